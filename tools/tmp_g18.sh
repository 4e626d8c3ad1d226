python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g18_build.log 2>&1
rm -f gpurun_out/ab.txt
REPS=1 LIBS="varlibs/final.so varlibs/pg4.so" CONFIGS="C4 --topics 100;C4 --topics 300;C4 --topics 1000;C3 --waves 4;C2" bash tools/ab_libs.sh
cat gpurun_out/ab.txt
timeout 900 python bench.py > gpurun_out/r2_bench_C3.json 2> gpurun_out/r2_bench_C3.err
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest_final.log 2>&1; tail -3 gpurun_out/r2_gputest_final.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; tail -2 gpurun_out/r2_smoke.log
