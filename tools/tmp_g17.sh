python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g17_build.log 2>&1
rm -f gpurun_out/ab.txt gpurun_out/variants.txt
REPS=1 LIBS="varlibs/final.so varlibs/pg2.so varlibs/pg4.so" CONFIGS="C3;C3 --waves 2;C5" bash tools/ab_libs.sh
VARIANTS="SPDP_CHUNK_TOKENS=256;SPDP_CHUNK_TOKENS=512;SPDP_CHUNK_TOKENS=1024" bash tools/variants.sh C3
VARIANTS="SPDP_CHUNK_TOKENS=256;SPDP_CHUNK_TOKENS=1024" bash tools/variants.sh C5 --steps 10
cat gpurun_out/ab.txt gpurun_out/variants.txt
timeout 900 python bench.py --config C5 --largest "" --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_C5.json 2> gpurun_out/r2_bench_C5.err
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest_final.log 2>&1; tail -3 gpurun_out/r2_gputest_final.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; tail -2 gpurun_out/r2_smoke.log
