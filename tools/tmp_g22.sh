python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g22_build.log 2>&1
timeout 900 python bench.py > gpurun_out/r2_bench_C3.json 2> gpurun_out/r2_bench_C3.err
NCU_PREFIX=r2 bash tools/ncu_round2.sh C5
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest_final.log 2>&1; tail -3 gpurun_out/r2_gputest_final.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; tail -2 gpurun_out/r2_smoke.log
