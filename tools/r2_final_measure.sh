#!/bin/bash
# Round-2 final measurement pass on one B200 (outputs under gpurun_out/; summaries copied to profiles/ by hand)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_final_build.log 2>&1
timeout 900 python bench.py > gpurun_out/r2_bench_C3.json 2> gpurun_out/r2_bench_C3.err
timeout 300 python tools/e2e_loop.py C3 50 > gpurun_out/r2_e2e_loop.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_C3.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --largest "" > /dev/null 2>&1
python tools/launch_shares.py gpurun_out/r2_launches_C3.csv gpurun_out/r2_launch_shares_C3.txt > /dev/null
bash tools/bench_matrix.sh > gpurun_out/r2_matrix.txt 2>&1
NCU_PREFIX=r2 bash tools/ncu_round2.sh C3 C5 C4K1000 C4K300 C4K100 C2 C4K20 C3W2
# (compute-sanitizer is closed on this GPU pool since round 2: tools/sanitize.sh is kept for pools that allow it)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest_final.log 2>&1; tail -3 gpurun_out/r2_gputest_final.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; tail -2 gpurun_out/r2_smoke.log
