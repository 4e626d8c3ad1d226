#!/bin/bash
# Round-2 measurement pass on one B200 (outputs under gpurun_out/, summaries copied to profiles/ by hand)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 900 python bench.py > gpurun_out/r2_bench_C3.json 2> gpurun_out/r2_bench_C3.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r2_bench_reference.json 2>>gpurun_out/r2_bench_C3.err
# N > 1 code path end to end on one GPU (functional, not a measurement): 2 ranks over the NCCL shim
gcc -O2 -shared -fPIC -I/usr/local/cuda/include tests/nccl_shim.c -o tests/libnccl_shim.so -L/usr/local/cuda/lib64 \
    -Wl,-rpath,/usr/local/cuda/lib64 -lcudart
SPDP_NCCL_LIB=$PWD/tests/libnccl_shim.so SPDP_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 \
    --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --config C2 --largest C3 \
    --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_shim2.json 2> gpurun_out/r2_bench_shim2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_C3.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --largest "" > /dev/null 2>&1
python tools/launch_shares.py gpurun_out/r2_launches_C3.csv gpurun_out/r2_launch_shares_C3.txt > /dev/null
bash tools/ncu_round2.sh C3 C5 C4K1000 C4K300 C4K100 C2 C4K20
bash tools/bench_matrix.sh > gpurun_out/r2_matrix.txt 2>&1
