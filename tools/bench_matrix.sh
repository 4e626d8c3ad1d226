#!/bin/bash
# Runs bench.py over the BASELINE configs on one GPU; JSON lines into gpurun_out/matrix.jsonl
mkdir -p gpurun_out
out=gpurun_out/matrix.jsonl
: > $out
run() { timeout 900 python bench.py --no-cpu-baseline --largest "" "$@" 2>>gpurun_out/matrix.err | tail -1 >> $out; tail -1 $out | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['ms_per_step'], '%.3g'%d['value'], d['roofline']['frac'], d['stats']['lanes_per_token'], d['stats']['topics_per_lane'])" || echo "FAILED $@"; }
run --config C2 --steps 100
for K in 20 100 300 1000; do run --config C4 --topics $K --steps 30; done
for W in 2 4 8; do run --config C3 --waves $W --steps 20; done
run --config C5 --steps 10 --warmup 3
