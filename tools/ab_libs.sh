#!/bin/bash
# A/B of library builds on one box: bench.py per config under each SPDP_LIB; one line per (lib, config) into
# gpurun_out/ab.txt: lib config ms_per_step sample_ms/sweep apply_ms/sweep merge_ms/sweep
# usage: LIBS="a.so b.so" CONFIGS="C3;C5;C4 --topics 300" bash tools/ab_libs.sh
mkdir -p gpurun_out
IFS=';' read -ra CS <<< "${CONFIGS:-C3}"
for rep in $(seq ${REPS:-2}); do
for cfg in "${CS[@]}"; do
  for lib in $LIBS; do
    st=30; [[ "$cfg" == C5* ]] && st=10
    SPDP_LIB=$lib timeout 600 python bench.py --config $cfg --no-cpu-baseline --largest "" --steps $st --warmup 3 2>>gpurun_out/ab.err | tail -1 | \
      python -c "
import json,sys
d=json.loads(sys.stdin.read()); t=d['timings_ms']; n=max(t['sweeps'],1)
print('$lib', '$cfg', d['ms_per_step'], round(t['sample_ms']/n,4), round(t['apply_ms']/n,4), round(t['merge_ms']/n,4))" >> gpurun_out/ab.txt || echo "$lib $cfg FAILED" >> gpurun_out/ab.txt
  done
done
done
