#!/bin/bash
# bench.py under env-var variants of the library (tuning knobs); one line per variant into gpurun_out/variants.txt:
#   config variant ms_per_step sample_ms/sweep apply_ms/sweep merge_ms/sweep roofline.frac LPTxKPL sparse_rows
# usage: bash tools/variants.sh CONFIG [extra bench args] ; variants from $VARIANTS (";"-separated "VAR=x VAR2=y")
mkdir -p gpurun_out
cfg=${1:-C3}; shift
IFS=';' read -ra VS <<< "${VARIANTS:-BASE=1}"
for v in "${VS[@]}"; do
  env $v timeout 300 python bench.py --config $cfg --no-cpu-baseline --largest "" --steps 30 --warmup 5 "$@" 2>/dev/null | tail -1 | \
    python -c "
import json,sys
d=json.loads(sys.stdin.read()); t=d['timings_ms']; n=max(t['sweeps'],1); st=d['stats']
print('$cfg', '$*', '$v', d['ms_per_step'], round(t['sample_ms']/n,4), round(t['apply_ms']/n,4), round(t['merge_ms']/n,4),
      d['roofline']['frac'], '%dx%d' % (st['lanes_per_token'], st['topics_per_lane']), 'sprows=%d/%d' % (st.get('sparse_rows',0), st.get('sparse_rows_lanes',0)))" >> gpurun_out/variants.txt || echo "$cfg $* $v FAILED" >> gpurun_out/variants.txt
done
