#!/bin/bash
# bench.py under env-var variants of the library (tuning knobs); one line per variant into gpurun_out/variants.txt
# usage: bash tools/variants.sh CONFIG [extra bench args] ; variants from $VARIANTS (";"-separated "VAR=x VAR2=y")
mkdir -p gpurun_out
cfg=${1:-C3}; shift
IFS=';' read -ra VS <<< "${VARIANTS:-BASE=1}"
for v in "${VS[@]}"; do
  env $v timeout 300 python bench.py --config $cfg --no-cpu-baseline --steps 30 --warmup 5 "$@" 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timings_ms']; print('$cfg', '$v', d['ms_per_step'], round(t['sample_ms']/t['sample_launches'],4), d['roofline']['frac'], d['stats']['lanes_per_token'], d['stats']['topics_per_lane'])" >> gpurun_out/variants.txt || echo "$cfg $v FAILED" >> gpurun_out/variants.txt
done
