#!/bin/bash
# compute-sanitizer (memcheck, racecheck, initcheck) over every sample-kernel variant on C1 / C2
# (SURVEY §5 race detection).  One summary line per (tool, variant) into gpurun_out/r2_sanitizer.txt;
# full logs under gpurun_out/sanit/.
mkdir -p gpurun_out/sanit
out=gpurun_out/r2_sanitizer.txt
: > $out
run() {  # name env... -- args
  local name=$1; shift
  local envs=()
  while [ "$1" != "--" ]; do envs+=("$1"); shift; done; shift
  for tool in memcheck racecheck initcheck; do
    local log=gpurun_out/sanit/${name}_${tool}.log
    env "${envs[@]}" timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
        python tools/prof_sweeps.py --sweeps 2 "$@" > $log 2>&1
    echo "$name $tool rc=$? $(grep -m1 'ERROR SUMMARY' $log)" >> $out
  done
}
run C1_K10_token X=1 -- --config C1
run C1_K100_chunk X=1 -- --config C1 --topics 100
run C1_K100_W3 X=1 -- --config C1 --topics 100 --waves 3
run C1_K10_W4_token X=1 -- --config C1 --waves 4
run C1_K200_row8 SPDP_ROW_BYTES=1 SPDP_PREFETCH_ROWS=1 -- --config C1 --topics 200
run C1_K300_row16 SPDP_ROW_BYTES=2 SPDP_PREFETCH_ROWS=1 -- --config C1 --topics 300
run C1_K1000 X=1 -- --config C1 --topics 1000
run C1_K50_async X=1 -- --config C1 --topics 50 --update async
run C1_K10_seq X=1 -- --config C1 --waves 0
run C1_K10_sparseP X=1 -- --config C1 --transform mix
run C1_K100_chunk64 SPDP_CHUNK_TOKENS=64 -- --config C1 --topics 100
run C2_K50 X=1 -- --config C2
run C1_K200_row8_scatter SPDP_ROW_BYTES=1 SPDP_PREFETCH_ROWS=1 SPDP_DOC_SCATTER=1 -- --config C1 --topics 200
run C1_K200_sprows SPDP_SPARSE_ROWS=1 -- --config C1 --topics 200
run C1_K100_chunkft SPDP_CHUNK_FACTORS=1 -- --config C1 --topics 100
