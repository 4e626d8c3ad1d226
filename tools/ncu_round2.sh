#!/bin/bash
# ncu --set full captures of the sample kernel on the HBM-bound and the bench configurations (round 2).
# Each report is summarised on the box (tools/ncu_summary.py -> JSON, tools/ncu_source_top.py -> top
# stall lines) and deleted unless KEEP_REP=1 (gpurun brings back <= 64 MiB).
mkdir -p gpurun_out
cap() {  # tag kernel-regex args...
  local tag=$1 kre=$2; shift 2
  local rep=/tmp/${NCU_PREFIX:-r2}_ncu_$tag
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -s 2 -c 1 \
    -o $rep -f python tools/prof_sweeps.py --sweeps 3 "$@" > gpurun_out/${NCU_PREFIX:-r2}_ncu_$tag.log 2>&1 \
    || echo "ncu $tag failed" >> gpurun_out/${NCU_PREFIX:-r2}_ncu_failures.txt
  python tools/ncu_summary.py $rep.ncu-rep gpurun_out/${NCU_PREFIX:-r2}_ncu_$tag.json > /dev/null 2>>gpurun_out/${NCU_PREFIX:-r2}_ncu_$tag.log
  python tools/ncu_source_top.py $rep.ncu-rep 50 > gpurun_out/${NCU_PREFIX:-r2}_ncu_${tag}_src.txt 2>>gpurun_out/${NCU_PREFIX:-r2}_ncu_$tag.log
  if [ "$KEEP_REP" = "1" ]; then cp $rep.ncu-rep gpurun_out/; fi
}
for spec in "$@"; do
  case $spec in
    C5) cap C5_K200_sample sample_kernel --config C5 ;;
    C4K1000) cap C4_K1000_sample sample_kernel --config C4 --topics 1000 ;;
    C4K300) cap C4_K300_sample sample_kernel --config C4 --topics 300 ;;
    C4K100) cap C4_K100_sample sample_kernel --config C4 --topics 100 ;;
    C4K20) cap C4_K20_token token_kernel --config C4 --topics 20 ;;
    C3) cap C3_K100_sample sample_kernel --config C3 ;;
    C3W2) cap C3_K100_W2_sample sample_kernel --config C3 --waves 2 ;;
    C2) cap C2_K50_token token_kernel --config C2 ;;
  esac
done
