for v in "varlibs/v9.so:1" "varlibs/v10.so:1" "varlibs/v10.so:0"; do
  lib=${v%%:*}; pool=${v#*:}
  echo "== $lib pool=$pool" >> gpurun_out/g9_load.txt
  SPDP_LIB=$lib SPDP_TEMP_POOL=$pool SPDP_VERBOSE=2 timeout 300 python tools/load_phases.py C3 >> gpurun_out/g9_load.txt 2>&1
done
cat gpurun_out/g9_load.txt
rm -f gpurun_out/variants.txt
VARIANTS="BASE=1;SPDP_DOC_SCATTER=0;SPDP_PREFETCH_ROWS=0;SPDP_DOC_SCATTER=0 SPDP_PREFETCH_ROWS=0" bash tools/variants.sh C5 --steps 10
cat gpurun_out/variants.txt
timeout 600 python -m pytest tests/test_gpu_validation.py -q > gpurun_out/g9_valtest.log 2>&1; tail -3 gpurun_out/g9_valtest.log
