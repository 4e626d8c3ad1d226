rm -f gpurun_out/g10_load.txt
for v in varlibs/v9.so varlibs/v10.so varlibs/v9.so varlibs/v10.so varlibs/v11.so; do
  echo "== $v" >> gpurun_out/g10_load.txt
  SPDP_LIB=$v SPDP_VERBOSE=2 timeout 300 python tools/load_phases.py C3 >> gpurun_out/g10_load.txt 2>&1
done
cat gpurun_out/g10_load.txt | grep -v "positions\|Stirling"
