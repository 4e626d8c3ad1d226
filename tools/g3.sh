rm -f gpurun_out/ab.txt
LIBS="varlibs/head.so varlibs/v3.so" CONFIGS="C3;C5;C2;C4 --topics 20;C4 --topics 300;C3 --waves 2" bash tools/ab_libs.sh
cat gpurun_out/ab.txt
for pool in 0 1; do
  SPDP_TEMP_POOL=$pool SPDP_VERBOSE=2 timeout 300 python tools/e2e_breakdown.py C3 20 > gpurun_out/g3_e2e_pool$pool.txt 2>&1
done
SPDP_LIB=varlibs/head.so SPDP_VERBOSE=2 timeout 300 python tools/e2e_breakdown.py C3 20 > gpurun_out/g3_e2e_head.txt 2>&1
timeout 900 python bench.py > gpurun_out/g3_bench.json 2> gpurun_out/g3_bench.err
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g3_gputest.log 2>&1; tail -3 gpurun_out/g3_gputest.log
