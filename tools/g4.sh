rm -f gpurun_out/ab.txt
LIBS="varlibs/head.so varlibs/v4.so" CONFIGS="C3;C5" bash tools/ab_libs.sh
for sc in 0 1; do
  SPDP_DOC_SCATTER=$sc timeout 600 python bench.py --config C5 --no-cpu-baseline --largest "" --steps 10 --warmup 3 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['timings_ms']; n=t['sweeps']; print('C5 scatter=$sc', d['ms_per_step'], t['sample_ms']/n, t['apply_ms']/n)" >> gpurun_out/ab.txt
done
cat gpurun_out/ab.txt
timeout 900 python bench.py --largest "" > gpurun_out/g4_bench.json 2> gpurun_out/g4_bench.err
NCU_PREFIX=r3 bash tools/ncu_round2.sh C3 C5
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g4_gputest.log 2>&1; tail -3 gpurun_out/g4_gputest.log
