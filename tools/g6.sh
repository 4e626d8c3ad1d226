rm -f gpurun_out/ab.txt
REPS=1 LIBS="varlibs/v5.so varlibs/v8.so varlibs/v8f4.so varlibs/v8f5.so varlibs/v8f6.so" CONFIGS="C3;C5;C3 --waves 2;C4 --topics 300;C4 --topics 1000" bash tools/ab_libs.sh
cat gpurun_out/ab.txt
timeout 900 python bench.py --largest "" > gpurun_out/g6_bench.json 2> gpurun_out/g6_bench.err
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g6_gputest.log 2>&1; tail -3 gpurun_out/g6_gputest.log
