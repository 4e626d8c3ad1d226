rm -f gpurun_out/ab.txt
REPS=1 LIBS="varlibs/v5.so varlibs/v9.so" CONFIGS="C3;C5;C3 --waves 2;C4 --topics 100;C4 --topics 300;C4 --topics 1000;C2;C4 --topics 20" bash tools/ab_libs.sh
cat gpurun_out/ab.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g7_gputest.log 2>&1; tail -3 gpurun_out/g7_gputest.log
