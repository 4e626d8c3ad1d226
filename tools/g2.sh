rm -f gpurun_out/ab.txt
LIBS="varlibs/head.so varlibs/unit.so" CONFIGS="C3;C5;C4 --topics 300;C4 --topics 1000;C3 --waves 2" bash tools/ab_libs.sh
cat gpurun_out/ab.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g2_gputest.log 2>&1; tail -3 gpurun_out/g2_gputest.log
