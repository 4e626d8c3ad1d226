rm -f gpurun_out/ab.txt
REPS=1 LIBS="varlibs/v5.so varlibs/v8.so varlibs/v8f4.so varlibs/v8f5.so varlibs/v8f6.so" CONFIGS="C3;C5;C3 --waves 2;C4 --topics 300;C4 --topics 1000" bash tools/ab_libs.sh
cat gpurun_out/ab.txt
