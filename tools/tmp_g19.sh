rm -f gpurun_out/ab.txt
REPS=2 LIBS="varlibs/pg4.so varlibs/pg8.so" CONFIGS="C4 --topics 300;C4 --topics 1000" bash tools/ab_libs.sh
cat gpurun_out/ab.txt
timeout 600 python bench.py --config C4 --topics 1000 --largest "" --steps 20 --no-cpu-baseline > gpurun_out/g19_k1000.json 2>/dev/null
