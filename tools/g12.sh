python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g12_build.log 2>&1
rm -f gpurun_out/variants.txt
VARIANTS="SPDP_RECOUNT_LPD=32;SPDP_RECOUNT_LPD=16" bash tools/variants.sh C5 --steps 10
VARIANTS="SPDP_RECOUNT_LPD=32;SPDP_RECOUNT_LPD=16" bash tools/variants.sh C3
cat gpurun_out/variants.txt
timeout 1200 python -m pytest tests/test_gpu_paths.py tests/test_gpu_validation.py -x -q > gpurun_out/g12_tests.log 2>&1; tail -3 gpurun_out/g12_tests.log
