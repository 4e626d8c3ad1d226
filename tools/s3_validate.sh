mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s3_build.log 2>&1
timeout 900 python bench.py > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s3_gputest.log 2>&1
tail -3 gpurun_out/s3_gputest.log
