#!/bin/bash
# Round-2 validation on one B200: the whole GPU suite (incl. slow), smoke, compute-sanitizer matrix
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_gputest_final.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
bash tools/sanitize.sh
