#!/bin/bash
# Round-2 GPU check: build, smoke, GPU tests, bench, launch list, one ncu full capture.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
bash tools/collect_profiles.sh > gpurun_out/collect.log 2>&1
tail -2 gpurun_out/smoke.log; tail -3 gpurun_out/gpu_tests.log; cat gpurun_out/bench.json
