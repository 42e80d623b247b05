#!/bin/bash
# Round-2 final evidence, part B (GPU box): smoke, GPU tests, bench (all configs + oracle parity),
# the reference arm.  Part A (tools/r02_refresh_a.sh) captures the profiles first so that
# bench.py's roofline.traffic reads the current ncu numbers (profiles/ncu_traffic.json).
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
tail -2 gpurun_out/smoke.log; tail -3 gpurun_out/gpu_tests.log; tail -3 gpurun_out/bench.err
