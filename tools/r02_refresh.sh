#!/bin/bash
# Round-2 evidence refresh on the GPU box: tests, smoke, bench (+ reference arm), launch list,
# ncu full capture, ablations.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
bash tools/collect_profiles.sh > gpurun_out/collect.log 2>&1
timeout 1200 python tools/ablation.py r02 5 > gpurun_out/ablation.log 2>&1
cp profiles/r02_ablation.md gpurun_out/ 2>/dev/null
tail -2 gpurun_out/smoke.log; tail -3 gpurun_out/gpu_tests.log; tail -3 gpurun_out/bench.err; tail -12 gpurun_out/ablation.log
