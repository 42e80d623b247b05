#!/bin/bash
# Round-2 final evidence, part A (GPU box): launch list + ncu full capture, ablations.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash tools/collect_profiles.sh > gpurun_out/collect.log 2>&1
timeout 1500 python tools/ablation.py r02 10 > gpurun_out/ablation.log 2>&1
cp profiles/r02_ablation.md gpurun_out/ 2>/dev/null
tail -14 gpurun_out/ablation.log
