#!/bin/bash
# GPU check: f4 link test, single-GPU bench (all configs), functional 2-rank bench (gloo, one GPU)
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_link.py tests/test_gpu_logt.py -q -x > gpurun_out/t_link.log 2>&1
timeout 900 python bench.py > gpurun_out/bench4.json 2> gpurun_out/bench4.err
FZ_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-configs > gpurun_out/dist2.json 2> gpurun_out/dist2.err
tail -3 gpurun_out/t_link.log; tail -3 gpurun_out/bench4.err; tail -5 gpurun_out/dist2.err; cat gpurun_out/dist2.json
