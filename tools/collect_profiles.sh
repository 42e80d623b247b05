#!/bin/bash
# Run on the GPU box (gpurun): launch list of the bench command + one ncu --set full capture.
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-configs > gpurun_out/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_compress|k_compact|k_decode|k_scan_walk|k_range|k_nnz|k_record|k_dzr|k_rowcodes|k_rowtiles" -s 10 -c 16 \
    -o gpurun_out/full python tools/prof_step.py --steps 4 > gpurun_out/full.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt
