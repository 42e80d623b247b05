#!/bin/bash
# A/B of the headline step: bench.py --no-configs --no-cpu-baseline alternating FZ_EXP values.
# usage: bash tools/ab_bench.sh "0 2097152" [rounds] [steps]
mkdir -p gpurun_out
V=${1:-"0 2097152"}; R=${2:-3}; S=${3:-20}
for r in $(seq $R); do for e in $V; do
  FZ_EXP=$e timeout 600 python bench.py --steps $S --warmup 5 --no-cpu-baseline --no-configs > gpurun_out/ab_$e.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_$e.json')); print('FZ_EXP=$e', d['value'], d['ms_per_step'], d['value_stream_launch'], d['compress_gbs'], d['decompress_gbs'])"
done; done
