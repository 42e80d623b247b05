mkdir -p gpurun_out
for e in 0 67108864 0 67108864; do
  FZ_EXP=$e timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-configs > gpurun_out/pdl_bench_$e.json 2> gpurun_out/pdl_bench_$e.err
  python -c "import json,sys; d=json.load(open('gpurun_out/pdl_bench_$e.json')); print('$e', d['value'], d['ms_per_step'], d['value_stream_launch'], d['compress_gbs'], d['decompress_gbs'], d['parity_vs_oracle'] if 'parity_vs_oracle' in d else '')" >> gpurun_out/pdl.log 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1
cat gpurun_out/pdl.log; tail -3 gpurun_out/gpu_tests.log; tail -3 gpurun_out/pdl_bench_0.err
