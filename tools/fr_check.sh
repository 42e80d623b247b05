mkdir -p gpurun_out
for e in 0 0; do FZ_EXP=$e timeout 120 python tools/time_compress.py child c4 >> gpurun_out/cp_time.log 2>&1; done
FZ_EXP=0 timeout 120 python tools/time_compress.py child c5 >> gpurun_out/cp_time.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused_range.py -q -x > gpurun_out/cp_tests.log 2>&1
cat gpurun_out/cp_time.log; tail -2 gpurun_out/cp_tests.log
