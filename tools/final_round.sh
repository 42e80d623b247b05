set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
bash tools/collect_profiles.sh > gpurun_out/collect.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_compress_zb|k_decode_cl|k_compact" -s 4 -c 3 -o gpurun_out/full_cl python tools/prof_step.py --steps 2 > gpurun_out/full_cl.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
tail -2 gpurun_out/smoke.log; tail -3 gpurun_out/gpu_tests.log; cat gpurun_out/bench.json
