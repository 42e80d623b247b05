"""Launch timeline of one single-process slab round trip (the multi-GPU protocol, 1 rank)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2304_12557_b200 import fz, synth, dist
import bench
field, shape, rel, _ = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
ranks = int(sys.argv[2]) if len(sys.argv) > 2 else 1
d = synth.generate(field, shape)
for _ in range(2):
    dist.roundtrip_sharded_single_process(d, fz.REL, rel, ranks)
torch.cuda.synchronize()
fz.profile_enable(True)
fz.profile_read()
dist.roundtrip_sharded_single_process(d, fz.REL, rel, ranks)
torch.cuda.synchronize()
prev = 0.0
for name, a, b in fz.profile_timeline():
    print(f"{name:18s} start {a*1e3:9.1f} dur {(b-a)*1e3:8.1f} gap {(a-prev)*1e3:8.1f}")
    prev = b
fz.profile_read()
