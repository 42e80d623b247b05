"""Profiling driver: N compress+decompress steps of one workload (used under ncu)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2304_12557_b200 import fz, synth
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c4")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--no-decompress", action="store_true")
a = ap.parse_args()
field, shape, rel, _ = bench.WORKLOADS[a.workload]
d = synth.generate(field, shape)
x = torch.from_numpy(d).cuda()
c = fz.Codec(shape, "cuda")
out = torch.empty_like(x)
for _ in range(a.steps):
    buf, size = c.compress(x, fz.REL, rel)
    if not a.no_decompress:
        c.decompress(buf, out=out)
torch.cuda.synchronize()
print("size", size, "CR", d.nbytes / size)
