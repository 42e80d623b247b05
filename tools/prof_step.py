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
ap.add_argument("--no-chunk-local", action="store_true", help="skip the f1 chunk-local steps")
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
if not a.no_chunk_local and len(shape) == 3:
    for _ in range(a.steps):   # f1 chunk-local mode: z-band compressor + one-pass chunk decoder
        buf, size = c.compress(x, fz.REL | fz.CHUNK_LOCAL, rel)
        if not a.no_decompress:
            c.decompress(buf, out=out)
    torch.cuda.synchronize()
    print("chunk-local size", size, "CR", d.nbytes / size)
