"""Per-launch timeline of one compress + decompress step (CUDA events), showing the gaps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2304_12557_b200 import fz, synth
import bench
wl = sys.argv[1] if len(sys.argv) > 1 else "c4"
field, shape, rel, _ = bench.WORKLOADS[wl]
d = synth.generate(field, shape)
x = torch.from_numpy(d).cuda()
c = fz.Codec(shape, "cuda")
out = torch.empty_like(x)
for _ in range(3):
    buf, size = c.compress(x, fz.REL, rel)
    c.decompress(buf, out=out)
torch.cuda.synchronize()
fz.profile_enable(True)
fz.profile_read()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
buf, size = c.compress(x, fz.REL, rel)
c.decompress(buf, out=out)
e1.record()
torch.cuda.synchronize()
tl = fz.profile_timeline()
print(f"step {e0.elapsed_time(e1)*1e3:.1f} us")
prev = 0.0
for name, a, b in tl:
    print(f"{name:18s} start {a*1e3:8.1f} end {b*1e3:8.1f} dur {(b-a)*1e3:7.1f} gap_before {(a-prev)*1e3:6.1f}")
    prev = b
fz.profile_read()
