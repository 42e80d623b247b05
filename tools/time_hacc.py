import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2304_12557_b200 import fz, synth
d = synth.generate("hacc_x")
x = torch.from_numpy(d).cuda()
c = fz.Codec(d.shape, "cuda")
out = torch.empty_like(x)
for _ in range(3):
    buf, size = c.compress(x, fz.PWREL, 1e-3); c.decompress(buf, out=out)
fz.profile_enable(True); fz.profile_read()
for _ in range(5):
    buf, size = c.compress(x, fz.PWREL, 1e-3); c.decompress(buf, out=out)
torch.cuda.synchronize()
p = fz.profile_read()
print("hacc", {k: round(ms / n * 1000, 1) for k, (ms, n) in p.items()})
