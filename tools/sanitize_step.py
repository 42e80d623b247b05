"""Small compress + decompress steps for compute-sanitizer (racecheck / memcheck / synccheck):
z-band compressor (global and chunk-local), plane decoder, chunk-local decoder, tile decoder."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2304_12557_b200 import fz, synth

for name, shape, mode in [("sines3d", (33, 8, 512), fz.REL), ("nyx_v", (20, 16, 256), fz.REL | fz.CHUNK_LOCAL),
                          ("hurr_u", (160, 8, 256), fz.REL), ("cesm_t", (40, 300), fz.REL)]:
    d = synth.generate(name, shape)
    x = torch.from_numpy(d).cuda()
    c = fz.Codec(shape, "cuda")
    buf, size = c.compress(x, mode, 1e-3)
    y = c.decompress(buf)
    torch.cuda.synchronize()
    info = fz.peek_header(buf[:128].cpu().numpy().tobytes())
    err = float((y.double() - x.double()).abs().max())
    assert err <= info.params.eb_abs, (name, err)
    print(name, shape, hex(mode), size, "ok", flush=True)
