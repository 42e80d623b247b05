"""Small compress + decompress steps for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck), one per kernel family: row-walking compressor + row-walking decoder (global and
chunk-local), z-band compressor + plane decoder, row-codes compressor (planes not whole tiles),
warp-specialized compressor + tile decoder (2-D), the f3 log transform, the device-parsed
asynchronous decode."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2304_12557_b200 import fz, synth

CASES = [
    ("nyx_v", (40, 32, 256), fz.REL),                    # k_compress_zr + k_dzr_*
    ("nyx_v", (32, 16, 256), fz.REL | fz.CHUNK_LOCAL),   # zr chunk-local + k_decode_cl
    ("sines3d", (33, 8, 512), fz.REL),                   # zr (ny % 16 != 0 -> zb) + plane decoder
    ("hurr_u", (12, 50, 52), fz.REL),                    # k_rowcodes + k_rowtiles, tile decoder
    ("cesm_t", (40, 300), fz.REL),                       # k_compress_ws (2-D)
    ("nyx_rho", (24, 32, 128), fz.PWREL),                # f3 log transform
    ("rtm", (256, 20, 96), fz.REL),                      # k_rowcodes + k_rowtiles, k_untile + k_dzg_*
]
for name, shape, mode in CASES:
    d = synth.generate(name, shape)
    x = torch.from_numpy(d).cuda()
    c = fz.Codec(shape, "cuda")
    buf, size = c.compress(x, mode, 1e-3)
    y = c.decompress(buf)
    z = c.decompress_device(buf) if not (mode & fz.CHUNK_LOCAL) else y
    if not (mode & fz.CHUNK_LOCAL):
        c.result()
    torch.cuda.synchronize()
    info = fz.peek_header(buf[:128].cpu().numpy().tobytes())
    if mode == fz.PWREL:
        err = float(((y.double() - x.double()).abs() / x.double().abs()).max())
        assert err <= 1e-3, (name, err)
    else:
        err = float((y.double() - x.double()).abs().max())
        assert err <= info.params.eb_abs, (name, err)
    assert torch.equal(y, z)
    print(name, shape, hex(mode), size, "ok", flush=True)
