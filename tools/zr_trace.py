"""Per-CTA residency trace of the row walker (variant 8388608): start / range-phase end / end
per CTA from globaltimer, for the fused and the separate-range compressor."""
import os, sys, ctypes as C, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2304_12557_b200 import fz, synth
import bench
field, shape, rel, _ = bench.WORKLOADS["c4"]
d = synth.generate(field, shape)
x = torch.from_numpy(d).cuda()
c = fz.Codec(shape, "cuda")
lib = fz.lib()
for extra in [int(v) for v in sys.argv[1:]] or [0, 2097152]:
    fz.debug_set_variant(8388608 | extra)
    for _ in range(3):
        c.compress(x, fz.REL, rel)
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * (4 * 2048))()
    lib.fz_debug_zr_trace(buf, 4 * 2048)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 4)[:444].astype(np.int64)
    t0 = a[:, 0].min()
    st = (a[:, 0] - t0) / 1000.0
    en = (a[:, 3] - t0) / 1000.0
    early = st < 3.0
    per_sm = collections.Counter(collections.Counter(a[early, 1]).values())
    msg = f"variant {extra}: early CTAs {early.sum()} (per SM {dict(per_sm)}), start q {np.round(np.percentile(st, [50, 90, 100]), 1)}, end q {np.round(np.percentile(en, [0, 50, 100]), 1)}"
    if not (extra & 2097152):
        rr = (a[:, 2] - t0) / 1000.0
        msg += f", range end q {np.round(np.percentile(rr, [0, 50, 100]), 1)}"
    print(msg, flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    np.save(f"gpurun_out/zr_trace_{extra}.npy", a)
fz.debug_set_variant(0)
