"""Times k_compress alone (CUDA-event profiling) for a workload; FZ_EXP=16 selects the generic
kernel instead of the warp-specialized one.  AS2D=1 reshapes the field to 2-D."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch
    import numpy as np
    from paper_2304_12557_b200 import fz, synth
    import bench
    wl = sys.argv[2] if len(sys.argv) > 2 else "c4"
    field, shape, rel, _ = bench.WORKLOADS[wl]
    cache = f"/tmp/field_{wl}.npy"
    d = np.load(cache) if os.path.exists(cache) else synth.generate(field, shape)
    if not os.path.exists(cache):
        np.save(cache, d)
    if os.environ.get("AS2D"):
        d = d.reshape(-1, shape[-1])
        shape = d.shape
    fz.debug_set_variant(int(os.environ.get("FZ_EXP", "0")))
    x = torch.from_numpy(d).cuda()
    c = fz.Codec(shape, "cuda")
    for _ in range(3):
        c.compress(x, fz.REL, rel)
    fz.profile_enable(True); fz.profile_read()
    for _ in range(10):
        c.compress(x, fz.REL, rel)
    p = fz.profile_read()
    ks = " ".join(f"{name} {ms / k * 1000:.1f}" for name, (ms, k) in p.items() if ms / k > 0.002)
    print(f"[{wl}] FZ_EXP={os.environ.get('FZ_EXP','0')} us/launch: {ks}")
else:
    for e in sys.argv[1:] or ["0", "16"]:
        env = dict(os.environ, FZ_EXP=e)
        subprocess.run([sys.executable, __file__, "child"], env=env)
