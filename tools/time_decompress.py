"""Times the decode kernels of one workload (CUDA-event profiling) under several env settings:
  python tools/time_decompress.py c4 "FZ_YS=8 FZ_ZC=16" "FZ_EXP=2048" ..."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch
    import numpy as np
    from paper_2304_12557_b200 import fz, synth
    import bench
    wl = sys.argv[2]
    field, shape, rel, _ = bench.WORKLOADS[wl]
    cache = f"/tmp/field_{wl}.npy"
    d = np.load(cache) if os.path.exists(cache) else synth.generate(field, shape)
    if not os.path.exists(cache):
        np.save(cache, d)
    fz.debug_set_variant(int(os.environ.get("FZ_EXP", "0")))
    x = torch.from_numpy(d).cuda()
    c = fz.Codec(shape, "cuda")
    buf, size = c.compress(x, fz.REL, rel)
    out = torch.empty_like(x)
    for _ in range(3):
        c.decompress(buf, out=out)
    fz.profile_enable(True); fz.profile_read()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(10):
        c.decompress(buf, out=out)
    s1.record(); torch.cuda.synchronize()
    p = fz.profile_read()
    ok = torch.equal(out, c.decompress(buf))
    ks = " ".join(f"{k} {ms / n * 1000:.1f}" for k, (ms, n) in p.items() if ms / n > 0.002)
    print(f"[{os.environ.get('TAG', '')}] wall/decompress {s0.elapsed_time(s1) / 10 * 1000:.1f} us | {ks}")
else:
    wl = sys.argv[1]
    for cfg in sys.argv[2:] or [""]:
        env = dict(os.environ, TAG=cfg)
        for kv in cfg.split():
            k, v = kv.split("=")
            env[k] = v
        subprocess.run([sys.executable, __file__, "child", wl], env=env)
