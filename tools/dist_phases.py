import os, sys, time
sys.path.insert(0, "/root/repo")
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1"); os.environ.setdefault("LOCAL_RANK", "0")
import torch, torch.distributed as tdist, numpy as np
from paper_2304_12557_b200 import dist, fz, synth
import bench
dev = torch.device("cuda", 0); torch.cuda.set_device(dev)
tdist.init_process_group("nccl", device_id=dev)
field, shape, rel, _ = bench.WORKLOADS["c4"]
d = synth.generate(field, shape); flat = d.reshape(-1)
pl = dist.plan(shape, 1, 0)
slab = torch.from_numpy(np.ascontiguousarray(flat[pl.slab_first: pl.slab_hi])).to(dev)
comp = dist.SlabCompressor(shape, pl, dev)
E = fz.slab_agg_elems(shape); nloc = pl.own_hi - pl.own_lo
q = torch.empty(nloc, dtype=torch.int32, device=dev); agg = torch.empty(E, dtype=torch.int32, device=dev); carry = torch.empty(E, dtype=torch.int32, device=dev)
dwork = torch.empty(max(16, fz.decompress_workspace_bytes(shape)), dtype=torch.uint8, device=dev)
out = [None]
def step(T):
    def tick(name):
        torch.cuda.synchronize(); T.append((name, time.perf_counter()))
    tick("start")
    mn, mx = comp.local_range(slab); tick("range")
    gmn, gmx = dist.exchange_range(mn, mx, device=dev); tick("xrange")
    params = fz.derive_params(gmn, gmx, fz.REL, rel); tick("params")
    counts = comp.compress_local(slab, params); tick("compress")
    before_all, totals = dist.exchange_counts((counts.nnz, counts.n_delta, counts.n_value), device=dev); tick("xcounts")
    total = 128 + 32 * pl.tiles + 16 * totals[0] + 8 * totals[1] + 8 * totals[2]
    if out[0] is None: out[0] = torch.empty(total, dtype=torch.uint8, device=dev)
    comp.place(counts, before_all[0], totals, params, out[0]); tick("place")
    comp.decode_local(counts, q, agg, dwork); tick("decode")
    aggs = dist.exchange_planes(agg); tick("xplanes")
    fz.slab_carry(aggs, 0, E, carry); tick("carry")
    comp.finish(q, carry, counts, params); tick("finish")
for _ in range(3): step([])
T = []; step(T)
for (n0, t0), (n1, t1) in zip(T, T[1:]): print(f"{n1:10s} {1e3*(t1-t0):8.3f} ms")
tdist.destroy_process_group()
