"""Multi-GPU bench path (torchrun, one process per GPU, NCCL): z-slab partitioned compress +
decompress of one global field.  Called by bench.py when WORLD_SIZE > 1.

Per rank and step:
  fz_slab_range -> all_gather(min, max) -> parameters -> fz_slab_compress -> all_gather(counts)
  -> fz_slab_place (the rank's share at its global offsets) -> fz_slab_decode ->
  all_gather(aggregate planes) -> fz_slab_carry -> fz_slab_finish.
Timing: barrier + device sync on both sides, CUDA events per step, max over ranks.
"""
from __future__ import annotations

import json
import os
import statistics

import numpy as np


def _clock_sampler(index: int):
    """bench.py's NVML sampler (SM clock + throttle reasons during the timed region)."""
    import importlib
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if root not in sys.path:
        sys.path.insert(0, root)
    return importlib.import_module("bench").ClockSampler(index)


def _peak():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


def run(args, wl, metric):
    import torch
    import torch.distributed as tdist

    from . import dist, fz, synth

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # FZ_DIST_BACKEND=gloo: a functional check of the multi-rank path with several ranks
    # sharing one GPU (collectives through host memory); the bench itself runs NCCL.
    backend = os.environ.get("FZ_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if backend == "nccl":
        tdist.init_process_group("nccl", device_id=dev)
    else:
        tdist.init_process_group(backend)
    xdev = dev if backend == "nccl" else torch.device("cpu")
    field_name, shape, rel, desc = wl
    d = synth.generate(field_name, shape)
    flat = d.reshape(-1)
    pl = dist.plan(shape, world, rank)
    # every rank needs a nonempty tile range (fz_slab_compress rejects an empty one, and a
    # rank that skipped the all_gathers would hang the others)
    nslabs = shape[0] if len(shape) == 3 else -(-int(np.prod(shape)) // 2048)
    if world > nslabs or pl.te <= pl.tb:
        raise SystemExit(f"bench_dist: {world} ranks but only {nslabs} slabs in {shape}")
    slab = torch.from_numpy(np.ascontiguousarray(flat[pl.slab_first: pl.slab_hi])).to(dev)
    comp = dist.SlabCompressor(shape, pl, dev)
    E = fz.slab_agg_elems(shape)
    nloc = pl.own_hi - pl.own_lo
    q = torch.empty(max(nloc, 4), dtype=torch.int32, device=dev)
    agg = torch.empty(E, dtype=torch.int32, device=dev)
    carry = torch.empty(E, dtype=torch.int32, device=dev)
    local_dims = (nloc // E,) + tuple(shape[1:]) if len(shape) > 1 else (nloc,)
    dwork = torch.empty(max(16, fz.decompress_workspace_bytes(local_dims)), dtype=torch.uint8, device=dev)
    out = None
    launches = [0]
    last_params = [None]

    coll = []   # CUDA-event pairs around the three exchange steps of the timed steps

    def timed(fn, *a, **k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = fn(*a, **k)
        e1.record()
        coll.append((e0, e1))
        return r

    def step():
        nonlocal out
        mn, mx = comp.local_range(slab)
        launches[0] += fz.last_launch_count()
        gmn, gmx = timed(dist.exchange_range, mn, mx, device=xdev)
        params = fz.derive_params(gmn, gmx, fz.REL, rel)
        last_params[0] = params
        counts = comp.compress_local(slab, params)
        launches[0] += fz.last_launch_count()
        before_all, totals = timed(dist.exchange_counts, (counts.nnz, counts.n_delta, counts.n_value), device=xdev)
        before = before_all[rank]
        total = 128 + 32 * pl.tiles + 16 * totals[0] + 8 * totals[1] + 8 * totals[2]
        if out is None or out.numel() < total:
            out = torch.empty(total, dtype=torch.uint8, device=dev)
        comp.place(counts, before, totals, params, out)
        comp.decode_local(counts, q, agg, dwork)
        launches[0] += fz.last_launch_count()
        aggs = timed(dist.exchange_planes, agg.to(xdev)).to(dev)
        fz.slab_carry(aggs, rank, E, carry)
        launches[0] += fz.last_launch_count()
        comp.finish(q, carry, counts, params)
        launches[0] += fz.last_launch_count()
        return total

    # warm-up mirrors the timed loop (barriers included: the first NCCL barrier is expensive)
    for _ in range(max(3, args.warmup)):
        tdist.barrier()
        torch.cuda.synchronize()
        total = step()
        torch.cuda.synchronize()
        tdist.barrier()
    torch.cuda.synchronize()
    times = []
    launches[0] = 0
    sampler = _clock_sampler(local)
    # per-kernel CUDA-event times of this rank's launches (the roofline of the compressor)
    fz.profile_enable(True)
    fz.profile_only(["k_range", "k_compress", "k_decode_tiles", "k_scan_walk", "k_scan_apply"])
    fz.profile_read()
    with sampler:
        for _ in range(args.steps):
            tdist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            total = step()
            e1.record()
            torch.cuda.synchronize()
            tdist.barrier()
            times.append(e0.elapsed_time(e1))
    prof = fz.profile_read()
    fz.profile_enable(False)
    if os.environ.get("FZ_DIST_DEBUG"):
        print(f"rank {rank} step ms {[round(x, 3) for x in times]}", flush=True)
    t = torch.tensor([statistics.mean(times)], dtype=torch.float64, device=xdev)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms = float(t.item())
    # time inside the three exchange steps (range, counts, carry planes), max over ranks
    nc = 3 * args.steps
    ct = torch.tensor([sum(a.elapsed_time(b) for a, b in coll[-nc:]) / max(1, args.steps)], dtype=torch.float64,
                      device=xdev)
    tdist.all_reduce(ct, op=tdist.ReduceOp.MAX)
    coll_ms = float(ct.item())

    # ---- end to end through the slab API with host buffers: per rank and step, H2D of the
    # slab (own + halo) from pinned memory, compress, D2H of the rank's compressed share (its
    # stage: flags, payload, outlier records), H2D of that share back, decode, D2H of the
    # decoded slab.  Bytes are summed over ranks.
    h_slab = torch.from_numpy(np.ascontiguousarray(flat[pl.slab_first: pl.slab_hi])).pin_memory()
    h_stage = torch.empty(comp.stage.numel(), dtype=torch.uint8).pin_memory()
    h_out = torch.empty(max(nloc, 1), dtype=torch.float32).pin_memory()
    io = [0, 0]

    def step_e2e():
        slab.copy_(h_slab, non_blocking=True)
        mn, mx = comp.local_range(slab)
        gmn, gmx = dist.exchange_range(mn, mx, device=xdev)
        params = fz.derive_params(gmn, gmx, fz.REL, rel)
        counts = comp.compress_local(slab, params)
        before_all, totals = dist.exchange_counts((counts.nnz, counts.n_delta, counts.n_value), device=xdev)
        total = 128 + 32 * pl.tiles + 16 * totals[0] + 8 * totals[1] + 8 * totals[2]
        comp.place(counts, before_all[rank], totals, params, out)
        sb = 32 * (pl.te - pl.tb) + 16 * counts.nnz + 8 * counts.n_delta + 8 * counts.n_value
        h_stage[:sb].copy_(comp.stage[:sb], non_blocking=True)
        comp.stage[:sb].copy_(h_stage[:sb], non_blocking=True)
        comp.decode_local(counts, q, agg, dwork)
        aggs = dist.exchange_planes(agg.to(xdev)).to(dev)
        fz.slab_carry(aggs, rank, E, carry)
        comp.finish(q, carry, counts, params)
        h_out[:nloc].copy_(q[:nloc].view(torch.float32), non_blocking=True)
        io[0] = 4 * slab.numel() + sb
        io[1] = sb + 4 * nloc
        return total

    for _ in range(max(3, args.warmup)):
        tdist.barrier()
        step_e2e()
        torch.cuda.synchronize()
    tdist.barrier()
    torch.cuda.synchronize()
    etimes = []
    for _ in range(args.steps):
        tdist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step_e2e()
        e1.record()
        torch.cuda.synchronize()
        tdist.barrier()
        etimes.append(e0.elapsed_time(e1))
    et = torch.tensor([statistics.mean(etimes)], dtype=torch.float64, device=xdev)
    tdist.all_reduce(et, op=tdist.ReduceOp.MAX)
    ebytes = torch.tensor([float(io[0]), float(io[1])], dtype=torch.float64, device=xdev)
    tdist.all_reduce(ebytes, op=tdist.ReduceOp.SUM)
    ems = float(et.item())
    # correctness spot check against the 1-GPU decode of the same stream: every rank's
    # decompressed slab must be within eb of its input
    xh = q[:nloc].view(torch.float32)
    ref = torch.from_numpy(np.ascontiguousarray(flat[pl.own_lo: pl.own_hi])).to(dev)
    err = float((xh.double() - ref.double()).abs().max().item()) if nloc else 0.0
    e = torch.tensor([err], dtype=torch.float64, device=xdev)
    tdist.all_reduce(e, op=tdist.ReduceOp.MAX)
    lt = torch.tensor([launches[0] / max(1, args.steps)], dtype=torch.float64, device=xdev)
    tdist.all_reduce(lt, op=tdist.ReduceOp.SUM)
    # a wrong multi-GPU decode must not print a valid bench line
    err = float(e.item())
    if err > last_params[0].eb_abs:
        raise SystemExit(f"bench_dist: max |x - x^| = {err} exceeds eb_abs = {last_params[0].eb_abs}")
    extra = _replica_and_link_legs(args, rank, world, dev, xdev, tdist, torch, fz, synth, d, shape, rel, pl)
    if rank == 0:
        gb = d.nbytes / 1e9
        roof = None
        if "k_compress" in prof:
            pk = prof["k_compress"][0] / prof["k_compress"][1]
            ab = 4 * nloc + (total - 128) * nloc / max(1, d.size)   # rank 0's share of the stream
            peak = _peak()
            ach = ab / (pk / 1e3) / 1e9
            roof = {"kernel": "k_compress (rank 0 slab)", "bound": "hbm", "achieved": round(ach, 1),
                    "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4), "traffic": None,
                    "ms_per_launch": round(pk, 4),
                    "kernels_ms": {k: round(v[0] / v[1], 4) for k, v in prof.items()}}
        line = {
            "metric": metric, "value": round(gb / (ms / 1e3), 3), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": desc, "dims": list(shape), "rel_eb": rel, "field_bytes": d.nbytes,
                       "parallelism": f"z-slabs x{world}, {'NCCL' if backend == 'nccl' else 'gloo (ranks sharing one GPU)'} "
                                      "all_gathers (range, counts, carry planes)",
                       "l2": "field 4.3x L2"},
            "cr": round(d.nbytes / total, 4),
            "max_abs_err_over_eb_abs": round(err / last_params[0].eb_abs, 6),
            "gpu_launches": int(lt.item() * args.steps),
            "clocks": sampler.summary(),
            "roofline": roof,
            "e2e": {"value": round(gb / (ems / 1e3), 3), "unit": "GB/s", "ms_per_step": round(ems, 4),
                    "h2d_bytes_per_step": int(ebytes[0].item()), "d2h_bytes_per_step": int(ebytes[1].item()),
                    "path": "slab API per rank: pinned H2D of the slab, compress, D2H + H2D of the rank's "
                            "compressed share, decode, D2H of the decoded slab"},
            "collectives_ms_per_step": round(coll_ms, 4),
            "value_without_collectives": round(gb / (max(ms - coll_ms, 1e-6) / 1e3), 3),
            **extra,
        }
        print(json.dumps(line), flush=True)
    tdist.barrier()
    tdist.destroy_process_group()


def _replica_and_link_legs(args, rank, world, dev, xdev, tdist, torch, fz, synth, d, shape, rel, pl):
    """c5 as replicas (SV 8.e: "c5 is replicas": every rank compresses + decompresses its own
    RTM field t = rank, no collective; aggregate = sum of fields / max over ranks), and f4
    (P:476-483): pairwise exchange of a field between ranks 2j and 2j+1 raw (the field's bytes
    over NCCL) against compressed (compress, send the stream, decompress), CUDA events, max
    over ranks.  Returns the keys for rank 0's JSON line."""
    import statistics as st_

    from . import link
    out = {}
    # ---- c5 replicas ----
    if not os.environ.get("FZ_DIST_NO_REPLICAS"):
        rshape = (1008, 1008, 352)
        r = torch.from_numpy(synth.generate("rtm", rshape, seed=5 + rank % 8)).to(dev)
        c = fz.Codec(rshape, dev)
        xr = torch.empty_like(r)
        for _ in range(3):
            c.compress(r, fz.REL, 1e-4, sync=False)
            c.decompress_device(c.out, out=xr)
        torch.cuda.synchronize()
        tdist.barrier()
        evs = []
        for _ in range(max(3, min(args.steps, 10))):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            c.compress(r, fz.REL, 1e-4, sync=False)
            c.decompress_device(c.out, out=xr)
            e1.record()
            evs.append((e0, e1))
        torch.cuda.synchronize()
        size = c.compress_result()
        c.result()
        tr = torch.tensor([st_.mean(a.elapsed_time(b) for a, b in evs)], dtype=torch.float64, device=xdev)
        tdist.all_reduce(tr, op=tdist.ReduceOp.MAX)
        out["c5_replicas"] = {"workload": f"c5 RTM-shaped 1008x1008x352 REL 1e-4, one field per rank (t = rank), "
                                          f"{world} replicas, no collective",
                              "value": round(world * r.numel() * 4 / 1e9 / (float(tr.item()) / 1e3), 3),
                              "unit": "GB/s (sum over ranks)", "ms_per_step": round(float(tr.item()), 4),
                              "cr_rank0": round(r.numel() * 4 / size, 4)}
        del r, xr, c
        torch.cuda.empty_cache()
    # ---- f4: compressed vs raw pairwise exchange ----
    if world >= 2 and world % 2 == 0:
        peer = rank ^ 1
        lshape = (max(1, (pl.own_hi - pl.own_lo) // (shape[1] * shape[2])),) + tuple(shape[1:])
        nloc = int(np.prod(lshape))
        flat = d.reshape(-1)
        mine = torch.from_numpy(np.ascontiguousarray(flat[pl.own_lo: pl.own_lo + nloc])).to(dev).reshape(lshape)
        got = torch.empty_like(mine)
        transport = "cuda" if xdev.type == "cuda" else "cpu"
        lk = link.CompressedLink(link.fz_codec(lshape, fz.REL, rel, dev), transport=transport)
        raw_t = mine if transport == "cuda" else mine.cpu()
        raw_o = torch.empty_like(raw_t)

        def run(fn, k):
            tdist.barrier()
            torch.cuda.synchronize()
            ts = []
            for _ in range(k):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            t = torch.tensor([st_.mean(ts)], dtype=torch.float64, device=xdev)
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
            return float(t.item())

        run(lambda: link.CompressedLink.exchange_raw(raw_t, peer, raw_o), 2)
        run(lambda: lk.exchange(mine, peer, got), 2)
        ms_raw = run(lambda: link.CompressedLink.exchange_raw(raw_t, peer, raw_o), max(3, min(args.steps, 10)))
        ms_cmp = run(lambda: lk.exchange(mine, peer, got), max(3, min(args.steps, 10)))
        # the received field decodes within the peer's REL bound
        from . import dist as fzd
        ppl = fzd.plan(shape, world, peer)
        pf = torch.from_numpy(np.ascontiguousarray(flat[ppl.own_lo: ppl.own_lo + nloc])).to(dev)
        perr = float((got.reshape(-1).double() - pf.double()).abs().max().item())
        pebs = rel * (float(pf.max().item()) - float(pf.min().item()))
        if perr > pebs:
            raise SystemExit(f"bench_dist f4: received field error {perr} exceeds the peer's bound {pebs}")
        gb = world * nloc * 4 / 1e9
        out["f4_compressed_link"] = {
            "what": "pairwise exchange of each rank's slab (ranks 2j <-> 2j+1): raw field bytes over "
                    f"{'NCCL' if transport == 'cuda' else 'gloo (host-staged)'} vs compress + send stream + decompress",
            "raw_gbs": round(gb / (ms_raw / 1e3), 3), "compressed_gbs": round(gb / (ms_cmp / 1e3), 3),
            "ms_raw": round(ms_raw, 4), "ms_compressed": round(ms_cmp, 4),
            "stream_bytes_rank0": lk.last_sent, "field_bytes_per_rank": nloc * 4,
            "max_err_over_eb_rank0": round(perr / pebs, 6) if pebs > 0 else None,
            "unit": "GB/s of original data, all ranks"}
    return out
