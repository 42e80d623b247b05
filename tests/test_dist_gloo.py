"""World-size-2 gloo tests (CPU) of the multi-GPU host logic: slab plans, the range and
count all_gathers, the carry-plane exchange and the prefix arithmetic."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2304_12557_b200 import dist as fzd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(rank)
        vals = rng.normal(size=100).astype(np.float32)
        mn, mx = fzd.exchange_range(float(vals.min()), float(vals.max()))
        counts = (10 * (rank + 1), rank, 2 * rank)
        before, totals = fzd.exchange_counts(counts)
        agg = torch.arange(6, dtype=torch.int32) * (rank + 1)
        planes = fzd.exchange_planes(agg)
        carry = planes[:rank].sum(dim=0) if rank else torch.zeros(6, dtype=torch.int64)
        q.put((rank, mn, mx, before, totals, planes.tolist(), carry.tolist()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchanges():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    mins = [float(np.random.default_rng(r).normal(size=100).astype(np.float32).min()) for r in range(world)]
    maxs = [float(np.random.default_rng(r).normal(size=100).astype(np.float32).max()) for r in range(world)]
    for r, mn, mx, before, totals, planes, carry in res:
        assert mn == min(mins) and mx == max(maxs)
        assert totals == (30, 1, 2)
        assert before == [(0, 0, 0), (10, 0, 0)]
        assert planes == [[0, 1, 2, 3, 4, 5], [0, 2, 4, 6, 8, 10]]
        assert carry == ([0] * 6 if r == 0 else [0, 1, 2, 3, 4, 5])


@pytest.mark.parametrize("dims,world", [((512, 512, 512), 8), ((64, 64, 64), 3), ((100, 500, 500), 4),
                                        ((1800, 3600), 5), ((280953,), 7), ((3, 5, 7), 4)])
def test_slab_plans_partition_and_halo(dims, world):
    n, nx, P, halo = fzd.geometry(dims)
    T = -(-n // 2048)
    plans = [fzd.plan(dims, world, k) for k in range(world)]
    assert plans[0].tb == 0 and plans[-1].te == T
    for a, b in zip(plans, plans[1:]):
        assert a.te == b.tb                      # contiguous, disjoint tile ranges
    for p in plans:
        assert p.slab_first % 4 == 0
        assert p.slab_first <= max(0, p.own_lo - halo)  # read-only Lorenzo halo held
        assert p.slab_hi == p.own_hi == min(n, p.te * 2048)
    if len(dims) == 3 and P % 2048 == 0:
        assert all((p.tb * 2048) % P == 0 for p in plans)   # plane-aligned: decodable slabs


def test_prefix_counts():
    before, totals = fzd.prefix_counts([(3, 1, 0), (0, 0, 0), (5, 2, 7)])
    assert before == [(0, 0, 0), (3, 1, 0), (3, 1, 0)] and totals == (8, 3, 7)


@pytest.mark.parametrize("world", [1, 2, 3, 5, 8])
def test_chunk_aligned_plan(world):
    """f1: chunk-local slabs are whole chunks of 16 planes, cover every tile once, in order."""
    from paper_2304_12557_b200 import dist
    dims = (100, 64, 128)
    P = dims[1] * dims[2]
    plans = [dist.plan(dims, world, k, chunk=16) for k in range(world)]
    assert plans[0].tb == 0 and plans[-1].te == plans[0].tiles
    for a, b in zip(plans, plans[1:]):
        assert a.te == b.tb
    for p in plans:
        if p.te > p.tb:
            assert (p.tb * 2048) % (16 * P) == 0
            assert p.te == p.tiles or (p.te * 2048) % (16 * P) == 0


# ---- f4: compressed transfer between ranks, protocol checked with the oracle as
# the codec (the CPU stand-in; the GPU test runs libfz through the same link) ----
def _oracle_codec(shape, eb):
    import oracle_lib as O
    from paper_2304_12557_b200 import link

    def compress(field):
        st, buf = O.compress(field.numpy(), O.REL, eb)
        assert st == O.OK
        return torch.from_numpy(buf)

    def decompress(stream, out):
        st, x = O.decompress(stream.numpy(), out.numel())
        assert st == O.OK
        out.copy_(torch.from_numpy(x).reshape(out.shape))

    return link.Codec(compress, decompress, O.compress_bound(shape))


def _link_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2304_12557_b200 import link, synth
        shape = (24, 40, 56)
        mine = torch.from_numpy(synth.generate("sines3d", shape, seed=11 + rank))
        lk = link.CompressedLink(_oracle_codec(shape, 1e-3), transport="cpu")
        got = torch.empty(shape, dtype=torch.float32)
        n = lk.exchange(mine, 1 - rank, got)
        raw = torch.empty(shape, dtype=torch.float32)
        link.CompressedLink.exchange_raw(mine, 1 - rank, raw)
        q.put((rank, n, lk.last_sent, got.numpy().copy(), raw.numpy().copy()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_compressed_link():
    import oracle_lib as O
    from paper_2304_12557_b200 import synth
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_link_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=120) for _ in range(world)), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    shape = (24, 40, 56)
    for rank, n, sent, got, raw in res:
        peer = synth.generate("sines3d", shape, seed=11 + (1 - rank))
        st, ref = O.compress(peer, O.REL, 1e-3)
        st, xr = O.decompress(ref, peer.size)
        assert n == ref.size                       # only the stream's bytes crossed
        assert np.array_equal(got.reshape(-1).view(np.uint32), xr.view(np.uint32))
        assert np.array_equal(raw, peer)
    assert res[0][2] == res[1][1] and res[1][2] == res[0][1]   # sizes agree both ways
