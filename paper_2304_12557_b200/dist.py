"""Multi-GPU z-slab partitioning of the compressor ("embarrassingly parallel";
SURVEY §8.e).  One process per GPU over torch.distributed (NCCL on B200s, gloo in CPU tests).

Rank k owns the global tiles [tb_k, te_k): tile-aligned z-slabs.  It holds its slab plus a
read-only Lorenzo halo of one plane + one row + one element (P + nx + 1 elements) before it.
The path has exactly two exchange steps, both tiny all_gathers:
  1. (min, max) of every rank -> identical Appendix-A parameters everywhere (REL needs the
     global range; the margin needs max|d|);
  2. (nnz, n_delta, n_value) of every rank -> exclusive prefixes = where each rank's share of
     every section goes in the global stream.
The concatenated stream is byte-identical to the 1-GPU stream for any rank count (R19).

Decompression of plane-aligned slabs (3-D: slab starts at multiples of P = ny*nx) has one
more exchange: each rank decodes its share locally (x and y prefix sums), reduces it to one
int32 plane (its z aggregate), the planes are all_gathered, and rank k seeds its z prefix sum
with the sum of the k lower planes (fz_slab_carry) before dequantizing (fz_slab_finish).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

TILE = 2048


@dataclass
class SlabPlan:
    rank: int
    world: int
    n: int
    tiles: int
    tb: int            # first owned tile
    te: int            # one past the last owned tile
    own_lo: int        # first owned element
    own_hi: int        # one past the last owned element
    slab_first: int    # first element held (halo included), multiple of 4
    slab_hi: int       # one past the last element held


def geometry(dims):
    dims = tuple(int(x) for x in dims)
    n = int(np.prod(dims))
    if len(dims) == 1:
        nx, P = n, n
        halo = 1
    elif len(dims) == 2:
        nx, P = dims[1], n
        halo = nx + 1
    else:
        nx, P = dims[2], dims[1] * dims[2]
        halo = P + nx + 1
    return n, nx, P, halo


def plan(dims, world: int, rank: int, chunk: int = 1) -> SlabPlan:
    """Tile-aligned z-slabs: rank k starts at the tile containing plane floor(k*nz/world)
    (plane-aligned whenever P % 2048 == 0).  chunk > 1 (f1 chunk-local streams): slabs are
    whole chunks of `chunk` planes, rank k starting at chunk floor(k * nchunks / world)."""
    dims = tuple(int(x) for x in dims)
    n, nx, P, halo = geometry(dims)
    T = -(-n // TILE)

    def start(k):
        if k >= world:
            return T
        if len(dims) == 3:
            if chunk > 1:
                z = (k * (-(-dims[0] // chunk)) // world) * chunk
            else:
                z = k * dims[0] // world
            return (z * P) // TILE
        return (k * T) // world

    tb, te = start(rank), start(rank + 1)
    own_lo, own_hi = tb * TILE, min(n, te * TILE)
    slab_first = max(0, own_lo - halo) & ~3
    return SlabPlan(rank, world, n, T, tb, te, own_lo, own_hi, slab_first, own_hi)


def combine_ranges(mins, maxs):
    """Global (min, max) from per-rank values (ranks with no elements pass None)."""
    lo = min(m for m in mins if m is not None)
    hi = max(m for m in maxs if m is not None)
    return float(np.float32(lo)), float(np.float32(hi))


def prefix_counts(all_counts):
    """all_counts: list over ranks of (nnz, nd, nv) -> (before[rank], totals)."""
    before, acc = [], np.zeros(3, dtype=np.uint64)
    for c in all_counts:
        before.append(tuple(int(v) for v in acc))
        acc = acc + np.asarray(c, dtype=np.uint64)
    return before, tuple(int(v) for v in acc)


# ----------------------------------------------------------------------------------------
# torch.distributed exchange steps (NCCL on GPUs, gloo in the CPU tests)
# ----------------------------------------------------------------------------------------
def exchange_range(mn: float, mx: float, device="cpu"):
    import torch
    import torch.distributed as dist
    t = torch.tensor([mn, mx], dtype=torch.float64, device=device)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    vals = torch.stack(out).cpu().numpy()
    return combine_ranges(vals[:, 0].tolist(), vals[:, 1].tolist())


def exchange_planes(agg, device=None):
    """all_gather of the per-rank aggregate planes (int32 tensors, same length)."""
    import torch
    import torch.distributed as dist
    out = [torch.empty_like(agg) for _ in range(dist.get_world_size())]
    dist.all_gather(out, agg)
    return torch.stack(out)


def exchange_counts(counts, device="cpu"):
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(counts), dtype=torch.int64, device=device)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    allc = torch.stack(out).cpu().numpy().tolist()
    return prefix_counts(allc)


# ----------------------------------------------------------------------------------------
# GPU slab compression
# ----------------------------------------------------------------------------------------
class SlabCompressor:
    """Per-rank device buffers for repeated slab compression of one global field."""

    def __init__(self, dims, pl: SlabPlan, device):
        import torch

        from . import fz
        self.fz = fz
        self.dims = tuple(int(x) for x in dims)
        self.pl = pl
        self.device = device
        self.stage = torch.empty(max(16, fz.slab_stage_bound(self.dims, pl.tb, pl.te)), dtype=torch.uint8,
                                 device=device)
        self.work = torch.empty(fz.workspace_bytes(self.dims), dtype=torch.uint8, device=device)
        self.out = None

    def local_range(self, slab):
        pl = self.pl
        own = slab[pl.own_lo - pl.slab_first: pl.own_hi - pl.slab_first]
        mn, mx, bad = self.fz.slab_range(own, self.work)
        if bad >= 0:
            raise self.fz.FZError(self.fz.ERR_NONFINITE, f"rank {pl.rank}: index {bad + pl.own_lo}")
        return mn, mx

    def compress_local(self, slab, params):
        pl = self.pl
        return self.fz.slab_compress(slab, pl.slab_first, self.dims, pl.tb, pl.te, params, self.stage, self.work)

    def decode_local(self, counts, q, agg, dwork):
        pl = self.pl
        self.fz.slab_decode(self.stage, counts, self.dims, pl.tb, pl.te, q, agg, dwork)

    def finish(self, q, carry, counts, params):
        pl = self.pl
        self.fz.slab_finish(q, carry, self.stage, counts, self.dims, pl.tb, pl.te, params)

    def place(self, counts, before, totals, params, out):
        fz = self.fz
        pl = self.pl
        fz.slab_place(self.stage, self.dims, pl.tb, pl.te, counts, fz.Counts(*before), fz.Counts(*totals),
                      params, pl.tb == 0, out)


def compress_sharded_single_process(d: np.ndarray, mode, eb, ranks: int, device="cuda:0") -> np.ndarray:
    """Runs the k-rank slab protocol sequentially on one GPU (the host plays the
    collectives).  Used by the parity tests: the result must equal the 1-GPU stream."""
    import torch

    from . import fz
    dims = d.shape
    flat = np.ascontiguousarray(d).reshape(-1)
    plans = [plan(dims, ranks, k) for k in range(ranks)]
    plans = [p for p in plans if p.te > p.tb]
    comps, slabs = [], []
    mins, maxs = [], []
    for p in plans:
        slab = torch.from_numpy(flat[p.slab_first: p.slab_hi].copy()).to(device)
        c = SlabCompressor(dims, p, device)
        mn, mx = c.local_range(slab)
        mins.append(mn)
        maxs.append(mx)
        comps.append(c)
        slabs.append(slab)
    gmn, gmx = combine_ranges(mins, maxs)
    params = fz.derive_params(gmn, gmx, mode, eb)
    counts = [c.compress_local(s, params) for c, s in zip(comps, slabs)]
    before, totals = prefix_counts([(c.nnz, c.n_delta, c.n_value) for c in counts])
    T = plans[0].tiles
    total = 128 + 32 * T + 16 * totals[0] + 8 * totals[1] + 8 * totals[2]
    out = torch.zeros(total, dtype=torch.uint8, device=device)
    for c, cnt, b in zip(comps, counts, before):
        c.place(cnt, b, totals, params, out)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def roundtrip_sharded_single_process(d: np.ndarray, mode, eb, ranks: int, device="cuda:0"):
    """Compress and decompress through the k-rank slab protocol sequentially on one GPU.
    Returns (stream bytes, decompressed field).  Requires plane-aligned slabs."""
    import torch

    from . import fz
    dims = d.shape
    flat = np.ascontiguousarray(d).reshape(-1)
    plans = [p for p in (plan(dims, ranks, k) for k in range(ranks)) if p.te > p.tb]
    comps, slabs, mins, maxs = [], [], [], []
    for p in plans:
        slab = torch.from_numpy(flat[p.slab_first: p.slab_hi].copy()).to(device)
        c = SlabCompressor(dims, p, device)
        mn, mx = c.local_range(slab)
        mins.append(mn)
        maxs.append(mx)
        comps.append(c)
        slabs.append(slab)
    params = fz.derive_params(*combine_ranges(mins, maxs), mode, eb)
    counts = [c.compress_local(s, params) for c, s in zip(comps, slabs)]
    before, totals = prefix_counts([(c.nnz, c.n_delta, c.n_value) for c in counts])
    T = plans[0].tiles
    out = torch.zeros(128 + 32 * T + 16 * totals[0] + 8 * totals[1] + 8 * totals[2], dtype=torch.uint8,
                      device=device)
    for c, cnt, b in zip(comps, counts, before):
        c.place(cnt, b, totals, params, out)
    # decode: local decode -> aggregates -> carries -> finish
    E = fz.slab_agg_elems(dims)
    aggs = torch.empty((len(plans), E), dtype=torch.int32, device=device)
    qs = []
    for k, (c, cnt, p) in enumerate(zip(comps, counts, plans)):
        q = torch.empty(p.own_hi - p.own_lo, dtype=torch.int32, device=device)
        local_dims = (int((p.own_hi - p.own_lo) // E),) + tuple(dims[1:]) if len(dims) > 1 else (p.own_hi - p.own_lo,)
        dwork = torch.empty(max(16, fz.decompress_workspace_bytes(local_dims)), dtype=torch.uint8, device=device)
        c.decode_local(cnt, q, aggs[k], dwork)
        qs.append(q)
    xhat = np.empty(flat.size, dtype=np.float32)
    for k, (c, cnt, p, q) in enumerate(zip(comps, counts, plans, qs)):
        carry = torch.empty(E, dtype=torch.int32, device=device)
        fz.slab_carry(aggs, k, E, carry)
        c.finish(q, carry, cnt, params)
        xhat[p.own_lo: p.own_hi] = q.view(torch.float32).cpu().numpy()
    torch.cuda.synchronize()
    return out.cpu().numpy(), xhat


def roundtrip_chunk_local_single_process(d: np.ndarray, mode, eb, ranks: int, device="cuda:0"):
    """f1: the k-rank slab protocol for a chunk-local stream, sequentially on one GPU.  The
    compress side is the usual one (range exchange, counts exchange, placement); the decode
    side needs no exchange at all -- each rank decodes its whole chunks on its own
    (fz_slab_decode_cl).  Returns (stream bytes, decompressed field)."""
    import torch

    from . import fz
    dims = d.shape
    flat = np.ascontiguousarray(d).reshape(-1)
    plans = [p for p in (plan(dims, ranks, k, chunk=16) for k in range(ranks)) if p.te > p.tb]
    comps, slabs, mins, maxs = [], [], [], []
    for p in plans:
        slab = torch.from_numpy(flat[p.slab_first: p.slab_hi].copy()).to(device)
        c = SlabCompressor(dims, p, device)
        mn, mx = c.local_range(slab)
        mins.append(mn)
        maxs.append(mx)
        comps.append(c)
        slabs.append(slab)
    params = fz.derive_params(*combine_ranges(mins, maxs), mode, eb)
    params.mode |= fz.CHUNK_LOCAL
    counts = [c.compress_local(s, params) for c, s in zip(comps, slabs)]
    before, totals = prefix_counts([(c.nnz, c.n_delta, c.n_value) for c in counts])
    T = plans[0].tiles
    out = torch.zeros(128 + 32 * T + 16 * totals[0] + 8 * totals[1] + 8 * totals[2], dtype=torch.uint8,
                      device=device)
    for c, cnt, b in zip(comps, counts, before):
        c.place(cnt, b, totals, params, out)
    xhat = np.empty(flat.size, dtype=np.float32)
    for c, cnt, p in zip(comps, counts, plans):
        local_dims = (int((p.own_hi - p.own_lo) // (dims[1] * dims[2])),) + tuple(dims[1:])
        dwork = torch.empty(max(16, fz.decompress_workspace_bytes(local_dims)), dtype=torch.uint8, device=device)
        x = torch.empty(p.own_hi - p.own_lo, dtype=torch.float32, device=device)
        fz.slab_decode_cl(c.stage, cnt, dims, p.tb, p.te, params, x, dwork)
        xhat[p.own_lo: p.own_hi] = x.cpu().numpy()
    torch.cuda.synchronize()
    return out.cpu().numpy(), xhat
