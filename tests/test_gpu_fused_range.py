"""C0 (the range pass, P:320 / R4 / R18) fused into the row walker's first phase (SV §8.f2,
P:509 "fusing all GPU kernels into one"): streams byte-identical to the oracle with the fused
phase and with the separate k_range launch (variant 2097152), the first non-finite index
decides the status, -0.0 canonicalized, one launch fewer, and no deadlock when two fused
compressions share the GPU from two streams (chunks are claimed, not assigned)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle_lib as O
from paper_2304_12557_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2304_12557_b200 import fz  # noqa: E402

DEV = "cuda:0"
SEPARATE_RANGE = 2097152   # fz_debug_set_variant bit: k_range launched before the walker

# row-walker shapes (nx in {128, 256, 512, 1024}, ny % 16 == 0): several runs per CTA,
# ragged run lengths (U not a multiple of the grid), one band per plane
ZR_SHAPES = [
    ("nyx_v", (40, 32, 256), 1e-3),
    ("nyx_rho", (33, 48, 128), 1e-3),
    ("sines3d", (20, 16, 512), 1e-4),
    ("rtm", (12, 16, 1024), 1e-3),
    ("nyx_v", (300, 64, 128), 1e-3),
    # shapes on the warp-specialized single-pass kernel (2-D, short 3-D): k_range either way
    ("cesm_t", (200, 400), 1e-3),
    ("hurr_u", (12, 50, 52), 1e-3),
    ("cesm_cld", (181, 359), 1e-4),
]


def _stream(d, mode, eb):
    codec = fz.Codec(d.shape, DEV)
    buf, size = codec.compress(torch.from_numpy(np.ascontiguousarray(d)).to(DEV), mode, eb)
    torch.cuda.synchronize()
    return buf.cpu().numpy().copy(), codec


@pytest.mark.parametrize("name,shape,eb", ZR_SHAPES)
@pytest.mark.parametrize("mode,omode", [(fz.REL, O.REL), (fz.ABS, O.ABS)])
def test_fused_range_stream_parity(name, shape, eb, mode, omode):
    d = synth.generate(name, shape)
    e = eb if mode == fz.REL else eb * float(d.max() - d.min())
    st, ref = O.compress(d, omode, e)
    assert st == O.OK
    for variant in (0, SEPARATE_RANGE):
        fz.debug_set_variant(variant)
        try:
            got, _ = _stream(d, mode, e)
        finally:
            fz.debug_set_variant(0)
        assert got.size == ref.size and np.array_equal(got, ref), f"{name}{shape} variant {variant}"


def test_fused_range_launches_one_kernel_fewer():
    d = synth.generate("nyx_v", (40, 32, 256))
    f = torch.from_numpy(d).to(DEV)
    codec = fz.Codec(d.shape, DEV)
    fz.profile_enable(True)
    try:
        fz.profile_read()
        codec.compress(f, fz.REL, 1e-3)
        torch.cuda.synchronize()
        fused = fz.profile_read()
        n_fused = fz.last_launch_count()
        fz.debug_set_variant(SEPARATE_RANGE)
        codec.compress(f, fz.REL, 1e-3)
        torch.cuda.synchronize()
        sep = fz.profile_read()
        n_sep = fz.last_launch_count()
    finally:
        fz.debug_set_variant(0)
        fz.profile_enable(False)
    assert "k_range" not in fused and "k_range" in sep
    assert n_fused == n_sep - 1


@pytest.mark.parametrize("shape", [(40, 32, 256), (60, 333)])
@pytest.mark.parametrize("where", ["first", "last", "middle", "two", "inf_neg"])
def test_fused_range_nonfinite(where, shape):
    d = synth.generate("nyx_v" if len(shape) == 3 else "cesm_t", shape).copy()
    flat = d.reshape(-1)
    n = flat.size
    if where == "first":
        flat[0] = np.nan
    elif where == "last":
        flat[n - 1] = np.inf
    elif where == "middle":
        flat[n // 2 + 7] = np.nan
    elif where == "two":
        flat[[n - 5, 1000]] = [np.nan, np.inf]
    else:
        flat[12345 % n] = -np.inf
    st, _ = O.compress(d, O.REL, 1e-3)
    assert st == O.ERR_NONFINITE
    codec = fz.Codec(d.shape, DEV)
    with pytest.raises(fz.FZError) as e:
        codec.compress(torch.from_numpy(d).to(DEV), fz.REL, 1e-3)
    assert e.value.status == fz.ERR_NONFINITE
    # the same codec compresses a finite field afterwards (the claim counters are per call)
    g = synth.generate("nyx_v" if len(shape) == 3 else "cesm_t", shape)
    st, ref = O.compress(g, O.REL, 1e-3)
    buf, size = codec.compress(torch.from_numpy(g).to(DEV), fz.REL, 1e-3)
    assert size == ref.size and np.array_equal(buf.cpu().numpy(), ref)


def test_fused_range_negative_zero():
    """R18: -0.0 counts as +0.0, so the header's min / max are unique bit patterns."""
    d = synth.generate("nyx_v", (24, 16, 128)).copy()
    d[d < 0] = np.float32(-0.0)          # min is -0.0 / +0.0
    st, ref = O.compress(d, O.REL, 1e-3)
    assert st == O.OK
    got, _ = _stream(d, fz.REL, 1e-3)
    assert np.array_equal(got, ref)
    z = np.full((8, 16, 128), np.float32(-0.0), dtype=np.float32)
    z[3, 5, 7] = np.float32(0.0)
    st, ref = O.compress(z, O.ABS, 1e-3)
    got, _ = _stream(z, fz.ABS, 1e-3)
    assert np.array_equal(got, ref)


def test_fused_range_two_streams_concurrently():
    """Two fused compressions in flight on two streams: the second kernel's CTAs may not be
    resident while the first one's wait -- claimed chunks keep both deadlock-free."""
    a = synth.generate("nyx_v", (256, 128, 512))
    b = synth.generate("nyx_rho", (256, 128, 512))
    refs = []
    for d in (a, b):
        st, r = O.compress(d, O.REL, 1e-3)
        assert st == O.OK
        refs.append(r)
    ca, cb = fz.Codec(a.shape, DEV), fz.Codec(b.shape, DEV)
    fa, fb = torch.from_numpy(a).to(DEV), torch.from_numpy(b).to(DEV)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    for _ in range(3):
        ca.compress(fa, fz.REL, 1e-3, stream=s1, sync=False)
        cb.compress(fb, fz.REL, 1e-3, stream=s2, sync=False)
        torch.cuda.synchronize()
        for c, r, s in ((ca, refs[0], s1), (cb, refs[1], s2)):
            size = c.compress_result(stream=s)
            assert size == r.size and np.array_equal(c.out[:size].cpu().numpy(), r)


@pytest.mark.parametrize("variant", [0, SEPARATE_RANGE, 67108864])
def test_fused_range_chunk_local_and_log_transform(variant):
    """The fused phase under f1 (chunk-local Lorenzo: the range stays field-global) and f3
    (FZ_EB_PWREL: the phase reads the log field in the workspace); variant 67108864 launches
    every kernel without programmatic dependent launch -- the same bytes."""
    d = synth.generate("nyx_v", (40, 32, 256))
    st, ref = O.compress_chunked(d, O.REL, 1e-3, 16, 2048 // d.shape[2])
    assert st == O.OK
    r = synth.generate("nyx_rho", (40, 32, 256))   # positive (log-normal): log domain
    st, ref_pw = O.compress(r, O.PWREL, 1e-3)
    assert st == O.OK
    fz.debug_set_variant(variant)
    try:
        codec = fz.Codec(d.shape, DEV)
        buf, size = codec.compress(torch.from_numpy(d).to(DEV), fz.REL | fz.CHUNK_LOCAL, 1e-3)
        got = buf.cpu().numpy().copy()
        xh = codec.decompress(buf).cpu().numpy().reshape(-1)
        buf2, size2 = codec.compress(torch.from_numpy(r).to(DEV), fz.PWREL, 1e-3)
        got2 = buf2.cpu().numpy().copy()
        xh2 = codec.decompress(buf2).cpu().numpy().reshape(-1)
        torch.cuda.synchronize()
    finally:
        fz.debug_set_variant(0)
    assert size == ref.size and np.array_equal(got, ref)
    st, xref = O.decompress(ref, d.size)
    assert np.array_equal(xh.view(np.uint32), xref.view(np.uint32))
    assert size2 == ref_pw.size and np.array_equal(got2, ref_pw)
    st, xref2 = O.decompress(ref_pw, r.size)
    assert np.array_equal(xh2.view(np.uint32), xref2.view(np.uint32))
