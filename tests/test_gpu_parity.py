"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, bit-exact.

Compared element by element on the same seeded inputs: the compressed byte stream, the
uint16 quant codes, both outlier lists, the reconstructed integer codes and the decompressed
fp32 array (BJ north star: "GPU output must match the oracle bit-exactly").
"""
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


def _gpu_stream(d: np.ndarray, mode, eb, params=None):
    codec = fz.Codec(d.shape, DEV)
    field = torch.from_numpy(np.ascontiguousarray(d)).to(DEV)
    buf, size = codec.compress(field, mode, eb, params)
    out = buf.cpu().numpy().copy()
    xh = codec.decompress(buf).cpu().numpy().reshape(-1)
    torch.cuda.synchronize()
    return out, xh, codec


def _assert_stream_equal(got: np.ndarray, ref: np.ndarray, name=""):
    if got.size != ref.size or not np.array_equal(got, ref):
        n = min(got.size, ref.size)
        diff = np.nonzero(got[:n] != ref[:n])[0]
        first = int(diff[0]) if diff.size else n
        raise AssertionError(f"{name}: sizes {got.size} vs {ref.size}, first differing byte {first}")


def _check_full(d: np.ndarray, mode, eb, name=""):
    st, ref = O.compress(d, mode, eb)
    assert st == O.OK
    got, xh, codec = _gpu_stream(d, mode, eb)
    _assert_stream_equal(got, ref, name)
    st, xref = O.decompress(ref, d.size)
    assert st == O.OK
    bad = np.nonzero(xh.view(np.uint32) != xref.view(np.uint32))[0]
    assert bad.size == 0, f"{name}: {bad.size} decoded values differ, first at {bad[:5]}"
    return ref


SMALL = [
    ("sines3d", lambda: synth.generate("sines3d", (64, 64, 64))),
    ("sines3d_ragged", lambda: synth.generate("sines3d", (33, 47, 61))),
    ("cesm_t", lambda: synth.generate("cesm_t", (180, 360))),
    ("cesm_cld", lambda: synth.generate("cesm_cld", (181, 359))),
    ("cesm_wide", lambda: synth.generate("cesm_t", (7, 5000))),          # nx > tile
    ("hurr_qsnow", lambda: synth.generate("hurr_qsnow", (10, 50, 50))),
    ("hurr_u", lambda: synth.generate("hurr_u", (10, 50, 50))),
    ("nyx_rho", lambda: synth.generate("nyx_rho", (32, 32, 32))),
    ("nyx_v", lambda: synth.generate("nyx_v", (32, 32, 32))),
    ("rtm", lambda: synth.generate("rtm", (40, 40, 22))),
    ("qmc", lambda: synth.generate("qmc", (60, 9, 9))),
    ("tiny_nx", lambda: synth.generate("sines3d", (9, 5, 3))),
    ("noise1d", lambda: synth.adversarial("noise", 10007)),
    ("ramp1d", lambda: synth.adversarial("ramp", 4097)),
    ("const1d", lambda: synth.adversarial("constant", 3000)),
    ("zeros", lambda: synth.adversarial("zeros", 2049)),
    ("one", lambda: np.array([1.5], np.float32)),
]


@pytest.mark.parametrize("name,gen", SMALL, ids=[s[0] for s in SMALL])
@pytest.mark.parametrize("rel", [1e-2, 1e-3, 1e-4])
def test_stream_and_decode_parity(name, gen, rel):
    _check_full(gen(), O.REL, rel, f"{name}@{rel}")


@pytest.mark.parametrize("eb", [0.5, 1e-3, 1e-6])
def test_abs_mode_parity(eb):
    _check_full(synth.generate("hurr_u", (12, 40, 40)), O.ABS, eb, f"abs{eb}")


def test_codes_and_outlier_lists_parity():
    """Stage hook C1-C3: uint16 codes and both outlier lists equal the oracle's."""
    cases = [synth.generate("sines3d", (40, 41, 42)), synth.adversarial("spike", 20000),
             synth.adversarial("offset", 9000), np.array([1e30, -1e30, 1.0, 0.0] * 700, np.float32)]
    for d, mode, eb in zip(cases, [O.REL, O.ABS, O.REL, O.ABS], [1e-3, 1e-3, 1e-6, 1e-3]):
        p = O.params_for(d, mode, eb)
        codes, didx, dval, vidx, vbits = O.quantize_field(d, p)
        gp = fz.derive_params(p.mn, p.mx, mode, eb)
        field = torch.from_numpy(d).to(DEV)
        c2, di2, dv2, vi2, vb2 = fz.debug_quantize(field, gp)
        assert np.array_equal(c2.cpu().numpy().view(np.uint16), codes)
        assert np.array_equal(di2.cpu().numpy().view(np.uint32), didx)
        assert np.array_equal(dv2.cpu().numpy(), dval)
        assert np.array_equal(vi2.cpu().numpy().view(np.uint32), vidx)
        assert np.array_equal(vb2.cpu().numpy().view(np.uint32), vbits)


def test_outlier_streams_and_staging_overflow():
    # delta outliers (spike), fallback + value outliers (offset), and a case with more value
    # outliers than the staging area holds (N/64 + 1024), which takes the rescan path
    _check_full(synth.adversarial("spike", 50000), O.ABS, 1e-3, "spike")
    _check_full(synth.adversarial("offset", 30000), O.REL, 1e-6, "offset")
    big = np.tile(np.array([1e30, -1e30, 1.0, 0.0], np.float32), 20000)
    ref = _check_full(big, O.ABS, 1e-3, "overflow")
    assert int.from_bytes(ref[104:112].tobytes(), "little") > big.size // 64 + 1024


def test_decode_q_parity():
    d = synth.generate("nyx_v", (24, 30, 33))
    st, ref = O.compress(d, O.REL, 1e-4)
    st, qref = O.decode_q(ref, d.size)
    buf = torch.from_numpy(ref).to(DEV)
    q = fz.debug_decode_q(buf, d.shape)
    assert np.array_equal(q.cpu().numpy(), qref)


def test_error_bound_and_idempotence():
    d = synth.generate("cesm_t", (200, 400))
    ref = _check_full(d, O.REL, 1e-4, "bound")
    info = fz.peek_header(ref[:128].tobytes())
    st, xh = O.decompress(ref, d.size)
    assert np.abs(xh.astype(np.float64) - d.reshape(-1)).max() <= info.params.eb_abs
    # with params pinned (ABS), recompressing x-hat on the GPU is byte-identical (R22)
    p = fz.derive_params(float(d.min()), float(d.max()), fz.ABS, 0.01)
    got1, xh1, _ = _gpu_stream(d, fz.ABS, 0.01, params=p)
    got2, _, _ = _gpu_stream(xh1.reshape(d.shape), fz.ABS, 0.01, params=p)
    assert np.array_equal(got1, got2)


def test_nonfinite_capacity_and_corrupt():
    d = synth.generate("sines3d", (16, 16, 16)).copy()
    d.reshape(-1)[1234] = np.nan
    codec = fz.Codec(d.shape, DEV)
    with pytest.raises(fz.FZError) as e:
        codec.compress(torch.from_numpy(d).to(DEV), fz.REL, 1e-3)
    assert e.value.status == fz.ERR_NONFINITE
    # capacity: snprintf convention, nothing written past the cap
    d = synth.generate("sines3d", (16, 16, 16))
    st, ref = O.compress(d, O.REL, 1e-3)
    field = torch.from_numpy(d).to(DEV)
    cap = ref.size - 1
    out = torch.full((cap + 64,), 0xAB, dtype=torch.uint8, device=DEV)
    work = torch.empty(fz.workspace_bytes(d.shape), dtype=torch.uint8, device=DEV)
    import ctypes as C
    size = C.c_size_t()
    stt = fz.lib().fz_compress(C.c_void_p(field.data_ptr()), C.byref(fz.make_shape(d.shape)), fz.REL, 1e-3,
                               C.c_void_p(out.data_ptr()), cap, C.byref(size), C.c_void_p(work.data_ptr()),
                               work.numel(), None)
    torch.cuda.synchronize()
    assert stt == fz.ERR_CAPACITY and size.value == ref.size
    assert (out[cap:].cpu().numpy() == 0xAB).all()
    # corrupt streams never crash: structured error or a decode
    rng = np.random.default_rng(3)
    codec = fz.Codec(d.shape, DEV)
    for k in range(60):
        m = ref.copy()
        for _ in range(rng.integers(1, 4)):
            i = int(rng.integers(0, m.size))
            m[i] ^= np.uint8(1 << int(rng.integers(0, 8)))
        try:
            codec.decompress(torch.from_numpy(m).to(DEV))
        except fz.FZError as e:
            assert e.status in (fz.ERR_CORRUPT, fz.ERR_ARG)
    torch.cuda.synchronize()


@pytest.mark.parametrize("ranks", [1, 2, 3, 8])
def test_fake_multirank_slabs_byte_identical(ranks):
    """SV §8.e: tile-aligned z-slabs with a read-only halo, counts exchanged, placed at
    global offsets -> byte-identical to the single-GPU stream (and the oracle's)."""
    from paper_2304_12557_b200 import dist
    d = synth.generate("nyx_v", (64, 64, 64))
    st, ref = O.compress(d, O.REL, 1e-3)
    out = dist.compress_sharded_single_process(d, fz.REL, 1e-3, ranks, DEV)
    _assert_stream_equal(out, ref, f"ranks={ranks}")


def test_host_buffer_entry_points():
    d = synth.generate("hurr_u", (10, 50, 50))
    st, ref = O.compress(d, O.REL, 1e-3)
    cap = fz.compress_bound(d.shape)
    d_field = torch.empty(d.shape, dtype=torch.float32, device=DEV)
    d_out = torch.empty(cap, dtype=torch.uint8, device=DEV)
    work = torch.empty(fz.workspace_bytes(d.shape), dtype=torch.uint8, device=DEV)
    h_out = np.empty(cap, np.uint8)
    size = fz.compress_host(np.ascontiguousarray(d), fz.REL, 1e-3, d_field, d_out, work, h_out)
    assert np.array_equal(h_out[:size], ref)
    h_x = np.empty(d.shape, np.float32)
    dwork = torch.empty(fz.decompress_workspace_bytes(d.shape), dtype=torch.uint8, device=DEV)
    fz.decompress_host(h_out, size, h_x, d_out, d_field, dwork)
    st, xref = O.decompress(ref, d.size)
    assert np.array_equal(h_x.reshape(-1).view(np.uint32), xref.view(np.uint32))


@pytest.mark.parametrize("ranks", [1, 2, 4, 8])
def test_fake_multirank_roundtrip(ranks):
    """Slab decompression with the carry-plane exchange (SV §8.e) reproduces the oracle's
    decompressed field bit for bit; the assembled stream equals the oracle's."""
    from paper_2304_12557_b200 import dist
    d = synth.generate("nyx_rho", (64, 32, 64))           # P = 2048: plane-aligned slabs
    st, ref = O.compress(d, O.REL, 1e-3)
    st, xref = O.decompress(ref, d.size)
    stream, xh = dist.roundtrip_sharded_single_process(d, fz.REL, 1e-3, ranks, DEV)
    _assert_stream_equal(stream, ref, f"ranks={ranks}")
    assert np.array_equal(xh.view(np.uint32), xref.view(np.uint32))


@pytest.mark.parametrize("shape", [(300, 2048), (6000,), (4, 64, 64)])
def test_fake_multirank_roundtrip_2d_1d(shape):
    from paper_2304_12557_b200 import dist
    d = synth.adversarial("noise", int(np.prod(shape))).reshape(shape) + np.float32(3)
    st, ref = O.compress(d, O.ABS, 1e-2)
    st, xref = O.decompress(ref, d.size)
    stream, xh = dist.roundtrip_sharded_single_process(d, fz.ABS, 1e-2, 3, DEV)
    _assert_stream_equal(stream, ref, f"{shape}")
    assert np.array_equal(xh.view(np.uint32), xref.view(np.uint32))


@pytest.mark.parametrize("n", [1, 3, 4, 7, 1000, 4 * 148 * 8 * 256 * 4 + 13, 5_000_003])
def test_range_kernel_vs_oracle(n):
    """C0: (min, max) with -0.0 canonicalized and the first non-finite index (R18), on sizes
    that hit the scalar tail, the single-load loop and the 4-deep unrolled loop."""
    rng = np.random.default_rng(n)
    d = rng.normal(size=n).astype(np.float32) * np.float32(3.0)
    work = torch.empty(fz.workspace_bytes((n,)), dtype=torch.uint8, device=DEV)
    for case in range(4):
        x = d.copy()
        if case == 1:
            x[:] = np.float32(-0.0)
            x[n // 2] = np.float32(0.0)
        if case == 2 and n > 2:
            x[[n - 1, n // 3]] = [np.inf, np.nan]
        if case == 3:
            x[n - 1] = np.float32(-1e30)
        mn, mx, bad = fz.slab_range(torch.from_numpy(x).to(DEV), work)
        st, omn, omx, obad = O.field_range(x)
        if st == O.ERR_NONFINITE:
            assert bad == obad
        else:
            assert bad == -1
            assert np.float32(mn).tobytes() == np.float32(omn).tobytes()
            assert np.float32(mx).tobytes() == np.float32(omx).tobytes()


# Shapes on the decoder's fused-y path (k_decode_planes: 3-D, nz >= 148, nx in
# {256..2048} dividing the tile, tiles inside planes): R = 8, 4, 2, 1 rows per tile with two
# or more tiles per plane, one tile per plane, and delta outliers inside fused planes.
FUSED_Y = [
    ("r8", lambda: synth.generate("nyx_rho", (296, 16, 256))),
    ("r4", lambda: synth.generate("nyx_v", (296, 8, 512))),
    ("r2", lambda: synth.generate("hurr_u", (300, 4, 1024))),
    ("r1", lambda: synth.generate("rtm", (300, 2, 2048))),
    ("one_tile_per_plane", lambda: synth.generate("sines3d", (300, 8, 256))),
    ("tpp4", lambda: synth.generate("sines3d", (300, 32, 256))),
    ("split_150", lambda: synth.generate("nyx_v", (150, 16, 512))),      # two CTAs per plane
    ("unsplit_600", lambda: synth.generate("nyx_rho", (600, 8, 512))),   # one CTA per plane
    ("odd_tpp", lambda: synth.generate("hurr_u", (160, 24, 256))),       # 3 tiles per plane
]


@pytest.mark.parametrize("name,gen", FUSED_Y, ids=[s[0] for s in FUSED_Y])
@pytest.mark.parametrize("rel", [1e-2, 1e-4])
def test_fused_y_decode_parity(name, gen, rel):
    _check_full(gen(), O.REL, rel, f"{name}@{rel}")


def test_fused_y_decode_with_outliers():
    d = synth.generate("nyx_rho", (296, 8, 512)).copy()
    eb = float(d.max() - d.min()) * 1e-4
    rng = np.random.default_rng(11)
    idx = rng.choice(d.size, 300, replace=False)
    d.reshape(-1)[idx] += np.float32(50.0) * np.float32(d.max() - d.min())
    ref = _check_full(d, O.ABS, eb, "fused_y_outliers")
    assert int.from_bytes(ref[96:104].tobytes(), "little") > 0      # delta outliers present
    st, qref = O.decode_q(ref, d.size)
    assert st == O.OK
    q = fz.debug_decode_q(torch.from_numpy(ref).to(DEV), d.shape)
    assert np.array_equal(q.cpu().numpy(), qref)


def test_host_header_decompress_matches():
    """fz_last_header returns the stream's own header bytes, and fz_decompress_hdr (no
    blocking header read) decodes bit-identically to fz_decompress."""
    import ctypes as C
    d = synth.generate("nyx_v", (300, 8, 512))
    codec = fz.Codec(d.shape, DEV)
    buf, size = codec.compress(torch.from_numpy(d).to(DEV), fz.REL, 1e-3)
    assert bytes(codec.hdr) == buf[:128].cpu().numpy().tobytes()
    a = codec.decompress(buf)                                     # header from the host copy
    b = torch.empty_like(a)
    st = fz.lib().fz_decompress(C.c_void_p(buf.data_ptr()), size, C.c_void_p(b.data_ptr()), d.size,
                                C.c_void_p(codec.dwork.data_ptr()), codec.dwork.numel(), None)
    assert st == fz.OK
    assert torch.equal(a.view(torch.int32), b.view(torch.int32))
    # asynchronous form: same result once fz_decompress_result returns OK
    c = torch.full_like(a, float("nan"))
    codec.decompress(buf, out=c, sync=False)
    codec.result()
    assert torch.equal(a.view(torch.int32), c.view(torch.int32))
    # a flipped flag bit makes popcount(flags) disagree with nnz: reported by the result call
    bad = buf.clone()
    bad[200] ^= 1
    codec.out[:size].copy_(bad)
    codec.decompress(codec.out[:size], out=c, sync=False)
    with pytest.raises(fz.FZError) as e:
        codec.result()
    assert e.value.status == fz.ERR_CORRUPT


def test_generic_vector_kernel_parity(monkeypatch):
    """Variant 16 (fz_debug_set_variant) routes compression through the generic padded-halo kernel (k_compress<NDIM,
    VEC>) instead of the warp-specialized one; its stream must be byte-identical too."""
    fz.debug_set_variant(16)
    try:
        for d in (synth.generate("nyx_v", (24, 40, 64)), synth.generate("cesm_t", (90, 256)),
                  synth.adversarial("spike", 30000)):
            _check_full(d, O.REL, 1e-3, f"generic{d.shape}")
    finally:
        fz.debug_set_variant(0)


ASYNC_SHAPES = [
    ("plane", lambda: synth.generate("nyx_v", (296, 8, 512))),         # k_decode_planes
    ("tiles3d", lambda: synth.generate("hurr_u", (20, 50, 52))),       # k_decode_tiles + walks
    ("ragged3d", lambda: synth.generate("sines3d", (33, 47, 61))),     # generic compressor (nx % 4)
    ("cesm2d", lambda: synth.generate("cesm_t", (180, 360))),          # chunked y scan
    ("wide2d", lambda: synth.generate("cesm_t", (7, 5000))),
    ("noise1d", lambda: synth.adversarial("noise", 10007)),            # x carries + 1-D dequant
    ("spike1d", lambda: synth.adversarial("spike", 50000)),            # delta outliers
    ("offset1d", lambda: synth.adversarial("offset", 30000)),          # staging overflow (reported)
    ("vout1d", lambda: synth.adversarial("offset", 1000)),             # value outliers below the cap
]


@pytest.mark.parametrize("name,gen", ASYNC_SHAPES, ids=[a[0] for a in ASYNC_SHAPES])
def test_async_pipeline_parity(name, gen):
    """fz_compress_async + fz_decompress_async (no host round trip, header parsed on the
    device): byte-identical stream and bit-identical field vs the oracle."""
    d = gen()
    mode, eb = (O.REL, 1e-6) if name in ("offset1d", "vout1d") else ((O.ABS, 1e-3) if name == "spike1d" else (O.REL, 1e-3))
    st, ref = O.compress(d, mode, eb)
    assert st == O.OK
    codec = fz.Codec(d.shape, DEV)
    buf, _ = codec.compress(torch.from_numpy(np.ascontiguousarray(d)).to(DEV), mode, eb, sync=False)
    if name == "offset1d":
        # more value outliers than the staging area holds: the asynchronous path cannot run the
        # rescan pass and says so (the synchronous fz_compress handles it)
        with pytest.raises(fz.FZError) as e:
            codec.compress_result()
        assert e.value.status == fz.ERR_WORKSPACE
        return
    xh = codec.decompress_device(buf)
    size = codec.compress_result()
    codec.result()
    _assert_stream_equal(buf[:size].cpu().numpy(), ref, name)
    st, xref = O.decompress(ref, d.size)
    assert np.array_equal(xh.cpu().numpy().reshape(-1).view(np.uint32), xref.view(np.uint32))


def test_async_decompress_rejects_bad_headers():
    d = synth.generate("nyx_v", (24, 30, 32))
    codec = fz.Codec(d.shape, DEV)
    buf, size = codec.compress(torch.from_numpy(d).to(DEV), fz.REL, 1e-3)
    good = buf.clone()
    for off, val in ((0, 0x00), (40, 0x07), (88, 0x7F), (67, 0x80)):   # magic, N, nnz, sign of w
        bad = good.clone()
        bad[off] = val if bad[off].item() != val else (val ^ 1)
        codec.decompress_device(bad)
        with pytest.raises(fz.FZError) as e:
            codec.result()
        assert e.value.status == fz.ERR_CORRUPT
    codec.decompress_device(good)
    codec.result()


# z-band two-pass compressor (3-D, P % 2048 == 0): chunk remainders, the smallest nz, a chunk
# boundary inside a field with outliers, and equality with the single-kernel path.
ZB_SHAPES = [
    ("nz2", lambda: synth.generate("nyx_v", (2, 32, 64))),
    ("nz17", lambda: synth.generate("sines3d", (17, 16, 128))),     # one full chunk + 1 plane
    ("nz33_r4", lambda: synth.generate("hurr_u", (33, 8, 512))),
    ("nz40_tpp3", lambda: synth.generate("rtm", (40, 24, 256))),    # 3 tiles per plane
]


@pytest.mark.parametrize("name,gen", ZB_SHAPES, ids=[z[0] for z in ZB_SHAPES])
def test_zband_compressor_parity(name, gen):
    _check_full(gen(), O.REL, 1e-3, name)


def test_zband_with_outliers_and_single_kernel_equality(monkeypatch):
    d = synth.generate("nyx_rho", (36, 16, 256)).copy()
    eb = float(d.max() - d.min()) * 1e-4
    rng = np.random.default_rng(5)
    d.reshape(-1)[rng.choice(d.size, 400, replace=False)] += np.float32(80.0) * np.float32(d.max() - d.min())
    ref = _check_full(d, O.ABS, eb, "zband_outliers")
    assert int.from_bytes(ref[96:104].tobytes(), "little") > 0
    fz.debug_set_variant(1024)                     # warp-specialized single kernel instead
    try:
        got, _, _ = _gpu_stream(d, O.ABS, eb)
    finally:
        fz.debug_set_variant(0)
    _assert_stream_equal(got, ref, "single_kernel")


# f1 chunk-local Lorenzo: chunks of 16 planes x one whole-row tile,
# bit-exact against the oracle's chunked compressor and decoder; partial last chunks, every
# rows-per-tile count R = 2048 / nx, outliers, and each decode entry point.
CL_SHAPES = [
    ("c1_64", lambda: synth.generate("sines3d", (64, 64, 64))),
    ("nz40_r4", lambda: synth.generate("nyx_v", (40, 16, 512))),       # 16 + 16 + 8 planes
    ("nz33_r16", lambda: synth.generate("hurr_u", (33, 32, 128))),     # 2 tiles per plane
    ("nz18_r8", lambda: synth.generate("rtm", (18, 16, 256))),
    ("nz17_r2", lambda: synth.generate("sines3d", (17, 2, 1024))),     # 1 tile per plane
    ("nz3_r1", lambda: synth.generate("nyx_rho", (3, 1, 2048))),
]


@pytest.mark.parametrize("name,gen", CL_SHAPES, ids=[c[0] for c in CL_SHAPES])
@pytest.mark.parametrize("rel", [1e-2, 1e-4])
def test_chunk_local_parity(name, gen, rel):
    d = gen()
    st, ref = O.compress_chunked(d, O.REL, rel, 16, 2048 // d.shape[2])
    assert st == O.OK
    got, xh, codec = _gpu_stream(d, O.REL | fz.CHUNK_LOCAL, rel)
    _assert_stream_equal(got, ref, name)
    st, xref = O.decompress(ref, d.size)
    assert st == O.OK
    assert np.array_equal(xh.view(np.uint32), xref.view(np.uint32)), name
    # decoded from a foreign buffer (blocking header read) and into integer codes
    buf = torch.from_numpy(ref).to(DEV)
    x2 = fz.decompress(buf).cpu().numpy().reshape(-1)
    assert np.array_equal(x2.view(np.uint32), xref.view(np.uint32))
    st, qref = O.decode_q(ref, d.size)
    assert np.array_equal(fz.debug_decode_q(buf, d.shape).cpu().numpy().reshape(-1), qref)


def test_chunk_local_outliers_async_and_errors():
    d = synth.generate("nyx_rho", (36, 16, 256)).copy()
    eb = float(d.max() - d.min()) * 1e-4
    rng = np.random.default_rng(7)
    d.reshape(-1)[rng.choice(d.size, 300, replace=False)] += np.float32(80.0) * np.float32(d.max() - d.min())
    st, ref = O.compress_chunked(d, O.ABS, eb, 16, 8)
    assert st == O.OK and int.from_bytes(ref[96:104].tobytes(), "little") > 0
    got, xh, codec = _gpu_stream(d, O.ABS | fz.CHUNK_LOCAL, eb)
    _assert_stream_equal(got, ref, "cl_outliers")
    st, xref = O.decompress(ref, d.size)
    assert np.array_equal(xh.view(np.uint32), xref.view(np.uint32))
    # asynchronous compress + host-header asynchronous decompress
    field = torch.from_numpy(d).to(DEV)
    codec.compress(field, O.ABS | fz.CHUNK_LOCAL, eb, sync=False)
    size = codec.compress_result()
    assert size == ref.size
    assert np.array_equal(codec.out[:size].cpu().numpy(), ref)
    # the device-parsed asynchronous decoder rejects chunk-local streams
    buf = torch.from_numpy(ref).to(DEV)
    codec.decompress_device(buf)
    with pytest.raises(fz.FZError) as e:
        codec.result()
    assert e.value.status == fz.ERR_ARG
    # shapes without whole-row tiles are refused
    bad = synth.generate("sines3d", (20, 10, 100))
    with pytest.raises(fz.FZError) as e:
        _gpu_stream(bad, O.REL | fz.CHUNK_LOCAL, 1e-3)
    assert e.value.status == fz.ERR_ARG


@pytest.mark.parametrize("ranks", [1, 2, 3, 4])
def test_chunk_local_multirank_no_exchange_decode(ranks):
    """f1 across ranks: chunk-aligned slabs compress to the oracle's chunk-local stream byte
    for byte, and every rank decodes its slab alone (no carry exchange), bit-exact."""
    from paper_2304_12557_b200 import dist
    d = synth.generate("nyx_v", (64, 32, 128))
    st, ref = O.compress_chunked(d, O.REL, 1e-3, 16, 2048 // 128)
    assert st == O.OK
    out, xh = dist.roundtrip_chunk_local_single_process(d, fz.REL, 1e-3, ranks, DEV)
    _assert_stream_equal(out, ref, f"cl ranks={ranks}")
    st, xref = O.decompress(ref, d.size)
    assert np.array_equal(xh.view(np.uint32), xref.view(np.uint32))



def test_cuda_graph_step_matches_direct_calls():
    """The asynchronous compress + device-parsed decompress captured into a CUDA graph (the
    bench's timed step) produces the same stream and field as direct calls, replay after
    replay."""
    d = synth.generate("nyx_v", (48, 64, 128))
    field = torch.from_numpy(d).to(DEV)
    ref_buf, ref_size = fz.Codec(d.shape, DEV).compress(field, fz.REL, 1e-3)
    ref = ref_buf.cpu().numpy().copy()
    codec = fz.Codec(d.shape, DEV)
    out = torch.empty_like(field)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        codec.compress(field, fz.REL, 1e-3, sync=False, stream=s)
        codec.decompress_device(codec.out, out=out, stream=s)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            codec.compress(field, fz.REL, 1e-3, sync=False, stream=s)
            codec.decompress_device(codec.out, out=out, stream=s)
    torch.cuda.synchronize()
    st, xref = O.decompress(ref, d.size)
    for _ in range(3):
        codec.out.zero_()
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert codec.compress_result() == ref_size
        codec.result()
        _assert_stream_equal(codec.out[:ref_size].cpu().numpy(), ref, "graph")
        assert np.array_equal(out.cpu().numpy().reshape(-1).view(np.uint32), xref.view(np.uint32))


def test_row_walker_fallback_value_outliers_across_runs():
    """Row-walking compressor (nx % 128 == 0, ny % 16 == 0) in fallback mode (R2) with value
    outliers (R20: |q| >= 2^21) spread over every plane, on a field whose band runs are long
    enough that CTAs take seed steps and then reuse the seed's stage: the seed plane's outlier
    marks must not reach a later plane's outlier lists."""
    nz, ny, nx = 512, 32, 128
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    s = np.sin(0.02 * z + 0.03 * y + 0.025 * x + 1.0)
    d = (2.0 ** 21 * 1.000001 * s).astype(np.float32)   # |d| >= 2^21 - 1/2 on ~0.1 % of elements
    # (2112 value outliers, 16788 delta-outliers: both below the N/64 + 1024 staging size, so
    # the single-pass path -- not the rescan -- produces the stream)
    ref = _check_full(d, O.ABS, 0.5, "fallback-runs")
    info = fz.peek_header(ref[:128].tobytes())
    assert info.params.fallback == 1 and 0 < info.counts.n_value < d.size // 64


# Row-walking decoder (fz_dzr.cu): 3-D, nx in {128, 256, 512, 1024}, ny % 16 == 0 -- bands of
# 16 rows, chunks of 16 planes (ragged last chunk), several bands and chunks, CTAs taking more
# than one unit; checked against the oracle's sequential recurrence bit for bit.
DZR = [
    ("nx128", lambda: synth.generate("sines3d", (37, 48, 128))),
    ("nx256", lambda: synth.generate("nyx_rho", (33, 32, 256))),
    ("nx512", lambda: synth.generate("nyx_v", (40, 64, 512))),
    ("nx1024", lambda: synth.generate("hurr_u", (18, 16, 1024))),
    ("one_band", lambda: synth.generate("rtm", (70, 16, 512))),
    ("many_units", lambda: synth.generate("nyx_v", (160, 128, 256))),
    ("nz2", lambda: synth.generate("sines3d", (2, 32, 128))),
]


@pytest.mark.parametrize("name,gen", DZR, ids=[s[0] for s in DZR])
@pytest.mark.parametrize("rel", [1e-2, 1e-4])
def test_row_walking_decoder_parity(name, gen, rel):
    d = gen()
    ref = _check_full(d, O.REL, rel, f"dzr-{name}@{rel}")
    # the device-parsed asynchronous decode and the integer-code hook take the same kernels
    codec = fz.Codec(d.shape, DEV)
    buf = torch.from_numpy(ref).to(DEV)
    xh = codec.decompress_device(buf)
    codec.result()
    st, xref = O.decompress(ref, d.size)
    assert np.array_equal(xh.cpu().numpy().reshape(-1).view(np.uint32), xref.view(np.uint32))
    st, qref = O.decode_q(ref, d.size)
    assert np.array_equal(fz.debug_decode_q(buf, d.shape).cpu().numpy().reshape(-1), qref)


def test_row_walking_decoder_outliers_and_old_path_equal():
    """delta- and value-outliers through the row-walking decoder, and the same stream decoded by
    the tile decoder + z walk (variant bit 32768) gives the same bits."""
    d = synth.generate("nyx_rho", (50, 32, 512)).copy()
    eb = float(d.max() - d.min()) * 1e-4
    rng = np.random.default_rng(12)
    idx = rng.choice(d.size, 400, replace=False)
    d.reshape(-1)[idx] += np.float32(50.0) * np.float32(d.max() - d.min())
    ref = _check_full(d, O.ABS, eb, "dzr_outliers")
    assert int.from_bytes(ref[96:104].tobytes(), "little") > 0      # delta outliers present
    buf = torch.from_numpy(ref).to(DEV)
    a = fz.decompress(buf)
    fz.debug_set_variant(32768)
    try:
        b = fz.decompress(buf)
    finally:
        fz.debug_set_variant(0)
    assert np.array_equal(a.cpu().numpy().view(np.uint32), b.cpu().numpy().view(np.uint32))


# General row-walking decoder (fz_dzg.cu): 3-D, nx % 4 == 0, 64 <= nx <= 512, nz >= 256 (or >= 64
# with N >= 2^22),
# rows that do not tile (partial bands, planes not whole tiles) -- un-shuffled code field, then
# the carries' two passes.
DZG = [
    ("nx96", lambda: synth.generate("sines3d", (300, 20, 96))),
    ("nx500_band9", lambda: synth.generate("hurr_u", (260, 9, 500))),
    ("nx352", lambda: synth.generate("rtm", (256, 33, 352))),
    ("nx1000", lambda: synth.generate("nyx_v", (257, 17, 1000))),
    # nz in [64, 256) with N >= 2^22 (c3-like), and a mostly-zero field (QSNOW: exact zeros,
    # the zero-tile / zero-warp fast paths next to dense warps)
    ("nz72_mid", lambda: synth.generate("hurr_u", (72, 120, 500))),
    ("qsnow_zero_paths", lambda: synth.generate("hurr_qsnow", (72, 120, 500))),
]


@pytest.mark.parametrize("name,gen", DZG, ids=[s[0] for s in DZG])
@pytest.mark.parametrize("rel", [1e-2, 1e-4])
def test_general_row_walking_decoder_parity(name, gen, rel):
    d = gen()
    ref = _check_full(d, O.REL, rel, f"dzg-{name}@{rel}")
    codec = fz.Codec(d.shape, DEV)
    buf = torch.from_numpy(ref).to(DEV)
    xh = codec.decompress_device(buf)
    codec.result()
    st, xr = O.decompress(ref, d.size)
    assert np.array_equal(xh.cpu().numpy().reshape(-1).view(np.uint32), xr.view(np.uint32))
    st, qref = O.decode_q(ref, d.size)
    assert np.array_equal(fz.debug_decode_q(buf, d.shape).cpu().numpy().reshape(-1), qref)


def test_general_row_walking_decoder_outliers_and_old_path_equal():
    d = synth.generate("hurr_u", (270, 12, 200)).copy()
    eb = float(d.max() - d.min()) * 1e-4
    rng = np.random.default_rng(13)
    idx = rng.choice(d.size, 500, replace=False)
    d.reshape(-1)[idx] += np.float32(50.0) * np.float32(d.max() - d.min())
    ref = _check_full(d, O.ABS, eb, "dzg_outliers")
    assert int.from_bytes(ref[96:104].tobytes(), "little") > 0      # delta outliers present
    buf = torch.from_numpy(ref).to(DEV)
    a = fz.decompress(buf)
    fz.debug_set_variant(32768)
    try:
        b = fz.decompress(buf)
    finally:
        fz.debug_set_variant(0)
    assert np.array_equal(a.cpu().numpy().view(np.uint32), b.cpu().numpy().view(np.uint32))
