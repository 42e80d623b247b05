"""Pins of the CPU oracle against things other than itself (no GPU needed).

Each test names the paper passage (P:n) or DESIGN.md reading (R#) it checks, and the
independent fact used: a closed form, a brute-force exact computation (fractions), a
numpy construction of the same definition, an invariant, or a hand-derived example.
"""
from __future__ import annotations

import json
import math
import os
import random
import struct
from fractions import Fraction

import numpy as np
import pytest

import oracle_lib as O
from paper_2304_12557_b200 import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def f32(x: float) -> float:
    return float(np.float32(x))


def f32bits(x: float) -> int:
    return struct.unpack("<I", struct.pack("<f", x))[0]


# --------------------------------------------------------------------------------------
# C0 / Appendix A parameters
# --------------------------------------------------------------------------------------

def test_params_w1_closed_form():
    """W1: M = 3.1 -> U = 2^-21, w = 1 - 2^-21, r = 1 + 2^-21."""
    g = json.load(open(os.path.join(GOLDEN, "w1.json")))
    st, p = O.derive_params(-0.5, f32(3.1), O.ABS, 0.5)
    assert st == O.OK
    assert f32bits(p.w) == int(g["w_bits"], 16)
    assert f32bits(p.r) == int(g["r_bits"], 16)
    assert p.w == 1 - 2.0 ** -21 and p.fallback == 0 and p.eb_abs == 0.5


def test_params_rel_range_and_constant_field():
    """eb_abs = REL * (max - min); constant field keeps eb (reading R4)."""
    st, p = O.derive_params(0.0, 2.0, O.REL, 1e-2)
    assert st == O.OK and p.eb_abs == 1e-2 * 2.0
    st, p = O.derive_params(5.0, 5.0, O.REL, 1e-3)
    assert st == O.OK and p.eb_abs == 1e-3


def test_params_margin_bounds():
    """w is the largest float <= 2 eb_abs - U (U = ulp of the binade above M), checked
    with exact rational arithmetic; fallback triggers exactly when M/w >= 2^21 - 1."""
    rnd = random.Random(11)
    for _ in range(400):
        M = f32(10 ** rnd.uniform(-6, 6))
        eb = 10 ** rnd.uniform(-8, 2)
        st, p = O.derive_params(-M, M, O.ABS, eb)
        if st != O.OK:
            assert st == O.ERR_EB_TOO_SMALL
            continue
        m, e = math.frexp(M)
        U = Fraction(2) ** (e - 23)
        target = 2 * Fraction(eb) - U
        w = Fraction(p.w)
        if not p.fallback:
            assert w <= target
            nxt = Fraction(float(np.nextafter(np.float32(p.w), np.float32(np.inf))))
            assert nxt > target
            assert Fraction(M) / w < 2 ** 21
        else:
            assert w <= 2 * Fraction(eb)


def test_params_errors():
    assert O.derive_params(0.0, 1.0, O.ABS, 0.0)[0] == O.ERR_ARG
    assert O.derive_params(0.0, 1.0, O.ABS, -1.0)[0] == O.ERR_ARG
    assert O.derive_params(0.0, 1.0, O.ABS, float("nan"))[0] == O.ERR_ARG
    assert O.derive_params(0.0, 1.0, O.ABS, 1e-50)[0] == O.ERR_EB_TOO_SMALL


def test_range_canonical_zero_and_nonfinite():
    st, mn, mx, bad = O.field_range(np.array([-0.0, 0.0, -0.0], np.float32))
    assert st == O.OK and f32bits(mn) == 0 and f32bits(mx) == 0
    st, *_rest, bad = O.field_range(np.array([1, 2, np.nan, np.inf], np.float32))
    assert st == O.ERR_NONFINITE and bad == 2


# --------------------------------------------------------------------------------------
# C1 prequantization: brute force with exact rationals
# --------------------------------------------------------------------------------------

def _exact_expect(d: float, p) -> tuple[int, int]:
    w = Fraction(p.w)
    qe = round(Fraction(d) / w)            # Python rounds Fractions half-to-even (R1)
    if abs(qe) >= 2 ** 21:
        return 0, 1
    xh = np.float32(np.float32(qe) * np.float32(p.w))   # fl32(fl32(q) * w)  (R21)
    viol = abs(Fraction(float(xh)) - Fraction(d)) > Fraction(p.eb_abs)
    return qe, int(viol)


@pytest.mark.parametrize("mode,eb,lo,hi", [
    (O.ABS, 0.5, -4.0, 4.0),
    (O.REL, 1e-3, -1.0, 1.0),
    (O.REL, 1e-4, 240.0, 290.0),     # offset field: exercises the ulp margin
    (O.REL, 1e-6, 1e6 - 1, 1e6 + 1),  # forces fallback mode (R2)
    (O.ABS, 1e-30, -1e-20, 1e-20),
])
def test_prequantize_bruteforce(mode, eb, lo, hi):
    rnd = random.Random(hash((mode, eb)) & 0xFFFF)
    vals = [f32(rnd.uniform(lo, hi)) for _ in range(3000)]
    mn, mx = min(vals), max(vals)
    st, p = O.derive_params(mn, mx, mode, eb)
    assert st == O.OK
    # add values within +-3 ulps of bin edges (q + 1/2) w
    for k in range(-40, 40):
        edge = (k + 0.5) * p.w
        x = np.float32(edge)
        for _ in range(3):
            if mn <= float(x) <= mx:
                vals.append(float(x))
            x = np.nextafter(x, np.float32(np.inf))
    q, flag = O.prequantize(np.array(vals, np.float32), p)
    for i, d in enumerate(vals):
        qe, fe = _exact_expect(d, p)
        assert (int(q[i]), int(flag[i])) == (qe, fe), (d, p.w)
    if not p.fallback:
        assert flag.sum() == 0   # Appendix A: the bound holds by construction in margin mode


def test_prequantize_exact_ties_to_even():
    """W2: exact half-integer multiples of w round to the even neighbour (R1)."""
    st, p = O.derive_params(-3.5, 3.5, O.ABS, 0.5)
    w = p.w
    assert w == 1 - 2.0 ** -21
    ties = [0.5, 1.5, 2.5, 3.5]
    for t in ties:
        for s in (1.0, -1.0):
            d = f32(s * t * w)
            assert Fraction(d) == Fraction(s * t) * Fraction(w)  # really a tie
            q, f = O.prequantize(np.array([d], np.float32), p)
            expect = s * (2 * round(t / 2)) if t != 0.5 else 0.0
            assert int(q[0]) == int(round(Fraction(s * t))) == int(expect)
            assert f[0] == 0


def test_prequantize_sign_symmetry():
    """prequantize(-d) = -prequantize(d) for the symmetric tie rule."""
    rnd = random.Random(5)
    vals = np.array([f32(rnd.uniform(-100, 100)) for _ in range(2000)], np.float32)
    st, p = O.derive_params(-100.0, 100.0, O.ABS, 0.01)
    q1, _ = O.prequantize(vals, p)
    q2, _ = O.prequantize(-vals, p)
    assert np.array_equal(q1, -q2)


# --------------------------------------------------------------------------------------
# C2 Lorenzo: closed form = repeated numpy.diff with a zero prepended
# --------------------------------------------------------------------------------------

def _np_lorenzo(q: np.ndarray) -> np.ndarray:
    v = q.astype(np.int64)
    for ax in range(q.ndim):
        v = np.diff(v, axis=ax, prepend=0)
    return v.astype(np.int32)      # wrap modulo 2^32 (R6)


def test_lorenzo_spec_examples():
    assert O.lorenzo(np.array([3, 3, 3, 3], np.int32)).tolist() == [3, 0, 0, 0]
    assert O.lorenzo(np.ones((2, 2), np.int32)).tolist() == [[1, 0], [0, 0]]
    ramp = np.arange(10, dtype=np.int32)
    assert O.lorenzo(ramp).tolist() == [0] + [1] * 9


@pytest.mark.parametrize("shape", [(1000,), (17, 33), (5, 7, 9), (1, 1, 64), (3, 1, 5)])
def test_lorenzo_closed_form(shape):
    rng = np.random.default_rng(3)
    q = rng.integers(-2 ** 31, 2 ** 31, size=shape, dtype=np.int64).astype(np.int32)
    assert np.array_equal(O.lorenzo(q), _np_lorenzo(q))
    q = rng.integers(-50, 50, size=shape).astype(np.int32)
    d = O.lorenzo(q)
    inv = d.astype(np.int64)
    for ax in range(q.ndim):
        inv = np.cumsum(inv, axis=ax)
    assert np.array_equal(inv.astype(np.int32), q)   # inverse = per-axis prefix sums


def test_lorenzo_annihilates_lower_dim_functions():
    """delta == 0 in the interior for q(z,y,x) = f(y,x) + g(z,x) + h(z,y)."""
    rng = np.random.default_rng(9)
    nz, ny, nx = 6, 7, 8
    f = rng.integers(-99, 99, (1, ny, nx))
    g = rng.integers(-99, 99, (nz, 1, nx))
    h = rng.integers(-99, 99, (nz, ny, 1))
    q = (f + g + h).astype(np.int32)
    d = O.lorenzo(q)
    assert not d[1:, 1:, 1:].any()


# --------------------------------------------------------------------------------------
# f1 chunk-local Lorenzo ("chunked data blocks can be compressed
# independently"): each chunk's residuals are the field-global closed form applied to the
# chunk alone, so chunks are independent (pinned with numpy, not with the oracle itself).
# --------------------------------------------------------------------------------------

def _np_lorenzo_chunked(q: np.ndarray, cz: int, cy: int) -> np.ndarray:
    out = np.empty_like(q)
    for z0 in range(0, q.shape[0], cz):
        for y0 in range(0, q.shape[1], cy):
            sub = q[z0:z0 + cz, y0:y0 + cy, :]
            out[z0:z0 + cz, y0:y0 + cy, :] = _np_lorenzo(sub)
    return out


@pytest.mark.parametrize("shape,cz,cy", [((35, 12, 8), 16, 4), ((16, 8, 64), 16, 32), ((7, 9, 5), 3, 2),
                                         ((5, 6, 7), 64, 64), ((33, 64, 64), 16, 32)])
def test_lorenzo_chunked_closed_form(shape, cz, cy):
    rng = np.random.default_rng(11)
    q = rng.integers(-2 ** 31, 2 ** 31, size=shape, dtype=np.int64).astype(np.int32)
    assert np.array_equal(O.lorenzo_chunked(q, cz, cy), _np_lorenzo_chunked(q, cz, cy))
    if cz >= shape[0] and cy >= shape[1]:   # one chunk: the field-global predictor
        assert np.array_equal(O.lorenzo_chunked(q, cz, cy), O.lorenzo(q))


def test_chunked_stream_roundtrip_and_independence():
    """Chunk-local stream: bound on every element, header bit 2 + chunk dims, and the codes
    of each chunk equal the global-mode codes of that chunk compressed as its own field
    with the same parameters (ABS: parameters do not depend on the rest of the field)."""
    from paper_2304_12557_b200 import synth
    d = synth.generate("sines3d", (40, 64, 64))
    cz, cy = 16, 32
    st, buf = O.compress_chunked(d, O.ABS, 1e-3, cz, cy)
    assert st == O.OK
    assert int.from_bytes(buf[6:8].tobytes(), "little") & 4
    assert int.from_bytes(buf[10:12].tobytes(), "little") == cz
    assert int.from_bytes(buf[12:14].tobytes(), "little") == cy
    st, x = O.decompress(buf, d.size)
    assert st == O.OK
    assert np.all(np.abs(x.astype(np.float64) - d.reshape(-1).astype(np.float64)) <= 1e-3)
    p = O.params_for(d, O.ABS, 1e-3)
    q, _ = O.prequantize(d[:cz, :cy], p)
    qz, _ = O.prequantize(d[cz:2 * cz, cy:2 * cy], p)
    full = O.lorenzo_chunked(O.prequantize(d, p)[0].reshape(d.shape), cz, cy)
    assert np.array_equal(full[:cz, :cy], _np_lorenzo(q.reshape(cz, cy, 64)))
    assert np.array_equal(full[cz:2 * cz, cy:2 * cy], _np_lorenzo(qz.reshape(cz, cy, 64)))
    st, qd = O.decode_q(buf, d.size)
    assert st == O.OK and np.array_equal(qd, O.prequantize(d, p)[0])


def test_chunked_single_chunk_equals_global_stream():
    """When one chunk covers the field, the stream equals the global one except the header's
    chunk fields."""
    from paper_2304_12557_b200 import synth
    d = synth.generate("sines3d", (8, 32, 64))
    st, g = O.compress(d, O.REL, 1e-3)
    st2, c = O.compress_chunked(d, O.REL, 1e-3, 8, 32)
    assert st == st2 == O.OK and g.size == c.size
    c2 = c.copy()
    c2[6] &= 0xFB
    c2[10:14] = 0
    assert np.array_equal(g, c2)


# --------------------------------------------------------------------------------------
# C3 codes
# --------------------------------------------------------------------------------------

def test_pack_examples_and_exhaustive_roundtrip():
    assert O.pack(0) == (0x0000, 0)
    assert O.pack(-3) == (0x8003, 0)
    assert O.pack(32767) == (0x7FFF, 0)
    assert O.pack(32768) == (0, 1) and O.pack(-32768) == (0, 1)
    assert O.unpack(0x8000) == 0              # R8
    for v in range(-32767, 32768, 1):
        c, o = O.pack(v)
        assert o == 0 and O.unpack(c) == v
        assert (c >> 15) == (1 if v < 0 else 0) and (c & 0x7FFF) == abs(v)


# --------------------------------------------------------------------------------------
# C5 bitshuffle and C6 flags: numpy constructions of the definitions
# --------------------------------------------------------------------------------------

def _np_shuffle(A: np.ndarray) -> np.ndarray:
    bits = (A.reshape(32, 32)[:, :, None].astype(np.uint64) >> np.arange(32, dtype=np.uint64)) & 1
    # bits[c, j, r]; O[r, c] = sum_j bits[c, j, r] << j
    Ob = bits.transpose(2, 0, 1)
    return (Ob << np.arange(32, dtype=np.uint64)).sum(axis=2).astype(np.uint32).reshape(1024)


def _np_flags(Ot: np.ndarray):
    nz = Ot.reshape(256, 4).any(axis=1)
    F = np.zeros(8, np.uint32)
    for b in np.nonzero(nz)[0]:
        F[b // 32] |= np.uint32(1 << (b % 32))
    return F, int(nz.sum())


def _tiles(n, seed=1):
    rng = np.random.default_rng(seed)
    out = [np.zeros(1024, np.uint32), np.full(1024, 0xFFFFFFFF, np.uint32)]
    for k in range(n):
        A = rng.integers(0, 2 ** 32, 1024, dtype=np.uint64).astype(np.uint32)
        if k % 2:
            A &= rng.integers(0, 2 ** 32, 1024, dtype=np.uint64).astype(np.uint32) & np.uint32(0x00070007)
        out.append(A)
    return out


def test_shuffle_example():
    A = np.zeros(1024, np.uint32)
    A[32 * 5 + 7] = 1 << 13
    O_ = O.shuffle_tile(A)
    expect = np.zeros(1024, np.uint32)
    expect[32 * 13 + 5] = 1 << 7
    assert np.array_equal(O_, expect)


def test_shuffle_matches_numpy_and_inverts():
    for A in _tiles(60):
        Ot = O.shuffle_tile(A)
        assert np.array_equal(Ot, _np_shuffle(A))
        assert np.array_equal(O.unshuffle_tile(Ot), A)
        # popcount preserved; shuffle^3 = identity (SURVEY App. B identity)
        assert np.unpackbits(Ot.view(np.uint8)).sum() == np.unpackbits(A.view(np.uint8)).sum()
        assert np.array_equal(O.shuffle_tile(O.shuffle_tile(Ot)), A)


def test_flags_examples_and_numpy():
    Ot = np.zeros(1024, np.uint32)
    Ot[7] = 5
    F, nnz = O.flags_tile(Ot)                       # word 7 -> block 1
    assert F.tolist() == [2, 0, 0, 0, 0, 0, 0, 0] and nnz == 1
    F, nnz = O.flags_tile(np.full(1024, 1, np.uint32))
    assert F.tolist() == [0xFFFFFFFF] * 8 and nnz == 256
    for A in _tiles(20, seed=4):
        Ot = O.shuffle_tile(A)
        F, nnz = O.flags_tile(Ot)
        F2, nnz2 = _np_flags(Ot)
        assert np.array_equal(F, F2) and nnz == nnz2
        # OR-reduction identity: block (r, x) nonzero iff bit r of OR(words 128x..128x+127)
        g = [int(np.bitwise_or.reduce(A[128 * x:128 * x + 128])) for x in range(8)]
        for b in range(256):
            r, x = divmod(b, 8)
            assert bool((F[b // 32] >> (b % 32)) & 1) == bool((g[x] >> r) & 1)


# --------------------------------------------------------------------------------------
# Whole stream: independent numpy assembly of C4-C9 from the codes; golden W1; size law
# --------------------------------------------------------------------------------------

HDR = 128


def _parse_header(buf: np.ndarray) -> dict:
    b = buf.tobytes()
    h = {"magic": b[0:4], "version": struct.unpack_from("<H", b, 4)[0],
         "flags": struct.unpack_from("<H", b, 6)[0], "ndim": b[8],
         "dims": struct.unpack_from("<3Q", b, 16), "n": struct.unpack_from("<Q", b, 40)[0],
         "eb_input": struct.unpack_from("<d", b, 48)[0], "eb_abs": struct.unpack_from("<d", b, 56)[0],
         "w": struct.unpack_from("<f", b, 64)[0], "r": struct.unpack_from("<f", b, 68)[0],
         "min": struct.unpack_from("<f", b, 72)[0], "max": struct.unpack_from("<f", b, 76)[0]}
    h["T"], h["nnz"], h["nd"], h["nv"], h["total"] = struct.unpack_from("<5Q", b, 80)
    return h


def _np_assemble(codes: np.ndarray, didx, dval, vidx, vbits) -> bytes:
    """C4-C9 written independently with numpy from the codes and outlier lists."""
    n = codes.size
    T = -(-n // 2048)
    c = np.zeros(T * 2048, np.uint32)
    c[:n] = codes
    words = (c[0::2] | (c[1::2] << 16)).astype(np.uint32).reshape(T, 1024)
    flags, payload = [], []
    for t in range(T):
        Ot = _np_shuffle(words[t])
        F, _ = _np_flags(Ot)
        flags.append(F)
        blocks = Ot.reshape(256, 4)
        payload.append(blocks[blocks.any(axis=1)])
    fl = np.concatenate(flags).astype("<u4").tobytes()
    pl = np.concatenate(payload).astype("<u4").tobytes() if payload else b""
    ds = np.stack([didx, dval.view(np.uint32)], axis=1).astype("<u4").tobytes() if len(didx) else b""
    vs = np.stack([vidx, vbits], axis=1).astype("<u4").tobytes() if len(vidx) else b""
    return fl + pl + ds + vs


def test_w1_golden_stream():
    g = json.load(open(os.path.join(GOLDEN, "w1.json")))
    d = np.array(g["d"], np.float32)
    st, buf = O.compress(d, O.ABS, g["eb"])
    assert st == O.OK and buf.size == g["size"] == 224
    h = _parse_header(buf)
    assert h["magic"] == b"FZB2" and h["T"] == 1 and h["nnz"] == 4 and h["nd"] == 0 and h["nv"] == 0
    assert f32bits(h["w"]) == int(g["w_bits"], 16)
    flags = np.frombuffer(buf[HDR:HDR + 32].tobytes(), "<u4")
    assert flags.tolist() == g["flags"]
    pay = np.frombuffer(buf[HDR + 32:].tobytes(), "<u4").reshape(-1, 4)
    assert pay.tolist() == g["payload"]
    p = O.params_for(d, O.ABS, 0.5)
    codes, *_ = O.quantize_field(d, p)
    assert codes.tolist() == g["codes"]
    st, xh = O.decompress(buf, 4)
    assert [hex(f32bits(float(v))) for v in xh] == g["xhat_bits"]


def _small_fields():
    return [
        ("sines3d", synth.generate("sines3d", (64, 64, 64))),
        ("cesm_t", synth.generate("cesm_t", (90, 180))),
        ("cesm_cld", synth.generate("cesm_cld", (90, 181))),
        ("hurr_qsnow", synth.generate("hurr_qsnow", (10, 50, 50))),
        ("hurr_u", synth.generate("hurr_u", (10, 50, 50))),
        ("nyx_rho", synth.generate("nyx_rho", (32, 32, 32))),
        ("nyx_v", synth.generate("nyx_v", (32, 32, 32))),
        ("rtm", synth.generate("rtm", (40, 40, 22))),
        ("qmc", synth.generate("qmc", (40, 9, 9))),
        ("noise1d", synth.adversarial("noise", 5000)),
        ("spike1d", synth.adversarial("spike", 4099)),
    ]


@pytest.mark.parametrize("rel", [1e-2, 1e-3, 1e-4])
def test_stream_matches_numpy_assembly_and_bound(rel):
    for name, d in _small_fields():
        p = O.params_for(d, O.REL, rel)
        codes, didx, dval, vidx, vbits = O.quantize_field(d, p)
        st, buf = O.compress(d, O.REL, rel)
        assert st == O.OK
        h = _parse_header(buf)
        n = d.size
        T = -(-n // 2048)
        assert h["n"] == n and h["T"] == T and h["nd"] == len(didx) and h["nv"] == len(vidx)
        # size law
        assert buf.size == h["total"] == HDR + 32 * T + 16 * h["nnz"] + 8 * h["nd"] + 8 * h["nv"]
        assert buf[HDR:].tobytes() == _np_assemble(codes, didx, dval, vidx, vbits), name
        # codes == pack(lorenzo(prequantize(d))) via the numpy closed-form stencil
        q, _ = (O.prequantize(d, p) if n <= 5000 else (None, None))
        if q is not None:
            dl = _np_lorenzo(q.reshape(d.shape)).reshape(-1)
            exp = np.where(np.abs(dl.astype(np.int64)) > 32767, 0,
                           np.where(dl < 0, 0x8000 | np.abs(dl), dl)).astype(np.uint16)
            assert np.array_equal(codes, exp)
        # error bound on every element, exact in float64
        st, xh = O.decompress(buf, n)
        assert st == O.OK
        err = np.abs(xh.astype(np.float64) - d.reshape(-1).astype(np.float64))
        assert err.max() <= h["eb_abs"], name
        # round trip of the integer codes: decode_q == per-axis cumsum of unpacked deltas
        st, qd = O.decode_q(buf, n)
        dd = np.where(codes & 0x8000, -(codes & 0x7FFF).astype(np.int64), (codes & 0x7FFF).astype(np.int64))
        dd[didx] = dval
        inv = dd.reshape(d.shape)
        for ax in range(d.ndim):
            inv = np.cumsum(inv, axis=ax)
        assert np.array_equal(qd, inv.astype(np.int32).reshape(-1)), name


def test_all_zero_field_cap():
    """An all-zero block costs exactly one flag bit; all-zero tile 4096 -> 32 B."""
    for n in (1, 64, 2047, 2048, 2049, 1 << 20):
        st, buf = O.compress(np.zeros(n, np.float32), O.ABS, 1e-3)
        T = -(-n // 2048)
        assert st == O.OK and buf.size == HDR + 32 * T
    st, buf = O.compress(np.zeros(1 << 20, np.float32), O.ABS, 1e-3)
    cr = (4 << 20) / buf.size
    assert 250 <= cr <= 256


def test_ragged_tails_and_shapes():
    rng = np.random.default_rng(2)
    for shape in [(1,), (2047,), (2049,), (3, 700), (2, 3, 345), (1, 1, 1), (4097, 1)]:
        d = rng.normal(size=shape).astype(np.float32)
        st, buf = O.compress(d, O.REL, 1e-3)
        assert st == O.OK
        st, xh = O.decompress(buf, d.size)
        h = _parse_header(buf)
        assert st == O.OK and np.abs(xh - d.reshape(-1)).max() <= h["eb_abs"]


def test_delta_and_value_outliers():
    # spike: |delta| > 32767 -> delta outliers, still exactly invertible (R7)
    d = synth.adversarial("spike", 9000)
    st, buf = O.compress(d, O.ABS, 1e-3)
    h = _parse_header(buf)
    assert st == O.OK and h["nd"] > 0 and h["nv"] == 0
    st, xh = O.decompress(buf, d.size)
    assert np.abs(xh.astype(np.float64) - d).max() <= h["eb_abs"]
    # offset 1e6 at REL 1e-6: fallback mode; value outliers carry the raw bits (R2)
    d = synth.adversarial("offset", 6000)
    st, buf = O.compress(d, O.REL, 1e-6)
    h = _parse_header(buf)
    assert st == O.OK
    st, xh = O.decompress(buf, d.size)
    assert np.abs(xh.astype(np.float64) - d).max() <= h["eb_abs"]
    # a value that is not representable within eb at all: huge spread, tiny ABS bound
    d = np.array([1e30, -1e30, 1.0, 0.0] * 600, np.float32)
    st, buf = O.compress(d, O.ABS, 1e-3)
    h = _parse_header(buf)
    assert st == O.OK and h["flags"] & 2 and h["nv"] >= 1200
    st, xh = O.decompress(buf, d.size)
    assert np.abs(xh.astype(np.float64) - d).max() <= h["eb_abs"]


def test_nonfinite_rejected():
    d = np.ones(100, np.float32)
    d[37] = np.inf
    st, _ = O.compress(d, O.REL, 1e-3)
    assert st == O.ERR_NONFINITE


def test_idempotence_abs_pinned_params():
    """S:113 / reading R22: with w pinned, recompressing x-hat gives the same bytes."""
    d = synth.generate("sines3d", (16, 16, 16))
    p = O.params_for(d, O.ABS, 1e-2)
    st, b1 = O.compress(d, O.ABS, 1e-2, params=p)
    st, xh = O.decompress(b1, d.size)
    st, b2 = O.compress(xh.reshape(d.shape), O.ABS, 1e-2, params=p)
    assert np.array_equal(b1, b2)


def test_corrupt_streams_never_crash():
    d = synth.generate("cesm_t", (40, 80))
    st, buf = O.compress(d, O.REL, 1e-3)
    rnd = random.Random(1)
    bad_magic = buf.copy()
    bad_magic[0] ^= 1
    assert O.decompress(bad_magic, d.size)[0] == O.ERR_CORRUPT
    assert O.decompress(buf[:-1], d.size)[0] == O.ERR_CORRUPT
    for _ in range(300):
        m = buf.copy()
        for _k in range(rnd.randint(1, 4)):
            m[rnd.randrange(m.size)] ^= 1 << rnd.randrange(8)
        st, _ = O.decompress(m, d.size)
        assert st in (O.OK, O.ERR_CORRUPT, O.ERR_ARG)
