"""Quantizer edge cases: exact ties d = (k + 1/2) w, values within +-3 ulps of bin edges, the
worked examples W1 / W2, in ABS-margin, REL-margin and fallback modes (reading R1:
ties to even, R2: margin / fallback, R20: value outliers), and pins of the oracle's range pass
(C0) against numpy.

CPU tests pin the oracle against things other than itself (numpy min/max, the REL bound
computed here from the field, exact rationals, hand-derived golden streams).  GPU tests
(marked gpu) compare the CUDA path with the oracle on the same inputs: codes, both outlier
lists, the stream and the decoded field.
"""
from __future__ import annotations

import json
import os
import struct
from fractions import Fraction

import numpy as np
import pytest

import oracle_lib as O
from paper_2304_12557_b200 import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
HDR = 128


def _hdr(buf: np.ndarray) -> dict:
    b = buf.tobytes()
    h = {"flags": struct.unpack_from("<H", b, 6)[0], "eb_input": struct.unpack_from("<d", b, 48)[0],
         "eb_abs": struct.unpack_from("<d", b, 56)[0], "w": struct.unpack_from("<f", b, 64)[0],
         "min": struct.unpack_from("<f", b, 72)[0], "max": struct.unpack_from("<f", b, 76)[0]}
    h["T"], h["nnz"], h["nd"], h["nv"], h["total"] = struct.unpack_from("<5Q", b, 80)
    return h


def _fields():
    return [
        ("sines3d", synth.generate("sines3d", (64, 64, 64))),
        ("cesm_t", synth.generate("cesm_t", (90, 180))),            # offset field, all positive
        ("cesm_cld", synth.generate("cesm_cld", (90, 181))),        # plateaus at exactly 0 and 1
        ("hurr_qsnow", synth.generate("hurr_qsnow", (10, 50, 50))),  # mostly exact zeros
        ("hurr_u", synth.generate("hurr_u", (10, 50, 50))),
        ("nyx_rho", synth.generate("nyx_rho", (32, 32, 32))),        # log-normal, heavy tail
        ("nyx_v", synth.generate("nyx_v", (32, 32, 32))),
        ("rtm", synth.generate("rtm", (40, 40, 22))),
        ("qmc", synth.generate("qmc", (40, 9, 9))),
        ("noise1d", synth.adversarial("noise", 5000)),
        ("spike1d", synth.adversarial("spike", 4099)),
        ("offset1d", synth.adversarial("offset", 3000)),
        ("mixed_zeros", np.array([-0.0, 3.5, -2.25, 0.0, -0.0, 1e-30, -1e-30], np.float32)),
        ("neg_only", -np.abs(synth.adversarial("noise", 777)) - np.float32(2)),
        ("negzero_min", np.array([-0.0, 1.0, 2.0], np.float32)),
        ("negzero_max", np.array([-0.0, -1.0, -2.0], np.float32)),
    ]


# --------------------------------------------------------------------------------------
# C0: the oracle's range against numpy; the header's REL bound against the field
# --------------------------------------------------------------------------------------

@pytest.mark.parametrize("name,d", _fields(), ids=[f[0] for f in _fields()])
def test_oracle_range_matches_numpy(name, d):
    """fzo_range (min, max) == numpy's min / max of the same fp32 array; -0.0 reported as
    +0.0 (R18), so the header's min / max are unique bit patterns."""
    st, mn, mx, bad = O.field_range(d)
    assert st == O.OK and bad == -1
    assert mn == float(np.min(d)) and mx == float(np.max(d)), name
    for v in (mn, mx):
        assert struct.pack("<f", v) != struct.pack("<f", -0.0), name


@pytest.mark.parametrize("rel", [1e-2, 1e-3, 1e-4])
def test_header_rel_bound_from_field(rel):
    """P:320 "relative to the value range": the stream's eb_abs equals REL * (max - min) of
    the field, computed here in float64 from numpy's min / max (R4), and the decoded field
    stays within it on every element."""
    for name, d in _fields():
        st, buf = O.compress(d, O.REL, rel)
        assert st == O.OK
        h = _hdr(buf)
        lo, hi = float(np.min(d)), float(np.max(d))
        want = rel * (hi - lo) if hi != lo else rel
        assert h["eb_abs"] == want, name
        assert h["eb_input"] == rel and h["min"] == lo and h["max"] == hi, name
        assert h["flags"] & 1, name
        st, xh = O.decompress(buf, d.size)
        err = np.abs(xh.astype(np.float64) - d.reshape(-1).astype(np.float64))
        assert err.max() <= want, name


def test_header_abs_bound():
    d = synth.generate("hurr_u", (10, 50, 50))
    st, buf = O.compress(d, O.ABS, 0.03)
    h = _hdr(buf)
    assert h["eb_abs"] == 0.03 and h["eb_input"] == 0.03 and not (h["flags"] & 1)


# --------------------------------------------------------------------------------------
# Worked example W2 (ties to even), hand-derived golden stream
# --------------------------------------------------------------------------------------

def _w2():
    g = json.load(open(os.path.join(GOLDEN, "w2.json")))
    d = np.array([int(b, 16) for b in g["d_bits"]], np.uint32).view(np.float32)
    return g, d


def test_w2_inputs_are_exact_ties():
    g, d = _w2()
    w = Fraction(float(np.array([int(g["w_bits"], 16)], np.uint32).view(np.float32)[0]))
    assert w == 1 - Fraction(1, 2 ** 21)
    for v, k2 in zip(d[:4].tolist(), (3, 5, -5, 1)):
        assert Fraction(v) / w == Fraction(k2, 2)


def test_w2_golden_stream():
    g, d = _w2()
    st, buf = O.compress(d, O.ABS, 0.5)
    assert st == O.OK and buf.size == g["size"]
    h = _hdr(buf)
    assert h["T"] == 1 and h["nnz"] == 5 and h["nd"] == 0 and h["nv"] == 0
    assert struct.pack("<f", h["w"]) == struct.pack("<I", int(g["w_bits"], 16))
    assert np.frombuffer(buf[HDR:HDR + 32].tobytes(), "<u4").tolist() == g["flags"]
    assert np.frombuffer(buf[HDR + 32:].tobytes(), "<u4").reshape(-1, 4).tolist() == g["payload"]
    p = O.params_for(d, O.ABS, 0.5)
    q, vf = O.prequantize(d, p)
    assert q.tolist() == g["q"] and not vf.any()
    codes, *_ = O.quantize_field(d, p)
    assert codes.tolist() == g["codes"]
    st, xh = O.decompress(buf, d.size)
    assert [f"0x{v:08x}" for v in xh.view(np.uint32).tolist()] == g["xhat_bits"]


# --------------------------------------------------------------------------------------
# Edge-value fields (shared by the oracle pins and the GPU parity tests)
# --------------------------------------------------------------------------------------

def _ulp_steps(x: np.ndarray, steps: np.ndarray) -> np.ndarray:
    """x moved by `steps` ulps (nextafter repeated), elementwise, fp32."""
    out = x.copy()
    for s in range(1, 4):
        up = steps >= s
        dn = steps <= -s
        out[up] = np.nextafter(out[up], np.float32(np.inf))
        out[dn] = np.nextafter(out[dn], np.float32(-np.inf))
    return out


def edge_field(mode_name: str, shape, seed: int = 0):
    """A smooth field of bin indices k (so Lorenzo residuals stay small), every value put on a
    bin edge (k + 1/2) w or within +-3 ulps of it; w is a power of two so the edges are exact
    floats.  Returns (field, mode, eb, w).  The two extreme values fix the parameters:
      abs:      M = 1000 -> U = 2^-13, eb = (2^-4 + 2^-13)/2 -> w = 2^-4 (margin mode)
      rel:      min -1024, max 1024 -> U = 2^-12, REL = (2^-3 + 2^-12)/4096 -> w = 2^-3
      fallback: M = 2^21 -> ABS eb = 0.5 fails the margin test (M/w = 2^22) -> w = 1, and
                values with |q| >= 2^21 become value outliers."""
    n = int(np.prod(shape))
    rng = np.random.default_rng(seed)
    i = np.arange(n, dtype=np.float64)
    if mode_name == "abs":
        mode, eb, w, kmax, ext = O.ABS, (2.0 ** -4 + 2.0 ** -13) / 2, 2.0 ** -4, 14000, 1000.0
    elif mode_name == "rel":
        mode, eb, w, kmax, ext = O.REL, (2.0 ** -3 + 2.0 ** -12) / 4096, 2.0 ** -3, 7000, 1024.0
    else:
        mode, eb, w, kmax, ext = O.ABS, 0.5, 1.0, 5000, float(2 ** 21)
    k = np.floor(kmax * np.sin(i / 97.0) * np.cos(i / 1301.0))
    k += rng.integers(-2, 3, n)                       # small roughness: codes beyond 0/+-1
    d = ((k + 0.5) * w).astype(np.float32)            # exact ties
    steps = rng.integers(-3, 4, n)
    steps[rng.random(n) < 0.3] = 0                    # 30 % stay exact ties
    d = _ulp_steps(d, steps)
    if mode_name == "fallback":
        # values around |q| = 2^21 (the outlier threshold) and exact ties there
        m = max(8, n // 200)
        pos = rng.choice(n, m, replace=False)
        kk = (2 ** 21 + rng.integers(-4, 4, m)) * rng.choice([-1, 1], m)
        d[pos] = _ulp_steps((kk + 0.5 * rng.integers(0, 2, m)).astype(np.float32), rng.integers(-2, 3, m))
    d[0], d[-1] = np.float32(-ext), np.float32(ext)
    return d.reshape(shape), mode, eb, w


EDGE_MODES = ["abs", "rel", "fallback"]


@pytest.mark.parametrize("mode_name", EDGE_MODES)
def test_edge_field_params_and_oracle_bruteforce(mode_name):
    """The edge fields hit the intended mode and bin width, and the oracle's q equals the
    exact rational nearest integer (ties to even) on every element, with the bound."""
    d, mode, eb, w = edge_field(mode_name, (6000,), seed=1)
    p = O.params_for(d, mode, eb)
    assert p.w == w and bool(p.fallback) == (mode_name == "fallback")
    q, vf = O.prequantize(d, p)
    W = Fraction(p.w)
    ties = 0
    for v, qi, fi in zip(d.tolist(), q.tolist(), vf.tolist()):
        x = Fraction(v) / W
        qe = round(x)                         # half-to-even on Fractions (R1)
        ties += x.denominator == 2
        if abs(qe) >= 2 ** 21:
            assert fi == 1 and qi == 0
            continue
        assert qi == qe
        xh = float(np.float32(np.float32(qe) * np.float32(p.w)))
        assert bool(fi) == (abs(Fraction(xh) - Fraction(v)) > Fraction(p.eb_abs))
    assert ties > 1000


# --------------------------------------------------------------------------------------
# GPU parity on the same inputs
# --------------------------------------------------------------------------------------

def _torch():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2304_12557_b200 import fz
    return torch, fz


def _gpu_check(d, mode, eb, name):
    torch, fz = _torch()
    dev = "cuda:0"
    st, ref = O.compress(d, mode, eb)
    assert st == O.OK
    codec = fz.Codec(d.shape, dev)
    x = torch.from_numpy(np.ascontiguousarray(d)).to(dev)
    buf, size = codec.compress(x, mode, eb)
    got = buf[:size].cpu().numpy()
    assert size == ref.size and np.array_equal(got, ref), f"{name}: stream differs"
    xh = codec.decompress(buf).cpu().numpy().reshape(-1)
    st, xref = O.decompress(ref, d.size)
    assert np.array_equal(xh.view(np.uint32), xref.view(np.uint32)), f"{name}: x-hat differs"
    # C1-C3 stage hook: codes and both outlier lists
    p = O.params_for(d, mode, eb)
    codes, didx, dval, vidx, vbits = O.quantize_field(d, p)
    gp = fz.derive_params(p.mn, p.mx, mode, eb)
    c2, di2, dv2, vi2, vb2 = fz.debug_quantize(x, gp)
    assert np.array_equal(c2.cpu().numpy().view(np.uint16), codes), f"{name}: codes differ"
    assert np.array_equal(di2.cpu().numpy().view(np.uint32), didx)
    assert np.array_equal(dv2.cpu().numpy(), dval)
    assert np.array_equal(vi2.cpu().numpy().view(np.uint32), vidx)
    assert np.array_equal(vb2.cpu().numpy().view(np.uint32), vbits)
    return ref


# 1-D (single-pass kernel), a 3-D shape with whole tiles per plane (the c4 kernel family) and a
# 3-D shape whose planes straddle tiles
EDGE_SHAPES = [(70001,), (12, 32, 128), (9, 30, 52), (5, 64, 512)]


@pytest.mark.gpu
@pytest.mark.parametrize("shape", EDGE_SHAPES, ids=["x".join(map(str, s)) for s in EDGE_SHAPES])
@pytest.mark.parametrize("mode_name", EDGE_MODES)
def test_gpu_edge_values_parity(mode_name, shape):
    d, mode, eb, w = edge_field(mode_name, shape, seed=len(shape))
    ref = _gpu_check(d, mode, eb, f"{mode_name}{shape}")
    h = _hdr(ref)
    assert h["w"] == w and bool(h["flags"] & 2) == (mode_name == "fallback")
    if mode_name == "fallback":
        assert h["nv"] > 0


@pytest.mark.gpu
def test_gpu_worked_examples_w1_w2():
    g1 = json.load(open(os.path.join(GOLDEN, "w1.json")))
    d1 = np.array(g1["d"], np.float32)
    ref = _gpu_check(d1, O.ABS, 0.5, "W1")
    assert ref.size == g1["size"]
    g2, d2 = _w2()
    ref = _gpu_check(d2, O.ABS, 0.5, "W2")
    assert ref.size == g2["size"]
    # the same tie values tiled over a 3-D field with whole tiles per plane
    d3 = np.tile(d2[:4], 8 * 32 * 128 // 4).reshape(8, 32, 128)
    d3[0, 0, 0] = d2[4]
    _gpu_check(d3, O.ABS, 0.5, "W2-3d")
