"""f3: point-wise relative error bound through a log transform -- pins of
the oracle's transform (reading R25: natural log / exp as fixed binary64 operation sequences
rounded once to binary32) and of the P:314 guarantee |x^ - x| <= eps |x| on every element.

The transform functions are pinned against numpy's libm log / exp (an implementation the
oracle shares nothing with): agreement to a few binary64 ulps, and binary32 results equal to
numpy's rounded value except where the binary64 values straddle a binary32 rounding boundary.
"""
from __future__ import annotations

import struct

import numpy as np
import pytest

import oracle_lib as O
from paper_2304_12557_b200 import synth

FLT_MIN = np.float32(np.finfo(np.float32).tiny)
FLT_MAX = np.float32(np.finfo(np.float32).max)


def _samples(n=60000, seed=3):
    rng = np.random.default_rng(seed)
    e = rng.uniform(-125.9, 127.9, n)
    x = np.exp2(e).astype(np.float32)                          # log-uniform over the normals
    x = np.concatenate([x, rng.uniform(0.5, 2.0, 20000).astype(np.float32),
                        (1.0 + rng.uniform(-1e-3, 1e-3, 5000)).astype(np.float32),
                        np.float32(2.0) ** np.arange(-126, 128, dtype=np.float32),
                        np.array([FLT_MIN, FLT_MAX, 1.0, np.nextafter(np.float32(1), 2),
                                  np.nextafter(np.float32(1), 0)], np.float32)])
    return x[(x >= FLT_MIN) & np.isfinite(x)]


def _f32_boundary_close(v64: np.ndarray, ulps64=8):
    """True where a binary64 value is within `ulps64` binary64 ulps of a binary32 rounding
    boundary (midpoint between two binary32 neighbours): there two correct binary64
    approximations may round to different binary32 values."""
    f = v64.astype(np.float32).astype(np.float64)
    lo = np.nextafter(v64.astype(np.float32), np.float32(-np.inf)).astype(np.float64)
    hi = np.nextafter(v64.astype(np.float32), np.float32(np.inf)).astype(np.float64)
    mid = np.minimum(np.abs(v64 - (f + lo) / 2), np.abs(v64 - (f + hi) / 2))
    return mid <= ulps64 * np.spacing(np.abs(v64))


def test_log64_exp64_against_numpy():
    L = O.lib()
    x = _samples()
    ours = np.array([L.fzo_log64(float(v)) for v in x[::7]])
    ref = np.log(x[::7].astype(np.float64))
    assert np.all(np.abs(ours - ref) <= 4 * np.spacing(np.maximum(np.abs(ref), 1e-300)) + 1e-300)
    t = np.linspace(-103.0, 88.7, 20011)
    ours = np.array([L.fzo_exp64(float(v)) for v in t])
    ref = np.exp(t)
    assert np.all(np.abs(ours - ref) <= 8 * np.spacing(ref))


def test_log32_exp32_round_once():
    L = O.lib()
    x = _samples()[::3]
    ours = np.array([L.fzo_log32(float(v)) for v in x], np.float32)
    r64 = np.log(x.astype(np.float64))
    ref = r64.astype(np.float32)
    bad = ours != ref
    assert np.all(_f32_boundary_close(r64[bad]))
    assert bad.sum() <= 2
    y = np.linspace(-87.0, 88.5, 30011).astype(np.float32)
    ours = np.array([L.fzo_exp32(float(v)) for v in y], np.float32)
    r64 = np.exp(y.astype(np.float64))
    ref = r64.astype(np.float32)
    bad = ours != ref
    assert np.all(_f32_boundary_close(r64[bad])) and bad.sum() <= 2


def test_special_values():
    L = O.lib()
    assert L.fzo_log64(1.0) == 0.0 and L.fzo_log32(1.0) == 0.0          # S:320 log 1 = 0
    assert L.fzo_exp64(0.0) == 1.0 and L.fzo_exp32(0.0) == 1.0
    assert abs(L.fzo_log64(2.0) - np.log(2.0)) <= np.spacing(np.log(2.0))
    assert L.fzo_exp32(89.0) == FLT_MAX                                    # clamped, not inf
    for k in (-126, -1, 1, 64, 127):   # log 2^k = k ln 2 to a few binary64 ulps
        v = L.fzo_log64(2.0 ** k)
        assert abs(v - k * np.log(2.0)) <= 4 * np.spacing(abs(k * np.log(2.0)))


def test_pwrel_bound_is_sound_and_tight():
    """eb(eps, M) < log(1 + eps) (sound side) and within U/4 + 2^-24 + 2^-39 of it (tight)."""
    L = O.lib()
    for eps in (1e-1, 1e-2, 1e-3, 1e-4):
        for M in (0.0, 0.5, 5.0, 88.0):
            b = L.fzo_pwrel_eb(eps, M)
            U = 0.0 if M == 0 else 2.0 ** (np.frexp(M)[1] - 23)
            assert 0 < b < np.log1p(eps)
            assert np.log1p(eps) - b <= U / 4 + 2 ** -23 + 2 ** -39
    assert L.fzo_pwrel_eb(1e-9, 88.0) <= 0      # below the binary32 resolution of log x


def _roundtrip(d: np.ndarray, eps: float):
    st, buf = O.compress(d, O.PWREL, eps)
    assert st == O.OK
    st, xh = O.decompress(buf, d.size)
    assert st == O.OK
    x = d.reshape(-1).astype(np.float64)
    err = np.abs(xh.astype(np.float64) - x)
    return buf, xh, err, x


FIELDS = [
    ("hacc_x", lambda: synth.generate("hacc_x", (300000,))),
    ("nyx_rho", lambda: synth.generate("nyx_rho", (24, 24, 24))),
    ("loguniform", lambda: np.exp2(np.random.default_rng(5).uniform(-120, 120, 50000)).astype(np.float32)),
    ("extremes", lambda: np.array([FLT_MIN, FLT_MAX, 1.0, 3.0, FLT_MAX, FLT_MIN] * 700, np.float32)),
    ("constant", lambda: np.full(5000, 7.25, np.float32)),
]


@pytest.mark.parametrize("name,gen", FIELDS, ids=[f[0] for f in FIELDS])
@pytest.mark.parametrize("eps", [1e-2, 1e-3, 1e-4])
def test_pointwise_relative_bound(name, gen, eps):
    """compressing log x with the derived ABS bound yields |x^ - x| <= eps |x|."""
    d = gen()
    buf, xh, err, x = _roundtrip(d, eps)
    assert np.all(err <= eps * np.abs(x)), f"worst {np.max(err / np.abs(x)) / eps:.6f} eps"
    assert np.all(np.isfinite(xh)) and np.all(xh > 0)
    hdr = buf[:128].tobytes()
    flags = struct.unpack_from("<H", hdr, 6)[0]
    eb_in, eb_abs = struct.unpack_from("<dd", hdr, 48)
    assert flags & 8 and not flags & 1 and eb_in == eps
    # the stream's own ABS guarantee holds on the log field: |y^ - log32(x)| <= eb_abs
    L = O.lib()
    y = np.array([L.fzo_log32(float(v)) for v in d.reshape(-1)[:3000]], np.float32)
    st, q = O.decode_q(buf, d.size)
    w = struct.unpack_from("<f", hdr, 64)[0]
    yh = (q[:3000].astype(np.float32) * np.float32(w)).astype(np.float32)
    nv = struct.unpack_from("<Q", hdr, 104)[0]
    if nv == 0:
        assert np.all(np.abs(yh.astype(np.float64) - y.astype(np.float64)) <= eb_abs)
    assert eb_abs > 0.9 * np.log1p(eps) - 2e-5


def test_domain_errors():
    for bad, st in [(0.0, O.ERR_ARG), (-1.0, O.ERR_ARG), (1e-40, O.ERR_ARG), (np.nan, O.ERR_NONFINITE),
                    (np.inf, O.ERR_NONFINITE)]:
        d = np.ones(100, np.float32)
        d[37] = bad
        assert O.compress(d, O.PWREL, 1e-3)[0] == st
    assert O.compress(np.ones(10, np.float32), O.PWREL, 1.0)[0] == O.ERR_ARG
    assert O.compress(np.ones(10, np.float32), O.PWREL, 1e-9)[0] == O.ERR_EB_TOO_SMALL


def test_all_ones_logs_to_zero():
    """an all-ones field transforms to all zeros -> every block is zero (P:373 cap)."""
    d = np.ones(4096, np.float32)
    st, buf = O.compress(d, O.PWREL, 1e-3)
    assert st == O.OK and buf.size == 128 + 32 * 2
    st, xh = O.decompress(buf, d.size)
    assert np.array_equal(xh, d)
