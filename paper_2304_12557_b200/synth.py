"""Seeded synthetic look-alike fields for the paper's workloads.

This module holds ONLY input generation: no step of the compression method lives here.
It is the one module shared by the CUDA path's tests/bench and the oracle's tests
(DESIGN.md §5 "input recipe").  Every field is evaluated in float64 on the host and
rounded once to float32, so the oracle and the GPU always see identical bytes.

Generators (dims slowest first, (z, y, x)):
  sines3d     c1  64^3 sum of separable sinusoids + uniform noise       ("smooth")
  cesm_t      c2  1800x3600 T-like field with a +250 offset and noise   (P:406 shape)
  cesm_cld    c2  1800x3600 cloud-fraction-like field clipped to [0,1]
  hurr_qsnow  c3  100x500x500 mostly exact zeros (QSNOW-like)
  hurr_u      c3  100x500x500 vortex wind + noise
  nyx_rho     c4  512^3 log-normal density exp(1.5 g)
  nyx_v       c4  512^3 velocity-like 3e7 * sines + noise
  rtm         c5  1008x1008x352 5 reflected Ricker shells over exact zeros
  qmc         alt 33120x69x69 oscillatory orbitals ("unsmooth")
  hacc_x      f3  280,953,867 particle coordinates in (0, 256) (P:314 HACC, "unsmooth")
Adversarial fields for parity edge cases live in `adversarial()`.

Random numbers: splitmix64 (Steele et al.), u(idx, s) = ((mix(s*G + idx + G) >> 40) + .5)
* 2^-24 in (0, 1); parameters come from a sequential splitmix64 stream seeded per config.
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

# name -> (default shape, seed)
FIELDS = {
    "sines3d": ((64, 64, 64), 1),
    "cesm_t": ((1800, 3600), 2),
    "cesm_cld": ((1800, 3600), 2),
    "hurr_qsnow": ((100, 500, 500), 3),
    "hurr_u": ((100, 500, 500), 3),
    "nyx_rho": ((512, 512, 512), 4),
    "nyx_v": ((512, 512, 512), 44),
    "rtm": ((1008, 1008, 352), 5),
    "qmc": ((33120, 69, 69), 6),
    "hacc_x": ((280953867,), 8),
}


def _mix(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


class SplitMix64:
    """Sequential splitmix64 stream for generator parameters."""

    def __init__(self, seed: int):
        self.state = int(seed) & 0xFFFFFFFFFFFFFFFF

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        return int(_mix(np.array([self.state], dtype=np.uint64))[0])

    def uniform(self, lo: float, hi: float) -> float:
        u = ((self.next_u64() >> 11) + 0.5) * 2.0 ** -53
        return lo + (hi - lo) * u


def uniform01(idx: np.ndarray, seed: int) -> np.ndarray:
    """Counter-based u(idx, s) in (0, 1), float64."""
    with np.errstate(over="ignore"):
        base = np.uint64(seed) * GAMMA
        z = idx.astype(np.uint64) + base + GAMMA
    return ((_mix(z) >> np.uint64(40)).astype(np.float64) + 0.5) * (2.0 ** -24)


def _noise(amp: float, start: int, count: int, seed: int) -> np.ndarray:
    idx = np.arange(start, start + count, dtype=np.uint64)
    return amp * (2.0 * uniform01(idx, seed) - 1.0)


def _sine_terms(shape, K, seed, fmin, fmax):
    rng = SplitMix64(seed)
    terms = []
    for _ in range(K):
        a = rng.uniform(0.5, 1.0)
        axes = []
        for n in shape:
            f = rng.uniform(fmin, fmax)
            phi = rng.uniform(0.0, 2.0 * math.pi)
            i = np.arange(n, dtype=np.float64)
            axes.append(np.sin(2.0 * math.pi * f * i / n + phi))
        terms.append((a, axes))
    return terms


def _sines_chunk(terms, shape, z0, z1):
    """Clean separable sum over planes [z0, z1) (3-D) or rows (2-D)."""
    nd = len(shape)
    out = None
    for a, axes in terms:
        if nd == 3:
            t = a * axes[0][z0:z1, None, None] * (axes[1][None, :, None] * axes[2][None, None, :])
        elif nd == 2:
            t = a * axes[0][z0:z1, None] * axes[1][None, :]
        else:
            t = a * axes[0][z0:z1]
        out = t if out is None else out + t
    return out


def _chunks(nz, per):
    z = 0
    while z < nz:
        yield z, min(nz, z + per)
        z += per


def _pmap(fn, chunks):
    """fn over the chunks on a thread pool (numpy releases the GIL in its array loops);
    results in chunk order, so reductions over them sum in the same order as a serial loop
    and every element is the same f64 expression -- bit-identical to the serial evaluation."""
    chunks = list(chunks)
    if len(chunks) <= 1:
        return [fn(*c) for c in chunks]
    with ThreadPoolExecutor(max_workers=min(len(chunks), os.cpu_count() or 1, 32)) as ex:
        return list(ex.map(lambda c: fn(*c), chunks))


def _plane(shape):
    return int(np.prod(shape[1:])) if len(shape) > 1 else 1


def sines3d(shape=(64, 64, 64), seed=1, K=6, fmin=0.5, fmax=4.0, noise_rel=1e-3):
    terms = _sine_terms(shape, K, seed, fmin, fmax)
    clean = np.empty(shape, dtype=np.float64)

    def fill(z0, z1):
        clean[z0:z1] = _sines_chunk(terms, shape, z0, z1)
    _pmap(fill, _chunks(shape[0], max(1, (1 << 23) // _plane(shape))))
    rng_ = float(clean.max() - clean.min())
    out = np.empty(shape, dtype=np.float32)
    P = _plane(shape)

    def put(z0, z1):
        n = (z1 - z0) * P
        v = clean[z0:z1].reshape(-1) + _noise(noise_rel * rng_, z0 * P, n, seed)
        out[z0:z1] = v.reshape((z1 - z0,) + tuple(shape[1:])).astype(np.float32)
    _pmap(put, _chunks(shape[0], max(1, (1 << 23) // P)))
    return out


def _latlon(ny, nx, y0, y1):
    lat = -math.pi / 2 + math.pi * (np.arange(y0, y1, dtype=np.float64) + 0.5) / ny
    lon = 2.0 * math.pi * np.arange(nx, dtype=np.float64) / nx
    return lat[:, None], lon[None, :]


def cesm_t(shape=(1800, 3600), seed=2):
    ny, nx = shape
    out = np.empty(shape, dtype=np.float32)
    for y0, y1 in _chunks(ny, max(1, (1 << 22) // nx)):
        lat, lon = _latlon(ny, nx, y0, y1)
        v = (250.0 + 40.0 * np.cos(lat) + 5.0 * np.sin(3 * lon) * np.cos(2 * lat)
             + 2.0 * np.sin(7 * lon + 3 * lat))
        v = v.reshape(-1) + _noise(0.1, y0 * nx, (y1 - y0) * nx, seed)
        out[y0:y1] = v.reshape(y1 - y0, nx).astype(np.float32)
    return out


def cesm_cld(shape=(1800, 3600), seed=2):
    ny, nx = shape
    out = np.empty(shape, dtype=np.float32)
    for y0, y1 in _chunks(ny, max(1, (1 << 22) // nx)):
        lat, lon = _latlon(ny, nx, y0, y1)
        v = 0.5 + 0.6 * np.sin(5 * lon) * np.cos(4 * lat) + 0.3 * np.sin(11 * lon + 2 * lat)
        out[y0:y1] = np.clip(v, 0.0, 1.0).astype(np.float32)
    return out


def _hurr_grid(shape, z0, z1):
    nz, ny, nx = shape
    cy, cx = ny / 2.0, nx / 2.0
    z = np.arange(z0, z1, dtype=np.float64)[:, None, None]
    y = np.arange(ny, dtype=np.float64)[None, :, None]
    x = np.arange(nx, dtype=np.float64)[None, None, :]
    r = np.hypot(y - cy, x - cx)
    return z, y, x, r, cy, cx


def hurr_qsnow(shape=(100, 500, 500), seed=3):
    out = np.empty(shape, dtype=np.float32)
    s = shape[1] / 500.0
    for z0, z1 in _chunks(shape[0], max(1, (1 << 22) // _plane(shape))):
        z, y, x, r, _, _ = _hurr_grid(shape, z0, z1)
        v = (1e-3 * np.exp(-(((r - 120 * s) / (50 * s)) ** 2)) * np.exp(-z / 60.0)
             * (1 + 0.3 * np.sin(x / (14 * s)) * np.sin(y / (18 * s))) - 2e-4)
        out[z0:z1] = np.maximum(0.0, v).astype(np.float32)
    return out


def hurr_u(shape=(100, 500, 500), seed=3):
    out = np.empty(shape, dtype=np.float32)
    s = shape[1] / 500.0
    P = _plane(shape)
    for z0, z1 in _chunks(shape[0], max(1, (1 << 22) // P)):
        z, y, x, r, cy, _ = _hurr_grid(shape, z0, z1)
        rs = r / (80 * s)
        v = 40.0 * rs * np.exp(1 - rs) * (-(y - cy) / np.maximum(r, 1.0)) * np.exp(-z / 80.0)
        v = np.broadcast_to(v, (z1 - z0,) + tuple(shape[1:])).reshape(-1)
        v = v + _noise(0.01, z0 * P, (z1 - z0) * P, seed)
        out[z0:z1] = v.reshape((z1 - z0,) + tuple(shape[1:])).astype(np.float32)
    return out


def nyx_rho(shape=(512, 512, 512), seed=4):
    terms = _sine_terms(shape, 12, seed, 1.0, 8.0)
    per = max(1, (1 << 23) // _plane(shape))
    n = float(np.prod(shape))
    s1 = 0.0
    for v in _pmap(lambda z0, z1: float(_sines_chunk(terms, shape, z0, z1).sum()), _chunks(shape[0], per)):
        s1 += v
    mean = s1 / n
    s2 = 0.0
    for v in _pmap(lambda z0, z1: float(((_sines_chunk(terms, shape, z0, z1) - mean) ** 2).sum()),
                   _chunks(shape[0], per)):
        s2 += v
    std = math.sqrt(s2 / n)
    out = np.empty(shape, dtype=np.float32)

    def put(z0, z1):
        g = (_sines_chunk(terms, shape, z0, z1) - mean) / std
        out[z0:z1] = np.exp(1.5 * g).astype(np.float32)
    _pmap(put, _chunks(shape[0], per))
    return out


def nyx_v(shape=(512, 512, 512), seed=44):
    terms = _sine_terms(shape, 6, seed, 0.5, 4.0)
    per = max(1, (1 << 23) // _plane(shape))
    lo, hi = math.inf, -math.inf

    def ext(z0, z1):
        c = _sines_chunk(terms, shape, z0, z1)
        return float(c.min()), float(c.max())
    for a, b in _pmap(ext, _chunks(shape[0], per)):
        lo, hi = min(lo, a), max(hi, b)
    amp = 2e-4 * 3e7 * (hi - lo)
    out = np.empty(shape, dtype=np.float32)
    P = _plane(shape)

    def put(z0, z1):
        v = 3e7 * _sines_chunk(terms, shape, z0, z1).reshape(-1)
        v = v + _noise(amp, z0 * P, (z1 - z0) * P, seed)
        out[z0:z1] = v.reshape((z1 - z0,) + tuple(shape[1:])).astype(np.float32)
    _pmap(put, _chunks(shape[0], per))
    return out


def rtm(shape=(1008, 1008, 352), seed=5):
    """Field t = seed - 5 of the c5 batch (seeds 5..12)."""
    t = seed - 5
    nz, ny, nx = shape
    sc = ny / 1008.0
    out = np.empty(shape, dtype=np.float32)
    y = np.arange(ny, dtype=np.float64)[None, :, None]
    x = np.arange(nx, dtype=np.float64)[None, None, :]
    def put(z0, z1):
        z = np.arange(z0, z1, dtype=np.float64)[:, None, None]
        rr = np.sqrt((z - 20 * sc) ** 2 + (y - ny / 2.0) ** 2 + (x - nx / 2.0) ** 2).reshape(-1)
        # ricker(s) is exactly 0 for |s| >= 6: the shells are evaluated only where some shell
        # is live (the same f64 expression per element; 0 / max(rr, 1) = +0 elsewhere)
        live = np.zeros(rr.shape, dtype=bool)
        for m in range(5):
            live |= np.abs((rr - (150 + 60 * t) * sc + 45 * m * sc) / (6 * sc)) < 6
        r_l = rr[live]
        acc = np.zeros_like(r_l)
        for m in range(5):
            s = (r_l - (150 + 60 * t) * sc + 45 * m * sc) / (6 * sc)
            rk = np.where(np.abs(s) < 6, (1 - 2 * s * s) * np.exp(-s * s), 0.0)
            acc += (0.6 ** m) * rk
        v = np.zeros(rr.shape, dtype=np.float32)
        v[live] = (acc / np.maximum(r_l, 1.0)).astype(np.float32)
        out[z0:z1] = v.reshape((z1 - z0, ny, nx))
    _pmap(put, _chunks(nz, max(1, (1 << 22) // _plane(shape))))
    return out


def qmc(shape=(33120, 69, 69), seed=6):
    """Oscillatory orbitals under a Gaussian envelope (low-CR stress field)."""
    nz, ny, nx = shape
    rng = SplitMix64(seed)
    kz, ky, kx = (rng.uniform(0.5, 1.5) for _ in range(3))
    out = np.empty(shape, dtype=np.float32)
    y = (np.arange(ny, dtype=np.float64)[None, :, None] - ny / 2) / ny
    x = (np.arange(nx, dtype=np.float64)[None, None, :] - nx / 2) / nx
    P = _plane(shape)
    for z0, z1 in _chunks(nz, max(1, (1 << 22) // P)):
        zi = np.arange(z0, z1, dtype=np.float64)[:, None, None]
        orb = (zi % 69) / 69.0 - 0.5
        env = np.exp(-(orb ** 2 + y ** 2 + x ** 2) * 8.0)
        v = env * np.cos(40 * kx * x + 37 * ky * y + 2.1 * kz * zi) * np.sin(23 * x * y + zi * 0.37)
        v = v.reshape(-1) + _noise(1e-3, z0 * P, (z1 - z0) * P, seed)
        out[z0:z1] = v.reshape((z1 - z0,) + tuple(shape[1:])).astype(np.float32)
    return out


def hacc_x(shape=(280953867,), seed=8):
    """HACC-like particle coordinate (1-D, SV 8.a: 280,953,867 particles): particles come in
    halos of 1000 consecutive indices; halo h has centre c_h = 256 u(h) and radius
    r_h = 0.05 + 2 u'(h); particle i sits at c_h + r_h (2 u(i) - 1), wrapped into the periodic
    box [0, 256) and shifted by 1/64 so every value is strictly positive (the log transform's
    domain).  Irregular within a halo, clustered across halos ("unsmooth")."""
    n = int(np.prod(shape))
    out = np.empty(n, dtype=np.float32)
    per = 1 << 22

    def put(a, b):
        i = np.arange(a, b, dtype=np.uint64)
        h = i // np.uint64(1000)
        c = 256.0 * uniform01(h, seed)
        r = 0.05 + 2.0 * uniform01(h, seed + 1)
        v = np.mod(c + r * (2.0 * uniform01(i, seed + 2) - 1.0), 256.0) + 1.0 / 64.0
        out[a:b] = v.astype(np.float32)
    _pmap(put, _chunks(n, per))
    return out.reshape(shape)


_GEN = {
    "sines3d": sines3d, "cesm_t": cesm_t, "cesm_cld": cesm_cld, "hurr_qsnow": hurr_qsnow,
    "hurr_u": hurr_u, "nyx_rho": nyx_rho, "nyx_v": nyx_v, "rtm": rtm, "qmc": qmc, "hacc_x": hacc_x,
}


def generate(name: str, shape=None, seed=None) -> np.ndarray:
    """Generate field `name` (optionally at a reduced look-alike `shape`)."""
    dshape, dseed = FIELDS[name]
    shape = tuple(shape) if shape is not None else dshape
    seed = dseed if seed is None else seed
    return _GEN[name](shape=shape, seed=seed)


# Workload configs of BASELINE.json (c1..c5): (field, shape, REL bounds)
CONFIGS = {
    "c1": [("sines3d", (64, 64, 64), (1e-3,))],
    "c2": [("cesm_t", (1800, 3600), (1e-2, 1e-3, 1e-4)),
           ("cesm_cld", (1800, 3600), (1e-2, 1e-3, 1e-4))],
    "c3": [("hurr_qsnow", (100, 500, 500), (1e-3,)), ("hurr_u", (100, 500, 500), (1e-3,))],
    "c4": [("nyx_v", (512, 512, 512), (1e-3, 1e-4)), ("nyx_rho", (512, 512, 512), (1e-3, 1e-4))],
    "c5": [("rtm", (1008, 1008, 352), (1e-4,))],
}


def adversarial(kind: str, n: int, seed: int = 7) -> np.ndarray:
    """1-D adversarial inputs: constant, ramp, zeros, spike, offset, noise."""
    i = np.arange(n, dtype=np.float64)
    if kind == "zeros":
        return np.zeros(n, dtype=np.float32)
    if kind == "constant":
        return np.full(n, 3.25, dtype=np.float32)
    if kind == "ramp":
        return (0.001 * i).astype(np.float32)
    if kind == "noise":
        return (2.0 * uniform01(i.astype(np.uint64), seed) - 1.0).astype(np.float32)
    if kind == "spike":
        v = np.sin(i / 50.0)
        v[:: max(1, n // 7)] = 100.0
        return v.astype(np.float32)
    if kind == "offset":
        return (1e6 + np.sin(i / 30.0)).astype(np.float32)
    raise KeyError(kind)
