"""ctypes access to the CPU oracle (oracle/liboracle.so) for tests and bench only.

The oracle is test infrastructure (oracle/fz_oracle.h header).  This wrapper is argument
marshalling only; it builds the library with gcc on first use if it is missing.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "fz_oracle.c")
LIB = os.path.join(ROOT, "oracle", "liboracle.so")

OK, ERR_ARG, ERR_NONFINITE, ERR_EB_TOO_SMALL, ERR_CAPACITY, ERR_CORRUPT = range(6)
ABS, REL, PWREL = 0, 1, 2


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call([
            "gcc", "-std=c99", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
            "-shared", "-o", LIB, SRC, "-lm"])
    return LIB


class Params(C.Structure):
    _fields_ = [("eb_input", C.c_double), ("eb_abs", C.c_double), ("w", C.c_float),
                ("r", C.c_float), ("eb32", C.c_float), ("mn", C.c_float), ("mx", C.c_float),
                ("mode", C.c_int), ("fallback", C.c_int)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P = C.c_void_p
        u64 = C.c_uint64
        L.fzo_range.argtypes = [P, u64, P, P, P]
        L.fzo_derive_params.argtypes = [C.c_float, C.c_float, C.c_int, C.c_double, C.POINTER(Params)]
        L.fzo_prequantize_one.argtypes = [C.c_float, C.POINTER(Params), P]
        L.fzo_lorenzo.argtypes = [P, C.c_int, P, P]
        L.fzo_pack.argtypes = [C.c_int32, P]
        L.fzo_unpack.argtypes = [C.c_uint16]
        L.fzo_unpack.restype = C.c_int32
        L.fzo_shuffle_tile.argtypes = [P, P]
        L.fzo_unshuffle_tile.argtypes = [P, P]
        L.fzo_flags_tile.argtypes = [P, P]
        L.fzo_quantize_field.argtypes = [P, C.c_int, P, C.POINTER(Params), P, P, P, u64, P, P, P, u64, P]
        L.fzo_compress_bound.argtypes = [C.c_int, P]
        L.fzo_compress_bound.restype = u64
        L.fzo_compress.argtypes = [P, C.c_int, P, C.c_int, C.c_double, P, u64, P]
        L.fzo_compress_with_params.argtypes = [P, C.c_int, P, C.POINTER(Params), P, u64, P]
        L.fzo_decompress.argtypes = [P, u64, P, u64]
        L.fzo_decode_q.argtypes = [P, u64, P, u64]
        L.fzo_lorenzo_chunked.argtypes = [P, P, u64, u64, P]
        L.fzo_compress_chunked.argtypes = [P, P, C.c_int, C.c_double, u64, u64, P, u64, P]
        L.fzo_log64.argtypes = [C.c_double]
        L.fzo_log64.restype = C.c_double
        L.fzo_exp64.argtypes = [C.c_double]
        L.fzo_exp64.restype = C.c_double
        L.fzo_log32.argtypes = [C.c_float]
        L.fzo_log32.restype = C.c_float
        L.fzo_exp32.argtypes = [C.c_float]
        L.fzo_exp32.restype = C.c_float
        L.fzo_pwrel_eb.argtypes = [C.c_double, C.c_float]
        L.fzo_pwrel_eb.restype = C.c_double
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _dims(shape):
    return np.array(list(shape), dtype=np.uint64)


def field_range(d: np.ndarray):
    d = np.ascontiguousarray(d, dtype=np.float32)
    mn, mx, bad = C.c_float(), C.c_float(), C.c_int64()
    st = lib().fzo_range(_ptr(d), d.size, C.byref(mn), C.byref(mx), C.byref(bad))
    return st, mn.value, mx.value, bad.value


def derive_params(mn: float, mx: float, mode: int, eb: float):
    p = Params()
    st = lib().fzo_derive_params(mn, mx, mode, eb, C.byref(p))
    return st, p


def params_for(d: np.ndarray, mode: int, eb: float) -> Params:
    st, mn, mx, _ = field_range(d)
    assert st == OK
    st, p = derive_params(mn, mx, mode, eb)
    assert st == OK, st
    return p


def prequantize(d: np.ndarray, p: Params):
    """Per-element C1: returns (q int32, value-outlier flags)."""
    d = np.ascontiguousarray(d, dtype=np.float32).reshape(-1)
    q = np.zeros(d.size, dtype=np.int32)
    f = np.zeros(d.size, dtype=np.uint8)
    one = C.c_int32()
    L = lib()
    for i, v in enumerate(d.tolist()):
        f[i] = L.fzo_prequantize_one(v, C.byref(p), C.byref(one))
        q[i] = one.value
    return q, f


def lorenzo(q: np.ndarray) -> np.ndarray:
    q = np.ascontiguousarray(q, dtype=np.int32)
    out = np.empty_like(q)
    dims = _dims(q.shape)
    lib().fzo_lorenzo(_ptr(q), q.ndim, _ptr(dims), _ptr(out))
    return out


def pack(delta: int):
    c = C.c_uint16()
    o = lib().fzo_pack(int(delta), C.byref(c))
    return c.value, o


def unpack(code: int) -> int:
    return lib().fzo_unpack(code)


def shuffle_tile(A: np.ndarray) -> np.ndarray:
    A = np.ascontiguousarray(A, dtype=np.uint32).reshape(1024)
    O = np.empty(1024, dtype=np.uint32)
    lib().fzo_shuffle_tile(_ptr(A), _ptr(O))
    return O


def unshuffle_tile(O: np.ndarray) -> np.ndarray:
    O = np.ascontiguousarray(O, dtype=np.uint32).reshape(1024)
    A = np.empty(1024, dtype=np.uint32)
    lib().fzo_unshuffle_tile(_ptr(O), _ptr(A))
    return A


def flags_tile(O: np.ndarray):
    O = np.ascontiguousarray(O, dtype=np.uint32).reshape(1024)
    F = np.empty(8, dtype=np.uint32)
    nnz = lib().fzo_flags_tile(_ptr(O), _ptr(F))
    return F, nnz


def quantize_field(d: np.ndarray, p: Params):
    """Codes and outlier lists of the whole field (stage hook)."""
    d = np.ascontiguousarray(d, dtype=np.float32)
    n = d.size
    codes = np.empty(n, dtype=np.uint16)
    cap = n
    didx = np.empty(cap, dtype=np.uint32)
    dval = np.empty(cap, dtype=np.int32)
    vidx = np.empty(cap, dtype=np.uint32)
    vbits = np.empty(cap, dtype=np.uint32)
    nd, nv = C.c_uint64(), C.c_uint64()
    dims = _dims(d.shape)
    st = lib().fzo_quantize_field(_ptr(d), d.ndim, _ptr(dims), C.byref(p), _ptr(codes),
                                  _ptr(didx), _ptr(dval), cap, C.byref(nd),
                                  _ptr(vidx), _ptr(vbits), cap, C.byref(nv))
    assert st == OK, st
    return (codes, didx[: nd.value].copy(), dval[: nd.value].copy(),
            vidx[: nv.value].copy(), vbits[: nv.value].copy())


def compress_bound(shape) -> int:
    dims = _dims(shape)
    return int(lib().fzo_compress_bound(len(shape), _ptr(dims)))


def compress(d: np.ndarray, mode: int, eb: float, params: Params | None = None):
    """Returns (status, bytes).  bytes is None on error."""
    d = np.ascontiguousarray(d, dtype=np.float32)
    dims = _dims(d.shape)
    cap = compress_bound(d.shape)
    out = np.empty(cap, dtype=np.uint8)
    size = C.c_uint64()
    if params is None:
        st = lib().fzo_compress(_ptr(d), d.ndim, _ptr(dims), mode, eb, _ptr(out), cap, C.byref(size))
    else:
        st = lib().fzo_compress_with_params(_ptr(d), d.ndim, _ptr(dims), C.byref(params),
                                            _ptr(out), cap, C.byref(size))
    if st != OK:
        return st, None
    return st, out[: size.value].copy()


def lorenzo_chunked(q: np.ndarray, cz: int, cy: int) -> np.ndarray:
    """f1: chunk-local Lorenzo of a 3-D array (chunks of cz planes x cy rows x full rows)."""
    q = np.ascontiguousarray(q, dtype=np.int32)
    assert q.ndim == 3
    out = np.empty_like(q)
    dims = _dims(q.shape)
    lib().fzo_lorenzo_chunked(_ptr(q), _ptr(dims), cz, cy, _ptr(out))
    return out


def compress_chunked(d: np.ndarray, mode: int, eb: float, cz: int, cy: int):
    """f1 chunk-local compressor (3-D).  Returns (status, bytes)."""
    d = np.ascontiguousarray(d, dtype=np.float32)
    dims = _dims(d.shape)
    cap = compress_bound(d.shape)
    out = np.empty(cap, dtype=np.uint8)
    size = C.c_uint64()
    st = lib().fzo_compress_chunked(_ptr(d), _ptr(dims), mode, eb, cz, cy, _ptr(out), cap, C.byref(size))
    if st != OK:
        return st, None
    return st, out[: size.value].copy()


def decompress(buf: np.ndarray, n: int):
    buf = np.ascontiguousarray(buf, dtype=np.uint8)
    out = np.empty(n, dtype=np.float32)
    st = lib().fzo_decompress(_ptr(buf), buf.size, _ptr(out), n)
    return st, out


def decode_q(buf: np.ndarray, n: int):
    buf = np.ascontiguousarray(buf, dtype=np.uint8)
    q = np.empty(n, dtype=np.int32)
    st = lib().fzo_decode_q(_ptr(buf), buf.size, _ptr(q), n)
    return st, q
