"""The oracle is plain C99 that is also valid C++17 (SURVEY §8.c asks for "plain single-threaded
C++"): built with g++ -x c++ (same -ffp-contract=off -fno-fast-math, no shared code with the GPU
path), it must produce byte-identical streams and bit-identical decoded fields to the C build
on every mode: REL / ABS / PWREL (f3), chunk-local (f1), outliers and fallback."""
import ctypes as C
import os
import shutil
import subprocess

import numpy as np
import pytest

import oracle_lib as O
from paper_2304_12557_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cpp_lib(tmp_path_factory):
    if shutil.which("g++") is None:
        pytest.skip("needs g++")
    so = str(tmp_path_factory.mktemp("cpp") / "liboracle_cpp.so")
    subprocess.run(["g++", "-std=c++17", "-x", "c++", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                    "-shared", "-Wall", "-Werror", os.path.join(ROOT, "oracle", "fz_oracle.c"), "-o", so],
                   check=True, capture_output=True)
    L = C.CDLL(so)
    P, u64 = C.c_void_p, C.c_uint64
    L.fzo_compress_bound.argtypes = [C.c_int, P]
    L.fzo_compress_bound.restype = u64
    L.fzo_compress.argtypes = [P, C.c_int, P, C.c_int, C.c_double, P, u64, P]
    L.fzo_compress_chunked.argtypes = [P, P, C.c_int, C.c_double, u64, u64, P, u64, P]
    L.fzo_decompress.argtypes = [P, u64, P, u64]
    return L


def _cpp_compress(L, d, mode, eb, chunk=None):
    d = np.ascontiguousarray(d, dtype=np.float32)
    dims = np.array(list(d.shape) + [1] * (3 - d.ndim), dtype=np.uint64)
    cap = L.fzo_compress_bound(d.ndim, dims.ctypes.data)
    out = np.empty(cap, dtype=np.uint8)
    size = C.c_uint64()
    if chunk is None:
        st = L.fzo_compress(d.ctypes.data, d.ndim, dims.ctypes.data, mode, eb, out.ctypes.data, cap, C.byref(size))
    else:
        st = L.fzo_compress_chunked(d.ctypes.data, dims.ctypes.data, mode, eb, chunk[0], chunk[1], out.ctypes.data,
                                    cap, C.byref(size))
    assert st == 0
    s = out[: size.value].copy()
    x = np.empty(d.size, dtype=np.float32)
    assert L.fzo_decompress(s.ctypes.data, s.size, x.ctypes.data, d.size) == 0
    return s, x


@pytest.mark.parametrize("name,shape,mode,eb,chunk", [
    ("nyx_v", (20, 16, 256), O.REL, 1e-3, None),
    ("hurr_u", (9, 30, 52), O.ABS, 1e-2, None),
    ("cesm_t", (60, 90), O.REL, 1e-4, None),
    ("hacc_x", (50001,), O.PWREL, 1e-3, None),
    ("nyx_v", (32, 16, 256), O.REL, 1e-3, (16, 8)),
])
def test_oracle_cpp_build_equals_c_build(cpp_lib, name, shape, mode, eb, chunk):
    d = synth.generate(name, shape).copy()
    if name == "hurr_u":   # spikes: delta and value outliers
        d.reshape(-1)[[17, 900, 5000]] += np.float32(1e4)
    if chunk is None:
        st, ref = O.compress(d, mode, eb)
    else:
        st, ref = O.compress_chunked(d, mode, eb, chunk[0], chunk[1])
    assert st == O.OK
    st, xref = O.decompress(ref, d.size)
    got, x = _cpp_compress(cpp_lib, d, mode, eb, chunk)
    assert got.size == ref.size and np.array_equal(got, ref)
    assert np.array_equal(x.view(np.uint32), xref.view(np.uint32))
