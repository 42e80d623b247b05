"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/fz.h declares,
and its host-side logic (sizes, parameter derivation, header parsing) is right.  No kernel
is launched here."""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle_lib as O
from paper_2304_12557_b200 import build as B
from paper_2304_12557_b200 import fz, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    B.build_libfz()
    return fz.lib()


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "fz.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(fz_[a-z_0-9]+)\s*\(", txt)))


def test_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) == 40
    L = C.CDLL(fz.LIB_PATH)
    for s in syms:
        assert hasattr(L, s), s


def test_sizes():
    assert fz.compress_bound((64, 64, 64)) == 128 + 32 * 128 + 4096 * 128 + 16 * 64 ** 3
    assert fz.compress_bound((0,)) == 0
    assert fz.compress_bound((1 << 32,)) == 0           # N >= 2^32 rejected (R16)
    assert fz.workspace_bytes((512, 512, 512)) > 0
    assert fz.decompress_workspace_bytes((100, 500, 500)) > 0
    assert fz.slab_stage_bound((512, 512, 512), 0, 128) == 32 * 128 + 4096 * 128 + 16 * 128 * 2048


@pytest.mark.parametrize("mode", [O.ABS, O.REL, O.PWREL])
def test_host_params_match_oracle(mode):
    """libfz's host parameter derivation equals the oracle's (independent implementations of
    Appendix A / R2; for PWREL also of R25's bound on the log field, incl. log64)."""
    rng = np.random.default_rng(0)
    for _ in range(2000):
        a = np.float32(rng.normal() * 10 ** rng.uniform(-5, 8))
        b = np.float32(a + abs(rng.normal()) * 10 ** rng.uniform(-8, 6))
        eb = 10 ** rng.uniform(-7, 0)
        st1, p1 = O.derive_params(float(a), float(b), mode, eb)
        try:
            p2 = fz.derive_params(float(a), float(b), mode, eb)
            st2 = O.OK
        except fz.FZError as e:
            st2 = e.status
        assert st1 == st2
        if st1 == O.OK:
            for k in ("eb_abs", "w", "r", "eb32", "fallback"):
                assert getattr(p1, k) == getattr(p2, k), k


def test_peek_header_on_oracle_stream():
    d = synth.generate("cesm_t", (90, 180))
    st, buf = O.compress(d, O.REL, 1e-3)
    info = fz.peek_header(buf[:128].tobytes())
    assert info.n == d.size and info.tiles == -(-d.size // 2048)
    assert info.total_size == buf.size and info.shape.ndim == 2
    assert tuple(info.shape.dims)[:2] == d.shape
    bad = bytearray(buf[:128].tobytes())
    bad[0] ^= 1
    with pytest.raises(fz.FZError):
        fz.peek_header(bytes(bad))
    bad = bytearray(buf[:128].tobytes())
    bad[88] ^= 1                                   # nnz breaks the size law
    with pytest.raises(fz.FZError):
        fz.peek_header(bytes(bad))


def test_peek_header_chunk_word_consistency():
    """Header flag bit 2 (f1 chunk-local, R23) and the chunk dims at bytes 10-13 must agree:
    bit 2 with a zero chunk word, or a nonzero word without bit 2, is a corrupt stream."""
    d = synth.generate("nyx_v", (32, 32, 64))
    st, g = O.compress(d, O.REL, 1e-3)
    st, c = O.compress_chunked(d, O.REL, 1e-3, 16, 2048 // 64)
    assert fz.peek_header(g[:128].tobytes()).flags & 4 == 0
    assert fz.peek_header(c[:128].tobytes()).flags & 4 == 4
    bad = bytearray(c[:128].tobytes())
    bad[10:14] = b"\0\0\0\0"                    # bit 2 set, chunk word zero
    with pytest.raises(fz.FZError) as e:
        fz.peek_header(bytes(bad))
    assert e.value.status == fz.ERR_CORRUPT
    bad = bytearray(g[:128].tobytes())
    bad[12] = 1                                    # chunk height without bit 2
    with pytest.raises(fz.FZError) as e:
        fz.peek_header(bytes(bad))
    assert e.value.status == fz.ERR_CORRUPT


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    monkeypatch.setattr(fz, "_lib", None)
    monkeypatch.setattr(fz, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(RuntimeError):
        fz.lib()
