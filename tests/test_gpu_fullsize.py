"""Full-size parity at the BASELINE.json shapes (c1..c5), in the launch configuration bench.py
times: the GPU stream must equal the oracle's byte for byte and the decompressed field must be
bit-identical (BJ north star "bit-exact agreement with the CPU oracle on all five configs")."""
from __future__ import annotations

import numpy as np
import pytest

import oracle_lib as O
from paper_2304_12557_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2304_12557_b200 import fz  # noqa: E402

CASES = [
    ("c1", "sines3d", (64, 64, 64), 1e-3),
    ("c2", "cesm_t", (1800, 3600), 1e-2),
    ("c2", "cesm_t", (1800, 3600), 1e-3),
    ("c2", "cesm_t", (1800, 3600), 1e-4),
    ("c2", "cesm_cld", (1800, 3600), 1e-3),
    ("c3", "hurr_qsnow", (100, 500, 500), 1e-3),
    ("c3", "hurr_u", (100, 500, 500), 1e-3),
    ("c4", "nyx_v", (512, 512, 512), 1e-3),
    ("c4", "nyx_rho", (512, 512, 512), 1e-4),
    ("c5", "rtm", (1008, 1008, 352), 1e-4),
]


@pytest.mark.parametrize("cfg,field,shape,rel", CASES, ids=[f"{c[0]}-{c[1]}-{c[3]}" for c in CASES])
def test_fullsize_parity(cfg, field, shape, rel):
    d = synth.generate(field, shape)
    st, ref = O.compress(d, O.REL, rel)
    assert st == O.OK
    codec = fz.Codec(shape, "cuda:0")
    x = torch.from_numpy(d).to("cuda:0")
    buf, size = codec.compress(x, fz.REL, rel)
    got = buf.cpu().numpy()
    assert size == ref.size, (size, ref.size)
    if not np.array_equal(got, ref):
        first = int(np.nonzero(got != ref)[0][0])
        raise AssertionError(f"stream differs from the oracle at byte {first} of {size}")
    del got
    xh = codec.decompress(buf).cpu().numpy().reshape(-1)
    del x, buf
    st, xref = O.decompress(ref, d.size)
    assert st == O.OK
    bad = np.count_nonzero(xh.view(np.uint32) != xref.view(np.uint32))
    assert bad == 0, f"{bad} decoded values differ"
    info = fz.peek_header(ref[:128].tobytes())
    assert np.abs(xh.astype(np.float64) - d.reshape(-1)).max() <= info.params.eb_abs


# f1 chunk-local mode at the full shapes it applies to (3-D, nx | 2048): c1 and c4, in the
# launch configuration bench.py's chunk-local leg times.
CL_CASES = [
    ("c1", "sines3d", (64, 64, 64), 1e-3),
    ("c4", "nyx_v", (512, 512, 512), 1e-3),
    ("c4", "nyx_rho", (512, 512, 512), 1e-4),
]


@pytest.mark.parametrize("cfg,field,shape,rel", CL_CASES, ids=[f"{c[0]}-{c[1]}-{c[3]}" for c in CL_CASES])
def test_fullsize_chunk_local_parity(cfg, field, shape, rel):
    d = synth.generate(field, shape)
    st, ref = O.compress_chunked(d, O.REL, rel, 16, 2048 // shape[2])
    assert st == O.OK
    codec = fz.Codec(shape, "cuda:0")
    x = torch.from_numpy(d).to("cuda:0")
    buf, size = codec.compress(x, fz.REL | fz.CHUNK_LOCAL, rel)
    got = buf.cpu().numpy()
    assert size == ref.size, (size, ref.size)
    if not np.array_equal(got, ref):
        first = int(np.nonzero(got != ref)[0][0])
        raise AssertionError(f"stream differs from the oracle at byte {first} of {size}")
    del got
    xh = codec.decompress(buf).cpu().numpy().reshape(-1)
    del x, buf
    st, xref = O.decompress(ref, d.size)
    assert st == O.OK
    assert np.count_nonzero(xh.view(np.uint32) != xref.view(np.uint32)) == 0


# f3: the HACC-shaped 1-D field (280,953,867 particle coordinates) under the
# point-wise relative bound, in the launch configuration bench.py times.
@pytest.mark.parametrize("eps", [1e-3])
def test_fullsize_hacc_pwrel_parity(eps):
    d = synth.generate("hacc_x")
    st, ref = O.compress(d, O.PWREL, eps)
    assert st == O.OK
    codec = fz.Codec(d.shape, "cuda:0")
    x = torch.from_numpy(d).to("cuda:0")
    buf, size = codec.compress(x, fz.PWREL, eps)
    assert size == ref.size and np.array_equal(buf.cpu().numpy(), ref)
    xh = codec.decompress(buf).cpu().numpy().reshape(-1)
    del x, buf
    st, xref = O.decompress(ref, d.size)
    assert np.count_nonzero(xh.view(np.uint32) != xref.view(np.uint32)) == 0
    assert np.all(np.abs(xh.astype(np.float64) - d) <= eps * d.astype(np.float64))
