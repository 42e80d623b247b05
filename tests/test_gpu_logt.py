"""GPU parity of f3 (FZ_EB_PWREL, P:314 log transform + the corresponding ABS bound, reading
R25): the CUDA path's stream and decoded field against the oracle's, bit for bit, and the
point-wise relative guarantee |x^ - x| <= eps |x| on every element."""
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
FLT_MIN = np.float32(np.finfo(np.float32).tiny)
FLT_MAX = np.float32(np.finfo(np.float32).max)

FIELDS = [
    ("hacc_x", lambda: synth.generate("hacc_x", (1_000_003,))),
    ("nyx_rho_zr", lambda: synth.generate("nyx_rho", (40, 32, 256))),      # row-walking paths
    ("nyx_rho_ragged", lambda: synth.generate("nyx_rho", (21, 33, 47))),
    ("loguniform_2d", lambda: np.exp2(np.random.default_rng(5).uniform(-120, 120, (300, 700))).astype(np.float32)),
    ("extremes", lambda: np.array([FLT_MIN, FLT_MAX, 1.0, 3.0, FLT_MAX, FLT_MIN] * 1700, np.float32)),
    ("ones", lambda: np.ones(10000, np.float32)),
]


def _check(d, eps, name):
    st, ref = O.compress(d, O.PWREL, eps)
    assert st == O.OK
    codec = fz.Codec(d.shape, DEV)
    x = torch.from_numpy(np.ascontiguousarray(d)).to(DEV)
    buf, size = codec.compress(x, fz.PWREL, eps)
    got = buf.cpu().numpy()
    assert size == ref.size and np.array_equal(got, ref), f"{name}: stream differs"
    xh = codec.decompress(buf).cpu().numpy().reshape(-1)
    st, xr = O.decompress(ref, d.size)
    assert np.array_equal(xh.view(np.uint32), xr.view(np.uint32)), f"{name}: decoded field differs"
    err = np.abs(xh.astype(np.float64) - d.reshape(-1).astype(np.float64))
    assert np.all(err <= eps * np.abs(d.reshape(-1).astype(np.float64)))
    return codec, x, ref


@pytest.mark.parametrize("name,gen", FIELDS, ids=[f[0] for f in FIELDS])
@pytest.mark.parametrize("eps", [1e-2, 1e-3, 1e-4])
def test_pwrel_parity(name, gen, eps):
    _check(gen(), eps, f"{name}@{eps}")


def test_pwrel_async_and_device_parsed_decode():
    d = synth.generate("nyx_rho", (40, 32, 256))
    codec, x, ref = _check(d, 1e-3, "async")
    codec.compress(x, fz.PWREL, 1e-3, sync=False)
    size = codec.compress_result()
    assert size == ref.size and np.array_equal(codec.out[:size].cpu().numpy(), ref)
    xh = codec.decompress_device(codec.out[:size])
    codec.result()
    st, xr = O.decompress(ref, d.size)
    assert np.array_equal(xh.cpu().numpy().reshape(-1).view(np.uint32), xr.view(np.uint32))
    # a non-log stream through the same device path is left alone by the exp kernel
    buf, size = codec.compress(x, fz.REL, 1e-3)
    xh = codec.decompress_device(buf)
    codec.result()
    st, ref2 = O.compress(d, O.REL, 1e-3)
    st, xr2 = O.decompress(ref2, d.size)
    assert np.array_equal(xh.cpu().numpy().reshape(-1).view(np.uint32), xr2.view(np.uint32))


@pytest.mark.parametrize("bad,status", [(0.0, fz.ERR_ARG), (-2.0, fz.ERR_ARG), (1e-40, fz.ERR_ARG),
                                        (np.nan, fz.ERR_NONFINITE), (np.inf, fz.ERR_NONFINITE)])
def test_pwrel_domain_errors(bad, status):
    d = np.ones((64, 64), np.float32)
    d.reshape(-1)[777] = bad
    codec = fz.Codec(d.shape, DEV)
    with pytest.raises(fz.FZError) as e:
        codec.compress(torch.from_numpy(d).to(DEV), fz.PWREL, 1e-3)
    assert e.value.status == status == O.compress(d, O.PWREL, 1e-3)[0]


def test_pwrel_first_bad_element_decides():
    d = np.ones(100000, np.float32)
    d[5000] = 0.0          # domain error first
    d[9000] = np.nan
    codec = fz.Codec(d.shape, DEV)
    with pytest.raises(fz.FZError) as e:
        codec.compress(torch.from_numpy(d).to(DEV), fz.PWREL, 1e-3)
    assert e.value.status == fz.ERR_ARG == O.compress(d, O.PWREL, 1e-3)[0]
    d[3000] = np.inf       # now the non-finite element comes first
    with pytest.raises(fz.FZError) as e:
        codec.compress(torch.from_numpy(d).to(DEV), fz.PWREL, 1e-3)
    assert e.value.status == fz.ERR_NONFINITE == O.compress(d, O.PWREL, 1e-3)[0]
