"""f4 on the GPU: two ranks exchange fields as libfz streams through the
compressed link (gloo transport through host memory, both ranks on cuda:0); the received,
decompressed field must equal the oracle's decompression of the peer's field, bit for bit,
and only the stream's bytes may cross."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

SHAPE = (48, 32, 256)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        from paper_2304_12557_b200 import fz, link, synth
        mine = torch.from_numpy(synth.generate("nyx_v", SHAPE, seed=21 + rank)).to("cuda:0")
        lk = link.CompressedLink(link.fz_codec(SHAPE, fz.REL, 1e-3, "cuda:0"), transport="cpu")
        got = torch.empty(SHAPE, dtype=torch.float32, device="cuda:0")
        n = lk.exchange(mine, 1 - rank, got)
        torch.cuda.synchronize()
        q.put((rank, n, got.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_compressed_link_two_ranks_one_gpu():
    import oracle_lib as O
    from paper_2304_12557_b200 import synth
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in range(2)), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, n, got in res:
        peer = synth.generate("nyx_v", SHAPE, seed=21 + (1 - rank))
        st, ref = O.compress(peer, O.REL, 1e-3)
        st, xr = O.decompress(ref, peer.size)
        assert n == ref.size
        assert np.array_equal(got.reshape(-1).view(np.uint32), xr.view(np.uint32))
