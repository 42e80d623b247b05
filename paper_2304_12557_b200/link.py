"""f4: move a field between ranks as its compressed stream.

P:478 models the throughput of compress-then-transfer as
    T_overall = ((BW x CR)^-1 + T_compr^-1)^-1
and leaves "the evaluation in node communication for future work".  Here a rank
compresses its field on its GPU (fz_compress), sends the stream's size and then only the
stream's bytes to the peer (torch.distributed send / recv: NCCL over NVLink on B200s, gloo in
the CPU tests), and the peer decompresses it on its GPU (fz_decompress).  Two equal-size
messages are exchanged per call: an int64 size, then `size` bytes of the stream.

The transfer logic is codec-agnostic: the link takes `compress(field) -> uint8 tensor` and
`decompress(stream, out)` callables.  `fz_codec()` builds the product pair from libfz (CUDA
path, no CPU fallback); the CPU tests pass the oracle as the codec to check the protocol.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable


def t_overall(bw_gbs: float, cr: float, t_compr_gbs: float) -> float:
    """((BW * CR)^-1 + T_compr^-1)^-1, GB/s of original data."""
    return 1.0 / (1.0 / (bw_gbs * cr) + 1.0 / t_compr_gbs)


def t_pipeline(bw_gbs: float, cr: float, t_c_gbs: float, t_d_gbs: float) -> float:
    """Compress, transfer and decompress back to back (no overlap): original GB/s."""
    return 1.0 / (1.0 / t_c_gbs + 1.0 / (bw_gbs * cr) + 1.0 / t_d_gbs)


@dataclass
class Codec:
    compress: Callable      # field tensor -> uint8 tensor (the stream)
    decompress: Callable    # (uint8 tensor, out tensor) -> None
    capacity: int           # upper bound of a stream's size (receive buffer)


def fz_codec(dims, mode, eb, device) -> Codec:
    """The product codec: libfz on `device` (blocking compress: the size is needed on the
    host to post the send)."""
    from . import fz
    c = fz.Codec(dims, device)

    def compress(field):
        buf, size = c.compress(field, mode, eb)
        return buf[:size]

    def decompress(stream, out):
        c.decompress(stream, out=out)

    return Codec(compress, decompress, fz.compress_bound(dims))


class CompressedLink:
    """Sends / receives fields as compressed streams over torch.distributed.

    transport: device of the tensors handed to torch.distributed ("cuda" for NCCL; "cpu" for
    gloo, which stages the stream through host memory)."""

    def __init__(self, codec: Codec, transport="cuda"):
        import torch
        self.codec = codec
        self.transport = torch.device(transport)
        self.rbuf = torch.empty(codec.capacity, dtype=torch.uint8, device=self.transport)
        self.last_sent = 0

    def exchange(self, field, peer: int, out):
        """Sends `field` (compressed) to `peer` and receives the peer's field into `out`
        (decompressed).  Both ranks call it with each other as the peer."""
        import torch
        import torch.distributed as dist
        stream = self.codec.compress(field)
        self.last_sent = int(stream.numel())
        sz = torch.tensor([stream.numel()], dtype=torch.int64, device=self.transport)
        rz = torch.empty(1, dtype=torch.int64, device=self.transport)
        ops = [dist.P2POp(dist.isend, sz, peer), dist.P2POp(dist.irecv, rz, peer)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        n = int(rz.item())
        if n > self.rbuf.numel():
            raise ValueError(f"peer stream of {n} bytes exceeds the receive capacity {self.rbuf.numel()}")
        send = stream.to(self.transport)
        recv = self.rbuf[:n]
        ops = [dist.P2POp(dist.isend, send, peer), dist.P2POp(dist.irecv, recv, peer)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        self.codec.decompress(recv.to(out.device) if out.device != self.transport else recv, out)
        return n

    @staticmethod
    def exchange_raw(field, peer: int, out):
        """The uncompressed baseline: the field's bytes both ways."""
        import torch.distributed as dist
        ops = [dist.P2POp(dist.isend, field, peer), dist.P2POp(dist.irecv, out, peer)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()
