"""Thin ctypes binding of libfz.so (include/fz.h): argument marshalling only.

Every step of the compression path runs in the CUDA kernels of libfz.so.  PyTorch provides
device memory and streams.  There is no CPU fallback: if libfz.so is missing the import of
this module's functions raises (run `python -m paper_2304_12557_b200.build` or
`__graft_entry__.build()`).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FZ_LIB") or os.path.join(PKG, "libfz.so")  # FZ_LIB: A/B builds

ABS, REL, PWREL = 0, 1, 2   # PWREL: f3 point-wise relative bound via the log transform
CHUNK_LOCAL = 0x100   # f1 chunk-local Lorenzo (fz.h FZ_CHUNK_LOCAL), OR into the mode
STATUS = {0: "OK", 1: "ERR_ARG", 2: "ERR_NONFINITE", 3: "ERR_EB_TOO_SMALL", 4: "ERR_CAPACITY",
          5: "ERR_CORRUPT", 6: "ERR_WORKSPACE", 7: "ERR_CUDA"}
OK, ERR_ARG, ERR_NONFINITE, ERR_EB_TOO_SMALL, ERR_CAPACITY, ERR_CORRUPT, ERR_WORKSPACE, ERR_CUDA = range(8)


class FZError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = f"{where}: {STATUS.get(status, status)}"
        if status == ERR_CUDA:
            msg += " (" + lib().fz_last_cuda_error().decode() + ")"
        super().__init__(msg)


class Shape(C.Structure):
    _fields_ = [("ndim", C.c_uint32), ("reserved", C.c_uint32), ("dims", C.c_uint64 * 3)]


class Params(C.Structure):
    _fields_ = [("eb_input", C.c_double), ("eb_abs", C.c_double), ("w", C.c_float), ("r", C.c_float),
                ("eb32", C.c_float), ("mn", C.c_float), ("mx", C.c_float), ("mode", C.c_uint32),
                ("fallback", C.c_uint32)]


class Counts(C.Structure):
    _fields_ = [("nnz", C.c_uint64), ("n_delta", C.c_uint64), ("n_value", C.c_uint64)]


class Info(C.Structure):
    _fields_ = [("shape", Shape), ("n", C.c_uint64), ("tiles", C.c_uint64), ("total_size", C.c_uint64),
                ("counts", Counts), ("params", Params), ("version", C.c_uint32), ("flags", C.c_uint32)]


_lib = None


def lib():
    """Load libfz.so (fails loudly when the CUDA library has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libfz.so not built at {LIB_PATH}; run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    P, S, u64, i = C.c_void_p, C.c_size_t, C.c_uint64, C.c_int
    pS, pP, pC = C.POINTER(Shape), C.POINTER(Params), C.POINTER(Counts)
    sig = {
        "fz_compress_bound": ([pS], S),
        "fz_workspace_bytes": ([pS], S),
        "fz_workspace_bytes_mode": ([pS, i], S),
        "fz_decompress_workspace_bytes": ([pS], S),
        "fz_derive_params": ([C.c_float, C.c_float, i, C.c_double, pP], i),
        "fz_compress": ([P, pS, i, C.c_double, P, S, C.POINTER(S), P, S, P], i),
        "fz_compress_with_params": ([P, pS, pP, P, S, C.POINTER(S), P, S, P], i),
        "fz_decompress": ([P, S, P, u64, P, S, P], i),
        "fz_decompress_hdr": ([P, S, P, P, u64, P, S, P], i),
        "fz_last_header": ([P], i),
        "fz_decompress_hdr_async": ([P, S, P, P, u64, P, S, P], i),
        "fz_decompress_result": ([P, P], i),
        "fz_decompress_async": ([P, S, pS, P, P, S, P], i),
        "fz_compress_async": ([P, pS, i, C.c_double, P, S, P, S, P], i),
        "fz_compress_result": ([P, S, C.POINTER(S), P], i),
        "fz_compress_host": ([P, pS, i, C.c_double, P, S, C.POINTER(S), P, P, S, P, S, P], i),
        "fz_decompress_host": ([P, S, P, u64, P, P, P, S, P], i),
        "fz_peek_header": ([P, S, C.POINTER(Info)], i),
        "fz_strerror": ([i], C.c_char_p),
        "fz_last_cuda_error": ([], C.c_char_p),
        "fz_slab_range": ([P, u64, C.POINTER(C.c_float), C.POINTER(C.c_float), C.POINTER(C.c_int64), P, S, P], i),
        "fz_slab_stage_bound": ([pS, u64, u64], S),
        "fz_slab_compress": ([P, u64, u64, pS, u64, u64, pP, P, S, pC, P, S, P], i),
        "fz_slab_place": ([P, pS, u64, u64, pC, pC, pC, pP, i, P, S, P], i),
        "fz_debug_workspace_bytes": ([pS], S),
        "fz_debug_quantize": ([P, pS, pP, P, P, P, u64, C.POINTER(u64), P, P, u64, C.POINTER(u64), P, S, P], i),
        "fz_debug_decode_q": ([P, S, P, u64, P, S, P], i),
        "fz_last_launch_count": ([], i),
        "fz_debug_set_variant": ([i], None),
        "fz_profile_enable": ([i], None),
        "fz_profile_mask": ([C.c_ulonglong], None),
        "fz_profile_read": ([C.POINTER(C.c_double), C.POINTER(C.c_int), i], i),
        "fz_kernel_name": ([i], C.c_char_p),
        "fz_profile_timeline": ([C.POINTER(C.c_int), C.POINTER(C.c_float), C.POINTER(C.c_float), i], i),
        "fz_slab_agg_elems": ([pS], u64),
        "fz_slab_decode": ([P, pC, pS, u64, u64, P, P, P, S, P], i),
        "fz_slab_carry": ([P, C.c_uint32, u64, P, P], i),
        "fz_slab_finish": ([P, P, P, pC, pS, u64, u64, pP, P], i),
        "fz_slab_decode_cl": ([P, pC, pS, u64, u64, pP, P, P, S, P], i),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _check(st: int, where: str):
    if st != OK:
        raise FZError(st, where)


def make_shape(dims) -> Shape:
    dims = tuple(int(d) for d in dims)
    s = Shape()
    s.ndim = len(dims)
    for k in range(3):
        s.dims[k] = dims[k] if k < len(dims) else 1
    return s


def _ptr(t) -> int:
    return C.c_void_p(t.data_ptr())


def _stream(stream=None):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def compress_bound(dims) -> int:
    return lib().fz_compress_bound(C.byref(make_shape(dims)))


def workspace_bytes(dims) -> int:
    return lib().fz_workspace_bytes(C.byref(make_shape(dims)))


def workspace_bytes_mode(dims, mode) -> int:
    """Compress workspace for `mode` (FZ_EB_PWREL adds the 4N-byte log field)."""
    return lib().fz_workspace_bytes_mode(C.byref(make_shape(dims)), int(mode))


def decompress_workspace_bytes(dims) -> int:
    return lib().fz_decompress_workspace_bytes(C.byref(make_shape(dims)))


def derive_params(mn: float, mx: float, mode: int, eb: float) -> Params:
    p = Params()
    _check(lib().fz_derive_params(mn, mx, mode, eb, C.byref(p)), "fz_derive_params")
    return p


def last_launch_count() -> int:
    return lib().fz_last_launch_count()


def profile_enable(on: bool = True):
    lib().fz_profile_enable(int(on))


def profile_timeline(max_records: int = 4096) -> list:
    """[(kernel name, start ms, end ms)] of the launches recorded since the last profile_read,
    relative to the first one (profiling on)."""
    ids = (C.c_int * max_records)()
    a = (C.c_float * max_records)()
    b = (C.c_float * max_records)()
    k = lib().fz_profile_timeline(ids, a, b, max_records)
    return [(lib().fz_kernel_name(ids[i]).decode(), a[i], b[i]) for i in range(k)]


def profile_only(names):
    """Record events only for the named kernels (others launch without event records)."""
    ids = {lib().fz_kernel_name(i).decode(): i for i in range(64) if lib().fz_kernel_name(i) != b"?"}
    mask = 0
    for n in names:
        mask |= 1 << ids[n]
    lib().fz_profile_mask(mask)


def profile_read() -> dict:
    """{kernel name: (total ms, launches)} since the last read (CUDA events per launch)."""
    ms = (C.c_double * 32)()
    cnt = (C.c_int * 32)()
    k = lib().fz_profile_read(ms, cnt, 32)
    return {lib().fz_kernel_name(i).decode(): (ms[i], cnt[i]) for i in range(k) if cnt[i]}


def _u8(n, device):
    import torch
    # 16-byte alignment: torch's caching allocator returns >= 512-byte aligned blocks
    return torch.empty(max(int(n), 16), dtype=torch.uint8, device=device)


class Codec:
    """Holds device buffers for repeated compress/decompress of one shape (no allocation
    inside the timed calls)."""

    def __init__(self, dims, device="cuda"):
        self.dims = tuple(int(d) for d in dims)
        self.shape = make_shape(self.dims)
        self.n = int(np.prod(self.dims))
        self.device = device
        self.cap = compress_bound(self.dims)
        self.out = _u8(self.cap, device)
        self.work = _u8(workspace_bytes(self.dims), device)
        self.dwork = _u8(decompress_workspace_bytes(self.dims), device)
        self.hdr = (C.c_uint8 * 128)()   # host copy of the last stream's header
        self.hdr_size = None             # size of the stream it belongs to (None: no header)

    def compress(self, field, mode=REL, eb=1e-3, params: Params | None = None, stream=None, sync=True):
        """Returns (uint8 view of the stream, size).  With sync=False the whole compression is
        only enqueued (fz_compress_async) and (the output buffer, None) is returned; the size
        comes from compress_result()."""
        need = workspace_bytes_mode(self.dims, (params.mode if params is not None else mode) & ~CHUNK_LOCAL)
        if self.work.numel() < need:      # FZ_EB_PWREL: room for the log field
            self.work = _u8(need, self.device)
        if not sync:
            assert params is None
            st = lib().fz_compress_async(_ptr(field), C.byref(self.shape), mode, eb, _ptr(self.out), self.cap,
                                         _ptr(self.work), self.work.numel(), _stream(stream))
            _check(st, "fz_compress_async")
            self.hdr_size = None
            return self.out, None
        size = C.c_size_t()
        if params is None:
            st = lib().fz_compress(_ptr(field), C.byref(self.shape), mode, eb, _ptr(self.out), self.cap,
                                   C.byref(size), _ptr(self.work), self.work.numel(), _stream(stream))
        else:
            st = lib().fz_compress_with_params(_ptr(field), C.byref(self.shape), C.byref(params),
                                               _ptr(self.out), self.cap, C.byref(size), _ptr(self.work),
                                               self.work.numel(), _stream(stream))
        _check(st, "fz_compress")
        _check(lib().fz_last_header(self.hdr), "fz_last_header")
        self.hdr_size = size.value
        return self.out[: size.value], size.value

    def decompress(self, buf, out=None, stream=None, sync=True):
        """Decompresses `buf`; when it is this codec's last output, the header comes from the
        host copy kept by compress (fz_decompress_hdr: no blocking header read).  With
        sync=False (own output only) the decode is only enqueued; call result() before using
        `out`."""
        import torch
        if out is None:
            out = torch.empty(self.dims, dtype=torch.float32, device=self.device)
        own = (self.hdr_size is not None and buf.data_ptr() == self.out.data_ptr()
               and buf.numel() == self.hdr_size)
        if own and not sync:
            st = lib().fz_decompress_hdr_async(_ptr(buf), buf.numel(), self.hdr, _ptr(out), self.n,
                                               _ptr(self.dwork), self.dwork.numel(), _stream(stream))
            _check(st, "fz_decompress_hdr_async")
            return out
        if own:
            st = lib().fz_decompress_hdr(_ptr(buf), buf.numel(), self.hdr, _ptr(out), self.n, _ptr(self.dwork),
                                         self.dwork.numel(), _stream(stream))
        else:
            st = lib().fz_decompress(_ptr(buf), buf.numel(), _ptr(out), self.n, _ptr(self.dwork),
                                     self.dwork.numel(), _stream(stream))
        _check(st, "fz_decompress")
        return out


def _codec_result(self, stream=None):
    """Waits for an asynchronous decompress and raises on a recorded stream error."""
    _check(lib().fz_decompress_result(_ptr(self.dwork), _stream(stream)), "fz_decompress_result")


def _codec_compress_result(self, stream=None) -> int:
    """Waits for an asynchronous compress; returns the stream size."""
    size = C.c_size_t()
    _check(lib().fz_compress_result(_ptr(self.work), self.cap, C.byref(size), _stream(stream)),
           "fz_compress_result")
    return size.value


def _codec_decompress_device(self, buf, out=None, stream=None):
    """Fully device-driven asynchronous decompress (fz_decompress_async): the header is parsed
    on the device, nothing waits for the host; call result() before using `out`."""
    import torch
    if out is None:
        out = torch.empty(self.dims, dtype=torch.float32, device=self.device)
    st = lib().fz_decompress_async(_ptr(buf), buf.numel(), C.byref(self.shape), _ptr(out), _ptr(self.dwork),
                                   self.dwork.numel(), _stream(stream))
    _check(st, "fz_decompress_async")
    return out


Codec.result = _codec_result
Codec.compress_result = _codec_compress_result
Codec.decompress_device = _codec_decompress_device


def compress(field, mode=REL, eb=1e-3, params: Params | None = None, stream=None):
    """fz_compress on a CUDA float32 tensor; returns a fresh uint8 tensor with the stream."""
    codec = Codec(tuple(field.shape), field.device)
    buf, size = codec.compress(field.contiguous(), mode, eb, params, stream)
    return buf.clone()


def decompress(buf, dims=None, stream=None):
    import torch
    info = peek_header(buf[:128].cpu().numpy().tobytes())
    if dims is None:
        dims = tuple(int(info.shape.dims[k]) for k in range(info.shape.ndim))
    n = int(np.prod(dims))
    out = torch.empty(dims, dtype=torch.float32, device=buf.device)
    dwork = _u8(decompress_workspace_bytes(dims), buf.device)
    st = lib().fz_decompress(_ptr(buf), buf.numel(), _ptr(out), n, _ptr(dwork), dwork.numel(), _stream(stream))
    _check(st, "fz_decompress")
    return out


def peek_header(hdr: bytes) -> Info:
    info = Info()
    b = C.create_string_buffer(bytes(hdr), len(hdr))
    _check(lib().fz_peek_header(b, len(hdr), C.byref(info)), "fz_peek_header")
    return info


def debug_quantize(field, params: Params, cap: int | None = None, stream=None):
    """Stage hook C1-C3: (codes uint16, didx, dval, vidx, vbits) as CUDA tensors."""
    import torch
    dims = tuple(field.shape)
    n = field.numel()
    cap = n if cap is None else cap
    dev = field.device
    codes = torch.empty(n, dtype=torch.int16, device=dev)
    didx = torch.empty(max(cap, 4), dtype=torch.int32, device=dev)
    dval = torch.empty(max(cap, 4), dtype=torch.int32, device=dev)
    vidx = torch.empty(max(cap, 4), dtype=torch.int32, device=dev)
    vbits = torch.empty(max(cap, 4), dtype=torch.int32, device=dev)
    work = _u8(lib().fz_debug_workspace_bytes(C.byref(make_shape(dims))), dev)
    nd, nv = C.c_uint64(), C.c_uint64()
    st = lib().fz_debug_quantize(_ptr(field), C.byref(make_shape(dims)), C.byref(params), _ptr(codes),
                                 _ptr(didx), _ptr(dval), cap, C.byref(nd), _ptr(vidx), _ptr(vbits), cap,
                                 C.byref(nv), _ptr(work), work.numel(), _stream(stream))
    _check(st, "fz_debug_quantize")
    return codes, didx[: nd.value], dval[: nd.value], vidx[: nv.value], vbits[: nv.value]


def debug_set_variant(bits: int) -> None:
    """A/B experiments only: process-wide kernel-variant bits (0 = product configuration)."""
    lib().fz_debug_set_variant(int(bits))


def debug_decode_q(buf, dims, stream=None):
    import torch
    n = int(np.prod(dims))
    q = torch.empty(n, dtype=torch.int32, device=buf.device)
    dwork = _u8(decompress_workspace_bytes(dims), buf.device)
    st = lib().fz_debug_decode_q(_ptr(buf), buf.numel(), _ptr(q), n, _ptr(dwork), dwork.numel(), _stream(stream))
    _check(st, "fz_debug_decode_q")
    return q


def compress_host(h_field: np.ndarray, mode, eb, d_field, d_out, work, h_out: np.ndarray, stream=None):
    """fz_compress_host: host fp32 array in, host stream bytes out (H2D + kernels + D2H)."""
    dims = h_field.shape
    size = C.c_size_t()
    st = lib().fz_compress_host(h_field.ctypes.data_as(C.c_void_p), C.byref(make_shape(dims)), mode, eb,
                                h_out.ctypes.data_as(C.c_void_p), h_out.nbytes, C.byref(size), _ptr(d_field),
                                _ptr(d_out), d_out.numel(), _ptr(work), work.numel(), _stream(stream))
    _check(st, "fz_compress_host")
    return size.value


def decompress_host(h_in: np.ndarray, size: int, h_field: np.ndarray, d_in, d_field, dwork, stream=None):
    st = lib().fz_decompress_host(h_in.ctypes.data_as(C.c_void_p), size, h_field.ctypes.data_as(C.c_void_p),
                                  h_field.size, _ptr(d_in), _ptr(d_field), _ptr(dwork), dwork.numel(),
                                  _stream(stream))
    _check(st, "fz_decompress_host")


# ---- slab API (multi-GPU) ------------------------------------------------------------
def slab_range(slab, work, stream=None):
    mn, mx, bad = C.c_float(), C.c_float(), C.c_int64()
    st = lib().fz_slab_range(_ptr(slab), slab.numel(), C.byref(mn), C.byref(mx), C.byref(bad), _ptr(work),
                             work.numel(), _stream(stream))
    if st == ERR_NONFINITE:
        return mn.value, mx.value, bad.value
    _check(st, "fz_slab_range")
    return mn.value, mx.value, -1


def slab_stage_bound(dims, tb, te) -> int:
    return lib().fz_slab_stage_bound(C.byref(make_shape(dims)), tb, te)


def slab_compress(slab, slab_first, dims, tb, te, params: Params, stage, work, stream=None) -> Counts:
    c = Counts()
    st = lib().fz_slab_compress(_ptr(slab), slab_first, slab.numel(), C.byref(make_shape(dims)), tb, te,
                                C.byref(params), _ptr(stage), stage.numel(), C.byref(c), _ptr(work),
                                work.numel(), _stream(stream))
    _check(st, "fz_slab_compress")
    return c


def slab_place(stage, dims, tb, te, local: Counts, before: Counts, totals: Counts, params: Params,
               write_header: bool, out, stream=None):
    st = lib().fz_slab_place(_ptr(stage), C.byref(make_shape(dims)), tb, te, C.byref(local), C.byref(before),
                             C.byref(totals), C.byref(params), int(write_header), _ptr(out), out.numel(),
                             _stream(stream))
    _check(st, "fz_slab_place")


def slab_agg_elems(dims) -> int:
    return lib().fz_slab_agg_elems(C.byref(make_shape(dims)))


def slab_decode(stage, counts: Counts, dims, tb, te, q, agg, work, stream=None):
    st = lib().fz_slab_decode(_ptr(stage), C.byref(counts), C.byref(make_shape(dims)), tb, te, _ptr(q), _ptr(agg),
                              _ptr(work), work.numel(), _stream(stream))
    _check(st, "fz_slab_decode")


def slab_decode_cl(stage, counts: Counts, dims, tb, te, params: Params, out, work, stream=None):
    """f1: decode a chunk-local slab on its own (no carry from other ranks) into fp32 `out`."""
    st = lib().fz_slab_decode_cl(_ptr(stage), C.byref(counts), C.byref(make_shape(dims)), tb, te, C.byref(params),
                                 _ptr(out), _ptr(work), work.numel(), _stream(stream))
    _check(st, "fz_slab_decode_cl")


def slab_carry(aggs, nbefore: int, elems: int, carry, stream=None):
    st = lib().fz_slab_carry(_ptr(aggs) if aggs is not None else None, nbefore, elems, _ptr(carry), _stream(stream))
    _check(st, "fz_slab_carry")


def slab_finish(q, carry, stage, counts: Counts, dims, tb, te, params: Params, stream=None):
    st = lib().fz_slab_finish(_ptr(q), _ptr(carry), _ptr(stage), C.byref(counts), C.byref(make_shape(dims)), tb, te,
                              C.byref(params), _stream(stream))
    _check(st, "fz_slab_finish")
