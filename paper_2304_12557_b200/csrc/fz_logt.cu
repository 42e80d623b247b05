// fz_logt.cu -- f3: the log transform of the point-wise relative mode
// (FZ_EB_PWREL, "transform the original data using a logarithmic function and compress
// the log-transformed data with the corresponding absolute error bound (computed from the
// point-wise relative error bound)"), reading R25 in DESIGN.md.
//
//   k_log_fwd   y = log32(x) over the field (16-byte loads / stores, grid-stride), the first
//               index outside the domain (x >= FLT_MIN, finite) into ctrl->log_bad
//   k_log_check the status of that element: FZ_ERR_NONFINITE (NaN / Inf) or FZ_ERR_ARG
//               (zero, negative, subnormal), kept only if no earlier error (R24)
//   k_exp_inv   x^ = exp32(y^) in place after the decode's value patch (host-parsed header),
//               or, device-parsed (fz_decompress_async), only when ctrl->dec_flags has bit 3
// Both are HBM-streaming passes (4 + 4 bytes per element) with ~25 binary64 operations per
// element (log32 / exp32 of fz_internal.cuh).
#include "fz_internal.cuh"
#include "fz_launch.h"

namespace fz {

__device__ __forceinline__ float log_elem(float x, uint64_t i, unsigned long long& bad)
{
    if (isfinite(x) && x >= 1.17549435e-38f) return log32(x);
    if (i < bad) bad = i;
    return 0.0f;
}

__global__ void __launch_bounds__(256) k_log_fwd(const float* __restrict__ x, float* __restrict__ y, uint64_t n,
                                                 Ctrl* ctrl)
{
    pdl_begin();
    unsigned long long bad = ~0ull;
    const uint64_t n4 = n / 4;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const float4 v = __ldcs(reinterpret_cast<const float4*>(x) + i);
        float4 o;
        o.x = log_elem(v.x, 4 * i, bad);
        o.y = log_elem(v.y, 4 * i + 1, bad);
        o.z = log_elem(v.z, 4 * i + 2, bad);
        o.w = log_elem(v.w, 4 * i + 3, bad);
        reinterpret_cast<float4*>(y)[i] = o;
    }
    for (uint64_t i = 4 * n4 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        y[i] = log_elem(x[i], i, bad);
    for (int o = 16; o; o >>= 1) bad = min(bad, __shfl_xor_sync(kFull, bad, o));
    if ((threadIdx.x & 31) == 0 && bad != ~0ull) atomicMin(&ctrl->log_bad, bad);
}

__global__ void k_log_check(const float* x, Ctrl* ctrl)
{
    pdl_begin();
    const unsigned long long b = ctrl->log_bad;
    if (b == ~0ull) return;
    atomicCAS(&ctrl->err, 0, isfinite(x[b]) ? (int)FZ_ERR_ARG : (int)FZ_ERR_NONFINITE);
}

__global__ void __launch_bounds__(256) k_exp_inv(float* __restrict__ v, uint64_t n, const Ctrl* ctrl)
{
    pdl_begin();
    if (ctrl != nullptr && (!(ctrl->dec_flags & 8u) || ctrl->err != 0)) return;
    const uint64_t n4 = n / 4;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 a = reinterpret_cast<float4*>(v)[i];
        a.x = exp32(a.x);
        a.y = exp32(a.y);
        a.z = exp32(a.z);
        a.w = exp32(a.w);
        __stcs(reinterpret_cast<float4*>(v) + i, a);
    }
    for (uint64_t i = 4 * n4 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) v[i] = exp32(v[i]);
}

// Device-parsed decode (fz_decompress_async): the value patch (R20) and, when the header has
// bit 3 (f3), x^ = exp32(y^) in one launch.  Without the flag every block patches its share of
// the value outliers (raw bits).  With it every block takes its share of the exp pass and the
// last block to finish (ticket in ctrl->scan_done, zero after the popcount scan, reset here)
// writes the value outliers as exp32 of their y bits -- the order of the separate patch + exp
// launches.
__global__ void __launch_bounds__(256) k_patch_exp_dev(float* __restrict__ v, const uint8_t* payload, Ctrl* ctrl,
                                                       uint64_t n)
{
    pdl_begin();
    __shared__ bool last;
    const bool do_exp = (ctrl->dec_flags & 8u) && ctrl->err == 0;
    const uint64_t cnt = ctrl->dec_nv;
    const uint2* rec = reinterpret_cast<const uint2*>(payload + 16 * ctrl->dec_nnz + 8 * ctrl->dec_nd);
    const uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (uint64_t)gridDim.x * blockDim.x;
    if (!do_exp) {
        for (uint64_t k = i0; k < cnt; k += stride) {
            const uint2 r = rec[k];
            if (r.x < n) v[r.x] = __uint_as_float(r.y);
        }
        return;
    }
    const uint64_t n4 = n / 4;
    for (uint64_t i = i0; i < n4; i += stride) {
        float4 a = reinterpret_cast<float4*>(v)[i];
        a.x = exp32(a.x);
        a.y = exp32(a.y);
        a.z = exp32(a.z);
        a.w = exp32(a.w);
        __stcs(reinterpret_cast<float4*>(v) + i, a);
    }
    for (uint64_t i = 4 * n4 + i0; i < n; i += stride) v[i] = exp32(v[i]);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&ctrl->scan_done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (uint64_t k = threadIdx.x; k < cnt; k += blockDim.x) {
        const uint2 r = rec[k];
        if (r.x < n) v[r.x] = exp32(__uint_as_float(r.y));
    }
    if (threadIdx.x == 0) ctrl->scan_done = 0;
}

static unsigned stream_grid(uint64_t n)
{
    const uint64_t want = (n / 4 + 255) / 256;
    const uint64_t cap = (uint64_t)num_sms() * 8;
    return (unsigned)(want < 1 ? 1 : (want > cap ? cap : want));
}

cudaError_t launch_log_fwd(const float* x, float* y, uint64_t n, Ctrl* ctrl, cudaStream_t st)
{
    {
        LaunchProf lp(K_LOGT, st);
        { const cudaError_t e_ = launch_pdl(k_log_fwd, dim3(stream_grid(n)), dim3(256), 0, st, x, y, n, ctrl); if (e_ != cudaSuccess) return e_; }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    LaunchProf lp(K_LOGT, st);
    { const cudaError_t e_ = launch_pdl(k_log_check, dim3(1), dim3(1), 0, st, x, ctrl); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

cudaError_t launch_exp_inv(float* v, uint64_t n, const Ctrl* dev_ctrl, cudaStream_t st)
{
    LaunchProf lp(K_LOGT, st);
    { const cudaError_t e_ = launch_pdl(k_exp_inv, dim3(stream_grid(n)), dim3(256), 0, st, v, n, dev_ctrl); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

cudaError_t launch_patch_exp_dev(float* v, const uint8_t* payload, Ctrl* ctrl, uint64_t n, cudaStream_t st)
{
    LaunchProf lp(K_VPATCH, st);
    return launch_pdl(k_patch_exp_dev, dim3(stream_grid(n)), dim3(256), 0, st, v, payload, ctrl, n);
}

}  // namespace fz
