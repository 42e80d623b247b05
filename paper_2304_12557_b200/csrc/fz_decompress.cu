// fz_decompress.cu -- decompression kernels of libfz (B200, sm_100a).
//
// "the decompression pipeline is highly symmetrical"; the paper gives no design.
//   k_decode_tiles  D1-D5(x): payload offsets from the flags (decoupled look-back), gather
//                   of the 16-byte blocks, register un-shuffle, unpack, delta-outlier patch,
//                   segmented inclusive x-scan (decoupled look-back carry); 1-D fields are
//                   dequantized here directly (D6).
//   k_scan_*        D5(y, z): inclusive prefix sums along y and z (reduce-then-scan in
//                   chunks of 32 rows), D6 dequantization fused into the last axis.
//   k_value_patch   D6: value outliers get their raw bits back.
#include "fz_internal.cuh"
#include "fz_launch.h"

namespace fz {

constexpr int kScanChunk = 32;

DecodeLayout decode_layout(const fz_shape& s)
{
    DecodeLayout L{};
    uint64_t d[3] = {1, 1, 1};
    for (uint32_t k = 0; k < s.ndim && k < 3; ++k) d[k] = s.dims[k];
    uint64_t nz = 1, ny = 1, nx = 1;
    if (s.ndim == 1) nx = d[0];
    else if (s.ndim == 2) { ny = d[0]; nx = d[1]; }
    else { nz = d[0]; ny = d[1]; nx = d[2]; }
    const uint64_t n = nz * ny * nx, T = (n + kTileCodes - 1) / kTileCodes;
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    const uint64_t ych = (ny + kScanChunk - 1) / kScanChunk, zch = (nz + kScanChunk - 1) / kScanChunk;
    uint64_t sums = 0;
    if (s.ndim >= 2) sums = nz * ych * nx;
    if (s.ndim == 3 && zch * ny * nx > sums) sums = zch * ny * nx;
    size_t off = 0;
    L.ctrl = off;   off += 512;
    L.st_nnz = off; off = al(off + 8 * T);
    L.st_x = off;   off = al(off + 8 * T);
    L.sums = off;   off = al(off + 4 * sums);
    L.sums_elems = sums;
    L.total = off;
    return L;
}

__global__ void k_decode_init(Ctrl* ctrl, unsigned long long* st_nnz, unsigned long long* st_x,
                              uint32_t ntiles)
{
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    for (uint32_t k = i; k < ntiles; k += gridDim.x * blockDim.x) { st_nnz[k] = 0; st_x[k] = 0; }
    if (i == 0) {
        ctrl->err = 0;
        ctrl->ticket = 0;
        ctrl->nnz = 0;
    }
}

// Outlier lists must be strictly increasing and inside the field.
__global__ void k_validate_outliers(const uint2* rec, uint64_t cnt, uint64_t n, Ctrl* ctrl)
{
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cnt;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t idx = rec[k].x;
        if (idx >= n || (k > 0 && rec[k - 1].x >= idx)) atomicExch(&ctrl->err, (int)FZ_ERR_CORRUPT);
    }
}

// Segmented-sum element: (reset flag, value).  combine(earlier, later).
struct Seg {
    uint32_t f, v;
};
__device__ __forceinline__ Seg seg_combine(Seg e, Seg l)
{
    return l.f ? l : Seg{e.f, e.v + l.v};
}

// ------------------------------------------------------------------------------------
// Tile decoder, a 3-stage software pipeline per CTA (tiles from a ticket):
//   stage 1 (tile t)  : read its 8 flag words, publish its block count (aggregate);
//   stage 2 (tile t1) : payload offset by wide look-back, gather the 16-byte blocks (D2),
//                       un-shuffle (D3), unpack + delta patch (D4), local segmented x-scan,
//                       publish the x aggregate (a tile holding a row start is terminal);
//   stage 3 (tile t2) : x carry by wide look-back, final x-scanned q written (D5 along x;
//                       1-D fields are dequantized here, D6).
// Each look-back targets a tile whose predecessors have had a whole iteration to publish.
// ------------------------------------------------------------------------------------
template <int NDIM>
__global__ void __launch_bounds__(kCta) k_decode_tiles(DecodeArgs a)
{
    __shared__ uint32_t Obuf[32 * 33];
    __shared__ int32_t D[kTileCodes];
    __shared__ uint32_t s_tile[2], s_F[2][8], s_tnnz[2], s_wf[8], s_wv[8];
    __shared__ unsigned long long s_off;
    __shared__ uint32_t s_carry;
    __shared__ uint32_t s_tagf[2], s_tagv[2];
    __shared__ uint64_t s_lo, s_hi;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    Ctrl* ctrl = a.ctrl;
    if (ctrl->err != 0) return;
    const uint32_t n = a.g.n, nx = a.g.nx;
    constexpr uint32_t NONE = 0xFFFFFFFFu;

    if (tid == 0) s_tile[0] = atomicAdd(&ctrl->ticket, 1u);
    __syncthreads();
    uint32_t t1 = NONE, t2 = NONE;
    // stage-3 state of tile t2, per thread
    uint32_t loc2[8];
    uint32_t rmask2 = 0;
    Seg wp2{0, 0}, lx2{0, 0};
#pragma unroll
    for (int u = 0; u < 8; ++u) loc2[u] = 0;

    for (int it = 0;; ++it) {
        const int cur = it & 1;
        const uint32_t t = s_tile[cur];
        const bool work = t < a.tiles;
        if (!work && t1 == NONE && t2 == NONE) break;

        // ---- stage 1: flags of tile t ----
        if (work && lane == 0) s_F[cur][warp] = reinterpret_cast<const uint32_t*>(a.flags)[8 * (uint64_t)t + warp];
        __syncthreads();
        if (tid == 0) s_tile[cur ^ 1] = work ? atomicAdd(&ctrl->ticket, 1u) : NONE;
        if (warp == 0) {
            if (work) {
                uint32_t tn = 0;
#pragma unroll
                for (int w = 0; w < 8; ++w) tn += __popc(s_F[cur][w]);
                if (lane == 0) {
                    s_tnnz[cur] = tn;
                    st_relaxed_u64(&a.st_nnz[t], (t == 0 ? kStInc : kStAgg) | tn);
                }
            }
            if (t1 != NONE) {
                unsigned long long ex = 0;
                if (t1 != 0) {
                    ex = lookback_wide<8, false>(a.st_nnz, t1, 0, kStAgg - 1, &ctrl->err);
                    if (lane == 0) st_relaxed_u64(&a.st_nnz[t1], kStInc | (ex + s_tnnz[cur ^ 1]));
                }
                if (lane == 0) {
                    s_off = ex;
                    if (t1 == a.tiles - 1) ctrl->nnz = ex + s_tnnz[cur ^ 1];
                }
            }
        }
        if (tid == 32 && t1 != NONE) {
            uint64_t lo = 0, hi = 0;
            if (a.nd > 0) {
                const int64_t s1 = (int64_t)t1 * kTileCodes;
                uint64_t l = 0, h = a.nd;
                while (l < h) { uint64_t m = (l + h) / 2; if ((int64_t)a.drec[m].x < s1) l = m + 1; else h = m; }
                lo = l;
                h = a.nd;
                while (l < h) { uint64_t m = (l + h) / 2; if ((int64_t)a.drec[m].x < s1 + kTileCodes) l = m + 1; else h = m; }
                hi = l;
            }
            s_lo = lo;
            s_hi = hi;
        }
        __syncthreads();

        // ---- stage 2: decode tile t1 ----
        uint32_t loc[8];
        uint32_t rmask = 0;
        Seg wp{0, 0}, lex{0, 0};
        if (t1 != NONE) {
            const int64_t s1 = (int64_t)t1 * kTileCodes;
            const uint32_t g0 = (uint32_t)s1 + 8u * tid;
            {
                const uint32_t F = s_F[cur ^ 1][warp];
                uint32_t wpre = 0;
#pragma unroll
                for (int w = 0; w < 8; ++w)
                    if (w < warp) wpre += __popc(s_F[cur ^ 1][w]);
                uint4 blk = make_uint4(0, 0, 0, 0);
                if ((F >> lane) & 1u) {
                    const uint64_t bi = s_off + wpre + __popc(F & ((1u << lane) - 1u));
                    if (bi < a.nnz_total) blk = reinterpret_cast<const uint4*>(a.payload)[bi];
                    else atomicExch(&ctrl->err, (int)FZ_ERR_CORRUPT);
                }
                uint32_t* row = Obuf + (tid >> 3) * 33 + 4 * (tid & 7);
                row[0] = blk.x; row[1] = blk.y; row[2] = blk.z; row[3] = blk.w;
            }
            __syncthreads();
            // D3: column c of O -> row c of A (the same 32x32 bit transpose)
            uint32_t w4[4];
            {
                const int c = tid >> 3, kk = tid & 7;
#pragma unroll
                for (int i = 0; i < 4; ++i) w4[i] = Obuf[(4 * kk + i) * 33 + c];
                transpose32_group8(w4, lane & 7);
            }
            // D4: unpack (0x8000 -> 0, R8), delta outliers
            int32_t dl[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t lo16 = w4[i] & 0xFFFFu, hi16 = w4[i] >> 16;
                dl[2 * i] = (lo16 & 0x8000u) ? -(int32_t)(lo16 & 0x7FFFu) : (int32_t)lo16;
                dl[2 * i + 1] = (hi16 & 0x8000u) ? -(int32_t)(hi16 & 0x7FFFu) : (int32_t)hi16;
            }
            if (s_hi > s_lo) {   // rare, block-uniform
#pragma unroll
                for (int u = 0; u < 8; ++u) D[8 * tid + u] = dl[u];
                __syncthreads();
                for (uint64_t k = s_lo + tid; k < s_hi; k += kCta) {
                    const uint2 r = a.drec[k];
                    D[r.x - (uint32_t)s1] = (int32_t)r.y;
                }
                __syncthreads();
#pragma unroll
                for (int u = 0; u < 8; ++u) dl[u] = D[8 * tid + u];
            }
            // local segmented inclusive x-scan, resets at row starts (x == 0)
            Seg me{0, 0};
            if (nx >= 8) {
                uint32_t x = fmod_(g0, a.dnx);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    if (x == 0) { me.f = 1; me.v = 0; }
                    me.v += (uint32_t)dl[u];
                    loc[u] = me.v;
                    if (me.f) rmask |= 1u << u;
                    if (++x == nx) x = 0;
                }
            } else {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    if (fmod_(g0 + u, a.dnx) == 0) { me.f = 1; me.v = 0; }
                    me.v += (uint32_t)dl[u];
                    loc[u] = me.v;
                    if (me.f) rmask |= 1u << u;
                }
            }
            Seg inc = me;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const Seg up{__shfl_up_sync(kFull, inc.f, o), __shfl_up_sync(kFull, inc.v, o)};
                if (lane >= o) inc = seg_combine(up, inc);
            }
            lex = Seg{__shfl_up_sync(kFull, inc.f, 1), __shfl_up_sync(kFull, inc.v, 1)};
            if (lane == 0) lex = Seg{0, 0};
            if (lane == 31) { s_wf[warp] = inc.f; s_wv[warp] = inc.v; }
            __syncthreads();
            Seg tagg{0, 0};
#pragma unroll
            for (int w = 0; w < 8; ++w) {
                const Seg sw{s_wf[w], s_wv[w]};
                if (w < warp) wp = seg_combine(wp, sw);
                tagg = seg_combine(tagg, sw);
            }
            if (tid == 0) {
                s_tagf[cur] = tagg.f;
                s_tagv[cur] = tagg.v;
                // a row start inside the tile makes its value carry-independent: terminal
                st_relaxed_u64(&a.st_x[t1], ((tagg.f || t1 == 0) ? kStInc : kStAgg) | tagg.v);
            }
        }

        // ---- stage 3: x carry of tile t2 ----
        if (warp == 0 && t2 != NONE) {
            uint32_t carry = 0;
            if (t2 != 0) {
                carry = (uint32_t)lookback_wide<8, false>(a.st_x, t2, 0, 0xFFFFFFFFull, &ctrl->err);
                if (lane == 0 && !s_tagf[cur ^ 1])
                    st_relaxed_u64(&a.st_x[t2], kStInc | (uint32_t)(carry + s_tagv[cur ^ 1]));
            }
            if (lane == 0) s_carry = carry;
        }
        __syncthreads();
        if (t2 != NONE) {
            const int64_t s2 = (int64_t)t2 * kTileCodes;
            Seg acc{0, s_carry};
            acc = seg_combine(acc, wp2);
            acc = seg_combine(acc, lx2);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t g = s2 + 8 * tid + u;
                if (g < (int64_t)n) {
                    const uint32_t qv = ((rmask2 >> u) & 1u) ? loc2[u] : acc.v + loc2[u];
                    if (NDIM == 1 && a.x_out != nullptr) a.x_out[g] = __fmul_rn(__int2float_rn((int32_t)qv), a.w);
                    else a.q_out[g] = (int32_t)qv;
                }
            }
        }
        t2 = t1;
        if (t1 != NONE) {
#pragma unroll
            for (int u = 0; u < 8; ++u) loc2[u] = loc[u];
            rmask2 = rmask;
            wp2 = wp;
            lx2 = lex;
        }
        t1 = work ? t : NONE;
    }
}

// ------------------------------------------------------------------------------------
// Reduce-then-scan along an axis of [outer][L][W] (wrap-around int32 sums).
// ------------------------------------------------------------------------------------
__global__ void k_scan_sums(const int32_t* __restrict__ v, uint64_t outer, uint64_t L, uint64_t W,
                            uint64_t nch, uint32_t* __restrict__ sums)
{
    const uint64_t total = outer * nch * W;
    for (uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; gid < total;
         gid += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t w = gid % W, rest = gid / W, c = rest % nch, o = rest / nch;
        const uint64_t l0 = c * kScanChunk, l1 = min(L, l0 + kScanChunk);
        const int32_t* p = v + (o * L + l0) * W + w;
        uint32_t acc = 0;
        for (uint64_t l = l0; l < l1; ++l, p += W) acc += (uint32_t)__ldg(p);
        sums[gid] = acc;
    }
}

__global__ void k_scan_chunks(uint64_t outer, uint64_t W, uint64_t nch, uint32_t* sums)
{
    const uint64_t total = outer * W;
    for (uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; gid < total;
         gid += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t w = gid % W, o = gid / W;
        uint32_t* p = sums + o * nch * W + w;
        uint32_t acc = 0;
        for (uint64_t c = 0; c < nch; ++c, p += W) {
            const uint32_t x = *p;
            *p = acc;
            acc += x;
        }
    }
}

__global__ void k_scan_apply(int32_t* v, uint64_t outer, uint64_t L, uint64_t W, uint64_t nch,
                             const uint32_t* __restrict__ sums, float dequant_w)
{
    const uint64_t total = outer * nch * W;
    for (uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; gid < total;
         gid += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t w = gid % W, rest = gid / W, c = rest % nch, o = rest / nch;
        const uint64_t l0 = c * kScanChunk, l1 = min(L, l0 + kScanChunk);
        int32_t* p = v + (o * L + l0) * W + w;
        uint32_t acc = sums[gid];
        for (uint64_t l = l0; l < l1; ++l, p += W) {
            acc += (uint32_t)*p;
            if (dequant_w > 0.0f) *reinterpret_cast<float*>(p) = __fmul_rn(__int2float_rn((int32_t)acc), dequant_w);
            else *p = (int32_t)acc;
        }
    }
}

// Single-pass inclusive scan along L when there are many independent columns: one thread
// per column walks L with 8 loads in flight (8 B/element of traffic instead of 12).
__global__ void __launch_bounds__(256) k_scan_walk(int32_t* v, uint64_t outer, uint64_t L, uint64_t W,
                                                   float dequant_w)
{
    const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= outer * W) return;
    const uint64_t w = gid % W, o = gid / W;
    int32_t* p = v + o * L * W + w;
    uint32_t acc = 0;
    uint64_t l = 0;
    for (; l + 8 <= L; l += 8) {
        uint32_t x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = (uint32_t)__ldcs(p + k * W);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            acc += x[k];
            if (dequant_w > 0.0f) __stcs(reinterpret_cast<float*>(p + k * W), __fmul_rn(__int2float_rn((int32_t)acc), dequant_w));
            else __stcs(p + k * W, (int32_t)acc);
        }
        p += 8 * W;
    }
    for (; l < L; ++l, p += W) {
        acc += (uint32_t)*p;
        if (dequant_w > 0.0f) *reinterpret_cast<float*>(p) = __fmul_rn(__int2float_rn((int32_t)acc), dequant_w);
        else *p = (int32_t)acc;
    }
}

__global__ void k_value_patch(float* out, const uint2* rec, uint64_t cnt, uint64_t n)
{
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cnt;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint2 r = rec[k];
        if (r.x < n) out[r.x] = __uint_as_float(r.y);
    }
}

// ------------------------------------------------------------------------------------
static unsigned grid_for(uint64_t work, int per_thread = 1)
{
    uint64_t g = (work / per_thread + 255) / 256;
    const uint64_t cap = (uint64_t)num_sms() * 16;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

cudaError_t launch_decode_init(Ctrl* ctrl, unsigned long long* st_nnz, unsigned long long* st_x,
                               uint32_t ntiles, cudaStream_t st)
{
    LaunchProf lp(K_DINIT, st);
    k_decode_init<<<grid_for(ntiles), 256, 0, st>>>(ctrl, st_nnz, st_x, ntiles);
    return cudaGetLastError();
}

cudaError_t launch_validate_outliers(const uint2* rec, uint64_t cnt, uint64_t n, Ctrl* ctrl,
                                     cudaStream_t st)
{
    if (cnt == 0) return cudaSuccess;
    LaunchProf lp(K_VALIDATE, st);
    k_validate_outliers<<<grid_for(cnt), 256, 0, st>>>(rec, cnt, n, ctrl);
    return cudaGetLastError();
}

template <int NDIM>
static cudaError_t launch_decode_t(const DecodeArgs& a_in, cudaStream_t st)
{
    DecodeArgs a = a_in;
    a.dnx = make_fastdiv(a.g.nx);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_decode_tiles<NDIM>, kCta, 0);
    if (per_sm < 1) per_sm = 1;
    uint64_t grid = (uint64_t)per_sm * num_sms();
    if (grid > a.tiles) grid = a.tiles;
    if (grid == 0) return cudaSuccess;
    k_decode_tiles<NDIM><<<(unsigned)grid, kCta, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_decode_tiles(const DecodeArgs& a, cudaStream_t st)
{
    LaunchProf lp(K_DECODE, st);
    switch (a.g.ndim) {
        case 1: return launch_decode_t<1>(a, st);
        case 2: return launch_decode_t<2>(a, st);
        default: return launch_decode_t<3>(a, st);
    }
}

cudaError_t launch_scan_axis(int32_t* data, uint64_t outer, uint64_t L, uint64_t W, uint32_t* sums,
                             float dequant_w, cudaStream_t st)
{
    if (outer * W >= 32768) {
        LaunchProf lp(K_SCAN_APPLY, st);
        k_scan_walk<<<(unsigned)((outer * W + 255) / 256), 256, 0, st>>>(data, outer, L, W, dequant_w);
        return cudaGetLastError();
    }
    const uint64_t nch = (L + kScanChunk - 1) / kScanChunk;
    const uint64_t work = outer * nch * W;
    {
        LaunchProf lp(K_SCAN_SUMS, st);
        k_scan_sums<<<grid_for(work), 256, 0, st>>>(data, outer, L, W, nch, sums);
    }
    {
        LaunchProf lp(K_SCAN_CHUNKS, st);
        k_scan_chunks<<<grid_for(outer * W), 256, 0, st>>>(outer, W, nch, sums);
    }
    {
        LaunchProf lp(K_SCAN_APPLY, st);
        k_scan_apply<<<grid_for(work), 256, 0, st>>>(data, outer, L, W, nch, sums, dequant_w);
    }
    return cudaGetLastError();
}

cudaError_t launch_value_patch(float* out, const uint2* vrec, uint64_t cnt, uint64_t n, cudaStream_t st)
{
    if (cnt == 0) return cudaSuccess;
    LaunchProf lp(K_VPATCH, st);
    k_value_patch<<<grid_for(cnt), 256, 0, st>>>(out, vrec, cnt, n);
    return cudaGetLastError();
}

}  // namespace fz
