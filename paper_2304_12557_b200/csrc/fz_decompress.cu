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

// Look-back with one 62-bit count (payload offsets).
__device__ __forceinline__ unsigned long long lookback_count(unsigned long long* st, uint32_t t,
                                                             unsigned long long cnt)
{
    const int lane = threadIdx.x & 31;
    const unsigned long long kAgg = 1ull << 62, kInc = 2ull << 62, kMask = kAgg - 1;
    if (t == 0) {
        if (lane == 0) st_release_u64(&st[0], kInc | cnt);
        return 0;
    }
    if (lane == 0) st_release_u64(&st[t], kAgg | cnt);
    unsigned long long ex = 0;
    int64_t p = (int64_t)t - 1;
    while (true) {
        const int64_t q = p - lane;
        unsigned long long s = kInc;
        if (q >= 0) {
            do { s = ld_acquire_u64(&st[q]); } while ((s >> 62) == 0);
        }
        const uint32_t incl = __ballot_sync(kFull, (s >> 62) == 2);
        const int stop = incl ? __ffs(incl) - 1 : 31;
        unsigned long long c = lane <= stop ? (s & kMask) : 0;
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
        ex += c;
        if (incl) break;
        p -= 32;
    }
    if (lane == 0) st_release_u64(&st[t], kInc | (ex + cnt));
    return ex;
}

// Segmented-sum element: (reset flag, value).  combine(earlier, later).
struct Seg {
    uint32_t f, v;
};
__device__ __forceinline__ Seg seg_combine(Seg e, Seg l)
{
    return l.f ? l : Seg{e.f, e.v + l.v};
}

// Look-back for the segmented x-scan: status = state(2) | reset(1) @32 | value(32).
// Returns the carry into tile t (sum since the last row start before the tile).
__device__ __forceinline__ uint32_t lookback_seg(unsigned long long* st, uint32_t t, Seg agg)
{
    const int lane = threadIdx.x & 31;
    const unsigned long long kAgg = 1ull << 62, kInc = 2ull << 62;
    auto pack = [](Seg s) { return ((unsigned long long)s.f << 32) | s.v; };
    if (t == 0) {
        if (lane == 0) st_release_u64(&st[0], kInc | pack(agg));
        return 0;
    }
    // a tile containing a row start has a carry-independent inclusive value
    if (lane == 0) st_release_u64(&st[t], (agg.f ? kInc : kAgg) | pack(agg));
    Seg acc{0, 0};
    int64_t p = (int64_t)t - 1;
    while (true) {
        const int64_t q = p - lane;
        unsigned long long s = kInc;   // before tile 0: identity, inclusive
        if (q >= 0) {
            do { s = ld_acquire_u64(&st[q]); } while ((s >> 62) == 0);
        }
        Seg e{(uint32_t)((s >> 32) & 1u), (uint32_t)s};
        const bool term = ((s >> 62) == 2) || e.f;
        const uint32_t tm = __ballot_sync(kFull, term);
        const int stop = tm ? __ffs(tm) - 1 : 31;
        if (lane > stop) e = Seg{0, 0};
        // ordered reduction: lane i holds range [i, i+o); higher lanes are earlier tiles
        for (int o = 1; o < 32; o <<= 1) {
            Seg hi{__shfl_down_sync(kFull, e.f, o), __shfl_down_sync(kFull, e.v, o)};
            if (lane + o < 32) e = seg_combine(hi, e);
        }
        acc = seg_combine(Seg{__shfl_sync(kFull, e.f, 0), __shfl_sync(kFull, e.v, 0)}, acc);
        if (tm) break;
        p -= 32;
    }
    if (lane == 0 && !agg.f) st_release_u64(&st[t], kInc | pack(seg_combine(acc, agg)));
    return acc.v;
}

template <int NDIM>
__global__ void __launch_bounds__(kCta) k_decode_tiles(DecodeArgs a)
{
    __shared__ uint32_t Obuf[32 * 33];
    __shared__ int32_t D[kTileCodes];
    __shared__ uint32_t s_tile[2], s_F[8], s_wf[8], s_wv[8];
    __shared__ unsigned long long s_off;
    __shared__ uint32_t s_carry;
    __shared__ uint64_t s_lo, s_hi;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    Ctrl* ctrl = a.ctrl;
    if (ctrl->err != 0) return;
    const uint32_t n = a.g.n, nx = a.g.nx;

    if (tid == 0) s_tile[0] = atomicAdd(&ctrl->ticket, 1u);
    __syncthreads();
    for (int it = 0;; ++it) {
        const uint32_t t = s_tile[it & 1];
        if (t >= a.tiles) break;
        const int64_t s = (int64_t)t * kTileCodes;
        const int64_t g0 = s + 8 * tid;

        // ---- D1: flags and payload offsets ----
        const uint32_t F = reinterpret_cast<const uint32_t*>(a.flags)[8 * (uint64_t)t + warp];
        const bool nz = (F >> lane) & 1u;
        if (lane == 0) s_F[warp] = F;
        if (tid == 0 && a.nd > 0) {
            uint64_t lo = 0, hi = a.nd;           // first record with idx >= s
            while (lo < hi) { uint64_t m = (lo + hi) / 2; if ((int64_t)a.drec[m].x < s) lo = m + 1; else hi = m; }
            s_lo = lo;
            hi = a.nd;                            // first record with idx >= s + 2048
            while (lo < hi) { uint64_t m = (lo + hi) / 2; if ((int64_t)a.drec[m].x < s + kTileCodes) lo = m + 1; else hi = m; }
            s_hi = lo;
        } else if (tid == 0) {
            s_lo = s_hi = 0;
        }
        __syncthreads();
        if (tid == 0) s_tile[(it + 1) & 1] = atomicAdd(&ctrl->ticket, 1u);
        uint32_t tnnz = 0, wpre = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            const uint32_t pc = __popc(s_F[w]);
            tnnz += pc;
            if (w < warp) wpre += pc;
        }
        if (warp == 0) {
            unsigned long long ex = lookback_count(a.st_nnz, t, tnnz);
            if (lane == 0) {
                s_off = ex;
                if (t == a.tiles - 1) ctrl->nnz = ex + tnnz;
            }
        }
        __syncthreads();

        // ---- D2: gather block b = tid into the shuffled tile O ----
        {
            uint4 blk = make_uint4(0, 0, 0, 0);
            if (nz) {
                const uint64_t bi = s_off + wpre + __popc(F & ((1u << lane) - 1u));
                if (bi < a.nnz_total) blk = reinterpret_cast<const uint4*>(a.payload)[bi];
                else atomicExch(&ctrl->err, (int)FZ_ERR_CORRUPT);
            }
            const int r = tid >> 3, xb = tid & 7;
            uint32_t* row = Obuf + r * 33 + 4 * xb;
            row[0] = blk.x; row[1] = blk.y; row[2] = blk.z; row[3] = blk.w;
        }
        __syncthreads();

        // ---- D3: un-shuffle: column c of O -> row c of A (same 32x32 bit transpose) ----
        uint32_t w4[4];
        {
            const int c = tid >> 3, kk = tid & 7;
#pragma unroll
            for (int i = 0; i < 4; ++i) w4[i] = Obuf[(4 * kk + i) * 33 + c];
            transpose32_group8(w4, lane & 7);
        }
        // ---- D4: unpack (0x8000 -> 0, R8) ----
        int32_t dl[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t lo16 = w4[i] & 0xFFFFu, hi16 = w4[i] >> 16;
            dl[2 * i] = (lo16 & 0x8000u) ? -(int32_t)(lo16 & 0x7FFFu) : (int32_t)lo16;
            dl[2 * i + 1] = (hi16 & 0x8000u) ? -(int32_t)(hi16 & 0x7FFFu) : (int32_t)hi16;
        }
        if (s_hi > s_lo) {   // delta outliers of this tile (rare; uniform branch)
#pragma unroll
            for (int u = 0; u < 8; ++u) D[8 * tid + u] = dl[u];
            __syncthreads();
            for (uint64_t k = s_lo + tid; k < s_hi; k += kCta) {
                const uint2 r = a.drec[k];
                D[r.x - (uint32_t)s] = (int32_t)r.y;
            }
            __syncthreads();
#pragma unroll
            for (int u = 0; u < 8; ++u) dl[u] = D[8 * tid + u];
        }

        // ---- D5 (x): segmented inclusive scan, resets at row starts x == 0 ----
        uint32_t loc[8];
        uint32_t rmask = 0;     // bit u: a row start at or before u inside this thread
        Seg me{0, 0};
        {
            uint32_t x = (uint32_t)(g0 % nx);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (x == 0) { me.f = 1; me.v = 0; }
                me.v += (uint32_t)dl[u];
                loc[u] = me.v;
                if (me.f) rmask |= 1u << u;
                if (++x == nx) x = 0;
            }
        }
        // warp inclusive segmented scan
        Seg inc = me;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            Seg up{__shfl_up_sync(kFull, inc.f, o), __shfl_up_sync(kFull, inc.v, o)};
            if (lane >= o) inc = seg_combine(up, inc);
        }
        Seg lex{__shfl_up_sync(kFull, inc.f, 1), __shfl_up_sync(kFull, inc.v, 1)};
        if (lane == 0) lex = Seg{0, 0};
        if (lane == 31) { s_wf[warp] = inc.f; s_wv[warp] = inc.v; }
        __syncthreads();
        Seg wp{0, 0}, tagg{0, 0};
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            const Seg sw{s_wf[w], s_wv[w]};
            if (w < warp) wp = seg_combine(wp, sw);
            tagg = seg_combine(tagg, sw);
        }
        if (warp == 0) {
            const uint32_t carry = lookback_seg(a.st_x, t, tagg);
            if (lane == 0) s_carry = carry;
        }
        __syncthreads();
        Seg acc{0, s_carry};
        acc = seg_combine(acc, wp);
        acc = seg_combine(acc, lex);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t g = g0 + u;
            if (g < (int64_t)n) {
                const uint32_t qv = ((rmask >> u) & 1u) ? loc[u] : acc.v + loc[u];
                if (NDIM == 1 && a.x_out != nullptr) a.x_out[g] = __fmul_rn(__int2float_rn((int32_t)qv), a.w);
                else a.q_out[g] = (int32_t)qv;
            }
        }
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
    count_launch();
    k_decode_init<<<grid_for(ntiles), 256, 0, st>>>(ctrl, st_nnz, st_x, ntiles);
    return cudaGetLastError();
}

cudaError_t launch_validate_outliers(const uint2* rec, uint64_t cnt, uint64_t n, Ctrl* ctrl,
                                     cudaStream_t st)
{
    if (cnt == 0) return cudaSuccess;
    count_launch();
    k_validate_outliers<<<grid_for(cnt), 256, 0, st>>>(rec, cnt, n, ctrl);
    return cudaGetLastError();
}

template <int NDIM>
static cudaError_t launch_decode_t(const DecodeArgs& a, cudaStream_t st)
{
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
    count_launch();
    switch (a.g.ndim) {
        case 1: return launch_decode_t<1>(a, st);
        case 2: return launch_decode_t<2>(a, st);
        default: return launch_decode_t<3>(a, st);
    }
}

cudaError_t launch_scan_axis(int32_t* data, uint64_t outer, uint64_t L, uint64_t W, uint32_t* sums,
                             float dequant_w, cudaStream_t st)
{
    const uint64_t nch = (L + kScanChunk - 1) / kScanChunk;
    const uint64_t work = outer * nch * W;
    count_launch();
    k_scan_sums<<<grid_for(work), 256, 0, st>>>(data, outer, L, W, nch, sums);
    count_launch();
    k_scan_chunks<<<grid_for(outer * W), 256, 0, st>>>(outer, W, nch, sums);
    count_launch();
    k_scan_apply<<<grid_for(work), 256, 0, st>>>(data, outer, L, W, nch, sums, dequant_w);
    return cudaGetLastError();
}

cudaError_t launch_value_patch(float* out, const uint2* vrec, uint64_t cnt, uint64_t n, cudaStream_t st)
{
    if (cnt == 0) return cudaSuccess;
    count_launch();
    k_value_patch<<<grid_for(cnt), 256, 0, st>>>(out, vrec, cnt, n);
    return cudaGetLastError();
}

}  // namespace fz
