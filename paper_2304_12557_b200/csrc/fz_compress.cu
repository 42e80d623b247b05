// fz_compress.cu -- compression kernels of libfz (B200, sm_100a).
//
//   k_init          reset the control block / tile status words (and optionally set params)
//   k_range         C0: min, max, first non-finite index
//   k_params        C0: Appendix-A parameters on the device (no host round trip)
//   k_compress      C1-C8 fused: prequantize -> Lorenzo -> codes -> bitshuffle -> block flags
//                   -> decoupled look-back scan -> compaction; persistent CTAs, tile ticket
//   k_finalize      C9: header
//   k_outlier_scan / k_outlier_place: outlier sections (only launched when outliers exist)
//
// Citation key: P:n = PAPER.md line n; R# = DESIGN.md §3 readings; SV = SURVEY.md.
#include <cfloat>
#include <cstdlib>

#include "fz_internal.cuh"
#include "fz_launch.h"

namespace fz {

// Shared q arrays: element m stored at m + (m >> 3) so that the stride-8 per-thread access
// pattern of the Lorenzo stage is (at most 2-way) bank-conflict free.
__device__ __forceinline__ int pad(int m) { return m + (m >> 3); }
inline uint32_t pad_words(uint32_t len) { return len + (len >> 3) + 8; }
constexpr uint32_t kUnionHaloMax = 4097;   // union arrays when the row halo nx+1 fits

// ------------------------------------------------------------------------------------
__global__ void k_init(Ctrl* ctrl, unsigned long long* status, uint2* ocnt, uint32_t ntiles,
                       int set_params, fz_params p, uint32_t chunk)
{
    pdl_begin();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    for (uint32_t k = i; k < ntiles; k += gridDim.x * blockDim.x) {
        status[k] = 0ull;   // per-unit look-back words (at most one per tile)
        ocnt[k] = make_uint2(0, 0);
    }
    if (i == 0) {
        // every byte of the control block defined (the host reads it back whole)
        for (uint32_t w = 0; w < sizeof(Ctrl) / 4; ++w) reinterpret_cast<uint32_t*>(ctrl)[w] = 0u;
        ctrl->mn_enc = 0xFFFFFFFFu;
        ctrl->mx_enc = 0u;
        ctrl->first_bad = ~0ull;
        ctrl->log_bad = ~0ull;
        ctrl->err = 0;
        ctrl->ticket = 0;
        ctrl->stage_overflow = 0;
        ctrl->nnz = ctrl->nd = ctrl->nv = ctrl->total = 0;
        ctrl->dcount = ctrl->vcount = 0;
        ctrl->done = 0;
        ctrl->chunk = chunk;
        if (set_params) {
            ctrl->p = p;
            set_quant_consts(ctrl);
        }
    }
}

// ------------------------------------------------------------------------------------
// C0 range: grid-stride, four 16-byte loads in flight per thread, float min/max with one
// finiteness test per element (the index of the first non-finite value is recovered on a
// rare path), -0.0 canonicalized to +0.0 once per warp (R18), one atomic per warp.
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_range(const float* __restrict__ d, uint64_t n, Ctrl* ctrl)
{
    pdl_begin();
    constexpr int U = 4;
    float lo = INFINITY, hi = -INFINITY;
    unsigned long long bad = ~0ull;
    const uint64_t nv4 = n / 4;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    auto first_bad = [&](uint64_t i0, int cnt) {
        for (int u = 0; u < cnt; ++u)
            if (!(fabsf(__ldg(d + i0 + u)) <= FLT_MAX)) { bad = min(bad, (unsigned long long)(i0 + u)); return; }
    };
    uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; k + (U - 1) * stride < nv4; k += U * stride) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ldg_f4(d + 4 * (k + u * stride));
        bool ok = true;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            lo = fminf(lo, fminf(fminf(v[u].x, v[u].y), fminf(v[u].z, v[u].w)));
            hi = fmaxf(hi, fmaxf(fmaxf(v[u].x, v[u].y), fmaxf(v[u].z, v[u].w)));
            ok &= fabsf(v[u].x) <= FLT_MAX && fabsf(v[u].y) <= FLT_MAX && fabsf(v[u].z) <= FLT_MAX &&
                  fabsf(v[u].w) <= FLT_MAX;
        }
        if (!ok)
            for (int u = 0; u < U; ++u) first_bad(4 * (k + u * stride), 4);
    }
    for (; k < nv4; k += stride) {
        const float4 v = ldg_f4(d + 4 * k);
        lo = fminf(lo, fminf(fminf(v.x, v.y), fminf(v.z, v.w)));
        hi = fmaxf(hi, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
        if (!(fabsf(v.x) <= FLT_MAX && fabsf(v.y) <= FLT_MAX && fabsf(v.z) <= FLT_MAX && fabsf(v.w) <= FLT_MAX))
            first_bad(4 * k, 4);
    }
    for (uint64_t j = 4 * nv4 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
        const float v = __ldg(d + j);
        lo = fminf(lo, v);
        hi = fmaxf(hi, v);
        if (!(fabsf(v) <= FLT_MAX)) bad = min(bad, (unsigned long long)j);
    }
    // fminf/fmaxf skip NaN; non-finite inputs are reported through first_bad anyway
    uint32_t elo = f2ord(__fadd_rn(lo, 0.0f)), ehi = f2ord(__fadd_rn(hi, 0.0f));
    if (lo == INFINITY) elo = 0xFFFFFFFFu;   // no element seen by this thread
    if (hi == -INFINITY) ehi = 0u;
    elo = __reduce_min_sync(kFull, elo);
    ehi = __reduce_max_sync(kFull, ehi);
    unsigned long long b = bad;
    for (int o = 16; o; o >>= 1) b = min(b, __shfl_xor_sync(kFull, b, o));
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&ctrl->mn_enc, elo);
        atomicMax(&ctrl->mx_enc, ehi);
        if (b != ~0ull) atomicMin(&ctrl->first_bad, b);
    }
}

__global__ void k_params(Ctrl* ctrl, int mode, double eb, uint64_t n)
{
    pdl_begin();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    fz_params p;
    if (ctrl->err != 0) return;   // an earlier device step failed (e.g. the f3 log transform)
    const int st = params_from_range(ctrl, mode, eb, n, &p);
    if (st != FZ_OK) { ctrl->err = st; return; }
    ctrl->p = p;
    set_quant_consts(ctrl);
}

// ------------------------------------------------------------------------------------
// Field loads: element g (may be negative or past N: 0 outside the field).
// ------------------------------------------------------------------------------------
__device__ __forceinline__ float load1(const CompressArgs& a, int64_t g)
{
    return (g >= (int64_t)a.base && g < (int64_t)a.g.n) ? __ldg(a.field + (g - (int64_t)a.base)) : 0.0f;
}

template <int K>
__device__ __forceinline__ void loadk(const CompressArgs& a, int64_t g0, float (&v)[K])
{
    const int64_t base = (int64_t)a.base;
    if (g0 >= base && g0 + K <= (int64_t)a.g.n) {   // g0 - base is a multiple of 4 here
        const float* p = a.field + (g0 - base);
#pragma unroll
        for (int c = 0; c < K / 4; ++c) {
            float4 x = ldg_f4(p + 4 * c);
            v[4 * c] = x.x; v[4 * c + 1] = x.y; v[4 * c + 2] = x.z; v[4 * c + 3] = x.w;
        }
    } else {
#pragma unroll
        for (int u = 0; u < K; ++u) v[u] = load1(a, g0 + u);
    }
}

// cp.async.bulk.prefetch.L2 of the field elements [g, g + cnt) (16-byte aligned, clamped).
__device__ __forceinline__ void prefetch_l2_range(const CompressArgs& a, uint64_t g, uint64_t cnt)
{
    if (g < a.base) return;
    uint64_t e = g + cnt;
    if (e > a.g.n) e = a.g.n;
    uint64_t lo = (g - a.base) & ~uint64_t(3), hi = (e - a.base) & ~uint64_t(3);
    while (lo < hi) {
        const uint64_t chunk = (hi - lo) > 16384 ? 16384 : (hi - lo);   // elements
        const float* p = a.field + lo;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"((uint32_t)(chunk * 4)) : "memory");
        lo += chunk;
    }
}

// ------------------------------------------------------------------------------------
// The fused compression kernels.  One CTA of 256 threads; thread t owns the elements
// 8t..8t+7 of the current tile (= words 4t..4t+3 = A[t/8][4(t%8)..+3]).
// Scan granularity: a "unit" of kUnitTiles consecutive tiles.  The CTA compacts each tile's
// nonzero blocks into a shared stage (double-buffered per unit), publishes the unit's block
// count once its last tile is done, and resolves the unit's global offset by a wide
// decoupled look-back one tile later (while computing the next unit's first tile), then
// copies the stage to the payload with coalesced 16-byte stores.
//
// Two front ends produce the Lorenzo residuals of a tile:
//   front_vec  (nx % 4 == 0, row halo <= 6140): quantized values live in power-of-two rings
//              in shared memory; per tile the CTA quantizes its 2048 own elements and the
//              2048 new elements of the previous plane (= the z neighbours, kept in
//              registers); the row and plane halos come from the unit's earlier tiles
//              (filled at a unit's first tile).  128-bit LDS/STS, x-1 neighbour by SHFL.
//   front_gen  (any shape): both halo ranges are re-quantized for every tile into padded
//              linear arrays (element m at m + m/8).
// Both feed the same tail (codes, bitshuffle, flags, outliers, staging, look-back).
// ------------------------------------------------------------------------------------
constexpr int kUnitTiles = 4;
constexpr int kFillBatch = 4;     // halo chunks (4 elements each) per thread per batch
constexpr int kStageBlocks = kUnitTiles * kTileBlocks;

// Fast-path prequantization (C1, R2/R3): magic-rounded q0 = rint(fl(d*r)) and the exact
// residual e = d - q0*w.  When |e| < hU (= w/2 - U, rounded down) q0 is the exact nearest
// bin (no tie) and |fl32(q0*w) - d| <= |e| + U/2 < w/2 <= eb: no correction and no bound
// check are needed.  Otherwise (rare; always in fallback mode, hU = -1) `hard` is set and
// the caller applies the exact rule + bound check.
__device__ __forceinline__ int pq_fast(float d, const QuantP& P, bool& hard)
{
    const float kMagic = 12582912.0f;
    const float t = __fadd_rn(__fmul_rn(d, P.r), kMagic);
    const float qf = __fsub_rn(t, kMagic);
    const float e = __fmaf_rn(-qf, P.w, d);
    hard = !(fabsf(e) < P.hU);
    return __float_as_int(t) - 0x4B400000;
}

// Quantizes K values (q only, halo elements) with the fast path and a warp-uniform slow path.
template <int K>
__device__ __forceinline__ void pq_many(const float (&v)[K], int (&q)[K], const QuantP& P)
{
    bool any = false;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        bool h;
        q[i] = pq_fast(v[i], P, h);
        any |= h;
    }
    if (__any_sync(kFull, any) && any) {
#pragma unroll
        for (int i = 0; i < K; ++i) {
            bool h;
            pq_fast(v[i], P, h);
            if (h) q[i] = prequant_q(v[i], P);
        }
    }
}

// Own elements: q plus the exact rule + bound check where the fast path does not apply.
__device__ __forceinline__ void pq_own(const float (&v)[8], int (&q)[8], uint32_t& vmask, const QuantP& P)
{
    bool any = false;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        bool h;
        q[i] = pq_fast(v[i], P, h);
        any |= h;
    }
    vmask = 0;
    if (__any_sync(kFull, any) && any) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            bool h;
            pq_fast(v[i], P, h);
            if (h) {
                bool vo;
                q[i] = prequant(v[i], P, vo);
                if (vo) vmask |= 1u << i;
            }
        }
    }
}

// Block-uniform shared state of the compression kernels.
struct CompShared {
    uint32_t lbok;          // pending unit's offset resolved this tile
    uint32_t unit[2];
    uint32_t F[8];
    uint32_t cd[8], cv[8];
    unsigned long long off;
    unsigned long long ob[2];
};

// Per-thread copy of the (block-uniform) unit bookkeeping.
struct UnitState {
    uint32_t pu;       // pending unit: aggregate published, offset unknown
    uint32_t pcnt;     // its block count
    uint32_t cnt;      // blocks staged for the current unit
    int buf;           // stage buffer of the current unit
    uint32_t nunits;
    int it;
};

constexpr uint32_t kNone = 0xFFFFFFFFu;

__device__ __forceinline__ void flush_unit(const CompressArgs& a, CompShared& sh, const uint4* ps,
                                           const UnitState& us, unsigned long long off)
{
    for (uint32_t i = threadIdx.x; i < us.pcnt; i += kCta) {
        const uint64_t bo = 16 * (off + i);
        if (bo + 16 <= a.payload_cap) *reinterpret_cast<uint4*>(a.payload_out + bo) = ps[i];
    }
    if (threadIdx.x == 0 && us.pu == us.nunits - 1) a.ctrl->nnz = off + us.pcnt;
}

constexpr int kLbLane = 16;   // look-back window: 32 x 16 = 512 units per round

__device__ __forceinline__ void lookback_unit(const CompressArgs& a, CompShared& sh, const UnitState& us,
                                              const unsigned long long* pre = nullptr)
{
    const int lane = threadIdx.x & 31;
    unsigned long long ex = 0;
    if (us.pu != 0) {
        ex = lookback_wide<kLbLane, false>(a.status, us.pu, 0, kStAgg - 1, &a.ctrl->err, pre);
        if (lane == 0) st_relaxed_u64(&a.status[us.pu], kStInc | (ex + us.pcnt));
    }
    if (lane == 0) sh.off = ex;
}

// ------------------------------------------------------------------------------------
// Tail of a tile: C3 codes, C5 bitshuffle, outlier records, C6 flags, C8 local compaction
// into the unit stage; at the first tile of a unit, the pending unit's look-back (C7) and
// its global compaction.  dl = Lorenzo residuals (already masked), vmask = value outliers.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ void tile_tail(const CompressArgs& a, CompShared& sh, uint32_t* Obuf, uint4* stage,
                                          UnitState& us, uint32_t t, bool first, bool lbt, uint32_t g0, uint32_t vm,
                                          const int32_t (&dl)[8], uint32_t vmask, const float (&dv)[8],
                                          const unsigned long long* pre)
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    Ctrl* ctrl = a.ctrl;
    const uint32_t n = a.g.n;
    // ---- C3 codes: sign-magnitude, |delta| > 32767 -> code 0 + delta outlier (R7) ----
    uint32_t code[8];
    uint32_t dmask = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const uint32_t dd = (uint32_t)dl[e];
        const uint32_t mag = (uint32_t)abs(dl[e]);
        const bool outl = mag > 32767u;
        code[e] = outl ? 0u : (((dd >> 16) & 0x8000u) | mag);
        if (outl) dmask |= 1u << e;
    }
    if (vm != 0xFFu) {
        dmask &= vm;
        vmask &= vm;
#pragma unroll
        for (int e = 0; e < 8; ++e)
            if (!((vm >> e) & 1u)) code[e] = 0u;
    }
    if (a.codes_out != nullptr) {
#pragma unroll
        for (int e = 0; e < 8; ++e)
            if (g0 + e < n) a.codes_out[g0 + e] = (uint16_t)code[e];
    }
    if (!a.rescan) {
        // ---- C4 words, C5 bitshuffle in registers: row c = tid/8 of A ----
        uint32_t w4[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) w4[i] = __byte_perm(code[2 * i], code[2 * i + 1], 0x5410);
        transpose32_group8(w4, lane & 7);
        const int c = tid >> 3, kk = tid & 7;
#pragma unroll
        for (int i = 0; i < 4; ++i) Obuf[(4 * kk + i) * 33 + c] = w4[i];
    }
    const int any_out = __syncthreads_or((dmask | vmask) != 0);
    if (first && tid == 0) {
        const uint32_t nu = atomicAdd(&ctrl->ticket, 1u);
        sh.unit[(us.it & 1) ^ 1] = nu;
        // TMA L2 prefetch of the next unit's input (~kUnitTiles tiles ahead)
        if (nu < us.nunits)
            prefetch_l2_range(a, (uint64_t)(a.tile_begin + nu * kUnitTiles) * kTileCodes,
                              (uint64_t)kUnitTiles * kTileCodes);
    }

    // ---- outlier records (rare; R7, R20): ascending element index ----
    if (any_out) {
        const int cd = __popc(dmask), cv = __popc(vmask);
        const int wd = __reduce_add_sync(kFull, cd), wv = __reduce_add_sync(kFull, cv);
        if (lane == 0) { sh.cd[warp] = wd; sh.cv[warp] = wv; }
        __syncthreads();
        uint32_t tnd = 0, tnv = 0, wpre_d = 0, wpre_v = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            tnd += sh.cd[w]; tnv += sh.cv[w];
            if (w < warp) { wpre_d += sh.cd[w]; wpre_v += sh.cv[w]; }
        }
        if (tid == 0) {
            if (a.rescan) {
                const uint2 o = a.opre[t];
                sh.ob[0] = o.x; sh.ob[1] = o.y;
            } else {
                sh.ob[0] = tnd ? atomicAdd(&ctrl->dcount, (unsigned long long)tnd) : 0ull;
                sh.ob[1] = tnv ? atomicAdd(&ctrl->vcount, (unsigned long long)tnv) : 0ull;
                a.ocnt[t] = make_uint2(tnd, tnv);
                a.obase[t] = make_uint2((uint32_t)sh.ob[0], (uint32_t)sh.ob[1]);
            }
        }
        int id = cd, iv = cv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int yd = __shfl_up_sync(kFull, id, o), yv = __shfl_up_sync(kFull, iv, o);
            if (lane >= o) { id += yd; iv += yv; }
        }
        __syncthreads();
        uint64_t pd = sh.ob[0] + wpre_d + (id - cd), pv = sh.ob[1] + wpre_v + (iv - cv);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const uint32_t gi = g0 + e;
            if (dmask & (1u << e)) {
                if (pd < a.dcap) {
                    if (a.o_didx) { a.o_didx[pd] = gi; a.o_dval[pd] = dl[e]; }
                    else a.dstage[pd] = make_uint2(gi, (uint32_t)dl[e]);
                } else {
                    atomicOr(&ctrl->stage_overflow, 1u);
                }
                ++pd;
            }
            if (vmask & (1u << e)) {
                if (pv < a.vcap) {
                    if (a.o_vidx) { a.o_vidx[pv] = gi; a.o_vbits[pv] = __float_as_uint(dv[e]); }
                    else a.vstage[pv] = make_uint2(gi, __float_as_uint(dv[e]));
                } else {
                    atomicOr(&ctrl->stage_overflow, 1u);
                }
                ++pv;
            }
        }
        __syncthreads();
    }
    if (a.rescan) return;

    // ---- C6 block flags: thread b owns block b = 8r + x of the shuffled tile ----
    const uint32_t* row = Obuf + (tid >> 3) * 33 + 4 * (tid & 7);
    const uint4 blk = make_uint4(row[0], row[1], row[2], row[3]);
    const bool nz = (blk.x | blk.y | blk.z | blk.w) != 0;
    const uint32_t F = __ballot_sync(kFull, nz);
    if (lane == 0) sh.F[warp] = F;
    // the pending unit's look-back (window prefetched at the top of the tile) overlaps the
    // other warps' flag work; it only blocks at the unit's last tile (lbt)
    if (us.pu != kNone && warp == 0) {
        unsigned long long ex = 0;
        bool ok = true;
        if (us.pu != 0) {
            if (pre != nullptr)
                ok = lookback_try<kLbLane>(a.status, us.pu, 0, kStAgg - 1, &ctrl->err,
                                           *reinterpret_cast<const unsigned long long (*)[kLbLane]>(pre), ex);
            else ok = false;
            if (!ok && lbt) {
                ex = lookback_wide<kLbLane, false>(a.status, us.pu, 0, kStAgg - 1, &ctrl->err);
                ok = true;
            }
            if (ok && lane == 0) st_relaxed_u64(&a.status[us.pu], kStInc | (ex + us.pcnt));
        }
        if (lane == 0) {
            sh.off = ex;
            sh.lbok = ok;
        }
    }
    __syncthreads();
    uint32_t tn = 0, wpre = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        const uint32_t pc = __popc(sh.F[w]);
        tn += pc;
        if (w < warp) wpre += pc;
    }
    if (tid < 8) {
        const uint64_t fo = (uint64_t)(t - a.tile_begin) * 32 + 4 * tid;
        if (fo + 4 <= a.flags_cap) *reinterpret_cast<uint32_t*>(a.flags_out + fo) = sh.F[tid];
    }
    // ---- C8 (local): compact the tile's nonzero blocks into the unit stage ----
    if (nz) stage[us.buf * kStageBlocks + us.cnt + wpre + __popc(F & ((1u << lane) - 1u))] = blk;
    us.cnt += tn;
    if (us.pu != kNone && sh.lbok) {
        // ---- C8 (global): the pending unit's stage goes to its final offset ----
        flush_unit(a, sh, stage + (us.buf ^ 1) * kStageBlocks, us, sh.off);
        us.pu = kNone;
    }
}

// ------------------------------------------------------------------------------------
// Lorenzo masks of a thread's 8 elements: bit e of xmask/ymask/zmask = the x-1 / y-1 / z-1
// neighbour of element g0+e exists (zero boundary outside the field, R5).  `fast` = all set.
// ------------------------------------------------------------------------------------
template <int NDIM>
__device__ __forceinline__ void lorenzo_masks(const CompressArgs& a, uint32_t g0, uint32_t& xm, uint32_t& ym,
                                              uint32_t& zm, bool& fast_yz)
{
    const uint32_t nx = a.g.nx, PL = a.g.P;
    xm = 0xFFu; ym = 0xFFu; zm = 0xFFu;
    fast_yz = true;
    if (nx >= 8) {
        const uint32_t x0 = fmod_(g0, a.dnx);
        const uint32_t us = x0 == 0 ? 0u : nx - x0;
        if (us < 8) xm &= ~(1u << us);
        if (NDIM >= 2) {
            const uint32_t p0 = fmod_(g0, a.dP);
            fast_yz = p0 >= nx && p0 + 7 < PL && (NDIM == 2 || g0 >= PL);
            if (!fast_yz) {
                uint32_t pp = p0;
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    if (pp < nx) ym &= ~(1u << e);
                    if (g0 + e < PL) zm &= ~(1u << e);
                    if (++pp == PL) pp = 0;
                }
            }
        }
    } else {
        fast_yz = false;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            if (fmod_(g0 + e, a.dnx) == 0) xm &= ~(1u << e);
            if (fmod_(g0 + e, a.dP) < nx) ym &= ~(1u << e);
            if (g0 + e < PL) zm &= ~(1u << e);
        }
    }
    if (NDIM == 1) { ym = 0; zm = 0; }
    if (NDIM == 2) zm = 0;
}

// Same masks from the thread's precomputed in-row (x0) and in-plane (p0) positions.
template <int NDIM>
__device__ __forceinline__ void lorenzo_masks_xp(const CompressArgs& a, uint32_t g0, uint32_t x0, uint32_t p0,
                                                 uint32_t& xm, uint32_t& ym, uint32_t& zm, bool& fast_yz)
{
    const uint32_t nx = a.g.nx, PL = a.g.P;
    if (nx < 8) {
        lorenzo_masks<NDIM>(a, g0, xm, ym, zm, fast_yz);
        return;
    }
    xm = 0xFFu; ym = 0xFFu; zm = 0xFFu;
    fast_yz = true;
    const uint32_t us = x0 == 0 ? 0u : nx - x0;
    if (us < 8) xm &= ~(1u << us);
    if (NDIM >= 2) {
        fast_yz = p0 >= nx && p0 + 7 < PL && (NDIM == 2 || g0 >= PL);
        if (!fast_yz) {
            uint32_t pp = p0;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                if (pp < nx) ym &= ~(1u << e);
                if (g0 + e < PL) zm &= ~(1u << e);
                if (++pp == PL) pp = 0;
            }
        }
    }
    if (NDIM == 1) { ym = 0; zm = 0; }
    if (NDIM == 2) zm = 0;
}

// delta(e) = S(e+1) - [x>0] S(e), with S(j) the y/z combination at element g0-1+j (C2).
__device__ __forceinline__ void residuals(const uint32_t (&S)[9], uint32_t xm, int32_t (&dl)[8])
{
#pragma unroll
    for (int e = 0; e < 8; ++e) dl[e] = (int32_t)(S[e + 1] - S[e]);
    if (xm != 0xFFu) {   // a row start among the 8 elements: its x-1 neighbour is outside
#pragma unroll
        for (int e = 0; e < 8; ++e)
            if (!((xm >> e) & 1u)) dl[e] = (int32_t)S[e + 1];
    }
}

// ------------------------------------------------------------------------------------
// front_gen: generic shapes (padded linear arrays, halos re-quantized per tile).
// ------------------------------------------------------------------------------------
// Cooperative prequantization of two ranges into shared arrays (word offsets o0, o1 in
// smem): element m of range r at o_r + m + (m >> 3).  4-element aligned chunks.
__device__ __forceinline__ void fill_halo(const CompressArgs& a, const QuantP& P, int* smem, int o0, int64_t g0lo,
                                          int len0, int o1, int64_t g1lo, int len1)
{
    const int64_t a0 = g0lo & ~(int64_t)3, a1 = g1lo & ~(int64_t)3;
    const int n0 = len0 > 0 ? (int)((g0lo + len0 - a0 + 3) >> 2) : 0;
    const int n1 = len1 > 0 ? (int)((g1lo + len1 - a1 + 3) >> 2) : 0;
    const int total = n0 + n1;
    for (int c0 = 0; c0 < total; c0 += kCta * kFillBatch) {
        float v[4 * kFillBatch];
        int64_t gc[kFillBatch];
#pragma unroll
        for (int i = 0; i < kFillBatch; ++i) {
            const int c = c0 + threadIdx.x + i * kCta;
            gc[i] = c < n0 ? a0 + 4 * (int64_t)c : a1 + 4 * (int64_t)(c - n0);
            float x[4];
            if (c < total) {
                loadk<4>(a, gc[i], x);
            } else {
                x[0] = x[1] = x[2] = x[3] = 0.0f;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) v[4 * i + u] = x[u];
        }
        int q[4 * kFillBatch];
        pq_many<4 * kFillBatch>(v, q, P);
#pragma unroll
        for (int i = 0; i < kFillBatch; ++i) {
            const int c = c0 + threadIdx.x + i * kCta;
            if (c >= total) continue;
            const bool r0 = c < n0;
            const int ob = r0 ? o0 : o1;
            const int m0 = (int)(gc[i] - (r0 ? g0lo : g1lo));
            const int len = r0 ? len0 : len1;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int m = m0 + u;
                if (m >= 0 && m < len) smem[ob + m + (m >> 3)] = q[4 * i + u];
            }
        }
    }
}

template <int NDIM>
__device__ __forceinline__ void front_gen(const CompressArgs& a, const QuantP& P, int* smem, uint32_t t,
                                          int32_t (&dl)[8], uint32_t& vmask, float (&dv)[8], uint32_t& vm)
{
    const int tid = threadIdx.x;
    const uint32_t n = a.g.n, nx = a.g.nx, PL = a.g.P;
    const int qs = (int)a.qstride;
    int ab[4], mo[4];
    if (NDIM == 1) {
        ab[0] = ab[1] = ab[2] = ab[3] = 0; mo[0] = mo[1] = mo[2] = mo[3] = 1;
    } else if (a.union_mode) {
        const int HA = (int)nx + 1;
        ab[0] = 0; mo[0] = HA; ab[1] = 0; mo[1] = 1;
        ab[2] = qs; mo[2] = HA; ab[3] = qs; mo[3] = 1;
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) { ab[k] = k * qs; mo[k] = 1; }
    }
    const int tb9 = 9 * tid;       // (8 tid) + ((8 tid) >> 3)
    const int64_t s = (int64_t)t * kTileCodes;
    const uint32_t g0 = (uint32_t)s + 8u * tid;
    loadk<8>(a, (int64_t)g0, dv);
    if (NDIM == 1) {
        fill_halo(a, P, smem, 0, s - 1, 1, 0, 0, 0);
    } else if (a.union_mode) {
        fill_halo(a, P, smem, 0, s - (int64_t)nx - 1, (int)nx + 1, qs, s - (int64_t)PL - nx - 1,
                  NDIM == 3 ? kTileCodes + (int)nx + 1 : 0);
    } else {
        fill_halo(a, P, smem, 0, s - 1, 1, ab[1], s - (int64_t)nx - 1, kTileCodes + 1);
        if (NDIM == 3)
            fill_halo(a, P, smem, ab[2], s - (int64_t)PL - 1, kTileCodes + 1, ab[3], s - (int64_t)PL - nx - 1,
                      kTileCodes + 1);
    }
    int qo[8];
    pq_own(dv, qo, vmask, P);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const int m = mo[0] + e;
        smem[ab[0] + tb9 + m + (m >> 3)] = qo[e];
    }
    vm = 0xFFu;
    if (s + kTileCodes > (int64_t)n) vm = (g0 >= n) ? 0u : ((n - g0 >= 8) ? 0xFFu : ((1u << (n - g0)) - 1u));
    __syncthreads();

    uint32_t xm, ym, zm;
    bool fast_yz;
    lorenzo_masks<NDIM>(a, g0, xm, ym, zm, fast_yz);
    uint32_t S[9];
#pragma unroll
    for (int j = 0; j < 9; ++j) {
        uint32_t ow;
        if (j == 0) {
            const int m = mo[0] - 1;
            ow = (uint32_t)smem[ab[0] + tb9 + m + (m >> 3)];
        } else {
            ow = (uint32_t)qo[j - 1];
        }
        uint32_t v = ow;
        if (NDIM >= 2) {
            const int m1 = mo[1] - 1 + j;
            const uint32_t qy = (uint32_t)smem[ab[1] + tb9 + m1 + (m1 >> 3)];
            uint32_t qz = 0, qyz = 0;
            if (NDIM == 3) {
                const int m2 = mo[2] - 1 + j, m3 = mo[3] - 1 + j;
                qz = (uint32_t)smem[ab[2] + tb9 + m2 + (m2 >> 3)];
                qyz = (uint32_t)smem[ab[3] + tb9 + m3 + (m3 >> 3)];
            }
            if (fast_yz) {
                v = ow - qy - (qz - qyz);
            } else {
                // masks of element j-1 for S(j), of element 0 for S(0)
                const int e = j == 0 ? 0 : j - 1;
                const uint32_t Y = (ym >> e) & 1u ? 0xFFFFFFFFu : 0u;
                const uint32_t Z = (zm >> e) & 1u ? 0xFFFFFFFFu : 0u;
                v = ow - (qy & Y) - ((qz - (qyz & Y)) & Z);
            }
        }
        S[j] = v;
    }
    residuals(S, xm, dl);
}

// ------------------------------------------------------------------------------------
// front_vec: nx % 4 == 0.  Rings RA (this plane) and RB (previous plane), R = rmask + 1
// elements each, element g at index g & rmask.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ void load8_vec(const CompressArgs& a, int64_t g, bool inb, float (&v)[8])
{
    if (inb) {
        const float* p = a.field + (g - (int64_t)a.base);
        const float4 x = ldg_f4(p), y = ldg_f4(p + 4);
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
        v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
    } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = load1(a, g + u);
    }
}

// Quantize the quads [lo4, hi) (lo4 4-aligned) of ring `R` (word offset ro) cooperatively.
__device__ __forceinline__ void fill_ring(const CompressArgs& a, const QuantP& P, int* smem, int ro,
                                          uint32_t rmask, int64_t lo4, int64_t hi)
{
    const int nq = (int)((hi - lo4 + 3) >> 2);
    const int64_t base = (int64_t)a.base;
    for (int c0 = 0; c0 < nq; c0 += kCta * 2) {
        float v[8];
        int64_t g[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int c = c0 + threadIdx.x + i * kCta;
            g[i] = lo4 + 4 * (int64_t)c;
            float x[4] = {0.0f, 0.0f, 0.0f, 0.0f};
            if (c < nq) {
                if (g[i] >= base && g[i] + 4 <= (int64_t)a.g.n) {
                    const float4 f = ldg_f4(a.field + (g[i] - base));
                    x[0] = f.x; x[1] = f.y; x[2] = f.z; x[3] = f.w;
                } else {
#pragma unroll
                    for (int u = 0; u < 4; ++u) x[u] = load1(a, g[i] + u);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) v[4 * i + u] = x[u];
        }
        int q[8];
        pq_many<8>(v, q, P);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int c = c0 + threadIdx.x + i * kCta;
            if (c < nq)
                *reinterpret_cast<int4*>(smem + ro + ((uint32_t)g[i] & rmask)) =
                    make_int4(q[4 * i], q[4 * i + 1], q[4 * i + 2], q[4 * i + 3]);
        }
    }
}

template <int NDIM>
__device__ __forceinline__ void front_vec(const CompressArgs& a, const QuantP& P, int* smem, uint32_t rmask,
                                          uint32_t t, bool first, int32_t (&dl)[8], uint32_t& vmask,
                                          float (&dv)[8], uint32_t& vm)
{
    const int tid = threadIdx.x, lane = tid & 31;
    const uint32_t n = a.g.n, nx = a.g.nx, PL = a.g.P;
    const int RB = (int)rmask + 1;                  // word offset of the previous-plane ring
    const int64_t s = (int64_t)t * kTileCodes;
    const uint32_t g0 = (uint32_t)s + 8u * tid;
    const int64_t base = (int64_t)a.base;
    const int64_t H = NDIM >= 2 ? (int64_t)nx + 1 : 1;
    const bool full = s + kTileCodes <= (int64_t)n;
    const bool own_in = full && s >= base;
    const bool b_in = full && s - (int64_t)PL >= base;
    // ---- A: loads (own + previous plane), halos at a unit's first tile ----
    float bz[8];
    load8_vec(a, (int64_t)g0, own_in, dv);
    if (NDIM == 3) load8_vec(a, (int64_t)g0 - PL, b_in, bz);
    if (first) {
        fill_ring(a, P, smem, 0, rmask, (s - H) & ~(int64_t)3, s);
        if (NDIM == 3) fill_ring(a, P, smem, RB, rmask, (s - (int64_t)PL - H) & ~(int64_t)3, s - (int64_t)PL);
    }
    int qo[8], qz[8];
    pq_own(dv, qo, vmask, P);
    if (NDIM == 3) pq_many<8>(bz, qz, P);
    *reinterpret_cast<int4*>(smem + (g0 & rmask)) = make_int4(qo[0], qo[1], qo[2], qo[3]);
    *reinterpret_cast<int4*>(smem + ((g0 + 4) & rmask)) = make_int4(qo[4], qo[5], qo[6], qo[7]);
    if (NDIM == 3) {
        const uint32_t gb = g0 - PL;
        *reinterpret_cast<int4*>(smem + RB + (gb & rmask)) = make_int4(qz[0], qz[1], qz[2], qz[3]);
        *reinterpret_cast<int4*>(smem + RB + ((gb + 4) & rmask)) = make_int4(qz[4], qz[5], qz[6], qz[7]);
    }
    vm = 0xFFu;
    if (!full) vm = (g0 >= n) ? 0u : ((n - g0 >= 8) ? 0xFFu : ((1u << (n - g0)) - 1u));
    __syncthreads();

    // ---- B: Lorenzo (C2) ----
    uint32_t xm, ym, zm;
    bool fast_yz;
    lorenzo_masks<NDIM>(a, g0, xm, ym, zm, fast_yz);
    uint32_t S[9];
    if (NDIM == 1) {
#pragma unroll
        for (int j = 1; j < 9; ++j) S[j] = (uint32_t)qo[j - 1];
    } else if (fast_yz) {
        uint32_t y[8], yz[8];
        {
            const int4 p = *reinterpret_cast<const int4*>(smem + ((g0 - nx) & rmask));
            const int4 q = *reinterpret_cast<const int4*>(smem + ((g0 - nx + 4) & rmask));
            y[0] = p.x; y[1] = p.y; y[2] = p.z; y[3] = p.w; y[4] = q.x; y[5] = q.y; y[6] = q.z; y[7] = q.w;
        }
        if (NDIM == 3) {
            const uint32_t gb = g0 - PL - nx;
            const int4 p = *reinterpret_cast<const int4*>(smem + RB + (gb & rmask));
            const int4 q = *reinterpret_cast<const int4*>(smem + RB + ((gb + 4) & rmask));
            yz[0] = p.x; yz[1] = p.y; yz[2] = p.z; yz[3] = p.w; yz[4] = q.x; yz[5] = q.y; yz[6] = q.z; yz[7] = q.w;
        }
#pragma unroll
        for (int j = 1; j < 9; ++j) {
            uint32_t v = (uint32_t)qo[j - 1] - y[j - 1];
            if (NDIM == 3) v -= (uint32_t)qz[j - 1] - yz[j - 1];
            S[j] = v;
        }
    } else {
        // boundary thread: every neighbour from the rings, masked per element
#pragma unroll
        for (int j = 1; j < 9; ++j) {
            const uint32_t pos = g0 + j - 1;
            const int e = j - 1;
            const uint32_t Y = (ym >> e) & 1u ? 0xFFFFFFFFu : 0u;
            const uint32_t Z = (zm >> e) & 1u ? 0xFFFFFFFFu : 0u;
            const uint32_t qy = (uint32_t)smem[(pos - nx) & rmask];
            uint32_t v = (uint32_t)qo[e] - (qy & Y);
            if (NDIM == 3) {
                const uint32_t qzz = (uint32_t)smem[RB + ((pos - PL) & rmask)];
                const uint32_t qyz = (uint32_t)smem[RB + ((pos - PL - nx) & rmask)];
                v -= (qzz - (qyz & Y)) & Z;
            }
            S[j] = v;
        }
    }
    // S(0) at element g0-1: S(8) of the previous lane, computed directly by lane 0
    S[0] = __shfl_up_sync(kFull, S[8], 1);
    if (lane == 0 || !fast_yz) {
        const uint32_t pos = g0 - 1;
        const uint32_t Y = (ym & 1u) ? 0xFFFFFFFFu : 0u;
        const uint32_t Z = (zm & 1u) ? 0xFFFFFFFFu : 0u;
        uint32_t v = (uint32_t)smem[pos & rmask];
        if (NDIM >= 2) v -= (uint32_t)smem[(pos - nx) & rmask] & Y;
        if (NDIM == 3)
            v -= ((uint32_t)smem[RB + ((pos - PL) & rmask)] - ((uint32_t)smem[RB + ((pos - PL - nx) & rmask)] & Y)) & Z;
        S[0] = v;
    }
    residuals(S, xm, dl);
}

// ------------------------------------------------------------------------------------
template <int NDIM, bool VEC>
__device__ __forceinline__ void compress_body(const CompressArgs& a)
{
    extern __shared__ int smem[];
    __shared__ CompShared sh;
    const int tid = threadIdx.x;
    Ctrl* ctrl = a.ctrl;
    if (ctrl->err != 0) return;
    QuantP P;
    P.w = ctrl->p.w; P.r = ctrl->p.r; P.h = ctrl->h; P.eb32 = ctrl->p.eb32; P.hU = ctrl->hU;
    uint32_t* Obuf = reinterpret_cast<uint32_t*>(smem + a.qwords);          // 32 x 33
    uint4* stage = reinterpret_cast<uint4*>(smem + a.qwords + 32 * 33 + 4);  // 16-byte aligned
    const uint32_t rmask = a.qstride - 1;                                    // ring mask (VEC)

    UnitState us;
    us.nunits = (a.tile_end - a.tile_begin + kUnitTiles - 1) / kUnitTiles;
    us.pu = kNone;
    us.pcnt = 0;
    us.buf = 0;
    if (tid == 0) sh.unit[0] = atomicAdd(&ctrl->ticket, 1u);
    __syncthreads();
    for (us.it = 0;; ++us.it) {
        const uint32_t u = sh.unit[us.it & 1];
        const bool work = u < us.nunits;
        if (!work && us.pu == kNone) break;
        if (!work) {
            // ---- flush the last pending unit ----
            if ((tid >> 5) == 0) lookback_unit(a, sh, us);
            __syncthreads();
            flush_unit(a, sh, stage + (us.buf ^ 1) * kStageBlocks, us, sh.off);
            break;
        }
        const uint32_t t_first = a.tile_begin + u * kUnitTiles;
        const uint32_t t_last = min(a.tile_end, t_first + kUnitTiles);
        us.cnt = 0;
        // the pending unit is resolved at the first tile where its window is complete, at
        // the latest at the unit's last tile (before its stage buffer is reused)
        for (uint32_t t = t_first; t < t_last; ++t) {
            const bool lbt = t == t_last - 1;
            unsigned long long pre[kLbLane];
            const bool use_pre = VEC && us.pu != kNone && us.pu != 0;
            if (use_pre && (tid >> 5) == 0) lookback_load<kLbLane>(a.status, (int64_t)us.pu - 1, 0, pre);
            int32_t dl[8];
            uint32_t vmask, vm;
            float dv[8];
            if (VEC) front_vec<NDIM>(a, P, smem, rmask, t, t == t_first, dl, vmask, dv, vm);
            else front_gen<NDIM>(a, P, smem, t, dl, vmask, dv, vm);
            tile_tail(a, sh, Obuf, stage, us, t, t == t_first, lbt, (uint32_t)t * kTileCodes + 8u * tid, vm,
                      dl, vmask, dv, use_pre ? pre : nullptr);
        }
        if (!a.rescan) {
            // ---- C7: publish the unit's aggregate (inclusive for unit 0) ----
            if (tid == 0) st_relaxed_u64(&a.status[u], (u == 0 ? kStInc : kStAgg) | us.cnt);
            us.pu = u;
            us.pcnt = us.cnt;
            us.buf ^= 1;
        }
        __syncthreads();
    }
}

// One kernel per (ndim, front end); the margin/fallback choice (R2) only changes the
// fast-path threshold hU (k_params / k_init set hU = -1 in fallback mode).
template <int NDIM, bool VEC>
__global__ void __launch_bounds__(kCta, 2) k_compress(CompressArgs a)
{
    pdl_begin();
    compress_body<NDIM, VEC>(a);
}

// ------------------------------------------------------------------------------------
// Warp-specialized vector kernel (k_compress_ws): 8 compute warps + 1 scanner warp.
//   compute warps : TMA-fed front (own tile and previous-plane tile arrive by
//                   cp.async.bulk into a 2-stage shared buffer while the previous tile is
//                   processed), Lorenzo, codes, bitshuffle, flags, local compaction into a
//                   unit stage; at a unit's end they publish its aggregate and hand the
//                   stage to the scanner (named barrier READY_b).
//   scanner warp  : decoupled look-back of the unit (C7), inclusive publication, copy of
//                   the stage to the payload (C8), then releases the stage (FREE_b).
// The compute warps never wait for the look-back unless they are two units ahead.
// Named barriers: 0 = whole CTA (start only), 1/2 = READY_0/1, 3/4 = FREE_0/1,
// 5 = compute warps only.
// ------------------------------------------------------------------------------------
constexpr int kWsThreads = kCta + 32;
constexpr int kBarCompute = 5;

struct WsDesc {
    uint32_t unit, start, cnt, pad;
};

struct WsShared {
    uint64_t mbar;                 // TMA input stage
    uint32_t tma_bits;             // bit0: own tile loaded by TMA, bit1: previous-plane tile
    uint32_t unit[2];
    uint32_t F[8];
    uint32_t cd[8], cv[8];
    unsigned long long ob[2];
    volatile uint32_t ring_tail;   // payload ring blocks released by the scanner
    uint64_t desc_full[kDescQ];    // mbarrier per descriptor slot: completes when it is written
    fz_params p;                   // parameters (derived in the prologue when a.derive)
    QuantP P;
    int perr;
    volatile uint32_t desc_head;   // descriptors published by the compute warps
    volatile uint32_t desc_tail;   // descriptors consumed by the scanner
    WsDesc desc[kDescQ];
};

// Issue the TMA loads of tile t into the input stage (thread 0 of the compute group).
template <int NDIM>
__device__ __forceinline__ void ws_issue(const CompressArgs& a, WsShared& sh, float* inbuf, uint32_t t)
{
    const int64_t s = (int64_t)t * kTileCodes, base = (int64_t)a.base;
    const bool full = s + kTileCodes <= (int64_t)a.g.n;
    uint32_t bits = 0, bytes = 0;
    if (full && s >= base) { bits |= 1; bytes += kTileCodes * 4; }
    if (NDIM == 3 && full && s - (int64_t)a.g.P >= base) { bits |= 2; bytes += kTileCodes * 4; }
    sh.tma_bits = bits;
    if (bytes) {
        mbar_expect_tx(&sh.mbar, bytes);
        if (bits & 1) tma_load_1d(inbuf, a.field + (s - base), kTileCodes * 4, &sh.mbar);
        if (bits & 2) tma_load_1d(inbuf + kTileCodes, a.field + (s - (int64_t)a.g.P - base), kTileCodes * 4, &sh.mbar);
    }
}

template <int NDIM, class OnFree>
__device__ __forceinline__ void front_ws(const CompressArgs& a, const QuantP& P, int* smem, uint32_t rmask,
                                         uint32_t t, bool first, const float* in_own, const float* in_b,
                                         uint32_t x0, uint32_t p0,
                                         int32_t (&dl)[8], uint32_t& vmask, float (&dv)[8], uint32_t& vm,
                                         OnFree&& on_input_free)
{
    const int tid = threadIdx.x, lane = tid & 31;
    const uint32_t n = a.g.n, nx = a.g.nx, PL = a.g.P;
    const int RB = (int)rmask + 1;
    const int64_t s = (int64_t)t * kTileCodes;
    const uint32_t g0 = (uint32_t)s + 8u * tid;
    const int64_t H = NDIM >= 2 ? (int64_t)nx + 1 : 1;
    const bool full = s + kTileCodes <= (int64_t)n;
    float bz[8];
    if (in_own) {
        const float4 x = *reinterpret_cast<const float4*>(in_own + 8 * tid);
        const float4 y = *reinterpret_cast<const float4*>(in_own + 8 * tid + 4);
        dv[0] = x.x; dv[1] = x.y; dv[2] = x.z; dv[3] = x.w; dv[4] = y.x; dv[5] = y.y; dv[6] = y.z; dv[7] = y.w;
    } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) dv[u] = load1(a, (int64_t)g0 + u);
    }
    if (NDIM == 3) {
        if (in_b) {
            const float4 x = *reinterpret_cast<const float4*>(in_b + 8 * tid);
            const float4 y = *reinterpret_cast<const float4*>(in_b + 8 * tid + 4);
            bz[0] = x.x; bz[1] = x.y; bz[2] = x.z; bz[3] = x.w; bz[4] = y.x; bz[5] = y.y; bz[6] = y.z; bz[7] = y.w;
        } else {
#pragma unroll
            for (int u = 0; u < 8; ++u) bz[u] = load1(a, (int64_t)g0 - PL + u);
        }
    }
    if (first) {
        fill_ring(a, P, smem, 0, rmask, (s - H) & ~(int64_t)3, s);
        if (NDIM == 3) fill_ring(a, P, smem, RB, rmask, (s - (int64_t)PL - H) & ~(int64_t)3, s - (int64_t)PL);
    }
    int qo[8], qz[8];
    pq_own(dv, qo, vmask, P);
    if (NDIM == 3) pq_many<8>(bz, qz, P);
    *reinterpret_cast<int4*>(smem + (g0 & rmask)) = make_int4(qo[0], qo[1], qo[2], qo[3]);
    *reinterpret_cast<int4*>(smem + ((g0 + 4) & rmask)) = make_int4(qo[4], qo[5], qo[6], qo[7]);
    if (NDIM == 3) {
        const uint32_t gb = g0 - PL;
        *reinterpret_cast<int4*>(smem + RB + (gb & rmask)) = make_int4(qz[0], qz[1], qz[2], qz[3]);
        *reinterpret_cast<int4*>(smem + RB + ((gb + 4) & rmask)) = make_int4(qz[4], qz[5], qz[6], qz[7]);
    }
    vm = 0xFFu;
    if (!full) vm = (g0 >= n) ? 0u : ((n - g0 >= 8) ? 0xFFu : ((1u << (n - g0)) - 1u));
    bar_sync(kBarCompute, kCta);
    on_input_free();   // every compute thread has read the TMA input stage

    uint32_t xm, ym, zm;
    bool fast_yz;
    lorenzo_masks_xp<NDIM>(a, g0, x0, p0, xm, ym, zm, fast_yz);
    uint32_t S[9];
    if (NDIM == 1) {
#pragma unroll
        for (int j = 1; j < 9; ++j) S[j] = (uint32_t)qo[j - 1];
    } else if (fast_yz) {
        uint32_t y[8], yz[8];
        {
            const int4 p = *reinterpret_cast<const int4*>(smem + ((g0 - nx) & rmask));
            const int4 q = *reinterpret_cast<const int4*>(smem + ((g0 - nx + 4) & rmask));
            y[0] = p.x; y[1] = p.y; y[2] = p.z; y[3] = p.w; y[4] = q.x; y[5] = q.y; y[6] = q.z; y[7] = q.w;
        }
        if (NDIM == 3) {
            const uint32_t gb = g0 - PL - nx;
            const int4 p = *reinterpret_cast<const int4*>(smem + RB + (gb & rmask));
            const int4 q = *reinterpret_cast<const int4*>(smem + RB + ((gb + 4) & rmask));
            yz[0] = p.x; yz[1] = p.y; yz[2] = p.z; yz[3] = p.w; yz[4] = q.x; yz[5] = q.y; yz[6] = q.z; yz[7] = q.w;
        }
#pragma unroll
        for (int j = 1; j < 9; ++j) {
            uint32_t v = (uint32_t)qo[j - 1] - y[j - 1];
            if (NDIM == 3) v -= (uint32_t)qz[j - 1] - yz[j - 1];
            S[j] = v;
        }
    } else {
#pragma unroll
        for (int j = 1; j < 9; ++j) {
            const uint32_t pos = g0 + j - 1;
            const int e = j - 1;
            const uint32_t Y = (ym >> e) & 1u ? 0xFFFFFFFFu : 0u;
            const uint32_t Z = (zm >> e) & 1u ? 0xFFFFFFFFu : 0u;
            const uint32_t qy = (uint32_t)smem[(pos - nx) & rmask];
            uint32_t v = (uint32_t)qo[e] - (qy & Y);
            if (NDIM == 3) {
                const uint32_t qzz = (uint32_t)smem[RB + ((pos - PL) & rmask)];
                const uint32_t qyz = (uint32_t)smem[RB + ((pos - PL - nx) & rmask)];
                v -= (qzz - (qyz & Y)) & Z;
            }
            S[j] = v;
        }
    }
    S[0] = __shfl_up_sync(kFull, S[8], 1);
    if (lane == 0 || !fast_yz) {
        const uint32_t pos = g0 - 1;
        uint32_t v = (uint32_t)smem[pos & rmask];
        if (fast_yz) {
            if (NDIM >= 2) v -= (uint32_t)smem[(pos - nx) & rmask];
            if (NDIM == 3) v -= (uint32_t)smem[RB + ((pos - PL) & rmask)] - (uint32_t)smem[RB + ((pos - PL - nx) & rmask)];
        } else {
            const uint32_t Y = (ym & 1u) ? 0xFFFFFFFFu : 0u;
            const uint32_t Z = (zm & 1u) ? 0xFFFFFFFFu : 0u;
            if (NDIM >= 2) v -= (uint32_t)smem[(pos - nx) & rmask] & Y;
            if (NDIM == 3)
                v -= ((uint32_t)smem[RB + ((pos - PL) & rmask)] - ((uint32_t)smem[RB + ((pos - PL - nx) & rmask)] & Y)) & Z;
        }
        S[0] = v;
    }
    residuals(S, xm, dl);
}

// Tail of a tile on the compute warps (no look-back): codes, bitshuffle, outliers, flags,
// local compaction.  Returns the tile's nonzero block count.
__device__ __forceinline__ uint32_t tail_ws(const CompressArgs& a, WsShared& sh, uint32_t* Obuf, uint4* ring,
                                            uint32_t head, uint32_t t, uint32_t g0, uint32_t vm,
                                            const int32_t (&dl)[8], uint32_t vmask, const float (&dv)[8])
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    Ctrl* ctrl = a.ctrl;
    const uint32_t n = a.g.n;
    // ---- C3 codes; |delta| > 32767 (rare) -> code 0 + delta outlier (R7) ----
    uint32_t code[8];
    uint32_t magor = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const uint32_t mag = (uint32_t)abs(dl[e]);
        code[e] = (((uint32_t)dl[e] >> 16) & 0x8000u) | mag;
        magor |= mag;
    }
    uint32_t dmask = 0;
    if (magor > 32767u) {
#pragma unroll
        for (int e = 0; e < 8; ++e)
            if ((uint32_t)abs(dl[e]) > 32767u) { dmask |= 1u << e; code[e] = 0u; }
    }
    if (vm != 0xFFu) {
        dmask &= vm;
        vmask &= vm;
#pragma unroll
        for (int e = 0; e < 8; ++e)
            if (!((vm >> e) & 1u)) code[e] = 0u;
    }
    if (a.codes_out != nullptr) {
#pragma unroll
        for (int e = 0; e < 8; ++e)
            if (g0 + e < n) a.codes_out[g0 + e] = (uint16_t)code[e];
    }
    if (!a.rescan) {
        uint32_t w4[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) w4[i] = __byte_perm(code[2 * i], code[2 * i + 1], 0x5410);
        transpose32_group8(w4, lane & 7);
        const int c = tid >> 3, kk = tid & 7;
#pragma unroll
        for (int i = 0; i < 4; ++i) Obuf[(4 * kk + i) * 33 + c] = w4[i];
    }
    const int any_out = bar_or(kBarCompute, kCta, (dmask | vmask) != 0);
    if (any_out) {
        const int cd = __popc(dmask), cv = __popc(vmask);
        const int wd = __reduce_add_sync(kFull, cd), wv = __reduce_add_sync(kFull, cv);
        if (lane == 0) { sh.cd[warp] = wd; sh.cv[warp] = wv; }
        bar_sync(kBarCompute, kCta);
        uint32_t tnd = 0, tnv = 0, wpre_d = 0, wpre_v = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            tnd += sh.cd[w]; tnv += sh.cv[w];
            if (w < warp) { wpre_d += sh.cd[w]; wpre_v += sh.cv[w]; }
        }
        if (tid == 0) {
            if (a.rescan) {
                const uint2 o = a.opre[t];
                sh.ob[0] = o.x; sh.ob[1] = o.y;
            } else {
                sh.ob[0] = tnd ? atomicAdd(&ctrl->dcount, (unsigned long long)tnd) : 0ull;
                sh.ob[1] = tnv ? atomicAdd(&ctrl->vcount, (unsigned long long)tnv) : 0ull;
                a.ocnt[t] = make_uint2(tnd, tnv);
                a.obase[t] = make_uint2((uint32_t)sh.ob[0], (uint32_t)sh.ob[1]);
            }
        }
        int id = cd, iv = cv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int yd = __shfl_up_sync(kFull, id, o), yv = __shfl_up_sync(kFull, iv, o);
            if (lane >= o) { id += yd; iv += yv; }
        }
        bar_sync(kBarCompute, kCta);
        uint64_t pd = sh.ob[0] + wpre_d + (id - cd), pv = sh.ob[1] + wpre_v + (iv - cv);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const uint32_t gi = g0 + e;
            if (dmask & (1u << e)) {
                if (pd < a.dcap) {
                    if (a.o_didx) { a.o_didx[pd] = gi; a.o_dval[pd] = dl[e]; }
                    else a.dstage[pd] = make_uint2(gi, (uint32_t)dl[e]);
                } else {
                    atomicOr(&ctrl->stage_overflow, 1u);
                }
                ++pd;
            }
            if (vmask & (1u << e)) {
                if (pv < a.vcap) {
                    if (a.o_vidx) { a.o_vidx[pv] = gi; a.o_vbits[pv] = __float_as_uint(dv[e]); }
                    else a.vstage[pv] = make_uint2(gi, __float_as_uint(dv[e]));
                } else {
                    atomicOr(&ctrl->stage_overflow, 1u);
                }
                ++pv;
            }
        }
        bar_sync(kBarCompute, kCta);
    }
    if (a.rescan) return 0;
    const uint32_t* row = Obuf + (tid >> 3) * 33 + 4 * (tid & 7);
    const uint4 blk = make_uint4(row[0], row[1], row[2], row[3]);
    const bool nz = (blk.x | blk.y | blk.z | blk.w) != 0;
    const uint32_t F = __ballot_sync(kFull, nz);
    if (lane == 0) sh.F[warp] = F;
    if (tid == 0) {
        // room for a whole tile (worst case 256 blocks) in the payload ring
        while (head + kTileBlocks - sh.ring_tail > (uint32_t)kRingBlocks) __nanosleep(32);
        __threadfence_block();
    }
    bar_sync(kBarCompute, kCta);
    // block counts of the 8 flag words: lane l < 8 holds word l; warp prefix by reductions
    const uint32_t fw = lane < 8 ? sh.F[lane] : 0u;
    const uint32_t pc = __popc(fw);
    const uint32_t tn = __reduce_add_sync(kFull, pc);
    const uint32_t wpre = __reduce_add_sync(kFull, lane < warp ? pc : 0u);
    if (tid < 8) {
        const uint64_t fo = (uint64_t)(t - a.tile_begin) * 32 + 4 * tid;
        if (fo + 4 <= a.flags_cap) *reinterpret_cast<uint32_t*>(a.flags_out + fo) = fw;
    }
    if (nz) ring[(head + wpre + __popc(F & ((1u << lane) - 1u))) & (kRingBlocks - 1)] = blk;
    return tn;
}

__device__ void finalize_stream(uint8_t* out, uint64_t out_cap, uint32_t ndim, uint64_t d0, uint64_t d1,
                                uint64_t d2, uint64_t n, uint64_t T, Ctrl* ctrl, const fz_params& p);

template <int NDIM>
__global__ void __launch_bounds__(kWsThreads, 3) k_compress_ws(CompressArgs a)
{
    pdl_begin();
    extern __shared__ __align__(16) int smem[];
    __shared__ WsShared sh;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    Ctrl* ctrl = a.ctrl;
    if (ctrl->err != 0) return;
    const uint32_t rmask = a.qstride - 1;
    uint32_t* Obuf = reinterpret_cast<uint32_t*>(smem + a.qwords);           // 32 x 33
    uint4* ring = reinterpret_cast<uint4*>(smem + a.qwords + 32 * 33 + 4);    // kRingBlocks
    float* inbuf = reinterpret_cast<float*>(ring + kRingBlocks);              // own, previous plane
    const uint32_t nunits = (a.tile_end - a.tile_begin + kUnitTiles - 1) / kUnitTiles;

    if (tid == 0) {
        sh.perr = 0;
        if (a.derive) {
            // C0 parameters from k_range's result (every CTA derives the same values; CTA 0
            // publishes them for the host and the header)
            fz_params p;
            const int st = params_from_range(ctrl, a.eb_mode, a.eb, a.n_hdr, &p);
            sh.perr = st;
            if (st == FZ_OK) {
                float h, hU;
                quant_consts(p, h, hU);
                sh.p = p;
                sh.P = QuantP{p.w, p.r, h, p.eb32, hU};
                if (blockIdx.x == 0) { ctrl->p = p; ctrl->h = h; ctrl->hU = hU; }
            } else if (blockIdx.x == 0) {
                ctrl->err = st;
            }
        } else {
            sh.p = ctrl->p;
            sh.P = QuantP{ctrl->p.w, ctrl->p.r, ctrl->h, ctrl->p.eb32, ctrl->hU};
        }
        if (sh.perr == 0) {
            mbar_init(&sh.mbar, 1);
            for (int k = 0; k < kDescQ; ++k) mbar_init(&sh.desc_full[k], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            sh.ring_tail = 0;
            sh.desc_head = 0;
            sh.desc_tail = 0;
            sh.unit[0] = atomicAdd(&ctrl->ticket, 1u);
            sh.tma_bits = 0;
            if (sh.unit[0] < nunits) ws_issue<NDIM>(a, sh, inbuf, a.tile_begin + sh.unit[0] * kUnitTiles);
        }
    }
    __syncthreads();
    if (sh.perr != 0) return;

    if (warp == kCta / 32) {
        // ================= scanner warp =================
        for (uint32_t dt = 0; !a.rescan; ++dt) {
            // sleeps in hardware until the compute warps publish descriptor dt
            while (!mbar_try_wait_sleep(&sh.desc_full[dt % kDescQ], (dt / kDescQ) & 1u, 20000)) {
            }
            const WsDesc d = sh.desc[dt % kDescQ];
            if (d.unit == kNone) break;
            unsigned long long ex = 0;
            if (d.unit != 0) {
                ex = lookback_adaptive<kLbLane>(a.status, d.unit, kStAgg - 1, &ctrl->err);
                if (lane == 0) st_relaxed_u64(&a.status[d.unit], kStInc | (ex + d.cnt));
            }
            for (uint32_t i = lane; i < d.cnt; i += 32) {
                const uint64_t bo = 16 * (ex + i);
                if (bo + 16 <= a.payload_cap)
                    *reinterpret_cast<uint4*>(a.payload_out + bo) = ring[(d.start + i) & (kRingBlocks - 1)];
            }
            if (lane == 0 && d.unit == nunits - 1) ctrl->nnz = ex + d.cnt;
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                sh.ring_tail = d.start + d.cnt;
                sh.desc_tail = dt + 1;
            }
            __syncwarp();
        }
    } else {
    // ================= compute warps =================
    const QuantP P = sh.P;
    uint32_t phase = 0;      // parity of the next wait on the input stage
    uint32_t head = 0;       // payload ring blocks written so far
    for (int it = 0;; ++it) {
        const uint32_t u = sh.unit[it & 1];
        if (u >= nunits) {
            if (!a.rescan && tid == 0) {
                while (sh.desc_head - sh.desc_tail >= (uint32_t)kDescQ) __nanosleep(32);
                const uint32_t dh = sh.desc_head;
                sh.desc[dh % kDescQ].unit = kNone;
                sh.desc_head = dh + 1;
                mbar_arrive(&sh.desc_full[dh % kDescQ]);
            }
            break;
        }
        const uint32_t t_first = a.tile_begin + u * kUnitTiles;
        const uint32_t t_last = min(a.tile_end, t_first + kUnitTiles);
        const uint32_t start = head;
        // thread's in-row / in-plane positions, advanced per tile without divisions
        uint32_t x0 = 0, p0 = 0;
        {
            const uint32_t g = t_first * kTileCodes + 8u * tid;
            if (a.g.nx >= 8) {
                x0 = fmod_(g, a.dnx);
                if (NDIM >= 2) p0 = fmod_(g, a.dP);
            }
        }
        for (uint32_t t = t_first; t < t_last; ++t) {
            const bool first = t == t_first;
            const uint32_t bits = sh.tma_bits;
            if (bits) {
                while (!mbar_try_wait(&sh.mbar, phase)) {
                }
                phase ^= 1u;
            }
            int32_t dl[8];
            uint32_t vmask, vm;
            float dv[8];
            // as soon as every compute thread has consumed the input stage: TMA of the next tile
            auto issue_next = [&]() {
                if (tid == 0) {
                    if (first) sh.unit[(it & 1) ^ 1] = atomicAdd(&ctrl->ticket, 1u);
                    const uint32_t nu = sh.unit[(it & 1) ^ 1];
                    uint32_t nt = kNone;
                    if (t + 1 < t_last) nt = t + 1;
                    else if (nu < nunits) nt = a.tile_begin + nu * kUnitTiles;
                    if (nt != kNone) ws_issue<NDIM>(a, sh, inbuf, nt);
                    else sh.tma_bits = 0;
                    if (first && nu < nunits)   // L2 prefetch of the next unit beyond the TMA stage
                        prefetch_l2_range(a, (uint64_t)(a.tile_begin + nu * kUnitTiles) * kTileCodes,
                                          (uint64_t)kUnitTiles * kTileCodes);
                }
            };
            front_ws<NDIM>(a, P, smem, rmask, t, first, (bits & 1) ? inbuf : nullptr,
                           (bits & 2) ? inbuf + kTileCodes : nullptr, x0, p0, dl, vmask, dv, vm, issue_next);
            x0 += a.sx;
            if (x0 >= a.g.nx) x0 -= a.g.nx;
            p0 += a.sp;
            if (p0 >= a.g.P) p0 -= a.g.P;
            head += tail_ws(a, sh, Obuf, ring, head, t, (uint32_t)t * kTileCodes + 8u * tid, vm, dl, vmask, dv);
        }
        bar_sync(kBarCompute, kCta);   // all ring writes of the unit are done
        if (!a.rescan && tid == 0) {
            st_relaxed_u64(&a.status[u], (u == 0 ? kStInc : kStAgg) | (head - start));
            while (sh.desc_head - sh.desc_tail >= (uint32_t)kDescQ) __nanosleep(32);
            const uint32_t dh = sh.desc_head;
            sh.desc[dh % kDescQ] = WsDesc{u, start, head - start, 0};
            sh.desc_head = dh + 1;
            mbar_arrive(&sh.desc_full[dh % kDescQ]);
        }
    }
    }
    // C9: the last CTA to finish writes the totals and the header (replaces k_finalize)
    __syncthreads();
    if (a.finalize && tid == 0) {
        __threadfence();
        const uint32_t prev = atomicAdd(&ctrl->done, 1u);
        if (prev == gridDim.x - 1) {
            __threadfence();
            if (*(volatile int32_t*)&ctrl->err == 0)
                finalize_stream(a.hdr_out, a.hdr_cap, a.ndim, a.dims[0], a.dims[1], a.dims[2], a.n_hdr, a.T_hdr,
                                ctrl, sh.p);
        }
    }
}

// ------------------------------------------------------------------------------------
// z-band compression, pass 1 (3-D fields with whole tiles per plane, P % 2048 == 0).
// A work item is a column of tiles: tile position p of the planes [z0, z0 + Zc).  The CTA
// walks it plane by plane, so the previous plane's quantized values are still in its shared
// ring from the step before (the two rings swap roles every step) -- no re-quantization of
// the previous plane, no previous-plane TMA.  Only the row halo (the nx+1 elements before the
// tile, from the neighbouring tile of the same plane) is quantized again, from the TMA
// stage.  Each tile's flags go straight to the stream; its nonzero blocks go to a staging
// slot of 256 blocks (pass 2, k_compact, moves them to their final offsets), so no ordering
// between CTAs is needed: no look-back, no scanner warp, any work order.
// ------------------------------------------------------------------------------------
constexpr int kZbChunk = 16;       // planes per work item

struct ZbShared {
    uint64_t mbar;
    uint32_t tma_bits;             // bit0 own tile, bit1 own row halo staged by TMA
    uint32_t item;
    uint32_t F[8];
    uint32_t cd[8], cv[8];
    unsigned long long ob[2];
    QuantP P;
    fz_params p;
    int perr;
};

__device__ __forceinline__ void zb_issue(const CompressArgs& a, ZbShared& sh, float* inbuf, uint32_t t)
{
    const int64_t s = (int64_t)t * kTileCodes, base = (int64_t)a.base;
    const int64_t hw = (int64_t)a.hwords;
    const bool full = s + kTileCodes <= (int64_t)a.g.n;
    uint32_t bits = 0, bytes = 0;
    if (full && s >= base) { bits |= 1; bytes += kTileCodes * 4; }
    if (hw > 0 && s - hw >= base) { bits |= 2; bytes += (uint32_t)hw * 4; }
    sh.tma_bits = bits;
    if (bytes) {
        mbar_expect_tx(&sh.mbar, bytes);
        if (bits & 1) tma_load_1d(inbuf, a.field + (s - base), kTileCodes * 4, &sh.mbar);
        if (bits & 2) tma_load_1d(inbuf + kTileCodes, a.field + (s - hw - base), (uint32_t)hw * 4, &sh.mbar);
    }
}

// Quantize the hw floats staged in shared memory (field elements [g_lo, g_lo + hw)) into ring
// `ro` (positions & rmask).  Element-strided over the whole CTA so every warp does about the
// same share (the front barrier follows); warp-uniform trip count (pq_many votes per warp).
__device__ __forceinline__ void zb_fill_halo(const QuantP& P, int* smem, int ro, uint32_t rmask, const float* src,
                                             int64_t g_lo, int hw)
{
    const int wbase = (int)(threadIdx.x & ~31u);
    for (int b0 = 0; b0 < hw; b0 += 2 * kCta) {
        if (b0 + wbase >= hw) break;   // warp-uniform: no element left for this warp
        const int c0 = b0 + (int)threadIdx.x, c1 = c0 + kCta;
        const bool has1 = b0 + kCta + wbase < hw;   // warp-uniform
        float v[2];
        int q[2];
        v[0] = c0 < hw ? src[c0] : 0.0f;
        v[1] = (has1 && c1 < hw) ? src[c1] : 0.0f;
        if (has1) {
            pq_many<2>(v, q, P);
        } else {
            float v1[1] = {v[0]};
            int q1[1];
            pq_many<1>(v1, q1, P);
            q[0] = q1[0];
        }
        const uint32_t g = (uint32_t)(g_lo + c0);
        if (c0 < hw) smem[ro + (g & rmask)] = q[0];
        if (has1 && c1 < hw) smem[ro + ((g + kCta) & rmask)] = q[1];
    }
}

// Front half of a z-band step.  The thread's 8 elements sit at the same in-plane positions
// in every plane of the work item, so the Lorenzo residual is built from the y-difference
// D(z, e) = q(z, e) - [y>0] q(z, e - nx): S(e) = D(z, e) - [z>0] D(z-1, e) and
// delta(e) = S(e) - [x>0] S(e-1) (C2).  D(z-1, .) is carried in registers (Dp, and
// Dp0 for element g0-1 on lane 0), so the previous plane is neither re-quantized nor
// re-read; only at a chunk start (z0 > 0) is the previous plane's tile (+ row halo)
// quantized once into ring rb to seed the carry.  Own tile + row halo go to ring ra.
// xm / ym (x-1 / y-1 neighbour exists, bit e) are per work item.
template <class OnFree>
__device__ __forceinline__ void front_zb(const CompressArgs& a, const QuantP& P, int* smem, uint32_t rmask, int ra,
                                         int rb, uint32_t t, bool bstart, const float* in_own, const float* in_halo,
                                         uint32_t xm, uint32_t ym, uint32_t (&Dp)[8], uint32_t& Dp0,
                                         int32_t (&dl)[8], uint32_t& vmask, float (&dv)[8], OnFree&& on_input_free)
{
    const int tid = threadIdx.x, lane = tid & 31;
    const uint32_t nx = a.g.nx, PL = a.g.P;
    const int64_t s = (int64_t)t * kTileCodes;
    const uint32_t g0 = (uint32_t)s + 8u * tid;
    const int64_t H = (int64_t)nx + 1;
    if (in_own) {
        const float4 x = *reinterpret_cast<const float4*>(in_own + 8 * tid);
        const float4 y = *reinterpret_cast<const float4*>(in_own + 8 * tid + 4);
        dv[0] = x.x; dv[1] = x.y; dv[2] = x.z; dv[3] = x.w; dv[4] = y.x; dv[5] = y.y; dv[6] = y.z; dv[7] = y.w;
    } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) dv[u] = load1(a, (int64_t)g0 + u);
    }
    // row halo (the y-1 neighbours of the tile's first row); chunk-local mode (f1) has none
    if (in_halo) zb_fill_halo(P, smem, ra, rmask, in_halo, s - (int64_t)a.hwords, (int)a.hwords);
    else if (!a.cl) fill_ring(a, P, smem, ra, rmask, (s - H) & ~(int64_t)3, s);
    if (bstart)   // first step of a chunk: the previous plane's tile and halo, once
        fill_ring(a, P, smem, rb, rmask, (s - (int64_t)PL - H) & ~(int64_t)3, s - (int64_t)PL + kTileCodes);
    int qo[8];
    pq_own(dv, qo, vmask, P);
    *reinterpret_cast<int4*>(smem + ra + (g0 & rmask)) = make_int4(qo[0], qo[1], qo[2], qo[3]);
    *reinterpret_cast<int4*>(smem + ra + ((g0 + 4) & rmask)) = make_int4(qo[4], qo[5], qo[6], qo[7]);
    bar_sync(kBarCompute, kCta);
    on_input_free();   // every thread has read the TMA stage

    if (bstart) {      // seed the carry with D(z0-1, .)
        const uint32_t gb = g0 - PL;
        uint32_t zz[8], zy[8];
        {
            const int4 p = *reinterpret_cast<const int4*>(smem + rb + (gb & rmask));
            const int4 q = *reinterpret_cast<const int4*>(smem + rb + ((gb + 4) & rmask));
            zz[0] = p.x; zz[1] = p.y; zz[2] = p.z; zz[3] = p.w; zz[4] = q.x; zz[5] = q.y; zz[6] = q.z; zz[7] = q.w;
        }
        {
            const int4 p = *reinterpret_cast<const int4*>(smem + rb + ((gb - nx) & rmask));
            const int4 q = *reinterpret_cast<const int4*>(smem + rb + ((gb - nx + 4) & rmask));
            zy[0] = p.x; zy[1] = p.y; zy[2] = p.z; zy[3] = p.w; zy[4] = q.x; zy[5] = q.y; zy[6] = q.z; zy[7] = q.w;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) Dp[e] = zz[e] - (((ym >> e) & 1u) ? zy[e] : 0u);
        if (lane == 0 && (xm & 1u)) {
            Dp0 = (uint32_t)smem[rb + ((gb - 1) & rmask)];
            if (ym & 1u) Dp0 -= (uint32_t)smem[rb + ((gb - 1 - nx) & rmask)];
        }
    }
    uint32_t y[8];
    {
        const int4 p = *reinterpret_cast<const int4*>(smem + ra + ((g0 - nx) & rmask));
        const int4 q = *reinterpret_cast<const int4*>(smem + ra + ((g0 - nx + 4) & rmask));
        y[0] = p.x; y[1] = p.y; y[2] = p.z; y[3] = p.w; y[4] = q.x; y[5] = q.y; y[6] = q.z; y[7] = q.w;
    }
    if (ym != 0xFFu) {   // first row of the plane among the 8 elements: no y-1 neighbour
#pragma unroll
        for (int e = 0; e < 8; ++e)
            if (!((ym >> e) & 1u)) y[e] = 0u;
    }
    uint32_t S[9];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const uint32_t D = (uint32_t)qo[e] - y[e];
        S[e + 1] = D - Dp[e];
        Dp[e] = D;
    }
    S[0] = __shfl_up_sync(kFull, S[8], 1);
    if (lane == 0 && (xm & 1u)) {   // element g0-1 (same row) belongs to the previous warp
        uint32_t D = (uint32_t)smem[ra + ((g0 - 1) & rmask)];
        if (ym & 1u) D -= (uint32_t)smem[ra + ((g0 - 1 - nx) & rmask)];
        S[0] = D - Dp0;
        Dp0 = D;
    }
    residuals(S, xm, dl);
}

// Tail of a z-band step: codes, bitshuffle, outliers, flags to the stream, nonzero blocks
// to the tile's staging slot.
__device__ __forceinline__ void tail_zb(const CompressArgs& a, ZbShared& sh, uint32_t* Obuf, uint32_t t, uint32_t g0,
                                        uint32_t vm, const int32_t (&dl)[8], uint32_t vmask)
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    Ctrl* ctrl = a.ctrl;
    const uint32_t n = a.g.n;
    // C3/C4: two sign-magnitude codes per word, built pairwise: magnitudes by PRMT, both
    // sign bits (bit 31 of each delta -> bits 15 and 31) by a second PRMT, merged by LOP3.
    uint32_t w4[4];
    uint32_t magor = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t m0 = (uint32_t)abs(dl[2 * i]), m1 = (uint32_t)abs(dl[2 * i + 1]);
        magor |= m0 | m1;
        w4[i] = bitsel(__byte_perm((uint32_t)dl[2 * i], (uint32_t)dl[2 * i + 1], 0x7030u), __byte_perm(m0, m1, 0x5410u),
                       0x80008000u);
    }
    uint32_t dmask = 0;
    if (magor > 32767u || vm != 0xFFu) {   // delta-outliers (R7) or a partial tile: code 0
#pragma unroll
        for (int i = 0; i < 4; ++i) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int e = 2 * i + h;
                const bool drop = (uint32_t)abs(dl[e]) > 32767u;
                if (drop) dmask |= 1u << e;
                if (drop || !((vm >> e) & 1u)) w4[i] &= h ? 0x0000FFFFu : 0xFFFF0000u;
            }
        }
        dmask &= vm;
        vmask &= vm;
    }
    if (a.codes_out != nullptr) {
#pragma unroll
        for (int e = 0; e < 8; ++e)
            if (g0 + e < n) a.codes_out[g0 + e] = (uint16_t)(w4[e >> 1] >> (16 * (e & 1)));
    }
    {
        transpose32_group8(w4, lane & 7);
        const int c = tid >> 3, kk = tid & 7;
#pragma unroll
        for (int i = 0; i < 4; ++i) Obuf[(4 * kk + i) * 33 + c] = w4[i];
    }
    const int any_out = bar_or(kBarCompute, kCta, (dmask | vmask) != 0);
    if (any_out) {
        const int cd = __popc(dmask), cv = __popc(vmask);
        const int wd = __reduce_add_sync(kFull, cd), wv = __reduce_add_sync(kFull, cv);
        if (lane == 0) { sh.cd[warp] = wd; sh.cv[warp] = wv; }
        bar_sync(kBarCompute, kCta);
        uint32_t tnd = 0, tnv = 0, wpre_d = 0, wpre_v = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            tnd += sh.cd[w]; tnv += sh.cv[w];
            if (w < warp) { wpre_d += sh.cd[w]; wpre_v += sh.cv[w]; }
        }
        if (tid == 0) {
            sh.ob[0] = tnd ? atomicAdd(&ctrl->dcount, (unsigned long long)tnd) : 0ull;
            sh.ob[1] = tnv ? atomicAdd(&ctrl->vcount, (unsigned long long)tnv) : 0ull;
            a.ocnt[t] = make_uint2(tnd, tnv);
            a.obase[t] = make_uint2((uint32_t)sh.ob[0], (uint32_t)sh.ob[1]);
        }
        int id = cd, iv = cv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int yd = __shfl_up_sync(kFull, id, o), yv = __shfl_up_sync(kFull, iv, o);
            if (lane >= o) { id += yd; iv += yv; }
        }
        bar_sync(kBarCompute, kCta);
        uint64_t pd = sh.ob[0] + wpre_d + (id - cd), pv = sh.ob[1] + wpre_v + (iv - cv);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const uint32_t gi = g0 + e;
            if (dmask & (1u << e)) {
                if (pd < a.dcap) a.dstage[pd] = make_uint2(gi, (uint32_t)dl[e]);
                else atomicOr(&ctrl->stage_overflow, 1u);
                ++pd;
            }
            if (vmask & (1u << e)) {
                // raw bits re-read from the field (rare path; keeps the 8 inputs out of registers)
                if (pv < a.vcap) a.vstage[pv] = make_uint2(gi, __float_as_uint(__ldg(a.field + (gi - a.base))));
                else atomicOr(&ctrl->stage_overflow, 1u);
                ++pv;
            }
        }
        bar_sync(kBarCompute, kCta);
    }
    // C6: thread tid holds block b = tid (O[r][4x..4x+3], r = tid/8, x = tid%8), so warp w's
    // ballot is flag word w.  Its nonzero blocks go to sub-slot w (32 blocks) of the tile's
    // staging slot in lane order; k_compact concatenates the sub-slots (C8 order b).  No
    // cross-warp exchange, no barrier.
    const uint32_t* row = Obuf + (tid >> 3) * 33 + 4 * (tid & 7);
    const uint4 blk = make_uint4(row[0], row[1], row[2], row[3]);
    const bool nz = (blk.x | blk.y | blk.z | blk.w) != 0;
    const uint32_t F = __ballot_sync(kFull, nz);
    if (lane == 0) {
        const uint64_t fo = (uint64_t)(t - a.tile_begin) * 32 + 4 * warp;
        if (fo + 4 <= a.flags_cap) *reinterpret_cast<uint32_t*>(a.flags_out + fo) = F;
    }
    if (nz) a.tstage[(uint64_t)(t - a.tile_begin) * kTileBlocks + 32 * warp + __popc(F & ((1u << lane) - 1u))] = blk;
}

__global__ void __launch_bounds__(kCta, 4) k_compress_zb(CompressArgs a)
{
    pdl_begin();
    extern __shared__ __align__(16) int smem[];
    __shared__ ZbShared sh;
    const int tid = threadIdx.x;
    Ctrl* ctrl = a.ctrl;
    if (ctrl->err != 0) return;
    const uint32_t rmask = a.qstride - 1;
    const int RB = (int)a.qstride;
    uint32_t* Obuf = reinterpret_cast<uint32_t*>(smem + a.qwords);              // 32 x 33
    float* inbuf = reinterpret_cast<float*>(smem + a.qwords + 32 * 33 + 4);    // own tile + row halo
    // planes [zbeg, zend) of this call (a slab's tile range is plane-aligned; see compress_uses_zb)
    const uint32_t tpp = a.g.P / kTileCodes, zbeg = a.tile_begin / tpp, zend = a.tile_end / tpp;
    const uint32_t nchunks = (zend - zbeg + kZbChunk - 1) / kZbChunk, nwork = tpp * nchunks;
    if (tid == 0) {
        sh.perr = 0;
        if (a.derive) {
            fz_params p;
            const int st = params_from_range(ctrl, a.eb_mode, a.eb, a.n_hdr, &p);
            sh.perr = st;
            if (st == FZ_OK) {
                float h, hU;
                quant_consts(p, h, hU);
                sh.p = p;
                sh.P = QuantP{p.w, p.r, h, p.eb32, hU};
                if (blockIdx.x == 0) { ctrl->p = p; ctrl->h = h; ctrl->hU = hU; }
            } else if (blockIdx.x == 0) {
                ctrl->err = st;
            }
        } else {
            sh.P = QuantP{ctrl->p.w, ctrl->p.r, ctrl->h, ctrl->p.eb32, ctrl->hU};
        }
        mbar_init(&sh.mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        sh.tma_bits = 0;
    }
    __syncthreads();
    if (sh.perr != 0) return;
    const QuantP P = sh.P;
    uint32_t phase = 0;
    for (;;) {
        if (tid == 0) sh.item = atomicAdd(&ctrl->ticket, 1u);
        __syncthreads();
        const uint32_t w = sh.item;
        if (w >= nwork) break;
        const uint32_t c = w / tpp, p = w - c * tpp;
        const uint32_t z0 = zbeg + c * kZbChunk, z1 = min(zend, z0 + kZbChunk);
        // the thread's in-row / in-plane positions are the same in every plane of the column
        const uint32_t pp = p * kTileCodes + 8u * tid;
        // pp + e < P: no plane wrap inside a thread's 8 elements.  nx >= 4, so x0 + e < 3 nx and
        // a row starts at element e iff x0 + e is 0, nx or 2 nx.
        uint32_t xm = 0xFFu, ym = 0xFFu;
        {
            const uint32_t x0 = fmod_(pp, a.dnx), nx = a.g.nx;
            // chunk-local (f1): a tile is one chunk plane, so its first row has no y-1 neighbour
            const uint32_t yoff = a.cl ? 8u * tid : pp;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const uint32_t xe = x0 + e;
                if (xe == 0 || xe == nx || xe == 2 * nx) xm &= ~(1u << e);
                if (yoff + e < nx) ym &= ~(1u << e);
            }
        }
        uint32_t Dp[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u}, Dp0 = 0u;
        if (tid == 0) zb_issue(a, sh, inbuf, z0 * tpp + p);
        for (uint32_t z = z0; z < z1; ++z) {
            const uint32_t t = z * tpp + p;
            // sh.tma_bits: at z0 written by thread 0 just above; later by issue_next in the
            // previous step's front, ordered by that step's tail barrier (bar_or)
            if (z == z0) __syncthreads();
            const uint32_t bits = sh.tma_bits;
            if (bits) {
                while (!mbar_try_wait(&sh.mbar, phase)) {
                }
                phase ^= 1u;
            }
            int32_t dl[8];
            uint32_t vmask;
            float dv[8];
            auto issue_next = [&]() {
                if (tid == 0) {
                    if (z + 1 < z1) zb_issue(a, sh, inbuf, t + tpp);
                    else sh.tma_bits = 0;
                }
            };
            // opaque per-step copies: keeps the compiler from hoisting 16 per-element mask
            // registers out of the z loop (they spill at 64 registers)
            uint32_t xmv, ymv;
            asm volatile("mov.b32 %0, %1;" : "=r"(xmv) : "r"(xm));
            asm volatile("mov.b32 %0, %1;" : "=r"(ymv) : "r"(ym));
            // chunk-local (f1): items are whole chunks, the z carry starts from zero
            front_zb(a, P, smem, rmask, 0, RB, t, z == z0 && z > 0 && !a.cl, (bits & 1) ? inbuf : nullptr,
                     (bits & 2) ? inbuf + kTileCodes : nullptr, xmv, ymv, Dp, Dp0, dl, vmask, dv, issue_next);
            tail_zb(a, sh, Obuf, t, (uint32_t)t * kTileCodes + 8u * tid, 0xFFu, dl, vmask);
        }
    }
}

// Pass 2: each tile's staged blocks to their final offsets (exclusive scan of the flag
// popcounts by k_nnz_block/k_nnz_top).  One warp per tile.
// C8: one warp per tile moves the tile's staged nonzero blocks to the payload at
// offset bpre + loc (the popcount scan).  Sub-slot w of the staging slot holds flag word w's
// nonzero blocks in block order, so the tile's k-th nonzero block is entry k - E[w] of
// sub-slot w, w = #{i : I[i] <= k} (I / E = inclusive / exclusive prefixes of the 8 flag
// words' popcounts).  Lanes take consecutive k (dense: a tile has ~50 of 256 blocks set on c4),
// every load of the tile is issued before its stores, and the next tile's flags and offsets
// are loaded while this tile's blocks move.
// C9 rides along: thread 0 of block 0 writes the totals and the header (k_finalize's work; the
// scan's nnz and the walker's outlier counts are complete when this kernel starts).
__global__ void __launch_bounds__(256, 6) k_compact(const uint32_t* __restrict__ flags, const uint32_t* __restrict__ loc,
                                                 const uint32_t* __restrict__ bpre, const uint4* __restrict__ tstage,
                                                 uint8_t* payload_out, uint64_t payload_cap, uint32_t ntiles,
                                                 uint8_t* hdr_out, uint64_t hdr_cap, uint32_t ndim, uint64_t d0,
                                                 uint64_t d1, uint64_t d2, uint64_t n_hdr, uint64_t T_hdr, Ctrl* ctrl)
{
    pdl_begin();
    if (blockIdx.x == 0 && threadIdx.x == 0 && ctrl->err == 0)
        finalize_stream(hdr_out, hdr_cap, ndim, d0, d1, d2, n_hdr, T_hdr, ctrl, ctrl->p);
    const int lane = threadIdx.x & 31;
    const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    uint32_t t = wid;
    if (t >= ntiles) return;
    uint32_t fw = lane < 8 ? __ldg(flags + 8 * (uint64_t)t + lane) : 0u;
    uint64_t off = (uint64_t)__ldg(bpre + (t >> 10)) + __ldg(loc + t);
    for (;;) {
        const uint32_t tn = t + nw;
        // the next tile's metadata in flight while this one moves
        uint32_t fwn = 0u;
        uint64_t offn = 0;
        if (tn < ntiles) {
            fwn = lane < 8 ? __ldg(flags + 8 * (uint64_t)tn + lane) : 0u;
            offn = (uint64_t)__ldg(bpre + (tn >> 10)) + __ldg(loc + tn);
        }
        const uint32_t pc = __popc(fw);
        uint32_t inc = pc;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, inc, o);
            if (lane >= o) inc += y;
        }
        uint32_t I[8];
#pragma unroll
        for (int w = 0; w < 8; ++w) I[w] = __shfl_sync(kFull, inc, w);
        const uint32_t total = I[7];
        const uint4* src = tstage + (uint64_t)t * kTileBlocks;
        // two rounds of 32 blocks per pass (a c4 tile has ~50 nonzero blocks): both loads in
        // flight before the stores, few registers (6 CTAs of 256 threads per SM)
#pragma unroll 1
        for (uint32_t r0 = 0; r0 < total; r0 += 64) {
            uint4 v[2];
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const uint32_t k = (uint32_t)lane + r0 + 32u * r;
                if (k < total) {
                    uint32_t w = 0, e = 0;
#pragma unroll
                    for (int i = 0; i < 7; ++i)
                        if (I[i] <= k) { w = i + 1; e = I[i]; }
                    v[r] = __ldcs(src + 32 * w + (k - e));
                }
            }
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const uint32_t k = (uint32_t)lane + r0 + 32u * r;
                if (k < total) {
                    const uint64_t bo = 16 * (off + k);
                    if (bo + 16 <= payload_cap) __stcs(reinterpret_cast<uint4*>(payload_out + bo), v[r]);
                }
            }
        }
        if (tn >= ntiles) break;
        t = tn;
        fw = fwn;
        off = offn;
    }
}

// ------------------------------------------------------------------------------------
// C9: header (outlier sections are placed by k_outlier_place when there are any).
// ------------------------------------------------------------------------------------
// C9 totals and header (one thread): k_finalize, or the last CTA of the ws kernel.
__device__ void finalize_stream(uint8_t* out, uint64_t out_cap, uint32_t ndim, uint64_t d0, uint64_t d1,
                                uint64_t d2, uint64_t n, uint64_t T, Ctrl* ctrl, const fz_params& p)
{
    const uint64_t nnz = *(volatile unsigned long long*)&ctrl->nnz;
    const uint64_t nd = *(volatile unsigned long long*)&ctrl->dcount;
    const uint64_t nv = *(volatile unsigned long long*)&ctrl->vcount;
    const uint64_t total = kHeaderBytes + 32 * T + 16 * nnz + 8 * nd + 8 * nv;
    ctrl->nd = nd;
    ctrl->nv = nv;
    ctrl->total = total;
    if (total > out_cap || out == nullptr) return;
    uint8_t h[128];
    for (int i = 0; i < 128; ++i) h[i] = 0;
    h[0] = 'F'; h[1] = 'Z'; h[2] = 'B'; h[3] = '2';
    const uint32_t chunk = ctrl->chunk;
    const uint16_t ver = 1,
                   fl = (uint16_t)((p.mode == FZ_EB_REL ? 1u : 0u) | (p.fallback ? 2u : 0u) | (chunk ? 4u : 0u) |
                                   (p.mode == FZ_EB_PWREL ? 8u : 0u));
    memcpy(h + 4, &ver, 2);
    memcpy(h + 6, &fl, 2);
    h[8] = (uint8_t)ndim;
    memcpy(h + 10, &chunk, 4);     // f1: chunk depth (u16) and height (u16), zero otherwise
    uint64_t dims[3] = {d0, d1, d2};
    memcpy(h + 16, dims, 24);
    memcpy(h + 40, &n, 8);
    memcpy(h + 48, &p.eb_input, 8);
    memcpy(h + 56, &p.eb_abs, 8);
    memcpy(h + 64, &p.w, 4);
    memcpy(h + 68, &p.r, 4);
    memcpy(h + 72, &p.mn, 4);
    memcpy(h + 76, &p.mx, 4);
    uint64_t cnt[5] = {T, nnz, nd, nv, total};
    memcpy(h + 80, cnt, 40);
    uint4* o = reinterpret_cast<uint4*>(out);
    const uint4* hs = reinterpret_cast<const uint4*>(h);
    for (int i = 0; i < 8; ++i) o[i] = hs[i];
}

__global__ void k_finalize(uint8_t* out, uint64_t out_cap, uint32_t ndim, uint64_t d0, uint64_t d1,
                           uint64_t d2, uint64_t n, uint64_t T, Ctrl* ctrl)
{
    pdl_begin();
    if (ctrl->err != 0 || threadIdx.x != 0) return;
    finalize_stream(out, out_cap, ndim, d0, d1, d2, n, T, ctrl, ctrl->p);
}

// Exclusive scan of the per-tile outlier counts (one block; only when outliers exist).
__global__ void __launch_bounds__(1024) k_outlier_scan(const uint2* ocnt, uint2* opre, uint32_t ntiles,
                                                       const Ctrl* ctrl)
{
    pdl_begin();
    __shared__ uint32_t wd[32], wv[32];
    __shared__ uint32_t carry_d, carry_v;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // device-driven mode: nothing to do without outliers (ctrl == null: the host checked)
    if (ctrl != nullptr && (ctrl->err != 0 || ctrl->dcount + ctrl->vcount == 0)) return;
    if (tid == 0) { carry_d = 0; carry_v = 0; }
    __syncthreads();
    for (uint32_t base = 0; base < ntiles; base += 1024) {
        const uint32_t t = base + tid;
        const uint2 c = t < ntiles ? ocnt[t] : make_uint2(0, 0);
        uint32_t id = c.x, iv = c.y;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t yd = __shfl_up_sync(kFull, id, o), yv = __shfl_up_sync(kFull, iv, o);
            if (lane >= o) { id += yd; iv += yv; }
        }
        if (lane == 31) { wd[warp] = id; wv[warp] = iv; }
        __syncthreads();
        uint32_t pd = carry_d, pv = carry_v;
        for (int w = 0; w < warp; ++w) { pd += wd[w]; pv += wv[w]; }
        if (t < ntiles) opre[t] = make_uint2(pd + id - c.x, pv + iv - c.y);
        __syncthreads();
        if (tid == 1023) { carry_d = pd + id; carry_v = pv + iv; }
        __syncthreads();
    }
}

// Copies each tile's staged records to its final place (records, or split lists).
__global__ void k_outlier_place(const uint2* ocnt, const uint2* obase, const uint2* opre, uint32_t ntiles,
                                const uint2* dstage, const uint2* vstage, uint2* dout, uint2* vout,
                                uint32_t* didx, int32_t* dval, uint32_t* vidx, uint32_t* vbits)
{
    pdl_begin();
    const int lane = threadIdx.x & 31;
    const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t t = wid; t < ntiles; t += nw) {
        const uint2 c = ocnt[t];
        if ((c.x | c.y) == 0) continue;
        const uint2 b = obase[t], p = opre[t];
        for (uint32_t k = lane; k < c.x; k += 32) {
            const uint2 r = dstage[b.x + k];
            if (didx) { didx[p.x + k] = r.x; dval[p.x + k] = (int32_t)r.y; }
            else dout[p.x + k] = r;
        }
        for (uint32_t k = lane; k < c.y; k += 32) {
            const uint2 r = vstage[b.y + k];
            if (vidx) { vidx[p.y + k] = r.x; vbits[p.y + k] = r.y; }
            else vout[p.y + k] = r;
        }
    }
}

// Device-driven placement (asynchronous compression): destinations from the totals in ctrl;
// a staging overflow (the rescan needs the host) is reported as FZ_ERR_WORKSPACE.
__global__ void k_outlier_place_dev(const uint2* ocnt, const uint2* obase, const uint2* opre, uint32_t ntiles,
                                    const uint2* dstage, const uint2* vstage, uint8_t* payload_out,
                                    uint64_t payload_cap, Ctrl* ctrl)
{
    pdl_begin();
    if (ctrl->err != 0) return;
    const uint64_t nd = ctrl->dcount, nv = ctrl->vcount, nnz = ctrl->nnz;
    if (nd + nv == 0) return;
    if (ctrl->stage_overflow) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicCAS(&ctrl->err, 0, (int)FZ_ERR_WORKSPACE);
        return;
    }
    if (16 * nnz + 8 * (nd + nv) > payload_cap) return;   // capacity: reported by the result call
    uint2* dout = reinterpret_cast<uint2*>(payload_out + 16 * nnz);
    uint2* vout = dout + nd;
    const int lane = threadIdx.x & 31;
    const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t t = wid; t < ntiles; t += nw) {
        const uint2 c = ocnt[t];
        if ((c.x | c.y) == 0) continue;
        const uint2 b = obase[t], p = opre[t];
        for (uint32_t k = lane; k < c.x; k += 32) dout[p.x + k] = dstage[b.x + k];
        for (uint32_t k = lane; k < c.y; k += 32) vout[p.y + k] = vstage[b.y + k];
    }
}

// ------------------------------------------------------------------------------------
// Host-side launch wrappers.
// ------------------------------------------------------------------------------------
static int g_sms = 0;
int num_sms()
{
    if (g_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_sms <= 0) g_sms = 148;
    }
    return g_sms;
}

// Shared q storage for a shape; fills a.union_mode / a.qstride / a.qwords and returns the
// dynamic shared memory bytes.  vec: rings of R = 2^k >= 2048 + halo + 4 elements.
static size_t plan_smem(CompressArgs& a, bool& vec)
{
    const uint32_t ndim = a.g.ndim, nx = a.g.nx;
    const uint32_t halo = ndim >= 2 ? nx + 1 : 1;
    vec = (ndim == 1 || (nx % 4) == 0) && (a.base % 4) == 0 && halo + kTileCodes + 4 <= 8192;
    if (vec) {
        uint32_t R = 1;
        while (R < halo + kTileCodes + 4) R <<= 1;
        a.union_mode = 1;
        a.qstride = R;
        a.qwords = (ndim == 3 ? 2 : 1) * R;
    } else {
        uint32_t narr, len;
        if (ndim == 1) {
            narr = 1;
            len = kTileCodes + 1;
            a.union_mode = 0;
        } else if (nx + 1 <= kUnionHaloMax) {
            a.union_mode = 1;
            narr = ndim == 3 ? 2 : 1;
            len = kTileCodes + nx + 1;
        } else {
            a.union_mode = 0;
            narr = ndim == 3 ? 4 : 2;
            len = kTileCodes + 1;
        }
        a.qstride = (pad_words(len) + 31) & ~31u;
        a.qwords = narr * a.qstride;
    }
    a.qwords = (a.qwords + 3) & ~3u;
    return sizeof(int) * ((size_t)a.qwords + 32 * 33 + 8) + 2 * 16 * (size_t)kStageBlocks;
}

template <int NDIM, bool VEC>
static cudaError_t launch_compress_t(const CompressArgs& a, size_t sm, uint32_t ntiles, cudaStream_t st)
{
    cudaFuncSetAttribute(k_compress<NDIM, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_compress<NDIM, VEC>, kCta, sm);
    if (per_sm < 1) per_sm = 1;
    uint64_t grid = (uint64_t)per_sm * num_sms();
    const uint32_t nunits = (ntiles + kUnitTiles - 1) / kUnitTiles;
    if (grid > nunits) grid = nunits;
    if (grid == 0) return cudaSuccess;
    { const cudaError_t e_ = launch_pdl(k_compress<NDIM, VEC>, dim3((unsigned)grid), dim3(kCta), sm, st, a); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

template <int NDIM>
static cudaError_t launch_compress_ws(const CompressArgs& a, size_t sm, uint32_t ntiles, cudaStream_t st)
{
    cudaFuncSetAttribute(k_compress_ws<NDIM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_compress_ws<NDIM>, kWsThreads, sm);
    if (per_sm < 1) per_sm = 1;
    uint64_t grid = (uint64_t)per_sm * num_sms();
    const uint32_t nunits = (ntiles + kUnitTiles - 1) / kUnitTiles;
    if (grid > nunits) grid = nunits;
    if (grid == 0) return cudaSuccess;
    { const cudaError_t e_ = launch_pdl(k_compress_ws<NDIM>, dim3((unsigned)grid), dim3(kWsThreads), sm, st, a); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

// z-band two-pass compression applies to 3-D fields with whole tiles per plane on the vector
// path (variant bit 1024, fz_debug_set_variant, turns it off for A/B timing).
bool compress_uses_zb(const CompressArgs& a_in)
{
    CompressArgs a = a_in;
    a.exp = variant_bits();
    if (a.g.ndim != 3 || ((a.exp & (16 | 1024)) && !a.cl) || a.rescan || a.tstage == nullptr) return false;
    if (a.g.P % kTileCodes != 0 || a.g.n / a.g.P < 2) return false;
    // a slab (multi-GPU, SV 8.e) takes it when its tile range is whole planes
    const uint32_t tpp = a.g.P / kTileCodes;
    if (a.tile_begin % tpp != 0 || a.tile_end % tpp != 0 || (a.base & 3) != 0) return false;
    bool vec = false;
    plan_smem(a, vec);
    return vec;
}

cudaError_t launch_compress_zb(const CompressArgs& a_in, cudaStream_t st)
{
    CompressArgs a = a_in;
    a.dnx = make_fastdiv(a.g.nx);
    a.dP = make_fastdiv(a.g.P);
    a.sx = a.g.nx ? (uint32_t)(kTileCodes % a.g.nx) : 0u;
    a.sp = a.g.P ? (uint32_t)(kTileCodes % a.g.P) : 0u;
    bool vec = false;
    plan_smem(a, vec);
    const uint32_t H = a.g.nx + 1;
    const uint32_t hw = (H + 3) & ~3u;
    a.hwords = (hw * 4 <= 8192 && !a.cl) ? hw : 0;
    const size_t sm = sizeof(int) * ((size_t)a.qwords + 32 * 33 + 4) + sizeof(float) * (kTileCodes + (size_t)a.hwords);
    cudaFuncSetAttribute(k_compress_zb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_compress_zb, kCta, sm);
    if (per_sm < 1) per_sm = 1;
    const uint32_t tpp = a.g.P / kTileCodes, nzr = (a.tile_end - a.tile_begin) / tpp;
    const uint64_t nwork = (uint64_t)tpp * ((nzr + kZbChunk - 1) / kZbChunk);
    uint64_t grid = (uint64_t)per_sm * num_sms();
    if (grid > nwork) grid = nwork;
    LaunchProf lp(K_COMPRESS, st);
    { const cudaError_t e_ = launch_pdl(k_compress_zb, dim3((unsigned)grid), dim3(kCta), sm, st, a); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

cudaError_t launch_compact(const uint8_t* flags, const uint32_t* loc, const uint32_t* bpre, const uint4* tstage,
                           uint8_t* payload_out, uint64_t payload_cap, uint32_t ntiles, uint8_t* hdr_out,
                           uint64_t hdr_cap, const fz_shape& s, uint64_t n, uint64_t T, Ctrl* ctrl, cudaStream_t st)
{
    uint64_t d[3] = {1, 1, 1};
    for (uint32_t k = 0; k < s.ndim; ++k) d[k] = s.dims[k];
    LaunchProf lp(K_COMPACT, st);
    unsigned grid = (unsigned)((ntiles + 7) / 8);
    if (grid > (unsigned)num_sms() * 16) grid = num_sms() * 16;
    if (grid < 1) grid = 1;
    return launch_pdl(k_compact, dim3(grid), dim3(256), 0, st, reinterpret_cast<const uint32_t*>(flags), loc, bpre,
                      tstage, payload_out, payload_cap, ntiles, hdr_out, hdr_cap, s.ndim, d[0], d[1], d[2], n, T,
                      ctrl);
}

bool compress_uses_ws(const CompressArgs& a_in)
{
    CompressArgs a = a_in;
    a.exp = variant_bits();
    bool vec = false;
    plan_smem(a, vec);
    return vec && !(a.exp & 16);
}

cudaError_t launch_compress(const CompressArgs& a_in, cudaStream_t st)
{
    CompressArgs a = a_in;
    a.exp = variant_bits();
    a.dnx = make_fastdiv(a.g.nx);
    a.dP = make_fastdiv(a.g.P);
    a.sx = a.g.nx ? (uint32_t)(kTileCodes % a.g.nx) : 0u;
    a.sp = a.g.P ? (uint32_t)(kTileCodes % a.g.P) : 0u;
    bool vec = false;
    size_t sm = plan_smem(a, vec);
    const uint32_t ntiles = a.tile_end - a.tile_begin;
    LaunchProf lp(K_COMPRESS, st);
    if (vec && !(a.exp & 16)) {
        // ws kernel: q storage + shuffle buffer + payload ring + one TMA input stage
        sm = sizeof(int) * ((size_t)a.qwords + 32 * 33 + 8) + 16 * (size_t)kRingBlocks +
             2 * kTileCodes * sizeof(float);
        switch (a.g.ndim) {
            case 1: return launch_compress_ws<1>(a, sm, ntiles, st);
            case 2: return launch_compress_ws<2>(a, sm, ntiles, st);
            default: return launch_compress_ws<3>(a, sm, ntiles, st);
        }
    }
    switch (a.g.ndim * 2 + (vec ? 1 : 0)) {
        case 2: return launch_compress_t<1, false>(a, sm, ntiles, st);
        case 3: return launch_compress_t<1, true>(a, sm, ntiles, st);
        case 4: return launch_compress_t<2, false>(a, sm, ntiles, st);
        case 5: return launch_compress_t<2, true>(a, sm, ntiles, st);
        case 6: return launch_compress_t<3, false>(a, sm, ntiles, st);
        default: return launch_compress_t<3, true>(a, sm, ntiles, st);
    }
}

cudaError_t launch_init(Ctrl* ctrl, unsigned long long* status, uint2* ocnt, uint32_t ntiles,
                        const fz_params* p, cudaStream_t st, uint32_t chunk)
{
    fz_params pp{};
    if (p) pp = *p;
    unsigned grid = (unsigned)((ntiles + 255) / 256);
    if (grid < 1) grid = 1;
    if (grid > 1024) grid = 1024;
    LaunchProf lp(K_INIT, st);
    { const cudaError_t e_ = launch_pdl(k_init, dim3(grid), dim3(256), 0, st, ctrl, status, ocnt, ntiles, p ? 1 : 0, pp, chunk); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

// C0 with the field streamed through shared memory by 1-D TMA bulk copies: a persistent CTA
// owns chunks i, i + G, ... of 4096 floats; a ring of kRgStages chunks is in flight (thread 0
// issues, an mbarrier per stage completes), every thread reduces 16 floats of the chunk.
constexpr int kRgStages = 4;
constexpr uint32_t kRgChunk = 4096;   // floats per chunk (16 KB)

__global__ void __launch_bounds__(256) k_range_tma(const float* __restrict__ d, uint64_t n, Ctrl* ctrl)
{
    pdl_begin();
    extern __shared__ __align__(128) float rgs[];
    __shared__ __align__(8) uint64_t full[kRgStages];
    const int tid = threadIdx.x;
    const uint64_t nch = n / kRgChunk;   // whole chunks (the rest below)
    if (tid == 0) {
        for (int s = 0; s < kRgStages; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](uint64_t c, int s) {
        mbar_expect_tx(&full[s], kRgChunk * 4);
        tma_load_1d(rgs + (size_t)s * kRgChunk, d + c * kRgChunk, kRgChunk * 4, &full[s]);
    };
    uint64_t c = blockIdx.x;
    if (tid == 0)
        for (int s = 0; s < kRgStages; ++s)
            if (c + (uint64_t)s * gridDim.x < nch) issue(c + (uint64_t)s * gridDim.x, s);
    float lo = INFINITY, hi = -INFINITY;
    unsigned long long bad = ~0ull;
    for (uint32_t k = 0; c < nch; c += gridDim.x, ++k) {
        const int s = k % kRgStages;
        while (!mbar_try_wait(&full[s], (k / kRgStages) & 1u)) {
        }
        const float4* p = reinterpret_cast<const float4*>(rgs + (size_t)s * kRgChunk);
        bool ok = true;
#pragma unroll
        for (int u = 0; u < (int)(kRgChunk / 4 / 256); ++u) {
            const float4 v = p[tid + 256 * u];
            lo = fminf(lo, fminf(fminf(v.x, v.y), fminf(v.z, v.w)));
            hi = fmaxf(hi, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
            ok &= fabsf(v.x) <= FLT_MAX && fabsf(v.y) <= FLT_MAX && fabsf(v.z) <= FLT_MAX && fabsf(v.w) <= FLT_MAX;
        }
        if (!ok) {   // rare: the first non-finite index of this thread's elements
            for (int u = 0; u < (int)(kRgChunk / 4 / 256); ++u)
                for (int e = 0; e < 4; ++e) {
                    const uint32_t o = 4 * (tid + 256 * u) + e;
                    if (!(fabsf(rgs[(size_t)s * kRgChunk + o]) <= FLT_MAX))
                        bad = min(bad, (unsigned long long)(c * kRgChunk + o));
                }
        }
        __syncthreads();   // the stage is consumed
        if (tid == 0) {
            const uint64_t nc = c + (uint64_t)kRgStages * gridDim.x;
            if (nc < nch) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(nc, s);
            }
        }
    }
    // the tail past the whole chunks (CTA 0)
    if (blockIdx.x == 0)
        for (uint64_t j = nch * kRgChunk + tid; j < n; j += 256) {
            const float v = __ldg(d + j);
            lo = fminf(lo, v);
            hi = fmaxf(hi, v);
            if (!(fabsf(v) <= FLT_MAX)) bad = min(bad, (unsigned long long)j);
        }
    uint32_t elo = f2ord(__fadd_rn(lo, 0.0f)), ehi = f2ord(__fadd_rn(hi, 0.0f));
    if (lo == INFINITY) elo = 0xFFFFFFFFu;
    if (hi == -INFINITY) ehi = 0u;
    elo = __reduce_min_sync(kFull, elo);
    ehi = __reduce_max_sync(kFull, ehi);
    unsigned long long b = bad;
    for (int o = 16; o; o >>= 1) b = min(b, __shfl_xor_sync(kFull, b, o));
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&ctrl->mn_enc, elo);
        atomicMax(&ctrl->mx_enc, ehi);
        if (b != ~0ull) atomicMin(&ctrl->first_bad, b);
    }
}

cudaError_t launch_range(const float* d, uint64_t n, Ctrl* ctrl, cudaStream_t st)
{
    if (n >= (uint64_t)kRgChunk * 1184 && (reinterpret_cast<uintptr_t>(d) & 15) == 0 && !(variant_bits() & 1048576)) {
        const size_t sm = (size_t)kRgStages * kRgChunk * 4;
        cudaFuncSetAttribute(k_range_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        uint64_t nch = n / kRgChunk, grid = (uint64_t)num_sms() * 3;
        if (grid > nch) grid = nch;
        LaunchProf lp(K_RANGE, st);
        { const cudaError_t e_ = launch_pdl(k_range_tma, dim3((unsigned)grid), dim3(256), sm, st, d, n, ctrl); if (e_ != cudaSuccess) return e_; }
        return cudaGetLastError();
    }
    uint64_t want = (n / 4 + 255) / 256;
    uint64_t cap = (uint64_t)num_sms() * 8;
    unsigned grid = (unsigned)(want < 1 ? 1 : (want > cap ? cap : want));
    LaunchProf lp(K_RANGE, st);
    { const cudaError_t e_ = launch_pdl(k_range, dim3(grid), dim3(256), 0, st, d, n, ctrl); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

cudaError_t launch_params(Ctrl* ctrl, int mode, double eb, uint64_t n, cudaStream_t st)
{
    LaunchProf lp(K_PARAMS, st);
    { const cudaError_t e_ = launch_pdl(k_params, dim3(1), dim3(32), 0, st, ctrl, mode, eb, n); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

cudaError_t launch_finalize(uint8_t* out, uint64_t cap, const fz_shape& s, uint64_t n, uint64_t T, Ctrl* ctrl,
                            cudaStream_t st)
{
    uint64_t d[3] = {1, 1, 1};
    for (uint32_t k = 0; k < s.ndim; ++k) d[k] = s.dims[k];
    LaunchProf lp(K_FINALIZE, st);
    { const cudaError_t e_ = launch_pdl(k_finalize, dim3(1), dim3(32), 0, st, out, cap, s.ndim, d[0], d[1], d[2], n, T, ctrl); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

cudaError_t launch_outlier_scan(const uint2* ocnt, uint2* opre, uint32_t ntiles, cudaStream_t st, const Ctrl* ctrl)
{
    LaunchProf lp(K_OUTLIERS, st);
    { const cudaError_t e_ = launch_pdl(k_outlier_scan, dim3(1), dim3(1024), 0, st, ocnt, opre, ntiles, ctrl); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

cudaError_t launch_outlier_place_dev(const uint2* ocnt, const uint2* obase, const uint2* opre, uint32_t ntiles,
                                     const uint2* dstage, const uint2* vstage, uint8_t* payload_out,
                                     uint64_t payload_cap, Ctrl* ctrl, cudaStream_t st)
{
    LaunchProf lp(K_OUTLIERS, st);
    unsigned grid = (unsigned)((ntiles + 7) / 8);
    if (grid > (unsigned)num_sms() * 8) grid = num_sms() * 8;
    if (grid < 1) grid = 1;
    { const cudaError_t e_ = launch_pdl(k_outlier_place_dev, dim3(grid), dim3(256), 0, st, ocnt, obase, opre, ntiles, dstage, vstage, payload_out, payload_cap,
                                              ctrl); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

cudaError_t launch_outlier_place(const uint2* ocnt, const uint2* obase, const uint2* opre, uint32_t ntiles,
                                 const uint2* dstage, const uint2* vstage, uint2* dout, uint2* vout,
                                 uint32_t* didx, int32_t* dval, uint32_t* vidx, uint32_t* vbits, cudaStream_t st)
{
    LaunchProf lp(K_OUTLIERS, st);
    unsigned grid = (unsigned)((ntiles + 7) / 8);
    if (grid > (unsigned)num_sms() * 8) grid = num_sms() * 8;
    if (grid < 1) grid = 1;
    { const cudaError_t e_ = launch_pdl(k_outlier_place, dim3(grid), dim3(256), 0, st, ocnt, obase, opre, ntiles, dstage, vstage, dout, vout, didx, dval,
                                          vidx, vbits); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

}  // namespace fz
