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
                       int set_params, fz_params p)
{
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    for (uint32_t k = i; k < ntiles; k += gridDim.x * blockDim.x) {
        status[k] = 0ull;   // per-unit look-back words (at most one per tile)
        ocnt[k] = make_uint2(0, 0);
    }
    if (i == 0) {
        ctrl->mn_enc = 0xFFFFFFFFu;
        ctrl->mx_enc = 0u;
        ctrl->first_bad = ~0ull;
        ctrl->err = 0;
        ctrl->ticket = 0;
        ctrl->stage_overflow = 0;
        ctrl->nnz = ctrl->nd = ctrl->nv = ctrl->total = 0;
        ctrl->dcount = ctrl->vcount = 0;
        if (set_params) {
            ctrl->p = p;
            ctrl->h = 0.5f * p.w;
        }
    }
}

// ------------------------------------------------------------------------------------
// C0 range: grid-stride, 16-byte loads, warp reductions, one atomic per warp.
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_range(const float* __restrict__ d, uint64_t n, Ctrl* ctrl)
{
    uint32_t lo = 0xFFFFFFFFu, hi = 0u;
    unsigned long long bad = ~0ull;
    const uint64_t nv4 = n / 4;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    auto take = [&](float v, uint64_t idx) {
        if (!isfinite(v)) { bad = min(bad, (unsigned long long)idx); return; }
        v = __fadd_rn(v, 0.0f);   // -0.0 -> +0.0 (R18)
        uint32_t e = f2ord(v);
        lo = min(lo, e);
        hi = max(hi, e);
    };
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nv4; k += stride) {
        float4 v = ldg_f4(d + 4 * k);
        take(v.x, 4 * k); take(v.y, 4 * k + 1); take(v.z, 4 * k + 2); take(v.w, 4 * k + 3);
    }
    for (uint64_t k = 4 * nv4 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride)
        take(__ldg(d + k), k);
    lo = __reduce_min_sync(kFull, lo);
    hi = __reduce_max_sync(kFull, hi);
    unsigned long long b = bad;
    for (int o = 16; o; o >>= 1) b = min(b, __shfl_xor_sync(kFull, b, o));
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&ctrl->mn_enc, lo);
        atomicMax(&ctrl->mx_enc, hi);
        if (b != ~0ull) atomicMin(&ctrl->first_bad, b);
    }
}

__global__ void k_params(Ctrl* ctrl, int mode, double eb, uint64_t n)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (ctrl->first_bad != ~0ull) { ctrl->err = FZ_ERR_NONFINITE; return; }
    float mn = n ? ord2f(ctrl->mn_enc) : 0.0f;
    float mx = n ? ord2f(ctrl->mx_enc) : 0.0f;
    fz_params p;
    int st = derive_params(mn, mx, mode, eb, &p);
    if (st != FZ_OK) { ctrl->err = st; return; }
    ctrl->p = p;
    ctrl->h = 0.5f * p.w;
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

// q of one halo element (no bound check needed: only own elements can be value outliers).
template <bool FB>
__device__ __forceinline__ int quant_q(float d, const QuantP& P)
{
    if (FB) return prequant_q(d, P);
    bool hard;
    float qf;
    int q = prequant_fast(d, P, hard, qf);
    if (hard) q = prequant_q(d, P);
    return q;
}

// Cooperative fill of arr[pad(g - g_lo)] = q(g) for g in [g_lo, g_lo + len), in 4-element
// aligned chunks (16-byte loads).  Elements outside the field get q = 0 (masked later).
template <bool FB>
__device__ __forceinline__ void fill_range(const CompressArgs& a, const QuantP& P, int* arr,
                                           int64_t g_lo, int len)
{
    if (len <= 0) return;
    const int64_t a0 = g_lo & ~(int64_t)3;
    const int nch = (int)((g_lo + len - a0 + 3) >> 2);
    for (int c = threadIdx.x; c < nch; c += kCta) {
        const int64_t gc = a0 + 4 * c;
        float v[4];
        loadk<4>(a, gc, v);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t m = gc + u - g_lo;
            if (m >= 0 && m < len) arr[pad((int)m)] = quant_q<FB>(v[u], P);
        }
    }
}

// ------------------------------------------------------------------------------------
// The fused compression kernel.  One CTA of 256 threads; thread t owns the elements
// 8t..8t+7 of the current tile (= words 4t..4t+3 = A[t/8][4(t%8)..+3]).
// Scan granularity: a "unit" of kUnitTiles consecutive tiles.  The CTA compacts each tile's
// nonzero blocks into a shared stage (double-buffered per unit), publishes the unit's block
// count once its last tile is done, and resolves the unit's global offset by a wide
// decoupled look-back one tile later (while computing the next unit's first tile), then
// copies the stage to the payload with coalesced 16-byte stores.
// ------------------------------------------------------------------------------------
constexpr int kUnitTiles = 4;

template <int NDIM, bool FB>
__device__ __forceinline__ void compress_body(const CompressArgs& a)
{
    extern __shared__ int smem[];
    __shared__ uint32_t s_unit[2];
    __shared__ uint32_t s_F[8];
    __shared__ uint32_t s_cd[8], s_cv[8];
    __shared__ unsigned long long s_off;
    __shared__ unsigned long long s_ob[2];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    Ctrl* ctrl = a.ctrl;
    if (ctrl->err != 0) return;
    QuantP P;
    P.w = ctrl->p.w; P.r = ctrl->p.r; P.h = ctrl->h; P.eb32 = ctrl->p.eb32;
    const uint32_t n = a.g.n, nx = a.g.nx, PL = a.g.P;
    const int qs = (int)a.qstride;
    // neighbour streams: array base (words) and m offset of own element j = 0
    int ab[4], mo[4];
    int narr;
    if (NDIM == 1) {
        ab[0] = 0; mo[0] = 1; narr = 1;
    } else if (a.union_mode) {
        const int HA = (int)nx + 1;
        ab[0] = 0; mo[0] = HA; ab[1] = 0; mo[1] = 1;
        ab[2] = qs; mo[2] = HA; ab[3] = qs; mo[3] = 1;
        narr = NDIM == 3 ? 2 : 1;
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) { ab[k] = k * qs; mo[k] = 1; }
        narr = NDIM == 3 ? 4 : 2;
    }
    uint32_t* Obuf = reinterpret_cast<uint32_t*>(smem + narr * qs);              // 32 x 33
    uint4* stage = reinterpret_cast<uint4*>(smem + narr * qs + 32 * 33 + 3);     // 2 x units
    stage = reinterpret_cast<uint4*>((reinterpret_cast<uintptr_t>(stage) + 15) & ~uintptr_t(15));
    constexpr int kStageBlocks = kUnitTiles * kTileBlocks;

    const uint32_t nunits = (a.tile_end - a.tile_begin + kUnitTiles - 1) / kUnitTiles;
    constexpr uint32_t NONE = 0xFFFFFFFFu;
    if (tid == 0) s_unit[0] = atomicAdd(&ctrl->ticket, 1u);
    __syncthreads();
    uint32_t pu = NONE;       // pending unit: aggregate published, offset unknown
    uint32_t pcnt = 0;        // its block count
    int buf = 0;              // stage buffer of the current unit
    for (int it = 0;; ++it) {
        const uint32_t u = s_unit[it & 1];
        const bool work = u < nunits;
        if (!work && pu == NONE) break;
        if (!work) {
            // ---- flush the last pending unit ----
            if (warp == 0) {
                unsigned long long ex = 0;
                if (pu != 0) {
                    ex = lookback_wide<8, false>(a.status, pu, 0, kStAgg - 1, &ctrl->err);
                    if (lane == 0) st_relaxed_u64(&a.status[pu], kStInc | (ex + pcnt));
                }
                if (lane == 0) s_off = ex;
            }
            __syncthreads();
            const uint4* ps = stage + (buf ^ 1) * kStageBlocks;
            for (uint32_t i = tid; i < pcnt; i += kCta) {
                const uint64_t bo = 16 * (s_off + i);
                if (bo + 16 <= a.payload_cap) *reinterpret_cast<uint4*>(a.payload_out + bo) = ps[i];
            }
            if (tid == 0 && pu == nunits - 1) ctrl->nnz = s_off + pcnt;
            break;
        }
        const uint32_t t_first = a.tile_begin + u * kUnitTiles;
        const uint32_t t_last = min(a.tile_end, t_first + kUnitTiles);
        uint32_t cnt = 0;                         // blocks staged for this unit (uniform)
        uint4* st = stage + buf * kStageBlocks;
        for (uint32_t t = t_first; t < t_last; ++t) {
            const int64_t s = (int64_t)t * kTileCodes;
            const uint32_t g0 = (uint32_t)s + 8u * tid;
            const bool full = s + kTileCodes <= (int64_t)n;

            // ---- A: prequantize own elements (+ bound check) and the halo ranges ----
            float dv[8];
            int qo[8];
            uint32_t vmask = 0;
            loadk<8>(a, (int64_t)g0, dv);
            if (NDIM == 1 || !a.union_mode) {
                if (tid == 0) smem[pad(0)] = quant_q<FB>(load1(a, s - 1), P);
                if (NDIM >= 2) fill_range<FB>(a, P, smem + ab[1], s - (int64_t)nx - 1, kTileCodes + 1);
                if (NDIM == 3) {
                    fill_range<FB>(a, P, smem + ab[2], s - (int64_t)PL - 1, kTileCodes + 1);
                    fill_range<FB>(a, P, smem + ab[3], s - (int64_t)PL - nx - 1, kTileCodes + 1);
                }
            } else {
                fill_range<FB>(a, P, smem, s - (int64_t)nx - 1, (int)nx + 1);
                if (NDIM == 3) fill_range<FB>(a, P, smem + qs, s - (int64_t)PL - nx - 1, kTileCodes + (int)nx + 1);
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                bool vo;
                if (FB) {
                    qo[e] = prequant(dv[e], P, vo);
                } else {
                    bool hard;
                    float qf;
                    qo[e] = prequant_fast(dv[e], P, hard, qf);
                    if (hard) {
                        qo[e] = prequant(dv[e], P, vo);
                    } else {
                        vo = fabsf(__fsub_rn(__fmul_rn(qf, P.w), dv[e])) > P.eb32;
                    }
                }
                if (vo) vmask |= 1u << e;
                smem[ab[0] + pad(mo[0] + 8 * tid + e)] = qo[e];
            }
            if (!full) vmask &= (g0 >= n) ? 0u : ((n - g0 >= 8) ? 0xFFu : ((1u << (n - g0)) - 1u));
            __syncthreads();
            if (t == t_first && tid == 0) {
                const uint32_t nu = atomicAdd(&ctrl->ticket, 1u);
                s_unit[(it & 1) ^ 1] = nu;
                // TMA L2 prefetch of the next unit's input (~kUnitTiles tiles ahead): keeps
                // HBM busy independently of how many loads the registers can hold
                if (nu < nunits) prefetch_l2_range(a, (uint64_t)(a.tile_begin + nu * kUnitTiles) * kTileCodes,
                                                   (uint64_t)kUnitTiles * kTileCodes);
            }

            // ---- B: Lorenzo residual (C2) as delta(e) = S(e+1) - [x>0] S(e), where S(j)
            // combines the element at j-1 with its y-1, z-1, (y-1,z-1) neighbours ----
            int S[9];
            bool fast_yz = true;
            uint32_t xmask = 0xFFu;
            if (NDIM == 1) {
                S[0] = smem[ab[0] + pad(mo[0] + 8 * tid - 1)];
#pragma unroll
                for (int j = 1; j < 9; ++j) S[j] = qo[j - 1];
                if (nx >= 8) {
                    const uint32_t x0 = fmod_(g0, a.dnx);
                    const uint32_t us = x0 == 0 ? 0u : nx - x0;
                    if (us < 8) xmask &= ~(1u << us);
                } else {
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        if (fmod_(g0 + e, a.dnx) == 0) xmask &= ~(1u << e);
                }
            } else {
                int qy[9], qz[9], qyz[9];
                const int o0 = ab[0] + pad(mo[0] + 8 * tid - 1);
                const int own0 = smem[o0];
#pragma unroll
                for (int j = 0; j < 9; ++j) qy[j] = smem[ab[1] + pad(mo[1] + 8 * tid - 1 + j)];
                if (NDIM == 3) {
#pragma unroll
                    for (int j = 0; j < 9; ++j) {
                        qz[j] = smem[ab[2] + pad(mo[2] + 8 * tid - 1 + j)];
                        qyz[j] = smem[ab[3] + pad(mo[3] + 8 * tid - 1 + j)];
                    }
                }
                uint32_t ymask = 0xFFu, zmask = 0xFFu;   // bit e: neighbour exists for element e
                if (nx >= 8) {
                    const uint32_t x0 = fmod_(g0, a.dnx);
                    const uint32_t us = x0 == 0 ? 0u : nx - x0;
                    if (us < 8) xmask &= ~(1u << us);
                    const uint32_t p0 = fmod_(g0, a.dP);
                    fast_yz = p0 >= nx && p0 + 7 < PL && (NDIM == 2 || g0 >= PL);
                    if (!fast_yz) {
                        uint32_t pp = p0;
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            if (pp < nx) ymask &= ~(1u << e);
                            if (g0 + e < PL) zmask &= ~(1u << e);
                            if (++pp == PL) pp = 0;
                        }
                    }
                } else {
                    fast_yz = false;
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        if (fmod_(g0 + e, a.dnx) == 0) xmask &= ~(1u << e);
                        if (fmod_(g0 + e, a.dP) < nx) ymask &= ~(1u << e);
                        if (g0 + e < PL) zmask &= ~(1u << e);
                    }
                }
                if (NDIM == 2) zmask = 0;
                if (fast_yz) {
                    S[0] = (int)((uint32_t)own0 - (uint32_t)qy[0] - (NDIM == 3 ? (uint32_t)qz[0] - (uint32_t)qyz[0] : 0u));
#pragma unroll
                    for (int j = 1; j < 9; ++j)
                        S[j] = (int)((uint32_t)qo[j - 1] - (uint32_t)qy[j] -
                                     (NDIM == 3 ? (uint32_t)qz[j] - (uint32_t)qyz[j] : 0u));
                } else {
                    // masks of element j-1 for S(j); of element 0 for S(0)
#pragma unroll
                    for (int j = 0; j < 9; ++j) {
                        const int e = j == 0 ? 0 : j - 1;
                        const uint32_t Y = (ymask >> e) & 1u ? 0xFFFFFFFFu : 0u;
                        const uint32_t Z = (zmask >> e) & 1u ? 0xFFFFFFFFu : 0u;
                        const uint32_t ow = j == 0 ? (uint32_t)own0 : (uint32_t)qo[j - 1];
                        uint32_t v = ow - ((uint32_t)qy[j] & Y);
                        if (NDIM == 3) v -= ((uint32_t)qz[j] - ((uint32_t)qyz[j] & Y)) & Z;
                        S[j] = (int)v;
                    }
                }
            }
            // ---- C3 codes, C4 words ----
            uint32_t code[8];
            int32_t dl[8];
            uint32_t dmask = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const uint32_t X = (xmask >> e) & 1u ? 0xFFFFFFFFu : 0u;
                const uint32_t dd = (uint32_t)S[e + 1] - ((uint32_t)S[e] & X);
                const int32_t di = (int32_t)dd;
                const uint32_t mag = (uint32_t)abs(di);
                const bool outl = mag > 32767u;
                code[e] = outl ? 0u : (((dd >> 16) & 0x8000u) | mag);
                dl[e] = di;
                if (outl) dmask |= 1u << e;
            }
            if (!full) {
                const uint32_t vm = (g0 >= n) ? 0u : ((n - g0 >= 8) ? 0xFFu : ((1u << (n - g0)) - 1u));
                dmask &= vm;
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
                // ---- C5 bitshuffle in registers: row c = tid/8 of A, lanes k = tid%8 ----
                uint32_t w4[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) w4[i] = __byte_perm(code[2 * i], code[2 * i + 1], 0x5410);
                transpose32_group8(w4, lane & 7);
                const int c = tid >> 3, kk = tid & 7;
#pragma unroll
                for (int i = 0; i < 4; ++i) Obuf[(4 * kk + i) * 33 + c] = w4[i];
            }
            const int any_out = __syncthreads_or((dmask | vmask) != 0);

            // ---- outlier records (rare; R7, R20): ascending element index ----
            if (any_out) {
                const int cd = __popc(dmask), cv = __popc(vmask);
                const int wd = __reduce_add_sync(kFull, cd), wv = __reduce_add_sync(kFull, cv);
                if (lane == 0) { s_cd[warp] = wd; s_cv[warp] = wv; }
                __syncthreads();
                uint32_t tnd = 0, tnv = 0, wpre_d = 0, wpre_v = 0;
#pragma unroll
                for (int w = 0; w < 8; ++w) {
                    tnd += s_cd[w]; tnv += s_cv[w];
                    if (w < warp) { wpre_d += s_cd[w]; wpre_v += s_cv[w]; }
                }
                if (tid == 0) {
                    if (a.rescan) {
                        const uint2 o = a.opre[t];
                        s_ob[0] = o.x; s_ob[1] = o.y;
                    } else {
                        s_ob[0] = tnd ? atomicAdd(&ctrl->dcount, (unsigned long long)tnd) : 0ull;
                        s_ob[1] = tnv ? atomicAdd(&ctrl->vcount, (unsigned long long)tnv) : 0ull;
                        a.ocnt[t] = make_uint2(tnd, tnv);
                        a.obase[t] = make_uint2((uint32_t)s_ob[0], (uint32_t)s_ob[1]);
                    }
                }
                int id = cd, iv = cv;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int yd = __shfl_up_sync(kFull, id, o), yv = __shfl_up_sync(kFull, iv, o);
                    if (lane >= o) { id += yd; iv += yv; }
                }
                __syncthreads();
                uint64_t pd = s_ob[0] + wpre_d + (id - cd), pv = s_ob[1] + wpre_v + (iv - cv);
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
            if (a.rescan) continue;

            // ---- C6 block flags: thread b owns block b = 8r + x of the shuffled tile ----
            const uint32_t* row = Obuf + (tid >> 3) * 33 + 4 * (tid & 7);
            const uint4 blk = make_uint4(row[0], row[1], row[2], row[3]);
            const bool nz = (blk.x | blk.y | blk.z | blk.w) != 0;
            const uint32_t F = __ballot_sync(kFull, nz);
            if (lane == 0) s_F[warp] = F;
            // the pending unit's look-back overlaps the other warps' flag work
            if (t == t_first && pu != NONE && warp == 0) {
                unsigned long long ex = 0;
                if (pu != 0) {
                    ex = lookback_wide<8, false>(a.status, pu, 0, kStAgg - 1, &ctrl->err);
                    if (lane == 0) st_relaxed_u64(&a.status[pu], kStInc | (ex + pcnt));
                }
                if (lane == 0) s_off = ex;
            }
            __syncthreads();
            uint32_t tn = 0, wpre = 0;
#pragma unroll
            for (int w = 0; w < 8; ++w) {
                const uint32_t pc = __popc(s_F[w]);
                tn += pc;
                if (w < warp) wpre += pc;
            }
            if (tid < 8) {
                const uint64_t fo = (uint64_t)(t - a.tile_begin) * 32 + 4 * tid;
                if (fo + 4 <= a.flags_cap) *reinterpret_cast<uint32_t*>(a.flags_out + fo) = s_F[tid];
            }
            // ---- C8 (local): compact the tile's nonzero blocks into the unit stage ----
            if (nz) st[cnt + wpre + __popc(F & ((1u << lane) - 1u))] = blk;
            cnt += tn;
            if (t == t_first && pu != NONE) {
                // ---- C8 (global): the pending unit's stage goes to its final offset ----
                const uint4* ps = stage + (buf ^ 1) * kStageBlocks;
                const unsigned long long off = s_off;
                for (uint32_t i = tid; i < pcnt; i += kCta) {
                    const uint64_t bo = 16 * (off + i);
                    if (bo + 16 <= a.payload_cap) *reinterpret_cast<uint4*>(a.payload_out + bo) = ps[i];
                }
                if (tid == 0 && pu == nunits - 1) ctrl->nnz = off + pcnt;
                pu = NONE;
            }
        }
        if (a.rescan) {
            __syncthreads();
            continue;
        }
        // ---- C7: publish the unit's aggregate (inclusive for unit 0) ----
        if (tid == 0) st_relaxed_u64(&a.status[u], (u == 0 ? kStInc : kStAgg) | cnt);
        pu = u;
        pcnt = cnt;
        buf ^= 1;
        __syncthreads();
    }
}

// The margin/fallback mode (R2) is known only on the device when fz_compress derives the
// parameters there, so the kernel dispatches on it (block-uniform branch).
template <int NDIM>
__global__ void __launch_bounds__(kCta, 2) k_compress(CompressArgs a)
{
    if (a.ctrl->p.fallback) compress_body<NDIM, true>(a);
    else compress_body<NDIM, false>(a);
}

// ------------------------------------------------------------------------------------
// C9: header (outlier sections are placed by k_outlier_place when there are any).
// ------------------------------------------------------------------------------------
__global__ void k_finalize(uint8_t* out, uint64_t out_cap, uint32_t ndim, uint64_t d0, uint64_t d1,
                           uint64_t d2, uint64_t n, uint64_t T, Ctrl* ctrl)
{
    if (ctrl->err != 0 || threadIdx.x != 0) return;
    const uint64_t nnz = ctrl->nnz, nd = ctrl->dcount, nv = ctrl->vcount;
    const uint64_t total = kHeaderBytes + 32 * T + 16 * nnz + 8 * nd + 8 * nv;
    ctrl->nd = nd;
    ctrl->nv = nv;
    ctrl->total = total;
    if (total > out_cap || out == nullptr) return;
    const fz_params& p = ctrl->p;
    uint8_t h[128];
    for (int i = 0; i < 128; ++i) h[i] = 0;
    h[0] = 'F'; h[1] = 'Z'; h[2] = 'B'; h[3] = '2';
    const uint16_t ver = 1, fl = (uint16_t)((p.mode == FZ_EB_REL ? 1u : 0u) | (p.fallback ? 2u : 0u));
    memcpy(h + 4, &ver, 2);
    memcpy(h + 6, &fl, 2);
    h[8] = (uint8_t)ndim;
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

// Exclusive scan of the per-tile outlier counts (one block; only when outliers exist).
__global__ void __launch_bounds__(1024) k_outlier_scan(const uint2* ocnt, uint2* opre, uint32_t ntiles)
{
    __shared__ uint32_t wd[32], wv[32];
    __shared__ uint32_t carry_d, carry_v;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
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

// Shared q arrays for a shape: fills a.union_mode / a.qstride; returns dynamic smem bytes.
static size_t plan_smem(CompressArgs& a)
{
    const uint32_t ndim = a.g.ndim;
    uint32_t narr, len;
    if (ndim == 1) {
        narr = 1;
        len = kTileCodes + 1;
        a.union_mode = 0;
    } else if (a.g.nx + 1 <= kUnionHaloMax) {
        a.union_mode = 1;
        narr = ndim == 3 ? 2 : 1;
        len = kTileCodes + a.g.nx + 1;
    } else {
        a.union_mode = 0;
        narr = ndim == 3 ? 4 : 2;
        len = kTileCodes + 1;
    }
    a.qstride = (pad_words(len) + 31) & ~31u;
    return sizeof(int) * ((size_t)narr * a.qstride + 32 * 33 + 8) + 2 * 16 * (size_t)kUnitTiles * kTileBlocks;
}

template <int NDIM>
static cudaError_t launch_compress_t(const CompressArgs& a, size_t sm, uint32_t ntiles, cudaStream_t st)
{
    cudaFuncSetAttribute(k_compress<NDIM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_compress<NDIM>, kCta, sm);
    if (per_sm < 1) per_sm = 1;
    uint64_t grid = (uint64_t)per_sm * num_sms();
    const uint32_t nunits = (ntiles + kUnitTiles - 1) / kUnitTiles;
    if (grid > nunits) grid = nunits;
    if (grid == 0) return cudaSuccess;
    k_compress<NDIM><<<(unsigned)grid, kCta, sm, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_compress(const CompressArgs& a_in, cudaStream_t st)
{
    CompressArgs a = a_in;
    a.dnx = make_fastdiv(a.g.nx);
    a.dP = make_fastdiv(a.g.P);
    const size_t sm = plan_smem(a);
    const uint32_t ntiles = a.tile_end - a.tile_begin;
    LaunchProf lp(K_COMPRESS, st);
    switch (a.g.ndim) {
        case 1: return launch_compress_t<1>(a, sm, ntiles, st);
        case 2: return launch_compress_t<2>(a, sm, ntiles, st);
        default: return launch_compress_t<3>(a, sm, ntiles, st);
    }
}

cudaError_t launch_init(Ctrl* ctrl, unsigned long long* status, uint2* ocnt, uint32_t ntiles,
                        const fz_params* p, cudaStream_t st)
{
    fz_params pp{};
    if (p) pp = *p;
    unsigned grid = (unsigned)((ntiles + 255) / 256);
    if (grid < 1) grid = 1;
    if (grid > 1024) grid = 1024;
    LaunchProf lp(K_INIT, st);
    k_init<<<grid, 256, 0, st>>>(ctrl, status, ocnt, ntiles, p ? 1 : 0, pp);
    return cudaGetLastError();
}

cudaError_t launch_range(const float* d, uint64_t n, Ctrl* ctrl, cudaStream_t st)
{
    uint64_t want = (n / 4 + 255) / 256;
    uint64_t cap = (uint64_t)num_sms() * 8;
    unsigned grid = (unsigned)(want < 1 ? 1 : (want > cap ? cap : want));
    LaunchProf lp(K_RANGE, st);
    k_range<<<grid, 256, 0, st>>>(d, n, ctrl);
    return cudaGetLastError();
}

cudaError_t launch_params(Ctrl* ctrl, int mode, double eb, uint64_t n, cudaStream_t st)
{
    LaunchProf lp(K_PARAMS, st);
    k_params<<<1, 32, 0, st>>>(ctrl, mode, eb, n);
    return cudaGetLastError();
}

cudaError_t launch_finalize(uint8_t* out, uint64_t cap, const fz_shape& s, uint64_t n, uint64_t T, Ctrl* ctrl,
                            cudaStream_t st)
{
    uint64_t d[3] = {1, 1, 1};
    for (uint32_t k = 0; k < s.ndim; ++k) d[k] = s.dims[k];
    LaunchProf lp(K_FINALIZE, st);
    k_finalize<<<1, 32, 0, st>>>(out, cap, s.ndim, d[0], d[1], d[2], n, T, ctrl);
    return cudaGetLastError();
}

cudaError_t launch_outlier_scan(const uint2* ocnt, uint2* opre, uint32_t ntiles, cudaStream_t st)
{
    LaunchProf lp(K_OUTLIERS, st);
    k_outlier_scan<<<1, 1024, 0, st>>>(ocnt, opre, ntiles);
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
    k_outlier_place<<<grid, 256, 0, st>>>(ocnt, obase, opre, ntiles, dstage, vstage, dout, vout, didx, dval,
                                          vidx, vbits);
    return cudaGetLastError();
}

}  // namespace fz
