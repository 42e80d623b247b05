// fz_compress.cu -- compression kernels of libfz (B200, sm_100a).
//
//   k_init      reset the control block / tile status words (and optionally set params)
//   k_range     C0: min, max, first non-finite index
//   k_params    C0: Appendix-A parameters on the device (no host round trip)
//   k_compress  C1-C8 fused: prequantize -> Lorenzo -> codes -> bitshuffle -> block flags ->
//               decoupled look-back scan -> compaction, persistent CTAs with a tile ticket
//   k_finalize  C9: header + outlier sections
//
// Citation key: P:n = PAPER.md line n; R# = DESIGN.md §3 readings; SV = SURVEY.md.
#include "fz_internal.cuh"
#include "fz_launch.h"

namespace fz {

// Q arrays hold q of 2049 consecutive elements; index m stored at m + (m >> 3) so that the
// stride-8 per-thread access pattern is bank-conflict free.
constexpr int kQStride = 2312;
__device__ __forceinline__ int qaddr(int m) { return m + (m >> 3); }

// ------------------------------------------------------------------------------------
__global__ void k_init(Ctrl* ctrl, unsigned long long* status, uint32_t ntiles, int set_params,
                       fz_params p)
{
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    for (uint32_t k = i; k < ntiles; k += gridDim.x * blockDim.x) status[k] = 0ull;
    if (i == 0) {
        ctrl->mn_enc = 0xFFFFFFFFu;
        ctrl->mx_enc = 0u;
        ctrl->first_bad = ~0ull;
        ctrl->err = 0;
        ctrl->ticket = 0;
        ctrl->ticket2 = 0;
        ctrl->stage_overflow = 0;
        ctrl->nnz = ctrl->nd = ctrl->nv = ctrl->total = 0;
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
// Loads 8 consecutive elements g0..g0+7 (g0 may be negative: zero outside the field).
// ------------------------------------------------------------------------------------
__device__ __forceinline__ void load8(const CompressArgs& a, int64_t g0, float (&v)[8])
{
    const int64_t n = a.g.n;
    const int64_t base = (int64_t)a.base;
    if (g0 >= base && g0 + 8 <= n && ((g0 - base) & 3) == 0) {
        const float* p = a.field + (g0 - base);
        float4 x = ldg_f4(p), y = ldg_f4(p + 4);
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
        v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
    } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            int64_t g = g0 + u;
            v[u] = (g >= base && g < n) ? __ldg(a.field + (g - base)) : 0.0f;
        }
    }
}

__device__ __forceinline__ float load1(const CompressArgs& a, int64_t g)
{
    return (g >= (int64_t)a.base && g < (int64_t)a.g.n) ? __ldg(a.field + (g - (int64_t)a.base)) : 0.0f;
}

// ------------------------------------------------------------------------------------
// Decoupled look-back over tiles (C7): status word = state(2) | nnz(30) | nd(32),
// value-outlier counts in companion arrays written before the release of the status word.
// Returns the exclusive prefix (nnz, nd, nv) of tile t.  Warp-wide call.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ void lookback3(const CompressArgs& a, uint32_t t, uint32_t nnz,
                                          uint32_t nd, uint32_t nv, unsigned long long& e_nnz,
                                          unsigned long long& e_nd, unsigned long long& e_nv)
{
    const int lane = threadIdx.x & 31;
    const unsigned long long kAgg = 1ull << 62, kInc = 2ull << 62;
    e_nnz = e_nd = e_nv = 0;
    if (t == a.tile_begin) {
        if (lane == 0) {
            a.inclv[t] = nv;
            st_release_u64(&a.status[t], kInc | ((unsigned long long)nnz << 32) | nd);
        }
        return;
    }
    if (lane == 0) {
        a.aggv[t] = nv;
        st_release_u64(&a.status[t], kAgg | ((unsigned long long)nnz << 32) | nd);
    }
    int64_t p = (int64_t)t - 1;
    while (true) {
        const int64_t q = p - lane;
        unsigned long long s = kInc;
        uint32_t v = 0;
        if (q >= (int64_t)a.tile_begin) {
            do { s = ld_acquire_u64(&a.status[q]); } while ((s >> 62) == 0);
            v = ((s >> 62) == 1) ? ld_relaxed_u32(&a.aggv[q]) : ld_relaxed_u32(&a.inclv[q]);
        }
        const uint32_t incl = __ballot_sync(kFull, (s >> 62) == 2);
        const int stop = incl ? __ffs(incl) - 1 : 31;
        unsigned long long cn = 0, cd = 0, cv = 0;
        if (lane <= stop) { cn = (s >> 32) & 0x3FFFFFFFull; cd = s & 0xFFFFFFFFull; cv = v; }
        for (int o = 16; o; o >>= 1) {
            cn += __shfl_xor_sync(kFull, cn, o);
            cd += __shfl_xor_sync(kFull, cd, o);
            cv += __shfl_xor_sync(kFull, cv, o);
        }
        e_nnz += cn; e_nd += cd; e_nv += cv;
        if (incl) break;
        p -= 32;
    }
    if (lane == 0) {
        a.inclv[t] = (uint32_t)(e_nv + nv);
        st_release_u64(&a.status[t], kInc | ((e_nnz + nnz) << 32) | (uint32_t)(e_nd + nd));
    }
}

// ------------------------------------------------------------------------------------
// The fused compression kernel.  One CTA of 256 threads works on one 2048-code tile at a
// time; thread t owns tile elements 8t..8t+7 (= words 4t..4t+3 = A[t/8][4(t%8)..+3]).
// ------------------------------------------------------------------------------------
template <int NDIM>
__global__ void __launch_bounds__(kCta) k_compress(CompressArgs a)
{
    constexpr int NQ = NDIM == 1 ? 1 : (NDIM == 2 ? 2 : 4);
    extern __shared__ int smem[];
    int* Q = smem;                                          // NQ x kQStride
    uint32_t* Obuf = reinterpret_cast<uint32_t*>(smem + NQ * kQStride);   // 32 x 33
    __shared__ uint32_t s_tile[2];
    __shared__ uint32_t s_F[8], s_cd[8], s_cv[8];
    __shared__ unsigned long long s_ex[3];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    Ctrl* ctrl = a.ctrl;
    if (ctrl->err != 0) return;
    QuantP P;
    P.w = ctrl->p.w; P.r = ctrl->p.r; P.h = ctrl->h; P.eb32 = ctrl->p.eb32;
    const uint32_t n = a.g.n, nx = a.g.nx, PL = a.g.P;
    // neighbour offsets of the Q ranges: own, y-1, z-1, y-1 & z-1
    const int64_t off[4] = {0, (int64_t)nx, (int64_t)PL, (int64_t)PL + nx};

    if (tid == 0) s_tile[0] = a.tile_begin + atomicAdd(&ctrl->ticket, 1u);
    __syncthreads();
    for (int it = 0;; ++it) {
        const uint32_t t = s_tile[it & 1];
        if (t >= a.tile_end) break;
        const int64_t s = (int64_t)t * kTileCodes;
        const int64_t g0 = s + 8 * tid;

        // ---- A: prequantize own elements (with bound check) and the halo ranges ----
        float dv[8];
        int qo[8];
        uint32_t vmask = 0;
        load8(a, g0, dv);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            bool vo;
            qo[u] = prequant(dv[u], P, vo);
            if (vo && g0 + u < (int64_t)n) vmask |= 1u << u;
            Q[qaddr(1 + 8 * tid + u)] = qo[u];
        }
        if (tid == 0) Q[qaddr(0)] = prequant_q(load1(a, s - 1), P);
#pragma unroll
        for (int k = 1; k < NQ; ++k) {
            float hv[8];
            load8(a, g0 - off[k], hv);
#pragma unroll
            for (int u = 0; u < 8; ++u) Q[k * kQStride + qaddr(1 + 8 * tid + u)] = prequant_q(hv[u], P);
            if (tid == 0) Q[k * kQStride + qaddr(0)] = prequant_q(load1(a, s - off[k] - 1), P);
        }
        __syncthreads();
        if (tid == 0) s_tile[(it + 1) & 1] = a.tile_begin + atomicAdd(&ctrl->ticket, 1u);

        // ---- B: Lorenzo residual (C2), codes (C3), words (C4) ----
        uint32_t x = (uint32_t)(g0 % nx), pp = (uint32_t)(g0 % PL);
        int qn[NQ][9];
        qn[0][0] = Q[qaddr(8 * tid)];
#pragma unroll
        for (int u = 0; u < 8; ++u) qn[0][u + 1] = qo[u];
#pragma unroll
        for (int k = 1; k < NQ; ++k)
#pragma unroll
            for (int u = 0; u < 9; ++u) qn[k][u] = Q[k * kQStride + qaddr(8 * tid + u)];
        uint32_t code[8];
        int32_t dl[8];
        uint32_t dmask = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const bool mx = x != 0, my = pp >= nx, mz = (g0 + u) >= (int64_t)PL;
            uint32_t r0 = (uint32_t)qn[0][u + 1] - (mx ? (uint32_t)qn[0][u] : 0u);
            uint32_t dd = r0;
            if (NDIM >= 2) {
                uint32_t r1 = (uint32_t)qn[1][u + 1] - (mx ? (uint32_t)qn[1][u] : 0u);
                if (NDIM == 3) {
                    uint32_t r2 = (uint32_t)qn[2][u + 1] - (mx ? (uint32_t)qn[2][u] : 0u);
                    uint32_t r3 = (uint32_t)qn[3][u + 1] - (mx ? (uint32_t)qn[3][u] : 0u);
                    dd -= my ? r1 : 0u;
                    dd -= mz ? (r2 - (my ? r3 : 0u)) : 0u;
                } else {
                    dd -= my ? r1 : 0u;
                }
            }
            const bool valid = (g0 + u) < (int64_t)n;
            const int32_t di = (int32_t)dd;
            const uint32_t mag = di < 0 ? (0u - dd) : dd;
            const bool out = valid && mag > 32767u;
            code[u] = (valid && !out) ? ((di < 0 ? 0x8000u : 0u) | mag) : 0u;
            dl[u] = di;
            if (out) dmask |= 1u << u;
            if (++x == nx) x = 0;
            if (++pp == PL) pp = 0;
        }
        if (a.codes_out != nullptr) {
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (g0 + u < (int64_t)n) a.codes_out[g0 + u] = (uint16_t)code[u];
        }
        const int cd = __popc(dmask), cv = __popc(vmask);
        const int wd = __reduce_add_sync(kFull, cd), wv = __reduce_add_sync(kFull, cv);

        if (!a.rescan) {
            // ---- C: bitshuffle (C5) in registers: row c = tid/8, lanes k = tid%8 ----
            uint32_t w4[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) w4[i] = code[2 * i] | (code[2 * i + 1] << 16);
            transpose32_group8(w4, lane & 7);
            const int c = tid >> 3, kk = tid & 7;
#pragma unroll
            for (int i = 0; i < 4; ++i) Obuf[(4 * kk + i) * 33 + c] = w4[i];
        }
        if (lane == 0) { s_cd[warp] = wd; s_cv[warp] = wv; }
        __syncthreads();

        // ---- D: block flags (C6): thread b owns block b = 8r + x ----
        uint4 blk = make_uint4(0, 0, 0, 0);
        uint32_t F = 0;
        bool nz = false;
        if (!a.rescan) {
            const int r = tid >> 3, xb = tid & 7;
            const uint32_t* row = Obuf + r * 33 + 4 * xb;
            blk = make_uint4(row[0], row[1], row[2], row[3]);
            nz = (blk.x | blk.y | blk.z | blk.w) != 0;
            F = __ballot_sync(kFull, nz);
            if (lane == 0) s_F[warp] = F;
        }
        __syncthreads();

        // ---- E: exclusive scan over tiles (C7) ----
        uint32_t tnd = 0, tnv = 0, wpre_d = 0, wpre_v = 0, tnnz = 0, wpre_n = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            tnd += s_cd[w]; tnv += s_cv[w];
            if (w < warp) { wpre_d += s_cd[w]; wpre_v += s_cv[w]; }
            if (!a.rescan) {
                const uint32_t pc = __popc(s_F[w]);
                tnnz += pc;
                if (w < warp) wpre_n += pc;
            }
        }
        if (!a.rescan) {
            if (warp == 0) {
                unsigned long long en, ed, ev;
                lookback3(a, t, tnnz, tnd, tnv, en, ed, ev);
                if (lane == 0) {
                    s_ex[0] = en; s_ex[1] = ed; s_ex[2] = ev;
                    a.tpre[t] = make_uint2((uint32_t)ed, (uint32_t)ev);
                    if (t == a.tile_end - 1) {
                        ctrl->nnz = en + tnnz;
                        ctrl->nd = ed + tnd;
                        ctrl->nv = ev + tnv;
                    }
                }
            }
            if (tid < 8) {
                const uint64_t fo = (uint64_t)(t - a.tile_begin) * 32 + 4 * tid;
                if (fo + 4 <= a.flags_cap) *reinterpret_cast<uint32_t*>(a.flags_out + fo) = s_F[tid];
            }
            __syncthreads();
            // ---- F: compaction (C8): nonzero blocks in (tile, block) order ----
            if (nz) {
                const uint64_t bi = s_ex[0] + wpre_n + __popc(F & ((1u << lane) - 1u));
                const uint64_t bo = 16 * bi;
                if (bo + 16 <= a.payload_cap) *reinterpret_cast<uint4*>(a.payload_out + bo) = blk;
            }
        } else {
            if (tid == 0) {
                const uint2 tp = a.tpre[t];
                s_ex[1] = tp.x; s_ex[2] = tp.y;
            }
            __syncthreads();
        }

        // ---- outlier records (rare): ascending element index (R7, R20) ----
        if (tnd + tnv != 0) {
            int id = cd, iv = cv;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int yd = __shfl_up_sync(kFull, id, o), yv = __shfl_up_sync(kFull, iv, o);
                if (lane >= o) { id += yd; iv += yv; }
            }
            uint64_t pd = s_ex[1] + wpre_d + (id - cd), pv = s_ex[2] + wpre_v + (iv - cv);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t gi = (uint32_t)(g0 + u);
                if (dmask & (1u << u)) {
                    if (pd < a.dcap) {
                        if (a.o_didx) { a.o_didx[pd] = gi; a.o_dval[pd] = dl[u]; }
                        else a.dstage[pd] = make_uint2(gi, (uint32_t)dl[u]);
                    } else {
                        atomicOr(&ctrl->stage_overflow, 1u);
                    }
                    ++pd;
                }
                if (vmask & (1u << u)) {
                    if (pv < a.vcap) {
                        if (a.o_vidx) { a.o_vidx[pv] = gi; a.o_vbits[pv] = __float_as_uint(dv[u]); }
                        else a.vstage[pv] = make_uint2(gi, __float_as_uint(dv[u]));
                    } else {
                        atomicOr(&ctrl->stage_overflow, 1u);
                    }
                    ++pv;
                }
            }
        }
    }
}

// ------------------------------------------------------------------------------------
// C9: header + outlier sections.  Grid-stride copy of the staged records.
// ------------------------------------------------------------------------------------
__global__ void k_finalize(uint8_t* out, uint64_t out_cap, uint32_t ndim, uint64_t d0,
                           uint64_t d1, uint64_t d2, uint64_t n, uint64_t T,
                           const uint2* dstage, const uint2* vstage, Ctrl* ctrl)
{
    if (ctrl->err != 0) return;
    const uint64_t nnz = ctrl->nnz, nd = ctrl->nd, nv = ctrl->nv;
    const uint64_t total = kHeaderBytes + 32 * T + 16 * nnz + 8 * nd + 8 * nv;
    if (blockIdx.x == 0 && threadIdx.x == 0) ctrl->total = total;
    if (total > out_cap) return;
    const uint64_t dbase = kHeaderBytes + 32 * T + 16 * nnz, vbase = dbase + 8 * nd;
    if (!ctrl->stage_overflow) {
        const uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
        const uint64_t st = (uint64_t)gridDim.x * blockDim.x;
        for (uint64_t k = i0; k < nd; k += st) {
            uint2 r = dstage[k];
            *reinterpret_cast<uint2*>(out + dbase + 8 * k) = r;
        }
        for (uint64_t k = i0; k < nv; k += st) {
            uint2 r = vstage[k];
            *reinterpret_cast<uint2*>(out + vbase + 8 * k) = r;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
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

static size_t compress_smem(int ndim)
{
    const int nq = ndim == 1 ? 1 : (ndim == 2 ? 2 : 4);
    return sizeof(int) * (size_t)(nq * kQStride + 32 * 33);
}

template <int NDIM>
static cudaError_t launch_compress_t(const CompressArgs& a, uint32_t ntiles, cudaStream_t st)
{
    const size_t sm = compress_smem(NDIM);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_compress<NDIM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        attr = true;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_compress<NDIM>, kCta, sm);
    if (per_sm < 1) per_sm = 1;
    uint64_t grid = (uint64_t)per_sm * num_sms();
    if (grid > ntiles) grid = ntiles;
    if (grid == 0) return cudaSuccess;
    k_compress<NDIM><<<(unsigned)grid, kCta, sm, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_compress(const CompressArgs& a, cudaStream_t st)
{
    const uint32_t ntiles = a.tile_end - a.tile_begin;
    count_launch();
    switch (a.g.ndim) {
        case 1: return launch_compress_t<1>(a, ntiles, st);
        case 2: return launch_compress_t<2>(a, ntiles, st);
        default: return launch_compress_t<3>(a, ntiles, st);
    }
}

cudaError_t launch_init(Ctrl* ctrl, unsigned long long* status, uint32_t ntiles, const fz_params* p,
                        cudaStream_t st)
{
    fz_params pp{};
    if (p) pp = *p;
    unsigned grid = (unsigned)((ntiles + 255) / 256);
    if (grid < 1) grid = 1;
    if (grid > 1024) grid = 1024;
    count_launch();
    k_init<<<grid, 256, 0, st>>>(ctrl, status, ntiles, p ? 1 : 0, pp);
    return cudaGetLastError();
}

cudaError_t launch_range(const float* d, uint64_t n, Ctrl* ctrl, cudaStream_t st)
{
    uint64_t want = (n / 4 + 255) / 256;
    uint64_t cap = (uint64_t)num_sms() * 8;
    unsigned grid = (unsigned)(want < 1 ? 1 : (want > cap ? cap : want));
    count_launch();
    k_range<<<grid, 256, 0, st>>>(d, n, ctrl);
    return cudaGetLastError();
}

cudaError_t launch_params(Ctrl* ctrl, int mode, double eb, uint64_t n, cudaStream_t st)
{
    count_launch();
    k_params<<<1, 32, 0, st>>>(ctrl, mode, eb, n);
    return cudaGetLastError();
}

cudaError_t launch_finalize(uint8_t* out, uint64_t cap, const fz_shape& s, uint64_t n, uint64_t T,
                            const uint2* dstage, const uint2* vstage, Ctrl* ctrl, cudaStream_t st)
{
    uint64_t d[3] = {1, 1, 1};
    for (uint32_t k = 0; k < s.ndim; ++k) d[k] = s.dims[k];
    count_launch();
    k_finalize<<<num_sms(), 256, 0, st>>>(out, cap, s.ndim, d[0], d[1], d[2], n, T, dstage, vstage, ctrl);
    return cudaGetLastError();
}

}  // namespace fz
