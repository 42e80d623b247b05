// fz_rowcodes.cu -- the row walker for shapes whose rows do not tile (C1-C6 in two passes):
// 3-D fields with planes that are not whole tiles (c3: 100x500x500, c5: 1008x1008x352) and
// 2-D fields (c2: 1800x3600); nx % 4 == 0, nx >= 64.  Citation key: P:n = PAPER.md line n;
// R# = DESIGN.md §3 readings; SV = SURVEY.md.
//
// The tile (2048 consecutive codes) does not line up with rows or planes here, so the
// walk and the tiling are split:
//   k_rowcodes   (pass A) walks (column segment, band of 16 rows, plane) steps exactly like
//                k_compress_zr's phase A -- TMA-staged rows, prequantization (C1) in place,
//                Lorenzo (C2) with the z carry in tensor memory, the row above (halo) and the
//                column left of the segment (shadow) -- and writes the 2-byte codes (C3) to a
//                code field in global memory at their flattened positions; the rare
//                delta-outliers (R7) and value outliers (R20) set bits in two bit masks
//   k_rowtiles   (pass B) one warp per tile in stream order: lane c loads A-row c (the tile's
//                codes 64c .. 64c + 63: 8 x 16-byte loads), bit-transposes it (C5), flags by
//                ballot (C6), stages the nonzero blocks and the tile's outlier records (read
//                back from the masks, delta recomputed exactly from the field) -- the layout of
//                k_compress_zr's phase B, so the popcount scan and k_compact (C7, C8) follow.
// The code field costs 2 + 2 bytes per element of traffic (mostly L2 for pass B, which reads
// the tiles a pass A wave has just written); in exchange every element is quantized once and
// the z carry never leaves the SM.
#include "fz_internal.cuh"
#include "fz_launch.h"
#include "fz_rowwalk.cuh"

namespace fz {

constexpr int kRcRows = 16;                 // band height
constexpr uint32_t kRcMagic = 0x4B400000u;  // t-bits of q = 0 (magic rounding)

bool compress_uses_rc(const CompressArgs& a)
{
    if (a.rescan || a.tstage == nullptr || a.rc_codes == nullptr || a.cl || (variant_bits() & 131072)) return false;
    // 3-D (c3, c5; 2-D fields measured slower than the single-pass kernel: a band is one
    // step with no z carry to reuse, and a 3600-wide row needs per-row copies)
    if (a.g.ndim != 3 && !(a.g.ndim == 2 && (variant_bits() & 262144))) return false;
    const uint32_t nx = a.g.nx;
    // runs of planes long enough to amortize the seed steps (c5: nz = 1008; c3's nz = 100
    // measured slower than the single-pass kernel)
    if (a.g.ndim == 3 && a.g.n / a.g.P < 256 && !(variant_bits() & 262144)) return false;
    // whole fields only (the slab API's tile ranges take the single-pass kernels)
    if (nx % 4 != 0 || nx < 64 || a.base != 0 || a.tile_begin != 0 ||
        (uint64_t)a.tile_end != ((uint64_t)a.g.n + kTileCodes - 1) / kTileCodes)
        return false;
    return true;
}

bool rc_layout_shape(const fz_shape& s)
{
    if (s.ndim != 2 && s.ndim != 3) return false;
    const uint64_t nx = s.dims[s.ndim - 1];
    return nx % 4 == 0 && nx >= 64;
}

// Exact q of (z, y, x), zero outside the field (the rare delta-outlier path).
__device__ int32_t rc_q(const CompressArgs& a, const QuantP& P, int64_t z, int64_t y, int64_t x)
{
    if (z < 0 || y < 0 || x < 0) return 0;
    bool vo;
    const uint64_t g = (uint64_t)z * a.g.P + (uint64_t)y * a.g.nx + (uint64_t)x;
    return prequant(__ldg(a.field + g), P, vo);
}

__device__ int32_t rc_delta(const CompressArgs& a, const QuantP& P, int64_t z, int64_t y, int64_t x)
{
    uint32_t s = 0;
#pragma unroll 1
    for (int k = 0; k < 8; ++k) {
        const int dz = k >> 2 & 1, dy = k >> 1 & 1, dx = k & 1;
        const uint32_t q = (uint32_t)rc_q(a, P, z - dz, y - dy, x - dx);
        s += ((dz + dy + dx) & 1) ? 0u - q : q;
    }
    return (int32_t)s;
}

struct RcShared {
    QuantP P;
    int perr;
    uint32_t tmem;
};

// t-bits of one row's 4 values in place (fast path, inline exact correction of hard elements
// in margin mode, the full exact rule + bound check in fallback mode: value-outlier bits).
__device__ __forceinline__ void rc_trow(float4& v, const QuantP& P, uint32_t& vb)
{
    const float kMagic = 12582912.0f;
    const float thr = P.hU < 0.0f ? -1.0f : P.h;
    float d[4] = {v.x, v.y, v.z, v.w};
    uint32_t t[4];
    float e[4];
    bool hard = false;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float tf = __fmaf_rn(d[k], P.r, kMagic);
        const float qf = __fsub_rn(tf, kMagic);
        e[k] = __fmaf_rn(-qf, P.w, d[k]);
        hard |= !(fabsf(e[k]) < thr);
        t[k] = __float_as_uint(tf);
    }
    vb = 0;
    if (__builtin_expect(hard, 0)) {
        if (P.hU < 0.0f) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                bool vo;
                t[k] = (uint32_t)prequant(d[k], P, vo) + kRcMagic;
                if (vo) vb |= 1u << k;
            }
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float ae = fabsf(e[k]);
                const bool step = ae > P.h || (ae == P.h && (t[k] & 1u));
                t[k] += step ? (e[k] > 0.0f ? 1u : 0xFFFFFFFFu) : 0u;
            }
        }
    }
    v = make_float4(__uint_as_float(t[0]), __uint_as_float(t[1]), __uint_as_float(t[2]), __uint_as_float(t[3]));
}

__device__ __forceinline__ uint32_t rc_pack2(int32_t d0, int32_t d1, uint32_t& mag)
{
    const uint32_t m0 = (uint32_t)abs(d0), m1 = (uint32_t)abs(d1);
    mag |= m0 | m1;
    return bitsel(__byte_perm((uint32_t)d0, (uint32_t)d1, 0x7030u), __byte_perm(m0, m1, 0x5410u), 0x80008000u);
}

// ---- pass A ----
// Steps: unit u = (segment s, band b, plane z), s-major, then b, then z; a CTA takes an equal
// share of the units, so it walks runs of planes of one (segment, band); a run starting at
// z0 > 0 first re-quantizes plane z0 - 1 (seed step) into the carry.
template <int NW>
__global__ void __launch_bounds__(32 * NW, 12 / NW) k_rowcodes(CompressArgs a, uint32_t nseg, uint32_t ny,
                                                               uint32_t nz)
{
    pdl_begin();
    extern __shared__ __align__(128) uint8_t rsm[];
    __shared__ RcShared sh;
    __shared__ __align__(8) uint64_t mbar[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    Ctrl* ctrl = a.ctrl;
    if (ctrl->err != 0) return;
    constexpr uint32_t SW = 128u * NW;                          // segment width
    constexpr uint32_t sbytes = (kRcRows + 1) * 4u * SW;
    const uint32_t nx = a.g.nx, PL = a.g.P;
    // shared row pitch: the field's own row pitch when one segment spans the row (the band's
    // rows are then one contiguous bulk copy), else the segment's width
    const uint32_t RP = nseg == 1 ? 4u * nx : 4u * SW;
    const uint32_t nbands = (ny + kRcRows - 1) / kRcRows;
    if (tid == 0) {
        sh.perr = 0;
        if (a.derive) {
            fz_params p;
            const int st = params_from_range(ctrl, a.eb_mode, a.eb, a.n_hdr, &p);
            sh.perr = st;
            if (st == FZ_OK) {
                float h, hU;
                quant_consts(p, h, hU);
                sh.P = QuantP{p.w, p.r, h, p.eb32, hU};
                if (blockIdx.x == 0) { ctrl->p = p; ctrl->h = h; ctrl->hU = hU; }
            } else if (blockIdx.x == 0) {
                ctrl->err = st;
            }
        } else {
            sh.P = QuantP{ctrl->p.w, ctrl->p.r, ctrl->h, ctrl->p.eb32, ctrl->hU};
        }
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    constexpr uint32_t kTmemCols = NW > 4 ? 256u : 128u;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"(smem_u32(&sh.tmem)), "n"(kTmemCols) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t taddr = sh.tmem + ((32u * (warp & 3)) << 16) + 68u * (warp >> 2);
    auto tmem_free = [&]() {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (warp == 0)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(sh.tmem), "n"(kTmemCols)
                         : "memory");
    };
    if (sh.perr != 0) {
        tmem_free();
        return;
    }
    const QuantP P = sh.P;
    const uint64_t U = (uint64_t)nseg * nbands * nz;
    const uint64_t u0 = U * blockIdx.x / gridDim.x, u1 = U * (blockIdx.x + 1) / gridDim.x;
    // the step sequence: (run, z) with a seed step before a run that starts at z > 0
    struct Step {
        uint32_t s, b, z;
        bool seed, run_start, valid;
    };
    struct Cur {
        uint64_t u;
        uint32_t sb, z;   // u = sb * nz + z
        bool seeded;
    };
    auto next = [&](Cur& c) -> Step {
        Step st{0, 0, 0, false, false, false};
        if (c.u >= u1) return st;
        st.valid = true;
        st.s = c.sb / nbands;
        st.b = c.sb - st.s * nbands;
        st.z = c.z;
        const bool start = c.u == u0 || c.z == 0;
        if (start && !c.seeded && st.z > 0) {
            c.seeded = true;
            st.seed = true;
            st.run_start = true;
            st.z -= 1;
            return st;
        }
        st.run_start = start && !c.seeded;
        c.seeded = false;
        ++c.u;
        if (++c.z == nz) { c.z = 0; ++c.sb; }
        return st;
    };
    auto cur0 = [&]() { return Cur{u0, (uint32_t)(u0 / nz), (uint32_t)(u0 % nz), false}; };
    // TMA of a step: rows y0 - 1 .. y0 + rows - 1 of columns [xs, xs + w) (one bulk copy per
    // row unless the segment is the whole row, then one copy)
    auto issue = [&](const Step& st, uint32_t k) {
        uint8_t* dst = rsm + (k & 1u) * sbytes;
        const uint32_t y0 = st.b * kRcRows, xs = st.s * SW;
        const uint32_t w = min(SW, nx - xs);
        const uint32_t rows = min((uint32_t)kRcRows, ny - y0) + (y0 > 0 ? 1u : 0u);
        const uint32_t ylo = y0 > 0 ? y0 - 1 : 0;
        uint8_t* d0 = dst + (y0 > 0 ? 0u : RP);
        const float* src = a.field + (uint64_t)st.z * PL + (uint64_t)ylo * nx + xs;
        mbar_expect_tx(&mbar[k & 1u], rows * w * 4u);
        if (nseg == 1) {
            tma_load_1d(d0, src, rows * w * 4u, &mbar[k & 1u]);
        } else {
            for (uint32_t r = 0; r < rows; ++r) tma_load_1d(d0 + r * RP, src + (uint64_t)r * nx, w * 4u, &mbar[k & 1u]);
        }
    };
    // both stages in flight: steps 0 and 1 now, step k + 2 once step k is consumed (pass A has
    // no tile phase to hide the copy behind)
    Cur ic = cur0();
    uint32_t kissue = 0;
    if (tid == 0) {
        for (int j = 0; j < 2; ++j) {
            const Step st = next(ic);
            if (st.valid) issue(st, kissue++);
        }
    }
    Cur pc = cur0();
    uint32_t th[4], tsh = kRcMagic;
    bool zfirst = true;
    for (uint32_t k = 0;; ++k) {
        const Step st = next(pc);
        if (!st.valid) break;
        uint8_t* stg = rsm + (k & 1u) * sbytes;
        const uint32_t y0 = st.b * kRcRows, xs = st.s * SW, z = st.z;
        const uint32_t rows = min((uint32_t)kRcRows, ny - y0);
        const uint32_t x0 = xs + 128u * warp + 4u * lane;
        const bool colv = x0 < nx;
        if (st.run_start) {
            zfirst = true;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) th[kk] = kRcMagic;
            tsh = kRcMagic;
        }
        // shadow column x0w - 1 of warp w (x0w = xs + 128 w), lane j = row y0 - 1 + j
        const uint32_t xsh = xs + 128u * warp;
        const bool shv = xsh > 0 && xsh < nx && lane <= (int)rows && (y0 + lane) > 0;
        float dsh = 0.0f;
        if (shv) dsh = __ldg(a.field + (uint64_t)z * PL + (uint64_t)(y0 + lane - 1) * nx + xsh - 1u);
        while (!mbar_try_wait(&mbar[k & 1u], (k >> 1) & 1u)) {
        }
        const bool halo = y0 > 0;
        // t-bits in place (own rows 1..rows, and row 0 when the halo is used), in groups of 8
        // rows whose loads are issued together; lanes past nx skip (they still join the
        // warp-wide shuffles below)
        if (colv) {
            if (halo) {
                float4* p = reinterpret_cast<float4*>(stg + 16u * tid);
                float4 v = *p;
                uint32_t vb;
                rc_trow(v, P, vb);
                *p = v;
            }
#pragma unroll
            for (int r0 = 1; r0 <= kRcRows; r0 += 8) {
                float4 v[8];
#pragma unroll
                for (int g = 0; g < 8; ++g)
                    if ((uint32_t)(r0 + g) <= rows) v[g] = *reinterpret_cast<const float4*>(stg + (r0 + g) * RP + 16u * tid);
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    if ((uint32_t)(r0 + g) > rows) continue;
                    uint32_t vb;
                    rc_trow(v[g], P, vb);
                    *reinterpret_cast<float4*>(stg + (r0 + g) * RP + 16u * tid) = v[g];
                    if (__builtin_expect(vb != 0, 0) && !st.seed) {   // value outliers (fallback mode)
                        const uint64_t gi = (uint64_t)z * PL + (uint64_t)(y0 + r0 + g - 1) * nx + x0;
                        atomicOr(a.rc_vmask + (gi >> 5), vb << (gi & 31));
                    }
                }
            }
        }
        uint32_t tshn = kRcMagic;
        if (shv) {
            bool vo;
            tshn = (uint32_t)prequant(dsh, P, vo) + kRcMagic;
        }
        __syncwarp();
        if (st.seed) {
#pragma unroll 1
            for (int g = 0; g < kRcRows / 4; ++g) {
                uint32_t tv[16];
#pragma unroll
                for (int ii = 0; ii < 4; ++ii) {
                    uint4 v = make_uint4(kRcMagic, kRcMagic, kRcMagic, kRcMagic);
                    if (colv && (uint32_t)(4 * g + ii) < rows)
                        v = *reinterpret_cast<const uint4*>(stg + (4 * g + ii + 1) * RP + 16u * tid);
                    tv[4 * ii] = v.x; tv[4 * ii + 1] = v.y; tv[4 * ii + 2] = v.z; tv[4 * ii + 3] = v.w;
                }
                tmem_st16(taddr + 16u * g, tv);
            }
            tmem_wait_st();
            zfirst = false;
            if (halo && colv) {
                const uint4 tv = *reinterpret_cast<const uint4*>(stg + 16u * tid);
                th[0] = tv.x; th[1] = tv.y; th[2] = tv.z; th[3] = tv.w;
            }
            if (shv) tsh = tshn;
            __syncthreads();
            if (tid == 0) {
                const Step nst = next(ic);
                if (nst.valid) issue(nst, kissue++);
            }
            continue;
        }
        uint32_t Zup[4] = {0u, 0u, 0u, 0u};
        if (halo && colv) {
            const uint4 tv = *reinterpret_cast<const uint4*>(stg + 16u * tid);
            const uint32_t t[4] = {tv.x, tv.y, tv.z, tv.w};
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) { Zup[kk] = t[kk] - th[kk]; th[kk] = t[kk]; }
        }
        uint32_t Ysh;
        {
            uint32_t Zs = 0u;
            if (shv) { Zs = tshn - tsh; tsh = tshn; }
            const uint32_t Zabove = __shfl_up_sync(kFull, Zs, 1);
            Ysh = Zs - Zabove;
        }
        if (zfirst) {
            uint32_t mg[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) mg[j] = kRcMagic;
#pragma unroll
            for (int g = 0; g < kRcRows / 4; ++g) tmem_st16(taddr + 16u * g, mg);
            tmem_wait_st();
        }
        uint32_t magor = 0;
        uint32_t tpb[2][8];
        tmem_ld8(taddr, tpb[0]);
        uint16_t* const co = a.rc_codes + (uint64_t)z * PL + (uint64_t)y0 * nx + x0;
#pragma unroll
        for (int i = 0; i < kRcRows; ++i) {
            uint32_t(&tpp)[8] = tpb[(i >> 1) & 1];
            if ((i & 1) == 0) {
                tmem_wait_ld8(tpp);
                if (i + 2 < kRcRows) tmem_ld8(taddr + 4u * (i + 2), tpb[((i >> 1) + 1) & 1]);
            }
            const uint32_t* tp = tpp + 4 * (i & 1);
            uint4 tv = make_uint4(kRcMagic, kRcMagic, kRcMagic, kRcMagic);
            if (colv && (uint32_t)i < rows) tv = *reinterpret_cast<const uint4*>(stg + (i + 1) * RP + 16u * tid);
            const uint32_t t[4] = {tv.x, tv.y, tv.z, tv.w};
            tmem_st4(taddr + 4u * i, t[0], t[1], t[2], t[3]);
            uint32_t Y[4];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const uint32_t Z = t[kk] - tp[kk];
                Y[kk] = Z - Zup[kk];
                Zup[kk] = Z;
            }
            uint32_t Yl = __shfl_up_sync(kFull, Y[3], 1);
            const uint32_t ysh = __shfl_sync(kFull, Ysh, i + 1);
            if (lane == 0) Yl = ysh;   // x = xs + 128 w - 1 (0 at x = 0: Ysh = 0 there)
            uint32_t mag = 0;
            const uint32_t w0 = rc_pack2((int32_t)(Y[0] - Yl), (int32_t)(Y[1] - Y[0]), mag);
            const uint32_t w1 = rc_pack2((int32_t)(Y[2] - Y[1]), (int32_t)(Y[3] - Y[2]), mag);
            if (colv && (uint32_t)i < rows) {
                magor |= mag;
                *reinterpret_cast<uint2*>(co + (uint64_t)i * nx) = make_uint2(w0, w1);
            }
        }
        tmem_wait_st();
        zfirst = false;
        // delta-outliers (R7): code 0 and a mask bit (the value is recomputed in pass B)
        if (__builtin_expect(magor > 32767u, 0)) {
#pragma unroll 1
            for (uint32_t i = 0; i < rows; ++i) {
                uint2 wv = *reinterpret_cast<uint2*>(co + (uint64_t)i * nx);
                uint32_t dbits = 0;
#pragma unroll 1
                for (int kk = 0; kk < 4; ++kk) {
                    const int32_t dl = rc_delta(a, P, z, y0 + i, x0 + kk);
                    if ((uint32_t)abs(dl) > 32767u) {
                        dbits |= 1u << kk;
                        uint32_t& wd = (kk < 2) ? wv.x : wv.y;
                        wd &= (kk & 1) ? 0x0000FFFFu : 0xFFFF0000u;
                    }
                }
                if (dbits) {
                    *reinterpret_cast<uint2*>(co + (uint64_t)i * nx) = wv;
                    const uint64_t g = (uint64_t)z * PL + (uint64_t)(y0 + i) * nx + x0;
                    atomicOr(a.rc_dmask + (g >> 5), dbits << (g & 31));
                }
            }
        }
        __syncthreads();
        if (tid == 0) {
            const Step nst = next(ic);
            if (nst.valid) issue(nst, kissue++);
        }
    }
    tmem_free();
}

// ---- pass B: one warp per tile (stream order), 8 warps per CTA, persistent ----
// The tile's 4 KB of codes arrive by coalesced 16-byte loads (lane L: bytes 16 L + 512 j) a
// tile ahead, are stored to the warp's shared buffer with A-row r at 144 r (16 bytes of skew
// per A-row: conflict-free), and lane c reads A-row c back (8 x 16 bytes).
__global__ void __launch_bounds__(256) k_rowtiles(CompressArgs a, uint32_t ntiles)
{
    pdl_begin();
    __shared__ __align__(16) uint8_t Bsh[8][32 * 144];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    Ctrl* ctrl = a.ctrl;
    if (ctrl->err != 0) return;
    const QuantP P{ctrl->p.w, ctrl->p.r, ctrl->h, ctrl->p.eb32, ctrl->hU};
    const uint64_t n = a.g.n;
    const uint32_t nx = a.g.nx, PL = a.g.P;
    uint8_t* const B = Bsh[warp];
    uint32_t* const Os = reinterpret_cast<uint32_t*>(B);
    const uint32_t stride = gridDim.x * 8;
    uint4 nxt[8];
    auto load_tile = [&](uint32_t t) {   // whole tiles only (the tail tile is read element-wise)
        const uint64_t g = (uint64_t)t * kTileCodes;
        if (t < ntiles && g + kTileCodes <= n) {
            const uint4* src = reinterpret_cast<const uint4*>(a.rc_codes + g);
#pragma unroll
            for (int j = 0; j < 8; ++j) nxt[j] = __ldcs(src + lane + 32 * j);
        }
    };
    load_tile(blockIdx.x * 8 + warp);
    for (uint32_t t = blockIdx.x * 8 + warp; t < ntiles; t += stride) {
        const uint64_t g0 = (uint64_t)t * kTileCodes + 64u * lane;   // A-row c = codes 64c ..
        // outlier mask words of A-row c (issued first: consumed after the flags)
        uint2 mv = make_uint2(0, 0), md = make_uint2(0, 0);
        if (g0 < n) {
            mv = *reinterpret_cast<const uint2*>(a.rc_vmask + (g0 >> 5));
            md = *reinterpret_cast<const uint2*>(a.rc_dmask + (g0 >> 5));
        }
        const bool whole = (uint64_t)t * kTileCodes + kTileCodes <= n;
        // a tile of zero codes (RTM's exact-zero regions) has zero flags and no blocks:
        // no staging, no transpose (its outlier marks below still count: a delta outlier's code is 0)
        bool zt = false;
        if (whole && a.codes_out == nullptr) {
            uint32_t o = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) o |= nxt[j].x | nxt[j].y | nxt[j].z | nxt[j].w;
            zt = !__any_sync(kFull, o != 0u);
        }
        if (zt) {
            load_tile(t + stride);
            if (lane < 8) {
                const uint64_t fo = (uint64_t)t * 32 + 4 * lane;
                if (fo + 4 <= a.flags_cap) *reinterpret_cast<uint32_t*>(a.flags_out + fo) = 0u;
            }
        } else {
        uint32_t A[32];
        if (whole) {
            // 16-byte chunk L + 32 j of the tile = A-row (L + 32 j) / 8, part (L + 32 j) % 8
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t c = (uint32_t)lane + 32u * j;
                *reinterpret_cast<uint4*>(B + 144u * (c >> 3) + 16u * (c & 7)) = nxt[j];
            }
            load_tile(t + stride);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint4 v = *reinterpret_cast<const uint4*>(B + 144u * lane + 16u * j);
                A[4 * j] = v.x; A[4 * j + 1] = v.y; A[4 * j + 2] = v.z; A[4 * j + 3] = v.w;
            }
        } else {   // the zero-padded tail (C4)
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const uint64_t e = g0 + 2 * j;
                const uint32_t lo = e < n ? a.rc_codes[e] : 0u, hi = e + 1 < n ? a.rc_codes[e + 1] : 0u;
                A[j] = lo | hi << 16;
            }
        }
        if (a.codes_out != nullptr) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                if (g0 + 2 * j < n) a.codes_out[g0 + 2 * j] = (uint16_t)A[j];
                if (g0 + 2 * j + 1 < n) a.codes_out[g0 + 2 * j + 1] = (uint16_t)(A[j] >> 16);
            }
        }
        transpose32_regs(A);
        __syncwarp();   // every lane has read its A-row: the buffer takes O
#pragma unroll
        for (int r = 0; r < 32; ++r) Os[32 * r + lane] = A[r];
        __syncwarp();
        uint4* stage = a.tstage + (uint64_t)t * kTileBlocks;
        uint32_t myF = 0;
#pragma unroll
        for (int f = 0; f < 8; ++f) {
            const uint4 blk = *reinterpret_cast<const uint4*>(Os + 128 * f + 4 * lane);
            const bool nz = (blk.x | blk.y | blk.z | blk.w) != 0;
            const uint32_t F = __ballot_sync(kFull, nz);
            if (lane == f) myF = F;
            if (nz) stage[32 * f + __popc(F & ((1u << lane) - 1u))] = blk;
        }
        if (lane < 8) {
            const uint64_t fo = (uint64_t)t * 32 + 4 * lane;
            if (fo + 4 <= a.flags_cap) *reinterpret_cast<uint32_t*>(a.flags_out + fo) = myF;
        }
        __syncwarp();   // the blocks are read: the next tile's codes may overwrite the buffer
        }
        // outliers of this tile: the mask bits of A-row c are words (g0 >> 5) and +1
        const uint64_t vm = (uint64_t)mv.x | (uint64_t)mv.y << 32, dm = (uint64_t)md.x | (uint64_t)md.y << 32;
        if (__any_sync(kFull, (vm | dm) != 0)) {
            const uint32_t cd = __popcll(dm), cv = __popcll(vm);
            uint32_t id = cd, iv = cv;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t yd = __shfl_up_sync(kFull, id, o), yv = __shfl_up_sync(kFull, iv, o);
                if (lane >= o) { id += yd; iv += yv; }
            }
            const uint32_t tnd = __shfl_sync(kFull, id, 31), tnv = __shfl_sync(kFull, iv, 31);
            unsigned long long bd = 0, bv = 0;
            if (lane == 0) {
                bd = tnd ? atomicAdd(&ctrl->dcount, (unsigned long long)tnd) : 0ull;
                bv = tnv ? atomicAdd(&ctrl->vcount, (unsigned long long)tnv) : 0ull;
                a.ocnt[t] = make_uint2(tnd, tnv);
                a.obase[t] = make_uint2((uint32_t)bd, (uint32_t)bv);
            }
            bd = __shfl_sync(kFull, bd, 0);
            bv = __shfl_sync(kFull, bv, 0);
            uint64_t pd = bd + id - cd, pv = bv + iv - cv;
#pragma unroll 1
            for (int j = 0; j < 64; ++j) {
                const uint64_t gi = g0 + j;
                if ((dm >> j) & 1u) {
                    const uint64_t zz = gi / PL, rem = gi - zz * PL, yy = rem / nx, xx = rem - yy * nx;
                    const int32_t dl = rc_delta(a, P, (int64_t)zz, (int64_t)yy, (int64_t)xx);
                    if (pd < a.dcap) a.dstage[pd] = make_uint2((uint32_t)gi, (uint32_t)dl);
                    else atomicOr(&ctrl->stage_overflow, 1u);
                    ++pd;
                }
                if ((vm >> j) & 1u) {
                    if (pv < a.vcap) a.vstage[pv] = make_uint2((uint32_t)gi, __float_as_uint(__ldg(a.field + gi)));
                    else atomicOr(&ctrl->stage_overflow, 1u);
                    ++pv;
                }
            }
        }
    }
}

template <int NW>
static cudaError_t rc_launch(const CompressArgs& a, uint32_t nseg, uint32_t ny, uint32_t nz, cudaStream_t st)
{
    auto kern = k_rowcodes<NW>;
    const size_t sm = 2ull * (kRcRows + 1) * 4 * 128 * NW;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kern);
    int dev = 0, smem_sm = 0, regs_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
    const int regs_cta = ((fa.numRegs + 7) & ~7) * 32 * NW;
    int per_sm = (int)(smem_sm / (sm + fa.sharedSizeBytes + 1024));
    if (regs_cta > 0 && regs_sm / regs_cta < per_sm) per_sm = regs_sm / regs_cta;
    const int tmem_cap = 512 / (NW > 4 ? 256 : 128);
    if (per_sm > tmem_cap) per_sm = tmem_cap;
    if (per_sm < 1) per_sm = 1;
    const uint64_t units = (uint64_t)nseg * ((ny + kRcRows - 1) / kRcRows) * nz;
    uint64_t grid = (uint64_t)per_sm * num_sms();
    if (grid > units) grid = units;
    LaunchProf lp(K_COMPRESS, st);
    { const cudaError_t e_ = launch_pdl(kern, dim3((unsigned)grid), dim3(32 * NW), sm, st, a, nseg, ny, nz); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

cudaError_t launch_compress_rc(const CompressArgs& a, cudaStream_t st)
{
    const uint32_t nx = a.g.nx;
    uint32_t ny, nz;
    if (a.g.ndim == 3) { ny = a.g.P / nx; nz = a.g.n / a.g.P; }
    else { ny = a.g.n / nx; nz = 1; }
    const uint32_t T = a.tile_end;
    // the masks start clear (pass A only ORs bits in)
    cudaError_t e = cudaMemsetAsync(a.rc_vmask, 0, 2 * 4 * (size_t)(((uint64_t)T * kTileCodes + 31) / 32 + 2), st);
    if (e != cudaSuccess) return e;
    if (nx <= 128) e = rc_launch<1>(a, 1, ny, nz, st);
    else if (nx <= 256) e = rc_launch<2>(a, 1, ny, nz, st);
    else if (nx <= 384) e = rc_launch<3>(a, 1, ny, nz, st);
    else if (nx <= 512) e = rc_launch<4>(a, 1, ny, nz, st);
    else if (nx <= 1024) e = rc_launch<8>(a, 1, ny, nz, st);
    else e = rc_launch<8>(a, (nx + 1023) / 1024, ny, nz, st);
    if (e != cudaSuccess) return e;
    const uint64_t want = ((uint64_t)T + 7) / 8;
    const uint64_t cap = (uint64_t)num_sms() * 8;
    LaunchProf lp(K_ROWTILES, st);
    { const cudaError_t e_ = launch_pdl(k_rowtiles, dim3((unsigned)(want < cap ? want : cap)), dim3(256), 0, st, a, T); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

}  // namespace fz
