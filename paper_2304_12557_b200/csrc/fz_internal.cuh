// fz_internal.cuh -- device-side building blocks of libfz (B200, sm_100a).
//
// Nothing here is shared with oracle/: the oracle is an independent C program.
// Citation key: P:n = PAPER.md line n; SV = SURVEY.md; R# = DESIGN.md §3 readings.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/fz.h"

namespace fz {

constexpr int kTileCodes = 2048;   // 32x32 u32 words, 2 codes per word
constexpr int kTileWords = 1024;
constexpr int kTileBlocks = 256;   // 16-byte blocks per tile (P:253, 256 byte flags)
constexpr int kCta = 256;          // threads per CTA: one 16-byte block per thread
constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr size_t kHeaderBytes = 128;

// ------------------------------------------------------------------------------------
// Device control block (first 512 bytes of every workspace).
// ------------------------------------------------------------------------------------
struct Ctrl {
    // range pass (C0)
    uint32_t mn_enc, mx_enc;         // order-preserving encodings of min / max
    unsigned long long first_bad;    // first non-finite index, ~0 if none
    // parameters (Appendix A), written by k_params or k_init
    fz_params p;
    float h;                         // w / 2
    float hU;                        // fast-path threshold (see pq_fast)
    int32_t err;                     // fz_status of the device-side steps
    uint32_t ticket;                 // persistent-tile ticket
    uint32_t stage_overflow;         // outlier staging overflowed -> rescan pass
    // results (written by the last tile / k_finalize)
    unsigned long long nnz, nd, nv, total;
    unsigned long long dcount, vcount;   // outlier staging allocation counters (= totals)
    uint32_t done;                       // CTAs finished (last one finalizes)
    // decoder, device-driven mode (k_decode_hdr parses the stream header on the device)
    unsigned long long dec_nnz, dec_nd, dec_nv;
    float dec_w;
    uint32_t chunk;                      // f1 chunk-local stream: cz | cy << 16 (0: field-global)
    uint32_t dec_flags;                  // header flags of the stream being decoded (dev mode)
    unsigned long long log_bad;          // f3: first index outside the log domain, ~0 if none
    uint32_t rclaim, rdone;              // fused range phase of the row walker: chunks claimed / done
    uint32_t scan_done;                  // flag-popcount scan: blocks finished (the last one scans the totals)
};
static_assert(sizeof(Ctrl) <= 512, "Ctrl too large");

// Workspace carve (host computes it identically for every call).
//   status : per-tile look-back word, state(2) | inclusive-or-aggregate nnz(62)
//   ocnt   : per-tile (n_delta, n_value); obase: staging offsets of the tile's records;
//   opre   : per-tile exclusive outlier offsets (filled only when outliers exist)
struct Layout {
    size_t ctrl, status, ocnt, obase, opre, dstage, vstage, tstage, zloc, zbsum, rcodes, rmask, total;
    uint64_t ntiles;
    uint64_t dcap, vcap;             // staging capacities in records
};

// zb: room for the z-band two-pass compressor (a 4 KB staging slot per tile + the offsets
// of its compaction pass).
inline uint64_t rc_mask_words(uint64_t tiles) { return tiles * 64 + 2; }   // even: 8-byte aligned pairs

inline Layout compress_layout(uint64_t n, uint64_t tiles, bool zb = false, bool rc = false)
{
    Layout L{};
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    size_t off = 0;
    L.ntiles = tiles;
    L.ctrl = off;   off += 512;
    L.status = off; off = al(off + 8 * tiles);
    L.ocnt = off;   off = al(off + 8 * tiles);
    L.obase = off;  off = al(off + 8 * tiles);
    L.opre = off;   off = al(off + 8 * tiles);
    L.dcap = n / 64 + 1024;
    L.vcap = n / 64 + 1024;
    L.dstage = off; off = al(off + 8 * L.dcap);
    L.vstage = off; off = al(off + 8 * L.vcap);
    L.tstage = L.zloc = L.zbsum = L.rcodes = L.rmask = 0;
    if (zb || rc) {
        L.tstage = off; off = al(off + 16 * 256 * tiles);
        L.zloc = off;   off = al(off + 4 * tiles);
        L.zbsum = off;  off = al(off + 4 * ((tiles + 1023) / 1024));
    }
    if (rc) {
        L.rcodes = off; off = al(off + 2 * 2048 * tiles);
        L.rmask = off;  off = al(off + 2 * 4 * rc_mask_words(tiles));
    }
    L.total = off;
    return L;
}

// 3-D, nx % 4 == 0 and whole tiles per plane: the shapes the z-band compressor may take.
inline bool zb_shape(uint32_t ndim, uint64_t ny, uint64_t nx, uint64_t nz)
{
    return ndim == 3 && nz >= 2 && nx % 4 == 0 && (ny * nx) % 2048 == 0 && nx + 1 + 2048 + 4 <= 8192;
}

// ------------------------------------------------------------------------------------
// Fast 32-bit unsigned division by a runtime constant (round-up multiplier method):
//   n / d = (umulhi(n, m) + n) >> s,  s = ceil(log2 d),  m = floor(2^32 (2^s - d) / d) + 1.
// ------------------------------------------------------------------------------------
struct FastDiv {
    uint32_t d, m, s;
};

inline FastDiv make_fastdiv(uint32_t d)
{
    FastDiv f{d, 0, 0};
    uint32_t s = 0;
    while ((1ull << s) < d) ++s;
    f.s = s;
    f.m = (uint32_t)((((1ull << s) - d) << 32) / d + 1);
    return f;
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f)
{
    const uint64_t hi = __umulhi(n, f.m);
    return (uint32_t)((hi + n) >> f.s);
}
__device__ __forceinline__ uint32_t fmod_(uint32_t n, const FastDiv& f)
{
    return n - fdiv(n, f) * f.d;
}

// ------------------------------------------------------------------------------------
// Order-preserving float <-> u32 (for atomicMin/Max of the range).
// ------------------------------------------------------------------------------------
__host__ __device__ inline uint32_t f2ord(float f)
{
    uint32_t b;
#ifdef __CUDA_ARCH__
    b = __float_as_uint(f);
#else
    memcpy(&b, &f, 4);
#endif
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__host__ __device__ inline float ord2f(uint32_t u)
{
    uint32_t b = (u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u;
    float f;
#ifdef __CUDA_ARCH__
    f = __uint_as_float(b);
#else
    memcpy(&f, &b, 4);
#endif
    return f;
}

// ------------------------------------------------------------------------------------
// Memory-model helpers for the decoupled look-back (gpu scope).
// ------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p)
{
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v)
{
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p)
{
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p)
{
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p)
{
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v)
{
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ------------------------------------------------------------------------------------
// Wide decoupled look-back (C7).  Status word of tile t: state(2) | value(62),
// state 1 = aggregate, 2 = inclusive prefix.  `term` additionally marks aggregates that do
// not depend on earlier tiles (segmented scans: a row start inside the tile, bit 61).
// One warp reads W = 32 * PER_LANE predecessors per round (relaxed gpu-scope loads, no L1
// invalidation: each status word is self-contained), finds the nearest terminal entry and
// sums the values from it up to t-1.  Entries before `first` count as inclusive zeros.
// Must be called by a full warp; returns the sum (exclusive prefix / carry) in every lane.
// ------------------------------------------------------------------------------------
constexpr unsigned long long kStAgg = 1ull << 62, kStInc = 2ull << 62;
constexpr unsigned long long kStTerm = 1ull << 61;

// Watchdog: a look-back that spins for ~seconds raises kErrStall in *err and returns, so a
// logic error can never hang the device (the caller reports FZ_ERR_CUDA).
constexpr int32_t kErrStall = 100;

// Window layout: entry (k, lane) is tile t-1-(32k + lane), i.e. distance 32k + lane: each
// load instruction reads 32 consecutive status words (two 128-byte lines).
template <int PER_LANE>
__device__ __forceinline__ void lookback_load(const unsigned long long* st, int64_t hi, int64_t first,
                                              unsigned long long (&v)[PER_LANE])
{
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < PER_LANE; ++k) {
        const int64_t idx = hi - 32 * k - lane;
        v[k] = idx >= first ? ld_relaxed_u64(st + idx) : kStInc;
    }
}

// Evaluates one loaded window: returns 0 = an entry nearer than the nearest terminal is
// unpublished (retry), 1 = terminal found (sum complete), 2 = no terminal (sum of the whole
// window, continue with the next window).
template <int PER_LANE, bool SEG>
__device__ __forceinline__ int lookback_eval(const unsigned long long (&v)[PER_LANE], unsigned long long vmask,
                                             unsigned long long& sum)
{
    const int lane = threadIdx.x & 31;
    // nearest terminal: smallest k with one, lowest lane within it
    int kt = PER_LANE;
    uint32_t tmask = 0;
#pragma unroll
    for (int k = PER_LANE - 1; k >= 0; --k) {
        const bool term = (v[k] >> 62) == 2 || (SEG && (v[k] & kStTerm));
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, term);
        if (m) { kt = k; tmask = m; }
    }
    const int tl = kt < PER_LANE ? __ffs(tmask) - 1 : 0;
    // every entry nearer than the terminal must be published
    bool missing = false;
#pragma unroll
    for (int k = 0; k < PER_LANE; ++k) {
        const bool nearer = k < kt || (k == kt && lane < tl);
        if (nearer && (v[k] >> 62) == 0) missing = true;
    }
    if (__any_sync(0xFFFFFFFFu, missing)) return 0;
    unsigned long long part = 0;
#pragma unroll
    for (int k = 0; k < PER_LANE; ++k) {
        const bool take = k < kt || (k == kt && lane <= tl);
        if (take) part += v[k] & vmask;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xFFFFFFFFu, part, o);
    sum = part;
    return kt < PER_LANE ? 1 : 2;
}

// `pre` (optional) is the first window, loaded earlier by lookback_load(st, t-1, first, pre)
// so that its latency overlaps other work.
template <int PER_LANE, bool SEG>
__device__ __forceinline__ unsigned long long lookback_wide(const unsigned long long* st, int64_t t,
                                                            int64_t first, unsigned long long vmask,
                                                            int32_t* err,
                                                            const unsigned long long* pre = nullptr,
                                                            unsigned long long* dbg = nullptr)
{
    const int lane = threadIdx.x & 31;
    unsigned long long sum = 0;
    int64_t hi = t - 1;
    uint32_t spins = 0;
    bool use_pre = pre != nullptr;
    while (hi >= first) {
        unsigned long long v[PER_LANE];
        for (;;) {
            if (++spins > (1u << 22)) {
                if (lane == 0) atomicExch(err, kErrStall);
                return sum;
            }
            if (use_pre) {
#pragma unroll
                for (int k = 0; k < PER_LANE; ++k) v[k] = pre[k];
                use_pre = false;
            } else {
                lookback_load<PER_LANE>(st, hi, first, v);
                if (dbg && lane == 0) atomicAdd(dbg, 1ull);
            }
            unsigned long long part;
            const int r = lookback_eval<PER_LANE, SEG>(v, vmask, part);
            if (r == 0) continue;
            sum += part;
            if (r == 1) return sum;
            break;
        }
        hi -= 32 * PER_LANE;
        use_pre = false;
    }
    return sum;
}

// Look-back that first polls the nearest 32 predecessors (one status word per lane, backing
// off while one is unpublished) and widens to WIDE words per lane only past them.
template <int WIDE>
__device__ __forceinline__ unsigned long long lookback_adaptive(const unsigned long long* st, int64_t t,
                                                                unsigned long long vmask, int32_t* err)
{
    for (uint32_t spins = 0;; ++spins) {
        if (spins > (1u << 22)) {
            if ((threadIdx.x & 31) == 0) atomicExch(err, kErrStall);
            return 0;
        }
        unsigned long long v[1], part;
        lookback_load<1>(st, t - 1, 0, v);
        const int r = lookback_eval<1, false>(v, vmask, part);
        if (r == 1) return part;
        if (r == 2) return part + lookback_wide<WIDE, false>(st, t - 32, 0, vmask, err);
        __nanosleep(128);
    }
}

// Non-blocking attempt on a window loaded earlier (lookback_load(st, t-1, first, v)).
template <int PER_LANE>
__device__ __forceinline__ bool lookback_try(const unsigned long long* st, int64_t t, int64_t first,
                                             unsigned long long vmask, int32_t* err,
                                             const unsigned long long (&v)[PER_LANE], unsigned long long& out,
                                             unsigned long long* dbg = nullptr)
{
    unsigned long long part;
    const int r = lookback_eval<PER_LANE, false>(v, vmask, part);
    if (r == 0) return false;
    if (r == 2) part += lookback_wide<PER_LANE, false>(st, t - 32 * PER_LANE, first, vmask, err);
    out = part;
    return true;
}


// 16-byte streaming load of the read-only field.
__device__ __forceinline__ float4 ldg_f4(const float* p)
{
    return __ldg(reinterpret_cast<const float4*>(p));
}

// ------------------------------------------------------------------------------------
// 32x32 bit transpose across an 8-lane group (C5).
// Lane k (= lane & 7) of the group holds words v[4k+i], i = 0..3, of one 32-word row
// (row c of A for the shuffle, column c of O for the un-shuffle).  Afterwards lane k
// holds T[4k+i] with T[r] bit j = v[j] bit r.  Each stage swaps word-index bit s with
// bit-position bit s; stages commute.  Stages 16/8/4 cross lanes (shfl_xor 4/2/1),
// stages 2/1 stay in registers.  ~6.5 ALU + 1.5 SHFL lane-ops per element.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ void xpose_pair(uint32_t& lo, uint32_t& hi, int s, uint32_t m)
{
    uint32_t t = ((lo >> s) ^ hi) & m;
    hi ^= t;
    lo ^= t << s;
}

// (a & c) | (b & ~c) as one LOP3 (the compiler splits it when c is lane-dependent).
__device__ __forceinline__ uint32_t bitsel(uint32_t a, uint32_t b, uint32_t c)
{
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

__device__ __forceinline__ void transpose32_group8(uint32_t (&a)[4], int k)
{
#pragma unroll
    for (int st = 0; st < 3; ++st) {
        const int s = 16 >> st;
        const int lm = s >> 2;
        const uint32_t m = st == 0 ? 0x0000FFFFu : (st == 1 ? 0x00FF00FFu : 0x0F0F0F0Fu);
        const bool lower = (k & lm) == 0;
        const uint32_t keep = lower ? m : ~m;
        const int rot = lower ? s : 32 - s;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            uint32_t p = __shfl_xor_sync(kFull, a[i], lm);
            // lower: (a & m) | ((p << s) & ~m); upper: (a & ~m) | ((p >> s) & m).
            // A rotate puts the wanted bits in place; wrapped bits fall in the kept field.
            uint32_t r = __funnelshift_l(p, p, rot);
            a[i] = bitsel(a[i], r, keep);
        }
    }
    xpose_pair(a[0], a[2], 2, 0x33333333u);
    xpose_pair(a[1], a[3], 2, 0x33333333u);
    xpose_pair(a[0], a[1], 1, 0x55555555u);
    xpose_pair(a[2], a[3], 1, 0x55555555u);
}

// ------------------------------------------------------------------------------------
// C1 prequantization, exact nearest bin with ties to even (R1, R3), fp32
// IEEE ops with explicit rounding (no contraction, no fast-math):
//   v = fl(d*r); t = fl(v + 1.5*2^23); q = bits(t) - bits(1.5*2^23); e = fma(-q, w, d)
//   exactly; +-1 correction; then the bound check |fl(fl(q)*w) - d| <= eb (R20).
// Returns q; *vout = value outlier.
// ------------------------------------------------------------------------------------
struct QuantP {
    float w, r, h, eb32, hU;
};

__device__ __forceinline__ int prequant(float d, const QuantP& P, bool& vout)
{
    const float kMagic = 12582912.0f;   // 1.5 * 2^23
    float v = __fmul_rn(d, P.r);
    bool big = fabsf(v) >= 4194302.0f;  // 2^22 - 2: magic rounding no longer exact
    float t = __fadd_rn(v, kMagic);
    int q = __float_as_int(t) - 0x4B400000;
    float qf = __fsub_rn(t, kMagic);
    float e = __fmaf_rn(-qf, P.w, d);   // exact residual d - q*w
    int adj = (e > P.h) - (e < -P.h);
    if (fabsf(e) == P.h && (q & 1)) adj = e > 0.0f ? 1 : -1;
    q += adj;
    bool toolarge = big || (q >= 2097152) || (q <= -2097152);   // |q| >= 2^21
    if (toolarge) q = 0;
    float qq = __fsub_rn(__int_as_float(q + 0x4B400000), kMagic);   // exact fl32(q)
    float xh = __fmul_rn(qq, P.w);
    float diff = __fsub_rn(xh, d);
    vout = toolarge || (fabsf(diff) > P.eb32);
    return q;
}

// Margin-mode fast path: the magic-rounded q is the exact nearest bin whenever the exact
// residual satisfies |e| < w/2 (no tie, no correction); otherwise `hard` is raised and the
// caller re-runs the full rule (rare: d/w within ~|d/w| 2^-23 of a half-integer).
// In margin mode |q| < 2^21 always (Appendix A), so no range checks are needed.
__device__ __forceinline__ int prequant_fast(float d, const QuantP& P, bool& hard, float& qf)
{
    const float kMagic = 12582912.0f;
    float v = __fmul_rn(d, P.r);
    float t = __fadd_rn(v, kMagic);
    qf = __fsub_rn(t, kMagic);
    float e = __fmaf_rn(-qf, P.w, d);
    hard = fabsf(e) >= P.h;
    return __float_as_int(t) - 0x4B400000;
}

// q only (halo elements): identical arithmetic, no bound check.
__device__ __forceinline__ int prequant_q(float d, const QuantP& P)
{
    const float kMagic = 12582912.0f;
    float v = __fmul_rn(d, P.r);
    bool big = fabsf(v) >= 4194302.0f;
    float t = __fadd_rn(v, kMagic);
    int q = __float_as_int(t) - 0x4B400000;
    float qf = __fsub_rn(t, kMagic);
    float e = __fmaf_rn(-qf, P.w, d);
    int adj = (e > P.h) - (e < -P.h);
    if (fabsf(e) == P.h && (q & 1)) adj = e > 0.0f ? 1 : -1;
    q += adj;
    if (big || q >= 2097152 || q <= -2097152) q = 0;
    return q;
}

// ------------------------------------------------------------------------------------
// Parameter derivation (Appendix A, R2/R4/R17), used on the host (fz_derive_params,
// slab API) and on the device (k_params).  Compiled with --fmad=false on the device and
// -ffp-contract=off on the host: every f64 op is one IEEE rounding on both sides.
// ------------------------------------------------------------------------------------
__host__ __device__ inline float rd32(double t)
{
    float f = (float)t;
    if ((double)f > t) f = nextafterf(f, -INFINITY);
    return f;
}

// ------------------------------------------------------------------------------------
// f3 log transform, reading R25: ln and exp as fixed binary64 operation sequences
// (every op one IEEE rounding: --fmad=false on the device, -ffp-contract=off on the host),
// rounded once to binary32 -- a defined function, so the decoder's exp and every rank's log
// agree bit for bit.  ln 2 is split (Cody-Waite): k * kLn2Hi is exact for |k| < 2^11.
// ------------------------------------------------------------------------------------
constexpr double kLn2Hi = 6.93147180369123816490e-01;
constexpr double kLn2Lo = 1.90821492927058770002e-10;
constexpr double kInvLn2 = 1.4426950408889634074;

// ln v (v > 0 finite) = e ln2 + 2 atanh(s): v = m 2^e, m in [sqrt(1/2), sqrt(2)),
// s = (m - 1) / (m + 1), 2 atanh(s) = 2 s sum_{k=0}^{11} s^{2k} / (2k + 1) (Horner from k = 11
// with fused multiply-adds, coefficients rounded once by constant folding)
__host__ __device__ inline double log64(double v)
{
    int e;
    double m = frexp(v, &e);
    if (m < 0.70710678118654752440) { m = m * 2.0; e = e - 1; }
    const double s = (m - 1.0) / (m + 1.0), z = s * s;
    double p = 1.0 / 23.0;
    p = fma(p, z, 1.0 / 21.0);
    p = fma(p, z, 1.0 / 19.0);
    p = fma(p, z, 1.0 / 17.0);
    p = fma(p, z, 1.0 / 15.0);
    p = fma(p, z, 1.0 / 13.0);
    p = fma(p, z, 1.0 / 11.0);
    p = fma(p, z, 1.0 / 9.0);
    p = fma(p, z, 1.0 / 7.0);
    p = fma(p, z, 1.0 / 5.0);
    p = fma(p, z, 1.0 / 3.0);
    p = fma(p, z, 1.0 / 1.0);
    return (double)e * kLn2Hi + ((double)e * kLn2Lo + 2.0 * s * p);
}

// exp t = 2^k e^r, k = rint(t / ln2), r = (t - k ln2_hi) - k ln2_lo, e^r = sum_{n<=17} r^n/n!
// by Horner steps p = fma(p, r, 1/n!) (coefficients rounded once by constant folding)
__host__ __device__ inline double exp64(double t)
{
    const double k = rint(t * kInvLn2);
    const double r = (t - k * kLn2Hi) - k * kLn2Lo;
    double p = 1.0 / 355687428096000.0;
    p = fma(p, r, 1.0 / 20922789888000.0);
    p = fma(p, r, 1.0 / 1307674368000.0);
    p = fma(p, r, 1.0 / 87178291200.0);
    p = fma(p, r, 1.0 / 6227020800.0);
    p = fma(p, r, 1.0 / 479001600.0);
    p = fma(p, r, 1.0 / 39916800.0);
    p = fma(p, r, 1.0 / 3628800.0);
    p = fma(p, r, 1.0 / 362880.0);
    p = fma(p, r, 1.0 / 40320.0);
    p = fma(p, r, 1.0 / 5040.0);
    p = fma(p, r, 1.0 / 720.0);
    p = fma(p, r, 1.0 / 120.0);
    p = fma(p, r, 1.0 / 24.0);
    p = fma(p, r, 1.0 / 6.0);
    p = fma(p, r, 1.0 / 2.0);
    p = fma(p, r, 1.0 / 1.0);
    p = fma(p, r, 1.0 / 1.0);
    return ldexp(p, (int)k);
}

__host__ __device__ inline float log32(float x) { return (float)log64((double)x); }

__host__ __device__ inline float exp32(float y)
{
    double v = exp64((double)y);
    if (v > 3.4028234663852886e38) v = 3.4028234663852886e38;   // FLT_MAX (x^ stays finite)
    return (float)v;
}

// R25: the ABS bound on y = log32(x) that keeps |exp32(y^) - x| <= eps |x|: with
// |y^ - y| <= b, |y - ln x| <= U/4 (binary32 rounding of y, |y| <= M) and the binary32
// rounding of exp (relative 2^-24, plus 2^-45 for the binary64 evaluations),
// b = min(ln((1+eps)/(1+k)), -ln((1-eps)/(1-k))) - U/4 - 2^-40, k = 2^-24 + 2^-45.
__host__ __device__ inline double pwrel_eb(double eps, float M)
{
    if (!(eps > 0.0) || !(eps < 1.0)) return 0.0;
    const double k = ldexp(1.0, -24) + ldexp(1.0, -45);
    double U = 0.0;
    if (M > 0.0f) {
        int e;
        frexp((double)M, &e);
        U = ldexp(1.0, e - 23);
    }
    const double up = log64((1.0 + eps) / (1.0 + k)), lo = -log64((1.0 - eps) / (1.0 - k));
    return (up < lo ? up : lo) - U / 4.0 - ldexp(1.0, -40);
}

__host__ __device__ inline int derive_params(float mn, float mx, int mode, double eb,
                                             fz_params* p)
{
    if (!(eb > 0.0) || !isfinite(eb)) return FZ_ERR_ARG;
    if (mode != FZ_EB_ABS && mode != FZ_EB_REL && mode != FZ_EB_PWREL) return FZ_ERR_ARG;
    if (mode == FZ_EB_PWREL && !(eb < 1.0)) return FZ_ERR_ARG;
    float M = fmaxf(fabsf(mn), fabsf(mx));
    double eb_abs = eb;
    if (mode == FZ_EB_REL && !(mx == mn)) eb_abs = eb * ((double)mx - (double)mn);
    if (mode == FZ_EB_PWREL) eb_abs = pwrel_eb(eb, M);
    if (!(eb_abs > 0.0) || !isfinite(eb_abs)) return FZ_ERR_EB_TOO_SMALL;
    double U = 0.0;
    if (M > 0.0f) {
        int e;
        frexp((double)M, &e);
        U = ldexp(1.0, e - 23);
    }
    float w = rd32(2.0 * eb_abs - U);
    uint32_t fallback = 0;
    if (!(w > 0.0f && (double)M * (1.0 / (double)w) < 2097151.0)) {
        fallback = 1;
        w = rd32(2.0 * eb_abs);
    }
    if (!(w >= 1.17549435e-38f)) return FZ_ERR_EB_TOO_SMALL;
    p->eb_input = eb;
    p->eb_abs = eb_abs;
    p->w = w;
    p->r = (float)(1.0 / (double)w);
    p->eb32 = rd32(eb_abs);
    p->mn = mn;
    p->mx = mx;
    p->mode = (uint32_t)mode;
    p->fallback = fallback;
    return FZ_OK;
}

// ------------------------------------------------------------------------------------
// h = w/2; hU = RD32(w/2 - U) with U = 2^(e-23), M = max|d| = m 2^e (Appendix A): the
// fast-path threshold of pq_fast.  Fallback mode: hU = -1 (every element takes the exact
// rule and the bound check).
// h = w/2 and the fast-path threshold hU = RD32(w/2 - U) (-1: fast path off, fallback mode).
__device__ inline void quant_consts(const fz_params& p, float& h, float& hU)
{
    h = 0.5f * p.w;
    if (p.fallback) {
        hU = -1.0f;
        return;
    }
    const float M = fmaxf(fabsf(p.mn), fabsf(p.mx));
    double U = 0.0;
    if (M > 0.0f) {
        int e;
        frexp((double)M, &e);
        U = ldexp(1.0, e - 23);
    }
    const double t = (double)h - U;
    hU = t > 0.0 ? rd32(t) : -1.0f;
}

__device__ inline void set_quant_consts(Ctrl* ctrl)
{
    quant_consts(ctrl->p, ctrl->h, ctrl->hU);
}

// Appendix-A parameters from the range pass's result (k_params and the ws-kernel prologue).
__device__ inline int params_from_range(const Ctrl* ctrl, int mode, double eb, uint64_t n, fz_params* p)
{
    if (ctrl->first_bad != ~0ull) return FZ_ERR_NONFINITE;
    const float mn = n ? ord2f(ctrl->mn_enc) : 0.0f;
    const float mx = n ? ord2f(ctrl->mx_enc) : 0.0f;
    return derive_params(mn, mx, mode, eb, p);
}

// ------------------------------------------------------------------------------------
// Named barriers, mbarriers and 1-D TMA bulk copies (cp.async.bulk).
// ------------------------------------------------------------------------------------
__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ int bar_or(int id, int n, int pred)
{
    int r;
    asm volatile("{ .reg .pred p, q; setp.ne.s32 p, %1, 0; bar.red.or.pred q, %2, %3, p; selp.s32 %0, 1, 0, q; }"
                 : "=r"(r) : "r"(pred), "r"(id), "r"(n) : "memory");
    return r;
}
// PDL (launch_pdl): wait for the stream predecessors, then let the successor launch.  A no-op
// for a kernel launched without the attribute.
__device__ __forceinline__ void pdl_begin()
{
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* m, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
// try_wait with a suspend-time hint (ns): the thread stays parked until the phase completes
// or the hint elapses, instead of returning after the default short timeout.
__device__ __forceinline__ bool mbar_try_wait_sleep(uint64_t* m, uint32_t parity, uint32_t ns)
{
    uint32_t ok;
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(smem_u32(m)), "r"(parity), "r"(ns) : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* m)
{
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(m)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* m, uint32_t parity)
{
    uint32_t ok;
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(smem_u32(m)), "r"(parity) : "memory");
    return ok != 0;
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* m)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(m)) : "memory");
}

constexpr int kRingBlocks = 1024;   // 16 KB elastic payload ring (per-tile allocation)
constexpr int kDescQ = 8;          // unit descriptors in flight to the scanner

// ------------------------------------------------------------------------------------
// Kernel argument bundles.
// ------------------------------------------------------------------------------------
struct Geom {
    uint32_t n;       // global N
    uint32_t nx;      // x extent (1-D: N)
    uint32_t P;       // plane size (1-D/2-D: N)
    uint32_t ndim;
};

struct CompressArgs {
    const float* field;       // element g at field[g - base]
    uint64_t base;
    Geom g;
    FastDiv dnx, dP;          // x extent, plane size
    uint32_t sx, sp;          // 2048 mod nx, 2048 mod P: per-tile position increments
    uint32_t tile_begin, tile_end;
    // neighbour streams (SV §7 hard part 3): q of the element and of its y-1, z-1, (y-1,z-1)
    // neighbours live in shared arrays; union = [s-nx-1, e) and [s-P-nx-1, e-P)
    int union_mode;           // 1: one array per plane; 0: one 2049-element array per stream
    uint32_t qstride;         // padded words per shared q array (vec: ring size, a power of 2)
    uint32_t qwords;          // words of shared q storage before the shuffle buffer
    uint8_t* flags_out;       // 32 B per tile, tile t at (t - tile_begin) * 32
    uint8_t* payload_out;     // 16 B blocks
    uint64_t flags_cap;       // bytes writable at flags_out
    uint64_t payload_cap;     // bytes writable at payload_out
    uint2* dstage;            // (idx, delta) records
    uint2* vstage;            // (idx, bits) records
    uint64_t dcap, vcap;      // staging capacities (records)
    unsigned long long* status;
    uint2* ocnt;              // per-tile (n_delta, n_value)
    uint2* obase;             // per-tile staging offsets
    const uint2* opre;        // rescan: per-tile final (exclusive) outlier offsets
    Ctrl* ctrl;
    uint16_t* codes_out;      // debug hook: codes at element index (may be null)
    uint32_t* o_didx;         // rescan into split lists (debug hook), else records
    int32_t* o_dval;
    uint32_t* o_vidx;
    uint32_t* o_vbits;
    int rescan;               // 1: outliers only, straight to final offsets via opre
    // ws kernel only: parameters derived in the prologue from k_range's result (replaces
    // k_params) and totals + header written by the last CTA to finish (replaces k_finalize)
    int derive, finalize;
    int eb_mode;
    double eb;
    uint8_t* hdr_out;         // 128-byte header destination (null: totals only)
    uint64_t hdr_cap;         // bytes writable at hdr_out (whole stream capacity)
    uint64_t dims[3];
    uint32_t ndim;
    uint64_t n_hdr, T_hdr;    // field size and tiles for the totals / header
    uint4* tstage;            // z-band pass 1: 256-block staging slot per tile (null: not available)
    uint32_t hwords;          // z-band: floats of the TMA-staged row halo (0: quantized from global)
    uint32_t cl;              // f1 chunk-local Lorenzo (z-band kernel only): chunks of kZbChunk planes x one tile
    uint32_t fuse_range;      // row walker: C0 (range) as the kernel's first phase (no k_range launch)
    int exp;                  // variant bits (fz_debug_set_variant), bit 16: generic kernel instead of the warp-specialized one
    // row-codes path (fz_rowcodes.cu): the code field (T x 2048 u16) and the two outlier bit
    // masks (value, delta; one bit per element, rc_dmask = rc_vmask + rc_mask_words)
    uint16_t* rc_codes;
    uint32_t* rc_vmask;
    uint32_t* rc_dmask;
};

}  // namespace fz
