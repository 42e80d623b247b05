// fz_zrow.cu -- the row-walking z-band compressor (C1-C6 fused, pass 1 of the 3-D path).
//
// Shapes: 3-D, nx % 128 == 0, nx <= 1024, ny % 16 == 0 (so every band of 16 rows is
// nx / 128 whole tiles and every plane a whole number of tiles).  Citation key: P:n =
// PAPER.md line n; R# = DESIGN.md §3 readings; SV = SURVEY.md.
//
// Work decomposition.  A band is 16 consecutive rows of one plane (16 nx elements = nx/128
// tiles).  A CTA of nx/128 warps walks a run of consecutive planes of one band (a persistent
// CTA takes an equal share of all (band, plane) steps, in band-major order, so a share is one
// or two runs).  In every plane:
//
//  phase A (coalesced, registers only): warp w owns the 128 columns [128w, 128w + 128) of
//   the band, lane L the 4 columns x0 = 128w + 4L, and walks the 16 rows.  Per row it loads
//   the 4 floats (one 16-byte load, consecutive lanes = consecutive addresses), prequantizes
//   them (C1: magic-rounded q by one FFMA, exact residual, exact rule only on the rare hard
//   elements), and builds the Lorenzo residual (C2) from
//       Z = q(z) - q(z-1)          (q(z-1) of the thread's 64 elements carried in registers)
//       Y = Z - Z(y-1)             (the previous row's Z, carried in registers)
//       delta = Y - Y(x-1)         (x-1 by SHFL; lane 0 takes it from a "shadow" column)
//   In-register values are the float bit patterns t = q + 0x4B400000 of the magic rounding:
//   the Lorenzo signs sum to zero, so differences of t are differences of q.  Codes (C3:
//   sign-magnitude by IABS/PRMT/LOP3) go two per word (C4) into a shared code buffer
//   laid out by A-row (64 codes) with 16 bytes of padding per A-row.
//  phase B (one warp per tile): lane c loads A-row c of the warp's tile (8 conflict-free
//   128-bit loads), bit-transposes its 32 words in registers (C5: O[r][c] =
//   transpose32(A[c])[r]; byte and half-word stages by PRMT), stages O row-major in shared
//   memory, and emits flag word f (C6: block 32f + c nonzero <=> any of O words
//   4(32f+c)..+3) by one ballot per f; each nonzero block goes to the tile's staging slot at
//   its rank within flag word f (the layout k_compact reads).
//
// The row above the band (halo) is prequantized in every plane (1/16 extra), the shadow
// column x = 128w - 1 (17 elements per plane, lanes 0..16) gives lane 0 its Y(x-1).  A run
// that starts at plane z0 > 0 first prequantizes plane z0 - 1 (the z carry).  Outliers
// (R7 delta-outliers, R20 value outliers) are rare: marked in the A-row padding in phase A,
// recorded per tile in phase B (delta recomputed exactly from the field).  One CTA barrier
// per plane (the code buffer is double-buffered).
#include "fz_internal.cuh"
#include "fz_launch.h"
#include "fz_rowwalk.cuh"

#include <cfloat>
#include <cstdio>
#include <cstdlib>

namespace fz {

constexpr int kZrRows = 16;              // band height
constexpr uint32_t kMagicBits = 0x4B400000u;
constexpr int kZrStages = 2;             // TMA stages (field rows of one step each)

// Exact t-bits (q + magic) of the element at global index g (prequant: exact rule, R1-R3).
__device__ __forceinline__ uint32_t zr_texact(const CompressArgs& a, const QuantP& P, uint64_t g, bool& vo)
{
    const float d = __ldg(a.field + (g - a.base));
    return (uint32_t)prequant(d, P, vo) + kMagicBits;
}

// Exact q of the element at (z, y, x) with zero outside the field / outside its chunk.
__device__ int32_t zr_q(const CompressArgs& a, const QuantP& P, int64_t z, int64_t y, int64_t x, int64_t zc,
                        int64_t yc, uint32_t cz, uint32_t cy)
{
    if (z < 0 || y < 0 || x < 0) return 0;
    if (cz && (z < zc || y < yc)) return 0;   // f1: a neighbour in another chunk counts as 0
    bool vo;
    const uint64_t g = (uint64_t)z * a.g.P + (uint64_t)y * a.g.nx + (uint64_t)x;
    return (int32_t)(zr_texact(a, P, g, vo) - kMagicBits);
}

// Lorenzo residual of one element recomputed from the field (rare path: delta-outliers).
__device__ int32_t zr_delta(const CompressArgs& a, const QuantP& P, int64_t z, int64_t y, int64_t x, uint32_t cz,
                            uint32_t cy)
{
    const int64_t zc = cz ? z - z % cz : 0, yc = cy ? y - y % cy : 0;
    uint32_t s = 0;
#pragma unroll 1
    for (int k = 0; k < 8; ++k) {
        const int dz = k >> 2 & 1, dy = k >> 1 & 1, dx = k & 1;
        const uint32_t q = (uint32_t)zr_q(a, P, z - dz, y - dy, x - dx, zc, yc, cz, cy);
        s += ((dz + dy + dx) & 1) ? 0u - q : q;
    }
    return (int32_t)s;
}

// A shared-memory load the compiler may not merge with an earlier load of the same address
// (volatile), and that stays ordered before later stores to it (it is a visible load).
__device__ __forceinline__ void lds_u4_volatile(const uint8_t* p, uint32_t (&v)[4])
{
    const volatile uint4* q = reinterpret_cast<const volatile uint4*>(p);
    v[0] = q->x; v[1] = q->y; v[2] = q->z; v[3] = q->w;
}

struct ZrShared {
    QuantP P;
    fz_params p;
    int perr;
    uint32_t tmem;   // TMEM base address (tcgen05.alloc)
};

// Prequantize 4 values: t-bits by the fast path; the exact rule when any is hard.
// vbits (own elements only): value-outlier flags in bits 0..3.
template <bool OWN>
__device__ __forceinline__ void zr_quant4(const float4 dv, const QuantP& P, uint32_t (&t)[4], uint32_t& vbits)
{
    const float kMagic = 12582912.0f;   // 1.5 * 2^23
    const float d[4] = {dv.x, dv.y, dv.z, dv.w};
    bool hard = false;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        // q0 = rint(d * r) by one rounding of d * r + 1.5 * 2^23 (|d r| < 2^22 in margin
        // mode); the exact residual e = d - q0 w decides: |e| < hU => q0 is the unique
        // nearest bin and the bound holds (R3, SV App. A) -- however q0 was rounded
        const float tf = __fmaf_rn(d[k], P.r, kMagic);
        const float qf = __fsub_rn(tf, kMagic);
        const float e = __fmaf_rn(-qf, P.w, d[k]);
        hard |= !(fabsf(e) < P.hU);
        t[k] = __float_as_uint(tf);
    }
    vbits = 0;
    if (__builtin_expect(hard, 0)) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            bool vo;
            t[k] = (uint32_t)prequant(d[k], P, vo) + kMagicBits;
            if (OWN && vo) vbits |= 1u << k;
        }
    }
}

// Two sign-magnitude codes per word (C3/C4): magnitudes by PRMT, both signs (bit 31 of each
// delta -> bits 15 and 31) by a second PRMT, merged by one LOP3.  |delta| > 32767 is caught
// by the caller through `mag` (OR of the magnitudes).
__device__ __forceinline__ uint32_t zr_pack2(int32_t d0, int32_t d1, uint32_t& mag)
{
    const uint32_t m0 = (uint32_t)abs(d0), m1 = (uint32_t)abs(d1);
    mag |= m0 | m1;
    return bitsel(__byte_perm((uint32_t)d0, (uint32_t)d1, 0x7030u), __byte_perm(m0, m1, 0x5410u), 0x80008000u);
}

// Step sequence of a CTA: its share [u0, u1) of the (band, plane) units, band-major, with a
// seed step (plane z - 1, prequantized only) before every run that starts inside the field
// (or inside an f1 chunk).  Two cursors walk it: the TMA issuer (thread 0, ahead) and the
// processing loop.
struct ZrCursor {
    uint64_t u;
    uint32_t band, zo;   // u = band * nzr + zo, tracked incrementally (no 64-bit division)
    bool seeded;         // the current run's seed step was returned already
};
struct ZrStep {
    uint32_t band, z;
    bool seed, run_start, valid;
};
__device__ __forceinline__ ZrCursor zr_cursor(uint64_t u0, uint32_t nzr)
{
    return ZrCursor{u0, (uint32_t)(u0 / nzr), (uint32_t)(u0 % nzr), false};
}
__device__ __forceinline__ ZrStep zr_next(ZrCursor& c, uint64_t u0, uint64_t u1, uint32_t nzr, uint32_t zbeg,
                                          bool cl, uint32_t cz)
{
    ZrStep s{0, 0, false, false, false};
    if (c.u >= u1) return s;
    s.valid = true;
    s.band = c.band;
    s.z = zbeg + c.zo;
    const bool start = c.u == u0 || c.zo == 0;
    if (start && !c.seeded && s.z > 0 && !(cl && s.z % cz == 0)) {
        c.seeded = true;
        s.seed = true;
        s.run_start = true;
        s.z -= 1;
        return s;
    }
    s.run_start = start && !c.seeded;
    c.seeded = false;
    ++c.u;
    if (++c.zo == nzr) { c.zo = 0; ++c.band; }
    return s;
}

// A0: the t-bits of G stage rows r0..r0+G-1 (row 0 = halo), in place, exact: the fast path
// for all, the exact rule (prequant) for the lanes of a group with a hard element (one warp
// vote per group), value-outlier marks for own rows (1..16).
// Out of line (cold, keeps the hot loop small for the instruction cache): the t-bits of G
// stage rows from their floats with the exact rule (R1-R3, R20) wherever the fast path does
// not apply, value-outlier marks for own rows (1..16).
__device__ __noinline__ void zr_tgroup_slow(uint8_t* stg, uint8_t* msk, uint32_t RP, uint32_t spr, int r0, int G,
                                            int tid, int lane, int warp, QuantP P)
{
    const float kMagic = 12582912.0f;
#pragma unroll 1
    for (int g = 0; g < G; ++g) {
        uint32_t* row = reinterpret_cast<uint32_t*>(stg + (r0 + g) * RP + 16u * tid);
        uint32_t vb = 0;
#pragma unroll 1
        for (int k = 0; k < 4; ++k) {
            const float d = __uint_as_float(row[k]);
            const float tf = __fmaf_rn(d, P.r, kMagic);
            const float qf = __fsub_rn(tf, kMagic);
            uint32_t t = __float_as_uint(tf);
            if (!(fabsf(__fmaf_rn(-qf, P.w, d)) < P.hU)) {
                bool vo;
                t = (uint32_t)prequant(d, P, vo) + kMagicBits;
                if (vo) vb |= 1u << k;
            }
            row[k] = t;
        }
        const int r = r0 + g;
        // own rows only (row 0 is the halo); no marks in a seed step (msk == null): its plane
        // is not encoded, and stale marks would reach the stage's next phase B
        if (vb && r >= 1 && msk != nullptr) {
            const uint32_t seg = 2u * warp + (lane >> 4);
            atomicOr(reinterpret_cast<unsigned long long*>(msk + 16 * ((r - 1) * spr + seg)),
                     (unsigned long long)vb << (4 * (lane & 15)));
        }
    }
}

// A0: the t-bits of G stage rows r0..r0+G-1 (row 0 = halo), in place.  The fast path for all
// (one FFMA + FADD + FFMA + FSETP per element).  A hard element (|e| >= w/2) in margin mode
// is corrected inline from its exact residual e = d - q0 w (|q0 - d/w| <= 1/2 + 1/8, so one
// step reaches the nearest bin; |e| = w/2 is a tie -> even, R1); margin mode has no value
// outliers (|fl(q w) - d| <= |e| + U/2 <= eb for |e| <= w/2, SV App. A) and |q| < 2^21.
// Fallback mode (hU < 0) takes the full exact rule with the bound check out of line.
template <int G>
__device__ __forceinline__ void zr_tgroup(uint8_t* stg, uint8_t* msk, uint32_t RP, uint32_t spr, int r0, int tid,
                                          int lane, int warp, const QuantP& P)
{
    const float kMagic = 12582912.0f;
    // |e| < w/2 suffices in margin mode: q0 is then the unique nearest bin and
    // |fl(q0 w) - d| < w/2 + U/2 <= eb (SV App. A), so the threshold is h, not h - U;
    // fallback mode (hU < 0) sends every element to the exact rule
    const float thr = P.hU < 0.0f ? -1.0f : P.h;
    float dv[G][4];
    uint32_t t[G][4];
    bool hard = false;
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const float4 d = *reinterpret_cast<const float4*>(stg + (r0 + g) * RP + 16u * tid);
        dv[g][0] = d.x; dv[g][1] = d.y; dv[g][2] = d.z; dv[g][3] = d.w;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            // q0 = rint(d r) by one rounding of d r + 1.5 2^23 (|d r| < 2^22 in margin mode);
            // the exact residual e = d - q0 w decides: |e| < hU => q0 is the unique nearest
            // bin and the bound holds (R3, SV App. A), however q0 was rounded
            const float tf = __fmaf_rn(dv[g][k], P.r, kMagic);
            const float qf = __fsub_rn(tf, kMagic);
            const float e = __fmaf_rn(-qf, P.w, dv[g][k]);
            hard |= !(fabsf(e) < thr);
            t[g][k] = __float_as_uint(tf);
        }
    }
    if (__any_sync(kFull, hard)) {   // rare
        if (P.hU < 0.0f) {           // fallback mode: exact rule + bound check for every element
            zr_tgroup_slow(stg, msk, RP, spr, r0, G, tid, lane, warp, P);
            __syncwarp();
            return;
        }
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float qf = __fsub_rn(__uint_as_float(t[g][k]), kMagic);
                const float e = __fmaf_rn(-qf, P.w, dv[g][k]);   // exact residual
                const float ae = fabsf(e);
                const bool step = ae > P.h || (ae == P.h && (t[g][k] & 1u));
                t[g][k] += step ? (e > 0.0f ? 1u : 0xFFFFFFFFu) : 0u;
            }
    }
#pragma unroll
    for (int g = 0; g < G; ++g)
        *reinterpret_cast<uint4*>(stg + (r0 + g) * RP + 16u * tid) = make_uint4(t[g][0], t[g][1], t[g][2], t[g][3]);
}

__device__ __forceinline__ void zr_tpass(uint8_t* stg, uint8_t* msk, uint32_t RP, uint32_t spr, bool halo, int tid,
                                         int lane, int warp, const QuantP& P)
{
    if (halo) zr_tgroup<1>(stg, msk, RP, spr, 0, tid, lane, warp, P);
    // two groups of 4 rows per call: the compiler may then interleave their loads
#pragma unroll
    for (int r0 = 1; r0 <= kZrRows; r0 += 8) zr_tgroup<8>(stg, msk, RP, spr, r0, tid, lane, warp, P);
}

// C0 (R4, R18) fused into the row walker as its first phase (SV §8.f2, "fusing
// all GPU kernels into one"): the field's min / max and first non-finite index, then a
// grid-wide wait, then the walk with the parameters every CTA derives from the result.
// The unit of work is half a step's own rows (8 rows of a band in one plane: contiguous,
// 32 nx bytes), copied by 1-D TMA into kZrRStages buffers carved from the walk's stages.
// Chunks are CLAIMED from a global counter (batches of kZrRClaim = 2: 8 left a longer tail at
// the wait, 1 cost more atomic round trips) instead of being assigned
// by blockIdx, so the wait cannot deadlock when fewer CTAs are resident than launched
// (another stream's kernels on the SMs): every claimed chunk is held by a running CTA.
// Claim order j -> chunk: position-major from the END of the compression runs (half-step
// pos = 2L - 1 - j / G of run r = j % G), so the chunks read last -- the ones L2 still holds
// at the wait -- are the first steps of every run of the walk.
constexpr int kZrRStages = 4;

// debug trace (variant 8388608): per CTA (start, smid, range-phase end, end) in globaltimer ns
__device__ unsigned long long g_zr_trace[4 * 2048];
constexpr uint32_t kZrRClaim = 2;

__device__ __noinline__ void zr_range_phase(const float* field, Ctrl* ctrl, uint8_t* zsm, uint64_t* mbar,
                                            int* ids, uint32_t nx, uint32_t PL, uint32_t nzr, uint32_t zbeg,
                                            uint32_t U, bool natural)
{
    const int tid = threadIdx.x, nthr = blockDim.x;
    const uint32_t G = gridDim.x, L2 = 2u * ((U + G - 1) / G), J = L2 * G;
    const uint32_t cbytes = (kZrRows / 2) * 4u * nx;   // half a step's own rows
    uint32_t jb = 0, je = 0;                          // thread 0: the claimed batch [jb, je)
    // next valid chunk (half-step index 2u + h), or -1 when every chunk is claimed
    auto claim = [&]() -> int {
        for (;;) {
            if (jb == je) {
                jb = atomicAdd(&ctrl->rclaim, kZrRClaim);
                je = jb + kZrRClaim;
            }
            if (jb >= J) return -1;
            const uint32_t j = jb++;
            if (natural) {   // A/B (variant 4194304): chunks in address order
                if (j < 2u * U) {
                    const uint32_t m = j >> 1, nb = U / nzr;
                    return (int)(2u * ((m % nb) * nzr + m / nb) + (j & 1u));
                }
                continue;
            }
            const uint32_t pos = L2 - 1u - j / G, r = j % G;
            const uint32_t a0 = (uint32_t)((uint64_t)U * r / G), a1 = (uint32_t)((uint64_t)U * (r + 1) / G);
            if (a0 + pos / 2 < a1) return (int)(2u * (a0 + pos / 2) + (pos & 1u));
        }
    };
    auto src_of = [&](int c) -> const float* {
        const uint32_t u = (uint32_t)c >> 1, band = u / nzr, z = zbeg + u % nzr;
        return field + (uint64_t)z * PL + ((uint64_t)band * kZrRows + (uint64_t)(c & 1) * (kZrRows / 2)) * nx;
    };
    auto issue = [&](int c, uint32_t s) {
        mbar_expect_tx(&mbar[s], cbytes);
        tma_load_1d(zsm + s * cbytes, src_of(c), cbytes, &mbar[s]);
    };
    if (tid == 0) {
        for (uint32_t s = 0; s < (uint32_t)kZrRStages; ++s) {
            const int c = claim();
            ids[s] = c;
            if (c >= 0) issue(c, s);
        }
    }
    __syncthreads();
    float lo = INFINITY, hi = -INFINITY;
    unsigned long long bad = ~0ull;
    uint32_t done = 0;
    const uint32_t nv = cbytes / 16;
    for (uint32_t k = 0;; ++k) {
        const uint32_t s = k % kZrRStages;
        const int c = ids[s];   // written by thread 0 before the barrier of iteration k - 3
        if (c < 0) break;
        while (!mbar_try_wait(&mbar[s], (k / kZrRStages) & 1u)) {
        }
        const float4* p = reinterpret_cast<const float4*>(zsm + s * cbytes);
        bool ok = true;
        for (uint32_t i = tid; i < nv; i += nthr) {
            const float4 v = p[i];
            lo = fminf(lo, fminf(fminf(v.x, v.y), fminf(v.z, v.w)));
            hi = fmaxf(hi, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
            ok &= fabsf(v.x) <= FLT_MAX && fabsf(v.y) <= FLT_MAX && fabsf(v.z) <= FLT_MAX && fabsf(v.w) <= FLT_MAX;
        }
        if (!ok) {   // rare: the first non-finite index among this thread's elements
            const uint64_t g0 = (uint64_t)(src_of(c) - field);
            const float* f = reinterpret_cast<const float*>(zsm + s * cbytes);
            for (uint32_t i = tid; i < nv; i += nthr)
                for (uint32_t e = 0; e < 4; ++e)
                    if (!(fabsf(f[4 * i + e]) <= FLT_MAX)) bad = min(bad, (unsigned long long)(g0 + 4 * i + e));
        }
        ++done;
        __syncthreads();   // the buffer is consumed (and ids[s] read by every thread)
        if (tid == 0) {
            const int cn = claim();
            ids[s] = cn;
            if (cn >= 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(cn, s);
            }
        }
    }
    uint32_t elo = f2ord(__fadd_rn(lo, 0.0f)), ehi = f2ord(__fadd_rn(hi, 0.0f));
    if (lo == INFINITY) elo = 0xFFFFFFFFu;
    if (hi == -INFINITY) ehi = 0u;
    elo = __reduce_min_sync(kFull, elo);
    ehi = __reduce_max_sync(kFull, ehi);
    unsigned long long b = bad;
    for (int o = 16; o; o >>= 1) b = min(b, __shfl_xor_sync(kFull, b, o));
    if ((tid & 31) == 0) {
        atomicMin(&ctrl->mn_enc, elo);
        atomicMax(&ctrl->mx_enc, ehi);
        if (b != ~0ull) atomicMin(&ctrl->first_bad, b);
    }
    __syncthreads();   // every read of the buffers is done: they go back to the walk's TMA
    if (tid == 0) {
        __threadfence();
        atomicAdd(&ctrl->rdone, done);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
}

// The grid-wide wait of the fused range phase (thread 0): every chunk's min / max is in ctrl.
__device__ __forceinline__ void zr_range_wait(Ctrl* ctrl, uint32_t U)
{
    uint32_t seen;
    for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(&ctrl->rdone) : "memory");
        if (seen >= 2u * U) break;
        __nanosleep(64);
    }
}

// NW = nx / 128 warps; at most ~170 registers per thread (12 warps per SM).
// Shared memory per stage: 17 rows of the field (row 0 = the band's halo row y0 - 1, rows
// 1..16 = the band) + the A-row outlier masks.  Codes of band row i are written over row i
// (the halo row / band row i - 1, already consumed by the same warp), A-row slot of segment
// (2k + p) at 512 k + 256 p + 16 ((i spr + 2k + p) & 7): 8 consecutive A-rows fall in 8
// distinct 16-byte bank groups, and the last 16 bytes of each warp's 512-byte row segment
// (its right neighbour's shadow element) are never overwritten.
template <int NW, bool CL, int NST>
__global__ void __launch_bounds__(32 * NW, 12 / NW) k_compress_zr(CompressArgs a, uint32_t cz, uint32_t cy)
{
    pdl_begin();
    extern __shared__ __align__(128) uint8_t zsm[];
    __shared__ ZrShared sh;
    __shared__ __align__(8) uint64_t mbar[NST];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    Ctrl* ctrl = a.ctrl;
    if (ctrl->err != 0) return;
    constexpr uint32_t nx = 128u * NW, spr = 2u * NW, RP = 4u * nx;   // row pitch (bytes)
    constexpr uint32_t dbytes = (kZrRows + 1) * RP, mbytes = kZrRows * spr * 16u;
    constexpr uint32_t sbytes = dbytes + mbytes;
    const uint32_t PL = a.g.P;
    const uint32_t tpp = PL / kTileCodes, nbands = PL / nx / kZrRows;
    const uint32_t zbeg = a.tile_begin / tpp, zend = a.tile_end / tpp, nzr = zend - zbeg;
    if ((a.exp & 8388608) && tid == 0 && blockIdx.x < 2048) {
        unsigned long long ts;
        uint32_t smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_zr_trace[4 * blockIdx.x] = ts;
        g_zr_trace[4 * blockIdx.x + 1] = smid;
    }
    // TMEM for the z carry: warp 0 allocates (power-of-two columns) and frees it at the end.
    // First thing: the SM launches its next CTA of this kernel only after this one relinquished
    // the allocation permit (measured: a range phase before it left one CTA per SM resident)
    constexpr uint32_t kTmemCols = NW > 4 ? 256u : 128u;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"(smem_u32(&sh.tmem)), "n"(kTmemCols) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    const uint64_t U = (uint64_t)nbands * nzr;
    const uint64_t u0 = U * blockIdx.x / gridDim.x, u1 = U * (blockIdx.x + 1) / gridDim.x;
    const bool clm = CL;
    // TMA issue of one step into its stage (thread 0): rows y0 - 1 .. y0 + 15 of plane z
    auto issue = [&](const ZrStep& st, uint32_t k) {
        const uint32_t s = k % NST;
        uint8_t* dst = zsm + s * sbytes;
        const uint32_t y0 = st.band * kZrRows;
        const uint64_t g = (uint64_t)st.z * PL + (uint64_t)(y0 > 0 ? y0 - 1 : 0) * nx;
        const uint32_t rows = y0 > 0 ? kZrRows + 1 : kZrRows;
        mbar_expect_tx(&mbar[s], rows * RP);
        tma_load_1d(dst + (y0 > 0 ? 0u : RP), a.field + (g - a.base), rows * RP, &mbar[s]);
    };
    ZrCursor ic = zr_cursor(u0, nzr);   // issue cursor (thread 0 only)
    uint32_t kissue = 0;
    // steps 0 .. NST-2 (thread 0); step k + NST - 1 once step k - 1 is done
    auto issue_first = [&]() {
        for (int s = 0; s + 1 < NST; ++s) {
            const ZrStep st = zr_next(ic, u0, u1, nzr, zbeg, clm, cz);
            if (!st.valid) break;
            issue(st, kissue++);
        }
    };
    if (tid == 0) {
        for (int s = 0; s < NST; ++s) mbar_init(&mbar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (a.fuse_range) {
        __shared__ __align__(8) uint64_t rbar[kZrRStages];
        __shared__ int rids[kZrRStages];
        static_assert(kZrRStages * (kZrRows / 2) <= NST * (kZrRows + 1), "range buffers exceed the stages");
        if (tid == 0) {
            for (int s = 0; s < kZrRStages; ++s) mbar_init(&rbar[s], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        zr_range_phase(a.field, ctrl, zsm, rbar, rids, nx, PL, nzr, zbeg, nbands * nzr, a.fuse_range == 2);
        if (tid == 0) {
            // the walk's first field rows do not depend on the range: in flight during the wait
            issue_first();
            zr_range_wait(ctrl, (uint32_t)U);
        }
        if ((a.exp & 8388608) && tid == 0 && blockIdx.x < 2048) {
            unsigned long long t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            g_zr_trace[4 * blockIdx.x + 2] = t1;
        }
    }
    if (tid == 0) {
        sh.perr = 0;
        if (a.derive) {
            fz_params p;
            int st;
            if (a.fuse_range) {   // other CTAs' atomics: read from L2, not a stale L1 line
                Ctrl rc;
                rc.mn_enc = __ldcg(&ctrl->mn_enc);
                rc.mx_enc = __ldcg(&ctrl->mx_enc);
                rc.first_bad = __ldcg(&ctrl->first_bad);
                st = params_from_range(&rc, a.eb_mode, a.eb, a.n_hdr, &p);
            } else {
                st = params_from_range(ctrl, a.eb_mode, a.eb, a.n_hdr, &p);
            }
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
    }
    // outlier masks start clear (phase B clears them after use)
    for (uint32_t s = 0; s < NST; ++s)
        for (uint32_t o = 16 * tid; o < mbytes; o += 16 * blockDim.x)
            *reinterpret_cast<uint4*>(zsm + s * sbytes + dbytes + o) = make_uint4(0, 0, 0, 0);
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
        // (fused range: the prefetched steps must land before the CTA exits)
        if (tid == 0)
            for (uint32_t k = 0; k < kissue; ++k)
                while (!mbar_try_wait(&mbar[k % NST], (k / NST) & 1u)) {
                }
        tmem_free();
        return;
    }
    const QuantP P = sh.P;
    if (tid == 0 && !a.fuse_range) issue_first();
    const uint32_t x0 = 128u * warp + 4u * lane;
    const bool has_shadow = warp > 0 && lane <= kZrRows;   // shadow column x = 128 w - 1
    ZrCursor pc = zr_cursor(u0, nzr);
    uint32_t th[4], tsh = kMagicBits;
    bool zfirst = true;   // the TMEM carry holds no plane yet (q(z-1) = 0)
    for (uint32_t k = 0;; ++k) {
        const ZrStep st = zr_next(pc, u0, u1, nzr, zbeg, clm, cz);
        if (!st.valid) break;
        const uint32_t s = k % NST;
        uint8_t* stg = zsm + s * sbytes;
        uint8_t* msk = stg + dbytes;
        const uint32_t y0 = st.band * kZrRows, z = st.z;
        // the z carry starts from q = 0 at a run start (a seed step then fills it) and at an
        // f1 chunk's first plane
        if (st.run_start || (CL && !st.seed && z % cz == 0)) {
            zfirst = true;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) th[kk] = kMagicBits;
            tsh = kMagicBits;
        }
        // shadow column x = 128 w - 1, lane j (0..16) = row y0 - 1 + j, read from the field
        // (an L2 hit: the stage's copy belongs to warp w - 1, which rewrites it); issued
        // before the stage wait so that its latency overlaps
        const bool shv = has_shadow && (y0 + lane) > 0 && !(CL && lane == 0 && y0 % cy == 0);
        float dsh = 0.0f;
        if (shv) dsh = __ldg(a.field + ((uint64_t)z * PL + (uint64_t)(y0 + lane - 1) * nx + 128u * warp - 1u - a.base));
        while (!mbar_try_wait(&mbar[s], (k / NST) & 1u)) {
        }
        const bool halo = y0 > 0 && !(CL && y0 % cy == 0);
        // A0: t-bits in place (rows 1..16, and row 0 when the halo row is used)
        zr_tpass(stg, st.seed ? nullptr : msk, RP, spr, halo, tid, lane, warp, P);
        __syncwarp();
        uint32_t tshn = kMagicBits;
        if (shv) {
            bool vo;
            tshn = (uint32_t)prequant(dsh, P, vo) + kMagicBits;
        }
        if (st.seed) {
#pragma unroll 1
            for (int g = 0; g < kZrRows / 4; ++g) {
                uint32_t tv[16];
#pragma unroll
                for (int ii = 0; ii < 4; ++ii) {
                    const uint4 v = *reinterpret_cast<const uint4*>(stg + (4 * g + ii + 1) * RP + 16u * tid);
                    tv[4 * ii] = v.x; tv[4 * ii + 1] = v.y; tv[4 * ii + 2] = v.z; tv[4 * ii + 3] = v.w;
                }
                tmem_st16(taddr + 16u * g, tv);
            }
            tmem_wait_st();
            zfirst = false;
            if (halo) {
                const uint4 tv = *reinterpret_cast<const uint4*>(stg + 16u * tid);
                th[0] = tv.x; th[1] = tv.y; th[2] = tv.z; th[3] = tv.w;
            }
            if (shv) tsh = tshn;
        } else {
            // halo row y0 - 1: its Z is the first row's Z(y-1)
            uint32_t Zup[4] = {0u, 0u, 0u, 0u};
            if (halo) {
                const uint4 tv = *reinterpret_cast<const uint4*>(stg + 16u * tid);
                const uint32_t t[4] = {tv.x, tv.y, tv.z, tv.w};
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) { Zup[kk] = t[kk] - th[kk]; th[kk] = t[kk]; }
            }
            // Ysh of lane i + 1 is row y0 + i's Y at x = 128 w - 1
            uint32_t Ysh;
            {
                uint32_t Zs = 0u;
                if (shv) { Zs = tshn - tsh; tsh = tshn; }
                const uint32_t Zabove = __shfl_up_sync(kFull, Zs, 1);
                const bool ystart = CL ? ((y0 + lane - 1) % cy == 0) : false;
                Ysh = Zs - (ystart ? 0u : Zabove);
            }
            // ---- A1: Lorenzo + codes, 16 rows in groups of 4; z carry in TMEM ----
            uint32_t magor = 0;
            // two carry buffers (the next group's load in flight while one is used)
            uint32_t tpb[2][8];   // two rows of the carry per load, the next pair in flight
            if (zfirst) {   // q(z-1) = 0: the carry starts as the t-bits of q = 0
                uint32_t mg[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) mg[j] = kMagicBits;
#pragma unroll
                for (int g = 0; g < kZrRows / 4; ++g) tmem_st16(taddr + 16u * g, mg);
                tmem_wait_st();
            }
            tmem_ld8(taddr, tpb[0]);
            // t of the next two rows loaded ahead: the compiler cannot move these loads above
            // the code stores (it cannot prove the addresses distinct)
            uint4 tvq[2];
            tvq[0] = *reinterpret_cast<const uint4*>(stg + 1 * RP + 16u * tid);
            tvq[1] = *reinterpret_cast<const uint4*>(stg + 2 * RP + 16u * tid);
#pragma unroll
            for (int i = 0; i < kZrRows; ++i) {
                uint32_t(&tpp)[8] = tpb[(i >> 1) & 1];
                if ((i & 1) == 0) {
                    tmem_wait_ld8(tpp);
                    if (i + 2 < kZrRows) tmem_ld8(taddr + 4u * (i + 2), tpb[((i >> 1) + 1) & 1]);
                }
                const uint32_t* tp = tpp + 4 * (i & 1);
                const uint4 tv = tvq[i & 1];
                if (i + 2 < kZrRows) tvq[i & 1] = *reinterpret_cast<const uint4*>(stg + (i + 3) * RP + 16u * tid);
                const uint32_t t[4] = {tv.x, tv.y, tv.z, tv.w};
                tmem_st4(taddr + 4u * i, t[0], t[1], t[2], t[3]);
                uint32_t Y[4];
                const bool ystart = CL && ((y0 + i) % cy == 0);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint32_t Z = t[kk] - tp[kk];
                    Y[kk] = ystart ? Z : Z - Zup[kk];
                    Zup[kk] = Z;
                }
                uint32_t Yl = __shfl_up_sync(kFull, Y[3], 1);
                const uint32_t ysh = __shfl_sync(kFull, Ysh, i + 1);
                if (lane == 0) Yl = ysh;          // warp 0: Ysh = 0 (x = 0, zero boundary)
                uint32_t mag = 0;
                const uint32_t w0 = zr_pack2((int32_t)(Y[0] - Yl), (int32_t)(Y[1] - Y[0]), mag);
                const uint32_t w1 = zr_pack2((int32_t)(Y[2] - Y[1]), (int32_t)(Y[3] - Y[2]), mag);
                magor |= mag;
                // codes of row i over row i - 1's t (read by this warp one row earlier)
                const uint32_t p = lane >> 4, seg = 2u * warp + p;
                uint8_t* sp = stg + i * RP + 512u * warp + 256u * p + 16u * ((i * spr + seg) & 7u);
                *reinterpret_cast<uint2*>(sp + 8 * (lane & 15)) = make_uint2(w0, w1);
            }
            tmem_wait_st();
            zfirst = false;
            // delta-outliers (R7): code 0 + a mark in the A-row's dmask (value recomputed in B)
            if (__builtin_expect(magor > 32767u, 0)) {
#pragma unroll 1
                for (int i = 0; i < kZrRows; ++i) {
                    const uint32_t p = lane >> 4, seg = 2u * warp + p;
                    uint8_t* sp = stg + i * RP + 512u * warp + 256u * p + 16u * ((i * spr + seg) & 7u);
                    uint2 wv = *reinterpret_cast<uint2*>(sp + 8 * (lane & 15));
                    uint32_t dbits = 0;
#pragma unroll 1
                    for (int kk = 0; kk < 4; ++kk) {
                        const int32_t dl = zr_delta(a, P, z, y0 + i, x0 + kk, CL ? cz : 0u, CL ? cy : 0u);
                        if ((uint32_t)abs(dl) > 32767u) {
                            dbits |= 1u << kk;
                            uint32_t& wd = (kk < 2) ? wv.x : wv.y;
                            wd &= (kk & 1) ? 0x0000FFFFu : 0xFFFF0000u;
                        }
                    }
                    if (dbits) {
                        *reinterpret_cast<uint2*>(sp + 8 * (lane & 15)) = wv;
                        atomicOr(reinterpret_cast<unsigned long long*>(msk + 16 * (i * spr + seg) + 8),
                                 (unsigned long long)dbits << (4 * (lane & 15)));
                    }
                }
            }
        }
        __syncthreads();
        // every warp is done with step k - 1: its stage takes step k + NST - 1
        if (tid == 0) {
            const ZrStep nx_st = zr_next(ic, u0, u1, nzr, zbeg, clm, cz);
            if (nx_st.valid) issue(nx_st, kissue++);
        }
        if (st.seed) continue;
        // ---- phase B: warp w = tile w of the band, lane c = A-row c ----
        const uint32_t t = z * tpp + st.band * NW + warp;
        constexpr uint32_t rpt = kTileCodes / nx;          // rows per tile
        const uint32_t R = warp * rpt + lane / spr, seg = lane % spr, kreg = seg >> 1, p = seg & 1;
        const uint8_t* my = stg + R * RP + 512u * kreg + 256u * p + 16u * ((R * spr + seg) & 7u);
        uint32_t A[32];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint4 v = *reinterpret_cast<const uint4*>(my + 16 * j);
            A[4 * j] = v.x; A[4 * j + 1] = v.y; A[4 * j + 2] = v.z; A[4 * j + 3] = v.w;
        }
        uint8_t* mym = msk + 16u * (32u * warp + lane);
        const uint4 om = *reinterpret_cast<const uint4*>(mym);
        if (a.codes_out != nullptr) {
            uint16_t* co = a.codes_out + (uint64_t)t * kTileCodes + 64 * lane;
#pragma unroll
            for (int j = 0; j < 32; ++j) { co[2 * j] = (uint16_t)A[j]; co[2 * j + 1] = (uint16_t)(A[j] >> 16); }
        }
        transpose32_regs(A);
        __syncwarp();
        uint32_t* Os = reinterpret_cast<uint32_t*>(stg + warp * rpt * RP);   // the tile's own rows
#pragma unroll
        for (int r = 0; r < 32; ++r) Os[32 * r + lane] = A[r];
        __syncwarp();
        const uint64_t tl = t - a.tile_begin;
        uint4* stage = a.tstage + tl * kTileBlocks;
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
            const uint64_t fo = tl * 32 + 4 * lane;
            if (fo + 4 <= a.flags_cap) *reinterpret_cast<uint32_t*>(a.flags_out + fo) = myF;
        }
        // outliers of this tile (rare): counts, staging offsets, records in index order
        const uint64_t vm = ((uint64_t)om.y << 32) | om.x, dm = ((uint64_t)om.w << 32) | om.z;
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
            const uint64_t g0 = (uint64_t)t * kTileCodes + 64u * lane;   // A-row c = tile codes 64c..
#pragma unroll 1
            for (int j = 0; j < 64; ++j) {
                const uint64_t gi = g0 + j;
                if ((dm >> j) & 1u) {
                    const uint64_t zz = gi / PL, rem = gi - zz * PL, yy = rem / nx, xx = rem - yy * nx;
                    const int32_t dl = zr_delta(a, P, (int64_t)zz, (int64_t)yy, (int64_t)xx, CL ? cz : 0u, CL ? cy : 0u);
                    if (pd < a.dcap) a.dstage[pd] = make_uint2((uint32_t)gi, (uint32_t)dl);
                    else atomicOr(&ctrl->stage_overflow, 1u);
                    ++pd;
                }
                if ((vm >> j) & 1u) {
                    if (pv < a.vcap) a.vstage[pv] = make_uint2((uint32_t)gi, __float_as_uint(__ldg(a.field + (gi - a.base))));
                    else atomicOr(&ctrl->stage_overflow, 1u);
                    ++pv;
                }
            }
            *reinterpret_cast<uint4*>(mym) = make_uint4(0, 0, 0, 0);   // clear for the stage's reuse
        }
    }
    if ((a.exp & 8388608) && tid == 0 && blockIdx.x < 2048) {
        unsigned long long t2;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));
        g_zr_trace[4 * blockIdx.x + 3] = t2;
    }
    tmem_free();
}

bool compress_uses_zr(const CompressArgs& a)
{
    if (a.g.ndim != 3 || a.rescan || a.tstage == nullptr || (variant_bits() & 8192)) return false;
    const uint32_t nx = a.g.nx, PL = a.g.P;
    if (nx % 128 != 0 || nx > 1024 || (nx & (nx - 1)) != 0 || PL % nx != 0 || (PL / nx) % kZrRows != 0) return false;
    if (a.g.n / PL < 2 || (a.base & 3) != 0) return false;
    const uint32_t tpp = PL / kTileCodes;
    if (a.tile_begin % tpp != 0 || a.tile_end % tpp != 0) return false;
    // f1 chunk-local streams: chunks of 16 planes x one tile of rows (2048 / nx, a power of 2)
    if (a.cl && (kTileCodes % nx != 0)) return false;
    return true;
}

template <int NW, int NST>
static size_t zr_smem()
{
    constexpr uint32_t nx = 128u * NW, spr = 2u * NW;
    return (size_t)NST * ((kZrRows + 1) * 4u * nx + kZrRows * spr * 16u);
}

template <int NST>
static void zr_pick(uint32_t nw, bool cl, void (*&kern)(CompressArgs, uint32_t, uint32_t), size_t& sm)
{
    switch (nw * 2 + (cl ? 1 : 0)) {
        case 2: kern = k_compress_zr<1, false, NST>; sm = zr_smem<1, NST>(); break;
        case 3: kern = k_compress_zr<1, true, NST>; sm = zr_smem<1, NST>(); break;
        case 4: kern = k_compress_zr<2, false, NST>; sm = zr_smem<2, NST>(); break;
        case 5: kern = k_compress_zr<2, true, NST>; sm = zr_smem<2, NST>(); break;
        case 8: kern = k_compress_zr<4, false, NST>; sm = zr_smem<4, NST>(); break;
        case 9: kern = k_compress_zr<4, true, NST>; sm = zr_smem<4, NST>(); break;
        case 16: kern = k_compress_zr<8, false, NST>; sm = zr_smem<8, NST>(); break;
        default: kern = k_compress_zr<8, true, NST>; sm = zr_smem<8, NST>(); break;
    }
}

cudaError_t launch_compress_zr(const CompressArgs& a, cudaStream_t st)
{
    const uint32_t nx = a.g.nx, nw = nx / 128;
    const uint32_t cz = a.cl ? 16u : 0u, cy = a.cl ? (uint32_t)(kTileCodes / nx) : 0u;
    void (*kern)(CompressArgs, uint32_t, uint32_t) = nullptr;
    size_t sm = 0;
    if (variant_bits() & 16384) zr_pick<3>(nw, a.cl != 0, kern, sm);   // A/B: three TMA stages
    else zr_pick<kZrStages>(nw, a.cl != 0, kern, sm);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (!(variant_bits() & 16777216))   // the whole carveout as shared memory (3 CTAs per SM)
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    // residency from registers and shared memory (the occupancy API reports one CTA per SM
    // for kernels that allocate tensor memory)
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kern);
    int dev = 0, smem_sm = 0, regs_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
    const int regs_cta = ((fa.numRegs + 7) & ~7) * 32 * (int)nw;
    int per_sm = (int)(smem_sm / (sm + fa.sharedSizeBytes + 1024));
    if (regs_cta > 0 && regs_sm / regs_cta < per_sm) per_sm = regs_sm / regs_cta;
    if (per_sm < 1) per_sm = 1;
    if (getenv("FZ_ZR_DEBUG")) fprintf(stderr, "zr: occupancy %d CTAs/SM, smem %zu\n", per_sm, sm);
    const int tmem_cap = 512 / (nw > 4 ? 256 : 128);   // TMEM columns per SM / per CTA
    if (per_sm > tmem_cap) per_sm = tmem_cap;
    const uint32_t tpp = a.g.P / kTileCodes, nbands = a.g.P / nx / kZrRows;
    const uint64_t units = (uint64_t)nbands * ((a.tile_end - a.tile_begin) / tpp);
    uint64_t grid = (uint64_t)per_sm * num_sms();
    if (grid > units) grid = units;
    if (grid == 0) return cudaSuccess;
    LaunchProf lp(K_COMPRESS, st);
    CompressArgs ax = a;
    ax.exp = variant_bits();
    { const cudaError_t e_ = launch_pdl(kern, dim3((unsigned)grid), dim3(32 * nw), sm, st, ax, cz, cy); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

}  // namespace fz

extern "C" int fz_debug_zr_trace(unsigned long long* host, int n)
{
    if (n > 4 * 2048) n = 4 * 2048;
    return cudaMemcpyFromSymbol(host, fz::g_zr_trace, sizeof(unsigned long long) * n) == cudaSuccess ? n : -1;
}
