// fz_dzg.cu -- the row-walking decoder for 3-D shapes whose rows do not tile (c3, c5; D1-D6,
// P:400).  Citation key as in fz_dzr.cu.
//
// fz_dzr.cu decodes a band's tiles straight into the band's rows; here a tile (2048
// consecutive codes) straddles rows and planes, so the un-shuffle and the walk are
// split (the mirror image of fz_rowcodes.cu):
//   k_untile    one warp per tile: gather (cp.async, zero-fill for clear flags), lane c reads
//               column c of O and bit-transposes it (C5 inverse) into A-row c, the A-rows are
//               staged (skewed) in shared memory and leave as coalesced 16-byte stores into a
//               code field at the elements' flattened positions; a delta-outlier (R7) is
//               marked by the never-emitted code 0x8000 (R8), its delta is looked up later
//   k_dzg_sum   pass 1: unit (band of 16 rows, chunk of cz planes); thread (w, l) owns the 4
//               columns 128 w + 4 l of the band's rows; per plane it unpacks its 4 codes of
//               every row (loaded a plane ahead) and accumulates the chunk sums (Dsum, per
//               element), the plane's column sums (Cd) and their chunk total (CD) -- the
//               same arrays as fz_dzr.cu, so k_dzr_prep1 / prep2 form V, Dpre and G
//   k_dzg_main  pass 2: the unit's z carry S_x(G + S_y Dpre) into tensor memory; per plane the
//               16 rows' deltas, their x prefix across the CTA (warp scans + one barrier for
//               the warp totals of all 16 rows), the y carry (V, a plane ahead), the z carry,
//               x^ = fl32(fl32(q) w) (D6) and 16-byte stores.
// Traffic ~ 2 (code field out) + 2 + 2 (in, twice) + 4 (x^) + ~1.5 (carries) B/elem, against
// ~20 for the tile decoder with separate y and z walks.
#include "fz_internal.cuh"
#include "fz_launch.h"
#include "fz_rowwalk.cuh"

namespace fz {

constexpr int kDzgRows = 16;

bool decode_uses_dzg(const fz_shape& s)
{
    if (s.ndim != 3 || decode_uses_dzr(s)) return false;
    const uint64_t nz = s.dims[0], ny = s.dims[1], nx = s.dims[2];
    // nz >= 256, or nz >= 64 with N >= 2^22: c3 (nz = 100, 25 M elements) decodes 18 % faster
    // than with the tile decoder + y / z walks, while a small field with few planes (c1, 64^3)
    // pays more in launches than it saves (variant 268435456: nz >= 256 only, for A/B)
    if (nx % 4 != 0 || nx < 64 || nx > 512 || ny < 1) return false;
    const bool deep = nz >= 256, mid = !(variant_bits() & 268435456) && nz >= 64 && nz * ny * nx >= (1ull << 22);
    if (!deep && !mid) return false;
    return nz * ny * nx < (1ull << 32);
}

static uint32_t dzg_grid_main(uint32_t nx);

DzrLayout dzg_layout(const fz_shape& s)
{
    DzrLayout L{};
    if (!decode_uses_dzg(s)) return L;
    const uint64_t nz = s.dims[0], ny = s.dims[1], nx = s.dims[2];
    L.nbands = (uint32_t)((ny + kDzgRows - 1) / kDzgRows);
    L.cz = dz_chunk_depth(nz, L.nbands, dzg_grid_main((uint32_t)nx));   // balanced units (fz_dzr.cu)
    L.nchunks = (uint32_t)((nz + L.cz - 1) / L.cz);
    const uint64_t nch16 = (nz + 15) / 16, nch_ws = L.nchunks > nch16 ? L.nchunks : nch16;
    L.cdelta_elems = (uint64_t)L.nbands * nz * nx;
    L.dsum_elems = (uint64_t)L.nbands * nch_ws * kDzgRows * nx;
    L.cd_elems = (uint64_t)L.nbands * nch_ws * nx;
    const uint64_t T = (nz * ny * nx + kTileCodes - 1) / kTileCodes;
    L.code_bytes = 2 * kTileCodes * T;
    return L;
}

__device__ __forceinline__ void dzg_resolve(DzrArgs& a)
{
    if (!a.dev) return;
    a.nnz_total = a.ctrl->dec_nnz;
    a.nd = a.ctrl->dec_nd;
    a.drec = reinterpret_cast<const uint2*>(a.payload + 16 * a.nnz_total);
    a.dev = 0;
}

// ---- k_untile ----
__global__ void __launch_bounds__(256) k_untile(DzrArgs a, uint64_t n)
{
    pdl_begin();
    dzg_resolve(a);
    __shared__ __align__(16) uint8_t Ush[8][32 * 144];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint8_t* const B = Ush[warp];
    const uint32_t lt = (1u << lane) - 1u;
    const uint4* pay = reinterpret_cast<const uint4*>(a.payload);
    for (uint32_t t = blockIdx.x * 8 + warp; t < a.ntiles; t += gridDim.x * 8) {
        // D1 + D2: flags, offset, gather (zero-filled blocks for clear bits)
        const uint4* fp = reinterpret_cast<const uint4*>(a.flags + 32ull * t);
        const uint4 f0 = __ldg(fp), f1 = __ldg(fp + 1);
        const uint32_t F[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
        if (((f0.x | f0.y | f0.z | f0.w) | (f1.x | f1.y | f1.z | f1.w)) == 0u) {
            // all 256 blocks zero: the tile's codes are 0 -- no gather, no transpose
#pragma unroll
            for (int j = 0; j < 8; ++j) *reinterpret_cast<uint4*>(B + 144u * lane + 16u * j) = make_uint4(0, 0, 0, 0);
            __syncwarp();
        } else {
        // 32-bit block indices (nnz < 2^29, R16); one corrupt-index check per lane (fz_dzr.cu)
        const uint32_t nnz = a.nnz_total < 0xFFFFFFFFull ? (uint32_t)a.nnz_total : 0xFFFFFFFFu;
        uint32_t pre = __ldg(a.bpre + (t >> 10)) + __ldg(a.loc + t);
        bool bad = false;
        const uint32_t Bb = smem_u32(B) + 16u * lane;
#pragma unroll
        for (int f = 0; f < 8; ++f) {
            const uint32_t bi = pre + __popc(F[f] & lt);
            const bool set = (F[f] >> lane) & 1u;
            const bool ok = bi < nnz;
            bad |= set && !ok;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(Bb + 512u * f),
                         "l"(pay + (ok ? bi : 0u)), "r"((set && ok) ? 16u : 0u) : "memory");
            pre += __popc(F[f]);
        }
        if (bad) atomicCAS(&a.ctrl->err, 0, (int)FZ_ERR_CORRUPT);
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
        // D3: column c of O (row-major at B), bit-transposed -> A-row c
        uint32_t A[32];
        {
            const uint32_t* O = reinterpret_cast<const uint32_t*>(B);
#pragma unroll
            for (int r = 0; r < 32; ++r) A[r] = O[32 * r + lane];
        }
        __syncwarp();
        transpose32_regs(A);
        // A-row c to the skewed staging (A-row r at 144 r)
#pragma unroll
        for (int j = 0; j < 8; ++j)
            *reinterpret_cast<uint4*>(B + 144u * lane + 16u * j) = make_uint4(A[4 * j], A[4 * j + 1], A[4 * j + 2], A[4 * j + 3]);
        __syncwarp();
        }
        // delta-outliers of the tile (rare): code 0 -> 0x8000, the escape the walk resolves
        if (a.nd > 0) {
            const uint32_t nd32 = (uint32_t)a.nd;
            uint32_t lo = __ldg(a.drange + t), hi = __ldg(a.drange + t + 1);
            lo = lo < nd32 ? lo : nd32;
            hi = hi < lo ? lo : (hi < nd32 ? hi : nd32);
            for (uint32_t k = lo + lane; k < hi; k += 32) {
                const uint64_t e = (uint64_t)a.drec[k].x - (uint64_t)t * kTileCodes;
                if (e < (uint64_t)kTileCodes)
                    *reinterpret_cast<uint16_t*>(B + 144u * (uint32_t)(e / 64) + 2u * (uint32_t)(e % 64)) = 0x8000u;
                else
                    atomicCAS(&a.ctrl->err, 0, (int)FZ_ERR_CORRUPT);
            }
            __syncwarp();
        }
        // coalesced stores: 16-byte chunk L + 32 j of the tile = A-row (L + 32 j) / 8, part % 8
        const uint64_t g = (uint64_t)t * kTileCodes;
        uint4* dst = reinterpret_cast<uint4*>(a.codes + g);
        if (g + kTileCodes <= n) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t c = (uint32_t)lane + 32u * j;
                __stcg(dst + c, *reinterpret_cast<const uint4*>(B + 144u * (c >> 3) + 16u * (c & 7)));
            }
        } else {   // the tail tile: codes past N are padding
            for (uint32_t e = lane; e < (uint32_t)(n - g); e += 32)
                a.codes[g + e] = *reinterpret_cast<const uint16_t*>(B + 144u * (e / 64) + 2u * (e % 64));
        }
        __syncwarp();
    }
}

// 4 sign-magnitude codes (two words) -> int32 deltas; the escape 0x8000 (a delta-outlier of
// k_untile) takes its delta from the sorted records by binary search (rare).
__device__ __forceinline__ void dzg_unpack4(const DzrArgs& a, uint2 w, uint64_t g, int32_t (&d)[4])
{
    const uint32_t wd[2] = {w.x, w.y};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        uint32_t mlo, mhi;
        asm("prmt.b32 %0, %1, 0, 0x9999;" : "=r"(mlo) : "r"(wd[k]));
        asm("prmt.b32 %0, %1, 0, 0xBBBB;" : "=r"(mhi) : "r"(wd[k]));
        d[2 * k] = (int32_t)(((wd[k] & 0x7FFFu) ^ mlo) - mlo);
        d[2 * k + 1] = (int32_t)((((wd[k] >> 16) & 0x7FFFu) ^ mhi) - mhi);
    }
    const bool esc = (w.x & 0xFFFFu) == 0x8000u || (w.x >> 16) == 0x8000u || (w.y & 0xFFFFu) == 0x8000u ||
                     (w.y >> 16) == 0x8000u;
    if (__builtin_expect(esc, 0)) {
#pragma unroll 1
        for (int k = 0; k < 4; ++k) {
            const uint32_t c = (k < 2 ? wd[0] : wd[1]) >> (16 * (k & 1)) & 0xFFFFu;
            if (c != 0x8000u) continue;
            uint64_t lo = 0, hi = a.nd;   // first record with idx >= g + k
            while (lo < hi) {
                const uint64_t mid = (lo + hi) / 2;
                if ((uint64_t)a.drec[mid].x < g + k) lo = mid + 1;
                else hi = mid;
            }
            d[k] = (lo < a.nd && (uint64_t)a.drec[lo].x == g + k) ? (int32_t)a.drec[lo].y : 0;
        }
    }
}

struct DzgCur {
    uint32_t u, b, c, z, z1, rows;
    bool valid;
};
__device__ __forceinline__ DzgCur dzg_unit(const DzrArgs& a, uint32_t u)
{
    DzgCur q;
    q.u = u;
    q.valid = u < a.nbands * a.nchunks;
    q.b = u / a.nchunks;
    q.c = u - q.b * a.nchunks;
    q.z = q.c * a.cz;
    q.z1 = min(a.nz, q.z + a.cz);
    q.rows = min((uint32_t)kDzgRows, a.ny - q.b * kDzgRows);
    return q;
}
__device__ __forceinline__ DzgCur dzg_next(const DzrArgs& a, DzgCur q)
{
    if (q.z + 1 < q.z1) { ++q.z; return q; }
    return dzg_unit(a, q.u + gridDim.x);
}

// The 16 rows' code pairs of the thread's 4 columns at plane q.z, by cp.async into the
// thread's own 16 shared slots (8 bytes each; zero-filled past the band / row); each thread
// reads back only its own slots, so no barrier -- cp.async.wait_group orders them.
__device__ __forceinline__ void dzg_load_async(const DzrArgs& a, const DzgCur& q, uint32_t x0, bool colv, uint2* slots)
{
    const uint16_t* p = a.codes + (uint64_t)q.z * a.P + (uint64_t)(q.b * kDzgRows) * a.nx + x0;
#pragma unroll
    for (int i = 0; i < kDzgRows; ++i) {
        const bool v = colv && q.valid && (uint32_t)i < q.rows;
        const uint16_t* src = v ? p + (uint64_t)i * a.nx : a.codes;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(slots + i * blockDim.x)),
                     "l"(src), "r"(v ? 8u : 0u) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// ---- pass 1 ----
template <int NW>
__global__ void __launch_bounds__(32 * NW, 16 / NW) k_dzg_sum(DzrArgs a)
{
    pdl_begin();
    dzg_resolve(a);
    extern __shared__ __align__(16) uint8_t gsm[];
    uint2 (*slots)[kDzgRows * 32 * NW] = reinterpret_cast<uint2 (*)[kDzgRows * 32 * NW]>(gsm);   // codes of plane k, k + 1
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t nx = a.nx, nz = a.nz;
    const uint32_t x0 = 128u * warp + 4u * lane;
    const bool colv = x0 < nx;
    DzgCur cur = dzg_unit(a, blockIdx.x);
    DzgCur nxt = dzg_next(a, cur);
    dzg_load_async(a, cur, x0, colv, slots[0] + tid);
    dzg_load_async(a, nxt, x0, colv, slots[1] + tid);
    uint32_t ds[kDzgRows][4];
    uint32_t cdu[4];
    for (uint32_t k = 0; cur.valid; ++k) {
        if (cur.z == cur.c * a.cz) {
#pragma unroll
            for (int i = 0; i < kDzgRows; ++i) ds[i][0] = ds[i][1] = ds[i][2] = ds[i][3] = 0u;
            cdu[0] = cdu[1] = cdu[2] = cdu[3] = 0u;
        }
        const DzgCur n2 = dzg_next(a, nxt);
        dzg_load_async(a, n2, x0, colv, slots[(k + 2) % 3] + tid);   // two planes ahead
        asm volatile("cp.async.wait_group 2;" ::: "memory");
        const uint2* sl = slots[k % 3] + tid;
        const uint64_t g0 = (uint64_t)cur.z * a.P + (uint64_t)(cur.b * kDzgRows) * nx + x0;
        uint32_t cs[4] = {0u, 0u, 0u, 0u};
        uint32_t orv = 0;   // all-zero codes (the warp's 16 rows): nothing to add
#pragma unroll
        for (int i = 0; i < kDzgRows; ++i) {
            const uint2 cv = sl[i * blockDim.x];
            orv |= cv.x | cv.y;
        }
        if (__any_sync(kFull, orv != 0u))
#pragma unroll
        for (int i = 0; i < kDzgRows; ++i) {
            int32_t d[4];
            dzg_unpack4(a, sl[i * blockDim.x], g0 + (uint64_t)i * nx, d);
#pragma unroll
            for (int q = 0; q < 4; ++q) { ds[i][q] += (uint32_t)d[q]; cs[q] += (uint32_t)d[q]; }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) cdu[q] += cs[q];
        if (colv) *reinterpret_cast<uint4*>(a.cdelta + ((uint64_t)cur.b * nz + cur.z) * nx + x0) = make_uint4(cs[0], cs[1], cs[2], cs[3]);
        if (cur.z + 1 == cur.z1 && colv) {
            int32_t* dsp = a.dsum + ((uint64_t)cur.b * a.nchunks + cur.c) * kDzgRows * nx + x0;
#pragma unroll
            for (int i = 0; i < kDzgRows; ++i)
                *reinterpret_cast<uint4*>(dsp + (uint64_t)i * nx) = make_uint4(ds[i][0], ds[i][1], ds[i][2], ds[i][3]);
            *reinterpret_cast<uint4*>(a.cd + ((uint64_t)cur.b * a.nchunks + cur.c) * nx + x0) =
                make_uint4(cdu[0], cdu[1], cdu[2], cdu[3]);
        }
        cur = nxt;
        nxt = n2;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// Inclusive x prefix of 16 rows held as 4 consecutive values per thread, across the CTA:
// warp scans of all rows, the warp totals through wt[16][NW], one barrier.
template <int NW>
__device__ __forceinline__ void dzg_rows_xscan(uint32_t (&v)[kDzgRows][4], uint32_t* wt, int lane, int warp)
{
#pragma unroll
    for (int i = 0; i < kDzgRows; ++i) {
        v[i][1] += v[i][0]; v[i][2] += v[i][1]; v[i][3] += v[i][2];
        uint32_t inc = v[i][3];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t up = __shfl_up_sync(kFull, inc, o);
            if (lane >= o) inc += up;
        }
        if (lane == 31) wt[i * NW + warp] = inc;
        const uint32_t ex = inc - v[i][3];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[i][q] += ex;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kDzgRows; ++i) {
        uint32_t pre = 0;
#pragma unroll
        for (int ww = 0; ww < NW; ++ww)
            if (ww < warp) pre += wt[i * NW + ww];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[i][q] += pre;
    }
}

// ---- pass 2 ----
template <int NW, bool LOGT>
__global__ void __launch_bounds__(32 * NW, 16 / NW) k_dzg_main(DzrArgs a)
{
    pdl_begin();
    dzg_resolve(a);
    __shared__ uint32_t wts[3][kDzgRows * NW];   // row-scan warp totals (unit start + 2 plane buffers)
    extern __shared__ __align__(16) uint8_t gsm[];
    uint2 (*slots)[kDzgRows * 32 * NW] = reinterpret_cast<uint2 (*)[kDzgRows * 32 * NW]>(gsm);   // codes of plane k, k + 1
    uint4* const xsl = reinterpret_cast<uint4*>(gsm + 3 * 8 * kDzgRows * 32 * NW);   // the thread's x-prefixed rows
    const int tid = threadIdx.x;
    __shared__ __align__(16) uint32_t tsh[4];   // tsh[3]: TMEM base
    uint32_t& tmem_base = tsh[3];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t nx = a.nx, nz = a.nz, PL = a.P;
    const float w = a.wp ? *a.wp : a.w;
    constexpr uint32_t kTmemCols = NW > 4 ? 256u : 128u;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     ::"r"(smem_u32(&tmem_base)), "n"(kTmemCols) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t taddr = tmem_base + ((32u * (warp & 3)) << 16) + 68u * (warp >> 2);
    const uint32_t x0 = 128u * warp + 4u * lane;
    const bool colv = x0 < nx;
    DzgCur cur = dzg_unit(a, blockIdx.x);
    DzgCur nxt = dzg_next(a, cur);
    dzg_load_async(a, cur, x0, colv, slots[0] + tid);
    dzg_load_async(a, nxt, x0, colv, slots[1] + tid);
    uint4 vy = make_uint4(0, 0, 0, 0);
    if (cur.valid && colv) vy = *reinterpret_cast<const uint4*>(a.cdelta + ((uint64_t)cur.b * nz + cur.z) * nx + x0);
    for (uint32_t k = 0; cur.valid; ++k) {
        const uint32_t b = cur.b, c = cur.c, z = cur.z;
        if (z == c * a.cz) {   // unit start: carry Q(z - 1) of the band = S_x( G + S_y Dpre )
            uint32_t v[kDzgRows][4];
            if (c == 0) {
#pragma unroll
                for (int i = 0; i < kDzgRows; ++i) v[i][0] = v[i][1] = v[i][2] = v[i][3] = 0u;
            } else {
                uint4 gv = make_uint4(0, 0, 0, 0);
                if (colv) gv = dz_gsum(a.cd + x0, (uint64_t)b * a.nchunks, c, nx);
                uint32_t run[4] = {gv.x, gv.y, gv.z, gv.w};
                const int32_t* dp = a.dsum + ((uint64_t)b * a.nchunks + c) * kDzgRows * nx + x0;
#pragma unroll
                for (int i = 0; i < kDzgRows; ++i) {
                    uint4 dv = make_uint4(0, 0, 0, 0);
                    if (colv) dv = *reinterpret_cast<const uint4*>(dp + (uint64_t)i * nx);
                    run[0] += dv.x; run[1] += dv.y; run[2] += dv.z; run[3] += dv.w;
                    v[i][0] = run[0]; v[i][1] = run[1]; v[i][2] = run[2]; v[i][3] = run[3];
                }
                dzg_rows_xscan<NW>(v, wts[2], lane, warp);
            }
#pragma unroll
            for (int g = 0; g < kDzgRows / 4; ++g) {
                uint32_t tv[16];
#pragma unroll
                for (int ii = 0; ii < 4; ++ii)
#pragma unroll
                    for (int q = 0; q < 4; ++q) tv[4 * ii + q] = v[4 * g + ii][q];
                tmem_st16(taddr + 16u * g, tv);
            }
            tmem_wait_st();
        }
        const DzgCur n2 = dzg_next(a, nxt);
        dzg_load_async(a, n2, x0, colv, slots[(k + 2) % 3] + tid);   // two planes ahead
        asm volatile("cp.async.wait_group 2;" ::: "memory");
        const uint2* sl = slots[k % 3] + tid;
        uint32_t cy[4] = {vy.x, vy.y, vy.z, vy.w};
        if (nxt.valid && colv) vy = *reinterpret_cast<const uint4*>(a.cdelta + ((uint64_t)nxt.b * nz + nxt.z) * nx + x0);
        // deltas of the 16 rows, x prefix across the row (D5, x): in the thread and the warp
        // now (kept in the thread's shared slots), the warps' totals after one barrier
        const uint64_t g0 = (uint64_t)z * PL + (uint64_t)(b * kDzgRows) * nx + x0;
        uint32_t* wt = wts[k & 1];
        uint4* xs = xsl + tid;
        // a warp whose 16 rows x 128 columns of codes are all zero (RTM's exact-zero regions,
        // P:372) has X = 0: no unpack, no scans, zero warp totals
        uint32_t orv = 0;
#pragma unroll
        for (int i = 0; i < kDzgRows; ++i) {
            const uint2 cv = sl[i * blockDim.x];
            orv |= cv.x | cv.y;
        }
        const bool zw = !__any_sync(kFull, orv != 0u);
        if (zw) {
            if (lane == 31)
#pragma unroll
                for (int i = 0; i < kDzgRows; ++i) wt[i * NW + warp] = 0u;
        } else
#pragma unroll
        for (int i = 0; i < kDzgRows; ++i) {
            int32_t d[4];
            dzg_unpack4(a, sl[i * blockDim.x], g0 + (uint64_t)i * nx, d);
            uint32_t v0 = (uint32_t)d[0], v1 = v0 + (uint32_t)d[1], v2 = v1 + (uint32_t)d[2], v3 = v2 + (uint32_t)d[3];
            uint32_t inc = v3;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t up = __shfl_up_sync(kFull, inc, o);
                if (lane >= o) inc += up;
            }
            if (lane == 31) wt[i * NW + warp] = inc;
            const uint32_t ex = inc - v3;
            xs[i * blockDim.x] = make_uint4(v0 + ex, v1 + ex, v2 + ex, v3 + ex);
        }
        __syncthreads();
        // y carry down the band, z carry in TMEM, D6
        uint32_t tpb[2][8];
        tmem_ld8(taddr, tpb[0]);
        int32_t* o = a.q_out + g0;
#pragma unroll
        for (int i = 0; i < kDzgRows; ++i, o += nx) {
            uint32_t(&tpp)[8] = tpb[(i >> 1) & 1];
            if ((i & 1) == 0) {
                tmem_wait_ld8(tpp);
                if (i + 2 < kDzgRows) tmem_ld8(taddr + 4u * (i + 2), tpb[((i >> 1) + 1) & 1]);
            }
            const uint32_t* qp = tpp + 4 * (i & 1);
            uint32_t pre = 0;
#pragma unroll
            for (int ww = 0; ww < NW; ++ww)
                if (ww < warp) pre += wt[i * NW + ww];
            const uint4 xv = zw ? make_uint4(0u, 0u, 0u, 0u) : xs[i * blockDim.x];
            cy[0] += xv.x + pre; cy[1] += xv.y + pre; cy[2] += xv.z + pre; cy[3] += xv.w + pre;
            const uint32_t q0 = qp[0] + cy[0], q1 = qp[1] + cy[1], q2 = qp[2] + cy[2], q3 = qp[3] + cy[3];
            tmem_st4(taddr + 4u * i, q0, q1, q2, q3);
            if (colv && (uint32_t)i < cur.rows) {
                if (w > 0.0f)
                    __stcs(reinterpret_cast<float4*>(o),
                           dzx<LOGT>(q0, q1, q2, q3, w));
                else
                    __stcs(reinterpret_cast<int4*>(o), make_int4((int)q0, (int)q1, (int)q2, (int)q3));
            }
        }
        tmem_wait_st();
        cur = nxt;
        nxt = n2;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(kTmemCols)
                     : "memory");
}

template <int NW>
static int dzg_per_sm(const void* kern, size_t dyn)
{
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kern);
    int dev = 0, regs_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
    const int regs_cta = ((fa.numRegs + 7) & ~7) * 32 * NW;
    int per = regs_cta > 0 ? regs_sm / regs_cta : 1;
    int smem_sm = 0;
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    const int by_smem = smem_sm / (int)(fa.sharedSizeBytes + dyn + 1024);
    if (by_smem < per) per = by_smem;
    if (per > 16) per = 16;
    return per < 1 ? 1 : per;
}

template <int NW>
static cudaError_t dzg_launch(const DzrArgs& a, cudaStream_t st)
{
    const uint32_t U = a.nbands * a.nchunks;
    constexpr size_t sm1 = 3 * 8 * kDzgRows * 32 * NW, sm2 = sm1 + 16 * kDzgRows * 32 * NW;
    {
        auto kern = k_dzg_sum<NW>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
        uint64_t grid = (uint64_t)dzg_per_sm<NW>((const void*)kern, sm1) * num_sms();
        if (grid > U) grid = U;
        LaunchProf lp(K_DZR_SUM, st);
        { const cudaError_t e_ = launch_pdl(kern, dim3((unsigned)grid), dim3(32 * NW), sm1, st, a); if (e_ != cudaSuccess) return e_; }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    cudaError_t e = launch_dzr_prep(a, st);
    if (e != cudaSuccess) return e;
    auto kern = a.logt > 0 ? k_dzg_main<NW, true> : k_dzg_main<NW, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
    int per = dzg_per_sm<NW>((const void*)kern, sm2);
    const int tmem_cap = 512 / (NW > 4 ? 256 : 128);
    if (per > tmem_cap) per = tmem_cap;
    uint64_t grid = (uint64_t)per * num_sms();
    if (grid > U) grid = U;
    LaunchProf lp(K_DZR_MAIN, st);
    { const cudaError_t e_ = launch_pdl(kern, dim3((unsigned)grid), dim3(32 * NW), sm2, st, a); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

template <int NW>
static uint32_t dzg_grid_nw()
{
    int per = dzg_per_sm<NW>((const void*)k_dzg_main<NW, false>, 3 * 8 * kDzgRows * 32 * NW + 16 * kDzgRows * 32 * NW);
    const int tmem_cap = 512 / (NW > 4 ? 256 : 128);
    if (per > tmem_cap) per = tmem_cap;
    return (uint32_t)per * (uint32_t)num_sms();
}

static uint32_t dzg_grid_main(uint32_t nx)
{
    static uint32_t cache[4] = {0, 0, 0, 0};
    const uint32_t nw = (nx + 127) / 128;
    if (nw < 1 || nw > 4) return 0;
    if (cache[nw - 1] == 0) {
        switch (nw) {
            case 1: cache[0] = dzg_grid_nw<1>(); break;
            case 2: cache[1] = dzg_grid_nw<2>(); break;
            case 3: cache[2] = dzg_grid_nw<3>(); break;
            default: cache[3] = dzg_grid_nw<4>(); break;
        }
    }
    return cache[nw - 1];
}

cudaError_t launch_decode_dzg(const DzrArgs& a, cudaStream_t st)
{
    const uint64_t n = (uint64_t)a.nz * a.P;
    {
        const uint64_t want = ((uint64_t)a.ntiles + 7) / 8, cap = (uint64_t)num_sms() * 8;
        LaunchProf lp(K_DECODE, st);
        { const cudaError_t e_ = launch_pdl(k_untile, dim3((unsigned)(want < cap ? want : cap)), dim3(256), 0, st, a, n); if (e_ != cudaSuccess) return e_; }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    const uint32_t nw = (a.nx + 127) / 128;
    switch (nw) {
        case 1: return dzg_launch<1>(a, st);
        case 2: return dzg_launch<2>(a, st);
        case 3: return dzg_launch<3>(a, st);
        default: return dzg_launch<4>(a, st);
    }
}

}  // namespace fz
