// fz_dzr.cu -- the row-walking decoder for field-global 3-D streams (D1-D6, "the
// decompression pipeline is highly symmetrical"; SV §8.a D1-D6, §8.f f2): the inverse Lorenzo
// q = S_z S_y S_x delta (S_a = inclusive prefix sum along axis a, mod 2^32) computed
// without an int32 intermediate field in HBM.
//
// Shapes: 3-D, nx % 128 == 0, nx <= 1024, ny % 16 == 0 (the row-walking compressor's shapes:
// a band of 16 rows of one plane is NW = nx / 128 whole tiles).  Citation key: P:n = PAPER.md
// line n; S:n = SPEC.md line n; SV = SURVEY.md; R# = DESIGN.md §3 readings.
//
// Decomposition.  A unit is (band b, chunk c): the band's 16 rows in planes [16c, 16c + 16).
// With X = S_x delta and, for an element (z, y, x) of band b (rows 16b .. 16b + 15):
//   Q(z, y, x) = Q(z - 1, y, x) + V_b(z, x) + sum_{16b <= y' <= y} X(z, y', x)
//   V_b(z, x)  = sum_{y' < 16b} X(z, y', x) = S_x( sum_{b' < b} Cd(b', z, .) )(x)
//   Q(16c - 1, y, x) = S_x( G(b, c, .) + sum_{16b <= y' <= y} Dpre(b, c, y', .) )(x)
// where Cd(b, z, x) = sum over the band's rows of delta (column sums, one plane), Dsum(b, c) =
// sum over the chunk's planes of delta (one value per band element), Dpre(b, c) = sum_{c' < c}
// Dsum(b, c'), CD(b, c, x) = column sums of Dsum(b, c), G(b, c, x) = sum_{b' < b} sum_{c' < c}
// CD(b', c', x).  Every term is linear in delta, so the sums are taken before the prefix
// operators and all arithmetic is mod 2^32, exactly like the oracle's recurrence.
//
//   k_dzr_sum   (pass 1) decodes every tile to delta: Cd per (band, plane), Dsum and CD per unit
//   k_dzr_prep1 V = S_x exscan_b Cd (in place); Dpre = exscan_c Dsum (in place); CD exscan_b
//   (G = exscan_c of that, summed by pass 2 at each unit start)
//   k_dzr_main  (pass 2) per unit: carry Q(16c - 1) from G and Dpre into tensor memory, then per
//               plane: decode the band's tiles (gather, un-shuffle, unpack, delta patch, x scan)
//               into shared memory, walk the 16 rows down y with the y carry from V, add the z
//               carry, dequantize (D6: x^ = fl32(fl32(q) w), one FMUL) and store fp32.
//
// Per tile (warp w of the CTA = tile w of the band), phase B: lane L gathers the tile's blocks
// 32f + L (f = 0..7; zero where the flag bit is clear) into O (row-major, 4 KB) in the
// tile's own rows of the shared buffer, lane c reads column c of O and bit-transposes it
// (O[r][c] = transpose32(A[c])[r] inverted: A[c] = transpose32(O[.][c])), which gives
// A-row c = codes 64c .. 64c + 63 of the tile; sign-magnitude unpack (R8: 0x8000 -> 0), delta
// patch (R7), and (pass 2) the x prefix: in the lane, then across the nx / 64 lanes of a row.
// Phase A: thread (w, lane) owns columns x0 = 128 w + 4 lane .. + 3 of all 16 rows.
// Shared X / delta buffer: row i at i RPX, 64-element segment s at 272 s (16 bytes of skew per
// segment: conflict-free 128-bit stores in phase B and loads in phase A); two buffers (plane k
// and k + 1), one CTA barrier per plane.
#include "fz_internal.cuh"
#include "fz_launch.h"
#include "fz_rowwalk.cuh"

namespace fz {

constexpr int kDzrRows = 16;   // band height (rows)
constexpr int kDzrChunk = 16;  // planes per unit

bool decode_uses_dzr(const fz_shape& s)
{
    if (s.ndim != 3) return false;
    const uint64_t nz = s.dims[0], ny = s.dims[1], nx = s.dims[2];
    if (nx % 128 != 0 || nx > 1024 || (nx & (nx - 1)) != 0 || ny % kDzrRows != 0 || nz < 2) return false;
    if (nz * ny * nx >= (1ull << 32)) return false;
    return true;
}

static uint32_t dzr_grid_main(uint32_t nx);

// Planes per unit.  Both passes hand units (band, chunk of cz planes) round-robin to a
// persistent grid of G CTAs, so a pass lasts ceil(U / G) units: with 16-plane chunks c4
// (32 bands x 32 chunks = 1024 units on 444 CTAs) ran 3 units where the mean is 2.3.  The
// depth is picked per shape to minimize ceil(U / G) (cz + 2) (2 plane-equivalents for a
// unit start: carry rebuild, first gather), cz in [8, 48]; c4 -> cz = 40 (ties with 19; the
// deeper chunk measured faster: fewer chunk sums for the prep).
// Variant 33554432 keeps cz = 16 (A/B).
uint32_t dz_chunk_depth(uint64_t nz, uint32_t nbands, uint64_t G)
{
    if ((variant_bits() & 33554432) || G == 0) return (uint32_t)kDzrChunk;   // A/B; no device
    uint32_t best = kDzrChunk;
    uint64_t bcost = ~0ull;
    for (uint32_t cz = 8; cz <= 48; ++cz) {
        const uint64_t U = (uint64_t)nbands * ((nz + cz - 1) / cz);
        const uint64_t cost = (U + G - 1) / G * ((cz < nz ? cz : nz) + 2);
        if (cost <= bcost) { bcost = cost; best = cz; }   // ties -> the deeper chunk (fewer starts)
    }
    return best;
}

DzrLayout dzr_layout(const fz_shape& s)
{
    DzrLayout L{};
    if (!decode_uses_dzr(s)) return L;
    const uint64_t nz = s.dims[0], ny = s.dims[1], nx = s.dims[2];
    L.nbands = (uint32_t)(ny / kDzrRows);
    L.cz = dz_chunk_depth(nz, L.nbands, dzr_grid_main((uint32_t)nx));
    L.nchunks = (uint32_t)((nz + L.cz - 1) / L.cz);
    // carry arrays sized for the larger of this depth and the A/B depth 16 (the workspace must
    // not depend on the variant bits)
    const uint64_t nch16 = (nz + kDzrChunk - 1) / kDzrChunk, nch_ws = L.nchunks > nch16 ? L.nchunks : nch16;
    L.cdelta_elems = (uint64_t)L.nbands * nz * nx;
    L.dsum_elems = (uint64_t)L.nbands * nch_ws * kDzrRows * nx;
    L.cd_elems = (uint64_t)L.nbands * nch_ws * nx;
    return L;
}

template <int NW>
struct DzrSmem {
    static constexpr uint32_t nx = 128u * NW, spl = nx / 64;      // A-rows per row
    static constexpr uint32_t RPX = 272u * spl;                   // bytes per row
    static constexpr uint32_t buf = kDzrRows * RPX;               // one plane of the band
    static constexpr uint32_t total = 2 * buf + 4 * kDzrRows * NW; // + row-scan warp totals
};

// Resolves the device-parsed counts (fz_decompress_async) into the CTA's copy of the args.
__device__ __forceinline__ void dzr_resolve(DzrArgs& a)
{
    if (!a.dev) return;
    a.nnz_total = a.ctrl->dec_nnz;
    a.nd = a.ctrl->dec_nd;
    a.drec = reinterpret_cast<const uint2*>(a.payload + 16 * a.nnz_total);
    a.dev = 0;
}

// D1 inputs of tile t: its 8 flag words and the payload offset of its first block, kept as
// the raw loaded words (combined only in dzr_gather, a plane later: no wait at the load).
struct DzrIn {
    uint4 f0, f1;
    uint32_t bpre, loc;
};
__device__ __forceinline__ DzrIn dzr_in(const DzrArgs& a, uint32_t t)
{
    DzrIn in;
    const uint4* fp = reinterpret_cast<const uint4*>(a.flags + 32ull * t);
    in.f0 = __ldg(fp);
    in.f1 = __ldg(fp + 1);
    in.bpre = __ldg(a.bpre + (t >> 10));
    in.loc = __ldg(a.loc + t);
    return in;
}

// D2: asynchronous gather of the tile's blocks 32 f + lane into O (row-major 4 KB at `O`, block
// b at 16 b; a clear flag bit zero-fills the block: cp.async with src-size 0).
__device__ __forceinline__ void dzr_gather(const DzrArgs& a, const DzrIn& in, uint8_t* O, int lane)
{
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t F[8] = {in.f0.x, in.f0.y, in.f0.z, in.f0.w, in.f1.x, in.f1.y, in.f1.z, in.f1.w};
    // 32-bit block indices: nnz <= 256 T < 2^29 for N < 2^32 (R16); a corrupt index (past the
    // stream's nnz) zero-fills its block and reports FZ_ERR_CORRUPT once per lane
    const uint32_t nnz = a.nnz_total < 0xFFFFFFFFull ? (uint32_t)a.nnz_total : 0xFFFFFFFFu;
    uint32_t pre = in.bpre + in.loc;
    bool bad = false;
    const uint4* pay = reinterpret_cast<const uint4*>(a.payload);
    const uint32_t Ob = smem_u32(O) + 16u * lane;
#pragma unroll
    for (int f = 0; f < 8; ++f) {
        const uint32_t bi = pre + __popc(F[f] & lt);
        const bool set = (F[f] >> lane) & 1u;
        const bool ok = bi < nnz;
        bad |= set && !ok;
        const uint32_t n = (set && ok) ? 16u : 0u;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(Ob + 512u * f),
                     "l"(pay + (ok ? bi : 0u)), "r"(n) : "memory");
        pre += __popc(F[f]);
    }
    if (bad) atomicCAS(&a.ctrl->err, 0, (int)FZ_ERR_CORRUPT);
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// D3-D5(x) for tile t (one warp), its O already gathered at `rows` (the tile's first row): its
// 2048 deltas (XSCAN: x-prefixed) into the shared buffer, 64 per lane: lane c = A-row c = row
// c / spl, x 64 (c % spl).
template <int NW, bool XSCAN>
__device__ __forceinline__ void dzr_tile(const DzrArgs& a, uint32_t t, uint8_t* rows, int lane)
{
    using S = DzrSmem<NW>;
    constexpr uint32_t spl = S::spl, RPX = S::RPX;
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    // D3: column c of O, bit-transposed -> A-row c
    uint32_t A[32];
    {
        const uint32_t* O = reinterpret_cast<const uint32_t*>(rows);
#pragma unroll
        for (int r = 0; r < 32; ++r) A[r] = O[32 * r + lane];
    }
    __syncwarp();
    transpose32_regs(A);
    // D4: sign-magnitude -> int32 (R8: 0x8000 decodes to 0): v = ((c & 0x7FFF) ^ m) - m with
    // m the sign replicated by PRMT (selector 9 = sign of byte 1, B = sign of byte 3)
    int32_t d[64];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const uint32_t w = A[j];
        uint32_t mlo, mhi;   // (inline PTX: __byte_perm masks the selector's sign bits away)
        asm("prmt.b32 %0, %1, 0, 0x9999;" : "=r"(mlo) : "r"(w));
        asm("prmt.b32 %0, %1, 0, 0xBBBB;" : "=r"(mhi) : "r"(w));
        d[2 * j] = (int32_t)(((w & 0x7FFFu) ^ mlo) - mlo);
        d[2 * j + 1] = (int32_t)((((w >> 16) & 0x7FFFu) ^ mhi) - mhi);
    }
    // the lane's 64 values live at row lane / spl, segment lane % spl of the tile
    uint8_t* const mine = rows + (uint32_t)(lane / spl) * RPX + 272u * (uint32_t)(lane % spl);
    // delta-outlier patch (R7; rare, warp-uniform): through the shared buffer
    uint32_t rlo = 0, rhi = 0;
    if (a.nd > 0) {
        rlo = __ldg(a.drange + t);
        rhi = __ldg(a.drange + t + 1);
        const uint32_t nd32 = (uint32_t)a.nd;
        rlo = rlo < nd32 ? rlo : nd32;
        rhi = rhi < rlo ? rlo : (rhi < nd32 ? rhi : nd32);
    }
    if (rhi > rlo) {
#pragma unroll
        for (int k = 0; k < 16; ++k)
            *reinterpret_cast<int4*>(mine + 16 * k) = make_int4(d[4 * k], d[4 * k + 1], d[4 * k + 2], d[4 * k + 3]);
        __syncwarp();
        for (uint32_t k = rlo + lane; k < rhi; k += 32) {
            const uint2 r = a.drec[k];
            const uint64_t e = (uint64_t)r.x - (uint64_t)t * kTileCodes;
            if (e < (uint64_t)kTileCodes) {
                const uint32_t rr = (uint32_t)e / S::nx, x = (uint32_t)e % S::nx;
                *reinterpret_cast<int32_t*>(rows + rr * RPX + 272u * (x / 64) + 4u * (x % 64)) = (int32_t)r.y;
            } else {
                atomicCAS(&a.ctrl->err, 0, (int)FZ_ERR_CORRUPT);
            }
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const int4 v = *reinterpret_cast<const int4*>(mine + 16 * k);
            d[4 * k] = v.x; d[4 * k + 1] = v.y; d[4 * k + 2] = v.z; d[4 * k + 3] = v.w;
        }
        __syncwarp();
    }
    if (XSCAN) {   // D5 (x): in the lane (8 groups of 8: independent chains), then across the row
        uint32_t gt[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
#pragma unroll
            for (int j = 1; j < 8; ++j) d[8 * g + j] = (int32_t)((uint32_t)d[8 * g + j] + (uint32_t)d[8 * g + j - 1]);
            gt[g] = (uint32_t)d[8 * g + 7];
        }
#pragma unroll
        for (int g = 1; g < 8; ++g) gt[g] += gt[g - 1];   // inclusive group prefixes
        const uint32_t acc = gt[7];
        uint32_t inc = acc;
#pragma unroll
        for (uint32_t o = 1; o < spl; o <<= 1) {
            const uint32_t up = __shfl_up_sync(kFull, inc, o);
            if ((uint32_t)lane % spl >= o) inc += up;
        }
        const uint32_t ex = inc - acc;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            const uint32_t add = ex + (g > 0 ? gt[g - 1] : 0u);
#pragma unroll
            for (int j = 0; j < 8; ++j) d[8 * g + j] = (int32_t)((uint32_t)d[8 * g + j] + add);
        }
    }
#pragma unroll
    for (int k = 0; k < 16; ++k)
        *reinterpret_cast<int4*>(mine + 16 * k) = make_int4(d[4 * k], d[4 * k + 1], d[4 * k + 2], d[4 * k + 3]);
}

// The CTA's plane sequence: units u = blockIdx.x + i gridDim.x (band-major), planes of each.
struct DzrCur {
    uint32_t u, b, c, z, z1;
    bool valid;
};
__device__ __forceinline__ DzrCur dzr_unit(const DzrArgs& a, uint32_t u)
{
    DzrCur q;
    q.u = u;
    q.valid = u < a.nbands * a.nchunks;
    q.b = u / a.nchunks;
    q.c = u - q.b * a.nchunks;
    q.z = q.c * a.cz;
    q.z1 = min(a.nz, q.z + a.cz);
    return q;
}
__device__ __forceinline__ DzrCur dzr_next(const DzrArgs& a, DzrCur q)
{
    if (q.z + 1 < q.z1) { ++q.z; return q; }
    return dzr_unit(a, q.u + gridDim.x);
}

// Phase A address of row i, columns x0 .. x0 + 3 (x0 = 128 w + 4 lane)
template <int NW>
__device__ __forceinline__ uint32_t dzr_aoff(int warp, int lane)
{
    return 272u * (2u * warp + (uint32_t)lane / 16) + 16u * ((uint32_t)lane % 16);
}

// ---- pass 1: Cd per (band, plane), Dsum and CD per unit ----
template <int NW>
__global__ void __launch_bounds__(32 * NW, 12 / NW) k_dzr_sum(DzrArgs a)
{
    pdl_begin();
    dzr_resolve(a);
    extern __shared__ __align__(128) uint8_t dsm[];
    using S = DzrSmem<NW>;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t nx = S::nx, tpp = a.tpp, nz = a.nz;
    const uint32_t aoff = dzr_aoff<NW>(warp, lane);
    const uint32_t x0 = 128u * warp + 4u * lane;
    const uint32_t trow = (uint32_t)warp * (kTileCodes / nx) * S::RPX;   // the tile's rows
    DzrCur cur = dzr_unit(a, blockIdx.x);
    if (!cur.valid) return;
    auto tile_of = [&](const DzrCur& q) { return q.z * tpp + q.b * NW + warp; };
    dzr_gather(a, dzr_in(a, tile_of(cur)), dsm + trow, lane);
    DzrCur nxt = dzr_next(a, cur);
    DzrIn in_next = dzr_in(a, nxt.valid ? tile_of(nxt) : tile_of(cur));
    uint32_t ds[kDzrRows][4];
    uint32_t cdu[4];
    for (uint32_t k = 0; cur.valid; ++k) {
        uint8_t* buf = dsm + (k & 1u) * S::buf;
        if (cur.z == cur.c * a.cz) {
#pragma unroll
            for (int i = 0; i < kDzrRows; ++i) ds[i][0] = ds[i][1] = ds[i][2] = ds[i][3] = 0u;
            cdu[0] = cdu[1] = cdu[2] = cdu[3] = 0u;
        }
        dzr_tile<NW, false>(a, tile_of(cur), buf + trow, lane);
        __syncthreads();
        // the next plane's gather into the other buffer (every warp is past its phase A)
        if (nxt.valid) {
            dzr_gather(a, in_next, dsm + ((k + 1) & 1u) * S::buf + trow, lane);
            const DzrCur n2 = dzr_next(a, nxt);
            if (n2.valid) in_next = dzr_in(a, tile_of(n2));
        }
        uint32_t cs[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int i = 0; i < kDzrRows; ++i) {
            const uint4 v = *reinterpret_cast<const uint4*>(buf + i * S::RPX + aoff);
            ds[i][0] += v.x; ds[i][1] += v.y; ds[i][2] += v.z; ds[i][3] += v.w;
            cs[0] += v.x; cs[1] += v.y; cs[2] += v.z; cs[3] += v.w;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) cdu[q] += cs[q];
        *reinterpret_cast<uint4*>(a.cdelta + ((uint64_t)cur.b * nz + cur.z) * nx + x0) = make_uint4(cs[0], cs[1], cs[2], cs[3]);
        if (cur.z + 1 == cur.z1) {   // unit end: its delta sums and their column sums
            int32_t* dsp = a.dsum + ((uint64_t)cur.b * a.nchunks + cur.c) * kDzrRows * nx + x0;
#pragma unroll
            for (int i = 0; i < kDzrRows; ++i)
                *reinterpret_cast<uint4*>(dsp + (uint64_t)i * nx) = make_uint4(ds[i][0], ds[i][1], ds[i][2], ds[i][3]);
            *reinterpret_cast<uint4*>(a.cd + ((uint64_t)cur.b * a.nchunks + cur.c) * nx + x0) =
                make_uint4(cdu[0], cdu[1], cdu[2], cdu[3]);
        }
        cur = nxt;
        nxt = dzr_next(a, cur);
    }
}

// ---- prep 1: blocks [0, nz): V rows of plane z; then Dpre (exclusive over chunks, in place);
// then CD exclusive over bands (in place) ----
__global__ void k_dzr_prep1(DzrArgs a, uint32_t dblocks)
{
    pdl_begin();
    __shared__ uint32_t wt8[8][8];   // [band of the round][warp] (nx / 4 <= 256 threads)
    const uint32_t nx = a.nx, nz = a.nz;
    if (blockIdx.x < nz) {   // V(b, z, .) = S_x( sum_{b' < b} Cd(b', z, .) ), blockDim >= nx / 4
        const uint32_t z = blockIdx.x, x0 = 4u * threadIdx.x;
        const bool act = x0 < nx;   // (blockDim is nx / 4 rounded up to whole warps)
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
        uint32_t run[4] = {0u, 0u, 0u, 0u};
        for (uint32_t b0 = 0; b0 < a.nbands; b0 += 8) {   // 8 bands per round: loads in flight
            const uint32_t m = min(8u, a.nbands - b0);
            uint4 cv[8];
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j)
                cv[j] = (j < m && act) ? *reinterpret_cast<const uint4*>(a.cdelta + ((uint64_t)(b0 + j) * nz + z) * nx + x0)
                                       : make_uint4(0, 0, 0, 0);
            uint32_t v[8][4];
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) {
                v[j][0] = run[0]; v[j][1] = run[1]; v[j][2] = run[2]; v[j][3] = run[3];
                if (j < m) { run[0] += cv[j].x; run[1] += cv[j].y; run[2] += cv[j].z; run[3] += cv[j].w; }
                v[j][1] += v[j][0]; v[j][2] += v[j][1]; v[j][3] += v[j][2];
                uint32_t inc = v[j][3];
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t up = __shfl_up_sync(kFull, inc, o);
                    if (lane >= o) inc += up;
                }
                if (lane == 31) wt8[j][warp] = inc;
                const uint32_t ex = inc - v[j][3];
#pragma unroll
                for (int q = 0; q < 4; ++q) v[j][q] += ex;
            }
            __syncthreads();
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) {
                uint32_t pre = 0;
                for (int w2 = 0; w2 < warp && w2 < nw; ++w2) pre += wt8[j][w2];
                if (j < m && act)
                    *reinterpret_cast<uint4*>(a.cdelta + ((uint64_t)(b0 + j) * nz + z) * nx + x0) =
                        make_uint4(v[j][0] + pre, v[j][1] + pre, v[j][2] + pre, v[j][3] + pre);
            }
            __syncthreads();
        }
        return;
    }
    const uint64_t band_q = (uint64_t)kDzrRows * nx / 4;   // uint4 per band element plane
    const uint64_t gi = (uint64_t)(blockIdx.x - nz) * blockDim.x + threadIdx.x;
    if (blockIdx.x < nz + dblocks) {   // Dpre: thread = (band, element quad), over chunks
        if (gi >= (uint64_t)a.nbands * band_q) return;
        const uint32_t b = (uint32_t)(gi / band_q);
        const uint64_t e = gi % band_q;
        uint4* p = reinterpret_cast<uint4*>(a.dsum) + (uint64_t)b * a.nchunks * band_q + e;
        uint4 run = make_uint4(0, 0, 0, 0);
        for (uint32_t c0 = 0; c0 < a.nchunks; c0 += 8) {
            uint4 v[8];
            const uint32_t m = min(8u, a.nchunks - c0);
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j)
                if (j < m) v[j] = p[(uint64_t)(c0 + j) * band_q];
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j)
                if (j < m) {
                    p[(uint64_t)(c0 + j) * band_q] = run;
                    run.x += v[j].x; run.y += v[j].y; run.z += v[j].z; run.w += v[j].w;
                }
        }
        return;
    }
    // CD exclusive over bands: thread = (chunk, x quad)
    const uint64_t hi = (uint64_t)(blockIdx.x - nz - dblocks) * blockDim.x + threadIdx.x;
    const uint32_t nq = nx / 4;
    if (hi >= (uint64_t)a.nchunks * nq) return;
    const uint32_t c = (uint32_t)(hi / nq), q = (uint32_t)(hi % nq);
    uint4* p = reinterpret_cast<uint4*>(a.cd) + (uint64_t)c * nq + q;
    const uint64_t bstride = (uint64_t)a.nchunks * nq;
    uint4 run = make_uint4(0, 0, 0, 0);
    for (uint32_t b0 = 0; b0 < a.nbands; b0 += 8) {
        uint4 v[8];
        const uint32_t m = min(8u, a.nbands - b0);
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j)
            if (j < m) v[j] = p[(uint64_t)(b0 + j) * bstride];
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j)
            if (j < m) {
                p[(uint64_t)(b0 + j) * bstride] = run;
                run.x += v[j].x; run.y += v[j].y; run.z += v[j].z; run.w += v[j].w;
            }
    }
}

// ---- prep 2: G = exclusive over chunks of (CD exclusive over bands): thread = (band, x quad) ----
__global__ void k_dzr_prep2(DzrArgs a)
{
    pdl_begin();
    const uint32_t nq = a.nx / 4;
    const uint64_t gi = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gi >= (uint64_t)a.nbands * nq) return;
    const uint32_t b = (uint32_t)(gi / nq), q = (uint32_t)(gi % nq);
    uint4* p = reinterpret_cast<uint4*>(a.cd) + (uint64_t)b * a.nchunks * nq + q;
    uint4 run = make_uint4(0, 0, 0, 0);
    for (uint32_t c0 = 0; c0 < a.nchunks; c0 += 8) {
        uint4 v[8];
        const uint32_t m = min(8u, a.nchunks - c0);
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j)
            if (j < m) v[j] = p[(uint64_t)(c0 + j) * nq];
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j)
            if (j < m) {
                p[(uint64_t)(c0 + j) * nq] = run;
                run.x += v[j].x; run.y += v[j].y; run.z += v[j].z; run.w += v[j].w;
            }
    }
}

// ---- pass 2 ----
template <int NW, bool LOGT>
__global__ void __launch_bounds__(32 * NW, 12 / NW) k_dzr_main(DzrArgs a)
{
    pdl_begin();
    dzr_resolve(a);
    extern __shared__ __align__(128) uint8_t dsm[];
    __shared__ __align__(16) uint32_t tsh[4];   // tsh[3]: TMEM base (kept off shared address 0)
    uint32_t& tmem_base = tsh[3];
    using S = DzrSmem<NW>;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t nx = S::nx, tpp = a.tpp, nz = a.nz, PL = a.P;
    uint32_t* const wt = reinterpret_cast<uint32_t*>(dsm + 2 * S::buf);   // [16][NW]
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
    const uint32_t aoff = dzr_aoff<NW>(warp, lane);
    const uint32_t x0 = 128u * warp + 4u * lane;
    const uint32_t trow = (uint32_t)warp * (kTileCodes / nx) * S::RPX;
    DzrCur cur = dzr_unit(a, blockIdx.x);
    auto tile_of = [&](const DzrCur& q) { return q.z * tpp + q.b * NW + warp; };
    DzrCur nxt = cur;
    DzrIn in_next;
    auto vrow = [&](const DzrCur& q) {   // the band's y carries at plane q.z
        return *reinterpret_cast<const uint4*>(a.cdelta + ((uint64_t)q.b * nz + q.z) * nx + x0);
    };
    uint4 vy = make_uint4(0, 0, 0, 0);
    if (cur.valid) {
        dzr_gather(a, dzr_in(a, tile_of(cur)), dsm + trow, lane);
        nxt = dzr_next(a, cur);
        in_next = dzr_in(a, nxt.valid ? tile_of(nxt) : tile_of(cur));
        vy = vrow(cur);
    }
    for (uint32_t k = 0; cur.valid; ++k) {
        const uint32_t b = cur.b, c = cur.c, z = cur.z;
        // ---- unit start: carry Q(16c - 1) of the band = S_x( G + S_y Dpre ) ----
        if (z == c * a.cz) {
            uint32_t v[kDzrRows][4];
            if (c == 0) {
#pragma unroll
                for (int i = 0; i < kDzrRows; ++i) v[i][0] = v[i][1] = v[i][2] = v[i][3] = 0u;
            } else {
                const uint4 g = dz_gsum(a.cd + x0, (uint64_t)b * a.nchunks, c, nx);
                uint32_t run[4] = {g.x, g.y, g.z, g.w};
                const int32_t* dp = a.dsum + ((uint64_t)b * a.nchunks + c) * kDzrRows * nx + x0;
                uint4 dv[kDzrRows];
#pragma unroll
                for (int i = 0; i < kDzrRows; ++i) dv[i] = *reinterpret_cast<const uint4*>(dp + (uint64_t)i * nx);
#pragma unroll
                for (int i = 0; i < kDzrRows; ++i) {
                    run[0] += dv[i].x; run[1] += dv[i].y; run[2] += dv[i].z; run[3] += dv[i].w;
                    v[i][0] = run[0];
                    v[i][1] = run[0] + run[1];
                    v[i][2] = v[i][1] + run[2];
                    v[i][3] = v[i][2] + run[3];
                }
#pragma unroll
                for (int i = 0; i < kDzrRows; ++i) {
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
                for (int i = 0; i < kDzrRows; ++i) {
                    uint32_t pre = 0;
#pragma unroll
                    for (int ww = 0; ww < NW; ++ww)
                        if (ww < warp) pre += wt[i * NW + ww];
#pragma unroll
                    for (int q = 0; q < 4; ++q) v[i][q] += pre;
                }
            }
#pragma unroll
            for (int g = 0; g < kDzrRows / 4; ++g) {
                uint32_t tv[16];
#pragma unroll
                for (int ii = 0; ii < 4; ++ii)
#pragma unroll
                    for (int q = 0; q < 4; ++q) tv[4 * ii + q] = v[4 * g + ii][q];
                tmem_st16(taddr + 16u * g, tv);
            }
            tmem_wait_st();
        }
        uint8_t* buf = dsm + (k & 1u) * S::buf;
        dzr_tile<NW, true>(a, tile_of(cur), buf + trow, lane);
        __syncthreads();
        uint32_t cy[4] = {vy.x, vy.y, vy.z, vy.w};
        // the next plane's gather into the other buffer (every warp is past its phase A) and
        // its y carries (a plane ahead)
        if (nxt.valid) {
            dzr_gather(a, in_next, dsm + ((k + 1) & 1u) * S::buf + trow, lane);
            const DzrCur n2 = dzr_next(a, nxt);
            if (n2.valid) in_next = dzr_in(a, tile_of(n2));
            vy = vrow(nxt);
        }
        uint32_t tpb[2][8];
        tmem_ld8(taddr, tpb[0]);
        int32_t* o = a.q_out + (uint64_t)z * PL + (uint64_t)(b * kDzrRows) * nx + x0;
#pragma unroll
        for (int i = 0; i < kDzrRows; ++i, o += nx) {
            uint32_t(&tpp)[8] = tpb[(i >> 1) & 1];
            if ((i & 1) == 0) {
                tmem_wait_ld8(tpp);
                if (i + 2 < kDzrRows) tmem_ld8(taddr + 4u * (i + 2), tpb[((i >> 1) + 1) & 1]);
            }
            const uint32_t* qp = tpp + 4 * (i & 1);
            const uint4 xv = *reinterpret_cast<const uint4*>(buf + i * S::RPX + aoff);
            cy[0] += xv.x; cy[1] += xv.y; cy[2] += xv.z; cy[3] += xv.w;
            const uint32_t q0 = qp[0] + cy[0], q1 = qp[1] + cy[1], q2 = qp[2] + cy[2], q3 = qp[3] + cy[3];
            tmem_st4(taddr + 4u * i, q0, q1, q2, q3);
            if (w > 0.0f) {   // D6: x^ = fl32(fl32(q) w), one FMUL (R21)
                __stcs(reinterpret_cast<float4*>(o),
                       dzx<LOGT>(q0, q1, q2, q3, w));
            } else {          // the integer codes (fz_debug_decode_q)
                __stcs(reinterpret_cast<int4*>(o), make_int4((int)q0, (int)q1, (int)q2, (int)q3));
            }
        }
        tmem_wait_st();
        cur = nxt;
        nxt = dzr_next(a, cur);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(kTmemCols)
                     : "memory");
}

// ---------------------------------------------------------------------------------------
// 1-D fields (f3's HACC-like particle arrays): the inverse Lorenzo is one prefix sum along the
// field, q = S_x delta, so the carry into tile t is the sum of every delta before it.  Two
// passes over the stream instead of an int32 field: k_dec1d<true> sums each tile's deltas
// (gather by cp.async, register un-shuffle, unpack, delta patch), a two-level exclusive scan of
// the tile sums gives the carries, and k_dec1d<false> decodes the tile again, scans it in the
// lane (8 chains of 8) and across the warp, adds the carry, dequantizes (D6; f3's exp when the
// header says so) and stores through a skewed shared staging as coalesced 16-byte stores.
// ---------------------------------------------------------------------------------------
template <bool SUM, bool LOGT>
__global__ void __launch_bounds__(256) k_dec1d(DzrArgs a, uint64_t n, uint32_t* tsum, const uint32_t* loc,
                                               const uint32_t* bpre)
{
    pdl_begin();
    dzr_resolve(a);
    extern __shared__ __align__(16) uint8_t dsm1[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint8_t* const B = dsm1 + (uint32_t)warp * (32 * 272);   // O (4 KB), then the output staging
    const float w = a.wp ? *a.wp : a.w;
    for (uint32_t t = blockIdx.x * 8 + warp; t < a.ntiles; t += gridDim.x * 8) {
        dzr_gather(a, dzr_in(a, t), B, lane);
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
        uint32_t A[32];
        {
            const uint32_t* O = reinterpret_cast<const uint32_t*>(B);
#pragma unroll
            for (int r = 0; r < 32; ++r) A[r] = O[32 * r + lane];
        }
        __syncwarp();
        transpose32_regs(A);
        int32_t d[64];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const uint32_t wd = A[j];
            uint32_t mlo, mhi;
            asm("prmt.b32 %0, %1, 0, 0x9999;" : "=r"(mlo) : "r"(wd));
            asm("prmt.b32 %0, %1, 0, 0xBBBB;" : "=r"(mhi) : "r"(wd));
            d[2 * j] = (int32_t)(((wd & 0x7FFFu) ^ mlo) - mlo);
            d[2 * j + 1] = (int32_t)((((wd >> 16) & 0x7FFFu) ^ mhi) - mhi);
        }
        // delta-outliers (R7; rare): through the staging buffer (lane c's 64 at 272 c)
        uint32_t rlo = 0, rhi = 0;
        if (a.nd > 0) {
            const uint32_t nd32 = (uint32_t)a.nd;
            rlo = __ldg(a.drange + t);
            rhi = __ldg(a.drange + t + 1);
            rlo = rlo < nd32 ? rlo : nd32;
            rhi = rhi < rlo ? rlo : (rhi < nd32 ? rhi : nd32);
        }
        if (rhi > rlo) {
#pragma unroll
            for (int k = 0; k < 16; ++k)
                *reinterpret_cast<int4*>(B + 272u * lane + 16u * k) = make_int4(d[4 * k], d[4 * k + 1], d[4 * k + 2], d[4 * k + 3]);
            __syncwarp();
            for (uint32_t k = rlo + lane; k < rhi; k += 32) {
                const uint2 r = a.drec[k];
                const uint64_t e = (uint64_t)r.x - (uint64_t)t * kTileCodes;
                if (e < (uint64_t)kTileCodes)
                    *reinterpret_cast<int32_t*>(B + 272u * (uint32_t)(e / 64) + 4u * (uint32_t)(e % 64)) = (int32_t)r.y;
                else
                    atomicCAS(&a.ctrl->err, 0, (int)FZ_ERR_CORRUPT);
            }
            __syncwarp();
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const int4 v = *reinterpret_cast<const int4*>(B + 272u * lane + 16u * k);
                d[4 * k] = v.x; d[4 * k + 1] = v.y; d[4 * k + 2] = v.z; d[4 * k + 3] = v.w;
            }
            __syncwarp();
        }
        if (SUM) {
            uint32_t sm = 0;
#pragma unroll
            for (int j = 0; j < 64; ++j) sm += (uint32_t)d[j];
            sm = __reduce_add_sync(kFull, sm);
            if (lane == 0) tsum[t] = sm;
            continue;
        }
        // the lane's inclusive prefix (8 independent chains of 8), the warp's, the tile carry
        uint32_t gt[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
#pragma unroll
            for (int j = 1; j < 8; ++j) d[8 * g + j] = (int32_t)((uint32_t)d[8 * g + j] + (uint32_t)d[8 * g + j - 1]);
            gt[g] = (uint32_t)d[8 * g + 7];
        }
#pragma unroll
        for (int g = 1; g < 8; ++g) gt[g] += gt[g - 1];
        uint32_t inc = gt[7];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t up = __shfl_up_sync(kFull, inc, o);
            if (lane >= o) inc += up;
        }
        const uint32_t carry = __ldg(bpre + (t >> 10)) + __ldg(loc + t);
        const uint32_t ex = carry + inc - gt[7];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            float4 v;
            const uint32_t a0 = ex + (k >= 2 ? gt[(k >> 1) - 1] : 0u);
            v.x = __uint_as_float((uint32_t)d[4 * k] + a0);
            v.y = __uint_as_float((uint32_t)d[4 * k + 1] + a0);
            v.z = __uint_as_float((uint32_t)d[4 * k + 2] + a0);
            v.w = __uint_as_float((uint32_t)d[4 * k + 3] + a0);
            if (w > 0.0f) {
                v = dzx<LOGT>(__float_as_uint(v.x), __float_as_uint(v.y), __float_as_uint(v.z), __float_as_uint(v.w), w);
            }
            *reinterpret_cast<float4*>(B + 272u * lane + 16u * k) = v;
        }
        __syncwarp();
        const uint64_t g = (uint64_t)t * kTileCodes;
        if (g + kTileCodes <= n) {
            float4* dst = reinterpret_cast<float4*>(a.q_out + g);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const uint32_t c = (uint32_t)lane + 32u * j;   // 16-byte chunk = lane c / 16, part c % 16
                __stcs(dst + c, *reinterpret_cast<const float4*>(B + 272u * (c >> 4) + 16u * (c & 15)));
            }
        } else {
            for (uint32_t e = lane; e < (uint32_t)(n - g); e += 32)
                a.q_out[g + e] = *reinterpret_cast<const int32_t*>(B + 272u * (e / 64) + 4u * (e % 64));
        }
        __syncwarp();
    }
}

// two-level exclusive scan of the tile sums: loc = within blocks of 1024 tiles, bpre = of the
// blocks (one block of 1024 threads for the second level)
__global__ void __launch_bounds__(1024) k_tsum_block(const uint32_t* __restrict__ tsum, uint32_t ntiles, uint32_t* loc,
                                                     uint32_t* bsum)
{
    pdl_begin();
    __shared__ uint32_t ws[33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t i = blockIdx.x * 1024 + threadIdx.x;
    const uint32_t x = i < ntiles ? tsum[i] : 0u;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) ws[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const uint32_t v = ws[lane];
        uint32_t vi = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, vi, o);
            if (lane >= o) vi += y;
        }
        ws[lane] = vi - v;
        if (lane == 31) ws[32] = vi;
    }
    __syncthreads();
    if (i < ntiles) loc[i] = ws[warp] + inc - x;
    if (threadIdx.x == 0) bsum[blockIdx.x] = ws[32];
}

__global__ void __launch_bounds__(1024) k_tsum_top(uint32_t* bsum, uint32_t nb)
{
    pdl_begin();
    __shared__ uint32_t ws[33];
    __shared__ uint32_t carry;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint32_t base = 0; base < nb; base += 1024) {
        const uint32_t i = base + threadIdx.x;
        const uint32_t x = i < nb ? bsum[i] : 0u;
        uint32_t inc = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) ws[warp] = inc;
        __syncthreads();
        if (warp == 0) {
            const uint32_t v = ws[lane];
            uint32_t vi = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, vi, o);
                if (lane >= o) vi += y;
            }
            ws[lane] = vi - v;
            if (lane == 31) ws[32] = vi;
        }
        __syncthreads();
        if (i < nb) bsum[i] = carry + ws[warp] + inc - x;
        __syncthreads();
        if (threadIdx.x == 0) carry += ws[32];
        __syncthreads();
    }
}

cudaError_t launch_decode_1d(const DzrArgs& a, uint64_t n, uint32_t* tsum, uint32_t* loc, uint32_t* bsum,
                             cudaStream_t st)
{
    const size_t sm = 8 * 32 * 272;
    const uint64_t want = ((uint64_t)a.ntiles + 7) / 8, cap = (uint64_t)num_sms() * 3;
    const unsigned grid = (unsigned)(want < cap ? want : cap);
    {
        cudaFuncSetAttribute(k_dec1d<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        LaunchProf lp(K_DZR_SUM, st);
        { const cudaError_t e_ = launch_pdl(k_dec1d<true, false>, dim3(grid), dim3(256), sm, st, a, n, tsum, nullptr, nullptr); if (e_ != cudaSuccess) return e_; }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const uint32_t nb = (a.ntiles + 1023) / 1024;
    {
        LaunchProf lp(K_DZR_PREP, st);
        { const cudaError_t e_ = launch_pdl(k_tsum_block, dim3(nb), dim3(1024), 0, st, tsum, a.ntiles, loc, bsum); if (e_ != cudaSuccess) return e_; }
    }
    {
        LaunchProf lp(K_DZR_PREP, st);
        { const cudaError_t e_ = launch_pdl(k_tsum_top, dim3(1), dim3(1024), 0, st, bsum, nb); if (e_ != cudaSuccess) return e_; }
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    auto kern = a.logt > 0 ? k_dec1d<false, true> : k_dec1d<false, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    LaunchProf lp(K_DZR_MAIN, st);
    { const cudaError_t e_ = launch_pdl(kern, dim3(grid), dim3(256), sm, st, a, n, nullptr, loc, bsum); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

template <int NW>
static int dzr_per_sm(const void* kern, size_t sm, bool tmem)
{
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kern);
    int dev = 0, smem_sm = 0, regs_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
    const int regs_cta = ((fa.numRegs + 7) & ~7) * 32 * NW;
    int per_sm = (int)(smem_sm / (sm + fa.sharedSizeBytes + 1024));
    if (regs_cta > 0 && regs_sm / regs_cta < per_sm) per_sm = regs_sm / regs_cta;
    if (tmem) {
        const int cap = 512 / (NW > 4 ? 256 : 128);
        if (per_sm > cap) per_sm = cap;
    }
    return per_sm < 1 ? 1 : per_sm;
}

// V, Dpre and G from pass 1's sums (shared by the row-walking decoders of fz_dzr.cu and
// fz_dzg.cu).  One block size for the three parts of prep 1: nx / 4 rounded up to whole warps
// (V takes one thread per x quad of a row); the Dpre and CD parts index by block * bs + thread.
cudaError_t launch_dzr_prep(const DzrArgs& a, cudaStream_t st)
{
    const uint32_t bs = (a.nx / 4 + 31) / 32 * 32;
    const uint64_t dq = (uint64_t)a.nbands * kDzrRows * (a.nx / 4);
    const uint32_t dblocks = (uint32_t)((dq + bs - 1) / bs);
    const uint32_t cblocks = (uint32_t)(((uint64_t)a.nchunks * (a.nx / 4) + bs - 1) / bs);
    {
        LaunchProf lp(K_DZR_PREP, st);
        const cudaError_t e = launch_pdl(k_dzr_prep1, dim3(a.nz + dblocks + cblocks), dim3(bs), 0, st, a, dblocks);
        if (e != cudaSuccess) return e;
    }
    // (G = the exclusive prefix over chunks of prep 1's CD scan is summed by pass 2 at each
    // unit start: dz_gsum; k_dzr_prep2 below does it as a separate pass, kept for reference)
    return cudaGetLastError();
}

template <int NW>
static cudaError_t dzr_launch(const DzrArgs& a, cudaStream_t st)
{
    using S = DzrSmem<NW>;
    const uint32_t U = a.nbands * a.nchunks;
    // pass 1
    {
        auto kern = k_dzr_sum<NW>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::total);
        uint64_t grid = (uint64_t)dzr_per_sm<NW>((const void*)kern, S::total, false) * num_sms();
        if (grid > U) grid = U;
        if (variant_bits() & 65536) {
            const uint64_t per = (U + grid - 1) / grid;
            grid = (U + per - 1) / per;
        }
        LaunchProf lp(K_DZR_SUM, st);
        const cudaError_t e = launch_pdl(kern, dim3((unsigned)grid), dim3(32 * NW), S::total, st, a);
        if (e != cudaSuccess) return e;
    }
    // prep
    {
        cudaError_t e = launch_dzr_prep(a, st);
        if (e != cudaSuccess) return e;
    }
    // pass 2
    {
        auto kern = a.logt > 0 ? k_dzr_main<NW, true> : k_dzr_main<NW, false>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::total);
        uint64_t grid = (uint64_t)dzr_per_sm<NW>((const void*)kern, S::total, true) * num_sms();
        if (grid > U) grid = U;
        if (variant_bits() & 65536) {   // A/B: every CTA the same number of units
            const uint64_t per = (U + grid - 1) / grid;
            grid = (U + per - 1) / per;
        }
        LaunchProf lp(K_DZR_MAIN, st);
        return launch_pdl(kern, dim3((unsigned)grid), dim3(32 * NW), S::total, st, a);
    }
}

static uint32_t dzr_grid_main(uint32_t nx)
{
    static uint32_t cache[4] = {0, 0, 0, 0};   // per NW (device attributes: one device per process)
    const int i = nx == 128 ? 0 : nx == 256 ? 1 : nx == 512 ? 2 : 3;
    if (cache[i] == 0) {
        int per = 1;
        switch (i) {
            case 0: per = dzr_per_sm<1>((const void*)k_dzr_main<1, false>, DzrSmem<1>::total, true); break;
            case 1: per = dzr_per_sm<2>((const void*)k_dzr_main<2, false>, DzrSmem<2>::total, true); break;
            case 2: per = dzr_per_sm<4>((const void*)k_dzr_main<4, false>, DzrSmem<4>::total, true); break;
            default: per = dzr_per_sm<8>((const void*)k_dzr_main<8, false>, DzrSmem<8>::total, true); break;
        }
        const int sms = num_sms();
        if (sms <= 0) return 0;
        cache[i] = (uint32_t)per * (uint32_t)sms;
    }
    return cache[i];
}

cudaError_t launch_decode_dzr(const DzrArgs& a, cudaStream_t st)
{
    switch (a.nx) {
        case 128: return dzr_launch<1>(a, st);
        case 256: return dzr_launch<2>(a, st);
        case 512: return dzr_launch<4>(a, st);
        default: return dzr_launch<8>(a, st);
    }
}

}  // namespace fz
