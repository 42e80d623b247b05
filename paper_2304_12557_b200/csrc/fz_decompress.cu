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
#include <cstdlib>
#include <type_traits>

#include "fz_internal.cuh"
#include "fz_launch.h"

namespace fz {

constexpr int kScanChunk = 32;

// The y prefix sum is fused into the tile decode when every tile holds whole rows
// (nx | 2048, nx >= 256 so a tile has at most 8 rows) and no tile straddles two planes.
bool decode_fuses_y(const fz_shape& s)
{
    if (s.ndim != 3) return false;
    const uint64_t nx = s.dims[2];
    if (nx < 256 || nx > (uint64_t)kTileCodes || kTileCodes % nx != 0) return false;
    if ((s.dims[1] * nx) % kTileCodes != 0) return false;
    return s.dims[0] >= 148;        // one or two CTAs per plane: enough planes to fill the GPU
}

// Decode workspace: control block, per-tile block offsets (two-level exclusive scan of the
// flag popcounts), per-tile x-scan aggregates and carries, chunk sums of the axis scans.
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
    const uint64_t nb = (T + 1023) / 1024;
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    const uint64_t ych = (ny + kScanChunk - 1) / kScanChunk, zch = (nz + kScanChunk - 1) / kScanChunk;
    uint64_t sums = 0;
    if (s.ndim >= 2) sums = nz * ych * nx;
    if (s.ndim == 3 && zch * ny * nx > sums) sums = zch * ny * nx;
    size_t off = 0;
    L.ctrl = off;   off += 512;
    L.loc = off;    off = al(off + 4 * T);
    L.bsum = off;   off = al(off + 4 * nb);
    L.xagg = off;   off = al(off + 8 * T);
    L.xloc = off;   off = al(off + 8 * T);
    L.xbagg = off;  off = al(off + 8 * nb);
    L.sums = off;   off = al(off + 4 * sums);
    L.drange = off; off = al(off + 4 * (T + 1));
    L.ycarry = off; off = al(off + (decode_fuses_y(s) ? 4 * kMaxYseg * nz * nx : 0));
    {
        // zero sizes unless a row-walking decoder applies (dzg adds the code field)
        const DzrLayout Z = decode_uses_dzr(s) ? dzr_layout(s) : dzg_layout(s);
        L.dzr_cdelta = off; off = al(off + 4 * Z.cdelta_elems);
        L.dzr_dsum = off;   off = al(off + 4 * Z.dsum_elems);
        L.dzr_cd = off;     off = al(off + 4 * Z.cd_elems);
        L.dzg_codes = off;  off = al(off + Z.code_bytes);
    }
    L.sums_elems = sums;
    L.total = off;
    return L;
}

__global__ void k_decode_init(Ctrl* ctrl)
{
    pdl_begin();
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        // every byte of the control block defined (the host reads it back whole)
        for (uint32_t w = 0; w < sizeof(Ctrl) / 4; ++w) reinterpret_cast<uint32_t*>(ctrl)[w] = 0u;
        ctrl->err = 0;
        ctrl->nnz = 0;
    }
}

// Device-driven decode: the stream header is parsed on the device (thread 0); the section
// counts and the bin width go to ctrl, where every later kernel reads them, so the host needs
// nothing from the stream.  A header that does not match (magic, version, shape, N, T, size
// law, capacity, bin width) sets FZ_ERR_CORRUPT and zero counts (the kernels then read nothing
// outside the flags).
__global__ void k_decode_hdr(Ctrl* ctrl, const uint8_t* in, uint64_t in_size, uint32_t ndim, uint64_t d0,
                             uint64_t d1, uint64_t d2, uint64_t n, uint64_t T)
{
    pdl_begin();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (uint32_t w = 0; w < sizeof(Ctrl) / 4; ++w) reinterpret_cast<uint32_t*>(ctrl)[w] = 0u;
    ctrl->err = 0;
    ctrl->nnz = 0;
    auto u64 = [&](int off) {
        uint64_t v;
        memcpy(&v, in + off, 8);
        return v;
    };
    uint32_t magic;
    uint16_t ver;
    float w;
    memcpy(&magic, in, 4);
    memcpy(&ver, in + 4, 2);
    memcpy(&w, in + 64, 4);
    const uint64_t cT = u64(80), nnz = u64(88), nd = u64(96), nv = u64(104), total = u64(112);
    const uint64_t dm[3] = {d0, d1, d2};
    bool ok = magic == 0x32425A46u /* "FZB2" */ && ver == 1 && in[8] == ndim && u64(40) == n && cT == T &&
              total <= in_size && nnz <= 256 * T && nd <= n && nv <= n &&
              total == kHeaderBytes + 32 * T + 16 * nnz + 8 * nd + 8 * nv && w > 0.0f && isfinite(w);
    for (uint32_t k = 0; k < 3; ++k) ok = ok && u64(16 + 8 * k) == (k < ndim ? dm[k] : 1);
    uint16_t fl;
    memcpy(&fl, in + 6, 2);
    if (ok && (fl & 4u)) {   // f1 chunk-local stream: decoded by the blocking entry points only
        ok = false;
        ctrl->err = FZ_ERR_ARG;
    } else if (!ok) {
        ctrl->err = FZ_ERR_CORRUPT;
    }
    if (!ok) {
        ctrl->dec_nnz = ctrl->dec_nd = ctrl->dec_nv = 0;
        ctrl->dec_w = 0.0f;
        ctrl->dec_flags = 0;
        return;
    }
    ctrl->dec_nnz = nnz;
    ctrl->dec_nd = nd;
    ctrl->dec_nv = nv;
    ctrl->dec_w = w;
    ctrl->dec_flags = fl;
}

// Outlier lists must be strictly increasing and inside the field.
__global__ void k_validate_outliers(const uint2* rec, uint64_t cnt, uint64_t n, Ctrl* ctrl)
{
    pdl_begin();
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cnt;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t idx = rec[k].x;
        if (idx >= n || (k > 0 && rec[k - 1].x >= idx)) atomicCAS(&ctrl->err, 0, (int)FZ_ERR_CORRUPT);
    }
}

// Per-tile delta-outlier ranges: records [drange[t], drange[t+1]) fall in tile t (records
// ascend; entries are clamped by the reader, so a corrupt list cannot index out of range).
// Device-driven forms: records and counts located from ctrl (payload = the stream's payload
// section; which = 0 delta records, 1 value records).
// Both record lists in one launch: index k < nd checks the delta list, the rest the value list.
// The same launch also records the per-tile delta-outlier ranges (k_record_tiles' device form:
// drange[t] = first delta record at or after element 2048 t; readers clamp the entries).
__device__ void validate_dev_work(const uint8_t* payload, uint64_t n, Ctrl* ctrl, uint32_t ntiles, uint32_t* drange)
{
    const uint64_t nnz = ctrl->dec_nnz, nd = ctrl->dec_nd, nv = ctrl->dec_nv;
    const uint2* drec = reinterpret_cast<const uint2*>(payload + 16 * nnz);
    const uint2* vrec = drec + nd;
    const uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, step = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = i0; k < nd + nv; k += step) {
        const uint2* rec = k < nd ? drec : vrec;
        const uint64_t j = k < nd ? k : k - nd;
        const uint32_t idx = rec[j].x;
        if (idx >= n || (j > 0 && rec[j - 1].x >= idx)) atomicCAS(&ctrl->err, 0, (int)FZ_ERR_CORRUPT);
    }
    if (nd == 0) return;   // readers skip the ranges without records
    for (uint64_t t = i0; t <= ntiles; t += step) {
        const int64_t e = (int64_t)(t * kTileCodes);
        uint64_t l = 0, h = nd;
        while (l < h) {
            const uint64_t m = (l + h) / 2;
            if ((int64_t)drec[m].x < e) l = m + 1;
            else h = m;
        }
        drange[t] = (uint32_t)l;
    }
}


__global__ void k_record_tiles(const uint2* __restrict__ rec, uint64_t nd, uint32_t ntiles, uint64_t gbase,
                               uint32_t* __restrict__ drange, const uint8_t* payload = nullptr,
                               const Ctrl* ctrl = nullptr)
{
    pdl_begin();
    if (ctrl != nullptr) {   // device-driven: records and count from the parsed header
        nd = ctrl->dec_nd;
        rec = reinterpret_cast<const uint2*>(payload + 16 * ctrl->dec_nnz);
    }
    if (nd == 0) return;     // readers skip the ranges without records
    // one tile boundary per thread: drange[t] = first record at or after element 2048 t
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t <= ntiles;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const int64_t e = (int64_t)(t * kTileCodes);
        uint64_t l = 0, h = nd;
        while (l < h) {
            const uint64_t m = (l + h) / 2;
            if ((int64_t)rec[m].x - (int64_t)gbase < e) l = m + 1;
            else h = m;
        }
        drange[t] = (uint32_t)l;
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

// Block-wide (1024 threads) exclusive scans: plain sums and segmented sums.
__device__ __forceinline__ uint32_t block_excl_sum(uint32_t x, uint32_t& total, uint32_t* wsum)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = wsum[lane], wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, wi, o);
            if (lane >= o) wi += y;
        }
        wsum[lane] = wi - w;          // exclusive warp prefix
        if (lane == 31) wsum[32] = wi;
    }
    __syncthreads();
    total = wsum[32];
    const uint32_t r = wsum[warp] + inc - x;
    __syncthreads();
    return r;
}

__device__ __forceinline__ Seg block_excl_seg(Seg x, Seg& total, uint32_t* wf, uint32_t* wv)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    Seg inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const Seg y{__shfl_up_sync(kFull, inc.f, o), __shfl_up_sync(kFull, inc.v, o)};
        if (lane >= o) inc = seg_combine(y, inc);
    }
    Seg ex{__shfl_up_sync(kFull, inc.f, 1), __shfl_up_sync(kFull, inc.v, 1)};
    if (lane == 0) ex = Seg{0, 0};
    if (lane == 31) { wf[warp] = inc.f; wv[warp] = inc.v; }
    __syncthreads();
    if (warp == 0) {
        const Seg w{wf[lane], wv[lane]};
        Seg wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const Seg y{__shfl_up_sync(kFull, wi.f, o), __shfl_up_sync(kFull, wi.v, o)};
            if (lane >= o) wi = seg_combine(y, wi);
        }
        Seg we{__shfl_up_sync(kFull, wi.f, 1), __shfl_up_sync(kFull, wi.v, 1)};
        if (lane == 0) we = Seg{0, 0};
        __syncwarp();
        wf[lane] = we.f;
        wv[lane] = we.v;
        if (lane == 31) { wf[32] = wi.f; wv[32] = wi.v; }
    }
    __syncthreads();
    total = Seg{wf[32], wv[32]};
    const Seg r = seg_combine(Seg{wf[warp], wv[warp]}, ex);
    __syncthreads();
    return r;
}

// D1 part 1: per-tile nonzero-block counts (popcount of the 8 flag words), exclusive scan
// inside blocks of 1024 tiles; block totals in bsum.
// D1 / C7: per-tile exclusive popcount prefixes of the flags inside blocks of
// 1024 tiles (loc), block totals (bsum); the last block to finish (ticket in ctrl->scan_done,
// zeroed with ctrl by k_init / k_decode_hdr / k_decode_init and reset here) scans the block
// totals in place (exclusive) and writes the grand total to ctrl->nnz -- one launch.
__device__ void validate_dev_work(const uint8_t* payload, uint64_t n, Ctrl* ctrl, uint32_t ntiles, uint32_t* drange);

__global__ void __launch_bounds__(1024) k_nnz_block(const uint32_t* __restrict__ flags, uint32_t ntiles,
                                                    uint32_t* loc, uint32_t* bsum, Ctrl* ctrl, uint64_t expect_nnz,
                                                    const uint8_t* vpay, uint64_t vn, uint32_t* drange)
{
    pdl_begin();
    // device-parsed decode: the outlier-list validation and the per-tile delta ranges ride
    // along (they need only the parsed header)
    if (vpay != nullptr) validate_dev_work(vpay, vn, ctrl, ntiles, drange);
    __shared__ uint32_t wsum[33];
    __shared__ bool last;
    __shared__ unsigned long long carry;
    const uint32_t t = blockIdx.x * 1024 + threadIdx.x;
    uint32_t c = 0;
    if (t < ntiles) {
        const uint4 a = reinterpret_cast<const uint4*>(flags)[2 * (uint64_t)t];
        const uint4 b = reinterpret_cast<const uint4*>(flags)[2 * (uint64_t)t + 1];
        c = __popc(a.x) + __popc(a.y) + __popc(a.z) + __popc(a.w) + __popc(b.x) + __popc(b.y) + __popc(b.z) +
            __popc(b.w);
    }
    uint32_t total;
    const uint32_t ex = block_excl_sum(c, total, wsum);
    if (t < ntiles) loc[t] = ex;
    if (threadIdx.x == 0) {
        bsum[blockIdx.x] = total;
        __threadfence();
        last = atomicAdd(&ctrl->scan_done, 1u) == gridDim.x - 1;
        carry = 0;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    const uint32_t nb = gridDim.x;
    for (uint32_t base = 0; base < nb; base += 1024) {
        const uint32_t i = base + threadIdx.x;
        const uint32_t x = i < nb ? __ldcg(bsum + i) : 0u;
        uint32_t tot;
        const uint32_t e = block_excl_sum(x, tot, wsum);
        if (i < nb) bsum[i] = (uint32_t)(carry + e);
        __syncthreads();
        if (threadIdx.x == 0) carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        ctrl->scan_done = 0;   // ready for the next scan on this workspace
        ctrl->nnz = carry;
        // expect_nnz: the header's nnz, ~0 = the device-parsed one, ~1 = no check (the row-walking
        // and z-band compressors use this scan to produce nnz)
        if (expect_nnz != ~1ull) {
            const uint64_t want = expect_nnz == ~0ull ? __ldcg(&ctrl->dec_nnz) : expect_nnz;
            if (carry != want) atomicCAS(&ctrl->err, 0, (int)FZ_ERR_CORRUPT);   // popcount(flags) != nnz
        }
    }
}

// x carries: segmented exclusive scan of the per-tile x aggregates (only when some tile
// starts inside a row).
// One launch: the last block to finish (ticket in ctrl->scan_done, zero after the popcount scan
// and reset here) scans the block aggregates in place (k_xseg_top's work).
__device__ void xseg_top_block(uint2* xbagg, uint32_t nb, uint32_t* wf, uint32_t* wv);

__global__ void __launch_bounds__(1024) k_xseg_block(const uint2* xagg, uint32_t ntiles, uint2* xloc, uint2* xbagg,
                                                     Ctrl* ctrl)
{
    pdl_begin();
    __shared__ uint32_t wf[33], wv[33];
    __shared__ bool last;
    const uint32_t t = blockIdx.x * 1024 + threadIdx.x;
    const uint2 g = t < ntiles ? xagg[t] : make_uint2(0, 0);
    Seg total;
    const Seg ex = block_excl_seg(Seg{g.x, g.y}, total, wf, wv);
    if (t < ntiles) xloc[t] = make_uint2(ex.f, ex.v);
    if (threadIdx.x == 0) {
        xbagg[blockIdx.x] = make_uint2(total.f, total.v);
        __threadfence();
        last = atomicAdd(&ctrl->scan_done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    xseg_top_block(xbagg, gridDim.x, wf, wv);
    if (threadIdx.x == 0) ctrl->scan_done = 0;
}

__device__ void xseg_top_block(uint2* xbagg, uint32_t nb, uint32_t* wf, uint32_t* wv)
{
    __shared__ uint32_t cf, cv;
    if (threadIdx.x == 0) { cf = 0; cv = 0; }
    __syncthreads();
    for (uint32_t base = 0; base < nb; base += 1024) {
        const uint32_t i = base + threadIdx.x;
        const uint2 g = i < nb ? __ldcg(xbagg + i) : make_uint2(0, 0);
        Seg total;
        const Seg ex = block_excl_seg(Seg{g.x, g.y}, total, wf, wv);
        const Seg c{cf, cv};
        if (i < nb) {
            const Seg r = seg_combine(c, ex);
            xbagg[i] = make_uint2(r.f, r.v);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const Seg r = seg_combine(c, total);
            cf = r.f;
            cv = r.v;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------------
// D1-D5(x) for one tile: payload offsets from the flags, gather of the 16-byte blocks,
// register un-shuffle, unpack, delta-outlier patch, segmented inclusive x-scan inside the
// tile.  Returns the thread's 8 x-prefixed values (elements 8*tid .. 8*tid+7 of the tile);
// elements before the thread's first row start carry only the in-tile prefix (the carry
// from earlier tiles is added by k_xfix where a row spans tiles).  (lo, hi): the tile's
// delta-outlier records, found by the caller.
// ------------------------------------------------------------------------------------
struct DecSmem {
    uint32_t Obuf[32 * 33];
    __align__(16) int32_t D[kTileCodes];
    uint32_t wf[8], wv[8];
};

// Independent loads of a tile: lanes 0-7 of every warp hold the tile's 8 flag words, every
// lane its payload base and delta-outlier record range.
struct TileIn {
    uint32_t fw;
    uint64_t tbase;
    uint32_t rlo, rhi;
};

__device__ __forceinline__ TileIn tile_in(const DecodeArgs& a, uint32_t t)
{
    const int lane = threadIdx.x & 31;
    TileIn in;
    in.fw = lane < 8 ? __ldg(reinterpret_cast<const uint32_t*>(a.flags) + 8 * (uint64_t)t + lane) : 0u;
    in.tbase = (uint64_t)__ldg(a.bpre + (t >> 10)) + __ldg(a.loc + t);
    in.rlo = in.rhi = 0;
    if ((a.dev ? a.ctrl->dec_nd : a.nd) > 0) {
        in.rlo = __ldg(a.drange + t);
        in.rhi = __ldg(a.drange + t + 1);
    }
    return in;
}

// The thread's 16-byte payload block of the tile (zero when its flag bit is clear).
__device__ __forceinline__ uint4 tile_blk(const DecodeArgs& a, const TileIn& in)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t F = __shfl_sync(kFull, in.fw, warp);
    const uint32_t wpre = __reduce_add_sync(kFull, lane < warp ? __popc(in.fw) : 0u);
    uint4 blk = make_uint4(0, 0, 0, 0);
    if ((F >> lane) & 1u) {
        const uint64_t bi = in.tbase + wpre + __popc(F & ((1u << lane) - 1u));
        if (bi < (a.dev ? a.ctrl->dec_nnz : a.nnz_total)) blk = __ldcs(reinterpret_cast<const uint4*>(a.payload) + bi);
        else atomicCAS(&a.ctrl->err, 0, (int)FZ_ERR_CORRUPT);
    }
    return blk;
}

// Sign-magnitude 16-bit codes (two per word) -> int32 (C3 inverse): with m = -sign,
// v = ((c & 0x7FFF) ^ m) - m.
__device__ __forceinline__ void unpack_codes(const uint32_t (&w4)[4], int32_t (&dl)[8])
{
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t w = w4[i];
        const uint32_t mlo = (uint32_t)((int32_t)(w << 16) >> 31), mhi = (uint32_t)((int32_t)w >> 31);
        dl[2 * i] = (int32_t)(((w & 0x7FFFu) ^ mlo) - mlo);
        dl[2 * i + 1] = (int32_t)((((w >> 16) & 0x7FFFu) ^ mhi) - mhi);
    }
}

// Delta-outlier patch of the thread's 8 deltas (records [rlo, rhi) of tile starting at s).
__device__ __forceinline__ void patch_deltas(const DecodeArgs& a, DecSmem& sm, int64_t s, uint32_t rlo, uint32_t rhi,
                                             int32_t (&dl)[8])
{
    const int tid = threadIdx.x;
    const uint32_t nd32 = (uint32_t)(a.dev ? a.ctrl->dec_nd : a.nd);
    const uint2* drec = a.dev ? reinterpret_cast<const uint2*>(a.payload + 16 * a.ctrl->dec_nnz) : a.drec;
    rlo = rlo < nd32 ? rlo : nd32;
    rhi = rhi < rlo ? rlo : (rhi < nd32 ? rhi : nd32);
    if (rhi > rlo) {   // rare, block-uniform
#pragma unroll
        for (int u = 0; u < 8; ++u) sm.D[8 * tid + u] = dl[u];
        __syncthreads();
        for (uint32_t k = rlo + tid; k < rhi; k += kCta) {
            const uint2 r = drec[k];
            const uint64_t e = (uint64_t)r.x - a.gbase - (uint64_t)s;
            if (e < (uint64_t)kTileCodes) sm.D[e] = (int32_t)r.y;
            else atomicCAS(&a.ctrl->err, 0, (int)FZ_ERR_CORRUPT);
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < 8; ++u) dl[u] = sm.D[8 * tid + u];
    }
}

// D3-D5(x) for a tile of R whole rows (nx = 2048 / R >= 256, so every warp lies inside one
// row and row starts fall on warp boundaries): plain scans, no segment flags.
template <int R>
__device__ __forceinline__ void decode_tile_rows(const DecodeArgs& a, DecSmem& sm, int64_t s, const uint4& blk,
                                                 uint32_t rlo, uint32_t rhi, uint32_t (&q)[8])
{
    constexpr int WPR = 8 / R;    // warps per row
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    {
        uint32_t* row = sm.Obuf + (tid >> 3) * 33 + 4 * (tid & 7);
        row[0] = blk.x; row[1] = blk.y; row[2] = blk.z; row[3] = blk.w;
    }
    __syncthreads();
    uint32_t w4[4];
    {
        const int c = tid >> 3, kk = tid & 7;
#pragma unroll
        for (int i = 0; i < 4; ++i) w4[i] = sm.Obuf[(4 * kk + i) * 33 + c];
        transpose32_group8(w4, lane & 7);
    }
    int32_t dl[8];
    unpack_codes(w4, dl);
    patch_deltas(a, sm, s, rlo, rhi, dl);
    uint32_t acc = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) { acc += (uint32_t)dl[u]; q[u] = acc; }
    uint32_t inc = acc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t up = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += up;
    }
    if (lane == 31) sm.wv[warp] = inc;
    uint32_t pre = inc - acc;      // exclusive prefix inside the warp
    if (WPR > 1) {
        __syncthreads();
#pragma unroll
        for (int w = 0; w < WPR - 1; ++w) {
            const int ww = (warp & ~(WPR - 1)) + w;
            if (ww < warp) pre += sm.wv[ww];
        }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) q[u] += pre;
}

template <int NDIM>
__device__ __forceinline__ Seg decode_tile_x(const DecodeArgs& a, DecSmem& sm, uint32_t t, const uint4& blk,
                                             uint32_t rlo, uint32_t rhi, uint32_t (&q)[8])
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t nx = a.g.nx;
    const int64_t s = (int64_t)t * kTileCodes;
    const uint32_t g0 = (uint32_t)s + 8u * tid;
    uint32_t xm_rs = 0;                      // row-start bit per element
    if (nx >= 8) {
        const uint32_t x0 = fmod_(g0, a.dnx);
        const uint32_t us = x0 == 0 ? 0u : nx - x0;
        if (us < 8) xm_rs = 1u << us;
    } else {
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (fmod_(g0 + u, a.dnx) == 0) xm_rs |= 1u << u;
    }
    {
        uint32_t* row = sm.Obuf + (tid >> 3) * 33 + 4 * (tid & 7);
        row[0] = blk.x; row[1] = blk.y; row[2] = blk.z; row[3] = blk.w;
    }
    __syncthreads();
    // ---- D3: column c of O -> row c of A ----
    uint32_t w4[4];
    {
        const int c = tid >> 3, kk = tid & 7;
#pragma unroll
        for (int i = 0; i < 4; ++i) w4[i] = sm.Obuf[(4 * kk + i) * 33 + c];
        transpose32_group8(w4, lane & 7);
    }
    // ---- D4: unpack, delta outliers ----
    int32_t dl[8];
    unpack_codes(w4, dl);
    patch_deltas(a, sm, s, rlo, rhi, dl);
    // ---- D5 (x, local): segmented inclusive scan, resets at row starts ----
    uint32_t loc[8];
    Seg me{0, 0};
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        if ((xm_rs >> u) & 1u) { me.f = 1; me.v = 0; }
        me.v += (uint32_t)dl[u];
        loc[u] = me.v;
    }
    Seg inc = me;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const Seg up{__shfl_up_sync(kFull, inc.f, o), __shfl_up_sync(kFull, inc.v, o)};
        if (lane >= o) inc = seg_combine(up, inc);
    }
    Seg lex{__shfl_up_sync(kFull, inc.f, 1), __shfl_up_sync(kFull, inc.v, 1)};
    if (lane == 0) lex = Seg{0, 0};
    if (lane == 31) { sm.wf[warp] = inc.f; sm.wv[warp] = inc.v; }
    __syncthreads();
    Seg wp{0, 0}, tagg{0, 0};
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        const Seg sw{sm.wf[w], sm.wv[w]};
        if (w < warp) wp = seg_combine(wp, sw);
        tagg = seg_combine(tagg, sw);
    }
    const Seg acc = seg_combine(wp, lex);
    const uint32_t pre = xm_rs ? ((xm_rs & (0u - xm_rs)) - 1u) : 0xFFu;   // elements before it
#pragma unroll
    for (int u = 0; u < 8; ++u) q[u] = ((pre >> u) & 1u) ? acc.v + loc[u] : loc[u];
    return tagg;
}

// Device-driven mode: the parsed counts are read once per CTA into the CTA's copy of the
// arguments (uniform registers), off every tile's critical path.
__device__ __forceinline__ void resolve_dev(DecodeArgs& a)
{
    if (!a.dev) return;
    a.nnz_total = a.ctrl->dec_nnz;
    a.nd = a.ctrl->dec_nd;
    a.drec = reinterpret_cast<const uint2*>(a.payload + 16 * a.nnz_total);
    a.dev = 0;
}

// One CTA per tile: many tiles in flight per SM.
template <int NDIM>
__global__ void __launch_bounds__(kCta) k_decode_tiles(DecodeArgs a)
{
    pdl_begin();
    resolve_dev(a);
    __shared__ DecSmem sm;
    const int tid = threadIdx.x;
    const uint32_t n = a.g.n;
    const uint32_t t = blockIdx.x;
    const int64_t s = (int64_t)t * kTileCodes;
    const uint32_t g0 = (uint32_t)s + 8u * tid;
    const TileIn in = tile_in(a, t);
    const uint4 blk = tile_blk(a, in);
    uint32_t q[8];
    const Seg tagg = decode_tile_x<NDIM>(a, sm, t, blk, in.rlo, in.rhi, q);
    if (tid == 0) a.xagg[t] = make_uint2(tagg.f, tagg.v);
    if (s + kTileCodes <= (int64_t)n) {
        int4* o = reinterpret_cast<int4*>(a.q_out + g0);
        __stcs(o, make_int4((int)q[0], (int)q[1], (int)q[2], (int)q[3]));
        __stcs(o + 1, make_int4((int)q[4], (int)q[5], (int)q[6], (int)q[7]));
    } else {
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (g0 + u < n) a.q_out[g0 + u] = (int32_t)q[u];
    }
}

// ------------------------------------------------------------------------------------
// D1-D5(x, y) for 3-D fields whose tiles hold R = 2048/nx whole rows of one plane
// (R in {1, 2, 4, 8}): one CTA per plane walks the plane's tiles in order.  After the x scan
// each thread takes C = 8/R whole columns of the tile (all R rows) from shared memory and
// runs the y prefix sum down them with its running column carries in registers, so the y
// scan costs no extra pass over HBM and no inter-CTA communication.  The z scan follows.
// ------------------------------------------------------------------------------------
// C consecutive int32 (or float bits) of one row, streaming store.
template <int C>
__device__ __forceinline__ void store_row(int32_t* o, const uint32_t (&v)[C])
{
    if constexpr (C == 1) {
        __stcs(o, (int32_t)v[0]);
    } else if constexpr (C == 2) {
        __stcs(reinterpret_cast<int2*>(o), make_int2((int)v[0], (int)v[1]));
    } else {
#pragma unroll
        for (int k = 0; k < C; k += 4)
            __stcs(reinterpret_cast<int4*>(o + k), make_int4((int)v[k], (int)v[k + 1], (int)v[k + 2], (int)v[k + 3]));
    }
}

template <int R>
__global__ void __launch_bounds__(kCta) k_decode_planes(DecodeArgs a)
{
    pdl_begin();
    resolve_dev(a);
    constexpr int C = 8 / R;
    __shared__ DecSmem sm;
    const int tid = threadIdx.x;
    // CTA = segment (blockIdx % yseg) of plane (blockIdx / yseg): tiles [k0, k0 + nk)
    const uint32_t nx = a.g.nx, z = blockIdx.x / a.yseg, seg = blockIdx.x % a.yseg;
    const uint32_t nk = a.tpp / a.yseg, t0 = z * a.tpp + seg * nk;
    uint32_t carry[C];
#pragma unroll
    for (int c = 0; c < C; ++c) carry[c] = 0;
    // two-stage software pipeline: payload block of tile k+1, flags/offsets of tile k+2
    TileIn in_cur = tile_in(a, t0);
    uint4 blk_next = tile_blk(a, in_cur);
    TileIn in_next = nk > 1 ? tile_in(a, t0 + 1) : in_cur;
    for (uint32_t k = 0; k < nk; ++k) {
        const uint32_t t = t0 + k;
        const int64_t s = (int64_t)t * kTileCodes;
        const uint4 blk = blk_next;
        const uint32_t rlo = in_cur.rlo, rhi = in_cur.rhi;
        if (k + 1 < nk) {
            blk_next = tile_blk(a, in_next);
            in_cur = in_next;
            if (k + 2 < nk) in_next = tile_in(a, t + 2);
        }
        uint32_t q[8];
        decode_tile_rows<R>(a, sm, s, blk, rlo, rhi, q);
        *reinterpret_cast<uint4*>(sm.D + 8 * tid) = make_uint4(q[0], q[1], q[2], q[3]);
        *reinterpret_cast<uint4*>(sm.D + 8 * tid + 4) = make_uint4(q[4], q[5], q[6], q[7]);
        __syncthreads();
        uint32_t v[R][C];
#pragma unroll
        for (int r = 0; r < R; ++r) {
#pragma unroll
            for (int c = 0; c < C; ++c) {
                carry[c] += (uint32_t)sm.D[r * nx + C * tid + c];
                v[r][c] = carry[c];
            }
        }
        int32_t* o = a.q_out + s + C * tid;
#pragma unroll
        for (int r = 0; r < R; ++r, o += nx) store_row<C>(o, v[r]);
        __syncthreads();    // sm.D and sm.Obuf are reused by the next tile
    }
    // a plane split into yseg segments (CTAs): every segment but the last leaves its column
    // totals; k_yprefix turns them into inclusive prefixes, the y carries the z walk adds to
    // the rows of the segments below
    if (seg + 1 < a.yseg) {
#pragma unroll
        for (int c = 0; c < C; ++c) a.ycarry[((size_t)z * a.yseg + seg) * nx + C * tid + c] = (int32_t)carry[c];
    }
}

// ------------------------------------------------------------------------------------
// f1 chunk-local decode ("highly symmetrical"): with the Lorenzo
// neighbours confined to chunks of cz planes x one tile (R whole rows), a chunk decodes on
// its own -- one pass, no carries between CTAs.  CTA = one chunk column (tile position p,
// planes [z0, z0 + cz)): per plane, gather + un-shuffle + unpack + delta patch + x scan
// (decode_tile_rows), the y prefix down the tile's R rows from shared memory, the z prefix
// in registers, then dequantization (D6) and a streaming store of the fp32 values.
// ------------------------------------------------------------------------------------
template <int R>
__global__ void __launch_bounds__(kCta, 5) k_decode_cl(DecodeArgs a, uint32_t cz)
{
    pdl_begin();
    resolve_dev(a);
    constexpr int C = 8 / R;
    __shared__ DecSmem sm;
    const int tid = threadIdx.x;
    const uint32_t nx = a.g.nx, tpp = a.tpp, nz = a.g.n / a.g.P;
    const uint32_t c = blockIdx.x / tpp, p = blockIdx.x - c * tpp;
    const uint32_t z0 = c * cz, z1 = min(nz, z0 + cz);
    const float w = a.wp ? *a.wp : a.w;
    uint32_t zr[R][C];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int k = 0; k < C; ++k) zr[r][k] = 0u;
    // two-stage software pipeline down z: payload block of plane z+1, flags/offsets of z+2
    TileIn in_cur = tile_in(a, z0 * tpp + p);
    uint4 blk_next = tile_blk(a, in_cur);
    TileIn in_next = z0 + 1 < z1 ? tile_in(a, (z0 + 1) * tpp + p) : in_cur;
    for (uint32_t z = z0; z < z1; ++z) {
        const uint32_t t = z * tpp + p;
        const int64_t s = (int64_t)t * kTileCodes;
        const uint4 blk = blk_next;
        const uint32_t rlo = in_cur.rlo, rhi = in_cur.rhi;
        if (z + 1 < z1) {
            blk_next = tile_blk(a, in_next);
            in_cur = in_next;
            if (z + 2 < z1) in_next = tile_in(a, t + 2 * tpp);
        }
        uint32_t q[8];
        decode_tile_rows<R>(a, sm, s, blk, rlo, rhi, q);
        *reinterpret_cast<uint4*>(sm.D + 8 * tid) = make_uint4(q[0], q[1], q[2], q[3]);
        *reinterpret_cast<uint4*>(sm.D + 8 * tid + 4) = make_uint4(q[4], q[5], q[6], q[7]);
        __syncthreads();
        uint32_t ycar[C];
#pragma unroll
        for (int k = 0; k < C; ++k) ycar[k] = 0u;
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int k = 0; k < C; ++k) {
                ycar[k] += (uint32_t)sm.D[r * nx + C * tid + k];
                zr[r][k] += ycar[k];
            }
        // D6 (or the integer codes for the decode_q hook), one row pointer stepped by nx
        int32_t* o = a.q_out + s + C * tid;
        if (w > 0.0f) {
#pragma unroll
            for (int r = 0; r < R; ++r, o += nx) {
                uint32_t v[C];
#pragma unroll
                for (int k = 0; k < C; ++k) v[k] = __float_as_uint(__fmul_rn(__int2float_rn((int32_t)zr[r][k]), w));
                store_row<C>(o, v);
            }
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r, o += nx) store_row<C>(o, zr[r]);
        }
        __syncthreads();    // sm.D and sm.Obuf are reused by the next plane
    }
}

// Same for short rows (nx < 256, R = 2048 / nx > 8 rows per tile): segmented x scan
// (decode_tile_x; the tile starts on a row), then thread t takes column x = t % nx, rows
// 8g .. 8g+7 (g = t / nx): a local prefix down its 8 rows plus the totals of the groups
// above it (shared memory), and the z prefix of those 8 elements in registers.
__global__ void __launch_bounds__(kCta) k_decode_cl_short(DecodeArgs a, uint32_t cz)
{
    pdl_begin();
    resolve_dev(a);
    __shared__ DecSmem sm;
    const int tid = threadIdx.x;
    const uint32_t nx = a.g.nx, tpp = a.tpp, nz = a.g.n / a.g.P;
    const uint32_t c = blockIdx.x / tpp, p = blockIdx.x - c * tpp;
    const uint32_t z0 = c * cz, z1 = min(nz, z0 + cz);
    const float w = a.wp ? *a.wp : a.w;
    const uint32_t x = (uint32_t)tid % nx, g = (uint32_t)tid / nx;
    uint32_t zr[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) zr[i] = 0u;
    for (uint32_t z = z0; z < z1; ++z) {
        const uint32_t t = z * tpp + p;
        const int64_t s = (int64_t)t * kTileCodes;
        const TileIn in = tile_in(a, t);
        const uint4 blk = tile_blk(a, in);
        uint32_t q[8];
        decode_tile_x<3>(a, sm, t, blk, in.rlo, in.rhi, q);
        __syncthreads();
        *reinterpret_cast<uint4*>(sm.D + 8 * tid) = make_uint4(q[0], q[1], q[2], q[3]);
        *reinterpret_cast<uint4*>(sm.D + 8 * tid + 4) = make_uint4(q[4], q[5], q[6], q[7]);
        __syncthreads();
        uint32_t v[8], acc = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            acc += (uint32_t)sm.D[(8 * g + i) * nx + x];
            v[i] = acc;
        }
        sm.Obuf[tid] = acc;
        __syncthreads();
        uint32_t pre = 0;
        for (uint32_t gg = 0; gg < g; ++gg) pre += sm.Obuf[gg * nx + x];
        int32_t* o = a.q_out + s + (int64_t)(8 * g) * nx + x;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            zr[i] += v[i] + pre;
            const uint32_t out = w > 0.0f ? __float_as_uint(__fmul_rn(__int2float_rn((int32_t)zr[i]), w)) : zr[i];
            __stcs(o + (int64_t)i * nx, (int32_t)out);
        }
        __syncthreads();    // sm.D / sm.Obuf are reused by the next plane
    }
}

// x carries into the elements of a tile whose row began in an earlier tile; 1-D fields are
// dequantized here (D6).  One CTA per tile.
template <int NDIM>
__global__ void __launch_bounds__(kCta) k_xfix(int32_t* q, const uint2* xloc, const uint2* xbpre, uint32_t ntiles,
                                               uint32_t n, uint32_t nx, float w_in, int carries, const float* wp)
{
    pdl_begin();
    const float w = wp ? *wp : w_in;
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint64_t s = (uint64_t)t * kTileCodes;
        uint32_t carry = 0;
        if (carries) {
            const uint2 b = xbpre[t >> 10], l = xloc[t];
            carry = seg_combine(Seg{b.x, b.y}, Seg{l.x, l.y}).v;
        }
        uint64_t e = s + kTileCodes;
        if (e > n) e = n;
        uint64_t r0 = e;           // first row start at or after s
        if (NDIM != 1) {
            const uint64_t rr = (s + nx - 1) / nx * nx;
            if (rr < r0) r0 = rr;
        } else if (s == 0) {
            r0 = 0;
        }
        if (NDIM == 1 && w > 0.0f) {
            for (uint64_t g = s + threadIdx.x; g < e; g += kCta) {
                const uint32_t v = (uint32_t)q[g] + (g < r0 ? carry : 0u);
                reinterpret_cast<float*>(q)[g] = __fmul_rn(__int2float_rn((int32_t)v), w);
            }
        } else if (carry != 0) {
            for (uint64_t g = s + threadIdx.x; g < r0; g += kCta) q[g] = (int32_t)((uint32_t)q[g] + carry);
        }
    }
}

// ------------------------------------------------------------------------------------
// Reduce-then-scan along an axis of [outer][L][W] (wrap-around int32 sums).
// ------------------------------------------------------------------------------------
__global__ void k_scan_sums(const int32_t* __restrict__ v, uint64_t outer, uint64_t L, uint64_t W,
                            uint64_t nch, uint32_t* __restrict__ sums)
{
    pdl_begin();
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
    pdl_begin();
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
                             const uint32_t* __restrict__ sums, float dequant_w_in, const float* wp)
{
    pdl_begin();
    const float dequant_w = wp ? *wp : dequant_w_in;
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
                                                   float dequant_w_in, const int32_t* __restrict__ carry,
                                                   const float* wp)
{
    pdl_begin();
    const float dequant_w = wp ? *wp : dequant_w_in;
    const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= outer * W) return;
    const uint64_t w = gid % W, o = gid / W;
    int32_t* p = v + o * L * W + w;
    uint32_t acc = carry ? (uint32_t)carry[w] : 0u;
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

// Vector walk: V adjacent columns per thread (W % V == 0, rows 16-byte aligned for V = 4),
// U rows in flight; same arithmetic as k_scan_walk.
// ycarry (optional): a column w in plane segment g = (w / ynx) / yrows > 0 also adds
// ycarry[(l * ys + g - 1) * ynx + w % ynx] at step l (the y carry
// of the upper half of a plane decoded as two segments by k_decode_planes).
template <int V, int U>
__global__ void __launch_bounds__(256) k_scan_walk_v(int32_t* v, uint64_t outer, uint64_t L, uint64_t W,
                                                     float dequant_w_in, const int32_t* __restrict__ carry,
                                                     const int32_t* __restrict__ ycarry, uint32_t ynx,
                                                     uint32_t yrows, uint32_t ys,
                                                     const float* wp)
{
    pdl_begin();
    const float dequant_w = wp ? *wp : dequant_w_in;
    using VT = typename std::conditional<V == 4, int4, int2>::type;
    const uint64_t Wv = W / V;
    const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= outer * Wv) return;
    const uint64_t w = (gid % Wv) * V, o = gid / Wv;
    int32_t* p = v + o * L * W + w;
    uint32_t acc[V];
#pragma unroll
    for (int c = 0; c < V; ++c) acc[c] = carry ? (uint32_t)carry[w + c] : 0u;
    auto emit = [&](int32_t* q, const uint32_t (&x)[V]) {
        uint32_t y[V];
#pragma unroll
        for (int c = 0; c < V; ++c) {
            acc[c] += x[c];
            y[c] = dequant_w > 0.0f ? __float_as_uint(__fmul_rn(__int2float_rn((int32_t)acc[c]), dequant_w)) : acc[c];
        }
        if constexpr (V == 4) __stcs(reinterpret_cast<int4*>(q), make_int4((int)y[0], (int)y[1], (int)y[2], (int)y[3]));
        else __stcs(reinterpret_cast<int2*>(q), make_int2((int)y[0], (int)y[1]));
    };
    const uint32_t yg = ycarry != nullptr ? (uint32_t)(w / ynx) / yrows : 0u;
    const int32_t* yc = yg > 0 ? ycarry + (size_t)(yg - 1) * ynx + w % ynx : nullptr;
    const uint64_t ystride = (uint64_t)ys * ynx;
    uint64_t l = 0;
    for (; l + U <= L; l += U) {
        VT x[U];
#pragma unroll
        for (int k = 0; k < U; ++k) x[k] = __ldcs(reinterpret_cast<const VT*>(p + k * W));
        if (yc != nullptr) {
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const VT c = __ldg(reinterpret_cast<const VT*>(yc + (l + k) * ystride));
                if constexpr (V == 4) { x[k].x += c.x; x[k].y += c.y; x[k].z += c.z; x[k].w += c.w; }
                else { x[k].x += c.x; x[k].y += c.y; }
            }
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            uint32_t e[V];
            if constexpr (V == 4) { e[0] = x[k].x; e[1] = x[k].y; e[2] = x[k].z; e[3] = x[k].w; }
            else { e[0] = x[k].x; e[1] = x[k].y; }
            emit(p + k * W, e);
        }
        p += U * W;
    }
    for (; l < L; ++l, p += W) {
        VT x = *reinterpret_cast<const VT*>(p);
        if (yc != nullptr) {
            const VT c = __ldg(reinterpret_cast<const VT*>(yc + l * ystride));
            if constexpr (V == 4) { x.x += c.x; x.y += c.y; x.z += c.z; x.w += c.w; }
            else { x.x += c.x; x.y += c.y; }
        }
        uint32_t e[V];
        if constexpr (V == 4) { e[0] = x.x; e[1] = x.y; e[2] = x.z; e[3] = x.w; }
        else { e[0] = x.x; e[1] = x.y; }
        emit(p, e);
    }
}

__global__ void k_value_patch(float* out, const uint2* rec, uint64_t cnt, uint64_t n, uint64_t base, int logt)
{
    pdl_begin();
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cnt;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint2 r = rec[k];
        if (r.x >= base && r.x - base < n) out[r.x - base] = logt ? exp32(__uint_as_float(r.y)) : __uint_as_float(r.y);
    }
}

// ---- multi-GPU slab decode helpers ----
// agg[w] = sum over l of v[l][w] (mod 2^32): a slab's aggregate along its slowest axis.
__global__ void __launch_bounds__(256) k_axis_sum(const int32_t* __restrict__ v, uint64_t L, uint64_t W,
                                                  int32_t* __restrict__ agg)
{
    pdl_begin();
    const uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= W) return;
    const int32_t* p = v + w;
    uint32_t acc = 0;
    uint64_t l = 0;
    for (; l + 8 <= L; l += 8) {
        uint32_t x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = (uint32_t)__ldcs(p + k * W);
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += x[k];
        p += 8 * W;
    }
    for (; l < L; ++l, p += W) acc += (uint32_t)*p;
    agg[w] = (int32_t)acc;
}

// carry[w] = sum over the lower ranks j < nbefore of aggs[j][w] (mod 2^32).
__global__ void k_slab_carry(const int32_t* __restrict__ aggs, uint32_t nbefore, uint64_t elems, int32_t* carry)
{
    pdl_begin();
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < elems;
         w += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t acc = 0;
        for (uint32_t j = 0; j < nbefore; ++j) acc += (uint32_t)aggs[(uint64_t)j * elems + w];
        carry[w] = (int32_t)acc;
    }
}

// 1-D slab finish: x = fl32(fl32(q + carry) * w).
__global__ void k_add_dequant(int32_t* q, uint64_t n, const int32_t* carry, float w)
{
    pdl_begin();
    const uint32_t c = (uint32_t)carry[0];
    for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n; g += (uint64_t)gridDim.x * blockDim.x)
        reinterpret_cast<float*>(q)[g] = __fmul_rn(__int2float_rn((int32_t)((uint32_t)q[g] + c)), w);
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

cudaError_t launch_decode_init(Ctrl* ctrl, cudaStream_t st)
{
    LaunchProf lp(K_DINIT, st);
    { const cudaError_t e_ = launch_pdl(k_decode_init, dim3(1), dim3(32), 0, st, ctrl); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

cudaError_t launch_validate_outliers(const uint2* rec, uint64_t cnt, uint64_t n, Ctrl* ctrl,
                                     cudaStream_t st)
{
    if (cnt == 0) return cudaSuccess;
    LaunchProf lp(K_VALIDATE, st);
    { const cudaError_t e_ = launch_pdl(k_validate_outliers, dim3(grid_for(cnt)), dim3(256), 0, st, rec, cnt, n, ctrl); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

cudaError_t launch_decode_hdr(Ctrl* ctrl, const uint8_t* in, uint64_t in_size, const fz_shape& s, uint64_t n,
                              uint64_t T, cudaStream_t st)
{
    uint64_t d[3] = {1, 1, 1};
    for (uint32_t k = 0; k < s.ndim && k < 3; ++k) d[k] = s.dims[k];
    LaunchProf lp(K_DINIT, st);
    { const cudaError_t e_ = launch_pdl(k_decode_hdr, dim3(1), dim3(32), 0, st, ctrl, in, in_size, s.ndim, d[0], d[1], d[2], n, T); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

// fixed grids: the record counts are only known on the device
cudaError_t launch_record_tiles(const uint2* drec, uint64_t nd, uint32_t ntiles, uint64_t gbase, uint32_t* drange,
                                cudaStream_t st)
{
    if (nd == 0) return cudaSuccess;
    LaunchProf lp(K_OFFSETS, st);
    { const cudaError_t e_ = launch_pdl(k_record_tiles, dim3(grid_for((uint64_t)ntiles + 1)), dim3(256), 0, st, drec, nd, ntiles, gbase, drange, (const uint8_t*)nullptr, (const Ctrl*)nullptr); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

cudaError_t launch_tile_offsets(const uint8_t* flags, uint32_t ntiles, uint32_t* loc, uint32_t* bsum, Ctrl* ctrl,
                                cudaStream_t st, uint64_t expect_nnz, const uint8_t* vpay, uint64_t vn,
                                uint32_t* drange)
{
    const uint32_t nb = ntiles == 0 ? 1u : (ntiles + 1023) / 1024;   // one block even for no tiles (nnz = 0)
    LaunchProf lp(K_OFFSETS, st);
    return launch_pdl(k_nnz_block, dim3(nb), dim3(1024), 0, st, reinterpret_cast<const uint32_t*>(flags), ntiles, loc,
                      bsum, ctrl, expect_nnz, vpay, vn, drange);
}

template <int NDIM>
static cudaError_t launch_decode_t(const DecodeArgs& a_in, cudaStream_t st)
{
    DecodeArgs a = a_in;
    a.dnx = make_fastdiv(a.g.nx);
    if (a.tiles == 0) return cudaSuccess;
    { const cudaError_t e_ = launch_pdl(k_decode_tiles<NDIM>, dim3(a.tiles), dim3(kCta), 0, st, a); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

cudaError_t launch_decode_tiles(const DecodeArgs& a_in, cudaStream_t st, bool fuse_y)
{
    LaunchProf lp(fuse_y ? K_DECODE_PLANES : K_DECODE, st);
    if (fuse_y) {
        DecodeArgs a = a_in;
        a.dnx = make_fastdiv(a.g.nx);
        const uint32_t ctas = a.g.n / a.g.P * a.yseg;
        switch (kTileCodes / a.g.nx) {
            case 1: { const cudaError_t e_ = launch_pdl(k_decode_planes<1>, dim3(ctas), dim3(kCta), 0, st, a); if (e_ != cudaSuccess) return e_; } break;
            case 2: { const cudaError_t e_ = launch_pdl(k_decode_planes<2>, dim3(ctas), dim3(kCta), 0, st, a); if (e_ != cudaSuccess) return e_; } break;
            case 4: { const cudaError_t e_ = launch_pdl(k_decode_planes<4>, dim3(ctas), dim3(kCta), 0, st, a); if (e_ != cudaSuccess) return e_; } break;
            default: { const cudaError_t e_ = launch_pdl(k_decode_planes<8>, dim3(ctas), dim3(kCta), 0, st, a); if (e_ != cudaSuccess) return e_; } break;
        }
        return cudaGetLastError();
    }
    switch (a_in.g.ndim) {
        case 1: return launch_decode_t<1>(a_in, st);
        case 2: return launch_decode_t<2>(a_in, st);
        default: return launch_decode_t<3>(a_in, st);
    }
}

cudaError_t launch_decode_cl(const DecodeArgs& a_in, uint32_t cz, cudaStream_t st)
{
    DecodeArgs a = a_in;
    a.dnx = make_fastdiv(a.g.nx);
    a.tpp = (uint32_t)(a.g.P / kTileCodes);
    const uint32_t nz = a.g.n / a.g.P;
    const uint64_t ctas = (uint64_t)((nz + cz - 1) / cz) * a.tpp;
    if (ctas == 0) return cudaSuccess;
    LaunchProf lp(K_DECODE_PLANES, st);
    switch (kTileCodes / a.g.nx) {
        case 1: { const cudaError_t e_ = launch_pdl(k_decode_cl<1>, dim3((unsigned)ctas), dim3(kCta), 0, st, a, cz); if (e_ != cudaSuccess) return e_; } break;
        case 2: { const cudaError_t e_ = launch_pdl(k_decode_cl<2>, dim3((unsigned)ctas), dim3(kCta), 0, st, a, cz); if (e_ != cudaSuccess) return e_; } break;
        case 4: { const cudaError_t e_ = launch_pdl(k_decode_cl<4>, dim3((unsigned)ctas), dim3(kCta), 0, st, a, cz); if (e_ != cudaSuccess) return e_; } break;
        case 8: { const cudaError_t e_ = launch_pdl(k_decode_cl<8>, dim3((unsigned)ctas), dim3(kCta), 0, st, a, cz); if (e_ != cudaSuccess) return e_; } break;
        default: { const cudaError_t e_ = launch_pdl(k_decode_cl_short, dim3((unsigned)ctas), dim3(kCta), 0, st, a, cz); if (e_ != cudaSuccess) return e_; } break;
    }
    return cudaGetLastError();
}

cudaError_t launch_xcarry(const DecodeArgs& a, uint2* xloc, uint2* xbagg, bool carries, cudaStream_t st)
{
    const uint32_t nb = (a.tiles + 1023) / 1024;
    if (carries) {
        {
            LaunchProf lp(K_XCARRY, st);
            { const cudaError_t e_ = launch_pdl(k_xseg_block, dim3(nb), dim3(1024), 0, st, a.xagg, a.tiles, xloc, xbagg, a.ctrl); if (e_ != cudaSuccess) return e_; }
        }
    }
    if (!carries && a.g.ndim != 1) return cudaGetLastError();
    unsigned grid = a.tiles < (uint32_t)num_sms() * 8 ? a.tiles : num_sms() * 8;
    LaunchProf lp(K_XCARRY, st);
    switch (a.g.ndim) {
        case 1: { const cudaError_t e_ = launch_pdl(k_xfix<1>, dim3(grid), dim3(kCta), 0, st, a.q_out, xloc, xbagg, a.tiles, a.g.n, a.g.nx, a.w, carries, a.wp); if (e_ != cudaSuccess) return e_; } break;
        case 2: { const cudaError_t e_ = launch_pdl(k_xfix<2>, dim3(grid), dim3(kCta), 0, st, a.q_out, xloc, xbagg, a.tiles, a.g.n, a.g.nx, a.w, carries, nullptr); if (e_ != cudaSuccess) return e_; } break;
        default: { const cudaError_t e_ = launch_pdl(k_xfix<3>, dim3(grid), dim3(kCta), 0, st, a.q_out, xloc, xbagg, a.tiles, a.g.n, a.g.nx, a.w, carries, nullptr); if (e_ != cudaSuccess) return e_; } break;
    }
    return cudaGetLastError();
}

static int walk_mode()
{
    return (variant_bits() >> 8) & 3;
}

// Column walk along L (stride W): vector columns when the rows allow it.
static void launch_walk(int32_t* data, uint64_t outer, uint64_t L, uint64_t W, float w, const int32_t* carry,
                        cudaStream_t st, const int32_t* ycarry = nullptr, uint32_t ynx = 0,
                        const float* wp = nullptr)
{
    const int m = walk_mode();
    const bool a16 = (reinterpret_cast<uintptr_t>(data) & 15) == 0;
    if (m != 3 && W % 4 == 0 && a16 && m != 1) {
        const uint64_t thr = outer * W / 4;
        { (void)launch_pdl(k_scan_walk_v<4, 8>, dim3((unsigned)((thr + 255) / 256)), dim3(256), 0, st, data, outer, L, W, w, carry, ycarry, ynx, 1u, 1u, wp);  /* errors: cudaGetLastError */ }
    } else if (m != 3 && W % 2 == 0 && a16) {
        const uint64_t thr = outer * W / 2;
        { (void)launch_pdl(k_scan_walk_v<2, 8>, dim3((unsigned)((thr + 255) / 256)), dim3(256), 0, st, data, outer, L, W, w, carry, ycarry, ynx, 1u, 1u, wp);  /* errors: cudaGetLastError */ }
    } else {
        { (void)launch_pdl(k_scan_walk, dim3((unsigned)((outer * W + 255) / 256)), dim3(256), 0, st, data, outer, L, W, w, carry, wp);  /* errors: cudaGetLastError */ }
    }
}

cudaError_t launch_scan_axis(int32_t* data, uint64_t outer, uint64_t L, uint64_t W, uint32_t* sums,
                             float dequant_w, cudaStream_t st, const float* wp)
{
    if (outer * W >= 32768) {
        LaunchProf lp(K_SCAN_WALK, st);
        launch_walk(data, outer, L, W, dequant_w, nullptr, st, nullptr, 0, wp);
        return cudaGetLastError();
    }
    const uint64_t nch = (L + kScanChunk - 1) / kScanChunk;
    const uint64_t work = outer * nch * W;
    {
        LaunchProf lp(K_SCAN_SUMS, st);
        { const cudaError_t e_ = launch_pdl(k_scan_sums, dim3(grid_for(work)), dim3(256), 0, st, data, outer, L, W, nch, sums); if (e_ != cudaSuccess) return e_; }
    }
    {
        LaunchProf lp(K_SCAN_CHUNKS, st);
        { const cudaError_t e_ = launch_pdl(k_scan_chunks, dim3(grid_for(outer * W)), dim3(256), 0, st, outer, W, nch, sums); if (e_ != cudaSuccess) return e_; }
    }
    {
        LaunchProf lp(K_SCAN_APPLY, st);
        { const cudaError_t e_ = launch_pdl(k_scan_apply, dim3(grid_for(work)), dim3(256), 0, st, data, outer, L, W, nch, sums, dequant_w, wp); if (e_ != cudaSuccess) return e_; }
    }
    return cudaGetLastError();
}

cudaError_t launch_value_patch(float* out, const uint2* vrec, uint64_t cnt, uint64_t n, cudaStream_t st,
                               uint64_t base, int logt)
{
    if (cnt == 0) return cudaSuccess;
    LaunchProf lp(K_VPATCH, st);
    { const cudaError_t e_ = launch_pdl(k_value_patch, dim3(grid_for(cnt)), dim3(256), 0, st, out, vrec, cnt, n, base, logt); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

cudaError_t launch_axis_sum(const int32_t* v, uint64_t L, uint64_t W, int32_t* agg, cudaStream_t st)
{
    LaunchProf lp(K_SLAB, st);
    { const cudaError_t e_ = launch_pdl(k_axis_sum, dim3((unsigned)((W + 255) / 256)), dim3(256), 0, st, v, L, W, agg); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

cudaError_t launch_slab_carry(const int32_t* aggs, uint32_t nbefore, uint64_t elems, int32_t* carry, cudaStream_t st)
{
    LaunchProf lp(K_SLAB, st);
    { const cudaError_t e_ = launch_pdl(k_slab_carry, dim3(grid_for(elems)), dim3(256), 0, st, aggs, nbefore, elems, carry); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

// in place: the segments' column totals -> inclusive prefixes over the segments of a plane
__global__ void k_yprefix(int32_t* ycarry, uint64_t nz, uint32_t nx, uint32_t ys)
{
    pdl_begin();
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nz * nx) return;
    const uint64_t z = i / nx, x = i - z * nx;
    int32_t* p = ycarry + z * ys * nx + x;
    uint32_t acc = (uint32_t)p[0];
    for (uint32_t g = 1; g + 1 < ys; ++g) {
        acc += (uint32_t)p[(size_t)g * nx];
        p[(size_t)g * nx] = (int32_t)acc;
    }
}

cudaError_t launch_zwalk_ycarry(int32_t* data, uint64_t L, uint64_t W, float w, int32_t* ycarry, uint32_t nx,
                               uint32_t ys, cudaStream_t st, const float* wp)
{
    if (ys > 2) {
        LaunchProf lp(K_OFFSETS, st);
        { const cudaError_t e_ = launch_pdl(k_yprefix, dim3((unsigned)((L * nx + 255) / 256)), dim3(256), 0, st, ycarry, L, nx, ys); if (e_ != cudaSuccess) return e_; }
    }
    LaunchProf lp(K_SCAN_WALK, st);
    if (W % 4 != 0 || (reinterpret_cast<uintptr_t>(data) & 15) != 0) return cudaErrorInvalidValue;
    const uint64_t thr = W / 4;
    { const cudaError_t e_ = launch_pdl(k_scan_walk_v<4, 8>, dim3((unsigned)((thr + 255) / 256)), dim3(256), 0, st, data, 1, L, W, w, nullptr, ycarry, nx,
                                                                        (uint32_t)(W / nx / ys), ys, wp); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

cudaError_t launch_walk_carry(int32_t* data, uint64_t L, uint64_t W, float w, const int32_t* carry, cudaStream_t st)
{
    LaunchProf lp(K_SCAN_WALK, st);
    launch_walk(data, 1, L, W, w, carry, st);
    return cudaGetLastError();
}

cudaError_t launch_add_dequant(int32_t* q, uint64_t n, const int32_t* carry, float w, cudaStream_t st)
{
    LaunchProf lp(K_SLAB, st);
    { const cudaError_t e_ = launch_pdl(k_add_dequant, dim3(grid_for(n)), dim3(256), 0, st, q, n, carry, w); if (e_ != cudaSuccess) return e_; }
    return cudaGetLastError();
}

}  // namespace fz
