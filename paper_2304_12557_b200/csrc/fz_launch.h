// fz_launch.h -- host-side launch wrappers shared by the libfz translation units.
#pragma once

#include <cuda_runtime.h>

#include <utility>

#include "fz_internal.cuh"

namespace fz {

int num_sms();

// Kernel-variant bits for A/B experiments, set only through fz_debug_set_variant (0 = the
// product configuration; never read from the environment).
int variant_bits();
void set_variant_bits(int v);

// Programmatic dependent launch (PDL, sm_90+): a kernel launched by launch_pdl may start
// while its stream predecessor drains; it calls pdl_begin() (griddepcontrol.wait: every
// predecessor grid complete and its memory visible, then launch_dependents) before touching
// anything a predecessor wrote, so the launch latency and CTA ramp-up of each pipeline step
// overlap the previous kernel's tail -- also inside a captured CUDA graph.  Variant bit
// 67108864 launches without the attribute (A/B).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = (variant_bits() & 67108864) ? 0 : 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Kernel kinds for launch accounting and per-kernel CUDA-event timing (fz_profile_*).
enum KernelId {
    K_INIT = 0, K_RANGE, K_PARAMS, K_COMPRESS, K_FINALIZE, K_DINIT, K_VALIDATE, K_DECODE,
    K_SCAN_SUMS, K_SCAN_CHUNKS, K_SCAN_APPLY, K_VPATCH, K_OUTLIERS, K_OFFSETS, K_XCARRY, K_SLAB, K_DECODE_PLANES, K_SCAN_WALK,
    K_COMPACT, K_DZR_SUM, K_DZR_PREP, K_DZR_MAIN, K_LOGT, K_ROWTILES, K_COUNT
};

// Counts one launch of `id` and, when profiling is on, brackets it with CUDA events on the
// launch stream.  Construct right before the <<<>>> launch; the destructor records the end.
struct LaunchProf {
    LaunchProf(KernelId id, cudaStream_t st);
    ~LaunchProf();
    KernelId id;
    cudaStream_t st;
    int slot;              // 1: events are being recorded for this launch
    void* rec = nullptr;   // its pending record (fz_api.cu)
};

// compression (fz_compress.cu)
cudaError_t launch_init(Ctrl* ctrl, unsigned long long* status, uint2* ocnt, uint32_t ntiles,
                        const fz_params* p, cudaStream_t st, uint32_t chunk = 0);
cudaError_t launch_range(const float* d, uint64_t n, Ctrl* ctrl, cudaStream_t st);
cudaError_t launch_params(Ctrl* ctrl, int mode, double eb, uint64_t n, cudaStream_t st);
cudaError_t launch_compress(const CompressArgs& a, cudaStream_t st);
bool compress_uses_ws(const CompressArgs& a);   // the warp-specialized kernel takes this launch
bool compress_uses_zb(const CompressArgs& a);   // the z-band two-pass compressor takes it
cudaError_t launch_compress_zb(const CompressArgs& a, cudaStream_t st);
bool compress_uses_rc(const CompressArgs& a);   // the row-codes two-pass path takes it (fz_rowcodes.cu)
bool rc_layout_shape(const fz_shape& s);
cudaError_t launch_compress_rc(const CompressArgs& a, cudaStream_t st);
bool compress_uses_zr(const CompressArgs& a);   // the row-walking z-band compressor takes it (fz_zrow.cu)
cudaError_t launch_compress_zr(const CompressArgs& a, cudaStream_t st);
// C8 + C9: compaction of the staged blocks, and (thread 0) the totals + header of k_finalize
cudaError_t launch_compact(const uint8_t* flags, const uint32_t* loc, const uint32_t* bpre, const uint4* tstage,
                           uint8_t* payload_out, uint64_t payload_cap, uint32_t ntiles, uint8_t* hdr_out,
                           uint64_t hdr_cap, const fz_shape& s, uint64_t n, uint64_t T, Ctrl* ctrl, cudaStream_t st);
cudaError_t launch_finalize(uint8_t* out, uint64_t cap, const fz_shape& s, uint64_t n,
                            uint64_t T, Ctrl* ctrl, cudaStream_t st);
cudaError_t launch_outlier_scan(const uint2* ocnt, uint2* opre, uint32_t ntiles, cudaStream_t st,
                                const Ctrl* ctrl = nullptr);
cudaError_t launch_outlier_place_dev(const uint2* ocnt, const uint2* obase, const uint2* opre, uint32_t ntiles,
                                     const uint2* dstage, const uint2* vstage, uint8_t* payload_out,
                                     uint64_t payload_cap, Ctrl* ctrl, cudaStream_t st);
cudaError_t launch_outlier_place(const uint2* ocnt, const uint2* obase, const uint2* opre,
                                 uint32_t ntiles, const uint2* dstage, const uint2* vstage,
                                 uint2* dout, uint2* vout, uint32_t* didx, int32_t* dval,
                                 uint32_t* vidx, uint32_t* vbits, cudaStream_t st);

// decompression (fz_decompress.cu)
struct DecodeArgs {
    const uint8_t* flags;       // 32 B per tile
    const uint8_t* payload;     // 16 B blocks
    const uint2* drec;          // (idx, delta) records, ascending idx
    uint64_t nnz_total;         // header nnz (bounds every payload read)
    uint64_t nd;
    Geom g;
    FastDiv dnx;
    uint32_t tiles;
    float w;
    int32_t* q_out;             // integer codes (aliases the output field)
    uint64_t gbase;             // global element index of local element 0 (slab decode)
    const uint32_t* loc;        // per-tile block offset inside its group of 1024 tiles
    const uint32_t* bpre;       // exclusive block offset of each group of 1024 tiles
    uint2* xagg;                // per-tile x-scan aggregate (row start seen, sum)
    Ctrl* ctrl;
    uint32_t tpp;               // tiles per plane (fused y scan)
    uint32_t yseg;              // CTAs (segments) per plane: 1, or 2 with the carry in ycarry
    int32_t* ycarry;            // [nz][nx] column totals of the lower segment (yseg == 2)
    const uint32_t* drange;     // per-tile delta-outlier record ranges (k_record_tiles)
    int dev;                    // 1: nnz / n_delta / delta records come from ctrl (k_decode_hdr)
    const float* wp;            // device bin width for dequantization (dev mode), else null
};

// The y scan runs inside the decode (one CTA per plane) when every tile holds whole rows of
// one plane and there are enough planes to fill the GPU.
bool decode_fuses_y(const fz_shape& s);

// f3 log transform (fz_logt.cu): y = log32(x) with the domain check (first bad index and
// status into ctrl), and x^ = exp32(y^) in place (dev_ctrl: only when its dec_flags bit 3)
cudaError_t launch_log_fwd(const float* x, float* y, uint64_t n, Ctrl* ctrl, cudaStream_t st);
cudaError_t launch_exp_inv(float* v, uint64_t n, const Ctrl* dev_ctrl, cudaStream_t st);
// device-parsed decode: value patch + (header bit 3) exp32 in one launch (fz_logt.cu)
cudaError_t launch_patch_exp_dev(float* v, const uint8_t* payload, Ctrl* ctrl, uint64_t n, cudaStream_t st);

// Row-walking decoder (fz_dzr.cu): 3-D, nx % 128 == 0, nx <= 1024, ny % 16 == 0.
struct DzrArgs {
    const uint8_t* flags;
    const uint8_t* payload;
    const uint2* drec;
    uint64_t nnz_total, nd;
    int dev;                    // 1: counts from ctrl (device-parsed header)
    const float* wp;            // device bin width (dev mode), else null
    float w;                    // > 0: dequantize; 0: integer codes out
    Ctrl* ctrl;
    const uint32_t* loc;
    const uint32_t* bpre;
    const uint32_t* drange;
    int32_t* q_out;
    uint32_t nx, nz, P, tpp, nbands, nchunks;
    int32_t* cdelta;            // [nbands][nz][nx]  column delta sums -> V (y carries)
    int32_t* dsum;              // [nbands][nchunks][16][nx] chunk delta sums -> prefixes
    int32_t* cd;                // [nbands][nchunks][nx] chunk column sums -> G
    uint16_t* codes;            // dzg: the un-shuffled code field (tiles x 2048), else null
    uint32_t ny, cz;            // dzg: rows (last band may be partial), planes per chunk
    uint32_t ntiles;
    int logt;                   // f3: x^ = exp32(fl32(q) w) (header flag bit 3); -1: from ctrl (dev)
};
struct DzrLayout {
    uint32_t nbands, nchunks, cz;
    uint64_t cdelta_elems, dsum_elems, cd_elems, code_bytes;
};
bool decode_uses_dzr(const fz_shape& s);
DzrLayout dzr_layout(const fz_shape& s);
// planes per unit of the row-walking decoders' persistent grids of G CTAs (fz_dzr.cu)
uint32_t dz_chunk_depth(uint64_t nz, uint32_t nbands, uint64_t G);
cudaError_t launch_decode_dzr(const DzrArgs& a, cudaStream_t st);
cudaError_t launch_dzr_prep(const DzrArgs& a, cudaStream_t st);
// 1-D fields: tile sums, their scan, then the decode with the carries (fz_dzr.cu)
cudaError_t launch_decode_1d(const DzrArgs& a, uint64_t n, uint32_t* tsum, uint32_t* loc, uint32_t* bsum,
                             cudaStream_t st);
// General row-walking decoder (fz_dzg.cu): 3-D, nx % 4 == 0, 64 <= nx <= 1024, nz >= 256;
// the tiles are first un-shuffled into a code field (k_untile), then pass 1 / prep / pass 2
// walk rows of that field.
bool decode_uses_dzg(const fz_shape& s);
DzrLayout dzg_layout(const fz_shape& s);
cudaError_t launch_decode_dzg(const DzrArgs& a, cudaStream_t st);

constexpr uint32_t kMaxYseg = 8;   // plane segments (CTAs) per plane in k_decode_planes
struct DecodeLayout {
    size_t ctrl, loc, bsum, xagg, xloc, xbagg, sums, drange, ycarry, dzr_cdelta, dzr_dsum, dzr_cd, dzg_codes, total;
    uint64_t sums_elems;
};
DecodeLayout decode_layout(const fz_shape& s);

cudaError_t launch_decode_init(Ctrl* ctrl, cudaStream_t st);
cudaError_t launch_validate_outliers(const uint2* rec, uint64_t cnt, uint64_t n, Ctrl* ctrl,
                                     cudaStream_t st);
cudaError_t launch_tile_offsets(const uint8_t* flags, uint32_t ntiles, uint32_t* loc, uint32_t* bsum, Ctrl* ctrl,
                                cudaStream_t st, uint64_t expect_nnz, const uint8_t* vpay = nullptr, uint64_t vn = 0,
                                uint32_t* drange = nullptr);
// device-driven decode (counts parsed from the stream header on the device)
cudaError_t launch_decode_hdr(Ctrl* ctrl, const uint8_t* in, uint64_t in_size, const fz_shape& s, uint64_t n,
                              uint64_t T, cudaStream_t st);
cudaError_t launch_record_tiles(const uint2* drec, uint64_t nd, uint32_t ntiles, uint64_t gbase, uint32_t* drange,
                                cudaStream_t st);
cudaError_t launch_decode_tiles(const DecodeArgs& a, cudaStream_t st, bool fuse_y = false);
cudaError_t launch_xcarry(const DecodeArgs& a, uint2* xloc, uint2* xbagg, bool carries, cudaStream_t st);
// f1 chunk-local decode (chunks of cz planes x one whole-row tile): one pass, dequantized
cudaError_t launch_decode_cl(const DecodeArgs& a, uint32_t cz, cudaStream_t st);
// inclusive prefix sum along an axis of a [outer][L][W] int32 array (mod 2^32); when
// dequant_w > 0 the final values are written as fl32(fl32(q) * w) floats in place.
// wp (device, optional) supplies the bin width instead of dequant_w (device-driven decode).
cudaError_t launch_scan_axis(int32_t* data, uint64_t outer, uint64_t L, uint64_t W,
                             uint32_t* sums, float dequant_w, cudaStream_t st, const float* wp = nullptr);
cudaError_t launch_value_patch(float* out, const uint2* vrec, uint64_t cnt, uint64_t n,
                               cudaStream_t st, uint64_t base = 0, int logt = 0);
cudaError_t launch_axis_sum(const int32_t* v, uint64_t L, uint64_t W, int32_t* agg, cudaStream_t st);
cudaError_t launch_slab_carry(const int32_t* aggs, uint32_t nbefore, uint64_t elems, int32_t* carry,
                              cudaStream_t st);
cudaError_t launch_zwalk_ycarry(int32_t* data, uint64_t L, uint64_t W, float w, int32_t* ycarry, uint32_t nx,
                               uint32_t ys, cudaStream_t st, const float* wp = nullptr);
cudaError_t launch_walk_carry(int32_t* data, uint64_t L, uint64_t W, float w, const int32_t* carry,
                              cudaStream_t st);
cudaError_t launch_add_dequant(int32_t* q, uint64_t n, const int32_t* carry, float w, cudaStream_t st);

}  // namespace fz
