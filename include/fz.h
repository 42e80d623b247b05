/*
 * fz.h -- C ABI of the B200-native FZ-GPU compressor (arXiv 2304.12557), libfz.so.
 *
 * Citation key: P:n = PAPER.md line n, S:n = SPEC.md line n, SV = SURVEY.md, DESIGN.md §3
 * lists the readings R1-R22 that fix everything the paper leaves open.
 *
 * Problem statement: the data is produced on the GPU and compressed "directly ...
 * from the GPU memory"; the compressed stream is cached in GPU memory and "decompressed on the
 * GPU directly", or saved to disk via the CPU.  Hence: every field/stream pointer below is a
 * DEVICE pointer unless its name starts with h_, and work is enqueued on `stream`
 * (a cudaStream_t passed as void*; NULL = legacy default stream).
 *
 * Ownership: the caller allocates every buffer (typically torch tensors).  The library never
 * allocates device memory and retains no pointer after a call returns.  Calls are re-entrant
 * given separate workspaces.  Device pointers must be 16-byte aligned.
 *
 * Errors: status codes only (fz_status); nothing crosses the ABI as an exception.  A CUDA
 * runtime failure returns FZ_ERR_CUDA (the CUDA error string is available from
 * fz_last_cuda_error()).
 */
#ifndef FZ_H
#define FZ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* FZ_EB_ABS: |x^ - x| <= eb.  FZ_EB_REL: eb_abs = eb * (max - min).
 * FZ_EB_PWREL (f3, "transform the original data using a logarithmic function and
 * compress the log-transformed data with the corresponding absolute error bound"): the
 * point-wise relative bound |x^ - x| <= eb |x|, 0 < eb < 1, for fields of positive normal
 * floats (x >= FLT_MIN; zero, negative or subnormal -> FZ_ERR_ARG, NaN/Inf ->
 * FZ_ERR_NONFINITE).  y = log x (reading R25: a fixed binary64 sequence rounded once) is
 * compressed with the ABS bound of R25 and the decoder returns x^ = exp y^; header flag bit 3.
 * Needs fz_workspace_bytes_mode(s, FZ_EB_PWREL) of compress workspace (the log field lives
 * there); not combinable with FZ_CHUNK_LOCAL or the slab API (FZ_ERR_ARG). */
typedef enum { FZ_EB_ABS = 0, FZ_EB_REL = 1, FZ_EB_PWREL = 2 } fz_eb_mode;

/* f1 ("chunked data blocks can be compressed independently"): OR
 * into eb_mode of fz_compress / fz_compress_async to select the chunk-local Lorenzo
 * predictor.  Neighbours in another chunk count as zero, a chunk being 16 planes x one tile
 * (2048 / nx whole rows) of a 3-D field, so each chunk decodes on its own in one pass.
 * Shapes: 3-D, nz >= 2, nx % 4 == 0, nx divides 2048, (ny * nx) % 2048 == 0; otherwise
 * FZ_ERR_ARG.  The stream sets header flag bit 2 and stores the chunk depth / height as
 * u16 at bytes 10 / 12.  fz_decompress and fz_decompress_hdr read either variant;
 * fz_decompress_async reports FZ_ERR_ARG for a chunk-local stream.  More than N/64 + 1024
 * outliers of one kind return FZ_ERR_WORKSPACE in this mode (no rescan pass). */
#define FZ_CHUNK_LOCAL 0x100

typedef enum {
    FZ_OK = 0,
    FZ_ERR_ARG = 1,          /* ndim not in {1,2,3}, zero extent, N >= 2^32, eb <= 0 or
                                non-finite, NULL or misaligned pointer                     */
    FZ_ERR_NONFINITE = 2,    /* NaN/Inf in the field; first index reported           */
    FZ_ERR_EB_TOO_SMALL = 3, /* bin width w below FLT_MIN (reading R17)                     */
    FZ_ERR_CAPACITY = 4,     /* output too small: *out_size = required size, nothing
                                written past out_cap (snprintf convention)                 */
    FZ_ERR_CORRUPT = 5,      /* stream fails magic/version/size-law/popcount/index checks   */
    FZ_ERR_WORKSPACE = 6,    /* workspace smaller than fz_*workspace_bytes()                */
    FZ_ERR_CUDA = 7
} fz_status;

/* Field shape: dims[0] slowest (z), dims[ndim-1] fastest (x); row-major fp32. */
typedef struct {
    uint32_t ndim;
    uint32_t reserved;
    uint64_t dims[3];
} fz_shape;

/* Quantization parameters (P:129-134 with reading R2 = SURVEY Appendix A). */
typedef struct {
    double eb_input;   /* eb as given                                             */
    double eb_abs;     /* eb (ABS) or eb*(max-min) (REL)                    */
    float w;           /* bin width: RD32(2 eb_abs - U), U = ulp of binade above M */
    float r;           /* (float)(1/(double)w)                                     */
    float eb32;        /* RD32(eb_abs)                                             */
    float mn, mx;      /* field range (-0.0 counted as +0.0, R18)                  */
    uint32_t mode;     /* fz_eb_mode                                               */
    uint32_t fallback; /* 1 when the margin mode is infeasible (R2)                */
} fz_params;

/* Section sizes of one stream (or of one slab's share of it). */
typedef struct {
    uint64_t nnz;      /* nonzero 16-byte blocks      */
    uint64_t n_delta;  /* delta outliers, |delta| > 32767 (R7) */
    uint64_t n_value;  /* value outliers (R20)                 */
} fz_counts;

/* Decoded 128-byte header. */
typedef struct {
    fz_shape shape;
    uint64_t n, tiles, total_size;
    fz_counts counts;
    fz_params params;
    uint32_t version, flags;
} fz_info;

/* ---------------------------------------------------------------------------------------
 * Sizes.  T = ceil(N / 2048) tiles of 32x32 words, 2 codes per word.
 * ------------------------------------------------------------------------------------- */
/* 128 + 32T + 4096T + 16N: safe upper bound of the stream (every block and every element
 * an outlier).  0 if the shape is invalid. */
size_t fz_compress_bound(const fz_shape* s);
/* Device workspace needed by fz_compress / fz_compress_with_params / slab calls. */
size_t fz_workspace_bytes(const fz_shape* s);
/* The same for a given eb_mode: FZ_EB_PWREL adds 4N bytes (the log field). */
size_t fz_workspace_bytes_mode(const fz_shape* s, int eb_mode);
/* Device workspace needed by fz_decompress. */
size_t fz_decompress_workspace_bytes(const fz_shape* s);

/* ---------------------------------------------------------------------------------------
 * Parameters (host).  Appendix A of SURVEY.md; identical on every rank for identical
 * (min, max, mode, eb).
 * ------------------------------------------------------------------------------------- */
fz_status fz_derive_params(float mn, float mx, int eb_mode, double eb, fz_params* h_params);

/* ---------------------------------------------------------------------------------------
 * Compression: range -> prequantize -> Lorenzo -> codes -> bitshuffle -> block
 * flags -> exclusive scan -> compaction.  3-D fields whose 16-row bands are whole tiles (c4):
 * one persistent kernel takes the range (its first phase) through the flags and staged blocks,
 * then one popcount-scan launch and one compaction launch (+ header); other shapes: a range
 * launch, then a row-codes walk + tiling pass or a single-pass kernel with a decoupled
 * look-back.  Blocks once on `stream` to return *out_size (host).
 *   d_field   : N fp32, device, row-major
 *   d_out     : device, out_cap bytes; receives header || flags || payload || outliers
 *   d_work    : device workspace of fz_workspace_bytes(s) bytes
 * A NaN / Inf anywhere in the field returns FZ_ERR_NONFINITE (fz_slab_range reports the
 * first such index).
 * ------------------------------------------------------------------------------------- */
fz_status fz_compress(const float* d_field, const fz_shape* s, int eb_mode, double eb,
                      void* d_out, size_t out_cap, size_t* h_out_size,
                      void* d_work, size_t work_bytes, void* stream);

/* Same with parameters supplied by the caller (skips the range pass; multi-GPU ranks and
 * idempotence tests use it).  h_params must come from fz_derive_params. */
fz_status fz_compress_with_params(const float* d_field, const fz_shape* s,
                                  const fz_params* h_params,
                                  void* d_out, size_t out_cap, size_t* h_out_size,
                                  void* d_work, size_t work_bytes, void* stream);

/* Decompression: parse, offsets from flags, gather, un-shuffle, unpack + delta patch,
 * inverse-Lorenzo prefix sums, x-hat = fl32(fl32(q) * w) + value patch.  Blocks once on
 * `stream` to read the header.  d_field receives n fp32 values (n must equal the header's N). */
fz_status fz_decompress(const void* d_in, size_t in_size, float* d_field, uint64_t n,
                        void* d_work, size_t work_bytes, void* stream);

/* Same, with the 128-byte header supplied from host memory (h_hdr, e.g. from fz_last_header
 * after the fz_compress that produced d_in): no blocking header read before the launches;
 * blocks once at the end for the status.  h_hdr must be the header of d_in -- the section
 * bounds it implies are checked against in_size, and every device read stays inside them,
 * but a header that does not belong to the stream decodes to garbage. */
fz_status fz_decompress_hdr(const void* d_in, size_t in_size, const void* h_hdr, float* d_field,
                            uint64_t n, void* d_work, size_t work_bytes, void* stream);

/* Asynchronous compression: the whole pipeline (range, parameters, fused kernel, outlier
 * placement) is enqueued on `stream` with no host round trip.  fz_compress_result waits for
 * `stream` and returns the status and the stream size (FZ_ERR_CAPACITY if it exceeds
 * out_cap).  A staging overflow (more than N/64 + 1024 outliers of one kind; the synchronous
 * fz_compress handles it with a second pass) is reported as FZ_ERR_WORKSPACE. */
fz_status fz_compress_async(const float* d_field, const fz_shape* s, int eb_mode, double eb,
                            void* d_out, size_t out_cap, void* d_work, size_t work_bytes, void* stream);
fz_status fz_compress_result(const void* d_work, size_t out_cap, size_t* h_out_size, void* stream);

/* Asynchronous form of fz_decompress_hdr: enqueues the decode on `stream` and returns without
 * waiting; argument errors are returned at once, stream errors (corrupt input, a popcount that
 * disagrees with nnz) are recorded in d_work and returned by fz_decompress_result, which waits
 * for `stream`.  d_field is valid only once fz_decompress_result returns FZ_OK. */
fz_status fz_decompress_hdr_async(const void* d_in, size_t in_size, const void* h_hdr, float* d_field,
                                  uint64_t n, void* d_work, size_t work_bytes, void* stream);
fz_status fz_decompress_result(const void* d_work, void* stream);

/* Fully device-driven asynchronous decompression: the host supplies only the expected shape
 * (launch configuration); the stream header is parsed and checked on the device (magic,
 * version, shape, N, tile count, size law against in_size) and every kernel takes the section
 * counts and the bin width from the workspace.  Nothing blocks; the status comes from
 * fz_decompress_result.  Lets a compress -> decompress pipeline run without host round trips
 * (and be captured in a CUDA graph). */
fz_status fz_decompress_async(const void* d_in, size_t in_size, const fz_shape* s, float* d_field,
                              void* d_work, size_t work_bytes, void* stream);

/* Copies the header of the last successful fz_compress / fz_compress_with_params on this
 * thread (128 bytes, the same bytes as the stream's header) to h_hdr.  FZ_ERR_ARG if none. */
fz_status fz_last_header(void* h_hdr);

/* Host-buffer variants (end-to-end path): H2D of the input, the device call, D2H of the
 * result, all on `stream`.  The caller passes device scratch of the stated sizes.
 *   compress  : d_field_scratch >= 4N bytes, d_out_scratch >= d_out_cap bytes.
 *   decompress: d_in_scratch >= in_size bytes, d_field_scratch >= 4n bytes. */
fz_status fz_compress_host(const float* h_field, const fz_shape* s, int eb_mode, double eb,
                           void* h_out, size_t out_cap, size_t* h_out_size,
                           float* d_field_scratch, void* d_out_scratch, size_t d_out_cap,
                           void* d_work, size_t work_bytes, void* stream);
fz_status fz_decompress_host(const void* h_in, size_t in_size, float* h_field, uint64_t n,
                             void* d_in_scratch, float* d_field_scratch,
                             void* d_work, size_t work_bytes, void* stream);

/* Parse and validate a header (host memory, n >= 128 bytes).  Checks magic, version, shape
 * and the size law; popcount and index checks need the whole stream (fz_decompress). */
fz_status fz_peek_header(const void* h_hdr, size_t n, fz_info* h_info);

const char* fz_strerror(int status);
const char* fz_last_cuda_error(void);

/* ---------------------------------------------------------------------------------------
 * Slab API for multi-GPU z-slab partitioning ("embarrassingly parallel"; SV §8.e).
 * Rank-local calls; the caller does the NCCL all_gathers.  Tiles are global: rank k owns
 * tiles [tile_begin, tile_end).  The slab buffer d_slab holds the global elements
 * [slab_first, slab_first + slab_elems), which must cover [2048*tile_begin - (P + nx + 1),
 * min(N, 2048*tile_end)) clamped at 0 (the read-only 1-plane + 1-row + 1-element Lorenzo
 * halo).  slab_first must be a multiple of 4.
 * ------------------------------------------------------------------------------------- */

/* Range of d_slab[0..n): min, max (R18), first non-finite index (-1 if none). */
fz_status fz_slab_range(const float* d_slab, uint64_t n, float* h_min, float* h_max,
                        int64_t* h_first_bad, void* d_work, size_t work_bytes, void* stream);

/* Compress the slab's tiles into d_stage laid out as the slab's share of every section:
 * flags (32 * ntiles) || payload (16 * nnz) || delta records (8 * n_delta) || value records
 * (8 * n_value).  *h_counts receives the local counts.  stage_cap >= fz_slab_stage_bound. */
size_t fz_slab_stage_bound(const fz_shape* global, uint64_t tile_begin, uint64_t tile_end);
fz_status fz_slab_compress(const float* d_slab, uint64_t slab_first, uint64_t slab_elems,
                           const fz_shape* global, uint64_t tile_begin, uint64_t tile_end,
                           const fz_params* h_params, void* d_stage, size_t stage_cap,
                           fz_counts* h_counts, void* d_work, size_t work_bytes, void* stream);

/* Copy a staged slab to its final place in the global stream buffer d_out (total bytes
 * out_cap): `before` = exclusive prefix of the counts of lower ranks, `totals` = global sums.
 * The rank owning tile 0 also passes write_header = 1. */
fz_status fz_slab_place(const void* d_stage, const fz_shape* global, uint64_t tile_begin,
                        uint64_t tile_end, const fz_counts* local, const fz_counts* before,
                        const fz_counts* totals, const fz_params* h_params, int write_header,
                        void* d_out, size_t out_cap, void* stream);

/* Slab decompression (plane-aligned z-slabs: 2048*tile_begin and 2048*tile_end are multiples
 * of the plane size P = ny*nx (3-D), of nx (2-D), or any tile boundary (1-D)).  The inverse
 * Lorenzo prefix sums need, besides the slab's own share of the stream (d_stage, as written
 * by fz_slab_compress), one carry from the lower ranks: the sum over all earlier planes
 * (3-D), rows (2-D) or elements (1-D).  Protocol per rank k:
 *   fz_slab_decode   : local decode; d_q (int32, the slab's elements) holds the x- (and y-)
 *                      scanned codes, d_agg (agg_elems int32) the slab's aggregate;
 *   all_gather of d_agg (NCCL), then fz_slab_carry over the k lower ranks' aggregates;
 *   fz_slab_finish   : carry-seeded scan along the slowest axis, x-hat = fl32(fl32(q) w)
 *                      written over d_q as fp32, value outliers patched.
 * agg_elems = P (3-D), nx (2-D), 1 (1-D): fz_slab_agg_elems.  d_work: fz_decompress_workspace_
 * bytes of the slab's own shape (<= that of the global shape). */
uint64_t fz_slab_agg_elems(const fz_shape* global);
fz_status fz_slab_decode(const void* d_stage, const fz_counts* local, const fz_shape* global,
                         uint64_t tile_begin, uint64_t tile_end, int32_t* d_q, int32_t* d_agg,
                         void* d_work, size_t work_bytes, void* stream);
fz_status fz_slab_carry(const int32_t* d_aggs, uint32_t nranks_before, uint64_t agg_elems,
                        int32_t* d_carry, void* stream);
fz_status fz_slab_finish(int32_t* d_q, const int32_t* d_carry, const void* d_stage,
                         const fz_counts* local, const fz_shape* global, uint64_t tile_begin,
                         uint64_t tile_end, const fz_params* h_params, void* stream);

/* f1 chunk-local slabs ("multi-GPU decode needs no exchange").  OR
 * FZ_CHUNK_LOCAL into h_params->mode for fz_slab_compress and fz_slab_place (the header then
 * carries flag bit 2 and the chunk dims); the slab's planes must start on a chunk boundary
 * (a multiple of 16 planes) and end on one or at nz, on a FZ_CHUNK_LOCAL shape, else
 * FZ_ERR_ARG.  Such a slab decodes on its own, with no carry from other ranks:
 *   d_out : the slab's own elements [2048*tile_begin, min(N, 2048*tile_end)) as fp32 x-hat,
 *           value outliers patched.  d_work as for fz_slab_decode. */
fz_status fz_slab_decode_cl(const void* d_stage, const fz_counts* local, const fz_shape* global,
                            uint64_t tile_begin, uint64_t tile_end, const fz_params* h_params,
                            float* d_out, void* d_work, size_t work_bytes, void* stream);

/* ---------------------------------------------------------------------------------------
 * Stage hooks for parity tests (north star: codes and outlier lists match the oracle).
 * ------------------------------------------------------------------------------------- */
/* Workspace of fz_debug_quantize: the compression workspace plus scratch for the flag and
 * payload sections the product kernels write (32 T + 4096 T bytes). */
size_t fz_debug_workspace_bytes(const fz_shape* s);
/* C1-C3: uint16 codes of every element and both outlier lists (ascending index), produced by
 * the same kernels fz_compress launches for the shape (codes written as a side output).
 * d_work: fz_debug_workspace_bytes(s) bytes, else FZ_ERR_WORKSPACE. */
fz_status fz_debug_quantize(const float* d_field, const fz_shape* s, const fz_params* h_params,
                            uint16_t* d_codes,
                            uint32_t* d_didx, int32_t* d_dval, uint64_t dcap, uint64_t* h_nd,
                            uint32_t* d_vidx, uint32_t* d_vbits, uint64_t vcap, uint64_t* h_nv,
                            void* d_work, size_t work_bytes, void* stream);
/* D1-D5: reconstructed integer codes q (before dequantization), n int32 values. */
fz_status fz_debug_decode_q(const void* d_in, size_t in_size, int32_t* d_q, uint64_t n,
                            void* d_work, size_t work_bytes, void* stream);

/* Kernel variants for A/B experiments (tools/ablation.py): process-wide bits, 0 = the
 * product configuration.  16: generic fused compressor; 1024: warp-specialized single-pass
 * compressor instead of the z-band one; 128: unfused decoder y scan; 512 / 4096: plane decoder
 * with one / two CTAs per plane; 2097152: k_range launched before the row walker instead of
 * the walker's fused range phase (SV 8.f2); 4194304: the fused range phase reads its chunks in
 * address order; 33554432: 16-plane units in the row-walking decoder instead of the balanced
 * depth; 8388608: per-CTA residency trace of the row walker (fz_debug_zr_trace); 67108864:
 * kernels launched without programmatic dependent launch; 268435456: the general row-walking
 * decoder only for nz >= 256 (the tile decoder below; set before sizing the decompress
 * workspace).  Streams are byte-identical under every variant. */
void fz_debug_set_variant(int bits);

/* Row-walker residency trace (variant 8388608): copies up to n (<= 8192) u64 to host_out,
 * 4 per CTA of the last walker launch: globaltimer ns at start, SM id, end of the fused range
 * phase (0 without it), end.  Returns the count copied, -1 on a CUDA error.  Debug only. */
int fz_debug_zr_trace(unsigned long long* host_out, int n);

/* Number of kernel launches issued by the last fz_compress / fz_decompress on this thread
 * (bench accounting of "gpu_launches"). */
int fz_last_launch_count(void);

/* Per-kernel CUDA-event timing (tracing).  When enabled, every libfz kernel launch is
 * bracketed by two CUDA events recorded on its launch stream.  fz_profile_read waits for
 * the pending events, writes the summed milliseconds and launch counts per kernel kind
 * (indices 0..n-1, names from fz_kernel_name) and resets the totals; returns n. */
void fz_profile_enable(int on);
/* Restrict profiling to the kernels whose ids (fz_kernel_name order) are set in `mask`; the
 * others launch without event records.  fz_profile_enable resets the mask to all kernels. */
void fz_profile_mask(unsigned long long mask);

int fz_profile_read(double* h_ms, int* h_launches, int max_kernels);

/* Timeline of the launches recorded since the last fz_profile_read (profiling on): kernel id,
 * start and end of each launch's event pair in ms relative to the first one.  Does not clear.
 * Returns the number of records written (<= max_records). */
int fz_profile_timeline(int* h_ids, float* h_start_ms, float* h_end_ms, int max_records);
const char* fz_kernel_name(int id);

#ifdef __cplusplus
}
#endif
#endif /* FZ_H */
