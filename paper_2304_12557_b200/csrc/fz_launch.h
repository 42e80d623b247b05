// fz_launch.h -- host-side launch wrappers shared by the libfz translation units.
#pragma once

#include <cuda_runtime.h>

#include "fz_internal.cuh"

namespace fz {

void count_launch();
int num_sms();

// compression (fz_compress.cu)
cudaError_t launch_init(Ctrl* ctrl, unsigned long long* status, uint32_t ntiles,
                        const fz_params* p, cudaStream_t st);
cudaError_t launch_range(const float* d, uint64_t n, Ctrl* ctrl, cudaStream_t st);
cudaError_t launch_params(Ctrl* ctrl, int mode, double eb, uint64_t n, cudaStream_t st);
cudaError_t launch_compress(const CompressArgs& a, cudaStream_t st);
cudaError_t launch_finalize(uint8_t* out, uint64_t cap, const fz_shape& s, uint64_t n,
                            uint64_t T, const uint2* dstage, const uint2* vstage, Ctrl* ctrl,
                            cudaStream_t st);

// decompression (fz_decompress.cu)
struct DecodeArgs {
    const uint8_t* flags;       // 32 B per tile
    const uint8_t* payload;     // 16 B blocks
    const uint2* drec;          // (idx, delta) records, ascending idx
    uint64_t nnz_total;         // header nnz (bounds every payload read)
    uint64_t nd;
    Geom g;
    uint32_t tiles;
    float w;
    int32_t* q_out;             // integer codes (2-D/3-D), aliases the output field
    float* x_out;               // 1-D: dequantized directly
    unsigned long long* st_nnz; // look-back status, payload offsets
    unsigned long long* st_x;   // look-back status, segmented x-scan carry
    Ctrl* ctrl;
};

struct DecodeLayout {
    size_t ctrl, st_nnz, st_x, sums, total;
    uint64_t sums_elems;
};
DecodeLayout decode_layout(const fz_shape& s);

cudaError_t launch_decode_init(Ctrl* ctrl, unsigned long long* st_nnz, unsigned long long* st_x,
                               uint32_t ntiles, cudaStream_t st);
cudaError_t launch_validate_outliers(const uint2* rec, uint64_t cnt, uint64_t n, Ctrl* ctrl,
                                     cudaStream_t st);
cudaError_t launch_decode_tiles(const DecodeArgs& a, cudaStream_t st);
// inclusive prefix sum along an axis of a [outer][L][W] int32 array (mod 2^32); when
// dequant_w > 0 the final values are written as fl32(fl32(q) * w) floats in place.
cudaError_t launch_scan_axis(int32_t* data, uint64_t outer, uint64_t L, uint64_t W,
                             uint32_t* sums, float dequant_w, cudaStream_t st);
cudaError_t launch_value_patch(float* out, const uint2* vrec, uint64_t cnt, uint64_t n,
                               cudaStream_t st);

}  // namespace fz
