// fz_rowwalk.cuh -- device helpers shared by the row-walking compressor (fz_zrow.cu) and
// the row-walking decoder (fz_dzr.cu): tensor-memory (TMEM) loads / stores of the per-thread
// z carry and the in-register 32x32 bit transpose (C5 bitshuffle and its inverse).
#pragma once

#include "fz_internal.cuh"

namespace fz {

// ---- tensor memory (TMEM) as the z-carry store: thread (warp w, lane l) owns TMEM lane
// 32 (w % 4) + l, columns [68 (w / 4), 68 (w / 4) + 64) hold q(z-1) of its 16 rows x 4.
// tcgen05.ld / st of 32x32b shape move 4 / 16 consecutive columns per thread.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(taddr));
}
// completes the loads; the +r operands keep every use of v after the wait
__device__ __forceinline__ void tmem_wait_ld(uint32_t (&v)[16])
{
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                   "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15])
                 :: "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16])
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 :: "r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                    "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
                 : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld8(uint32_t (&v)[8])
{
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7])
                 :: "memory");
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};"
                 :: "r"(taddr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void tmem_wait_st()
{
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// 32x32 bit transpose of the thread's 32 words (C5): T[r] bit j = A[j] bit r.  Stages 16 and
// 8 are byte permutes, stages 4/2/1 a shift and a bit-select per word.
__device__ __forceinline__ void transpose32_regs(uint32_t (&A)[32])
{
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const uint32_t a = A[j], b = A[j + 16];
        A[j] = __byte_perm(a, b, 0x5410u);
        A[j + 16] = __byte_perm(a, b, 0x7632u);
    }
#pragma unroll
    for (int j0 = 0; j0 < 32; j0 += 16) {
#pragma unroll
        for (int j = j0; j < j0 + 8; ++j) {
            const uint32_t a = A[j], b = A[j + 8];
            A[j] = __byte_perm(a, b, 0x6240u);
            A[j + 8] = __byte_perm(a, b, 0x7351u);
        }
    }
#pragma unroll
    for (int st = 0; st < 3; ++st) {
        const int s = 4 >> st;
        const uint32_t m = st == 0 ? 0x0F0F0F0Fu : (st == 1 ? 0x33333333u : 0x55555555u);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            if (j & s) continue;
            const uint32_t a = A[j], b = A[j + s];
            A[j] = bitsel(a, b << s, m);        // (a & m) | ((b << s) & ~m)
            A[j + s] = bitsel(a >> s, b, m);    // ((a >> s) & m) | (b & ~m)
        }
    }
}

// G(b, c, x0..x0+3) = sum over chunks c' < c of R(b, c', .) (R: the chunk column sums after
// k_dzr_prep1's exclusive scan over bands), summed at a unit start with the loads in flight
__device__ __forceinline__ uint4 dz_gsum(const int32_t* cd, uint64_t row0, uint32_t c, uint32_t nx)
{
    uint4 g = make_uint4(0, 0, 0, 0);
    for (uint32_t c0 = 0; c0 < c; c0 += 8) {
        uint4 v[8];
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j)
            v[j] = c0 + j < c ? *reinterpret_cast<const uint4*>(cd + (row0 + c0 + j) * nx) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j) { g.x += v[j].x; g.y += v[j].y; g.z += v[j].z; g.w += v[j].w; }
    }
    return g;
}

// D6 (R21): x^ = fl32(fl32(q) w) for 4 codes; f3 (R25, header flag bit 3): then exp32 (the
// decoder's exp fused into its dequantization)
template <bool LOGT>
__device__ __forceinline__ float4 dzx(uint32_t q0, uint32_t q1, uint32_t q2, uint32_t q3, float w)
{
    float4 v = make_float4(__fmul_rn(__int2float_rn((int32_t)q0), w), __fmul_rn(__int2float_rn((int32_t)q1), w),
                           __fmul_rn(__int2float_rn((int32_t)q2), w), __fmul_rn(__int2float_rn((int32_t)q3), w));
    if (LOGT) {
        v.x = exp32(v.x);
        v.y = exp32(v.y);
        v.z = exp32(v.z);
        v.w = exp32(v.w);
    }
    return v;
}

}  // namespace fz
