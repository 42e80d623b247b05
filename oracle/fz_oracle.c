/*
 * fz_oracle.c -- CPU ORACLE for FZ-GPU (arXiv 2304.12557).  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load this library.  It shares no code with the CUDA path.  See fz_oracle.h for
 * the parity pins of every function.  Every step follows the paper's order: range ->
 * prequantization -> Lorenzo -> 2-byte sign-magnitude codes -> 32x32-word tiles ->
 * bitshuffle -> 16-byte block flags -> exclusive prefix sum -> compaction,
 * and the decoder inverts each step.
 *
 * Build: gcc -std=c99 -O2 -ffp-contract=off -fno-fast-math -fPIC -shared
 */
#include "fz_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------ */
/* Container layout (the paper defines no format).                  */
/* ------------------------------------------------------------------------------------ */
#define HDR_BYTES 128u
#define TILE_CODES 2048u   /* 32x32 words x 2 codes per word */
#define TILE_WORDS 1024u
#define TILE_BLOCKS 256u   /* 16-byte blocks per tile, "ByteFlagArr[256]" */

static void put_u16(uint8_t* b, uint16_t v) { memcpy(b, &v, 2); }
static void put_u32(uint8_t* b, uint32_t v) { memcpy(b, &v, 4); }
static void put_u64(uint8_t* b, uint64_t v) { memcpy(b, &v, 8); }
static void put_f32(uint8_t* b, float v) { memcpy(b, &v, 4); }
static void put_f64(uint8_t* b, double v) { memcpy(b, &v, 8); }
static uint16_t get_u16(const uint8_t* b) { uint16_t v; memcpy(&v, b, 2); return v; }
static uint32_t get_u32(const uint8_t* b) { uint32_t v; memcpy(&v, b, 4); return v; }
static uint64_t get_u64(const uint8_t* b) { uint64_t v; memcpy(&v, b, 8); return v; }
static float get_f32(const uint8_t* b) { float v; memcpy(&v, b, 4); return v; }

/* dims slowest first -> (nz, ny, nx) */
static void dims3(int ndim, const uint64_t* dims, uint64_t* nz, uint64_t* ny, uint64_t* nx)
{
    *nz = 1; *ny = 1; *nx = 1;
    if (ndim == 1) { *nx = dims[0]; }
    else if (ndim == 2) { *ny = dims[0]; *nx = dims[1]; }
    else { *nz = dims[0]; *ny = dims[1]; *nx = dims[2]; }
}

static int check_shape(int ndim, const uint64_t* dims, uint64_t* n_out)
{
    uint64_t n = 1;
    int k;
    if (ndim < 1 || ndim > 3 || dims == NULL) return FZO_ERR_ARG;
    for (k = 0; k < ndim; ++k) {
        if (dims[k] == 0) return FZO_ERR_ARG;
        if (dims[k] > 0xFFFFFFFFull) return FZO_ERR_ARG;
        n *= dims[k];
        if (n > 0xFFFFFFFFull) return FZO_ERR_ARG; /* indices are u32 (reading R16) */
    }
    *n_out = n;
    return FZO_OK;
}

/* ------------------------------------------------------------------------------------ */
/* C0  Range ("relative to the value range of the data field").                    */
/* -0.0 is counted as +0.0 (reading R18) so that min/max are unique bit patterns.        */
/* ------------------------------------------------------------------------------------ */
int fzo_range(const float* d, uint64_t n, float* mn, float* mx, int64_t* first_bad)
{
    uint64_t i;
    float lo = 0.0f, hi = 0.0f;
    int have = 0;
    *first_bad = -1;
    for (i = 0; i < n; ++i) {
        float v = d[i];
        if (!isfinite(v)) { *first_bad = (int64_t)i; return FZO_ERR_NONFINITE; }
        if (v == 0.0f) v = 0.0f; /* canonical zero */
        if (!have) { lo = v; hi = v; have = 1; }
        else {
            if (v < lo) lo = v;
            if (v > hi) hi = v;
        }
    }
    *mn = lo;
    *mx = hi;
    return FZO_OK;
}

/* ------------------------------------------------------------------------------------ */
/* f3 log transform, reading R25: natural log and exp as fixed binary64 operation  */
/* sequences (no libm, no FMA contraction), so the transform is a defined function.       */
/* ------------------------------------------------------------------------------------ */
/* ln 2 split (Cody-Waite): LN2_HI has 32 trailing zero bits, so k * LN2_HI is exact */
#define FZO_LN2_HI 6.93147180369123816490e-01
#define FZO_LN2_LO 1.90821492927058770002e-10
#define FZO_INV_LN2 1.4426950408889634074
#define FZO_SQRT_HALF 0.70710678118654752440

/* log v = e ln2 + 2 atanh(s), v = m 2^e, m in [sqrt(1/2), sqrt(2)), s = (m - 1) / (m + 1):
 * 2 atanh(s) = 2 s (1 + s^2/3 + s^4/5 + ... + s^22/23), |s| <= 0.1716 (truncation < 1e-20);
 * the polynomial in z = s^2 by Horner steps p = fma(p, z, 1/(2k+1)). */
double fzo_log64(double v)
{
    int e;
    double m = frexp(v, &e), s, z, p;
    if (m < FZO_SQRT_HALF) { m = m * 2.0; e = e - 1; }
    s = (m - 1.0) / (m + 1.0);
    z = s * s;
    /* Horner with fused multiply-adds, coefficients 1/(2k+1) rounded once (constant folding) */
    p = 1.0 / 23.0;
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
    return (double)e * FZO_LN2_HI + ((double)e * FZO_LN2_LO + 2.0 * s * p);
}

/* exp t = 2^k e^r, k = rint(t / ln2), r = (t - k LN2_HI) - k LN2_LO (|r| <= 0.35):
 * e^r = sum_{n<=17} r^n / n! by Horner steps p = fma(p, r, 1/n!) (truncation < 1e-21). */
double fzo_exp64(double t)
{
    double k = nearbyint(t * FZO_INV_LN2), r = (t - k * FZO_LN2_HI) - k * FZO_LN2_LO;
    /* Horner with fused multiply-adds, coefficients 1/n! rounded once (constant folding) */
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

float fzo_log32(float x) { return (float)fzo_log64((double)x); }

float fzo_exp32(float y)
{
    double v = fzo_exp64((double)y);
    if (v > (double)FLT_MAX) v = (double)FLT_MAX;
    return (float)v;
}

double fzo_pwrel_eb(double eps, float M)
{
    const double k = ldexp(1.0, -24) + ldexp(1.0, -45);
    double U = 0.0, up, lo, b;
    int e;
    if (!(eps > 0.0) || !(eps < 1.0)) return 0.0;
    if (M > 0.0f) {
        (void)frexp((double)M, &e);
        U = ldexp(1.0, e - 23);
    }
    up = fzo_log64((1.0 + eps) / (1.0 + k));
    lo = -fzo_log64((1.0 - eps) / (1.0 - k));
    b = up < lo ? up : lo;
    return b - U / 4.0 - ldexp(1.0, -40);
}

/* Largest float <= t (round toward -inf to binary32). */
static float rd32(double t)
{
    float f = (float)t;
    if ((double)f > t) f = nextafterf(f, -INFINITY);
    return f;
}

/* ------------------------------------------------------------------------------------ */
/* Appendix A of SURVEY.md (reading R2 in DESIGN.md): the paper's bin width 2*eb */
/* reduced by U = one ulp of the binade above max|d| so that the fp32 reconstruction     */
/* fl32(q*w) still satisfies |xhat - d| <= eb_abs.                                       */
/* ------------------------------------------------------------------------------------ */
int fzo_derive_params(float mn, float mx, int mode, double eb, fzo_params* p)
{
    double eb_abs, U, t;
    float M, w;
    int fallback = 0;

    if (p == NULL) return FZO_ERR_ARG;
    if (!(eb > 0.0) || !isfinite(eb)) return FZO_ERR_ARG;
    if (mode != FZO_ABS && mode != FZO_REL && mode != FZO_PWREL) return FZO_ERR_ARG;
    if (mode == FZO_PWREL && !(eb < 1.0)) return FZO_ERR_ARG;

    M = fabsf(mn);
    if (fabsf(mx) > M) M = fabsf(mx);
    /* REL bound = eb * value range; a constant field keeps eb (reading R4).
     * P:314 (f3): the log field's ABS bound from the point-wise relative bound (R25). */
    if (mode == FZO_REL) {
        if (mx == mn) eb_abs = eb;
        else eb_abs = eb * ((double)mx - (double)mn);
    } else if (mode == FZO_PWREL) {
        eb_abs = fzo_pwrel_eb(eb, M);
    } else {
        eb_abs = eb;
    }
    if (!(eb_abs > 0.0) || !isfinite(eb_abs)) return FZO_ERR_EB_TOO_SMALL;

    U = 0.0;
    if (M > 0.0f) {
        int e;
        (void)frexp((double)M, &e);   /* M = m * 2^e, m in [1/2, 1) */
        U = ldexp(1.0, e - 23);       /* ulp of the binade above M  */
    }
    t = 2.0 * eb_abs - U;
    w = rd32(t);
    /* margin mode iff every |d|/w < 2^21 - 1, so |q| < 2^21 for every element */
    if (!(w > 0.0f && (double)M * (1.0 / (double)w) < 2097151.0)) {
        fallback = 1;
        w = rd32(2.0 * eb_abs);
    }
    if (!(w >= FLT_MIN)) return FZO_ERR_EB_TOO_SMALL;  /* reading R17 */

    p->eb_input = eb;
    p->eb_abs = eb_abs;
    p->w = w;
    p->r = (float)(1.0 / (double)w);
    p->eb32 = rd32(eb_abs);
    p->mn = mn;
    p->mx = mx;
    p->mode = mode;
    p->fallback = fallback;
    return FZO_OK;
}

/* ------------------------------------------------------------------------------------ */
/* C1  Prequantization:  q = round(d / (2 eb)),                              */
/*     |round(d/(2eb)) * 2eb - d| <= eb.                                                 */
/* Written as the definition: q is the integer nearest to d/w, ties to even (reading R1), */
/* computed exactly in binary64; the reconstruction is the fp32 product fl32(fl32(q)*w)   */
/* (reading R21) and the inequality is checked exactly in binary64.                      */
/* ------------------------------------------------------------------------------------ */
int fzo_prequantize_one(float d, const fzo_params* p, int32_t* q)
{
    const double w = (double)p->w;
    const double ratio = (double)d / w;
    double q0, R, h;
    float xh;

    if (fabs(ratio) >= 4194304.0) {        /* |d/w| >= 2^22: nearest |q| >= 2^21 */
        *q = 0;
        return 1;
    }
    q0 = nearbyint(ratio);                 /* default rounding mode: nearest-even */
    R = (double)d - q0 * w;                /* exact: q0 < 2^22 and w has 24 bits */
    h = 0.5 * w;
    if (R > h) q0 += 1.0;
    else if (R < -h) q0 -= 1.0;
    else if (fabs(R) == h && fmod(q0, 2.0) != 0.0) q0 += (R > 0.0) ? 1.0 : -1.0;

    if (fabs(q0) >= 2097152.0) {           /* |q| >= 2^21: value outlier, q := 0 */
        *q = 0;
        return 1;
    }
    *q = (int32_t)q0;
    xh = (float)(*q) * p->w;               /* fl32(fl32(q) * w) */
    if (fabs((double)xh - (double)d) > p->eb_abs) return 1;  /* P:133 violated */
    return 0;
}

/* ------------------------------------------------------------------------------------ */
/* C2  Lorenzo predictor on the prequantized integers:          */
/*     delta(z,y,x) = sum_{a,b,c in {0,1}} (-1)^(a+b+c) q(z-a, y-b, x-c),                */
/*     neighbours outside the field are 0 (field-global boundary, reading R5),           */
/*     arithmetic modulo 2^32 (reading R6).                                              */
/* ------------------------------------------------------------------------------------ */
/* f1 ("chunked data blocks can be compressed independently"):  */
/* the chunk-local variant treats a neighbour in another chunk like one outside the     */
/* field.  A chunk is cz planes x cy rows x the whole row of a 3-D field; cz = cy = 0    */
/* means no chunking (the paper's field-global predictor, reading R5).                  */
static int no_nb(uint64_t i, uint64_t c)
{
    return i == 0 || (c != 0 && i % c == 0);
}

static void lorenzo_cc(const int32_t* q, int ndim, const uint64_t* dims, uint64_t cz, uint64_t cy,
                       int32_t* delta)
{
    uint64_t nz, ny, nx, z, y, x;
    dims3(ndim, dims, &nz, &ny, &nx);
    for (z = 0; z < nz; ++z)
        for (y = 0; y < ny; ++y)
            for (x = 0; x < nx; ++x) {
                int64_t s = 0;
                int a, b, c;
                for (a = 0; a <= 1; ++a)
                    for (b = 0; b <= 1; ++b)
                        for (c = 0; c <= 1; ++c) {
                            int sign = ((a + b + c) & 1) ? -1 : 1;
                            if ((a && no_nb(z, cz)) || (b && no_nb(y, cy)) || (c && x == 0)) continue;
                            s += sign * (int64_t)q[((z - a) * ny + (y - b)) * nx + (x - c)];
                        }
                delta[(z * ny + y) * nx + x] = (int32_t)(uint32_t)(uint64_t)s;
            }
}

void fzo_lorenzo(const int32_t* q, int ndim, const uint64_t* dims, int32_t* delta)
{
    lorenzo_cc(q, ndim, dims, 0, 0, delta);
}

void fzo_lorenzo_chunked(const int32_t* q, const uint64_t* dims, uint64_t cz, uint64_t cy, int32_t* delta)
{
    lorenzo_cc(q, 3, dims, cz, cy, delta);
}

/* ------------------------------------------------------------------------------------ */
/* C3  Two-byte sign-magnitude code: "use two bytes", negative numbers are   */
/* "the corresponding positive number with the most significant bit set as one".         */
/* |delta| > 32767 becomes code 0 plus a delta outlier (reading R7).                     */
/* ------------------------------------------------------------------------------------ */
int fzo_pack(int32_t delta, uint16_t* code)
{
    int64_t v = delta;
    int64_t m = v < 0 ? -v : v;
    if (m > 32767) { *code = 0; return 1; }
    *code = (uint16_t)(v < 0 ? (0x8000 | (uint16_t)m) : (uint16_t)m);
    return 0;
}

int32_t fzo_unpack(uint16_t code)
{
    int32_t m = code & 0x7FFF;
    return (code & 0x8000) ? -m : m;   /* 0x8000 decodes to 0 (reading R8) */
}

/* ------------------------------------------------------------------------------------ */
/* C5  Bitshuffle (listing P:264-270, reading R11):                           */
/*     O[r][c] bit j = A[c][j] bit r, naive bit-by-bit gather.                           */
/* ------------------------------------------------------------------------------------ */
void fzo_shuffle_tile(const uint32_t* A, uint32_t* O)
{
    int r, c, j;
    for (r = 0; r < 32; ++r)
        for (c = 0; c < 32; ++c) {
            uint32_t v = 0;
            for (j = 0; j < 32; ++j) v |= ((A[32 * c + j] >> r) & 1u) << j;
            O[32 * r + c] = v;
        }
}

void fzo_unshuffle_tile(const uint32_t* O, uint32_t* A)
{
    int r, c, j;
    for (c = 0; c < 32; ++c)
        for (j = 0; j < 32; ++j) {
            uint32_t v = 0;
            for (r = 0; r < 32; ++r) v |= ((O[32 * r + c] >> j) & 1u) << r;
            A[32 * c + j] = v;
        }
}

/* ------------------------------------------------------------------------------------ */
/* C6  Bit-flag array ("bit-flag array", listing P:272-278, R12-R13):   */
/*     block b = words 4b..4b+3 of the row-major shuffled tile; flag word b/32, bit b%32. */
/* ------------------------------------------------------------------------------------ */
int fzo_flags_tile(const uint32_t* O, uint32_t* F)
{
    int b, k, nnz = 0;
    for (k = 0; k < 8; ++k) F[k] = 0;
    for (b = 0; b < (int)TILE_BLOCKS; ++b) {
        int nonzero = (O[4 * b] | O[4 * b + 1] | O[4 * b + 2] | O[4 * b + 3]) != 0;
        if (nonzero) { F[b / 32] |= 1u << (b % 32); ++nnz; }
    }
    return nnz;
}

/* ------------------------------------------------------------------------------------ */
/* Field-level quantization stage (C1 -> C2 -> C3).                                      */
/* ------------------------------------------------------------------------------------ */
static int quantize_all(const float* d, int ndim, const uint64_t* dims, const fzo_params* p,
                        uint64_t cz, uint64_t cy,
                        uint64_t n, uint16_t* codes, uint8_t* dflag, int32_t* dval,
                        uint8_t* vflag)
{
    int32_t* q = (int32_t*)calloc(n, sizeof(int32_t));
    uint64_t i;
    if (q == NULL) return FZO_ERR_ARG;
    for (i = 0; i < n; ++i) vflag[i] = (uint8_t)fzo_prequantize_one(d[i], p, &q[i]);
    lorenzo_cc(q, ndim, dims, cz, cy, dval);
    free(q);
    for (i = 0; i < n; ++i) dflag[i] = (uint8_t)fzo_pack(dval[i], &codes[i]);
    return FZO_OK;
}

int fzo_quantize_field(const float* d, int ndim, const uint64_t* dims, const fzo_params* p,
                       uint16_t* codes,
                       uint32_t* didx, int32_t* dval_out, uint64_t dcap, uint64_t* nd,
                       uint32_t* vidx, uint32_t* vbits, uint64_t vcap, uint64_t* nv)
{
    uint64_t n, i, kd = 0, kv = 0;
    uint8_t *dflag, *vflag;
    int32_t* dval;
    int st = check_shape(ndim, dims, &n);
    if (st != FZO_OK) return st;
    dflag = (uint8_t*)malloc(n);
    vflag = (uint8_t*)malloc(n);
    dval = (int32_t*)malloc(n * sizeof(int32_t));
    if (!dflag || !vflag || !dval) { free(dflag); free(vflag); free(dval); return FZO_ERR_ARG; }
    quantize_all(d, ndim, dims, p, 0, 0, n, codes, dflag, dval, vflag);
    for (i = 0; i < n; ++i) {
        if (dflag[i]) {
            if (kd < dcap) { didx[kd] = (uint32_t)i; dval_out[kd] = dval[i]; }
            ++kd;
        }
        if (vflag[i]) {
            uint32_t bits;
            memcpy(&bits, &d[i], 4);
            if (kv < vcap) { vidx[kv] = (uint32_t)i; vbits[kv] = bits; }
            ++kv;
        }
    }
    *nd = kd;
    *nv = kv;
    free(dflag); free(vflag); free(dval);
    return (kd > dcap || kv > vcap) ? FZO_ERR_CAPACITY : FZO_OK;
}

uint64_t fzo_compress_bound(int ndim, const uint64_t* dims)
{
    uint64_t n, T;
    if (check_shape(ndim, dims, &n) != FZO_OK) return 0;
    T = (n + TILE_CODES - 1) / TILE_CODES;
    return HDR_BYTES + 32u * T + 4096u * T + 16u * n;
}

/* ------------------------------------------------------------------------------------ */
/* Compressor: C4 tiles, C5 shuffle, C6 flags, C7 exclusive prefix sum over the blocks   */
/* (a block is written iff its offset differs from the previous one),  */
/* C8 compaction, C9 container.                                                          */
/* ------------------------------------------------------------------------------------ */
static int compress_cc(const float* d, int ndim, const uint64_t* dims, const fzo_params* p,
                       uint64_t cz, uint64_t cy, uint8_t* out, uint64_t cap, uint64_t* size)
{
    uint64_t n, T, t, i, k, nnz = 0, nd = 0, nv = 0, total, pos;
    uint16_t* codes;
    uint8_t *dflag, *vflag;
    int32_t* dval;
    uint32_t* flags;          /* 8 words per tile           */
    uint32_t* shuffled;       /* 1024 words per tile        */
    uint64_t* presum;         /* exclusive scan over blocks */
    uint32_t A[TILE_WORDS];
    int st = check_shape(ndim, dims, &n);
    if (st != FZO_OK) return st;
    if (size == NULL || p == NULL) return FZO_ERR_ARG;

    T = (n + TILE_CODES - 1) / TILE_CODES;
    codes = (uint16_t*)calloc(T * TILE_CODES, sizeof(uint16_t));   /* zero-padded tail */
    dflag = (uint8_t*)malloc(n);
    vflag = (uint8_t*)malloc(n);
    dval = (int32_t*)malloc(n * sizeof(int32_t));
    flags = (uint32_t*)calloc(T * 8, sizeof(uint32_t));
    shuffled = (uint32_t*)malloc(T * TILE_WORDS * sizeof(uint32_t));
    presum = (uint64_t*)malloc((T * TILE_BLOCKS + 1) * sizeof(uint64_t));
    if (!codes || !dflag || !vflag || !dval || !flags || !shuffled || !presum) {
        st = FZO_ERR_ARG;
        goto done;
    }

    /* C1-C3 */
    quantize_all(d, ndim, dims, p, cz, cy, n, codes, dflag, dval, vflag);
    for (i = 0; i < n; ++i) { nd += dflag[i]; nv += vflag[i]; }

    /* C4 + C5 + C6 per tile: word k = code[2k] | code[2k+1] << 16 (reading R9) */
    for (t = 0; t < T; ++t) {
        const uint16_t* tc = codes + t * TILE_CODES;
        for (k = 0; k < TILE_WORDS; ++k)
            A[k] = (uint32_t)tc[2 * k] | ((uint32_t)tc[2 * k + 1] << 16);
        fzo_shuffle_tile(A, shuffled + t * TILE_WORDS);
        fzo_flags_tile(shuffled + t * TILE_WORDS, flags + 8 * t);
    }

    /* C7: exclusive prefix sum of the per-block byte flags over the whole field */
    presum[0] = 0;
    for (k = 0; k < T * TILE_BLOCKS; ++k) {
        uint64_t tt = k / TILE_BLOCKS, b = k % TILE_BLOCKS;
        uint64_t flag = (flags[8 * tt + b / 32] >> (b % 32)) & 1u;
        presum[k + 1] = presum[k] + flag;
    }
    nnz = presum[T * TILE_BLOCKS];

    total = HDR_BYTES + 32u * T + 16u * nnz + 8u * nd + 8u * nv;
    *size = total;
    if (total > cap || out == NULL) { st = FZO_ERR_CAPACITY; goto done; }

    /* C9 header */
    memset(out, 0, HDR_BYTES);
    memcpy(out, "FZB2", 4);
    put_u16(out + 4, 1);
    put_u16(out + 6, (uint16_t)((p->mode == FZO_REL ? 1u : 0u) | (p->fallback ? 2u : 0u) |
                                (p->mode == FZO_PWREL ? 8u : 0u) |
                                (cz ? 4u : 0u)));
    out[8] = (uint8_t)ndim;
    if (cz) {                 /* f1: chunk depth and height (bytes 10-13, zero otherwise) */
        put_u16(out + 10, (uint16_t)cz);
        put_u16(out + 12, (uint16_t)cy);
    }
    for (k = 0; k < 3; ++k) put_u64(out + 16 + 8 * k, k < (uint64_t)ndim ? dims[k] : 1u);
    put_u64(out + 40, n);
    put_f64(out + 48, p->eb_input);
    put_f64(out + 56, p->eb_abs);
    put_f32(out + 64, p->w);
    put_f32(out + 68, p->r);
    put_f32(out + 72, p->mn);
    put_f32(out + 76, p->mx);
    put_u64(out + 80, T);
    put_u64(out + 88, nnz);
    put_u64(out + 96, nd);
    put_u64(out + 104, nv);
    put_u64(out + 112, total);

    /* flags section */
    for (k = 0; k < 8 * T; ++k) put_u32(out + HDR_BYTES + 4 * k, flags[k]);

    /* C8 compaction: block k is written iff presum[k+1] != presum[k] (P:284 footnote) */
    pos = HDR_BYTES + 32u * T;
    for (k = 0; k < T * TILE_BLOCKS; ++k) {
        if (presum[k + 1] != presum[k]) {
            uint64_t tt = k / TILE_BLOCKS, b = k % TILE_BLOCKS, m;
            uint8_t* dst = out + pos + 16u * presum[k];
            for (m = 0; m < 4; ++m) put_u32(dst + 4 * m, shuffled[tt * TILE_WORDS + 4 * b + m]);
        }
    }

    /* outlier sections, ascending index (reading R7) */
    pos = HDR_BYTES + 32u * T + 16u * nnz;
    for (i = 0; i < n; ++i)
        if (dflag[i]) {
            put_u32(out + pos, (uint32_t)i);
            put_u32(out + pos + 4, (uint32_t)dval[i]);
            pos += 8;
        }
    for (i = 0; i < n; ++i)
        if (vflag[i]) {
            uint32_t bits;
            memcpy(&bits, &d[i], 4);
            put_u32(out + pos, (uint32_t)i);
            put_u32(out + pos + 4, bits);
            pos += 8;
        }
    st = FZO_OK;
done:
    free(codes); free(dflag); free(vflag); free(dval); free(flags); free(shuffled); free(presum);
    return st;
}

int fzo_compress_with_params(const float* d, int ndim, const uint64_t* dims,
                             const fzo_params* p, uint8_t* out, uint64_t cap,
                             uint64_t* size)
{
    return compress_cc(d, ndim, dims, p, 0, 0, out, cap, size);
}

/* f1: chunk-local compressor (3-D only; 1 <= cz, cy <= 65535). */
int fzo_compress_chunked(const float* d, const uint64_t* dims, int mode, double eb, uint64_t cz,
                         uint64_t cy, uint8_t* out, uint64_t cap, uint64_t* size)
{
    uint64_t n;
    float mn, mx;
    int64_t bad;
    fzo_params p;
    int st = check_shape(3, dims, &n);
    if (st != FZO_OK) return st;
    if (d == NULL || size == NULL || cz < 1 || cy < 1 || cz > 65535 || cy > 65535) return FZO_ERR_ARG;
    st = fzo_range(d, n, &mn, &mx, &bad);
    if (st != FZO_OK) return st;
    st = fzo_derive_params(mn, mx, mode, eb, &p);
    if (st != FZO_OK) return st;
    return compress_cc(d, 3, dims, &p, cz, cy, out, cap, size);
}

static int compress_pwrel(const float* d, int ndim, const uint64_t* dims, uint64_t n, double eps,
                          uint8_t* out, uint64_t cap, uint64_t* size)
{
    /* f3: y = log(x) elementwise, then the ABS pipeline on y with the bound that
     * guarantees |x^ - x| <= eps |x| after x^ = exp(y^) (reading R25) */
    uint64_t i;
    float mn, mx;
    int64_t bad;
    fzo_params p;
    int st;
    float* y = (float*)malloc(n * sizeof(float));
    if (y == NULL) return FZO_ERR_ARG;
    for (i = 0; i < n; ++i) {
        if (!isfinite(d[i])) { free(y); return FZO_ERR_NONFINITE; }
        if (!(d[i] >= FLT_MIN)) { free(y); return FZO_ERR_ARG; }   /* domain: normal x > 0 */
        y[i] = fzo_log32(d[i]);
    }
    st = fzo_range(y, n, &mn, &mx, &bad);
    if (st == FZO_OK) st = fzo_derive_params(mn, mx, FZO_PWREL, eps, &p);
    if (st == FZO_OK) st = fzo_compress_with_params(y, ndim, dims, &p, out, cap, size);
    free(y);
    return st;
}

int fzo_compress(const float* d, int ndim, const uint64_t* dims, int mode, double eb,
                 uint8_t* out, uint64_t cap, uint64_t* size)
{
    uint64_t n;
    float mn, mx;
    int64_t bad;
    fzo_params p;
    int st = check_shape(ndim, dims, &n);
    if (st != FZO_OK) return st;
    if (d == NULL || size == NULL) return FZO_ERR_ARG;
    if (mode == FZO_PWREL) {
        if (!(eb > 0.0) || !(eb < 1.0)) return FZO_ERR_ARG;
        return compress_pwrel(d, ndim, dims, n, eb, out, cap, size);
    }
    st = fzo_range(d, n, &mn, &mx, &bad);
    if (st != FZO_OK) return st;
    st = fzo_derive_params(mn, mx, mode, eb, &p);
    if (st != FZO_OK) return st;
    return fzo_compress_with_params(d, ndim, dims, &p, out, cap, size);
}

/* ------------------------------------------------------------------------------------ */
/* Decoder ("highly symmetrical"): parse, scatter blocks (D1-D2), naive un-gather   */
/* (D3), unpack + delta patch (D4), sequential SZ-style Lorenzo recurrence (D5),          */
/* dequantize + value patch (D6).                                                         */
/* ------------------------------------------------------------------------------------ */
typedef struct {
    int ndim;
    uint64_t cz, cy;          /* f1 chunk depth / height, 0 = field-global Lorenzo */
    int logt;                 /* f3: the stream holds log(x) (flag bit 3)          */
    uint64_t dims[3], n, T, nnz, nd, nv, total;
    float w;
    const uint8_t *flags, *payload, *dsec, *vsec;
} parsed_t;

static int popc32(uint32_t v)
{
    int c = 0;
    while (v) { c += (int)(v & 1u); v >>= 1; }
    return c;
}

static int parse(const uint8_t* in, uint64_t size, parsed_t* h)
{
    uint64_t k, n = 1, cnt = 0, prev;
    if (in == NULL || size < HDR_BYTES) return FZO_ERR_CORRUPT;
    if (memcmp(in, "FZB2", 4) != 0 || get_u16(in + 4) != 1) return FZO_ERR_CORRUPT;
    h->ndim = in[8];
    if (h->ndim < 1 || h->ndim > 3) return FZO_ERR_CORRUPT;
    h->cz = h->cy = 0;
    h->logt = (get_u16(in + 6) & 8u) ? 1 : 0;
    if (get_u16(in + 6) & 4u) {
        h->cz = get_u16(in + 10);
        h->cy = get_u16(in + 12);
        if (h->ndim != 3 || h->cz == 0 || h->cy == 0) return FZO_ERR_CORRUPT;
    }
    for (k = 0; k < 3; ++k) {
        h->dims[k] = get_u64(in + 16 + 8 * k);
        if (h->dims[k] == 0 || h->dims[k] > 0xFFFFFFFFull) return FZO_ERR_CORRUPT;
        if (k >= (uint64_t)h->ndim && h->dims[k] != 1) return FZO_ERR_CORRUPT;
        n *= h->dims[k];
        if (n > 0xFFFFFFFFull) return FZO_ERR_CORRUPT;
    }
    h->n = get_u64(in + 40);
    if (h->n != n) return FZO_ERR_CORRUPT;
    h->w = get_f32(in + 64);
    if (!(h->w > 0.0f) || !isfinite(h->w)) return FZO_ERR_CORRUPT;
    h->T = get_u64(in + 80);
    h->nnz = get_u64(in + 88);
    h->nd = get_u64(in + 96);
    h->nv = get_u64(in + 104);
    h->total = get_u64(in + 112);
    if (h->T != (n + TILE_CODES - 1) / TILE_CODES) return FZO_ERR_CORRUPT;
    if (h->nnz > h->T * TILE_BLOCKS || h->nd > n || h->nv > n) return FZO_ERR_CORRUPT;
    if (h->total != HDR_BYTES + 32u * h->T + 16u * h->nnz + 8u * h->nd + 8u * h->nv)
        return FZO_ERR_CORRUPT;
    if (size < h->total) return FZO_ERR_CORRUPT;
    h->flags = in + HDR_BYTES;
    h->payload = h->flags + 32u * h->T;
    h->dsec = h->payload + 16u * h->nnz;
    h->vsec = h->dsec + 8u * h->nd;
    for (k = 0; k < 8 * h->T; ++k) cnt += (uint64_t)popc32(get_u32(h->flags + 4 * k));
    if (cnt != h->nnz) return FZO_ERR_CORRUPT;
    /* outlier indices strictly increasing and < n (SURVEY §5 corrupt-stream checks) */
    prev = 0;
    for (k = 0; k < h->nd; ++k) {
        uint64_t idx = get_u32(h->dsec + 8 * k);
        if (idx >= n || (k > 0 && idx <= prev)) return FZO_ERR_CORRUPT;
        prev = idx;
    }
    prev = 0;
    for (k = 0; k < h->nv; ++k) {
        uint64_t idx = get_u32(h->vsec + 8 * k);
        if (idx >= n || (k > 0 && idx <= prev)) return FZO_ERR_CORRUPT;
        prev = idx;
    }
    return FZO_OK;
}

/* D1-D5: integer codes q */
static int decode_q(const parsed_t* h, int32_t* q)
{
    uint64_t t, k, used = 0, nz, ny, nx, z, y, x;
    uint32_t O[TILE_WORDS], A[TILE_WORDS];
    int32_t* delta = (int32_t*)malloc(h->T * TILE_CODES * sizeof(int32_t));
    if (delta == NULL) return FZO_ERR_ARG;
    for (t = 0; t < h->T; ++t) {
        int b;
        for (b = 0; b < (int)TILE_BLOCKS; ++b) {          /* D2 scatter */
            uint32_t f = get_u32(h->flags + 32u * t + 4u * (uint64_t)(b / 32));
            int m;
            if ((f >> (b % 32)) & 1u) {
                for (m = 0; m < 4; ++m) O[4 * b + m] = get_u32(h->payload + 16u * used + 4u * (uint64_t)m);
                ++used;
            } else {
                for (m = 0; m < 4; ++m) O[4 * b + m] = 0;
            }
        }
        fzo_unshuffle_tile(O, A);                          /* D3 */
        for (k = 0; k < TILE_WORDS; ++k) {                 /* D4 unpack */
            delta[t * TILE_CODES + 2 * k] = fzo_unpack((uint16_t)(A[k] & 0xFFFFu));
            delta[t * TILE_CODES + 2 * k + 1] = fzo_unpack((uint16_t)(A[k] >> 16));
        }
    }
    for (k = 0; k < h->nd; ++k)                            /* D4 delta patch */
        delta[get_u32(h->dsec + 8 * k)] = (int32_t)get_u32(h->dsec + 8 * k + 4);

    /* D5: sequential recurrence q = delta + pred, pred from reconstructed neighbours */
    dims3(h->ndim, h->dims, &nz, &ny, &nx);
    for (z = 0; z < nz; ++z)
        for (y = 0; y < ny; ++y)
            for (x = 0; x < nx; ++x) {
                uint32_t s = (uint32_t)delta[(z * ny + y) * nx + x];
                int a, b, c;
                for (a = 0; a <= 1; ++a)
                    for (b = 0; b <= 1; ++b)
                        for (c = 0; c <= 1; ++c) {
                            uint32_t v;
                            if (a + b + c == 0) continue;
                            if ((a && no_nb(z, h->cz)) || (b && no_nb(y, h->cy)) || (c && x == 0)) continue;
                            v = (uint32_t)q[((z - a) * ny + (y - b)) * nx + (x - c)];
                            /* pred = -sum_{(a,b,c) != 0} (-1)^(a+b+c) q(...) */
                            if ((a + b + c) & 1) s += v; else s -= v;
                        }
                q[(z * ny + y) * nx + x] = (int32_t)s;
            }
    free(delta);
    return FZO_OK;
}

int fzo_decode_q(const uint8_t* in, uint64_t size, int32_t* q, uint64_t n)
{
    parsed_t h;
    int st = parse(in, size, &h);
    if (st != FZO_OK) return st;
    if (n != h.n || q == NULL) return FZO_ERR_ARG;
    return decode_q(&h, q);
}

int fzo_decompress(const uint8_t* in, uint64_t size, float* out, uint64_t n)
{
    parsed_t h;
    uint64_t i, k;
    int32_t* q;
    int st = parse(in, size, &h);
    if (st != FZO_OK) return st;
    if (n != h.n || out == NULL) return FZO_ERR_ARG;
    q = (int32_t*)malloc(n * sizeof(int32_t));
    if (q == NULL) return FZO_ERR_ARG;
    st = decode_q(&h, q);
    if (st == FZO_OK) {
        for (i = 0; i < n; ++i) out[i] = (float)q[i] * h.w;   /* D6: fl32(fl32(q) * w) */
        for (k = 0; k < h.nv; ++k) {                          /* D6 value patch */
            uint32_t bits = get_u32(h.vsec + 8 * k + 4);
            memcpy(&out[get_u32(h.vsec + 8 * k)], &bits, 4);
        }
        if (h.logt)                                           /* f3: x^ = exp(y^) */
            for (i = 0; i < n; ++i) out[i] = fzo_exp32(out[i]);
    }
    free(q);
    return st;
}
