/*
 * fz_oracle.h -- CPU ORACLE for the FZ-GPU compression path (arXiv 2304.12557).
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  It shares no code,
 * header, table or constant generator with the CUDA path (paper_2304_12557_b200/csrc/,
 * include/fz.h); the two are written independently from the paper and from the readings
 * listed in DESIGN.md §3.
 *
 * Plain, slow, single-threaded C99.  Compiled with -O2 -ffp-contract=off -fno-fast-math
 * (SSE2 arithmetic, no x87, no FMA contraction) so that every float/double operation is
 * one IEEE-754 round-to-nearest-even operation as written.
 *
 * Citation key: P:n = PAPER.md line n, S:n = SPEC.md line n, SV = SURVEY.md section.
 *
 * Parity pins (tests/test_oracle_*.py, all "-m 'not gpu'"):
 *   derive_params  : Appendix-A closed forms (frexp / nextafter by hand), worked example W1.
 *   prequantize    : exact nearest integer from Python fractions.Fraction (brute force),
 *                    the P:133 inequality on every element, sign symmetry.
 *   lorenzo        : numpy.diff-with-zero-prepend along each axis (closed form).
 *   pack/unpack    : exhaustive over [-32767, 32767].
 *   shuffle_tile   : numpy bit-tensor transpose (independent construction).
 *   flags_tile     : numpy any() over 16-byte blocks of the numpy-shuffled tile.
 *   compress       : size law, all-zero field = 128 + 32T, worked example W1 byte stream
 *                    (tests/golden/w1.hex), P:373 cap.
 *   decompress     : |x - xhat| <= eb_abs on every element, code round trip,
 *                    numpy cumsum inverse of the stencil.
 * No function is "parity unpinned".
 */
#ifndef FZ_ORACLE_H
#define FZ_ORACLE_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status values.  Numerically equal to fz.h's fz_status by convention;
 * declared independently here. */
enum {
    FZO_OK = 0,
    FZO_ERR_ARG = 1,
    FZO_ERR_NONFINITE = 2,
    FZO_ERR_EB_TOO_SMALL = 3,
    FZO_ERR_CAPACITY = 4,
    FZO_ERR_CORRUPT = 5
};

enum { FZO_ABS = 0, FZO_REL = 1, FZO_PWREL = 2 };

typedef struct {
    double eb_input;  /* eb as given by the user                                  */
    double eb_abs;    /* absolute bound: eb (ABS) or eb*(max-min) (REL)     */
    float  w;         /* bin width, ~2*eb_abs less a ulp margin (SV App. A)        */
    float  r;         /* (float)(1/(double)w), recorded in the header              */
    float  eb32;      /* largest float <= eb_abs                                   */
    float  mn, mx;    /* field range (canonical: -0.0 counted as +0.0)            */
    int    mode;      /* FZO_ABS / FZO_REL / FZO_PWREL (f3: log transform)         */
    int    fallback;  /* 1 when the margin ("fast") mode is infeasible             */
} fzo_params;

/* C0 range: min, max over the field, first non-finite index (-1 if none). */
int fzo_range(const float* d, uint64_t n, float* mn, float* mx, int64_t* first_bad);

/* Appendix A parameter derivation (P:129-134 with reading R2 of DESIGN.md). */
int fzo_derive_params(float mn, float mx, int mode, double eb, fzo_params* p);

/* C1 prequantization of ONE value: returns 1 if the element is a value
 * outlier (bound check failed, or |q| >= 2^21), else 0; *q receives the integer code. */
int fzo_prequantize_one(float d, const fzo_params* p, int32_t* q);

/* C2 Lorenzo residual: delta = sum over the unit cube of (-1)^k q, zero
 * outside the field, int32 wrap-around.  dims slowest first, ndim in {1,2,3}. */
void fzo_lorenzo(const int32_t* q, int ndim, const uint64_t* dims, int32_t* delta);

/* f1 chunk-local Lorenzo: as fzo_lorenzo on a 3-D field, but a
 * neighbour in another chunk (cz planes x cy rows x the whole row) counts as 0. */
void fzo_lorenzo_chunked(const int32_t* q, const uint64_t* dims, uint64_t cz, uint64_t cy, int32_t* delta);

/* C3 sign-magnitude packing: returns 1 if |delta| > 32767 (delta outlier,
 * code 0), else 0. */
int fzo_pack(int32_t delta, uint16_t* code);
int32_t fzo_unpack(uint16_t code);

/* C5 bitshuffle of one tile by naive bit gather:
 * O[r][c] bit j = A[c][j] bit r, A[c][j] = word 32c+j. */
void fzo_shuffle_tile(const uint32_t* A, uint32_t* O);
void fzo_unshuffle_tile(const uint32_t* O, uint32_t* A);

/* C6 flags of one shuffled tile: block b = words 4b..4b+3 of O;
 * flag word b/32 bit b%32 set iff the block has a nonzero word.  Returns nnz. */
int fzo_flags_tile(const uint32_t* O, uint32_t* F);

/* Stage hook: quantize + Lorenzo + pack for the whole field (parity of codes and lists).
 * codes: n entries.  Lists are in ascending index order.  Capacities in entries. */
int fzo_quantize_field(const float* d, int ndim, const uint64_t* dims, const fzo_params* p,
                       uint16_t* codes,
                       uint32_t* didx, int32_t* dval, uint64_t dcap, uint64_t* nd,
                       uint32_t* vidx, uint32_t* vbits, uint64_t vcap, uint64_t* nv);

/* Upper bound of the container size. */
uint64_t fzo_compress_bound(int ndim, const uint64_t* dims);

/* Full compressor: header || flags || payload || delta outliers || value outliers. */
int fzo_compress(const float* d, int ndim, const uint64_t* dims, int mode, double eb,
                 uint8_t* out, uint64_t cap, uint64_t* size);

/* Same with parameters supplied (used by idempotence tests). */
int fzo_compress_with_params(const float* d, int ndim, const uint64_t* dims,
                             const fzo_params* p, uint8_t* out, uint64_t cap,
                             uint64_t* size);

/* f1 chunk-local compressor (3-D): header flag bit 2, chunk depth/height at bytes 10-13;
 * the decompressors below read both variants. */
int fzo_compress_chunked(const float* d, const uint64_t* dims, int mode, double eb, uint64_t cz,
                         uint64_t cy, uint8_t* out, uint64_t cap, uint64_t* size);

/* Full decompressor.  out: n floats, n must equal the header's element count. */
int fzo_decompress(const uint8_t* in, uint64_t size, float* out, uint64_t n);

/* f3 ("transform the original data using a logarithmic function and
 * compress the log-transformed data with the corresponding absolute error bound (computed
 * from the point-wise relative error bound)"), reading R25 in DESIGN.md.  The transform is a
 * defined function: a fixed sequence of binary64 operations rounded once to binary32, so two
 * independent implementations agree bit for bit.  Pins: tests/test_oracle_pins.py (numpy log /
 * exp within half an ulp of binary32 plus the binary64 error, special values, the P:314
 * guarantee |x^ - x| <= eps |x| on every element). */
double fzo_log64(double v);            /* v > 0, finite                                     */
double fzo_exp64(double t);            /* |t| < 700                                         */
float fzo_log32(float x);              /* x >= FLT_MIN, finite                              */
float fzo_exp32(float y);              /* fl32(min(exp64(y), FLT_MAX))                      */
/* ABS bound on the log field that guarantees the point-wise relative bound eps (reading R25):
 * min(log64((1+eps)/(1+k)), -log64((1-eps)/(1-k))) - U/4 - 2^-40, k = 2^-24 + 2^-45, U the
 * binade-above ulp of M = max|y|.  <= 0 -> FZO_ERR_EB_TOO_SMALL. */
double fzo_pwrel_eb(double eps, float M);

/* Decoder stage hook: reconstructed integer codes q (before dequantization). */
int fzo_decode_q(const uint8_t* in, uint64_t size, int32_t* q, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif
