/* ASan + UBSan driver for the C oracle (test infrastructure; SURVEY §5 "ASan/UBSan on the
 * oracle").  Runs every public oracle entry point on small synthetic fields -- smooth, noise,
 * spikes (delta outliers), offset data in fallback mode (value outliers), all-zero, ragged
 * tails, NaN / Inf, the f1 chunked and f3 log variants -- round-trips them, checks the P:133
 * bound, then feeds truncated and bit-flipped streams to the decompressor (must fail cleanly
 * or succeed, never read or write out of bounds).
 *   gcc -std=c99 -O1 -g -fsanitize=address,undefined -fno-sanitize-recover=all \
 *       -ffp-contract=off tools/oracle_asan.c oracle/fz_oracle.c -lm -o /tmp/oracle_asan
 *   /tmp/oracle_asan   (tools/oracle_asan.sh) */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../oracle/fz_oracle.h"

static uint64_t sm64(uint64_t* s)
{
    uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static double u01(uint64_t* s) { return ((sm64(s) >> 11) + 0.5) * (1.0 / 9007199254740992.0); }

static int failures = 0, cases = 0;

static void roundtrip(const char* name, const float* d, int ndim, const uint64_t* dims, int mode, double eb,
                      int expect)
{
    uint64_t n = 1;
    for (int k = 0; k < ndim; ++k) n *= dims[k];
    const uint64_t cap = fzo_compress_bound(ndim, dims);
    uint8_t* out = (uint8_t*)malloc(cap);
    float* x = (float*)malloc(sizeof(float) * (n ? n : 1));
    uint64_t size = 0;
    ++cases;
    int st = fzo_compress(d, ndim, dims, mode, eb, out, cap, &size);
    if (st != expect) {
        printf("FAIL %s: compress status %d, expected %d\n", name, st, expect);
        ++failures;
    }
    if (st == FZO_OK) {
        st = fzo_decompress(out, size, x, n);
        double ebabs;
        memcpy(&ebabs, out + 56, 8);
        double worst = 0.0;
        for (uint64_t i = 0; i < n; ++i) {
            const double e = fabs((double)x[i] - (double)d[i]);
            const double b = mode == FZO_PWREL ? eb * fabs((double)d[i]) : ebabs;
            if (e > b && e - b > worst) worst = e - b;
        }
        if (st != FZO_OK || worst > 0.0) {
            printf("FAIL %s: decompress status %d, bound exceeded by %g\n", name, st, worst);
            ++failures;
        }
        /* corrupt streams: every truncation length class and single bit flips in each section */
        uint8_t* bad = (uint8_t*)malloc(size + 1);
        const uint64_t cuts[] = {0, 1, 64, 127, 128, 129, size / 2, size - 1};
        for (int c = 0; c < 8; ++c) {
            if (cuts[c] > size) continue;
            memcpy(bad, out, cuts[c]);
            (void)fzo_decompress(bad, cuts[c], x, n);
        }
        uint64_t rs = 12345;
        for (int f = 0; f < 64 && size > 0; ++f) {
            memcpy(bad, out, size);
            const uint64_t pos = sm64(&rs) % size;
            bad[pos] ^= (uint8_t)(1u << (sm64(&rs) & 7));
            (void)fzo_decompress(bad, size, x, n);
        }
        free(bad);
    }
    free(out);
    free(x);
}

int main(void)
{
    uint64_t s = 7;
    /* 3-D smooth + noise, ragged tail */
    {
        const uint64_t dims[3] = {9, 17, 33};
        const uint64_t n = dims[0] * dims[1] * dims[2];
        float* d = (float*)malloc(4 * n);
        for (uint64_t i = 0; i < n; ++i) {
            const uint64_t z = i / (dims[1] * dims[2]), y = (i / dims[2]) % dims[1], x = i % dims[2];
            d[i] = (float)(sin(0.3 * x) * cos(0.2 * y) + 0.1 * z + 1e-3 * (u01(&s) - 0.5));
        }
        roundtrip("3d smooth REL", d, 3, dims, FZO_REL, 1e-3, FZO_OK);
        roundtrip("3d smooth ABS", d, 3, dims, FZO_ABS, 1e-4, FZO_OK);
        d[77] = 1e9f;   /* spike: delta outliers */
        roundtrip("3d spike", d, 3, dims, FZO_REL, 1e-6, FZO_OK);
        d[n - 1] = NAN;
        roundtrip("3d nan", d, 3, dims, FZO_REL, 1e-3, FZO_ERR_NONFINITE);
        d[n - 1] = INFINITY;
        roundtrip("3d inf", d, 3, dims, FZO_REL, 1e-3, FZO_ERR_NONFINITE);
        free(d);
    }
    /* 2-D noise, offset data in fallback mode (value outliers) */
    {
        const uint64_t dims[2] = {37, 61};
        const uint64_t n = dims[0] * dims[1];
        float* d = (float*)malloc(4 * n);
        for (uint64_t i = 0; i < n; ++i) d[i] = (float)(1e6 + u01(&s));
        roundtrip("2d offset REL 1e-6", d, 2, dims, FZO_REL, 1e-6, FZO_OK);
        for (uint64_t i = 0; i < n; ++i) d[i] = (float)(u01(&s) * 2.0 - 1.0);
        roundtrip("2d noise ABS", d, 2, dims, FZO_ABS, 1e-2, FZO_OK);
        free(d);
    }
    /* 1-D: all-zero tails of 1, 64, 2047, 2049 codes; constant; ramp */
    {
        const uint64_t lens[] = {1, 64, 2047, 2049, 5000};
        for (int k = 0; k < 5; ++k) {
            const uint64_t dims[1] = {lens[k]};
            float* d = (float*)calloc(lens[k], 4);
            roundtrip("1d zeros", d, 1, dims, FZO_REL, 1e-3, FZO_OK);
            for (uint64_t i = 0; i < lens[k]; ++i) d[i] = 3.5f;
            roundtrip("1d constant", d, 1, dims, FZO_ABS, 1e-3, FZO_OK);
            for (uint64_t i = 0; i < lens[k]; ++i) d[i] = (float)i * 0.25f;
            roundtrip("1d ramp", d, 1, dims, FZO_REL, 1e-4, FZO_OK);
            free(d);
        }
    }
    /* f3: log transform on a positive field; domain errors */
    {
        const uint64_t dims[1] = {3001};
        float* d = (float*)malloc(4 * dims[0]);
        for (uint64_t i = 0; i < dims[0]; ++i) d[i] = (float)(1.0 / 64 + 256.0 * u01(&s));
        roundtrip("1d pwrel", d, 1, dims, FZO_PWREL, 1e-3, FZO_OK);
        d[100] = 0.0f;
        roundtrip("1d pwrel zero", d, 1, dims, FZO_PWREL, 1e-3, FZO_ERR_ARG);
        free(d);
    }
    /* f1: chunk-local compressor */
    {
        const uint64_t dims[3] = {20, 8, 256};
        const uint64_t n = dims[0] * dims[1] * dims[2];
        float* d = (float*)malloc(4 * n);
        for (uint64_t i = 0; i < n; ++i) d[i] = (float)(sin(1e-3 * (double)i) + 1e-3 * u01(&s));
        const uint64_t cap = fzo_compress_bound(3, dims);
        uint8_t* out = (uint8_t*)malloc(cap);
        float* x = (float*)malloc(4 * n);
        uint64_t size = 0;
        ++cases;
        int st = fzo_compress_chunked(d, dims, FZO_REL, 1e-3, 16, 8, out, cap, &size);
        if (st == FZO_OK) st = fzo_decompress(out, size, x, n);
        if (st != FZO_OK) {
            printf("FAIL chunked: status %d\n", st);
            ++failures;
        }
        free(d);
        free(out);
        free(x);
    }
    printf("oracle ASan/UBSan driver: %d cases, %d failures\n", cases, failures);
    return failures != 0;
}
