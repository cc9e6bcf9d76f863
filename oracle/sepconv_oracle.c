/*
 * sepconv_oracle.c -- CPU restatement of the reference's separable-convolution
 * arithmetic. TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library,
 * and only as the checker or the reported CPU baseline. The product path
 * (paper_1711_09791_b200) never links or calls it.
 *
 * Reference = sepconv_lab 0.1.0 (pure Python + numpy), cited as
 *   S/ = /root/reference/pkg/src/sepconv_lab/
 * Parity is PINNED: tests/test_oracle_golden.py checks every function here
 * against fixtures produced by the reference itself (tests/golden/make_golden.py)
 * and against the reference tests' constants (T/test_conv.py:34, :119;
 * T/test_image.py:25-26).
 *
 * Arithmetic contract (S/conv.py:1-15): every product is one IEEE float32
 * multiply, every sum one float32 add, folded left-to-right from the first
 * product. numpy executes each `*` and `+=` as a separate correctly rounded
 * ufunc, so the restatement must never contract a*b+c into an FMA. This file
 * is compiled with -ffp-contract=off (see Makefile); auto-vectorisation
 * across pixels is allowed because it keeps each pixel's operation sequence
 * intact.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------------
 * Two-pass bodies.
 * horizontal_rows_vec, S/conv.py:215-240: for y in [lo,hi), x in [r,C-r):
 *   acc = s[y, x-r] * w0; acc += s[y, x-r+m] * w_m (m = 1..W-1); dst[y,x] = acc.
 * dst outside [r, C-r) of those rows is untouched (S/conv.py:240).
 */
ORC_API void orc_horizontal_rows(const float *src, float *dst, int rows, int cols,
                                 const float *w, int width, int row_lo, int row_hi)
{
    const int r = width / 2;
    (void)rows;
    for (int y = row_lo; y < row_hi; ++y) {
        const float *s = src + (int64_t)y * cols;
        float *d = dst + (int64_t)y * cols;
        for (int x = r; x < cols - r; ++x) {
            float acc = s[x - r] * w[0];
            for (int m = 1; m < width; ++m) {
                float term = s[x - r + m] * w[m];
                acc = acc + term;
            }
            d[x] = acc;
        }
    }
}

/* vertical_rows_vec, S/conv.py:269-293: rows [lo,hi) inside [r, R-r):
 *   acc = s[y-r, x] * w0; acc += s[y-r+m, x] * w_m; dst[y, x] = acc, x in [r, C-r). */
ORC_API void orc_vertical_rows(const float *src, float *dst, int rows, int cols,
                               const float *w, int width, int row_lo, int row_hi)
{
    const int r = width / 2;
    (void)rows;
    for (int y = row_lo; y < row_hi; ++y) {
        float *d = dst + (int64_t)y * cols;
        const float *s0 = src + (int64_t)(y - r) * cols;
        for (int x = r; x < cols - r; ++x) {
            d[x] = s0[x] * w[0];
        }
        for (int m = 1; m < width; ++m) {
            const float *sm = src + (int64_t)(y - r + m) * cols;
            for (int x = r; x < cols - r; ++x) {
                float term = sm[x] * w[m];
                d[x] = d[x] + term;
            }
        }
    }
}

/* single_pass_rows_vec, S/conv.py:86-114 (and its unrolled twin :146-175, same
 * order): D(y,x) folds K[i][j]*A(y-r+i, x-r+j) row-major (i outer, j inner),
 * left to right, starting from the first product. dst ring untouched. */
ORC_API void orc_single_pass_rows(const float *src, const float *dense, float *dst,
                                  int rows, int cols, int width, int row_lo, int row_hi)
{
    const int r = width / 2;
    (void)rows;
    for (int y = row_lo; y < row_hi; ++y) {
        float *d = dst + (int64_t)y * cols;
        for (int i = 0; i < width; ++i) {
            const float *s = src + (int64_t)(y - r + i) * cols;
            for (int j = 0; j < width; ++j) {
                const float k = dense[i * width + j];
                if (i == 0 && j == 0) {
                    for (int x = r; x < cols - r; ++x) d[x] = s[x - r + j] * k;
                } else {
                    for (int x = r; x < cols - r; ++x) {
                        float term = s[x - r + j] * k;
                        d[x] = d[x] + term;
                    }
                }
            }
        }
    }
}

/* conv_two_pass, S/conv.py:392-421, identical to the convolve_image two-pass
 * branch S/executors.py:308-326 + :361-365: scratch := 0; H over [r, R-r)
 * (faithful) or [0, R) (extended); V from scratch back into `plane` on [r, R-r). */
ORC_API void orc_two_pass(float *plane, float *scratch, int rows, int cols,
                          const float *w, int width, int extended)
{
    const int r = width / 2;
    memset(scratch, 0, sizeof(float) * (size_t)rows * (size_t)cols);
    if (extended)
        orc_horizontal_rows(plane, scratch, rows, cols, w, width, 0, rows);
    else
        orc_horizontal_rows(plane, scratch, rows, cols, w, width, r, rows - r);
    orc_vertical_rows(scratch, plane, rows, cols, w, width, r, rows - r);
}

/* copy_back, S/conv.py:424-440: dst[region] := src[region]. */
ORC_API void orc_copy_region(const float *src, float *dst, int rows, int cols,
                             int row_lo, int row_hi, int col_lo, int col_hi)
{
    (void)rows;
    for (int y = row_lo; y < row_hi; ++y)
        memcpy(dst + (int64_t)y * cols + col_lo, src + (int64_t)y * cols + col_lo,
               sizeof(float) * (size_t)(col_hi - col_lo));
}

/* outer_product, S/kernels.py:66-72: K[i][j] = fl32(w[i] * w[j]). */
ORC_API void orc_outer_product(const float *w, int width, float *out)
{
    for (int i = 0; i < width; ++i)
        for (int j = 0; j < width; ++j)
            out[i * width + j] = w[i] * w[j];
}

/* ------------------------------------------------------------------------
 * Deterministic inputs. splitmix64, S/image.py:131-141: draw n (0-based) mixes
 * seed + (n+1)*gamma. `offset` lets a shard start mid-stream (counter-based).
 * kind 0: make_synthetic's [0,256) mapping, S/image.py:158-160: (x>>40)*2^-16.
 * kind 1: U[0,1): (x>>40)*2^-24 (exact float32).
 * kind 2: U[0,255): fl32((x>>40)*255) * 2^-24 (one rounding, then exact scale).
 */
static inline uint64_t orc_mix(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

ORC_API void orc_splitmix64(uint64_t seed, uint64_t offset, uint64_t count, uint64_t *out)
{
    for (uint64_t i = 0; i < count; ++i)
        out[i] = orc_mix(seed + (offset + i + 1) * 0x9E3779B97F4A7C15ULL);
}

ORC_API void orc_fill_synthetic(float *dst, uint64_t count, uint64_t seed, uint64_t offset, int kind)
{
    for (uint64_t i = 0; i < count; ++i) {
        uint64_t top = orc_mix(seed + (offset + i + 1) * 0x9E3779B97F4A7C15ULL) >> 40;
        float v;
        if (kind == 0)
            v = (float)top * (1.0f / 65536.0f);
        else if (kind == 1)
            v = (float)top * (1.0f / 16777216.0f);
        else
            v = (float)(top * 255ULL) * (1.0f / 16777216.0f);
        dst[i] = v;
    }
}

ORC_API int orc_abi_version(void) { return 1; }

/* Row band of the faithful/extended two-pass (the multi-GPU partitioner's unit,
 * SURVEY.md section 8e) restated directly from the reference's rules with
 * GLOBAL row indices: src holds global rows [src_row0, src_row0+src_rows), dst
 * row 0 is global row dst_row0; output rows [out_lo, out_hi) are produced.
 * Ring rows/cols (outside [r,R-r)x[r,C-r)) copy the input, as the in-place
 * reference leaves them (S/conv.py:392-421); valid samples are V(H0). */
ORC_API int orc_two_pass_band(const float *src, float *dst, int global_rows, int cols,
                              int src_row0, int src_rows, int dst_row0, int out_lo, int out_hi,
                              const float *w, int width, int extended)
{
    const int r = width / 2;
    float *scr = (float *)calloc((size_t)src_rows * (size_t)cols, sizeof(float));
    if (!scr) return -1;
    for (int i = 0; i < src_rows; ++i) {
        const int g = src_row0 + i;
        if (extended || (g >= r && g < global_rows - r))
            orc_horizontal_rows(src + (int64_t)i * cols - 0, scr + (int64_t)i * cols, 1, cols, w, width, 0, 1);
    }
    for (int y = out_lo; y < out_hi; ++y) {
        const float *a = src + (int64_t)(y - src_row0) * cols;
        float *d = dst + (int64_t)(y - dst_row0) * cols;
        memcpy(d, a, sizeof(float) * (size_t)cols);
        if (y < r || y >= global_rows - r) continue;
        for (int x = r; x < cols - r; ++x) d[x] = scr[(int64_t)(y - r - src_row0) * cols + x] * w[0];
        for (int m = 1; m < width; ++m) {
            const float *s = scr + (int64_t)(y - r + m - src_row0) * cols;
            for (int x = r; x < cols - r; ++x) {
                float term = s[x] * w[m];
                d[x] = d[x] + term;
            }
        }
    }
    free(scr);
    return 0;
}
