/*
 * CPU ORACLE - test infrastructure only.  Not part of the product and never
 * called by it: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs load this library, as the checker.
 *
 * A plain-C restatement of the reference's float64 "parallel phase"
 * (dequantise -> IDCT -> [chroma upsample] -> YCbCr->RGB), performing the
 * identical IEEE-754 double operation sequence so results are bit-exact:
 *
 *   _round_u8          pkg/src/hetjpeg/kernels/_native.pyx:312-318, fallback.py:37-38
 *   aan_1d             _native.pyx:321-351, fallback.py:67-91
 *   direct_1d          _native.pyx:354-361, fallback.py:51-64
 *   idct_block         _native.pyx:364-388, fallback.py:94-100,194-197
 *   color_px           _native.pyx:391-395, fallback.py:142-150
 *   render 4:4:4 row   _native.pyx:402-438, fallback.py:224-243
 *   render 4:2:2 row   _native.pyx:441-490, fallback.py:200-212,246-260
 *
 * 4:2:0 is NOT supported by the reference (parser.py:223-229 rejects it).
 * render 4:2:0 below is this repository's documented extension (DESIGN.md
 * "4:2:0 extension"): the same IDCT/colour/rounding, 16x16 MCUs with four
 * Y blocks per MCU in raster order, and the libjpeg h2v2 "fancy" triangle
 * filter over the PADDED chroma plane (mcus_per_row*8 x mcu_rows*8) with
 * edge replication at its first/last row and column - the padded-plane
 * convention the reference uses horizontally for 4:2:2.  Parity for 4:2:0
 * is self-consistency pinned only.
 *
 * Build with -ffp-contract=off and without -ffast-math (oracle/Makefile):
 * any FMA contraction would change the float64 bits.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oracle_tables.h"

static const double PRE[64] = OR_PRESCALE_INIT;
static const double BASIS[64] = OR_BASIS_INIT; /* BASIS[u*8+x] */

static inline uint8_t round_u8(double x) {
    x = floor(x + 0.5);
    if (x < 0.0) return 0;
    if (x > 255.0) return 255;
    return (uint8_t)x;
}

static inline void aan_1d(const double *x, int xs, double *y, int ys) {
    double d0 = x[0], d1 = x[xs], d2 = x[2 * xs], d3 = x[3 * xs];
    double d4 = x[4 * xs], d5 = x[5 * xs], d6 = x[6 * xs], d7 = x[7 * xs];
    double tmp10 = d0 + d4;
    double tmp11 = d0 - d4;
    double tmp13 = d2 + d6;
    double tmp12 = (d2 - d6) * OR_SQRT2 - tmp13;
    double e0 = tmp10 + tmp13;
    double e3 = tmp10 - tmp13;
    double e1 = tmp11 + tmp12;
    double e2 = tmp11 - tmp12;
    double z13 = d5 + d3;
    double z10 = d5 - d3;
    double z11 = d1 + d7;
    double z12 = d1 - d7;
    double t7 = z11 + z13;
    double t11 = (z11 - z13) * OR_SQRT2;
    double z5 = (z10 + z12) * OR_ROT;
    double t10 = OR_ROT_P * z12 - z5;
    double t12 = (-OR_ROT_M) * z10 + z5;
    double t6 = t12 - t7;
    double t5 = t11 - t6;
    double t4 = t10 + t5;
    y[0] = e0 + t7;
    y[ys] = e1 + t6;
    y[2 * ys] = e2 + t5;
    y[3 * ys] = e3 - t4;
    y[4 * ys] = e3 + t4;
    y[5 * ys] = e2 - t5;
    y[6 * ys] = e1 - t6;
    y[7 * ys] = e0 - t7;
}

static inline void direct_1d(const double *x, int xs, double *y, int ys) {
    for (int k = 0; k < 8; ++k) {
        double acc = 0.0;
        for (int r = 0; r < 8; ++r) acc += BASIS[r * 8 + k] * x[r * xs];
        y[k * ys] = acc;
    }
}

/* Pre-rounding transform core over dequantised input (no +128). */
void or_idct_core_f64(const int32_t *deq, double *out, int fast) {
    double d[64], g[64];
    if (fast) {
        for (int i = 0; i < 64; ++i) d[i] = (double)deq[i] * PRE[i];
        for (int c = 0; c < 8; ++c) aan_1d(&d[c], 8, &g[c], 8);
        for (int r = 0; r < 8; ++r) aan_1d(&g[8 * r], 1, &out[8 * r], 1);
    } else {
        for (int i = 0; i < 64; ++i) d[i] = (double)deq[i];
        for (int c = 0; c < 8; ++c) direct_1d(&d[c], 8, &g[c], 8);
        for (int r = 0; r < 8; ++r) direct_1d(&g[8 * r], 1, &out[8 * r], 1);
    }
}

/* Dequantise + transform + level shift + round one block into an 8x8
 * window of a sample plane with row stride `stride`. */
static void idct_block(const int16_t *coef, const int32_t *q, uint8_t *out,
                       int stride, int fast) {
    int32_t deq[64];
    double s[64];
    for (int i = 0; i < 64; ++i) deq[i] = (int32_t)coef[i] * q[i];
    or_idct_core_f64(deq, s, fast);
    for (int r = 0; r < 8; ++r)
        for (int c = 0; c < 8; ++c) out[r * stride + c] = round_u8(s[8 * r + c] + 128.0);
}

void or_idct_blocks(const int16_t *coef, const int32_t *q, uint8_t *out, long n, int fast) {
    for (long b = 0; b < n; ++b) idct_block(coef + 64 * b, q, out + 64 * b, 8, fast);
}

static inline void color_px(double y, double cb, double cr, uint8_t *rgb) {
    rgb[0] = round_u8(y + OR_CR_TO_R * (cr - 128.0));
    rgb[1] = round_u8(y - OR_CB_TO_G * (cb - 128.0) - OR_CR_TO_G * (cr - 128.0));
    rgb[2] = round_u8(y + OR_CB_TO_B * (cb - 128.0));
}

void or_ycbcr_to_rgb(const uint8_t *y, const uint8_t *cb, const uint8_t *cr,
                     uint8_t *rgb, long n) {
    for (long i = 0; i < n; ++i) color_px(y[i], cb[i], cr[i], rgb + 3 * i);
}

/* ------------------------------------------------------------------ */
/* per-MCU-row renderers                                               */
/* ------------------------------------------------------------------ */

typedef struct {
    const int16_t *y, *cb, *cr;
    const int32_t *q; /* 3 x 64, natural order */
    uint8_t *rgb;
    int width, height, mpr, mcu_rows, fast;
} job_t;

static void row_444(const job_t *j, int row, uint8_t *scratch) {
    const int sw = j->mpr * 8;
    uint8_t *ys = scratch, *cbs = scratch + 8 * sw, *crs = scratch + 16 * sw;
    for (int m = 0; m < j->mpr; ++m) {
        long b = (long)row * j->mpr + m;
        idct_block(j->y + 64 * b, j->q, ys + 8 * m, sw, j->fast);
        idct_block(j->cb + 64 * b, j->q + 64, cbs + 8 * m, sw, j->fast);
        idct_block(j->cr + 64 * b, j->q + 128, crs + 8 * m, sw, j->fast);
    }
    int y0 = row * 8;
    int nr = j->height - y0 < 8 ? j->height - y0 : 8;
    int nx = j->width < sw ? j->width : sw;
    for (int by = 0; by < nr; ++by) {
        uint8_t *px = j->rgb + (size_t)(y0 + by) * j->width * 3;
        for (int x = 0; x < nx; ++x)
            color_px(ys[by * sw + x], cbs[by * sw + x], crs[by * sw + x], px + 3 * x);
    }
}

/* h2v1 fancy upsample over the padded chroma stripe; even output pixel
 * (3c[k]+c[k-1]+1)>>2, odd (3c[k]+c[k+1]+2)>>2, edge copy at the stripe ends. */
static void row_422(const job_t *j, int row, uint8_t *scratch) {
    const int cw = j->mpr * 8, yw = j->mpr * 16;
    uint8_t *ys = scratch, *cbs = scratch + 8 * yw, *crs = cbs + 8 * cw;
    for (int m = 0; m < j->mpr; ++m) {
        long mcu = (long)row * j->mpr + m;
        idct_block(j->y + 64 * (2 * mcu), j->q, ys + 16 * m, yw, j->fast);
        idct_block(j->y + 64 * (2 * mcu + 1), j->q, ys + 16 * m + 8, yw, j->fast);
        idct_block(j->cb + 64 * mcu, j->q + 64, cbs + 8 * m, cw, j->fast);
        idct_block(j->cr + 64 * mcu, j->q + 128, crs + 8 * m, cw, j->fast);
    }
    int y0 = row * 8;
    int nr = j->height - y0 < 8 ? j->height - y0 : 8;
    for (int by = 0; by < nr; ++by) {
        uint8_t *px = j->rgb + (size_t)(y0 + by) * j->width * 3;
        const uint8_t *cbr = cbs + by * cw, *crr = crs + by * cw;
        for (int k = 0; k < cw; ++k) {
            int cbp = cbr[k > 0 ? k - 1 : 0], crp = crr[k > 0 ? k - 1 : 0];
            int cbn = cbr[k + 1 < cw ? k + 1 : cw - 1], crn = crr[k + 1 < cw ? k + 1 : cw - 1];
            int x = 2 * k;
            if (x < j->width)
                color_px(ys[by * yw + x], (3 * cbr[k] + cbp + 1) >> 2,
                         (3 * crr[k] + crp + 1) >> 2, px + 3 * x);
            ++x;
            if (x < j->width)
                color_px(ys[by * yw + x], (3 * cbr[k] + cbn + 2) >> 2,
                         (3 * crr[k] + crn + 2) >> 2, px + 3 * x);
        }
    }
}

/* 4:2:0 extension (see header comment).  Chroma rows of MCU rows row-1 and
 * row+1 provide the vertical context, replicated at the padded plane's top
 * and bottom edge. */
static void chroma_stripe(const job_t *j, const int16_t *plane, const int32_t *q,
                          int row, uint8_t *out) {
    const int cw = j->mpr * 8;
    for (int m = 0; m < j->mpr; ++m)
        idct_block(plane + 64 * ((long)row * j->mpr + m), q, out + 8 * m, cw, j->fast);
}

static void row_420(const job_t *j, int row, uint8_t *scratch) {
    const int cw = j->mpr * 8, yw = j->mpr * 16;
    uint8_t *ys = scratch;                 /* 16 x yw */
    uint8_t *cb3 = ys + 16 * yw;           /* 24 x cw : rows of MCU row-1,row,row+1 */
    uint8_t *cr3 = cb3 + 24 * cw;
    int *colsum_b = (int *)(cr3 + 24 * cw);
    int *colsum_r = colsum_b + cw;
    for (int m = 0; m < j->mpr; ++m) {
        long mcu = (long)row * j->mpr + m;
        for (int b = 0; b < 4; ++b)
            idct_block(j->y + 64 * (4 * mcu + b), j->q,
                       ys + (b >> 1) * 8 * yw + 16 * m + (b & 1) * 8, yw, j->fast);
    }
    chroma_stripe(j, j->cb, j->q + 64, row, cb3 + 8 * cw);
    chroma_stripe(j, j->cr, j->q + 128, row, cr3 + 8 * cw);
    if (row > 0) {
        chroma_stripe(j, j->cb, j->q + 64, row - 1, cb3);
        chroma_stripe(j, j->cr, j->q + 128, row - 1, cr3);
    }
    if (row + 1 < j->mcu_rows) {
        chroma_stripe(j, j->cb, j->q + 64, row + 1, cb3 + 16 * cw);
        chroma_stripe(j, j->cr, j->q + 128, row + 1, cr3 + 16 * cw);
    }
    const int ch = j->mcu_rows * 8; /* padded chroma plane height */
    int y0 = row * 16;
    int nr = j->height - y0 < 16 ? j->height - y0 : 16;
    for (int oy = 0; oy < nr; ++oy) {
        int ci = row * 8 + (oy >> 1);                 /* nearer chroma row */
        int cf = ci + ((oy & 1) ? 1 : -1);            /* farther chroma row */
        if (cf < 0) cf = 0;
        if (cf > ch - 1) cf = ch - 1;
        const uint8_t *bn = cb3 + (ci - (row - 1) * 8) * cw;
        const uint8_t *bf = cb3 + (cf - (row - 1) * 8) * cw;
        const uint8_t *rn = cr3 + (ci - (row - 1) * 8) * cw;
        const uint8_t *rf = cr3 + (cf - (row - 1) * 8) * cw;
        for (int k = 0; k < cw; ++k) {
            colsum_b[k] = 3 * bn[k] + bf[k];
            colsum_r[k] = 3 * rn[k] + rf[k];
        }
        uint8_t *px = j->rgb + (size_t)(y0 + oy) * j->width * 3;
        const uint8_t *yrow = ys + oy * yw;
        for (int k = 0; k < cw; ++k) {
            int bp = colsum_b[k > 0 ? k - 1 : 0], rp = colsum_r[k > 0 ? k - 1 : 0];
            int bq = colsum_b[k + 1 < cw ? k + 1 : cw - 1], rq = colsum_r[k + 1 < cw ? k + 1 : cw - 1];
            int x = 2 * k;
            if (x < j->width)
                color_px(yrow[x], (3 * colsum_b[k] + bp + 8) >> 4,
                         (3 * colsum_r[k] + rp + 8) >> 4, px + 3 * x);
            ++x;
            if (x < j->width)
                color_px(yrow[x], (3 * colsum_b[k] + bq + 7) >> 4,
                         (3 * colsum_r[k] + rq + 7) >> 4, px + 3 * x);
        }
    }
}

typedef struct {
    const job_t *job;
    int subsamp, r0, r1;
} span_t;

static size_t scratch_bytes(int mpr) {
    size_t yw = (size_t)mpr * 16, cw = (size_t)mpr * 8;
    return 16 * yw + 48 * cw + 2 * cw * sizeof(int) + 64;
}

static void *run_span(void *arg) {
    span_t *s = (span_t *)arg;
    uint8_t *scratch = (uint8_t *)malloc(scratch_bytes(s->job->mpr));
    for (int r = s->r0; r < s->r1; ++r) {
        if (s->subsamp == 0) row_444(s->job, r, scratch);
        else if (s->subsamp == 1) row_422(s->job, r, scratch);
        else row_420(s->job, r, scratch);
    }
    free(scratch);
    return NULL;
}

/*
 * Render MCU rows [row0, row0+n_rows) of one image into rgb (h x w x 3).
 * subsamp: 0 = 4:4:4 (8x8 MCU), 1 = 4:2:2 (16x8), 2 = 4:2:0 (16x16, extension).
 * mcu_rows is only used by 4:2:0 (vertical edge of the padded chroma plane).
 * threads > 1 splits the row range into contiguous stripes (one pthread each),
 * the way the reference's host lane splits stripes (executors.py:205-218).
 */
void or_render_rows(const int16_t *y, const int16_t *cb, const int16_t *cr,
                    const int32_t *q, uint8_t *rgb, int width, int height,
                    int mpr, int mcu_rows, int row0, int n_rows, int subsamp,
                    int fast, int threads) {
    if (n_rows <= 0) return;
    job_t job = {y, cb, cr, q, rgb, width, height, mpr, mcu_rows, fast};
    if (threads < 1) threads = 1;
    if (threads > n_rows) threads = n_rows;
    span_t *spans = (span_t *)calloc((size_t)threads, sizeof(span_t));
    pthread_t *tid = (pthread_t *)calloc((size_t)threads, sizeof(pthread_t));
    int base = n_rows / threads, extra = n_rows % threads, r = row0;
    for (int t = 0; t < threads; ++t) {
        int n = base + (t < extra ? 1 : 0);
        spans[t].job = &job;
        spans[t].subsamp = subsamp;
        spans[t].r0 = r;
        spans[t].r1 = r + n;
        r += n;
    }
    for (int t = 1; t < threads; ++t) pthread_create(&tid[t], NULL, run_span, &spans[t]);
    run_span(&spans[0]);
    for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
    free(spans);
    free(tid);
}
