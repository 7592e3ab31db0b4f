/*
 * CPU ORACLE - test infrastructure only (tests/, smoke, bench's CPU legs).
 *
 * The "islow" decode mode: the parallel phase as libjpeg(-turbo) computes it,
 * which BASELINE.json's north_star names ("the fixed-point IDCT (libjpeg
 * jidctint 'islow')").  The reference package has no such path (its IDCT is
 * float64), so this restates the third-party
 * algorithm - libjpeg-turbo 3.1.x as bundled with Pillow 12.2 (the encoder
 * of every synthetic JPEG here) - and is pinned to Pillow's own decode of the
 * same JPEGs (tests/golden/make_islow_golden.py):
 *
 *   islow_block   jidctint.c jpeg_idct_islow: CONST_BITS 13, PASS1_BITS 2,
 *                 column pass DESCALE(., 11) into an int workspace, row pass
 *                 DESCALE(., 18), output range_limit[x & 1023] (IDCT
 *                 range-limit table of jdmaster.c prepare_range_limit_table),
 *                 i.e. sat_u8(sign_extend_10(x) + 128).  The zero-AC
 *                 column/row shortcuts are exact and omitted.  Arithmetic is
 *                 32-bit two's complement (JLONG as on ILP32 builds): on every
 *                 realistic stream it equals the LP64 C and the SIMD
 *                 implementations; for adversarial coefficients (|coef*q|
 *                 beyond the JPEG 8-bit range) libjpeg-turbo's own builds
 *                 disagree with each other, and this mode is defined as the
 *                 wrapping 32-bit arithmetic.
 *   upsampling    jdsample.c: h2v1 / h2v2 fancy triangle filter when the
 *                 component's downsampled_width > 2, else box replication
 *                 (h2v1_upsample / h2v2_upsample); edges replicated at the
 *                 REAL chroma size ceil(w/2) x ceil(h/2) (jdsample.c first /
 *                 last column cases; jdmainct.c context rows: the row above
 *                 the first and below the last real row repeat it).
 *   colour        jdcolor.c ycc_rgb_convert with build_ycc_rgb_table
 *                 (SCALEBITS 16): R = y + Cr_r_tab[cr], B = y + Cb_b_tab[cb],
 *                 G = y + ((Cb_g_tab[cb] + Cr_g_tab[cr]) >> 16), clamped.
 *
 * Coefficient layout = the reference's CoefficientBuffer (entropy.py:31-56).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define CB 13 /* CONST_BITS */
#define P1 2  /* PASS1_BITS */
enum {
    F0298 = 2446, F0390 = 3196, F0541 = 4433, F0765 = 6270, F0899 = 7373, F1175 = 9633,
    F1501 = 12299, F1847 = 15137, F1961 = 16069, F2053 = 16819, F2562 = 20995, F3072 = 25172
};

/* 32-bit wrapping arithmetic */
static inline int32_t w_add(int32_t a, int32_t b) { return (int32_t)((uint32_t)a + (uint32_t)b); }
static inline int32_t w_sub(int32_t a, int32_t b) { return (int32_t)((uint32_t)a - (uint32_t)b); }
static inline int32_t w_mul(int32_t a, int32_t b) { return (int32_t)((uint32_t)a * (uint32_t)b); }
static inline int32_t w_shl(int32_t a, int n) { return (int32_t)((uint32_t)a << n); }
static inline int32_t descale(int32_t x, int n) { return w_add(x, 1 << (n - 1)) >> n; } /* arithmetic */

/* One 1-D pass of jidctint (either direction): in[0..7] -> out[0..7]
 * before the final DESCALE (returned scaled by 2^CONST_BITS). */
static void islow_1d(const int32_t *in, int32_t *out) {
    int32_t z1, z2, z3, z4, z5, t0, t1, t2, t3, t10, t11, t12, t13;
    /* even part */
    z2 = in[2];
    z3 = in[6];
    z1 = w_mul(w_add(z2, z3), F0541);
    t2 = w_add(z1, w_mul(z3, -F1847));
    t3 = w_add(z1, w_mul(z2, F0765));
    t0 = w_shl(w_add(in[0], in[4]), CB);
    t1 = w_shl(w_sub(in[0], in[4]), CB);
    t10 = w_add(t0, t3);
    t13 = w_sub(t0, t3);
    t11 = w_add(t1, t2);
    t12 = w_sub(t1, t2);
    /* odd part */
    t0 = in[7];
    t1 = in[5];
    t2 = in[3];
    t3 = in[1];
    z1 = w_add(t0, t3);
    z2 = w_add(t1, t2);
    z3 = w_add(t0, t2);
    z4 = w_add(t1, t3);
    z5 = w_mul(w_add(z3, z4), F1175);
    t0 = w_mul(t0, F0298);
    t1 = w_mul(t1, F2053);
    t2 = w_mul(t2, F3072);
    t3 = w_mul(t3, F1501);
    z1 = w_mul(z1, -F0899);
    z2 = w_mul(z2, -F2562);
    z3 = w_mul(z3, -F1961);
    z4 = w_mul(z4, -F0390);
    z3 = w_add(z3, z5);
    z4 = w_add(z4, z5);
    t0 = w_add(t0, w_add(z1, z3));
    t1 = w_add(t1, w_add(z2, z4));
    t2 = w_add(t2, w_add(z2, z3));
    t3 = w_add(t3, w_add(z1, z4));
    out[0] = w_add(t10, t3);
    out[7] = w_sub(t10, t3);
    out[1] = w_add(t11, t2);
    out[6] = w_sub(t11, t2);
    out[2] = w_add(t12, t1);
    out[5] = w_sub(t12, t1);
    out[3] = w_add(t13, t0);
    out[4] = w_sub(t13, t0);
}

static inline uint8_t range_limit(int32_t x) {
    int32_t v = (int32_t)((uint32_t)x << 22) >> 22; /* x & 1023 read as a signed 10-bit value */
    v += 128;
    return (uint8_t)(v < 0 ? 0 : v > 255 ? 255 : v);
}

/* coef: 64 int16 natural order; q: 64 int32 natural order; out: 8x8 u8 row-major */
void lj_islow_block(const int16_t *coef, const int32_t *q, uint8_t *out) {
    int32_t ws[64], col[8], res[8];
    for (int c = 0; c < 8; ++c) {
        for (int r = 0; r < 8; ++r) col[r] = w_mul(coef[r * 8 + c], q[r * 8 + c]);
        islow_1d(col, res);
        for (int r = 0; r < 8; ++r) ws[r * 8 + c] = descale(res[r], CB - P1);
    }
    for (int r = 0; r < 8; ++r) {
        islow_1d(ws + r * 8, res);
        for (int c = 0; c < 8; ++c) out[r * 8 + c] = range_limit(descale(res[c], CB + P1 + 3));
    }
}

void lj_islow_blocks(const int16_t *coef, const int32_t *q, uint8_t *out, long n) {
    for (long i = 0; i < n; ++i) lj_islow_block(coef + 64 * i, q, out + 64 * i);
}

/* jdcolor.c build_ycc_rgb_table / ycc_rgb_convert */
#define SCALEBITS 16
#define ONE_HALF (1 << (SCALEBITS - 1))
#define FIX(x) ((int32_t)((x) * (1 << SCALEBITS) + 0.5))
static inline uint8_t clamp255(int v) { return (uint8_t)(v < 0 ? 0 : v > 255 ? 255 : v); }
static inline void lj_color(int y, int cb, int cr, uint8_t *rgb) {
    const int xb = cb - 128, xr = cr - 128;
    const int r_off = (FIX(1.40200) * xr + ONE_HALF) >> SCALEBITS;
    const int b_off = (FIX(1.77200) * xb + ONE_HALF) >> SCALEBITS;
    const int g_off = ((-FIX(0.34414)) * xb + ONE_HALF + (-FIX(0.71414)) * xr) >> SCALEBITS;
    rgb[0] = clamp255(y + r_off);
    rgb[1] = clamp255(y + g_off);
    rgb[2] = clamp255(y + b_off);
}

void lj_ycc_rgb(const uint8_t *y, const uint8_t *cb, const uint8_t *cr, uint8_t *rgb, long n) {
    for (long i = 0; i < n; ++i) lj_color(y[i], cb[i], cr[i], rgb + 3 * i);
}

static inline int clampi(int v, int lo, int hi) { return v < lo ? lo : v > hi ? hi : v; }

/* Whole image (rows [y0, y1) of RGB written).  sub: 0 = 4:4:4, 1 = 4:2:2,
 * 2 = 4:2:0.  Planes are MCU-ordered as in the reference's buffer. */
void lj_render(const int16_t *yb, const int16_t *cbb, const int16_t *crb, const int32_t *q, uint8_t *rgb,
               int w, int h, int sub, int y0, int y1) {
    const int mw = sub == 0 ? 8 : 16, mh = sub == 2 ? 16 : 8, ypm = sub == 0 ? 1 : sub == 1 ? 2 : 4;
    const int mpr = (w + mw - 1) / mw, rows = (h + mh - 1) / mh;
    const int pw = mpr * mw, ph = rows * mh;   /* padded luma plane */
    const int cpw = mpr * 8, cph = rows * 8;   /* padded chroma plane */
    uint8_t *Y = malloc((size_t)pw * ph), *Cb = malloc((size_t)cpw * cph), *Cr = malloc((size_t)cpw * cph);
    uint8_t blk[64];
    for (int m = 0; m < mpr * rows; ++m) {
        const int mx = m % mpr, my = m / mpr;
        for (int j = 0; j < ypm; ++j) {
            lj_islow_block(yb + ((size_t)m * ypm + j) * 64, q, blk);
            const int bx = mx * mw + (j % (mw / 8)) * 8, by = my * mh + (j / (mw / 8)) * 8;
            for (int r = 0; r < 8; ++r) memcpy(Y + (size_t)(by + r) * pw + bx, blk + 8 * r, 8);
        }
        lj_islow_block(cbb + (size_t)m * 64, q + 64, blk);
        for (int r = 0; r < 8; ++r) memcpy(Cb + (size_t)(my * 8 + r) * cpw + mx * 8, blk + 8 * r, 8);
        lj_islow_block(crb + (size_t)m * 64, q + 128, blk);
        for (int r = 0; r < 8; ++r) memcpy(Cr + (size_t)(my * 8 + r) * cpw + mx * 8, blk + 8 * r, 8);
    }
    const int cw = sub == 0 ? w : (w + 1) / 2;          /* downsampled_width */
    const int ch = sub == 2 ? (h + 1) / 2 : h;          /* downsampled_height */
    const int fancy = sub == 0 || cw > 2;
    int *cs = malloc(sizeof(int) * (size_t)(cw + 2) * 2);
    for (int y = y0; y < y1; ++y) {
        uint8_t *out = rgb + (size_t)y * w * 3;
        if (sub == 0) {
            for (int x = 0; x < w; ++x)
                lj_color(Y[(size_t)y * pw + x], Cb[(size_t)y * cpw + x], Cr[(size_t)y * cpw + x], out + 3 * x);
            continue;
        }
        /* chroma column sums (x 4 for 4:2:2 so both filters share the form) */
        for (int p = 0; p < 2; ++p) {
            const uint8_t *pl = p ? Cr : Cb;
            int *s = cs + p * (cw + 2) + 1;
            for (int k = 0; k < cw; ++k) {
                if (sub == 1) {
                    s[k] = pl[(size_t)y * cpw + k];
                } else if (!fancy) {
                    s[k] = pl[(size_t)(y / 2) * cpw + k];
                } else {
                    const int rn = y / 2, rf = clampi(y & 1 ? rn + 1 : rn - 1, 0, ch - 1);
                    s[k] = 3 * pl[(size_t)rn * cpw + k] + pl[(size_t)rf * cpw + k];
                }
            }
            s[-1] = s[0];
            s[cw] = s[cw - 1];
        }
        for (int x = 0; x < w; ++x) {
            const int k = x / 2;
            int c[2];
            for (int p = 0; p < 2; ++p) {
                const int *s = cs + p * (cw + 2) + 1;
                if (!fancy) c[p] = s[k];
                else if (sub == 1) c[p] = x & 1 ? (3 * s[k] + s[k + 1] + 2) >> 2 : (3 * s[k] + s[k - 1] + 1) >> 2;
                else c[p] = x & 1 ? (3 * s[k] + s[k + 1] + 7) >> 4 : (3 * s[k] + s[k - 1] + 8) >> 4;
            }
            lj_color(Y[(size_t)y * pw + x], c[0], c[1], out + 3 * x);
        }
    }
    free(cs);
    free(Y);
    free(Cb);
    free(Cr);
}
