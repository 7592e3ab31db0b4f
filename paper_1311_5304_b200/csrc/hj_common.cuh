// Device helpers shared by the render and per-block kernels.
//
//  * exact float64 AAN / direct-basis passes in the reference's operation
//    order (kernels/_native.pyx:312-388) with explicitly rounded
//    __dadd_rn/__dmul_rn (no FMA contraction);
//  * the integer colour formulas proven equal to the reference's float64
//    rounding over all 2^24 inputs (tools/gen_constants.py);
//  * byte packing through the saturating I2IP instruction
//    (cvt.pack.sat.u8.s32.b32: d = c<<16 | sat(a)<<8 | sat(b)).
#pragma once

#include <cstdint>

#include "hj_tables.h"

namespace hj {

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// Exact int32 -> float64 without the quarter-rate I2F.F64 conversion:
// as_double(0x43300000 : x ^ 0x80000000) == 2^52 + 2^31 + x.
__device__ __forceinline__ double i2d(int x) {
    return dsub(__hiloint2double(0x43300000, x ^ (int)0x80000000), 4503601774854144.0);
}

// _round_u8(s + 128.0) (_native.pyx:312-318, 388): floor(fl(fl(s+128)+0.5)),
// clamped to [0,255].  fl(a+0.5) never changes floor() for |a| < 2^51, so
// floor(fl(a+0.5)) = floor(a+0.5) is read off one round-down add into the
// 0.5-spaced binade [2^51, 2^52): lo32(rd(a + 1.5*2^51 + 0.5)) = floor(2a+1).
__device__ __forceinline__ int round_sample(double s) {
    double a = dadd(s, 128.0);
    double t = __dadd_rd(a, 3377699720527872.5);
    int n = __double2loint(t) >> 1;
    return min(max(n, 0), 255);
}

// One scaled-AAN 1-D pass, operation order of _native.pyx:321-351.
__device__ __forceinline__ void aan8(double &x0, double &x1, double &x2, double &x3, double &x4,
                                     double &x5, double &x6, double &x7) {
    double tmp10 = dadd(x0, x4);
    double tmp11 = dsub(x0, x4);
    double tmp13 = dadd(x2, x6);
    double tmp12 = dsub(dmul(dsub(x2, x6), HJ_SQRT2), tmp13);
    double e0 = dadd(tmp10, tmp13);
    double e3 = dsub(tmp10, tmp13);
    double e1 = dadd(tmp11, tmp12);
    double e2 = dsub(tmp11, tmp12);
    double z13 = dadd(x5, x3);
    double z10 = dsub(x5, x3);
    double z11 = dadd(x1, x7);
    double z12 = dsub(x1, x7);
    double t7 = dadd(z11, z13);
    double t11 = dmul(dsub(z11, z13), HJ_SQRT2);
    double z5 = dmul(dadd(z10, z12), HJ_ROT);
    double t10 = dsub(dmul(HJ_ROT_P, z12), z5);
    double t12 = dadd(dmul(-HJ_ROT_M, z10), z5);
    double t6 = dsub(t12, t7);
    double t5 = dsub(t11, t6);
    double t4 = dadd(t10, t5);
    x0 = dadd(e0, t7);
    x1 = dadd(e1, t6);
    x2 = dadd(e2, t5);
    x3 = dsub(e3, t4);
    x4 = dadd(e3, t4);
    x5 = dsub(e2, t5);
    x6 = dsub(e1, t6);
    x7 = dsub(e0, t7);
}

// One direct-basis 1-D pass (_native.pyx:354-361): y[k] = sum_r T[r][k]*x[r],
// accumulated from 0.0 in ascending r.  `basis` is T row-major.
__device__ __forceinline__ void direct8(double *x, const double *basis) {
    double y[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        double acc = 0.0;
#pragma unroll
        for (int r = 0; r < 8; ++r) acc = dadd(acc, dmul(basis[r * 8 + k], x[r]));
        y[k] = acc;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = y[k];
}

// ------------------------------------------------------------ colour

// Colour offsets (tools/gen_constants.py colour_constants): with K = 20,
//   R = clamp(Y + ((AR*Cr + CR) >> K)),  B = clamp(Y + ((AB*Cb + CB) >> K)),
//   G = clamp(Y + ((AGB*Cb + AGR*Cr + CG) >> K))  except the float64 tie pair
// (Cb, Cr) = (78, 178), where G loses 1 more for 47 <= Y <= 82.
// The G accumulator of that pair is a unique value (checked exhaustively),
// so it is detected from `gsum` alone.
constexpr int kColK = HJ_COL_K;
constexpr int kGSpecial = HJ_COL_AGB * 78 + HJ_COL_AGR * 178 + HJ_COL_CG;

struct Rgb {
    int r, g, b;
};

// Unclamped R, G, B of one pixel; sets `special` when the tie pair occurs.
__device__ __forceinline__ Rgb colour(int y, int cb, int cr, bool &special) {
    int rs = HJ_COL_AR * cr + HJ_COL_CR;
    int bs = HJ_COL_AB * cb + HJ_COL_CB;
    int gs = HJ_COL_AGB * cb + HJ_COL_AGR * cr + HJ_COL_CG;
    special |= (gs == kGSpecial);
    return Rgb{y + (rs >> kColK), y + (gs >> kColK), y + (bs >> kColK)};
}

// The additive colour constants held in registers: the multiplier goes into
// IMAD's immediate slot and the constant stays in a register instead of
// being rematerialised per pixel (IMAD takes one immediate).  The empty asm
// hides the values from constant folding.
struct ColourRegs {
    int cr, cb, cg, ar, ab, agb, agr;
};
__device__ __forceinline__ ColourRegs colour_regs() {
    ColourRegs k{HJ_COL_CR, HJ_COL_CB, HJ_COL_CG, HJ_COL_AR, HJ_COL_AB, HJ_COL_AGB, HJ_COL_AGR};
    asm("" : "+r"(k.cr), "+r"(k.cb), "+r"(k.cg), "+r"(k.ar), "+r"(k.ab), "+r"(k.agb), "+r"(k.agr));
    return k;
}
__device__ __forceinline__ Rgb colour(int y, int cb, int cr, bool &special, const ColourRegs &k) {
    int rs = k.ar * cr + k.cr;
    int bs = k.ab * cb + k.cb;
    int gs = k.agb * cb + (k.agr * cr + k.cg);
    special |= (gs == kGSpecial);
    return Rgb{y + (rs >> kColK), y + (gs >> kColK), y + (bs >> kColK)};
}

// Colour of the islow (libjpeg) decode mode: jdcolor.c ycc_rgb_convert with
// build_ycc_rgb_table (SCALEBITS 16, FIX(x) = (int)(x * 65536 + 0.5)):
//   R = y + ((FIX(1.402) * (cr-128) + 2^15) >> 16), B likewise with FIX(1.772),
//   G = y + ((-FIX(0.34414) * (cb-128) + 2^15 - FIX(0.71414) * (cr-128)) >> 16)
// in the same IMAD + arithmetic-shift form (no float64 tie: exact integers).
constexpr int kLjColK = 16;
__device__ __forceinline__ ColourRegs colour_regs_libjpeg() {
    ColourRegs k{32768 - 128 * 91881, 32768 - 128 * 116130, 32768 + 128 * (22554 + 46802), 91881, 116130,
                 -22554, -46802};
    asm("" : "+r"(k.cr), "+r"(k.cb), "+r"(k.cg), "+r"(k.ar), "+r"(k.ab), "+r"(k.agb), "+r"(k.agr));
    return k;
}
__device__ __forceinline__ Rgb colour_libjpeg(int y, int cb, int cr, const ColourRegs &k) {
    const int rs = k.ar * cr + k.cr;
    const int bs = k.ab * cb + k.cb;
    const int gs = k.agb * cb + (k.agr * cr + k.cg);
    return Rgb{y + (rs >> kLjColK), y + (gs >> kLjColK), y + (bs >> kLjColK)};
}

// The tie-pair correction for one pixel (rarely executed).
__device__ __forceinline__ int colour_g_exact(int y, int cb, int cr) {
    int g = y + ((HJ_COL_AGB * cb + HJ_COL_AGR * cr + HJ_COL_CG) >> kColK);
    if (cb == 78 && cr == 178 && (unsigned)(y - 47) <= 35u) g -= 1;
    return g;
}

// Saturating pack: returns c << 16 | sat_u8(a) << 8 | sat_u8(b).
__device__ __forceinline__ uint32_t pack2(int a, int b, uint32_t c) {
    uint32_t d;
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// bytes [b0 b1 b2 b3] (each saturated to [0,255])
__device__ __forceinline__ uint32_t pack4(int b0, int b1, int b2, int b3) {
    return pack2(b1, b0, pack2(b3, b2, 0u));
}

// 8 pixels -> 24 interleaved RGB bytes (6 words), saturating each channel.
__device__ __forceinline__ void pack_rgb8(const Rgb (&p)[8], uint32_t (&w)[6]) {
    w[0] = pack4(p[0].r, p[0].g, p[0].b, p[1].r);
    w[1] = pack4(p[1].g, p[1].b, p[2].r, p[2].g);
    w[2] = pack4(p[2].b, p[3].r, p[3].g, p[3].b);
    w[3] = pack4(p[4].r, p[4].g, p[4].b, p[5].r);
    w[4] = pack4(p[5].g, p[5].b, p[6].r, p[6].g);
    w[5] = pack4(p[6].b, p[7].r, p[7].g, p[7].b);
}

// Store 24 bytes (8 pixels) at dst, cropped to npx pixels.
__device__ __forceinline__ void store_rgb8(uint8_t *__restrict__ dst, const uint32_t (&w)[6], int npx) {
    uintptr_t a = reinterpret_cast<uintptr_t>(dst);
    if (npx == 8 && (a & 7) == 0) {
        uint2 *d = reinterpret_cast<uint2 *>(dst);
        d[0] = make_uint2(w[0], w[1]);
        d[1] = make_uint2(w[2], w[3]);
        d[2] = make_uint2(w[4], w[5]);
    } else if (npx == 8 && (a & 3) == 0) {
        uint32_t *d = reinterpret_cast<uint32_t *>(dst);
#pragma unroll
        for (int i = 0; i < 6; ++i) d[i] = w[i];
    } else {
#pragma unroll
        for (int i = 0; i < 24; ++i)
            if (i < npx * 3) dst[i] = (uint8_t)(w[i >> 2] >> (8 * (i & 3)));
    }
}

}  // namespace hj
