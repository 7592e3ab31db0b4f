// sm_100a render kernel (v3): dequantise -> IDCT -> [h2v1 / h2v2 fancy
// upsample] -> YCbCr->RGB, bit-exact against the reference's float64 path
// (kernels/_native.pyx:312-549, kernels/fallback.py:37-260).
//
// IDCT numerics: every block is first transformed
// in binary32 with the reference's AAN operation order, two lanes per
// FADD2/FFMA2 instruction: screen_rows (4:2:0) pairs two columns in the
// column pass and two rows in the row pass, with 2x2 register transposes
// (explicit PRMT copies) between; screen_cols (4:4:4 / 4:2:2) puts two rows
// of ONE column transform in a register (aan_col) so the row pass needs no
// transposes.  A rigorous first-order error bound E = u * sum_i K_i |x_i|
// (K from tools/analysis/screen_constants.py) brackets each sample; if no
// rounding boundary of floor(s + 128.5) lies inside [s - E, s + E] for all
// 64 samples, the binary32 result provably rounds like the reference's
// float64 one.  Otherwise (a few percent of real blocks; every block in
// "direct" mode) the block is queued and recomputed in exact float64
// (explicitly rounded __dadd_rn/__dmul_rn, the reference's operation order)
// by 8 cooperating threads.
//
// Work decomposition: a CTA (64 threads for 4:4:4 / 4:2:2, 128 for 4:2:0)
// owns a strip of MCU columns of one image and sweeps down a range of MCU
// rows.  Step s is two phases:
//   A. screen: one job (two blocks) per thread - the Y blocks of MCU row s
//      and the chroma (Cb, Cr) pairs of MCU row s (s+1 for 4:2:0, whose
//      vertical filter needs the next row) -> sample planes in shared memory;
//      blocks the screen cannot prove are queued.  Coefficients arrive as
//      256-bit L1::no_allocate loads.
//   B. the queued blocks' exact recompute, overlapped with the pixel stage
//      of MCU row s-1 (16-pixel items handed out through a shared counter,
//      so the threads busy with float64 simply take fewer items):
//      upsample (SWAR, both chroma planes per 32-bit op) + integer colour +
//      saturating I2IP byte packing + 16-byte RGB stores.
// Sample planes are double (Y) / triple (4:2:0 chroma) buffered across steps.
// One thread prefetches the next step's coefficient ranges into L2 with
// bulk prefetches (cp.async.bulk.prefetch.L2).
#include <atomic>
#include <cstdint>

#include "hj_common.cuh"
#include "hj_render.cuh"
#include "hj_screen.h"
#include "hj_mtable.h"
#include "hj_tc.cuh"

namespace hj {

namespace {

__constant__ double kPre64[64] = HJ_PRESCALE_INIT;
__constant__ double kBasis64[64] = HJ_BASIS_INIT;
__constant__ float kScreenK[64] = HJ_SCREEN_K_INIT;

typedef unsigned long long u64;

// Blocks recomputed by the exact float64 path (all launches; diagnostics).
__device__ unsigned long long g_exact_blocks;

// ---------------------------------------------------------- packed f32x2
__device__ __forceinline__ u64 pk(float lo, float hi) {
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float plo(u64 v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float phi(u64 v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
    u64 d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
    u64 d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
    u64 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
    u64 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}

// binary32 rotators (the reference's decimal literals, constants.py:31-35)
#define F_SQRT2 1.414213562f
#define F_ROT 1.847759065f
#define F_ROT_P 1.082392200f
#define F_ROT_M 2.613125930f

// One AAN pass on 2 independent lanes, the node structure analysed by
// tools/analysis/screen_constants.py: FFMA at tmp12 / t10 / t12, products at
// t11 / z5, everything else one rounded add/sub.  tmp12 and t10 are carried
// negated (exactly: round-to-nearest is sign-symmetric).
__device__ __forceinline__ void aan_x2(u64 &d0, u64 &d1, u64 &d2, u64 &d3, u64 &d4, u64 &d5, u64 &d6,
                                       u64 &d7) {
    const u64 sq = pk(F_SQRT2, F_SQRT2), nsq = pk(-F_SQRT2, -F_SQRT2);
    const u64 rot = pk(F_ROT, F_ROT), nrotp = pk(-F_ROT_P, -F_ROT_P), nrotm = pk(-F_ROT_M, -F_ROT_M);
    u64 tmp10 = add2(d0, d4);
    u64 tmp11 = sub2(d0, d4);
    u64 tmp13 = add2(d2, d6);
    u64 ntmp12 = fma2(sub2(d2, d6), nsq, tmp13);  // = -(a*SQRT2 - tmp13)
    u64 e0 = add2(tmp10, tmp13);
    u64 e3 = sub2(tmp10, tmp13);
    u64 e1 = sub2(tmp11, ntmp12);
    u64 e2 = add2(tmp11, ntmp12);
    u64 z13 = add2(d5, d3);
    u64 z10 = sub2(d5, d3);
    u64 z11 = add2(d1, d7);
    u64 z12 = sub2(d1, d7);
    u64 t7 = add2(z11, z13);
    u64 t11 = mul2(sub2(z11, z13), sq);
    u64 z5 = mul2(add2(z10, z12), rot);
    u64 nt10 = fma2(z12, nrotp, z5);  // = -(ROT_P*z12 - z5)
    u64 t12 = fma2(z10, nrotm, z5);   // = -ROT_M*z10 + z5
    u64 t6 = sub2(t12, t7);
    u64 t5 = sub2(t11, t6);
    u64 t4 = sub2(t5, nt10);
    d0 = add2(e0, t7);
    d1 = add2(e1, t6);
    d2 = add2(e2, t5);
    d3 = sub2(e3, t4);
    d4 = add2(e3, t4);
    d5 = sub2(e2, t5);
    d6 = sub2(e1, t6);
    d7 = sub2(e0, t7);
}

// Bracket constants of one block: E = u*B*(1 + 2.5e-3) + 2^-16 (rounding of
// t) + 2^-30 (float64 side), rounded up to the 2^-15 grid so 384.5 -/+ Eq is
// exact in binary32.
__device__ __forceinline__ float bracket(float B) {
    float e = fmaf(B, 5.9754e-8f, 1.5260e-5f);
    return ceilf(e * 32768.0f) * (1.0f / 32768.0f);
}

__device__ __forceinline__ float4 lds128f(const float *p) {
    float4 v;
    unsigned a = (unsigned)__cvta_generic_to_shared(p);
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}

// Per-sample rounding test of one f32x2 output pair (DESIGN.md "FP32
// screen").  t = v + C with C = 384.5 -/+ Eq lands in the binade [256, 512)
// (ulp 2^-15) for v in [-128.5, 127.5), where floor(v + 128.5) =
// (bits >> 15) - 0x8700.  `acc` collects bits(t-) ^ bits(t+): any bit >= 15
// means some bracket straddles a rounding boundary or a binade edge.
// Outside the binade the integer read-out saturates the right way with an
// ARITHMETIC shift of the signed bit pattern: t >= 512 gives n >= 256 (255 -
// the true sample exceeds 255.5 - E); 0 <= t < 256 gives n < 0 and a negative
// t (v < -384.5) a negative pattern, both 0 - the true sample is below
// -0.5 + E.  So no clamp is needed.
__device__ __forceinline__ void round_pair(u64 v, u64 cm, u64 cp, uint32_t &acc, int &n_lo, int &n_hi) {
    u64 tm = add2(v, cm), tp = add2(v, cp);
    uint32_t a0 = __float_as_uint(plo(tm)), a1 = __float_as_uint(phi(tm));
    uint32_t b0 = __float_as_uint(plo(tp)), b1 = __float_as_uint(phi(tp));
    acc |= (a0 ^ b0) | (a1 ^ b1);
    n_lo = ((int)a0 >> 15) - 0x8700;
    n_hi = ((int)a1 >> 15) - 0x8700;
}

// One block row pair (32 B = one sector) per load: 256-bit LDG on sm_100.
// L1::no_allocate: the stream is read once, and keeping it out of L1 leaves
// the spill slots and the exact path L1-resident (measured +3 %).
#ifndef HJ_LDG_NA
#define HJ_LDG_NA 1
#endif
#ifndef HJ_LDG256
#define HJ_LDG256 1
#endif
__device__ __forceinline__ void ldg_rows2(const int4 *p, int4 &a, int4 &b) {
#if HJ_LDG256
#if HJ_LDG_NA
    asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
#else
    asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
#endif
                 : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
                 : "l"(p));
#else
    a = __ldg(p);
    b = __ldg(p + 1);
#endif
}

// HJ_CVT_LO: the low int16 half converted as a PRMT sign extension + I2FP
// (integer ALU) instead of I2F.S16 (the quarter-rate XU pipe).
#ifndef HJ_CVT_LO
#define HJ_CVT_LO 0
#endif
__device__ __forceinline__ float cvt_lo16(int w) {
#if HJ_CVT_LO
    int x;
    asm("prmt.b32 %0, %1, 0, 0x9910;" : "=r"(x) : "r"(w));
    float f;
    asm("cvt.rn.f32.s32 %0, %1;" : "=f"(f) : "r"(x));
    return f;
#else
    return (float)(short)(w & 0xffff);
#endif
}
#ifndef HJ_CVT_H1
#define HJ_CVT_H1 0
#endif
// The 2x2 transposes between the passes as explicit PRMT copies: ptxas
// otherwise emits IMAD.MOV, on the FMA pipe the screen already saturates.
#ifndef HJ_PRMT_T
#define HJ_PRMT_T 1
#endif
__device__ __forceinline__ float alu_mov(float x) {
    uint32_t d;
    asm volatile("prmt.b32 %0, %1, 0, 0x3210;" : "=r"(d) : "r"(__float_as_uint(x)));
    return __uint_as_float(d);
}

// FP32 screen of one block: returns true (and the 64 samples, u8 row-major,
// 4 per word) when every sample is proven equal to the reference's float64
// result; false = recompute exactly.  Two f32x2 formulations of the same
// operations: screen_rows (lanes = two columns in the column pass, 2x2
// register transposes before the row pass) and screen_cols (aan_col below).
__device__ __forceinline__ bool screen_rows(const int16_t *__restrict__ src, const float *qf,
                                             uint32_t (&out)[16]) {
    int4 raw[8];
    const int4 *s4 = reinterpret_cast<const int4 *>(src);
#pragma unroll
    for (int r = 0; r < 8; r += 2) ldg_rows2(s4 + r, raw[r], raw[r + 1]);
    u64 X[4][8];  // X[cp][r] = (x[r][2cp], x[r][2cp+1])
    float b0 = 0.f, b1 = 0.f, b2 = 0.f, b3 = 0.f;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        float4 qa = lds128f(qf + r * 8), qb = lds128f(qf + r * 8 + 4);
        const int w[4] = {raw[r].x, raw[r].y, raw[r].z, raw[r].w};
        const float q[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
#pragma unroll
        for (int cp = 0; cp < 4; ++cp) {
            float c0 = cvt_lo16(w[cp]);
            float c1 = (float)(w[cp] >> 16);
            u64 x = mul2(pk(c0, c1), pk(q[2 * cp], q[2 * cp + 1]));
            X[cp][r] = x;
            if (cp & 1) {
                b1 = fmaf(fabsf(plo(x)), kScreenK[r * 8 + 2 * cp], b1);
                b3 = fmaf(fabsf(phi(x)), kScreenK[r * 8 + 2 * cp + 1], b3);
            } else {
                b0 = fmaf(fabsf(plo(x)), kScreenK[r * 8 + 2 * cp], b0);
                b2 = fmaf(fabsf(phi(x)), kScreenK[r * 8 + 2 * cp + 1], b2);
            }
        }
    }
    // bound: E = u*B*(1 + 2.5e-3) + 2^-16 (rounding of t) + 2^-30 (float64
    // side), rounded up to the 2^-15 grid so 384.5 -/+ Eq is exact in binary32
    const float eq = bracket((b0 + b1) + (b2 + b3));
    u64 cm = pk(384.5f - eq, 384.5f - eq), cpl = pk(384.5f + eq, 384.5f + eq);

#pragma unroll
    for (int cp = 0; cp < 4; ++cp)
        aan_x2(X[cp][0], X[cp][1], X[cp][2], X[cp][3], X[cp][4], X[cp][5], X[cp][6], X[cp][7]);

    uint32_t acc = 0;
#pragma unroll
    for (int rp = 0; rp < 4; ++rp) {
        const int r0 = 2 * rp, r1 = 2 * rp + 1;
        u64 Q[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            u64 a = X[j >> 1][r0], b = X[j >> 1][r1];
#if HJ_PRMT_T
            Q[j] = (j & 1) ? pk(alu_mov(phi(a)), alu_mov(phi(b))) : pk(alu_mov(plo(a)), alu_mov(plo(b)));
#else
            Q[j] = (j & 1) ? pk(phi(a), phi(b)) : pk(plo(a), plo(b));
#endif
        }
        aan_x2(Q[0], Q[1], Q[2], Q[3], Q[4], Q[5], Q[6], Q[7]);
        int n0[8], n1[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) round_pair(Q[c], cm, cpl, acc, n0[c], n1[c]);
        out[r0 * 2] = pack4(n0[0], n0[1], n0[2], n0[3]);
        out[r0 * 2 + 1] = pack4(n0[4], n0[5], n0[6], n0[7]);
        out[r1 * 2] = pack4(n1[0], n1[1], n1[2], n1[3]);
        out[r1 * 2 + 1] = pack4(n1[4], n1[5], n1[6], n1[7]);
    }
    return (acc >> 15) == 0;
}

// Column pass with the two f32x2 lanes inside ONE column transform (two rows
// of the column per register), so that its outputs are already the row pairs
// the row pass consumes: no 2x2 register transposes between the passes.
// Every lane computes exactly the IEEE operation of aan_x2 on the same
// operands (x*(+-1) + y inside an FMA is the rounded sum / difference), so
// the screen's values - and its error bound - are unchanged.
//   in:  A = (x0, x2)  B = (x4, x6)  C = (x5, x1)  D = (x3, x7)
//   out: A = (y0, y3)  B = (y7, y4)  C = (y1, y2)  D = (y6, y5)
__device__ __forceinline__ u64 bc(float x) { return pk(x, x); }
// (1, -1), (-1, 1), (-ROT_M, -ROT_P) as constant-bank pairs: ptxas keeps them
// in uniform registers and uses them as FFMA2 operands directly (built from
// immediates they would be re-materialised into register pairs at each use)
__constant__ __align__(8) float kColPairs[6] = {1.0f, -1.0f, -1.0f, 1.0f, -F_ROT_M, -F_ROT_P};
__device__ __forceinline__ u64 col_pair(int i) { return reinterpret_cast<const u64 *>(kColPairs)[i]; }
__device__ __forceinline__ void aan_col(u64 &A, u64 &B, u64 &C, u64 &D, u64 pm, u64 mp, u64 nrot) {
    const u64 U = add2(A, B);   // (tmp10, tmp13)
    const u64 V = sub2(A, B);   // (tmp11, d2 - d6)
    const u64 Z1 = add2(C, D);  // (z13, z11)
    const u64 Z2 = sub2(C, D);  // (z10, z12)
    const float ntmp12 = fmaf(phi(V), -F_SQRT2, phi(U));
    const u64 E03 = fma2(bc(phi(U)), pm, bc(plo(U)));   // (e0, e3) = tmp10 +- tmp13
    const u64 E12 = fma2(bc(ntmp12), mp, bc(plo(V)));   // (e1, e2) = tmp11 -+ ntmp12
    const u64 T7S = fma2(bc(plo(Z1)), pm, bc(phi(Z1))); // (t7, z11 - z13)
    const float t11 = phi(T7S) * F_SQRT2;
    const float z5 = (plo(Z2) + phi(Z2)) * F_ROT;
    const u64 T12 = fma2(Z2, nrot, bc(z5));             // (t12, nt10)
    const float t7 = plo(T7S);
    const float t6 = plo(T12) - t7;
    const float t5 = t11 - t6;
    const float t4 = t5 - phi(T12);
    const u64 T74 = pk(t7, t4), T65 = pk(t6, t5);
    A = fma2(T74, pm, E03);  // (e0 + t7, e3 - t4)
    B = fma2(T74, mp, E03);  // (e0 - t7, e3 + t4)
    C = add2(E12, T65);      // (e1 + t6, e2 + t5)
    D = sub2(E12, T65);      // (e1 - t6, e2 - t5)
}

// Shared-memory order of the binary32 dequantisation factors: row-major for
// screen_rows; for screen_cols column c holds rows (0, 2, 4, 6, 5, 1, 3, 7)
// at [8c, 8c + 8).
__host__ __device__ constexpr int qf_slot(bool cols, int r, int c) {
    return !cols ? 8 * r + c
                 : 8 * c + (r == 0 ? 0 : r == 2 ? 1 : r == 4 ? 2 : r == 6 ? 3 : r == 5 ? 4 : r == 1 ? 5 : r == 3 ? 6 : 7);
}

__device__ __forceinline__ bool screen_cols(const int16_t *__restrict__ src, const float *qf,
                                             uint32_t (&out)[16]) {
    int4 raw[8];
    const int4 *s4 = reinterpret_cast<const int4 *>(src);
#pragma unroll
    for (int r = 0; r < 8; r += 2) ldg_rows2(s4 + r, raw[r], raw[r + 1]);
    const u64 pm = col_pair(0), mp = col_pair(1), nrot = col_pair(2);
    u64 Y[8][4];  // Y[c][k]: column c, row pair k
    float b0 = 0.f, b1 = 0.f, b2 = 0.f, b3 = 0.f;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        float f[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int w = c < 2 ? raw[r].x : c < 4 ? raw[r].y : c < 6 ? raw[r].z : raw[r].w;
#if HJ_CVT_H1
            f[r] = (c & 1) ? (float)(short)((unsigned)w >> 16) : (float)(short)(w & 0xffff);
#else
            f[r] = (c & 1) ? (float)(w >> 16) : cvt_lo16(w);
#endif
        }
        const float4 qa = lds128f(qf + 8 * c), qb = lds128f(qf + 8 * c + 4);
        u64 A = mul2(pk(f[0], f[2]), pk(qa.x, qa.y));
        u64 B = mul2(pk(f[4], f[6]), pk(qa.z, qa.w));
        u64 C = mul2(pk(f[5], f[1]), pk(qb.x, qb.y));
        u64 D = mul2(pk(f[3], f[7]), pk(qb.z, qb.w));
        b0 = fmaf(fabsf(plo(A)), kScreenK[0 * 8 + c], b0);
        b1 = fmaf(fabsf(phi(A)), kScreenK[2 * 8 + c], b1);
        b2 = fmaf(fabsf(plo(B)), kScreenK[4 * 8 + c], b2);
        b3 = fmaf(fabsf(phi(B)), kScreenK[6 * 8 + c], b3);
        b0 = fmaf(fabsf(plo(C)), kScreenK[5 * 8 + c], b0);
        b1 = fmaf(fabsf(phi(C)), kScreenK[1 * 8 + c], b1);
        b2 = fmaf(fabsf(plo(D)), kScreenK[3 * 8 + c], b2);
        b3 = fmaf(fabsf(phi(D)), kScreenK[7 * 8 + c], b3);
        aan_col(A, B, C, D, pm, mp, nrot);
        Y[c][0] = A;
        Y[c][1] = B;
        Y[c][2] = C;
        Y[c][3] = D;
    }
    const float eq = bracket((b0 + b1) + (b2 + b3));
    const u64 cm = pk(384.5f - eq, 384.5f - eq), cpl = pk(384.5f + eq, 384.5f + eq);
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        // row pairs (0,3) (7,4) (1,2) (6,5)
        const int ra = k == 0 ? 0 : k == 1 ? 7 : k == 2 ? 1 : 6;
        const int rb = k == 0 ? 3 : k == 1 ? 4 : k == 2 ? 2 : 5;
        aan_x2(Y[0][k], Y[1][k], Y[2][k], Y[3][k], Y[4][k], Y[5][k], Y[6][k], Y[7][k]);
        int n0[8], n1[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) round_pair(Y[c][k], cm, cpl, acc, n0[c], n1[c]);
        out[ra * 2] = pack4(n0[0], n0[1], n0[2], n0[3]);
        out[ra * 2 + 1] = pack4(n0[4], n0[5], n0[6], n0[7]);
        out[rb * 2] = pack4(n1[0], n1[1], n1[2], n1[3]);
        out[rb * 2 + 1] = pack4(n1[4], n1[5], n1[6], n1[7]);
    }
    return (acc >> 15) == 0;
}

// 4:4:4 takes screen_cols (measured +4 %).  4:2:0 and 4:2:2 keep
// screen_rows: the 4:2:0 kernel sits at the 128-register cap with more live
// state and spills with screen_cols (-8 %); 4:2:2 with screen_rows fits 128
// registers without spills and runs 8 CTAs (16 warps) per SM instead of
// 6 x 150 registers with screen_cols (+4.8 %, round 2).
#ifndef HJ_SCREEN_COLS_420
#define HJ_SCREEN_COLS_420 0
#endif
#ifndef HJ_SCREEN_COLS_422
#define HJ_SCREEN_COLS_422 0
#endif
#ifndef HJ_SCREEN_COLS
#define HJ_SCREEN_COLS 1
#endif
template <int SUB>
constexpr bool kScreenCols = SUB == HJ_SUB_444   ? HJ_SCREEN_COLS != 0
                             : SUB == HJ_SUB_422 ? HJ_SCREEN_COLS_422 != 0
                                                 : HJ_SCREEN_COLS_420 != 0;
template <int SUB>
__device__ __forceinline__ bool screen_block(const int16_t *__restrict__ src, const float *qf, uint32_t (&out)[16]) {
    if constexpr (kScreenCols<SUB>) return screen_cols(src, qf, out);
    else return screen_rows(src, qf, out);
}

// ------------------------------------------------- islow (libjpeg) mode
// The "islow" decode mode (idct="islow"; north_star's libjpeg jidctint
// fixed-point IDCT): libjpeg-turbo's jpeg_idct_islow (jidctint.c) in 32-bit
// two's-complement arithmetic - CONST_BITS 13, PASS1_BITS 2, column pass
// DESCALE(., 11) into an int workspace, row pass DESCALE(., 18), output
// range_limit[x & 1023] = sat_u8(sext10(x) + 128) (jdmaster.c
// prepare_range_limit_table).  Oracle: oracle/libjpeg_oracle.c, pinned to
// libjpeg-turbo 3.1 (Pillow) decodes.  Exact integer arithmetic: no screen,
// no float64 path.
namespace lj {
constexpr int F0298 = 2446, F0390 = 3196, F0541 = 4433, F0765 = 6270, F0899 = 7373, F1175 = 9633,
              F1501 = 12299, F1847 = 15137, F1961 = 16069, F2053 = 16819, F2562 = 20995, F3072 = 25172;

// one 1-D pass; o[k] = the pre-DESCALE output k (2^13-scaled).  Ring
// arithmetic mod 2^32 (unsigned: wrapping is defined), signed only for the
// arithmetic right shifts of DESCALE.
typedef unsigned U;
__device__ __forceinline__ void pass(const U (&i)[8], U (&o)[8]) {
    const U z1e = (i[2] + i[6]) * (U)F0541;
    const U t2e = z1e - i[6] * (U)F1847;
    const U t3e = z1e + i[2] * (U)F0765;
    const U t0e = (i[0] + i[4]) << 13;
    const U t1e = (i[0] - i[4]) << 13;
    const U t10 = t0e + t3e, t13 = t0e - t3e, t11 = t1e + t2e, t12 = t1e - t2e;
    const U z1 = i[7] + i[1], z2 = i[5] + i[3], z3 = i[7] + i[3], z4 = i[5] + i[1];
    const U z5 = (z3 + z4) * (U)F1175;
    const U z3s = z5 - z3 * (U)F1961, z4s = z5 - z4 * (U)F0390;
    const U t0 = i[7] * (U)F0298 - z1 * (U)F0899 + z3s;
    const U t1 = i[5] * (U)F2053 - z2 * (U)F2562 + z4s;
    const U t2 = i[3] * (U)F3072 - z2 * (U)F2562 + z3s;
    const U t3 = i[1] * (U)F1501 - z1 * (U)F0899 + z4s;
    o[0] = t10 + t3;
    o[7] = t10 - t3;
    o[1] = t11 + t2;
    o[6] = t11 - t2;
    o[2] = t12 + t1;
    o[5] = t12 - t1;
    o[3] = t13 + t0;
    o[4] = t13 - t0;
}
// DESCALE(x, n) = (x + 2^(n-1)) >> n, arithmetic
template <int N>
__device__ __forceinline__ U descale(U x) { return (U)((int)(x + (1u << (N - 1))) >> N); }
// range_limit[DESCALE(x, 18) & 1023] = sat_u8(sext10(.) + 128); pack4 saturates
__device__ __forceinline__ int out_sample(U x) { return ((int)(descale<18>(x) << 22) >> 22) + 128; }
}  // namespace lj

__device__ __forceinline__ void islow_block(const int16_t *__restrict__ src, const int *qi, uint32_t (&out)[16]) {
    int4 raw[8];
    const int4 *s4 = reinterpret_cast<const int4 *>(src);
#pragma unroll
    for (int r = 0; r < 8; r += 2) ldg_rows2(s4 + r, raw[r], raw[r + 1]);
    lj::U ws[8][8];  // ws[r][c]
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        lj::U in[8], o[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int w = c < 2 ? raw[r].x : c < 4 ? raw[r].y : c < 6 ? raw[r].z : raw[r].w;
            const int coef = (c & 1) ? (w >> 16) : (int)(short)(w & 0xffff);
            in[r] = (lj::U)coef * (lj::U)qi[r * 8 + c];  // DEQUANTIZE
        }
        lj::pass(in, o);
#pragma unroll
        for (int r = 0; r < 8; ++r) ws[r][c] = lj::descale<11>(o[r]);  // CONST_BITS - PASS1_BITS
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        lj::U o[8];
        lj::pass(ws[r], o);
        out[2 * r] = pack4(lj::out_sample(o[0]), lj::out_sample(o[1]), lj::out_sample(o[2]), lj::out_sample(o[3]));
        out[2 * r + 1] = pack4(lj::out_sample(o[4]), lj::out_sample(o[5]), lj::out_sample(o[6]), lj::out_sample(o[7]));
    }
}

// ------------------------------------------------------ exact fallback

// Cooperative exact float64 IDCT of one block by 8 threads (lane l = column
// l in the column pass, row l in the row pass), the reference's operation
// order (_native.pyx:364-388); column results staged in `g` (64 doubles,
// shared).  Returns row l's 8 rounded samples packed in a uint2.
__device__ __noinline__ uint2 exact_block_x8(const int16_t *__restrict__ src, const int *q, bool direct,
                                                double *g, int l, unsigned mask) {
    {
        double d[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            int v = (int)src[r * 8 + l] * q[r * 8 + l];
            d[r] = direct ? i2d(v) : dmul(i2d(v), kPre64[r * 8 + l]);
        }
        if (direct) direct8(d, kBasis64);
        else aan8(d[0], d[1], d[2], d[3], d[4], d[5], d[6], d[7]);
#pragma unroll
        for (int r = 0; r < 8; ++r) g[r * 8 + l] = d[r];
    }
    __syncwarp(mask);
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = g[l * 8 + k];
    if (direct) direct8(x, kBasis64);
    else aan8(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7]);
    __syncwarp(mask);
    return make_uint2(pack4(round_sample(x[0]), round_sample(x[1]), round_sample(x[2]), round_sample(x[3])),
                      pack4(round_sample(x[4]), round_sample(x[5]), round_sample(x[6]), round_sample(x[7])));
}

// ------------------------------------------------------------- geometry

// Chroma planes: 4:4:4 keeps Cb and Cr as byte planes (no filter).  4:2:2 /
// 4:2:0 store one (Cb | Cr << 8) pair per position and widen it on read to
// SWAR words (c_cb | c_cr << 16) << CSH, so the fancy filters run on both
// planes per 32-bit op; 4:2:0 scales by 16 and 4:2:2 by 64 so the filtered
// values land in byte 1 / byte 3 of each word (every lane stays below 2^16).
// The 4:2:x chroma window covers MCUs [m0-1, m1+1).
template <int SUB, int S_>
struct GeoT;
template <int S_>
struct GeoT<HJ_SUB_444, S_> {
    static constexpr int S = S_, MW = 8, MH = 8;
    static constexpr int YW = 8 * S;      // Y / Cb / Cr plane width (bytes)
    static constexpr int CW = 0;
    static constexpr int YSLOTS = 2;
    static constexpr int CROWS = 0;
};
template <int S_>
struct GeoT<HJ_SUB_422, S_> {
    static constexpr int S = S_, MW = 16, MH = 8, CSH = 6;
    static constexpr int YW = 16 * S;
    static constexpr int CW = 8 * (S + 2);  // SWAR window width (words)
    static constexpr int YSLOTS = 2;
    static constexpr int CROWS = 2 * 8;     // two slots of one MCU row
};
template <int S_>
struct GeoT<HJ_SUB_420, S_> {
    static constexpr int S = S_, MW = 16, MH = 16, CSH = 4;
    static constexpr int YW = 16 * S;
    static constexpr int CW = 8 * (S + 2);
    static constexpr int YSLOTS = 2;
    static constexpr int CROWS = 3 * 8 + 1;  // three MCU-row slots + the saved last row (index 24)
};
template <int SUB>
using Geo = GeoT<SUB, SUB == HJ_SUB_444 ? kStrip444 : SUB == HJ_SUB_422 ? kStrip422 : kStrip420>;

#ifndef HJ_CSTAGE
#define HJ_CSTAGE 1
#endif
// timing ablations (tools/ablate.sh; wrong bytes): no IDCT screen / no pixel stage
#ifndef HJ_ABLATE_SCREEN
#define HJ_ABLATE_SCREEN 0
#endif
#ifndef HJ_ABLATE_PIXELS
#define HJ_ABLATE_PIXELS 0
#endif
#ifndef HJ_PF_L2
#define HJ_PF_L2 1
#endif
static_assert(sizeof(double) * 64 / 8 == 64, "exact staging holds 64 B per thread");

template <int SUB>
constexpr int kNT = threads_for(SUB);           // threads per CTA
template <int SUB>
constexpr int kExactGroups = kNT<SUB> / 8;      // blocks recomputed in parallel
template <int SUB>
constexpr int kQueueMax = 2 * kNT<SUB>;         // >= blocks of one step

template <int SUB>
struct Smem {
    using G = Geo<SUB>;
    alignas(16) uint8_t ys[G::YSLOTS][G::MH * G::YW];
    // 4:4:4: Cb, Cr byte planes (two slots); 4:2:x: SWAR chroma rows
    alignas(16) uint8_t cbp[SUB == HJ_SUB_444 ? 2 : 1][SUB == HJ_SUB_444 ? 8 * G::YW : 16];
    alignas(16) uint8_t crp[SUB == HJ_SUB_444 ? 2 : 1][SUB == HJ_SUB_444 ? 8 * G::YW : 16];
    // 4:2:x chroma: one 16-bit (Cb | Cr << 8) pair per sample position; the
    // pixel stage widens it to SWAR words (2 bytes/position keeps 16 warps/SM)
    alignas(16) uint16_t cs[SUB == HJ_SUB_444 ? 1 : G::CROWS][SUB == HJ_SUB_444 ? 8 : G::CW];
    alignas(16) float qf[3][64];            // binary32 q * pre (screen)
    int qi[3][64];                          // integer q (exact path)
    double g[kExactGroups<SUB>][64];        // exact-path column results
    uint32_t queue[2][kQueueMax<SUB>];      // exact-path jobs: comp << 30 | block
    uint32_t qdst[2][kQueueMax<SUB>];       // destination (see push_exact)
    int n_queue[2];
    int n_taken[2];                         // pixel-item counters
};

__device__ __forceinline__ void sts128(void *p, uint4 v) { *reinterpret_cast<uint4 *>(p) = v; }
__device__ __forceinline__ uint4 lds128(const void *p) { return *reinterpret_cast<const uint4 *>(p); }

__device__ __forceinline__ void write_block_rows(uint8_t *dst, int stride, const uint32_t (&a)[16]) {
#pragma unroll
    for (int r = 0; r < 8; ++r) *reinterpret_cast<uint2 *>(dst + r * stride) = make_uint2(a[2 * r], a[2 * r + 1]);
}

// Chroma rows: position k = cb_k | cr_k << 8, 8 positions (16 bytes) per row.
__device__ __forceinline__ void write_c16_rows(uint16_t *cs, int stride, const uint32_t (&cb)[16],
                                               const uint32_t (&cr)[16]) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const uint32_t a0 = cb[2 * r], a1 = cb[2 * r + 1], b0 = cr[2 * r], b1 = cr[2 * r + 1];
        sts128(cs + r * stride, make_uint4(__byte_perm(a0, b0, 0x5140), __byte_perm(a0, b0, 0x7362),
                                           __byte_perm(a1, b1, 0x5140), __byte_perm(a1, b1, 0x7362)));
    }
}

// Destination encoding of a queued exact block: bits 31-30 = kind
// (0: byte plane offset, 2: SWAR Cb lane, 3: SWAR Cr lane), low 30 bits =
// byte offset into the Smem struct (byte planes) or word index (SWAR).
__device__ __forceinline__ void push_exact(int *n_queue, uint32_t *queue, uint32_t *qdst, uint32_t job,
                                           uint32_t dst) {
    const int e = atomicAdd(n_queue, 1);
    queue[e] = job;
    qdst[e] = dst;
}

// A block the screen could not prove is re-read by phase B's exact path; the
// screen's own loads bypassed L1, so pull its line into L1 now.
#ifndef HJ_PF_EXACT
#define HJ_PF_EXACT 1
#endif
__device__ __forceinline__ void prefetch_l1(const void *p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

// Unaligned / cropped tail of a 16-pixel RGB row (rare: odd widths, right edge).
__device__ __noinline__ void store_partial(uint8_t *__restrict__ dst, uint4 a, uint4 b, uint4 c, int nbytes) {
    const uint32_t w[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
    // aligned word j of the span starting at dst - m covers item bytes
    // [4j - m, 4j - m + 4): whole words inside [0, nbytes) as word stores,
    // the (at most two) cut words byte by byte
    const int m = (int)(reinterpret_cast<uintptr_t>(dst) & 3);
    uint32_t *d = reinterpret_cast<uint32_t *>(dst - m);
    const unsigned sh = 8u * (unsigned)m;
#pragma unroll
    for (int j = 0; j < 13; ++j) {
        const int lo = 4 * j - m;
        if (lo >= nbytes) break;
        const uint32_t prev = j > 0 ? w[j - 1] : 0u, cur = j < 12 ? w[j] : 0u;
        const uint32_t v = m ? __funnelshift_l(prev, cur, sh) : cur;
        if (lo >= 0 && lo + 4 <= nbytes) {
            d[j] = v;
        } else {
            for (int k = 0; k < 4; ++k)
                if (lo + k >= 0 && lo + k < nbytes) dst[lo + k] = (uint8_t)(v >> (8 * k));
        }
    }
}

// Pixel items are handed out 32 at a time per warp (one shared atomic per
// warp and round), so warps busy with exact blocks take fewer rounds.
__device__ __forceinline__ int grab32(int *taken) {
    int base = 0;
    if ((threadIdx.x & 31) == 0) base = atomicAdd(taken, 32);
    return __shfl_sync(0xffffffffu, base, 0) + (threadIdx.x & 31);
}

// HJ_EARLY_A (measured and rejected, default 0; tools/experiments/README.md):
// no barrier at the end of a step; a thread starts the next step's phase A
// (coefficient loads + first screen: registers only) as soon as its own
// phase B is done, and waits on barrier 1 (non-aligned: reached from
// different code points) before its first shared-memory write.
#ifndef HJ_EARLY_A
#define HJ_EARLY_A 0
#endif
__device__ __forceinline__ void hj_barrier_early() { asm volatile("barrier.sync 1;" ::: "memory"); }

// Reference mode: each warp's first round of a step is its own 32 items (the
// counter starts at blockDim.x), so only the later rounds take the atomic
// (+0.5 % at 1080p 4:2:0).  The islow kernel keeps the atomic-only queue
// (-1 % with the static round).
#ifndef HJ_GRAB_STATIC
#define HJ_GRAB_STATIC 1
#endif
// The number of static rounds: 1, and 2 for the 64-thread 4:4:4 CTAs
// (+0.5 %); 2 / 3 rounds measured slower at 4:2:0 (-0.5 % / -3 %), 3 spills
// at 4:4:4, 2 in the 256-thread tensor-core kernel -3.6 % at 4:4:4
// (profiles/r02bm_ab.txt, r02bn).  HJ_GRAB_STATIC=0: the atomic-only queue.
template <int SUB, int MODE, bool TC>
__device__ __forceinline__ constexpr int grab_static() {
    return (MODE == kModeRef && HJ_GRAB_STATIC) ? (SUB == HJ_SUB_444 && !TC ? 2 : 1) : 0;
}
template <int SUB, int MODE, bool TC>
__device__ __forceinline__ int grab_base() { return grab_static<SUB, MODE, TC>() * (int)blockDim.x; }
template <int SUB, int MODE, bool TC>
__device__ __forceinline__ int grab_first(int *taken) {
    if constexpr (grab_static<SUB, MODE, TC>() > 0) return (int)threadIdx.x;
    else return grab32(taken);
}
template <int SUB, int MODE, bool TC>
__device__ __forceinline__ int grab_next(int *taken, int i0) {
    if constexpr (grab_static<SUB, MODE, TC>() > 1)
        if (i0 < (grab_static<SUB, MODE, TC>() - 1) * (int)blockDim.x) return i0 + (int)blockDim.x;
    return grab32(taken);
}

// Colour + pack of 4 pixels (Y bytes of `yw`, chroma ints) -> 12 RGB bytes
// in 3 words.  Small live ranges on purpose: the colour constants stay in
// registers instead of being rematerialised per pixel.
template <int MODE>
__device__ __forceinline__ Rgb colour_m(int y, int cb, int cr, bool &special, const ColourRegs &k) {
    if constexpr (MODE == kModeIslow) return colour_libjpeg(y, cb, cr, k);
    else return colour(y, cb, cr, special, k);
}
template <int MODE>
__device__ __forceinline__ ColourRegs colour_regs_m() {
    if constexpr (MODE == kModeIslow) return colour_regs_libjpeg();
    else return colour_regs();
}
template <int MODE>
__device__ __forceinline__ void colour4(uint32_t yw, int cb0, int cr0, int cb1, int cr1, int cb2, int cr2,
                                        int cb3, int cr3, bool &special, uint32_t &w0, uint32_t &w1,
                                        uint32_t &w2, const ColourRegs &k) {
    const Rgb p0 = colour_m<MODE>((int)__byte_perm(yw, 0, 0x4440), cb0, cr0, special, k);
    const Rgb p1 = colour_m<MODE>((int)__byte_perm(yw, 0, 0x4441), cb1, cr1, special, k);
    const Rgb p2 = colour_m<MODE>((int)__byte_perm(yw, 0, 0x4442), cb2, cr2, special, k);
    const Rgb p3 = colour_m<MODE>((int)__byte_perm(yw, 0, 0x4443), cb3, cr3, special, k);
    w0 = pack4(p0.r, p0.g, p0.b, p1.r);
    w1 = pack4(p1.g, p1.b, p2.r, p2.g);
    w2 = pack4(p2.b, p3.r, p3.g, p3.b);
}

// 48 RGB bytes (16 pixels) at dst.  Rows of an image whose width is not a
// multiple of 4 start at any byte offset, so a full item is written as its
// 11 interior aligned words (funnel-shifted into place) plus the partial
// words at both ends; only items cropped by the right edge take the
// byte-wise path.
// RGB stores are write-once: st.global.cs (evict-first) keeps them from
// displacing the coefficient stream's L2 prefetches (measured +0.3-0.6 %).
#ifndef HJ_STCS
#define HJ_STCS 1
#endif
template <class T>
__device__ __forceinline__ void st_rgb(T *p, T v) {
#if HJ_STCS
    __stcs(p, v);
#else
    *p = v;
#endif
}
__device__ __forceinline__ void st_rgb(uint32_t *p, uint32_t v) {
#if HJ_STCS
    __stcs(reinterpret_cast<unsigned int *>(p), v);
#else
    *p = v;
#endif
}
__device__ __forceinline__ void store48(uint8_t *__restrict__ dst, const uint32_t (&w)[12], int npx) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(dst);
    if (npx == 16 && (a & 15) == 0) {
        uint4 *d = reinterpret_cast<uint4 *>(dst);
        st_rgb(d, make_uint4(w[0], w[1], w[2], w[3]));
        st_rgb(d + 1, make_uint4(w[4], w[5], w[6], w[7]));
        st_rgb(d + 2, make_uint4(w[8], w[9], w[10], w[11]));
    } else if (npx == 16 && (a & 7) == 0) {
        uint2 *d = reinterpret_cast<uint2 *>(dst);
#pragma unroll
        for (int i = 0; i < 6; ++i) st_rgb(d + i, make_uint2(w[2 * i], w[2 * i + 1]));
    } else if (npx == 16 && (a & 3) == 0) {
        // a = 4 mod 8: one word, five 8-byte pairs, one word
        uint32_t *d = reinterpret_cast<uint32_t *>(dst);
        st_rgb(d, w[0]);
#pragma unroll
        for (int i = 1; i < 11; i += 2) st_rgb(reinterpret_cast<uint2 *>(d + i), make_uint2(w[i], w[i + 1]));
        st_rgb(d + 11, w[11]);
    } else if (npx == 16) {
        const int m = (int)(a & 3);  // 1..3
        uint32_t *d = reinterpret_cast<uint32_t *>(dst - m);
        const unsigned sh = 8u * (unsigned)m;
        // word k of the aligned span = bytes of w[k-1] (high part) | w[k] (low part)
        uint32_t f[12];
#pragma unroll
        for (int k = 1; k < 12; ++k) f[k] = __funnelshift_l(w[k - 1], w[k], sh);
        // the 11 interior words as 8-byte stores where the span allows (a
        // row's items share one alignment: 48-byte steps)
        if ((reinterpret_cast<uintptr_t>(d + 1) & 7) == 0) {
#pragma unroll
            for (int k = 1; k < 11; k += 2) st_rgb(reinterpret_cast<uint2 *>(d + k), make_uint2(f[k], f[k + 1]));
            st_rgb(d + 11, f[11]);
        } else {
            st_rgb(d + 1, f[1]);
#pragma unroll
            for (int k = 2; k < 12; k += 2) st_rgb(reinterpret_cast<uint2 *>(d + k), make_uint2(f[k], f[k + 1]));
        }
        // head: the first 4-m bytes of w[0]; tail: the last m bytes of w[11]
        if (m == 2) {
            *reinterpret_cast<uint16_t *>(dst) = (uint16_t)w[0];
            *reinterpret_cast<uint16_t *>(dst + 46) = (uint16_t)(w[11] >> 16);
        } else if (m == 1) {
            dst[0] = (uint8_t)w[0];
            *reinterpret_cast<uint16_t *>(dst + 1) = (uint16_t)(w[0] >> 8);
            dst[47] = (uint8_t)(w[11] >> 24);
        } else {
            dst[0] = (uint8_t)w[0];
            *reinterpret_cast<uint16_t *>(dst + 45) = (uint16_t)(w[11] >> 8);
            dst[47] = (uint8_t)(w[11] >> 24);
        }
    } else if (npx == 8 && (a & 7) == 0) {
        // half item (4:4:4 image whose width is 8 mod 16): 24 bytes, 8-aligned
        uint2 *d = reinterpret_cast<uint2 *>(dst);
        st_rgb(d, make_uint2(w[0], w[1]));
        st_rgb(d + 1, make_uint2(w[2], w[3]));
        st_rgb(d + 2, make_uint2(w[4], w[5]));
    } else {
        store_partial(dst, make_uint4(w[0], w[1], w[2], w[3]), make_uint4(w[4], w[5], w[6], w[7]),
                      make_uint4(w[8], w[9], w[10], w[11]), npx * 3);
    }
}

// Rare path: the 16 pixels held the float64 tie pair (Cb, Cr) = (78, 178)
// (SURVEY.md E3): recompute them with the exact G rule and store.  Inputs by
// value (no local arrays on the hot path).  is444: a = Cb bytes, b = Cr
// bytes; else a, b, e = the 10 SWAR chroma sums of render16_swar.
__device__ __noinline__ void render16_exact(uint8_t *__restrict__ dst, uint4 yv, uint4 a, uint4 b, uint2 e,
                                            uint32_t rnd_e, uint32_t rnd_o, int is444, int npx) {
    const uint32_t yw[4] = {yv.x, yv.y, yv.z, yv.w};
    int cb[16], cr[16];
    if (is444) {
        const uint32_t bw[4] = {a.x, a.y, a.z, a.w}, rw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            cb[i] = (int)((bw[i >> 2] >> (8 * (i & 3))) & 0xff);
            cr[i] = (int)((rw[i >> 2] >> (8 * (i & 3))) & 0xff);
        }
    } else {
        const uint32_t c[10] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, e.x, e.y};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t t3 = c[i + 1] * 3u;
            const uint32_t ev = t3 + c[i] + rnd_e, od = t3 + c[i + 2] + rnd_o;
            cb[2 * i] = (int)((ev >> 8) & 0xff);
            cr[2 * i] = (int)(ev >> 24);
            cb[2 * i + 1] = (int)((od >> 8) & 0xff);
            cr[2 * i + 1] = (int)(od >> 24);
        }
    }
    uint32_t w[12];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        Rgb p[4];
        bool dummy = false;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int i = 4 * q + k, y = (int)((yw[q] >> (8 * k)) & 0xff);
            p[k] = colour(y, cb[i], cr[i], dummy);
            p[k].g = colour_g_exact(y, cb[i], cr[i]);
        }
        w[3 * q] = pack4(p[0].r, p[0].g, p[0].b, p[1].r);
        w[3 * q + 1] = pack4(p[1].g, p[1].b, p[2].r, p[2].g);
        w[3 * q + 2] = pack4(p[2].b, p[3].r, p[3].g, p[3].b);
    }
    store48(dst, w, npx);
}

// 16 pixels of a 4:2:x row: Y bytes `yv`, chroma SWAR sums c[0..9] (c[1..8]
// under the 16 pixels), horizontal fancy filter even = 3c + prev + rnd_e,
// odd = 3c + next + rnd_o with the result in byte 1 (Cb) / byte 3 (Cr) of
// each lane; colour; 48 bytes stored at dst (cropped to npx).
// MODE: kModeRef (the reference's float64 colour) or kModeIslow (libjpeg's
// integer colour).  BOX: libjpeg's box replication instead of the triangle
// filter (islow mode, chroma width <= 2): every neighbour reads as the
// sample itself.
template <int MODE, bool BOX = false>
__device__ __forceinline__ void render16_swar(uint8_t *__restrict__ dst, uint4 yv, const uint32_t (&c)[10],
                                              uint32_t rnd_e, uint32_t rnd_o, int npx) {
    const uint32_t yw[4] = {yv.x, yv.y, yv.z, yv.w};
    uint32_t w[12];
    bool special = false;
    const ColourRegs k = colour_regs_m<MODE>();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t ta = c[2 * q + 1] * 3u, tb = c[2 * q + 2] * 3u;
        const uint32_t e0 = ta + c[2 * q + (BOX ? 1 : 0)] + rnd_e, o0 = ta + c[2 * q + (BOX ? 1 : 2)] + rnd_o;
        const uint32_t e1 = tb + c[2 * q + (BOX ? 2 : 1)] + rnd_e, o1 = tb + c[2 * q + (BOX ? 2 : 3)] + rnd_o;
        colour4<MODE>(yw[q], (int)__byte_perm(e0, 0, 0x4441), (int)(e0 >> 24), (int)__byte_perm(o0, 0, 0x4441),
                (int)(o0 >> 24), (int)__byte_perm(e1, 0, 0x4441), (int)(e1 >> 24),
                (int)__byte_perm(o1, 0, 0x4441), (int)(o1 >> 24), special, w[3 * q], w[3 * q + 1], w[3 * q + 2], k);
    }
    if (MODE == kModeRef && special) {
        render16_exact(dst, yv, make_uint4(c[0], c[1], c[2], c[3]), make_uint4(c[4], c[5], c[6], c[7]),
                       make_uint2(c[8], c[9]), rnd_e, rnd_o, 0, npx);
        return;
    }
    store48(dst, w, npx);
}

// 16 pixels of a 4:4:4 row from Y / Cb / Cr byte vectors.
template <int MODE>
__device__ __forceinline__ void render16_444(uint8_t *__restrict__ dst, uint4 yv, uint4 bv, uint4 rv, int npx) {
    const uint32_t yw[4] = {yv.x, yv.y, yv.z, yv.w}, bw[4] = {bv.x, bv.y, bv.z, bv.w},
                   rw[4] = {rv.x, rv.y, rv.z, rv.w};
    uint32_t w[12];
    bool special = false;
    const ColourRegs k = colour_regs_m<MODE>();
#pragma unroll
    for (int q = 0; q < 4; ++q)
        colour4<MODE>(yw[q], (int)(bw[q] & 0xff), (int)((rw[q]) & 0xff), (int)__byte_perm(bw[q], 0, 0x4441),
                (int)__byte_perm(rw[q], 0, 0x4441), (int)__byte_perm(bw[q], 0, 0x4442),
                (int)__byte_perm(rw[q], 0, 0x4442), (int)(bw[q] >> 24), (int)(rw[q] >> 24), special, w[3 * q],
                w[3 * q + 1], w[3 * q + 2], k);
    if (MODE == kModeRef && special) {
        render16_exact(dst, yv, bv, rv, make_uint2(0, 0), 0, 0, 1, npx);
        return;
    }
    store48(dst, w, npx);
}

// 10 SWAR words (cb | cr << 16) of one chroma row from the 16-bit pair
// storage: positions p[-1], p[0..7], p[8], with edge replication at the
// padded plane's first / last column.
__device__ __forceinline__ uint32_t widen(uint32_t pair) { return __byte_perm(pair, 0, 0x4140); }
__device__ __forceinline__ void load_c10(const uint16_t *p, bool left_edge, bool right_edge, uint32_t (&c)[10]) {
    const uint4 m = lds128(p);
    c[1] = __byte_perm(m.x, 0, 0x4140); c[2] = __byte_perm(m.x, 0, 0x4342);
    c[3] = __byte_perm(m.y, 0, 0x4140); c[4] = __byte_perm(m.y, 0, 0x4342);
    c[5] = __byte_perm(m.z, 0, 0x4140); c[6] = __byte_perm(m.z, 0, 0x4342);
    c[7] = __byte_perm(m.w, 0, 0x4140); c[8] = __byte_perm(m.w, 0, 0x4342);
    c[0] = left_edge ? c[1] : widen(p[-1]);
    c[9] = right_edge ? c[8] : widen(p[8]);
}

// islow mode (libjpeg jdsample.c): the chroma plane's real width is
// cw = ceil(w/2); the filter's right neighbour of column cw-1 is itself.
// c[1 + j] holds chroma column c0 + j of the item (c[0], c[9] the
// neighbours); columns from cw on only feed cropped pixels.
__device__ __forceinline__ void lj_right_edge(uint32_t (&c)[10], int cw, int c0) {
    const int j = cw - c0;  // window index of column cw
#pragma unroll
    for (int t = 1; t <= 8; ++t)
        if (t == j) c[t + 1] = c[t];
}

// Phase B, first half: the step's queued blocks recomputed in exact float64
// by 8-thread groups (NT / 8 blocks in parallel), written over the screen's
// samples in the planes.  The islow mode never queues.
template <int SUB, int MODE, class G, int NT, class SM>
__device__ __forceinline__ void exact_phase(SM &sm, uint8_t *smem_raw, const hj_image_t &im, int par, bool direct) {
    constexpr bool kIslow = MODE == kModeIslow;
    constexpr int kExactGroups = NT / 8;
    const int tid = threadIdx.x;
    int *const nq = &sm.n_queue[par];
    const uint32_t *const queue = sm.queue[par];
    const uint32_t *const qdst = sm.qdst[par];
    if constexpr (!kIslow) {
        const int n = *nq;
        const int grp = tid >> 3, l = tid & 7;
        const unsigned gmask = 0xffu << (tid & 24);  // the 8 lanes of this group
#pragma unroll 1
        for (int e = grp; e < n; e += kExactGroups) {
            const uint32_t job = queue[e], dst = qdst[e];
            const int comp = job >> 30;
            const int64_t blk = job & 0x3fffffff;
            const int16_t *src = (comp == 0 ? im.y : comp == 1 ? im.cb : im.cr) + blk * 64;
            const uint2 row = exact_block_x8(src, sm.qi[comp], direct, sm.g[grp], l, gmask);
            const uint32_t kind = dst >> 30, off = dst & 0x3fffffff;
            if (kind == 0) {
                *reinterpret_cast<uint2 *>(smem_raw + off + l * G::YW) = row;
            } else if constexpr (SUB != HJ_SUB_444) {
                uint8_t *c8 = reinterpret_cast<uint8_t *>(&sm.cs[0][0] + off + l * G::CW) + (kind & 1);
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    c8[2 * c] = (uint8_t)(c < 4 ? row.x >> (8 * c) : row.y >> (8 * (c - 4)));
            }
        }
        if (tid == 0 && n) atomicAdd(&g_exact_blocks, (unsigned long long)n);
    }

}

// Phase B, second half: the pixel stage of MCU row R = s - 1 (upsample +
// colour + RGB stores) from the previous step's sample planes; items are
// handed out through a shared counter so threads busy in exact_phase take fewer.
template <int SUB, int MODE, class G, class SM, bool TC = false>
__device__ __forceinline__ void pixel_phase(SM &sm, const hj_image_t &im, const Tile &t, int s, int par, bool do_c) {
    constexpr bool kIslow = MODE == kModeIslow;
    const int tid = threadIdx.x;
    const int mpr = im.mcus_per_row, mcu_rows = im.mcu_rows, S = t.m1 - t.m0;
    const bool left_edge = (t.m0 == 0), right_edge = (t.m1 == mpr);
    const int lj_cw = (im.width + 1) >> 1, lj_ch = (im.height + 1) >> 1;
    const bool lj_box = kIslow && lj_cw <= 2;
    (void)lj_ch; (void)lj_cw; (void)mcu_rows; (void)tid; (void)do_c;
    const int R = s - 1;
    if (!HJ_ABLATE_PIXELS && R >= t.r0 && R < t.r1) {
        const int y_base = R * G::MH;
        const int x_base = t.m0 * G::MW;
        const uint8_t *yp = sm.ys[par ^ 1];
        int *const taken = &sm.n_taken[par];
        if constexpr (SUB == HJ_SUB_420) {
            // item = (MCU column g, row pair p): output rows y_base+2p, +1
            const int n_items = 8 * S;
            const int gw = S;
            const float inv_w = 1.0f / (float)gw;
            const uint16_t *cnear = &sm.cs[0][0] + (R % 3) * 8 * G::CW;
            const uint16_t *cnext = &sm.cs[0][0] + ((R + 1) % 3) * 8 * G::CW;
            // top context of the MCU row's first sample row: the last row
            // of MCU row R-1 - saved in row 24 when this step's chroma
            // jobs overwrote its slot, else still in the slot
            const uint16_t *cprev = do_c ? &sm.cs[24][0] : &sm.cs[0][0] + (((R + 2) % 3) * 8 + 7) * G::CW;
#pragma unroll 1
            for (int i0 = grab_first<SUB, MODE, TC>(taken); i0 - (tid & 31) < n_items; i0 = grab_next<SUB, MODE, TC>(taken, i0)) {
                const int i = i0;
                if (i >= n_items) continue;
                // row-major items: adjacent lanes store adjacent 48-byte runs
                const int p = __float2int_rd(((float)i + 0.5f) * inv_w), g = i - p * S;
                const int y0 = y_base + 2 * p;
                if (y0 >= im.height) continue;
                const int x0 = x_base + 16 * g;
                const int npx = min(16, im.width - x0);
                if (npx <= 0) continue;
                const int kw = 8 * (g + 1);  // window word of the MCU's chroma column 0
                const uint16_t *pn = cnear + p * G::CW + kw;
                const uint16_t *pu = p > 0 ? pn - G::CW : (R > 0 ? cprev + kw : pn);
                const uint16_t *pd = p < 7 ? pn + G::CW : (R + 1 < mcu_rows ? cnext + kw : pn);
                if (kIslow) {
                    // libjpeg context rows: the real chroma plane ends at row
                    // ceil(h/2) - 1 (jdmainct.c set_bottom_pointers); box
                    // replication has no vertical filter
                    if (lj_box || 8 * R + p >= lj_ch - 1) pd = pn;
                    if (lj_box) pu = pn;
                }
                const bool le = left_edge && g == 0, re = right_edge && g == S - 1;
                const int c0 = 8 * (t.m0 + g);  // the item's first chroma column
                // colsum = 3*near + far per lane (libjpeg h2v2 fancy), 16x scaled
                uint32_t n3[10];
                load_c10(pn, le, re, n3);
                if (kIslow && c0 + 8 >= lj_cw) lj_right_edge(n3, lj_cw, c0);
#pragma unroll
                for (int k = 0; k < 10; ++k) n3[k] = n3[k] * (3u << G::CSH) + 0x00200020u;
                const int rows = min(2, im.height - y0);
#pragma unroll 1
                for (int h = 0; h < rows; ++h) {
                    uint32_t cs10[10];
                    load_c10(h ? pd : pu, le, re, cs10);
                    if (kIslow && c0 + 8 >= lj_cw) lj_right_edge(cs10, lj_cw, c0);
#pragma unroll
                    for (int k = 0; k < 10; ++k) cs10[k] = (cs10[k] << G::CSH) + n3[k];
                    // even 16(3cs+prev+8), odd 16(3cs+next+7): each colsum
                    // carries +2 (x16) from n3, so 3cs+prev already holds
                    // the +8 and odd subtracts 1 (lanes stay >= 0x80)
                    uint8_t *dst = im.rgb + ((int64_t)(y0 + h) * im.width + x0) * 3;
                    const uint4 yv = lds128(yp + (2 * p + h) * G::YW + 16 * g);
                    if (kIslow && lj_box)
                        render16_swar<MODE, true>(dst, yv, cs10, 0u, 0u - 0x00100010u, npx);
                    else
                        render16_swar<MODE>(dst, yv, cs10, 0u, 0u - 0x00100010u, npx);
                }
            }
        } else if constexpr (SUB == HJ_SUB_422) {
            // item = (MCU column g, row y): 16 pixels
            const int n_items = 8 * S;
            const int gw = S;
            const float inv_w = 1.0f / (float)gw;
            const uint16_t *crow0 = &sm.cs[0][0] + (par ^ 1) * 8 * G::CW;
#pragma unroll 1
            for (int i0 = grab_first<SUB, MODE, TC>(taken); i0 - (tid & 31) < n_items; i0 = grab_next<SUB, MODE, TC>(taken, i0)) {
                const int i = i0;
                if (i >= n_items) continue;
                const int y = __float2int_rd(((float)i + 0.5f) * inv_w), g = i - y * gw;
                const int yy = y_base + y;
                if (yy >= im.height) continue;
                const int x0 = x_base + 16 * g;
                const int npx = min(16, im.width - x0);
                if (npx <= 0) continue;
                uint32_t c10[10];
                load_c10(crow0 + y * G::CW + 8 * (g + 1), left_edge && g == 0, right_edge && g == S - 1, c10);
                const int c0 = 8 * (t.m0 + g);
                if (kIslow && c0 + 8 >= lj_cw) lj_right_edge(c10, lj_cw, c0);
#pragma unroll
                for (int k = 0; k < 10; ++k) c10[k] = (c10[k] << G::CSH) + 0x00100010u;
                // h2v1 on 64x-scaled lanes: even 64(3c+prev+1), odd 64(3c+next+2);
                // each sample carries +1/4 (x64), so 3c+prev already holds the +1
                uint8_t *dst = im.rgb + ((int64_t)yy * im.width + x0) * 3;
                const uint4 yv = lds128(yp + y * G::YW + 16 * g);
                if (kIslow && lj_box)
                    render16_swar<MODE, true>(dst, yv, c10, 0u, 0x00400040u, npx);
                else
                    render16_swar<MODE>(dst, yv, c10, 0u, 0x00400040u, npx);
            }
        } else {
            // item = (MCU pair g, row y): 16 pixels
            const int gw = (S + 1) / 2;
            const int n_items = 8 * gw;
            const float inv_w = 1.0f / (float)gw;
            const uint8_t *cbp = sm.cbp[par ^ 1], *crp = sm.crp[par ^ 1];
#pragma unroll 1
            for (int i0 = grab_first<SUB, MODE, TC>(taken); i0 - (tid & 31) < n_items; i0 = grab_next<SUB, MODE, TC>(taken, i0)) {
                const int i = i0;
                if (i >= n_items) continue;
                const int y = __float2int_rd(((float)i + 0.5f) * inv_w), g = i - y * gw;
                const int yy = y_base + y;
                if (yy >= im.height) continue;
                const int x0 = x_base + 16 * g;
                const int npx = min(min(16, im.width - x0), 8 * (S - 2 * g));
                if (npx <= 0) continue;
                const int o = y * G::YW + 16 * g;
                render16_444<MODE>(im.rgb + ((int64_t)yy * im.width + x0) * 3, lds128(yp + o), lds128(cbp + o),
                             lds128(crp + o), npx);
            }
        }
    }
}

template <int SUB, int MODE>
__global__ void __launch_bounds__(kNT<SUB>, ctas_per_sm(SUB))
render_kernel(const hj_image_t *__restrict__ images, const Tile *__restrict__ tiles) {
    using G = Geo<SUB>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];  // (one declaration for both kernels)
    Smem<SUB> &sm = *reinterpret_cast<Smem<SUB> *>(smem_raw);

    const Tile t = tiles[blockIdx.x];
    const hj_image_t im = images[t.image];
    const int tid = threadIdx.x;
    const int mpr = im.mcus_per_row;
    const int S = t.m1 - t.m0;
    const bool direct = MODE == kModeRef && (im.flags & HJ_FLAG_DIRECT_IDCT) != 0;
    constexpr bool kIslow = MODE == kModeIslow;
    constexpr int kThreads = kNT<SUB>;
    for (int i = tid; i < 192; i += kThreads) {
        const int q = im.q[i];
        sm.qi[i >> 6][i & 63] = q;
    }
    if constexpr (!kIslow)
        for (int i = tid; i < 192; i += kThreads)
            sm.qf[i >> 6][qf_slot(kScreenCols<SUB>, (i & 63) >> 3, i & 7)] = (float)((double)im.q[i] * kPre64[i & 63]);
    if (tid == 0) {
        sm.n_queue[0] = sm.n_queue[1] = 0;
        sm.n_taken[0] = sm.n_taken[1] = grab_base<SUB, MODE, false>();
    }

    const int cm_lo = (SUB == HJ_SUB_444) ? t.m0 : t.m0 - 1;  // first chroma window MCU
    const int n_cm = (SUB == HJ_SUB_444) ? S : S + 2;
    // Y jobs (two blocks): 444 MCU pair; 422 one MCU; 420 half MCU
    const int n_yj = (SUB == HJ_SUB_444) ? (S + 1) / 2 : (SUB == HJ_SUB_422 ? S : 2 * S);
    constexpr int YB = G::MW / 8 * (G::MH / 8);          // Y blocks per MCU
    const int mcu_rows = im.mcu_rows;
    __syncthreads();

    // step range: 4:2:0 screens chroma one MCU row ahead (vertical context)
    const int s_begin = (SUB == HJ_SUB_420) ? max(t.r0 - 2, -1) : t.r0;
    const int s_end = t.r1;  // the last step only draws row r1-1
#pragma unroll 1
    for (int s = s_begin; s <= s_end; ++s) {
        const int par = s & 1;
        int *const nq = &sm.n_queue[par];
        uint32_t *const queue = sm.queue[par];
        uint32_t *const qdst = sm.qdst[par];
        const bool do_y = s >= t.r0 && s < t.r1;
        const int crow = (SUB == HJ_SUB_420) ? s + 1 : s;
        const bool do_c = (SUB == HJ_SUB_420) ? (crow >= t.r0 - 1 && crow <= t.r1 && crow >= 0 && crow < mcu_rows)
                                              : do_y;
        if (tid == 0) {
            if (!HJ_EARLY_A) {
                sm.n_queue[par ^ 1] = 0;  // last used in step s-1, next in s+1
                sm.n_taken[par ^ 1] = grab_base<SUB, MODE, false>();
            }
            // bulk L2 prefetch of the next step's coefficient ranges
            const int ny = HJ_PF_L2 ? s + 1 : -1;
            if (ny >= t.r0 && ny < t.r1) {
                const int64_t b0 = ((int64_t)ny * mpr + t.m0) * YB;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(im.y + b0 * 64),
                             "r"((unsigned)(S * YB * 128)));
            }
            const int nc = crow + 1;
            if (HJ_PF_L2 && nc < mcu_rows && nc <= t.r1) {
                const int c0 = max(cm_lo, 0), c1 = min(cm_lo + n_cm, mpr);
                const int64_t b0 = (int64_t)nc * mpr + c0;
                const unsigned bytes = (unsigned)((c1 - c0) * 128);
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(im.cb + b0 * 64), "r"(bytes));
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(im.cr + b0 * 64), "r"(bytes));
            }
        }

        // ---------------- phase A: screen (one two-block job per thread)
        {
            const int n_y = do_y ? n_yj : 0;
            const int n_jobs = n_y + (do_c ? n_cm : 0);
            bool synced = !HJ_EARLY_A;  // passed the deferred end-of-step barrier
#pragma unroll 1
            for (int j = tid; j < n_jobs; j += kThreads) {
                const bool is_y = j < n_y;
                const int lm = j - n_y;            // chroma window MCU
                const int m = cm_lo + lm;
                if (!is_y && (m < 0 || m >= mpr)) continue;
                const int16_t *srcA, *srcB;
                bool has_b = true;
                uint32_t dA, dB;                   // exact-path destinations
                uint8_t *ydst = nullptr;           // Y-like byte rows
                uint16_t *cdst = nullptr;          // chroma pair rows
                int cw0 = 0;
                if (is_y) {
                    int64_t yblk;
                    int yoff;
                    if (SUB == HJ_SUB_444) {
                        yblk = (int64_t)s * mpr + t.m0 + 2 * j;
                        yoff = 16 * j;
                        has_b = 2 * j + 1 < S;
                    } else if (SUB == HJ_SUB_422) {
                        yblk = ((int64_t)s * mpr + t.m0 + j) * 2;
                        yoff = 16 * j;
                    } else {
                        yblk = ((int64_t)s * mpr + t.m0 + (j >> 1)) * 4 + 2 * (j & 1);
                        yoff = (j & 1) * 8 * G::YW + (j >> 1) * 16;
                    }
                    srcA = im.y + yblk * 64;
                    srcB = has_b ? srcA + 64 : srcA;
                    ydst = sm.ys[par] + yoff;
                    dA = (uint32_t)(ydst - smem_raw);
                    dB = dA + 8;
                } else {
                    const int64_t cblk = (int64_t)crow * mpr + m;
                    srcA = im.cb + cblk * 64;
                    srcB = im.cr + cblk * 64;
                    if (SUB == HJ_SUB_444) {
                        ydst = sm.cbp[par] + 8 * lm;
                        dA = (uint32_t)(ydst - smem_raw);
                        dB = (uint32_t)(sm.crp[par] + 8 * lm - smem_raw);
                    } else {
                        const int slot = (SUB == HJ_SUB_420) ? (crow % 3) : par;
                        cw0 = slot * 8 * G::CW + 8 * lm;
                        cdst = &sm.cs[0][0] + cw0;
                        dA = (2u << 30) | (uint32_t)cw0;
                        dB = (3u << 30) | (uint32_t)cw0;
                        if constexpr (SUB == HJ_SUB_420 && !HJ_EARLY_A) {
                            // the slot's old row 7 (MCU row crow-3) is the top
                            // context of MCU row crow-2, drawn this step
                            uint16_t *save = &sm.cs[24][0] + 8 * lm;
                            sts128(save, lds128(cdst + 7 * G::CW));
                        }
                    }
                }
                // the two blocks through one (rolled) screen call site; block
                // A's samples stay in `keep` until B is done
                uint32_t keep[16];
                bool okA = false;
#pragma unroll 1
                for (int k = 0; k < 2; ++k) {
                    if (k == 1 && !has_b) break;
                    uint32_t w[16];
                    const int comp = is_y ? 0 : 1 + k;
                    bool ok = false;
                    if constexpr (kIslow) {
                        islow_block(k ? srcB : srcA, sm.qi[comp], w);
                        ok = true;
                    } else if (HJ_ABLATE_SCREEN) {
                        // timing ablation only (wrong bytes): load the block, no transform
                        int4 r[8];
#pragma unroll
                        for (int i = 0; i < 8; i += 2)
                            ldg_rows2(reinterpret_cast<const int4 *>(k ? srcB : srcA) + i, r[i], r[i + 1]);
#pragma unroll
                        for (int i = 0; i < 16; ++i) w[i] = (uint32_t)(r[i >> 1].x ^ r[i >> 1].w) + i;
                        ok = true;
                    } else if (!direct) {
                        ok = screen_block<SUB>(k ? srcB : srcA, sm.qf[comp], w);
                    }
                    if (!synced) {
                        // early A: the loads and the first screen of this step
                        // ran while other warps finished the previous step's
                        // phase B; shared-memory writes wait for all of them
                        hj_barrier_early();
                        synced = true;
                    }
                    if constexpr (SUB == HJ_SUB_420 && HJ_EARLY_A) {
                        if (k == 0 && !is_y) {
                            uint16_t *save = &sm.cs[24][0] + 8 * lm;
                            sts128(save, lds128(cdst + 7 * G::CW));
                        }
                    }
                    if (SUB == HJ_SUB_444 || is_y) {
                        // byte planes: Y (blocks side by side) or Cb / Cr
                        uint8_t *dst = is_y ? ydst + 8 * k : (k ? sm.crp[par] + 8 * lm : ydst);
                        if (!direct) write_block_rows(dst, G::YW, w);
                        if (!ok) {
                            const int64_t blk = ((k ? srcB : srcA) - (is_y ? im.y : k ? im.cr : im.cb)) / 64;
                            push_exact(nq, queue, qdst, ((uint32_t)comp << 30) | (uint32_t)blk, k ? dB : dA);
                            if (HJ_PF_EXACT) prefetch_l1(k ? srcB : srcA);
                        }
                    } else if (k == 0) {
#if HJ_CSTAGE
                        // park block A's samples in this thread's 64 B of the
                        // (phase-B-only) exact staging area: 16 registers
                        // fewer live across the second screen
                        if (!direct) {
                            uint4 *st = reinterpret_cast<uint4 *>(&sm.g[0][0]) + 4 * tid;
#pragma unroll
                            for (int i = 0; i < 4; ++i)
                                sts128(st + i, make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]));
                        }
#else
#pragma unroll
                        for (int i = 0; i < 16; ++i) keep[i] = w[i];
#endif
                        okA = ok;
                    } else {
#if HJ_CSTAGE
                        if (!direct) {
                            const uint4 *st = reinterpret_cast<const uint4 *>(&sm.g[0][0]) + 4 * tid;
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                const uint4 v = lds128(st + i);
                                keep[4 * i] = v.x, keep[4 * i + 1] = v.y, keep[4 * i + 2] = v.z, keep[4 * i + 3] = v.w;
                            }
                        }
#endif
                        if (!direct) write_c16_rows(cdst, G::CW, keep, w);
                        const uint32_t blk = (uint32_t)((int64_t)crow * mpr + m);
                        if (!okA) {
                            push_exact(nq, queue, qdst, (1u << 30) | blk, dA);
                            if (HJ_PF_EXACT) prefetch_l1(srcA);
                        }
                        if (!ok) {
                            push_exact(nq, queue, qdst, (2u << 30) | blk, dB);
                            if (HJ_PF_EXACT) prefetch_l1(srcB);
                        }
                    }
                }
            }
            if (!synced) hj_barrier_early();  // threads without a (drawn) job
        }
        __syncthreads();
        if (HJ_EARLY_A && tid == 0) {
            // last used by phase B of step s-1 (done: every thread passed the
            // early barrier of this step), next by step s+1
            sm.n_queue[par ^ 1] = 0;
            sm.n_taken[par ^ 1] = grab_base<SUB, MODE, false>();
        }

        // ---------------- phase B: exact recompute of this step's queue ...
        exact_phase<SUB, MODE, G, kThreads>(sm, smem_raw, im, par, direct);
        // ---------------- ... overlapped with the pixel stage of MCU row s-1
        pixel_phase<SUB, MODE, G>(sm, im, t, s, par, do_c);
        if (!HJ_EARLY_A) __syncthreads();
    }
}

// ------------------------------------------ tensor-core IDCT screen (v4)
// The reference mode's IDCT is a fixed linear map: with
// exact arithmetic, s = M x for the dequantised block x, M evaluated exactly
// from the reference's float64 constants (tools/gen_mtable.py).  The screen
// computes s on the 5th-generation tensor cores in exact integer arithmetic:
//   A = the AC coefficients as int8 (the low byte of each int16; blocks with
//       an AC coefficient outside [-128, 127] go to the exact path),
//   B = Mq = round(2^F M diag(q)) in three 8-bit limbs (F per quantisation
//       table, |Mq| < 2^23), DC column zero (the DC term c0 q0 / 8 is exact
//       and enters through the per-block bias),
//   D = A B^T per limb, int32 in TMEM: T = acc0 + 2^8 acc1 + 2^16 acc2 + bias
//       = 2^F (s_tc + 128.5) - e  (mod 2^32; a per-block guard proves no wrap),
// with the rigorous bound |s_tc - s_ref| <= e 2^-F, e from ||c_AC||_2 and
// the exact quantisation residual of Mq (Cauchy-Schwarz) plus the float64
// rounding of the reference.  A sample is proven when floor(T / 2^F) ==
// floor((T + 2e) / 2^F): then it equals floor(s_ref + 128.5).  Blocks with
// any unproven sample are recomputed by the exact float64 path as before.
//
// CTA: 256 threads, 2 CTAs / SM (TMEM: 256 columns each).  Step s:
//   staging  - every thread loads its blocks (256-bit loads), writes the
//              int8 rows into the M=128 operand tiles (K-major, no swizzle)
//              and the block's bias / bound (int8 DC-free ||c||^2 by DP4A);
//   units    - Y tiles in two N=32 halves, the chroma tile (Cb and Cr side
//              by side in TMEM, same rows = same MCU) in four N=16 quarters;
//              thread 0 issues each unit's 6 / 12 MMAs into one of two TMEM
//              buffers (mbarrier ping-pong), all 8 warps read their lanes
//              (warp w: lanes 32(w%4).., half of the unit's columns) and
//              write the proven u8 samples into the planes of the v3 kernel;
//   phase B  - exact recompute + the pixel stage of row s-1 (shared with v3).
namespace tcs {
constexpr int kThreads = 256;
constexpr int kCols = 256;                 // TMEM columns per CTA
constexpr int kFmax = 21;                  // |s| + 128.5 < 2^(31-F) = 1024 at F = 21
// A unit = kUnitOut outputs of one operand tile: one MMA of N = 3 kUnitOut
// (limb-stacked) per K step into one of kNBuf TMEM buffers; the MMAs run
// kNBuf units ahead of the epilogue.  Fewer, larger units win (per-unit
// handshake and index overhead): 64 outputs (N = 192, one buffer released
// by the epilogue's last TMEM load) > 32 (N = 96 x 2) by 11 % > 16 (x 5).
#ifndef HJ_TC_UNIT_OUT
#define HJ_TC_UNIT_OUT 64
#endif
constexpr int kUnitOut = HJ_TC_UNIT_OUT;   // 64, 32 or 16
constexpr int kParts = 64 / kUnitOut;      // units per operand tile
constexpr int kUnitN = 3 * kUnitOut;       // MMA N (TMEM columns per unit)
constexpr int kNBuf = kCols / kUnitN;      // 1 (N = 192), 2 (N = 96) or 5 (N = 48)
constexpr int kPartB = kUnitN * 64;        // B operand bytes of one unit's outputs
constexpr int kNS = kUnitOut / 2;          // samples per thread per unit (two warps per lane quadrant)
template <int SUB>
constexpr int kStrip = SUB == HJ_SUB_444 ? 96 : SUB == HJ_SUB_422 ? 64 : 48;
template <int SUB>
struct Dims {
    static constexpr int S = kStrip<SUB>;
    static constexpr int NY = SUB == HJ_SUB_444 ? S : SUB == HJ_SUB_422 ? 2 * S : 4 * S;  // Y blocks / step
    static constexpr int NC = SUB == HJ_SUB_444 ? S : S + 2;                               // chroma MCUs / step
    static constexpr int YT = (NY + 127) / 128;                                            // Y operand tiles
    static constexpr int NB = NY + 2 * NC;                                                 // blocks / step
    static_assert(NC <= 128, "one chroma tile");
};
}  // namespace tcs

__device__ const double kMtab[64 * 64] = HJ_MTAB_INIT;
__device__ const double kMtabDirect[64 * 64] = HJ_MTAB_DIRECT_INIT;  // idct="direct"

template <int SUB>
struct SmemTc {
    using G = GeoT<SUB, tcs::kStrip<SUB>>;
    using D = tcs::Dims<SUB>;
    union {
        struct {
            alignas(128) uint8_t ay[D::YT][tc::kTileBytes];
            alignas(128) uint8_t acb[tc::kTileBytes];
            alignas(128) uint8_t acr[tc::kTileBytes];
        } a;                                      // MMA A operands (phase A)
        double g[tcs::kThreads / 8][64];          // exact-path staging (phase B)
    };
    alignas(128) uint8_t bm[2][tcs::kParts * tcs::kPartB];  // MMA B: [Y, chroma] x parts (limb-stacked)
    alignas(16) uint8_t ys[G::YSLOTS][G::MH * G::YW];
    alignas(16) uint8_t cbp[SUB == HJ_SUB_444 ? 2 : 1][SUB == HJ_SUB_444 ? 8 * G::YW : 16];
    alignas(16) uint8_t crp[SUB == HJ_SUB_444 ? 2 : 1][SUB == HJ_SUB_444 ? 8 * G::YW : 16];
    alignas(16) uint16_t cs[SUB == HJ_SUB_444 ? 1 : G::CROWS][SUB == HJ_SUB_444 ? 8 : G::CW];
    int qi[3][64];
    int2 meta[D::NB];                             // per staged block: bias, 2e
    int flag[D::NB];                              // 1 = queued for the exact path
    uint32_t queue[2][D::NB];
    uint32_t qdst[2][D::NB];
    int n_queue[2];
    int n_taken[2];
    alignas(8) uint64_t full[tcs::kNBuf];
    alignas(8) uint64_t empty[tcs::kNBuf];
    uint32_t tmem;
    int F[2];
    float dd[2], gg[2];                           // per table: error and magnitude factors
    unsigned long long mx[2], dmax[2], gmax[2];   // reductions (positive doubles as bits)
    int cr_differs;                               // Cr table != Cb table
    double dcc;                                   // the DC column's constant (M[0][i], all i)
};

// Build B (3 limbs of round(2^F M q), canonical K-major) for the luma table
// (c = 0) and the chroma table (c = 1), and the per-table factors of the
// screen bound.  128 threads: (c, output i), 64 coefficients each.
template <int SUB>
__device__ __forceinline__ void tc_build_b(SmemTc<SUB> &sm, const hj_image_t &im) {
    const int tid = threadIdx.x;
    const int c = tid >> 6, i = tid & 63;
    const int *q = im.q + (c ? 64 : 0);
    // the AAN map (fast) or the direct-basis map (idct="direct"); their DC
    // columns are constants (exactly 1/8 for AAN) and enter through the bias
    const double *kMtab = (im.flags & HJ_FLAG_DIRECT_IDCT) ? ::hj::kMtabDirect : ::hj::kMtab;
    if (tid == 0) sm.dcc = kMtab[0];
    if (tid < 2) sm.mx[tid] = sm.dmax[tid] = sm.gmax[tid] = 0ull;
    if (tid == 0) sm.cr_differs = 0;
    __syncthreads();
    if (tid < 128) {
        double mx = 0.0;
        for (int j = 1; j < 64; ++j) mx = fmax(mx, fabs(kMtab[j * 64 + i] * (double)q[j]));
        atomicMax(&sm.mx[c], (unsigned long long)__double_as_longlong(mx));
    }
    __syncthreads();
    if (tid < 128) {
        const double mx = __longlong_as_double((long long)sm.mx[c]);
        int F = tcs::kFmax;
        if (mx > 0.0) F = min(F, (int)floor(log2(8355711.0 / mx)));  // balanced 3-limb range
        const double sc = ldexp(1.0, F), isc = ldexp(1.0, -F);
        double dsum = 0.0, gsum = 0.0;
        // output i of part p = i / kUnitOut is row kUnitOut d + (i % kUnitOut)
        // of that part's N = 3 kUnitOut operand, d = limb: one MMA yields all
        // three limb products
        uint8_t *bh = sm.bm[c] + (i / tcs::kUnitOut) * tcs::kPartB;
        const int r0 = i % tcs::kUnitOut;
        for (int j0 = 0; j0 < 64; j0 += 4) {
            uint32_t w0 = 0, w1 = 0, w2 = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int j = j0 + k;
                const double mq = kMtab[j * 64 + i] * (double)q[j];
                int v = 0;
                if (j > 0) {
                    v = (int)__double2ll_rn(mq * sc);
                    const double d = (double)v * isc - mq;
                    dsum = fma(d, d, dsum);
                    gsum = fma(mq, mq, gsum);
                }
                // balanced signed limbs: v = l0 + 2^8 l1 + 2^16 l2, each in [-128, 127]
                const int l0 = ((v + 128) & 255) - 128;
                const int v1 = (v - l0) >> 8;
                const int l1 = ((v1 + 128) & 255) - 128;
                const int l2 = (v1 - l1) >> 8;
                w0 |= (uint32_t)(l0 & 255) << (8 * k);
                w1 |= (uint32_t)(l1 & 255) << (8 * k);
                w2 |= (uint32_t)(l2 & 255) << (8 * k);
            }
            *reinterpret_cast<uint32_t *>(bh + tc::kmaj(r0, j0)) = w0;
            *reinterpret_cast<uint32_t *>(bh + tc::kmaj(tcs::kUnitOut + r0, j0)) = w1;
            *reinterpret_cast<uint32_t *>(bh + tc::kmaj(2 * tcs::kUnitOut + r0, j0)) = w2;
        }
        atomicMax(&sm.dmax[c], (unsigned long long)__double_as_longlong(sqrt(dsum)));
        atomicMax(&sm.gmax[c], (unsigned long long)__double_as_longlong(sqrt(gsum)));
        if (i == 0) sm.F[c] = F;
        // the chroma B operand is built from the Cb table; a Cr table that
        // differs (rare: libjpeg and Pillow share table 1) sends Cr blocks
        // to the exact path
        if (c == 1 && im.q[64 + i] != im.q[128 + i]) sm.cr_differs = 1;
    }
    tc::fence_proxy_async();
    __syncthreads();
    if (tid < 2) {
        // error factor per unit ||c_AC||_2, in value units: the quantisation
        // residual (rounded up) + the reference's float64 rounding and the
        // table's own rounding, <= 2^-44 q_max sqrt(63) per unit of ||c||
        int qmax = 1;
        for (int j = 0; j < 64; ++j) qmax = max(qmax, im.q[(tid ? 64 : 0) + j]);
        const double d = __longlong_as_double((long long)sm.dmax[tid]) * (1.0 + 0x1p-20) + 0x1p-41 * qmax;
        sm.dd[tid] = __double2float_ru(d);
        sm.gg[tid] = __double2float_ru(__longlong_as_double((long long)sm.gmax[tid]) * (1.0 + 0x1p-20));
    }
    __syncthreads();
}

// Y-block geometry of a step: block b of the step's MCU-row strip ->
// coefficient index (relative to the row strip start) and plane offset.
template <int SUB, class G>
__device__ __forceinline__ int tc_y_off(int b) {
    if (SUB == HJ_SUB_444) return 8 * b;
    if (SUB == HJ_SUB_422) return 16 * (b >> 1) + 8 * (b & 1);
    return ((b & 3) >> 1) * 8 * G::YW + (b >> 2) * 16 + (b & 1) * 8;
}

// Stage one block: int8 row of the operand tile, bias / bound, range guard.
// Returns true when the block must take the exact path.
__device__ __forceinline__ bool tc_stage(const int16_t *__restrict__ src, uint8_t *arow_tile, int row, int q0,
                                         int F, float dd, float gg, double dcc, bool bad_in, int2 &meta) {
    int4 raw[8];
    const int4 *s4 = reinterpret_cast<const int4 *>(src);
#pragma unroll
    for (int r = 0; r < 8; r += 2) ldg_rows2(s4 + r, raw[r], raw[r + 1]);
    uint32_t lo[16];
    uint32_t rng = 0;
    int n2 = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int4 &v = raw[i >> 1];
        const uint32_t a = (uint32_t)((i & 1) ? v.z : v.x), b = (uint32_t)((i & 1) ? v.w : v.y);
        const uint32_t L = __byte_perm(a, b, 0x6420);   // low bytes of 4 coefficients
        const uint32_t H = __byte_perm(a, b, 0x7531);   // high bytes
        uint32_t Sg;  // sign of each low byte, replicated (PRMT sign mode; __byte_perm masks it off)
        asm("prmt.b32 %0, %1, %2, 0xECA8;" : "=r"(Sg) : "r"(a), "r"(b));
        const uint32_t m = i == 0 ? 0xFFFFFF00u : 0xFFFFFFFFu;  // DC excluded
        rng |= (H ^ Sg) & m;
        n2 = __dp4a((int)(L & m), (int)(L & m), n2);
        lo[i] = L;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
        sts128(arow_tile + tc::kmaj(row, 16 * k), make_uint4(lo[4 * k], lo[4 * k + 1], lo[4 * k + 2], lo[4 * k + 3]));
    const int dc = (int)(short)(raw[0].x & 0xffff);
    // |dc q0| < 2^31; the float product is within 2^-24 relative, covered by
    // the (1 + 2^-23) factors where it enters the bounds
    const float dcq = fabsf((float)dc * (float)q0);
    const float nrm = __fsqrt_ru((float)n2);
    const float scale = __int_as_float((127 + F) << 23);  // 2^F
    const float eu = __fmul_ru(__fmaf_ru(nrm, dd, __fmul_ru(__fmul_ru(dcq, 1.0000001f), 0x1p-44f)), scale);
    const int e = (int)ceilf(eu) + 3;  // + the bias rounding below
    // no-wrap guard: |T|, |T + 2e| < 2^31 with |s| <= |dc q0| / 8 + ||c_AC|| G
    const float sb = __fmaf_ru(nrm, gg, __fmul_ru(__fmul_ru(dcq, 1.0000001f), 0.125f));
    const bool wrap = __fadd_ru(__fmul_ru(__fadd_ru(sb, 129.0f), scale), 2.0f * (float)e + 8.0f) >= 2.0e9f;
    // 2^F (128.5 + dcc dc q0), rounded: dcc = 1/8 (AAN, exact) or the direct
    // basis' T00^2 (its double and this product err < 2^-24 absolute)
    const long long bias = __double2ll_rn(ldexp(fma(dcc, (double)dc * (double)q0, 128.5), F)) - e;
    meta = make_int2((int)bias, 2 * e);
    return bad_in || rng != 0 || wrap;
}

template <int SUB>
__global__ void __launch_bounds__(tcs::kThreads, 2)
render_tc_kernel(const hj_image_t *__restrict__ images, const Tile *__restrict__ tiles) {
    using Sm = SmemTc<SUB>;
    using G = typename Sm::G;
    using D = tcs::Dims<SUB>;
    constexpr int NT = tcs::kThreads;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    Sm &sm = *reinterpret_cast<Sm *>(smem_raw);

    const Tile t = tiles[blockIdx.x];
    const hj_image_t im = images[t.image];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int mpr = im.mcus_per_row;
    const int S = t.m1 - t.m0;
    // idct="direct" is screened too (its own exact map); the exact path
    // below still recomputes unproven blocks with the direct basis
    const bool direct = (im.flags & HJ_FLAG_DIRECT_IDCT) != 0;
    for (int i = tid; i < 192; i += NT) sm.qi[i >> 6][i & 63] = im.q[i];
    if (tid == 0) {
        sm.n_queue[0] = sm.n_queue[1] = 0; sm.n_taken[0] = sm.n_taken[1] = grab_base<SUB, kModeRef, true>();
        for (int b = 0; b < tcs::kNBuf; ++b) {
            tc::mbar_init(&sm.full[b], 1);
            tc::mbar_init(&sm.empty[b], NT / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) tc::tmem_alloc<tcs::kCols>(&sm.tmem);
    tc_build_b<SUB>(sm, im);  // (contains the barriers that publish the above)
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = sm.tmem;
    const int F0 = sm.F[0], F1 = sm.F[1];
    const float dd0 = sm.dd[0], dd1 = sm.dd[1], gg0 = sm.gg[0], gg1 = sm.gg[1];
    const bool cr_exact = sm.cr_differs != 0;
    const double dcc = sm.dcc;

    const int cm_lo = (SUB == HJ_SUB_444) ? t.m0 : t.m0 - 1;
    const int n_cm = (SUB == HJ_SUB_444) ? S : S + 2;
    const int n_yb = (SUB == HJ_SUB_444) ? S : (SUB == HJ_SUB_422 ? 2 * S : 4 * S);
    constexpr int YB = G::MW / 8 * (G::MH / 8);
    const int mcu_rows = im.mcu_rows;
    uint32_t unit = 0;  // running unit counter (TMEM buffer = unit % kNBuf)

    const int s_begin = (SUB == HJ_SUB_420) ? max(t.r0 - 2, -1) : t.r0;
    const int s_end = t.r1;
#pragma unroll 1
    for (int s = s_begin; s <= s_end; ++s) {
        const int par = s & 1;
        int *const nq = &sm.n_queue[par];
        uint32_t *const queue = sm.queue[par];
        uint32_t *const qdst = sm.qdst[par];
        const bool do_y = s >= t.r0 && s < t.r1;
        const int crow = (SUB == HJ_SUB_420) ? s + 1 : s;
        const bool do_c = (SUB == HJ_SUB_420) ? (crow >= t.r0 - 1 && crow <= t.r1 && crow >= 0 && crow < mcu_rows)
                                              : do_y;
        const int64_t yblk0 = ((int64_t)s * mpr + t.m0) * YB;  // first Y block of the step
        if (tid == 0) {
            sm.n_queue[par ^ 1] = 0;
            sm.n_taken[par ^ 1] = grab_base<SUB, kModeRef, true>();
            const int ny = HJ_PF_L2 ? s + 1 : -1;
            if (ny >= t.r0 && ny < t.r1) {
                const int64_t b0 = ((int64_t)ny * mpr + t.m0) * YB;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(im.y + b0 * 64),
                             "r"((unsigned)(S * YB * 128)));
            }
            const int nc = crow + 1;
            if (HJ_PF_L2 && nc < mcu_rows && nc <= t.r1) {
                const int c0 = max(cm_lo, 0), c1 = min(cm_lo + n_cm, mpr);
                const int64_t b0 = (int64_t)nc * mpr + c0;
                const unsigned bytes = (unsigned)((c1 - c0) * 128);
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(im.cb + b0 * 64), "r"(bytes));
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(im.cr + b0 * 64), "r"(bytes));
            }
        }

        // ---------------- staging: int8 operand rows + per-block bounds
        const int n_y = do_y ? n_yb : 0;
        const int n_c = do_c ? n_cm : 0;
#pragma unroll 1
        for (int j = tid; j < n_y + 2 * n_c; j += NT) {
            if (j < n_y) {
                int2 meta;
                const bool bad = tc_stage(im.y + (yblk0 + j) * 64, sm.a.ay[j >> 7], j & 127, sm.qi[0][0], F0, dd0,
                                          gg0, dcc, false, meta);
                sm.meta[j] = meta;
                sm.flag[j] = bad;
                if (bad) {
                    const uint32_t dst = (uint32_t)(sm.ys[par] + tc_y_off<SUB, G>(j) - smem_raw);
                    push_exact(nq, queue, qdst, (uint32_t)(yblk0 + j), dst);
                }
            } else {
                const int k = (j - n_y) >= n_c;           // 0: Cb, 1: Cr
                const int lm = j - n_y - k * n_c;         // chroma window MCU
                const int m = cm_lo + lm;
                if (m < 0 || m >= mpr) {
                    sm.flag[D::NY + k * D::NC + lm] = 1;  // no block: never written, never queued
                    continue;
                }
                const int64_t cblk = (int64_t)crow * mpr + m;
                int2 meta;
                const bool bad = tc_stage((k ? im.cr : im.cb) + cblk * 64, k ? sm.a.acr : sm.a.acb, lm, sm.qi[1 + k][0],
                                          F1, dd1, gg1, dcc, k && cr_exact, meta);
                sm.meta[D::NY + k * D::NC + lm] = meta;
                sm.flag[D::NY + k * D::NC + lm] = bad;
                uint32_t dst;
                if (SUB == HJ_SUB_444) {
                    dst = (uint32_t)((k ? sm.crp[par] : sm.cbp[par]) + 8 * lm - smem_raw);
                } else {
                    const int cslot = (SUB == HJ_SUB_420) ? (crow % 3) : par;
                    const int cw0 = cslot * 8 * G::CW + 8 * lm;
                    dst = ((2u + k) << 30) | (uint32_t)cw0;
                    if (SUB == HJ_SUB_420 && k == 0) {
                        // the slot's old row 7 (MCU row crow-3) is the top
                        // context of MCU row crow-2, drawn this step
                        uint16_t *save = &sm.cs[24][0] + 8 * lm;
                        sts128(save, lds128(&sm.cs[0][0] + cw0 + 7 * G::CW));
                    }
                }
                if (bad) push_exact(nq, queue, qdst, ((1u + k) << 30) | (uint32_t)cblk, dst);
            }
        }
        tc::fence_proxy_async();
        __syncthreads();

        // ---------------- units: MMA (thread 0) -> TMEM -> proven samples
        constexpr int P = tcs::kParts, NS = tcs::kNS;
        const int n_yunits = do_y ? P * ((n_yb + 127) >> 7) : 0;
        const int n_units = n_yunits + (do_c ? 2 * P : 0);
        // Y unit k: tile k / P, part k % P; chroma unit: (Cb, Cr) x part, order Cb0 Cr0 Cb1 Cr1 ...
        auto issue = [&](int k, uint32_t u) {
            const uint32_t b = u % tcs::kNBuf, dcol = tbase + b * tcs::kUnitN;
            if (u >= (uint32_t)tcs::kNBuf) tc::mbar_wait(&sm.empty[b], ((u - tcs::kNBuf) / tcs::kNBuf) & 1);
            tc::fence_after();
            constexpr uint32_t id = tc::idesc_i8(tcs::kUnitN, true, true);
            const int cu = k - n_yunits;
            const uint32_t a0 = k < n_yunits ? tc::smem_u32(sm.a.ay[k / P]) : tc::smem_u32((cu & 1) ? sm.a.acr : sm.a.acb);
            const uint32_t b0 = tc::smem_u32(sm.bm[k < n_yunits ? 0 : 1]) + (k < n_yunits ? k % P : cu >> 1) * tcs::kPartB;
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) tc::mma_i8(dcol, tc::sdesc(a0 + ks * 256), tc::sdesc(b0 + ks * 256), id, ks);
            tc::commit(&sm.full[b]);
        };
        if (tid == 0)
            for (int k = 0; k < n_units && k < tcs::kNBuf; ++k) issue(k, unit + k);
        const int qd = warp & 3, grp = warp >> 2;
        const int row = 32 * qd + lane;
        uint32_t cbk[NS / 4];  // 4:2:x: Cb samples held for the paired Cr unit
#pragma unroll 1
        for (int k = 0; k < n_units; ++k, ++unit) {
            const uint32_t b = unit % tcs::kNBuf;
            const uint32_t tl = tbase + ((uint32_t)(32 * qd) << 16) + b * tcs::kUnitN;
            tc::mbar_wait(&sm.full[b], (unit / tcs::kNBuf) & 1);
            tc::fence_after();
            __syncwarp();  // the tcgen05.ld below are warp-collective (.sync.aligned)
            // this thread's block (TMEM lane) and its NS / 8 sample rows,
            // read in chunks of CH outputs (the last chunk's loads release
            // the buffer to the next unit's MMAs)
            constexpr int CH = NS < 16 ? NS : 16, NCH = NS / CH;
            const bool is_y = k < n_yunits;
            const int cu = k - n_yunits, cc = cu & 1;
            const int part = is_y ? (k % P) : (cu >> 1);
            const int yb = (k / P) * 128 + row, lm = row;
            const int fi = is_y ? yb : D::NY + cc * D::NC + lm;
            const bool valid = is_y ? yb < n_yb : (lm < n_cm && cm_lo + lm >= 0 && cm_lo + lm < mpr);
            const int Fk = is_y ? F0 : F1;
            const int flagged = valid ? sm.flag[fi] : 1;
            const int2 mt = valid ? sm.meta[fi] : make_int2(0, 0);
            const int srow0 = part * (tcs::kUnitOut / 8) + grp * (NS / 8);
            const int cslot = (SUB == HJ_SUB_420) ? (crow % 3) : par;
            uint32_t fail = 0;
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) {
                uint32_t a0[CH], a1[CH], a2[CH];  // limbs 0..2 of CH outputs
                const uint32_t ta = tl + NS * grp + CH * ch;
                if constexpr (CH == 16) {
                    tc::ld16(ta, a0);
                    tc::ld16(ta + tcs::kUnitOut, a1);
                    tc::ld16(ta + 2 * tcs::kUnitOut, a2);
                } else {
                    tc::ld8(ta, a0);
                    tc::ld8(ta + tcs::kUnitOut, a1);
                    tc::ld8(ta + 2 * tcs::kUnitOut, a2);
                }
                tc::wait_ld();
                if (ch == NCH - 1) {
                    tc::fence_before();
                    __syncwarp();
                    if (lane == 0) tc::mbar_arrive(&sm.empty[b]);
                    if (tid == 0 && k + tcs::kNBuf < n_units) issue(k + tcs::kNBuf, unit + tcs::kNBuf);
                }
                if (!valid) continue;
                int n[CH];
#pragma unroll
                for (int i = 0; i < CH; ++i) {
                    const uint32_t T = a0[i] + (uint32_t)mt.x + (a1[i] << 8) + (a2[i] << 16);
                    fail |= T ^ (T + (uint32_t)mt.y);
                    n[i] = (int)T >> Fk;
                }
                uint32_t w[CH / 4];
#pragma unroll
                for (int q = 0; q < CH / 4; ++q) w[q] = pack4(n[4 * q], n[4 * q + 1], n[4 * q + 2], n[4 * q + 3]);
                const int srow = srow0 + ch * (CH / 8);
                if (is_y || SUB == HJ_SUB_444) {
                    uint8_t *dst = (is_y ? sm.ys[par] + tc_y_off<SUB, G>(yb) : (cc ? sm.crp[par] : sm.cbp[par]) + 8 * lm) +
                                   srow * G::YW;
#pragma unroll
                    for (int r = 0; r < CH / 8; ++r)
                        *reinterpret_cast<uint2 *>(dst + r * G::YW) = make_uint2(w[2 * r], w[2 * r + 1]);
                } else if (cc == 0) {
#pragma unroll
                    for (int q = 0; q < CH / 4; ++q) cbk[ch * (CH / 4) + q] = w[q];  // paired with the Cr unit next
                } else {
                    uint16_t *cdst = &sm.cs[0][0] + cslot * 8 * G::CW + 8 * lm + srow * G::CW;
                    const uint32_t *cb = cbk + ch * (CH / 4);
#pragma unroll
                    for (int r = 0; r < CH / 8; ++r)
                        sts128(cdst + r * G::CW,
                               make_uint4(__byte_perm(cb[2 * r], w[2 * r], 0x5140), __byte_perm(cb[2 * r], w[2 * r], 0x7362),
                                          __byte_perm(cb[2 * r + 1], w[2 * r + 1], 0x5140),
                                          __byte_perm(cb[2 * r + 1], w[2 * r + 1], 0x7362)));
                }
            }
            if (valid) {
                if (!flagged && (fail >> Fk) != 0 && atomicExch(&sm.flag[fi], 1) == 0) {
                    if (is_y) {
                        push_exact(nq, queue, qdst, (uint32_t)(yblk0 + yb),
                                   (uint32_t)(sm.ys[par] + tc_y_off<SUB, G>(yb) - smem_raw));
                        if (HJ_PF_EXACT) prefetch_l1(im.y + (yblk0 + yb) * 64);
                    } else {
                        const int64_t cblk = (int64_t)crow * mpr + cm_lo + lm;
                        const uint32_t dst = SUB == HJ_SUB_444
                                                 ? (uint32_t)((cc ? sm.crp[par] : sm.cbp[par]) + 8 * lm - smem_raw)
                                                 : ((2u + cc) << 30) | (uint32_t)(cslot * 8 * G::CW + 8 * lm);
                        push_exact(nq, queue, qdst, ((1u + cc) << 30) | (uint32_t)cblk, dst);
                        if (HJ_PF_EXACT) prefetch_l1((cc ? im.cr : im.cb) + cblk * 64);
                    }
                }
            }
        }
        __syncthreads();

        // ---------------- phase B: exact recompute ∥ pixel stage of row s-1
        exact_phase<SUB, kModeRef, G, NT>(sm, smem_raw, im, par, direct);
        pixel_phase<SUB, kModeRef, G, SmemTc<SUB>, true>(sm, im, t, s, par, do_c);
        __syncthreads();
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<tcs::kCols>(tbase);
}

// two CTAs per SM: (228 KB - 2 x 1 KB reserved) / 2
static_assert(sizeof(SmemTc<HJ_SUB_444>) <= 113 * 1024, "4:4:4 tensor-core smem");
static_assert(sizeof(SmemTc<HJ_SUB_422>) <= 113 * 1024, "4:2:2 tensor-core smem");
static_assert(sizeof(SmemTc<HJ_SUB_420>) <= 113 * 1024, "4:2:0 tensor-core smem");

std::atomic<unsigned long long> g_tc_launches{0};

template <int SUB>
cudaError_t launch_tc(const hj_image_t *images, const Tile *tiles, int n_tiles, cudaStream_t stream) {
    g_tc_launches.fetch_add(1, std::memory_order_relaxed);
    static std::atomic<uint64_t> configured{0};
    const int bytes = (int)sizeof(SmemTc<SUB>);
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = 1ull << (dev & 63);
    if (!(configured.load(std::memory_order_acquire) & bit)) {
        e = cudaFuncSetAttribute(render_tc_kernel<SUB>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        if (e != cudaSuccess) return e;
        configured.fetch_or(bit, std::memory_order_release);
    }
    render_tc_kernel<SUB><<<n_tiles, tcs::kThreads, bytes, stream>>>(images, tiles);
    return cudaGetLastError();
}

template <int SUB, int MODE>
cudaError_t launch_sub(const hj_image_t *images, const Tile *tiles, int n_tiles, cudaStream_t stream) {
    // the dynamic shared-memory opt-in is per device; set it once per device
    // (thread-safe: a racing second setter is harmless and idempotent)
    static std::atomic<uint64_t> configured{0};
    const int bytes = (int)sizeof(Smem<SUB>);
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = 1ull << (dev & 63);
    if (!(configured.load(std::memory_order_acquire) & bit)) {
        e = cudaFuncSetAttribute(render_kernel<SUB, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        if (e != cudaSuccess) return e;
        configured.fetch_or(bit, std::memory_order_release);
    }
    render_kernel<SUB, MODE><<<n_tiles, kNT<SUB>, bytes, stream>>>(images, tiles);
    return cudaGetLastError();
}

}  // namespace

unsigned long long tc_launch_count() { return g_tc_launches.load(); }

unsigned long long exact_block_count() {
    unsigned long long v = 0;
    cudaMemcpyFromSymbol(&v, g_exact_blocks, sizeof(v));
    return v;
}

size_t render_smem_bytes_tc(int sub) {
    return sub == HJ_SUB_444 ? sizeof(SmemTc<HJ_SUB_444>)
         : sub == HJ_SUB_422 ? sizeof(SmemTc<HJ_SUB_422>) : sizeof(SmemTc<HJ_SUB_420>);
}

size_t render_smem_bytes(int sub) {
    return sub == HJ_SUB_444 ? sizeof(Smem<HJ_SUB_444>)
         : sub == HJ_SUB_422 ? sizeof(Smem<HJ_SUB_422>) : sizeof(Smem<HJ_SUB_420>);
}

// mode: kModeRef (AAN / direct chosen per image by HJ_FLAG_DIRECT_IDCT) or
// kModeIslow (every image of the group decoded with libjpeg's arithmetic).
cudaError_t launch_render(int sub, int mode, const hj_image_t *images, const Tile *tiles, int n_tiles,
                          cudaStream_t stream) {
    if (n_tiles <= 0) return cudaSuccess;
    if (mode == kModeRefTc) {
        if (sub == HJ_SUB_444) return launch_tc<HJ_SUB_444>(images, tiles, n_tiles, stream);
        if (sub == HJ_SUB_422) return launch_tc<HJ_SUB_422>(images, tiles, n_tiles, stream);
        return launch_tc<HJ_SUB_420>(images, tiles, n_tiles, stream);
    }
    if (mode == kModeIslow) {
        if (sub == HJ_SUB_444) return launch_sub<HJ_SUB_444, kModeIslow>(images, tiles, n_tiles, stream);
        if (sub == HJ_SUB_422) return launch_sub<HJ_SUB_422, kModeIslow>(images, tiles, n_tiles, stream);
        return launch_sub<HJ_SUB_420, kModeIslow>(images, tiles, n_tiles, stream);
    }
    if (sub == HJ_SUB_444) return launch_sub<HJ_SUB_444, kModeRef>(images, tiles, n_tiles, stream);
    if (sub == HJ_SUB_422) return launch_sub<HJ_SUB_422, kModeRef>(images, tiles, n_tiles, stream);
    return launch_sub<HJ_SUB_420, kModeRef>(images, tiles, n_tiles, stream);
}

}  // namespace hj
