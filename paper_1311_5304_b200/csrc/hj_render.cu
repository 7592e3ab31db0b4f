// sm_100a render kernel: dequantise -> IDCT -> [h2v1 / h2v2 fancy upsample]
// -> YCbCr->RGB, bit-exact against the reference's float64 path.
//
// IDCT numerics:  every block is first transformed
// in binary32 with the reference's AAN operation order, packed two columns /
// two rows per f32x2 instruction (FFMA2/FADD2).  A rigorous first-order
// error bound E = u * sum_i K_i |x_i| (K from tools/analysis/
// screen_constants.py) brackets each sample; if no rounding boundary of
// floor(s + 128.5) lies inside [s - E, s + E] for all 64 samples, the binary32
// result provably rounds like the reference's float64 one.  Otherwise (a few
// percent of real blocks, all blocks in "direct" mode) the block is queued and
// recomputed in exact float64 (explicitly rounded __dadd_rn/__dmul_rn, the
// reference's operation order) by the CTA's fallback pass.
//
// Work decomposition: a CTA (128 threads) owns a strip of MCU columns of one
// image and sweeps down a range of MCU rows.  Per MCU row:
//   (1) screen: each thread takes one job of two blocks (two Y blocks, or
//       the Cb+Cr pair of one MCU), writes Y samples as u8 and chroma as SWAR
//       words (Cb | Cr << 16) so the upsampler filters both planes per op;
//   (2) exact fallback for queued blocks (float64, few threads);
//   (3) upsample + colour + store: 8 pixels per item, integer colour
//       formulas, saturating I2IP byte packing, 8-byte RGB stores.
// 4:2:2 / 4:2:0 strips include the chroma MCU left/right of the strip; 4:2:0
// keeps the previous / next chroma MCU row resident (vertical context).
#include <cstdint>

#include "hj_common.cuh"
#include "hj_render.cuh"
#include "hj_screen.h"

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

// FP32 screen of one block: returns true (and the 64 samples, u8 row-major,
// 4 per word) when every sample is proven equal to the reference's float64
// result; false = recompute exactly.
__device__ __forceinline__ bool screen_block(const int16_t *__restrict__ src, const float *qf,
                                             uint32_t (&out)[16]) {
    int4 raw[8];
    const int4 *s4 = reinterpret_cast<const int4 *>(src);
#pragma unroll
    for (int r = 0; r < 8; ++r) raw[r] = __ldg(s4 + r);
    u64 X[4][8];  // X[cp][r] = (x[r][2cp], x[r][2cp+1])
    float b0 = 0.f, b1 = 0.f, b2 = 0.f, b3 = 0.f;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        float4 qa = lds128f(qf + r * 8), qb = lds128f(qf + r * 8 + 4);
        const int w[4] = {raw[r].x, raw[r].y, raw[r].z, raw[r].w};
        const float q[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
#pragma unroll
        for (int cp = 0; cp < 4; ++cp) {
            float c0 = (float)(short)(w[cp] & 0xffff);
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
    float B = (b0 + b1) + (b2 + b3);
    float e = fmaf(B, 5.9754e-8f, 1.5260e-5f);
    float eq = ceilf(e * 32768.0f) * (1.0f / 32768.0f);
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
            Q[j] = (j & 1) ? pk(phi(a), phi(b)) : pk(plo(a), plo(b));
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

// ------------------------------------------------------ exact fallback

// Cooperative exact float64 IDCT of one block by 8 threads (lane l = column
// l in the column pass, row l in the row pass), the reference's operation
// order (_native.pyx:364-388); column results staged in `g` (64 doubles,
// shared).  Returns row l's 8 rounded samples packed in a uint2.
__device__ __forceinline__ uint2 exact_block_x8(const int16_t *__restrict__ src, const int *q, bool direct,
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

template <int SUB>
struct Geo;
// Chroma SWAR words hold (c << CSH) | (c << CSH) << 16: 4:2:0 scales by 16 and
// 4:2:2 by 64 so the fancy filters' results land byte-aligned (the filtered
// value is byte 1 / byte 3 of the word; every lane stays below 2^16).
template <>
struct Geo<HJ_SUB_444> {
    static constexpr int S = kStrip444, MW = 8, MH = 8, CSH = 0;
    static constexpr int YW = 8 * S;   // Y plane width (bytes)
    static constexpr int CW = 8 * S;   // chroma window width (words)
    static constexpr int CROWS = 8;
};
template <>
struct Geo<HJ_SUB_422> {
    static constexpr int S = kStrip422, MW = 16, MH = 8, CSH = 6;
    static constexpr int YW = 16 * S;
    static constexpr int CW = 8 * (S + 2);
    static constexpr int CROWS = 8;
};
template <>
struct Geo<HJ_SUB_420> {
    static constexpr int S = kStrip420, MW = 16, MH = 16, CSH = 4;
    static constexpr int YW = 16 * S;
    static constexpr int CW = 8 * (S + 2);
    static constexpr int CROWS = 17;  // MCU rows c (slot c&1, 8 rows each) + row 16: last row of r-1
};

constexpr int kExactGroups = kThreads / 8;  // blocks recomputed in parallel
constexpr int kQueueMax = 2 * kThreads;     // >= blocks of one sweep step

template <int SUB>
struct Smem {
    using G = Geo<SUB>;
    uint8_t ys[G::MH * G::YW];
    uint32_t cs[G::CROWS * G::CW];          // SWAR chroma: Cb | Cr << 16
    float qf[3][64];                        // binary32 q * pre (screen)
    int qi[3][64];                          // integer q (exact path)
    double g[kExactGroups][64];             // exact-path column results
    uint32_t queue[kQueueMax];              // exact-path jobs
    uint32_t qdst[kQueueMax];
    uint4 cscratch[kThreads][4];            // Cb samples of a chroma job
    int n_queue[2];                         // per iteration parity (reset lag)
};

__device__ __forceinline__ void write_y_rows(uint8_t *ys, int yoff, int stride, const uint32_t (&w)[16]) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
        *reinterpret_cast<uint2 *>(ys + yoff + r * stride) = make_uint2(w[2 * r], w[2 * r + 1]);
}

// Interleave Cb and Cr sample rows into SWAR words:
// word k = (cb_k | cr_k << 16) << CSH.
template <int CSH>
__device__ __forceinline__ void write_c_rows(uint32_t *cs, int coff, int stride, const uint4 *cb,
                                             const uint32_t (&cr)[16]) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        uint4 cbv = cb[r >> 1];
        const uint32_t cbw[2] = {(r & 1) ? cbv.z : cbv.x, (r & 1) ? cbv.w : cbv.y};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            uint32_t a = cbw[h], b = cr[2 * r + h];
            uint32_t t0 = __byte_perm(a, b, 0x5140), t1 = __byte_perm(a, b, 0x7362);
            uint4 v = make_uint4(__byte_perm(t0, 0, 0x4140) << CSH, __byte_perm(t0, 0, 0x4342) << CSH,
                                 __byte_perm(t1, 0, 0x4140) << CSH, __byte_perm(t1, 0, 0x4342) << CSH);
            *reinterpret_cast<uint4 *>(cs + coff + r * stride + 4 * h) = v;
        }
    }
}

template <int SUB>
__global__ void __launch_bounds__(kThreads, HJ_MIN_CTAS)
render_kernel(const hj_image_t *__restrict__ images, const Tile *__restrict__ tiles) {
    using G = Geo<SUB>;
    extern __shared__ __align__(16) uint8_t smem_raw[];
    Smem<SUB> &sm = *reinterpret_cast<Smem<SUB> *>(smem_raw);

    const Tile t = tiles[blockIdx.x];
    const hj_image_t im = images[t.image];
    const int tid = threadIdx.x;
    const int mpr = im.mcus_per_row;
    const int S = t.m1 - t.m0;
    const bool direct = (im.flags & HJ_FLAG_DIRECT_IDCT) != 0;
    for (int i = tid; i < 192; i += kThreads) {
        int q = im.q[i];
        sm.qi[i >> 6][i & 63] = q;
        sm.qf[i >> 6][i & 63] = (float)((double)q * kPre64[i & 63]);
    }
    if (tid == 0) sm.n_queue[0] = sm.n_queue[1] = 0;

    // chroma MCU window of the strip: [m0-1, m1+1) for 4:2:2/4:2:0
    const int cm_lo = (SUB == HJ_SUB_444) ? t.m0 : t.m0 - 1;
    const int n_cm = (SUB == HJ_SUB_444) ? S : S + 2;
    // Y jobs: two blocks each (444: MCU pair; 422: one MCU; 420: half MCU)
    const int n_yj = (SUB == HJ_SUB_444) ? (S + 1) / 2 : (SUB == HJ_SUB_422 ? S : 2 * S);
    const bool left_edge = (t.m0 == 0), right_edge = (t.m1 == mpr);
    const int n_groups = (G::MW / 8) * S;  // 8-pixel groups per pixel row of the strip
    const int oy0 = tid / n_groups, gx0 = tid - oy0 * n_groups;
    const int ystep = kThreads / n_groups, gstep = kThreads - ystep * n_groups;
    __syncthreads();

    // One transform job = two blocks through one screen call site, kept
    // branch-free up to the call so a warp mixing Y and chroma jobs runs the
    // screen once per block slot (no divergent duplication).  Y job: blocks
    // side by side in the Y plane; chroma job (job >= n_yj): the Cb and Cr
    // block of one MCU of chroma row crow, combined into SWAR words.
    // Exact-path queue entry: comp << 30 | block index; destination: Y byte
    // offset, or 1 << 31 | lane << 30 | chroma word offset.
    auto run_job = [&](int job, int yrow, int crow, int *n_queue, bool active) {
        const bool is_y = job < n_yj;
        const int lm = job - n_yj;                 // chroma window MCU
        const int m = cm_lo + lm;
        const bool valid = active && (is_y || (m >= 0 && m < mpr));
        const int nb = (SUB == HJ_SUB_444 && is_y && 2 * job + 1 >= S) ? 1 : 2;
        // Y: first block index and plane offset of the job
        int64_t yblk;
        int yoff0;
        if (SUB == HJ_SUB_444) {
            yblk = (int64_t)yrow * mpr + t.m0 + 2 * job;
            yoff0 = 2 * job * 8;
        } else if (SUB == HJ_SUB_422) {
            yblk = ((int64_t)yrow * mpr + t.m0 + job) * 2;
            yoff0 = job * 16;
        } else {  // MCU job/2, blocks 0,1 (top) or 2,3 (bottom)
            yblk = ((int64_t)yrow * mpr + t.m0 + (job >> 1)) * 4 + 2 * (job & 1);
            yoff0 = (job & 1) * 8 * G::YW + (job >> 1) * 16;
        }
        const int64_t cblk = (int64_t)crow * mpr + m;
        const int coff = (SUB == HJ_SUB_420 ? (crow & 1) * 8 * G::CW : 0) + lm * 8;
        if constexpr (SUB == HJ_SUB_420) {
            // copy-on-overwrite: the slot's old row 7 (chroma MCU row crow-2)
            // becomes row 16, the context of MCU row crow-1
            if (valid && !is_y) {
#pragma unroll
                for (int i = 0; i < 8; i += 4)
                    *reinterpret_cast<uint4 *>(sm.cs + 16 * G::CW + lm * 8 + i) =
                        *reinterpret_cast<const uint4 *>(sm.cs + coff + 7 * G::CW + i);
            }
        }
        // the same job of the next iteration reads the blocks one MCU row
        // down: pull them into L2 now (hides DRAM latency next iteration)
        if (valid) {
            const bool more = is_y ? (yrow + 1 < t.r1) : (crow + 1 < im.mcu_rows && crow + 1 <= t.r1);
            if (more) {
                const int64_t ystep = (int64_t)mpr * (G::MW / 8) * (G::MH / 8);  // Y blocks per MCU row
                const int16_t *p0 = is_y ? im.y + (yblk + ystep) * 64 : im.cb + (cblk + mpr) * 64;
                const int16_t *p1 = is_y ? p0 + 64 : im.cr + (cblk + mpr) * 64;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(p0));
                if (nb > 1) asm volatile("prefetch.global.L2 [%0];" ::"l"(p1));
            }
        }
        bool ok0 = false;
#pragma unroll 1
        for (int k = 0; k < 2; ++k) {
            const bool run = valid && k < nb;
            const int64_t blk = is_y ? yblk + k : cblk;
            const int16_t *src = (is_y ? im.y : (k == 0 ? im.cb : im.cr)) + blk * 64;
            const float *qf = sm.qf[is_y ? 0 : 1 + k];
            uint32_t w[16];
            bool ok = false;
            if (run) ok = !direct && screen_block(src, qf, w);
            if (!run) continue;
            if (is_y) {
                const int yoff = yoff0 + k * 8;
                if (ok) {
                    write_y_rows(sm.ys, yoff, G::YW, w);
                } else {
                    int e = atomicAdd(n_queue, 1);
                    sm.queue[e] = (uint32_t)blk;
                    sm.qdst[e] = (uint32_t)yoff;
                }
            } else if (k == 0) {
                ok0 = ok;
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    sm.cscratch[tid][i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
            } else if (ok && ok0) {
                write_c_rows<G::CSH>(sm.cs, coff, G::CW, sm.cscratch[tid], w);
            } else {
                int e = atomicAdd(n_queue, 2);
                sm.queue[e] = (uint32_t)blk | (1u << 30);
                sm.qdst[e] = (uint32_t)coff | (1u << 31);
                sm.queue[e + 1] = (uint32_t)blk | (2u << 30);
                sm.qdst[e + 1] = (uint32_t)coff | (1u << 31) | (1u << 30);
            }
        }
    };

    // 4:2:0 sweeps one iteration ahead on chroma: iteration `it` transforms
    // the Y blocks of MCU row it and the chroma of MCU row it+1, starting two
    // iterations early (transform-only) to bring in rows r0-1 and r0.
    const int it0 = (SUB == HJ_SUB_420) ? max(t.r0 - 2, -1) : t.r0;
#pragma unroll 1
    for (int it = it0; it < t.r1; ++it) {
        const bool draw = it >= t.r0;
        int crow = it, n_c = n_cm;
        if (SUB == HJ_SUB_420) {
            crow = it + 1;
            n_c = (crow >= t.r0 - 1 && crow >= 0 && crow < im.mcu_rows) ? n_cm : 0;
        }
        const int n_y = draw ? n_yj : 0;
        // ---- (1) binary32 screen of this iteration's blocks
        int *const nq = &sm.n_queue[it & 1];
        // every lane runs the job loop the same number of times (inactive
        // lanes ride along) so the screen is never split by divergence
        const int n_jobs = n_y + n_c;
#pragma unroll 1
        for (int j0 = 0; j0 < n_jobs; j0 += kThreads) {
            const int j = j0 + tid;
            run_job(j < n_y ? j : n_yj + (j - n_y), it, crow, nq, j < n_jobs);
        }
        __syncthreads();
        // ---- (2) exact float64 recompute of the unproven blocks, 8 threads each
        {
            const int n = *nq;
            const int grp = tid >> 3, l = tid & 7;
            const unsigned gmask = 0xffu << (tid & 24);  // the 8 lanes of this group
#pragma unroll 1
            for (int e = grp; e < n; e += kExactGroups) {
                const uint32_t job = sm.queue[e], dst = sm.qdst[e];
                const int comp = job >> 30;
                const int64_t blk = job & 0x3fffffff;
                const int16_t *src = (comp == 0 ? im.y : comp == 1 ? im.cb : im.cr) + blk * 64;
                const uint2 row = exact_block_x8(src, sm.qi[comp], direct, sm.g[grp], l, gmask);
                if (!(dst >> 31)) {
                    *reinterpret_cast<uint2 *>(sm.ys + dst + l * G::YW) = row;
                } else {
                    const int coff = dst & 0x3fffffff, lane = (dst >> 30) & 1;
                    uint16_t *c16 = reinterpret_cast<uint16_t *>(sm.cs + coff + l * G::CW) + lane;
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        c16[2 * c] = (uint16_t)(((c < 4 ? row.x >> (8 * c) : row.y >> (8 * (c - 4))) & 0xff) << G::CSH);
                }
            }
            if (tid == 0 && n) atomicAdd(&g_exact_blocks, (unsigned long long)n);
        }
        __syncthreads();
        // this parity's counter is next used two iterations (>= 2 barriers) later
        if (tid == 0) *nq = 0;
        if (!draw) continue;

        // ---- (3) upsample + colour + store MCU row `it`
        const int y_base = it * G::MH;
        const int x_base = t.m0 * G::MW;
        const int ylim = min(G::MH, im.height - y_base);
        // items (oy, gx) = 8 pixels, walked without a division per item
        int oy = oy0, gx = gx0;
#pragma unroll 1
        for (; oy < ylim; gx += gstep, oy += ystep) {
            if (gx >= n_groups) {
                gx -= n_groups;
                ++oy;
                if (oy >= ylim) break;
            }
            const int x0 = x_base + gx * 8;
            const int npx = min(8, im.width - x0);
            if (npx <= 0) continue;
            const uint2 yv = *reinterpret_cast<const uint2 *>(sm.ys + oy * G::YW + gx * 8);
            int Y[8], cbv[8], crv[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                Y[i] = (int)__byte_perm(yv.x, 0, 0x4440 + i);
                Y[4 + i] = (int)__byte_perm(yv.y, 0, 0x4440 + i);
            }
            if (SUB == HJ_SUB_444) {
                const uint32_t *cr = sm.cs + oy * G::CW + gx * 8;
                uint4 a = *reinterpret_cast<const uint4 *>(cr), b = *reinterpret_cast<const uint4 *>(cr + 4);
                const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    cbv[i] = (int)__byte_perm(w[i], 0, 0x4440);
                    crv[i] = (int)__byte_perm(w[i], 0, 0x4442);
                }
            } else {
                // chroma samples k0-1 .. k0+4 (k0 = 8*m0 + 4*gx) as window-local
                // words; the padded plane's first/last column is replicated
                // (fallback.py:200-212, _native.pyx:477-480)
                const int kl = 8 * (t.m0 - cm_lo) + 4 * gx;
                const int dl = (left_edge && gx == 0) ? 0 : -1;
                const int dr = (right_edge && gx == n_groups - 1) ? 3 : 4;
                uint32_t c[6];
                uint32_t rnd_e, rnd_o;
                if (SUB == HJ_SUB_422) {
                    const uint32_t *cr = sm.cs + oy * G::CW + kl;
                    uint4 mid = *reinterpret_cast<const uint4 *>(cr);
                    c[0] = cr[dl];
                    c[1] = mid.x;
                    c[2] = mid.y;
                    c[3] = mid.z;
                    c[4] = mid.w;
                    c[5] = cr[dr];
                    // h2v1 on 64x-scaled lanes: even 64(3c+prev+1), odd 64(3c+next+2)
                    rnd_e = 0x00400040u;
                    rnd_o = 0x00800080u;
                } else {
                    // near chroma row ci, far row cf (clamped to the padded plane)
                    const int ch_img = 8 * im.mcu_rows;
                    const int ci = 8 * it + (oy >> 1);
                    const int cf = min(max(ci + ((oy & 1) ? 1 : -1), 0), ch_img - 1);
                    // row 8*it-1: saved in row 16 when this iteration overwrote
                    // its slot with MCU row it+1, else still in slot (it-1)&1
                    const int rn = (it & 1) * 8 + (ci & 7);
                    const int rf = cf >= 8 * it ? (((cf >> 3) & 1) * 8 + (cf & 7))
                                 : (it + 1 < im.mcu_rows ? 16 : ((it - 1) & 1) * 8 + 7);
                    const uint32_t *cn = sm.cs + rn * G::CW + kl;
                    const uint32_t *cfp = sm.cs + rf * G::CW + kl;
                    uint4 mn = *reinterpret_cast<const uint4 *>(cn), mf = *reinterpret_cast<const uint4 *>(cfp);
                    // colsum = 3*near + far per lane (libjpeg h2v2 fancy), 16x scaled
                    c[0] = cn[dl] * 3u + cfp[dl];
                    c[1] = mn.x * 3u + mf.x;
                    c[2] = mn.y * 3u + mf.y;
                    c[3] = mn.z * 3u + mf.z;
                    c[4] = mn.w * 3u + mf.w;
                    c[5] = cn[dr] * 3u + cfp[dr];
                    // even 16(3cs+prev+8), odd 16(3cs+next+7)
                    rnd_e = 0x00800080u;
                    rnd_o = 0x00700070u;
                }
                // filtered value = byte 1 (Cb) / byte 3 (Cr) of each word
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint32_t t3 = c[i + 1] * 3u;
                    const uint32_t ev = t3 + c[i] + rnd_e, od = t3 + c[i + 2] + rnd_o;
                    cbv[2 * i] = (int)__byte_perm(ev, 0, 0x4441);
                    crv[2 * i] = (int)(ev >> 24);
                    cbv[2 * i + 1] = (int)__byte_perm(od, 0, 0x4441);
                    crv[2 * i + 1] = (int)(od >> 24);
                }
            }
            Rgb p[8];
            bool special = false;
#pragma unroll
            for (int i = 0; i < 8; ++i) p[i] = colour(Y[i], cbv[i], crv[i], special);
            if (special) {
#pragma unroll
                for (int i = 0; i < 8; ++i) p[i].g = colour_g_exact(Y[i], cbv[i], crv[i]);
            }
            uint32_t w[6];
            pack_rgb8(p, w);
            store_rgb8(im.rgb + ((int64_t)(y_base + oy) * im.width + x0) * 3, w, npx);
        }
        __syncthreads();
    }
}

template <int SUB>
cudaError_t launch_sub(const hj_image_t *images, const Tile *tiles, int n_tiles, cudaStream_t stream) {
    static bool configured = false;
    const int bytes = (int)sizeof(Smem<SUB>);
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(render_kernel<SUB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              bytes);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    render_kernel<SUB><<<n_tiles, kThreads, bytes, stream>>>(images, tiles);
    return cudaGetLastError();
}

}  // namespace

unsigned long long exact_block_count() {
    unsigned long long v = 0;
    cudaMemcpyFromSymbol(&v, g_exact_blocks, sizeof(v));
    return v;
}

size_t render_smem_bytes(int sub) {
    return sub == HJ_SUB_444 ? sizeof(Smem<HJ_SUB_444>)
         : sub == HJ_SUB_422 ? sizeof(Smem<HJ_SUB_422>) : sizeof(Smem<HJ_SUB_420>);
}

cudaError_t launch_render(int sub, bool /*direct is per image*/, const hj_image_t *images, const Tile *tiles,
                          int n_tiles, cudaStream_t stream) {
    if (n_tiles <= 0) return cudaSuccess;
    if (sub == HJ_SUB_444) return launch_sub<HJ_SUB_444>(images, tiles, n_tiles, stream);
    if (sub == HJ_SUB_422) return launch_sub<HJ_SUB_422>(images, tiles, n_tiles, stream);
    return launch_sub<HJ_SUB_420>(images, tiles, n_tiles, stream);
}

}  // namespace hj
