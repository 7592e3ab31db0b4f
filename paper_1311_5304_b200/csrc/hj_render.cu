// sm_100a kernels for the hetjpeg parallel phase:
//   dequantise -> IDCT -> [h2v1 / h2v2 fancy upsample] -> YCbCr->RGB.
//
// Bit-exactness contract: the IDCT reproduces the reference's float64
// operation sequence (kernels/_native.pyx:321-388, fallback.py:67-100)
// with explicitly-rounded __dadd_rn/__dmul_rn (no FMA contraction), and the
// colour conversion uses integer formulas proven equal to the reference's
// float64 rounding over all 2^24 inputs (tools/gen_constants.py).
//
// Work decomposition: one CTA of 128 threads owns a
// strip of MCU columns of one image and sweeps down a range of MCU rows.
// Each sweep step
//   (1) IDCTs one MCU row of the strip, one 8x8 block per thread, entirely
//       in registers (no transposes), into u8 sample planes in shared memory;
//       4:2:2/4:2:0 also transform the chroma blocks of the MCU to the left
//       and right of the strip (horizontal filter context), and 4:2:0 keeps a
//       3-MCU-row chroma ring so the vertical context is transformed once;
//   (2) upsamples + colour-converts from shared memory and stores
//       interleaved RGB8 with 8-byte vector stores.
#include <cstdint>

#include "hj_render.cuh"
#include "hj_tables.h"

namespace hj {

namespace {

__constant__ double kPre[64] = HJ_PRESCALE_INIT;
__constant__ double kBasis[64] = HJ_BASIS_INIT;

// ---------------------------------------------------------------- float64

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// Exact int32 -> float64 without the (quarter-rate) I2F.F64 conversion:
// as_double(0x43300000 : x ^ 0x80000000) == 2^52 + 2^31 + x.
__device__ __forceinline__ double i2d(int x) {
    return dsub(__hiloint2double(0x43300000, x ^ (int)0x80000000), 4503601774854144.0);
}

// _round_u8(s + 128.0) (_native.pyx:312-318, 388): floor(fl(fl(s+128)+0.5))
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
__device__ __forceinline__ void aan8(double &x0, double &x1, double &x2, double &x3,
                                     double &x4, double &x5, double &x6, double &x7) {
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
// accumulated from 0.0 in ascending r.
__device__ __forceinline__ void direct8(double *x) {
    double y[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        double acc = 0.0;
#pragma unroll
        for (int r = 0; r < 8; ++r) acc = dadd(acc, dmul(kBasis[r * 8 + k], x[r]));
        y[k] = acc;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = y[k];
}

__device__ __forceinline__ int coef_at(const int4 (&raw)[8], int r, int c) {
    int w = (c >> 1) == 0 ? raw[r].x : (c >> 1) == 1 ? raw[r].y : (c >> 1) == 2 ? raw[r].z : raw[r].w;
    return (c & 1) ? (w >> 16) : (int)(short)(w & 0xffff);
}

// Shared-memory int4 load that the compiler may not hoist out of the
// block loop (a hoisted q table would pin 64 registers for the whole sweep).
__device__ __forceinline__ int4 lds128_volatile(const int *p) {
    int4 v;
    unsigned a = (unsigned)__cvta_generic_to_shared(p);
    asm volatile("ld.shared.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}

// Pre-rounding float64 core of one block of dequantised coefficients
// dq[64] (natural order).  Result in g[64].
template <bool DIRECT>
__device__ __forceinline__ void idct_core(const int (&dq)[64], double (&g)[64]) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        double d[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            int v = dq[r * 8 + c];
            d[r] = DIRECT ? i2d(v) : dmul(i2d(v), kPre[r * 8 + c]);
        }
        if (DIRECT) {
            direct8(d);
        } else {
            aan8(d[0], d[1], d[2], d[3], d[4], d[5], d[6], d[7]);
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) g[r * 8 + c] = d[r];
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        double *x = &g[r * 8];
        if (DIRECT) {
            direct8(x);
        } else {
            aan8(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7]);
        }
    }
}

// Dequantise + IDCT + round one block (global) into an 8x8 window of a u8
// plane in shared memory (row stride `stride`, 8-byte aligned).
template <bool DIRECT>
__device__ __noinline__ void idct_block(const int16_t *__restrict__ src, const int *q,
                                           uint8_t *dst, int stride) {
    int4 raw[8];
    const int4 *s4 = reinterpret_cast<const int4 *>(src);
#pragma unroll
    for (int r = 0; r < 8; ++r) raw[r] = __ldg(s4 + r);
    int dq[64];  // dequantise: int16 coefficient * qtable entry (fallback.py:194-195)
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        int4 q0 = lds128_volatile(q + r * 8), q1 = lds128_volatile(q + r * 8 + 4);
        const int qa[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
        for (int c = 0; c < 8; ++c) dq[r * 8 + c] = coef_at(raw, r, c) * qa[c];
    }
    double g[64];
    idct_core<DIRECT>(dq, g);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        uint32_t lo = 0, hi = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) lo |= (uint32_t)round_sample(g[r * 8 + c]) << (8 * c);
#pragma unroll
        for (int c = 0; c < 4; ++c) hi |= (uint32_t)round_sample(g[r * 8 + 4 + c]) << (8 * c);
        *reinterpret_cast<uint2 *>(dst + r * stride) = make_uint2(lo, hi);
    }
}

// ---------------------------------------------------------------- colour

// Integer forms of _color_px (_native.pyx:391-395), exhaustively verified
// (tools/gen_constants.py colour_constants).  Returns 0x00BBGGRR.
__device__ __forceinline__ uint32_t colour(int y, int cb, int cr) {
    int yk = y << HJ_COL_K;
    int r = (yk + HJ_COL_AR * cr + HJ_COL_CR) >> HJ_COL_K;
    int g = (yk + HJ_COL_AGB * cb + HJ_COL_AGR * cr + HJ_COL_CG) >> HJ_COL_K;
    int b = (yk + HJ_COL_AB * cb + HJ_COL_CB) >> HJ_COL_K;
    // the one float64 tie whose offset depends on Y
    if (cb == 78 && cr == 178 && (unsigned)(y - 47) <= 35u) g -= 1;
    r = min(max(r, 0), 255);
    g = min(max(g, 0), 255);
    b = min(max(b, 0), 255);
    return (uint32_t)r | ((uint32_t)g << 8) | ((uint32_t)b << 16);
}

// Store 8 pixels (packed 0x00BBGGRR each) as 24 interleaved bytes at
// rgb + off, cropping to `npx` pixels.
__device__ __forceinline__ void store8(uint8_t *__restrict__ dst, const uint32_t (&px)[8], int npx) {
    uint32_t w[6];
    w[0] = px[0] | (px[1] << 24);
    w[1] = (px[1] >> 8) | (px[2] << 16);
    w[2] = (px[2] >> 16) | (px[3] << 8);
    w[3] = px[4] | (px[5] << 24);
    w[4] = (px[5] >> 8) | (px[6] << 16);
    w[5] = (px[6] >> 16) | (px[7] << 8);
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
        for (int i = 0; i < npx * 3; ++i) dst[i] = (uint8_t)(w[i >> 2] >> (8 * (i & 3)));
    }
}

// ---------------------------------------------------------------- kernel

template <int SUB>
struct Geo;
template <>
struct Geo<HJ_SUB_444> {
    static constexpr int S = kStrip444, YPM = 1, MW = 8, MH = 8;
    static constexpr int YW = 8 * S, CW = 8 * S, CROWS = 8;
};
template <>
struct Geo<HJ_SUB_422> {
    static constexpr int S = kStrip422, YPM = 2, MW = 16, MH = 8;
    static constexpr int YW = 16 * S, CW = 8 * (S + 2), CROWS = 8;
};
template <>
struct Geo<HJ_SUB_420> {
    static constexpr int S = kStrip420, YPM = 4, MW = 16, MH = 16;
    static constexpr int YW = 16 * S, CW = 8 * (S + 2), CROWS = 24;  // 3-row ring
};

template <int SUB, bool DIRECT>
__global__ void __launch_bounds__(kThreads, 2)
render_kernel(const hj_image_t *__restrict__ images, const Tile *__restrict__ tiles) {
    using G = Geo<SUB>;
    __shared__ __align__(16) uint8_t ys[G::MH * G::YW];
    __shared__ __align__(16) uint8_t cbs[G::CROWS * G::CW];
    __shared__ __align__(16) uint8_t crs[G::CROWS * G::CW];
    __shared__ __align__(16) int qs[3 * 64];

    const Tile t = tiles[blockIdx.x];
    const hj_image_t im = images[t.image];
    const int tid = threadIdx.x;
    const int mpr = im.mcus_per_row;
    const int S = t.m1 - t.m0;
    for (int i = tid; i < 192; i += kThreads) qs[i] = im.q[i];

    // chroma MCU window of the strip: [m0-1, m1+1) for 4:2:2/4:2:0
    const int cm_lo = (SUB == HJ_SUB_444) ? t.m0 : t.m0 - 1;
    const int n_cm = (SUB == HJ_SUB_444) ? S : S + 2;
    __syncthreads();

    // Resolve chroma job j of MCU row `row` (j in [0, 2*n_cm): component
    // j / n_cm, window MCU j % n_cm) to its source block and plane window.
    auto chroma_job = [&](int row, int slot, int j, const int16_t *&src, const int *&q,
                          uint8_t *&dst) -> bool {
        int comp = j / n_cm, lm = j - comp * n_cm;
        int m = cm_lo + lm;
        if (m < 0 || m >= mpr) return false;
        src = (comp == 0 ? im.cb : im.cr) + ((int64_t)row * mpr + m) * 64;
        q = qs + 64 * (1 + comp);
        dst = (comp == 0 ? cbs : crs) + slot * 8 * G::CW + lm * 8;
        return true;
    };

    if (SUB == HJ_SUB_420) {
        // prime the ring with MCU rows r0-1 (if any) and r0
        int pre_lo = t.r0 > 0 ? t.r0 - 1 : t.r0;
        int n_pre = (t.r0 - pre_lo + 1) * 2 * n_cm;
#pragma unroll 1
        for (int j = tid; j < n_pre; j += kThreads) {
            int rr = pre_lo + j / (2 * n_cm);
            const int16_t *src;
            const int *q;
            uint8_t *dst;
            if (chroma_job(rr, rr % 3, j % (2 * n_cm), src, q, dst)) idct_block<DIRECT>(src, q, dst, G::CW);
        }
    }

#pragma unroll 1
    for (int row = t.r0; row < t.r1; ++row) {
        // ---- (1) transforms of this step
        const int n_y = G::YPM * S;
        int n_c = 0, c_row = row;
        if (SUB == HJ_SUB_420) {
            c_row = row + 1;
            n_c = (c_row < im.mcu_rows) ? 2 * n_cm : 0;
        } else {
            n_c = 2 * n_cm;
        }
#pragma unroll 1
        for (int j = tid; j < n_y + n_c; j += kThreads) {
            const int16_t *src;
            const int *q;
            uint8_t *dst;
            int stride;
            if (j < n_y) {
                int lm = j / G::YPM, b = j - lm * G::YPM;
                int64_t blk = ((int64_t)row * mpr + t.m0 + lm) * G::YPM + b;
                // Y block b of the MCU: 4:2:2 left/right, 4:2:0 raster 2x2
                int bx = (G::YPM == 1) ? 0 : (b & 1), by = (G::YPM == 4) ? (b >> 1) : 0;
                src = im.y + blk * 64;
                q = qs;
                dst = ys + by * 8 * G::YW + (lm * (G::MW / 8) + bx) * 8;
                stride = G::YW;
            } else {
                if (!chroma_job(c_row, SUB == HJ_SUB_420 ? c_row % 3 : 0, j - n_y, src, q, dst)) continue;
                stride = G::CW;
            }
            idct_block<DIRECT>(src, q, dst, stride);
        }
        __syncthreads();

        // ---- (2) upsample + colour + store
        const int y_base = row * G::MH;
        const int n_groups = (G::MW / 8) * S;  // 8-pixel groups per pixel row
        const int x_base = t.m0 * G::MW;
        const int cw_img = 8 * mpr;            // padded chroma plane width
#pragma unroll 1
        for (int it = tid; it < G::MH * n_groups; it += kThreads) {
            int oy = it / n_groups, gx = it - oy * n_groups;
            int y = y_base + oy;
            int x0 = x_base + gx * 8;
            int npx = min(8, im.width - x0);
            if (y >= im.height || npx <= 0) continue;
            const uint8_t *yrow = ys + oy * G::YW + gx * 8;
            uint32_t px[8];
            if (SUB == HJ_SUB_444) {
                const uint8_t *cbr = cbs + oy * G::CW + gx * 8;
                const uint8_t *crr = crs + oy * G::CW + gx * 8;
#pragma unroll
                for (int i = 0; i < 8; ++i) px[i] = colour(yrow[i], cbr[i], crr[i]);
            } else {
                // chroma samples k0-1 .. k0+4 of this group, clamped to the
                // padded plane (edge copy), as window-local columns
                const int k0 = 8 * t.m0 + 4 * gx;
                int cb_s[6], cr_s[6];
                if (SUB == HJ_SUB_422) {
                    const uint8_t *cbr = cbs + oy * G::CW;
                    const uint8_t *crr = crs + oy * G::CW;
#pragma unroll
                    for (int i = 0; i < 6; ++i) {
                        int k = min(max(k0 - 1 + i, 0), cw_img - 1) - 8 * cm_lo;
                        cb_s[i] = cbr[k];
                        cr_s[i] = crr[k];
                    }
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        int cb3 = 3 * cb_s[i + 1], cr3 = 3 * cr_s[i + 1];
                        px[2 * i] = colour(yrow[2 * i], (cb3 + cb_s[i] + 1) >> 2, (cr3 + cr_s[i] + 1) >> 2);
                        px[2 * i + 1] = colour(yrow[2 * i + 1], (cb3 + cb_s[i + 2] + 2) >> 2,
                                               (cr3 + cr_s[i + 2] + 2) >> 2);
                    }
                } else {
                    const int ch_img = 8 * im.mcu_rows;
                    int ci = 8 * row + (oy >> 1);
                    int cf = min(max(ci + ((oy & 1) ? 1 : -1), 0), ch_img - 1);
                    const int on = ((ci >> 3) % 3) * 8 + (ci & 7);
                    const int of = ((cf >> 3) % 3) * 8 + (cf & 7);
                    const uint8_t *cbn = cbs + on * G::CW, *cbf = cbs + of * G::CW;
                    const uint8_t *crn = crs + on * G::CW, *crf = crs + of * G::CW;
#pragma unroll
                    for (int i = 0; i < 6; ++i) {
                        int k = min(max(k0 - 1 + i, 0), cw_img - 1) - 8 * cm_lo;
                        cb_s[i] = 3 * cbn[k] + cbf[k];
                        cr_s[i] = 3 * crn[k] + crf[k];
                    }
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        int cb3 = 3 * cb_s[i + 1], cr3 = 3 * cr_s[i + 1];
                        px[2 * i] = colour(yrow[2 * i], (cb3 + cb_s[i] + 8) >> 4, (cr3 + cr_s[i] + 8) >> 4);
                        px[2 * i + 1] = colour(yrow[2 * i + 1], (cb3 + cb_s[i + 2] + 7) >> 4,
                                               (cr3 + cr_s[i + 2] + 7) >> 4);
                    }
                }
            }
            store8(im.rgb + ((int64_t)y * im.width + x0) * 3, px, npx);
        }
        __syncthreads();
    }
}

// ------------------------------------------------------- per-block kernels

template <bool DIRECT>
__global__ void idct_blocks_kernel(const int32_t *__restrict__ deq, int64_t n,
                                   uint8_t *__restrict__ out, double *__restrict__ out_f64) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= n) return;
    // reuse the block core with q == 1 over the int32 input split in halves:
    // the dequantised product is passed through an int4 view per row.
    int dq[64];
    const int4 *src = reinterpret_cast<const int4 *>(deq + b * 64);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        int4 v = src[i];
        dq[4 * i] = v.x;
        dq[4 * i + 1] = v.y;
        dq[4 * i + 2] = v.z;
        dq[4 * i + 3] = v.w;
    }
    double g[64];
    idct_core<DIRECT>(dq, g);
    if (out_f64) {
#pragma unroll
        for (int i = 0; i < 64; ++i) out_f64[b * 64 + i] = g[i];
    } else {
#pragma unroll
        for (int i = 0; i < 64; ++i) out[b * 64 + i] = (uint8_t)round_sample(g[i]);
    }
}

__global__ void ycbcr_kernel(const uint8_t *__restrict__ y, const uint8_t *__restrict__ cb,
                             const uint8_t *__restrict__ cr, uint8_t *__restrict__ rgb, int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t p = colour(y[i], cb[i], cr[i]);
    rgb[3 * i] = (uint8_t)p;
    rgb[3 * i + 1] = (uint8_t)(p >> 8);
    rgb[3 * i + 2] = (uint8_t)(p >> 16);
}

// Algorithm 1 on one 8-sample row, floor division:
// out[2k] = (3s[k] + s[k-1] + 1) / 4, out[2k+1] = (3s[k] + s[k+1] + 2) / 4,
// with the end samples copied unless a neighbour is given.
__global__ void upsample_422_kernel(const uint8_t *__restrict__ rows, const int16_t *__restrict__ left,
                                    const int16_t *__restrict__ right, int32_t *__restrict__ out, int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int s[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) s[k] = rows[i * 8 + k];
    int32_t *o = out + i * 16;
    int l = left[i], r = right[i];
    o[0] = l < 0 ? s[0] : (3 * s[0] + l + 1) >> 2;
#pragma unroll
    for (int k = 1; k < 8; ++k) o[2 * k] = (3 * s[k] + s[k - 1] + 1) >> 2;
#pragma unroll
    for (int k = 0; k < 7; ++k) o[2 * k + 1] = (3 * s[k] + s[k + 1] + 2) >> 2;
    o[15] = r < 0 ? s[7] : (3 * s[7] + r + 2) >> 2;
}

}  // namespace

cudaError_t launch_upsample_422(const uint8_t *rows, const int16_t *left, const int16_t *right,
                               int32_t *out, int64_t n, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    upsample_422_kernel<<<(unsigned)((n + 127) / 128), 128, 0, stream>>>(rows, left, right, out, n);
    return cudaGetLastError();
}

cudaError_t launch_render(int sub, bool direct, const hj_image_t *images, const Tile *tiles,
                          int n_tiles, cudaStream_t stream) {
    if (n_tiles <= 0) return cudaSuccess;
    dim3 grid(n_tiles), block(kThreads);
#define HJ_LAUNCH(S, D) render_kernel<S, D><<<grid, block, 0, stream>>>(images, tiles)
    if (sub == HJ_SUB_444) {
        if (direct) HJ_LAUNCH(HJ_SUB_444, true); else HJ_LAUNCH(HJ_SUB_444, false);
    } else if (sub == HJ_SUB_422) {
        if (direct) HJ_LAUNCH(HJ_SUB_422, true); else HJ_LAUNCH(HJ_SUB_422, false);
    } else {
        if (direct) HJ_LAUNCH(HJ_SUB_420, true); else HJ_LAUNCH(HJ_SUB_420, false);
    }
#undef HJ_LAUNCH
    return cudaGetLastError();
}

cudaError_t launch_idct_blocks(const int32_t *deq, int64_t n, uint8_t *out, double *out_f64,
                               bool direct, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    int64_t grid = (n + 127) / 128;
    if (direct) idct_blocks_kernel<true><<<(unsigned)grid, 128, 0, stream>>>(deq, n, out, out_f64);
    else idct_blocks_kernel<false><<<(unsigned)grid, 128, 0, stream>>>(deq, n, out, out_f64);
    return cudaGetLastError();
}

cudaError_t launch_ycbcr(const uint8_t *y, const uint8_t *cb, const uint8_t *cr, uint8_t *rgb,
                         int64_t n, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    int64_t grid = (n + 255) / 256;
    ycbcr_kernel<<<(unsigned)grid, 256, 0, stream>>>(y, cb, cr, rgb, n);
    return cudaGetLastError();
}

}  // namespace hj
