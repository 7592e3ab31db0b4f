// Per-block kernels behind the reference's single-block API
// (block_transforms.py / kernels/fallback.py:103-180): exact float64 IDCT of
// independent dequantised blocks, colour conversion of sample triples, and
// the single-row Algorithm 1 upsample.  Not on the render hot path.
#include <cstdint>

#include "hj_common.cuh"
#include "hj_render.cuh"

namespace hj {

namespace {

__constant__ double kPre64b[64] = HJ_PRESCALE_INIT;
__constant__ double kBasis64b[64] = HJ_BASIS_INIT;

template <bool DIRECT>
__global__ void idct_blocks_kernel(const int32_t *__restrict__ deq, int64_t n, uint8_t *__restrict__ out,
                                   double *__restrict__ out_f64) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= n) return;
    double g[64];
    const int32_t *src = deq + b * 64;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        double d[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            int v = src[r * 8 + c];
            d[r] = DIRECT ? i2d(v) : dmul(i2d(v), kPre64b[r * 8 + c]);
        }
        if (DIRECT) direct8(d, kBasis64b);
        else aan8(d[0], d[1], d[2], d[3], d[4], d[5], d[6], d[7]);
#pragma unroll
        for (int r = 0; r < 8; ++r) g[r * 8 + c] = d[r];
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        double *x = &g[r * 8];
        if (DIRECT) direct8(x, kBasis64b);
        else aan8(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7]);
    }
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
    bool special = false;
    Rgb p = colour(y[i], cb[i], cr[i], special);
    if (special) p.g = colour_g_exact(y[i], cb[i], cr[i]);
    uint32_t w = pack4(p.r, p.g, p.b, 0);
    rgb[3 * i] = (uint8_t)w;
    rgb[3 * i + 1] = (uint8_t)(w >> 8);
    rgb[3 * i + 2] = (uint8_t)(w >> 16);
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

// Packed coefficient transfer (hj_pack.h): expand one block per thread back
// into the dense int16 CoefficientBuffer layout (lossless).
template <bool WIDE>
__device__ __forceinline__ void unpack_one(uint64_t m, int dc, const uint8_t *__restrict__ v, uint32_t (&w)[32]) {
    int idx = 0;
#pragma unroll
    for (int k = 0; k < 64; k += 2) {
        int a = 0, c = 0;
        if (k == 0) {
            a = dc;
        } else if ((m >> k) & 1) {
            a = WIDE ? (int)*reinterpret_cast<const int16_t *>(v + 2 * idx) : (int)(int8_t)v[idx];
            ++idx;
        }
        if ((m >> (k + 1)) & 1) {
            c = WIDE ? (int)*reinterpret_cast<const int16_t *>(v + 2 * idx) : (int)(int8_t)v[idx];
            ++idx;
        }
        w[k >> 1] = (uint32_t)(uint16_t)a | ((uint32_t)(uint16_t)c << 16);
    }
}

// Records of `chunk` blocks at byte offsets tab[k] of `pack`: masks (8 B per
// block slot) | offsets (4) | DC (2) | values at rec_hdr.
__global__ void unpack_blocks_kernel(const uint8_t *__restrict__ pack, const uint64_t *__restrict__ tab,
                                     int64_t chunk, size_t rec_hdr, int64_t n, int16_t *__restrict__ out) {
    const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= n) return;
    const int64_t k = b / chunk, i = b - k * chunk;
    const uint8_t *rec = pack + tab[k];
    const uint64_t m = reinterpret_cast<const uint64_t *>(rec)[i];
    const uint32_t o = reinterpret_cast<const uint32_t *>(rec + chunk * 8)[i];
    const int dc = reinterpret_cast<const int16_t *>(rec + chunk * 12)[i];
    const uint8_t *v = rec + rec_hdr + (o & 0x7fffffffu);
    uint32_t w[32];
    if (o >> 31) unpack_one<true>(m, dc, v, w);
    else unpack_one<false>(m, dc, v, w);
    uint4 *d = reinterpret_cast<uint4 *>(out + b * 64);
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
}

}  // namespace

cudaError_t launch_upsample_422(const uint8_t *rows, const int16_t *left, const int16_t *right, int32_t *out,
                               int64_t n, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    upsample_422_kernel<<<(unsigned)((n + 127) / 128), 128, 0, stream>>>(rows, left, right, out, n);
    return cudaGetLastError();
}

cudaError_t launch_idct_blocks(const int32_t *deq, int64_t n, uint8_t *out, double *out_f64, bool direct,
                               cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    unsigned grid = (unsigned)((n + 127) / 128);
    if (direct) idct_blocks_kernel<true><<<grid, 128, 0, stream>>>(deq, n, out, out_f64);
    else idct_blocks_kernel<false><<<grid, 128, 0, stream>>>(deq, n, out, out_f64);
    return cudaGetLastError();
}

cudaError_t launch_ycbcr(const uint8_t *y, const uint8_t *cb, const uint8_t *cr, uint8_t *rgb, int64_t n,
                         cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    ycbcr_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(y, cb, cr, rgb, n);
    return cudaGetLastError();
}

}  // namespace hj

namespace hj {
cudaError_t launch_unpack_blocks(const uint8_t *pack, const uint64_t *tab, int64_t chunk, size_t rec_hdr, int64_t n,
                                 int16_t *out, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    const int t = 256;
    unpack_blocks_kernel<<<(unsigned)((n + t - 1) / t), t, 0, stream>>>(pack, tab, chunk, rec_hdr, n, out);
    return cudaGetLastError();
}
}  // namespace hj
