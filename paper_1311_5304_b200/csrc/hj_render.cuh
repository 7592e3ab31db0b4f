// Internal interface between the C-ABI host layer (hj_api.cu) and the
// sm_100a render kernels (hj_render.cu).  Not part of the public ABI.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/hetjpeg_b200.h"

namespace hj {

// A CTA's work unit: one vertical strip of MCU columns [m0, m1) of one
// image, swept over MCU rows [r0, r1).  The sweep carries the chroma rows
// of the previous MCU row (4:2:0 vertical context) in shared memory.
struct Tile {
    int32_t image;
    int32_t m0, m1;
    int32_t r0, r1;
    int32_t pad[3];
};
static_assert(sizeof(Tile) == 32, "Tile layout");

// CTA size and residency: small CTAs sweep their strips independently, so
// barrier waits stay local to a strip.  4:2:0 uses 4-warp CTAs (its wider
// per-step pixel work balances the float64 fallback better), 4:4:4 / 4:2:2
// 2-warp CTAs.  CTAs per SM (launch bounds): 4:4:4 and 4:2:2 run 8 CTAs and
// 4:2:0 4 CTAs (16 warps, 128 registers; 4:2:x chroma is stored as 2-byte
// pairs to fit; 4:2:2 with the row-pair screen, hj_render.cu kScreenCols).
// Measured: tools/experiments/README.md.
#ifndef HJ_THREADS_420
#define HJ_THREADS_420 128
#endif
#ifndef HJ_THREADS_422
#define HJ_THREADS_422 64
#endif
#ifndef HJ_THREADS
#define HJ_THREADS 64
#endif
constexpr int threads_for(int sub) {
    return sub == HJ_SUB_420 ? HJ_THREADS_420 : sub == HJ_SUB_422 ? HJ_THREADS_422 : HJ_THREADS;
}
#ifndef HJ_CTAS_444
#define HJ_CTAS_444 8
#endif
#ifndef HJ_CTAS_422
#define HJ_CTAS_422 8
#endif
#ifndef HJ_CTAS_420
#define HJ_CTAS_420 4
#endif
constexpr int ctas_per_sm(int sub) {
    return sub == HJ_SUB_444 ? HJ_CTAS_444 : sub == HJ_SUB_422 ? HJ_CTAS_422 : HJ_CTAS_420;
}
// Strip widths (MCUs per CTA) so one sweep step has ~threads two-block jobs:
// 444 -> ceil(S/2) + S, 422 -> S + (S+2), 420 -> 2S + (S+2).
constexpr int strip_for(int sub) {
    return sub == HJ_SUB_444 ? ((2 * threads_for(sub)) / 3) & ~1   // even: 16-byte plane rows
         : sub == HJ_SUB_422 ? (threads_for(sub) - 2) / 2
                             : (threads_for(sub) - 2) / 3;
}
constexpr int kStrip444 = strip_for(HJ_SUB_444);
constexpr int kStrip422 = strip_for(HJ_SUB_422);
constexpr int kStrip420 = strip_for(HJ_SUB_420);

inline int strip_width(int sub) {
    return sub == HJ_SUB_444 ? kStrip444 : sub == HJ_SUB_422 ? kStrip422 : kStrip420;
}

// Decode modes of the render kernel: the reference's float64 arithmetic
// (AAN "fast" or "direct" per image flag) or libjpeg's integer "islow".
// kModeRefTc: the reference's arithmetic with the IDCT screen on the tensor
// cores (render_tc_kernel, v4); kModeRef keeps the FP32-screen kernel (v3),
// used for "direct" images and chroma tables that differ between Cb and Cr.
enum { kModeRef = 0, kModeIslow = 1, kModeRefTc = 2 };

// Tensor-core kernel geometry: 256-thread CTAs, 2 per SM (TMEM), strips of
// 96 / 64 / 48 MCUs for 4:4:4 / 4:2:2 / 4:2:0.
constexpr int kTcThreads = 256;
constexpr int kTcCtasPerSm = 2;
constexpr int tc_strip(int sub) { return sub == HJ_SUB_444 ? 96 : sub == HJ_SUB_422 ? 64 : 48; }

// Plan group kinds (hj_api.cu): the IDCT path an image takes.
enum { kKindTc = 0, kKindDirect = 1, kKindIslow = 2, kKindSimt = 3 };
inline int mode_of_kind(int kind) {
    return kind == kKindTc ? kModeRefTc : kind == kKindIslow ? kModeIslow : kModeRef;
}

// Launch the render kernel for `n_tiles` tiles of one subsampling family.
// `images` and `tiles` are device arrays.
cudaError_t launch_render(int subsampling, int mode, const hj_image_t *images,
                          const Tile *tiles, int n_tiles, cudaStream_t stream);

// Blocks the FP32 screen sent to the exact float64 path, all launches so far.
unsigned long long exact_block_count();
// Tensor-core screen kernel launches so far.
unsigned long long tc_launch_count();

// Single-block transforms (reference per-block API).
cudaError_t launch_idct_blocks(const int32_t *deq, int64_t n, uint8_t *out, double *out_f64,
                               bool direct, cudaStream_t stream);
cudaError_t launch_upsample_422(const uint8_t *rows, const int16_t *left, const int16_t *right,
                               int32_t *out, int64_t n, cudaStream_t stream);
// Packed coefficient transfer (hj_pack.h): dense int16 blocks from records of
// `chunk` blocks (masks | offsets | DC | values at rec_hdr) at offsets tab[k].
cudaError_t launch_unpack_blocks(const uint8_t *pack, const uint64_t *tab, int64_t chunk, size_t rec_hdr, int64_t n,
                                 int16_t *out, cudaStream_t stream);
cudaError_t launch_ycbcr(const uint8_t *y, const uint8_t *cb, const uint8_t *cr, uint8_t *rgb,
                         int64_t n, cudaStream_t stream);

}  // namespace hj
