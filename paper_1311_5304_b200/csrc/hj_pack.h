// Packed coefficient transfer for the synchronous drop-in (render_rows):
// the host->device copy of a CoefficientBuffer region is PCIe-bound and the
// blocks are mostly zeros, so the host packs each 64-coefficient block into
//   mask[b]  uint64   bit k set <=> AC coefficient k (natural order) != 0
//   off[b]   uint32   byte offset of the block's values in `vals`; bit 31 set
//                     when they are int16 (any AC coefficient outside
//                     [-128, 127], offset 2-aligned), else int8
//   dc[b]    int16    the DC coefficient (often outside the int8 range)
//   vals     the nonzero AC coefficients in order
// and the device expands it back into the dense int16 layout before the
// render kernel runs (hj_blockops.cu unpack_blocks_kernel).  Lossless for
// every int16 input; 1080p q90: ~47 B instead of 128 B per block.
#pragma once

#include <cstddef>
#include <cstdint>

namespace hj {

// Worst-case bytes of `vals` for n blocks (+ slack for the vector stores).
inline size_t pack_vals_bound(int64_t n) { return (size_t)n * 130 + 128; }

// Pack n blocks; returns the bytes of `vals` written (offsets relative to
// `vals`, starting at `base`).  Uses AVX-512 (VBMI2) when the CPU has it.
size_t pack_blocks(const int16_t *src, int64_t n, uint64_t *mask, uint32_t *off, int16_t *dc, uint8_t *vals,
                   size_t base);

// Reference unpacker (host), for tests.
void unpack_blocks_host(const uint64_t *mask, const uint32_t *off, const int16_t *dc, const uint8_t *vals,
                        int64_t n, int16_t *dst);

// True when pack_blocks runs the AVX-512 path on this CPU.
bool pack_has_avx512();

}  // namespace hj
