// Host side of the packed coefficient transfer (hj_pack.h).
#include "hj_pack.h"

#include <cstdlib>
#include <cstring>
#include <immintrin.h>

namespace hj {

namespace {

inline bool in_i8(int v) { return v >= -128 && v <= 127; }

size_t pack_scalar(const int16_t *src, int64_t n, uint64_t *mask, uint32_t *off, int16_t *dc, uint8_t *vals,
                   size_t base) {
    size_t o = base;
    for (int64_t b = 0; b < n; ++b) {
        const int16_t *c = src + b * 64;
        uint64_t m = 0;
        bool wide = false;
        for (int k = 1; k < 64; ++k) {
            if (c[k]) m |= 1ull << k;
            wide |= !in_i8(c[k]);
        }
        if (wide) o = (o + 1) & ~(size_t)1;
        mask[b] = m;
        dc[b] = c[0];
        off[b] = (uint32_t)o | (wide ? 0x80000000u : 0u);
        for (int k = 1; k < 64; ++k) {
            if (!c[k]) continue;
            if (wide) {
                std::memcpy(vals + (o - base), &c[k], 2);
                o += 2;
            } else {
                vals[o - base] = (uint8_t)(int8_t)c[k];
                o += 1;
            }
        }
    }
    return o - base;
}

__attribute__((target("avx512f,avx512bw,avx512vl,avx512vbmi2,popcnt"))) size_t
pack_avx512(const int16_t *src, int64_t n, uint64_t *mask, uint32_t *off, int16_t *dc, uint8_t *vals, size_t base) {
    size_t o = base;
    const __m512i k128 = _mm512_set1_epi16(128), k255 = _mm512_set1_epi16(255);
    for (int64_t b = 0; b < n; ++b) {
        const __m512i v0 = _mm512_loadu_si512(src + b * 64);
        const __m512i v1 = _mm512_loadu_si512(src + b * 64 + 32);
        // AC only: the DC coefficient travels separately as int16
        const __mmask32 m0 = _mm512_test_epi16_mask(v0, v0) & ~1u, m1 = _mm512_test_epi16_mask(v1, v1);
        // outside [-128, 127] <=> (c + 128) as u16 > 255
        const __mmask32 w = (_mm512_cmpgt_epu16_mask(_mm512_add_epi16(v0, k128), k255) & ~1u) |
                            _mm512_cmpgt_epu16_mask(_mm512_add_epi16(v1, k128), k255);
        dc[b] = src[b * 64];
        mask[b] = (uint64_t)m0 | ((uint64_t)m1 << 32);
        const unsigned p0 = (unsigned)_mm_popcnt_u32(m0), p1 = (unsigned)_mm_popcnt_u32(m1);
        if (!w) {
            off[b] = (uint32_t)o;
            uint8_t *d = vals + (o - base);
            _mm256_storeu_si256(reinterpret_cast<__m256i *>(d), _mm512_cvtepi16_epi8(_mm512_maskz_compress_epi16(m0, v0)));
            _mm256_storeu_si256(reinterpret_cast<__m256i *>(d + p0),
                                _mm512_cvtepi16_epi8(_mm512_maskz_compress_epi16(m1, v1)));
            o += p0 + p1;
        } else {
            o = (o + 1) & ~(size_t)1;
            off[b] = (uint32_t)o | 0x80000000u;
            uint8_t *d = vals + (o - base);
            _mm512_storeu_si512(d, _mm512_maskz_compress_epi16(m0, v0));
            _mm512_storeu_si512(d + 2 * p0, _mm512_maskz_compress_epi16(m1, v1));
            o += 2 * (p0 + p1);
        }
    }
    return o - base;
}

}  // namespace

bool pack_has_avx512() {
    // HJ_PACK_SCALAR=1 forces the portable path (tests)
    static const bool has = [] {
        const char *v = std::getenv("HJ_PACK_SCALAR");
        if (v && v[0] && v[0] != '0') return false;
        return __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
               __builtin_cpu_supports("avx512vl") && __builtin_cpu_supports("avx512vbmi2");
    }();
    return has;
}

size_t pack_blocks(const int16_t *src, int64_t n, uint64_t *mask, uint32_t *off, int16_t *dc, uint8_t *vals,
                   size_t base) {
    return pack_has_avx512() ? pack_avx512(src, n, mask, off, dc, vals, base)
                             : pack_scalar(src, n, mask, off, dc, vals, base);
}

void unpack_blocks_host(const uint64_t *mask, const uint32_t *off, const int16_t *dc, const uint8_t *vals,
                        int64_t n, int16_t *dst) {
    for (int64_t b = 0; b < n; ++b) {
        const bool wide = (off[b] & 0x80000000u) != 0;
        size_t o = off[b] & 0x7fffffffu;
        dst[b * 64] = dc[b];
        for (int k = 1; k < 64; ++k) {
            int16_t v = 0;
            if ((mask[b] >> k) & 1) {
                if (wide) {
                    std::memcpy(&v, vals + o, 2);
                    o += 2;
                } else {
                    v = (int8_t)vals[o++];
                }
            }
            dst[b * 64 + k] = v;
        }
    }
}

}  // namespace hj
