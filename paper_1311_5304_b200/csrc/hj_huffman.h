// Host Huffman core shared by the whole-scan decoder and the resumable
// per-row cursor of the drop-in API (both in hj_huffman.cpp).
// Internal header, not part of the C ABI.
//
// Reader: a left-aligned 64-bit bit buffer topped up to >= 57 bits per
// refill (one big-endian 8-byte load when the next bytes hold no 0xFF),
// 0xFF00 unstuffing, and - like the reference's reader - no bits past a
// marker (kernels/_native.pyx:74-88).
//
// Decoding: 11-bit lookahead tables.  One lookup yields code length, run and
// the EXTENDed value when code + magnitude bits fit in 11 bits; otherwise the
// code alone (magnitude read from the buffer) or the canonical
// mincode/maxcode walk for codes longer than 11 bits.  Block semantics
// follow _native.pyx:141-184: DC category <= 15, predictor accumulated in
// 64 bits and wrapped to int16 on store, AC run/size with ZRL, any other
// size-0 symbol ends the block, run past coefficient 63 = bad code.
//
// Reference-equivalent reader state.  The reference loads bytes lazily
// (`_refill(need)`: a byte only while fewer than `need` bits are buffered;
// need = 8 for a Huffman lookahead, k for a k-bit take), so its position
// after a run of operations is the smallest byte count covering every
// operation's need: B = max_i ceil((C_i + need_i - bits0) / 8) data bytes
// past the origin (C_i = bits consumed before operation i, bits0 = bits
// buffered at the origin), capped where a marker stops the reader.  Only
// the last Huffman lookahead can reach past the consumed bits, so tracking
// `need_hi = C + 8` at each symbol is enough; a failed take means the
// reference read everything up to the stop.  `ref_state` converts this
// reader into the reference's {pos, bitbuf, bits} - the restart check
// (_native.pyx:238-257) and the int64[8] cursor write-back
// (_native.pyx:289-296) are then the reference's own.
#pragma once

#include <cstdint>
#include <cstring>

#include "../../include/hetjpeg_b200.h"
#include "hj_tables.h"

namespace hj {
namespace huff {

constexpr int kLook = 11;
#ifndef HJ_PAIR_LOOK
#define HJ_PAIR_LOOK 13
#endif
constexpr int kPairLook = HJ_PAIR_LOOK;  // lookahead of the two-symbol table

// fast[] entry: bits 0-15 value (int16), 16-19 run, 20-24 bits consumed
// (code + magnitude), 25-27 kind, 28-31 code length.
enum Kind : uint32_t { kSlow = 0, kCoef = 1, kEob = 2, kZrl = 3, kCodeOnly = 4 };

// pair[] entry (AC tables, whole-scan decoder): two consecutive AC
// coefficients whose codes and magnitudes both lie inside the 11-bit
// lookahead.  bits 0-9 value 1, 10-19 value 2 (signed; 0 = the second
// symbol is the block's EOB), 20-23 run 1, 24-27 run 2, 28-31 bits consumed
// by both (0 = no pair: fall back to fast[]).  (q90 symbols average ~5 bits
// with their magnitudes.)
struct Table {
    uint16_t look[1 << kLook];  // (len << 8) | symbol, len 0 = code longer than kLook
    uint32_t fast[1 << kLook];
    uint32_t pair[1 << kPairLook];
    int32_t mincode[17], maxcode[17], valptr[17];
    uint8_t symbols[256];
};

struct Tables {
    Table t[8];
    int comp_dc[3], comp_ac[3];
};

// Builds the lookahead tables of the slots a scan uses; false = a component
// names a slot outside 0..7.
bool build_tables(const hj_scan_tables_t *scan, Tables &out);

inline int extend(int v, int t) { return v < (1 << (t - 1)) ? v - ((1 << t) - 1) : v; }

extern const int kZigzag[64];

struct Reader {
    const uint8_t *org = nullptr, *p = nullptr, *end = nullptr;
    uint64_t acc = 0;     // next bit = bit 63
    int nbits = 0;
    int bits0 = 0;        // bits buffered at the origin
    int64_t loaded = 0;   // data bytes appended since the origin
    bool stopped = false; // a refill met a marker or the end of the data

    Reader() = default;
    Reader(const uint8_t *pos, const uint8_t *e, uint64_t buf = 0, int bits = 0)
        : org(pos), p(pos), end(e), acc(bits ? buf << (64 - bits) : 0), nbits(bits), bits0(bits) {}

    // bits consumed since the origin
    inline int64_t consumed() const { return 8 * loaded + bits0 - nbits; }

    inline void refill() {
        if (nbits <= 56 && end - p >= 8) {
            uint64_t w;
            std::memcpy(&w, p, 8);
            w = __builtin_bswap64(w);
            const int nb = (64 - nbits) >> 3;  // 1..8 whole bytes fit
            const uint64_t top = nb == 8 ? ~0ull : ~(~0ull >> (8 * nb));
            const uint64_t x = ~w & top;       // a 0xFF byte -> a zero byte of x
            const uint64_t has_ff = (x - 0x0101010101010101ull) & ~x & 0x8080808080808080ull & top;
            if (!has_ff) {
                acc |= (w & top) >> nbits;
                p += nb;
                loaded += nb;
                nbits += 8 * nb;
                return;
            }
        }
        while (nbits <= 56) {
            if (p >= end) {
                stopped = true;
                return;
            }
            const uint8_t b = *p;
            if (b == 0xFF) {
                if (p + 1 < end && p[1] == 0x00) {
                    p += 2;
                } else {
                    stopped = true;  // marker: stop delivering bits
                    return;
                }
            } else {
                ++p;
            }
            acc |= (uint64_t)b << (56 - nbits);
            nbits += 8;
            ++loaded;
        }
    }
    inline uint32_t peek(int n) const { return (uint32_t)(acc >> (64 - n)); }
    inline void skip(int n) {
        acc <<= n;
        nbits -= n;
    }
};

// Lazy-reader bookkeeping of one decode run (see the header comment).
struct Track {
    int64_t need_hi = 0;  // max over operations of C_i + need_i (relative to the origin)
    bool starved = false; // a take found too few bits: the reference read to the stop
};

// Generic symbol decode: lookahead table, then the canonical walk.  Bit
// consumption on every outcome equals the reference's _huffdecode
// (_native.pyx:105-132): a code is consumed whole; "no code within 16
// bits" consumes 16 bits; running out mid-walk consumes the bits taken.
template <bool kTrack>
inline int decode_sym(Reader &br, const Table &t, int &err, Track *tr) {
    if (br.nbits < 16) br.refill();
    if (br.nbits >= 1) {
        const uint16_t e = t.look[br.peek(kLook)];  // bits past nbits read as 0:
        const int len = e >> 8;                      // only codes within nbits count
        if (len != 0 && len <= br.nbits) {
            br.skip(len);
            return e & 0xff;
        }
    }
    if (br.nbits >= 16) {
        for (int l = kLook + 1; l < 17; ++l) {
            const int code = (int)br.peek(l);
            if (t.maxcode[l] >= 0 && code <= t.maxcode[l]) {
                br.skip(l);
                return t.symbols[t.valptr[l] + code - t.mincode[l]];
            }
        }
        br.skip(16);
        err = HJ_ERR_BADCODE;
        return 0;
    }
    // fewer than 16 bits before a marker / the end: bit by bit
    int code = 0;
    for (int l = 1; l < 17; ++l) {
        if (br.nbits < 1) {
            if (kTrack) tr->starved = true;
            err = HJ_ERR_EXHAUSTED;
            return 0;
        }
        code = (code << 1) | (int)br.peek(1);
        br.skip(1);
        if (t.maxcode[l] >= 0 && code <= t.maxcode[l]) return t.symbols[t.valptr[l] + code - t.mincode[l]];
    }
    err = HJ_ERR_BADCODE;
    return 0;
}

// k-bit take (k <= 16); false = exhausted (nothing consumed).
template <bool kTrack>
inline bool take(Reader &br, int k, int &v, Track *tr) {
    if (br.nbits < k) br.refill();
    if (br.nbits < k) {
        if (kTrack) tr->starved = true;
        return false;
    }
    v = (int)br.peek(k);
    br.skip(k);
    return true;
}

// One block.  kZero: clear the 64 outputs first (whole-scan decoder; the
// drop-in cursor writes only decoded positions, like the reference).
// kTrack: keep the lazy-reader bookkeeping (Track) for ref_state.
template <bool kZero, bool kTrack>
inline int decode_block(Reader &br, const Table &dc, const Table &ac, int16_t *out, int64_t &pred, Track *tr) {
    if (kZero) std::memset(out, 0, 64 * sizeof(int16_t));
    int err = HJ_OK;
    int diff = 0;
    if (br.nbits < 32) br.refill();
    if (kTrack) tr->need_hi = br.consumed() + 8;
    const uint32_t de = br.nbits >= 32 ? dc.fast[br.peek(kLook)] : 0u;
    const uint32_t dkind = (de >> 25) & 7;
    if (dkind == kCoef) {
        br.skip((de >> 20) & 31);
        diff = (int16_t)(de & 0xffff);
    } else if (dkind == kCodeOnly) {
        const int t = de & 0xff;  // 1..15; >= 16 buffered bits remain
        br.skip((de >> 20) & 31);
        diff = extend((int)br.peek(t), t);
        br.skip(t);
    } else {
        const int t = decode_sym<kTrack>(br, dc, err, tr);
        if (err) return err;
        if (t > 15) return HJ_ERR_BADCODE;
        if (t) {
            int v;
            if (!take<kTrack>(br, t, v, tr)) return HJ_ERR_EXHAUSTED;
            diff = extend(v, t);
        }
    }
    pred += diff;
    out[0] = (int16_t)pred;
    int k = 1;
    while (k < 64) {
        if (br.nbits < 32) br.refill();
        if (kTrack) tr->need_hi = br.consumed() + 8;
        if (!kTrack && br.nbits >= kPairLook) {
            // two coefficients per lookup when both fit the lookahead and
            // stay inside the block (else the single-symbol path below,
            // which also reports any error exactly)
            const uint32_t pe = ac.pair[br.peek(kPairLook)];
            const int r1 = (int)(pe >> 20) & 15, r2 = (int)(pe >> 24) & 15;
            const int v2 = (int32_t)(pe << 12) >> 22;
            // (an EOB pair needs room after its coefficient: a block whose
            // coefficient 63 is coded ends there without an EOB)
            if ((pe >> 28) != 0 && k + r1 + (v2 ? r2 + 1 : 1) <= 63) {
                br.skip((int)(pe >> 28));
                k += r1;
                out[kZigzag[k]] = (int16_t)((int32_t)(pe << 22) >> 22);
                if (!v2) break;  // coefficient + EOB
                k += 1 + r2;
                out[kZigzag[k]] = (int16_t)v2;
                ++k;
                continue;
            }
        }
        if (br.nbits >= kLook) {
            const uint32_t e = ac.fast[br.peek(kLook)];
            const uint32_t kind = (e >> 25) & 7;
            if (kind == kCoef) {
                const int run = (e >> 16) & 15;
                if (k + run > 63) {
                    br.skip(e >> 28);  // the code is consumed, the magnitude is not
                    return HJ_ERR_BADCODE;
                }
                br.skip((e >> 20) & 31);
                k += run;
                out[kZigzag[k]] = (int16_t)(e & 0xffff);
                ++k;
                continue;
            }
            if (kind == kEob) {
                br.skip((e >> 20) & 31);
                break;
            }
            if (kind == kZrl) {
                br.skip((e >> 20) & 31);
                k += 16;
                continue;
            }
            if (kind == kCodeOnly && br.nbits >= 32) {
                const int r = (e >> 4) & 15, sz = e & 15;
                br.skip((e >> 20) & 31);
                k += r;
                if (k > 63) return HJ_ERR_BADCODE;
                out[kZigzag[k]] = (int16_t)extend((int)br.peek(sz), sz);
                br.skip(sz);
                ++k;
                continue;
            }
        }
        const int rs = decode_sym<kTrack>(br, ac, err, tr);
        if (err) return err;
        const int r = rs >> 4, s = rs & 15;
        if (s == 0) {
            if (r == 15) {
                k += 16;
                continue;
            }
            break;
        }
        k += r;
        if (k > 63) return HJ_ERR_BADCODE;
        int v;
        if (!take<kTrack>(br, s, v, tr)) {
            // the reference stores EXTEND of the failed take's 0 before it
            // checks the error (_native.pyx:180-182)
            out[kZigzag[k]] = (int16_t)extend(0, s);
            return HJ_ERR_EXHAUSTED;
        }
        out[kZigzag[k]] = (int16_t)extend(v, s);
        ++k;
    }
    return HJ_OK;
}

// The reference reader's {pos, bitbuf, bits} equivalent to `br` after a
// run whose lazy bookkeeping is `tr` (header comment); `data` = the byte
// that positions are counted from.
struct RefState {
    int64_t pos;
    uint64_t buf;
    int bits;
};

inline RefState ref_state(Reader &br, const uint8_t *data, const Track &tr) {
    const int64_t c = br.consumed();
    int64_t b;
    if (tr.starved) {
        b = INT64_MAX;
    } else {
        const int64_t hi = tr.need_hi > c ? tr.need_hi : c;
        b = hi <= br.bits0 ? 0 : (hi - br.bits0 + 7) / 8;
    }
    if (b > br.loaded && !br.stopped) br.refill();
    if (b > br.loaded) b = br.loaded;  // the reader stopped first
    // walk back over the (loaded - b) data bytes appended after byte b
    const uint8_t *q = br.p;
    for (int64_t i = br.loaded - b; i > 0; --i)
        q -= (q - 2 >= br.org && q[-1] == 0x00 && q[-2] == 0xFF) ? 2 : 1;
    RefState s;
    s.pos = q - data;
    s.bits = (int)(br.bits0 + 8 * b - c);
    s.buf = s.bits ? (br.acc >> (64 - s.bits)) : 0;
    return s;
}

// The reference's restart consumption at `pos` (_native.pyx:240-257):
// HJ_OK when an RSTn with the expected index sits there.
inline int check_restart(const uint8_t *data, int64_t n, int64_t pos, int64_t next_rst) {
    if (pos + 1 >= n || data[pos] != 0xFF) return HJ_ERR_EXHAUSTED;
    const uint8_t m = data[pos + 1];
    if (m < 0xD0 || m > 0xD7) return HJ_ERR_MARKER;
    if (m - 0xD0 != next_rst) return HJ_ERR_RST_SEQ;
    return HJ_OK;
}

}  // namespace huff
}  // namespace hj
