// Host entropy stage: baseline Huffman decoding of MCU rows into the planar
// coefficient buffer.  This is the serial producer of the parallel phase and
// stays on the CPU (BASELINE.json north_star "Entropy stage").
//
// Behavioural contract = the reference's native decoder
// (kernels/_native.pyx:66-305; numpy twin fallback.py:282-417):
//   * bit reader: byte-wise refill, 0xFF00 unstuffing, stops delivering bits
//     at any marker (_native.pyx:74-88);
//   * Huffman: 8-bit lookahead table, else the per-length maxcode walk with
//     1-bit takes; truncated streams pad the lookahead with 1-bits
//     (_native.pyx:105-132);
//   * blocks: DC category <= 15, EXTEND, predictor accumulate with a wrap to
//     int16 on store, AC run/size with ZRL/EOB, natural-order store through
//     the zigzag table (_native.pyx:141-184);
//   * restart intervals: byte-align, expect RSTn in sequence, reset the
//     predictors (_native.pyx:238-257);
//   * the int64[8] state {pos, bitbuf, bits, mcus_since_rst, next_rst,
//     predY, predCb, predCr} is written back even on error
//     (_native.pyx:289-296).
#include <cstdint>
#include <cstring>

#include "../../include/hetjpeg_b200.h"
#include "hj_tables.h"

namespace {

const int kZigzag[64] = HJ_ZIGZAG_INIT;

struct BitReader {
    const uint8_t *data;
    int64_t n;
    int64_t pos;
    uint64_t buf;
    int bits;

    inline void refill(int need) {
        while (bits < need) {
            if (pos >= n) return;
            uint8_t b = data[pos];
            if (b == 0xFF) {
                if (pos + 1 < n && data[pos + 1] == 0x00) pos += 2;
                else return;  // marker: stop delivering bits
            } else {
                pos += 1;
            }
            buf = (buf << 8) | b;
            bits += 8;
        }
    }

    inline int take(int k, int &err) {
        if (k == 0) return 0;
        refill(k);
        if (bits < k) {
            err = HJ_ERR_EXHAUSTED;
            return 0;
        }
        bits -= k;
        int v = (int)((buf >> bits) & ((1ull << k) - 1));
        buf &= (1ull << bits) - 1;
        return v;
    }
};

struct Table {
    const uint8_t *lut_sym, *lut_len, *symbols;
    const int32_t *mincode, *maxcode, *valptr;
};

inline Table slot(const hj_scan_tables_t *s, int k) {
    return Table{s->lut_sym[k], s->lut_len[k], s->symbols[k], s->mincode[k], s->maxcode[k], s->valptr[k]};
}

inline int huffdecode(BitReader &br, const Table &t, int &err) {
    br.refill(8);
    unsigned v;
    if (br.bits >= 8) {
        v = (unsigned)((br.buf >> (br.bits - 8)) & 0xFF);
    } else {
        int pad = 8 - br.bits;
        v = (unsigned)(((br.buf << pad) | ((1ull << pad) - 1)) & 0xFF);
    }
    int len = t.lut_len[v];
    if (len != 0 && len <= br.bits) {
        br.bits -= len;
        br.buf &= (1ull << br.bits) - 1;
        return t.lut_sym[v];
    }
    int code = 0;
    for (int l = 1; l < 17; ++l) {
        code = (code << 1) | br.take(1, err);
        if (err != HJ_OK) return 0;
        if (t.maxcode[l] >= 0 && code <= t.maxcode[l]) return t.symbols[t.valptr[l] + code - t.mincode[l]];
    }
    err = HJ_ERR_BADCODE;
    return 0;
}

inline int extend(int v, int t) { return v < (1 << (t - 1)) ? v - ((1 << t) - 1) : v; }

inline int decode_block(BitReader &br, const Table &dc, const Table &ac, int16_t *out, int64_t &pred) {
    int err = HJ_OK;
    int t = huffdecode(br, dc, err);
    if (err != HJ_OK) return err;
    if (t > 15) return HJ_ERR_BADCODE;
    int diff = 0;
    if (t) {
        diff = extend(br.take(t, err), t);
        if (err != HJ_OK) return err;
    }
    pred += diff;
    out[0] = (int16_t)pred;
    int k = 1;
    while (k < 64) {
        int rs = huffdecode(br, ac, err);
        if (err != HJ_OK) return err;
        int r = rs >> 4, s = rs & 0x0F;
        if (s == 0) {
            if (r == 15) {
                k += 16;
                continue;
            }
            break;  // end of block
        }
        k += r;
        if (k > 63) return HJ_ERR_BADCODE;
        out[kZigzag[k]] = (int16_t)extend(br.take(s, err), s);
        if (err != HJ_OK) return err;
        k += 1;
    }
    return HJ_OK;
}

}  // namespace

extern "C" {

hj_status hj_decode_mcu_rows(const uint8_t *data, int64_t n_bytes, int64_t *state,
                             const hj_scan_tables_t *scan, int16_t *y_out, int16_t *cb_out,
                             int16_t *cr_out, int32_t row0, int32_t n_rows, int32_t mcus_per_row,
                             int32_t y_per_mcu, int32_t restart_interval) {
    if (!state || !scan || !y_out || !cb_out || !cr_out || n_bytes < 0) return HJ_ERR_ARG;
    for (int c = 0; c < 3; ++c)
        if (scan->comp_dc[c] < 0 || scan->comp_dc[c] > 7 || scan->comp_ac[c] < 0 || scan->comp_ac[c] > 7)
            return HJ_ERR_ARG;
    BitReader br{data, n_bytes, state[0], (uint64_t)state[1], (int)state[2]};
    int64_t mcus_since = state[3];
    int64_t next_rst = state[4];
    int64_t preds[3] = {state[5], state[6], state[7]};
    Table dc[3], ac[3];
    for (int c = 0; c < 3; ++c) {
        dc[c] = slot(scan, scan->comp_dc[c]);
        ac[c] = slot(scan, scan->comp_ac[c]);
    }
    int err = HJ_OK;
    for (int row = row0; row < row0 + n_rows && err == HJ_OK; ++row) {
        for (int m = 0; m < mcus_per_row; ++m) {
            if (restart_interval != 0 && mcus_since == restart_interval) {
                br.buf = 0;
                br.bits = 0;
                if (br.pos + 1 >= br.n || br.data[br.pos] != 0xFF) {
                    err = HJ_ERR_EXHAUSTED;
                    break;
                }
                uint8_t marker = br.data[br.pos + 1];
                if (marker < 0xD0 || marker > 0xD7) {
                    err = HJ_ERR_MARKER;
                    break;
                }
                if (marker - 0xD0 != next_rst) {
                    err = HJ_ERR_RST_SEQ;
                    break;
                }
                br.pos += 2;
                next_rst = (next_rst + 1) & 7;
                preds[0] = preds[1] = preds[2] = 0;
                mcus_since = 0;
            }
            int64_t mcu = (int64_t)row * mcus_per_row + m;
            for (int j = 0; j < y_per_mcu && err == HJ_OK; ++j)
                err = decode_block(br, dc[0], ac[0], y_out + (mcu * y_per_mcu + j) * 64, preds[0]);
            if (err == HJ_OK) err = decode_block(br, dc[1], ac[1], cb_out + mcu * 64, preds[1]);
            if (err == HJ_OK) err = decode_block(br, dc[2], ac[2], cr_out + mcu * 64, preds[2]);
            if (err != HJ_OK) break;
            mcus_since += 1;
        }
    }
    state[0] = br.pos;
    state[1] = (int64_t)br.buf;
    state[2] = br.bits;
    state[3] = mcus_since;
    state[4] = next_rst;
    state[5] = preds[0];
    state[6] = preds[1];
    state[7] = preds[2];
    return (hj_status)err;
}

int64_t hj_scan_entropy_end(const uint8_t *data, int64_t n, int64_t start) {
    int64_t pos = start;
    while (pos < n - 1) {
        const void *ff = std::memchr(data + pos, 0xFF, (size_t)(n - 1 - pos));
        if (!ff) return -1;
        pos = static_cast<const uint8_t *>(ff) - data;
        uint8_t nxt = data[pos + 1];
        if (nxt == 0x00 || (nxt >= 0xD0 && nxt <= 0xD7)) {
            pos += 2;
            continue;
        }
        if (nxt == 0xFF) {  // fill byte
            pos += 1;
            continue;
        }
        return pos;
    }
    return -1;
}

}  // extern "C"
