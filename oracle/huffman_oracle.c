/*
 * CPU ORACLE - test infrastructure only (see render_oracle.c).  Never linked
 * or called by the product: tests/, __graft_entry__.smoke() and bench.py's
 * CPU legs load it as the checker and as the reference arm's decoder.
 *
 * A plain-C restatement of the reference's resumable baseline Huffman
 * decoder, kernels/_native.pyx:66-305 (numpy twin kernels/fallback.py:282-417):
 *
 *   or_refill        _native.pyx:74-88   byte-wise refill, 0xFF00 unstuffing,
 *                                        stops delivering bits at any marker
 *   or_take          _native.pyx:91-102
 *   or_huffdecode    _native.pyx:105-132 8-bit lookahead (1-bit padded when
 *                                        short), then the per-length maxcode walk
 *   or_extend        _native.pyx:135-138
 *   or_decode_block  _native.pyx:141-184 DC category <= 15, predictor with a
 *                                        wrap to int16 on store, AC run/size,
 *                                        ZRL / EOB, natural-order store
 *   or_decode_mcu_rows _native.pyx:195-305 restart intervals (byte-align,
 *                                        RSTn in sequence, predictor reset),
 *                                        int64[8] state written back on error
 *
 * The slot tables are the reference's _pack_scan_tables layout
 * (entropy.py:59-84): slots 0-3 DC, 4-7 AC.
 */
#include <stdint.h>
#include <string.h>

enum { OR_OK = 0, OR_EXHAUSTED = 1, OR_BADCODE = 2, OR_MARKER = 3, OR_RST_SEQ = 4, OR_ARG = 16 };

typedef struct {
    uint8_t lut_sym[8][256];
    uint8_t lut_len[8][256];
    int32_t mincode[8][17];
    int32_t maxcode[8][17];
    int32_t valptr[8][17];
    uint8_t symbols[8][256];
    int32_t comp_dc[3];
    int32_t comp_ac[3];
} or_scan_tables;

static const int ZZ[64] = {0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,
                           12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6,  7,  14, 21, 28,
                           35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
                           58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};

typedef struct {
    const uint8_t *data;
    int64_t n, pos;
    uint64_t buf;
    int bits;
} or_reader;

static void or_refill(or_reader *r, int need) {
    while (r->bits < need) {
        if (r->pos >= r->n) return;
        uint8_t b = r->data[r->pos];
        if (b == 0xFF) {
            if (r->pos + 1 < r->n && r->data[r->pos + 1] == 0x00) r->pos += 2;
            else return;
        } else {
            r->pos += 1;
        }
        r->buf = (r->buf << 8) | b;
        r->bits += 8;
    }
}

static int or_take(or_reader *r, int k, int *err) {
    if (k == 0) return 0;
    or_refill(r, k);
    if (r->bits < k) {
        *err = OR_EXHAUSTED;
        return 0;
    }
    r->bits -= k;
    int v = (int)((r->buf >> r->bits) & ((1ull << k) - 1));
    r->buf &= (1ull << r->bits) - 1;
    return v;
}

static int or_huffdecode(or_reader *r, const or_scan_tables *t, int s, int *err) {
    or_refill(r, 8);
    unsigned v;
    if (r->bits >= 8) {
        v = (unsigned)((r->buf >> (r->bits - 8)) & 0xFF);
    } else {
        int pad = 8 - r->bits;
        v = (unsigned)(((r->buf << pad) | ((1ull << pad) - 1)) & 0xFF);
    }
    int len = t->lut_len[s][v];
    if (len != 0 && len <= r->bits) {
        r->bits -= len;
        r->buf &= (1ull << r->bits) - 1;
        return t->lut_sym[s][v];
    }
    int code = 0;
    for (int l = 1; l < 17; ++l) {
        code = (code << 1) | or_take(r, 1, err);
        if (*err) return 0;
        if (t->maxcode[s][l] >= 0 && code <= t->maxcode[s][l])
            return t->symbols[s][t->valptr[s][l] + code - t->mincode[s][l]];
    }
    *err = OR_BADCODE;
    return 0;
}

static int or_extend(int v, int t) { return v < (1 << (t - 1)) ? v - ((1 << t) - 1) : v; }

static int or_decode_block(or_reader *r, const or_scan_tables *t, int dc, int ac, int16_t *out,
                           int64_t *pred) {
    int err = OR_OK;
    int cat = or_huffdecode(r, t, dc, &err);
    if (err) return err;
    if (cat > 15) return OR_BADCODE;
    int diff = 0;
    if (cat) {
        diff = or_extend(or_take(r, cat, &err), cat);
        if (err) return err;
    }
    *pred += diff;
    out[0] = (int16_t)*pred;
    for (int k = 1; k < 64;) {
        int rs = or_huffdecode(r, t, ac, &err);
        if (err) return err;
        int run = rs >> 4, sz = rs & 15;
        if (sz == 0) {
            if (run == 15) {
                k += 16;
                continue;
            }
            break;
        }
        k += run;
        if (k > 63) return OR_BADCODE;
        out[ZZ[k]] = (int16_t)or_extend(or_take(r, sz, &err), sz);
        if (err) return err;
        k += 1;
    }
    return OR_OK;
}

int or_decode_mcu_rows(const uint8_t *data, int64_t n, int64_t *state, const or_scan_tables *t,
                       int16_t *y, int16_t *cb, int16_t *cr, int row0, int n_rows, int mpr, int ypm,
                       int restart_interval) {
    if (!state || !t || n < 0) return OR_ARG;
    or_reader r = {data, n, state[0], (uint64_t)state[1], (int)state[2]};
    int64_t since = state[3], next_rst = state[4];
    int64_t pred[3] = {state[5], state[6], state[7]};
    int err = OR_OK;
    for (int row = row0; row < row0 + n_rows && !err; ++row) {
        for (int m = 0; m < mpr && !err; ++m) {
            if (restart_interval && since == restart_interval) {
                r.buf = 0;
                r.bits = 0;
                if (r.pos + 1 >= r.n || r.data[r.pos] != 0xFF) {
                    err = OR_EXHAUSTED;
                    break;
                }
                int mk = r.data[r.pos + 1];
                if (mk < 0xD0 || mk > 0xD7) {
                    err = OR_MARKER;
                    break;
                }
                if (mk - 0xD0 != next_rst) {
                    err = OR_RST_SEQ;
                    break;
                }
                r.pos += 2;
                next_rst = (next_rst + 1) & 7;
                pred[0] = pred[1] = pred[2] = 0;
                since = 0;
            }
            int64_t mcu = (int64_t)row * mpr + m;
            for (int j = 0; j < ypm && !err; ++j)
                err = or_decode_block(&r, t, t->comp_dc[0], t->comp_ac[0], y + (mcu * ypm + j) * 64, &pred[0]);
            if (!err) err = or_decode_block(&r, t, t->comp_dc[1], t->comp_ac[1], cb + mcu * 64, &pred[1]);
            if (!err) err = or_decode_block(&r, t, t->comp_dc[2], t->comp_ac[2], cr + mcu * 64, &pred[2]);
            if (!err) since += 1;
        }
    }
    state[0] = r.pos;
    state[1] = (int64_t)r.buf;
    state[2] = r.bits;
    state[3] = since;
    state[4] = next_rst;
    state[5] = pred[0];
    state[6] = pred[1];
    state[7] = pred[2];
    return err;
}
