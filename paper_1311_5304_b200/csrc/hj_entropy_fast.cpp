// Throughput Huffman decoder for the pipelined / batched decode path.
//
// Produces coefficient planes bit-identical to the reference decoder
// (kernels/_native.pyx:66-305; same code construction, same EXTEND, EOB/ZRL,
// predictor wrap to int16, restart handling and error conditions), but
//   * keeps a left-aligned 64-bit bit buffer refilled up to 56 bits at a time
//     (stops at any marker, like _refill, _native.pyx:74-88);
//   * decodes with 11-bit lookahead tables; for DC and AC, one lookup yields
//     code length (+ run) + the EXTENDed value whenever code + magnitude bits
//     fit in 11 bits (most coefficients), else the code alone with the
//     magnitude bits read straight from the buffer; codes longer than 11 bits
//     continue the canonical maxcode walk (_native.pyx:124-132) on the
//     buffered bits;
//   * splits a scan at its restart markers and decodes the intervals on
//     several host threads - exact, because every RSTn resets the DC
//     predictors (_native.pyx:238-257).
// The resumable per-row cursor of the drop-in API stays in hj_entropy.cpp.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/hetjpeg_b200.h"
#include "hj_tables.h"

namespace {

const int kZigzag[64] = HJ_ZIGZAG_INIT;
constexpr int kLook = 11;

// AC fast entry: bits 0-15 value (int16), 16-19 run, 20-24 consumed length,
// 25-27 kind.
enum Kind { kSlow = 0, kCoef = 1, kEob = 2, kZrl = 3, kCodeOnly = 4 };

struct Table {
    uint16_t look[1 << kLook];  // (len << 8) | symbol, len 0 = longer code
    int32_t ac[1 << kLook];     // AC fast entries (AC tables only)
    int32_t mincode[17], maxcode[17], valptr[17];
    uint8_t symbols[256];
};

struct Fast {
    Table t[8];
    int comp_dc[3], comp_ac[3];
};

inline int extend(int v, int t) { return v < (1 << (t - 1)) ? v - ((1 << t) - 1) : v; }

void build_table(const hj_scan_tables_t *s, int slot, Table &t, bool ac) {
    std::memcpy(t.mincode, s->mincode[slot], sizeof(t.mincode));
    std::memcpy(t.maxcode, s->maxcode[slot], sizeof(t.maxcode));
    std::memcpy(t.valptr, s->valptr[slot], sizeof(t.valptr));
    std::memcpy(t.symbols, s->symbols[slot], sizeof(t.symbols));
    std::memset(t.look, 0, sizeof(t.look));
    std::memset(t.ac, 0, sizeof(t.ac));
    for (int len = 1; len <= kLook; ++len) {
        if (t.maxcode[len] < 0) continue;
        for (int code = t.mincode[len]; code <= t.maxcode[len]; ++code) {
            int idx = t.valptr[len] + code - t.mincode[len];
            if (idx < 0 || idx > 255) continue;
            int sym = t.symbols[idx];
            int lo = code << (kLook - len), n = 1 << (kLook - len);
            for (int v = lo; v < lo + n; ++v) {
                t.look[v] = (uint16_t)((len << 8) | sym);
                if (!ac) {
                    // DC: the symbol is the magnitude category; > 15 is a bad
                    // code (left to the generic path)
                    int32_t e = kSlow << 25;
                    if (sym == 0) e = kCoef << 25 | len << 20;
                    else if (sym <= 15 && len + sym <= kLook)
                        e = kCoef << 25 | (len + sym) << 20 |
                            (extend((v >> (kLook - len - sym)) & ((1 << sym) - 1), sym) & 0xffff);
                    else if (sym <= 15) e = kCodeOnly << 25 | len << 20 | sym;
                    t.ac[v] = e;
                    continue;
                }
                int r = sym >> 4, sz = sym & 15;
                int32_t e;
                if (sz == 0) {
                    // r == 15: ZRL; any other run with size 0 ends the block
                    // (reference: `if s == 0: ... break`, _native.pyx:172-176)
                    e = (r == 15 ? kZrl : kEob) << 25 | len << 20;
                } else if (len + sz <= kLook) {
                    int bits = (v >> (kLook - len - sz)) & ((1 << sz) - 1);
                    int val = extend(bits, sz);
                    e = kCoef << 25 | (len + sz) << 20 | r << 16 | (val & 0xffff);
                } else {
                    e = kCodeOnly << 25 | len << 20 | (sym & 0xff);
                }
                t.ac[v] = e;
            }
        }
    }
}

struct Reader {
    const uint8_t *p, *end;
    uint64_t acc = 0;  // next bit = bit 63
    int nbits = 0;

    inline void refill() {
        // fast path: the next whole bytes that fit contain no 0xFF (no
        // stuffing, no marker): append them with one big-endian 64-bit load
        if (nbits <= 56 && end - p >= 8) {
            uint64_t w;
            std::memcpy(&w, p, 8);
            w = __builtin_bswap64(w);
            const int nb = (64 - nbits) >> 3;          // 1..8 whole bytes fit
            const uint64_t top = nb == 8 ? ~0ull : ~(~0ull >> (8 * nb));
            const uint64_t x = ~w & top;               // a 0xFF byte -> a zero byte of x
            const uint64_t has_ff = (x - 0x0101010101010101ull) & ~x & 0x8080808080808080ull & top;
            if (!has_ff) {
                acc |= (w & top) >> nbits;
                p += nb;
                nbits += 8 * nb;
                return;
            }
        }
        while (nbits <= 56) {
            if (p >= end) return;
            uint8_t b = *p;
            if (b == 0xFF) {
                if (p + 1 < end && p[1] == 0x00) p += 2;
                else return;  // marker: stop delivering bits
            } else {
                ++p;
            }
            acc |= (uint64_t)b << (56 - nbits);
            nbits += 8;
        }
    }
    inline uint32_t peek(int n) const { return (uint32_t)(acc >> (64 - n)); }
    inline void skip(int n) {
        acc <<= n;
        nbits -= n;
    }
    // take k bits (k <= 16); false = stream exhausted (reference _take)
    inline bool take(int k, int &v) {
        if (k == 0) {
            v = 0;
            return true;
        }
        if (nbits < k) refill();
        if (nbits < k) return false;
        v = (int)peek(k);
        skip(k);
        return true;
    }
};

// Generic Huffman decode, reference semantics (_native.pyx:105-132).
inline int decode_sym(Reader &br, const Table &t, int &err) {
    if (br.nbits < 16) br.refill();
    if (br.nbits >= 1) {
        uint16_t e = t.look[br.peek(kLook)];  // bits past nbits are 0: only codes of
                                              // length <= nbits are accepted
        int len = e >> 8;
        if (len != 0 && len <= br.nbits) {
            br.skip(len);
            return e & 0xff;
        }
    }
    if (br.nbits >= 16) {
        // no code of <= kLook bits prefixes the stream (the table): walk the
        // longer lengths on the buffered bits (_native.pyx:124-132 order)
        for (int l = kLook + 1; l < 17; ++l) {
            const int code = (int)br.peek(l);
            if (t.maxcode[l] >= 0 && code <= t.maxcode[l]) {
                br.skip(l);
                return t.symbols[t.valptr[l] + code - t.mincode[l]];
            }
        }
        err = HJ_ERR_BADCODE;
        return 0;
    }
    int code = 0;
    for (int l = 1; l < 17; ++l) {
        int bit;
        if (!br.take(1, bit)) {
            err = HJ_ERR_EXHAUSTED;
            return 0;
        }
        code = (code << 1) | bit;
        if (t.maxcode[l] >= 0 && code <= t.maxcode[l]) return t.symbols[t.valptr[l] + code - t.mincode[l]];
    }
    err = HJ_ERR_BADCODE;
    return 0;
}

inline int decode_block(Reader &br, const Table &dc, const Table &ac, int16_t *out, int64_t &pred) {
    std::memset(out, 0, 64 * sizeof(int16_t));  // the block is about to be hot anyway
    int err = HJ_OK;
    int diff = 0;
    if (br.nbits < 32) br.refill();
    const int32_t de = br.nbits >= 32 ? dc.ac[br.peek(kLook)] : 0;
    if ((de >> 25) == kCoef) {
        br.skip((de >> 20) & 31);
        diff = (int16_t)(de & 0xffff);
    } else if ((de >> 25) == kCodeOnly) {
        const int t = de & 0xff;  // 1..15; >= 16 buffered bits remain
        br.skip((de >> 20) & 31);
        diff = extend((int)br.peek(t), t);
        br.skip(t);
    } else {
        int t = decode_sym(br, dc, err);
        if (err) return err;
        if (t > 15) return HJ_ERR_BADCODE;
        if (t) {
            int v;
            if (!br.take(t, v)) return HJ_ERR_EXHAUSTED;
            diff = extend(v, t);
        }
    }
    pred += diff;
    out[0] = (int16_t)pred;
    int k = 1;
    while (k < 64) {
        if (br.nbits < 32) br.refill();
        if (br.nbits >= kLook) {
            int32_t e = ac.ac[br.peek(kLook)];
            int kind = e >> 25, len = (e >> 20) & 31;
            if (kind == kCoef) {
                br.skip(len);
                k += (e >> 16) & 15;
                if (k > 63) return HJ_ERR_BADCODE;
                out[kZigzag[k]] = (int16_t)(e & 0xffff);
                ++k;
                continue;
            }
            if (kind == kEob) {
                br.skip(len);
                break;
            }
            if (kind == kZrl) {
                br.skip(len);
                k += 16;
                continue;
            }
            if (kind == kCodeOnly && br.nbits >= 32) {
                // code in the table, magnitude bits past it: still buffered
                const int r = (e >> 4) & 15, sz = e & 15;
                br.skip(len);
                k += r;
                if (k > 63) return HJ_ERR_BADCODE;
                out[kZigzag[k]] = (int16_t)extend((int)br.peek(sz), sz);
                br.skip(sz);
                ++k;
                continue;
            }
        }
        int rs = decode_sym(br, ac, err);
        if (err) return err;
        int r = rs >> 4, s = rs & 15;
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
        if (!br.take(s, v)) return HJ_ERR_EXHAUSTED;
        out[kZigzag[k]] = (int16_t)extend(v, s);
        ++k;
    }
    return HJ_OK;
}

struct Segment {
    int64_t byte0;    // first entropy byte of the interval
    int64_t mcu0, mcu1;
    int expect_rst;   // RSTn that must precede it (-1 for the first)
};

int decode_segment(const Fast &f, const uint8_t *data, int64_t n, const Segment &sg, int16_t *y, int16_t *cb,
                   int16_t *cr, int ypm) {
    Reader br{data + sg.byte0, data + n};
    int64_t preds[3] = {0, 0, 0};
    const Table &dy = f.t[f.comp_dc[0]], &ay = f.t[f.comp_ac[0]];
    const Table &dcb = f.t[f.comp_dc[1]], &acb = f.t[f.comp_ac[1]];
    const Table &dcr = f.t[f.comp_dc[2]], &acr = f.t[f.comp_ac[2]];
    for (int64_t mcu = sg.mcu0; mcu < sg.mcu1; ++mcu) {
        for (int j = 0; j < ypm; ++j) {
            int e = decode_block(br, dy, ay, y + (mcu * ypm + j) * 64, preds[0]);
            if (e) return e;
        }
        int e = decode_block(br, dcb, acb, cb + mcu * 64, preds[1]);
        if (!e) e = decode_block(br, dcr, acr, cr + mcu * 64, preds[2]);
        if (e) return e;
    }
    return HJ_OK;
}

}  // namespace

extern "C" {

hj_status hj_huff_build(const hj_scan_tables_t *scan, void **out) {
    if (!scan || !out) return HJ_ERR_ARG;
    Fast *f = new Fast();
    bool used[8] = {false};
    for (int c = 0; c < 3; ++c) {
        if (scan->comp_dc[c] < 0 || scan->comp_dc[c] > 7 || scan->comp_ac[c] < 0 || scan->comp_ac[c] > 7) {
            delete f;
            return HJ_ERR_ARG;
        }
        f->comp_dc[c] = scan->comp_dc[c];
        f->comp_ac[c] = scan->comp_ac[c];
        used[scan->comp_dc[c]] = used[scan->comp_ac[c]] = true;
    }
    for (int s = 0; s < 8; ++s)
        if (used[s]) build_table(scan, s, f->t[s], s >= 4);
    *out = f;
    return HJ_OK;
}

void hj_huff_free(void *fast) { delete static_cast<Fast *>(fast); }

// Decode a whole scan (all MCUs) into the planes (every block is written,
// zeros included).  With a
// restart interval the intervals are decoded on up to n_threads threads.
hj_status hj_decode_scan_fast(const void *fast, const uint8_t *data, int64_t n, int16_t *y, int16_t *cb,
                              int16_t *cr, int32_t mcus_per_row, int32_t mcu_rows, int32_t y_per_mcu,
                              int32_t restart_interval, int32_t n_threads) {
    const Fast *f = static_cast<const Fast *>(fast);
    if (!f || (!data && n) || !y || !cb || !cr || n < 0) return HJ_ERR_ARG;
    const int64_t total = (int64_t)mcus_per_row * mcu_rows;
    std::vector<Segment> segs;
    if (restart_interval <= 0) {
        segs.push_back({0, 0, total, -1});
    } else {
        // interval boundaries = RSTn markers, in order
        int64_t pos = 0, mcu = 0;
        int k = 0;
        segs.push_back({0, 0, std::min<int64_t>(total, restart_interval), -1});
        mcu = segs.back().mcu1;
        while (mcu < total) {
            // next RSTn after `pos`: skip stuffed 0xFF00 and fill bytes; any
            // other marker ends the scan data (reference: "expected a
            // restart marker", _native.pyx:242-244)
            int64_t q = pos;
            bool found = false;
            while (q + 1 < n) {
                const void *ff = std::memchr(data + q, 0xFF, (size_t)(n - 1 - q));
                if (!ff) break;
                q = static_cast<const uint8_t *>(ff) - data;
                uint8_t b = data[q + 1];
                if (b == 0x00) {
                    q += 2;
                } else if (b == 0xFF) {
                    q += 1;
                } else {
                    found = (b >= 0xD0 && b <= 0xD7);
                    break;
                }
            }
            if (!found) return HJ_ERR_EXHAUSTED;
            if (data[q + 1] - 0xD0 != (k & 7)) return HJ_ERR_RST_SEQ;
            pos = q + 2;
            segs.push_back({pos, mcu, std::min<int64_t>(total, mcu + restart_interval), k & 7});
            mcu = segs.back().mcu1;
            ++k;
        }
    }
    const int nt = std::max(1, std::min<int>(n_threads, (int)segs.size()));
    std::atomic<int64_t> next{0};
    std::vector<int> errs(segs.size(), HJ_OK);
    auto work = [&]() {
        for (int64_t i; (i = next.fetch_add(1)) < (int64_t)segs.size();)
            errs[i] = decode_segment(*f, data, n, segs[i], y, cb, cr, y_per_mcu);
    };
    std::vector<std::thread> th;
    for (int i = 1; i < nt; ++i) th.emplace_back(work);
    work();
    for (auto &t : th) t.join();
    for (int e : errs)
        if (e) return (hj_status)e;
    return HJ_OK;
}

}  // extern "C"
