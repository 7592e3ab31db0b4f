// Host entropy stage (CPU, C++): the serial producer of the parallel phase,
// kept on the host cores (BASELINE.json north_star "Entropy stage").  One
// Huffman core (hj_huffman.h) behind three C-ABI entry points:
//
//   hj_decode_mcu_rows   the drop-in backend's resumable decoder
//                        (kernels/_native.pyx:195-305): MCU rows
//                        [row0, row0+n) from an int64[8] cursor state,
//                        written back on success and on error;
//   hj_decode_scan_fast  a whole scan for the pipelined / batched path,
//                        split at its restart markers and decoded on
//                        several threads (exact: every RSTn resets the DC
//                        predictors, _native.pyx:238-257);
//   hj_scan_entropy_end  the parser's entropy-span scan (parser.py:277-293).
//
// Both decoders reproduce the reference's outputs, errors and - for the
// cursor - its reader state, including on corrupt streams: the restart check
// is made where the reference's lazily-filled reader would stand
// (hj_huffman.h, "Reference-equivalent reader state").
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/hetjpeg_b200.h"
#include "hj_error.h"
#include "hj_huffman.h"
#include "hj_tables.h"

namespace hj {
namespace huff {

const int kZigzag[64] = HJ_ZIGZAG_INIT;

namespace {

void build_table(const hj_scan_tables_t *s, int slot, Table &t, bool ac) {
    std::memcpy(t.mincode, s->mincode[slot], sizeof(t.mincode));
    std::memcpy(t.maxcode, s->maxcode[slot], sizeof(t.maxcode));
    std::memcpy(t.valptr, s->valptr[slot], sizeof(t.valptr));
    std::memcpy(t.symbols, s->symbols[slot], sizeof(t.symbols));
    std::memset(t.look, 0, sizeof(t.look));
    std::memset(t.fast, 0, sizeof(t.fast));
    std::memset(t.pair, 0, sizeof(t.pair));
    // every code of <= kLook bits owns the 2^(kLook - len) lookahead values it prefixes
    for (int len = 1; len <= kLook; ++len) {
        if (t.maxcode[len] < 0) continue;
        for (int code = t.mincode[len]; code <= t.maxcode[len]; ++code) {
            const int idx = t.valptr[len] + code - t.mincode[len];
            if (idx < 0 || idx > 255) continue;
            const int sym = t.symbols[idx];
            const int span = kLook - len;
            for (int v = code << span, v1 = (code + 1) << span; v < v1; ++v) {
                t.look[v] = (uint16_t)((len << 8) | sym);
                const uint32_t clen = (uint32_t)len << 28;
                uint32_t e;
                const int run = ac ? sym >> 4 : 0, size = ac ? sym & 15 : sym;
                if (!ac && size > 15) {
                    e = kSlow << 25;  // bad DC category: the generic path reports it
                } else if (ac && size == 0) {
                    // ZRL (15/0); any other run with size 0 ends the block
                    e = (run == 15 ? kZrl : kEob) << 25 | clen | (uint32_t)len << 20;
                } else if (size == 0) {
                    e = kCoef << 25 | clen | (uint32_t)len << 20;  // DC difference 0
                } else if (len + size <= kLook) {
                    const int mag = (v >> (span - size)) & ((1 << size) - 1);
                    e = kCoef << 25 | clen | (uint32_t)(len + size) << 20 | (uint32_t)run << 16 |
                        ((uint32_t)extend(mag, size) & 0xffff);
                } else {
                    e = kCodeOnly << 25 | clen | (uint32_t)len << 20 | (uint32_t)(ac ? sym : size);
                }
                t.fast[v] = e;
            }
        }
    }
    if (!ac) return;
    // pairs: a complete first coefficient (kCoef with a nonzero size) whose
    // remaining lookahead bits hold a complete second one
    for (int v = 0; v < (1 << kPairLook); ++v) {
        const uint32_t e1 = t.fast[v >> (kPairLook - kLook)];
        if (((e1 >> 25) & 7) != kCoef || (e1 >> 28) == 0) continue;
        const int l1 = (e1 >> 20) & 31;
        const int rest = kPairLook - l1;
        if (rest <= 0) continue;
        // the next kLook bits after the first coefficient (known: `rest` of them)
        const int nxt = (int)(((uint32_t)v << l1) & ((1u << kPairLook) - 1));
        const uint32_t e2 = t.fast[nxt >> (kPairLook - kLook)];
        const uint32_t k2 = (e2 >> 25) & 7;
        if (k2 != kCoef && k2 != kEob) continue;
        const int l2 = (e2 >> 20) & 31;
        if (l2 > rest) continue;  // the second code / magnitude needs bits past the lookahead
        const int v1 = (int16_t)(e1 & 0xffff), v2 = k2 == kEob ? 0 : (int16_t)(e2 & 0xffff);
        if (v1 < -512 || v1 > 511 || v2 < -512 || v2 > 511) continue;
        t.pair[v] = ((uint32_t)v1 & 1023) | ((uint32_t)v2 & 1023) << 10 | ((e1 >> 16) & 15) << 20 |
                    (k2 == kEob ? 0u : ((e2 >> 16) & 15) << 24) | (uint32_t)(l1 + l2) << 28;
    }
}

}  // namespace

bool build_tables(const hj_scan_tables_t *scan, Tables &f) {
    bool used[8] = {false};
    for (int c = 0; c < 3; ++c) {
        if (scan->comp_dc[c] < 0 || scan->comp_dc[c] > 7 || scan->comp_ac[c] < 0 || scan->comp_ac[c] > 7)
            return false;
        f.comp_dc[c] = scan->comp_dc[c];
        f.comp_ac[c] = scan->comp_ac[c];
        used[scan->comp_dc[c]] = used[scan->comp_ac[c]] = true;
    }
    for (int s = 0; s < 8; ++s)
        if (used[s]) build_table(scan, s, f.t[s], s >= 4);
    return true;
}

}  // namespace huff
}  // namespace hj

namespace {

using namespace hj::huff;

// Decodes MCUs [mcu0, mcu1) of one MCU-ordered plane set, with the
// lazy-reader bookkeeping when `tr` is given: on every MCU (kTrackAll, the
// cursor, whose state must be exact after an error too) or on the last MCU
// only (whose blocks hold the run's final Huffman lookahead).
template <bool kZero, bool kTrackAll>
int decode_mcus(const Tables &f, Reader &br, int64_t mcu0, int64_t mcu1, int ypm, int16_t *y, int16_t *cb,
                int16_t *cr, int64_t *preds, Track *tr, int64_t *done) {
    const Table &dy = f.t[f.comp_dc[0]], &ay = f.t[f.comp_ac[0]];
    const Table &dcb = f.t[f.comp_dc[1]], &acb = f.t[f.comp_ac[1]];
    const Table &dcr = f.t[f.comp_dc[2]], &acr = f.t[f.comp_ac[2]];
    const int64_t plain_end = !tr ? mcu1 : kTrackAll ? mcu0 : mcu1 - 1;
    int64_t mcu = mcu0;
    for (; mcu < plain_end; ++mcu) {
        int e = HJ_OK;
        for (int j = 0; j < ypm && !e; ++j)
            e = decode_block<kZero, false>(br, dy, ay, y + (mcu * ypm + j) * 64, preds[0], nullptr);
        if (!e) e = decode_block<kZero, false>(br, dcb, acb, cb + mcu * 64, preds[1], nullptr);
        if (!e) e = decode_block<kZero, false>(br, dcr, acr, cr + mcu * 64, preds[2], nullptr);
        if (e) {
            if (done) *done = mcu - mcu0;
            return e;
        }
    }
    for (; mcu < mcu1; ++mcu) {  // the tracked last MCU
        int e = HJ_OK;
        for (int j = 0; j < ypm && !e; ++j)
            e = decode_block<kZero, true>(br, dy, ay, y + (mcu * ypm + j) * 64, preds[0], tr);
        if (!e) e = decode_block<kZero, true>(br, dcb, acb, cb + mcu * 64, preds[1], tr);
        if (!e) e = decode_block<kZero, true>(br, dcr, acr, cr + mcu * 64, preds[2], tr);
        if (e) {
            if (done) *done = mcu - mcu0;
            return e;
        }
    }
    if (done) *done = mcu1 - mcu0;
    return HJ_OK;
}

// One restart interval of a whole scan.  `end` = the reader's stop point
// after it (the first 0xFF not followed by 0x00, or the end of the data).
struct Segment {
    int64_t byte0;  // first entropy byte of the interval
    int64_t mcu0, mcu1;
    int64_t end;
    bool last;      // no restart marker is consumed after it
};

int decode_segment(const Tables &f, const uint8_t *data, int64_t n, const Segment &sg, int16_t *y,
                   int16_t *cb, int16_t *cr, int ypm, int expect_rst) {
    Reader br(data + sg.byte0, data + n);
    int64_t preds[3] = {0, 0, 0};
    Track tr;
    int e = decode_mcus<true, false>(f, br, sg.mcu0, sg.mcu1, ypm, y, cb, cr, preds, sg.last ? nullptr : &tr, nullptr);
    if (e || sg.last) return e;
    // the reference consumes RSTn where its own reader stands
    const RefState rs = ref_state(br, data, tr);
    return check_restart(data, n, rs.pos, expect_rst);
}

// First byte at or after `q` where the reader stops: 0xFF not followed by 0x00.
int64_t stop_point(const uint8_t *data, int64_t n, int64_t q) {
    while (q < n) {
        const void *ff = std::memchr(data + q, 0xFF, (size_t)(n - q));
        if (!ff) return n;
        q = static_cast<const uint8_t *>(ff) - data;
        if (q + 1 < n && data[q + 1] == 0x00) {
            q += 2;
            continue;
        }
        return q;
    }
    return n;
}

// Thread-local cache of the tables of the last scan header seen by the
// drop-in cursor (one call per MCU row; the packed header is ~8.5 KB).
struct CursorCache {
    hj_scan_tables_t key;
    Tables tables;
    bool valid = false;
};

const Tables *cursor_tables(const hj_scan_tables_t *scan) {
    thread_local std::unique_ptr<CursorCache> c(new CursorCache());  // large: heap, per thread
    if (!c->valid || std::memcmp(&c->key, scan, sizeof(*scan)) != 0) {
        if (!build_tables(scan, c->tables)) return nullptr;
        std::memcpy(&c->key, scan, sizeof(*scan));
        c->valid = true;
    }
    return &c->tables;
}

const char *status_name(int s) {
    switch (s) {
        case HJ_ERR_EXHAUSTED: return "ran out of entropy-coded bits";
        case HJ_ERR_BADCODE: return "no Huffman symbol matches within 16 bits";
        case HJ_ERR_MARKER: return "non-restart marker inside the scan";
        case HJ_ERR_RST_SEQ: return "restart marker out of sequence";
        default: return "entropy decode failed";
    }
}

}  // namespace

extern "C" {

hj_status hj_huff_build(const hj_scan_tables_t *scan, void **out) {
    if (!scan || !out) return hj::fail(HJ_ERR_ARG, "hj_huff_build: null pointer");
    Tables *f = new Tables();
    if (!build_tables(scan, *f)) {
        delete f;
        return hj::fail(HJ_ERR_ARG, "hj_huff_build: component table slot outside 0..7");
    }
    *out = f;
    return HJ_OK;
}

void hj_huff_free(void *fast) { delete static_cast<Tables *>(fast); }

// Decode a whole scan (all MCUs; every block written, zeros included).
// With a restart interval the intervals are located first (each one ends
// where the reader stops), decoded on up to n_threads threads, and each
// interval's end is checked where the reference's reader would stand.  The
// first failing interval in scan order decides the status, as in the
// reference's sequential decode.
}  // extern "C"

namespace {

// Decodes the restart intervals of a scan that overlap MCUs [m_lo, m_hi).
// Interval boundaries are found by a byte scan from the start (each interval
// ends where the reader stops); only the overlapping intervals are Huffman
// decoded, on up to n_threads threads.  Without restart intervals the scan is
// one interval and is decoded whole.
hj_status decode_scan_mcus(const Tables *f, const uint8_t *data, int64_t n, int16_t *y, int16_t *cb, int16_t *cr,
                           int32_t mcus_per_row, int32_t mcu_rows, int32_t y_per_mcu, int32_t restart_interval,
                           int64_t m_lo, int64_t m_hi, int32_t n_threads) {
    const int64_t total = (int64_t)mcus_per_row * mcu_rows;
    m_lo = std::max<int64_t>(0, m_lo);
    m_hi = std::min<int64_t>(total, m_hi);
    std::vector<Segment> segs;
    std::vector<int> expect;  // RSTn index after each segment
    if (restart_interval <= 0 || total <= restart_interval) {
        segs.push_back({0, 0, total, n, true});
        expect.push_back(0);
    } else {
        int64_t pos = 0, mcu = 0, k = 0;
        while (mcu < total && mcu < m_hi) {
            const int64_t m1 = std::min<int64_t>(total, mcu + restart_interval);
            const bool last = m1 == total;
            const int64_t end = last ? n : stop_point(data, n, pos);
            segs.push_back({pos, mcu, m1, end, last});
            expect.push_back((int)(k & 7));
            if (last) break;
            // an interval that does not end on the expected RSTn fails its
            // own check; nothing after it is decoded (first error wins)
            if (check_restart(data, n, end, k & 7) != HJ_OK) break;
            pos = end + 2;
            mcu = m1;
            ++k;
        }
    }
    std::vector<size_t> todo;
    for (size_t i = 0; i < segs.size(); ++i)
        if (segs[i].mcu1 > m_lo && segs[i].mcu0 < m_hi) todo.push_back(i);
    if (!segs.empty() && segs.back().mcu1 < m_hi && todo.empty()) todo.push_back(segs.size() - 1);
    const int nt = std::max(1, std::min<int>(n_threads, (int)todo.size()));
    std::atomic<int64_t> next{0};
    std::vector<int> errs(todo.size(), HJ_OK);
    auto work = [&]() {
        for (int64_t t; (t = next.fetch_add(1)) < (int64_t)todo.size();) {
            const size_t i = todo[(size_t)t];
            errs[(size_t)t] = decode_segment(*f, data, n, segs[i], y, cb, cr, y_per_mcu, expect[i]);
        }
    };
    std::vector<std::thread> th;
    for (int i = 1; i < nt; ++i) th.emplace_back(work);
    work();
    for (auto &t : th) t.join();
    for (size_t t = 0; t < errs.size(); ++t)
        if (errs[t]) return hj::fail((hj_status)errs[t], std::string("restart interval ") + std::to_string(todo[t]) +
                                                           ": " + status_name(errs[t]));
    return HJ_OK;
}

}  // namespace

extern "C" {

// Decode a whole scan (all MCUs; every block written, zeros included).
// With a restart interval the intervals are located first (each one ends
// where the reader stops), decoded on up to n_threads threads, and each
// interval's end is checked where the reference's reader would stand.  The
// first failing interval in scan order decides the status, as in the
// reference's sequential decode.
hj_status hj_decode_scan_fast(const void *fast, const uint8_t *data, int64_t n, int16_t *y, int16_t *cb,
                              int16_t *cr, int32_t mcus_per_row, int32_t mcu_rows, int32_t y_per_mcu,
                              int32_t restart_interval, int32_t n_threads) {
    const Tables *f = static_cast<const Tables *>(fast);
    if (!f || (!data && n) || !y || !cb || !cr || n < 0 || mcus_per_row < 0 || mcu_rows < 0 ||
        y_per_mcu < 1 || y_per_mcu > 4)
        return hj::fail(HJ_ERR_ARG, "hj_decode_scan_fast: bad arguments");
    return decode_scan_mcus(f, data, n, y, cb, cr, mcus_per_row, mcu_rows, y_per_mcu, restart_interval, 0,
                            (int64_t)mcus_per_row * mcu_rows, n_threads);
}

// MCU rows [row0, row0+n_rows) of a scan: the restart intervals covering
// them (every block of those intervals written); a shard of a large image
// (BASELINE config 4) decodes only its own intervals.
hj_status hj_decode_scan_rows(const void *fast, const uint8_t *data, int64_t n, int16_t *y, int16_t *cb,
                              int16_t *cr, int32_t mcus_per_row, int32_t mcu_rows, int32_t y_per_mcu,
                              int32_t restart_interval, int32_t row0, int32_t n_rows, int32_t n_threads) {
    const Tables *f = static_cast<const Tables *>(fast);
    if (!f || (!data && n) || !y || !cb || !cr || n < 0 || mcus_per_row < 0 || mcu_rows < 0 ||
        y_per_mcu < 1 || y_per_mcu > 4 || row0 < 0 || n_rows < 0 || row0 + n_rows > mcu_rows)
        return hj::fail(HJ_ERR_ARG, "hj_decode_scan_rows: bad arguments");
    if (n_rows == 0) return HJ_OK;
    return decode_scan_mcus(f, data, n, y, cb, cr, mcus_per_row, mcu_rows, y_per_mcu, restart_interval,
                            (int64_t)row0 * mcus_per_row, (int64_t)(row0 + n_rows) * mcus_per_row, n_threads);
}

// The drop-in cursor: MCU rows [row0, row0+n_rows) from / to the reference's
// int64[8] state {pos, bitbuf, bits, mcus_since_rst, next_rst, predY, predCb,
// predCr} (kernels/_native.pyx:195-305), written back on error too.
hj_status hj_decode_mcu_rows(const uint8_t *data, int64_t n, int64_t *state, const hj_scan_tables_t *scan,
                             int16_t *y_out, int16_t *cb_out, int16_t *cr_out, int32_t row0, int32_t n_rows,
                             int32_t mcus_per_row, int32_t y_per_mcu, int32_t restart_interval) {
    if (!state || !scan || !y_out || !cb_out || !cr_out || n < 0 || (!data && n))
        return hj::fail(HJ_ERR_ARG, "hj_decode_mcu_rows: null pointer or negative length");
    if (y_per_mcu < 1 || y_per_mcu > 4 || mcus_per_row < 0 || n_rows < 0)
        return hj::fail(HJ_ERR_ARG, "hj_decode_mcu_rows: bad geometry");
    if (state[0] < 0 || state[0] > n || state[2] < 0 || state[2] > 56)
        return hj::fail(HJ_ERR_ARG, "hj_decode_mcu_rows: cursor state outside the data");
    const Tables *f = cursor_tables(scan);
    if (!f) return hj::fail(HJ_ERR_ARG, "hj_decode_mcu_rows: component table slot outside 0..7");

    Reader br(data + state[0], data + n, (uint64_t)state[1], (int)state[2]);
    Track tr;
    bool touched = false;  // any operation since the reader's origin
    int64_t since = state[3], next_rst = state[4];
    int64_t preds[3] = {state[5], state[6], state[7]};
    int err = HJ_OK;
    int64_t pos_override = -1;  // reader parked at a restart check

    const int64_t m_begin = (int64_t)row0 * mcus_per_row, m_end = m_begin + (int64_t)n_rows * mcus_per_row;
    int64_t mcu = m_begin;
    while (mcu < m_end && err == HJ_OK) {
        if (restart_interval != 0 && since == restart_interval) {
            const int64_t pos = touched ? ref_state(br, data, tr).pos : (br.org - data);
            err = check_restart(data, n, pos, next_rst);
            if (err) {
                pos_override = pos;  // the reference cleared its buffer before the check
                break;
            }
            br = Reader(data + pos + 2, data + n);
            tr = Track();
            touched = false;
            next_rst = (next_rst + 1) & 7;
            preds[0] = preds[1] = preds[2] = 0;
            since = 0;
        }
        // decode up to the next restart point (or the end of the range)
        int64_t run = m_end - mcu;
        if (restart_interval != 0) run = std::min<int64_t>(run, restart_interval - since);
        int64_t done = 0;
        touched = touched || run > 0;
        err = decode_mcus<false, true>(*f, br, mcu, mcu + run, y_per_mcu, y_out, cb_out, cr_out, preds, &tr, &done);
        mcu += done;
        since += done;
    }

    if (pos_override >= 0) {
        state[0] = pos_override;
        state[1] = 0;
        state[2] = 0;
    } else if (touched) {
        const RefState rs = ref_state(br, data, tr);
        state[0] = rs.pos;
        state[1] = (int64_t)rs.buf;
        state[2] = rs.bits;
    }
    state[3] = since;
    state[4] = next_rst;
    state[5] = preds[0];
    state[6] = preds[1];
    state[7] = preds[2];
    if (err) return hj::fail((hj_status)err, status_name(err));
    return HJ_OK;
}

int64_t hj_scan_entropy_end(const uint8_t *data, int64_t n, int64_t start) {
    int64_t pos = start;
    while (pos < n - 1) {
        const void *ff = std::memchr(data + pos, 0xFF, (size_t)(n - 1 - pos));
        if (!ff) return -1;
        pos = static_cast<const uint8_t *>(ff) - data;
        const uint8_t nxt = data[pos + 1];
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
