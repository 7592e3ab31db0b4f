"""Host Huffman decoders on corrupt streams, against the REFERENCE.

tests/golden/huffman_fuzz.json (tests/golden/make_huffman_fuzz.py) holds 600
seeded corruptions of golden entropy-coded spans (RST and non-RST, 4:4:4 /
4:2:2 / 4:2:0) with the reference native decoder's cursor state after every
MCU row, its first error and the coefficient planes' SHA-256.  Replayed here:

  * the drop-in cursor (kernels.cuda.decode_mcu_rows -> hj_decode_mcu_rows):
    identical state after every row, identical error class on the same row,
    identical planes;
  * the whole-scan decoder (FastScan -> hj_decode_scan_fast, 1 and 4
    threads): the same first error class, identical planes when the
    reference succeeds - in particular an interval whose bits do not end at
    its RSTn fails as in the reference (_native.pyx:238-257).
"""
import hashlib
import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.join(HERE, "golden"))

from paper_1311_5304_b200 import _lib, entropy, errors, parser  # noqa: E402
from paper_1311_5304_b200.kernels import cuda  # noqa: E402

from make_huffman_fuzz import apply_ops  # noqa: E402

with open(os.path.join(HERE, "golden", "huffman_fuzz.json")) as fh:
    FUZZ = json.load(fh)["cases"]

ERR = {errors.BitstreamExhausted: "exhausted", errors.BadCode: "badcode", errors.MarkerInScan: "marker"}
_SPANS = {}


def _base(name):
    if name not in _SPANS:
        z = np.load(os.path.join(HERE, "golden", name + ".npz"))
        blob = bytes(z["jpeg"])
        p = parser.parse_stream(blob)
        sp = p.entropy_span
        packed = entropy._pack_scan_tables(p)
        _SPANS[name] = (p, blob[sp.offset:sp.offset + sp.length], cuda.prepare_scan(*packed))
    return _SPANS[name]


def _planes(c):
    n = c["mcus_per_row"] * c["mcu_rows"]
    return (np.zeros((n * c["ypm"], 64), np.int16), np.zeros((n, 64), np.int16), np.zeros((n, 64), np.int16))


def _sha(y, cb, cr):
    return hashlib.sha256(y.tobytes() + cb.tobytes() + cr.tobytes()).hexdigest()


@pytest.mark.parametrize("k", range(0, len(FUZZ), 10))
def test_cursor_matches_reference_on_corrupt_streams(k):
    for c in FUZZ[k:k + 10]:
        p, span, scan = _base(c["base"])
        data = apply_ops(span, c["ops"])
        y, cb, cr = _planes(c)
        st = np.zeros(8, np.int64)
        states, err = [], None
        for row in range(c["mcu_rows"]):
            try:
                cuda.decode_mcu_rows(data, st, scan, y, cb, cr, row, 1, c["mcus_per_row"], c["ypm"],
                                     c["restart_interval"])
            except tuple(ERR) as e:
                err = [row, ERR[type(e)]]
                states.append(st.tolist())
                break
            states.append(st.tolist())
        want_err = c["error"][:2] if c["error"] else None
        assert err == want_err, (c["base"], c["ops"])
        assert states == c["states"], (c["base"], c["ops"])
        assert _sha(y, cb, cr) == c["sha256"], (c["base"], c["ops"])


_STATUS = {_lib.HJ_ERR_EXHAUSTED: "exhausted", _lib.HJ_ERR_BADCODE: "badcode", _lib.HJ_ERR_MARKER: "marker",
           _lib.HJ_ERR_RST_SEQ: "marker"}


@pytest.mark.parametrize("threads", [1, 4])
def test_fast_scan_matches_reference_on_corrupt_streams(threads):
    import ctypes as C
    bad = []
    for c in FUZZ:
        p, span, scan = _base(c["base"])
        data = np.frombuffer(apply_ops(span, c["ops"]), np.uint8)
        y, cb, cr = _planes(c)
        h = C.c_void_p()
        _lib.check(_lib.lib.hj_huff_build(C.byref(scan), C.byref(h)), "hj_huff_build")
        try:
            st = _lib.lib.hj_decode_scan_fast(h.value, data.ctypes.data if len(data) else None, len(data),
                                              y.ctypes.data, cb.ctypes.data, cr.ctypes.data, c["mcus_per_row"],
                                              c["mcu_rows"], c["ypm"], c["restart_interval"], threads)
        finally:
            _lib.lib.hj_huff_free(h.value)
        got = None if st == 0 else _STATUS.get(st, f"status {st}")
        want = c["error"][1] if c["error"] else None
        if got != want or (want is None and _sha(y, cb, cr) != c["sha256"]):
            bad.append((c["base"], c["ops"], got, want))
    assert not bad, f"{len(bad)} of {len(FUZZ)} differ, e.g. {bad[:5]}"


def test_fuzz_fixture_exercises_restart_errors():
    # the corpus covers the restart-specific failure modes of ADVICE r01
    rst_err = [c for c in FUZZ if c["restart_interval"] and c["error"]]
    assert len(rst_err) > 100
    assert {c["error"][1] for c in rst_err} >= {"exhausted", "badcode", "marker"}


def test_cursor_state_is_chunking_invariant():
    # the reference's cursor state after row r does not depend on how the
    # rows were grouped into calls; ours neither (3-row chunks here)
    for c in FUZZ[::7]:
        p, span, scan = _base(c["base"])
        data = apply_ops(span, c["ops"])
        y, cb, cr = _planes(c)
        st = np.zeros(8, np.int64)
        row = 0
        while row < c["mcu_rows"]:
            n = min(3, c["mcu_rows"] - row)
            try:
                cuda.decode_mcu_rows(data, st, scan, y, cb, cr, row, n, c["mcus_per_row"], c["ypm"],
                                     c["restart_interval"])
            except tuple(ERR):
                assert c["error"] and row <= c["error"][0] < row + n
                assert st.tolist() == c["states"][-1]
                break
            row += n
            assert st.tolist() == c["states"][row - 1], (c["base"], c["ops"], row)
        assert _sha(y, cb, cr) == c["sha256"]


def _dc_wrap_cases():
    z = np.load(os.path.join(HERE, "golden", "dc_wrap.npz"))
    return [(k[:-5], bytes(z[k]), z[k[:-5] + "_y"], z[k[:-5] + "_cb"], z[k[:-5] + "_cr"])
            for k in z.files if k.endswith("_jpeg")]


@pytest.mark.parametrize("case", _dc_wrap_cases(), ids=lambda c: c[0])
@pytest.mark.parametrize("threads", [1, 3])
def test_dc_predictor_wraps_like_the_reference(case, threads):
    """DC predictors run far past int16 (crafted scans, tests/golden/
    make_dc_wrap.py): accumulate in 64 bits, wrap on store
    (_native.pyx:162-163) - the cursor and the whole-scan decoder."""
    name, blob, y, cb, cr = case
    p = parser.parse_stream(blob)
    c, cur = entropy.decode_all(p, blob)
    assert np.array_equal(c.y_blocks, y) and np.array_equal(c.cb_blocks, cb) and np.array_equal(c.cr_blocks, cr)
    assert max(abs(v) for v in cur.dc_predictors) < 2 ** 40
    fs = entropy.FastScan(p)
    out = fs.decode(blob, threads=threads)
    assert np.array_equal(out.y_blocks, y) and np.array_equal(out.cb_blocks, cb) and np.array_equal(out.cr_blocks, cr)
