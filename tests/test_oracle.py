"""The CPU oracle against the reference's own outputs (golden fixtures made
by tests/golden/make_golden.py from /root/reference) and the SPEC.md
known-answer vectors.  CPU only."""
import os

import numpy as np
import pytest

from conftest import GOLDEN_CASES
from oracle import oracle

REF_CASES = [g for g in GOLDEN_CASES if g.sub in (0, 1)]


@pytest.mark.parametrize("g", REF_CASES, ids=repr)
@pytest.mark.parametrize("fast", [True, False])
def test_oracle_matches_reference_render(g, fast):
    want = g.rgb if fast else g.rgb_direct
    got = oracle.render(g.y, g.cb, g.cr, g.q, g.width, g.height, g.sub, fast=fast)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("g", REF_CASES, ids=repr)
def test_oracle_row_chunks_and_threads(g):
    # rendering in chunks / threads must not change bytes (SPEC "determinism")
    rows = -(-g.height // 8)
    rgb = np.zeros((g.height, g.width, 3), np.uint8)
    r = 0
    while r < rows:
        n = min(3, rows - r)
        oracle.render(g.y, g.cb, g.cr, g.q, g.width, g.height, g.sub, row0=r, n_rows=n, rgb=rgb)
        r += n
    assert np.array_equal(rgb, g.rgb)
    assert np.array_equal(oracle.render(g.y, g.cb, g.cr, g.q, g.width, g.height, g.sub,
                                        threads=4), g.rgb)


def test_oracle_blocks_match_reference(blocks_golden):
    deq = blocks_golden["deq"]
    q1 = np.ones(64, np.int32)
    # deq values exceed int16: route through the f64 core instead
    for i in range(0, 256, 7):
        for fast, key in ((True, "f64_fast"), (False, "f64_direct")):
            core = oracle.idct_core_f64(deq[i], fast)
            assert np.array_equal(core.view(np.uint64), blocks_golden[key][i].view(np.uint64))
    small = np.abs(deq).max(axis=1) < 32768
    coef = deq[small].astype(np.int16)
    assert np.array_equal(oracle.idct_blocks(coef, q1, True), blocks_golden["fast"][small])
    assert np.array_equal(oracle.idct_blocks(coef, q1, False), blocks_golden["direct"][small])


def test_spec_vectors():
    # zero block -> 128, DC 240 -> 158 (both IDCTs)
    q1 = np.ones(64, np.int32)
    z = np.zeros((1, 64), np.int16)
    dc = z.copy()
    dc[0, 0] = 240
    for fast in (True, False):
        assert (oracle.idct_blocks(z, q1, fast) == 128).all()
        assert (oracle.idct_blocks(dc, q1, fast) == 158).all()
    # SPEC.md:199-201 colour conversion
    out = oracle.ycbcr_to_rgb([128, 76, 255], [128, 85, 128], [128, 255, 128])
    assert out.tolist() == [[128, 128, 128], [254, 0, 0], [255, 255, 255]]


def test_oracle_single_mcu_forms_match_reference_vectors():
    """The oracle's render / colour on the reference's single-MCU vectors
    (tests/golden/single_ops.npz, from fallback.py:122-180)."""
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "single_ops.npz"))
    for blk, q, wf, wd in zip(z["f444_blocks"][:60], z["f444_q"][:60], z["f444_fast"][:60], z["f444_direct"][:60]):
        for fast, want in ((True, wf), (False, wd)):
            got = oracle.render(blk[0:1], blk[1:2], blk[2:3], q, 8, 8, 0, fast)
            assert np.array_equal(got.reshape(64, 3), want)
    # colour of the reference-upsampled rows = the reference's fused 4:2:2 rows
    up = lambda r, a, b: [(int(r[0]) if a < 0 else (3 * int(r[0]) + int(a) + 1) // 4)] + [  # noqa: E731
        v for k in range(8) for v in ((3 * int(r[k]) + int(r[k - 1]) + 1) // 4 if k else None,
                                      (3 * int(r[k]) + int(r[k + 1]) + 2) // 4 if k < 7 else None)
        if v is not None] + [int(r[7]) if b < 0 else (3 * int(r[7]) + int(b) + 2) // 4]
    for r, a, b, want in zip(z["up_rows"], z["up_left"], z["up_right"], z["up_out"]):
        assert up(r, a, b) == want.tolist()
    for y, cb, cr, k, want in zip(z["f422_y"], z["f422_cb"], z["f422_cr"], z["f422_nb"], z["f422_out"]):
        got = oracle.ycbcr_to_rgb(y, up(cb, k[0], k[1]), up(cr, k[2], k[3]))
        assert np.array_equal(np.asarray(got).reshape(16, 3), want)


def _h2v2_pin_cases():
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "h2v2_pin.npz"))
    return [(k[:-5], bytes(z[k]), z[k[:-5] + "_rgb"]) for k in z.files if k.endswith("_jpeg")]


@pytest.mark.parametrize("case", _h2v2_pin_cases(), ids=lambda c: c[0])
def test_oracle_420_upsampler_pinned_to_libjpeg_turbo(case):
    """4:2:0 extension vs libjpeg-turbo's h2v2_fancy_upsample on DC-only
    16-aligned images (tests/golden/make_h2v2_pin.py): the RGB the reference
    would produce from libjpeg-turbo's upsampled planes."""
    from paper_1311_5304_b200 import entropy, parser
    from paper_1311_5304_b200.perf_model import qtable_stack
    name, blob, want = case
    p = parser.parse_stream(blob)
    c, _ = entropy.decode_all(p, blob)
    assert not any(np.count_nonzero(b[:, 1:]) for b in (c.y_blocks, c.cb_blocks, c.cr_blocks))  # DC-only
    got = oracle.render(c.y_blocks, c.cb_blocks, c.cr_blocks, qtable_stack(p), p.width, p.height, 2)
    assert np.array_equal(got, want)


from conftest import ISLOW_CASES, rgb_sha  # noqa: E402


@pytest.mark.parametrize("case", ISLOW_CASES, ids=repr)
def test_islow_oracle_matches_libjpeg_turbo(case):
    """The islow-mode oracle (libjpeg_oracle.c) reproduces libjpeg-turbo's
    decode of the same JPEG (tests/golden/make_islow_golden.py)."""
    from paper_1311_5304_b200 import entropy, parser
    from paper_1311_5304_b200.perf_model import qtable_stack
    p = parser.parse_stream(case.jpeg)
    c, _ = entropy.decode_all(p, case.jpeg)
    sub = {8: 0}.get(c.geometry.mcu_width, 1 if c.geometry.mcu_height == 8 else 2)
    got = oracle.render_islow(c.y_blocks, c.cb_blocks, c.cr_blocks, qtable_stack(p), p.width, p.height, sub)
    assert rgb_sha(got) == case.sha


def test_islow_oracle_row_ranges_compose():
    from paper_1311_5304_b200 import entropy, parser
    from paper_1311_5304_b200.perf_model import qtable_stack
    case = [c for c in ISLOW_CASES if "160x96_420" in c.name][0]
    p = parser.parse_stream(case.jpeg)
    c, _ = entropy.decode_all(p, case.jpeg)
    q = qtable_stack(p)
    rgb = np.zeros((p.height, p.width, 3), np.uint8)
    for r0 in range(c.geometry.mcu_rows):
        oracle.render_islow(c.y_blocks, c.cb_blocks, c.cr_blocks, q, p.width, p.height, 2, r0, 1, rgb)
    assert rgb_sha(rgb) == case.sha
