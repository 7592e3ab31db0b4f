"""The CPU oracle against the reference's own outputs (golden fixtures made
by tests/golden/make_golden.py from /root/reference) and the SPEC.md
known-answer vectors.  CPU only."""
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
