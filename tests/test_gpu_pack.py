"""The drop-in's packed coefficient transfer (csrc/hj_pack.{h,cpp}, device
unpack in hj_blockops.cu) under the whole GPU parity suite with
packing forced on (HJ_PACK_H2D=1; by default it engages only when several
host threads call the drop-in at once): goldens, partial row ranges, the
4:2:0 chroma context rows, BASELINE sizes, adversarial int16 coefficients
(wide blocks) - bit-exact RGB, in a subprocess because the switch is read
once per process."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_parity_suite_with_packed_transfer():
    env = dict(os.environ, HJ_PACK_H2D="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_parity_suite_with_banded_transfer():
    """The banded path of large packed calls, forced onto every call above 96
    blocks (bands of one or a few MCU rows: the 4:2:0 chroma context row of
    each band comes from the next band's upload)."""
    env = dict(os.environ, HJ_PACK_H2D="1", HJ_PACK_BAND="96")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("sub", ["420", "422", "444"])
def test_large_call_packed_in_bands(sub):
    """A call above the 64k-block single-record limit, packing forced: sent in
    bands at the default band size, bit-exact, fewer bytes than dense; also a
    partial MCU-row window of it."""
    from oracle import oracle
    from paper_1311_5304_b200 import _lib, entropy, parser
    from paper_1311_5304_b200.block_transforms import alloc_pixels, render_rows
    from paper_1311_5304_b200.perf_model import qtable_stack
    from paper_1311_5304_b200.synth import synth_jpeg
    _lib.require_device()
    w, h = {"420": (2400, 1800), "422": (2000, 1500), "444": (1600, 1200)}[sub]
    blob = synth_jpeg(w, h, 85, sub, seed=9)
    p = parser.parse_stream(blob)
    co, _ = entropy.decode_all(p, blob)
    g = co.geometry
    q = qtable_stack(p)
    dense = 128 * (co.y_blocks.shape[0] + 2 * co.cb_blocks.shape[0])
    assert dense // 128 > 1 << 16
    want = oracle.render(co.y_blocks, co.cb_blocks, co.cr_blocks, q, w, h, {"444": 0, "422": 1, "420": 2}[sub])
    try:
        assert _lib.lib.hj_set_packed_h2d(1) == 0
        px = alloc_pixels(w, h)
        b0 = _lib.lib.hj_h2d_bytes()
        render_rows(co, q, px, 0, g.mcu_rows)
        moved = _lib.lib.hj_h2d_bytes() - b0
        assert np.array_equal(px.data, want)
        assert moved < 0.6 * dense, (moved, dense)
        # rows [r0, r0 + n) of the same image (a band boundary inside, chroma context at both ends)
        r0, n = g.mcu_rows // 5, g.mcu_rows // 2
        assert _lib.lib.hj_set_pack_band(4000) == 0
        px2 = alloc_pixels(w, h)
        render_rows(co, q, px2, r0, n)
        mh = g.mcu_height
        y0, y1 = r0 * mh, min(h, (r0 + n) * mh)
        assert np.array_equal(px2.data[y0:y1], want[y0:y1])
    finally:
        _lib.lib.hj_set_packed_h2d(-1)
        _lib.lib.hj_set_pack_band(0)


def test_packed_transfer_moves_fewer_bytes():
    from oracle import oracle
    from paper_1311_5304_b200 import _lib, entropy, parser
    from paper_1311_5304_b200.block_transforms import alloc_pixels, render_rows
    from paper_1311_5304_b200.perf_model import qtable_stack
    from paper_1311_5304_b200.synth import synth_jpeg
    _lib.require_device()
    blob = synth_jpeg(1920, 1080, 90, "420", seed=5)
    p = parser.parse_stream(blob)
    co, _ = entropy.decode_all(p, blob)
    g = co.geometry
    q = qtable_stack(p)
    want = oracle.render(co.y_blocks, co.cb_blocks, co.cr_blocks, q, g.width, g.height, 2)
    dense = 128 * (co.y_blocks.shape[0] + 2 * co.cb_blocks.shape[0])
    moved = {}
    try:
        for mode in (1, 0):
            assert _lib.lib.hj_set_packed_h2d(mode) == 0
            px = alloc_pixels(g.width, g.height)
            b0 = _lib.lib.hj_h2d_bytes()
            render_rows(co, q, px, 0, g.mcu_rows)
            moved[mode] = _lib.lib.hj_h2d_bytes() - b0
            assert np.array_equal(px.data, want), mode
    finally:
        _lib.lib.hj_set_packed_h2d(-1)
    assert moved[0] >= dense
    assert moved[1] < 0.5 * dense, (moved, dense)


@pytest.mark.parametrize("band", [0, 96])
def test_packed_transfer_concurrent_mixed_calls(band):
    """8 threads calling the drop-in at once (the automatic packing policy's
    trigger) on different sizes, subsamplings, qualities and IDCT modes - every
    output bit-exact against the oracle."""
    import threading

    from oracle import oracle
    from paper_1311_5304_b200 import _lib, entropy, parser
    from paper_1311_5304_b200.block_transforms import alloc_pixels, render_rows
    from paper_1311_5304_b200.perf_model import qtable_stack
    from paper_1311_5304_b200.synth import synth_jpeg
    _lib.require_device()
    cases = []
    rng = np.random.default_rng(11)
    for i in range(16):
        w, h = int(rng.integers(64, 700)), int(rng.integers(48, 500))
        sub = ["444", "422", "420"][i % 3]
        blob = synth_jpeg(w, h, int(rng.integers(40, 96)), sub, seed=i)
        p = parser.parse_stream(blob)
        co, _ = entropy.decode_all(p, blob)
        q = qtable_stack(p)
        fast = bool(i % 4)
        want = oracle.render(co.y_blocks, co.cb_blocks, co.cr_blocks, q, w, h, {"444": 0, "422": 1, "420": 2}[sub], fast)
        cases.append((co, q, w, h, fast, want))
    errs = []

    def work(k):
        try:
            for rep in range(3):
                for co, q, w, h, fast, want in cases[k::8]:
                    px = alloc_pixels(w, h)
                    render_rows(co, q, px, 0, co.geometry.mcu_rows, fast=fast)
                    if not np.array_equal(px.data, want):
                        errs.append((w, h, fast))
        except Exception as e:  # pragma: no cover
            errs.append(e)

    b0 = _lib.lib.hj_h2d_bytes()
    # 96: every call that packs goes in bands, each band packed while >= 4 calls are in flight, else dense
    assert _lib.lib.hj_set_pack_band(band) == 0
    try:
        ts = [threading.Thread(target=work, args=(k,)) for k in range(8)]
        [t.start() for t in ts]
        [t.join() for t in ts]
    finally:
        _lib.lib.hj_set_pack_band(0)
    assert not errs, errs[:3]
    assert _lib.lib.hj_h2d_bytes() > b0
