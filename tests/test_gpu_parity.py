"""Parity of the sm_100a parallel phase with the reference (golden fixtures:
the reference's own render_rows output for 4:4:4/4:2:2) and with the CPU
oracle (4:2:0 extension, full BASELINE sizes, adversarial inputs).
Bar: bit-exact RGB.  Calls go through the C ABI (ctypes)."""
import os
import threading

import numpy as np
import pytest

from conftest import GOLDEN_CASES
from oracle import oracle

pytestmark = pytest.mark.gpu

RENDER = {0: "render_rows_444", 1: "render_rows_422", 2: "render_rows_420"}


@pytest.fixture(scope="module")
def cuda():
    from paper_1311_5304_b200 import _lib
    from paper_1311_5304_b200.kernels import cuda as backend
    _lib.require_device()
    return backend


def _render(cuda, g, fast=True, row0=0, n_rows=None, rgb=None, y=None, cb=None, cr=None, q=None):
    mh = 16 if g.sub == 2 else 8
    mw = 8 if g.sub == 0 else 16
    rows = -(-g.height // mh)
    n_rows = rows - row0 if n_rows is None else n_rows
    rgb = np.zeros((g.height, g.width, 3), np.uint8) if rgb is None else rgb
    getattr(cuda, RENDER[g.sub])(g.y if y is None else y, g.cb if cb is None else cb,
                                 g.cr if cr is None else cr, g.q if q is None else q, rgb,
                                 g.width, g.height, -(-g.width // mw), row0, n_rows, fast, True)
    return rgb


@pytest.mark.parametrize("g", GOLDEN_CASES, ids=repr)
@pytest.mark.parametrize("fast", [True, False], ids=["aan", "direct"])
def test_render_matches_golden(cuda, g, fast):
    assert np.array_equal(_render(cuda, g, fast), g.rgb if fast else g.rgb_direct)


@pytest.mark.parametrize("g", [c for c in GOLDEN_CASES if c.meta["mcu_rows"] >= 3], ids=repr)
def test_partial_row_ranges(cuda, g):
    rows = g.meta["mcu_rows"]
    rng = np.random.default_rng(len(g.name))
    rgb = np.full((g.height, g.width, 3), 7, np.uint8)
    r = 0
    while r < rows:
        n = int(rng.integers(1, 4))
        n = min(n, rows - r)
        _render(cuda, g, True, r, n, rgb)
        r += n
    assert np.array_equal(rgb, g.rgb)
    # a zero-row call is a no-op
    _render(cuda, g, True, 0, 0, rgb)


def test_concurrent_disjoint_ranges(cuda):
    g = max((c for c in GOLDEN_CASES if c.sub == 1), key=lambda c: c.width * c.height)
    rows = g.meta["mcu_rows"]
    rgb = np.zeros((g.height, g.width, 3), np.uint8)
    spans = [(r, min(4, rows - r)) for r in range(0, rows, 4)]
    errs = []

    def work(chunk):
        try:
            for r0, n in chunk:
                _render(cuda, g, True, r0, n, rgb)
        except Exception as e:  # pragma: no cover
            errs.append(e)

    ts = [threading.Thread(target=work, args=(spans[i::4],)) for i in range(4)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    assert not errs
    assert np.array_equal(rgb, g.rgb)


def test_idct_blocks_match_reference(blocks_golden):
    from paper_1311_5304_b200 import block_transforms as bt
    deq = blocks_golden["deq"]
    assert np.array_equal(bt.idct_fast(deq), blocks_golden["fast"])
    assert np.array_equal(bt.idct_direct(deq), blocks_golden["direct"])
    f64 = bt.idct_fast_f64(deq[:256]).reshape(256, 64)
    assert np.array_equal(f64.view(np.uint64), blocks_golden["f64_fast"].view(np.uint64))
    f64d = bt.idct_direct_f64(deq[:256]).reshape(256, 64)
    assert np.array_equal(f64d.view(np.uint64), blocks_golden["f64_direct"].view(np.uint64))
    # SPEC.md:173-174,181-182
    z = np.zeros(64, np.int32)
    dc = z.copy()
    dc[0] = 240
    assert (bt.idct_fast(z) == 128).all() and (bt.idct_direct(dc) == 158).all()


def test_colour_exhaustive_on_gpu():
    from paper_1311_5304_b200 import block_transforms as bt
    v = np.arange(256, dtype=np.uint8)
    y, cb, cr = (a.reshape(-1) for a in np.meshgrid(v, v, v, indexing="ij"))
    r, g, b = bt.ycbcr_to_rgb(y, cb, cr)
    want = oracle.ycbcr_to_rgb(y, cb, cr)
    assert np.array_equal(np.stack([r, g, b], -1), want)
    # SPEC.md:199-201
    assert [int(c) for c in bt.ycbcr_to_rgb(76, 85, 255)] == [254, 0, 0]


def test_upsample_row_422_spec():
    from paper_1311_5304_b200 import block_transforms as bt
    ramp = np.arange(0, 32, 4)
    assert bt.upsample_row_422(ramp).tolist() == [0, 1, 3, 5, 7, 9, 11, 13, 15, 17, 19, 21, 23,
                                                  25, 27, 28]
    assert (bt.upsample_row_422([9] * 8) == 9).all()
    out = bt.upsample_row_422(ramp, left=10, right=40)
    assert out[0] == (0 * 3 + 10 + 1) // 4 and out[15] == (28 * 3 + 40 + 2) // 4
    rgb = bt.fused_upsample_color_422(np.full(16, 90), ramp, ramp[::-1])
    r, g, b = bt.ycbcr_to_rgb(np.full(16, 90), bt.upsample_row_422(ramp),
                              bt.upsample_row_422(ramp[::-1]))
    assert np.array_equal(rgb, np.stack([r, g, b], -1))


def test_fused_444_single_mcu(cuda):
    from paper_1311_5304_b200 import block_transforms as bt
    rng = np.random.default_rng(3)
    blocks = rng.integers(-60, 60, size=(3, 64)).astype(np.int16)
    q = rng.integers(1, 40, size=(3, 64)).astype(np.int32)
    got = bt.fused_idct_color_444(blocks[0], blocks[1], blocks[2], q[0], q[1], q[2])
    want = oracle.render(blocks[0:1], blocks[1:2], blocks[2:3], q, 8, 8, 0)
    assert np.array_equal(got, want.reshape(64, 3))


def _synthetic(width, height, quality, sub, **kw):
    from paper_1311_5304_b200 import entropy, parser
    from paper_1311_5304_b200.perf_model import qtable_stack
    from paper_1311_5304_b200.synth import synth_jpeg
    blob = synth_jpeg(width, height, quality, sub, **kw)
    p = parser.parse_stream(blob)
    coeffs, _ = entropy.decode_all(p, blob)
    return p, coeffs, qtable_stack(p)


@pytest.mark.parametrize("w,h,q,sub,kw", [
    (512, 512, 75, "420", {}),
    (1920, 1080, 90, "420", {}),
    (4096, 4096, 95, "444", {}),
    (4096, 4096, 95, "422", {}),
    (6000, 4000, 90, "420", {"restart_rows": 1}),
    (1023, 769, 85, "422", {"restart_blocks": 5}),
    (1001, 999, 80, "420", {}),
    (1922, 700, 70, "444", {}),   # rows start 2 bytes off a word: funnel-shifted stores
    (1928, 300, 80, "444", {}),   # width 8 mod 16: every row ends in a 24-byte half item
    (1925, 300, 60, "422", {}),   # rows at every byte offset
], ids=["512_420", "1080p_420", "4096_444", "4096_422", "24MP_420_rst", "odd_422", "odd_420", "w2mod4_444",
        "w8mod16_444", "w1mod4_422"])
def test_full_size_against_oracle(w, h, q, sub, kw):
    from paper_1311_5304_b200.block_transforms import alloc_pixels, render_rows
    p, coeffs, qt = _synthetic(w, h, q, sub, **kw)
    px = alloc_pixels(w, h)
    render_rows(coeffs, qt, px, 0, coeffs.geometry.mcu_rows)
    want = oracle.render(coeffs.y_blocks, coeffs.cb_blocks, coeffs.cr_blocks, qt, w, h,
                         {"444": 0, "422": 1, "420": 2}[sub], True, threads=16)
    assert np.array_equal(px.data, want)


@pytest.mark.parametrize("w,h,q,sub,kw", [
    (1920, 1080, 90, "420", {}),
    (1001, 999, 80, "420", {}),
    (1925, 300, 60, "422", {"restart_blocks": 7}),
    (1922, 700, 70, "444", {}),
], ids=["1080p_420", "odd_420", "w1mod4_422_rst", "w2mod4_444"])
def test_direct_idct_full_size_against_oracle(w, h, q, sub, kw):
    """idct="direct" at BASELINE-like sizes: by default these images run on the
    tensor-core screen kernel - its exact direct-basis map,
    the rounded T00^2 DC bias and the exact fallback against the oracle."""
    from paper_1311_5304_b200.block_transforms import alloc_pixels, render_rows
    p, coeffs, qt = _synthetic(w, h, q, sub, **kw)
    px = alloc_pixels(w, h)
    render_rows(coeffs, qt, px, 0, coeffs.geometry.mcu_rows, fast=False)
    want = oracle.render(coeffs.y_blocks, coeffs.cb_blocks, coeffs.cr_blocks, qt, w, h,
                         {"444": 0, "422": 1, "420": 2}[sub], False, threads=16)
    assert np.array_equal(px.data, want)


@pytest.mark.parametrize("sub", [0, 1, 2])
def test_adversarial_coefficients(cuda, sub):
    """Extreme int16 coefficients, q up to 255 (saturation on both ends),
    sparse DC-only blocks and rounding-tie DC values."""
    rng = np.random.default_rng(100 + sub)
    w, h = 203, 77
    mw, mh, ypm = {0: (8, 8, 1), 1: (16, 8, 2), 2: (16, 16, 4)}[sub]
    mpr, rows = -(-w // mw), -(-h // mh)
    n_c = mpr * rows
    y = rng.integers(-32768, 32768, size=(n_c * ypm, 64)).astype(np.int16)
    cb = rng.integers(-3000, 3000, size=(n_c, 64)).astype(np.int16)
    cr = (rng.integers(-40, 40, size=(n_c, 64)) * (rng.random((n_c, 64)) < 0.2)).astype(np.int16)
    cr[::3, 1:] = 0
    cr[::3, 0] = rng.integers(-64, 64, size=len(cr[::3])) * 4 + 1  # DC-only, tie family
    q = np.stack([rng.integers(1, 256, 64), rng.integers(1, 256, 64), np.full(64, 1)]).astype(np.int32)

    class G:  # minimal golden-like record
        pass
    g = G()
    g.sub, g.width, g.height, g.y, g.cb, g.cr, g.q = sub, w, h, y, cb, cr, q
    for fast in (True, False):
        got = _render(cuda, g, fast)
        want = oracle.render(y, cb, cr, q, w, h, sub, fast)
        assert np.array_equal(got, want)


def test_device_batch_mixed_subsamplings(cuda):
    from paper_1311_5304_b200 import device, entropy, parser
    cases = [c for c in GOLDEN_CASES if c.width * c.height > 1000]
    geos, coeffs = [], []
    for c in cases:
        p = parser.parse_stream(c.jpeg)
        cf, _ = entropy.decode_all(p, c.jpeg)
        geos.append(cf.geometry)
        coeffs.append(cf)
    batch = device.DeviceBatch(geos)
    s = device.Stream()
    for i, (c, cf) in enumerate(zip(cases, coeffs)):
        batch.upload_coefficients(i, cf, s)
        batch.upload_qtables(i, c.q, s)
    batch.render(stream=s)
    outs = [np.zeros((c.height, c.width, 3), np.uint8) for c in cases]
    for i, o in enumerate(outs):
        batch.download_rgb(i, o, s)
    s.synchronize()
    for c, o in zip(cases, outs):
        assert np.array_equal(o, c.rgb), c.name


@pytest.mark.parametrize("world", [2, 3, 8])
def test_mcu_row_sharding_with_only_local_coefficients(cuda, world):
    """BASELINE config 4: one large 4:2:0 image with restart intervals split
    into contiguous MCU-row shards, each 'rank' holding ONLY its rows plus
    one chroma MCU row of context on each side (shard.chroma_context) on its
    own device batch; the stitched RGB equals the oracle's whole-image render."""
    from paper_1311_5304_b200 import device, entropy, parser, shard
    from paper_1311_5304_b200.perf_model import qtable_stack
    from paper_1311_5304_b200.synth import synth_jpeg
    blob = synth_jpeg(1200, 800, 90, "420", seed=5, restart_rows=1)
    p = parser.parse_stream(blob)
    c, _ = entropy.decode_all(p, blob, pinned=True)
    q = qtable_stack(p)
    g = c.geometry
    want = oracle.render(c.y_blocks, c.cb_blocks, c.cr_blocks, q, g.width, g.height, 2)
    got = np.zeros_like(want)
    s = device.Stream()
    for row0, n in shard.split_rows(g.mcu_rows, world):
        lo, hi = shard.chroma_context(row0, n, g.mcu_rows)
        db = device.DeviceBatch([g])
        _lib_memset_poison(db)
        db.upload_coefficients(0, c, s, row0=lo, n_rows=hi - lo)
        db.upload_qtables(0, q, s)
        db.render_items([(0, row0, n)], s)
        y0, y1 = row0 * 16, min(g.height, (row0 + n) * 16)
        db.download_rgb(0, got, s, y0=y0, y1=y1)
        s.synchronize()
        db.close()
    assert np.array_equal(got, want)


def _lib_memset_poison(db):
    """Fill the device coefficients with a pattern, so a shard reading rows it
    does not own would change the output."""
    from paper_1311_5304_b200 import _lib
    _lib.check(_lib.lib.hj_memset_device(db.coef.ptr, 0x5A, db.coef.nbytes, None), "poison")
    _lib.check(_lib.lib.hj_device_synchronize(), "sync")


@pytest.mark.parametrize("sub", ["444", "422", "420"])
def test_strip_widths_sweep(cuda, sub):
    """Widths around every strip / MCU-pair boundary, rendered as one small
    batch (narrowed strips) and one image at a time, against the oracle:
    the tile planner must cover every MCU column exactly once."""
    from paper_1311_5304_b200 import device, entropy, parser
    from paper_1311_5304_b200.perf_model import qtable_stack
    from paper_1311_5304_b200.synth import synth_jpeg
    widths = [8, 16, 24, 40, 72, 88, 168, 328, 336, 344, 352, 680, 696, 1000]
    imgs = []
    for k, w in enumerate(widths):
        blob = synth_jpeg(w, 40, 70 + k, sub, seed=k)
        p = parser.parse_stream(blob)
        c, _ = entropy.decode_all(p, blob)
        imgs.append((c, qtable_stack(p)))
    code = {"444": 0, "422": 1, "420": 2}[sub]
    for group in (list(range(len(imgs))), [len(imgs) - 1], [0]):
        batch = device.DeviceBatch([imgs[i][0].geometry for i in group])
        s = device.Stream()
        for j, i in enumerate(group):
            batch.upload_coefficients(j, imgs[i][0], s)
            batch.upload_qtables(j, imgs[i][1], s)
        batch.render(stream=s)
        for j, i in enumerate(group):
            c, q = imgs[i]
            g = c.geometry
            out = np.zeros((g.height, g.width, 3), np.uint8)
            batch.download_rgb(j, out, s)
            s.synchronize()
            want = oracle.render(c.y_blocks, c.cb_blocks, c.cr_blocks, q, g.width, g.height, code, True)
            assert np.array_equal(out, want), (sub, g.width)
        batch.close()


def _single_ops():
    return np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "single_ops.npz"))


def test_single_mcu_forms_match_reference_vectors(cuda):
    """upsample_row_422 / fused_upsample_color_422 / fused_idct_color_444
    against the reference's own outputs (tests/golden/make_single_ops.py),
    including the float64 G tie pair (Cb, Cr) = (78, 178)."""
    from paper_1311_5304_b200 import block_transforms as bt
    z = _single_ops()
    nb = lambda v: None if v < 0 else int(v)  # noqa: E731
    for r, a, b, want in zip(z["up_rows"], z["up_left"], z["up_right"], z["up_out"]):
        assert bt.upsample_row_422(r, nb(a), nb(b)).tolist() == want.tolist()
    for y, cb, cr, k, want in zip(z["f422_y"], z["f422_cb"], z["f422_cr"], z["f422_nb"], z["f422_out"]):
        got = bt.fused_upsample_color_422(y, cb, cr, *[nb(v) for v in k])
        assert np.array_equal(got, want)
    for blk, q, wf, wd in zip(z["f444_blocks"], z["f444_q"], z["f444_fast"], z["f444_direct"]):
        assert np.array_equal(bt.fused_idct_color_444(*blk, *q, fast=True), wf)
        assert np.array_equal(bt.fused_idct_color_444(*blk, *q, fast=False), wd)


def _h2v2_pin_cases():
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "h2v2_pin.npz"))
    return [(k[:-5], bytes(z[k]), z[k[:-5] + "_rgb"]) for k in z.files if k.endswith("_jpeg")]


@pytest.mark.parametrize("case", _h2v2_pin_cases(), ids=lambda c: c[0])
def test_render_420_pinned_to_libjpeg_turbo(cuda, case):
    """The 4:2:0 render kernel against libjpeg-turbo's h2v2 fancy upsampler
    (DC-only 16-aligned images, tests/golden/make_h2v2_pin.py), through the
    drop-in render_rows and through a device batch."""
    from paper_1311_5304_b200 import device, entropy, parser
    from paper_1311_5304_b200.block_transforms import alloc_pixels, render_rows
    from paper_1311_5304_b200.perf_model import qtable_stack
    name, blob, want = case
    p = parser.parse_stream(blob)
    c, _ = entropy.decode_all(p, blob)
    q = qtable_stack(p)
    px = alloc_pixels(p.width, p.height)
    render_rows(c, q, px, 0, c.geometry.mcu_rows)
    assert np.array_equal(px.data, want)
    db = device.DeviceBatch([c.geometry, c.geometry])
    st = device.Stream()
    for i in range(2):
        db.upload_coefficients(i, c, st)
        db.upload_qtables(i, q, st)
    db.render(stream=st)
    out = np.zeros_like(want)
    db.download_rgb(1, out, st)
    st.synchronize()
    db.close()
    assert np.array_equal(out, want)
