"""The islow decode mode on the B200 (north_star's libjpeg jidctint path):
the render kernel with idct="islow" against libjpeg-turbo's own decode of the
same JPEGs (tests/golden/islow_golden.npz: SHA-256 of Pillow's RGB) and
against the C restatement (oracle/libjpeg_oracle.c) on adversarial and
BASELINE-size inputs."""
import numpy as np
import pytest

from conftest import ISLOW_CASES, has_gpu, rgb_sha
from oracle import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not has_gpu():
        pytest.fail("islow GPU tests need a CUDA device (the product has no CPU path)")


def _decode(blob):
    from paper_1311_5304_b200 import entropy, parser
    from paper_1311_5304_b200.perf_model import qtable_stack
    p = parser.parse_stream(blob)
    c, _ = entropy.decode_all(p, blob)
    g = c.geometry
    sub = {8: 0}.get(g.mcu_width, 1 if g.mcu_height == 8 else 2)
    return p, c, qtable_stack(p), sub


@pytest.mark.parametrize("case", ISLOW_CASES, ids=repr)
def test_islow_render_rows_matches_libjpeg_turbo(case):
    from paper_1311_5304_b200.block_transforms import alloc_pixels, render_rows
    p, c, q, sub = _decode(case.jpeg)
    px = alloc_pixels(p.width, p.height)
    render_rows(c, q, px, 0, c.geometry.mcu_rows, fast="islow")
    if rgb_sha(px.data) != case.sha:
        want = oracle.render_islow(c.y_blocks, c.cb_blocks, c.cr_blocks, q, p.width, p.height, sub)
        d = np.argwhere((px.data != want).any(-1))
        pytest.fail(f"{case}: {len(d)} pixels differ from the oracle, first {d[:4].tolist()}")


def test_islow_device_batch_mixed_and_row_ranges():
    from paper_1311_5304_b200 import device
    from paper_1311_5304_b200.block_transforms import alloc_pixels
    from paper_1311_5304_b200.kernels import cuda
    cases = [c for c in ISLOW_CASES if not c.name.startswith("i00")][::3]
    dec = [_decode(c.jpeg) for c in cases]
    db = device.DeviceBatch([d[1].geometry for d in dec], fast="islow")
    st = device.Stream()
    for i, (p, c, q, sub) in enumerate(dec):
        db.upload_coefficients(i, c, st)
        db.upload_qtables(i, q, st)
    db.render(stream=st)
    for i, (case, (p, c, q, sub)) in enumerate(zip(cases, dec)):
        out = np.zeros((p.height, p.width, 3), np.uint8)
        db.download_rgb(i, out, st)
        st.synchronize()
        assert rgb_sha(out) == case.sha, case
    db.close()
    # the drop-in over random MCU-row ranges composes to the whole image
    rng = np.random.default_rng(11)
    fns = {0: cuda.render_rows_444, 1: cuda.render_rows_422, 2: cuda.render_rows_420}
    for case, (p, c, q, sub) in list(zip(cases, dec))[:12]:
        g = c.geometry
        px = alloc_pixels(p.width, p.height)
        r = 0
        while r < g.mcu_rows:
            n = int(rng.integers(1, 4))
            fns[sub](c.y_blocks, c.cb_blocks, c.cr_blocks, q, px.data, p.width, p.height, g.mcus_per_row, r,
                     min(n, g.mcu_rows - r), "islow", True)
            r += n
        assert rgb_sha(px.data) == case.sha, case


@pytest.mark.parametrize("sub", [0, 1, 2])
@pytest.mark.parametrize("w,h", [(64, 48), (37, 29), (3, 5)])
def test_islow_adversarial_coefficients_match_oracle(sub, w, h):
    """Full int16 coefficient range with q up to 255: the mode's 32-bit
    wrapping arithmetic and the 10-bit range-limit window, as the oracle."""
    from paper_1311_5304_b200.kernels import cuda
    rng = np.random.default_rng(100 * sub + w)
    mw, mh, ypm = {0: (8, 8, 1), 1: (16, 8, 2), 2: (16, 16, 4)}[sub]
    mpr, rows = -(-w // mw), -(-h // mh)
    n = mpr * rows
    planes = []
    for nb in (n * ypm, n, n):
        a = rng.integers(-40, 40, size=(nb, 64)).astype(np.int16)
        big = rng.random((nb, 64)) < 0.1
        a[big] = rng.integers(-32768, 32767, size=int(big.sum()))
        a[rng.random(nb) < 0.2, 1:] = 0
        planes.append(a)
    q = rng.integers(1, 256, size=(3, 64)).astype(np.int32)
    q[:, 10:] = rng.integers(1, 8, size=(3, 54))
    rgb = np.zeros((h, w, 3), np.uint8)
    {0: cuda.render_rows_444, 1: cuda.render_rows_422, 2: cuda.render_rows_420}[sub](
        *planes, q, rgb, w, h, mpr, 0, rows, "islow", True)
    want = oracle.render_islow(*planes, q, w, h, sub)
    assert np.array_equal(rgb, want)


@pytest.mark.parametrize("mode", ["seq", "par", "accel", "accel-pipe", "sps", "pps"])
def test_islow_orchestrator_modes(mode):
    import os

    from paper_1311_5304_b200 import executors, orchestrator, parser, perf_model
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    prof = perf_model.load_profile(os.path.join(root, "profiles", "b200_profile.json"))
    lanes = executors.make_lanes(host_workers=2, transfer_latency_ns=0.0, transfer_bytes_per_ns=0.0)
    try:
        for case in [c for c in ISLOW_CASES if "_420_" in c.name or "_422_" in c.name][-6:]:
            p = parser.parse_stream(case.jpeg)
            px, rep = orchestrator.decode(p, mode, prof, lanes, data=case.jpeg, idct="islow")
            assert rgb_sha(px.data) == case.sha, (mode, case)
    finally:
        lanes.shutdown()


@pytest.mark.parametrize("w,h,q,sub", [(1920, 1080, 90, "420"), (4096, 4096, 95, "444"), (4096, 4096, 95, "422"),
                                       (6000, 4000, 90, "420")])
def test_islow_baseline_sizes_match_oracle_and_libjpeg(w, h, q, sub):
    import io

    from PIL import Image

    from paper_1311_5304_b200.block_transforms import alloc_pixels, render_rows
    from paper_1311_5304_b200.synth import synth_jpeg
    blob = synth_jpeg(w, h, q, sub, seed=5, restart_rows=1 if w == 6000 else 0)
    p, c, qt, s = _decode(blob)
    px = alloc_pixels(w, h)
    render_rows(c, qt, px, 0, c.geometry.mcu_rows, fast="islow")
    want = oracle.render_islow(c.y_blocks, c.cb_blocks, c.cr_blocks, qt, w, h, s)
    assert np.array_equal(px.data, want)
    assert np.array_equal(px.data, np.asarray(Image.open(io.BytesIO(blob)).convert("RGB")))
