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
