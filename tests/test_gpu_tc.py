"""The tensor-core IDCT screen (render_tc_kernel) under the
whole GPU parity suite with HJ_RENDER_TC=1 (AAN images on it too; by default
only idct="direct" runs on it, covered by the default suite's direct cases):
every golden case (AAN and direct), partial row ranges, concurrent threads,
BASELINE sizes vs the oracle, adversarial int16 coefficients (out-of-range AC,
huge DC, Cb and Cr tables that differ: the exact path), mixed-subsampling
device batches, MCU-row shards and strip sweeps - bit-exact RGB, in a
subprocess because the switch is read once per process."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_parity_suite_on_tensor_core_kernel():
    env = dict(os.environ, HJ_RENDER_TC="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_tensor_core_kernel_runs_and_screens():
    """The switch really selects the tcgen05 kernel, and its screen proves
    almost every block of a BASELINE-config image (exact-path share < 3 %)."""
    code = r"""
import numpy as np
from paper_1311_5304_b200 import _lib, entropy, parser
from paper_1311_5304_b200.block_transforms import alloc_pixels, render_rows
from paper_1311_5304_b200.perf_model import qtable_stack
from paper_1311_5304_b200.synth import synth_jpeg
from oracle import oracle
_lib.require_device()
blob = synth_jpeg(1920, 1080, 90, "420", seed=3)
p = parser.parse_stream(blob)
co, _ = entropy.decode_all(p, blob)
g = co.geometry
q = qtable_stack(p)
px = alloc_pixels(g.width, g.height)
t0, e0 = _lib.lib.hj_tc_launch_count(), _lib.lib.hj_exact_block_count()
render_rows(co, q, px, 0, g.mcu_rows)
t1, e1 = _lib.lib.hj_tc_launch_count(), _lib.lib.hj_exact_block_count()
want = oracle.render(co.y_blocks, co.cb_blocks, co.cr_blocks, q, g.width, g.height, 2)
n_blocks = co.y_blocks.shape[0] + co.cb_blocks.shape[0] + co.cr_blocks.shape[0]
assert np.array_equal(px.data, want), "tensor-core kernel differs from the oracle"
assert t1 > t0, "HJ_RENDER_TC=1 did not launch the tensor-core kernel"
assert (e1 - e0) < 0.03 * n_blocks, (e1 - e0, n_blocks)
print("ok", t1 - t0, (e1 - e0) / n_blocks)
"""
    env = dict(os.environ, HJ_RENDER_TC="1")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_tensor_core_extreme_tables_and_coefficients():
    """F selection and the no-wrap guard at the table extremes: all-1 tables
    (F capped at 21, every block near the wrap limit), all-255 tables (small
    F, many exact-path blocks), 16-bit entries (beyond the reference's 8-bit
    DQT; the C ABI accepts them) - AAN and direct, every subsampling, against
    the oracle on the tensor-core kernel."""
    code = r"""
import numpy as np
from paper_1311_5304_b200 import _lib
from paper_1311_5304_b200.kernels import cuda
from oracle import oracle
_lib.require_device()
t0 = _lib.lib.hj_tc_launch_count()
rng = np.random.default_rng(7)
fns = {0: cuda.render_rows_444, 1: cuda.render_rows_422, 2: cuda.render_rows_420}
for sub in (0, 1, 2):
    w, h = 97, 53
    mw, mh, ypm = {0: (8, 8, 1), 1: (16, 8, 2), 2: (16, 16, 4)}[sub]
    mpr, rows = -(-w // mw), -(-h // mh)
    n_c = mpr * rows
    for qv in (1, 255, 4000):
        q = np.full((3, 64), qv, np.int32)
        y = (rng.integers(-60, 60, (n_c * ypm, 64)) * (rng.random((n_c * ypm, 64)) < 0.3)).astype(np.int16)
        y[:, 0] = rng.integers(-1024 // qv - 1, 1024 // qv + 2, n_c * ypm)
        cb = (rng.integers(-20, 20, (n_c, 64)) * (rng.random((n_c, 64)) < 0.2)).astype(np.int16)
        cr = cb[::-1].copy()
        for fast in (True, False):
            rgb = np.zeros((h, w, 3), np.uint8)
            fns[sub](y, cb, cr, q, rgb, w, h, mpr, 0, rows, fast, True)
            want = oracle.render(y, cb, cr, q, w, h, sub, fast)
            assert np.array_equal(rgb, want), (sub, qv, fast)
assert _lib.lib.hj_tc_launch_count() > t0
print("ok")
"""
    env = dict(os.environ, HJ_RENDER_TC="1")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
