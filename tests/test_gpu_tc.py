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
