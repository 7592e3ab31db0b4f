"""Known-answer vectors for the reference's single-MCU forms, from the REFERENCE.

Run in the build container only (reference build in oracle/_ref):

    python tests/golden/make_single_ops.py

Writes tests/golden/single_ops.npz with, from the reference's
kernels/fallback.py (the numpy backend, bit-identical to _native):
  up_rows/up_left/up_right/up_out     upsample_row_422 (fallback.py:122-139);
                                      neighbour -1 = None (end pixel copied)
  f422_y/f422_cb/f422_cr/f422_nb/f422_out  fused_upsample_color_422
                                      (fallback.py:168-180); nb = (cb_left,
                                      cb_right, cr_left, cr_right), -1 = None
  f444_blocks/f444_q/f444_fast/f444_direct  fused_idct_color_444
                                      (fallback.py:153-165), fast and direct
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref", "patched"))

from hetjpeg.kernels import fallback  # noqa: E402


def nb(v):
    return None if v < 0 else int(v)


def main():
    rng = np.random.default_rng(1311)
    n = 400
    up_rows = rng.integers(0, 256, size=(n, 8)).astype(np.uint8)
    up_rows[:40] = rng.integers(0, 2, size=(40, 8)) * 255  # extremes
    up_left = np.where(rng.random(n) < 0.5, -1, rng.integers(0, 256, n)).astype(np.int16)
    up_right = np.where(rng.random(n) < 0.5, -1, rng.integers(0, 256, n)).astype(np.int16)
    up_out = np.stack([fallback.upsample_row_422(r, nb(a), nb(b)) for r, a, b in zip(up_rows, up_left, up_right)])

    f422_y = rng.integers(0, 256, size=(n, 16)).astype(np.uint8)
    f422_cb = rng.integers(0, 256, size=(n, 8)).astype(np.uint8)
    f422_cr = rng.integers(0, 256, size=(n, 8)).astype(np.uint8)
    f422_cb[:8] = 78  # the float64 G tie pair with Y inside / outside [47, 82]
    f422_cr[:8] = 178
    f422_y[:4] = 60
    f422_nb = np.where(rng.random((n, 4)) < 0.5, -1, rng.integers(0, 256, (n, 4))).astype(np.int16)
    f422_out = np.stack([fallback.fused_upsample_color_422(y, cb, cr, *[nb(v) for v in k])
                         for y, cb, cr, k in zip(f422_y, f422_cb, f422_cr, f422_nb)]).astype(np.uint8)

    m = 200
    f444_blocks = np.zeros((m, 3, 64), np.int16)
    dense = rng.random((m, 3, 64)) < 0.35
    f444_blocks[dense] = rng.integers(-300, 300, size=int(dense.sum()))
    f444_blocks[:, :, 0] = rng.integers(-1024, 1016, size=(m, 3)) // 8
    f444_q = rng.integers(1, 100, size=(m, 3, 64)).astype(np.int32)
    f444_fast = np.stack([fallback.fused_idct_color_444(*b, *q, fast=True) for b, q in zip(f444_blocks, f444_q)])
    f444_direct = np.stack([fallback.fused_idct_color_444(*b, *q, fast=False) for b, q in zip(f444_blocks, f444_q)])
    np.savez_compressed(os.path.join(HERE, "single_ops.npz"), up_rows=up_rows, up_left=up_left, up_right=up_right,
                        up_out=up_out.astype(np.int32), f422_y=f422_y, f422_cb=f422_cb, f422_cr=f422_cr,
                        f422_nb=f422_nb, f422_out=f422_out, f444_blocks=f444_blocks, f444_q=f444_q,
                        f444_fast=f444_fast.astype(np.uint8), f444_direct=f444_direct.astype(np.uint8))
    print("single_ops.npz:", n, "upsample rows,", n, "fused 4:2:2 rows,", m, "fused 4:4:4 MCUs")


if __name__ == "__main__":
    main()
