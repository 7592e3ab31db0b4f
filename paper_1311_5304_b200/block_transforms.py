"""Pixel kernels - the public surface of the reference's
`hetjpeg.block_transforms` (pkg/src/hetjpeg/block_transforms.py:1-75 and the
single-block functions it re-exports from kernels/fallback.py:45-180).

Every transform runs on the GPU through the C ABI; single-block calls are
batched per call (pass a stack of blocks to amortise the launch).  Results
are bit-identical to the reference's float64 definitions.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib, kernels

__all__ = [
    "PixelBuffer", "alloc_pixels", "render_rows", "dequantize", "idct_direct",
    "idct_direct_f64", "idct_fast", "idct_fast_f64", "upsample_row_422", "ycbcr_to_rgb",
    "fused_idct_color_444", "fused_upsample_color_422",
]


@dataclass
class PixelBuffer:
    """Interleaved RGB8, row-major from the top-left pixel."""
    width: int
    height: int
    data: np.ndarray  # uint8 (height, width, 3)

    def tobytes(self) -> bytes:
        return self.data.tobytes()


def alloc_pixels(width: int, height: int, pinned: bool = False) -> PixelBuffer:
    if pinned:
        from .entropy import PinnedArray
        owner = PinnedArray((height, width, 3), np.uint8)
        owner.array[...] = 0
        buf = PixelBuffer(width, height, owner.array)
        buf._owner = owner  # keep the page-locked allocation alive
        return buf
    return PixelBuffer(width, height, np.zeros((height, width, 3), np.uint8))


def render_rows(coeffs, qtables, pixels: PixelBuffer, row0: int, n_rows: int,
                fast=True, fused: bool = True, backend=None) -> None:
    """Parallel phase over MCU rows [row0, row0 + n_rows) (block_transforms.py:60-75).

    Dispatches on the MCU shape: 8x8 -> 4:4:4, 16x8 -> 4:2:2, 16x16 -> 4:2:0.
    Safe to call concurrently for disjoint row ranges."""
    if n_rows <= 0:
        return
    impl = backend if backend is not None else kernels.active()
    geo = coeffs.geometry
    if geo.mcu_width == 8:
        fn = impl.render_rows_444
    elif geo.mcu_height == 8:
        fn = impl.render_rows_422
    else:
        fn = impl.render_rows_420
    fn(coeffs.y_blocks, coeffs.cb_blocks, coeffs.cr_blocks, qtables, pixels.data, geo.width,
       geo.height, geo.mcus_per_row, row0, n_rows, fast, fused)


# ----------------------------------------------------------------- per block

def dequantize(block, qtable) -> np.ndarray:
    """Elementwise coefficient * qtable, natural order (fallback.py:45-48)."""
    return (np.asarray(block, np.int32).reshape(64) * np.asarray(qtable, np.int32).reshape(64))


def _blocks(deq) -> tuple:
    a = np.ascontiguousarray(deq, dtype=np.int32)
    single = a.size == 64 and a.ndim <= 2 and (a.ndim < 2 or a.shape[0] in (1, 8))
    return a.reshape(-1, 64), single


def _idct(deq, fast: bool) -> np.ndarray:
    _lib.require_device()
    a, single = _blocks(deq)
    out = np.empty((len(a), 64), np.uint8)
    _lib.check(_lib.lib.hj_idct_blocks(a.ctypes.data, len(a), out.ctypes.data, int(fast)), "idct")
    return out[0] if single else out


def _idct_f64(deq, fast: bool) -> np.ndarray:
    _lib.require_device()
    a, single = _blocks(deq)
    out = np.empty((len(a), 64), np.float64)
    _lib.check(_lib.lib.hj_idct_blocks_f64(a.ctypes.data, len(a), out.ctypes.data, int(fast)),
               "idct_f64")
    return out[0].reshape(8, 8) if single else out.reshape(-1, 8, 8)


def idct_direct(block) -> np.ndarray:
    """Direct two-pass transform -> 64 samples (fallback.py:108-110)."""
    return _idct(block, fast=False)


def idct_fast(block) -> np.ndarray:
    """Scaled AAN transform -> 64 samples (fallback.py:117-119)."""
    return _idct(block, fast=True)


def idct_direct_f64(block) -> np.ndarray:
    """Pre-rounding float64 core, no level shift (fallback.py:103-105)."""
    return _idct_f64(block, fast=False)


def idct_fast_f64(block) -> np.ndarray:
    return _idct_f64(block, fast=True)


def upsample_row_422(row, left=None, right=None):
    """Algorithm 1 on an 8-sample row (fallback.py:122-139), on the GPU.
    Accepts one row (8,) or a stack (n, 8) with per-row neighbour arrays."""
    _lib.require_device()
    rows = np.asarray(row)
    single = rows.ndim == 1
    if rows.shape not in ((8,),) and not (rows.ndim == 2 and rows.shape[1] == 8):
        raise ValueError("expected an 8-sample chroma row")
    rows = rows.reshape(-1, 8)
    n = len(rows)

    def nb(v):
        if v is None:
            return np.full(n, -1, np.int16)
        return np.broadcast_to(np.asarray(v, np.int16), (n,)).copy()

    r8 = np.ascontiguousarray(rows, dtype=np.uint8)
    out = np.empty((n, 16), np.int32)
    lf, rt = nb(left), nb(right)
    _lib.check(_lib.lib.hj_upsample_422(r8.ctypes.data, lf.ctypes.data, rt.ctypes.data,
                                        out.ctypes.data, n), "upsample_422")
    return out[0] if single else out


def ycbcr_to_rgb(y, cb, cr):
    """Colour conversion (fallback.py:142-150): scalars or arrays of samples
    -> (r, g, b) uint8 arrays of the broadcast shape.  The exact integer
    conversion (proven over all 2^24 inputs) covers what a decoder produces:
    integer-valued samples in [0, 255], of any numeric dtype.  Other values
    (fractional or out of range), which the reference would convert in
    float64, are rejected rather than truncated."""
    _lib.require_device()
    yb, cbb, crb = np.broadcast_arrays(np.asarray(y), np.asarray(cb), np.asarray(cr))
    shape = yb.shape
    for a in (yb, cbb, crb):
        if a.dtype.kind not in "biuf":
            raise TypeError(f"samples must be numeric, got {a.dtype}")
        if a.size and (a.min() < 0 or a.max() > 255):
            raise ValueError("samples must lie in [0, 255]")
        if a.dtype.kind == "f" and a.size and not np.array_equal(a, np.floor(a)):
            raise ValueError("samples must be integer-valued (the exact conversion is defined on 8-bit samples)")
    flat = [np.ascontiguousarray(a, dtype=np.uint8).reshape(-1) for a in (yb, cbb, crb)]
    n = flat[0].size
    rgb = np.empty((n, 3), np.uint8)
    if n:
        _lib.check(_lib.lib.hj_ycbcr_to_rgb(flat[0].ctypes.data, flat[1].ctypes.data,
                                            flat[2].ctypes.data, rgb.ctypes.data, n), "ycbcr")
    return tuple(rgb[:, k].reshape(shape) for k in range(3))


def fused_idct_color_444(y_block, cb_block, cr_block, qy, qcb, qcr, fast=True):
    """One 4:4:4 MCU -> (64, 3) RGB (fallback.py:153-165), through the render
    kernel itself (a 8x8 image)."""
    coeffs = np.stack([np.asarray(b, np.int16).reshape(64) for b in (y_block, cb_block, cr_block)])
    q = np.stack([np.asarray(t, np.int32).reshape(64) for t in (qy, qcb, qcr)])
    rgb = np.zeros((8, 8, 3), np.uint8)
    kernels.active().render_rows_444(coeffs[0:1].copy(), coeffs[1:2].copy(), coeffs[2:3].copy(), q,
                                     rgb, 8, 8, 1, 0, 1, fast, True)
    return rgb.reshape(64, 3)


def fused_upsample_color_422(y_row, cb_row, cr_row, cb_left=None, cb_right=None,
                             cr_left=None, cr_right=None):
    """16-pixel row: Algorithm 1 on Cb and Cr + colour (fallback.py:168-180)."""
    cb16 = upsample_row_422(cb_row, cb_left, cb_right)
    cr16 = upsample_row_422(cr_row, cr_left, cr_right)
    r, g, b = ycbcr_to_rgb(np.asarray(y_row), cb16, cr16)
    return np.stack([r, g, b], axis=-1)
