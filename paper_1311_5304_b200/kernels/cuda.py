"""The `cuda` kernel backend: the module contract of the reference's
`_native` / `fallback` backends (kernels/_native.pyx:187-549,
kernels/fallback.py:224-417) implemented on the B200.

  NAME              "cuda"
  prepare_scan      packs the slot tables into the C struct hj_scan_tables_t
  decode_mcu_rows   host C++ Huffman decoder (hj_decode_mcu_rows)
  render_rows_444   GPU parallel phase, synchronous drop-in (hj_render_rows)
  render_rows_422   "
  render_rows_420   the 4:2:0 extension (no reference counterpart)

render_rows_* keep the reference contract: caller-owned host numpy arrays,
RGB rows [8*row0, min(h, 8*(row0+n_rows))) written in place, no references
kept, safe to call from several threads on disjoint row ranges (each thread
gets its own CUDA stream and staging inside the library).  `fused` never
changes bytes.  For device-resident batches use `paper_1311_5304_b200.device`.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from .. import _lib

NAME = "cuda"

_SUB_MCU_H = {_lib.SUB_444: 8, _lib.SUB_422: 8, _lib.SUB_420: 16}


def prepare_scan(lut_sym, lut_len, mincode, maxcode, valptr, symbols, comp_dc, comp_ac):
    t = _lib.hj_scan_tables_t()
    for name, arr, dt in (("lut_sym", lut_sym, np.uint8), ("lut_len", lut_len, np.uint8),
                          ("mincode", mincode, np.int32), ("maxcode", maxcode, np.int32),
                          ("valptr", valptr, np.int32), ("symbols", symbols, np.uint8),
                          ("comp_dc", comp_dc, np.int32), ("comp_ac", comp_ac, np.int32)):
        src = np.ascontiguousarray(arr, dtype=dt)
        dst = np.ctypeslib.as_array(getattr(t, name))
        if src.shape != dst.shape:
            raise ValueError(f"{name}: expected shape {dst.shape}, got {src.shape}")
        dst[...] = src
    return t


def _i16_blocks(a, what):
    if not isinstance(a, np.ndarray) or a.dtype != np.int16 or a.ndim != 2 or a.shape[1] != 64 \
            or not a.flags.c_contiguous:
        raise ValueError(f"{what}: expected a C-contiguous int16 (n, 64) array")
    return a


def decode_mcu_rows(data, state, scan, y_out, cb_out, cr_out, row0, n_rows, mcus_per_row,
                    y_per_mcu, restart_interval):
    """Huffman-decode MCU rows [row0, row0+n_rows); `state` (int64[8]) is
    updated in place even when an error is raised (native semantics)."""
    if not isinstance(state, np.ndarray) or state.dtype != np.int64 or state.shape != (8,):
        raise ValueError("state must be an int64[8] array")
    for a, w in ((y_out, "y_out"), (cb_out, "cb_out"), (cr_out, "cr_out")):
        _i16_blocks(a, w)
        if not a.flags.writeable:
            raise ValueError(f"{w} is read-only")
    end_mcu = (row0 + n_rows) * mcus_per_row
    if n_rows > 0 and (len(cb_out) < end_mcu or len(cr_out) < end_mcu
                       or len(y_out) < end_mcu * y_per_mcu):
        raise ValueError("coefficient planes too small for the requested rows")
    buf = np.frombuffer(data, dtype=np.uint8) if len(data) else np.zeros(1, np.uint8)
    st = _lib.lib.hj_decode_mcu_rows(buf.ctypes.data, len(data), state.ctypes.data, C.byref(scan),
                                     y_out.ctypes.data, cb_out.ctypes.data, cr_out.ctypes.data,
                                     int(row0), int(n_rows), int(mcus_per_row), int(y_per_mcu),
                                     int(restart_interval))
    _lib.check(st, "decode_mcu_rows")


def _render(sub, y_blocks, cb_blocks, cr_blocks, qtables, rgb, width, height, mcus_per_row,
            row0, n_rows, fast, fused):
    if n_rows <= 0:
        return
    _lib.require_device()
    _i16_blocks(y_blocks, "y_blocks")
    _i16_blocks(cb_blocks, "cb_blocks")
    _i16_blocks(cr_blocks, "cr_blocks")
    q = np.ascontiguousarray(qtables, dtype=np.int32)
    if q.shape != (3, 64):
        raise ValueError("qtables must be (3, 64)")
    if not isinstance(rgb, np.ndarray) or rgb.dtype != np.uint8 or rgb.shape != (height, width, 3) \
            or not rgb.flags.c_contiguous:
        raise ValueError("rgb must be a C-contiguous uint8 (height, width, 3) array")
    mcu_rows = -(-int(height) // _SUB_MCU_H[sub])
    ptr = _lib.ptr
    st = _lib.lib.hj_render_rows(ptr(y_blocks), ptr(cb_blocks), ptr(cr_blocks),
                                 ptr(q), ptr(rgb), int(width), int(height),
                                 int(mcus_per_row), mcu_rows, int(row0), int(n_rows), sub,
                                 _lib.idct_code(fast), int(bool(fused)), len(y_blocks), len(cb_blocks))
    _lib.check(st, "render_rows")


def render_rows_444(y_blocks, cb_blocks, cr_blocks, qtables, rgb, width, height, mcus_per_row,
                    row0, n_rows, fast=True, fused=True):
    _render(_lib.SUB_444, y_blocks, cb_blocks, cr_blocks, qtables, rgb, width, height,
            mcus_per_row, row0, n_rows, fast, fused)


def render_rows_422(y_blocks, cb_blocks, cr_blocks, qtables, rgb, width, height, mcus_per_row,
                    row0, n_rows, fast=True, fused=True):
    _render(_lib.SUB_422, y_blocks, cb_blocks, cr_blocks, qtables, rgb, width, height,
            mcus_per_row, row0, n_rows, fast, fused)


def render_rows_420(y_blocks, cb_blocks, cr_blocks, qtables, rgb, width, height, mcus_per_row,
                    row0, n_rows, fast=True, fused=True):
    """4:2:0 extension; reads chroma of MCU rows row0-1 and row0+n_rows
    (vertical filter context) when they exist - decode them first."""
    _render(_lib.SUB_420, y_blocks, cb_blocks, cr_blocks, qtables, rgb, width, height,
            mcus_per_row, row0, n_rows, fast, fused)
