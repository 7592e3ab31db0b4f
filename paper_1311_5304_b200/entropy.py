"""Host entropy stage: resumable MCU-row Huffman decoding into the planar
coefficient buffer the GPU consumes.

API of the reference's `hetjpeg.entropy` (pkg/src/hetjpeg/entropy.py):
`dezigzag`, `CoefficientBuffer`, `alloc_coefficients`, `EntropyCursor`,
`new_cursor`, `decode_rows`, `decode_all`, with the same int64[8] cursor
state layout.  Decoding runs in the native C++ decoder
(`hj_decode_mcu_rows`, csrc/hj_huffman.cpp) with the GIL released (ctypes),
so several host threads decode different images truly in parallel - the
reference's Cython decoder re-takes the GIL per helper call.

Coefficient buffers can be allocated in page-locked memory
(`alloc_coefficients(geo, pinned=True)`) so the GPU lane copies them with
async DMA.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .parser import ImageGeometry, ParsedJpeg, build_huffman_table, geometry_of

ZIGZAG = np.array([
    0, 1, 8, 16, 9, 2, 3, 10, 17, 24, 32, 25, 18, 11, 4, 5,
    12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6, 7, 14, 21, 28,
    35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
    58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63], dtype=np.int32)


def dezigzag(block_zz) -> np.ndarray:
    """Zigzag scan order -> natural row-major order (entropy.py:21-28)."""
    block_zz = np.asarray(block_zz)
    if block_zz.shape != (64,):
        raise ValueError("expected 64 coefficients")
    out = np.empty_like(block_zz)
    out[ZIGZAG] = block_zz
    return out


class PinnedArray:
    """A numpy view over page-locked host memory owned by the native library."""

    def __init__(self, shape, dtype):
        nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = _lib.C.c_void_p()
        _lib.check(_lib.lib.hj_malloc_host(_lib.C.byref(p), max(nbytes, 1)), "hj_malloc_host")
        self._ptr = p.value
        buf = (_lib.C.c_uint8 * max(nbytes, 1)).from_address(self._ptr)
        self.array = np.frombuffer(buf, dtype=np.uint8, count=nbytes).view(dtype).reshape(shape)

    def __del__(self):
        if getattr(self, "_ptr", None):
            _lib.lib.hj_free_host(self._ptr)
            self._ptr = None


@dataclass
class CoefficientBuffer:
    """Planar int16 blocks: all Y (MCU order), all Cb, all Cr; natural order."""
    geometry: ImageGeometry
    y_blocks: np.ndarray
    cb_blocks: np.ndarray
    cr_blocks: np.ndarray
    _owners: tuple = field(default=(), repr=False, compare=False)

    @property
    def y_blocks_per_mcu(self) -> int:
        return self.geometry.y_blocks_per_mcu


def alloc_coefficients(geometry: ImageGeometry, pinned: bool = False) -> CoefficientBuffer:
    n_c = geometry.total_mcus
    n_y = n_c * geometry.y_blocks_per_mcu
    if not pinned:
        return CoefficientBuffer(geometry, np.zeros((n_y, 64), np.int16),
                                 np.zeros((n_c, 64), np.int16), np.zeros((n_c, 64), np.int16))
    owner = PinnedArray((n_y + 2 * n_c, 64), np.int16)
    a = owner.array
    a[...] = 0
    return CoefficientBuffer(geometry, a[:n_y], a[n_y:n_y + n_c], a[n_y + n_c:], (owner,))


def _pack_scan_tables(parsed: ParsedJpeg):
    """Slot-indexed table arrays (slots 0-3 DC, 4-7 AC), entropy.py:59-84."""
    lut_sym = np.zeros((8, 256), np.uint8)
    lut_len = np.zeros((8, 256), np.uint8)
    mincode = np.zeros((8, 17), np.int32)
    maxcode = np.full((8, 17), -1, np.int32)
    valptr = np.zeros((8, 17), np.int32)
    symbols = np.zeros((8, 256), np.uint8)
    for spec in parsed.huffman_specs:
        k = spec.table_class.value * 4 + spec.table_id
        t = build_huffman_table(spec)
        lut_sym[k], lut_len[k] = t.lut_symbol, t.lut_length
        mincode[k], maxcode[k], valptr[k] = t.mincode, t.maxcode, t.valptr
        symbols[k, :len(t.symbols)] = t.symbols
    comp_dc = np.array([c.dc_table_id for c in parsed.components], np.int32)
    comp_ac = np.array([4 + c.ac_table_id for c in parsed.components], np.int32)
    return lut_sym, lut_len, mincode, maxcode, valptr, symbols, comp_dc, comp_ac


# int64[8] state layout (entropy.py:87-88)
_POS, _BITBUF, _BITS, _MCUS_SINCE_RST, _NEXT_RST, _PRED_Y, _PRED_CB, _PRED_CR = range(8)


@dataclass
class EntropyCursor:
    data: bytes
    geometry: ImageGeometry
    restart_interval: int
    scan: object
    backend: object
    state: np.ndarray = field(default_factory=lambda: np.zeros(8, np.int64))
    rows_decoded: int = 0
    row_times_ns: list = field(default_factory=list)

    @property
    def bit_position(self) -> int:
        return int(self.state[_POS]) * 8 - int(self.state[_BITS])

    @property
    def dc_predictors(self) -> tuple:
        return int(self.state[_PRED_Y]), int(self.state[_PRED_CB]), int(self.state[_PRED_CR])


def new_cursor(parsed: ParsedJpeg, data: bytes | None = None) -> EntropyCursor:
    from . import kernels
    data = parsed.stream if data is None else data
    sp = parsed.entropy_span
    backend = kernels.active()
    return EntropyCursor(bytes(data[sp.offset:sp.offset + sp.length]), geometry_of(parsed),
                         parsed.restart_interval, backend.prepare_scan(*_pack_scan_tables(parsed)),
                         backend)


def decode_rows(cursor: EntropyCursor, parsed: ParsedJpeg, out: CoefficientBuffer,
                n_rows: int, record_rows: bool = True) -> EntropyCursor:
    """Decode the next n_rows MCU rows (strictly in order), timing each row
    for the re-partitioner (entropy.py:133-155).  `record_rows=False` decodes
    the whole range in one native call (no per-row timestamps)."""
    geo = out.geometry
    left = geo.mcu_rows - cursor.rows_decoded
    if n_rows > left:
        raise ValueError(f"{n_rows} rows requested with only {left} remaining")
    args = (cursor.data, cursor.state, cursor.scan, out.y_blocks, out.cb_blocks, out.cr_blocks)
    if not record_rows:
        t0 = time.perf_counter_ns()
        cursor.backend.decode_mcu_rows(*args, cursor.rows_decoded, n_rows, geo.mcus_per_row,
                                       out.y_blocks_per_mcu, cursor.restart_interval)
        if n_rows:
            cursor.row_times_ns.extend([(time.perf_counter_ns() - t0) // n_rows] * n_rows)
        cursor.rows_decoded += n_rows
        return cursor
    for _ in range(n_rows):
        t0 = time.perf_counter_ns()
        cursor.backend.decode_mcu_rows(*args, cursor.rows_decoded, 1, geo.mcus_per_row,
                                       out.y_blocks_per_mcu, cursor.restart_interval)
        cursor.row_times_ns.append(time.perf_counter_ns() - t0)
        cursor.rows_decoded += 1
    return cursor


class FastScan:
    """Whole-scan throughput decoder (hj_decode_scan_fast) for one parsed
    header; bit-identical coefficients to `decode_all`."""

    def __init__(self, parsed: ParsedJpeg):
        self.parsed = parsed
        self.geometry = geometry_of(parsed)
        tables = _lib.hj_scan_tables_t()
        from .kernels import cuda as _backend
        tables = _backend.prepare_scan(*_pack_scan_tables(parsed))
        h = _lib.C.c_void_p()
        _lib.check(_lib.lib.hj_huff_build(_lib.C.byref(tables), _lib.C.byref(h)), "hj_huff_build")
        self._h = h.value

    def decode(self, data: bytes | None = None, out: CoefficientBuffer | None = None,
               threads: int = 1, pinned: bool = False) -> CoefficientBuffer:
        p = self.parsed
        data = p.stream if data is None else data
        sp = p.entropy_span
        buf = np.frombuffer(data, dtype=np.uint8)[sp.offset:sp.offset + sp.length]
        if out is None:
            out = alloc_coefficients(self.geometry, pinned=pinned)
        g = self.geometry
        st = _lib.lib.hj_decode_scan_fast(self._h, buf.ctypes.data, len(buf), out.y_blocks.ctypes.data,
                                          out.cb_blocks.ctypes.data, out.cr_blocks.ctypes.data,
                                          g.mcus_per_row, g.mcu_rows, g.y_blocks_per_mcu,
                                          p.restart_interval, int(threads))
        _lib.check(st, "decode_scan_fast")
        return out

    def decode_rows(self, row0: int, n_rows: int, data: bytes | None = None, out: CoefficientBuffer | None = None,
                    threads: int = 1) -> CoefficientBuffer:
        """Only the restart intervals covering MCU rows [row0, row0+n_rows)
        (hj_decode_scan_rows; the whole scan when it has no restart markers)."""
        p = self.parsed
        data = p.stream if data is None else data
        sp = p.entropy_span
        buf = np.frombuffer(data, dtype=np.uint8)[sp.offset:sp.offset + sp.length]
        if out is None:
            out = alloc_coefficients(self.geometry)
        g = self.geometry
        st = _lib.lib.hj_decode_scan_rows(self._h, buf.ctypes.data, len(buf), out.y_blocks.ctypes.data,
                                          out.cb_blocks.ctypes.data, out.cr_blocks.ctypes.data, g.mcus_per_row,
                                          g.mcu_rows, g.y_blocks_per_mcu, p.restart_interval, int(row0),
                                          int(n_rows), int(threads))
        _lib.check(st, "decode_scan_rows")
        return out

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.lib.hj_huff_free(self._h)
            self._h = None


def decode_all(parsed: ParsedJpeg, data: bytes | None = None, pinned: bool = False):
    cursor = new_cursor(parsed, data)
    buf = alloc_coefficients(cursor.geometry, pinned=pinned)
    decode_rows(cursor, parsed, buf, cursor.geometry.mcu_rows, record_rows=False)
    return buf, cursor
