"""CPU ORACLE: baseline-JPEG front end - TEST INFRASTRUCTURE ONLY.

Parses a synthetic baseline JPEG and Huffman-decodes it with the oracle's C
restatement of the reference decoder (huffman_oracle.c), producing the
reference CoefficientBuffer layout (entropy.py:31-56) that the parallel
phase consumes.  Used by tests/ (as an independent check of the product's
host decoders), by bench.py's --impl reference / cpu_baseline legs (so the
reference arm never loads the product library), and never by the product.

  parse        restates parser.parse_stream (parser.py:296-380) for SOF0
               frames, extended to 4:2:0 (the reference rejects it,
               parser.py:223-229)
  scan_tables  restates build_huffman_table + _pack_scan_tables
               (parser.py:133-177, entropy.py:59-84)
  qtables      restates perf_model._qtable_stack (perf_model.py:306-311)
  decode       restates entropy.decode_all (entropy.py:158-164)
  synth_jpeg   the SURVEY.md Appendix B generator (Pillow encoder)
"""
from __future__ import annotations

import ctypes as C
import io
import os
import struct
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

ZIGZAG = np.array([
    0, 1, 8, 16, 9, 2, 3, 10, 17, 24, 32, 25, 18, 11, 4, 5,
    12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6, 7, 14, 21, 28,
    35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
    58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63], dtype=np.int32)

# (h, v) sampling factors of Y -> (subsampling code, mcu_w, mcu_h, Y blocks per MCU)
LAYOUTS = {(1, 1): (0, 8, 8, 1), (2, 1): (1, 16, 8, 2), (2, 2): (2, 16, 16, 4)}


class OracleDecodeError(Exception):
    pass


class ScanTables(C.Structure):
    _fields_ = [("lut_sym", C.c_uint8 * 256 * 8), ("lut_len", C.c_uint8 * 256 * 8),
                ("mincode", C.c_int32 * 17 * 8), ("maxcode", C.c_int32 * 17 * 8),
                ("valptr", C.c_int32 * 17 * 8), ("symbols", C.c_uint8 * 256 * 8),
                ("comp_dc", C.c_int32 * 3), ("comp_ac", C.c_int32 * 3)]


_lib = None


def _clib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            subprocess.run(["make", "-s", "-C", HERE], check=True)
        _lib = C.CDLL(LIB_PATH)
        _lib.or_decode_mcu_rows.restype = C.c_int
        _lib.or_decode_mcu_rows.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.POINTER(ScanTables),
                                            C.c_void_p, C.c_void_p, C.c_void_p] + [C.c_int] * 5
    return _lib


@dataclass
class Parsed:
    width: int
    height: int
    subsampling: int
    mcu_w: int
    mcu_h: int
    ypm: int
    comps: list            # [(id, h, v, tq, td, ta)]
    qt: dict
    huff: list             # [(class, id, counts, symbols)]
    restart_interval: int
    scan: bytes

    @property
    def mcus_per_row(self):
        return -(-self.width // self.mcu_w)

    @property
    def mcu_rows(self):
        return -(-self.height // self.mcu_h)


def parse(data: bytes) -> Parsed:
    if len(data) < 2 or data[0] != 0xFF or data[1] != 0xD8:
        raise OracleDecodeError("no SOI")
    pos = 2
    frame = None
    qt, huff = {}, []
    dri = 0
    scan = None
    while True:
        if pos >= len(data) or data[pos] != 0xFF:
            raise OracleDecodeError("expected marker")
        while pos < len(data) and data[pos] == 0xFF:
            pos += 1
        m = data[pos]
        pos += 1
        if m == 0xD9:
            break
        if m == 0x01 or 0xD0 <= m <= 0xD7:
            continue
        ln = struct.unpack_from(">H", data, pos)[0]
        pay = data[pos + 2:pos + ln]
        pos += ln
        if m == 0xC0:
            _, h, w, nc = struct.unpack_from(">BHHB", pay)
            frame = (w, h, [(pay[6 + 3 * i], pay[7 + 3 * i] >> 4, pay[7 + 3 * i] & 15, pay[8 + 3 * i])
                            for i in range(nc)])
        elif 0xC1 <= m <= 0xCF and m not in (0xC4, 0xC8, 0xCC):
            raise OracleDecodeError("not a baseline frame")
        elif m == 0xC4:
            k = 0
            while k < len(pay):
                tc, th = pay[k] >> 4, pay[k] & 15
                counts = tuple(pay[k + 1:k + 17])
                syms = tuple(pay[k + 17:k + 17 + sum(counts)])
                huff.append((tc, th, counts, syms))
                k += 17 + sum(counts)
        elif m == 0xDB:
            k = 0
            while k < len(pay):
                qt[pay[k] & 15] = tuple(pay[k + 1:k + 65])
                k += 65
        elif m == 0xDD:
            dri = struct.unpack_from(">H", pay)[0]
        elif m == 0xDA:
            ns = pay[0]
            sel = {pay[1 + 2 * i]: (pay[2 + 2 * i] >> 4, pay[2 + 2 * i] & 15) for i in range(ns)}
            comps = [c + sel[c[0]] for c in frame[2]]
            end = pos
            while end < len(data) - 1:  # parser._scan_entropy_end (parser.py:277-293)
                if data[end] != 0xFF:
                    end += 1
                elif data[end + 1] == 0x00 or 0xD0 <= data[end + 1] <= 0xD7:
                    end += 2
                elif data[end + 1] == 0xFF:
                    end += 1
                else:
                    break
            scan = data[pos:end]
            frame = (frame[0], frame[1], comps)
            pos = end
    w, h, comps = frame
    key = (comps[0][1], comps[0][2])
    if key not in LAYOUTS or any((c[1], c[2]) != (1, 1) for c in comps[1:]):
        raise OracleDecodeError(f"unsupported sampling {[(c[1], c[2]) for c in comps]}")
    sub, mw, mh, ypm = LAYOUTS[key]
    return Parsed(w, h, sub, mw, mh, ypm, comps, qt, huff, dri, scan)


def scan_tables(p: Parsed) -> ScanTables:
    t = ScanTables()
    for s in range(8):
        for l in range(17):
            t.maxcode[s][l] = -1
    for tc, th, counts, syms in p.huff:
        s = tc * 4 + th
        code = k = 0
        for length in range(1, 17):
            cnt = counts[length - 1]
            if cnt:
                t.mincode[s][length] = code
                t.maxcode[s][length] = code + cnt - 1
                t.valptr[s][length] = k
                for _ in range(cnt):
                    if length <= 8:
                        lo = code << (8 - length)
                        for v in range(lo, lo + (1 << (8 - length))):
                            t.lut_sym[s][v] = syms[k]
                            t.lut_len[s][v] = length
                    code += 1
                    k += 1
            code <<= 1
        for i, v in enumerate(syms):
            t.symbols[s][i] = v
    for i, c in enumerate(p.comps):
        t.comp_dc[i] = c[4]
        t.comp_ac[i] = 4 + c[5]
    return t


def qtables(p: Parsed) -> np.ndarray:
    out = np.zeros((3, 64), np.int32)
    for i, c in enumerate(p.comps):
        out[i, ZIGZAG] = np.array(p.qt[c[3]], np.int32)
    return out


@dataclass
class Decoded:
    parsed: Parsed
    y: np.ndarray
    cb: np.ndarray
    cr: np.ndarray
    q: np.ndarray


def decode(data: bytes, row0: int = 0, n_rows: int | None = None) -> Decoded:
    p = parse(data)
    n_c = p.mcus_per_row * p.mcu_rows
    y = np.zeros((n_c * p.ypm, 64), np.int16)
    cb = np.zeros((n_c, 64), np.int16)
    cr = np.zeros((n_c, 64), np.int16)
    st = np.zeros(8, np.int64)
    t = scan_tables(p)
    buf = np.frombuffer(p.scan, np.uint8) if p.scan else np.zeros(1, np.uint8)
    rows = p.mcu_rows if n_rows is None else n_rows
    err = _clib().or_decode_mcu_rows(buf.ctypes.data, len(p.scan), st.ctypes.data, C.byref(t),
                                     y.ctypes.data, cb.ctypes.data, cr.ctypes.data, row0, rows,
                                     p.mcus_per_row, p.ypm, p.restart_interval)
    if err:
        raise OracleDecodeError(f"huffman error {err}")
    return Decoded(p, y, cb, cr, qtables(p))


def synth_rgb(width, height, seed=0, sigma=20.0):
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:height, 0:width].astype(np.float32)
    rgb = np.stack([128 + 100 * np.sin(xx / 37 + yy / 53),
                    128 + 90 * np.cos(xx / 23 - yy / 41),
                    128 + 80 * np.sin((xx + yy) / 61)], axis=-1)
    rgb += rng.normal(0.0, sigma, size=rgb.shape).astype(np.float32)
    return np.clip(rgb, 0, 255).astype(np.uint8)


def synth_jpeg(width, height, quality=90, subsampling="420", seed=0, restart_rows=0, restart_blocks=0,
               sigma=20.0) -> bytes:
    from PIL import Image
    kw = {}
    if restart_rows:
        kw["restart_marker_rows"] = restart_rows
    if restart_blocks:
        kw["restart_marker_blocks"] = restart_blocks
    b = io.BytesIO()
    Image.fromarray(synth_rgb(width, height, seed, sigma)).save(
        b, "JPEG", quality=quality, subsampling={"444": 0, "422": 1, "420": 2}[subsampling], **kw)
    return b.getvalue()
