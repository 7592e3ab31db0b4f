"""ctypes binding of libhetjpeg_b200.so (C ABI: include/hetjpeg_b200.h).

The product path has no CPU fallback: importing this module fails loudly
(ImportError) when the library is missing, and every compute call raises when
no CUDA device is visible.  Build with `python -m paper_1311_5304_b200._build`
(or `__graft_entry__.build()`).
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import BadCode, BitstreamExhausted, HetJpegError, MarkerInScan

_LIB_PATH = os.environ.get("HETJPEG_B200_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libhetjpeg_b200.so")

HJ_OK = 0
HJ_ERR_EXHAUSTED = 1
HJ_ERR_BADCODE = 2
HJ_ERR_MARKER = 3
HJ_ERR_RST_SEQ = 4
HJ_ERR_ARG = 16
HJ_ERR_CUDA = 17
HJ_ERR_NOMEM = 18
HJ_ERR_NODEVICE = 19

SUB_444, SUB_422, SUB_420 = 0, 1, 2
FLAG_DIRECT_IDCT = 1
FLAG_ISLOW_IDCT = 2
IDCT_DIRECT, IDCT_FAST, IDCT_ISLOW = 0, 1, 2


def idct_code(fast) -> int:
    """The IDCT path of a `fast` argument: True = the reference's AAN, False =
    its direct basis (both float64, kernels/_native.pyx:364-388), "islow" =
    libjpeg's integer decode (north_star's jidctint mode; HJ_IDCT_ISLOW)."""
    if isinstance(fast, str):
        if fast == "islow":
            return IDCT_ISLOW
        if fast in ("fast", "direct"):
            return IDCT_FAST if fast == "fast" else IDCT_DIRECT
        raise ValueError(f"unknown idct path {fast!r}")
    return IDCT_FAST if fast else IDCT_DIRECT


def image_flags(fast) -> int:
    return {IDCT_FAST: 0, IDCT_DIRECT: FLAG_DIRECT_IDCT, IDCT_ISLOW: FLAG_ISLOW_IDCT}[idct_code(fast)]


class CudaError(HetJpegError, RuntimeError):
    """A CUDA runtime failure inside the native library."""


class NoDevice(HetJpegError, RuntimeError):
    """No CUDA device is visible: the parallel phase has no CPU fallback."""


class hj_image_t(C.Structure):  # noqa: N801 - C name
    _fields_ = [
        ("y", C.c_void_p), ("cb", C.c_void_p), ("cr", C.c_void_p), ("q", C.c_void_p),
        ("rgb", C.c_void_p),
        ("width", C.c_int32), ("height", C.c_int32),
        ("mcus_per_row", C.c_int32), ("mcu_rows", C.c_int32),
        ("row0", C.c_int32), ("n_rows", C.c_int32),
        ("subsampling", C.c_int32), ("flags", C.c_int32),
    ]


class hj_scan_tables_t(C.Structure):  # noqa: N801
    _fields_ = [
        ("lut_sym", C.c_uint8 * 256 * 8), ("lut_len", C.c_uint8 * 256 * 8),
        ("mincode", C.c_int32 * 17 * 8), ("maxcode", C.c_int32 * 17 * 8),
        ("valptr", C.c_int32 * 17 * 8), ("symbols", C.c_uint8 * 256 * 8),
        ("comp_dc", C.c_int32 * 3), ("comp_ac", C.c_int32 * 3),
    ]


class hj_pipe_image_t(C.Structure):  # noqa: N801
    _fields_ = [
        ("huff", C.c_void_p), ("scan", C.c_void_p), ("scan_bytes", C.c_int64),
        ("y", C.c_void_p), ("cb", C.c_void_p), ("cr", C.c_void_p),
        ("dev_y", C.c_void_p), ("dev_cb", C.c_void_p), ("dev_cr", C.c_void_p),
        ("n_y", C.c_int64), ("n_c", C.c_int64),
        ("mcus_per_row", C.c_int32), ("mcu_rows", C.c_int32), ("y_per_mcu", C.c_int32),
        ("restart_interval", C.c_int32),
        ("plan", C.c_void_p), ("dev_rgb", C.c_void_p), ("rgb", C.c_void_p), ("rgb_bytes", C.c_int64),
    ]


class hj_stream_image_t(C.Structure):  # noqa: N801
    _fields_ = [
        ("huff", C.c_void_p), ("scan", C.c_void_p), ("scan_bytes", C.c_int64), ("q", C.c_void_p),
        ("width", C.c_int32), ("height", C.c_int32), ("subsampling", C.c_int32), ("flags", C.c_int32),
        ("restart_interval", C.c_int32), ("rgb_out", C.c_void_p), ("row0", C.c_int32), ("n_rows", C.c_int32),
    ]


class hj_stream_stats_t(C.Structure):  # noqa: N801
    _fields_ = [
        ("images", C.c_int64), ("launches", C.c_int64), ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64),
        ("pinned_bytes", C.c_int64), ("device_bytes", C.c_int64), ("huffman_thread_s", C.c_double),
        ("wall_s", C.c_double),
    ]


class hj_balance_term_t(C.Structure):  # noqa: N801
    _fields_ = [("coef", C.c_void_p), ("n", C.c_int32), ("reflected", C.c_int32), ("sign", C.c_double)]


class hj_partition_t(C.Structure):  # noqa: N801
    _fields_ = [("x_root", C.c_double), ("accel_mcu_rows", C.c_int32), ("cpu_mcu_rows", C.c_int32),
                ("accel_rows", C.c_int32), ("cpu_rows", C.c_int32)]


if not os.path.exists(_LIB_PATH):
    raise ImportError(
        f"native library missing: {_LIB_PATH} (build it with "
        "`python -m paper_1311_5304_b200._build`); there is no CPU fallback")

lib = C.CDLL(_LIB_PATH)

_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_SIG = {
    "hj_version": (C.c_char_p, []),
    "hj_last_error": (C.c_char_p, []),
    "hj_device_count": (C.c_int, []),
    "hj_set_device": (C.c_int, [C.c_int]),
    "hj_malloc_device": (C.c_int, [C.POINTER(_P), C.c_size_t]),
    "hj_free_device": (C.c_int, [_P]),
    "hj_malloc_host": (C.c_int, [C.POINTER(_P), C.c_size_t]),
    "hj_free_host": (C.c_int, [_P]),
    "hj_memcpy_h2d": (C.c_int, [_P, _P, C.c_size_t, _P]),
    "hj_memcpy_d2h": (C.c_int, [_P, _P, C.c_size_t, _P]),
    "hj_memset_device": (C.c_int, [_P, C.c_int, C.c_size_t, _P]),
    "hj_stream_create": (C.c_int, [C.POINTER(_P)]),
    "hj_stream_destroy": (C.c_int, [_P]),
    "hj_stream_synchronize": (C.c_int, [_P]),
    "hj_device_synchronize": (C.c_int, []),
    "hj_event_create": (C.c_int, [C.POINTER(_P)]),
    "hj_event_destroy": (C.c_int, [_P]),
    "hj_event_record": (C.c_int, [_P, _P]),
    "hj_event_elapsed_ms": (C.c_int, [_P, _P, C.POINTER(C.c_float)]),
    "hj_stream_wait_event": (C.c_int, [_P, _P]),
    "hj_render_batch": (C.c_int, [C.POINTER(hj_image_t), C.c_int, _P]),
    "hj_plan_create": (C.c_int, [C.POINTER(hj_image_t), C.c_int, C.POINTER(_P)]),
    "hj_plan_launch": (C.c_int, [_P, _P]),
    "hj_plan_destroy": (C.c_int, [_P]),
    "hj_launch_count": (C.c_uint64, []),
    "hj_exact_block_count": (C.c_uint64, []),
    "hj_tc_launch_count": (C.c_uint64, []),
    "hj_set_packed_h2d": (C.c_int, [C.c_int32]),
    "hj_packed_h2d_active": (C.c_int32, []),
    "hj_set_pack_band": (C.c_int, [C.c_int64]),
    "hj_h2d_bytes": (C.c_uint64, []),
    "hj_pack_blocks": (C.c_int64, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "hj_unpack_blocks_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "hj_render_rows": (C.c_int, [_P, _P, _P, _P, _P, _I32, _I32, _I32, _I32, _I32, _I32, _I32,
                                 _I32, _I32, _I64, _I64]),
    "hj_render_rows_timed": (C.c_int, [_P, _P, _P, _P, _P, _I32, _I32, _I32, _I32, _I32, _I32,
                                       _I32, _I32, _I32, _I64, _I64, _P]),
    "hj_idct_blocks": (C.c_int, [_P, _I64, _P, _I32]),
    "hj_idct_blocks_f64": (C.c_int, [_P, _I64, _P, _I32]),
    "hj_ycbcr_to_rgb": (C.c_int, [_P, _P, _P, _P, _I64]),
    "hj_upsample_422": (C.c_int, [_P, _P, _P, _P, _I64]),
    "hj_decode_mcu_rows": (C.c_int, [_P, _I64, _P, C.POINTER(hj_scan_tables_t), _P, _P, _P, _I32,
                                     _I32, _I32, _I32, _I32]),
    "hj_scan_entropy_end": (C.c_int64, [_P, _I64, _I64]),
    "hj_huff_build": (C.c_int, [C.POINTER(hj_scan_tables_t), C.POINTER(_P)]),
    "hj_huff_free": (None, [_P]),
    "hj_decode_scan_fast": (C.c_int, [_P, _P, _I64, _P, _P, _P, _I32, _I32, _I32, _I32, _I32]),
    "hj_decode_scan_rows": (C.c_int, [_P, _P, _I64, _P, _P, _P, _I32, _I32, _I32, _I32, _I32, _I32, _I32]),
    "hj_pipeline_run": (C.c_int, [C.POINTER(hj_pipe_image_t), _I32, _I32, C.POINTER(_P)]),
    "hj_partition_solve": (C.c_int, [C.POINTER(hj_balance_term_t), _I32, _I32, _I32, C.POINTER(hj_partition_t)]),
    "hj_balance_eval": (C.c_double, [C.POINTER(hj_balance_term_t), _I32, C.c_double, C.c_double,
                                     C.POINTER(C.c_double)]),
    "hj_stream_run": (C.c_int, [C.POINTER(hj_stream_image_t), _I32, _I32, _I32, _I32,
                                C.POINTER(hj_stream_stats_t)]),
    "hj_pipeline_huffman": (C.c_int, [C.POINTER(hj_pipe_image_t), _I32, _I32]),
}
for _name, (_res, _args) in _SIG.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

EXPORTED = tuple(_SIG)


def last_error() -> str:
    return lib.hj_last_error().decode(errors="replace")


def check(status: int, what: str = "") -> None:
    """Map an hj_status onto the reference exception classes."""
    if status == HJ_OK:
        return
    msg = last_error() or what
    # entropy errors carry the reference's messages (_native.pyx:298-305); the
    # library's context (which image / restart interval) is appended when it has one
    ref = {HJ_ERR_EXHAUSTED: (BitstreamExhausted, "ran out of entropy-coded bits"),
           HJ_ERR_BADCODE: (BadCode, "no Huffman symbol matches within 16 bits"),
           HJ_ERR_MARKER: (MarkerInScan, "non-restart marker inside the scan"),
           HJ_ERR_RST_SEQ: (MarkerInScan, "restart marker out of sequence")}.get(status)
    if ref is not None:
        cls, text = ref
        raise cls(text if not msg or msg == text else f"{text} ({msg})")
    if status == HJ_ERR_ARG:
        raise ValueError(msg)
    if status == HJ_ERR_NODEVICE:
        raise NoDevice(msg)
    raise CudaError(f"{what}: {msg}")


_device_lock = threading.Lock()
_device_ready = False


def require_device() -> None:
    """Fail loudly when no GPU is visible (no CPU fallback exists)."""
    global _device_ready
    if _device_ready:
        return
    with _device_lock:
        if lib.hj_device_count() <= 0:
            raise NoDevice("no CUDA device visible; the hetjpeg-b200 parallel phase "
                           "runs only on the GPU")
        _device_ready = True


def ptr(a: np.ndarray) -> int:
    """Address of a contiguous array's data.  ctypes' from_buffer is ~3x
    cheaper than `a.ctypes.data` (which builds a helper object per call) - it
    matters for the drop-in's many small per-image calls from lane threads,
    which hold the GIL while they marshal arguments; read-only or empty
    arrays take the generic path."""
    try:
        return C.addressof(C.c_char.from_buffer(a))
    except (TypeError, ValueError, BufferError):
        return a.ctypes.data


def version() -> str:
    return lib.hj_version().decode()
