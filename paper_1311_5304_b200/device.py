"""Device-resident batches: the B200 "accelerator lane" without per-call
staging.  Coefficients and RGB of many images live in HBM; one
`hj_plan_launch` renders the whole batch (one kernel launch per subsampling
family).  Used by the pipelined orchestrator modes, the multi-image scheduler
and bench.py.

Only plain device pointers cross the C ABI; this module owns them through
small RAII wrappers over hj_malloc_device / hj_malloc_host.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib

_SUB = {(8, 8): _lib.SUB_444, (16, 8): _lib.SUB_422, (16, 16): _lib.SUB_420}


class DeviceBuffer:
    def __init__(self, nbytes: int):
        _lib.require_device()
        p = C.c_void_p()
        _lib.check(_lib.lib.hj_malloc_device(C.byref(p), max(int(nbytes), 1)), "hj_malloc_device")
        self.ptr = p.value
        self.nbytes = int(nbytes)

    def free(self):
        if self.ptr:
            _lib.lib.hj_free_device(self.ptr)
            self.ptr = None

    def __del__(self):
        self.free()


class Stream:
    def __init__(self):
        _lib.require_device()
        p = C.c_void_p()
        _lib.check(_lib.lib.hj_stream_create(C.byref(p)), "hj_stream_create")
        self.handle = p.value

    def synchronize(self):
        _lib.check(_lib.lib.hj_stream_synchronize(self.handle), "hj_stream_synchronize")

    def wait(self, event: "Event") -> None:
        """Device-side wait of this stream for `event`."""
        _lib.check(_lib.lib.hj_stream_wait_event(self.handle, event.handle), "hj_stream_wait_event")

    def __del__(self):
        if getattr(self, "handle", None):
            _lib.lib.hj_stream_destroy(self.handle)
            self.handle = None


class Event:
    def __init__(self):
        p = C.c_void_p()
        _lib.check(_lib.lib.hj_event_create(C.byref(p)), "hj_event_create")
        self.handle = p.value

    def record(self, stream: "Stream | None" = None):
        _lib.check(_lib.lib.hj_event_record(self.handle, stream.handle if stream else None), "record")

    def elapsed_ms(self, end: "Event") -> float:
        ms = C.c_float()
        _lib.check(_lib.lib.hj_event_elapsed_ms(self.handle, end.handle, C.byref(ms)), "elapsed")
        return float(ms.value)

    def __del__(self):
        if getattr(self, "handle", None):
            _lib.lib.hj_event_destroy(self.handle)
            self.handle = None


def subsampling_code(geometry) -> int:
    return _SUB[(geometry.mcu_width, geometry.mcu_height)]


@dataclass
class ImageSlot:
    """Device placement of one image inside a DeviceBatch."""
    geometry: object
    y_off: int          # byte offsets into the coefficient arena
    cb_off: int
    cr_off: int
    coef_bytes: int
    q_off: int
    rgb_off: int        # byte offset into the RGB arena
    rgb_bytes: int
    n_y: int
    n_c: int


class DeviceBatch:
    """A fixed set of images resident on the device.

    `geometries` lists ImageGeometry objects; each image gets a contiguous
    coefficient region [Y | Cb | Cr] (the host CoefficientBuffer layout, so
    one H2D copy moves it) and an RGB region (h*w*3).  `fast=False` selects
    the direct-basis IDCT for every image, `fast="islow"` libjpeg's integer
    decode (the islow mode).
    """

    def __init__(self, geometries, fast=True):
        _lib.require_device()
        self.slots = []
        coef = rgb = 0
        for geo in geometries:
            n_c = geo.total_mcus
            n_y = n_c * geo.y_blocks_per_mcu
            cb = (n_y + 2 * n_c) * 128
            rb = geo.width * geo.height * 3
            self.slots.append(ImageSlot(geo, coef, coef + n_y * 128, coef + (n_y + n_c) * 128, cb,
                                        len(self.slots) * 768, rgb, rb, n_y, n_c))
            coef += (cb + 255) // 256 * 256
            rgb += (rb + 255) // 256 * 256
        self.coef = DeviceBuffer(coef)
        self.rgb = DeviceBuffer(rgb)
        self.q = DeviceBuffer(768 * max(1, len(self.slots)))
        self.fast = fast
        self._plan = None
        self._plans = {}  # cached plans for item tuples (tile lists stay resident)

    # ---- descriptors
    def image_desc(self, i: int, row0: int = 0, n_rows: int | None = None) -> _lib.hj_image_t:
        s = self.slots[i]
        g = s.geometry
        d = _lib.hj_image_t()
        d.y = self.coef.ptr + s.y_off
        d.cb = self.coef.ptr + s.cb_off
        d.cr = self.coef.ptr + s.cr_off
        d.q = self.q.ptr + s.q_off
        d.rgb = self.rgb.ptr + s.rgb_off
        d.width, d.height = g.width, g.height
        d.mcus_per_row, d.mcu_rows = g.mcus_per_row, g.mcu_rows
        d.row0 = row0
        d.n_rows = g.mcu_rows - row0 if n_rows is None else n_rows
        d.subsampling = subsampling_code(g)
        d.flags = _lib.image_flags(self.fast)
        return d

    def descs(self, items) -> C.Array:
        """items: iterable of (image index, row0, n_rows)."""
        items = list(items)
        arr = (_lib.hj_image_t * max(1, len(items)))()
        for k, (i, r0, n) in enumerate(items):
            arr[k] = self.image_desc(i, r0, n)
        return arr, len(items)

    # ---- transfers (host arrays must stay alive until the stream syncs)
    def upload_coefficients(self, i: int, coeffs, stream: Stream | None = None, row0: int = 0,
                            n_rows: int | None = None) -> int:
        """H2D of MCU rows [row0, row0+n_rows) of image i (all planes)."""
        s = self.slots[i]
        g = s.geometry
        n_rows = g.mcu_rows - row0 if n_rows is None else n_rows
        ypm = g.y_blocks_per_mcu
        h = stream.handle if stream else None
        moved = 0
        for arr, off, per_row in ((coeffs.y_blocks, s.y_off, g.mcus_per_row * ypm),
                                  (coeffs.cb_blocks, s.cb_off, g.mcus_per_row),
                                  (coeffs.cr_blocks, s.cr_off, g.mcus_per_row)):
            nbytes = n_rows * per_row * 128
            if nbytes == 0:
                continue
            src = arr.ctypes.data + row0 * per_row * 128
            _lib.check(_lib.lib.hj_memcpy_h2d(self.coef.ptr + off + row0 * per_row * 128, src,
                                              nbytes, h), "h2d coefficients")
            moved += nbytes
        return moved

    def upload_qtables(self, i: int, q: np.ndarray, stream: Stream | None = None) -> None:
        q = np.ascontiguousarray(q, np.int32)
        if q.shape != (3, 64):
            raise ValueError("qtables must be (3, 64)")
        self._keep_q = getattr(self, "_keep_q", {})
        self._keep_q[i] = q
        _lib.check(_lib.lib.hj_memcpy_h2d(self.q.ptr + self.slots[i].q_off, q.ctypes.data, 768,
                                          stream.handle if stream else None), "h2d q")

    def download_rgb(self, i: int, out: np.ndarray, stream: Stream | None = None, y0: int = 0,
                     y1: int | None = None) -> int:
        s = self.slots[i]
        g = s.geometry
        y1 = g.height if y1 is None else y1
        row_b = g.width * 3
        nbytes = (y1 - y0) * row_b
        if nbytes <= 0:
            return 0
        if out.dtype != np.uint8 or out.shape != (g.height, g.width, 3) or not out.flags.c_contiguous:
            raise ValueError("out must be a C-contiguous uint8 (h, w, 3) array")
        _lib.check(_lib.lib.hj_memcpy_d2h(out.ctypes.data + y0 * row_b,
                                          self.rgb.ptr + s.rgb_off + y0 * row_b, nbytes,
                                          stream.handle if stream else None), "d2h rgb")
        return nbytes

    # ---- launches
    def render(self, items=None, stream: Stream | None = None) -> None:
        """Render (image, row0, n_rows) items; default = every image fully.
        The whole-batch plan is cached (tile list resident on the device)."""
        h = stream.handle if stream else None
        if items is None:
            if self._plan is None:
                arr, n = self.descs((i, 0, s.geometry.mcu_rows) for i, s in enumerate(self.slots))
                p = C.c_void_p()
                _lib.check(_lib.lib.hj_plan_create(arr, n, C.byref(p)), "hj_plan_create")
                self._plan = p.value
            _lib.check(_lib.lib.hj_plan_launch(self._plan, h), "hj_plan_launch")
            return
        arr, n = self.descs(items)
        p = C.c_void_p()
        _lib.check(_lib.lib.hj_plan_create(arr, n, C.byref(p)), "hj_plan_create")
        try:
            _lib.check(_lib.lib.hj_plan_launch(p.value, h), "hj_plan_launch")
            if stream is not None:
                stream.synchronize()
            else:
                _lib.check(_lib.lib.hj_device_synchronize(), "sync")
        finally:
            _lib.lib.hj_plan_destroy(p.value)

    def render_items(self, items, stream: Stream | None = None) -> None:
        """Asynchronous render of (image, row0, n_rows) items on `stream`
        with a cached plan (no host synchronisation)."""
        key = tuple(items)
        plan = self._plans.get(key)
        if plan is None:
            arr, n = self.descs(key)
            p = C.c_void_p()
            _lib.check(_lib.lib.hj_plan_create(arr, n, C.byref(p)), "hj_plan_create")
            plan = self._plans[key] = p.value
        _lib.check(_lib.lib.hj_plan_launch(plan, stream.handle if stream else None),
                   "hj_plan_launch")

    def algorithmic_bytes(self) -> int:
        """Coefficient bytes in (MCU padding included) + RGB bytes out:
        WorkItem.write_bytes + read_bytes of the whole batch (executors.py:75-86)."""
        return sum(s.coef_bytes + s.rgb_bytes for s in self.slots)

    def pixels(self) -> int:
        return sum(s.geometry.width * s.geometry.height for s in self.slots)

    def close(self):
        if self._plan:
            _lib.lib.hj_plan_destroy(self._plan)
            self._plan = None
        for plan in self._plans.values():
            _lib.lib.hj_plan_destroy(plan)
        self._plans = {}
        self.coef.free()
        self.rgb.free()
        self.q.free()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
