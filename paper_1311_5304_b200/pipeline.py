"""The GPU lane: chunked, stream-overlapped H2D -> render -> D2H over
page-locked host buffers.

This is the real counterpart of the reference's simulated accelerator lane
(executors.py:131-197, whose transfers are `sleep(latency + bytes/bw)`):
chunks of images (or MCU-row ranges) alternate between CUDA streams so the
PCIe copies of chunk k+1 / k-1 overlap the kernel of chunk k.
"""
from __future__ import annotations

import numpy as np

from . import _lib, device
from .entropy import PinnedArray


class GpuLane:
    """Render many host-resident coefficient buffers into host RGB buffers."""

    def __init__(self, geometries, n_streams: int = 3, chunk: int = 8, fast: bool = True):
        self.batch = device.DeviceBatch(geometries, fast=fast)
        self.streams = [device.Stream() for _ in range(n_streams)]
        self.chunk = max(1, int(chunk))
        self.n = len(geometries)
        self._q = PinnedArray((max(1, self.n), 3, 64), np.int32)  # staging for the qtables

    def run(self, coeffs, qtables, outs) -> dict:
        """coeffs[i]: CoefficientBuffer (pinned for async DMA), qtables[i]:
        (3, 64), outs[i]: (h, w, 3) uint8 host array.  Returns byte counts."""
        h2d = d2h = 0
        b = self.batch
        for k, start in enumerate(range(0, self.n, self.chunk)):
            s = self.streams[k % len(self.streams)]
            idx = range(start, min(self.n, start + self.chunk))
            for i in idx:
                h2d += b.upload_coefficients(i, coeffs[i], s)
                self._q.array[i] = qtables[i]
            nq = 768 * len(idx)
            _lib.check(_lib.lib.hj_memcpy_h2d(b.q.ptr + b.slots[start].q_off,
                                              self._q.array[start:].ctypes.data, nq, s.handle),
                       "h2d q")
            h2d += nq
            b.render_items([(i, 0, b.slots[i].geometry.mcu_rows) for i in idx], s)
            for i in idx:
                d2h += b.download_rgb(i, outs[i], s)
        for s in self.streams:
            s.synchronize()
        return {"h2d_bytes": h2d, "d2h_bytes": d2h}

    def close(self):
        self.batch.close()


def render_batch(coeffs, qtables, outs=None, chunk: int = 8, n_streams: int = 3):
    """Public one-shot API: render a list of decoded images on the GPU.
    Returns the list of RGB arrays."""
    geos = [c.geometry for c in coeffs]
    if outs is None:
        outs = [np.zeros((g.height, g.width, 3), np.uint8) for g in geos]
    lane = GpuLane(geos, n_streams=n_streams, chunk=chunk)
    try:
        lane.run(coeffs, qtables, outs)
    finally:
        lane.close()
    return outs
