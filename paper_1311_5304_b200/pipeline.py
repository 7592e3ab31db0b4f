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
    """Render many host-resident coefficient buffers into host RGB buffers.

    Three-stage pipeline over chunks of images on three CUDA streams joined
    by events: the H2D stream copies chunk k+1 while the compute stream
    renders chunk k and the D2H stream drains chunk k-1, so both PCIe
    directions stay busy (the copy engines are independent: ~92 GB/s
    duplex on this box, tools/microbench/pcie.py)."""

    def __init__(self, geometries, n_streams: int = 3, chunk: int = 4, fast=True):
        self.batch = device.DeviceBatch(geometries, fast=fast)
        self.h2d, self.comp, self.d2h = device.Stream(), device.Stream(), device.Stream()
        self.streams = [self.h2d, self.comp, self.d2h]
        self.chunk = max(1, int(chunk))
        self.n = len(geometries)
        n_chunks = -(-self.n // self.chunk)
        self._up = [device.Event() for _ in range(n_chunks)]
        self._done = [device.Event() for _ in range(n_chunks)]
        self._q = PinnedArray((max(1, self.n), 3, 64), np.int32)  # staging for the qtables

    def run(self, coeffs, qtables, outs) -> dict:
        """coeffs[i]: CoefficientBuffer (pinned for async DMA), qtables[i]:
        (3, 64), outs[i]: (h, w, 3) uint8 host array.  Returns byte counts."""
        h2d = d2h = 0
        b = self.batch
        for k, start in enumerate(range(0, self.n, self.chunk)):
            idx = range(start, min(self.n, start + self.chunk))
            for i in idx:
                h2d += b.upload_coefficients(i, coeffs[i], self.h2d)
                self._q.array[i] = qtables[i]
            nq = 768 * len(idx)
            _lib.check(_lib.lib.hj_memcpy_h2d(b.q.ptr + b.slots[start].q_off,
                                              self._q.array[start:].ctypes.data, nq, self.h2d.handle),
                       "h2d q")
            h2d += nq
            self._up[k].record(self.h2d)
            self.comp.wait(self._up[k])
            b.render_items([(i, 0, b.slots[i].geometry.mcu_rows) for i in idx], self.comp)
            self._done[k].record(self.comp)
            self.d2h.wait(self._done[k])
            for i in idx:
                d2h += b.download_rgb(i, outs[i], self.d2h)
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


class BatchDecoder:
    """End-to-end batch decode: host Huffman on a thread pool (native C++,
    GIL released) pipelined with the B200 parallel phase.

    Each host worker entropy-decodes an image (into page-locked coefficient
    buffers) and then queues that image's H2D -> render -> D2H on its own
    CUDA stream, so the GPU work of finished images overlaps the Huffman
    decoding of the rest with no central dispatcher in the way - the paper's
    pipelined scheme (§5.3) at batch granularity.  `huffman_only()` times the same
    host stage alone (same decoder, same thread count): T_huff of the Amdahl
    bound wall / huffman (orchestrator.py:71-75).
    """

    def __init__(self, blobs, threads: int = 0, n_streams: int = 4, fast=True):
        import os

        from . import entropy, parser
        from .block_transforms import alloc_pixels
        from .perf_model import qtable_stack
        self.threads = threads or len(os.sched_getaffinity(0))
        self.blobs = [bytes(b) for b in blobs]
        self.parsed = [parser.parse_stream(b) for b in self.blobs]
        self.scans = [entropy.FastScan(p) for p in self.parsed]
        self.geos = [s.geometry for s in self.scans]
        self.q = [qtable_stack(p) for p in self.parsed]
        self.coeffs = [entropy.alloc_coefficients(g, pinned=True) for g in self.geos]
        self.pixels = [alloc_pixels(g.width, g.height, pinned=True) for g in self.geos]
        self.batch = device.DeviceBatch(self.geos, fast=fast)
        # one CUDA stream per host worker: a worker that finishes an image's
        # entropy decode queues that image's H2D -> render -> D2H itself
        self.streams = [device.Stream() for _ in range(max(1, n_streams, self.threads))]
        for i in range(len(self.geos)):
            self.batch.upload_qtables(i, self.q[i], self.streams[0])
            self.batch.render_items([(i, 0, self.geos[i].mcu_rows)], self.streams[0])  # cache the plans
        self.streams[0].synchronize()
        self._native = self._pipe_descriptors()

    def _pipe_descriptors(self):
        """hj_pipe_image_t per image for the native pipeline (hj_pipeline_run)."""
        import ctypes as C

        import numpy as np
        b = self.batch
        arr = (_lib.hj_pipe_image_t * max(1, len(self.geos)))()
        self._scan_views = []
        for i, g in enumerate(self.geos):
            sp = self.parsed[i].entropy_span
            view = np.frombuffer(self.blobs[i], dtype=np.uint8)[sp.offset:sp.offset + sp.length]
            self._scan_views.append(view)
            c, slot = self.coeffs[i], b.slots[i]
            d = arr[i]
            d.huff = self.scans[i]._h
            d.scan, d.scan_bytes = view.ctypes.data, len(view)
            d.y, d.cb, d.cr = c.y_blocks.ctypes.data, c.cb_blocks.ctypes.data, c.cr_blocks.ctypes.data
            d.dev_y, d.dev_cb, d.dev_cr = (b.coef.ptr + slot.y_off, b.coef.ptr + slot.cb_off,
                                           b.coef.ptr + slot.cr_off)
            d.n_y, d.n_c = len(c.y_blocks), len(c.cb_blocks)
            d.mcus_per_row, d.mcu_rows, d.y_per_mcu = g.mcus_per_row, g.mcu_rows, g.y_blocks_per_mcu
            d.restart_interval = self.parsed[i].restart_interval
            d.plan = b._plans[((i, 0, g.mcu_rows),)]
            d.dev_rgb = b.rgb.ptr + slot.rgb_off
            d.rgb, d.rgb_bytes = self.pixels[i].data.ctypes.data, g.width * g.height * 3
        handles = (C.c_void_p * len(self.streams))(*[s.handle for s in self.streams])
        self._h2d = sum(2 * len(c.y_blocks) * 64 + 2 * 2 * len(c.cb_blocks) * 64 for c in self.coeffs)
        self._d2h = sum(g.width * g.height * 3 for g in self.geos)
        return arr, handles

    def _huff(self, i: int) -> int:
        self.scans[i].decode(self.blobs[i], out=self.coeffs[i], threads=1)
        return i

    def huffman_only(self) -> float:
        """Wall seconds of the host entropy stage alone over the batch (native
        threads, hj_pipeline_huffman: the same work as run() minus the GPU)."""
        import time
        arr, _ = self._native
        t0 = time.perf_counter()
        _lib.check(_lib.lib.hj_pipeline_huffman(arr, len(self.geos), self.threads), "pipeline huffman")
        return time.perf_counter() - t0

    def run(self) -> dict:
        """Decode the whole batch into self.pixels (native pipeline,
        hj_pipeline_run: no Python between an image's Huffman and its GPU work);
        returns wall seconds and bytes moved."""
        import time
        arr, handles = self._native
        t0 = time.perf_counter()
        _lib.check(_lib.lib.hj_pipeline_run(arr, len(self.geos), self.threads, handles), "pipeline run")
        return {"wall_s": time.perf_counter() - t0, "h2d_bytes": self._h2d, "d2h_bytes": self._d2h}

    def huffman_only_threads(self) -> float:
        """huffman_only() through a Python thread pool (comparison)."""
        import time
        from concurrent.futures import ThreadPoolExecutor
        t0 = time.perf_counter()
        with ThreadPoolExecutor(self.threads) as ex:
            list(ex.map(self._huff, range(len(self.blobs))))
        return time.perf_counter() - t0

    def run_threads(self) -> dict:
        """run() through a Python thread pool, one ctypes call per step
        (comparison: the GIL between the calls costs small images)."""
        import threading
        import time
        from concurrent.futures import ThreadPoolExecutor
        b = self.batch
        slot = threading.local()
        counter = iter(range(len(self.streams)))
        lock = threading.Lock()

        def work(i):
            if not hasattr(slot, "stream"):
                with lock:
                    slot.stream = self.streams[next(counter)]
            self._huff(i)
            s = slot.stream
            h2d = b.upload_coefficients(i, self.coeffs[i], s)
            b.render_items([(i, 0, self.geos[i].mcu_rows)], s)
            return h2d, b.download_rgb(i, self.pixels[i].data, s)

        t0 = time.perf_counter()
        with ThreadPoolExecutor(self.threads) as ex:
            moved = list(ex.map(work, range(len(self.blobs))))
        for s in self.streams:
            s.synchronize()
        return {"wall_s": time.perf_counter() - t0, "h2d_bytes": sum(m[0] for m in moved),
                "d2h_bytes": sum(m[1] for m in moved)}

    def close(self):
        self.batch.close()


class StreamDecoder:
    """Whole-corpus decode with bounded memory (BASELINE config 5: 10k mixed
    images): a ring of `slots` reusable page-locked + device slots sized to
    the largest image (hj_stream_run).  Host threads Huffman-decode into free
    slots; the calling thread queues each slot's H2D -> render -> D2H and
    recycles finished ones - memory is O(slots), not O(corpus), unlike
    BatchDecoder, which keeps every image resident.

    `blobs` may repeat the same bytes object (a corpus drawn from a pool):
    each distinct blob is parsed and gets its Huffman tables once.  `keep`:
    indices whose RGB is copied out to page-locked arrays (self.kept[i]);
    the others are delivered into the ring and overwritten.  `order`: the
    processing order (default: largest first, which shortens the tail).
    `shards[i]` = (row0, n_rows): decode and render only those MCU rows of
    image i (BASELINE config 4: a rank's share of one large image; only its
    restart intervals are Huffman-decoded)."""

    def __init__(self, blobs, threads: int = 0, slots: int = 0, fast=True, keep=(), order=None, shards=None):
        import ctypes as C
        import os

        from . import entropy, parser
        from .perf_model import qtable_stack
        self.threads = threads or len(os.sched_getaffinity(0))
        self.slots = slots or self.threads + 4
        self._distinct = {}
        self._keep_alive = []
        per = []
        for b in blobs:
            key = id(b)
            if key not in self._distinct:
                p = parser.parse_stream(b)
                fs = entropy.FastScan(p)
                sp = p.entropy_span
                view = np.frombuffer(b, dtype=np.uint8)[sp.offset:sp.offset + sp.length]
                q = np.ascontiguousarray(qtable_stack(p), np.int32)
                self._distinct[key] = (b, p, fs, view, q)
            per.append(self._distinct[key])
        self.n = len(per)
        self.geometries = [d[2].geometry for d in per]
        self.pixels = sum(g.width * g.height for g in self.geometries)
        if shards is not None:
            self.pixels = sum(
                g.width * (min(g.height, (sh[0] + sh[1]) * g.mcu_height) - sh[0] * g.mcu_height) if sh
                else g.width * g.height for g, sh in zip(self.geometries, shards))
        if order is None:
            order = sorted(range(self.n), key=lambda i: -self.geometries[i].width * self.geometries[i].height)
        self.order = list(order)
        self.kept = {}
        keep = set(keep) if _lib.lib.hj_device_count() > 0 else set()  # page-locked outputs need a driver
        arr = (_lib.hj_stream_image_t * max(1, self.n))()
        for k, i in enumerate(self.order):
            b, p, fs, view, q = per[i]
            g = self.geometries[i]
            d = arr[k]
            d.huff = fs._h
            d.scan, d.scan_bytes = view.ctypes.data, len(view)
            d.q = q.ctypes.data
            d.width, d.height = g.width, g.height
            d.subsampling = device.subsampling_code(g)
            d.flags = _lib.image_flags(fast)
            d.restart_interval = p.restart_interval
            if shards is not None and shards[i] is not None:
                d.row0, d.n_rows = int(shards[i][0]), int(shards[i][1])
            if i in keep:
                out = PinnedArray((g.height, g.width, 3), np.uint8)
                self.kept[i] = out
                d.rgb_out = out.array.ctypes.data
        self._arr = arr
        self._C = C

    def _run(self, gpu: int) -> dict:
        import time
        stats = _lib.hj_stream_stats_t()
        t0 = time.perf_counter()
        _lib.check(_lib.lib.hj_stream_run(self._arr, self.n, self.threads, self.slots, gpu,
                                          self._C.byref(stats)), "hj_stream_run")
        call = time.perf_counter() - t0
        return {"wall_s": stats.wall_s, "call_s": call, "images": stats.images, "launches": stats.launches,
                "h2d_bytes": stats.h2d_bytes, "d2h_bytes": stats.d2h_bytes,
                "pinned_bytes": stats.pinned_bytes, "device_bytes": stats.device_bytes,
                "huffman_thread_s": stats.huffman_thread_s}

    def run(self) -> dict:
        """Decode the whole corpus (host Huffman pipelined with the B200)."""
        _lib.require_device()
        return self._run(1)

    def huffman_only(self) -> dict:
        """The same host stage alone: same decoder, threads and ring (T_huff)."""
        return self._run(0)

    def rgb(self, i: int) -> np.ndarray:
        return self.kept[i].array
