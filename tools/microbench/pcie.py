"""Pinned host <-> device copy bandwidth on this box: H2D alone, D2H alone,
and both directions concurrently on two streams (the e2e ceiling)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1311_5304_b200 import _lib, device  # noqa: E402
from paper_1311_5304_b200.entropy import PinnedArray  # noqa: E402
import numpy as np  # noqa: E402

N = 512 << 20
h1, h2 = PinnedArray((N,), np.uint8), PinnedArray((N,), np.uint8)
d1, d2 = device.DeviceBuffer(N), device.DeviceBuffer(N)
s1, s2 = device.Stream(), device.Stream()
L = _lib.lib


def run(kind, reps=5, chunk=N):
    t0 = time.perf_counter()
    for _ in range(reps):
        for off in range(0, N, chunk):
            n = min(chunk, N - off)
            if kind in ("h2d", "both"):
                L.hj_memcpy_h2d(d1.ptr + off, h1.array.ctypes.data + off, n, s1.handle)
            if kind in ("d2h", "both"):
                L.hj_memcpy_d2h(h2.array.ctypes.data + off, d2.ptr + off, n, s2.handle)
    s1.synchronize()
    s2.synchronize()
    dt = time.perf_counter() - t0
    mult = 2 if kind == "both" else 1
    return reps * N * mult / dt / 1e9


for k in ("h2d", "d2h", "both"):
    run(k, 1)
    print(k, "GB/s", round(run(k), 1), "chunked 8MB:", round(run(k, chunk=8 << 20), 1))
