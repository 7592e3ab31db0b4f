import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np
import bench
from paper_1311_5304_b200 import pipeline, device, _lib
from paper_1311_5304_b200.entropy import PinnedArray
wl = bench.WORKLOADS["1080p420"]
images = bench.make_inputs(wl, 0, 128)
geos = [images[i % 8][2].geometry for i in range(128)]
coeffs = [images[i % 8][2] for i in range(128)]
qts = [images[i % 8][3] for i in range(128)]
owners = [PinnedArray((g.height, g.width, 3), np.uint8) for g in geos]
outs = [o.array for o in owners]
lane = pipeline.GpuLane(geos, chunk=4)
b = lane.batch
for _ in range(2): lane.run(coeffs, qts, outs)
def t(f, n=5):
    f(); ts=[]
    for _ in range(n):
        t0=time.perf_counter(); f(); ts.append(time.perf_counter()-t0)
    return min(ts)*1e3
def h2d_only():
    for i in range(128): b.upload_coefficients(i, coeffs[i], lane.h2d)
    lane.h2d.synchronize()
def d2h_only():
    for i in range(128): b.download_rgb(i, outs[i], lane.d2h)
    lane.d2h.synchronize()
def both():
    for i in range(128):
        b.upload_coefficients(i, coeffs[i], lane.h2d); b.download_rgb(i, outs[i], lane.d2h)
    lane.h2d.synchronize(); lane.d2h.synchronize()
def issue_only():
    t0=time.perf_counter()
    for i in range(128): b.upload_coefficients(i, coeffs[i], lane.h2d)
    dt=time.perf_counter()-t0; lane.h2d.synchronize(); return dt
print("h2d ms", t(h2d_only), "d2h ms", t(d2h_only), "both ms", t(both), "lane.run ms", t(lambda: lane.run(coeffs, qts, outs)))
print("issue-only h2d ms", issue_only()*1e3)

