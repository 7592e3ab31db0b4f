"""Per-image render throughput over the bench's mixed manifest (diagnostic)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
from paper_1311_5304_b200 import device, entropy, parser  # noqa: E402
from paper_1311_5304_b200.perf_model import qtable_stack  # noqa: E402
from paper_1311_5304_b200.synth import synth_jpeg  # noqa: E402

man = bench.mixed_manifest(24)
st = device.Stream()
for k, (w, h, q, sub) in enumerate(man):
    blob = synth_jpeg(w, h, q, sub, seed=k)
    p = parser.parse_stream(blob)
    c, _ = entropy.decode_all(p, blob, pinned=True)
    db = device.DeviceBatch([c.geometry] * 4)
    for i in range(4):
        db.upload_coefficients(i, c, st)
        db.upload_qtables(i, qtable_stack(p), st)
    for _ in range(3):
        db.render(stream=st)
    e0, e1 = device.Event(), device.Event()
    e0.record(st)
    for _ in range(20):
        db.render(stream=st)
    e1.record(st)
    st.synchronize()
    ms = e0.elapsed_ms(e1) / 20
    print(f"{w}x{h} q{q} {sub}: {4 * w * h / ms / 1e3:9.0f} Mpix/s  ({ms * 1e3:.0f} us for 4 images)")
    db.close()
