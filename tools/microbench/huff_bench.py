"""Single-thread host Huffman (hj_decode_scan_fast) throughput on synthetic
scans: best of N whole-scan decodes, MB/s of entropy-coded data and Mpix/s."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

from paper_1311_5304_b200 import entropy, parser  # noqa: E402
from paper_1311_5304_b200.synth import synth_jpeg  # noqa: E402

for (w, h, q, sub) in [(1920, 1080, 90, "420"), (1920, 1080, 50, "420"), (2048, 2048, 95, "444")]:
    blob = synth_jpeg(w, h, q, sub, seed=3)
    p = parser.parse_stream(blob)
    fs = entropy.FastScan(p)
    out = entropy.alloc_coefficients(fs.geometry)
    ref, _ = entropy.decode_all(p, blob)
    fs.decode(blob, out=out)
    assert np.array_equal(out.y_blocks, ref.y_blocks) and np.array_equal(out.cr_blocks, ref.cr_blocks)
    best = 1e9
    for _ in range(int(os.environ.get("HB_REPS", "30"))):
        t0 = time.perf_counter()
        fs.decode(blob, out=out)
        best = min(best, time.perf_counter() - t0)
    mb = p.entropy_span.length / 1e6
    print(f"{w}x{h} q{q} {sub}: {best * 1e3:.2f} ms  {mb / best:.0f} MB/s  {w * h / best / 1e6:.0f} Mpix/s per thread",
          flush=True)
