"""Native batch pipeline (hj_pipeline_run) vs its Huffman stage alone, by
image size and host thread count (diagnostic for the Amdahl fraction)."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

from paper_1311_5304_b200.pipeline import BatchDecoder  # noqa: E402
from paper_1311_5304_b200.synth import synth_jpeg  # noqa: E402

for (w, h, q, n) in [(512, 512, 75, 32), (512, 512, 75, 128), (1920, 1080, 90, 32)]:
    blobs = [synth_jpeg(w, h, q, "420", seed=i) for i in range(8)]
    for threads in (4, 8, 16):
        dec = BatchDecoder([blobs[i % 8] for i in range(n)], threads=threads, n_streams=4)
        dec.run()
        hs, ws, ts = [], [], []
        for _ in range(5):
            hs.append(dec.huffman_only())
            ws.append(dec.run()["wall_s"])
            t0 = time.perf_counter()
            dec.run_threads()
            ts.append(time.perf_counter() - t0)
        dec.close()
        th, tw, tt = (float(np.median(x)) * 1e3 for x in (hs, ws, ts))
        print(f"{w}x{h} n={n} threads={threads}: huff {th:.2f} ms  native {tw:.2f} ms (frac {th / tw:.2f})"
              f"  python-threads {tt:.2f} ms (frac {th / tt:.2f})", flush=True)
