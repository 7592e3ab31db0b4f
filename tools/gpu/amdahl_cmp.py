"""Amdahl fraction of the two pipeline APIs on the same batch (diagnostic):
BatchDecoder (hj_pipeline_run, every worker queues its own image's CUDA work)
vs StreamDecoder (hj_stream_run, workers only decode, one submitter)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.getcwd())
from paper_1311_5304_b200 import pipeline  # noqa: E402
from paper_1311_5304_b200.synth import synth_jpeg  # noqa: E402

for (w, h, q, sub, n) in [(1920, 1080, 90, "420", 128), (512, 512, 75, "420", 240)]:
    blobs = [synth_jpeg(w, h, q, sub, seed=i) for i in range(8)]
    batch = [blobs[i % 8] for i in range(n)]
    bd = pipeline.BatchDecoder(batch, threads=16, n_streams=4, fast=True)
    bd.run()
    hb, wb = [], []
    for _ in range(5):
        hb.append(bd.huffman_only())
        wb.append(bd.run()["wall_s"])
    bd.close()
    for keep in ((), tuple(range(n))):
        sd = pipeline.StreamDecoder(batch, threads=16, keep=keep)
        sd.huffman_only()
        sd.run()
        hs, ws = [], []
        for _ in range(5):
            hs.append(sd.huffman_only()["wall_s"])
            ws.append(sd.run()["wall_s"])
        print(f"{w}x{h} n={n}: batch {np.median(hb)/np.median(wb):.3f} (huff {np.median(hb)*1e3:.1f} wall {np.median(wb)*1e3:.1f} ms)"
              f" | stream keep={len(keep)} {np.median(hs)/np.median(ws):.3f} (huff {np.median(hs)*1e3:.1f} wall {np.median(ws)*1e3:.1f} ms)", flush=True)
