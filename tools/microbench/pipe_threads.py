import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1311_5304_b200.pipeline import BatchDecoder
from paper_1311_5304_b200.synth import synth_jpeg
print("cores", len(os.sched_getaffinity(0)))
blobs = [synth_jpeg(1920, 1080, 90, "420", seed=i) for i in range(8)]
for n in (32, 64):
    for threads in (12, 14, 15, 16):
        dec = BatchDecoder([blobs[i % 8] for i in range(n)], threads=threads, n_streams=4)
        dec.run()
        hs, ws = [], []
        for _ in range(7):
            hs.append(dec.huffman_only()); ws.append(dec.run()["wall_s"])
        dec.close()
        th, tw = float(np.median(hs)) * 1e3, float(np.median(ws)) * 1e3
        print(f"n={n} threads={threads}: huff {th:.2f} ms (min {min(hs)*1e3:.2f})  wall {tw:.2f} ms (min {min(ws)*1e3:.2f})  frac {th/tw:.3f}", flush=True)
