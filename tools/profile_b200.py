"""Recalibrate the paper's offline performance model on this B200 box
(perf_model.run_profiling, §5.1) and write the DeviceProfile JSON
(the reference's schema) to profiles/b200_profile.json.

    python tools/profile_b200.py [--out profiles/b200_profile.json] [--images 24]

Training set: synthetic JPEGs (SURVEY.md Appendix B content), 4:4:4 / 4:2:2 /
4:2:0 at q50-95, on a (w, h) grid from 320 to 6000 px - the size range of
BASELINE config 5 (0.3-24 MP) - so the fitted degree can carry the w*h
(area) term; max degree 3 (10 bivariate terms).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1311_5304_b200 import executors, perf_model  # noqa: E402
from paper_1311_5304_b200.synth import synth_jpeg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "b200_profile.json"))
    ap.add_argument("--images", type=int, default=40)
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--max-degree", type=int, default=3)
    args = ap.parse_args()
    sizes = [320, 640, 1024, 1600, 2400, 3200, 4000, 4800, 6000]
    blobs = []
    k = 0
    while len(blobs) < args.images:
        w = sizes[k % len(sizes)]
        h = sizes[(k * 4 + 3) % len(sizes)]
        if w * h > 24.5e6:  # config 5's largest images are 24 MP
            h = int(24e6 // w) // 16 * 16
        q = (50, 75, 90, 95)[k % 4]
        sub = ("420", "422", "444")[k % 3]
        blobs.append(synth_jpeg(w, h, q, sub, seed=k))
        k += 1
    lanes = executors.make_lanes()
    t0 = time.time()
    try:
        prof = perf_model.run_profiling(blobs, lanes, repeats=args.repeats, max_degree=args.max_degree,
                                        device_description="NVIDIA B200 (sm_100a) + host Huffman "
                                                           f"({lanes.meta['host_workers']} host workers)")
    finally:
        lanes.shutdown()
    perf_model.save_profile(prof, args.out)
    print(json.dumps({"out": args.out, "seconds": round(time.time() - t0, 1), "chunk_rows": prof.chunk_rows,
                      "degrees": {n: getattr(prof, n).degree for n in ("p_cpu", "p_gpu", "t_disp",
                                                                          "t_huff_per_pixel")}}))


if __name__ == "__main__":
    main()
