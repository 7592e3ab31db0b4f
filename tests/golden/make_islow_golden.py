"""Golden vectors of the "islow" decode mode, from libjpeg-turbo itself.

Run in the build container (Pillow with its bundled libjpeg-turbo):

    python tests/golden/make_islow_golden.py

north_star names libjpeg's fixed-point "islow" IDCT (jidctint.c); the
reference has no such path, so its oracle is libjpeg-turbo's own decode of
the same synthetic JPEGs: Pillow's default decode = jpeg_idct_islow +
fancy upsampling (jdsample.c) + integer YCbCr->RGB (jdcolor.c).  Written to
tests/golden/islow_golden.npz per case: the JPEG bytes (SURVEY.md Appendix B
generator, Pillow encoder) and the SHA-256 of the RGB libjpeg-turbo decodes,
plus the libjpeg-turbo version.  Covers widths 1..8 (box vs fancy
upsampling: libjpeg filters only when the chroma width exceeds 2), odd sizes,
q50-100, restart intervals, all three subsamplings, and BASELINE configs[0]
(512x512 4:2:0 q75).
"""
import hashlib
import io
import os
import sys

import numpy as np
from PIL import Image, features

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from paper_1311_5304_b200.synth import synth_jpeg  # noqa: E402

SIZES = [(1, 1), (2, 2), (3, 5), (4, 4), (5, 3), (6, 7), (7, 2), (8, 8), (9, 9), (17, 9), (31, 33), (64, 48),
         (97, 61), (200, 130)]


def main():
    out = {"libjpeg": np.array(f"libjpeg-turbo {features.version('libjpeg_turbo')}")}
    cases = [(w, h, q, sub, 0) for (w, h) in SIZES for sub in ("444", "422", "420") for q in (60, 95)]
    cases += [(512, 512, 75, "420", 0), (333, 211, 95, "422", 0), (256, 256, 90, "444", 0),
              (200, 130, 70, "422", 1), (160, 96, 85, "420", 1)]
    for k, (w, h, q, sub, rst) in enumerate(cases):
        blob = synth_jpeg(w, h, q, sub, seed=7 * k + 1, restart_rows=rst)
        rgb = np.asarray(Image.open(io.BytesIO(blob)).convert("RGB"))
        name = f"i{k:02d}_{w}x{h}_{sub}_q{q}" + ("_rst" if rst else "")
        out[name + "_jpeg"] = np.frombuffer(blob, np.uint8)
        out[name + "_sha"] = np.array(hashlib.sha256(np.ascontiguousarray(rgb).tobytes()).hexdigest())
    np.savez_compressed(os.path.join(HERE, "islow_golden.npz"), **out)
    print(len(cases), "cases;", out["libjpeg"])


if __name__ == "__main__":
    main()
