"""Reference hashes at BASELINE sizes the reference itself decodes.

Run in the build container only (reference build in oracle/_ref):

    python tests/golden/make_big_hashes.py

BASELINE.json configs[2] are 4096x4096 4:4:4 and 4:2:2 at q95 - the two
BASELINE configurations the reference accepts.  For each, the synthetic JPEG
(paper_1311_5304_b200.synth, SURVEY.md Appendix B generator, Pillow encoder)
is decoded by the REFERENCE (native build, oracle/_ref/patched): its
entropy.decode_all and its render_rows with idct fast and direct.  Only
SHA-256 digests are committed (tests/golden/big_hashes.json): of the JPEG
bytes (detects encoder drift), of the coefficient planes and of each RGB.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
from paper_1311_5304_b200.synth import synth_jpeg  # noqa: E402

sys.path.insert(0, os.path.join(REPO, "oracle", "_ref", "patched"))
from hetjpeg import entropy, parser  # noqa: E402
from hetjpeg.block_transforms import alloc_pixels, render_rows  # noqa: E402
from hetjpeg.perf_model import _qtable_stack  # noqa: E402

CASES = [("4096p444q95", 4096, 4096, 95, "444", 0), ("4096p422q95", 4096, 4096, 95, "422", 0),
         ("1080p422q90rst", 1920, 1080, 90, "422", 2)]


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    out = {}
    for name, w, h, q, sub, rst in CASES:
        blob = synth_jpeg(w, h, q, sub, seed=0, restart_rows=rst)
        p = parser.parse_stream(blob)
        c, _ = entropy.decode_all(p, blob)
        g = c.geometry
        qt = _qtable_stack(p)
        rec = {"w": w, "h": h, "q": q, "sub": sub, "restart_rows": rst, "seed": 0,
               "jpeg_sha256": hashlib.sha256(blob).hexdigest(), "coef_sha256": sha(c.y_blocks, c.cb_blocks, c.cr_blocks)}
        for fast in (True, False):
            px = alloc_pixels(g.width, g.height)
            render_rows(c, qt, px, 0, g.mcu_rows, fast=fast)
            rec["rgb_fast_sha256" if fast else "rgb_direct_sha256"] = sha(px.data)
        out[name] = rec
        print(name, rec["coef_sha256"][:16], rec["rgb_fast_sha256"][:16])
    with open(os.path.join(HERE, "big_hashes.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_big_hashes.py (reference native build, oracle/_ref/patched)",
                   "cases": out}, fh, indent=1)


if __name__ == "__main__":
    main()
