"""Pins the 4:2:0 extension's h2v2 fancy upsampler to libjpeg-turbo.

Run in the build container only (Pillow with its bundled libjpeg-turbo, and
the reference build in oracle/_ref for its float64 colour conversion):

    python tests/golden/make_h2v2_pin.py

The reference rejects 4:2:0 (parser.py:223-229), so the repo's 4:2:0 path
 has no reference RGB.  Its h2v2 rule is libjpeg's
h2v2_fancy_upsample (jdsample.c: colsum = 3*near + far, (3*cs + prev + 8)
>> 4, (3*cs + next + 7) >> 4, edges replicated).  This script pins it to
the real libjpeg-turbo on inputs where every other stage provably agrees:

  * images of constant 16x16 tiles, w and h multiples of 16: every 8x8
    block of every plane is DC-only, where the reference's float64 IDCT and
    libjpeg's islow IDCT are both exactly clamp((c*q + 1028) >> 3)
    (SURVEY.md E5), and the padded chroma plane equals libjpeg's
    downsampled_width x downsampled_height plane (same edge replication);
  * Pillow decodes with fancy upsampling but WITHOUT colour conversion
    (draft("YCbCr")), giving libjpeg-turbo's upsampled Y/Cb/Cr planes;
  * those planes go through the reference's own float64 colour conversion
    (kernels/fallback.py:142-150).

The result is the RGB the reference would produce if it accepted 4:2:0 with
libjpeg's upsampler.  tests/golden/h2v2_pin.npz holds, per case, the JPEG and
that RGB; tests check the oracle (CPU) and the render kernel (GPU) against it.
"""
import io
import os
import sys

import numpy as np
from PIL import Image, features

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(REPO, "oracle", "_ref", "patched"))

from hetjpeg.kernels import fallback  # noqa: E402

CASES = [(16, 16, 75), (64, 48, 90), (160, 96, 50), (256, 256, 95), (512, 512, 75), (1920, 1088, 90)]


def main():
    rng = np.random.default_rng(4202)
    out = {"libjpeg": np.array(f"libjpeg-turbo {features.version('libjpeg_turbo')} (Pillow "
                               f"{Image.__version__ if hasattr(Image, '__version__') else ''})")}
    for k, (w, h, q) in enumerate(CASES):
        tiles = rng.integers(0, 256, size=(h // 16, w // 16, 3)).astype(np.uint8)
        tiles[rng.random(tiles.shape) < 0.15] = 0      # saturating colours
        tiles[rng.random(tiles.shape) < 0.15] = 255
        rgb = np.repeat(np.repeat(tiles, 16, 0), 16, 1)
        buf = io.BytesIO()
        Image.fromarray(rgb).save(buf, "JPEG", quality=q, subsampling=2)
        blob = buf.getvalue()
        im = Image.open(io.BytesIO(blob))
        im.draft("YCbCr", None)  # libjpeg output colour space YCbCr: upsampled, not converted
        assert im.mode == "YCbCr"
        ycc = np.asarray(im)
        r, g, b = fallback.ycbcr_to_rgb(ycc[..., 0], ycc[..., 1], ycc[..., 2])
        name = f"c{k}_{w}x{h}_q{q}"
        out[name + "_jpeg"] = np.frombuffer(blob, np.uint8)
        out[name + "_rgb"] = np.stack([r, g, b], -1).astype(np.uint8)
    np.savez_compressed(os.path.join(HERE, "h2v2_pin.npz"), **out)
    print("wrote", len(CASES), "cases;", out["libjpeg"])


if __name__ == "__main__":
    main()
