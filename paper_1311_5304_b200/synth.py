"""Deterministic synthetic baseline JPEGs (SURVEY.md Appendix B generator),
for profiling, benchmarks and tests.  Needs Pillow (libjpeg-turbo encoder);
there are no datasets on the GPU boxes.
"""
from __future__ import annotations

import io

import numpy as np

SUBSAMPLING = {"444": 0, "422": 1, "420": 2}


def synth_rgb(width: int, height: int, seed: int = 0, sigma: float = 20.0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:height, 0:width].astype(np.float32)
    rgb = np.stack([128 + 100 * np.sin(xx / 37 + yy / 53),
                    128 + 90 * np.cos(xx / 23 - yy / 41),
                    128 + 80 * np.sin((xx + yy) / 61)], axis=-1)
    rgb += rng.normal(0.0, sigma, size=rgb.shape).astype(np.float32)
    return np.clip(rgb, 0, 255).astype(np.uint8)


def synth_jpeg(width: int, height: int, quality: int = 90, subsampling: str = "420",
               seed: int = 0, restart_rows: int = 0, restart_blocks: int = 0,
               sigma: float = 20.0) -> bytes:
    from PIL import Image
    kw = {}
    if restart_rows:
        kw["restart_marker_rows"] = restart_rows
    if restart_blocks:
        kw["restart_marker_blocks"] = restart_blocks
    buf = io.BytesIO()
    Image.fromarray(synth_rgb(width, height, seed, sigma)).save(
        buf, "JPEG", quality=quality, subsampling=SUBSAMPLING[subsampling], **kw)
    return buf.getvalue()
