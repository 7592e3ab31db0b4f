"""BASELINE-size parity against the REFERENCE's own decode (digests in
tests/golden/big_hashes.json, made by tests/golden/make_big_hashes.py with
the reference's native build): 4096x4096 4:4:4 and 4:2:2 q95 (BASELINE
configs[2]) and a 1080p 4:2:2 scan with restart intervals.

CPU: the host Huffman decoders (cursor and whole-scan, 1 and 8 threads)
reproduce the reference's coefficient planes.  GPU: the render kernel
reproduces the reference's RGB for idct fast and direct."""
import hashlib
import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

with open(os.path.join(HERE, "golden", "big_hashes.json")) as fh:
    CASES = json.load(fh)["cases"]


def _sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _jpeg(rec):
    from paper_1311_5304_b200.synth import synth_jpeg
    blob = synth_jpeg(rec["w"], rec["h"], rec["q"], rec["sub"], seed=rec["seed"], restart_rows=rec["restart_rows"])
    assert hashlib.sha256(blob).hexdigest() == rec["jpeg_sha256"], "synthetic encoder output drifted"
    return blob


@pytest.mark.parametrize("name", sorted(CASES))
def test_host_huffman_matches_reference_at_baseline_size(name):
    from paper_1311_5304_b200 import entropy, parser
    rec = CASES[name]
    blob = _jpeg(rec)
    p = parser.parse_stream(blob)
    c, _ = entropy.decode_all(p, blob)
    assert _sha(c.y_blocks, c.cb_blocks, c.cr_blocks) == rec["coef_sha256"]
    fs = entropy.FastScan(p)
    for threads in (1, 8):
        o = fs.decode(blob, threads=threads)
        assert _sha(o.y_blocks, o.cb_blocks, o.cr_blocks) == rec["coef_sha256"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_render_matches_reference_at_baseline_size(name):
    from paper_1311_5304_b200 import _lib, entropy, parser
    from paper_1311_5304_b200.block_transforms import alloc_pixels, render_rows
    from paper_1311_5304_b200.perf_model import qtable_stack
    _lib.require_device()
    rec = CASES[name]
    blob = _jpeg(rec)
    p = parser.parse_stream(blob)
    c = entropy.FastScan(p).decode(blob, threads=8)
    q = qtable_stack(p)
    for fast, key in ((True, "rgb_fast_sha256"), (False, "rgb_direct_sha256")):
        px = alloc_pixels(p.width, p.height)
        render_rows(c, q, px, 0, c.geometry.mcu_rows, fast=fast)
        assert _sha(px.data) == rec[key], key
