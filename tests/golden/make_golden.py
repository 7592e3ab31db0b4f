"""Generate the committed golden fixtures from the REFERENCE itself.

Run in the build container only (needs /root/reference and Pillow):

    python tests/golden/make_golden.py

What it writes (tests/golden/*.npz), per case:
  jpeg   - the synthetic baseline JPEG bytes (Pillow/libjpeg-turbo encoder,
           generator = SURVEY.md Appendix B)
  y, cb, cr, q - coefficient planes (int16, natural order, MCU-ordered Y) and
           the de-zigzagged (3, 64) qtable stack, produced by the reference's
           own Huffman decoder (`entropy.decode_all`, or for 4:2:0 - which the
           reference parser rejects - the reference `decode_mcu_rows` driven
           with y_per_mcu=4 over the reference's packed scan tables)
  rgb, rgb_direct - RGB decoded by the reference's `render_rows` with
           idct fast / direct (both reference backends, asserted equal).
           For 4:2:0 these come from this repo's C oracle (the documented
           extension; the reference has no 4:2:0 path).
Plus blocks.npz: random + adversarial coefficient blocks with the reference's
single-block idct_fast / idct_direct outputs and pre-rounding float64 cores.

The reference is imported from a scratch Cython build (/tmp/refbuild, made by
oracle/build_ref.sh or `python setup.py build_ext --inplace` on a copy) when
present, else straight from /root/reference with the numpy fallback backend.
"""
from __future__ import annotations

import ctypes
import io
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
for cand in ("/tmp/refbuild/src", "/root/reference/pkg/src"):
    if os.path.isdir(cand):
        sys.path.insert(0, cand)
        break

from PIL import Image  # noqa: E402

import hetjpeg  # noqa: E402,F401
from hetjpeg import entropy, kernels, parser  # noqa: E402
from hetjpeg.block_transforms import alloc_pixels, render_rows  # noqa: E402
from hetjpeg.kernels import fallback  # noqa: E402
from hetjpeg.perf_model import _qtable_stack  # noqa: E402


def synth(w: int, h: int, seed: int = 0, sigma: float = 20.0) -> np.ndarray:
    """SURVEY.md Appendix B synthetic content (smooth waves + gaussian noise)."""
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    rgb = np.stack([128 + 100 * np.sin(xx / 37 + yy / 53),
                    128 + 90 * np.cos(xx / 23 - yy / 41),
                    128 + 80 * np.sin((xx + yy) / 61)], axis=-1)
    rgb = rgb + rng.normal(0.0, sigma, size=rgb.shape)
    return np.clip(rgb, 0, 255).astype(np.uint8)


def encode(rgb: np.ndarray, quality: int, sub: int, rst_rows: int = 0,
           rst_blocks: int = 0) -> bytes:
    buf = io.BytesIO()
    kw = {}
    if rst_rows:
        kw["restart_marker_rows"] = rst_rows
    if rst_blocks:
        kw["restart_marker_blocks"] = rst_blocks
    Image.fromarray(rgb).save(buf, "JPEG", quality=quality, subsampling=sub, **kw)
    return buf.getvalue()


def _parse_any(blob: bytes):
    """Reference parse; for 4:2:0 temporarily accept the factors so the
    reference's own table/segment parsing can be reused (geometry is then
    recomputed here for 16x16 MCUs)."""
    orig = parser._classify_subsampling
    try:
        parser._classify_subsampling = lambda comps: parser.Subsampling.S444
        return parser.parse_stream(blob)
    finally:
        parser._classify_subsampling = orig


def reference_coefficients(blob: bytes, sub: int):
    if sub in (0, 1):
        parsed = parser.parse_stream(blob)
        coeffs, _ = entropy.decode_all(parsed, blob)
        geo = coeffs.geometry
        return (parsed, coeffs.y_blocks, coeffs.cb_blocks, coeffs.cr_blocks,
                geo.mcus_per_row, geo.mcu_rows)
    parsed = _parse_any(blob)
    factors = [(c.h_sampling, c.v_sampling) for c in parsed.components]
    assert factors == [(2, 2), (1, 1), (1, 1)], factors
    mpr = -(-parsed.width // 16)
    rows = -(-parsed.height // 16)
    y = np.zeros((mpr * rows * 4, 64), np.int16)
    cb = np.zeros((mpr * rows, 64), np.int16)
    cr = np.zeros((mpr * rows, 64), np.int16)
    span = parsed.entropy_span
    data = blob[span.offset:span.offset + span.length]
    backend = kernels.active()
    scan = backend.prepare_scan(*entropy._pack_scan_tables(parsed))
    state = np.zeros(8, np.int64)
    backend.decode_mcu_rows(data, state, scan, y, cb, cr, 0, rows, mpr, 4,
                            parsed.restart_interval)
    return parsed, y, cb, cr, mpr, rows


def oracle_lib():
    path = os.path.join(REPO, "oracle", "liboracle.so")
    if not os.path.exists(path):
        os.system(f"make -C {os.path.join(REPO, 'oracle')} >/dev/null")
    return ctypes.CDLL(path)


def oracle_render(lib, y, cb, cr, q, w, h, mpr, rows, sub, fast):
    rgb = np.zeros((h, w, 3), np.uint8)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    q = np.ascontiguousarray(q, np.int32)
    lib.or_render_rows(p(y), p(cb), p(cr), p(q), p(rgb), w, h, mpr, rows, 0, rows,
                       sub, int(fast), 1)
    return rgb


CASES = [
    # name, w, h, quality, sub, rst_rows, rst_blocks, seed
    ("t1x1_444_q90", 1, 1, 90, 0, 0, 0, 1),
    ("t8x8_444_q75", 8, 8, 75, 0, 0, 0, 2),
    ("t17x9_422_q90", 17, 9, 90, 1, 0, 0, 3),
    ("t64x48_444_q75", 64, 48, 75, 0, 0, 0, 4),
    ("t200x130_422_q60_rst13", 200, 130, 60, 1, 0, 13, 5),
    ("t256x256_444_q95_rst7", 256, 256, 95, 0, 0, 7, 6),
    ("t333x211_422_q95", 333, 211, 95, 1, 0, 0, 7),
    ("t97x61_444_q100", 97, 61, 100, 0, 0, 0, 8),
    ("t1x1_420_q90", 1, 1, 90, 2, 0, 0, 11),
    ("t16x16_420_q75", 16, 16, 75, 2, 0, 0, 12),
    ("t17x9_420_q90", 17, 9, 90, 2, 0, 0, 13),
    ("t31x33_420_q50", 31, 33, 50, 2, 0, 0, 14),
    ("t64x48_420_q75", 64, 48, 75, 2, 0, 0, 15),
    ("t200x130_420_q60_rstrow1", 200, 130, 60, 2, 1, 0, 16),
    ("t333x211_420_q95", 333, 211, 95, 2, 0, 0, 17),
    ("t512x512_420_q75", 512, 512, 75, 2, 0, 0, 0),   # BASELINE config 1 (smaller noise file)
]


def make_case(lib, name, w, h, quality, sub, rst_rows, rst_blocks, seed):
    blob = encode(synth(w, h, seed), quality, sub, rst_rows, rst_blocks)
    parsed, y, cb, cr, mpr, rows = reference_coefficients(blob, sub)
    q = _qtable_stack(parsed).astype(np.int32)
    out = {"jpeg": np.frombuffer(blob, np.uint8), "y": y, "cb": cb, "cr": cr, "q": q}
    if sub in (0, 1):
        coeffs, _ = entropy.decode_all(parsed, blob)
        results = {}
        for backend in sorted(kernels.available_backends()):
            with kernels.use(backend):
                for fast in (True, False):
                    px = alloc_pixels(w, h)
                    render_rows(coeffs, q, px, 0, coeffs.geometry.mcu_rows, fast=fast)
                    results[(backend, fast)] = px.data.copy()
        for fast in (True, False):
            per = [v for (b, f), v in results.items() if f == fast]
            assert all(np.array_equal(per[0], v) for v in per), f"backends differ {name}"
        out["rgb"] = results[(sorted(kernels.available_backends())[0], True)]
        out["rgb_direct"] = results[(sorted(kernels.available_backends())[0], False)]
        # the C oracle must reproduce the reference on every 4:4:4/4:2:2 case
        for fast, key in ((True, "rgb"), (False, "rgb_direct")):
            mine = oracle_render(lib, y, cb, cr, q, w, h, mpr, rows, sub, fast)
            assert np.array_equal(mine, out[key]), f"oracle != reference on {name} fast={fast}"
    else:
        out["rgb"] = oracle_render(lib, y, cb, cr, q, w, h, mpr, rows, sub, True)
        out["rgb_direct"] = oracle_render(lib, y, cb, cr, q, w, h, mpr, rows, sub, False)
    meta = {"name": name, "width": w, "height": h, "quality": quality, "subsampling": sub,
            "restart_rows": rst_rows, "restart_blocks": rst_blocks, "seed": seed,
            "mcus_per_row": mpr, "mcu_rows": rows,
            "restart_interval": parsed.restart_interval,
            "source_rgb": "reference render_rows" if sub in (0, 1) else "oracle (4:2:0 extension)",
            "reference_backends": sorted(kernels.available_backends())}
    out["meta"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    return meta


def make_blocks(seed: int = 1234):
    """Random + adversarial dequantised blocks through the reference's
    single-block transforms (fallback.py:103-119)."""
    rng = np.random.default_rng(seed)
    n = 4000
    coef = np.zeros((n, 64), np.int32)
    dense = rng.random((n, 64)) < 0.3
    coef[dense] = rng.integers(-1024, 1024, size=dense.sum())
    coef[:, 0] = rng.integers(-2048, 2048, size=n)
    q = rng.integers(1, 256, size=(n, 64)).astype(np.int32)
    deq = coef * q
    # adversarial: saturation, extreme int16 magnitudes, DC-only, zero blocks
    deq[0] = 0
    deq[1] = 0; deq[1, 0] = 240
    deq[2] = 0; deq[2, 0] = 32767 * 255
    deq[3] = 0; deq[3, 0] = -32768 * 255
    deq[4] = rng.integers(-32768, 32768, size=64) * 255
    deq[5] = np.where(np.arange(64) % 2 == 0, 32767 * 255, -32768 * 255)
    deq[6] = 0; deq[6, 1] = 1
    deq[7] = 0; deq[7, 0] = -1028  # DC rounding tie family
    out_fast = fallback._round_u8(fallback._idct_fast_batch(deq) + 128.0).reshape(n, 64)
    out_direct = fallback._round_u8(fallback._idct_direct_batch(deq) + 128.0).reshape(n, 64)
    f64_fast = fallback._idct_fast_batch(deq[:256]).reshape(256, 64)
    f64_direct = fallback._idct_direct_batch(deq[:256]).reshape(256, 64)
    # single-block API spot checks use the reference's public functions
    for i in range(8):
        assert np.array_equal(fallback.idct_fast(deq[i]), out_fast[i])
        assert np.array_equal(fallback.idct_direct(deq[i]), out_direct[i])
    np.savez_compressed(os.path.join(HERE, "blocks.npz"), deq=deq, fast=out_fast,
                        direct=out_direct, f64_fast=f64_fast, f64_direct=f64_direct)


def main():
    lib = oracle_lib()
    manifest = {"pillow": Image.__version__, "numpy": np.__version__,
                "reference_import": hetjpeg.__file__, "cases": []}
    for case in CASES:
        manifest["cases"].append(make_case(lib, *case))
        print("wrote", case[0])
    make_blocks()
    with open(os.path.join(HERE, "MANIFEST.json"), "w") as fh:
        json.dump(manifest, fh, indent=1)
    print("done")


if __name__ == "__main__":
    main()
