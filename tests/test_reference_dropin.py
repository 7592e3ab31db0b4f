"""The drop-in claim, tested through the UNMODIFIED reference package.

The reference's own package (built from /root/reference by
oracle/build_ref.sh into oracle/_ref/shipped - git-ignored, shipped to the
GPU box with the snapshot like the product .so) is driven in a fresh
interpreter:

  1. unpatched: the reference's parser and entropy stage, then its own
     `block_transforms.render_rows(..., backend=paper_1311_5304_b200.kernels
     .cuda)` (block_transforms.py:60-75) on every 4:4:4 / 4:2:2 golden, idct
     fast and direct, against the RGB the reference's native backend makes;
  2. registered: a temporary copy of the reference with INTEGRATION.md
     section 2's patch applied to kernels/__init__.py and
     HETJPEG_BACKEND=cuda, running the reference's own `orchestrator.decode`
     in all six modes (its lanes call render_rows without a backend,
     executors.py:175-177) against the same golden RGB.

Both legs must launch this repo's render kernel (library launch counter).
"""
import json
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PKG = os.path.join(ROOT, "oracle", "_ref", "shipped", "hetjpeg")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.isdir(REF_PKG), reason="reference build (oracle/build_ref.sh) absent")]

# INTEGRATION.md section 2, as (old, new) replacements on kernels/__init__.py
PATCH = [
    ("_native = None\n_forced = os.environ.get(\"HETJPEG_BACKEND\")\nif _forced != \"fallback\":",
     "_native = None\n_cuda = None\n_forced = os.environ.get(\"HETJPEG_BACKEND\")\nif _forced == \"cuda\":\n"
     "    from paper_1311_5304_b200.kernels import cuda as _cuda   # raises if no library/GPU\n"
     "elif _forced != \"fallback\":"),
    ("_active = _native if _native is not None else fallback",
     "_active = _cuda or (_native if _native is not None else fallback)"),
    ("        out[\"native\"] = _native\n    return out",
     "        out[\"native\"] = _native\n    if _cuda is not None:\n        out[\"cuda\"] = _cuda\n    return out"),
]

SCRIPT = r"""
import json, os, sys
import numpy as np
ROOT, MODE = sys.argv[1], sys.argv[2]
import hetjpeg
from hetjpeg import block_transforms, entropy, kernels, orchestrator, parser, perf_model
from hetjpeg.executors import make_lanes
from paper_1311_5304_b200 import _lib
from paper_1311_5304_b200.kernels import cuda
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import GOLDEN_CASES
out = {"reference_file": hetjpeg.__file__, "backend": kernels.backend_name(), "cases": 0, "bad": []}
l0 = _lib.lib.hj_launch_count()
cases = [g for g in GOLDEN_CASES if g.sub in (0, 1)]
if MODE == "unpatched":
    for g in cases:
        p = parser.parse_stream(g.jpeg)
        c, _ = entropy.decode_all(p, g.jpeg)
        geo = c.geometry
        qt = perf_model._qtable_stack(p)
        for fast, want in ((True, g.rgb), (False, g.rgb_direct)):
            px = block_transforms.alloc_pixels(geo.width, geo.height)
            block_transforms.render_rows(c, qt, px, 0, geo.mcu_rows, fast=fast, backend=cuda)
            out["cases"] += 1
            if not np.array_equal(px.data, want):
                out["bad"].append([g.name, fast])
else:
    prof = perf_model.load_profile(os.path.join(ROOT, "profiles", "b200_profile.json"))
    lanes = make_lanes(host_workers=2, transfer_latency_ns=0.0, transfer_bytes_per_ns=0.0)
    try:
        for g in cases:
            p = parser.parse_stream(g.jpeg)
            for mode in orchestrator.MODES:
                for idct, want in (("fast", g.rgb), ("direct", g.rgb_direct)):
                    px, rep = orchestrator.decode(p, mode, prof, lanes, data=g.jpeg, idct=idct)
                    out["cases"] += 1
                    if not np.array_equal(px.data, want):
                        out["bad"].append([g.name, mode, idct])
    finally:
        lanes.shutdown()
out["launches"] = _lib.lib.hj_launch_count() - l0
print("RESULT " + json.dumps(out))
"""


def _run(pkg_parent, mode, env_extra):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([pkg_parent, ROOT])
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, mode], capture_output=True, text=True, env=env,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")][-1]
    return json.loads(line[7:])


def test_reference_render_rows_with_cuda_backend_argument():
    res = _run(os.path.dirname(REF_PKG), "unpatched", {})
    assert res["reference_file"].startswith(REF_PKG)
    assert res["cases"] > 0 and not res["bad"], res["bad"]
    assert res["launches"] >= res["cases"]


def test_reference_orchestrator_all_modes_on_registered_cuda_backend(tmp_path):
    dst = tmp_path / "hetjpeg"
    shutil.copytree(REF_PKG, dst)
    init = dst / "kernels" / "__init__.py"
    src = init.read_text()
    for old, new in PATCH:
        assert old in src, f"INTEGRATION.md patch no longer applies: {old!r}"
        src = src.replace(old, new)
    init.write_text(src)
    res = _run(str(tmp_path), "registered", {"HETJPEG_BACKEND": "cuda"})
    assert res["reference_file"].startswith(str(dst))
    assert res["backend"] == "cuda"
    assert res["cases"] >= 6 * 2 and not res["bad"], res["bad"]
    assert res["launches"] > 0
