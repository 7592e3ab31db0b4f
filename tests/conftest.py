import glob
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


class Golden:
    def __init__(self, path):
        z = np.load(path)
        self.meta = json.loads(bytes(z["meta"]).decode())
        self.name = self.meta["name"]
        self.jpeg = bytes(z["jpeg"])
        self.y, self.cb, self.cr, self.q = z["y"], z["cb"], z["cr"], z["q"]
        self.rgb, self.rgb_direct = z["rgb"], z["rgb_direct"]
        self.width, self.height = self.meta["width"], self.meta["height"]
        self.sub = self.meta["subsampling"]

    def __repr__(self):
        return self.name


def golden_cases():
    return [Golden(p) for p in sorted(glob.glob(os.path.join(GOLDEN, "t*.npz")))]


GOLDEN_CASES = golden_cases()


@pytest.fixture(scope="session")
def blocks_golden():
    return np.load(os.path.join(GOLDEN, "blocks.npz"))


def has_gpu() -> bool:
    try:
        from paper_1311_5304_b200 import _lib
        return _lib.lib.hj_device_count() > 0
    except Exception:
        return False


class IslowCase:
    """One libjpeg-turbo golden of the islow mode (tests/golden/make_islow_golden.py)."""

    def __init__(self, name, jpeg, sha):
        self.name, self.jpeg, self.sha = name, jpeg, sha

    def __repr__(self):
        return self.name


def islow_cases():
    z = np.load(os.path.join(GOLDEN, "islow_golden.npz"))
    return [IslowCase(k[:-5], bytes(z[k]), str(z[k[:-5] + "_sha"])) for k in sorted(z.files) if k.endswith("_jpeg")]


ISLOW_CASES = islow_cases()


def rgb_sha(rgb) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(rgb).tobytes()).hexdigest()
