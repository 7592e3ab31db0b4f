"""Build the native library in-tree: nvcc for sm_100a, no JIT, no torch.

    python -m paper_1311_5304_b200._build          # library only
    python -m paper_1311_5304_b200._build --all    # + the CPU oracle (tests only)

Output: paper_1311_5304_b200/libhetjpeg_b200.so (git-ignored, travels with
gpurun snapshots).  Rebuilds whenever the SHA-256 of the sources, headers,
flags and nvcc version differs from the one recorded next to the library
(libhetjpeg_b200.so.sha256), so a stale prebuilt binary is never reused.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libhetjpeg_b200.so")
SOURCES = ["hj_render.cu", "hj_blockops.cu", "hj_api.cu", "hj_huffman.cpp", "hj_sched.cpp", "hj_pack.cpp"]
HEADERS = ["hj_render.cuh", "hj_common.cuh", "hj_screen.h", "hj_tables.h", "hj_huffman.h", "hj_error.h",
           os.path.join("..", "..", "include", "hetjpeg_b200.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3,-ffp-contract=off", "-shared",
         "-Xptxas", "-warn-spills"]


def source_hash() -> str:
    import hashlib
    h = hashlib.sha256()
    for name in SOURCES + HEADERS:
        h.update(name.encode())
        with open(os.path.join(CSRC, name), "rb") as fh:
            h.update(fh.read())
    h.update(" ".join(ARCH + FLAGS).encode())
    try:
        h.update(subprocess.run([NVCC, "--version"], capture_output=True, text=True).stdout.encode())
    except OSError:
        pass
    return h.hexdigest()


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    try:
        with open(LIB + ".sha256") as fh:
            return fh.read().strip() != source_hash()
    except OSError:
        return True


def build_library(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    cmd = [NVCC, *ARCH, *FLAGS, "-o", LIB + ".tmp", *[os.path.join(CSRC, s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd))
    res = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    os.replace(LIB + ".tmp", LIB)
    with open(LIB + ".sha256", "w") as fh:
        fh.write(source_hash() + "\n")
    return LIB


def build_oracle() -> str:
    """The CPU oracle is test infrastructure; built here only so build() can
    prepare it next to the product."""
    res = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], capture_output=True,
                         text=True)
    if res.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{res.stdout}\n{res.stderr}")
    return os.path.join(ROOT, "oracle", "liboracle.so")


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose=True))
    if "--all" in sys.argv:
        print(build_oracle())
