"""Kernel-backend registry, API of the reference's `hetjpeg.kernels`
(pkg/src/hetjpeg/kernels/__init__.py:17-60): `active()`, `backend_name()`,
`available_backends()`, `use(name)`.

There is exactly one backend here, `cuda` (kernels/cuda.py): the sm_100a
parallel phase plus the native host Huffman decoder.  Unlike the reference
there is no silent numpy fallback - importing this package fails if the
native library is missing, and `HETJPEG_BACKEND` may only name `cuda`.
A reference installation selects the same module by adding it to its own
registry.
"""
from __future__ import annotations

import contextlib
import os
import threading

from . import cuda

_BACKENDS = {"cuda": cuda}
_requested = os.environ.get("HETJPEG_BACKEND")
if _requested not in (None, "", "cuda"):
    raise ImportError(f"HETJPEG_BACKEND={_requested!r}: this package provides only the "
                      "'cuda' backend (there is no CPU fallback)")

_active = cuda
_lock = threading.Lock()


def active():
    return _active


def backend_name() -> str:
    return _active.NAME


def available_backends() -> dict:
    return dict(_BACKENDS)


@contextlib.contextmanager
def use(name: str):
    """Temporarily select a backend by name (thread-safe swap)."""
    global _active
    if name not in _BACKENDS:
        raise ValueError(f"backend {name!r} not available (have {sorted(_BACKENDS)})")
    with _lock:
        previous, _active = _active, _BACKENDS[name]
    try:
        yield _active
    finally:
        with _lock:
            _active = previous
