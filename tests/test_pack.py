"""Packed coefficient transfer (csrc/hj_pack.{h,cpp}): the
host packer (AVX-512 VBMI2 path where the CPU has it, else scalar) and its
reference unpacker are lossless on every int16 input - sparse and dense
blocks, int8-range and wide values, the int16 extremes.  CPU only; the device
expansion is covered by the GPU parity suite, which runs the drop-in through it."""
import ctypes as C

import numpy as np
import pytest

from paper_1311_5304_b200 import _lib


def _roundtrip(blocks):
    n = blocks.shape[0]
    src = np.ascontiguousarray(blocks, np.int16)
    mask = np.zeros(n, np.uint64)
    off = np.zeros(n, np.uint32)
    dc = np.zeros(n, np.int16)
    vals = np.zeros(130 * n + 128, np.uint8)
    nb = _lib.lib.hj_pack_blocks(src.ctypes.data, n, mask.ctypes.data, off.ctypes.data, dc.ctypes.data,
                                 vals.ctypes.data)
    assert nb >= 0
    out = np.full_like(src, 12345)
    assert _lib.lib.hj_unpack_blocks_host(mask.ctypes.data, off.ctypes.data, dc.ctypes.data, vals.ctypes.data,
                                          n, out.ctypes.data) == 0
    assert np.array_equal(out, src)
    # the masks are the nonzero AC sets, the DC travels as int16
    want = (src != 0)
    want[:, 0] = False
    got = ((mask[:, None] >> np.arange(64, dtype=np.uint64)) & np.uint64(1)).astype(bool)
    assert np.array_equal(got, want)
    assert np.array_equal(dc, src[:, 0] if n else dc)
    wide = (off >> 31).astype(bool)
    assert np.array_equal(wide, ((src[:, 1:] < -128) | (src[:, 1:] > 127)).any(1))
    return nb


@pytest.mark.parametrize("seed", range(4))
def test_pack_roundtrip_random(seed):
    rng = np.random.default_rng(seed)
    n = 777
    b = np.zeros((n, 64), np.int16)
    nnz = rng.integers(0, 65, n)
    for i in range(n):
        pos = rng.choice(64, nnz[i], replace=False)
        scale = [4, 127, 2000, 32767][i % 4]
        b[i, pos] = rng.integers(-scale, scale + 1, nnz[i])
    _roundtrip(b)


def test_pack_edge_values_and_sizes():
    ext = np.array([-32768, 32767, -129, 128, -128, 127, -1, 1, 0], np.int16)
    b = np.zeros((40, 64), np.int16)
    for i in range(40):
        b[i, :] = np.roll(np.resize(ext, 64), i)
    b[3] = 0
    b[7] = -32768
    _roundtrip(b)
    _roundtrip(np.zeros((1, 64), np.int16))
    _roundtrip(np.zeros((0, 64), np.int16))


def test_pack_size_on_a_q90_image():
    from paper_1311_5304_b200 import entropy, parser
    from paper_1311_5304_b200.synth import synth_jpeg
    blob = synth_jpeg(320, 240, 90, "420", seed=1)
    p = parser.parse_stream(blob)
    co, _ = entropy.decode_all(p, blob)
    y = np.asarray(co.y_blocks).reshape(-1, 64)
    nb = _roundtrip(y)
    assert 14 * len(y) + nb < 0.5 * 128 * len(y)  # well under half the dense bytes


def test_scalar_path_matches():
    """The portable packer (hosts without AVX-512 VBMI2) produces the same bytes."""
    import os
    import subprocess
    import sys
    code = ("import numpy as np, sys; sys.path[:0] = ['.', 'tests']; from test_pack import _roundtrip;"
            "rng = np.random.default_rng(9); b = rng.integers(-300, 300, (300, 64)).astype(np.int16);"
            "b[rng.random((300, 64)) < 0.7] = 0; b[::3, 1:] = np.clip(b[::3, 1:], -128, 127); _roundtrip(b); print('ok')")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, HJ_PACK_SCALAR="1"),
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
