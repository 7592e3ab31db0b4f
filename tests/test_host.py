"""Host-side logic on the CPU: the C ABI exports, the parser (incl. the 4:2:0
extension), and the native C++ Huffman decoder against the reference's own
coefficients (golden fixtures).  No GPU calls."""
import os
import re

import numpy as np
import pytest

from conftest import GOLDEN_CASES, ROOT, has_gpu
from paper_1311_5304_b200 import _lib, entropy, errors, parser
from paper_1311_5304_b200.kernels import cuda


def test_library_exports_every_header_symbol():
    header = open(os.path.join(ROOT, "include", "hetjpeg_b200.h")).read()
    header = re.sub(r"/\*.*?\*/", "", header, flags=re.S)
    declared = set(re.findall(r"\b(hj_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations found"
    for name in declared:
        assert hasattr(_lib.lib, name), f"{name} not exported"
    assert declared <= set(_lib.EXPORTED) | {"hj_version"}, declared - set(_lib.EXPORTED)


def test_compiled_for_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          os.path.join(ROOT, "paper_1311_5304_b200", "libhetjpeg_b200.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


@pytest.mark.parametrize("g", GOLDEN_CASES, ids=repr)
def test_parse_geometry(g):
    p = parser.parse_stream(g.jpeg)
    geo = parser.geometry_of(p)
    assert (geo.width, geo.height) == (g.width, g.height)
    assert geo.mcus_per_row == g.meta["mcus_per_row"]
    assert geo.mcu_rows == g.meta["mcu_rows"]
    assert p.restart_interval == g.meta["restart_interval"]
    assert p.subsampling is [parser.Subsampling.S444, parser.Subsampling.S422,
                             parser.Subsampling.S420][g.sub]
    # header round trip (SPEC parser invariant)
    sp = p.entropy_span
    blob = parser.serialize_headers(p) + g.jpeg[sp.offset:sp.offset + sp.length] + b"\xff\xd9"
    p2 = parser.parse_stream(blob)
    assert (p2.width, p2.height, p2.components, p2.quant_tables, p2.huffman_specs,
            p2.restart_interval) == (p.width, p.height, p.components, p.quant_tables,
                                     p.huffman_specs, p.restart_interval)


@pytest.mark.parametrize("g", GOLDEN_CASES, ids=repr)
def test_native_huffman_matches_reference_coefficients(g):
    p = parser.parse_stream(g.jpeg)
    coeffs, cur = entropy.decode_all(p, g.jpeg)
    assert np.array_equal(coeffs.y_blocks, g.y)
    assert np.array_equal(coeffs.cb_blocks, g.cb)
    assert np.array_equal(coeffs.cr_blocks, g.cr)
    assert cur.rows_decoded == parser.geometry_of(p).mcu_rows


@pytest.mark.parametrize("g", [c for c in GOLDEN_CASES if c.meta["mcu_rows"] > 2], ids=repr)
def test_chunked_decode_is_deterministic(g):
    # SPEC entropy invariant: R rows in one call == R calls of 1 row; pinned buffers too
    p = parser.parse_stream(g.jpeg)
    geo = parser.geometry_of(p)
    cur = entropy.new_cursor(p, g.jpeg)
    buf = entropy.alloc_coefficients(geo, pinned=has_gpu())
    entropy.decode_rows(cur, p, buf, 2)
    entropy.decode_rows(cur, p, buf, geo.mcu_rows - 2, record_rows=True)
    assert np.array_equal(buf.y_blocks, g.y) and np.array_equal(buf.cr_blocks, g.cr)
    assert len(cur.row_times_ns) == geo.mcu_rows
    with pytest.raises(ValueError):
        entropy.decode_rows(cur, p, buf, 1)


def test_truncated_scan_raises_and_writes_state_back():
    g = GOLDEN_CASES[-1]
    p = parser.parse_stream(g.jpeg)
    sp = p.entropy_span
    data = g.jpeg[sp.offset:sp.offset + sp.length // 3]
    geo = parser.geometry_of(p)
    buf = entropy.alloc_coefficients(geo)
    scan = cuda.prepare_scan(*entropy._pack_scan_tables(p))
    state = np.zeros(8, np.int64)
    with pytest.raises(errors.BitstreamExhausted):
        cuda.decode_mcu_rows(data, state, scan, buf.y_blocks, buf.cb_blocks, buf.cr_blocks, 0,
                             geo.mcu_rows, geo.mcus_per_row, geo.y_blocks_per_mcu, 0)
    assert 0 < state[0] <= len(data)


def test_restart_out_of_sequence_raises():
    g = next(c for c in GOLDEN_CASES if c.meta["restart_interval"])
    p = parser.parse_stream(g.jpeg)
    sp = p.entropy_span
    data = bytearray(g.jpeg[sp.offset:sp.offset + sp.length])
    i = next(k for k in range(len(data) - 1) if data[k] == 0xFF and 0xD0 <= data[k + 1] <= 0xD7)
    data[i + 1] = 0xD5
    geo = parser.geometry_of(p)
    buf = entropy.alloc_coefficients(geo)
    scan = cuda.prepare_scan(*entropy._pack_scan_tables(p))
    with pytest.raises(errors.MarkerInScan):
        cuda.decode_mcu_rows(bytes(data), np.zeros(8, np.int64), scan, buf.y_blocks,
                             buf.cb_blocks, buf.cr_blocks, 0, geo.mcu_rows, geo.mcus_per_row,
                             geo.y_blocks_per_mcu, p.restart_interval)


def test_parser_rejections():
    g = GOLDEN_CASES[0]
    with pytest.raises(errors.MissingMarker):
        parser.parse_stream(b"\x00\x00")
    with pytest.raises(errors.CorruptSegment):
        parser.parse_stream(g.jpeg[: len(g.jpeg) // 2])
    sof2 = bytearray(g.jpeg)
    k = sof2.find(b"\xff\xc0")
    sof2[k + 1] = 0xC2
    with pytest.raises(errors.UnsupportedFeature):
        parser.parse_stream(bytes(sof2))


def test_huffman_table_spec_examples():
    # SPEC.md build_huffman_table examples
    t = parser.build_huffman_table(parser.HuffmanSpec(parser.TableClass.DC, 0,
                                                      (1, 1) + (0,) * 14, (7, 9)))
    assert t.decode_map == {(0, 1): 7, (2, 2): 9}
    with pytest.raises(errors.InvalidTable):
        parser.build_huffman_table(parser.HuffmanSpec(parser.TableClass.DC, 0,
                                                      (3,) + (0,) * 15, (1, 2, 3)))


def test_zigzag_and_dezigzag():
    assert entropy.ZIGZAG[1] == 1 and entropy.ZIGZAG[2] == 8
    blk = np.arange(64)
    nat = entropy.dezigzag(blk)
    assert nat[1] == 1 and nat[8] == 2


def test_entropy_end_scan_matches_python_walk():
    for g in GOLDEN_CASES[:6]:
        p = parser.parse_stream(g.jpeg)
        start = p.entropy_span.offset
        pos, n = start, len(g.jpeg)
        while pos < n - 1:  # parser.py:277-293 restated
            if g.jpeg[pos] != 0xFF:
                pos += 1
                continue
            nxt = g.jpeg[pos + 1]
            if nxt == 0 or 0xD0 <= nxt <= 0xD7:
                pos += 2
                continue
            if nxt == 0xFF:
                pos += 1
                continue
            break
        assert parser.scan_entropy_end(g.jpeg, start) == pos


@pytest.mark.parametrize("g", GOLDEN_CASES, ids=repr)
@pytest.mark.parametrize("threads", [1, 4])
def test_fast_scan_decoder_matches_reference(g, threads):
    p = parser.parse_stream(g.jpeg)
    out = entropy.FastScan(p).decode(g.jpeg, threads=threads)
    assert np.array_equal(out.y_blocks, g.y)
    assert np.array_equal(out.cb_blocks, g.cb)
    assert np.array_equal(out.cr_blocks, g.cr)


def test_fast_scan_decoder_truncated_raises():
    g = GOLDEN_CASES[-1]
    p = parser.parse_stream(g.jpeg)
    sp = p.entropy_span
    cut = g.jpeg[:sp.offset + sp.length // 2] + b"\xff\xd9"
    with pytest.raises(errors.BitstreamExhausted):
        entropy.FastScan(p).decode(cut)
