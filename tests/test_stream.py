"""Bounded-memory streaming decode (hj_stream_run / pipeline.StreamDecoder,
BASELINE config 5) and restart-interval shard decoding (hj_decode_scan_rows,
config 4).  CPU: the host stage; GPU: bit-exact RGB out of the ring."""
import numpy as np
import pytest

from conftest import has_gpu
from oracle import oracle


def _rst_jpeg(w=640, h=480, sub="420", q=85, rows=1, seed=3):
    from paper_1311_5304_b200.synth import synth_jpeg
    return synth_jpeg(w, h, q, sub, seed=seed, restart_rows=rows)


@pytest.mark.parametrize("sub", ["444", "422", "420"])
def test_scan_rows_decodes_only_the_covering_intervals(sub):
    from paper_1311_5304_b200 import entropy, parser
    blob = _rst_jpeg(sub=sub)
    p = parser.parse_stream(blob)
    full, _ = entropy.decode_all(p, blob)
    fs = entropy.FastScan(p)
    g = fs.geometry
    rng = np.random.default_rng(0)
    for _ in range(12):
        r0 = int(rng.integers(0, g.mcu_rows))
        n = int(rng.integers(1, g.mcu_rows - r0 + 1))
        out = entropy.alloc_coefficients(g)
        out.y_blocks[...] = 7777
        out.cb_blocks[...] = 7777
        fs.decode_rows(r0, n, blob, out=out, threads=3)
        ypr = g.mcus_per_row * g.y_blocks_per_mcu
        assert np.array_equal(out.y_blocks[r0 * ypr:(r0 + n) * ypr], full.y_blocks[r0 * ypr:(r0 + n) * ypr])
        cpr = g.mcus_per_row
        assert np.array_equal(out.cb_blocks[r0 * cpr:(r0 + n) * cpr], full.cb_blocks[r0 * cpr:(r0 + n) * cpr])
        # one interval = one MCU row here: nothing outside the range was decoded
        assert (out.y_blocks[:r0 * ypr] == 7777).all() and (out.cb_blocks[(r0 + n) * cpr:] == 7777).all()


def test_scan_rows_without_restarts_decodes_the_whole_scan():
    from paper_1311_5304_b200 import entropy, parser
    blob = _rst_jpeg(rows=0)
    p = parser.parse_stream(blob)
    full, _ = entropy.decode_all(p, blob)
    out = entropy.FastScan(p).decode_rows(5, 3, blob)
    assert np.array_equal(out.y_blocks, full.y_blocks)


def test_stream_host_stage_counts_and_bounded_ring():
    from paper_1311_5304_b200 import pipeline
    from paper_1311_5304_b200.synth import synth_jpeg
    blobs = [synth_jpeg(w, h, q, s, seed=k) for k, (w, h, q, s) in
             enumerate([(640, 480, 90, "420"), (333, 211, 60, "422"), (96, 64, 95, "444"), (1024, 768, 75, "420")])]
    corpus = [blobs[k % 4] for k in range(200)]
    sd = pipeline.StreamDecoder(corpus, threads=4, slots=3)
    st = sd.huffman_only()
    assert st["images"] == 200
    # the ring is 3 slots of the largest image, whatever the corpus length
    biggest = max((g.mcus_per_row * g.mcu_rows * (g.y_blocks_per_mcu + 2) * 128) for g in sd.geometries)
    assert st["pinned_bytes"] == 3 * biggest


@pytest.mark.gpu
def test_stream_gpu_bit_exact_and_shards():
    if not has_gpu():
        pytest.fail("needs a GPU")
    from paper_1311_5304_b200 import entropy, parser, pipeline
    from paper_1311_5304_b200.perf_model import qtable_stack
    from paper_1311_5304_b200.synth import synth_jpeg
    spec = [(640, 480, 90, "420", 1), (333, 211, 60, "422", 0), (96, 64, 95, "444", 2), (1024, 768, 75, "420", 0),
            (17, 9, 80, "420", 0)]
    blobs = [synth_jpeg(w, h, q, s, seed=k, restart_rows=r) for k, (w, h, q, s, r) in enumerate(spec)]
    corpus = [blobs[k % len(blobs)] for k in range(60)]
    keep = (0, 1, 2, 3, 4, 57)
    sd = pipeline.StreamDecoder(corpus, threads=4, slots=5, keep=keep)
    st = sd.run()
    assert st["images"] == 60 and st["launches"] >= 60
    for i in keep:
        b = corpus[i]
        p = parser.parse_stream(b)
        c, _ = entropy.decode_all(p, b)
        g = c.geometry
        sub = {8: 0}.get(g.mcu_width, 1 if g.mcu_height == 8 else 2)
        want = oracle.render(c.y_blocks, c.cb_blocks, c.cr_blocks, qtable_stack(p), g.width, g.height, sub)
        assert np.array_equal(sd.rgb(i), want), i
    # MCU-row shards of the RST image: every shard's rows bit-exact
    b = blobs[0]
    p = parser.parse_stream(b)
    c, _ = entropy.decode_all(p, b)
    g = c.geometry
    want = oracle.render(c.y_blocks, c.cb_blocks, c.cr_blocks, qtable_stack(p), g.width, g.height, 2)
    cuts = [0, 3, 11, 12, g.mcu_rows]
    shards = [(a, z - a) for a, z in zip(cuts, cuts[1:])]
    sd = pipeline.StreamDecoder([b] * len(shards), threads=3, slots=2, keep=tuple(range(len(shards))),
                                shards=shards)
    sd.run()
    for k, (r0, n) in enumerate(shards):
        y0, y1 = r0 * 16, min(g.height, (r0 + n) * 16)
        assert np.array_equal(sd.rgb(k)[y0:y1], want[y0:y1]), (r0, n)


def test_stream_reports_the_first_failing_image():
    from paper_1311_5304_b200 import errors, parser, pipeline
    from paper_1311_5304_b200.synth import synth_jpeg
    good = synth_jpeg(200, 120, 80, "422", seed=1)
    p = parser.parse_stream(good)
    sp = p.entropy_span
    bad = bytearray(good)
    # scramble the middle of the scan: a Huffman error or an early stop
    mid = sp.offset + sp.length // 2
    bad[mid:mid + 40] = bytes([0xFF, 0xD9]) * 20
    bad = bytes(bad)
    sd = pipeline.StreamDecoder([good, good, bad, good], threads=2, slots=2, order=[0, 1, 2, 3])
    with pytest.raises((errors.BitstreamExhausted, errors.BadCode, errors.MarkerInScan)) as ei:
        sd.huffman_only()
    assert "image 2" in str(ei.value)
