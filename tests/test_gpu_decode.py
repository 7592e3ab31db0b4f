"""End-to-end decode on the B200: every orchestrator mode (orchestrator.py:87-145
of the reference) and the pipelined batch decoder must reproduce the
reference's RGB bit-exactly."""
import numpy as np
import pytest

from conftest import GOLDEN_CASES, has_gpu
from paper_1311_5304_b200 import executors, orchestrator, parser, perf_model
from paper_1311_5304_b200.pipeline import BatchDecoder

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


def _profile(chunk_rows):
    # B200-shaped: accelerator cheaper than the host lane per pixel, small
    # dispatch cost; degree-2 bivariate basis 1, w, w^2, h, w*h, h^2
    return perf_model.DeviceProfile(
        p_cpu=perf_model.PolyModel(2, 2, [5e4, 0, 0, 0, 4.0, 0]),
        p_gpu=perf_model.PolyModel(2, 2, [3e4, 0, 0, 0, 0.5, 0]),
        t_disp=perf_model.PolyModel(2, 2, [1e4, 0, 0, 0, 0, 0]),
        t_huff_per_pixel=perf_model.PolyModel(1, 1, [2.0, 10.0]), chunk_rows=chunk_rows)


@pytest.fixture(scope="module")
def lanes():
    lp = executors.make_lanes(host_workers=4)
    yield lp
    lp.shutdown()


@pytest.mark.parametrize("case", GOLDEN_CASES, ids=repr)
@pytest.mark.parametrize("mode", orchestrator.MODES)
def test_modes_bit_exact(case, mode, lanes):
    p = parser.parse_stream(case.jpeg)
    geo = parser.geometry_of(p)
    prof = _profile(chunk_rows=geo.mcu_height * 2)
    px, rep = orchestrator.decode(p, mode, prof, lanes, data=case.jpeg)
    assert np.array_equal(px.data, case.rgb), f"{mode} differs from the reference"
    assert rep.wall_ns > 0 and rep.huffman_ns > 0
    if mode in ("accel", "accel-pipe", "sps", "pps") and rep.accel_busy_ns:
        assert rep.accel_busy_ns >= rep.accel_compute_ns >= 0


@pytest.mark.parametrize("case", [c for c in GOLDEN_CASES if c.height > 64], ids=repr)
def test_direct_idct_and_pps_without_repartition(case, lanes):
    p = parser.parse_stream(case.jpeg)
    px, _ = orchestrator.decode(p, "accel-pipe", None, lanes, data=case.jpeg, idct="direct", chunk_mcu_rows=1)
    assert np.array_equal(px.data, case.rgb_direct)
    px, rep = orchestrator.decode(p, "pps", _profile(16), lanes, data=case.jpeg, enable_repartition=False)
    assert np.array_equal(px.data, case.rgb) and not rep.repartitioned


def test_pps_plan_partitions_rows(lanes):
    case = max(GOLDEN_CASES, key=lambda c: c.width * c.height)
    p = parser.parse_stream(case.jpeg)
    geo = parser.geometry_of(p)
    # a host lane as cheap as the accelerator: the plan must split the rows
    prof = perf_model.DeviceProfile(
        p_cpu=perf_model.PolyModel(2, 2, [0, 0, 0, 0, 1.0, 0]),
        p_gpu=perf_model.PolyModel(2, 2, [0, 0, 0, 0, 1.0, 0]),
        t_disp=perf_model.PolyModel(2, 2, [0, 0, 0, 0, 0, 0]),
        t_huff_per_pixel=perf_model.PolyModel(1, 1, [1.0, 1.0]), chunk_rows=geo.mcu_height * 4)
    px, rep = orchestrator.decode(p, "sps", prof, lanes, data=case.jpeg)
    assert 0 < rep.plan.accel_mcu_rows < geo.mcu_rows
    assert np.array_equal(px.data, case.rgb)
    px, rep = orchestrator.decode(p, "pps", prof, lanes, data=case.jpeg)
    assert np.array_equal(px.data, case.rgb)
    assert len(rep.chunks) >= 1


def test_batch_decoder_pipelined_matches_reference():
    cases = GOLDEN_CASES
    dec = BatchDecoder([c.jpeg for c in cases], threads=4, n_streams=3)
    try:
        t_h = dec.huffman_only()
        io = dec.run()
        for c, px in zip(cases, dec.pixels):
            assert np.array_equal(px.data, c.rgb), c.name
        assert t_h > 0 and io["wall_s"] > 0
        assert io["d2h_bytes"] == sum(c.width * c.height * 3 for c in cases)
        # the Python-thread form of the same pipeline agrees (and repeated
        # native runs over the same buffers stay exact)
        for px in dec.pixels:
            px.data[...] = 0
        dec.run_threads()
        assert all(np.array_equal(px.data, c.rgb) for c, px in zip(cases, dec.pixels))
        for px in dec.pixels:
            px.data[...] = 0
        dec.run()
        assert all(np.array_equal(px.data, c.rgb) for c, px in zip(cases, dec.pixels))
        assert dec.huffman_only_threads() > 0
    finally:
        dec.close()


def test_batch_decoder_reports_a_truncated_scan():
    """A scan cut short by an EOI in the middle of the entropy data: the
    native pipeline's Huffman workers stop and the error surfaces as one of
    the reference's exceptions (BitstreamExhausted / BadCode); a batch of
    intact images afterwards decodes exactly."""
    from paper_1311_5304_b200.errors import HetJpegError
    good = max(GOLDEN_CASES, key=lambda c: c.width * c.height)
    p = parser.parse_stream(good.jpeg)
    sp = p.entropy_span
    cut = good.jpeg[:sp.offset + sp.length // 2] + b"\xff\xd9"
    dec = BatchDecoder([good.jpeg, cut], threads=2, n_streams=2)
    try:
        with pytest.raises(HetJpegError):
            dec.run()
        with pytest.raises(HetJpegError):
            dec.huffman_only()
    finally:
        dec.close()
    dec = BatchDecoder([good.jpeg], threads=1)
    try:
        dec.run()
        assert np.array_equal(dec.pixels[0].data, good.rgb)
    finally:
        dec.close()
