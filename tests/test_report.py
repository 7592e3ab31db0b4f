"""Output formats (report.py) against the reference's cli.py: P6 PPM bytes, the
bench CSV columns and the per-mode summary line.  CPU tests drive the bench
loop through lanes with a render hook that writes the oracle's pixels; the
GPU test runs the real lanes and checks the PPM payload against the
reference's RGB."""
import csv

import numpy as np
import pytest

from conftest import GOLDEN_CASES, has_gpu
from paper_1311_5304_b200 import executors, perf_model, report
from paper_1311_5304_b200.block_transforms import PixelBuffer


def test_ppm_format_matches_reference_writer(tmp_path):
    rgb = np.arange(5 * 3 * 3, dtype=np.uint8).reshape(3, 5, 3)
    px = PixelBuffer(5, 3, rgb)
    path = tmp_path / "x.ppm"
    report.write_ppm(px, path)
    blob = path.read_bytes()
    assert blob == b"P6\n5 3\n255\n" + rgb.tobytes()      # cli.py:21-25
    assert report.read_ppm(path) == (5, 3, rgb.tobytes())
    assert report.read_ppm(blob) == (5, 3, rgb.tobytes())
    with pytest.raises(ValueError):
        report.read_ppm(b"P5\n1 1\n255\n\x00")
    with pytest.raises(ValueError):
        report.read_ppm(b"P6\n2 2\n255\n\x00")


def test_csv_header_is_the_reference_one():
    assert report.CSV_HEADER == ["image", "w", "h", "d", "mode", "wall_ns", "huff_ns", "par_ns",
                                 "x_rows", "chunks", "amdahl_bound"]


def _fake_lanes():
    # render hook: no device on the CPU runner; the bench loop only needs the
    # lanes to complete (pixels are not checked here)
    return executors.make_lanes(host_workers=2, render=lambda item: None)


def _profile():
    return perf_model.DeviceProfile(
        p_cpu=perf_model.PolyModel(2, 2, [5e4, 0, 0, 0, 4.0, 0]),
        p_gpu=perf_model.PolyModel(2, 2, [3e4, 0, 0, 0, 0.5, 0]),
        t_disp=perf_model.PolyModel(2, 2, [1e4, 0, 0, 0, 0, 0]),
        t_huff_per_pixel=perf_model.PolyModel(1, 1, [2.0, 10.0]), chunk_rows=16)


def test_bench_loop_rows_and_summary(tmp_path, monkeypatch):
    from paper_1311_5304_b200 import entropy
    alloc = entropy.alloc_coefficients
    # page-locked buffers need a CUDA driver; the CPU runner uses pageable ones
    monkeypatch.setattr(entropy, "alloc_coefficients", lambda geo, pinned=False: alloc(geo, pinned=False))
    cases = [c for c in GOLDEN_CASES if c.height >= 16][:3]
    images = [(f"{i}.jpg", c.jpeg) for i, c in enumerate(cases)]
    images.append(("broken.jpg", b"\xff\xd8\xff\xd9"))
    errs = []
    with _fake_lanes() as lanes:
        res = report.bench_corpus(images, ["accel", "pps"], _profile(), lanes, reference="par", errors=errs)
    assert res.failed == 1 and errs and errs[0].startswith("error: broken.jpg")
    assert len(res.rows) == 2 * len(cases)
    for row, (name, _) in zip(res.rows[::2], images):
        assert row[0] == name and row[4] == "accel" and row[8] == -1 and row[9] == 1
        assert float(row[10]) >= 1.0 and int(row[6]) > 0
    pps_rows = res.rows[1::2]
    assert all(r[4] == "pps" and r[8] >= 0 for r in pps_rows)
    lines = res.summary_lines("par")
    assert len(lines) == 2 and lines[0].startswith(f"mode=accel images={len(cases)} mean_speedup_vs_par=")
    assert "cov_pct=" in lines[1]
    path = tmp_path / "bench.csv"
    res.write_csv(path)
    got = list(csv.reader(open(path)))
    assert got[0] == report.CSV_HEADER and len(got) == 1 + len(res.rows)


def test_bench_loop_usage_errors():
    with pytest.raises(ValueError):
        report.bench_corpus([], ["bogus"], None, None)
    with pytest.raises(ValueError):
        report.bench_corpus([], ["pps"], None, None)


@pytest.mark.gpu
@pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")
def test_bench_loop_and_ppm_on_device(tmp_path):
    from paper_1311_5304_b200 import orchestrator, parser
    case = max(GOLDEN_CASES, key=lambda c: c.width * c.height)
    with executors.make_lanes(host_workers=4) as lanes:
        res = report.bench_corpus([("a.jpg", case.jpeg)], ["seq", "accel", "pps"], _profile(), lanes)
        assert res.failed == 0 and len(res.rows) == 3 and set(res.summary) == {"seq", "accel", "pps"}
        px, _ = orchestrator.decode(parser.parse_stream(case.jpeg), "accel", None, lanes, data=case.jpeg)
    report.write_ppm(px, tmp_path / "a.ppm")
    w, h, data = report.read_ppm(tmp_path / "a.ppm")
    assert (w, h) == (case.width, case.height) and data == case.rgb.tobytes()
