"""Output formats of the reference's front end: the P6 PPM
writer, the per-image bench CSV and the per-mode speed-up summary
(reference `cli.py:21-25` write_ppm, `cli.py:171-234` cmd_bench).

Only the formats and the bench loop are kept - the argparse CLI itself is out
of scope.  `bench_corpus` runs exactly the reference's loop:
every image is decoded in each requested mode plus the reference mode, the
reference run's Amdahl bound is recorded, one CSV row per (image, mode) with
the reference's columns, and one summary line per mode with the mean speed-up
over the reference mode and its coefficient of variation.
"""
from __future__ import annotations

import csv
import statistics
from dataclasses import dataclass, field
from pathlib import Path

from .errors import HetJpegError
from .orchestrator import MODES, amdahl_bound, decode
from .parser import parse_stream

# cli.py:171-172
CSV_HEADER = ["image", "w", "h", "d", "mode", "wall_ns", "huff_ns", "par_ns",
              "x_rows", "chunks", "amdahl_bound"]


def ppm_bytes(pixels) -> bytes:
    """Binary PPM (P6, maxval 255) of a PixelBuffer (cli.py:21-25)."""
    return f"P6\n{pixels.width} {pixels.height}\n255\n".encode("ascii") + pixels.tobytes()


def write_ppm(pixels, path) -> None:
    """Write `pixels` as binary PPM (cli.py:21-25)."""
    with open(path, "wb") as fh:
        fh.write(ppm_bytes(pixels))


def read_ppm(path_or_bytes) -> tuple:
    """Parse a P6 maxval-255 PPM written by `write_ppm`: (width, height, rgb bytes)."""
    blob = path_or_bytes if isinstance(path_or_bytes, (bytes, bytearray)) else Path(path_or_bytes).read_bytes()
    parts, pos = [], 0
    while len(parts) < 4:
        while blob[pos:pos + 1].isspace():
            pos += 1
        end = pos
        while not blob[end:end + 1].isspace():
            end += 1
        parts.append(blob[pos:end])
        pos = end
    if parts[0] != b"P6" or parts[3] != b"255":
        raise ValueError("not a P6 maxval-255 PPM")
    w, h = int(parts[1]), int(parts[2])
    data = bytes(blob[pos + 1:])
    if len(data) != 3 * w * h:
        raise ValueError(f"PPM payload {len(data)} B != 3*{w}*{h}")
    return w, h, data


def csv_row(image: str, report, bound: float) -> list:
    """One bench CSV row (cli.py:212-216)."""
    plan_x = report.plan.x_cpu_rows if report.plan else -1
    return [image, report.width, report.height, f"{report.density:.6f}", report.mode, report.wall_ns,
            report.huffman_ns, report.parallel_host_ns, plan_x, len(report.chunks), f"{bound:.6f}"]


@dataclass
class BenchResult:
    rows: list = field(default_factory=list)        # CSV rows (CSV_HEADER order)
    failed: int = 0
    summary: dict = field(default_factory=dict)     # mode -> (images, mean speed-up, cov %)

    def summary_lines(self, reference: str) -> list:
        """The reference's per-mode stdout lines (cli.py:223-233)."""
        return [f"mode={m} images={n} mean_speedup_vs_{reference}={mean:.3f} cov_pct={cov:.2f}"
                for m, (n, mean, cov) in self.summary.items()]

    def write_csv(self, path) -> None:
        with open(path, "w", newline="", encoding="utf-8") as fh:
            writer = csv.writer(fh)
            writer.writerow(CSV_HEADER)
            writer.writerows(self.rows)


def bench_corpus(images, modes, profile, lanes, reference: str = "seq", errors=None) -> BenchResult:
    """The reference's bench loop (cli.py:174-234) over `images`, an iterable of
    (name, jpeg bytes) or paths.  Unknown modes raise ValueError (the CLI's
    usage error); model-driven modes need a profile."""
    modes = list(modes)
    for m in modes:
        if m not in MODES:
            raise ValueError(f"unknown mode {m!r}")
    if profile is None and any(m in ("sps", "pps", "accel-pipe") for m in modes):
        raise ValueError("model-driven modes require a profile")
    res = BenchResult()
    wall_by_mode: dict = {m: {} for m in modes}
    ref_by_image: dict = {}
    for item in images:
        if isinstance(item, tuple):
            name, blob = item
        else:
            name, blob = Path(item).name, Path(item).read_bytes()
        try:
            parsed = parse_stream(blob)
            run_modes = modes + ([reference] if reference not in modes else [])
            reports = {m: decode(parsed, m, profile, lanes, data=blob)[1] for m in run_modes}
            bound = amdahl_bound(reports[reference])
            ref_by_image[name] = (reports[reference].wall_ns, bound)
            for m in modes:
                res.rows.append(csv_row(name, reports[m], bound))
                wall_by_mode[m][name] = reports[m].wall_ns
        except HetJpegError as exc:
            res.failed += 1
            if errors is not None:
                errors.append(f"error: {name}: {exc}")
    for m in modes:
        speedups = [ref_by_image[img][0] / wall for img, wall in wall_by_mode[m].items() if wall > 0]
        if not speedups:
            continue
        mean = statistics.fmean(speedups)
        cov = statistics.stdev(speedups) / mean * 100.0 if len(speedups) > 1 and mean > 0 else 0.0
        res.summary[m] = (len(speedups), mean, cov)
    return res
