"""bench.py contract on CPU: the reference arm's JSON line (same metric as
ours, no product library in its process), `--gpus N` spawning N ranks by
itself, and bench's own N-rank helpers (dist_setup / barrier / max- and
sum-reductions) under a world-size-2 gloo group."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _run(args, env=None, timeout=240):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, env=e, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    return lines


def test_reference_arm_line_is_clean():
    (line,) = _run(["--impl", "reference", "--workload", "512p420", "--steps", "3", "--warmup", "1"])
    assert line["impl"] == "reference"
    assert line["metric"] == bench.METRIC and line["unit"] == "Mpix/s" and line["higher_is_better"]
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["value"] == line["value"]
    # the reference arm never maps the product library
    assert not any("paper_1311_5304_b200" in p for p in line["repo_libs_loaded"])


def test_gpus_flag_spawns_ranks():
    # two ranks (torch.distributed.run on 127.0.0.1); only rank 0 prints
    lines = _run(["--gpus", "2", "--impl", "reference", "--workload", "512p420", "--steps", "2", "--warmup", "1"])
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, port, q):
    os.environ.update(WORLD_SIZE="2", RANK=str(rank), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    world, r, local, pg = bench.dist_setup()
    bench.barrier(pg)
    mx = bench.allreduce_max(pg, 1.0 + rank)
    sm = bench.allreduce_sum(pg, 10.0 * (rank + 1))
    q.put((r, world, local, mx, sm))
    pg.destroy_process_group()


def test_bench_dist_helpers_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_rank, args=(r, port, q)) for r in range(2)]
    [p.start() for p in ps]
    res = sorted(q.get(timeout=120) for _ in ps)
    [p.join(timeout=60) for p in ps]
    assert [r[0] for r in res] == [0, 1] and all(r[1] == 2 for r in res)
    assert all(r[3] == 2.0 and r[4] == 30.0 for r in res)  # max over ranks, whole-job sum


@pytest.mark.skipif(not os.path.isdir(os.path.join(ROOT, "oracle", "_ref", "patched", "hetjpeg")),
                    reason="reference build (oracle/build_ref.sh) not present")
def test_reference_arm_runs_the_reference_for_422():
    (line,) = _run(["--impl", "reference", "--workload", "1080p444q50", "--steps", "2", "--warmup", "1"],
                   timeout=400)
    assert line["cpu_baseline"]["kind"] == "reference"
    assert line["metric"] == bench.METRIC
