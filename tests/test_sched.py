"""Profile-driven corpus scheduling (paper_1311_5304_b200/sched.py)."""
import os

import numpy as np

from paper_1311_5304_b200 import perf_model, sched

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _profile():
    return perf_model.load_profile(os.path.join(ROOT, "profiles", "b200_profile.json"))


def test_predict_scales_with_area_and_density():
    p = _profile()
    a = sched.predict(p, 1920, 1080, 1920 * 1080)
    b = sched.predict(p, 3840, 2160, 4 * 1920 * 1080)
    assert b.t_huff_ns > 3.5 * a.t_huff_ns and a.t_huff_ns > 0
    c = sched.predict(p, 1920, 1080, 2 * 1920 * 1080)  # denser
    assert c.t_huff_ns > a.t_huff_ns


def test_lpt_partitions_exactly_and_balances():
    rng = np.random.default_rng(0)
    costs = [sched.ImageCost(float(t), float(g)) for t, g in zip(rng.uniform(1e6, 5e7, 500), rng.uniform(1e4, 1e5, 500))]
    for ranks in (1, 2, 3, 8):
        parts = sched.assign_lpt(costs, ranks, host_threads=2)
        assert sorted(i for p in parts for i in p) == list(range(500))
        rep = sched.balance_report(costs, parts, 2)
        assert rep["imbalance"] < 1.02
    # GPU-bound corpus: the GPU column decides
    gpu_heavy = [sched.ImageCost(1.0, 1e6)] * 9
    parts = sched.assign_lpt(gpu_heavy, 3, host_threads=16)
    assert [len(p) for p in parts] == [3, 3, 3]


def test_makespan_model():
    cs = [sched.ImageCost(8e6, 1e6)] * 4
    assert sched.makespan(cs, 4) == 8e6
    assert sched.makespan(cs, 64) == 4e6
