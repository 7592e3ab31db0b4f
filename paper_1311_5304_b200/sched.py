"""Batch / multi-GPU scheduling on the recalibrated B200 DeviceProfile.

The reference partitions ONE image between a host lane and an accelerator
lane with its fitted cost models (partitioner.py, perf_model.py:212-239;
PAPER.md section 5).  On a B200 box the parallel phase never runs on the
host, so what the models schedule is different: a corpus of images over
GPUs, each GPU fed by its own share of the host cores, where every image
costs one host-Huffman task (t_huff, estimate_huffman_time:
rate(d) * w * h) overlapped with its GPU lane work (p_gpu(w, h): H2D +
kernel + D2H).  A rank's makespan is about

    max( sum t_huff / host_threads ,  sum p_gpu )

(the paper's pipelined scheme at corpus granularity: the GPU work hides
behind the Huffman stream unless the GPU side is the larger one).  Images
are assigned by LPT (longest predicted cost first, each to the rank whose
modelled makespan grows least), the standard 4/3-approximation for
identical machines.
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass

from .perf_model import DeviceProfile, entropy_density, estimate_huffman_time


@dataclass(frozen=True)
class ImageCost:
    t_huff_ns: float  # host entropy decode, one thread
    t_gpu_ns: float   # GPU lane: H2D + render + D2H


def predict(profile: DeviceProfile, width: int, height: int, file_size: int) -> ImageCost:
    """Modelled costs of one image from the profile (d = bytes per pixel)."""
    d = entropy_density(file_size, width, height).d
    return ImageCost(estimate_huffman_time(profile, width, height, d), profile.predict_p_gpu(width, height))


def makespan(costs, host_threads: int) -> float:
    """Modelled wall time of one rank decoding `costs` with `host_threads`."""
    th = sum(c.t_huff_ns for c in costs) / max(1, host_threads)
    return max(th, sum(c.t_gpu_ns for c in costs))


def assign_lpt(costs, n_ranks: int, host_threads: int) -> list:
    """Partition image indices over ranks: LPT on each image's modelled
    share of a rank's makespan.  Returns one index list per rank."""
    if n_ranks < 1:
        raise ValueError("n_ranks must be >= 1")
    weight = [max(c.t_huff_ns / max(1, host_threads), c.t_gpu_ns) for c in costs]
    order = sorted(range(len(costs)), key=lambda i: (-weight[i], i))
    heap = [(0.0, r) for r in range(n_ranks)]
    out = [[] for _ in range(n_ranks)]
    # per-rank running sums of both resources; key = the rank's makespan
    huff = [0.0] * n_ranks
    gpu = [0.0] * n_ranks
    for i in order:
        _, r = heapq.heappop(heap)
        out[r].append(i)
        huff[r] += costs[i].t_huff_ns
        gpu[r] += costs[i].t_gpu_ns
        heapq.heappush(heap, (max(huff[r] / max(1, host_threads), gpu[r]), r))
    return out


def balance_report(costs, parts, host_threads: int) -> dict:
    """Modelled per-rank makespans and the imbalance max / mean."""
    spans = [makespan([costs[i] for i in p], host_threads) for p in parts]
    mean = sum(spans) / max(1, len(spans))
    return {"makespans_ms": [round(s / 1e6, 3) for s in spans],
            "imbalance": round(max(spans) / mean, 4) if mean > 0 else 1.0}
