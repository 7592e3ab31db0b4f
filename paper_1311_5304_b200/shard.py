"""Multi-GPU work assignment: images (or MCU-row ranges of one large image)
shard across ranks with no data exchange.

* `assign_lpt`   - longest-processing-time-first assignment of images to ranks
                   by a predicted cost (pixels, or a DeviceProfile prediction).
* `split_rows`   - contiguous MCU-row ranges of one image for N ranks; 4:2:0
                   ranges read one chroma MCU row of context on each side
                   (`chroma_context`), which each rank decodes/ships itself.
* `max_over_ranks` - timing reduction (the only collective: a scalar max).
"""
from __future__ import annotations

import heapq


def assign_lpt(costs, world: int) -> list:
    """Return, per rank, the list of item indices (LPT greedy, deterministic)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    heap = [(0.0, r) for r in range(world)]
    out = [[] for _ in range(world)]
    for i in sorted(range(len(costs)), key=lambda k: (-costs[k], k)):
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + float(costs[i]), r))
    for lst in out:
        lst.sort()
    return out


def split_rows(mcu_rows: int, world: int) -> list:
    """Contiguous (row0, n_rows) per rank covering [0, mcu_rows) exactly."""
    base, extra = divmod(mcu_rows, world)
    out, r = [], 0
    for k in range(world):
        n = base + (1 if k < extra else 0)
        out.append((r, n))
        r += n
    return out


def chroma_context(row0: int, n_rows: int, mcu_rows: int) -> tuple:
    """MCU rows whose coefficients a 4:2:0 render of [row0, row0+n) reads."""
    return max(0, row0 - 1), min(mcu_rows, row0 + n_rows + 1)


def max_over_ranks(value: float, group=None) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
