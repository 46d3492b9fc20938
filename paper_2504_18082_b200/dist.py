"""Host-side multi-GPU logic of the step (no data-path collective).

Mini-batches are independent units given (graph, seed, batch id) (readings R11, R22): rank r
of a world of size W runs global batches r, r+W, r+2W, ...; the graph and features are
replicated.  The only collectives are for measurement: the max of the per-rank timed
durations and the sum of the per-rank counters."""
from __future__ import annotations

from typing import Iterable, List, Tuple

import torch
import torch.distributed as dist


def global_batch(rank: int, world: int, t: int) -> int:
    """Global batch id of this rank's t-th step (round-robin over ranks)."""
    return t * world + rank


def rank_batches(rank: int, world: int, steps: int) -> List[int]:
    return [global_batch(rank, world, t) for t in range(steps)]


def epoch_and_index(gb: int, n_batches: int) -> Tuple[int, int]:
    """Global batch id -> (epoch, batch index inside the epoch's order)."""
    return divmod(int(gb), int(n_batches))


def reduce_timing(ms: float, counters: Iterable[float], device=None) -> Tuple[float, List[float]]:
    """(max over ranks of `ms`, sum over ranks of each counter).  Identity when not distributed."""
    c = [float(x) for x in counters]
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(ms), c
    dev = device if device is not None else torch.device("cpu")
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    s = torch.tensor(c, dtype=torch.float64, device=dev)
    dist.all_reduce(s, op=dist.ReduceOp.SUM)
    return float(t.item()), [float(x) for x in s.tolist()]
