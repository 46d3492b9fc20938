"""Host-side multi-GPU logic of the step (no data-path collective).

Mini-batches are independent units given (graph, seed, batch id) (readings R11, R22): rank r
of a world of size W runs global batches r, r+W, r+2W, ...; the graph and features are
replicated.  The only collectives are for measurement: the max of the per-rank timed
durations and the sum of the per-rank counters."""
from __future__ import annotations

from typing import Iterable, List, Tuple

import numpy as np

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


# ---------------------------------------------------------------- NEXT-1: shard-aligned placement
def shard_owner(v, rows_per_shard: int):
    """Owner rank of node / feature row v under contiguous row sharding (a6: S = ceil(N / W))."""
    return v // rows_per_shard


def aligned_schedule(order, batch_size: int, num_nodes: int, world: int) -> List[List[int]]:
    """Community-aware batch -> GPU placement (second half).

    With a community-ordered graph the feature shards are contiguous id ranges, i.e. runs
    of whole communities, and the community-aware Knob-1 orders (COMM-MIX-k) give each batch
    roots from a few communities.  Placing batch b on the rank that owns the median id of its
    roots keeps its input rows (mostly intra-community at high p_intra) in the local
    shard, so the one-sided gather reads them from local HBM instead of over NVLink -- the
    paper's reuse argument applied to the sharded table.

    Returns, per rank, the epoch-local batch indices it runs, in epoch order.  Balance: every rank
    gets floor(nb / W) or ceil(nb / W) batches (first come first served at the home rank; a
    batch whose home is full goes to the least-loaded rank, ties to the lowest shard distance,
    then the lowest rank).  Deterministic: every rank computes the same schedule from the same
    epoch order, with no collective.
    """
    o = order.cpu().numpy() if isinstance(order, torch.Tensor) else np.asarray(order)
    n = int(o.shape[0])
    nb = (n + batch_size - 1) // batch_size
    S = (int(num_nodes) + world - 1) // world
    base, spare = divmod(nb, world)  # every rank runs base batches, `spare` ranks one more
    load = [0] * world
    n_full = 0                       # ranks already at base + 1
    out: List[List[int]] = [[] for _ in range(world)]
    for b in range(nb):
        roots = o[b * batch_size: min((b + 1) * batch_size, n)]
        home = min(int(shard_owner(int(np.median(roots)), S)), world - 1)

        def has_room(r):
            return load[r] < base or (load[r] == base and n_full < spare)

        r = home if has_room(home) else min(
            (q for q in range(world) if has_room(q)), key=lambda q: (load[q], abs(q - home), q))
        n_full += load[r] == base
        load[r] += 1
        out[r].append(b)
    return out


def remote_fraction(nodes: torch.Tensor, n_rows: int, rank: int, rows_per_shard: int) -> float:
    """Fraction of a batch's input rows nodes[0:n_rows) that another rank owns."""
    if n_rows == 0:
        return 0.0
    own = shard_owner(nodes[:n_rows].to(torch.int64), rows_per_shard)
    return float((own != rank).sum().item()) / float(n_rows)
