"""a6: input-feature gather from a ROW-SHARDED feature table (north_star: papers100M-scale
tables are row-sharded over the GPUs, with an NCCL all-to-all over NVLink for remote rows).

Rank r of W owns rows [r*S, min(N, (r+1)*S)), S = ceil(N / W).  For a batch's input nodes
nodes[0:U) the exchange is (all ranks call it in lockstep, one call per batch):

    plan      cmb_shard_plan: stable bucketing by owner -> send_ids (owner-major), perm, counts
    counts    all_to_all_single of the W counts        (NCCL)
    ids       all_to_all_single of the requested ids   (NCCL)
    gather    cmb_gather_rows from the local shard
    rows      all_to_all_single of the rows back       (NCCL)
    scatter   cmb_scatter_rows: X_in[perm[k]] = row k

The result is byte-identical to the replicated gather (oracle O5).  The device steps go
through the C ABI (`CudaOps`); the host protocol (splits, ordering, collectives) is this
class.  Tests on CPU substitute a numpy `ops` object (a fake backend) to check the protocol
with world-size-2 gloo; the product path has no CPU fallback.
"""
from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

from . import _check, _ptr, _stream, _workspace, lib


class CudaOps:
    """Device steps of the exchange through the C ABI (include/cmb.h, a6)."""

    def __init__(self):
        self._ws = {}

    def plan(self, nodes, n_dev, n_cap, rows_per_shard, world):
        dev = nodes.device
        key = (dev, n_cap)
        if key not in self._ws:
            self._ws[key] = _workspace(lib().cmb_shard_plan_workspace_bytes(n_cap), dev)
        ws = self._ws[key]
        counts = torch.empty(world, dtype=torch.int64, device=dev)
        send_ids = torch.empty(n_cap, dtype=torch.int32, device=dev)
        perm = torch.empty(n_cap, dtype=torch.int32, device=dev)
        _check(lib().cmb_shard_plan(_ptr(nodes), _ptr(n_dev), n_cap, int(rows_per_shard),
                                    int(world), _ptr(counts), _ptr(send_ids), _ptr(perm),
                                    _ptr(ws), ws.numel(), _stream()))
        return counts, send_ids, perm

    def gather_rows(self, x_local, row0, feat_dim, ids, out):
        n = torch.tensor([ids.shape[0]], dtype=torch.int64, device=ids.device)
        if ids.shape[0]:
            _check(lib().cmb_gather_rows(_ptr(x_local), x_local.stride(0), int(row0),
                                         int(feat_dim), _ptr(ids), _ptr(n), ids.shape[0],
                                         _ptr(out), out.stride(0), _stream()))
        return out

    def scatter_rows(self, rows, perm, n, feat_dim, out):
        nd = torch.tensor([n], dtype=torch.int64, device=rows.device)
        if n:
            _check(lib().cmb_scatter_rows(_ptr(rows), rows.stride(0), _ptr(perm), _ptr(nd), n,
                                          int(feat_dim), _ptr(out), out.stride(0), _stream()))
        return out


class ShardedFeatures:
    """This rank's shard of the feature table + the all-to-all exchange of one batch."""

    def __init__(self, x_local: torch.Tensor, num_nodes: int, feat_dim: int, world: int,
                 rank: int, group=None, ops=None):
        self.x = x_local
        self.N = int(num_nodes)
        self.F = int(feat_dim)
        self.world = int(world)
        self.rank = int(rank)
        self.S = (self.N + self.world - 1) // self.world   # rows per shard
        self.row0 = self.rank * self.S
        self.group = group
        self.ops = ops if ops is not None else CudaOps()

    @staticmethod
    def shard_bounds(num_nodes: int, world: int, rank: int):
        S = (num_nodes + world - 1) // world
        return rank * S, min(num_nodes, (rank + 1) * S)

    def _a2a(self, out, inp, out_splits, in_splits):
        if self.world == 1:
            out.copy_(inp)
            return out
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)
        return out

    def gather(self, nodes: torch.Tensor, n: int, out: torch.Tensor) -> torch.Tensor:
        """out[i, :F] = X[nodes[i], :F] for i < n, X the row-sharded table (collective)."""
        dev = self.x.device
        n_dev = torch.tensor([n], dtype=torch.int64, device=dev)
        n_cap = max(1, int(n))
        counts, send_ids, perm = self.ops.plan(nodes, n_dev, n_cap, self.S, self.world)
        recv_counts = torch.empty_like(counts)
        self._a2a(recv_counts, counts, [1] * self.world, [1] * self.world)
        # NCCL's all-to-all takes its variable splits on the host: ONE device->host read of both
        # count vectors per batch is this protocol's synchronisation cost (the one-sided form,
        # cmb_gather_aggregate_sharded, has none)
        both = torch.cat([counts, recv_counts]).cpu().tolist()
        sc = [int(c) for c in both[: self.world]]
        rc = [int(c) for c in both[self.world:]]
        req = torch.empty(sum(rc), dtype=torch.int32, device=dev)
        self._a2a(req, send_ids[: sum(sc)].contiguous(), rc, sc)
        rows = torch.empty(sum(rc), self.x.stride(0), dtype=self.x.dtype, device=dev)
        self.ops.gather_rows(self.x, self.row0, self.F, req, rows)
        back = torch.empty(sum(sc), self.x.stride(0), dtype=self.x.dtype, device=dev)
        self._a2a(back, rows, sc, rc)
        self.ops.scatter_rows(back, perm, int(n), self.F, out)
        return out
