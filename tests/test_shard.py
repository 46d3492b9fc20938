"""a6 row-sharded feature exchange.

CPU (world-size-2 gloo): the host protocol of ShardedFeatures.gather (owner bucketing, the
count / id / row all-to-alls, scatter) with a numpy fake backend standing in for the device
steps, against X[nodes] of the full table.
GPU (-m gpu): the device steps through the C ABI with W virtual shards in one process (no NCCL),
and the world-size-1 path, byte-identical to the oracle gather (O5)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_18082_b200.shard import ShardedFeatures


class NumpyOps:
    """Fake backend (test infrastructure): the three device steps in numpy."""

    def plan(self, nodes, n_dev, n_cap, rows_per_shard, world):
        n = int(n_dev[0])
        v = nodes[:n].numpy()
        own = v // rows_per_shard
        perm = np.argsort(own, kind="stable").astype(np.int32)
        counts = np.bincount(own, minlength=world).astype(np.int64)
        send = np.zeros(n_cap, np.int32)
        send[:n] = v[perm]
        p = np.zeros(n_cap, np.int32)
        p[:n] = perm
        return torch.from_numpy(counts), torch.from_numpy(send), torch.from_numpy(p)

    def gather_rows(self, x_local, row0, feat_dim, ids, out):
        if ids.shape[0]:
            out[: ids.shape[0], :feat_dim] = x_local[ids.long() - row0, :feat_dim]
        return out

    def scatter_rows(self, rows, perm, n, feat_dim, out):
        out[perm[:n].long(), :feat_dim] = rows[:n, :feat_dim]
        return out


def _table(N=1000, F=8, ld=8):
    g = torch.Generator().manual_seed(3)
    return torch.randn(N, ld, generator=g)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    X = _table()
    N, F = X.shape[0], 8
    lo, hi = ShardedFeatures.shard_bounds(N, world, rank)
    sf = ShardedFeatures(X[lo:hi].clone(), N, F, world, rank, ops=NumpyOps())
    ok = True
    for trial in range(3):
        g = torch.Generator().manual_seed(100 * rank + trial)
        n = int(torch.randint(1, 300, (1,), generator=g))
        nodes = torch.randperm(N, generator=g)[:n].to(torch.int32)
        out = torch.zeros(n, F)
        sf.gather(nodes, n, out)
        ok &= torch.equal(out, X[nodes.long(), :F])
    q.put((rank, bool(ok)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_exchange_protocol_gloo():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res)


def test_shard_bounds_cover_table():
    for N, W in ((1000, 3), (7, 8), (111_059_956, 8)):
        b = [ShardedFeatures.shard_bounds(N, W, r) for r in range(W)]
        assert b[0][0] == 0 and b[-1][1] == N
        assert all(b[i][1] == b[i + 1][0] or b[i + 1][0] >= N for i in range(W - 1))


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("W", [1, 2, 4, 8])
def test_virtual_shards_match_oracle_gather(W):
    import oracle
    import paper_2504_18082_b200 as cmb
    from paper_2504_18082_b200.shard import CudaOps
    from gen import CONFIGS, generate, scaled
    b = generate(scaled(CONFIGS["products"], 0.01))
    cfg = b.cfg
    X = torch.from_numpy(b.X).cuda()
    rng = np.random.default_rng(W)
    nodes_np = rng.choice(cfg.num_nodes, 5000, replace=False).astype(np.int32)
    nodes = torch.from_numpy(nodes_np).cuda()
    n = nodes.shape[0]
    ops = CudaOps()
    S = (cfg.num_nodes + W - 1) // W
    counts, send_ids, perm = ops.plan(nodes, torch.tensor([n], device="cuda"), n, S, W)
    cnt = counts.cpu().tolist()
    rows = torch.empty(n, X.stride(0), device="cuda")
    off = 0
    for r in range(W):  # every owner serves its slice of the requests from its shard
        lo, hi = ShardedFeatures.shard_bounds(cfg.num_nodes, W, r)
        ops.gather_rows(X[lo:hi], lo, cfg.feat_dim, send_ids[off: off + cnt[r]], rows[off:])
        off += cnt[r]
    out = torch.zeros(n, X.stride(0), device="cuda")
    ops.scatter_rows(rows, perm, n, cfg.feat_dim, out)
    torch.cuda.synchronize()
    ref = oracle.gather(nodes_np, b.X, cfg.feat_dim)
    assert out[:, : cfg.feat_dim].cpu().numpy().tobytes() == ref.tobytes()
    # the world-size-1 exchange (no process group): the same bytes through ShardedFeatures
    if W == 1:
        sf = ShardedFeatures(X, cfg.num_nodes, cfg.feat_dim, 1, 0)
        out2 = torch.zeros(n, X.stride(0), device="cuda")
        sf.gather(nodes, n, out2)
        torch.cuda.synchronize()
        assert out2[:, : cfg.feat_dim].cpu().numpy().tobytes() == ref.tobytes()


# ------------------------------------------------------------------ NEXT-1 host logic (CPU)
def test_shard_table_layout_and_validation():
    from paper_2504_18082_b200 import ShardTable
    N, F = 1001, 8
    X = torch.zeros(N, 8)
    W = 3
    S = (N + W - 1) // W
    t = ShardTable([X[r * S:(r + 1) * S] for r in range(W)], N, F)
    assert t.world == W and t.rows_per_shard == S and t.shard_ld == 8
    assert list(t.ptr_array) == [X[r * S:].data_ptr() for r in range(W)]
    # raw pointers need the row stride
    t2 = ShardTable([X.data_ptr(), X[S:].data_ptr()], N, F, shard_ld=8)
    assert t2.world == 2 and t2.rows_per_shard == (N + 1) // 2
    with pytest.raises(ValueError):
        ShardTable([X, torch.zeros(N, 12)], N, F)          # mixed strides
    with pytest.raises(ValueError):
        ShardTable([X] * 9, N, F)                           # more than 8 shards
    with pytest.raises(ValueError):
        ShardTable([X.data_ptr()], N, F)                    # pointer without a stride


def test_owner_formula_matches_division():
    # the device's owner computation (gather_row.cuh ShardedRows::row), restated on the host
    rng = np.random.default_rng(5)
    for S in (1, 2, 3, 7, 1000, 1_388_237, 13_882_495, 2 ** 30):
        inv = ((1 << 32) + S - 1) // S
        us = np.concatenate([[0, 1, S - 1, S, S + 1, 2 * S - 1, 2 * S, 2 ** 31 - 1],
                             rng.integers(0, 2 ** 31, 3000)])
        for u in us.tolist():
            r = (u * inv) >> 32
            if r * S > u:
                r -= 1
            assert r == u // S
