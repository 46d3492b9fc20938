"""NEXT-1: the one-sided sharded gather (cmb_gather_aggregate_sharded) -- the fused a4 + a5
reading every feature row from its owner's shard through a pointer table.

* virtual shards: W separate allocations on one GPU, W in {1, 2, 3, 8}; X_in and H
  byte-identical to the oracle (and so to the replicated path).
* CUDA IPC: two processes on the same GPU, each owning half of the table, exchange handles
  over a gloo group (ShardTable.exchange) and read the other's half through the mapping --
  the same code path that reads peer HBM over NVLink on a multi-GPU node."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
from gen import CONFIGS, generate, scaled

pytestmark = pytest.mark.gpu
cmb = pytest.importorskip("paper_2504_18082_b200")
SEED = 42


def _setup():
    b = generate(scaled(CONFIGS["products"], 0.01))
    prep = oracle.graph_prep(b)
    g = cmb.Graph.from_bundle(b, features=False)
    order = oracle.order_roots(b.train, b.comm, b.cfg.num_communities, oracle.MODE_RAND, 0, SEED, 0)
    return b, prep, g, order


def _check(b, prep, x_in, h, roots_np, n, batch):
    cfg = b.cfg
    ref = oracle.run_batch(prep, b.X, cfg.feat_dim, roots_np, cfg.fanouts, cfg.p_intra, SEED, batch)
    assert n == ref["n"]
    L = len(cfg.fanouts)
    F = cfg.feat_dim
    assert x_in[: n[L], :F].cpu().numpy().tobytes() == ref["X_in"].tobytes()
    assert h[: n[L - 1], :F].cpu().numpy().tobytes() == ref["H"].tobytes()


@pytest.mark.parametrize("W", [1, 2, 3, 8])
def test_virtual_shards(W):
    b, prep, g, order = _setup()
    cfg = b.cfg
    X = torch.from_numpy(b.X).cuda()
    S = (cfg.num_nodes + W - 1) // W
    shards = [X[r * S: (r + 1) * S].clone() for r in range(W)]  # separate allocations
    table = cmb.ShardTable(shards, cfg.num_nodes, cfg.feat_dim)
    s = cmb.Sampler(g, cfg.batch_size, cfg.fanouts)
    for bb in (0, 1):
        roots = oracle.batch_roots(order, cfg.batch_size, bb)
        view = s.sample(torch.from_numpy(roots).cuda(), cfg.p_intra, SEED, bb)
        x_in, h = s.gather_aggregate_sharded(table)
        torch.cuda.synchronize()
        assert s.status() == 0
        n, _ = view.host_sizes()
        _check(b, prep, x_in, h, roots, n, bb)


def test_sharded_rejects_bad_cover():
    b, prep, g, order = _setup()
    cfg = b.cfg
    X = torch.from_numpy(b.X).cuda()
    table = cmb.ShardTable([X[:10].clone(), X[10:20].clone()], cfg.num_nodes, cfg.feat_dim)
    table.rows_per_shard = 10  # does not cover num_nodes
    s = cmb.Sampler(g, cfg.batch_size, cfg.fanouts)
    s.sample(torch.arange(8, dtype=torch.int32, device="cuda"), cfg.p_intra, SEED, 0)
    with pytest.raises(cmb.CmbError) as ei:
        s.gather_aggregate_sharded(table)
    assert ei.value.code == 1


def _ipc_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b, prep, g, order = _setup()
        cfg = b.cfg
        S = (cfg.num_nodes + world - 1) // world
        mine = torch.from_numpy(b.X[rank * S: (rank + 1) * S]).cuda()
        table = cmb.ShardTable.exchange(mine, cfg.num_nodes, cfg.feat_dim, rank, world)
        s = cmb.Sampler(g, cfg.batch_size, cfg.fanouts)
        bb = rank
        roots = oracle.batch_roots(order, cfg.batch_size, bb)
        view = s.sample(torch.from_numpy(roots).cuda(), cfg.p_intra, SEED, bb)
        x_in, h = s.gather_aggregate_sharded(table)
        torch.cuda.synchronize()
        n, _ = view.host_sizes()
        _check(b, prep, x_in, h, roots, n, bb)
        dist.barrier()          # the peer has finished reading my shard
        table.close()
        q.put((rank, "ok"))
    except Exception as e:  # report instead of hanging the other rank
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_ipc_two_processes_one_gpu():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(2))
    for p in ps:
        p.join(timeout=120)
    assert res == {0: "ok", 1: "ok"}, res
