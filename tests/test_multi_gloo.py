"""World-size-2 CPU (gloo) test of the multi-GPU host logic: batches are
partitioned round-robin over ranks with no data-path collective, the timed duration is the
max over ranks and the counters are summed, and every batch's output is independent of the
world size (reading R11: results depend only on (graph, seed, batch id)).  The per-batch
work runs on the CPU oracle, which stands in for the GPU step here."""
import hashlib
import os
import socket
import sys
import time

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from gen import CONFIGS, generate
from paper_2504_18082_b200 import dist as cmb_dist

STEPS, SEED, P = 7, 42, 0.9


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run_batches(rank, world):
    b = generate(CONFIGS["tiny"])
    cfg = b.cfg
    prep = oracle.graph_prep(b)
    nb = (cfg.n_train + cfg.batch_size - 1) // cfg.batch_size
    out = {}
    for gb in cmb_dist.rank_batches(rank, world, STEPS):
        epoch, bi = cmb_dist.epoch_and_index(gb, nb)
        order = oracle.order_roots(b.train, b.comm, cfg.num_communities, oracle.MODE_COMM, 0.5,
                                   SEED, epoch)
        blk = oracle.sample_blocks(prep, oracle.batch_roots(order, cfg.batch_size, bi),
                                   cfg.fanouts, P, SEED, gb)
        h = hashlib.sha1(blk["nodes"].tobytes())
        for ix in blk["indices"]:
            h.update(ix.tobytes())
        out[gb] = h.hexdigest()
    return out


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t0 = time.perf_counter()
    res = _run_batches(rank, world)
    ms = (time.perf_counter() - t0) * 1e3 + 10.0 * rank  # skew: rank 1 is "slower"
    ms_max, (n_tot,) = cmb_dist.reduce_timing(ms, [len(res)])
    gathered = [None] * world
    dist.all_gather_object(gathered, res)
    q.put((rank, ms, ms_max, n_tot, gathered))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_partition_timing_and_invariance():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    rows = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rows.sort()
    ms_each = [r[1] for r in rows]
    for _, ms, ms_max, n_tot, gathered in rows:
        assert ms_max == max(ms_each)          # max over ranks
        assert n_tot == world * STEPS          # summed counters
        batches = [set(g) for g in gathered]
        assert not (batches[0] & batches[1])    # disjoint
        assert set().union(*batches) == set(range(world * STEPS))  # round-robin covers all
    # world-size invariance: the same batch ids computed by one process give the same bytes
    merged = {}
    for g in rows[0][4]:
        merged.update(g)
    single = _run_batches(0, 1)
    for gb, hx in single.items():
        assert merged[gb] == hx


def test_rank_batch_helpers():
    assert cmb_dist.rank_batches(1, 4, 3) == [1, 5, 9]
    assert cmb_dist.epoch_and_index(200, 193) == (1, 7)
    ms, c = cmb_dist.reduce_timing(3.5, [1, 2])   # not initialised: identity
    assert ms == 3.5 and c == [1.0, 2.0]
    assert np.array_equal(np.sort(sum((cmb_dist.rank_batches(r, 3, 4) for r in range(3)), [])),
                          np.arange(12))


# ---------------------------------------------------------------- NEXT-1: shard-aligned placement
def test_aligned_schedule_partition_and_balance():
    rng = np.random.default_rng(0)
    for world in (1, 2, 3, 8):
        for n in (1, 100, 1024 * 5 + 7, 20000):
            o = rng.permutation(100000)[:n].astype(np.int32)
            sch = cmb_dist.aligned_schedule(o, 1024, 100000, world)
            nb = (n + 1023) // 1024
            assert sorted(b for r in sch for b in r) == list(range(nb))
            loads = [len(r) for r in sch]
            assert max(loads) - min(loads) <= 1
            assert all(r == sorted(r) for r in sch)    # epoch order kept on every rank


def test_aligned_schedule_follows_the_shards():
    """Batches whose roots sit in one shard go to that shard's owner when quotas allow."""
    world, N, B = 4, 4000, 100
    S = N // world
    # 8 batches: two per shard, roots drawn inside the shard
    rng = np.random.default_rng(1)
    order = np.concatenate([rng.choice(np.arange(r * S, (r + 1) * S), B, replace=False)
                            for r in (2, 0, 3, 1, 1, 3, 0, 2)]).astype(np.int32)
    sch = cmb_dist.aligned_schedule(order, B, N, world)
    assert sch == [[1, 6], [3, 4], [0, 7], [2, 5]]
    # a skewed order (all roots in shard 0) still balances
    sch = cmb_dist.aligned_schedule(np.arange(800, dtype=np.int32), B, N, world)
    assert [len(r) for r in sch] == [2, 2, 2, 2] and sch[0] == [0, 1]


def test_remote_fraction_counts_foreign_rows():
    import torch
    nodes = torch.tensor([0, 5, 10, 15, 19, 3], dtype=torch.int32)
    assert cmb_dist.remote_fraction(nodes, 5, 0, 10) == 3 / 5    # rows 10, 15, 19 are rank 1's
    assert cmb_dist.remote_fraction(nodes, 6, 1, 10) == 3 / 6
    assert cmb_dist.remote_fraction(nodes, 0, 0, 10) == 0.0


def test_bench_relaunches_under_torchrun(monkeypatch):
    """`python bench.py --gpus N` outside torchrun starts N ranks through torch.distributed.run
    on 127.0.0.1 with the same arguments (the driver's command form)."""
    import bench
    seen = {}

    def fake_call(cmd, env=None):
        seen["cmd"], seen["env"] = cmd, env
        return 0

    monkeypatch.setattr(bench.subprocess, "call", fake_call)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "7"])
    assert bench.main() == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "7"]
    assert os.path.basename(cmd[cmd.index("--master-addr=127.0.0.1") + 2]) == "bench.py"
