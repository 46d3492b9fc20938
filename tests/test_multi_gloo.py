"""World-size-2 CPU (gloo) test of the multi-GPU host logic: batches are
partitioned round-robin over ranks with no data-path collective, the timed duration is the
max over ranks and the counters are summed, and every batch's output is independent of the
world size (reading R11: results depend only on (graph, seed, batch id)).  The per-batch
work runs on the CPU oracle, which stands in for the GPU step here."""
import hashlib
import os
import socket
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
