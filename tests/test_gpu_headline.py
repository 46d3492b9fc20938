"""GPU parity of the EXACT benchmarked path (bench.py's default run), every batch of an epoch.

bench.py times products-shaped input (BASELINE.json configs[3], full size) through
``BatchedPipeline.step_group`` -> ``cmb_step_group``: one cooperative sampler launch for
``cmb.DEFAULT_BATCHES_PER_LAUNCH`` = 6 batches (the SMs split into 6 virtual grids of 24 blocks)
followed by the ONE fused gather + aggregate launch over all of them.  This file runs that same call, with the same pipeline
object and the same global batch ids (epoch 0: 0 .. n_batches - 1, the last group ragged),
and compares EVERY batch of epoch 0 with the oracle:

* nodes (relabel map), sizes, indptr and indices of every hop: bit-exact;
* X_in bit-exact and H bit-exact with the CSR-order fp32 oracle (O5, O6);
* H within the 1e-5 bound of the fp64 shadow on a few batches (first, middle, ragged last);

at the bench's default knob point (RAND, p = 0.5) and the paper's best total-training point
(COMM-RAND-MIX-12.5 %, p = 1.0).  The oracle batches run in a thread pool (the oracle's
C functions release the GIL), each thread with its own scratch map.

The RAND point must reach the sampler's uncached row branch (``sample_persist.cuh``: a virtual
block owning more than kRowCap = 3072 dst rows of a hop re-reads the row info from global
memory instead of its shared-memory cache); the test asserts that some batch does.
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

import oracle
from gen import CONFIGS, generate

pytestmark = pytest.mark.gpu
cmb = pytest.importorskip("paper_2504_18082_b200")

SEED = 42
K_ROW_CAP = 3072  # sample_persist.cuh kRowCap
_CACHE = {}


def _products():
    if "p" not in _CACHE:
        b = generate(CONFIGS["products"])
        _CACHE["p"] = (b, oracle.graph_prep(b), cmb.Graph.from_bundle(b))
    return _CACHE["p"]


def _mode(m):
    return {"rand": oracle.MODE_RAND, "norand": oracle.MODE_NORAND, "comm": oracle.MODE_COMM,
            "comm_static": oracle.MODE_COMM_STATIC}[m]


def _agg_tol_ok(H, H64, Xin, ip, idx):
    deg = np.diff(ip)
    scale = np.zeros_like(H64)
    np.add.at(scale, np.repeat(np.arange(deg.shape[0]), deg), np.abs(Xin[idx]).astype(np.float64))
    scale[deg > 0] /= deg[deg > 0, None]
    return bool(np.all(np.abs(H.astype(np.float64) - H64)
                       <= 1e-5 * np.maximum(np.abs(H64), scale) + 1e-30))


def _host_batch(s, L, F):
    """Host copies of one sampler's outputs (valid prefix only)."""
    sz = s.sizes.cpu().numpy()
    n, e = [int(x) for x in sz[: L + 1]], [int(x) for x in sz[L + 1:]]
    return {"n": n, "e": e, "nodes": s.nodes[: n[L]].cpu().numpy(),
            "indptr": [s.indptr[h][: n[h] + 1].cpu().numpy().astype(np.int64) for h in range(L)],
            "indices": [s.indices[h][: e[h]].cpu().numpy() for h in range(L)],
            "X_in": s.x_in[: n[L], :F].cpu().numpy(), "H": s.h[: n[L - 1], :F].cpu().numpy()}


@pytest.mark.parametrize("mode,k,p", [("rand", 0.0, 0.5), ("comm", 0.125, 1.0)])
def test_bench_launch_config_every_batch_of_epoch0(mode, k, p):
    b, prep, g = _products()
    cfg = b.cfg
    L, F, B = len(cfg.fanouts), cfg.feat_dim, cfg.batch_size
    G = cmb.DEFAULT_BATCHES_PER_LAUNCH  # bench.py --batches-per-launch default (6)
    pipe = cmb.BatchedPipeline(g, torch.from_numpy(b.train), B, cfg.fanouts, mode=mode, mix=k,
                               p=p, seed=SEED, nb=G)
    nb = pipe.n_batches
    order = oracle.order_roots(b.train, b.comm, cfg.num_communities, _mode(mode), k, SEED, 0)
    full_check = {0, nb // 2, nb - 1}
    workers = max(1, min(16, (os.cpu_count() or 2) - 1))
    scratch = [np.full(prep.num_nodes, -1, dtype=np.int32) for _ in range(workers)]
    free = list(range(workers))

    def verify(bb, got):
        slot = free.pop()
        try:
            ref = oracle.run_batch(prep, b.X, F, oracle.batch_roots(order, B, bb), cfg.fanouts, p,
                                   SEED, bb, scratch[slot])
        finally:
            free.append(slot)
        assert got["n"] == ref["n"] and got["e"] == ref["e"], (bb, got["n"], ref["n"])
        assert np.array_equal(got["nodes"], ref["nodes"]), bb
        for h in range(L):
            assert np.array_equal(got["indptr"][h], ref["indptr"][h]), (bb, h)
            assert np.array_equal(got["indices"][h], ref["indices"][h]), (bb, h)
        assert got["X_in"].tobytes() == ref["X_in"].tobytes(), f"X_in batch {bb}"
        assert got["H"].tobytes() == ref["H"].tobytes(), f"H batch {bb}"
        if bb in full_check:
            assert _agg_tol_ok(got["H"], ref["H64"], ref["X_in"], ref["indptr"][L - 1],
                               ref["indices"][L - 1]), f"H tolerance batch {bb}"
        return got["n"]

    sms = torch.cuda.get_device_properties(0).multi_processor_count
    vgrid = (sms - sms % G) // G  # blocks per batch in a G-batch launch (sample.cu)
    sizes = {}
    with ThreadPoolExecutor(max_workers=workers) as ex:
        futs = []
        for t0 in range(0, nb, G):
            ids = list(range(t0, min(nb, t0 + G)))
            ss = pipe.step_group(ids)          # cmb_step_group, as bench.py calls it
            torch.cuda.synchronize()
            for s in ss:
                assert s.status() == 0
            for bb, s in zip(ids, ss):
                futs.append((bb, ex.submit(verify, bb, _host_batch(s, L, F))))
            while sum(not f.done() for _, f in futs) > workers:  # bound host memory
                next(f for _, f in futs if not f.done()).result()
        for bb, f in futs:
            sizes[bb] = f.result()
    assert len(sizes) == nb and order.shape[0] % B != 0  # the ragged last batch was included
    per_block = max(-(-n[h] // vgrid) for n in sizes.values() for h in range(L))
    if mode == "rand":
        assert per_block > K_ROW_CAP, (per_block, vgrid)
