"""Pins for a0 (community offsets + per-row intra segment) and the generator's
input invariants (CSR symmetric/sorted/simple, community-ordered).  CPU only."""
import numpy as np
import pytest

import oracle
from gen import CONFIGS, generate, scaled


def _check_csr(b):
    n = b.num_nodes
    ip, ix = b.indptr, b.indices
    assert ip[0] == 0 and ip[-1] == ix.shape[0]
    assert np.all(np.diff(ip) >= 0)
    assert ix.min() >= 0 and ix.max() < n
    src = np.repeat(np.arange(n), np.diff(ip))
    # strictly ascending rows (sorted, no duplicates), no self-loops
    same_row = src[1:] == src[:-1]
    assert np.all(ix[1:][same_row] > ix[:-1][same_row])
    assert not np.any(src == ix)
    # symmetric: the set {(u,v)} equals {(v,u)}
    k1 = np.sort(src.astype(np.int64) * n + ix)
    k2 = np.sort(ix.astype(np.int64) * n + src)
    assert np.array_equal(k1, k2)
    # community-ordered, every community present
    assert np.all(np.diff(b.comm) >= 0)
    assert np.array_equal(np.unique(b.comm), np.arange(b.cfg.num_communities))
    # train: ascending unique, right count
    assert b.train.shape[0] == b.cfg.n_train
    assert np.all(np.diff(b.train) > 0)


@pytest.mark.parametrize("name,factor", [("tiny", None), ("arxiv", 0.05), ("products", 0.01),
                                         ("reddit", 0.02)])
def test_generator_invariants(name, factor):
    cfg = CONFIGS[name] if factor is None else scaled(CONFIGS[name], factor)
    b = generate(cfg, features=True)
    _check_csr(b)
    assert abs(b.nnz - cfg.nnz_target) / cfg.nnz_target < 0.05
    # features: exactly k*2^-23 - 1 with 0 <= k < 2^24, pad columns zero
    X = b.X[:, : cfg.feat_dim].astype(np.float64)
    k = (X + 1.0) * 2.0 ** 23
    assert np.all(k == np.round(k)) and k.min() >= 0 and k.max() < 2 ** 24
    assert np.all(b.X[:, cfg.feat_dim:] == 0)
    # determinism
    b2 = generate(cfg, features=False, cache=False)
    assert np.array_equal(b.indices, b2.indices) and np.array_equal(b.train, b2.train)


def test_generator_intra_fraction():
    cfg = scaled(CONFIGS["products"], 0.01)
    b = generate(cfg, features=False)
    # stubs stay inside the community w.p. 1 - mu, plus global stubs landing inside
    assert 0.70 < b.meta["intra_edge_fraction"] < 0.95


def test_graph_prep_brute_force(small_products):
    b = small_products
    p = oracle.graph_prep(b)
    assert p.status == 0
    cb = np.searchsorted(b.comm, np.arange(b.cfg.num_communities + 1))
    assert np.array_equal(p.cbeg, cb)
    rng = np.random.default_rng(1)
    for v in rng.integers(0, b.num_nodes, 500):
        row = b.indices[b.indptr[v]: b.indptr[v + 1]]
        c = b.comm[v]
        intra = [q for q, u in enumerate(row) if b.comm[u] == c]
        if intra:
            assert (p.lo[v], p.hi[v]) == (intra[0], intra[-1] + 1)
            assert len(intra) == intra[-1] + 1 - intra[0]   # contiguous segment
        else:
            assert p.lo[v] == p.hi[v]


def test_graph_prep_rejects_bad_input():
    from conftest import star_graph
    ip, ix, comm, C, hub = star_graph(3, 2, 2)
    assert oracle.Prep(ip, ix, comm, C).status == 0
    bad = ix.copy()
    r0, r1 = ip[hub], ip[hub + 1]
    bad[r0], bad[r0 + 1] = bad[r0 + 1], bad[r0]          # unsorted row
    assert oracle.Prep(ip, bad, comm, C).status == 1
    oob = ix.copy()
    oob[-1] = ip.shape[0] + 5                               # id out of range
    assert oracle.Prep(ip, oob, comm, C).status == 1
    unordered = comm.copy()
    unordered[0], unordered[-1] = unordered[-1], unordered[0]
    assert oracle.Prep(ip, ix, unordered, C).status == 2
    assert oracle.Prep(ip, ix, comm, C + 1).status == 2     # empty community
