"""Pins for a3 (dedup + relabel, Alg. 1 "Build sub-graph S_i"),
a4 (input-feature gather) and a5 (GraphSAGE mean aggregation, P:512,
P:770), plus the method-level footprint trend.  CPU only."""
import numpy as np
import pytest

import oracle


def brute_relabel(prefix, nbr):
    """First-occurrence order with a Python dict (reading R8)."""
    m = {int(u): i for i, u in enumerate(prefix)}
    nodes = [int(u) for u in prefix]
    local = []
    for u in nbr:
        u = int(u)
        if u not in m:
            m[u] = len(nodes)
            nodes.append(u)
        local.append(m[u])
    return np.array(nodes, np.int32), np.array(local, np.int32)


def test_relabel_brute_force():
    rng = np.random.default_rng(0)
    for trial in range(50):
        N = int(rng.integers(5, 300))
        nd = int(rng.integers(1, min(N, 40) + 1))
        prefix = rng.choice(N, nd, replace=False).astype(np.int32)
        nbr = rng.integers(0, N, int(rng.integers(0, 200))).astype(np.int32)
        nodes, local = oracle.relabel_hop(prefix, nbr, N)
        bn, bl = brute_relabel(prefix, nbr)
        assert np.array_equal(nodes, bn) and np.array_equal(local, bl)
        # invariants: dst prefix kept, dense injective map, global(local) == nbr
        assert np.array_equal(nodes[:nd], prefix)
        assert np.unique(nodes).shape[0] == nodes.shape[0]
        assert np.array_equal(nodes[local], nbr)


def test_blocks_invariants(small_products):
    b = small_products
    prep = oracle.graph_prep(b)
    order = oracle.order_roots(b.train, b.comm, b.cfg.num_communities, oracle.MODE_COMM, 0.125, 42, 0)
    roots = oracle.batch_roots(order, 512, 3)
    blk = oracle.sample_blocks(prep, roots, (15, 10, 5), 0.9, 42, 3)
    nodes = blk["nodes"]
    assert np.array_equal(nodes[: roots.shape[0]], roots)
    assert np.unique(nodes).shape[0] == nodes.shape[0]
    for h in range(3):
        n_h, n_next = blk["n"][h], blk["n"][h + 1]
        loc = blk["indices"][h]
        assert loc.shape[0] == blk["e"][h] == blk["indptr"][h][-1]
        assert blk["indptr"][h].shape[0] == n_h + 1
        assert loc.max(initial=0) < n_next
        assert np.array_equal(nodes[loc], blk["nbr"][h])
        # every new node of hop h is referenced by hop h (no phantom nodes)
        assert np.unique(loc[loc >= n_h]).shape[0] == n_next - n_h


def test_gather_is_row_copy(small_products):
    b = small_products
    rng = np.random.default_rng(2)
    nodes = rng.choice(b.num_nodes, 777, replace=False).astype(np.int32)
    out = oracle.gather(nodes, b.X, b.cfg.feat_dim)
    assert out.tobytes() == np.ascontiguousarray(b.X[nodes, : b.cfg.feat_dim]).tobytes()


def test_sage_mean_closed_forms():
    rng = np.random.default_rng(3)
    F = 37
    Xs = rng.standard_normal((50, F)).astype(np.float32)
    # rows: deg 0, deg 1, deg 2 (equal rows: x+x and /2 are exact in fp32), deg 7 (random)
    rows = [[], [5], [9, 9], list(rng.integers(0, 50, 7))]
    ip = np.zeros(len(rows) + 1, np.int64)
    ip[1:] = np.cumsum([len(r) for r in rows])
    idx = np.array(sum(rows, []), np.int32)
    H, H64 = oracle.sage_mean(ip, idx, Xs)
    assert np.all(H[0] == 0)                                  # empty row -> 0
    assert np.array_equal(H[1], Xs[5])                        # deg 1 -> exact copy
    assert np.array_equal(H[2], Xs[9])                        # (x + x) / 2 == x exactly
    ref = Xs[rows[3]].astype(np.float64).mean(axis=0)         # fp64 closed form
    assert np.allclose(H64[3], ref, rtol=0, atol=1e-12)
    tol = 1e-5 * np.maximum(np.abs(ref), np.abs(Xs[rows[3]]).astype(np.float64).mean(axis=0))
    assert np.all(np.abs(H[3] - ref) <= tol)
    # src_map form reads X[src_map[idx]] (the fused reading)
    smap = rng.permutation(50).astype(np.int32)
    inv = np.argsort(smap)
    Hm, _ = oracle.sage_mean(ip, inv[idx].astype(np.int32), Xs, src_map=smap)
    assert np.array_equal(Hm, H)


def test_sage_mean_on_batch_within_tolerance(small_products):
    b = small_products
    prep = oracle.graph_prep(b)
    order = oracle.order_roots(b.train, b.comm, b.cfg.num_communities, oracle.MODE_RAND, 0, 42, 0)
    out = oracle.run_batch(prep, b.X, b.cfg.feat_dim, oracle.batch_roots(order, 256, 0),
                           (15, 10, 5), 0.5, 42, 0)
    L = 3
    ip, idx, Xin = out["indptr"][L - 1], out["indices"][L - 1], out["X_in"]
    assert Xin.shape[0] == out["n"][L]
    deg = np.diff(ip)
    ref = np.zeros((ip.shape[0] - 1, Xin.shape[1]))
    np.add.at(ref, np.repeat(np.arange(deg.shape[0]), deg), Xin[idx].astype(np.float64))
    ref[deg > 0] /= deg[deg > 0, None]
    assert np.allclose(out["H64"], ref, rtol=1e-12, atol=1e-12)
    scale = np.zeros_like(ref)
    np.add.at(scale, np.repeat(np.arange(deg.shape[0]), deg), np.abs(Xin[idx]).astype(np.float64))
    scale[deg > 0] /= deg[deg > 0, None]
    assert np.all(np.abs(out["H"] - ref) <= 1e-5 * np.maximum(np.abs(ref), scale) + 1e-30)


@pytest.mark.slow
def test_footprint_trend_with_knobs(small_products):
    """the input-feature footprint falls as community bias rises.
    Mean U (unique input rows per batch) is non-increasing in p and along
    RAND -> MIX-50 -> MIX-12.5 -> MIX-0 -> NORAND (sign test over seeds)."""
    b = small_products
    prep = oracle.graph_prep(b)
    C = b.cfg.num_communities
    fan = (10, 10, 5)
    B = 256
    pol = [(oracle.MODE_RAND, 0), (oracle.MODE_COMM, 0.5), (oracle.MODE_COMM, 0.125),
           (oracle.MODE_COMM, 0.0), (oracle.MODE_NORAND, 0)]

    def mean_U(mode, k, p, seed):
        o = oracle.order_roots(b.train, b.comm, C, mode, k, seed, 0)
        us = [oracle.sample_blocks(prep, oracle.batch_roots(o, B, bb), fan, p, seed, bb)["n"][-1]
              for bb in range(3)]
        return float(np.mean(us))

    wins = 0
    total = 0
    for seed in range(6):
        u = [mean_U(m, k, 0.5, seed) for m, k in pol]
        wins += sum(u[i] >= u[i + 1] for i in range(len(u) - 1))
        total += len(u) - 1
        up = [mean_U(oracle.MODE_RAND, 0, p, seed) for p in (0.5, 0.9, 1.0)]
        wins += sum(up[i] >= up[i + 1] for i in range(2))
        total += 2
    # sign test: far more non-increasing steps than chance
    from scipy import stats
    assert stats.binomtest(wins, total, 0.5, alternative="greater").pvalue < 1e-3
