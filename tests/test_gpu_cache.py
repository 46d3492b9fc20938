"""NEXT-3: the HBM feature cache over a pinned host table (cmb_cache_gather_aggregate).

The bytes never depend on the cache: X_in and H equal the oracle on every batch, whether the
rows come from hits or from misses read over the host link, and the hit/miss counters obey the
cache's own invariants (first touch = all misses, an immediate repeat = no misses, a cache of
exactly one batch keeps missing on new batches)."""
import numpy as np
import pytest
import torch

import oracle
from gen import CONFIGS, generate, scaled

pytestmark = pytest.mark.gpu
cmb = pytest.importorskip("paper_2504_18082_b200")
SEED = 42


@pytest.fixture(scope="module")
def env():
    b = generate(scaled(CONFIGS["products"], 0.01))
    prep = oracle.graph_prep(b)
    g = cmb.Graph.from_bundle(b, features=False)
    host = torch.from_numpy(b.X).pin_memory()
    order = oracle.order_roots(b.train, b.comm, b.cfg.num_communities, oracle.MODE_RAND, 0, SEED, 0)
    return b, prep, g, host, order


def _run(b, prep, s, cache, roots, bid):
    cfg = b.cfg
    L = len(cfg.fanouts)
    view = s.sample(torch.from_numpy(roots).cuda(), cfg.p_intra, SEED, bid)
    before = cache.stats.clone()
    x_in, h = s.gather_aggregate_cached(cache)
    torch.cuda.synchronize()
    assert s.status() == 0
    n, _ = view.host_sizes()
    ref = oracle.run_batch(prep, b.X, cfg.feat_dim, roots, cfg.fanouts, cfg.p_intra, SEED, bid)
    F = cfg.feat_dim
    assert x_in[: n[L], :F].cpu().numpy().tobytes() == ref["X_in"].tobytes()
    assert h[: n[L - 1], :F].cpu().numpy().tobytes() == ref["H"].tobytes()
    d = (cache.stats - before).tolist()
    assert d[0] == n[L]
    return d[1], n[L]


def test_cache_bytes_and_counters(env):
    b, prep, g, host, order = env
    cfg = b.cfg
    s = cmb.Sampler(g, cfg.batch_size, cfg.fanouts)
    big = cmb.FeatureCache(g, host, cfg.feat_dim, capacity=cfg.num_nodes,
                           max_rows=s.n_cap[-1], max_edges=s.e_cap[-1])
    r0 = oracle.batch_roots(order, cfg.batch_size, 0)
    m, u = _run(b, prep, s, big, r0, 0)
    assert m == u                                   # cold cache: every row misses
    m, u = _run(b, prep, s, big, r0, 0)
    assert m == 0                                   # the same batch again: all hits
    r1 = oracle.batch_roots(order, cfg.batch_size, 1)
    m1, u1 = _run(b, prep, s, big, r1, 1)
    assert 0 < m1 < u1                              # overlap with batch 0 hits


def test_small_cache_evicts_and_stays_exact(env):
    b, prep, g, host, order = env
    cfg = b.cfg
    s = cmb.Sampler(g, cfg.batch_size, cfg.fanouts)
    small = cmb.FeatureCache(g, host, cfg.feat_dim, capacity=s.n_cap[-1],
                             max_rows=s.n_cap[-1], max_edges=s.e_cap[-1])
    for bid in (0, 1, 0, 1):
        m, u = _run(b, prep, s, small, oracle.batch_roots(order, cfg.batch_size, bid), bid)
        assert 0 <= m <= u
    assert small.miss_rate() > 0


def test_cache_rejects_oversized_batch(env):
    b, prep, g, host, order = env
    cfg = b.cfg
    s = cmb.Sampler(g, cfg.batch_size, cfg.fanouts)
    tiny = cmb.FeatureCache(g, host, cfg.feat_dim, capacity=16, max_rows=16, max_edges=16)
    s.sample(torch.from_numpy(oracle.batch_roots(order, cfg.batch_size, 0)).cuda(), cfg.p_intra,
             SEED, 0)
    with pytest.raises(cmb.CmbError) as ei:
        s.gather_aggregate_cached(tiny)
    assert ei.value.code == 1
