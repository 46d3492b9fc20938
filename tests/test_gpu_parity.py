"""GPU parity: the CUDA path (through the C ABI) versus the oracle, element by element.

Bar (BASELINE.json north_star): bit-exact root order, sampled blocks, relabel maps
and gathered rows; aggregation within 1e-5 relative of the fp64 shadow (and, in
practice, bit-exact with the fp32 oracle because both sum in CSR order).
All tests need a B200 (-m gpu)."""
import numpy as np
import pytest
import torch

import oracle
from gen import CONFIGS, generate, scaled

pytestmark = pytest.mark.gpu

cmb = pytest.importorskip("paper_2504_18082_b200")

SEED = 42
_CACHE = {}


def _bundle(name, factor=None):
    key = (name, factor)
    if key not in _CACHE:
        cfg = CONFIGS[name] if factor is None else scaled(CONFIGS[name], factor)
        b = generate(cfg)
        _CACHE[key] = (b, oracle.graph_prep(b), cmb.Graph.from_bundle(b))
    return _CACHE[key]


def _mode(m):
    return {"rand": oracle.MODE_RAND, "norand": oracle.MODE_NORAND, "comm": oracle.MODE_COMM,
            "comm_static": oracle.MODE_COMM_STATIC}[m]


def agg_tol_ok(H, H64, Xin, ip, idx):
    deg = np.diff(ip)
    scale = np.zeros_like(H64)
    np.add.at(scale, np.repeat(np.arange(deg.shape[0]), deg), np.abs(Xin[idx]).astype(np.float64))
    scale[deg > 0] /= deg[deg > 0, None]
    return np.all(np.abs(H.astype(np.float64) - H64) <= 1e-5 * np.maximum(np.abs(H64), scale) + 1e-30)


def check_batch(bundle, prep, graph, sampler, roots_np, fanouts, p, batch_id, features=True,
                law=oracle.LAW_A):
    roots = torch.from_numpy(roots_np).cuda()
    view = sampler.sample(roots, p, SEED, batch_id, law)
    if features:
        x_in, h = sampler.gather_aggregate()
    torch.cuda.synchronize()
    assert sampler.status() == 0
    L = len(fanouts)
    if features:
        ref = oracle.run_batch(prep, bundle.X, bundle.cfg.feat_dim, roots_np, fanouts, p, SEED,
                               batch_id, law=law)
    else:
        ref = oracle.sample_blocks(prep, roots_np, fanouts, p, SEED, batch_id, law=law)
    n, e = view.host_sizes()
    assert n == ref["n"], (n, ref["n"])
    assert e == ref["e"], (e, ref["e"])
    assert np.array_equal(view.nodes[: n[L]].cpu().numpy(), ref["nodes"])
    for h_ in range(L):
        assert np.array_equal(view.indptr[h_][: n[h_] + 1].cpu().numpy().astype(np.int64),
                              ref["indptr"][h_])
        assert np.array_equal(view.indices[h_][: e[h_]].cpu().numpy(), ref["indices"][h_])
    if features:
        F = bundle.cfg.feat_dim
        xg = x_in[: n[L], :F].cpu().numpy()
        assert xg.tobytes() == ref["X_in"].tobytes(), "X_in not bit-exact"
        hg = h[: n[L - 1], :F].cpu().numpy()
        assert agg_tol_ok(hg, ref["H64"], ref["X_in"], ref["indptr"][L - 1], ref["indices"][L - 1])
        assert hg.tobytes() == ref["H"].tobytes(), "H not bit-exact with the CSR-order fp32 oracle"
    return n, e


# ------------------------------------------------------------------ a0
@pytest.mark.parametrize("name,factor", [("tiny", None), ("products", 0.01), ("arxiv", None)])
def test_graph_prep_parity(name, factor):
    b, prep, g = _bundle(name, factor)
    cbeg, bounds = g.arrays()
    torch.cuda.synchronize()
    assert g.status() == 0
    assert np.array_equal(cbeg.cpu().numpy(), prep.cbeg)
    bd = bounds.cpu().numpy().view(np.uint32)
    assert np.array_equal(bd[:, 0], prep.lo) and np.array_equal(bd[:, 1], prep.hi)


def test_load_graph_rejects_bad_input():
    from conftest import star_graph
    ip, ix, comm, C, hub = star_graph(3, 2, 2)
    cmb.Graph(ip, ix, comm, C)  # ok
    bad = ix.copy()
    bad[ip[hub]], bad[ip[hub] + 1] = bad[ip[hub] + 1], bad[ip[hub]]
    with pytest.raises(cmb.CmbError) as ei:
        cmb.Graph(ip, bad, comm, C)
    assert ei.value.code == 2
    unordered = comm.copy()
    unordered[0], unordered[-1] = unordered[-1], unordered[0]
    with pytest.raises(cmb.CmbError) as ei:
        cmb.Graph(ip, ix, unordered, C)
    assert ei.value.code == 3
    with pytest.raises(cmb.CmbError) as ei:
        cmb.Graph(ip, ix, comm, C + 1)   # empty community
    assert ei.value.code == 3


# ------------------------------------------------------------------ a1
@pytest.mark.parametrize("name,factor", [("tiny", None), ("arxiv", None), ("products", None)])
@pytest.mark.parametrize("mode,k", [("rand", 0.0), ("norand", 0.0), ("comm", 0.0),
                                    ("comm", 0.125), ("comm", 0.5), ("comm", 1.0),
                                    ("comm_static", 0.0), ("comm_static", 0.125),
                                    ("comm_static", 1.0)])
def test_order_roots_parity(name, factor, mode, k):
    b, prep, g = _bundle(name, factor)
    ro = cmb.RootOrderer(g, torch.from_numpy(b.train))
    for epoch in (0, 3):
        got = ro.order(mode, k, SEED, epoch).cpu().numpy()
        ref = oracle.order_roots(b.train, b.comm, b.cfg.num_communities, _mode(mode), k, SEED, epoch)
        assert np.array_equal(got, ref)
    assert ro.status() == 0


# ------------------------------------------------------------------ a2-a5
def test_tiny_every_batch_two_epochs():
    b, prep, g = _bundle("tiny")
    cfg = b.cfg
    s = cmb.Sampler(g, cfg.batch_size, cfg.fanouts)
    nb = (cfg.n_train + cfg.batch_size - 1) // cfg.batch_size
    for epoch in range(2):
        for mode, k in (("comm", 0.5), ("rand", 0.0)):
            order = oracle.order_roots(b.train, b.comm, cfg.num_communities, _mode(mode), k, SEED,
                                       epoch)
            for bb in range(nb):
                check_batch(b, prep, g, s, oracle.batch_roots(order, cfg.batch_size, bb),
                            cfg.fanouts, cfg.p_intra, epoch * nb + bb)


@pytest.mark.parametrize("p", [0.0, 0.5, 0.9, 1.0])
@pytest.mark.parametrize("fanouts", [(15, 10, 5), (25, 10), (1, 32), (3,)])
def test_products_scaled_knobs(p, fanouts):
    b, prep, g = _bundle("products", 0.01)
    s = cmb.Sampler(g, 512, fanouts)
    order = oracle.order_roots(b.train, b.comm, b.cfg.num_communities, oracle.MODE_COMM, 0.125,
                               SEED, 0)
    for bb in (0, 3):
        check_batch(b, prep, g, s, oracle.batch_roots(order, 512, bb), fanouts, p, bb)


@pytest.mark.parametrize("p", [0.0, 0.5, 0.9, 1.0])
@pytest.mark.parametrize("fanouts", [(15, 10, 5), (25, 10), (1, 32)])
def test_slot_law_products_scaled(p, fanouts):
    # NEXT-2 (i): the slot law (reading R23) through cmb_sample_blocks_law
    b, prep, g = _bundle("products", 0.01)
    s = cmb.Sampler(g, 512, fanouts)
    order = oracle.order_roots(b.train, b.comm, b.cfg.num_communities, oracle.MODE_COMM, 0.5,
                               SEED, 0)
    for bb in (0, 3):
        n, e = check_batch(b, prep, g, s, oracle.batch_roots(order, 512, bb), fanouts, p, bb,
                           law=oracle.LAW_SLOT)
    if p == 1.0:  # rows with fewer intra neighbours than f return short (no refill)
        assert e[0] < 512 * fanouts[0]


def test_slot_law_rejects_unknown_law():
    b, prep, g = _bundle("tiny")
    s = cmb.Sampler(g, 64, (5, 5))
    roots = torch.arange(10, dtype=torch.int32, device="cuda")
    with pytest.raises(cmb.CmbError) as ei:
        s.sample(roots, 0.9, SEED, 0, law=7)
    assert ei.value.code == 1


def test_ragged_last_batch_and_single_root():
    b, prep, g = _bundle("products", 0.01)
    s = cmb.Sampler(g, 512, (15, 10, 5))
    order = oracle.order_roots(b.train, b.comm, b.cfg.num_communities, oracle.MODE_RAND, 0, SEED, 0)
    nb = (order.shape[0] + 511) // 512
    last = oracle.batch_roots(order, 512, nb - 1)
    assert last.shape[0] < 512
    check_batch(b, prep, g, s, last, (15, 10, 5), 0.9, nb - 1)
    check_batch(b, prep, g, s, order[:1].copy(), (15, 10, 5), 0.9, 7)


def test_isolated_and_hub_rows():
    # a graph with isolated nodes (deg 0) and a hub of degree >> fanout
    from conftest import star_graph
    ip, ix, comm, C, hub = star_graph(60, 40, 45)
    n = ip.shape[0] - 1
    # append 5 isolated nodes to the last community
    ip2 = np.concatenate([ip, np.full(5, ip[-1])])
    comm2 = np.concatenate([comm, np.full(5, comm[-1], np.int32)])
    from types import SimpleNamespace
    X = np.random.default_rng(0).standard_normal((n + 5, 12)).astype(np.float32)
    cfg = SimpleNamespace(num_communities=C, feat_dim=12)
    bnd = SimpleNamespace(indptr=ip2, indices=ix, comm=comm2, X=X, cfg=cfg)
    prep = oracle.Prep(ip2, ix, comm2, C)
    g = cmb.Graph(ip2, ix, comm2, C, torch.from_numpy(X), 12)
    roots = np.array([hub, n, n + 4, 0, hub + 3], np.int32)
    for fan in ((5, 3), (32, 32), (1,)):
        s = cmb.Sampler(g, 8, fan)
        for p in (0.5, 0.9, 1.0, 0.0):
            check_batch(bnd, prep, g, s, roots, fan, p, 11)


def test_arxiv_full_size():
    b, prep, g = _bundle("arxiv")
    cfg = b.cfg
    s = cmb.Sampler(g, cfg.batch_size, cfg.fanouts)
    for mode, k in (("rand", 0.0), ("comm", 0.0)):
        order = oracle.order_roots(b.train, b.comm, cfg.num_communities, _mode(mode), k, SEED, 0)
        for bb in (0, 88):
            check_batch(b, prep, g, s, oracle.batch_roots(order, cfg.batch_size, bb), cfg.fanouts,
                        0.9, bb)


def test_products_full_size_launch_config():
    """BASELINE configs[3] at full size, one batch per sampler launch (all SMs on one batch).
    The bench's own launch configuration (4 batches per launch) is tested batch by batch over a
    whole epoch in test_gpu_headline.py."""
    b, prep, g = _bundle("products")
    cfg = b.cfg
    s = cmb.Sampler(g, cfg.batch_size, cfg.fanouts)
    for mode, k, p in (("rand", 0.0, 0.5), ("comm", 0.125, 1.0)):
        order = oracle.order_roots(b.train, b.comm, cfg.num_communities, _mode(mode), k, SEED, 0)
        check_batch(b, prep, g, s, oracle.batch_roots(order, cfg.batch_size, 5), cfg.fanouts, p, 5)


@pytest.mark.slow
def test_reddit_full_size():
    b, prep, g = _bundle("reddit")
    cfg = b.cfg
    s = cmb.Sampler(g, cfg.batch_size, cfg.fanouts)
    order = oracle.order_roots(b.train, b.comm, cfg.num_communities, oracle.MODE_COMM, 0.125, SEED, 0)
    for p in (0.5, 1.0):
        check_batch(b, prep, g, s, oracle.batch_roots(order, cfg.batch_size, 2), cfg.fanouts, p, 2)


# ------------------------------------------------------------------ unfused a4 / a5 entry points
def test_unfused_gather_and_aggregate():
    b, prep, g = _bundle("products", 0.01)
    F = b.cfg.feat_dim
    s = cmb.Sampler(g, 256, (10, 5))
    order = oracle.order_roots(b.train, b.comm, b.cfg.num_communities, oracle.MODE_RAND, 0, SEED, 1)
    roots = oracle.batch_roots(order, 256, 2)
    view = s.sample(torch.from_numpy(roots).cuda(), 0.9, SEED, 2)
    ref = oracle.run_batch(prep, b.X, F, roots, (10, 5), 0.9, SEED, 2)
    L = 2
    xin = torch.zeros(s.n_cap[L], F, device="cuda")
    cmb.gather_features(g, view.nodes, view.sizes[L: L + 1], xin)
    h = torch.zeros(s.n_cap[L - 1], F, device="cuda")
    cmb.sage_mean_aggregate(view.indptr[L - 1], view.indices[L - 1], view.sizes[L - 1: L], xin, F, h)
    # fused form reading the feature table through the relabel map
    h2 = torch.zeros(s.n_cap[L - 1], F + 4, device="cuda")
    cmb.sage_mean_aggregate(view.indptr[L - 1], view.indices[L - 1], view.sizes[L - 1: L],
                            g.features, F, h2, src_map=view.nodes)
    torch.cuda.synchronize()
    n = ref["n"]
    assert xin[: n[L]].cpu().numpy().tobytes() == ref["X_in"].tobytes()
    assert h[: n[L - 1]].cpu().numpy().tobytes() == ref["H"].tobytes()
    assert h2[: n[L - 1], :F].cpu().numpy().tobytes() == ref["H"].tobytes()
    # unaligned leading dimension -> scalar path, same bytes
    xo = torch.zeros(s.n_cap[L], F + 1, device="cuda")
    cmb.gather_features(g, view.nodes, view.sizes[L: L + 1], xo)
    torch.cuda.synchronize()
    assert xo[: n[L], :F].cpu().numpy().tobytes() == ref["X_in"].tobytes()


# ------------------------------------------------------------------ errors / determinism
def test_capacity_and_argument_errors():
    b, prep, g = _bundle("tiny")
    s = cmb.Sampler(g, 64, (5, 5))
    roots = torch.from_numpy(b.train[:64]).cuda()
    s._blocks.indices_cap[1] = 10
    with pytest.raises(cmb.CmbError) as ei:
        s.sample(roots, 0.5, SEED, 0)
    assert ei.value.code == 4
    s2 = cmb.Sampler(g, 64, (5, 5))
    with pytest.raises(cmb.CmbError) as ei:
        s2.sample(roots, 1.5, SEED, 0)
    assert ei.value.code == 1
    dup = torch.tensor([3, 5, 3], dtype=torch.int32, device="cuda")
    s2.sample(dup, 0.5, SEED, 0)
    torch.cuda.synchronize()
    assert s2.status() == 7          # duplicate roots: device-detected invalid input
    assert s2.status() == 0          # sticky word cleared by the read


def test_out_of_range_ids_are_flagged_not_followed():
    """A root id outside [0, N) (or negative) sets CMB_ERR_INVALID_INPUT and is never used as an
    address: its row samples nothing, node 0 stands in for it in the outputs, the fused gather
    stays inside the table, and the other roots' rows are unaffected.  Train ids outside [0, N)
    in the root order are flagged the same way."""
    b, prep, g = _bundle("tiny")
    cfg = b.cfg
    N = cfg.num_nodes
    s = cmb.Sampler(g, 8, (5, 5))
    good = b.train[:3].astype(np.int32)
    for bad in (N, N + 12345, -7, 2 ** 31 - 1):
        roots = np.array([good[0], bad, good[1], good[2]], dtype=np.int32)
        view = s.sample(torch.from_numpy(roots).cuda(), 0.9, SEED, 3)
        x_in, h = s.gather_aggregate()
        torch.cuda.synchronize()
        assert s.status() == 7
        n, e = view.host_sizes()
        nodes = view.nodes[: n[-1]].cpu().numpy()
        assert nodes[1] == 0 and np.all((nodes >= 0) & (nodes < N))
        ip0 = view.indptr[0][: n[0] + 1].cpu().numpy()
        assert ip0[2] - ip0[1] == 0           # the bad root's row is empty
        # the first root's picks depend only on (root, hop, batch): the oracle's, in global ids
        ref = oracle.sample_blocks(prep, good[:1], (5,), 0.9, SEED, 3)
        got = nodes[view.indices[0][: ip0[1]].cpu().numpy()]
        assert np.array_equal(got, ref["nbr"][0])
    ro = cmb.RootOrderer(g, torch.tensor([1, 5, N + 3], dtype=torch.int32))
    ro.order("comm", 0.5, SEED, 0)
    torch.cuda.synchronize()
    assert ro.status() == 7


def test_load_graph_checks_row_offsets():
    """validate=1: indptr[0] != 0 or indptr[N] != nnz (a tail past the index array) is rejected
    before any row is read."""
    from conftest import star_graph
    ip, ix, comm, C, hub = star_graph(3, 2, 2)
    bad = ip.copy()
    bad[-1] += 5                      # the last row claims entries past nnz
    with pytest.raises(cmb.CmbError) as ei:
        cmb.Graph(bad, ix, comm, C)
    assert ei.value.code == 2
    bad = ip.copy()
    bad[0] = 1
    with pytest.raises(cmb.CmbError) as ei:
        cmb.Graph(bad, ix, comm, C)
    assert ei.value.code == 2


def test_deterministic_repeat():
    b, prep, g = _bundle("products", 0.01)
    s = cmb.Sampler(g, 512, (15, 10, 5))
    roots = torch.from_numpy(b.train[:512]).cuda()
    outs = []
    for _ in range(2):
        view = s.sample(roots, 0.9, SEED, 4)
        x_in, h = s.gather_aggregate()
        torch.cuda.synchronize()
        n, e = view.host_sizes()
        outs.append((view.nodes[: n[-1]].cpu().numpy().copy(),
                     view.indices[2][: e[2]].cpu().numpy().copy(),
                     h[: n[2]].cpu().numpy().copy()))
    for a, c in zip(outs[0], outs[1]):
        assert a.tobytes() == c.tobytes()


def test_overlapped_pipeline_matches_sequential():
    """Two batches in flight on two streams (OverlappedPipeline) give the same bytes as the
    sequential pipeline (double-buffered outputs, event-ordered reuse)."""
    b, prep, g = _bundle("products", 0.01)
    cfg = b.cfg
    train = torch.from_numpy(b.train)
    seq = cmb.MiniBatchPipeline(g, train, 512, (15, 10, 5), mode="comm", mix=0.125, p=0.9)
    ov = cmb.OverlappedPipeline(g, train, 512, (15, 10, 5), mode="comm", mix=0.125, p=0.9)
    ref = []
    for t in range(6):
        view, x_in, h = seq.step(t)
        torch.cuda.synchronize()
        n, e = view.host_sizes()
        ref.append((view.nodes[: n[-1]].cpu().numpy().copy(), h[: n[2]].cpu().numpy().copy()))
    for t in range(6):
        s = ov.step(t)
        j = t % ov.depth
        ov.ev_gathered[j].synchronize()
        n = s.sizes.cpu().tolist()
        nodes = s.nodes[: n[3]].cpu().numpy()
        hh = s.h[: n[2]].cpu().numpy()
        assert nodes.tobytes() == ref[t][0].tobytes()
        assert hh.tobytes() == ref[t][1].tobytes()
    ov.join()
    torch.cuda.synchronize()
