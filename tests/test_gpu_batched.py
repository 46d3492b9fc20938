"""GPU parity of the multi-batch sampler launch (cmb_sample_blocks_multi) and of the
BatchedPipeline: several batches per launch give the same bytes as one batch per launch,
and both match the oracle."""
import numpy as np
import pytest
import torch

import oracle
from gen import CONFIGS, generate, scaled

pytestmark = pytest.mark.gpu
cmb = pytest.importorskip("paper_2504_18082_b200")

SEED = 42


@pytest.fixture(scope="module")
def small():
    b = generate(scaled(CONFIGS["products"], 0.01))
    return b, oracle.graph_prep(b), cmb.Graph.from_bundle(b)


@pytest.mark.parametrize("nb,law", [(2, 0), (3, 0), (4, 0), (4, 1)])
def test_sample_multi_matches_oracle(small, nb, law):
    b, prep, g = small
    fan = (15, 10, 5)
    order = oracle.order_roots(b.train, b.comm, b.cfg.num_communities, oracle.MODE_RAND, 0, SEED, 0)
    samplers = [cmb.Sampler(g, 256, fan) for _ in range(nb)]
    roots = [torch.from_numpy(oracle.batch_roots(order, 256 - 37 * i, i)).cuda() for i in range(nb)]
    ids = [100 + i for i in range(nb)]
    for rep in range(2):  # a second launch reuses the workspaces (tagged dedup maps)
        views = cmb.sample_multi(samplers, roots, ids, 0.9, SEED, law)
        torch.cuda.synchronize()
        for s, v, r, bid in zip(samplers, views, roots, ids):
            assert s.status() == 0
            ref = oracle.sample_blocks(prep, r.cpu().numpy(), fan, 0.9, SEED, bid, law=law)
            n, e = v.host_sizes()
            assert n == ref["n"] and e == ref["e"]
            assert np.array_equal(v.nodes[: n[-1]].cpu().numpy(), ref["nodes"])
            for h in range(3):
                assert np.array_equal(v.indices[h][: e[h]].cpu().numpy(), ref["indices"][h])
                assert np.array_equal(v.indptr[h][: n[h] + 1].cpu().numpy().astype(np.int64),
                                      ref["indptr"][h])


def test_batched_pipeline_matches_sequential(small):
    b, prep, g = small
    train = torch.from_numpy(b.train)
    seq = cmb.MiniBatchPipeline(g, train, 512, (15, 10, 5), mode="comm", mix=0.125, p=1.0)
    bat = cmb.BatchedPipeline(g, train, 512, (15, 10, 5), mode="comm", mix=0.125, p=1.0, nb=2)
    nbat = seq.n_batches
    first = nbat - 1  # the group straddles an epoch boundary
    ref = []
    for t in (first, first + 1):
        view, x_in, h = seq.step(t)
        torch.cuda.synchronize()
        n, e = view.host_sizes()
        ref.append((view.nodes[: n[-1]].cpu().numpy().copy(), x_in[: n[-1]].cpu().numpy().copy(),
                    h[: n[2]].cpu().numpy().copy()))
    ss = bat.step_group([first, first + 1])
    torch.cuda.synchronize()
    for s, (nodes, xin, hh) in zip(ss, ref):
        n = s.sizes.cpu().tolist()
        assert s.nodes[: n[3]].cpu().numpy().tobytes() == nodes.tobytes()
        assert s.x_in[: n[3]].cpu().numpy().tobytes() == xin.tobytes()
        assert s.h[: n[2]].cpu().numpy().tobytes() == hh.tobytes()


@pytest.mark.parametrize("nb", [1, 4])
def test_dst_order_is_a_bucketed_permutation(small, nb):
    """cmb_blocks.dst_order: the sampler writes a permutation of the last hop's dst rows whose
    node ids (v >> s, s = max(0, bits(N) - 12)) are non-decreasing by bucket; the fused gather's
    bytes do not depend on it (checked against the natural order)."""
    b, prep, g = small
    fan = (15, 10, 5)
    L = len(fan)
    order = oracle.order_roots(b.train, b.comm, b.cfg.num_communities, oracle.MODE_RAND, 0, SEED, 0)
    samplers = [cmb.Sampler(g, 256, fan) for _ in range(nb)]
    roots = [torch.from_numpy(oracle.batch_roots(order, 256, i)).cuda() for i in range(nb)]
    cmb.sample_multi(samplers, roots, list(range(nb)), 0.9, SEED)
    torch.cuda.synchronize()
    N = b.cfg.num_nodes
    shift = max(0, int(N - 1).bit_length() - 12)
    for s in samplers:
        assert s.status() == 0
        n = int(s.sizes[L - 1].item())
        o = s.dst_order[:n].cpu().numpy()
        assert np.array_equal(np.sort(o), np.arange(n))
        bucket = s.nodes[:n].cpu().numpy()[o] >> shift
        assert np.all(np.diff(bucket) >= 0)
        x1, h1 = (t.clone() for t in s.gather_aggregate())
        s.set_dst_order(False)
        x0, h0 = s.gather_aggregate()
        s.set_dst_order(True)
        torch.cuda.synchronize()
        nl = int(s.sizes[L].item())
        assert torch.equal(x0[:nl], x1[:nl]) and torch.equal(h0[:n], h1[:n])


def test_step_group_unaligned_rows_fall_back_per_batch():
    """cmb_step_group with feature rows that are not 16-byte multiples (F = ld = 15): the
    one-launch gather needs vector rows, so each batch goes through cmb_gather_aggregate's
    scalar path -- same bytes as the oracle."""
    from gen import CONFIGS
    b = generate(CONFIGS["tiny"])
    F = 15
    X = np.ascontiguousarray(b.X[:, :F])
    g = cmb.Graph(b.indptr, b.indices, b.comm, b.cfg.num_communities, torch.from_numpy(X), F)
    prep = oracle.graph_prep(b)
    pipe = cmb.BatchedPipeline(g, torch.from_numpy(b.train), 64, (5, 5), mode="rand", p=0.9,
                               nb=3)
    ss = pipe.step_group([0, 1, 2])
    torch.cuda.synchronize()
    order = oracle.order_roots(b.train, b.comm, b.cfg.num_communities, oracle.MODE_RAND, 0.0,
                               42, 0)
    for bb, s in enumerate(ss):
        assert s.status() == 0
        ref = oracle.run_batch(prep, X, F, oracle.batch_roots(order, 64, bb), (5, 5), 0.9, 42, bb)
        n = s.sizes.cpu().tolist()
        assert s.x_in[: n[2], :F].cpu().numpy().tobytes() == ref["X_in"].tobytes()
        assert s.h[: n[1], :F].cpu().numpy().tobytes() == ref["H"].tobytes()
