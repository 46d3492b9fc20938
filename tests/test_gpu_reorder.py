"""NEXT-2 (iii) on the GPU: cmb_community_order against the oracle (bit-exact permutation and
CSR), then the relabelled graph runs the whole path against the oracle on the same relabelling."""
import numpy as np
import pytest
import torch

import oracle
from test_oracle_reorder import _shuffled

pytestmark = pytest.mark.gpu
cmb = pytest.importorskip("paper_2504_18082_b200")
SEED = 42


@pytest.mark.parametrize("seed", [0, 1])
def test_community_order_matches_oracle(seed):
    b, ip, ix, cm = _shuffled(seed)
    C = b.cfg.num_communities
    ref = oracle.community_order(ip, ix, cm)
    got = [t.cpu().numpy() for t in cmb.community_order(ip, ix, cm, C)]
    for r, g_ in zip(ref, got):
        assert np.array_equal(r.astype(np.int64), g_.astype(np.int64))


def test_reordered_graph_runs_the_path():
    b, ip, ix, cm = _shuffled(2)
    C = b.cfg.num_communities
    perm, inv, ip2, ix2, cm2 = cmb.community_order(ip, ix, cm, C)
    perm_h = perm.cpu().numpy()
    # features and train set follow the relabelling: shuffled id s holds original row old_of[s]
    n = ip.shape[0] - 1
    rng = np.random.default_rng(2)
    new_of = rng.permutation(n).astype(np.int32)
    old_of = np.argsort(new_of)
    X_shuf = b.X[old_of]
    X2 = np.ascontiguousarray(X_shuf[perm_h])
    train_shuf = np.sort(new_of[b.train]).astype(np.int32)
    train2 = np.sort(inv.cpu().numpy()[train_shuf]).astype(np.int32)
    g = cmb.Graph(ip2, ix2, cm2, C, torch.from_numpy(X2), b.cfg.feat_dim)
    prep = oracle.Prep(ip2.cpu().numpy(), ix2.cpu().numpy(), cm2.cpu().numpy(), C)
    assert prep.status == 0
    order = oracle.order_roots(train2, cm2.cpu().numpy(), C, oracle.MODE_COMM, 0.25, SEED, 0)
    s = cmb.Sampler(g, 256, (10, 5))
    roots = oracle.batch_roots(order, 256, 1)
    view = s.sample(torch.from_numpy(roots).cuda(), 0.9, SEED, 1)
    x_in, h = s.gather_aggregate()
    torch.cuda.synchronize()
    ref = oracle.run_batch(prep, X2, b.cfg.feat_dim, roots, (10, 5), 0.9, SEED, 1)
    nn, _ = view.host_sizes()
    assert nn == ref["n"]
    assert np.array_equal(view.nodes[: nn[2]].cpu().numpy(), ref["nodes"])
    F = b.cfg.feat_dim
    assert x_in[: nn[2], :F].cpu().numpy().tobytes() == ref["X_in"].tobytes()
    assert h[: nn[1], :F].cpu().numpy().tobytes() == ref["H"].tobytes()
