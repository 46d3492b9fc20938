"""GPU parity of the sampler's tagged dedup map across its word layouts
(sample_persist.cuh MapWord): the 32-bit words' 7-bit batch tag wraps after 127 batches on one
workspace (the wrapping batch clears the map), and a workspace alternating between batches that
need 64-bit words (an id or edge position of the batch's capacity >= 2^24) and batches that fit
32-bit words is cleared on every switch.  Every checked batch must equal the oracle
(oracle.sample_blocks, which has no map at all: it dedups with a dictionary)."""
import numpy as np
import pytest
import torch

import oracle
from gen import CONFIGS, generate, scaled

pytestmark = pytest.mark.gpu
cmb = pytest.importorskip("paper_2504_18082_b200")

SEED = 7


def _check(view, ref, L):
    n, e = view.host_sizes()
    assert n == ref["n"] and e == ref["e"]
    assert np.array_equal(view.nodes[: n[L]].cpu().numpy(), ref["nodes"])
    for h in range(L):
        assert np.array_equal(view.indices[h][: e[h]].cpu().numpy(), ref["indices"][h])
        assert np.array_equal(view.indptr[h][: n[h] + 1].cpu().numpy().astype(np.int64),
                              ref["indptr"][h])


def test_tag_wrap_every_127_batches():
    b = generate(scaled(CONFIGS["products"], 0.01))
    prep = oracle.graph_prep(b)
    g = cmb.Graph.from_bundle(b)
    fan = (15, 10, 5)
    s = cmb.Sampler(g, 256, fan)
    order = oracle.order_roots(b.train, b.comm, b.cfg.num_communities, oracle.MODE_RAND, 0, SEED, 0)
    nb = len(order) // 256
    check = {0, 1, 125, 126, 127, 128, 129, 252, 253, 254, 255, 256, 299}
    for t in range(300):  # batch t runs with counter t + 1: tags wrap (and clear) at t = 127, 254
        roots_np = oracle.batch_roots(order, 256, t % nb)
        view = s.sample(torch.from_numpy(roots_np).cuda(), 0.9, SEED, t)
        if t in check:
            torch.cuda.synchronize()
            assert s.status() == 0
            ref = oracle.sample_blocks(prep, roots_np, fan, 0.9, SEED, t)
            _check(view, ref, len(fan))


def test_wide_and_narrow_words_share_a_workspace():
    b = generate(scaled(CONFIGS["products"], 0.3), features=False)
    prep = oracle.graph_prep(b)
    g = cmb.Graph.from_bundle(b, features=False)
    fan = (32, 32)
    big = 25000
    n_cap, e_cap = cmb.blocks_capacity(big, fan, g.num_nodes)
    assert max(e_cap) >= 1 << 24, "the big batch must need 64-bit map words"
    n_cap_s, e_cap_s = cmb.blocks_capacity(300, fan, g.num_nodes)
    assert max(max(e_cap_s), n_cap_s[-1]) < (1 << 24) - 1, "the small batch fits 32-bit words"
    s = cmb.Sampler(g, big, fan)
    order = oracle.order_roots(b.train, b.comm, b.cfg.num_communities, oracle.MODE_RAND, 0, SEED, 0)
    assert len(order) >= 2 * big
    seq = [(big, 0), (300, 1), (300, 2), (big, 3), (big, 4), (300, 5)]
    for n_roots, t in seq:
        roots_np = order[t * 400: t * 400 + n_roots] if n_roots < big else \
            order[(t % 2) * big:(t % 2 + 1) * big]
        roots_np = np.ascontiguousarray(roots_np, dtype=np.int32)
        view = s.sample(torch.from_numpy(roots_np).cuda(), 0.7, SEED, t)
        torch.cuda.synchronize()
        assert s.status() == 0
        ref = oracle.sample_blocks(prep, roots_np, fan, 0.7, SEED, t)
        _check(view, ref, len(fan))
