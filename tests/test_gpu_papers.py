"""papers100M-shaped parity (BASELINE.json configs[4]) on one GPU, graph and features replicated.

The feature table is generated on the GPU (gen.device, 57 GB at full size); the oracle's rows
come from the same counter formula on the host (gen.planted.feature_rows), so X_in[i] must equal
X[nodes[i]] byte for byte and H must equal the oracle's CSR-order fp32 mean.

* ``test_papers_scaled`` (default): 1 % of the nodes, same degree / mu / F / fanouts.
* ``test_papers_full`` (default; ~4 min, mostly generation): the full 111M-node, 3.2G-entry
  CSR -- positions beyond 2^31 exercise the int64 CSR offsets of every kernel -- batches
  compared in full (blocks, X_in, H).  CMB_TEST_PAPERS=0 skips it."""
import os

import numpy as np
import pytest
import torch

import oracle
from gen import CONFIGS, generate, scaled
from gen.device import feature_table
from gen.planted import feature_rows

pytestmark = pytest.mark.gpu
cmb = pytest.importorskip("paper_2504_18082_b200")
SEED = 42


def _check(bundle, prep, graph, roots_np, p, batch_id):
    cfg = bundle.cfg
    L = len(cfg.fanouts)
    s = cmb.Sampler(graph, cfg.batch_size, cfg.fanouts)
    view = s.sample(torch.from_numpy(roots_np).cuda(), p, SEED, batch_id)
    x_in, h = s.gather_aggregate()
    torch.cuda.synchronize()
    assert s.status() == 0
    ref = oracle.sample_blocks(prep, roots_np, cfg.fanouts, p, SEED, batch_id)
    n, e = view.host_sizes()
    assert n == ref["n"] and e == ref["e"]
    assert np.array_equal(view.nodes[: n[L]].cpu().numpy(), ref["nodes"])
    for hh in range(L):
        assert np.array_equal(view.indptr[hh][: n[hh] + 1].cpu().numpy().astype(np.int64),
                              ref["indptr"][hh])
        assert np.array_equal(view.indices[hh][: e[hh]].cpu().numpy(), ref["indices"][hh])
    F = cfg.feat_dim
    xin_ref = np.ascontiguousarray(feature_rows(bundle, ref["nodes"]))
    assert x_in[: n[L], :F].cpu().numpy().tobytes() == xin_ref.tobytes()
    H, _ = oracle.sage_mean(ref["indptr"][L - 1], ref["indices"][L - 1], xin_ref, F)
    assert h[: n[L - 1], :F].cpu().numpy().tobytes() == H.tobytes()
    return n, e


def _run(cfg, batches):
    b = generate(cfg)
    assert b.X is None and cfg.device_features
    prep = oracle.graph_prep(b)
    g = cmb.Graph.from_bundle(b, features=feature_table(b, "cuda"))
    order = oracle.order_roots(b.train, b.comm, cfg.num_communities, oracle.MODE_RAND, 0.0, SEED, 0)
    out = []
    for bb, p in batches:
        out.append(_check(b, prep, g, oracle.batch_roots(order, cfg.batch_size, bb), p, bb))
    return b, out


def test_papers_scaled():
    _run(scaled(CONFIGS["papers100m"], 0.01), [(0, 0.5), (5, 1.0)])


@pytest.mark.skipif(os.environ.get("CMB_TEST_PAPERS") == "0", reason="CMB_TEST_PAPERS=0")
def test_papers_full():
    b, out = _run(CONFIGS["papers100m"], [(3, 0.5)])
    assert b.indptr[-1] > 2 ** 31  # the int64 CSR offsets are exercised
    n, e = out[0]
    print("papers100M batch 3: n =", n, "e =", e)
