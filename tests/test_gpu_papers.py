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


@pytest.mark.skipif(os.environ.get("CMB_TEST_PAPERS") == "0", reason="CMB_TEST_PAPERS=0")
def test_papers_community_order_beyond_int32():
    """NEXT-2 (iii) at papers100M scale (3.2G CSR entries > 2^31 - 1: the row sort runs in
    chunks).  Input: the community-ordered graph with its two halves (split at a community
    boundary) swapped -- node v of the first half becomes v + |B|, of the second v - |A| -- so
    the communities are out of order and every row's neighbour ids are unsorted.  Reading R25
    (new order = (community, old id)) must give back the original graph exactly: perm = the
    swap, indptr / indices / communities identical to the generated ones."""
    cfg = CONFIGS["papers100m"]
    b = generate(cfg, features=False)
    n, nnz, C = cfg.num_nodes, int(b.indptr[-1]), cfg.num_communities
    assert nnz > 2 ** 31
    cut = int(np.searchsorted(b.comm, C // 2))       # first node of community C/2
    e0 = int(b.indptr[cut])
    dev = torch.device("cuda")
    ip = torch.from_numpy(b.indptr).to(dev)
    ix = torch.from_numpy(b.indices).to(dev)
    cm = torch.from_numpy(b.comm).to(dev)
    nb_ = n - cut                                      # |B|
    ip_in = torch.cat([ip[cut:] - e0, ip[1:cut + 1] + (nnz - e0)])
    cm_in = torch.cat([cm[cut:], cm[:cut]])
    ix_in = torch.cat([ix[e0:], ix[:e0]])
    step = 1 << 28
    for s0 in range(0, nnz, step):                     # rename in place, chunk by chunk
        t = ix_in[s0:s0 + step]
        t.copy_(torch.where(t < cut, t + nb_, t - cut))
    perm, inv, ip2, ix2, cm2 = cmb.community_order(ip_in, ix_in, cm_in, C, device=dev)
    torch.cuda.synchronize()
    want_perm = torch.cat([torch.arange(nb_, n, device=dev), torch.arange(0, nb_, device=dev)])
    assert torch.equal(perm.long(), want_perm)
    assert torch.equal(ip2, ip) and torch.equal(cm2, cm)
    assert torch.equal(ix2, ix)
