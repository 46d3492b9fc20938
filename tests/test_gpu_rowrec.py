"""GPU parity of the sampler's row reads through a0's packed row records (graph.cu
k_intra_bounds: row start 40 bits, degree 24 bits, lo, hi in one 16-byte record) at the record's
limit: a hub whose degree (2^24 + 7) does not fit the 24-bit degree field is stored with the
sentinel degree and read from indptr / bounds instead.  Hub and leaf rows, both Knob-2 classes,
against the oracle (which reads the CSR directly)."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu
cmb = pytest.importorskip("paper_2504_18082_b200")


def _big_star():
    """Community-ordered star: communities 0 = [0, 4), 1 = [4, 5 + I), 2 = the last 3 nodes; the
    hub (node 4) is adjacent to every other node, every other node only to the hub."""
    intra = 1 << 24
    n = 4 + 1 + intra + 3
    hub = 4
    deg = np.ones(n, dtype=np.int64)
    deg[hub] = n - 1
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(deg, out=indptr[1:])
    indices = np.full(indptr[-1], hub, dtype=np.int32)
    others = np.concatenate([np.arange(hub, dtype=np.int32), np.arange(hub + 1, n, dtype=np.int32)])
    indices[indptr[hub]:indptr[hub + 1]] = others
    comm = np.concatenate([np.zeros(4, np.int32), np.ones(1 + intra, np.int32),
                           np.full(3, 2, np.int32)])
    return indptr, indices, comm, 3, hub


def test_hub_degree_beyond_the_record_field():
    ip, ix, comm, C, hub = _big_star()
    n = ip.shape[0] - 1
    assert ip[hub + 1] - ip[hub] >= (1 << 24) - 1
    prep = oracle.Prep(ip, ix, comm, C)
    g = cmb.Graph(ip, ix, comm, C, None, None)
    roots = np.array([hub, 0, 5, n - 1, n // 2], np.int32)
    fan = (5, 3)
    s = cmb.Sampler(g, 8, fan)
    for p, bid in ((0.5, 1), (1.0, 2), (0.0, 3), (0.9, 4)):
        view = s.sample(torch.from_numpy(roots).cuda(), p, 17, bid)
        torch.cuda.synchronize()
        assert s.status() == 0
        ref = oracle.sample_blocks(prep, roots, fan, p, 17, bid)
        nn, e = view.host_sizes()
        assert nn == ref["n"] and e == ref["e"]
        assert np.array_equal(view.nodes[: nn[-1]].cpu().numpy(), ref["nodes"])
        for h in range(len(fan)):
            assert np.array_equal(view.indices[h][: e[h]].cpu().numpy(), ref["indices"][h])
            assert np.array_equal(view.indptr[h][: nn[h] + 1].cpu().numpy().astype(np.int64),
                                  ref["indptr"][h])
