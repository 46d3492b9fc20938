import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long CPU test")


@pytest.fixture(scope="session")
def tiny_bundle():
    from gen import CONFIGS, generate
    return generate(CONFIGS["tiny"])


@pytest.fixture(scope="session")
def tiny_prep(tiny_bundle):
    import oracle
    p = oracle.graph_prep(tiny_bundle)
    assert p.status == 0
    return p


@pytest.fixture(scope="session")
def small_products():
    """products-shaped graph at 1/100 scale (24K nodes, mean degree ~50)."""
    from gen import CONFIGS, generate, scaled
    return generate(scaled(CONFIGS["products"], 0.01), features=True)


def star_graph(intra, inter_left, inter_right=0):
    """Community-ordered CSR whose hub node h has `intra` neighbours in its own
    community (community 1) and `inter_left` / `inter_right` neighbours in the
    communities before / after it, so the hub's intra segment sits strictly
    inside its sorted row.  Returns (indptr, indices, comm, num_comm, hub)."""
    nl, nr = max(inter_left, 1), max(inter_right, 1)
    hub = nl
    n = nl + 1 + intra + nr
    comm = np.array([0] * nl + [1] * (1 + intra) + [2] * nr, dtype=np.int32)
    nbrs = list(range(inter_left)) + list(range(hub + 1, hub + 1 + intra)) + \
        list(range(hub + 1 + intra, hub + 1 + intra + inter_right))
    adj = {v: set() for v in range(n)}
    for u in nbrs:
        adj[hub].add(u)
        adj[u].add(hub)
    indptr = np.zeros(n + 1, dtype=np.int64)
    idx = []
    for v in range(n):
        row = sorted(adj[v])
        idx.extend(row)
        indptr[v + 1] = indptr[v] + len(row)
    return indptr, np.array(idx, dtype=np.int32), comm, 3, hub
