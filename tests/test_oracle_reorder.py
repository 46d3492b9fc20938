"""Pins for NEXT-2 (iii), community reordering of a graph that is not community-ordered
(reading R25; the paper assumes community-ordered inputs).  CPU only."""
import numpy as np

import oracle
from gen import CONFIGS, generate, scaled


def _shuffled(seed=0):
    """A community-ordered synthetic graph under a random node relabelling (the input a user
    without a community-ordered file has), plus the relabelling."""
    b = generate(scaled(CONFIGS["products"], 0.002))
    n = b.num_nodes
    rng = np.random.default_rng(seed)
    new_of = rng.permutation(n).astype(np.int32)            # old (ordered) id -> shuffled id
    old_of = np.argsort(new_of).astype(np.int32)
    deg = np.diff(b.indptr)
    ip = np.zeros(n + 1, np.int64)
    np.cumsum(deg[old_of], out=ip[1:])
    ix = np.concatenate([np.sort(new_of[b.indices[b.indptr[o]: b.indptr[o + 1]]]) for o in old_of])
    return b, ip, ix.astype(np.int32), b.comm[old_of].astype(np.int32)


def _edges(ip, ix):
    src = np.repeat(np.arange(ip.shape[0] - 1), np.diff(ip))
    return set(zip(src.tolist(), ix.tolist()))


def test_reorder_is_an_isomorphism_onto_a_community_ordered_csr():
    b, ip, ix, cm = _shuffled()
    perm, inv, ip2, ix2, cm2 = oracle.community_order(ip, ix, cm)
    n = ip.shape[0] - 1
    assert np.array_equal(np.sort(perm), np.arange(n)) and np.array_equal(inv[perm], np.arange(n))
    assert np.all(np.diff(cm2) >= 0)                                    # community-ordered
    assert np.array_equal(cm2, cm[perm])
    for i in range(n):                                                  # rows sorted, simple
        r = ix2[ip2[i]: ip2[i + 1]]
        assert np.all(np.diff(r) > 0)
    # edge set maps exactly: (u, w) in the input <=> (inv[u], inv[w]) in the output
    e_in = _edges(ip, ix)
    e_out = _edges(ip2, ix2)
    assert {(int(inv[u]), int(inv[w])) for u, w in e_in} == e_out
    # ties inside a community keep the old id order
    for c in np.unique(cm2)[:50]:
        assert np.all(np.diff(perm[cm2 == c]) > 0)
    # prep accepts the output (the a0 community-order check passes)
    assert oracle.Prep(ip2, ix2, cm2, int(cm2.max()) + 1).status == 0


def test_reorder_brute_force_tiny():
    ip = np.array([0, 2, 3, 5, 6], np.int64)       # 4 nodes, communities [1, 0, 1, 0]
    ix = np.array([1, 3, 0, 0, 3, 2], np.int32)
    cm = np.array([1, 0, 1, 0], np.int32)
    perm, inv, ip2, ix2, cm2 = oracle.community_order(ip, ix, cm)
    assert perm.tolist() == [1, 3, 0, 2] and inv.tolist() == [2, 0, 3, 1]
    assert cm2.tolist() == [0, 0, 1, 1]
    # new rows: old 1 -> [0] -> {2}; old 3 -> [2] -> {3}; old 0 -> [1, 3] -> {0, 1};
    # old 2 -> [0, 3] -> {2, 1} sorted {1, 2}
    assert ip2.tolist() == [0, 1, 2, 4, 6] and ix2.tolist() == [2, 3, 0, 1, 1, 2]


def test_reorder_of_an_ordered_graph_is_the_identity():
    b = generate(scaled(CONFIGS["products"], 0.002))
    perm, inv, ip2, ix2, cm2 = oracle.community_order(b.indptr, b.indices, b.comm)
    assert np.array_equal(perm, np.arange(b.num_nodes))
    assert np.array_equal(ip2, b.indptr) and np.array_equal(ix2, b.indices)
