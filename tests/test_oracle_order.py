"""Pins for a1, Knob-1 root ordering (Table 1; S4.1 P:653-680).

What the paper fixes: NORAND is the unshuffled training set, "static across
epochs"; RAND is a uniform shuffle; COMM-RAND-MIX shuffles
communities as whole blocks and the contents inside each (super-)block
(P:671-678).  CPU only."""
import numpy as np
import pytest
from scipy import stats

import oracle
from oracle import MODE_COMM, MODE_NORAND, MODE_RAND


def _setup(n=3000, C=37, ntr=1200, seed=0):
    rng = np.random.default_rng(seed)
    sizes = rng.integers(max(2, n // C // 2), max(3, 3 * n // C // 2), C)
    comm = np.repeat(np.arange(C, dtype=np.int32), sizes)
    train = np.sort(rng.choice(comm.shape[0], ntr, replace=False)).astype(np.int32)
    return train, comm, C


def test_norand_is_static_identity():
    train, comm, C = _setup()
    for e in range(3):
        assert np.array_equal(oracle.order_roots(train, comm, C, MODE_NORAND, epoch=e), train)


@pytest.mark.parametrize("mode,k", [(MODE_RAND, 0.0), (MODE_COMM, 0.0), (MODE_COMM, 0.125),
                                    (MODE_COMM, 0.5), (MODE_COMM, 1.0)])
def test_order_is_bijection_and_epoch_dependent(mode, k):
    train, comm, C = _setup()
    o0 = oracle.order_roots(train, comm, C, mode, k, seed=7, epoch=0)
    o1 = oracle.order_roots(train, comm, C, mode, k, seed=7, epoch=1)
    assert np.array_equal(np.sort(o0), train) and np.array_equal(np.sort(o1), train)
    assert not np.array_equal(o0, o1)        # re-randomised every epoch
    assert np.array_equal(o0, oracle.order_roots(train, comm, C, mode, k, seed=7, epoch=0))


def test_comm_k1_equals_rand_bitwise():
    # one super-block holding every training community == uniform shuffle (reading R10)
    train, comm, C = _setup()
    for e in range(4):
        assert np.array_equal(oracle.order_roots(train, comm, C, MODE_COMM, 1.0, 3, e),
                              oracle.order_roots(train, comm, C, MODE_RAND, 0.0, 3, e))


def _superblocks(order, comm):
    """Merge the position spans of every community; returns list of sets of communities."""
    c = comm[order]
    spans = {}
    for pos, cc in enumerate(c):
        lo, hi = spans.get(cc, (pos, pos))
        spans[cc] = (min(lo, pos), max(hi, pos))
    iv = sorted((lo, hi, cc) for cc, (lo, hi) in spans.items())
    groups, cur, end = [], set(), -1
    for lo, hi, cc in iv:
        if lo > end and cur:
            groups.append(cur)
            cur = set()
        cur.add(cc)
        end = max(end, hi)
    groups.append(cur)
    return groups


@pytest.mark.parametrize("k", [0.0, 0.125, 0.25, 0.5])
def test_comm_superblock_structure(k):
    train, comm, C = _setup(n=20000, C=40, ntr=8000, seed=3)
    c_tr = np.unique(comm[train]).shape[0]
    S = max(1, int(np.floor(k * c_tr + 0.5)))
    for e in range(3):
        o = oracle.order_roots(train, comm, C, MODE_COMM, k, 11, e)
        groups = _superblocks(o, comm)
        sizes = [len(g) for g in groups]
        # consecutive super-blocks of exactly S communities (the last may be smaller)
        assert all(s == S for s in sizes[:-1]) and 1 <= sizes[-1] <= S, sizes
        assert sum(sizes) == c_tr


def test_comm_mix0_community_of_size_B_gives_single_community_batches():
    # k = 0 and every training community holds exactly B nodes
    B, C = 16, 12
    comm = np.repeat(np.arange(C, dtype=np.int32), B)
    train = np.arange(C * B, dtype=np.int32)
    for e in range(5):
        o = oracle.order_roots(train, comm, C, MODE_COMM, 0.0, 5, e)
        for b in range(C):
            assert np.unique(comm[oracle.batch_roots(o, B, b)]).shape[0] == 1


@pytest.mark.parametrize("mode,k", [(MODE_RAND, 0.0), (MODE_COMM, 1.0)])
def test_batch_index_uniform_chi2(mode, k):
    # with one super-block each node's batch index is uniform over batches
    train, comm, C = _setup(n=200, C=5, ntr=40, seed=4)
    B, nb, E = 8, 5, 3000
    counts = np.zeros((train.shape[0], nb), dtype=np.int64)
    pos_of = {v: i for i, v in enumerate(train)}
    for e in range(E):
        o = oracle.order_roots(train, comm, C, mode, k, 99, e)
        for pos, v in enumerate(o):
            counts[pos_of[v], pos // B] += 1
    chi2 = ((counts - E / nb) ** 2 / (E / nb)).sum()
    dof = train.shape[0] * (nb - 1)
    assert stats.chi2.sf(chi2, dof) > 1e-3, chi2


def test_comm_mix0_within_block_uniform_chi2():
    # contents of each community are shuffled uniformly
    C, size = 3, 6
    comm = np.repeat(np.arange(C, dtype=np.int32), size)
    train = np.arange(C * size, dtype=np.int32)
    E = 3000
    counts = np.zeros((C * size, size), dtype=np.int64)
    firsts = np.zeros(C, dtype=np.int64)
    for e in range(E):
        o = oracle.order_roots(train, comm, C, MODE_COMM, 0.0, 1, e)
        firsts[comm[o[0]]] += 1
        for pos, v in enumerate(o):
            counts[v, pos % size] += 1
    chi2 = ((counts - E / size) ** 2 / (E / size)).sum()
    assert stats.chi2.sf(chi2, C * size * (size - 1)) > 1e-3
    # communities are shuffled as whole blocks: the first block is uniform over communities
    chi2c = ((firsts - E / C) ** 2 / (E / C)).sum()
    assert stats.chi2.sf(chi2c, C - 1) > 1e-3


def test_train_communities_only():
    # communities without training nodes do not change the super-block size
    train, comm, C = _setup(n=3000, C=37, ntr=1200, seed=0)
    keep = comm[train] < 20
    tr = train[keep]
    a = oracle.order_roots(tr, comm, C, MODE_COMM, 0.25, 5, 0)
    groups = _superblocks(a, comm)
    S = max(1, int(np.floor(0.25 * 20 + 0.5)))
    assert all(len(g) == S for g in groups[:-1])


# ------------------------------------------------------------------ static super-blocks (R24)
from oracle import MODE_COMM_STATIC  # noqa: E402


@pytest.mark.parametrize("k", [0.0, 0.1, 0.25, 0.5])
def test_static_superblocks_are_adjacent_runs(k):
    """Each super-block is a contiguous run of the order holding the train nodes of S
    communities that are ADJACENT in id order (the same groups every epoch), and inside a run
    the nodes follow the RAND order restricted to them (same node keys)."""
    train, comm, C = _setup()
    ctr_ids = np.unique(comm[train])                  # train communities, ascending
    S = max(1, int(np.floor(k * ctr_ids.shape[0] + 0.5)))
    group = {c: j // S for j, c in enumerate(ctr_ids)}
    for epoch in (0, 1, 2):
        o = oracle.order_roots(train, comm, C, MODE_COMM_STATIC, k, seed=11, epoch=epoch)
        r = oracle.order_roots(train, comm, C, MODE_RAND, 0.0, seed=11, epoch=epoch)
        assert np.array_equal(np.sort(o), train)
        g = np.array([group[c] for c in comm[o]])
        runs = g[np.r_[True, g[1:] != g[:-1]]]
        assert len(runs) == len(set(runs.tolist())) == len(set(group.values()))  # contiguous
        pos_in_rand = {v: i for i, v in enumerate(r.tolist())}
        for b in set(runs.tolist()):
            run = o[g == b]
            assert np.all(np.diff([pos_in_rand[v] for v in run.tolist()]) > 0)
    o0 = oracle.order_roots(train, comm, C, MODE_COMM_STATIC, k, seed=11, epoch=0)
    o1 = oracle.order_roots(train, comm, C, MODE_COMM_STATIC, k, seed=11, epoch=1)
    assert not np.array_equal(o0, o1)


def test_static_k1_equals_rand_bitwise():
    train, comm, C = _setup()
    for e in range(3):
        assert np.array_equal(oracle.order_roots(train, comm, C, MODE_COMM_STATIC, 1.0, 5, e),
                              oracle.order_roots(train, comm, C, MODE_RAND, 0.0, 5, e))


def test_static_superblock_order_is_uniform_chi2():
    """The super-block sequence is a uniformly random permutation: the position of super-block
    0 among nsb super-blocks is uniform over epochs."""
    train, comm, C = _setup()
    ctr_ids = np.unique(comm[train])
    S = 5
    k = S / ctr_ids.shape[0]
    group = {c: j // S for j, c in enumerate(ctr_ids)}
    nsb = (ctr_ids.shape[0] + S - 1) // S
    cnt = np.zeros(nsb)
    for e in range(1500):
        o = oracle.order_roots(train, comm, C, MODE_COMM_STATIC, k, seed=3, epoch=e)
        g = np.array([group[c] for c in comm[o]])
        runs = g[np.r_[True, g[1:] != g[:-1]]]
        cnt[int(np.nonzero(runs == 0)[0][0])] += 1
    assert stats.chisquare(cnt).pvalue > 1e-4
