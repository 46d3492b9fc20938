"""Pins for a2, Knob-2 biased fanout sampling (S4.2 PAPER.md P:683-691; S5 P:717).

The paper fixes: per-edge unnormalised probability p (intra-community) and
1-p (inter) passed to DGL's NeighborSampler, i.e. weighted sampling WITHOUT
replacement; p = 0.5 is "equal likelihood of selecting all neighbors"
(P:691); p = 0.9 makes an intra neighbour "9 times higher";
p = 1.0 "only select[s] neighbors from the same community".

The oracle's urn + Floyd procedure is checked against the DEFINITION of
successive weighted sampling without replacement, enumerated exactly on tiny
rows (a different computation), plus textbook closed forms.  CPU only."""
import itertools

import numpy as np
import pytest
from scipy import stats

import oracle
from conftest import star_graph


def _p16(p):
    q = int(np.floor(p * 65536 + 0.5))
    return q, 65536 - q


def exact_set_law(weights, f):
    """P(selected set) under successive sampling w/o replacement, by enumerating
    every ordered draw sequence: P(i1..if) = prod_t w_it / (W - sum_{s<t} w_is)."""
    items = [i for i, w in enumerate(weights) if w > 0]
    law = {}
    for seq in itertools.permutations(items, f):
        pr, rem = 1.0, float(sum(weights))
        for i in seq:
            pr *= weights[i] / rem
            rem -= weights[i]
        key = tuple(sorted(seq))
        law[key] = law.get(key, 0.0) + pr
    return law


def _sample_sets(intra, left, right, f, p, nbatch, hop=0, law=oracle.LAW_A):
    ip, ix, comm, C, hub = star_graph(intra, left, right)
    prep = oracle.Prep(ip, ix, comm, C)
    assert prep.status == 0
    row = ix[ip[hub]: ip[hub + 1]]
    out = {}
    for b in range(nbatch):
        iph, nbr = oracle.sample_hop(prep, np.array([hub], np.int32), f, p, 42, hop, b, law)
        key = tuple(np.searchsorted(row, nbr).tolist())   # row positions of the picks
        out[key] = out.get(key, 0) + 1
    return out, row, comm, hub


def _chi2_pvalue(obs, law, n):
    keys = sorted(law)
    exp = np.array([law[k] * n for k in keys])
    o = np.array([obs.get(k, 0) for k in keys])
    assert sum(obs.get(k, 0) for k in obs if k not in law) == 0, "impossible set sampled"
    # merge tiny-expectation cells
    small = exp < 5
    if small.any():
        exp = np.append(exp[~small], exp[small].sum())
        o = np.append(o[~small], o[small].sum())
    chi2 = ((o - exp) ** 2 / exp).sum()
    return stats.chi2.sf(chi2, max(1, len(exp) - 1))


@pytest.mark.parametrize("intra,left,right,f,p", [
    (2, 2, 1, 2, 0.9), (3, 1, 2, 3, 0.9), (2, 2, 2, 2, 0.5), (3, 3, 0, 2, 0.7),
    (1, 2, 2, 3, 0.6), (4, 1, 1, 1, 0.9)])
def test_exact_without_replacement_law(intra, left, right, f, p):
    n = 20000
    obs, row, comm, hub = _sample_sets(intra, left, right, f, p, n)
    wi, wo = _p16(p)
    weights = [wi if comm[u] == comm[hub] else wo for u in row]
    law = exact_set_law(weights, f)
    assert abs(sum(law.values()) - 1) < 1e-12
    assert _chi2_pvalue(obs, law, n) > 1e-4


def test_worked_K_distribution_values():
    # (ni, no, f, p) = (3, 5, 2, 0.9): P(K = 0, 1, 2) from the enumerated law
    wi, wo = _p16(0.9)
    law = exact_set_law([wi] * 3 + [wo] * 5, 2)
    pk = np.zeros(3)
    for s, pr in law.items():
        pk[sum(1 for i in s if i < 3)] += pr
    assert np.allclose(pk, [0.020164, 0.319527, 0.660309], atol=2e-6)


def test_p05_is_uniform_hypergeometric():
    # p = 0.5: uniform f-subset, K ~ Hypergeometric(deg, ni, f); inclusion rate f/deg
    intra, left, right, f, n = 4, 3, 3, 4, 20000
    obs, row, comm, hub = _sample_sets(intra, left, right, f, 0.5, n)
    deg = len(row)
    assert all(len(k) == f for k in obs)
    incl = np.zeros(deg)
    kh = np.zeros(f + 1)
    for key, c in obs.items():
        incl[list(key)] += c
        kh[sum(1 for q in key if comm[row[q]] == comm[hub])] += c
    assert np.all(np.abs(incl / n - f / deg) < 5 * np.sqrt(f / deg * (1 - f / deg) / n))
    pmf = stats.hypergeom(deg, intra, f).pmf(np.arange(f + 1))
    sel = pmf * n >= 5
    chi2 = ((kh[sel] - pmf[sel] * n) ** 2 / (pmf[sel] * n)).sum()
    assert stats.chi2.sf(chi2, sel.sum() - 1) > 1e-4


def test_p09_nine_times_more_likely():
    # P:721 / S:225: one intra + one inter neighbour, fanout 1: P(intra) = wi/(wi+wo)
    n = 100000
    obs, row, comm, hub = _sample_sets(1, 1, 0, 1, 0.9, n)
    n_intra = sum(c for k, c in obs.items() if comm[row[k[0]]] == comm[hub])
    pi = 58982 / 65536
    assert abs(n_intra - n * pi) < 4 * np.sqrt(n * pi * (1 - pi))
    ratio = n_intra / (n - n_intra)
    assert 8.5 < ratio < 9.5


def test_p1_intra_only_and_empty_without_intra():
    obs, row, comm, hub = _sample_sets(3, 4, 4, 2, 1.0, 2000)
    assert all(comm[row[q]] == comm[hub] for k in obs for q in k)
    # fanout >= #intra at p = 1: exactly the intra neighbours
    obs, row, comm, hub = _sample_sets(3, 4, 4, 10, 1.0, 50)
    assert list(obs) == [tuple(q for q in range(len(row)) if comm[row[q]] == comm[hub])]
    # no intra neighbour at p = 1: empty sample (reading R3)
    obs, row, comm, hub = _sample_sets(0, 3, 3, 2, 1.0, 50)
    assert list(obs) == [()]


def test_full_neighbourhood_when_fanout_ge_degree():
    for p in (0.5, 0.9):
        obs, row, comm, hub = _sample_sets(3, 2, 2, 7, p, 20)
        assert list(obs) == [tuple(range(len(row)))]
        obs, row, comm, hub = _sample_sets(3, 2, 2, 8, p, 20)
        assert list(obs) == [tuple(range(len(row)))]


def _check_hop(prep, dst, f, p, iph, nbr):
    for i, v in enumerate(dst):
        row = prep.indices[prep.indptr[v]: prep.indptr[v + 1]]
        picks = nbr[iph[i]: iph[i + 1]]
        pos = np.searchsorted(row, picks)
        assert np.all(pos < row.shape[0]) and np.array_equal(row[np.minimum(pos, len(row) - 1)], picks)
        assert np.all(np.diff(pos) > 0)          # distinct, ascending position
        ni = int(prep.hi[v]) - int(prep.lo[v])
        wi, wo = _p16(p)
        m = (ni if wi else 0) + (row.shape[0] - ni if wo else 0)
        assert picks.shape[0] == min(f, m)
        intra = (pos >= prep.lo[v]) & (pos < prep.hi[v])
        if wo == 0:
            assert intra.all()
        if wi == 0:
            assert not intra.any()


@pytest.mark.parametrize("p", [0.0, 0.5, 0.9, 1.0])
def test_structural_invariants_on_graph(small_products, p):
    b = small_products
    prep = oracle.graph_prep(b)
    order = oracle.order_roots(b.train, b.comm, b.cfg.num_communities, oracle.MODE_RAND, 0, 42, 0)
    roots = oracle.batch_roots(order, 256, 0)
    blk = oracle.sample_blocks(prep, roots, (15, 10, 5), p, 42, 0)
    for h, f in enumerate((15, 10, 5)):
        dst = blk["nodes"][: blk["n"][h]]
        _check_hop(prep, dst, f, p, blk["indptr"][h], blk["nbr"][h])


def test_batch_and_hop_keying():
    # the same dst node draws independent samples per batch id and per hop (reading R11)
    a, _, _, _ = _sample_sets(5, 5, 5, 3, 0.7, 1)
    ip, ix, comm, C, hub = star_graph(5, 5, 5)
    prep = oracle.Prep(ip, ix, comm, C)
    outs = {tuple(oracle.sample_hop(prep, np.array([hub], np.int32), 3, 0.7, 42, h, b)[1])
            for h in range(3) for b in range(5)}
    assert len(outs) > 5
    # deterministic: same (seed, hop, batch) -> same picks
    x = oracle.sample_hop(prep, np.array([hub], np.int32), 3, 0.7, 42, 1, 1)[1]
    y = oracle.sample_hop(prep, np.array([hub], np.int32), 3, 0.7, 42, 1, 1)[1]
    assert np.array_equal(x, y)


# ------------------------------------------------------------------ slot law (NEXT-2 (i), R23)
def exact_slot_law(is_intra, f, p):
    """P(selected set) under the slot law, from its definition (a different computation from
    the oracle's loop): K_draw ~ Binomial(f, P16/65536) (each slot intra independently, the
    16-bit comparison being exact); K = min(K_draw, ni), kb = min(f - K_draw, no); the intra
    and inter subsets are uniform of those sizes.  Take-all when f >= ni_e + no_e."""
    from math import comb
    wi, wo = _p16(p)
    ni = sum(is_intra) if wi else 0
    no = (len(is_intra) - sum(is_intra)) if wo else 0
    elig = [i for i, x in enumerate(is_intra) if (x and wi) or (not x and wo)]
    if f >= ni + no:
        return {tuple(elig): 1.0}
    q = wi / 65536.0
    intra = [i for i, x in enumerate(is_intra) if x]
    inter = [i for i, x in enumerate(is_intra) if not x]
    law = {}
    for kd in range(f + 1):
        pk = comb(f, kd) * q ** kd * (1 - q) ** (f - kd)
        if pk == 0:
            continue
        K, kb = min(kd, ni), min(f - kd, no)
        subsets = [(a, b) for a in itertools.combinations(intra if wi else [], K)
                   for b in itertools.combinations(inter if wo else [], kb)]
        for a, b in subsets:
            key = tuple(sorted(a + b))
            law[key] = law.get(key, 0.0) + pk / len(subsets)
    return law


@pytest.mark.parametrize("intra,left,right,f,p", [
    (2, 2, 1, 2, 0.9), (3, 1, 2, 3, 0.7), (2, 2, 2, 2, 0.5), (1, 2, 2, 3, 0.6), (4, 1, 1, 3, 1.0),
    (1, 3, 2, 3, 1.0), (2, 1, 1, 3, 0.0), (3, 2, 2, 4, 0.25)])
def test_slot_law_exact(intra, left, right, f, p):
    n = 20000
    obs, row, comm, hub = _sample_sets(intra, left, right, f, p, n, law=oracle.LAW_SLOT)
    law = exact_slot_law([comm[u] == comm[hub] for u in row], f, p)
    assert abs(sum(law.values()) - 1) < 1e-12
    assert _chi2_pvalue(obs, law, n) > 1e-4


def test_slot_law_p1_returns_fewer_than_f():
    # 1 intra + 4 inter neighbours, f = 3 < m: p = 1 -> the single intra neighbour only
    obs, row, comm, hub = _sample_sets(1, 2, 2, 3, 1.0, 200, law=oracle.LAW_SLOT)
    assert list(obs) == [tuple(i for i, u in enumerate(row) if comm[u] == comm[hub])]


def test_slot_law_intra_count_is_binomial():
    # ample neighbours in both classes: #intra picks = K_draw ~ Binomial(f, P16 / 65536)
    f, p, n = 5, 0.7, 20000
    obs, row, comm, hub = _sample_sets(12, 6, 6, f, p, n, law=oracle.LAW_SLOT)
    cnt = np.zeros(f + 1)
    for key, c in obs.items():
        assert len(key) == f
        cnt[sum(comm[row[i]] == comm[hub] for i in key)] += c
    wi, _ = _p16(p)
    exp = stats.binom.pmf(np.arange(f + 1), f, wi / 65536.0) * n
    assert stats.chisquare(cnt, exp).pvalue > 1e-4


def test_slot_law_take_all_and_same_words_as_law_a():
    # f >= m: both laws take the whole eligible row; and at p = 1 with enough intra
    # neighbours both laws pick f intra positions from the same words (the urn is
    # then all-intra too), so the two laws coincide exactly there
    ip, ix, comm, C, hub = star_graph(20, 3, 3)
    prep = oracle.Prep(ip, ix, comm, C)
    d = np.array([hub], np.int32)
    for b in range(50):
        a = oracle.sample_hop(prep, d, 40, 0.7, 42, 0, b, oracle.LAW_A)
        s_ = oracle.sample_hop(prep, d, 40, 0.7, 42, 0, b, oracle.LAW_SLOT)
        assert np.array_equal(a[1], s_[1])
        a = oracle.sample_hop(prep, d, 5, 1.0, 42, 1, b, oracle.LAW_A)
        s_ = oracle.sample_hop(prep, d, 5, 1.0, 42, 1, b, oracle.LAW_SLOT)
        assert np.array_equal(a[1], s_[1])
