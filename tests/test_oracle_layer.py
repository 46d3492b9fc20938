"""Pins for the oracle's first SAGEConv layer (NEXT-4, reading R26; Eq. (1)
in the GraphSAGE-mean form of its footnote; GraphSAGE trained with hidden dim 256,
P:770-774).  CPU only: a hand-computed worked example (tests/golden/), the special cases that
reduce the layer to a copy of X_dst or of H, an explicit-loop brute force on tiny inputs, the
linearity / ReLU / column-permutation laws, and the composition with the C oracle's a5 mean."""
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "sage_layer_worked.txt")


def _golden():
    out = {}
    with open(GOLD) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            key, rest = line.split(None, 1)
            rows = [[float(t) for t in r.split()] for r in rest.split(";")]
            out[key] = np.array(rows if len(rows) > 1 else rows[0], dtype=np.float64)
    return out


def test_worked_example():
    g = _golden()
    y = oracle.sage_conv(g["X_dst"], g["H"], g["W_self"], g["W_neigh"], g["bias"], relu=False)
    assert np.array_equal(y, g["Y_linear"])
    y = oracle.sage_conv(g["X_dst"], g["H"], g["W_self"], g["W_neigh"], g["bias"], relu=True)
    assert np.array_equal(y, g["Y_relu"])


def test_special_cases_reduce_to_copies():
    rng = np.random.default_rng(1)
    n, F = 37, 11
    X = rng.standard_normal((n, F))
    H = rng.standard_normal((n, F))
    eye, zero = np.eye(F), np.zeros((F, F))
    assert np.array_equal(oracle.sage_conv(X, H, eye, zero), X)      # self path only
    assert np.array_equal(oracle.sage_conv(X, H, zero, eye), H)      # neighbour path only
    # a unit column picks one feature of each path: Y[:, 0] = X[:, 3] + H[:, 5]
    ws, wn = np.zeros((F, 2)), np.zeros((F, 2))
    ws[3, 0] = 1.0
    wn[5, 0] = 1.0
    wn[7, 1] = -2.0
    y = oracle.sage_conv(X, H, ws, wn, bias=np.array([0.0, 0.25]))
    assert np.array_equal(y[:, 0], X[:, 3] + H[:, 5])
    assert np.array_equal(y[:, 1], -2.0 * H[:, 7] + 0.25)


def test_brute_force_loops():
    rng = np.random.default_rng(2)
    for trial in range(5):
        n, F, Fo = int(rng.integers(1, 6)), int(rng.integers(1, 7)), int(rng.integers(1, 5))
        X, H = rng.standard_normal((n, F)), rng.standard_normal((n, F))
        Ws, Wn = rng.standard_normal((F, Fo)), rng.standard_normal((F, Fo))
        b = rng.standard_normal(Fo)
        y = oracle.sage_conv(X, H, Ws, Wn, b, relu=True)
        for d in range(n):
            for o in range(Fo):
                s = b[o]
                for f in range(F):
                    s += X[d, f] * Ws[f, o]
                for f in range(F):
                    s += H[d, f] * Wn[f, o]
                assert abs(y[d, o] - max(s, 0.0)) <= 1e-12 * (1 + abs(s))


def test_linearity_relu_and_permutation():
    rng = np.random.default_rng(3)
    n, F, Fo = 50, 9, 6
    X, H = rng.standard_normal((n, F)), rng.standard_normal((n, F))
    Ws, Wn = rng.standard_normal((F, Fo)), rng.standard_normal((F, Fo))
    b = rng.standard_normal(Fo)
    y = oracle.sage_conv(X, H, Ws, Wn, b)
    # linear in the weights (exact for a power-of-two scale), additive in the bias
    assert np.array_equal(oracle.sage_conv(X, H, 4 * Ws, 4 * Wn, 4 * b), 4 * y)
    assert np.allclose(oracle.sage_conv(X, H, Ws, Wn), y - b[None, :], rtol=0, atol=1e-12)
    # ReLU is max(0, .) of the linear output
    assert np.array_equal(oracle.sage_conv(X, H, Ws, Wn, b, relu=True), np.maximum(y, 0))
    # permuting output columns of the weights permutes Y's columns (no transposed operand)
    perm = rng.permutation(Fo)
    assert np.array_equal(oracle.sage_conv(X, H, Ws[:, perm], Wn[:, perm], b[perm]), y[:, perm])
    # swapping the two paths swaps the roles of X_dst and H
    assert np.array_equal(oracle.sage_conv(H, X, Wn, Ws, b), y)


def test_composes_with_a5_mean(tiny_prep, tiny_bundle):
    """W_self = 0, W_neigh = I returns the C oracle's fp64 a5 mean of the input-side block."""
    from gen import CONFIGS
    cfg = CONFIGS["tiny"]
    order = oracle.order_roots(tiny_bundle.train, tiny_bundle.comm, cfg.num_communities,
                               oracle.MODE_RAND, 0.0, 7, 0)
    roots = oracle.batch_roots(order, cfg.batch_size, 0)
    ref = oracle.run_batch(tiny_prep, tiny_bundle.X, cfg.feat_dim, roots, cfg.fanouts,
                           cfg.p_intra, 7, 0)
    L = len(cfg.fanouts)
    nd = ref["n"][L - 1]
    F = cfg.feat_dim
    y = oracle.sage_conv(ref["X_in"][:nd], ref["H64"], np.zeros((F, F)), np.eye(F))
    assert np.array_equal(y, ref["H64"])
    y = oracle.sage_conv(ref["X_in"][:nd], ref["H64"], np.eye(F), np.zeros((F, F)))
    assert np.array_equal(y, ref["X_in"][:nd].astype(np.float64))


# ---------------------------------------------------------------- backward (reading R27)
def _loss(X, H, Ws, Wn, b, G, relu):
    """L = sum(G * Y): dL/dY = G, so its gradient in W is what sage_conv_backward returns."""
    return float(np.sum(G * oracle.sage_conv(X, H, Ws, Wn, b, relu=relu)))


@pytest.mark.parametrize("relu", [False, True])
def test_backward_matches_finite_differences(relu):
    """Central differences of the forward oracle (exact for the linear layer up to rounding; for
    ReLU away from the kinks) -- a check that does not reuse the transpose formula."""
    rng = np.random.default_rng(5)
    n, F, Fo = 12, 5, 4
    X, H = rng.standard_normal((n, F)), rng.standard_normal((n, F))
    Ws, Wn, b = rng.standard_normal((F, Fo)), rng.standard_normal((F, Fo)), rng.standard_normal(Fo)
    G = rng.standard_normal((n, Fo))
    Y = oracle.sage_conv(X, H, Ws, Wn, b, relu=relu)
    dWs, dWn, db = oracle.sage_conv_backward(X, H, G, Y, relu=relu)
    eps = 1e-6
    for (W, dW) in ((Ws, dWs), (Wn, dWn)):
        for i in range(F):
            for j in range(Fo):
                W[i, j] += eps
                lp = _loss(X, H, Ws, Wn, b, G, relu)
                W[i, j] -= 2 * eps
                lm = _loss(X, H, Ws, Wn, b, G, relu)
                W[i, j] += eps
                assert abs((lp - lm) / (2 * eps) - dW[i, j]) <= 1e-6 * (1 + abs(dW[i, j]))
    for j in range(Fo):
        b[j] += eps
        lp = _loss(X, H, Ws, Wn, b, G, relu)
        b[j] -= 2 * eps
        lm = _loss(X, H, Ws, Wn, b, G, relu)
        b[j] += eps
        assert abs((lp - lm) / (2 * eps) - db[j]) <= 1e-6 * (1 + abs(db[j]))


def test_backward_worked_example():
    """Hand arithmetic on the golden layer: with dY = ones and no activation,
    dW_self[f, o] = sum_d X_dst[d, f] = [0, 2.5], dW_neigh[f, o] = sum_d H[d, f] = [2.5, 1],
    db = [2, 2, 2] (n = 2 rows)."""
    g = _golden()
    dY = np.ones((2, 3))
    dWs, dWn, db = oracle.sage_conv_backward(g["X_dst"], g["H"], dY)
    assert np.array_equal(dWs, np.array([[0.0] * 3, [2.5] * 3]))
    assert np.array_equal(dWn, np.array([[2.5] * 3, [1.0] * 3]))
    assert np.array_equal(db, np.array([2.0, 2.0, 2.0]))
    # ReLU masks the rows whose output is not positive: Y_relu has zeros at (0,2) and (1,1)
    dWs, dWn, db = oracle.sage_conv_backward(g["X_dst"], g["H"], dY, g["Y_relu"], relu=True)
    assert np.array_equal(db, np.array([2.0, 1.0, 1.0]))
    assert np.array_equal(dWs[:, 2], np.array([-1.0, 0.5]))   # only row 1 contributes to col 2
    assert np.array_equal(dWn[:, 1], np.array([0.5, -1.0]))   # only row 0 contributes to col 1


# ---------------------------------------------------------------- GCN variant (reading R28)
def test_gcn_worked_example():
    """Block with 2 dst nodes over 4 src nodes: row 0 has edges to src 2 and 3, row 1 none.
    Hand arithmetic: A' row 0 = (X0 + X2 + X3) / 3 = ([1,2] + [3,0] + [2,1]) / 3 = [2, 1];
    A' row 1 = X1 / 1 = [-1, 4].  W = [[1, 0, 2], [0, 1, -1]], b = [0, 0, 1]:
    Y0 = [2, 1, 4 - 1 + 1] = [2, 1, 4], Y1 = [-1, 4, -2 - 4 + 1] = [-1, 4, -5]."""
    X = np.array([[1, 2], [-1, 4], [3, 0], [2, 1]], dtype=np.float64)
    W = np.array([[1, 0, 2], [0, 1, -1]], dtype=np.float64)
    y = oracle.gcn_conv([0, 2, 2], [2, 3], X, W, bias=[0, 0, 1])
    assert np.array_equal(y, np.array([[2, 1, 4], [-1, 4, -5]], dtype=np.float64))
    assert np.array_equal(oracle.gcn_conv([0, 2, 2], [2, 3], X, W, bias=[0, 0, 1], relu=True),
                          np.array([[2, 1, 4], [0, 4, 0]], dtype=np.float64))


def test_gcn_brute_force_and_identities(tiny_prep, tiny_bundle):
    from gen import CONFIGS
    cfg = CONFIGS["tiny"]
    order = oracle.order_roots(tiny_bundle.train, tiny_bundle.comm, cfg.num_communities,
                               oracle.MODE_RAND, 0.0, 3, 0)
    ref = oracle.run_batch(tiny_prep, tiny_bundle.X, cfg.feat_dim,
                           oracle.batch_roots(order, cfg.batch_size, 0), cfg.fanouts,
                           cfg.p_intra, 3, 0)
    L = len(cfg.fanouts)
    ip, ix, X = ref["indptr"][L - 1], ref["indices"][L - 1], ref["X_in"].astype(np.float64)
    nd, F = ip.shape[0] - 1, cfg.feat_dim
    rng = np.random.default_rng(8)
    W = rng.standard_normal((F, 6))
    y = oracle.gcn_conv(ip, ix, X, W)
    for d in range(0, nd, 17):   # explicit loops over a sample of rows
        row = X[d].copy()
        for e in range(ip[d], ip[d + 1]):
            row = row + X[ix[e]]
        row = row / (ip[d + 1] - ip[d] + 1)
        assert np.allclose(y[d], row @ W, rtol=1e-12, atol=1e-12)
    # W = I: every output row is the mean over the node and its sampled neighbours
    yi = oracle.gcn_conv(ip, ix, X, np.eye(F))
    deg = np.diff(ip)
    H64 = ref["H64"]
    assert np.allclose(yi, (X[:nd] + deg[:, None] * H64) / (deg[:, None] + 1), rtol=1e-12, atol=1e-12)
    # rows of equal degree k: GCN(W) == SAGE(W_self = W/(k+1), W_neigh = k W/(k+1)) on them
    for k in np.unique(deg):
        rows = np.nonzero(deg == k)[0]
        ys = oracle.sage_conv(X[rows], H64[rows], W / (k + 1), k * W / (k + 1))
        assert np.allclose(y[rows], ys, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("relu", [False, True])
def test_gcn_backward_matches_finite_differences(tiny_prep, tiny_bundle, relu):
    """GCN weight gradients (reading R35) against central differences of the GCN forward oracle
    (gcn_conv) on a real sampled block -- the transpose formula is not reused."""
    from gen import CONFIGS
    cfg = CONFIGS["tiny"]
    order = oracle.order_roots(tiny_bundle.train, tiny_bundle.comm, cfg.num_communities,
                               oracle.MODE_COMM, 0.5, 4, 0)
    ref = oracle.run_batch(tiny_prep, tiny_bundle.X, cfg.feat_dim,
                           oracle.batch_roots(order, cfg.batch_size, 1), cfg.fanouts,
                           cfg.p_intra, 4, 1)
    L = len(cfg.fanouts)
    ip, ix, X = ref["indptr"][L - 1], ref["indices"][L - 1], ref["X_in"].astype(np.float64)
    nd, F, Fo = ip.shape[0] - 1, cfg.feat_dim, 5
    rng = np.random.default_rng(11)
    W, b, Gup = rng.standard_normal((F, Fo)), rng.standard_normal(Fo), rng.standard_normal((nd, Fo))
    Y = oracle.gcn_conv(ip, ix, X, W, b, relu=relu)
    dW, db = oracle.gcn_conv_backward(ip, ix, X, Gup, Y, relu=relu)

    def loss():
        return float(np.sum(Gup * oracle.gcn_conv(ip, ix, X, W, b, relu=relu)))

    eps = 1e-6
    for i in range(0, F, 3):
        for j in range(Fo):
            W[i, j] += eps
            lp = loss()
            W[i, j] -= 2 * eps
            lm = loss()
            W[i, j] += eps
            assert abs((lp - lm) / (2 * eps) - dW[i, j]) <= 1e-6 * (1 + abs(dW[i, j]))
    for j in range(Fo):
        b[j] += eps
        lp = loss()
        b[j] -= 2 * eps
        lm = loss()
        b[j] += eps
        assert abs((lp - lm) / (2 * eps) - db[j]) <= 1e-6 * (1 + abs(db[j]))


def test_gcn_backward_worked_example():
    """The worked block of test_gcn_worked_example: A' X = [[2, 1], [-1, 4]].  With dY = ones:
    dW = (A'X)^T 1 = [[1, 1, 1], [5, 5, 5]], db = [2, 2, 2].  With the ReLU outputs
    Y = [[2, 1, 4], [0, 4, 0]] only (0, *) and (1, 1) pass: dW = [[2, 1, 2], [1, 5, 1]],
    db = [1, 2, 1]."""
    X = np.array([[1, 2], [-1, 4], [3, 0], [2, 1]], dtype=np.float64)
    dW, db = oracle.gcn_conv_backward([0, 2, 2], [2, 3], X, np.ones((2, 3)))
    assert np.array_equal(dW, np.array([[1, 1, 1], [5, 5, 5]], dtype=np.float64))
    assert np.array_equal(db, np.array([2, 2, 2], dtype=np.float64))
    Y = np.array([[2, 1, 4], [0, 4, 0]], dtype=np.float64)
    dW, db = oracle.gcn_conv_backward([0, 2, 2], [2, 3], X, np.ones((2, 3)), Y, relu=True)
    assert np.array_equal(dW, np.array([[2, 1, 2], [1, 5, 1]], dtype=np.float64))
    assert np.array_equal(db, np.array([1, 2, 1], dtype=np.float64))


def test_sage_mean64_matches_the_c_oracle(tiny_prep, tiny_bundle):
    """The numpy fp64 mean used for the hidden layers (R29) equals the C oracle's fp64 shadow of
    a5 on the same (fp32) inputs, including empty rows."""
    from gen import CONFIGS
    cfg = CONFIGS["tiny"]
    order = oracle.order_roots(tiny_bundle.train, tiny_bundle.comm, cfg.num_communities,
                               oracle.MODE_NORAND, 0.0, 5, 0)
    ref = oracle.run_batch(tiny_prep, tiny_bundle.X, cfg.feat_dim,
                           oracle.batch_roots(order, cfg.batch_size, 0), cfg.fanouts, 1.0, 5, 0)
    for h in range(len(cfg.fanouts)):
        ip, ix = ref["indptr"][h], ref["indices"][h]
        Xs = ref["X_in"][: ref["n"][h + 1]]
        _, h64 = oracle.sage_mean(ip, ix, Xs)
        assert np.array_equal(oracle.sage_mean64(ip, ix, Xs), h64)
    assert np.array_equal(oracle.sage_mean64([0, 0, 2], [1, 2], np.array([[1.0], [2.0], [6.0]])),
                          np.array([[0.0], [4.0]]))


# ---------------------------------------------------------------- a5 backward (reading R30)
def test_mean_backward_is_the_adjoint(tiny_prep, tiny_bundle):
    """<mean(X), G> == <X, mean^T(G)> for random X, G on real sampled blocks of every hop -- the
    defining property of the transposed-block scatter-add, independent of how either side sums."""
    from gen import CONFIGS
    cfg = CONFIGS["tiny"]
    order = oracle.order_roots(tiny_bundle.train, tiny_bundle.comm, cfg.num_communities,
                               oracle.MODE_RAND, 0.0, 9, 0)
    ref = oracle.sample_blocks(tiny_prep, oracle.batch_roots(order, cfg.batch_size, 0),
                               cfg.fanouts, 0.7, 9, 0)
    rng = np.random.default_rng(4)
    for h in range(len(cfg.fanouts)):
        ip, ix = ref["indptr"][h], ref["indices"][h]
        n_src, n_dst = ref["n"][h + 1], ref["n"][h]
        X = rng.standard_normal((n_src, 7))
        G = rng.standard_normal((n_dst, 7))
        lhs = np.sum(oracle.sage_mean64(ip, ix, X) * G)
        rhs = np.sum(X * oracle.sage_mean_backward(ip, ix, G, n_src))
        assert abs(lhs - rhs) <= 1e-10 * (1 + abs(lhs))


def test_mean_backward_worked_example():
    """Rows: d0 -> {1, 2}, d1 -> {2}, d2 -> {} over 4 src rows; dH = [[2], [3], [5]]:
    dX[1] = 2/2 = 1, dX[2] = 2/2 + 3/1 = 4, dX[0] = dX[3] = 0 (d2 has no edges)."""
    dX = oracle.sage_mean_backward([0, 2, 3, 3], [1, 2, 2], np.array([[2.0], [3.0], [5.0]]), 4)
    assert np.array_equal(dX, np.array([[0.0], [1.0], [4.0], [0.0]]))


# ---------------------------------------------------------------- hidden backward (reading R31)
@pytest.mark.parametrize("relu", [False, True])
def test_hidden_backward_matches_finite_differences(tiny_prep, tiny_bundle, relu):
    """R31: the weight gradients of a hidden layer are R27's on (Yp[0:n_dst], mean of Yp over the
    hop's block).  Central differences of the hidden forward chain (sage_mean64 -> sage_conv)
    on a real sampled block of the tiny graph, a check that does not reuse the transpose."""
    from gen import CONFIGS
    cfg = CONFIGS["tiny"]
    order = oracle.order_roots(tiny_bundle.train, tiny_bundle.comm, cfg.num_communities,
                               oracle.MODE_RAND, 0.0, 7, 0)
    roots = oracle.batch_roots(order, cfg.batch_size, 0)
    blk = oracle.sample_blocks(tiny_prep, roots, cfg.fanouts, cfg.p_intra, 7, 0)
    h = 0
    ip, ix = blk["indptr"][h], blk["indices"][h]
    nd, ns = blk["n"][h], blk["n"][h + 1]
    rng = np.random.default_rng(11)
    Fin, Fo = 3, 2
    Yp = rng.standard_normal((ns, Fin))
    Ws, Wn, b = rng.standard_normal((Fin, Fo)), rng.standard_normal((Fin, Fo)), rng.standard_normal(Fo)
    G = rng.standard_normal((nd, Fo))

    def loss():
        Y = oracle.sage_conv(Yp[:nd], oracle.sage_mean64(ip, ix, Yp), Ws, Wn, b, relu=relu)
        return float(np.sum(G * Y))

    H = oracle.sage_mean64(ip, ix, Yp)
    Y = oracle.sage_conv(Yp[:nd], H, Ws, Wn, b, relu=relu)
    dWs, dWn, db = oracle.sage_conv_backward(Yp[:nd], H, G, Y, relu=relu)
    eps = 1e-6
    for W, dW in ((Ws, dWs), (Wn, dWn)):
        for i in range(Fin):
            for j in range(Fo):
                W[i, j] += eps
                lp = loss()
                W[i, j] -= 2 * eps
                lm = loss()
                W[i, j] += eps
                assert abs((lp - lm) / (2 * eps) - dW[i, j]) <= 1e-6 * (1 + abs(dW[i, j]))
    for j in range(Fo):
        b[j] += eps
        lp = loss()
        b[j] -= 2 * eps
        lm = loss()
        b[j] += eps
        assert abs((lp - lm) / (2 * eps) - db[j]) <= 1e-6 * (1 + abs(db[j]))


# ---------------------------------------------------------------- hidden input gradient (R32)
@pytest.mark.parametrize("relu", [False, True])
def test_hidden_input_grad_matches_finite_differences(tiny_prep, tiny_bundle, relu):
    """R32: dYp of L = sum(G * sigma(Yp[:nd] W_self + mean(Yp) W_neigh + b)) by central
    differences in every entry of Yp on a real sampled block (hop 1 of tiny: shared and unused
    src rows, an independent check of both the prefix path and the transposed block)."""
    from gen import CONFIGS
    cfg = CONFIGS["tiny"]
    order = oracle.order_roots(tiny_bundle.train, tiny_bundle.comm, cfg.num_communities,
                               oracle.MODE_RAND, 0.0, 7, 0)
    roots = oracle.batch_roots(order, cfg.batch_size, 0)[:6]
    blk = oracle.sample_blocks(tiny_prep, roots, cfg.fanouts, cfg.p_intra, 7, 0)
    h = 1
    ip, ix = blk["indptr"][h], blk["indices"][h]
    nd, ns = blk["n"][h], blk["n"][h + 1]
    rng = np.random.default_rng(13)
    Fin, Fo = 2, 3
    Yp = rng.standard_normal((ns + 2, Fin))   # two rows past n_src: no gradient may reach them
    Ws, Wn, b = rng.standard_normal((Fin, Fo)), rng.standard_normal((Fin, Fo)), rng.standard_normal(Fo)
    G = rng.standard_normal((nd, Fo))

    def fwd():
        return oracle.sage_conv(Yp[:nd], oracle.sage_mean64(ip, ix, Yp[:ns]), Ws, Wn, b, relu=relu)

    Y = fwd()
    dZ = G * (Y > 0) if relu else G
    dX = oracle.sage_hidden_input_grad(ip, ix, dZ, Ws, Wn, ns)
    assert dX.shape == (ns, Fin)
    eps = 1e-6
    for i in range(ns + 2):
        for j in range(Fin):
            Yp[i, j] += eps
            lp = float(np.sum(G * fwd()))
            Yp[i, j] -= 2 * eps
            lm = float(np.sum(G * fwd()))
            Yp[i, j] += eps
            want = dX[i, j] if i < ns else 0.0
            assert abs((lp - lm) / (2 * eps) - want) <= 1e-6 * (1 + abs(want)), (i, j)
