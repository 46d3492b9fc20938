"""GPU parity of NEXT-4, the input-side SAGEConv-mean layer fused with a4 + a5 on the tensor cores
(cmb_sage_layer_forward, reading R26), through the C ABI, against oracle.sage_conv on the
oracle's own blocks, X_in and fp64 H.

Bound (R26, derived from the arithmetic): bf16 operands (2^-9 relative each), fp32 accumulation
over K <= 256 terms, optional bf16 output:
    |Y_gpu - Y| <= 2^-7 * S + 2^-8 * |Y| (bf16 out),  S = |X_dst||W_self| + |H||W_neigh| + |b|.
With bf16-representable features and weights and W_neigh = 0 the operands are exact and only fp32
accumulation is left: 2^-16 * S."""
import copy

import numpy as np
import pytest
import torch

import oracle
from gen import CONFIGS, generate, scaled

pytestmark = pytest.mark.gpu

cmb = pytest.importorskip("paper_2504_18082_b200")

SEED = 42
_CACHE = {}


def _bundle(name, factor=None):
    key = (name, factor)
    if key not in _CACHE:
        cfg = CONFIGS[name] if factor is None else scaled(CONFIGS[name], factor)
        b = generate(cfg)
        _CACHE[key] = (b, oracle.graph_prep(b), cmb.Graph.from_bundle(b))
    return _CACHE[key]


def _weights(F, fo, seed, bf16_exact=False):
    g = torch.Generator().manual_seed(seed)
    ws = torch.randn(F, fo, generator=g) / np.sqrt(F)
    wn = torch.randn(F, fo, generator=g) / np.sqrt(F)
    b = torch.randn(fo, generator=g) * 0.1
    if bf16_exact:
        ws, wn, b = (t.to(torch.bfloat16).float() for t in (ws, wn, b))
    return ws, wn, b


def _run(bundle, prep, graph, fanouts, roots_np, batch_id, layer, p):
    sampler = cmb.Sampler(graph, len(roots_np), fanouts)
    sampler.sample(torch.from_numpy(roots_np).cuda(), p, SEED, batch_id)
    y = sampler.sage_layer(layer)
    torch.cuda.synchronize()
    assert sampler.status() == 0
    ref = oracle.run_batch(prep, bundle.X, bundle.cfg.feat_dim, roots_np, fanouts, p, SEED,
                           batch_id)
    L = len(fanouts)
    nd = ref["n"][L - 1]
    return y[:nd].float().cpu().numpy().astype(np.float64), ref, nd


def _check(yg, ref, nd, F, ws, wn, b, relu, out_bf16, exact=False):
    Xd = ref["X_in"][:nd, :F].astype(np.float64)
    H = ref["H64"][:, :F]
    Y = oracle.sage_conv(Xd, H, ws.double().numpy(), wn.double().numpy(), b.double().numpy(),
                         relu=relu)
    S = np.abs(Xd) @ np.abs(ws.double().numpy()) + np.abs(H) @ np.abs(wn.double().numpy()) + \
        np.abs(b.double().numpy())[None, :]
    tol = (2.0 ** -16 if exact else 2.0 ** -7) * S + (2.0 ** -8 * np.abs(Y) if out_bf16 else 0.0)
    err = np.abs(yg - Y)
    bad = err > tol + 1e-30
    assert not bad.any(), (f"{bad.sum()} of {bad.size} outside the R26 bound; worst "
                           f"{np.max(err - tol)} at {np.unravel_index(np.argmax(err - tol), err.shape)}")
    return float(np.max(err / np.maximum(S, 1e-30)))


@pytest.mark.parametrize("name,factor,fo,relu,out_bf16", [
    ("tiny", None, 256, True, False),        # F = 16: one swizzle atom per half
    ("tiny", None, 48, False, False),        # narrow N, no activation
    ("products", 0.01, 256, True, False),    # F = 100: two atoms per half, ragged F and tail
    ("products", 0.01, 128, False, True),    # bf16 output
    ("arxiv", None, 256, True, True),        # F = 128: full K = 256
])
def test_layer_parity(name, factor, fo, relu, out_bf16):
    b, prep, g = _bundle(name, factor)
    cfg = b.cfg
    F = cfg.feat_dim
    ws, wn, bias = _weights(F, fo, 7)
    layer = cmb.SageLayer(ws, wn, bias, relu=relu, out_bf16=out_bf16)
    order = oracle.order_roots(b.train, b.comm, cfg.num_communities, oracle.MODE_RAND, 0.0, SEED, 0)
    for bid in (0, 1):
        roots = oracle.batch_roots(order, cfg.batch_size, bid)
        yg, ref, nd = _run(b, prep, g, cfg.fanouts, roots, bid, layer, cfg.p_intra)
        assert nd > 0
        _check(yg, ref, nd, F, ws, wn, bias, relu, out_bf16)


def test_layer_exact_operands():
    """bf16-representable X and W, W_neigh = 0: only fp32 accumulation separates GPU and oracle,
    so a layout / indexing / descriptor error cannot hide under the bf16 tolerance."""
    b0, _, _ = _bundle("products", 0.01)
    b = copy.copy(b0)
    b.X = torch.from_numpy(b0.X).to(torch.bfloat16).float().numpy()
    prep = oracle.graph_prep(b)
    g = cmb.Graph.from_bundle(b)
    F = b.cfg.feat_dim
    ws, _, bias = _weights(F, 256, 11, bf16_exact=True)
    wn = torch.zeros_like(ws)
    layer = cmb.SageLayer(ws, wn, bias, relu=False)
    order = oracle.order_roots(b.train, b.comm, b.cfg.num_communities, oracle.MODE_COMM, 0.25,
                               SEED, 1)
    roots = oracle.batch_roots(order, b.cfg.batch_size, 1)
    yg, ref, nd = _run(b, prep, g, b.cfg.fanouts, roots, 1, layer, 1.0)
    _check(yg, ref, nd, F, ws, wn, bias, False, False, exact=True)
    # and the neighbour path alone (W_self = 0): H is not bf16-exact, so the R26 bound applies
    ws2, wn2, _ = _weights(F, 256, 12)
    layer2 = cmb.SageLayer(torch.zeros_like(ws2), wn2, None, relu=False)
    yg, ref, nd = _run(b, prep, g, b.cfg.fanouts, roots, 1, layer2, 1.0)
    _check(yg, ref, nd, F, torch.zeros_like(ws2), wn2, torch.zeros(256), False, False)


def test_layer_full_size_products():
    """The bench configuration (products-shaped, full size, RAND, p = 0.5): every row of one
    batch against the oracle (one oracle batch is ~0.3 s)."""
    b, prep, g = _bundle("products")
    cfg = b.cfg
    F = cfg.feat_dim
    ws, wn, bias = _weights(F, 256, 5)
    layer = cmb.SageLayer(ws, wn, bias, relu=True)
    order = oracle.order_roots(b.train, b.comm, cfg.num_communities, oracle.MODE_RAND, 0.0, SEED, 0)
    roots = oracle.batch_roots(order, cfg.batch_size, 5)
    yg, ref, nd = _run(b, prep, g, cfg.fanouts, roots, 5, layer, 0.5)
    assert nd > 100_000  # spans ~1000 tiles of 128 rows
    _check(yg, ref, nd, F, ws, wn, bias, True, False)


def test_layer_edge_cases():
    b, prep, g = _bundle("tiny")
    F = b.cfg.feat_dim
    ws, wn, bias = _weights(F, 64, 3)
    layer = cmb.SageLayer(ws, wn, bias, relu=False)
    # a single root (one partial tile) and a zero-degree-heavy p = 1 batch
    order = oracle.order_roots(b.train, b.comm, b.cfg.num_communities, oracle.MODE_NORAND, 0.0,
                               SEED, 0)
    for roots in (order[:1], order[:129]):
        roots = np.ascontiguousarray(roots)
        yg, ref, nd = _run(b, prep, g, b.cfg.fanouts, roots, 0, layer, 1.0)
        _check(yg, ref, nd, F, ws, wn, bias, False, False)
    # unsupported shapes are host-checked errors
    with pytest.raises(ValueError):
        cmb.SageLayer(torch.zeros(F, 20), torch.zeros(F, 20))
    with pytest.raises(ValueError):
        cmb.SageLayer(torch.zeros(200, 64), torch.zeros(200, 64))


@pytest.mark.parametrize("fanouts", [(10, 8), (4, 15), (3, 32)])
def test_layer_wide_fanouts(fanouts):
    """Last-hop fanouts above 5 take the DMAX = 10 kernel; above 10 the long-row loop (edges
    folded in CSR order in chunks of DMAX), up to the 32-edge maximum."""
    b, prep, g = _bundle("products", 0.01)
    F = b.cfg.feat_dim
    ws, wn, bias = _weights(F, 128, 9)
    layer = cmb.SageLayer(ws, wn, bias, relu=True)
    order = oracle.order_roots(b.train, b.comm, b.cfg.num_communities, oracle.MODE_RAND, 0.0,
                               SEED, 0)
    roots = np.ascontiguousarray(oracle.batch_roots(order, 512, 1))
    yg, ref, nd = _run(b, prep, g, list(fanouts), roots, 1, layer, 0.7)
    _check(yg, ref, nd, F, ws, wn, bias, True, False)


# ---------------------------------------------------------------- backward (reading R27)
def _bwd_check(b, prep, g, fanouts, roots, bid, p, fo, relu, seed=21):
    F = b.cfg.feat_dim
    ws, wn, bias = _weights(F, fo, seed)
    layer = cmb.SageLayer(ws, wn, bias, relu=relu, out_bf16=True)
    sampler = cmb.Sampler(g, len(roots), fanouts)
    sampler.sample(torch.from_numpy(roots).cuda(), p, SEED, bid)
    ref = oracle.run_batch(prep, b.X, F, roots, fanouts, p, SEED, bid)
    L = len(fanouts)
    nd = ref["n"][L - 1]
    Xd = ref["X_in"][:nd, :F].astype(np.float64)
    H = ref["H64"][:, :F]
    # upstream gradient and (for ReLU) the mask source: test inputs in bf16, the same values on
    # both sides; Y is the oracle's forward output rounded to bf16 (never the GPU's)
    gen = torch.Generator().manual_seed(seed + 1)
    dY = (torch.randn(nd, fo, generator=gen) * 0.01).to(torch.bfloat16)
    Yo = torch.from_numpy(oracle.sage_conv(Xd, H, ws.double().numpy(), wn.double().numpy(),
                                           bias.double().numpy(), relu=True)).to(torch.bfloat16)
    dy_d = torch.zeros(sampler.n_cap[L - 1], fo, dtype=torch.bfloat16, device="cuda")
    dy_d[:nd] = dY.cuda()
    y_d = None
    if relu:
        y_d = torch.zeros_like(dy_d)
        y_d[:nd] = Yo.cuda()
    dws, dwn, db = sampler.sage_layer_backward(layer, dy_d, y_d)
    torch.cuda.synchronize()
    assert sampler.status() == 0
    dZ = dY.double().numpy()
    if relu:
        dZ = dZ * (Yo.double().numpy() > 0)
    rs, rn, rb = oracle.sage_conv_backward(Xd, H, dZ)
    for got, ref_, A in ((dws, rs, Xd), (dwn, rn, H)):
        S = np.abs(A).T @ np.abs(dZ)
        err = np.abs(got.double().cpu().numpy() - ref_)
        assert np.all(err <= 2.0 ** -7 * S + 1e-30), float(np.max(err - 2.0 ** -7 * S))
    errb = np.abs(db.double().cpu().numpy() - rb)
    assert np.all(errb <= 2.0 ** -12 * np.abs(dZ).sum(0) + 1e-30), float(np.max(errb))
    return nd


@pytest.mark.parametrize("name,factor,fo,relu", [
    ("tiny", None, 256, False),      # F = 16: M = 128 covers both halves (kh = 1)
    ("tiny", None, 64, True),
    ("products", 0.01, 256, True),   # F = 100: two M blocks, ragged F
    ("arxiv", None, 128, False),     # F = 128
])
def test_layer_backward_parity(name, factor, fo, relu):
    b, prep, g = _bundle(name, factor)
    order = oracle.order_roots(b.train, b.comm, b.cfg.num_communities, oracle.MODE_RAND, 0.0,
                               SEED, 0)
    roots = oracle.batch_roots(order, b.cfg.batch_size, 1)
    assert _bwd_check(b, prep, g, b.cfg.fanouts, roots, 1, b.cfg.p_intra, fo, relu) > 0


def test_layer_backward_full_size_products():
    b, prep, g = _bundle("products")
    order = oracle.order_roots(b.train, b.comm, b.cfg.num_communities, oracle.MODE_RAND, 0.0,
                               SEED, 0)
    roots = oracle.batch_roots(order, b.cfg.batch_size, 5)
    assert _bwd_check(b, prep, g, b.cfg.fanouts, roots, 5, 0.5, 256, True) > 100_000


def test_layer_backward_edge_cases():
    b, prep, g = _bundle("tiny")
    order = oracle.order_roots(b.train, b.comm, b.cfg.num_communities, oracle.MODE_NORAND, 0.0,
                               SEED, 0)
    for roots in (order[:1], order[:129]):   # one partial tile; fewer tiles than SMs
        _bwd_check(b, prep, g, b.cfg.fanouts, np.ascontiguousarray(roots), 0, 1.0, 32, True)
    with pytest.raises(ValueError):   # backward needs a power-of-two out_dim
        layer = cmb.SageLayer(torch.zeros(16, 48), torch.zeros(16, 48))
        layer.backward_workspace()


# ---------------------------------------------------------------- wide rows (cmb_sage_dense_*)
@pytest.mark.parametrize("name,factor,fo,relu,out_bf16", [
    ("reddit", 0.01, 256, True, True),       # F = 602 (ld 604): the case the fused layer can't hold
    ("reddit", 0.01, 64, False, False),
    ("products", 0.01, 256, True, True),     # F = 100: the same layer through the unfused path
])
def test_dense_layer_parity(name, factor, fo, relu, out_bf16):
    """NEXT-4 for F > 128 (R26 / R27 on the a4 + a5 outputs, bf16 operands, cuBLASLt GEMMs):
    forward within the R26 bound, weight gradients within the R27 bound, rows past n zero."""
    b, prep, g = _bundle(name, factor)
    cfg = b.cfg
    F, L = cfg.feat_dim, len(cfg.fanouts)
    ws, wn, bias = _weights(F, fo, 9)
    layer = cmb.DenseSageLayer(ws, wn, bias, relu=relu, out_bf16=out_bf16)
    order = oracle.order_roots(b.train, b.comm, cfg.num_communities, oracle.MODE_RAND, 0.0, SEED, 0)
    roots = oracle.batch_roots(order, cfg.batch_size, 1)
    sampler = cmb.Sampler(g, len(roots), cfg.fanouts)
    sampler.sample(torch.from_numpy(roots).cuda(), cfg.p_intra, SEED, 1)
    y = sampler.sage_dense_layer(layer)
    torch.cuda.synchronize()
    assert sampler.status() == 0
    ref = oracle.run_batch(prep, b.X, F, roots, cfg.fanouts, cfg.p_intra, SEED, 1)
    nd = ref["n"][L - 1]
    _check(y[:nd].float().cpu().numpy().astype(np.float64), ref, nd, F, ws, wn, bias, relu,
           out_bf16)
    assert torch.all(y[nd:] == 0)
    # backward on the same batch: dY bf16 test input, Y the oracle's bf16 forward (mask source)
    Xd = ref["X_in"][:nd, :F].astype(np.float64)
    H = ref["H64"][:, :F]
    gen = torch.Generator().manual_seed(4)
    dY = (torch.randn(nd, fo, generator=gen) * 0.01).to(torch.bfloat16)
    Yo = torch.from_numpy(oracle.sage_conv(Xd, H, ws.double().numpy(), wn.double().numpy(),
                                           bias.double().numpy(), relu=True)).to(torch.bfloat16)
    cap = sampler.n_cap[L - 1]
    dy_d = torch.zeros(cap, fo, dtype=torch.bfloat16, device="cuda")
    dy_d[:nd] = dY.cuda()
    y_d = None
    if relu:
        y_d = torch.zeros_like(dy_d)
        y_d[:nd] = Yo.cuda()
    dws, dwn, db = sampler.sage_dense_backward(layer, dy_d, y_d)
    torch.cuda.synchronize()
    dZ = dY.double().numpy()
    if relu:
        dZ = dZ * (Yo.double().numpy() > 0)
    rs, rn, rb = oracle.sage_conv_backward(Xd, H, dZ)
    for got, ref_, A in ((dws, rs, Xd), (dwn, rn, H)):
        S = np.abs(A).T @ np.abs(dZ)
        err = np.abs(got.double().cpu().numpy() - ref_)
        assert np.all(err <= 2.0 ** -7 * S + 1e-30), float(np.max(err - 2.0 ** -7 * S))
    errb = np.abs(db.double().cpu().numpy() - rb)
    assert np.all(errb <= 2.0 ** -12 * np.abs(dZ).sum(0) + 1e-30), float(np.max(errb))


# ---------------------------------------------------------------- GCN variant (reading R28)
@pytest.mark.parametrize("name,factor,fo,relu,out_bf16", [
    ("tiny", None, 64, True, False),
    ("products", 0.01, 256, False, True),
    ("arxiv", None, 256, True, False),
])
def test_gcn_layer_parity(name, factor, fo, relu, out_bf16):
    b, prep, g = _bundle(name, factor)
    F = b.cfg.feat_dim
    gen = torch.Generator().manual_seed(13)
    W = torch.randn(F, fo, generator=gen) / np.sqrt(F)
    bias = torch.randn(fo, generator=gen) * 0.1
    layer = cmb.GcnLayer(W, bias, relu=relu, out_bf16=out_bf16)
    order = oracle.order_roots(b.train, b.comm, b.cfg.num_communities, oracle.MODE_COMM, 0.5,
                               SEED, 0)
    roots = oracle.batch_roots(order, b.cfg.batch_size, 1)
    sampler = cmb.Sampler(g, len(roots), b.cfg.fanouts)
    sampler.sample(torch.from_numpy(roots).cuda(), b.cfg.p_intra, SEED, 1)
    y = sampler.gcn_layer(layer)
    torch.cuda.synchronize()
    ref = oracle.run_batch(prep, b.X, F, roots, b.cfg.fanouts, b.cfg.p_intra, SEED, 1)
    L = len(b.cfg.fanouts)
    nd = ref["n"][L - 1]
    ip, ix = ref["indptr"][L - 1], ref["indices"][L - 1]
    X = ref["X_in"][:, :F].astype(np.float64)
    Y = oracle.gcn_conv(ip, ix, X, W.double().numpy(), bias.double().numpy(), relu=relu)
    Aabs = oracle.gcn_conv(ip, ix, np.abs(X), np.abs(W.double().numpy()),
                           np.abs(bias.double().numpy()))  # |A'X|·|W| + |b| bound (A' >= 0)
    tol = 2.0 ** -7 * Aabs + (2.0 ** -8 * np.abs(Y) if out_bf16 else 0.0)
    err = np.abs(y[:nd].float().cpu().numpy().astype(np.float64) - Y)
    assert np.all(err <= tol + 1e-30), float(np.max(err - tol))


@pytest.mark.parametrize("name,factor,fo,relu", [
    ("tiny", None, 64, True),        # F = 16: kh = 1, the M block spans an unused atom
    ("tiny", None, 256, False),
    ("products", 0.01, 256, True),   # F = 100: kh = 2, one M block
    ("arxiv", None, 128, False),     # F = 128
    ("products", None, 256, True),   # full size
])
def test_gcn_layer_backward_parity(name, factor, fo, relu):
    """GCN weight gradients (reading R35) against oracle.gcn_conv_backward on the oracle's own
    block and X_in, within the R27 bound 2^-7 |A'X|^T |dZ| (dW) and 2^-12 sum |dZ| (db)."""
    b, prep, g = _bundle(name, factor)
    F, L = b.cfg.feat_dim, len(b.cfg.fanouts)
    gen = torch.Generator().manual_seed(17)
    W = torch.randn(F, fo, generator=gen) / np.sqrt(F)
    bias = torch.randn(fo, generator=gen) * 0.1
    layer = cmb.GcnLayer(W, bias, relu=relu, out_bf16=True)
    order = oracle.order_roots(b.train, b.comm, b.cfg.num_communities, oracle.MODE_COMM, 0.5,
                               SEED, 0)
    roots = oracle.batch_roots(order, b.cfg.batch_size, 1)   # every config has >= 2 batches
    assert len(roots) > 0
    sampler = cmb.Sampler(g, len(roots), b.cfg.fanouts)
    sampler.sample(torch.from_numpy(roots).cuda(), b.cfg.p_intra, SEED, 1)
    ref = oracle.run_batch(prep, b.X, F, roots, b.cfg.fanouts, b.cfg.p_intra, SEED, 1)
    nd = ref["n"][L - 1]
    ip, ix = ref["indptr"][L - 1], ref["indices"][L - 1]
    X = ref["X_in"][:, :F].astype(np.float64)
    dY = (torch.randn(nd, fo, generator=gen) * 0.01).to(torch.bfloat16)
    Yo = torch.from_numpy(oracle.gcn_conv(ip, ix, X, W.double().numpy(), bias.double().numpy(),
                                          relu=True)).to(torch.bfloat16)
    dy_d = torch.zeros(sampler.n_cap[L - 1], fo, dtype=torch.bfloat16, device="cuda")
    dy_d[:nd] = dY.cuda()
    y_d = None
    if relu:
        y_d = torch.zeros_like(dy_d)
        y_d[:nd] = Yo.cuda()
    dw, db = sampler.gcn_layer_backward(layer, dy_d, y_d)
    torch.cuda.synchronize()
    assert sampler.status() == 0
    dZ = dY.double().numpy()
    if relu:
        dZ = dZ * (Yo.double().numpy() > 0)
    rw, rb = oracle.gcn_conv_backward(ip, ix, X, dZ)
    S = np.abs(oracle.gcn_aggregate64(ip, ix, X)).T @ np.abs(dZ)
    err = np.abs(dw.double().cpu().numpy() - rw)
    assert np.all(err <= 2.0 ** -7 * S + 1e-30), float(np.max(err - 2.0 ** -7 * S))
    errb = np.abs(db.double().cpu().numpy() - rb)
    assert np.all(errb <= 2.0 ** -12 * np.abs(dZ).sum(0) + 1e-30), float(np.max(errb))


# ---------------------------------------------------------------- the 3-layer model (R26, R29)
def _prop(T, ip, ix, nd):
    """Elementwise bound of a layer input error T through (self row, neighbour mean)."""
    return T[:nd], oracle.sage_mean64(ip, ix, T)


@pytest.mark.parametrize("name,factor", [("tiny", None), ("products", 0.01)])
def test_three_layer_forward(name, factor):
    """Layer 1 fused with the gather, layers 2 and 3 on the previous layer's bf16 output, the last
    without activation and with a class-sized output (48).  The oracle chain runs in fp64; the
    bound of each layer is its own R26/R29 term plus the previous layer's bound propagated
    through |W| (ReLU is 1-Lipschitz)."""
    b, prep, g = _bundle(name, factor)
    cfg = b.cfg
    F, L = cfg.feat_dim, len(cfg.fanouts)
    gen = torch.Generator().manual_seed(31)
    dims = [F] + [256] * (L - 1) + [48]
    Ws = [(torch.randn(dims[i], dims[i + 1], generator=gen) / np.sqrt(dims[i]),
           torch.randn(dims[i], dims[i + 1], generator=gen) / np.sqrt(dims[i]),
           torch.randn(dims[i + 1], generator=gen) * 0.1) for i in range(L)]
    order = oracle.order_roots(b.train, b.comm, cfg.num_communities, oracle.MODE_RAND, 0.0, SEED, 0)
    roots = oracle.batch_roots(order, cfg.batch_size, 0)
    sampler = cmb.Sampler(g, len(roots), cfg.fanouts)
    sampler.sample(torch.from_numpy(roots).cuda(), cfg.p_intra, SEED, 0)
    ref = oracle.run_batch(prep, b.X, F, roots, cfg.fanouts, cfg.p_intra, SEED, 0)
    # GPU chain
    ys = []
    for l in range(L):
        ws, wn, bias = Ws[l]
        last = l == L - 1
        layer = cmb.SageLayer(ws, wn, bias, relu=not last, out_bf16=not last, hidden=l > 0)
        ys.append(sampler.sage_layer(layer) if l == 0 else
                  sampler.sage_hidden(layer, L - 1 - l, ys[-1]))
    torch.cuda.synchronize()
    assert sampler.status() == 0
    # oracle chain with propagated bounds
    X = ref["X_in"][:, :F].astype(np.float64)
    Y, T = None, None
    for l in range(L):
        h = L - 1 - l
        ip, ix, nd = ref["indptr"][h], ref["indices"][h], ref["n"][h]
        ws, wn, bias = (t.double().numpy() for t in Ws[l])
        last = l == L - 1
        src = X if l == 0 else Y
        Xd, Hn = src[:nd], oracle.sage_mean64(ip, ix, src)
        Yn = oracle.sage_conv(Xd, Hn, ws, wn, bias, relu=not last)
        S = np.abs(Xd) @ np.abs(ws) + np.abs(Hn) @ np.abs(wn) + np.abs(bias)[None, :]
        tol = 2.0 ** -7 * S + (0.0 if last else 2.0 ** -8 * np.abs(Yn))
        if T is not None:
            Td, Tn = _prop(T, ip, ix, nd)
            tol = tol + Td @ np.abs(ws) + Tn @ np.abs(wn) + 2.0 ** -7 * (Td @ np.abs(ws) + Tn @ np.abs(wn))
        got = ys[l][:nd].float().cpu().numpy().astype(np.float64)
        err = np.abs(got - Yn)
        assert np.all(err <= tol + 1e-30), (l, float(np.max(err - tol)))
        Y, T = Yn, tol


# ---------------------------------------------------------------- a5 backward (reading R30)
@pytest.mark.parametrize("name,factor,F,ld", [("tiny", None, 16, 16), ("products", 0.01, 100, 100),
                                              ("products", 0.01, 7, 8), ("arxiv", None, 256, 256)])
def test_mean_backward_parity(name, factor, F, ld):
    """dX += M^T dH on every hop of a sampled batch (the GPU's blocks are bit-exact with the
    oracle's, tested above); dx starts at 1 to check that the kernel adds into it."""
    b, prep, g = _bundle(name, factor)
    cfg = b.cfg
    order = oracle.order_roots(b.train, b.comm, cfg.num_communities, oracle.MODE_RAND, 0.0, SEED, 0)
    roots = oracle.batch_roots(order, cfg.batch_size, 0)
    sampler = cmb.Sampler(g, len(roots), cfg.fanouts)
    sampler.sample(torch.from_numpy(roots).cuda(), cfg.p_intra, SEED, 0)
    ref = oracle.sample_blocks(prep, roots, cfg.fanouts, cfg.p_intra, SEED, 0)
    gen = torch.Generator().manual_seed(17)
    for h in range(len(cfg.fanouts)):
        nd, ns = ref["n"][h], ref["n"][h + 1]
        dH = torch.randn(nd, ld, generator=gen)
        dx = torch.ones(ns, ld, device="cuda")
        cmb.sage_mean_backward(sampler.indptr[h], sampler.indices[h], sampler.sizes[h:h + 1],
                               dH.cuda(), dx, F)
        torch.cuda.synchronize()
        ip, ix = ref["indptr"][h], ref["indices"][h]
        want = 1.0 + oracle.sage_mean_backward(ip, ix, dH[:, :F].double().numpy(), ns)
        S = oracle.sage_mean_backward(ip, ix, np.abs(dH[:, :F].double().numpy()), ns)
        cnt = np.bincount(np.asarray(ix, dtype=np.int64), minlength=ns)[:, None]
        got = dx.cpu().double().numpy()
        err = np.abs(got[:, :F] - want)
        tol = (cnt + 2) * 2.0 ** -24 * (S + 1.0) + 2.0 ** -126
        assert np.all(err <= tol), (h, float(np.max(err - tol)))
        assert np.all(got[:, F:] == 1.0)   # columns past feat_dim untouched


# ---------------------------------------------------------------- hidden backward (reading R31)
@pytest.mark.parametrize("name,factor,hop,fin,ld,fo,relu", [
    ("tiny", None, 0, 64, 64, 64, True),           # 64 dst rows: 32-row tiles, padding atom
    ("products", 0.01, 1, 256, 264, 256, True),    # layer 2 at the paper's widths, padded rows
    ("products", 0.01, 0, 192, 192, 128, False),   # odd atom count, no activation
    ("arxiv", None, 1, 256, 256, 256, True),
    ("products", None, 1, 256, 256, 256, True),    # full-size layer 2: 16K dst rows
    ("products", None, 0, 256, 256, 64, True),     # full-size layer 3: 1024 roots, 32-row tiles
    ("arxiv", None, 0, 128, 128, 128, True),       # fp32 dY (as the training step passes it)
])
def test_hidden_backward_parity(name, factor, hop, fin, ld, fo, relu):
    """Weight gradients of a hidden layer (R31) on a sampled batch's hop against
    oracle.sage_conv_backward on (Yp[0:n_dst], sage_mean64(Yp)); Yp, dY and Y are bf16 test
    inputs, the same values on both sides (Y only decides the ReLU mask)."""
    b, prep, g = _bundle(name, factor)
    cfg = b.cfg
    order = oracle.order_roots(b.train, b.comm, cfg.num_communities, oracle.MODE_RAND, 0.0, SEED, 0)
    roots = oracle.batch_roots(order, cfg.batch_size, 1)
    sampler = cmb.Sampler(g, len(roots), cfg.fanouts)
    sampler.sample(torch.from_numpy(roots).cuda(), cfg.p_intra, SEED, 1)
    ref = oracle.sample_blocks(prep, roots, cfg.fanouts, cfg.p_intra, SEED, 1)
    nd, ns = ref["n"][hop], ref["n"][hop + 1]
    ip, ix = ref["indptr"][hop], ref["indices"][hop]
    gen = torch.Generator().manual_seed(23 + hop)
    yp = (torch.randn(sampler.n_cap[hop + 1], ld, generator=gen) * 0.5).to(torch.bfloat16)
    dY = (torch.randn(nd, fo, generator=gen) * 0.01).to(torch.bfloat16)
    Y = torch.randn(nd, fo, generator=gen)
    Y[torch.rand(nd, fo, generator=gen) < 0.1] = 0.0   # exact zeros are masked out too
    Y = Y.to(torch.bfloat16)
    dy_d = torch.zeros(sampler.n_cap[hop], fo, dtype=torch.bfloat16, device="cuda")
    dy_d[:nd] = dY.cuda()
    y_d = None
    if relu:
        y_d = torch.zeros_like(dy_d)
        y_d[:nd] = Y.cuda()
    layer = cmb.SageLayer(torch.zeros(fin, fo), torch.zeros(fin, fo), relu=relu, out_bf16=True,
                          hidden=True)
    dz_d = torch.full((sampler.n_cap[hop], fo), float("nan"), dtype=torch.bfloat16, device="cuda")
    if name == "arxiv" and hop == 0:   # the fp32 dY path: the same (bf16-exact) values in fp32
        dy_d = dy_d.float()
    dws, dwn, db = sampler.sage_hidden_backward(layer, hop, yp.cuda(), dy_d, y_d, dz_out=dz_d)
    torch.cuda.synchronize()
    assert sampler.status() == 0
    mz = torch.where(Y > 0, dY, torch.zeros_like(dY)) if relu else dY   # R31's dZ, bit for bit
    assert torch.equal(dz_d[:nd].cpu().view(torch.int16), mz.view(torch.int16))
    Yp = yp[:ns, :fin].double().numpy()
    Xd, H = Yp[:nd], oracle.sage_mean64(ip, ix, Yp)
    dZ = dY.double().numpy()
    if relu:
        dZ = dZ * (Y.double().numpy() > 0)
    rs, rn, rb = oracle.sage_conv_backward(Xd, H, dZ)
    for got, want, A in ((dws, rs, Xd), (dwn, rn, H)):
        S = np.abs(A).T @ np.abs(dZ)
        err = np.abs(got.double().cpu().numpy() - want)
        assert np.all(err <= 2.0 ** -7 * S + 1e-30), float(np.max(err - 2.0 ** -7 * S))
    errb = np.abs(db.double().cpu().numpy() - rb)
    assert np.all(errb <= 2.0 ** -12 * np.abs(dZ).sum(0) + 1e-30), float(np.max(errb))


def test_hidden_backward_errors():
    layer = cmb.SageLayer(torch.zeros(256, 48), torch.zeros(256, 48), hidden=True)
    with pytest.raises(ValueError):   # needs a power-of-two out_dim
        layer.backward_workspace()
    first = cmb.SageLayer(torch.zeros(64, 64), torch.zeros(64, 64))
    b, prep, g = _bundle("tiny")
    sampler = cmb.Sampler(g, 8, b.cfg.fanouts)
    z = torch.zeros(8, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):   # a first-layer weight image is not a hidden layer's
        sampler.sage_hidden_backward(first, 0, z, z)


# ---------------------------------------------------------------- hidden input gradient (R32)
class _TLayer:
    """Only what sage_hidden_input_grad needs, for widths the hidden forward does not take
    (in_dim not a multiple of 64): the transposed image packed by cmb_sage_hidden_pack_weights_t."""

    def __init__(self, ws, wn):
        import ctypes
        self.hidden, self.feat_dim, self.out_dim = True, int(ws.shape[0]), int(ws.shape[1])
        self.device = torch.device("cuda")
        self.w_self, self.w_neigh = ws.cuda().contiguous(), wn.cuda().contiguous()
        n = cmb.lib().cmb_sage_hidden_weights_t_bytes(self.feat_dim, self.out_dim)
        assert n > 0
        self._wt = torch.zeros(n, dtype=torch.uint8, device="cuda")
        assert cmb.lib().cmb_sage_hidden_pack_weights_t(
            ctypes.c_void_p(self.w_self.data_ptr()), ctypes.c_void_p(self.w_neigh.data_ptr()),
            self.feat_dim, self.out_dim, ctypes.c_void_p(self._wt.data_ptr()), n, None) == 0

    def transposed_image(self):
        return self._wt


@pytest.mark.parametrize("name,factor,hop,fin,fo", [
    ("tiny", None, 0, 64, 64),
    ("tiny", None, 1, 192, 32),          # K = 32 padded to one 64-column atom (zero columns)
    ("products", 0.01, 1, 48, 16),       # N = 48 (not a multiple of 64), K = 16
    ("products", 0.01, 1, 256, 256),     # layer 2's input gradient at the paper's widths
    ("products", 0.01, 0, 128, 64),      # layer 3 (1024-root batches scaled down)
    ("arxiv", None, 1, 256, 256),
    ("products", None, 1, 256, 256),     # full size: 16K dst rows, ~145K src rows
])
def test_hidden_input_grad_parity(name, factor, hop, fin, fo):
    """dYp = P^T dZ W_self^T + M^T dZ W_neigh^T (R32) against oracle.sage_hidden_input_grad;
    every row of the output past n_src is zero."""
    b, prep, g = _bundle(name, factor)
    cfg = b.cfg
    order = oracle.order_roots(b.train, b.comm, cfg.num_communities, oracle.MODE_RAND, 0.0, SEED, 0)
    roots = oracle.batch_roots(order, cfg.batch_size, 1)
    sampler = cmb.Sampler(g, len(roots), cfg.fanouts)
    sampler.sample(torch.from_numpy(roots).cuda(), cfg.p_intra, SEED, 1)
    ref = oracle.sample_blocks(prep, roots, cfg.fanouts, cfg.p_intra, SEED, 1)
    nd, ns = ref["n"][hop], ref["n"][hop + 1]
    ip, ix = ref["indptr"][hop], ref["indices"][hop]
    gen = torch.Generator().manual_seed(41 + hop)
    ws = torch.randn(fin, fo, generator=gen) / np.sqrt(fo)
    wn = torch.randn(fin, fo, generator=gen) / np.sqrt(fo)
    dZ = (torch.randn(nd, fo, generator=gen) * 0.01).to(torch.bfloat16)
    ld = ((fo + 63) // 64) * 64
    dz_d = torch.zeros(sampler.n_cap[hop], ld, dtype=torch.bfloat16, device="cuda")
    dz_d[:nd, :fo] = dZ.cuda()
    layer = cmb.SageLayer(ws, wn, hidden=True) if fin % 64 == 0 else _TLayer(ws, wn)
    dx = torch.full((sampler.n_cap[hop + 1], fin), float("nan"), device="cuda")
    sampler.sage_hidden_input_grad(layer, hop, dz_d, dx)
    torch.cuda.synchronize()
    assert sampler.status() == 0
    Z = dZ.double().numpy()
    want = oracle.sage_hidden_input_grad(ip, ix, Z, ws.double().numpy(), wn.double().numpy(), ns)
    S = oracle.sage_hidden_input_grad(ip, ix, np.abs(Z), np.abs(ws.double().numpy()),
                                      np.abs(wn.double().numpy()), ns)
    got = dx.cpu().double().numpy()
    err = np.abs(got[:ns] - want)
    tol = 2.0 ** -7 * S + 1e-30
    assert np.all(err <= tol), float(np.max(err - tol))
    assert np.all(got[ns:] == 0.0)


# ---------------------------------------------------------------- saved operand tiles (§7)
@pytest.mark.parametrize("name,factor,relu", [("tiny", None, True), ("products", 0.01, True),
                                              ("arxiv", None, False), ("products", None, True)])
def test_layer_saved_operand_is_bit_exact(name, factor, relu):
    """The forward that saves its operand tiles returns the same Y, and the backward that reloads
    them returns the same dW / db, bit for bit, as the re-gathering pair (same operand bytes, same
    MMAs, same reduction order); the R27 bound is checked on the re-gathering pair above."""
    b, prep, g = _bundle(name, factor)
    cfg = b.cfg
    F, L, fo = cfg.feat_dim, len(cfg.fanouts), 256
    ws, wn, bias = _weights(F, fo, 5)
    layer = cmb.SageLayer(ws, wn, bias, relu=relu, out_bf16=True)
    order = oracle.order_roots(b.train, b.comm, cfg.num_communities, oracle.MODE_RAND, 0.0, SEED, 0)
    roots = oracle.batch_roots(order, cfg.batch_size, 1)
    sampler = cmb.Sampler(g, len(roots), cfg.fanouts)
    sampler.sample(torch.from_numpy(roots).cuda(), cfg.p_intra, SEED, 1)
    y0 = sampler.sage_layer(layer).clone()
    y1 = sampler.sage_layer(layer, save_a=True)
    gen = torch.Generator(device="cuda").manual_seed(3)
    dy = torch.randn(sampler.n_cap[L - 1], fo, generator=gen, device="cuda") * 0.01   # fp32 dY
    r0 = [t.clone() for t in sampler.sage_layer_backward(layer, dy, y1 if relu else None)]
    r1 = sampler.sage_layer_backward(layer, dy, y1 if relu else None, saved=True)
    torch.cuda.synchronize()
    assert sampler.status() == 0
    nd = int(sampler.sizes[L - 1].item())
    assert torch.equal(y0[:nd].view(torch.int16), y1[:nd].view(torch.int16))
    for a, c in zip(r0, r1):
        assert torch.equal(a.view(torch.int32), c.view(torch.int32))
