"""GPU parity of the training-step stages added for NEXT-4 -- the loss (R33), Adam (R34) -- each
elementwise within its stated bound against the fp64 oracle, and one whole training step of
the 3-layer GraphSAGE (forward, loss, every gradient, Adam) against the fp64 oracle chain."""
import numpy as np
import pytest
import torch

import oracle
from gen import CONFIGS, generate, make_labels, num_classes, scaled

pytestmark = pytest.mark.gpu

cmb = pytest.importorskip("paper_2504_18082_b200")

SEED = 42


@pytest.mark.parametrize("n,C,ld,dy_cols", [(1024, 47, 64, 64), (3000, 256, 256, 256),
                                            (1, 1, 16, 16), (777, 40, 40, 64), (0, 8, 16, 16)])
def test_xent_parity(n, C, ld, dy_cols):
    gen = torch.Generator().manual_seed(n + C)
    logits = torch.randn(max(n, 1), ld, generator=gen) * 4 + 20   # large offsets: stable lse
    N = 5000
    node_labels = torch.randint(0, C, (N,), generator=gen, dtype=torch.int32)
    nodes = torch.randperm(N, generator=gen)[:max(n, 1)].to(torch.int32)
    dy = torch.full((max(n, 1), dy_cols), float("nan"), dtype=torch.bfloat16, device="cuda")
    loss = torch.full((1,), float("nan"), dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    cmb.softmax_xent(logits.cuda(), node_labels.cuda(), nodes.cuda(),
                     torch.tensor([n], dtype=torch.int64, device="cuda"), C, dy, loss, status)
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    Y = logits[:n, :C].double().numpy()
    lab = node_labels[nodes[:n].long()].numpy()
    want_loss, want_dy = oracle.softmax_xent(Y, lab)
    got = dy[:n].float().cpu().double().numpy()
    tol = 2.0 ** -8 * np.abs(want_dy) + 2.0 ** -20 / max(n, 1)
    assert np.all(np.abs(got[:, :C] - want_dy) <= tol), float(np.max(np.abs(got[:, :C] - want_dy) - tol))
    assert np.all(got[:, C:] == 0.0)
    mx = np.abs(Y.max(axis=1)).mean() if n else 0.0
    assert abs(loss.item() - want_loss) <= 2.0 ** -20 * (mx + 1.0)


def test_xent_bad_label_sets_status():
    logits = torch.zeros(4, 16, device="cuda")
    labels = torch.tensor([0, 1, 99, 2], dtype=torch.int32, device="cuda")
    nodes = torch.arange(4, dtype=torch.int32, device="cuda")
    dy = torch.zeros(4, 16, dtype=torch.bfloat16, device="cuda")
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    cmb.softmax_xent(logits, labels, nodes, torch.tensor([4], device="cuda"), 16, dy, loss, status)
    torch.cuda.synchronize()
    assert int(status.item()) == 1   # CMB_ERR_INVALID_ARGUMENT
    assert torch.all(dy[2] == 0)


def _adam_tol(w0, g, ow, om, ov, step, wd, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8):
    """R34's bound on the updated parameters: fp32 rounding of the update (2^-22 |w| + 2^-18 lr
    (|u| + 1)) plus the first-order effect of the fp32 rounding of the decayed gradient
    g' = g + wd w (|delta| <= 2^-23 (|g| + |wd w|), large where g ~ -wd w cancels):
    |du| <= |delta| (c1 (1 - b1) + |u| sqrt(c2 (1 - b2))) / (sqrt(v_hat) + eps)."""
    c1, c2 = 1.0 / (1 - b1 ** step), 1.0 / (1 - b2 ** step)
    den = np.sqrt(ov * c2) + eps
    u = om * c1 / den
    delta = 2.0 ** -23 * (np.abs(g) + np.abs(wd * w0))
    du = 2 * delta * (c1 * (1 - b1) + np.abs(u) * np.sqrt(c2 * (1 - b2))) / den
    return 2.0 ** -22 * np.abs(ow) + lr * (2.0 ** -18 * (np.abs(u) + 1.0) + du)


@pytest.mark.parametrize("step,wd", [(1, 0.0), (1, 5e-4), (7, 5e-4)])
def test_adam_parity(step, wd):
    rng = np.random.default_rng(step)
    n = 1 << 16
    w = rng.standard_normal(n).astype(np.float32)
    g = (rng.standard_normal(n) * 10.0 ** rng.integers(-6, 1, n)).astype(np.float32)
    m = (rng.standard_normal(n) * 1e-3).astype(np.float32) if step > 1 else np.zeros(n, np.float32)
    v = (rng.random(n) * 1e-5).astype(np.float32) if step > 1 else np.zeros(n, np.float32)
    tw, tg, tm, tv = (torch.from_numpy(a).cuda() for a in (w, g, m, v))
    cmb.adam_step(tw, tg, tm, tv, step, lr=1e-3, weight_decay=wd)
    torch.cuda.synchronize()
    ow, om, ov = oracle.adam_step(w, g, m, v, step, lr=1e-3, weight_decay=wd)
    tol = _adam_tol(w.astype(np.float64), g.astype(np.float64), ow, om, ov, step, wd)
    assert np.all(np.abs(tw.cpu().double().numpy() - ow) <= tol)
    ga = np.abs(g.astype(np.float64)) + np.abs(wd * w.astype(np.float64))   # |g| + |wd w|
    assert np.all(np.abs(tm.cpu().double().numpy() - om) <=
                  2.0 ** -21 * (np.abs(om) + 0.9 * np.abs(m) + 0.1 * ga) + 1e-38)
    assert np.all(np.abs(tv.cpu().double().numpy() - ov) <=
                  2.0 ** -20 * (np.abs(ov) + 0.999 * v + 1e-3 * ga * ga) + 1e-38)


def _bf16(t):
    return t.to(torch.bfloat16).float().cpu().double().numpy()


@pytest.mark.parametrize("name,factor", [("tiny", None), ("products", 0.01), ("arxiv", None),
                                         ("reddit", 0.01)])
def test_train_step_matches_the_oracle_chain(name, factor):
    """One step of the model (layers = hops) on a RAND batch, in two parts.
    (1) Plumbing, elementwise: every layer's weight gradient equals oracle.sage_conv_backward on
    the GPU's OWN layer input (X_in for layer 1, the previous layer's bf16 output otherwise), its
    own upstream dY (bf16-rounded, as the kernel stages it) and its own ReLU mask, within the
    R27 / R31 bound; every hidden layer's input gradient equals oracle.sage_hidden_input_grad of
    the GPU's dZ within R32; the loss and dY of the last layer equal oracle.softmax_xent of the
    GPU's logits within R33; the parameters equal oracle.adam_step of the GPU's gradients (R34).
    (2) End to end against the independent fp64 oracle chain from the same parameters, element by
    element: every activation, the loss, every weight / bias gradient and every hidden-layer input
    gradient within a bound propagated through the chain from the per-stage bounds (R26-R33),
    with ReLU masks that may flip near zero accounted for (see the comment in the test)."""
    cfg = CONFIGS[name] if factor is None else scaled(CONFIGS[name], factor)
    b = generate(cfg)
    C = num_classes(cfg)
    labels = make_labels(b, C)
    prep = oracle.graph_prep(b)
    g = cmb.Graph.from_bundle(b)
    F, L = cfg.feat_dim, len(cfg.fanouts)
    model = cmb.GraphSAGE(F, C, num_layers=L, seed=3)
    p0 = model.params.cpu().double().numpy().copy()
    order = oracle.order_roots(b.train, b.comm, cfg.num_communities, oracle.MODE_RAND, 0.0, SEED, 0)
    roots = oracle.batch_roots(order, cfg.batch_size, 0)
    sampler = cmb.Sampler(g, len(roots), cfg.fanouts)
    sampler.sample(torch.from_numpy(roots).cuda(), cfg.p_intra, SEED, 0)
    loss = model.train_step(sampler, torch.from_numpy(labels).cuda())
    torch.cuda.synchronize()
    assert sampler.status() == 0 and int(model.status.item()) == 0
    ref = oracle.run_batch(prep, b.X, F, roots, cfg.fanouts, cfg.p_intra, SEED, 0)
    got_g = model.grads.cpu().double().numpy()
    got_p = model.params.cpu().double().numpy()

    def views(flat, l):
        fi, fo = model.dims[l], model.dims[l + 1]
        o = model.offsets[l]
        return (flat[o:o + fi * fo].reshape(fi, fo), flat[o + fi * fo:o + 2 * fi * fo].reshape(fi, fo),
                flat[o + 2 * fi * fo:o + 2 * fi * fo + fo])

    X = ref["X_in"][:, :F].astype(np.float64)
    n0 = ref["n"][0]
    lab0 = labels[ref["nodes"][:n0]]
    # ---- (1) plumbing, stage by stage on the GPU's own intermediates
    ys = [model._bufs[("y", l)] for l in range(L)]
    logits = ys[-1][:n0].cpu().double().numpy()
    l_want, dy_want = oracle.softmax_xent(logits[:, :C], lab0)
    assert abs(loss.item() - l_want) <= 2.0 ** -20 * (np.abs(logits[:, :C].max(axis=1)).mean() + 1)
    dY = model._bufs["dyL"][:n0].float().cpu().double().numpy()
    assert np.all(np.abs(dY[:, :C] - dy_want) <= 2.0 ** -8 * np.abs(dy_want) + 2.0 ** -20 / n0)
    for l in range(L - 1, -1, -1):
        h = L - 1 - l
        ip, ix, nd, ns = ref["indptr"][h], ref["indices"][h], ref["n"][h], ref["n"][h + 1]
        src = X if l == 0 else ys[l - 1][:ns].float().cpu().double().numpy()
        Xd, Hn = src[:nd], oracle.sage_mean64(ip, ix, src)
        dZ = dY[:nd]
        if l < L - 1:
            dZ = dZ * (ys[l][:nd].float().cpu().double().numpy() > 0)
        want = oracle.sage_conv_backward(Xd, Hn, dZ)
        for got, w_, A in zip(views(got_g, l), want, (Xd, Hn, None)):
            if A is None:
                tol = 2.0 ** -12 * np.abs(dZ).sum(0)
            else:
                tol = 2.0 ** -7 * (np.abs(A).T @ np.abs(dZ))
            assert np.all(np.abs(got - w_) <= tol + 1e-30), (l, float(np.max(np.abs(got - w_) - tol)))
        if l > 0:
            dz_gpu = model._bufs[("dz", l)][:nd, :model.dims[l + 1]].float().cpu().double().numpy()
            assert np.array_equal(dz_gpu, dZ)   # the fused mask, bit for bit
            ws, wn, _ = views(p0, l)
            want_dx = oracle.sage_hidden_input_grad(ip, ix, dZ, ws, wn, ns)
            S = oracle.sage_hidden_input_grad(ip, ix, np.abs(dZ), np.abs(ws), np.abs(wn), ns)
            dx = model._bufs[("dx", l)][:ns].cpu().double().numpy()
            assert np.all(np.abs(dx - want_dx) <= 2.0 ** -7 * S + 1e-30), l
            dY = _bf16(model._bufs[("dx", l)][:ns])   # the next layer stages it in bf16
    z = np.zeros_like(p0)
    want_p, om, ov = oracle.adam_step(p0, got_g, z, z, 1)
    assert np.all(np.abs(got_p - want_p) <= _adam_tol(p0, got_g, want_p, om, ov, 1, 5e-4))
    # ---- (2) end to end against the independent fp64 chain, ELEMENTWISE with propagated bounds:
    # forward as test_three_layer_forward (each layer's own R26 / R29 term + the previous layer's
    # bound through |W|); the loss and dY through the softmax (a logit row perturbed by at most m
    # moves every probability by at most s (e^{2m} - 1)); backward: a ReLU mask entry is certain
    # where |Y*| > T (the GPU's Y lies in [Y* - T, Y* + T]) and may flip elsewhere (there the
    # error of dZ is bounded by |dY*| + E); weight gradients add the operand errors to their own
    # R27 / R31 term, input gradients add the dZ error through |W| to their own R32 term, and the
    # next layer's bf16 staging of dY adds 2^-8 |dY|.
    acts, ins, T_in, T_out = [], [], [], []
    src, Tsrc = X, None
    for l in range(L):
        h = L - 1 - l
        ip, ix, nd = ref["indptr"][h], ref["indices"][h], ref["n"][h]
        ws, wn, bias = views(p0, l)
        last = l == L - 1
        Xd, Hn = src[:nd], oracle.sage_mean64(ip, ix, src)
        if Tsrc is None:   # layer 1: exact features, H summed in fp32 (<= 32 terms)
            Td = np.zeros_like(Xd)
            Tn = 2.0 ** -18 * oracle.sage_mean64(ip, ix, np.abs(src))
        else:
            Td, Tn = Tsrc[:nd], oracle.sage_mean64(ip, ix, Tsrc)
        Y = oracle.sage_conv(Xd, Hn, ws, wn, bias, relu=not last)
        S = (np.abs(Xd) + Td) @ np.abs(ws) + (np.abs(Hn) + Tn) @ np.abs(wn) + np.abs(bias)[None, :]
        T = 2.0 ** -7 * S + Td @ np.abs(ws) + Tn @ np.abs(wn) + (0.0 if last else 2.0 ** -8 * np.abs(Y))
        got_y = ys[l][:nd].float().cpu().double().numpy()
        assert np.all(np.abs(got_y - Y) <= T + 1e-30), ("forward", l, float(np.max(np.abs(got_y - Y) - T)))
        acts.append(Y)
        ins.append((Xd, Hn))
        T_in.append((Td, Tn))
        T_out.append(T)
        src, Tsrc = Y, T
    logit = acts[-1][:, :C]
    want_loss, dYc = oracle.softmax_xent(logit, lab0)
    m = T_out[-1][:, :C].max(axis=1, keepdims=True)
    row_term = 2.0 * m[:, 0] + 2.0 ** -20 * (np.abs(logit.max(axis=1)) + 1.0)
    assert abs(loss.item() - want_loss) <= row_term.mean() + 1e-30
    sm_ = np.exp(logit - logit.max(axis=1, keepdims=True))
    sm_ /= sm_.sum(axis=1, keepdims=True)
    dY = np.zeros_like(acts[-1])
    dY[:, :C] = dYc
    E = np.zeros_like(dY)
    E[:, :C] = (sm_ * np.expm1(2.0 * m) / n0) * (1 + 2.0 ** -8) + 2.0 ** -8 * np.abs(dYc) + 2.0 ** -20 / n0
    for l in range(L - 1, -1, -1):
        h = L - 1 - l
        ip, ix, nd, ns = ref["indptr"][h], ref["indices"][h], ref["n"][h], ref["n"][h + 1]
        Xd, Hn = ins[l]
        Td, Tn = T_in[l]
        if l < L - 1:
            certain1 = acts[l] > T_out[l]
            uncertain = (acts[l] <= T_out[l]) & (acts[l] + T_out[l] > 0)
            dZ = dY * certain1
            EZ = E * certain1 + uncertain * (np.abs(dY) + E)
        else:
            dZ, EZ = dY, E
        aZ = np.abs(dZ) + EZ
        want = oracle.sage_conv_backward(Xd, Hn, dZ)
        for part, (A, TA) in enumerate(((Xd, Td), (Hn, Tn))):
            bound = TA.T @ aZ + np.abs(A).T @ EZ + 2.0 ** -7 * ((np.abs(A) + TA).T @ aZ)
            err = np.abs(views(got_g, l)[part] - want[part])
            assert np.all(err <= bound + 1e-30), ("dW", l, part, float(np.max(err - bound)))
        bound_b = EZ.sum(axis=0) + 2.0 ** -12 * aZ.sum(axis=0)
        assert np.all(np.abs(views(got_g, l)[2] - want[2]) <= bound_b + 1e-30), ("db", l)
        if l > 0:
            ws, wn, _ = views(p0, l)
            dYp = oracle.sage_hidden_input_grad(ip, ix, dZ, ws, wn, ns)
            Ep = oracle.sage_hidden_input_grad(ip, ix, EZ, np.abs(ws), np.abs(wn), ns) + \
                2.0 ** -7 * oracle.sage_hidden_input_grad(ip, ix, aZ, np.abs(ws), np.abs(wn), ns)
            dx = model._bufs[("dx", l)][:ns].cpu().double().numpy()
            assert np.all(np.abs(dx - dYp) <= Ep + 1e-30), ("dX", l, float(np.max(np.abs(dx - dYp) - Ep)))
            dY, E = dYp, Ep + 2.0 ** -8 * (np.abs(dYp) + Ep)   # staged as bf16 by the next kernel
    # padded logit columns: no gradient reaches them, their parameters stay zero
    assert np.all(views(got_g, L - 1)[0][:, C:] == 0.0)
    assert np.all(views(got_p, L - 1)[0][:, C:] == 0.0)


def test_training_fits_one_batch():
    """Sanity of the whole step as an optimizer: repeated steps on ONE batch (tiny graph) must
    drive its loss down (the classic overfit-a-batch check; a sign error anywhere in the chain
    makes the loss rise)."""
    cfg = CONFIGS["tiny"]
    b = generate(cfg)
    C = num_classes(cfg)
    g = cmb.Graph.from_bundle(b)
    model = cmb.GraphSAGE(cfg.feat_dim, C, num_layers=len(cfg.fanouts), seed=5, lr=1e-2,
                          weight_decay=0.0)
    order = oracle.order_roots(b.train, b.comm, cfg.num_communities, oracle.MODE_RAND, 0.0, SEED, 0)
    roots = oracle.batch_roots(order, cfg.batch_size, 0)
    sampler = cmb.Sampler(g, len(roots), cfg.fanouts)
    sampler.sample(torch.from_numpy(roots).cuda(), cfg.p_intra, SEED, 0)
    labels = torch.from_numpy(make_labels(b, C)).cuda()
    losses = [float(model.train_step(sampler, labels).item()) for _ in range(40)]
    assert losses[0] > 1.0 and losses[-1] < 0.25 * losses[0], losses


def test_fused_adam_repack_equals_adam_then_pack():
    """cmb_adam_step_pack (one launch) = cmb_adam_step + a fresh pack of every image, bit for
    bit: parameters, moments, forward images and transposed images after three steps."""
    cfg = scaled(CONFIGS["products"], 0.01)
    b = generate(cfg)
    C = num_classes(cfg)
    g = cmb.Graph.from_bundle(b)
    L = len(cfg.fanouts)
    labels = torch.from_numpy(make_labels(b, C)).cuda()
    order = oracle.order_roots(b.train, b.comm, cfg.num_communities, oracle.MODE_RAND, 0.0, SEED, 0)
    sampler = cmb.Sampler(g, cfg.batch_size, cfg.fanouts)
    model = cmb.GraphSAGE(cfg.feat_dim, C, num_layers=L, seed=2)
    for k in range(3):
        roots = oracle.batch_roots(order, cfg.batch_size, k % 2)   # the scaled graph has 2
        sampler.sample(torch.from_numpy(roots).cuda(), cfg.p_intra, SEED, k)
        p_before, m_before, v_before = (t.clone() for t in (model.params, model.m, model.v))
        model.train_step(sampler, labels)
        # the unfused reference from the same state and gradients
        w, m, v = p_before.clone(), m_before.clone(), v_before.clone()
        cmb.adam_step(w, model.grads, m, v, model.step_count, model.lr,
                      weight_decay=model.weight_decay)
        for got, want in ((model.params, w), (model.m, m), (model.v, v)):
            assert torch.equal(got.view(torch.int32), want.view(torch.int32))
        for layer in model.layers:
            ref = cmb.SageLayer(layer.w_self, layer.w_neigh, layer.bias, hidden=layer.hidden)
            assert torch.equal(layer.w_img, ref.w_img)
            if layer.hidden:
                assert torch.equal(layer.transposed_image(), ref.transposed_image())
    torch.cuda.synchronize()


def test_graph_replayed_train_step_matches_eager():
    """GraphSAGE.train_step(graph=True): the first call runs the step eagerly and captures it as
    a CUDA graph, later calls replay it on whatever batch the sampler holds.  Per batch (5
    different batches) the replayed model starts from the eager model's state (parameters,
    moments, weight images): same loss and gradients as the eager step up to the fp32 rounding
    order of the aggregation backward's atomics (R30), the device step counter in step, and the
    replayed Adam + repack bit-exact against the unfused reference from its own gradients.
    (Trajectories are not compared: Adam turns a last-bit gradient difference on a parameter
    whose gradient is near zero into an lr-sized update difference.)"""
    cfg = scaled(CONFIGS["products"], 0.01)
    b = generate(cfg)
    C = num_classes(cfg)
    g = cmb.Graph.from_bundle(b)
    L = len(cfg.fanouts)
    labels = torch.from_numpy(make_labels(b, C)).cuda()
    order = oracle.order_roots(b.train, b.comm, cfg.num_communities, oracle.MODE_RAND, 0.0, SEED, 0)
    sampler = cmb.Sampler(g, cfg.batch_size, cfg.fanouts)
    eager = cmb.GraphSAGE(cfg.feat_dim, C, num_layers=L, seed=4)
    replay = cmb.GraphSAGE(cfg.feat_dim, C, num_layers=L, seed=4)
    for k in range(5):
        roots = oracle.batch_roots(order, cfg.batch_size // 2, k % 4)
        sampler.sample(torch.from_numpy(roots).cuda(), cfg.p_intra, SEED, 10 + k)
        for a, e in ((replay.params, eager.params), (replay.m, eager.m), (replay.v, eager.v)):
            a.copy_(e)
        for la, le_ in zip(replay.layers, eager.layers):
            la.w_img.copy_(le_.w_img)
            if la.hidden:
                la.transposed_image().copy_(le_.transposed_image())
        p_before, m_before, v_before = (t.clone() for t in (eager.params, eager.m, eager.v))
        le = float(eager.train_step(sampler, labels).item())
        lr_ = float(replay.train_step(sampler, labels, graph=True).item())
        torch.cuda.synchronize()
        assert replay.status.item() == 0 and eager.status.item() == 0
        assert replay.step_count == eager.step_count == k + 1
        assert int(replay._step_dev.item()) == k + 1
        assert len(replay._graphs) == 1
        assert abs(le - lr_) <= 1e-6 * abs(le) + 1e-9, (k, le, lr_)
        scale = eager.grads.abs().max().item()
        assert torch.allclose(replay.grads, eager.grads, rtol=1e-3, atol=1e-5 * scale), k
        w, m, v = p_before.clone(), m_before.clone(), v_before.clone()
        cmb.adam_step(w, replay.grads, m, v, replay.step_count, replay.lr,
                      weight_decay=replay.weight_decay)
        for got, want in ((replay.params, w), (replay.m, m), (replay.v, v)):
            assert torch.equal(got.view(torch.int32), want.view(torch.int32)), k
