"""Pins for the oracle's loss (reading R33) and optimizer step (reading R34), CPU only: hand
arithmetic, closed forms, finite differences of the loss, shift invariance, and the library
optimizer (torch.optim.Adam in fp64, a different implementation of the same textbook rule)."""
import math

import numpy as np
import pytest
import torch

import oracle


def test_xent_worked_example():
    # two roots, two classes: logits (0, 0) label 0 and (log 3, 0) label 1
    Y = np.array([[0.0, 0.0], [math.log(3.0), 0.0]])
    loss, dY = oracle.softmax_xent(Y, [0, 1])
    # row 0: log 2; row 1: log(3 + 1) - 0 = log 4; mean = (log 2 + log 4) / 2 = 1.5 log 2
    assert loss == pytest.approx(1.5 * math.log(2.0), rel=1e-15)
    # softmax rows (1/2, 1/2) and (3/4, 1/4); minus one-hot; over n = 2
    assert np.allclose(dY, np.array([[-0.25, 0.25], [0.375, -0.375]]), rtol=0, atol=1e-16)


def test_xent_uniform_logits_is_log_c():
    for C in (1, 2, 47, 256):
        loss, dY = oracle.softmax_xent(np.full((5, C), 3.25), np.arange(5) % C)
        assert loss == pytest.approx(math.log(C), abs=1e-14)
        assert np.allclose(dY.sum(axis=1), 0.0, atol=4e-16)   # rows of dY sum to 0 (C roundings)


def test_xent_gradient_is_the_derivative_and_shift_invariant():
    rng = np.random.default_rng(3)
    Y = rng.standard_normal((6, 5)) * 2
    lab = rng.integers(0, 5, 6)
    loss, dY = oracle.softmax_xent(Y, lab)
    eps = 1e-6
    for i in range(6):
        for c in range(5):
            Y[i, c] += eps
            lp, _ = oracle.softmax_xent(Y, lab)
            Y[i, c] -= 2 * eps
            lm, _ = oracle.softmax_xent(Y, lab)
            Y[i, c] += eps
            assert (lp - lm) / (2 * eps) == pytest.approx(dY[i, c], abs=1e-9)
    l2, d2 = oracle.softmax_xent(Y + rng.standard_normal((6, 1)) * 50, lab)   # per-row shifts
    assert l2 == pytest.approx(loss, rel=1e-12) and np.allclose(d2, dY, atol=1e-15)


def test_adam_first_step_closed_form():
    # step 1, no decay: m_hat = g, v_hat = g^2, so w moves by lr * g / (|g| + eps)
    g = np.array([0.5, -2.0, 1e-3, 0.0])
    w0 = np.array([1.0, 2.0, 3.0, 4.0])
    w, m, v = oracle.adam_step(w0, g, np.zeros(4), np.zeros(4), 1, lr=0.1, weight_decay=0.0)
    assert np.allclose(w, w0 - 0.1 * g / (np.abs(g) + 1e-8), rtol=0, atol=1e-15)
    assert np.allclose(m, 0.1 * g) and np.allclose(v, 0.001 * g * g)


@pytest.mark.parametrize("wd", [0.0, 5e-4])
def test_adam_matches_torch_optim(wd):
    rng = np.random.default_rng(9)
    w0 = rng.standard_normal(37)
    p = torch.nn.Parameter(torch.from_numpy(w0.copy()))
    opt = torch.optim.Adam([p], lr=1e-3, weight_decay=wd)
    w, m, v = w0.copy(), np.zeros(37), np.zeros(37)
    for t in range(1, 6):
        g = rng.standard_normal(37) * 10.0 ** rng.integers(-4, 1)
        p.grad = torch.from_numpy(g.copy())
        opt.step()
        w, m, v = oracle.adam_step(w, g, m, v, t, weight_decay=wd)
        assert np.allclose(w, p.detach().numpy(), rtol=1e-13, atol=1e-15)
