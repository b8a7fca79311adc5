"""Pins for oracle.update (readings R6, R13).

Pinned against: the textbook/library optimizers the paper says the rule reduces to
 -- torch.optim.SGD(momentum) and torch.optim.RMSprop(momentum),
which the oracle does not call; hand-computed single steps; the momentum-correction
property (Delta carries no eta); fixed points and m >= 0.
"""
import math

import numpy as np
import pytest
import torch

from oracle import schedule as sch
from oracle import update as upd


def _run_oracle(theta, grads, etas, a_sgd, a_rms):
    th, d, m = theta.copy(), np.zeros_like(theta), np.zeros_like(theta)
    for g, eta in zip(grads, etas):
        th, d, m = upd.step(th, g, m, d, eta, a_sgd, a_rms)
    return th, d, m


def _grads(n, steps, seed):
    r = np.random.default_rng(seed)
    return [r.standard_normal(n) * 10.0 ** r.uniform(-4, 0, n) for _ in range(steps)]


def _etas(steps):   # LR changes mid-run (the paper's piecewise schedule)
    return [0.1 if i < 30 else 0.01 for i in range(steps)]


def _torch_run(opt_factory, theta, grads, etas):
    p = torch.nn.Parameter(torch.tensor(theta, dtype=torch.float64))
    opt = opt_factory([p])
    for g, eta in zip(grads, etas):
        for group in opt.param_groups:
            group["lr"] = eta
        p.grad = torch.tensor(g, dtype=torch.float64)
        opt.step()
    return p.detach().numpy(), opt.state[p]


def test_alpha_rmsprop_zero_is_momentum_sgd():
    # alpha_RMSprop = 0 -> standard momentum SGD
    theta = np.random.default_rng(1).standard_normal(1000)
    grads, etas = _grads(1000, 50, 2), _etas(50)
    th, d, _ = _run_oracle(theta, grads, etas, 1.0, 0.0)
    ref, st = _torch_run(lambda ps: torch.optim.SGD(ps, lr=0.1, momentum=0.9), theta, grads, etas)
    assert np.max(np.abs(th - ref)) <= 1e-12
    assert np.max(np.abs(-d - st["momentum_buffer"].numpy())) <= 1e-12   # Delta = -v


def test_alpha_sgd_zero_is_rmsprop_with_momentum():
    # alpha_SGD = 0 -> RMSprop (the momentum variant)
    theta = np.random.default_rng(3).standard_normal(1000)
    grads, etas = _grads(1000, 50, 4), _etas(50)
    th, d, m = _run_oracle(theta, grads, etas, 0.0, 1.0)
    ref, st = _torch_run(lambda ps: torch.optim.RMSprop(ps, lr=0.1, alpha=0.99, eps=1e-8,
                                                        momentum=0.9, centered=False),
                         theta, grads, etas)
    assert np.max(np.abs(th - ref)) <= 1e-12
    assert np.max(np.abs(m - st["square_avg"].numpy())) <= 1e-15
    assert np.max(np.abs(-d - st["momentum_buffer"].numpy())) <= 1e-9


def test_hand_step_sgd():
    # mu1 = 0.9, Delta = 0, g = 1, eta = 0.1, theta = 0 -> Delta = -1, theta = -0.1
    th, d, m = upd.step(0.0, 1.0, 0.0, 0.0, 0.1, 1.0, 0.0)
    assert d == -1.0 and th == pytest.approx(-0.1, abs=1e-17)


def test_hand_step_rmsprop():
    # m = 0.01 * 4 = 0.04, Delta = -2 / (0.2 + 1e-8)
    th, d, m = upd.step(0.0, 2.0, 0.0, 0.0, 1.0, 0.0, 1.0)
    assert m == pytest.approx(0.04, rel=1e-15)
    assert d == pytest.approx(-2.0 / (0.2 + 1e-8), rel=1e-15)
    assert d == pytest.approx(-9.9999995, rel=1e-8)


def test_hand_step_blended_epoch0_32k():
    # step 1 at 32k, g = 1e-3, theta = 0.05 (values worked by hand):
    # m = 0.01 * 1e-6 = 1e-8; sqrt(m) = 1e-4;
    # c = e^-4/2 + (1 - e^-4/2) 3e-4 / 6.4 / (1e-4 + 1e-8) = 0.473566...
    c = sch.coeffs_at(1)
    th, d, m = upd.step(0.05, 1e-3, 0.0, 0.0, c.eta, c.alpha_sgd, c.alpha_rmsprop)
    a = 0.5 * math.exp(-4)
    coef = a + (1 - a) * 3e-4 / 6.4 / (1e-4 + 1e-8)
    assert m == pytest.approx(1e-8, rel=1e-14)
    assert d == pytest.approx(-coef * 1e-3, rel=1e-14)
    assert d == pytest.approx(-4.7357e-4, rel=1e-4)
    assert th == pytest.approx(0.0469692, rel=1e-6)


def test_delta_independent_of_eta():
    # Delta_t must not depend on the learning-rate sequence.
    r = np.random.default_rng(9)
    grads = [r.standard_normal(64) for _ in range(500)]
    e1 = list(r.uniform(0.001, 10, 500))
    e2 = list(r.uniform(0.001, 10, 500))
    cl = sch.Cluster()
    t1 = np.zeros(64); t2 = np.ones(64)
    d1 = d2 = m1 = m2 = np.zeros(64)
    for i, g in enumerate(grads):
        c = sch.coeffs_at(1 + 7 * i, sch.Hyper(), cl)
        t1, d1, m1 = upd.step(t1, g, m1, d1, e1[i], c.alpha_sgd, c.alpha_rmsprop)
        t2, d2, m2 = upd.step(t2, g, m2, d2, e2[i], c.alpha_sgd, c.alpha_rmsprop)
        assert np.array_equal(d1, d2) and np.array_equal(m1, m2)


def test_zero_gradient_fixed_point_and_m_nonneg():
    th, d, m = upd.step(np.full(8, 0.3), np.zeros(8), np.zeros(8), np.zeros(8), 6.4, 0.01, 5e-5)
    assert np.array_equal(th, np.full(8, 0.3)) and not d.any() and not m.any()
    r = np.random.default_rng(10)
    m = np.zeros(100)
    d = np.zeros(100)
    for _ in range(100):
        _, d, m = upd.step(np.zeros(100), r.standard_normal(100), m, d, 1.0, 0.5, 0.5)
        assert np.all(m >= 0)


def test_inputs_not_modified():
    th = np.ones(4); g = np.ones(4); m = np.ones(4); d = np.ones(4)
    upd.step(th, g, m, d, 0.1, 0.5, 0.5)
    assert th.tolist() == g.tolist() == m.tolist() == d.tolist() == [1.0] * 4


def test_weight_decay_is_torch_weight_decay():
    """R12 (Goyal's settings): g + lambda theta before the m update --
    torch.optim.SGD / RMSprop(weight_decay=lambda) at the two endpoints."""
    theta = np.random.default_rng(11).standard_normal(500)
    grads, etas = _grads(500, 40, 12), _etas(40)
    lam = 1e-4
    for (a_sgd, a_rms), fac in (((1.0, 0.0), lambda ps: torch.optim.SGD(ps, lr=0.1, momentum=0.9, weight_decay=lam)),
                                ((0.0, 1.0), lambda ps: torch.optim.RMSprop(ps, lr=0.1, alpha=0.99, eps=1e-8,
                                                                           momentum=0.9, weight_decay=lam))):
        th, d, m = theta.copy(), np.zeros(500), np.zeros(500)
        for g, eta in zip(grads, etas):
            th, d, m = upd.step(th, g, m, d, eta, a_sgd, a_rms, weight_decay=lam)
        ref, _ = _torch_run(fac, theta, grads, etas)
        assert np.max(np.abs(th - ref)) <= 1e-12


def test_weight_decay_prefix_only():
    th = np.ones(10)
    a = upd.step(th, np.zeros(10), np.zeros(10), np.zeros(10), 1.0, 1.0, 0.0, weight_decay=0.5, n_decay=4)
    assert np.array_equal(a[1][:4], np.full(4, -0.5)) and not a[1][4:].any()
