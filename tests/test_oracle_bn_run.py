"""Pins for oracle.bn (reading R16) and oracle.run (the loop).

bn: SPEC S:367-369 worked values, identity/fixed-point cases, dyadic exactness,
    permutation invariance.
run: the loop equals an independently written momentum-SGD loop once alpha_SGD = 1,
     and the tiny configuration C1 runs in well under the time budget.
"""
import time

import numpy as np
import pytest

import synth
from oracle import bn, exchange, run, schedule, update


def test_bn_worked_values():
    m, v = bn.sync_statistics(np.array([[0.0, 4.0], [2.0, 6.0]]), np.array([[1.0, 0.5], [3.0, 1.5]]))
    assert m.tolist() == [1.0, 5.0] and v.tolist() == [2.0, 1.0]   # simple mean, not pooled


def test_bn_identity_and_fixed_point():
    mean, var = synth.bn_stats(1, 1000)
    assert np.array_equal(bn.average(mean), mean[0])
    assert np.array_equal(bn.average(np.repeat(var, 8, axis=0)), var[0])


def test_bn_dyadic_exact_and_permutation():
    r = np.random.default_rng(1)
    x = (r.integers(-2 ** 20, 2 ** 20, (8, 512)) / 2.0 ** 12).astype(np.float32)
    avg = bn.average(x)
    assert np.array_equal(avg.astype(np.float64), x.astype(np.float64).sum(0) / 8)
    assert np.array_equal(bn.average(x[::-1]), avg)


def _c1():
    # C1 tiny: 4,096 params, 2 workers x minibatch 32, 20 steps; N_train = 64 so
    # epoch = t - 1 crosses every alpha branch (exp: t<=10, 1/2: t=11, linear 12-13, 1: t>=14)
    return schedule.Cluster(n_workers=2, b_local=32, n_train=64)


def test_run_c1_fast_and_consistent():
    n, k, T = 4096, 2, 20
    a = synth.grad_scale(n)
    th0 = synth.theta0(n, None)
    t0 = time.perf_counter()
    res = run.run(th0, lambda t: synth.grads(k, t, n, a), k, T, 1024.0, cluster=_c1())
    assert time.perf_counter() - t0 < 5.0
    a_sgd = [c.alpha_sgd for c in res.coeffs]
    assert a_sgd[10] == 0.5 and a_sgd[12] == pytest.approx(0.9) and a_sgd[13] == 1.0
    assert all(x < 0.5 for x in a_sgd[:10])
    for t in range(1, T + 1):
        assert np.array_equal(res.ghat[t - 1], exchange.exchange(list(synth.grads(k, t, n, a)), 1024.0).ghat)


def test_run_tail_equals_plain_momentum_sgd():
    """From t = 14 on (alpha_SGD = 1, alpha_RMS = 0) the loop must equal
    v <- mu1 v - ghat; theta <- theta + eta v, written out here."""
    n, k = 512, 2
    a = synth.grad_scale(n)
    cl = _c1()
    gfn = lambda t: synth.grads(k, t, n, a)  # noqa: E731
    head = run.run(synth.theta0(n, None), gfn, k, 13, 1.0, cluster=cl)
    th, v = head.theta.copy(), head.delta.copy()
    tail = run.run(synth.theta0(n, None), gfn, k, 20, 1.0, cluster=cl)
    for t in range(14, 21):
        c = schedule.coeffs_at(t, schedule.Hyper(), cl)
        assert c.alpha_sgd == 1.0 and c.alpha_rmsprop == 0.0
        ghat = exchange.exchange(list(gfn(t)), 1.0).ghat.astype(np.float64)
        v = 0.9 * v - ghat
        th = th + c.eta * v
    assert np.max(np.abs(th - tail.theta)) <= 1e-15
    assert np.array_equal(v, tail.delta)


def test_resync_step_and_scaled_error():
    c = schedule.coeffs_at(1)
    g = np.array([1e-3], dtype=np.float32)
    th, d, m = run.resync_step(np.array([0.05]), np.zeros(1), np.zeros(1), g, c)
    assert (th, d, m) == update.step(np.array([0.05]), g, np.zeros(1), np.zeros(1), c.eta,
                                     c.alpha_sgd, c.alpha_rmsprop)
    assert run.scaled_error(np.array([1.0, 2.0]), np.array([1.0, 2.0 + 1e-7]), np.array([1.0, 1.0])) \
        == pytest.approx(1e-7)
