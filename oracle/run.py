"""The whole per-iteration hot path for T steps and k workers (oracle; test
infrastructure).

PAPER.md:113-116 (an iteration = forward/backward, communication, optimization);
the communication and optimization halves are simulated here, the gradients are
inputs.  For t = 1..T:
  1. coefficients (epoch, eta, alpha_SGD, alpha_RMSprop)     schedule.coeffs_at
  2.-5. pack, exact reduce, fp16 wire, unpack + average        exchange.exchange
  6. blended update in float64                                  update.step
Starts from m_0 = Delta_0 = 0 (R13).

``resync_step`` is the one-step form used for tolerance checks: it starts from a
given (fp32) state and a given ghat, so one-step errors do not compound.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import exchange, schedule, update


@dataclass
class RunResult:
    theta: np.ndarray
    delta: np.ndarray
    m: np.ndarray
    ghat: list = field(default_factory=list)       # per step fp32 [n]
    coeffs: list = field(default_factory=list)     # per step schedule.Coeffs


def run(theta0, grads_fn, k: int, T: int, s: float = 1.0,
        hyper: schedule.Hyper = schedule.Hyper(),
        cluster: schedule.Cluster = schedule.Cluster(),
        t0: int = 1, keep_ghat: bool = True) -> RunResult:
    """grads_fn(t) -> fp32 [k, n] worker gradients of step t."""
    theta = np.asarray(theta0, dtype=np.float64).copy()
    delta = np.zeros_like(theta)
    m = np.zeros_like(theta)
    res = RunResult(theta, delta, m)
    for t in range(t0, t0 + T):
        c = schedule.coeffs_at(t, hyper, cluster)
        ex = exchange.exchange(list(grads_fn(t)), s)
        theta, delta, m = update.step(theta, ex.ghat, m, delta, c.eta, c.alpha_sgd,
                                      c.alpha_rmsprop, hyper.mu1, hyper.mu2, hyper.eps)
        if keep_ghat:
            res.ghat.append(ex.ghat)
        res.coeffs.append(c)
    res.theta, res.delta, res.m = theta, delta, m
    return res


def resync_step(theta_prev, delta_prev, m_prev, ghat, c: schedule.Coeffs,
                hyper: schedule.Hyper = schedule.Hyper(), weight_decay=0.0, n_decay=None):
    """Float64 update from a given state and ghat (the GPU's fp32 values)."""
    return update.step(theta_prev, ghat, m_prev, delta_prev, c.eta, c.alpha_sgd,
                       c.alpha_rmsprop, hyper.mu1, hyper.mu2, hyper.eps, weight_decay, n_decay)


def scaled_error(x_gpu, x_ora, scale) -> float:
    """max_j |x_gpu - x_ora| / scale_j with scale_j > 0 (DESIGN.md tolerances)."""
    x_gpu = np.asarray(x_gpu, dtype=np.float64)
    scale = np.asarray(scale, dtype=np.float64)
    err = np.abs(x_gpu - x_ora)
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(scale > 0, err / scale, np.where(err == 0, 0.0, np.inf))
    return float(r.max()) if r.size else 0.0
