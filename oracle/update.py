"""The blended RMSprop / momentum-SGD update rule (oracle; test infrastructure).

PAPER.md:152-157 (Appendix A.1, "Our update rule is a simple combination of
momentum SGD and RMSprop"):

    m_t     = mu2 m_{t-1} + (1 - mu2) g_t^2
    Delta_t = mu1 Delta_{t-1} - (alpha_SGD + alpha_RMSprop / (sqrt(m_t) + eps)) g_t
    theta_t = theta_{t-1} + eta Delta_t

Inputs g_t, theta_{t-1}, Delta_{t-1}, m_{t-1}; outputs theta_t, Delta_t, m_t
(PAPER.md:160-161).  Reading R6: eps is added after the square root, as displayed.
Reading R13: m_0 = Delta_0 = 0, no bias correction.  Reading R12: optional weight
decay inherited from Goyal et al. ("the same settings are used unless otherwise
specified"): g <- g + lambda theta on the first n_decay elements,
before the m update (the torch.optim convention); off by default.  Float64.
"""
from __future__ import annotations

import numpy as np


def step(theta, g, m, delta, eta, alpha_sgd, alpha_rmsprop, mu1=0.9, mu2=0.99, eps=1e-8,
         weight_decay=0.0, n_decay=None):
    """One application of the rule, in the paper's order m, then Delta, then theta.
    Returns (theta_t, Delta_t, m_t) as float64 arrays; inputs are not modified."""
    theta = np.asarray(theta, dtype=np.float64)
    g = np.asarray(g, dtype=np.float64)
    m = np.asarray(m, dtype=np.float64)
    delta = np.asarray(delta, dtype=np.float64)
    if weight_decay:
        lam = np.zeros_like(g)
        lam[..., : (g.shape[-1] if n_decay is None else n_decay)] = weight_decay
        g = g + lam * theta
    m_t = mu2 * m + (1.0 - mu2) * g * g
    delta_t = mu1 * delta - (alpha_sgd + alpha_rmsprop / (np.sqrt(m_t) + eps)) * g
    theta_t = theta + eta * delta_t
    return theta_t, delta_t, m_t
