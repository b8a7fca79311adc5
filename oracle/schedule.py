"""Learning-rate and blend schedule (oracle; test infrastructure).

PAPER.md:174-196 (Appendix A.1, RMSprop warm-up): the ELU-like alpha_SGD
transition, beta_center = 10, beta_period = 5, eta_RMSprop = 0.0003,
eta = eta_SGD, alpha_RMSprop = (1 - alpha_SGD) eta_RMSprop / eta_SGD.
PAPER.md:216-230 (Appendix A.2): eta_base = 0.1 b_total / 256; slow-start
multipliers 0.5 / 0.075 / 0.01 / 0.001 for 40 / 30 / 15 / 5 epochs; Goyal et al.'s
1 / 0.1 / 0.01 / 0.001 for 30 / 30 / 20 / 10 epochs.

Readings: R1 linear-branch slope 1/beta_period (the displayed "2" at
PAPER.md:180 contradicts PAPER.md:186-188); R2 fractional epoch per iteration;
R3 step t uses epoch (t-1) b_total / N_train; R4 right-open phase boundaries tested
with integers; R5 N_train = 1,281,167.  R20: the other transition
functions the paper examined -- linear, sigmoid and a sudden switch
-- are not written out in the paper; R20 fixes them (below, alpha_sgd_at).

All arithmetic is IEEE double in the operation order written below (the C++ host
schedule is checked bit-exact against these doubles).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

# (end epoch, multiplier of eta_base)
SLOW_START = ((40, 0.5), (70, 0.075), (85, 0.01), (90, 0.001))
# PAPER.md:222
GOYAL = ((30, 1.0), (60, 0.1), (80, 0.01), (90, 0.001))
SCHEDULES = {"slow_start": SLOW_START, "goyal": GOYAL}

N_TRAIN_IMAGENET = 1_281_167  # R5


@dataclass(frozen=True)
class Hyper:
    """PAPER.md:167 (mu1, mu2, eps), PAPER.md:190 (beta_center, beta_period),
    PAPER.md:192 (eta_RMSprop)."""
    mu1: float = 0.9
    mu2: float = 0.99
    eps: float = 1e-8
    eta_rmsprop: float = 0.0003
    beta_center: float = 10.0
    beta_period: float = 5.0


@dataclass(frozen=True)
class Cluster:
    """Logical cluster shape that drives eta_base."""
    n_workers: int = 1024
    b_local: int = 32
    n_train: int = N_TRAIN_IMAGENET
    schedule: str = "slow_start"
    transition: str = "elu"      # R20: "elu" (the paper's), "linear", "sigmoid", "sudden"

    @property
    def b_total(self) -> int:
        return self.n_workers * self.b_local


@dataclass(frozen=True)
class Coeffs:
    epoch: float
    eta: float
    alpha_sgd: float
    alpha_rmsprop: float
    phase: int


class ScheduleRangeError(ValueError):
    pass


def eta_base(n_workers: int, b_local: int) -> float:
    """eta_base = 0.1 * b_total / 256 = 0.1 * n b_local / 256."""
    b_total = n_workers * b_local
    return 0.1 * b_total / 256


def alpha_sgd_at(epoch: float, beta_center: float = 10.0, beta_period: float = 5.0,
                 transition: str = "elu") -> float:
    """PAPER.md:178-182 with reading R1 (slope 1/beta_period on the linear branch):
        1/2 exp(2 (epoch - beta_c) / beta_p)      epoch < beta_c
        1/2 + (epoch - beta_c) / beta_p             epoch < beta_c + beta_p / 2
        1                                           otherwise
    Reading R20, the alternatives PAPER.md:205-210 names without formulas, each
    through 1/2 at beta_c with the ELU's slope 1/beta_p there:
        linear   min(max(1/2 + (epoch - beta_c) / beta_p, 0), 1)
        sigmoid  1 / (1 + exp(-4 (epoch - beta_c) / beta_p))
        sudden   0 if epoch < beta_c else 1       (Wu et al.'s switch)
    """
    if beta_period <= 0:
        raise ValueError("beta_period must be > 0")
    if epoch < 0:
        raise ValueError("epoch must be >= 0")
    if transition == "elu":
        if epoch < beta_center:
            return 0.5 * math.exp(2.0 * (epoch - beta_center) / beta_period)
        if epoch < beta_center + 0.5 * beta_period:
            return 0.5 + (epoch - beta_center) / beta_period
        return 1.0
    if transition == "linear":
        return min(max(0.5 + (epoch - beta_center) / beta_period, 0.0), 1.0)
    if transition == "sigmoid":
        return 1.0 / (1.0 + math.exp(-4.0 * (epoch - beta_center) / beta_period))
    if transition == "sudden":
        return 0.0 if epoch < beta_center else 1.0
    raise ValueError(f"unknown transition {transition!r}")


def phase_at(t: int, cl: Cluster) -> int:
    """Index of the LR phase containing step t: the first p with
    (t-1) b_total < E_p N_train (integer test, right-open, R3/R4)."""
    num = (t - 1) * cl.b_total
    for p, (end, _) in enumerate(SCHEDULES[cl.schedule]):
        if num < end * cl.n_train:
            return p
    raise ScheduleRangeError(f"step {t} is past the last epoch of the schedule")


def n_steps(cl: Cluster) -> int:
    """Number of iterations T covering the schedule: the largest t with
    (t-1) b_total < E_last N_train."""
    end = SCHEDULES[cl.schedule][-1][0]
    return -(-(end * cl.n_train) // cl.b_total)


def coeffs_at(t: int, hyper: Hyper = Hyper(), cl: Cluster = Cluster()) -> Coeffs:
    """Coefficients for step t (t >= 1), PAPER.md:192-196 and PAPER.md:216-230:
        epoch   = ((t-1) b_total) / N_train
        eta     = mult_phase * eta_base                       (eta = eta_SGD)
        a_SGD   = alpha_sgd_at(epoch)
        a_RMS   = ((1 - a_SGD) eta_RMSprop) / eta
    """
    if t < 1:
        raise ValueError("t must be >= 1")
    epoch = ((t - 1) * cl.b_total) / cl.n_train
    p = phase_at(t, cl)
    eta = SCHEDULES[cl.schedule][p][1] * eta_base(cl.n_workers, cl.b_local)
    if not eta > 0:
        raise ValueError("eta must be > 0")
    a_sgd = alpha_sgd_at(epoch, hyper.beta_center, hyper.beta_period, cl.transition)
    a_rms = ((1.0 - a_sgd) * hyper.eta_rmsprop) / eta
    return Coeffs(epoch, eta, a_sgd, a_rms, p)


def lr_at_epoch(epoch: float, base: float, schedule: str = "slow_start") -> float:
    """Piecewise-constant LR at a real epoch, right-open phases (R4); used by the
    schedule pins."""
    for end, mult in SCHEDULES[schedule]:
        if epoch < end:
            return mult * base
    raise ScheduleRangeError("epoch past the schedule")
