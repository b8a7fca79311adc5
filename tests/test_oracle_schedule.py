"""Pins for oracle.schedule (readings R1-R5).

Pinned against: paper-printed values (tests/golden/paper_values.json), closed forms
(alpha(0) = e^-4 / 2, alpha_RMSprop at epoch 0/10), the prose constraints the
paper states (continuity, "reaches 1/2", "becomes 1", monotone increase), the
integral of the slow-start schedule, and the linear scaling rule.
"""
import math

import numpy as np
import pytest

from oracle import schedule as sch


def test_hyper_defaults_match_paper(golden):
    h = sch.Hyper()
    for k in ("mu1", "mu2", "eps", "beta_center", "beta_period", "eta_rmsprop"):
        assert getattr(h, k) == golden["hyper"][k]["value"]


def test_eta_base(golden):
    eb = golden["eta_base"]
    assert sch.eta_base(eb["n_workers"], eb["b_local"]) == eb["value"]   # PAPER.md:221, exact
    assert sch.eta_base(8, 32) == 0.1                                     # b_total = 256 anchor
    assert sch.eta_base(4, 8) == 0.0125
    for k in (2, 3, 7, 64):                                               # linear in b_total
        assert math.isclose(sch.eta_base(1024 * k, 32), k * 12.8, rel_tol=1e-15)


@pytest.mark.parametrize("name", ["slow_start", "goyal"])
def test_lr_phases(golden, name):
    for start, end, mult in golden[name]["phases"]:
        for e in (start, (start + end) / 2, end - 1e-9):
            assert sch.lr_at_epoch(e, 12.8, name) == pytest.approx(mult * 12.8, rel=1e-15)
    with pytest.raises(sch.ScheduleRangeError):
        sch.lr_at_epoch(90.0, 12.8, name)


def test_slow_start_values_at_phase_starts():
    # SPEC acceptance #2: {6.4, 0.96, 0.128, 0.0128} at epochs {0, 40, 70, 85}
    got = [sch.lr_at_epoch(e, 12.8) for e in (0, 40, 70, 85)]
    assert got == pytest.approx([6.4, 0.96, 0.128, 0.0128], rel=1e-15)


def test_slow_start_integral():
    # sum of lr over a 0.001-epoch grid, eta_base = 1: 0.5*40 + 0.075*30 + 0.01*15 + 0.001*5
    grid = np.arange(0, 90, 0.001)
    total = sum(sch.lr_at_epoch(float(e), 1.0) for e in grid) * 0.001
    assert abs(total - 22.405) < 1e-3


def test_alpha_paper_points(golden):
    for p in golden["alpha_sgd_points"]:
        assert sch.alpha_sgd_at(p["epoch"]) == p["value"]


def test_alpha_closed_forms():
    assert sch.alpha_sgd_at(0.0) == pytest.approx(0.5 * math.exp(-4.0), rel=1e-15)
    assert sch.alpha_sgd_at(0.0) == pytest.approx(0.00915781944436709, rel=1e-14)
    assert sch.alpha_sgd_at(11.25) == 0.75           # linear branch, slope 1/beta_period (R1)
    assert sch.alpha_sgd_at(5.0) == pytest.approx(0.5 * math.exp(-2.0), rel=1e-15)


def test_alpha_continuity_pins_reading_R1():
    # PAPER.md:186-188 prose: reaches 1/2 at beta_c, becomes 1 at beta_c + beta_p/2.
    # The displayed slope 2/beta_p would jump 1.5 -> 1 at 12.5.
    d = 1e-6
    for e in (10.0, 12.5):
        assert abs(sch.alpha_sgd_at(e - d) - sch.alpha_sgd_at(e + d)) < 1e-5
    # C^1 at beta_c: one-sided slopes both 1/beta_p = 0.2
    h = 1e-7
    left = (sch.alpha_sgd_at(10.0) - sch.alpha_sgd_at(10.0 - h)) / h
    right = (sch.alpha_sgd_at(10.0 + h) - sch.alpha_sgd_at(10.0)) / h
    assert left == pytest.approx(0.2, rel=1e-5) and right == pytest.approx(0.2, rel=1e-5)


def test_alpha_monotone_and_bounded():
    grid = np.linspace(0, 90, 90001)
    a = np.array([sch.alpha_sgd_at(float(e)) for e in grid])
    assert np.all(np.diff(a) >= 0) and a.min() > 0 and a.max() == 1.0


def test_alpha_errors():
    with pytest.raises(ValueError):
        sch.alpha_sgd_at(-1.0)
    with pytest.raises(ValueError):
        sch.alpha_sgd_at(1.0, 10.0, 0.0)


def test_alpha_rmsprop_closed_forms():
    # alpha_RMSprop = (1 - alpha_SGD) eta_RMSprop / eta_SGD
    cl = sch.Cluster()
    # epoch 10 at 32k: (1 - 1/2) * 3e-4 / 6.4 = 2.34375e-5
    t10 = next(t for t in range(1, 1000) if sch.coeffs_at(t).epoch >= 10.0)
    c0 = sch.coeffs_at(1)
    assert c0.epoch == 0.0 and c0.eta == pytest.approx(6.4, rel=1e-15) and c0.phase == 0
    assert c0.alpha_rmsprop == pytest.approx((1 - 0.5 * math.exp(-4)) * 3e-4 / 6.4, rel=1e-14)
    assert c0.alpha_rmsprop == pytest.approx(4.644572721354529e-05, rel=1e-14)
    c = sch.coeffs_at(t10, sch.Hyper(), cl)
    assert c.alpha_sgd >= 0.5
    # exactly at epoch 10 (construct a cluster where (t-1) b / N lands on 10):
    cl10 = sch.Cluster(n_workers=2, b_local=32, n_train=64)
    c = sch.coeffs_at(11, sch.Hyper(), cl10)
    assert c.epoch == 10.0 and c.alpha_sgd == 0.5
    assert c.alpha_rmsprop == pytest.approx(0.5 * 3e-4 / 0.0125, rel=1e-15)


def test_breakpoints_at_32k():
    """Start-of-step epoch (R3) with N_train = 1,281,167 (R5): the first steps at
    which alpha reaches 1/2 and 1 and the LR phases change, computed here by
    integer ceiling division, independently of coeffs_at's branch logic."""
    cl = sch.Cluster()
    def first_t(epoch_num, epoch_den=1):   # smallest t with (t-1) b >= epoch * N
        return -(-(epoch_num * cl.n_train) // (epoch_den * cl.b_total)) + 1
    assert first_t(10) == 392 and first_t(25, 2) == 490
    assert (first_t(40), first_t(70), first_t(85)) == (1565, 2738, 3325)
    assert sch.n_steps(cl) == 3519
    assert sch.coeffs_at(391).alpha_sgd < 0.5 <= sch.coeffs_at(392).alpha_sgd
    assert sch.coeffs_at(489).alpha_sgd < 1.0 == sch.coeffs_at(490).alpha_sgd
    assert sch.coeffs_at(490).alpha_rmsprop == 0.0
    for t, p in ((1564, 0), (1565, 1), (2737, 1), (2738, 2), (3324, 2), (3325, 3), (3519, 3)):
        assert sch.coeffs_at(t).phase == p
    with pytest.raises(sch.ScheduleRangeError):
        sch.coeffs_at(3520)


def test_coeffs_phase_matches_float_lookup():
    cl = sch.Cluster()
    for t in range(1, sch.n_steps(cl) + 1, 7):
        c = sch.coeffs_at(t)
        assert c.eta == sch.lr_at_epoch(c.epoch, 12.8)


def test_operation_order_of_alpha_rmsprop():
    # ((1 - a) * eta_R) / eta, in that order (the C++ schedule is checked bit-exact
    # against these doubles; the order is part of the contract)
    cl = sch.Cluster(n_workers=2, b_local=32, n_train=64)
    for t in range(1, 21):
        c = sch.coeffs_at(t, sch.Hyper(), cl)
        assert c.alpha_rmsprop == ((1.0 - c.alpha_sgd) * 0.0003) / c.eta


# ---- R20: the transition functions PAPER.md:205-210 names (f3) -------------------

@pytest.mark.parametrize("tr", ["elu", "linear", "sigmoid"])
def test_transition_half_at_center_with_elu_slope(tr):
    """Each smooth variant passes 1/2 at beta_center with the ELU's
    slope there, 1/beta_p (the exp branch's derivative, reading R1)."""
    for bc, bp in ((10.0, 5.0), (3.0, 2.0)):
        assert sch.alpha_sgd_at(bc, bc, bp, tr) == 0.5
        h = 1e-6
        slope = (sch.alpha_sgd_at(bc + h, bc, bp, tr) - sch.alpha_sgd_at(bc - h, bc, bp, tr)) / (2 * h)
        assert slope == pytest.approx(1.0 / bp, rel=1e-6)


def test_transition_closed_forms():
    # sigmoid: 1 / (1 + e^{-4 (e - 10) / 5}); at e = 15: 1/(1+e^-4), at e = 0: 1/(1+e^8)
    assert sch.alpha_sgd_at(15.0, transition="sigmoid") == pytest.approx(0.9820137900379085, rel=1e-15)
    assert sch.alpha_sgd_at(0.0, transition="sigmoid") == pytest.approx(3.353501304664781e-4, rel=1e-14)
    # linear: 0 up to beta_c - beta_p/2 = 7.5, 3/4 at 11.25, 1 from 12.5 on
    assert [sch.alpha_sgd_at(e, transition="linear") for e in (0.0, 7.5, 8.75, 11.25, 12.5, 80.0)] == \
           [0.0, 0.0, 0.25, 0.75, 1.0, 1.0]
    # sudden switch (Wu et al.) at beta_center
    assert [sch.alpha_sgd_at(e, transition="sudden") for e in (0.0, 9.999999, 10.0, 50.0)] == [0.0, 0.0, 1.0, 1.0]
    with pytest.raises(ValueError):
        sch.alpha_sgd_at(1.0, transition="cosine")


@pytest.mark.parametrize("tr", ["elu", "linear", "sigmoid", "sudden"])
def test_transition_monotone_bounded_and_rms_closed_form(tr):
    cl = sch.Cluster(transition=tr)
    prev = -1.0
    for t in range(1, sch.n_steps(cl) + 1, 5):
        c = sch.coeffs_at(t, sch.Hyper(), cl)
        assert 0.0 <= c.alpha_sgd <= 1.0 and c.alpha_sgd >= prev
        prev = c.alpha_sgd
        assert c.alpha_rmsprop == ((1.0 - c.alpha_sgd) * 3e-4) / c.eta
    # sudden at 32k: pure RMSprop (alpha_RMS = eta_R / eta) until t = 392, then SGD
    if tr == "sudden":
        assert sch.coeffs_at(391, sch.Hyper(), cl).alpha_rmsprop == 3e-4 / 6.4
        assert sch.coeffs_at(392, sch.Hyper(), cl).alpha_rmsprop == 0.0
