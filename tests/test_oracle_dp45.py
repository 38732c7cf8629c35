"""Pins of the oracle's Dormand-Prince integrator (reading C-DP):
fifth-order convergence of the propagated solution, fourth/fifth-order scaling of the embedded
error estimate, the adaptive driver against the damped-macrospin closed form, and the cavity
recursion with variable steps equal to the same run re-stepped with the accepted step list."""
import math

import numpy as np
import pytest

from oracle import sim as S
from oracle import llg
from oracle.constants import GAMMA


def _nonlinear_sim(alpha=0.0, **kw):
    rng = np.random.default_rng(3)
    m0 = rng.normal(size=(2 * 3 * 4, 3)) * 0.3 + np.array([0, 0, 1.0])
    m0 /= np.linalg.norm(m0, axis=1, keepdims=True)
    return S.Simulation((4, 3, 2), (5e-9, 5e-9, 5e-9), 8e5, 1.3e-11, alpha, m0, bext=(0.01, 0.0, 0.1),
                        aniso={"ku1": 5e4, "u": (0.3, 0.0, 1.0)}, demag="brute", **kw)


def test_tableau_consistency():
    # row sums equal the nodes and both weight sets sum to one (the order conditions of degree 1)
    for c, a in zip(llg.DP_C, llg.DP_A):
        assert sum(a) == pytest.approx(c, abs=1e-15)
    assert sum(llg.DP_B5) == pytest.approx(1.0, abs=1e-15) and sum(llg.DP_B4) == pytest.approx(1.0, abs=1e-15)
    assert llg.DP_A[6] == tuple(llg.DP_B5[:6])


def test_dp5_fifth_order_and_error_estimate_scaling():
    T_ = 10e-12
    ref = _nonlinear_sim()
    for _ in range(1280):
        ref.step_dp(T_ / 1280)
    errs, ests = [], []
    for n in (40, 80, 160):
        s = _nonlinear_sim()
        e = [s.step_dp(T_ / n) for _ in range(n)]
        errs.append(np.abs(s.m - ref.m).max())
        ests.append(max(e))
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 25 < r1 < 50 and 26 < r2 < 40, errs              # global error ~ dt^5 (RK4 gave 16x)
    q1, q2 = ests[0] / ests[1], ests[1] / ests[2]
    assert 25 < q1 < 40 and 25 < q2 < 40, ests              # local estimate ~ dt^5
    rk = _nonlinear_sim()
    rk.run(T_ / 40, 40)
    assert errs[0] < 0.2 * np.abs(rk.m - ref.m).max()      # DP5 beats RK4 at equal dt


def test_adaptive_damped_macrospin_closed_form():
    B, alpha, th0 = 0.5, 0.1, 2.0
    T = 6 * 2 * math.pi / (GAMMA * B)
    th = 2 * math.atan(math.tan(th0 / 2) * math.exp(-alpha * GAMMA * B * T / (1 + alpha**2)))
    errs, steps = [], []
    for tol in (1e-5, 1e-7):
        sim = S.Simulation((1, 1, 1), (5e-9,) * 3, 1.4e5, 0.0, alpha,
                           np.array([[math.sin(th0), 0, math.cos(th0)]]), bext=(0, 0, B), demag="off")
        acc, rej, dt, dts = sim.run_adaptive(T, 1e-13, tol)
        assert sim.mem.t == pytest.approx(T, rel=1e-12) and sum(dts) == pytest.approx(T, rel=1e-12)
        errs.append(abs(math.acos(sim.m[0, 0, 0, 2]) - th))
        steps.append(acc)
    assert errs[0] < 1e-3 and errs[1] < errs[0] / 10        # tighter tolerance, smaller error
    assert 1.5 < steps[1] / steps[0] < 4.0                  # steps ~ tol^(-1/5): 100^(1/5) = 2.5


def test_variable_step_cavity_recursion_replays():
    """The cavity memory advanced with the accepted variable steps equals a re-run that takes
    exactly those steps (the recursion has no hidden state beyond (S, C) / alpha)."""
    kw = dict(brms_uniform=(2e-3, 0.0, 0.0), f_c=12e9, kappa=2 * math.pi * 30e6, x0=0.1, p0=-0.05)
    a = _nonlinear_sim(alpha=0.01, **kw)
    acc, rej, dt, dts = a.run_adaptive(20e-12, 1e-13, 1e-6)
    assert acc > 5 and len(set(np.round(np.array(dts) / 1e-15))) > 2   # the steps did vary
    b = _nonlinear_sim(alpha=0.01, **kw)
    for h in dts:
        b.step_dp(h)
    assert np.array_equal(a.m, b.m)
    assert a.mem.alpha() == b.mem.alpha() and a.mem.t == b.mem.t
