"""Pins for oracle.llg / oracle.sim / oracle.cavity: closed-form dynamics, convergence orders,
the literal memory recursion against brute-force re-summation and the complex-alpha form."""
import math

import numpy as np
import pytest

from oracle import sim as S
from oracle import cavity as C
from oracle.constants import GAMMA, HBAR


def macrospin(m0, bext, alpha=0.0, cell=(5e-9,) * 3, demag="off", **kw):
    return S.Simulation((1, 1, 1), cell, 1.4e5, 3.7e-12, alpha, np.asarray(m0, float)[None],
                        bext=bext, demag=demag, **kw)


def test_larmor_precession_phase():
    B = 0.2
    th = 0.4
    sim = macrospin([math.sin(th), 0, math.cos(th)], (0, 0, B))
    w = GAMMA * B
    dt = 2 * math.pi / w / 200
    sim.run(dt, 1000)
    t = 1000 * dt
    expect = np.array([math.sin(th) * math.cos(w * t), math.sin(th) * math.sin(w * t), math.cos(th)])
    assert np.allclose(sim.m[0, 0, 0], expect, atol=5e-7)   # RK4 phase error ~(w dt)^4 w t/120


def test_damped_macrospin_closed_form():
    B, alpha, th0 = 0.5, 0.1, 2.0
    sim = macrospin([math.sin(th0), 0, math.cos(th0)], (0, 0, B), alpha=alpha)
    dt = 2 * math.pi / (GAMMA * B) / 100
    sim.run(dt, 600)
    t = 600 * dt
    th = 2 * math.atan(math.tan(th0 / 2) * math.exp(-alpha * GAMMA * B * t / (1 + alpha**2)))
    assert abs(math.acos(sim.m[0, 0, 0, 2]) - th) < 1e-6   # RK4 truncation at 100 steps/period


def _nonlinear_sim(alpha=0.0):
    rng = np.random.default_rng(3)
    m0 = rng.normal(size=(2 * 3 * 4, 3)) * 0.3 + np.array([0, 0, 1.0])
    m0 /= np.linalg.norm(m0, axis=1, keepdims=True)
    return S.Simulation((4, 3, 2), (5e-9, 5e-9, 5e-9), 8e5, 1.3e-11, alpha, m0, bext=(0.01, 0.0, 0.1),
                        aniso={"ku1": 5e4, "u": (0.3, 0.0, 1.0)}, demag="brute")


def test_rk4_fourth_order():
    T_ = 10e-12
    ref = _nonlinear_sim()
    ref.run(T_ / 1280, 1280)
    errs = []
    for n in (40, 80, 160):
        s = _nonlinear_sim()
        s.run(T_ / n, n)
        errs.append(np.abs(s.m - ref.m).max())
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 12 < r1 < 20 and 12 < r2 < 20, errs


def test_unit_norm_and_energy_conservation_rate():
    drifts = []
    for n in (40, 80):
        s = _nonlinear_sim(alpha=0.0)
        e0 = s.energy()
        s.run(10e-12 / n, n)
        assert np.allclose(np.linalg.norm(s.m, axis=-1), 1.0, atol=1e-14)
        drifts.append(abs(s.energy() - e0) / abs(e0))
    assert drifts[0] / drifts[1] > 10          # ~dt^4 (RK4 order, cavity off)


def test_damping_decreases_energy():
    s = _nonlinear_sim(alpha=0.05)
    e = [s.energy()]
    for _ in range(5):
        s.run(1e-12, 10)
        e.append(s.energy())
    assert all(b < a for a, b in zip(e, e[1:]))


# ------------------------------------------------------------------ cavity memory

def test_gamma_initial_value_and_ringdown():
    wc, k = 2 * math.pi * 5e9, 2 * math.pi * 50e6
    mem = C.CavityMemory(wc, k, x0=0.7, p0=-0.3, vcell=1e-25)
    assert mem.gamma(0.0) == pytest.approx(0.7)
    dt = 1e-12
    for _ in range(1000):
        mem.update(0.0, dt)
    t = mem.t
    expect = math.exp(-k * t) * (0.7 * math.cos(wc * t) + 0.3 * math.sin(wc * t))
    assert mem.gamma(t) == pytest.approx(expect, rel=1e-12)
    a = mem.alpha()
    a0 = complex(0.7, 0.3) / 2
    assert a == pytest.approx(a0 * complex(math.cos(-wc * t), math.sin(-wc * t)) * math.exp(-k * t), rel=1e-12)
    assert 2 * a.real == pytest.approx(mem.gamma(t), rel=1e-12)


def test_literal_recursion_equals_resummation_and_complex_alpha():
    """the recursion equals brute-force re-summation of the memory integral; reading C5:
    it also equals alpha_{n+1} = e^{-(kappa+i w)dt} alpha_n + i (Vc/hbar) W dt."""
    rng = np.random.default_rng(1)
    wc, k, vc = 2 * math.pi * 13.2e9, 2 * math.pi * 1e8, 4.77e-25
    x0, p0 = 0.2, -0.1
    mem = C.CavityMemory(wc, k, x0, p0, vc)
    dt = 0.5e-12
    a = complex(x0, -p0) / 2
    ts, Ws = [], []
    scale = HBAR / vc / dt * 1e-3
    for n in range(10_000):
        W = scale * rng.normal()
        mem.update(W, dt)
        ts.append(mem.t)
        Ws.append(W)
        a = complex(math.cos(-wc * dt), math.sin(-wc * dt)) * math.exp(-k * dt) * a + 1j * vc / HBAR * W * dt
        if n % 997 == 0 or n == 9999:
            g = mem.gamma(mem.t)
            assert 2 * a.real == pytest.approx(g, rel=1e-9, abs=1e-12)
            assert mem.alpha() == pytest.approx(a, rel=1e-9, abs=1e-12)
    g_lit = mem.gamma(mem.t)
    g_brute = C.gamma_resummed(ts, Ws, mem.t, wc, k, x0, p0, vc)
    assert abs(g_lit - g_brute) <= 1e-10 * max(1.0, abs(g_brute))


def test_reset_idempotent():
    mem = C.CavityMemory(1e10, 1e7, 0.5, 0.1, 1e-24)
    mem.update(3.0, 1e-12)
    mem.reset()
    st = (mem.S, mem.C, mem.t, mem.step)
    mem.reset()
    assert (mem.S, mem.C, mem.t, mem.step) == st == (0.0, 0.0, 0.0, 0)


def test_overflow_guard():
    mem = C.CavityMemory(1e10, 1e12, vcell=1e-24)
    with pytest.raises(OverflowError):
        mem.gamma(1e-9)


def test_zero_brms_cavity_is_bitwise_cavity_off():
    """Reading C14: B_rms = 0, x0 = p0 = 0 gives exactly the cavity-off trajectory."""
    a = _nonlinear_sim(alpha=0.01)
    b = _nonlinear_sim(alpha=0.01)
    b.mem = C.CavityMemory(2 * math.pi * 10e9, 1e7, 0.0, 0.0, b.vcell)
    a.run(0.5e-12, 20)
    b.run(0.5e-12, 20)
    assert np.array_equal(a.m, b.m)
    assert not b.cavity_enabled


def test_relax_reaches_tolerance_and_resets_memory():
    s = _nonlinear_sim(alpha=0.0)
    s.mem.update(1.0, 1e-12)
    n = s.relax(2e-13, 1e-4, 20000, check_every=50)
    assert n < 20000 and n % 50 == 0
    assert s.max_torque() < 1e-4
    assert s.mem.t == 0.0 and s.mem.S == 0.0
