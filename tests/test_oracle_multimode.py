"""Pins of the oracle's multimode cavity (reading C-MM in DESIGN.md):
each extra mode is its own damped oscillator driven by its own overlap, the field is the sum.

* an extra mode with B_rms = 0 changes nothing (bit for bit);
* two degenerate modes with maps c1 b and c2 b act exactly like one mode with map s b,
  s^2 = c1^2 + c2^2 (the magnet couples to the bright combination; the orthogonal one is dark) —
  a dropped mode, a shared overlap or a wrong sum in the field breaks it;
* a macrospin coupled to two modes at different frequencies shows the three normal modes of
  three position-coupled oscillators, the textbook generalisation of the two-oscillator formula
  pinned in test_oracle_physics.py (P:419 with lambda -> g)."""
import math

import numpy as np
import pytest

from oracle import sim as S
from oracle import analytic as A
from oracle.constants import GAMMA

CELL = (5e-9, 5e-9, 5e-9)
MS = 1.4e5
V = float(np.prod(CELL))


def _bperp(g):
    return g / (GAMMA * math.sqrt(MS * V / (A.HBAR * GAMMA) / 2))


def _macrospin(brms, f_c, modes=(), kappa=0.0, B=0.3):
    return S.Simulation((1, 1, 1), CELL, MS, 0.0, 0.0, np.array([[0.0, 0.02, 1.0]]), bext=(0, 0, B),
                        brms_uniform=brms, f_c=f_c, kappa=kappa, demag="brute", modes=modes)


def test_zero_extra_mode_is_identity():
    w = GAMMA * 0.3
    b = (_bperp(0.05 * w), 0.0, 0.0)
    a = _macrospin(b, w / (2 * math.pi))
    c = _macrospin(b, w / (2 * math.pi), modes=[{"brms_uniform": (0.0, 0.0, 0.0), "f_c": 3e9}])
    dt = 2 * math.pi / w / 25
    a.run(dt, 200)
    c.run(dt, 200)
    assert np.array_equal(a.m, c.m)
    assert a.mem.alpha() == c.mem.alpha()


def test_degenerate_modes_equal_one_bright_mode():
    w = GAMMA * 0.3
    bp = _bperp(0.05 * w)
    fc, kap = w / (2 * math.pi), 2 * math.pi * 20e6
    one = _macrospin((bp, 0.0, 0.0), fc, kappa=kap)
    two = _macrospin((0.6 * bp, 0.0, 0.0), fc, kappa=kap,
                     modes=[{"brms_uniform": (0.8 * bp, 0.0, 0.0), "f_c": fc, "kappa": kap}])
    dt = 2 * math.pi / w / 25
    for _ in range(600):
        one.step(dt)
        two.step(dt)
    assert np.abs(one.m - two.m).max() < 1e-12
    a = one.mem.alpha()
    assert abs(two.mem.alpha() - 0.6 * a) < 1e-9 * abs(a)
    assert abs(two.extra[0][1].alpha() - 0.8 * a) < 1e-9 * abs(a)
    # a wrong split (0.6, 0.6) is not equivalent
    bad = _macrospin((0.6 * bp, 0.0, 0.0), fc, kappa=kap,
                     modes=[{"brms_uniform": (0.6 * bp, 0.0, 0.0), "f_c": fc, "kappa": kap}])
    for _ in range(600):
        bad.step(dt)
    assert np.abs(one.m - bad.m).max() > 1e-4


def test_two_modes_three_normal_modes():
    B = 0.3
    wz = GAMMA * B
    w1, w2 = wz, 1.1 * wz
    g1, g2 = 0.03 * wz, 0.03 * wz
    sim = _macrospin((_bperp(g1), 0.0, 0.0), w1 / (2 * math.pi), B=B,
                     modes=[{"brms_uniform": (_bperp(g2), 0.0, 0.0), "f_c": w2 / (2 * math.pi)}])
    dt = 2 * math.pi / wz / 25
    ys = []
    for _ in range(12000):
        sim.step(dt)
        ys.append(sim.m[0, 0, 0, 1])
    got = A.peaks(ys, dt, 3, window="hann", pad=8)
    # position-coupled oscillators: Omega^2 = eig([[wz^2, 2 g1 sqrt(wz w1), 2 g2 sqrt(wz w2)], ...])
    Mx = np.array([[wz * wz, 2 * g1 * math.sqrt(wz * w1), 2 * g2 * math.sqrt(wz * w2)],
                   [2 * g1 * math.sqrt(wz * w1), w1 * w1, 0.0],
                   [2 * g2 * math.sqrt(wz * w2), 0.0, w2 * w2]])
    want = np.sort(np.sqrt(np.linalg.eigvalsh(Mx))) / (2 * math.pi)
    # the 2x2 case of the same matrix is the pinned two-oscillator formula
    lo, hi = A.two_oscillator(wz, w1, g1)
    assert np.sqrt(np.linalg.eigvalsh(Mx[:2, :2])) == pytest.approx([lo, hi], rel=1e-12)
    assert np.array(got) == pytest.approx(want, rel=5e-3)
