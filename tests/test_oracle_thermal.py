"""Pins of the oracle's thermal field (reading C-TH; P:188 lists the thermal field among the
Mumax3 terms).  The generator is pinned to SplitMix64's published output, the normals to their
distribution, and the field's scale to physics: an ensemble of non-interacting macrospins in a
field relaxes to the Langevin magnetisation <m_z> = coth x - 1/x, x = M_s V B / (k_B T)
(Boltzmann statistics on the sphere) — a wrong factor 2, alpha, gamma, M_s V or dt in sigma, or
noise redrawn per stage, moves <m_z> far outside the tolerance."""
import math

import numpy as np
import pytest

from oracle import thermal as TH
from oracle import sim as S
from oracle.constants import KB, GAMMA


def test_splitmix64_reference_outputs():
    # SplitMix64 (Steele, Lea & Flood 2014; Vigna's splitmix64.c) started at state 0: the
    # first four outputs of the reference generator
    got = [int(x) for x in TH.splitmix64(0, np.arange(4))]
    assert got == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F, 0xF88BB8A8724C81EC]
    # counter c of the stream started at s is the (c+1)-th step of the same recurrence
    s = 0x0123456789ABCDEF
    assert int(TH.splitmix64(s, np.array([5]))[0]) == int(TH.splitmix64(s + 5 * 0x9E3779B97F4A7C15 % 2**64, np.array([0]))[0])


def test_eta_is_standard_normal_and_independent():
    from scipy import stats
    e = TH.eta((64, 64, 16), seed=12345, step=3).reshape(-1, 3)
    n = e.shape[0]
    for c in range(3):
        x = e[:, c]
        assert abs(x.mean()) < 5 / math.sqrt(n)
        assert abs(x.var() - 1.0) < 5 * math.sqrt(2.0 / n)
        assert stats.kstest(x, "norm").pvalue > 1e-4
    cc = np.corrcoef(e.T)
    assert np.all(np.abs(cc - np.eye(3)) < 5 / math.sqrt(n))
    nxt = TH.eta((64, 64, 16), seed=12345, step=4).reshape(-1, 3)         # the next step's draw
    other = TH.eta((64, 64, 16), seed=54321, step=3).reshape(-1, 3)       # another seed
    for f in (nxt, other):
        assert abs(np.corrcoef(e[:, 0], f[:, 0])[0, 1]) < 5 / math.sqrt(n)
    assert np.array_equal(e, TH.eta((64, 64, 16), seed=12345, step=3).reshape(-1, 3))


def test_thermal_field_zero_in_vacuum_and_off_at_zero_temperature():
    grid = (6, 5, 2)
    mask = np.zeros((2, 5, 6), bool)
    mask[:, 1:4, 2:5] = True
    m0 = np.tile([0.0, 0.0, 1.0], (60, 1))
    sim = S.Simulation(grid, (5e-9,) * 3, 1.4e5, 0.0, 0.5, m0, mask=mask.reshape(-1), temperature=300.0, seed=9)
    sim.run(1e-13, 2)
    B = sim.field(sim.m, sim.mem.t, S.THERM)
    assert np.all(B[~mask] == 0) and np.all(B[mask] != 0)
    sig = TH.sigma(0.5, 300.0, GAMMA, 1.4e5, 1.25e-25, 1e-13)
    assert np.allclose(B[mask], sig * TH.eta((2, 5, 6), 9, 2)[mask], rtol=1e-15, atol=0)
    cold = S.Simulation(grid, (5e-9,) * 3, 1.4e5, 0.0, 0.5, m0, mask=mask.reshape(-1))
    cold.run(1e-13, 2)
    assert np.all(cold.field(cold.m, cold.mem.t, S.THERM) == 0)
    with pytest.raises(RuntimeError):
        sim.step_dp(1e-13)


def test_langevin_equilibrium_of_independent_macrospins():
    """256 uncoupled cells (A = 0, Zeeman only) in B = 0.5 T along z at x = 2."""
    grid, cell, Ms, alpha, B = (16, 16, 1), (5e-9,) * 3, 1.4e5, 1.0, 0.5
    V = cell[0] * cell[1] * cell[2]
    x = 2.0
    T = Ms * V * B / (KB * x)
    rng = np.random.default_rng(1)
    m0 = rng.normal(size=(256, 3))
    m0 /= np.linalg.norm(m0, axis=1, keepdims=True)
    sim = S.Simulation(grid, cell, Ms, 0.0, alpha, m0, bext=(0.0, 0.0, B), terms=S.ZEEMAN,
                       temperature=T, seed=2024)
    dt = 1e-13                                   # relaxation time (1 + a^2)/(a gamma B) = 230 dt
    sim.run(dt, 1000)
    acc = []
    for _ in range(50):
        sim.run(dt, 100)
        acc.append(sim.m[..., 2].mean())
    langevin = 1.0 / math.tanh(x) - 1.0 / x      # 0.5373
    assert abs(np.mean(acc) - langevin) < 0.03, (np.mean(acc), langevin)
    # the same ensemble at 3x the temperature sits at L(x/3) = 0.2143: the scale is not fixed
    # by the test's choice of T
    hot = S.Simulation(grid, cell, Ms, 0.0, alpha, m0, bext=(0.0, 0.0, B), terms=S.ZEEMAN,
                       temperature=3 * T, seed=7)
    hot.run(dt, 1000)
    acc = []
    for _ in range(50):
        hot.run(dt, 100)
        acc.append(hot.m[..., 2].mean())
    assert abs(np.mean(acc) - (1.0 / math.tanh(x / 3) - 3.0 / x)) < 0.03
