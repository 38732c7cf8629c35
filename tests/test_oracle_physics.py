"""Physics pins of the oracle: the paper's Dicke benchmark, Kittel frequencies, the
coupling law g ~ B_rms sqrt(V), the anticrossing and i_rms."""
import json
import math
import os

import numpy as np
import pytest

from oracle import sim as S
from oracle import dicke as D
from oracle import analytic as A
from oracle.constants import GAMMA, MU0

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))
CELL = (5e-9, 5e-9, 5e-9)
MS = 1.4e5
DICKE_TERMS = S.ZEEMAN | S.CAVITY | S.EXCITATION     # B_eff = B_ext + B_cav


def dicke_sim(wz, wc, lam, m0, alpha=0.0, kappa=0.0):
    bext, brms = D.mapping(wz, lam, MS, np.prod(CELL))
    return S.Simulation((1, 1, 1), CELL, MS, 0.0, alpha, np.asarray(m0, float)[None], bext=bext,
                        brms_uniform=brms, f_c=wc / (2 * math.pi), kappa=kappa, demag="off",
                        terms=DICKE_TERMS)


def zero_crossing_freq(x, dt):
    """Mean frequency (Hz) from linearly interpolated upward zero crossings (test helper)."""
    x = np.asarray(x) - np.mean(x)
    idx = np.nonzero((x[:-1] < 0) & (x[1:] >= 0))[0]
    tc = (idx + (-x[idx]) / (x[idx + 1] - x[idx])) * dt
    return (len(tc) - 1) / (tc[-1] - tc[0])


def test_golden_paper_values():
    g = GOLD["dicke_superradiant_mx"]
    w = 2 * math.pi * 10e9
    lc = D.lambda_c(w, w)
    assert abs(D.mx_equilibrium(g["lambda_over_lambda_c"] * lc, w, w) - g["abs_mx"]) < g["tol"]
    g = GOLD["i_rms_nA"]
    assert abs(A.i_rms(2 * math.pi * g["omega0_over_2pi"], g["Z0"]) * 1e9 - g["value"]) < g["tol"]
    g = GOLD["dark_current_ratio"]
    assert abs(g["i_bright_nA"] * g["f_dark_GHz"] / g["f_bright_GHz"] - g["i_dark_nA"]) < 0.5


def test_polariton_closed_forms():
    w = 1.0
    lam = 0.2
    om, op = D.polaritons(w, w, lam)
    assert om == pytest.approx(math.sqrt(w * w - 2 * lam * w)) and op == pytest.approx(math.sqrt(w * w + 2 * lam * w))
    # reading C18: both branches are real and Omega_- -> 0 continuously at lambda_c
    for wz, wc in [(1.0, 1.0), (0.7, 1.3)]:
        lc = D.lambda_c(wc, wz)
        below = D.polaritons(wz, wc, lc * (1 - 1e-6))[0]
        above = D.polaritons(wz, wc, lc * (1 + 1e-6))[0]
        assert below < 1e-2 and above < 1e-2
        for r in (1.1, 1.4, 3.0):
            a, b = D.polaritons(wz, wc, r * lc)
            assert 0 < a < b


def test_ide_converges_to_explicit_ode_first_order():
    """the memory-kernel (IDE) integration 'matches the evolution computed with
    Python' (the explicit joint ODE).  Under reading C3 (S_n, C_n frozen inside a step) the
    difference is first order in dt: the relative L2 error of m_x halves when dt halves."""
    w = 2 * math.pi * 10e9
    lam = 0.3 * D.lambda_c(w, w)
    m0 = np.array([0.05, 0.0, 1.0]); m0 /= np.linalg.norm(m0)
    bext, brms = D.mapping(w, lam, MS, np.prod(CELL))
    kw = dict(bext=bext, brms=brms, alpha=0.0, omega_c=w, kappa=0.0, Ms=MS, vcell=np.prod(CELL))
    errs = []
    for per in (50, 100, 200):
        sim = dicke_sim(w, w, lam, m0)
        dt = 2 * math.pi / w / per
        n = 10 * per
        mx_ide = [sim.m[0, 0, 0, 0]]
        for _ in range(n):
            sim.step(dt)
            mx_ide.append(sim.m[0, 0, 0, 0])
        ms, _ = D.explicit_rk4(m0, 0.0, dt, n, **kw)
        errs.append(np.linalg.norm(np.array(mx_ide) - ms[:, 0]) / np.linalg.norm(ms[:, 0]))
    assert 1.8 < errs[0] / errs[1] < 2.2 and 1.8 < errs[1] / errs[2] < 2.2, errs
    assert errs[2] < 5e-3
    # the explicit RK4 reference itself agrees with SciPy's DOP853 (the paper's own route)
    t = np.arange(n + 1) * dt
    ms2, _ = D.explicit_scipy(m0, 0.0, t, **kw)
    assert np.abs(ms2 - ms).max() < 1e-6


def test_dicke_polariton_peaks_normal_phase():
    """the spectrum of m_x peaks at Omega_+- (eq:dickepolaritons); 0.5% (BJ)."""
    w = 2 * math.pi * 10e9
    lam = 0.3 * D.lambda_c(w, w)
    m0 = np.array([0.02, 0.0, 1.0]); m0 /= np.linalg.norm(m0)
    sim = dicke_sim(w, w, lam, m0)
    dt = 2 * math.pi / w / 25
    xs = []
    for _ in range(6000):
        sim.step(dt)
        xs.append(sim.m[0, 0, 0, 0])
    pk = A.peaks(xs, dt, 2)
    om, op = D.polaritons(w, w, lam)
    assert pk[0] == pytest.approx(om / (2 * math.pi), rel=5e-3)
    assert pk[1] == pytest.approx(op / (2 * math.pi), rel=5e-3)


def test_dicke_superradiant_attractor_with_loss():
    """P:433-440 + reading C19: the dissipative superradiant run settles at |m_x| = sqrt(1-mu_k^2)."""
    w = 2 * math.pi * 10e9
    kappa = 0.05 * w
    lam = 1.4 * D.lambda_c(w, w)
    m0 = np.array([0.05, 0.0, 1.0]); m0 /= np.linalg.norm(m0)
    sim = dicke_sim(w, w, lam, m0, alpha=0.05, kappa=kappa)
    dt = 2 * math.pi / w / 40
    sim.run(dt, 8000)
    assert abs(abs(sim.m[0, 0, 0, 0]) - D.mx_equilibrium(lam, w, w, kappa)) < 2e-3


def test_kittel_single_cubic_cell():
    """A uniformly magnetised cube (N = 1/3 each) precesses at gamma B / 2 pi (BJ north_star)."""
    B = 0.3
    sim = S.Simulation((1, 1, 1), CELL, MS, 3.7e-12, 0.0, np.array([[0.05, 0.0, 1.0]]), bext=(0, 0, B),
                       demag="brute")
    dt = 2 * math.pi / (GAMMA * B) / 40
    xs = []
    for _ in range(2000):
        sim.step(dt)
        xs.append(sim.m[0, 0, 0, 0])
    assert zero_crossing_freq(xs, dt) == pytest.approx(GAMMA * B / (2 * math.pi), rel=1e-5)


def test_kittel_flat_cell_with_aharoni_factors():
    """Single flat cell, bias along x: w = gamma sqrt((B+(Ny-Nx)mu0Ms)(B+(Nz-Nx)mu0Ms))."""
    cell = (10e-9, 10e-9, 2e-9)
    Ms, B = 8.6e5, 0.1
    sim = S.Simulation((1, 1, 1), cell, Ms, 1.3e-11, 0.0, np.array([[1.0, 0.0, 0.01]]), bext=(B, 0, 0),
                       demag="brute")
    w = A.kittel_box(B, Ms, A.aharoni(*cell))
    dt = 2 * math.pi / w / 60
    zs = []
    for _ in range(3000):
        sim.step(dt)
        zs.append(sim.m[0, 0, 0, 2])
    assert zero_crossing_freq(zs, dt) == pytest.approx(w / (2 * math.pi), rel=1e-4)
    # thin-film limit of the box formula (dz/dx -> 0)
    assert A.kittel_box(B, Ms, A.aharoni(1e4, 1e4, 1.0)) == pytest.approx(A.kittel_film(B, Ms), rel=2e-3)


def _splitting(cell, Bperp, B=0.3, n=5000, per=25):
    w = GAMMA * B
    sim = S.Simulation((1, 1, 1), cell, MS, 0.0, 0.0, np.array([[0.0, 0.02, 1.0]]), bext=(0, 0, B),
                       brms_uniform=(Bperp, 0, 0), f_c=w / (2 * math.pi), demag="brute")
    dt = 2 * math.pi / w / per
    xs = []
    for _ in range(n):
        sim.step(dt)
        xs.append(sim.m[0, 0, 0, 1])
    lo, hi = A.peaks(xs, dt, 2, window="hann", pad=8)
    return 2 * math.pi * (hi - lo), w


def test_coupling_law_and_anticrossing():
    """g = gamma B_rms sqrt(S/2) with S = Ms V/(hbar gamma): the resonant splitting is
    Omega_+ - Omega_- of the two-oscillator model, and g ~ sqrt(V)."""
    V = np.prod(CELL)
    g_target = 0.05 * GAMMA * 0.3
    Bperp = g_target / (GAMMA * math.sqrt(MS * V / (A.HBAR * GAMMA) / 2))
    split1, w = _splitting(CELL, Bperp)
    om, op = A.two_oscillator(w, w, A.coupling_g(Bperp, MS, V))
    assert split1 == pytest.approx(op - om, rel=5e-3)
    cell2 = (CELL[0] * 2 ** (1 / 3),) * 3
    split2, _ = _splitting(cell2, Bperp)
    om2, op2 = A.two_oscillator(w, w, A.coupling_g(Bperp, MS, 2 * V))
    assert split2 == pytest.approx(op2 - om2, rel=5e-3)
    assert A.coupling_g(Bperp, MS, 2 * V) / A.coupling_g(Bperp, MS, V) == pytest.approx(math.sqrt(2))


def test_anticrossing_detuned():
    """Off resonance the two peaks follow the two-oscillator Omega_+- (lambda -> g)."""
    V = np.prod(CELL)
    B = 0.3
    wz = GAMMA * B
    wc = 1.1 * wz
    g = 0.04 * wz
    Bperp = g / (GAMMA * math.sqrt(MS * V / (A.HBAR * GAMMA) / 2))
    sim = S.Simulation((1, 1, 1), CELL, MS, 0.0, 0.0, np.array([[0.0, 0.02, 1.0]]), bext=(0, 0, B),
                       brms_uniform=(Bperp, 0, 0), f_c=wc / (2 * math.pi), demag="brute")
    dt = 2 * math.pi / wz / 25
    xs = []
    for _ in range(5000):
        sim.step(dt)
        xs.append(sim.m[0, 0, 0, 1])
    lo, hi = A.peaks(xs, dt, 2, window="hann", pad=8)
    om, op = A.two_oscillator(wz, wc, g)
    assert lo == pytest.approx(om / (2 * math.pi), rel=5e-3)
    assert hi == pytest.approx(op / (2 * math.pi), rel=5e-3)
