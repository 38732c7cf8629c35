"""Dicke-model benchmark (oracle).  Test infrastructure only.

Mapping: B_eff = B_ext = (0, 0, w_z/gamma), B_rms = (sqrt(2/S) lambda/gamma, 0, 0),
with S = M_s V_c / (hbar gamma).  lambda_c = sqrt(w_c w_z)/2.
Equilibrium m_x (eq:dickeeqmag); polaritons (eq:dickepolaritons; the
superradiant branch is read with (w_z^2/mu^2 - w_c^2)^2 under the root, reading C18).
The explicit reference integrates the joint spin + cavity ODE
(eq:eqmotionspinclasical / eq:eqmotionaclasical) with kappa via w_c -> w_c - i kappa.
"""
from __future__ import annotations

import math

import numpy as np

from .constants import GAMMA, HBAR
from .llg import normalize


def spin_S(Ms, vcell, hbar=HBAR, gamma=GAMMA):
    """S = M_s V_c / (hbar gamma)."""
    return Ms * vcell / (hbar * gamma)


def mapping(omega_z, lam, Ms, vcell, hbar=HBAR, gamma=GAMMA):
    """(B_ext, B_rms) of P:403-404."""
    S = spin_S(Ms, vcell, hbar, gamma)
    return (0.0, 0.0, omega_z / gamma), (math.sqrt(2.0 / S) * lam / gamma, 0.0, 0.0)


def lambda_c(omega_c, omega_z):
    return math.sqrt(omega_c * omega_z) / 2


def mx_equilibrium(lam, omega_c, omega_z, kappa=0.0):
    """|m_x| at equilibrium: 0 below lambda_c, sqrt(1 - mu^2) above, mu = (lambda_c/lambda)^2
    (P:410-416); with cavity loss mu -> mu (1 + kappa^2/w_c^2) (reading C19)."""
    lc = lambda_c(omega_c, omega_z)
    mu = (lc / lam) ** 2 * (1 + kappa**2 / omega_c**2)
    return 0.0 if mu >= 1 else math.sqrt(1 - mu * mu)


def polaritons(omega_z, omega_c, lam):
    """(Omega_-, Omega_+) of eq:dickepolaritons (reading C18)."""
    lc = lambda_c(omega_c, omega_z)
    if lam < lc:
        a = omega_z**2 + omega_c**2
        b = math.sqrt((omega_z**2 - omega_c**2) ** 2 + 16 * lam**2 * omega_z * omega_c)
    else:
        mu = (lc / lam) ** 2
        a = omega_z**2 / mu**2 + omega_c**2
        b = math.sqrt((omega_z**2 / mu**2 - omega_c**2) ** 2 + 4 * omega_z**2 * omega_c**2)
    return math.sqrt((a - b) / 2), math.sqrt((a + b) / 2)


def joint_rhs(m, a, bext, brms, alpha, omega_c, kappa, Ms, vcell, hbar=HBAR, gamma=GAMMA):
    """Explicit joint ODE: dm/dt = LLG with B' = B_ext + B_rms 2Re(a);
    da/dt = -(i w_c + kappa) a + i (V_c/hbar) M_s m . B_rms (P:220 with S = -M_s V_c m/gamma)."""
    B = np.asarray(bext) + np.asarray(brms) * 2 * a.real
    mxB = np.cross(m, B)
    dm = -gamma / (1 + alpha**2) * (mxB + alpha * np.cross(m, mxB))
    W = Ms * float(np.dot(m, brms))
    da = -(1j * omega_c + kappa) * a + 1j * (vcell / hbar) * W
    return dm, da


def explicit_rk4(m0, a0, dt, steps, record_every=1, **kw):
    """Fixed-step RK4 on the joint (m, alpha) system, m renormalised each stage (as C2)."""
    m = np.asarray(m0, float).copy()
    a = complex(a0)
    out_m, out_a = [m.copy()], [a]
    for n in range(steps):
        k1m, k1a = joint_rhs(m, a, **kw)
        m2, a2 = normalize(m + 0.5 * dt * k1m), a + 0.5 * dt * k1a
        k2m, k2a = joint_rhs(m2, a2, **kw)
        m3, a3 = normalize(m + 0.5 * dt * k2m), a + 0.5 * dt * k2a
        k3m, k3a = joint_rhs(m3, a3, **kw)
        m4, a4 = normalize(m + dt * k3m), a + dt * k3a
        k4m, k4a = joint_rhs(m4, a4, **kw)
        m = normalize(m + dt / 6 * (k1m + 2 * k2m + 2 * k3m + k4m))
        a = a + dt / 6 * (k1a + 2 * k2a + 2 * k3a + k4a)
        if (n + 1) % record_every == 0:
            out_m.append(m.copy())
            out_a.append(a)
    return np.array(out_m), np.array(out_a)


def explicit_scipy(m0, a0, t_eval, rtol=1e-10, atol=1e-12, **kw):
    """The paper's reference route: SciPy's default-family integrator (DOP853 here)."""
    from scipy.integrate import solve_ivp

    def f(t, y):
        m = y[:3]
        a = complex(y[3], y[4])
        dm, da = joint_rhs(m, a, **kw)
        return np.concatenate([dm, [da.real, da.imag]])

    y0 = np.concatenate([np.asarray(m0, float), [complex(a0).real, complex(a0).imag]])
    sol = solve_ivp(f, (0.0, float(t_eval[-1])), y0, method="DOP853", t_eval=t_eval, rtol=rtol, atol=atol)
    return sol.y[:3].T, sol.y[3] + 1j * sol.y[4]
