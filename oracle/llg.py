"""LLG torque and the fixed-step RK4 integrator (oracle, fp64).  Test infrastructure only.

dm/dt = -gamma/(1+alpha^2) [ m x B' + alpha m x (m x B') ]      (eq:llg; B' = B_eff +
B_cav in both terms).  Integrator: classical RK4 with a fixed step (reading C1)
and renormalisation of every stage state and of the step result (reading C2):
  k1 = f(m_n, t_n);            m2 = norm(m_n + dt/2 k1)
  k2 = f(m2, t_n + dt/2);      m3 = norm(m_n + dt/2 k2)
  k3 = f(m3, t_n + dt/2);      m4 = norm(m_n + dt k3)
  k4 = f(m4, t_n + dt);        m_{n+1} = norm(m_n + dt/6 (k1 + 2k2 + 2k3 + k4))
"""
from __future__ import annotations

import numpy as np

from .constants import GAMMA


def torque(m, B, alpha, gamma=GAMMA):
    mxB = np.cross(m, B)
    return -gamma / (1 + alpha * alpha) * (mxB + alpha * np.cross(m, mxB))


def relax_torque(m, B, gamma=GAMMA):
    """Damping-only flow used by relax (reading C15): -gamma m x (m x B)."""
    return -gamma * np.cross(m, np.cross(m, B))


def normalize(v):
    """v/|v|, with v = 0 (vacuum) kept at 0."""
    n = np.linalg.norm(v, axis=-1, keepdims=True)
    return np.where(n > 0, v / np.where(n > 0, n, 1.0), 0.0)


def rk4_step(f, m, t, dt):
    """One RK4 step of dm/dt = f(m, t) with stage renormalisation.  Returns m_{n+1}."""
    k1 = f(m, t)
    m2 = normalize(m + 0.5 * dt * k1)
    k2 = f(m2, t + 0.5 * dt)
    m3 = normalize(m + 0.5 * dt * k2)
    k3 = f(m3, t + 0.5 * dt)
    m4 = normalize(m + dt * k3)
    k4 = f(m4, t + dt)
    return normalize(m + dt / 6.0 * (k1 + 2 * k2 + 2 * k3 + k4))


# ---------------------------------------------------------------- Dormand-Prince 5(4) (NEXT-1)
# Mumax3 integrates with its own (adaptive) solvers, unmodified; SURVEY §8(f) NEXT-1 names
# Dormand-Prince RK45.  Reading C-DP: the standard DP5(4) tableau (Dormand & Prince 1980), every
# stage state renormalised like C2, the 5th-order solution propagated (a_7j = b5_j, so stage 7's
# state is the step result), and the local error estimate e = dt sum_j (b5_j - b4_j) k_j with
# err = max_i |e_i| over cells.  No FSAL reuse (k7 is evaluated for the estimate only).
DP_C = (0.0, 1 / 5, 3 / 10, 4 / 5, 8 / 9, 1.0, 1.0)
DP_A = ((),
        (1 / 5,),
        (3 / 40, 9 / 40),
        (44 / 45, -56 / 15, 32 / 9),
        (19372 / 6561, -25360 / 2187, 64448 / 6561, -212 / 729),
        (9017 / 3168, -355 / 33, 46732 / 5247, 49 / 176, -5103 / 18656),
        (35 / 384, 0.0, 500 / 1113, 125 / 192, -2187 / 6784, 11 / 84))
DP_B5 = (35 / 384, 0.0, 500 / 1113, 125 / 192, -2187 / 6784, 11 / 84, 0.0)
DP_B4 = (5179 / 57600, 0.0, 7571 / 16695, 393 / 640, -92097 / 339200, 187 / 2100, 1 / 40)


def dp45_step(f, m, t, dt):
    """One Dormand-Prince step of dm/dt = f(m, t): returns (m_{n+1} (5th order, renormalised),
    err = max_i |dt sum_j (b5_j - b4_j) k_j|)."""
    ks = []
    ms = m
    for s in range(7):
        if s > 0:
            ms = normalize(m + dt * sum(a * k for a, k in zip(DP_A[s], ks)))
        ks.append(f(ms, t + DP_C[s] * dt))
    e = dt * sum((b5 - b4) * k for b5, b4, k in zip(DP_B5, DP_B4, ks))
    return ms, float(np.max(np.linalg.norm(e, axis=-1)))


def dp_controller(dt, err, tol):
    """Next step size after an attempt (standard 5th-order controller, safety 0.9, growth in
    [0.2, 5]); err == 0 grows by the maximum factor."""
    if err <= 0.0:
        return dt * 5.0
    return dt * min(5.0, max(0.2, 0.9 * (tol / err) ** 0.2))
