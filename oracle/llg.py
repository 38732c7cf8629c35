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
