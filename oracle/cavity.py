"""Cavity memory term (oracle, fp64), literally as P:330-346.  Test infrastructure only.

Gamma(t_n) = e^{-k t_n} cos(w t_n)(x0 - 2Vc/hbar S_n) - e^{-k t_n} sin(w t_n)(p0 - 2Vc/hbar C_n)
                                                                       (eq:gammadiscretefinal)
S_n = S_{n-1} + e^{k t_n} sin(w t_n) W_n dt,  C_n = C_{n-1} + e^{k t_n} cos(w t_n) W_n dt,
S_0 = C_0 = 0                                           (eq:Sdiscrete / eq:Cdiscrete)
W_n = sum_i M_s,i m_i(t_n) . B_rms(r_i)
alpha(t) = e^{-(k+iw)t}[alpha0 - (Vc/hbar) S + i (Vc/hbar) C], alpha0 = (x0 - i p0)/2
                                                        (P:254 discretised; readings C4, C6)
Inside a step Gamma is evaluated at the stage time with S_n, C_n frozen (reading C3).
"""
from __future__ import annotations

import math

from .constants import HBAR


class CavityMemory:
    def __init__(self, omega_c, kappa, x0=0.0, p0=0.0, vcell=1.0, hbar=HBAR):
        self.omega_c = float(omega_c)
        self.kappa = float(kappa)
        self.x0 = float(x0)
        self.p0 = float(p0)
        self.vcell = float(vcell)
        self.hbar = float(hbar)
        self.reset()

    def reset(self):
        """ResetMemoryTerm(): the current state becomes t = 0 of the coupling."""
        self.S = 0.0
        self.C = 0.0
        self.t = 0.0
        self.step = 0
        self.W = 0.0

    def gamma(self, t):
        """Gamma(t) from P:343 with the S_n, C_n of the last completed step."""
        if self.kappa * t > 700:
            raise OverflowError("kappa*t > 700: literal e^{kappa t} recursion overflows (reading C5)")
        k = 2 * self.vcell / self.hbar
        e = math.exp(-self.kappa * t)
        return e * math.cos(self.omega_c * t) * (self.x0 - k * self.S) \
            - e * math.sin(self.omega_c * t) * (self.p0 - k * self.C)

    def update(self, W, dt):
        """Advance t_n -> t_{n+1} and accumulate S, C with the right-endpoint rule."""
        t = self.t + dt
        if self.kappa * t > 700:
            raise OverflowError("kappa*t > 700 (reading C5)")
        ek = math.exp(self.kappa * t)
        self.S += ek * math.sin(self.omega_c * t) * W * dt
        self.C += ek * math.cos(self.omega_c * t) * W * dt
        self.t = t
        self.step += 1
        self.W = W

    def alpha(self):
        """alpha(t_n) reconstructed a posteriori."""
        a0 = complex(self.x0, -self.p0) / 2
        c = self.vcell / self.hbar
        inner = a0 - c * self.S + 1j * c * self.C
        return complex(math.exp(-self.kappa * self.t) * complex(math.cos(self.omega_c * self.t),
                                                                  -math.sin(self.omega_c * self.t)) * inner)

    def photons(self):
        """|alpha|^2 = <a^dagger a>."""
        return abs(self.alpha()) ** 2


def gamma_resummed(ts, Ws, t, omega_c, kappa, x0, p0, vcell, hbar=HBAR):
    """Brute-force re-summation of the memory integral with the same right-endpoint
    quadrature (S:659 style): Gamma(t) = 2 e^{-kt} Re(alpha0 e^{-iwt})
    - (2Vc/hbar) sum_j dt_j e^{k(t_j - t)} sin(w(t_j - t)) W_j  (eq:gammafinal)."""
    a0 = complex(x0, -p0) / 2
    g = 2 * math.exp(-kappa * t) * (a0 * complex(math.cos(omega_c * t), -math.sin(omega_c * t))).real
    prev = 0.0
    acc = 0.0
    for tj, Wj in zip(ts, Ws):
        dtj = tj - prev
        prev = tj
        acc += dtj * math.exp(kappa * (tj - t)) * math.sin(omega_c * (tj - t)) * Wj
    return g - 2 * vcell / hbar * acc
