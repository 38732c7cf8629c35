"""Closed forms used as pins (oracle).  Test infrastructure only.

* Aharoni's demagnetising factor of a rectangular prism (used to pin Newell's tensor).
* Kittel frequencies (BJ north_star): sphere / cube f = gamma B / 2 pi; box with bias along x
  w = gamma sqrt((B + (N_y - N_x) mu0 Ms)(B + (N_z - N_x) mu0 Ms)); thin film
  gamma sqrt(B (B + mu0 Ms)).
* Coupling law g = gamma B_rms,perp sqrt(S/2) (g ~ B_rms sqrt(V_m)), S = Ms V/(hbar gamma).
* Two-oscillator anticrossing Omega_+- (P:419 with lambda -> g, w_z -> w_Kittel).
* Zero-point current i_rms = w_0 sqrt(hbar pi / (4 Z_0)) (eq:irms; 11.3 nA).
* Spectrum peak: FFT of the mean-subtracted signal, parabolic interpolation on the
  log amplitude (reading C23).
"""
from __future__ import annotations

import math

import numpy as np

from .constants import GAMMA, HBAR, MU0  # noqa: F401 (HBAR re-exported for tests)


def aharoni_z(a, b, c):
    """D_z of a prism with half-edges a, b, c along x, y, z (Aharoni, J. Appl. Phys. 83, 3432)."""
    abc = a * b * c
    r = math.sqrt(a * a + b * b + c * c)
    rab = math.sqrt(a * a + b * b)
    rbc = math.sqrt(b * b + c * c)
    rac = math.sqrt(a * a + c * c)
    v = (b * b - c * c) / (2 * b * c) * math.log((r - a) / (r + a))
    v += (a * a - c * c) / (2 * a * c) * math.log((r - b) / (r + b))
    v += b / (2 * c) * math.log((rab + a) / (rab - a))
    v += a / (2 * c) * math.log((rab + b) / (rab - b))
    v += c / (2 * a) * math.log((rbc - b) / (rbc + b))
    v += c / (2 * b) * math.log((rac - a) / (rac + a))
    v += 2 * math.atan(a * b / (c * r))
    v += (a**3 + b**3 - 2 * c**3) / (3 * abc)
    v += (a * a + b * b - 2 * c * c) / (3 * abc) * r
    v += c / (a * b) * (rac + rbc)
    v -= (rab**3 + rbc**3 + rac**3) / (3 * abc)
    return v / math.pi


def aharoni(lx, ly, lz):
    """(D_x, D_y, D_z) of a prism with full edges lx, ly, lz."""
    a, b, c = lx / 2, ly / 2, lz / 2
    return aharoni_z(b, c, a), aharoni_z(c, a, b), aharoni_z(a, b, c)


def kittel_box(B, Ms, N):
    """Angular Kittel frequency of a uniformly magnetised box, bias along x, factors N."""
    Nx, Ny, Nz = N
    return GAMMA * math.sqrt((B + (Ny - Nx) * MU0 * Ms) * (B + (Nz - Nx) * MU0 * Ms))


def kittel_film(B, Ms):
    return GAMMA * math.sqrt(B * (B + MU0 * Ms))


def coupling_g(Bperp, Ms, volume):
    """g (rad/s) = gamma B_perp sqrt(S/2), S = M_s V / (hbar gamma)."""
    S = Ms * volume / (HBAR * GAMMA)
    return GAMMA * Bperp * math.sqrt(S / 2)


def two_oscillator(w1, w2, g):
    """Normal modes of two coupled oscillators (P:419 with lambda -> g, w_z -> w1, w_c -> w2)."""
    a = w1 * w1 + w2 * w2
    b = math.sqrt((w1 * w1 - w2 * w2) ** 2 + 16 * g * g * w1 * w2)
    return math.sqrt((a - b) / 2), math.sqrt((a + b) / 2)


def i_rms(omega0, Z0):
    return omega0 * math.sqrt(HBAR * math.pi / (4 * Z0))


def spectrum(signal, dt, window=None, pad=1):
    """|FFT| of the mean-subtracted signal; optional Hann window and zero padding."""
    x = np.asarray(signal, float)
    x = x - x.mean()
    if window == "hann":
        x = x * np.hanning(x.size)
    n = x.size * int(pad)
    amp = np.abs(np.fft.rfft(x, n))
    freqs = np.fft.rfftfreq(n, dt)
    return freqs, amp


def peaks(signal, dt, n=2, fmin=0.0, window=None, pad=1):
    """The n largest local maxima (Hz), refined by a parabola through log-amplitudes (C23)."""
    f, a = spectrum(signal, dt, window, pad)
    la = np.log(a + 1e-300)
    cand = [k for k in range(1, a.size - 1) if a[k] >= a[k - 1] and a[k] > a[k + 1] and f[k] >= fmin]
    cand.sort(key=lambda k: -a[k])
    out = []
    for k in cand[:n]:
        y0, y1, y2 = la[k - 1], la[k], la[k + 1]
        d = y0 - 2 * y1 + y2
        delta = 0.5 * (y0 - y2) / d if d != 0 else 0.0
        out.append((k + delta) * (f[1] - f[0]))
    return sorted(out)


def fit_two_oscillator(w_mag, lo, hi, wc0, g0):
    """Least-squares (omega_c, g) (rad/s) of the two_oscillator normal modes (w1 = w_mag,
    w2 = omega_c) to measured branches lo < hi (the anticrossing read-out of P:14-22, P:419 with
    lambda -> g), with SciPy's least_squares from (wc0, g0); parameters scaled by wc0."""
    from scipy.optimize import least_squares

    w_mag, lo, hi = (np.asarray(v, float) for v in (w_mag, lo, hi))

    def res(q):
        m = np.array([two_oscillator(w, q[0] * wc0, q[1] * wc0) for w in w_mag])
        return np.concatenate([m[:, 0] - lo, m[:, 1] - hi]) / wc0

    r = least_squares(res, [1.0, g0 / wc0], xtol=1e-15, ftol=1e-15, gtol=1e-15)
    return float(r.x[0] * wc0), float(abs(r.x[1]) * wc0)
