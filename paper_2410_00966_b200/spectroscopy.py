"""Spectroscopy driver: the paper's spectra are the numerical Fourier
transform of the spatially averaged magnetisation, and its couplings are read off
anticrossings of such spectra over a bias sweep.  This module runs a sweep as
independent replicas on their own CUDA streams (every replica records its per-step <m> with the
on-device trace, no host round trip per step), then does the small host-side analysis: windowed
FFT, parabolic peak interpolation, and a least-squares fit of the two-oscillator normal modes
(position-coupled oscillators, P:419 with lambda -> g) for g and omega_c.

The simulation itself runs entirely in libmcq's kernels; this is analysis of the recorded
traces (numpy), not part of the per-step hot path."""
from __future__ import annotations

import math

import numpy as np


def spectrum(signal, dt, window="hann", pad=8):
    """|FFT| of the mean-subtracted signal with a Hann window and zero padding: (freqs Hz, amp)."""
    x = np.asarray(signal, np.float64)
    x = x - x.mean()
    if window == "hann":
        x = x * np.hanning(x.size)
    n = x.size * int(pad)
    return np.fft.rfftfreq(n, dt), np.abs(np.fft.rfft(x, n))


def peaks(signal, dt, n=2, fmin=0.0, window="hann", pad=8):
    """The n strongest local maxima (Hz, ascending), refined by a parabola through log |FFT|."""
    f, a = spectrum(signal, dt, window, pad)
    la = np.log(a + 1e-300)
    k = np.nonzero((a[1:-1] >= a[:-2]) & (a[1:-1] > a[2:]) & (f[1:-1] >= fmin))[0] + 1
    k = k[np.argsort(-a[k])][:n]
    out = []
    for i in k:
        y0, y1, y2 = la[i - 1], la[i], la[i + 1]
        d = y0 - 2 * y1 + y2
        out.append((i + (0.5 * (y0 - y2) / d if d != 0 else 0.0)) * (f[1] - f[0]))
    return sorted(out)


def normal_modes(w1, w2, g):
    """Normal-mode angular frequencies of two position-coupled oscillators with coupling g
    (eigenvalues of [[w1^2, 2g sqrt(w1 w2)], [2g sqrt(w1 w2), w2^2]])."""
    w1, w2 = np.asarray(w1, float), np.asarray(w2, float)
    a = w1 * w1 + w2 * w2
    b = np.sqrt((w1 * w1 - w2 * w2) ** 2 + 16 * g * g * w1 * w2)
    return np.sqrt((a - b) / 2), np.sqrt((a + b) / 2)


def fit_anticrossing(w_mag, lo, hi, wc0, g0):
    """Least-squares (omega_c, g) of the two branches lo(w_mag), hi(w_mag) (angular)."""
    from scipy.optimize import least_squares

    w_mag, lo, hi = (np.asarray(v, float) for v in (w_mag, lo, hi))
    ok = np.isfinite(lo) & np.isfinite(hi)
    w_mag, lo, hi = w_mag[ok], lo[ok], hi[ok]

    def res(q):  # parameters in units of wc0 (well-conditioned for the solver)
        m, pl = normal_modes(w_mag, q[0] * wc0, q[1] * wc0)
        return np.concatenate([m - lo, pl - hi]) / wc0

    r = least_squares(res, [1.0, g0 / wc0], xtol=1e-14, ftol=1e-14, gtol=1e-14)
    return float(r.x[0] * wc0), float(abs(r.x[1]) * wc0)


def sweep(make_solver, points, dt, steps, component=1, every=1):
    """Run one replica per sweep point concurrently (one CUDA stream each) and return the two
    dominant spectral peaks (Hz) of <m_component> per point, shape (len(points), 2).

    make_solver(point, stream) -> a Solver whose state is set (bias, B_rms, cavity, m)."""
    import torch

    from . import mcq_get_trace, mcq_set_trace

    streams = [torch.cuda.Stream() for _ in points]
    solvers = [make_solver(p, s.cuda_stream) for p, s in zip(points, streams)]
    for sv in solvers:
        mcq_set_trace(sv.ctx, steps // every + 1, every)
    for sv in solvers:                       # enqueue all: the replicas overlap on the GPU
        sv.run(dt, steps)
    torch.cuda.synchronize()
    out = []
    for sv in solvers:
        tr = mcq_get_trace(sv.ctx)
        pk = peaks(tr[:, 1 + component], dt * every, 2)
        out.append(pk + [math.nan] * (2 - len(pk)))
        sv.close()
    return np.array(out)
