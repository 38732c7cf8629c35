"""Spectroscopy driver: the paper's spectra are the numerical Fourier
transform of the spatially averaged magnetisation, and its couplings are read off
anticrossings of such spectra over a bias sweep.  A sweep runs as independent
replicas on their own CUDA streams (every replica records its per-step <m> with the on-device
trace, no host round trip per step); the analysis then also runs on the device
(csrc/spectro.cu through include/mcq.h): the FFT of every replica's trace in one batched pass,
the parabolic peak interpolation (reading C23), and the least-squares fit of the two-oscillator
normal modes (position-coupled oscillators, P:419 with lambda -> g) for omega_c and g.
Argument marshalling only; the one formula kept here (normal_modes) documents the model."""
from __future__ import annotations

import math

import numpy as np


def normal_modes(w1, w2, g):
    """Normal-mode angular frequencies of two position-coupled oscillators with coupling g
    (eigenvalues of [[w1^2, 2g sqrt(w1 w2)], [2g sqrt(w1 w2), w2^2]]): the model the device fit
    (mcq_fit_anticrossing) uses."""
    w1, w2 = np.asarray(w1, float), np.asarray(w2, float)
    a = w1 * w1 + w2 * w2
    b = np.sqrt((w1 * w1 - w2 * w2) ** 2 + 16 * g * g * w1 * w2)
    return np.sqrt((a - b) / 2), np.sqrt((a + b) / 2)


def peaks(solver, component=1, npeaks=2, pad=8, window=1, fmin=0.0):
    """The npeaks strongest spectral peaks (Hz, ascending) of <m_component> from the solver's
    recorded trace, computed on the device."""
    from . import mcq_trace_peaks
    f, _ = mcq_trace_peaks(solver.ctx, 1 + component, pad, window, fmin, npeaks)
    return list(f)


def fit_anticrossing(w_mag, lo, hi, wc0, g0):
    """Device least-squares (omega_c, g) (rad/s) of the two branches lo(w_mag), hi(w_mag);
    points with a missing peak (NaN) are dropped."""
    from . import mcq_fit_anticrossing
    w_mag, lo, hi = (np.asarray(v, float) for v in (w_mag, lo, hi))
    ok = np.isfinite(lo) & np.isfinite(hi)
    return mcq_fit_anticrossing(w_mag[ok], lo[ok], hi[ok], wc0, g0)


def sweep(make_solver, points, dt, steps, component=1, every=1, pad=8, window=1):
    """Run one replica per sweep point concurrently (one CUDA stream each) and return the two
    dominant spectral peaks (Hz) of <m_component> per point, shape (len(points), 2), from one
    batched device pass over all replicas' traces.

    make_solver(point, stream) -> a Solver whose state is set (bias, B_rms, cavity, m)."""
    import torch

    from . import mcq_set_trace, mcq_trace_peaks_batch

    from . import mcq_set_persistent_2d

    streams = [torch.cuda.Stream() for _ in points]
    solvers = [make_solver(p, s.cuda_stream) for p, s in zip(points, streams)]
    for sv in solvers:
        mcq_set_trace(sv.ctx, steps // every + 1, every)
        mcq_set_persistent_2d(sv.ctx, 1)  # 2D replicas: one persistent kernel each (no-op in 3D)
    for sv in solvers:                       # enqueue all: the replicas overlap on the GPU
        sv.run(dt, steps)
    torch.cuda.synchronize()
    res = mcq_trace_peaks_batch([sv.ctx for sv in solvers], 1 + component, pad, window, 0.0, 2)
    out = [list(f) + [math.nan] * (2 - len(f)) for f, _ in res]
    for sv in solvers:
        sv.close()
    return np.array(out)
