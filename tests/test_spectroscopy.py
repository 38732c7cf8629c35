"""CPU side of the spectroscopy driver (NEXT-3): the normal-mode model the device fit uses equals
the oracle's pinned two-oscillator result, and the oracle's own anticrossing fit (the reference
for tests/test_gpu_spectroscopy.py) recovers known (omega_c, g) from noisy synthetic branches."""
import importlib.util
import math
import os

import numpy as np
import pytest

from oracle import analytic as A

_P = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2410_00966_b200",
                  "spectroscopy.py")
_spec = importlib.util.spec_from_file_location("mcq_spectroscopy", _P)   # no libmcq needed
SP = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(SP)


def test_oracle_peaks_of_two_tones():
    dt = 1e-12
    t = np.arange(20000) * dt
    x = np.sin(2 * math.pi * 11.3e9 * t) + 0.4 * np.sin(2 * math.pi * 12.9e9 * t + 0.3) + 0.2
    lo, hi = A.peaks(x, dt, 2, window="hann", pad=8)
    assert lo == pytest.approx(11.3e9, rel=2e-4) and hi == pytest.approx(12.9e9, rel=2e-4)


def test_normal_modes_equal_oracle_two_oscillator():
    for w1, w2, g in ((7e10, 7e10, 2e9), (7e10, 8e10, 1e9), (5e10, 3e10, 4e9)):
        m, p = SP.normal_modes(w1, w2, g)
        om, op = A.two_oscillator(w1, w2, g)
        assert float(m) == pytest.approx(om, rel=1e-13) and float(p) == pytest.approx(op, rel=1e-13)


def test_oracle_fit_recovers_parameters():
    wc, g = 7.0e10, 2.2e9
    w = np.linspace(0.92, 1.08, 9) * wc
    lo = np.array([A.two_oscillator(x, wc * 1.004, g)[0] for x in w])
    hi = np.array([A.two_oscillator(x, wc * 1.004, g)[1] for x in w])
    lo = lo * (1 + 1e-5 * np.sin(np.arange(9)))               # small measurement noise
    wc_fit, g_fit = A.fit_two_oscillator(w, lo, hi, wc, 0.5 * g)
    assert wc_fit == pytest.approx(wc * 1.004, rel=1e-4) and g_fit == pytest.approx(g, rel=1e-3)
