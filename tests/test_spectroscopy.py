"""Host analysis of the spectroscopy driver (paper_2410_00966_b200.spectroscopy, NEXT-3): peak
finding on synthetic signals with known frequencies, the normal-mode formula against the
oracle's pinned two-oscillator result, and the anticrossing fit recovering known (w_c, g)."""
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


def test_peaks_of_two_tones():
    dt = 1e-12
    t = np.arange(20000) * dt
    x = np.sin(2 * math.pi * 11.3e9 * t) + 0.4 * np.sin(2 * math.pi * 12.9e9 * t + 0.3) + 0.2
    lo, hi = SP.peaks(x, dt, 2)
    assert lo == pytest.approx(11.3e9, rel=2e-4) and hi == pytest.approx(12.9e9, rel=2e-4)


def test_normal_modes_equal_oracle_two_oscillator():
    for w1, w2, g in ((7e10, 7e10, 2e9), (7e10, 8e10, 1e9), (5e10, 3e10, 4e9)):
        m, p = SP.normal_modes(w1, w2, g)
        om, op = A.two_oscillator(w1, w2, g)
        assert float(m) == pytest.approx(om, rel=1e-13) and float(p) == pytest.approx(op, rel=1e-13)


def test_fit_recovers_parameters():
    wc, g = 7.0e10, 2.2e9
    w = np.linspace(0.92, 1.08, 9) * wc
    lo, hi = SP.normal_modes(w, wc * 1.004, g)
    lo = lo * (1 + 1e-5 * np.sin(np.arange(9)))               # small measurement noise
    wc_fit, g_fit = SP.fit_anticrossing(w, lo, hi, wc, 0.5 * g)
    assert wc_fit == pytest.approx(wc * 1.004, rel=1e-4) and g_fit == pytest.approx(g, rel=1e-3)
    lo[3] = np.nan                                              # a missing peak is dropped
    assert SP.fit_anticrossing(w, lo, hi, wc, 0.5 * g)[1] == pytest.approx(g, rel=1e-3)
