"""Pins of the oracle's interfacial DMI field (reading C-DMI): the discrete closed form on a
Neel spiral, the variational identity B = -(1/(M_s V)) dE/dm of the discrete energy in the
interior, the vanishing field of uniform states, and the sign convention (chirality)."""
import math

import numpy as np
import pytest

from oracle import fields as F

CELL = (2e-9, 3e-9, 1e-9)
MS, D = 8.6e5, 3e-3


def test_neel_spiral_discrete_closed_form():
    nx, ny, nz = 24, 5, 2
    k = 2 * math.pi / (10 * CELL[0])
    x = np.arange(nx)
    m = np.zeros((nz, ny, nx, 3))
    m[..., 0] = np.sin(k * x * CELL[0])
    m[..., 2] = np.cos(k * x * CELL[0])
    mag = np.ones((nz, ny, nx), bool)
    B = F.dmi_interfacial(m, mag, CELL, D, MS)
    # interior: d_x sin = sin(k dx)/dx cos, d_x cos = -sin(k dx)/dx sin  =>  B = -(2D/Ms) s m, s = sin(k dx)/dx
    s = math.sin(k * CELL[0]) / CELL[0]
    inner = (slice(None), slice(None), slice(1, nx - 1))
    assert np.allclose(B[inner], -(2 * D / MS) * s * m[inner], rtol=0, atol=1e-12 * 2 * D / MS * s)
    # the opposite chirality costs energy: field parallel to m for the reversed spiral
    m2 = m.copy()
    m2[..., 0] *= -1
    B2 = F.dmi_interfacial(m2, mag, CELL, D, MS)
    assert np.allclose(B2[inner], (2 * D / MS) * s * m2[inner], atol=1e-12 * 2 * D / MS * s)


def _energy(m, mag):
    """Discrete energy V sum_i D [m_z (d_x m_x + d_y m_y) - (m_x d_x m_z + m_y d_y m_z)] with the
    same central differences (boundary handling irrelevant for interior perturbations)."""
    def d(f, axis, h):
        return (np.roll(f, -1, axis) - np.roll(f, 1, axis)) / (2 * h)
    mx, my, mz = m[..., 0], m[..., 1], m[..., 2]
    e = mz * (d(mx, 2, CELL[0]) + d(my, 1, CELL[1])) - (mx * d(mz, 2, CELL[0]) + my * d(mz, 1, CELL[1]))
    return D * np.prod(CELL) * float(np.sum(e * mag))


def test_field_is_minus_energy_gradient_in_the_interior():
    rng = np.random.default_rng(4)
    nz, ny, nx = 1, 9, 10
    m = rng.normal(size=(nz, ny, nx, 3))
    m /= np.linalg.norm(m, axis=-1, keepdims=True)
    mag = np.ones((nz, ny, nx), bool)
    B = F.dmi_interfacial(m, mag, CELL, D, MS)
    V = np.prod(CELL)
    for (y, x) in ((4, 5), (3, 3), (6, 7)):
        for c in range(3):
            h = 1e-6
            mp, mm = m.copy(), m.copy()
            mp[0, y, x, c] += h
            mm[0, y, x, c] -= h
            g = (_energy(mp, mag) - _energy(mm, mag)) / (2 * h)
            assert B[0, y, x, c] == pytest.approx(-g / (MS * V), rel=1e-6, abs=1e-9 * 2 * D / MS / CELL[0])


def test_uniform_state_and_vacuum():
    m = np.zeros((2, 4, 5, 3))
    m[..., 1] = 1.0
    mag = np.ones((2, 4, 5), bool)
    assert np.abs(F.dmi_interfacial(m, mag, CELL, D, MS)).max() == 0.0
    mag[0, 1, 1] = False
    m[0, 1, 1] = 0.0
    B = F.dmi_interfacial(m, mag, CELL, D, MS)
    assert np.abs(B).max() == 0.0          # vacuum neighbours act as Neumann ghosts (C-DMI)
