"""Pins for oracle.fields: closed forms, hand values, invariants, and two independent demag routes."""
import math

import numpy as np
import pytest

from oracle import fields as F
from oracle import tensor as T
from oracle import analytic as A
from oracle.constants import MU0

rng = np.random.default_rng(42)


def _rand_m(shape, mag=None):
    v = rng.normal(size=shape + (3,))
    v /= np.linalg.norm(v, axis=-1, keepdims=True)
    if mag is not None:
        v *= mag[..., None]
    return v


def test_exchange_uniform_and_single_cell_zero():
    m = np.zeros((3, 4, 5, 3)); m[..., 2] = 1
    mag = np.ones((3, 4, 5), bool)
    assert np.abs(F.exchange(m, mag, (1e-9, 2e-9, 3e-9), 1e-11, 8e5)).max() == 0
    m1 = _rand_m((1, 1, 1))
    assert np.abs(F.exchange(m1, np.ones((1, 1, 1), bool), (1e-9,) * 3, 1e-11, 8e5)).max() == 0


def test_exchange_two_cell_hand_value():
    # two cells along x: B_0 = (2A/Ms)(m_1 - m_0)/dx^2 (S:143 style hand value)
    A_, Ms, dx = 1.3e-11, 8.6e5, 2e-9
    m = np.array([[[[1.0, 0, 0], [0, 1.0, 0]]]])
    B = F.exchange(m, np.ones((1, 1, 2), bool), (dx, 1e-9, 1e-9), A_, Ms)
    expect0 = 2 * A_ / Ms * (np.array([0, 1.0, 0]) - np.array([1.0, 0, 0])) / dx**2
    assert np.allclose(B[0, 0, 0], expect0, rtol=1e-14)
    assert np.allclose(B[0, 0, 1], -expect0, rtol=1e-14)


def test_exchange_vacuum_neighbour_contributes_nothing():
    A_, Ms, dx = 1e-11, 1e6, 1e-9
    m = np.array([[[[1.0, 0, 0], [0, 1.0, 0], [0, 0, 0]]]])
    mag = np.array([[[True, True, False]]])
    B = F.exchange(m, mag, (dx,) * 3, A_, Ms)
    assert np.allclose(B[0, 0, 1], 2 * A_ / Ms * (np.array([1.0, 0, 0]) - np.array([0, 1.0, 0])) / dx**2)
    assert np.all(B[0, 0, 2] == 0)


def test_exchange_discrete_spin_wave_closed_form():
    # interior cells of m = (cos kx, sin kx, 0): B = -(2A/Ms)(2 - 2cos(k dx))/dx^2 m (derived)
    nx, k, dx, A_, Ms = 40, 0.3, 1e-9, 1e-11, 1e6
    x = np.arange(nx) * dx
    m = np.zeros((1, 1, nx, 3))
    m[0, 0, :, 0] = np.cos(k * x / dx)
    m[0, 0, :, 1] = np.sin(k * x / dx)
    B = F.exchange(m, np.ones((1, 1, nx), bool), (dx, 5e-9, 5e-9), A_, Ms)
    expect = -(2 * A_ / Ms) * (2 - 2 * math.cos(k)) / dx**2 * m
    assert np.allclose(B[0, 0, 1:-1], expect[0, 0, 1:-1], rtol=1e-12, atol=1e-9)


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_exchange_spin_wave_along_each_axis_anisotropic_cell(axis):
    """the spin-wave pin along x alone left the y / z scaling unpinned (a swap
    of dy and dz passed every test).  With three distinct cell sizes, a discrete spin wave along
    axis a gives B = -(2A/Ms)(2 - 2cos(k))/d_a^2 m in the interior — only the right d_a passes."""
    cell = (1.0e-9, 1.7e-9, 2.9e-9)
    n, k, A_, Ms = 24, 0.4, 1.2e-11, 9e5
    shape = [3, 3, 3]
    shape[2 - axis] = n                          # array axes are (z, y, x)
    j = np.arange(n).reshape([n if a == 2 - axis else 1 for a in range(3)])
    m = np.zeros(tuple(shape) + (3,))
    m[..., 0] = np.cos(k * j)
    m[..., 1] = np.sin(k * j)
    B = F.exchange(m, np.ones(tuple(shape), bool), cell, A_, Ms)
    expect = -(2 * A_ / Ms) * (2 - 2 * math.cos(k)) / cell[axis] ** 2 * m
    inner = [slice(1, -1) if a == 2 - axis else slice(1, 2) for a in range(3)]   # interior, centre row
    assert np.allclose(B[tuple(inner)], expect[tuple(inner)], rtol=1e-12, atol=1e-12 * np.abs(expect).max())


def test_exchange_total_torque_vanishes():
    mag = rng.random((4, 5, 6)) > 0.2
    m = _rand_m((4, 5, 6), mag)
    B = F.exchange(m, mag, (1e-9, 1.5e-9, 2e-9), 1e-11, 1e6)
    assert np.abs(np.cross(m, B).sum(axis=(0, 1, 2))).max() < 1e-6 * np.abs(B).max()


def test_uniaxial_cases():
    Ku, Ms = 5e4, 8e5
    u = np.array([0.0, 0.6, 0.8])
    mag = np.ones((1, 1, 1), bool)
    assert np.allclose(F.uniaxial(u[None, None, None], mag, Ku, u, Ms)[0, 0, 0], 2 * Ku / Ms * u)
    perp = np.array([[[[1.0, 0, 0]]]])
    assert np.allclose(F.uniaxial(perp, mag, Ku, u, Ms), 0)


def _cubic_energy(m, Kc1, c1, c2):
    c1 = np.asarray(c1, float) / np.linalg.norm(c1)
    c2 = np.asarray(c2, float) / np.linalg.norm(c2)
    c3 = np.cross(c1, c2)
    a, b, c = m @ c1, m @ c2, m @ c3
    return Kc1 * (a * a * b * b + b * b * c * c + c * c * a * a)


def test_cubic_field_is_minus_energy_gradient():
    Kc1, Ms = -610.0, 1.4e5
    c1, c2 = (1, 1, 0), (-1, 1, 0)
    m = np.array([0.3, -0.5, 0.81])
    m /= np.linalg.norm(m)
    B = F.cubic(m[None, None, None], np.ones((1, 1, 1), bool), Kc1, c1, c2, Ms)[0, 0, 0]
    h = 1e-6
    grad = np.array([(_cubic_energy(m + h * e, Kc1, c1, c2) - _cubic_energy(m - h * e, Kc1, c1, c2)) / (2 * h)
                     for e in np.eye(3)])
    assert np.allclose(B, -grad / Ms, rtol=1e-7, atol=1e-12)


def test_cubic_axes():
    Kc1, Ms = 1e4, 1e6
    mag = np.ones((1, 1, 1), bool)
    for m in ([1, 0, 0], [0, 0, -1]):
        assert np.allclose(F.cubic(np.array(m, float)[None, None, None], mag, Kc1, (1, 0, 0), (0, 1, 0), Ms), 0)
    m111 = np.ones(3) / math.sqrt(3)
    B = F.cubic(m111[None, None, None], mag, Kc1, (1, 0, 0), (0, 1, 0), Ms)[0, 0, 0]
    assert np.allclose(np.cross(m111, B), 0, atol=1e-12)


def test_single_cell_demag_is_self_factor():
    cell = (2e-9, 3e-9, 1e-9)
    Ms = 8e5
    m = _rand_m((1, 1, 1))
    B = F.demag_bruteforce(m, np.ones((1, 1, 1), bool), cell, Ms)
    D = np.array(A.aharoni(*cell))
    assert np.allclose(B[0, 0, 0], -MU0 * Ms * D * m[0, 0, 0], rtol=1e-12)


def test_demag_bruteforce_equals_direct_dft_masked():
    grid = (7, 6, 3)
    cell = (2e-9, 2.5e-9, 3e-9)
    mag = rng.random((3, 6, 7)) > 0.3
    m = _rand_m((3, 6, 7), mag)
    Ms = 1.4e5
    a = F.demag_bruteforce(m, mag, cell, Ms)
    b = F.demag_dft(m, mag, cell, Ms)
    assert np.max(np.abs(a - b)) < 1e-12 * np.max(np.abs(a)) * 1e3
    pts = [(0, 0, 0), (6, 5, 2), (3, 2, 1)]
    c = F.demag_at(m, mag, cell, Ms, pts, T.tensor_octant(grid, cell))
    for p, v in zip(pts, c):
        assert np.allclose(v, a[p[2], p[1], p[0]], rtol=1e-12, atol=1e-18)


def test_demag_linear_and_odd():
    grid, cell, Ms = (5, 4, 2), (1e-9,) * 3, 1e6
    mag = np.ones((2, 4, 5), bool)
    m1, m2 = _rand_m((2, 4, 5)), _rand_m((2, 4, 5))
    oc = T.tensor_octant(grid, cell)
    f = lambda m: F.demag_bruteforce(m, mag, cell, Ms, oc)
    assert np.allclose(f(-m1), -f(m1))
    assert np.allclose(f(0.3 * m1 + 0.7 * m2), 0.3 * f(m1) + 0.7 * f(m2), atol=1e-12)


def test_uniform_box_mean_field_is_aharoni():
    grid, cell, Ms = (10, 8, 3), (2e-9, 2e-9, 1e-9), 1e6
    m = np.zeros((3, 8, 10, 3)); m[..., 0] = 1
    B = F.demag_bruteforce(m, np.ones((3, 8, 10), bool), cell, Ms)
    D = A.aharoni(20e-9, 16e-9, 3e-9)
    assert abs(B[..., 0].mean() / (-MU0 * Ms) - D[0]) < 1e-9


def test_sinc():
    assert F.sinc(0.0) == 1.0
    assert abs(F.sinc(math.pi)) < 1e-16
    assert abs(F.sinc(0.5) - math.sin(0.5) / 0.5) < 1e-16
