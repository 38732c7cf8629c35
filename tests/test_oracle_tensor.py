"""Pins for oracle.tensor (reading C11) against closed forms that do not use the oracle's code."""
import json
import math
import os

import numpy as np
import pytest

from oracle import tensor as T
from oracle import analytic as A

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_cube_self_term_is_one_third():
    n = T.newell(0.0, 0.0, 0.0, 2e-9, 2e-9, 2e-9)
    g = GOLD["cube_self_demag"]
    assert np.allclose(n[:3], g["value"], atol=g["tol"], rtol=0)
    assert np.allclose(n[3:], 0.0, atol=1e-15)


@pytest.mark.parametrize("box", [(1.0, 1.3, 0.2), (5.0, 5.0, 2.5), (1.953125, 1.953125, 2.5), (3.0, 1.0, 7.0)])
def test_self_term_equals_aharoni_prism(box):
    n = T.newell(0.0, 0.0, 0.0, *box)
    ah = A.aharoni(*box)
    assert np.allclose(n[:3], ah, rtol=0, atol=1e-12)
    assert abs(n[:3].sum() - 1.0) < 1e-12          # trace of the self term is 1


def test_aharoni_closed_form_sanity():
    # independent checks of the Aharoni routine itself: cube, trace, thin-film and needle limits
    assert abs(A.aharoni(1, 1, 1)[2] - 1 / 3) < 1e-14
    assert abs(sum(A.aharoni(2.0, 0.7, 0.3)) - 1.0) < 1e-12
    assert 0.99 < A.aharoni(1000, 1000, 1)[2] < A.aharoni(1e5, 1e5, 1)[2] < 1.0
    assert A.aharoni(1, 1, 1000)[2] < 0.01


def test_component_parity_by_direct_evaluation():
    d = (1.0, 1.2, 0.8)
    X, Y, Z = 2.0, 3.6, 1.6
    base = T.newell(X, Y, Z, *d)
    for sx, sy, sz in [(-1, 1, 1), (1, -1, 1), (1, 1, -1), (-1, -1, -1)]:
        v = T.newell(sx * X, sy * Y, sz * Z, *d)
        expect = base * np.array([1, 1, 1, sx * sy, sx * sz, sy * sz])
        assert np.allclose(v, expect, rtol=1e-10, atol=1e-14)


def test_far_field_tends_to_point_dipole():
    for n, tol in [(10, 1e-3), (30, 1e-5)]:
        X, Y, Z = n * 1.0, 0.7 * n, 0.3 * n
        a = T.newell(X, Y, Z, 1.0, 1.0, 1.0)
        b = T.point_dipole(X, Y, Z, 1.0)
        assert np.max(np.abs(a - b)) / np.max(np.abs(b)) < tol


def test_dipole_sign_and_trace():
    # on-axis dipole: N_xx = -2V/(4 pi r^3), N_yy = N_zz = V/(4 pi r^3); trace 0 off the source
    r = 7.0
    d = T.point_dipole(r, 0.0, 0.0, 1.0)
    assert np.allclose(d[:3], np.array([-2, 1, 1]) / (4 * math.pi * r**3))
    a = T.newell(20.0, 13.0, 5.0, 1.0, 1.0, 1.0)
    assert abs(a[:3].sum()) < 1e-9


def test_newell_and_gauss_legendre_agree_in_overlap_band():
    rng = np.random.default_rng(0)
    for cell in [(1.0, 1.0, 1.0), (1.953125, 1.953125, 2.5), (5.0, 5.0, 5.0)]:
        for _ in range(6):
            i, j, k = rng.integers(8, 17, size=3)
            X, Y, Z = i * cell[0], j * cell[1], k * cell[2]
            a = T.newell(X, Y, Z, *cell)
            b = T.far_field(X, Y, Z, *cell)
            assert np.max(np.abs(a - b)) / np.max(np.abs(a)) < 2e-7


@pytest.mark.parametrize("grid,cell", [((6, 5, 4), (1.0, 1.0, 1.0)), ((40, 24, 2), (5.0, 5.0, 3.0)),
                                       ((20, 20, 20), (1.0, 1.0, 1.0))])
def test_sum_rule_box_equals_aharoni(grid, cell):
    """Uniform magnetisation of a box of cells: the cell-averaged tensor summed over sources and
    averaged over targets is the prism's demagnetising factor (exact for Newell; the Gauss-Legendre
    far field must keep it to ~1e-6)."""
    nx, ny, nz = grid
    oc = T.tensor_octant(grid, cell)
    # sum over targets of sum over sources = sum over offsets of multiplicity * N(offset)
    tot = np.zeros(6)
    for k in range(-(nz - 1), nz):
        for j in range(-(ny - 1), ny):
            mult_jk = (ny - abs(j)) * (nz - abs(k))
            i = np.arange(-(nx - 1), nx)
            vals = T.signed_lookup(oc, i, np.full_like(i, j), np.full_like(i, k))
            tot += (vals * ((nx - np.abs(i)) * mult_jk)).sum(axis=1)
    mean = tot / (nx * ny * nz)
    ah = A.aharoni(nx * cell[0], ny * cell[1], nz * cell[2])
    assert np.allclose(mean[:3], ah, atol=2e-6, rtol=0)
    assert np.allclose(mean[3:], 0.0, atol=1e-12)


def test_padded_layout_plain_definition():
    grid, cell = (3, 4, 1), (1.0, 1.0, 1.0)
    P = T.padded_tensor(grid, cell)
    assert P.shape == (6, 1, 8, 6)
    oc = T.tensor_octant(grid, cell)
    # offset -1 in x at index L-1, offset +-n slot zero
    assert np.allclose(P[:, 0, 0, 5], oc[:, 0, 0, 1] * np.array([1, 1, 1, -1, -1, 1]))
    assert np.allclose(P[:, 0, :, 3], 0.0) and np.allclose(P[:, 0, 4, :], 0.0)
