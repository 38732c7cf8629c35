"""Thermal (stochastic) field (oracle, fp64).  Test infrastructure only.

P:188 lists the thermal field among the Mumax3 terms the cavity field is added to; the paper
gives no formula.  Reading C-TH: Mumax3's Brown field
    B_th,i = eta_i * sqrt(2 alpha k_B T / (gamma M_s V_cell dt)),
eta_i a standard normal 3-vector per cell, drawn once per time step and held for all stages of
that step, zero in vacuum cells.  The random numbers are a counter-based stream that the CUDA
path implements independently from the same definition (SplitMix64, Steele, Lea & Flood 2014):
    h(seed, c) = mix(seed + (c + 1) * 0x9E3779B97F4A7C15)      (mod 2^64)
    mix(z):  z = (z ^ z>>30) * 0xBF58476D1CE4E5B9;  z = (z ^ z>>27) * 0x94D049BB133111EB;  z ^ z>>31
i.e. the c-th output of the SplitMix64 generator started at state `seed`.  Cell g (global
index (z ny + y) nx + x) at step n uses counters c = 2 (n N + g) + j, j = 0, 1 (N cells); each
64-bit word gives a Box-Muller pair from u1 = (h>>40 + 1) 2^-24 in (0, 1] and
u2 = (h & 0xFFFFFF) 2^-24:  r = sqrt(-2 ln u1),  (r cos 2 pi u2, r sin 2 pi u2).
eta = (pair0.cos, pair0.sin, pair1.cos).
"""
from __future__ import annotations

import math

import numpy as np

from .constants import KB

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed, counters):
    """The counters-th outputs (uint64 array) of SplitMix64 started at state `seed`."""
    c = np.asarray(counters, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (c + np.uint64(1)) * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


def box_muller(h):
    """Two standard normals per 64-bit word (see the module docstring)."""
    u1 = ((h >> np.uint64(40)).astype(np.float64) + 1.0) * 2.0 ** -24
    u2 = (h & np.uint64(0xFFFFFF)).astype(np.float64) * 2.0 ** -24
    r = np.sqrt(-2.0 * np.log(u1))
    return r * np.cos(2 * math.pi * u2), r * np.sin(2 * math.pi * u2)


def eta(shape, seed, step):
    """eta of every cell at step n: shape (nz, ny, nx, 3)."""
    n_cells = int(np.prod(shape))
    g = np.arange(n_cells, dtype=np.uint64)
    base = (np.uint64(step) * np.uint64(n_cells) + g) * np.uint64(2)
    c0, s0 = box_muller(splitmix64(seed, base))
    c1, _ = box_muller(splitmix64(seed, base + np.uint64(1)))
    return np.stack([c0, s0, c1], axis=-1).reshape(tuple(shape) + (3,))


def sigma(alpha, temperature, gamma, Ms, vcell, dt):
    """Standard deviation (T) of each component of B_th (reading C-TH)."""
    return math.sqrt(2.0 * alpha * KB * temperature / (gamma * Ms * vcell * dt))


def thermal_field(shape, mag, seed, step, sig):
    """B_th = sig * eta at step n, zero in vacuum cells."""
    return np.where(np.asarray(mag)[..., None], sig * eta(shape, seed, step), 0.0)
