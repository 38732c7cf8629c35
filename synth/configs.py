"""Synthetic workloads shaped like the paper's (BASELINE.json configs).

Everything here is an *input recipe*: geometry, initial state, B_rms map and the
scalar parameters handed to both the oracle and the CUDA path.  The physical
constants below are only used to scale inputs (e.g. to normalise a B_rms map to
a target coupling g via the coupling law g ~ gamma*B_rms*sqrt(S/2)); the
oracle and the CUDA library each define their own copies for the method.

Materials: YIG Ms=1.4e5 A/m, A=3.7e-12 J/m, alpha=1e-4;
                   Py  Ms=8.6e5 A/m, A=1.3e-11 J/m, alpha=1e-2.
RNG: numpy.random.default_rng(seed).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

GAMMA = 1.7595e11          # rad s^-1 T^-1
MU0 = 4e-7 * math.pi       # T m / A
HBAR = 1.05457182e-34      # J s

YIG = dict(Ms=1.4e5, Aex=3.7e-12, alpha=1e-4)
PY = dict(Ms=8.6e5, Aex=1.3e-11, alpha=1e-2)


@dataclasses.dataclass
class Config:
    name: str
    grid: tuple                      # (nx, ny, nz)
    cell: tuple                      # (dx, dy, dz) metres
    Ms: float
    Aex: float
    alpha: float
    m0: np.ndarray                   # float32 (N, 3), x fastest; 0 in vacuum
    mask: Optional[np.ndarray] = None  # uint8 (N,), 1 = magnetic; None = full box
    bext: tuple = (0.0, 0.0, 0.0)
    brms_map: Optional[np.ndarray] = None   # float32 (N, 3) tesla, or None
    brms_uniform: tuple = (0.0, 0.0, 0.0)   # used when brms_map is None
    f_c: float = 10e9                # Hz
    kappa: float = 2 * math.pi * 1e6  # rad/s
    x0: float = 0.0
    p0: float = 0.0
    exc_amp: float = 0.0             # dimensionless factor on B_rms
    exc_omega: float = 0.0           # rad/s, sinc cut-off
    aniso: Optional[dict] = None     # {ku1,u,kc1,c1,c2}
    dt: float = 0.5e-12
    seed: int = 0
    relax_first: bool = False

    @property
    def n(self) -> int:
        nx, ny, nz = self.grid
        return nx * ny * nz

    def n_magnetic(self) -> int:
        return self.n if self.mask is None else int(self.mask.sum())


# ---------------------------------------------------------------- geometry

def cell_centres(grid, cell):
    """Cell-centre coordinates relative to the box centre, arrays shaped (nz, ny, nx)."""
    nx, ny, nz = grid
    dx, dy, dz = cell
    x = (np.arange(nx) + 0.5) * dx - nx * dx / 2
    y = (np.arange(ny) + 0.5) * dy - ny * dy / 2
    z = (np.arange(nz) + 0.5) * dz - nz * dz / 2
    Z, Y, X = np.meshgrid(z, y, x, indexing="ij")
    return X, Y, Z


def sphere_mask(grid, cell, radius):
    X, Y, Z = cell_centres(grid, cell)
    return ((X**2 + Y**2 + Z**2) <= radius**2).astype(np.uint8).ravel()


def disc_mask(grid, cell, radius):
    X, Y, _ = cell_centres(grid, cell)
    return ((X**2 + Y**2) <= radius**2).astype(np.uint8).ravel()


# ---------------------------------------------------------------- states

def _apply_mask(m, mask):
    if mask is not None:
        m = m * mask[:, None]
    return m.astype(np.float32)


def random_unit(n, rng, mask=None):
    """Isotropic random unit vectors ("rand" parity state)."""
    v = rng.normal(size=(n, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return _apply_mask(v, mask)


def tilted_uniform(n, rng, axis=(0, 0, 1), noise=0.05, mask=None):
    """m = norm(axis + noise * N(0,1)^3) ("phys" state of SURVEY §8(d))."""
    v = np.asarray(axis, float)[None, :] + noise * rng.normal(size=(n, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return _apply_mask(v, mask)


def vortex_state(grid, cell, circulation=1, polarity=1, core=10e-9, mask=None):
    """Vortex ansatz: in-plane curl c*(-sin phi, cos phi), m_z = p exp(-rho^2/(2 core^2))."""
    X, Y, _ = cell_centres(grid, cell)
    rho2 = X**2 + Y**2
    phi = np.arctan2(Y, X)
    mz = polarity * np.exp(-rho2 / (2 * core**2))
    s = np.sqrt(np.clip(1 - mz**2, 0, 1))
    m = np.stack([-circulation * np.sin(phi) * s, circulation * np.cos(phi) * s, mz], axis=-1)
    return _apply_mask(m.reshape(-1, 3), mask)


# ---------------------------------------------------------------- B_rms maps

def _coupling_scale(Bperp_mean, Ms, n_mag, vcell, g_target):
    """Amplitude factor so that gamma*sqrt(S/2)*|<B_perp>| = 2*pi*g."""
    S = Ms * n_mag * vcell / (HBAR * GAMMA)
    return 2 * math.pi * g_target / (GAMMA * math.sqrt(S / 2) * Bperp_mean)


def two_wire_field(grid, cell, current, signs, offset=0.0, sep_factor=1.875):
    """In-plane field of two infinite line currents || z at x = +-sep*Lx/2 + offset, y = 0
    (two-post re-entrant cavity stand-in, P:8).  Returns float64 (N,3)."""
    nx, ny, nz = grid
    X, Y, _ = cell_centres((nx, ny, 1), cell)
    X, Y = X[0], Y[0]
    lx = nx * cell[0]
    bx = np.zeros_like(X)
    by = np.zeros_like(X)
    for s, xw in zip(signs, (+sep_factor * lx / 2 + offset, -sep_factor * lx / 2 + offset)):
        dx_, dy_ = X - xw, Y
        r2 = dx_**2 + dy_**2
        pref = s * MU0 * current / (2 * math.pi)
        bx += pref * (-dy_) / r2
        by += pref * dx_ / r2
    b = np.stack([bx, by, np.zeros_like(bx)], axis=-1)      # (ny, nx, 3)
    b = np.broadcast_to(b[None], (nz, ny, nx, 3)).reshape(-1, 3)
    return np.ascontiguousarray(b)


def _mean_perp(b, mask):
    sel = b if mask is None else b[mask.astype(bool)]
    return float(np.linalg.norm(sel[:, :2].mean(axis=0)))


def two_wire_map(grid, cell, Ms, mask, g_target, mode="bright", dark_current_ratio=498 / 785):
    """Bright (antiparallel) or dark (parallel, offset) two-wire B_rms map normalised to g."""
    n_mag = int(mask.sum()) if mask is not None else int(np.prod(grid))
    vcell = float(np.prod(cell))
    unit = two_wire_field(grid, cell, 1.0, (+1, -1))
    i_bright = _coupling_scale(_mean_perp(unit, mask), Ms, n_mag, vcell, 1e9)
    if mode == "bright":
        cur = i_bright * g_target / 1e9
        return (two_wire_field(grid, cell, cur, (+1, -1))).astype(np.float32), cur, 0.0
    cur = i_bright * dark_current_ratio
    lx = grid[0] * cell[0]
    lo, hi = 0.0, 0.4 * lx

    def g_of(off):
        b = two_wire_field(grid, cell, cur, (+1, +1), offset=off)
        S = Ms * n_mag * vcell / (HBAR * GAMMA)
        return GAMMA * math.sqrt(S / 2) * _mean_perp(b, mask) / (2 * math.pi)

    for _ in range(60):
        mid = 0.5 * (lo + hi)
        if g_of(mid) < g_target:
            lo = mid
        else:
            hi = mid
    off = 0.5 * (lo + hi)
    return two_wire_field(grid, cell, cur, (+1, +1), offset=off).astype(np.float32), cur, off


def strip_map(grid, cell, current=11.3e-9, width=100e-9, thickness=50e-9, gap=10e-9, nq=16):
    """Field of an infinite strip conductor || x (cpw centre line) below the film,
    uniform current density, 2D Gauss-Legendre Biot-Savart over the cross-section."""
    nx, ny, nz = grid
    X, Y, Z = cell_centres(grid, cell)
    zb = -nz * cell[2] / 2           # bottom face of the magnet
    zc = zb - gap - thickness / 2    # strip centre
    xg, wg = np.polynomial.legendre.leggauss(nq)
    by = np.zeros_like(Y)
    bz = np.zeros_like(Y)
    jw = current / (width * thickness)
    for yi, wy in zip(xg * width / 2, wg * width / 2):
        for zi, wz in zip(xg * thickness / 2 + zc, wg * thickness / 2):
            dy_, dz_ = Y - yi, Z - zi
            r2 = dy_**2 + dz_**2
            pref = MU0 * jw * wy * wz / (2 * math.pi)
            by += pref * (-dz_) / r2
            bz += pref * dy_ / r2
    b = np.stack([np.zeros_like(by), by, bz], axis=-1).reshape(-1, 3)
    return b.astype(np.float32)


def uniform_brms_for_g(grid, cell, Ms, mask, g_target, direction=(0, 1, 0)):
    n_mag = int(mask.sum()) if mask is not None else int(np.prod(grid))
    d = np.asarray(direction, float)
    d /= np.linalg.norm(d)
    amp = _coupling_scale(1.0, Ms, n_mag, float(np.prod(cell)), g_target)
    return tuple(float(v) for v in amp * d)


def film_kittel_bias(f, Ms):
    """B with gamma*sqrt(B(B+mu0 Ms)) = 2 pi f (thin-film Kittel; input choice for configs[0])."""
    w = 2 * math.pi * f / GAMMA
    a = MU0 * Ms
    return (-a + math.sqrt(a * a + 4 * w * w)) / 2


# ---------------------------------------------------------------- BJ configs

def _excitation(brms_map, brms_uniform, target=1e-3):
    bmax = float(np.abs(brms_map).max()) if brms_map is not None else float(np.linalg.norm(brms_uniform))
    return (target / bmax) if bmax > 0 else 0.0


def make_config(k: int, grid=None, seed=None, state="phys") -> Config:
    """BASELINE.json configs[k] (k = 0..4), optionally on a smaller grid with the same
    construction (used for parity tests).  ``state`` = "phys" | "rand"."""
    if k == 0:
        grid = grid or (64, 64, 1)
        cell = (5e-9, 5e-9, 5e-9)
        seed = 1001 if seed is None else seed
        rng = np.random.default_rng(seed)
        mat = YIG
        f_c = 10e9
        b = film_kittel_bias(f_c, mat["Ms"])
        brms_u = uniform_brms_for_g(grid, cell, mat["Ms"], None, 100e6, (0, 1, 0))
        m0 = tilted_uniform(int(np.prod(grid)), rng, (1, 0, 0), 0.05) if state == "phys" \
            else random_unit(int(np.prod(grid)), rng)
        return Config("configs[0] thin film", grid, cell, m0=m0, bext=(b, 0.0, 0.0),
                      brms_uniform=brms_u, f_c=f_c, exc_amp=_excitation(None, brms_u),
                      exc_omega=2 * math.pi * 30e9, dt=0.5e-12, seed=seed, **mat)
    if k in (1, 2):
        grid = grid or (128, 128, 128)
        box = 1e-6
        cell = (box / 128,) * 3 if grid == (128, 128, 128) else (box / grid[0], box / grid[1], box / grid[2])
        seed = (1002 if k == 1 else 1003) if seed is None else seed
        rng = np.random.default_rng(seed)
        mat = YIG
        mask = sphere_mask(grid, cell, 500e-9)
        f_c = 13.2e9 if k == 1 else 20.8e9
        bz = 2 * math.pi * f_c / GAMMA
        if k == 1:
            brms, _, _ = two_wire_map(grid, cell, mat["Ms"], mask, 1e9, "bright")
        else:
            brms, _, _ = two_wire_map(grid, cell, mat["Ms"], mask, 30e6, "dark")
        n = int(np.prod(grid))
        m0 = tilted_uniform(n, rng, (0, 0, 1), 0.05, mask) if state == "phys" else random_unit(n, rng, mask)
        return Config(f"configs[{k}] YIG sphere {'bright' if k == 1 else 'dark'}", grid, cell, m0=m0,
                      mask=mask, bext=(0.0, 0.0, bz), brms_map=brms, f_c=f_c,
                      exc_amp=_excitation(brms, None), exc_omega=2 * math.pi * 30e9,
                      dt=0.5e-12, seed=seed, **mat)
    if k == 3:
        grid = grid or (512, 512, 8)
        cell = (1e-6 / grid[0], 1e-6 / grid[1], 20e-9 / grid[2])
        seed = 1004 if seed is None else seed
        rng = np.random.default_rng(seed)
        mat = PY
        mask = disc_mask(grid, cell, 500e-9)
        brms = strip_map(grid, cell)
        n = int(np.prod(grid))
        m0 = vortex_state(grid, cell, mask=mask) if state == "phys" else random_unit(n, rng, mask)
        return Config("configs[3] Py vortex disc", grid, cell, m0=m0, mask=mask,
                      brms_map=brms, f_c=0.55e9, exc_amp=_excitation(brms, None),
                      exc_omega=2 * math.pi * 30e9, dt=0.1e-12, seed=seed,
                      relax_first=True, **mat)
    if k == 4:
        grid = grid or (512, 512, 256)
        cell = (7.8125e-9,) * 3
        seed = 1005 if seed is None else seed
        rng = np.random.default_rng(seed)
        mat = YIG
        f_c = 13.2e9
        brms, _, _ = two_wire_map(grid, cell, mat["Ms"], None, 1e9, "bright")
        n = int(np.prod(grid))
        m0 = tilted_uniform(n, rng, (0, 0, 1), 0.05) if state == "phys" else random_unit(n, rng)
        return Config("configs[4] large slab", grid, cell, m0=m0, bext=(0.0, 0.0, 2 * math.pi * f_c / GAMMA),
                      brms_map=brms, f_c=f_c, exc_amp=_excitation(brms, None),
                      exc_omega=2 * math.pi * 30e9, dt=0.5e-12, seed=seed, **mat)
    raise ValueError(k)


CONFIGS = {0: "64x64x1 thin film", 1: "YIG sphere 128^3 bright", 2: "YIG sphere 128^3 dark",
           3: "Py vortex disc 512x512x8", 4: "large slab 512x512x256"}


def small_config(kind: str, grid, seed=7, aniso=None, state="rand") -> Config:
    """Small parity cases spanning several tiles with ragged tails.  ``kind`` picks the
    construction: 'film' (full box, uniform B_rms), 'sphere' (masked, map), 'disc'."""
    rng = np.random.default_rng(seed)
    n = int(np.prod(grid))
    if kind == "film":
        cell = (5e-9, 5e-9, 5e-9)
        mat = YIG
        brms_u = uniform_brms_for_g(grid, cell, mat["Ms"], None, 100e6, (0, 1, 0))
        m0 = random_unit(n, rng) if state == "rand" else tilted_uniform(n, rng, (1, 0, 0), 0.1)
        return Config(f"film{grid}", grid, cell, m0=m0, bext=(0.28, 0.01, 0.02), brms_uniform=brms_u,
                      f_c=10e9, exc_amp=50.0, exc_omega=2 * math.pi * 30e9, aniso=aniso,
                      x0=0.3, p0=-0.2, seed=seed, **mat)
    if kind == "sphere":
        cell = (7.8125e-9,) * 3
        mat = YIG
        r = 0.45 * min(g * c for g, c in zip(grid, cell))
        mask = sphere_mask(grid, cell, r)
        brms, _, _ = two_wire_map(grid, cell, mat["Ms"], mask, 1e9, "bright")
        m0 = random_unit(n, rng, mask) if state == "rand" else tilted_uniform(n, rng, (0, 0, 1), 0.1, mask)
        return Config(f"sphere{grid}", grid, cell, m0=m0, mask=mask, bext=(0.0, 0.0, 0.4714),
                      brms_map=brms, f_c=13.2e9, exc_amp=_excitation(brms, None),
                      exc_omega=2 * math.pi * 30e9, aniso=aniso, x0=0.1, p0=0.05, seed=seed, **mat)
    if kind == "disc":
        cell = (1.953125e-9, 1.953125e-9, 2.5e-9)
        mat = PY
        r = 0.48 * min(grid[0] * cell[0], grid[1] * cell[1])
        mask = disc_mask(grid, cell, r)
        brms = strip_map(grid, cell)
        m0 = vortex_state(grid, cell, mask=mask, core=4e-9) if state == "phys" else random_unit(n, rng, mask)
        return Config(f"disc{grid}", grid, cell, m0=m0, mask=mask, brms_map=brms, f_c=0.55e9,
                      exc_amp=_excitation(brms, None), exc_omega=2 * math.pi * 30e9, aniso=aniso,
                      dt=0.1e-12, seed=seed, **mat)
    raise ValueError(kind)


def bias_sweep(center, n=41, rel=0.1):
    """Bias-field sweep points for an anticrossing (configs[0], configs[1] replicas)."""
    return list(np.linspace(center * (1 - rel), center * (1 + rel), n))
