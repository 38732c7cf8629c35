"""Test helpers: build the oracle and the CUDA solver from the same synthetic Config."""
import numpy as np

from oracle import sim as S


def oracle_from(cfg, demag="auto", octant=None):
    return S.Simulation(cfg.grid, cfg.cell, cfg.Ms, cfg.Aex, cfg.alpha, cfg.m0, mask=cfg.mask, bext=cfg.bext,
                        brms_map=cfg.brms_map, brms_uniform=cfg.brms_uniform, f_c=cfg.f_c, kappa=cfg.kappa,
                        x0=cfg.x0, p0=cfg.p0, exc_amp=cfg.exc_amp, exc_omega=cfg.exc_omega, aniso=cfg.aniso,
                        demag=demag, octant=octant)


def magmask(cfg):
    return np.ones(cfg.n, bool) if cfg.mask is None else cfg.mask.astype(bool)


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


# oracle term bits == ABI term bits (both follow the same list; asserted in test_abi.py)
TERMS = {"zeeman": 1, "exchange": 2, "anis": 4, "demag": 8, "cavity": 16, "excitation": 32}
