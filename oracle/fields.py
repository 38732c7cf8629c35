"""Effective-field terms (oracle, fp64).  Test infrastructure only.

Arrays: m has shape (nz, ny, nx, 3), x fastest; ``mag`` is the boolean
magnetic mask of shape (nz, ny, nx) (vacuum cells carry m = 0, M_s = 0).
Every term returns B in tesla with shape (nz, ny, nx, 3).

B_eff' = B_ext + B_exch + B_anis + B_demag + a sinc(w t) B_rms + B_rms Gamma(t)
(P:188 lists the Mumax3 terms; P:237-239 adds B_cav = B_rms Gamma; P:165 the
excitation).  The summation order is fixed in ``total`` (reading C12).
"""
from __future__ import annotations

import numpy as np

from .constants import MU0
from . import tensor as _tensor


def zeeman(shape, bext):
    """Uniform external field B_ext."""
    return np.broadcast_to(np.asarray(bext, dtype=np.float64), tuple(shape) + (3,)).copy()


def exchange(m, mag, cell, Aex, Ms):
    """6-neighbour exchange (reading C9): B_i = (2A/M_s) sum_axes sum_+- (m_j - m_i)/d^2,
    only over neighbours j inside the mesh and magnetic (free/Neumann boundary)."""
    out = np.zeros_like(m)
    nz, ny, nx, _ = m.shape
    for axis, d in ((2, cell[0]), (1, cell[1]), (0, cell[2])):
        n = m.shape[axis]
        for shift in (-1, +1):
            nb = np.roll(m, -shift, axis=axis)        # nb[i] = m[i + shift]
            nbmag = np.roll(mag, -shift, axis=axis)
            valid = nbmag.copy()
            idx = [slice(None)] * 3
            idx[axis] = n - 1 if shift == +1 else 0   # neighbour outside the mesh
            valid[tuple(idx)] = False
            out += np.where(valid[..., None], (nb - m) / (d * d), 0.0)
    out *= 2 * Aex / Ms
    return np.where(mag[..., None], out, 0.0)


def _neighbour(m, mag, axis, shift):
    """m at i + shift along `axis`, with the cell's own m where the neighbour is outside the
    mesh or in vacuum (Neumann ghost, reading C-DMI)."""
    nb = np.roll(m, -shift, axis=axis)
    valid = np.roll(mag, -shift, axis=axis).copy()
    idx = [slice(None)] * 3
    idx[axis] = m.shape[axis] - 1 if shift == +1 else 0
    valid[tuple(idx)] = False
    return np.where(valid[..., None], nb, m)


def dmi_interfacial(m, mag, cell, D, Ms):
    """Interfacial DMI (P:188 lists DMI among Mumax3's field terms; reading C-DMI):
    energy density D [m_z div m - (m . grad) m_z] (in-plane derivatives), field
    B = (2D/M_s) (d_x m_z, d_y m_z, -(d_x m_x + d_y m_y)) with central differences
    d_x f = (f_{x+1} - f_{x-1}) / (2 dx) and Neumann ghosts at mesh / vacuum boundaries (the
    DMI-tilted boundary condition of Mumax3 is not modelled)."""
    dxp, dxm = _neighbour(m, mag, 2, +1), _neighbour(m, mag, 2, -1)
    dyp, dym = _neighbour(m, mag, 1, +1), _neighbour(m, mag, 1, -1)
    ddx = (dxp - dxm) / (2 * cell[0])
    ddy = (dyp - dym) / (2 * cell[1])
    out = np.zeros_like(m)
    out[..., 0] = ddx[..., 2]
    out[..., 1] = ddy[..., 2]
    out[..., 2] = -(ddx[..., 0] + ddy[..., 1])
    return np.where(mag[..., None], (2 * D / Ms) * out, 0.0)


def uniaxial(m, mag, Ku1, u, Ms):
    """First-order uniaxial anisotropy (reading C10): B = (2K_u1/M_s)(m.u)u."""
    u = np.asarray(u, dtype=np.float64)
    u = u / np.linalg.norm(u)
    mu = m @ u
    return np.where(mag[..., None], (2 * Ku1 / Ms) * mu[..., None] * u, 0.0)


def cubic(m, mag, Kc1, c1, c2, Ms):
    """Cubic anisotropy, energy K_c1 (m1^2 m2^2 + m2^2 m3^2 + m3^2 m1^2), c3 = c1 x c2 (C10):
    B = -(2K_c1/M_s)[m1(m2^2+m3^2)c1 + m2(m1^2+m3^2)c2 + m3(m1^2+m2^2)c3]."""
    c1 = np.asarray(c1, dtype=np.float64)
    c2 = np.asarray(c2, dtype=np.float64)
    c1 = c1 / np.linalg.norm(c1)
    c2 = c2 / np.linalg.norm(c2)
    c3 = np.cross(c1, c2)
    m1, m2, m3 = m @ c1, m @ c2, m @ c3
    b = (m1 * (m2**2 + m3**2))[..., None] * c1 + (m2 * (m1**2 + m3**2))[..., None] * c2 \
        + (m3 * (m1**2 + m2**2))[..., None] * c3
    return np.where(mag[..., None], -(2 * Kc1 / Ms) * b, 0.0)


def demag_bruteforce(m, mag, cell, Ms, octant=None):
    """Plain real-space sum B_i = -mu0 sum_j N(r_i - r_j) M_j, M = M_s m (C11).  O(N^2)."""
    nz, ny, nx, _ = m.shape
    if octant is None:
        octant = _tensor.tensor_octant((nx, ny, nz), cell)
    K, J, I = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    I, J, K = I.ravel(), J.ravel(), K.ravel()
    M = (Ms * m * mag[..., None]).reshape(-1, 3)
    src = np.nonzero(mag.ravel())[0]
    out = np.zeros((I.size, 3))
    blk = max(1, (1 << 22) // max(1, src.size))
    for s in range(0, I.size, blk):
        t = np.arange(s, min(I.size, s + blk))
        N = _tensor.signed_lookup(octant, I[t, None] - I[None, src], J[t, None] - J[None, src],
                                  K[t, None] - K[None, src])          # (6, nt, ns)
        Ms_ = M[src]
        bx = N[0] @ Ms_[:, 0] + N[3] @ Ms_[:, 1] + N[4] @ Ms_[:, 2]
        by = N[3] @ Ms_[:, 0] + N[1] @ Ms_[:, 1] + N[5] @ Ms_[:, 2]
        bz = N[4] @ Ms_[:, 0] + N[5] @ Ms_[:, 1] + N[2] @ Ms_[:, 2]
        out[t] = -MU0 * np.stack([bx, by, bz], axis=1)
    return out.reshape(nz, ny, nx, 3)


def demag_at(m, mag, cell, Ms, points, octant):
    """Brute-force demag field at selected cells ``points`` = [(x,y,z), ...] (sampled parity
    at full size).  Same definition as demag_bruteforce."""
    nz, ny, nx, _ = m.shape
    K, J, I = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    sel = mag.ravel()
    I, J, K = I.ravel()[sel], J.ravel()[sel], K.ravel()[sel]
    M = (Ms * m.reshape(-1, 3))[sel]
    out = []
    for (x, y, z) in points:
        N = _tensor.signed_lookup(octant, x - I, y - J, z - K)
        b = np.array([N[0] @ M[:, 0] + N[3] @ M[:, 1] + N[4] @ M[:, 2],
                      N[3] @ M[:, 0] + N[1] @ M[:, 1] + N[5] @ M[:, 2],
                      N[4] @ M[:, 0] + N[5] @ M[:, 1] + N[2] @ M[:, 2]])
        out.append(-MU0 * b)
    return np.array(out)


def _dft_matrix(L, inverse=False):
    k = np.arange(L)
    sign = 1.0 if inverse else -1.0
    return np.exp(sign * 2j * np.pi * np.outer(k, k) / L)


def demag_dft(m, mag, cell, Ms, padded=None):
    """Same convolution via an explicit direct DFT (no FFT library): zero-pad M to
    (2nz, 2ny, 2nx), apply the DFT matrices per axis, multiply by the DFT of the cyclic
    padded tensor, invert, crop.  Exact because padding >= 2n-1 (C11)."""
    nz, ny, nx, _ = m.shape
    if padded is None:
        padded = _tensor.padded_tensor((nx, ny, nz), cell)
    _, Lz, Ly, Lx = padded.shape
    Fx, Fy, Fz = _dft_matrix(Lx), _dft_matrix(Ly), _dft_matrix(Lz)

    def fwd(a):   # a: (c, Lz, Ly, Lx) complex; DFT over the last three axes (matmuls)
        c = a.shape[0]
        a = a @ Fx.T                                       # x
        a = Fy @ a                                         # y (broadcast over c, z)
        a = (Fz @ a.reshape(c, Lz, Ly * Lx)).reshape(c, Lz, Ly, Lx)   # z
        return a

    Mp = np.zeros((3, Lz, Ly, Lx), dtype=np.complex128)
    Mp[:, :nz, :ny, :nx] = np.moveaxis(Ms * m * mag[..., None], -1, 0)
    Mh = fwd(Mp)
    del Mp
    Nh = fwd(padded.astype(np.complex128))
    xx, yy, zz, xy, xz, yz = Nh
    Bh = np.stack([xx * Mh[0] + xy * Mh[1] + xz * Mh[2],
                   xy * Mh[0] + yy * Mh[1] + yz * Mh[2],
                   xz * Mh[0] + yz * Mh[1] + zz * Mh[2]])
    del Nh, Mh
    Gx, Gy, Gz = _dft_matrix(Lx, True)[:nx], _dft_matrix(Ly, True)[:ny], _dft_matrix(Lz, True)[:nz]
    b = (Gz @ Bh.reshape(3, Lz, Ly * Lx)).reshape(3, nz, Ly, Lx)
    b = Gy @ b
    b = b @ Gx.T
    b = b.real / (Lx * Ly * Lz)
    return np.moveaxis(-MU0 * b, 0, -1)


def sinc(x):
    """Unnormalised sinc, sinc(0) = 1 (reading C13)."""
    x = np.asarray(x, dtype=np.float64)
    return np.where(x == 0, 1.0, np.sin(x) / np.where(x == 0, 1.0, x))
