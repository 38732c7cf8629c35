"""Demagnetising tensor of orthorhombic cells (oracle, fp64).  Test infrastructure only.

PAPER.md only names the demag field and defers to Mumax3; the definition
used here is reading C11:

* near field, max(|i|,|j|,|k|) <= NEAR (=16): Newell's cell-averaged tensor,
  the 27-point second difference of f (diagonal) / g (off-diagonal);
* far field: the point-dipole tensor (V/4 pi r^3)(I - 3 r^ r^) averaged over the
  source and target cells with 3-point Gauss-Legendre quadrature per axis.

Components are ordered XX, YY, ZZ, XY, XZ, YZ.  B_demag,i = -mu0 sum_j N(r_i - r_j) M_j.
Pins (tests/test_oracle_tensor.py): cube self-term 1/3, self-term trace 1, self-term
equal to Aharoni's closed-form prism factor, far field -> dipole, Newell vs
Gauss-Legendre in the overlap band, sum rule over a box = Aharoni of the box.
"""
from __future__ import annotations

import math

import numpy as np

NEAR = 16
COMPONENTS = ("xx", "yy", "zz", "xy", "xz", "yz")


def _asinh_ratio(num, den):
    """asinh(num/den) with den==0 mapped to 0 (callers zero the coefficient there)."""
    safe = np.where(den > 0, den, 1.0)
    return np.where(den > 0, np.arcsinh(num / safe), 0.0)


def _atan_ratio(num, den):
    safe = np.where(den != 0, den, 1.0)
    return np.where(den != 0, np.arctan(num / safe), 0.0)


def newell_f(x, y, z):
    """Newell's f(x,y,z); terms whose coefficient vanishes are 0."""
    x, y, z = (np.asarray(a, dtype=np.float64) for a in (x, y, z))
    x2, y2, z2 = x * x, y * y, z * z
    R = np.sqrt(x2 + y2 + z2)
    t1 = 0.5 * y * (z2 - x2) * _asinh_ratio(y, np.sqrt(x2 + z2))
    t2 = 0.5 * z * (y2 - x2) * _asinh_ratio(z, np.sqrt(x2 + y2))
    t3 = -x * y * z * _atan_ratio(y * z, x * R)
    t4 = (2 * x2 - y2 - z2) * R / 6.0
    return t1 + t2 + t3 + t4


def newell_g(x, y, z):
    """Newell's g(x,y,z)."""
    x, y, z = (np.asarray(a, dtype=np.float64) for a in (x, y, z))
    x2, y2, z2 = x * x, y * y, z * z
    R = np.sqrt(x2 + y2 + z2)
    t1 = x * y * z * _asinh_ratio(z, np.sqrt(x2 + y2))
    t2 = y / 6.0 * (3 * z2 - y2) * _asinh_ratio(x, np.sqrt(y2 + z2))
    t3 = x / 6.0 * (3 * z2 - x2) * _asinh_ratio(y, np.sqrt(x2 + z2))
    t4 = -z2 * z / 6.0 * _atan_ratio(x * y, z * R)
    t5 = -z * y2 / 2.0 * _atan_ratio(x * z, y * R)
    t6 = -z * x2 / 2.0 * _atan_ratio(y * z, x * R)
    t7 = -x * y * R / 3.0
    return t1 + t2 + t3 + t4 + t5 + t6 + t7


_W = {-1: -1.0, 0: 2.0, 1: -1.0}


def _second_difference(fun, X, Y, Z, dx, dy, dz):
    acc = np.zeros(np.broadcast(X, Y, Z).shape)
    for a in (-1, 0, 1):
        for b in (-1, 0, 1):
            for c in (-1, 0, 1):
                acc = acc + _W[a] * _W[b] * _W[c] * fun(X + a * dx, Y + b * dy, Z + c * dz)
    return acc


def newell(X, Y, Z, dx, dy, dz):
    """All six Newell components at offsets (X,Y,Z) (metres).  Returns (6, ...)."""
    pre = 1.0 / (4 * math.pi * dx * dy * dz)
    nxx = _second_difference(newell_f, X, Y, Z, dx, dy, dz)
    nyy = _second_difference(lambda a, b, c: newell_f(b, a, c), X, Y, Z, dx, dy, dz)
    nzz = _second_difference(lambda a, b, c: newell_f(c, b, a), X, Y, Z, dx, dy, dz)
    nxy = _second_difference(newell_g, X, Y, Z, dx, dy, dz)
    nxz = _second_difference(lambda a, b, c: newell_g(a, c, b), X, Y, Z, dx, dy, dz)
    nyz = _second_difference(lambda a, b, c: newell_g(b, c, a), X, Y, Z, dx, dy, dz)
    return pre * np.stack([nxx, nyy, nzz, nxy, nxz, nyz])


def point_dipole(X, Y, Z, V):
    """(V / 4 pi r^3)(I - 3 r^ r^) at r = (X,Y,Z); r must be nonzero."""
    r2 = X * X + Y * Y + Z * Z
    r = np.sqrt(r2)
    pre = V / (4 * math.pi * r2 * r)
    return np.stack([pre * (1 - 3 * X * X / r2), pre * (1 - 3 * Y * Y / r2), pre * (1 - 3 * Z * Z / r2),
                     pre * (-3 * X * Y / r2), pre * (-3 * X * Z / r2), pre * (-3 * Y * Z / r2)])


def _gl3_difference_rule():
    """Nodes/weights of (xi_s - xi_t) for 3-point Gauss-Legendre on [-1/2,1/2]^2 (merged)."""
    a = math.sqrt(3.0 / 5.0) / 2.0
    nodes = (-a, 0.0, a)
    w = (5.0 / 18.0, 8.0 / 18.0, 5.0 / 18.0)
    rule = {}
    for i in range(3):
        for j in range(3):
            key = round((nodes[i] - nodes[j]) / a)
            rule[key] = rule.get(key, 0.0) + w[i] * w[j]
    return [(k * a, wt) for k, wt in sorted(rule.items())]


GL3_RULE = _gl3_difference_rule()


def far_field(X, Y, Z, dx, dy, dz):
    """Cell-pair-averaged point-dipole tensor, 3-point Gauss-Legendre per axis (C11)."""
    V = dx * dy * dz
    acc = 0.0
    for u, wu in GL3_RULE:
        for v, wv in GL3_RULE:
            for s, ws in GL3_RULE:
                acc = acc + (wu * wv * ws) * point_dipole(X + u * dx, Y + v * dy, Z + s * dz, V)
    return acc


def tensor_octant(m, cell, near=NEAR, chunk=1 << 20):
    """N_ab for index offsets (i,j,k), 0<=i<mx, 0<=j<my, 0<=k<mz.  Returns (6, mz, my, mx)."""
    mx, my, mz = m
    dx, dy, dz = cell
    out = np.empty((6, mz, my, mx))
    K, J, I = np.meshgrid(np.arange(mz), np.arange(my), np.arange(mx), indexing="ij")
    I, J, K = I.ravel(), J.ravel(), K.ravel()
    flat = out.reshape(6, -1)
    for s in range(0, I.size, chunk):
        i, j, k = I[s:s + chunk], J[s:s + chunk], K[s:s + chunk]
        isnear = np.maximum(np.maximum(i, j), k) <= near
        vals = np.empty((6, i.size))
        if (~isnear).any():
            f = ~isnear
            vals[:, f] = far_field(i[f] * dx, j[f] * dy, k[f] * dz, dx, dy, dz)
        if isnear.any():
            vals[:, isnear] = newell(i[isnear] * dx, j[isnear] * dy, k[isnear] * dz, dx, dy, dz)
        flat[:, s:s + chunk] = vals
    return out


# parity of each component under a sign flip of (x, y, z) offsets
PARITY = np.array([[1, 1, 1], [1, 1, 1], [1, 1, 1], [-1, -1, 1], [-1, 1, -1], [1, -1, -1]])


def signed_lookup(octant, di, dj, dk):
    """N(di,dj,dk) for signed integer offsets from an octant table (6, mz, my, mx)."""
    di, dj, dk = (np.asarray(a) for a in (di, dj, dk))
    vals = octant[:, np.abs(dk), np.abs(dj), np.abs(di)]
    sx, sy, sz = np.sign(di), np.sign(dj), np.sign(dk)
    signs = np.stack([np.ones_like(sx), np.ones_like(sx), np.ones_like(sx), sx * sy, sx * sz, sy * sz])
    return vals * signs


def padded_length(n):
    """Oracle's own zero-padded length: 2n (n>1), 1 (n==1); any L >= 2n-1 is exact."""
    return 1 if n == 1 else 2 * n


def padded_tensor(grid, cell, octant=None):
    """Full cyclic zero-padded tensor (6, Lz, Ly, Lx): offset -o sits at index L-o, other
    slots (|offset| >= n) are zero."""
    nx, ny, nz = grid
    if octant is None:
        octant = tensor_octant((nx, ny, nz), cell)
    L = [padded_length(n) for n in (nx, ny, nz)]

    def offsets(n, Ln):
        p = np.arange(Ln)
        o = np.where(p < n, p, p - Ln)
        valid = (p < n) | (p > Ln - n)
        return o, valid

    ox, vx = offsets(nx, L[0])
    oy, vy = offsets(ny, L[1])
    oz, vz = offsets(nz, L[2])
    OZ, OY, OX = np.meshgrid(oz, oy, ox, indexing="ij")
    V = (vz[:, None, None] & vy[None, :, None] & vx[None, None, :])
    T = signed_lookup(octant, np.where(V, OX, 0), np.where(V, OY, 0), np.where(V, OZ, 0))
    return T * V[None]
