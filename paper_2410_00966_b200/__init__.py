"""B200-native Mumax3-cQED hot path (arXiv 2410.00966): LLG + single damped cavity mode.

Thin Python binding of the C ABI in ``include/mcq.h`` — the functions below carry the ABI's
names and only marshal arguments (numpy host arrays, or integer device pointers such as
``torch.Tensor.data_ptr()``).  All computation happens in ``libmcq.so`` (sm_100a CUDA).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import (lib, MCQError, mcq_aniso, mcq_dist, mcq_cavity_state, EXPORTED,  # noqa: F401
                   TERM_ZEEMAN, TERM_EXCHANGE, TERM_ANIS, TERM_DEMAG, TERM_CAVITY, TERM_EXCITATION,
                   TERM_DMI, TERM_ALL, TERM_THERM, NKCLASS, KCLASS_NAMES, K_YFWD, K_ZCONV, K_YINV, K_Y2D, K_UPDATE, K_CAVITY)

__all__ = [n for n in EXPORTED] + ["Solver", "MCQError"]


def _check(ctx, rc):
    if rc != 0:
        msg = lib.mcq_last_error(ctx)
        raise MCQError(rc, msg.decode() if msg else "")


def _vec(a, n=None, dtype=np.float32):
    arr = np.ascontiguousarray(a, dtype=dtype).reshape(-1)
    if n is not None and arr.size != n:
        raise ValueError(f"expected {n} values, got {arr.size}")
    return arr


def _d3(v):
    return (C.c_double * 3)(*[float(x) for x in v])


# ---------------------------------------------------------------- ABI-named functions

def mcq_nccl_get_unique_id():
    """128-byte NCCL unique id (bytes) for a multi-process context (include/mcq.h)."""
    buf = (C.c_ubyte * 128)()
    rc = lib.mcq_nccl_get_unique_id(buf)
    if rc != 0:
        raise MCQError(rc, "mcq_nccl_get_unique_id failed (libnccl.so.2 not loadable)")
    return bytes(buf)


def mcq_create(grid, cell, Ms, Aex, alpha, K=None, dist=None):
    """dist: None or {"rank", "world", "device", "nccl_id" (bytes), "stream"}; rank < 0 = loopback
    slabs in this process (include/mcq.h, mcq_dist)."""
    h = C.c_void_p()
    g = (C.c_int * 3)(*[int(x) for x in grid])
    c = (C.c_double * 3)(*[float(x) for x in cell])
    kp = None
    if K:
        k = mcq_aniso()
        k.ku1 = float(K.get("ku1", 0.0))
        k.u = _d3(K.get("u", (0, 0, 1)))
        k.kc1 = float(K.get("kc1", 0.0))
        k.c1 = _d3(K.get("c1", (1, 0, 0)))
        k.c2 = _d3(K.get("c2", (0, 1, 0)))
        kp = C.pointer(k)
    dp = None
    idbuf = None
    if dist is not None:
        nid = dist.get("nccl_id")
        if nid is not None:
            idbuf = (C.c_ubyte * 128).from_buffer_copy(bytes(nid))
        d = mcq_dist(int(dist.get("rank", 0)), int(dist.get("world", 1)), int(dist.get("device", -1)),
                     C.cast(idbuf, C.c_void_p) if idbuf is not None else None, dist.get("stream"))
        dp = C.pointer(d)
    rc = lib.mcq_create(C.byref(h), g, c, float(Ms), float(Aex), float(alpha), kp, dp)
    if rc != 0:
        raise MCQError(rc, "mcq_create failed (invalid arguments, no device or out of memory)")
    return h


def mcq_set_persistent_2d(ctx, on):
    """nz == 1 grids: one persistent kernel per mcq_run (1) or per-step graphs (0) (include/mcq.h)."""
    _check(ctx, lib.mcq_set_persistent_2d(ctx, 1 if on else 0))


def mcq_set_slab_overlap(ctx, on):
    """z slabs: overlap the transposes with the per-component y passes (include/mcq.h)."""
    _check(ctx, lib.mcq_set_slab_overlap(ctx, 1 if on else 0))


def mcq_set_stream(ctx, stream):
    _check(ctx, lib.mcq_set_stream(ctx, C.c_void_p(stream) if stream else None))


def mcq_set_geometry(ctx, mask):
    if mask is None:
        _check(ctx, lib.mcq_set_geometry(ctx, None))
        return
    m = np.ascontiguousarray(mask, dtype=np.uint8).reshape(-1)
    _check(ctx, lib.mcq_set_geometry(ctx, m.ctypes.data))


def mcq_set_m(ctx, m):
    a = _vec(m)
    _check(ctx, lib.mcq_set_m(ctx, a.ctypes.data))


def mcq_set_m_device(ctx, dptr):
    _check(ctx, lib.mcq_set_m_device(ctx, C.c_void_p(int(dptr))))


def mcq_set_bext(ctx, B):
    _check(ctx, lib.mcq_set_bext(ctx, _d3(B)))


def mcq_set_brms(ctx, map=None, uniform=(0.0, 0.0, 0.0)):
    if map is not None:
        a = _vec(map)
        _check(ctx, lib.mcq_set_brms(ctx, a.ctypes.data, _d3(uniform)))
    else:
        _check(ctx, lib.mcq_set_brms(ctx, None, _d3(uniform)))


def mcq_set_cavity(ctx, f_c, kappa, x0=0.0, p0=0.0):
    _check(ctx, lib.mcq_set_cavity(ctx, float(f_c), float(kappa), float(x0), float(p0)))


def mcq_set_excitation(ctx, amplitude, omega_cut):
    _check(ctx, lib.mcq_set_excitation(ctx, float(amplitude), float(omega_cut)))


def mcq_set_dmi(ctx, D):
    """Interfacial DMI constant D (J/m^2), reading C-DMI (include/mcq.h)."""
    _check(ctx, lib.mcq_set_dmi(ctx, float(D)))


def mcq_set_temperature(ctx, T, seed=0):
    """Temperature (K) and thermal-stream seed, reading C-TH (include/mcq.h)."""
    _check(ctx, lib.mcq_set_temperature(ctx, float(T), int(seed) & (2**64 - 1)))


def mcq_get_thermal_step(ctx):
    """The thermal noise step n (counts mcq_run steps since mcq_set_temperature; reading C-TH)."""
    n = C.c_longlong()
    _check(ctx, lib.mcq_get_thermal_step(ctx, C.byref(n)))
    return n.value


def mcq_set_thermal_step(ctx, n):
    _check(ctx, lib.mcq_set_thermal_step(ctx, int(n)))


def mcq_reset_memory(ctx):
    _check(ctx, lib.mcq_reset_memory(ctx))


MAX_MODES = 4


def mcq_set_modes(ctx, nmodes):
    """Number of cavity modes (include/mcq.h, NEXT-2); mode 0 is the single-mode API's."""
    _check(ctx, lib.mcq_set_modes(ctx, int(nmodes)))


def mcq_set_brms_mode(ctx, k, map=None, uniform=(0.0, 0.0, 0.0)):
    a = _vec(map) if map is not None else None
    _check(ctx, lib.mcq_set_brms_mode(ctx, int(k), a.ctypes.data if a is not None else None, _d3(uniform)))


def mcq_set_cavity_mode(ctx, k, f_c, kappa, x0=0.0, p0=0.0):
    _check(ctx, lib.mcq_set_cavity_mode(ctx, int(k), float(f_c), float(kappa), float(x0), float(p0)))


def mcq_set_excitation_mode(ctx, k, amplitude, omega_cut):
    _check(ctx, lib.mcq_set_excitation_mode(ctx, int(k), float(amplitude), float(omega_cut)))


def mcq_get_cavity_mode(ctx, k):
    s = mcq_cavity_state()
    _check(ctx, lib.mcq_get_cavity_mode(ctx, int(k), C.byref(s)))
    return s.as_dict()


def mcq_set_cavity_state_mode(ctx, k, state):
    s = mcq_cavity_state()
    s.t = float(state["t"])
    s.re_alpha = float(state["re_alpha"])
    s.im_alpha = float(state["im_alpha"])
    s.step = int(state.get("step", 0))
    _check(ctx, lib.mcq_set_cavity_state_mode(ctx, int(k), C.byref(s)))


def mcq_relax(ctx, dt, torque_tol, max_steps):
    n = C.c_longlong(0)
    _check(ctx, lib.mcq_relax(ctx, float(dt), float(torque_tol), int(max_steps), C.byref(n)))
    return n.value


def mcq_run(ctx, dt, steps):
    _check(ctx, lib.mcq_run(ctx, float(dt), int(steps)))


def mcq_run_dp(ctx, dt, steps):
    """Fixed-step Dormand-Prince 5(4) (include/mcq.h, NEXT-1)."""
    _check(ctx, lib.mcq_run_dp(ctx, float(dt), int(steps)))


def mcq_run_adaptive(ctx, duration, dt0, tol, max_attempts=10**7):
    """Adaptive Dormand-Prince over `duration` s; returns (accepted, rejected, dt_next)."""
    a, r, d = C.c_longlong(), C.c_longlong(), C.c_double()
    _check(ctx, lib.mcq_run_adaptive(ctx, float(duration), float(dt0), float(tol), int(max_attempts),
                                     C.byref(a), C.byref(r), C.byref(d)))
    return a.value, r.value, d.value


def mcq_ovf_last_error():
    return lib.mcq_ovf_last_error().decode()


def mcq_ovf_read(path):
    """OVF 2.0 file -> (values (N, 3) float32 x-fastest, grid (nx, ny, nz), cell (dx, dy, dz))."""
    g = (C.c_int * 3)()
    c = (C.c_double * 3)()
    p = str(path).encode()
    rc = lib.mcq_ovf_read(p, g, c, None, 0)
    if rc != 0:
        raise MCQError(rc, mcq_ovf_last_error())
    n = g[0] * g[1] * g[2]
    out = np.empty(3 * n, np.float32)
    rc = lib.mcq_ovf_read(p, g, c, out.ctypes.data, out.size)
    if rc != 0:
        raise MCQError(rc, mcq_ovf_last_error())
    return out.reshape(n, 3), tuple(g), tuple(c)


def mcq_ovf_write(path, values, grid, cell, representation="binary4"):
    """Write a (N, 3) field as OVF 2.0: representation "text", "binary4" or "binary8"."""
    rep = {"text": 0, "binary4": 4, "binary8": 8}[representation]
    a = _vec(values)
    g = (C.c_int * 3)(*[int(x) for x in grid])
    c = (C.c_double * 3)(*[float(x) for x in cell])
    if a.size != 3 * g[0] * g[1] * g[2]:
        raise ValueError("values do not match the grid")
    rc = lib.mcq_ovf_write(str(path).encode(), g, c, a.ctypes.data, rep)
    if rc != 0:
        raise MCQError(rc, mcq_ovf_last_error())


def mcq_synchronize(ctx):
    _check(ctx, lib.mcq_synchronize(ctx))


def mcq_get_m(ctx, n_cells, out=None):
    out = np.empty(3 * n_cells, np.float32) if out is None else out
    _check(ctx, lib.mcq_get_m(ctx, out.ctypes.data))
    return out.reshape(n_cells, 3)


def mcq_get_m_device(ctx, dptr):
    _check(ctx, lib.mcq_get_m_device(ctx, C.c_void_p(int(dptr))))


def mcq_get_field(ctx, n_cells, terms=TERM_ALL):
    out = np.empty(3 * n_cells, np.float32)
    _check(ctx, lib.mcq_get_field(ctx, out.ctypes.data, C.c_uint(terms)))
    return out.reshape(n_cells, 3)


def mcq_get_cavity(ctx):
    s = mcq_cavity_state()
    _check(ctx, lib.mcq_get_cavity(ctx, C.byref(s)))
    return s.as_dict()


def mcq_cavity_state_bytes():
    """Bytes one mcq_get_cavity call copies device -> host."""
    return int(lib.mcq_cavity_state_bytes())


def mcq_set_cavity_state(ctx, state):
    s = mcq_cavity_state()
    s.t = float(state["t"])
    s.re_alpha = float(state["re_alpha"])
    s.im_alpha = float(state["im_alpha"])
    s.step = int(state.get("step", 0))
    _check(ctx, lib.mcq_set_cavity_state(ctx, C.byref(s)))


def mcq_cavity_status(ctx):
    rc = lib.mcq_cavity_status(ctx)
    if rc < 0:
        _check(ctx, rc)
    return rc


TRACE_COLS = ("t", "mx", "my", "mz", "re_alpha", "im_alpha", "W", "step")


def mcq_set_trace(ctx, capacity, every=1):
    """Record the per-step observables on the device (include/mcq.h, NEXT-3)."""
    _check(ctx, lib.mcq_set_trace(ctx, int(capacity), int(every)))


def mcq_get_trace(ctx, max_rows=None):
    """Recorded trace rows as an (n, 8) float64 array, columns TRACE_COLS."""
    n = C.c_longlong()
    _check(ctx, lib.mcq_get_trace(ctx, None, 0, C.byref(n)))
    rows = n.value if max_rows is None else min(n.value, int(max_rows))
    out = np.zeros((max(rows, 0), len(TRACE_COLS)), np.float64)
    got = C.c_longlong()
    if rows > 0:
        _check(ctx, lib.mcq_get_trace(ctx, out.ctypes.data, rows, C.byref(got)))
        out = out[:min(rows, got.value)]
    return out


# ---------------------------------------------------------------- NEXT-3: device spectroscopy
def mcq_trace_peaks(ctx, column=2, pad=8, window=1, fmin=0.0, npeaks=2):
    """Peaks (Hz, |X|) of a recorded trace column (1..7: <mx>, <my>, <mz>, Re a, Im a, W, step),
    computed on the device (include/mcq.h: FFT, parabolic interpolation, reading C23)."""
    f = np.zeros(npeaks)
    a = np.zeros(npeaks)
    n = C.c_int()
    _check(ctx, lib.mcq_trace_peaks(ctx, int(column), int(pad), int(window), float(fmin), int(npeaks),
                                    f.ctypes.data, a.ctypes.data, C.byref(n)))
    return f[:n.value].copy(), a[:n.value].copy()


def mcq_trace_peaks_batch(ctxs, column=2, pad=8, window=1, fmin=0.0, npeaks=2):
    """mcq_trace_peaks for several contexts (a sweep's replicas) in one batched device pass:
    list of (f, a) per context."""
    n = len(ctxs)
    arr = (C.c_void_p * n)(*[int(c) if not isinstance(c, C.c_void_p) else c.value for c in ctxs])
    f = np.zeros((n, npeaks))
    a = np.zeros((n, npeaks))
    nf = np.zeros(n, np.int32)
    rc = lib.mcq_trace_peaks_batch(arr, n, int(column), int(pad), int(window), float(fmin), int(npeaks),
                                   f.ctypes.data, a.ctypes.data, nf.ctypes.data)
    if rc != 0:
        raise MCQError(rc, lib.mcq_last_error(ctxs[0]).decode())
    return [(f[i, :nf[i]].copy(), a[i, :nf[i]].copy()) for i in range(n)]


def mcq_spectrum_peaks(signal, dt, pad=8, window=1, fmin=0.0, npeaks=2):
    """Device spectrum peaks of a host signal (context-free; include/mcq.h)."""
    x = np.ascontiguousarray(signal, np.float64)
    f = np.zeros(npeaks)
    a = np.zeros(npeaks)
    n = C.c_int()
    rc = lib.mcq_spectrum_peaks(x.ctypes.data, x.size, float(dt), int(pad), int(window), float(fmin), int(npeaks),
                                f.ctypes.data, a.ctypes.data, C.byref(n))
    if rc != 0:
        raise MCQError(rc, "mcq_spectrum_peaks")
    return f[:n.value].copy(), a[:n.value].copy()


def mcq_fit_anticrossing(w_mag, lo, hi, wc0, g0):
    """Device least-squares (omega_c, g) (rad/s) of the two-oscillator normal modes to two branches."""
    w = np.ascontiguousarray(w_mag, np.float64)
    lo = np.ascontiguousarray(lo, np.float64)
    hi = np.ascontiguousarray(hi, np.float64)
    wc, g = C.c_double(), C.c_double()
    rc = lib.mcq_fit_anticrossing(w.size, w.ctypes.data, lo.ctypes.data, hi.ctypes.data, float(wc0), float(g0),
                                  C.byref(wc), C.byref(g))
    if rc != 0:
        raise MCQError(rc, "mcq_fit_anticrossing")
    return wc.value, g.value


def mcq_kernel_launches(ctx):
    return int(lib.mcq_kernel_launches(ctx))


def mcq_profile_run(ctx, dt, steps):
    ms = (C.c_double * NKCLASS)()
    per = (C.c_int * NKCLASS)()
    _check(ctx, lib.mcq_profile_run(ctx, float(dt), int(steps), ms, per))
    return {KCLASS_NAMES[k]: (ms[k], per[k]) for k in range(NKCLASS)}


def mcq_debug_layout(ctx):
    out = (C.c_longlong * 6)()
    _check(ctx, lib.mcq_debug_layout(ctx, out))
    return dict(zip(("Lx", "Ly", "Lz", "NKX", "P", "n_partials"), list(out)))


def mcq_debug_tensor_octant(ctx):
    L = mcq_debug_layout(ctx)
    shape = (6, L["Lz"] // 2 + 1, L["Ly"] // 2 + 1, L["Lx"] // 2 + 1)
    out = np.empty(shape, np.float64)
    _check(ctx, lib.mcq_debug_tensor_octant(ctx, out.ctypes.data))
    return out


def mcq_debug_khat(ctx):
    L = mcq_debug_layout(ctx)
    shape = (L["Lz"] // 2 + 1, L["Ly"] // 2 + 1, L["P"], 6)
    out = np.empty(shape, np.float32)
    _check(ctx, lib.mcq_debug_khat(ctx, out.ctypes.data))
    return np.moveaxis(out, 3, 0)[..., :L["NKX"]]      # (6, kz, ky, kx) view


def mcq_last_error(ctx):
    return lib.mcq_last_error(ctx).decode()


def mcq_destroy(ctx):
    lib.mcq_destroy(ctx)


# ---------------------------------------------------------------- convenience wrapper

class Solver:
    """Owns one context; methods forward to the ABI functions above."""

    def __init__(self, grid, cell, Ms, Aex, alpha, aniso=None, stream=None, dist=None):
        self.grid = tuple(int(g) for g in grid)
        self.cell = tuple(float(c) for c in cell)
        self.n = self.grid[0] * self.grid[1] * self.grid[2]
        d = dict(dist or {})
        if stream:
            d["stream"] = stream
        self.ctx = mcq_create(grid, cell, Ms, Aex, alpha, aniso, d or None)

    @classmethod
    def from_config(cls, cfg, stream=None, set_state=True, dist=None):
        s = cls(cfg.grid, cfg.cell, cfg.Ms, cfg.Aex, cfg.alpha, cfg.aniso, stream, dist)
        if cfg.mask is not None:
            mcq_set_geometry(s.ctx, cfg.mask)
        mcq_set_bext(s.ctx, cfg.bext)
        mcq_set_brms(s.ctx, cfg.brms_map, cfg.brms_uniform)
        mcq_set_cavity(s.ctx, cfg.f_c, cfg.kappa, cfg.x0, cfg.p0)
        mcq_set_excitation(s.ctx, cfg.exc_amp, cfg.exc_omega)
        if set_state:
            mcq_set_m(s.ctx, cfg.m0)
        return s

    def set_m(self, m):
        mcq_set_m(self.ctx, m)

    def run(self, dt, steps):
        mcq_run(self.ctx, dt, steps)

    def relax(self, dt, tol, max_steps):
        return mcq_relax(self.ctx, dt, tol, max_steps)

    def m(self):
        return mcq_get_m(self.ctx, self.n)

    def field(self, terms=TERM_ALL):
        return mcq_get_field(self.ctx, self.n, terms)

    def cavity(self):
        return mcq_get_cavity(self.ctx)

    def set_brms_ovf(self, path, mode=0, rtol=1e-9):
        """B_rms of `mode` from an OVF 2.0 file: the node counts must equal the grid and
        the step sizes must match the cell within rtol (no resampling)."""
        vals, g, c = mcq_ovf_read(path)
        if tuple(g) != self.grid:
            raise ValueError(f"OVF grid {g} != solver grid {self.grid}")
        if any(abs(a - b) > rtol * abs(b) for a, b in zip(c, self.cell)):
            raise ValueError(f"OVF cell {c} != solver cell {self.cell}")
        mcq_set_brms_mode(self.ctx, mode, vals)

    def trace(self, capacity=None, every=1):
        """trace(capacity): start recording; trace(): the rows recorded so far."""
        if capacity is not None:
            mcq_set_trace(self.ctx, capacity, every)
            return None
        return mcq_get_trace(self.ctx)

    def sync(self):
        mcq_synchronize(self.ctx)

    def close(self):
        if getattr(self, "ctx", None) is not None:
            mcq_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
