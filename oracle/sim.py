"""The whole hot path, step by step (oracle, fp64).  Test infrastructure only.

Follows SURVEY §8(c) "Oracle algorithm": field B'(m, t) (step 3), torque (4), RK4 (5),
memory update after the step on the new state (6), relax (7).  Inputs come in as the
CUDA path receives them (fp32 m, B_rms), widened to fp64.

Multimode (P:24 runs each mode separately and calls a native multimode
cavity "straightforward"): reading C-MM — every extra mode k is its own damped oscillator with
its own B_rms,k, f_k, kappa_k, x0_k, p0_k and excitation; it is driven by its own overlap
W_k = sum_i M_s m_i . B_rms,k(r_i) through the same recursion, and the field gains
a_k sinc(w_k t) B_rms,k + B_rms,k Gamma_k(t).  The modes couple only through m.
"""
from __future__ import annotations

import math

import numpy as np

from .constants import GAMMA, HBAR
from . import fields as F
from . import tensor as T
from . import thermal as TH
from .cavity import CavityMemory
from .llg import torque, relax_torque, normalize, rk4_step, dp45_step, dp_controller

ZEEMAN, EXCHANGE, ANIS, DEMAG, CAVITY, EXCITATION, DMI = 1, 2, 4, 8, 16, 32, 64
ALL = ZEEMAN | EXCHANGE | ANIS | DEMAG | CAVITY | EXCITATION | DMI
THERM = 128    # the thermal field (reading C-TH): stochastic, so not part of ALL
RELAX_CHECK_EVERY = 50


class Simulation:
    def __init__(self, grid, cell, Ms, Aex, alpha, m0, mask=None, bext=(0.0, 0.0, 0.0),
                 brms_map=None, brms_uniform=(0.0, 0.0, 0.0), f_c=1e9, kappa=0.0, x0=0.0, p0=0.0,
                 exc_amp=0.0, exc_omega=0.0, aniso=None, demag="auto", octant=None, hbar=HBAR,
                 gamma=GAMMA, terms=ALL, modes=(), dmi=0.0, temperature=0.0, seed=0):
        self.grid = tuple(int(g) for g in grid)
        nx, ny, nz = self.grid
        self.shape = (nz, ny, nx)
        self.cell = tuple(float(c) for c in cell)
        self.vcell = self.cell[0] * self.cell[1] * self.cell[2]
        self.Ms, self.Aex, self.alpha = float(Ms), float(Aex), float(alpha)
        self.gamma = gamma
        self.mag = np.ones(self.shape, bool) if mask is None else np.asarray(mask).reshape(self.shape).astype(bool)
        self.m = np.asarray(m0, dtype=np.float64).reshape(self.shape + (3,)) * self.mag[..., None]
        self.m = normalize(self.m)
        self.bext = np.asarray(bext, dtype=np.float64)
        if brms_map is not None:
            self.brms = np.asarray(brms_map, dtype=np.float64).reshape(self.shape + (3,))
        else:
            self.brms = F.zeeman(self.shape, brms_uniform)
        self.aniso = aniso or {}
        self.dmi = float(dmi)       # interfacial DMI constant D (J/m^2), reading C-DMI
        self.temperature, self.seed = float(temperature), int(seed)   # reading C-TH
        # noise step n of the thermal stream: RK4 steps since the temperature / seed were set;
        # independent of the cavity memory clock (reset_memory / relax do not restart it, so
        # the segments of one run never reuse a draw) — reading C-TH
        self.th_step = 0
        self.th_dt = None           # dt of the last run: the thermal field's scale
        self._bth = None            # B_th of the step in progress
        self.exc_amp, self.exc_omega = float(exc_amp), float(exc_omega)
        self.mem = CavityMemory(2 * math.pi * f_c, kappa, x0, p0, self.vcell, hbar)
        # extra modes k >= 1 (reading C-MM): dicts with brms_map | brms_uniform, f_c, kappa,
        # x0, p0, exc_amp, exc_omega
        self.extra = []
        for md in modes:
            if md.get("brms_map") is not None:
                b = np.asarray(md["brms_map"], dtype=np.float64).reshape(self.shape + (3,))
            else:
                b = F.zeeman(self.shape, md.get("brms_uniform", (0.0, 0.0, 0.0)))
            mem = CavityMemory(2 * math.pi * md.get("f_c", 1e9), md.get("kappa", 0.0), md.get("x0", 0.0),
                               md.get("p0", 0.0), self.vcell, hbar)
            self.extra.append((b, mem, float(md.get("exc_amp", 0.0)), float(md.get("exc_omega", 0.0))))
        n = nx * ny * nz
        self.demag_mode = ("brute" if n <= 4096 else "dft") if demag == "auto" else demag
        self._octant = octant
        self._padded = None
        self.terms = terms          # enabled field terms (e.g. the Dicke mapping uses B_ext + cavity only)

    # ---------------------------------------------------------------- state
    @property
    def cavity_enabled(self):
        """CavityFeatureStatus: 1 iff B_rms set and nonzero (reading C14)."""
        return bool(np.any(self.brms != 0))

    def octant(self):
        if self._octant is None:
            nx, ny, nz = self.grid
            self._octant = T.tensor_octant((nx, ny, nz), self.cell)
        return self._octant

    # ---------------------------------------------------------------- field (step 3)
    def demag(self, m):
        if self.demag_mode == "brute":
            return F.demag_bruteforce(m, self.mag, self.cell, self.Ms, self.octant())
        if self.demag_mode == "dft":
            if self._padded is None:
                self._padded = T.padded_tensor(self.grid, self.cell, self.octant())
            return F.demag_dft(m, self.mag, self.cell, self.Ms, self._padded)
        return np.zeros_like(m)

    def field(self, m, t, terms=ALL):
        """B'(m, t) summed in the fixed order Zeeman, exchange, anisotropy, demag, excitation,
        cavity; vacuum cells get 0.  Gamma uses the S_n, C_n of the last completed step (C3)."""
        B = np.zeros_like(m)
        therm = terms & THERM
        terms &= self.terms
        if terms & ZEEMAN:
            B += F.zeeman(self.shape, self.bext)
        if terms & EXCHANGE and self.Aex != 0.0:
            B += F.exchange(m, self.mag, self.cell, self.Aex, self.Ms)
        if terms & ANIS:
            a = self.aniso
            if a.get("ku1", 0.0):
                B += F.uniaxial(m, self.mag, a["ku1"], a["u"], self.Ms)
            if a.get("kc1", 0.0):
                B += F.cubic(m, self.mag, a["kc1"], a["c1"], a["c2"], self.Ms)
        if terms & DEMAG and self.demag_mode != "off":
            B += self.demag(m)
        if terms & DMI and self.dmi != 0.0:
            B += F.dmi_interfacial(m, self.mag, self.cell, self.dmi, self.Ms)
        if terms & EXCITATION and self.exc_amp != 0.0:
            B += self.exc_amp * float(F.sinc(self.exc_omega * t)) * self.brms
        if terms & CAVITY and self.cavity_enabled:
            B += self.brms * self.mem.gamma(t)
        for b, mem, a_k, w_k in self.extra:          # modes k >= 1, in order (C-MM)
            if terms & EXCITATION and a_k != 0.0:
                B += a_k * float(F.sinc(w_k * t)) * b
            if terms & CAVITY and np.any(b != 0):
                B += b * mem.gamma(t)
        if therm and self.temperature > 0.0:       # the next step's draw (reading C-TH)
            if self.th_dt is None:
                raise RuntimeError("thermal field before any run (its scale needs dt)")
            B += self.thermal(self.th_dt)
        return np.where(self.mag[..., None], B, 0.0)

    def set_temperature(self, temperature, seed):
        """mcq_set_temperature: new T and seed; the noise step restarts at 0 (reading C-TH)."""
        self.temperature, self.seed, self.th_step = float(temperature), int(seed), 0

    def thermal(self, dt):
        """B_th of noise step n = th_step (RK4 steps since set_temperature), for time step dt
        (reading C-TH)."""
        sig = TH.sigma(self.alpha, self.temperature, self.gamma, self.Ms, self.vcell, dt)
        return TH.thermal_field(self.shape, self.mag, self.seed, self.th_step, sig)

    def W(self, m):
        """Overlap W = sum_i M_s,i m_i . B_rms(r_i)."""
        return float(np.sum(self.Ms * np.sum(m * self.brms, axis=-1) * self.mag))

    # ---------------------------------------------------------------- stepping (steps 4-6)
    def rhs(self, m, t):
        B = self.field(m, t)
        if self._bth is not None:                  # held for all stages of the step (C-TH)
            B = B + self._bth
        return torque(m, B, self.alpha, self.gamma)

    def step(self, dt):
        if self.temperature > 0.0:
            self.th_dt = dt
            self._bth = self.thermal(dt)
        self.m = rk4_step(self.rhs, self.m, self.mem.t, dt)
        self._bth = None
        self.th_step += 1
        W = self.W(self.m) if self.cavity_enabled else 0.0
        self.mem.update(W, dt)
        for b, mem, _, _ in self.extra:              # every mode advances on its own overlap
            Wk = float(np.sum(self.Ms * np.sum(self.m * b, axis=-1) * self.mag)) if np.any(b != 0) else 0.0
            mem.update(Wk, dt)

    def run(self, dt, steps):
        for _ in range(int(steps)):
            self.step(dt)
        return self.m

    # ---------------------------------------------------------------- Dormand-Prince (NEXT-1)
    def _advance_memory(self, dt):
        W = self.W(self.m) if self.cavity_enabled else 0.0
        self.mem.update(W, dt)
        for b, mem, _, _ in self.extra:
            Wk = float(np.sum(self.Ms * np.sum(self.m * b, axis=-1) * self.mag)) if np.any(b != 0) else 0.0
            mem.update(Wk, dt)

    def step_dp(self, dt):
        """One fixed Dormand-Prince step (reading C-DP), memory advanced with this dt (C3-C5).
        Returns the error estimate."""
        if self.temperature > 0.0:
            raise RuntimeError("the thermal field is defined for the fixed-step RK4 path only (C-TH)")
        self.m, err = dp45_step(self.rhs, self.m, self.mem.t, dt)
        self._advance_memory(dt)
        return err

    def run_adaptive(self, duration, dt0, tol, max_attempts=10**6):
        """Adaptive Dormand-Prince over `duration`: an attempt with err <= tol is accepted (state
        and memory advance by its dt, the step variable of eq:Sdiscrete/eq:Cdiscrete), a rejected
        one leaves both untouched; the next dt follows dp_controller, clipped to the end time.
        Returns (accepted, rejected, dt_next, accepted dts)."""
        if self.temperature > 0.0:
            raise RuntimeError("the thermal field is defined for the fixed-step RK4 path only (C-TH)")
        t_end = self.mem.t + duration
        dt, acc, rej, dts = dt0, 0, 0, []
        while t_end - self.mem.t > 1e-12 * max(duration, 1e-30) and acc + rej < max_attempts:
            h = min(dt, t_end - self.mem.t)
            m_new, err = dp45_step(self.rhs, self.m, self.mem.t, h)
            if err <= tol:
                self.m = m_new
                self._advance_memory(h)
                acc += 1
                dts.append(h)
            else:
                rej += 1
            dt = dp_controller(h, err, tol)
        return acc, rej, dt, dts

    # ---------------------------------------------------------------- relax (step 7)
    def max_torque(self, m=None):
        m = self.m if m is None else m
        B = self.field(m, self.mem.t, ALL & ~(CAVITY | EXCITATION))
        return float(np.max(np.linalg.norm(np.cross(m, B), axis=-1)))

    def relax(self, dt, tol, max_steps, check_every=RELAX_CHECK_EVERY):
        """RK4 on -gamma m x (m x B') with cavity and excitation off and t frozen; every
        ``check_every`` steps stop if max_i |m_i x B'_i| < tol; then reset memory (C15)."""
        t0 = self.mem.t
        terms = ALL & ~(CAVITY | EXCITATION)

        def f(m, t):
            return relax_torque(m, self.field(m, t0, terms), self.gamma)

        steps = 0
        while steps < max_steps:
            k = min(check_every, max_steps - steps)
            for _ in range(k):
                self.m = rk4_step(f, self.m, t0, dt)
            steps += k
            if self.max_torque() < tol:
                break
        self.reset_memory()
        return steps

    def reset_memory(self):
        self.mem.reset()
        for _, mem, _, _ in self.extra:
            mem.reset()

    # ---------------------------------------------------------------- diagnostics (pins)
    def energy(self, m=None):
        """E = Vc sum_i [-M_s m.B_ext - 1/2 M_s m.(B_exch + B_demag) + e_anis]
        - Vc W Gamma + hbar w_c |alpha|^2  (P:214 with S = -M_s Vc m / gamma; reading C22)."""
        m = self.m if m is None else m
        Ms = self.Ms * self.mag
        e = -Ms * np.sum(m * self.bext, -1)
        e = e - 0.5 * Ms * np.sum(m * F.exchange(m, self.mag, self.cell, self.Aex, self.Ms), -1)
        if self.demag_mode != "off":
            e = e - 0.5 * Ms * np.sum(m * self.demag(m), -1)
        a = self.aniso
        if a.get("ku1", 0.0):
            u = np.asarray(a["u"], float)
            u = u / np.linalg.norm(u)
            e = e - a["ku1"] * (m @ u) ** 2 * self.mag
        if a.get("kc1", 0.0):
            c1 = np.asarray(a["c1"], float); c1 /= np.linalg.norm(c1)
            c2 = np.asarray(a["c2"], float); c2 /= np.linalg.norm(c2)
            c3 = np.cross(c1, c2)
            m1, m2, m3 = m @ c1, m @ c2, m @ c3
            e = e + a["kc1"] * (m1**2 * m2**2 + m2**2 * m3**2 + m3**2 * m1**2) * self.mag
        E = self.vcell * float(np.sum(e))
        if self.cavity_enabled:
            al = self.mem.alpha()
            E += -self.vcell * self.W(m) * 2 * al.real + self.mem.hbar * self.mem.omega_c * abs(al) ** 2
        return E

    def mean_m(self):
        return (self.m * self.mag[..., None]).sum(axis=(0, 1, 2)) / self.mag.sum()
