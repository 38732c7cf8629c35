"""Multimode cavity on the GPU (reading C-MM) against the oracle's
multimode Simulation (pinned in test_oracle_multimode.py): fields, 100-step parity, the
degenerate bright-mode equivalence on the GPU, API validation and the single-mode fallback."""
import math

import numpy as np
import pytest

from helpers import oracle_from, magmask, rel_l2
from synth import small_config
from synth.configs import two_wire_map

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2410_00966_b200 as mcq  # noqa: E402


def _two_mode_cfg():
    cfg = small_config("sphere", (16, 12, 8), seed=9, state="phys")
    dark, _, _ = two_wire_map(cfg.grid, cfg.cell, cfg.Ms, cfg.mask, 3e8, "dark")
    extra = {"brms_map": dark, "f_c": 15.1e9, "kappa": 2 * math.pi * 5e6, "x0": 0.05, "p0": -0.02,
             "exc_amp": 3.0, "exc_omega": 2 * math.pi * 20e9}
    return cfg, extra


def _gpu(cfg, extra):
    s = mcq.Solver.from_config(cfg, set_state=False)
    mcq.mcq_set_modes(s.ctx, 2)
    mcq.mcq_set_brms_mode(s.ctx, 1, extra["brms_map"])
    mcq.mcq_set_cavity_mode(s.ctx, 1, extra["f_c"], extra["kappa"], extra["x0"], extra["p0"])
    mcq.mcq_set_excitation_mode(s.ctx, 1, extra["exc_amp"], extra["exc_omega"])
    s.set_m(cfg.m0)
    return s


def _oracle(cfg, extra):
    ref = oracle_from(cfg)
    from oracle import sim as S
    return S.Simulation(cfg.grid, cfg.cell, cfg.Ms, cfg.Aex, cfg.alpha, cfg.m0, mask=cfg.mask, bext=cfg.bext,
                        brms_map=cfg.brms_map, brms_uniform=cfg.brms_uniform, f_c=cfg.f_c, kappa=cfg.kappa,
                        x0=cfg.x0, p0=cfg.p0, exc_amp=cfg.exc_amp, exc_omega=cfg.exc_omega, aniso=cfg.aniso,
                        demag=ref.demag_mode, modes=[extra])


def test_two_mode_field_and_100_steps_parity():
    cfg, extra = _two_mode_cfg()
    s = _gpu(cfg, extra)
    ref = _oracle(cfg, extra)
    mag = magmask(cfg)
    for bit in (16, 32, 63):                         # cavity, excitation, total
        b = s.field(bit)[mag]
        r = ref.field(ref.m, 0.0, bit).reshape(-1, 3)[mag]
        assert rel_l2(b, r) < 1e-5, bit
    s.run(cfg.dt, 100)
    ref.run(cfg.dt, 100)
    assert rel_l2(s.m()[mag], ref.m.reshape(-1, 3)[mag]) < 1e-4
    for k, mem in ((0, ref.mem), (1, ref.extra[0][1])):
        cav = mcq.mcq_get_cavity_mode(s.ctx, k)
        a = mem.alpha()
        assert cav["step"] == 100 and cav["t"] == pytest.approx(mem.t, rel=1e-14)
        assert abs(complex(cav["re_alpha"], cav["im_alpha"]) - a) <= 1e-4 * max(abs(a), 1e-12), k
        assert cav["W"] == pytest.approx(mem.W, rel=1e-4, abs=1e-9 * abs(mem.W) + 1e-30), k
        assert cav["S"] == pytest.approx(mem.S, rel=1e-3, abs=1e-6 * abs(mem.S) + 1e-30), k
    s.close()


def test_degenerate_modes_equal_one_bright_mode_on_gpu():
    cfg = small_config("film", (16, 16, 1), seed=4, state="phys")
    cfg.brms_uniform = (2e-4, 0.0, 0.0)
    cfg.kappa = 2 * math.pi * 50e6
    cfg.exc_amp = 0.0
    cfg.x0 = cfg.p0 = 0.0
    one = mcq.Solver.from_config(cfg)
    two = mcq.Solver.from_config(cfg, set_state=False)
    mcq.mcq_set_modes(two.ctx, 2)
    mcq.mcq_set_brms(two.ctx, None, (0.6 * 2e-4, 0.0, 0.0))
    mcq.mcq_set_brms_mode(two.ctx, 1, None, (0.8 * 2e-4, 0.0, 0.0))
    mcq.mcq_set_cavity_mode(two.ctx, 1, cfg.f_c, cfg.kappa)
    two.set_m(cfg.m0)
    one.run(cfg.dt, 200)
    two.run(cfg.dt, 200)
    assert rel_l2(two.m(), one.m()) < 1e-5
    a = complex(one.cavity()["re_alpha"], one.cavity()["im_alpha"])
    a0 = mcq.mcq_get_cavity_mode(two.ctx, 0)
    a1 = mcq.mcq_get_cavity_mode(two.ctx, 1)
    assert abs(complex(a0["re_alpha"], a0["im_alpha"]) - 0.6 * a) < 1e-4 * abs(a)
    assert abs(complex(a1["re_alpha"], a1["im_alpha"]) - 0.8 * a) < 1e-4 * abs(a)
    one.close()
    two.close()


def test_mode_api_validation_and_single_mode_fallback():
    cfg = small_config("sphere", (16, 12, 8), seed=8, state="phys")
    a = mcq.Solver.from_config(cfg)
    for bad in (0, mcq.MAX_MODES + 1):
        with pytest.raises(mcq.MCQError) as e:
            mcq.mcq_set_modes(a.ctx, bad)
        assert e.value.code == -1
    with pytest.raises(mcq.MCQError):
        mcq.mcq_set_cavity_mode(a.ctx, 1, 1e9, 0.0)          # only mode 0 exists
    mcq.mcq_set_modes(a.ctx, 3)
    mcq.mcq_set_brms_mode(a.ctx, 2, None, (1e-4, 0.0, 0.0))
    mcq.mcq_set_modes(a.ctx, 1)                            # drops modes 1, 2 back to defaults
    a.set_m(cfg.m0)
    a.run(cfg.dt, 20)
    b = mcq.Solver.from_config(cfg)
    b.run(cfg.dt, 20)
    assert np.array_equal(a.m(), b.m())
    assert a.cavity()["re_alpha"] == b.cavity()["re_alpha"]
    a.close()
    b.close()


def test_brms_from_ovf_file_equals_direct_map(tmp_path):
    """the B_rms map handed over as an OVF 2.0 file (binary 4) drives the same run bit
    for bit; a file on another grid is refused (no resampling)."""
    cfg = small_config("sphere", (16, 12, 8), seed=5, state="phys")
    p = tmp_path / "brmsfile.ovf"
    mcq.mcq_ovf_write(p, cfg.brms_map, cfg.grid, cfg.cell, "binary4")
    a = mcq.Solver.from_config(cfg)
    b = mcq.Solver.from_config(cfg, set_state=False)
    mcq.mcq_set_brms(b.ctx, None, (0.0, 0.0, 0.0))
    b.set_brms_ovf(p)
    b.set_m(cfg.m0)
    a.run(cfg.dt, 20)
    b.run(cfg.dt, 20)
    assert np.array_equal(a.m(), b.m()) and a.cavity()["re_alpha"] == b.cavity()["re_alpha"]
    q = tmp_path / "other.ovf"
    mcq.mcq_ovf_write(q, np.zeros((8 * 8 * 8, 3), np.float32), (8, 8, 8), cfg.cell, "binary4")
    with pytest.raises(ValueError):
        b.set_brms_ovf(q)
    a.close()
    b.close()
