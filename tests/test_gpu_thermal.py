"""Thermal field on the GPU (reading C-TH) against the oracle's
(pinned in test_oracle_thermal.py).  Both sides implement the same counter-based stream
(SplitMix64 + Box-Muller) independently, so parity is element by element: the thermal field of
a step, 100 noisy steps, the slab decomposition, and the Langevin equilibrium of uncoupled
macrospins on the GPU path at scale."""
import math

import numpy as np
import pytest

from helpers import oracle_from, magmask, rel_l2
from synth import small_config

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2410_00966_b200 as mcq  # noqa: E402
from oracle import sim as S  # noqa: E402

T_K, SEED = 300.0, 0xC0FFEE


def _pair(cfg):
    s = mcq.Solver.from_config(cfg)
    mcq.mcq_set_temperature(s.ctx, T_K, SEED)
    ref = oracle_from(cfg)
    ref.set_temperature(T_K, SEED)
    return s, ref


@pytest.mark.parametrize("kind,grid", [("sphere", (16, 12, 8)), ("film", (40, 24, 1))])
def test_thermal_field_and_100_steps_parity(kind, grid):
    cfg = small_config(kind, grid, seed=21, state="phys")
    s, ref = _pair(cfg)
    mag = magmask(cfg)
    with pytest.raises(mcq.MCQError) as e:                 # its scale needs a run's dt
        s.field(mcq.TERM_THERM)
    assert e.value.code == -2
    s.run(cfg.dt, 3)
    ref.run(cfg.dt, 3)
    b = s.field(mcq.TERM_THERM)
    r = ref.field(ref.m, ref.mem.t, S.THERM).reshape(-1, 3)
    assert np.all(b[~mag] == 0)
    assert rel_l2(b[mag], r[mag]) < 1e-5
    assert rel_l2(s.field(mcq.TERM_ALL | mcq.TERM_THERM)[mag],
                  ref.field(ref.m, ref.mem.t, S.ALL | S.THERM).reshape(-1, 3)[mag]) < 1e-5
    s.run(cfg.dt, 97)
    ref.run(cfg.dt, 97)
    assert rel_l2(s.m()[mag], ref.m.reshape(-1, 3)[mag]) < 1e-4
    a = ref.mem.alpha()
    cav = s.cavity()
    assert abs(complex(cav["re_alpha"], cav["im_alpha"]) - a) <= 1e-4 * max(abs(a), 1e-12)
    s.close()


def test_temperature_api_zero_is_bitwise_off_and_slabs_match():
    cfg = small_config("sphere", (16, 12, 8), seed=22, state="phys")
    cold = mcq.Solver.from_config(cfg)
    zero = mcq.Solver.from_config(cfg)
    mcq.mcq_set_temperature(zero.ctx, 0.0, 5)
    cold.run(cfg.dt, 20)
    zero.run(cfg.dt, 20)
    assert np.array_equal(cold.m(), zero.m())
    hot = mcq.Solver.from_config(cfg)
    mcq.mcq_set_temperature(hot.ctx, T_K, SEED)
    loop = mcq.Solver.from_config(cfg, dist={"rank": -1, "world": 2})   # two z slabs, one process
    mcq.mcq_set_temperature(loop.ctx, T_K, SEED)
    hot.run(cfg.dt, 20)
    loop.run(cfg.dt, 20)
    assert np.array_equal(hot.m(), loop.m())                # global cell index: same draws
    assert not np.array_equal(hot.m(), cold.m())
    other = mcq.Solver.from_config(cfg)
    mcq.mcq_set_temperature(other.ctx, T_K, SEED + 1)
    other.run(cfg.dt, 20)
    assert not np.array_equal(hot.m(), other.m())
    for bad in (-1.0, math.nan, math.inf):
        with pytest.raises(mcq.MCQError):
            mcq.mcq_set_temperature(hot.ctx, bad, 0)
    with pytest.raises(mcq.MCQError) as e:                 # RK4 path only
        mcq.mcq_run_dp(hot.ctx, cfg.dt, 1)
    assert e.value.code == -2
    for sv in (cold, zero, hot, loop, other):
        sv.close()


def test_langevin_equilibrium_on_gpu():
    """1024 isolated cubic cells (every 4th cell of a 128 x 128 x 1 mesh: no exchange partner;
    a cube's self-demag is isotropic, the dipolar coupling at 4 cells is ~1e-3 of B) in 0.5 T
    along z at x = M_s V B / (k_B T) = 2 relax to <m_z> = coth 2 - 1/2 = 0.537."""
    grid, cell, Ms, alpha, B = (128, 128, 1), (5e-9,) * 3, 1.4e5, 1.0, 0.5
    V = cell[0] * cell[1] * cell[2]
    x = 2.0
    T = Ms * V * B / (1.380649e-23 * x)
    mask = np.zeros((128, 128), np.uint8)
    mask[::4, ::4] = 1
    mask = mask.reshape(-1)
    rng = np.random.default_rng(3)
    m0 = rng.normal(size=(mask.size, 3)).astype(np.float32)
    m0 /= np.linalg.norm(m0, axis=1, keepdims=True)
    m0 *= mask[:, None]
    s = mcq.Solver(grid, cell, Ms, 1e-11, alpha)
    mcq.mcq_set_geometry(s.ctx, mask)
    mcq.mcq_set_bext(s.ctx, (0.0, 0.0, B))
    mcq.mcq_set_temperature(s.ctx, T, 99)
    s.set_m(m0)
    dt = 1e-13
    s.run(dt, 2000)
    acc = []
    for _ in range(60):
        s.run(dt, 500)
        acc.append(s.m()[mask.astype(bool), 2].mean())
    langevin = 1.0 / math.tanh(x) - 1.0 / x
    assert abs(np.mean(acc) - langevin) < 0.02, (np.mean(acc), langevin)
    s.close()


def test_stored_draw_follows_temperature_and_dt_changes():
    """Stage 1 stores the step's draw and stages 2-4 reload it (12 B per cell): the stored draw
    must always be the current step's, across changes of T, seed and dt between runs and after
    a run with the thermal term off."""
    cfg = small_config("sphere", (16, 12, 8), seed=23, state="phys")
    s, ref = _pair(cfg)
    mag = magmask(cfg)
    plan = [(T_K, SEED, cfg.dt, 3), (100.0, SEED + 7, 0.5 * cfg.dt, 4), (0.0, SEED, cfg.dt, 2),
            (T_K, SEED, cfg.dt, 3)]
    for T, seed, dt, n in plan:
        mcq.mcq_set_temperature(s.ctx, T, seed)
        ref.set_temperature(T, seed)
        s.run(dt, n)
        ref.run(dt, n)
        assert rel_l2(s.m()[mag], ref.m.reshape(-1, 3)[mag]) < 1e-4
    s.close()


def test_noise_step_is_not_restarted_by_memory_resets():
    """the thermal stream is keyed on its own noise step (RK4 steps since
    mcq_set_temperature), not on the cavity step count, so mcq_reset_memory / relax / the cavity
    setters never make a later segment reuse an earlier segment's draws."""
    cfg = small_config("sphere", (16, 12, 8), seed=24, state="phys")
    s, ref = _pair(cfg)
    mag = magmask(cfg)
    s.run(cfg.dt, 3)
    ref.run(cfg.dt, 3)
    assert mcq.mcq_get_thermal_step(s.ctx) == 3 == ref.th_step
    before = s.field(mcq.TERM_THERM)
    mcq.mcq_reset_memory(s.ctx)                   # cavity step back to 0, noise step stays 3
    ref.reset_memory()
    after = s.field(mcq.TERM_THERM)
    assert np.array_equal(before, after)
    assert mcq.mcq_get_thermal_step(s.ctx) == 3
    s.run(cfg.dt, 2)
    ref.run(cfg.dt, 2)
    assert rel_l2(s.m()[mag], ref.m.reshape(-1, 3)[mag]) < 1e-4
    nxt = s.field(mcq.TERM_THERM)                 # noise step 5: a fresh draw
    assert rel_l2(nxt[mag], ref.field(ref.m, ref.mem.t, S.THERM).reshape(-1, 3)[mag]) < 1e-5
    assert not np.allclose(nxt[mag], before[mag])
    # checkpoint / resume of the noise step
    mcq.mcq_set_thermal_step(s.ctx, 40)
    ref.th_step = 40
    assert rel_l2(s.field(mcq.TERM_THERM)[mag], ref.field(ref.m, ref.mem.t, S.THERM).reshape(-1, 3)[mag]) < 1e-5
    with pytest.raises(mcq.MCQError):
        mcq.mcq_set_thermal_step(s.ctx, -1)
    s.close()
