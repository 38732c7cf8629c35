"""Edge cases of the grid (include/mcq.h mcq_create: 2 <= nx, ny <= 512, 1 <= nz <= 512) against
the oracle: the smallest mesh, odd sizes, each axis at its maximum with the others minimal (the
largest row FFTs: Lx, Ly or Lz = 1024), and a single magnetic cell in vacuum.  Field terms
within 1e-5 and 20 steps within 1e-4, as in test_gpu_parity.py."""
import numpy as np
import pytest

from helpers import oracle_from, magmask, rel_l2, TERMS
from synth import small_config

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2410_00966_b200 as mcq  # noqa: E402

GRIDS = [(2, 2, 1), (3, 5, 2), (2, 3, 7), (512, 2, 1), (2, 512, 1), (2, 2, 512), (511, 3, 2)]


def _check(cfg, steps=20):
    s = mcq.Solver.from_config(cfg)
    ref = oracle_from(cfg)
    ref.m = s.m().astype(np.float64).reshape(ref.m.shape)
    mag = magmask(cfg)
    for name, bit in list(TERMS.items()) + [("total", 63)]:
        b = s.field(bit)[mag]
        r = ref.field(ref.m, 0.0, bit).reshape(-1, 3)[mag]
        if np.all(r == 0):
            assert np.all(b == 0), name
            continue
        assert rel_l2(b, r) < 1e-5, (name, rel_l2(b, r))
    s.run(cfg.dt, steps)
    ref.run(cfg.dt, steps)
    assert rel_l2(s.m()[mag], ref.m.reshape(-1, 3)[mag]) < 1e-4
    a = ref.mem.alpha()
    cav = s.cavity()
    assert abs(complex(cav["re_alpha"], cav["im_alpha"]) - a) <= 1e-4 * max(abs(a), 1e-12)
    s.close()


@pytest.mark.parametrize("grid", GRIDS)
def test_extreme_grids(grid):
    _check(small_config("film", grid, seed=5, state="phys"))


def test_single_magnetic_cell_in_vacuum():
    cfg = small_config("film", (8, 6, 3), seed=6, state="phys")
    mask = np.zeros(cfg.n, np.uint8)
    mask[(1 * 6 + 2) * 8 + 5] = 1                     # cell (x=5, y=2, z=1)
    cfg.mask = mask
    cfg.m0 = (cfg.m0 * mask[:, None]).astype(np.float32)
    _check(cfg)


def test_geometry_growing_the_magnet_needs_a_fresh_state():
    """a geometry change that makes former vacuum cells (m = 0) magnetic is applied,
    reports ESTATE and blocks the run until mcq_set_m; shrinking the magnet keeps the state."""
    cfg = small_config("sphere", (12, 10, 6), seed=7, state="phys")
    s = mcq.Solver.from_config(cfg)
    mask = cfg.mask.copy()
    smaller = mask.copy()
    smaller[np.flatnonzero(mask)[:5]] = 0
    mcq.mcq_set_geometry(s.ctx, smaller)           # shrink: fine, vacuum zeroed
    assert np.all(s.m()[~smaller.astype(bool)] == 0)
    s.run(cfg.dt, 2)
    with pytest.raises(mcq.MCQError) as e:         # grow back: the 5 cells have no m
        mcq.mcq_set_geometry(s.ctx, mask)
    assert e.value.code == -2
    with pytest.raises(mcq.MCQError) as e:
        s.run(cfg.dt, 1)
    assert e.value.code == -2
    s.set_m(cfg.m0)
    s.run(cfg.dt, 1)
    with pytest.raises(mcq.MCQError) as e:         # removing the mask: every vacuum cell has m = 0
        mcq.mcq_set_geometry(s.ctx, None)
    assert e.value.code == -2
    s.close()


def test_rescaled_accumulators_stay_finite():
    """S, C grow as e^{kappa t}; the rescaled pair e^{-kappa t}(S, C) is finite for any
    t and equals the literal pair times e^{-kappa t} while that is representable."""
    cfg = small_config("film", (8, 6, 1), seed=8, state="phys")
    cfg.kappa = 2e11                                # kappa t = 700 after 3.5 ns
    s = mcq.Solver.from_config(cfg)
    ref = oracle_from(cfg)
    s.run(1e-12, 200)
    ref.run(1e-12, 200)
    cav = s.cavity()
    k = np.exp(-cfg.kappa * cav["t"])
    assert np.isfinite(cav["S"]) and abs(cav["S_resc"] - ref.mem.S * k) <= 1e-4 * abs(ref.mem.S * k) + 1e-30
    assert abs(cav["C_resc"] - ref.mem.C * k) <= 1e-4 * abs(ref.mem.C * k) + 1e-30
    s.run(1e-12, 4000)                              # kappa t = 840: S, C overflow
    cav = s.cavity()
    assert not np.isfinite(cav["S"]) or not np.isfinite(cav["C"]) or abs(cav["S"]) > 1e300
    assert np.isfinite(cav["S_resc"]) and np.isfinite(cav["C_resc"])
    s.close()
