"""Dormand-Prince 5(4) on the GPU (reading C-DP) against the oracle's
integrator (pinned in test_oracle_dp45.py): fixed-step parity with the cavity on, the adaptive
driver replayed step for step in the oracle (the accepted step list comes from the device
trace), accuracy improving with the tolerance, and the decomposed (loopback) run bit for bit."""
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


def _cmp_cav(s, ref, tol=1e-4):
    cav = s.cavity()
    a = ref.mem.alpha()
    assert cav["t"] == pytest.approx(ref.mem.t, rel=1e-12)
    assert abs(complex(cav["re_alpha"], cav["im_alpha"]) - a) <= tol * max(abs(a), 1e-12)


def test_fixed_step_dp_parity():
    cfg = small_config("sphere", (16, 12, 8), seed=3, state="phys")
    s = mcq.Solver.from_config(cfg)
    ref = oracle_from(cfg)
    mag = magmask(cfg)
    mcq.mcq_run_dp(s.ctx, cfg.dt, 30)
    for _ in range(30):
        ref.step_dp(cfg.dt)
    assert rel_l2(s.m()[mag], ref.m.reshape(-1, 3)[mag]) < 1e-4
    assert np.allclose(np.linalg.norm(s.m()[mag], axis=1), 1.0, atol=1e-6)
    _cmp_cav(s, ref)
    assert s.cavity()["step"] == 30
    s.close()


def test_adaptive_replayed_in_oracle():
    cfg = small_config("sphere", (12, 10, 6), seed=2, state="rand")
    s = mcq.Solver.from_config(cfg)
    s.trace(10000, every=1)
    acc, rej, dt_next = mcq.mcq_run_adaptive(s.ctx, 6e-12, 0.01e-12, 1e-5)
    assert acc > 6 and dt_next > 0
    tr = s.trace()
    assert tr.shape[0] == acc and tr[-1, 0] == pytest.approx(6e-12, rel=1e-12)
    dts = np.diff(np.concatenate([[0.0], tr[:, 0]]))
    assert dts.max() > 1.5 * dts.min()                      # the controller did vary the step
    ref = oracle_from(cfg)
    for h in dts:
        ref.step_dp(h)
    mag = magmask(cfg)
    assert rel_l2(s.m()[mag], ref.m.reshape(-1, 3)[mag]) < 1e-4
    _cmp_cav(s, ref)
    s.close()


def test_adaptive_accuracy_improves_with_tolerance():
    cfg = small_config("film", (16, 16, 1), seed=6, state="phys")
    T = 60e-12
    ref = mcq.Solver.from_config(cfg)
    ref.run(T / 6000, 6000)                                 # RK4 at 0.01 ps: the reference
    errs = []
    for tol in (1e-4, 1e-6):
        s = mcq.Solver.from_config(cfg)
        acc, rej, _ = mcq.mcq_run_adaptive(s.ctx, T, 0.1e-12, tol)
        assert s.cavity()["t"] == pytest.approx(T, rel=1e-12)
        errs.append(np.abs(s.m() - ref.m()).max())
        s.close()
    assert errs[1] < errs[0] and errs[1] < 1e-4, errs
    ref.close()


def test_dp_loopback_slabs_bitwise():
    cfg = small_config("sphere", (16, 12, 8), seed=21, state="rand")
    one = mcq.Solver.from_config(cfg)
    two = mcq.Solver.from_config(cfg, dist={"rank": -1, "world": 2})
    mcq.mcq_run_dp(one.ctx, cfg.dt, 12)
    mcq.mcq_run_dp(two.ctx, cfg.dt, 12)
    assert np.array_equal(one.m(), two.m())
    assert one.cavity()["re_alpha"] == two.cavity()["re_alpha"]
    r1 = mcq.mcq_run_adaptive(one.ctx, 5e-12, 0.05e-12, 1e-5)
    r2 = mcq.mcq_run_adaptive(two.ctx, 5e-12, 0.05e-12, 1e-5)
    assert r1 == r2 and np.array_equal(one.m(), two.m())
    one.close()
    two.close()
