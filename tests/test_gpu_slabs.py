"""z-slab decomposition in loopback mode: all slabs of the decomposed schedule —
one-plane halo exchanges, the z-slab <-> kx-slab all-to-all around K-Z, W partials in global z
order — run inside one context on one GPU with device copies standing in for NCCL (the
profiling guide forbids emulating ranks as processes on one GPU).  The decomposition changes
no arithmetic, so every output must be BITWISE equal to the undecomposed run, and (through
that) within the oracle tolerances of test_gpu_parity.py.  Also checks the oracle directly for
one decomposed case, the launch-count claim and argument validation."""
import numpy as np
import pytest

from helpers import oracle_from, magmask, rel_l2
from synth import small_config

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2410_00966_b200 as mcq  # noqa: E402

UNI = {"ku1": 2e4, "u": (0.2, 0.3, 1.0)}
CUBIC = {"kc1": -610.0, "c1": (1, 1, 0), "c2": (-1, 1, 0)}

# (kind, grid, aniso, worlds): several kx slabs incl. empty ones (NKX small vs NS * 16),
# one-plane slabs (both halos from different ranks), non-power-of-two world, masks and maps
CASES = [
    ("sphere", (16, 12, 8), None, (2, 4, 8)),
    ("disc", (48, 40, 4), UNI, (2, 4)),
    ("sphere", (30, 18, 6), CUBIC, (2, 3, 6)),
    ("disc", (32, 32, 2), None, (2,)),
    ("film", (64, 24, 16), None, (4, 16)),
    ("film", (2, 8, 4), None, (2, 4)),          # NKX = 3 < world: empty kx slabs
    ("disc", (40, 72, 6), None, (3, 6)),        # NKX = 65 split 16/16/33 and 8-column blocks
]


def _loop(cfg, world):
    return mcq.Solver.from_config(cfg, dist={"rank": -1, "world": world})


def _cav_equal(a, b):
    ca, cb = a.cavity(), b.cavity()
    for k in ("t", "re_alpha", "im_alpha", "W", "step"):
        assert ca[k] == cb[k], (k, ca[k], cb[k])


@pytest.mark.parametrize("kind,grid,aniso,worlds", CASES)
def test_loopback_slabs_bitwise_equal_single(kind, grid, aniso, worlds):
    cfg = small_config(kind, grid, seed=21, aniso=aniso, state="rand")
    ref = mcq.Solver.from_config(cfg)
    ref_m0 = ref.m().copy()
    fields = {bit: ref.field(bit).copy() for bit in (1, 2, 4, 8, 16, 32, 63)}
    ref.run(cfg.dt, 37)
    m_ref = ref.m().copy()
    for w in worlds:
        s = _loop(cfg, w)
        assert np.array_equal(s.m(), ref_m0), w      # set_m / get_m plane ranges of every slab
        for bit, f in fields.items():
            assert np.array_equal(s.field(bit), f), (w, bit)
        s.run(cfg.dt, 37)
        assert np.array_equal(s.m(), m_ref), w
        _cav_equal(s, ref)
        s.close()
    ref.close()


def test_loopback_slabs_oracle_parity():
    """Decomposed run vs the fp64 oracle directly (north_star: m within 1e-4 after 100 steps)."""
    cfg = small_config("sphere", (24, 20, 12), seed=3, aniso=CUBIC, state="phys")
    s = _loop(cfg, 4)
    ref = oracle_from(cfg)
    mag = magmask(cfg)
    s.run(cfg.dt, 100)
    ref.run(cfg.dt, 100)
    assert rel_l2(s.m()[mag], ref.m.reshape(-1, 3)[mag]) < 1e-4
    a = ref.mem.alpha()
    cav = s.cavity()
    assert abs(complex(cav["re_alpha"], cav["im_alpha"]) - a) <= 1e-4 * max(abs(a), 1e-12)
    s.close()


def test_loopback_relax_and_resume():
    cfg = small_config("disc", (32, 32, 4), seed=2, state="phys")
    a = mcq.Solver.from_config(cfg)
    b = _loop(cfg, 2)
    na = a.relax(0.2e-12, 2e-3, 3000)
    nb = b.relax(0.2e-12, 2e-3, 3000)
    assert na == nb
    assert np.array_equal(a.m(), b.m())
    # resume a decomposed run from a state saved by an undecomposed one
    a.run(cfg.dt, 10)
    m_mid, cav_mid = a.m().copy(), a.cavity()
    a.run(cfg.dt, 10)
    c = _loop(cfg, 4)
    c.set_m(m_mid)
    mcq.mcq_set_cavity_state(c.ctx, cav_mid)
    c.run(cfg.dt, 10)
    assert np.array_equal(a.m(), c.m())
    for s in (a, b, c):
        s.close()


def test_loopback_launch_count_and_layout():
    cfg = small_config("sphere", (16, 12, 8), seed=8, state="phys")
    one = mcq.Solver.from_config(cfg)
    s = _loop(cfg, 4)
    assert mcq.mcq_debug_layout(s.ctx) == mcq.mcq_debug_layout(one.ctx)   # global layout + partials
    n0 = mcq.mcq_kernel_launches(s.ctx)
    s.run(cfg.dt, 11)
    s.sync()
    assert mcq.mcq_kernel_launches(s.ctx) - n0 == 1 + 11 * (4 * 4 * (3 + 1) + 1)
    # overlapped schedule: K-Y and K-YI one launch per component (each component's transpose
    # runs on the side stream during the next one's pass)
    mcq.mcq_set_slab_overlap(s.ctx, 1)
    n0 = mcq.mcq_kernel_launches(s.ctx)
    s.run(cfg.dt, 11)
    s.sync()
    assert mcq.mcq_kernel_launches(s.ctx) - n0 == 1 + 11 * (4 * 4 * (3 + 1 + 3 + 1) + 1)
    s.close()
    one.close()


def test_slab_argument_validation():
    g, c = (16, 16, 6), (5e-9,) * 3
    with pytest.raises(mcq.MCQError) as e:
        mcq.mcq_create(g, c, 1e5, 1e-11, 0.01, dist={"rank": -1, "world": 4})   # 4 does not divide 6
    assert e.value.code == -1
    with pytest.raises(mcq.MCQError) as e:
        mcq.mcq_create(g, c, 1e5, 1e-11, 0.01, dist={"rank": 0, "world": 2})    # NCCL rank, no id
    assert e.value.code == -1
    with pytest.raises(mcq.MCQError) as e:
        mcq.mcq_create(g, c, 1e5, 1e-11, 0.01, dist={"rank": 2, "world": 2, "nccl_id": bytes(128)})
    assert e.value.code == -1


@pytest.mark.parametrize("grid,slabs", [((16, 12, 8), 4), ((16, 6, 100), 5)])
def test_overlapped_slab_schedule_is_bitwise_the_serial_one(grid, slabs):
    """The side-stream schedule (per-component y passes, transposes overlapped: the NCCL default)
    gives the same bits as one slab."""
    cfg = small_config("sphere", grid, seed=9, state="phys")
    one = mcq.Solver.from_config(cfg)
    lb = _loop(cfg, slabs)
    mcq.mcq_set_slab_overlap(lb.ctx, 1)
    one.run(cfg.dt, 13)
    lb.run(cfg.dt, 13)
    assert np.array_equal(one.m(), lb.m())
    assert one.cavity()["re_alpha"] == lb.cavity()["re_alpha"]
    one.close()
    lb.close()
