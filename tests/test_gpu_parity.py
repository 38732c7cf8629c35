"""GPU-vs-oracle parity through the C ABI (BJ north_star acceptance):
  fp32 field within 1e-5 relative L2 per term and in total; m after 100 fixed steps within 1e-4;
  integer layout maps bit-exact; cavity state; relax; edge cases."""
import math

import numpy as np
import pytest

from helpers import oracle_from, magmask, rel_l2, TERMS
from synth import small_config, make_config
from oracle import tensor as T
from oracle import fields as F
from oracle.constants import MU0

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2410_00966_b200 as mcq  # noqa: E402

CUBIC = {"kc1": -610.0, "c1": (1, 1, 0), "c2": (-1, 1, 0)}
UNI = {"ku1": 2e4, "u": (0.2, 0.3, 1.0)}

# several tiles and ragged tails: NKX not a multiple of the column tile, ny not a multiple of
# the row tile, non-power-of-two sizes (padding beyond 2n), 2D and 3D, masks, maps, anisotropy
CASES = [
    ("film", (40, 24, 1), None),
    ("film", (64, 64, 1), UNI),
    ("sphere", (24, 20, 12), None),
    ("sphere", (16, 16, 16), CUBIC),
    ("disc", (48, 40, 3), UNI),
    ("sphere", (30, 18, 5), None),
    ("disc", (40, 72, 3), UNI),      # NKX = 65 = 4 full 16-column tiles + a 1-column tile
]


def _solver(cfg):
    return mcq.Solver.from_config(cfg)


@pytest.mark.parametrize("kind,grid,aniso", CASES)
def test_field_terms_parity(kind, grid, aniso):
    cfg = small_config(kind, grid, seed=11, aniso=aniso, state="rand")
    s = _solver(cfg)
    ref = oracle_from(cfg)
    ref.m = s.m().astype(np.float64).reshape(ref.m.shape)   # the exact fp32 state the GPU holds
    mag = magmask(cfg)
    for name, bit in list(TERMS.items()) + [("total", 63)]:
        if name == "anis" and not aniso:
            continue
        b = s.field(bit)[mag]
        r = ref.field(ref.m, 0.0, bit).reshape(-1, 3)[mag]
        err = rel_l2(b, r)
        assert err < 1e-5, (name, err)
    s.close()


def test_tensor_octant_matches_oracle():
    cfg = small_config("sphere", (24, 20, 12), seed=1)
    s = _solver(cfg)
    L = mcq.mcq_debug_layout(s.ctx)
    gpu = mcq.mcq_debug_tensor_octant(s.ctx)
    nx, ny, nz = cfg.grid
    ref = T.tensor_octant((nx, ny, nz), cfg.cell)
    assert gpu.shape == (6, L["Lz"] // 2 + 1, L["Ly"] // 2 + 1, L["Lx"] // 2 + 1)
    assert np.abs(gpu[:, :nz, :ny, :nx] - ref).max() < 1e-9
    assert np.all(gpu[:, nz:] == 0) and np.all(gpu[:, :, ny:] == 0) and np.all(gpu[..., nx:] == 0)
    s.close()


def test_khat_matches_direct_dft_of_padded_tensor():
    cfg = small_config("sphere", (16, 8, 4), seed=1)
    s = _solver(cfg)
    kh = mcq.mcq_debug_khat(s.ctx)
    P = T.padded_tensor(cfg.grid, cfg.cell)             # oracle's own padding, 2n (== GPU for pow2 n)
    _, Lz, Ly, Lx = P.shape
    Fx = np.exp(-2j * np.pi * np.outer(np.arange(Lx), np.arange(Lx)) / Lx)
    Fy = np.exp(-2j * np.pi * np.outer(np.arange(Ly), np.arange(Ly)) / Ly)
    Fz = np.exp(-2j * np.pi * np.outer(np.arange(Lz), np.arange(Lz)) / Lz)
    Nh = np.einsum("ax,by,cz,nzyx->ncba", Fx, Fy, Fz, P)
    assert np.abs(Nh.imag).max() < 1e-9 * np.abs(Nh.real).max()
    expect = -MU0 * cfg.Ms / (Lx * Ly * Lz) * Nh.real[:, :Lz // 2 + 1, :Ly // 2 + 1, :Lx // 2 + 1]
    assert kh.shape == expect.shape                     # (6, kz, ky, kx) as the ABI states
    assert np.abs(kh - expect).max() <= 2e-7 * np.abs(expect).max()
    s.close()


def test_layout_maps_bit_exact():
    """Padded lengths and spectral row layout are the plain definitions."""
    for grid in [(40, 24, 1), (24, 20, 12), (128, 128, 128), (512, 512, 8), (30, 18, 5)]:
        s = mcq.Solver(grid, (5e-9,) * 3, 1e5, 1e-11, 0.01)
        L = mcq.mcq_debug_layout(s.ctx)

        def pad(n):
            return 1 if n == 1 else 1 << int(math.ceil(math.log2(2 * n)))

        assert (L["Lx"], L["Ly"], L["Lz"]) == tuple(pad(n) for n in grid)
        assert L["NKX"] == L["Lx"] // 2 + 1 and L["P"] == (L["NKX"] + 15) // 16 * 16
        s.close()


def test_unaligned_rows_fallback_path():
    """nx not a multiple of 4: the update kernel stages rows with plain loads instead of TMA bulk
    copies (16-byte alignment); same results."""
    cfg = small_config("sphere", (30, 18, 5), seed=12, state="rand")
    s = _solver(cfg)
    ref = oracle_from(cfg)
    ref.m = s.m().astype(np.float64).reshape(ref.m.shape)
    mag = magmask(cfg)
    assert rel_l2(s.field(63)[mag], ref.field(ref.m, 0.0).reshape(-1, 3)[mag]) < 1e-5
    s.close()


def test_set_get_m_roundtrip_index_map():
    grid = (24, 20, 12)
    n = int(np.prod(grid))
    s = mcq.Solver(grid, (5e-9,) * 3, 1e5, 1e-11, 0.01)
    rng = np.random.default_rng(0)
    axes = np.eye(3, dtype=np.float32)[rng.integers(0, 3, n)] * rng.choice([-1, 1], n)[:, None]
    s.set_m(axes)
    assert np.array_equal(s.m(), axes.astype(np.float32))
    s.close()


@pytest.mark.parametrize("kind,grid,aniso", [("film", (40, 24, 1), None), ("sphere", (24, 20, 12), CUBIC),
                                             ("disc", (48, 40, 3), UNI)])
def test_100_steps_parity(kind, grid, aniso):
    cfg = small_config(kind, grid, seed=3, aniso=aniso, state="phys")
    s = _solver(cfg)
    ref = oracle_from(cfg)
    mag = magmask(cfg)
    s.run(cfg.dt, 100)
    ref.run(cfg.dt, 100)
    m = s.m()[mag]
    mr = ref.m.reshape(-1, 3)[mag]
    assert rel_l2(m, mr) < 1e-4
    assert np.allclose(np.linalg.norm(s.m()[mag], axis=1), 1.0, atol=1e-6)
    cav = s.cavity()
    a = ref.mem.alpha()
    assert cav["step"] == 100 and cav["t"] == pytest.approx(ref.mem.t, rel=1e-14)
    assert abs(complex(cav["re_alpha"], cav["im_alpha"]) - a) <= 1e-4 * max(abs(a), 1e-12)
    assert cav["W"] == pytest.approx(ref.mem.W, rel=1e-4, abs=1e-9 * abs(ref.mem.W) + 1e-30)
    s.close()


def test_strong_coupling_cavity_parity():
    """Uniform B_rms strong enough that the cavity feedback visibly changes m (Dicke-like)."""
    cfg = small_config("film", (16, 16, 1), seed=4, state="phys")
    cfg.brms_uniform = (2e-4, 0.0, 0.0)
    cfg.kappa = 2 * math.pi * 50e6
    cfg.exc_amp = 0.0
    s = _solver(cfg)
    ref = oracle_from(cfg)
    s.run(cfg.dt, 200)
    ref.run(cfg.dt, 200)
    assert rel_l2(s.m(), ref.m.reshape(-1, 3)) < 1e-4
    cav = s.cavity()
    a = ref.mem.alpha()
    assert abs(complex(cav["re_alpha"], cav["im_alpha"]) - a) <= 1e-4 * abs(a)
    # literal accumulators reconstructed from alpha equal the oracle's S_n, C_n
    assert cav["S"] == pytest.approx(ref.mem.S, rel=1e-4)
    assert cav["C"] == pytest.approx(ref.mem.C, rel=1e-4)
    s.close()


def test_relax_parity_fixed_steps():
    cfg = small_config("disc", (32, 32, 2), seed=2, state="phys")
    s = _solver(cfg)
    ref = oracle_from(cfg)
    n = s.relax(0.05e-12, 0.0, 100)
    nr = ref.relax(0.05e-12, 0.0, 100)
    assert n == nr == 100
    mag = magmask(cfg)
    assert rel_l2(s.m()[mag], ref.m.reshape(-1, 3)[mag]) < 1e-4
    assert s.cavity()["t"] == 0.0 and s.cavity()["step"] == 0


def test_relax_reaches_tolerance():
    cfg = small_config("film", (32, 16, 1), seed=2, state="phys")
    s = _solver(cfg)
    n = s.relax(0.2e-12, 1e-3, 20000)
    assert n < 20000 and n % 50 == 0
    ref = oracle_from(cfg)
    ref.m = s.m().astype(np.float64).reshape(ref.m.shape)
    assert ref.max_torque() < 1.05e-3
    s.close()


def test_zero_brms_is_cavity_off_and_status():
    cfg = small_config("film", (16, 16, 1), seed=6, state="phys")
    cfg.x0 = cfg.p0 = 0.0
    cfg.exc_amp = 0.0
    a = _solver(cfg)
    assert mcq.mcq_cavity_status(a.ctx) == 1
    cfg.brms_uniform = (0.0, 0.0, 0.0)
    b = _solver(cfg)
    assert mcq.mcq_cavity_status(b.ctx) == 0
    b.run(cfg.dt, 30)
    c = mcq.Solver(cfg.grid, cfg.cell, cfg.Ms, cfg.Aex, cfg.alpha)
    mcq.mcq_set_bext(c.ctx, cfg.bext)
    c.set_m(cfg.m0)
    c.run(cfg.dt, 30)
    assert np.array_equal(b.m(), c.m())


def test_resume_from_saved_state_is_bit_exact():
    cfg = small_config("sphere", (16, 12, 8), seed=8, state="phys")
    a = _solver(cfg)
    a.run(cfg.dt, 20)
    b = _solver(cfg)
    b.run(cfg.dt, 10)
    m_mid, cav_mid = b.m().copy(), b.cavity()
    c = _solver(cfg)
    c.set_m(m_mid)
    mcq.mcq_set_cavity_state(c.ctx, cav_mid)
    c.run(cfg.dt, 10)
    assert np.array_equal(a.m(), c.m())
    assert a.cavity()["re_alpha"] == c.cavity()["re_alpha"]


def test_error_paths():
    s = mcq.Solver((8, 8, 2), (5e-9,) * 3, 1e5, 1e-11, 0.01)
    with pytest.raises(mcq.MCQError) as e:
        s.run(1e-12, 1)
    assert e.value.code == -2                     # ESTATE: run before set_m
    m = np.zeros((128, 3), np.float32)
    m[:, 2] = 1
    m[5] = 0
    with pytest.raises(mcq.MCQError) as e:
        s.set_m(m)
    assert e.value.code == -1                     # EINVAL: zero vector in a magnetic cell
    m[5] = (1, 0, 0)
    s.set_m(m)
    with pytest.raises(mcq.MCQError):
        s.run(-1e-12, 1)
    with pytest.raises(mcq.MCQError):
        mcq.mcq_set_cavity(s.ctx, -1.0, 0.0)
    mask = np.ones(128, np.uint8)
    mask[:10] = 0
    mcq.mcq_set_geometry(s.ctx, mask)
    assert np.all(s.m()[:10] == 0)
    s.close()


def test_launch_count_claim():
    cfg = small_config("sphere", (16, 12, 8), seed=8, state="phys")
    s = _solver(cfg)
    n0 = mcq.mcq_kernel_launches(s.ctx)
    s.run(cfg.dt, 11)
    s.sync()
    assert mcq.mcq_kernel_launches(s.ctx) - n0 == 1 + 11 * (4 * (3 + 1) + 1)
    s.close()


# ---------------------------------------------------------------- full-size configs (bench launch)

@pytest.mark.parametrize("k", [1, 3])
def test_full_size_sampled_field_parity(k):
    """BJ configs at full size in the bench's launch configuration.  Demag (the size-dependent
    FFT path) at sampled magnetic cells against the brute-force sum at those cells; every local
    term on the whole grid; the total at the samples relative to the scale of its terms (the
    vortex total is ~1e-3 of its demag/exchange parts, so fp32 terms each good to 1e-5 cannot
    give the cancelled total to 1e-5 of itself)."""
    cfg = make_config(k)
    s = _solver(cfg)
    nx, ny, nz = cfg.grid
    ref = oracle_from(cfg, demag="off")
    ref.m = s.m().astype(np.float64).reshape(ref.m.shape)   # the exact fp32 state the GPU holds
    mag = magmask(cfg)
    oc = T.tensor_octant((nx, ny, nz), cfg.cell)
    rng = np.random.default_rng(k)
    bd = s.field(TERMS["demag"])
    idx = np.concatenate([rng.choice(np.nonzero(mag)[0], 8, replace=False),
                          [int(np.argmax(np.linalg.norm(bd, axis=1) * mag))]])
    pts = [(i % nx, (i // nx) % ny, i // (nx * ny)) for i in idx]
    dem = F.demag_at(ref.m, ref.mag, cfg.cell, cfg.Ms, pts, oc)
    # relative L2 over the grid, estimated from the samples: rms sample error / rms grid field
    rms_grid = np.linalg.norm(bd[mag]) / np.sqrt(mag.sum())
    rms_err = np.linalg.norm(bd[idx] - dem) / np.sqrt(len(idx))
    assert rms_err / rms_grid < 1e-5, rms_err / rms_grid
    local_bits = 63 & ~TERMS["demag"]
    for name, bit in TERMS.items():
        if name == "demag" or (name == "anis" and not cfg.aniso):
            continue
        r = ref.field(ref.m, 0.0, bit).reshape(-1, 3)[mag]
        if np.linalg.norm(r) == 0:
            assert np.abs(s.field(bit)[mag]).max() == 0
            continue
        assert rel_l2(s.field(bit)[mag], r) < 1e-5, name
    local = ref.field(ref.m, 0.0, local_bits).reshape(-1, 3)[idx]
    btot = s.field(63)
    rms_grid = np.linalg.norm(btot[mag]) / np.sqrt(mag.sum())
    rms_err = np.linalg.norm(btot[idx] - (local + dem)) / np.sqrt(len(idx))
    assert rms_err / rms_grid < 1e-5, rms_err / rms_grid
    s.close()


def test_full_size_run_properties():
    """configs[1] in the bench configuration: |m| = 1 on magnetic cells, vacuum stays 0, and the
    device overlap W equals the oracle's W evaluated on the device state."""
    cfg = make_config(1)
    s = _solver(cfg)
    s.run(cfg.dt, 20)
    m = s.m()
    mag = magmask(cfg)
    assert np.allclose(np.linalg.norm(m[mag], axis=1), 1.0, atol=1e-6)
    assert np.all(m[~mag] == 0)
    ref = oracle_from(cfg, demag="off")
    W = ref.W(m.astype(np.float64).reshape(ref.m.shape))
    assert s.cavity()["W"] == pytest.approx(W, rel=1e-5)
    s.close()


def test_khat_bitwise_reproducible_across_contexts():
    """The device precompute of Khat must not depend on timing (it once did: transform matrices
    uploaded outside the work stream's order)."""
    cfg = small_config("disc", (40, 72, 3), seed=11, aniso=UNI, state="rand")
    first = None
    for _ in range(8):
        s = _solver(cfg)
        k = mcq.mcq_debug_khat(s.ctx)
        if first is None:
            first = k
        assert np.array_equal(k, first)
        s.close()


@pytest.mark.parametrize("kind,grid,D", [("disc", (48, 40, 3), 3e-3), ("film", (40, 24, 1), 1e-4)])
def test_dmi_field_and_steps_parity(kind, grid, D):
    """Interfacial DMI (reading C-DMI) through the general K-U instance: the DMI term alone and
    the total field within 1e-5, and 100 steps within 1e-4, against the oracle (D sized so that
    2D/(M_s dx) stays below the step's stability limit: 3.6 T for the Py disc, 0.3 T for YIG)."""
    from oracle import sim as S
    cfg = small_config(kind, grid, seed=13, state="rand")
    s = _solver(cfg)
    mcq.mcq_set_dmi(s.ctx, D)
    ref = oracle_from(cfg)
    ref.dmi = D
    ref.m = s.m().astype(np.float64).reshape(ref.m.shape)
    mag = magmask(cfg)
    for bit in (64, 127):
        b = s.field(bit)[mag]
        r = ref.field(ref.m, 0.0, bit).reshape(-1, 3)[mag]
        assert rel_l2(b, r) < 1e-5, bit
    assert S.DMI == mcq.TERM_DMI
    cfg2 = small_config(kind, grid, seed=13, state="phys")
    s2 = _solver(cfg2)
    mcq.mcq_set_dmi(s2.ctx, D)
    ref2 = oracle_from(cfg2)
    ref2.dmi = D
    s2.run(cfg2.dt, 100)
    ref2.run(cfg2.dt, 100)
    assert rel_l2(s2.m()[mag], ref2.m.reshape(-1, 3)[mag]) < 1e-4
    s.close()
    s2.close()


def test_divergence_is_detected_and_cleared_by_set_m():
    """Failure detection (include/mcq.h, mcq_synchronize): an absurd time step overflows the
    stage slopes, the step's m_{n+1} turns non-finite, and mcq_synchronize reports ESTATE
    "diverged" until a fresh state is installed (m and, since alpha diverged with it, the cavity
    memory); a sane run on the same context is then clean."""
    cfg = small_config("sphere", (16, 12, 8), seed=3, state="phys")
    s = mcq.Solver.from_config(cfg)
    s.run(cfg.dt, 5)
    mcq.mcq_synchronize(s.ctx)                       # healthy: no error
    s.run(1e30, 3)
    with pytest.raises(mcq.MCQError) as e:
        mcq.mcq_synchronize(s.ctx)
    assert e.value.code == -2 and "diverged" in str(e.value)
    assert not np.all(np.isfinite(s.m()))
    s.set_m(cfg.m0)                                  # clears the flag ...
    s.run(cfg.dt, 1)
    with pytest.raises(mcq.MCQError):                # ... but the cavity memory diverged too
        mcq.mcq_synchronize(s.ctx)
    s.set_m(cfg.m0)
    mcq.mcq_reset_memory(s.ctx)                      # a fresh state: m and alpha
    s.run(cfg.dt, 5)
    mcq.mcq_synchronize(s.ctx)
    assert np.all(np.isfinite(s.m()))
    s.close()
