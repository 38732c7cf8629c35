"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck): every kernel family
of the hot path on small grids — the RK4 step with cavity and map (3D: K-Y, K-Z v2 at Lz = 256 and 512 (TMA, lone tiles),
K-YI, K-U, K-CAV; 2D: K-Y2D), the old K-Z at other Lz, relax, field evaluation, Dormand-Prince,
two cavity modes, thermal + DMI, and a loopback z-slab decomposition.  Run under
tests/test_gpu_sanitizer.py (opt-in) or by hand:
    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_small.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2410_00966_b200 as mcq  # noqa: E402
from synth import small_config  # noqa: E402


def main():
    for kind, grid in [("film", (12, 10, 1)), ("sphere", (8, 6, 70)), ("sphere", (10, 6, 9)), ("film", (6, 3, 129)),
                       ("film", (8, 6, 200))]:
        cfg = small_config(kind, grid, seed=3, state="phys")
        s = mcq.Solver.from_config(cfg)
        s.run(cfg.dt, 3)
        s.field(127)
        s.relax(cfg.dt, 0.0, 2)
        mcq.mcq_run_dp(s.ctx, cfg.dt, 2)
        s.sync()
        s.close()
    cfg = small_config("sphere", (10, 6, 9), seed=4, state="phys")
    s = mcq.Solver.from_config(cfg)
    mcq.mcq_set_modes(s.ctx, 2)
    mcq.mcq_set_brms_mode(s.ctx, 1, cfg.brms_map)
    s.set_m(cfg.m0)
    mcq.mcq_set_dmi(s.ctx, 1e-4)
    mcq.mcq_set_temperature(s.ctx, 300.0, 7)
    s.run(cfg.dt, 3)
    s.sync()
    s.close()
    lb = mcq.Solver.from_config(small_config("sphere", (8, 6, 70), seed=5, state="phys"), dist={"rank": -1, "world": 2})
    lb.run(cfg.dt, 2)
    lb.sync()
    lb.close()
    print("sanitize_small: done")


if __name__ == "__main__":
    main()
