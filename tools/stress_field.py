"""Determinism stress: the demag field of the same state, evaluated repeatedly (fresh contexts
and repeated calls), must be bitwise identical.  Usage: python tools/stress_field.py [reps]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2410_00966_b200 as mcq  # noqa: E402
from synth import small_config  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
cases = [("disc", (40, 72, 3), {"ku1": 2e4, "u": (0.2, 0.3, 1.0)}), ("sphere", (24, 20, 12), None),
         ("film", (64, 64, 1), None), ("sphere", (30, 18, 5), None)]
for kind, grid, an in cases:
    cfg = small_config(kind, grid, seed=11, aniso=an, state="rand")
    ref = None
    bad = 0
    for r in range(reps):
        s = mcq.Solver.from_config(cfg)
        for k in range(3):
            f = s.field(8)
            if ref is None:
                ref = f.copy()
            elif not np.array_equal(f, ref):
                bad += 1
                d = np.abs(f - ref).max(axis=1)
                idx = np.nonzero(d)[0]
                if bad <= 3:
                    nx, ny, nz = grid
                    print(f"  {kind}{grid} rep {r} call {k}: {idx.size} cells differ, max {d.max():.3e};"
                          f" z of first {[(i // (nx * ny)) for i in idx[:8]]} y {[(i // nx) % ny for i in idx[:8]]}"
                          f" x {[i % nx for i in idx[:8]]}")
        s.close()
    print(f"{kind}{grid}: {bad} mismatching evaluations of {3 * reps}")
