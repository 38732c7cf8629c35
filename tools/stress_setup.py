"""Determinism of per-context setup: Khat, the tensor octant and m after set_m, over fresh
contexts.  Usage: python tools/stress_setup.py [reps]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2410_00966_b200 as mcq  # noqa: E402
from synth import small_config  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
cfg = small_config("disc", (40, 72, 3), seed=11, aniso={"ku1": 2e4, "u": (0.2, 0.3, 1.0)}, state="rand")
ref = {}
bad = {}
for r in range(reps):
    s = mcq.Solver.from_config(cfg)
    got = {"khat": mcq.mcq_debug_khat(s.ctx), "m": s.m().copy(), "demag": s.field(8).copy(),
           "octant": mcq.mcq_debug_tensor_octant(s.ctx)}
    got["khat2"] = mcq.mcq_debug_khat(s.ctx)   # after the octant rebuild (same buffer)
    for k, v in got.items():
        if k not in ref:
            ref[k] = v
        elif not np.array_equal(v, ref[k]):
            bad[k] = bad.get(k, 0) + 1
            if bad[k] <= 2:
                d = np.argwhere(v != ref[k])
                print(f"rep {r} {k}: {len(d)} entries differ; first {d[:4].tolist()}")
    s.close()
print("mismatches:", bad, "of", reps)
