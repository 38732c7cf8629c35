#!/usr/bin/env python
"""One LLG step of a bench workload bracketed by cudaProfilerStart/Stop, for
`ncu --profile-from-start off` captures of exactly the kernels one step launches (4 RK4 RHS
evaluations + the cavity kernel), after two untimed warm-up steps.

    ncu --set full --profile-from-start off -o rep python tools/ncu_step.py CONFIG [persist]

(`persist`: the persistent cooperative 2D kernel for nz = 1 configs, 20 steps in one launch.)"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from synth import make_config  # noqa: E402
import paper_2410_00966_b200 as mcq  # noqa: E402


def main(k, persist=False):
    cfg = make_config(k)
    s = mcq.Solver.from_config(cfg)
    if persist:
        mcq.mcq_set_persistent_2d(s.ctx, 1)
    s.run(cfg.dt, 2)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    s.run(cfg.dt, 20 if persist else 1)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    s.close()


if __name__ == "__main__":
    main(int(sys.argv[1]), len(sys.argv) > 2 and sys.argv[2] == "persist")
