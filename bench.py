#!/usr/bin/env python
"""Benchmark: LLG + cavity RK4 steps (cell-updates/s) on BASELINE.json configs[4] by default
(512 x 512 x 256: the grid the metric's 1/2/4/8-GPU strong-scaling target is quoted on).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config k] [--impl mcq|reference]

One process per GPU (torchrun for N > 1).  N > 1 (default --decomp slab): the SAME grid z-slab
decomposed over the ranks (libmcq's NCCL halos, demag all-to-all transpose and W all-gather;
"scaling": "strong"), with a bitwise self-check against the undecomposed run
("self_check"); --decomp replicas: independent replicas, one bias-field sweep point per rank
("scaling": "weak").  Timing: W untimed warm-up steps, then exactly K steps between barrier +
synchronize, CUDA events on the library's stream, max over ranks.  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "LLG cell-updates/sec & % HBM roofline at 1/2/4/8 B200"


def ncu_traffic(config, kernel):
    """Per-launch DRAM bytes of `kernel` from the committed ncu capture (tools/ncu_traffic.py), or
    None; the file names the report it came from."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))[f"config{config}"]
        return d.get(kernel), d.get("_source")
    except Exception:
        return None, None


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


# ---------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) >= 9:
                rows.append(p)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        busy = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": float(np.median(busy)), "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------- algorithmic bytes
def alg_bytes(L, grid, has_map, slabs=1):
    """Algorithmic HBM bytes per launch of each kernel class (fp32 state, complex64 spectra);
    with z slabs, one launch covers 1/slabs of the grid (and of the Khat columns in K-Z)."""
    nx, ny, nz = grid
    nz //= slabs
    N = nx * ny * nz
    nkx, Ly, Lz = L["NKX"], L["Ly"], L["Lz"]
    X = 3 * nz * ny * nkx * 8
    Y = 3 * nz * Ly * nkx * 8
    K = 6 * (Lz // 2 + 1) * (Ly // 2 + 1) * nkx * 4 // slabs
    state = (36 + 60 + 60 + 48) / 4 * N           # RK4 state traffic averaged over the 4 stages
    out = {"yfwd": X + Y, "zconv": 2 * Y + K, "yinv": Y + X,
           "y2d": 2 * X + 6 * ((Ly // 2 + 1) * nkx * 4),
           "update": 2 * X + state + (12 * N if has_map else 0), "cavity": 0}
    return out


def step_alg_bytes(L, grid, has_map, slabs=1):
    b = alg_bytes(L, grid, has_map, slabs)
    if grid[2] > 1:
        return 4 * (b["yfwd"] + b["zconv"] + b["yinv"] + b["update"])
    return 4 * (b["y2d"] + b["update"])


# ---------------------------------------------------------------- oracle timing
def cpu_baseline(cfg, rhs_evals=1, full=None):
    """Oracle (fp64 NumPy, as it stands) on the same workload, bounded sample: `rhs_evals`
    right-hand-side evaluations (one RK4 step = 4), scaled to cell-updates/s = N * evals/4 / t.
    `full`: the full-size config when `cfg` is its downscaled construction (configs[4]: the
    direct-DFT oracle needs ~100 GB and hours per RHS at 512 x 512 x 256); the line then also
    carries the per-cell rate extrapolated to the full grid by the oracle's cost model
    N (Lx + Ly + Lz) (one DFT-matrix product per padded axis)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from helpers import oracle_from
    t0 = time.perf_counter()
    ref = oracle_from(cfg)
    ref.octant()
    if ref.demag_mode == "dft":
        from oracle import tensor as T
        ref._padded = T.padded_tensor(ref.grid, ref.cell, ref.octant())
    setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    for _ in range(rhs_evals):
        ref.rhs(ref.m, 0.0)
    dt = time.perf_counter() - t0
    out = {"value": cfg.n * rhs_evals / 4 / dt, "unit": "cell-updates/s", "cores": len(os.sched_getaffinity(0)),
           "kind": "oracle", "sample": f"{rhs_evals} RHS evaluation(s) (1/4 RK4 step each) of {cfg.name} "
           f"{tuple(cfg.grid)}, direct-DFT demag in fp64; tensor setup {setup:.1f} s untimed", "seconds": dt}
    if full is not None:
        def pad(n):
            return 1 if n == 1 else 1 << math.ceil(math.log2(2 * n))
        ls = sum(pad(g) for g in cfg.grid)
        lf = sum(pad(g) for g in full.grid)
        out["sample"] = ("downscaled construction: " + out["sample"] +
                         f"; the full {tuple(full.grid)} grid does not fit the oracle's direct DFT")
        out["extrapolated_full_grid"] = {"value": out["value"] * ls / lf, "unit": "cell-updates/s",
                                         "model": "oracle cost per cell ~ Lx + Ly + Lz (padded)"}
    return out


def run_reference(args):
    """--impl reference: the oracle is this tier's reference arm (CPU, host cores)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from synth import make_config
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from helpers import oracle_from
    full = make_config(args.config)
    sample_grid = {0: (64, 64, 1), 1: (32, 32, 32), 2: (32, 32, 32), 3: (64, 64, 8), 4: (64, 64, 32)}[args.config]
    cfg = make_config(args.config, grid=sample_grid) if args.config in (1, 2, 3) else full
    if args.config == 4:
        cfg = make_config(4, grid=sample_grid)
    ref = oracle_from(cfg)
    ref.rhs(ref.m, 0.0)
    for _ in range(args.warmup):
        ref.step(cfg.dt)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ref.step(cfg.dt)
    el = time.perf_counter() - t0
    v = cfg.n * args.steps / el
    cores = len(os.sched_getaffinity(0))
    line = {"metric": METRIC, "value": v, "unit": "cell-updates/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": full.name, "sample_grid": list(cfg.grid), "full_grid": list(full.grid)},
            "cpu_baseline": {"value": v, "unit": "cell-updates/s", "cores": cores, "kind": "oracle",
                             "sample": f"{args.steps} RK4 steps of the {full.name} construction on "
                                       f"{cfg.grid} (same recipe, reduced grid)"},
            "e2e": {"value": v, "unit": "cell-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="default: 40 (configs[4]), 500 (others)")
    ap.add_argument("--warmup", type=int, default=None, help="default: 5 (configs[4]), 20 (others)")
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--e2e-steps", type=int, default=None, help="steps of the end-to-end run (default: --steps)")
    ap.add_argument("--check-steps", type=int, default=2, help="N > 1 slab runs: steps of the bitwise self-check")
    ap.add_argument("--impl", default="mcq", choices=["mcq", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=5)
    ap.add_argument("--decomp", default="slab", choices=["slab", "replicas"],
                    help="N > 1: z-slab decomposition of one grid (strong) or independent replicas (weak)")
    ap.add_argument("--loopback", type=int, default=0,
                    help="N == 1: run the decomposed schedule with this many z slabs on the one GPU")
    ap.add_argument("--batch", type=int, default=1,
                    help="independent replicas per GPU (one bias point each, own stream; latency-bound grids)")
    ap.add_argument("--integrator", default="rk4", choices=["rk4", "dp"],
                    help="dp: fixed-step Dormand-Prince 5(4) steps (7 RHS each, NEXT-1)")
    ap.add_argument("--modes", type=int, default=1, help="cavity modes (NEXT-2; extra modes: dark map)")
    ap.add_argument("--temperature", type=float, default=0.0, help="thermal field, K (NEXT-4)")
    ap.add_argument("--dmi", type=float, default=0.0, help="interfacial DMI constant, J/m^2 (NEXT-4)")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 40 if args.config == 4 else 500
    if args.warmup is None:
        args.warmup = 5 if args.config == 4 else 20
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return run_reference(args)
    if args.batch > 1:  # more hardware work queues than the default 8 for concurrent replica streams
        os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2410_00966_b200 as mcq
    from synth import make_config

    from paper_2410_00966_b200.replicas import replica_bias, max_over_ranks
    from paper_2410_00966_b200.slabs import slab_dist
    cfg = make_config(args.config)
    slab = world > 1 and args.decomp == "slab"
    R = max(1, args.batch) if not slab and args.loopback <= 1 else 1
    # replica (rank, j): its own bias point of the sweep (replicas for small grids)
    bext0 = cfg.bext
    streams, solvers = [], []
    for j in range(R):
        if (world > 1 and not slab) or R > 1:
            cfg.bext = replica_bias(bext0, world * R, rank * R + j)
        s_j = torch.cuda.Stream()         # a real stream: the library's kernels and our events share it
        dd = slab_dist(rank, world, local) if slab else None
        if world == 1 and args.loopback > 1:
            dd = {"rank": -1, "world": args.loopback}
        sv = mcq.Solver.from_config(cfg, stream=s_j.cuda_stream, dist=dd, set_state=args.modes <= 1)
        if args.modes > 1:  # extra modes k >= 1: the dark two-wire map, f_c shifted by 0.3 GHz per mode
            from synth.configs import two_wire_map
            dark, _, _ = two_wire_map(cfg.grid, cfg.cell, cfg.Ms, cfg.mask, 1e9, "dark")
            mcq.mcq_set_modes(sv.ctx, args.modes)
            for k in range(1, args.modes):
                mcq.mcq_set_brms_mode(sv.ctx, k, dark)
                mcq.mcq_set_cavity_mode(sv.ctx, k, cfg.f_c + 0.3e9 * k, cfg.kappa)
            sv.set_m(cfg.m0)
        if R > 1 and cfg.grid[2] == 1:  # concurrent 2D replicas: one persistent kernel per run call
            mcq.mcq_set_persistent_2d(sv.ctx, 1)
        if args.temperature > 0:
            mcq.mcq_set_temperature(sv.ctx, args.temperature, 1234 + j)
        if args.dmi != 0:
            mcq.mcq_set_dmi(sv.ctx, args.dmi)
        if cfg.relax_first:
            sv.relax(cfg.dt * 0.5, 1e-3, 2000)
            mcq.mcq_reset_memory(sv.ctx)
        streams.append(s_j)
        solvers.append(sv)
    stream, solver = streams[0], solvers[0]
    torch.cuda.set_stream(stream)
    jobs = (1 if slab else world) * R     # grids the job advances per step
    L = mcq.mcq_debug_layout(solver.ctx)

    def barrier():
        # drain this rank's work (incl. libmcq's own NCCL calls) before torch's collective, so
        # the two communicators never have kernels in flight at the same time
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def advance(sv, steps):
        if args.integrator == "dp":
            mcq.mcq_run_dp(sv.ctx, cfg.dt, steps)
        else:
            sv.run(cfg.dt, steps)

    def run_all(steps):  # every replica on its own stream, fork / join through events
        fork = torch.cuda.Event()
        fork.record(stream)
        for s_j, sv in zip(streams, solvers):
            s_j.wait_event(fork)
            advance(sv, steps)
        for s_j in streams[1:]:
            join = torch.cuda.Event()
            join.record(s_j)
            stream.wait_event(join)

    # warm-up (captures the graphs)
    run_all(args.warmup)
    barrier()
    launches0 = sum(mcq.mcq_kernel_launches(sv.ctx) for sv in solvers)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        run_all(args.steps)
        ev1.record(stream)
        barrier()
    launches = sum(mcq.mcq_kernel_launches(sv.ctx) for sv in solvers) - launches0
    ms_max = max_over_ranks(ev0.elapsed_time(ev1), device="cuda")
    value = cfg.n * args.steps * jobs / (ms_max * 1e-3)

    # e2e through the public API with host buffers, timed on the host: the state in from pinned
    # host memory (mcq_set_m, H2D), then every step one mcq_run(dt, 1) call and a device-to-host
    # read of that step's result (mcq_get_cavity: alpha, W, t, S, C; it synchronises), and the
    # final state out (mcq_get_m, D2H).  Bytes per step count these copies.
    m_host = torch.from_numpy(np.ascontiguousarray(cfg.m0, np.float32)).pin_memory()
    out_host = torch.empty_like(m_host).pin_memory()
    e2e_steps = args.e2e_steps or args.steps
    cav_bytes = mcq.mcq_cavity_state_bytes()
    for sv in solvers:                       # the 1-step graphs are captured before timing
        mcq.mcq_set_m(sv.ctx, m_host.numpy())
        advance(sv, 1)
    barrier()
    t0 = time.perf_counter()
    for sv in solvers:
        mcq.mcq_set_m(sv.ctx, m_host.numpy())
    for _ in range(e2e_steps):
        for sv in solvers:
            advance(sv, 1)
        for sv in solvers:
            mcq.mcq_get_cavity(sv.ctx)
    for sv in solvers:
        mcq.mcq_get_m(sv.ctx, cfg.n, out_host.numpy().reshape(-1))
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0, device="cuda")
    e2e_val = cfg.n * e2e_steps * jobs / e2e_s
    h2d_step = 12 * cfg.n * jobs / e2e_steps / (world if slab else 1)
    d2h_step = (12 * cfg.n * jobs / e2e_steps / (world if slab else 1)) + cav_bytes * len(solvers)

    # N > 1 slab decomposition: every rank replays `check_steps` steps of the undecomposed grid on
    # its own GPU and compares its planes bitwise with the decomposed result
    self_check = None
    if slab:
        k = args.check_steps
        for sv in solvers:
            sv.set_m(cfg.m0)
            mcq.mcq_reset_memory(sv.ctx)
            advance(sv, k)
        got = solvers[0].m()
        ref1 = mcq.Solver.from_config(cfg, stream=stream.cuda_stream)
        advance(ref1, k)
        want = ref1.m()
        ref1.close()
        from paper_2410_00966_b200.slabs import cell_range
        i0, i1 = cell_range(cfg.grid, world, rank)
        same = bool(np.array_equal(got[i0:i1], want[i0:i1]))
        allsame = max_over_ranks(0.0 if same else 1.0, device="cuda") == 0.0
        self_check = {"bitwise_vs_p1": allsame, "steps": k,
                      "what": "each rank's planes of m after k steps from the same state vs the "
                              "undecomposed 1-GPU run of the same grid on that rank's GPU"}

    # per-kernel timing (CUDA events around each launch, same stream) -> roofline of the top kernel
    prof = mcq.mcq_profile_run(solver.ctx, cfg.dt, args.profile_steps)
    ns = world if slab else (args.loopback if args.loopback > 1 else 1)  # slabs per launch
    ab = alg_bytes(L, cfg.grid, cfg.brms_map is not None, ns)
    share = {k: v[0] * v[1] for k, v in prof.items() if v[1] > 0}
    top = max(share, key=share.get)
    pk = peaks()
    achieved = ab[top] / (prof[top][0] * 1e-3) / 1e9
    step_bytes = step_alg_bytes(L, cfg.grid, cfg.brms_map is not None, ns)
    if not slab and args.loopback > 1:  # every slab's launches run on this GPU in one step
        step_bytes *= ns
    traffic, traffic_src = ncu_traffic(args.config, top) if (world == 1 and args.loopback <= 1) else (None, None)
    ms_step = ms_max / args.steps
    # resident working set of one replica: 4 state arrays, X, Y, Khat (+ map), vs the 126 MB L2
    ws = (4 * 12 * cfg.n + 3 * cfg.grid[2] * cfg.grid[1] * L["P"] * 8 * (1 + (L["Ly"] if cfg.grid[2] > 1 else 0)
          / max(cfg.grid[1], 1)) + 6 * (L["Lz"] // 2 + 1) * (L["Ly"] // 2 + 1) * L["P"] * 4
          + (12 * cfg.n if cfg.brms_map is not None else 0)) * R
    l2_note = (f"working set {ws / 1e6:.0f} MB > 126 MB L2: streamed from HBM every step (no flush needed)"
               if ws > 126e6 else
               f"working set {ws / 1e6:.1f} MB fits in the 126 MB L2 (latency-bound workload; not flushed)")

    if rank == 0:
        res = {
            "metric": METRIC, "value": value, "unit": "cell-updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if slab else "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg.name, "grid": list(cfg.grid), "cells": cfg.n,
                       "magnetic_cells": cfg.n_magnetic(), "dt_s": cfg.dt,
                       "integrator": "RK4 (4 RHS/step)" if args.integrator == "rk4" else
                       "Dormand-Prince 5(4), fixed dt (7 RHS/step; roofline/kernels from an RK4 profile)",
                       "parallelism": (f"z-slab x{world} (NCCL)" if slab else f"replicas x{world}")
                       if world > 1 else (f"single GPU, loopback z-slab x{args.loopback}"
                                          if args.loopback > 1 else "single GPU"),
                       "replicas_per_gpu": R,
                       **({"variant": {"modes": args.modes, "temperature_K": args.temperature, "dmi": args.dmi}}
                          if (args.modes > 1 or args.temperature > 0 or args.dmi != 0) else {}),
                       "l2": l2_note,
                       "padded_fft": [L["Lx"], L["Ly"], L["Lz"]]},
            "roofline": {"bound": "hbm", "kernel": top, "achieved": achieved, "peak": pk["hbm_gbs"],
                         "unit": "GB/s", "frac": achieved / pk["hbm_gbs"], "traffic": traffic,
                         "traffic_source": (f"profiles/ncu_traffic.json from {traffic_src} (ncu --set full, dram "
                                            f"bytes read+write per RHS stage of this kernel class, i.e. per timed 'launch' here; "
                                            f"summary profiles/r2_final_ncu.md)"
                                            if traffic_src else None),
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if not pk.get("_fallback") else "fallback",
                         "alg_bytes_per_launch": ab[top], "ms_per_launch": prof[top][0]},
            "step_roofline": {"alg_bytes_per_step": step_bytes, "achieved_gbs": step_bytes / (ms_step * 1e-3) / 1e9,
                              "frac": step_bytes / (ms_step * 1e-3) / 1e9 / pk["hbm_gbs"]},
            "kernels": {k: {"ms": v[0], "per_step": v[1], "share": share.get(k, 0.0) / max(1e-12, sum(share.values())),
                            "alg_gbs": (ab[k] / (v[0] * 1e-3) / 1e9) if v[0] > 0 else None}
                        for k, v in prof.items() if v[1] > 0},
            "rhs_evals_per_s": (4 if args.integrator == "rk4" else 7) * value,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "e2e": {"value": e2e_val, "unit": "cell-updates/s", "h2d_bytes_per_step": h2d_step,
                    "d2h_bytes_per_step": d2h_step, "steps": e2e_steps,
                    "calls": "mcq_set_m (pinned H2D) once; per step mcq_run(dt, 1) + mcq_get_cavity "
                             "(D2H of the step's cavity state, synchronising); mcq_get_m (D2H) at the end"},
        }
        if self_check is not None:
            res["self_check"] = self_check
        if world == 1 and not args.no_cpu_baseline:
            if args.config == 4:
                res["cpu_baseline"] = cpu_baseline(make_config(4, grid=(128, 128, 64)), rhs_evals=2, full=cfg)
            else:
                res["cpu_baseline"] = cpu_baseline(cfg)
        print(json.dumps(res), flush=True)
    for sv in solvers:
        sv.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
