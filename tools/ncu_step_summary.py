#!/usr/bin/env python
"""Markdown summary of a tools/ncu_step.py capture (its `--page raw --csv` export): per kernel
class, launches, device time, DRAM bytes against the algorithmic bytes (bench.alg_bytes), the
shared-memory wavefronts and bank conflicts with their time floor, issue / warp occupancy and
the top stall reasons.

    python tools/ncu_step_summary.py CSV CONFIG > profiles/...md"""
import csv
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import bench  # noqa: E402
from ncu_traffic import classify  # noqa: E402
from synth import make_config  # noqa: E402

SM, CLK = 148, 1.965e9  # SMs, SM clock under load (bench clocks lines)
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e-3, "us": 1e-6, "usecond": 1e-6,
         "msecond": 1e-3, "nsecond": 1e-9, "ns": 1e-9, "s": 1.0, "second": 1.0}


def main(path, k):
    rows = list(csv.reader(open(path)))
    h, u, data = rows[0], rows[1], rows[2:]
    col = {n: i for i, n in enumerate(h)}

    def val(r, n):
        i = col[n]
        return float(r[i].replace(",", "") or 0) * SCALE.get(u[i], 1)

    cfg = make_config(int(k))
    pad = [1 if n == 1 else 1 << (2 * n - 1).bit_length() for n in cfg.grid]  # 2 n rounded up to 2^k
    L = {"NKX": pad[0] // 2 + 1, "Ly": pad[1], "Lz": pad[2]}
    ab = bench.alg_bytes(L, cfg.grid, cfg.brms_map is not None)
    peak = bench.peaks()["hbm_gbs"]
    acc = {}
    for r in data:
        kc = classify(r[col["Kernel Name"]])
        if not kc:
            continue
        a = acc.setdefault(kc, {"n": 0, "t": 0, "dram": 0, "wf": 0, "cf": 0, "ia": [], "wa": [], "st": {},
                                "names": set(), "regs": set()})
        a["n"] += 1
        a["t"] += val(r, "gpu__time_duration.sum")
        a["dram"] += val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
        a["wf"] += val(r, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
        a["cf"] += val(r, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")
        a["ia"].append(val(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"))
        a["wa"].append(val(r, "sm__warps_active.avg.pct_of_peak_sustained_active"))
        a["names"].add(r[col["Kernel Name"]].split("(")[0].replace("void ", ""))
        a["regs"].add(r[col["launch__registers_per_thread"]])
        for n, i in col.items():
            if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
                key = n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]
                a["st"][key] = a["st"].get(key, 0) + float(r[i] or 0)
    stages = 4
    print(f"| class | kernels | launches/step | ms per stage | DRAM GB per stage | alg GB | DRAM/alg | alg GB/s (frac of {peak:.0f}) "
          f"| smem wavefronts (conflict share) | smem floor ms | DRAM floor ms | issue active | warps active | regs | top stalls per issue |")
    print("|" + "---|" * 15)
    for kc, a in acc.items():
        per = 1 if kc == "cavity" else stages
        t = a["t"] / per
        dram = a["dram"] / per
        alg = ab.get(kc, 0)
        gbs = alg / t / 1e9 if t else 0
        wf = a["wf"] / per
        st = sorted(a["st"].items(), key=lambda x: -x[1])[:4]
        n = len(a["ia"])
        print(f"| {kc} | {', '.join(sorted(a['names']))} | {a['n'] // per if per > 1 else a['n']} | {t * 1e3:.3f} | "
              f"{dram / 1e9:.3f} | {alg / 1e9:.3f} | {dram / alg if alg else 0:.2f} | {gbs:.0f} ({gbs / peak:.2f}) | "
              f"{wf / 1e6:.1f} M ({a['cf'] / max(1, a['wf']):.0%}) | {wf / (SM * CLK) * 1e3:.3f} | {dram / peak / 1e9 * 1e3:.3f} | "
              f"{sum(a['ia']) / n:.0f} % | {sum(a['wa']) / n:.0f} % | {'/'.join(sorted(a['regs']))} | "
              f"{', '.join(f'{k_} {v / n:.2f}' for k_, v in st)} |")


if __name__ == "__main__":
    main(*sys.argv[1:3])
