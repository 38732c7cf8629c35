"""Hottest SASS instructions of one kernel from an ncu report (source page, SASS view):
python tools/ncu_hot.py report.ncu-rep kernel_regex [N]  — prints the top-N instructions by warp
stall samples with their stall-reason breakdown, and totals by opcode class."""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep, rx = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{rx}"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    # stop at the next kernel block if several
    rows = [r for r in rows if r.get("Address", "").startswith("0x")]
    tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
    stall_cols = [k for k in rows[0] if k.startswith("stall_") or "Stall" in k and k not in (
        "Warp Stall Sampling (All Samples)", "Warp Stall Sampling (Not-issued Samples)")]
    print(f"total samples {tot}, instructions {len(rows)}")
    by = collections.Counter()
    for r in rows:
        op = r["Source"].split()[0] if r["Source"].split() else "?"
        if op.startswith("@"):
            op = r["Source"].split()[1]
        by[op.split(".")[0]] += int(r["Warp Stall Sampling (All Samples)"] or 0)
    print("by opcode:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in by.most_common(14)))
    rows.sort(key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))
    for r in rows[:n]:
        s = int(r["Warp Stall Sampling (All Samples)"] or 0)
        print(f"{100 * s / tot:5.1f}%  {r['Address'][-5:]}  {r['Source'].strip()[:70]}")


if __name__ == "__main__":
    main()
