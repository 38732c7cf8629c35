#!/usr/bin/env python
"""Warp-stall samples of one kernel aggregated per CUDA source line.

  python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX LIB.so [N]
  NCU_COL="L1 Wavefronts Shared" python tools/ncu_lines.py ...   (any per-instruction column)

ncu's SASS source page carries the samples per instruction address; the line table comes from
`nvdisasm -g` on the cubin of LIB.so (the library the report was taken with: build it from the
same tree, -lineinfo).  Prints the N hottest source lines with their share of the samples."""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


COL = os.environ.get("NCU_COL", "Warp Stall Sampling (All Samples)")


def sass_samples(rep, rx):
    # a report, or its `ncu -i REP --page source --csv` export (taken on the GPU box when the
    # report is too large to bring back)
    out = open(rep).read() if rep.endswith(".csv") else subprocess.run(
        ["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{rx}"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    name = lines[0].split('","')[1].rstrip('",') if lines else "?"
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = [r for r in csv.DictReader(io.StringIO("\n".join(lines[start:]))) if r["Address"].startswith("0x")]
    base = min(int(r["Address"], 16) for r in rows)
    return name, {int(r["Address"], 16) - base: int(float(r[COL] or 0)) for r in rows}


def line_table(lib, mangled_hint):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
    table = {}
    for f in os.listdir(d):
        txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, f)], capture_output=True, text=True).stdout
        cur_fun, cur_line = None, None
        for l in txt.splitlines():
            m = re.match(r"\s*\.text\.(\S+):", l)
            if m:
                cur_fun = m.group(1)
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', l)
            if m:
                cur_line = (os.path.basename(m.group(1)), int(m.group(2)))
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
            if m and cur_fun and cur_line:
                table.setdefault(cur_fun, {})[int(m.group(1), 16)] = cur_line
    return table


def main():
    rep, rx, lib = sys.argv[1:4]
    n = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    kname, samp = sass_samples(rep, rx)
    tab = line_table(lib, rx)
    cands = [f for f in tab if re.search(rx, f)]
    # pick the function whose instruction count matches the report's
    fun = min(cands, key=lambda f: abs(len(tab[f]) - len(samp)))
    lt = tab[fun]
    per = collections.Counter()
    for off, s in samp.items():
        per[lt.get(off, ("?", 0))] += s
    tot = sum(samp.values())
    srcs = {}
    print(f"{kname}\n  function {fun}: {tot} samples")
    for (f, ln), s in per.most_common(n):
        if f not in srcs:
            p = next((os.path.join(r, f) for r, _, fs in os.walk(os.path.dirname(os.path.abspath(lib))) if f in fs), None)
            srcs[f] = open(p).read().splitlines() if p else []
        text = srcs[f][ln - 1].strip() if 0 < ln <= len(srcs[f]) else ""
        print(f"{100 * s / tot:5.1f}%  {f}:{ln}  {text[:90]}")


if __name__ == "__main__":
    main()
