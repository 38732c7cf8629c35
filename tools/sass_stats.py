#!/usr/bin/env python
"""Compile one csrc/*.cu for sm_100a and report, per kernel matching a regex: registers, spill
bytes and the static SASS instruction mix (FP32 packed / scalar, shared, global, integer, ...).

  python tools/sass_stats.py passes.cu 'k_zconv_seqILi(256|512)ELb0' [-D MCQ_X=1 ...]
"""
from __future__ import annotations

import collections
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2410_00966_b200", "csrc")

CLASSES = [
    ("fp2", r"^(FADD2|FMUL2|FFMA2)"), ("fp", r"^(FADD|FMUL|FFMA|FMNMX|FSEL|FSETP|MUFU|FCHK)"),
    ("lds", r"^LDS"), ("sts", r"^STS"), ("ldg", r"^(LDG|LD\.)"), ("stg", r"^(STG|ST\.)"),
    ("shfl", r"^SHFL"), ("bar", r"^(BAR|SYNCS|WARPSYNC)"), ("tma", r"^(UTMA|UBLKCP)"),
    ("int", r"^(IMAD|IADD|LOP|SHF|LEA|ISETP|SEL|IMNMX|PRMT|I2F|F2I|IABS|BMSK|POPC|FLO)"),
    ("mov", r"^(MOV|UMOV|R2UR|S2R|S2UR|CS2R|LDC|ULDC)"), ("ctrl", r"^(BRA|EXIT|BSYNC|BSSY|CALL|RET|NOP)"),
]


def main():
    src, pat = sys.argv[1], sys.argv[2]
    defs = sys.argv[3:]
    obj = os.path.join(tempfile.mkdtemp(), "k.o")
    cmd = ["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
           "--expt-relaxed-constexpr", "-Xptxas", "-v", *defs, "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        print(r.stderr)
        sys.exit(1)
    regs, spill, cur = {}, {}, None
    for line in r.stderr.splitlines():
        m = re.search(r"Function properties for (\S+)", line)
        if m:
            cur = m.group(1)
        m = re.search(r"(\d+) bytes spill stores", line)
        if m and cur:
            spill[cur] = int(m.group(1))
        m = re.search(r"Used (\d+) registers", line)
        if m and cur:
            regs[cur] = int(m.group(1))
    sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    funcs, name = collections.defaultdict(list), None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            name = m.group(1)
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if m and name:
            funcs[name].append(m.group(2))
    for fn, ops in funcs.items():
        if not re.search(pat, fn):
            continue
        mix = collections.Counter()
        for op in ops:
            for cls, rx in CLASSES:
                if re.match(rx, op):
                    mix[cls] += 1
                    break
            else:
                mix["other"] += 1
        body = sum(v for k, v in mix.items() if k != "ctrl") + mix["ctrl"] - ops.count("NOP")
        print(f"{fn}\n  regs {regs.get(fn)}  spill {spill.get(fn, 0)}  instr {body}  " +
              "  ".join(f"{k} {v}" for k, v in sorted(mix.items(), key=lambda kv: -kv[1])))


if __name__ == "__main__":
    main()
