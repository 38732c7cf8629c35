"""Extract per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the hot-path
kernels from an `ncu --set full` report and store it for bench.py's roofline "traffic" field.

    python tools/ncu_traffic.py report.ncu-rep profiles/ncu_traffic.json config1 [STAGES]

The JSON maps a workload key to {kernel class: bytes per stage, "_source": report name}; kernel
classes follow bench.py (yfwd, zconv, yinv, y2d, update, cavity), whose live timings bracket one
RHS stage of a class (several launches: per-component K-Y passes, the K-Z normal + lone-tile
launches).  With STAGES given (a tools/ncu_step.py capture of one RK4 step: 4), the bytes of all
launches of a class are summed and divided by STAGES (the cavity kernel runs once per step);
without it, the per-launch average is stored (the round-1 captures)."""
import csv
import json
import os
import subprocess
import sys

def classify(name):
    """Kernel class of an ncu kernel name (template arguments: k_ypass<L, INV, ...>,
    k_conv<L, Y2D>)."""
    n = name.split("(")[0].replace("void ", "").replace("mcq::", "").strip()
    base = n.split("<")[0]
    targs = [x.strip(" >") for x in n.split("<", 1)[1].split(",")] if "<" in n else []
    if base == "k_ypass":
        return "yinv" if len(targs) > 1 and targs[1] in ("1", "true") else "yfwd"
    if base == "k_conv":
        return "y2d" if len(targs) > 1 and targs[1] in ("1", "true") else "zconv"
    return {"k_zconv_seq": "zconv", "k_zconv2": "zconv", "k_zconv3": "zconv", "k_zconv_tma": "zconv", "k_update": "update", "k_cavity": "cavity"}.get(base)


def main(rep, out, key, stages=None):
    # a report, or its `ncu -i REP --page raw --csv` export (full-set step captures exceed what
    # gpurun copies back; they are exported on the box)
    txt = open(rep).read() if rep.endswith(".csv") else subprocess.run(
        ["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, data = rows[0], rows[2:]
    iname = hdr.index("Kernel Name")
    ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    iu = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    acc = {}
    for d in data:
        k = classify(d[iname])
        if not k:
            continue
        b = float(d[ir]) * scale.get(iu[ir], 1) + float(d[iw]) * scale.get(iu[iw], 1)
        acc.setdefault(k, []).append(b)
    res = json.load(open(out)) if os.path.exists(out) else {}
    if stages:
        res[key] = {k: sum(v) / (1 if k == "cavity" else int(stages)) for k, v in acc.items()}
        res[key]["_launches"] = {k: len(v) for k, v in acc.items()}
    else:
        res[key] = {k: sum(v) / len(v) for k, v in acc.items()}
    res[key]["_source"] = os.path.basename(rep)
    json.dump(res, open(out, "w"), indent=1, sort_keys=True)
    print(json.dumps(res[key]))


if __name__ == "__main__":
    main(*sys.argv[1:5])
