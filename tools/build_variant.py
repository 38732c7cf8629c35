"""Build a tuning variant of libmcq.so with extra -D flags (experiments only; the product build is
paper_2410_00966_b200/build.py).  Usage: python tools/build_variant.py OUT.so -DMCQ_UE=4 ..."""
import importlib.util
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("b", os.path.join(ROOT, "paper_2410_00966_b200", "build.py"))
b = importlib.util.module_from_spec(spec)
spec.loader.exec_module(b)
out, defs = sys.argv[1], sys.argv[2:]
objs, procs = [], []
for src in b.SOURCES:
    obj = f"/tmp/variant_{os.getpid()}_{src}.o"
    procs.append(subprocess.Popen(["/usr/local/cuda/bin/nvcc", *b.FLAGS, *defs, "-c", os.path.join(b.CSRC, src), "-o", obj]))
    objs.append(obj)
assert all(p.wait() == 0 for p in procs)
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out, *objs, "-lcudart", "-ldl"])
print(out)
