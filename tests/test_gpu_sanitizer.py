"""compute-sanitizer (memcheck, racecheck, synccheck) over every kernel family on small grids
(VERDICT r1 hygiene; tools/sanitize_small.py).  Opt-in: the B200 profiling guide records that
compute-sanitizer runs on this driver have left GPUs unusable, so the round-end suite does not
start it unless MCQ_RUN_SANITIZER names the tool(s) to run, one per gpurun call
(MCQ_RUN_SANITIZER=memcheck, =racecheck or =synccheck).  The logs of the runs made are kept
in profiles/r2_sanitizer_*.log.  (Round 2: the GPU pool refuses compute-sanitizer runs
outright, so no log could be taken.)"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOLS = [t for t in os.environ.get("MCQ_RUN_SANITIZER", "").split(",") if t]


@pytest.mark.skipif(not TOOLS, reason="opt-in: set MCQ_RUN_SANITIZER=memcheck|racecheck|synccheck")
@pytest.mark.parametrize("tool", TOOLS or ["memcheck"])
def test_compute_sanitizer(tool):
    assert tool in ("memcheck", "racecheck", "synccheck", "initcheck")
    cmd = ["compute-sanitizer", "--tool", tool, "--error-exitcode", "9", sys.executable,
           os.path.join(ROOT, "tools", "sanitize_small.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1800)
    log = os.path.join(ROOT, "gpurun_out", f"sanitizer_{tool}.log")
    os.makedirs(os.path.dirname(log), exist_ok=True)
    open(log, "w").write(r.stdout + r.stderr)
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    assert "ERROR SUMMARY: 0 errors" in r.stdout + r.stderr
