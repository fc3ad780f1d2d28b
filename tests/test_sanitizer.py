"""compute-sanitizer over the kernel families.

The kernels stage gathered rows through shared memory with cp.async groups,
warp-synchronous hand-offs and mbarrier rings; memcheck, racecheck and
synccheck run tools/sanitize_cases.py (every kernel family on small graphs
that reach each code path, outputs checked against the oracle) and must
report 0 errors.

Opt-in: AUTOSAGE_SANITIZER=<memcheck|racecheck|synccheck|initcheck>.  The
B200 profiling recipe allows one sanitizer tool per GPU session (several in
one session have left a GPU unusable), so the default `pytest -m gpu` run
skips this test; each tool is run in its own session and its log is kept
under profiles/ (r02_sanitizer_<tool>.log).
"""
import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

TOOL = os.environ.get("AUTOSAGE_SANITIZER", "")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not TOOL, reason="opt-in: set AUTOSAGE_SANITIZER to one compute-sanitizer tool")
def test_kernels_clean_under_compute_sanitizer():
    assert TOOL in ("memcheck", "racecheck", "synccheck", "initcheck")
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    cmd = [exe, "--tool", TOOL, "--error-exitcode", "17", "--print-limit", "50"]
    if TOOL == "memcheck":
        cmd += ["--leak-check", "no"]
    if TOOL == "racecheck":
        cmd += ["--racecheck-report", "all"]
    cmd += [sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py")]
    env = dict(os.environ, PYTHONPATH=ROOT)
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=3000)
    log = r.stdout + r.stderr
    out = os.environ.get("AUTOSAGE_SANITIZER_LOG")
    if out:
        with open(out, "w") as fh:
            fh.write(" ".join(cmd) + "\n" + log)
    assert "SANITIZE_CASES_OK" in r.stdout, log[-4000:]
    m = re.search(r"ERROR SUMMARY: (\d+) error", log)
    assert r.returncode == 0 and m and int(m.group(1)) == 0, log[-4000:]
