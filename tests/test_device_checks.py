"""Memory-safety check of the kernels with the checked build (VERDICT r1
item 8).  compute-sanitizer is closed on the B200 pool ("runs under it have
left GPUs needing a reset"), so `make checked` compiles the same sources with
device-side bounds checks (csrc/dcheck.cuh: every gathered row index, entry
range and row lookup of the SpMM lane-group and ring kernels and the SDDMM
pair kernel is asserted; a failed check traps the launch).  The parity
workload tools/sanitize_cases.py -- every kernel family on graphs shaped to
reach each path, outputs compared with the oracle -- must pass on it.
tests/test_sanitizer.py keeps the compute-sanitizer form for pools where the
tool is open.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2511_17594_b200", "libautosage_b200_checked.so")


@pytest.mark.skipif(not os.path.exists(CHECKED), reason="checked build absent (make -C paper_2511_17594_b200 checked)")
def test_parity_workload_passes_the_checked_build():
    env = dict(os.environ, AUTOSAGE_DEV_LIB=CHECKED, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=1200)
    log = r.stdout + r.stderr
    assert "autosage device check failed" not in log, log[-4000:]
    assert r.returncode == 0 and "SANITIZE_CASES_OK" in r.stdout, log[-4000:]


@pytest.mark.skipif(not os.path.exists(CHECKED), reason="checked build absent")
def test_checked_build_is_the_library_loaded():
    code = ("import paper_2511_17594_b200._capi as c, os; "
            "print(os.path.basename(c.LIB_PATH))")
    env = dict(os.environ, AUTOSAGE_DEV_LIB=CHECKED, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.stdout.strip() == "libautosage_b200_checked.so", r.stdout + r.stderr
