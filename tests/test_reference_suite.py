"""The reference's own doctest suites, compiled unchanged against the B200
library.

tests/compat/Makefile compiles /root/reference/proj/tests/<suite>.cpp in
place with -Iinclude/compat, so their `#include "autosage/..."` lines resolve
to include/autosage_b200_compat.hpp -- the reference's namespace autosage
re-declared over the C-ABI -- and with the doctest shim tests/compat/doctest.h.
Each binary must report every test case passed.  test_cache and test_io need
no device (cache lines, signatures, ASCR files are host work); the others run
the GPU kernels and scheduler.  test_cli needs the reference's CLI binary and
CLI11 (absent) and is replaced by tests/test_cli.py.
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "compat", "_bin")

HOST_SUITES = ["test_cache", "test_io"]
GPU_SUITES = ["test_csr", "test_kernels", "test_cost", "test_scheduler", "test_attention", "test_generate"]


def _run(suite, tmp_path):
    exe = os.path.join(BIN, suite)
    if not os.path.exists(exe):
        pytest.skip(f"{suite} not built (make -C tests/compat; needs /root/reference at build time)")
    env = {k: v for k, v in os.environ.items() if not k.startswith("AUTOSAGE_")}
    env["TMPDIR"] = str(tmp_path)
    r = subprocess.run([exe], cwd=str(tmp_path), env=env, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    m = re.search(r"test cases: (\d+) \| passed: (\d+) \| failed: (\d+)", out)
    assert m, out[-3000:]
    total, passed, failed = (int(x) for x in m.groups())
    assert r.returncode == 0 and failed == 0 and passed == total > 0, out[-6000:]
    return total


@pytest.mark.parametrize("suite", HOST_SUITES)
def test_reference_suite_host(suite, tmp_path):
    _run(suite, tmp_path)


@pytest.mark.gpu
@pytest.mark.parametrize("suite", GPU_SUITES)
def test_reference_suite_gpu(suite, tmp_path):
    _run(suite, tmp_path)
