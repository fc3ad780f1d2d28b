import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); parity tests proper")


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(autouse=True)
def _clean_autosage_env(monkeypatch):
    """Tests set AUTOSAGE_* knobs explicitly; never inherit them.  One knob
    is set for every test: AUTOSAGE_DEV_MIX_MIN_WORK=0 scans the dense
    operand for Inf/NaN at every size, so the small parity graphs exercise
    the ALU re-bias widening the large workloads run (by default small
    products skip the scan and widen on the XU only; the two give the same
    bits -- tests/test_gpu_kernels.py::test_small_work_scan_rule_keeps_bits)."""
    for k in list(os.environ):
        if k.startswith("AUTOSAGE_"):
            monkeypatch.delenv(k, raising=False)
    monkeypatch.setenv("AUTOSAGE_DEV_MIX_MIN_WORK", "0")
    yield
