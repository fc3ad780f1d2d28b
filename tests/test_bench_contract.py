"""bench.py's reference arm on CPU (it needs no GPU): the driver's JSON-line
contract -- exactly one line on stdout, the metric / unit / config of our own
arm, `impl: reference`, a `cpu_baseline` describing the run and an `e2e`
with zero copy bytes -- and the helpers that define the bench's bytes."""
import json
import os
import subprocess
import sys

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_contract_line():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["PYTHONPATH"] = ROOT
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                        "--steps", "2", "--warmup", "3"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "config", "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3
    assert d["metric"] == bench.metric_name("c1", 64) and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["config"]["workload"] == bench.workload_name("c1", 64)
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["sample"] and cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_bench_byte_models():
    """proj/src/cost.cpp:21-27 (gather model) and the compulsory floor."""
    n, nnz, f = 1000, 50_000, 64
    assert bench.gather_bytes("spmm", n, nnz, f) == 8 * nnz + 4 * nnz * f + 4 * n * f + 8 * (n + 1)
    assert bench.gather_bytes("sddmm", n, nnz, f) == 8 * nnz + 8 * nnz * f + 4 * nnz
    assert bench.compulsory_bytes("spmm", n, n, nnz, f) == 8 * (n + 1) + 8 * nnz + 4 * n * f + 4 * n * f
    assert bench.compulsory_bytes("sddmm", n, n, nnz, f) == 8 * (n + 1) + 4 * nnz + 8 * n * f + 4 * nnz
