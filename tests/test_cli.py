"""autosage-bench CLI (paper_2511_17594_b200/cli.py), mirroring
proj/tests/test_cli.cpp: subcommands, CSV schemas, sidecar, exit codes."""
import csv
import json
import os

import numpy as np
import pytest

import paper_2511_17594_b200 as asb
from paper_2511_17594_b200 import cli


def rows_of(path):
    with open(path) as fh:
        return list(csv.reader(fh))


def test_gen_shapes_and_closed_form_nnz(tmp_path):
    """proj/tests/test_cli.cpp:101-111: hubfixed nnz = hubs*hub_deg + (n-hubs)*other_deg."""
    out = str(tmp_path / "hf.ascr")
    assert cli.main(["gen", "hubfixed", "--n", "2000", "--hubs", "1", "--hub-deg", "500",
                     "--other-deg", "8", "--seed", "3", "--out", out]) == cli.EXIT_OK
    m = asb.load_csr(out)
    assert m.nnz == 500 + 1999 * 8 and asb.validate(m) is None
    out2 = str(tmp_path / "hs.ascr")
    assert cli.main(["gen", "hubskew", "--n", "3000", "--k", "4", "--hub-frac", "0.1", "--factor", "16",
                     "--out", out2]) == cli.EXIT_OK
    d = asb.load_csr(out2).degrees()
    assert set(np.unique(d)) <= {4, 64}
    out3 = str(tmp_path / "er.ascr")
    assert cli.main(["gen", "er", "--n", "1000", "--p", "0.01", "--out", out3]) == cli.EXIT_OK
    m3 = asb.load_csr(out3)
    assert asb.validate(m3) is None and 5000 < m3.nnz < 15000


def test_usage_and_io_exit_codes(tmp_path):
    assert cli.main(["bench"]) == cli.EXIT_USAGE                      # missing required options
    assert cli.main(["nope"]) == cli.EXIT_USAGE
    assert cli.main(["bench", "--graph", str(tmp_path / "missing.ascr"),
                     "--out", str(tmp_path / "o.csv")]) == cli.EXIT_IO
    assert cli.main(["--help"]) == cli.EXIT_OK


@pytest.mark.gpu
def test_bench_sweep_ablate_attention_replay(tmp_path, monkeypatch):
    g = str(tmp_path / "hub.ascr")
    assert cli.main(["gen", "hubfixed", "--n", "3000", "--hubs", "2", "--hub-deg", "2500",
                     "--other-deg", "12", "--out", g]) == 0
    cache = str(tmp_path / "sched.cache")
    out = str(tmp_path / "bench.csv")
    assert cli.main(["bench", "--graph", g, "--op", "spmm", "--f", "32,64", "--iters", "3",
                     "--warmups", "1", "--cache", cache, "--out", out]) == 0
    r = rows_of(out)
    assert r[0] == ["dataset", "F", "op", "choice", "baseline_ms", "chosen_ms", "speedup"]
    assert [x[1] for x in r[1:]] == ["32", "64"] and all(x[0] == "hub" for x in r[1:])
    assert all(x[3] in ("autosage", "baseline") for x in r[1:])
    meta = json.load(open(out + ".meta.json"))
    assert meta["command"] == "bench" and meta["config"]["f_list"] == [32, 64]
    assert meta["device"]["device_sig"].startswith("NVIDIA") and "probe" in meta["config"]
    assert meta["versions"]["sm"].startswith("sm_") and meta["versions"]["torch"]

    out = str(tmp_path / "sddmm.csv")
    assert cli.main(["bench", "--graph", g, "--op", "sddmm", "--f", "64", "--iters", "3",
                     "--cache", cache, "--out", out]) == 0
    assert rows_of(out)[1][2] == "sddmm"

    out = str(tmp_path / "split.csv")
    assert cli.main(["sweep-split", "--graph", g, "--f", "64", "--thresholds", "64,1024",
                     "--iters", "3", "--out", out]) == 0
    r = rows_of(out)
    assert r[0] == ["dataset", "F", "threshold", "baseline_ms", "hubsplit_ms", "speedup"]
    assert [x[2] for x in r[1:]] == ["64", "1024"]

    out = str(tmp_path / "ablate.csv")
    assert cli.main(["ablate-vec", "--graph", g, "--f", "64,30", "--iters", "3", "--out", out]) == 0
    r = rows_of(out)
    assert r[0] == ["dataset", "F", "op", "variant", "off_ms", "on_ms", "speedup"]
    assert r[2][-1] == "ineligible" and r[1][3].startswith("spmm:")

    out = str(tmp_path / "att.csv")
    acache = str(tmp_path / "att.cache")
    assert cli.main(["attention", "--graph", g, "--f", "32", "--iters", "2", "--cache", acache,
                     "--out", out]) == 0
    r = rows_of(out)
    assert r[0][:2] == ["dataset", "phase"] and [x[1] for x in r[1:]] == ["cold", "warm", "replay"]
    assert int(r[1][8]) > 0 and r[2][8] == "0" and r[3][8] == "0"   # probes only when cold
    assert r[3][6] == "replayed" and r[3][7] == "replayed"

    assert cli.main(["replay", "--cache", cache, "--graph", g, "--op", "spmm", "--f", "64",
                     "--iters", "2"]) == 0
    # strict replay miss -> exit 3 (autosage_bench.cpp:733-736)
    assert cli.main(["replay", "--cache", cache, "--graph", g, "--op", "spmm", "--f", "48",
                     "--strict", "--iters", "2"]) == cli.EXIT_REPLAY_MISS
