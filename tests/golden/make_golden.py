#!/usr/bin/env python3
"""Regenerate tests/golden/*.npz from the REFERENCE LIBRARY ITSELF.

Runs only where /root/reference exists (oracle/Makefile builds
oracle/_ref/libautosage_ref.so from its untouched sources).  The fixtures pin
the C restatement (oracle/oracle.c) and, through it, the B200 kernels on
machines where the reference library is unavailable.  Inputs come from the
reference's own generators (gen_er / gen_hubskew / gen_hub_fixed) and seeded
U(-1,1) dense operands; outputs from its kernels, row_softmax, graph_sig,
extract_features, sample_row_indices and shortlist.

  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2511_17594_b200 as asb  # noqa: E402


def dense(seed, rows, cols):
    """U[-1,1) from the counter-based generator (stable across numpy versions)."""
    return asb.fill_uniform(rows * cols, seed, (rows, cols))


CASES = [
    # name, generator kwargs, F list, hubsplit thresholds
    ("er_small", dict(kind="er", n=300, p=0.03, seed=3), [1, 33, 64], [1, 8]),
    ("hubskew", dict(kind="hubskew", n=800, k=4, p=0.15, seed=11), [16, 20], [64, 256]),
    ("hub_fixed", dict(kind="hub_fixed", n=2600, hubs=2, hub_deg=2500, other_deg=5, seed=9),
     [8, 12], [128, 2048]),
]


def main():
    if not oracle.ref_available():
        sys.exit("reference library not built (make -C oracle needs /root/reference)")
    for name, gk, fs, hubts in CASES:
        kind = gk.pop("kind")
        n_rows, n_cols, rp, ci, va = oracle.ref_gen(kind, **gk)
        m = asb.CsrMatrix(n_rows, n_cols, rp, ci, va)
        rg = oracle.RefGraph(m)
        out = {"rowptr": rp, "colind": ci, "val": va, "shape": np.array([n_rows, n_cols])}
        out["graph_sig"] = np.array([oracle.ref_graph_sig(rg)], dtype=np.uint64)
        feats = oracle.ref_extract_features(rg, 256)
        out["features"] = np.array([feats[k] for k in sorted(feats)], dtype=np.float64)
        out["sample_002_512"] = oracle.ref_sample_row_indices(rg, 0.02, 512)
        out["sample_01_16"] = oracle.ref_sample_row_indices(rg, 0.1, 16)
        for f in fs:
            b = dense(100 + f, n_cols, f)
            x = dense(200 + f, n_rows, f)
            rb, rx = oracle.RefDense(b), oracle.RefDense(x)
            out[f"spmm_F{f}"] = oracle.ref_spmm_baseline(rg, rb)
            for t in hubts:
                v = f"spmm:hubsplit:ft=64:rpc=4:vec=0:hubt={t}"
                out[f"hub{t}_F{f}"] = oracle.ref_spmm_dispatch(v, rg, rb)[0]
            out[f"sddmm_F{f}"] = oracle.ref_sddmm_baseline(rg, rx, rb)
            for ft in (32, 64):
                v = f"sddmm:rowparallel:ft={ft}:rpc=4:vec=1:hubt=256"
                out[f"sddmm_vec_ft{ft}_F{f}"] = oracle.ref_sddmm_dispatch(v, rg, rx, rb)
            sl = "\n".join(oracle.ref_shortlist(rg, f, 0, 20e9, 40e9, 4))
            out[f"shortlist_spmm_F{f}"] = np.frombuffer(sl.encode(), dtype=np.uint8)
        sm = oracle.ref_row_softmax(rg)
        out["softmax"] = sm
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print("wrote", name, {k: v.shape for k, v in out.items() if hasattr(v, "shape")})


if __name__ == "__main__":
    main()
