"""Test helpers: seeded CSR / dense generators and comparison utilities
(the reference's proj/tests/test_util.hpp restated for numpy)."""
from __future__ import annotations

import numpy as np

import paper_2511_17594_b200 as asb


def close(got, want, rel=1e-5, abs_=1e-6) -> bool:
    """|got - want| <= abs + rel*|want| (proj/tests/test_util.hpp:28-30)."""
    return abs(float(got) - float(want)) <= abs_ + rel * abs(float(want))


def max_err(got, want, rel=1e-5, abs_=1e-6) -> float:
    """Worst |got-want| / (abs + rel*|want|); <= 1.0 is within tolerance."""
    got = np.asarray(got, dtype=np.float64).ravel()
    want = np.asarray(want, dtype=np.float64).ravel()
    if got.shape != want.shape:
        return 1e30
    if got.size == 0:
        return 0.0
    return float(np.max(np.abs(got - want) / (abs_ + rel * np.abs(want))))


def bits(a) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    return a.view(np.uint32)


def bit_equal(a, b) -> bool:
    a = np.asarray(a, dtype=np.float32)
    b = np.asarray(b, dtype=np.float32)
    return a.shape == b.shape and np.array_equal(bits(a), bits(b))


def n_bit_diff(a, b) -> int:
    return int(np.sum(bits(a) != bits(b)))


def ulp_diff(a, b) -> int:
    """Max distance in f32 units-in-last-place (finite values)."""
    ia = bits(a).astype(np.int64)
    ib = bits(b).astype(np.int64)
    ia = np.where(ia >= 1 << 31, (1 << 31) - ia, ia)
    ib = np.where(ib >= 1 << 31, (1 << 31) - ib, ib)
    return int(np.max(np.abs(ia - ib))) if ia.size else 0


def random_csr(rng, n_rows, n_cols, max_deg, with_values=True, val_lo=-1.0, val_hi=1.0):
    """Degrees U[0, max_deg], distinct sorted columns, values U[lo, hi)
    (proj/tests/test_util.hpp:45-66)."""
    deg = rng.integers(0, min(max_deg, n_cols) + 1, size=n_rows)
    return csr_from_degrees(rng, n_rows, n_cols, deg, with_values, val_lo, val_hi)


def csr_from_degrees(rng, n_rows, n_cols, deg, with_values=True, val_lo=-1.0, val_hi=1.0):
    deg = np.asarray(deg, dtype=np.int64)
    rowptr = np.zeros(n_rows + 1, dtype=np.uint64)
    rowptr[1:] = np.cumsum(deg)
    cols = [np.sort(rng.choice(n_cols, size=int(d), replace=False)) for d in deg]
    colind = np.concatenate(cols).astype(np.uint32) if cols else np.zeros(0, np.uint32)
    val = (rng.uniform(val_lo, val_hi, size=colind.size).astype(np.float32)
           if with_values else None)
    return asb.CsrMatrix(n_rows, n_cols, rowptr, colind, val)


def random_dense(rng, rows, cols):
    return rng.uniform(-1.0, 1.0, size=(rows, cols)).astype(np.float32)


def identity(n, with_values=False):
    return asb.CsrMatrix(n, n, np.arange(n + 1, dtype=np.uint64), np.arange(n, dtype=np.uint32),
                         np.ones(n, np.float32) if with_values else None)


def hub_graph(rng, n, hub_degs, other_deg, with_values=True):
    deg = np.full(n, other_deg, dtype=np.int64)
    deg[:len(hub_degs)] = hub_degs
    return csr_from_degrees(rng, n, n, deg, with_values)


def empty_rows(n_rows, n_cols):
    return asb.CsrMatrix(n_rows, n_cols, np.zeros(n_rows + 1, np.uint64), np.zeros(0, np.uint32),
                         None)


class FakeTimer:
    """Scripted ProbeTimer (proj/tests/test_util.hpp:172-189): returns the
    recorded values in call order, raises when the script runs dry."""

    def __init__(self, script, run_kernels=False):
        self.script = list(script)
        self.next = 0
        self.run_kernels = run_kernels

    def __call__(self, label, run):
        if self.run_kernels:
            run()
        if self.next >= len(self.script):
            raise RuntimeError("FakeTimer: script exhausted")
        v = self.script[self.next]
        self.next += 1
        return v

    def calls(self):
        return self.next


def cuda(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()
