"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the B200 library.

Two checkers, both loaded through ctypes:

* ``port``: oracle/_oracle.so, the plain-C restatement of the reference
  algorithm in oracle/oracle.c (each function cites reference file:line);
* ``ref``: oracle/_ref/libautosage_ref.so, the reference library itself,
  compiled from /root/reference/proj/src by oracle/Makefile (namespace
  renamed to autosage_ref) with the extern "C" shim oracle/ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker
or the timed CPU baseline -- never as the thing measured or shipped.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(HERE, "_oracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libautosage_ref.so")

vp, u64, dbl = C.c_void_p, C.c_uint64, C.c_double


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class orc_features(C.Structure):
    _fields_ = [("n_rows", u64), ("n_cols", u64), ("nnz", u64), ("deg_p25", u64),
                ("deg_p50", u64), ("deg_p75", u64), ("deg_p90", u64), ("deg_p99", u64),
                ("deg_max", u64), ("mean_degree", dbl), ("heavy_row_fraction", dbl),
                ("empty_row_fraction", dbl), ("hub_threshold", u64)]


class orc_variant(C.Structure):
    _fields_ = [("op", C.c_int), ("mapping", C.c_int), ("f_tile", u64),
                ("rows_per_chunk", u64), ("vectorized", C.c_int), ("hub_threshold", u64)]


class orc_timed_stats(C.Structure):
    _fields_ = [("median_ms", dbl), ("completed", C.c_int), ("capped", C.c_int),
                ("launches", C.c_int), ("max_run_ms", dbl)]


_port = None
_ref = None


def port():
    """The C restatement (always available once built)."""
    global _port
    if _port is None:
        if not os.path.exists(PORT_PATH):
            raise ImportError(f"{PORT_PATH} not built (make -C oracle)")
        lib = C.CDLL(PORT_PATH)
        lib.orc_graph_sig.restype = u64
        lib.orc_graph_sig.argtypes = [vp, vp, u64, u64, u64]
        lib.orc_estimate_cost.restype = dbl
        lib.orc_estimate_cost.argtypes = [C.POINTER(orc_variant), C.POINTER(orc_features), u64,
                                          dbl, dbl, u64]
        lib.orc_sample_row_indices.restype = u64
        lib.orc_sample_row_indices.argtypes = [vp, u64, dbl, u64, vp]
        lib.orc_slice_rows.restype = u64
        lib.orc_slice_rows.argtypes = [vp, vp, vp, vp, u64, vp, vp, vp]
        for name, args in {
            "orc_spmm_baseline": [vp, vp, vp, u64, vp, u64, vp],
            "orc_spmm_hubsplit": [vp, vp, vp, u64, vp, u64, u64, vp],
            "orc_spmm_blocked": [vp, vp, vp, u64, vp, u64, u64, vp, C.c_uint32, vp],
            "orc_sddmm": [vp, vp, u64, vp, vp, u64, u64, C.c_int, vp],
            "orc_row_softmax": [vp, u64, vp, vp],
            "orc_attention": [vp, vp, u64, vp, vp, u64, vp, u64, u64, C.c_int, u64, vp],
            "orc_extract_features": [vp, u64, u64, u64, C.POINTER(orc_features)],
            "orc_partition_rows": [vp, u64, C.c_uint32, vp],
            "orc_transpose": [vp, vp, u64, u64, vp, vp, vp],
            "orc_row_softmax_backward": [vp, u64, vp, vp, vp],
        }.items():
            fn = getattr(lib, name)
            fn.restype = None
            fn.argtypes = args
        lib.orc_shortlist.restype = C.c_int
        lib.orc_shortlist.argtypes = [C.POINTER(orc_features), u64, C.c_int, dbl, dbl, u64,
                                      C.POINTER(orc_variant)]
        lib.orc_gen_powerlaw_degrees.restype = C.c_int
        lib.orc_gen_powerlaw_degrees.argtypes = [u64, u64, u64, dbl, u64, u64, u64, vp]
        lib.orc_gen_powerlaw_columns.restype = None
        lib.orc_gen_powerlaw_columns.argtypes = [u64, u64, u64, vp, vp, vp]
        lib.orc_fill_uniform.restype = None
        lib.orc_fill_uniform.argtypes = [vp, u64, u64]
        lib.orc_time_kernel_policy.restype = C.c_int
        lib.orc_time_kernel_policy.argtypes = [C.POINTER(dbl), C.c_int, C.c_int, dbl, dbl,
                                               C.POINTER(orc_timed_stats)]
        _port = lib
    return _port


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    """The reference library itself (None-safe check with ref_available())."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_PATH):
            raise ImportError(f"{REF_PATH} not built (needs /root/reference; make -C oracle)")
        lib = C.CDLL(REF_PATH)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_graph_new.restype = vp
        lib.ref_graph_new.argtypes = [vp, vp, vp, u64, u64, u64]
        lib.ref_graph_free.argtypes = [vp]
        lib.ref_dense_new.restype = vp
        lib.ref_dense_new.argtypes = [vp, u64, u64]
        lib.ref_dense_free.argtypes = [vp]
        sigs = {
            "ref_spmm_baseline": [vp, vp, vp],
            "ref_spmm_dispatch": [C.c_char_p, vp, vp, u64, vp, C.POINTER(C.c_int)],
            "ref_sddmm_baseline": [vp, vp, vp, vp],
            "ref_sddmm_dispatch": [C.c_char_p, vp, vp, vp, u64, vp],
            "ref_row_softmax": [vp, u64, vp],
            "ref_graph_sig": [vp, C.POINTER(u64)],
            "ref_extract_features": [vp, u64, C.POINTER(dbl)],
            "ref_sample_row_indices": [vp, dbl, u64, vp, C.POINTER(u64)],
            "ref_shortlist": [vp, u64, C.c_int, dbl, dbl, u64, C.c_char_p, u64],
            "ref_estimate_cost": [vp, C.c_char_p, u64, dbl, dbl, u64, C.POINTER(dbl)],
            "ref_record_line": [C.c_char_p, u64, u64, C.c_int, C.c_char_p, dbl, dbl, dbl, u64,
                                C.c_char_p, C.c_char_p, u64],
            "ref_gen": [C.c_int, u64, dbl, u64, u64, u64, u64, u64, C.POINTER(vp), C.POINTER(vp),
                        C.POINTER(vp), C.POINTER(u64), C.POINTER(u64), C.POINTER(u64)],
            "ref_decide": [vp, vp, vp, C.c_int, C.c_char_p, u64, C.POINTER(dbl)],
            "ref_attention": [vp, vp, vp, vp, vp],
        }
        for name, args in sigs.items():
            fn = getattr(lib, name)
            fn.restype = C.c_int
            fn.argtypes = args
        lib.ref_free.argtypes = [vp]
        lib.ref_default_workers.restype = u64
        _ref = lib
    return _ref


def _rcheck(rc):
    if rc != 0:
        raise RuntimeError("reference: " + ref().ref_last_error().decode())


# ---------------------------------------------------------------------------
# C-restatement wrappers (numpy in, numpy out)
# ---------------------------------------------------------------------------
def spmm_baseline(m, b: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(b, dtype=np.float32)
    f = b.shape[1]
    c = np.empty((m.n_rows, f), dtype=np.float32)
    port().orc_spmm_baseline(_ptr(m.rowptr), _ptr(m.colind), _ptr(m.val if m.has_values() else None),
                             m.n_rows, _ptr(b), f, _ptr(c))
    return c


def spmm_hubsplit(m, b: np.ndarray, hub_t: int) -> np.ndarray:
    b = np.ascontiguousarray(b, dtype=np.float32)
    f = b.shape[1]
    c = np.empty((m.n_rows, f), dtype=np.float32)
    port().orc_spmm_hubsplit(_ptr(m.rowptr), _ptr(m.colind), _ptr(m.val if m.has_values() else None),
                             m.n_rows, _ptr(b), f, hub_t, _ptr(c))
    return c


def spmm_blocked(m, b: np.ndarray, cuts, hub_t: int = 0) -> np.ndarray:
    """Column-blocked SpMM restatement (segment accumulators carried across
    ascending column blocks); equals spmm_baseline / spmm_hubsplit bit for bit."""
    b = np.ascontiguousarray(b, dtype=np.float32)
    cuts = np.ascontiguousarray(cuts, dtype=np.uint64)
    c = np.empty((m.n_rows, b.shape[1]), dtype=np.float32)
    port().orc_spmm_blocked(_ptr(m.rowptr), _ptr(m.colind), _ptr(m.val if m.has_values() else None), m.n_rows,
                            _ptr(b), b.shape[1], hub_t, _ptr(cuts), cuts.size - 1, _ptr(c))
    return c


def sddmm(m, x: np.ndarray, y: np.ndarray, f_tile: int = 64, vec: bool = False) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.ascontiguousarray(y, dtype=np.float32)
    out = np.empty(max(m.nnz, 1), dtype=np.float32)
    port().orc_sddmm(_ptr(m.rowptr), _ptr(m.colind), m.n_rows, _ptr(x), _ptr(y), x.shape[1],
                     f_tile, 1 if vec else 0, _ptr(out))
    return out[:m.nnz]


def row_softmax(m, vals: Optional[np.ndarray] = None) -> np.ndarray:
    vin = np.ascontiguousarray(m.val if vals is None else vals, dtype=np.float32)
    out = vin.copy()
    port().orc_row_softmax(_ptr(m.rowptr), m.n_rows, _ptr(vin), _ptr(out))
    return out


def transpose(m):
    """(A^T as (rowptr, colind, val-or-None), perm): stable counting sort by
    column; perm[k] = source entry of transposed entry k."""
    rp = np.zeros(m.n_cols + 1, dtype=np.uint64)
    ci = np.zeros(max(m.nnz, 1), dtype=np.uint32)
    perm = np.zeros(max(m.nnz, 1), dtype=np.uint32)
    port().orc_transpose(_ptr(m.rowptr), _ptr(m.colind), m.n_rows, m.n_cols, _ptr(rp), _ptr(ci),
                         _ptr(perm))
    perm = perm[:m.nnz]
    val = m.val[perm] if m.has_values() else None
    return (rp, ci[:m.nnz], val), perm


def row_softmax_backward(m, p: np.ndarray, g: np.ndarray) -> np.ndarray:
    p = np.ascontiguousarray(p, dtype=np.float32)
    g = np.ascontiguousarray(g, dtype=np.float32)
    out = np.zeros(max(m.nnz, 1), dtype=np.float32)
    port().orc_row_softmax_backward(_ptr(m.rowptr), m.n_rows, _ptr(p), _ptr(g), _ptr(out))
    return out[:m.nnz]


def attention(m, q, k, v, sddmm_ft=64, sddmm_vec=False, spmm_hub_t=0) -> np.ndarray:
    q, k, v = (np.ascontiguousarray(t, dtype=np.float32) for t in (q, k, v))
    out = np.empty((m.n_rows, v.shape[1]), dtype=np.float32)
    port().orc_attention(_ptr(m.rowptr), _ptr(m.colind), m.n_rows, _ptr(q), _ptr(k), q.shape[1],
                         _ptr(v), v.shape[1], sddmm_ft, 1 if sddmm_vec else 0, spmm_hub_t,
                         _ptr(out))
    return out


def graph_sig(m) -> int:
    return int(port().orc_graph_sig(_ptr(m.rowptr), _ptr(m.colind), m.n_rows, m.n_cols, m.nnz))


def extract_features(m, hub_t: int = 256) -> dict:
    f = orc_features()
    port().orc_extract_features(_ptr(m.rowptr), m.n_rows, m.n_cols, hub_t, C.byref(f))
    return {n: getattr(f, n) for n, _ in orc_features._fields_}


def sample_row_indices(m, frac: float, min_rows: int) -> np.ndarray:
    rows = np.zeros(max(m.n_rows, 1), dtype=np.uint64)
    n = port().orc_sample_row_indices(_ptr(m.rowptr), m.n_rows, frac, min_rows, _ptr(rows))
    if n == (1 << 64) - 1:
        raise ValueError("sample: frac must be in (0,1]")
    return rows[:n].copy()


def slice_rows(m, rows: np.ndarray):
    rows = np.ascontiguousarray(rows, dtype=np.uint64)
    rp = np.zeros(rows.size + 1, dtype=np.uint64)
    nnz = int(sum(m.degree(int(r)) for r in rows))
    ci = np.zeros(max(nnz, 1), dtype=np.uint32)
    va = np.zeros(max(nnz, 1), dtype=np.float32) if m.has_values() else None
    port().orc_slice_rows(_ptr(m.rowptr), _ptr(m.colind), _ptr(m.val if m.has_values() else None),
                          _ptr(rows), rows.size, _ptr(rp), _ptr(ci), _ptr(va))
    return rp, ci[:nnz], None if va is None else va[:nnz]


def shortlist(feat: dict, f: int, op: int, bw: float, flops: float, cores: int):
    cf = orc_features(*[feat[n] for n, _ in orc_features._fields_])
    out = (orc_variant * 36)()
    n = port().orc_shortlist(C.byref(cf), f, op, bw, flops, cores, out)
    return [(out[i].op, out[i].mapping, out[i].f_tile, out[i].rows_per_chunk,
             bool(out[i].vectorized), out[i].hub_threshold) for i in range(n)]


def estimate_cost(variant: tuple, feat: dict, f: int, bw: float, flops: float, cores: int):
    cf = orc_features(*[feat[n] for n, _ in orc_features._fields_])
    cv = orc_variant(*variant)
    return port().orc_estimate_cost(C.byref(cv), C.byref(cf), f, bw, flops, cores)


def time_kernel_policy(script, iters: int, cap_ms: float, warmup_ms: float = 0.0):
    arr = (dbl * max(len(script), 1))(*script)
    st = orc_timed_stats()
    rc = port().orc_time_kernel_policy(arr, len(script), iters, cap_ms, warmup_ms, C.byref(st))
    if rc == -1:
        raise ValueError("time_kernel: iters must be >= 1")
    if rc == -2:
        raise RuntimeError("FakeTimer: script exhausted")
    return {"median_ms": st.median_ms, "completed": st.completed, "capped": bool(st.capped),
            "launches": st.launches, "max_run_ms": st.max_run_ms}


def partition_rows(rowptr: np.ndarray, g: int) -> np.ndarray:
    rowptr = np.ascontiguousarray(rowptr, dtype=np.uint64)
    cuts = np.zeros(g + 1, dtype=np.uint64)
    port().orc_partition_rows(_ptr(rowptr), rowptr.size - 1, g, _ptr(cuts))
    return cuts


# ---------------------------------------------------------------------------
# Input generators (oracle/gen.c): the bench workload without the package
# ---------------------------------------------------------------------------
class HostCsr:
    """A host CSR with the attributes the oracle functions read (the same
    duck type as the package's CsrMatrix, so the reference arm and the tests
    can build inputs without importing the B200 package)."""

    def __init__(self, n_rows, n_cols, rowptr, colind, val=None):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.rowptr = np.ascontiguousarray(rowptr, dtype=np.uint64)
        self.colind = np.ascontiguousarray(colind, dtype=np.uint32)
        self.val = None if val is None else np.ascontiguousarray(val, dtype=np.float32)

    @property
    def nnz(self) -> int:
        return int(self.colind.size)

    def has_values(self) -> bool:
        return self.val is not None and self.val.size > 0


def gen_powerlaw(n_rows: int, n_cols: int, nnz_target: int, alpha: float, d_min: int, d_max: int,
                 seed: int, with_values: bool = True) -> HostCsr:
    """Same bytes as the package's gen_powerlaw (checked in test_oracle)."""
    rowptr = np.zeros(n_rows + 1, dtype=np.uint64)
    if port().orc_gen_powerlaw_degrees(n_rows, n_cols, nnz_target, alpha, d_min, d_max, seed,
                                       _ptr(rowptr)) != 0:
        raise ValueError("gen_powerlaw: bad arguments")
    nnz = int(rowptr[-1])
    colind = np.empty(nnz, dtype=np.uint32)
    val = np.empty(nnz, dtype=np.float32) if with_values else None
    port().orc_gen_powerlaw_columns(n_rows, n_cols, seed, _ptr(rowptr), _ptr(colind), _ptr(val))
    return HostCsr(n_rows, n_cols, rowptr, colind, val)


def fill_uniform(n: int, seed: int, shape=None) -> np.ndarray:
    """U[-1, 1) f32, the same bytes as the package's fill_uniform."""
    out = np.empty(n, dtype=np.float32)
    port().orc_fill_uniform(_ptr(out), n, seed)
    return out.reshape(shape) if shape is not None else out


# ---------------------------------------------------------------------------
# Reference-library wrappers
# ---------------------------------------------------------------------------
class RefGraph:
    """A CsrMatrix living inside the reference library (autosage_ref::)."""

    def __init__(self, m):
        self.m = m
        self.h = ref().ref_graph_new(_ptr(m.rowptr), _ptr(m.colind) if m.nnz else None,
                                     _ptr(m.val if m.has_values() else None), m.n_rows, m.n_cols,
                                     m.nnz)

    def __del__(self):
        try:
            ref().ref_graph_free(self.h)
        except Exception:
            pass


class RefDense:
    def __init__(self, a: np.ndarray):
        a = np.ascontiguousarray(a, dtype=np.float32)
        self.shape = a.shape
        self.h = ref().ref_dense_new(_ptr(a), a.shape[0], a.shape[1])

    def __del__(self):
        try:
            ref().ref_dense_free(self.h)
        except Exception:
            pass


def ref_spmm_baseline(g: RefGraph, b: RefDense) -> np.ndarray:
    out = np.empty((g.m.n_rows, b.shape[1]), dtype=np.float32)
    _rcheck(ref().ref_spmm_baseline(g.h, b.h, _ptr(out)))
    return out


def ref_spmm_dispatch(variant: str, g: RefGraph, b: RefDense, workers: int = 0,
                      out: Optional[np.ndarray] = None):
    vec = C.c_int()
    if out is None:
        out = np.empty((g.m.n_rows, b.shape[1]), dtype=np.float32)
    _rcheck(ref().ref_spmm_dispatch(variant.encode(), g.h, b.h, workers, _ptr(out), C.byref(vec)))
    return out, bool(vec.value)


def ref_sddmm_baseline(g: RefGraph, x: RefDense, y: RefDense) -> np.ndarray:
    out = np.empty(max(g.m.nnz, 1), dtype=np.float32)
    _rcheck(ref().ref_sddmm_baseline(g.h, x.h, y.h, _ptr(out)))
    return out[:g.m.nnz]


def ref_sddmm_dispatch(variant: str, g: RefGraph, x: RefDense, y: RefDense,
                       workers: int = 0) -> np.ndarray:
    out = np.empty(max(g.m.nnz, 1), dtype=np.float32)
    _rcheck(ref().ref_sddmm_dispatch(variant.encode(), g.h, x.h, y.h, workers, _ptr(out)))
    return out[:g.m.nnz]


def ref_row_softmax(g: RefGraph, workers: int = 0) -> np.ndarray:
    out = np.empty(max(g.m.nnz, 1), dtype=np.float32)
    _rcheck(ref().ref_row_softmax(g.h, workers, _ptr(out)))
    return out[:g.m.nnz]


def ref_graph_sig(g: RefGraph) -> int:
    out = u64()
    _rcheck(ref().ref_graph_sig(g.h, C.byref(out)))
    return out.value


def ref_extract_features(g: RefGraph, hub_t: int = 256) -> dict:
    arr = (dbl * 14)()
    _rcheck(ref().ref_extract_features(g.h, hub_t, arr))
    names = ["n_rows", "n_cols", "nnz", "deg_p25", "deg_p50", "deg_p75", "deg_p90", "deg_p99",
             "deg_max", "mean_degree", "heavy_row_fraction", "empty_row_fraction",
             "hub_threshold"]
    return {n: arr[i] for i, n in enumerate(names)}


def ref_sample_row_indices(g: RefGraph, frac: float, min_rows: int) -> np.ndarray:
    rows = np.zeros(max(g.m.n_rows, 1), dtype=np.uint64)
    n = u64()
    _rcheck(ref().ref_sample_row_indices(g.h, frac, min_rows, _ptr(rows), C.byref(n)))
    return rows[:n.value].copy()


def ref_shortlist(g: RefGraph, f: int, op: int, bw: float, flops: float, cores: int):
    buf = C.create_string_buffer(8192)
    _rcheck(ref().ref_shortlist(g.h, f, op, bw, flops, cores, buf, 8192))
    return [s for s in buf.value.decode().split("\n") if s]


def ref_record_line(dev, sig, f, op, choice, t_b, t_star, alpha, ts, tool) -> str:
    buf = C.create_string_buffer(2048)
    _rcheck(ref().ref_record_line(dev.encode(), sig, f, op, choice.encode(), t_b, t_star, alpha,
                                  ts, tool.encode(), buf, 2048))
    return buf.value.decode()


def ref_gen(kind: str, n: int, p: float = 0.0, k: int = 0, hubs: int = 0, hub_deg: int = 0,
            other_deg: int = 0, seed: int = 1, hub_factor: int = 64):
    """gen_er / gen_hubskew / gen_hub_fixed from the reference (returns arrays)."""
    kinds = {"er": 0, "hubskew": 1, "hub_fixed": 2}
    rp, ci, va = vp(), vp(), vp()
    nr, nc, nz = u64(), u64(), u64()
    hubs_arg = hub_factor if kind == "hubskew" else hubs
    _rcheck(ref().ref_gen(kinds[kind], n, p, k, hubs_arg, hub_deg, other_deg, seed, C.byref(rp),
                          C.byref(ci), C.byref(va), C.byref(nr), C.byref(nc), C.byref(nz)))
    n_rows, n_cols, nnz = nr.value, nc.value, nz.value
    rowptr = np.ctypeslib.as_array(C.cast(rp, C.POINTER(C.c_uint64)), (n_rows + 1,)).copy()
    colind = (np.ctypeslib.as_array(C.cast(ci, C.POINTER(C.c_uint32)), (nnz,)).copy()
              if nnz else np.zeros(0, dtype=np.uint32))
    val = None
    if va.value:
        val = (np.ctypeslib.as_array(C.cast(va, C.POINTER(C.c_float)), (nnz,)).copy()
               if nnz else np.zeros(0, dtype=np.float32))
    for ptr in (rp, ci, va):
        if ptr.value:
            ref().ref_free(ptr)
    return n_rows, n_cols, rowptr, colind, val


def ref_decide(g: RefGraph, x: Optional[RefDense], y: RefDense, op: int):
    buf = C.create_string_buffer(256)
    probe_ms = dbl()
    _rcheck(ref().ref_decide(g.h, x.h if x is not None else None, y.h, op, buf, 256,
                             C.byref(probe_ms)))
    return buf.value.decode(), probe_ms.value


def ref_attention(g: RefGraph, q: RefDense, k: RefDense, v: RefDense) -> np.ndarray:
    out = np.empty((g.m.n_rows, v.shape[1]), dtype=np.float32)
    _rcheck(ref().ref_attention(g.h, q.h, k.h, v.h, _ptr(out)))
    return out


def ref_default_workers() -> int:
    return int(ref().ref_default_workers())
