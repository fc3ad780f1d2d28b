"""B200-native AutoSAGE: Python face of libautosage_b200.so.

The product is the C++/CUDA library behind ``include/autosage_b200.h``; this
module is a thin ctypes mirror of the reference's operator API
(/root/reference/proj/include/autosage/*.hpp) so callers and tests read like
the reference's own:

    spmm_baseline(a, b)            kernels.hpp:46-48
    spmm_rowparallel(a, b, v)      kernels.hpp:50-55
    spmm_hubsplit(a, b, v)         kernels.hpp:57-61
    sddmm_baseline(p, x, y)        kernels.hpp:63-66
    sddmm_rowparallel(p, x, y, v)  kernels.hpp:68-73
    row_softmax(m)                 kernels.hpp:75-77
    dispatch(v, a, b[, y])         kernels.hpp:79-85
    decide_spmm / decide_sddmm / spmm_auto / sddmm_auto     scheduler.hpp:71-87
    csr_attention_forward / attention_probe_breakdown        attention.hpp:19-25
    ScheduleCache, graph_sig, record_to_line/from_line       cache.hpp:23-91
    estimate_cost, shortlist, extract_features, validate     cost.hpp, csr.hpp
    time_kernel, ProbeConfig, ReplayPolicy, DeviceProfile    timing.hpp, ...

Host numpy operands use the library's host-buffer entry points (H2D, kernel,
D2H inside the call -- the reference's by-value convention); torch CUDA
tensors go straight to the device entry points.  Every operator runs on the
sm_100a kernels; nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _capi as _c
from ._capi import lib as _lib

__all__ = [
    "SPMM", "SDDMM", "BASELINE", "ROWPARALLEL", "HUBSPLIT", "DEFAULT_HUB_THRESHOLD",
    "InvalidArgument", "CacheError", "IoError", "ReplayMiss", "CudaError", "LogicError",
    "CsrMatrix", "KernelVariant", "KernelResult", "Graph", "GraphFeatures", "DeviceProfile",
    "ProbeConfig", "ReplayPolicy", "ScheduleKey", "CacheRecord", "ScheduleCache",
    "ScheduleContext", "ScheduleDecision", "TimedKernelStats", "variant_to_string",
    "variant_from_string", "vec4_eligible", "validate", "graph_sig", "extract_features",
    "sample_row_indices", "slice_rows", "estimate_cost", "shortlist", "time_kernel",
    "spmm_baseline", "spmm_rowparallel", "spmm_hubsplit", "sddmm_baseline",
    "sddmm_rowparallel", "row_softmax", "dispatch", "decide_spmm", "decide_sddmm",
    "spmm_auto", "sddmm_auto", "probe_launch_count", "reset_probe_launch_count",
    "decide_host", "csr_attention_forward", "attention_probe_breakdown", "partition_rows",
    "gen_powerlaw", "fill_uniform", "save_csr", "load_csr", "record_to_line",
    "record_from_line", "toolchain_tag", "kernel_launch_count", "LIB_PATH",
]

LIB_PATH = _c.LIB_PATH
SPMM, SDDMM = 0, 1
BASELINE, ROWPARALLEL, HUBSPLIT = 0, 1, 2
DEFAULT_HUB_THRESHOLD = 256
SOURCES = {0: "probed", 1: "cached", 2: "replayed", 3: "forced-env"}
PROBED, CACHED, REPLAYED, FORCED_ENV = 0, 1, 2, 3


# ---- errors (reference exception roles) --------------------------------------
class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class CacheError(RuntimeError):
    """CacheError, include/autosage/cache.hpp:16-18."""


class IoError(RuntimeError):
    """IoError, include/autosage/io.hpp:10-12."""


class ReplayMiss(RuntimeError):
    """ReplayMiss, include/autosage/cache.hpp:78-81."""


class CudaError(RuntimeError):
    pass


class LogicError(RuntimeError):
    pass


_ERRORS = {
    _c.AS_INVALID_ARGUMENT: InvalidArgument, _c.AS_CACHE_ERROR: CacheError,
    _c.AS_IO_ERROR: IoError, _c.AS_REPLAY_MISS: ReplayMiss, _c.AS_CUDA_ERROR: CudaError,
    _c.AS_OUT_OF_MEMORY: MemoryError, _c.AS_LOGIC_ERROR: LogicError,
    _c.AS_INTERNAL: RuntimeError,
}

_pending_exc: list = []


def _check(status: int) -> None:
    if _pending_exc:
        exc = _pending_exc.pop()
        _pending_exc.clear()
        raise exc
    if status != _c.AS_OK:
        msg = _lib.as_last_error().decode(errors="replace")
        raise _ERRORS.get(status, RuntimeError)(msg)


def kernel_launch_count() -> int:
    return int(_lib.as_kernel_launch_count())


def toolchain_tag() -> str:
    return _lib.as_toolchain_tag().decode()


# ---- host containers --------------------------------------------------------------
class CsrMatrix:
    """Host CSR (include/autosage/csr.hpp:24-45): u64 rowptr, u32 colind,
    optional f32 values (None = pattern-only, implicit 1.0)."""

    def __init__(self, n_rows: int, n_cols: int, rowptr, colind, val=None):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.rowptr = np.ascontiguousarray(rowptr, dtype=np.uint64)
        self.colind = np.ascontiguousarray(colind, dtype=np.uint32)
        self.val = None if val is None else np.ascontiguousarray(val, dtype=np.float32)

    @property
    def nnz(self) -> int:
        return int(self.colind.size)

    def has_values(self) -> bool:
        return self.val is not None and self.val.size > 0

    def degree(self, i: int) -> int:
        return int(self.rowptr[i + 1] - self.rowptr[i])

    def degrees(self) -> np.ndarray:
        return np.diff(self.rowptr).astype(np.int64)

    def row_cols(self, i: int) -> np.ndarray:
        return self.colind[int(self.rowptr[i]):int(self.rowptr[i + 1])]

    def row_vals(self, i: int) -> np.ndarray:
        return self.val[int(self.rowptr[i]):int(self.rowptr[i + 1])]

    def with_values(self, val) -> "CsrMatrix":
        return CsrMatrix(self.n_rows, self.n_cols, self.rowptr, self.colind, val)

    def __eq__(self, o) -> bool:
        if not isinstance(o, CsrMatrix):
            return NotImplemented
        hv = self.has_values(), o.has_values()
        return (self.n_rows == o.n_rows and self.n_cols == o.n_cols
                and np.array_equal(self.rowptr, o.rowptr)
                and np.array_equal(self.colind, o.colind) and hv[0] == hv[1]
                and (not hv[0] or np.array_equal(self.val.view(np.uint32), o.val.view(np.uint32))))


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclasses.dataclass
class KernelVariant:
    """KernelVariant, include/autosage/kernels.hpp:21-30 (defaults included)."""
    op: int = SPMM
    mapping: int = ROWPARALLEL
    f_tile: int = 64
    rows_per_chunk: int = 4
    vectorized: bool = False
    hub_threshold: int = DEFAULT_HUB_THRESHOLD

    def to_c(self) -> _c.as_variant:
        return _c.as_variant(int(self.op), int(self.mapping), int(self.f_tile),
                             int(self.rows_per_chunk), 1 if self.vectorized else 0,
                             int(self.hub_threshold))

    @staticmethod
    def from_c(v: _c.as_variant) -> "KernelVariant":
        return KernelVariant(v.op, v.mapping, v.f_tile, v.rows_per_chunk, bool(v.vectorized),
                             v.hub_threshold)


def variant_to_string(v: KernelVariant) -> str:
    buf = C.create_string_buffer(256)
    cv = v.to_c()
    _check(_lib.as_variant_to_string(C.byref(cv), buf, 256))
    return buf.value.decode()


def variant_from_string(s: str) -> KernelVariant:
    out = _c.as_variant()
    _check(_lib.as_variant_from_string(s.encode(), C.byref(out)))
    return KernelVariant.from_c(out)


def vec4_eligible(f: int, *arrays) -> bool:
    """src/kernels.cpp:202-208 on the operands' base addresses."""
    bases = (C.c_void_p * max(len(arrays), 1))(*[_base(a) for a in arrays])
    return bool(_lib.as_vec4_eligible(int(f), bases, len(arrays)))


def _base(a) -> int:
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return int(a.data_ptr())


@dataclasses.dataclass
class KernelResult:
    """KernelResult, include/autosage/kernels.hpp:36-42."""
    output: Optional[np.ndarray]
    values: Optional[np.ndarray]
    variant: KernelVariant
    vectorized_path: bool
    elapsed_ms: float


# ---- device graphs -----------------------------------------------------------------
class Graph:
    """A device-resident CSR (as_graph).  Owns its HBM copy."""

    def __init__(self, handle: int, device: int):
        self._h = C.c_void_p(handle)
        self.device = device
        nr, nc, nz, hv = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_int()
        _check(_lib.as_graph_shape(self._h, C.byref(nr), C.byref(nc), C.byref(nz), C.byref(hv)))
        self.n_rows, self.n_cols, self.nnz = nr.value, nc.value, nz.value
        self._has_val = bool(hv.value)

    @staticmethod
    def from_csr(m: CsrMatrix, device: int = 0) -> "Graph":
        h = C.c_void_p()
        val = m.val if m.has_values() else None
        _check(_lib.as_graph_create(_ptr(m.rowptr), _ptr(m.colind) if m.nnz else None, _ptr(val),
                                    m.n_rows, m.n_cols, m.nnz, device, C.byref(h)))
        return Graph(h.value, device)

    def synchronize(self) -> None:
        """Wait for every queued host-buffer operation (as_graph_synchronize)."""
        _check(_lib.as_graph_synchronize(self._h))

    def close(self) -> None:
        if self._h:
            _lib.as_graph_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def has_values(self) -> bool:
        return self._has_val

    def device_arrays(self):
        r, c, v = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _check(_lib.as_graph_device_arrays(self._h, C.byref(r), C.byref(c), C.byref(v)))
        return r.value, c.value, v.value

    def set_values(self, vals) -> None:
        if vals is None:
            _check(_lib.as_graph_set_values(self._h, None, 0))
        elif isinstance(vals, np.ndarray):
            vals = np.ascontiguousarray(vals, dtype=np.float32)
            _check(_lib.as_graph_set_values(self._h, _ptr(vals), 0))
        else:
            _check(_lib.as_graph_set_values(self._h, C.c_void_p(vals.data_ptr()), 1))
        self._has_val = vals is not None and self.nnz > 0

    def sig(self) -> int:
        out = C.c_uint64()
        _check(_lib.as_graph_sig(self._h, C.byref(out)))
        return out.value

    def features(self, hub_threshold: int = DEFAULT_HUB_THRESHOLD) -> "GraphFeatures":
        out = _c.as_features()
        _check(_lib.as_graph_features(self._h, hub_threshold, C.byref(out)))
        return GraphFeatures.from_c(out)

    def sample_row_indices(self, frac: float, min_rows: int) -> np.ndarray:
        rows = np.zeros(max(self.n_rows, 1), dtype=np.uint64)
        n = C.c_uint64()
        _check(_lib.as_sample_row_indices(self._h, frac, min_rows, _ptr(rows), C.byref(n)))
        return rows[:n.value].copy()

    def slice_rows(self, rows) -> "Graph":
        rows = np.ascontiguousarray(rows, dtype=np.uint64)
        h = C.c_void_p()
        _check(_lib.as_slice_rows(self._h, _ptr(rows), rows.size, C.byref(h)))
        return Graph(h.value, self.device)

    def row_range(self, r0: int, r1: int) -> "Graph":
        h = C.c_void_p()
        _check(_lib.as_graph_row_range(self._h, r0, r1, C.byref(h)))
        return Graph(h.value, self.device)

    def transpose(self) -> "Graph":
        """A^T on device (as_graph_transpose; backward pass):
        entries of each new row in source row order, values permuted, the
        entry permutation kept on the new handle."""
        h = C.c_void_p()
        _check(_lib.as_graph_transpose(self._h, C.byref(h)))
        return Graph(h.value, self.device)

    def transpose_perm_ptr(self) -> int:
        """Device address of a transpose's u32[nnz] permutation (perm[k] = source entry)."""
        p = C.c_void_p()
        _check(_lib.as_graph_transpose_perm(self._h, C.byref(p)))
        return p.value or 0

    def download(self) -> CsrMatrix:
        rp = np.zeros(self.n_rows + 1, dtype=np.uint64)
        ci = np.zeros(max(self.nnz, 1), dtype=np.uint32)
        va = np.zeros(max(self.nnz, 1), dtype=np.float32) if self._has_val else None
        _check(_lib.as_graph_download(self._h, _ptr(rp), _ptr(ci), _ptr(va)))
        return CsrMatrix(self.n_rows, self.n_cols, rp, ci[:self.nnz],
                         None if va is None else va[:self.nnz])


def _as_graph(m, device: int = 0):
    """(Graph, owned) for a CsrMatrix or Graph argument."""
    if isinstance(m, Graph):
        return m, False
    if isinstance(m, CsrMatrix):
        return Graph.from_csr(m, device), True
    raise TypeError(f"expected CsrMatrix or Graph, got {type(m).__name__}")


@dataclasses.dataclass
class GraphFeatures:
    """GraphFeatures, include/autosage/csr.hpp:93-107."""
    n_rows: int = 0
    n_cols: int = 0
    nnz: int = 0
    deg_p25: int = 0
    deg_p50: int = 0
    deg_p75: int = 0
    deg_p90: int = 0
    deg_p99: int = 0
    deg_max: int = 0
    mean_degree: float = 0.0
    heavy_row_fraction: float = 0.0
    empty_row_fraction: float = 0.0
    hub_threshold: int = DEFAULT_HUB_THRESHOLD

    @staticmethod
    def from_c(f: _c.as_features) -> "GraphFeatures":
        return GraphFeatures(*[getattr(f, n) for n, _ in _c.as_features._fields_])

    def to_c(self) -> _c.as_features:
        return _c.as_features(*[getattr(self, n) for n, _ in _c.as_features._fields_])


# ---- policy helpers ------------------------------------------------------------------
def validate(m: CsrMatrix):
    """validate, src/csr.cpp:62-93: None, or (invariant, index)."""
    viol, idx = C.c_int(), C.c_uint64()
    buf = C.create_string_buffer(128)
    rp = m.rowptr if m.rowptr.size else np.zeros(1, dtype=np.uint64)
    _check(_lib.as_validate(_ptr(rp), _ptr(m.colind), None, m.rowptr.size, m.n_rows, m.n_cols,
                            m.nnz, 0 if m.val is None else m.val.size, C.byref(viol), buf, 128,
                            C.byref(idx)))
    return (buf.value.decode(), idx.value) if viol.value else None


def graph_sig(m) -> int:
    """graph_sig, src/cache.cpp:66-74 (host arrays, or memoized on a Graph)."""
    if isinstance(m, Graph):
        return m.sig()
    return int(_lib.as_graph_sig_host(_ptr(m.rowptr), _ptr(m.colind), m.n_rows, m.n_cols, m.nnz))


def extract_features(m, hub_threshold: int = DEFAULT_HUB_THRESHOLD) -> GraphFeatures:
    g, own = _as_graph(m)
    try:
        return g.features(hub_threshold)
    finally:
        if own:
            g.close()


def sample_row_indices(m, frac: float, min_rows: int) -> np.ndarray:
    g, own = _as_graph(m)
    try:
        return g.sample_row_indices(frac, min_rows)
    finally:
        if own:
            g.close()


def slice_rows(m, rows) -> CsrMatrix:
    g, own = _as_graph(m)
    try:
        s = g.slice_rows(rows)
        out = s.download()
        s.close()
        return out
    finally:
        if own:
            g.close()


@dataclasses.dataclass
class DeviceProfile:
    """DeviceProfile, include/autosage/device.hpp:12-27."""
    device_sig: str = ""
    bw_eff: float = 0.0
    flops_eff: float = 0.0
    cores: int = 1
    model: int = 0  # 0: reference cost model, 1: B200 refinement (GPU profiles)

    @staticmethod
    def fixed(bw_eff: float, flops_eff: float, cores: int, sig_tag: str = "fixed"):
        out = _c.as_device_profile()
        _lib.as_device_profile_fixed(bw_eff, flops_eff, cores, sig_tag.encode(), C.byref(out))
        return DeviceProfile.from_c(out)

    @staticmethod
    def gpu(device: int = 0) -> "DeviceProfile":
        out = _c.as_device_profile()
        _check(_lib.as_device_profile_gpu(device, C.byref(out)))
        return DeviceProfile.from_c(out)

    @staticmethod
    def from_c(d) -> "DeviceProfile":
        return DeviceProfile(d.device_sig.decode(), d.bw_eff, d.flops_eff, d.cores, d.model)

    def to_c(self) -> _c.as_device_profile:
        return _c.as_device_profile(self.device_sig.encode(), self.bw_eff, self.flops_eff,
                                    self.cores, self.model)


def estimate_cost(v: KernelVariant, gf: GraphFeatures, f: int, dp: DeviceProfile) -> float:
    out = C.c_double()
    cv, cf, cd = v.to_c(), gf.to_c(), dp.to_c()
    _check(_lib.as_estimate_cost(C.byref(cv), C.byref(cf), f, C.byref(cd), C.byref(out)))
    return out.value


def shortlist(gf: GraphFeatures, f: int, op: int, dp: DeviceProfile) -> List[KernelVariant]:
    arr = (_c.as_variant * _c.AS_MAX_CANDIDATES)()
    n = C.c_int()
    cf, cd = gf.to_c(), dp.to_c()
    _check(_lib.as_shortlist(C.byref(cf), f, op, C.byref(cd), arr, C.byref(n)))
    return [KernelVariant.from_c(arr[i]) for i in range(n.value)]


@dataclasses.dataclass
class TimedKernelStats:
    median_ms: float
    completed: int
    capped: bool
    max_run_ms: float
    wall_ms: float
    launches: int


# A timer is a Python callable (label, run) -> ms, the ProbeTimer interface
# (include/autosage/timing.hpp:10-15); run() executes one kernel launch.
def _make_timer(timer):
    if timer is None:
        return _c.TIME_ONCE_FN(), None

    def cb(user, label, run_fn, run_arg):
        try:
            ms = timer(label.decode() if label else "", lambda: run_fn(run_arg))
            return float(ms)
        except Exception as e:  # surfaced after the C call returns
            _pending_exc.append(e)
            return -1.0
    fn = _c.TIME_ONCE_FN(cb)
    return fn, fn


def time_kernel(label: str, run: Callable[[], None], iters: int, cap_ms: float,
                timer=None) -> TimedKernelStats:
    """time_kernel, src/timing.cpp:22-61."""
    def _run(_arg):
        run()
    run_fn = _c.RUN_FN(_run)
    tfn, keep = _make_timer(timer)
    out = _c.as_timed_stats()
    _check(_lib.as_time_kernel(label.encode(), run_fn, None, iters, cap_ms, tfn, None,
                               C.byref(out)))
    del keep
    return TimedKernelStats(out.median_ms, out.completed, bool(out.capped), out.max_run_ms,
                            out.wall_ms, out.launches)


# ---- operands ------------------------------------------------------------------------
def _is_torch_cuda(x) -> bool:
    return hasattr(x, "data_ptr") and getattr(getattr(x, "device", None), "type", "") == "cuda"


def _np2d(a) -> np.ndarray:
    a = np.asarray(a)
    if a.ndim != 2:
        raise InvalidArgument("dense operand must be 2-D")
    if a.dtype != np.float32 or not a.flags.c_contiguous:
        a = np.ascontiguousarray(a, dtype=np.float32)
    return a


def _vptr(x):
    return C.c_void_p(x.data_ptr())


def torch_stream_handle(device=None) -> int:
    """torch's current stream as a C-ABI stream argument.  The legacy default
    stream (handle 0) maps to cudaStreamLegacy (0x1): NULL in the C-ABI means
    the graph's own internal stream."""
    import torch
    s = torch.cuda.current_stream(device).cuda_stream
    return s if s else 1


def _variant_arg(v: Optional[KernelVariant]):
    return None if v is None else C.byref(v.to_c())


def _result(r: _c.as_kernel_result, output=None, values=None) -> KernelResult:
    return KernelResult(output, values, KernelVariant.from_c(r.variant), bool(r.vectorized_path),
                        r.elapsed_ms)


def _spmm_call(v, a, b, result: bool):
    g, own = _as_graph(a)
    try:
        res = _c.as_kernel_result()
        if _is_torch_cuda(b):
            import torch
            f = int(b.shape[1])
            c = torch.empty((g.n_rows, f), dtype=torch.float32, device=b.device)
            stream = torch_stream_handle(b.device)
            _check(_lib.as_spmm(_variant_arg(v), g.handle, _vptr(b), int(b.shape[0]), f, _vptr(c),
                                C.c_void_p(stream), C.byref(res) if result else None))
            return c, res
        b = _np2d(b)
        f = b.shape[1]
        c = np.empty((g.n_rows, f), dtype=np.float32)
        _check(_lib.as_spmm_host(_variant_arg(v), g.handle, _ptr(b), b.shape[0], f, _ptr(c),
                                 C.byref(res)))
        return c, res
    finally:
        if own:
            g.close()


def spmm_host_async(v: Optional[KernelVariant], g: "Graph", b: np.ndarray, c: np.ndarray) -> None:
    """Queue H2D(b) -> SpMM -> D2H(c) on the graph's pipeline and return
    (as_spmm_host_async); c is valid after g.synchronize().  b and c should
    be pinned (e.g. torch.empty(..., pin_memory=True).numpy())."""
    res = _c.as_kernel_result()
    _check(_lib.as_spmm_host_async(_variant_arg(v), g.handle, _ptr(b), b.shape[0], b.shape[1],
                                   _ptr(c), C.byref(res)))


def sddmm_host_async(v: Optional[KernelVariant], g: "Graph", x: np.ndarray, y: np.ndarray,
                     out: np.ndarray) -> None:
    """Queue H2D(x, y) -> SDDMM (in slices) -> D2H(out) (as_sddmm_host_async)."""
    res = _c.as_kernel_result()
    _check(_lib.as_sddmm_host_async(_variant_arg(v), g.handle, _ptr(x), x.shape[0], _ptr(y),
                                    y.shape[0], x.shape[1], _ptr(out), C.byref(res)))


def spmm_baseline(a, b):
    """C = A*B with the guardrail baseline kernel (src/kernels.cpp:210-228)."""
    return _spmm_call(None, a, b, False)[0]


def _mapped(fn, v: KernelVariant, a, b):
    g, own = _as_graph(a)
    try:
        if _is_torch_cuda(b):
            import torch
            f = int(b.shape[1])
            c = torch.empty((g.n_rows, f), dtype=torch.float32, device=b.device)
            stream = torch_stream_handle(b.device)
            _check(fn(C.byref(v.to_c()), g.handle, _vptr(b), int(b.shape[0]), f, _vptr(c),
                      C.c_void_p(stream)))
            return c
        import torch
        bt = torch.from_numpy(_np2d(b)).cuda(g.device)
        c = torch.empty((g.n_rows, bt.shape[1]), dtype=torch.float32, device=bt.device)
        stream = torch_stream_handle(bt.device)
        _check(fn(C.byref(v.to_c()), g.handle, _vptr(bt), int(bt.shape[0]), int(bt.shape[1]),
                  _vptr(c), C.c_void_p(stream)))
        return c.cpu().numpy()
    finally:
        if own:
            g.close()


def spmm_rowparallel(a, b, v: KernelVariant, workers: int = 0):
    """src/kernels.cpp:230-258 (workers is a CPU knob; ignored on the GPU)."""
    return _mapped(_lib.as_spmm_rowparallel, v, a, b)


def spmm_hubsplit(a, b, v: KernelVariant, workers: int = 0):
    """src/kernels.cpp:260-334."""
    return _mapped(_lib.as_spmm_hubsplit, v, a, b)


def _sddmm_call(v, p, x, y, result: bool):
    g, own = _as_graph(p)
    try:
        res = _c.as_kernel_result()
        if _is_torch_cuda(x):
            import torch
            if x.shape[1] != y.shape[1]:
                raise InvalidArgument("sddmm: x.n_cols != y.n_cols")
            out = torch.empty(max(g.nnz, 0), dtype=torch.float32, device=x.device)
            stream = torch_stream_handle(x.device)
            _check(_lib.as_sddmm(_variant_arg(v), g.handle, _vptr(x), int(x.shape[0]), _vptr(y),
                                 int(y.shape[0]), int(x.shape[1]), _vptr(out) if g.nnz else None,
                                 C.c_void_p(stream), C.byref(res) if result else None))
            return out, res
        x, y = _np2d(x), _np2d(y)
        if x.shape[1] != y.shape[1]:
            raise InvalidArgument("sddmm: x.n_cols != y.n_cols")
        out = np.empty(max(g.nnz, 1), dtype=np.float32)
        _check(_lib.as_sddmm_host(_variant_arg(v), g.handle, _ptr(x), x.shape[0], _ptr(y),
                                  y.shape[0], x.shape[1], _ptr(out), C.byref(res)))
        return out[:g.nnz], res
    finally:
        if own:
            g.close()


def sddmm_baseline(p, x, y):
    """out[e] = <X[i,:], Y[col[e],:]> (src/kernels.cpp:336-355)."""
    return _sddmm_call(None, p, x, y, False)[0]


def sddmm_rowparallel(p, x, y, v: KernelVariant, workers: int = 0):
    """src/kernels.cpp:357-429 (mapping must not be baseline; no env overrides)."""
    import torch
    g, own = _as_graph(p)
    try:
        host = not _is_torch_cuda(x)
        xd, yd = _to_device(x, g.device), _to_device(y, g.device)
        if xd.shape[1] != yd.shape[1]:
            raise InvalidArgument("sddmm: x.n_cols != y.n_cols")
        out = torch.empty(max(g.nnz, 1), dtype=torch.float32, device=xd.device)
        stream = torch_stream_handle(xd.device)
        vv = dataclasses.replace(v, op=SDDMM).to_c()
        _check(_lib.as_sddmm_rowparallel(C.byref(vv), g.handle, _vptr(xd), int(xd.shape[0]),
                                         _vptr(yd), int(yd.shape[0]), int(xd.shape[1]),
                                         _vptr(out), C.c_void_p(stream)))
        out = out[:g.nnz]
        return out.cpu().numpy() if host else out
    finally:
        if own:
            g.close()


def row_softmax(m, workers: int = 0):
    """Row softmax over the matrix's values (src/kernels.cpp:431-461).
    CsrMatrix in -> CsrMatrix out (pattern copied); Graph in -> values array."""
    if isinstance(m, CsrMatrix):
        if m.nnz > 0 and not m.has_values():
            raise InvalidArgument("row_softmax: values required")
        if m.nnz == 0 or m.n_rows == 0:
            return CsrMatrix(m.n_rows, m.n_cols, m.rowptr.copy(), m.colind.copy(),
                             None if m.val is None else m.val.copy())
        g = Graph.from_csr(m.with_values(None))
        try:
            out = np.empty(m.nnz, dtype=np.float32)
            _check(_lib.as_row_softmax_host(g.handle, _ptr(m.val), _ptr(out)))
        finally:
            g.close()
        return CsrMatrix(m.n_rows, m.n_cols, m.rowptr.copy(), m.colind.copy(), out)
    out = np.empty(max(m.nnz, 1), dtype=np.float32)
    _check(_lib.as_row_softmax_host(m.handle, None, _ptr(out)))
    return out[:m.nnz]


def dispatch(v: KernelVariant, a, b, y=None, workers: int = 0) -> KernelResult:
    """dispatch(v, a, b) for SpMM, dispatch(v, pattern, x, y) for SDDMM
    (src/kernels.cpp:485-531): env overrides, vec4 gate, elapsed_ms."""
    if y is None:
        out, res = _spmm_call(v, a, b, True)
        return _result(res, output=out)
    vals, res = _sddmm_call(v, a, b, y, True)
    return _result(res, values=vals)


# ---- schedule cache ---------------------------------------------------------------
@dataclasses.dataclass(frozen=True, order=True)
class ScheduleKey:
    device_sig: str
    graph_sig: int
    f: int
    op: int

    def to_c(self) -> _c.as_key:
        return _c.as_key(self.device_sig.encode(), self.graph_sig, self.f, self.op)

    @staticmethod
    def from_c(k: _c.as_key) -> "ScheduleKey":
        return ScheduleKey(k.device_sig.decode(), k.graph_sig, k.f, k.op)

    def to_string(self) -> str:
        buf = C.create_string_buffer(512)
        ck = self.to_c()
        _check(_lib.as_key_to_string(C.byref(ck), buf, 512))
        return buf.value.decode()


@dataclasses.dataclass
class CacheRecord:
    key: ScheduleKey
    choice: str
    t_b: float = 0.0
    t_star: float = 0.0
    alpha: float = 0.0
    timestamp: int = 0
    schema_version: int = 1
    toolchain: str = ""

    def to_c(self) -> _c.as_record:
        return _c.as_record(self.key.to_c(), self.choice.encode(), self.t_b, self.t_star,
                            self.alpha, self.timestamp, self.schema_version,
                            self.toolchain.encode())

    @staticmethod
    def from_c(r: _c.as_record) -> "CacheRecord":
        return CacheRecord(ScheduleKey.from_c(r.key), r.choice.decode(), r.t_b, r.t_star,
                           r.alpha, r.timestamp, r.schema_version, r.toolchain.decode())


def record_to_line(rec: CacheRecord) -> str:
    buf = C.create_string_buffer(1024)
    cr = rec.to_c()
    _check(_lib.as_record_to_line(C.byref(cr), buf, 1024))
    return buf.value.decode()


def record_from_line(line: str) -> CacheRecord:
    out = _c.as_record()
    _check(_lib.as_record_from_line(line.encode(), C.byref(out)))
    return CacheRecord.from_c(out)


class ScheduleCache:
    """ScheduleCache, include/autosage/cache.hpp:48-76."""

    def __init__(self):
        h = C.c_void_p()
        _check(_lib.as_cache_create(C.byref(h)))
        self._h = h

    def __del__(self):
        try:
            if self._h:
                _lib.as_cache_destroy(self._h)
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def get(self, key: ScheduleKey) -> Optional[CacheRecord]:
        out, found = _c.as_record(), C.c_int()
        ck = key.to_c()
        _check(_lib.as_cache_get(self._h, C.byref(ck), C.byref(out), C.byref(found)))
        return CacheRecord.from_c(out) if found.value else None

    def put(self, rec: CacheRecord) -> None:
        cr = rec.to_c()
        _check(_lib.as_cache_put(self._h, C.byref(cr)))

    def size(self) -> int:
        n = C.c_uint64()
        _check(_lib.as_cache_size(self._h, C.byref(n)))
        return n.value

    def snapshot(self) -> List[CacheRecord]:
        n = C.c_uint64()
        _check(_lib.as_cache_snapshot(self._h, None, 0, C.byref(n)))
        arr = (_c.as_record * max(n.value, 1))()
        _check(_lib.as_cache_snapshot(self._h, arr, n.value, C.byref(n)))
        return [CacheRecord.from_c(arr[i]) for i in range(n.value)]

    def clear(self) -> None:
        _check(_lib.as_cache_clear(self._h))

    def load(self, path: str) -> None:
        _check(_lib.as_cache_load(self._h, os.fspath(path).encode()))

    def store(self, path: str) -> None:
        _check(_lib.as_cache_store(self._h, os.fspath(path).encode()))


# ---- scheduler -------------------------------------------------------------------------
@dataclasses.dataclass
class ProbeConfig:
    """ProbeConfig, include/autosage/scheduler.hpp:16-28."""
    frac: float = 0.02
    min_rows: int = 512
    iters: int = 5
    cap_ms: float = 1.0
    top_k: int = 3
    alpha: float = 0.95

    @staticmethod
    def from_env() -> "ProbeConfig":
        out = _c.as_probe_config()
        _lib.as_probe_config_from_env(C.byref(out))
        return ProbeConfig(out.frac, out.min_rows, out.iters, out.cap_ms, out.top_k, out.alpha)

    def to_c(self) -> _c.as_probe_config:
        return _c.as_probe_config(self.frac, self.min_rows, self.iters, self.cap_ms, self.top_k,
                                  self.alpha)


@dataclasses.dataclass
class ReplayPolicy:
    replay_only: bool = False
    strict: bool = False

    @staticmethod
    def from_env() -> "ReplayPolicy":
        out = _c.as_replay_policy()
        _lib.as_replay_policy_from_env(C.byref(out))
        return ReplayPolicy(bool(out.replay_only), bool(out.strict))


@dataclasses.dataclass
class ScheduleContext:
    """ScheduleContext, include/autosage/scheduler.hpp:61-69."""
    device: Optional[DeviceProfile] = None
    cache: Optional[ScheduleCache] = None
    timer: Optional[Callable] = None
    replay: ReplayPolicy = dataclasses.field(default_factory=ReplayPolicy)
    stream: Optional[int] = None

    def to_c(self):
        keep = []
        dev = None
        if self.device is not None:
            dev = self.device.to_c()
            keep.append(dev)
        tfn, tkeep = _make_timer(self.timer)
        keep.append(tfn)
        ctx = _c.as_context(C.pointer(dev) if dev is not None else None,
                            self.cache.handle if self.cache else None, tfn, None,
                            _c.as_replay_policy(int(self.replay.replay_only),
                                                int(self.replay.strict)),
                            self.stream)
        return ctx, keep


@dataclasses.dataclass
class CandidateTiming:
    variant: KernelVariant
    median_ms: float
    completed: int
    capped: bool


@dataclasses.dataclass
class ScheduleDecision:
    """ScheduleDecision + ProbeReport, include/autosage/scheduler.hpp:36-59."""
    choice: Optional[KernelVariant]
    source: int
    key: ScheduleKey
    alpha: float
    baseline_ms: float
    baseline_completed: int
    baseline_capped: bool
    candidates: List[CandidateTiming]
    best_index: int
    t_star: float
    sample_rows: int
    probe_wall_ms: float
    max_single_run_ms: float
    sig_ms: float = 0.0
    features_ms: float = 0.0
    sample_ms: float = 0.0
    decide_wall_ms: float = 0.0

    def choice_string(self) -> str:
        return variant_to_string(self.choice) if self.choice is not None else "baseline"

    @property
    def source_name(self) -> str:
        return SOURCES[self.source]

    @staticmethod
    def from_c(d: _c.as_decision) -> "ScheduleDecision":
        cands = [CandidateTiming(KernelVariant.from_c(d.candidates[i].variant),
                                 d.candidates[i].median_ms, d.candidates[i].completed,
                                 bool(d.candidates[i].capped)) for i in range(d.n_candidates)]
        return ScheduleDecision(KernelVariant.from_c(d.choice) if d.has_choice else None,
                                d.source, ScheduleKey.from_c(d.key), d.alpha, d.baseline_ms,
                                d.baseline_completed, bool(d.baseline_capped), cands,
                                d.best_index, d.t_star, d.sample_rows, d.probe_wall_ms,
                                d.max_single_run_ms, d.sig_ms, d.features_ms, d.sample_ms,
                                d.decide_wall_ms)


def _to_device(a, device: int):
    import torch
    if _is_torch_cuda(a):
        return a
    return torch.from_numpy(_np2d(a)).cuda(device)


def decide_spmm(a, b, cfg: Optional[ProbeConfig] = None,
                ctx: Optional[ScheduleContext] = None) -> ScheduleDecision:
    cfg = cfg or ProbeConfig()
    ctx = ctx or ScheduleContext()
    g, own = _as_graph(a)
    try:
        bd = _to_device(b, g.device)
        cctx, keep = ctx.to_c()
        ccfg = cfg.to_c()
        out = _c.as_decision()
        _check(_lib.as_decide_spmm(C.byref(cctx), C.byref(ccfg), g.handle, _vptr(bd),
                                   int(bd.shape[0]), int(bd.shape[1]), C.byref(out)))
        del keep
        return ScheduleDecision.from_c(out)
    finally:
        if own:
            g.close()


def decide_sddmm(p, x, y, cfg: Optional[ProbeConfig] = None,
                 ctx: Optional[ScheduleContext] = None) -> ScheduleDecision:
    cfg = cfg or ProbeConfig()
    ctx = ctx or ScheduleContext()
    g, own = _as_graph(p)
    try:
        xd, yd = _to_device(x, g.device), _to_device(y, g.device)
        if xd.shape[1] != yd.shape[1]:
            raise InvalidArgument("decide_sddmm: dimension mismatch")
        cctx, keep = ctx.to_c()
        ccfg = cfg.to_c()
        out = _c.as_decision()
        _check(_lib.as_decide_sddmm(C.byref(cctx), C.byref(ccfg), g.handle, _vptr(xd),
                                    int(xd.shape[0]), _vptr(yd), int(yd.shape[0]),
                                    int(xd.shape[1]), C.byref(out)))
        del keep
        return ScheduleDecision.from_c(out)
    finally:
        if own:
            g.close()


def spmm_auto(a, b, cfg: Optional[ProbeConfig] = None, ctx: Optional[ScheduleContext] = None,
              return_decision: bool = False):
    """decide + dispatch on the full input (src/scheduler.cpp:226-231)."""
    import torch
    cfg = cfg or ProbeConfig()
    ctx = ctx or ScheduleContext()
    g, own = _as_graph(a)
    try:
        host = not _is_torch_cuda(b)
        bd = _to_device(b, g.device)
        c = torch.empty((g.n_rows, int(bd.shape[1])), dtype=torch.float32, device=bd.device)
        cctx, keep = ctx.to_c()
        ccfg = cfg.to_c()
        out = _c.as_decision()
        _check(_lib.as_spmm_auto(C.byref(cctx), C.byref(ccfg), g.handle, _vptr(bd),
                                 int(bd.shape[0]), int(bd.shape[1]), _vptr(c), C.byref(out)))
        torch.cuda.synchronize(bd.device)
        del keep
        res = c.cpu().numpy() if host else c
        return (res, ScheduleDecision.from_c(out)) if return_decision else res
    finally:
        if own:
            g.close()


def sddmm_auto(p, x, y, cfg: Optional[ProbeConfig] = None,
               ctx: Optional[ScheduleContext] = None, return_decision: bool = False):
    import torch
    cfg = cfg or ProbeConfig()
    ctx = ctx or ScheduleContext()
    g, own = _as_graph(p)
    try:
        host = not _is_torch_cuda(x)
        xd, yd = _to_device(x, g.device), _to_device(y, g.device)
        o = torch.empty(max(g.nnz, 1), dtype=torch.float32, device=xd.device)
        cctx, keep = ctx.to_c()
        ccfg = cfg.to_c()
        out = _c.as_decision()
        _check(_lib.as_sddmm_auto(C.byref(cctx), C.byref(ccfg), g.handle, _vptr(xd),
                                  int(xd.shape[0]), _vptr(yd), int(yd.shape[0]),
                                  int(xd.shape[1]), _vptr(o), C.byref(out)))
        torch.cuda.synchronize(xd.device)
        del keep
        o = o[:g.nnz]
        res = o.cpu().numpy() if host else o
        return (res, ScheduleDecision.from_c(out)) if return_decision else res
    finally:
        if own:
            g.close()


def probe_launch_count() -> int:
    return int(_lib.as_probe_launch_count())


def reset_probe_launch_count() -> None:
    _lib.as_reset_probe_launch_count()


def decide_host(ctx: ScheduleContext, cfg: ProbeConfig, graph_sig_value: int,
                gf: GraphFeatures, f: int, op: int, sample_rows: int = 0) -> ScheduleDecision:
    """decide_common over precomputed inputs; no kernels run (host-only)."""
    cctx, keep = ctx.to_c()
    ccfg, cf = cfg.to_c(), gf.to_c()
    out = _c.as_decision()
    _check(_lib.as_decide_host(C.byref(cctx), C.byref(ccfg), graph_sig_value, C.byref(cf), f, op,
                               sample_rows, C.byref(out)))
    del keep
    return ScheduleDecision.from_c(out)


# ---- attention -----------------------------------------------------------------------------
@dataclasses.dataclass
class AttentionRun:
    output: object
    sddmm_decision: ScheduleDecision
    spmm_decision: ScheduleDecision


def attention_probe_breakdown(pattern, q, k, v, cfg: Optional[ProbeConfig] = None,
                              ctx: Optional[ScheduleContext] = None,
                              fused: bool = False) -> AttentionRun:
    """src/attention.cpp:9-40.  fused=True: SDDMM -> per-row (max, sum) -> SpMM
    that applies the softmax to each score as it loads it (no probability
    array); the same bits as the staged pipeline (fused=False)."""
    import torch
    cfg = cfg or ProbeConfig()
    ctx = ctx or ScheduleContext()
    g, own = _as_graph(pattern)
    try:
        host = not _is_torch_cuda(q)
        qd, kd, vd = (_to_device(t, g.device) for t in (q, k, v))
        if qd.shape[1] != kd.shape[1]:
            raise InvalidArgument("attention: q.n_cols != k.n_cols")
        out = torch.empty((g.n_rows, int(vd.shape[1])), dtype=torch.float32, device=qd.device)
        cctx, keep = ctx.to_c()
        ccfg = cfg.to_c()
        sd, pd = _c.as_decision(), _c.as_decision()
        _check(_lib.as_csr_attention_forward(
            C.byref(cctx), C.byref(ccfg), g.handle, _vptr(qd), int(qd.shape[0]), _vptr(kd),
            int(kd.shape[0]), _vptr(vd), int(vd.shape[0]), int(qd.shape[1]), int(vd.shape[1]),
            _vptr(out), 1 if fused else 0, C.byref(sd), C.byref(pd)))
        torch.cuda.synchronize(qd.device)
        del keep
        res = out.cpu().numpy() if host else out
        return AttentionRun(res, ScheduleDecision.from_c(sd), ScheduleDecision.from_c(pd))
    finally:
        if own:
            g.close()


def csr_attention_forward(pattern, q, k, v, cfg: Optional[ProbeConfig] = None,
                          ctx: Optional[ScheduleContext] = None, fused: bool = False):
    return attention_probe_breakdown(pattern, q, k, v, cfg, ctx, fused).output


def csr_attention_forward_heads(pattern: "Graph", qs, ks, vs, cfg: Optional[ProbeConfig] = None,
                                ctx: Optional[ScheduleContext] = None, fused: bool = True):
    """Several heads on one device pattern graph in one call
    (as_csr_attention_forward_heads): head 1 decides, the rest reuse its
    decisions (a call-local cache when ctx has none).  qs / ks / vs: lists of
    CUDA float32 tensors (n_rows x F, n_cols x F, n_cols x Fv); returns the
    list of n_rows x Fv outputs, each equal to the single-head call."""
    import torch
    h = len(qs)
    if not (len(ks) == h and len(vs) == h):
        raise InvalidArgument("attention_heads: q, k, v head counts differ")
    cfg = cfg or ProbeConfig()
    ctx = ctx or ScheduleContext()
    qs, ks, vs = ([t.contiguous().float() for t in seq] for seq in (qs, ks, vs))
    f = int(qs[0].shape[1]) if h else 0
    fv = int(vs[0].shape[1]) if h else 0
    outs = [torch.empty((pattern.n_rows, fv), dtype=torch.float32, device=qs[0].device) for _ in range(h)]
    arr = lambda ts: (C.c_void_p * max(h, 1))(*[t.data_ptr() for t in ts])  # noqa: E731
    if ctx.stream is None and h:
        ctx = dataclasses.replace(ctx, stream=torch_stream_handle(qs[0].device))
    cctx, keep = ctx.to_c()
    ccfg = cfg.to_c()
    sd, pd = _c.as_decision(), _c.as_decision()
    _check(_lib.as_csr_attention_forward_heads(
        C.byref(cctx), C.byref(ccfg), pattern.handle, h, arr(qs), int(qs[0].shape[0]) if h else 0, arr(ks),
        int(ks[0].shape[0]) if h else 0, arr(vs), int(vs[0].shape[0]) if h else 0, f, fv, arr(outs), int(fused),
        C.byref(sd), C.byref(pd)))
    del keep
    return outs


# ---- multi-GPU partition, synthetic inputs, I/O -------------------------------------------
class BlockedSpmm:
    """Column-blocked SpMM plan (as_spmm_blocked_*): C = A B consumed one
    column block of B per run(), in ascending block order on one stream, so a
    rank can start on each B row shard as it lands (dist.py).  Bit-identical
    to as_spmm with the same variant (None: baseline)."""

    def __init__(self, g: "Graph", variant: Optional[KernelVariant], cuts):
        self.g = g
        self.cuts = np.ascontiguousarray(cuts, dtype=np.uint64)
        self.n_blocks = int(self.cuts.size - 1)
        h = C.c_void_p()
        cv = variant.to_c() if variant is not None else None
        _check(_lib.as_spmm_blocked_create(g.handle, C.byref(cv) if cv is not None else None, _ptr(self.cuts),
                                           self.n_blocks, C.byref(h)))
        self._h = h.value

    def run(self, block: int, b, c, vals=None, stream=None) -> None:
        """Block `block` of C = A B (b, c, vals: CUDA tensors; the last block
        writes c)."""
        s = stream if stream is not None else torch_stream_handle(b.device)
        _check(_lib.as_spmm_blocked_run(self._h, block, _vptr(vals) if vals is not None else None, _vptr(b),
                                        int(b.shape[0]), int(b.shape[1]), _vptr(c), C.c_void_p(s)))

    def close(self) -> None:
        if self._h:
            _lib.as_spmm_blocked_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def partition_rows(rowptr, g: int) -> np.ndarray:
    """nnz-balanced row cuts (g+1 entries), SURVEY 8(e)."""
    rowptr = np.ascontiguousarray(rowptr, dtype=np.uint64)
    cuts = np.zeros(g + 1, dtype=np.uint64)
    _check(_lib.as_partition_rows(_ptr(rowptr), rowptr.size - 1, g, _ptr(cuts)))
    return cuts


def _take_csr(rp, ci, va, n_rows, n_cols, nnz) -> CsrMatrix:
    rowptr = np.ctypeslib.as_array(C.cast(rp, C.POINTER(C.c_uint64)), (n_rows + 1,)).copy()
    colind = (np.ctypeslib.as_array(C.cast(ci, C.POINTER(C.c_uint32)), (nnz,)).copy()
              if nnz else np.zeros(0, dtype=np.uint32))
    val = None
    if va:
        val = (np.ctypeslib.as_array(C.cast(va, C.POINTER(C.c_float)), (nnz,)).copy()
               if nnz else np.zeros(0, dtype=np.float32))
    for p in (rp, ci, va):
        if p:
            _lib.as_free(p)
    return CsrMatrix(n_rows, n_cols, rowptr, colind, val)


def gen_powerlaw(n_rows: int, n_cols: int, nnz_target: int, alpha: float, d_min: int,
                 d_max: int, seed: int, with_values: bool = True) -> CsrMatrix:
    rp, ci, va, nnz = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_uint64()
    _check(_lib.as_gen_powerlaw(n_rows, n_cols, nnz_target, alpha, d_min, d_max, seed,
                                1 if with_values else 0, C.byref(rp), C.byref(ci), C.byref(va),
                                C.byref(nnz)))
    return _take_csr(rp.value, ci.value, va.value, n_rows, n_cols, nnz.value)


def fill_uniform(n: int, seed: int, shape=None) -> np.ndarray:
    """U[-1, 1) f32, counter-based (deterministic, thread-count independent)."""
    out = np.empty(n, dtype=np.float32)
    _check(_lib.as_fill_uniform(_ptr(out), n, seed))
    return out.reshape(shape) if shape is not None else out


def save_csr(m: CsrMatrix, path: str) -> None:
    _check(_lib.as_save_csr(os.fspath(path).encode(), _ptr(m.rowptr), _ptr(m.colind),
                            _ptr(m.val) if m.has_values() else None, m.n_rows, m.n_cols, m.nnz))


def load_csr(path: str) -> CsrMatrix:
    rp, ci, va = C.c_void_p(), C.c_void_p(), C.c_void_p()
    nr, nc, nz = C.c_uint64(), C.c_uint64(), C.c_uint64()
    _check(_lib.as_load_csr(os.fspath(path).encode(), C.byref(rp), C.byref(ci), C.byref(va),
                            C.byref(nr), C.byref(nc), C.byref(nz)))
    return _take_csr(rp.value, ci.value, va.value, nr.value, nc.value, nz.value)
