"""PyTorch custom operators over the C-ABI (the paper's
integration surface).

    import paper_2511_17594_b200.torch_ops  # registers torch.ops.autosage.*
    c = torch.ops.autosage.spmm_csr(crow, col, val, b, "spmm:hubsplit:ft=64:rpc=4:vec=1:hubt=256")
    c = torch.ops.autosage.spmm_csr_auto(crow, col, val, b)       # decide (cached) + run
    c = torch.ops.autosage.spmm_csr_split(crow, col, val, b, 256, 64, True)  # hub split at hubT 256
    s = torch.ops.autosage.sddmm_csr_auto(crow, col, x, y)         # decide (cached) + run
    s = torch.ops.autosage.sddmm_csr(crow, col, x, y, "")          # "" = baseline
    o = torch.ops.autosage.csr_attention(crow, col, q, k, v, False)
    p = torch.ops.autosage.row_softmax_csr(crow, col, s, n_cols)

CSR arrays are CUDA tensors: crow int64 [n_rows + 1], col int32 [nnz],
values float32 [nnz] (optional: pass an empty tensor for pattern-only).  The
number of columns is the dense operand's row count.  Results are computed on
torch's current stream by the sm_100a kernels, with the same numerics as the
reference (bit-exact SpMM/SDDMM).  Device graph handles (upload, degree
order, hub plans) are cached per CSR storage, so repeated calls on a static
graph pay the setup once.

Backward (the reference has no gradients): every op has a
registered autograd formula built from the same kernels -- A^T products run
the SpMM on a cached device transpose (as_graph_transpose) with the values
carried through its entry permutation, value gradients are SDDMMs, and the
softmax gradient is as_row_softmax_backward.  SpMM mappings are bit-identical
to each other, so the backward SpMMs use the hub-split mapping (`_BWD_SPMM`)
whatever the forward variant was; the SDDMMs use a scalar (sequential-order)
mapped variant (`_BWD_SDDMM`), the same bits as the baseline.  csr_attention's backward recomputes the
scores and probabilities (staged) rather than keeping them from the forward.
"""
from __future__ import annotations

import ctypes as C
import os
from collections import OrderedDict

import torch

from . import (Graph, ProbeConfig, ReplayPolicy, ScheduleCache, ScheduleContext, _check, _lib,
               torch_stream_handle, variant_from_string)
from . import _capi as _c

_GRAPHS: "OrderedDict[tuple, _Entry]" = OrderedDict()
_TRANSPOSES: "OrderedDict[tuple, _Entry]" = OrderedDict()
_MAX_GRAPHS = 8
_CACHE = None


class _Entry:
    """A cached device graph and the CSR tensors it was built from.  Holding
    the tensors keeps their storage alive, so while the entry is cached no
    other tensor can be allocated at the same addresses and hit it."""

    __slots__ = ("graph", "crow", "col")

    def __init__(self, graph: Graph, crow: torch.Tensor, col: torch.Tensor):
        self.graph, self.crow, self.col = graph, crow, col


def _key(crow, col, n_cols):
    # structure only: edge weights are passed per call (as_spmm_values /
    # as_spmm_auto_values), so updating them never rebuilds the graph
    return (crow.data_ptr(), col.data_ptr(), crow.numel() - 1, int(n_cols), col.numel(), crow._version,
            col._version, crow.device.index)


def _check_csr(crow: torch.Tensor, col: torch.Tensor):
    if not (crow.is_cuda and col.is_cuda):
        raise ValueError("autosage ops take CUDA CSR tensors")
    if crow.dtype != torch.int64 or col.dtype != torch.int32:
        raise ValueError("crow must be int64 and col int32")
    if crow.dim() != 1 or col.dim() != 1 or crow.numel() < 1:
        raise ValueError("crow and col must be 1-D (crow has n_rows + 1 entries)")


def _graph(crow: torch.Tensor, col: torch.Tensor, n_cols: int) -> Graph:
    """The pattern graph of (crow, col) with n_cols columns, uploaded and
    validated on the device once (columns in range and increasing per row),
    then cached per CSR storage."""
    _check_csr(crow, col)
    k = _key(crow, col, n_cols)
    e = _GRAPHS.get(k)
    if e is not None:
        _GRAPHS.move_to_end(k)
        return e.graph
    crow_c, col_c = crow.contiguous(), col.contiguous()
    h = C.c_void_p()
    # the copies are ordered after torch's current stream (which produced the arrays)
    _check(_lib.as_graph_create_device(C.c_void_p(crow_c.data_ptr()), C.c_void_p(col_c.data_ptr()), None,
                                       crow_c.numel() - 1, int(n_cols), col_c.numel(),
                                       crow.device.index or 0, _stream(crow), C.byref(h)))
    g = Graph(h.value, crow.device.index or 0)
    _GRAPHS[k] = _Entry(g, crow, col)
    while len(_GRAPHS) > _MAX_GRAPHS:
        _GRAPHS.popitem(last=False)[1].graph.close()
    return g


def _transpose(crow: torch.Tensor, col: torch.Tensor, n_cols: int) -> Graph:
    """Pattern-only A^T (device), cached per CSR storage like _graph."""
    k = _key(crow, col, n_cols)
    e = _TRANSPOSES.get(k)
    if e is not None:
        _TRANSPOSES.move_to_end(k)
        return e.graph
    g = _graph(crow, col, n_cols).transpose()
    _TRANSPOSES[k] = _Entry(g, crow, col)
    while len(_TRANSPOSES) > _MAX_GRAPHS:
        _TRANSPOSES.popitem(last=False)[1].graph.close()
    return g


def _values(val: torch.Tensor, nnz: int):
    """Edge weights as f32 (None: pattern-only, implicit 1.0)."""
    if val.numel() == 0:
        return None
    if val.numel() != nnz:
        raise ValueError(f"values must have nnz = {nnz} entries (got {val.numel()})")
    return val.contiguous().float()


def _vptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


# 16-bit operand words (csrc/half.cuh): dtype -> (SpMM, SDDMM, word type)
_HALF = {
    torch.bfloat16: (_lib.as_spmm_bf16, _lib.as_sddmm_bf16, 1),
    torch.float16: (_lib.as_spmm_f16, _lib.as_sddmm_f16, 2),
}


def _variant(s: str):
    return None if not s or s == "baseline" else C.byref(variant_from_string(s).to_c())


def _stream(t: torch.Tensor):
    return C.c_void_p(torch_stream_handle(t.device))


def _ctx(t: torch.Tensor):
    """The process-wide schedule context of the *_auto ops.  The paper's
    toggles apply: AUTOSAGE_CACHE names a cache file loaded on
    first use and rewritten whenever a decision is added (persistent replay
    across processes; the same TSV as the reference's), and
    AUTOSAGE_REPLAY_ONLY / AUTOSAGE_REPLAY_STRICT set the replay policy
    (ReplayPolicy::from_env)."""
    global _CACHE
    if _CACHE is None:
        _CACHE = ScheduleCache()
        path = os.environ.get("AUTOSAGE_CACHE", "")
        if path and os.path.exists(path):
            _CACHE.load(path)
    return ScheduleContext(cache=_CACHE, stream=torch_stream_handle(t.device), replay=ReplayPolicy.from_env())


def _persist(n_before: int) -> None:
    """Write the cache back to AUTOSAGE_CACHE when a decision was added."""
    path = os.environ.get("AUTOSAGE_CACHE", "")
    if path and _CACHE is not None and _CACHE.size() != n_before:
        _CACHE.store(path)


def _cache_size() -> int:
    return _CACHE.size() if _CACHE is not None else 0


@torch.library.custom_op("autosage::spmm_csr", mutates_args=())
def spmm_csr(crow: torch.Tensor, col: torch.Tensor, val: torch.Tensor, b: torch.Tensor,
             variant: str) -> torch.Tensor:
    """C = A B (dispatch(variant, A, B), src/kernels.cpp:485-506; "" = baseline).
    A bfloat16 / float16 B is read as 16-bit words (as_spmm_bf16 / as_spmm_f16: half the gather bytes, the
    f32 result on float(B) bit for bit); C is float32 either way."""
    return _spmm_impl(crow, col, val, b, variant)


def _spmm_impl(crow, col, val, b, variant: str) -> torch.Tensor:
    if b.dim() != 2:
        raise ValueError("spmm_csr: b must be 2-D")
    g = _graph(crow, col, b.shape[0])
    vals = _values(val, g.nnz)
    c = torch.empty((g.n_rows, b.shape[1]), dtype=torch.float32, device=b.device)
    if b.dtype in _HALF:
        b = b.contiguous()
        _check(_HALF[b.dtype][0](_variant(variant), g.handle, _vptr(vals), C.c_void_p(b.data_ptr()), b.shape[0],
                                 b.shape[1], C.c_void_p(c.data_ptr()), _stream(b), None))
        return c
    b = b.contiguous().float()
    if vals is None:
        _check(_lib.as_spmm(_variant(variant), g.handle, C.c_void_p(b.data_ptr()), b.shape[0], b.shape[1],
                            C.c_void_p(c.data_ptr()), _stream(b), None))
    else:
        _check(_lib.as_spmm_values(_variant(variant), g.handle, _vptr(vals), C.c_void_p(b.data_ptr()),
                                   b.shape[0], b.shape[1], C.c_void_p(c.data_ptr()), _stream(b), None))
    return c


@spmm_csr.register_fake
def _(crow, col, val, b, variant):
    return b.new_empty((crow.shape[0] - 1, b.shape[1]), dtype=torch.float32)


@torch.library.custom_op("autosage::spmm_csr_split", mutates_args=())
def spmm_csr_split(crow: torch.Tensor, col: torch.Tensor, val: torch.Tensor, b: torch.Tensor,
                   hub_threshold: int, f_tile: int, vec: bool) -> torch.Tensor:
    """The paper's split SpMM (light rows + hubs): the hub-split
    mapping (src/kernels.cpp:260-334) with rows of degree >= hub_threshold cut
    into 2048-entry pieces whose f64 partials are summed in piece order;
    f_tile 0 = 64.  AUTOSAGE_HUB_T / AUTOSAGE_FTILE override as in dispatch."""
    if hub_threshold <= 0:
        raise ValueError("spmm_csr_split: hub_threshold must be > 0")
    variant = f"spmm:hubsplit:ft={f_tile if f_tile > 0 else 64}:rpc=1:vec={int(bool(vec))}:hubt={hub_threshold}"
    return _spmm_impl(crow, col, val, b, variant)


@spmm_csr_split.register_fake
def _(crow, col, val, b, hub_threshold, f_tile, vec):
    return b.new_empty((crow.shape[0] - 1, b.shape[1]), dtype=torch.float32)


@torch.library.custom_op("autosage::spmm_csr_auto", mutates_args=())
def spmm_csr_auto(crow: torch.Tensor, col: torch.Tensor, val: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """spmm_auto (src/scheduler.cpp:226-232) with a process-wide schedule cache."""
    if b.dim() != 2:
        raise ValueError("spmm_csr_auto: b must be 2-D")
    b = b.contiguous().float()
    g = _graph(crow, col, b.shape[0])
    vals = _values(val, g.nnz)
    c = torch.empty((g.n_rows, b.shape[1]), dtype=torch.float32, device=b.device)
    cctx, keep = _ctx(b).to_c()
    n0 = _cache_size()
    ccfg = ProbeConfig.from_env().to_c()
    d = _c.as_decision()
    if vals is None:
        _check(_lib.as_spmm_auto(C.byref(cctx), C.byref(ccfg), g.handle, C.c_void_p(b.data_ptr()), b.shape[0],
                                 b.shape[1], C.c_void_p(c.data_ptr()), C.byref(d)))
    else:
        _check(_lib.as_spmm_auto_values(C.byref(cctx), C.byref(ccfg), g.handle, _vptr(vals),
                                        C.c_void_p(b.data_ptr()), b.shape[0], b.shape[1],
                                        C.c_void_p(c.data_ptr()), C.byref(d)))
    del keep
    _persist(n0)
    return c


@spmm_csr_auto.register_fake
def _(crow, col, val, b):
    return b.new_empty((crow.shape[0] - 1, b.shape[1]))


@torch.library.custom_op("autosage::sddmm_csr", mutates_args=())
def sddmm_csr(crow: torch.Tensor, col: torch.Tensor, x: torch.Tensor, y: torch.Tensor,
              variant: str) -> torch.Tensor:
    """out[e] = <x[i], y[col[e]]> on A's pattern (src/kernels.cpp:336-429).
    bfloat16 / float16 x and y are read as 16-bit words (as_sddmm_bf16 / _f16; the f32 result on the
    widened operands, bit for bit); out is float32 either way."""
    _check_dense_pair("sddmm_csr", crow, x, y)
    g = _graph(crow, col, y.shape[0])
    out = torch.empty(col.numel(), dtype=torch.float32, device=x.device)
    if x.dtype in _HALF and y.dtype == x.dtype:
        x, y = x.contiguous(), y.contiguous()
        _check(_HALF[x.dtype][1](_variant(variant), g.handle, C.c_void_p(x.data_ptr()), x.shape[0],
                                  C.c_void_p(y.data_ptr()), y.shape[0], x.shape[1],
                                  C.c_void_p(out.data_ptr()) if out.numel() else None, _stream(x), None))
        return out
    x, y = x.contiguous().float(), y.contiguous().float()
    _check(_lib.as_sddmm(_variant(variant), g.handle, C.c_void_p(x.data_ptr()), x.shape[0],
                         C.c_void_p(y.data_ptr()), y.shape[0], x.shape[1],
                         C.c_void_p(out.data_ptr()) if out.numel() else None, _stream(x), None))
    return out


@torch.library.custom_op("autosage::sddmm_csr_auto", mutates_args=())
def sddmm_csr_auto(crow: torch.Tensor, col: torch.Tensor, x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
    """sddmm_auto (src/scheduler.cpp:234-239; the paper's sddmm_csr_auto,
    PAPER.md:286) with the process-wide schedule cache."""
    _check_dense_pair("sddmm_csr_auto", crow, x, y)
    x, y = x.contiguous().float(), y.contiguous().float()
    g = _graph(crow, col, y.shape[0])
    out = torch.empty(col.numel(), dtype=torch.float32, device=x.device)
    cctx, keep = _ctx(x).to_c()
    n0 = _cache_size()
    ccfg = ProbeConfig.from_env().to_c()
    d = _c.as_decision()
    _check(_lib.as_sddmm_auto(C.byref(cctx), C.byref(ccfg), g.handle, C.c_void_p(x.data_ptr()), x.shape[0],
                              C.c_void_p(y.data_ptr()), y.shape[0], x.shape[1],
                              C.c_void_p(out.data_ptr()) if out.numel() else None, C.byref(d)))
    del keep
    _persist(n0)
    return out


@sddmm_csr_auto.register_fake
def _(crow, col, x, y):
    return x.new_empty((col.shape[0],), dtype=torch.float32)


def _check_dense_pair(name, crow, x, y):
    """x: n_rows x F (one row per CSR row), y: n_cols x F (same F)."""
    if x.dim() != 2 or y.dim() != 2:
        raise ValueError(f"{name}: dense operands must be 2-D")
    if x.shape[0] != crow.numel() - 1:
        raise ValueError(f"{name}: x has {x.shape[0]} rows, the CSR {crow.numel() - 1}")
    if x.shape[1] != y.shape[1]:
        raise ValueError(f"{name}: feature widths differ ({x.shape[1]} vs {y.shape[1]})")


@sddmm_csr.register_fake
def _(crow, col, x, y, variant):
    return x.new_empty((col.shape[0],), dtype=torch.float32)


@torch.library.custom_op("autosage::csr_attention", mutates_args=())
def csr_attention(crow: torch.Tensor, col: torch.Tensor, q: torch.Tensor, k: torch.Tensor,
                  v: torch.Tensor, fused: bool) -> torch.Tensor:
    """csr_attention_forward (src/attention.cpp:9-40), decisions cached.
    bfloat16 / float16 q, k and v take the 16-bit route (_attention_half,
    fused or staged)."""
    _check_attention(crow, q, k, v)
    if _all_half(q, k, v):
        return _attention_half(crow, col, q, k, v, fused=fused)[0]
    q, k, v = q.contiguous().float(), k.contiguous().float(), v.contiguous().float()
    g = _graph(crow, col, k.shape[0])
    out = torch.empty((g.n_rows, v.shape[1]), dtype=torch.float32, device=q.device)
    cctx, keep = _ctx(q).to_c()
    n0 = _cache_size()
    ccfg = ProbeConfig.from_env().to_c()
    sd, pd = _c.as_decision(), _c.as_decision()
    _check(_lib.as_csr_attention_forward(C.byref(cctx), C.byref(ccfg), g.handle, C.c_void_p(q.data_ptr()),
                                         q.shape[0], C.c_void_p(k.data_ptr()), k.shape[0],
                                         C.c_void_p(v.data_ptr()), v.shape[0], q.shape[1], v.shape[1],
                                         C.c_void_p(out.data_ptr()), 1 if fused else 0, C.byref(sd),
                                         C.byref(pd)))
    del keep
    _persist(n0)
    return out


@csr_attention.register_fake
def _(crow, col, q, k, v, fused):
    return q.new_empty((crow.shape[0] - 1, v.shape[1]), dtype=torch.float32)


def _check_attention(crow, q, k, v):
    _check_dense_pair("csr_attention", crow, q, k)
    if v.dim() != 2 or v.shape[0] != k.shape[0]:
        raise ValueError("csr_attention: k and v need the same row count")


def _all_half(*ts) -> bool:
    return ts[0].dtype in _HALF and all(t.dtype == ts[0].dtype for t in ts)


def _attention_half(crow, col, q, k, v, fused=False, keep_p=False):
    """CSR attention on 16-bit q, k, v (bf16 or f16) through
    as_csr_attention_half with fixed variants (_BWD_SDDMM: the sequential dot
    order, src/kernels.cpp:336-355; _BWD_SPMM): (out, p) equal the f32
    pipeline sddmm_csr -> row_softmax_csr -> spmm_csr on q.float(), k.float(),
    v.float() with the same variants, bit for bit, while the Q/K/V gathers
    read half the bytes.  fused (and not keep_p): the probabilities are
    applied inside the SpMM and never stored (p returned empty).  out and p
    are float32."""
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    _check_attention(crow, q, k, v)
    pat = _graph(crow, col, k.shape[0])
    out = torch.empty((pat.n_rows, v.shape[1]), dtype=torch.float32, device=q.device)
    p = torch.empty(col.numel() if keep_p or not fused else 0, dtype=torch.float32, device=q.device)
    sv, pv = variant_from_string(_BWD_SDDMM).to_c(), variant_from_string(_BWD_SPMM).to_c()
    _check(_lib.as_csr_attention_half(pat.handle, C.byref(sv), C.byref(pv), C.c_void_p(q.data_ptr()), q.shape[0],
                                      C.c_void_p(k.data_ptr()), k.shape[0], C.c_void_p(v.data_ptr()), v.shape[0],
                                      q.shape[1], v.shape[1], C.c_void_p(out.data_ptr()),
                                      C.c_void_p(p.data_ptr()) if p.numel() else None, _HALF[q.dtype][2],
                                      0 if p.numel() else 1, _stream(q)))
    return out, p


# ---------------------------------------------------------------------------
# Backward
# ---------------------------------------------------------------------------
_BWD_SPMM = "spmm:hubsplit:ft=64:rpc=1:vec=1:hubt=256"
# sequential-order SDDMM (scalar variant: the same bits as the baseline, src/kernels.cpp:103-127)
_BWD_SDDMM = "sddmm:rowparallel:ft=32:rpc=1:vec=0:hubt=256"


def _spmm_vals(g: Graph, vals, b: torch.Tensor) -> torch.Tensor:
    """C = G[vals] B on torch's stream (vals None: G's own values / implicit 1)."""
    b = b.contiguous().float()
    c = torch.empty((g.n_rows, b.shape[1]), dtype=torch.float32, device=b.device)
    if vals is None:
        _check(_lib.as_spmm(_variant(_BWD_SPMM), g.handle, C.c_void_p(b.data_ptr()), b.shape[0],
                            b.shape[1], C.c_void_p(c.data_ptr()), _stream(b), None))
    else:
        vals = vals.contiguous().float()
        _check(_lib.as_spmm_values(_variant(_BWD_SPMM), g.handle,
                                   C.c_void_p(vals.data_ptr()) if vals.numel() else None,
                                   C.c_void_p(b.data_ptr()), b.shape[0], b.shape[1],
                                   C.c_void_p(c.data_ptr()), _stream(b), None))
    return c


def _spmm_t(crow, col, vals, n_cols: int, dc: torch.Tensor) -> torch.Tensor:
    """A^T[vals] dC: SpMM on the cached transpose, vals (source order) permuted."""
    gt = _transpose(crow, col, n_cols)
    if vals is None or vals.numel() == 0:
        return _spmm_vals(gt, None, dc)
    vals = vals.contiguous().float()
    dc = dc.contiguous().float()
    c = torch.empty((gt.n_rows, dc.shape[1]), dtype=torch.float32, device=dc.device)
    # the kernels read vals through the transpose's permutation (no permuted copy)
    _check(_lib.as_spmm_transpose_values(_variant(_BWD_SPMM), gt.handle, C.c_void_p(vals.data_ptr()),
                                         C.c_void_p(dc.data_ptr()), dc.shape[0], dc.shape[1],
                                         C.c_void_p(c.data_ptr()), _stream(dc), None))
    return c


@torch.library.custom_op("autosage::row_softmax_csr", mutates_args=())
def row_softmax_csr(crow: torch.Tensor, col: torch.Tensor, s: torch.Tensor, n_cols: int) -> torch.Tensor:
    """row_softmax over explicit values (src/kernels.cpp:431-461)."""
    s = s.contiguous().float()
    g = _graph(crow, col, n_cols)
    if s.numel() != g.nnz:
        raise ValueError(f"row_softmax_csr: {s.numel()} values for {g.nnz} entries")
    out = torch.empty_like(s)
    if s.numel():
        _check(_lib.as_row_softmax(g.handle, C.c_void_p(s.data_ptr()), C.c_void_p(out.data_ptr()),
                                   _stream(s)))
    return out


@row_softmax_csr.register_fake
def _(crow, col, s, n_cols):
    return torch.empty_like(s)


@torch.library.custom_op("autosage::row_softmax_csr_backward", mutates_args=())
def row_softmax_csr_backward(crow: torch.Tensor, col: torch.Tensor, p: torch.Tensor,
                             grad: torch.Tensor, n_cols: int) -> torch.Tensor:
    """ds = p * (grad - sum_row p*grad) (as_row_softmax_backward)."""
    p, grad = p.contiguous().float(), grad.contiguous().float()
    g = _graph(crow, col, n_cols)
    if p.numel() != g.nnz or grad.numel() != g.nnz:
        raise ValueError("row_softmax_csr_backward: p and grad need nnz entries")
    ds = torch.empty_like(p)  # every entry is written (empty rows have none)
    if p.numel():
        _check(_lib.as_row_softmax_backward(g.handle, C.c_void_p(p.data_ptr()), C.c_void_p(grad.data_ptr()),
                                            C.c_void_p(ds.data_ptr()), _stream(p)))
    return ds


@row_softmax_csr_backward.register_fake
def _(crow, col, p, grad, n_cols):
    return torch.empty_like(p)


def _softmax_setup(ctx, inputs, output):
    crow, col, _, n_cols = inputs
    ctx.n_cols = n_cols
    ctx.save_for_backward(crow, col, output)


def _softmax_bwd(ctx, grad):
    crow, col, p = ctx.saved_tensors
    return None, None, row_softmax_csr_backward(crow, col, p, grad, ctx.n_cols), None


row_softmax_csr.register_autograd(_softmax_bwd, setup_context=_softmax_setup)


def _spmm_setup(ctx, inputs, output):
    crow, col, val, b = inputs[:4]
    ctx.save_for_backward(crow, col, val, b)


def _spmm_bwd(ctx, dc):
    crow, col, val, b = ctx.saved_tensors
    dval = db = None
    if ctx.needs_input_grad[2] and val.numel():
        dval = sddmm_csr(crow, col, dc, b.float(), _BWD_SDDMM)
    if ctx.needs_input_grad[3]:
        db = _spmm_t(crow, col, val if val.numel() else None, b.shape[0], dc).to(b.dtype)
    return (None, None, dval, db) + (None,) * (ctx.n_extra)


def _spmm_setup_v(ctx, inputs, output):
    _spmm_setup(ctx, inputs, output)
    ctx.n_extra = 1


def _spmm_setup_auto(ctx, inputs, output):
    _spmm_setup(ctx, inputs, output)
    ctx.n_extra = 0


def _spmm_setup_split(ctx, inputs, output):
    _spmm_setup(ctx, inputs, output)
    ctx.n_extra = 3


spmm_csr.register_autograd(_spmm_bwd, setup_context=_spmm_setup_v)
spmm_csr_split.register_autograd(_spmm_bwd, setup_context=_spmm_setup_split)
spmm_csr_auto.register_autograd(_spmm_bwd, setup_context=_spmm_setup_auto)


def _sddmm_setup(ctx, inputs, output):
    crow, col, x, y = inputs[:4]
    ctx.save_for_backward(crow, col, x, y)
    ctx.n_extra = len(inputs) - 4


def _sddmm_bwd(ctx, dout):
    crow, col, x, y = ctx.saved_tensors
    dx = dy = None
    if ctx.needs_input_grad[2]:
        dx = _spmm_vals(_graph(crow, col, y.shape[0]), dout, y).to(x.dtype)
    if ctx.needs_input_grad[3]:
        dy = _spmm_t(crow, col, dout, y.shape[0], x).to(y.dtype)
    return (None, None, dx, dy) + (None,) * ctx.n_extra


sddmm_csr.register_autograd(_sddmm_bwd, setup_context=_sddmm_setup)
sddmm_csr_auto.register_autograd(_sddmm_bwd, setup_context=_sddmm_setup)


def _attention_setup(ctx, inputs, output):
    crow, col, q, k, v, _ = inputs
    ctx.save_for_backward(crow, col, q, k, v)


def _attention_bwd(ctx, do):
    """Staged recompute: s = SDDMM(q, k), p = softmax(s); then dv = A^T[p] dO,
    dp = SDDMM(dO, v), ds = softmax'(p, dp), dq = A[ds] k, dk = A^T[ds] q."""
    crow, col, q, k, v = ctx.saved_tensors
    s = sddmm_csr(crow, col, q, k, _BWD_SDDMM)
    p = row_softmax_csr(crow, col, s, k.shape[0])
    dv = _spmm_t(crow, col, p, k.shape[0], do) if ctx.needs_input_grad[4] else None
    dp = sddmm_csr(crow, col, do, v, _BWD_SDDMM)
    ds = row_softmax_csr_backward(crow, col, p, dp, k.shape[0])
    pat = _graph(crow, col, k.shape[0])
    dq = _spmm_vals(pat, ds, k).to(q.dtype) if ctx.needs_input_grad[2] else None
    dk = _spmm_t(crow, col, ds, k.shape[0], q).to(k.dtype) if ctx.needs_input_grad[3] else None
    return None, None, dq, dk, None if dv is None else dv.to(v.dtype), None


csr_attention.register_autograd(_attention_bwd, setup_context=_attention_setup)


# ---------------------------------------------------------------------------
# Training form of the attention: keeps p for the backward
# ---------------------------------------------------------------------------
@torch.library.custom_op("autosage::csr_attention_with_probs", mutates_args=())
def csr_attention_with_probs(crow: torch.Tensor, col: torch.Tensor, q: torch.Tensor, k: torch.Tensor,
                             v: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """(out, p): the staged pipeline (as_csr_attention_forward_p), p = the row
    softmax of the scores (nnz floats).  out is bit-identical to csr_attention;
    its backward reuses p instead of recomputing SDDMM + softmax.  bfloat16 /
    float16 q, k and v take the 16-bit route (_attention_half, p kept)."""
    _check_attention(crow, q, k, v)
    if _all_half(q, k, v):
        return _attention_half(crow, col, q, k, v, keep_p=True)
    q, k, v = q.contiguous().float(), k.contiguous().float(), v.contiguous().float()
    g = _graph(crow, col, k.shape[0])
    out = torch.empty((g.n_rows, v.shape[1]), dtype=torch.float32, device=q.device)
    p = torch.empty(col.numel(), dtype=torch.float32, device=q.device)
    cctx, keep = _ctx(q).to_c()
    n0 = _cache_size()
    ccfg = ProbeConfig.from_env().to_c()
    sd, pd = _c.as_decision(), _c.as_decision()
    _check(_lib.as_csr_attention_forward_p(C.byref(cctx), C.byref(ccfg), g.handle, C.c_void_p(q.data_ptr()),
                                           q.shape[0], C.c_void_p(k.data_ptr()), k.shape[0],
                                           C.c_void_p(v.data_ptr()), v.shape[0], q.shape[1], v.shape[1],
                                           C.c_void_p(out.data_ptr()), C.c_void_p(p.data_ptr()) if p.numel() else None,
                                           C.byref(sd), C.byref(pd)))
    del keep
    _persist(n0)
    return out, p


@csr_attention_with_probs.register_fake
def _(crow, col, q, k, v):
    return (q.new_empty((crow.shape[0] - 1, v.shape[1]), dtype=torch.float32),
            q.new_empty((col.shape[0],), dtype=torch.float32))


def _attention_p_setup(ctx, inputs, output):
    crow, col, q, k, v = inputs
    ctx.save_for_backward(crow, col, q, k, v, output[1])


def _attention_p_bwd(ctx, do, gp):
    """dv = A^T[p] dO, dp = SDDMM(dO, v) (+ the gradient reaching p directly),
    ds = softmax'(p, dp), dq = A[ds] k, dk = A^T[ds] q -- p from the forward."""
    crow, col, q, k, v, p = ctx.saved_tensors
    n_cols = k.shape[0]
    dv = dq = dk = None
    if do is None:
        do = torch.zeros((crow.shape[0] - 1, v.shape[1]), dtype=torch.float32, device=q.device)
    if ctx.needs_input_grad[4]:
        dv = _spmm_t(crow, col, p, n_cols, do)
    dp = sddmm_csr(crow, col, do, v, _BWD_SDDMM)
    if gp is not None:
        dp = dp + gp
    ds = row_softmax_csr_backward(crow, col, p, dp, n_cols)
    if ctx.needs_input_grad[2]:
        dq = _spmm_vals(_graph(crow, col, n_cols), ds, k).to(q.dtype)
    if ctx.needs_input_grad[3]:
        dk = _spmm_t(crow, col, ds, n_cols, q).to(k.dtype)
    return None, None, dq, dk, None if dv is None else dv.to(v.dtype)


csr_attention_with_probs.register_autograd(_attention_p_bwd, setup_context=_attention_p_setup)


def csr_attention_train(crow, col, q, k, v) -> torch.Tensor:
    """CSR attention for training: the forward keeps p (4 bytes per nonzero)
    so the backward skips the SDDMM + softmax recompute of csr_attention."""
    return csr_attention_with_probs(crow, col, q, k, v)[0]
