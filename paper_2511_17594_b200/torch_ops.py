"""PyTorch custom operators over the C-ABI (the paper's
integration surface).

    import paper_2511_17594_b200.torch_ops  # registers torch.ops.autosage.*
    c = torch.ops.autosage.spmm_csr(crow, col, val, b, "spmm:hubsplit:ft=64:rpc=4:vec=1:hubt=256")
    c = torch.ops.autosage.spmm_csr_auto(crow, col, val, b)       # decide (cached) + run
    s = torch.ops.autosage.sddmm_csr(crow, col, x, y, "")          # "" = baseline
    o = torch.ops.autosage.csr_attention(crow, col, q, k, v, False)

CSR arrays are CUDA tensors: crow int64 [n_rows + 1], col int32 [nnz],
values float32 [nnz] (optional: pass an empty tensor for pattern-only).  The
number of columns is the dense operand's row count.  Results are computed on
torch's current stream by the sm_100a kernels, with the same numerics as the
reference (bit-exact SpMM/SDDMM).  Device graph handles (upload, degree
order, hub plans) are cached per CSR storage, so repeated calls on a static
graph pay the setup once.  Forward only (backward kernels are SURVEY 8(f) N4).
"""
from __future__ import annotations

import ctypes as C
from collections import OrderedDict

import torch

from . import (Graph, ProbeConfig, ScheduleCache, ScheduleContext, _check, _lib, torch_stream_handle,
               variant_from_string)
from . import _capi as _c

_GRAPHS: "OrderedDict[tuple, Graph]" = OrderedDict()
_MAX_GRAPHS = 8
_CACHE = None


def _key(crow, col, val, n_cols):
    return (crow.data_ptr(), col.data_ptr(), val.data_ptr() if val.numel() else 0, crow.numel() - 1,
            int(n_cols), col.numel(), crow._version, col._version, val._version, crow.device.index)


def _graph(crow: torch.Tensor, col: torch.Tensor, val: torch.Tensor, n_cols: int) -> Graph:
    if not (crow.is_cuda and col.is_cuda):
        raise ValueError("autosage ops take CUDA CSR tensors")
    if crow.dtype != torch.int64 or col.dtype != torch.int32:
        raise ValueError("crow must be int64 and col int32")
    k = _key(crow, col, val, n_cols)
    g = _GRAPHS.get(k)
    if g is not None:
        _GRAPHS.move_to_end(k)
        return g
    crow_c, col_c = crow.contiguous(), col.contiguous()
    has_val = val.numel() > 0
    val_c = val.contiguous().float() if has_val else None
    h = C.c_void_p()
    _check(_lib.as_graph_create_device(C.c_void_p(crow_c.data_ptr()), C.c_void_p(col_c.data_ptr()),
                                       C.c_void_p(val_c.data_ptr()) if has_val else None,
                                       crow_c.numel() - 1, int(n_cols), col_c.numel(),
                                       crow.device.index or 0, C.byref(h)))
    g = Graph(h.value, crow.device.index or 0)
    _GRAPHS[k] = g
    while len(_GRAPHS) > _MAX_GRAPHS:
        _GRAPHS.popitem(last=False)[1].close()
    return g


def _variant(s: str):
    return None if not s or s == "baseline" else C.byref(variant_from_string(s).to_c())


def _stream(t: torch.Tensor):
    return C.c_void_p(torch_stream_handle(t.device))


def _ctx(t: torch.Tensor):
    global _CACHE
    if _CACHE is None:
        _CACHE = ScheduleCache()
    return ScheduleContext(cache=_CACHE, stream=torch_stream_handle(t.device))


@torch.library.custom_op("autosage::spmm_csr", mutates_args=())
def spmm_csr(crow: torch.Tensor, col: torch.Tensor, val: torch.Tensor, b: torch.Tensor,
             variant: str) -> torch.Tensor:
    """C = A B (dispatch(variant, A, B), src/kernels.cpp:485-506; "" = baseline)."""
    b = b.contiguous().float()
    g = _graph(crow, col, val, b.shape[0])
    c = torch.empty((g.n_rows, b.shape[1]), dtype=torch.float32, device=b.device)
    _check(_lib.as_spmm(_variant(variant), g.handle, C.c_void_p(b.data_ptr()), b.shape[0], b.shape[1],
                        C.c_void_p(c.data_ptr()), _stream(b), None))
    return c


@spmm_csr.register_fake
def _(crow, col, val, b, variant):
    return b.new_empty((crow.shape[0] - 1, b.shape[1]))


@torch.library.custom_op("autosage::spmm_csr_auto", mutates_args=())
def spmm_csr_auto(crow: torch.Tensor, col: torch.Tensor, val: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """spmm_auto (src/scheduler.cpp:226-232) with a process-wide schedule cache."""
    b = b.contiguous().float()
    g = _graph(crow, col, val, b.shape[0])
    c = torch.empty((g.n_rows, b.shape[1]), dtype=torch.float32, device=b.device)
    cctx, keep = _ctx(b).to_c()
    ccfg = ProbeConfig.from_env().to_c()
    d = _c.as_decision()
    _check(_lib.as_spmm_auto(C.byref(cctx), C.byref(ccfg), g.handle, C.c_void_p(b.data_ptr()), b.shape[0],
                             b.shape[1], C.c_void_p(c.data_ptr()), C.byref(d)))
    del keep
    return c


@spmm_csr_auto.register_fake
def _(crow, col, val, b):
    return b.new_empty((crow.shape[0] - 1, b.shape[1]))


@torch.library.custom_op("autosage::sddmm_csr", mutates_args=())
def sddmm_csr(crow: torch.Tensor, col: torch.Tensor, x: torch.Tensor, y: torch.Tensor,
              variant: str) -> torch.Tensor:
    """out[e] = <x[i], y[col[e]]> on A's pattern (src/kernels.cpp:336-429)."""
    x, y = x.contiguous().float(), y.contiguous().float()
    empty = torch.empty(0, dtype=torch.float32, device=x.device)
    g = _graph(crow, col, empty, y.shape[0])
    out = torch.empty(col.numel(), dtype=torch.float32, device=x.device)
    _check(_lib.as_sddmm(_variant(variant), g.handle, C.c_void_p(x.data_ptr()), x.shape[0],
                         C.c_void_p(y.data_ptr()), y.shape[0], x.shape[1],
                         C.c_void_p(out.data_ptr()) if out.numel() else None, _stream(x), None))
    return out


@sddmm_csr.register_fake
def _(crow, col, x, y, variant):
    return x.new_empty((col.shape[0],))


@torch.library.custom_op("autosage::csr_attention", mutates_args=())
def csr_attention(crow: torch.Tensor, col: torch.Tensor, q: torch.Tensor, k: torch.Tensor,
                  v: torch.Tensor, fused: bool) -> torch.Tensor:
    """csr_attention_forward (src/attention.cpp:9-40), decisions cached."""
    q, k, v = q.contiguous().float(), k.contiguous().float(), v.contiguous().float()
    empty = torch.empty(0, dtype=torch.float32, device=q.device)
    g = _graph(crow, col, empty, k.shape[0])
    out = torch.empty((g.n_rows, v.shape[1]), dtype=torch.float32, device=q.device)
    cctx, keep = _ctx(q).to_c()
    ccfg = ProbeConfig.from_env().to_c()
    sd, pd = _c.as_decision(), _c.as_decision()
    _check(_lib.as_csr_attention_forward(C.byref(cctx), C.byref(ccfg), g.handle, C.c_void_p(q.data_ptr()),
                                         q.shape[0], C.c_void_p(k.data_ptr()), k.shape[0],
                                         C.c_void_p(v.data_ptr()), v.shape[0], q.shape[1], v.shape[1],
                                         C.c_void_p(out.data_ptr()), 1 if fused else 0, C.byref(sd),
                                         C.byref(pd)))
    del keep
    return out


@csr_attention.register_fake
def _(crow, col, q, k, v, fused):
    return q.new_empty((crow.shape[0] - 1, v.shape[1]))
