"""ctypes declarations for include/autosage_b200.h (the library's C-ABI).

Loads ``libautosage_b200.so`` from this package directory and fails loudly
when it is missing: there is no CPU fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# AUTOSAGE_DEV_LIB: an alternative in-tree build for developer A/B runs
LIB_PATH = os.environ.get("AUTOSAGE_DEV_LIB") or os.path.join(_HERE, "libautosage_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
        "(or `make -C paper_2511_17594_b200`). The B200 library has no CPU fallback."
    )

lib = C.CDLL(LIB_PATH)

u64, i32, u32, dbl = C.c_uint64, C.c_int32, C.c_uint32, C.c_double
vp, cp = C.c_void_p, C.c_char_p
P = C.POINTER

AS_OK = 0
AS_INVALID_ARGUMENT = 1
AS_CACHE_ERROR = 2
AS_IO_ERROR = 3
AS_REPLAY_MISS = 4
AS_CUDA_ERROR = 5
AS_OUT_OF_MEMORY = 6
AS_LOGIC_ERROR = 7
AS_INTERNAL = 8

AS_MAX_CANDIDATES = 36


class as_variant(C.Structure):
    _fields_ = [("op", i32), ("mapping", i32), ("f_tile", u64), ("rows_per_chunk", u64),
                ("vectorized", i32), ("hub_threshold", u64)]


class as_kernel_result(C.Structure):
    _fields_ = [("variant", as_variant), ("vectorized_path", i32), ("elapsed_ms", dbl)]


class as_features(C.Structure):
    _fields_ = [("n_rows", u64), ("n_cols", u64), ("nnz", u64), ("deg_p25", u64),
                ("deg_p50", u64), ("deg_p75", u64), ("deg_p90", u64), ("deg_p99", u64),
                ("deg_max", u64), ("mean_degree", dbl), ("heavy_row_fraction", dbl),
                ("empty_row_fraction", dbl), ("hub_threshold", u64)]


class as_device_profile(C.Structure):
    _fields_ = [("device_sig", C.c_char * 256), ("bw_eff", dbl), ("flops_eff", dbl),
                ("cores", u64), ("model", C.c_int32)]


class as_timed_stats(C.Structure):
    _fields_ = [("median_ms", dbl), ("completed", i32), ("capped", i32), ("max_run_ms", dbl),
                ("wall_ms", dbl), ("launches", i32)]


class as_key(C.Structure):
    _fields_ = [("device_sig", C.c_char * 256), ("graph_sig", u64), ("f", u64), ("op", i32)]


class as_record(C.Structure):
    _fields_ = [("key", as_key), ("choice", C.c_char * 128), ("t_b", dbl), ("t_star", dbl),
                ("alpha", dbl), ("timestamp", u64), ("schema_version", u32),
                ("toolchain", C.c_char * 64)]


class as_probe_config(C.Structure):
    _fields_ = [("frac", dbl), ("min_rows", u64), ("iters", i32), ("cap_ms", dbl),
                ("top_k", i32), ("alpha", dbl)]


class as_replay_policy(C.Structure):
    _fields_ = [("replay_only", i32), ("strict", i32)]


class as_candidate_timing(C.Structure):
    _fields_ = [("variant", as_variant), ("median_ms", dbl), ("completed", i32), ("capped", i32)]


class as_decision(C.Structure):
    _fields_ = [("has_choice", i32), ("choice", as_variant), ("source", i32), ("key", as_key),
                ("alpha", dbl), ("baseline_ms", dbl), ("baseline_completed", i32),
                ("baseline_capped", i32), ("n_candidates", i32),
                ("candidates", as_candidate_timing * AS_MAX_CANDIDATES), ("best_index", i32),
                ("t_star", dbl), ("sample_rows", u64), ("probe_wall_ms", dbl),
                ("max_single_run_ms", dbl), ("sig_ms", dbl), ("features_ms", dbl),
                ("sample_ms", dbl), ("decide_wall_ms", dbl)]


RUN_FN = C.CFUNCTYPE(None, vp)
TIME_ONCE_FN = C.CFUNCTYPE(dbl, vp, cp, RUN_FN, vp)


class as_context(C.Structure):
    _fields_ = [("device", P(as_device_profile)), ("cache", vp), ("timer", TIME_ONCE_FN),
                ("timer_user", vp), ("replay", as_replay_policy), ("stream", vp)]


def _proto(name, restype, *argtypes):
    fn = getattr(lib, name)
    fn.restype = restype
    fn.argtypes = list(argtypes)
    return fn


st = C.c_int  # as_status

_proto("as_last_error", cp)
_proto("as_abi_version", C.c_int)
_proto("as_artifact_version", cp)
_proto("as_kernel_launch_count", u64)
_proto("as_variant_default", None, P(as_variant))
_proto("as_variant_to_string", st, P(as_variant), C.c_char_p, C.c_size_t)
_proto("as_variant_from_string", st, cp, P(as_variant))
_proto("as_vec4_eligible", C.c_int, u64, P(vp), C.c_int)
_proto("as_graph_create", st, vp, vp, vp, u64, u64, u64, C.c_int, P(vp))
_proto("as_graph_create_device", st, vp, vp, vp, u64, u64, u64, C.c_int, vp, P(vp))
_proto("as_graph_destroy", st, vp)
_proto("as_graph_shape", st, vp, P(u64), P(u64), P(u64), P(C.c_int))
_proto("as_graph_device_arrays", st, vp, P(vp), P(vp), P(vp))
_proto("as_graph_set_values", st, vp, vp, C.c_int)
_proto("as_validate", st, vp, vp, vp, u64, u64, u64, u64, u64, P(C.c_int), C.c_char_p,
       C.c_size_t, P(u64))
_proto("as_graph_sig", st, vp, P(u64))
_proto("as_graph_sig_host", u64, vp, vp, u64, u64, u64)
_proto("as_graph_features", st, vp, u64, P(as_features))
_proto("as_sample_row_indices", st, vp, dbl, u64, vp, P(u64))
_proto("as_slice_rows", st, vp, vp, u64, P(vp))
_proto("as_graph_download", st, vp, vp, vp, vp)
_proto("as_spmm", st, P(as_variant), vp, vp, u64, u64, vp, vp, P(as_kernel_result))
_proto("as_spmm_rowparallel", st, P(as_variant), vp, vp, u64, u64, vp, vp)
_proto("as_spmm_hubsplit", st, P(as_variant), vp, vp, u64, u64, vp, vp)
_proto("as_sddmm", st, P(as_variant), vp, vp, u64, vp, u64, u64, vp, vp, P(as_kernel_result))
_proto("as_sddmm_rowparallel", st, P(as_variant), vp, vp, u64, vp, u64, u64, vp, vp)
_proto("as_row_softmax", st, vp, vp, vp, vp)
_proto("as_spmm_host", st, P(as_variant), vp, vp, u64, u64, vp, P(as_kernel_result))
_proto("as_sddmm_host", st, P(as_variant), vp, vp, u64, vp, u64, u64, vp, P(as_kernel_result))
_proto("as_row_softmax_host", st, vp, vp, vp)
_proto("as_spmm_host_async", st, P(as_variant), vp, vp, u64, u64, vp, P(as_kernel_result))
_proto("as_sddmm_host_async", st, P(as_variant), vp, vp, u64, vp, u64, u64, vp, P(as_kernel_result))
_proto("as_graph_synchronize", st, vp)
_proto("as_device_profile_gpu", st, C.c_int, P(as_device_profile))
_proto("as_device_profile_fixed", None, dbl, dbl, u64, cp, P(as_device_profile))
_proto("as_estimate_cost", st, P(as_variant), P(as_features), u64, P(as_device_profile),
       P(dbl))
_proto("as_shortlist", st, P(as_features), u64, C.c_int, P(as_device_profile), P(as_variant),
       P(C.c_int))
_proto("as_time_kernel", st, cp, RUN_FN, vp, C.c_int, dbl, TIME_ONCE_FN, vp, P(as_timed_stats))
_proto("as_cache_create", st, P(vp))
_proto("as_cache_destroy", st, vp)
_proto("as_cache_get", st, vp, P(as_key), P(as_record), P(C.c_int))
_proto("as_cache_put", st, vp, P(as_record))
_proto("as_cache_size", st, vp, P(u64))
_proto("as_cache_snapshot", st, vp, P(as_record), u64, P(u64))
_proto("as_cache_clear", st, vp)
_proto("as_cache_load", st, vp, cp)
_proto("as_cache_store", st, vp, cp)
_proto("as_record_to_line", st, P(as_record), C.c_char_p, C.c_size_t)
_proto("as_record_from_line", st, cp, P(as_record))
_proto("as_key_to_string", st, P(as_key), C.c_char_p, C.c_size_t)
_proto("as_toolchain_tag", cp)
_proto("as_probe_config_default", None, P(as_probe_config))
_proto("as_probe_config_from_env", None, P(as_probe_config))
_proto("as_replay_policy_from_env", None, P(as_replay_policy))
_proto("as_decide_spmm", st, P(as_context), P(as_probe_config), vp, vp, u64, u64,
       P(as_decision))
_proto("as_decide_sddmm", st, P(as_context), P(as_probe_config), vp, vp, u64, vp, u64, u64,
       P(as_decision))
_proto("as_spmm_auto", st, P(as_context), P(as_probe_config), vp, vp, u64, u64, vp,
       P(as_decision))
_proto("as_spmm_auto_values", st, P(as_context), P(as_probe_config), vp, vp, vp, u64, u64, vp,
       P(as_decision))
_proto("as_sddmm_auto", st, P(as_context), P(as_probe_config), vp, vp, u64, vp, u64, u64, vp,
       P(as_decision))
_proto("as_probe_launch_count", u64)
_proto("as_reset_probe_launch_count", None)
_proto("as_decide_host", st, P(as_context), P(as_probe_config), u64, P(as_features), u64,
       C.c_int, u64, P(as_decision))
_proto("as_csr_attention_forward", st, P(as_context), P(as_probe_config), vp, vp, u64, vp, u64,
       vp, u64, u64, u64, vp, C.c_int, P(as_decision), P(as_decision))
_proto("as_csr_attention_forward_heads", st, P(as_context), P(as_probe_config), vp, u32, vp, u64, vp, u64,
       vp, u64, u64, u64, vp, C.c_int, P(as_decision), P(as_decision))
_proto("as_csr_attention_forward_p", st, P(as_context), P(as_probe_config), vp, vp, u64, vp, u64,
       vp, u64, u64, u64, vp, vp, P(as_decision), P(as_decision))
_proto("as_partition_rows", st, vp, u64, u32, vp)
_proto("as_graph_row_range", st, vp, u64, u64, P(vp))
_proto("as_spmm_blocked_create", st, vp, P(as_variant), vp, u32, P(vp))
_proto("as_spmm_blocked_run", st, vp, u32, vp, vp, u64, u64, vp, vp)
_proto("as_spmm_blocked_destroy", st, vp)
_proto("as_graph_transpose", st, vp, P(vp))
_proto("as_graph_transpose_perm", st, vp, P(vp))
_proto("as_permute_values", st, vp, vp, vp, vp)
_proto("as_spmm_values", st, P(as_variant), vp, vp, vp, u64, u64, vp, vp, P(as_kernel_result))
_proto("as_row_softmax_backward", st, vp, vp, vp, vp, vp)
_proto("as_spmm_bf16", st, P(as_variant), vp, vp, vp, u64, u64, vp, vp, P(as_kernel_result))
_proto("as_spmm_transpose_values", st, P(as_variant), vp, vp, vp, u64, u64, vp, vp, P(as_kernel_result))
_proto("as_sddmm_bf16", st, P(as_variant), vp, vp, u64, vp, u64, u64, vp, vp, P(as_kernel_result))
_proto("as_csr_attention_half", st, vp, P(as_variant), P(as_variant), vp, u64, vp, u64, vp, u64, u64, u64, vp, vp,
       C.c_int, C.c_int, vp)
_proto("as_spmm_f16", st, P(as_variant), vp, vp, vp, u64, u64, vp, vp, P(as_kernel_result))
_proto("as_sddmm_f16", st, P(as_variant), vp, vp, u64, vp, u64, u64, vp, vp, P(as_kernel_result))
_proto("as_gen_powerlaw", st, u64, u64, u64, dbl, u64, u64, u64, C.c_int, P(vp), P(vp), P(vp),
       P(u64))
_proto("as_fill_uniform", st, vp, u64, u64)
_proto("as_free", None, vp)
_proto("as_save_csr", st, cp, vp, vp, vp, u64, u64, u64)
_proto("as_load_csr", st, cp, P(vp), P(vp), P(vp), P(u64), P(u64), P(u64))
_proto("as_host_alloc", st, P(vp), u64)
_proto("as_host_free", st, vp)

# every symbol the header declares (checked by tests/test_capi.py)
EXPORTED = [
    "as_last_error", "as_abi_version", "as_artifact_version", "as_variant_default",
    "as_variant_to_string", "as_variant_from_string", "as_vec4_eligible", "as_graph_create",
    "as_graph_create_device", "as_graph_destroy", "as_graph_shape", "as_graph_device_arrays",
    "as_graph_set_values", "as_validate", "as_graph_sig", "as_graph_sig_host",
    "as_graph_features", "as_sample_row_indices", "as_slice_rows", "as_graph_download",
    "as_spmm", "as_spmm_rowparallel", "as_spmm_hubsplit", "as_sddmm", "as_sddmm_rowparallel",
    "as_row_softmax",
    "as_spmm_host", "as_sddmm_host", "as_row_softmax_host", "as_spmm_host_async",
    "as_sddmm_host_async", "as_graph_synchronize", "as_device_profile_gpu",
    "as_device_profile_fixed", "as_estimate_cost", "as_shortlist", "as_time_kernel",
    "as_cache_create", "as_cache_destroy", "as_cache_get", "as_cache_put", "as_cache_size",
    "as_cache_snapshot", "as_cache_clear", "as_cache_load", "as_cache_store",
    "as_record_to_line", "as_record_from_line", "as_key_to_string", "as_toolchain_tag",
    "as_probe_config_default", "as_probe_config_from_env", "as_replay_policy_from_env",
    "as_decide_spmm", "as_decide_sddmm", "as_spmm_auto", "as_sddmm_auto",
    "as_probe_launch_count", "as_reset_probe_launch_count", "as_decide_host",
    "as_csr_attention_forward", "as_partition_rows", "as_graph_row_range", "as_gen_powerlaw",
    "as_fill_uniform", "as_free", "as_save_csr", "as_load_csr", "as_host_alloc",
    "as_host_free", "as_kernel_launch_count", "as_graph_transpose", "as_graph_transpose_perm",
    "as_permute_values", "as_spmm_values", "as_row_softmax_backward", "as_spmm_bf16",
    "as_sddmm_bf16", "as_spmm_transpose_values", "as_csr_attention_forward_p", "as_spmm_auto_values",
    "as_spmm_blocked_create", "as_spmm_blocked_run", "as_spmm_blocked_destroy", "as_spmm_f16", "as_sddmm_f16",
    "as_csr_attention_half", "as_csr_attention_forward_heads",
]
