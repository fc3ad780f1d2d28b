/*
 * autosage_b200.h -- C-ABI of the B200-native AutoSAGE library
 * (libautosage_b200.so, built from paper_2511_17594_b200/csrc).
 *
 * The reference (arxiv 2511.17594, /root/reference/proj) is a C++20 static
 * library whose public interface is the headers under
 * proj/include/autosage/<name>.hpp; it ships no FFI.  Each entry point below
 * names the reference declaration it replaces (file:line, relative to
 * proj/).  Plain pointers and sizes only; no C++ or torch types cross the
 * boundary.
 *
 * Conventions
 *  - Every call returns as_status; on failure as_last_error() holds the
 *    message (thread-local), using the reference's exception texts where the
 *    reference throws (std::invalid_argument -> AS_INVALID_ARGUMENT,
 *    CacheError -> AS_CACHE_ERROR, IoError -> AS_IO_ERROR,
 *    ReplayMiss -> AS_REPLAY_MISS).
 *  - "dev" pointers are CUDA device pointers on the graph's device; "host"
 *    pointers are host memory (pinned or pageable).  Dense matrices are
 *    row-major with row stride == number of columns (the reference's
 *    DenseMatrix layout, include/autosage/csr.hpp:51-89).
 *  - stream == NULL selects the graph's internal stream.  Calls that return
 *    an as_kernel_result with a non-NULL pointer synchronize that stream (the
 *    reference's dispatch is synchronous and reports elapsed_ms); calls with
 *    NULL result pointers are asynchronous on the stream.
 */
#ifndef AUTOSAGE_B200_H
#define AUTOSAGE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AS_ABI_VERSION 2

typedef enum {
    AS_OK = 0,
    AS_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference       */
    AS_CACHE_ERROR = 2,      /* CacheError, include/autosage/cache.hpp:16-18 */
    AS_IO_ERROR = 3,         /* IoError, include/autosage/io.hpp:10-12       */
    AS_REPLAY_MISS = 4,      /* ReplayMiss, include/autosage/cache.hpp:78-81 */
    AS_CUDA_ERROR = 5,
    AS_OUT_OF_MEMORY = 6,
    AS_LOGIC_ERROR = 7,      /* e.g. a scripted timer running dry            */
    AS_INTERNAL = 8
} as_status;

/* Thread-local text of the last failure on this thread. */
const char* as_last_error(void);
int as_abi_version(void);
/* Artifact version folded into device signatures
 * (include/autosage/version.hpp:6 kArtifactVersion). */
const char* as_artifact_version(void);

/* ------------------------------------------------------------------ */
/* Variants -- include/autosage/kernels.hpp:12-34                      */
/* ------------------------------------------------------------------ */
enum { AS_OP_SPMM = 0, AS_OP_SDDMM = 1 };
enum { AS_MAP_BASELINE = 0, AS_MAP_ROWPARALLEL = 1, AS_MAP_HUBSPLIT = 2 };
#define AS_DEFAULT_HUB_THRESHOLD 256 /* include/autosage/csr.hpp:18 */

typedef struct {
    int32_t op;              /* AS_OP_*                                     */
    int32_t mapping;         /* AS_MAP_*                                    */
    uint64_t f_tile;         /* features per (sub)warp pass                 */
    uint64_t rows_per_chunk; /* GPU: warps per CTA (AUTOSAGE_WPB)           */
    int32_t vectorized;      /* float4 path when the vec4 gate passes       */
    uint64_t hub_threshold;  /* degree >= hub_threshold => heavy (HubSplit)  */
} as_variant;

/* KernelVariant{} defaults (include/autosage/kernels.hpp:21-30). */
void as_variant_default(as_variant* v);
/* variant_to_string, src/kernels.cpp:159-165 ("spmm:hubsplit:ft=..."). */
as_status as_variant_to_string(const as_variant* v, char* buf, size_t cap);
/* variant_from_string, src/kernels.cpp:167-200. */
as_status as_variant_from_string(const char* s, as_variant* out);
/* vec4_eligible, src/kernels.cpp:202-208, on raw base pointers. */
int as_vec4_eligible(uint64_t f, const void* const* bases, int n_bases);

typedef struct {
    as_variant variant;      /* variant after env overrides                 */
    int32_t vectorized_path; /* the 4-wide path actually ran                */
    double elapsed_ms;       /* CUDA-event time of the launch(es)           */
} as_kernel_result;          /* KernelResult, include/autosage/kernels.hpp:36-42 */

/* ------------------------------------------------------------------ */
/* Graphs: a device-resident CsrMatrix (include/autosage/csr.hpp:24-45) */
/* ------------------------------------------------------------------ */
typedef struct as_graph_s* as_graph;

/* Validates (src/csr.cpp:62-93, first violation -> AS_INVALID_ARGUMENT
 * naming invariant and index) and uploads.  val == NULL: pattern-only CSR
 * (implicit 1.0).  device < 0: current device. */
as_status as_graph_create(const uint64_t* rowptr_host, const uint32_t* colind_host,
                          const float* val_host, uint64_t n_rows, uint64_t n_cols,
                          uint64_t nnz, int device, as_graph* out);
/* Same from device arrays (copied).  The copies are ordered after the work
 * already enqueued on `stream` (the stream that produced the arrays; NULL =
 * the legacy default stream).  Validated on the device: rowptr as for
 * as_graph_create; columns < n_cols and strictly increasing in each row. */
as_status as_graph_create_device(const uint64_t* rowptr_dev, const uint32_t* colind_dev,
                                 const float* val_dev, uint64_t n_rows, uint64_t n_cols,
                                 uint64_t nnz, int device, void* stream, as_graph* out);
as_status as_graph_destroy(as_graph g);
as_status as_graph_shape(as_graph g, uint64_t* n_rows, uint64_t* n_cols, uint64_t* nnz,
                         int* has_values);
/* Device views of the stored arrays (owned by the graph). */
as_status as_graph_device_arrays(as_graph g, const uint64_t** rowptr, const uint32_t** colind,
                                 const float** val);
/* Replace the value array (host or device source, nnz floats); NULL drops
 * values (pattern-only). */
as_status as_graph_set_values(as_graph g, const float* vals, int vals_on_device);

/* validate, src/csr.cpp:62-93, on host arrays.  Returns AS_OK and
 * *violated = 0 when canonical; else *violated = 1, invariant name in buf. */
as_status as_validate(const uint64_t* rowptr, const uint32_t* colind, const float* val,
                      uint64_t rowptr_len, uint64_t n_rows, uint64_t n_cols, uint64_t nnz,
                      uint64_t val_len, int* violated, char* invariant_buf, size_t cap,
                      uint64_t* index);

/* graph_sig, src/cache.cpp:66-74 (FNV-1a 64); memoized per graph. */
as_status as_graph_sig(as_graph g, uint64_t* out);
/* graph_sig on host arrays (no graph needed). */
uint64_t as_graph_sig_host(const uint64_t* rowptr, const uint32_t* colind, uint64_t n_rows,
                           uint64_t n_cols, uint64_t nnz);

/* GraphFeatures, include/autosage/csr.hpp:93-107; computed on device. */
typedef struct {
    uint64_t n_rows, n_cols, nnz;
    uint64_t deg_p25, deg_p50, deg_p75, deg_p90, deg_p99, deg_max;
    double mean_degree, heavy_row_fraction, empty_row_fraction;
    uint64_t hub_threshold;
} as_features;
/* extract_features, src/csr.cpp:108-135. */
as_status as_graph_features(as_graph g, uint64_t hub_threshold, as_features* out);

/* sample_row_indices, src/generate.cpp:134-153 (device stable radix sort).
 * rows_out (host) must hold n_rows entries; *count receives the size. */
as_status as_sample_row_indices(as_graph g, double frac, uint64_t min_rows, uint64_t* rows_out,
                                uint64_t* count);
/* slice_rows, src/generate.cpp:155-176 -> new device graph. */
as_status as_slice_rows(as_graph g, const uint64_t* rows_host, uint64_t n_sel, as_graph* out);
/* Download a graph's arrays into host buffers (sizes from as_graph_shape). */
as_status as_graph_download(as_graph g, uint64_t* rowptr, uint32_t* colind, float* val);

/* ------------------------------------------------------------------ */
/* Operators -- include/autosage/kernels.hpp:44-85                      */
/* ------------------------------------------------------------------ */
/* spmm_baseline (src/kernels.cpp:210-228) / spmm_rowparallel (:230-258) /
 * spmm_hubsplit (:260-334) via dispatch (:485-510): C = A * B.
 * b_dev: n_cols x f, c_dev: n_rows x f.  v == NULL -> baseline kernel. */
as_status as_spmm(const as_variant* v, as_graph a, const float* b_dev, uint64_t b_rows,
                  uint64_t f, float* c_dev, void* stream, as_kernel_result* res);
/* The strict per-mapping entry points: mapping mismatch -> invalid argument
 * ("spmm_rowparallel: variant mapping mismatch"). */
as_status as_spmm_rowparallel(const as_variant* v, as_graph a, const float* b_dev,
                              uint64_t b_rows, uint64_t f, float* c_dev, void* stream);
as_status as_spmm_hubsplit(const as_variant* v, as_graph a, const float* b_dev, uint64_t b_rows,
                           uint64_t f, float* c_dev, void* stream);

/* sddmm_baseline (src/kernels.cpp:336-355) / sddmm_rowparallel (:357-429) via
 * dispatch (:512-531): out[e] = <X[i,:], Y[colind[e],:]>.  v == NULL ->
 * baseline.  out_dev holds nnz floats aligned with the pattern. */
as_status as_sddmm(const as_variant* v, as_graph pattern, const float* x_dev, uint64_t x_rows,
                   const float* y_dev, uint64_t y_rows, uint64_t f, float* out_dev, void* stream,
                   as_kernel_result* res);

/* sddmm_rowparallel, src/kernels.cpp:357-429: the strict entry point (no env
 * overrides; a Baseline mapping is "sddmm_rowparallel: variant mapping
 * mismatch"). */
as_status as_sddmm_rowparallel(const as_variant* v, as_graph pattern, const float* x_dev,
                               uint64_t x_rows, const float* y_dev, uint64_t y_rows, uint64_t f,
                               float* out_dev, void* stream);

/* row_softmax, src/kernels.cpp:431-461, over explicit values (vals_dev ==
 * NULL uses the graph's own values; a pattern-only graph with nnz > 0 is
 * "row_softmax: values required"). */
as_status as_row_softmax(as_graph m, const float* vals_dev, float* out_dev, void* stream);

/* Host-buffer forms (the reference's own by-value calling convention:
 * host operands in, host result out; H2D/D2H inside the call). */
as_status as_spmm_host(const as_variant* v, as_graph a, const float* b_host, uint64_t b_rows,
                       uint64_t f, float* c_host, as_kernel_result* res);
as_status as_sddmm_host(const as_variant* v, as_graph pattern, const float* x_host,
                        uint64_t x_rows, const float* y_host, uint64_t y_rows, uint64_t f,
                        float* out_host, as_kernel_result* res);
as_status as_row_softmax_host(as_graph m, const float* vals_host, float* out_host);
/* Asynchronous host-buffer forms: queue H2D, kernels and D2H on the graph's
 * pipeline streams and return; results are in the host buffers after
 * as_graph_synchronize().  Host buffers should be pinned (as_host_alloc) and
 * must stay valid until then.  An SpMM and an SDDMM on the same graph may be
 * in flight together (separate staging); calls of one op are ordered. */
as_status as_spmm_host_async(const as_variant* v, as_graph a, const float* b_host, uint64_t b_rows,
                             uint64_t f, float* c_host, as_kernel_result* res);
as_status as_sddmm_host_async(const as_variant* v, as_graph pattern, const float* x_host,
                              uint64_t x_rows, const float* y_host, uint64_t y_rows, uint64_t f,
                              float* out_host, as_kernel_result* res);
as_status as_graph_synchronize(as_graph g);

/* ------------------------------------------------------------------ */
/* Device profile -- include/autosage/device.hpp:12-27                  */
/* ------------------------------------------------------------------ */
typedef struct {
    char device_sig[256];
    double bw_eff;    /* bytes/s */
    double flops_eff; /* FLOP/s  */
    uint64_t cores;   /* GPU: SM count */
    int32_t model;    /* AS_MODEL_REFERENCE: proj/src/cost.cpp as is;
                         AS_MODEL_B200: the GPU refinement (as_estimate_cost) */
} as_device_profile;
enum { AS_MODEL_REFERENCE = 0, AS_MODEL_B200 = 1 };
/* DeviceProfile::host() re-targeted: calibrated once per device per process
 * (triad + FMA kernels, src/device.cpp:42-95 analogue). */
as_status as_device_profile_gpu(int device, as_device_profile* out);
/* DeviceProfile::fixed, src/device.cpp:103-111. */
void as_device_profile_fixed(double bw_eff, double flops_eff, uint64_t cores,
                             const char* sig_tag, as_device_profile* out);

/* estimate_cost / shortlist, include/autosage/cost.hpp:17-26. */
as_status as_estimate_cost(const as_variant* v, const as_features* gf, uint64_t f,
                           const as_device_profile* dp, double* out_ms);
/* out must hold 36 entries; *count = 36 (F%4==0) or 18. */
as_status as_shortlist(const as_features* gf, uint64_t f, int op, const as_device_profile* dp,
                       as_variant* out, int* count);

/* ------------------------------------------------------------------ */
/* Timing -- include/autosage/timing.hpp:10-36                          */
/* ------------------------------------------------------------------ */
/* ProbeTimer::time_once_ms as a callback: must call run(run_arg) (or not,
 * as a scripted timer may) and return milliseconds; a negative return is a
 * logic error ("script exhausted"). */
typedef double (*as_time_once_fn)(void* user, const char* label, void (*run)(void*),
                                  void* run_arg);
typedef struct {
    double median_ms;
    int32_t completed;
    int32_t capped;
    double max_run_ms;
    double wall_ms;
    int32_t launches;
} as_timed_stats;
/* time_kernel, src/timing.cpp:22-61.  timer == NULL: CUDA events on the
 * current device's legacy stream around a synchronous run. */
as_status as_time_kernel(const char* label, void (*run)(void*), void* run_arg, int iters,
                         double cap_ms, as_time_once_fn timer, void* timer_user,
                         as_timed_stats* out);

/* ------------------------------------------------------------------ */
/* Schedule cache -- include/autosage/cache.hpp:23-91                   */
/* ------------------------------------------------------------------ */
typedef struct as_cache_s* as_cache;
typedef struct {
    char device_sig[256];
    uint64_t graph_sig;
    uint64_t f;
    int32_t op;
} as_key;
typedef struct {
    as_key key;
    char choice[128]; /* "baseline" or a variant string */
    double t_b, t_star, alpha;
    uint64_t timestamp;
    uint32_t schema_version;
    char toolchain[64];
} as_record;

as_status as_cache_create(as_cache* out);
as_status as_cache_destroy(as_cache c);
/* *found = 0 on miss. */
as_status as_cache_get(as_cache c, const as_key* key, as_record* out, int* found);
as_status as_cache_put(as_cache c, const as_record* rec);
as_status as_cache_size(as_cache c, uint64_t* n);
/* Records in canonical key order; out may be NULL to query the count. */
as_status as_cache_snapshot(as_cache c, as_record* out, uint64_t cap, uint64_t* n);
as_status as_cache_clear(as_cache c);
as_status as_cache_load(as_cache c, const char* path);
as_status as_cache_store(as_cache c, const char* path);
/* record_to_line / record_from_line, src/cache.cpp:97-158. */
as_status as_record_to_line(const as_record* rec, char* buf, size_t cap);
as_status as_record_from_line(const char* line, as_record* out);
as_status as_key_to_string(const as_key* key, char* buf, size_t cap);
const char* as_toolchain_tag(void);

/* ------------------------------------------------------------------ */
/* Scheduler -- include/autosage/scheduler.hpp:16-92                    */
/* ------------------------------------------------------------------ */
typedef struct {
    double frac;       /* 0.02 */
    uint64_t min_rows; /* 512  */
    int32_t iters;     /* 5    */
    double cap_ms;     /* 1.0  */
    int32_t top_k;     /* 3    */
    double alpha;      /* 0.95 */
} as_probe_config;
void as_probe_config_default(as_probe_config* out);
/* ProbeConfig::from_env, src/scheduler.cpp:171-179. */
void as_probe_config_from_env(as_probe_config* out);

typedef struct {
    int32_t replay_only;
    int32_t strict;
} as_replay_policy;
/* ReplayPolicy::from_env, src/cache.cpp:223-228. */
void as_replay_policy_from_env(as_replay_policy* out);

enum { AS_SRC_PROBED = 0, AS_SRC_CACHED = 1, AS_SRC_REPLAYED = 2, AS_SRC_FORCED_ENV = 3 };

#define AS_MAX_CANDIDATES 36
typedef struct {
    as_variant variant;
    double median_ms;
    int32_t completed;
    int32_t capped;
} as_candidate_timing;

typedef struct {
    int32_t has_choice; /* 0: baseline */
    as_variant choice;
    int32_t source; /* AS_SRC_* */
    as_key key;
    double alpha;
    /* ProbeReport, include/autosage/scheduler.hpp:36-46 */
    double baseline_ms;
    int32_t baseline_completed;
    int32_t baseline_capped;
    int32_t n_candidates;
    as_candidate_timing candidates[AS_MAX_CANDIDATES];
    int32_t best_index;
    double t_star;
    uint64_t sample_rows;
    double probe_wall_ms;
    double max_single_run_ms;
    /* cold-decide phases (new; host wall clock, ms): graph signature
     * (memoised per graph: 0 after the first decide), features, the probe
     * sample (rows + slice), and the whole decide call */
    double sig_ms;
    double features_ms;
    double sample_ms;
    double decide_wall_ms;
} as_decision;

/* ScheduleContext, include/autosage/scheduler.hpp:61-69.  Every pointer
 * member may be NULL (process defaults: calibrated GPU profile, no cache,
 * CUDA-event timer). */
typedef struct {
    const as_device_profile* device;
    as_cache cache;
    as_time_once_fn timer;
    void* timer_user;
    as_replay_policy replay;
    void* stream;
} as_context;

/* decide_spmm / decide_sddmm, src/scheduler.cpp:195-224. */
as_status as_decide_spmm(const as_context* ctx, const as_probe_config* cfg, as_graph a,
                         const float* b_dev, uint64_t b_rows, uint64_t f, as_decision* out);
as_status as_decide_sddmm(const as_context* ctx, const as_probe_config* cfg, as_graph pattern,
                          const float* x_dev, uint64_t x_rows, const float* y_dev,
                          uint64_t y_rows, uint64_t f, as_decision* out);
/* spmm_auto / sddmm_auto, src/scheduler.cpp:226-239 (decision optional). */
as_status as_spmm_auto(const as_context* ctx, const as_probe_config* cfg, as_graph a,
                       const float* b_dev, uint64_t b_rows, uint64_t f, float* c_dev,
                       as_decision* decision);
/* spmm_auto over explicit values vals_dev (nnz floats, device) instead of
 * the graph's own: the same decision key (graph_sig excludes values,
 * src/cache.cpp:66-74), so one cached pattern graph serves any edge
 * weights (new; the torch ops pass weights per call). */
as_status as_spmm_auto_values(const as_context* ctx, const as_probe_config* cfg, as_graph a,
                              const float* vals_dev, const float* b_dev, uint64_t b_rows, uint64_t f,
                              float* c_dev, as_decision* decision);
as_status as_sddmm_auto(const as_context* ctx, const as_probe_config* cfg, as_graph pattern,
                        const float* x_dev, uint64_t x_rows, const float* y_dev,
                        uint64_t y_rows, uint64_t f, float* out_dev, as_decision* decision);
/* probe_launch_count / reset_probe_launch_count, src/scheduler.cpp:241-247. */
uint64_t as_probe_launch_count(void);
void as_reset_probe_launch_count(void);

/* Pure decision procedure (decide_common, src/scheduler.cpp:86-167) over
 * precomputed inputs, for host-only use: no kernels are launched; timer is
 * required and its run callback is a no-op.  Used to test the guardrail on
 * machines without a GPU. */
as_status as_decide_host(const as_context* ctx, const as_probe_config* cfg, uint64_t graph_sig,
                         const as_features* gf, uint64_t f, int op, uint64_t sample_rows,
                         as_decision* out);

/* ------------------------------------------------------------------ */
/* Attention -- include/autosage/attention.hpp:13-25                    */
/* ------------------------------------------------------------------ */
/* attention_probe_breakdown, src/attention.cpp:9-40: sddmm_auto ->
 * row_softmax -> spmm_auto, each decided under its own key.  q: n_rows x f,
 * k: n_cols x f, v: n_cols x fv, out: n_rows x fv (device).  Decisions are
 * optional outputs.  fused != 0: SDDMM -> per-row (max, sum) -> SpMM that
 * turns each score into its probability as it loads it (no probability
 * array, the same bits as fused == 0); it needs a mapped SpMM decision and
 * fv % 4 == 0 with 16-byte aligned v, else the staged pipeline runs. */
as_status as_csr_attention_forward(const as_context* ctx, const as_probe_config* cfg,
                                   as_graph pattern, const float* q_dev, uint64_t q_rows,
                                   const float* k_dev, uint64_t k_rows, const float* v_dev,
                                   uint64_t v_rows, uint64_t f, uint64_t fv, float* out_dev,
                                   int fused, as_decision* sddmm_decision,
                                   as_decision* spmm_decision);

/* Batched heads (the optional batched-heads variant of
 * csr_attention_forward): n_heads independent heads on one pattern, head h
 * reading q_devs[h], k_devs[h], v_devs[h] and writing out_devs[h] (same
 * shapes as above for every head), in head order on one stream.  Every head
 * decides under the same keys as the single-head call (src/attention.cpp:
 * 21-38: head 1 probes, the rest hit the cache); without a cache in ctx a
 * cache local to the call plays that role.  Decisions: those of the last
 * head.  Each head's out equals the single-head call's bit for bit. */
as_status as_csr_attention_forward_heads(const as_context* ctx, const as_probe_config* cfg,
                                         as_graph pattern, uint32_t n_heads, const float* const* q_devs,
                                         uint64_t q_rows, const float* const* k_devs, uint64_t k_rows,
                                         const float* const* v_devs, uint64_t v_rows, uint64_t f,
                                         uint64_t fv, float* const* out_devs, int fused,
                                         as_decision* sddmm_decision, as_decision* spmm_decision);

/* The staged pipeline with the probabilities p = row_softmax(SDDMM(q, k))
 * also written to p_dev (nnz floats, device): the training forward keeps p
 * for the backward instead of recomputing it (new).  out is
 * bit-identical to as_csr_attention_forward. */
as_status as_csr_attention_forward_p(const as_context* ctx, const as_probe_config* cfg,
                                     as_graph pattern, const float* q_dev, uint64_t q_rows,
                                     const float* k_dev, uint64_t k_rows, const float* v_dev,
                                     uint64_t v_rows, uint64_t f, uint64_t fv, float* out_dev,
                                     float* p_dev, as_decision* sddmm_decision,
                                     as_decision* spmm_decision);

/* ------------------------------------------------------------------ */
/* Multi-GPU row partition (new)                           */
/* ------------------------------------------------------------------ */
/* cut_k = lower_bound(rowptr, floor(k*nnz/g)); cuts has g+1 entries. */
as_status as_partition_rows(const uint64_t* rowptr_host, uint64_t n_rows, uint32_t g,
                            uint64_t* cuts);
/* Row range [r0, r1) of g as a new graph with rebased rowptr and global
 * column indices. */
as_status as_graph_row_range(as_graph g, uint64_t r0, uint64_t r1, as_graph* out);

/* Column-blocked SpMM (new): C = A * B consumed one column
 * block of B at a time, so a rank can start on each B row shard as the
 * all-gather lands it.  col_cuts[0..n_blocks] split [0, n_cols); run blocks
 * 0, 1, ..., n_blocks-1 in order on one stream (block 0 resets the f64 row
 * state, the last writes C).  Every row / HubSplit piece keeps an f64
 * accumulator across blocks, so C is bit-identical to as_spmm with the same
 * variant (v == NULL: baseline; RowParallel = row chains; HubSplit = the
 * 2048-nnz pieces of rows >= hub_threshold, src/kernels.cpp:260-334).  A
 * plan references its graph (which must outlive it) and is single-stream. */
typedef struct as_blocked_s* as_blocked;
as_status as_spmm_blocked_create(as_graph a, const as_variant* v, const uint64_t* col_cuts, uint32_t n_blocks,
                                 as_blocked* out);
/* vals_dev == NULL: the graph's own values (implicit 1.0 when pattern-only). */
as_status as_spmm_blocked_run(as_blocked p, uint32_t block, const float* vals_dev, const float* b_dev,
                              uint64_t b_rows, uint64_t f, float* c_dev, void* stream);
as_status as_spmm_blocked_destroy(as_blocked p);

/* ------------------------------------------------------------------ */
/* Backward pass (new, PAPER.md:334 -- the reference has  */
/* no gradients).  C = A B gives dB = A^T dC (as_spmm_values on the      */
/* transpose, values permuted) and dval = SDDMM(A, dC, B); out =          */
/* SDDMM(A, X, Y) gives dX = A[dout] Y and dY = A^T[dout] X.              */
/* ------------------------------------------------------------------ */
/* CSR transpose on device (n_cols x n_rows; entries of each new row in
 * source row order, so canonical, csr.hpp:24-45).  Values are permuted when
 * g has them; the entry permutation is kept on the new handle. */
as_status as_graph_transpose(as_graph g, as_graph* out);
/* Device view of a transpose's permutation: perm[k] = source entry of entry
 * k (nnz u32).  Not a transpose -> AS_INVALID_ARGUMENT. */
as_status as_graph_transpose_perm(as_graph gt, const uint32_t** perm);
/* dst_dev[k] = src_dev[perm[k]] for a transpose's nnz entries (a source
 * value array carried into the transposed order). */
as_status as_permute_values(as_graph gt, const float* src_dev, float* dst_dev, void* stream);
/* as_spmm with an explicit value array (nnz floats, device) in place of the
 * graph's own: the same kernels and numerics (dispatch, src/kernels.cpp:485-510). */
as_status as_spmm_values(const as_variant* v, as_graph a, const float* vals_dev, const float* b_dev,
                         uint64_t b_rows, uint64_t f, float* c_dev, void* stream,
                         as_kernel_result* res);
/* SpMM with a bf16 dense operand (new):
 * b_dev holds b_rows x f bf16 values (raw 16-bit words), vals_dev f32 or
 * NULL (graph's own values), f64 accumulation, f32 C.  bf16 -> f32 is exact,
 * so C equals as_spmm on the f32 copy of B bit for bit, with half the gather
 * bytes.  v == NULL -> baseline kernel; env overrides as in dispatch. */
as_status as_spmm_bf16(const as_variant* v, as_graph a, const float* vals_dev, const uint16_t* b_dev,
                       uint64_t b_rows, uint64_t f, float* c_dev, void* stream, as_kernel_result* res);
/* SDDMM on bf16 X (x_rows x f) and Y (y_rows x f) words, f64 accumulation,
 * f32 out: as_sddmm on the f32 copies of X and Y with the same variant, bit
 * for bit (the vec order applies whenever f % 4 == 0).  v == NULL -> baseline. */
as_status as_sddmm_bf16(const as_variant* v, as_graph pattern, const uint16_t* x_dev, uint64_t x_rows,
                        const uint16_t* y_dev, uint64_t y_rows, uint64_t f, float* out_dev, void* stream,
                        as_kernel_result* res);
/* CSR attention on 16-bit q, k, v words (wt 1 = bf16, 2 = f16; new, SURVEY
 * 8(f) N4) with given variants (NULL = baseline): scores = SDDMM(q, k), p =
 * row_softmax(scores), out = SpMM(p, v) (f32 out, n_rows x fv).  fused != 0
 * and p_out == NULL: SDDMM -> per-row (max, sum) -> an SpMM that turns each
 * score into its probability as it loads it (needs a mapped SpMM variant and
 * fv % 4 == 0 with an 8-byte aligned v; else staged).  p_out (nnz floats)
 * receives p (staged).  The bits equal the f32 staged pipeline on the widened
 * operands with the same variants. */
as_status as_csr_attention_half(as_graph pattern, const as_variant* sddmm_v, const as_variant* spmm_v,
                                const uint16_t* q_dev, uint64_t q_rows, const uint16_t* k_dev, uint64_t k_rows,
                                const uint16_t* v_dev, uint64_t v_rows, uint64_t f, uint64_t fv, float* out_dev,
                                float* p_dev, int wt, int fused, void* stream);
/* The same two operators on IEEE binary16 words (new): f16
 * -> f32 is exact too, so the results equal as_spmm / as_sddmm on the f32
 * copies bit for bit (Inf/NaN included; a device scan gates the re-bias
 * widening as for f32). */
as_status as_spmm_f16(const as_variant* v, as_graph a, const float* vals_dev, const uint16_t* b_dev,
                      uint64_t b_rows, uint64_t f, float* c_dev, void* stream, as_kernel_result* res);
as_status as_sddmm_f16(const as_variant* v, as_graph pattern, const uint16_t* x_dev, uint64_t x_rows,
                       const uint16_t* y_dev, uint64_t y_rows, uint64_t f, float* out_dev, void* stream,
                       as_kernel_result* res);
/* A^T[vals] * B on a transpose gt, with vals in the SOURCE graph's entry
 * order (nnz floats, device): the kernels read val[perm[k]] at the value
 * load, so no permuted copy is written (as_permute_values + as_spmm_values
 * in one pass, the same bits).  gt not a transpose -> AS_INVALID_ARGUMENT. */
as_status as_spmm_transpose_values(const as_variant* v, as_graph gt, const float* vals_src_dev,
                                   const float* b_dev, uint64_t b_rows, uint64_t f, float* c_dev, void* stream,
                                   as_kernel_result* res);
/* Gradient of row_softmax (src/kernels.cpp:431-461): ds = p * (g - dot),
 * dot = sum_row p*g in f64 (32 strided partials, fixed pairwise fold;
 * oracle/oracle.c orc_row_softmax_backward). */
as_status as_row_softmax_backward(as_graph m, const float* p_dev, const float* grad_dev,
                                  float* ds_dev, void* stream);

/* ------------------------------------------------------------------ */
/* Synthetic inputs + ASCR I/O (include/autosage/generate.hpp, io.hpp)  */
/* ------------------------------------------------------------------ */
/* Heavy-tailed degree CSR: degrees d_i = clamp(floor(d_min * u^(-1/(a-1))),
 * 0, d_max) rescaled to hit nnz_target exactly (when > 0); columns distinct
 * uniform in [0, n_cols), sorted; values U[0,1).  Deterministic in seed and
 * independent of the thread count.  Arrays are malloc'ed: free with as_free. */
as_status as_gen_powerlaw(uint64_t n_rows, uint64_t n_cols, uint64_t nnz_target, double alpha,
                          uint64_t d_min, uint64_t d_max, uint64_t seed, int with_values,
                          uint64_t** rowptr, uint32_t** colind, float** val, uint64_t* nnz);
/* Dense U(-1,1) f32 matrix from a seed (splitmix64 per element). */
as_status as_fill_uniform(float* host, uint64_t n, uint64_t seed);
void as_free(void* p);
/* save_csr / load_csr, src/io.cpp:48-93 (ASCR v1). */
as_status as_save_csr(const char* path, const uint64_t* rowptr, const uint32_t* colind,
                      const float* val, uint64_t n_rows, uint64_t n_cols, uint64_t nnz);
as_status as_load_csr(const char* path, uint64_t** rowptr, uint32_t** colind, float** val,
                      uint64_t* n_rows, uint64_t* n_cols, uint64_t* nnz);

/* Pinned host memory helpers for host-buffer entry points. */
as_status as_host_alloc(void** p, uint64_t bytes);
as_status as_host_free(void* p);

/* Count of this library's kernel launches since process start (for the
 * bench's gpu_launches claim). */
uint64_t as_kernel_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* AUTOSAGE_B200_H */
