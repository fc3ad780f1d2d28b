// engine.hpp -- operator dispatch, the input-aware scheduler and the
// attention pipeline over device graphs (host C++).
#pragma once

#include "cache.hpp"
#include "graph.hpp"
#include "policy.hpp"

namespace asb {

const as_device_profile& gpu_profile(int device);

struct KernelResult {
    as_variant variant{};
    bool vectorized_path = false;
    double elapsed_ms = 0.0;
};

// Value array a graph operator reads: explicit override, else the graph's.
inline const float* graph_values(const Graph& g, const float* override_vals) {
    if (override_vals) return override_vals;
    return g.has_val ? g.val.get() : nullptr;
}

// spmm_baseline (src/kernels.cpp:210-228): no variant, no env overrides.
void spmm_baseline(Graph& a, const float* vals, const float* b, std::uint64_t b_rows,
                   std::uint64_t f, float* c, cudaStream_t s);
// spmm_rowparallel / spmm_hubsplit with the reference's mapping checks.
void spmm_mapped(const as_variant& v, int expect_mapping, Graph& a, const float* vals,
                 const float* b, std::uint64_t b_rows, std::uint64_t f, float* c, cudaStream_t s);
// dispatch (src/kernels.cpp:485-531); `timed` synchronizes and fills
// elapsed_ms from CUDA events.
KernelResult dispatch_spmm(const as_variant& v, Graph& a, const float* vals, const float* b,
                           std::uint64_t b_rows, std::uint64_t f, float* c, cudaStream_t s,
                           bool timed);
// SpMM with 16-bit B words (wt: 1 bf16, 2 f16; v == nullptr: baseline); the
// f32 result on float(B).
KernelResult dispatch_spmm_half(const as_variant* v, Graph& a, const float* vals, const std::uint16_t* b,
                                std::uint64_t b_rows, std::uint64_t f, float* c, cudaStream_t s, bool timed,
                                int wt);
// CSR attention on 16-bit q, k, v words with given variants (staged or
// fused), the f32 staged pipeline's bits on the widened operands.
void attention_half(Graph& pattern, const as_variant* sv, const as_variant* pv, const std::uint16_t* q,
                    std::uint64_t q_rows, const std::uint16_t* k, std::uint64_t k_rows, const std::uint16_t* v,
                    std::uint64_t v_rows, std::uint64_t f, std::uint64_t fv, float* out, float* p_out, bool fused,
                    int wt, cudaStream_t s);
// SDDMM on 16-bit X, Y words (v == nullptr: baseline); the f32 result on
// float(X), float(Y).
KernelResult dispatch_sddmm_half(const as_variant* v, Graph& p, const std::uint16_t* x, std::uint64_t x_rows,
                                 const std::uint16_t* y, std::uint64_t y_rows, std::uint64_t f, float* out,
                                 cudaStream_t s, bool timed, int wt);
void sddmm_baseline(Graph& p, const float* x, std::uint64_t x_rows, const float* y,
                    std::uint64_t y_rows, std::uint64_t f, float* out, cudaStream_t s);
// sddmm_rowparallel (src/kernels.cpp:357-429): variant as given, no env.
void sddmm_mapped(const as_variant& v, Graph& p, const float* x, std::uint64_t x_rows,
                  const float* y, std::uint64_t y_rows, std::uint64_t f, float* out,
                  cudaStream_t s);
KernelResult dispatch_sddmm(const as_variant& v, Graph& p, const float* x, std::uint64_t x_rows,
                            const float* y, std::uint64_t y_rows, std::uint64_t f, float* out,
                            cudaStream_t s, bool timed);
void row_softmax(Graph& m, const float* vin, float* vout, cudaStream_t s);

// Host-buffer operators (the reference's by-value API).  Copies in on the
// graph's h2d stream, kernels on its stream, copies out on its d2h stream;
// SDDMM values leave in slices so the D2H overlaps the remaining kernels.
// v == nullptr: baseline.  sync = false returns once everything is queued
// (host buffers must stay valid -- and should be pinned -- until
// host_synchronize()).
KernelResult spmm_host(const as_variant* v, Graph& a, const float* b_host, std::uint64_t b_rows,
                       std::uint64_t f, float* c_host, bool sync);
KernelResult sddmm_host(const as_variant* v, Graph& p, const float* x_host, std::uint64_t x_rows,
                        const float* y_host, std::uint64_t y_rows, std::uint64_t f,
                        float* out_host, bool sync);
void host_synchronize(Graph& g);

// ScheduleContext (include/autosage/scheduler.hpp:61-69)
struct Context {
    const as_device_profile* device = nullptr;  // nullptr: calibrated GPU profile
    ScheduleCache* cache = nullptr;
    TimeOnce timer;                              // empty: CUDA events
    as_replay_policy replay{};
    cudaStream_t stream = nullptr;               // nullptr: the graph's stream
};

as_decision decide_spmm(const Context& ctx, const as_probe_config& cfg, Graph& a,
                        const float* vals, const float* b, std::uint64_t b_rows, std::uint64_t f);
as_decision decide_sddmm(const Context& ctx, const as_probe_config& cfg, Graph& p,
                         const float* x, std::uint64_t x_rows, const float* y,
                         std::uint64_t y_rows, std::uint64_t f);
as_decision decide_host(const Context& ctx, const as_probe_config& cfg, std::uint64_t sig,
                        const as_features& gf, std::uint64_t f, int op, std::uint64_t sample_rows);
void spmm_auto(const Context& ctx, const as_probe_config& cfg, Graph& a, const float* vals,
               const float* b, std::uint64_t b_rows, std::uint64_t f, float* c, as_decision* d);
void sddmm_auto(const Context& ctx, const as_probe_config& cfg, Graph& p, const float* x,
                std::uint64_t x_rows, const float* y, std::uint64_t y_rows, std::uint64_t f,
                float* out, as_decision* d);

std::uint64_t probe_launch_count();
void reset_probe_launch_count();

// p_out (nnz floats, nullable): also keep the probabilities there (staged
// pipeline; the training path saves them for the backward)
void attention_forward(const Context& ctx, const as_probe_config& cfg, Graph& pattern,
                       const float* q, std::uint64_t q_rows, const float* k, std::uint64_t k_rows,
                       const float* v, std::uint64_t v_rows, std::uint64_t f, std::uint64_t fv,
                       float* out, bool fused, as_decision* sd, as_decision* pd,
                       float* p_out = nullptr);

} // namespace asb
