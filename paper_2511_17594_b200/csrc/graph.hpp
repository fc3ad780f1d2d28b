// graph.hpp -- device-resident CSR graph handle (the B200 home of the
// reference's CsrMatrix, include/autosage/csr.hpp:24-45) and the derived
// per-graph schedule data memoized on it.
//
// HBM layout per graph (one allocation each, 256-B aligned by cudaMalloc):
//   rowptr  u64[n_rows+1]   colind u32[nnz]   val f32[nnz] (optional)
//   order   u32[n_rows]     rows sorted by degree descending, stable
//                           (the probe sampling order, src/generate.cpp:143-147;
//                           also the LPT launch order of the row kernels)
//   chunk_row u32[ceil(nnz/32)]  row holding nnz 32*k (SDDMM nnz-chunk map)
//   hub plans (per threshold): light-row list, 2048-nnz pieces, reduce list
#pragma once

#include "internal.hpp"

#include <future>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

namespace asb {

template <class T>
class DevBuf {
public:
    DevBuf() = default;
    explicit DevBuf(std::uint64_t n) { alloc(n); }
    ~DevBuf() { release(); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); p_ = o.p_; n_ = o.n_; o.p_ = nullptr; o.n_ = 0; }
        return *this;
    }
    void alloc(std::uint64_t n) {
        release();
        if (n == 0) return;
        ASB_CUDA(cudaMalloc(&p_, n * sizeof(T)));
        n_ = n;
    }
    void ensure(std::uint64_t n) { if (n > n_) alloc(n); }
    void release() {
        if (p_) cudaFree(p_);
        p_ = nullptr;
        n_ = 0;
    }
    T* get() const { return p_; }
    std::uint64_t size() const { return n_; }

private:
    T* p_ = nullptr;
    std::uint64_t n_ = 0;
};

// Heavy/light split for HubSplit at one threshold (src/kernels.cpp:271-286).
struct HubPlan {
    std::uint64_t threshold = 0;
    std::uint64_t n_light = 0;
    DevBuf<std::uint32_t> light_rows;  // light rows, degree-descending
    std::uint64_t n_pieces = 0;
    DevBuf<std::uint32_t> piece_row;
    DevBuf<std::uint64_t> piece_e0;
    DevBuf<std::uint32_t> piece_len;
    DevBuf<std::uint32_t> piece_slot;  // partial slot, or UINT32_MAX: write C directly
    std::uint64_t n_slots = 0;         // partial rows needed (pieces of multi-piece rows)
    std::uint64_t n_red = 0;           // multi-piece heavy rows
    DevBuf<std::uint32_t> red_row;
    DevBuf<std::uint32_t> red_first;   // first slot
    DevBuf<std::uint32_t> red_count;   // pieces
    std::uint64_t n_heavy = 0;
    // one item list for a single launch: the pieces (longest first) followed
    // by the light rows as direct-write items (degree-descending)
    DevBuf<std::uint32_t> all_row, all_len, all_slot;
    DevBuf<std::uint64_t> all_e0;
};

struct Graph {
    int device = 0;
    int sms = 148;  // multiprocessors of `device` (queried once at creation)
    std::uint64_t n_rows = 0, n_cols = 0, nnz = 0;
    bool has_val = false;
    // kernel-path heuristics see this many entries (a probe sample stands in
    // for its parent graph, so it takes the parent's paths); 0 = own nnz
    std::uint64_t plan_nnz = 0;
    DevBuf<std::uint64_t> rowptr;
    DevBuf<std::uint32_t> colind;
    DevBuf<float> val;
    std::vector<std::uint64_t> h_rowptr;  // host mirror (8 B/row)
    cudaStream_t stream = nullptr;

    std::mutex mu;
    std::optional<std::uint64_t> sig;
    // graph_sig computed in the background from creation on (FNV-1a is a
    // serial ~1 GB/s pass over rowptr + colind); graph_sig() waits for it
    std::future<std::uint64_t> sig_future;
    bool order_ready = false;
    DevBuf<std::uint32_t> order;       // degree-descending stable row order
    DevBuf<std::uint32_t> sorted_deg;  // degrees in that order
    bool chunk_ready = false;
    DevBuf<std::uint32_t> chunk_row;
    std::map<std::uint64_t, std::unique_ptr<HubPlan>> hub_plans;
    std::map<std::uint64_t, as_features> features;
    DevBuf<double> scratch;            // hub partials
    DevBuf<double> sddmm_state;        // pass-major SDDMM: per-entry f64 chains
    DevBuf<float> att_buf;             // attention: scores | probabilities (staged)
    DevBuf<float> att_max;             // fused attention: per-row score max ...
    DevBuf<double> att_sum;            // ... and softmax denominator
    DevBuf<std::uint32_t> sm_chain_row; // row softmax: long rows whose sum needs
    DevBuf<float> sm_chain_mx;          // the entry-order chain (row, max) ...
    DevBuf<unsigned> sm_chain_n;        // ... and their count
    DevBuf<float> stage_in, stage_out; // host-buffer row softmax
    std::map<std::uint64_t, std::uint64_t> ge_count;  // rows with degree >= key
    DevBuf<unsigned> flag;             // finiteness flag of the current dense operand
    bool flag_frozen = false;          // probe sample: flag computed once per decide
    DevBuf<double> xwide;              // SDDMM: X widened to f64 (fixed-width path)
    bool is_transpose = false;         // built by transpose_graph (backward.cu) ...
    DevBuf<std::uint32_t> src_perm;    // ... entry k came from source entry src_perm[k]
    // set for the duration of one SpMM call (ValPermScope, engine.cpp): the
    // value array is in source order and entry k reads val[val_perm[k]]
    const std::uint32_t* val_perm = nullptr;
    cudaStream_t aux = nullptr;        // fork/join stream for concurrent kernels
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;

    // operator serialisation (GraphUse): the scratch above is per graph, so
    // operators on one handle run one at a time -- host side under op_mu,
    // device side ordered across streams by ev_last_op
    std::recursive_mutex op_mu;
    int op_depth = 0;
    cudaStream_t last_op_stream = nullptr;
    cudaEvent_t ev_last_op = nullptr;

    // host-buffer pipeline (as_*_host, as_*_host_async): copies in on h2d,
    // kernels on `stream`, copies out on d2h; per-op staging so an SpMM and
    // an SDDMM can be in flight together.
    struct HostPipe {
        cudaStream_t h2d = nullptr, d2h = nullptr;
        DevBuf<float> b, c, x, y, v;
        // per op: inputs landed / kernels done (staging readable again) /
        // outputs copied (staging writable again)
        cudaEvent_t spmm_in = nullptr, spmm_done = nullptr, spmm_out = nullptr;
        cudaEvent_t sddmm_in = nullptr, sddmm_done = nullptr, sddmm_out = nullptr;
        std::vector<cudaEvent_t> slice;    // SDDMM output slices computed
        std::vector<cudaEvent_t> slice_x;  // ... and their X rows landed
    } pipe;

    ~Graph();
};

// RAII device guard
struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (dev != prev) ASB_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = 0;
        cudaGetDevice(&cur);
        if (cur != prev) cudaSetDevice(prev);
    }
};

// One operator call on a graph handle.  The handle's scratch (X widening,
// hub partials, finite flag, attention buffers, the transpose's value
// permutation) is shared by every operator on it, so calls serialise: a
// recursive host mutex (entry points nest: attention -> SDDMM -> SpMM), and
// on the device the outermost call on stream s waits for the previous call's
// work when that was enqueued on another stream (one event per graph).  A
// graph can therefore be used from several threads and streams; its
// operators never overlap one another.
class GraphUse {
public:
    GraphUse(Graph& g, cudaStream_t s);
    ~GraphUse();
    GraphUse(const GraphUse&) = delete;
    GraphUse& operator=(const GraphUse&) = delete;

private:
    Graph& g_;
    cudaStream_t s_;
    std::unique_lock<std::recursive_mutex> lk_;
};

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) and the occupancy query
// of a kernel, once per (kernel, device, smem, threads) -- off the per-launch
// path.  Returns resident CTAs per SM.
int kernel_setup(const void* kernel, std::size_t smem, int threads);
template <class K>
int kernel_setup(K* kernel, std::size_t smem, int threads) {
    return kernel_setup(reinterpret_cast<const void*>(kernel), smem, threads);
}
// multiprocessors of the current device (cached per device)
int device_sms();

std::unique_ptr<Graph> graph_create_host(const std::uint64_t* rowptr, const std::uint32_t* colind,
                                         const float* val, std::uint64_t n_rows,
                                         std::uint64_t n_cols, std::uint64_t nnz, int device,
                                         bool validate);
// Device arrays in: the copies run after the work already enqueued on
// `caller` (the stream that produced them; nullptr = legacy default stream),
// and the structure is validated on the device (columns in range and
// strictly increasing per row, src/csr.cpp:62-93).
std::unique_ptr<Graph> graph_create_device(const std::uint64_t* rowptr, const std::uint32_t* colind,
                                           const float* val, std::uint64_t n_rows,
                                           std::uint64_t n_cols, std::uint64_t nnz, int device,
                                           cudaStream_t caller);
cudaStream_t resolve_stream(Graph& g, void* stream);

std::uint64_t graph_sig(Graph& g);
void start_sig(Graph& g);  // background graph_sig at creation (graph.cu)
// number of rows with degree >= d (host count from the rowptr mirror, cached)
std::uint64_t rows_with_degree_at_least(Graph& g, std::uint64_t d);
// fork: returns the graph's aux stream ordered after `s`; join: `s` waits
// for the aux stream's work
cudaStream_t graph_fork(Graph& g, cudaStream_t s);
void graph_join(Graph& g, cudaStream_t s);
void ensure_order(Graph& g);
void ensure_chunk_rows(Graph& g);
const HubPlan& ensure_hub_plan(Graph& g, std::uint64_t threshold);
as_features graph_features(Graph& g, std::uint64_t hub_threshold);
std::vector<std::uint64_t> sample_row_indices(Graph& g, double frac, std::uint64_t min_rows);
// vals: the value array to slice (nullptr: pattern-only sample).
std::unique_ptr<Graph> slice_rows(Graph& g, const std::vector<std::uint64_t>& rows,
                                  const float* vals);
std::unique_ptr<Graph> row_range(Graph& g, std::uint64_t r0, std::uint64_t r1);
// Gathers rows of a dense n x f device matrix (SDDMM probe x-sample,
// src/scheduler.cpp:214-220).
// CSR transpose (backward.cu): rows = source columns, entries in source row
// order, values permuted, src_perm kept for permuting later value arrays.
std::unique_ptr<Graph> transpose_graph(Graph& g);
void gather_dense_rows(const float* src, std::uint64_t f, const std::vector<std::uint64_t>& rows,
                       float* dst, cudaStream_t s);

} // namespace asb
