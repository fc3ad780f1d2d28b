// graph.cu -- device graph handles and the per-graph schedule data:
// stable degree ordering (CUB radix sort), GraphFeatures, probe sampling,
// row slicing, hub plans and the SDDMM nnz-chunk row map.
#include "graph.hpp"
#include "half.cuh"
#include "policy.hpp"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <thread>
#include <tuple>

namespace asb {

namespace {

__global__ void degrees_iota_kernel(const std::uint64_t* __restrict__ rowptr, std::uint64_t n,
                                    std::uint32_t* __restrict__ deg, std::uint32_t* __restrict__ idx) {
    for (std::uint64_t i = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += std::uint64_t(gridDim.x) * blockDim.x) {
        deg[i] = std::uint32_t(rowptr[i + 1] - rowptr[i]);
        idx[i] = std::uint32_t(i);
    }
}

__global__ void count_heavy_empty_kernel(const std::uint32_t* __restrict__ deg, std::uint64_t n,
                                         std::uint64_t thr, unsigned long long* __restrict__ out) {
    unsigned long long heavy = 0, empty = 0;
    for (std::uint64_t i = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += std::uint64_t(gridDim.x) * blockDim.x) {
        heavy += deg[i] >= thr;
        empty += deg[i] == 0;
    }
    for (int o = 16; o > 0; o >>= 1) {
        heavy += __shfl_xor_sync(0xffffffffu, heavy, o);
        empty += __shfl_xor_sync(0xffffffffu, empty, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&out[0], heavy);
        atomicAdd(&out[1], empty);
    }
}

__global__ void gather_u32_strided_kernel(const std::uint32_t* __restrict__ src, std::uint64_t s,
                                          std::uint64_t stride, std::uint64_t* __restrict__ dst) {
    std::uint64_t r = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x;
    if (r < s) dst[r] = src[r * stride];
}

// warp per selected row: segmented copy of colind (and values)
__global__ void slice_copy_kernel(const std::uint64_t* __restrict__ rowptr,
                                  const std::uint32_t* __restrict__ colind,
                                  const float* __restrict__ val,
                                  const std::uint64_t* __restrict__ rows, std::uint64_t s,
                                  const std::uint64_t* __restrict__ out_rowptr,
                                  std::uint32_t* __restrict__ out_col, float* __restrict__ out_val) {
    std::uint64_t w = (blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (w >= s) return;
    const std::uint64_t src0 = rowptr[rows[w]], src1 = rowptr[rows[w] + 1];
    const std::uint64_t dst0 = out_rowptr[w];
    for (std::uint64_t k = lane; k < src1 - src0; k += 32) {
        out_col[dst0 + k] = colind[src0 + k];
        if (val) out_val[dst0 + k] = val[src0 + k];
    }
}

__global__ void rebase_rowptr_kernel(const std::uint64_t* __restrict__ src, std::uint64_t n1,
                                     std::uint64_t base, std::uint64_t* __restrict__ dst) {
    std::uint64_t i = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x;
    if (i < n1) dst[i] = src[i] - base;
}

// chunk_row[k] = row containing nnz 32*k
__global__ void chunk_row_kernel(const std::uint64_t* __restrict__ rowptr, std::uint64_t n,
                                 std::uint32_t* __restrict__ chunk_row) {
    for (std::uint64_t i = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += std::uint64_t(gridDim.x) * blockDim.x) {
        const std::uint64_t e0 = rowptr[i], e1 = rowptr[i + 1];
        if (e0 == e1) continue;
        for (std::uint64_t k = (e0 + 31) / 32; k * 32 < e1; ++k) chunk_row[k] = std::uint32_t(i);
    }
}

__global__ void gather_rows_kernel(const float* __restrict__ src, std::uint64_t f,
                                   const std::uint64_t* __restrict__ rows, std::uint64_t s,
                                   float* __restrict__ dst) {
    std::uint64_t total = s * f;
    for (std::uint64_t i = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; i < total;
         i += std::uint64_t(gridDim.x) * blockDim.x) {
        std::uint64_t r = i / f, c = i - r * f;
        dst[i] = src[rows[r] * f + c];
    }
}

// Structure check of a device-built CSR (src/csr.cpp:62-93: columns in range,
// strictly increasing within each row): bit 0 = a column >= n_cols, bit 1 =
// a row whose columns do not increase.  Warp per row, lanes over entries.
__global__ void validate_cols_kernel(const std::uint64_t* __restrict__ rowptr, std::uint64_t n_rows,
                                     const std::uint32_t* __restrict__ colind, std::uint64_t n_cols,
                                     unsigned* __restrict__ bad) {
    const unsigned lane = threadIdx.x & 31;
    unsigned mine = 0;
    for (std::uint64_t i = (blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x) >> 5; i < n_rows;
         i += (std::uint64_t(gridDim.x) * blockDim.x) >> 5) {
        const std::uint64_t e0 = rowptr[i], e1 = rowptr[i + 1];
        for (std::uint64_t e = e0 + lane; e < e1; e += 32) {
            const std::uint32_t c = colind[e];
            if (c >= n_cols) mine |= 1u;
            if (e > e0 && colind[e - 1] >= c) mine |= 2u;
        }
    }
    mine = __reduce_or_sync(0xffffffffu, mine);
    if (lane == 0 && mine) atomicOr(bad, mine);
}

// grid-stride launches: at most `cap` CTAs (default 16 per SM of the device)
unsigned grid_for(std::uint64_t n, unsigned block, unsigned cap = 0) {
    if (cap == 0) cap = unsigned(device_sms()) * 16u;
    std::uint64_t g = (n + block - 1) / block;
    if (g == 0) g = 1;
    return unsigned(std::min<std::uint64_t>(g, cap));
}

} // namespace

Graph::~Graph() {
    if (sig_future.valid()) sig_future.wait();  // the background hash reads colind
    if (stream) {
        cudaStreamSynchronize(stream);
        cudaStreamDestroy(stream);
    }
    if (aux) {
        cudaStreamSynchronize(aux);
        cudaStreamDestroy(aux);
    }
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (ev_last_op) cudaEventDestroy(ev_last_op);
    for (cudaStream_t q : {pipe.h2d, pipe.d2h}) {
        if (q) {
            cudaStreamSynchronize(q);
            cudaStreamDestroy(q);
        }
    }
    for (cudaEvent_t e : {pipe.spmm_in, pipe.spmm_done, pipe.spmm_out, pipe.sddmm_in, pipe.sddmm_done,
                          pipe.sddmm_out})
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : pipe.slice) cudaEventDestroy(e);
    for (cudaEvent_t e : pipe.slice_x) cudaEventDestroy(e);
}

std::uint64_t rows_with_degree_at_least(Graph& g, std::uint64_t d) {
    std::lock_guard<std::mutex> lk(g.mu);
    auto it = g.ge_count.find(d);
    if (it != g.ge_count.end()) return it->second;
    std::uint64_t n = 0;
    for (std::uint64_t i = 0; i < g.n_rows; ++i) n += (g.h_rowptr[i + 1] - g.h_rowptr[i]) >= d;
    g.ge_count[d] = n;
    return n;
}

cudaStream_t graph_fork(Graph& g, cudaStream_t s) {
    if (!g.aux) {
        ASB_CUDA(cudaStreamCreateWithFlags(&g.aux, cudaStreamNonBlocking));
        ASB_CUDA(cudaEventCreateWithFlags(&g.ev_fork, cudaEventDisableTiming));
        ASB_CUDA(cudaEventCreateWithFlags(&g.ev_join, cudaEventDisableTiming));
    }
    ASB_CUDA(cudaEventRecord(g.ev_fork, s));
    ASB_CUDA(cudaStreamWaitEvent(g.aux, g.ev_fork, 0));
    return g.aux;
}

void graph_join(Graph& g, cudaStream_t s) {
    ASB_CUDA(cudaEventRecord(g.ev_join, g.aux));
    ASB_CUDA(cudaStreamWaitEvent(s, g.ev_join, 0));
}

cudaStream_t resolve_stream(Graph& g, void* stream) {
    return stream ? static_cast<cudaStream_t>(stream) : g.stream;
}

static std::unique_ptr<Graph> alloc_graph(std::uint64_t n_rows, std::uint64_t n_cols,
                                          std::uint64_t nnz, bool has_val, int device) {
    if (device < 0) ASB_CUDA(cudaGetDevice(&device));
    if (n_rows >= (1ull << 32) || n_cols > (1ull << 32))
        throw InvalidArgument("graph: n_rows and n_cols must fit 32-bit indices");
    DeviceGuard dg(device);
    auto g = std::make_unique<Graph>();
    g->device = device;
    g->n_rows = n_rows;
    g->n_cols = n_cols;
    g->nnz = nnz;
    g->has_val = has_val;
    g->sms = device_sms();
    ASB_CUDA(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
    ASB_CUDA(cudaEventCreateWithFlags(&g->ev_last_op, cudaEventDisableTiming));
    g->rowptr.alloc(n_rows + 1);
    g->colind.alloc(nnz);
    if (has_val) g->val.alloc(nnz);
    return g;
}

std::unique_ptr<Graph> graph_create_host(const std::uint64_t* rowptr, const std::uint32_t* colind,
                                         const float* val, std::uint64_t n_rows,
                                         std::uint64_t n_cols, std::uint64_t nnz, int device,
                                         bool validate) {
    if (rowptr == nullptr) throw InvalidArgument("graph: rowptr required");
    if (nnz > 0 && colind == nullptr) throw InvalidArgument("graph: colind required");
    if (validate) {
        auto v = validate_csr(rowptr, n_rows + 1, colind, nnz, val ? nnz : 0, n_rows, n_cols);
        if (v) throw InvalidArgument("graph: " + v->invariant + " at index " + std::to_string(v->index));
    }
    auto g = alloc_graph(n_rows, n_cols, nnz, val != nullptr && nnz > 0, device);
    DeviceGuard dg(g->device);
    g->h_rowptr.assign(rowptr, rowptr + n_rows + 1);
    ASB_CUDA(cudaMemcpyAsync(g->rowptr.get(), rowptr, (n_rows + 1) * 8, cudaMemcpyHostToDevice,
                             g->stream));
    if (nnz) {
        ASB_CUDA(cudaMemcpyAsync(g->colind.get(), colind, nnz * 4, cudaMemcpyHostToDevice, g->stream));
        if (g->has_val)
            ASB_CUDA(cudaMemcpyAsync(g->val.get(), val, nnz * 4, cudaMemcpyHostToDevice, g->stream));
    }
    ASB_CUDA(cudaStreamSynchronize(g->stream));
    start_sig(*g);
    return g;
}

std::unique_ptr<Graph> graph_create_device(const std::uint64_t* rowptr, const std::uint32_t* colind,
                                           const float* val, std::uint64_t n_rows,
                                           std::uint64_t n_cols, std::uint64_t nnz, int device,
                                           cudaStream_t caller) {
    if (rowptr == nullptr) throw InvalidArgument("graph: rowptr required");
    if (nnz > 0 && colind == nullptr) throw InvalidArgument("graph: colind required");
    auto g = alloc_graph(n_rows, n_cols, nnz, val != nullptr && nnz > 0, device);
    DeviceGuard dg(g->device);
    // the caller's arrays may still be in flight on its stream: copy after them
    cudaEvent_t ready = nullptr;
    ASB_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    ASB_CUDA(cudaEventRecord(ready, caller));
    ASB_CUDA(cudaStreamWaitEvent(g->stream, ready, 0));
    cudaEventDestroy(ready);
    ASB_CUDA(cudaMemcpyAsync(g->rowptr.get(), rowptr, (n_rows + 1) * 8, cudaMemcpyDeviceToDevice,
                             g->stream));
    if (nnz) {
        ASB_CUDA(cudaMemcpyAsync(g->colind.get(), colind, nnz * 4, cudaMemcpyDeviceToDevice, g->stream));
        if (g->has_val)
            ASB_CUDA(cudaMemcpyAsync(g->val.get(), val, nnz * 4, cudaMemcpyDeviceToDevice, g->stream));
    }
    g->h_rowptr.resize(n_rows + 1);
    ASB_CUDA(cudaMemcpyAsync(g->h_rowptr.data(), rowptr, (n_rows + 1) * 8, cudaMemcpyDeviceToHost,
                             g->stream));
    ASB_CUDA(cudaStreamSynchronize(g->stream));
    if (g->h_rowptr[0] != 0) throw InvalidArgument("graph: rowptr[0] != 0 at index 0");
    if (g->h_rowptr[n_rows] != nnz) throw InvalidArgument("graph: rowptr[n_rows] != nnz at index " +
                                                          std::to_string(n_rows));
    for (std::uint64_t i = 1; i <= n_rows; ++i)
        if (g->h_rowptr[i] < g->h_rowptr[i - 1])
            throw InvalidArgument("graph: rowptr non-decreasing at index " + std::to_string(i));
    if (nnz) {
        DevBuf<unsigned> bad(1);
        ASB_CUDA(cudaMemsetAsync(bad.get(), 0, 4, g->stream));
        validate_cols_kernel<<<grid_for(n_rows * 32, 256, unsigned(g->sms) * 8u), 256, 0, g->stream>>>(
            g->rowptr.get(), n_rows, g->colind.get(), n_cols, bad.get());
        check_launch("validate_cols_kernel");
        unsigned hb = 0;
        ASB_CUDA(cudaMemcpyAsync(&hb, bad.get(), 4, cudaMemcpyDeviceToHost, g->stream));
        ASB_CUDA(cudaStreamSynchronize(g->stream));
        if (hb & 1u) throw InvalidArgument("graph: column index >= n_cols");
        if (hb & 2u) throw InvalidArgument("graph: columns not strictly increasing within a row");
    }
    start_sig(*g);
    return g;
}

// ---- operator serialisation and launch setup ---------------------------------------
GraphUse::GraphUse(Graph& g, cudaStream_t s) : g_(g), s_(s), lk_(g.op_mu) {
    if (!g_.ev_last_op) ASB_CUDA(cudaEventCreateWithFlags(&g_.ev_last_op, cudaEventDisableTiming));
    if (g_.op_depth++ == 0 && g_.last_op_stream && g_.last_op_stream != s_)
        ASB_CUDA(cudaStreamWaitEvent(s_, g_.ev_last_op, 0));
}

GraphUse::~GraphUse() {
    if (--g_.op_depth == 0) {
        if (cudaEventRecord(g_.ev_last_op, s_) == cudaSuccess) {
            g_.last_op_stream = s_;
        } else {
            g_.last_op_stream = nullptr;
            (void)cudaGetLastError();  // a destructor cannot throw: do not leave it sticky
        }
    }
}

int device_sms() {
    static std::mutex mu;
    static std::map<int, int> cache;
    int dev = 0;
    ASB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    int sms = 148;
    ASB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    cache[dev] = sms;
    return sms;
}

int kernel_setup(const void* kernel, std::size_t smem, int threads) {
    static std::mutex mu;
    static std::map<std::tuple<const void*, int, std::size_t, int>, int> done;
    // the attribute is per function: only ever raise it, so a launch with a
    // larger footprint is never left under a later, smaller setting
    static std::map<std::pair<const void*, int>, std::size_t> smem_set;
    int dev = 0;
    ASB_CUDA(cudaGetDevice(&dev));
    const auto key = std::make_tuple(kernel, dev, smem, threads);
    std::lock_guard<std::mutex> lk(mu);
    auto it = done.find(key);
    if (it != done.end()) return it->second;
    std::size_t& cur = smem_set[std::make_pair(kernel, dev)];
    if (smem > 48 * 1024 && smem > cur) {
        ASB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        cur = smem;
    }
    int per_sm = 1;
    ASB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
    done[key] = per_sm;
    return per_sm;
}

// graph_sig (src/cache.cpp:66-74).  colind streams down in chunks on `s`
// while the previous chunk is hashed (FNV-1a is inherently serial).  Reads
// only what never changes after creation (sizes, h_rowptr, colind).
// Pinned staging buffers of compute_sig, kept for the process: cudaMallocHost
// and cudaFreeHost synchronise with the device, which a hash running in the
// background must not do to the caller's streams on every graph.
namespace {
constexpr std::uint64_t kSigChunk = 8u << 20;  // elements per staging buffer
// never destroyed: a background hash may still return its buffers while the
// process tears down its statics
struct SigPool {
    std::mutex mu;
    std::vector<std::uint32_t*> free;
};
SigPool& sig_pool() {
    static SigPool* pool = new SigPool;
    return *pool;
}

std::uint32_t* sig_buf_acquire() {
    {
        std::lock_guard<std::mutex> lk(sig_pool().mu);
        if (!sig_pool().free.empty()) {
            std::uint32_t* p = sig_pool().free.back();
            sig_pool().free.pop_back();
            return p;
        }
    }
    std::uint32_t* p = nullptr;
    ASB_CUDA(cudaMallocHost(&p, kSigChunk * 4));
    return p;
}

void sig_buf_release(std::uint32_t* p) {
    std::lock_guard<std::mutex> lk(sig_pool().mu);
    sig_pool().free.push_back(p);
}
}  // namespace

static std::uint64_t compute_sig(const Graph& g, cudaStream_t s) {
    std::uint64_t h = kFnvOffset;
    h = fnv1a(h, &g.n_rows, 8);
    h = fnv1a(h, &g.n_cols, 8);
    h = fnv1a(h, &g.nnz, 8);
    h = fnv1a(h, g.h_rowptr.data(), (g.n_rows + 1) * 8);
    if (g.nnz) {
        const std::uint64_t chunk = kSigChunk;
        struct Bufs {
            std::uint32_t* p[2] = {nullptr, nullptr};
            ~Bufs() {
                for (auto* q : p)
                    if (q) sig_buf_release(q);
            }
        } bufs;
        bufs.p[0] = sig_buf_acquire();
        bufs.p[1] = sig_buf_acquire();
        std::uint32_t* const* pinned = bufs.p;
        cudaEvent_t ev[2];
        ASB_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
        ASB_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
        const std::uint64_t n_chunks = (g.nnz + chunk - 1) / chunk;
        auto issue = [&](std::uint64_t k) {
            const std::uint64_t off = k * chunk, len = std::min(chunk, g.nnz - off);
            ASB_CUDA(cudaMemcpyAsync(pinned[k & 1], g.colind.get() + off, len * 4,
                                     cudaMemcpyDeviceToHost, s));
            ASB_CUDA(cudaEventRecord(ev[k & 1], s));
        };
        issue(0);
        for (std::uint64_t k = 0; k < n_chunks; ++k) {
            ASB_CUDA(cudaEventSynchronize(ev[k & 1]));
            if (k + 1 < n_chunks) issue(k + 1);
            const std::uint64_t off = k * chunk, len = std::min(chunk, g.nnz - off);
            h = fnv1a(h, pinned[k & 1], len * 4);
        }
        cudaEventDestroy(ev[0]);
        cudaEventDestroy(ev[1]);
    }
    return h;
}

// memoized; waits for the background computation when one was started
std::uint64_t graph_sig(Graph& g) {
    std::lock_guard<std::mutex> lk(g.mu);
    if (g.sig) return *g.sig;
    DeviceGuard dg(g.device);
    if (g.sig_future.valid()) {
        g.sig = g.sig_future.get();  // rethrows a failure of the background pass
        return *g.sig;
    }
    g.sig = compute_sig(g, g.stream);
    return *g.sig;
}

// Start graph_sig in the background at creation (graphs of >= 1M entries;
// AUTOSAGE_EAGER_SIG=0 turns it off): the first decide then finds the key
// ready instead of spending ~0.5 s per 460 MB of colind on it.
void start_sig(Graph& g) {
    const auto knob = env::get_int("AUTOSAGE_EAGER_SIG");
    if ((knob && *knob == 0) || g.nnz < (1u << 20)) return;
    Graph* gp = &g;
    g.sig_future = std::async(std::launch::async, [gp] {
        ASB_CUDA(cudaSetDevice(gp->device));
        cudaStream_t s = nullptr;
        ASB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        struct StreamGuard {
            cudaStream_t s;
            ~StreamGuard() { cudaStreamDestroy(s); }
        } sg{s};
        return compute_sig(*gp, s);
    });
}

// Stable sort of rows by degree, descending (std::stable_sort with
// deg(a) > deg(b), src/generate.cpp:145-147): CUB's radix sort is stable.
void ensure_order(Graph& g) {
    std::lock_guard<std::mutex> lk(g.mu);
    if (g.order_ready) return;
    DeviceGuard dg(g.device);
    const std::uint64_t n = g.n_rows;
    g.order.alloc(std::max<std::uint64_t>(n, 1));
    g.sorted_deg.alloc(std::max<std::uint64_t>(n, 1));
    if (n > 0) {
        DevBuf<std::uint32_t> deg(n), idx(n);
        degrees_iota_kernel<<<grid_for(n, 256), 256, 0, g.stream>>>(g.rowptr.get(), n, deg.get(),
                                                                     idx.get());
        check_launch("degrees_iota_kernel");
        std::size_t temp_bytes = 0;
        ASB_CUDA(cub::DeviceRadixSort::SortPairsDescending(
            nullptr, temp_bytes, deg.get(), g.sorted_deg.get(), idx.get(), g.order.get(), int(n), 0,
            32, g.stream));
        DevBuf<unsigned char> temp(temp_bytes);
        ASB_CUDA(cub::DeviceRadixSort::SortPairsDescending(
            temp.get(), temp_bytes, deg.get(), g.sorted_deg.get(), idx.get(), g.order.get(), int(n),
            0, 32, g.stream));
        count_launch(4);
        ASB_CUDA(cudaStreamSynchronize(g.stream));
    }
    g.order_ready = true;
}

void ensure_chunk_rows(Graph& g) {
    std::lock_guard<std::mutex> lk(g.mu);
    if (g.chunk_ready) return;
    DeviceGuard dg(g.device);
    const std::uint64_t n_chunks = (g.nnz + 31) / 32;
    g.chunk_row.alloc(std::max<std::uint64_t>(n_chunks, 1));
    if (g.n_rows > 0 && g.nnz > 0) {
        chunk_row_kernel<<<grid_for(g.n_rows, 256), 256, 0, g.stream>>>(g.rowptr.get(), g.n_rows,
                                                                         g.chunk_row.get());
        check_launch("chunk_row_kernel");
        ASB_CUDA(cudaStreamSynchronize(g.stream));
    }
    g.chunk_ready = true;
}

// extract_features (src/csr.cpp:108-135) on device: the stable descending
// degree sort gives nearest-rank quantiles as asc[r-1] == desc[n-r].
as_features graph_features(Graph& g, std::uint64_t hub_threshold) {
    {
        std::lock_guard<std::mutex> lk(g.mu);
        auto it = g.features.find(hub_threshold);
        if (it != g.features.end()) return it->second;
    }
    as_features gf{};
    gf.n_rows = g.n_rows;
    gf.n_cols = g.n_cols;
    gf.nnz = g.nnz;
    gf.hub_threshold = hub_threshold;
    if (g.n_rows > 0) {
        ensure_order(g);
        DeviceGuard dg(g.device);
        const std::uint64_t n = g.n_rows;
        auto rank_of = [&](double q) {
            std::uint64_t r = std::uint64_t(std::ceil(q * double(n)));
            if (r == 0) r = 1;
            if (r > n) r = n;
            return r;
        };
        const double qs[5] = {0.25, 0.50, 0.75, 0.90, 0.99};
        std::uint32_t vals[6];
        for (int i = 0; i < 5; ++i) {
            const std::uint64_t r = rank_of(qs[i]);
            ASB_CUDA(cudaMemcpyAsync(&vals[i], g.sorted_deg.get() + (n - r), 4,
                                     cudaMemcpyDeviceToHost, g.stream));
        }
        ASB_CUDA(cudaMemcpyAsync(&vals[5], g.sorted_deg.get(), 4, cudaMemcpyDeviceToHost, g.stream));
        DevBuf<unsigned long long> cnt(2);
        ASB_CUDA(cudaMemsetAsync(cnt.get(), 0, 16, g.stream));
        count_heavy_empty_kernel<<<grid_for(n, 256, 592), 256, 0, g.stream>>>(
            g.sorted_deg.get(), n, hub_threshold, cnt.get());
        check_launch("count_heavy_empty_kernel");
        unsigned long long hc[2];
        ASB_CUDA(cudaMemcpyAsync(hc, cnt.get(), 16, cudaMemcpyDeviceToHost, g.stream));
        ASB_CUDA(cudaStreamSynchronize(g.stream));
        gf.deg_p25 = vals[0];
        gf.deg_p50 = vals[1];
        gf.deg_p75 = vals[2];
        gf.deg_p90 = vals[3];
        gf.deg_p99 = vals[4];
        gf.deg_max = vals[5];
        gf.mean_degree = double(g.nnz) / double(n);
        gf.heavy_row_fraction = double(hc[0]) / double(n);
        gf.empty_row_fraction = double(hc[1]) / double(n);
    }
    std::lock_guard<std::mutex> lk(g.mu);
    g.features[hub_threshold] = gf;
    return gf;
}

// sample_row_indices (src/generate.cpp:134-153)
std::vector<std::uint64_t> sample_row_indices(Graph& g, double frac, std::uint64_t min_rows) {
    if (frac <= 0.0 || frac > 1.0) throw InvalidArgument("sample: frac must be in (0,1]");
    std::vector<std::uint64_t> rows;
    const std::uint64_t n = g.n_rows;
    if (n == 0) return rows;
    std::uint64_t s = std::uint64_t(std::ceil(frac * double(n)));
    s = std::max(s, min_rows);
    s = std::min(s, n);
    const std::uint64_t stride = std::max<std::uint64_t>(1, n / s);
    ensure_order(g);
    DeviceGuard dg(g.device);
    DevBuf<std::uint64_t> out(s);
    gather_u32_strided_kernel<<<unsigned((s + 255) / 256), 256, 0, g.stream>>>(g.order.get(), s,
                                                                               stride, out.get());
    check_launch("gather_u32_strided_kernel");
    rows.resize(s);
    ASB_CUDA(cudaMemcpyAsync(rows.data(), out.get(), s * 8, cudaMemcpyDeviceToHost, g.stream));
    ASB_CUDA(cudaStreamSynchronize(g.stream));
    return rows;
}

// slice_rows (src/generate.cpp:155-176), on device
std::unique_ptr<Graph> slice_rows(Graph& g, const std::vector<std::uint64_t>& rows,
                                  const float* vals) {
    DeviceGuard dg(g.device);
    const std::uint64_t s = rows.size();
    for (auto r : rows)
        if (r >= g.n_rows) throw InvalidArgument("slice_rows: row index out of range");
    std::uint64_t nnz = 0;
    for (auto r : rows) nnz += g.h_rowptr[r + 1] - g.h_rowptr[r];
    auto out = alloc_graph(s, g.n_cols, nnz, vals != nullptr, g.device);
    out->plan_nnz = g.plan_nnz ? g.plan_nnz : g.nnz;
    out->h_rowptr.resize(s + 1);
    out->h_rowptr[0] = 0;
    for (std::uint64_t r = 0; r < s; ++r)
        out->h_rowptr[r + 1] = out->h_rowptr[r] + (g.h_rowptr[rows[r] + 1] - g.h_rowptr[rows[r]]);
    ASB_CUDA(cudaMemcpyAsync(out->rowptr.get(), out->h_rowptr.data(), (s + 1) * 8,
                             cudaMemcpyHostToDevice, g.stream));
    if (s > 0 && nnz > 0) {
        DevBuf<std::uint64_t> d_rows(s);
        ASB_CUDA(cudaMemcpyAsync(d_rows.get(), rows.data(), s * 8, cudaMemcpyHostToDevice, g.stream));
        const unsigned blocks = unsigned((s * 32 + 255) / 256);
        slice_copy_kernel<<<blocks, 256, 0, g.stream>>>(
            g.rowptr.get(), g.colind.get(), vals, d_rows.get(), s,
            out->rowptr.get(), out->colind.get(), out->has_val ? out->val.get() : nullptr);
        check_launch("slice_copy_kernel");
        ASB_CUDA(cudaStreamSynchronize(g.stream));
    }
    ASB_CUDA(cudaStreamSynchronize(g.stream));
    return out;
}

std::unique_ptr<Graph> row_range(Graph& g, std::uint64_t r0, std::uint64_t r1) {
    if (r0 > r1 || r1 > g.n_rows) throw InvalidArgument("row_range: bad range");
    DeviceGuard dg(g.device);
    const std::uint64_t e0 = g.h_rowptr[r0], e1 = g.h_rowptr[r1];
    auto out = alloc_graph(r1 - r0, g.n_cols, e1 - e0, g.has_val, g.device);
    out->h_rowptr.resize(r1 - r0 + 1);
    for (std::uint64_t i = r0; i <= r1; ++i) out->h_rowptr[i - r0] = g.h_rowptr[i] - e0;
    rebase_rowptr_kernel<<<unsigned((r1 - r0 + 1 + 255) / 256), 256, 0, g.stream>>>(
        g.rowptr.get() + r0, r1 - r0 + 1, e0, out->rowptr.get());
    check_launch("rebase_rowptr_kernel");
    if (e1 > e0) {
        ASB_CUDA(cudaMemcpyAsync(out->colind.get(), g.colind.get() + e0, (e1 - e0) * 4,
                                 cudaMemcpyDeviceToDevice, g.stream));
        if (g.has_val)
            ASB_CUDA(cudaMemcpyAsync(out->val.get(), g.val.get() + e0, (e1 - e0) * 4,
                                     cudaMemcpyDeviceToDevice, g.stream));
    }
    ASB_CUDA(cudaStreamSynchronize(g.stream));
    return out;
}

// Heavy rows (degree >= threshold) cut into 2048-nnz pieces
// (src/kernels.cpp:129-142).  A heavy row with a single piece reduces to
// 0.0 + partial == partial (the partial is never -0.0), so it writes C
// directly; multi-piece rows get partial slots and an ordered reduce.
// the light rows of a hub plan as direct-write items (HubPlan::all_*)
__global__ void light_items_kernel(const std::uint32_t* __restrict__ rows, std::uint64_t n,
                                   const std::uint64_t* __restrict__ rowptr, std::uint32_t* __restrict__ row,
                                   std::uint64_t* __restrict__ e0, std::uint32_t* __restrict__ len,
                                   std::uint32_t* __restrict__ slot) {
    for (std::uint64_t i = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += std::uint64_t(gridDim.x) * blockDim.x) {
        const std::uint32_t r = rows[i];
        const std::uint64_t a = rowptr[r];
        row[i] = r;
        e0[i] = a;
        len[i] = std::uint32_t(rowptr[r + 1] - a);
        slot[i] = 0xffffffffu;
    }
}

const HubPlan& ensure_hub_plan(Graph& g, std::uint64_t threshold) {
    {
        std::lock_guard<std::mutex> lk(g.mu);
        auto it = g.hub_plans.find(threshold);
        if (it != g.hub_plans.end()) return *it->second;
    }
    ensure_order(g);
    DeviceGuard dg(g.device);
    auto plan = std::make_unique<HubPlan>();
    plan->threshold = threshold;
    std::vector<std::uint32_t> prow, plen, pslot, rrow, rfirst, rcount;
    std::vector<std::uint64_t> pe0;
    std::uint64_t slots = 0, heavy = 0;
    for (std::uint64_t i = 0; i < g.n_rows; ++i) {
        const std::uint64_t e0 = g.h_rowptr[i], e1 = g.h_rowptr[i + 1];
        if (e1 - e0 < threshold) continue;
        ++heavy;
        const std::uint64_t np = (e1 - e0 + kHubNnzChunk - 1) / kHubNnzChunk;
        if (np > 1) {
            rrow.push_back(std::uint32_t(i));
            rfirst.push_back(std::uint32_t(slots));
            rcount.push_back(std::uint32_t(np));
        }
        for (std::uint64_t p = 0; p < np; ++p) {
            const std::uint64_t p0 = e0 + p * kHubNnzChunk;
            prow.push_back(std::uint32_t(i));
            pe0.push_back(p0);
            plen.push_back(std::uint32_t(std::min(kHubNnzChunk, e1 - p0)));
            pslot.push_back(np > 1 ? std::uint32_t(slots + p) : 0xffffffffu);
        }
        if (np > 1) slots += np;
    }
    plan->n_heavy = heavy;
    plan->n_light = g.n_rows - heavy;
    plan->n_pieces = prow.size();
    plan->n_slots = slots;
    plan->n_red = rrow.size();
    // light rows are the degree-descending order's tail past the heavy prefix
    // (launched by offset); pieces go longest-first so a warp's groups get
    // equal-length pieces and the long ones start early (LPT)
    {
        std::vector<std::uint32_t> perm(prow.size());
        for (std::size_t i = 0; i < perm.size(); ++i) perm[i] = std::uint32_t(i);
        std::stable_sort(perm.begin(), perm.end(),
                         [&](std::uint32_t a, std::uint32_t b) { return plen[a] > plen[b]; });
        auto apply = [&](auto& v) {
            auto tmp = v;
            for (std::size_t i = 0; i < perm.size(); ++i) v[i] = tmp[perm[i]];
        };
        apply(prow);
        apply(pe0);
        apply(plen);
        apply(pslot);
    }
    auto up32 = [&](DevBuf<std::uint32_t>& d, const std::vector<std::uint32_t>& h) {
        d.alloc(std::max<std::size_t>(h.size(), 1));
        if (!h.empty())
            ASB_CUDA(cudaMemcpyAsync(d.get(), h.data(), h.size() * 4, cudaMemcpyHostToDevice, g.stream));
    };
    up32(plan->piece_row, prow);
    up32(plan->piece_len, plen);
    up32(plan->piece_slot, pslot);
    up32(plan->red_row, rrow);
    up32(plan->red_first, rfirst);
    up32(plan->red_count, rcount);
    plan->piece_e0.alloc(std::max<std::size_t>(pe0.size(), 1));
    if (!pe0.empty())
        ASB_CUDA(cudaMemcpyAsync(plan->piece_e0.get(), pe0.data(), pe0.size() * 8,
                                 cudaMemcpyHostToDevice, g.stream));
    {
        const std::uint64_t n_all = plan->n_pieces + plan->n_light;
        plan->all_row.alloc(std::max<std::uint64_t>(n_all, 1));
        plan->all_len.alloc(std::max<std::uint64_t>(n_all, 1));
        plan->all_slot.alloc(std::max<std::uint64_t>(n_all, 1));
        plan->all_e0.alloc(std::max<std::uint64_t>(n_all, 1));
        if (plan->n_pieces) {
            const std::uint64_t np = plan->n_pieces;
            ASB_CUDA(cudaMemcpyAsync(plan->all_row.get(), plan->piece_row.get(), np * 4, cudaMemcpyDeviceToDevice,
                                     g.stream));
            ASB_CUDA(cudaMemcpyAsync(plan->all_len.get(), plan->piece_len.get(), np * 4, cudaMemcpyDeviceToDevice,
                                     g.stream));
            ASB_CUDA(cudaMemcpyAsync(plan->all_slot.get(), plan->piece_slot.get(), np * 4, cudaMemcpyDeviceToDevice,
                                     g.stream));
            ASB_CUDA(cudaMemcpyAsync(plan->all_e0.get(), plan->piece_e0.get(), np * 8, cudaMemcpyDeviceToDevice,
                                     g.stream));
        }
        if (plan->n_light) {
            light_items_kernel<<<grid_for(plan->n_light, 256), 256, 0, g.stream>>>(
                g.order.get() + plan->n_heavy, plan->n_light, g.rowptr.get(), plan->all_row.get() + plan->n_pieces,
                plan->all_e0.get() + plan->n_pieces, plan->all_len.get() + plan->n_pieces,
                plan->all_slot.get() + plan->n_pieces);
            check_launch("light_items_kernel");
        }
    }
    ASB_CUDA(cudaStreamSynchronize(g.stream));
    std::lock_guard<std::mutex> lk(g.mu);
    auto& slot = g.hub_plans[threshold];
    if (!slot) slot = std::move(plan);
    return *slot;
}

void gather_dense_rows(const float* src, std::uint64_t f, const std::vector<std::uint64_t>& rows,
                       float* dst, cudaStream_t s) {
    if (rows.empty() || f == 0) return;
    DevBuf<std::uint64_t> d_rows(rows.size());
    ASB_CUDA(cudaMemcpyAsync(d_rows.get(), rows.data(), rows.size() * 8, cudaMemcpyHostToDevice, s));
    gather_rows_kernel<<<grid_for(rows.size() * f, 256), 256, 0, s>>>(src, f, d_rows.get(),
                                                                      rows.size(), dst);
    check_launch("gather_rows_kernel");
    ASB_CUDA(cudaStreamSynchronize(s));
}

} // namespace asb

namespace asb {

namespace {
__global__ void finite_check_kernel(const float* __restrict__ p, std::uint64_t n,
                                    unsigned* __restrict__ flag) {
    bool bad = false;
    const std::uint64_t stride = std::uint64_t(gridDim.x) * blockDim.x;
    std::uint64_t i = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x;
    if ((reinterpret_cast<std::uintptr_t>(p) & 15) == 0) {
        const std::uint64_t n4 = n / 4;
        const uint4* p4 = reinterpret_cast<const uint4*>(p);
        for (std::uint64_t k = i; k < n4; k += stride) {
            const uint4 v = __ldg(p4 + k);
            bad |= ((v.x & 0x7F800000u) == 0x7F800000u) | ((v.y & 0x7F800000u) == 0x7F800000u) |
                   ((v.z & 0x7F800000u) == 0x7F800000u) | ((v.w & 0x7F800000u) == 0x7F800000u);
        }
        for (std::uint64_t k = n4 * 4 + i; k < n; k += stride)
            bad |= (__float_as_uint(p[k]) & 0x7F800000u) == 0x7F800000u;
    } else {
        for (std::uint64_t k = i; k < n; k += stride)
            bad |= (__float_as_uint(p[k]) & 0x7F800000u) == 0x7F800000u;
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *flag = 0u;
}

// 16-bit words (half.cuh): exponent field all ones (bf16 0x7F80, f16 0x7C00)
// = Inf/NaN
template <unsigned M>
__global__ void finite_check_half_kernel(const unsigned short* __restrict__ p, std::uint64_t n,
                                         unsigned* __restrict__ flag) {
    bool bad = false;
    const std::uint64_t stride = std::uint64_t(gridDim.x) * blockDim.x;
    const std::uint64_t i = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x;
    if ((reinterpret_cast<std::uintptr_t>(p) & 15) == 0) {
        const std::uint64_t n8 = n / 8;
        const uint4* p8 = reinterpret_cast<const uint4*>(p);
        for (std::uint64_t k = i; k < n8; k += stride) {
            const uint4 v = __ldg(p8 + k);
            for (unsigned w : {v.x, v.y, v.z, v.w})
                bad |= ((w & M) == M) | ((w & (M << 16)) == (M << 16));
        }
        for (std::uint64_t k = n8 * 8 + i; k < n; k += stride) bad |= (p[k] & M) == M;
    } else {
        for (std::uint64_t k = i; k < n; k += stride) bad |= (p[k] & M) == M;
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *flag = 0u;
}
}  // namespace

const unsigned* finite_flag_half(Graph& g, const std::uint16_t* p, std::uint64_t n, cudaStream_t s, int wt) {
    g.flag.ensure(1);
    // nothing to widen: 0, the safe path; else 0x01010101 (nonzero = finite)
    // until the scan clears it -- one memset
    const bool empty = n == 0 || p == nullptr;
    ASB_CUDA(cudaMemsetAsync(g.flag.get(), empty ? 0 : 1, 4, s));
    if (empty) return g.flag.get();
    const std::uint64_t want = (n / 8 + 255) / 256 + 1;
    const unsigned blocks = unsigned(std::min<std::uint64_t>(want, std::uint64_t(g.sms) * 8));
    if (wt == kWtF16) finite_check_half_kernel<half_inf_mask<kWtF16>()><<<blocks, 256, 0, s>>>(p, n, g.flag.get());
    else finite_check_half_kernel<half_inf_mask<kWtBF16>()><<<blocks, 256, 0, s>>>(p, n, g.flag.get());
    check_launch("finite_check_half_kernel");
    return g.flag.get();
}

const unsigned* finite_flag(Graph& g, const float* p, std::uint64_t n, cudaStream_t s) {
    g.flag.ensure(1);
    // nothing to widen: 0, the safe path; else 0x01010101 (nonzero = finite)
    // until the scan clears it -- one memset
    const bool empty = n == 0 || p == nullptr;
    ASB_CUDA(cudaMemsetAsync(g.flag.get(), empty ? 0 : 1, 4, s));
    if (empty) return g.flag.get();
    const std::uint64_t want = (n / 4 + 255) / 256 + 1;
    const unsigned blocks = unsigned(std::min<std::uint64_t>(want, std::uint64_t(g.sms) * 8));
    finite_check_kernel<<<blocks, 256, 0, s>>>(p, n, g.flag.get());
    check_launch("finite_check_kernel");
    return g.flag.get();
}

}  // namespace asb
