// backward.cu -- the pieces the operators' gradients need beyond SpMM and
// SDDMM themselves (the reference has no backward pass,
// PAPER.md:334).  With C = A B and out = SDDMM(A, X, Y):
//   dB   = A^T dC          SpMM on the transposed graph, values permuted
//   dval = SDDMM(A, dC, B)
//   dX   = A[dout] Y       SpMM with the SDDMM gradient as values
//   dY   = A^T[dout] X
// and the row softmax's gradient ds = p * (g - sum_row p*g).
//
// Transpose: stable CUB radix sort of (column, entry) pairs over the column
// bits only, so entries of one column keep source (= row) order and the
// result is canonical CSR; counts -> exclusive scan give rowptr.  It runs once
// per graph (the torch ops cache the transposed handle), so it is built from
// library passes rather than a hand-fused kernel: every pass is a coalesced
// stream except the sort's scatter and the fill's two gathers.
//
// Softmax backward: HBM-bound (12 B per entry + 8 B per row).  The exact
// products f64(p)*f64(g) are summed as 256 strided partials folded in a fixed
// tree, so the sum is deterministic and equals oracle/oracle.c
// orc_row_softmax_backward bit for bit; a warp per row (eight chains per lane)
// or, for rows of >= 4096 entries, a CTA per row (one chain per thread).
#include "graph.hpp"
#include "ops.hpp"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>

namespace asb {

namespace {

// grid-stride launches: at most `cap` CTAs (default 16 per SM of the device)
unsigned grid_for(std::uint64_t n, unsigned block, unsigned cap = 0) {
    if (cap == 0) cap = unsigned(device_sms()) * 16u;
    std::uint64_t g = (n + block - 1) / block;
    if (g == 0) g = 1;
    return unsigned(std::min<std::uint64_t>(g, cap));
}

__global__ void col_count_kernel(const std::uint32_t* __restrict__ colind, std::uint64_t nnz,
                                 unsigned long long* __restrict__ cnt) {
    for (std::uint64_t e = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; e < nnz;
         e += std::uint64_t(gridDim.x) * blockDim.x)
        atomicAdd(&cnt[colind[e]], 1ull);
}

__global__ void iota_u32_kernel(std::uint32_t* __restrict__ p, std::uint64_t n) {
    for (std::uint64_t i = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += std::uint64_t(gridDim.x) * blockDim.x)
        p[i] = std::uint32_t(i);
}

// erow[e] = row of entry e (warp per row, lanes stride the row)
__global__ void entry_row_kernel(const std::uint64_t* __restrict__ rowptr, std::uint64_t n_rows,
                                 std::uint32_t* __restrict__ erow) {
    const int lane = threadIdx.x & 31;
    for (std::uint64_t w = (blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x) >> 5; w < n_rows;
         w += (std::uint64_t(gridDim.x) * blockDim.x) >> 5) {
        const std::uint64_t e1 = rowptr[w + 1];
        for (std::uint64_t e = rowptr[w] + lane; e < e1; e += 32) erow[e] = std::uint32_t(w);
    }
}

__global__ void transpose_fill_kernel(const std::uint32_t* __restrict__ perm,
                                      const std::uint32_t* __restrict__ erow,
                                      const float* __restrict__ val, std::uint64_t nnz,
                                      std::uint32_t* __restrict__ colind_t, float* __restrict__ val_t) {
    for (std::uint64_t k = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; k < nnz;
         k += std::uint64_t(gridDim.x) * blockDim.x) {
        const std::uint32_t e = perm[k];
        colind_t[k] = erow[e];
        if (val) val_t[k] = val[e];
    }
}

__global__ void permute_kernel(const float* __restrict__ src, const std::uint32_t* __restrict__ perm,
                               std::uint64_t n, float* __restrict__ dst) {
    for (std::uint64_t k = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; k < n;
         k += std::uint64_t(gridDim.x) * blockDim.x)
        dst[k] = src[perm[k]];
}

// Softmax gradient.  dot = the fixed fold of 256 strided partials (partial
// l sums entries e0 + l, e0 + l + 256, ... in order; then part[l] +=
// part[l + o] for o = 128 .. 1), the order oracle/oracle.c restates.
//
// Warp kernel: lane l owns partials l + 32j, j = 0..7 -- eight independent
// f64 chains and 16 loads in flight per lane; the o = 128, 64, 32 steps of
// the fold are inside the lane, o = 16 .. 1 are xor shuffles (lane 0 then
// holds the oracle's association).
__device__ __forceinline__ void sbw_fma(double& part, float p, float g) {
    part = __dadd_rn(part, __dmul_rn(double(p), double(g)));
}

__device__ __forceinline__ void sbw_write(const float* __restrict__ p, const float* __restrict__ g,
                                          float* __restrict__ ds, std::uint64_t k0, std::uint64_t e1,
                                          std::uint64_t step, double dot) {
    std::uint64_t k = k0;
    for (; k + 3 * step < e1; k += 4 * step) {
        float pv[4], gv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            pv[u] = p[k + u * step];
            gv[u] = g[k + u * step];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            ds[k + u * step] = float(__dmul_rn(double(pv[u]), __dsub_rn(double(gv[u]), dot)));
    }
    for (; k < e1; k += step) ds[k] = float(__dmul_rn(double(p[k]), __dsub_rn(double(g[k]), dot)));
}

__global__ void __launch_bounds__(256)
softmax_backward_kernel(const std::uint64_t* __restrict__ rowptr, const std::uint32_t* __restrict__ order,
                        std::uint64_t n_rows, const float* __restrict__ p, const float* __restrict__ g,
                        float* __restrict__ ds) {
    const int lane = threadIdx.x & 31;
    for (std::uint64_t w = (blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x) >> 5; w < n_rows;
         w += (std::uint64_t(gridDim.x) * blockDim.x) >> 5) {
        const std::uint32_t row = order[w];
        const std::uint64_t e0 = rowptr[row], e1 = rowptr[row + 1];
        if (e0 == e1) continue;
        double part[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        std::uint64_t base = e0;
        for (; base + 256 <= e1; base += 256) {
            float pv[8], gv[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                pv[j] = __ldg(p + base + 32 * j + lane);
                gv[j] = __ldg(g + base + 32 * j + lane);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) sbw_fma(part[j], pv[j], gv[j]);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const std::uint64_t k = base + 32 * j + lane;
            if (k < e1) sbw_fma(part[j], __ldg(p + k), __ldg(g + k));
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) part[j] = __dadd_rn(part[j], part[j + 4]);  // o = 128
#pragma unroll
        for (int j = 0; j < 2; ++j) part[j] = __dadd_rn(part[j], part[j + 2]);  // o = 64
        double v = __dadd_rn(part[0], part[1]);                                // o = 32
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
        const double dot = __shfl_sync(0xffffffffu, v, 0);
        sbw_write(p, g, ds, e0 + lane, e1, 32, dot);  // the row was just read: L2 hits
    }
}

// CTA kernel for long rows (the first rows of the degree-descending order):
// warp w of 8 owns partials 32w + lane, so each chain has deg/256 terms; the
// o = 128, 64, 32 steps combine warps through shared memory in the same
// tree, o = 16 .. 1 are shuffles in warp 0.
__global__ void __launch_bounds__(256)
softmax_backward_cta_kernel(const std::uint64_t* __restrict__ rowptr, const std::uint32_t* __restrict__ order,
                            std::uint64_t n_long, const float* __restrict__ p, const float* __restrict__ g,
                            float* __restrict__ ds) {
    __shared__ double sp[256];
    __shared__ double sdot;
    const int t = threadIdx.x;
    for (std::uint64_t r = blockIdx.x; r < n_long; r += gridDim.x) {
        const std::uint32_t row = order[r];
        const std::uint64_t e0 = rowptr[row], e1 = rowptr[row + 1];
        double a = 0.0;  // partial t: one chain per thread, loads unrolled ahead of it
        std::uint64_t k = e0 + t;
        for (; k + 3 * 256 < e1; k += 4 * 256) {
            float pv[4], gv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                pv[u] = __ldg(p + k + 256 * u);
                gv[u] = __ldg(g + k + 256 * u);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) sbw_fma(a, pv[u], gv[u]);
        }
        for (; k < e1; k += 256) sbw_fma(a, __ldg(p + k), __ldg(g + k));
        sp[t] = a;
        __syncthreads();
        for (int o = 128; o >= 32; o >>= 1) {
            if (t < o) sp[t] = __dadd_rn(sp[t], sp[t + o]);
            __syncthreads();
        }
        if (t < 32) {
            double v = sp[t];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
            if (t == 0) sdot = v;
        }
        __syncthreads();
        const double dot = sdot;
        sbw_write(p, g, ds, e0 + t, e1, 256, dot);
        __syncthreads();  // sp / sdot reused by the next row
    }
}

} // namespace

std::unique_ptr<Graph> transpose_graph(Graph& g) {
    DeviceGuard dg(g.device);
    if (g.nnz >= (1ull << 31)) throw InvalidArgument("transpose: nnz must be < 2^31");
    auto t = std::make_unique<Graph>();
    t->device = g.device;
    t->n_rows = g.n_cols;
    t->n_cols = g.n_rows;
    t->nnz = g.nnz;
    t->has_val = g.has_val;
    t->sms = g.sms;
    ASB_CUDA(cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking));
    ASB_CUDA(cudaEventCreateWithFlags(&t->ev_last_op, cudaEventDisableTiming));
    t->rowptr.alloc(t->n_rows + 1);
    t->colind.alloc(g.nnz);
    if (t->has_val) t->val.alloc(g.nnz);
    t->src_perm.alloc(std::max<std::uint64_t>(g.nnz, 1));
    cudaStream_t s = g.stream;
    const std::uint64_t nnz = g.nnz, nc = g.n_cols;
    {
        DevBuf<unsigned long long> cnt(nc + 1);
        ASB_CUDA(cudaMemsetAsync(cnt.get(), 0, (nc + 1) * 8, s));
        if (nnz) {
            col_count_kernel<<<grid_for(nnz, 256), 256, 0, s>>>(g.colind.get(), nnz, cnt.get());
            check_launch("col_count_kernel");
        }
        std::size_t tb = 0;
        ASB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.get(), t->rowptr.get(), int(nc + 1), s));
        DevBuf<unsigned char> tmp(std::max<std::size_t>(tb, 1));
        ASB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, cnt.get(), t->rowptr.get(), int(nc + 1), s));
        count_launch(2);
    }
    if (nnz) {
        DevBuf<std::uint32_t> keys_out(nnz), iota(nnz), erow(nnz);
        iota_u32_kernel<<<grid_for(nnz, 256), 256, 0, s>>>(iota.get(), nnz);
        check_launch("iota_u32_kernel");
        entry_row_kernel<<<grid_for(g.n_rows * 32, 256), 256, 0, s>>>(g.rowptr.get(), g.n_rows, erow.get());
        check_launch("entry_row_kernel");
        int end_bit = 1;
        while (end_bit < 32 && (1ull << end_bit) < nc) ++end_bit;
        std::size_t tb = 0;
        ASB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, g.colind.get(), keys_out.get(), iota.get(),
                                                 t->src_perm.get(), int(nnz), 0, end_bit, s));
        DevBuf<unsigned char> tmp(std::max<std::size_t>(tb, 1));
        ASB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, g.colind.get(), keys_out.get(), iota.get(),
                                                 t->src_perm.get(), int(nnz), 0, end_bit, s));
        count_launch(4);
        transpose_fill_kernel<<<grid_for(nnz, 256), 256, 0, s>>>(
            t->src_perm.get(), erow.get(), g.has_val ? g.val.get() : nullptr, nnz, t->colind.get(),
            t->has_val ? t->val.get() : nullptr);
        check_launch("transpose_fill_kernel");
    }
    t->h_rowptr.resize(t->n_rows + 1);
    ASB_CUDA(cudaMemcpyAsync(t->h_rowptr.data(), t->rowptr.get(), (t->n_rows + 1) * 8,
                             cudaMemcpyDeviceToHost, s));
    ASB_CUDA(cudaStreamSynchronize(s));
    t->is_transpose = true;
    return t;
}

void launch_permute(const float* src, const std::uint32_t* perm, std::uint64_t n, float* dst,
                    cudaStream_t s) {
    if (n == 0) return;
    permute_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, perm, n, dst);
    check_launch("permute_kernel");
}

// Rows of at least kSbwLongRow entries (a prefix of the degree order) take
// the CTA kernel: one warp would run their 256 partials as deg/256-term chains
// eight at a time and set the kernel's tail (Reddit-shape's 21,657-entry hub).
constexpr std::uint64_t kSbwLongRow = 4096;

void launch_row_softmax_backward(Graph& g, const float* p, const float* grad, float* ds, cudaStream_t s) {
    if (g.n_rows == 0 || g.nnz == 0) return;
    ensure_order(g);
    const std::uint64_t n_long = rows_with_degree_at_least(g, kSbwLongRow);
    if (n_long) {
        softmax_backward_cta_kernel<<<unsigned(std::min<std::uint64_t>(n_long, unsigned(device_sms()) * 8u)), 256, 0, s>>>(
            g.rowptr.get(), g.order.get(), n_long, p, grad, ds);
        check_launch("softmax_backward_cta_kernel");
    }
    const std::uint64_t n_rest = g.n_rows - n_long;
    if (n_rest) {
        softmax_backward_kernel<<<grid_for(n_rest * 32, 256, unsigned(device_sms()) * 8u), 256, 0, s>>>(
            g.rowptr.get(), g.order.get() + n_long, n_rest, p, grad, ds);
        check_launch("softmax_backward_kernel");
    }
}

} // namespace asb
