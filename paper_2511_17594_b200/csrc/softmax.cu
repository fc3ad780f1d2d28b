// softmax.cu -- CSR row softmax for sm_100a (src/kernels.cpp:431-461).
//
// Per non-empty row: mx = max over the f32 values; ex_e = f32(exp(f64 v_e -
// f64 mx)); sum = f64 sum of ex_e in entry order; out_e = f32(f64 ex_e /
// sum).  Empty rows produce nothing.  The sum is accumulated sequentially
// in entry order (lane 0 folds each 32-entry chunk from shared memory), so
// the only difference from the CPU reference can come from exp() itself
// (CUDA's f64 exp vs libm, both within 1 ulp of f64, rounded to f32).
// The max ignores NaN where std::max would latch it; either way a NaN in a
// row makes every ex (or the sum) NaN, so all outputs of that row are NaN
// exactly as in the reference.
#include "ops.hpp"

#include <algorithm>

namespace asb {

namespace {

constexpr unsigned FULL = 0xffffffffu;

// lane 0 folds 32 staged f64 values into the row's sum, in entry order
__device__ __forceinline__ double fold_stage(double sum, const double* st, int n) {
    if (n == 32) {
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
            const double2 d = *reinterpret_cast<const double2*>(st + j);
            sum = __dadd_rn(sum, d.x);
            sum = __dadd_rn(sum, d.y);
        }
    } else {
        for (int j = 0; j < n; ++j) sum = __dadd_rn(sum, st[j]);
    }
    return sum;
}

// Warp per row, rows in degree-descending order.  Rows of at most kRowSmem
// entries stage their ex values in the warp's shared memory (one read of
// vin, one write of vout); longer rows take three passes over memory.
// Both: row max; ex_e = f32(exp(f64 v_e - f64 mx)) for 32 entries at a time,
// staged as f64 and folded into the row's sum by lane 0 in entry order (one
// DADD per entry on the chain, no shuffles); out_e = f32(f64 ex_e / sum).
constexpr int kRowSmem = 1024;
__global__ void __launch_bounds__(256) row_softmax_kernel(const std::uint64_t* __restrict__ rowptr,
                                                          const std::uint32_t* __restrict__ order,
                                                          std::uint64_t n_rows, const float* __restrict__ vin,
                                                          float* __restrict__ vout) {
    __shared__ __align__(16) double stage[8][32];
    __shared__ __align__(16) float exs_all[8][kRowSmem];
    const int lane = threadIdx.x & 31;
    double* st = stage[threadIdx.x >> 5];
    float* exs = exs_all[threadIdx.x >> 5];
    const std::uint64_t total_warps = std::uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (std::uint64_t w = (std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < n_rows;
         w += total_warps) {
        const std::uint64_t row = order[w];
        const std::uint64_t e0 = rowptr[row], e1 = rowptr[row + 1];
        if (e0 == e1) continue;
        const std::uint32_t deg = std::uint32_t(e1 - e0);
        if (deg <= std::uint32_t(kRowSmem)) {
            // ---- shared-memory path: values land in exs once
#pragma unroll 4
            for (std::uint32_t k = lane; k < deg; k += 32) exs[k] = __ldg(vin + e0 + k);
            __syncwarp();
            float mx = -INFINITY;
            for (std::uint32_t k = lane; k < deg; k += 32) mx = fmaxf(mx, exs[k]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, o));
            const double dmx = double(mx);
            double sum = 0.0;  // lane 0
            for (std::uint32_t base = 0; base < deg; base += 32) {
                const std::uint32_t k = base + lane;
                double exd = 0.0;
                if (k < deg) {
                    const float ex = float(exp(double(exs[k]) - dmx));
                    exs[k] = ex;
                    exd = double(ex);
                }
                st[lane] = exd;
                __syncwarp();
                if (lane == 0) sum = fold_stage(sum, st, (deg - base) < 32 ? int(deg - base) : 32);
                __syncwarp();
            }
            sum = __shfl_sync(FULL, sum, 0);
            for (std::uint32_t k = lane; k < deg; k += 32) vout[e0 + k] = float(__ddiv_rn(double(exs[k]), sum));
            __syncwarp();
            continue;
        }
        // ---- long rows: three passes
        float mx = -INFINITY;
#pragma unroll 8
        for (std::uint64_t e = e0 + lane; e < e1; e += 32) mx = fmaxf(mx, __ldg(vin + e));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, o));
        const double dmx = double(mx);
        double sum = 0.0;  // lane 0
        float vnext = e0 + lane < e1 ? __ldg(vin + e0 + lane) : 0.f;
        for (std::uint64_t base = e0; base < e1; base += 32) {
            const std::uint64_t e = base + lane;
            const float v = vnext;
            vnext = base + 32 + lane < e1 ? __ldg(vin + base + 32 + lane) : 0.f;
            double exd = 0.0;
            if (e < e1) {
                const float ex = float(exp(double(v) - dmx));
                vout[e] = ex;
                exd = double(ex);
            }
            st[lane] = exd;
            __syncwarp();
            if (lane == 0) sum = fold_stage(sum, st, (e1 - base) < 32 ? int(e1 - base) : 32);
            __syncwarp();
        }
        sum = __shfl_sync(FULL, sum, 0);
#pragma unroll 4
        for (std::uint64_t e = e0 + lane; e < e1; e += 32) vout[e] = float(__ddiv_rn(double(vout[e]), sum));
    }
}

} // namespace

void launch_row_softmax(Graph& g, const float* vin, float* vout, cudaStream_t s) {
    if (g.n_rows == 0 || g.nnz == 0) return;
    ensure_order(g);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const std::uint64_t want = (g.n_rows * 32 + 255) / 256;
    const unsigned blocks = unsigned(std::min<std::uint64_t>(want, std::uint64_t(sms) * 8));
    row_softmax_kernel<<<blocks, 256, 0, s>>>(g.rowptr.get(), g.order.get(), g.n_rows, vin, vout);
    check_launch("row_softmax_kernel");
}

} // namespace asb
