// softmax.cu -- CSR row softmax for sm_100a (src/kernels.cpp:431-461).
//
// Per non-empty row: mx = max over the f32 values; ex_e = f32(exp(f64 v_e -
// f64 mx)); sum = f64 sum of ex_e in entry order; out_e = f32(f64 ex_e /
// sum).  Empty rows produce nothing.  The sum is accumulated sequentially
// in entry order (lane 0 folds each 32-entry chunk via shuffles), so the
// only difference from the CPU reference can come from exp() itself
// (CUDA's f64 exp vs libm, both within 1 ulp of f64, rounded to f32).
// The max ignores NaN where std::max would latch it; either way a NaN in a
// row makes every ex (or the sum) NaN, so all outputs of that row are NaN
// exactly as in the reference.
#include "ops.hpp"

#include <algorithm>

namespace asb {

namespace {

constexpr unsigned FULL = 0xffffffffu;

__global__ void row_softmax_kernel(const std::uint64_t* __restrict__ rowptr,
                                   const std::uint32_t* __restrict__ order, std::uint64_t n_rows,
                                   const float* __restrict__ vin, float* __restrict__ vout) {
    const int lane = threadIdx.x & 31;
    const std::uint64_t total_warps = std::uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (std::uint64_t w = (std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < n_rows;
         w += total_warps) {
        const std::uint64_t row = order ? order[w] : w;
        const std::uint64_t e0 = rowptr[row], e1 = rowptr[row + 1];
        if (e0 == e1) continue;
        float mx = -INFINITY;
        for (std::uint64_t e = e0 + lane; e < e1; e += 32) mx = fmaxf(mx, vin[e]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, o));
        const double dmx = double(mx);
        double sum = 0.0;  // meaningful in lane 0
        for (std::uint64_t base = e0; base < e1; base += 32) {
            const std::uint64_t e = base + lane;
            double exd = 0.0;
            if (e < e1) {
                const float ex = float(exp(double(vin[e]) - dmx));
                vout[e] = ex;
                exd = double(ex);
            }
            const int n = (e1 - base) < 32 ? int(e1 - base) : 32;
            for (int j = 0; j < n; ++j) {
                const double t = __shfl_sync(FULL, exd, j);
                sum = __dadd_rn(sum, t);
            }
        }
        sum = __shfl_sync(FULL, sum, 0);
        for (std::uint64_t e = e0 + lane; e < e1; e += 32)
            vout[e] = float(__ddiv_rn(double(vout[e]), sum));
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
    const unsigned blocks = unsigned(std::min<std::uint64_t>(want, std::uint64_t(sms) * 16));
    row_softmax_kernel<<<blocks, 256, 0, s>>>(g.rowptr.get(), g.order.get(), g.n_rows, vin, vout);
    check_launch("row_softmax_kernel");
}

} // namespace asb
