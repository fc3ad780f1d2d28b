// attention.cu -- fused CSR attention for sm_100a.
//
// The reference pipeline (src/attention.cpp:9-40) is three passes with two
// CSR copies: scores = sddmm(pattern, q, k); p = row_softmax(scores);
// out = spmm(p, v).  Here one warp owns one row (rows in degree-descending
// order) and runs all three phases back to back:
//   A  scores of 32 entries at a time: the warp stages the 32 gathered K
//      rows and the row's q in shared memory, each lane computes one dot in
//      the chosen SDDMM order (sequential, or the vec f_tile order);
//   B  row max, f32(exp(f64)), sequential f64 sum, p_e = f32(ex/sum) --
//      the row_softmax arithmetic;
//   C  out[i,:] = sum_e p_e * V[col_e,:] in CSR order with f64 accumulators
//      (the row-parallel SpMM arithmetic).
// Scores live in a per-graph nnz scratch that is re-read by the same warp
// immediately (L2-resident), so HBM sees q, K/V gathers, the pattern and
// out once.  Results equal the unfused pipeline bit for bit.
#include "ops.hpp"

#include <algorithm>

namespace asb {

namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ double dfma(float x, float y, double acc) {
    return __fma_rn(double(x), double(y), acc);
}

template <int ORD>
__device__ __forceinline__ double att_dot(const float* xr, const float* yr, std::uint32_t f,
                                          std::uint32_t ft) {
    if constexpr (ORD == 0) {
        double acc = 0.0;
#pragma unroll 4
        for (std::uint32_t t = 0; t < f; t += 4) {
            const float4 x = *reinterpret_cast<const float4*>(xr + t);
            const float4 y = *reinterpret_cast<const float4*>(yr + t);
            acc = dfma(x.x, y.x, acc);
            acc = dfma(x.y, y.y, acc);
            acc = dfma(x.z, y.z, acc);
            acc = dfma(x.w, y.w, acc);
        }
        return acc;
    } else {
        double acc = 0.0;
        for (std::uint32_t b0 = 0; b0 < f; b0 += ft) {
            const std::uint32_t fw = min(ft, f - b0);
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll 2
            for (std::uint32_t t = 0; t < fw; t += 4) {
                const float4 x = *reinterpret_cast<const float4*>(xr + b0 + t);
                const float4 y = *reinterpret_cast<const float4*>(yr + b0 + t);
                a0 = dfma(x.x, y.x, a0);
                a1 = dfma(x.y, y.y, a1);
                a2 = dfma(x.z, y.z, a2);
                a3 = dfma(x.w, y.w, a3);
            }
            acc = __dadd_rn(acc, __dadd_rn(__dadd_rn(a0, a1), __dadd_rn(a2, a3)));  // tail == 0.0
        }
        return acc;
    }
}

// Requires f % 4 == 0 and fv % 4 == 0 with 16-byte aligned q/k/v (the host
// falls back to the unfused pipeline otherwise); ORD 1 also needs ft % 4 == 0
// so every block is a whole number of float4s and the tail sum is +0.0.
template <int ORD, int NCH>
__global__ void __launch_bounds__(256)
    attention_fused_kernel(const std::uint64_t* __restrict__ rowptr,
                           const std::uint32_t* __restrict__ colind,
                           const std::uint32_t* __restrict__ order, std::uint64_t n_rows,
                           const float* __restrict__ q, const float* __restrict__ k,
                           const float* __restrict__ v, float* __restrict__ out,
                           float* __restrict__ scratch, std::uint32_t f, std::uint32_t fv,
                           std::uint32_t S, std::uint32_t ft, std::uint64_t hub_t) {
    extern __shared__ __align__(16) float smem[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    float* ks = smem + std::uint64_t(wib) * 33 * S;
    float* qs = ks + 32 * S;
    const std::uint32_t nv = f / 4;
    const std::uint32_t dj = 32 / nv, dq = 32 % nv;
    const std::uint32_t j_start = std::uint32_t(lane) / nv, q_start = std::uint32_t(lane) % nv;
    const std::uint64_t total_warps = std::uint64_t(gridDim.x) * (blockDim.x >> 5);

    for (std::uint64_t w = std::uint64_t(blockIdx.x) * (blockDim.x >> 5) + wib; w < n_rows;
         w += total_warps) {
        const std::uint64_t row = order[w];
        const std::uint64_t e0 = rowptr[row], e1 = rowptr[row + 1];
        if (e0 == e1) {
            for (std::uint32_t t = lane; t < fv; t += 32) out[row * fv + t] = 0.f;
            continue;
        }
        // q row -> smem
        for (std::uint32_t t = lane; t < nv; t += 32)
            *reinterpret_cast<float4*>(qs + 4 * t) =
                __ldg(reinterpret_cast<const float4*>(q + row * f) + t);
        // ---- A: scores
        float mx = -INFINITY;
        for (std::uint64_t base = e0; base < e1; base += 32) {
            const std::uint64_t e = base + lane;
            const bool valid = e < e1;
            const std::uint32_t c = valid ? colind[e] : 0u;
            __syncwarp();
            std::uint32_t j = j_start, qq = q_start;
            for (std::uint32_t it = 0; it < nv; ++it) {
                const std::uint32_t cj = __shfl_sync(FULL, c, int(j));
                float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
                if (base + j < e1) val = __ldg(reinterpret_cast<const float4*>(k + std::uint64_t(cj) * f) + qq);
                *reinterpret_cast<float4*>(ks + j * S + 4 * qq) = val;
                j += dj;
                qq += dq;
                if (qq >= nv) {
                    qq -= nv;
                    ++j;
                }
            }
            __syncwarp();
            if (valid) {
                const float sc = float(att_dot<ORD>(qs, ks + lane * S, f, ft));
                scratch[e] = sc;
                mx = fmaxf(mx, sc);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, o));
        // ---- B: exp + sequential f64 sum (same lane wrote scratch[e])
        const double dmx = double(mx);
        double sum = 0.0;
        for (std::uint64_t base = e0; base < e1; base += 32) {
            const std::uint64_t e = base + lane;
            double exd = 0.0;
            if (e < e1) {
                const float ex = float(exp(double(scratch[e]) - dmx));
                scratch[e] = ex;
                exd = double(ex);
            }
            const int n = (e1 - base) < 32 ? int(e1 - base) : 32;
            for (int jj = 0; jj < n; ++jj) sum = __dadd_rn(sum, __shfl_sync(FULL, exd, jj));
        }
        sum = __shfl_sync(FULL, sum, 0);
        __syncwarp();
        // ---- C: out row = sum_e p_e * V[col_e] in CSR order
        // HubSplit numerics on heavy rows (src/kernels.cpp:284-332): f64
        // partials per 2048-entry piece, folded into tot in piece order.
        const bool split = hub_t != 0 && (e1 - e0) >= hub_t;
        double acc[NCH][4], tot[NCH][4];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
            for (int t = 0; t < 4; ++t) acc[ch][t] = tot[ch][t] = 0.0;
        bool fok[NCH];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) fok[ch] = std::uint32_t(ch * 32 + lane) * 4 < fv;
        for (std::uint64_t base = e0; base < e1; base += 32) {
            if (split && base > e0 && (base - e0) % 2048 == 0) {
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        tot[ch][t] = __dadd_rn(tot[ch][t], acc[ch][t]);
                        acc[ch][t] = 0.0;
                    }
            }
            const std::uint64_t e = base + lane;
            std::uint32_t c = 0;
            float p = 0.f;
            if (e < e1) {
                c = colind[e];
                p = float(__ddiv_rn(double(scratch[e]), sum));
            }
            const int n = (e1 - base) < 32 ? int(e1 - base) : 32;
            constexpr int U = NCH >= 4 ? 2 : (NCH == 2 ? 4 : 8);
            for (int j0 = 0; j0 < n; j0 += U) {
                std::uint32_t cj[U];
                float pj[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    cj[u] = __shfl_sync(FULL, c, (j0 + u) & 31);
                    pj[u] = __shfl_sync(FULL, p, (j0 + u) & 31);
                }
                float4 bv[U][NCH];
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int ch = 0; ch < NCH; ++ch)
                        if (j0 + u < n && fok[ch])
                            bv[u][ch] = __ldg(reinterpret_cast<const float4*>(v + std::uint64_t(cj[u]) * fv) +
                                              ch * 32 + lane);
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (j0 + u >= n) break;
                    const double dp = double(pj[u]);
#pragma unroll
                    for (int ch = 0; ch < NCH; ++ch) {
                        if (!fok[ch]) continue;
                        acc[ch][0] = __fma_rn(dp, double(bv[u][ch].x), acc[ch][0]);
                        acc[ch][1] = __fma_rn(dp, double(bv[u][ch].y), acc[ch][1]);
                        acc[ch][2] = __fma_rn(dp, double(bv[u][ch].z), acc[ch][2]);
                        acc[ch][3] = __fma_rn(dp, double(bv[u][ch].w), acc[ch][3]);
                    }
                }
            }
        }
        if (split) {
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
                for (int t = 0; t < 4; ++t) acc[ch][t] = __dadd_rn(tot[ch][t], acc[ch][t]);
        }
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
            if (!fok[ch]) continue;
            float* op = out + row * fv + std::uint64_t(ch * 32 + lane) * 4;
            op[0] = float(acc[ch][0]);
            op[1] = float(acc[ch][1]);
            op[2] = float(acc[ch][2]);
            op[3] = float(acc[ch][3]);
        }
    }
}

} // namespace

void launch_attention_fused(Graph& g, const float* q, const float* k, const float* v,
                            std::uint32_t f, std::uint32_t fv, float* out, std::uint64_t sddmm_ft,
                            bool sddmm_vec, std::uint64_t spmm_hub_t, cudaStream_t s) {
    if (g.n_rows == 0) return;
    ensure_order(g);
    g.tmp.ensure(std::max<std::uint64_t>(g.nnz, 1));
    const std::uint32_t ft = std::uint32_t(effective_tile(sddmm_ft, f));
    const std::uint32_t S = 4 * ((f / 4) | 1u);
    const std::uint32_t wpb = 8;
    const std::size_t smem = std::size_t(33) * S * 4 * wpb;
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const std::uint32_t lanes4 = (fv / 4 + 31) / 32;  // float4 chunks per lane
    auto go = [&](auto kernel) {
        ASB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        ASB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, int(wpb * 32), smem));
        const std::uint64_t want = (g.n_rows + wpb - 1) / wpb;
        const std::uint64_t cap = std::uint64_t(sms) * std::max(per_sm, 1) * 4;
        const unsigned blocks = unsigned(std::max<std::uint64_t>(1, std::min(want, cap)));
        kernel<<<blocks, wpb * 32, smem, s>>>(g.rowptr.get(), g.colind.get(), g.order.get(), g.n_rows,
                                              q, k, v, out, g.tmp.get(), f, fv, S, ft, spmm_hub_t);
        check_launch("attention_fused_kernel");
    };
    const bool ord1 = sddmm_vec;
    if (lanes4 <= 1) ord1 ? go(attention_fused_kernel<1, 1>) : go(attention_fused_kernel<0, 1>);
    else if (lanes4 <= 2) ord1 ? go(attention_fused_kernel<1, 2>) : go(attention_fused_kernel<0, 2>);
    else if (lanes4 <= 4) ord1 ? go(attention_fused_kernel<1, 4>) : go(attention_fused_kernel<0, 4>);
    else throw InvalidArgument("attention fused: fv > 512 unsupported (use the unfused path)");
}

} // namespace asb
