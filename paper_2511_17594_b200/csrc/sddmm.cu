// sddmm.cu -- CSR SDDMM kernels for sm_100a: out[e] = <X[i,:], Y[col[e],:]>.
//
// Numerics: one double accumulator per entry in the reference's order.
//   order 0 (baseline and every scalar variant, src/kernels.cpp:343-353 and
//            :120-123): acc += x[t]*y[t] for t = 0..F-1.
//   order 1 (vec variants, src/kernels.cpp:105-119): per f_tile block, four
//            stride-4 partial sums plus a scalar tail, folded into acc as
//            ((a0+a1)+(a2+a3))+tail.
// Products of f32 pairs are exact in f64, so each DFMA equals the
// reference's multiply-then-add.
//
// Mapping: nnz-chunk per warp (32 consecutive entries, one per lane), so
// rows of any degree -- hubs included -- spread over the whole grid; this
// is the GPU form of both RowParallel and HubSplit (whose SDDMM pieces are
// independent, src/kernels.cpp:396-428).  The warp stages the 32 gathered
// Y rows (coalesced, float4 when the vec4 gate passes) and the chunk's X
// rows in shared memory with an odd 16-byte row pitch, so each lane's
// sequential dot reads conflict-free LDS.128.
#include "ops.hpp"

#include <algorithm>

namespace asb {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kXRows = 8;  // X rows staged per chunk; further rows read global

__device__ __forceinline__ double dfma(float x, float y, double acc) {
    return __fma_rn(double(x), double(y), acc);
}

// Sequential dot over [0, f): VLDS uses 16-byte reads (f % 4 == 0, both
// pointers 16-byte aligned).
template <bool VLDS>
__device__ __forceinline__ double dot_seq(const float* xr, const float* yr, std::uint32_t f) {
    double acc = 0.0;
    if constexpr (VLDS) {
#pragma unroll 4
        for (std::uint32_t t = 0; t < f; t += 4) {
            const float4 x = *reinterpret_cast<const float4*>(xr + t);
            const float4 y = *reinterpret_cast<const float4*>(yr + t);
            acc = dfma(x.x, y.x, acc);
            acc = dfma(x.y, y.y, acc);
            acc = dfma(x.z, y.z, acc);
            acc = dfma(x.w, y.w, acc);
        }
    } else {
#pragma unroll 4
        for (std::uint32_t t = 0; t < f; ++t) acc = dfma(xr[t], yr[t], acc);
    }
    return acc;
}

// src/kernels.cpp:103-127 vec path.  VLDS requires ft % 4 == 0 too.
template <bool VLDS>
__device__ __forceinline__ double dot_vec4blk(const float* xr, const float* yr, std::uint32_t f,
                                              std::uint32_t ft) {
    double acc = 0.0;
    for (std::uint32_t b0 = 0; b0 < f; b0 += ft) {
        const std::uint32_t fw = min(ft, f - b0);
        const std::uint32_t fw4 = fw & ~3u;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        std::uint32_t t = 0;
#pragma unroll 2
        for (; t < fw4; t += 4) {
            float4 x, y;
            if constexpr (VLDS) {
                x = *reinterpret_cast<const float4*>(xr + b0 + t);
                y = *reinterpret_cast<const float4*>(yr + b0 + t);
            } else {
                x = make_float4(xr[b0 + t], xr[b0 + t + 1], xr[b0 + t + 2], xr[b0 + t + 3]);
                y = make_float4(yr[b0 + t], yr[b0 + t + 1], yr[b0 + t + 2], yr[b0 + t + 3]);
            }
            a0 = dfma(x.x, y.x, a0);
            a1 = dfma(x.y, y.y, a1);
            a2 = dfma(x.z, y.z, a2);
            a3 = dfma(x.w, y.w, a3);
        }
        double tail = 0.0;
        for (; t < fw; ++t) tail = dfma(xr[b0 + t], yr[b0 + t], tail);
        acc = __dadd_rn(acc, __dadd_rn(__dadd_rn(__dadd_rn(a0, a1), __dadd_rn(a2, a3)), tail));
    }
    return acc;
}

template <int ORD, bool VLDS>
__device__ __forceinline__ double dot_ord(const float* xr, const float* yr, std::uint32_t f,
                                          std::uint32_t ft) {
    if constexpr (ORD == 0) return dot_seq<VLDS>(xr, yr, f);
    else return dot_vec4blk<VLDS>(xr, yr, f, ft);
}

// Row of entry e, starting from the chunk's first row (chunk_row map).
__device__ __forceinline__ std::uint32_t row_of(const std::uint64_t* __restrict__ rowptr,
                                                std::uint32_t r, std::uint64_t e) {
    while (rowptr[r + 1] <= e) ++r;
    return r;
}

// VLOAD: 16-byte global gathers (vec4 gate passed).  S: smem row pitch in
// floats (multiple of 4 when VLOAD).
template <bool VLOAD, int ORD, bool VLDS>
__global__ void __launch_bounds__(512)
    sddmm_chunk_kernel(const std::uint64_t* __restrict__ rowptr,
                       const std::uint32_t* __restrict__ colind,
                       const std::uint32_t* __restrict__ chunk_row, const float* __restrict__ x,
                       const float* __restrict__ y, float* __restrict__ out, std::uint64_t nnz,
                       std::uint32_t f, std::uint32_t S, std::uint32_t ft) {
    extern __shared__ __align__(16) float smem[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    float* ys = smem + std::uint64_t(wib) * (32 + kXRows) * S;
    float* xs = ys + 32 * S;
    const std::uint64_t n_chunks = (nnz + 31) / 32;
    const std::uint64_t total_warps = std::uint64_t(gridDim.x) * (blockDim.x >> 5);
    // element walk over a (rows x nv) tile: 32 = dj*nv + dq
    const std::uint32_t nv = VLOAD ? f / 4 : f;
    const std::uint32_t dj = 32 / nv, dq = 32 % nv;
    const std::uint32_t j_start = std::uint32_t(lane) / nv, q_start = std::uint32_t(lane) % nv;

    for (std::uint64_t ch = std::uint64_t(blockIdx.x) * (blockDim.x >> 5) + wib; ch < n_chunks;
         ch += total_warps) {
        const std::uint64_t e0 = ch * 32;
        const std::uint64_t e = e0 + lane;
        const bool valid = e < nnz;
        const std::uint32_t r_first = chunk_row[ch];
        const std::uint32_t r = valid ? row_of(rowptr, r_first, e) : r_first;
        const std::uint32_t c = valid ? colind[e] : 0u;
        const std::uint32_t r_last = __reduce_max_sync(FULL, r);
        const std::uint32_t nx = min(r_last - r_first + 1, std::uint32_t(kXRows));

        // stage 32 Y rows
        {
            std::uint32_t j = j_start, q = q_start;
            for (std::uint32_t it = 0; it < nv; ++it) {
                const std::uint32_t cj = __shfl_sync(FULL, c, int(j));
                const bool ok = e0 + j < nnz;
                if constexpr (VLOAD) {
                    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (ok) v = __ldg(reinterpret_cast<const float4*>(y + std::uint64_t(cj) * f) + q);
                    *reinterpret_cast<float4*>(ys + j * S + 4 * q) = v;
                } else {
                    ys[j * S + q] = ok ? __ldg(y + std::uint64_t(cj) * f + q) : 0.f;
                }
                j += dj;
                q += dq;
                if (q >= nv) {
                    q -= nv;
                    ++j;
                }
            }
        }
        // stage up to kXRows X rows
        {
            const std::uint32_t total = nx * nv;
            std::uint32_t j = j_start, q = q_start;
            for (std::uint32_t idx = std::uint32_t(lane); idx < total; idx += 32) {
                const float* xsrc = x + std::uint64_t(r_first + j) * f;
                if constexpr (VLOAD) {
                    *reinterpret_cast<float4*>(xs + j * S + 4 * q) =
                        __ldg(reinterpret_cast<const float4*>(xsrc) + q);
                } else {
                    xs[j * S + q] = __ldg(xsrc + q);
                }
                j += dj;
                q += dq;
                if (q >= nv) {
                    q -= nv;
                    ++j;
                }
            }
        }
        __syncwarp();
        if (valid) {
            const float* yr = ys + lane * S;
            double acc;
            if (r - r_first < nx) acc = dot_ord<ORD, VLDS>(xs + (r - r_first) * S, yr, f, ft);
            else acc = dot_ord<ORD, false>(x + std::uint64_t(r) * f, yr, f, ft);
            out[e] = float(acc);
        }
        __syncwarp();
    }
}

// Guardrail baseline / large-F fallback: lane per entry, both rows read
// straight from global memory, scalar loads.
template <int ORD>
__global__ void sddmm_direct_kernel(const std::uint64_t* __restrict__ rowptr,
                                    const std::uint32_t* __restrict__ colind,
                                    const std::uint32_t* __restrict__ chunk_row,
                                    const float* __restrict__ x, const float* __restrict__ y,
                                    float* __restrict__ out, std::uint64_t nnz, std::uint32_t f,
                                    std::uint32_t ft) {
    const std::uint64_t ch = (std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const std::uint64_t e = ch * 32 + (threadIdx.x & 31);
    if (e >= nnz) return;
    const std::uint32_t r = row_of(rowptr, chunk_row[ch], e);
    const float* xr = x + std::uint64_t(r) * f;
    const float* yr = y + std::uint64_t(colind[e]) * f;
    out[e] = float(dot_ord<ORD, false>(xr, yr, f, ft));
}

} // namespace

void launch_sddmm_baseline(Graph& g, const float* x, const float* y, std::uint32_t f, float* out,
                           cudaStream_t s) {
    if (g.nnz == 0) return;
    ensure_chunk_rows(g);
    const std::uint64_t n_chunks = (g.nnz + 31) / 32;
    const unsigned blocks = unsigned((n_chunks * 32 + 255) / 256);
    sddmm_direct_kernel<0><<<blocks, 256, 0, s>>>(g.rowptr.get(), g.colind.get(), g.chunk_row.get(),
                                                  x, y, out, g.nnz, f, f ? f : 1);
    check_launch("sddmm_direct_kernel");
}

void launch_sddmm_chunks(Graph& g, const float* x, const float* y, std::uint32_t f, float* out,
                         std::uint64_t f_tile, bool vec, std::uint32_t wpb, cudaStream_t s) {
    if (g.nnz == 0) return;
    ensure_chunk_rows(g);
    const std::uint32_t ft = std::uint32_t(effective_tile(f_tile, f));
    const int ord = vec ? 1 : 0;
    const std::uint64_t n_chunks = (g.nnz + 31) / 32;
    if (f == 0) {
        // empty dot products: the reference writes 0.0f for every entry
        ASB_CUDA(cudaMemsetAsync(out, 0, g.nnz * 4, s));
        return;
    }
    const bool vload = vec;  // vec4 gate already applied by dispatch
    const bool vlds = vload && (ord == 0 || ft % 4 == 0);
    std::uint32_t S = vload ? 4 * ((f / 4) | 1u) : (f | 1u);
    const std::uint64_t per_warp = std::uint64_t(32 + kXRows) * S * 4;
    constexpr std::uint64_t kSmemMax = 200 * 1024;
    wpb = std::clamp<std::uint32_t>(wpb, 1, 16);
    while (wpb > 1 && per_warp * wpb > kSmemMax) --wpb;
    if (per_warp > kSmemMax) {
        const unsigned blocks = unsigned((n_chunks * 32 + 255) / 256);
        if (ord == 0)
            sddmm_direct_kernel<0><<<blocks, 256, 0, s>>>(g.rowptr.get(), g.colind.get(),
                                                          g.chunk_row.get(), x, y, out, g.nnz, f, ft);
        else
            sddmm_direct_kernel<1><<<blocks, 256, 0, s>>>(g.rowptr.get(), g.colind.get(),
                                                          g.chunk_row.get(), x, y, out, g.nnz, f, ft);
        check_launch("sddmm_direct_kernel");
        return;
    }
    const std::size_t smem = std::size_t(per_warp * wpb);
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);

    auto go = [&](auto kernel) {
        ASB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        ASB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, int(wpb * 32), smem));
        const std::uint64_t want = (n_chunks + wpb - 1) / wpb;
        const std::uint64_t cap = std::uint64_t(sms) * std::max(per_sm, 1) * 4;
        const unsigned blocks = unsigned(std::max<std::uint64_t>(1, std::min(want, cap)));
        kernel<<<blocks, wpb * 32, smem, s>>>(g.rowptr.get(), g.colind.get(), g.chunk_row.get(), x, y,
                                              out, g.nnz, f, S, ft);
        check_launch("sddmm_chunk_kernel");
    };
    if (vload) {
        if (ord == 0) go(sddmm_chunk_kernel<true, 0, true>);
        else if (vlds) go(sddmm_chunk_kernel<true, 1, true>);
        else go(sddmm_chunk_kernel<true, 1, false>);
    } else {
        if (ord == 0) go(sddmm_chunk_kernel<false, 0, false>);
        else go(sddmm_chunk_kernel<false, 1, false>);
    }
}

} // namespace asb
