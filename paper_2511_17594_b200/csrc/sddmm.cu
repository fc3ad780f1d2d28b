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
#include "widen.cuh"

#include <algorithm>
#include <cstdlib>

namespace asb {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kXRows = 8;  // X rows staged per chunk; further rows read global

__device__ __forceinline__ double dfma(double x, float y, double acc) {
    return __fma_rn(x, double(y), acc);
}

// widen y by re-bias (ALU pipe) when MIX; x carries the 2^896 (widen.cuh)
template <int MIX>
__device__ __forceinline__ double dfma_r(double x, float y, double acc) {
    if constexpr (MIX) return __fma_rn(x * kWidenUp, widen_scaled(y), acc);
    else return __fma_rn(x, double(y), acc);
}

// x components: f32 from global memory, or f64 pre-widened in shared memory
struct X4 {
    double a, b, c, d;
};
__device__ __forceinline__ X4 load_x4(const float* p) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    return {double(v.x), double(v.y), double(v.z), double(v.w)};
}
__device__ __forceinline__ X4 load_x4(const double* p) {
    const double2 lo = *reinterpret_cast<const double2*>(p);
    const double2 hi = *reinterpret_cast<const double2*>(p + 2);
    return {lo.x, lo.y, hi.x, hi.y};
}
__device__ __forceinline__ double x_at(const float* p, std::uint32_t t) { return double(p[t]); }
__device__ __forceinline__ double x_at(const double* p, std::uint32_t t) { return p[t]; }

// Sequential dot over [0, f): VLDS uses 16-byte reads (f % 4 == 0, both
// pointers 16-byte aligned).
template <bool VLDS, int MIX, class XT>
__device__ __forceinline__ double dot_seq(const XT* xr, const float* yr, std::uint32_t f) {
    double acc = 0.0;
    if constexpr (VLDS) {
#pragma unroll 4
        for (std::uint32_t t = 0; t < f; t += 4) {
            const X4 x = load_x4(xr + t);
            const float4 y = *reinterpret_cast<const float4*>(yr + t);
            acc = dfma(x.a, y.x, acc);
            acc = dfma(x.b, y.y, acc);
            acc = dfma_r<MIX>(x.c, y.z, acc);
            acc = dfma_r<MIX>(x.d, y.w, acc);
        }
    } else {
#pragma unroll 4
        for (std::uint32_t t = 0; t < f; ++t) acc = dfma(x_at(xr, t), yr[t], acc);
    }
    return acc;
}

// src/kernels.cpp:103-127 vec path.  VLDS requires ft % 4 == 0 too.
template <bool VLDS, int MIX, class XT>
__device__ __forceinline__ double dot_vec4blk(const XT* xr, const float* yr, std::uint32_t f,
                                              std::uint32_t ft) {
    double acc = 0.0;
    for (std::uint32_t b0 = 0; b0 < f; b0 += ft) {
        const std::uint32_t fw = min(ft, f - b0);
        const std::uint32_t fw4 = fw & ~3u;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        std::uint32_t t = 0;
#pragma unroll 2
        for (; t < fw4; t += 4) {
            X4 x;
            float4 y;
            if constexpr (VLDS) {
                x = load_x4(xr + b0 + t);
                y = *reinterpret_cast<const float4*>(yr + b0 + t);
            } else {
                x = {x_at(xr, b0 + t), x_at(xr, b0 + t + 1), x_at(xr, b0 + t + 2), x_at(xr, b0 + t + 3)};
                y = make_float4(yr[b0 + t], yr[b0 + t + 1], yr[b0 + t + 2], yr[b0 + t + 3]);
            }
            a0 = dfma(x.a, y.x, a0);
            a1 = dfma(x.b, y.y, a1);
            a2 = dfma_r<MIX>(x.c, y.z, a2);
            a3 = dfma_r<MIX>(x.d, y.w, a3);
        }
        double tail = 0.0;
        for (; t < fw; ++t) tail = dfma(x_at(xr, b0 + t), yr[b0 + t], tail);
        acc = __dadd_rn(acc, __dadd_rn(__dadd_rn(__dadd_rn(a0, a1), __dadd_rn(a2, a3)), tail));
    }
    return acc;
}

template <int ORD, bool VLDS, int MIX, class XT>
__device__ __forceinline__ double dot_ord(const XT* xr, const float* yr, std::uint32_t f,
                                          std::uint32_t ft) {
    if constexpr (ORD == 0) return dot_seq<VLDS, MIX>(xr, yr, f);
    else return dot_vec4blk<VLDS, MIX>(xr, yr, f, ft);
}

// Row of entry e, starting from the chunk's first row (chunk_row map).
__device__ __forceinline__ std::uint32_t row_of(const std::uint64_t* __restrict__ rowptr,
                                                std::uint32_t r, std::uint64_t e) {
    while (rowptr[r + 1] <= e) ++r;
    return r;
}

// VLOAD: 16-byte global gathers (vec4 gate passed).  S: smem row pitch in
// floats (multiple of 4 when VLOAD).
template <bool VLOAD, int ORD, bool VLDS, int MIX>
__device__ __forceinline__ void sddmm_chunk_body(
    const std::uint64_t* __restrict__ rowptr, const std::uint32_t* __restrict__ colind,
    const std::uint32_t* __restrict__ chunk_row, const float* __restrict__ x,
    const float* __restrict__ y, float* __restrict__ out, std::uint64_t nnz, std::uint32_t f,
    std::uint32_t S, std::uint32_t ft, float* smem) {
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    // per warp: 32 Y rows (f32, pitch S) then kXRows X rows widened to f64
    float* ys = reinterpret_cast<float*>(reinterpret_cast<char*>(smem) +
                                         std::uint64_t(wib) * (32ull * S * 4 + kXRows * 8ull * f));
    double* xs = reinterpret_cast<double*>(ys + 32 * S);
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
        // stage up to kXRows X rows, widened to f64 once per chunk (not once
        // per product): rows r_first.. are contiguous in X
        {
            const float* xsrc = x + std::uint64_t(r_first) * f;
            const std::uint32_t total = nx * f;
            for (std::uint32_t idx = std::uint32_t(lane); idx < total; idx += 32)
                xs[idx] = double(__ldg(xsrc + idx));
        }
        __syncwarp();
        if (valid) {
            const float* yr = ys + lane * S;
            double acc;
            if (r - r_first < nx) acc = dot_ord<ORD, VLDS, MIX>(xs + std::uint64_t(r - r_first) * f, yr, f, ft);
            else acc = dot_ord<ORD, false, 0>(x + std::uint64_t(r) * f, yr, f, ft);
            out[e] = float(acc);
        }
        __syncwarp();
    }
}

// MIX (re-bias half of the Y widening on the ALU pipe) only when the
// device-side scan found Y finite and the float4 smem path is in use.
template <bool VLOAD, int ORD, bool VLDS>
__global__ void __launch_bounds__(512)
    sddmm_chunk_kernel(const std::uint64_t* __restrict__ rowptr,
                       const std::uint32_t* __restrict__ colind,
                       const std::uint32_t* __restrict__ chunk_row, const float* __restrict__ x,
                       const float* __restrict__ y, float* __restrict__ out, std::uint64_t nnz,
                       std::uint32_t f, std::uint32_t S, std::uint32_t ft,
                       const unsigned* __restrict__ finite) {
    extern __shared__ __align__(16) float smem[];
    if (VLDS && finite && *finite)
        sddmm_chunk_body<VLOAD, ORD, VLDS, 1>(rowptr, colind, chunk_row, x, y, out, nnz, f, S, ft, smem);
    else
        sddmm_chunk_body<VLOAD, ORD, VLDS, 0>(rowptr, colind, chunk_row, x, y, out, nnz, f, S, ft, smem);
}

// ---------------------------------------------------------------------------
// TMA-staged chunk kernel (vec4-eligible operands): per warp, two staging
// buffers; each lane issues ONE bulk copy (cp.async.bulk, complete_tx on the
// buffer's mbarrier) for its entry's Y row, lanes < nx copy the chunk's X
// rows.  The next chunk's copies are in flight while the current chunk's
// dots run; chunk metadata (colind, chunk_row) is prefetched one chunk ahead
// in registers, so the warp never stalls on a dependent load before issuing.
constexpr int kTX = 4;  // X rows staged per chunk

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return unsigned(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(std::uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(std::uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "SDDMM_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra SDDMM_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, std::uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

struct TmaLayout {
    std::uint32_t ybuf, xbuf, xd, bar, per_warp;  // byte offsets within a warp's slice
};
__host__ __device__ inline TmaLayout tma_layout(std::uint32_t f, std::uint32_t S) {
    TmaLayout L{};
    std::uint32_t o = 0;
    L.ybuf = o;
    o += 2u * 32u * S * 4u;  // 2 buffers x 32 Y rows (pitch S floats)
    L.xbuf = o;
    o += 2u * kTX * f * 4u;  // 2 buffers x kTX X rows (f32)
    o = (o + 15) & ~15u;
    L.xd = o;
    o += kTX * (f + 2) * 8u;  // widened X rows, padded pitch
    o = (o + 15) & ~15u;
    L.bar = o;
    o += 16;
    L.per_warp = (o + 127) & ~127u;
    return L;
}

template <int ORD, int MIX>
__device__ __forceinline__ void sddmm_tma_body(const std::uint64_t* __restrict__ rowptr,
                                               const std::uint32_t* __restrict__ colind,
                                               const std::uint32_t* __restrict__ chunk_row,
                                               std::uint64_t n_rows, const float* __restrict__ x,
                                               const float* __restrict__ y, float* __restrict__ out,
                                               std::uint64_t nnz, std::uint32_t f, std::uint32_t S,
                                               std::uint32_t ft, char* wsm) {
    const TmaLayout L = tma_layout(f, S);
    float* ybuf = reinterpret_cast<float*>(wsm + L.ybuf);
    float* xbuf = reinterpret_cast<float*>(wsm + L.xbuf);
    double* xd = reinterpret_cast<double*>(wsm + L.xd);
    std::uint64_t* bar = reinterpret_cast<std::uint64_t*>(wsm + L.bar);
    const int lane = threadIdx.x & 31;
    const std::uint32_t xpitch = f + 2;
    const unsigned row_bytes = f * 4;
    const std::uint64_t n_chunks = (nnz + 31) / 32;
    const std::uint64_t stride = std::uint64_t(gridDim.x) * (blockDim.x >> 5);
    const std::uint64_t c0 = std::uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);

    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();

    struct Meta {
        std::uint32_t col, r_first, nx;
        bool valid;
    };
    auto load_meta = [&](std::uint64_t c) {
        Meta m{0, 0, 0, false};
        if (c >= n_chunks) return m;
        const std::uint64_t e = c * 32 + lane;
        m.valid = e < nnz;
        m.col = m.valid ? __ldg(colind + e) : 0u;
        m.r_first = __ldg(chunk_row + c);
        const std::uint32_t r_bound =
            c + 1 < n_chunks ? __ldg(chunk_row + c + 1) : std::uint32_t(n_rows - 1);
        m.nx = min(r_bound - m.r_first + 1, std::uint32_t(kTX));
        return m;
    };
    auto issue = [&](std::uint64_t c, const Meta& m, int b) {
        const unsigned nvalid = nnz - c * 32 < 32 ? unsigned(nnz - c * 32) : 32u;
        if (lane == 0) mbar_arrive_expect_tx(&bar[b], (nvalid + m.nx) * row_bytes);
        __syncwarp();
        if (m.valid)
            bulk_g2s(ybuf + std::uint64_t(b) * 32 * S + std::uint64_t(lane) * S,
                     y + std::uint64_t(m.col) * f, row_bytes, &bar[b]);
        if (std::uint32_t(lane) < m.nx)
            bulk_g2s(xbuf + (std::uint64_t(b) * kTX + lane) * f, x + std::uint64_t(m.r_first + lane) * f,
                     row_bytes, &bar[b]);
    };

    unsigned phase[2] = {0u, 0u};
    Meta cur = load_meta(c0);
    if (c0 < n_chunks) issue(c0, cur, 0);
    Meta nxt = load_meta(c0 + stride);
    int b = 0;
    for (std::uint64_t c = c0; c < n_chunks; c += stride, b ^= 1) {
        const std::uint64_t cn = c + stride;
        if (cn < n_chunks) issue(cn, nxt, b ^ 1);
        const Meta m = cur;
        cur = nxt;
        nxt = load_meta(cn + stride);  // in flight during this chunk's dots
        mbar_wait(&bar[b], phase[b]);
        phase[b] ^= 1u;
        // widen this chunk's X rows once
        const float* xs = xbuf + std::uint64_t(b) * kTX * f;
        for (std::uint32_t idx = lane; idx < m.nx * f; idx += 32) {
            const std::uint32_t rr = idx / f, t = idx - rr * f;
            xd[rr * xpitch + t] = double(xs[idx]);
        }
        __syncwarp();
        const std::uint64_t e = c * 32 + lane;
        if (m.valid) {
            const std::uint32_t r = row_of(rowptr, m.r_first, e);
            const float* yr = ybuf + std::uint64_t(b) * 32 * S + std::uint64_t(lane) * S;
            double acc;
            if (r - m.r_first < m.nx) acc = dot_ord<ORD, true, MIX>(xd + (r - m.r_first) * xpitch, yr, f, ft);
            else acc = dot_ord<ORD, false, 0>(x + std::uint64_t(r) * f, yr, f, ft);
            out[e] = float(acc);
        }
        __syncwarp();  // buffer b and xd free before they are refilled
    }
}

template <int ORD>
__global__ void __launch_bounds__(512)
    sddmm_tma_kernel(const std::uint64_t* __restrict__ rowptr,
                     const std::uint32_t* __restrict__ colind,
                     const std::uint32_t* __restrict__ chunk_row, std::uint64_t n_rows,
                     const float* __restrict__ x, const float* __restrict__ y,
                     float* __restrict__ out, std::uint64_t nnz, std::uint32_t f, std::uint32_t S,
                     std::uint32_t ft, const unsigned* __restrict__ finite) {
    extern __shared__ __align__(128) char tsmem[];
    char* wsm = tsmem + std::uint64_t(threadIdx.x >> 5) * tma_layout(f, S).per_warp;
    if (finite && *finite)
        sddmm_tma_body<ORD, 1>(rowptr, colind, chunk_row, n_rows, x, y, out, nnz, f, S, ft, wsm);
    else
        sddmm_tma_body<ORD, 0>(rowptr, colind, chunk_row, n_rows, x, y, out, nnz, f, S, ft, wsm);
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
    out[e] = float(dot_ord<ORD, false, 0>(xr, yr, f, ft));
}

bool tma_path_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("AUTOSAGE_DEV_SDDMM_TMA");
        return !(e && e[0] == '0');
    }();
    return on;
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
                         std::uint64_t f_tile, bool vec, std::uint32_t wpb, cudaStream_t s,
                         const unsigned* finite) {
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
    int dev0 = 0, sms0 = 148;
    cudaGetDevice(&dev0);
    cudaDeviceGetAttribute(&sms0, cudaDevAttrMultiProcessorCount, dev0);
    if (vlds && tma_path_enabled()) {
        const std::uint32_t per_warp = tma_layout(f, S).per_warp;
        std::uint32_t w = std::clamp<std::uint32_t>(wpb, 1, 16);
        while (w > 1 && std::uint64_t(per_warp) * w > 200 * 1024) --w;
        if (per_warp <= 200 * 1024) {
            const std::size_t smem = std::size_t(per_warp) * w;
            auto kern = ord == 0 ? sddmm_tma_kernel<0> : sddmm_tma_kernel<1>;
            int per_sm = 1;
            ASB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            ASB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, int(w * 32), smem));
            const std::uint64_t want = (n_chunks + w - 1) / w;
            const std::uint64_t cap = std::uint64_t(sms0) * std::max(per_sm, 1);
            const unsigned blocks = unsigned(std::max<std::uint64_t>(1, std::min(want, cap)));
            kern<<<blocks, w * 32, smem, s>>>(g.rowptr.get(), g.colind.get(), g.chunk_row.get(), g.n_rows,
                                              x, y, out, g.nnz, f, S, ft, finite);
            check_launch("sddmm_tma_kernel");
            return;
        }
    }
    const std::uint64_t per_warp = 32ull * S * 4 + kXRows * 8ull * f;
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
                                              out, g.nnz, f, S, ft, finite);
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
