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
// independent, src/kernels.cpp:396-428).  Each lane's dot is a sequential
// chain, so the 32 gathered Y rows are transposed through shared memory:
// the warp stages them with cp.async (all copies in flight at once, no
// register round trip), together with the chunk's X rows, while it
// resolves the next chunk's column indices and rows; X is widened to f64
// once per chunk, and half of every Y float4 is widened on the ALU pipe
// (widen.cuh) when Y is finite.  Row pitch: an odd number of 16-byte units,
// so each lane's LDS.128 walk along its own row is conflict-free.
#include "ops.hpp"
#include "dcheck.cuh"
#include "half.cuh"
#include "l2hint.cuh"
#include "widen.cuh"

#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace asb {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kXRows = 4;  // X rows staged per chunk; further rows read global

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
__device__ __forceinline__ X4 load_x4(const double* p) {
    const double2 lo = *reinterpret_cast<const double2*>(p);
    const double2 hi = *reinterpret_cast<const double2*>(p + 2);
    return {lo.x, lo.y, hi.x, hi.y};
}
__device__ __forceinline__ double x_at(const float* p, std::uint32_t t) { return double(p[t]); }
__device__ __forceinline__ double x_at(const double* p, std::uint32_t t) { return p[t]; }
// bf16 operands (raw 16-bit words): bf16 -> f32 is exact, so every product
// is the f32 path's on float(X), float(Y)
__device__ __forceinline__ float bf16f(unsigned short h) { return half_to_f32<kWtBF16>(h); }
__device__ __forceinline__ double x_at(const unsigned short* p, std::uint32_t t) { return double(bf16f(p[t])); }
__device__ __forceinline__ float y_at(const float* p, std::uint32_t t) { return p[t]; }
__device__ __forceinline__ float y_at(const unsigned short* p, std::uint32_t t) { return bf16f(p[t]); }
// IEEE half words as their own element type, so the generic dot loops pick
// the f16 conversion by overload
struct f16w {
    unsigned short v;
};
__device__ __forceinline__ double x_at(const f16w* p, std::uint32_t t) { return double(half_to_f32<kWtF16>(p[t].v)); }
__device__ __forceinline__ float y_at(const f16w* p, std::uint32_t t) { return half_to_f32<kWtF16>(p[t].v); }

// Sequential dot over [0, f): VLDS uses 16-byte reads (f % 4 == 0, both
// pointers 16-byte aligned).
template <bool VLDS, int MIX, class XT, class YT>
__device__ __forceinline__ double dot_seq(const XT* xr, const YT* yr, std::uint32_t f) {
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
        for (std::uint32_t t = 0; t < f; ++t) acc = dfma(x_at(xr, t), y_at(yr, t), acc);
    }
    return acc;
}

// src/kernels.cpp:103-127 vec path.  VLDS requires ft % 4 == 0 too.
template <bool VLDS, int MIX, class XT, class YT>
__device__ __forceinline__ double dot_vec4blk(const XT* xr, const YT* yr, std::uint32_t f,
                                              std::uint32_t ft) {
    double acc = 0.0;
    for (std::uint32_t b0 = 0; b0 < f; b0 += ft) {
        const std::uint32_t fw = min(ft, f - b0);
        const std::uint32_t fw4 = fw & ~3u;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        std::uint32_t t = 0;
#pragma unroll 4
        for (; t < fw4; t += 4) {
            X4 x;
            float4 y;
            if constexpr (VLDS) {
                x = load_x4(xr + b0 + t);
                y = *reinterpret_cast<const float4*>(yr + b0 + t);
            } else {
                x = {x_at(xr, b0 + t), x_at(xr, b0 + t + 1), x_at(xr, b0 + t + 2), x_at(xr, b0 + t + 3)};
                y = make_float4(y_at(yr, b0 + t), y_at(yr, b0 + t + 1), y_at(yr, b0 + t + 2),
                                y_at(yr, b0 + t + 3));
            }
            a0 = dfma(x.a, y.x, a0);
            a1 = dfma(x.b, y.y, a1);
            a2 = dfma_r<MIX>(x.c, y.z, a2);
            a3 = dfma_r<MIX>(x.d, y.w, a3);
        }
        double tail = 0.0;
        for (; t < fw; ++t) tail = dfma(x_at(xr, b0 + t), y_at(yr, b0 + t), tail);
        acc = __dadd_rn(acc, __dadd_rn(__dadd_rn(__dadd_rn(a0, a1), __dadd_rn(a2, a3)), tail));
    }
    return acc;
}

template <int ORD, bool VLDS, int MIX, class XT, class YT>
__device__ __forceinline__ double dot_ord(const XT* xr, const YT* yr, std::uint32_t f,
                                          std::uint32_t ft) {
    if constexpr (ORD == 0) return dot_seq<VLDS, MIX>(xr, yr, f);
    else return dot_vec4blk<VLDS, MIX>(xr, yr, f, ft);
}

// Row of entry e, starting from the chunk's first row (chunk_row map).
__device__ __forceinline__ std::uint32_t row_of(const std::uint64_t* __restrict__ rowptr,
                                                std::uint32_t r, std::uint64_t e) {
    while (__ldg(rowptr + r + 1) <= e) ++r;
    return r;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = unsigned(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const unsigned s = unsigned(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}

// Per-warp shared-memory slice of the generic chunk kernel: {32 Y rows (f32,
// pitch S), kXRows X rows (f32, pitch f)}, then the X rows widened to f64
// (pitch f+2).
__host__ __device__ inline std::uint64_t stage_bytes(std::uint32_t f, std::uint32_t S) {
    return (32ull * S * 4 + std::uint64_t(kXRows) * f * 4 + 15) / 16 * 16;
}
__host__ __device__ inline std::uint64_t warp_slice_bytes(std::uint32_t f, std::uint32_t S) {
    const std::uint64_t xd = std::uint64_t(kXRows) * (f + 2) * 8;
    return stage_bytes(f, S) + ((xd + 15) / 16 * 16);
}

int dev_knob(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

struct ChunkMeta {
    std::uint32_t col, r_first, r, nx;
    bool valid;
};

// Generic widths (any F): VLOAD = 16-byte copies (vec4 gate passed); S =
// smem row pitch in floats (multiple of 4 when VLOAD).  One staging buffer
// per warp: a second one (copies of the next chunk overlapping this chunk's
// dots) halved the resident warps and measured slower.
template <bool VLOAD, int ORD, bool VLDS, int MIX>
__device__ __forceinline__ void sddmm_chunk_body(
    const std::uint64_t* __restrict__ rowptr, const std::uint32_t* __restrict__ colind,
    const std::uint32_t* __restrict__ chunk_row, std::uint64_t n_rows, const float* __restrict__ x,
    const float* __restrict__ y, float* __restrict__ out, std::uint64_t nnz, std::uint64_t c_begin,
    std::uint64_t c_end, std::uint32_t f, std::uint32_t S, std::uint32_t ft, char* wsm) {
    const int lane = threadIdx.x & 31;
    const std::uint64_t sbytes = stage_bytes(f, S);
    double* xd = reinterpret_cast<double*>(wsm + sbytes);
    const std::uint32_t xpitch = f + 2;
    const std::uint64_t n_chunks = (nnz + 31) / 32;
    const std::uint64_t stride = std::uint64_t(gridDim.x) * (blockDim.x >> 5);
    // element walk over a (rows x nv) tile: 32 = dj*nv + dq
    const std::uint32_t nv = VLOAD ? f / 4 : f;
    const std::uint32_t dj = 32 / nv, dq = 32 % nv;
    const std::uint32_t j_start = std::uint32_t(lane) / nv, q_start = std::uint32_t(lane) % nv;

    auto meta = [&](std::uint64_t c) {
        ChunkMeta m{0, 0, 0, 0, false};
        if (c >= c_end) return m;
        const std::uint64_t e = c * 32 + lane;
        m.valid = e < nnz;
        m.col = m.valid ? __ldg(colind + e) : 0u;
        m.r_first = __ldg(chunk_row + c);
        const std::uint32_t r_bound = c + 1 < n_chunks ? __ldg(chunk_row + c + 1) : std::uint32_t(n_rows - 1);
        m.nx = min(r_bound - m.r_first + 1, std::uint32_t(kXRows));
        m.r = m.valid ? row_of(rowptr, m.r_first, e) : m.r_first;
        return m;
    };
    // async copies of chunk c's 32 Y rows and X rows
    auto issue = [&](const ChunkMeta& m, std::uint64_t c) {
        float* ys = reinterpret_cast<float*>(wsm);
        float* xs = ys + 32 * S;
        const std::uint64_t e0 = c * 32;
        std::uint32_t j = j_start, q = q_start;
        for (std::uint32_t it = 0; it < nv; ++it) {
            const std::uint32_t cj = __shfl_sync(FULL, m.col, int(j));
            if (e0 + j < nnz) {
                if constexpr (VLOAD) cp_async16(ys + j * S + 4 * q, y + std::uint64_t(cj) * f + 4 * q);
                else cp_async4(ys + j * S + q, y + std::uint64_t(cj) * f + q);
            }
            j += dj;
            q += dq;
            if (q >= nv) {
                q -= nv;
                ++j;
            }
        }
        const float* xsrc = x + std::uint64_t(m.r_first) * f;
        const std::uint32_t xn = m.nx * nv;
        for (std::uint32_t idx = std::uint32_t(lane); idx < xn; idx += 32) {
            if constexpr (VLOAD) cp_async16(xs + 4 * idx, xsrc + 4 * idx);
            else cp_async4(xs + idx, xsrc + idx);
        }
    };

    std::uint64_t c = c_begin + std::uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    ChunkMeta cur = meta(c);
    for (; c < c_end; c += stride) {
        issue(cur, c);
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        const ChunkMeta nxt = meta(c + stride);  // resolve the next chunk while the copies fly
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncwarp();
        const float* ys = reinterpret_cast<const float*>(wsm);
        const float* xs = ys + 32 * S;
        for (std::uint32_t idx = std::uint32_t(lane); idx < cur.nx * f; idx += 32) {
            const std::uint32_t rr = idx / f;
            xd[rr * xpitch + (idx - rr * f)] = double(xs[idx]);
        }
        __syncwarp();
        if (cur.valid) {
            const float* yr = ys + lane * S;
            const std::uint32_t rel = cur.r - cur.r_first;
            double acc;
            if (rel < cur.nx) acc = dot_ord<ORD, VLDS, MIX>(xd + std::uint64_t(rel) * xpitch, yr, f, ft);
            else acc = dot_ord<ORD, false, 0>(x + std::uint64_t(cur.r) * f, yr, f, ft);
            out[c * 32 + lane] = float(acc);
        }
        __syncwarp();
        cur = nxt;
    }
}

// MIX (re-bias half of the Y widening on the ALU pipe) only when the
// device-side scan found Y finite and the float4 smem path is in use.
template <bool VLOAD, int ORD, bool VLDS>
__global__ void __launch_bounds__(512)
    sddmm_chunk_kernel(const std::uint64_t* __restrict__ rowptr,
                       const std::uint32_t* __restrict__ colind,
                       const std::uint32_t* __restrict__ chunk_row, std::uint64_t n_rows,
                       const float* __restrict__ x, const float* __restrict__ y,
                       float* __restrict__ out, std::uint64_t nnz, std::uint64_t c_begin,
                       std::uint64_t c_end, std::uint32_t f, std::uint32_t S, std::uint32_t ft,
                       const unsigned* __restrict__ finite, int allow_mix) {
    extern __shared__ __align__(16) char smem[];
    char* wsm = smem + std::uint64_t(threadIdx.x >> 5) * warp_slice_bytes(f, S);
    if (VLDS && allow_mix && finite && *finite)
        sddmm_chunk_body<VLOAD, ORD, VLDS, 1>(rowptr, colind, chunk_row, n_rows, x, y, out, nnz, c_begin,
                                                  c_end, f, S, ft, wsm);
    else
        sddmm_chunk_body<VLOAD, ORD, VLDS, 0>(rowptr, colind, chunk_row, n_rows, x, y, out, nnz, c_begin,
                                                  c_end, f, S, ft, wsm);
}

// ---------------------------------------------------------------------------
// Fixed-width path (F in {16, 32, 64, 128}, X/Y 16-byte aligned): the copy
// and dot loops unroll completely, X is read pre-widened (f64, one prepass
// per call) with broadcast loads instead of being staged per chunk, and
// each lane finds its row from one coalesced read of the 32 row boundaries
// after the chunk's first row.  Shared memory holds only the 32 staged Y
// rows (pitch: odd number of 16-byte units).
// ---------------------------------------------------------------------------
// X -> f64.  When Y is finite (flag from finite_check_kernel) components 2
// and 3 of every float4 carry the 2^896 that widen_scaled() takes out of
// the matching Y components (widen.cuh).
__global__ void widen_kernel(const float4* __restrict__ x, double2* __restrict__ xd, std::uint64_t n4,
                             const unsigned* __restrict__ finite, int mix_all) {
    const double up = (finite && *finite) ? kWidenUp : 1.0;
    const double up01 = mix_all ? up : 1.0;
    for (std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
         i += std::uint64_t(gridDim.x) * blockDim.x) {
        const float4 v = __ldg(x + i);
        xd[2 * i] = make_double2(double(v.x) * up01, double(v.y) * up01);
        xd[2 * i + 1] = make_double2(double(v.z) * up, double(v.w) * up);
    }
}

// 16-bit X (4 words per uint2, half.cuh) -> f64, the same layout and scaling
template <int WT>
__global__ void widen_half_kernel(const uint2* __restrict__ x, double2* __restrict__ xd, std::uint64_t n4,
                                  const unsigned* __restrict__ finite, int mix_all) {
    const double up = (finite && *finite) ? kWidenUp : 1.0;
    const double up01 = mix_all ? up : 1.0;
    for (std::uint64_t i = std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
         i += std::uint64_t(gridDim.x) * blockDim.x) {
        const uint2 v = __ldg(x + i);
        const float a = half_lo<WT>(v.x), b = half_hi<WT>(v.x);
        const float c = half_lo<WT>(v.y), d = half_hi<WT>(v.y);
        xd[2 * i] = make_double2(double(a) * up01, double(b) * up01);
        xd[2 * i + 1] = make_double2(double(c) * up, double(d) * up);
    }
}

// FW = features staged per pass (F = npass * FW, runtime F).
template <int FW>
struct FixedShape {
    static constexpr int NV = FW / 4;                 // 16-byte units per row slice
    static constexpr int S = FW;                      // smem pitch in floats: rows 16-B aligned,
                                                      // 16-B chunks XOR-swizzled (see swz)
    static constexpr int kCopies = NV;                // cp.async per lane per pass (32 rows)
    static constexpr int KX = FW >= 64 ? 1 : 64 / FW; // X rows (f64) staged per chunk
    static constexpr int kXUnits = KX * FW / 2;       // their 16-byte units per pass
    static constexpr std::uint64_t kYBytes = 32ull * S * 4;
    static constexpr std::uint64_t kWarpBytes = kYBytes + std::uint64_t(KX) * FW * 8;
};

// Y rows sit unpadded in shared memory, so each 256-B row is written as two
// whole 128-B wavefronts; 16-byte chunk c of row j is stored at c ^ swz(j).
// When lane j then reads chunk c of its own row, any 8 consecutive lanes hit
// 8 distinct 16-B bank groups (NV >= 8: j & 7 permutes the chunk index
// within 128 B; NV == 4: rows are 64 B, so alternate lanes already sit in
// opposite halves of a 128-B segment and (j >> 1) & 3 separates the rest).
// An odd unit count per row (F = 100: 25 units) needs no swizzle: row j then
// starts at 16-byte bank group 25j mod 8, distinct for any 8 consecutive rows.
template <int NV>
__device__ __forceinline__ int swz(int j) {
    static_assert(NV % 2 == 1 || NV % 8 == 0 || NV == 4, "XOR swizzle must stay inside the row");
    if constexpr (NV % 2 == 1) return 0;
    else if constexpr (NV >= 8) return j & 7;
    else return (j >> 1) & 3;
}

template <bool SMEM>
__device__ __forceinline__ double2 ld_x2(const double* p) {
    if constexpr (SMEM) return *reinterpret_cast<const double2*>(p);
    else return __ldg(reinterpret_cast<const double2*>(p));
}

__device__ __forceinline__ void fold4(double& acc, double& a0, double& a1, double& a2, double& a3) {
    // src/kernels.cpp:103-127: block end; F % 4 == 0, so the scalar tail is empty
    const double tail = 0.0;
    acc = __dadd_rn(acc, __dadd_rn(__dadd_rn(__dadd_rn(a0, a1), __dadd_rn(a2, a3)), tail));
    a0 = a1 = a2 = a3 = 0.0;
}

// One pass (features [p*FW, (p+1)*FW)) of the lane's dot, continuing the
// chain(s).  ORD 0: one sequential chain.  ORD 1: four stride-4 partials per
// f_tile block; FT = 0 means one block over all F.
template <int FW, int ORD, int FT, bool XS, int MIX>
__device__ __forceinline__ void fixed_pass(const double* __restrict__ xr, const float* yr, int key, int p,
                                           int npass, double& acc, double& a0, double& a1, double& a2,
                                           double& a3) {
#pragma unroll 8
    for (int t = 0; t < FW; t += 4) {
        const float4 y4 = *reinterpret_cast<const float4*>(yr + 4 * ((t >> 2) ^ key));
        const double2 x01 = ld_x2<XS>(xr + t);
        const double2 x23 = ld_x2<XS>(xr + t + 2);
        if constexpr (ORD == 0) {
            // MIX 1: components 2,3 re-biased (ALU); MIX 2: all four
            acc = __fma_rn(x01.x, widen<(MIX >= 2)>(y4.x), acc);
            acc = __fma_rn(x01.y, widen<(MIX >= 2)>(y4.y), acc);
            acc = __fma_rn(x23.x, widen<(MIX >= 1)>(y4.z), acc);
            acc = __fma_rn(x23.y, widen<(MIX >= 1)>(y4.w), acc);
        } else {
            a0 = __fma_rn(x01.x, widen<(MIX >= 2)>(y4.x), a0);
            a1 = __fma_rn(x01.y, widen<(MIX >= 2)>(y4.y), a1);
            a2 = __fma_rn(x23.x, widen<(MIX >= 1)>(y4.z), a2);
            a3 = __fma_rn(x23.y, widen<(MIX >= 1)>(y4.w), a3);
            if constexpr (FT != 0 && FT <= FW)
                if ((t + 4) % FT == 0) fold4(acc, a0, a1, a2, a3);
        }
    }
    if constexpr (ORD == 1 && (FT == 0 || FT > FW)) {
        const bool end = p == npass - 1 || (FT != 0 && ((p + 1) * FW) % (FT != 0 ? FT : 1) == 0);
        if (end) fold4(acc, a0, a1, a2, a3);
    }
}

template <int FW, int ORD, int FT, int MIX, int NP>
__device__ __forceinline__ void sddmm_fixed_body(const std::uint64_t* __restrict__ rowptr,
                                                 const std::uint32_t* __restrict__ colind,
                                                 const std::uint32_t* __restrict__ chunk_row,
                                                 std::uint64_t n_rows, const double* __restrict__ xd,
                                                 const float* __restrict__ y, float* __restrict__ out,
                                                 std::uint64_t nnz, std::uint32_t F, std::uint64_t c_begin,
                                                 std::uint64_t c_end) {
    using Sh = FixedShape<FW>;
    extern __shared__ __align__(16) char smem[];
    char* wsm = smem + std::uint64_t(threadIdx.x >> 5) * Sh::kWarpBytes;
    float* ys = reinterpret_cast<float*>(wsm);
    double* xs = reinterpret_cast<double*>(wsm + Sh::kYBytes);
    const int lane = threadIdx.x & 31;
    // NP > 0: F = NP * FW known at compile time (single-pass shapes)
    const int npass = NP > 0 ? NP : int(F / FW);
    if constexpr (NP > 0) F = NP * FW;
    const std::uint64_t stride = std::uint64_t(gridDim.x) * (blockDim.x >> 5);

    struct Meta {
        std::uint32_t col, r_first;
        std::uint64_t bound;  // rowptr[r_first + 1 + lane] (or past-the-end)
    };
    auto meta = [&](std::uint64_t c) {
        Meta m{0u, 0u, ~0ull};
        if (c >= c_end) return m;
        const std::uint64_t e = c * 32 + lane;
        m.col = e < nnz ? __ldg(colind + e) : 0u;  // row 0 stands in for the tail's copies
        m.r_first = __ldg(chunk_row + c);
        const std::uint64_t bi = std::uint64_t(m.r_first) + 1 + lane;
        if (bi <= n_rows) m.bound = __ldg(rowptr + bi);
        return m;
    };
    // this pass's Y slice of the 32 rows and X slice of rows r_first.. (+KX)
    auto issue = [&](const Meta& m, int p) {
#pragma unroll
        for (int it = 0; it < Sh::kCopies; ++it) {
            const int idx = it * 32 + lane;
            const int j = idx / Sh::NV, q = idx % Sh::NV;
            const std::uint32_t cj = __shfl_sync(FULL, m.col, j);
            cp_async16(ys + j * Sh::S + 4 * (q ^ swz<Sh::NV>(j)), y + std::uint64_t(cj) * F + p * FW + 4 * q);
        }
#pragma unroll
        for (int u = lane; u < Sh::kXUnits; u += 32) {
            const int k = u / (FW / 2), uu = u % (FW / 2);
            const std::uint64_t xr = std::uint64_t(m.r_first) + k;
            if (xr < n_rows) cp_async16(xs + 2 * u, xd + xr * F + p * FW + 2 * uu);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };

    std::uint64_t c = c_begin + std::uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    Meta cur = meta(c);
    for (; c < c_end; c += stride) {
        issue(cur, 0);
        const Meta nxt = meta(c + stride);
        // the lane's row: count the chunk's row boundaries at or before e
        // (sorted, so the k boundaries inside the chunk sit in lanes 0..k-1)
        const std::uint64_t e0 = c * 32, e = e0 + lane;
        std::uint32_t r = cur.r_first;
        const unsigned inside = __ballot_sync(FULL, cur.bound <= e0 + 31);
        if (inside) {
            const int k = __popc(inside);
#pragma unroll 1
            for (int b = 0; b < k; ++b) r += __shfl_sync(FULL, cur.bound, b) <= e ? 1u : 0u;
            // more rows meet in this chunk; the tail's idle lanes search
            // for the last entry's row (rowptr ends at nnz)
            if (k == 32) r = row_of(rowptr, r, e < nnz ? e : nnz - 1);
        }
        const std::uint32_t rel = r - cur.r_first;
        const float* yr = ys + lane * Sh::S;
        const int key = swz<Sh::NV>(lane);
        double acc = 0.0, a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        for (int p = 0; p < npass; ++p) {
            if (p > 0) issue(cur, p);
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
            __syncwarp();
            if (e < nnz) {
                if (rel < Sh::KX)
                    fixed_pass<FW, ORD, FT, true, MIX>(xs + rel * FW, yr, key, p, npass, acc, a0, a1, a2, a3);
                else
                    fixed_pass<FW, ORD, FT, false, MIX>(xd + std::uint64_t(r) * F + p * FW, yr, key, p, npass, acc,
                                                        a0, a1, a2, a3);
            }
            __syncwarp();
        }
        if (e < nnz) out[e] = float(acc);
        cur = nxt;
    }
}

template <int FW, int ORD, int FT, int NP>
__global__ void __launch_bounds__(256, 3)
    sddmm_fixed_kernel(const std::uint64_t* __restrict__ rowptr, const std::uint32_t* __restrict__ colind,
                       const std::uint32_t* __restrict__ chunk_row, std::uint64_t n_rows,
                       const double* __restrict__ xd, const float* __restrict__ y,
                       float* __restrict__ out, std::uint64_t nnz, std::uint32_t f, std::uint64_t c_begin,
                       std::uint64_t c_end, const unsigned* __restrict__ finite, int mix_all) {
    if (finite && *finite && mix_all)
        sddmm_fixed_body<FW, ORD, FT, 2, NP>(rowptr, colind, chunk_row, n_rows, xd, y, out, nnz, f, c_begin,
                                             c_end);
    else if (finite && *finite)
        sddmm_fixed_body<FW, ORD, FT, 1, NP>(rowptr, colind, chunk_row, n_rows, xd, y, out, nnz, f, c_begin,
                                             c_end);
    else
        sddmm_fixed_body<FW, ORD, FT, 0, NP>(rowptr, colind, chunk_row, n_rows, xd, y, out, nnz, f, c_begin,
                                             c_end);
}

// ---------------------------------------------------------------------------
// Pair path (F = 32, or F a multiple of 64 in passes of FW = 64 features):
// each lane owns two entries, e and e + 32, of a 64-entry chunk.  The
// broadcast X reads (half of the shared-memory wavefronts of a 32-entry
// chunk) then serve two dot chains, and each lane has two independent
// chains in flight.  64 staged Y rows (of the pass's FW features) per warp.
// ---------------------------------------------------------------------------
template <int FW>
struct PairShape {
    static constexpr int NV = FW / 4;
    static constexpr int kCopies = 2 * NV;  // cp.async per lane per pass (64 rows)
    static constexpr int KX = 2;            // X rows staged
    static constexpr int kXUnits = KX * FW / 2;
    static constexpr std::uint64_t kYBytes = 64ull * FW * 4;
    static constexpr std::uint64_t kWarpBytes = kYBytes + std::uint64_t(KX) * FW * 8;
};

// One pass (features [p*FW, (p+1)*FW)) of both chains.  FT = 0: one f_tile
// block over all of F.
// SAME: both entries of every lane sit in one row (warp-uniform), so the
// second X read is skipped without a per-step branch
template <int FW, int ORD, int FT, bool XS, int MIX, bool SAME>
__device__ __forceinline__ void pair_pass(const double* __restrict__ xa, const double* __restrict__ xb,
                                          const float* ya, const float* yb, int ka, int kb, int p, int npass,
                                          double (&c)[2][5]) {
#pragma unroll 4
    for (int t = 0; t < FW; t += 4) {
        const float4 u = *reinterpret_cast<const float4*>(ya + 4 * ((t >> 2) ^ ka));
        const float4 w = *reinterpret_cast<const float4*>(yb + 4 * ((t >> 2) ^ kb));
        const double2 x01 = ld_x2<XS>(xa + t);
        const double2 x23 = ld_x2<XS>(xa + t + 2);
        double2 z01 = x01, z23 = x23;
        if constexpr (!SAME) {
            z01 = ld_x2<XS>(xb + t);
            z23 = ld_x2<XS>(xb + t + 2);
        }
        if constexpr (ORD == 0) {
            c[0][0] = __fma_rn(x01.x, widen<0>(u.x), c[0][0]);
            c[1][0] = __fma_rn(z01.x, widen<0>(w.x), c[1][0]);
            c[0][0] = __fma_rn(x01.y, widen<0>(u.y), c[0][0]);
            c[1][0] = __fma_rn(z01.y, widen<0>(w.y), c[1][0]);
            c[0][0] = __fma_rn(x23.x, widen<MIX>(u.z), c[0][0]);
            c[1][0] = __fma_rn(z23.x, widen<MIX>(w.z), c[1][0]);
            c[0][0] = __fma_rn(x23.y, widen<MIX>(u.w), c[0][0]);
            c[1][0] = __fma_rn(z23.y, widen<MIX>(w.w), c[1][0]);
        } else {
            c[0][1] = __fma_rn(x01.x, widen<0>(u.x), c[0][1]);
            c[1][1] = __fma_rn(z01.x, widen<0>(w.x), c[1][1]);
            c[0][2] = __fma_rn(x01.y, widen<0>(u.y), c[0][2]);
            c[1][2] = __fma_rn(z01.y, widen<0>(w.y), c[1][2]);
            c[0][3] = __fma_rn(x23.x, widen<MIX>(u.z), c[0][3]);
            c[1][3] = __fma_rn(z23.x, widen<MIX>(w.z), c[1][3]);
            c[0][4] = __fma_rn(x23.y, widen<MIX>(u.w), c[0][4]);
            c[1][4] = __fma_rn(z23.y, widen<MIX>(w.w), c[1][4]);
            if constexpr (FT != 0 && FT <= FW) {
                if ((t + 4) % FT == 0) {
                    fold4(c[0][0], c[0][1], c[0][2], c[0][3], c[0][4]);
                    fold4(c[1][0], c[1][1], c[1][2], c[1][3], c[1][4]);
                }
            }
        }
    }
    if constexpr (ORD == 1 && (FT == 0 || FT > FW)) {
        const bool end = p == npass - 1 || (FT != 0 && ((p + 1) * FW) % (FT != 0 ? FT : 1) == 0);
        if (end) {
            fold4(c[0][0], c[0][1], c[0][2], c[0][3], c[0][4]);
            fold4(c[1][0], c[1][1], c[1][2], c[1][3], c[1][4]);
        }
    }
}

template <int FW, int ORD, int FT, int MIX, int NP>
__device__ __forceinline__ void sddmm_pair_body(const std::uint64_t* __restrict__ rowptr,
                                                const std::uint32_t* __restrict__ colind,
                                                const std::uint32_t* __restrict__ chunk_row, std::uint64_t n_rows,
                                                const double* __restrict__ xd, const float* __restrict__ y,
                                                float* __restrict__ out, std::uint64_t nnz, std::uint32_t F,
                                                std::uint64_t c_begin, std::uint64_t c_end) {
    using Sh = PairShape<FW>;
    extern __shared__ __align__(16) char smem[];
    char* wsm = smem + std::uint64_t(threadIdx.x >> 5) * Sh::kWarpBytes;
    float* ys = reinterpret_cast<float*>(wsm);
    double* xs = reinterpret_cast<double*>(wsm + Sh::kYBytes);
    const int lane = threadIdx.x & 31;
    const int npass = NP > 0 ? NP : int(F / FW);
    if constexpr (NP > 0) F = NP * FW;
    const std::uint64_t e_end = min(c_end * 32, nnz);
    const std::uint64_t n_pairs = (c_end - c_begin + 1) / 2;
    const std::uint64_t stride = std::uint64_t(gridDim.x) * (blockDim.x >> 5);

    struct Meta {
        std::uint32_t ca, cb, r_first;
        std::uint64_t bound;
    };
    auto meta = [&](std::uint64_t pc) {
        Meta m{0u, 0u, 0u, ~0ull};
        if (pc >= n_pairs) return m;
        const std::uint64_t e0 = (c_begin + 2 * pc) * 32;
        m.ca = e0 + lane < e_end ? __ldg(colind + e0 + lane) : 0u;
        m.cb = e0 + 32 + lane < e_end ? __ldg(colind + e0 + 32 + lane) : 0u;
        m.r_first = __ldg(chunk_row + c_begin + 2 * pc);
        const std::uint64_t bi = std::uint64_t(m.r_first) + 1 + lane;
        if (bi <= n_rows) m.bound = __ldg(rowptr + bi);
        return m;
    };
    auto issue = [&](const Meta& m, int p) {
#pragma unroll
        for (int it = 0; it < Sh::kCopies; ++it) {
            const int idx = it * 32 + lane;
            const int j = idx / Sh::NV, q = idx % Sh::NV;
            const std::uint32_t cj = __shfl_sync(FULL, j < 32 ? m.ca : m.cb, j & 31);
            cp_async16(ys + j * FW + 4 * (q ^ swz<Sh::NV>(j)), y + std::uint64_t(cj) * F + p * FW + 4 * q);
        }
#pragma unroll
        for (int u = lane; u < Sh::kXUnits; u += 32) {
            const int k = u / (FW / 2), uu = u % (FW / 2);
            const std::uint64_t xr = std::uint64_t(m.r_first) + k;
            if (xr < n_rows) cp_async16(xs + 2 * u, xd + xr * F + p * FW + 2 * uu);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };

    std::uint64_t pc = std::uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    Meta cur = meta(pc);
    for (; pc < n_pairs; pc += stride) {
        issue(cur, 0);
        const Meta nxt = meta(pc + stride);
        const std::uint64_t e0 = (c_begin + 2 * pc) * 32, ea = e0 + lane, eb = ea + 32;
        std::uint32_t ra = cur.r_first, rb = cur.r_first;
        const unsigned inside = __ballot_sync(FULL, cur.bound <= e0 + 63);
        if (inside) {
            const int k = __popc(inside);
#pragma unroll 1
            for (int b = 0; b < k; ++b) {
                const std::uint64_t bb = __shfl_sync(FULL, cur.bound, b);
                ra += bb <= ea ? 1u : 0u;
                rb += bb <= eb ? 1u : 0u;
            }
            if (k == 32) {  // more than 32 rows meet in these 64 entries
                ra = row_of(rowptr, ra, ea < e_end ? ea : e_end - 1);
                rb = row_of(rowptr, rb, eb < e_end ? eb : e_end - 1);
            }
        }
        // lanes past the last entry (tail chunk) counted the trailing empty
        // rows' boundaries too and may sit at n_rows: park them on a real row
        // (their results are not stored; found by the checked build)
        if (ea >= e_end) ra = cur.r_first;
        if (eb >= e_end) rb = cur.r_first;
        const std::uint32_t rela = ra - cur.r_first, relb = rb - cur.r_first;
        const bool staged = rela < Sh::KX && relb < Sh::KX;
        double c[2][5] = {{0.0, 0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0, 0.0}};
        const float* ya = ys + lane * FW;
        const float* yb = ys + (lane + 32) * FW;
        const int ka = swz<Sh::NV>(lane), kb = swz<Sh::NV>(lane + 32);
        // warp-uniform, taken before the per-lane staged/unstaged split
        const bool all_same = __all_sync(FULL, rela == relb);
        auto run_pass = [&](int p) {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
            __syncwarp();
            if (staged) {
                if (all_same)
                    pair_pass<FW, ORD, FT, true, MIX, true>(xs + rela * FW, xs + relb * FW, ya, yb, ka, kb, p,
                                                            npass, c);
                else
                    pair_pass<FW, ORD, FT, true, MIX, false>(xs + rela * FW, xs + relb * FW, ya, yb, ka, kb, p,
                                                             npass, c);
            } else {
                pair_pass<FW, ORD, FT, false, MIX, false>(xd + std::uint64_t(ra) * F + p * FW,
                                                          xd + std::uint64_t(rb) * F + p * FW, ya, yb, ka, kb, p,
                                                          npass, c);
            }
        };
        if constexpr (NP == 1) {
            run_pass(0);
        } else {
            for (int p = 0; p < npass; ++p) {
                if (p > 0) {
                    __syncwarp();  // every lane done reading the previous pass
                    issue(cur, p);
                }
                run_pass(p);
            }
        }
        __syncwarp();
        if (ea < e_end) out[ea] = float(c[0][0]);
        if (eb < e_end) out[eb] = float(c[1][0]);
        cur = nxt;
    }
}

template <int FW, int ORD, int FT, int NP>
__global__ void __launch_bounds__(128, 3)
    sddmm_pair_kernel(const std::uint64_t* __restrict__ rowptr, const std::uint32_t* __restrict__ colind,
                      const std::uint32_t* __restrict__ chunk_row, std::uint64_t n_rows,
                      const double* __restrict__ xd, const float* __restrict__ y, float* __restrict__ out,
                      std::uint64_t nnz, std::uint32_t f, std::uint64_t c_begin, std::uint64_t c_end,
                      const unsigned* __restrict__ finite, int /*mix_all*/) {
    if (finite && *finite)
        sddmm_pair_body<FW, ORD, FT, 1, NP>(rowptr, colind, chunk_row, n_rows, xd, y, out, nnz, f, c_begin, c_end);
    else
        sddmm_pair_body<FW, ORD, FT, 0, NP>(rowptr, colind, chunk_row, n_rows, xd, y, out, nnz, f, c_begin, c_end);
}

// Single-pass F in {32, 64}: the same pair mapping with F compiled in (this
// specialisation measured 6% faster than the pass loop at F = 64).
// BF: Y rows staged as bf16 (half the cp.async and LDS wavefronts; one
// 16-byte unit holds 8 features)
#ifndef ASB_PAIR_RF_PREFETCH
#define ASB_PAIR_RF_PREFETCH 1  // chunk_row loaded an iteration ahead (A/B build knob)
#endif
#ifndef ASB_PAIR_KX
#define ASB_PAIR_KX 2  // X rows a pair-kernel warp stages for F <= 64 (A/B build knob)
#endif
template <int F, bool BF = false>
struct Pair1Shape {
    static constexpr int kYElem = BF ? 2 : 4;
    static constexpr int NV = F * kYElem / 16;  // 16-byte units per Y row
    static constexpr int kCopies = 2 * NV;      // cp.async per lane per chunk (64 rows)
    // X rows staged: the first KX rows of the 64-entry window are read from
    // shared memory, lanes in later rows read the widened X from L1/L2
    static constexpr int KX = F <= 64 ? ASB_PAIR_KX : 2;
    static constexpr int kXUnits = KX * F / 2;
    static constexpr std::uint64_t kYBytes = 64ull * F * kYElem;
    static constexpr std::uint64_t kWarpBytes = kYBytes + std::uint64_t(KX) * F * 8;
};

// Y features [t, t+4) of the lane's two rows as f32 (u for entry a, w for b)
template <int F, int WT>
__device__ __forceinline__ void pair1_y4(const void* ya, const void* yb, int ka, int kb, int t, float4& u,
                                         float4& w) {
    if constexpr (WT != kWtF32) {
        const unsigned short* pa = static_cast<const unsigned short*>(ya);
        const unsigned short* pb = static_cast<const unsigned short*>(yb);
        const uint2 ua = *reinterpret_cast<const uint2*>(pa + 8 * ((t >> 3) ^ ka) + (t & 4));
        const uint2 wb = *reinterpret_cast<const uint2*>(pb + 8 * ((t >> 3) ^ kb) + (t & 4));
        u = make_float4(half_lo<WT>(ua.x), half_hi<WT>(ua.x), half_lo<WT>(ua.y), half_hi<WT>(ua.y));
        w = make_float4(half_lo<WT>(wb.x), half_hi<WT>(wb.x), half_lo<WT>(wb.y), half_hi<WT>(wb.y));
    } else {
        u = *reinterpret_cast<const float4*>(static_cast<const float*>(ya) + 4 * ((t >> 2) ^ ka));
        w = *reinterpret_cast<const float4*>(static_cast<const float*>(yb) + 4 * ((t >> 2) ^ kb));
    }
}

// X features [t, t+4) of a row read as f32 from global memory and widened
// here (the F=100 path has no f64 prepass): components 2, 3 pre-scaled by
// 2^896 under MIX, as the prepass would have stored them
template <int MIX>
__device__ __forceinline__ void ld_xf4(const double* p, double2& x01, double2& x23) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(p));
    const double up = MIX ? kWidenUp : 1.0;
    x01 = make_double2(double(v.x), double(v.y));
    x23 = make_double2(double(v.z) * up, double(v.w) * up);
}

// XF: the X pointers are f32 rows (reinterpreted; see ld_xf4) when !XS
template <int F, int ORD, int FT, bool XS, int MIX, bool SAME, int WT = kWtF32, bool XF = false>
__device__ __forceinline__ void pair1_pass(const double* __restrict__ xa, const double* __restrict__ xb,
                                          const void* ya, const void* yb, int ka, int kb, double (&c)[2][5]) {
#pragma unroll 4
    for (int t = 0; t < F; t += 4) {
        float4 u, w;
        pair1_y4<F, WT>(ya, yb, ka, kb, t, u, w);
        double2 x01, x23;
        if constexpr (XF && !XS) {
            ld_xf4<MIX>(reinterpret_cast<const double*>(reinterpret_cast<const float*>(xa) + t), x01, x23);
        } else {
            x01 = ld_x2<XS>(xa + t);
            x23 = ld_x2<XS>(xa + t + 2);
        }
        double2 z01 = x01, z23 = x23;
        if constexpr (!SAME) {
            if constexpr (XF && !XS) {
                ld_xf4<MIX>(reinterpret_cast<const double*>(reinterpret_cast<const float*>(xb) + t), z01, z23);
            } else {
                z01 = ld_x2<XS>(xb + t);
                z23 = ld_x2<XS>(xb + t + 2);
            }
        }
        if constexpr (ORD == 0) {
            c[0][0] = __fma_rn(x01.x, widen<0>(u.x), c[0][0]);
            c[1][0] = __fma_rn(z01.x, widen<0>(w.x), c[1][0]);
            c[0][0] = __fma_rn(x01.y, widen<0>(u.y), c[0][0]);
            c[1][0] = __fma_rn(z01.y, widen<0>(w.y), c[1][0]);
            c[0][0] = __fma_rn(x23.x, widen<MIX>(u.z), c[0][0]);
            c[1][0] = __fma_rn(z23.x, widen<MIX>(w.z), c[1][0]);
            c[0][0] = __fma_rn(x23.y, widen<MIX>(u.w), c[0][0]);
            c[1][0] = __fma_rn(z23.y, widen<MIX>(w.w), c[1][0]);
        } else {
            c[0][1] = __fma_rn(x01.x, widen<0>(u.x), c[0][1]);
            c[1][1] = __fma_rn(z01.x, widen<0>(w.x), c[1][1]);
            c[0][2] = __fma_rn(x01.y, widen<0>(u.y), c[0][2]);
            c[1][2] = __fma_rn(z01.y, widen<0>(w.y), c[1][2]);
            c[0][3] = __fma_rn(x23.x, widen<MIX>(u.z), c[0][3]);
            c[1][3] = __fma_rn(z23.x, widen<MIX>(w.z), c[1][3]);
            c[0][4] = __fma_rn(x23.y, widen<MIX>(u.w), c[0][4]);
            c[1][4] = __fma_rn(z23.y, widen<MIX>(w.w), c[1][4]);
            const bool block_end = FT == 0 ? t + 4 == F : ((t + 4) % FT == 0 || t + 4 == F);
            if (block_end) {
                fold4(c[0][0], c[0][1], c[0][2], c[0][3], c[0][4]);
                fold4(c[1][0], c[1][1], c[1][2], c[1][3], c[1][4]);
            }
        }
    }
}

// Pass-major form (PM; F = 64 features of a wider row): features
// [f0, f0 + 64) of rows of width ld, each entry's f64 chain continued from
// state[e] (f0 > 0) and left in state[e] (not last) or rounded to out[e]
// (last).  One launch per 64-feature pass keeps the pass's 64-column Y slice
// L2-resident where the whole Y (n_cols x ld) is not; the chains and the
// ORD 1 blocks (ft 32 / 64: every block ends inside a pass) fold exactly as
// in the single-launch kernels, so the result is unchanged bit for bit.
struct PassArgs {
    std::uint32_t ld = 0, f0 = 0;
    double* state = nullptr;
    int last = 1;
};

template <int F, int ORD, int FT, int MIX, int WT = kWtF32, bool PM = false, bool XF = false>
__device__ __forceinline__ void sddmm_pair1_body(const std::uint64_t* __restrict__ rowptr,
                                                const std::uint32_t* __restrict__ colind,
                                                const std::uint32_t* __restrict__ chunk_row, std::uint64_t n_rows,
                                                const double* __restrict__ xd, const void* __restrict__ yv,
                                                float* __restrict__ out, std::uint64_t nnz, std::uint64_t c_begin,
                                                std::uint64_t c_end, int keep, std::uint64_t n_cols,
                                                PassArgs pa = PassArgs{}) {
    (void)n_cols;  // bounds of the checked build
    // row stride of X and Y, and the pass's first feature
    const std::uint64_t LD = PM ? pa.ld : F;
    const std::uint32_t F0 = PM ? pa.f0 : 0u;
    using Sh = Pair1Shape<F, WT != kWtF32>;
    using YT = typename std::conditional<WT != kWtF32, unsigned short, float>::type;
    constexpr int kUnitElems = 16 / Sh::kYElem;  // Y elements per 16-byte unit
    const YT* __restrict__ y = static_cast<const YT*>(yv);
    extern __shared__ __align__(16) char smem[];
    char* wsm = smem + std::uint64_t(threadIdx.x >> 5) * Sh::kWarpBytes;
    YT* ys = reinterpret_cast<YT*>(wsm);
    double* xs = reinterpret_cast<double*>(wsm + Sh::kYBytes);
    const int lane = threadIdx.x & 31;
    const std::uint64_t e_end = min(c_end * 32, nnz);
    const std::uint64_t n_pairs = (c_end - c_begin + 1) / 2;
    const std::uint64_t stride = std::uint64_t(gridDim.x) * (blockDim.x >> 5);
    // colind and the outputs stream once (evict_first); Y rows and the
    // widened X are re-read for every entry that hits them (evict_last)
    // keep bit 0: Y fits the L2 budget; bits 2:1 the widened X's policy
    // (0 as Y, 1 evict_normal, 2 evict_first: X rows are read by the
    // neighbouring chunk pairs only, so they need not outlive them)
    const std::uint64_t pol_s = l2_evict_first(), pol_k = l2_reuse_policy((keep & 1) != 0);
    const int xp = (keep >> 1) & 3;
    const std::uint64_t pol_x = xp == 0 ? pol_k : xp == 1 ? l2_evict_normal() : pol_s;

    struct Meta {
        std::uint32_t ca, cb, r_first;
        std::uint64_t bound;
    };
    // the chunk's first row is loaded one iteration before the rest of its
    // metadata: the rowptr bounds load depends on it, and issuing both back
    // to back stalled every iteration on the chunk_row load (the hottest
    // stall line of the r02ak capture)
    auto first_row = [&](std::uint64_t pc) {
        return pc < n_pairs ? __ldg(chunk_row + c_begin + 2 * pc) : 0u;
    };
    auto meta = [&](std::uint64_t pc, std::uint32_t r_first) {
        Meta m{0u, 0u, r_first, ~0ull};
        if (pc >= n_pairs) return m;
        const std::uint64_t e0 = (c_begin + 2 * pc) * 32;
        m.ca = e0 + lane < e_end ? ld_stream(colind + e0 + lane, pol_s) : 0u;
        m.cb = e0 + 32 + lane < e_end ? ld_stream(colind + e0 + 32 + lane, pol_s) : 0u;
        const std::uint64_t bi = std::uint64_t(r_first) + 1 + lane;
        if (bi <= n_rows) m.bound = __ldg(rowptr + bi);
        return m;
    };

    std::uint64_t pc = std::uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    Meta cur = meta(pc, first_row(pc));
#if ASB_PAIR_RF_PREFETCH
    std::uint32_t rf_next = first_row(pc + stride);
#endif
    for (; pc < n_pairs; pc += stride) {
#pragma unroll
        for (int it = 0; it < Sh::kCopies; ++it) {
            const int idx = it * 32 + lane;
            const int j = idx / Sh::NV, q = idx % Sh::NV;
            const std::uint32_t cj = __shfl_sync(FULL, j < 32 ? cur.ca : cur.cb, j & 31);
            ASB_DCHECK(cj < n_cols);
            cp_async16_pol(ys + j * F + kUnitElems * (q ^ swz<Sh::NV>(j)), y + std::uint64_t(cj) * LD + F0 + kUnitElems * q,
                           pol_k);
        }
        // XF: the f32 X rows are loaded here and widened into shared memory
        // after the row search below, so the loads' latency overlaps it
        constexpr int kXf = XF ? (Sh::KX * F / 4 + 31) / 32 : 1;  // float4 per lane
        float4 xv[kXf];
        if constexpr (XF) {
            const float* xf = reinterpret_cast<const float*>(xd);
#pragma unroll
            for (int i = 0; i < kXf; ++i) {
                const int u = lane + 32 * i;
                const int k = u / (F / 4), uu = u % (F / 4);
                const std::uint64_t xr = std::uint64_t(cur.r_first) + k;
                if (u < Sh::KX * F / 4 && xr < n_rows)
                    xv[i] = __ldg(reinterpret_cast<const float4*>(xf + xr * LD + 4 * uu));
            }
        } else {
#pragma unroll
            for (int u = lane; u < Sh::kXUnits; u += 32) {
                const int k = u / (F / 2), uu = u % (F / 2);
                const std::uint64_t xr = std::uint64_t(cur.r_first) + k;
                if (xr < n_rows) cp_async16_pol(xs + 2 * u, xd + xr * LD + F0 + 2 * uu, pol_x);
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
#if ASB_PAIR_RF_PREFETCH
        const Meta nxt = meta(pc + stride, rf_next);
        rf_next = first_row(pc + 2 * stride);
#else
        const Meta nxt = meta(pc + stride, first_row(pc + stride));
#endif
        const std::uint64_t e0 = (c_begin + 2 * pc) * 32, ea = e0 + lane, eb = ea + 32;
        std::uint32_t ra = cur.r_first, rb = cur.r_first;
        const unsigned inside = __ballot_sync(FULL, cur.bound <= e0 + 63);
        if (inside) {
            const int k = __popc(inside);
#pragma unroll 1
            for (int b = 0; b < k; ++b) {
                const std::uint64_t bb = __shfl_sync(FULL, cur.bound, b);
                ra += bb <= ea ? 1u : 0u;
                rb += bb <= eb ? 1u : 0u;
            }
            if (k == 32) {  // more than 32 rows meet in these 64 entries
                ra = row_of(rowptr, ra, ea < e_end ? ea : e_end - 1);
                rb = row_of(rowptr, rb, eb < e_end ? eb : e_end - 1);
            }
        }
        if constexpr (XF) {
            const double up = MIX ? kWidenUp : 1.0;
#pragma unroll
            for (int i = 0; i < kXf; ++i) {
                const int u = lane + 32 * i;
                const int k = u / (F / 4), uu = u % (F / 4);
                const std::uint64_t xr = std::uint64_t(cur.r_first) + k;
                if (u < Sh::KX * F / 4 && xr < n_rows) {
                    double2* dst = reinterpret_cast<double2*>(xs + k * F + 4 * uu);
                    dst[0] = make_double2(double(xv[i].x), double(xv[i].y));
                    dst[1] = make_double2(double(xv[i].z) * up, double(xv[i].w) * up);
                }
            }
        }
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncwarp();
        // lanes past the last entry (tail chunk) counted the trailing empty
        // rows' boundaries too and may sit at n_rows: park them on a real row
        // (their results are not stored; found by the checked build)
        if (ea >= e_end) ra = cur.r_first;
        if (eb >= e_end) rb = cur.r_first;
        const std::uint32_t rela = ra - cur.r_first, relb = rb - cur.r_first;
        ASB_DCHECK(ra < n_rows && rb < n_rows);
        ASB_DCHECK(ea >= e_end || (rowptr[ra] <= ea && ea < rowptr[ra + 1]));
        ASB_DCHECK(eb >= e_end || (rowptr[rb] <= eb && eb < rowptr[rb + 1]));
        double c[2][5] = {{0.0, 0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0, 0.0}};
        if constexpr (PM) {
            if (F0 > 0) {
                if (ea < e_end) c[0][0] = ld_state(pa.state + ea, pol_s);
                if (eb < e_end) c[1][0] = ld_state(pa.state + eb, pol_s);
            }
        }
        const YT* ya = ys + lane * F;
        const YT* yb = ys + (lane + 32) * F;
        const int ka = swz<Sh::NV>(lane), kb = swz<Sh::NV>(lane + 32);
        const bool all_same = __all_sync(FULL, rela == relb);  // warp-uniform, before the split
        if (rela < Sh::KX && relb < Sh::KX) {
            if (all_same)
                pair1_pass<F, ORD, FT, true, MIX, true, WT>(xs + rela * F, xs + relb * F, ya, yb, ka, kb, c);
            else
                pair1_pass<F, ORD, FT, true, MIX, false, WT>(xs + rela * F, xs + relb * F, ya, yb, ka, kb, c);
        } else if constexpr (XF) {
            const float* xf = reinterpret_cast<const float*>(xd);
            pair1_pass<F, ORD, FT, false, MIX, false, WT, true>(
                reinterpret_cast<const double*>(xf + std::uint64_t(ra) * LD),
                reinterpret_cast<const double*>(xf + std::uint64_t(rb) * LD), ya, yb, ka, kb, c);
        } else {
            pair1_pass<F, ORD, FT, false, MIX, false, WT>(xd + std::uint64_t(ra) * LD + F0,
                                                         xd + std::uint64_t(rb) * LD + F0, ya, yb, ka, kb, c);
        }
        if (PM && !pa.last) {
            if (ea < e_end) st_state(pa.state + ea, c[0][0], pol_s);
            if (eb < e_end) st_state(pa.state + eb, c[1][0], pol_s);
        } else {
            if (ea < e_end) st_stream(out + ea, float(c[0][0]), pol_s);
            if (eb < e_end) st_stream(out + eb, float(c[1][0]), pol_s);
        }
        __syncwarp();
        cur = nxt;
    }
}

// MINB: resident CTAs per SM the register budget is cut for.  f32 Y staging
// (17.4 KB per warp at F=64) caps residency at 3 CTAs through shared memory
// anyway; bf16 staging halves that, so its kernels can trade registers for
// occupancy.
// XF: xd is the f32 X itself (widened in the kernel, no prepass)
template <int F, int ORD, int FT, int WT = kWtF32, int MINB = 3, bool XF = false>
__global__ void __launch_bounds__(128, MINB)
    sddmm_pair1_kernel(const std::uint64_t* __restrict__ rowptr, const std::uint32_t* __restrict__ colind,
                      const std::uint32_t* __restrict__ chunk_row, std::uint64_t n_rows,
                      const double* __restrict__ xd, const void* __restrict__ y, float* __restrict__ out,
                      std::uint64_t nnz, std::uint32_t /*f*/, std::uint64_t c_begin, std::uint64_t c_end,
                      const unsigned* __restrict__ finite, int keep, std::uint64_t n_cols) {
    // keep: Y fits the L2 (kKeepMaxBytes) -- the Y and X staging reads evict_last
    if (finite && *finite)
        sddmm_pair1_body<F, ORD, FT, 1, WT, false, XF>(rowptr, colind, chunk_row, n_rows, xd, y, out, nnz, c_begin,
                                                       c_end, keep, n_cols);
    else
        sddmm_pair1_body<F, ORD, FT, 0, WT, false, XF>(rowptr, colind, chunk_row, n_rows, xd, y, out, nnz, c_begin,
                                                       c_end, keep, n_cols);
}

// One 64-feature pass of an F >= 128 SDDMM (PassArgs above)
template <int ORD, int FT>
__global__ void __launch_bounds__(128, 3)
    sddmm_pair1_pm_kernel(const std::uint64_t* __restrict__ rowptr, const std::uint32_t* __restrict__ colind,
                          const std::uint32_t* __restrict__ chunk_row, std::uint64_t n_rows,
                          const double* __restrict__ xd, const void* __restrict__ y, float* __restrict__ out,
                          std::uint64_t nnz, std::uint64_t c_begin, std::uint64_t c_end,
                          const unsigned* __restrict__ finite, int keep, std::uint64_t n_cols, PassArgs pa) {
    if (finite && *finite)
        sddmm_pair1_body<64, ORD, FT, 1, kWtF32, true>(rowptr, colind, chunk_row, n_rows, xd, y, out, nnz, c_begin,
                                                       c_end, keep, n_cols, pa);
    else
        sddmm_pair1_body<64, ORD, FT, 0, kWtF32, true>(rowptr, colind, chunk_row, n_rows, xd, y, out, nnz, c_begin,
                                                       c_end, keep, n_cols, pa);
}

// Guardrail baseline / large-F fallback: lane per entry, both rows read
// straight from global memory, scalar loads.
template <int ORD, class T = float>
__global__ void sddmm_direct_kernel(const std::uint64_t* __restrict__ rowptr,
                                    const std::uint32_t* __restrict__ colind,
                                    const std::uint32_t* __restrict__ chunk_row,
                                    const T* __restrict__ x, const T* __restrict__ y,
                                    float* __restrict__ out, std::uint64_t nnz, std::uint64_t c_begin,
                                    std::uint64_t c_end, std::uint32_t f, std::uint32_t ft) {
    const std::uint64_t ch = c_begin + ((std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
    const std::uint64_t e = ch * 32 + (threadIdx.x & 31);
    if (ch >= c_end || e >= nnz) return;
    const std::uint32_t r = row_of(rowptr, chunk_row[ch], e);
    const T* xr = x + std::uint64_t(r) * f;
    const T* yr = y + std::uint64_t(colind[e]) * f;
    out[e] = float(dot_ord<ORD, false, 0>(xr, yr, f, ft));
}

bool aligned16(const void* p) { return (reinterpret_cast<std::uintptr_t>(p) & 15u) == 0; }

// Fixed-width path: F a multiple of 16, X/Y 16-byte aligned, and an f_tile
// whose blocks line up with the passes.  FW = features staged per pass.
int fixed_fw(std::uint32_t f) {
    if (f == 16 || f == 32 || f == 64) return int(f);
    if (f % 64 == 0) return 64;
    if (f % 32 == 0) return 32;
    if (f % 16 == 0) return 16;
    return 0;
}

// F = 100 (the Products-shape width): the pair kernel with an odd 25-unit
// row pitch; its f_tile blocks (32, 64 or all of F) end inside the row
constexpr std::uint32_t kPairOddF = 100;

bool fixed_eligible(const float* x, const float* y, std::uint32_t f, std::uint32_t ft, int ord) {
    if (!dev_knob("AUTOSAGE_DEV_SDDMM_FIXED", 1)) return false;
    if (f == kPairOddF)
        return dev_knob("AUTOSAGE_DEV_SDDMM_PAIR", 1) && aligned16(x) && aligned16(y) &&
               (ord == 0 || ft >= f || ft == 32 || ft == 64);
    const int fw = fixed_fw(f);
    if (!fw || f > 4096) return false;
    if (!aligned16(x) || !aligned16(y)) return false;
    if (ord == 0 || ft >= f) return true;
    if (!(ft == 32 || ft == 64 || ft == 128)) return false;
    return int(ft) % fw == 0 || fw % int(ft) == 0;
}

// L2 policy of the pair kernels' widened-X staging (keep bits 2:1; see
// sddmm_pair1_body).  AUTOSAGE_DEV_SDDMM_XPOL: 0 as Y (default), 1 normal,
// 2 first.  A/B on Reddit-shape F = 64 / 128 / 256: within 0.5% for 0 and 1,
// 2 is 1-2% slower (profiles/r02m_pass_major.md).
int x_policy_bits() { return (dev_knob("AUTOSAGE_DEV_SDDMM_XPOL", 0) & 3) << 1; }

// Pass-major SDDMM (sddmm_pair1_pm_kernel) for F = 128, 192, ...: every
// f_tile block must end inside a 64-feature pass (ord 0, or ft 32 / 64).
// Auto: when Y is more than twice the L2 budget the streams leave it
// (kKeepMaxBytes) but one pass's 64-column slice fits; the carried chains
// cost 16 B of DRAM traffic per entry per pass boundary, plus one more read
// of colind per pass.  Reddit-shape, sequential order, with the finite
// scan (profiles/r02m_pass_major.md, r02p): F=256 11.62 -> 11.25 ms; F=128
// 4.76 -> 5.41 ms and F=192 7.85 -> 8.86 ms (slower: single launch there).
// AUTOSAGE_DEV_SDDMM_PM: -1 auto (default), 0 never, 1 whenever eligible.
bool pass_major(const Graph& g, std::uint32_t f, std::uint32_t ft, int ord) {
    if (f < 128 || f % 64 != 0) return false;
    if (!(ord == 0 || ft == 32 || ft == 64)) return false;
    const int knob = dev_knob("AUTOSAGE_DEV_SDDMM_PM", -1);
    if (knob >= 0) return knob != 0;
    return std::uint64_t(g.n_cols) * f * 4 > 2 * kKeepMaxBytes && std::uint64_t(g.n_cols) * 64 * 4 <= kKeepMaxBytes;
}

// all four components re-biased on the ALU pipe (dev knob; default: half)
int mix_all() { return dev_knob("AUTOSAGE_DEV_SDDMM_MIXALL", 0); }

int sm_count() { return device_sms(); }

// X widened to f64 (prepass of the fixed-width path, once per call)
// rows [r0, r1) of X (the host pipeline widens each slice's rows as they land)
void widen_x(Graph& g, const float* x, std::uint32_t f, cudaStream_t s, const unsigned* finite,
             std::uint64_t r0 = 0, std::uint64_t r1 = ~0ull) {
    g.xwide.ensure(std::max<std::uint64_t>(g.n_rows * f, 1));
    r1 = std::min(r1, g.n_rows);
    if (r0 >= r1) return;
    const std::uint64_t off4 = r0 * f / 4, n4 = (r1 - r0) * f / 4;
    if (!n4) return;
    const unsigned blocks = unsigned(std::min<std::uint64_t>((n4 + 255) / 256, std::uint64_t(sm_count()) * 8));
    widen_kernel<<<std::max(blocks, 1u), 256, 0, s>>>(reinterpret_cast<const float4*>(x) + off4,
                                                      reinterpret_cast<double2*>(g.xwide.get()) + 2 * off4, n4,
                                                      finite, mix_all());
    check_launch("widen_kernel");
}

// F=100: the pair kernel widens f32 X itself (no f64 prepass, half the X
// bytes); AUTOSAGE_DEV_SDDMM_XF32=0 restores the prepass (A/B)
bool x_widened_in_kernel(std::uint32_t f) { return f == kPairOddF && dev_knob("AUTOSAGE_DEV_SDDMM_XF32", 1) != 0; }

void launch_sddmm_fixed(Graph& g, const float* x, const float* y, std::uint32_t f, float* out, std::uint32_t ft,
                        int ord, cudaStream_t s, const unsigned* finite, std::uint64_t c_begin,
                        std::uint64_t c_end) {
    // Y (re-read by every entry of its column) fits the L2 beside the
    // streams: the staging reads evict_last
    const int keep_y = int(std::uint64_t(g.n_cols) * f * 4 <= kKeepMaxBytes) | x_policy_bits();
    const int sms = sm_count();
    auto go = [&](auto kernel, std::uint64_t warp_bytes) {
        constexpr int kWarps = 8;
        const std::size_t smem = std::size_t(warp_bytes * kWarps);
        const int per_sm = kernel_setup(kernel, smem, int(kWarps * 32));
        const std::uint64_t want = (c_end - c_begin + kWarps - 1) / kWarps;
        const std::uint64_t cap = std::uint64_t(sms) * std::max(per_sm, 1);
        const unsigned blocks = unsigned(std::max<std::uint64_t>(1, std::min(want, cap)));
        kernel<<<blocks, kWarps * 32, smem, s>>>(g.rowptr.get(), g.colind.get(), g.chunk_row.get(), g.n_rows,
                                                 g.xwide.get(), y, out, g.nnz, f, c_begin, c_end, finite,
                                                 mix_all());
        check_launch("sddmm_fixed_kernel");
    };
    // FT: 0 = one block over all of F (ft >= f); else the block width
    auto by_fw = [&](auto fc, auto npc) {
        constexpr int FW = decltype(fc)::value, NP = decltype(npc)::value;
        constexpr std::uint64_t wb = FixedShape<FW>::kWarpBytes;
        if (ord == 0) go(sddmm_fixed_kernel<FW, 0, 0, NP>, wb);
        else if (ft >= f) go(sddmm_fixed_kernel<FW, 1, 0, NP>, wb);
        else if (ft == 32) go(sddmm_fixed_kernel<FW, 1, 32, NP>, wb);
        else if (ft == 64) go(sddmm_fixed_kernel<FW, 1, 64, NP>, wb);
        else go(sddmm_fixed_kernel<FW, 1, 128, NP>, wb);
    };
    const bool pair_ok = (f == 32 || f % 64 == 0 || f == kPairOddF) &&
                         (ord == 0 || ft >= f || ft == 32 || ft % 64 == 0);
    if (pair_ok && dev_knob("AUTOSAGE_DEV_SDDMM_PAIR", 1)) {
        auto pair = [&](auto fc, auto npc) {
            constexpr int FW = decltype(fc)::value, NP = decltype(npc)::value;
            const std::uint64_t wb = PairShape<FW>::kWarpBytes;
            const int kWarps = 4;
            auto run = [&](auto kernel) {
                const std::size_t smem = std::size_t(wb * kWarps);
                const int per_sm = kernel_setup(kernel, smem, int(kWarps * 32));
                const std::uint64_t pairs = (c_end - c_begin + 1) / 2;
                const std::uint64_t want = (pairs + kWarps - 1) / kWarps;
                const std::uint64_t cap = std::uint64_t(sms) * std::max(per_sm, 1);
                const unsigned blocks = unsigned(std::max<std::uint64_t>(1, std::min(want, cap)));
                kernel<<<blocks, kWarps * 32, smem, s>>>(g.rowptr.get(), g.colind.get(), g.chunk_row.get(),
                                                         g.n_rows, g.xwide.get(), y, out, g.nnz, f, c_begin, c_end,
                                                         finite, mix_all());
                check_launch("sddmm_pair_kernel");
            };
            // FT: 0 = one block over all of F
            if (ord == 0 || ft >= f) {
                if (ord == 0) run(sddmm_pair_kernel<FW, 0, 0, NP>);
                else run(sddmm_pair_kernel<FW, 1, 0, NP>);
            } else if (ft == 32) run(sddmm_pair_kernel<FW, 1, 32, NP>);
            else if (ft == 64) run(sddmm_pair_kernel<FW, 1, 64, NP>);
            else run(sddmm_pair_kernel<FW, 1, 128, NP>);
        };
        if (f == 32 || f == 64) {
            auto pair1 = [&](auto fc) {
                constexpr int F = decltype(fc)::value;
                const std::uint64_t wb = Pair1Shape<F>::kWarpBytes;
                const int kWarps = 4;
                auto run = [&](auto kernel) {
                    const std::size_t smem = std::size_t(wb * kWarps);
                    const int per_sm = kernel_setup(kernel, smem, int(kWarps * 32));
                    const std::uint64_t pairs = (c_end - c_begin + 1) / 2;
                    const std::uint64_t want = (pairs + kWarps - 1) / kWarps;
                    const std::uint64_t cap = std::uint64_t(sms) * std::max(per_sm, 1);
                    const unsigned blocks = unsigned(std::max<std::uint64_t>(1, std::min(want, cap)));
                    kernel<<<blocks, kWarps * 32, smem, s>>>(g.rowptr.get(), g.colind.get(), g.chunk_row.get(),
                                                             g.n_rows, g.xwide.get(), y, out, g.nnz, f, c_begin,
                                                             c_end, finite, keep_y, g.n_cols);
                    check_launch("sddmm_pair_kernel");
                };
                // F=32 stages 8.7 KB per warp, so shared memory admits more than 3
                // CTAs; 4 (<= 128 registers) measured 1.378 -> 1.221 ms on Reddit-shape
                // (5: 1.236).  F=64 (17.4 KB per warp) stays at 3, the shared-memory
                // limit.  AUTOSAGE_DEV_SDDMM_MINB=3/4/5 overrides at F=32 (A/B knob).
                const int minb = F == 32 ? dev_knob("AUTOSAGE_DEV_SDDMM_MINB", 4) : 3;
                if (ord == 0) {
                    if (minb == 4) run(sddmm_pair1_kernel<F, 0, 0, false, 4>);
                    else if (minb == 5) run(sddmm_pair1_kernel<F, 0, 0, false, 5>);
                    else run(sddmm_pair1_kernel<F, 0, 0>);
                } else if (minb == 4) {
                    if (ft >= f) run(sddmm_pair1_kernel<F, 1, 0, false, 4>);
                    else run(sddmm_pair1_kernel<F, 1, 32, false, 4>);
                } else if (ft >= f) run(sddmm_pair1_kernel<F, 1, 0>);
                else run(sddmm_pair1_kernel<F, 1, 32>);
            };
            if (f == 32) pair1(std::integral_constant<int, 32>{});
            else pair1(std::integral_constant<int, 64>{});
        } else if (f == kPairOddF) {
            // 27.2 KB per warp: 2 CTAs of 4 warps per SM
            constexpr int F = int(kPairOddF);
            const std::uint64_t wb = Pair1Shape<F>::kWarpBytes;
            const int kWarps = 4;
            auto run = [&](auto kernel) {
                const std::size_t smem = std::size_t(wb * kWarps);
                const int per_sm = kernel_setup(kernel, smem, int(kWarps * 32));
                const std::uint64_t pairs = (c_end - c_begin + 1) / 2;
                const std::uint64_t want = (pairs + kWarps - 1) / kWarps;
                const std::uint64_t cap = std::uint64_t(sms) * std::max(per_sm, 1);
                const unsigned blocks = unsigned(std::max<std::uint64_t>(1, std::min(want, cap)));
                const double* xop = x_widened_in_kernel(f) ? reinterpret_cast<const double*>(x) : g.xwide.get();
                kernel<<<blocks, kWarps * 32, smem, s>>>(g.rowptr.get(), g.colind.get(), g.chunk_row.get(),
                                                         g.n_rows, xop, y, out, g.nnz, f, c_begin, c_end,
                                                         finite, keep_y, g.n_cols);
                check_launch("sddmm_pair_kernel");
            };
            if (x_widened_in_kernel(f)) {
                if (ord == 0) run(sddmm_pair1_kernel<F, 0, 0, kWtF32, 2, true>);
                else if (ft >= f) run(sddmm_pair1_kernel<F, 1, 0, kWtF32, 2, true>);
                else if (ft == 32) run(sddmm_pair1_kernel<F, 1, 32, kWtF32, 2, true>);
                else run(sddmm_pair1_kernel<F, 1, 64, kWtF32, 2, true>);
            } else {
                if (ord == 0) run(sddmm_pair1_kernel<F, 0, 0, kWtF32, 2>);
                else if (ft >= f) run(sddmm_pair1_kernel<F, 1, 0, kWtF32, 2>);
                else if (ft == 32) run(sddmm_pair1_kernel<F, 1, 32, kWtF32, 2>);
                else run(sddmm_pair1_kernel<F, 1, 64, kWtF32, 2>);
            }
        } else if (pass_major(g, f, ft, ord)) {
            // one launch per 64-feature pass (PassArgs): the slice of Y a
            // pass gathers fits the L2 where the whole Y does not
            const int npass = int(f / 64);
            g.sddmm_state.ensure(std::max<std::uint64_t>(g.nnz, 1));
            const int keep_slice = int(std::uint64_t(g.n_cols) * 64 * 4 <= kKeepMaxBytes) | x_policy_bits();
            const int kWarps = 4;
            const std::size_t smem = std::size_t(Pair1Shape<64>::kWarpBytes * kWarps);
            auto run = [&](auto kernel) {
                const int per_sm = kernel_setup(kernel, smem, int(kWarps * 32));
                const std::uint64_t pairs = (c_end - c_begin + 1) / 2;
                const std::uint64_t want = (pairs + kWarps - 1) / kWarps;
                const std::uint64_t cap = std::uint64_t(sms) * std::max(per_sm, 1);
                const unsigned blocks = unsigned(std::max<std::uint64_t>(1, std::min(want, cap)));
                for (int p = 0; p < npass; ++p) {
                    PassArgs pa;
                    pa.ld = f;
                    pa.f0 = std::uint32_t(p * 64);
                    pa.state = g.sddmm_state.get();
                    pa.last = p == npass - 1;
                    kernel<<<blocks, kWarps * 32, smem, s>>>(g.rowptr.get(), g.colind.get(), g.chunk_row.get(),
                                                             g.n_rows, g.xwide.get(), y, out, g.nnz, c_begin, c_end,
                                                             finite, keep_slice, g.n_cols, pa);
                    check_launch("sddmm_pair1_pm_kernel");
                }
            };
            if (ord == 0) run(sddmm_pair1_pm_kernel<0, 0>);
            else if (ft == 32) run(sddmm_pair1_pm_kernel<1, 32>);
            else run(sddmm_pair1_pm_kernel<1, 0>);  // ft 64: one block per pass
        } else {
            pair(std::integral_constant<int, 64>{}, std::integral_constant<int, 0>{});
        }
        return;
    }
    using I = std::integral_constant<int, 1>;
    using R = std::integral_constant<int, 0>;
    switch (f) {  // single-pass widths compile F in; the rest loop over passes
    case 16: by_fw(std::integral_constant<int, 16>{}, I{}); break;
    case 32: by_fw(std::integral_constant<int, 32>{}, I{}); break;
    case 64: by_fw(std::integral_constant<int, 64>{}, I{}); break;
    default:
        switch (fixed_fw(f)) {
        case 16: by_fw(std::integral_constant<int, 16>{}, R{}); break;
        case 32: by_fw(std::integral_constant<int, 32>{}, R{}); break;
        default: by_fw(std::integral_constant<int, 64>{}, R{}); break;
        }
    }
}

void launch_direct(Graph& g, const float* x, const float* y, std::uint32_t f, std::uint32_t ft, int ord,
                   float* out, cudaStream_t s, std::uint64_t c_begin, std::uint64_t c_end) {
    const unsigned blocks = unsigned(((c_end - c_begin) * 32 + 255) / 256);
    if (ord == 0)
        sddmm_direct_kernel<0><<<blocks, 256, 0, s>>>(g.rowptr.get(), g.colind.get(), g.chunk_row.get(), x, y,
                                                      out, g.nnz, c_begin, c_end, f, ft);
    else
        sddmm_direct_kernel<1><<<blocks, 256, 0, s>>>(g.rowptr.get(), g.colind.get(), g.chunk_row.get(), x, y,
                                                      out, g.nnz, c_begin, c_end, f, ft);
    check_launch("sddmm_direct_kernel");
}

} // namespace

void launch_sddmm_baseline(Graph& g, const float* x, const float* y, std::uint32_t f, float* out,
                           cudaStream_t s, std::uint64_t c_begin, std::uint64_t c_end) {
    if (g.nnz == 0) return;
    ensure_chunk_rows(g);
    c_end = std::min(c_end, (g.nnz + 31) / 32);
    if (c_begin >= c_end) return;
    launch_direct(g, x, y, f, f ? f : 1, 0, out, s, c_begin, c_end);
}

void sddmm_chunks_prepare(Graph& g, const float* x, const float* y, std::uint32_t f,
                          std::uint64_t f_tile, bool vec, cudaStream_t s, const unsigned* finite,
                          std::uint64_t r0, std::uint64_t r1) {
    if (g.nnz == 0 || f == 0) return;
    ensure_chunk_rows(g);
    const std::uint32_t ft = std::uint32_t(effective_tile(f_tile, f));
    if (fixed_eligible(x, y, f, ft, vec ? 1 : 0) && !x_widened_in_kernel(f))
        widen_x(g, x, f, s, dev_knob("AUTOSAGE_DEV_SDDMM_MIX", 1) ? finite : nullptr, r0, r1);
}

void launch_sddmm_chunks(Graph& g, const float* x, const float* y, std::uint32_t f, float* out,
                         std::uint64_t f_tile, bool vec, std::uint32_t wpb, cudaStream_t s,
                         const unsigned* finite, std::uint64_t c_begin, std::uint64_t c_end,
                         bool prepare) {
    if (g.nnz == 0) return;
    ensure_chunk_rows(g);
    const std::uint32_t ft = std::uint32_t(effective_tile(f_tile, f));
    const int ord = vec ? 1 : 0;
    c_end = std::min(c_end, (g.nnz + 31) / 32);
    if (c_begin >= c_end) return;
    if (f == 0) {
        // empty dot products: the reference writes 0.0f for every entry
        const std::uint64_t e0 = c_begin * 32, e1 = std::min(c_end * 32, g.nnz);
        ASB_CUDA(cudaMemsetAsync(out + e0, 0, (e1 - e0) * 4, s));
        return;
    }
    if (fixed_eligible(x, y, f, ft, ord)) {
        const unsigned* fin = dev_knob("AUTOSAGE_DEV_SDDMM_MIX", 1) ? finite : nullptr;
        if (prepare && !x_widened_in_kernel(f)) widen_x(g, x, f, s, fin);
        launch_sddmm_fixed(g, x, y, f, out, ft, ord, s, fin, c_begin, c_end);
        return;
    }
    const bool vload = vec;  // vec4 gate already applied by dispatch
    const bool vlds = vload && (ord == 0 || ft % 4 == 0);
    const std::uint32_t S = vload ? 4 * ((f / 4) | 1u) : (f | 1u);
    const int allow_mix = dev_knob("AUTOSAGE_DEV_SDDMM_MIX", 0);
    const std::uint64_t per_warp = warp_slice_bytes(f, S);
    constexpr std::uint64_t kSmemMax = 200 * 1024;
    wpb = std::clamp<std::uint32_t>(wpb, 1, 16);
    while (wpb > 1 && per_warp * wpb > kSmemMax) --wpb;
    if (per_warp > kSmemMax) {
        launch_direct(g, x, y, f, ft, ord, out, s, c_begin, c_end);
        return;
    }
    const std::size_t smem = std::size_t(per_warp * wpb);
    const int sms = sm_count();
    auto go = [&](auto kernel) {
        const int per_sm = kernel_setup(kernel, smem, int(wpb * 32));
        const std::uint64_t want = (c_end - c_begin + wpb - 1) / wpb;
        const std::uint64_t cap = std::uint64_t(sms) * std::max(per_sm, 1);
        const unsigned blocks = unsigned(std::max<std::uint64_t>(1, std::min(want, cap)));
        kernel<<<blocks, wpb * 32, smem, s>>>(g.rowptr.get(), g.colind.get(), g.chunk_row.get(), g.n_rows,
                                              x, y, out, g.nnz, c_begin, c_end, f, S, ft, finite, allow_mix);
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

// SDDMM on 16-bit X and Y (half.cuh: bf16 or f16): the pair
// kernel with 16-bit Y staging for F in {32, 64} (16-byte aligned operands,
// blocks that line up), the direct kernel otherwise.  ord/ft as in
// launch_sddmm_chunks; the result is the f32 SDDMM on float(X), float(Y) bit
// for bit.
template <int WT>
void launch_sddmm_half_t(Graph& g, const std::uint16_t* x, const std::uint16_t* y, std::uint32_t f, float* out,
                         std::uint32_t ft, int ord, bool baseline, cudaStream_t s) {
    if (g.nnz == 0) return;
    ensure_chunk_rows(g);
    const std::uint64_t c_end = (g.nnz + 31) / 32;
    if (f == 0) {
        ASB_CUDA(cudaMemsetAsync(out, 0, g.nnz * 4, s));
        return;
    }
    // element type of the direct kernel's generic loops: ushort = bf16, f16w = half
    using ET = typename std::conditional<WT == kWtF16, f16w, unsigned short>::type;
    const auto* xs = reinterpret_cast<const ET*>(x);
    const auto* ys = reinterpret_cast<const ET*>(y);
    const bool pair_ok = !baseline && (f == 32 || f == 64) && aligned16(x) && aligned16(y) &&
                         (ord == 0 || ft >= f || ft == 32) && dev_knob("AUTOSAGE_DEV_SDDMM_PAIR", 1);
    if (!pair_ok) {
        const unsigned blocks = unsigned((c_end * 32 + 255) / 256);
        if (ord == 0)
            sddmm_direct_kernel<0><<<blocks, 256, 0, s>>>(g.rowptr.get(), g.colind.get(), g.chunk_row.get(), xs, ys,
                                                          out, g.nnz, 0, c_end, f, ft);
        else
            sddmm_direct_kernel<1><<<blocks, 256, 0, s>>>(g.rowptr.get(), g.colind.get(), g.chunk_row.get(), xs, ys,
                                                          out, g.nnz, 0, c_end, f, ft);
        check_launch("sddmm_direct_kernel");
        return;
    }
    const unsigned* fin = nullptr;
    // scanned at any size, as the f32 SDDMM's Y (engine.cpp mix_flag)
    if (dev_knob("AUTOSAGE_DEV_SDDMM_MIX", 1)) fin = finite_flag_half(g, y, g.n_cols * f, s, WT);
    g.xwide.ensure(std::max<std::uint64_t>(g.n_rows * f, 1));
    const std::uint64_t n4 = g.n_rows * f / 4;
    if (n4) {
        const unsigned wb = unsigned(std::min<std::uint64_t>((n4 + 255) / 256, std::uint64_t(sm_count()) * 8));
        widen_half_kernel<WT><<<std::max(wb, 1u), 256, 0, s>>>(reinterpret_cast<const uint2*>(x),
                                                           reinterpret_cast<double2*>(g.xwide.get()), n4, fin,
                                                           mix_all());
        check_launch("widen_half_kernel");
    }
    const int sms = sm_count();
    auto pair1 = [&](auto fc) {
        constexpr int F = decltype(fc)::value;
        const std::uint64_t wbytes = Pair1Shape<F, WT != kWtF32>::kWarpBytes;
        const int kWarps = 4;
        auto run = [&](auto kernel) {
            const std::size_t smem = std::size_t(wbytes * kWarps);
            const int per_sm = kernel_setup(kernel, smem, int(kWarps * 32));
            const std::uint64_t pairs = (c_end + 1) / 2;
            const std::uint64_t want = (pairs + kWarps - 1) / kWarps;
            const std::uint64_t cap = std::uint64_t(sms) * std::max(per_sm, 1);
            const unsigned blocks = unsigned(std::max<std::uint64_t>(1, std::min(want, cap)));
            kernel<<<blocks, kWarps * 32, smem, s>>>(g.rowptr.get(), g.colind.get(), g.chunk_row.get(), g.n_rows,
                                                     g.xwide.get(), y, out, g.nnz, f, 0, c_end, fin,
                                                     int(std::uint64_t(g.n_cols) * f * 2 <= kKeepMaxBytes) |
                                                         x_policy_bits(),
                                                     g.n_cols);
            check_launch("sddmm_pair_kernel");
        };
        // 4 resident CTAs (<= 128 registers): Reddit-shape F=32 1.32 -> 1.16 ms,
        // F=64 2.03 -> 1.95 ms against 3; 5 (96 registers) is slower at F=64
        const int minb = dev_knob("AUTOSAGE_DEV_SDDMM_BF16_MINB", 4);
        if (ord == 0) {
            if (minb == 3) run(sddmm_pair1_kernel<F, 0, 0, WT, 3>);
            else if (minb == 5) run(sddmm_pair1_kernel<F, 0, 0, WT, 5>);
            else run(sddmm_pair1_kernel<F, 0, 0, WT, 4>);
        } else if (ft >= f) run(sddmm_pair1_kernel<F, 1, 0, WT, 4>);
        else run(sddmm_pair1_kernel<F, 1, 32, WT, 4>);
    };
    if (f == 32) pair1(std::integral_constant<int, 32>{});
    else pair1(std::integral_constant<int, 64>{});
}

void launch_sddmm_half(Graph& g, const std::uint16_t* x, const std::uint16_t* y, std::uint32_t f, float* out,
                       std::uint32_t ft, int ord, bool baseline, cudaStream_t s, int wt) {
    if (wt == kWtF16) launch_sddmm_half_t<kWtF16>(g, x, y, f, out, ft, ord, baseline, s);
    else launch_sddmm_half_t<kWtBF16>(g, x, y, f, out, ft, ord, baseline, s);
}

} // namespace asb
