// spmm.cu -- CSR SpMM kernels for sm_100a.
//
// Numerics (all mappings): each output C[i,f] is a double accumulator that
// adds val[e] * B[col[e], f] for the row's entries in CSR order, one
// rounding per add, then rounds to f32 -- exactly the reference's
// `acc[t] += v * brow[t]` (src/kernels.cpp:63-80, :217-226).  The product
// of two f32 values is exact in f64, so the DFMA below equals the
// reference's separate multiply and add bit for bit.  HubSplit heavy rows
// follow src/kernels.cpp:284-332: 2048-nnz pieces, f64 partials, summed in
// piece order from 0.0.
//
// Performance shape: B gathers dominate (4*F bytes per nnz).  Row groups of
// LPR lanes cover one row's feature tile with float4 (vec) or scalar loads;
// colind/val are fetched cooperatively (one coalesced load per LPR entries)
// and broadcast by shuffle, and U gathers per lane are issued before their
// DFMAs so each warp keeps U*LPR*16 bytes in flight.  Rows are visited in
// degree-descending order (the graph's stable sort), which packs rows of
// equal length into a warp and starts the longest rows first.
#include "ops.hpp"

#include <algorithm>

namespace asb {

namespace {

constexpr unsigned FULL = 0xffffffffu;

template <int VEC>
struct VecT;
template <>
struct VecT<1> {
    using T = float;
};
template <>
struct VecT<4> {
    using T = float4;
};

__device__ __forceinline__ float comp(const float& v, int) { return v; }
__device__ __forceinline__ float comp(const float4& v, int q) {
    return q == 0 ? v.x : (q == 1 ? v.y : (q == 2 ? v.z : v.w));
}

__host__ __device__ constexpr int unroll_for(int vec, int nch) {
    return vec * nch >= 32 ? 1 : (vec * nch >= 16 ? 2 : (vec * nch >= 8 ? 4 : 8));
}

struct SegArgs {
    const std::uint64_t* rowptr;
    const std::uint32_t* colind;
    const float* val;
    const float* b;
    float* c;
    double* scratch;
    const std::uint32_t* rowlist;     // row mode: row ids (nullptr: identity)
    const std::uint32_t* piece_row;   // piece mode when non-null
    const std::uint64_t* piece_e0;
    const std::uint32_t* piece_len;
    const std::uint32_t* piece_slot;
    std::uint64_t n_items;
    std::uint32_t n_tiles;
    std::uint32_t f;
    std::uint32_t tile_w;
};

// K2/K3 gather kernel.  One group of LPR lanes owns one (segment, feature
// tile) item; segment = a whole row (row mode) or a hub piece.
template <int VEC, int LPR, int NCH, bool HAS_VAL>
__global__ void __launch_bounds__(512) spmm_seg_kernel(SegArgs a) {
    using VT = typename VecT<VEC>::T;
    constexpr int GPW = 32 / LPR;
    constexpr int U = unroll_for(VEC, NCH);
    constexpr int W = LPR > U ? LPR : U;
    constexpr int S = W / LPR;
    const int lane = threadIdx.x & 31;
    const int grp = lane / LPR;
    const int gl = lane % LPR;
    const std::uint64_t warp = (std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const std::uint64_t item = warp * GPW + grp;
    const bool active = item < a.n_items;

    std::uint32_t row = 0, tile = 0, deg = 0, slot = 0xffffffffu;
    std::uint64_t e0 = 0;
    if (active) {
        const std::uint64_t si = item / a.n_tiles;
        tile = std::uint32_t(item - si * a.n_tiles);
        if (a.piece_row) {
            row = a.piece_row[si];
            e0 = a.piece_e0[si];
            deg = a.piece_len[si];
            slot = a.piece_slot[si];
        } else {
            row = a.rowlist ? a.rowlist[si] : std::uint32_t(si);
            e0 = a.rowptr[row];
            deg = std::uint32_t(a.rowptr[row + 1] - e0);
        }
    }
    std::uint32_t maxdeg = deg;
    if constexpr (GPW > 1) maxdeg = __reduce_max_sync(FULL, deg);

    const std::uint32_t f0 = tile * a.tile_w;
    const std::uint32_t fend = min(a.f, f0 + a.tile_w);
    std::uint32_t fidx[NCH];
    bool fok[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
        fidx[ch] = f0 + std::uint32_t(ch * LPR + gl) * VEC;
        fok[ch] = active && fidx[ch] < fend;
    }
    double acc[NCH][VEC];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
        for (int q = 0; q < VEC; ++q) acc[ch][q] = 0.0;

    const unsigned gbase = unsigned(grp * LPR);
    const std::uint32_t* colp = a.colind + e0;
    const float* valp = HAS_VAL ? a.val + e0 : nullptr;
    const float* __restrict__ bmat = a.b;

    for (std::uint32_t base = 0; base < maxdeg; base += W) {
        std::uint32_t cs[S];
        float vs[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const std::uint32_t k = base + std::uint32_t(s * LPR + gl);
            const bool ok = k < deg;
            cs[s] = ok ? __ldg(colp + k) : 0u;
            if constexpr (HAS_VAL) vs[s] = ok ? __ldg(valp + k) : 0.f;
            else vs[s] = 1.f;
        }
#pragma unroll
        for (int j0 = 0; j0 < W; j0 += U) {
            if (base + std::uint32_t(j0) >= maxdeg) break;
            std::uint32_t cj[U];
            float vj[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = j0 + u;
                cj[u] = __shfl_sync(FULL, cs[j / LPR], int(gbase) + (j % LPR));
                if constexpr (HAS_VAL) vj[u] = __shfl_sync(FULL, vs[j / LPR], int(gbase) + (j % LPR));
                else vj[u] = 1.f;
            }
            VT bv[U][NCH];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const bool okj = base + std::uint32_t(j0 + u) < deg;
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) {
                    if (okj && fok[ch])
                        bv[u][ch] = __ldg(reinterpret_cast<const VT*>(
                            bmat + std::uint64_t(cj[u]) * a.f + fidx[ch]));
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const bool okj = base + std::uint32_t(j0 + u) < deg;
                const double dv = HAS_VAL ? double(vj[u]) : 1.0;
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) {
                    if (okj && fok[ch]) {
#pragma unroll
                        for (int q = 0; q < VEC; ++q)
                            acc[ch][q] = __fma_rn(dv, double(comp(bv[u][ch], q)), acc[ch][q]);
                    }
                }
            }
        }
    }

    if (!active) return;
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
        if (!fok[ch]) continue;
        if (slot == 0xffffffffu) {
            float* cp = a.c + std::uint64_t(row) * a.f + fidx[ch];
#pragma unroll
            for (int q = 0; q < VEC; ++q) cp[q] = float(acc[ch][q]);
        } else {
            double* sp = a.scratch + std::uint64_t(slot) * a.f + fidx[ch];
#pragma unroll
            for (int q = 0; q < VEC; ++q) sp[q] = acc[ch][q];
        }
    }
}

// K3 epilogue: s = 0.0; s += partial[p] in piece order; C = f32(s)
// (src/kernels.cpp:320-331).
__global__ void hub_reduce_kernel(const std::uint32_t* __restrict__ red_row,
                                  const std::uint32_t* __restrict__ red_first,
                                  const std::uint32_t* __restrict__ red_count, std::uint64_t n_red,
                                  const double* __restrict__ scratch, float* __restrict__ c,
                                  std::uint32_t f) {
    const std::uint64_t total = n_red * f;
    for (std::uint64_t i = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; i < total;
         i += std::uint64_t(gridDim.x) * blockDim.x) {
        const std::uint64_t r = i / f, t = i - r * f;
        const std::uint64_t first = red_first[r], cnt = red_count[r];
        double s = 0.0;
        for (std::uint64_t p = 0; p < cnt; ++p) s = __dadd_rn(s, scratch[(first + p) * f + t]);
        c[std::uint64_t(red_row[r]) * f + t] = float(s);
    }
}

// K1: the guardrail baseline.  Warp per row in natural order, lane per
// feature (NF features per lane per pass), scalar loads, no prefetch.
template <int NF>
__global__ void spmm_baseline_kernel(const std::uint64_t* __restrict__ rowptr,
                                     const std::uint32_t* __restrict__ colind,
                                     const float* __restrict__ val, const float* __restrict__ b,
                                     float* __restrict__ c, std::uint64_t n_rows, std::uint32_t f) {
    const std::uint64_t row = (std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (row >= n_rows) return;
    const int lane = threadIdx.x & 31;
    const std::uint64_t e0 = rowptr[row], e1 = rowptr[row + 1];
    for (std::uint32_t f0 = 0; f0 < f; f0 += 32 * NF) {
        double acc[NF];
#pragma unroll
        for (int q = 0; q < NF; ++q) acc[q] = 0.0;
        for (std::uint64_t e = e0; e < e1; ++e) {
            const float* brow = b + std::uint64_t(colind[e]) * f + f0;
            const double v = val ? double(val[e]) : 1.0;
#pragma unroll
            for (int q = 0; q < NF; ++q) {
                const std::uint32_t t = std::uint32_t(lane + 32 * q);
                if (f0 + t < f) acc[q] = __fma_rn(v, double(brow[t]), acc[q]);
            }
        }
#pragma unroll
        for (int q = 0; q < NF; ++q) {
            const std::uint32_t t = std::uint32_t(lane + 32 * q);
            if (f0 + t < f) c[row * f + f0 + t] = float(acc[q]);
        }
    }
}

template <int VEC, int LPR, int NCH>
void launch_seg(const SegArgs& a, bool has_val, std::uint32_t wpb, cudaStream_t s) {
    constexpr int GPW = 32 / LPR;
    const std::uint64_t groups_per_block = std::uint64_t(wpb) * GPW;
    const std::uint64_t blocks = (a.n_items + groups_per_block - 1) / groups_per_block;
    if (blocks == 0) return;
    if (has_val)
        spmm_seg_kernel<VEC, LPR, NCH, true><<<unsigned(blocks), wpb * 32, 0, s>>>(a);
    else
        spmm_seg_kernel<VEC, LPR, NCH, false><<<unsigned(blocks), wpb * 32, 0, s>>>(a);
    check_launch("spmm_seg_kernel");
}

template <int VEC>
void launch_seg_vec(const SegArgs& a, bool has_val, std::uint32_t lanes, std::uint32_t wpb,
                    cudaStream_t s) {
    if (lanes <= 1) launch_seg<VEC, 1, 1>(a, has_val, wpb, s);
    else if (lanes <= 2) launch_seg<VEC, 2, 1>(a, has_val, wpb, s);
    else if (lanes <= 4) launch_seg<VEC, 4, 1>(a, has_val, wpb, s);
    else if (lanes <= 8) launch_seg<VEC, 8, 1>(a, has_val, wpb, s);
    else if (lanes <= 16) launch_seg<VEC, 16, 1>(a, has_val, wpb, s);
    else if (lanes <= 32) launch_seg<VEC, 32, 1>(a, has_val, wpb, s);
    else if (lanes <= 64) launch_seg<VEC, 32, 2>(a, has_val, wpb, s);
    else if (lanes <= 128) launch_seg<VEC, 32, 4>(a, has_val, wpb, s);
    else launch_seg<VEC, 32, 8>(a, has_val, wpb, s);
}

struct TileShape {
    std::uint32_t tile_w, n_tiles, lanes;
};

// GPU meaning of (f_tile, vec): a work item covers tile_w features; tiles
// are independent items.  Any tiling gives the same bits (per-feature
// accumulation order is always CSR order).
TileShape tile_shape(std::uint32_t f, std::uint64_t f_tile, bool vec) {
    const int v = vec ? 4 : 1;
    std::uint64_t tw = effective_tile(f_tile, f);
    if (vec) tw = (tw + 3) / 4 * 4;                       // keep float4 alignment
    tw = std::min<std::uint64_t>(tw, std::uint64_t(32 * 8 * v));  // at most 8 chunks / lane
    TileShape t;
    t.tile_w = std::uint32_t(std::max<std::uint64_t>(tw, 1));
    t.n_tiles = (f + t.tile_w - 1) / t.tile_w;
    t.lanes = (t.tile_w + v - 1) / v;
    return t;
}

} // namespace

void launch_spmm_baseline(Graph& g, const float* val, const float* b, std::uint32_t f, float* c, cudaStream_t s) {
    if (g.n_rows == 0 || f == 0) return;
    const std::uint64_t threads = g.n_rows * 32;
    const unsigned blocks = unsigned((threads + 255) / 256);
    if (f <= 32)
        spmm_baseline_kernel<1><<<blocks, 256, 0, s>>>(g.rowptr.get(), g.colind.get(), val, b, c,
                                                       g.n_rows, f);
    else if (f <= 64)
        spmm_baseline_kernel<2><<<blocks, 256, 0, s>>>(g.rowptr.get(), g.colind.get(), val, b, c,
                                                       g.n_rows, f);
    else if (f <= 128)
        spmm_baseline_kernel<4><<<blocks, 256, 0, s>>>(g.rowptr.get(), g.colind.get(), val, b, c,
                                                       g.n_rows, f);
    else
        spmm_baseline_kernel<8><<<blocks, 256, 0, s>>>(g.rowptr.get(), g.colind.get(), val, b, c,
                                                       g.n_rows, f);
    check_launch("spmm_baseline_kernel");
}

void launch_spmm_rows(Graph& g, const float* val, const std::uint32_t* rowlist, std::uint64_t n_list, const float* b,
                      std::uint32_t f, float* c, std::uint64_t f_tile, bool vec, std::uint32_t wpb,
                      cudaStream_t s) {
    if (n_list == 0 || f == 0) return;
    const TileShape t = tile_shape(f, f_tile, vec);
    SegArgs a{};
    a.rowptr = g.rowptr.get();
    a.colind = g.colind.get();
    a.val = val;
    a.b = b;
    a.c = c;
    a.rowlist = rowlist;
    a.n_items = n_list * t.n_tiles;
    a.n_tiles = t.n_tiles;
    a.f = f;
    a.tile_w = t.tile_w;
    wpb = std::clamp<std::uint32_t>(wpb, 1, 16);
    if (vec) launch_seg_vec<4>(a, val != nullptr, t.lanes, wpb, s);
    else launch_seg_vec<1>(a, val != nullptr, t.lanes, wpb, s);
}

void launch_spmm_hubsplit(Graph& g, const float* val, const float* b, std::uint32_t f, float* c,
                          std::uint64_t f_tile, bool vec, std::uint32_t wpb,
                          std::uint64_t hub_threshold, cudaStream_t s) {
    if (g.n_rows == 0 || f == 0) return;
    const HubPlan& plan = ensure_hub_plan(g, hub_threshold);
    wpb = std::clamp<std::uint32_t>(wpb, 1, 16);
    const TileShape t = tile_shape(f, f_tile, vec);
    if (plan.n_slots) g.scratch.ensure(plan.n_slots * f);
    if (plan.n_pieces) {
        SegArgs a{};
        a.rowptr = g.rowptr.get();
        a.colind = g.colind.get();
        a.val = val;
        a.b = b;
        a.c = c;
        a.scratch = g.scratch.get();
        a.piece_row = plan.piece_row.get();
        a.piece_e0 = plan.piece_e0.get();
        a.piece_len = plan.piece_len.get();
        a.piece_slot = plan.piece_slot.get();
        a.n_items = plan.n_pieces * t.n_tiles;
        a.n_tiles = t.n_tiles;
        a.f = f;
        a.tile_w = t.tile_w;
        if (vec) launch_seg_vec<4>(a, val != nullptr, t.lanes, wpb, s);
        else launch_seg_vec<1>(a, val != nullptr, t.lanes, wpb, s);
    }
    if (plan.n_light)
        launch_spmm_rows(g, val, plan.light_rows.get(), plan.n_light, b, f, c, f_tile, vec, wpb, s);
    if (plan.n_red) {
        const std::uint64_t total = plan.n_red * f;
        const unsigned blocks = unsigned(std::min<std::uint64_t>((total + 255) / 256, 148 * 32));
        hub_reduce_kernel<<<blocks, 256, 0, s>>>(plan.red_row.get(), plan.red_first.get(),
                                                 plan.red_count.get(), plan.n_red, g.scratch.get(),
                                                 c, f);
        check_launch("hub_reduce_kernel");
    }
}

} // namespace asb
