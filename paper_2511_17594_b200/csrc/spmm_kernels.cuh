// spmm_kernels.cuh -- the lane-group SpMM kernel template (K2/K3) and its
// argument block, shared by spmm.cu (f32 B) and the translation units that
// instantiate its bf16 (spmm_bf16.cu) and permuted-value (spmm_vp.cu)
// variants, so the three compile in parallel.  Numerics: see spmm.cu.
#pragma once

#include "ops.hpp"
#include "dcheck.cuh"
#include "half.cuh"
#include "l2hint.cuh"
#include "softmax.cuh"
#include "widen.cuh"

#include <algorithm>
#include <cstdlib>
#include <string>
#include <type_traits>

namespace asb {

// kernel argument block (named namespace: the launch entry points of the
// other translation units take it)
struct SegArgs {
    const std::uint64_t* rowptr;
    const std::uint32_t* colind;
    const float* val;
    const void* b;                    // f32, or 16-bit words (half.cuh) when wt != 0
    float* c;
    double* scratch;
    const std::uint32_t* rowlist;     // row mode: row ids (nullptr: identity)
    const std::uint32_t* piece_row;   // piece mode
    const std::uint64_t* piece_e0;
    const std::uint32_t* piece_len;
    const std::uint32_t* piece_slot;
    const unsigned* finite;           // device flag: B has no Inf/NaN (nullable)
    const std::uint32_t* vperm;       // values in source order: entry e reads val[vperm[e]] (nullable)
    const float* rmax;                // softmax mode (non-null): val holds each entry's ex from
    const double* rsum;               // the stats pass, p_e = sm_prob(ex, row sum) (softmax.cuh)
    int off32;                        // n_cols * f < 2^32: 32-bit element offsets
    int wt;                           // B word type (half.cuh): 0 f32, 1 bf16, 2 f16
    int keep_b;                       // B fits L2 (kKeepMaxBytes): gathers evict_last
    int tile_major;                   // items numbered tile-major (n_tiles > 1)
    std::uint64_t n_items;
    std::uint64_t n_rows, n_cols, nnz;  // bounds of the checked build (dcheck.cuh)
    std::uint32_t n_tiles;
    std::uint32_t f;
    std::uint32_t tile_w;
};

namespace {

constexpr unsigned FULL = 0xffffffffu;
// carried-state slot flags of the column-blocked SpMM (CARRY mode)
constexpr std::uint32_t kCarryFirst = 1u << 30, kCarryFinal = 1u << 31, kCarrySlotMask = (1u << 30) - 1;

#ifndef ASB_SEG_E64_MAXLPR
#define ASB_SEG_E64_MAXLPR 16  // widest lane group that takes the 8-byte entry (A/B build knob)
#endif
constexpr int kSegMaxS = 8;  // max entries per lane per fast-loop block (seg_smem)

// Load type of VEC consecutive B elements: f32 (float / float4) or, for the
// 16-bit word types (WT, half.cuh), raw words: ushort / uint2 (8-byte loads
// for 4 features) / uint4 (8 features).
template <int VEC, int WT = kWtF32>
struct VecT;
template <>
struct VecT<1, kWtF32> {
    using T = float;
};
template <>
struct VecT<4, kWtF32> {
    using T = float4;
};
template <int WT>
struct VecT<1, WT> {
    using T = unsigned short;
};
template <int WT>
struct VecT<4, WT> {
    using T = uint2;
};
template <int WT>
struct VecT<8, WT> {
    using T = uint4;
};

template <int WT>
__device__ __forceinline__ float comp(const float& v, int) { return v; }
template <int WT>
__device__ __forceinline__ float comp(const float4& v, int q) {
    return q == 0 ? v.x : (q == 1 ? v.y : (q == 2 ? v.z : v.w));
}
// 16-bit words -> f32 is exact (half.cuh), so every later widening and
// product is the f32 path's on float(B)
template <int WT>
__device__ __forceinline__ float comp(const unsigned short& h, int) { return half_to_f32<WT>(h); }
template <int WT>
__device__ __forceinline__ float comp(const uint2& w, int q) {
    const unsigned x = q < 2 ? w.x : w.y;
    return (q & 1) ? half_hi<WT>(x) : half_lo<WT>(x);
}
template <int WT>
__device__ __forceinline__ float comp(const uint4& w, int q) {
    const unsigned x = q < 2 ? w.x : (q < 4 ? w.y : (q < 6 ? w.z : w.w));
    return (q & 1) ? half_hi<WT>(x) : half_lo<WT>(x);
}

[[maybe_unused]] __host__ __device__ constexpr int unroll_for(int vec, int nch) {
    return vec >= 4 ? (nch == 1 ? 4 : (nch == 2 ? 2 : 1)) : (nch >= 8 ? 1 : 8 / nch);
}

[[maybe_unused]] __host__ __device__ constexpr int maxreg_for(int vec, int nch) {
    // float4 single-chunk tiles at 64 registers (32 warps/SM): 48 spilled the
    // 4 in-flight entries and cost Reddit-shape 2.35 -> 2.41 ms (hubsplit) and
    // 3.24 -> 4.01 ms (rowparallel); wider tiles keep their loads in registers
    // bf16 8-wide tiles (uint4 = 8 features per lane) carry 8 f64 accumulators per chunk
    return vec == 1 ? (nch == 1 ? 64 : (nch == 2 ? 96 : 128))
                    : (vec == 8 ? (nch == 1 ? 96 : 128) : (nch == 1 ? 64 : (nch == 2 ? 80 : 128)));
}


// acc[ch][q] += v * B component, one DFMA each, with MIX's widening split
// first component of a VEC-wide load re-biased on the ALU (MIX): f32 float4
// splits half/half with the XU's F2F; a bf16 component's re-bias is two ALU
// ops (its low mantissa word is zero), so bf16 loads put 3/4 on the ALU (an
// f16 word is first converted to f32, then split like f32)
template <int VEC, int WT>
#ifndef ASB_SEG_MIX_FROM
#define ASB_SEG_MIX_FROM 2  // f32 float4 tiles: components [MIX_FROM, 4) re-biased on the ALU (A/B build knob)
#endif
__host__ __device__ constexpr int mix_from() {
    return VEC == 1 ? 0 : (WT == kWtBF16 ? VEC / 4 : (WT == kWtF32 ? ASB_SEG_MIX_FROM : 2));
}

template <int VEC, int NCH, int MIX, class VT, int MQ = mix_from<VEC, kWtF32>(), int WT = kWtF32>
__device__ __forceinline__ void seg_accumulate(double (&acc)[NCH][VEC], double v, const VT (&bv)[NCH]) {
    const double vu = MIX ? v * kWidenUp : v;
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
        for (int q = 0; q < VEC; ++q) {
            if (MIX && q >= MQ)
                acc[ch][q] = __fma_rn(vu, widen_scaled(comp<WT>(bv[ch], q)), acc[ch][q]);
            else
                acc[ch][q] = __fma_rn(v, double(comp<WT>(bv[ch], q)), acc[ch][q]);
        }
}

// One group of LPR lanes owns one (segment, feature tile) item; segment =
// a whole row (row mode) or a hub piece (PIECES).  MIX selects the widening
// of B: 0 = F2F only, 1 = components 2,3 of each float4 (or every scalar)
// re-biased on the ALU pipe.  SMX: the entry values are softmax
// probabilities computed from the stats pass's ex and the row's sum by the
// lane that loads them (fused attention), instead of stored values.
// CARRY (column-blocked SpMM, spmm_blocked.cu): every item is a segment
// with an f64 state slot; the accumulators start from scratch[slot] instead
// of 0.0 and are written back there, so a row's entries can be consumed in
// ascending column blocks across launches with the reference's order.  Slot
// flags (kCarryFirst: the segment's first block -- start from 0.0, nothing
// to load; kCarryFinal: the last block of a single-segment row -- round into
// C instead of storing the state) keep the carried traffic to one store and
// one load per block boundary.
template <int VEC, int LPR, int NCH, bool HAS_VAL, bool PIECES, int U, int MIX, bool SMX, int WT, bool VP,
          bool CARRY = false>
__device__ __forceinline__ void seg_body(const SegArgs& a) {
    using VT = typename VecT<VEC, WT>::T;
    using BT = typename std::conditional<WT != kWtF32, unsigned short, float>::type;
    constexpr int GPW = 32 / LPR;
    constexpr int W = LPR > U ? LPR : U;
    constexpr int S = W / LPR;
    // the fast loop walks W-entry blocks U entries at a time (a U that does
    // not divide W read past the block: the removed 6-wide dev tunings)
    static_assert(W % U == 0, "entries in flight must divide the block");
    const int lane = threadIdx.x & 31;
    const int grp = lane / LPR;
    const int gl = lane % LPR;
    const std::uint64_t warp = (std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const std::uint64_t item = warp * GPW + grp;
    const bool active = item < a.n_items;

    std::uint32_t row = 0, tile = 0, deg = 0, slot = 0xffffffffu;
    std::uint64_t e0 = 0;
    if (active) {
        std::uint64_t si = item;
        if (a.n_tiles != 1) {
            if (a.tile_major) {
                // feature tile outermost: the grid sweeps every row's tile 0
                // before tile 1, so the B columns in flight (one tile of
                // every gathered row) stay L2-resident at large F
                const std::uint64_t n_seg = a.n_items / a.n_tiles;
                tile = std::uint32_t(item / n_seg);
                si = item - std::uint64_t(tile) * n_seg;
            } else {
                si = item / a.n_tiles;
                tile = std::uint32_t(item - si * a.n_tiles);
            }
        }
        if constexpr (PIECES) {
            row = a.piece_row[si];
            e0 = a.piece_e0[si];
            deg = a.piece_len[si];
            slot = a.piece_slot[si];
        } else {
            row = a.rowlist ? a.rowlist[si] : std::uint32_t(si);
            ASB_DCHECK(row < a.n_rows);
            e0 = a.rowptr[row];
            deg = std::uint32_t(a.rowptr[row + 1] - e0);
        }
        ASB_DCHECK(row < a.n_rows && e0 + deg <= a.nnz);
    }
    std::uint32_t maxdeg = deg;
    if constexpr (GPW > 1) maxdeg = __reduce_max_sync(FULL, deg);
    double rsm = 1.0, rrc = 1.0;
    if constexpr (SMX) {
        if (active && deg) {
            rsm = a.rsum[row];
            rrc = sm_rcp(rsm);
        }
    }

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
    bool carry_final = false;
    if constexpr (CARRY) {
        static_assert(PIECES, "carry mode runs on segment lists");
        const bool carry_first = (slot & kCarryFirst) != 0;
        carry_final = (slot & kCarryFinal) != 0;
        slot &= kCarrySlotMask;
        if (active && !carry_first) {
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch)
                if (fok[ch]) {
                    const double* sp = a.scratch + std::uint64_t(slot) * a.f + fidx[ch];
#pragma unroll
                    for (int q = 0; q < VEC; ++q) acc[ch][q] = sp[q];
                }
        }
    }

    const unsigned gbase = unsigned(grp * LPR);
    const std::uint32_t* colp = a.colind + e0;
    const float* valp = HAS_VAL ? a.val + e0 : nullptr;
    // VP (A^T products of the backward): entry k's value is val[vperm[e0 + k]]
    // (a separate instantiation: a runtime branch here cost the forward kernel ~3%)
    const std::uint32_t* vpp = VP ? a.vperm + e0 : nullptr;
    const BT* __restrict__ bmat = static_cast<const BT*>(a.b);
    // CSR streams once (evict_first); B is re-gathered ~mean-degree times (evict_last)
    const std::uint64_t pol_s = l2_evict_first(), pol_k = l2_reuse_policy(a.keep_b != 0);

    // Fast path: while every group of the warp still has W whole entries
    // left and every lane's features are in range, no predicates at all (a
    // lane-constant feature predicate measured 25% slower: the compiler
    // branches around each entry again); the loading lane pre-multiplies the
    // column by f so each gather address is one IMAD off a per-lane row base.
    // Same entries, same order.
    std::uint32_t base = 0;
    {
        std::uint32_t mindeg = deg;
        if constexpr (GPW > 1) mindeg = __reduce_min_sync(FULL, deg);
        bool lane_full = true;
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) lane_full = lane_full && fok[ch];
        const std::uint32_t fast_end = mindeg / W * W;
        if (a.off32 && fast_end && __all_sync(FULL, lane_full)) {
            const BT* bl[NCH];
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) bl[ch] = bmat + fidx[ch];
            const std::uint32_t f = a.f;
            // (value, offset) of the warp's W*GPW entries go through shared
            // memory: one STS per lane per block and one broadcast LDS per
            // entry, instead of three shuffles per entry (the shuffles held
            // ~40% of the LSU data pipe).  With several groups per warp
            // (LPR <= 16) the entry is 8 bytes (f32 value + offset, LDS.64)
            // and every lane widens the value itself: F=64 rowparallel 2.59 ->
            // 2.29 ms, F=32 1.07 -> 0.97; one group per warp (F >= 128) keeps
            // the 16-byte pre-widened entry (F=128: 4.19 vs 4.37 ms).
            constexpr bool E64 = LPR <= ASB_SEG_E64_MAXLPR;
            using Ent = typename std::conditional<E64, uint2, double2>::type;
            extern __shared__ __align__(16) double2 seg_ent[];
            static_assert(S <= kSegMaxS, "seg_smem too small");
            Ent* ent = reinterpret_cast<Ent*>(seg_ent) + (threadIdx.x >> 5) * (32 * S);
            for (; base < fast_end; base += W) {
                __syncwarp();  // the previous block's readers are done
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const std::uint32_t k = base + std::uint32_t(s * LPR + gl);
                    const std::uint32_t col = ld_stream(colp + k, pol_s);
                    ASB_DCHECK(k < deg && col < a.n_cols);
                    const std::uint32_t o = col * f;
                    float v;
                    if constexpr (SMX) v = sm_prob(ld_stream(valp + k, pol_s), rsm, rrc);
                    else if constexpr (VP) v = __ldg(a.val + ld_stream(vpp + k, pol_s));
                    else if constexpr (HAS_VAL) v = ld_stream(valp + k, pol_s);
                    else v = 1.f;
                    if constexpr (E64) ent[s * 32 + lane] = make_uint2(__float_as_uint(v), o);
                    else ent[s * 32 + lane] = make_double2(double(v), __hiloint2double(0, int(o)));
                }
                __syncwarp();
#pragma unroll
                for (int j0 = 0; j0 < W; j0 += U) {
                    std::uint32_t oj[U];
                    double vj[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int j = j0 + u;
                        const Ent e = ent[(j / LPR) * 32 + int(gbase) + (j % LPR)];
                        if constexpr (E64) {
                            oj[u] = e.y;
                            vj[u] = double(__uint_as_float(e.x));
                        } else {
                            oj[u] = unsigned(__double2loint(e.y));
                            vj[u] = e.x;
                        }
                    }
                    VT bv[U][NCH];
#pragma unroll
                    for (int u = 0; u < U; ++u)
#pragma unroll
                        for (int ch = 0; ch < NCH; ++ch)
                            bv[u][ch] = ld_keep(reinterpret_cast<const VT*>(bl[ch] + oj[u]), pol_k);
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        seg_accumulate<VEC, NCH, MIX, VT, mix_from<VEC, WT>(), WT>(acc, vj[u], bv[u]);
                }
            }
        }
    }

    for (; base < maxdeg; base += W) {
        std::uint32_t cs[S];
        double vs[S];  // widened once here, by the lane that loaded it
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const std::uint32_t k = base + std::uint32_t(s * LPR + gl);
            const bool ok = k < deg;
            cs[s] = ok ? ld_stream(colp + k, pol_s) : 0u;
            ASB_DCHECK(cs[s] < a.n_cols);
            if constexpr (SMX) vs[s] = ok ? double(sm_prob(ld_stream(valp + k, pol_s), rsm, rrc)) : 0.0;
            else if constexpr (VP) vs[s] = ok ? double(__ldg(a.val + ld_stream(vpp + k, pol_s))) : 0.0;
            else if constexpr (HAS_VAL) vs[s] = ok ? double(ld_stream(valp + k, pol_s)) : 0.0;
            else vs[s] = 1.0;
        }
#pragma unroll
        for (int j0 = 0; j0 < W; j0 += U) {
            if (base + std::uint32_t(j0) >= maxdeg) break;
            std::uint32_t cj[U];
            double vj[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = j0 + u;
                cj[u] = __shfl_sync(FULL, cs[j / LPR], int(gbase) + (j % LPR));
                if constexpr (HAS_VAL) vj[u] = __shfl_sync(FULL, vs[j / LPR], int(gbase) + (j % LPR));
                else vj[u] = 1.0;
            }
            VT bv[U][NCH];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const bool okj = base + std::uint32_t(j0 + u) < deg;
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) {
                    if (okj && fok[ch])
                        bv[u][ch] = ld_keep(reinterpret_cast<const VT*>(
                            bmat + std::uint64_t(cj[u]) * a.f + fidx[ch]), pol_k);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const bool okj = base + std::uint32_t(j0 + u) < deg;
                const double v = vj[u];
                const double vu = MIX ? v * kWidenUp : v;
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) {
                    if (okj && fok[ch]) {
#pragma unroll
                        for (int q = 0; q < VEC; ++q) {
                            const bool rebias = MIX && q >= mix_from<VEC, WT>();
                            if (rebias)
                                acc[ch][q] = __fma_rn(vu, widen_scaled(comp<WT>(bv[u][ch], q)), acc[ch][q]);
                            else
                                acc[ch][q] = __fma_rn(v, double(comp<WT>(bv[u][ch], q)), acc[ch][q]);
                        }
                    }
                }
            }
        }
    }

    if (!active) return;
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
        if (!fok[ch]) continue;
        if (!PIECES || (!CARRY && slot == 0xffffffffu) || carry_final) {
            float* cp = a.c + std::uint64_t(row) * a.f + fidx[ch];
#pragma unroll
            for (int q = 0; q < VEC; ++q) st_stream(cp + q, float(acc[ch][q]), pol_s);
        } else {
            double* sp = a.scratch + std::uint64_t(slot) * a.f + fidx[ch];
#pragma unroll
            for (int q = 0; q < VEC; ++q) sp[q] = acc[ch][q];
        }
    }
}

template <int VEC, int LPR, int NCH, bool HAS_VAL, bool PIECES, int U = unroll_for(VEC, NCH),
          int MAXR = maxreg_for(VEC, NCH), bool SMX = false, int WT = kWtF32, bool VP = false, bool CARRY = false>
__global__ void __launch_bounds__(512) __maxnreg__(MAXR) spmm_seg_kernel(SegArgs a) {
    if (a.finite && *a.finite) seg_body<VEC, LPR, NCH, HAS_VAL, PIECES, U, 1, SMX, WT, VP, CARRY>(a);
    else seg_body<VEC, LPR, NCH, HAS_VAL, PIECES, U, 0, SMX, WT, VP, CARRY>(a);
}

// dynamic shared memory of the lane-group kernels: the fast loop's
// (value, offset) staging, 32 x S double2 per warp (S = max(LPR, U) / LPR
// <= 8, reached by scalar single-lane groups)
inline std::size_t seg_smem(unsigned threads) { return std::size_t(threads / 32) * 32 * kSegMaxS * sizeof(double2); }

}  // namespace

// Lane-group launches of the other translation units: (vec, lanes-per-group,
// chunks) select the instantiation at run time.
void launch_seg_bf16(int vec, int lpr, int nch, const SegArgs& a, bool has_val, bool pieces, unsigned nb,
                     unsigned nt, cudaStream_t s);
void launch_seg_f16(int vec, int lpr, int nch, const SegArgs& a, bool has_val, bool pieces, unsigned nb,
                    unsigned nt, cudaStream_t s);
void launch_seg_vp(int vec, int lpr, int nch, const SegArgs& a, bool pieces, unsigned nb, unsigned nt,
                   cudaStream_t s);

}  // namespace asb
