// spmm_half.cuh -- lane-group SpMM instantiations for a B of 16-bit words
// (half.cuh: bf16 or f16; exact -> f32, so the f32 path's bits on float(B)):
// 1-, 4- and 8-wide tiles, with and without values, rows or hub pieces.
// spmm_bf16.cu and spmm_f16.cu instantiate it, one translation unit each so
// they compile in parallel.
#pragma once

#include "spmm_kernels.cuh"

namespace asb {

namespace {

// (LPR, NCH) pairs the lane-group launcher uses: groups of 1..32 lanes with one
// chunk, and whole warps with 2, 4 or 8 chunks per lane
template <class F>
void by_shape(int lpr, int nch, F&& f) {
    switch (lpr) {
    case 1: f(std::integral_constant<int, 1>{}, std::integral_constant<int, 1>{}); return;
    case 2: f(std::integral_constant<int, 2>{}, std::integral_constant<int, 1>{}); return;
    case 4: f(std::integral_constant<int, 4>{}, std::integral_constant<int, 1>{}); return;
    case 8: f(std::integral_constant<int, 8>{}, std::integral_constant<int, 1>{}); return;
    case 16: f(std::integral_constant<int, 16>{}, std::integral_constant<int, 1>{}); return;
    default: break;
    }
    switch (nch) {
    case 1: f(std::integral_constant<int, 32>{}, std::integral_constant<int, 1>{}); return;
    case 2: f(std::integral_constant<int, 32>{}, std::integral_constant<int, 2>{}); return;
    case 4: f(std::integral_constant<int, 32>{}, std::integral_constant<int, 4>{}); return;
    default: f(std::integral_constant<int, 32>{}, std::integral_constant<int, 8>{}); return;
    }
}

}  // namespace

template <int WT>
void launch_seg_half_t(int vec, int lpr, int nch, const SegArgs& a, bool has_val, bool pieces, unsigned nb,
                       unsigned nt, cudaStream_t s) {
    auto go = [&](auto vc) {
        constexpr int VEC = decltype(vc)::value;
        by_shape(lpr, nch, [&](auto lc, auto cc) {
            constexpr int LPR = decltype(lc)::value, NCH = decltype(cc)::value;
            if constexpr (VEC == 8 && NCH == 8) {
                throw LogicError("8-wide tiles take at most 4 chunks per lane");
            } else {
                // register caps: the 16-bit -> f32 step needs more live registers
                // than the f32 kernels' caps leave in the scalar tiles (they
                // spilled 24-160 B at 64).  Softmax mode keeps the f32 caps: 16
                // more registers there cost the fused 16-bit attention 4%
                // (occupancy), more than its small spills do.
                constexpr int U = unroll_for(VEC, NCH);
                constexpr int R0 = maxreg_for(VEC, NCH);
                constexpr int R = VEC == 1 && R0 < 96 ? 96 : R0;
                constexpr int RS = R;
                const std::size_t sm = seg_smem(nt);
                if (a.rmax) {  // softmax mode (fused attention over 16-bit V): values are the stats pass ex
                    if (!has_val) throw LogicError("spmm softmax mode needs the score values");
                    if (pieces) spmm_seg_kernel<VEC, LPR, NCH, true, true, U, RS, true, WT><<<nb, nt, sm, s>>>(a);
                    else spmm_seg_kernel<VEC, LPR, NCH, true, false, U, RS, true, WT><<<nb, nt, sm, s>>>(a);
                } else if (has_val) {
                    if (pieces) spmm_seg_kernel<VEC, LPR, NCH, true, true, U, R, false, WT><<<nb, nt, sm, s>>>(a);
                    else spmm_seg_kernel<VEC, LPR, NCH, true, false, U, R, false, WT><<<nb, nt, sm, s>>>(a);
                } else {
                    if (pieces) spmm_seg_kernel<VEC, LPR, NCH, false, true, U, R, false, WT><<<nb, nt, sm, s>>>(a);
                    else spmm_seg_kernel<VEC, LPR, NCH, false, false, U, R, false, WT><<<nb, nt, sm, s>>>(a);
                }
            }
        });
    };
    if (vec == 8) go(std::integral_constant<int, 8>{});
    else if (vec == 4) go(std::integral_constant<int, 4>{});
    else go(std::integral_constant<int, 1>{});
    check_launch("spmm_seg_kernel");
}

}  // namespace asb
