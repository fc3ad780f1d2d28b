// spmm_vp.cu -- lane-group SpMM instantiations whose owner lane loads each
// value through a transpose's entry permutation (val[vperm[e]]; the backward's
// A^T products, as_spmm_transpose_values).  f32 B, values present.
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

void launch_seg_vp(int vec, int lpr, int nch, const SegArgs& a, bool pieces, unsigned nb, unsigned nt,
                   cudaStream_t s) {
    auto go = [&](auto vc) {
        constexpr int VEC = decltype(vc)::value;
        by_shape(lpr, nch, [&](auto lc, auto cc) {
            constexpr int LPR = decltype(lc)::value, NCH = decltype(cc)::value;
            constexpr int U = unroll_for(VEC, NCH), R = maxreg_for(VEC, NCH);
            const std::size_t sm = seg_smem(nt);
            if (pieces) spmm_seg_kernel<VEC, LPR, NCH, true, true, U, R, false, false, true><<<nb, nt, sm, s>>>(a);
            else spmm_seg_kernel<VEC, LPR, NCH, true, false, U, R, false, false, true><<<nb, nt, sm, s>>>(a);
        });
    };
    if (vec == 4) go(std::integral_constant<int, 4>{});
    else go(std::integral_constant<int, 1>{});
    check_launch("spmm_seg_kernel");
}

}  // namespace asb
