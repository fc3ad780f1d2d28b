// spmm_f16.cu -- the lane-group SpMM on an IEEE half B (spmm_half.cuh, WT = f16).
#include "spmm_half.cuh"

namespace asb {

void launch_seg_f16(int vec, int lpr, int nch, const SegArgs& a, bool has_val, bool pieces, unsigned nb,
                    unsigned nt, cudaStream_t s) {
    launch_seg_half_t<kWtF16>(vec, lpr, nch, a, has_val, pieces, nb, nt, s);
}

}  // namespace asb
