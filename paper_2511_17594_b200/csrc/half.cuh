// half.cuh -- 16-bit operand words.
//
// Dense operands may arrive as raw 16-bit words of either format:
//   WT 1 = bfloat16  (f32's top 16 bits),
//   WT 2 = binary16  (IEEE half: 1 sign, 5 exponent, 10 mantissa bits).
// Both widen to f32 exactly, so every kernel computes the f32 path's bits on
// float(operand); the gathers read half the bytes.  WT 0 is plain f32.
#pragma once

#include <cuda_fp16.h>

#include <cstdint>

namespace asb {

enum : int { kWtF32 = 0, kWtBF16 = 1, kWtF16 = 2 };

template <int WT>
__device__ __forceinline__ float half_to_f32(unsigned short h) {
    static_assert(WT == kWtBF16 || WT == kWtF16, "16-bit word type");
    if constexpr (WT == kWtBF16) return __uint_as_float(unsigned(h) << 16);
    else return __half2float(__ushort_as_half(h));
}

// the low / high 16-bit word of a 32-bit pair as f32
template <int WT>
__device__ __forceinline__ float half_lo(unsigned x) {
    if constexpr (WT == kWtBF16) return __uint_as_float(x << 16);
    else return half_to_f32<WT>((unsigned short)(x & 0xffffu));
}
template <int WT>
__device__ __forceinline__ float half_hi(unsigned x) {
    if constexpr (WT == kWtBF16) return __uint_as_float(x & 0xffff0000u);
    else return half_to_f32<WT>((unsigned short)(x >> 16));
}

// exponent field all ones = Inf/NaN (the finite scan gating the re-bias widening)
template <int WT>
constexpr unsigned half_inf_mask() {
    return WT == kWtBF16 ? 0x7F80u : 0x7C00u;
}

}  // namespace asb
