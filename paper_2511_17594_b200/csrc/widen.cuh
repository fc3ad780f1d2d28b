// widen.cuh -- exact f32 -> f64 widening split across SM pipes.
//
// Every product of the bit-exact f64 accumulation needs its f32 operand
// widened.  The hardware conversion (F2F.F64.F32) issues on the XU pipe at
// 16 lanes/clk/SM, which caps an F=64 gather at ~17 TB/s; tools/
// gather_roofline.cu measures 19.8 TB/s when half of each float4 is widened
// instead by an integer re-bias on the ALU pipe:
//
//   widen_scaled(f) = bits (sign | exp_f | mant_f << 29) as a double
//                   = f * 2^-896        exactly, for every finite f32
//                                        (zero and subnormals included)
//
// The 2^-896 is folded into the other factor (pre-multiplied by 2^896, an
// exact power-of-two scaling that cannot overflow for an f32 magnitude), so
// fma(v * 2^896, widen_scaled(b), acc) == fma(double(v), double(b), acc)
// bit for bit.  Inf/NaN operands do not survive the re-bias, so kernels take
// this path only when a device-side scan (finite_check_kernel) has cleared
// the operand; otherwise the same kernel runs the all-F2F path.
#pragma once

#include <cstdint>

namespace asb {

constexpr double kWidenUp = 0x1p896;

__device__ __forceinline__ double widen_scaled(float f) {
    const int u = __float_as_int(f);
    const unsigned hi = unsigned(u >> 3) & 0x8FFFFFFFu;  // sign | 8-bit exp | mantissa[22:3]
    const unsigned lo = unsigned(u) << 29;               // mantissa[2:0]
    return __hiloint2double(int(hi), int(lo));
}

// MIX = 0: all hardware conversions; MIX = 1: re-bias this operand.
template <int MIX>
__device__ __forceinline__ double widen(float f) {
    if constexpr (MIX) return widen_scaled(f);
    else return double(f);
}


}  // namespace asb
