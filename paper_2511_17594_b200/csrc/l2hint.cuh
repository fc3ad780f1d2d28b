// l2hint.cuh -- L2 eviction-priority hints for the gather kernels.
//
// The CSR arrays (colind, val) and the outputs stream through once, while
// the gathered dense operand (B for SpMM, Y and the widened X for SDDMM) is
// re-read ~500 times per row on Reddit-shape graphs.  Without hints the
// streams evict the operand: ncu counted 2.29 GB of DRAM traffic per SDDMM
// launch against 1.04 GB of compulsory bytes (profiles/r02a_launches.md).
// Streaming accesses carry an L2 evict_first policy, the reused operand
// evict_last (createpolicy, PTX ISA 7.4+).  ASB_L2_HINTS=0 at build time
// turns every hint into the plain access (A/B builds).
#pragma once

#include <cstdint>

#ifndef ASB_L2_HINTS
#define ASB_L2_HINTS 1
#endif

namespace asb {

__device__ __forceinline__ std::uint64_t l2_evict_first() {
    std::uint64_t p = 0;
#if ASB_L2_HINTS
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
#endif
    return p;
}

__device__ __forceinline__ std::uint64_t l2_evict_last() {
    std::uint64_t p = 0;
#if ASB_L2_HINTS
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
#endif
    return p;
}

__device__ __forceinline__ std::uint64_t l2_evict_normal() {
    std::uint64_t p = 0;
#if ASB_L2_HINTS
    asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
#endif
    return p;
}

// evict_last only pays while the reused operand fits the L2 with room for
// the streams: a Products-shape B (980 MB) gathered from DRAM measured 0.4%
// slower with it (profiles/r02d_l2hint_ab.md)
constexpr std::uint64_t kKeepMaxBytes = std::uint64_t(96) << 20;
__device__ __forceinline__ std::uint64_t l2_reuse_policy(bool fits) {
    return fits ? l2_evict_last() : l2_evict_normal();
}

// read-only streaming loads (non-coherent path, like __ldg)
__device__ __forceinline__ std::uint32_t ld_stream(const std::uint32_t* p, std::uint64_t pol) {
#if ASB_L2_HINTS
    std::uint32_t v;
    asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
#else
    (void)pol;
    return __ldg(p);
#endif
}

__device__ __forceinline__ float ld_stream(const float* p, std::uint64_t pol) {
#if ASB_L2_HINTS
    float v;
    asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
#else
    (void)pol;
    return __ldg(p);
#endif
}

template <class T>
__device__ __forceinline__ T ld_keep(const T* p, std::uint64_t pol);
template <>
__device__ __forceinline__ float4 ld_keep<float4>(const float4* p, std::uint64_t pol) {
#if ASB_L2_HINTS
    float4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p), "l"(pol));
    return v;
#else
    (void)pol;
    return __ldg(p);
#endif
}

// the gathered operand: f32 float4 / scalar loads take the evict_last
// policy; the bf16 word types keep the plain read-only load
template <class T>
__device__ __forceinline__ T ld_keep(const T* p, std::uint64_t) {
    return __ldg(p);
}
template <>
__device__ __forceinline__ float ld_keep<float>(const float* p, std::uint64_t pol) {
#if ASB_L2_HINTS
    float v;
    asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
#else
    (void)pol;
    return __ldg(p);
#endif
}

__device__ __forceinline__ void st_stream(float* p, float v, std::uint64_t pol) {
#if ASB_L2_HINTS
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
#else
    (void)pol;
    *p = v;
#endif
}

// f64 carried state of a multi-launch reduction (written by the previous
// launch, so the coherent path)
__device__ __forceinline__ double ld_state(const double* p, std::uint64_t pol) {
#if ASB_L2_HINTS
    double v;
    asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
#else
    (void)pol;
    return *p;
#endif
}

__device__ __forceinline__ void st_state(double* p, double v, std::uint64_t pol) {
#if ASB_L2_HINTS
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
#else
    (void)pol;
    *p = v;
#endif
}

// 16-byte cp.async of a reused row with an L2 policy
__device__ __forceinline__ void cp_async16_pol(void* smem, const void* gmem, std::uint64_t pol) {
    const unsigned s = unsigned(__cvta_generic_to_shared(smem));
#if ASB_L2_HINTS
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "l"(pol)
                 : "memory");
#else
    (void)pol;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
#endif
}

}  // namespace asb
