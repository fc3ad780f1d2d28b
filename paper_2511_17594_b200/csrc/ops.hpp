// ops.hpp -- kernel launchers (device pointers, one stream) used by the
// dispatch layer and the scheduler.
#pragma once

#include "graph.hpp"

namespace asb {

// ---- SpMM (src/kernels.cpp:210-334) ------------------------------------
// K1: warp per row, lane per feature, scalar loads, natural row order.
// b: f32, or 16-bit words when wt != 0 (half.cuh: 1 bf16, 2 f16; every
// kernel reads B through an exact -> f32 step, so the result is the f32
// result on float(B) bit for bit)
void launch_spmm_baseline(Graph& g, const float* val, const void* b, std::uint32_t f, float* c, cudaStream_t s,
                          int wt = 0);
// K2: row groups over rows in degree-descending order; f_tile splits the
// feature dimension into independent work items; wpb warps per CTA.
// Rows order[offset, offset+n_list) of the degree-descending order; rows of
// degree >= 2048 among them go to the CTA-per-row cp.async ring kernel on a
// forked stream (same numerics).
void launch_spmm_rows(Graph& g, const float* val, std::uint64_t offset, std::uint64_t n_list,
                      const void* b, std::uint32_t f, float* c, std::uint64_t f_tile, bool vec,
                      std::uint32_t wpb, cudaStream_t s, const unsigned* finite = nullptr,
                      const float* rmax = nullptr, const double* rsum = nullptr, int wt = 0);
// K3: hub split -- light rows via K2 plus 2048-nnz pieces with ordered
// fp64 partial reduction.
void launch_spmm_hubsplit(Graph& g, const float* val, const void* b, std::uint32_t f, float* c,
                          std::uint64_t f_tile, bool vec, std::uint32_t wpb,
                          std::uint64_t hub_threshold, cudaStream_t s,
                          const unsigned* finite = nullptr, const float* rmax = nullptr,
                          const double* rsum = nullptr, int wt = 0);
// Softmax mode of K2/K3 (rmax != nullptr): `val` holds each entry's ex =
// f32(exp(score - max)) from launch_row_softmax_stats and each entry's value
// is p_e = sm_prob(ex, rsum[row]) (softmax.cuh), computed by the loading lane
// -- the SpMM half of the fused attention, bit-equal to SpMM over
// row_softmax's output.

// ---- SDDMM (src/kernels.cpp:336-429) -----------------------------------
// order: 0 = sequential (scalar variants and the baseline), 1 = per-f_tile
// four-way partial sums (vec variants, src/kernels.cpp:103-127).
// [c_begin, c_end): range of 32-entry chunks (entries 32*c_begin ..
// min(32*c_end, nnz)); the host-buffer pipeline launches slices of it so
// that the D2H of each slice overlaps the next slice's kernel.
constexpr std::uint64_t kAllChunks = ~0ull;
void launch_sddmm_baseline(Graph& g, const float* x, const float* y, std::uint32_t f, float* out,
                           cudaStream_t s, std::uint64_t c_begin = 0, std::uint64_t c_end = kAllChunks);
// prepare = run the per-call prepass (X widening of the fixed-width path);
// slices after the first pass false (sddmm_chunks_prepare runs it alone).
void launch_sddmm_chunks(Graph& g, const float* x, const float* y, std::uint32_t f, float* out,
                         std::uint64_t f_tile, bool vec, std::uint32_t wpb, cudaStream_t s,
                         const unsigned* finite = nullptr, std::uint64_t c_begin = 0,
                         std::uint64_t c_end = kAllChunks, bool prepare = true);
// rows [r0, r1) of X only (the host pipeline streams X in row slices)
void sddmm_chunks_prepare(Graph& g, const float* x, const float* y, std::uint32_t f,
                          std::uint64_t f_tile, bool vec, cudaStream_t s, const unsigned* finite,
                          std::uint64_t r0 = 0, std::uint64_t r1 = ~0ull);

// SDDMM on 16-bit X, Y words (wt: 1 bf16, 2 f16; half.cuh): ord 0
// sequential, 1 the four-way vec blocks of width ft; baseline = the direct
// kernel (guardrail mapping)
void launch_sddmm_half(Graph& g, const std::uint16_t* x, const std::uint16_t* y, std::uint32_t f, float* out,
                       std::uint32_t ft, int ord, bool baseline, cudaStream_t s, int wt);

// Device flag: 1 iff p[0..n) has no Inf/NaN (gates the re-bias widening,
// widen.cuh).  Written into g.flag (one flag per graph; a graph handle runs
// one operator at a time).
const unsigned* finite_flag(Graph& g, const float* p, std::uint64_t n, cudaStream_t s);
// the same over n 16-bit words of type wt (1 bf16, 2 f16)
const unsigned* finite_flag_half(Graph& g, const std::uint16_t* p, std::uint64_t n, cudaStream_t s, int wt);

// ---- row softmax (src/kernels.cpp:431-461) ----------------------------
void launch_row_softmax(Graph& g, const float* vin, float* vout, cudaStream_t s);
// per-row (max, sum) and per-entry ex (fused attention; ex must not alias
// vin); rows of degree 0 are not written
void launch_row_softmax_stats(Graph& g, const float* vin, float* ex, float* rmax, double* rsum, cudaStream_t s);

// ---- backward (backward.cu) ----------------------------
// dst[k] = src[perm[k]]
void launch_permute(const float* src, const std::uint32_t* perm, std::uint64_t n, float* dst,
                    cudaStream_t s);
// ds = p * (g - sum_row p*g), f64 dot in a fixed strided/tree order
void launch_row_softmax_backward(Graph& g, const float* p, const float* grad, float* ds, cudaStream_t s);

// ---- calibration (src/device.cpp:42-95 analogue) ------------------------
double measure_gpu_bandwidth(int device);
double measure_gpu_flops(int device);

} // namespace asb
