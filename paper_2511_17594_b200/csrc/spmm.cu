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
// Performance shape (F=64, Reddit-shaped): B gathers are L2 hits, so the
// budget is the L2 gather rate (~20 TB/s measured, tools/gather_roofline.cu)
// and the XU pipe that widens f32 to f64.  Hence:
//  * the group kernel runs small lane groups (float4 per lane) at high
//    occupancy (register cap), rows in degree-descending order;
//  * each entry's value is widened once by the lane that loaded it and
//    shuffled as f64; half of every B float4 is widened by an exact integer
//    re-bias on the ALU pipe (widen.cuh) when B is known finite;
//  * on small graphs, long rows (degree >= 256) and hub pieces (whose
//    dependent round trips would dominate a lane group) go to a CTA-per-item
//    kernel that streams the gathered B rows through a cp.async
//    shared-memory ring, concurrently on a forked stream.
#include "spmm_kernels.cuh"

#include <algorithm>
#include <cstdlib>
#include <string>
#include <type_traits>

namespace asb {

namespace {

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

// ---------------------------------------------------------------------------
// K2L: one CTA per long row or hub piece with the group kernel's numerics,
// warp-specialized around an mbarrier ring:
//   warp 0 (producer): streams the item's column indices/values into an index
//     ring with 4-byte cp.async (kIdxAhead chunks ahead, so no dependent
//     global load sits on its path), widens the values once into a f64 ring,
//     and gathers each stage's B rows with 16-byte cp.async spread over the
//     warp (whole 128-byte lines per instruction) into a kLongStages-deep
//     shared-memory ring.  A stage's "full" mbarrier counts, per producer
//     lane, one release arrive (its value stores) and one
//     cp.async.mbarrier.arrive.noinc (its copies landed).  One TMA bulk copy
//     per 256-byte row measured ~10% slower (c1 rowparallel 0.13 ms vs 0.116).
//   warps 1.. (consumers): F/FPL threads each run FPL f64 chains in CSR order
//     out of shared memory, then release the stage on its "empty" mbarrier.
// No __syncthreads in the steady state; a stage holds ch B rows.  Bit-equal
// to the group kernel.
// Ring shape (-D overridable for sweeps): 4 stages of 16 KB (64 rows of F=64
// per stage, 256 entries in flight per row).  Each stage costs a producer/
// consumer mbarrier round trip and the producer's cp.async group wait, so
// fewer, larger stages win on the
// c1 long rows (hub-split SpMM 0.101 -> 0.074 ms; 8 x 4 KB, 8 x 8 KB, 12 x
// 8 KB, 6 x 12 KB, 8 x 16 KB measured in profiles/r02g_c1_ring.md).
#ifndef ASB_LONG_STAGES
#define ASB_LONG_STAGES 4
#endif
#ifndef ASB_LONG_STAGE_BYTES
#define ASB_LONG_STAGE_BYTES 16384
#endif
#ifndef ASB_LONG_IDX_AHEAD
#define ASB_LONG_IDX_AHEAD 3
#endif
constexpr int kLongStages = ASB_LONG_STAGES;
constexpr std::uint32_t kLongStageBytes = ASB_LONG_STAGE_BYTES;
constexpr int kIdxAhead = ASB_LONG_IDX_AHEAD;
constexpr int kIdxRing = 2 * ASB_LONG_IDX_AHEAD;
static_assert(kIdxRing > kIdxAhead, "index ring too small");
constexpr int kLongMaxConsumers = 256;  // consumer threads; features beyond loop

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return unsigned(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void mbar_init(std::uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(std::uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "LONGROW_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra LONGROW_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

struct LongLayout {
    std::uint32_t ring_off, vd_off, cidx_off, vidx_off, bar_off, total;
};
__host__ __device__ inline LongLayout long_layout(std::uint32_t f, std::uint32_t ch) {
    LongLayout L{};
    std::uint32_t o = 0;
    L.ring_off = o;
    o += std::uint32_t(kLongStages) * ch * f * 4;  // B rows
    o = (o + 15) & ~15u;
    L.vd_off = o;
    o += std::uint32_t(kLongStages) * ch * 8;  // widened values
    L.cidx_off = o;
    o += std::uint32_t(kIdxRing) * ch * 4;  // column index ring
    L.vidx_off = o;
    o += std::uint32_t(kIdxRing) * ch * 4;  // value ring (f32)
    o = (o + 15) & ~15u;
    L.bar_off = o;
    o += 2 * kLongStages * 8;  // full + empty mbarriers
    L.total = o;
    return L;
}

template <int FPL>
struct LongVec;
template <>
struct LongVec<1> {
    using T = float;
};
template <>
struct LongVec<2> {
    using T = float2;
};
template <>
struct LongVec<4> {
    using T = float4;
};
__device__ __forceinline__ float long_comp(float v, int) { return v; }
__device__ __forceinline__ float long_comp(float2 v, int i) { return i == 0 ? v.x : v.y; }
__device__ __forceinline__ float long_comp(float4 v, int i) {
    return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

// Row mode: item = a.rowlist[blockIdx.x]; piece mode: hub piece blockIdx.x,
// written to its f64 partial slot (or straight to C when it is the row's
// only piece) exactly like the lane-group piece path.
template <int MIX, bool HAS_VAL, int FPL, bool PIECES, bool SMX>
__device__ __forceinline__ void longrow_body(const SegArgs& A, std::uint32_t ch, char* smem) {
    const std::uint64_t* __restrict__ rowptr = A.rowptr;
    const std::uint32_t* __restrict__ colind = A.colind;
    const float* __restrict__ val = A.val;
    const float* __restrict__ b = static_cast<const float*>(A.b);
    float* __restrict__ c = A.c;
    const std::uint32_t f = A.f;
    constexpr int S = kLongStages;
    const LongLayout L = long_layout(f, ch);
    float* ring = reinterpret_cast<float*>(smem + L.ring_off);
    double* vd = reinterpret_cast<double*>(smem + L.vd_off);
    std::uint32_t* cidx = reinterpret_cast<std::uint32_t*>(smem + L.cidx_off);
    float* vidx = reinterpret_cast<float*>(smem + L.vidx_off);
    std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + L.bar_off);
    std::uint64_t* empty = full + S;
    const std::uint32_t n_cons_warps = (blockDim.x >> 5) - 1;

    std::uint32_t row, deg, slot = 0xffffffffu;
    std::uint64_t e0;
    if constexpr (PIECES) {
        row = A.piece_row[blockIdx.x];
        e0 = A.piece_e0[blockIdx.x];
        deg = A.piece_len[blockIdx.x];
        slot = A.piece_slot[blockIdx.x];
    } else {
        row = A.rowlist[blockIdx.x];
        ASB_DCHECK(row < A.n_rows);
        e0 = rowptr[row];
        deg = std::uint32_t(rowptr[row + 1] - e0);
    }
    ASB_DCHECK(row < A.n_rows && e0 + deg <= A.nnz);
    const std::uint32_t nchunks = (deg + ch - 1) / ch;
    const int warp = int(threadIdx.x >> 5), lane = int(threadIdx.x & 31);
    double rsm = 1.0, rrc = 1.0;
    if constexpr (SMX) {
        rsm = A.rsum[row];
        rrc = sm_rcp(rsm);
    }

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 64);  // per producer lane: values written + its copies landed
            mbar_init(&empty[s], n_cons_warps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    if (warp == 0) {
        // ---------------- producer warp ----------------
        const std::uint32_t per_row = f / 4;  // 16-byte units per B row
        const std::uint32_t dj = 32 / per_row, dq = 32 % per_row;
        const std::uint32_t j0 = std::uint32_t(lane) / per_row, q0 = std::uint32_t(lane) % per_row;
        auto issue_idx = [&](std::uint32_t k) {
            if (k < nchunks) {
                const std::uint32_t base = k * ch, n = min(ch, deg - base);
                std::uint32_t* cd = cidx + (k % kIdxRing) * ch;
                float* vdst = vidx + (k % kIdxRing) * ch;
                for (std::uint32_t j = lane; j < n; j += 32) {
                    cp_async4(cd + j, colind + e0 + base + j);
                    if constexpr (HAS_VAL) cp_async4(vdst + j, val + e0 + base + j);
                }
            }
            cp_async_commit();  // one group per call keeps the wait count uniform
        };
        for (int k = 0; k < kIdxAhead; ++k) issue_idx(std::uint32_t(k));
        for (std::uint32_t k = 0; k < nchunks; ++k) {
            issue_idx(k + kIdxAhead);
            cp_async_wait<kIdxAhead>();  // chunk k's indices are in (this lane's copies)
            __syncwarp();                // ... and visible to the whole warp
            const int s = int(k % S);
            if (k >= std::uint32_t(S)) mbar_wait(&empty[s], ((k / S) - 1) & 1);
            const std::uint32_t n = min(ch, deg - k * ch);
            const std::uint32_t* cs = cidx + (k % kIdxRing) * ch;
            const float* vs = vidx + (k % kIdxRing) * ch;
            double* vdst = vd + std::uint64_t(s) * ch;
            for (std::uint32_t j = lane; j < n; j += 32)
                vdst[j] = SMX ? double(sm_prob(vs[j], rsm, rrc)) : (HAS_VAL ? double(vs[j]) : 1.0);
            __syncwarp();
            mbar_arrive(&full[s]);  // release: this lane's value stores
            // the stage's B rows as 16-byte cp.async pieces spread over the
            // warp (whole 128-byte lines per instruction); each lane's
            // arrive fires when its own copies have landed
            float* dst = ring + std::uint64_t(s) * ch * f;
            // piece p = lane + 32 i -> (row j, 16-byte unit qq), stepped
            // incrementally (no division in the loop)
            std::uint32_t j = j0, qq = q0;
            for (std::uint32_t pidx = lane; pidx < n * per_row; pidx += 32) {
                ASB_DCHECK(j < n && cs[j] < A.n_cols);
                cp_async16(dst + j * f + 4 * qq, b + std::uint64_t(cs[j]) * f + 4 * qq);
                j += dj;
                qq += dq;
                if (qq >= per_row) {
                    qq -= per_row;
                    ++j;
                }
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&full[s]))
                         : "memory");
        }
        cp_async_wait<0>();
        return;
    }

    // ---------------- consumer warps ----------------
    // thread q owns features [FPL*q, FPL*q + FPL): FPL independent f64 chains
    // fed by one FPL-wide LDS per entry; the entry value is a broadcast f64
    // read.  FPL is chosen so a row's features fill whole warps (F=64: 32
    // lanes x 2), which minimises instructions per entry.
    using VT = typename LongVec<FPL>::T;
    const std::uint32_t q = threadIdx.x - 32;
    const std::uint32_t nq = f / FPL;
    const bool active = q < nq;
    double acc[FPL];
#pragma unroll
    for (int i = 0; i < FPL; ++i) acc[i] = 0.0;
    for (std::uint32_t k = 0; k < nchunks; ++k) {
        const int s = int(k % S);
        mbar_wait(&full[s], (k / S) & 1);
        const std::uint32_t n = min(ch, deg - k * ch);
        if (active) {
            const VT* src = reinterpret_cast<const VT*>(ring + std::uint64_t(s) * ch * f) + q;
            const double* vv = vd + std::uint64_t(s) * ch;
#pragma unroll 4
            for (std::uint32_t j = 0; j < n; ++j) {
                const double v = vv[j];
                const VT bv = src[std::uint64_t(j) * nq];
#pragma unroll
                for (int i = 0; i < FPL; ++i) {
                    const float bi = long_comp(bv, i);
                    // odd components widen by re-bias when MIX (half the F2F)
                    if (MIX && (i & 1)) acc[i] = __fma_rn(v * kWidenUp, widen_scaled(bi), acc[i]);
                    else acc[i] = __fma_rn(v, double(bi), acc[i]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (active) {  // scalar stores: c need not be aligned beyond 4 bytes
        if (PIECES && slot != 0xffffffffu) {
            double* pr = A.scratch + std::uint64_t(slot) * f + FPL * q;
#pragma unroll
            for (int i = 0; i < FPL; ++i) pr[i] = acc[i];
        } else {
            float* cr = c + std::uint64_t(row) * f + FPL * q;
#pragma unroll
            for (int i = 0; i < FPL; ++i) cr[i] = float(acc[i]);
        }
    }
}

template <bool HAS_VAL, int FPL, bool PIECES, bool SMX = false>
__global__ void __launch_bounds__(32 + kLongMaxConsumers) spmm_longrow_kernel(SegArgs a, std::uint32_t ch) {
    extern __shared__ __align__(16) char lsmem[];
    if (a.finite && *a.finite) longrow_body<1, HAS_VAL, FPL, PIECES, SMX>(a, ch, lsmem);
    else longrow_body<0, HAS_VAL, FPL, PIECES, SMX>(a, ch, lsmem);
}

// Launch the ring kernel over n items (rows of a.rowlist, or hub pieces).
template <bool PIECES>
void launch_longrow(const SegArgs& a, std::uint64_t n, cudaStream_t s) {
    const std::uint32_t f = a.f;
    const std::uint32_t ch = std::max<std::uint32_t>(4, kLongStageBytes / (4 * f));
    const std::size_t smem = long_layout(f, ch).total;
    // features per consumer lane.  The ring kernel only runs when its items
    // are few (small graphs' long rows, a handful of hub pieces), so it is
    // latency-bound: each consumer warp advances its chains one entry per
    // ~6 instructions, and more warps per row shorten the longest row.  One
    // feature per lane while f fits kLongMaxConsumers (c1 F=64: 2 consumer
    // warps instead of 1, 73 -> see profiles/r02g_c1_fpl.md); the old
    // warp-filling choice (F=64 -> 2 per lane) via AUTOSAGE_DEV_LONG_FPL=2.
    static const int fpl_knob = [] {
        const char* e = std::getenv("AUTOSAGE_DEV_LONG_FPL");
        return e ? std::atoi(e) : 0;
    }();
    int fpl = f <= std::uint32_t(kLongMaxConsumers) ? 1 : (f <= 2u * kLongMaxConsumers ? 2 : 4);
    if (fpl_knob == 1 || fpl_knob == 2 || fpl_knob == 4) fpl = std::max(fpl, fpl_knob);
    const unsigned threads = 32 + (f / fpl + 31) / 32 * 32;
    auto go = [&](auto kern) {
        kernel_setup(kern, smem, int(threads));
        kern<<<unsigned(n), threads, smem, s>>>(a, ch);
        check_launch("spmm_longrow_kernel");
    };
    auto by_val = [&](auto fc) {
        constexpr int FPL = decltype(fc)::value;
        if (a.rmax) go(spmm_longrow_kernel<true, FPL, PIECES, true>);
        else if (a.val) go(spmm_longrow_kernel<true, FPL, PIECES>);
        else go(spmm_longrow_kernel<false, FPL, PIECES>);
    };
    if (fpl == 1) by_val(std::integral_constant<int, 1>{});
    else if (fpl == 2) by_val(std::integral_constant<int, 2>{});
    else by_val(std::integral_constant<int, 4>{});
}

// The ring kernel handles f % 4 == 0 with 16-byte B rows (bulk copies).
bool longrow_ok(std::uint32_t f, bool vec) {
    if (!(vec && f % 4 == 0 && f <= 4 * kLongMaxConsumers)) return false;
    const std::uint32_t ch = std::max<std::uint32_t>(4, kLongStageBytes / (4 * f));
    return long_layout(f, ch).total <= 200 * 1024;
}

// ---------------------------------------------------------------------------
// K1: the guardrail baseline.  Warp per row in natural order, lane per
// feature (NF features per lane per pass), scalar loads, no prefetch.
template <int NF, class BT = float, int WT = kWtF32>
__global__ void spmm_baseline_kernel(const std::uint64_t* __restrict__ rowptr,
                                     const std::uint32_t* __restrict__ colind,
                                     const float* __restrict__ val, const BT* __restrict__ b,
                                     float* __restrict__ c, std::uint64_t n_rows, std::uint32_t f,
                                     const std::uint32_t* __restrict__ vperm = nullptr) {
    const std::uint64_t row = (std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (row >= n_rows) return;
    const int lane = threadIdx.x & 31;
    const std::uint64_t e0 = rowptr[row], e1 = rowptr[row + 1];
    for (std::uint32_t f0 = 0; f0 < f; f0 += 32 * NF) {
        double acc[NF];
#pragma unroll
        for (int q = 0; q < NF; ++q) acc[q] = 0.0;
        for (std::uint64_t e = e0; e < e1; ++e) {
            const BT* brow = b + std::uint64_t(colind[e]) * f + f0;
            const double v = val ? double(val[vperm ? vperm[e] : e]) : 1.0;
#pragma unroll
            for (int q = 0; q < NF; ++q) {
                const std::uint32_t t = std::uint32_t(lane + 32 * q);
                if (f0 + t < f) acc[q] = __fma_rn(v, double(comp<WT>(brow[t], 0)), acc[q]);
            }
        }
#pragma unroll
        for (int q = 0; q < NF; ++q) {
            const std::uint32_t t = std::uint32_t(lane + 32 * q);
            if (f0 + t < f) c[row * f + f0 + t] = float(acc[q]);
        }
    }
}


// developer tuning knob (AUTOSAGE_DEV_SPMM_TUNE=<U>x<MAXR>) for the F=64
// shapes; default = the tuned constants above
int dev_tune() {
    static const int t = [] {
        const char* e = std::getenv("AUTOSAGE_DEV_SPMM_TUNE");
        if (!e) return 0;
        const std::string v(e);
        if (v == "2x40") return 1;
        if (v == "4x40") return 2;
        if (v == "4x48") return 3;
        if (v == "8x48") return 4;
        if (v == "8x64") return 5;
        if (v == "8x128") return 6;
        if (v == "2x48") return 7;
        if (v == "4x56") return 8;
        if (v == "4x64") return 9;
        if (v == "8x80") return 12;
        if (v == "8x96") return 13;
        if (v == "4x72") return 14;
        return 0;
    }();
    return t;
}

template <int VEC, int LPR, int NCH, bool HV, bool PC>
void launch_tuned(const SegArgs& a, unsigned blocks, unsigned threads, cudaStream_t s) {
    if constexpr (VEC == 4 && NCH == 1 && (LPR == 16 || LPR == 8) && HV) {
        switch (dev_tune()) {
            case 1: spmm_seg_kernel<VEC, LPR, NCH, HV, PC, 2, 40><<<blocks, threads, seg_smem(threads), s>>>(a); return;
            case 2: spmm_seg_kernel<VEC, LPR, NCH, HV, PC, 4, 40><<<blocks, threads, seg_smem(threads), s>>>(a); return;
            case 3: spmm_seg_kernel<VEC, LPR, NCH, HV, PC, 4, 48><<<blocks, threads, seg_smem(threads), s>>>(a); return;
            case 4: spmm_seg_kernel<VEC, LPR, NCH, HV, PC, 8, 48><<<blocks, threads, seg_smem(threads), s>>>(a); return;
            case 5: spmm_seg_kernel<VEC, LPR, NCH, HV, PC, 8, 64><<<blocks, threads, seg_smem(threads), s>>>(a); return;
            case 6: spmm_seg_kernel<VEC, LPR, NCH, HV, PC, 8, 128><<<blocks, threads, seg_smem(threads), s>>>(a); return;
            case 7: spmm_seg_kernel<VEC, LPR, NCH, HV, PC, 2, 48><<<blocks, threads, seg_smem(threads), s>>>(a); return;
            case 8: spmm_seg_kernel<VEC, LPR, NCH, HV, PC, 4, 56><<<blocks, threads, seg_smem(threads), s>>>(a); return;
            case 9: spmm_seg_kernel<VEC, LPR, NCH, HV, PC, 4, 64><<<blocks, threads, seg_smem(threads), s>>>(a); return;
            case 12: spmm_seg_kernel<VEC, LPR, NCH, HV, PC, 8, 80><<<blocks, threads, seg_smem(threads), s>>>(a); return;
            case 13: spmm_seg_kernel<VEC, LPR, NCH, HV, PC, 8, 96><<<blocks, threads, seg_smem(threads), s>>>(a); return;
            case 14: spmm_seg_kernel<VEC, LPR, NCH, HV, PC, 4, 72><<<blocks, threads, seg_smem(threads), s>>>(a); return;
            default: break;
        }
    }
    spmm_seg_kernel<VEC, LPR, NCH, HV, PC><<<blocks, threads, seg_smem(threads), s>>>(a);
}

// Warps per CTA of the lane-group kernels.  The reference's rows_per_chunk
// (a CPU parallel_for grain) has no GPU meaning that changes results; one
// CTA of 1 warp caps residency at 32 warps/SM and 16 warps gives coarse
// tails, so every rpc runs 4 warps (measured best on Reddit-shape, see
// DESIGN.md).  AUTOSAGE_DEV_SPMM_WPB overrides for experiments.
std::uint32_t warps_per_cta(std::uint32_t /*rpc*/) {
    static const int knob = [] {
        const char* e = std::getenv("AUTOSAGE_DEV_SPMM_WPB");
        return e ? std::atoi(e) : 0;
    }();
    return knob > 0 ? std::uint32_t(std::min(knob, 16)) : 4u;
}

template <int VEC, int LPR, int NCH>
void launch_seg(const SegArgs& a, bool has_val, std::uint32_t wpb, cudaStream_t s) {
    constexpr int GPW = 32 / LPR;
    const std::uint64_t groups_per_block = std::uint64_t(wpb) * GPW;
    const std::uint64_t blocks = (a.n_items + groups_per_block - 1) / groups_per_block;
    if (blocks == 0) return;
    const bool pieces = a.piece_row != nullptr;
    const unsigned nb = unsigned(blocks), nt = wpb * 32;
    // the permuted-value (spmm_vp.cu) and bf16 (spmm_bf16.cu) instantiations
    // live in their own translation units so the three compile in parallel
    if (a.vperm) {  // values read through a transpose permutation (f32 B, values present)
        if (VEC == 8 || a.wt || a.rmax || !has_val)
            throw LogicError("spmm: permuted values take f32 B and values");
        launch_seg_vp(VEC, LPR, NCH, a, pieces, nb, nt, s);
        return;
    }
    if (VEC == 8 || a.wt) {  // 16-bit B (bf16 / f16): default tuning (softmax mode included)
        if (a.wt == kWtF16) launch_seg_f16(VEC, LPR, NCH, a, has_val, pieces, nb, nt, s);
        else launch_seg_bf16(VEC, LPR, NCH, a, has_val, pieces, nb, nt, s);
        return;
    }
    if constexpr (VEC == 8) {
        throw LogicError("8-wide SpMM tiles are bf16-only");
    } else if (a.rmax) {  // softmax mode (fused attention): float4 tiles only
        if constexpr (VEC == 4) {
            if (pieces) spmm_seg_kernel<VEC, LPR, NCH, true, true, unroll_for(VEC, NCH), maxreg_for(VEC, NCH), true><<<nb, nt, seg_smem(nt), s>>>(a);
            else spmm_seg_kernel<VEC, LPR, NCH, true, false, unroll_for(VEC, NCH), maxreg_for(VEC, NCH), true><<<nb, nt, seg_smem(nt), s>>>(a);
        } else {
            throw LogicError("spmm softmax mode needs float4 tiles");
        }
    } else if (has_val) {
        if (pieces) launch_tuned<VEC, LPR, NCH, true, true>(a, nb, nt, s);
        else launch_tuned<VEC, LPR, NCH, true, false>(a, nb, nt, s);
    } else {
        if (pieces) launch_tuned<VEC, LPR, NCH, false, true>(a, nb, nt, s);
        else launch_tuned<VEC, LPR, NCH, false, false>(a, nb, nt, s);
    }
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
    else if constexpr (VEC == 8) throw LogicError("8-wide tiles take at most 4 chunks per lane");
    else launch_seg<VEC, 32, 8>(a, has_val, wpb, s);
}

struct TileShape {
    std::uint32_t tile_w, n_tiles, lanes;
};

// GPU meaning of (f_tile, vec): a work item covers tile_w features; tiles
// are independent items.  Any tiling gives the same bits (per-feature
// accumulation order is always CSR order).
// vec8: bf16 B with f % 8 == 0 and a 16-byte base (uint4 = 8 features per
// lane).  Below f = 64 the 4-wide tiles keep more lanes per row in flight
// (Reddit-shape F=32: 0.90 ms 4-wide vs 1.10 ms 8-wide; F=64: 1.72 vs 1.56;
// F=128: 3.80 vs 3.29).
bool vec8_ok(const void* b, std::uint32_t f, bool vec, int wt) {
    return wt != kWtF32 && vec && f >= 64 && f % 8 == 0 && (reinterpret_cast<std::uintptr_t>(b) & 15) == 0;
}

TileShape tile_shape(std::uint32_t f, std::uint64_t f_tile, bool vec, bool vec8 = false) {
    const int v = vec8 ? 8 : (vec ? 4 : 1);
    std::uint64_t tw = effective_tile(f_tile, f);
    if (vec) tw = (tw + v - 1) / v * v;                             // keep the vector alignment
    // at most 8 chunks per lane (4 for the 8-wide tiles: 8 f64 accumulators each)
    tw = std::min<std::uint64_t>(tw, std::uint64_t(32 * (v == 8 ? 4 : 8) * v));
    TileShape t;
    t.tile_w = std::uint32_t(std::max<std::uint64_t>(tw, 1));
    t.n_tiles = (f + t.tile_w - 1) / t.tile_w;
    t.lanes = (t.tile_w + v - 1) / v;
    return t;
}

// AUTOSAGE_DEV_TILE_MAJOR=0: items row-major (the round-1 numbering; A/B knob)
int tile_major() {
    static const int v = [] {
        const char* e = std::getenv("AUTOSAGE_DEV_TILE_MAJOR");
        return e ? std::atoi(e) : 1;
    }();
    return v;
}

// 32-bit gather offsets (col * f) fit; AUTOSAGE_DEV_SPMM_NOFAST=1 disables
// the predicate-free fast loop (developer A/B knob)
int fast_gather_ok(const Graph& g, std::uint32_t f) {
    static const bool off = [] {
        const char* e = std::getenv("AUTOSAGE_DEV_SPMM_NOFAST");
        return e && std::atoi(e) != 0;
    }();
    return !off && std::uint64_t(g.n_cols) * f < (std::uint64_t(1) << 32);
}

// Rows at least this long go to the CTA-per-row ring kernel.  In the
// lane-group kernel a row is a chain of dependent L2 round trips (U entries
// in flight), so on a small graph its longest rows set the kernel time; on
// a large graph other rows hide them and the group kernel's throughput wins
// (Reddit-shape: 4.10 ms without the ring kernel, 4.34 ms from 2048).
std::uint64_t long_row_min(const Graph& g) {
    static const long long knob = [] {
        const char* e = std::getenv("AUTOSAGE_DEV_LONG_ROW");
        return e ? std::strtoll(e, nullptr, 10) : -1ll;
    }();
    if (knob >= 0) return std::uint64_t(knob);
    const std::uint64_t n = g.plan_nnz ? g.plan_nnz : g.nnz;
    return n < (std::uint64_t(16) << 20) ? 256 : 1ull << 62;
}

} // namespace

void launch_spmm_baseline(Graph& g, const float* val, const void* bv, std::uint32_t f, float* c,
                          cudaStream_t s, int wt) {
    if (g.n_rows == 0 || f == 0) return;
    const std::uint64_t threads = g.n_rows * 32;
    const unsigned blocks = unsigned((threads + 255) / 256);
    if (wt != kWtF32) {
        const auto* b = static_cast<const unsigned short*>(bv);
        auto go = [&](auto wc) {
            constexpr int W = decltype(wc)::value;
            if (f <= 32)
                spmm_baseline_kernel<1, unsigned short, W><<<blocks, 256, 0, s>>>(g.rowptr.get(), g.colind.get(), val, b, c, g.n_rows, f, g.val_perm);
            else if (f <= 64)
                spmm_baseline_kernel<2, unsigned short, W><<<blocks, 256, 0, s>>>(g.rowptr.get(), g.colind.get(), val, b, c, g.n_rows, f, g.val_perm);
            else
                spmm_baseline_kernel<4, unsigned short, W><<<blocks, 256, 0, s>>>(g.rowptr.get(), g.colind.get(), val, b, c, g.n_rows, f, g.val_perm);
        };
        if (wt == kWtF16) go(std::integral_constant<int, kWtF16>{});
        else go(std::integral_constant<int, kWtBF16>{});
        check_launch("spmm_baseline_kernel");
        return;
    }
    const auto* b = static_cast<const float*>(bv);
    if (f <= 32)
        spmm_baseline_kernel<1><<<blocks, 256, 0, s>>>(g.rowptr.get(), g.colind.get(), val, b, c, g.n_rows, f, g.val_perm);
    else if (f <= 64)
        spmm_baseline_kernel<2><<<blocks, 256, 0, s>>>(g.rowptr.get(), g.colind.get(), val, b, c, g.n_rows, f, g.val_perm);
    else if (f <= 128)
        spmm_baseline_kernel<4><<<blocks, 256, 0, s>>>(g.rowptr.get(), g.colind.get(), val, b, c, g.n_rows, f, g.val_perm);
    else
        spmm_baseline_kernel<8><<<blocks, 256, 0, s>>>(g.rowptr.get(), g.colind.get(), val, b, c, g.n_rows, f, g.val_perm);
    check_launch("spmm_baseline_kernel");
}

void launch_spmm_rows(Graph& g, const float* val, std::uint64_t offset, std::uint64_t n_list,
                      const void* b, std::uint32_t f, float* c, std::uint64_t f_tile, bool vec,
                      std::uint32_t wpb, cudaStream_t s, const unsigned* finite, const float* rmax,
                      const double* rsum, int wt) {
    if (rmax) vec = true;  // softmax mode runs float4 tiles (same numerics, engine gates f % 4)
    if (n_list == 0 || f == 0) return;
    ensure_order(g);
    // long rows (a prefix of the degree-descending order) -> CTA-per-row ring
    // kernel on a forked stream, concurrent with the group kernel
    const std::uint64_t lmin = long_row_min(g);
    std::uint64_t n_long = 0;
    if (lmin > 0 && !wt && !g.val_perm && longrow_ok(f, vec)) {
        const std::uint64_t ge = rows_with_degree_at_least(g, lmin);
        n_long = ge > offset ? std::min(ge - offset, n_list) : 0;
    }
    if (n_long) {
        SegArgs a{};
        a.rowptr = g.rowptr.get();
        a.colind = g.colind.get();
        a.val = val;
        a.vperm = g.val_perm;
        a.b = b;
        a.c = c;
        a.rowlist = g.order.get() + offset;
        a.finite = finite;
        a.rmax = rmax;
        a.rsum = rsum;
        a.f = f;
        a.n_rows = g.n_rows;
        a.n_cols = g.n_cols;
        a.nnz = g.nnz;
        a.off32 = fast_gather_ok(g, f);
        launch_longrow<false>(a, n_long, graph_fork(g, s));
        offset += n_long;
        n_list -= n_long;
    }
    if (n_list) {
        const bool v8 = vec8_ok(b, f, vec, wt);
        const TileShape t = tile_shape(f, f_tile, vec, v8);
        SegArgs a{};
        a.rowptr = g.rowptr.get();
        a.colind = g.colind.get();
        a.val = val;
        a.vperm = g.val_perm;
        a.b = b;
        a.c = c;
        a.rowlist = g.order.get() + offset;
        a.finite = finite;
        a.rmax = rmax;
        a.rsum = rsum;
        a.n_items = n_list * t.n_tiles;
        a.n_tiles = t.n_tiles;
        a.f = f;
        a.n_rows = g.n_rows;
        a.n_cols = g.n_cols;
        a.nnz = g.nnz;
        a.off32 = fast_gather_ok(g, f);
        a.wt = wt;
        a.keep_b = std::uint64_t(g.n_cols) * f * (wt ? 2 : 4) <= kKeepMaxBytes;
        a.tile_major = tile_major();
        a.tile_w = t.tile_w;
        wpb = warps_per_cta(wpb);
        if (v8) launch_seg_vec<8>(a, val != nullptr, t.lanes, wpb, s);
        else if (vec) launch_seg_vec<4>(a, val != nullptr, t.lanes, wpb, s);
        else launch_seg_vec<1>(a, val != nullptr, t.lanes, wpb, s);
    }
    if (n_long) graph_join(g, s);
}

void launch_spmm_hubsplit(Graph& g, const float* val, const void* b, std::uint32_t f, float* c,
                          std::uint64_t f_tile, bool vec, std::uint32_t wpb,
                          std::uint64_t hub_threshold, cudaStream_t s, const unsigned* finite,
                          const float* rmax, const double* rsum, int wt) {
    if (g.n_rows == 0 || f == 0) return;
    if (rmax) vec = true;
    const HubPlan& plan = ensure_hub_plan(g, hub_threshold);
    wpb = warps_per_cta(wpb);
    const bool v8 = vec8_ok(b, f, vec, wt);
    const TileShape t = tile_shape(f, f_tile, vec, v8);
    if (plan.n_slots) g.scratch.ensure(plan.n_slots * f);
    // light rows on the forked stream, concurrent with the pieces: their
    // blocks fill the SMs the pieces kernel's last wave leaves idle
    static const bool concurrent = [] {
        const char* e = std::getenv("AUTOSAGE_DEV_SPMM_CONCURRENT");
        return e ? std::atoi(e) != 0 : true;
    }();
    // one launch over pieces + light rows (HubPlan::all_*: pieces longest
    // first, then the light rows degree-descending) instead of two kernels on
    // forked streams: one tail instead of two and no fork/join.  Same items,
    // same bits; Products F=100 9.03 -> 8.71 ms, its 8-way shard 1.22 -> 1.19,
    // c4 1.13 -> 1.10, Reddit unchanged (profiles/r02z_merged.md).
    // AUTOSAGE_DEV_SPMM_MERGED=0 restores the two-kernel form, =2 forces the
    // one launch also where the pieces would take the ring kernel (tests).
    const int merged_knob = [] {
        const char* e = std::getenv("AUTOSAGE_DEV_SPMM_MERGED");
        return e ? std::atoi(e) : 1;
    }();
    const bool few_pieces = plan.n_pieces <= std::uint64_t(4) * std::uint64_t(g.sms);
    if (merged_knob && plan.n_pieces && plan.n_light && (!few_pieces || merged_knob == 2)) {
        SegArgs a{};
        a.rowptr = g.rowptr.get();
        a.colind = g.colind.get();
        a.val = val;
        a.vperm = g.val_perm;
        a.b = b;
        a.c = c;
        a.scratch = g.scratch.get();
        a.piece_row = plan.all_row.get();
        a.piece_e0 = plan.all_e0.get();
        a.piece_len = plan.all_len.get();
        a.piece_slot = plan.all_slot.get();
        a.finite = finite;
        a.rmax = rmax;
        a.rsum = rsum;
        a.n_items = (plan.n_pieces + plan.n_light) * t.n_tiles;
        a.n_tiles = t.n_tiles;
        a.f = f;
        a.n_rows = g.n_rows;
        a.n_cols = g.n_cols;
        a.nnz = g.nnz;
        a.off32 = fast_gather_ok(g, f);
        a.wt = wt;
        a.keep_b = std::uint64_t(g.n_cols) * f * (wt ? 2 : 4) <= kKeepMaxBytes;
        a.tile_major = tile_major();
        a.tile_w = t.tile_w;
        if (v8) launch_seg_vec<8>(a, val != nullptr, t.lanes, wpb, s);
        else if (vec) launch_seg_vec<4>(a, val != nullptr, t.lanes, wpb, s);
        else launch_seg_vec<1>(a, val != nullptr, t.lanes, wpb, s);
        if (plan.n_red) {
            const std::uint64_t total = plan.n_red * f;
            const unsigned blocks = unsigned(std::min<std::uint64_t>((total + 255) / 256, std::uint64_t(g.sms) * 32));
            hub_reduce_kernel<<<blocks, 256, 0, s>>>(plan.red_row.get(), plan.red_first.get(),
                                                     plan.red_count.get(), plan.n_red, g.scratch.get(), c, f);
            check_launch("hub_reduce_kernel");
        }
        return;
    }
    const bool fork_light = concurrent && plan.n_light && plan.n_pieces;
    if (fork_light) {
        cudaStream_t aux = graph_fork(g, s);
        launch_spmm_rows(g, val, plan.n_heavy, plan.n_light, b, f, c, f_tile, vec, wpb, aux, finite, rmax, rsum,
                         wt);
    }
    if (plan.n_pieces) {
        SegArgs a{};
        a.rowptr = g.rowptr.get();
        a.colind = g.colind.get();
        a.val = val;
        a.vperm = g.val_perm;
        a.b = b;
        a.c = c;
        a.scratch = g.scratch.get();
        a.piece_row = plan.piece_row.get();
        a.piece_e0 = plan.piece_e0.get();
        a.piece_len = plan.piece_len.get();
        a.piece_slot = plan.piece_slot.get();
        a.finite = finite;
        a.rmax = rmax;
        a.rsum = rsum;
        a.n_items = plan.n_pieces * t.n_tiles;
        a.n_tiles = t.n_tiles;
        a.f = f;
        a.n_rows = g.n_rows;
        a.n_cols = g.n_cols;
        a.nnz = g.nnz;
        a.off32 = fast_gather_ok(g, f);
        a.wt = wt;
        a.keep_b = std::uint64_t(g.n_cols) * f * (wt ? 2 : 4) <= kKeepMaxBytes;
        a.tile_major = tile_major();
        a.tile_w = t.tile_w;
        // pieces are up to 2048-entry dependent chains: when there are too
        // few of them to fill the lane-group kernel (under a wave), the ring
        // kernel's deep per-piece prefetch wins (c1: 0.163 -> 0.106 ms); with
        // thousands of pieces the group kernel's throughput wins (Products
        // 8-way shard: 1.36 ms vs 1.72 ms)
        const bool few = plan.n_pieces <= std::uint64_t(4) * std::uint64_t(g.sms);
        if (few && !wt && !g.val_perm && longrow_ok(f, vec)) launch_longrow<true>(a, plan.n_pieces, s);
        else if (v8) launch_seg_vec<8>(a, val != nullptr, t.lanes, wpb, s);
        else if (vec) launch_seg_vec<4>(a, val != nullptr, t.lanes, wpb, s);
        else launch_seg_vec<1>(a, val != nullptr, t.lanes, wpb, s);
    }
    if (fork_light) graph_join(g, s);
    else if (plan.n_light)
        launch_spmm_rows(g, val, plan.n_heavy, plan.n_light, b, f, c, f_tile, vec, wpb, s, finite, rmax, rsum,
                         wt);
    if (plan.n_red) {
        const std::uint64_t total = plan.n_red * f;
        const unsigned blocks = unsigned(std::min<std::uint64_t>((total + 255) / 256, std::uint64_t(g.sms) * 32));
        hub_reduce_kernel<<<blocks, 256, 0, s>>>(plan.red_row.get(), plan.red_first.get(),
                                                 plan.red_count.get(), plan.n_red, g.scratch.get(),
                                                 c, f);
        check_launch("hub_reduce_kernel");
    }
}

} // namespace asb
