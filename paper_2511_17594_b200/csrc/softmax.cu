// softmax.cu -- CSR row softmax for sm_100a (src/kernels.cpp:431-461).
//
// Per non-empty row: mx = max over the f32 values; ex_e = f32(exp(f64 v_e -
// f64 mx)); sum = f64 sum of ex_e in entry order; out_e = f32(f64 ex_e /
// sum).  Empty rows produce nothing.  The arithmetic lives in softmax.cuh
// (shared with the SpMM that applies probabilities on the fly); the sum is
// reduced in parallel and is bit-equal to the reference's sequential chain
// whenever the exactness certificate of softmax.cuh holds, else the row
// re-runs the chain in entry order.  The only difference from the CPU
// reference can therefore come from exp() itself (CUDA's f64 exp vs libm,
// both within 1 ulp of f64, rounded to f32).
// The max ignores NaN where std::max would latch a leading NaN; either way a
// NaN in a row makes every ex (or the sum) NaN, so all outputs of that row
// are NaN exactly as in the reference.
//
// Mapping: rows in degree-descending order.  Rows longer than kRowSmem
// entries get a CTA each (staged in shared memory up to kCtaSmem entries,
// else three passes); the rest get a warp each, software-pipelined so the
// next row's values stream in (cp.async) while the current one computes.
// Either way one global read and one write per entry.  The CTA kernel runs
// on a forked stream, concurrently with the warp kernel.
//
// Stats mode (OUT = false) writes (mx, sum) per row and, into vout, each
// entry's ex = f32(exp(v - mx)): the fused attention SpMM turns ex into p_e
// with the same sm_prob as the output pass, so it never recomputes the f64
// exp.  Every path that computes a row's ex writes it (vout must not alias
// vin: a row deferred to the chain kernel is read again there).
#include "ops.hpp"
#include "softmax.cuh"

#include <algorithm>
#include <cstdlib>

namespace asb {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kRowSmem = 512;        // warp kernel: rows up to this many entries
constexpr int kCtaSmem = 8192;       // CTA kernel: rows staged in shared memory
constexpr int kWarpsPerCta = 8;

struct SoftmaxArgs {
    const std::uint64_t* rowptr;
    const std::uint32_t* order;  // rows of this launch: order[0, n)
    std::uint64_t n;
    const float* vin;
    float* vout;    // OUT: probabilities; !OUT: ex (see above)
    float* rmax;    // !OUT
    double* rsum;   // !OUT
    int force_seq;  // developer/test knob: always run the sequential chain
    // CTA kernel: defer a row straight to the chain kernel when its value
    // range already proves the exactness certificate fails (see below)
    int predefer;
    // CTA kernel: rows whose certificate failed are handed to the chain
    // kernel (row, max) instead of serialising the CTA on one sum chain
    std::uint32_t* chain_row;
    float* chain_mx;
    unsigned* chain_n;
};

// LIB: exp() itself instead of the written-out sm_exp (test knob
// AUTOSAGE_DEV_SOFTMAX_LIBEXP; the two must agree bit for bit)
template <bool LIB>
__device__ __forceinline__ float ex_of(float v, double dmx) {
    if constexpr (LIB) return float(exp(double(v) - dmx));
    else return sm_ex(v, dmx);
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return unsigned(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// Warp per row (rows of at most kRowSmem entries).  Software pipeline: while
// a warp works on its row out of shared memory, the next row's values are
// already in flight (cp.async into the other buffer) and the row after
// that has its (row, e0, deg) loads issued, so neither global latency sits
// on the path of a row.
template <bool OUT, bool LIB>
__global__ void __launch_bounds__(256, 3) softmax_warp_kernel(SoftmaxArgs a) {
    __shared__ __align__(16) float buf_all[kWarpsPerCta][2][kRowSmem];
    const int lane = threadIdx.x & 31;
    float (*buf)[kRowSmem] = buf_all[threadIdx.x >> 5];
    const std::uint64_t tw = std::uint64_t(gridDim.x) * (blockDim.x >> 5);
    std::uint64_t w = (std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;

    struct RowRef {
        std::uint32_t row, deg;
        std::uint64_t e0;
    };
    auto fetch = [&](std::uint64_t wi) {  // index loads (not waited on here)
        RowRef r{0, 0, 0};
        if (wi < a.n) {
            r.row = a.order[wi];
            r.e0 = a.rowptr[r.row];
            r.deg = std::uint32_t(a.rowptr[r.row + 1] - r.e0);
        }
        return r;
    };
    auto issue = [&](const RowRef& r, int slot) {
        const float* src = a.vin + r.e0;
        for (std::uint32_t k = lane; k < r.deg; k += 32) cp_async4(&buf[slot][k], src + k);
        cp_async_commit();
    };
    RowRef cur = fetch(w);
    RowRef nxt = fetch(w + tw);
    issue(cur, 0);
    for (int it = 0; w < a.n; w += tw, ++it) {
        const int slot = it & 1;
        const RowRef nn = fetch(w + 2 * tw);
        issue(nxt, slot ^ 1);
        cp_async_wait1();  // this lane's copies of `cur` landed
        __syncwarp();      // ... and everyone's
        const float* exs_in = buf[slot];
        float* exs = buf[slot];
        const std::uint32_t deg = cur.deg;
        if (deg) {
            float mx = -INFINITY;
            for (std::uint32_t k = lane; k < deg; k += 32) mx = fmaxf(mx, exs_in[k]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, o));
            const double dmx = double(mx);
            double sum = 0.0;
            unsigned mn = 0xffffffffu;
#pragma unroll 2
            for (std::uint32_t k = lane; k < deg; k += 32) {
                const float ex = ex_of<LIB>(exs[k], dmx);
                exs[k] = ex;
                sum += double(ex);
                mn = sm_cert_acc(mn, ex);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(FULL, sum, o);
            mn = __reduce_min_sync(FULL, mn);
            __syncwarp();
            if (a.force_seq || !__all_sync(FULL, sm_sum_exact(sum, mn))) {
                // the reference's chain, in entry order
                if (lane == 0) {
                    sum = 0.0;
                    for (std::uint32_t k = 0; k < deg; ++k) sum = __dadd_rn(sum, double(exs[k]));
                }
                sum = __shfl_sync(FULL, sum, 0);
            }
            if constexpr (OUT) {
                const double rcp = sm_rcp(sum);
                float* vout = a.vout + cur.e0;
#pragma unroll 4
                for (std::uint32_t k = lane; k < deg; k += 32) vout[k] = sm_prob(exs[k], sum, rcp);
            } else {
                float* vex = a.vout + cur.e0;
#pragma unroll 4
                for (std::uint32_t k = lane; k < deg; k += 32) vex[k] = exs[k];
                if (lane == 0) {
                    a.rmax[cur.row] = mx;
                    a.rsum[cur.row] = sum;
                }
            }
        }
        __syncwarp();  // buffer `slot` is refilled by the next iteration's issue
        cur = nxt;
        nxt = nn;
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// block-wide reductions over the 8 warps (every thread gets the result)
struct CtaRed {
    float f[kWarpsPerCta];
    float g[kWarpsPerCta];
    double d[kWarpsPerCta];
    unsigned u[kWarpsPerCta];
    double seq;
};
__device__ __forceinline__ float cta_max(CtaRed& r, float v) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(FULL, v, o));
    if (lane == 0) r.f[warp] = v;
    __syncthreads();
    v = r.f[0];
#pragma unroll
    for (int i = 1; i < kWarpsPerCta; ++i) v = fmaxf(v, r.f[i]);
    return v;
}
// max and min in one pass (one barrier)
__device__ __forceinline__ void cta_max_min(CtaRed& r, float& mx, float& mn) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, o));
        mn = fminf(mn, __shfl_xor_sync(FULL, mn, o));
    }
    if (lane == 0) {
        r.f[warp] = mx;
        r.g[warp] = mn;
    }
    __syncthreads();
    mx = r.f[0];
    mn = r.g[0];
#pragma unroll
    for (int i = 1; i < kWarpsPerCta; ++i) {
        mx = fmaxf(mx, r.f[i]);
        mn = fminf(mn, r.g[i]);
    }
}
// sum (exact under the certificate, so any order) and certificate minimum
__device__ __forceinline__ void cta_sum(CtaRed& r, double& sum, unsigned& mn) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(FULL, sum, o);
    mn = __reduce_min_sync(FULL, mn);
    if (lane == 0) {
        r.d[warp] = sum;
        r.u[warp] = mn;
    }
    __syncthreads();
    sum = r.d[0];
    mn = r.u[0];
#pragma unroll
    for (int i = 1; i < kWarpsPerCta; ++i) {
        sum += r.d[i];
        mn = min(mn, r.u[i]);
    }
}

// CTA per long row, persistent over rows order[blockIdx.x + k*gridDim.x]
// with the same software pipeline as the warp kernel: rows of at most
// kCtaSmem entries stream into one of two shared-memory buffers (cp.async)
// while the CTA works on the other, so the global read of a row overlaps
// the previous row's compute; ex is computed once and kept there for the
// output pass.  Longer rows take three passes over global memory (max; ex
// and sum; output with ex recomputed).  A failed certificate re-runs the
// sum as the entry-order chain (thread 0 over 256-entry blocks of ex).
template <bool OUT, bool LIB>
__global__ void __launch_bounds__(256, 3) softmax_cta_kernel(SoftmaxArgs a) {
    extern __shared__ __align__(16) float cbuf[];  // 2 x kCtaSmem floats
    __shared__ CtaRed red;
    const int tid = threadIdx.x;
    struct RowRef {
        std::uint32_t row, deg;
        std::uint64_t e0;
    };
    auto fetch = [&](std::uint64_t i) {
        RowRef r{0, 0, 0};
        if (i < a.n) {
            r.row = a.order[i];
            r.e0 = a.rowptr[r.row];
            r.deg = std::uint32_t(a.rowptr[r.row + 1] - r.e0);
        }
        return r;
    };
    auto issue = [&](const RowRef& r, int slot) {
        if (r.deg <= std::uint32_t(kCtaSmem)) {
            const float* src = a.vin + r.e0;
            float* dst = cbuf + slot * kCtaSmem;
            for (std::uint32_t k = tid; k < r.deg; k += 256) cp_async4(dst + k, src + k);
        }
        cp_async_commit();
    };
    const std::uint64_t G = gridDim.x;
    std::uint64_t i = blockIdx.x;
    RowRef cur = fetch(i);
    RowRef nxt = fetch(i + G);
    issue(cur, 0);
    for (int it = 0; i < a.n; i += G, ++it) {
        const int slot = it & 1;
        const RowRef nn = fetch(i + 2 * G);
        issue(nxt, slot ^ 1);
        cp_async_wait1();
        __syncthreads();
        const std::uint32_t deg = cur.deg;
        const bool staged = deg <= std::uint32_t(kCtaSmem);
        float* cexs = cbuf + slot * kCtaSmem;
        const float* vin = a.vin + cur.e0;

        float mx = -INFINITY, mnv = INFINITY;
        if (staged) {
#pragma unroll 8
            for (std::uint32_t k = tid; k < deg; k += 256) {
                mx = fmaxf(mx, cexs[k]);
                mnv = fminf(mnv, cexs[k]);
            }
        } else {
#pragma unroll 8
            for (std::uint32_t k = tid; k < deg; k += 256) {
                const float v = __ldg(vin + k);
                mx = fmaxf(mx, v);
                mnv = fminf(mnv, v);
            }
        }
        if (a.predefer && !a.force_seq) cta_max_min(red, mx, mnv);
        else mx = cta_max(red, mx);
        const double dmx = double(mx);
        // The row's maximum contributes ex = 1, so the total is >= 1.  If the
        // smallest value gives a normal, non-zero ex below 2^-31 (mnv - mx in
        // (-87, -22)), its ulp is below 2^-54 and the certificate
        // (total < 2^(q+53), softmax.cuh) cannot hold: skip the parallel
        // exp + sum and hand the row to the chain kernel at once.  Deferring
        // is always exact -- the chain is the reference's own order -- so
        // this only saves work.
        if (a.predefer && !a.force_seq) {
            const double span = double(mnv) - dmx;
            // predefer 2 adds an estimate: values spread over [mnv, mx] put the
            // total near deg / |span|, so the certificate likely fails once
            // log2(deg / |span|) >= span / ln 2 + 30 (a wrong guess only
            // moves the row to the other exact path)
            const bool certain = span < -22.0 && span > -87.0;
            const bool likely = a.predefer == 2 && span < -1.0 && span > -87.0 &&
                                log2(double(deg) / -span) >= span * 1.4426950408889634 + 30.0;
            if (certain || likely) {  // block-uniform
                if (tid == 0) {
                    const unsigned i = atomicAdd(a.chain_n, 1u);
                    a.chain_row[i] = cur.row;
                    a.chain_mx[i] = mx;
                }
                __syncthreads();
                cur = nxt;
                nxt = nn;
                continue;
            }
        }

        double sum = 0.0;
        unsigned mn = 0xffffffffu;
        if (staged) {
#pragma unroll 2
            for (std::uint32_t k = tid; k < deg; k += 256) {
                const float ex = ex_of<LIB>(cexs[k], dmx);
                cexs[k] = ex;
                sum += double(ex);
                mn = sm_cert_acc(mn, ex);
            }
        } else {
#pragma unroll 2
            for (std::uint32_t k = tid; k < deg; k += 256) {
                const float ex = ex_of<LIB>(__ldg(vin + k), dmx);
                sum += double(ex);
                mn = sm_cert_acc(mn, ex);
            }
        }
        cta_sum(red, sum, mn);
        if (a.force_seq || !sm_sum_exact(sum, mn)) {  // block-uniform
            // the sum needs the entry-order chain: defer the row to the
            // chain kernel (one lane per row there, many rows in flight)
            if (tid == 0) {
                const unsigned i = atomicAdd(a.chain_n, 1u);
                a.chain_row[i] = cur.row;
                a.chain_mx[i] = mx;
            }
            __syncthreads();  // buffer `slot` / `red` reuse
            cur = nxt;
            nxt = nn;
            continue;
        }
        if constexpr (OUT) {
            const double rcp = sm_rcp(sum);
            float* vout = a.vout + cur.e0;
            if (staged) {
#pragma unroll 4
                for (std::uint32_t k = tid; k < deg; k += 256) vout[k] = sm_prob(cexs[k], sum, rcp);
            } else {
                // plain loads: vout may alias vin (each entry is read, then
                // written, by the same thread)
#pragma unroll 4
                for (std::uint32_t k = tid; k < deg; k += 256)
                    vout[k] = sm_prob(ex_of<LIB>(vin[k], dmx), sum, rcp);
            }
        } else {
            float* vex = a.vout + cur.e0;
            if (staged) {
#pragma unroll 4
                for (std::uint32_t k = tid; k < deg; k += 256) vex[k] = cexs[k];
            } else {
#pragma unroll 4
                for (std::uint32_t k = tid; k < deg; k += 256) vex[k] = ex_of<LIB>(__ldg(vin + k), dmx);
            }
            if (tid == 0) {
                a.rmax[cur.row] = mx;
                a.rsum[cur.row] = sum;
            }
        }
        __syncthreads();  // buffer `slot` and `red` are reused next iteration
        cur = nxt;
        nxt = nn;
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// Rows deferred by the CTA kernel: warp per row, many warps per SM so many
// chains are in flight.  64 entries at a time the lanes recompute ex in
// parallel (next step's values already loaded) and stage it as f64; lane 0
// folds them into the row's sum in entry order (the reference's chain, one
// DADD per entry, two entries per LDS.128).  Then the output pass (ex
// recomputed, coalesced) or the stats write.  (Lane per row -- 32 chains per
// warp, each lane walking its own row -- measured 10x slower: the
// uncoalesced per-lane streams thrash L1.)
template <bool OUT, bool LIB>
__global__ void __launch_bounds__(256, 4) softmax_chain_kernel(SoftmaxArgs a) {
    __shared__ __align__(16) double stage_all[kWarpsPerCta][2 * 32];
    const int lane = threadIdx.x & 31;
    double* st = stage_all[threadIdx.x >> 5];
    const unsigned n = *a.chain_n;
    const std::uint64_t tw = std::uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (std::uint64_t w = (std::uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < n; w += tw) {
        const std::uint32_t row = a.chain_row[w];
        const float mx = a.chain_mx[w];
        const double dmx = double(mx);
        const std::uint64_t e0 = a.rowptr[row];
        const std::uint32_t deg = std::uint32_t(a.rowptr[row + 1] - e0);
        const float* vin = a.vin + e0;
        double sum = 0.0;
        // 64 entries per step: each lane's two exps run as independent
        // chains, and the warp syncs once per 64 adds
        float vn0 = lane < int(deg) ? __ldg(vin + lane) : 0.f;
        float vn1 = 32u + lane < deg ? __ldg(vin + 32 + lane) : 0.f;
        for (std::uint32_t base = 0; base < deg; base += 64) {
            const float v0 = vn0, v1 = vn1;
            const std::uint32_t k0 = base + lane, k1 = k0 + 32;
            vn0 = k0 + 64 < deg ? __ldg(vin + k0 + 64) : 0.f;
            vn1 = k1 + 64 < deg ? __ldg(vin + k1 + 64) : 0.f;
            const float ex0 = ex_of<LIB>(v0, dmx), ex1 = ex_of<LIB>(v1, dmx);
            st[lane] = k0 < deg ? double(ex0) : 0.0;
            st[32 + lane] = k1 < deg ? double(ex1) : 0.0;
            if constexpr (!OUT) {
                if (k0 < deg) a.vout[e0 + k0] = ex0;
                if (k1 < deg) a.vout[e0 + k1] = ex1;
            }
            __syncwarp();
            if (lane == 0) {
                const std::uint32_t m = deg - base < 64 ? deg - base : 64;
                if (m == 64) {
                    // whole step: the shared-memory loads are issued ahead of
                    // the dependent adds (16 at a time), so the chain runs at
                    // the DADD latency instead of LDS + DADD per pair
                    const double2* sp = reinterpret_cast<const double2*>(st);
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        double2 d[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) d[i] = sp[8 * h + i];
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            sum = __dadd_rn(sum, d[i].x);
                            sum = __dadd_rn(sum, d[i].y);
                        }
                    }
                } else {
                    std::uint32_t j = 0;
                    for (; j + 2 <= m; j += 2) {
                        const double2 d = *reinterpret_cast<const double2*>(st + j);
                        sum = __dadd_rn(sum, d.x);
                        sum = __dadd_rn(sum, d.y);
                    }
                    if (j < m) sum = __dadd_rn(sum, st[j]);
                }
            }
            __syncwarp();
        }
        sum = __shfl_sync(FULL, sum, 0);
        if constexpr (OUT) {
            const double rcp = sm_rcp(sum);
            float* vout = a.vout + e0;
            // plain loads: vout may alias vin (read, then written, by one lane)
#pragma unroll 4
            for (std::uint32_t k = lane; k < deg; k += 32) vout[k] = sm_prob(ex_of<LIB>(vin[k], dmx), sum, rcp);
        } else if (lane == 0) {
            a.rmax[row] = mx;
            a.rsum[row] = sum;
        }
    }
}

bool env_flag(const char* name) {
    const char* e = std::getenv(name);
    return e && std::atoi(e) != 0;
}

template <bool OUT>
void launch_softmax(Graph& g, const float* vin, float* vout, float* rmax, double* rsum, cudaStream_t s) {
    if (g.n_rows == 0 || g.nnz == 0) return;
    ensure_order(g);
    SoftmaxArgs a{};
    a.rowptr = g.rowptr.get();
    a.vin = vin;
    a.vout = vout;
    a.rmax = rmax;
    a.rsum = rsum;
    a.force_seq = env_flag("AUTOSAGE_DEV_SOFTMAX_SEQ") ? 1 : 0;
    {
        // 0 off, 1 certain failures only, 2 (default) also likely ones:
        // Reddit-shape fused attention 5.233 -> 5.197 ms, row softmax over
        // N(0, 8^2) values 2.045 -> 1.837 ms (profiles/r02ad_predefer.log)
        const char* e = std::getenv("AUTOSAGE_DEV_SOFTMAX_PREDEFER");
        a.predefer = e ? std::atoi(e) : 2;
    }
    const bool lib = env_flag("AUTOSAGE_DEV_SOFTMAX_LIBEXP");
    const std::uint64_t n_long = rows_with_degree_at_least(g, kRowSmem + 1);
    const std::uint64_t n_short = g.n_rows - n_long;
    if (n_long) {
        SoftmaxArgs al = a;
        al.order = g.order.get();
        al.n = n_long;
        cudaStream_t aux = n_short ? graph_fork(g, s) : s;
        constexpr int smem = 2 * kCtaSmem * 4;
        const int sms = g.sms;
        const unsigned grid = unsigned(std::min<std::uint64_t>(n_long, std::uint64_t(sms) * 3));
        auto go = [&](auto kern) {
            kernel_setup(kern, smem, 256);
            kern<<<grid, 256, smem, aux>>>(al);
        };
        g.sm_chain_row.ensure(n_long);
        g.sm_chain_mx.ensure(n_long);
        g.sm_chain_n.ensure(1);
        al.chain_row = g.sm_chain_row.get();
        al.chain_mx = g.sm_chain_mx.get();
        al.chain_n = g.sm_chain_n.get();
        ASB_CUDA(cudaMemsetAsync(al.chain_n, 0, sizeof(unsigned), aux));
        if (lib) go(softmax_cta_kernel<OUT, true>);
        else go(softmax_cta_kernel<OUT, false>);
        check_launch("softmax_cta_kernel");
        const unsigned cgrid = unsigned(std::min<std::uint64_t>((n_long + kWarpsPerCta - 1) / kWarpsPerCta,
                                                                std::uint64_t(sms) * 4));
        if (lib) softmax_chain_kernel<OUT, true><<<cgrid, 32 * kWarpsPerCta, 0, aux>>>(al);
        else softmax_chain_kernel<OUT, false><<<cgrid, 32 * kWarpsPerCta, 0, aux>>>(al);
        check_launch("softmax_chain_kernel");
    }
    if (n_short) {
        const int sms = g.sms;
        a.order = g.order.get() + n_long;
        a.n = n_short;
        const std::uint64_t want = (n_short + kWarpsPerCta - 1) / kWarpsPerCta;
        const unsigned blocks = unsigned(std::min<std::uint64_t>(want, std::uint64_t(sms) * 6));
        if (lib) softmax_warp_kernel<OUT, true><<<blocks, 32 * kWarpsPerCta, 0, s>>>(a);
        else softmax_warp_kernel<OUT, false><<<blocks, 32 * kWarpsPerCta, 0, s>>>(a);
        check_launch("softmax_warp_kernel");
    }
    if (n_long && n_short) graph_join(g, s);
}

} // namespace

void launch_row_softmax(Graph& g, const float* vin, float* vout, cudaStream_t s) {
    launch_softmax<true>(g, vin, vout, nullptr, nullptr, s);
}

void launch_row_softmax_stats(Graph& g, const float* vin, float* ex, float* rmax, double* rsum, cudaStream_t s) {
    if (ex == vin) throw LogicError("softmax stats: ex must not alias the scores");
    launch_softmax<false>(g, vin, ex, rmax, rsum, s);
}

} // namespace asb
