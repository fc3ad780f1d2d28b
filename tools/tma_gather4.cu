// tma_gather4.cu -- A/B of the SDDMM Y-row staging: 16-byte cp.async
// (LDGSTS, what sddmm_pair1_kernel does) against TMA tile::gather4
// (cp.async.bulk.tensor.2d ... tile::gather4: four 128-byte row halves per
// instruction, 128B-swizzled into shared memory, mbarrier completion).
//
// Workload: 232,965 x 64 f32 Y (L2-resident, Reddit-shape), 114.6M random
// row ids in 64-entry chunks per warp; each lane then walks its two staged
// rows with LDS.128 (the pair kernel's read pattern) and folds them into one
// f32 (the compute is deliberately trivial: this measures staging + reads).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_gather4 tools/tma_gather4.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                           \
    do {                                                                                \
        cudaError_t e_ = (x);                                                           \
        if (e_ != cudaSuccess) {                                                        \
            std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            return 1;                                                                   \
        }                                                                               \
    } while (0)

constexpr int F = 64;
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return unsigned(__cvta_generic_to_shared(p));
}

// ---- A: cp.async staging (XOR-swizzled 16-byte units, like the pair kernel) ----
template <int NV>
__device__ __forceinline__ int swz(int j) { return j & (NV - 1); }

__global__ void __launch_bounds__(128, 3) stage_cpasync(const float* __restrict__ y, const unsigned* __restrict__ idx,
                                                        unsigned long long m, float* __restrict__ out) {
    extern __shared__ __align__(1024) char smem[];
    constexpr int NV = F / 4;
    float* ys = reinterpret_cast<float*>(smem + (threadIdx.x >> 5) * (64 * F * 4));
    const int lane = threadIdx.x & 31;
    const unsigned long long chunks = m / 64;
    const unsigned long long stride = gridDim.x * 4ull;
    float acc = 0.f;
    for (unsigned long long c = blockIdx.x * 4ull + (threadIdx.x >> 5); c < chunks; c += stride) {
        const unsigned ca = __ldg(idx + c * 64 + lane), cb = __ldg(idx + c * 64 + 32 + lane);
#pragma unroll
        for (int it = 0; it < 2 * NV; ++it) {
            const int id = it * 32 + lane;
            const int j = id / NV, q = id % NV;
            const unsigned cj = __shfl_sync(FULL, j < 32 ? ca : cb, j & 31);
            const float* src = y + std::uint64_t(cj) * F + 4 * q;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(ys + j * F + 4 * (q ^ swz<NV>(j)))),
                         "l"(src));
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
        __syncwarp();
        const float* ya = ys + lane * F;
        const float* yb = ys + (lane + 32) * F;
#pragma unroll 4
        for (int t = 0; t < F; t += 4) {
            const float4 u = *reinterpret_cast<const float4*>(ya + 4 * ((t >> 2) ^ swz<NV>(lane)));
            const float4 w = *reinterpret_cast<const float4*>(yb + 4 * ((t >> 2) ^ swz<NV>(lane + 32)));
            acc += u.x + u.y + u.z + u.w + w.x + w.y + w.z + w.w;
        }
        __syncwarp();
    }
    if (acc == 1234.5f) out[threadIdx.x] = acc;
}

// ---- B: TMA tile::gather4 ----------------------------------------------------------
// Per warp buffer: half 0 (features 0-31) of the 64 rows, then half 1; each
// 64 x 128 B region 1024-aligned, 128B swizzle: 16-byte chunk c of row j sits
// at chunk c ^ (j & 7).
__device__ __forceinline__ void mbar_init(std::uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, unsigned phase) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, int x, int r0, int r1, int r2, int r3,
                                            std::uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<std::uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}

template <int NBUF>
__global__ void __launch_bounds__(128) stage_gather4(const __grid_constant__ CUtensorMap ymap,
                                                     const unsigned* __restrict__ idx, unsigned long long m,
                                                     float* __restrict__ out) {
    extern __shared__ __align__(1024) char smem[];
    constexpr int kBuf = 64 * F * 4;  // 16 KB: two 8 KB halves
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    char* wbase = smem + warp * (NBUF * kBuf + 1024);
    std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(wbase + NBUF * kBuf);
    if (lane == 0)
        for (int b = 0; b < NBUF; ++b) mbar_init(bars + b, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncwarp();
    const unsigned long long chunks = m / 64;
    const unsigned long long stride = gridDim.x * 4ull;
    auto issue = [&](unsigned long long c, int b) {
        if (c >= chunks) return;
        // lanes 0..15: entries 4g..4g+3 of the chunk
        if (lane < 16) {
            const uint4 cols = __ldg(reinterpret_cast<const uint4*>(idx + c * 64) + lane);
            char* buf = wbase + b * kBuf;
            if (lane == 0) mbar_expect_tx(bars + b, kBuf);
            __syncwarp(0xffffu);
            tma_gather4(buf + lane * 4 * 128, &ymap, 0, int(cols.x), int(cols.y), int(cols.z), int(cols.w), bars + b);
            tma_gather4(buf + 8192 + lane * 4 * 128, &ymap, 32, int(cols.x), int(cols.y), int(cols.z), int(cols.w),
                        bars + b);
        }
    };
    unsigned long long c = blockIdx.x * 4ull + warp;
    unsigned phase[NBUF] = {};
    for (int b = 0; b < NBUF - 1; ++b) issue(c + b * stride, b);
    float acc = 0.f;
    int b = 0;
    for (; c < chunks; c += stride) {
        if (NBUF > 1) issue(c + (NBUF - 1) * stride, (b + NBUF - 1) % NBUF);
        else issue(c, 0);
        mbar_wait(bars + b, phase[b]);
        phase[b] ^= 1u;
        const char* buf = wbase + b * kBuf;
#pragma unroll 4
        for (int t = 0; t < F; t += 4) {
            const int h = t >> 5, q = (t & 31) >> 2;
            const float4 u = *reinterpret_cast<const float4*>(buf + h * 8192 + lane * 128 + 16 * (q ^ (lane & 7)));
            const float4 w =
                *reinterpret_cast<const float4*>(buf + h * 8192 + (lane + 32) * 128 + 16 * (q ^ (lane & 7)));
            acc += u.x + u.y + u.z + u.w + w.x + w.y + w.z + w.w;
        }
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        b = (b + 1) % NBUF;
    }
    if (acc == 1234.5f) out[threadIdx.x] = acc;
}

// reference sums (host check that both stagings read the right rows)
__global__ void direct_sum(const float* __restrict__ y, const unsigned* __restrict__ idx, unsigned long long m,
                           double* __restrict__ total) {
    double acc = 0.0;
    for (unsigned long long e = blockIdx.x * 256ull + threadIdx.x; e < m; e += gridDim.x * 256ull)
        for (int t = 0; t < F; ++t) acc += y[std::uint64_t(idx[e]) * F + t];
    atomicAdd(total, acc);
}

template <class K>
float time_it(K k, int reps) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        k();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    return best;
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const unsigned n = 232965;
    const unsigned long long m = 114615872ull;  // multiple of 64
    std::vector<float> hy(std::size_t(n) * F);
    std::vector<unsigned> hidx(m);
    unsigned long long s = 88172645463325252ull;
    for (auto& v : hy) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        v = float(s % 1000) * 1e-3f;
    }
    for (auto& v : hidx) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        v = unsigned(s % n);
    }
    float *y, *out;
    unsigned* idx;
    CK(cudaMalloc(&y, hy.size() * 4));
    CK(cudaMalloc(&idx, m * 4));
    CK(cudaMalloc(&out, 4096));
    CK(cudaMemcpy(y, hy.data(), hy.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(idx, hidx.data(), m * 4, cudaMemcpyHostToDevice));

    EncodeTiled encode = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q));
    CUtensorMap map;
    const cuuint64_t gdim[2] = {F, n};
    const cuuint64_t gstride[1] = {F * 4};
    const cuuint32_t box[2] = {32, 1};
    const cuuint32_t estride[2] = {1, 1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, y, gdim, gstride, box, estride,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        std::printf("cuTensorMapEncodeTiled failed: %d\n", int(r));
        return 1;
    }
    const double gb = double(m) * F * 4 / 1e9;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);

    const int smA = 4 * 64 * F * 4;
    CK(cudaFuncSetAttribute(stage_cpasync, cudaFuncAttributeMaxDynamicSharedMemorySize, smA));
    int occA = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occA, stage_cpasync, 128, smA);
    float tA = time_it([&] { stage_cpasync<<<sms * occA, 128, smA>>>(y, idx, m, out); }, 5);
    CK(cudaGetLastError());
    std::printf("cp.async staging : %.3f ms  %.1f GB/s of staged rows  (%d CTAs/SM)\n", tA, gb / tA * 1e3, occA);

    auto runB = [&](auto kern, int nbuf, const char* name) -> int {
        const int sm = 4 * (nbuf * 64 * F * 4 + 1024) + 1024;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, sm);
        float t = time_it([&] { kern<<<sms * occ, 128, sm>>>(map, idx, m, out); }, 5);
        CK(cudaGetLastError());
        std::printf("%s: %.3f ms  %.1f GB/s of staged rows  (%d CTAs/SM)\n", name, t, gb / t * 1e3, occ);
        return 0;
    };
    if (runB(stage_gather4<1>, 1, "TMA gather4, 1 buffer  ")) return 1;
    if (runB(stage_gather4<2>, 2, "TMA gather4, 2 buffers ")) return 1;
    CK(cudaDeviceSynchronize());
    std::printf("done\n");
    return 0;
}
