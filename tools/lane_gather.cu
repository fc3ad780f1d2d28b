// lane_gather.cu -- is staging Y rows through shared memory (SDDMM) needed?
// Compares, on an L2-resident 232965 x 64 f32 matrix with hashed random rows:
//   A: lane per row, 16 LDG.128 per lane (32 distinct rows per instruction)
//   B: 16 lanes per row, one LDG.128 per lane (2 rows per instruction)
//   C: lane per row via cp.async into shared memory + LDS.128 (SDDMM today)
//   D: lane per row via one TMA bulk copy per row (cp.async.bulk, mbarrier
//      completion) + LDS.128 -- does the async proxy relieve the LSU pipe?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lane_gather tools/lane_gather.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ unsigned hsh(unsigned x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
constexpr int F = 64;

__global__ void __launch_bounds__(128) lane_row(const float* __restrict__ b, unsigned n, unsigned long long m,
                                                float* __restrict__ out) {
    const unsigned long long tid = blockIdx.x * 128ull + threadIdx.x;
    const unsigned long long nt = gridDim.x * 128ull;
    float acc = 0.f;
    for (unsigned long long e = tid; e < m; e += nt) {
        const float4* r = reinterpret_cast<const float4*>(b + std::uint64_t(hsh(unsigned(e)) % n) * F);
        float4 v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = __ldg(r + q);
#pragma unroll
        for (int q = 0; q < 16; ++q) acc += v[q].x + v[q].y + v[q].z + v[q].w;
    }
    if (acc == 12345.f) out[tid] = acc;
}

__global__ void __launch_bounds__(128) group_row(const float* __restrict__ b, unsigned n, unsigned long long m,
                                                 float* __restrict__ out) {
    const unsigned long long tid = blockIdx.x * 128ull + threadIdx.x;
    const unsigned long long nt = gridDim.x * 128ull;
    const int gl = threadIdx.x & 15;
    float acc = 0.f;
    // each group of 16 lanes: 4 rows in flight
    for (unsigned long long base = (tid >> 4) * 4; base < m; base += (nt >> 4) * 4) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const unsigned row = hsh(unsigned(base + u)) % n;
            v[u] = __ldg(reinterpret_cast<const float4*>(b + std::uint64_t(row) * F) + gl);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
    if (acc == 12345.f) out[tid] = acc;
}

__device__ __forceinline__ void cp16(void* s, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(unsigned(__cvta_generic_to_shared(s))), "l"(g) : "memory");
}
__global__ void __launch_bounds__(128) smem_row(const float* __restrict__ b, unsigned n, unsigned long long m,
                                                float* __restrict__ out) {
    extern __shared__ __align__(16) float sm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    float* ys = sm + w * 32 * F;
    const unsigned long long wid = blockIdx.x * 4ull + w, nw = gridDim.x * 4ull;
    float acc = 0.f;
    for (unsigned long long c = wid * 32; c < m; c += nw * 32) {
        const unsigned myrow = hsh(unsigned(c + lane)) % n;
#pragma unroll
        for (int it = 0; it < 16; ++it) {
            const int idx = it * 32 + lane, j = idx / 16, q = idx % 16;
            const unsigned rj = __shfl_sync(0xffffffffu, myrow, j);
            cp16(ys + j * F + 4 * (q ^ (j & 15)), b + std::uint64_t(rj) * F + 4 * q);
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const float4 v = *reinterpret_cast<const float4*>(ys + lane * F + 4 * (q ^ (lane & 15)));
            acc += v.x + v.y + v.z + v.w;
        }
        __syncwarp();
    }
    if (acc == 12345.f) out[blockIdx.x * 128 + threadIdx.x] = acc;
}

__global__ void __launch_bounds__(128) tma_row(const float* __restrict__ b, unsigned n, unsigned long long m,
                                               float* __restrict__ out) {
    extern __shared__ __align__(16) float smt[];
    __shared__ __align__(8) unsigned long long bar[4];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    float* ys = smt + w * 32 * F;
    const unsigned bs = unsigned(__cvta_generic_to_shared(&bar[w]));
    if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bs));
    __syncwarp();
    const unsigned long long wid = blockIdx.x * 4ull + w, nw = gridDim.x * 4ull;
    float acc = 0.f;
    unsigned phase = 0;
    for (unsigned long long c = wid * 32; c < m; c += nw * 32) {
        const unsigned myrow = hsh(unsigned(c + lane)) % n;
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bs), "r"(32u * F * 4) : "memory");
        __syncwarp();
        const unsigned dst = unsigned(__cvta_generic_to_shared(ys + lane * F));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                     ::"r"(dst), "l"(b + std::uint64_t(myrow) * F), "r"(F * 4), "r"(bs) : "memory");
        asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}\n"
                     ::"r"(bs), "r"(phase) : "memory");
        phase ^= 1;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const float4 v = *reinterpret_cast<const float4*>(ys + lane * F + 4 * q);
            acc += v.x + v.y + v.z + v.w;
        }
        __syncwarp();
    }
    if (acc == 12345.f) out[blockIdx.x * 128 + threadIdx.x] = acc;
}

int main() {
    const unsigned n = 232965;
    const unsigned long long m = 114615892ull;
    float *b, *out;
    cudaMalloc(&b, std::uint64_t(n) * F * 4);
    cudaMemset(b, 0, std::uint64_t(n) * F * 4);
    cudaMalloc(&out, 1 << 24);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double bytes = double(m) * F * 4;
    cudaFuncSetAttribute(smem_row, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32 * F * 4);
    cudaFuncSetAttribute(tma_row, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32 * F * 4);
    for (int blocks_per_sm : {4, 8, 16}) {
        const int grid = 148 * blocks_per_sm;
        for (int k = 0; k < 4; ++k) {
            float t[3];
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(e0);
                if (k == 0) lane_row<<<grid, 128>>>(b, n, m, out);
                if (k == 1) group_row<<<grid, 128>>>(b, n, m, out);
                if (k == 2) smem_row<<<grid, 128, 4 * 32 * F * 4>>>(b, n, m, out);
                if (k == 3) tma_row<<<grid, 128, 4 * 32 * F * 4>>>(b, n, m, out);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&t[rep], e0, e1);
            }
            const char* nm[] = {"lane-per-row LDG.128", "16-lanes-per-row LDG.128", "cp.async smem + LDS.128",
                                "TMA bulk row + LDS.128"};
            std::printf("%-28s blocks/SM %2d: %.3f ms  %.1f TB/s\n", nm[k], blocks_per_sm, t[2], bytes / (t[2] * 1e-3) / 1e12);
        }
    }
    std::printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
