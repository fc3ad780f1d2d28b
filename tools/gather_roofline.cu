// gather_roofline.cu -- microbenchmarks that bound the SpMM/SDDMM hot loop on
// B200: streaming copy (HBM), random row gathers from an L2-resident and an
// HBM-resident matrix, and the cost of the f32->f64 widening every product
// of the bit-exact f64 accumulation needs (F2F on the XU pipe vs an integer
// re-bias + exact DMUL scale on the ALU/FP64 pipes).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_roofline tools/gather_roofline.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e = (x);                                                         \
        if (e != cudaSuccess) {                                                      \
            std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            return 1;                                                                \
        }                                                                            \
    } while (0)

__global__ void copy_kernel(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        b[i] = a[i];
}

// widening modes: 0 = f32 accumulate (no widening), 1 = F2F + DFMA,
// 2 = integer re-bias + DFMA with 2^896-prescaled multiplier
__device__ __forceinline__ double widen_bits(float f) {
    // (double)f * 2^-896 for finite f: arithmetic shift replicates the sign
    // into bits 31..28, the mask keeps bit 31 and the 28 exponent/mantissa bits
    const int u = __float_as_int(f);
    const unsigned hi = unsigned(u >> 3) & 0x8FFFFFFFu;
    const unsigned lo = unsigned(u) << 29;
    return __hiloint2double(int(hi), int(lo));
}

template <int MODE, int U>
__global__ void __launch_bounds__(128) gather_kernel(const float* __restrict__ b,
                                                     const unsigned* __restrict__ idx, size_t nnz_per_row,
                                                     size_t n_out_rows, unsigned f, float* __restrict__ out) {
    // 16 lanes x float4 = 64 features per group; 2 groups per warp
    const int lane = threadIdx.x & 31, grp = lane >> 4, gl = lane & 15;
    const size_t row = ((blockIdx.x * size_t(blockDim.x) + threadIdx.x) >> 5) * 2 + grp;
    if (row >= n_out_rows) return;
    const unsigned* ip = idx + row * nnz_per_row;
    float facc[4] = {0, 0, 0, 0};
    double dacc[4] = {0, 0, 0, 0};
    const double scale = 0x1p896;
    for (size_t base = 0; base < nnz_per_row; base += 16) {
        const unsigned c = __ldg(ip + base + gl);
#pragma unroll
        for (int j0 = 0; j0 < 16; j0 += U) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const unsigned cj = __shfl_sync(0xffffffffu, c, grp * 16 + j0 + u);
                v[u] = __ldg(reinterpret_cast<const float4*>(b + size_t(cj) * f) + gl);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (MODE == 0) {
                    facc[0] += v[u].x; facc[1] += v[u].y; facc[2] += v[u].z; facc[3] += v[u].w;
                } else if (MODE == 1) {
                    dacc[0] = __fma_rn(0.75, double(v[u].x), dacc[0]);
                    dacc[1] = __fma_rn(0.75, double(v[u].y), dacc[1]);
                    dacc[2] = __fma_rn(0.75, double(v[u].z), dacc[2]);
                    dacc[3] = __fma_rn(0.75, double(v[u].w), dacc[3]);
                } else if (MODE == 3) {  // mixed: x,y on XU, z,w on ALU
                    const double s = 0.75 * scale;
                    dacc[0] = __fma_rn(0.75, double(v[u].x), dacc[0]);
                    dacc[1] = __fma_rn(0.75, double(v[u].y), dacc[1]);
                    dacc[2] = __fma_rn(s, widen_bits(v[u].z), dacc[2]);
                    dacc[3] = __fma_rn(s, widen_bits(v[u].w), dacc[3]);
                } else if (MODE == 4) {  // mixed: x on XU, y,z,w on ALU
                    const double s = 0.75 * scale;
                    dacc[0] = __fma_rn(0.75, double(v[u].x), dacc[0]);
                    dacc[1] = __fma_rn(s, widen_bits(v[u].y), dacc[1]);
                    dacc[2] = __fma_rn(s, widen_bits(v[u].z), dacc[2]);
                    dacc[3] = __fma_rn(s, widen_bits(v[u].w), dacc[3]);
                } else {
                    const double s = 0.75 * scale;
                    dacc[0] = __fma_rn(s, widen_bits(v[u].x), dacc[0]);
                    dacc[1] = __fma_rn(s, widen_bits(v[u].y), dacc[1]);
                    dacc[2] = __fma_rn(s, widen_bits(v[u].z), dacc[2]);
                    dacc[3] = __fma_rn(s, widen_bits(v[u].w), dacc[3]);
                }
            }
        }
    }
    float* o = out + row * f + gl * 4;
    if (MODE == 0) { o[0] = facc[0]; o[1] = facc[1]; o[2] = facc[2]; o[3] = facc[3]; }
    else { o[0] = float(dacc[0]); o[1] = float(dacc[1]); o[2] = float(dacc[2]); o[3] = float(dacc[3]); }
}

// exactness check of widen_bits*2^896 against the hardware conversion
__global__ void widen_check(unsigned* bad, unsigned long long start, unsigned long long count) {
    for (unsigned long long i = start + blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
         i < start + count; i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned u = unsigned(i);
        if (((u >> 23) & 0xFF) == 0xFF) continue;  // inf / nan handled separately
        const float f = __uint_as_float(u);
        const double a = double(f), b = widen_bits(f) * 0x1p896;
        if (__double_as_longlong(a) != __double_as_longlong(b)) atomicAdd(bad, 1u);
    }
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

int main() {
    // 1. HBM copy
    const size_t n4 = (size_t(1) << 30) / 16;  // 1 GiB
    float4 *a, *b;
    CK(cudaMalloc(&a, n4 * 16));
    CK(cudaMalloc(&b, n4 * 16));
    cudaMemset(a, 0, n4 * 16);
    float ms = time_it([&] { copy_kernel<<<148 * 16, 256>>>(a, b, n4); }, 5);
    std::printf("copy 1GiB: %.3f ms  %.1f GB/s (read+write)\n", ms, 2.0 * n4 * 16 / ms / 1e6);

    // 2. random gathers: 64 features (256 B rows), 512 nnz per row
    const unsigned f = 64;
    const size_t per_row = 512;
    const size_t out_rows = 224000;  // ~114.7M gathers
    std::vector<unsigned> h_idx(out_rows * per_row);
    unsigned long long s = 12345;
    for (int which = 0; which < 2; ++which) {
        const size_t n_b = which == 0 ? 232965 : 4000000;  // 60 MB (L2) vs 1 GB (HBM)
        for (auto& v : h_idx) {
            s = s * 6364136223846793005ULL + 1442695040888963407ULL;
            v = unsigned((s >> 33) % n_b);
        }
        unsigned* idx;
        float *bm, *out;
        CK(cudaMalloc(&idx, h_idx.size() * 4));
        CK(cudaMalloc(&bm, n_b * f * 4));
        CK(cudaMalloc(&out, out_rows * f * 4));
        cudaMemset(bm, 0, n_b * f * 4);
        CK(cudaMemcpy(idx, h_idx.data(), h_idx.size() * 4, cudaMemcpyHostToDevice));
        const double gbytes = double(out_rows) * per_row * f * 4 / 1e9;
        const unsigned blocks = unsigned((out_rows / 2 * 32 + 127) / 128);
        auto run = [&](auto kern, const char* name) {
            float t = time_it([&] { kern<<<blocks, 128>>>(bm, idx, per_row, out_rows, f, out); }, 3);
            std::printf("gather %s B=%s: %.3f ms  %.1f GB/s of gathered rows\n", name,
                        which == 0 ? "60MB(L2)" : "1GB(HBM)", t, gbytes / t * 1e3);
        };
        run(gather_kernel<0, 8>, "f32-acc  U=8 ");
        run(gather_kernel<0, 16>, "f32-acc  U=16");
        run(gather_kernel<1, 8>, "F2F+DFMA U=8 ");
        run(gather_kernel<1, 16>, "F2F+DFMA U=16");
        run(gather_kernel<2, 8>, "int+DFMA U=8 ");
        run(gather_kernel<2, 16>, "int+DFMA U=16");
        run(gather_kernel<3, 8>, "mix2+DFMA U=8 ");
        run(gather_kernel<4, 8>, "mix3+DFMA U=8 ");
        cudaFree(idx);
        cudaFree(bm);
        cudaFree(out);
    }
    // 3. exactness of the integer widening (all finite f32 bit patterns)
    unsigned* bad;
    CK(cudaMalloc(&bad, 4));
    cudaMemset(bad, 0, 4);
    widen_check<<<148 * 32, 256>>>(bad, 0, 1ull << 32);
    unsigned hb = 0;
    CK(cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost));
    std::printf("widen_bits * 2^896 != (double)f for %u finite f32 bit patterns\n", hb);
    return 0;
}
