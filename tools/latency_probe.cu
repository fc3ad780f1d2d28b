// latency_probe.cu -- dependent-chain latencies on B200 (clock64 cycles per op):
// DFMA, F2F.F64.F32 feeding DFMA, LDS -> F2F -> DFMA (the long-row consumer body).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_chain(double* out, long long* cyc, int n, double m, double a) {
    double x = threadIdx.x * 1e-3;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __fma_rn(x, m, a);
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = x; cyc[0] = t1 - t0; }
}
__global__ void lds_f2f_dfma_chain(const float* g, double* out, long long* cyc, int n) {
    __shared__ float s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = g[i];
    __syncthreads();
    double acc = 0.0;
    long long t0 = clock64();
    for (int j = 0; j < n; ++j) {
        const double v = double(s[(j * 7) & 4095]);
        const double bb = double(s[(j * 13 + threadIdx.x) & 4095]);
        acc = __fma_rn(v, bb, acc);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = acc; cyc[0] = t1 - t0; }
}
int main() {
    double* out; long long* cyc; float* g;
    cudaMalloc(&out, 8); cudaMalloc(&cyc, 8); cudaMalloc(&g, 4096 * 4); cudaMemset(g, 0, 4096 * 4);
    const int n = 1 << 16;
    long long h;
    dfma_chain<<<1, 32>>>(out, cyc, n, 0.999, 1e-3); cudaDeviceSynchronize();
    dfma_chain<<<1, 32>>>(out, cyc, n, 0.999, 1e-3); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent chain: %.2f cycles/op\n", double(h) / n);
    lds_f2f_dfma_chain<<<1, 64>>>(g, out, cyc, n); cudaDeviceSynchronize();
    lds_f2f_dfma_chain<<<1, 64>>>(g, out, cyc, n); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("LDS+F2F+DFMA loop (1 chain/thread, 2 warps): %.2f cycles/iter\n", double(h) / n);
    lds_f2f_dfma_chain<<<1, 256>>>(g, out, cyc, n); cudaDeviceSynchronize();
    lds_f2f_dfma_chain<<<1, 256>>>(g, out, cyc, n); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("LDS+F2F+DFMA loop (1 chain/thread, 8 warps): %.2f cycles/iter\n", double(h) / n);
    return 0;
}
