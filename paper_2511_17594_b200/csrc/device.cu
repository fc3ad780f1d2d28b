// device.cu -- GPU DeviceProfile (include/autosage/device.hpp:12-27
// re-targeted): device_sig = "<GPU name> sm_<cc>|cores=<SMs>|<artifact
// version>" (no UUID, so every B200 of a box shares cached decisions), and
// bw_eff / flops_eff from one-time calibration kernels: a streaming f64
// triad a = b + s*c (src/device.cpp:42-62 analogue) and independent DFMA
// chains (src/device.cpp:66-95 analogue; f64 because the operators
// accumulate in f64).
#include "graph.hpp"
#include "ops.hpp"

#include <algorithm>
#include <cstdio>
#include <map>
#include <mutex>

namespace asb {

namespace {

__global__ void triad_kernel(double* __restrict__ a, const double* __restrict__ b,
                             const double* __restrict__ c, double s, std::uint64_t n) {
    for (std::uint64_t i = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += std::uint64_t(gridDim.x) * blockDim.x)
        a[i] = b[i] + s * c[i];
}

__global__ void fill_kernel(double* a, double v, std::uint64_t n) {
    for (std::uint64_t i = blockIdx.x * std::uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += std::uint64_t(gridDim.x) * blockDim.x)
        a[i] = v;
}

__global__ void dfma_kernel(double* sink, int iters, double seed) {
    constexpr int kChains = 8;
    double x[kChains];
#pragma unroll
    for (int k = 0; k < kChains; ++k) x[k] = seed + 0.01 * k + 1e-9 * threadIdx.x;
    const double m = 0.999999, d = 1e-7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < kChains; ++k) x[k] = __fma_rn(x[k], m, d);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < kChains; ++k) s += x[k];
    if (s == 12345.678) sink[0] = s;  // keep the chains observable
}

int sm_count(int device) {
    int sms = 0;
    ASB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    return sms;
}

} // namespace

double measure_gpu_bandwidth(int device) {
    DeviceGuard dg(device);
    const std::uint64_t n = 32ull << 20;  // 3 x 256 MiB of doubles
    DevBuf<double> a(n), b(n), c(n);
    cudaStream_t s;
    ASB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const unsigned blocks = unsigned(sm_count(device) * 8);
    fill_kernel<<<blocks, 256, 0, s>>>(b.get(), 1.0, n);
    fill_kernel<<<blocks, 256, 0, s>>>(c.get(), 2.0, n);
    count_launch(2);
    cudaEvent_t e0, e1;
    ASB_CUDA(cudaEventCreate(&e0));
    ASB_CUDA(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int pass = 0; pass < 4; ++pass) {
        ASB_CUDA(cudaEventRecord(e0, s));
        triad_kernel<<<blocks, 256, 0, s>>>(a.get(), b.get(), c.get(), 1.0 + pass, n);
        check_launch("triad_kernel");
        ASB_CUDA(cudaEventRecord(e1, s));
        ASB_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        ASB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        if (pass > 0) best = std::min(best, ms);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s);
    return 3.0 * double(n) * sizeof(double) / (double(best) * 1e-3);
}

double measure_gpu_flops(int device) {
    DeviceGuard dg(device);
    DevBuf<double> sink(1);
    cudaStream_t s;
    ASB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const unsigned blocks = unsigned(sm_count(device) * 8);
    const int threads = 256, iters = 1 << 14;
    cudaEvent_t e0, e1;
    ASB_CUDA(cudaEventCreate(&e0));
    ASB_CUDA(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int pass = 0; pass < 4; ++pass) {
        ASB_CUDA(cudaEventRecord(e0, s));
        dfma_kernel<<<blocks, threads, 0, s>>>(sink.get(), iters, 0.5 + 1e-3 * pass);
        check_launch("dfma_kernel");
        ASB_CUDA(cudaEventRecord(e1, s));
        ASB_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        ASB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        if (pass > 0) best = std::min(best, ms);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s);
    const double flops = 2.0 * 8.0 * double(iters) * double(blocks) * threads;
    return flops / (double(best) * 1e-3);
}

std::string gpu_device_tag(int device) {
    cudaDeviceProp p{};
    ASB_CUDA(cudaGetDeviceProperties(&p, device));
    char buf[320];
    std::snprintf(buf, sizeof buf, "%s sm_%d%d", p.name, p.major, p.minor);
    return buf;
}

// DeviceProfile::host() analogue: calibrated once per device per process.
const as_device_profile& gpu_profile(int device) {
    static std::mutex mu;
    static std::map<int, as_device_profile> profiles;
    std::lock_guard<std::mutex> lk(mu);
    auto it = profiles.find(device);
    if (it != profiles.end()) return it->second;
    as_device_profile dp{};
    dp.cores = std::uint64_t(sm_count(device));
    std::snprintf(dp.device_sig, sizeof dp.device_sig, "%s|cores=%llu|%s",
                  gpu_device_tag(device).c_str(), (unsigned long long)dp.cores, kArtifactVersion);
    dp.bw_eff = measure_gpu_bandwidth(device);
    dp.flops_eff = measure_gpu_flops(device);
    dp.model = AS_MODEL_B200;
    return profiles.emplace(device, dp).first->second;
}

} // namespace asb
