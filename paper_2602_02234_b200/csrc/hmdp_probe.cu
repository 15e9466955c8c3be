// hmdp_probe.cu — measured FP32 FFMA throughput (the roofline denominator of
// the SIMT kernels).  16 independent FMA chains per thread, 8 x 256-thread CTAs
// per SM; timed with CUDA events.
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <string>

namespace hmdp {

__global__ __launch_bounds__(256) void k_ffma_probe(float* out, int iters, float b, float c) {
    float a[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) a[k] = threadIdx.x * 1e-7f + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int k = 0; k < 16; ++k) a[k] = fmaf(a[k], b, c);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += a[k];
    if (s == 1234.5f) out[blockIdx.x] = s;  // keep the chains alive
}

double probe_fp32_tflops(int ms) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = sms * 8, block = 256;
    float* out = nullptr;
    if (cudaMalloc(&out, grid * sizeof(float)) != cudaSuccess) throw std::runtime_error("probe alloc");
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](int iters) {
        cudaEventRecord(e0);
        k_ffma_probe<<<grid, block>>>(out, iters, 0.99999f, 1e-7f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float t = 0.f;
        cudaEventElapsedTime(&t, e0, e1);
        return static_cast<double>(t);
    };
    run(64);  // warm-up
    int iters = 256;
    double t = run(iters);
    while (t < ms * 0.5 && iters < (1 << 24)) {
        iters *= 2;
        t = run(iters);
    }
    double best = 1e30;
    for (int r = 0; r < 5; ++r) best = std::min(best, run(iters));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    const double flops = 2.0 * grid * block * static_cast<double>(iters) * 8 * 16;
    return flops / (best * 1e-3) / 1e12;
}

}  // namespace hmdp
