// Cost of a chain of dependent kernels in one CUDA graph (dev probe):
// N kernels, each grid x block with S bytes of dynamic smem, optionally PDL.
// Each kernel does a trivial dependent read/write so the chain is real.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", #x, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)
__global__ void k_step(float* buf, int iters) {
    extern __shared__ float sm[];
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    float v = buf[i];
    for (int k = 0; k < iters; ++k) v = v * 0.999f + 0.001f;
    sm[threadIdx.x] = v;
    buf[i] = v + sm[(threadIdx.x + 1) % blockDim.x] * 0.f;
}
int main() {
    float* buf;
    CK(cudaMalloc(&buf, 1 << 24));
    cudaMemset(buf, 0, 1 << 24);
    cudaFuncSetAttribute(k_step, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    const int N = 70;
    int grids[] = {146, 146, 146, 292, 582};
    int blocks[] = {512, 512, 128, 256, 128};
    int smems[] = {0, 90 * 1024, 0, 16 * 1024, 0};
    for (int pdl = 0; pdl < 2; ++pdl)
        for (int c = 0; c < 5; ++c) {
            cudaGraph_t g;
            CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            for (int k = 0; k < N; ++k) {
                cudaLaunchConfig_t cfg{};
                cfg.gridDim = dim3(grids[c]);
                cfg.blockDim = dim3(blocks[c]);
                cfg.dynamicSmemBytes = smems[c] > blocks[c] * 4 ? smems[c] : blocks[c] * 4;
                cfg.stream = st;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at;
                cfg.numAttrs = pdl;
                CK(cudaLaunchKernelEx(&cfg, k_step, buf, 4));
            }
            CK(cudaStreamEndCapture(st, &g));
            cudaGraphExec_t ex;
            CK(cudaGraphInstantiate(&ex, g, 0));
            for (int w = 0; w < 5; ++w) cudaGraphLaunch(ex, st);
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a, st);
            const int R = 50;
            for (int r = 0; r < R; ++r) cudaGraphLaunch(ex, st);
            cudaEventRecord(b, st);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("pdl=%d grid=%d block=%d smem=%dK: %.2f us per kernel\n", pdl, grids[c], blocks[c],
                   smems[c] / 1024, ms * 1e3 / (R * N));
            cudaGraphExecDestroy(ex);
            cudaGraphDestroy(g);
        }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
