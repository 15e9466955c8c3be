// hmdp_tc.cu — 5th-generation tensor cores (tcgen05) for the dense atom-level MLP
// contractions, in 3xTF32 (FP32-accurate: single-pass TF32 misses the north-star
// tolerance by 2-4 orders of magnitude).
//
//   k_tc_chain   a chain of up to 3 dense layers y = act(x W^T + b) over 128-row
//                tiles (one CTA of 4 warps per tile): operands staged in shared
//                memory in the canonical no-swizzle K-major UMMA layout, hi/lo TF32
//                split (x = x_hi + x_lo, W = W_hi + W_lo; x W^T ~ x_hi W_hi^T +
//                x_hi W_lo^T + x_lo W_hi^T), one elected thread issues
//                tcgen05.mma.cta_group::1.kind::tf32 (M = 128, N = layer width,
//                K = 8 per instruction) into an FP32 accumulator in TMEM, completion
//                through tcgen05.commit -> mbarrier, epilogue by tcgen05.ld
//                (32x32b: warp w reads TMEM lanes 32w..32w+31 = its 32 rows) +
//                bias + tanh in registers; intermediate layers go back to shared
//                memory (re-split hi/lo) as the next layer's A operand, the last
//                layer to global memory.
//   k_tc_probe   raw kind::tf32 MMA throughput (M = 128, N = 256, K = 8 back to
//                back into one TMEM accumulator, one CTA per SM) -- the measured
//                tensor-core denominator; 3xTF32 delivers a third of it.
//
// The reference's dense contractions are MlpT::forward / backward
// (/root/reference/proj/src/nn/inference.cpp:87-138): W row-major [out][in], which is
// exactly the K-major B operand (N = out rows, K = in contiguous).
#include <cuda_runtime.h>

#include <cstdint>

#include <algorithm>
#include <stdexcept>

#include "hmdp_common.cuh"

namespace hmdp {

namespace tc {

constexpr int kRows = 128;  // UMMA M (cta_group::1)
constexpr int kMaxK = 64;
constexpr int kMaxN = 64;
constexpr int kMaxLayers = 3;

struct Layer {
    const float* W;  // [N][ldw] row-major (the model's [out][in]), first K columns used
    const float* b;  // [N] (nullable)
    int K, N, ldw;   // K % 8 == 0, K <= 64; N in {32, 64}
    int act;         // 0 linear, 1 tanh
    int res;         // 1: + the chain input's first N columns (residual), after act
    float* out;      // [rows][ld_out] this layer's output (nullable except the last)
    int ld_out;
};
struct Chain {
    Layer L[kMaxLayers];
    int n_layers;
    const float* x;  // [rows][ldx], first K0 columns used
    int ldx;
    int rows;
};

// Byte offset of element (r, k) in the canonical no-swizzle K-major layout:
// 8 x 16-byte core matrices (8 rows x 4 tf32), k-chunks LBO = 128 B apart, 8-row
// groups SBO = (K/4) * 128 B apart.
__device__ __forceinline__ uint32_t kmajor_off(int r, int k, int K) {
    return static_cast<uint32_t>((r >> 3) * (K >> 2) * 128 + (k >> 2) * 128 + (r & 7) * 16 +
                                 (k & 3) * 4);
}

// UMMA shared-memory descriptor (sm_100): start >> 4 [0,14), LBO >> 4 [16,30),
// SBO >> 4 [32,46), version 1 [46,48), layout SWIZZLE_NONE (0) [61,64).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) |
           (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
           (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// Instruction descriptor, kind::tf32: D F32 [4,6) = 1, A TF32 [7,10) = 2,
// B TF32 [10,13) = 2, both K-major, N >> 3 at [17,23), M >> 4 at [24,29).
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ float to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void commit(uint64_t* mbar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"l"(
                     static_cast<uint64_t>(__cvta_generic_to_shared(mbar)))
                 : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* mbar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                     static_cast<unsigned>(__cvta_generic_to_shared(mbar))),
                 "r"(count)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* mbar, unsigned parity) {
    const unsigned mb = static_cast<unsigned>(__cvta_generic_to_shared(mbar));
    unsigned done = 0;
    while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
            "selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(mb), "r"(parity)
            : "memory");
}

// 32 consecutive TMEM columns of this thread's lane (row) -> registers.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
        "%28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int c = 0; c < 32; ++c) v[c] = __uint_as_float(r[c]);
}

// fp32 value -> hi/lo tf32 pair in the two A (or B) images at byte offset `off`
__device__ __forceinline__ void put_split(char* hi, char* lo, uint32_t off, float x) {
    const float h = to_tf32(x);
    *reinterpret_cast<float*>(hi + off) = h;
    *reinterpret_cast<float*>(lo + off) = to_tf32(x - h);
}

// Shared memory: A hi/lo (128 x 64 tf32 each), B hi/lo (64 x 64 each), barrier, TMEM slot.
struct Smem {
    alignas(128) char a_hi[kRows * kMaxK * 4];
    alignas(128) char a_lo[kRows * kMaxK * 4];
    alignas(128) char b_hi[kMaxN * kMaxK * 4];
    alignas(128) char b_lo[kMaxN * kMaxK * 4];
    uint64_t mbar;
    uint32_t tmem_base;
};

__global__ __launch_bounds__(128, 1) void k_tc_chain(Chain ch) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5;
    const int row0 = blockIdx.x * kRows;
    const int r = row0 + tid;  // this thread's row (TMEM lane tid)
    if (warp == 0) {  // TMEM: 64 columns (one FP32 accumulator of N <= 64)
        asm volatile(
            "tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(
                static_cast<unsigned>(__cvta_generic_to_shared(&sm.tmem_base)))
            : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        mbar_init(&sm.mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // layer 0 input: this thread's row, hi/lo split into the A images
    {
        const int K = ch.L[0].K;
        const float* xr = ch.x + static_cast<long long>(r) * ch.ldx;
        for (int k = 0; k < K; k += 4) {
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (r < ch.rows) v = *reinterpret_cast<const float4*>(xr + k);
            put_split(sm.a_hi, sm.a_lo, kmajor_off(tid, k, K), v.x);
            put_split(sm.a_hi, sm.a_lo, kmajor_off(tid, k + 1, K), v.y);
            put_split(sm.a_hi, sm.a_lo, kmajor_off(tid, k + 2, K), v.z);
            put_split(sm.a_hi, sm.a_lo, kmajor_off(tid, k + 3, K), v.w);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = sm.tmem_base;
    unsigned parity = 0;
    for (int li = 0; li < ch.n_layers; ++li) {
        const Layer& L = ch.L[li];
        const int K = L.K, N = L.N;
        // B = W [N][K]: the whole CTA splits it into the B images
        for (int t = tid; t < N * K; t += kRows) {
            const int n = t / K, k = t - n * K;
            put_split(sm.b_hi, sm.b_lo, kmajor_off(n, k, K), __ldg(L.W + n * L.ldw + k));
        }
        // generic-proxy smem writes -> visible to the tensor core (async proxy)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t a_hi = static_cast<uint32_t>(__cvta_generic_to_shared(sm.a_hi));
            const uint32_t a_lo = static_cast<uint32_t>(__cvta_generic_to_shared(sm.a_lo));
            const uint32_t b_hi = static_cast<uint32_t>(__cvta_generic_to_shared(sm.b_hi));
            const uint32_t b_lo = static_cast<uint32_t>(__cvta_generic_to_shared(sm.b_lo));
            const uint32_t sbo = static_cast<uint32_t>(K >> 2) * 128;
            const uint32_t idesc = idesc_tf32(kRows, N);
            for (int ks = 0; ks < K / 8; ++ks) {  // K = 8 per instruction = 2 k-chunks
                const uint32_t o = ks * 256;
                const uint64_t ah = smem_desc(a_hi + o, 128, sbo), al = smem_desc(a_lo + o, 128, sbo);
                const uint64_t bh = smem_desc(b_hi + o, 128, sbo), bl = smem_desc(b_lo + o, 128, sbo);
                // small terms first, then the leading hi x hi product
                mma_tf32(tmem, al, bh, idesc, ks > 0 ? 1u : 0u);
                mma_tf32(tmem, ah, bl, idesc, 1u);
                mma_tf32(tmem, ah, bh, idesc, 1u);
            }
            commit(&sm.mbar);
        }
        mbar_wait(&sm.mbar, parity);
        parity ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // epilogue: warp w holds rows 32w..32w+31 (TMEM lanes), N columns
        const bool last = li == ch.n_layers - 1;
        for (int c0 = 0; c0 < N; c0 += 32) {
            float v[32];
            tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                float y = v[c] + (L.b ? __ldg(L.b + c0 + c) : 0.f);
                if (L.act == 1) y = tanhf(y);
                v[c] = y;
            }
            if (L.res && r < ch.rows) {
                const float* xr = ch.x + static_cast<long long>(r) * ch.ldx + c0;
#pragma unroll
                for (int c = 0; c < 32; c += 4) {
                    const float4 q = *reinterpret_cast<const float4*>(xr + c);
                    v[c] += q.x;
                    v[c + 1] += q.y;
                    v[c + 2] += q.z;
                    v[c + 3] += q.w;
                }
            }
            if (L.out && r < ch.rows) {
                float* yr = L.out + static_cast<long long>(r) * L.ld_out + c0;
#pragma unroll
                for (int c = 0; c < 32; c += 4)
                    *reinterpret_cast<float4*>(yr + c) = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
            }
            if (!last) {  // next layer's A operand (its K = this N)
#pragma unroll
                for (int c = 0; c < 32; ++c) put_split(sm.a_hi, sm.a_lo, kmajor_off(tid, c0 + c, N), v[c]);
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();  // A / B images and the accumulator are free for the next layer
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem) : "memory");
}

// Raw kind::tf32 MMA issue rate: M = 128, N = 256, K = 8, `iters` instructions back
// to back into one accumulator (operands: whatever the shared memory holds).
__global__ __launch_bounds__(128, 1) void k_tc_probe(int iters, float* out) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x;
    for (int t = tid; t < (128 + 256) * 8; t += blockDim.x)
        reinterpret_cast<float*>(smem_raw)[t] = 0.f;
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                         static_cast<unsigned>(__cvta_generic_to_shared(&tmem_base)))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        mbar_init(&mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base;
    if (tid == 0) {
        const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
        const uint32_t b = a + 128 * 8 * 4;
        const uint64_t ad = smem_desc(a, 128, 256), bd = smem_desc(b, 128, 256);
        const uint32_t idesc = idesc_tf32(128, 256);
        for (int i = 0; i < iters; ++i) mma_tf32(tmem, ad, bd, idesc, i > 0 ? 1u : 0u);
        commit(&mbar);
    }
    mbar_wait(&mbar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    float v[32];
    tmem_ld32(tmem + (static_cast<uint32_t>((tid >> 5) * 32) << 16), v);
    if (v[0] == 1234.5f) out[blockIdx.x] = v[1];
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid < 32)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

}  // namespace tc

cudaError_t tc_configure() {
    return cudaFuncSetAttribute(tc::k_tc_chain, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(sizeof(tc::Smem)));
}

// One dense layer of a chain (host description).
struct TcLayer {
    const float* W;
    const float* b;
    int K, N, ldw, act, res;
    float* out;
    int ld_out;
};

// y_l = act_l(y_{l-1} W_l^T + b_l) [+ x residual], y_0 = x: rows x K0 in, every layer's
// output optionally stored; FP32 in / out, 3xTF32 on the tensor cores.
void launch_tc_chain(int rows, const float* x, int ldx, int n_layers, const TcLayer* L,
                     cudaStream_t st) {
    tc::Chain ch{};
    if (n_layers < 1 || n_layers > tc::kMaxLayers) throw std::invalid_argument("1..3 layers");
    for (int l = 0; l < n_layers; ++l) {
        const TcLayer& q = L[l];
        if (q.K % 8 || q.K < 8 || q.K > tc::kMaxK || q.N % 32 || q.N < 32 || q.N > tc::kMaxN)
            throw std::invalid_argument("tcgen05 chain: K % 8 == 0, K <= 64, N in {32, 64}");
        if (l > 0 && q.K != L[l - 1].N) throw std::invalid_argument("tcgen05 chain: K_l != N_{l-1}");
        ch.L[l] = tc::Layer{q.W, q.b, q.K, q.N, q.ldw, q.act, q.res, q.out, q.ld_out};
    }
    if (!L[n_layers - 1].out) throw std::invalid_argument("tcgen05 chain: last layer needs out");
    ch.n_layers = n_layers;
    ch.x = x;
    ch.ldx = ldx;
    ch.rows = rows;
    const int grid = (rows + tc::kRows - 1) / tc::kRows;
    if (grid > 0) tc::k_tc_chain<<<grid, 128, sizeof(tc::Smem), st>>>(ch);
}

// Raw tcgen05 kind::tf32 throughput (TFLOP/s), one CTA per SM, timed with events.
double probe_tcgen05_tf32_tflops(int ms) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    float* out = nullptr;
    if (cudaMalloc(&out, sms * sizeof(float)) != cudaSuccess) throw std::runtime_error("probe alloc");
    const size_t smem = (128 + 256) * 8 * 4;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](int iters) {
        cudaEventRecord(e0);
        tc::k_tc_probe<<<sms, 128, smem>>>(iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float t = 0.f;
        cudaEventElapsedTime(&t, e0, e1);
        return static_cast<double>(t);
    };
    run(64);
    int iters = 1024;
    double t = run(iters);
    while (t < ms * 0.5 && iters < (1 << 24)) {
        iters *= 2;
        t = run(iters);
    }
    double best = 1e30;
    for (int rep = 0; rep < 5; ++rep) best = std::min(best, run(iters));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string("tcgen05 probe: ") + cudaGetErrorString(e));
    return 2.0 * 128 * 256 * 8 * static_cast<double>(iters) * sms / (best * 1e-3) / 1e12;
}

}  // namespace hmdp
