// hmdp_net.cu — the DP network kernels (embedding, message layers, fitting,
// reverse mode, forces/virial), sm_100a.
//
// Decomposition: ONE WARP PER ATOM, lane = feature channel.  A CTA of W warps
// (W = 2..16, chosen from the system size so every SM gets work) stages the
// weight matrices its phase needs into shared memory once, then its warps
// grid-stride over atoms independently — no CTA barrier inside the atom loop,
// only __syncwarp.  Per atom:
//   * per-edge work runs lane = channel with edges taken 8 at a time (8 row loads
//     in flight per lane, every row access one coalesced 128-byte line); the
//     per-edge scalars are loaded lane = edge and staged in the warp's shared
//     scratch, so the edge loop reads them as shared-memory broadcasts;
//   * the atom-level MLP layers are warp mat-vecs (wmv): lane o reads row o of
//     the staged matrix with 128-bit loads (rows padded by 16 bytes, so the 8
//     lanes of each quarter-warp phase hit distinct banks) and x as broadcasts.
// Many atoms are in flight per SM (up to 32 warps), which is what this
// latency-bound workload needs (the FLOPs per step are a few hundred MFLOP).
//
// Dataflow is "push" into mirror slots (DevGraph, hmdp_device.cuh): the producer
// of a per-neighbour quantity writes it into the slot its consumer reads
// contiguously, so no kernel chases an index to gather a neighbour's row:
//   P_j = W1h h_j        pushed by j into the out-slots of j's in-edges
//   dz_e (h_j adjoint)   pushed by the edge's source into e's mirror slot
//   g_e                  pushed by the edge's source into e's mirror slot
// Every slot is written by exactly one lane and every sum runs in a fixed
// order: deterministic, no float atomics (the reference's scatters dh_j += ...,
// F_j -= ..., inference.cpp:343, :380, become these pushes + local sums).
//
// Linearity of the message MLP is exploited exactly (same function, fewer FLOPs):
//   forward   z_e = tanh(W1h h_j + W1b b_e + b1) with the per-ATOM projection
//             P_j = W1h h_j computed once per layer instead of once per edge;
//             msum_i = sum_e s_e (W2 z_e + b2) = W2 (sum_e s_e z_e) + (sum_e s_e) b2,
//             and msum enters the update MLP only through U1m msum, so W2 is folded
//             into it once at upload: U1m msum = (U1m W2) t + ssum (U1m b2) with
//             t = sum_e s_e z_e (one 64-input mat-vec [h; t] instead of two)
//   backward  with dmsum_i from the update MLP, v = W2^T dmsum_i, c0 = dmsum_i.b2;
//             folded likewise: v = (U1m W2)^T dz_u (the second half of the fused
//             transposed update matrix), c0 = dz_u . (U1m b2):
//             dsc_e = dmsum_i . mo_e = v . z_e + c0,  dz_e = s_e v (1 - z_e^2),
//             dE/dr_e += dsc_e s'(r_e) + sum_k b'_e[k] (W1b^T dz_e)[k],
//             dE/dh_j += W1h^T sum_{e in in(j)} dz_e  (one mat-vec per atom).
//
// Reference correspondence (paths relative to /root/reference/proj):
//   k_embed        edge radial + descriptor + embedding fwd   src/nn/inference.cpp:214-249
//                  [FUSE_FIT: + fitting fwd/bwd + embedding bwd, :288-311, :355-370]
//   k_msg_fwd      message layer fwd                          :251-286
//                  [LAST: + fitting fwd/bwd + top message layer bwd, :288-353]
//   k_msg_bwd      message layer bwd (lower layers)           :313-353
//   k_embed_bwd    embedding + descriptor adjoint             :355-370
//   k_force        force / virial (gather form) + E, W sums   :288-298, :372-387
//                  [+ velocity Verlet tail, src/integrators.cpp:32-47]
#include <algorithm>
#include <cstdio>
#include <map>
#include <mutex>
#include <tuple>
#include <cstdlib>

#include "hmdp_common.cuh"

namespace hmdp {

int num_sms();  // hmdp_nbr.cu
struct TcLayer {  // hmdp_tc.cu
    const float* W;
    const float* b;
    int K, N, ldw, act, res;
    float* out;
    int ld_out;
};
void launch_tc_chain(int rows, const float* x, int ldx, int n_layers, const TcLayer* L,
                     cudaStream_t st);
// Embedding MLP + P^0 on the tensor cores (tcgen05 3xTF32 chain) instead of the SIMT
// team mat-vecs: HMDP_TC_EMBED=1 on, 0 off, unset -> from kTcEmbedMinAtoms atoms up.
// A/B on B200 (DPA3 MD step, profiles/round2/tcgen05.md): SIMT 6218 vs tcgen05 5433
// steps/s at 2PTC (4114 atoms), 996 vs 978 at 2PTC x (2,2,2) (32 912 atoms) -- the
// K = N = 32 chain is latency-bound (tensor pipe active 1-6 %), so the fused SIMT
// path stays the default at every measured size.
constexpr int kTcEmbedMinAtoms = 1 << 30;
static bool tc_embed_on(int n) {
    static const int env = [] {
        const char* e = std::getenv("HMDP_TC_EMBED");
        return e ? std::atoi(e) : -1;
    }();
    return env >= 0 ? env != 0 : n >= kTcEmbedMinAtoms;
}

// Dev-only stage timing (build with HMDP_NVCC_DEFS=-DHMDP_TPROBE): lane 0 of every
// warp adds the clock64 cycles spent between consecutive TP(k) marks.
#ifdef HMDP_TPROBE
__device__ unsigned long long g_tprobe[32];
#define TP_START long long tp_last_ = clock64()
#define TP(k)                                                       \
    do {                                                            \
        if ((threadIdx.x & 31) == 0) {                              \
            const long long t_ = clock64();                         \
            atomicAdd(&g_tprobe[k], (unsigned long long)(t_ - tp_last_)); \
            tp_last_ = t_;                                          \
        }                                                           \
    } while (0)
#else
#define TP_START
#define TP(k)
#endif

// 20: measured against 16 on B200 (DPA3 FP32, flushed L2): 2PTC 6.94k -> 7.48k,
// 3LZM 9.13k -> 10.10k, 1UBQ 12.5k -> 16.7k steps/s (1UBQ: 9 teams per CTA no
// longer need a second wave of CTAs); 24 spills more (2PTC 7.04k).
#ifndef HMDP_TEAM_CTA_WARPS
#define HMDP_TEAM_CTA_WARPS 20
#endif
constexpr int kMaxWarps = 16;  // warps per CTA (network kernels, 1-warp teams)
// warps per CTA of the 2- and 4-warp-team kernels (one CTA per SM: the register
// budget per thread is 65536 / (32 x this))
// (FP64, the parity mode, keeps 16: its registers would not fit more).  WIDE: a
// second build of the FP32 2-warp-team kernels for 28-warp CTAs (72 registers),
// taken when 14 teams per SM need fewer rounds of atoms than 10 (net_shape).
#ifndef HMDP_WIDE_CTA_WARPS
#define HMDP_WIDE_CTA_WARPS 28
#endif
template <typename T, int G, bool WIDE = false>
constexpr int kCtaWarps = (G == 1 || sizeof(T) > 4) ? kMaxWarps
                          : (WIDE ? HMDP_WIDE_CTA_WARPS : HMDP_TEAM_CTA_WARPS);
// The push-form message kernels (domain decomposition, general CSR graphs) keep
// 16-warp CTAs: their backward holds the pushed-row batches and spills at 96
// registers (k_msg_bwd 400 B); net_shape(push) sizes their launches.
constexpr int kPushWarps = kMaxWarps;
// Message layers: store every layer's z_e rows (false) or only the LAST layer's and
// recompute z_e = tanh(W1b b_e + b1 + P^l_j) in the lower layers' backward (true:
// a tanh + 8 FMAs per edge channel instead of a 128-byte row that spills to HBM at
// 2PTC).  Measured on B200 (DPA3 2PTC, FP32): recompute made k_msg_bwd 31.7 -> 52.4
// us (step 152 -> 177 us) -- the kernel is issue/latency-bound, not HBM-bound.
constexpr bool kRecomputeZ = false;
// Resident CTAs per SM the register budget is sized for: 2 (64 registers) for the
// 1-warp teams of large systems — more atoms in flight; 1 (128 registers) for
// the 2/4-warp teams of small systems, whose chains would spill at 64 (measured:
// DPA2 2PTC +11 %, DPA3 2PTC +2 %, DPA3 1YRF -33 % if forced to 2).
template <int G>
constexpr int kNetMinCTAs = G == 1 ? 2 : 1;
#ifndef HMDP_FORCE_CTA
#define HMDP_FORCE_CTA 128
#endif
constexpr int kForceCTA = HMDP_FORCE_CTA;  // small CTAs: every SM gets atoms in small systems
// edges per unrolled batch (row loads in flight per lane; fewer for FP64 registers)
template <typename T>
constexpr int kU = sizeof(T) == 4 ? 8 : 4;

// Staged matrices: rows padded by 16 bytes (row stride in elements).
template <typename T>
__host__ __device__ constexpr int pad_ld(int cols) {
    return cols + 16 / static_cast<int>(sizeof(T));
}
template <typename T>
__host__ __device__ constexpr int mat_elems(int rows, int cols) {
    return rows * pad_ld<T>(cols);
}

// Per-warp shared scratch.
template <typename T>
struct WarpSmem {
    alignas(16) T x[64];
    alignas(16) T y[64];
    alignas(16) T t[32];
    alignas(16) T ed[32][20];  // edge scalars: (s, s', c0 | -, -, b or b'[8], [b[8]])
    alignas(16) T red[2][64];  // team-sum partials (double-buffered)
    T reds[2];
    int emir[32];  // staged mirror slots
    int ety[32];   // staged neighbour types
    int enb[32];   // staged neighbour indices (P_j row gathers)
};

// Bump allocator over the dynamic shared memory: staged matrices, then the
// warps' scratch.  view() only assigns the layout; load() fills it with ONE bulk
// copy (TMA engine, cp.async.bulk) of the kernel's pre-laid-out weight image
// (DevModel::img_*, built at upload in exactly this order), completed on an
// mbarrier — no per-thread copy loop.
template <typename T>
struct Smem {
    T* base;
    T* cur;
    __device__ explicit Smem(T* b) : base(b), cur(b) {}
    template <int R, int C>
    __device__ const T* view() {
        T* dst = cur;
        cur += R * pad_ld<T>(C);
        return dst;
    }
    // thread 0: arm the mbarrier and issue the copy; callers then __syncthreads()
    // (publishes the mbarrier init) and wait()
    __device__ void load(const T* img, unsigned long long* mbar) const {
        if (threadIdx.x != 0) return;
        const unsigned bytes = static_cast<unsigned>((cur - base) * sizeof(T));
        const unsigned mb = static_cast<unsigned>(__cvta_generic_to_shared(mbar));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes)
                     : "memory");
        constexpr unsigned kChunk = 32768;
        for (unsigned off = 0; off < bytes; off += kChunk) {
            const unsigned n = bytes - off < kChunk ? bytes - off : kChunk;
            const unsigned dst = static_cast<unsigned>(
                __cvta_generic_to_shared(reinterpret_cast<char*>(base) + off));
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
                "[%3];" ::"r"(dst),
                "l"(reinterpret_cast<const char*>(img) + off), "r"(n), "r"(mb)
                : "memory");
        }
    }
    __device__ static void wait(unsigned long long* mbar) {
        const unsigned mb = static_cast<unsigned>(__cvta_generic_to_shared(mbar));
        unsigned done = 0;
        while (!done)
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; "
                "selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(mb)
                : "memory");
    }
    // The staged matrices end 16-byte aligned (rows padded to a multiple of 16
    // bytes), so the scratch follows directly.  Pointer arithmetic from the
    // __shared__ base (no integer round trip) keeps the shared state space visible
    // to the compiler: LDS/STS instead of generic loads that may alias global
    // stores and so pin the edge loops' schedule.
    __device__ WarpSmem<T>& warp_scratch() const {
        return reinterpret_cast<WarpSmem<T>*>(cur)[threadIdx.x >> 5];
    }
};

// Warp mat-vec: returns sum_{k<NIN} W[row][k] x[k] (W staged, padded rows; x in
// shared memory, 16-byte aligned).  Four partial accumulators, fixed order.
template <typename T, int NIN>
__device__ __forceinline__ T wmv(const T* W, const T* x, int row) {
    const T* w = W + row * pad_ld<T>(NIN);
    T a0 = T(0), a1 = T(0), a2 = T(0), a3 = T(0);
#pragma unroll
    for (int k = 0; k < NIN; k += 4) {
        const V4<T> wv = ld4c(w + k), xv = ld4c(x + k);
        a0 += wv.x * xv.x;
        a1 += wv.y * xv.y;
        a2 += wv.z * xv.z;
        a3 += wv.w * xv.w;
    }
    return (a0 + a1) + (a2 + a3);
}

// Sum each of 8 per-lane values over the warp (reduce-scatter butterfly, fixed
// order): returns, in lane l, the total of value (l >> 2).  9 shuffles instead
// of the 40 of eight separate warp reductions.
template <typename T>
__device__ __forceinline__ T reduce8(T (&a)[8], int lane) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const bool hi = lane & 16;
        const T keep = hi ? a[j + 4] : a[j], send = hi ? a[j] : a[j + 4];
        a[j] = keep + __shfl_xor_sync(FULL_MASK, send, 16);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const bool hi = lane & 8;
        const T keep = hi ? a[j + 2] : a[j], send = hi ? a[j] : a[j + 2];
        a[j] = keep + __shfl_xor_sync(FULL_MASK, send, 8);
    }
    {
        const bool hi = lane & 4;
        const T keep = hi ? a[1] : a[0], send = hi ? a[0] : a[1];
        a[0] = keep + __shfl_xor_sync(FULL_MASK, send, 4);
    }
    a[0] += __shfl_xor_sync(FULL_MASK, a[0], 2);
    a[0] += __shfl_xor_sync(FULL_MASK, a[0], 1);
    return a[0];
}

// An atom "team" of G consecutive warps of a CTA processes one atom at a time
// (grid-stride over atoms).  The atom's edges (and in-edge slots) are split
// round-robin over the team's warps (local edge k of warp w is q = w + G k);
// per-atom mat-vecs are computed redundantly by every warp of the team, so the
// only team synchronisation is the fixed-order sum of the warps' edge partials.
// G = 1 for large systems (throughput); G = 2, 4 for small ones, where the SMs
// would otherwise hold a single warp per scheduler and the per-atom dependency
// chain sets the step time.
template <int G>
struct Team {
    int lane, w, first, stride, bar, rb;
    __device__ Team() : rb(0) {
        lane = threadIdx.x & 31;
        const int warp = threadIdx.x >> 5;
        const int tpc = (blockDim.x >> 5) / G;  // teams per CTA
        w = warp % G;
        first = blockIdx.x * tpc + warp / G;
        stride = gridDim.x * tpc;
        bar = 1 + warp / G;
    }
    __device__ __forceinline__ void sync() const {
        if constexpr (G > 1)
            asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(G * 32) : "memory");
        else
            __syncwarp();
    }
    // Sum of v (per lane) and s (warp-uniform) over the team's warps in a fixed
    // order; every warp gets the totals.  Double-buffered scratch: one barrier.
    template <typename T>
    __device__ __forceinline__ T sum(T v, T& s, WarpSmem<T>& sm) {
        if constexpr (G == 1) {
            return v;
        } else {
            sm.red[rb][lane] = v;
            if (lane == 0) sm.reds[rb] = s;
            sync();
            const WarpSmem<T>* b = &sm - w;
            T a = b[0].red[rb][lane], as = b[0].reds[rb];
#pragma unroll
            for (int q = 1; q < G; ++q) {
                a += b[q].red[rb][lane];
                as += b[q].reds[rb];
            }
            s = as;
            rb ^= 1;
            return a;
        }
    }
    template <typename T>
    __device__ __forceinline__ T sum(T v, WarpSmem<T>& sm) {
        T dummy = T(0);
        return sum(v, dummy, sm);
    }
    // two per-lane values summed with one barrier
    template <typename T>
    __device__ __forceinline__ void sum2(T& v0, T& v1, WarpSmem<T>& sm) {
        if constexpr (G > 1) {
            sm.red[rb][lane] = v0;
            sm.red[rb][32 + lane] = v1;
            sync();
            const WarpSmem<T>* b = &sm - w;
            T a0 = b[0].red[rb][lane], a1 = b[0].red[rb][32 + lane];
#pragma unroll
            for (int q = 1; q < G; ++q) {
                a0 += b[q].red[rb][lane];
                a1 += b[q].red[rb][32 + lane];
            }
            v0 = a0;
            v1 = a1;
            rb ^= 1;
        }
    }
    // number of this warp's local edges among cnt
    __device__ __forceinline__ int local(int cnt) const { return (cnt - w + G - 1) / G; }
};

// Team mat-vec: sum_{k<NIN} W[row][k] x[k] with the inputs split over the
// team's warps (warp w: inputs [w NIN/G, (w+1) NIN/G)) and the partials summed
// in a fixed order — one copy of the weight traffic per team, not per warp.
template <typename T, int NIN, int G>
__device__ __forceinline__ T twmv(const T* W, const T* x, int row, Team<G>& tm,
                                  WarpSmem<T>& sm) {
    if constexpr (G == 1) {
        return wmv<T, NIN>(W, x, row);
    } else {
        constexpr int KC = NIN / G;
        static_assert(KC % 4 == 0, "bad team split");
        const T* wr = W + row * pad_ld<T>(NIN) + tm.w * KC;
        const T* xr = x + tm.w * KC;
        T a0 = T(0), a1 = T(0), a2 = T(0), a3 = T(0);
#pragma unroll
        for (int k = 0; k < KC; k += 4) {
            const V4<T> wv = ld4c(wr + k), xv = ld4c(xr + k);
            a0 += wv.x * xv.x;
            a1 += wv.y * xv.y;
            a2 += wv.z * xv.z;
            a3 += wv.w * xv.w;
        }
        return tm.sum((a0 + a1) + (a2 + a3), sm);
    }
}
// Two rows of the same matrix (e.g. both halves of a 64-row transposed layer).
template <typename T, int NIN, int G>
__device__ __forceinline__ void twmv2(const T* W, const T* x, int row0, int row1, T& y0, T& y1,
                                      Team<G>& tm, WarpSmem<T>& sm) {
    if constexpr (G == 1) {
        y0 = wmv<T, NIN>(W, x, row0);
        y1 = wmv<T, NIN>(W, x, row1);
    } else {
        constexpr int KC = NIN / G;
        const T* w0 = W + row0 * pad_ld<T>(NIN) + tm.w * KC;
        const T* w1 = W + row1 * pad_ld<T>(NIN) + tm.w * KC;
        const T* xr = x + tm.w * KC;
        T a0 = T(0), a1 = T(0), b0 = T(0), b1 = T(0);
#pragma unroll
        for (int k = 0; k < KC; k += 4) {
            const V4<T> xv = ld4c(xr + k), u = ld4c(w0 + k), v = ld4c(w1 + k);
            a0 += u.x * xv.x;
            a1 += u.y * xv.y;
            a0 += u.z * xv.z;
            a1 += u.w * xv.w;
            b0 += v.x * xv.x;
            b1 += v.y * xv.y;
            b0 += v.z * xv.z;
            b1 += v.w * xv.w;
        }
        y0 = a0 + a1;
        y1 = b0 + b1;
        tm.sum2(y0, y1, sm);
    }
}

// Rows `row` of two matrices over the same input vector: ya = A[row] . x[0..NA),
// yb = B[row] . x[0..NB) (NB <= NA: B reads a prefix of x), one team barrier.
template <typename T, int NA, int NB, int G>
__device__ __forceinline__ void twmv_pair(const T* A, const T* B, const T* x, int row, T& ya, T& yb,
                                          Team<G>& tm, WarpSmem<T>& sm) {
    if constexpr (G == 1) {
        ya = wmv<T, NA>(A, x, row);
        yb = wmv<T, NB>(B, x, row);
    } else {
        constexpr int KA = NA / G, KB = NB / G;
        static_assert(KA % 4 == 0 && KB % 4 == 0, "bad team split");
        const T* wa = A + row * pad_ld<T>(NA) + tm.w * KA;
        const T* wb = B + row * pad_ld<T>(NB) + tm.w * KB;
        const T* xa = x + tm.w * KA;
        const T* xb = x + tm.w * KB;
        T a0 = T(0), a1 = T(0), b0 = T(0), b1 = T(0);
#pragma unroll
        for (int k = 0; k < KA; k += 4) {
            const V4<T> w = ld4c(wa + k), v = ld4c(xa + k);
            a0 += w.x * v.x;
            a1 += w.y * v.y;
            a0 += w.z * v.z;
            a1 += w.w * v.w;
        }
#pragma unroll
        for (int k = 0; k < KB; k += 4) {
            const V4<T> w = ld4c(wb + k), v = ld4c(xb + k);
            b0 += w.x * v.x;
            b1 += w.y * v.y;
            b0 += w.z * v.z;
            b1 += w.w * v.w;
        }
        ya = a0 + a1;
        yb = b0 + b1;
        tm.sum2(ya, yb, sm);
    }
}

// Sum of the pushed adjoint rows in i's mirror slots (+ remote partials in
// domain decomposition), lane = channel, fixed order.
template <typename T, int G>
__device__ __forceinline__ T gather_in(const T* D, const DevWork<T>& ws, const DevGraph& gr, int i,
                                       Team<G>& tm, WarpSmem<T>& sm) {
    const int ic = tm.local(gr.in_cnt[i]);
    const T* drow = D + static_cast<long long>(gr.in_start[i] + tm.w) * kH + tm.lane;
    T acc = T(0);
    constexpr int B = 2 * kU<T>;  // rows in flight
    for (int k0 = 0; k0 < ic; k0 += B) {
        T r[B];
#pragma unroll
        for (int u = 0; u < B; ++u)
            if (k0 + u < ic) r[u] = drow[(k0 + u) * G * kH];
#pragma unroll
        for (int u = 0; u < B; ++u)
            if (k0 + u < ic) acc += r[u];
    }
    acc = tm.sum(acc, sm);
    // domain decomposition: partial sums pushed to ghost copies of i on other ranks
    if (ws.s_remote) acc += ws.s_remote[static_cast<long long>(i) * kH + tm.lane];
    return acc;
}

// ---------------------------------------------------------------------------
// Edge radial features + descriptor + embedding; pushes P^0 (message layer 0's
// neighbour projection) or, for depth 1 (FUSE_FIT), runs the whole fitting and
// backward chain.  rev (periodic path): computes the reverse slot of every
// edge, which is the in-edge array of the symmetric graph (in_edge == rev).
// ---------------------------------------------------------------------------
// DESC_ONLY: the edge work and the descriptor only; the embedding MLP and the P^0
// projection then run as one tcgen05 layer chain over all atoms (hmdp_tc.cu).
template <typename T, int G, bool FUSE_FIT, bool LIST = false, bool DESC_ONLY = false, bool WIDE = false>
__global__ __launch_bounds__(kCtaWarps<T, G, WIDE> * 32, kNetMinCTAs<G>) void k_embed(DevModel<T> md, DevGraph gr,
                                                             DevWork<T> ws, int* __restrict__ rev,
                                                             MdFuse mf) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    pdl_launch_dependents();
    Smem<T> sg(reinterpret_cast<T*>(smem_raw));
    __shared__ unsigned long long s_mbar;
    const T* eW1 = sg.template view<32, 32>();
    // [eW2 ; Q]: the embedding output layer and, folded through it, the next
    // consumer of h^0: Q = W1h^0 eW2 (P^0) or Q = fW1 eW2 (the fitting net, FUSE_FIT)
    const T* eX2 = sg.template view<64, 32>();
    const T *fQT = nullptr, *eW1T = nullptr;
    if constexpr (FUSE_FIT) {
        fQT = sg.template view<32, 32>();  // (fW1 eW2)^T: dE/dz1 from the fitting adjoint
        eW1T = sg.template view<32, 32>();
    }
    if constexpr (!DESC_ONLY) sg.load(md.img_embed, &s_mbar);
    WarpSmem<T>& sm = sg.warp_scratch();
    Team<G> tm;
    const int lane = tm.lane;
    const bool lead = tm.w == 0;
    const T eb1 = md.embed.b1[lane], eb2 = md.embed.b2[lane];
    const T qb = md.eqb[lane];  // W1h^0 eb2 (P^0) or fW1 eb2 + fb1 (the fitting pre-activation)
    const T fw2 = FUSE_FIT ? md.fit.W2[lane] : T(0);
    const T fb2 = FUSE_FIT ? md.fit.b2[0] : T(0);
    const int nd = md.n_types * kK;
    __syncthreads();  // publishes the mbarrier init; the copy is awaited at first use
    bool staged = false;
    pdl_wait();
    // this step's neighbour search is complete: clear the cell counts for the
    // binning fused into the force kernel (device MD) / keep the zero invariant
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < mf.n_cells_zero;
         c += gridDim.x * blockDim.x)
        mf.cell_count[c] = 0;
    auto sb = sm.ed;
    // LIST (global-index DD): the atoms alist[0 .. *alist_n); else [0, n_active)
    const int n_run = LIST ? *gr.alist_n : gr.n_active;
    for (int k_at = tm.first; k_at < n_run; k_at += tm.stride) {
        const int i = LIST ? gr.alist[k_at] : k_at;
        const int start = gr.row_start[i] + tm.w, cnt = gr.nnei[i];
        const int mloc = tm.local(cnt);
        T desc = T(0);  // lane q < nd accumulates descriptor component q
        for (int base = 0; base < mloc; base += 32) {
            const int m = min(32, mloc - base);
            const int e = start + G * (base + lane);
            int j = 0;
            if (lane < m) {
                if (rev) j = gr.nbr[e];
                T x, y, z;
                const T r = edge_len<T>(gr.dr + 3ll * e, x, y, z);
                if (!(r > T(0))) atomicOr(ws.err, kErrZeroEdge);
                const T s = sw_val(r, md.rc), ds = sw_der(r, md.rc);
                T b[kK], db[kK];
#pragma unroll
                for (int k = 0; k < kK; ++k) {
                    const T d = r - md.mu[k];
                    const T gk = d_exp(-d * d * md.inv2w2);
                    b[k] = gk * s;
                    db[k] = -d * md.invw2 * gk * s + gk * ds;  // BasisT::derivatives
                }
                ws.es[e] = s;
                ws.eds[e] = ds;
                st4(ws.eb + 8ll * e, b[0], b[1], b[2], b[3]);
                st4(ws.eb + 8ll * e + 4, b[4], b[5], b[6], b[7]);
                st4(ws.edb + 8ll * e, db[0], db[1], db[2], db[3]);
                st4(ws.edb + 8ll * e + 4, db[4], db[5], db[6], db[7]);
                st4(&sb[lane][4], b[0], b[1], b[2], b[3]);
                st4(&sb[lane][8], b[4], b[5], b[6], b[7]);
                sm.ety[lane] = gr.ety[e];
            }
            if (rev) {
                // rev(e) = slot of i in nbr(j) (symmetric, sorted list).  Each pair is
                // searched once, by its lower atom: the edges with j > i (a suffix of
                // the warp's lanes, the list being sorted) find i in j's list and set
                // both rev(e) and rev(rev(e)) = e; the others are set by their j.  Lane
                // l reads entry l of each neighbour's list (one memory latency per 8
                // edges); a ballot finds i.  rev is read only by later kernels.
                // (pull-form DD, ws.dd_role set: an owned atom also searches for its
                // halo neighbours, which run no embedding here)
                bool up;
                int lo_lane;
                if constexpr (LIST) {
                    up = lane < m && (j > i || (ws.dd_role && ws.dd_role[j] != 1));
                    const unsigned upb = __ballot_sync(FULL_MASK, up);
                    lo_lane = upb ? __ffs(upb) - 1 : m;
                } else {
                    up = lane < m && j > i;
                    lo_lane = __popc(__ballot_sync(FULL_MASK, lane < m && !up));
                }
                const int rs_l = up ? gr.row_start[j] : 0;
                const int nn_l = up ? gr.nnei[j] : 0;
                int found = -1;
                for (int q0 = lo_lane; q0 < m; q0 += 8) {
                    int val[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int rsq = __shfl_sync(FULL_MASK, rs_l, (q0 + u) & 31);
                        const int nnq = __shfl_sync(FULL_MASK, nn_l, (q0 + u) & 31);
                        val[u] = (q0 + u < m && lane < nnq) ? gr.nbr[rsq + lane] : -1;
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const unsigned bal = __ballot_sync(FULL_MASK, val[u] == i);
                        if (lane == q0 + u && bal) found = rs_l + __ffs(bal) - 1;
                    }
                }
                if (up) {
                    if (found < 0 && nn_l > 32) {
                        int lo = rs_l, hi = rs_l + nn_l - 1;
                        while (lo <= hi) {
                            const int mid = (lo + hi) >> 1;
                            const int vv = gr.nbr[mid];
                            if (vv == i) {
                                found = mid;
                                break;
                            }
                            if (vv < i) lo = mid + 1;
                            else hi = mid - 1;
                        }
                    }
                    rev[e] = found;
                    if (found < 0) atomicOr(ws.err, kErrAsymmetric);
                    else rev[found] = e;
                }
            }
            __syncwarp();
            if (lane < nd) {  // descriptor: edge order within the warp, as inference.cpp:228-238
                const int ty = lane >> 3, k = lane & 7;
                for (int r = 0; r < m; ++r) desc += (sm.ety[r] == ty) ? sb[r][4 + k] : T(0);
            }
            __syncwarp();
        }
        desc = tm.sum(desc, sm);
        if constexpr (DESC_ONLY) {  // the tcgen05 chain takes it from here
            if (lead) ws.desc[static_cast<long long>(i) * 32 + lane] = lane < nd ? desc : T(0);
            __syncwarp();
            continue;
        }
        if (!staged) {  // weights (bulk copy issued at kernel entry) needed from here on
            Smem<T>::wait(&s_mbar);
            staged = true;
        }
        sm.x[lane] = lane < nd ? desc : T(0);
        if (lead && lane < nd) ws.desc[static_cast<long long>(i) * 32 + lane] = desc;
        __syncwarp();
        // embedding forward nd (zero-padded to 32) -> 32 (tanh) -> 32
        const T z1 = d_tanh(twmv<T, 32>(eW1, sm.x, lane, tm, sm) + eb1);
        if (lead) ws.ez1[static_cast<long long>(i) * kH + lane] = z1;
        sm.y[lane] = z1;
        __syncwarp();
        T h0, qz;  // h^0 - eb2 and Q z1
        twmv2<T, 32>(eX2, sm.y, lane, lane + 32, h0, qz, tm, sm);
        h0 += eb2;
        if (lead) ws.h[static_cast<long long>(i) * kH + lane] = h0;
        if constexpr (FUSE_FIT) {
            // fitting forward on h^0 (pre-activation fW1 h^0 + fb1 = Q z1 + qb) and its
            // adjoint straight to z1: dE/dz1 = (fW1 eW2)^T (fw2 (1 - zf^2))
            const bool owned = !(gr.is_ghost && gr.is_ghost[i]);
            const T zf = d_tanh(qz + qb);
            const T en = warp_sum(fw2 * zf) + fb2;
            if (lead && lane == 0) ws.e_atom[i] = owned ? static_cast<double>(en) : 0.0;
            sm.t[lane] = owned ? fw2 * (T(1) - zf * zf) : T(0);
            __syncwarp();
            // embedding backward: tanh layer 1 (W1^T, padded)
            const T dz1 = twmv<T, 32>(fQT, sm.t, lane, tm, sm) * (T(1) - z1 * z1);
            __syncwarp();
            sm.t[lane] = dz1;
            __syncwarp();
            const T dd = twmv<T, 32>(eW1T, sm.t, lane, tm, sm);
            sm.x[lane] = dd;
            __syncwarp();
            for (int q = lane; q < mloc; q += 32) {
                const long long e = start + G * q;
                const V4<T> d0 = ld4c(ws.edb + 8 * e), d1 = ld4c(ws.edb + 8 * e + 4);
                const T* dv = sm.x + gr.ety[e] * kK;
                T acc = dv[0] * d0.x;
                acc += dv[1] * d0.y;
                acc += dv[2] * d0.z;
                acc += dv[3] * d0.w;
                acc += dv[4] * d1.x;
                acc += dv[5] * d1.y;
                acc += dv[6] * d1.z;
                acc += dv[7] * d1.w;
                ws.g[e] = acc;
                // mirror for the force gather; on the periodic path the mirror slots are
                // still being written by the pairs' lower atoms, so the force kernel
                // gathers g[rev(q)] itself (DevWork::gather_mirror_g)
                if (!rev) ws.grev[gr.inv_pos[e]] = acc;
            }
        } else {
            // P^0 = W1h^(0) h^0 = Q z1 + W1h^(0) eb2, one row per atom (L2-resident;
            // gathered by the sources of i's in-edges in the message layer)
            const T p = qz + qb;
            if (lead) {
                ws.pa[static_cast<long long>(i) * kH + lane] = p;
                if (ws.p_atom) ws.p_atom[static_cast<long long>(i) * kH + lane] = p;
            }
        }
        __syncwarp();
    }
    if constexpr (!DESC_ONLY)
        if (!staged) Smem<T>::wait(&s_mbar);  // no CTA exits with its weight copy in flight
}

// ---------------------------------------------------------------------------
// Atom prologue.  On the periodic (ELL) graph atom i's slots are
// [i*ell, i*ell + ell), so a warp can issue its first batch of edge loads before
// the neighbour count arrives — every per-atom kernel then waits for ONE memory
// round trip before computing, instead of count -> rows -> ... chains.  Loads past
// the count read valid (ELL padding) memory and are never used.
// ---------------------------------------------------------------------------
template <int G>
struct AtomRow {
    long long e0;  // this warp's first slot: local edge k is e0 + G k
    int room;      // local slots addressable before the count is known
    int cnt;       // neighbour count (valid after finish())
    const int* nnei;
    int i;
    __device__ __forceinline__ AtomRow(const DevGraph& gr, int i_, const Team<G>& tm)
        : nnei(gr.nnei), i(i_) {
        if (gr.ell) {
            e0 = static_cast<long long>(i) * gr.ell + tm.w;
            room = tm.local(gr.ell);
            cnt = -1;
        } else {
            e0 = gr.row_start[i] + tm.w;
            cnt = gr.nnei[i];
            room = tm.local(cnt);
        }
    }
    __device__ __forceinline__ int finish(const Team<G>& tm) {
        if (cnt < 0) cnt = nnei[i];
        return tm.local(cnt);  // this warp's local edges
    }
};

// First batch of a warp's backward edge loop, loaded early (lane = local edge
// for the scalars, lane = channel for the rows).  Stored mode: the rows are z_e,
// written by the layer's forward.  RECOMP mode: nothing per edge is stored by the
// forward; the rows are the gathered P^l_j and z_e = tanh(W1b b_e + b1 + P^l_j) is
// recomputed in the edge loop (kRecomputeZ, defined with the team constants).
template <typename T>
struct BwdPre {
    T zr[8];  // z rows (stored mode) or P^l_j rows (RECOMP)
    T s, ds;
    V4<T> d0, d1;
    V4<T> b0, b1;  // RECOMP: basis b_e
    int mir, nb;
};
template <typename T, int G, bool RECOMP>
__device__ __forceinline__ void bwd_prefetch(BwdPre<T>& p, const T* Z, const DevWork<T>& ws,
                                             const DevGraph& gr, long long e0, int room,
                                             int lane) {
    if constexpr (!RECOMP) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (u < room) p.zr[u] = Z[(e0 + static_cast<long long>(G) * u) * kH + lane];
    }
    if (lane < room) {
        const long long e = e0 + static_cast<long long>(G) * lane;
        p.s = ws.es[e];
        p.ds = ws.eds[e];
        p.d0 = ld4c(ws.edb + 8 * e);
        p.d1 = ld4c(ws.edb + 8 * e + 4);
        p.mir = gr.inv_pos[e];
        if constexpr (RECOMP) {
            p.b0 = ld4c(ws.eb + 8 * e);
            p.b1 = ld4c(ws.eb + 8 * e + 4);
            p.nb = min(max(gr.nbr[e], 0), gr.n - 1);  // ELL padding: any valid row
        }
    }
    if constexpr (RECOMP) {  // Z = P^l rows [n][32]
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = __shfl_sync(FULL_MASK, p.nb, u);
            if (u < room) p.zr[u] = Z[static_cast<long long>(j) * kH + lane];
        }
    }
}

// Sum of the pushed adjoint rows in i's mirror slots (fixed order), symmetric
// ELL graph: the in-slots are the atom's own out-slots, so the first batch is
// loaded speculatively (see AtomRow).  General graphs use gather_in.
template <typename T, int G>
struct GatherPre {
    static constexpr int B = 2 * kU<T>;
    T r[B];
    __device__ __forceinline__ void load(const T* D, long long e0, int room, int lane) {
#pragma unroll
        for (int u = 0; u < B; ++u)
            if (u < room) r[u] = D[(e0 + static_cast<long long>(G) * u) * kH + lane];
    }
    __device__ __forceinline__ T sum(const T* D, long long e0, int ic, int lane) const {
        T acc = T(0);
#pragma unroll
        for (int u = 0; u < B; ++u)
            if (u < ic) acc += r[u];
        for (int k0 = B; k0 < ic; k0 += B) {
            T q[B];
#pragma unroll
            for (int u = 0; u < B; ++u)
                if (k0 + u < ic) q[u] = D[(e0 + static_cast<long long>(G) * (k0 + u)) * kH + lane];
#pragma unroll
            for (int u = 0; u < B; ++u)
                if (k0 + u < ic) acc += q[u];
        }
        return acc;
    }
};

// ---------------------------------------------------------------------------
// Message-layer backward for atom i, given dE/dh^{l+1}_i (dh, lane = channel)
// and the update hidden activation zu.  Pushes dz_e to e's mirror slot and
// accumulates dE/dr_e into g (this warp's share of the edges).  `pre` holds the
// first batch of the edge loop, loaded before the atom's mat-vecs.
// ---------------------------------------------------------------------------
template <typename T, int G, bool RECOMP>
__device__ __forceinline__ void msg_backward_warp(const T* uW2T, const T* uW1T, T mb1, T c1,
                                                  T w_in, const T (&w1b)[kK], const DevGraph& gr,
                                                  const DevWork<T>& ws, WarpSmem<T>& sm, int l,
                                                  int i, T dh, T zu, bool first_g,
                                                  Team<G>& tm, BwdPre<T>& pre, long long e0,
                                                  int mloc) {
    const int lane = tm.lane;
    const long long S = ws.slots;
    // update MLP backward (64 -> 32 tanh -> 32); uW2T null: w_in = uW2^T dh given
    T dz;
    if (uW2T) {
        sm.t[lane] = dh;
        __syncwarp();
        dz = twmv<T, 32>(uW2T, sm.t, lane, tm, sm) * (T(1) - zu * zu);
    } else {
        dz = w_in * (T(1) - zu * zu);
    }
    sm.y[lane] = dz;
    __syncwarp();
    // rows 0..31: dE/dh (update input); rows 32..63 (folded): v = W2^T U1m^T dz
    T din_h, v;
    twmv2<T, 32>(uW1T, sm.y, lane, lane + 32, din_h, v, tm, sm);
    if (tm.w == 0)
        ws.dhown[static_cast<long long>(i) * kH + lane] = dh + din_h;  // residual + update
    const T c0 = warp_sum(dz * c1);  // dmsum . b2
    // stored z rows (LAST layer) or this layer's P rows (RECOMP)
    const T* Z = RECOMP ? ws.pa + static_cast<long long>(l) * gr.n * kH
                        : ws.z + (kRecomputeZ ? 0 : static_cast<long long>(l) * S * kH);
    T* D = ws.d + (l & 1) * S * kH;
    for (int base = 0; base < mloc; base += 32) {
        const int m = min(32, mloc - base);
        const long long eb = e0 + static_cast<long long>(G) * base;  // local edge k: eb + G k
        const T* zrow = Z + eb * kH + lane;
        if (base > 0) bwd_prefetch<T, G, RECOMP>(pre, Z, ws, gr, eb, m, lane);
        // lane u stages edge u's scalars; the edge loop reads them as broadcasts
        if (lane < m) {
            T* row = sm.ed[lane];
            row[0] = pre.s;
            row[1] = pre.ds;
            st4(row + 4, pre.d0.x, pre.d0.y, pre.d0.z, pre.d0.w);
            st4(row + 8, pre.d1.x, pre.d1.y, pre.d1.z, pre.d1.w);
            if constexpr (RECOMP) {
                st4(row + 12, pre.b0.x, pre.b0.y, pre.b0.z, pre.b0.w);
                st4(row + 16, pre.b1.x, pre.b1.y, pre.b1.z, pre.b1.w);
                sm.enb[lane] = pre.nb;
            }
            sm.emir[lane] = pre.mir;
        }
        __syncwarp();
        T* zr = pre.zr;
        for (int u0 = 0; u0 < m; u0 += 8) {
            const int mu = min(8, m - u0);
            T zn[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (u0 + 8 + u < m)
                    zn[u] = RECOMP ? Z[static_cast<long long>(sm.enb[u0 + 8 + u]) * kH + lane]
                                   : zrow[(u0 + 8 + u) * G * kH];
            T term[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                term[u] = T(0);
                if (u < mu) {
                    const T* row = sm.ed[u0 + u];
                    const T s = row[0], ds = row[1];
                    const V4<T> d0 = ld4c(row + 4), d1 = ld4c(row + 8);
                    T wv = w1b[0] * d0.x;
                    wv += w1b[1] * d0.y;
                    wv += w1b[2] * d0.z;
                    wv += w1b[3] * d0.w;
                    wv += w1b[4] * d1.x;
                    wv += w1b[5] * d1.y;
                    wv += w1b[6] * d1.z;
                    wv += w1b[7] * d1.w;
                    T z;
                    if constexpr (RECOMP) {  // z_e = tanh(W1b b_e + b1 + P^l_j), as the forward
                        const V4<T> b0 = ld4c(row + 12), bb = ld4c(row + 16);
                        T a = mb1;
                        a += w1b[0] * b0.x;
                        a += w1b[1] * b0.y;
                        a += w1b[2] * b0.z;
                        a += w1b[3] * b0.w;
                        a += w1b[4] * bb.x;
                        a += w1b[5] * bb.y;
                        a += w1b[6] * bb.z;
                        a += w1b[7] * bb.w;
                        z = d_tanh(a + zr[u]);
                    } else {
                        z = zr[u];
                    }
                    const T d = s * v * (T(1) - z * z);
                    D[static_cast<long long>(sm.emir[u0 + u]) * kH + lane] = d;
                    term[u] = ds * v * z + d * wv;
                }
            }
            // reduce-scatter butterfly: 8 edge sums in 9 shuffles; lane 4u holds edge u
            const T tot = reduce8(term, lane);
            if ((lane & 3) == 0 && (lane >> 2) < mu) {
                const int u = u0 + (lane >> 2);
                const long long e = eb + static_cast<long long>(G) * u;
                ws.g[e] = (first_g ? T(0) : ws.g[e]) + (tot + sm.ed[u][1] * c0);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) zr[u] = zn[u];
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// Pull form of the message backward (symmetric periodic graph, every atom runs
// the network).  The push form above has each RECEIVER i push dz_e = s_e v_i
// (1 - z_e^2) into a per-edge row that the sender k later gathers: two 128-byte
// rows per edge and layer that spill out of L2 at 2PTC.  Every quantity of
// message e = (i <- k) depends only on (v_i, c0_i) of the receiver and on z_e,
// so the SENDER can compute all of it over its own slots: it gathers the
// receiver's per-atom row v_i (an [n][32] array that stays in L2, like the P
// rows of the forward), sums dz_e in registers, and adds the message's dE/dr to
// g at its own slot (the force kernel sums g_q + g_rev(q), so either end of a
// pair may hold a term).  z_e is either stored by the forward at the sender's
// mirror slot (PULL = 1) or recomputed by the sender from its OWN P row,
// z_e = tanh(W1b b_e + b1 + P_k), no gather (PULL = 2).  Same function as the
// push form; only the summation points of the per-pair terms move.
// ---------------------------------------------------------------------------
// Update-MLP backward of layer l for atom i (dE/dh^{l+1}_i = dh, update hidden
// activation zu): writes dhown (residual + update input), v^l_i = W2^T dmsum and
// c0^l_i = dmsum . b2 for the senders of i's messages.
template <typename T, int G>
__device__ __forceinline__ void upd_bwd_pull(const T* uW2T, const T* uW1T, T c1, T w_in,
                                             const DevWork<T>& ws, WarpSmem<T>& sm, int n, int l,
                                             int i, T dh, T zu, Team<G>& tm) {
    const int lane = tm.lane;
    T dz;  // uW2T null: w_in = uW2^T dh given
    if (uW2T) {
        sm.t[lane] = dh;
        __syncwarp();
        dz = twmv<T, 32>(uW2T, sm.t, lane, tm, sm) * (T(1) - zu * zu);
    } else {
        dz = w_in * (T(1) - zu * zu);
    }
    sm.y[lane] = dz;
    __syncwarp();
    // rows 0..31: dE/dh (update input); rows 32..63 (folded): v = W2^T U1m^T dz
    T din_h, v;
    twmv2<T, 32>(uW1T, sm.y, lane, lane + 32, din_h, v, tm, sm);
    const T c0 = warp_sum(dz * c1);  // dmsum . b2
    if (tm.w == 0) {
        const long long b = static_cast<long long>(l & 1) * n + i;
        ws.dhown[static_cast<long long>(i) * kH + lane] = dh + din_h;
        ws.vrow[b * kH + lane] = v;
        if (lane == 0) ws.vc0[b] = c0;
    }
    __syncwarp();
}

// Sender-side backward of one message layer over this warp's local slots of atom
// k (local edge q: slot e0 + G q, neighbour = the message's receiver i).  Returns
// the warp's sum of dz_e (lane = channel); adds each message's dE/dr to g at the
// slot (first_g: the first backward kernel to touch g overwrites it).
//   z_e  = stored row (PULL 1) | tanh(W1b b_e + b1 + P_k) (PULL 2, pk = P_k[lane])
//   dz_e = s_e v_i (1 - z_e^2);  dE/dr_e += s'_e (v_i . z_e + c0_i) + b'_e . (W1b^T dz_e)
// DD (halo-exchange domain decomposition, PULL = 1): the sender k is any searched
// row (owned or halo) and only messages into OWNED receivers are this rank's; the
// others contribute nothing (mask row[3]; their v / z rows are stale and never used).
// A halo sender's edge scalars were computed by the owned receiver's embedding at
// the mirror slot (same |r|, bit-identical), so they are read there.
template <typename T, int G, int PULL, bool DD = false>
__device__ __forceinline__ T pull_edges(const T (&w1b)[kK], T mb1, T pk, const T* Z, const T* V,
                                        const T* C0, const DevGraph& gr, const DevWork<T>& ws,
                                        WarpSmem<T>& sm, long long e0, int mloc, bool first_g,
                                        int lane, bool own_sender = true) {
    static_assert(!DD || PULL == 1, "DD pull form: stored z only");
    T sdz = T(0);
    for (int base = 0; base < mloc; base += 32) {
        const int m = min(32, mloc - base);
        const long long eb = e0 + static_cast<long long>(G) * base;  // local edge k: eb + G k
        // lane u stages edge u's scalars (read as broadcasts by the edge loop)
        if (lane < m) {
            const long long e = eb + static_cast<long long>(G) * lane;
            const int nb = gr.nbr[e];
            T* row = sm.ed[lane];
            if constexpr (DD) {
                const bool rcv = ws.dd_role[nb] == 1;
                const long long es = own_sender ? e : static_cast<long long>(gr.inv_pos[e]);
                const V4<T> d0 = rcv ? ld4c(ws.edb + 8 * es) : V4<T>{},
                            d1 = rcv ? ld4c(ws.edb + 8 * es + 4) : V4<T>{};
                row[0] = rcv ? ws.es[es] : T(0);
                row[1] = rcv ? ws.eds[es] : T(0);
                row[2] = rcv ? C0[nb] : T(0);
                row[3] = rcv ? T(1) : T(0);
                st4(row + 4, d0.x, d0.y, d0.z, d0.w);
                st4(row + 8, d1.x, d1.y, d1.z, d1.w);
            } else {
                row[0] = ws.es[e];
                row[1] = ws.eds[e];
                const V4<T> d0 = ld4c(ws.edb + 8 * e), d1 = ld4c(ws.edb + 8 * e + 4);
                st4(row + 4, d0.x, d0.y, d0.z, d0.w);
                st4(row + 8, d1.x, d1.y, d1.z, d1.w);
                if constexpr (PULL == 2) {
                    const V4<T> b0 = ld4c(ws.eb + 8 * e), b1 = ld4c(ws.eb + 8 * e + 4);
                    st4(row + 12, b0.x, b0.y, b0.z, b0.w);
                    st4(row + 16, b1.x, b1.y, b1.z, b1.w);
                }
                row[2] = C0[nb];
            }
            sm.enb[lane] = nb;
        }
        __syncwarp();
        constexpr int U = kU<T>;
        T vr[U], zr[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (u < m) {
                vr[u] = V[static_cast<long long>(sm.enb[u]) * kH + lane];
                if constexpr (PULL == 1) zr[u] = Z[(eb + static_cast<long long>(G) * u) * kH + lane];
            }
        for (int u0 = 0; u0 < m; u0 += U) {
            const int mu = min(U, m - u0);
            T vn[U], zn[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (u0 + U + u < m) {
                    vn[u] = V[static_cast<long long>(sm.enb[u0 + U + u]) * kH + lane];
                    if constexpr (PULL == 1)
                        zn[u] = Z[(eb + static_cast<long long>(G) * (u0 + U + u)) * kH + lane];
                }
            T term[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                term[u] = T(0);
                if (u < U && u < mu) {
                    const T* row = sm.ed[u0 + u];
                    const T s = row[0], ds = row[1];
                    const V4<T> d0 = ld4c(row + 4), d1 = ld4c(row + 8);
                    T wv = w1b[0] * d0.x;
                    wv += w1b[1] * d0.y;
                    wv += w1b[2] * d0.z;
                    wv += w1b[3] * d0.w;
                    wv += w1b[4] * d1.x;
                    wv += w1b[5] * d1.y;
                    wv += w1b[6] * d1.z;
                    wv += w1b[7] * d1.w;
                    T z;
                    if constexpr (PULL == 2) {  // bit-identical to the forward's z_e
                        const V4<T> b0 = ld4c(row + 12), bb = ld4c(row + 16);
                        T a = mb1;
                        a += w1b[0] * b0.x;
                        a += w1b[1] * b0.y;
                        a += w1b[2] * b0.z;
                        a += w1b[3] * b0.w;
                        a += w1b[4] * bb.x;
                        a += w1b[5] * bb.y;
                        a += w1b[6] * bb.z;
                        a += w1b[7] * bb.w;
                        z = d_tanh(a + pk);
                    } else {
                        z = zr[u];
                    }
                    T v = vr[u];
                    if constexpr (DD)
                        if (row[3] == T(0)) v = z = T(0);  // not this rank's message
                    const T d = s * v * (T(1) - z * z);
                    sdz += d;
                    term[u] = ds * v * z + d * wv;
                }
            }
            // reduce-scatter butterfly: 8 edge sums in 9 shuffles; lane 4u holds edge u
            const T tot = reduce8(term, lane);
            if ((lane & 3) == 0 && (lane >> 2) < mu) {
                const int u = u0 + (lane >> 2);
                const long long e = eb + static_cast<long long>(G) * u;
                const T* row = sm.ed[u];
                ws.g[e] = (first_g ? T(0) : ws.g[e]) + (tot + row[1] * row[2]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                vr[u] = vn[u];
                if constexpr (PULL == 1) zr[u] = zn[u];
            }
        }
        __syncwarp();
    }
    return sdz;
}

// ---------------------------------------------------------------------------
// Message layer l forward; LAST fuses the fitting net and the top layer's
// backward (all atom-local).
// ---------------------------------------------------------------------------
template <typename T, int G, bool LAST, bool LIST = false, int PULL = 0, bool WIDE = false>
__global__ __launch_bounds__((PULL == 0 ? kPushWarps : kCtaWarps<T, G, WIDE>) * 32, kNetMinCTAs<G>) void k_msg_fwd(DevModel<T> md, DevGraph gr,
                                                               DevWork<T> ws, int l) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TP_START;
    pdl_launch_dependents();
    const DevMlp<T>& msg = md.msg[l];
    const DevMlp<T>& upd = md.upd[l];
    Smem<T> sg(reinterpret_cast<T*>(smem_raw));
    __shared__ unsigned long long s_mbar;
    const T* uW1 = sg.template view<32, 64>();  // [U1h | U1m W2] (folded)
    const T *uW2 = nullptr, *nW1h = nullptr, *fW1 = nullptr, *uX3 = nullptr, *fY3 = nullptr,
            *uW1T = nullptr;
    if constexpr (LAST) {
        // the fitting net folded through the top update's output layer:
        // fW1 h^M = fW1 h + (fW1 U2) zu + fW1 b2u, and its adjoint back to zu
        fW1 = sg.template view<32, 32>();
        uX3 = sg.template view<64, 32>();  // [U2 ; fW1 U2]
        fY3 = sg.template view<64, 32>();  // [fW1^T ; (fW1 U2)^T]
        uW1T = sg.template view<64, 32>();  // [U1h^T ; (U1m W2)^T]
    } else {
        uW2 = sg.template view<32, 32>();
        nW1h = sg.template view<32, 32>();
    }
    sg.load(md.img_fwd[l], &s_mbar);
    WarpSmem<T>& sm = sg.warp_scratch();
    Team<G> tm;
    const int lane = tm.lane;
    const bool lead = tm.w == 0;
    T w1b[kK];
#pragma unroll
    for (int k = 0; k < kK; ++k) w1b[k] = msg.W1T[(kH + k) * kH + lane];
    const T mb1 = msg.b1[lane], ub1 = upd.b1[lane], ub2 = upd.b2[lane];
    const T c1 = md.uc1[l][lane];  // U1m b2 (folded message output bias)
    const T fcl = LAST ? md.fcl[lane] : T(0);  // fW1 b2u + fb1
    const T fw2 = LAST ? md.fit.W2[lane] : T(0);
    const T fb2 = LAST ? md.fit.b2[0] : T(0);
    __syncthreads();  // publishes the mbarrier init; the copy is awaited at first use
    bool staged = false;
    TP(0);
    pdl_wait();
    TP(1);
    const int n = gr.n;
    // P^l_j rows: one per atom, gathered by neighbour index (the [n][32] array stays
    // in L2 at every paper size; per-edge pushed copies would not)
    const T* Pl = ws.pa + static_cast<long long>(l) * n * kH;
    // z_e rows of this layer (read back by the layer's backward); with kRecomputeZ only
    // the LAST layer's are stored (the lower layers' backward recomputes them)
    T* Z = ws.z + (kRecomputeZ && PULL == 0 ? 0 : static_cast<long long>(l) * ws.slots * kH);
    // LIST (global-index DD): the atoms alist[0 .. *alist_n); else [0, n_active)
    const int n_run = LIST ? *gr.alist_n : gr.n_active;
    for (int k_at = tm.first; k_at < n_run; k_at += tm.stride) {
        const int i = LIST ? gr.alist[k_at] : k_at;
        AtomRow<G> ar(gr, i, tm);
        const T hi = ws.h[(static_cast<long long>(l) * n + i) * kH + lane];
        // first batch: edge scalars and neighbour indices (lane = local edge; on the
        // ELL graph issued before the count arrives), then the P rows they select
        T es_l = T(0);
        V4<T> b0_l{}, bb_l{};
        int nb_l = 0, mir_l = 0;
        if (lane < ar.room) {
            const long long e = ar.e0 + static_cast<long long>(G) * lane;
            es_l = ws.es[e];
            b0_l = ld4c(ws.eb + 8 * e);
            bb_l = ld4c(ws.eb + 8 * e + 4);
            nb_l = min(max(gr.nbr[e], 0), n - 1);  // padding slots: any valid row
            if constexpr (PULL == 1) mir_l = gr.inv_pos[e];
        }
        T pr[kU<T>];
#pragma unroll
        for (int u = 0; u < kU<T>; ++u) {
            const int j = __shfl_sync(FULL_MASK, nb_l, u);
            if (u < ar.room) pr[u] = Pl[static_cast<long long>(j) * kH + lane];
        }
        const int mloc = ar.finish(tm);
        sm.x[lane] = hi;
        TP(2);
        T acc = T(0), ssum = T(0);
        for (int base = 0; base < mloc; base += 32) {
            const int m = min(32, mloc - base);
            const long long e0 = ar.e0 + static_cast<long long>(G) * base;  // local k: e0 + G k
            if (base > 0) {
                if (lane < m) {
                    const long long e = e0 + G * lane;
                    es_l = ws.es[e];
                    b0_l = ld4c(ws.eb + 8 * e);
                    bb_l = ld4c(ws.eb + 8 * e + 4);
                    nb_l = gr.nbr[e];
                    if constexpr (PULL == 1) mir_l = gr.inv_pos[e];
                }
#pragma unroll
                for (int u = 0; u < kU<T>; ++u) {
                    const int j = __shfl_sync(FULL_MASK, nb_l, u);
                    if (u < m) pr[u] = Pl[static_cast<long long>(j) * kH + lane];
                }
            }
            if (lane < m) {
                T* row = sm.ed[lane];
                row[0] = es_l;
                st4(row + 4, b0_l.x, b0_l.y, b0_l.z, b0_l.w);
                st4(row + 8, bb_l.x, bb_l.y, bb_l.z, bb_l.w);
                sm.enb[lane] = nb_l;
                if constexpr (PULL == 1) sm.emir[lane] = mir_l;
            }
            __syncwarp();
            for (int u0 = 0; u0 < m; u0 += kU<T>) {
                T pn[kU<T>];
#pragma unroll
                for (int u = 0; u < kU<T>; ++u)
                    if (u0 + kU<T> + u < m)
                        pn[u] = Pl[static_cast<long long>(sm.enb[u0 + kU<T> + u]) * kH + lane];
#pragma unroll
                for (int u = 0; u < kU<T>; ++u) {
                    if (u0 + u >= m) break;
                    const T* row = sm.ed[u0 + u];
                    const T s = row[0];
                    const V4<T> b0 = ld4c(row + 4), bb = ld4c(row + 8);
                    T a = mb1;
                    a += w1b[0] * b0.x;
                    a += w1b[1] * b0.y;
                    a += w1b[2] * b0.z;
                    a += w1b[3] * b0.w;
                    a += w1b[4] * bb.x;
                    a += w1b[5] * bb.y;
                    a += w1b[6] * bb.z;
                    a += w1b[7] * bb.w;
                    const T z = d_tanh(a + pr[u]);
                    if constexpr (PULL == 1)  // the sender's mirror slot (its backward reads it)
                        Z[static_cast<long long>(sm.emir[u0 + u]) * kH + lane] = z;
                    else if constexpr (PULL == 0)
                        if (LAST || !kRecomputeZ)
                            Z[(e0 + static_cast<long long>(G) * (u0 + u)) * kH + lane] = z;
                    acc += s * z;
                    ssum += s;
                }
#pragma unroll
                for (int u = 0; u < kU<T>; ++u) pr[u] = pn[u];
            }
            __syncwarp();
        }
        // LAST: the backward edge loop's first batch (z rows just written by this
        // warp) is loaded now, under the atom-level mat-vecs below
        TP(3);
        BwdPre<T> pre;
        if constexpr (LAST && PULL == 0)
            bwd_prefetch<T, G, false>(pre, Z, ws, gr, ar.e0, min(mloc, 32), lane);
        acc = tm.sum(acc, ssum, sm);
        TP(4);
        if (!staged) {  // weights (bulk copy issued at kernel entry) needed from here on
            Smem<T>::wait(&s_mbar);
            staged = true;
        }
        // update MLP on [h_i, msum] (64 -> 32 tanh -> 32), residual, with W2 folded:
        // U1 [h; msum] = [U1h | U1m W2] [h; t] + ssum U1m b2,  t = sum_e s_e z_e
        sm.x[kH + lane] = acc;
        __syncwarp();
        if constexpr (!LAST) {
            const T zu = d_tanh((twmv<T, 64>(uW1, sm.x, lane, tm, sm) + ssum * c1) + ub1);
            if (lead) ws.uz1[(static_cast<long long>(l) * n + i) * kH + lane] = zu;
            sm.y[lane] = zu;
            __syncwarp();
            const T hn = hi + (twmv<T, 32>(uW2, sm.y, lane, tm, sm) + ub2);
            if (lead) ws.h[(static_cast<long long>(l + 1) * n + i) * kH + lane] = hn;
            sm.t[lane] = hn;
            __syncwarp();
            TP(5);
            // P^{l+1}_i, one row per atom
            const T p = twmv<T, 32>(nW1h, sm.t, lane, tm, sm);
            if (lead) {
                ws.pa[(static_cast<long long>(l + 1) * n + i) * kH + lane] = p;
                if (ws.p_atom) ws.p_atom[static_cast<long long>(i) * kH + lane] = p;
            }
            TP(6);
        } else {
            // update input [h; t] for U1 and, on its h half, fW1 h (one team barrier)
            T pu, fh;
            twmv_pair<T, 64, 32>(uW1, fW1, sm.x, lane, pu, fh, tm, sm);
            const T zu = d_tanh((pu + ssum * c1) + ub1);
            if (lead) ws.uz1[(static_cast<long long>(l) * n + i) * kH + lane] = zu;
            sm.y[lane] = zu;
            __syncwarp();
            T uh, up;  // U2 zu and (fW1 U2) zu
            twmv2<T, 32>(uX3, sm.y, lane, lane + 32, uh, up, tm, sm);
            const T hn = hi + (uh + ub2);
            if (lead) ws.h[(static_cast<long long>(l + 1) * n + i) * kH + lane] = hn;
            TP(5);
            // fitting (inference.cpp:288-311): pre-activation fW1 h^M + fb1
            const bool owned = !(gr.is_ghost && gr.is_ghost[i]);
            const T zf = d_tanh((fh + up) + fcl);
            const T en = warp_sum(fw2 * zf) + fb2;
            if (lead && lane == 0) ws.e_atom[i] = owned ? static_cast<double>(en) : 0.0;
            sm.t[lane] = owned ? fw2 * (T(1) - zf * zf) : T(0);
            __syncwarp();
            T dh, w;  // dE/dh^M = fW1^T dzf and U2^T dE/dh^M = (fW1 U2)^T dzf
            twmv2<T, 32>(fY3, sm.t, lane, lane + 32, dh, w, tm, sm);
            __syncwarp();
            TP(7);
            if constexpr (PULL == 0)
                msg_backward_warp<T, G, false>(nullptr, uW1T, mb1, c1, w, w1b, gr, ws, sm, l, i,
                                               dh, zu, true, tm, pre, ar.e0, mloc);
            else  // the edges' share runs at their senders (k_msg_bwd_pull / k_embed_bwd_pull)
                upd_bwd_pull<T, G>(nullptr, uW1T, c1, w, ws, sm, n, l, i, dh, zu, tm);
            TP(8);
        }
        __syncwarp();
    }
    if (!staged) Smem<T>::wait(&s_mbar);  // no CTA exits with its weight copy in flight
}

// Message layer l < M-1 backward: gather dE/dh^{l+1}, then the layer body.
template <typename T, int G, bool LIST = false>
__global__ __launch_bounds__(kPushWarps * 32, kNetMinCTAs<G>) void k_msg_bwd(DevModel<T> md, DevGraph gr,
                                                               DevWork<T> ws, int l) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    pdl_launch_dependents();
    const DevMlp<T>& msg = md.msg[l];
    const DevMlp<T>& upd = md.upd[l];
    Smem<T> sg(reinterpret_cast<T*>(smem_raw));
    __shared__ unsigned long long s_mbar;
    // W1h^(l+1)^T: rows 0..31 of msg[l+1].W1T ([in][32])
    const T* nW1hT = sg.template view<32, 32>();
    const T* uW2T = sg.template view<32, 32>();
    const T* uW1T = sg.template view<64, 32>();  // [U1h^T ; (U1m W2)^T]
    sg.load(md.img_bwd[l], &s_mbar);
    WarpSmem<T>& sm = sg.warp_scratch();
    Team<G> tm;
    const int lane = tm.lane;
    T w1b[kK];
#pragma unroll
    for (int k = 0; k < kK; ++k) w1b[k] = msg.W1T[(kH + k) * kH + lane];
    const T mb1 = msg.b1[lane], c1 = md.uc1[l][lane];
    __syncthreads();  // publishes the mbarrier init; the copy is awaited at first use
    bool staged = false;
    pdl_wait();
    const T* Dn = ws.d + ((l + 1) & 1) * ws.slots * kH;
    // kRecomputeZ: z_e recomputed from P^l_j; else the rows the forward stored
    const T* Pl = kRecomputeZ ? ws.pa + static_cast<long long>(l) * gr.n * kH
                              : ws.z + static_cast<long long>(l) * ws.slots * kH;
    // LIST (global-index DD): the atoms alist[0 .. *alist_n); else [0, n_active)
    const int n_run = LIST ? *gr.alist_n : gr.n_active;
    for (int k_at = tm.first; k_at < n_run; k_at += tm.stride) {
        const int i = LIST ? gr.alist[k_at] : k_at;
        AtomRow<G> ar(gr, i, tm);
        // one round trip: own adjoint, update activations, the pushed adjoint rows
        // and the backward edge loop's first batch
        const T own = ws.dhown[static_cast<long long>(i) * kH + lane];
        const T zu = ws.uz1[(static_cast<long long>(l) * gr.n + i) * kH + lane];
        GatherPre<T, G> gp;
        if (gr.sym) gp.load(Dn, ar.e0, ar.room, lane);
        BwdPre<T> pre;
        bwd_prefetch<T, G, kRecomputeZ>(pre, Pl, ws, gr, ar.e0, min(ar.room, 32), lane);
        const int mloc = ar.finish(tm);
        T sv;
        if (gr.sym) {
            sv = tm.sum(gp.sum(Dn, ar.e0, mloc, lane), sm);
            if (ws.s_remote) sv += ws.s_remote[static_cast<long long>(i) * kH + lane];
        } else {
            sv = gather_in(Dn, ws, gr, i, tm, sm);
        }
        if (!staged) {  // weights (bulk copy issued at kernel entry) needed from here on
            Smem<T>::wait(&s_mbar);
            staged = true;
        }
        sm.t[lane] = sv;
        __syncwarp();
        // dE/dh^{l+1}_i = own + W1h^(l+1)^T S_i
        const T dh = own + twmv<T, 32>(nW1hT, sm.t, lane, tm, sm);
        __syncwarp();
        msg_backward_warp<T, G, kRecomputeZ>(uW2T, uW1T, mb1, c1, T(0), w1b, gr, ws, sm, l, i, dh,
                                             zu, false, tm, pre, ar.e0, mloc);
        __syncwarp();
    }
    if (!staged) Smem<T>::wait(&s_mbar);  // no CTA exits with its weight copy in flight
}

// Embedding backward + descriptor adjoint (depth > 1); pushes g to the mirrors.
template <typename T, int G, bool LIST = false>
__global__ __launch_bounds__(kPushWarps * 32, kNetMinCTAs<G>) void k_embed_bwd(DevModel<T> md, DevGraph gr,
                                                                 DevWork<T> ws) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    pdl_launch_dependents();
    Smem<T> sg(reinterpret_cast<T*>(smem_raw));
    __shared__ unsigned long long s_mbar;
    const T* m0W1hT = sg.template view<32, 32>();
    const T* eW2T = sg.template view<32, 32>();
    const T* eW1T = sg.template view<32, 32>();
    sg.load(md.img_embed_bwd, &s_mbar);
    WarpSmem<T>& sm = sg.warp_scratch();
    Team<G> tm;
    const int lane = tm.lane;
    __syncthreads();  // publishes the mbarrier init; the copy is awaited at first use
    bool staged = false;
    pdl_wait();
    // LIST (global-index DD): the atoms alist[0 .. *alist_n); else [0, n_active)
    const int n_run = LIST ? *gr.alist_n : gr.n_active;
    for (int k_at = tm.first; k_at < n_run; k_at += tm.stride) {
        const int i = LIST ? gr.alist[k_at] : k_at;
        AtomRow<G> ar(gr, i, tm);
        const T own = ws.dhown[static_cast<long long>(i) * kH + lane];
        const T z1 = ws.ez1[static_cast<long long>(i) * kH + lane];
        GatherPre<T, G> gp;
        if (gr.sym) gp.load(ws.d, ar.e0, ar.room, lane);
        // first batch of the per-edge descriptor adjoint (lane = local edge)
        V4<T> d0_l{}, d1_l{};
        T g_l = T(0);
        int ty_l = 0, mir_l = 0;
        if (lane < ar.room) {
            const long long e = ar.e0 + static_cast<long long>(G) * lane;
            d0_l = ld4c(ws.edb + 8 * e);
            d1_l = ld4c(ws.edb + 8 * e + 4);
            g_l = ws.g[e];
            ty_l = gr.ety[e];
            mir_l = gr.inv_pos[e];
        }
        const int mloc = ar.finish(tm);
        T sv;
        if (gr.sym) {
            sv = tm.sum(gp.sum(ws.d, ar.e0, mloc, lane), sm);
            if (ws.s_remote) sv += ws.s_remote[static_cast<long long>(i) * kH + lane];
        } else {
            sv = gather_in(ws.d, ws, gr, i, tm, sm);
        }
        if (!staged) {  // weights (bulk copy issued at kernel entry) needed from here on
            Smem<T>::wait(&s_mbar);
            staged = true;
        }
        sm.t[lane] = sv;
        __syncwarp();
        const T dh = own + twmv<T, 32>(m0W1hT, sm.t, lane, tm, sm);
        sm.x[lane] = dh;
        __syncwarp();
        const T dz1 = twmv<T, 32>(eW2T, sm.x, lane, tm, sm) * (T(1) - z1 * z1);
        sm.y[lane] = dz1;
        __syncwarp();
        const T dd = twmv<T, 32>(eW1T, sm.y, lane, tm, sm);
        sm.t[lane] = dd;
        __syncwarp();
        for (int q = lane; q < mloc; q += 32) {
            const long long e = ar.e0 + static_cast<long long>(G) * q;
            if (q >= 32) {
                d0_l = ld4c(ws.edb + 8 * e);
                d1_l = ld4c(ws.edb + 8 * e + 4);
                g_l = ws.g[e];
                ty_l = gr.ety[e];
                mir_l = gr.inv_pos[e];
            }
            const T* dv = sm.t + ty_l * kK;
            T acc = dv[0] * d0_l.x;
            acc += dv[1] * d0_l.y;
            acc += dv[2] * d0_l.z;
            acc += dv[3] * d0_l.w;
            acc += dv[4] * d1_l.x;
            acc += dv[5] * d1_l.y;
            acc += dv[6] * d1_l.z;
            acc += dv[7] * d1_l.w;
            const T gv = g_l + acc;
            ws.g[e] = gv;
            ws.grev[mir_l] = gv;  // mirror for the force gather
        }
        __syncwarp();
    }
    if (!staged) Smem<T>::wait(&s_mbar);  // no CTA exits with its weight copy in flight
}

// Pull form, lower layers (l < M-1): the sender-side backward of layer l+1's
// messages (gathering the receivers' v^{l+1} rows), dE/dh^{l+1}_k, then layer l's
// update backward (v^l_k, c0^l_k for the next kernel).
//
// DD (halo-exchange domain decomposition, alist-driven): 1 = the sender-side half
// over the searched rows (owned + halo), dE/dh partial sums into ws.dd_sum (the
// halo rows' travel to their owners in the SUMS round); 2 = the update half over
// the owned rows, from dd_sum + s_remote.
template <typename T, int G, int PULL, bool WIDE = false, int DD = 0>
__global__ __launch_bounds__(kCtaWarps<T, G, WIDE> * 32, kNetMinCTAs<G>) void k_msg_bwd_pull(DevModel<T> md,
                                                                    DevGraph gr, DevWork<T> ws,
                                                                    int l) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    pdl_launch_dependents();
    const DevMlp<T>& msgn = md.msg[l + 1];  // the messages whose backward runs here
    Smem<T> sg(reinterpret_cast<T*>(smem_raw));
    __shared__ unsigned long long s_mbar;
    const T* nW1hT = sg.template view<32, 32>();  // W1h^(l+1)^T
    const T* uW2T = sg.template view<32, 32>();
    const T* uW1T = sg.template view<64, 32>();  // [U1h^T ; (U1m W2)^T]
    sg.load(md.img_bwd[l], &s_mbar);
    WarpSmem<T>& sm = sg.warp_scratch();
    Team<G> tm;
    const int lane = tm.lane;
    T w1b[kK];
#pragma unroll
    for (int k = 0; k < kK; ++k) w1b[k] = msgn.W1T[(kH + k) * kH + lane];
    const T mb1n = msgn.b1[lane], c1 = md.uc1[l][lane];
    __syncthreads();  // publishes the mbarrier init; the copy is awaited at first use
    bool staged = false;
    pdl_wait();
    const int n = gr.n;
    const T* Z = ws.z + static_cast<long long>(l + 1) * ws.slots * kH;
    const T* V = ws.vrow + static_cast<long long>((l + 1) & 1) * n * kH;
    const T* C0 = ws.vc0 + static_cast<long long>((l + 1) & 1) * n;
    // the first backward kernel overwrites g; DD: at every slot of every searched row
    // (masked slots get 0), so no zeroing pass is needed
    const bool first_g = l == md.n_msg - 2;
    const int n_run = DD ? *gr.alist_n : gr.n_active;
    for (int k_at = tm.first; k_at < n_run; k_at += tm.stride) {
        const int k = DD ? gr.alist[k_at] : k_at;
        if (DD == 2 && !ws.dd_bnd[k]) continue;  // finished by the sender half
        const T own = ws.dhown[static_cast<long long>(k) * kH + lane];
        const T zu = ws.uz1[(static_cast<long long>(l) * n + k) * kH + lane];
        T sdz;
        if constexpr (DD == 2) {
            sdz = ws.dd_sum[static_cast<long long>(k) * kH + lane] +
                  ws.s_remote[static_cast<long long>(k) * kH + lane];
        } else {
            AtomRow<G> ar(gr, k, tm);
            const T pk =
                PULL == 2 ? ws.pa[(static_cast<long long>(l + 1) * n + k) * kH + lane] : T(0);
            const int mloc = ar.finish(tm);
            sdz = pull_edges<T, G, PULL, DD == 1>(w1b, mb1n, pk, Z, V, C0, gr, ws, sm, ar.e0, mloc,
                                                  first_g, lane,
                                                  DD == 0 || ws.dd_role[k] == 1);
            sdz = tm.sum(sdz, sm);
            if constexpr (DD == 1) {
                // owned rows no peer sends partial sums to are finished here; the
                // rest wait for the SUMS round (DD = 2)
                if (ws.dd_role[k] != 1 || ws.dd_bnd[k]) {
                    if (tm.w == 0) {
                        ws.dd_sum[static_cast<long long>(k) * kH + lane] = sdz;
                        if (ws.dd_role[k] == 1)  // the SUMS round adds the peers' rows here
                            ws.s_remote[static_cast<long long>(k) * kH + lane] = T(0);
                    }
                    __syncwarp();
                    continue;
                }
            }
        }
        if (!staged) {  // weights (bulk copy issued at kernel entry) needed from here on
            Smem<T>::wait(&s_mbar);
            staged = true;
        }
        sm.t[lane] = sdz;
        __syncwarp();
        // dE/dh^{l+1}_k = own + W1h^(l+1)^T sum_e dz_e
        const T dh = own + twmv<T, 32>(nW1hT, sm.t, lane, tm, sm);
        __syncwarp();
        upd_bwd_pull<T, G>(uW2T, uW1T, c1, T(0), ws, sm, n, l, k, dh, zu, tm);
    }
    if (!staged) Smem<T>::wait(&s_mbar);  // no CTA exits with its weight copy in flight
}

// Pull form, embedding backward: the sender-side backward of layer 0's messages,
// dE/dh^0_k, the embedding backward and the descriptor adjoint; pushes the final
// g to the mirrors for the force gather.
// DD: as k_msg_bwd_pull (1 = sender half over the searched rows, 2 = the rest over
// the owned rows; the force kernel then gathers the mirror g itself, no grev).
template <typename T, int G, int PULL, bool WIDE = false, int DD = 0>
__global__ __launch_bounds__(kCtaWarps<T, G, WIDE> * 32, kNetMinCTAs<G>) void k_embed_bwd_pull(DevModel<T> md,
                                                                      DevGraph gr,
                                                                      DevWork<T> ws) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    pdl_launch_dependents();
    const DevMlp<T>& msg0 = md.msg[0];
    Smem<T> sg(reinterpret_cast<T*>(smem_raw));
    __shared__ unsigned long long s_mbar;
    const T* m0W1hT = sg.template view<32, 32>();
    const T* eW2T = sg.template view<32, 32>();
    const T* eW1T = sg.template view<32, 32>();
    sg.load(md.img_embed_bwd, &s_mbar);
    WarpSmem<T>& sm = sg.warp_scratch();
    Team<G> tm;
    const int lane = tm.lane;
    T w1b[kK];
#pragma unroll
    for (int k = 0; k < kK; ++k) w1b[k] = msg0.W1T[(kH + k) * kH + lane];
    const T mb1 = msg0.b1[lane];
    __syncthreads();  // publishes the mbarrier init; the copy is awaited at first use
    bool staged = false;
    pdl_wait();
    const int n = gr.n;
    const bool first_g = md.n_msg == 1;  // (see k_msg_bwd_pull)
    const int n_run = DD ? *gr.alist_n : gr.n_active;
    for (int k_at = tm.first; k_at < n_run; k_at += tm.stride) {
        const int k = DD ? gr.alist[k_at] : k_at;
        if (DD == 2 && !ws.dd_bnd[k]) continue;  // finished by the sender half
        AtomRow<G> ar(gr, k, tm);
        const T own = ws.dhown[static_cast<long long>(k) * kH + lane];
        const T z1 = ws.ez1[static_cast<long long>(k) * kH + lane];
        const int mloc = ar.finish(tm);
        T sdz;
        if constexpr (DD == 2) {
            sdz = ws.dd_sum[static_cast<long long>(k) * kH + lane] +
                  ws.s_remote[static_cast<long long>(k) * kH + lane];
        } else {
            const T pk = PULL == 2 ? ws.pa[static_cast<long long>(k) * kH + lane] : T(0);
            sdz = pull_edges<T, G, PULL, DD == 1>(w1b, mb1, pk, ws.z, ws.vrow, ws.vc0, gr, ws, sm,
                                                  ar.e0, mloc, first_g, lane,
                                                  DD == 0 || ws.dd_role[k] == 1);
            sdz = tm.sum(sdz, sm);
            if constexpr (DD == 1) {
                // owned rows no peer sends partial sums to are finished here; the
                // rest wait for the SUMS round (DD = 2)
                if (ws.dd_role[k] != 1 || ws.dd_bnd[k]) {
                    if (tm.w == 0) {
                        ws.dd_sum[static_cast<long long>(k) * kH + lane] = sdz;
                        if (ws.dd_role[k] == 1)  // the SUMS round adds the peers' rows here
                            ws.s_remote[static_cast<long long>(k) * kH + lane] = T(0);
                    }
                    __syncwarp();
                    continue;
                }
            }
        }
        if (!staged) {  // weights (bulk copy issued at kernel entry) needed from here on
            Smem<T>::wait(&s_mbar);
            staged = true;
        }
        sm.t[lane] = sdz;
        __syncwarp();
        const T dh = own + twmv<T, 32>(m0W1hT, sm.t, lane, tm, sm);
        sm.x[lane] = dh;
        __syncwarp();
        const T dz1 = twmv<T, 32>(eW2T, sm.x, lane, tm, sm) * (T(1) - z1 * z1);
        sm.y[lane] = dz1;
        __syncwarp();
        const T dd = twmv<T, 32>(eW1T, sm.y, lane, tm, sm);
        sm.t[lane] = dd;
        __syncwarp();
        // descriptor adjoint per edge (lane = local edge), on top of the message
        // terms this warp just wrote; then the mirror copy for the force gather
        for (int q = lane; q < mloc; q += 32) {
            const long long e = ar.e0 + static_cast<long long>(G) * q;
            const V4<T> d0 = ld4c(ws.edb + 8 * e), d1 = ld4c(ws.edb + 8 * e + 4);
            const T* dv = sm.t + gr.ety[e] * kK;
            T acc = dv[0] * d0.x;
            acc += dv[1] * d0.y;
            acc += dv[2] * d0.z;
            acc += dv[3] * d0.w;
            acc += dv[4] * d1.x;
            acc += dv[5] * d1.y;
            acc += dv[6] * d1.z;
            acc += dv[7] * d1.w;
            const T gv = ws.g[e] + acc;
            ws.g[e] = gv;
            if constexpr (DD == 0) ws.grev[gr.inv_pos[e]] = gv;  // mirror for the force gather
        }
        __syncwarp();
    }
    if (!staged) Smem<T>::wait(&s_mbar);  // no CTA exits with its weight copy in flight
}

// ---------------------------------------------------------------------------
// Forces (gather form), per-atom energy, virial, and the velocity-Verlet tail of
// the device MD loop.  A group of FG lanes per atom (FG = 32: one warp per atom
// for small systems, where every SM should get atoms; FG = 8: four atoms per warp
// for large ones -- 3-level group sums instead of 5-level warp sums, the MD tail
// of four atoms at once, and a grid that fits one wave of resident CTAs).
//   F_i = sum_{e in out(i)} u_e g_e - sum_{e' in in(i)} u_e' g_e'
//       = sum_q u_q (g_q + grev_q)            (symmetric list: u_rev(e) = -u_e)
//   W   = -sum_e g_e r_e ;  W_ab = -sum_e g_e dr_a u_b
// CTA partials of (E, W, W_ab) in a fixed order, then the last CTA to finish
// reduces all CTAs' partials in a fixed order (deterministic).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void reduce_partials(const double* partial, unsigned nb, double* out,
                                                double (*s_part)[12]);

template <int FG>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
    for (int o = FG / 2; o > 0; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
    return v;
}

// DDG: the pull-form DD's variant (mirror gathers skip pairs of two non-owned rows).
template <typename T, int FG, bool DDG = false>
__global__ __launch_bounds__(kForceCTA) void k_force(DevGraph gr, DevWork<T> ws,
                                                     double* __restrict__ forces,
                                                     double* __restrict__ per_atom,
                                                     double* __restrict__ out, MdFuse mf) {
    __shared__ double s_part[kForceCTA / 32][12];
    __shared__ bool s_last;
    pdl_launch_dependents();
    pdl_wait();
    constexpr int APW = 32 / FG;  // atoms per warp
    const int lane = threadIdx.x & 31, wc = threadIdx.x >> 5;
    const int sub = lane % FG, grp = lane / FG;
    const int gw = blockIdx.x * (blockDim.x >> 5) + wc, nw = gridDim.x * (blockDim.x >> 5);
    double acc[11];
#pragma unroll
    for (int q = 0; q < 11; ++q) acc[q] = 0.0;
    for (int base = gw * APW; base < gr.n; base += nw * APW) {  // warp-uniform trip count
        const int i = base + grp;
        const bool act = i < gr.n;
        // MD state of atom i, loaded early (independent of the edge loads)
        double xv[3] = {0, 0, 0}, vv[3] = {0, 0, 0}, xr[3] = {0, 0, 0}, mi = 1.0, ei = 0.0;
        if (act && sub == 0) {
            ei = ws.e_atom[i];
            if (mf.mode) {
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    vv[a] = mf.v[3 * i + a];
                    xv[a] = mf.x[3 * i + a];
                }
                mi = mf.m[i];
                if (mf.vflag)  // Verlet-row reference position, for the drift's check
#pragma unroll
                    for (int a = 0; a < 3; ++a) xr[a] = mf.xref[3 * i + a];
            }
        }
        double fx = 0.0, fy = 0.0, fz = 0.0;
        const int start = act ? gr.row_start[i] : 0, cnt = act ? gr.nnei[i] : 0;
        if (ws.gv) {  // DeePMD-style families: vector dE/d(edge_dr) (hmdp_dp.cu)
            //   F_i = sum_q (gv_q - gv_rev(q));  W_ab = -sum_q dr_a gv_b
            for (int q = sub; q < cnt; q += FG) {
                const int e = start + q;
                const V4<T> g = ld4c(ws.gv + 4ll * e);
                const double* d = gr.dr + 3ll * e;
                const double g3[3] = {static_cast<double>(g.x), static_cast<double>(g.y),
                                      static_cast<double>(g.z)};
                fx += g3[0];
                fy += g3[1];
                fz += g3[2];
                if (gr.sym) {
                    const V4<T> m = ld4c(ws.gvrev + 4ll * e);
                    fx -= static_cast<double>(m.x);
                    fy -= static_cast<double>(m.y);
                    fz -= static_cast<double>(m.z);
                }
                acc[1] -= d[0] * g3[0] + d[1] * g3[1] + d[2] * g3[2];
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int b = 0; b < 3; ++b) acc[2 + 3 * a + b] -= d[a] * g3[b];
            }
            if (!gr.sym && act) {
                const int is = gr.in_start[i], ic = gr.in_cnt[i];
                for (int q = sub; q < ic; q += FG) {
                    const V4<T> m = ld4c(ws.gvrev + 4ll * (is + q));
                    fx -= static_cast<double>(m.x);
                    fy -= static_cast<double>(m.y);
                    fz -= static_cast<double>(m.z);
                }
            }
        } else {
            for (int q = sub; q < cnt; q += FG) {
                const int e = start + q;
                const T gg = ws.g[e];
                T gm = T(0);
                if (gr.sym) {
                    if (ws.gather_mirror_g) {
                        // (pull-form DD: pairs of two non-owned rows carry no terms and
                        // have no mirror slot)
                        const int mq = gr.inv_pos[e];
                        if (mq >= 0 && (!DDG || ws.dd_role[i] == 1 ||
                                        ws.dd_role[gr.nbr[e]] == 1))
                            gm = ws.g[mq];
                    } else {
                        gm = ws.grev[e];
                    }
                }
                T x, y, z;
                const double* d = gr.dr + 3ll * e;
                const T r = edge_len<T>(d, x, y, z);
                const T ux = x / r, uy = y / r, uz = z / r;
                fx += static_cast<double>(ux * gg) + static_cast<double>(ux * gm);
                fy += static_cast<double>(uy * gg) + static_cast<double>(uy * gm);
                fz += static_cast<double>(uz * gg) + static_cast<double>(uz * gm);
                acc[1] -= static_cast<double>(gg * r);
                const double gd = static_cast<double>(gg);
                const double u3[3] = {static_cast<double>(ux), static_cast<double>(uy),
                                      static_cast<double>(uz)};
#pragma unroll
                for (int a = 0; a < 3; ++a)
#pragma unroll
                    for (int b = 0; b < 3; ++b) acc[2 + 3 * a + b] -= gd * d[a] * u3[b];
            }
            if (!gr.sym && act) {  // generic CSR: the pushed g of each in-edge, its own geometry
                const int is = gr.in_start[i], ic = gr.in_cnt[i];
                for (int q = sub; q < ic; q += FG) {
                    const int e = gr.in_edge[is + q];
                    const T gg = ws.grev[is + q];
                    T x, y, z;
                    const T r = edge_len<T>(gr.dr + 3ll * e, x, y, z);
                    fx -= static_cast<double>((x / r) * gg);
                    fy -= static_cast<double>((y / r) * gg);
                    fz -= static_cast<double>((z / r) * gg);
                }
            }
        }
        fx = group_sum<FG>(fx);
        fy = group_sum<FG>(fy);
        fz = group_sum<FG>(fz);
        // forces (and per-atom energies) of the warp's APW consecutive atoms as one
        // contiguous store per array (3 APW doubles): one wide write instead of 3 APW
        // scattered ones, which matters when the output is host-mapped memory
        // (hmdp_compute's graph path writes across PCIe)
        const bool full = ws.wide_out && base + APW <= gr.n;  // warp-uniform
        if (full) {
            const int src = ((lane % (3 * APW)) / 3) * FG;
            const double vx = __shfl_sync(FULL_MASK, fx, src);
            const double vy = __shfl_sync(FULL_MASK, fy, src);
            const double vz = __shfl_sync(FULL_MASK, fz, src);
            const int c = lane % 3;
            if (lane < 3 * APW) forces[3ll * base + lane] = c == 0 ? vx : (c == 1 ? vy : vz);
            if (per_atom) {
                const double e = __shfl_sync(FULL_MASK, ei, (lane % APW) * FG);
                if (lane < APW) per_atom[base + lane] = e;
            }
        }
        if (act && sub == 0) {
            const double f3[3] = {fx, fy, fz};
            if (!full) {
                forces[3 * i] = fx;
                forces[3 * i + 1] = fy;
                forces[3 * i + 2] = fz;
                if (per_atom) per_atom[i] = ei;
            }
            acc[0] += ei;
            if (mf.mode) {
                const double s = mf.half / mi;
                const bool finite = isfinite(fx) && isfinite(fy) && isfinite(fz);
                if (!finite) atomicOr(ws.err, kErrNonFinite);
                double x3[3];
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    double va = __dadd_rn(vv[a], __dmul_rn(f3[a], s));  // closing kick
                    if (mf.vs) {  // completed step: the state hmdp_md_get returns
                        mf.vs[3 * i + a] = va;
                        mf.xs[3 * i + a] = xv[a];
                    }
                    if (mf.mode == 2) {
                        va = __dadd_rn(va, __dmul_rn(f3[a], s));  // next step's opening kick
                        x3[a] = __dadd_rn(xv[a], __dmul_rn(va, mf.dt));
                        mf.x[3 * i + a] = x3[a];
                    }
                    mf.v[3 * i + a] = va;
                }
                if (mf.mode == 2) {
                    vlist_check(x3, xr, mf);
                    bin_atom(i, x3, mf.cg, mf.cell_count, mf.members, mf.cell_of, ws.err);
                }
            }
        }
    }
#pragma unroll
    for (int q = 0; q < 11; ++q) acc[q] = warp_sum(acc[q]);
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < 11; ++q) s_part[wc][q] = acc[q];
    __syncthreads();
    if (threadIdx.x < 11) {
        double v = 0.0;
        for (int q = 0; q < kForceCTA / 32; ++q) v += s_part[q][threadIdx.x];
        ws.partial[blockIdx.x * 16 + threadIdx.x] = v;
    }
    // device MD: the (E, W) totals are reduced on demand (hmdp_md_get ->
    // k_reduce_partials); a single evaluation reduces here, in the last CTA
    if (mf.mode) return;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(ws.ticket, 1u) == gridDim.x - 1);
    __syncthreads();
    if (s_last) {
        __threadfence();
        reduce_partials(ws.partial, gridDim.x, out, s_part);
        if (threadIdx.x == 0) {
            *ws.ticket = 0u;  // re-arm for the next launch / graph replay
            if (ws.export_err) {
                out[12] = static_cast<double>(*ws.err);
                *ws.err = 0u;
            }
        }
    }
}

// Fixed-order sum of nb CTA partials (E, W, W_ab) into out[0..10], by one CTA of
// kForceCTA threads.
__device__ __forceinline__ void reduce_partials(const double* partial, unsigned nb, double* out,
                                                double (*s_part)[12]) {
    const int lane = threadIdx.x & 31, wc = threadIdx.x >> 5;
    double v[11];
#pragma unroll
    for (int q = 0; q < 11; ++q) v[q] = 0.0;
    for (unsigned b = threadIdx.x; b < nb; b += kForceCTA)
#pragma unroll
        for (int q = 0; q < 11; ++q) v[q] += __ldcg(partial + b * 16 + q);
#pragma unroll
    for (int q = 0; q < 11; ++q) v[q] = warp_sum(v[q]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < 11; ++q) s_part[wc][q] = v[q];
    __syncthreads();
    if (threadIdx.x < 11) {
        double tot = 0.0;
        for (int q = 0; q < kForceCTA / 32; ++q) tot += s_part[q][threadIdx.x];
        out[threadIdx.x] = tot;
    }
}

__global__ __launch_bounds__(kForceCTA) void k_reduce_partials(const double* partial, int nb,
                                                               double* out) {
    __shared__ double s_part[kForceCTA / 32][12];
    reduce_partials(partial, nb, out, s_part);
}

// ---------------------------------------------------------------------------
// Domain-decomposition helpers (halo ghosts are atoms [n_active, n)).
// ---------------------------------------------------------------------------
// The received per-atom projections P of halo ghosts into the layer's P rows
// (what the owner would have written had the ghost been local).
template <typename T>
__global__ void k_dd_ghost_p(DevGraph gr, const T* __restrict__ p_atom, T* __restrict__ pa) {
    const int i = gr.n_active + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= gr.n) return;
    pa[static_cast<long long>(i) * kH + lane] = p_atom[static_cast<long long>(i) * kH + lane];
}
// Partial dE/dh adjoint sums collected at halo ghosts (sent back to the owners).
template <typename T>
__global__ void k_dd_ghost_sums(DevGraph gr, const T* __restrict__ d, T* __restrict__ out) {
    const int i = gr.n_active + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= gr.n) return;
    const int is = gr.in_start[i], ic = gr.in_cnt[i];
    T s = T(0);
    for (int k = 0; k < ic; ++k) s += d[static_cast<long long>(is + k) * kH + lane];
    out[static_cast<long long>(i) * kH + lane] = s;
}

// ---------------------------------------------------------------------------
// launch
// ---------------------------------------------------------------------------
// Staged weight elements per kernel (must follow the kernels' staging order).
enum class Phase { EmbedFit, Embed, MsgFwd, MsgFwdLast, MsgBwd, EmbedBwd };
template <typename T>
static int staged_elems(Phase p) {
    const int m32 = mat_elems<T>(32, 32), m64 = mat_elems<T>(32, 64), t64 = mat_elems<T>(64, 32);
    switch (p) {
        case Phase::EmbedFit: return 3 * m32 + t64;
        case Phase::Embed: return m32 + t64;
        case Phase::MsgFwd: return 2 * m32 + m64;
        case Phase::MsgFwdLast: return m32 + m64 + 3 * t64;
        case Phase::MsgBwd: return 2 * m32 + t64;
        case Phase::EmbedBwd: return 3 * m32;
    }
    return 0;
}

// Launch shape: team size G (warps per atom) from the system size — the
// largest of 4, 2, 1 that keeps every atom's team resident at 16 warps per SM —
// then enough teams per CTA that the atoms fill every SM, grid-stride beyond
// two CTAs per SM.
struct NetShape {
    int G, warps, grid;
    int wide = 0;  // 1: the 28-warp-CTA (WIDE) build of the 2-warp-team kernels
};
static bool wide_on() {  // HMDP_WIDE=0 keeps the 20-warp build (A/B experiments)
    static const bool v = [] {
        const char* e = std::getenv("HMDP_WIDE");
        return !(e && std::atoi(e) == 0);
    }();
    return v;
}
int team_override() {  // HMDP_TEAM=1|2|4 pins the team size (tuning experiments)
    static const int v = [] {
        const char* e = std::getenv("HMDP_TEAM");
        const int t = e ? std::atoi(e) : 0;
        return (t == 1 || t == 2 || t == 4) ? t : 0;
    }();
    return v;
}
// Team size by system size and model (measured on B200): 4 warps per
// atom up to 4 atoms per SM (1YRF); 2 warps per atom for the message-passing model
// up to ~40 atoms per SM (1UBQ 7.5k -> 11.4k, 3LZM 6.8k -> 8.1k steps/s vs 1 warp;
// 2PTC on par, warm L2 6.3k vs 3.9k) and for embed_fit up to ~10 atoms per SM
// (1UBQ 24.2k -> 28.9k; 3LZM and 2PTC prefer 1 warp); 1 warp beyond.
// FP64 (the oracle-of-record mode) caps a CTA at 8 warps: its per-warp scratch and
// staged matrices are twice as large and 16 warps would not fit in shared memory.
static NetShape net_shape(int n, int n_msg, int elem_bytes, bool allow_wide = false,
                          bool push = false) {
    const int sms = num_sms();
    const int two_upto = (n_msg > 0 ? 40 : 10) * sms;
    int G = (4 * n <= kMaxWarps * sms) ? 4 : (n <= two_upto ? 2 : 1);
    if (team_override()) G = team_override();
    const int max_warps = elem_bytes > 4 ? kMaxWarps / 2
                          : (G == 1 ? kCtaWarps<float, 1> : (push ? kPushWarps : kCtaWarps<float, 2>));
    int max_teams = max_warps / G;
    // Every team takes whole atoms, so a kernel runs ceil(n / teams) rounds of them:
    // take the fewest teams per CTA that keep the fewest rounds (more registers and
    // issue slots per warp at the same round count; 3LZM: 9 teams, 2 rounds).  For
    // FP32 2-warp teams, the 28-warp build (WIDE, 14 teams) is taken when it needs
    // fewer rounds than the 20-warp one (2PTC: 2 rounds instead of 3).
    bool wide = false;
    auto rounds = [&](int t) { return (n + sms * t - 1) / (sms * t); };
    if (allow_wide && G == 2 && elem_bytes == 4 && n_msg > 0 && wide_on()) {
        const int tw = kCtaWarps<float, 2, true> / 2;
        if (rounds(tw) < rounds(max_teams)) {
            wide = true;
            max_teams = tw;
        }
    }
    const int r = rounds(max_teams);
    int teams = (n + sms * r - 1) / (sms * r);
    teams = teams < 1 ? 1 : (teams > max_teams ? max_teams : teams);
    if (G == 1 && teams < 2) teams = 2;
    int grid = (n + teams - 1) / teams;
    if (grid > 2 * sms) grid = 2 * sms;
    return {G, teams * G, grid < 1 ? 1 : grid, wide ? 1 : 0};
}

// CTAs of a kernel resident per SM at a given block / shared-memory size (cached;
// launches are capped at one wave of them).
static int resident_ctas(const void* fn, int threads, size_t smem) {
    static std::mutex mu;
    static std::map<std::tuple<const void*, int, size_t>, int> cache;
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(fn, threads, smem);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, threads, smem) != cudaSuccess || nb < 1) {
        cudaGetLastError();
        nb = 1;
    }
    cache.emplace(key, nb);
    return nb;
}

template <typename T, typename... Params, typename... Args>
static void launch_net(void (*kernel)(Params...), Phase p, const NetShape& sh, cudaStream_t st,
                       Args... args) {
    const size_t smem = static_cast<size_t>(staged_elems<T>(p)) * sizeof(T) + 16 +
                        static_cast<size_t>(sh.warps) * sizeof(WarpSmem<T>);
    // at most one wave of resident CTAs: the teams grid-stride over the remaining
    // atoms instead of a partial second wave of CTAs doubling the kernel time
    int grid = sh.grid;
    const int per_sm = resident_ctas(reinterpret_cast<const void*>(kernel), 32 * sh.warps, smem);
    const int g = per_sm * num_sms();
    grid = g < grid ? g : grid;
    const cudaError_t e = launch_pdl(kernel, dim3(grid), dim3(32 * sh.warps), smem, st, args...);
    if (e != cudaSuccess && std::getenv("HMDP_DEBUG_LAUNCH")) {
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, kernel);
        std::fprintf(stderr,
                     "launch_net failed: %s grid %d block %d smem %zu | attr maxThreads %d regs %d "
                     "static smem %zu maxDyn %d\n",
                     cudaGetErrorString(e), sh.grid, 32 * sh.warps, smem, fa.maxThreadsPerBlock,
                     fa.numRegs, fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes);
    }
}

// Lanes per atom of the force kernel: a warp per atom while the atoms do not fill
// the SMs' resident warps (every SM gets atoms), 16 up to 64 atoms per SM, 8 beyond
// (HMDP_FORCE_FG pins it).  Measured (profiles/round2/ab/force_fg16.txt, force_fg2.txt):
// at 3LZM / 2PTC (18 / 28 atoms per SM) 16 lanes beat 8 by 2 % (DPA3) and 5-7 % (DPA2);
// at 1YRF / 1UBQ 32 lanes stay best, at 2PTC x8 (222 atoms per SM) 8.
int force_fg(int n) {
    static const int env = [] {
        const char* e = std::getenv("HMDP_FORCE_FG");
        const int v = e ? std::atoi(e) : 0;
        return (v == 8 || v == 16 || v == 32) ? v : 0;
    }();
    if (env) return env;
    return n <= num_sms() * 16 ? 32 : (n <= num_sms() * 64 ? 16 : 8);
}
int force_grid(int n) {
    const int apc = (kForceCTA / 32) * (32 / force_fg(n));  // atoms per CTA
    const int want = (n + apc - 1) / apc;
    const int cap = num_sms() * 16;
    return want < 1 ? 1 : (want < cap ? want : cap);
}
template <typename T>
static void launch_force_k(const DevGraph& gr, const DevWork<T>& ws, double* forces,
                           double* per_atom, double* out, cudaStream_t st, const MdFuse& mf,
                           bool ddg = false) {
    const dim3 grid(force_grid(gr.n)), block(kForceCTA);
    auto go = [&](auto k) { launch_pdl(k, grid, block, 0, st, gr, ws, forces, per_atom, out, mf); };
    switch (force_fg(gr.n)) {
        case 8: ddg ? go(k_force<T, 8, true>) : go(k_force<T, 8>); break;
        case 16: ddg ? go(k_force<T, 16, true>) : go(k_force<T, 16>); break;
        default: ddg ? go(k_force<T, 32, true>) : go(k_force<T, 32>); break;
    }
}

constexpr int kMaxSmem = 200 * 1024;

// Message backward form (see pull_edges): the pull form needs the symmetric
// periodic graph with every atom running the network (no halo ghosts, no global
// list, no domain-decomposition rows); everything else runs the push form.
// Stored z rows (PULL 1) while the M layers' rows fit comfortably in L2, recomputed
// (PULL 2) beyond.  Measured on B200 (DPA3 FP32, flushed L2, steps/s):
//              push (0)   stored z (1)   recomputed z (2)   DRAM/step (ncu, 0/1/2)
//   2PTC        6443        7483           7343             112.5 / 23.1 / 1.6 MB
//   2PTC x8     1114        1223           1451
//   2PTC x64     145         164            195
// HMDP_PULL=0|1|2 pins it (A/B experiments).
constexpr size_t kZRowsL2Budget = 48u << 20;  // bytes of stored z rows (126 MB L2)
template <typename T>
static int pull_mode(const DevGraph& gr, const DevWork<T>& ws, int n_msg) {
    static const int env = [] {
        const char* e = std::getenv("HMDP_PULL");
        const int v = e ? std::atoi(e) : -1;
        return (v >= 0 && v <= 2) ? v : -1;
    }();
    if (!gr.sym || gr.alist || gr.n_active != gr.n || ws.s_remote || ws.p_atom || !ws.vrow) return 0;
    if (env >= 0) return env;
    // ~32 neighbours per atom at the paper density
    const size_t zbytes = static_cast<size_t>(gr.n_active) * n_msg * 32 * kH * sizeof(T);
    return zbytes > kZRowsL2Budget ? 2 : 1;
}

// The network phases for one element type and team size (WIDE: the 28-warp-CTA
// build of the FP32 2-warp-team kernels, single-domain periodic path only).
template <typename T, int G, bool LIST = false, bool WIDE = false>
struct Net {
    static_assert(!WIDE || (G == 2 && sizeof(T) == 4), "WIDE: FP32 2-warp teams only");
    template <int PULL>
    static cudaError_t configure_p() {
        const cudaFuncAttribute a = cudaFuncAttributeMaxDynamicSharedMemorySize;
        cudaError_t e = cudaSuccess;
        for (cudaError_t r : {cudaFuncSetAttribute(k_msg_fwd<T, G, true, LIST, PULL, WIDE>, a, kMaxSmem),
                              cudaFuncSetAttribute(k_msg_fwd<T, G, false, LIST, PULL, WIDE>, a, kMaxSmem)})
            if (r != cudaSuccess) e = r;
        if constexpr (PULL == 0) {
            for (cudaError_t r : {cudaFuncSetAttribute(k_msg_bwd<T, G, LIST>, a, kMaxSmem),
                                  cudaFuncSetAttribute(k_embed_bwd<T, G, LIST>, a, kMaxSmem)})
                if (r != cudaSuccess) e = r;
        } else {
            for (cudaError_t r : {cudaFuncSetAttribute(k_msg_bwd_pull<T, G, PULL, WIDE>, a, kMaxSmem),
                                  cudaFuncSetAttribute(k_embed_bwd_pull<T, G, PULL, WIDE>, a, kMaxSmem)})
                if (r != cudaSuccess) e = r;
        }
        return e;
    }
    static cudaError_t configure() {
        const cudaFuncAttribute a = cudaFuncAttributeMaxDynamicSharedMemorySize;
        cudaError_t e = cudaSuccess;
        if constexpr (WIDE && LIST) {  // the halo-exchange DD's pull form, 28-warp CTAs
            for (cudaError_t r :
                 {cudaFuncSetAttribute(k_embed<T, G, false, true, false, true>, a, kMaxSmem),
                  cudaFuncSetAttribute(k_msg_fwd<T, G, true, true, 1, true>, a, kMaxSmem),
                  cudaFuncSetAttribute(k_msg_fwd<T, G, false, true, 1, true>, a, kMaxSmem),
                  cudaFuncSetAttribute(k_msg_bwd_pull<T, G, 1, true, 1>, a, kMaxSmem),
                  cudaFuncSetAttribute(k_msg_bwd_pull<T, G, 1, true, 2>, a, kMaxSmem),
                  cudaFuncSetAttribute(k_embed_bwd_pull<T, G, 1, true, 1>, a, kMaxSmem),
                  cudaFuncSetAttribute(k_embed_bwd_pull<T, G, 1, true, 2>, a, kMaxSmem)})
                if (r != cudaSuccess) e = r;
            return e;
        } else if constexpr (WIDE) {
            for (cudaError_t r : {cudaFuncSetAttribute(k_embed<T, G, true, false, false, true>, a, kMaxSmem),
                                  cudaFuncSetAttribute(k_embed<T, G, false, false, false, true>, a, kMaxSmem),
                                  configure_p<1>(), configure_p<2>()})
                if (r != cudaSuccess) e = r;
            return e;
        } else {
            for (cudaError_t r : {cudaFuncSetAttribute(k_embed<T, G, true, LIST>, a, kMaxSmem),
                                  cudaFuncSetAttribute(k_embed<T, G, false, LIST>, a, kMaxSmem),
                                  cudaFuncSetAttribute(k_embed<T, G, false, LIST, true>, a, kMaxSmem),
                                  configure_p<0>()})
                if (r != cudaSuccess) e = r;
            if constexpr (!LIST) {
                for (cudaError_t r : {configure_p<1>(), configure_p<2>()})
                    if (r != cudaSuccess) e = r;
            } else {  // the halo-exchange DD's pull form
                for (cudaError_t r :
                     {cudaFuncSetAttribute(k_msg_fwd<T, G, true, true, 1>, a, kMaxSmem),
                      cudaFuncSetAttribute(k_msg_fwd<T, G, false, true, 1>, a, kMaxSmem),
                      cudaFuncSetAttribute(k_msg_bwd_pull<T, G, 1, false, 1>, a, kMaxSmem),
                      cudaFuncSetAttribute(k_msg_bwd_pull<T, G, 1, false, 2>, a, kMaxSmem),
                      cudaFuncSetAttribute(k_embed_bwd_pull<T, G, 1, false, 1>, a, kMaxSmem),
                      cudaFuncSetAttribute(k_embed_bwd_pull<T, G, 1, false, 2>, a, kMaxSmem)})
                    if (r != cudaSuccess) e = r;
            }
            return e;
        }
    }
    // returns the kernels launched (2 with the tcgen05 embedding chain)
    static int embed(const NetShape& sh, const DevModel<T>& md, const DevGraph& gr,
                     const DevWork<T>& ws, int* rev, const MdFuse& mf, cudaStream_t st) {
        if (md.n_msg == 0) {
            launch_net<T>(k_embed<T, G, true, LIST, false, WIDE>, Phase::EmbedFit, sh, st, md, gr,
                          ws, rev, mf);
            return 1;
        }
        if constexpr (sizeof(T) == 4 && !LIST && !WIDE) {
            if (tc_embed_on(gr.n_active) && !ws.p_atom) {
                launch_net<T>(k_embed<T, G, false, LIST, true>, Phase::Embed, sh, st, md, gr, ws,
                              rev, mf);
                // desc (nd, zero-padded to 32) -> tanh(32) = ez1 -> h^0 -> P^0 = W1h h^0
                const TcLayer L[3] = {
                    {md.embed.W1, md.embed.b1, 32, 32, 32, 1, 0, ws.ez1, kH},
                    {md.embed.W2, md.embed.b2, 32, 32, 32, 0, 0, ws.h, kH},
                    {md.msg[0].W1, nullptr, 32, 32, kH + kK, 0, 0, ws.pa, kH}};
                launch_tc_chain(gr.n_active, ws.desc, 32, 3, L, st);
                return 2;
            }
        }
        launch_net<T>(k_embed<T, G, false, LIST, false, WIDE>, Phase::Embed, sh, st, md, gr, ws, rev,
                      mf);
        return 1;
    }
    template <int PULL>
    static void msg_fwd(const NetShape& sh, const DevModel<T>& md, const DevGraph& gr,
                        const DevWork<T>& ws, int l, cudaStream_t st) {
        if (l == md.n_msg - 1)
            launch_net<T>(k_msg_fwd<T, G, true, LIST, PULL, WIDE>, Phase::MsgFwdLast, sh, st, md, gr,
                          ws, l);
        else
            launch_net<T>(k_msg_fwd<T, G, false, LIST, PULL, WIDE>, Phase::MsgFwd, sh, st, md, gr, ws,
                          l);
    }
    template <int PULL>
    static void msg_bwd(const NetShape& sh, const DevModel<T>& md, const DevGraph& gr,
                        const DevWork<T>& ws, int l, cudaStream_t st) {
        if constexpr (PULL == 0)
            launch_net<T>(k_msg_bwd<T, G, LIST>, Phase::MsgBwd, sh, st, md, gr, ws, l);
        else
            launch_net<T>(k_msg_bwd_pull<T, G, PULL, WIDE>, Phase::MsgBwd, sh, st, md, gr, ws, l);
    }
    template <int PULL>
    static void embed_bwd(const NetShape& sh, const DevModel<T>& md, const DevGraph& gr,
                          const DevWork<T>& ws, cudaStream_t st) {
        if constexpr (PULL == 0)
            launch_net<T>(k_embed_bwd<T, G, LIST>, Phase::EmbedBwd, sh, st, md, gr, ws);
        else
            launch_net<T>(k_embed_bwd_pull<T, G, PULL, WIDE>, Phase::EmbedBwd, sh, st, md, gr, ws);
    }
    // One evaluation's network kernels.
    template <int PULL>
    static int network_p(const NetShape& sh, const DevModel<T>& md, const DevGraph& gr,
                         const DevWork<T>& ws, int* rev, cudaStream_t st, const Marker& mk,
                         const MdFuse& mf) {
        const int M = md.n_msg;
        const int ne = embed(sh, md, gr, ws, rev, mf, st);
        mk(M == 0 ? "embed_fit" : "embed", st);
        if (M == 0) return 1;
        for (int l = 0; l < M; ++l) {
            msg_fwd<PULL>(sh, md, gr, ws, l, st);
            mk(l == M - 1 ? "msg_fwd_last" : "msg_fwd", st);
        }
        for (int l = M - 2; l >= 0; --l) {
            msg_bwd<PULL>(sh, md, gr, ws, l, st);
            mk("msg_bwd", st);
        }
        embed_bwd<PULL>(sh, md, gr, ws, st);
        mk("embed_bwd", st);
        return ne + 1 + M + (M - 1);
    }
    static int network(const NetShape& sh, const DevModel<T>& md, const DevGraph& gr,
                       const DevWork<T>& ws, int* rev, cudaStream_t st, const Marker& mk,
                       const MdFuse& mf) {
        if constexpr (!LIST) {
            const int pull = pull_mode(gr, ws, md.n_msg);
            if (pull == 1) return network_p<1>(sh, md, gr, ws, rev, st, mk, mf);
            if (pull == 2) return network_p<2>(sh, md, gr, ws, rev, st, mk, mf);
        }
        if constexpr (WIDE)
            return -1;  // never: the WIDE build is chosen only on the pull-form path
        else
            return network_p<0>(sh, md, gr, ws, rev, st, mk, mf);
    }
    static void dd_phase(const NetShape& sh, const DevModel<T>& md, const DevGraph& gr,
                         const DevWork<T>& ws, int phase, int l, cudaStream_t st, int* rev) {
        const MdFuse none{};
        if (phase == 0) embed(sh, md, gr, ws, rev, none, st);
        if constexpr (!WIDE) {  // push form
            switch (phase) {
                case 2: msg_fwd<0>(sh, md, gr, ws, l, st); break;
                case 4: msg_bwd<0>(sh, md, gr, ws, l, st); break;
                case 5: embed_bwd<0>(sh, md, gr, ws, st); break;
            }
        }
        if constexpr (LIST) {  // halo-exchange DD, pull form (stored z)
            switch (phase) {
                case 12: msg_fwd<1>(sh, md, gr, ws, l, st); break;
                case 13:  // sender half of layer l's backward over the searched rows
                    if (l > 0)
                        launch_net<T>(k_msg_bwd_pull<T, G, 1, WIDE, 1>, Phase::MsgBwd, sh, st, md,
                                      gr, ws, l - 1);
                    else
                        launch_net<T>(k_embed_bwd_pull<T, G, 1, WIDE, 1>, Phase::EmbedBwd, sh, st,
                                      md, gr, ws);
                    break;
                case 14:  // layer l's update backward over the owned rows
                    launch_net<T>(k_msg_bwd_pull<T, G, 1, WIDE, 2>, Phase::MsgBwd, sh, st, md, gr,
                                  ws, l);
                    break;
                case 15:
                    launch_net<T>(k_embed_bwd_pull<T, G, 1, WIDE, 2>, Phase::EmbedBwd, sh, st, md,
                                  gr, ws);
                    break;
            }
        }
    }
};

// Per device: allow the staged-weight kernels > 48 KB of dynamic shared memory
// (set when a context is created, never during stream capture).
cudaError_t net_configure() {
    cudaError_t e = cudaSuccess;
    for (cudaError_t r : {Net<float, 1>::configure(), Net<float, 2>::configure(),
                          Net<float, 2, false, true>::configure(),
                          Net<float, 2, true, true>::configure(),
                          Net<float, 4>::configure(), Net<double, 1>::configure(),
                          Net<double, 2>::configure(), Net<double, 4>::configure(),
                          Net<float, 1, true>::configure(), Net<float, 2, true>::configure(),
                          Net<float, 4, true>::configure(), Net<double, 1, true>::configure(),
                          Net<double, 2, true>::configure(), Net<double, 4, true>::configure()})
        if (r != cudaSuccess) e = r;
    return e;
}

template <typename T>
int launch_network(const DevModel<T>& md, const DevGraph& gr, const DevWork<T>& ws,
                   double* forces, double* per_atom, double* out, int* rev, cudaStream_t st,
                   const Marker& mk, const MdFuse& mf) {
    // the WIDE build exists for the pull-form (single-domain periodic) path only
    const bool pull = !gr.alist && pull_mode(gr, ws, md.n_msg) != 0;
    const bool wide_ok = sizeof(T) == 4 && pull;
    const NetShape sh = net_shape(gr.n_active, md.n_msg, static_cast<int>(sizeof(T)), wide_ok,
                                  !pull && md.n_msg > 0);
    int launches;
    if constexpr (sizeof(T) == 4)
        if (sh.G == 2 && sh.wide) {
            launches = Net<T, 2, false, true>::network(sh, md, gr, ws, rev, st, mk, mf);
            launch_force_k<T>(gr, ws, forces, per_atom, out, st, mf);
            mk("force", st);
            return launches + 1;
        }
    if (sh.G == 4)
        launches = Net<T, 4>::network(sh, md, gr, ws, rev, st, mk, mf);
    else if (sh.G == 2)
        launches = Net<T, 2>::network(sh, md, gr, ws, rev, st, mk, mf);
    else
        launches = Net<T, 1>::network(sh, md, gr, ws, rev, st, mk, mf);
    DevWork<T> wf = ws;
    wf.gather_mirror_g = (md.n_msg == 0 && rev) ? 1 : 0;  // k_embed<FUSE_FIT> pushed no mirrors
    launch_force_k<T>(gr, wf, forces, per_atom, out, st, mf);
    mk("force", st);
    return launches + 1;
}

// Force kernel alone (the DeePMD-style families' last phase, hmdp_dp.cu).
template <typename T>
void launch_force(const DevGraph& gr, const DevWork<T>& ws, double* forces, double* per_atom,
                  double* out, cudaStream_t st, const MdFuse& mf) {
    launch_force_k<T>(gr, ws, forces, per_atom, out, st, mf);
}
template void launch_force<float>(const DevGraph&, const DevWork<float>&, double*, double*,
                                  double*, cudaStream_t, const MdFuse&);
template void launch_force<double>(const DevGraph&, const DevWork<double>&, double*, double*,
                                   double*, cudaStream_t, const MdFuse&);

// Device MD: (E, W, W_ab) of the last step from the force kernel's CTA partials.
void launch_reduce_partials(const double* partial, int n, double* out, cudaStream_t st) {
    k_reduce_partials<<<1, kForceCTA, 0, st>>>(partial, force_grid(n), out);
}

// One phase of a domain-decomposed evaluation (the caller exchanges halo rows
// between phases).  Phases: 0 embed, 1 ghost P rows (into layer `l`), 2 message
// layer l forward, 3 ghost adjoint sums of layer l, 4 message layer l backward,
// 5 embedding backward, 6 forces.
template <typename T>
void launch_dd_phase(const DevModel<T>& md, const DevGraph& gr, const DevWork<T>& ws, int phase,
                     int l, T* s_ghost, double* forces, double* out, cudaStream_t st, int* rev) {
    // the pull-form DD (ws.dd_role set) takes the pull form's CTA shapes, 28-warp included
    const NetShape sh = net_shape(gr.n_active, md.n_msg, static_cast<int>(sizeof(T)),
                                  ws.dd_role != nullptr, md.n_msg > 0 && !ws.dd_role);
    const int ng = gr.n - gr.n_active;
    switch (phase) {
        case 1:
            if (ng > 0)
                k_dd_ghost_p<T><<<(ng * 32 + 255) / 256, 256, 0, st>>>(
                    gr, ws.p_atom, ws.pa + static_cast<long long>(l) * gr.n * kH);
            break;
        case 3:
            if (ng > 0)
                k_dd_ghost_sums<T><<<(ng * 32 + 255) / 256, 256, 0, st>>>(
                    gr, ws.d + (l & 1) * ws.slots * kH, s_ghost);
            break;
        case 6:
            launch_force_k<T>(gr, ws, forces, static_cast<double*>(nullptr), out, st, MdFuse{});
            break;
        case 16: {  // pull form: each pair's terms sit at either end; gather the mirror g
            DevWork<T> wf = ws;
            wf.gather_mirror_g = 1;
            launch_force_k<T>(gr, wf, forces, static_cast<double*>(nullptr), out, st, MdFuse{},
                              true);
            break;
        }
        default:
            if (gr.alist) {  // global-index DD: the owned-atom list variants
                if constexpr (sizeof(T) == 4)
                    if (sh.wide) {
                        Net<T, 2, true, true>::dd_phase(sh, md, gr, ws, phase, l, st, rev);
                        break;
                    }
                if (sh.G == 4)
                    Net<T, 4, true>::dd_phase(sh, md, gr, ws, phase, l, st, rev);
                else if (sh.G == 2)
                    Net<T, 2, true>::dd_phase(sh, md, gr, ws, phase, l, st, rev);
                else
                    Net<T, 1, true>::dd_phase(sh, md, gr, ws, phase, l, st, rev);
            } else if (sh.G == 4)
                Net<T, 4>::dd_phase(sh, md, gr, ws, phase, l, st, rev);
            else if (sh.G == 2)
                Net<T, 2>::dd_phase(sh, md, gr, ws, phase, l, st, rev);
            else
                Net<T, 1>::dd_phase(sh, md, gr, ws, phase, l, st, rev);
    }
}
template void launch_dd_phase<float>(const DevModel<float>&, const DevGraph&,
                                     const DevWork<float>&, int, int, float*, double*, double*,
                                     cudaStream_t, int*);
template void launch_dd_phase<double>(const DevModel<double>&, const DevGraph&,
                                      const DevWork<double>&, int, int, double*, double*, double*,
                                      cudaStream_t, int*);
template int launch_network<float>(const DevModel<float>&, const DevGraph&, const DevWork<float>&,
                                   double*, double*, double*, int*, cudaStream_t, const Marker&,
                                   const MdFuse&);
template int launch_network<double>(const DevModel<double>&, const DevGraph&,
                                    const DevWork<double>&, double*, double*, double*, int*,
                                    cudaStream_t, const Marker&, const MdFuse&);

}  // namespace hmdp

#ifdef HMDP_TPROBE
extern "C" int hmdp_debug_tprobe(unsigned long long* out, int reset) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, hmdp::g_tprobe, sizeof(hmdp::g_tprobe));
    if (reset) {
        unsigned long long z[32] = {};
        cudaMemcpyToSymbol(hmdp::g_tprobe, z, sizeof(z));
    }
    return 0;
}
#endif
