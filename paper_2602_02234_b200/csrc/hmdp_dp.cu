// hmdp_dp.cu — DeePMD-style families (north-star ops with no reference
// function, SURVEY.md §8(a'); parity against the FP64 oracle oracle/dpfamily.py,
// "parity unpinned"): the smooth environment matrix, per-neighbour-type
// embedding nets with the G^T.R.R^T.G descriptor contraction (se_a), and the
// DPA2-style repformer stack with gated, smoothly switched neighbour
// self-attention.  Model definition: oracle/dpfamily.py and DESIGN.md §11.
//
// Decomposition: one warp per atom (the reference's per-atom loop,
// inference.cpp:183-416, is the same shape), 4 warps per CTA, grid-stride over
// atoms.  Two lane layouts, chosen per phase:
//   * lane = feature channel for atom-level vectors (descriptor, g1, MLPs):
//     weights read as coalesced 128-byte rows of the transposed matrix, inputs
//     broadcast by shuffle or shared memory;
//   * lane = edge row for per-neighbour work (embedding, q/k/v/o projections,
//     attention): the row lives in registers, weights are read at uniform
//     addresses (one broadcast transaction per load), the attention loops over
//     the atom's neighbours f with an online softmax (running max / sum), so
//     no n_nei x n_nei matrix is materialised.
// Everything an atom's edges need stays inside that atom's warp: the softmax,
// the attention backward (row pass over e, column pass over f), the dE/dw and
// dE/dh accumulators.  Cross-atom terms (the neighbour projection P_j in conv,
// its adjoint) are gathered by the consumer over the symmetric list's mirror
// slots (rev), so there are no float atomics and runs are deterministic.
//
// se_a (depth 1) is ONE kernel per atom plus the force kernel.  The embedding's
// output layer is linear, so the contraction R^T G is taken through it exactly:
//   A[c][b] = (1/N) sum_t ( sum_o W2_t[b][o] Z_t[c][o] + b2_t[b] Rsum_t[c] ),
//   Z_t[c][o] = sum_{e of type t} R_e[c] z_e[o],  z_e = tanh(w1_t s_e + b1_t),
// and backward V_t[c][o] = sum_b W2_t[b][o] dA[c][b] gives per edge
//   dR_e[c] = V_t[c] . z_e + b2_t . dA[c],  dz_e = (sum_c R_e[c] V_t[c]) (1 - z_e^2),
// so an edge costs one tanh and a few FMAs per lane instead of a 32x32 mat-vec.
//
// Geometry (edge e = i -> j, d = edge_dr, r = |d|, u = d / r):
//   R = (s, q d),  s = sw/r,  q = sw/r^2
//   dE/dd = (dE/ds) s' u + q dE/dR[1:4] + q' u (dE/dR[1:4] . d) + (dE/dw) sw' u
//   with s' = sw'/r - sw/r^2 and q' = sw'/r^2 - 2 sw/r^3; the vector goes to the
//   edge slot and its mirror, and k_force (hmdp_net.cu) gathers
//   F_i = sum_q (gv_q - gv_rev(q)), W_ab = -sum_q d_a gv_b.
#include <cstdlib>

#include <type_traits>

#include "hmdp_common.cuh"

namespace hmdp {

int num_sms();  // hmdp_nbr.cu
template <typename T>
void launch_force(const DevGraph&, const DevWork<T>&, double*, double*, double*, cudaStream_t,
                  const MdFuse&);

namespace {

constexpr int kDpWarps = 4;
constexpr int kDpCTA = 32 * kDpWarps;
constexpr double kShift = 20.0;  // smooth-softmax logit shift (oracle SHIFT)

template <typename T>
struct Env {
    T r, ux, uy, uz, sw, dsw, s;
};

// Smooth environment of one edge (DeePMD switch, oracle smooth_switch).
template <typename T>
__device__ __forceinline__ Env<T> dp_env(const double* d, T rc, T rcs) {
    Env<T> v;
    T x, y, z;
    v.r = edge_len<T>(d, x, y, z);
    v.ux = x / v.r;
    v.uy = y / v.r;
    v.uz = z / v.r;
    if (v.r < rcs) {
        v.sw = T(1);
        v.dsw = T(0);
    } else if (v.r < rc) {
        const T inv = T(1) / (rc - rcs);
        const T u = (v.r - rcs) * inv;
        const T u2 = u * u;
        v.sw = u2 * u * (T(-6) * u2 + T(15) * u - T(10)) + T(1);
        v.dsw = T(-30) * u2 * (u - T(1)) * (u - T(1)) * inv;
    } else {
        v.sw = T(0);
        v.dsw = T(0);
    }
    v.s = v.sw / v.r;
    return v;
}

// dE/d(edge_dr) from the adjoints of s (total), R[1:4] (dh) and w = sw.
template <typename T>
__device__ __forceinline__ void dp_gvec(const Env<T>& v, const double* d, T dEds, T dh0, T dh1,
                                        T dh2, T dEdw, T g[3]) {
    const T r = v.r, ir = T(1) / r;
    const T sp = v.dsw * ir - v.sw * ir * ir;            // s'
    const T q = v.sw * ir * ir;                           // q = sw / r^2
    const T qp = v.dsw * ir * ir - T(2) * v.sw * ir * ir * ir;  // q'
    const T dx = static_cast<T>(d[0]), dy = static_cast<T>(d[1]), dz = static_cast<T>(d[2]);
    const T dot = dh0 * dx + dh1 * dy + dh2 * dz;
    const T radial = dEds * sp + qp * dot + dEdw * v.dsw;
    g[0] = radial * v.ux + q * dh0;
    g[1] = radial * v.uy + q * dh1;
    g[2] = radial * v.uz + q * dh2;
}

template <typename T>
__device__ __forceinline__ T shfl(T v, int src) {
    return __shfl_sync(FULL_MASK, v, src);
}

// Lane = channel mat-vec, x distributed (lane k holds x_k): y_lane = b + sum_k WT[k][lane] x_k.
template <typename T>
__device__ __forceinline__ T cmv(const T* __restrict__ WT, const T* __restrict__ b, T x) {
    const int lane = threadIdx.x & 31;
    T acc = b ? __ldg(b + lane) : T(0);
#pragma unroll 8
    for (int k = 0; k < 32; ++k) acc += __ldg(WT + k * 32 + lane) * shfl(x, k);
    return acc;
}


// A (lane b holds A[c][b], c < 4) -> D[a][b] = sum_c A[c][a] A[c][b], a < 4.
template <typename T>
__device__ __forceinline__ void gram4(const T (&A)[4], T (&D)[4]) {
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        T v = T(0);
#pragma unroll
        for (int c = 0; c < 4; ++c) v += shfl(A[c], a) * A[c];
        D[a] = v;
    }
}
// Adjoint of gram4 over NC rows: dA[c][b] = sum_a dD[a][b] A[c][a] + [b < 4] sum_b' dD[b][b'] A[c][b'].
template <typename T, int NC>
__device__ __forceinline__ void gram4_bwd(const T (&A)[NC], const T (&dD)[4], T (&dA)[NC]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        T v = T(0);
#pragma unroll
        for (int a = 0; a < 4; ++a) v += dD[a] * shfl(A[c], a);
        dA[c] = v;
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const T x = warp_sum(dD[a] * A[c]);
            if (lane == a) dA[c] += x;
        }
}


struct DpWarpSmem {
    double s[32];
    double R[32][4];
    int t[32];
    double x[160];  // descriptor / MLP input staging
    double zs[kMaxTypes][4][32];
};

__device__ __forceinline__ void zero_cells(const MdFuse& mf) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < mf.n_cells_zero;
         c += gridDim.x * blockDim.x)
        mf.cell_count[c] = 0;
}

struct WarpIdx {
    int lane, wid, first, stride;
    __device__ WarpIdx()
        : lane(threadIdx.x & 31),
          wid(threadIdx.x >> 5),
          first(blockIdx.x * kDpWarps + (threadIdx.x >> 5)),
          stride(gridDim.x * kDpWarps) {}
};

// ---------------------------------------------------------------------------
// se_a: environment, embedding, G^T R R^T G, fitting, and the whole backward to
// per-edge dE/d(edge_dr), one warp per atom.
// ---------------------------------------------------------------------------
template <typename T>
__global__ __launch_bounds__(kDpCTA) void k_sea(DevDp<T> md, DevGraph gr, DevWork<T> ws,
                                                int* __restrict__ rev, MdFuse mf) {
    __shared__ DpWarpSmem s_w[kDpWarps];
    pdl_launch_dependents();
    const WarpIdx wi;
    const int lane = wi.lane;
    DpWarpSmem& sm = s_w[wi.wid];
    T w1[kMaxTypes], b1[kMaxTypes];
#pragma unroll
    for (int t = 0; t < kMaxTypes; ++t) {
        w1[t] = t < md.n_types ? md.emb_w1[t][lane] : T(0);
        b1[t] = t < md.n_types ? md.emb_b1[t][lane] : T(0);
    }
    const T fb1 = md.fit1.b[lane], fw2 = md.fit2.W[lane], fb2 = md.fit2.b[0];
    pdl_wait();
    zero_cells(mf);
    for (int i = wi.first; i < gr.n_active; i += wi.stride) {
        const int start = gr.row_start[i], cnt = gr.nnei[i];
        T Z[kMaxTypes][4], Rs[kMaxTypes][4];
#pragma unroll
        for (int t = 0; t < kMaxTypes; ++t)
#pragma unroll
            for (int c = 0; c < 4; ++c) Z[t][c] = Rs[t][c] = T(0);
        // pass 1: env (lane = edge) then Z_t, Rsum_t (lane = channel o)
        for (int base = 0; base < cnt; base += 32) {
            const int m = min(32, cnt - base);
            const int e = start + base + lane;
            int j = 0;
            if (lane < m) {
                j = gr.nbr[e];
                const Env<T> v = dp_env<T>(gr.dr + 3ll * e, md.rc, md.rcs);
                if (!(v.r > T(0))) atomicOr(ws.err, kErrZeroEdge);
                sm.s[lane] = v.s;
                sm.R[lane][0] = v.s;
                sm.R[lane][1] = v.s * v.ux;
                sm.R[lane][2] = v.s * v.uy;
                sm.R[lane][3] = v.s * v.uz;
                sm.t[lane] = gr.ety[e];
            }
            if (rev) {
                const int f = find_rev(i, j, m, gr);
                if (lane < m) {
                    rev[e] = f;
                    if (f < 0) atomicOr(ws.err, kErrAsymmetric);
                }
            }
            __syncwarp();
            for (int u = 0; u < m; ++u) {
                const int t = sm.t[u];
                const T s = static_cast<T>(sm.s[u]);
                const T R0 = static_cast<T>(sm.R[u][0]), R1 = static_cast<T>(sm.R[u][1]),
                        R2 = static_cast<T>(sm.R[u][2]), R3 = static_cast<T>(sm.R[u][3]);
#pragma unroll
                for (int tt = 0; tt < kMaxTypes; ++tt)
                    if (tt == t) {
                        const T z = d_tanh(w1[tt] * s + b1[tt]);
                        Z[tt][0] += R0 * z;
                        Z[tt][1] += R1 * z;
                        Z[tt][2] += R2 * z;
                        Z[tt][3] += R3 * z;
                        Rs[tt][0] += R0;
                        Rs[tt][1] += R1;
                        Rs[tt][2] += R2;
                        Rs[tt][3] += R3;
                    }
            }
            __syncwarp();
        }
        // A[c][b] (lane b)
#pragma unroll
        for (int t = 0; t < kMaxTypes; ++t)
#pragma unroll
            for (int c = 0; c < 4; ++c) sm.zs[t][c][lane] = Z[t][c];
        __syncwarp();
        T A[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
        for (int t = 0; t < kMaxTypes; ++t) {
            if (t >= md.n_types) break;
            const T* W2T = md.emb2[t].WT;
            for (int o = 0; o < 32; ++o) {
                const T w = __ldg(W2T + o * 32 + lane);
#pragma unroll
                for (int c = 0; c < 4; ++c) A[c] += w * static_cast<T>(sm.zs[t][c][o]);
            }
            const T bb = md.emb2[t].b[lane];
#pragma unroll
            for (int c = 0; c < 4; ++c) A[c] += bb * Rs[t][c];
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) A[c] *= md.inv_nnorm;
        T Dv[4];
        gram4(A, Dv);
        __syncwarp();
#pragma unroll
        for (int a = 0; a < 4; ++a) sm.x[a * 32 + lane] = Dv[a];
        __syncwarp();
        // fitting [128 -> 32 -> 1]
        T y = fb1;
        for (int k = 0; k < 128; ++k) y += __ldg(md.fit1.WT + k * 32 + lane) * static_cast<T>(sm.x[k]);
        y = d_tanh(y);
        const T e_i = warp_sum(fw2 * y);
        if (lane == 0) ws.e_atom[i] = static_cast<double>(e_i + fb2 + md.ebias[gr.types[i]]);
        const T dy = fw2 * (T(1) - y * y);
        T dD[4] = {T(0), T(0), T(0), T(0)};
        for (int o = 0; o < 32; ++o) {
            const T d_o = shfl(dy, o);
#pragma unroll
            for (int a = 0; a < 4; ++a) dD[a] += __ldg(md.fit1.W + o * 128 + a * 32 + lane) * d_o;
        }
        T dA[4];
        gram4_bwd<T, 4>(A, dD, dA);
#pragma unroll
        for (int c = 0; c < 4; ++c) dA[c] *= md.inv_nnorm;
        __syncwarp();
#pragma unroll
        for (int c = 0; c < 4; ++c) sm.zs[0][c][lane] = dA[c];
        __syncwarp();
        // V_t[c][o] = sum_b W2_t[b][o] dA[c][b] (lane o) into zs[t][c][o]; c0_t[c]
        T c0[kMaxTypes][4];
        T V[kMaxTypes][4];
#pragma unroll
        for (int t = 0; t < kMaxTypes; ++t) {
#pragma unroll
            for (int c = 0; c < 4; ++c) V[t][c] = c0[t][c] = T(0);
            if (t < md.n_types) {
                const T* W2 = md.emb2[t].W;
                for (int b = 0; b < 32; ++b) {
                    const T w = __ldg(W2 + b * 32 + lane);
#pragma unroll
                    for (int c = 0; c < 4; ++c) V[t][c] += w * static_cast<T>(sm.zs[0][c][b]);
                }
                const T bb = md.emb2[t].b[lane];
#pragma unroll
                for (int c = 0; c < 4; ++c) c0[t][c] = warp_sum(bb * dA[c]);
            }
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < kMaxTypes; ++t)
#pragma unroll
            for (int c = 0; c < 4; ++c) sm.zs[t][c][lane] = V[t][c];
        __syncwarp();
        // pass 2: per-edge adjoints -> dE/d(edge_dr), LANE = EDGE: each lane runs the
        // 32 channels of its own edge (no cross-lane reductions)
        //   z_o = tanh(w1_o s + b1_o), dR_c = sum_o V[c][o] z_o + c0[c],
        //   ds = sum_o w1_o (sum_c R_c V[c][o]) (1 - z_o^2)
        for (int base = 0; base < cnt; base += 32) {
            const int m = min(32, cnt - base);
            const int e = start + base + lane;
            Env<T> v{};
            T mdR[4] = {T(0), T(0), T(0), T(0)}, mds = T(0);
            if (lane < m) {
                v = dp_env<T>(gr.dr + 3ll * e, md.rc, md.rcs);
                const int t = gr.ety[e];
                const T sv = v.s, R1 = v.s * v.ux, R2 = v.s * v.uy, R3 = v.s * v.uz;
                const T* w1t = md.emb_w1[0];
                const T* b1t = md.emb_b1[0];
#pragma unroll
                for (int tt = 0; tt < kMaxTypes; ++tt)
                    if (tt == t) {
                        w1t = md.emb_w1[tt];
                        b1t = md.emb_b1[tt];
                        mdR[0] = c0[tt][0];
                        mdR[1] = c0[tt][1];
                        mdR[2] = c0[tt][2];
                        mdR[3] = c0[tt][3];
                    }
                const double* Vt = &sm.zs[t][0][0];
#pragma unroll 4
                for (int o = 0; o < 32; ++o) {
                    const T w = __ldg(w1t + o);
                    const T z = d_tanh(w * sv + __ldg(b1t + o));
                    const T v0 = static_cast<T>(Vt[o]), v1 = static_cast<T>(Vt[32 + o]),
                            v2 = static_cast<T>(Vt[64 + o]), v3 = static_cast<T>(Vt[96 + o]);
                    mdR[0] += v0 * z;
                    mdR[1] += v1 * z;
                    mdR[2] += v2 * z;
                    mdR[3] += v3 * z;
                    mds += w * (sv * v0 + R1 * v1 + R2 * v2 + R3 * v3) * (T(1) - z * z);
                }
            }
            if (lane < m) {
                T g[3];
                const double* d = gr.dr + 3ll * e;
                dp_gvec(v, d, mds + mdR[0], mdR[1], mdR[2], mdR[3], T(0), g);
                st4(ws.gv + 4ll * e, g[0], g[1], g[2], T(0));
                const int mir = rev ? rev[e] : gr.inv_pos[e];
                if (mir >= 0) st4(ws.gvrev + 4ll * mir, g[0], g[1], g[2], T(0));
            }
            __syncwarp();
        }
    }
}

// ---------------------------------------------------------------------------
// repformer: ONE ATOM PER CTA (a team of 4 warps, 128 threads), grid-stride.
//   * per-edge 32x32 projections (q, k, v, o and their transposes): warp w takes
//     the atom's edges q = w, w+4, ...; lane c keeps row c of the matrix in
//     registers and reads the edge's input row at a uniform address (broadcast);
//   * attention: a QUAD of lanes per edge row (lane 4r + p holds channels
//     8p..8p+7 of row r), 32 rows per pass; the q.k and do.v dot products are
//     8 FMAs + 2 quad shuffles; the loop over the atom's neighbours f keeps an
//     online softmax (running max / sum); the backward runs a row pass
//     (dq, row-side dw/dh) and a column pass (dk, dv, column-side dw/dh);
//   * atom-level vectors (conv, grrg, update MLP, fitting, g1 map) by warp 0
//     from per-warp partials summed in a fixed order in shared memory.
// ---------------------------------------------------------------------------
constexpr int kRfT = 128;
// Resident CTAs per SM the register budget targets for the lighter kernels (embed,
// forward layers, embed backward): 6 in FP32 (<= 80 registers, 24 warps per SM for
// these latency-bound atom teams), 2 in FP64.  The top / backward layer kernels keep
// the compiler's choice (128 registers): forcing 80 spills and measured slower.
template <typename T>
constexpr int kRfMinB = sizeof(T) == 4 ? 6 : 2;
constexpr double kInvSqrt32 = 0.17677669529663688;  // 1 / sqrt(32)

template <typename T>
struct RfSmem {
    T x[160];       // MLP input staging (warp 0)
    T red[4][128];  // per-warp partial sums
    T bc[128];      // values broadcast to the team (dconv + dT, dA)
    int alist[256];  // repflow: local rows of the angle neighbours (r < rca), ascending
    int na;
};

// repflow: the atom's angle-neighbour rows (omega > 0, i.e. r < rca) in ascending
// order, by warp 0 with a ballot per 32 rows.  Ends with a CTA barrier.
template <typename T>
__device__ __forceinline__ void rf_angle_list(const DevDpWork<T>& dw, int start, int cnt,
                                              RfSmem<T>& sm) {
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        int na = 0;
        for (int base = 0; base < cnt; base += 32) {
            const int r = base + lane;
            const bool in = r < cnt && dw.envA[8ll * (start + r)] > T(0);
            const unsigned b = __ballot_sync(FULL_MASK, in);
            if (in) sm.alist[na + __popc(b & ((1u << lane) - 1u))] = r;
            na += __popc(b);
        }
        if (lane == 0) sm.na = na;
    }
    __syncthreads();
}

// out_q = [res_q] + b + W x_q over the atom's cnt edge rows (warp w: q = w, w+4,
// ...), W [32][32] row-major (lane c holds row c); rows of 32 at `in + q*ld_in`,
// `out + q*ld_out` (local row index q; shared or global memory); ADD accumulates
// into out instead of a residual.  Two rows per iteration (loads in flight).
template <typename T, bool ADD>
__device__ __forceinline__ void proj_simt(const T* __restrict__ W, const T* __restrict__ b,
                                          const T* in, int ld_in, const T* res, int ld_res, T* out,
                                          int ld_out, int cnt) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    T wr[32];
#pragma unroll
    for (int k = 0; k < 32; k += 4) {
        const V4<T> v = ld4(W + lane * 32 + k);
        wr[k] = v.x;
        wr[k + 1] = v.y;
        wr[k + 2] = v.z;
        wr[k + 3] = v.w;
    }
    const T bb = b ? __ldg(b + lane) : T(0);
#pragma unroll 1
    for (int q = w; q < cnt; q += 8) {
        const bool two = q + 4 < cnt;
        const T* x = in + (long long)q * ld_in;
        const T* y = in + (long long)(two ? q + 4 : q) * ld_in;
        T a0 = bb, a1 = T(0), c0 = bb, c1 = T(0);
#pragma unroll
        for (int k = 0; k < 32; k += 8) {
            const V4<T> u = ld4c(x + k), v = ld4c(x + k + 4);
            const V4<T> u2 = ld4c(y + k), v2 = ld4c(y + k + 4);
            a0 += wr[k] * u.x + wr[k + 1] * u.y + wr[k + 2] * u.z + wr[k + 3] * u.w;
            a1 += wr[k + 4] * v.x + wr[k + 5] * v.y + wr[k + 6] * v.z + wr[k + 7] * v.w;
            c0 += wr[k] * u2.x + wr[k + 1] * u2.y + wr[k + 2] * u2.z + wr[k + 3] * u2.w;
            c1 += wr[k + 4] * v2.x + wr[k + 5] * v2.y + wr[k + 6] * v2.z + wr[k + 7] * v2.w;
        }
        T* o = out + (long long)q * ld_out + lane;
        if (ADD) *o += a0 + a1;
        else *o = (res ? res[(long long)q * ld_res + lane] : T(0)) + a0 + a1;
        if (two) {
            T* o2 = out + (long long)(q + 4) * ld_out + lane;
            if (ADD) *o2 += c0 + c1;
            else *o2 = (res ? res[(long long)(q + 4) * ld_res + lane] : T(0)) + c0 + c1;
        }
    }
}

// ---- tensor-core projection (FP32 path): mma.sync m16n8k8 TF32 with the 3-pass
// hi/lo split (x = hi + lo, x*y ~ hi*hi + hi*lo + lo*hi), which keeps FP32-level
// accuracy (single-pass TF32 fails the force tolerance).  Warp w
// owns output channels 8w..8w+7 for every 16-row tile of the atom's edge rows.
__device__ __forceinline__ void tf32_split(float x, uint32_t& hi, uint32_t& lo) {
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(x));
    const float r = x - __uint_as_float(hi);
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lo) : "f"(r));
}
__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
template <bool ADD>
__device__ __forceinline__ void proj_tc(const float* __restrict__ W, const float* __restrict__ b,
                                        const float* in, int ld_in, const float* res, int ld_res,
                                        float* out, int ld_out, int cnt) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    // B[k][n] = W[n][k] for this warp's 8 output channels, all four k-steps, split
    uint32_t bh[4][2], bl[4][2];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
        tf32_split(__ldg(W + (8 * w + g) * 32 + 8 * kk + t), bh[kk][0], bl[kk][0]);
        tf32_split(__ldg(W + (8 * w + g) * 32 + 8 * kk + t + 4), bh[kk][1], bl[kk][1]);
    }
    const int col = 8 * w + 2 * t;
    const float bias0 = b ? __ldg(b + col) : 0.f, bias1 = b ? __ldg(b + col + 1) : 0.f;
    for (int m0 = 0; m0 < cnt; m0 += 16) {
        const int r0 = m0 + g, r1 = r0 + 8;
        const bool v0 = r0 < cnt, v1 = r1 < cnt;
        const float* x0 = in + (long long)(v0 ? r0 : 0) * ld_in;
        const float* x1 = in + (long long)(v1 ? r1 : 0) * ld_in;
        float c[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            const int k0 = 8 * kk + t;
            const float a[4] = {v0 ? x0[k0] : 0.f, v1 ? x1[k0] : 0.f, v0 ? x0[k0 + 4] : 0.f,
                                v1 ? x1[k0 + 4] : 0.f};
            uint32_t ah[4], al[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) tf32_split(a[q], ah[q], al[q]);
            mma_tf32(c, al, bh[kk][0], bh[kk][1]);
            mma_tf32(c, ah, bl[kk][0], bl[kk][1]);
            mma_tf32(c, ah, bh[kk][0], bh[kk][1]);
        }
        if (v0) {
            float* o = out + (long long)r0 * ld_out + col;
            if (ADD) {
                o[0] += c[0];
                o[1] += c[1];
            } else {
                const float* rr = res ? res + (long long)r0 * ld_res + col : nullptr;
                o[0] = (rr ? rr[0] : 0.f) + bias0 + c[0];
                o[1] = (rr ? rr[1] : 0.f) + bias1 + c[1];
            }
        }
        if (v1) {
            float* o = out + (long long)r1 * ld_out + col;
            if (ADD) {
                o[0] += c[2];
                o[1] += c[3];
            } else {
                const float* rr = res ? res + (long long)r1 * ld_res + col : nullptr;
                o[0] = (rr ? rr[0] : 0.f) + bias0 + c[2];
                o[1] = (rr ? rr[1] : 0.f) + bias1 + c[3];
            }
        }
    }
}

// out_q = [res_q] + b + W x_q over the atom's edge rows: tensor cores (3xTF32) in
// FP32, SIMT in FP64 (the FP64 check mode).
template <typename T, bool ADD>
__device__ __forceinline__ void proj(const T* __restrict__ W, const T* __restrict__ b,
                                     const T* in, int ld_in, const T* res, int ld_res, T* out,
                                     int ld_out, int cnt) {
    if constexpr (sizeof(T) == 4)
        proj_tc<ADD>(W, b, in, ld_in, res, ld_res, out, ld_out, cnt);
    else
        proj_simt<T, ADD>(W, b, in, ld_in, res, ld_res, out, ld_out, cnt);
}

template <typename T>
__device__ __forceinline__ T quad_sum(T v) {
    v += __shfl_xor_sync(FULL_MASK, v, 1);
    return v + __shfl_xor_sync(FULL_MASK, v, 2);
}
template <typename T>
__device__ __forceinline__ void ld8(const T* p, T (&x)[8]) {
    const V4<T> a = ld4c(p), b = ld4c(p + 4);
    x[0] = a.x, x[1] = a.y, x[2] = a.z, x[3] = a.w, x[4] = b.x, x[5] = b.y, x[6] = b.z, x[7] = b.w;
}
template <typename T>
__device__ __forceinline__ void st8(T* p, const T (&x)[8]) {
    st4(p, x[0], x[1], x[2], x[3]);
    st4(p + 4, x[4], x[5], x[6], x[7]);
}
template <typename T>
__device__ __forceinline__ T dot8(const T (&a)[8], const T* p) {
    const V4<T> u = ld4c(p), v = ld4c(p + 4);
    return (a[0] * u.x + a[1] * u.y + a[2] * u.z + a[3] * u.w) +
           (a[4] * v.x + a[5] * v.y + a[6] * v.z + a[7] * v.w);
}

// Per-atom q/k/v and attention-output-adjoint rows: in the CTA's dynamic shared
// memory when the ELL capacity fits (kRfSmemRows rows: 64 x 128 values), else
// in the global per-slot scratch (capacity grown for dense clusters).
constexpr int kRfSmemRows = 64;
template <typename T>
__device__ __forceinline__ T* rf_smem_rows() {
    extern __shared__ __align__(16) unsigned char rf_dyn[];
    return reinterpret_cast<T*>(rf_dyn);
}
// SR (compile time, = DevDpWork::smem_rows): the shared-memory rows, so every access
// through these pointers compiles to LDS/STS instead of a generic load
template <typename T, bool SR>
__device__ __forceinline__ T* rf_rows_qkv(const DevDpWork<T>& dw, int start) {
    if constexpr (SR) return rf_smem_rows<T>();
    else return dw.qkv + 96ll * start;
}
template <typename T, bool SR>
__device__ __forceinline__ T* rf_rows_dob(const DevDpWork<T>& dw, int start) {
    if constexpr (SR) return rf_smem_rows<T>() + 96 * kRfSmemRows;
    else return dw.dob + 32ll * start;
}

// Per-edge env row: s, w, h0, h1 | h2, dsw, r, type.
template <typename T>
struct EnvRow {
    T s, w, h0, h1, h2;
};
template <typename T>
__device__ __forceinline__ EnvRow<T> env_row(const T* env, long long e) {
    const V4<T> a = ld4c(env + 8 * e);
    return {a.x, a.y, a.z, a.w, env[8 * e + 4]};
}

// embedding + descriptor + g1 map + P^0, one atom per CTA
template <typename T>
__global__ __launch_bounds__(kRfT, kRfMinB<T>) void k_rf_embed(DevDp<T> md, DevGraph gr, DevWork<T> ws,
                                                   DevDpWork<T> dw, int* __restrict__ rev,
                                                   MdFuse mf) {
    __shared__ RfSmem<T> sm;
    pdl_launch_dependents();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    T w1[kMaxTypes], b1[kMaxTypes], b2[kMaxTypes];
#pragma unroll
    for (int t = 0; t < kMaxTypes; ++t) {
        w1[t] = t < md.n_types ? md.emb_w1[t][lane] : T(0);
        b1[t] = t < md.n_types ? md.emb_b1[t][lane] : T(0);
        b2[t] = t < md.n_types ? md.emb2[t].b[lane] : T(0);
    }
    pdl_wait();
    zero_cells(mf);
    for (int i = blockIdx.x; i < gr.n_active; i += gridDim.x) {
        const int start = gr.row_start[i], cnt = gr.nnei[i];
        // env rows + mirror slots (warp w: edge chunks 32 w + 128 k)
        for (int base = 32 * w; base < cnt; base += kRfT) {
            const int m = min(32, cnt - base);
            const int e = start + base + lane;
            int j = 0;
            if (lane < m) {
                j = gr.nbr[e];
                const Env<T> v = dp_env<T>(gr.dr + 3ll * e, md.rc, md.rcs);
                if (!(v.r > T(0))) atomicOr(ws.err, kErrZeroEdge);
                T* en = dw.env + 8ll * e;
                st4(en, v.s, v.sw, v.s * v.ux, v.s * v.uy);
                st4(en + 4, v.s * v.uz, v.dsw, v.r, static_cast<T>(gr.ety[e]));
                if (md.family == kRepflow) {  // angle switch omega(r) on [rcas, rca)
                    const Env<T> a = dp_env<T>(gr.dr + 3ll * e, md.rca, md.rcas);
                    T* ea = dw.envA + 8ll * e;
                    st4(ea, a.sw, a.dsw, v.ux, v.uy);
                    st4(ea + 4, v.uz, T(0), T(0), T(0));
                }
            }
            if (rev) {
                const int f = find_rev(i, j, m, gr);
                if (lane < m) {
                    rev[e] = f;
                    if (f < 0) atomicOr(ws.err, kErrAsymmetric);
                }
            }
        }
        __syncthreads();
        // embedding G_e (lane = channel) and R^T G partials
        T A[4] = {T(0), T(0), T(0), T(0)};
        for (int q = w; q < cnt; q += 4) {
            const long long e = start + q;
            const V4<T> a = ld4c(dw.env + 8 * e), b = ld4c(dw.env + 8 * e + 4);
            const int t = static_cast<int>(b.w);
            T z = T(0), bb = T(0);
            const T* W2T = md.emb2[0].WT;
#pragma unroll
            for (int tt = 0; tt < kMaxTypes; ++tt)
                if (tt == t) {
                    z = d_tanh(w1[tt] * a.x + b1[tt]);
                    bb = b2[tt];
                    W2T = md.emb2[tt].WT;
                }
            T G0 = bb, G1 = T(0);
#pragma unroll 8
            for (int o = 0; o < 32; o += 2) {
                G0 += __ldg(W2T + o * 32 + lane) * shfl(z, o);
                G1 += __ldg(W2T + (o + 1) * 32 + lane) * shfl(z, o + 1);
            }
            const T G = G0 + G1;
            dw.g2[32 * e + lane] = G;
            A[0] += a.x * G;
            A[1] += a.z * G;
            A[2] += a.w * G;
            A[3] += b.x * G;
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) sm.red[w][32 * c + lane] = A[c];
        __syncthreads();
        if (w == 0) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                A[c] = ((sm.red[0][32 * c + lane] + sm.red[1][32 * c + lane]) +
                        sm.red[2][32 * c + lane]) + sm.red[3][32 * c + lane];
                A[c] *= md.inv_nnorm;
                dw.A[128ll * i + 32 * c + lane] = A[c];
            }
            T Dv[4];
            gram4(A, Dv);
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                sm.x[a * 32 + lane] = Dv[a];
                dw.D[128ll * i + 32 * a + lane] = Dv[a];
            }
            __syncwarp();
            T m0 = md.map1.b[lane], m1 = T(0);
            for (int k = 0; k < 128; k += 2) {
                m0 += __ldg(md.map1.WT + k * 32 + lane) * sm.x[k];
                m1 += __ldg(md.map1.WT + (k + 1) * 32 + lane) * sm.x[k + 1];
            }
            const T mz = d_tanh(m0 + m1);
            const T g1 = cmv(md.map2.WT, md.map2.b, mz);
            dw.mz[32ll * i + lane] = mz;
            dw.g1[32ll * i + lane] = g1;
            dw.P[32ll * i + lane] = cmv(md.L[0].c.WT, md.L[0].c.b, g1);
        }
        __syncthreads();
    }
}

// Gated, switched neighbour self-attention of one atom (forward), a quad per
// row: o_e = sum_f softmax_f(l_ef) w_e w_f (h_e . h_f) v_f into TMP rows; the
// row max / normaliser go to dw.stat for the backward.
template <typename T>
__device__ __forceinline__ void rf_attn_fwd(const DevDp<T>& md, const DevDpLayer<T>& L, const DevDpWork<T>& dw,
                            T* Q, T* TMP, long long S, int l, int start, int cnt) {
    proj<T, false>(L.q.W, L.q.b, dw.g2 + (long long)l * S * 32 + 32ll * start, 32, nullptr, 0, Q,
                   96, cnt);
    proj<T, false>(L.k.W, L.k.b, dw.g2 + (long long)l * S * 32 + 32ll * start, 32, nullptr, 0,
                   Q + 32, 96, cnt);
    proj<T, false>(L.v.W, L.v.b, dw.g2 + (long long)l * S * 32 + 32ll * start, 32, nullptr, 0,
                   Q + 64, 96, cnt);
    __syncthreads();
    const T sh = static_cast<T>(kShift), isq = static_cast<T>(kInvSqrt32);
    const int rq = threadIdx.x >> 2, p = threadIdx.x & 3;
    for (int rb = 0; rb < cnt; rb += 32) {
        const int r = rb + rq;
        const bool valid = r < cnt;
        const long long e = start + (valid ? r : 0);
        T q[8], o[8];
        ld8(Q + 96 * (valid ? r : 0) + 8 * p, q);
        const EnvRow<T> er = env_row(dw.env, e);
#pragma unroll
        for (int c = 0; c < 8; ++c) o[c] = T(0);
        T mx = T(-1e30), Z = T(0);
#pragma unroll 2
        for (int f = 0; f < cnt; ++f) {
            const long long ef = start + f;
            const T lam = quad_sum(dot8(q, Q + 96 * f + 32 + 8 * p)) * isq;
            const EnvRow<T> fr = env_row(dw.env, ef);
            const T ww = er.w * fr.w;
            const T gam = er.h0 * fr.h0 + er.h1 * fr.h1 + er.h2 * fr.h2;
            const T lt = (lam + sh) * ww - sh;
            if (lt > mx) {
                const T sc = d_exp(mx - lt);
                Z *= sc;
#pragma unroll
                for (int c = 0; c < 8; ++c) o[c] *= sc;
                mx = lt;
            }
            const T pe = d_exp(lt - mx);
            Z += pe;
            const T coef = pe * ww * gam;
            T v[8];
            ld8(Q + 96 * f + 64 + 8 * p, v);
#pragma unroll
            for (int c = 0; c < 8; ++c) o[c] += coef * v[c];
        }
        if (valid) {
            const T iz = T(1) / Z;
#pragma unroll
            for (int c = 0; c < 8; ++c) o[c] *= iz;
            st8(TMP + 96 * r + 8 * p, o);
            if (p == 0) {
                T* st = dw.stat + ((long long)l * S + e) * 2;
                st[0] = mx;
                st[1] = Z;
            }
        }
    }
}

// repflow edge/angle message of one atom (forward), a quad per row:
// m_e = (1/anorm) sum_{f in A(i), f != e} omega_e omega_f tanh(aw c_ef + ab) * v_f
// into TMP rows (zero for rows outside A(i)).  v rows are in Q + 64.
template <typename T>
__device__ __forceinline__ void rf_angle_fwd(const DevDp<T>& md, const DevDpLayer<T>& L, const DevDpWork<T>& dw,
                             const T* Q, T* TMP, int start, int cnt, const RfSmem<T>& sm) {
    const int rq = threadIdx.x >> 2, p = threadIdx.x & 3;
    T aw[8], ab[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        aw[c] = L.aw[8 * p + c];
        ab[c] = L.ab[8 * p + c];
    }
    const int na = sm.na;
    for (int rb = 0; rb < cnt; rb += 32) {
        const int r = rb + rq;
        if (r >= cnt) continue;
        const V4<T> ea = ld4c(dw.envA + 8ll * (start + r));
        T m[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) m[c] = T(0);
        if (ea.x > T(0)) {
            const T ux = ea.z, uy = ea.w, uz = dw.envA[8ll * (start + r) + 4];
            for (int a = 0; a < na; ++a) {
                const int f = sm.alist[a];
                if (f == r) continue;
                const V4<T> fa = ld4c(dw.envA + 8ll * (start + f));
                const T cs = ux * fa.z + uy * fa.w + uz * dw.envA[8ll * (start + f) + 4];
                const T coef = ea.x * fa.x * md.inv_anorm;
                T v[8];
                ld8(Q + 96 * f + 64 + 8 * p, v);
#pragma unroll
                for (int c = 0; c < 8; ++c) m[c] += coef * d_tanh(aw[c] * cs + ab[c]) * v[c];
            }
        }
        st8(TMP + 96 * r + 8 * p, m);
    }
}

// Layer l forward for the CTA's atom i; returns g1^{l+1}_i in warp 0 (lane = channel).
template <typename T, bool SR>
__device__ __forceinline__ T rf_layer_fwd(const DevDp<T>& md, const DevGraph& gr, const DevDpWork<T>& dw,
                          long long S, int n, int l, int i, RfSmem<T>& sm) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const DevDpLayer<T>& L = md.L[l];
    const int start = gr.row_start[i], cnt = gr.nnei[i];
    const T* g2l = dw.g2 + (long long)l * S * 32;
    T* g2n = dw.g2 + (long long)(l + 1) * S * 32;
    T* Q = rf_rows_qkv<T, SR>(dw, start);
    T* TMP = dw.tmp + 96ll * start;
    if (md.family == kRepflow) {
        proj<T, false>(L.v.W, L.v.b, g2l + 32ll * start, 32, nullptr, 0, Q + 64, 96, cnt);
        rf_angle_list(dw, start, cnt, sm);
        rf_angle_fwd(md, L, dw, Q, TMP, start, cnt, sm);
    } else {
        rf_attn_fwd(md, L, dw, Q, TMP, S, l, start, cnt);
    }
    __syncthreads();
    // g2hat = g2 + Wo o + bo
    proj<T, false>(L.o.W, L.o.b, TMP, 96, g2l + 32ll * start, 32, g2n + 32ll * start, 32, cnt);
    __syncthreads();
    // conv and T partials (lane = channel), summed over warps in a fixed order
    const T* Pl = dw.P + (long long)l * n * 32;
    T conv = T(0), T3[3] = {T(0), T(0), T(0)};
    for (int q2 = w; q2 < cnt; q2 += 4) {
        const long long e = start + q2;
        const T gh = g2n[32 * e + lane];
        const T pj = Pl[32ll * gr.nbr[e] + lane];
        const EnvRow<T> er = env_row(dw.env, e);
        conv += er.w * gh * pj;
        T3[0] += er.h0 * gh;
        T3[1] += er.h1 * gh;
        T3[2] += er.h2 * gh;
    }
    sm.red[w][lane] = conv;
#pragma unroll
    for (int c = 0; c < 3; ++c) sm.red[w][32 + 32 * c + lane] = T3[c];
    __syncthreads();
    T g1 = T(0);
    if (w == 0) {
        auto tot = [&](int k) {
            return ((sm.red[0][k] + sm.red[1][k]) + sm.red[2][k]) + sm.red[3][k];
        };
        conv = tot(lane) * md.inv_nnorm;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            T3[c] = tot(32 + 32 * c + lane) * md.inv_nnorm;
            dw.Ts[((long long)l * n + i) * 96 + 32 * c + lane] = T3[c];
        }
        T gr4[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            T v = T(0);
#pragma unroll
            for (int c = 0; c < 3; ++c) v += shfl(T3[c], a) * T3[c];
            gr4[a] = v;
        }
        sm.x[lane] = conv;
#pragma unroll
        for (int a = 0; a < 4; ++a) sm.x[32 + 32 * a + lane] = gr4[a];
        __syncwarp();
        T u0 = L.u1.b[lane], u1 = T(0);
        for (int k = 0; k < 160; k += 2) {
            u0 += __ldg(L.u1.WT + k * 32 + lane) * sm.x[k];
            u1 += __ldg(L.u1.WT + (k + 1) * 32 + lane) * sm.x[k + 1];
        }
        const T uz = d_tanh(u0 + u1);
        dw.uz[((long long)l * n + i) * 32 + lane] = uz;
        g1 = dw.g1[((long long)l * n + i) * 32 + lane] + cmv(L.u2.WT, L.u2.b, uz);
        dw.g1[((long long)(l + 1) * n + i) * 32 + lane] = g1;
    }
    return g1;
}

// Attention backward of one atom: q/k/v recomputed, do = Wo^T dg2hat, row pass
// (S_e, dq_e, row-side dw/dh), column pass (dk_f, dv_f, column-side dw/dh), then
// dg2 = dg2hat + Wq^T dq + Wk^T dk + Wv^T dv.
template <typename T>
__device__ __forceinline__ void rf_attn_bwd(const DevDp<T>& md, const DevDpLayer<T>& L, const DevDpWork<T>& dw,
                            const T* g2l, T* Q, T* DOB, T* TMP, T* DG2, long long S, int l,
                            int start, int cnt, bool have_qkv) {
    // q, k, v (recomputed unless the forward of this layer just left them in Q)
    // and do = Wo^T dg2hat
    if (!have_qkv) {
        proj<T, false>(L.q.W, L.q.b, g2l + 32ll * start, 32, nullptr, 0, Q, 96, cnt);
        proj<T, false>(L.k.W, L.k.b, g2l + 32ll * start, 32, nullptr, 0, Q + 32, 96, cnt);
        proj<T, false>(L.v.W, L.v.b, g2l + 32ll * start, 32, nullptr, 0, Q + 64, 96, cnt);
    }
    proj<T, false>(L.o.WT, nullptr, DG2, 32, nullptr, 0, DOB, 32, cnt);
    __syncthreads();
    const T sh = static_cast<T>(kShift), isq = static_cast<T>(kInvSqrt32);
    const int rq = threadIdx.x >> 2, p = threadIdx.x & 3;
    // row pass (quad per row e): S_e, dq_e, row-side dw/dh
    for (int rb = 0; rb < cnt; rb += 32) {
        const int r = rb + rq;
        const bool valid = r < cnt;
        const long long e = start + (valid ? r : 0);
        T q[8], dov[8];
        ld8(Q + 96 * (valid ? r : 0) + 8 * p, q);
        ld8(DOB + 32 * (valid ? r : 0) + 8 * p, dov);
        const T* st = dw.stat + ((long long)l * S + e) * 2;
        const T mx = st[0], iz = T(1) / st[1];
        const EnvRow<T> er = env_row(dw.env, e);
        // one pass: with dlt_ef = a_ef (da_ef - S_e), every S_e-dependent sum splits
        // into two S_e-free sums combined after the loop
        //   dq_e  = isq (sum a da ww k_f - S_e sum a ww k_f)
        //   dw_e += sum db a gam w_f + sum a da (lam+sh) w_f - S_e sum a (lam+sh) w_f
        T Ssum = T(0), k1[8], k2[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) k1[c] = k2[c] = T(0);
        T dwe = T(0), dwa = T(0), dwb = T(0), dh0 = T(0), dh1 = T(0), dh2 = T(0);
#pragma unroll 2
        for (int f = 0; f < cnt; ++f) {
            const long long ef = start + f;
            const T* kf = Q + 96 * f + 32 + 8 * p;
            const T lam = quad_sum(dot8(q, kf)) * isq;
            const T db = quad_sum(dot8(dov, Q + 96 * f + 64 + 8 * p));
            const EnvRow<T> fr = env_row(dw.env, ef);
            const T ww = er.w * fr.w;
            const T gam = er.h0 * fr.h0 + er.h1 * fr.h1 + er.h2 * fr.h2;
            const T al = d_exp((lam + sh) * ww - sh - mx) * iz;
            const T da = db * ww * gam;
            Ssum += al * da;
            const T aw = al * ww, ada = aw * da;
            T k[8];
            ld8(kf, k);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                k1[c] += ada * k[c];
                k2[c] += aw * k[c];
            }
            const T lw = (lam + sh) * fr.w;
            dwe += db * al * gam * fr.w;
            dwa += al * da * lw;
            dwb += al * lw;
            const T dgam = db * aw;
            dh0 += dgam * fr.h0;
            dh1 += dgam * fr.h1;
            dh2 += dgam * fr.h2;
        }
        T dq[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) dq[c] = isq * (k1[c] - Ssum * k2[c]);
        dwe += dwa - Ssum * dwb;
        if (valid) {
            st8(TMP + 96 * r + 8 * p, dq);
            if (p == 0) {
                dw.aux[2 * e] = Ssum;
                T* pw = dw.dwh + 4 * e;
                const V4<T> old = ld4c(pw);
                st4(pw, old.x + dwe, old.y + dh0, old.z + dh1, old.w + dh2);
            }
        }
    }
    __syncthreads();
    // column pass (quad per column f): dk_f, dv_f, column-side dw/dh
    for (int rb = 0; rb < cnt; rb += 32) {
        const int r = rb + rq;
        const bool valid = r < cnt;
        const long long f = start + (valid ? r : 0);
        T k[8], v[8], dk[8], dv[8];
        const int rl = valid ? r : 0;
        ld8(Q + 96 * rl + 32 + 8 * p, k);
        ld8(Q + 96 * rl + 64 + 8 * p, v);
#pragma unroll
        for (int c = 0; c < 8; ++c) dk[c] = dv[c] = T(0);
        const EnvRow<T> fr = env_row(dw.env, f);
        T dwf = T(0), dh0 = T(0), dh1 = T(0), dh2 = T(0);
#pragma unroll 2
        for (int r2 = 0; r2 < cnt; ++r2) {
            const long long e = start + r2;
            const T* qe = Q + 96 * r2 + 8 * p;
            const T* de = DOB + 32 * r2 + 8 * p;
            const T lam = quad_sum(dot8(k, qe)) * isq;
            const T db = quad_sum(dot8(v, de));
            const EnvRow<T> er = env_row(dw.env, e);
            const T ww = er.w * fr.w;
            const T gam = er.h0 * fr.h0 + er.h1 * fr.h1 + er.h2 * fr.h2;
            const T* st = dw.stat + ((long long)l * S + e) * 2;
            const T al = d_exp((lam + sh) * ww - sh - st[0]) / st[1];
            const T da = db * ww * gam;
            const T dlt = al * (da - dw.aux[2 * e]);
            const T dlam = dlt * ww * isq;
            const T bet = al * ww * gam;
            T qv[8], dv8[8];
            ld8(qe, qv);
            ld8(de, dv8);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                dk[c] += dlam * qv[c];
                dv[c] += bet * dv8[c];
            }
            const T dww = db * al * gam + dlt * (lam + sh);
            const T dgam = db * al * ww;
            dwf += dww * er.w;
            dh0 += dgam * er.h0;
            dh1 += dgam * er.h1;
            dh2 += dgam * er.h2;
        }
        if (valid) {
            st8(TMP + 96 * r + 32 + 8 * p, dk);
            st8(TMP + 96 * r + 64 + 8 * p, dv);
            if (p == 0) {
                T* pw = dw.dwh + 4 * f;
                const V4<T> old = ld4c(pw);
                st4(pw, old.x + dwf, old.y + dh0, old.z + dh1, old.w + dh2);
            }
        }
    }
    __syncthreads();
    // dg2 = dg2hat + Wq^T dq + Wk^T dk + Wv^T dv
    proj<T, true>(L.q.WT, nullptr, TMP, 96, nullptr, 0, DG2, 32, cnt);
    proj<T, true>(L.k.WT, nullptr, TMP + 32, 96, nullptr, 0, DG2, 32, cnt);
    proj<T, true>(L.v.WT, nullptr, TMP + 64, 96, nullptr, 0, DG2, 32, cnt);
    __syncthreads();
}

// repflow angle-message backward of one atom (v rows in Q + 64, dm = Wo^T dg2hat
// rows in DOB), one pass over rows e (a quad per row) that also takes the terms
// of every m_f that depend on row e (c_ef = c_fe, v_e):
//   dv_e  = sum_f coef z_ef dm_f,                coef = omega_e omega_f / anorm
//   dE/dc = coef sum_c (dm_e v_f + dm_f v_e) (1 - z^2) aw   -> dE/du_e += dE/dc u_f
//   dE/domega_e = sum_f omega_f / anorm sum_c (dm_e v_f + dm_f v_e) z
// dv rows go to TMP + 64 (zero outside A(i)); (domega, du) accumulate into dua.
template <typename T>
__device__ __forceinline__ void rf_angle_bwd(const DevDp<T>& md, const DevDpLayer<T>& L, const DevDpWork<T>& dw,
                             const T* Q, const T* DOB, T* TMP, int start, int cnt, bool top,
                             const RfSmem<T>& sm) {
    const int rq = threadIdx.x >> 2, p = threadIdx.x & 3;
    T aw[8], ab[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        aw[c] = L.aw[8 * p + c];
        ab[c] = L.ab[8 * p + c];
    }
    const int na = sm.na;
    for (int rb = 0; rb < cnt; rb += 32) {
        const int r = rb + rq;
        const bool valid = r < cnt;
        const int rl = valid ? r : 0;
        const long long e = start + rl;
        const V4<T> ea = ld4c(dw.envA + 8 * e);
        const T ux = ea.z, uy = ea.w, uz = dw.envA[8 * e + 4];
        T dv[8], ve[8], dme[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) dv[c] = T(0);
        ld8(Q + 96 * rl + 64 + 8 * p, ve);
        ld8(DOB + 32 * rl + 8 * p, dme);
        T dom = T(0), du0 = T(0), du1 = T(0), du2 = T(0);
        if (valid && ea.x > T(0)) {
            for (int a = 0; a < na; ++a) {
                const int f = sm.alist[a];
                if (f == r) continue;
                const V4<T> fa = ld4c(dw.envA + 8ll * (start + f));
                const T fz = dw.envA[8ll * (start + f) + 4];
                const T cs = ux * fa.z + uy * fa.w + uz * fz;
                const T coef = ea.x * fa.x * md.inv_anorm;
                T vf[8], dmf[8];
                ld8(Q + 96 * f + 64 + 8 * p, vf);
                ld8(DOB + 32 * f + 8 * p, dmf);
                T sdc = T(0), sz = T(0);
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const T z = d_tanh(aw[c] * cs + ab[c]);
                    const T t = dme[c] * vf[c] + dmf[c] * ve[c];
                    sdc += t * (T(1) - z * z) * aw[c];
                    sz += t * z;
                    dv[c] += coef * z * dmf[c];
                }
                const T dc = coef * sdc;
                du0 += dc * fa.z;
                du1 += dc * fa.w;
                du2 += dc * fz;
                dom += fa.x * md.inv_anorm * sz;
            }
        }
        dom = quad_sum(dom);
        du0 = quad_sum(du0);
        du1 = quad_sum(du1);
        du2 = quad_sum(du2);
        if (valid) {
            st8(TMP + 96 * r + 64 + 8 * p, dv);
            if (p == 0) {
                T* pa = dw.dua + 4 * e;
                if (top) {
                    st4(pa, dom, du0, du1, du2);
                } else {
                    const V4<T> old = ld4c(pa);
                    st4(pa, old.x + dom, old.y + du0, old.z + du1, old.w + du2);
                }
            }
        }
    }
}

// Layer l backward for the CTA's atom i.  dg1_out (warp 0, lane = channel): the
// adjoint of g1^{l+1}_i.  top: no g2 adjoint from above.  Writes dconv (scaled by
// 1/nnorm) for the neighbours' P gather, the residual part of dg1^l (dw.dg1),
// dg2 (adjoint of g2^l), and accumulates dwh.
template <typename T, bool SR>
__device__ __forceinline__ void rf_layer_bwd(const DevDp<T>& md, const DevGraph& gr, const DevDpWork<T>& dw,
                             long long S, int n, int l, int i, T dg1_out, bool top,
                             RfSmem<T>& sm) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const DevDpLayer<T>& L = md.L[l];
    const int start = gr.row_start[i], cnt = gr.nnei[i];
    const T* g2l = dw.g2 + (long long)l * S * 32;
    const T* g2n = dw.g2 + (long long)(l + 1) * S * 32;
    if (w == 0) {
        // update MLP backward -> dconv, dgrrg -> dT
        const T uz = dw.uz[((long long)l * n + i) * 32 + lane];
        T du = T(0);
#pragma unroll 8
        for (int c = 0; c < 32; ++c) du += __ldg(L.u2.W + c * 32 + lane) * shfl(dg1_out, c);
        du *= (T(1) - uz * uz);
        T dx[5] = {T(0), T(0), T(0), T(0), T(0)};
        for (int o = 0; o < 32; ++o) {
            const T d_o = shfl(du, o);
#pragma unroll
            for (int jj = 0; jj < 5; ++jj) dx[jj] += __ldg(L.u1.W + o * 160 + 32 * jj + lane) * d_o;
        }
        const T dconv = dx[0] * md.inv_nnorm;
        T T3[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) T3[c] = dw.Ts[((long long)l * n + i) * 96 + 32 * c + lane];
        const T dgr[4] = {dx[1], dx[2], dx[3], dx[4]};
        T dT[3];
        gram4_bwd<T, 3>(T3, dgr, dT);
        sm.bc[lane] = dconv;
#pragma unroll
        for (int c = 0; c < 3; ++c) sm.bc[32 + 32 * c + lane] = dT[c] * md.inv_nnorm;
        dw.dconv[((long long)(l & 1) * n + i) * 32 + lane] = dconv;
        dw.dg1[32ll * i + lane] = dg1_out;
    }
    __syncthreads();
    // per-edge adjoints of g2hat (lane = channel)
    {
        const T dconv = sm.bc[lane], dT0 = sm.bc[32 + lane], dT1 = sm.bc[64 + lane],
                dT2 = sm.bc[96 + lane];
        const T* Pl = dw.P + (long long)l * n * 32;
        for (int q = w; q < cnt; q += 4) {
            const long long e = start + q;
            const T gh = g2n[32 * e + lane];
            const T pj = Pl[32ll * gr.nbr[e] + lane];
            const EnvRow<T> er = env_row(dw.env, e);
            T d = top ? T(0) : dw.dg2[32 * e + lane];
            d += er.w * dconv * pj + er.h0 * dT0 + er.h1 * dT1 + er.h2 * dT2;
            dw.dg2[32 * e + lane] = d;
            const T a0 = warp_sum(dconv * gh * pj);
            const T a1 = warp_sum(dT0 * gh);
            const T a2 = warp_sum(dT1 * gh);
            const T a3 = warp_sum(dT2 * gh);
            if (lane == 0) {
                T* pw = dw.dwh + 4 * e;
                if (top) {
                    st4(pw, a0, a1, a2, a3);
                } else {
                    const V4<T> old = ld4c(pw);
                    st4(pw, old.x + a0, old.y + a1, old.z + a2, old.w + a3);
                }
            }
        }
    }
    __syncthreads();
    T* Q = rf_rows_qkv<T, SR>(dw, start);
    T* DOB = rf_rows_dob<T, SR>(dw, start);
    T* TMP = dw.tmp + 96ll * start;
    T* DG2 = dw.dg2 + 32ll * start;
    if (md.family == kRepflow) {
        if (!top)  // the top kernel's forward left v in Q + 64 (and the angle list)
            proj<T, false>(L.v.W, L.v.b, g2l + 32ll * start, 32, nullptr, 0, Q + 64, 96, cnt);
        proj<T, false>(L.o.WT, nullptr, DG2, 32, nullptr, 0, DOB, 32, cnt);
        if (!top) rf_angle_list(dw, start, cnt, sm);
        else __syncthreads();
        rf_angle_bwd(md, L, dw, Q, DOB, TMP, start, cnt, top, sm);
        __syncthreads();
        proj<T, true>(L.v.WT, nullptr, TMP + 64, 96, nullptr, 0, DG2, 32, cnt);
        __syncthreads();
    } else {
        rf_attn_bwd(md, L, dw, g2l, Q, DOB, TMP, DG2, S, l, start, cnt, top);
    }
}

// dg1^l_j = dg1(residual) + Wc^T dP_j with dP_j = sum_{q in out(j)} w_q g2hat^l_{rev q}
// * dconv^l_{nbr q}; per-warp partials, warp 0 returns the result (lane = channel).
template <typename T>
__device__ __forceinline__ T rf_gather_dg1(const DevDp<T>& md, const DevGraph& gr,
                                           const DevDpWork<T>& dw, long long S, int n, int l,
                                           int j, RfSmem<T>& sm) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int start = gr.row_start[j], cnt = gr.nnei[j];
    const T* g2n = dw.g2 + (long long)(l + 1) * S * 32;
    const T* dcv = dw.dconv + (long long)(l & 1) * n * 32;
    T dP = T(0);
    for (int q = w; q < cnt; q += 4) {
        const long long e = start + q;
        const long long mir = gr.inv_pos[e];
        dP += dw.env[8 * mir + 1] * g2n[32 * mir + lane] * dcv[32ll * gr.nbr[e] + lane];
    }
    sm.red[w][lane] = dP;
    __syncthreads();
    T acc = T(0);
    if (w == 0) {
        dP = ((sm.red[0][lane] + sm.red[1][lane]) + sm.red[2][lane]) + sm.red[3][lane];
        acc = dw.dg1[32ll * j + lane];
#pragma unroll 8
        for (int k = 0; k < 32; ++k) acc += __ldg(md.L[l].c.W + k * 32 + lane) * shfl(dP, k);
    }
    __syncthreads();
    return acc;
}

template <typename T>
__device__ __forceinline__ T rf_fit(const DevDp<T>& md, const DevGraph& gr, const DevWork<T>& ws,
                                    int i, T g1) {
    const int lane = threadIdx.x & 31;
    const T y = d_tanh(cmv(md.fit1.WT, md.fit1.b, g1));
    const T fw2 = md.fit2.W[lane];
    const T e = warp_sum(fw2 * y);
    if (lane == 0) ws.e_atom[i] = static_cast<double>(e + md.fit2.b[0] + md.ebias[gr.types[i]]);
    const T dy = fw2 * (T(1) - y * y);
    T dg = T(0);
#pragma unroll 8
    for (int o = 0; o < 32; ++o) dg += __ldg(md.fit1.W + o * 32 + lane) * shfl(dy, o);
    return dg;
}

// Layer l forward (l < L - 1): g1^{l+1}, P^{l+1}.
template <typename T, bool SR>
__global__ __launch_bounds__(kRfT, kRfMinB<T>) void k_rf_fwd(DevDp<T> md, DevGraph gr, DevWork<T> ws,
                                                 DevDpWork<T> dw, int l) {
    __shared__ RfSmem<T> sm;
    pdl_launch_dependents();
    pdl_wait();
    const int n = gr.n;
    for (int i = blockIdx.x; i < gr.n_active; i += gridDim.x) {
        const T g1 = rf_layer_fwd<T, SR>(md, gr, dw, ws.slots, n, l, i, sm);
        if (threadIdx.x < 32)
            dw.P[((long long)(l + 1) * n + i) * 32 + threadIdx.x] =
                cmv(md.L[l + 1].c.WT, md.L[l + 1].c.b, g1);
        __syncthreads();
    }
}

// Top layer forward + fitting + top layer backward (atom-local part).
template <typename T, bool SR>
__global__ __launch_bounds__(kRfT) void k_rf_top(DevDp<T> md, DevGraph gr, DevWork<T> ws,
                                                 DevDpWork<T> dw) {
    __shared__ RfSmem<T> sm;
    pdl_launch_dependents();
    pdl_wait();
    const int n = gr.n, l = md.n_layers - 1;
    for (int i = blockIdx.x; i < gr.n_active; i += gridDim.x) {
        const T g1 = rf_layer_fwd<T, SR>(md, gr, dw, ws.slots, n, l, i, sm);
        T dg1 = T(0);
        if (threadIdx.x < 32) dg1 = rf_fit(md, gr, ws, i, g1);
        rf_layer_bwd<T, SR>(md, gr, dw, ws.slots, n, l, i, dg1, true, sm);
    }
}

// Gather for layer l + 1, then layer l backward.
template <typename T, bool SR>
__global__ __launch_bounds__(kRfT) void k_rf_bwd(DevDp<T> md, DevGraph gr, DevWork<T> ws,
                                                 DevDpWork<T> dw, int l) {
    __shared__ RfSmem<T> sm;
    pdl_launch_dependents();
    pdl_wait();
    const int n = gr.n;
    for (int i = blockIdx.x; i < gr.n_active; i += gridDim.x) {
        const T dg1 = rf_gather_dg1(md, gr, dw, ws.slots, n, l + 1, i, sm);
        rf_layer_bwd<T, SR>(md, gr, dw, ws.slots, n, l, i, dg1, false, sm);
    }
}

// Gather for layer 0, g1 map + descriptor + embedding backward -> dE/d(edge_dr).
template <typename T>
__global__ __launch_bounds__(kRfT, kRfMinB<T>) void k_rf_embed_bwd(DevDp<T> md, DevGraph gr, DevWork<T> ws,
                                                       DevDpWork<T> dw) {
    __shared__ RfSmem<T> sm;
    pdl_launch_dependents();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    T w1[kMaxTypes], b1[kMaxTypes];
#pragma unroll
    for (int t = 0; t < kMaxTypes; ++t) {
        w1[t] = t < md.n_types ? md.emb_w1[t][lane] : T(0);
        b1[t] = t < md.n_types ? md.emb_b1[t][lane] : T(0);
    }
    pdl_wait();
    const int n = gr.n;
    for (int i = blockIdx.x; i < gr.n_active; i += gridDim.x) {
        const int start = gr.row_start[i], cnt = gr.nnei[i];
        const T dg1 = rf_gather_dg1(md, gr, dw, ws.slots, n, 0, i, sm);
        if (w == 0) {
            // g1 map backward -> dD -> dA (broadcast to the team)
            const T mz = dw.mz[32ll * i + lane];
            T dm = T(0);
#pragma unroll 8
            for (int c = 0; c < 32; ++c) dm += __ldg(md.map2.W + c * 32 + lane) * shfl(dg1, c);
            dm *= (T(1) - mz * mz);
            T dD[4] = {T(0), T(0), T(0), T(0)};
            for (int o = 0; o < 32; ++o) {
                const T d_o = shfl(dm, o);
#pragma unroll
                for (int a = 0; a < 4; ++a) dD[a] += __ldg(md.map1.W + o * 128 + a * 32 + lane) * d_o;
            }
            T A[4], dA[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) A[c] = dw.A[128ll * i + 32 * c + lane];
            gram4_bwd<T, 4>(A, dD, dA);
#pragma unroll
            for (int c = 0; c < 4; ++c) sm.bc[32 * c + lane] = dA[c] * md.inv_nnorm;
        }
        __syncthreads();
        const T dA0 = sm.bc[lane], dA1 = sm.bc[32 + lane], dA2 = sm.bc[64 + lane],
                dA3 = sm.bc[96 + lane];
        for (int q = w; q < cnt; q += 4) {
            const long long e = start + q;
            const V4<T> a = ld4c(dw.env + 8 * e), b = ld4c(dw.env + 8 * e + 4);
            const T s = a.x;
            const int t = static_cast<int>(b.w);
            const T G = dw.g2[32 * e + lane];
            const T dG = dw.dg2[32 * e + lane] + dA0 * s + dA1 * a.z + dA2 * a.w + dA3 * b.x;
            const T dR0 = warp_sum(dA0 * G), dR1 = warp_sum(dA1 * G), dR2 = warp_sum(dA2 * G),
                    dR3 = warp_sum(dA3 * G);
            T ds = T(0);
#pragma unroll
            for (int tt = 0; tt < kMaxTypes; ++tt)
                if (tt == t) {
                    const T z = d_tanh(w1[tt] * s + b1[tt]);
                    T dz0 = T(0), dz1 = T(0);
#pragma unroll 8
                    for (int bq = 0; bq < 32; bq += 2) {
                        dz0 += __ldg(md.emb2[tt].W + bq * 32 + lane) * shfl(dG, bq);
                        dz1 += __ldg(md.emb2[tt].W + (bq + 1) * 32 + lane) * shfl(dG, bq + 1);
                    }
                    ds = warp_sum(w1[tt] * (dz0 + dz1) * (T(1) - z * z));
                }
            if (lane == 0) {
                const V4<T> wh = ld4c(dw.dwh + 4 * e);
                const double* d = gr.dr + 3ll * e;
                const Env<T> v = dp_env<T>(d, md.rc, md.rcs);
                T g[3];
                dp_gvec(v, d, ds + dR0, dR1 + wh.y, dR2 + wh.z, dR3 + wh.w, wh.x, g);
                if (md.family == kRepflow) {
                    // omega(r) and u = d / r:  + dE/domega omega' u + (du - (du.u) u) / r
                    const V4<T> ea = ld4c(dw.envA + 8 * e), da = ld4c(dw.dua + 4 * e);
                    const T dot = da.y * v.ux + da.z * v.uy + da.w * v.uz;
                    const T rad = da.x * ea.y - dot / v.r;
                    const T ir = T(1) / v.r;
                    g[0] += rad * v.ux + da.y * ir;
                    g[1] += rad * v.uy + da.z * ir;
                    g[2] += rad * v.uz + da.w * ir;
                }
                st4(ws.gv + 4 * e, g[0], g[1], g[2], T(0));
                st4(ws.gvrev + 4ll * gr.inv_pos[e], g[0], g[1], g[2], T(0));
            }
        }
        __syncthreads();
    }
}

template <typename T>
cudaError_t rf_configure() {
    const cudaFuncAttribute a = cudaFuncAttributeMaxDynamicSharedMemorySize;
    const int bytes = kRfSmemRows * 128 * sizeof(T);
    cudaError_t e = cudaSuccess;
    for (cudaError_t r : {cudaFuncSetAttribute(k_rf_fwd<T, true>, a, bytes),
                          cudaFuncSetAttribute(k_rf_top<T, true>, a, bytes),
                          cudaFuncSetAttribute(k_rf_bwd<T, true>, a, bytes)})
        if (r != cudaSuccess) e = r;
    return e;
}

int dp_grid(int n) {  // one warp per atom (se_a)
    const int want = (n + kDpWarps - 1) / kDpWarps;
    const int cap = num_sms() * 8;
    return want < 1 ? 1 : (want < cap ? want : cap);
}

int rf_grid(int n) {  // one atom per CTA; as many CTAs as fit (the scheduler queues the rest)
    const int cap = num_sms() * 16;
    return n < 1 ? 1 : (n < cap ? n : cap);
}


}  // namespace

// Per device: allow the repformer kernels their shared-memory rows (FP64 > 48 KB).
cudaError_t dp_configure() {
    const cudaError_t a = rf_configure<float>(), b = rf_configure<double>();
    return a != cudaSuccess ? a : b;
}

// Launches the whole DeePMD-style network + forces; returns the kernel count.
template <typename T>
int launch_dp(const DevDp<T>& md, const DevGraph& gr, const DevWork<T>& ws,
              const DevDpWork<T>& dw, double* forces, double* per_atom, double* out, int* rev,
              cudaStream_t st, const Marker& mk, const MdFuse& mf) {
    const dim3 block(kDpCTA);
    if (md.family == kSeA) {
        launch_pdl(k_sea<T>, dim3(dp_grid(gr.n_active)), block, 0, st, md, gr, ws, rev, mf);
        mk("sea", st);
        launch_force<T>(gr, ws, forces, per_atom, out, st, mf);
        mk("force", st);
        return 2;
    }
    // rev is computed by k_rf_embed; the later kernels read it as gr.inv_pos
    DevGraph g2 = gr;
    if (rev) g2.inv_pos = rev;
    const int L = md.n_layers;
    const dim3 rgrid(rf_grid(gr.n_active)), rblock(kRfT);
    DevDpWork<T> dws = dw;
    dws.smem_rows = gr.ell > 0 && gr.ell <= kRfSmemRows;
    const size_t rsm = dws.smem_rows ? size_t(kRfSmemRows) * 128 * sizeof(T) : 0;
    launch_pdl(k_rf_embed<T>, rgrid, rblock, 0, st, md, gr, ws, dw, rev, mf);
    mk("rf_embed", st);
    auto layers = [&](auto sr) {
        constexpr bool SR = decltype(sr)::value;
        for (int l = 0; l + 1 < L; ++l) {
            launch_pdl(k_rf_fwd<T, SR>, rgrid, rblock, rsm, st, md, g2, ws, dws, l);
            mk("rf_fwd", st);
        }
        launch_pdl(k_rf_top<T, SR>, rgrid, rblock, rsm, st, md, g2, ws, dws);
        mk("rf_top", st);
        for (int l = L - 2; l >= 0; --l) {
            launch_pdl(k_rf_bwd<T, SR>, rgrid, rblock, rsm, st, md, g2, ws, dws, l);
            mk("rf_bwd", st);
        }
    };
    if (dws.smem_rows)
        layers(std::true_type{});
    else
        layers(std::false_type{});
    launch_pdl(k_rf_embed_bwd<T>, rgrid, rblock, 0, st, md, g2, ws, dw);
    mk("rf_embed_bwd", st);
    launch_force<T>(g2, ws, forces, per_atom, out, st, mf);
    mk("force", st);
    return 2 * L + 2;
}

template int launch_dp<float>(const DevDp<float>&, const DevGraph&, const DevWork<float>&,
                              const DevDpWork<float>&, double*, double*, double*, int*,
                              cudaStream_t, const Marker&, const MdFuse&);
template int launch_dp<double>(const DevDp<double>&, const DevGraph&, const DevWork<double>&,
                               const DevDpWork<double>&, double*, double*, double*, int*,
                               cudaStream_t, const Marker&, const MdFuse&);

}  // namespace hmdp
