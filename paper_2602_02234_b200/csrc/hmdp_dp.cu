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

// rev(e) for the lanes' edges (lane l < m holds edge (i -> j_l)): the slot of i
// in nbr(j_l), found with 8 neighbour-list rows in flight per lane and a ballot;
// lists longer than 32 fall back to a binary search (lists are sorted).
__device__ __forceinline__ int find_rev(int i, int j, int m, const DevGraph& gr) {
    const int lane = threadIdx.x & 31;
    const int rs_l = lane < m ? gr.row_start[j] : 0;
    const int nn_l = lane < m ? gr.nnei[j] : 0;
    int found = -1;
    for (int q0 = 0; q0 < m; q0 += 8) {
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
    if (lane < m && found < 0 && nn_l > 32) {
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
    return found;
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
// Lane = channel mat-vec with x in shared memory (nin inputs, WT [nin][32]).
template <typename T>
__device__ __forceinline__ T cmv_s(const T* __restrict__ WT, const T* __restrict__ b,
                                   const T* xs, int nin) {
    const int lane = threadIdx.x & 31;
    T acc = b ? __ldg(b + lane) : T(0);
#pragma unroll 8
    for (int k = 0; k < nin; ++k) acc += __ldg(WT + k * 32 + lane) * xs[k];
    return acc;
}

// Lane = row mat-vec: y = W x (+ b), W [32][32] row-major read at uniform
// addresses (broadcast), x and y in registers.
template <typename T>
__device__ __forceinline__ void rmv(const T* __restrict__ W, const T* __restrict__ b,
                                    const T (&x)[32], T (&y)[32]) {
#pragma unroll
    for (int c = 0; c < 32; ++c) {
        T acc = b ? __ldg(b + c) : T(0);
#pragma unroll
        for (int k = 0; k < 32; k += 4) {
            const V4<T> w = ld4(W + c * 32 + k);
            acc += w.x * x[k] + w.y * x[k + 1] + w.z * x[k + 2] + w.w * x[k + 3];
        }
        y[c] = acc;
    }
}
template <typename T>
__device__ __forceinline__ void load_row(const T* p, T (&x)[32]) {  // coherent (same-kernel data)
#pragma unroll
    for (int k = 0; k < 32; k += 4) {
        const V4<T> v = ld4c(p + k);
        x[k] = v.x;
        x[k + 1] = v.y;
        x[k + 2] = v.z;
        x[k + 3] = v.w;
    }
}
template <typename T>
__device__ __forceinline__ void store_row(T* p, const T (&x)[32]) {
#pragma unroll
    for (int k = 0; k < 32; k += 4) st4(p + k, x[k], x[k + 1], x[k + 2], x[k + 3]);
}
template <typename T>
__device__ __forceinline__ T dot32(const T (&a)[32], const T* p) {  // a . row p (coherent)
    T acc = T(0);
#pragma unroll
    for (int k = 0; k < 32; k += 4) {
        const V4<T> v = ld4c(p + k);
        acc += a[k] * v.x + a[k + 1] * v.y + a[k + 2] * v.z + a[k + 3] * v.w;
    }
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
        T V[kMaxTypes][4], c0[kMaxTypes][4];
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
        // pass 2: per-edge adjoints -> dE/d(edge_dr)
        for (int base = 0; base < cnt; base += 32) {
            const int m = min(32, cnt - base);
            const int e = start + base + lane;
            Env<T> v{};
            if (lane < m) {
                v = dp_env<T>(gr.dr + 3ll * e, md.rc, md.rcs);
                sm.s[lane] = v.s;
                sm.R[lane][0] = v.s;
                sm.R[lane][1] = v.s * v.ux;
                sm.R[lane][2] = v.s * v.uy;
                sm.R[lane][3] = v.s * v.uz;
                sm.t[lane] = gr.ety[e];
            }
            __syncwarp();
            T mdR[4] = {T(0), T(0), T(0), T(0)}, mds = T(0);
            for (int u = 0; u < m; ++u) {
                const int t = sm.t[u];
                const T s = static_cast<T>(sm.s[u]);
                const T R0 = static_cast<T>(sm.R[u][0]), R1 = static_cast<T>(sm.R[u][1]),
                        R2 = static_cast<T>(sm.R[u][2]), R3 = static_cast<T>(sm.R[u][3]);
#pragma unroll
                for (int tt = 0; tt < kMaxTypes; ++tt)
                    if (tt == t) {
                        const T z = d_tanh(w1[tt] * s + b1[tt]);
                        const T dz = (R0 * V[tt][0] + R1 * V[tt][1] + R2 * V[tt][2] + R3 * V[tt][3]) *
                                     (T(1) - z * z);
                        const T p0 = warp_sum(V[tt][0] * z) + c0[tt][0];
                        const T p1 = warp_sum(V[tt][1] * z) + c0[tt][1];
                        const T p2 = warp_sum(V[tt][2] * z) + c0[tt][2];
                        const T p3 = warp_sum(V[tt][3] * z) + c0[tt][3];
                        const T ds = warp_sum(w1[tt] * dz);
                        if (lane == u) {
                            mdR[0] = p0;
                            mdR[1] = p1;
                            mdR[2] = p2;
                            mdR[3] = p3;
                            mds = ds;
                        }
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
// repformer: embedding + descriptor + g1 map + P^0 (one warp per atom).
// ---------------------------------------------------------------------------
template <typename T>
__global__ __launch_bounds__(kDpCTA) void k_rf_embed(DevDp<T> md, DevGraph gr, DevWork<T> ws,
                                                     DevDpWork<T> dw, int* __restrict__ rev,
                                                     MdFuse mf) {
    __shared__ DpWarpSmem s_w[kDpWarps];
    pdl_launch_dependents();
    const WarpIdx wi;
    const int lane = wi.lane;
    DpWarpSmem& sm = s_w[wi.wid];
    T w1[kMaxTypes], b1[kMaxTypes], b2[kMaxTypes];
#pragma unroll
    for (int t = 0; t < kMaxTypes; ++t) {
        w1[t] = t < md.n_types ? md.emb_w1[t][lane] : T(0);
        b1[t] = t < md.n_types ? md.emb_b1[t][lane] : T(0);
        b2[t] = t < md.n_types ? md.emb2[t].b[lane] : T(0);
    }
    const long long S = ws.slots;
    pdl_wait();
    zero_cells(mf);
    for (int i = wi.first; i < gr.n_active; i += wi.stride) {
        const int start = gr.row_start[i], cnt = gr.nnei[i];
        T A[4] = {T(0), T(0), T(0), T(0)};
        for (int base = 0; base < cnt; base += 32) {
            const int m = min(32, cnt - base);
            const int e = start + base + lane;
            int j = 0;
            if (lane < m) {
                j = gr.nbr[e];
                const Env<T> v = dp_env<T>(gr.dr + 3ll * e, md.rc, md.rcs);
                if (!(v.r > T(0))) atomicOr(ws.err, kErrZeroEdge);
                const int t = gr.ety[e];
                sm.s[lane] = v.s;
                sm.R[lane][0] = v.s;
                sm.R[lane][1] = v.s * v.ux;
                sm.R[lane][2] = v.s * v.uy;
                sm.R[lane][3] = v.s * v.uz;
                sm.t[lane] = t;
                T* en = dw.env + 8ll * e;
                st4(en, v.s, v.sw, v.s * v.ux, v.s * v.uy);
                st4(en + 4, v.s * v.uz, v.dsw, v.r, static_cast<T>(t));
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
                T z = T(0), bb = T(0);
                const T* W2T = md.emb2[0].WT;
#pragma unroll
                for (int tt = 0; tt < kMaxTypes; ++tt)
                    if (tt == t) {
                        z = d_tanh(w1[tt] * s + b1[tt]);
                        bb = b2[tt];
                        W2T = md.emb2[tt].WT;
                    }
                T G = bb;
#pragma unroll 8
                for (int o = 0; o < 32; ++o) G += __ldg(W2T + o * 32 + lane) * shfl(z, o);
                dw.g2[(long long)(start + base + u) * 32 + lane] = G;
#pragma unroll
                for (int c = 0; c < 4; ++c) A[c] += static_cast<T>(sm.R[u][c]) * G;
            }
            __syncwarp();
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
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
        T xs_t = T(0);
        (void)xs_t;
        // g1 map [128 -> 32 -> 32]
        T mz = md.map1.b[lane];
        for (int k = 0; k < 128; ++k) mz += __ldg(md.map1.WT + k * 32 + lane) * static_cast<T>(sm.x[k]);
        mz = d_tanh(mz);
        const T g1 = cmv(md.map2.WT, md.map2.b, mz);
        dw.mz[32ll * i + lane] = mz;
        dw.g1[32ll * i + lane] = g1;
        dw.P[32ll * i + lane] = cmv(md.L[0].c.WT, md.L[0].c.b, g1);
        __syncwarp();
    }
    (void)S;
}

// ---------------------------------------------------------------------------
// repformer layer pieces (device functions, one warp per atom i)
// ---------------------------------------------------------------------------
constexpr double kInvSqrt32 = 0.17677669529663688;  // 1 / sqrt(32)

// q, k, v of every edge of atom i from g2^l (lane = row).
template <typename T>
__device__ __forceinline__ void rf_qkv(const DevDpLayer<T>& L, const T* g2l, T* qkv, int start,
                                       int cnt) {
    const int lane = threadIdx.x & 31;
    for (int rb = 0; rb < cnt; rb += 32) {
        if (rb + lane < cnt) {
            const long long e = start + rb + lane;
            T x[32], y[32];
            load_row(g2l + 32 * e, x);
            rmv(L.q.W, L.q.b, x, y);
            store_row(qkv + 96 * e, y);
            rmv(L.k.W, L.k.b, x, y);
            store_row(qkv + 96 * e + 32, y);
            rmv(L.v.W, L.v.b, x, y);
            store_row(qkv + 96 * e + 64, y);
        }
    }
    __syncwarp();
}

// Layer l forward for atom i: attention (lane = row), conv / grrg / update
// (lane = channel).  Returns g1^{l+1}_i (lane = channel).
template <typename T>
__device__ T rf_layer_fwd(const DevDp<T>& md, const DevGraph& gr, const DevDpWork<T>& dw,
                          long long S, int n, int l, int i, DpWarpSmem& sm) {
    const int lane = threadIdx.x & 31;
    const DevDpLayer<T>& L = md.L[l];
    const int start = gr.row_start[i], cnt = gr.nnei[i];
    const T* g2l = dw.g2 + (long long)l * S * 32;
    T* g2n = dw.g2 + (long long)(l + 1) * S * 32;
    rf_qkv(L, g2l, dw.qkv, start, cnt);
    const T sh = static_cast<T>(kShift), isq = static_cast<T>(kInvSqrt32);
    for (int rb = 0; rb < cnt; rb += 32) {
        const bool valid = rb + lane < cnt;
        const long long e = start + rb + (valid ? lane : 0);
        T q[32], o[32];
        load_row(dw.qkv + 96 * e, q);
        const V4<T> en0 = ld4c(dw.env + 8 * e), en1 = ld4c(dw.env + 8 * e + 4);
        const T we = en0.y, he0 = en0.z, he1 = en0.w, he2 = en1.x;
#pragma unroll
        for (int c = 0; c < 32; ++c) o[c] = T(0);
        T mx = T(-1e30), Z = T(0);
        for (int f = 0; f < cnt; ++f) {
            const long long ef = start + f;
            const T lam = dot32(q, dw.qkv + 96 * ef + 32) * isq;
            const V4<T> fn0 = ld4c(dw.env + 8 * ef), fn1 = ld4c(dw.env + 8 * ef + 4);
            const T ww = we * fn0.y;
            const T gam = he0 * fn0.z + he1 * fn0.w + he2 * fn1.x;
            const T lt = (lam + sh) * ww - sh;
            if (lt > mx) {
                const T sc = d_exp(mx - lt);
                Z *= sc;
#pragma unroll
                for (int c = 0; c < 32; ++c) o[c] *= sc;
                mx = lt;
            }
            const T p = d_exp(lt - mx);
            Z += p;
            const T coef = p * ww * gam;
            const T* vf = dw.qkv + 96 * ef + 64;
#pragma unroll
            for (int c = 0; c < 32; c += 4) {
                const V4<T> vv = ld4c(vf + c);
                o[c] += coef * vv.x;
                o[c + 1] += coef * vv.y;
                o[c + 2] += coef * vv.z;
                o[c + 3] += coef * vv.w;
            }
        }
        if (valid) {
            const T iz = T(1) / Z;
#pragma unroll
            for (int c = 0; c < 32; ++c) o[c] *= iz;
            T g[32], y[32];
            load_row(g2l + 32 * e, g);
            rmv(L.o.W, L.o.b, o, y);
#pragma unroll
            for (int c = 0; c < 32; ++c) y[c] += g[c];
            store_row(g2n + 32 * e, y);
            T* st = dw.stat + ((long long)l * S + e) * 2;
            st[0] = mx;
            st[1] = Z;
        }
    }
    __syncwarp();
    // conv, T (lane = channel)
    const T* Pl = dw.P + (long long)l * n * 32;
    T conv = T(0), T3[3] = {T(0), T(0), T(0)};
    for (int q = 0; q < cnt; ++q) {
        const long long e = start + q;
        const T gh = g2n[32 * e + lane];
        const int j = gr.nbr[e];
        const T pj = Pl[32ll * j + lane];
        const V4<T> en0 = ld4c(dw.env + 8 * e);
        const T h2 = dw.env[8 * e + 4];
        conv += en0.y * gh * pj;
        T3[0] += en0.z * gh;
        T3[1] += en0.w * gh;
        T3[2] += h2 * gh;
    }
    conv *= md.inv_nnorm;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        T3[c] *= md.inv_nnorm;
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
    __syncwarp();
    sm.x[lane] = conv;
#pragma unroll
    for (int a = 0; a < 4; ++a) sm.x[32 + 32 * a + lane] = gr4[a];
    __syncwarp();
    T uz = L.u1.b[lane];
    for (int k = 0; k < 160; ++k) uz += __ldg(L.u1.WT + k * 32 + lane) * static_cast<T>(sm.x[k]);
    uz = d_tanh(uz);
    __syncwarp();
    dw.uz[((long long)l * n + i) * 32 + lane] = uz;
    const T g1 = dw.g1[((long long)l * n + i) * 32 + lane] + cmv(L.u2.WT, L.u2.b, uz);
    dw.g1[((long long)(l + 1) * n + i) * 32 + lane] = g1;
    return g1;
}

// Layer l backward, atom-local part: update MLP, grrg and conv adjoints, the
// per-edge adjoints of g2hat, and the attention backward (row + column pass).
// dg1_out: adjoint of g1^{l+1}_i (lane = channel).  top: no g2 adjoint from above.
// Writes dconv (scaled by 1/nnorm) for the neighbours' P gather, the residual
// part of dg1^l (dw.dg1), dg2 (adjoint of g2^l) and accumulates dwh.
template <typename T>
__device__ void rf_layer_bwd(const DevDp<T>& md, const DevGraph& gr, const DevDpWork<T>& dw,
                             long long S, int n, int l, int i, T dg1_out, bool top,
                             DpWarpSmem& sm) {
    const int lane = threadIdx.x & 31;
    const DevDpLayer<T>& L = md.L[l];
    const int start = gr.row_start[i], cnt = gr.nnei[i];
    const T* g2l = dw.g2 + (long long)l * S * 32;
    const T* g2n = dw.g2 + (long long)(l + 1) * S * 32;
    // update MLP backward
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
#pragma unroll
    for (int c = 0; c < 3; ++c) dT[c] *= md.inv_nnorm;
    dw.dconv[((long long)(l & 1) * n + i) * 32 + lane] = dconv;
    dw.dg1[32ll * i + lane] = dg1_out;
    // per-edge adjoints of g2hat (lane = channel)
    const T* Pl = dw.P + (long long)l * n * 32;
    for (int q = 0; q < cnt; ++q) {
        const long long e = start + q;
        const T gh = g2n[32 * e + lane];
        const int j = gr.nbr[e];
        const T pj = Pl[32ll * j + lane];
        const V4<T> en0 = ld4c(dw.env + 8 * e);
        const T h2 = dw.env[8 * e + 4];
        T d = top ? T(0) : dw.dg2[32 * e + lane];
        d += en0.y * dconv * pj + en0.z * dT[0] + en0.w * dT[1] + h2 * dT[2];
        dw.dg2[32 * e + lane] = d;
        const T a0 = warp_sum(dconv * gh * pj);
        const T a1 = warp_sum(dT[0] * gh);
        const T a2 = warp_sum(dT[1] * gh);
        const T a3 = warp_sum(dT[2] * gh);
        if (lane == 0) {
            T* p = dw.dwh + 4 * e;
            if (top) {
                st4(p, a0, a1, a2, a3);
            } else {
                const V4<T> old = ld4c(p);
                st4(p, old.x + a0, old.y + a1, old.z + a2, old.w + a3);
            }
        }
    }
    __syncwarp();
    // attention backward
    rf_qkv(L, g2l, dw.qkv, start, cnt);
    const T sh = static_cast<T>(kShift), isq = static_cast<T>(kInvSqrt32);
    // row pass (lane = e): do_e, S_e, dq_e, row-side dw/dh; dg2_e += Wq^T dq_e
    for (int rb = 0; rb < cnt; rb += 32) {
        const bool valid = rb + lane < cnt;
        const long long e = start + rb + (valid ? lane : 0);
        T x[32], dov[32];
        load_row(dw.dg2 + 32 * e, x);
        rmv(L.o.WT, static_cast<const T*>(nullptr), x, dov);
        if (valid) store_row(dw.dob + 32 * e, dov);
        const T* st = dw.stat + ((long long)l * S + e) * 2;
        const T mx = st[0], iz = T(1) / st[1];
        T q[32];
        load_row(dw.qkv + 96 * e, q);
        const V4<T> en0 = ld4c(dw.env + 8 * e), en1 = ld4c(dw.env + 8 * e + 4);
        const T we = en0.y, he0 = en0.z, he1 = en0.w, he2 = en1.x;
        T Ssum = T(0);
        for (int f = 0; f < cnt; ++f) {
            const long long ef = start + f;
            const T lam = dot32(q, dw.qkv + 96 * ef + 32) * isq;
            const V4<T> fn0 = ld4c(dw.env + 8 * ef), fn1 = ld4c(dw.env + 8 * ef + 4);
            const T ww = we * fn0.y;
            const T gam = he0 * fn0.z + he1 * fn0.w + he2 * fn1.x;
            const T al = d_exp((lam + sh) * ww - sh - mx) * iz;
            const T db = dot32(dov, dw.qkv + 96 * ef + 64);
            Ssum += al * db * ww * gam;
        }
        T dq[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) dq[c] = T(0);
        T dwe = T(0), dh0 = T(0), dh1 = T(0), dh2 = T(0);
        for (int f = 0; f < cnt; ++f) {
            const long long ef = start + f;
            const T* kf = dw.qkv + 96 * ef + 32;
            const T lam = dot32(q, kf) * isq;
            const V4<T> fn0 = ld4c(dw.env + 8 * ef), fn1 = ld4c(dw.env + 8 * ef + 4);
            const T wf = fn0.y, ww = we * wf;
            const T gam = he0 * fn0.z + he1 * fn0.w + he2 * fn1.x;
            const T al = d_exp((lam + sh) * ww - sh - mx) * iz;
            const T db = dot32(dov, dw.qkv + 96 * ef + 64);
            const T da = db * ww * gam;
            const T dlt = al * (da - Ssum);
            const T dlam = dlt * ww * isq;
#pragma unroll
            for (int c = 0; c < 32; c += 4) {
                const V4<T> kv = ld4c(kf + c);
                dq[c] += dlam * kv.x;
                dq[c + 1] += dlam * kv.y;
                dq[c + 2] += dlam * kv.z;
                dq[c + 3] += dlam * kv.w;
            }
            const T dww = db * al * gam + dlt * (lam + sh);
            const T dgam = db * al * ww;
            dwe += dww * wf;
            dh0 += dgam * fn0.z;
            dh1 += dgam * fn0.w;
            dh2 += dgam * fn1.x;
        }
        T y[32];
        rmv(L.q.WT, static_cast<const T*>(nullptr), dq, y);
        if (valid) {
#pragma unroll
            for (int c = 0; c < 32; ++c) y[c] += x[c];
            store_row(dw.dg2 + 32 * e, y);
            dw.aux[2 * e] = Ssum;
            T* p = dw.dwh + 4 * e;
            const V4<T> old = ld4c(p);
            st4(p, old.x + dwe, old.y + dh0, old.z + dh1, old.w + dh2);
        }
    }
    __syncwarp();
    // column pass (lane = f): dk_f, dv_f, column-side dw/dh; dg2_f += Wk^T dk_f + Wv^T dv_f
    for (int rb = 0; rb < cnt; rb += 32) {
        const bool valid = rb + lane < cnt;
        const long long f = start + rb + (valid ? lane : 0);
        T k[32], v[32], dk[32], dv[32];
        load_row(dw.qkv + 96 * f + 32, k);
        load_row(dw.qkv + 96 * f + 64, v);
#pragma unroll
        for (int c = 0; c < 32; ++c) dk[c] = dv[c] = T(0);
        const V4<T> fn0 = ld4c(dw.env + 8 * f), fn1 = ld4c(dw.env + 8 * f + 4);
        const T wf = fn0.y, hf0 = fn0.z, hf1 = fn0.w, hf2 = fn1.x;
        T dwf = T(0), dh0 = T(0), dh1 = T(0), dh2 = T(0);
        for (int r = 0; r < cnt; ++r) {
            const long long e = start + r;
            const T* qe = dw.qkv + 96 * e;
            const T* de = dw.dob + 32 * e;
            const T lam = dot32(k, qe) * isq;
            const T db = dot32(v, de);
            const V4<T> en0 = ld4c(dw.env + 8 * e), en1 = ld4c(dw.env + 8 * e + 4);
            const T we = en0.y, ww = we * wf;
            const T gam = en0.z * hf0 + en0.w * hf1 + en1.x * hf2;
            const T* st = dw.stat + ((long long)l * S + e) * 2;
            const T al = d_exp((lam + sh) * ww - sh - st[0]) / st[1];
            const T da = db * ww * gam;
            const T dlt = al * (da - dw.aux[2 * e]);
            const T dlam = dlt * ww * isq;
            const T bet = al * ww * gam;
#pragma unroll
            for (int c = 0; c < 32; c += 4) {
                const V4<T> qv = ld4c(qe + c);
                const V4<T> dv4 = ld4c(de + c);
                dk[c] += dlam * qv.x;
                dk[c + 1] += dlam * qv.y;
                dk[c + 2] += dlam * qv.z;
                dk[c + 3] += dlam * qv.w;
                dv[c] += bet * dv4.x;
                dv[c + 1] += bet * dv4.y;
                dv[c + 2] += bet * dv4.z;
                dv[c + 3] += bet * dv4.w;
            }
            const T dww = db * al * gam + dlt * (lam + sh);
            const T dgam = db * al * ww;
            dwf += dww * we;
            dh0 += dgam * en0.z;
            dh1 += dgam * en0.w;
            dh2 += dgam * en1.x;
        }
        T y[32];
        rmv(L.k.WT, static_cast<const T*>(nullptr), dk, y);
        T y2[32];
        rmv(L.v.WT, static_cast<const T*>(nullptr), dv, y2);
        if (valid) {
            T x[32];
            load_row(dw.dg2 + 32 * f, x);
#pragma unroll
            for (int c = 0; c < 32; ++c) x[c] += y[c] + y2[c];
            store_row(dw.dg2 + 32 * f, x);
            T* p = dw.dwh + 4 * f;
            const V4<T> old = ld4c(p);
            st4(p, old.x + dwf, old.y + dh0, old.z + dh1, old.w + dh2);
        }
    }
    __syncwarp();
}

// Gather of the neighbour-projection adjoint for atom j and layer l:
// dP_j = sum_{q in out(j)} w_q g2hat^l_{rev q} * dconv^l_{nbr q}, returns
// dg1^l_j = dg1(residual) + Wc^T dP_j (lane = channel).
template <typename T>
__device__ __forceinline__ T rf_gather_dg1(const DevDp<T>& md, const DevGraph& gr,
                                           const DevDpWork<T>& dw, long long S, int n, int l,
                                           int j) {
    const int lane = threadIdx.x & 31;
    const int start = gr.row_start[j], cnt = gr.nnei[j];
    const T* g2n = dw.g2 + (long long)(l + 1) * S * 32;
    const T* dcv = dw.dconv + (long long)(l & 1) * n * 32;
    T dP = T(0);
    for (int q = 0; q < cnt; ++q) {
        const long long e = start + q;
        const int mir = gr.inv_pos[e];
        const int i = gr.nbr[e];
        dP += dw.env[8ll * mir + 1] * g2n[32ll * mir + lane] * dcv[32ll * i + lane];
    }
    T acc = dw.dg1[32ll * j + lane];
#pragma unroll 8
    for (int k = 0; k < 32; ++k) acc += __ldg(md.L[l].c.W + k * 32 + lane) * shfl(dP, k);
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
template <typename T>
__global__ __launch_bounds__(kDpCTA) void k_rf_fwd(DevDp<T> md, DevGraph gr, DevWork<T> ws,
                                                   DevDpWork<T> dw, int l) {
    __shared__ DpWarpSmem s_w[kDpWarps];
    pdl_launch_dependents();
    const WarpIdx wi;
    pdl_wait();
    const int n = gr.n;
    for (int i = wi.first; i < gr.n_active; i += wi.stride) {
        const T g1 = rf_layer_fwd(md, gr, dw, ws.slots, n, l, i, s_w[wi.wid]);
        dw.P[((long long)(l + 1) * n + i) * 32 + wi.lane] = cmv(md.L[l + 1].c.WT, md.L[l + 1].c.b, g1);
        __syncwarp();
    }
}

// Top layer forward + fitting + top layer backward (atom-local part).
template <typename T>
__global__ __launch_bounds__(kDpCTA) void k_rf_top(DevDp<T> md, DevGraph gr, DevWork<T> ws,
                                                   DevDpWork<T> dw) {
    __shared__ DpWarpSmem s_w[kDpWarps];
    pdl_launch_dependents();
    const WarpIdx wi;
    pdl_wait();
    const int n = gr.n, l = md.n_layers - 1;
    for (int i = wi.first; i < gr.n_active; i += wi.stride) {
        const T g1 = rf_layer_fwd(md, gr, dw, ws.slots, n, l, i, s_w[wi.wid]);
        const T dg1 = rf_fit(md, gr, ws, i, g1);
        rf_layer_bwd(md, gr, dw, ws.slots, n, l, i, dg1, true, s_w[wi.wid]);
    }
}

// Gather for layer l + 1, then layer l backward.
template <typename T>
__global__ __launch_bounds__(kDpCTA) void k_rf_bwd(DevDp<T> md, DevGraph gr, DevWork<T> ws,
                                                   DevDpWork<T> dw, int l) {
    __shared__ DpWarpSmem s_w[kDpWarps];
    pdl_launch_dependents();
    const WarpIdx wi;
    pdl_wait();
    const int n = gr.n;
    for (int i = wi.first; i < gr.n_active; i += wi.stride) {
        const T dg1 = rf_gather_dg1(md, gr, dw, ws.slots, n, l + 1, i);
        __syncwarp();
        rf_layer_bwd(md, gr, dw, ws.slots, n, l, i, dg1, false, s_w[wi.wid]);
    }
}

// Gather for layer 0, g1 map + descriptor + embedding backward -> dE/d(edge_dr).
template <typename T>
__global__ __launch_bounds__(kDpCTA) void k_rf_embed_bwd(DevDp<T> md, DevGraph gr, DevWork<T> ws,
                                                         DevDpWork<T> dw) {
    __shared__ DpWarpSmem s_w[kDpWarps];
    pdl_launch_dependents();
    const WarpIdx wi;
    const int lane = wi.lane;
    T w1[kMaxTypes], b1[kMaxTypes];
#pragma unroll
    for (int t = 0; t < kMaxTypes; ++t) {
        w1[t] = t < md.n_types ? md.emb_w1[t][lane] : T(0);
        b1[t] = t < md.n_types ? md.emb_b1[t][lane] : T(0);
    }
    pdl_wait();
    const int n = gr.n;
    for (int i = wi.first; i < gr.n_active; i += wi.stride) {
        const int start = gr.row_start[i], cnt = gr.nnei[i];
        const T dg1 = rf_gather_dg1(md, gr, dw, ws.slots, n, 0, i);
        // g1 map backward
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
        for (int c = 0; c < 4; ++c) dA[c] *= md.inv_nnorm;
        for (int q = 0; q < cnt; ++q) {
            const long long e = start + q;
            const V4<T> en0 = ld4c(dw.env + 8 * e), en1 = ld4c(dw.env + 8 * e + 4);
            const T s = en0.x;
            const int t = static_cast<int>(en1.w);
            const T G = dw.g2[32 * e + lane];
            const T dG = dw.dg2[32 * e + lane] + dA[0] * s + dA[1] * en0.z + dA[2] * en0.w +
                         dA[3] * en1.x;
            const T dR0 = warp_sum(dA[0] * G), dR1 = warp_sum(dA[1] * G),
                    dR2 = warp_sum(dA[2] * G), dR3 = warp_sum(dA[3] * G);
            T ds = T(0);
#pragma unroll
            for (int tt = 0; tt < kMaxTypes; ++tt)
                if (tt == t) {
                    const T z = d_tanh(w1[tt] * s + b1[tt]);
                    T dz = T(0);
#pragma unroll 8
                    for (int b = 0; b < 32; ++b) dz += __ldg(md.emb2[tt].W + b * 32 + lane) * shfl(dG, b);
                    dz *= (T(1) - z * z);
                    ds = warp_sum(w1[tt] * dz);
                }
            if (lane == 0) {
                const V4<T> wh = ld4c(dw.dwh + 4 * e);
                const double* d = gr.dr + 3ll * e;
                const Env<T> v = dp_env<T>(d, md.rc, md.rcs);
                T g[3];
                dp_gvec(v, d, ds + dR0, dR1 + wh.y, dR2 + wh.z, dR3 + wh.w, wh.x, g);
                st4(ws.gv + 4 * e, g[0], g[1], g[2], T(0));
                st4(ws.gvrev + 4ll * gr.inv_pos[e], g[0], g[1], g[2], T(0));
            }
        }
        __syncwarp();
    }
    (void)s_w;
}

int dp_grid(int n) {
    const int want = (n + kDpWarps - 1) / kDpWarps;
    const int cap = num_sms() * 8;
    return want < 1 ? 1 : (want < cap ? want : cap);
}

}  // namespace

// Launches the whole DeePMD-style network + forces; returns the kernel count.
template <typename T>
int launch_dp(const DevDp<T>& md, const DevGraph& gr, const DevWork<T>& ws,
              const DevDpWork<T>& dw, double* forces, double* per_atom, double* out, int* rev,
              cudaStream_t st, const Marker& mk, const MdFuse& mf) {
    const dim3 grid(dp_grid(gr.n_active)), block(kDpCTA);
    if (md.family == kSeA) {
        launch_pdl(k_sea<T>, grid, block, 0, st, md, gr, ws, rev, mf);
        mk("sea", st);
        launch_force<T>(gr, ws, forces, per_atom, out, st, mf);
        mk("force", st);
        return 2;
    }
    // rev is computed by k_rf_embed; the later kernels read it as gr.inv_pos
    DevGraph g2 = gr;
    if (rev) g2.inv_pos = rev;
    const int L = md.n_layers;
    launch_pdl(k_rf_embed<T>, grid, block, 0, st, md, gr, ws, dw, rev, mf);
    mk("rf_embed", st);
    for (int l = 0; l + 1 < L; ++l) {
        launch_pdl(k_rf_fwd<T>, grid, block, 0, st, md, g2, ws, dw, l);
        mk("rf_fwd", st);
    }
    launch_pdl(k_rf_top<T>, grid, block, 0, st, md, g2, ws, dw);
    mk("rf_top", st);
    for (int l = L - 2; l >= 0; --l) {
        launch_pdl(k_rf_bwd<T>, grid, block, 0, st, md, g2, ws, dw, l);
        mk("rf_bwd", st);
    }
    launch_pdl(k_rf_embed_bwd<T>, grid, block, 0, st, md, g2, ws, dw);
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
