// hmdp_net.cu — the DP network kernels (embedding, message layers, fitting,
// reverse mode, forces/virial), sm_100a.
//
// Decomposition: one 128-thread CTA per atom (grid-stride over atoms).  Atom-level
// MLPs are 4-way split mat-vecs (bmv, hmdp_common.cuh) with the activation vector
// in shared memory; per-edge work is split over the 4 warps (edge q -> warp q % 4)
// with lane = channel, so every per-edge row access is one coalesced 128-byte line.
// Edge -> atom sums are reduced in a fixed order (deterministic, no float atomics):
// the reference's scatters dh_j += ..., F_j -= ... (inference.cpp:343, :380) become
// gathers over each atom's in-edges.
//
// Linearity of the message MLP is exploited exactly (same function, fewer FLOPs):
//   forward   z_e = tanh(W1h h_j + W1b b_e + b1), and W1h h_j is a per-ATOM
//             projection P_j computed once per layer instead of once per edge;
//             msum_i = sum_e s_e (W2 z_e + b2) = W2 (sum_e s_e z_e) + (sum_e s_e) b2
//   backward  with dmsum_i from the update MLP, v = W2^T dmsum_i, c0 = dmsum_i.b2:
//             dsc_e = dmsum_i . mo_e = v . z_e + c0,  dz_e = s_e v (1 - z_e^2),
//             dE/dr_e += dsc_e s'(r_e) + sum_k b'_e[k] (W1b^T dz_e)[k],
//             dE/dh_j += W1h^T sum_{e in in(j)} dz_e  (one mat-vec per atom).
//
// Reference correspondence (paths relative to /root/reference/proj):
//   k_embed      edge radial + descriptor + embedding fwd   src/nn/inference.cpp:214-249
//                [FUSE_FIT: + fitting fwd/bwd + embedding bwd, :288-311, :355-370]
//   k_msg_fwd    message layer fwd                          :251-286
//                [LAST: + fitting fwd/bwd + top message layer bwd, :288-353]
//   k_msg_bwd    message layer bwd (lower layers)           :313-353
//   k_embed_bwd  embedding + descriptor adjoint             :355-370
//   k_force      force / virial (gather form) + E, W sums   :288-298, :372-387
#include "hmdp_common.cuh"

namespace hmdp {

int atom_grid(int n);  // hmdp_nbr.cu

// Shared per-CTA scratch for one atom.
template <typename T>
struct AtomSmem {
    T v0[64], v1[64], v2[64], v3[64];  // activation vectors
    T part[4][32];                     // per-warp partial channel sums
    T s4[4];                           // block_sum scratch
    T sc[4];                           // per-warp scalar partials
};

// ---------------------------------------------------------------------------
// Fitting net forward + backward on h (in sm.v0 ... written by the caller into
// `h_s`), leaves dE/dh in dh_s.  inference.cpp:288-311.  Returns nothing; writes
// e_i for owned atoms (0 for ghosts) and dh = 0 for ghosts.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void fit_fwd_bwd(const DevMlp<T>& fit, const T* h_s, T* z_s, T* dz_s,
                                            T* dh_s, bool owned, double* e_out, T* s4, int t) {
    constexpr int O = 32;
    const int o = bmv_out<O>(t);
    const bool lead = bmv_lead<O>(t);
    const T zf = d_tanh(bmv<T, 32, 32>(fit.W1, 32, h_s, t) + __ldg(fit.b1 + o));
    if (lead) z_s[o] = zf;
    __syncthreads();
    // linear head 32 -> 1 and its adjoint (dout = 1)
    T ez = (t < 32) ? __ldg(fit.W2 + t) * z_s[t] : T(0);
    const T e = block_sum(ez, s4) + __ldg(fit.b2);
    if (t == 0) *e_out = owned ? static_cast<double>(e) : 0.0;
    if (t < 32) dz_s[t] = (__ldg(fit.W2 + t) * T(1)) * (T(1) - z_s[t] * z_s[t]);
    __syncthreads();
    const T dh = bmv<T, 32, 32>(fit.W1T, 32, dz_s, t);
    __syncthreads();  // dh_s may alias dz_s
    if (lead) dh_s[o] = owned ? dh : T(0);
    __syncthreads();
}

// ---------------------------------------------------------------------------
// Edge radial features + descriptor + embedding (and the message-layer-0 atom
// projection, or for depth 1 the whole fitting/backward chain).
// ---------------------------------------------------------------------------
template <typename T, bool FUSE_FIT>
__global__ __launch_bounds__(kAT) void k_embed(DevModel<T> md, DevGraph gr, DevWork<T> ws,
                                               int* __restrict__ rev, MdFuse mf) {
    __shared__ AtomSmem<T> sm;
    __shared__ T s_b[kAT][kK + 1];
    __shared__ int s_ty[kAT];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    // this step's neighbour search is complete: clear the cell counts for the
    // binning fused into the force kernel (device MD) / keep the zero invariant
    for (int c = blockIdx.x * blockDim.x + t; c < mf.n_cells_zero; c += gridDim.x * blockDim.x)
        mf.cell_count[c] = 0;
    const int nd = md.n_types * kK;
    constexpr int O = 32;
    const int o = bmv_out<O>(t);
    const bool lead = bmv_lead<O>(t);
    for (int i = blockIdx.x; i < gr.n; i += gridDim.x) {
        const int start = gr.row_start[i], cnt = gr.nnei[i];
        T desc = T(0);  // thread q < nd accumulates descriptor component q
        for (int base = 0; base < cnt; base += kAT) {
            const int m = min(kAT, cnt - base);
            const int e = start + base + t;
            int j = 0;
            if (t < m) {
                j = gr.nbr[e];
                const int ty = gr.types[j];
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
                ws.er[e] = r;
                ws.es[e] = s;
                ws.eds[e] = ds;
                st4(ws.eb + 8ll * e, b[0], b[1], b[2], b[3]);
                st4(ws.eb + 8ll * e + 4, b[4], b[5], b[6], b[7]);
                st4(ws.edb + 8ll * e, db[0], db[1], db[2], db[3]);
                st4(ws.edb + 8ll * e + 4, db[4], db[5], db[6], db[7]);
#pragma unroll
                for (int k = 0; k < kK; ++k) s_b[t][k] = b[k];
                s_ty[t] = ty;
            }
            if (rev) {
                // rev(e) = slot of i in nbr(j) (symmetric, sorted list).  Lane l of the
                // warp owning edges [32w, 32w+32) reads entry l of each neighbour's
                // list (one memory latency for the warp); a ballot finds i.
                const int mw = min(32, max(0, m - 32 * w));
                const int rs_l = t < m ? gr.row_start[j] : 0;
                const int nn_l = t < m ? gr.nnei[j] : 0;
                int val[32];
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    const int rsq = __shfl_sync(FULL_MASK, rs_l, q);
                    const int nnq = __shfl_sync(FULL_MASK, nn_l, q);
                    val[q] = (q < mw && lane < nnq) ? gr.nbr[rsq + lane] : -1;
                }
                int found = -1;
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    const unsigned bal = __ballot_sync(FULL_MASK, val[q] == i);
                    if (lane == q && bal) found = rs_l + __ffs(bal) - 1;
                }
                if (t < m) {
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
                }
            }
            __syncthreads();
            if (t < nd) {  // descriptor: CSR edge order, as inference.cpp:228-238
                const int ty = t >> 3, k = t & 7;
                for (int r = 0; r < m; ++r) desc += (s_ty[r] == ty) ? s_b[r][k] : T(0);
            }
            __syncthreads();
        }
        if (t < 32) {
            sm.v0[t] = t < nd ? desc : T(0);
            if (t < nd) ws.desc[static_cast<long long>(i) * 32 + t] = desc;
        }
        __syncthreads();
        // embedding forward nd (zero-padded to 32) -> 32 (tanh) -> 32
        const T z1 = d_tanh(bmv<T, 32, 32>(md.embed.W1, 32, sm.v0, t) + __ldg(md.embed.b1 + o));
        if (lead) {
            sm.v1[o] = z1;
            ws.ez1[static_cast<long long>(i) * kH + o] = z1;
        }
        __syncthreads();
        const T h0 = bmv<T, 32, 32>(md.embed.W2, 32, sm.v1, t) + __ldg(md.embed.b2 + o);
        if (lead) {
            sm.v2[o] = h0;
            ws.h[static_cast<long long>(i) * kH + o] = h0;
        }
        __syncthreads();
        if constexpr (FUSE_FIT) {
            const bool owned = !(gr.is_ghost && gr.is_ghost[i]);
            fit_fwd_bwd(md.fit, sm.v2, sm.v3, sm.v0, sm.v3, owned, ws.e_atom + i, sm.s4, t);
            // embedding backward: linear layer 2 (W2^T), tanh layer 1 (W1^T, padded)
            const T dz1 = bmv<T, 32, 32>(md.embed.W2T, 32, sm.v3, t) * (T(1) - z1 * z1);
            if (lead) sm.v0[o] = dz1;
            __syncthreads();
            const T dd = bmv<T, 32, 32>(md.embed.W1T, 32, sm.v0, t);
            if (lead) sm.v1[o] = dd;
            __syncthreads();
            for (int base = 0; base < cnt; base += kAT) {
                const int m = min(kAT, cnt - base);
                if (t < m) {
                    const long long e = start + base + t;
                    const int ty = gr.types[gr.nbr[e]];
                    const V4<T> d0 = ld4c(ws.edb + 8 * e), d1 = ld4c(ws.edb + 8 * e + 4);
                    const T* dv = sm.v1 + ty * kK;
                    T acc = dv[0] * d0.x;
                    acc += dv[1] * d0.y;
                    acc += dv[2] * d0.z;
                    acc += dv[3] * d0.w;
                    acc += dv[4] * d1.x;
                    acc += dv[5] * d1.y;
                    acc += dv[6] * d1.z;
                    acc += dv[7] * d1.w;
                    ws.g[e] = acc;
                }
            }
        } else {
            // P^0 = W1h^(0) h^0: the neighbour projection of message layer 0
            const T p = bmv<T, 32, 32>(md.msg[0].W1, kH + kK, sm.v2, t);
            if (lead) ws.p[static_cast<long long>(i) * kH + o] = p;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Message-layer backward body for atom i, given dE/dh^{l+1}_i in sm.v0 and the
// update hidden activations in sm.v2.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void msg_backward_body(const DevModel<T>& md, const DevGraph& gr,
                                                  const DevWork<T>& ws, AtomSmem<T>& sm, int l,
                                                  int i, bool first_g) {
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const long long S = ws.slots;
    const DevMlp<T> msg = md.msg[l];
    const DevMlp<T> upd = md.upd[l];
    constexpr int O = 32;
    const int o = bmv_out<O>(t);
    const bool lead = bmv_lead<O>(t);
    // update MLP backward (64 -> 32 tanh -> 32)
    const T zu = sm.v2[o];
    const T dz = bmv<T, 32, 32>(upd.W2T, 32, sm.v0, t) * (T(1) - zu * zu);
    if (lead) sm.v3[o] = dz;
    __syncthreads();
    const T din = bmv<T, 64, 32>(upd.W1T, 32, sm.v3, t);  // 64 outputs, 2 parts each
    if (bmv_lead<64>(t)) {
        const int k = bmv_out<64>(t);
        if (k < kH)
            ws.dhown[static_cast<long long>(i) * kH + k] = sm.v0[k] + din;  // residual + update
        else
            sm.v1[k - kH] = din;  // dmsum
    }
    __syncthreads();
    const T v = bmv<T, 32, 32>(msg.W2T, 32, sm.v1, t);  // v = W2^T dmsum
    if (lead) sm.v2[o] = v;
    const T c0 = block_sum(t < 32 ? sm.v1[t] * __ldg(msg.b2 + t) : T(0), sm.s4);
    // (block_sum's barriers also publish sm.v2)
    T w1b[kK];
#pragma unroll
    for (int k = 0; k < kK; ++k) w1b[k] = __ldg(msg.W1T + (kH + k) * kH + lane);
    const T vl = sm.v2[lane];
    const T* __restrict__ Z = ws.z + l * S * kH;
    T* __restrict__ D = ws.d + (l & 1) * S * kH;
    const int start = gr.row_start[i], cnt = gr.nnei[i];
    for (int base = 0; base < cnt; base += kAT) {
        // warp w owns edges base + w + 4u; lane u prefetches edge u's scalars
        const int mw = max(0, (min(kAT, cnt - base) - w + 3) / 4);
        const long long el = start + base + w + 4 * (lane < mw ? lane : 0);
        const T s_l = ws.es[el], ds_l = ws.eds[el];
        const V4<T> d0_l = ld4(ws.edb + 8 * el), d1_l = ld4(ws.edb + 8 * el + 4);
        T zr[32];
#pragma unroll
        for (int u = 0; u < 32; ++u)
            if (u < mw) zr[u] = Z[(start + base + w + 4 * u) * static_cast<long long>(kH) + lane];
        T tot_l = T(0);
#pragma unroll
        for (int u = 0; u < 32; ++u) {
            if (u >= mw) break;
            const long long e = start + base + w + 4 * u;
            const T z = zr[u];
            const T s = __shfl_sync(FULL_MASK, s_l, u), ds = __shfl_sync(FULL_MASK, ds_l, u);
            T wv = w1b[0] * __shfl_sync(FULL_MASK, d0_l.x, u);
            wv += w1b[1] * __shfl_sync(FULL_MASK, d0_l.y, u);
            wv += w1b[2] * __shfl_sync(FULL_MASK, d0_l.z, u);
            wv += w1b[3] * __shfl_sync(FULL_MASK, d0_l.w, u);
            wv += w1b[4] * __shfl_sync(FULL_MASK, d1_l.x, u);
            wv += w1b[5] * __shfl_sync(FULL_MASK, d1_l.y, u);
            wv += w1b[6] * __shfl_sync(FULL_MASK, d1_l.z, u);
            wv += w1b[7] * __shfl_sync(FULL_MASK, d1_l.w, u);
            const T d = s * vl * (T(1) - z * z);
            D[e * kH + lane] = d;
            const T tot = warp_sum(ds * vl * z + d * wv);
            if (lane == u) tot_l = tot;
        }
        if (lane < mw) ws.g[el] = (first_g ? T(0) : ws.g[el]) + (tot_l + ds_l * c0);
    }
}

// S_i = sum over in-edges of dz_e (layer l) -> sm.v1, split over the 4 warps
template <typename T>
__device__ __forceinline__ void gather_in(const DevGraph& gr, const DevWork<T>& ws,
                                          AtomSmem<T>& sm, int l, int i) {
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const T* __restrict__ D = ws.d + (l & 1) * ws.slots * kH;
    const int is = gr.in_start[i], ic = gr.in_cnt[i];
    T sg = T(0);
    for (int base = 0; base < ic; base += kAT) {
        const int mw = max(0, (min(kAT, ic - base) - w + 3) / 4);
        const int idx = lane < mw ? gr.in_edge[is + base + w + 4 * lane] : 0;
        T dr_[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) {
            const long long e = __shfl_sync(FULL_MASK, idx, u);
            if (u < mw) dr_[u] = D[e * kH + lane];
        }
#pragma unroll
        for (int u = 0; u < 32; ++u)
            if (u < mw) sg += dr_[u];
    }
    sm.part[w][lane] = sg;
    __syncthreads();
    if (t < 32) sm.v1[t] = ((sm.part[0][t] + sm.part[1][t]) + sm.part[2][t]) + sm.part[3][t];
    __syncthreads();
}

// ---------------------------------------------------------------------------
// Message layer l forward; LAST fuses the fitting net and the top layer's
// backward (all atom-local).
// ---------------------------------------------------------------------------
template <typename T, bool LAST>
__global__ __launch_bounds__(kAT) void k_msg_fwd(DevModel<T> md, DevGraph gr, DevWork<T> ws,
                                                 int l) {
    __shared__ AtomSmem<T> sm;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int n = gr.n;
    const long long S = ws.slots;
    const DevMlp<T> msg = md.msg[l];
    const DevMlp<T> upd = md.upd[l];
    const T* __restrict__ Pin = ws.p + (l & 1) * static_cast<long long>(n) * kH;
    T* __restrict__ Z = ws.z + l * S * kH;
    T w1b[kK];
#pragma unroll
    for (int k = 0; k < kK; ++k) w1b[k] = __ldg(msg.W1T + (kH + k) * kH + lane);
    const T b1 = __ldg(msg.b1 + lane);
    constexpr int O = 32;
    const int o = bmv_out<O>(t);
    const bool lead = bmv_lead<O>(t);
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const int start = gr.row_start[i], cnt = gr.nnei[i];
        T acc = T(0), ssum = T(0);
        for (int base = 0; base < cnt; base += kAT) {
            const int mw = max(0, (min(kAT, cnt - base) - w + 3) / 4);
            const long long el = start + base + w + 4 * (lane < mw ? lane : 0);
            const int jl = gr.nbr[el];
            const T s_l = ws.es[el];
            const V4<T> b0_l = ld4(ws.eb + 8 * el), b1_l = ld4(ws.eb + 8 * el + 4);
            T pr[32];
#pragma unroll
            for (int u = 0; u < 32; ++u) {
                const int j = __shfl_sync(FULL_MASK, jl, u);
                if (u < mw) pr[u] = Pin[static_cast<long long>(j) * kH + lane];
            }
#pragma unroll
            for (int u = 0; u < 32; ++u) {
                if (u >= mw) break;
                const long long e = start + base + w + 4 * u;
                const T s = __shfl_sync(FULL_MASK, s_l, u);
                T a = b1;
                a += w1b[0] * __shfl_sync(FULL_MASK, b0_l.x, u);
                a += w1b[1] * __shfl_sync(FULL_MASK, b0_l.y, u);
                a += w1b[2] * __shfl_sync(FULL_MASK, b0_l.z, u);
                a += w1b[3] * __shfl_sync(FULL_MASK, b0_l.w, u);
                a += w1b[4] * __shfl_sync(FULL_MASK, b1_l.x, u);
                a += w1b[5] * __shfl_sync(FULL_MASK, b1_l.y, u);
                a += w1b[6] * __shfl_sync(FULL_MASK, b1_l.z, u);
                a += w1b[7] * __shfl_sync(FULL_MASK, b1_l.w, u);
                const T z = d_tanh(a + pr[u]);
                Z[e * kH + lane] = z;
                acc += s * z;
                ssum += s;
            }
        }
        sm.part[w][lane] = acc;
        if (lane == 0) sm.sc[w] = ssum;
        if (t < 32) sm.v1[t] = ws.h[(static_cast<long long>(l) * n + i) * kH + t];  // h_i
        __syncthreads();
        if (t < 32) sm.v0[t] = ((sm.part[0][t] + sm.part[1][t]) + sm.part[2][t]) + sm.part[3][t];
        const T stot = ((sm.sc[0] + sm.sc[1]) + sm.sc[2]) + sm.sc[3];
        __syncthreads();
        // msum = W2 (sum_e s_e z_e) + (sum_e s_e) b2  -> second half of the update input
        const T msum = bmv<T, 32, 32>(msg.W2, 32, sm.v0, t) + stot * __ldg(msg.b2 + o);
        if (lead) sm.v1[kH + o] = msum;
        __syncthreads();
        // update MLP on [h_i, msum] (64 -> 32 tanh -> 32), residual
        const T zu = d_tanh(bmv<T, 32, 64>(upd.W1, 2 * kH, sm.v1, t) + __ldg(upd.b1 + o));
        if (lead) {
            sm.v2[o] = zu;
            ws.uz1[(static_cast<long long>(l) * n + i) * kH + o] = zu;
        }
        __syncthreads();
        const T hn = sm.v1[o] + (bmv<T, 32, 32>(upd.W2, 32, sm.v2, t) + __ldg(upd.b2 + o));
        if (lead) {
            sm.v3[o] = hn;
            ws.h[(static_cast<long long>(l + 1) * n + i) * kH + o] = hn;
        }
        __syncthreads();
        if constexpr (!LAST) {
            const T p = bmv<T, 32, 32>(md.msg[l + 1].W1, kH + kK, sm.v3, t);
            if (lead)
                ws.p[((l + 1) & 1) * static_cast<long long>(n) * kH + static_cast<long long>(i) * kH + o] = p;
        } else {
            const bool owned = !(gr.is_ghost && gr.is_ghost[i]);
            // fitting: h^M in v3 -> dE/dh^M in v0 (v1 scratch for the fit hidden layer)
            fit_fwd_bwd(md.fit, sm.v3, sm.v1, sm.v0, sm.v0, owned, ws.e_atom + i, sm.s4, t);
            msg_backward_body(md, gr, ws, sm, l, i, true);
        }
        __syncthreads();
    }
}

// Message layer l < M-1 backward: gather dE/dh^{l+1}, then the layer body.
template <typename T>
__global__ __launch_bounds__(kAT) void k_msg_bwd(DevModel<T> md, DevGraph gr, DevWork<T> ws,
                                                 int l) {
    __shared__ AtomSmem<T> sm;
    const int t = threadIdx.x;
    constexpr int O = 32;
    const int o = bmv_out<O>(t);
    const bool lead = bmv_lead<O>(t);
    for (int i = blockIdx.x; i < gr.n; i += gridDim.x) {
        gather_in(gr, ws, sm, l + 1, i);
        // dE/dh^{l+1}_i = own + W1h^(l+1)^T S_i
        const T dh = ws.dhown[static_cast<long long>(i) * kH + o] +
                     bmv<T, 32, 32>(md.msg[l + 1].W1T, 32, sm.v1, t);
        if (lead) {
            sm.v0[o] = dh;
            sm.v2[o] = ws.uz1[(static_cast<long long>(l) * gr.n + i) * kH + o];
        }
        __syncthreads();
        msg_backward_body(md, gr, ws, sm, l, i, false);
        __syncthreads();
    }
}

// Embedding backward + descriptor adjoint (depth > 1).
template <typename T>
__global__ __launch_bounds__(kAT) void k_embed_bwd(DevModel<T> md, DevGraph gr, DevWork<T> ws) {
    __shared__ AtomSmem<T> sm;
    const int t = threadIdx.x;
    constexpr int O = 32;
    const int o = bmv_out<O>(t);
    const bool lead = bmv_lead<O>(t);
    for (int i = blockIdx.x; i < gr.n; i += gridDim.x) {
        gather_in(gr, ws, sm, 0, i);
        const T dh = ws.dhown[static_cast<long long>(i) * kH + o] +
                     bmv<T, 32, 32>(md.msg[0].W1T, 32, sm.v1, t);
        if (lead) sm.v0[o] = dh;
        __syncthreads();
        const T z1 = ws.ez1[static_cast<long long>(i) * kH + o];
        const T dz1 = bmv<T, 32, 32>(md.embed.W2T, 32, sm.v0, t) * (T(1) - z1 * z1);
        if (lead) sm.v2[o] = dz1;
        __syncthreads();
        const T dd = bmv<T, 32, 32>(md.embed.W1T, 32, sm.v2, t);
        if (lead) sm.v3[o] = dd;
        __syncthreads();
        const int start = gr.row_start[i], cnt = gr.nnei[i];
        for (int q = t; q < cnt; q += kAT) {
            const long long e = start + q;
            const int ty = gr.types[gr.nbr[e]];
            const V4<T> d0 = ld4(ws.edb + 8 * e), d1 = ld4(ws.edb + 8 * e + 4);
            const T* dv = sm.v3 + ty * kK;
            T acc = dv[0] * d0.x;
            acc += dv[1] * d0.y;
            acc += dv[2] * d0.z;
            acc += dv[3] * d0.w;
            acc += dv[4] * d1.x;
            acc += dv[5] * d1.y;
            acc += dv[6] * d1.z;
            acc += dv[7] * d1.w;
            ws.g[e] = ws.g[e] + acc;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Forces (gather form), per-atom energy, virial, and the fused velocity-Verlet
// tail of the device MD loop; deterministic grid reduction of E, W, W_ab.
//   F_i = sum_{e in out(i)} u_e g_e - sum_{e in in(i)} u_e g_e
//   W   = -sum_e g_e r_e ;  W_ab = -sum_e g_e dr_a u_b
// ---------------------------------------------------------------------------
template <typename T>
__global__ __launch_bounds__(kAT) void k_force(DevGraph gr, DevWork<T> ws, double* __restrict__ forces,
                                               double* __restrict__ per_atom, double* __restrict__ out,
                                               MdFuse mf) {
    __shared__ double s_f[4][3];
    __shared__ double s_part[4][12];
    __shared__ bool s_last;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    double acc[11];
#pragma unroll
    for (int q = 0; q < 11; ++q) acc[q] = 0.0;
    for (int i = blockIdx.x; i < gr.n; i += gridDim.x) {
        double fx = 0.0, fy = 0.0, fz = 0.0;
        const int start = gr.row_start[i], cnt = gr.nnei[i];
        for (int q = t; q < cnt; q += kAT) {
            const int e = start + q;
            const T g = ws.g[e];
            T x, y, z;
            const double* d = gr.dr + 3ll * e;
            const T r = edge_len<T>(d, x, y, z);
            const T ux = x / r, uy = y / r, uz = z / r;
            fx += static_cast<double>(ux * g);
            fy += static_cast<double>(uy * g);
            fz += static_cast<double>(uz * g);
            acc[1] -= static_cast<double>(g * r);
            const double gd = static_cast<double>(g);
            const double u3[3] = {static_cast<double>(ux), static_cast<double>(uy),
                                  static_cast<double>(uz)};
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b) acc[2 + 3 * a + b] -= gd * d[a] * u3[b];
        }
        const int is = gr.in_start[i], ic = gr.in_cnt[i];
        for (int q = t; q < ic; q += kAT) {
            const int e = gr.in_edge[is + q];
            const T g = ws.g[e];
            T x, y, z;
            const T r = edge_len<T>(gr.dr + 3ll * e, x, y, z);
            fx -= static_cast<double>((x / r) * g);
            fy -= static_cast<double>((y / r) * g);
            fz -= static_cast<double>((z / r) * g);
        }
        fx = warp_sum(fx);
        fy = warp_sum(fy);
        fz = warp_sum(fz);
        if (lane == 0) {
            s_f[w][0] = fx;
            s_f[w][1] = fy;
            s_f[w][2] = fz;
        }
        __syncthreads();
        if (t == 0) {
            const double f3[3] = {((s_f[0][0] + s_f[1][0]) + s_f[2][0]) + s_f[3][0],
                                  ((s_f[0][1] + s_f[1][1]) + s_f[2][1]) + s_f[3][1],
                                  ((s_f[0][2] + s_f[1][2]) + s_f[2][2]) + s_f[3][2]};
            forces[3 * i] = f3[0];
            forces[3 * i + 1] = f3[1];
            forces[3 * i + 2] = f3[2];
            const double ei = ws.e_atom[i];
            if (per_atom) per_atom[i] = ei;
            acc[0] += ei;
            if (mf.mode) {
                const double s = mf.half / mf.m[i];
                const bool finite = isfinite(f3[0]) && isfinite(f3[1]) && isfinite(f3[2]);
                if (!finite) atomicOr(ws.err, kErrNonFinite);
                double x3[3];
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    double va = __dadd_rn(mf.v[3 * i + a], __dmul_rn(f3[a], s));  // closing kick
                    if (mf.mode == 2) {
                        va = __dadd_rn(va, __dmul_rn(f3[a], s));  // next step's opening kick
                        x3[a] = __dadd_rn(mf.x[3 * i + a], __dmul_rn(va, mf.dt));
                        mf.x[3 * i + a] = x3[a];
                    }
                    mf.v[3 * i + a] = va;
                }
                if (mf.mode == 2)
                    bin_atom(i, x3, mf.cg, mf.cell_count, mf.members, mf.cell_of, ws.err);
            }
        }
        __syncthreads();
    }
    // CTA partials (fixed order), then the last CTA reduces them in fixed order
#pragma unroll
    for (int q = 0; q < 11; ++q) acc[q] = warp_sum(acc[q]);
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < 11; ++q) s_part[w][q] = acc[q];
    __syncthreads();
    if (t < 11)
        ws.partial[blockIdx.x * 16 + t] =
            ((s_part[0][t] + s_part[1][t]) + s_part[2][t]) + s_part[3][t];
    __threadfence();
    __syncthreads();
    if (t == 0) s_last = (atomicAdd(ws.ticket, 1u) == gridDim.x - 1);
    __syncthreads();
    if (s_last) {
        __threadfence();
        double v[11];
#pragma unroll
        for (int q = 0; q < 11; ++q) v[q] = 0.0;
        for (unsigned b = t; b < gridDim.x; b += kAT)
#pragma unroll
            for (int q = 0; q < 11; ++q) v[q] += __ldcg(ws.partial + b * 16 + q);
#pragma unroll
        for (int q = 0; q < 11; ++q) v[q] = warp_sum(v[q]);
        if (lane == 0)
#pragma unroll
            for (int q = 0; q < 11; ++q) s_part[w][q] = v[q];
        __syncthreads();
        if (t < 11) out[t] = ((s_part[0][t] + s_part[1][t]) + s_part[2][t]) + s_part[3][t];
        if (t == 0) *ws.ticket = 0u;  // re-arm for the next launch / graph replay
    }
}

// ---------------------------------------------------------------------------
template <typename T>
int launch_network(const DevModel<T>& md, const DevGraph& gr, const DevWork<T>& ws,
                   double* forces, double* per_atom, double* out, int* rev, cudaStream_t st,
                   const Marker& mk, const MdFuse& mf) {
    const int nb = atom_grid(gr.n);
    const int M = md.n_msg;
    int launches = 0;
    if (M == 0) {
        k_embed<T, true><<<nb, kAT, 0, st>>>(md, gr, ws, rev, mf);
        mk("embed_fit", st);
        ++launches;
    } else {
        k_embed<T, false><<<nb, kAT, 0, st>>>(md, gr, ws, rev, mf);
        mk("embed", st);
        for (int l = 0; l < M; ++l) {
            if (l == M - 1) {
                k_msg_fwd<T, true><<<nb, kAT, 0, st>>>(md, gr, ws, l);
                mk("msg_fwd_last", st);
            } else {
                k_msg_fwd<T, false><<<nb, kAT, 0, st>>>(md, gr, ws, l);
                mk("msg_fwd", st);
            }
        }
        for (int l = M - 2; l >= 0; --l) {
            k_msg_bwd<T><<<nb, kAT, 0, st>>>(md, gr, ws, l);
            mk("msg_bwd", st);
        }
        k_embed_bwd<T><<<nb, kAT, 0, st>>>(md, gr, ws);
        mk("embed_bwd", st);
        launches += 2 + M + (M - 1);
    }
    k_force<T><<<nb, kAT, 0, st>>>(gr, ws, forces, per_atom, out, mf);
    mk("force", st);
    return launches + 1;
}
template int launch_network<float>(const DevModel<float>&, const DevGraph&, const DevWork<float>&,
                                   double*, double*, double*, int*, cudaStream_t, const Marker&,
                                   const MdFuse&);
template int launch_network<double>(const DevModel<double>&, const DevGraph&,
                                    const DevWork<double>&, double*, double*, double*, int*,
                                    cudaStream_t, const Marker&, const MdFuse&);

}  // namespace hmdp
