// hmdp_net.cu — the DP network kernels (embedding, message layers, fitting,
// reverse mode, forces/virial), sm_100a.
//
// Decomposition: a 512-thread CTA holds four independent 128-thread "atom
// groups"; each group processes one atom at a time (grid-stride over atoms) and
// synchronises with its own named barrier, so the groups never wait on each
// other.  Kernels stage the MLP weights they need into shared memory (once per
// CTA, ~1 CTA per SM), so the atom-level mat-vecs (bmv: 4-way split, xor-shuffle
// reduction) read weights and activations from shared memory only.  Per-edge
// work is split over the group's 4 warps (edge q -> warp q % 4) with lane =
// channel, so every per-edge row access is one coalesced 128-byte line; the
// per-edge scalars are staged in shared memory and read as broadcasts.
//
// Every phase is a per-group __device__ body (grid-stride over atoms) wrapped by
// a thin kernel that stages the weights it needs.
//
// Dataflow is "push" into mirror slots (DevGraph, hmdp_device.cuh): the producer
// of a per-neighbour quantity writes it into the slot its consumer reads
// contiguously, so no kernel chases an index to gather a neighbour's row:
//   P_j = W1h h_j        pushed by j into the out-slots of j's in-edges
//   dz_e (h_j adjoint)   pushed by the edge's source into e's mirror slot
//   g_e                  pushed by the edge's source into e's mirror slot
// Every slot is written by exactly one thread and every sum runs in a fixed
// order: deterministic, no float atomics (the reference's scatters dh_j += ...,
// F_j -= ..., inference.cpp:343, :380, become these pushes + local sums).
//
// Linearity of the message MLP is exploited exactly (same function, fewer FLOPs):
//   forward   z_e = tanh(W1h h_j + W1b b_e + b1) with the per-ATOM projection
//             P_j = W1h h_j computed once per layer instead of once per edge;
//             msum_i = sum_e s_e (W2 z_e + b2) = W2 (sum_e s_e z_e) + (sum_e s_e) b2
//   backward  with dmsum_i from the update MLP, v = W2^T dmsum_i, c0 = dmsum_i.b2:
//             dsc_e = dmsum_i . mo_e = v . z_e + c0,  dz_e = s_e v (1 - z_e^2),
//             dE/dr_e += dsc_e s'(r_e) + sum_k b'_e[k] (W1b^T dz_e)[k],
//             dE/dh_j += W1h^T sum_{e in in(j)} dz_e  (one mat-vec per atom).
//
// Reference correspondence (paths relative to /root/reference/proj):
//   embed_body       edge radial + descriptor + embedding fwd   src/nn/inference.cpp:214-249
//                    [FUSE_FIT: + fitting fwd/bwd + embedding bwd, :288-311, :355-370]
//   msg_fwd_body     message layer fwd                          :251-286
//                    [LAST: + fitting fwd/bwd + top message layer bwd, :288-353]
//   msg_bwd_body     message layer bwd (lower layers)           :313-353
//   embed_bwd_body   embedding + descriptor adjoint             :355-370
//   force_body       force / virial (gather form) + E, W sums   :288-298, :372-387
//                    [+ velocity Verlet tail, src/integrators.cpp:32-47]
#include "hmdp_common.cuh"

namespace hmdp {

int num_sms();  // hmdp_nbr.cu

constexpr int kG = 4;             // atom groups per CTA
constexpr int kCTA = kG * kAT;    // 512 threads
constexpr int kEdgePass = 64;     // edges per pass of a group (16 per warp)
constexpr int kPW = kEdgePass / 4;

// group-local barrier (named barrier 1 + g over the group's 128 threads)
__device__ __forceinline__ void gsync(int g) { group_bar(g + 1); }

// Sum over a group's 128 threads (every thread gets the total); fixed order.
template <typename T>
__device__ __forceinline__ T group_sum(T v, T* s4, int g) {
    v = warp_sum(v);
    gsync(g);
    if ((threadIdx.x & 31) == 0) s4[(threadIdx.x >> 5) & 3] = v;
    gsync(g);
    return ((s4[0] + s4[1]) + s4[2]) + s4[3];
}

// Per-group shared scratch for one atom.
template <typename T>
struct AtomSmem {
    T v0[64], v1[64], v2[64], v3[64];  // activation vectors
    T part[4][32];                     // per-warp partial channel sums
    T s4[4];                           // group_sum scratch
    T sc[4];                           // per-warp scalar partials
    alignas(16) T ed[4][16][12];       // per-warp staged edge scalars (s, s', b or b')
    int emir[4][16];                   // per-warp staged mirror slots
    double f[4][3];                    // per-warp force partials
};

// ---------------------------------------------------------------------------
// Weight staging: whole MLPs [in, 32, out] copied to shared memory.
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int mlp_elems(int in, int out) {
    return 32 * in + in * 32 + 32 + ((out * 32 + 3) / 4) * 4 * 2 + ((out + 3) / 4) * 4;
}
constexpr int kInEmbed = 32, kInFit = 32, kInMsg = kH + kK, kInUpd = 2 * kH;

template <typename T>
struct Stager {
    T* base;
    int off;
    __device__ const T* put(const T* src, int count) {
        T* dst = base + off;
        for (int q = threadIdx.x * 4; q < count; q += kCTA * 4) {
            const V4<T> v = ld4(src + q);
            st4(dst + q, v.x, v.y, v.z, v.w);
        }
        off += (count + 3) / 4 * 4;
        return dst;
    }
    // per-group scratch placed after the staged weights (same dynamic region)
    template <class S>
    __device__ S* scratch(int skip_bytes = 0) const {
        const size_t a = (reinterpret_cast<size_t>(base + off) + 15) & ~size_t(15);
        return reinterpret_cast<S*>(a + skip_bytes);
    }
    __device__ DevMlp<T> mlp(const DevMlp<T>& m, int in, int out) {
        DevMlp<T> d;
        d.W1 = put(m.W1, 32 * in);
        d.W1T = put(m.W1T, in * 32);
        d.b1 = put(m.b1, 32);
        d.W2 = put(m.W2, (out * 32 + 3) / 4 * 4);
        d.W2T = put(m.W2T, (32 * out + 3) / 4 * 4);
        d.b2 = put(m.b2, (out + 3) / 4 * 4);
        return d;
    }
};
// (the device weight buffer pads every array to a multiple of 32 elements, so
// the rounded-up copies above never read past an array's allocation)

// Group coordinates of this thread.
struct Grp {
    int g, t, gid, ngroups;
    __device__ Grp()
        : g(threadIdx.x / kAT),
          t(threadIdx.x % kAT),
          gid(blockIdx.x * kG + threadIdx.x / kAT),
          ngroups(gridDim.x * kG) {}
};

// Push a 32-vector (smem) into the rows `dst + in_edge[in_start + k] * 32` for
// k < in_cnt (the out-slots of i's in-edges): 4 rows per group iteration.
template <typename T>
__device__ __forceinline__ void push_rows(T* __restrict__ dst, const T* vec, const DevGraph& gr,
                                          int i, int t) {
    const int is = gr.in_start[i], ic = gr.in_cnt[i];
    const T v = vec[t & 31];
    for (int k = t >> 5; k < ic; k += 4) {
        const long long slot = gr.in_edge[is + k];
        dst[slot * kH + (t & 31)] = v;
    }
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

// ---------------------------------------------------------------------------
// Fitting net forward + backward on h_s: writes e_i for owned atoms (0 for
// ghosts), leaves dE/dh (0 for ghosts) in dh_s.  inference.cpp:288-311.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void fit_fwd_bwd(const DevMlp<T>& fit, const T* h_s, T* z_s, T* dz_s,
                                            T* dh_s, bool owned, double* e_out, T* s4, int t,
                                            int g) {
    const int o = bmv_out<32>(t);
    const bool lead = bmv_lead<32>(t);
    const T zf = d_tanh(bmv<T, 32, 32>(fit.W1, 32, h_s, t) + fit.b1[o]);
    if (lead) z_s[o] = zf;
    gsync(g);
    // linear head 32 -> 1 and its adjoint (dout = 1)
    const T ez = (t < 32) ? fit.W2[t] * z_s[t] : T(0);
    const T e = group_sum(ez, s4, g) + fit.b2[0];
    if (t == 0) *e_out = owned ? static_cast<double>(e) : 0.0;
    if (t < 32) dz_s[t] = (fit.W2[t] * T(1)) * (T(1) - z_s[t] * z_s[t]);
    gsync(g);
    const T dh = bmv<T, 32, 32>(fit.W1T, 32, dz_s, t);
    gsync(g);  // dh_s may alias dz_s
    if (lead) dh_s[o] = owned ? dh : T(0);
    gsync(g);
}

// ---------------------------------------------------------------------------
// Edge radial features + descriptor + embedding; pushes P^0 (message layer 0's
// neighbour projection) or, for depth 1 (FUSE_FIT), runs the whole fitting and
// backward chain.  rev (periodic path): computes the reverse slot of every
// edge, which is the in-edge array of the symmetric graph (in_edge == rev).
// `second` is the fitting net (FUSE_FIT) or message layer 0 (otherwise).
// ---------------------------------------------------------------------------
template <typename T, bool FUSE_FIT>
__device__ void embed_body(const DevModel<T>& md, const DevMlp<T>& emb, const DevMlp<T>& second,
                           const DevGraph& gr, const DevWork<T>& ws, int* __restrict__ rev,
                           const MdFuse& mf, AtomSmem<T>* sms, const Grp& G) {
    // this step's neighbour search is complete: clear the cell counts for the
    // binning fused into the force phase (device MD) / keep the zero invariant
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < mf.n_cells_zero;
         c += gridDim.x * blockDim.x)
        mf.cell_count[c] = 0;
    const int g = G.g, t = G.t, lane = t & 31, w = t >> 5;
    AtomSmem<T>& sm = sms[g];
    T(*s_b)[kK + 1] = reinterpret_cast<T(*)[kK + 1]>(&sm.ed[0][0][0]);  // [64][9] alias
    int* s_ty = &sm.emir[0][0];                                          // [64] alias
    const int nd = md.n_types * kK;
    const int o = bmv_out<32>(t);
    const bool lead = bmv_lead<32>(t);
    for (int i = G.gid; i < gr.n_active; i += G.ngroups) {
        const int start = gr.row_start[i], cnt = gr.nnei[i];
        T desc = T(0);  // thread q < nd accumulates descriptor component q
        for (int base = 0; base < cnt; base += kEdgePass) {
            const int m = min(kEdgePass, cnt - base);
            const int e = start + base + t;
            int j = 0;
            if (t < m) {
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
                ws.er[e] = r;
                ws.es[e] = s;
                ws.eds[e] = ds;
                st4(ws.eb + 8ll * e, b[0], b[1], b[2], b[3]);
                st4(ws.eb + 8ll * e + 4, b[4], b[5], b[6], b[7]);
                st4(ws.edb + 8ll * e, db[0], db[1], db[2], db[3]);
                st4(ws.edb + 8ll * e + 4, db[4], db[5], db[6], db[7]);
#pragma unroll
                for (int k = 0; k < kK; ++k) s_b[t][k] = b[k];
                s_ty[t] = gr.ety[e];
            }
            if (rev && w < 2) {
                // rev(e) = slot of i in nbr(j) (symmetric, sorted list).  Lane l of the
                // warp owning edges [32w, 32w+32) reads entry l of each neighbour's
                // list (one memory latency per 8 edges); a ballot finds i.
                const int mw = min(32, max(0, m - 32 * w));
                const int rs_l = t < m ? gr.row_start[j] : 0;
                const int nn_l = t < m ? gr.nnei[j] : 0;
                int found = -1;
                for (int q0 = 0; q0 < mw; q0 += 8) {
                    int val[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int rsq = __shfl_sync(FULL_MASK, rs_l, q0 + u);
                        const int nnq = __shfl_sync(FULL_MASK, nn_l, q0 + u);
                        val[u] = (q0 + u < mw && lane < nnq) ? gr.nbr[rsq + lane] : -1;
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const unsigned bal = __ballot_sync(FULL_MASK, val[u] == i);
                        if (lane == q0 + u && bal) found = rs_l + __ffs(bal) - 1;
                    }
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
            gsync(g);
            if (t < nd) {  // descriptor: CSR edge order, as inference.cpp:228-238
                const int ty = t >> 3, k = t & 7;
                for (int r = 0; r < m; ++r) desc += (s_ty[r] == ty) ? s_b[r][k] : T(0);
            }
            gsync(g);
        }
        if (t < 32) {
            sm.v0[t] = t < nd ? desc : T(0);
            if (t < nd) ws.desc[static_cast<long long>(i) * 32 + t] = desc;
        }
        gsync(g);
        // embedding forward nd (zero-padded to 32) -> 32 (tanh) -> 32
        const T z1 = d_tanh(bmv<T, 32, 32>(emb.W1, 32, sm.v0, t) + emb.b1[o]);
        if (lead) {
            sm.v1[o] = z1;
            ws.ez1[static_cast<long long>(i) * kH + o] = z1;
        }
        gsync(g);
        const T h0 = bmv<T, 32, 32>(emb.W2, 32, sm.v1, t) + emb.b2[o];
        if (lead) {
            sm.v2[o] = h0;
            ws.h[static_cast<long long>(i) * kH + o] = h0;
        }
        gsync(g);
        if constexpr (FUSE_FIT) {
            const bool owned = !(gr.is_ghost && gr.is_ghost[i]);
            fit_fwd_bwd(second, sm.v2, sm.v3, sm.v0, sm.v3, owned, ws.e_atom + i, sm.s4, t, g);
            // embedding backward: linear layer 2 (W2^T), tanh layer 1 (W1^T, padded)
            const T dz1 = bmv<T, 32, 32>(emb.W2T, 32, sm.v3, t) * (T(1) - z1 * z1);
            if (lead) sm.v0[o] = dz1;
            gsync(g);
            const T dd = bmv<T, 32, 32>(emb.W1T, 32, sm.v0, t);
            if (lead) sm.v1[o] = dd;
            gsync(g);
            for (int q = t; q < cnt; q += kAT) {
                const long long e = start + q;
                const V4<T> d0 = ld4c(ws.edb + 8 * e), d1 = ld4c(ws.edb + 8 * e + 4);
                const T* dv = sm.v1 + gr.ety[e] * kK;
                T acc = dv[0] * d0.x;
                acc += dv[1] * d0.y;
                acc += dv[2] * d0.z;
                acc += dv[3] * d0.w;
                acc += dv[4] * d1.x;
                acc += dv[5] * d1.y;
                acc += dv[6] * d1.z;
                acc += dv[7] * d1.w;
                ws.g[e] = acc;
                ws.grev[gr.inv_pos[e]] = acc;  // mirror for the force gather
            }
        } else {
            // P^0 = W1h^(0) h^0, pushed into the out-slots of i's in-edges
            const T p = bmv<T, 32, 32>(second.W1, kInMsg, sm.v2, t);
            if (lead) {
                sm.v3[o] = p;
                if (ws.p_atom) ws.p_atom[static_cast<long long>(i) * kH + o] = p;
            }
            gsync(g);
            push_rows(ws.pe, sm.v3, gr, i, t);
        }
        gsync(g);
    }
}

// ---------------------------------------------------------------------------
// Message-layer backward for atom i, given dE/dh^{l+1}_i in sm.v0 and the
// update hidden activations in sm.v2.  Pushes dz_e to e's mirror slot.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void msg_backward_atom(const DevMlp<T>& msg, const DevMlp<T>& upd,
                                                  const DevGraph& gr, const DevWork<T>& ws,
                                                  AtomSmem<T>& sm, int l, int i, bool first_g,
                                                  int t, int g) {
    const int lane = t & 31, w = t >> 5;
    const long long S = ws.slots;
    const int o = bmv_out<32>(t);
    const bool lead = bmv_lead<32>(t);
    // update MLP backward (64 -> 32 tanh -> 32)
    const T zu = sm.v2[o];
    const T dz = bmv<T, 32, 32>(upd.W2T, 32, sm.v0, t) * (T(1) - zu * zu);
    if (lead) sm.v3[o] = dz;
    gsync(g);
    const T din = bmv<T, 64, 32>(upd.W1T, 32, sm.v3, t);  // 64 outputs, 2 parts each
    if (bmv_lead<64>(t)) {
        const int k = bmv_out<64>(t);
        if (k < kH)
            ws.dhown[static_cast<long long>(i) * kH + k] = sm.v0[k] + din;  // residual + update
        else
            sm.v1[k - kH] = din;  // dmsum
    }
    gsync(g);
    const T v = bmv<T, 32, 32>(msg.W2T, 32, sm.v1, t);  // v = W2^T dmsum
    if (lead) sm.v2[o] = v;
    const T c0 = group_sum(t < 32 ? sm.v1[t] * msg.b2[t] : T(0), sm.s4, g);
    // (group_sum's barriers also publish sm.v2)
    T w1b[kK];
#pragma unroll
    for (int k = 0; k < kK; ++k) w1b[k] = msg.W1T[(kH + k) * kH + lane];
    const T vl = sm.v2[lane];
    const T* Z = ws.z + l * S * kH;
    T* __restrict__ D = ws.d + (l & 1) * S * kH;
    const int start = gr.row_start[i], cnt = gr.nnei[i];
    for (int base = 0; base < cnt; base += kEdgePass) {
        // warp w owns edges base + w + 4u, taken 8 at a time
        const int mw = max(0, (min(kEdgePass, cnt - base) - w + 3) / 4);
        for (int u0 = 0; u0 < mw; u0 += 8) {
            const int mu = min(8, mw - u0);
            const long long e0 = start + base + w + 4 * u0;  // edge of u = 0
            // lane u stages edge u's scalars (one memory round trip for the batch);
            // the edge loop then reads them as shared-memory broadcasts
            if (lane < mu) {
                const long long e = e0 + 4 * lane;
                T* row = sm.ed[w][lane];
                row[0] = ws.es[e];
                row[1] = ws.eds[e];
                const V4<T> d0 = ld4c(ws.edb + 8 * e), d1 = ld4c(ws.edb + 8 * e + 4);
                st4(row + 4, d0.x, d0.y, d0.z, d0.w);
                st4(row + 8, d1.x, d1.y, d1.z, d1.w);
                sm.emir[w][lane] = gr.inv_pos[e];
            }
            const T* zrow = Z + e0 * kH + lane;
            T zr[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (u < mu) zr[u] = zrow[4 * u * kH];
            __syncwarp();
            T term[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                term[u] = T(0);
                if (u < mu) {
                    const T* row = sm.ed[w][u];
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
                    const T z = zr[u];
                    const T d = s * vl * (T(1) - z * z);
                    D[static_cast<long long>(sm.emir[w][u]) * kH + lane] = d;
                    term[u] = ds * vl * z + d * wv;
                }
            }
            // reduce-scatter butterfly: 8 edge sums in 9 shuffles; lane 4u holds edge u
            const T tot = reduce8(term, lane);
            if ((lane & 3) == 0 && (lane >> 2) < mu) {
                const long long e = e0 + 4 * (lane >> 2);
                ws.g[e] = (first_g ? T(0) : ws.g[e]) + (tot + sm.ed[w][lane >> 2][1] * c0);
            }
            __syncwarp();
        }
    }
}

// S_i = sum over i's mirror slots of the pushed dz (layer l) (+ remote partials
// in domain decomposition) -> sm.v1; contiguous rows, fixed summation order.
template <typename T>
__device__ __forceinline__ void gather_in(const DevGraph& gr, const DevWork<T>& ws,
                                          AtomSmem<T>& sm, int l, int i, int t, int g) {
    const int lane = t & 31, w = t >> 5;
    const T* D = ws.d + (l & 1) * ws.slots * kH;
    const int is = gr.in_start[i], ic = gr.in_cnt[i];
    T acc = T(0);
    for (int base = 0; base < ic; base += kEdgePass) {
        const int mw = max(0, (min(kEdgePass, ic - base) - w + 3) / 4);
        const T* drow = D + static_cast<long long>(is + base + w) * kH + lane;
        T dr_[kPW];
#pragma unroll
        for (int u = 0; u < kPW; ++u)
            if (u < mw) dr_[u] = drow[4 * u * kH];
#pragma unroll
        for (int u = 0; u < kPW; ++u)
            if (u < mw) acc += dr_[u];
    }
    sm.part[w][lane] = acc;
    gsync(g);
    if (t < 32) {
        T s = ((sm.part[0][t] + sm.part[1][t]) + sm.part[2][t]) + sm.part[3][t];
        // domain decomposition: partial sums pushed to ghost copies of i on other ranks
        if (ws.s_remote) s += ws.s_remote[static_cast<long long>(i) * kH + t];
        sm.v1[t] = s;
    }
    gsync(g);
}

// ---------------------------------------------------------------------------
// Message layer l forward; LAST fuses the fitting net and the top layer's
// backward (all atom-local).  `third` is message layer l+1 (for P^{l+1}) or the
// fitting net (LAST).
// ---------------------------------------------------------------------------
template <typename T, bool LAST>
__device__ void msg_fwd_body(const DevMlp<T>& msg, const DevMlp<T>& upd, const DevMlp<T>& third,
                             const DevGraph& gr, const DevWork<T>& ws, int l, AtomSmem<T>* sms,
                             const Grp& G) {
    const int g = G.g, t = G.t, lane = t & 31, w = t >> 5;
    AtomSmem<T>& sm = sms[g];
    const int n = gr.n;
    const long long S = ws.slots;
    const T* Pin = ws.pe + (l & 1) * S * kH;
    T* __restrict__ Z = ws.z + l * S * kH;
    T w1b[kK];
#pragma unroll
    for (int k = 0; k < kK; ++k) w1b[k] = msg.W1T[(kH + k) * kH + lane];
    const T b1 = msg.b1[lane];
    const int o = bmv_out<32>(t);
    const bool lead = bmv_lead<32>(t);
    for (int i = G.gid; i < gr.n_active; i += G.ngroups) {
        const int start = gr.row_start[i], cnt = gr.nnei[i];
        if (t < 32) sm.v1[t] = ws.h[(static_cast<long long>(l) * n + i) * kH + t];  // h_i
        T acc = T(0), ssum = T(0);
        for (int base = 0; base < cnt; base += kEdgePass) {
            const int mw = max(0, (min(kEdgePass, cnt - base) - w + 3) / 4);
            const long long e0 = start + base + w;
            // lane u stages edge u's scalars (one memory round trip for the pass);
            // the edge loop reads them as shared-memory broadcasts
            if (lane < mw) {
                const long long e = e0 + 4 * lane;
                T* row = sm.ed[w][lane];
                row[0] = ws.es[e];
                const V4<T> b0 = ld4c(ws.eb + 8 * e), bb = ld4c(ws.eb + 8 * e + 4);
                st4(row + 4, b0.x, b0.y, b0.z, b0.w);
                st4(row + 8, bb.x, bb.y, bb.z, bb.w);
            }
            const T* prow = Pin + e0 * kH + lane;
            T pr[kPW];
#pragma unroll
            for (int u = 0; u < kPW; ++u)
                if (u < mw) pr[u] = prow[4 * u * kH];
            __syncwarp();
#pragma unroll
            for (int u = 0; u < kPW; ++u) {
                if (u >= mw) break;
                const long long e = e0 + 4 * u;
                const T* row = sm.ed[w][u];
                const T s = row[0];
                const V4<T> b0 = ld4c(row + 4), bb = ld4c(row + 8);
                T a = b1;
                a += w1b[0] * b0.x;
                a += w1b[1] * b0.y;
                a += w1b[2] * b0.z;
                a += w1b[3] * b0.w;
                a += w1b[4] * bb.x;
                a += w1b[5] * bb.y;
                a += w1b[6] * bb.z;
                a += w1b[7] * bb.w;
                const T z = d_tanh(a + pr[u]);
                Z[e * kH + lane] = z;
                acc += s * z;
                ssum += s;
            }
            __syncwarp();
        }
        sm.part[w][lane] = acc;
        if (lane == 0) sm.sc[w] = ssum;
        gsync(g);
        if (t < 32) sm.v0[t] = ((sm.part[0][t] + sm.part[1][t]) + sm.part[2][t]) + sm.part[3][t];
        const T stot = ((sm.sc[0] + sm.sc[1]) + sm.sc[2]) + sm.sc[3];
        gsync(g);
        // msum = W2 (sum_e s_e z_e) + (sum_e s_e) b2  -> second half of the update input
        const T msum = bmv<T, 32, 32>(msg.W2, 32, sm.v0, t) + stot * msg.b2[o];
        if (lead) sm.v1[kH + o] = msum;
        gsync(g);
        // update MLP on [h_i, msum] (64 -> 32 tanh -> 32), residual
        const T zu = d_tanh(bmv<T, 32, 64>(upd.W1, kInUpd, sm.v1, t) + upd.b1[o]);
        if (lead) {
            sm.v2[o] = zu;
            ws.uz1[(static_cast<long long>(l) * n + i) * kH + o] = zu;
        }
        gsync(g);
        const T hn = sm.v1[o] + (bmv<T, 32, 32>(upd.W2, 32, sm.v2, t) + upd.b2[o]);
        if (lead) {
            sm.v3[o] = hn;
            ws.h[(static_cast<long long>(l + 1) * n + i) * kH + o] = hn;
        }
        gsync(g);
        if constexpr (!LAST) {
            const T p = bmv<T, 32, 32>(third.W1, kInMsg, sm.v3, t);
            if (lead) {
                sm.v0[o] = p;
                if (ws.p_atom) ws.p_atom[static_cast<long long>(i) * kH + o] = p;
            }
            gsync(g);
            push_rows(ws.pe + ((l + 1) & 1) * S * kH, sm.v0, gr, i, t);
        } else {
            const bool owned = !(gr.is_ghost && gr.is_ghost[i]);
            // fitting: h^M in v3 -> dE/dh^M in v0 (v1 scratch for the fit hidden layer)
            fit_fwd_bwd(third, sm.v3, sm.v1, sm.v0, sm.v0, owned, ws.e_atom + i, sm.s4, t, g);
            msg_backward_atom(msg, upd, gr, ws, sm, l, i, true, t, g);
        }
        gsync(g);
    }
}

// Message layer l < M-1 backward: gather dE/dh^{l+1}, then the layer body.
// `nxt` is message layer l+1 (its W1h^T maps the gathered adjoints).
template <typename T>
__device__ void msg_bwd_body(const DevMlp<T>& msg, const DevMlp<T>& upd, const DevMlp<T>& nxt,
                             const DevGraph& gr, const DevWork<T>& ws, int l, AtomSmem<T>* sms,
                             const Grp& G) {
    const int g = G.g, t = G.t;
    AtomSmem<T>& sm = sms[g];
    const int o = bmv_out<32>(t);
    const bool lead = bmv_lead<32>(t);
    for (int i = G.gid; i < gr.n_active; i += G.ngroups) {
        const T own = ws.dhown[static_cast<long long>(i) * kH + o];
        const T zu = ws.uz1[(static_cast<long long>(l) * gr.n + i) * kH + o];
        gather_in(gr, ws, sm, l + 1, i, t, g);
        // dE/dh^{l+1}_i = own + W1h^(l+1)^T S_i
        const T dh = own + bmv<T, 32, 32>(nxt.W1T, 32, sm.v1, t);
        if (lead) {
            sm.v0[o] = dh;
            sm.v2[o] = zu;
        }
        gsync(g);
        msg_backward_atom(msg, upd, gr, ws, sm, l, i, false, t, g);
        gsync(g);
    }
}

// Embedding backward + descriptor adjoint (depth > 1); pushes g to the mirrors.
template <typename T>
__device__ void embed_bwd_body(const DevMlp<T>& emb, const DevMlp<T>& msg0, const DevGraph& gr,
                               const DevWork<T>& ws, AtomSmem<T>* sms, const Grp& G) {
    const int g = G.g, t = G.t;
    AtomSmem<T>& sm = sms[g];
    const int o = bmv_out<32>(t);
    const bool lead = bmv_lead<32>(t);
    for (int i = G.gid; i < gr.n_active; i += G.ngroups) {
        const T own = ws.dhown[static_cast<long long>(i) * kH + o];
        const T z1 = ws.ez1[static_cast<long long>(i) * kH + o];
        gather_in(gr, ws, sm, 0, i, t, g);
        const T dh = own + bmv<T, 32, 32>(msg0.W1T, 32, sm.v1, t);
        if (lead) sm.v0[o] = dh;
        gsync(g);
        const T dz1 = bmv<T, 32, 32>(emb.W2T, 32, sm.v0, t) * (T(1) - z1 * z1);
        if (lead) sm.v2[o] = dz1;
        gsync(g);
        const T dd = bmv<T, 32, 32>(emb.W1T, 32, sm.v2, t);
        if (lead) sm.v3[o] = dd;
        gsync(g);
        const int start = gr.row_start[i], cnt = gr.nnei[i];
        for (int q = t; q < cnt; q += kAT) {
            const long long e = start + q;
            const V4<T> d0 = ld4c(ws.edb + 8 * e), d1 = ld4c(ws.edb + 8 * e + 4);
            const T* dv = sm.v3 + gr.ety[e] * kK;
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
            ws.grev[gr.inv_pos[e]] = gv;  // mirror for the force gather
        }
        gsync(g);
    }
}

// ---------------------------------------------------------------------------
// Forces (gather form), per-atom energy, virial, and the velocity-Verlet tail
// of the device MD loop; accumulates this thread's E, W, W_ab into acc[11].
//   F_i = sum_{e in out(i)} u_e g_e - sum_{e' in in(i)} u_e' g_e'
//       = sum_q u_q (g_q + grev_q)            (symmetric list: u_rev(e) = -u_e)
//   W   = -sum_e g_e r_e ;  W_ab = -sum_e g_e dr_a u_b
// ---------------------------------------------------------------------------
template <typename T>
__device__ void force_body(const DevGraph& gr, const DevWork<T>& ws, double* __restrict__ forces,
                           double* __restrict__ per_atom, const MdFuse& mf, AtomSmem<T>* sms,
                           double (&acc)[11], const Grp& G) {
    const int g = G.g, t = G.t, lane = t & 31, w = t >> 5;
    AtomSmem<T>& sm = sms[g];
    for (int i = G.gid; i < gr.n; i += G.ngroups) {
        // MD state of atom i, loaded early (independent of the edge loads)
        double xv[3] = {0, 0, 0}, vv[3] = {0, 0, 0}, mi = 1.0;
        if (mf.mode && t == 0) {
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                vv[a] = mf.v[3 * i + a];
                xv[a] = mf.x[3 * i + a];
            }
            mi = mf.m[i];
        }
        double fx = 0.0, fy = 0.0, fz = 0.0;
        const int start = gr.row_start[i], cnt = gr.nnei[i];
        for (int q = t; q < cnt; q += kAT) {
            const int e = start + q;
            const T gg = ws.g[e];
            const T gm = gr.sym ? ws.grev[e] : T(0);
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
        if (!gr.sym) {  // generic CSR: the pushed g of each in-edge, its own geometry
            const int is = gr.in_start[i], ic = gr.in_cnt[i];
            for (int q = t; q < ic; q += kAT) {
                const int e = gr.in_edge[is + q];
                const T gg = ws.grev[is + q];
                T x, y, z;
                const T r = edge_len<T>(gr.dr + 3ll * e, x, y, z);
                fx -= static_cast<double>((x / r) * gg);
                fy -= static_cast<double>((y / r) * gg);
                fz -= static_cast<double>((z / r) * gg);
            }
        }
        fx = warp_sum(fx);
        fy = warp_sum(fy);
        fz = warp_sum(fz);
        if (lane == 0) {
            sm.f[w][0] = fx;
            sm.f[w][1] = fy;
            sm.f[w][2] = fz;
        }
        gsync(g);
        if (t == 0) {
            double f3[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) f3[a] = ((sm.f[0][a] + sm.f[1][a]) + sm.f[2][a]) + sm.f[3][a];
            forces[3 * i] = f3[0];
            forces[3 * i + 1] = f3[1];
            forces[3 * i + 2] = f3[2];
            const double ei = ws.e_atom[i];
            if (per_atom) per_atom[i] = ei;
            acc[0] += ei;
            if (mf.mode) {
                const double s = mf.half / mi;
                const bool finite = isfinite(f3[0]) && isfinite(f3[1]) && isfinite(f3[2]);
                if (!finite) atomicOr(ws.err, kErrNonFinite);
                double x3[3];
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    double va = __dadd_rn(vv[a], __dmul_rn(f3[a], s));  // closing kick
                    if (mf.mode == 2) {
                        va = __dadd_rn(va, __dmul_rn(f3[a], s));  // next step's opening kick
                        x3[a] = __dadd_rn(xv[a], __dmul_rn(va, mf.dt));
                        mf.x[3 * i + a] = x3[a];
                    }
                    mf.v[3 * i + a] = va;
                }
                if (mf.mode == 2)
                    bin_atom(i, x3, mf.cg, mf.cell_count, mf.members, mf.cell_of, ws.err);
            }
        }
        gsync(g);
    }
}

// CTA partials of (E, W, W_ab) in a fixed order, then the last CTA to finish
// reduces all CTAs' partials in a fixed order into out[0..10] (deterministic).
template <typename T>
__device__ void reduce_energy_virial(double (&acc)[11], const DevWork<T>& ws,
                                     double* __restrict__ out, double (*s_part)[12], bool* s_last) {
    const int lane = threadIdx.x & 31, wc = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < 11; ++q) acc[q] = warp_sum(acc[q]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < 11; ++q) s_part[wc][q] = acc[q];
    __syncthreads();
    if (threadIdx.x < 11) {
        double v = 0.0;
        for (int q = 0; q < kCTA / 32; ++q) v += s_part[q][threadIdx.x];
        ws.partial[blockIdx.x * 16 + threadIdx.x] = v;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) *s_last = (atomicAdd(ws.ticket, 1u) == gridDim.x - 1);
    __syncthreads();
    if (*s_last) {
        __threadfence();
        double v[11];
#pragma unroll
        for (int q = 0; q < 11; ++q) v[q] = 0.0;
        for (unsigned b = threadIdx.x; b < gridDim.x; b += kCTA)
#pragma unroll
            for (int q = 0; q < 11; ++q) v[q] += __ldcg(ws.partial + b * 16 + q);
#pragma unroll
        for (int q = 0; q < 11; ++q) v[q] = warp_sum(v[q]);
        __syncthreads();
        if (lane == 0)
#pragma unroll
            for (int q = 0; q < 11; ++q) s_part[wc][q] = v[q];
        __syncthreads();
        if (threadIdx.x < 11) {
            double tot = 0.0;
            for (int q = 0; q < kCTA / 32; ++q) tot += s_part[q][threadIdx.x];
            out[threadIdx.x] = tot;
        }
        if (threadIdx.x == 0) *ws.ticket = 0u;  // re-arm for the next launch / step
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// Standalone kernels (one phase each; weights staged per launch)
// ---------------------------------------------------------------------------
template <typename T, bool FUSE_FIT>
__global__ __launch_bounds__(kCTA, 1) void k_embed(DevModel<T> md, DevGraph gr, DevWork<T> ws,
                                                   int* __restrict__ rev, MdFuse mf) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    pdl_launch_dependents();
    Stager<T> sg{reinterpret_cast<T*>(smem_raw), 0};
    const DevMlp<T> emb = sg.mlp(md.embed, kInEmbed, kH);
    const DevMlp<T> second =
        FUSE_FIT ? sg.mlp(md.fit, kInFit, 1) : sg.mlp(md.msg[0], kInMsg, kH);
    __syncthreads();
    pdl_wait();
    embed_body<T, FUSE_FIT>(md, emb, second, gr, ws, rev, mf,
                            sg.template scratch<AtomSmem<T>>(), Grp());
}

template <typename T, bool LAST>
__global__ __launch_bounds__(kCTA, 1) void k_msg_fwd(DevModel<T> md, DevGraph gr, DevWork<T> ws,
                                                     int l) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    pdl_launch_dependents();
    Stager<T> sg{reinterpret_cast<T*>(smem_raw), 0};
    const DevMlp<T> msg = sg.mlp(md.msg[l], kInMsg, kH);
    const DevMlp<T> upd = sg.mlp(md.upd[l], kInUpd, kH);
    const DevMlp<T> third = LAST ? sg.mlp(md.fit, kInFit, 1) : sg.mlp(md.msg[l + 1], kInMsg, kH);
    __syncthreads();
    pdl_wait();
    msg_fwd_body<T, LAST>(msg, upd, third, gr, ws, l, sg.template scratch<AtomSmem<T>>(), Grp());
}

template <typename T>
__global__ __launch_bounds__(kCTA, 1) void k_msg_bwd(DevModel<T> md, DevGraph gr, DevWork<T> ws,
                                                     int l) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    pdl_launch_dependents();
    Stager<T> sg{reinterpret_cast<T*>(smem_raw), 0};
    const DevMlp<T> msg = sg.mlp(md.msg[l], kInMsg, kH);
    const DevMlp<T> upd = sg.mlp(md.upd[l], kInUpd, kH);
    const DevMlp<T> nxt = sg.mlp(md.msg[l + 1], kInMsg, kH);
    __syncthreads();
    pdl_wait();
    msg_bwd_body<T>(msg, upd, nxt, gr, ws, l, sg.template scratch<AtomSmem<T>>(), Grp());
}

template <typename T>
__global__ __launch_bounds__(kCTA, 1) void k_embed_bwd(DevModel<T> md, DevGraph gr, DevWork<T> ws) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    pdl_launch_dependents();
    Stager<T> sg{reinterpret_cast<T*>(smem_raw), 0};
    const DevMlp<T> emb = sg.mlp(md.embed, kInEmbed, kH);
    const DevMlp<T> msg0 = sg.mlp(md.msg[0], kInMsg, kH);
    __syncthreads();
    pdl_wait();
    embed_bwd_body<T>(emb, msg0, gr, ws, sg.template scratch<AtomSmem<T>>(), Grp());
}

template <typename T>
__global__ __launch_bounds__(kCTA, 1) void k_force(DevGraph gr, DevWork<T> ws,
                                                   double* __restrict__ forces,
                                                   double* __restrict__ per_atom,
                                                   double* __restrict__ out, MdFuse mf) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double s_part[kCTA / 32][12];
    __shared__ bool s_last;
    pdl_launch_dependents();
    pdl_wait();
    double acc[11];
#pragma unroll
    for (int q = 0; q < 11; ++q) acc[q] = 0.0;
    force_body<T>(gr, ws, forces, per_atom, mf, reinterpret_cast<AtomSmem<T>*>(smem_raw), acc,
                  Grp());
    reduce_energy_virial<T>(acc, ws, out, s_part, &s_last);
}

// ---------------------------------------------------------------------------
// Domain-decomposition helpers (halo ghosts are atoms [n_active, n)).
// ---------------------------------------------------------------------------
// Push the received per-atom projections P of halo ghosts into their in-edge
// slots (what the owner would have pushed had the ghost been local).
template <typename T>
__global__ void k_dd_push_ghosts(DevGraph gr, const T* __restrict__ p_atom, T* __restrict__ pe) {
    const int i = gr.n_active + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= gr.n) return;
    const T v = p_atom[static_cast<long long>(i) * kH + lane];
    const int is = gr.in_start[i], ic = gr.in_cnt[i];
    for (int k = 0; k < ic; ++k) pe[static_cast<long long>(gr.in_edge[is + k]) * kH + lane] = v;
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
static int net_grid(int n) {
    const int want = (n + kG - 1) / kG;
    const int cap = num_sms() * 2;  // grid-stride beyond two CTAs per SM
    return want < 1 ? 1 : (want < cap ? want : cap);
}

template <typename T>
static size_t smem_bytes(int weight_elems) {
    return static_cast<size_t>(weight_elems) * sizeof(T) + 16 + kG * sizeof(AtomSmem<T>);
}

// Launch with the staged weights + the groups' AtomSmem in dynamic shared memory
// (the > 48 KB opt-in is set by net_configure() when a context is created, never
// during stream capture).
template <typename T, typename... Params, typename... Args>
static void launch_staged(void (*kernel)(Params...), int grid, int smem_elems, cudaStream_t st,
                          Args... args) {
    launch_pdl(kernel, dim3(grid), dim3(kCTA), smem_bytes<T>(smem_elems), st, args...);
}

constexpr int kMaxSmem = 224 * 1024;

template <typename T>
static cudaError_t configure_t() {
    const cudaFuncAttribute a = cudaFuncAttributeMaxDynamicSharedMemorySize;
    cudaError_t e = cudaSuccess;
    for (cudaError_t r : {cudaFuncSetAttribute(k_embed<T, true>, a, kMaxSmem),
                          cudaFuncSetAttribute(k_embed<T, false>, a, kMaxSmem),
                          cudaFuncSetAttribute(k_msg_fwd<T, true>, a, kMaxSmem),
                          cudaFuncSetAttribute(k_msg_fwd<T, false>, a, kMaxSmem),
                          cudaFuncSetAttribute(k_msg_bwd<T>, a, kMaxSmem),
                          cudaFuncSetAttribute(k_embed_bwd<T>, a, kMaxSmem),
                          cudaFuncSetAttribute(k_force<T>, a, kMaxSmem)})
        if (r != cudaSuccess) e = r;
    return e;
}
// Per device: allow the staged-weight kernels up to 224 KB of dynamic smem.
cudaError_t net_configure() {
    const cudaError_t a = configure_t<float>();
    const cudaError_t b = configure_t<double>();
    return a != cudaSuccess ? a : b;
}

template <typename T>
int launch_network(const DevModel<T>& md, const DevGraph& gr, const DevWork<T>& ws,
                   double* forces, double* per_atom, double* out, int* rev, cudaStream_t st,
                   const Marker& mk, const MdFuse& mf) {
    const int nb = net_grid(gr.n);
    const int M = md.n_msg;
    const int e_emb = mlp_elems(kInEmbed, kH), e_fit = mlp_elems(kInFit, 1);
    const int e_msg = mlp_elems(kInMsg, kH), e_upd = mlp_elems(kInUpd, kH);
    int launches = 0;
    if (M == 0) {
        launch_staged<T>(k_embed<T, true>, nb, e_emb + e_fit, st, md, gr, ws, rev, mf);
        mk("embed_fit", st);
        ++launches;
    } else {
        launch_staged<T>(k_embed<T, false>, nb, e_emb + e_msg, st, md, gr, ws, rev, mf);
        mk("embed", st);
        for (int l = 0; l < M; ++l) {
            if (l == M - 1) {
                launch_staged<T>(k_msg_fwd<T, true>, nb, e_msg + e_upd + e_fit, st, md, gr, ws, l);
                mk("msg_fwd_last", st);
            } else {
                launch_staged<T>(k_msg_fwd<T, false>, nb, 2 * e_msg + e_upd, st, md, gr, ws, l);
                mk("msg_fwd", st);
            }
        }
        for (int l = M - 2; l >= 0; --l) {
            launch_staged<T>(k_msg_bwd<T>, nb, 2 * e_msg + e_upd, st, md, gr, ws, l);
            mk("msg_bwd", st);
        }
        launch_staged<T>(k_embed_bwd<T>, nb, e_emb + e_msg, st, md, gr, ws);
        mk("embed_bwd", st);
        launches += 2 + M + (M - 1);
    }
    launch_staged<T>(k_force<T>, nb, 0, st, gr, ws, forces, per_atom, out, mf);
    mk("force", st);
    return launches + 1;
}

// One phase of a domain-decomposed evaluation (the caller exchanges halo rows
// between phases).  Phases: 0 embed, 1 push ghost P (into parity `l`), 2 message
// layer l forward, 3 ghost adjoint sums of layer l, 4 message layer l backward,
// 5 embedding backward, 6 forces.
template <typename T>
void launch_dd_phase(const DevModel<T>& md, const DevGraph& gr, const DevWork<T>& ws, int phase,
                     int l, T* s_ghost, double* forces, double* out, cudaStream_t st) {
    const int nb = net_grid(gr.n_active);
    const int M = md.n_msg;
    const int e_emb = mlp_elems(kInEmbed, kH), e_fit = mlp_elems(kInFit, 1);
    const int e_msg = mlp_elems(kInMsg, kH), e_upd = mlp_elems(kInUpd, kH);
    const int ng = gr.n - gr.n_active;
    const MdFuse none{};
    switch (phase) {
        case 0:
            if (M == 0)
                launch_staged<T>(k_embed<T, true>, nb, e_emb + e_fit, st, md, gr, ws,
                                 static_cast<int*>(nullptr), none);
            else
                launch_staged<T>(k_embed<T, false>, nb, e_emb + e_msg, st, md, gr, ws,
                                 static_cast<int*>(nullptr), none);
            break;
        case 1:
            if (ng > 0)
                k_dd_push_ghosts<T><<<(ng * 32 + 255) / 256, 256, 0, st>>>(
                    gr, ws.p_atom, ws.pe + (l & 1) * ws.slots * kH);
            break;
        case 2:
            if (l == M - 1)
                launch_staged<T>(k_msg_fwd<T, true>, nb, e_msg + e_upd + e_fit, st, md, gr, ws, l);
            else
                launch_staged<T>(k_msg_fwd<T, false>, nb, 2 * e_msg + e_upd, st, md, gr, ws, l);
            break;
        case 3:
            if (ng > 0)
                k_dd_ghost_sums<T><<<(ng * 32 + 255) / 256, 256, 0, st>>>(
                    gr, ws.d + (l & 1) * ws.slots * kH, s_ghost);
            break;
        case 4:
            launch_staged<T>(k_msg_bwd<T>, nb, 2 * e_msg + e_upd, st, md, gr, ws, l);
            break;
        case 5:
            launch_staged<T>(k_embed_bwd<T>, nb, e_emb + e_msg, st, md, gr, ws);
            break;
        case 6:
            launch_staged<T>(k_force<T>, net_grid(gr.n), 0, st, gr, ws, forces,
                             static_cast<double*>(nullptr), out, none);
            break;
    }
}
template void launch_dd_phase<float>(const DevModel<float>&, const DevGraph&,
                                     const DevWork<float>&, int, int, float*, double*, double*,
                                     cudaStream_t);
template void launch_dd_phase<double>(const DevModel<double>&, const DevGraph&,
                                      const DevWork<double>&, int, int, double*, double*, double*,
                                      cudaStream_t);
template int launch_network<float>(const DevModel<float>&, const DevGraph&, const DevWork<float>&,
                                   double*, double*, double*, int*, cudaStream_t, const Marker&,
                                   const MdFuse&);
template int launch_network<double>(const DevModel<double>&, const DevGraph&,
                                    const DevWork<double>&, double*, double*, double*, int*,
                                    cudaStream_t, const Marker&, const MdFuse&);

}  // namespace hmdp
