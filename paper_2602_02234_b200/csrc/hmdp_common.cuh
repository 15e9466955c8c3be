// hmdp_common.cuh — device helpers shared by the neighbour-search and network
// kernels (math overloads for the FP32/FP64 template paths, vector loads, warp
// reductions, the switch function, FP64 geometry with explicit rounding).
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstdint>

#include "hmdp_device.cuh"

namespace hmdp {

#define FULL_MASK 0xffffffffu
constexpr int kAT = 128;       // threads per atom-CTA (4 warps)

// ---------------------------------------------------------------------------
// small device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ float d_tanh(float x) { return tanhf(x); }
__device__ __forceinline__ double d_tanh(double x) { return tanh(x); }
__device__ __forceinline__ float d_exp(float x) { return expf(x); }
__device__ __forceinline__ double d_exp(double x) { return exp(x); }
__device__ __forceinline__ float d_sqrt(float x) { return sqrtf(x); }
__device__ __forceinline__ double d_sqrt(double x) { return sqrt(x); }
__device__ __forceinline__ float d_cos(float x) { return cosf(x); }
__device__ __forceinline__ double d_cos(double x) { return cos(x); }
__device__ __forceinline__ float d_sin(float x) { return sinf(x); }
__device__ __forceinline__ double d_sin(double x) { return sin(x); }

template <typename T>
struct V4 {
    T x, y, z, w;
};
__device__ __forceinline__ V4<float> ld4(const float* p) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(p));
    return {v.x, v.y, v.z, v.w};
}
__device__ __forceinline__ V4<double> ld4(const double* p) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p));
    const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    return {a.x, a.y, b.x, b.y};
}
// coherent (non-.nc) variant for buffers written earlier in the same kernel
__device__ __forceinline__ V4<float> ld4c(const float* p) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    return {v.x, v.y, v.z, v.w};
}
__device__ __forceinline__ V4<double> ld4c(const double* p) {
    const double2 a = *reinterpret_cast<const double2*>(p);
    const double2 b = *(reinterpret_cast<const double2*>(p) + 1);
    return {a.x, a.y, b.x, b.y};
}
__device__ __forceinline__ void st4(float* p, float a, float b, float c, float d) {
    *reinterpret_cast<float4*>(p) = make_float4(a, b, c, d);
}
__device__ __forceinline__ void st4(double* p, double a, double b, double c, double d) {
    reinterpret_cast<double2*>(p)[0] = make_double2(a, b);
    reinterpret_cast<double2*>(p)[1] = make_double2(c, d);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
    return v;
}

// switch_value_t / switch_derivative_t (inference.cpp:49-62), in T.
template <typename T>
__device__ __forceinline__ T sw_val(T r, T rc) {
    const T onset = T(0.9) * rc;
    if (r <= onset) return T(1);
    if (r >= rc) return T(0);
    return T(0.5) * (d_cos(T(M_PI) * (r - onset) / (T(0.1) * rc)) + T(1));
}
template <typename T>
__device__ __forceinline__ T sw_der(T r, T rc) {
    const T onset = T(0.9) * rc;
    if (r <= onset || r >= rc) return T(0);
    return T(-0.5) * d_sin(T(M_PI) * (r - onset) / (T(0.1) * rc)) * T(M_PI) / (T(0.1) * rc);
}

// Edge geometry in T from the FP64 displacement (to_vec<T> + norm, inference.cpp:219-223).
template <typename T>
__device__ __forceinline__ T edge_len(const double* dr3, T& x, T& y, T& z) {
    x = static_cast<T>(dr3[0]);
    y = static_cast<T>(dr3[1]);
    z = static_cast<T>(dr3[2]);
    return d_sqrt(x * x + y * y + z * z);
}

// FP64 helpers with explicit rounding (no FMA contraction) for the bit-exact
// neighbour test: minimum_image (box.hpp:24-31) and norm2 (vec3.hpp:57-70).
// d - L * nearbyint(d / L) (box.hpp:27).  For |d| <= L/2 the rounded quotient
// has magnitude <= 0.5, which rounds (half to even) to zero: the result is d
// itself (+ 0.0 reproduces the +0 the full expression gives for d = -0), so the
// FP64 division is only paid by the pairs that actually wrap.
__device__ __forceinline__ double min_image1(double d, double L) {
    if (fabs(d) <= 0.5 * L) return __dadd_rn(d, 0.0);
    return __dsub_rn(d, __dmul_rn(L, rint(__ddiv_rn(d, L))));
}
__device__ __forceinline__ double norm2_rn(double x, double y, double z) {
    return __dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z));
}


// ---------------------------------------------------------------------------
// Atom-CTA (128 threads) mat-vec: y[o] = sum_{k<NIN} W[o*ldw + k] * x[k] for
// o < NOUT, with x in shared memory.  Thread t computes the partial sum of part
// p = t % P (P = 128/NOUT parts of NIN/P consecutive inputs) for output
// o = t / P; the P partials sit in adjacent lanes and are combined with xor
// shuffles, so every thread of the group returns y[o].  W and x both live in
// shared memory (the kernel stages its weights once per CTA).
// ---------------------------------------------------------------------------
template <typename T, int NOUT, int NIN>
__device__ __forceinline__ T bmv(const T* __restrict__ W, int ldw, const T* xs, int t) {
    constexpr int P = kAT / NOUT;
    constexpr int KP = NIN / P;
    static_assert(P * NOUT == kAT && KP * P == NIN && KP % 4 == 0, "bad bmv shape");
    const int o = t / P, p = t % P;
    const T* wr = W + o * ldw + p * KP;
    const T* xr = xs + p * KP;
    T acc = T(0);
#pragma unroll
    for (int q = 0; q < KP; q += 4) {
        const V4<T> w = ld4c(wr + q);  // weights staged in shared memory
        acc += w.x * xr[q];
        acc += w.y * xr[q + 1];
        acc += w.z * xr[q + 2];
        acc += w.w * xr[q + 3];
    }
#pragma unroll
    for (int m = 1; m < P; m <<= 1) acc += __shfl_xor_sync(FULL_MASK, acc, m);
    return acc;
}
// output index and "group leader" flag of thread t for an NOUT-output bmv
template <int NOUT>
__device__ __forceinline__ int bmv_out(int t) { return t / (kAT / NOUT); }
template <int NOUT>
__device__ __forceinline__ bool bmv_lead(int t) { return (t % (kAT / NOUT)) == 0; }

// Sum over the 128 threads of a CTA (every thread gets the total); s4 is a
// 4-entry shared scratch.  Fixed order: warp tree, then warps 0..3.
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* s4) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) s4[w] = v;
    __syncthreads();
    return ((s4[0] + s4[1]) + s4[2]) + s4[3];
}

// cell of a position: wrap_position, then static_cast<int>(r / L * n_cells)
// clamped (neighborlist.cpp:31-33), in exactly rounded FP64 (no contraction)
__device__ __forceinline__ int cell_index(const double* x3, const CellGrid& cg) {
    int c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double L = cg.L[a];
        double r = x3[a];
        r = __dsub_rn(r, __dmul_rn(L, floor(__ddiv_rn(r, L))));
        if (r >= L) r = 0.0;
        int v = static_cast<int>(__dmul_rn(__ddiv_rn(r, L), static_cast<double>(cg.nc[a])));
        v = v < 0 ? 0 : (v > cg.nc[a] - 1 ? cg.nc[a] - 1 : v);
        c[a] = v;
    }
    return (c[2] * cg.nc[1] + c[1]) * cg.nc[0] + c[0];
}

__device__ __forceinline__ void bin_atom(int i, const double* x3, const CellGrid& cg, int* cell_count,
                         int* members, int* cell_of, unsigned* err) {
    const int cid = cell_index(x3, cg);
    cell_of[i] = cid;
    const int slot = atomicAdd(cell_count + cid, 1);
    if (slot < cg.ccap)
        members[cid * cg.ccap + slot] = i;
    else
        atomicOr(err, kErrCellOverflow);
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

// Programmatic dependent launch (PDL): a kernel lets its successor start
// launching right away (the successor's CTAs take SMs as ours retire and stage
// their weights), and waits for its predecessor's results before touching them.
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Host: launch with the programmatic-stream-serialization attribute (also valid
// under stream capture, where it becomes a programmatic graph edge).
template <typename... Params, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(Params...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    static const bool no_pdl = std::getenv("HMDP_NO_PDL") != nullptr;  // A/B experiments
    cfg.numAttrs = no_pdl ? 0 : 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<Params>(args)...);
}

// ---------------------------------------------------------------------------
// Neighbour search body, one warp per atom.  The deduplicated 27 neighbouring
// cells' member lists form one candidate index space enumerated 32 lanes at a
// time; every j with FP64 minimum-image |dr|^2 <= rc^2 (neighborlist.cpp:91-93,
// box.hpp:27, no FMA contraction) survives a ballot compaction into the warp's
// shared list; survivors are ranked ascending (the reference's sorted full pair
// list, neighborlist.cpp:104-111) and written with their FP64 edge_dr
// (inference.cpp:474-485) and neighbour type.
// ---------------------------------------------------------------------------
constexpr int kCandDr = 64;  // survivors whose FP64 displacement is kept for the write
struct NbrSmem {
    int cand[kCandMax];  // this warp's surviving candidates
    int cnt;
    double cdr[kCandDr][3];  // their displacements as the pair test computed them
};

// G warps (a "team", named barrier `bar`) search one atom: warp w takes the
// candidate blocks q in [32 (w + G k), 32 (w + G k) + 32); each warp compacts its
// survivors into its own list, and ranks them against the whole team's lists.
template <int G>
__device__ __forceinline__ void nbr_search_team(int i, const double* pos, const CellGrid& cg,
                                                const int* cell_count, const int* members,
                                                const int* cell_of, double range2, int cap,
                                                int* __restrict__ nnei, int* __restrict__ row_start,
                                                int* __restrict__ nbr, double* __restrict__ dr,
                                                const int* __restrict__ types,
                                                int* __restrict__ ety, unsigned* err,
                                                NbrSmem* team_sm, int w, int lane, int bar) {
    NbrSmem& sm = team_sm[w];
    const double L0 = cg.L[0], L1 = cg.L[1], L2 = cg.L[2];
    const double xi = pos[3 * i], yi = pos[3 * i + 1], zi = pos[3 * i + 2];
    const int ci = cell_of[i];
    const int cx = ci % cg.nc[0], cy = (ci / cg.nc[0]) % cg.nc[1], cz = ci / (cg.nc[0] * cg.nc[1]);
    int nid = -1;
    if (lane < 27) {
        const int dz = lane / 9 - 1, dy = (lane / 3) % 3 - 1, dx = lane % 3 - 1;
        const int x = ((cx + dx) % cg.nc[0] + cg.nc[0]) % cg.nc[0];
        const int y = ((cy + dy) % cg.nc[1] + cg.nc[1]) % cg.nc[1];
        const int z = ((cz + dz) % cg.nc[2] + cg.nc[2]) % cg.nc[2];
        nid = (z * cg.nc[1] + y) * cg.nc[0] + x;
    }
    bool unique = lane < 27;
    if (cg.nc[0] < 3 || cg.nc[1] < 3 || cg.nc[2] < 3)  // small grids: a cell can repeat
        for (int q = 0; q < 27; ++q) {
            const int other = __shfl_sync(FULL_MASK, nid, q);
            if (q < lane && other == nid) unique = false;
        }
    int cnt = 0;
    if (unique) {
        cnt = cell_count[nid];
        cnt = cnt < cg.ccap ? cnt : cg.ccap;
    }
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(FULL_MASK, incl, o);
        if (lane >= o) incl += v;
    }
    const int off = incl - cnt;  // exclusive offset of lane's cell
    const int base = nid * cg.ccap;
    const int ncand = __shfl_sync(FULL_MASK, incl, 31);
    constexpr int U = G >= 4 ? 2 : 4;  // candidate blocks per warp per pass
    int total = 0;
    for (int b0 = w; 32 * b0 < ncand; b0 += G * U) {
        int jr[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {  // candidate q -> (cell slot, member): independent loads
            const int q = 32 * (b0 + G * u) + lane;
            int lo = 0;  // largest cell slot whose offset <= q (always a non-empty cell)
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const int mid = lo + step;
                const int om = __shfl_sync(FULL_MASK, off, mid & 31);
                if (mid < 27 && om <= q) lo = mid;
            }
            const int ob = __shfl_sync(FULL_MASK, off, lo);
            const int bb = __shfl_sync(FULL_MASK, base, lo);
            jr[u] = q < ncand ? members[bb + (q - ob)] : -1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {  // FP64 pair test (no FMA contraction) + compaction
            bool pass = false;
            double dx = 0.0, dy = 0.0, dz = 0.0;
            const int j = jr[u];
            if (j >= 0 && j != i) {
                dx = min_image1(__dsub_rn(pos[3 * j], xi), L0);
                dy = min_image1(__dsub_rn(pos[3 * j + 1], yi), L1);
                dz = min_image1(__dsub_rn(pos[3 * j + 2], zi), L2);
                pass = !(norm2_rn(dx, dy, dz) > range2);
            }
            const unsigned bal = __ballot_sync(FULL_MASK, pass);
            if (pass) {
                const int idx = total + __popc(bal & ((1u << lane) - 1u));
                if (idx < kCandMax) sm.cand[idx] = j;
                if (idx < kCandDr) {  // kept for the write below
                    sm.cdr[idx][0] = dx;
                    sm.cdr[idx][1] = dy;
                    sm.cdr[idx][2] = dz;
                }
            }
            total += __popc(bal);
        }
    }
    if (lane == 0) sm.cnt = total;
    if constexpr (G > 1)
        asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(G * 32) : "memory");
    else
        __syncwarp();
    int m = 0;
#pragma unroll
    for (int q = 0; q < G; ++q) m += team_sm[q].cnt;
    const bool over = m > cap || total > kCandMax;
    if (over && w == 0 && lane == 0) atomicOr(err, kErrNbrOverflow);
    const int mine = total < kCandMax ? total : kCandMax;
    for (int q = lane; q < mine; q += 32) {
        const int v = sm.cand[q];
        int rank = 0;
#pragma unroll
        for (int t = 0; t < G; ++t) {
            const NbrSmem& o = team_sm[t];
            const int c = o.cnt < kCandMax ? o.cnt : kCandMax;
            for (int p = 0; p < c; ++p) rank += o.cand[p] < v;
        }
        if (rank >= cap) continue;  // overflow: flagged above, the caller re-runs
        const long long slot = static_cast<long long>(i) * cap + rank;
        nbr[slot] = v;
        if (ety) ety[slot] = types[v];
        if (q < kCandDr && dr) {  // the displacement the pair test computed
            dr[3 * slot] = sm.cdr[q][0];
            dr[3 * slot + 1] = sm.cdr[q][1];
            dr[3 * slot + 2] = sm.cdr[q][2];
        } else if (dr) {  // (dr null: a Verlet candidate row, indices only)
            dr[3 * slot] = min_image1(__dsub_rn(pos[3 * v], xi), L0);
            dr[3 * slot + 1] = min_image1(__dsub_rn(pos[3 * v + 1], yi), L1);
            dr[3 * slot + 2] = min_image1(__dsub_rn(pos[3 * v + 2], zi), L2);
        }
    }
    if (w == 0 && lane == 0) {
        nnei[i] = m < cap ? m : cap;
        if (row_start) row_start[i] = i * cap;
    }
    // the lists are reused by the team's next atom
    if constexpr (G > 1)
        asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(G * 32) : "memory");
    else
        __syncwarp();
}

// Verlet filter (device MD loop with a skin): atom i's exact rc list out of its
// candidate row.  The row is ascending in j, so the survivors come out in the
// reference's sorted order (neighborlist.cpp:104-111) without a rank sort; the
// pair test and edge_dr are nbr_search_team's (FP64, no FMA), so the list is the
// one the full search builds.  G == 1: one pass with a running offset; G > 1:
// the team's warps take interleaved 32-candidate blocks, count survivors per
// block (shared), then recompute and write at the prefix offsets.
template <int G>
__device__ __forceinline__ void nbr_filter_team(int i, const double* __restrict__ pos,
                                                const CellGrid& cg, const VList& vl,
                                                double range2, int cap, int* __restrict__ nnei,
                                                int* __restrict__ row_start,
                                                int* __restrict__ nbr, double* __restrict__ dr,
                                                const int* __restrict__ types,
                                                int* __restrict__ ety, unsigned* err,
                                                NbrSmem* team_sm, int w, int lane, int bar) {
    const double L[3] = {cg.L[0], cg.L[1], cg.L[2]};
    const double xi[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
    const int c = min(vl.cnt[i], vl.cap);
    const int* row = vl.list + static_cast<long long>(i) * vl.cap;
    const int nb = (c + 31) >> 5;
    const long long base = static_cast<long long>(i) * cap;
    // 32-candidate blocks in flight per warp: 4 for one-warp teams (a 2PTC row in two
    // rounds), 2 for the multi-warp teams of small boxes (A/B profiles/round2/ab/filter_u.txt:
    // 2PTC DPA2 U=4 +1.7 %, 1UBQ DPA2 U=2 +3.4 %, 1YRF DPA3 U=2 +0.9 %)
#ifdef HMDP_FILTER_U
    constexpr int U = HMDP_FILTER_U;
#else
    constexpr int U = G == 1 ? 4 : 2;
#endif
    int* bcnt = team_sm[0].cand;  // G > 1: survivors per block (nb <= vl.cap / 32)
    // one group of up to U of this warp's blocks: candidates, positions, pair test
    auto test = [&](int b0, int bstep, int (&jr)[U], double (&d)[U][3], unsigned (&bal)[U]) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            // the row load does not wait for the count (slots past it hold stale valid
            // indices or zeros); the count only masks
            const int q = 32 * (b0 + bstep * u) + lane;
            const int raw = q < vl.cap ? row[q] : -1;
            jr[u] = q < c ? raw : -1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int a = 0; a < 3; ++a) d[u][a] = jr[u] >= 0 ? pos[3 * jr[u] + a] : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            bool pass = false;
            if (jr[u] >= 0) {
#pragma unroll
                for (int a = 0; a < 3; ++a) d[u][a] = min_image1(__dsub_rn(d[u][a], xi[a]), L[a]);
                pass = !(norm2_rn(d[u][0], d[u][1], d[u][2]) > range2);
            }
            bal[u] = __ballot_sync(FULL_MASK, pass);
        }
    };
    auto write = [&](int off, unsigned b, int j, const double (&d3)[3]) {
        if (!((b >> lane) & 1u)) return;
        const int idx = off + __popc(b & ((1u << lane) - 1u));
        if (idx >= cap) return;  // overflow: flagged below
        const long long slot = base + idx;
        nbr[slot] = j;
        if (ety) ety[slot] = types[j];
        dr[3 * slot] = d3[0];
        dr[3 * slot + 1] = d3[1];
        dr[3 * slot + 2] = d3[2];
    };
    int total = 0;
    if constexpr (G == 1) {
        int b0 = 0;
        do {  // (do-while: the first group's loads need not wait for the count)
            int jr[U];
            double d[U][3];
            unsigned bal[U];
            test(b0, 1, jr, d, bal);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                write(total, bal[u], jr[u], d[u]);
                total += __popc(bal[u]);
            }
            b0 += U;
        } while (b0 < nb);
        __syncwarp();
    } else {
        for (int b0 = w; b0 < nb; b0 += G * U) {
            int jr[U];
            double d[U][3];
            unsigned bal[U];
            test(b0, G, jr, d, bal);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (lane == 0 && b0 + G * u < nb) bcnt[b0 + G * u] = __popc(bal[u]);
        }
        asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(G * 32) : "memory");
        for (int t = 0; t < nb; ++t) total += bcnt[t];
        for (int b0 = w; b0 < nb; b0 += G * U) {
            int jr[U];
            double d[U][3];
            unsigned bal[U];
            test(b0, G, jr, d, bal);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int b = b0 + G * u;
                if (b >= nb) break;
                int off = 0;
                for (int t = 0; t < b; ++t) off += bcnt[t];
                write(off, bal[u], jr[u], d[u]);
            }
        }
        asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(G * 32) : "memory");  // bcnt reuse
    }
    if (w == 0 && lane == 0) {
        if (total > cap) atomicOr(err, kErrNbrOverflow);
        nnei[i] = total < cap ? total : cap;
        row_start[i] = i * cap;
    }
}

// Device MD loop with a Verlet skin: after the drift, an atom farther than skin/2
// from where the candidate rows were last built raises the rebuild flag.
__device__ __forceinline__ void vlist_check(const double* x3, const double* xr, const MdFuse& mf) {
    if (!mf.vflag) return;
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double d = min_image1(x3[a] - xr[a], mf.cg.L[a]);
        s += d * d;
    }
    if (!(s <= mf.vhalf2)) *mf.vflag = 1;  // (a NaN position rebuilds too)
}

// Opening of a device-MD chunk for atom i: first half kick + drift + binning
// (integrators.cpp:35-39 after the finite check of :12-18).
__device__ __forceinline__ void vv_kick_drift_bin_atom(int i, const MdFuse& mf,
                                                       const double* f, unsigned* err) {
    const double s = mf.half / mf.m[i];
    bool finite = true;
    double x3[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double fa = f[3 * i + a];
        finite &= isfinite(fa);
        const double va = __dadd_rn(mf.v[3 * i + a], __dmul_rn(fa, s));
        mf.v[3 * i + a] = va;
        x3[a] = __dadd_rn(mf.x[3 * i + a], __dmul_rn(va, mf.dt));
        mf.x[3 * i + a] = x3[a];
    }
    if (!finite) atomicOr(err, kErrNonFinite);
    if (mf.vflag) {
        const double xr[3] = {mf.xref[3 * i], mf.xref[3 * i + 1], mf.xref[3 * i + 2]};
        vlist_check(x3, xr, mf);
    }
    bin_atom(i, x3, mf.cg, mf.cell_count, mf.members, mf.cell_of, err);
}
}  // namespace hmdp
