// hmdp_gdd.cu — device-resident domain decomposition on the GLOBAL index space.
//
// Every rank keeps the whole system's positions (replicated: all ranks integrate
// all atoms with the same all-reduced forces) and the global periodic ELL graph,
// but runs the network only for the atoms its region owns.  Per step, entirely on
// the device with fixed-size buffers (so the step is capturable in one CUDA graph,
// collectives included):
//   roles      owner = region of the wrapped position (dd.owners); halo = within rc
//              of this rank's region; lists of owned / halo / searched atoms
//   search     rows for owned + halo atoms only (other rows empty)
//   rev        mirror slots of every searched row (halo rows too: halo atoms push
//              their received P into their in-edge slots, and collect partial sums)
//   zero       slots whose SOURCE is not owned here never receive a push on this
//              rank: their pushed adjoints (d) and pushed g are zeroed, and so are
//              halo rows' own g and the per-atom energies of non-owned atoms
//   network    the single-GPU kernels over the owned list (DevGraph::alist), with
//              the per-layer exchanges of the reference DD protocol (dd.py) done as
//              SUM all-reduces of global-index per-atom buffers in which only this
//              rank's rows are non-zero:
//                P^l rows of owned atoms  -> every rank (halo copies pushed into slots)
//                dE/dh partial sums at halo atoms -> owners (DevWork::s_remote)
//                partial forces at halo atoms -> owners; (E, W, W9) totals
//   integrate  velocity Verlet on all atoms from the all-reduced forces.
// The collectives are the caller's (NCCL all_reduce on the bound buffers, between
// phases, on the same stream); an in-process sum over simulated ranks exercises the
// same phases on one GPU.
//
// Halo-exchange mode (the default multi-GPU engine; hmdp_api.cu "gdd halo"): the
// same phases, but nothing is replicated and nothing is all-reduced except (E, W,
// W9).  Each rank integrates ONLY its owned atoms; per step, point-to-point rounds
// with every peer move exactly the halo:
//   POS     (x, v) of owned atoms near peer q's region      -> q   (+ migration)
//   P^l     P rows of owned atoms near q's region           -> q   (per layer)
//   SUMS^l  dE/dh partial sums at halo atoms                 -> their owners
//   FORCES  partial forces at halo atoms                     -> their owners
// Ownership is re-derived every step from the received positions (owner = region
// of the wrapped position), so an atom that drifts into a neighbour's region is
// migrated by the POS round itself (it is near -- inside -- that region).
#include "hmdp_common.cuh"

namespace hmdp {

struct GddGeom {
    int d[3];      // rank grid
    double L[3];   // box
    int rank;
    double halo;   // halo width (rc)
};

// Buffers the roles kernel clears on the way (phase 10's former memset nodes):
// up to four int ranges and one byte range, nullable.
struct GddZero {
    int* i32[4];
    int n32[4];
    unsigned char* u8;
    int n8;
    double* e_atom;  // per-atom energies of the rows this rank does not own
};

// Wrapped coordinate (wrap_position, box.hpp:34-42, as dd.owners).
__device__ __forceinline__ double gdd_wrap(double r, double L) {
    r = r - L * floor(r / L);
    return r >= L ? 0.0 : r;
}
// Region (rank) owning a wrapped position: its cell of the rank grid.
__device__ __forceinline__ int gdd_owner(const double* p, const GddGeom& g) {
    int c3[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double r = gdd_wrap(p[a], g.L[a]);
        int c = static_cast<int>(r / g.L[a] * g.d[a]);
        c3[a] = c < 0 ? 0 : (c > g.d[a] - 1 ? g.d[a] - 1 : c);
    }
    return c3[0] + g.d[0] * (c3[1] + g.d[1] * c3[2]);
}
// Periodic distance from a position to rank q's region, tested against the halo
// width.  The ONE predicate for "q needs this atom": the sender's send lists and
// the receiver's halo role both use it on bitwise-identical positions, so they
// always agree.  The ownership test and the slab bounds may disagree at a boundary
// by rounding: the region's own atoms are always "near".
__device__ __forceinline__ bool gdd_near(const double* p, const GddGeom& g, int q) {
    const int q3[3] = {q % g.d[0], (q / g.d[0]) % g.d[1], q / (g.d[0] * g.d[1])};
    double dist2 = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (g.d[a] <= 1) continue;
        const double L = g.L[a];
        const double r = gdd_wrap(p[a], L);
        const double lo = L * q3[a] / g.d[a], hi = L * (q3[a] + 1) / g.d[a];
        double da = 0.0;
        if (r < lo || r >= hi) {  // periodic distance to the slab [lo, hi)
            double a1 = lo - r, a2 = r - hi;
            a1 -= L * floor(a1 / L);
            a2 -= L * floor(a2 / L);
            da = a1 < a2 ? a1 : a2;
        }
        dist2 += da * da;
    }
    return dist2 <= g.halo * g.halo * (1.0 + 1e-9) + 1e-24;
}

// roles + lists: lists[0..n) owned, lists[n..2n) halo, lists[2n..3n) searched
// (owned + halo); counts[0..2] their lengths (zeroed by the caller each step).
// Halo-exchange mode (stamp != null): only atoms whose position is current on this
// rank take part -- owned here last step (role 1) or received this step (stamp ==
// *cur); every other row of the global arrays is stale.
__global__ void k_gdd_roles(int n, const double* __restrict__ pos, GddGeom g,
                            unsigned char* __restrict__ role, int* __restrict__ lists,
                            int* __restrict__ counts, const int* __restrict__ stamp,
                            const int* __restrict__ cur, GddZero z) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int nt = gridDim.x * blockDim.x;
#pragma unroll
    for (int r = 0; r < 4; ++r)
        if (z.i32[r])
            for (int t = i; t < z.n32[r]; t += nt) z.i32[r][t] = 0;
    if (z.u8)
        for (int t = i; t < z.n8; t += nt) z.u8[t] = 0;
    if (i >= n) return;
    if (stamp && role[i] != 1 && stamp[i] != *cur) {
        role[i] = 0;
        if (z.e_atom) z.e_atom[i] = 0.0;
        return;
    }
    const bool owned = gdd_owner(pos + 3 * i, g) == g.rank;
    const bool halo = !owned && gdd_near(pos + 3 * i, g, g.rank);
    const unsigned char ro = owned ? 1 : (halo ? 2 : 0);
    role[i] = ro;
    if (z.e_atom && !owned) z.e_atom[i] = 0.0;
    if (owned) lists[atomicAdd(counts + 0, 1)] = i;
    if (halo) lists[n + atomicAdd(counts + 1, 1)] = i;
    if (ro) lists[2 * n + atomicAdd(counts + 2, 1)] = i;
}

// ---------------------------------------------------------------------------
// Halo exchange (point-to-point, per peer; hmdp_gdd halo mode).  Per round every
// rank fills one fixed-capacity packet per peer and the transport (grouped
// ncclSend/ncclRecv, or the caller) moves packet s->r into r's receive slot s.
// Packet (C rows, C % 4 == 0): int count, 3 pad, int gidx[C], payload[C][W] (E).
// Lists are [world][C] global indices; counts[world].
// ---------------------------------------------------------------------------
__host__ __device__ inline size_t gdd_pkt_bytes(int C, int W, int esz) {
    return 16 + static_cast<size_t>(C) * 4 + static_cast<size_t>(C) * W * esz;
}

// send lists: src atoms (a list) that are near peer q's region, for every q != rank
// (forward rounds: owned atoms -> the peers whose halo they are in), or grouped by
// owner (reverse rounds: halo atoms -> their owners, by_owner = 1).  blockIdx.y
// selects one of two sets (phase 10 builds both directions in one launch).
struct SendSet {
    const int* src;
    const int* src_n;
    int by_owner;
    int* lists;
    int* counts;
    unsigned char* mark;  // forward: 1 for every atom in some peer's halo (nullable)
};
__global__ void k_gdd_send_lists(SendSet s0, SendSet s1, const double* __restrict__ pos, GddGeom g,
                                 int world, int C, unsigned* err, int* tick) {
    if (tick && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0)
        *tick += 1;  // the POS round's new stamp
    const SendSet& ss = blockIdx.y ? s1 : s0;
    const int ns = *ss.src_n;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < ns; k += gridDim.x * blockDim.x) {
        const int i = ss.src[k];
        const double* p = pos + 3 * i;
        if (ss.by_owner) {
            const int q = gdd_owner(p, g);
            if (q == g.rank) continue;
            const int s = atomicAdd(ss.counts + q, 1);
            if (s < C) ss.lists[q * C + s] = i;
            else atomicOr(err, kErrHaloOverflow);
        } else {
            for (int q = 0; q < world; ++q) {
                if (q == g.rank || !gdd_near(p, g, q)) continue;
                if (ss.mark) ss.mark[i] = 1;
                const int s = atomicAdd(ss.counts + q, 1);
                if (s < C) ss.lists[q * C + s] = i;
                else atomicOr(err, kErrHaloOverflow);
            }
        }
    }
}

// pack: payload columns [0, w0) from src0 rows, [w0, w0 + w1) from src1 rows
template <typename E>
__global__ void k_gdd_pack(int world, int rank, const int* __restrict__ lists,
                           const int* __restrict__ counts, int C, const E* __restrict__ src0,
                           int w0, const E* __restrict__ src1, int w1, char* __restrict__ pkts,
                           size_t pkt_bytes) {
    const int q = blockIdx.y;
    if (q == rank) return;
    const int W = w0 + w1;
    const int cnt = min(counts[q], C);
    char* pk = pkts + q * pkt_bytes;
    int* head = reinterpret_cast<int*>(pk);
    int* gid = head + 4;
    E* pay = reinterpret_cast<E*>(pk + 16 + static_cast<size_t>(C) * 4);
    if (blockIdx.x == 0 && threadIdx.x == 0) head[0] = cnt;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt * W; t += gridDim.x * blockDim.x) {
        const int k = t / W, c = t - k * W;
        const long long i = lists[q * C + k];
        if (c == 0) gid[k] = static_cast<int>(i);
        pay[static_cast<size_t>(k) * W + c] = c < w0 ? src0[i * w0 + c] : src1[i * w1 + (c - w0)];
    }
}

// unpack (copy): rows of every peer's packet into dst0/dst1 at their global index;
// stamp (nullable) marks the received atoms current for this step
template <typename E>
__global__ void k_gdd_unpack_copy(int world, int rank, int C, const char* __restrict__ pkts,
                                  size_t pkt_bytes, E* __restrict__ dst0, int w0,
                                  E* __restrict__ dst1, int w1, int* __restrict__ stamp,
                                  const int* __restrict__ cur) {
    const int q = blockIdx.y;
    if (q == rank) return;
    const int W = w0 + w1;
    const char* pk = pkts + q * pkt_bytes;
    const int* head = reinterpret_cast<const int*>(pk);
    const int* gid = head + 4;
    const E* pay = reinterpret_cast<const E*>(pk + 16 + static_cast<size_t>(C) * 4);
    const int cnt = min(head[0], C);
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt * W; t += gridDim.x * blockDim.x) {
        const int k = t / W, c = t - k * W;
        const long long i = gid[k];
        const E v = pay[static_cast<size_t>(k) * W + c];
        if (c < w0) dst0[i * w0 + c] = v;
        else dst1[i * w1 + (c - w0)] = v;
        if (stamp && c == 0) stamp[i] = *cur;
    }
}

// unpack (add): peer q's rows added into dst at their global index.  One launch per
// peer, in rank order: an atom that is a halo atom on several peers receives their
// partials in a fixed order (bitwise-deterministic sums, no float atomics).
template <typename E>
__global__ void k_gdd_unpack_add(int q, int C, const char* __restrict__ pkts, size_t pkt_bytes,
                                 E* __restrict__ dst, int W) {
    const char* pk = pkts + q * pkt_bytes;
    const int* head = reinterpret_cast<const int*>(pk);
    const int* gid = head + 4;
    const E* pay = reinterpret_cast<const E*>(pk + 16 + static_cast<size_t>(C) * 4);
    const int cnt = min(head[0], C);
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt * W; t += gridDim.x * blockDim.x) {
        const int k = t / W, c = t - k * W;
        dst[static_cast<long long>(gid[k]) * W + c] += pay[static_cast<size_t>(k) * W + c];
    }
}

// OUT round: (E, W, W9) partials into every peer's packet slot; the totals are the
// rank-ordered sum of all ranks' partials (own partial read from `out` itself), so
// every rank ends with bitwise the same totals.
__global__ void k_gdd_out_pack(int world, int rank, const double* __restrict__ out,
                               char* __restrict__ pkts, size_t stride) {
    const int q = blockIdx.x, k = threadIdx.x;
    if (q != rank && k < 16) reinterpret_cast<double*>(pkts + q * stride)[k] = out[k];
}
__global__ void k_gdd_sum_out(int world, int rank, const char* __restrict__ pkts, size_t stride,
                              double* __restrict__ out) {
    const int k = threadIdx.x;
    if (k >= 11) return;
    double s = 0.0;
    for (int q = 0; q < world; ++q)
        s += q == rank ? out[k] : reinterpret_cast<const double*>(pkts + q * stride)[k];
    __syncwarp();
    out[k] = s;
}
__global__ void k_gdd_stamp_all(int n, int* __restrict__ stamp, const int* __restrict__ cur) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) stamp[i] = *cur + 1;  // current for the next step
}

// Mirror slots of the searched rows (one warp per atom); rows of atoms that are
// not searched are empty, so the mirror of an edge into them is -1 (never used).
__global__ void k_gdd_rev(DevGraph gr, int* __restrict__ rev) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int n_run = *gr.alist_n;
    for (int k = warp; k < n_run; k += nw) {
        const int i = gr.alist[k];
        const int start = gr.row_start[i], cnt = gr.nnei[i];
        for (int base = 0; base < cnt; base += 32) {
            const int m = min(32, cnt - base);
            const int e = start + base + lane;
            const int j = lane < m ? gr.nbr[e] : 0;
            const int f = find_rev(i, j, m, gr);
            if (lane < m) rev[e] = f;
        }
    }
}

// Zero what no kernel on this rank will write this step (one warp per searched atom).
template <typename T>
__global__ void k_gdd_zero(DevGraph gr, const unsigned char* __restrict__ role, T* __restrict__ d,
                           long long slots, T* __restrict__ grev, T* __restrict__ g,
                           double* __restrict__ e_atom) {
    // per-atom energies of every row this rank does not own
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < gr.n; i += gridDim.x * blockDim.x)
        if (role[i] != 1) e_atom[i] = 0.0;
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int n_run = *gr.alist_n;
    for (int k = warp; k < n_run; k += nw) {
        const int i = gr.alist[k];
        const int start = gr.row_start[i], cnt = gr.nnei[i];
        const bool own_row = role[i] == 1;
        for (int base = 0; base < cnt; base += 32) {  // lane = slot, then the flagged rows
            const int q = base + lane;
            const long long e = start + q;
            const bool flag = q < cnt && role[gr.nbr[e]] != 1;
            if (flag) grev[e] = T(0);
            if (!own_row && q < cnt) g[e] = T(0);
            if (d) {
                unsigned bal = __ballot_sync(FULL_MASK, flag);
                while (bal) {
                    const long long ef = start + base + (__ffs(bal) - 1);
                    bal &= bal - 1;
                    d[ef * kH + lane] = T(0);
                    d[(slots + ef) * kH + lane] = T(0);
                }
            }
        }
    }
}

// Halo atoms take the P rows received from their owners into the layer's per-atom
// P rows (gathered by the owned sources' edges).
template <typename T>
__global__ void k_gdd_push_halo(DevGraph gr, const T* __restrict__ p_atom, T* __restrict__ pa,
                                const int* __restrict__ hlist, const int* __restrict__ hcount) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int nh = *hcount;
    for (int k = warp; k < nh; k += nw) {
        const long long i = hlist[k];
        pa[i * kH + lane] = p_atom[i * kH + lane];
    }
}

// Partial dE/dh sums collected at halo atoms (pushed by owned sources), into the
// global-index exchange buffer (rows of other atoms stay zero).
template <typename T>
__global__ void k_gdd_halo_sums(DevGraph gr, const T* __restrict__ d, T* __restrict__ out,
                                const int* __restrict__ hlist, const int* __restrict__ hcount) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int nh = *hcount;
    for (int k = warp; k < nh; k += nw) {
        const int i = hlist[k];
        const int start = gr.row_start[i], cnt = gr.nnei[i];
        T s = T(0);
        for (int q = 0; q < cnt; ++q) s += d[static_cast<long long>(start + q) * kH + lane];
        out[static_cast<long long>(i) * kH + lane] = s;
    }
}

// Velocity Verlet on every atom from the all-reduced forces: closing kick of this
// step, opening kick of the next, drift (integrators.cpp:32-47, the split the
// single-GPU device MD loop fuses into its force kernel).
// (Halo mode: only the atoms of `list` -- this rank's owned atoms.)
__global__ void k_gdd_integrate(int n, const double* __restrict__ f, double* __restrict__ x,
                                double* __restrict__ v, const double* __restrict__ m, double half,
                                double dt, int mode, unsigned* err, const int* __restrict__ list,
                                const int* __restrict__ list_n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (list) {
        if (i >= *list_n) return;
        i = list[i];
    }
    if (i >= n) return;
    const double s = half / m[i];
    bool finite = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double fa = f[3 * i + a];
        finite = finite && isfinite(fa);
        double va = v[3 * i + a];
        if (mode != 1) va = __dadd_rn(va, __dmul_rn(fa, s));  // closing kick
        va = __dadd_rn(va, __dmul_rn(fa, s));                  // next opening kick
        x[3 * i + a] = __dadd_rn(x[3 * i + a], __dmul_rn(va, dt));
        v[3 * i + a] = va;
    }
    if (!finite) atomicOr(err, kErrNonFinite);
}

void launch_gdd_roles(int n, const double* pos, const GddGeom& g, unsigned char* role, int* lists,
                      int* counts, cudaStream_t st, const int* stamp, const int* cur,
                      const GddZero* zero) {
    k_gdd_roles<<<(n + 255) / 256, 256, 0, st>>>(n, pos, g, role, lists, counts, stamp, cur,
                                                 zero ? *zero : GddZero{});
}
void launch_gdd_send_lists(const int* src, const int* src_n, int n_est, const double* pos,
                           const GddGeom& g, int world, int by_owner, int C, int* lists,
                           int* counts, unsigned* err, cudaStream_t st, unsigned char* mark,
                           int* tick) {
    const int blocks = (n_est + 255) / 256;
    const SendSet s0{src, src_n, by_owner, lists, counts, mark};
    k_gdd_send_lists<<<blocks < 1 ? 1 : blocks, 256, 0, st>>>(s0, s0, pos, g, world, C, err, tick);
}
// Both directions of phase 10 in one launch: owned -> peers' halos (forward, with the
// boundary marks) and halo -> owners.
void launch_gdd_send_lists2(const int* own, const int* own_n, const int* halo, const int* halo_n,
                            int n_est, const double* pos, const GddGeom& g, int world, int C,
                            int* flist, int* fcnt, int* rlist, int* rcnt, unsigned* err,
                            unsigned char* mark, cudaStream_t st) {
    const int blocks = (n_est + 255) / 256;
    const SendSet s0{own, own_n, 0, flist, fcnt, mark}, s1{halo, halo_n, 1, rlist, rcnt, nullptr};
    k_gdd_send_lists<<<dim3(blocks < 1 ? 1 : blocks, 2), 256, 0, st>>>(s0, s1, pos, g, world, C, err,
                                                                    nullptr);
}
template <typename E>
void launch_gdd_pack(int world, int rank, const int* lists, const int* counts, int C, const E* src0,
                     int w0, const E* src1, int w1, char* pkts, size_t pkt_bytes, cudaStream_t st) {
    const int work = C * (w0 + w1);
    const int bx = (work + 255) / 256;
    k_gdd_pack<E><<<dim3(bx < 1 ? 1 : (bx > 64 ? 64 : bx), world), 256, 0, st>>>(
        world, rank, lists, counts, C, src0, w0, src1, w1, pkts, pkt_bytes);
}
template <typename E>
void launch_gdd_unpack_copy(int world, int rank, int C, const char* pkts, size_t pkt_bytes, E* dst0,
                            int w0, E* dst1, int w1, int* stamp, const int* cur, cudaStream_t st) {
    const int work = C * (w0 + w1);
    const int bx = (work + 255) / 256;
    k_gdd_unpack_copy<E><<<dim3(bx < 1 ? 1 : (bx > 64 ? 64 : bx), world), 256, 0, st>>>(
        world, rank, C, pkts, pkt_bytes, dst0, w0, dst1, w1, stamp, cur);
}
template <typename E>
void launch_gdd_unpack_add(int world, int rank, int C, const char* pkts, size_t pkt_bytes, E* dst,
                           int W, cudaStream_t st) {
    const int bx = (C * W + 255) / 256;
    for (int q = 0; q < world; ++q)
        if (q != rank)
            k_gdd_unpack_add<E><<<bx < 1 ? 1 : (bx > 64 ? 64 : bx), 256, 0, st>>>(q, C, pkts,
                                                                              pkt_bytes, dst, W);
}
void launch_gdd_out_pack(int world, int rank, const double* out, char* pkts, size_t stride,
                         cudaStream_t st) {
    k_gdd_out_pack<<<world, 32, 0, st>>>(world, rank, out, pkts, stride);
}
void launch_gdd_sum_out(int world, int rank, const char* pkts, size_t stride, double* out,
                        cudaStream_t st) {
    k_gdd_sum_out<<<1, 32, 0, st>>>(world, rank, pkts, stride, out);
}
void launch_gdd_stamp_all(int n, int* stamp, const int* cur, cudaStream_t st) {
    k_gdd_stamp_all<<<(n + 255) / 256, 256, 0, st>>>(n, stamp, cur);
}
static int warp_grid(int n_est) {
    const int blocks = (n_est * 32 + 255) / 256;
    return blocks < 1 ? 1 : (blocks > 4096 ? 4096 : blocks);
}
void launch_gdd_rev(const DevGraph& gr, int n_est, int* rev, cudaStream_t st) {
    k_gdd_rev<<<warp_grid(n_est), 256, 0, st>>>(gr, rev);
}
template <typename T>
void launch_gdd_zero(const DevGraph& gr, int n_est, const unsigned char* role, T* d,
                     long long slots, T* grev, T* g, double* e_atom, cudaStream_t st) {
    k_gdd_zero<T><<<warp_grid(n_est), 256, 0, st>>>(gr, role, d, slots, grev, g, e_atom);
}
template <typename T>
void launch_gdd_push_halo(const DevGraph& gr, int n_est, const T* p_atom, T* pe,
                          const int* hlist, const int* hcount, cudaStream_t st) {
    k_gdd_push_halo<T><<<warp_grid(n_est), 256, 0, st>>>(gr, p_atom, pe, hlist, hcount);
}
template <typename T>
void launch_gdd_halo_sums(const DevGraph& gr, int n_est, const T* d, T* out, const int* hlist,
                          const int* hcount, cudaStream_t st) {
    k_gdd_halo_sums<T><<<warp_grid(n_est), 256, 0, st>>>(gr, d, out, hlist, hcount);
}
void launch_gdd_integrate(int n, const double* f, double* x, double* v, const double* m,
                          double dt, int mode, unsigned* err, cudaStream_t st, const int* list,
                          const int* list_n) {
    k_gdd_integrate<<<(n + 255) / 256, 256, 0, st>>>(n, f, x, v, m, 0.5 * dt, dt, mode, err, list,
                                                     list_n);
}

#define HMDP_GDD_INST(T)                                                                       \
    template void launch_gdd_zero<T>(const DevGraph&, int, const unsigned char*, T*, long long, \
                                     T*, T*, double*, cudaStream_t);                            \
    template void launch_gdd_push_halo<T>(const DevGraph&, int, const T*, T*, const int*,       \
                                          const int*, cudaStream_t);                            \
    template void launch_gdd_halo_sums<T>(const DevGraph&, int, const T*, T*, const int*,       \
                                          const int*, cudaStream_t);
HMDP_GDD_INST(float)
HMDP_GDD_INST(double)
#define HMDP_GDD_PKT_INST(E)                                                                      \
    template void launch_gdd_pack<E>(int, int, const int*, const int*, int, const E*, int,        \
                                     const E*, int, char*, size_t, cudaStream_t);                 \
    template void launch_gdd_unpack_copy<E>(int, int, int, const char*, size_t, E*, int, E*, int, \
                                            int*, const int*, cudaStream_t);                      \
    template void launch_gdd_unpack_add<E>(int, int, int, const char*, size_t, E*, int,           \
                                           cudaStream_t);
HMDP_GDD_PKT_INST(float)
HMDP_GDD_PKT_INST(double)

// ---------------------------------------------------------------------------
// Gather-to-root mode (the paper's strategy: the group's atoms are
// aggregated on one rank for a single inference, forces scattered back to the
// owners).  GATHER: every rank's owned atoms -> root; SCATTER: root answers each
// peer with the rows of the atoms that peer sent, in the same order.
// ---------------------------------------------------------------------------
// send lists of the GATHER round: this rank's owned list to `root`, nothing to the
// other peers (lists are [world][C]).
__global__ void k_gdd_gather_list(int world, int root, const int* __restrict__ owned,
                                  const int* __restrict__ n_owned, int C, int* __restrict__ lists,
                                  int* __restrict__ counts, unsigned* err) {
    const int no = *n_owned;
    if (blockIdx.x == 0 && threadIdx.x < world)
        counts[threadIdx.x] = threadIdx.x == root ? (no < C ? no : C) : 0;
    if (blockIdx.x == 0 && threadIdx.x == 0 && no > C) atomicOr(err, kErrHaloOverflow);
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < no && k < C; k += gridDim.x * blockDim.x)
        lists[root * C + k] = owned[k];
}

// reply packets: for every peer q, the rows src[gid] of the atoms listed in the
// packet received from q (count 0 answers an empty packet)
template <typename E>
__global__ void k_gdd_pack_reply(int world, int rank, int C, const char* __restrict__ rpk,
                                 char* __restrict__ spk, size_t pkt_bytes, const E* __restrict__ src,
                                 int W) {
    const int q = blockIdx.y;
    if (q == rank) return;
    const int* rhead = reinterpret_cast<const int*>(rpk + q * pkt_bytes);
    const int* rgid = rhead + 4;
    int* shead = reinterpret_cast<int*>(spk + q * pkt_bytes);
    int* sgid = shead + 4;
    E* pay = reinterpret_cast<E*>(spk + q * pkt_bytes + 16 + static_cast<size_t>(C) * 4);
    const int cnt = min(rhead[0], C);
    if (blockIdx.x == 0 && threadIdx.x == 0) shead[0] = cnt;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt * W; t += gridDim.x * blockDim.x) {
        const int k = t / W, c = t - k * W;
        const long long i = rgid[k];
        if (c == 0) sgid[k] = static_cast<int>(i);
        pay[static_cast<size_t>(k) * W + c] = src[i * W + c];
    }
}

void launch_gdd_gather_list(int world, int root, const int* owned, const int* n_owned, int C,
                            int* lists, int* counts, unsigned* err, cudaStream_t st) {
    const int b = (C + 255) / 256;
    k_gdd_gather_list<<<b < 1 ? 1 : (b > 64 ? 64 : b), 256, 0, st>>>(world, root, owned, n_owned,
                                                                     C, lists, counts, err);
}
template <typename E>
void launch_gdd_pack_reply(int world, int rank, int C, const char* rpk, char* spk,
                           size_t pkt_bytes, const E* src, int W, cudaStream_t st) {
    const int bx = (C * W + 255) / 256;
    k_gdd_pack_reply<E><<<dim3(bx < 1 ? 1 : (bx > 64 ? 64 : bx), world), 256, 0, st>>>(
        world, rank, C, rpk, spk, pkt_bytes, src, W);
}
template void launch_gdd_pack_reply<double>(int, int, int, const char*, char*, size_t,
                                            const double*, int, cudaStream_t);

}  // namespace hmdp
