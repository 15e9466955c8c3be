// hmdp_nbr.cu — cell-list neighbour search, CSR/in-edge plumbing, the FP64
// descriptor API and the velocity-Verlet opening kernel of the device MD loop.
// The per-atom bodies (bin_atom, nbr_search_atom, vv_kick_drift_bin_atom) live
// in hmdp_common.cuh so the persistent MD kernel (hmdp_net.cu) reuses them.
//
// Reference correspondence (paths relative to /root/reference/proj):
//   k_cell_bin          build_grid + wrap_position   src/neighborlist.cpp:21-38,
//                                                    include/halomd/box.hpp:34-42
//   k_nbr_search        build_neighbor_list (full)   src/neighborlist.cpp:42-113
//                       + CSR edge_dr                src/nn/inference.cpp:474-485
//   k_descriptors_f64   descriptors()                src/nn/inference.cpp:430-447
//   k_vv_kick_drift_bin velocity_verlet_step         src/integrators.cpp:12-47
#include <cstdlib>

#include "hmdp_common.cuh"

namespace hmdp {

__global__ void k_cell_bin(int n, const double* __restrict__ pos, CellGrid cg,
                           int* __restrict__ cell_count, int* __restrict__ members,
                           int* __restrict__ cell_of, unsigned* err) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    bin_atom(i, pos + 3 * i, cg, cell_count, members, cell_of, err);
}

// hmdp_compute's graph path: stage one atom's inputs from host-mapped memory into
// the device arrays and bin it — one kernel where a stage-in kernel and the binning
// were two (-4 µs per DPA3 1YRF call, tools/ab_e2e.sh).
__global__ void k_stage_bin(int n, const double* __restrict__ hx, const int* __restrict__ ht,
                            double* __restrict__ pos, int* __restrict__ types, CellGrid cg,
                            int* __restrict__ cell_count, int* __restrict__ members,
                            int* __restrict__ cell_of, unsigned* err,
                            const double* __restrict__ xref, int* vflag, double vhalf2) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double x3[3] = {hx[3 * i], hx[3 * i + 1], hx[3 * i + 2]};
    types[i] = ht[i];
    pos[3 * i] = x3[0];
    pos[3 * i + 1] = x3[1];
    pos[3 * i + 2] = x3[2];
    if (vflag) {  // Verlet rows of the graph path: this call's atom moved past skin/2?
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double d = min_image1(x3[a] - xref[3 * i + a], cg.L[a]);
            s += d * d;
        }
        if (!(s <= vhalf2)) *vflag = 1;  // (a NaN position rebuilds too)
    }
    bin_atom(i, x3, cg, cell_count, members, cell_of, err);
}

// G warps per atom (G = 4 / 2 / 1 by system size, as the network kernels), 16
// warps per CTA, grid-stride over atoms.
constexpr int kSearchCTA = 512;
template <int G>
__global__ __launch_bounds__(kSearchCTA, 2) void k_nbr_search(
    int n, const double* __restrict__ pos, CellGrid cg, const int* __restrict__ cell_count,
    const int* __restrict__ members, const int* __restrict__ cell_of, double range2, int cap,
    int* __restrict__ nnei, int* __restrict__ row_start, int* __restrict__ nbr,
    double* __restrict__ dr, const int* __restrict__ types, int* __restrict__ ety,
    unsigned* err, const int* __restrict__ alist, const int* __restrict__ alist_n) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    NbrSmem* sm = reinterpret_cast<NbrSmem*>(smem_raw);
    pdl_launch_dependents();
    pdl_wait();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tpc = (blockDim.x >> 5) / G, team = warp / G, w = warp % G;
    const int nt = gridDim.x * tpc;
    // alist (global-index domain decomposition): only this rank's owned + halo atoms
    const int n_run = alist ? *alist_n : n;
    for (int k = blockIdx.x * tpc + team; k < n_run; k += nt)
        nbr_search_team<G>(alist ? alist[k] : k, pos, cg, cell_count, members, cell_of, range2,
                           cap, nnei, row_start, nbr, dr, types, ety, err, sm + team * G, w, lane,
                           1 + team);
}

// Device MD loop with a Verlet skin: the exact rc list filtered out of each atom's
// candidate row (within rc + skin), the rows rebuilt by the cell-list scan only on
// steps whose flag a drift set (some atom moved more than skin/2 since the last
// build).  Every CTA reads the flag first; the last CTA to finish a rebuild clears
// it, so the force kernel's drift can raise it again for the next step.
template <int G>
__global__ __launch_bounds__(kSearchCTA, 2) void k_nbr_search_v(
    int n, const double* __restrict__ pos, CellGrid cg, const int* __restrict__ cell_count,
    const int* __restrict__ members, const int* __restrict__ cell_of, double range2, int cap,
    int* __restrict__ nnei, int* __restrict__ row_start, int* __restrict__ nbr,
    double* __restrict__ dr, const int* __restrict__ types, int* __restrict__ ety,
    unsigned* err, VList vl) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    NbrSmem* sm = reinterpret_cast<NbrSmem*>(smem_raw);
    pdl_launch_dependents();
    pdl_wait();
    const bool rebuild = *reinterpret_cast<volatile int*>(vl.flag) != 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tpc = (blockDim.x >> 5) / G, team = warp / G, w = warp % G;
    const int nt = gridDim.x * tpc;
    for (int i = blockIdx.x * tpc + team; i < n; i += nt) {
        if (rebuild) {  // candidate row (indices only, ascending) + reference position
            nbr_search_team<G>(i, pos, cg, cell_count, members, cell_of, vl.range2, vl.cap,
                               vl.cnt, nullptr, vl.list, nullptr, types, nullptr, err,
                               sm + team * G, w, lane, 1 + team);
            if (w == 0 && lane < 3) vl.xref[3 * i + lane] = pos[3 * i + lane];
        }
        nbr_filter_team<G>(i, pos, cg, vl, range2, cap, nnei, row_start, nbr, dr, types, ety, err,
                           sm + team * G, w, lane, 1 + team);
    }
    if (rebuild) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            auto* done = reinterpret_cast<unsigned*>(vl.flag + 1);
            if (atomicAdd(done, 1u) == gridDim.x - 1) {
                *done = 0u;
                vl.flag[0] = 0;
                ++vl.flag[2];  // rebuild count (hmdp_md_stats)
            }
        }
    }
}

// CSR offsets -> (row_start, nnei)
__global__ void k_csr_rows(int n, const int* __restrict__ offset, int* __restrict__ row_start,
                           int* __restrict__ nnei) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    row_start[i] = offset[i];
    nnei[i] = offset[i + 1] - offset[i];
}

// Generic in-edge lists (transpose of an arbitrary CSR, e.g. a caller-built
// NnInput with ghosts): count, single-CTA exclusive scan, fill, then a per-atom
// sort by edge id so that every gather sums in a fixed order.
__global__ void k_in_count(int ne, const int* __restrict__ nbr, int* __restrict__ in_cnt) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= ne) return;
    atomicAdd(in_cnt + nbr[e], 1);
}
__global__ void k_scan_single(int n, const int* __restrict__ cnt, int* __restrict__ start) {
    __shared__ int s_carry;
    __shared__ int s_w[32];
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int base = 0; base < n; base += blockDim.x) {
        const int i = base + threadIdx.x;
        const int own = i < n ? cnt[i] : 0;
        int v = own;
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(FULL_MASK, v, o);
            if (lane >= o) v += u;
        }
        if (lane == 31) s_w[w] = v;
        __syncthreads();
        if (w == 0) {
            int x = lane < static_cast<int>(blockDim.x >> 5) ? s_w[lane] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(FULL_MASK, x, o);
                if (lane >= o) x += u;
            }
            s_w[lane] = x;
        }
        __syncthreads();
        const int incl = v + (w > 0 ? s_w[w - 1] : 0) + s_carry;
        if (i < n) start[i] = incl - own;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) s_carry = incl;
        __syncthreads();
    }
}
__global__ void k_in_fill(int ne, const int* __restrict__ nbr, const int* __restrict__ in_start,
                          int* __restrict__ cursor, int* __restrict__ in_edge) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= ne) return;
    const int j = nbr[e];
    const int slot = atomicAdd(cursor + j, 1);
    in_edge[in_start[j] + slot] = e;
}
__global__ void k_in_sort(int n, const int* __restrict__ in_start, const int* __restrict__ in_cnt,
                          int* __restrict__ in_edge) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int* a = in_edge + in_start[i];
    const int m = in_cnt[i];
    for (int p = 1; p < m; ++p) {  // insertion sort: lists are ~30 long
        const int v = a[p];
        int q = p - 1;
        while (q >= 0 && a[q] > v) {
            a[q + 1] = a[q];
            --q;
        }
        a[q + 1] = v;
    }
}

// Generic CSR path: neighbour types per edge and the mirror index of each edge.
__global__ void k_edge_meta(int ne, const int* __restrict__ nbr, const int* __restrict__ types,
                            int* __restrict__ ety) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < ne) ety[e] = types[nbr[e]];
}
__global__ void k_inv_pos(int ne, const int* __restrict__ in_edge, int* __restrict__ inv_pos) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < ne) inv_pos[in_edge[q]] = q;
}

// FP64 descriptors() (inference.cpp:430-447): one warp per atom, lane = (type, k).
__global__ __launch_bounds__(128) void k_descriptors_f64(DevModel<double> md, DevGraph gr,
                                                         double* __restrict__ desc) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i = blockIdx.x * 4 + w;
    if (i >= gr.n) return;
    const int nd = md.n_types * kK;
    if (lane >= nd) return;
    const int ty = lane >> 3, k = lane & 7;
    double acc = 0.0;
    const int start = gr.row_start[i], cnt = gr.nnei[i];
    const double rc = static_cast<double>(md.rc), onset = 0.9 * rc;
    for (int q = 0; q < cnt; ++q) {  // CSR order, as the reference
        const int e = start + q;
        if (gr.types[gr.nbr[e]] != ty) continue;
        const double* d = gr.dr + 3ll * e;
        const double r = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        double s;  // switch_value (FP64 API form, inference.cpp:34-39)
        if (r <= onset) s = 1.0;
        else if (r >= rc) s = 0.0;
        else s = 0.5 * (cos(M_PI * (r - onset) / (0.1 * rc)) + 1.0);
        const double x = r - md.mu[k];
        acc += exp(-x * x * md.inv2w2) * s;
    }
    desc[static_cast<long long>(i) * nd + lane] = acc;
}

__global__ void k_vv_kick_drift_bin(int n, MdFuse mf, const double* __restrict__ f,
                                    unsigned* err) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    vv_kick_drift_bin_atom(i, mf, f, err);
}

// NNPot extraction: group-local positions and types.
__global__ void k_gather_group(int ng, const int* __restrict__ idx, const double* __restrict__ xyz,
                               const int* __restrict__ types, double* __restrict__ pos_out,
                               int* __restrict__ types_out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= ng) return;
    const int j = idx[k];
    pos_out[3 * k] = xyz[3 * j];
    pos_out[3 * k + 1] = xyz[3 * j + 1];
    pos_out[3 * k + 2] = xyz[3 * j + 2];
    types_out[k] = types[j];
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
int team_override();  // hmdp_net.cu

int num_sms() {
    static thread_local int dev_cached = -1, sms_cached = 148;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != dev_cached) {
        cudaDeviceGetAttribute(&sms_cached, cudaDevAttrMultiProcessorCount, dev);
        dev_cached = dev;
    }
    return sms_cached;
}

// Binning of a list of atoms only (halo-exchange DD: the other rows are stale).
__global__ void k_cell_bin_list(const int* __restrict__ list, const int* __restrict__ list_n,
                                const double* __restrict__ pos, CellGrid cg,
                                int* __restrict__ cell_count, int* __restrict__ members,
                                int* __restrict__ cell_of, unsigned* err) {
    const int cnt = *list_n;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < cnt; k += gridDim.x * blockDim.x) {
        const int i = list[k];
        bin_atom(i, pos + 3 * i, cg, cell_count, members, cell_of, err);
    }
}
void launch_cell_bin_list(const int* list, const int* list_n, int n_max, const double* pos,
                          const CellGrid& cg, int* cell_count, int* members, int* cell_of,
                          unsigned* err, cudaStream_t st) {
    k_cell_bin_list<<<(n_max + 127) / 128, 128, 0, st>>>(list, list_n, pos, cg, cell_count,
                                                         members, cell_of, err);
}
void launch_cell_bin(int n, const double* pos, const CellGrid& cg, int* cell_count, int* members,
                     int* cell_of, unsigned* err, cudaStream_t st) {
    k_cell_bin<<<(n + 127) / 128, 128, 0, st>>>(n, pos, cg, cell_count, members, cell_of, err);
}
void launch_stage_bin(int n, const double* hx, const int* ht, double* pos, int* types,
                      const CellGrid& cg, int* cell_count, int* members, int* cell_of,
                      unsigned* err, cudaStream_t st, const double* xref, int* vflag,
                      double vhalf2) {
    k_stage_bin<<<(n + 127) / 128, 128, 0, st>>>(n, hx, ht, pos, types, cg, cell_count, members,
                                                 cell_of, err, xref, vflag, vhalf2);
}
void launch_nbr_search(int n, const double* pos, const CellGrid& cg, const int* cell_count,
                       const int* members, const int* cell_of, double range2, int cap, int* nnei,
                       int* row_start, int* nbr, double* dr, const int* types, int* ety,
                       unsigned* err, cudaStream_t st, const int* alist, const int* alist_n,
                       const VList* vl) {
    const int sms = num_sms();
    // team size by system size: 4 warps per atom up to 4 atoms per SM, 2 up to 16 per
    // SM (one round of 2-warp teams), then 1 (measured: 3LZM, 18 atoms per SM, with 1
    // instead of 2: DPA3 +2.2 %, DPA2 +6.7 %; 1UBQ with 1: -7 %)
    int G = (4 * n <= 16 * sms) ? 4 : (n <= 16 * sms ? 2 : 1);
    if (team_override()) G = team_override();
    static const int g_env = [] {
        const char* e = std::getenv("HMDP_SEARCH_G");
        const int v = e ? std::atoi(e) : 0;
        return (v == 1 || v == 2 || v == 4) ? v : 0;
    }();
    if (g_env) G = g_env;
    // The kernel holds 32 warps per SM (64 registers): 2 CTAs of up to 16 warps.
    // Atoms per SM m = ceil(n / sms); one round when m teams fit on the SM, and the
    // CTAs are shaped so that every SM carries the same number of atoms (2PTC: two
    // 14-warp CTAs per SM, 28 atoms each, instead of 258 16-warp CTAs that left 38 SMs
    // half loaded); never more CTAs than one resident wave (3LZM had 331: a partial
    // second wave), the teams grid-stride over the rest.
    const int m = (n + sms - 1) / sms;
    const int per_sm_teams = 32 / G;
    int teams;
    if (m <= 16 / G) {
        teams = m < 1 ? 1 : m;  // one CTA per SM
    } else {
        const int round_teams = m <= per_sm_teams ? m : per_sm_teams;
        teams = (round_teams + 1) / 2;  // two CTAs per SM
        teams = teams > 16 / G ? 16 / G : teams;
    }
    static const int t_env = [] {
        const char* e = std::getenv("HMDP_SEARCH_T");
        return e ? std::atoi(e) : 0;
    }();
    if (t_env > 0 && t_env * G <= 16) teams = t_env;
    const int threads = 32 * G * teams;
    int grid = (n + teams - 1) / teams;
    const int resident = sms * (32 / (G * teams));  // 64 registers: 32 warps per SM
    grid = grid < resident ? grid : resident;
    const size_t smem = static_cast<size_t>(G * teams) * sizeof(NbrSmem);
    auto args = [&](auto kernel) {
        launch_pdl(kernel, dim3(grid > 0 ? grid : 1), dim3(threads), smem, st, n, pos, cg,
                   cell_count, members, cell_of, range2, cap, nnei, row_start, nbr, dr, types, ety,
                   err, alist, alist_n);
    };
    if (vl) {
        auto vargs = [&](auto kernel) {
            launch_pdl(kernel, dim3(grid > 0 ? grid : 1), dim3(threads), smem, st, n, pos, cg,
                       cell_count, members, cell_of, range2, cap, nnei, row_start, nbr, dr, types,
                       ety, err, *vl);
        };
        if (G == 4) vargs(k_nbr_search_v<4>);
        else if (G == 2) vargs(k_nbr_search_v<2>);
        else vargs(k_nbr_search_v<1>);
        return;
    }
    if (G == 4) args(k_nbr_search<4>);
    else if (G == 2) args(k_nbr_search<2>);
    else args(k_nbr_search<1>);
}
cudaError_t nbr_configure() {
    const cudaFuncAttribute a = cudaFuncAttributeMaxDynamicSharedMemorySize;
    cudaError_t e = cudaSuccess;
    for (cudaError_t r : {cudaFuncSetAttribute(k_nbr_search<1>, a, 16 * sizeof(NbrSmem)),
                          cudaFuncSetAttribute(k_nbr_search<2>, a, 16 * sizeof(NbrSmem)),
                          cudaFuncSetAttribute(k_nbr_search<4>, a, 16 * sizeof(NbrSmem)),
                          cudaFuncSetAttribute(k_nbr_search_v<1>, a, 16 * sizeof(NbrSmem)),
                          cudaFuncSetAttribute(k_nbr_search_v<2>, a, 16 * sizeof(NbrSmem)),
                          cudaFuncSetAttribute(k_nbr_search_v<4>, a, 16 * sizeof(NbrSmem))})
        if (r != cudaSuccess) e = r;
    return e;
}
void launch_edge_meta(int ne, const int* nbr, const int* types, int* ety, const int* in_edge,
                      int* inv_pos, cudaStream_t st) {
    if (ne <= 0) return;
    k_edge_meta<<<(ne + 255) / 256, 256, 0, st>>>(ne, nbr, types, ety);
    k_inv_pos<<<(ne + 255) / 256, 256, 0, st>>>(ne, in_edge, inv_pos);
}
void launch_csr_rows(int n, const int* offset, int* row_start, int* nnei, cudaStream_t st) {
    k_csr_rows<<<(n + 127) / 128, 128, 0, st>>>(n, offset, row_start, nnei);
}
void launch_in_edges(int n, int ne, const int* nbr, int* in_cnt, int* in_start, int* cursor,
                     int* in_edge, cudaStream_t st) {
    cudaMemsetAsync(in_cnt, 0, sizeof(int) * n, st);
    cudaMemsetAsync(cursor, 0, sizeof(int) * n, st);
    if (ne > 0) k_in_count<<<(ne + 255) / 256, 256, 0, st>>>(ne, nbr, in_cnt);
    k_scan_single<<<1, 1024, 0, st>>>(n, in_cnt, in_start);
    if (ne > 0) k_in_fill<<<(ne + 255) / 256, 256, 0, st>>>(ne, nbr, in_start, cursor, in_edge);
    k_in_sort<<<(n + 127) / 128, 128, 0, st>>>(n, in_start, in_cnt, in_edge);
}
void launch_descriptors_f64(const DevModel<double>& md, const DevGraph& gr, double* desc,
                            cudaStream_t st) {
    k_descriptors_f64<<<(gr.n + 3) / 4, 128, 0, st>>>(md, gr, desc);
}
void launch_vv_kick_drift_bin(int n, const MdFuse& mf, const double* f, unsigned* err,
                              cudaStream_t st) {
    k_vv_kick_drift_bin<<<(n + 127) / 128, 128, 0, st>>>(n, mf, f, err);
}

void launch_gather_group(int ng, const int* idx, const double* xyz, const int* types,
                         double* pos_out, int* types_out, cudaStream_t st) {
    k_gather_group<<<(ng + 127) / 128, 128, 0, st>>>(ng, idx, xyz, types, pos_out, types_out);
}

}  // namespace hmdp
