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
#include "hmdp_common.cuh"

namespace hmdp {

struct GddGeom {
    int d[3];      // rank grid
    double L[3];   // box
    int rank;
    double halo;   // halo width (rc)
};

// roles + lists: lists[0..n) owned, lists[n..2n) halo, lists[2n..3n) searched
// (owned + halo); counts[0..2] their lengths (zeroed by the caller each step).
__global__ void k_gdd_roles(int n, const double* __restrict__ pos, GddGeom g,
                            unsigned char* __restrict__ role, int* __restrict__ lists,
                            int* __restrict__ counts) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int rc3[3] = {g.rank % g.d[0], (g.rank / g.d[0]) % g.d[1], g.rank / (g.d[0] * g.d[1])};
    bool owned = true;
    double dist2 = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double L = g.L[a];
        double r = pos[3 * i + a];
        r = r - L * floor(r / L);  // wrap_position (box.hpp:34-42), as dd.owners
        if (r >= L) r = 0.0;
        int c = static_cast<int>(r / L * g.d[a]);
        c = c < 0 ? 0 : (c > g.d[a] - 1 ? g.d[a] - 1 : c);
        if (c != rc3[a]) owned = false;
        if (g.d[a] > 1) {  // periodic distance to this rank's slab [lo, hi)
            const double lo = L * rc3[a] / g.d[a], hi = L * (rc3[a] + 1) / g.d[a];
            double da = 0.0;
            if (r < lo || r >= hi) {
                double a1 = lo - r, a2 = r - hi;
                a1 -= L * floor(a1 / L);
                a2 -= L * floor(a2 / L);
                da = a1 < a2 ? a1 : a2;
            }
            dist2 += da * da;
        }
    }
    // the ownership test and the slab bounds may disagree at a boundary by rounding:
    // an owned atom is always searched
    const bool halo = !owned && dist2 <= g.halo * g.halo * (1.0 + 1e-9) + 1e-24;
    const unsigned char ro = owned ? 1 : (halo ? 2 : 0);
    role[i] = ro;
    if (owned) lists[atomicAdd(counts + 0, 1)] = i;
    if (halo) lists[n + atomicAdd(counts + 1, 1)] = i;
    if (ro) lists[2 * n + atomicAdd(counts + 2, 1)] = i;
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
                           long long slots, T* __restrict__ grev, T* __restrict__ g) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    const int n_run = *gr.alist_n;
    for (int k = warp; k < n_run; k += nw) {
        const int i = gr.alist[k];
        const int start = gr.row_start[i], cnt = gr.nnei[i];
        const bool own_row = role[i] == 1;
        for (int q = 0; q < cnt; ++q) {
            const long long e = start + q;
            if (role[gr.nbr[e]] != 1) {
                if (d) {
                    d[e * kH + lane] = T(0);
                    d[(slots + e) * kH + lane] = T(0);
                }
                if (lane == 0) grev[e] = T(0);
            }
            if (!own_row && lane == 0) g[e] = T(0);
        }
    }
}

__global__ void k_gdd_zero_energy(int n, const unsigned char* __restrict__ role,
                                  double* __restrict__ e_atom) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && role[i] != 1) e_atom[i] = 0.0;
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
__global__ void k_gdd_integrate(int n, const double* __restrict__ f, double* __restrict__ x,
                                double* __restrict__ v, const double* __restrict__ m, double half,
                                double dt, int mode, unsigned* err) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
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
                      int* counts, cudaStream_t st) {
    k_gdd_roles<<<(n + 255) / 256, 256, 0, st>>>(n, pos, g, role, lists, counts);
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
    k_gdd_zero<T><<<warp_grid(n_est), 256, 0, st>>>(gr, role, d, slots, grev, g);
    k_gdd_zero_energy<<<(gr.n + 255) / 256, 256, 0, st>>>(gr.n, role, e_atom);
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
                          double dt, int mode, unsigned* err, cudaStream_t st) {
    k_gdd_integrate<<<(n + 255) / 256, 256, 0, st>>>(n, f, x, v, m, 0.5 * dt, dt, mode, err);
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

}  // namespace hmdp
