// hmdp_ff.cu — the reference's classical force field on the device (SURVEY §8(f)
// item 4: the solvent / cross-group terms of the protein-in-water hybrid), so the
// whole hybrid step can stay on the GPU.  Same functions as
// /root/reference/proj/src/forcefield.cpp:
//   bonded_impl   :50-134  harmonic bonds, harmonic angles (clamped derivative near
//                          collinear), periodic dihedrals
//   pair_loop     :139-193 + lj_impl :195-216 (potential-shifted LJ, Lorentz-Berthelot)
//                 + coulomb_impl :218-245 (cutoff_shifted or reaction_field)
//   compute_classical :265-279
// Pairs: the device cell-list neighbour list at the pair cutoff (the pairs of
// build_neighbor_list(.., rc, skin 0), neighborlist.cpp:42-113) minus the
// topology's exclusions; one warp per atom gathers its own force over its FULL
// list (no atomics), each pair's energy and virial are counted once (j > i).
// Bonded terms: one thread per term writes its per-atom contributions to fixed
// slots, one thread per atom then sums its slots in a fixed order — runs are
// deterministic.  T = the reference's Precision (float or double arithmetic);
// forces, energies and virials accumulate in FP64.
#include "hmdp_common.cuh"

namespace hmdp {

struct FfDev {
    int n, n_types, scheme;  // scheme 0 cutoff_shifted, 1 reaction_field
    double rc_lj, rc_c, k_rf, c_rf, fpre;
    const double* sigma;
    const double* eps;
    const double* q;
    const int* type;
    const int* exo;  // exclusion CSR (sorted per atom)
    const int* exc;
    int nb, na, nd;
    const int* bi;      // [nb][2]
    const double* bp;   // [nb][2] k_b, r0
    const int* ai;      // [na][3]
    const double* ap;   // [na][2] k_a, theta0
    const int* di;      // [nd][4]
    const double* dp;   // [nd][3] k_d, phase, multiplicity
    const int* aso;     // atom -> contribution slots (CSR, slot order)
    const int* asl;
    double L[3];
};

constexpr int kFfCTA = 128;

__device__ __forceinline__ bool ff_excluded(const FfDev& f, int i, int j) {
    int lo = f.exo[i], hi = f.exo[i + 1] - 1;
    while (lo <= hi) {
        const int mid = (lo + hi) >> 1;
        const int v = f.exc[mid];
        if (v == j) return true;
        if (v < j) lo = mid + 1;
        else hi = mid - 1;
    }
    return false;
}

// part[blk][0..2] = E_lj, E_coulomb, pair virial of this CTA's atoms
template <typename T>
__global__ __launch_bounds__(kFfCTA) void k_ff_pairs(FfDev f, DevGraph gr, double* __restrict__ F,
                                                     double* __restrict__ part, unsigned* err) {
    __shared__ double s[kFfCTA / 32][3];
    const int lane = threadIdx.x & 31, wc = threadIdx.x >> 5;
    const int nw = gridDim.x * (kFfCTA / 32);
    double elj = 0.0, ec = 0.0, vir = 0.0;
    const T rlj = T(f.rc_lj), rcc = T(f.rc_c), fpre = T(f.fpre), krf = T(f.k_rf), crf = T(f.c_rf);
    for (int i = blockIdx.x * (kFfCTA / 32) + wc; i < f.n; i += nw) {
        const int start = gr.row_start[i], cnt = gr.nnei[i];
        const int ti = f.type[i];
        const T qi = T(f.q[i]);
        double fx = 0.0, fy = 0.0, fz = 0.0;
        for (int q = lane; q < cnt; q += 32) {
            const int e = start + q;
            const int j = gr.nbr[e];
            if (ff_excluded(f, i, j)) continue;
            const T x = T(gr.dr[3ll * e]), y = T(gr.dr[3ll * e + 1]), z = T(gr.dr[3ll * e + 2]);
            const T r2 = x * x + y * y + z * z;
            if (r2 < T(1e-8)) {  // kOverlapDistance^2 (forcefield.cpp:15, :161-165)
                atomicOr(err, kErrZeroEdge);
                continue;
            }
            const T r = d_sqrt(r2);
            T dv = T(0), vlj = T(0), vc = T(0);
            if (r <= rlj) {  // lj_impl :198-215
                const int tj = f.type[j];
                const T sig = T(0.5 * (f.sigma[ti] + f.sigma[tj]));
                const T ep = T(sqrt(f.eps[ti] * f.eps[tj]));
                if (ep != T(0)) {
                    const T sr2 = (sig / r) * (sig / r);
                    const T sr6 = sr2 * sr2 * sr2, sr12 = sr6 * sr6;
                    const T sc2 = (sig / rlj) * (sig / rlj);
                    const T sc6 = sc2 * sc2 * sc2;
                    dv += -T(24) * ep / r * (T(2) * sr12 - sr6);
                    vlj = T(4) * ep * (sr12 - sr6) - T(4) * ep * (sc6 * sc6 - sc6);
                }
            }
            if (r <= rcc) {  // coulomb_impl :221-244
                const T qq = qi * T(f.q[j]);
                if (qq != T(0)) {
                    if (f.scheme == 0) {
                        dv += -fpre * qq / (r * r);
                        vc = fpre * qq * (T(1) / r - T(1) / rcc);
                    } else {
                        dv += fpre * qq * (-T(1) / (r * r) + T(2) * krf * r);
                        vc = fpre * qq * (T(1) / r + krf * r * r - crf);
                    }
                }
            }
            // f_j = dr (-dV/dr / r), f_i = -f_j
            const T c = dv / r;
            fx += static_cast<double>(x * c);
            fy += static_cast<double>(y * c);
            fz += static_cast<double>(z * c);
            if (j > i) {
                elj += static_cast<double>(vlj);
                ec += static_cast<double>(vc);
                vir += -static_cast<double>(dv * r);
            }
        }
        fx = warp_sum(fx);
        fy = warp_sum(fy);
        fz = warp_sum(fz);
        if (lane == 0) {
            F[3 * i] = fx;
            F[3 * i + 1] = fy;
            F[3 * i + 2] = fz;
        }
    }
    elj = warp_sum(elj);
    ec = warp_sum(ec);
    vir = warp_sum(vir);
    if (lane == 0) {
        s[wc][0] = elj;
        s[wc][1] = ec;
        s[wc][2] = vir;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        double v = 0.0;
        for (int w = 0; w < kFfCTA / 32; ++w) v += s[w][threadIdx.x];
        part[3 * blockIdx.x + threadIdx.x] = v;
    }
}

template <typename T>
struct V3 {
    T x, y, z;
};
template <typename T>
__device__ __forceinline__ V3<T> ff_dr(const FfDev& f, const double* pos, int a, int b) {
    // ts.min_image(ts.pos[b] - ts.pos[a]) in T (forcefield.cpp:29-35)
    T d[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const T L = T(f.L[k]);
        T v = T(pos[3 * b + k]) - T(pos[3 * a + k]);
        v -= L * rint(v / L);
        d[k] = v;
    }
    return {d[0], d[1], d[2]};
}
template <typename T>
__device__ __forceinline__ T dot3(V3<T> a, V3<T> b) {
    return a.x * b.x + a.y * b.y + a.z * b.z;
}
template <typename T>
__device__ __forceinline__ V3<T> cross3(V3<T> a, V3<T> b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
template <typename T>
__device__ __forceinline__ V3<T> scl(V3<T> a, T s) {
    return {a.x * s, a.y * s, a.z * s};
}
template <typename T>
__device__ __forceinline__ V3<T> sub(V3<T> a, V3<T> b) {
    return {a.x - b.x, a.y - b.y, a.z - b.z};
}
template <typename T>
__device__ __forceinline__ void put(double* c, long long slot, V3<T> v) {
    c[3 * slot] = static_cast<double>(v.x);
    c[3 * slot + 1] = static_cast<double>(v.y);
    c[3 * slot + 2] = static_cast<double>(v.z);
}

// one thread per bonded term: contributions to slots, (E, W) per term
template <typename T>
__global__ void k_ff_bonded(FfDev f, const double* __restrict__ pos, double* __restrict__ contrib,
                            double* __restrict__ term_ew, int* collinear) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int nt = f.nb + f.na + f.nd;
    if (t >= nt) return;
    T e = T(0), w = T(0);
    if (t < f.nb) {  // bonds :58-67
        const int i = f.bi[2 * t], j = f.bi[2 * t + 1];
        const V3<T> dr = ff_dr<T>(f, pos, i, j);
        const T r = d_sqrt(dot3(dr, dr));
        const T dev = r - T(f.bp[2 * t + 1]);
        e = T(0.5) * T(f.bp[2 * t]) * dev * dev;
        const V3<T> fj = scl(dr, -(T(f.bp[2 * t]) * dev) / r);
        put(contrib, 2ll * t, scl(fj, T(-1)));  // i
        put(contrib, 2ll * t + 1, fj);          // j
        w = dot3(dr, fj);
    } else if (t < f.nb + f.na) {  // angles :69-93
        const int a = t - f.nb;
        const int i = f.ai[3 * a], j = f.ai[3 * a + 1], k = f.ai[3 * a + 2];
        const V3<T> u = ff_dr<T>(f, pos, j, i), v = ff_dr<T>(f, pos, j, k);
        const T nu = d_sqrt(dot3(u, u)), nv = d_sqrt(dot3(v, v));
        T cs = dot3(u, v) / (nu * nv);
        cs = cs < T(-1) ? T(-1) : (cs > T(1) ? T(1) : cs);
        T sn = d_sqrt(T(1) - cs * cs);
        if (sn < T(1e-9)) {
            sn = T(1e-9);
            atomicAdd(collinear, 1);
        }
        const T theta = acos(cs);
        const T dev = theta - T(f.ap[2 * a + 1]);
        e = T(0.5) * T(f.ap[2 * a]) * dev * dev;
        const T dEdt = T(f.ap[2 * a]) * dev;
        const V3<T> dtu = scl(sub(scl(v, T(1) / nv), scl(u, cs / nu)), T(-1) / (nu * sn));
        const V3<T> dtv = scl(sub(scl(u, T(1) / nu), scl(v, cs / nv)), T(-1) / (nv * sn));
        const V3<T> fi = scl(dtu, -dEdt), fk = scl(dtv, -dEdt);
        const long long base = 2ll * f.nb + 3ll * a;
        put(contrib, base, fi);
        put(contrib, base + 1, scl(V3<T>{fi.x + fk.x, fi.y + fk.y, fi.z + fk.z}, T(-1)));
        put(contrib, base + 2, fk);
        w = dot3(u, fi) + dot3(v, fk);
    } else {  // dihedrals :95-126
        const int d = t - f.nb - f.na;
        const int i = f.di[4 * d], j = f.di[4 * d + 1], k = f.di[4 * d + 2], l = f.di[4 * d + 3];
        const V3<T> b1 = ff_dr<T>(f, pos, i, j), b2 = ff_dr<T>(f, pos, j, k),
                    b3 = ff_dr<T>(f, pos, k, l);
        const V3<T> n1 = cross3(b1, b2), n2 = cross3(b2, b3);
        const T nb2 = d_sqrt(dot3(b2, b2));
        T n1sq = dot3(n1, n1), n2sq = dot3(n2, n2);
        n1sq = n1sq > T(1e-12) ? n1sq : T(1e-12);
        n2sq = n2sq > T(1e-12) ? n2sq : T(1e-12);
        const T phi = atan2(dot3(cross3(n1, n2), b2) / nb2, dot3(n1, n2));
        const T kd = T(f.dp[3 * d]), ph = T(f.dp[3 * d + 1]), mu = T(f.dp[3 * d + 2]);
        const T arg = mu * phi - ph;
        e = kd * (T(1) + cos(arg));
        const T dEdp = -kd * mu * sin(arg);
        const V3<T> dpi = scl(n1, -nb2 / n1sq), dpl = scl(n2, nb2 / n2sq);
        const T t1 = dot3(b1, b2) / (nb2 * nb2), t3 = dot3(b3, b2) / (nb2 * nb2);
        const V3<T> dpj = sub(scl(dpi, t1 - T(1)), scl(dpl, t3));
        const V3<T> dpk = sub(scl(dpl, t3 - T(1)), scl(dpi, t1));
        const V3<T> fi = scl(dpi, -dEdp), fj = scl(dpj, -dEdp), fk = scl(dpk, -dEdp),
                    fl = scl(dpl, -dEdp);
        const long long base = 2ll * f.nb + 3ll * f.na + 4ll * d;
        put(contrib, base, fi);
        put(contrib, base + 1, fj);
        put(contrib, base + 2, fk);
        put(contrib, base + 3, fl);
        const V3<T> b12 = {b1.x + b2.x, b1.y + b2.y, b1.z + b2.z};
        const V3<T> b123 = {b12.x + b3.x, b12.y + b3.y, b12.z + b3.z};
        w = dot3(b1, fj) + dot3(b12, fk) + dot3(b123, fl);
    }
    term_ew[2 * t] = static_cast<double>(e);
    term_ew[2 * t + 1] = static_cast<double>(w);
}

// F[i] += sum of i's bonded contribution slots (fixed slot order)
__global__ void k_ff_gather(FfDev f, const double* __restrict__ contrib, double* __restrict__ F) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= f.n) return;
    double s[3] = {0, 0, 0};
    for (int k = f.aso[i]; k < f.aso[i + 1]; ++k) {
        const long long sl = f.asl[k];
#pragma unroll
        for (int a = 0; a < 3; ++a) s[a] += contrib[3 * sl + a];
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) F[3 * i + a] += s[a];
}

// out[0..3] = E_bonded, E_lj, E_coulomb, virial (one CTA, fixed order)
__global__ void k_ff_reduce(int nblk, const double* __restrict__ part, int nt,
                            const double* __restrict__ term_ew, double* __restrict__ out) {
    __shared__ double s[4][kFfCTA];
    double v[4] = {0, 0, 0, 0};
    for (int b = threadIdx.x; b < nblk; b += kFfCTA) {
        v[1] += part[3 * b];
        v[2] += part[3 * b + 1];
        v[3] += part[3 * b + 2];
    }
    for (int t = threadIdx.x; t < nt; t += kFfCTA) {
        v[0] += term_ew[2 * t];
        v[3] += term_ew[2 * t + 1];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) s[k][threadIdx.x] = v[k];
    __syncthreads();
    if (threadIdx.x < 4) {
        double tot = 0.0;
        for (int q = 0; q < kFfCTA; ++q) tot += s[threadIdx.x][q];
        out[threadIdx.x] = tot;
    }
}

// dst[group[k]] += src[k] (the NNPot scatter of group forces)
__global__ void k_scatter_add3(int ng, const int* __restrict__ grp, const double* __restrict__ src,
                               double* __restrict__ dst) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= ng) return;
    const int i = grp[k];
#pragma unroll
    for (int a = 0; a < 3; ++a) dst[3 * i + a] += src[3 * k + a];
}
void launch_scatter_add3(int ng, const int* grp, const double* src, double* dst, cudaStream_t st) {
    if (ng > 0) k_scatter_add3<<<(ng + 127) / 128, 128, 0, st>>>(ng, grp, src, dst);
}

int ff_grid(int n) {
    const int want = (n + kFfCTA / 32 - 1) / (kFfCTA / 32);
    return want < 1 ? 1 : (want > 4096 ? 4096 : want);
}

template <typename T>
void launch_ff(const FfDev& f, const DevGraph& gr, const double* pos, double* F, double* part,
               double* contrib, double* term_ew, int* collinear, double* out, unsigned* err,
               cudaStream_t st) {
    const int nblk = ff_grid(f.n);
    k_ff_pairs<T><<<nblk, kFfCTA, 0, st>>>(f, gr, F, part, err);
    const int nt = f.nb + f.na + f.nd;
    if (nt > 0) {
        k_ff_bonded<T><<<(nt + 127) / 128, 128, 0, st>>>(f, pos, contrib, term_ew, collinear);
        k_ff_gather<<<(f.n + 127) / 128, 128, 0, st>>>(f, contrib, F);
    }
    k_ff_reduce<<<1, kFfCTA, 0, st>>>(nblk, part, nt, term_ew, out);
}
template void launch_ff<float>(const FfDev&, const DevGraph&, const double*, double*, double*,
                               double*, double*, int*, double*, unsigned*, cudaStream_t);
template void launch_ff<double>(const FfDev&, const DevGraph&, const double*, double*, double*,
                                double*, double*, int*, double*, unsigned*, cudaStream_t);

}  // namespace hmdp
