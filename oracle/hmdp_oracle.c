/* hmdp_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * CPU restatement of the reference hot path, compiled twice by oracle/Makefile:
 *   -DORA_REAL=double -DORA_SFX=f64   (Precision::fp64, evaluate_impl<double>)
 *   -DORA_REAL=float  -DORA_SFX=f32   (Precision::fp32, evaluate_impl<float>)
 * with -ffp-contract=off so every expression rounds exactly as written, in the
 * same operation order as the reference C++ (cited per function below).
 * Reference paths are relative to /root/reference/proj.
 */
#include "hmdp_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <tgmath.h>

#ifndef ORA_REAL
#define ORA_REAL double
#define ORA_SFX f64
#endif
typedef ORA_REAL real;
#define ORA_CAT2(a, b) a##_##b
#define ORA_CAT(a, b) ORA_CAT2(a, b)
#define ORA_FN(name) ORA_CAT(name, ORA_SFX)

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

#ifndef ORA_NO_COMMON
static _Thread_local char g_err[512];
const char* ora_last_error(void) { return g_err; }
void ora_set_error(const char* msg) {
    strncpy(g_err, msg, sizeof g_err - 1);
    g_err[sizeof g_err - 1] = 0;
}
#else
void ora_set_error(const char* msg);
#endif

/* ------------------------------------------------------------------------- */
/* Shared FP64 geometry + neighbour search (built once, in the f64 TU).       */
/* ------------------------------------------------------------------------- */
#ifndef ORA_NO_COMMON

/* minimum_image, include/halomd/box.hpp:24-31 (all axes periodic, L > 0). */
static void min_image(double d[3], const double box[3]) {
    for (int a = 0; a < 3; ++a)
        if (box[a] > 0.0) d[a] -= box[a] * nearbyint(d[a] / box[a]);
}

/* wrap_position, include/halomd/box.hpp:34-42. */
static double wrap1(double r, double L) {
    if (L > 0.0) {
        r -= L * floor(r / L);
        if (r >= L) r = 0.0;
    }
    return r;
}

/* norm2 = dot(a,a) = (x*x + y*y) + z*z, include/halomd/vec3.hpp:57-70. */
static double norm2_3(const double d[3]) { return d[0] * d[0] + d[1] * d[1] + d[2] * d[2]; }

static int cmp_pair(const void* a, const void* b) {
    const long long x = *(const long long*)a, y = *(const long long*)b;
    return (x > y) - (x < y);
}
static int cmp_int(const void* a, const void* b) {
    const int x = *(const int*)a, y = *(const int*)b;
    return (x > y) - (x < y);
}

static int geometry_check(const double box[3], double rc) {
    /* neighborlist.cpp:44-49 (skin = 0 in build_input_periodic, inference.cpp:473). */
    for (int a = 0; a < 3; ++a)
        if (rc > 0.5 * box[a]) {
            char msg[128];
            snprintf(msg, sizeof msg, "rc+skin exceeds half the box length on axis %d", a);
            ora_set_error(msg);
            return -1;
        }
    return 0;
}

/* Half pairs (lo,hi) packed as lo<<32|hi -> sorted full CSR (neighborlist.cpp:104-111,
 * inference.cpp:474-485).  edge_dr = minimum_image(x_j - x_i) recomputed in FP64. */
static int emit_csr(int n, const double* xyz, const double box[3], long long* half, long nh,
                    int cap, int* offset, int* nbr, double* dr) {
    qsort(half, (size_t)nh, sizeof(long long), cmp_pair);
    long long* full = (long long*)malloc(sizeof(long long) * (size_t)(2 * nh + 1));
    for (long k = 0; k < nh; ++k) {
        const long long lo = half[k] >> 32, hi = half[k] & 0xffffffffLL;
        full[2 * k] = half[k];
        full[2 * k + 1] = (hi << 32) | lo;
    }
    qsort(full, (size_t)(2 * nh), sizeof(long long), cmp_pair);
    for (int i = 0; i <= n; ++i) offset[i] = 0;
    for (long k = 0; k < 2 * nh; ++k) offset[(full[k] >> 32) + 1]++;
    for (int i = 1; i <= n; ++i) offset[i] += offset[i - 1];
    const long ne = 2 * nh;
    for (long e = 0; e < ne && e < cap; ++e) {
        const int i = (int)(full[e] >> 32), j = (int)(full[e] & 0xffffffffLL);
        nbr[e] = j;
        double d[3] = {xyz[3 * j] - xyz[3 * i], xyz[3 * j + 1] - xyz[3 * i + 1],
                       xyz[3 * j + 2] - xyz[3 * i + 2]};
        min_image(d, box);
        dr[3 * e] = d[0];
        dr[3 * e + 1] = d[1];
        dr[3 * e + 2] = d[2];
    }
    free(full);
    return (int)ne;
}

/* build_grid (neighborlist.cpp:21-38) + 27-cell deduplicated scan over cells
 * c2 >= c (neighborlist.cpp:62-102). */
int ora_neighbor_csr(int n, const double* xyz, const double* box, double rc, int cap,
                     int* offset, int* nbr, double* dr) {
    if (geometry_check(box, rc)) return -1;
    const double range2 = rc * rc;
    int nc[3];
    for (int a = 0; a < 3; ++a) {
        const int c = (int)floor(box[a] / rc);
        nc[a] = c > 1 ? c : 1;
    }
    const int ncell = nc[0] * nc[1] * nc[2];
    int* cell_of = (int*)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
    int* cstart = (int*)calloc((size_t)ncell + 1, sizeof(int));
    int* members = (int*)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
    for (int i = 0; i < n; ++i) {
        int c[3];
        for (int a = 0; a < 3; ++a) {
            const double r = wrap1(xyz[3 * i + a], box[a]);
            int v = (int)(r / box[a] * nc[a]);
            if (v < 0) v = 0;
            if (v > nc[a] - 1) v = nc[a] - 1;
            c[a] = v;
        }
        cell_of[i] = (c[2] * nc[1] + c[1]) * nc[0] + c[0];
        cstart[cell_of[i] + 1]++;
    }
    for (int c = 0; c < ncell; ++c) cstart[c + 1] += cstart[c];
    {   /* members in ascending atom order, as push_back in i order */
        int* fill = (int*)malloc(sizeof(int) * (size_t)ncell);
        memcpy(fill, cstart, sizeof(int) * (size_t)ncell);
        for (int i = 0; i < n; ++i) members[fill[cell_of[i]]++] = i;
        free(fill);
    }
    long hcap = 1024, nh = 0;
    long long* half = (long long*)malloc(sizeof(long long) * (size_t)hcap);
    for (int cz = 0; cz < nc[2]; ++cz)
        for (int cy = 0; cy < nc[1]; ++cy)
            for (int cx = 0; cx < nc[0]; ++cx) {
                const int c = (cz * nc[1] + cy) * nc[0] + cx;
                if (cstart[c + 1] == cstart[c]) continue;
                int neigh[27], nn = 0;
                for (int dz = -1; dz <= 1; ++dz)
                    for (int dy = -1; dy <= 1; ++dy)
                        for (int dx = -1; dx <= 1; ++dx) {
                            const int x = ((cx + dx) % nc[0] + nc[0]) % nc[0];
                            const int y = ((cy + dy) % nc[1] + nc[1]) % nc[1];
                            const int z = ((cz + dz) % nc[2] + nc[2]) % nc[2];
                            neigh[nn++] = (z * nc[1] + y) * nc[0] + x;
                        }
                qsort(neigh, (size_t)nn, sizeof(int), cmp_int);
                int nu = 0;
                for (int k = 0; k < nn; ++k)
                    if (nu == 0 || neigh[nu - 1] != neigh[k]) neigh[nu++] = neigh[k];
                for (int k = 0; k < nu; ++k) {
                    const int c2 = neigh[k];
                    if (c2 < c) continue;
                    for (int ai = cstart[c]; ai < cstart[c + 1]; ++ai) {
                        const int i = members[ai];
                        const int b0 = (c2 == c) ? ai + 1 : cstart[c2];
                        for (int bi = b0; bi < cstart[c2 + 1]; ++bi) {
                            const int j = members[bi];
                            double d[3] = {xyz[3 * j] - xyz[3 * i], xyz[3 * j + 1] - xyz[3 * i + 1],
                                           xyz[3 * j + 2] - xyz[3 * i + 2]};
                            min_image(d, box);
                            if (norm2_3(d) > range2) continue;
                            const long long lo = i < j ? i : j, hi = i < j ? j : i;
                            if (nh == hcap) {
                                hcap *= 2;
                                half = (long long*)realloc(half, sizeof(long long) * (size_t)hcap);
                            }
                            half[nh++] = (lo << 32) | hi;
                        }
                    }
                }
            }
    const int ne = emit_csr(n, xyz, box, half, nh, cap, offset, nbr, dr);
    free(half);
    free(members);
    free(cstart);
    free(cell_of);
    return ne;
}

int ora_neighbor_bruteforce(int n, const double* xyz, const double* box, double rc, int cap,
                            int* offset, int* nbr, double* dr) {
    if (geometry_check(box, rc)) return -1;
    const double range2 = rc * rc;
    long hcap = 1024, nh = 0;
    long long* half = (long long*)malloc(sizeof(long long) * (size_t)hcap);
    for (int i = 0; i < n; ++i)
        for (int j = i + 1; j < n; ++j) {
            double d[3] = {xyz[3 * j] - xyz[3 * i], xyz[3 * j + 1] - xyz[3 * i + 1],
                           xyz[3 * j + 2] - xyz[3 * i + 2]};
            min_image(d, box);
            if (norm2_3(d) > range2) continue;
            if (nh == hcap) {
                hcap *= 2;
                half = (long long*)realloc(half, sizeof(long long) * (size_t)hcap);
            }
            half[nh++] = ((long long)i << 32) | j;
        }
    const int ne = emit_csr(n, xyz, box, half, nh, cap, offset, nbr, dr);
    free(half);
    return ne;
}

/* switch_value / switch_derivative, inference.cpp:34-45 (FP64 API versions). */
double ora_switch_value(double r, double rc) {
    const double onset = 0.9 * rc;
    if (r <= onset) return 1.0;
    if (r >= rc) return 0.0;
    return 0.5 * (cos(M_PI * (r - onset) / (0.1 * rc)) + 1.0);
}
double ora_switch_derivative(double r, double rc) {
    const double onset = 0.9 * rc;
    if (r <= onset || r >= rc) return 0.0;
    return -0.5 * sin(M_PI * (r - onset) / (0.1 * rc)) * M_PI / (0.1 * rc);
}
#endif /* ORA_NO_COMMON */

/* ------------------------------------------------------------------------- */
/* Model unpacking                                                            */
/* ------------------------------------------------------------------------- */
#define ORA_MAX_LAYERS 8
typedef struct {
    int n_layers;
    int sizes[ORA_MAX_LAYERS + 1];
    real* w[ORA_MAX_LAYERS]; /* cast to T like MlpT's constructor, inference.cpp:73-83 */
    real* b[ORA_MAX_LAYERS];
    int act_offset[ORA_MAX_LAYERS + 1];
    int act_size;
} mlp_t;

typedef struct {
    int family, n_types, K, H, n_msg, n_mlp;
    double rc_d, width_d;
    const double* centers_d;
    mlp_t* mlp; /* embedding, fitting, msg0, upd0, ... */
} model_t;

static int unpack(const int* ilay, const double* dpar, model_t* m) {
    m->family = ilay[0];
    m->n_types = ilay[1];
    m->K = ilay[2];
    m->H = ilay[3];
    m->n_msg = ilay[4];
    m->n_mlp = ilay[5];
    m->rc_d = dpar[0];
    m->width_d = dpar[1];
    m->centers_d = dpar + 2;
    m->mlp = (mlp_t*)calloc((size_t)m->n_mlp, sizeof(mlp_t));
    const int* ip = ilay + 6;
    const double* dp = dpar + 2 + m->K;
    for (int q = 0; q < m->n_mlp; ++q) {
        mlp_t* p = &m->mlp[q];
        p->n_layers = *ip++;
        if (p->n_layers < 1 || p->n_layers > ORA_MAX_LAYERS) return -1;
        for (int l = 0; l <= p->n_layers; ++l) p->sizes[l] = *ip++;
        for (int l = 0; l < p->n_layers; ++l) {
            const int in = p->sizes[l], out = p->sizes[l + 1];
            p->w[l] = (real*)malloc(sizeof(real) * (size_t)in * out);
            p->b[l] = (real*)malloc(sizeof(real) * (size_t)out);
            for (int k = 0; k < in * out; ++k) p->w[l][k] = (real)*dp++;
            for (int k = 0; k < out; ++k) p->b[l][k] = (real)*dp++;
        }
        p->act_size = 0;
        for (int l = 0; l <= p->n_layers; ++l) {
            p->act_offset[l] = p->act_size;
            p->act_size += p->sizes[l];
        }
    }
    return 0;
}

static void release(model_t* m) {
    for (int q = 0; q < m->n_mlp; ++q)
        for (int l = 0; l < m->mlp[q].n_layers; ++l) {
            free(m->mlp[q].w[l]);
            free(m->mlp[q].b[l]);
        }
    free(m->mlp);
}

/* MlpT::forward, inference.cpp:87-101 */
static void mlp_forward(const mlp_t* p, const real* input, real* acts) {
    memcpy(acts, input, sizeof(real) * (size_t)p->sizes[0]);
    for (int l = 0; l < p->n_layers; ++l) {
        const real* x = acts + p->act_offset[l];
        real* y = acts + p->act_offset[l + 1];
        const int in = p->sizes[l], out = p->sizes[l + 1];
        const int last = l == p->n_layers - 1;
        for (int o = 0; o < out; ++o) {
            real z = p->b[l][o];
            const real* row = p->w[l] + (size_t)o * in;
            for (int i = 0; i < in; ++i) z += row[i] * x[i];
            y[o] = last ? z : tanh(z);
        }
    }
}

/* MlpT::backward without weight grads, inference.cpp:107-138 */
static void mlp_backward(const mlp_t* p, const real* dout, const real* acts, real* din,
                         real* scratch /* 2 * max width */) {
    int maxw = 0;
    for (int l = 0; l <= p->n_layers; ++l)
        if (p->sizes[l] > maxw) maxw = p->sizes[l];
    real* cur = scratch;
    real* next = scratch + maxw;
    const int nl = p->n_layers;
    memcpy(cur, dout, sizeof(real) * (size_t)p->sizes[nl]);
    for (int l = nl - 1; l >= 0; --l) {
        const int in = p->sizes[l], out = p->sizes[l + 1];
        const real* y = acts + p->act_offset[l + 1];
        if (l != nl - 1)
            for (int o = 0; o < out; ++o) cur[o] *= ((real)1 - y[o] * y[o]);
        for (int i = 0; i < in; ++i) next[i] = (real)0;
        for (int o = 0; o < out; ++o) {
            const real dz = cur[o];
            const real* row = p->w[l] + (size_t)o * in;
            for (int i = 0; i < in; ++i) next[i] += row[i] * dz;
        }
        real* t = cur;
        cur = next;
        next = t;
    }
    memcpy(din, cur, sizeof(real) * (size_t)p->sizes[0]);
}

static unsigned long long mlp_fwd_flops(const mlp_t* p) {
    unsigned long long f = 0;
    for (int l = 0; l < p->n_layers; ++l)
        f += 2ull * p->sizes[l] * p->sizes[l + 1] + 4ull * p->sizes[l + 1];
    return f;
}

/* switch_value_t / switch_derivative_t, inference.cpp:49-62 (in T). */
static real sw_val(real r, real rc) {
    const real onset = (real)0.9 * rc;
    if (r <= onset) return (real)1;
    if (r >= rc) return (real)0;
    return (real)0.5 * (cos((real)M_PI * (r - onset) / ((real)0.1 * rc)) + (real)1);
}
static real sw_der(real r, real rc) {
    const real onset = (real)0.9 * rc;
    if (r <= onset || r >= rc) return (real)0;
    return (real)(-0.5) * sin((real)M_PI * (r - onset) / ((real)0.1 * rc)) * (real)M_PI /
           ((real)0.1 * rc);
}

/* BasisT::values / derivatives, inference.cpp:162-180 */
static void basis_values(const real* mu, int K, real width, real r, real s, real* out) {
    const real inv = (real)1 / ((real)2 * width * width);
    for (int k = 0; k < K; ++k) {
        const real d = r - mu[k];
        out[k] = exp(-d * d * inv) * s;
    }
}
static void basis_derivs(const real* mu, int K, real width, real r, real s, real ds, real* out) {
    const real inv = (real)1 / ((real)2 * width * width);
    const real inv_w2 = (real)1 / (width * width);
    for (int k = 0; k < K; ++k) {
        const real d = r - mu[k];
        const real g = exp(-d * d * inv);
        out[k] = -d * inv_w2 * g * s + g * ds;
    }
}

/* NnInput::check, inference.cpp:19-32 (+ the type-range check the reference
 * lacks, SURVEY.md §4 "Unchecked types"). */
static int check_input(int n, const int* types, const int* offset, const int* nbr, int n_types) {
    const int ne = offset[n];
    if (offset[0] != 0) {
        ora_set_error("NnInput CSR offsets inconsistent");
        return ORA_INVALID_ARGUMENT;
    }
    for (int e = 0; e < ne; ++e)
        if (nbr[e] < 0 || nbr[e] >= n) {
            ora_set_error("NnInput edge neighbor out of range");
            return ORA_INVALID_ARGUMENT;
        }
    for (int i = 0; i < n; ++i)
        if (types[i] < 0 || types[i] >= n_types) {
            ora_set_error("NnInput atom type out of range");
            return ORA_INVALID_ARGUMENT;
        }
    return ORA_OK;
}

/* evaluate_impl<T>, inference.cpp:183-416 */
int ORA_FN(ora_evaluate)(const int* ilay, const double* dpar, int n, const int* types,
                         const unsigned char* is_ghost, const int* offset, const int* nbr,
                         const double* dr, double coverage, int skip_cov, double* energy_out,
                         double* per_atom, double* forces, double* virial_out,
                         unsigned long long* counters, double* desc_out, double* h_out,
                         double* edge_g_out) {
    model_t m;
    if (unpack(ilay, dpar, &m)) {
        ora_set_error("bad model layout");
        return ORA_INVALID_ARGUMENT;
    }
    int st = check_input(n, types, offset, nbr, m.n_types);
    if (st) {
        release(&m);
        return st;
    }
    const double needed = (1 + m.n_msg) * m.rc_d; /* receptive_radius, model.hpp:51-52 */
    if (!skip_cov && coverage < needed - 1e-12) {
        char msg[256];
        snprintf(msg, sizeof msg,
                 "receptive-field error: model needs %f nm of environment but input covers %f "
                 "nm; widen the halo to L×rc or gather to one rank",
                 needed, coverage);
        ora_set_error(msg);
        release(&m);
        return ORA_RUNTIME_ERROR;
    }
    const int ne = offset[n], K = m.K, H = m.H, nd = m.n_types * K, M = m.n_msg;
    for (int i = 0; i < n; ++i) {
        if (per_atom) per_atom[i] = 0.0;
        forces[3 * i] = forces[3 * i + 1] = forces[3 * i + 2] = 0.0;
    }
    *energy_out = 0.0;
    if (virial_out) *virial_out = 0.0;
    if (n == 0) {
        release(&m);
        return ORA_OK;
    }
    const mlp_t* embed = &m.mlp[0];
    const mlp_t* fit = &m.mlp[1];
    real* mu = (real*)malloc(sizeof(real) * (size_t)K);
    for (int k = 0; k < K; ++k) mu[k] = (real)m.centers_d[k];
    const real width = (real)m.width_d, rcT = (real)m.rc_d;

    /* edge radial quantities, inference.cpp:214-226 */
    real* er = (real*)malloc(sizeof(real) * (size_t)(ne + 1));
    real* es = (real*)malloc(sizeof(real) * (size_t)(ne + 1));
    real* eb = (real*)malloc(sizeof(real) * (size_t)(ne + 1) * K);
    real* eu = (real*)malloc(sizeof(real) * (size_t)(ne + 1) * 3);
    for (int e = 0; e < ne; ++e) {
        const real x = (real)dr[3 * e], y = (real)dr[3 * e + 1], z = (real)dr[3 * e + 2];
        const real r = sqrt(x * x + y * y + z * z);
        if (r <= (real)0) {
            ora_set_error("zero-length edge in NN input");
            free(mu), free(er), free(es), free(eb), free(eu);
            release(&m);
            return ORA_RUNTIME_ERROR;
        }
        er[e] = r;
        eu[3 * e] = x / r;
        eu[3 * e + 1] = y / r;
        eu[3 * e + 2] = z / r;
        es[e] = sw_val(r, rcT);
        basis_values(mu, K, width, r, es[e], eb + (size_t)e * K);
    }
    /* descriptors, inference.cpp:228-238 */
    real* desc = (real*)calloc((size_t)n * nd, sizeof(real));
    for (int i = 0; i < n; ++i)
        for (int e = offset[i]; e < offset[i + 1]; ++e) {
            real* slot = desc + (size_t)i * nd + types[nbr[e]] * K;
            for (int k = 0; k < K; ++k) slot[k] += eb[(size_t)e * K + k];
        }
    if (desc_out)
        for (size_t q = 0; q < (size_t)n * nd; ++q) desc_out[q] = (double)desc[q];

    /* forward, inference.cpp:240-286 */
    real* embed_acts = (real*)malloc(sizeof(real) * (size_t)n * embed->act_size);
    real* h = (real*)calloc((size_t)(M + 1) * n * H, sizeof(real));
    for (int i = 0; i < n; ++i) {
        real* acts = embed_acts + (size_t)i * embed->act_size;
        mlp_forward(embed, desc + (size_t)i * nd, acts);
        memcpy(h + (size_t)i * H, acts + embed->act_offset[embed->n_layers], sizeof(real) * H);
    }
    real** msg_acts = (real**)calloc((size_t)(M + 1), sizeof(real*));
    real** upd_acts = (real**)calloc((size_t)(M + 1), sizeof(real*));
    real* msg_in = (real*)malloc(sizeof(real) * (size_t)(H + K));
    real* upd_in = (real*)malloc(sizeof(real) * (size_t)(2 * H));
    real* msum = (real*)malloc(sizeof(real) * (size_t)n * H);
    for (int l = 0; l < M; ++l) {
        const mlp_t* msg = &m.mlp[2 + 2 * l];
        const mlp_t* upd = &m.mlp[3 + 2 * l];
        msg_acts[l] = (real*)malloc(sizeof(real) * (size_t)(ne + 1) * msg->act_size);
        upd_acts[l] = (real*)malloc(sizeof(real) * (size_t)n * upd->act_size);
        const real* hp = h + (size_t)l * n * H;
        real* hn = h + (size_t)(l + 1) * n * H;
        for (size_t q = 0; q < (size_t)n * H; ++q) msum[q] = (real)0;
        for (int i = 0; i < n; ++i) {
            real* ms = msum + (size_t)i * H;
            for (int e = offset[i]; e < offset[i + 1]; ++e) {
                const int j = nbr[e];
                memcpy(msg_in, hp + (size_t)j * H, sizeof(real) * H);
                memcpy(msg_in + H, eb + (size_t)e * K, sizeof(real) * K);
                real* acts = msg_acts[l] + (size_t)e * msg->act_size;
                mlp_forward(msg, msg_in, acts);
                const real* mo = acts + msg->act_offset[msg->n_layers];
                for (int c = 0; c < H; ++c) ms[c] += es[e] * mo[c];
            }
            memcpy(upd_in, hp + (size_t)i * H, sizeof(real) * H);
            memcpy(upd_in + H, ms, sizeof(real) * H);
            real* ua = upd_acts[l] + (size_t)i * upd->act_size;
            mlp_forward(upd, upd_in, ua);
            const real* u = ua + upd->act_offset[upd->n_layers];
            for (int c = 0; c < H; ++c) hn[(size_t)i * H + c] = hp[(size_t)i * H + c] + u[c];
        }
    }
    if (h_out)
        for (size_t q = 0; q < (size_t)(M + 1) * n * H; ++q) h_out[q] = (double)h[q];

    /* fitting + energy, inference.cpp:288-298 */
    real* fit_acts = (real*)calloc((size_t)n * fit->act_size, sizeof(real));
    double energy = 0.0;
    const real* hM = h + (size_t)M * n * H;
    for (int i = 0; i < n; ++i) {
        if (is_ghost && is_ghost[i]) continue;
        real* acts = fit_acts + (size_t)i * fit->act_size;
        mlp_forward(fit, hM + (size_t)i * H, acts);
        const double ei = (double)acts[fit->act_offset[fit->n_layers]];
        if (per_atom) per_atom[i] = ei;
        energy += ei;
    }
    *energy_out = energy;

    /* backward, inference.cpp:300-370 */
    int maxw = 2 * H + K + nd + 8;
    real* scratch = (real*)malloc(sizeof(real) * (size_t)(2 * maxw));
    real* g = (real*)calloc((size_t)(ne + 1), sizeof(real));
    real* dh = (real*)calloc((size_t)n * H, sizeof(real));
    real* dh_prev = (real*)malloc(sizeof(real) * (size_t)n * H);
    real* dtmp = (real*)malloc(sizeof(real) * (size_t)maxw);
    real* dmo = (real*)malloc(sizeof(real) * (size_t)H);
    real* dbd = (real*)malloc(sizeof(real) * (size_t)K);
    const real one = (real)1;
    for (int i = 0; i < n; ++i) {
        if (is_ghost && is_ghost[i]) continue;
        mlp_backward(fit, &one, fit_acts + (size_t)i * fit->act_size, dtmp, scratch);
        for (int c = 0; c < H; ++c) dh[(size_t)i * H + c] += dtmp[c];
    }
    for (int l = M - 1; l >= 0; --l) {
        const mlp_t* msg = &m.mlp[2 + 2 * l];
        const mlp_t* upd = &m.mlp[3 + 2 * l];
        memcpy(dh_prev, dh, sizeof(real) * (size_t)n * H);
        for (int i = 0; i < n; ++i) {
            mlp_backward(upd, dh + (size_t)i * H, upd_acts[l] + (size_t)i * upd->act_size, dtmp,
                         scratch);
            for (int c = 0; c < H; ++c) dh_prev[(size_t)i * H + c] += dtmp[c];
            real dmsum[256];
            for (int c = 0; c < H; ++c) dmsum[c] = dtmp[H + c];
            for (int e = offset[i]; e < offset[i + 1]; ++e) {
                const int j = nbr[e];
                const real* acts = msg_acts[l] + (size_t)e * msg->act_size;
                const real* mo = acts + msg->act_offset[msg->n_layers];
                const real s = es[e];
                real dsc = (real)0;
                for (int c = 0; c < H; ++c) dsc += dmsum[c] * mo[c];
                g[e] += dsc * sw_der(er[e], rcT);
                for (int c = 0; c < H; ++c) dmo[c] = s * dmsum[c];
                real dmsg_in[512];
                mlp_backward(msg, dmo, acts, dmsg_in, scratch);
                for (int c = 0; c < H; ++c) dh_prev[(size_t)j * H + c] += dmsg_in[c];
                basis_derivs(mu, K, width, er[e], es[e], sw_der(er[e], rcT), dbd);
                real acc = (real)0;
                for (int k = 0; k < K; ++k) acc += dmsg_in[H + k] * dbd[k];
                g[e] += acc;
            }
        }
        real* t = dh;
        dh = dh_prev;
        dh_prev = t;
    }
    for (int i = 0; i < n; ++i) {
        real ddesc[512];
        mlp_backward(embed, dh + (size_t)i * H, embed_acts + (size_t)i * embed->act_size, ddesc,
                     scratch);
        for (int e = offset[i]; e < offset[i + 1]; ++e) {
            const int t = types[nbr[e]];
            basis_derivs(mu, K, width, er[e], es[e], sw_der(er[e], rcT), dbd);
            real acc = (real)0;
            for (int k = 0; k < K; ++k) acc += ddesc[t * K + k] * dbd[k];
            g[e] += acc;
        }
    }
    if (edge_g_out)
        for (int e = 0; e < ne; ++e) edge_g_out[e] = (double)g[e];

    /* force / virial scatter, inference.cpp:372-387 */
    double virial = 0.0;
    for (int i = 0; i < n; ++i)
        for (int e = offset[i]; e < offset[i + 1]; ++e) {
            const int j = nbr[e];
            const real d = g[e];
            if (d == (real)0) continue;
            const real fx = eu[3 * e] * d, fy = eu[3 * e + 1] * d, fz = eu[3 * e + 2] * d;
            forces[3 * j] -= (double)fx;
            forces[3 * j + 1] -= (double)fy;
            forces[3 * j + 2] -= (double)fz;
            forces[3 * i] += (double)fx;
            forces[3 * i + 1] += (double)fy;
            forces[3 * i + 2] += (double)fz;
            virial -= (double)(d * er[e]);
        }
    if (virial_out) *virial_out = virial;

    /* analytic counters, inference.cpp:389-414 */
    if (counters) {
        unsigned long long fl = 0, act = 0;
        int n_owned = 0;
        for (int i = 0; i < n; ++i) n_owned += !(is_ghost && is_ghost[i]);
        fl += (unsigned long long)ne * (20ull + 10ull * K);
        fl += (unsigned long long)n * 3ull * mlp_fwd_flops(embed);
        fl += (unsigned long long)n_owned * 3ull * mlp_fwd_flops(fit);
        for (int l = 0; l < M; ++l) {
            const mlp_t* msg = &m.mlp[2 + 2 * l];
            const mlp_t* upd = &m.mlp[3 + 2 * l];
            fl += (unsigned long long)ne * (3ull * mlp_fwd_flops(msg) + 6ull * H + 3ull * K);
            fl += (unsigned long long)n * (3ull * mlp_fwd_flops(upd) + 2ull * H);
        }
        act += (unsigned long long)n * (nd + embed->act_size + fit->act_size);
        act += (unsigned long long)n * (M + 1) * H;
        for (int l = 0; l < M; ++l) {
            act += (unsigned long long)ne * m.mlp[2 + 2 * l].act_size;
            act += (unsigned long long)n * (m.mlp[3 + 2 * l].act_size + H);
        }
        act += (unsigned long long)ne * (2 + K);
        counters[0] = fl;
        counters[1] = act * sizeof(real);
    }

    for (int l = 0; l < M; ++l) {
        free(msg_acts[l]);
        free(upd_acts[l]);
    }
    free(msg_acts), free(upd_acts), free(msg_in), free(upd_in), free(msum);
    free(fit_acts), free(scratch), free(g), free(dh), free(dh_prev), free(dtmp), free(dmo);
    free(dbd), free(embed_acts), free(h), free(desc), free(mu), free(er), free(es), free(eb);
    free(eu);
    release(&m);
    return ORA_OK;
}

#ifndef ORA_NO_COMMON
/* descriptors(), inference.cpp:430-447 — FP64 with the FP64 switch API. */
int ora_descriptors(const int* ilay, const double* dpar, int n, const int* types,
                    const int* offset, const int* nbr, const double* dr, double* desc) {
    const int K = ilay[2], nd = ilay[1] * K;
    const double rc = dpar[0], width = dpar[1];
    const double* mu = dpar + 2;
    int st = check_input(n, types, offset, nbr, ilay[1]);
    if (st) return st;
    for (size_t q = 0; q < (size_t)n * nd; ++q) desc[q] = 0.0;
    const double inv = 1.0 / (2.0 * width * width);
    for (int i = 0; i < n; ++i)
        for (int e = offset[i]; e < offset[i + 1]; ++e) {
            const double* d = dr + 3 * (size_t)e;
            const double r = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
            const double s = ora_switch_value(r, rc);
            for (int k = 0; k < K; ++k) {
                const double x = r - mu[k];
                desc[(size_t)i * nd + types[nbr[e]] * K + k] += exp(-x * x * inv) * s;
            }
        }
    return ORA_OK;
}
#endif
