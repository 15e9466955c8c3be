/* hmdp_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's DP force-evaluation hot path
 * (/root/reference/proj/src/neighborlist.cpp, src/nn/inference.cpp), used
 * exclusively as the checker in tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg.  The product (libhmdp.so) never links or calls it.
 *
 * Parity of this restatement is pinned against the reference itself, compiled
 * from its own sources into oracle/_ref (see Makefile, tests/test_oracle.py)
 * and against the committed golden vectors in tests/golden/.
 *
 * Model encoding (shared with the product's flat weight layout):
 *   ilay = [family, n_types, K, H, n_msg, n_mlp,
 *           for each mlp: n_layers, sizes[0..n_layers]]
 *   dpar = [rc, width, centers[K],
 *           for each mlp, for each layer l: W_l (out*in, row-major [out][in]), b_l (out)]
 *   mlp order: embedding, fitting, (message_0, update_0), (message_1, update_1), ...
 *   (the same order make_model draws them, proj/src/nn/model.cpp:88-97)
 */
#ifndef HMDP_ORACLE_H
#define HMDP_ORACLE_H
#ifdef __cplusplus
extern "C" {
#endif

#define ORA_OK 0
#define ORA_INVALID_ARGUMENT 1
#define ORA_RUNTIME_ERROR 2

const char* ora_last_error(void);

/* build_input_periodic CSR (inference.cpp:449-487 over neighborlist.cpp:42-113).
 * Returns the number of directed edges (writes at most `cap` of them) or -1. */
int ora_neighbor_csr(int n, const double* xyz, const double* box, double rc, int cap,
                     int* offset, int* nbr, double* dr);

/* O(N^2) minimum-image pair set; same output format; the brute-force oracle
 * of SPEC.md:141,641. */
int ora_neighbor_bruteforce(int n, const double* xyz, const double* box, double rc, int cap,
                            int* offset, int* nbr, double* dr);

/* evaluate_impl<T> (inference.cpp:183-416).  Optional outputs may be NULL:
 * per_atom[n], virial, counters[2] = {flops, activation bytes},
 * desc_out[n*nd], h_out[(n_msg+1)*n*H], edge_g_out[ne]. */
int ora_evaluate_f64(const int* ilay, const double* dpar, int n, const int* types,
                     const unsigned char* is_ghost, const int* offset, const int* nbr,
                     const double* dr, double coverage, int skip_cov, double* energy,
                     double* per_atom, double* forces, double* virial,
                     unsigned long long* counters, double* desc_out, double* h_out,
                     double* edge_g_out);
int ora_evaluate_f32(const int* ilay, const double* dpar, int n, const int* types,
                     const unsigned char* is_ghost, const int* offset, const int* nbr,
                     const double* dr, double coverage, int skip_cov, double* energy,
                     double* per_atom, double* forces, double* virial,
                     unsigned long long* counters, double* desc_out, double* h_out,
                     double* edge_g_out);

/* descriptors() (inference.cpp:430-447), FP64. */
int ora_descriptors(const int* ilay, const double* dpar, int n, const int* types,
                    const int* offset, const int* nbr, const double* dr, double* desc);

double ora_switch_value(double r, double rc);      /* inference.cpp:34-39 */
double ora_switch_derivative(double r, double rc); /* inference.cpp:41-45 */

#ifdef __cplusplus
}
#endif
#endif
