/* hmdp.h — C-ABI of the B200-native deep-potential force evaluation.
 *
 * This is the drop-in boundary for the reference's NN force-provider API
 * (/root/reference/proj/include/halomd/nn/inference.hpp).  Every entry point
 * takes plain pointers and sizes; no C++ or torch types cross it.  Each
 * function names the reference interface it replaces.
 *
 * Units follow the reference (include/halomd/units.hpp:1-5): nm, kJ/mol, ps,
 * amu.  Positions, box, energies, forces and virials are FP64 on the host
 * side, exactly as in NnInput/NnOutput (inference.hpp:18-44).
 *
 * Error model (inference.cpp / model.cpp exceptions mapped to codes):
 *   HMDP_OK                0
 *   HMDP_INVALID_ARGUMENT  1   std::invalid_argument (shapes, model, geometry)
 *   HMDP_RUNTIME_ERROR     2   std::runtime_error (receptive field, zero-length
 *                              edge, non-finite force)
 *   HMDP_CUDA_ERROR        3   device failure
 * The message of the last failure on the calling thread is hmdp_last_error().
 *
 * Threading: a context owns one CUDA stream and its device buffers; it may be
 * used from one thread at a time.  Distinct contexts are independent
 * ("multiple inferences may run concurrently on disjoint inputs").
 */
#ifndef HMDP_H
#define HMDP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HMDP_OK 0
#define HMDP_INVALID_ARGUMENT 1
#define HMDP_RUNTIME_ERROR 2
#define HMDP_CUDA_ERROR 3

/* Precision, include/halomd/forcefield.hpp:10 (enum class Precision {fp32, fp64}).
 * HMDP_FP64 runs the whole network in FP64 (the oracle-of-record mode);
 * HMDP_FP32 runs it in FP32 with FP64 geometry, energy and force accumulation. */
#define HMDP_FP32 0
#define HMDP_FP64 1

typedef struct hmdp_ctx hmdp_ctx;
typedef struct hmdp_md hmdp_md;

/* Thread-local message of the last failed call ("" if none). */
const char* hmdp_last_error(void);

/* ---------------------------------------------------------------------------
 * Model + context.
 * Replaces: halomd::nn::model_from_json (model.cpp:165-197) + NnModel::validate
 * (model.cpp:30-48).  `model_json` is the reference's versioned JSON
 * ({"format":"halomd-model","version":1,...}, model.cpp:147-163).
 * max_atoms sizes the device buffers (grown on demand); max_neighbors is the
 * per-atom edge capacity of the device neighbour list (0 = default 64; grown
 * and retried automatically on overflow outside graph capture).
 * model_json may be NULL (len 0) for a geometry-only context that serves
 * hmdp_build_neighbors; model-dependent calls then fail with
 * HMDP_INVALID_ARGUMENT.
 * ------------------------------------------------------------------------- */
int hmdp_create(const char* model_json, size_t len, int device, int max_atoms,
                int max_neighbors, hmdp_ctx** out);
int hmdp_destroy(hmdp_ctx* ctx);

/* Host-only model check (no device work): model_from_json + validate. */
int hmdp_model_validate(const char* model_json, size_t len);

/* Model facts: family (0 embed_fit, 1 message_passing, 2 se_a, 3 repformer), depth, rc, n_types,
 * hidden, n_basis; receptive radius = depth * rc (model.hpp:51-52). */
int hmdp_model_info(const hmdp_ctx* ctx, int* family, int* depth, double* rc, int* n_types,
                    int* hidden, int* n_basis);

/* ---------------------------------------------------------------------------
 * Single-domain periodic evaluation = build_input_periodic + evaluate.
 * Replaces: halomd::nn::build_input_periodic (inference.cpp:449-487) followed by
 *           halomd::nn::evaluate (inference.cpp:420-424), all atoms owned,
 *           identity global_index, coverage = infinity.
 * xyz[3n], types[n], box[3] (orthorhombic, fully periodic).
 * Outputs: energy (required), per_atom[n] (nullable), forces[3n] (required),
 * virial9[9] (nullable; W_ab = -sum_e g_e dr_a dr_b / r), virial (nullable;
 * the reference's scalar, = trace of virial9 up to rounding).
 * ------------------------------------------------------------------------- */
int hmdp_compute(hmdp_ctx* ctx, int n, const double* xyz, const int* types, const double* box,
                 int precision, double* energy, double* per_atom, double* forces,
                 double* virial9, double* virial);

/* ---------------------------------------------------------------------------
 * Evaluation on an explicit environment (NnInput, inference.hpp:18-38):
 * directed CSR edges (offset[n+1], nbr[offset[n]], dr[3*offset[n]] = r_j - r_i
 * image-corrected), is_ghost[n] (nullable = all owned), coverage_radius and the
 * skip_coverage_check test hook (inference.hpp:31-32).
 * Replaces: halomd::nn::evaluate (inference.cpp:183-416).  Energies for owned
 * atoms only, forces for every input atom (ghost forces returned for routing).
 * Optional stage outputs for per-kernel parity (nullable):
 *   desc[n * n_types * n_basis], h[(depth) * n * hidden] (h^0..h^{depth-1}),
 *   edge_g[offset[n]] (dE/dr per edge).
 * counters (nullable) = {flops, peak_activation_bytes}, the reference's analytic
 * NnCounters (inference.cpp:389-414).
 * ------------------------------------------------------------------------- */
int hmdp_compute_csr(hmdp_ctx* ctx, int n, const int* types, const unsigned char* is_ghost,
                     const int* offset, const int* nbr, const double* dr,
                     double coverage_radius, int skip_coverage_check, int precision,
                     double* energy, double* per_atom, double* forces, double* virial9,
                     double* virial, double* desc, double* h, double* edge_g,
                     uint64_t* counters);

/* ---------------------------------------------------------------------------
 * Device neighbour list exported in the reference's CSR form.
 * Replaces: halomd::nn::build_input_periodic's CSR (inference.cpp:472-485) over
 *           halomd::build_neighbor_list(.., rc, skin=0, full) (neighborlist.cpp:42-113).
 * Pair set and order are bit-exact with the reference (FP64 test, no FMA).
 * Writes up to `cap` edges; returns the edge count via *n_edges (call again
 * with a larger cap when *n_edges > cap).  rc > L/2 -> HMDP_INVALID_ARGUMENT.
 * ------------------------------------------------------------------------- */
int hmdp_build_neighbors(hmdp_ctx* ctx, int n, const double* xyz, const double* box, double rc,
                         int cap, int* offset, int* nbr, double* dr, int* n_edges);

/* descriptors() (inference.cpp:430-447), computed on the device in FP64. */
int hmdp_descriptors(hmdp_ctx* ctx, int n, const int* types, const int* offset, const int* nbr,
                     const double* dr, double* desc);

/* switch_value / switch_derivative (inference.cpp:34-45); host functions. */
double hmdp_switch_value(double r, double rc);
double hmdp_switch_derivative(double r, double rc);

/* Analytic counters for an evaluation of n atoms (n_owned owned) with ne
 * directed edges (inference.cpp:389-414): out[0] flops, out[1] activation
 * bytes for the given precision. */
int hmdp_counters(const hmdp_ctx* ctx, int n, int n_owned, long long ne, int precision,
                  uint64_t* out);

/* ---------------------------------------------------------------------------
 * Device-resident entry point for in-process callers that already hold device
 * buffers (the MD loop, domain decomposition, graph capture).  All pointers are
 * device pointers; `stream` is a cudaStream_t (NULL = the context's stream).
 * Neighbour list is rebuilt on the device from d_xyz (skin 0).  Outputs:
 * d_energy[1], d_forces[3n] (FP64), d_virial9[9] (nullable), d_per_atom[n]
 * (nullable).  Nothing is synchronised; errors are latched in the context's
 * device error word and reported by hmdp_check(ctx).
 * Capturable in a CUDA graph once hmdp_prepare() has sized buffers for n.
 * ------------------------------------------------------------------------- */
int hmdp_prepare(hmdp_ctx* ctx, int n, const double* box, int precision);
int hmdp_compute_device(hmdp_ctx* ctx, int n, const double* d_xyz, const int* d_types,
                        const double* box, int precision, double* d_energy, double* d_forces,
                        double* d_virial9, double* d_per_atom, void* stream);
int hmdp_check(hmdp_ctx* ctx);

/* Number of kernels hmdp_compute_device launches per call for this context's
 * model (for launch accounting in benchmarks). */
int hmdp_kernels_per_eval(const hmdp_ctx* ctx);

/* ---------------------------------------------------------------------------
 * NNPot-style group provider (the paper's Fig. 2 coupling):
 * the DP model runs on the atoms listed in group[n_group] (sorted, duplicate-
 * free indices into the n_total-atom periodic system, e.g. Topology::groups
 * ["protein"]); their NN forces are ADDED into forces_accum[3 n_total] (other
 * atoms untouched), the NN energy is returned.  Classical terms — including
 * every cross-group interaction — stay with the caller.  Positions are gathered
 * on the device; equivalent to hmdp_compute on the extracted group.
 * ------------------------------------------------------------------------- */
int hmdp_compute_group(hmdp_ctx* ctx, int n_total, const double* xyz, const int* types,
                       const int* group, int n_group, const double* box, int precision,
                       double* energy, double* forces_accum, double* virial9, double* virial);

/* ---------------------------------------------------------------------------
 * Device MD loop: velocity Verlet (integrators.cpp:32-47) with the finite-force
 * check (integrators.cpp:12-18) and the NN force provider, all on the device and
 * captured as one CUDA graph per `steps_per_graph` steps.  Every step evaluates
 * the exact rc neighbour list of build_input_periodic (same pairs, order and
 * edge_dr); it is filtered out of Verlet candidate rows within rc + skin that
 * are rebuilt by the cell-list search only after some atom moved more than
 * skin/2 (skin from HMDP_SKIN at hmdp_md_create, default 0.1 nm; 0, or a box
 * where rc + skin exceeds half a length, searches every step).
 * ------------------------------------------------------------------------- */
int hmdp_md_create(hmdp_ctx* ctx, int n, const double* xyz, const double* vel,
                   const double* masses, const int* types, const double* box, double dt_ps,
                   int precision, int steps_per_graph, hmdp_md** out);
int hmdp_md_run(hmdp_md* md, int steps);
/* Asynchronous variant: enqueues the steps on the context's stream and returns;
 * errors are reported by the next hmdp_check / hmdp_md_run / hmdp_md_get. */
int hmdp_md_enqueue(hmdp_md* md, int steps);
/* Copies the current state back; any pointer may be NULL. */
int hmdp_md_get(hmdp_md* md, double* xyz, double* vel, double* forces, double* epot);
/* The loop's Verlet skin (nm, 0 = none) and how many steps rebuilt the candidate
 * rows so far (the first step always does); either pointer may be NULL. */
int hmdp_md_stats(hmdp_md* md, double* skin, long long* rebuilds);
int hmdp_md_destroy(hmdp_md* md);

/* ---------------------------------------------------------------------------
 * Domain decomposition (multi-GPU, per-layer rc halo).  A rank's local system is
 * its n_own owned atoms (local 0..n_own-1) followed by halo ghosts; the CSR
 * carries edges only for owned atoms (their rows of the global periodic list,
 * neighbour indices remapped to local ids; ghost rows empty).  The caller runs
 * the phases in order and exchanges halo rows between them with its transport
 * (NCCL over NVLink in production), through the device buffers returned by
 * hmdp_dd_buffer (rows of n_loc x 32 in the compute precision, forces n_loc x 3
 * FP64):
 *   phase 0 embed                      -> P rows of owned atoms (buffer 0)
 *   [P rows of ghosts <- their owners]  phase 1 (layer 0) pushes them
 *   phase 2 layer l forward            -> P rows (l < depth-2) / top backward
 *   [exchange P, phase 1 (layer l+1)]
 *   phase 3 layer l ghost sums         -> buffer 2 rows of ghosts
 *   [owners add the ghosts' sums of their atoms into buffer 1 (zeroed first)]
 *   phase 4 layer l backward (l = depth-3 .. 0), then phase 3 / exchange again
 *   phase 5 embedding backward         (reads buffer 1)
 *   phase 6 forces                     -> buffer 3 rows; ghosts' rows go to owners
 * hmdp_dd_result: this rank's partial energy (owned atoms) and virial.
 * Replaces: the SPEC's halo_inference with rc-deep halos
 * exchanged per message layer instead of one L*rc-deep halo.
 * ------------------------------------------------------------------------- */
int hmdp_dd_setup(hmdp_ctx* ctx, int n_loc, int n_own, const int* offset, const int* nbr,
                  const double* dr, const int* types, int precision);
int hmdp_dd_phase(hmdp_ctx* ctx, int phase, int layer);
int hmdp_dd_buffer(hmdp_ctx* ctx, int kind, void** dptr);
int hmdp_dd_result(hmdp_ctx* ctx, double* energy, double* virial9, double* virial);

/* ---------------------------------------------------------------------------
 * Device-resident domain decomposition on the global index space (hmdp_gdd.cu).
 * Every rank holds all n positions (replicated; all ranks integrate all atoms
 * with the same all-reduced forces) and runs the network for the atoms its region
 * of the dims[0] x dims[1] x dims[2] rank grid owns; plans are built on the device
 * each step (no host work, fixed sizes: the whole step is capturable in a CUDA
 * graph together with the caller's collectives).  The caller binds device buffers
 * (kind 0 positions [n][3] f64, 1 P rows [n][32] T, 2 halo sums [n][32] T,
 * 3 forces [n][3] f64, 4 out[16] f64 = (E, W, W9), 5 velocities, 6 masses) and
 * runs, on the context's stream, with a SUM all-reduce of the named buffer at "|":
 *   10 ; 0 ; for l < depth-1: |1| 1(l) 2(l) ;
 *   for l = depth-2 .. 0: 3(l) |2| then 4(l-1) or 5 ; 6 |3| |4| ; 7(dt)
 * (phase 8(dt) = the initial opening kick + drift).  Same results as the
 * single-domain evaluation up to the summation order of halo partials.
 * Replaces: the SPEC's halo_inference, per-layer rc halo.
 * ------------------------------------------------------------------------- */
int hmdp_gdd_setup(hmdp_ctx* ctx, int n, const int* types, const double* box, const int* dims,
                   int rank, int precision);
int hmdp_gdd_bind(hmdp_ctx* ctx, int kind, void* dptr);
int hmdp_gdd_phase(hmdp_ctx* ctx, int phase, int layer, double dt);
int hmdp_gdd_counts(hmdp_ctx* ctx, int* counts3); /* owned, halo, searched (syncs) */
/* Kernels enqueued by hmdp_gdd_phase on this context so far (launch accounting). */
int hmdp_gdd_launches(const hmdp_ctx* ctx, long long* launches);

/* ---------------------------------------------------------------------------
 * 5th-generation tensor cores (hmdp_tc.cu): a chain of up to 3 dense layers
 * y = act(x W^T + b) (the reference's MlpT::forward, inference.cpp:87-101) on
 * tcgen05.mma kind::tf32 with the 3xTF32 hi/lo split and FP32 accumulation in
 * TMEM.  Host arrays: x [rows][sizes[0]], weights = W_1 [sizes[1]][sizes[0]], W_2
 * [sizes[2]][sizes[1]], ... concatenated, biases likewise, act[l] 0 linear / 1 tanh;
 * y [rows][sizes[n_layers]].  K % 8 == 0, K <= 64, N in {32, 64}.
 * hmdp_peak_tcgen05_tf32: measured raw kind::tf32 MMA throughput (TFLOP/s);
 * 3xTF32 delivers a third of it.
 * ------------------------------------------------------------------------- */
int hmdp_tc_mlp(int device, int rows, const float* x, int n_layers, const int* sizes,
                const float* weights, const float* biases, const int* act, float* y);
int hmdp_peak_tcgen05_tf32(int device, int ms, double* tflops);

/* ---------------------------------------------------------------------------
 * Halo-exchange mode of the device DD (the multi-GPU engine; SPEC.md:474-524
 * message kinds ghost_positions / ghost_forces, per-layer rc halo).
 * Nothing is replicated: each rank integrates only the atoms its region owns, and
 * every step moves exactly the halo with point-to-point rounds to every peer:
 *   POS (x, v of owned atoms within rc of the peer's region; migration included),
 *   P^l per message layer (P rows of owned atoms near the peer),
 *   SUMS^l per layer (dE/dh partial sums at halo atoms -> their owners),
 *   FORCES (partial forces at halo atoms -> their owners), OUT ((E, W, W9) partials,
 *   summed in rank order on every rank).
 * Each round packs one fixed-capacity packet per peer on the device (capacity
 * planned once from the initial geometry, x1.5 + 64 rows headroom; overflow latches
 * an error), so a whole MD step -- collectives included -- is one CUDA graph.
 * The network runs in its pull form (senders -- owned and halo rows -- pull the
 * owned receivers' adjoint rows; the SUMS round carries the halo senders' sums);
 * the environment variable HMDP_DD_PULL=0 selects the push form.  Same results up
 * to the summation order of the partial sums.
 * Transports: NCCL (grouped ncclSend/ncclRecv on the context's stream; libnccl is
 * loaded at run time), an in-process hub (simulated ranks = contexts on one GPU,
 * one host thread each), or a caller callback (e.g. gloo in tests).
 *   hmdp_gdd_set_mode(ctx, 1) after hmdp_gdd_setup, bind buffers 0 (positions),
 *   3 (forces), 4 (out[16]) and, for MD, 5 (velocities) and 6 (masses), load the
 *   positions, then hmdp_gdd_plan (capacity; syncs) and hmdp_gdd_step per step.
 * ------------------------------------------------------------------------- */
typedef struct hmdp_gdd_hub hmdp_gdd_hub;
/* Caller transport: move, for every peer q != rank, the first `bytes` of
 * send + q*stride (device) to peer q's recv + rank*stride (device); return 0 on
 * success.  Called with the context's stream synchronized. */
typedef int (*hmdp_gdd_exchange_fn)(void* user, int round, const void* send, void* recv,
                                    size_t stride, size_t bytes);
/* Gather-to-root mode (2; the paper's NNPot strategy, reference SPEC.md:505,
 * nn_inference_decomposed(strategy = gather_to_root)): the same POS round (migration),
 * then GATHER (every rank's owned positions -> rank 0), one single-domain evaluation
 * of the whole system on rank 0, SCATTER (each owner's forces, in the order it sent
 * its atoms) and OUT; owners integrate their atoms.  Same buffers, plan and step
 * calls as halo mode; the comparison path for the halo-exchange engine. */
int hmdp_gdd_set_mode(hmdp_ctx* ctx, int mode); /* 0 all-reduce, 1 halo, 2 gather-to-root */
/* NCCL transport: 128-byte ncclUniqueId (generated on rank 0 by hmdp_nccl_unique_id
 * and broadcast by the caller), world size and this rank (= DD rank). */
int hmdp_nccl_unique_id(void* id128);
int hmdp_gdd_attach_nccl(hmdp_ctx* ctx, const void* id128, int world, int rank);
int hmdp_gdd_hub_create(int world, hmdp_gdd_hub** out);
int hmdp_gdd_hub_destroy(hmdp_gdd_hub* hub);
int hmdp_gdd_attach_hub(hmdp_ctx* ctx, hmdp_gdd_hub* hub);
int hmdp_gdd_attach_callback(hmdp_ctx* ctx, hmdp_gdd_exchange_fn fn, void* user);
/* Packet capacity from the loaded positions; marks every atom current (syncs). */
int hmdp_gdd_plan(hmdp_ctx* ctx);
/* One step on the context's stream: kind 0 evaluation (E, F, W into the bound
 * buffers), 1 MD step (evaluation + closing kick + next opening kick + drift of
 * the owned atoms), 2 the initial opening kick + drift only.  Capturable with the
 * NCCL transport. */
int hmdp_gdd_step(hmdp_ctx* ctx, int kind, double dt);
/* Halo statistics of the last step (syncs): out[0] packet rows capacity C,
 * out[1] rounds per step, out[2] useful halo bytes sent by this rank per step
 * (rows x row bytes over every round), out[3] bytes actually transferred per step
 * (fixed-capacity packets), out[4] peers. */
int hmdp_gdd_halo_stats(hmdp_ctx* ctx, long long* out5);
/* Roles of the last step (syncs): out[n] = 1 owned here, 2 halo, 0 neither; the
 * forces of the owned rows are this rank's share of the global result. */
int hmdp_gdd_roles(hmdp_ctx* ctx, unsigned char* out);

/* ---------------------------------------------------------------------------
 * Classical force field on the device: the reference's
 * compute_classical (forcefield.cpp:265-279) — harmonic bonds, angles, periodic
 * dihedrals, potential-shifted LJ (Lorentz-Berthelot), Coulomb cutoff_shifted (0)
 * or reaction_field (1) — over the device cell-list pairs within max(rc_lj,
 * rc_coulomb) minus the exclusions (excl_offset[n+1] / excl: each atom's sorted
 * list).  bonds[2 nb] + bond_params[2 nb] = (k_b, r0); angles[3 na] (j = vertex) +
 * angle_params[2 na] = (k_a, theta0); dihedrals[4 nd] + dihedral_params[3 nd] =
 * (k_d, phase, multiplicity).  energies[3] = (bonded, lj, coulomb); forces[3n]
 * are SET (as compute_classical zeroes first); virial = sum r.F over all terms;
 * collinear = angles evaluated with the clamped derivative.
 * precision: HMDP_FP32 / HMDP_FP64 arithmetic as the reference's Precision.
 * ------------------------------------------------------------------------- */
typedef struct hmdp_ff hmdp_ff;
int hmdp_ff_create(int device, int n, const int* types, const double* charges, int n_types,
                   const double* sigma, const double* epsilon, int coulomb_scheme,
                   double rc_coulomb, double eps_rf, double rc_lj, const int* excl_offset,
                   const int* excl, int n_bonds, const int* bonds, const double* bond_params,
                   int n_angles, const int* angles, const double* angle_params, int n_dihedrals,
                   const int* dihedrals, const double* dihedral_params, hmdp_ff** out);
int hmdp_ff_compute(hmdp_ff* ff, const double* xyz, const double* box, int precision,
                    double* energies, double* forces, double* virial, int* collinear);
int hmdp_ff_destroy(hmdp_ff* ff);

/* Hybrid device MD (the paper's NNPot coupling): every step the
 * classical force field (ff) on all n atoms + the DP model (ctx) on the sorted
 * group[n_group], forces summed, velocity Verlet on all atoms — captured as one CUDA
 * graph per steps_per_graph steps.  energies[4] = (bonded, lj, coulomb, nn) of the
 * last evaluated configuration. */
typedef struct hmdp_hmd hmdp_hmd;
int hmdp_hybrid_create(hmdp_ctx* ctx, hmdp_ff* ff, int n, const int* group, int n_group,
                       const double* xyz, const double* vel, const double* masses, const int* types,
                       const double* box, double dt_ps, int precision, int steps_per_graph,
                       hmdp_hmd** out);
int hmdp_hybrid_run(hmdp_hmd* h, int steps);
int hmdp_hybrid_get(hmdp_hmd* h, double* xyz, double* vel, double* forces, double* energies);
int hmdp_hybrid_destroy(hmdp_hmd* h);

/* ---------------------------------------------------------------------------
 * Measurement hooks.
 * hmdp_set_stream: run the context's work on an external cudaStream_t (e.g. the
 *   caller's current stream) instead of its own (NULL restores it).
 * hmdp_profile: when enabled, a CUDA event is recorded after every kernel of an
 *   evaluation / MD step (also inside captured graphs); hmdp_profile_read returns
 *   the per-kernel durations (ms) of the most recent execution and
 *   hmdp_profile_name(i) the i-th kernel's name.
 * hmdp_peak_fp32: measured FP32 FFMA throughput of the device (TFLOP/s), the
 *   roofline denominator for the SIMT kernels.
 * hmdp_peak_tf32x3: measured FP32-accurate 3xTF32 mma.sync throughput (TFLOP/s,
 *   each hi/lo triple of m16n8k8 MMAs counted as one product), the denominator for
 *   the tensor-core projections of the DeePMD-style families.
 * ------------------------------------------------------------------------- */
int hmdp_set_stream(hmdp_ctx* ctx, void* stream);
int hmdp_profile(hmdp_ctx* ctx, int enable);
int hmdp_profile_read(hmdp_ctx* ctx, float* ms, int cap, int* count);
const char* hmdp_profile_name(const hmdp_ctx* ctx, int i);
int hmdp_peak_fp32(int device, int ms, double* tflops);
int hmdp_peak_tf32x3(int device, int ms, double* tflops);

/* ---------------------------------------------------------------------------
 * Host fixtures (no device work).
 * hmdp_make_model_json: make_model (model.cpp:70-100) + model_to_json
 *   (model.cpp:147-163); deterministic mt19937_64 draw order; returns the JSON
 *   length (excluding NUL) and writes it if buf/cap allow, or -code on error.
 * hmdp_synthetic_system: generate_synthetic_system (synthetic.cpp:36-130):
 *   positions, types, masses, velocities (300 K draw) and box.
 * ------------------------------------------------------------------------- */
long hmdp_make_model_json(int family, int depth, double rc, int n_types, int n_basis,
                          int hidden, uint64_t seed, char* buf, long cap);
/* DeePMD-style families (no reference function; SURVEY.md §8(a')):
 * family 2 = se_a (smooth env matrix, per-neighbour-type embedding, G^T R R^T G,
 * fitting; depth 1), family 3 = repformer (se_a descriptor + depth-1 repformer
 * layers with gated neighbour self-attention).  Same Rng / MLP init as
 * hmdp_make_model_json; the JSON carries "family":"se_a"|"repformer".
 * Every compute entry point accepts these models except hmdp_descriptors, the
 * domain-decomposition phases, the per-stage outputs of hmdp_compute_csr, and
 * (repformer) hmdp_compute_csr itself. */
long hmdp_make_dp_model_json(int family, int depth, double rc, double rc_smooth, int n_types,
                             int axis, uint64_t seed, char* buf, long cap);
int hmdp_synthetic_system(int n, double density, double fraction_grouped, uint64_t seed,
                          double temperature, double* xyz, int* types, double* masses,
                          double* vel, double* box);

#ifdef __cplusplus
}
#endif
#endif /* HMDP_H */
