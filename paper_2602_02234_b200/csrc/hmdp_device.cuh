// hmdp_device.cuh — device-side data structures shared by the kernels and the
// host orchestration (hmdp_api.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "hmdp_model.h"

namespace hmdp {

// Device error word bits (latched with atomicOr, read back after each call).
enum : unsigned {
    kErrNbrOverflow = 1u << 0,   // an atom has more neighbours than the ELL capacity
    kErrCellOverflow = 1u << 1,  // a cell has more members than the cell capacity
    kErrZeroEdge = 1u << 2,      // zero-length edge (inference.cpp:221)
    kErrAsymmetric = 1u << 3,    // reverse edge missing in a "symmetric" list
    kErrNonFinite = 1u << 4,     // non-finite force (integrators.cpp:12-18)
    kErrHaloOverflow = 1u << 5,  // a halo-exchange packet exceeded its row capacity
};

// One two-layer MLP [in, 32, out] on the device, stored both row-major (as in
// the model file, [out][in]) and transposed ([in][out]) so that the warp
// kernels always read contiguous rows.
template <typename T>
struct DevMlp {
    const T* W1;   // [32][in]
    const T* W1T;  // [in][32]
    const T* b1;   // [32]
    const T* W2;   // [out][32]
    const T* W2T;  // [32][out]
    const T* b2;   // [out]
};

template <typename T>
struct DevModel {
    DevMlp<T> embed, fit;
    DevMlp<T> msg[kMaxMsg], upd[kMaxMsg];
    T mu[kK];
    T rc;       // T(model.rc_model)
    T width;    // T(basis.width)
    T inv2w2;   // T(1)/(T(2)*width*width)  (inference.cpp:164)
    T invw2;    // T(1)/(width*width)        (inference.cpp:174)
    int n_types;
    int n_msg;
    // Shared-memory images of the matrices each network kernel stages, laid out
    // exactly as in shared memory (rows padded by 16 bytes), one bulk copy each
    // (hmdp_net.cu, Smem::load): embedding (or embed_fit when n_msg == 0), message
    // layer forward (the fused last-layer layout at n_msg - 1), message layer
    // backward (l < n_msg - 1), embedding backward.  Forward: [U1h | U1m W2] (the
    // message output layer folded into the update MLP), backward [U1h^T ; (U1m W2)^T].
    const T* img_embed;
    // U1m b2 per message layer (the message MLP's output bias through the update
    // MLP's msum half; W2 itself is folded into the update matrices of the images)
    const T* uc1[kMaxMsg];
    // the embedding output layer folded into its consumer: eqb = W1h^0 eb2 (P^0 bias) or
    // fW1 eb2 + fb1 (the fitting pre-activation, depth 1); fcl = fW1 b2u + fb1 (the
    // fitting through the top update's output layer)
    const T* eqb;
    const T* fcl;
    const T* img_fwd[kMaxMsg];
    const T* img_bwd[kMaxMsg];
    const T* img_embed_bwd;
};

// Directed edge graph of one evaluation.  Out-edges of atom i occupy slots
// [row_start[i], row_start[i] + nnei[i]) sorted by neighbour index; in-edges
// (edges e = (k -> i)) are listed in in_edge[in_start[i] .. + in_cnt[i]).
// For the symmetric periodic list in_start/in_cnt alias row_start/nnei and
// in_edge[e] = rev(e), the slot of the mirrored edge.
//
// "Mirror" slots: the in-edge array position of edge e (e's slot in the list of
// its target j) is inv_pos[e].  Producers push per-neighbour data there (P_j for
// message layers, the h_j adjoint dz_e, and g_e for the force), so consumers
// read their own contiguous range [in_start[i], in_start[i] + in_cnt[i]) without
// an index indirection.  For the symmetric periodic list the in-edge array IS
// the out-slot array: in_edge = inv_pos = rev and in_start/in_cnt alias
// row_start/nnei (sym = 1).
struct DevGraph {
    int n;
    int n_active;  // atoms [0, n_active) run the network; the rest are halo ghosts
    int sym;       // 1: in-edge array aliases the out-slots (rev), see above
    int ell;       // > 0: ELL rows, row_start[i] = i * ell (periodic path); 0: general CSR
    const int* row_start;
    const int* nnei;
    const int* nbr;
    const int* ety;    // [slot] type of the neighbour (written by the search)
    const double* dr;  // [slot][3], r_j - r_i image-corrected (FP64)
    const int* in_start;
    const int* in_cnt;
    const int* in_edge;  // [in-position] -> edge slot
    const int* inv_pos;  // [edge slot] -> in-position (mirror slot)
    const int* types;
    const unsigned char* is_ghost;  // nullable
    // nullable: run the network only for the atoms alist[0 .. *alist_n) (global-index
    // domain decomposition, hmdp_gdd_*: this rank's owned atoms); else [0, n_active)
    const int* alist;
    const int* alist_n;
};

// Per-evaluation device workspace (element type T for the network tensors).
template <typename T>
struct DevWork {
    // per edge slot
    T* es;    // s(r)
    T* eds;   // s'(r)
    T* eb;    // [slot][8] b_k
    T* edb;   // [slot][8] b_k'
    T* g;     // dE/dr
    T* grev;  // [in-position] g of the edge mirrored there (pushed by its source)
    T* z;     // [M][slot][32] message hidden (tanh) activations z_e (push form: at the
              // receiver's slot; pull-store form: at the sender's mirror slot)
    T* d;     // [2][in-position][32] pushed adjoints dz_e (push form only)
    T* pa;    // [M][n][32] per-atom neighbour projections P^l_i = W1h^l h^l_i, gathered
              // by the edges' sources (nbr index); L2-resident at every paper size
    // pull-form backward (symmetric graph, every atom runs the network): per-atom
    // v^l_i = W2^T dmsum^l_i rows and c0^l_i = dmsum^l_i . b2, double-buffered by layer;
    // the SENDER of each message gathers its receiver's row (hmdp_net.cu, k_msg_bwd_pull)
    T* vrow;  // [2][n][32]
    T* vc0;   // [2][n]
    // domain decomposition (nullable otherwise)
    T* p_atom;    // [n][32] per-atom P of the layer just produced (sent to ghost copies)
    T* s_remote;  // [n][32] adjoint partial sums received from ghost copies elsewhere
    // halo-exchange DD, pull form (nullable otherwise): roles of the global-index rows
    // (1 = owned) and the per-row dE/dh partial sums of the sender-side backward
    const unsigned char* dd_role;
    const unsigned char* dd_bnd;  // 1: owned row in some peer's halo (receives s_remote)
    T* dd_sum;  // [n][32]
    // per atom
    T* desc;   // [n][32] descriptor (n_types*8 used)
    T* ez1;    // [n][32] embedding hidden activations
    T* h;      // [M+1][n][32]
    T* uz1;    // [M][n][32] update hidden activations
    T* dhown;  // [n][32] atom-local part of dE/dh
    double* e_atom;   // [n]
    double* forces;   // [n][3]
    double* partial;  // [blocks][16] per-block E, W, W9
    unsigned* ticket;
    double* out;  // [16]: E, W, W9[9]
    long long slots;  // edge-slot capacity of the per-edge arrays
    unsigned* err;
    // DeePMD-style families: dE/d(edge_dr) as a vector per edge slot ([slot][4],
    // xyz + pad) and its mirror copy pushed by the edge's source (gv of rev(e) at
    // slot e); the force kernel gathers both when gv != nullptr.
    T* gv;
    T* gvrev;
    // 1: the force kernel gathers the mirror g of each slot as g[inv_pos[q]] instead of
    // reading the pushed grev[q] (the fused depth-1 network on the periodic path)
    int gather_mirror_g;
    // 1: the force kernel's last CTA also exports the device error word into out[12]
    // and clears it (hmdp_compute's graph path, outputs in host-mapped memory)
    int export_err;
    // 1: forces / per-atom energies go to host-mapped memory (hmdp_compute's graph
    // path): the force kernel writes each warp's atoms as one contiguous store
    int wide_out;
};

// ---------------------------------------------------------------------------
// DeePMD-style families (se_a, repformer, hmdp_dp.cu).
// Linear layer y = W x + b with W row-major [out][in] and its transpose.
template <typename T>
struct DevLin {
    const T* W;   // [out][in]
    const T* WT;  // [in][out]
    const T* b;   // [out]
};

template <typename T>
struct DevDpLayer {
    DevLin<T> q, k, v, o, c;   // [32][32] each (repflow: no q, k)
    const T* aw;               // repflow angle embedding z = tanh(aw c + ab), [32] each
    const T* ab;
    DevLin<T> u1, u2;          // update MLP [32 + 4*32 -> 32 -> 32]
};

template <typename T>
struct DevDp {
    T rc, rcs, inv_nnorm;
    T rca, rcas, inv_anorm;         // repflow angle neighbours
    int n_types, n_layers, family;  // family: kSeA / kRepformer / kRepflow
    T ebias[kMaxTypes];
    // per neighbour type embedding [1 -> 32 -> 32]: w1/b1 [32], layer 2 as DevLin
    const T* emb_w1[kMaxTypes];
    const T* emb_b1[kMaxTypes];
    DevLin<T> emb2[kMaxTypes];
    DevLin<T> fit1, fit2;  // fitting [in -> 32 -> 1]
    DevLin<T> map1, map2;  // repformer g1 map [128 -> 32 -> 32]
    DevDpLayer<T> L[kMaxMsg];
};

// Per-evaluation workspace of the repformer kernels (per edge slot / per atom).
template <typename T>
struct DevDpWork {
    T* env;    // [slot][8]: s, w, h0, h1, h2, dsw, r, type (as T)
    T* g2;     // [L+1][slot][32] edge channel g2 per layer (g2^{l+1} = after attention l)
    T* qkv;    // [slot][96] q, k, v of the current layer
    T* dg2;    // [slot][32] adjoint of g2 (in place, layer by layer)
    T* dwh;    // [slot][4]  accumulated dE/dw, dE/dh (from every layer)
    T* g1;     // [L+1][n][32]
    T* P;      // [L][n][32] neighbour projections P^l = Wc g1^l + bc
    T* uz;     // [L][n][32] update MLP hidden activations
    T* mz;     // [n][32] g1 map hidden activations
    T* D;      // [n][128] descriptor
    T* A;      // [n][128] R^T G / nnorm (4 x 32)
    T* Ts;     // [L][n][96] h^T g2 / nnorm per layer (3 x 32)
    T* stat;   // [L][slot][2] softmax row max and normaliser per layer
    T* dob;    // [slot][32] attention output adjoint do_e = Wo^T dg2hat_e
    T* aux;    // [slot][2] row sums S_e = sum_f a_ef da_ef
    T* tmp;    // [slot][96] attention output o_e (forward); dq, dk, dv (backward)
    T* dconv;  // [2][n][32] adjoint of conv_i / nnorm (double-buffered by layer)
    T* dg1;    // [n][32] adjoint of g1 (residual part) of the current layer
    int smem_rows;  // 1: per-atom q/k/v and do rows live in shared memory (ELL cap <= 64)
    T* envA;   // repflow [slot][8]: omega, omega', u_x, u_y, u_z
    T* dua;    // repflow [slot][4]: dE/domega, dE/du (accumulated over layers)
};

// Optional per-kernel timing hook: called after every kernel launch with the
// kernel's name (records a CUDA event when profiling is enabled; capturable).
struct Marker {
    void (*fn)(void*, const char*, cudaStream_t) = nullptr;
    void* user = nullptr;
    void operator()(const char* name, cudaStream_t st) const {
        if (fn) fn(user, name, st);
    }
};

constexpr int kCandMax = 512;  // neighbour candidates kept per atom (search warp list)

struct CellGrid {
    int nc[3];
    double L[3];
    int ccap;
};

// Velocity-Verlet work fused into the force kernel (device MD loop):
//   mode 0: none
//   mode 1: second half kick            v += F * (dt/2)/m
//   mode 2: second half kick, then the next step's first half kick, drift and
//           cell binning:  v += F*(dt/2)/m; v += F*(dt/2)/m; x += v*dt; bin(x)
// The device MD loop runs every step in mode 2 (the opening kick of the next
// step is fused into this one) and writes the completed step to (xs, vs).
// (integrators.cpp:32-47, with the finite-force check of :12-18 on F).
// zero_cells (embed kernel): cell counts to clear once the search consumed them.
struct MdFuse {
    int mode = 0;
    double* x = nullptr;
    double* v = nullptr;
    const double* m = nullptr;
    double half = 0.0, dt = 0.0;
    CellGrid cg{};
    int* cell_count = nullptr;
    int* members = nullptr;
    int* cell_of = nullptr;
    int n_cells_zero = 0;  // > 0: embed kernel zeroes cell_count[0..n)
    double* xs = nullptr;  // nullable: completed-step snapshot (x, v after the
    double* vs = nullptr;  // closing kick), what hmdp_md_get returns
    // Verlet candidate list (device MD loop with a skin, VList): after the drift,
    // any atom farther than skin/2 from its position at the last candidate build
    // (xref, minimum image) sets *vflag, and the next search rebuilds.
    const double* xref = nullptr;
    int* vflag = nullptr;
    double vhalf2 = 0.0;  // (skin/2)^2, slightly shrunk
};

// Verlet candidate list of the device MD loop (k_nbr_search_v): every step the
// exact rc list is filtered out of the rows of candidates within rc + skin,
// which are rebuilt by the cell-list scan only when *flag is set.
struct VList {
    int* list = nullptr;   // [n][cap] candidates, ascending j
    int* cnt = nullptr;    // [n]
    double* xref = nullptr;  // [n][3] positions at the last build
    int* flag = nullptr;   // [0] rebuild flag, [1] CTA-done counter, [2] rebuilds so far
    int cap = 0;
    double range2 = 0.0;   // (rc + skin)^2
};

}  // namespace hmdp
