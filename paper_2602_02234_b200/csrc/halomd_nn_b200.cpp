// halomd_nn_b200.cpp — exact-signature C++ drop-in for the reference's NN
// force-provider API, over the C-ABI in include/hmdp.h.
//
// This translation unit DEFINES the functions the reference DECLARES in
// /root/reference/proj/include/halomd/nn/inference.hpp:
//
//   NnInput::n_owned, NnInput::check            inference.hpp:35-36   (inference.cpp:12-32)
//   build_input_periodic(positions, types,       inference.hpp:63-65   (inference.cpp:449-487)
//                        global_index, box, rc)
//   evaluate(model, input, prec, counters)       inference.hpp:69-70   (inference.cpp:420-424)
//   descriptors(model, input)                    inference.hpp:73      (inference.cpp:430-447)
//   switch_value / switch_derivative             inference.hpp:76-77   (inference.cpp:34-45)
//
// with exactly the declared signatures, so libhalomd_nn_b200.so links in place of
// the reference's inference.o and reference call sites compile and run unchanged
// (plain `nn::evaluate(model, in, prec, &c)`).  It is compiled against the
// reference's own headers (-I<reference>/proj/include; nothing is copied), which is
// why it is built only where the reference tree exists (build.py) and travels to
// the GPU box as a built artefact, like oracle/_ref.
//
// Semantics kept: value semantics, std::invalid_argument / std::runtime_error with
// the reference's messages, energies for owned atoms only, forces for every input
// atom, the scalar virial, the reference's analytic NnCounters.  One device context
// per (model JSON, device), each behind its own mutex, so concurrent calls on
// disjoint inputs are allowed.  Device: HMDP_DEVICE (default 0).
// Documented divergence: the device neighbour search is fully periodic, so a box
// with a non-periodic axis is rejected with std::invalid_argument.
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "halomd/nn/inference.hpp"
#include "hmdp.h"

namespace {

void check_code(int code) {
    if (code == HMDP_OK) return;
    const std::string msg = hmdp_last_error();
    if (code == HMDP_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

int device_ordinal() {
    static const int dev = [] {
        const char* e = std::getenv("HMDP_DEVICE");
        return e ? std::atoi(e) : 0;
    }();
    return dev;
}

struct Slot {
    hmdp_ctx* ctx = nullptr;
    std::mutex mu;  // a context is not shared across threads without a lock (hmdp.h)
    ~Slot() {
        if (ctx) hmdp_destroy(ctx);
    }
};

// One context per model JSON ("" = geometry-only context for build_input_periodic).
class Contexts {
   public:
    static Contexts& get() {
        static Contexts c;
        return c;
    }
    Slot& slot(const std::string& json) {
        std::lock_guard<std::mutex> lk(mu_);
        auto& s = map_[json];
        if (!s) {
            auto fresh = std::make_unique<Slot>();
            check_code(hmdp_create(json.empty() ? nullptr : json.data(), json.size(),
                                   device_ordinal(), 1024, 0, &fresh->ctx));
            s = std::move(fresh);
        }
        return *s;
    }

   private:
    std::mutex mu_;
    std::map<std::string, std::unique_ptr<Slot>> map_;
};

void require_periodic(const halomd::SimBox& box) {
    for (int a = 0; a < 3; ++a)
        if (!box.periodic[a])
            throw std::invalid_argument(
                "B200 neighbour search supports fully periodic boxes only (axis " +
                std::to_string(a) + " is not periodic)");
}

std::vector<double> flat3(const std::vector<halomd::Vec3>& v) {
    std::vector<double> out(3 * v.size());
    for (std::size_t i = 0; i < v.size(); ++i) {
        out[3 * i] = v[i].x;
        out[3 * i + 1] = v[i].y;
        out[3 * i + 2] = v[i].z;
    }
    return out;
}

}  // namespace

namespace halomd::nn {

int NnInput::n_owned() const {
    int n = 0;
    for (char g : is_ghost)
        if (!g) ++n;
    return n;
}

// Same checks and messages as inference.cpp:19-32.
void NnInput::check() const {
    const std::size_t n = types.size();
    if (positions.size() != n || global_index.size() != n || is_ghost.size() != n)
        throw std::invalid_argument("NnInput arrays disagree on atom count");
    if (edge_offset.size() != n + 1) throw std::invalid_argument("NnInput edge_offset has wrong size");
    if (edge_neighbor.size() != edge_dr.size())
        throw std::invalid_argument("NnInput edge arrays disagree");
    if (!edge_offset.empty() && edge_offset.back() != static_cast<int>(edge_neighbor.size()))
        throw std::invalid_argument("NnInput CSR offsets inconsistent");
    for (int j : edge_neighbor)
        if (j < 0 || j >= static_cast<int>(n))
            throw std::invalid_argument("NnInput edge neighbor out of range");
}

double switch_value(double r, double rc) { return hmdp_switch_value(r, rc); }
double switch_derivative(double r, double rc) { return hmdp_switch_derivative(r, rc); }

// Device cell-list search (hmdp_build_neighbors): the reference's pair set, order
// and FP64 edge_dr bit for bit.
NnInput build_input_periodic(const std::vector<Vec3>& positions, const std::vector<int>& types,
                             const std::vector<int>& global_index, const SimBox& box,
                             double rc_model) {
    if (positions.size() != types.size() || positions.size() != global_index.size())
        throw std::invalid_argument("positions/types/global_index size mismatch");
    require_periodic(box);
    const int n = static_cast<int>(positions.size());
    NnInput in;
    in.positions = positions;
    in.types = types;
    in.global_index = global_index;
    in.is_ghost.assign(positions.size(), 0);
    const std::vector<double> x = flat3(positions);
    const double b[3] = {box.lengths.x, box.lengths.y, box.lengths.z};
    Slot& s = Contexts::get().slot("");
    std::lock_guard<std::mutex> lk(s.mu);
    in.edge_offset.assign(static_cast<std::size_t>(n) + 1, 0);
    int cap = 48 * (n > 0 ? n : 1), ne = 0;
    std::vector<int> nbr;
    std::vector<double> dr;
    for (;;) {
        nbr.resize(static_cast<std::size_t>(cap));
        dr.resize(3 * static_cast<std::size_t>(cap));
        check_code(hmdp_build_neighbors(s.ctx, n, x.data(), b, rc_model, cap, in.edge_offset.data(),
                                        nbr.data(), dr.data(), &ne));
        if (ne <= cap) break;
        cap = ne;
    }
    in.edge_neighbor.assign(nbr.begin(), nbr.begin() + ne);
    in.edge_dr.resize(static_cast<std::size_t>(ne));
    for (int e = 0; e < ne; ++e) in.edge_dr[e] = Vec3{dr[3 * e], dr[3 * e + 1], dr[3 * e + 2]};
    return in;
}

// evaluate_impl<T> (inference.cpp:183-416) on the device: input.check() and
// model.validate() first, then the receptive-field check, then E / F / W.
NnOutput evaluate(const NnModel& model, const NnInput& input, Precision prec,
                  NnCounters* counters) {
    input.check();
    model.validate();
    const int n = input.n_atoms();
    Slot& s = Contexts::get().slot(model_to_json(model));
    std::lock_guard<std::mutex> lk(s.mu);
    const std::vector<double> dr = flat3(input.edge_dr);
    const std::vector<unsigned char> ghost(input.is_ghost.begin(), input.is_ghost.end());
    NnOutput out;
    out.per_atom_energy.assign(static_cast<std::size_t>(n), 0.0);
    std::vector<double> f(3 * static_cast<std::size_t>(n));
    uint64_t cnt[2] = {0, 0};
    double e = 0.0, w = 0.0;
    const double cov = std::isfinite(input.coverage_radius) ? input.coverage_radius : 1e300;
    check_code(hmdp_compute_csr(s.ctx, n, input.types.data(), ghost.data(), input.edge_offset.data(),
                                input.edge_neighbor.data(), dr.data(), cov,
                                input.skip_coverage_check ? 1 : 0,
                                prec == Precision::fp64 ? HMDP_FP64 : HMDP_FP32, &e,
                                out.per_atom_energy.data(), f.data(), nullptr, &w, nullptr, nullptr,
                                nullptr, cnt));
    out.energy = e;
    out.virial = w;
    out.forces.resize(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) out.forces[i] = Vec3{f[3 * i], f[3 * i + 1], f[3 * i + 2]};
    if (counters && n > 0) {  // n == 0 returns before the tally (inference.cpp:205)
        NnCounters c;
        c.flops = cnt[0];
        c.peak_activation_bytes = cnt[1];
        c.inferences = 1;
        counters->merge(c);
    }
    return out;
}

// descriptors (inference.cpp:430-447), FP64 on the device.
std::vector<std::vector<double>> descriptors(const NnModel& model, const NnInput& input) {
    input.check();
    const int n = input.n_atoms();
    const int nd = model.descriptor_dim();
    std::vector<std::vector<double>> out(static_cast<std::size_t>(n), std::vector<double>(nd, 0.0));
    if (n == 0) return out;
    Slot& s = Contexts::get().slot(model_to_json(model));
    std::lock_guard<std::mutex> lk(s.mu);
    std::vector<double> flat(static_cast<std::size_t>(n) * nd);
    const std::vector<double> dr = flat3(input.edge_dr);
    check_code(hmdp_descriptors(s.ctx, n, input.types.data(), input.edge_offset.data(),
                                input.edge_neighbor.data(), dr.data(), flat.data()));
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < nd; ++k) out[i][k] = flat[static_cast<std::size_t>(i) * nd + k];
    return out;
}

}  // namespace halomd::nn
