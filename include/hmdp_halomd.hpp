// hmdp_halomd.hpp — header-only C++ drop-in for the reference's NN force-provider
// API (/root/reference/proj/include/halomd/nn/inference.hpp), over the C-ABI in
// hmdp.h.
//
// Include it after the reference's headers; every function is a template over
// the caller's own types (NnModel, NnInput, NnOutput, SimBox, Vec3, State), so a
// reference-side call site switches to the B200 path by changing the namespace:
//
//   halomd::nn::build_input_periodic(pos, types, gidx, box, rc)  -> hmdp::halomd::build_input_periodic<NnInput>(...)
//   halomd::nn::evaluate(model, input, prec, &counters)          -> hmdp::halomd::evaluate<NnOutput>(model, input, prec, &counters)
//   halomd::nn::descriptors(model, input)                        -> hmdp::halomd::descriptors(model, input)
//   halomd::nn::switch_value / switch_derivative                 -> hmdp::halomd::switch_value / switch_derivative
//   ForceFunction (integrators.hpp:35)                           -> hmdp::halomd::force_function(model, types, prec)
//   NNPot hybrid coupling (no reference code):
//     plan_group_preprocessing(topo, "protein")                  -> hmdp::halomd::plan_group_preprocessing(topo, name)
//     nn_force_provider(state, topo', plan, model)               -> hmdp::halomd::nn_force_provider(state, plan, model, prec)
//
// Semantics follow the reference: same argument meaning, energies for owned
// atoms only, forces for every input atom, std::invalid_argument /
// std::runtime_error with the reference's messages.  Model weights reach the
// device through the reference's own JSON (model_to_json, model.cpp:147-163),
// passed in by the caller as `to_json` (halomd::nn::model_to_json).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <algorithm>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "hmdp.h"

namespace hmdp::halomd {

inline void check(int code) {
    if (code == HMDP_OK) return;
    const std::string msg = hmdp_last_error();
    if (code == HMDP_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

// One device context per model JSON (contexts are not shared across threads
// without this lock, include/hmdp.h).
class ContextCache {
   public:
    static ContextCache& get() {
        static ContextCache c;
        return c;
    }
    hmdp_ctx* ctx(const std::string& json, int device = 0) {
        std::lock_guard<std::mutex> lk(mu_);
        auto key = std::make_pair(json, device);
        auto it = map_.find(key);
        if (it != map_.end()) return it->second.get();
        hmdp_ctx* c = nullptr;
        check(hmdp_create(json.empty() ? nullptr : json.data(), json.size(), device, 1024, 0, &c));
        map_.emplace(key, std::unique_ptr<hmdp_ctx, int (*)(hmdp_ctx*)>(c, &hmdp_destroy));
        return c;
    }
    std::mutex& lock() { return mu_; }

   private:
    std::mutex mu_;
    std::map<std::pair<std::string, int>, std::unique_ptr<hmdp_ctx, int (*)(hmdp_ctx*)>> map_;
};

// The device neighbour search is fully periodic (SimBox::periodic, box.hpp:10-13):
// a box with an open axis is rejected instead of being silently wrapped.
template <class SimBox>
void require_periodic(const SimBox& box) {
    for (int a = 0; a < 3; ++a)
        if (!box.periodic[a])
            throw std::invalid_argument(
                "B200 neighbour search supports fully periodic boxes only (axis " +
                std::to_string(a) + " is not periodic)");
}

template <class Vec3>
std::vector<double> flat3(const std::vector<Vec3>& v) {
    std::vector<double> out(3 * v.size());
    for (std::size_t i = 0; i < v.size(); ++i) {
        out[3 * i] = v[i].x;
        out[3 * i + 1] = v[i].y;
        out[3 * i + 2] = v[i].z;
    }
    return out;
}

// build_input_periodic (inference.cpp:449-487): device cell-list search,
// bit-exact pair set and order, FP64 edge_dr.
template <class NnInput, class Vec3, class SimBox>
NnInput build_input_periodic(const std::vector<Vec3>& positions, const std::vector<int>& types,
                             const std::vector<int>& global_index, const SimBox& box,
                             double rc_model, int device = 0) {
    if (positions.size() != types.size() || positions.size() != global_index.size())
        throw std::invalid_argument("positions/types/global_index size mismatch");
    const int n = static_cast<int>(positions.size());
    NnInput in;
    in.positions = positions;
    in.types = types;
    in.global_index = global_index;
    in.is_ghost.assign(n, 0);
    const std::vector<double> x = flat3(positions);
    require_periodic(box);
    const double b[3] = {box.lengths.x, box.lengths.y, box.lengths.z};
    hmdp_ctx* c = ContextCache::get().ctx("", device);
    std::lock_guard<std::mutex> lk(ContextCache::get().lock());
    std::vector<int> offset(n + 1);
    int cap = 48 * (n > 0 ? n : 1), ne = 0;
    std::vector<int> nbr;
    std::vector<double> dr;
    for (;;) {
        nbr.resize(cap);
        dr.resize(3 * static_cast<std::size_t>(cap));
        check(hmdp_build_neighbors(c, n, x.data(), b, rc_model, cap, offset.data(), nbr.data(),
                                   dr.data(), &ne));
        if (ne <= cap) break;
        cap = ne;
    }
    in.edge_offset = offset;
    in.edge_neighbor.assign(nbr.begin(), nbr.begin() + ne);
    in.edge_dr.resize(ne);
    for (int e = 0; e < ne; ++e) {
        in.edge_dr[e].x = dr[3 * e];
        in.edge_dr[e].y = dr[3 * e + 1];
        in.edge_dr[e].z = dr[3 * e + 2];
    }
    return in;
}

// evaluate (inference.cpp:420-424): prec is the caller's Precision enum
// (forcefield.hpp:10; fp32 = 0, fp64 = 1, the same values as HMDP_FP32/FP64).
template <class NnOutput, class NnModel, class NnInput, class Precision, class Counters,
          class ToJson>
NnOutput evaluate(const NnModel& model, const NnInput& in, Precision prec, Counters* counters,
                  ToJson&& to_json, int device = 0) {
    const int n = static_cast<int>(in.types.size());
    if (in.positions.size() != static_cast<std::size_t>(n) ||
        in.global_index.size() != static_cast<std::size_t>(n) ||
        in.is_ghost.size() != static_cast<std::size_t>(n))
        throw std::invalid_argument("NnInput arrays disagree on atom count");
    if (in.edge_offset.size() != static_cast<std::size_t>(n) + 1)
        throw std::invalid_argument("NnInput edge_offset has wrong size");
    if (in.edge_neighbor.size() != in.edge_dr.size())
        throw std::invalid_argument("NnInput edge arrays disagree");
    hmdp_ctx* c = ContextCache::get().ctx(to_json(model), device);
    std::lock_guard<std::mutex> lk(ContextCache::get().lock());
    const std::vector<double> dr = flat3(in.edge_dr);
    std::vector<unsigned char> ghost(in.is_ghost.begin(), in.is_ghost.end());
    NnOutput out;
    out.per_atom_energy.assign(n, 0.0);
    out.forces.resize(n);
    std::vector<double> f(3 * static_cast<std::size_t>(n)), w9(9);
    uint64_t cnt[2] = {0, 0};
    double e = 0.0, w = 0.0;
    const double cov = std::isfinite(in.coverage_radius) ? in.coverage_radius : 1e300;
    check(hmdp_compute_csr(c, n, in.types.data(), ghost.data(), in.edge_offset.data(),
                           in.edge_neighbor.data(), dr.data(), cov, in.skip_coverage_check ? 1 : 0,
                           static_cast<int>(prec) == 1 ? HMDP_FP64 : HMDP_FP32, &e,
                           out.per_atom_energy.data(), f.data(), w9.data(), &w, nullptr, nullptr,
                           nullptr, cnt));
    out.energy = e;
    out.virial = w;
    for (int i = 0; i < n; ++i) {
        out.forces[i].x = f[3 * i];
        out.forces[i].y = f[3 * i + 1];
        out.forces[i].z = f[3 * i + 2];
    }
    if (counters) {
        counters->flops += cnt[0];
        if (cnt[1] > counters->peak_activation_bytes) counters->peak_activation_bytes = cnt[1];
        counters->inferences += 1;
    }
    return out;
}

// descriptors (inference.cpp:430-447), FP64.
template <class NnModel, class NnInput, class ToJson>
std::vector<std::vector<double>> descriptors(const NnModel& model, const NnInput& in,
                                             ToJson&& to_json, int device = 0) {
    const int n = static_cast<int>(in.types.size());
    hmdp_ctx* c = ContextCache::get().ctx(to_json(model), device);
    std::lock_guard<std::mutex> lk(ContextCache::get().lock());
    const int nd = model.descriptor_dim();
    std::vector<double> flat(static_cast<std::size_t>(n) * nd), dr = flat3(in.edge_dr);
    check(hmdp_descriptors(c, n, in.types.data(), in.edge_offset.data(), in.edge_neighbor.data(),
                           dr.data(), flat.data()));
    std::vector<std::vector<double>> out(n, std::vector<double>(nd));
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < nd; ++k) out[i][k] = flat[static_cast<std::size_t>(i) * nd + k];
    return out;
}

inline double switch_value(double r, double rc) { return hmdp_switch_value(r, rc); }
inline double switch_derivative(double r, double rc) { return hmdp_switch_derivative(r, rc); }

// NNPot-style ForceFunction (integrators.hpp:35): recompute
// forces for the current positions (all atoms owned, periodic box), store them
// in state.forces, return the potential energy.
template <class State, class NnModel, class ToJson>
std::function<double(State&)> force_function(const NnModel& model, std::vector<int> types,
                                             int prec, ToJson&& to_json, int device = 0) {
    hmdp_ctx* c = ContextCache::get().ctx(to_json(model), device);
    return [c, types = std::move(types), prec](State& st) -> double {
        std::lock_guard<std::mutex> lk(ContextCache::get().lock());
        const int n = static_cast<int>(st.positions.size());
        if (static_cast<int>(types.size()) != n)
            throw std::invalid_argument("positions/types/global_index size mismatch");
        const std::vector<double> x = flat3(st.positions);
        require_periodic(st.box);
        const double b[3] = {st.box.lengths.x, st.box.lengths.y, st.box.lengths.z};
        std::vector<double> f(3 * static_cast<std::size_t>(n));
        double e = 0.0;
        check(hmdp_compute(c, n, x.data(), types.data(), b, prec == 1 ? HMDP_FP64 : HMDP_FP32,
                           &e, nullptr, f.data(), nullptr, nullptr));
        st.forces.resize(n);
        for (int i = 0; i < n; ++i) {
            st.forces[i].x = f[3 * i];
            st.forces[i].y = f[3 * i + 1];
            st.forces[i].z = f[3 * i + 2];
        }
        return e;
    };
}

// ---------------------------------------------------------------------------
// NNPot-style hybrid coupling (SPEC.md:375-383 plan_group_preprocessing,
// :411-419 nn_force_provider; the paper's Fig. 2).  The reference declares the
// contract but ships no code; these follow it on the caller's own Topology /
// State types (topology.hpp, state.hpp).
// ---------------------------------------------------------------------------

// Everything plan_group_preprocessing removed or added, so it can be undone.
template <class Topology>
struct NnGroupPlan {
    std::string group;
    std::vector<int> atoms;  // sorted, duplicate-free (Topology::groups)
    std::vector<typename decltype(Topology::bonds)::value_type> removed_bonds;
    std::vector<typename decltype(Topology::angles)::value_type> removed_angles;
    std::vector<typename decltype(Topology::dihedrals)::value_type> removed_dihedrals;
    std::vector<std::pair<int, int>> added_exclusions;  // i < j, previously not excluded
};

// Removes every bonded term whose atoms all lie in the group and excludes every
// in-group pair (symmetrically); cross-group terms and pairs are untouched.  An
// empty group is a no-op.  Throws std::invalid_argument for an unknown group.
template <class Topology>
NnGroupPlan<Topology> plan_group_preprocessing(Topology& topo, const std::string& group) {
    auto it = topo.groups.find(group);
    if (it == topo.groups.end()) throw std::invalid_argument("unknown atom group: " + group);
    NnGroupPlan<Topology> plan;
    plan.group = group;
    plan.atoms = it->second;
    if (plan.atoms.empty()) return plan;
    std::vector<char> in(static_cast<std::size_t>(topo.n_atoms), 0);
    for (int a : plan.atoms) in[static_cast<std::size_t>(a)] = 1;
    auto split = [](auto& terms, auto& removed, auto inside) {
        auto keep = terms.begin();
        for (auto t = terms.begin(); t != terms.end(); ++t) {
            if (inside(*t)) removed.push_back(*t);
            else *keep++ = *t;
        }
        terms.erase(keep, terms.end());
    };
    split(topo.bonds, plan.removed_bonds, [&](const auto& b) { return in[b.i] && in[b.j]; });
    split(topo.angles, plan.removed_angles,
          [&](const auto& a) { return in[a.i] && in[a.j] && in[a.k]; });
    split(topo.dihedrals, plan.removed_dihedrals,
          [&](const auto& d) { return in[d.i] && in[d.j] && in[d.k] && in[d.l]; });
    for (std::size_t p = 0; p < plan.atoms.size(); ++p)
        for (std::size_t q = p + 1; q < plan.atoms.size(); ++q) {
            const int i = plan.atoms[p], j = plan.atoms[q];
            if (!topo.excluded(i, j)) {
                topo.add_exclusion(i, j);
                plan.added_exclusions.emplace_back(i, j);
            }
        }
    return plan;
}

// Reverts plan_group_preprocessing (bonded terms re-appended, added exclusions
// dropped).
template <class Topology>
void undo_group_preprocessing(Topology& topo, const NnGroupPlan<Topology>& plan) {
    topo.bonds.insert(topo.bonds.end(), plan.removed_bonds.begin(), plan.removed_bonds.end());
    topo.angles.insert(topo.angles.end(), plan.removed_angles.begin(), plan.removed_angles.end());
    topo.dihedrals.insert(topo.dihedrals.end(), plan.removed_dihedrals.begin(),
                          plan.removed_dihedrals.end());
    for (const auto& [i, j] : plan.added_exclusions) {
        auto drop = [&](int a, int b) {
            auto& v = topo.exclusions[static_cast<std::size_t>(a)];
            v.erase(std::remove(v.begin(), v.end(), b), v.end());
        };
        drop(i, j);
        drop(j, i);
    }
}

// The coupling layer: extracts the group's positions (on the device), runs the DP
// model on them, ADDS the group's NN forces into state.forces and returns the NN
// energy.  The caller's classical force field supplies everything else, including
// every cross-group interaction.
template <class State, class Topology, class NnModel, class ToJson>
double nn_force_provider(State& state, const std::vector<int>& type_of,
                         const NnGroupPlan<Topology>& plan, const NnModel& model, int prec,
                         ToJson&& to_json, int device = 0) {
    hmdp_ctx* c = ContextCache::get().ctx(to_json(model), device);
    std::lock_guard<std::mutex> lk(ContextCache::get().lock());
    const int n = static_cast<int>(state.positions.size());
    if (static_cast<int>(type_of.size()) != n)
        throw std::invalid_argument("positions/types/global_index size mismatch");
    if (static_cast<int>(state.forces.size()) != n) state.forces.resize(n);
    const std::vector<double> x = flat3(state.positions);
    std::vector<double> f = flat3(state.forces);
    require_periodic(state.box);
    const double b[3] = {state.box.lengths.x, state.box.lengths.y, state.box.lengths.z};
    double e = 0.0;
    check(hmdp_compute_group(c, n, x.data(), type_of.data(), plan.atoms.data(),
                             static_cast<int>(plan.atoms.size()), b,
                             prec == 1 ? HMDP_FP64 : HMDP_FP32, &e, f.data(), nullptr, nullptr));
    for (int i = 0; i < n; ++i) {
        state.forces[i].x = f[3 * i];
        state.forces[i].y = f[3 * i + 1];
        state.forces[i].z = f[3 * i + 2];
    }
    return e;
}

}  // namespace hmdp::halomd
