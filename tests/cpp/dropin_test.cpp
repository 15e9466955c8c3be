// dropin_test.cpp — TEST INFRASTRUCTURE: the reference's own call sites with the
// B200 path swapped in through include/hmdp_halomd.hpp.  Linked against the
// reference compiled from its sources (oracle/Makefile target `dropin`); the
// binary lands in oracle/_ref/ and runs on the GPU box (tests/test_gpu_dropin.py).
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "halomd/forcefield.hpp"
#include "halomd/integrators.hpp"
#include "halomd/neighborlist.hpp"
#include "halomd/nn/inference.hpp"
#include "halomd/nn/model.hpp"
#include "halomd/synthetic.hpp"
#include "hmdp_halomd.hpp"

using namespace halomd;

static int fails = 0;
#define EXPECT(cond, ...)                  \
    do {                                   \
        if (!(cond)) {                     \
            std::printf("FAIL: " __VA_ARGS__); \
            std::printf("\n");             \
            ++fails;                       \
        }                                  \
    } while (0)

static double rms(const std::vector<Vec3>& f) {
    double s = 0;
    for (const auto& v : f) s += norm2(v);
    return std::sqrt(s / f.size());
}

int main() {
    SyntheticParams p;
    p.n_atoms = 582;
    p.density = 33.4;
    p.fraction_grouped = 0.35;
    p.seed = 7;
    auto [topo, st] = generate_synthetic_system(p);
    const int n = st.n_atoms();
    std::vector<int> gidx(n);
    for (int i = 0; i < n; ++i) gidx[i] = i;
    auto to_json = [](const nn::NnModel& m) { return nn::model_to_json(m); };

    // build_input_periodic: bit-exact CSR
    auto ref_in = nn::build_input_periodic(st.positions, topo.type_of, gidx, st.box, 0.6);
    auto our_in = hmdp::halomd::build_input_periodic<nn::NnInput>(st.positions, topo.type_of, gidx,
                                                                   st.box, 0.6);
    EXPECT(ref_in.edge_offset == our_in.edge_offset, "edge_offset differs");
    EXPECT(ref_in.edge_neighbor == our_in.edge_neighbor, "edge_neighbor differs");
    EXPECT(ref_in.edge_dr == our_in.edge_dr, "edge_dr differs (must be bit-exact)");

    // an open axis is rejected (the device search is fully periodic), not wrapped
    {
        SimBox open_box = st.box;
        open_box.periodic[2] = false;
        bool threw = false;
        try {
            hmdp::halomd::build_input_periodic<nn::NnInput>(st.positions, topo.type_of, gidx,
                                                           open_box, 0.6);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        EXPECT(threw, "non-periodic axis must raise std::invalid_argument");
    }

    for (auto fam : {nn::ModelFamily::embed_fit, nn::ModelFamily::message_passing}) {
        const int depth = fam == nn::ModelFamily::embed_fit ? 1 : 3;
        auto model = nn::make_model(fam, depth, 0.6, 2, 8, 32, 1);
        nn::NnCounters rc, oc;
        auto ref = nn::evaluate(model, ref_in, Precision::fp64, &rc);
        for (auto prec : {Precision::fp64, Precision::fp32}) {
            auto out = hmdp::halomd::evaluate<nn::NnOutput>(model, ref_in, prec, &oc, to_json);
            const double etol = prec == Precision::fp64 ? 1e-11 : 1e-6;
            const double ftol = prec == Precision::fp64 ? 1e-10 : 1e-4;
            double df = 0;
            for (int i = 0; i < n; ++i) df = std::max(df, std::sqrt(norm2(out.forces[i] - ref.forces[i])));
            EXPECT(std::fabs(out.energy - ref.energy) <= etol * std::fabs(ref.energy),
                   "depth %d energy %.12f vs %.12f", depth, out.energy, ref.energy);
            EXPECT(df <= ftol * rms(ref.forces), "depth %d force err %.3e", depth, df / rms(ref.forces));
            EXPECT(std::fabs(out.virial - ref.virial) <= ftol * std::max(std::fabs(ref.virial), rms(ref.forces)),
                   "depth %d virial %.10f vs %.10f", depth, out.virial, ref.virial);
        }
        EXPECT(oc.flops == 2 * rc.flops, "counters %llu vs %llu", (unsigned long long)oc.flops,
               (unsigned long long)rc.flops);
        // receptive-field error with the reference's message
        auto in2 = ref_in;
        in2.coverage_radius = 0.5;
        if (depth > 1) {
            bool threw = false;
            try {
                hmdp::halomd::evaluate<nn::NnOutput>(model, in2, Precision::fp64, (nn::NnCounters*)nullptr, to_json);
            } catch (const std::runtime_error& e) {
                threw = std::string(e.what()).rfind("receptive-field error", 0) == 0;
            }
            EXPECT(threw, "receptive-field error not raised");
        }
        // ForceFunction drop-in: 5 velocity-Verlet steps, reference vs B200 provider (FP64)
        State a = st, b = st;
        ForceFunction ref_ff = [&](State& s) {
            auto in = nn::build_input_periodic(s.positions, topo.type_of, gidx, s.box, 0.6);
            auto o = nn::evaluate(model, in, Precision::fp64);
            s.forces = o.forces;
            return o.energy;
        };
        ForceFunction our_ff = hmdp::halomd::force_function<State>(model, topo.type_of, 1, to_json);
        ref_ff(a);
        our_ff(b);
        for (int s = 0; s < 5; ++s) {
            velocity_verlet_step(a, ref_ff, 0.001, topo.mass);
            velocity_verlet_step(b, our_ff, 0.001, topo.mass);
        }
        double dx = 0;
        for (int i = 0; i < n; ++i) dx = std::max(dx, std::sqrt(norm2(a.positions[i] - b.positions[i])));
        EXPECT(dx < 1e-11, "depth %d MD trajectory differs by %.3e nm", depth, dx);
    }
    auto d_ref = nn::descriptors(nn::make_model(nn::ModelFamily::embed_fit, 1, 0.6, 2, 8, 32, 1), ref_in);
    auto d_our = hmdp::halomd::descriptors(nn::make_model(nn::ModelFamily::embed_fit, 1, 0.6, 2, 8, 32, 1),
                                           ref_in, to_json);
    double dd = 0;
    for (int i = 0; i < n; ++i)
        for (std::size_t k = 0; k < d_ref[i].size(); ++k) dd = std::max(dd, std::fabs(d_ref[i][k] - d_our[i][k]));
    EXPECT(dd < 1e-12, "descriptors differ by %.3e", dd);
    EXPECT(hmdp::halomd::switch_value(0.57, 0.6) == nn::switch_value(0.57, 0.6), "switch_value");

    // NNPot hybrid coupling on the reference's own
    // Topology/State: group preprocessing, the group provider against the reference
    // evaluate() on the extracted group, and hybrid velocity-Verlet steps with the
    // reference's classical force field on the preprocessed topology.
    {
        Topology t2 = topo;
        auto plan = hmdp::halomd::plan_group_preprocessing(t2, "protein");
        const auto& grp = topo.groups.at("protein");
        const int ng = static_cast<int>(grp.size());
        std::vector<char> in(n, 0);
        for (int a : grp) in[a] = 1;
        bool ok = true;
        for (const auto& b : t2.bonds) ok &= !(in[b.i] && in[b.j]);
        for (const auto& a : t2.angles) ok &= !(in[a.i] && in[a.j] && in[a.k]);
        for (const auto& d : t2.dihedrals) ok &= !(in[d.i] && in[d.j] && in[d.k] && in[d.l]);
        EXPECT(ok, "in-group bonded term survived preprocessing");
        EXPECT(t2.bonds.size() + plan.removed_bonds.size() == topo.bonds.size(), "bond bookkeeping");
        bool excl = true;
        for (int p2 = 0; p2 < ng && excl; ++p2)
            for (int q = p2 + 1; q < ng; ++q) excl &= t2.excluded(grp[p2], grp[q]);
        EXPECT(excl, "in-group pair not excluded");
        t2.validate();

        auto model = nn::make_model(nn::ModelFamily::message_passing, 3, 0.6, 2, 8, 32, 1);
        State s = st;
        s.forces.assign(n, Vec3{});
        const double e_nn = hmdp::halomd::nn_force_provider(s, topo.type_of, plan, model, 1, to_json);
        std::vector<Vec3> gpos;
        std::vector<int> gty, ggi;
        for (int k = 0; k < ng; ++k) {
            gpos.push_back(st.positions[grp[k]]);
            gty.push_back(topo.type_of[grp[k]]);
            ggi.push_back(k);
        }
        auto gin = nn::build_input_periodic(gpos, gty, ggi, st.box, 0.6);
        auto gref = nn::evaluate(model, gin, Precision::fp64);
        EXPECT(std::fabs(e_nn - gref.energy) <= 1e-11 * std::fabs(gref.energy),
               "group energy %.12f vs %.12f", e_nn, gref.energy);
        double dfg = 0, other = 0;
        Vec3 sum{};
        for (int k = 0; k < ng; ++k) {
            dfg = std::max(dfg, std::sqrt(norm2(s.forces[grp[k]] - gref.forces[k])));
            sum = sum + s.forces[grp[k]];
        }
        for (int i = 0; i < n; ++i)
            if (!in[i]) other = std::max(other, std::sqrt(norm2(s.forces[i])));
        EXPECT(dfg <= 1e-10 * rms(gref.forces), "group forces differ %.3e", dfg);
        EXPECT(other == 0.0, "NN provider touched a non-group atom");
        EXPECT(std::sqrt(norm2(sum)) <= 1e-8 * rms(gref.forces) * ng, "group NN forces sum %.3e",
               std::sqrt(norm2(sum)));

        // hybrid MD: classical(topo') + NN(protein); energy stays finite and the
        // hybrid potential equals classical + NN
        ForceFieldParams ffp;
        ffp.lj.sigma = {0.33, 0.30};
        ffp.lj.epsilon = {0.40, 0.50};
        ffp.rc = 0.7;
        ffp.coulomb.rc = 0.7;
        double last_cl = 0, last_nn = 0;
        ForceFunction hybrid = [&](State& x) {
            auto nl = build_neighbor_list(x, t2, 0.7, 0.0);
            const EnergyReport rep = compute_classical(x, t2, nl, ffp);
            last_cl = rep.total_potential();
            last_nn = hmdp::halomd::nn_force_provider(x, topo.type_of, plan, model, 1, to_json);
            return last_cl + last_nn;
        };
        State h = st;
        const double e0 = hybrid(h);
        EXPECT(std::fabs(e0 - (last_cl + last_nn)) == 0.0, "hybrid energy composition");
        for (int k = 0; k < 5; ++k) velocity_verlet_step(h, hybrid, 0.001, topo.mass);
        bool finite = true;
        for (int i = 0; i < n; ++i) finite &= std::isfinite(h.positions[i].x + h.forces[i].x);
        EXPECT(finite, "hybrid MD produced non-finite state");

        hmdp::halomd::undo_group_preprocessing(t2, plan);
        EXPECT(t2.bonds.size() == topo.bonds.size() && t2.angles.size() == topo.angles.size() &&
                   t2.dihedrals.size() == topo.dihedrals.size(),
               "undo did not restore bonded terms");
        EXPECT(t2.exclusions == topo.exclusions, "undo did not restore exclusions");
    }
    std::printf(fails ? "DROPIN FAIL (%d)\n" : "DROPIN PASS\n", fails);
    return fails ? 1 : 0;
}
