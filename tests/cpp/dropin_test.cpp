// dropin_test.cpp — TEST INFRASTRUCTURE: the reference's own call sites with the
// B200 path swapped in through include/hmdp_halomd.hpp.  Linked against the
// reference compiled from its sources (oracle/Makefile target `dropin`); the
// binary lands in oracle/_ref/ and runs on the GPU box (tests/test_gpu_dropin.py).
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "halomd/integrators.hpp"
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
    std::printf(fails ? "DROPIN FAIL (%d)\n" : "DROPIN PASS\n", fails);
    return fails ? 1 : 0;
}
