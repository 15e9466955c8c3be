// dropin_exact.cpp — TEST INFRASTRUCTURE: reference call sites, written exactly as
// reference code calls the NN force-provider API (halomd::nn::build_input_periodic,
// evaluate, descriptors, switch_value / switch_derivative, a ForceFunction inside
// velocity_verlet_step), with NO B200 header and NO change at any call site.
//
// oracle/Makefile `dropin_exact` links it against the reference objects MINUS
// inference.o plus libhalomd_nn_b200.so (paper_2602_02234_b200/csrc/halomd_nn_b200.cpp),
// so every nn:: call below runs on the GPU.  It writes its results as raw arrays
// into the directory argv[1]; tests/test_gpu_dropin.py compares them with the
// reference itself (oracle/_ref/libhalomd_ref.so, loaded in the test process).
#include <cstdio>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "halomd/integrators.hpp"
#include "halomd/nn/inference.hpp"
#include "halomd/nn/model.hpp"
#include "halomd/synthetic.hpp"

using namespace halomd;

static std::string g_dir;

template <class T>
static void dump(const std::string& name, const std::vector<T>& v) {
    std::ofstream f(g_dir + "/" + name, std::ios::binary);
    f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(T)));
}

static std::vector<double> flat(const std::vector<Vec3>& v) {
    std::vector<double> o;
    for (const auto& x : v) o.insert(o.end(), {x.x, x.y, x.z});
    return o;
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    g_dir = argv[1];
    std::ofstream log(g_dir + "/log.txt");
    for (int natoms : {582, 1231}) {
        SyntheticParams p;
        p.n_atoms = natoms;
        p.density = 33.4;
        p.fraction_grouped = 0.35;
        p.seed = 7;
        auto [topo, st] = generate_synthetic_system(p);
        const int n = st.n_atoms();
        std::vector<int> gidx(n);
        for (int i = 0; i < n; ++i) gidx[i] = i;
        const std::string tag = std::to_string(natoms);

        nn::NnInput in = nn::build_input_periodic(st.positions, topo.type_of, gidx, st.box, 0.6);
        dump("offset_" + tag, in.edge_offset);
        dump("nbr_" + tag, in.edge_neighbor);
        dump("dr_" + tag, flat(in.edge_dr));

        for (auto fam : {nn::ModelFamily::embed_fit, nn::ModelFamily::message_passing}) {
            const int depth = fam == nn::ModelFamily::embed_fit ? 1 : 3;
            const nn::NnModel model = nn::make_model(fam, depth, 0.6, 2, 8, 32, 1);
            for (auto prec : {Precision::fp64, Precision::fp32}) {
                nn::NnCounters c;
                const nn::NnOutput out = nn::evaluate(model, in, prec, &c);
                const std::string k = tag + "_d" + std::to_string(depth) +
                                      (prec == Precision::fp64 ? "_f64" : "_f32");
                dump("forces_" + k, flat(out.forces));
                dump("pae_" + k, out.per_atom_energy);
                dump("scalars_" + k, std::vector<double>{out.energy, out.virial,
                                                         static_cast<double>(c.flops),
                                                         static_cast<double>(c.peak_activation_bytes),
                                                         static_cast<double>(c.inferences)});
            }
            if (natoms == 582) {
                // receptive-field error (inference.cpp:188-193)
                nn::NnInput narrow = in;
                narrow.coverage_radius = 0.5;
                try {
                    nn::evaluate(model, narrow, Precision::fp64);
                    log << "coverage_d" << depth << " no-throw\n";
                } catch (const std::runtime_error& e) {
                    log << "coverage_d" << depth << " runtime_error " << e.what() << "\n";
                }
                // the ForceFunction call site (integrators.hpp:35) in 5 velocity-Verlet steps
                State s = st;
                const Precision pr = Precision::fp64;
                ForceFunction ff = [&](State& x) {
                    auto input = nn::build_input_periodic(x.positions, topo.type_of, gidx, x.box,
                                                          model.rc_model);
                    auto o = nn::evaluate(model, input, pr);
                    x.forces = o.forces;
                    return o.energy;
                };
                ff(s);
                for (int k = 0; k < 5; ++k) velocity_verlet_step(s, ff, 0.001, topo.mass);
                dump("md_x_d" + std::to_string(depth), flat(s.positions));
                dump("md_v_d" + std::to_string(depth), flat(s.velocities));
            }
        }
        if (natoms == 582) {
            const nn::NnModel m1 = nn::make_model(nn::ModelFamily::embed_fit, 1, 0.6, 2, 8, 32, 1);
            std::vector<double> d;
            for (const auto& row : nn::descriptors(m1, in)) d.insert(d.end(), row.begin(), row.end());
            dump("desc_582", d);
            std::vector<double> sw;
            for (double r : {0.1, 0.54, 0.55, 0.57, 0.59, 0.6, 0.7})
                sw.insert(sw.end(), {nn::switch_value(r, 0.6), nn::switch_derivative(r, 0.6)});
            dump("switch", sw);
            // argument errors (inference.cpp:19-32, :452-453)
            try {
                std::vector<int> short_types(topo.type_of.begin(), topo.type_of.end() - 1);
                nn::build_input_periodic(st.positions, short_types, gidx, st.box, 0.6);
                log << "mismatch no-throw\n";
            } catch (const std::invalid_argument& e) {
                log << "mismatch invalid_argument " << e.what() << "\n";
            }
            try {
                nn::NnInput bad = in;
                bad.edge_neighbor[0] = n + 5;
                nn::evaluate(m1, bad, Precision::fp64);
                log << "badnbr no-throw\n";
            } catch (const std::invalid_argument& e) {
                log << "badnbr invalid_argument " << e.what() << "\n";
            }
            try {
                nn::build_input_periodic(st.positions, topo.type_of, gidx, st.box, 0.6 * 3);
                log << "halfbox no-throw\n";
            } catch (const std::invalid_argument& e) {
                log << "halfbox invalid_argument " << e.what() << "\n";
            }
        }
    }
    log << "DONE\n";
    std::printf("DROPIN_EXACT DONE\n");
    return 0;
}
