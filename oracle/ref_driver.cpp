// ref_driver.cpp — TEST INFRASTRUCTURE ONLY (checker + CPU baseline, never the product).
//
// A thin extern "C" surface over the *unmodified* reference sources compiled
// from /root/reference/proj/src (see oracle/Makefile), so that Python tests,
// the golden-vector generator and bench.py's `--impl reference` arm can call
// the reference's own hot path:
//   halomd::generate_synthetic_system   proj/src/synthetic.cpp:36
//   halomd::nn::make_model              proj/src/nn/model.cpp:70
//   halomd::nn::model_to_json           proj/src/nn/model.cpp:147
//   halomd::nn::build_input_periodic    proj/src/nn/inference.cpp:449
//   halomd::nn::evaluate                proj/src/nn/inference.cpp:420
//   halomd::nn::descriptors             proj/src/nn/inference.cpp:430
//   halomd::velocity_verlet_step        proj/src/integrators.cpp:32
// Exceptions are mapped to return codes 1 (invalid_argument) / 2 (runtime_error)
// with the message retrievable through ref_last_error().
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "halomd/forcefield.hpp"
#include "halomd/integrators.hpp"
#include "halomd/neighborlist.hpp"
#include "halomd/nn/inference.hpp"
#include "halomd/nn/model.hpp"
#include "halomd/synthetic.hpp"

using namespace halomd;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

std::vector<Vec3> to_vec3(int n, const double* xyz) {
    std::vector<Vec3> v(n);
    for (int i = 0; i < n; ++i) v[i] = Vec3(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
    return v;
}

struct InputHandle {
    nn::NnInput in;
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- fixtures -------------------------------------------------------------
int ref_synthetic(int n, double density, double fraction, uint64_t seed, double temperature,
                  double* pos, int* types, double* masses, double* vel, double* box) {
    return guarded([&] {
        SyntheticParams p;
        p.n_atoms = n;
        p.density = density;
        p.fraction_grouped = fraction;
        p.seed = seed;
        p.temperature = temperature;
        auto [topo, st] = generate_synthetic_system(p);
        for (int i = 0; i < n; ++i) {
            for (int a = 0; a < 3; ++a) {
                pos[3 * i + a] = st.positions[i][a];
                vel[3 * i + a] = st.velocities[i][a];
            }
            types[i] = topo.type_of[i];
            masses[i] = topo.mass[i];
        }
        for (int a = 0; a < 3; ++a) box[a] = st.box.lengths[a];
    });
}

// ---- classical force field (forcefield.cpp) on the synthetic topology -------
// The synthetic system's topology (synthetic.cpp:36-130) exported as flat arrays
// (call with NULL arrays to get the counts: counts[0..3] = bonds, angles,
// dihedrals, exclusion entries).
int ref_synthetic_topology(int n, double density, double fraction, uint64_t seed, int* counts,
                           double* charges, int* excl_offset, int* excl, int* bonds,
                           double* bond_p, int* angles, double* angle_p, int* dih, double* dih_p) {
    return guarded([&] {
        SyntheticParams p;
        p.n_atoms = n;
        p.density = density;
        p.fraction_grouped = fraction;
        p.seed = seed;
        auto [topo, st] = generate_synthetic_system(p);
        (void)st;
        long ne = 0;
        for (const auto& e : topo.exclusions) ne += static_cast<long>(e.size());
        counts[0] = static_cast<int>(topo.bonds.size());
        counts[1] = static_cast<int>(topo.angles.size());
        counts[2] = static_cast<int>(topo.dihedrals.size());
        counts[3] = static_cast<int>(ne);
        if (!charges) return;
        int k = 0;
        excl_offset[0] = 0;
        for (int i = 0; i < n; ++i) {
            charges[i] = topo.charge[i];
            for (int j : topo.exclusions[i]) excl[k++] = j;
            excl_offset[i + 1] = k;
        }
        for (size_t t = 0; t < topo.bonds.size(); ++t) {
            const auto& b = topo.bonds[t];
            bonds[2 * t] = b.i, bonds[2 * t + 1] = b.j;
            bond_p[2 * t] = b.k_b, bond_p[2 * t + 1] = b.r0;
        }
        for (size_t t = 0; t < topo.angles.size(); ++t) {
            const auto& a = topo.angles[t];
            angles[3 * t] = a.i, angles[3 * t + 1] = a.j, angles[3 * t + 2] = a.k;
            angle_p[2 * t] = a.k_a, angle_p[2 * t + 1] = a.theta0;
        }
        for (size_t t = 0; t < topo.dihedrals.size(); ++t) {
            const auto& d = topo.dihedrals[t];
            dih[4 * t] = d.i, dih[4 * t + 1] = d.j, dih[4 * t + 2] = d.k, dih[4 * t + 3] = d.l;
            dih_p[3 * t] = d.k_d, dih_p[3 * t + 1] = d.phase, dih_p[3 * t + 2] = d.multiplicity;
        }
    });
}

// compute_classical (forcefield.cpp:265-279) on the synthetic topology with the
// given positions; pair list = build_neighbor_list(.., rc, skin 0, half).
int ref_classical(int n, double density, double fraction, uint64_t seed, const double* xyz,
                  const double* sigma, const double* eps, int scheme, double rc_c, double eps_rf,
                  double rc_lj, int fp64, double* energies, double* forces, double* virial,
                  int* collinear) {
    return guarded([&] {
        SyntheticParams p;
        p.n_atoms = n;
        p.density = density;
        p.fraction_grouped = fraction;
        p.seed = seed;
        auto [topo, st] = generate_synthetic_system(p);
        for (int i = 0; i < n; ++i) st.positions[i] = Vec3{xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
        ForceFieldParams ffp;
        ffp.lj.sigma = {sigma[0], sigma[1]};
        ffp.lj.epsilon = {eps[0], eps[1]};
        ffp.rc = rc_lj;
        ffp.coulomb.rc = rc_c;
        ffp.coulomb.eps_rf = eps_rf;
        ffp.coulomb.scheme = scheme ? CoulombScheme::reaction_field : CoulombScheme::cutoff_shifted;
        auto nl = build_neighbor_list(st, topo, std::max(rc_c, rc_lj), 0.0);
        ForceDiagnostics diag;
        const EnergyReport rep = compute_classical(st, topo, nl, ffp, &diag,
                                                   fp64 ? Precision::fp64 : Precision::fp32);
        energies[0] = rep.bonded;
        energies[1] = rep.lj;
        energies[2] = rep.coulomb;
        for (int i = 0; i < n; ++i)
            for (int a = 0; a < 3; ++a) forces[3 * i + a] = st.forces[i][a];
        *virial = diag.virial;
        *collinear = diag.collinear_angles;
    });
}

// Writes the model JSON into buf (NUL-terminated); returns the length needed
// (excluding NUL) or a negative error code.
long ref_make_model_json(int family, int depth, double rc, int n_types, int n_basis, int hidden,
                         uint64_t seed, char* buf, long cap) {
    std::string s;
    int rc_code = guarded([&] {
        auto m = nn::make_model(family == 0 ? nn::ModelFamily::embed_fit
                                            : nn::ModelFamily::message_passing,
                                depth, rc, n_types, n_basis, hidden, seed);
        s = nn::model_to_json(m);
    });
    if (rc_code) return -rc_code;
    if (buf && cap > static_cast<long>(s.size())) std::memcpy(buf, s.c_str(), s.size() + 1);
    return static_cast<long>(s.size());
}

void* ref_model_load(const char* json, long len) {
    nn::NnModel* m = nullptr;
    int rc = guarded([&] { m = new nn::NnModel(nn::model_from_json(std::string(json, len))); });
    return rc ? nullptr : m;
}
void ref_model_free(void* m) { delete static_cast<nn::NnModel*>(m); }

// ---- build_input_periodic -------------------------------------------------
void* ref_input_build(int n, const double* xyz, const int* types, const double* box, double rc) {
    InputHandle* h = nullptr;
    int code = guarded([&] {
        std::vector<int> gidx(n);
        for (int i = 0; i < n; ++i) gidx[i] = i;
        auto in = nn::build_input_periodic(to_vec3(n, xyz), std::vector<int>(types, types + n),
                                           gidx, SimBox(box[0], box[1], box[2]), rc);
        h = new InputHandle{std::move(in)};
    });
    return code ? nullptr : h;
}
int ref_input_nedges(void* h) {
    return static_cast<int>(static_cast<InputHandle*>(h)->in.edge_neighbor.size());
}
void ref_input_get(void* h, int* offset, int* nbr, double* dr) {
    auto& in = static_cast<InputHandle*>(h)->in;
    for (std::size_t i = 0; i < in.edge_offset.size(); ++i) offset[i] = in.edge_offset[i];
    for (std::size_t e = 0; e < in.edge_neighbor.size(); ++e) {
        nbr[e] = in.edge_neighbor[e];
        for (int a = 0; a < 3; ++a) dr[3 * e + a] = in.edge_dr[e][a];
    }
}
void ref_input_free(void* h) { delete static_cast<InputHandle*>(h); }

// ---- evaluate on an explicit CSR input --------------------------------------
// is_ghost may be NULL. prec: 0 = fp64, 1 = fp32. virial/flops/act may be NULL.
int ref_evaluate_csr(void* model, int n, const double* xyz, const int* types,
                     const unsigned char* is_ghost, const int* offset, const int* nbr,
                     const double* dr, double coverage, int skip_cov, int prec, double* energy,
                     double* per_atom, double* forces, double* virial, uint64_t* flops,
                     uint64_t* act_bytes) {
    return guarded([&] {
        nn::NnInput in;
        in.positions = to_vec3(n, xyz);
        in.types.assign(types, types + n);
        in.global_index.resize(n);
        for (int i = 0; i < n; ++i) in.global_index[i] = i;
        in.is_ghost.assign(n, 0);
        if (is_ghost)
            for (int i = 0; i < n; ++i) in.is_ghost[i] = static_cast<char>(is_ghost[i]);
        in.edge_offset.assign(offset, offset + n + 1);
        const int ne = offset[n];
        in.edge_neighbor.assign(nbr, nbr + ne);
        in.edge_dr = to_vec3(ne, dr);
        in.coverage_radius = coverage;
        in.skip_coverage_check = skip_cov != 0;
        nn::NnCounters c;
        auto out = nn::evaluate(*static_cast<nn::NnModel*>(model), in,
                                prec == 0 ? Precision::fp64 : Precision::fp32, &c);
        *energy = out.energy;
        if (virial) *virial = out.virial;
        if (per_atom)
            for (int i = 0; i < n; ++i) per_atom[i] = out.per_atom_energy[i];
        for (int i = 0; i < n; ++i)
            for (int a = 0; a < 3; ++a) forces[3 * i + a] = out.forces[i][a];
        if (flops) *flops = c.flops;
        if (act_bytes) *act_bytes = c.peak_activation_bytes;
    });
}

// build_input_periodic + evaluate: the reference's single-domain hot path.
int ref_evaluate_periodic(void* model, int n, const double* xyz, const int* types,
                          const double* box, int prec, double* energy, double* per_atom,
                          double* forces, double* virial) {
    return guarded([&] {
        const auto& m = *static_cast<nn::NnModel*>(model);
        std::vector<int> gidx(n);
        for (int i = 0; i < n; ++i) gidx[i] = i;
        auto in = nn::build_input_periodic(to_vec3(n, xyz), std::vector<int>(types, types + n),
                                           gidx, SimBox(box[0], box[1], box[2]), m.rc_model);
        auto out = nn::evaluate(m, in, prec == 0 ? Precision::fp64 : Precision::fp32);
        *energy = out.energy;
        if (virial) *virial = out.virial;
        if (per_atom)
            for (int i = 0; i < n; ++i) per_atom[i] = out.per_atom_energy[i];
        for (int i = 0; i < n; ++i)
            for (int a = 0; a < 3; ++a) forces[3 * i + a] = out.forces[i][a];
    });
}

int ref_descriptors(void* model, int n, const double* xyz, const int* types, const int* offset,
                    const int* nbr, const double* dr, double* desc) {
    return guarded([&] {
        const auto& m = *static_cast<nn::NnModel*>(model);
        nn::NnInput in;
        in.positions = to_vec3(n, xyz);
        in.types.assign(types, types + n);
        in.global_index.resize(n);
        in.is_ghost.assign(n, 0);
        in.edge_offset.assign(offset, offset + n + 1);
        in.edge_neighbor.assign(nbr, nbr + offset[n]);
        in.edge_dr = to_vec3(offset[n], dr);
        auto d = nn::descriptors(m, in);
        const int nd = m.descriptor_dim();
        for (int i = 0; i < n; ++i)
            for (int k = 0; k < nd; ++k) desc[i * nd + k] = d[i][k];
    });
}

double ref_switch_value(double r, double rc) { return nn::switch_value(r, rc); }
double ref_switch_derivative(double r, double rc) { return nn::switch_derivative(r, rc); }

// ---- CPU baseline timing ----------------------------------------------------
// Runs `steps` force evaluations (build_input_periodic + evaluate) on each of
// `threads` std::threads concurrently (evaluate is pure and reentrant,
// SPEC.md:445), returns wall seconds. Each thread owns a private copy of the
// positions, so this is P independent replicas of the same workload.
double ref_bench_eval(void* model, int n, const double* xyz, const int* types, const double* box,
                      int prec, int steps, int threads) {
    const auto& m = *static_cast<nn::NnModel*>(model);
    const auto pos = to_vec3(n, xyz);
    const std::vector<int> ty(types, types + n);
    std::vector<int> gidx(n);
    for (int i = 0; i < n; ++i) gidx[i] = i;
    const SimBox b(box[0], box[1], box[2]);
    auto work = [&] {
        for (int s = 0; s < steps; ++s) {
            auto in = nn::build_input_periodic(pos, ty, gidx, b, m.rc_model);
            auto out = nn::evaluate(m, in, prec == 0 ? Precision::fp64 : Precision::fp32);
            (void)out;
        }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(work);
    for (auto& th : pool) th.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// Velocity-Verlet MD loop (proj/src/integrators.cpp:32-47) with the NN force
// provider as ForceFunction; one replica per thread. Positions/velocities are
// updated in place for thread 0's replica (the trajectory the tests compare).
double ref_md_run(void* model, int n, double* xyz, double* vel, const int* types,
                  const double* masses, const double* box, double dt_ps, int prec, int steps,
                  int threads, double* epot_out) {
    const auto& m = *static_cast<nn::NnModel*>(model);
    const std::vector<int> ty(types, types + n);
    const std::vector<double> mass(masses, masses + n);
    std::vector<int> gidx(n);
    for (int i = 0; i < n; ++i) gidx[i] = i;
    const SimBox b(box[0], box[1], box[2]);
    std::vector<double> epots(threads, 0.0);
    std::vector<State> states(threads);
    for (auto& st : states) {
        st.positions = to_vec3(n, xyz);
        st.velocities = to_vec3(n, vel);
        st.forces.assign(n, Vec3{});
        st.box = b;
    }
    auto force_fn_for = [&](int t) {
        return [&, t](State& st) {
            auto in = nn::build_input_periodic(st.positions, ty, gidx, st.box, m.rc_model);
            auto out = nn::evaluate(m, in, prec == 0 ? Precision::fp64 : Precision::fp32);
            st.forces = out.forces;
            epots[t] = out.energy;
            return out.energy;
        };
    };
    // each replica times its own step loop (initial force evaluation excluded);
    // the reported wall time is the slowest replica's
    std::vector<double> walls(threads, 0.0);
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&, t] {
            State& st = states[t];
            auto ff = force_fn_for(t);
            ff(st);  // initial forces
            const auto t0 = std::chrono::steady_clock::now();
            for (int s = 0; s < steps; ++s) velocity_verlet_step(st, ff, dt_ps, mass);
            walls[t] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        });
    for (auto& th : pool) th.join();
    double wall = 0.0;
    for (double w : walls) wall = std::max(wall, w);
    for (int i = 0; i < n; ++i)
        for (int a = 0; a < 3; ++a) {
            xyz[3 * i + a] = states[0].positions[i][a];
            vel[3 * i + a] = states[0].velocities[i][a];
        }
    if (epot_out) *epot_out = epots[0];
    return wall;
}

}  // extern "C"
