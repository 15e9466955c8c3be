// hmdp_model.h — host-side model representation for the B200 DP force path.
//
// Mirrors halomd::nn::NnModel (include/halomd/nn/model.hpp:40-56): family,
// rc_model, n_types, hidden width H, seed, radial basis (centres, width),
// embedding / fitting MLPs and (for message_passing) depth-1 message layers,
// each an MLP with tanh hidden layers and a linear output, weights row-major
// [out][in] (model.hpp:12-22).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace hmdp {

constexpr int kH = 32;  // hidden width of every device MLP (lane = channel)

struct Mlp {
    std::vector<int> sizes;                   // [in, hidden..., out]
    std::vector<std::vector<double>> weights; // per layer, [out][in]
    std::vector<std::vector<double>> biases;  // per layer, [out]
    int n_layers() const { return static_cast<int>(sizes.size()) - 1; }
    std::uint64_t forward_flops() const;      // inference.cpp:140-145
    int act_size() const;                     // Σ sizes (inference.cpp:78-82)
};

// One repformer layer of the DeePMD-style "repformer" family:
// attention projections q, k, v, o and the neighbour projection c are single
// linear layers [32, 32] (Mlp with one layer); update is [32 + axis*32, 32, 32].
// repflow layers carry `angle` [1, 32] (the elementwise angle embedding) instead
// of q and k.
struct RfLayer {
    Mlp q, k, v, o, c, update, angle;
};

// Model families: the reference's two (model.hpp:9) plus the DeePMD-style
// families of the north star that have no reference function (SURVEY §8(a')).
enum Family : int { kEmbedFit = 0, kMessagePassing = 1, kSeA = 2, kRepformer = 3, kRepflow = 4 };

struct Model {
    int family = 0;  // Family
    double rc = 0.6;
    int n_types = 2;
    int hidden = 32;
    std::uint64_t seed = 0;
    std::vector<double> centers;
    double width = 0.1;
    Mlp embedding, fitting;
    std::vector<Mlp> message, update;
    // DeePMD-style families (kSeA, kRepformer): smooth env matrix with switch
    // onset rcs, per-neighbour-type embedding nets [1, 32, 32], axis neurons,
    // descriptor normaliser nnorm, per-type energy bias, repformer layers.
    double rcs = 0.0;
    int axis = 4;
    double nnorm = 32.0;
    std::vector<Mlp> embeds;
    std::vector<double> ebias;
    Mlp g1map;
    std::vector<RfLayer> rf;
    // repflow: angle neighbours r < rca, switch onset rcas, angle normaliser anorm
    double rca = 0.4, rcas = 0.2, anorm = 8.0;

    bool is_dp() const { return family >= kSeA; }
    int n_basis() const { return static_cast<int>(centers.size()); }
    int depth() const {
        return 1 + static_cast<int>(is_dp() ? rf.size() : message.size());
    }
    double receptive_radius() const { return depth() * rc; }
    int descriptor_dim() const { return is_dp() ? axis * kH : n_types * n_basis(); }
    // NnModel::validate (model.cpp:30-48) plus the shape limits of the device
    // kernels (two-layer MLPs, H = 32, n_basis = 8, n_types <= 4).
    void validate() const;
    // Analytic NnCounters (inference.cpp:389-414).
    void counters(int n, int n_owned, long long ne, int real_bytes, std::uint64_t out[2]) const;
};

Model model_from_json(const std::string& text);  // model.cpp:165-197
std::string model_to_json(const Model& m);        // model.cpp:147-163
Model make_model(int family, int depth, double rc, int n_types, int n_basis, int hidden,
                 std::uint64_t seed);             // model.cpp:70-100
// Random-init DeePMD-style model (kSeA: depth 1; kRepformer: depth - 1 layers),
// same Rng and MLP init as make_model (model.cpp:52-66).
Model make_dp_model(int family, int depth, double rc, double rcs, int n_types, int axis,
                    std::uint64_t seed);

struct SyntheticSystem {
    std::vector<double> xyz, vel, masses;
    std::vector<int> types;
    double box[3];
};
SyntheticSystem synthetic_system(int n, double density, double fraction, std::uint64_t seed,
                                 double temperature);  // synthetic.cpp:36-130

// Kernel shape limits.
constexpr int kAxis = 4;
constexpr int kK = 8;
constexpr int kMaxTypes = 4;
constexpr int kMaxMsg = 8;

}  // namespace hmdp
