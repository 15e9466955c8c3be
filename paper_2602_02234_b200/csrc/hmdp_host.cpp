// hmdp_host.cpp — host-side model I/O, validation and the deterministic fixtures
// (random-init model, synthetic protein-in-water box).  No device code.
//
// The JSON reader is a small self-contained recursive-descent parser for the
// reference's model format (model.cpp:128-197); numbers are parsed with strtod,
// which is correctly rounded, so weights round-trip bit-exactly.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <random>

#include "hmdp_model.h"

namespace hmdp {

// ---------------------------------------------------------------------------
// Minimal JSON value + parser
// ---------------------------------------------------------------------------
namespace {

struct JVal {
    enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
    double num = 0.0;
    bool b = false;
    std::string str;
    std::vector<JVal> arr;
    std::vector<std::pair<std::string, JVal>> obj;

    const JVal* find(const char* key) const {
        for (const auto& kv : obj)
            if (kv.first == key) return &kv.second;
        return nullptr;
    }
    const JVal& at(const char* key) const {
        const JVal* v = find(key);
        if (!v) throw std::invalid_argument(std::string("model JSON missing key '") + key + "'");
        return *v;
    }
    double as_num() const {
        if (kind != Num) throw std::invalid_argument("model JSON: expected a number");
        return num;
    }
    int as_int() const {
        const double v = as_num();
        if (v != std::floor(v) || std::fabs(v) > 2147483647.0)
            throw std::invalid_argument("model JSON: expected an integer");
        return static_cast<int>(v);
    }
    std::vector<double> as_vec() const {
        if (kind != Arr) throw std::invalid_argument("model JSON: expected an array");
        std::vector<double> out;
        out.reserve(arr.size());
        for (const auto& e : arr) out.push_back(e.as_num());
        return out;
    }
};

class Parser {
   public:
    explicit Parser(const std::string& s) : s_(s) {}
    JVal parse() {
        JVal v = value();
        ws();
        if (p_ != s_.size()) fail("trailing characters");
        return v;
    }

   private:
    const std::string& s_;
    std::size_t p_ = 0;

    [[noreturn]] void fail(const char* what) {
        throw std::invalid_argument(std::string("model JSON parse error: ") + what +
                                    " at byte " + std::to_string(p_));
    }
    void ws() {
        while (p_ < s_.size() && (s_[p_] == ' ' || s_[p_] == '\n' || s_[p_] == '\r' ||
                                  s_[p_] == '\t'))
            ++p_;
    }
    bool lit(const char* w) {
        const std::size_t n = std::strlen(w);
        if (s_.compare(p_, n, w) == 0) {
            p_ += n;
            return true;
        }
        return false;
    }
    JVal value() {
        ws();
        if (p_ >= s_.size()) fail("unexpected end of input");
        const char c = s_[p_];
        JVal v;
        if (c == '{') {
            v.kind = JVal::Obj;
            ++p_;
            ws();
            if (p_ < s_.size() && s_[p_] == '}') {
                ++p_;
                return v;
            }
            for (;;) {
                ws();
                if (p_ >= s_.size() || s_[p_] != '"') fail("expected object key");
                std::string key = string();
                ws();
                if (p_ >= s_.size() || s_[p_] != ':') fail("expected ':'");
                ++p_;
                v.obj.emplace_back(std::move(key), value());
                ws();
                if (p_ < s_.size() && s_[p_] == ',') {
                    ++p_;
                    continue;
                }
                if (p_ < s_.size() && s_[p_] == '}') {
                    ++p_;
                    return v;
                }
                fail("expected ',' or '}'");
            }
        }
        if (c == '[') {
            v.kind = JVal::Arr;
            ++p_;
            ws();
            if (p_ < s_.size() && s_[p_] == ']') {
                ++p_;
                return v;
            }
            for (;;) {
                v.arr.push_back(value());
                ws();
                if (p_ < s_.size() && s_[p_] == ',') {
                    ++p_;
                    continue;
                }
                if (p_ < s_.size() && s_[p_] == ']') {
                    ++p_;
                    return v;
                }
                fail("expected ',' or ']'");
            }
        }
        if (c == '"') {
            v.kind = JVal::Str;
            v.str = string();
            return v;
        }
        if (lit("true")) {
            v.kind = JVal::Bool;
            v.b = true;
            return v;
        }
        if (lit("false")) {
            v.kind = JVal::Bool;
            return v;
        }
        if (lit("null")) return v;
        if (c == '-' || (c >= '0' && c <= '9')) {
            const char* begin = s_.c_str() + p_;
            char* end = nullptr;
            v.kind = JVal::Num;
            v.num = std::strtod(begin, &end);
            if (end == begin) fail("bad number");
            p_ += static_cast<std::size_t>(end - begin);
            return v;
        }
        fail("unexpected character");
    }
    std::string string() {
        ++p_;  // opening quote
        std::string out;
        while (p_ < s_.size() && s_[p_] != '"') {
            char c = s_[p_++];
            if (c == '\\') {
                if (p_ >= s_.size()) fail("bad escape");
                const char e = s_[p_++];
                switch (e) {
                    case 'n': out += '\n'; break;
                    case 't': out += '\t'; break;
                    case 'r': out += '\r'; break;
                    case 'b': out += '\b'; break;
                    case 'f': out += '\f'; break;
                    case 'u': {
                        if (p_ + 4 > s_.size()) fail("bad \\u escape");
                        const unsigned cp = std::strtoul(s_.substr(p_, 4).c_str(), nullptr, 16);
                        p_ += 4;
                        if (cp < 0x80) out += static_cast<char>(cp);
                        else if (cp < 0x800) {
                            out += static_cast<char>(0xC0 | (cp >> 6));
                            out += static_cast<char>(0x80 | (cp & 0x3F));
                        } else {
                            out += static_cast<char>(0xE0 | (cp >> 12));
                            out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
                            out += static_cast<char>(0x80 | (cp & 0x3F));
                        }
                        break;
                    }
                    default: out += e;
                }
            } else {
                out += c;
            }
        }
        if (p_ >= s_.size()) fail("unterminated string");
        ++p_;
        return out;
    }
};

Mlp mlp_from(const JVal& j) {  // model.cpp:134-145
    Mlp m;
    for (double v : j.at("sizes").as_vec()) {
        if (v != std::floor(v) || v < 1 || v > 1e6)
            throw std::invalid_argument("MLP sizes must be positive integers");
        m.sizes.push_back(static_cast<int>(v));
    }
    const JVal& w = j.at("weights");
    const JVal& b = j.at("biases");
    if (w.kind != JVal::Arr || b.kind != JVal::Arr)
        throw std::invalid_argument("MLP weights/biases must be arrays");
    if (m.sizes.size() < 2 || w.arr.size() != m.sizes.size() - 1 ||
        b.arr.size() != m.sizes.size() - 1)
        throw std::invalid_argument("MLP layer count mismatch");
    for (int l = 0; l < m.n_layers(); ++l) {
        m.weights.push_back(w.arr[l].as_vec());
        m.biases.push_back(b.arr[l].as_vec());
        if (m.weights[l].size() != static_cast<std::size_t>(m.sizes[l]) * m.sizes[l + 1] ||
            m.biases[l].size() != static_cast<std::size_t>(m.sizes[l + 1]))
            throw std::invalid_argument("MLP weight shape mismatch");
    }
    return m;
}

void put_num(std::string& o, double v) {
    char buf[40];
    if (v == std::floor(v) && std::fabs(v) < 1e15) {
        std::snprintf(buf, sizeof buf, "%.1f", v);
    } else {
        std::snprintf(buf, sizeof buf, "%.17g", v);
    }
    o += buf;
}
void put_vec(std::string& o, const std::vector<double>& v) {
    o += '[';
    for (std::size_t k = 0; k < v.size(); ++k) {
        if (k) o += ',';
        put_num(o, v[k]);
    }
    o += ']';
}
void put_mlp(std::string& o, const Mlp& m) {
    o += "{\"sizes\":[";
    for (std::size_t k = 0; k < m.sizes.size(); ++k) {
        if (k) o += ',';
        o += std::to_string(m.sizes[k]);
    }
    o += "],\"weights\":[";
    for (std::size_t l = 0; l < m.weights.size(); ++l) {
        if (l) o += ',';
        put_vec(o, m.weights[l]);
    }
    o += "],\"biases\":[";
    for (std::size_t l = 0; l < m.biases.size(); ++l) {
        if (l) o += ',';
        put_vec(o, m.biases[l]);
    }
    o += "]}";
}

// Rng, include/halomd/rng.hpp:11-44: mt19937_64 with hand-rolled distributions.
struct Rng {
    std::mt19937_64 gen;
    bool have_spare = false;
    double spare = 0.0;
    explicit Rng(std::uint64_t seed) : gen(seed) {}
    double uniform() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    double gaussian() {
        if (have_spare) {
            have_spare = false;
            return spare;
        }
        double u1 = 0.0;
        do {
            u1 = uniform();
        } while (u1 <= 0.0);
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 2.0 * M_PI * u2;
        spare = r * std::sin(a);
        have_spare = true;
        return r * std::cos(a);
    }
};

Mlp random_mlp(const std::vector<int>& sizes, Rng& rng) {  // model.cpp:52-66
    Mlp m;
    m.sizes = sizes;
    for (std::size_t l = 0; l + 1 < sizes.size(); ++l) {
        const int in = sizes[l], out = sizes[l + 1];
        const double scale = 1.0 / std::sqrt(static_cast<double>(in));
        std::vector<double> w(static_cast<std::size_t>(in) * out);
        for (auto& v : w) v = rng.uniform(-scale, scale);
        std::vector<double> b(out);
        for (auto& v : b) v = rng.uniform(-0.1, 0.1);
        m.weights.push_back(std::move(w));
        m.biases.push_back(std::move(b));
    }
    return m;
}

}  // namespace

// ---------------------------------------------------------------------------
std::uint64_t Mlp::forward_flops() const {
    std::uint64_t f = 0;
    for (int l = 0; l < n_layers(); ++l) f += 2ull * sizes[l] * sizes[l + 1] + 4ull * sizes[l + 1];
    return f;
}
int Mlp::act_size() const {
    int s = 0;
    for (int v : sizes) s += v;
    return s;
}

namespace {
void validate_dp(const Model& m) {
    // DeePMD-style families (no reference function).
    auto shape = [](const Mlp& p, std::vector<int> want, const char* name) {
        if (p.sizes != want)
            throw std::invalid_argument(std::string("unsupported ") + name +
                                        " MLP shape for this model family");
    };
    if (m.rc <= 0.0) throw std::invalid_argument("rc_model must be positive");
    if (!(m.rcs >= 0.0 && m.rcs < m.rc))
        throw std::invalid_argument("rc_smooth must satisfy 0 <= rc_smooth < rc_model");
    if (m.n_types < 1) throw std::invalid_argument("n_types must be >= 1");
    if (m.n_types > kMaxTypes) throw std::invalid_argument("unsupported n_types (kernels take <= 4)");
    if (m.hidden != kH) throw std::invalid_argument("unsupported hidden width (kernels take H=32)");
    if (m.axis != kAxis) throw std::invalid_argument("unsupported axis neurons (kernels take 4)");
    if (!(m.nnorm > 0.0)) throw std::invalid_argument("nnorm must be positive");
    if (static_cast<int>(m.embeds.size()) != m.n_types)
        throw std::invalid_argument("one embedding net per neighbour type required");
    for (const Mlp& e : m.embeds) shape(e, {1, kH, kH}, "embedding");
    if (static_cast<int>(m.ebias.size()) != m.n_types)
        throw std::invalid_argument("energy_bias must have n_types entries");
    const int nd = m.axis * kH;
    if (m.family == kSeA) {
        shape(m.fitting, {nd, kH, 1}, "fitting");
        if (!m.rf.empty()) throw std::invalid_argument("se_a model cannot carry repformer layers");
        return;
    }
    if (m.rf.empty()) throw std::invalid_argument("repformer needs depth >= 2 (one layer or more)");
    shape(m.g1map, {nd, kH, kH}, "g1map");
    shape(m.fitting, {kH, kH, 1}, "fitting");
    if (static_cast<int>(m.rf.size()) > kMaxMsg)
        throw std::invalid_argument("unsupported depth (kernels take <= 9)");
    if (m.family == kRepflow) {
        if (!(m.rcas >= 0.0 && m.rcas < m.rca && m.rca <= m.rc))
            throw std::invalid_argument("repflow needs 0 <= rc_angle_smooth < rc_angle <= rc_model");
        if (!(m.anorm > 0.0)) throw std::invalid_argument("anorm must be positive");
    }
    for (const RfLayer& l : m.rf) {
        if (m.family == kRepflow) {
            shape(l.angle, {1, kH}, "angle");
            for (const Mlp* p : {&l.v, &l.o, &l.c}) shape(*p, {kH, kH}, "edge");
        } else {
            for (const Mlp* p : {&l.q, &l.k, &l.v, &l.o, &l.c}) shape(*p, {kH, kH}, "attention");
        }
        shape(l.update, {kH + nd, kH, kH}, "update");
    }
}
}  // namespace

void Model::validate() const {
    if (is_dp()) return validate_dp(*this);
    // NnModel::validate, model.cpp:30-48 (same messages).
    if (rc <= 0.0) throw std::invalid_argument("rc_model must be positive");
    if (n_types < 1) throw std::invalid_argument("n_types must be >= 1");
    if (n_basis() < 1) throw std::invalid_argument("radial basis must not be empty");
    if (embedding.sizes.front() != descriptor_dim())
        throw std::invalid_argument("embedding input dim != descriptor dim");
    if (embedding.sizes.back() != hidden || fitting.sizes.front() != hidden)
        throw std::invalid_argument("embedding/fitting width mismatch");
    if (fitting.sizes.back() != 1) throw std::invalid_argument("fitting net must output 1 value");
    if (family == 0 && !message.empty())
        throw std::invalid_argument("embed_fit model cannot carry message layers");
    for (std::size_t l = 0; l < message.size(); ++l) {
        if (message[l].sizes.front() != hidden + n_basis() || message[l].sizes.back() != hidden)
            throw std::invalid_argument("message MLP dims mismatch");
        if (update[l].sizes.front() != 2 * hidden || update[l].sizes.back() != hidden)
            throw std::invalid_argument("update MLP dims mismatch");
    }
    // Device-kernel limits (documented divergence: the reference is shape-generic).
    auto two_layer = [&](const Mlp& m, const char* name) {
        if (m.n_layers() != 2 || m.sizes[1] != kH)
            throw std::invalid_argument(std::string("unsupported ") + name +
                                        " MLP shape: the B200 kernels take [in, 32, out]");
    };
    if (hidden != kH) throw std::invalid_argument("unsupported hidden width (kernels take H=32)");
    if (n_basis() != kK) throw std::invalid_argument("unsupported n_basis (kernels take K=8)");
    if (n_types > kMaxTypes) throw std::invalid_argument("unsupported n_types (kernels take <= 4)");
    if (static_cast<int>(message.size()) > kMaxMsg)
        throw std::invalid_argument("unsupported depth (kernels take <= 9)");
    if (width <= 0.0) throw std::invalid_argument("radial basis width must be positive");
    two_layer(embedding, "embedding");
    two_layer(fitting, "fitting");
    for (std::size_t l = 0; l < message.size(); ++l) {
        two_layer(message[l], "message");
        two_layer(update[l], "update");
    }
}

void Model::counters(int n, int n_owned, long long ne, int real_bytes,
                     std::uint64_t out[2]) const {
    if (is_dp()) {
        // Algorithmic count in the reference's convention (forward + 2x forward
        // for the reverse pass, inference.cpp:389-402), written out for the
        // DeePMD-style operators: env matrix, embedding, R^T G, G^T R R^T G,
        // fitting; repformer: q/k/v/o projections, attention over the n_e^2
        // neighbour pairs of each atom (n_e = ne / n), conv, grrg, update.
        const double H = kH, nd = axis * kH;
        const double m2 = n > 0 ? static_cast<double>(ne) * ne / n : 0.0;
        double fl = 0.0, act = 0.0;
        fl += ne * (30.0 + 3.0 * embeds[0].forward_flops() + 3.0 * 2 * 4 * H);
        fl += n * 3.0 * (2.0 * axis * 4 * H);
        fl += n_owned * 3.0 * fitting.forward_flops();
        act += static_cast<double>(ne) * (8 + 2 * H) + n * (nd + fitting.act_size());
        if (family >= kRepformer) {
            fl += n * 3.0 * g1map.forward_flops();
            for (const RfLayer& l : rf) {
                fl += ne * 3.0 * (4.0 * l.q.forward_flops() + 6 * H);
                fl += m2 * 3.0 * (4.0 * H + 12);
                fl += n * 3.0 * (l.c.forward_flops() + 2.0 * 3 * axis * H + l.update.forward_flops());
                act += static_cast<double>(ne) * 5 * H + m2 + n * (nd + 2 * H + l.update.act_size());
            }
        }
        out[0] = static_cast<std::uint64_t>(fl);
        out[1] = static_cast<std::uint64_t>(act) * static_cast<std::uint64_t>(real_bytes);
        return;
    }
    // inference.cpp:389-414
    const std::uint64_t K = n_basis(), H = hidden;
    std::uint64_t fl = 0, act = 0;
    fl += static_cast<std::uint64_t>(ne) * (20 + 10 * K);
    fl += static_cast<std::uint64_t>(n) * 3 * embedding.forward_flops();
    fl += static_cast<std::uint64_t>(n_owned) * 3 * fitting.forward_flops();
    for (std::size_t l = 0; l < message.size(); ++l) {
        fl += static_cast<std::uint64_t>(ne) * (3 * message[l].forward_flops() + 6 * H + 3 * K);
        fl += static_cast<std::uint64_t>(n) * (3 * update[l].forward_flops() + 2 * H);
    }
    act += static_cast<std::uint64_t>(n) *
           (descriptor_dim() + embedding.act_size() + fitting.act_size());
    act += static_cast<std::uint64_t>(n) * (message.size() + 1) * H;
    for (std::size_t l = 0; l < message.size(); ++l) {
        act += static_cast<std::uint64_t>(ne) * message[l].act_size();
        act += static_cast<std::uint64_t>(n) * (update[l].act_size() + H);
    }
    act += static_cast<std::uint64_t>(ne) * (2 + K);
    out[0] = fl;
    out[1] = act * static_cast<std::uint64_t>(real_bytes);
}

Model model_from_json(const std::string& text) {
    const JVal j = Parser(text).parse();
    if (j.kind != JVal::Obj) throw std::invalid_argument("not a halomd model file");
    const JVal* fmt = j.find("format");
    if (!fmt || fmt->kind != JVal::Str || fmt->str != "halomd-model")
        throw std::invalid_argument("not a halomd model file");
    const JVal* ver = j.find("version");
    const int version = (ver && ver->kind == JVal::Num) ? ver->as_int() : 0;
    if (version != 1)
        throw std::invalid_argument("unsupported model version " + std::to_string(version));
    Model m;
    const JVal& fam = j.at("family");
    if (fam.kind == JVal::Str && fam.str == "embed_fit")
        m.family = kEmbedFit;
    else if (fam.kind == JVal::Str && fam.str == "message_passing")
        m.family = kMessagePassing;
    else if (fam.kind == JVal::Str && fam.str == "se_a")
        m.family = kSeA;
    else if (fam.kind == JVal::Str && fam.str == "repformer")
        m.family = kRepformer;
    else if (fam.kind == JVal::Str && fam.str == "repflow")
        m.family = kRepflow;
    else
        throw std::invalid_argument("unknown model family '" + fam.str + "'");
    if (m.is_dp()) {
        m.rc = j.at("rc_model").as_num();
        m.rcs = j.at("rc_smooth").as_num();
        m.n_types = j.at("n_types").as_int();
        m.hidden = j.at("hidden").as_int();
        m.axis = j.at("axis").as_int();
        m.nnorm = j.at("nnorm").as_num();
        if (const JVal* s = j.find("seed"); s && s->kind == JVal::Num)
            m.seed = static_cast<std::uint64_t>(s->num);
        const JVal& em = j.at("embeddings");
        if (em.kind != JVal::Arr) throw std::invalid_argument("model JSON: embeddings must be an array");
        for (const auto& e : em.arr) m.embeds.push_back(mlp_from(e));
        m.ebias = j.at("energy_bias").as_vec();
        m.fitting = mlp_from(j.at("fitting"));
        if (m.family == kRepflow) {
            m.rca = j.at("rc_angle").as_num();
            m.rcas = j.at("rc_angle_smooth").as_num();
            m.anorm = j.at("anorm").as_num();
        }
        if (m.family >= kRepformer) {
            m.g1map = mlp_from(j.at("g1map"));
            const JVal& layers = j.at("layers");
            if (layers.kind != JVal::Arr)
                throw std::invalid_argument("model JSON: layers must be an array");
            for (const auto& jl : layers.arr) {
                RfLayer l;
                if (m.family == kRepflow) {
                    l.angle = mlp_from(jl.at("angle"));
                } else {
                    l.q = mlp_from(jl.at("q"));
                    l.k = mlp_from(jl.at("k"));
                }
                l.v = mlp_from(jl.at("v"));
                l.o = mlp_from(jl.at("o"));
                l.c = mlp_from(jl.at("c"));
                l.update = mlp_from(jl.at("update"));
                m.rf.push_back(std::move(l));
            }
        }
        m.validate();
        return m;
    }
    m.rc = j.at("rc_model").as_num();
    m.n_types = j.at("n_types").as_int();
    m.hidden = j.at("hidden").as_int();
    if (const JVal* s = j.find("seed"); s && s->kind == JVal::Num)
        m.seed = static_cast<std::uint64_t>(s->num);
    m.centers = j.at("basis").at("centers").as_vec();
    m.width = j.at("basis").at("width").as_num();
    m.embedding = mlp_from(j.at("embedding"));
    m.fitting = mlp_from(j.at("fitting"));
    const JVal& layers = j.at("layers");
    if (layers.kind != JVal::Arr) throw std::invalid_argument("model JSON: layers must be an array");
    for (const auto& jl : layers.arr) {
        m.message.push_back(mlp_from(jl.at("message")));
        m.update.push_back(mlp_from(jl.at("update")));
    }
    m.validate();
    return m;
}

namespace {
std::string dp_to_json(const Model& m) {
    std::string o;
    o.reserve(400000);
    o += "{\"format\":\"halomd-model\",\"version\":1,\"family\":\"";
    o += m.family == kSeA ? "se_a" : (m.family == kRepformer ? "repformer" : "repflow");
    o += "\",\"rc_model\":";
    put_num(o, m.rc);
    o += ",\"rc_smooth\":";
    put_num(o, m.rcs);
    o += ",\"n_types\":" + std::to_string(m.n_types);
    o += ",\"hidden\":" + std::to_string(m.hidden);
    o += ",\"axis\":" + std::to_string(m.axis);
    o += ",\"nnorm\":";
    put_num(o, m.nnorm);
    o += ",\"seed\":" + std::to_string(m.seed);
    o += ",\"embeddings\":[";
    for (std::size_t t = 0; t < m.embeds.size(); ++t) {
        if (t) o += ',';
        put_mlp(o, m.embeds[t]);
    }
    o += "],\"energy_bias\":";
    put_vec(o, m.ebias);
    o += ",\"fitting\":";
    put_mlp(o, m.fitting);
    if (m.family == kRepflow) {
        o += ",\"rc_angle\":";
        put_num(o, m.rca);
        o += ",\"rc_angle_smooth\":";
        put_num(o, m.rcas);
        o += ",\"anorm\":";
        put_num(o, m.anorm);
    }
    if (m.family >= kRepformer) {
        o += ",\"g1map\":";
        put_mlp(o, m.g1map);
        o += ",\"layers\":[";
        for (std::size_t l = 0; l < m.rf.size(); ++l) {
            if (l) o += ',';
            const RfLayer& L = m.rf[l];
            const bool flow = m.family == kRepflow;
            const std::pair<const char*, const Mlp*> parts[] = {
                {flow ? "angle" : "q", flow ? &L.angle : &L.q}, {"k", &L.k}, {"v", &L.v},
                {"o", &L.o}, {"c", &L.c}, {"update", &L.update}};
            o += '{';
            bool first = true;
            for (int p = 0; p < 6; ++p) {
                if (flow && p == 1) continue;
                if (!first) o += ',';
                first = false;
                o += std::string("\"") + parts[p].first + "\":";
                put_mlp(o, *parts[p].second);
            }
            o += '}';
        }
        o += ']';
    }
    o += '}';
    return o;
}
}  // namespace

std::string model_to_json(const Model& m) {
    if (m.is_dp()) return dp_to_json(m);
    std::string o;
    o.reserve(400000);
    o += "{\"format\":\"halomd-model\",\"version\":1,\"family\":\"";
    o += m.family == 0 ? "embed_fit" : "message_passing";
    o += "\",\"rc_model\":";
    put_num(o, m.rc);
    o += ",\"n_types\":" + std::to_string(m.n_types);
    o += ",\"hidden\":" + std::to_string(m.hidden);
    o += ",\"seed\":" + std::to_string(m.seed);
    o += ",\"basis\":{\"centers\":";
    put_vec(o, m.centers);
    o += ",\"width\":";
    put_num(o, m.width);
    o += "},\"embedding\":";
    put_mlp(o, m.embedding);
    o += ",\"fitting\":";
    put_mlp(o, m.fitting);
    o += ",\"layers\":[";
    for (std::size_t l = 0; l < m.message.size(); ++l) {
        if (l) o += ',';
        o += "{\"message\":";
        put_mlp(o, m.message[l]);
        o += ",\"update\":";
        put_mlp(o, m.update[l]);
        o += '}';
    }
    o += "]}";
    return o;
}

Model make_model(int family, int depth, double rc, int n_types, int n_basis, int hidden,
                 std::uint64_t seed) {
    // model.cpp:70-100
    if (depth < 1) throw std::invalid_argument("depth must be >= 1");
    if (family == 0 && depth != 1)
        throw std::invalid_argument("embed_fit has depth 1 by construction");
    Model m;
    m.family = family;
    m.rc = rc;
    m.n_types = n_types;
    m.hidden = hidden;
    m.seed = seed;
    m.centers.resize(n_basis);
    for (int k = 0; k < n_basis; ++k) m.centers[k] = n_basis > 1 ? rc * k / (n_basis - 1) : 0.0;
    m.width = n_basis > 1 ? rc / (n_basis - 1) : rc;
    Rng rng(seed);
    const int nd = n_types * n_basis;
    m.embedding = random_mlp({nd, hidden, hidden}, rng);
    m.fitting = random_mlp({hidden, hidden, 1}, rng);
    for (int l = 1; l < depth; ++l) {
        m.message.push_back(random_mlp({hidden + n_basis, hidden, hidden}, rng));
        m.update.push_back(random_mlp({2 * hidden, hidden, hidden}, rng));
    }
    m.validate();
    return m;
}

Model make_dp_model(int family, int depth, double rc, double rcs, int n_types, int axis,
                    std::uint64_t seed) {
    if (family != kSeA && family != kRepformer && family != kRepflow)
        throw std::invalid_argument("make_dp_model: family must be se_a, repformer or repflow");
    if (depth < 1) throw std::invalid_argument("depth must be >= 1");
    if (family == kSeA && depth != 1) throw std::invalid_argument("se_a has depth 1 by construction");
    Model m;
    m.family = family;
    m.rc = rc;
    m.rcs = rcs;
    m.n_types = n_types;
    m.hidden = kH;
    m.axis = axis;
    m.nnorm = 32.0;
    m.seed = seed;
    Rng rng(seed);
    for (int t = 0; t < n_types; ++t) m.embeds.push_back(random_mlp({1, kH, kH}, rng));
    const int nd = axis * kH;
    m.fitting = random_mlp({family == kSeA ? nd : kH, kH, 1}, rng);
    for (int t = 0; t < n_types; ++t) m.ebias.push_back(rng.uniform(-1.0, 1.0));
    if (family >= kRepformer) {
        m.g1map = random_mlp({nd, kH, kH}, rng);
        for (int l = 1; l < depth; ++l) {
            RfLayer L;
            if (family == kRepflow) {
                L.angle = random_mlp({1, kH}, rng);
            } else {
                L.q = random_mlp({kH, kH}, rng);
                L.k = random_mlp({kH, kH}, rng);
            }
            L.v = random_mlp({kH, kH}, rng);
            L.o = random_mlp({kH, kH}, rng);
            L.c = random_mlp({kH, kH}, rng);
            L.update = random_mlp({kH + nd, kH, kH}, rng);
            m.rf.push_back(std::move(L));
        }
    }
    m.validate();
    return m;
}

SyntheticSystem synthetic_system(int n, double density, double fraction, std::uint64_t seed,
                                 double temperature) {
    // generate_synthetic_system, synthetic.cpp:36-130 (the NN-relevant outputs:
    // positions, types, masses, velocities, box; charges/bonded terms are not
    // on this path).
    if (n < 2) throw std::invalid_argument("n_atoms must be >= 2");
    if (density <= 0.0) throw std::invalid_argument("density must be positive");
    if (fraction < 0.0 || fraction > 1.0)
        throw std::invalid_argument("fraction_grouped must be in [0, 1]");
    SyntheticSystem s;
    const double box_len = std::cbrt(n / density);
    const int m = static_cast<int>(std::ceil(std::cbrt(static_cast<double>(n))));
    const double spacing = box_len / m;
    const double sigma_max = 0.33;  // max(sigma_protein 0.33, sigma_solvent 0.30)
    if (spacing < 0.8 * sigma_max)
        throw std::runtime_error("density too high: lattice spacing " + std::to_string(spacing) +
                                 " nm < 0.8 sigma");
    const int n_group = static_cast<int>(std::ceil(fraction * n));
    s.box[0] = s.box[1] = s.box[2] = box_len;
    s.xyz.resize(3 * static_cast<std::size_t>(n));
    s.vel.assign(3 * static_cast<std::size_t>(n), 0.0);
    s.types.resize(n);
    s.masses.resize(n);
    // snake_sites, synthetic.cpp:14-31
    std::vector<int> site(3 * static_cast<std::size_t>(n));
    {
        int cnt = 0;
        for (int z = 0; z < m && cnt < n; ++z) {
            const bool flip_y = (z % 2) != 0;
            for (int yy = 0; yy < m && cnt < n; ++yy) {
                const int y = flip_y ? m - 1 - yy : yy;
                const bool flip_x = (yy % 2) != 0;
                for (int xx = 0; xx < m && cnt < n; ++xx) {
                    const int x = flip_x ? m - 1 - xx : xx;
                    site[3 * cnt] = x;
                    site[3 * cnt + 1] = y;
                    site[3 * cnt + 2] = z;
                    ++cnt;
                }
            }
        }
    }
    Rng rng(seed);
    for (int i = 0; i < n; ++i) {
        const bool grouped = i < n_group;
        s.types[i] = grouped ? 0 : 1;
        s.masses[i] = grouped ? 12.0 : 18.0;
        const double jitter = (grouped ? 0.05 : 0.10) * spacing;
        for (int a = 0; a < 3; ++a) {
            double r = (site[3 * i + a] + 0.5) * spacing + rng.uniform(-jitter, jitter);
            // wrap_position, box.hpp:34-42
            r -= box_len * std::floor(r / box_len);
            if (r >= box_len) r = 0.0;
            s.xyz[3 * i + a] = r;
        }
    }
    if (temperature > 0.0) {
        constexpr double kB = 0.008314462618;  // units.hpp:10
        for (int i = 0; i < n; ++i) {
            const double sd = std::sqrt(kB * temperature / s.masses[i]);
            for (int a = 0; a < 3; ++a) s.vel[3 * i + a] = sd * rng.gaussian();
        }
        double mom[3] = {0, 0, 0}, total_mass = 0.0;
        for (int i = 0; i < n; ++i) {
            for (int a = 0; a < 3; ++a) mom[a] += s.vel[3 * i + a] * s.masses[i];
            total_mass += s.masses[i];
        }
        double vcom[3];
        for (int a = 0; a < 3; ++a) vcom[a] = mom[a] / total_mass;
        for (int i = 0; i < n; ++i)
            for (int a = 0; a < 3; ++a) s.vel[3 * i + a] -= vcom[a];
        // kinetic_energy_and_temperature, state.cpp:9-19
        double ke = 0.0;
        for (int i = 0; i < n; ++i) {
            const double* v = &s.vel[3 * i];
            ke += 0.5 * s.masses[i] * (v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
        }
        const int ndf = 3 * n - 3;
        const double t_now = 2.0 * ke / (ndf * kB);
        if (t_now > 0.0) {
            const double lambda = std::sqrt(temperature / t_now);
            for (auto& v : s.vel) v *= lambda;
        }
    }
    return s;
}

}  // namespace hmdp
