// Model<R> (nn.hpp:68-222), layers (nn.hpp:344-453), SENSE fragments
// (recon.hpp:345-451) and the MoDL / VarNet constructors (recon.hpp:499-904),
// built over the device Nlop engine with fused B200 nodes in place of the
// reference's TenMul/FFT fragment chains.
#pragma once

#include "nodes.h"

#include <cmath>
#include <functional>
#include <map>

namespace mdnn {

// ---- deterministic RNG, restated from common.hpp:86-147 (bitwise) ---------------
inline uint64_t splitmix64(uint64_t& state)
{
    uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
inline uint64_t hash_rand(uint64_t key, uint64_t counter)
{
    uint64_t s = key ^ (0x9e3779b97f4a7c15ULL + counter * 0xbf58476d1ce4e5b9ULL);
    splitmix64(s);
    return splitmix64(s);
}
class Rng {
public:
    explicit Rng(uint64_t seed) : state_(seed ^ 0x5851f42d4c957f2dULL) { splitmix64(state_); }
    uint64_t next() { return splitmix64(state_); }
    double uniform() { return double(next() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    double gauss()
    {
        if (have_spare_) {
            have_spare_ = false;
            return spare_;
        }
        double u1 = 0.0;
        while (u1 == 0.0)
            u1 = uniform();
        double u2 = uniform();
        double r = std::sqrt(-2.0 * std::log(u1));
        spare_ = r * std::sin(2.0 * M_PI * u2);
        have_spare_ = true;
        return r * std::cos(2.0 * M_PI * u2);
    }
    uint64_t below(uint64_t n) { return next() % n; }

private:
    uint64_t state_;
    double spare_ = 0.0;
    bool have_spare_ = false;
};
inline uint64_t derive_seed(uint64_t seed, const std::string& label)
{
    uint64_t h = 0xcbf29ce484222325ULL;
    for (unsigned char c : label)
        h = (h ^ c) * 0x100000001b3ULL;
    return hash_rand(seed, h);
}

enum class ArgKind { Data = 0, Weights = 1, MovingStats = 2 };

struct Initializer {
    enum Kind { None, Constant, GlorotUniform } kind = None;
    double value = 0;
    long fan_in = 0, fan_out = 0;
    static Initializer constant(double v)
    {
        Initializer i;
        i.kind = Constant;
        i.value = v;
        return i;
    }
    static Initializer glorot(long fi, long fo)
    {
        Initializer i;
        i.kind = GlorotUniform;
        i.fan_in = fi;
        i.fan_out = fo;
        return i;
    }
};

enum class ProxKind { None = 0, NonNeg = 1 };

struct Arg {
    std::string name;
    ArgKind kind = ArgKind::Data;
    Initializer init;
    ProxKind prox = ProxKind::None;
    bool real_weights = false;
};

inline Arg data_arg(const std::string& n) { return Arg{n, ArgKind::Data, {}, ProxKind::None, false}; }

struct Model {
    Nlop op;
    std::vector<Arg> args;
    std::vector<std::string> out_names;
    std::function<Model(long)> rebatch;

    bool valid() const { return op.valid(); }
    int arg_index(const std::string& name) const;
    int output_index(const std::string& name) const;
    long num_real_params() const;
    // host values (interleaved complex) of one weights / moving-stats arg
    std::vector<std::complex<float>> init_weight(uint64_t seed, int i) const;
};

Model model_chain(const Model& a, const Model& b, const std::string& b_in, int a_out = -1);
Model model_link(Model m, int out_idx, const std::string& arg);
Model model_combine(const Model& a, const Model& b);
Model model_dedupe(Model m);

Model conv_layer(const std::string& name, const ConvSpec& spec, bool bias);
Model batchnorm_layer(const std::string& name, const Dims& dims, unsigned long flags, bool train,
                      double eps = 1e-5, double momentum = 0.1);
Model loss_model_mse(const Dims& dims);

Model sense_normal_fragment(const SenseDims& sd);
struct ModlConfig;
struct VarNetConfig;
Model modl_denoiser(const ModlConfig& cfg, const std::string& stat_suffix);
Model bn_block_fragment(const std::string& ln, const Dims& cur);
Model varnet_reg(const VarNetConfig& cfg, const std::string& prefix);
Model sense_adjoint_fragment(const SenseDims& sd);
Model modl_normal_plus_lambda(const SenseDims& sd);

struct ModlConfig {
    long iterations = 10, layers = 5, filters = 32, kernel = 3, cg_iter = 10;
    double cg_tol = 1e-7, lambda_init = 0.05;
    long im_x = 0, im_y = 0, coils = 1, maps = 1, batch = 1;
    bool train_mode = true;
    SenseDims sense() const { return SenseDims{im_x, im_y, coils, maps, batch}; }
    void validate() const;
};
struct VarNetConfig {
    long iterations = 10, filters = 24, kernel = 11, rbf = 31;
    long im_x = 0, im_y = 0, coils = 1, maps = 1, batch = 1;
    SenseDims sense() const { return SenseDims{im_x, im_y, coils, maps, batch}; }
    void validate() const;
};
Model build_modl(const ModlConfig& cfg);
Model build_varnet(const VarNetConfig& cfg);

// simulate.hpp:40-133 restated (fixture generators; host double math)
void sim_phantom(std::complex<float>* img, long nx, long ny, Rng& rng);
void sim_coils(std::complex<float>* maps, long nx, long ny, long nc, Rng& rng);
void sim_pattern(std::complex<float>* p, long size, long accel, long acl);

} // namespace mdnn
