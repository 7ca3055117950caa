// TEST INFRASTRUCTURE ONLY - never linked into the product.
//
// C-ABI shim over the *unmodified* reference hot path (turbda::analyze and
// friends), compiled from the sources where they lie under
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/.  Tests and
// bench.py's cpu_baseline / --impl reference leg load the result via ctypes.
//
// Every entry point forwards to the reference implementation:
//   ref_analyze          -> turbda::analyze        proj/src/ensf.cpp:132-223
//   ref_relax_spread     -> turbda::relax_spread   proj/src/ensf.cpp:225-258
//   ref_prior_score      -> turbda::prior_score    proj/src/ensf.cpp:68-82
//   ref_posterior_score  -> turbda::posterior_score proj/src/ensf.cpp:96-106
//   ref_philox4x32       -> turbda::philox4x32     proj/src/rng.cpp:23-31
//   ref_splitmix64       -> turbda::splitmix64     proj/src/rng.cpp:33-38
//   ref_stream_*         -> turbda::RngStream      proj/src/rng.cpp:40-84
//   ref_fast_exp_nonpos  -> turbda::fast_exp_nonpos proj/include/turbda/fastexp.hpp:13-50
//   ref_synthesize_obs   -> turbda::synthesize_observations proj/src/observation.cpp:62-81
//   ref_rmse / ref_spread -> proj/src/ensemble.cpp:18-43
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "turbda/ensemble.hpp"
#include "turbda/ensf.hpp"
#include "turbda/errors.hpp"
#include "turbda/fastexp.hpp"
#include "turbda/observation.hpp"
#include "turbda/parallel.hpp"
#include "turbda/rng.hpp"

using namespace turbda;

namespace {

enum : int { kOk = 0, kConfig = 1, kDimension = 2, kDiverged = 3, kDomain = 4, kOther = 5 };

void put_msg(char* msg, int len, const char* what) {
    if (!msg || len <= 0) return;
    std::strncpy(msg, what, size_t(len - 1));
    msg[len - 1] = '\0';
}

template <class F>
int guarded(char* msg, int msglen, double* div_t, F&& f) {
    try {
        f();
        return kOk;
    } catch (const SamplerDivergedError& e) {
        if (div_t) *div_t = e.pseudo_time;
        put_msg(msg, msglen, e.what());
        return kDiverged;
    } catch (const ConfigError& e) {
        put_msg(msg, msglen, e.what());
        return kConfig;
    } catch (const DimensionError& e) {
        put_msg(msg, msglen, e.what());
        return kDimension;
    } catch (const std::domain_error& e) {
        put_msg(msg, msglen, e.what());
        return kDomain;
    } catch (const std::exception& e) {
        put_msg(msg, msglen, e.what());
        return kOther;
    }
}

Ensemble make_ensemble(const double* members, int m, int64_t d, double time) {
    Ensemble ens;
    ens.valid_time = time;
    ens.members.resize(size_t(m));
    ens.member_seeds.resize(size_t(m));
    for (int j = 0; j < m; ++j) {
        ens.members[size_t(j)].assign(members + size_t(j) * size_t(d),
                                      members + size_t(j + 1) * size_t(d));
        ens.member_seeds[size_t(j)] = uint64_t(j) + 1;
    }
    return ens;
}

// obs_kind 0 = identity (y, r have d entries), 1 = index_selection
Observation make_observation(int64_t d, const double* y, const double* r,
                             const int64_t* idx, int64_t obs_dim, int obs_kind,
                             double time) {
    Observation obs;
    obs.op.state_dim = size_t(d);
    obs.op.kind = obs_kind == 0 ? ObsOperatorKind::identity
                                : ObsOperatorKind::index_selection;
    if (obs_kind != 0)
        for (int64_t q = 0; q < obs_dim; ++q) obs.op.indices.push_back(size_t(idx[q]));
    obs.y.assign(y, y + obs_dim);
    obs.r_diag.assign(r, r + obs_dim);
    obs.locations.assign(size_t(obs_dim), {0.0, 0.0});
    obs.time = time;
    return obs;
}

void flatten(const Ensemble& e, double* out) {
    const size_t d = e.dim();
    for (int j = 0; j < e.size(); ++j)
        std::memcpy(out + size_t(j) * d, e.members[size_t(j)].data(), d * sizeof(double));
}

}  // namespace

extern "C" {

int ref_analyze(const double* members, int m, int64_t d, const double* y,
                const double* r, const int64_t* idx, int64_t obs_dim,
                int obs_kind, int n_steps, double eps, int minibatch_j,
                double damping_t, double relax_factor, uint64_t seed,
                uint64_t cycle, int workers, double* out, double* diverged_t,
                char* msg, int msglen) {
    return guarded(msg, msglen, diverged_t, [&] {
        const Ensemble ens = make_ensemble(members, m, d, 0.0);
        const Observation obs = make_observation(d, y, r, idx, obs_dim, obs_kind, 0.0);
        EnsfConfig cfg;
        cfg.n_steps = n_steps;
        cfg.eps = eps;
        cfg.minibatch_j = minibatch_j;
        cfg.damping_t = damping_t;
        cfg.relax_factor = relax_factor;
        const Ensemble post = analyze(ens, obs, cfg, seed, cycle, workers);
        flatten(post, out);
    });
}

int ref_relax_spread(const double* analysis, const double* forecast, int m,
                     int64_t d, double factor, double* out) {
    return guarded(nullptr, 0, nullptr, [&] {
        const Ensemble a = make_ensemble(analysis, m, d, 0.0);
        const Ensemble f = make_ensemble(forecast, m, d, 0.0);
        flatten(relax_spread(a, f, factor), out);
    });
}

int ref_prior_score(const double* z, int64_t d, double t, const double* members,
                    int m, const int* batch, int nbatch, double eps, double* out) {
    return guarded(nullptr, 0, nullptr, [&] {
        const Ensemble ens = make_ensemble(members, m, d, 0.0);
        std::vector<int> b(batch, batch + nbatch);
        const auto s = prior_score(std::vector<double>(z, z + d), t, ens, b, eps);
        std::memcpy(out, s.data(), size_t(d) * sizeof(double));
    });
}

int ref_posterior_score(const double* z, int64_t d, double t,
                        const double* members, int m, const double* y,
                        const double* r, const int64_t* idx, int64_t obs_dim,
                        int obs_kind, double eps, double damping_t, double* out) {
    return guarded(nullptr, 0, nullptr, [&] {
        const Ensemble ens = make_ensemble(members, m, d, 0.0);
        const Observation obs = make_observation(d, y, r, idx, obs_dim, obs_kind, 0.0);
        EnsfConfig cfg;
        cfg.eps = eps;
        cfg.damping_t = damping_t;
        const auto s = posterior_score(std::vector<double>(z, z + d), t, ens, obs, cfg);
        std::memcpy(out, s.data(), size_t(d) * sizeof(double));
    });
}

void ref_philox4x32(const uint32_t* ctr, const uint32_t* key, uint32_t* out) {
    const auto r = philox4x32({ctr[0], ctr[1], ctr[2], ctr[3]}, {key[0], key[1]});
    for (int q = 0; q < 4; ++q) out[q] = r[size_t(q)];
}

uint64_t ref_splitmix64(uint64_t x) { return splitmix64(x); }

void ref_stream_normals(uint64_t seed, uint64_t use, uint64_t entity, int64_t n,
                        double* out) {
    RngStream rs(seed, static_cast<StreamUse>(use), entity);
    for (int64_t q = 0; q < n; ++q) out[q] = rs.normal();
}

void ref_stream_uniforms(uint64_t seed, uint64_t use, uint64_t entity, int64_t n,
                         double* out) {
    RngStream rs(seed, static_cast<StreamUse>(use), entity);
    for (int64_t q = 0; q < n; ++q) out[q] = rs.uniform();
}

void ref_stream_u64(uint64_t seed, uint64_t use, uint64_t entity, int64_t n,
                    uint64_t* out) {
    RngStream rs(seed, static_cast<StreamUse>(use), entity);
    for (int64_t q = 0; q < n; ++q) out[q] = rs.next_u64();
}

double ref_fast_exp_nonpos(double x) { return fast_exp_nonpos(x); }

int ref_synthesize_obs(const double* truth, int64_t d, const int64_t* idx,
                       int64_t obs_dim, int obs_kind, double r_variance,
                       uint64_t seed, uint64_t cycle, double* y_out) {
    return guarded(nullptr, 0, nullptr, [&] {
        GridSpec g;  // only used for locations, which are not returned
        g.nx = int(d);
        g.ny = 1;
        ObsOperator op;
        op.state_dim = size_t(d);
        op.kind = obs_kind == 0 ? ObsOperatorKind::identity
                                : ObsOperatorKind::index_selection;
        if (obs_kind != 0)
            for (int64_t q = 0; q < obs_dim; ++q) op.indices.push_back(size_t(idx[q]));
        const Observation o = synthesize_observations(
            std::vector<double>(truth, truth + d), g, op, r_variance, 0.0, seed, cycle);
        std::memcpy(y_out, o.y.data(), o.y.size() * sizeof(double));
    });
}

double ref_rmse(const double* mean, const double* truth, int64_t d) {
    return rmse(std::vector<double>(mean, mean + d), std::vector<double>(truth, truth + d));
}

double ref_spread(const double* members, int m, int64_t d) {
    return spread(make_ensemble(members, m, d, 0.0));
}

int ref_default_worker_count(void) { return default_worker_count(); }

}  // extern "C"
