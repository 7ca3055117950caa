// C++ host of the turbda API (include/turbda/*.hpp) above the C-ABI.
//
// analyze / relax_spread / prior_score / posterior_score keep the reference
// signatures and validation order (proj/src/ensf.cpp:68-258) and run on the
// GPU through include/turbda_b200.h; status codes come back as the
// reference's exception types.  The remaining functions are the small host
// utilities of the same API (RNG, operators, ensemble statistics).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <exception>
#include <stdexcept>
#include <thread>
#include <vector>

#include "host_rng.h"
#include "turbda/ensemble.hpp"
#include "turbda/ensf.hpp"
#include "turbda/errors.hpp"
#include "turbda/letkf.hpp"
#include "turbda/observation.hpp"
#include "turbda/parallel.hpp"
#include "turbda/rng.hpp"
#include "turbda_b200.h"

namespace turbda {

namespace {

[[noreturn]] void raise(int code, const turbda_status& st) {
    switch (code) {
        case TURBDA_CONFIG: throw ConfigError(st.msg);
        case TURBDA_DIMENSION: throw DimensionError(st.msg);
        case TURBDA_DIVERGED: throw SamplerDivergedError(st.diverged_t);
        case TURBDA_DOMAIN: throw std::domain_error(st.msg);
        case TURBDA_SINGULAR: throw SingularAnalysisError(st.diverged_particle, st.diverged_step);
        case TURBDA_IO: throw IoError(st.msg);
        default: throw std::runtime_error(std::string("turbda_b200: ") + st.msg);
    }
}

void check(int code, const turbda_status& st) {
    if (code != TURBDA_OK) raise(code, st);
}

struct FlatObs {
    std::vector<int64_t> idx;
    int kind = 0;
};

// C-ABI operator kind: 0 identity, 1 index_selection, 2 arctan, 3 arctan_selection
int abi_kind(ObsOperatorKind k) {
    switch (k) {
        case ObsOperatorKind::identity: return 0;
        case ObsOperatorKind::index_selection: return 1;
        case ObsOperatorKind::arctan: return 2;
        case ObsOperatorKind::arctan_selection: return 3;
    }
    return 0;
}

FlatObs flatten_obs(const Observation& obs) {
    FlatObs f;
    f.kind = abi_kind(obs.op.kind);
    if (!is_dense(obs.op.kind)) f.idx.assign(obs.op.indices.begin(), obs.op.indices.end());
    return f;
}

}  // namespace

// ---------------------------------------------------------------- rng -----
std::array<std::uint32_t, 4> philox4x32(std::array<std::uint32_t, 4> ctr,
                                        std::array<std::uint32_t, 2> key) {
    return tb200::philox4x32_10(ctr, key);
}

std::uint64_t splitmix64(std::uint64_t x) { return tb200::splitmix64(x); }

RngStream::RngStream(std::uint64_t seed, StreamUse use, std::uint64_t entity) {
    const std::uint64_t k = tb200::stream_key(seed, static_cast<std::uint64_t>(use));
    key_ = {std::uint32_t(k), std::uint32_t(k >> 32)};
    entity_ = {std::uint32_t(entity), std::uint32_t(entity >> 32)};
}

std::uint32_t RngStream::next_u32() {
    if (pos_ >= 4) {
        buf_ = tb200::philox4x32_10(
            {std::uint32_t(block_), std::uint32_t(block_ >> 32), entity_[0], entity_[1]}, key_);
        ++block_;
        pos_ = 0;
    }
    return buf_[size_t(pos_++)];
}

std::uint64_t RngStream::next_u64() {
    const std::uint64_t lo = next_u32();
    return lo | (std::uint64_t(next_u32()) << 32);
}

double RngStream::uniform() { return (double(next_u64() >> 11) + 0.5) * 0x1.0p-53; }

double RngStream::normal() {
    if (has_spare_) {
        has_spare_ = false;
        return spare_;
    }
    const double u1 = uniform();
    const double u2 = uniform();
    const double rad = std::sqrt(-2.0 * std::log(u1));
    const double ang = 2.0 * 3.14159265358979323846 * u2;
    spare_ = rad * std::sin(ang);
    has_spare_ = true;
    return rad * std::cos(ang);
}

// ----------------------------------------------------------- parallel -----
int default_worker_count() {
    if (const char* env = std::getenv("TURBDA_WORKERS")) {
        const long v = std::strtol(env, nullptr, 10);
        if (v >= 1) return int(v);
    }
    const unsigned hc = std::thread::hardware_concurrency();
    return hc ? int(hc) : 1;
}

void parallel_for(std::size_t n, int workers, const std::function<void(std::size_t)>& fn) {
    if (n == 0) return;
    const std::size_t nw = std::min<std::size_t>(std::size_t(std::max(workers, 1)), n);
    if (nw == 1) {
        for (std::size_t i = 0; i < n; ++i) fn(i);
        return;
    }
    const std::size_t q = n / nw, rem = n % nw;
    std::vector<std::exception_ptr> errs(nw);
    std::vector<std::size_t> where(nw, n);
    std::vector<std::thread> pool;
    for (std::size_t b = 0; b < nw; ++b) {
        const std::size_t lo = b * q + std::min(b, rem);
        const std::size_t hi = lo + q + (b < rem ? 1 : 0);
        pool.emplace_back([&, b, lo, hi] {
            for (std::size_t i = lo; i < hi; ++i) {
                try {
                    fn(i);
                } catch (...) {
                    errs[b] = std::current_exception();
                    where[b] = i;
                    return;
                }
            }
        });
    }
    for (auto& t : pool) t.join();
    std::size_t first = n, owner = nw;
    for (std::size_t b = 0; b < nw; ++b)
        if (errs[b] && where[b] < first) {
            first = where[b];
            owner = b;
        }
    if (owner < nw) std::rethrow_exception(errs[owner]);
}

// ----------------------------------------------------------- ensemble -----
std::vector<double> ensemble_mean(const Ensemble& ens) {
    ens.validate(false);
    std::vector<double> mean(ens.dim(), 0.0);
    for (const auto& v : ens.members)
        for (std::size_t k = 0; k < mean.size(); ++k) mean[k] += v[k];
    const double inv = 1.0 / ens.size();
    for (double& v : mean) v *= inv;
    return mean;
}

double rmse(const std::vector<double>& mean, const std::vector<double>& truth) {
    if (mean.size() != truth.size()) throw DimensionError("rmse: dimension mismatch");
    double acc = 0.0;
    for (std::size_t k = 0; k < mean.size(); ++k) acc += (mean[k] - truth[k]) * (mean[k] - truth[k]);
    return std::sqrt(acc / double(mean.size()));
}

double spread(const Ensemble& ens) {
    ens.validate(false);
    if (ens.size() < 2) return 0.0;
    const std::vector<double> mean = ensemble_mean(ens);
    double acc = 0.0;
    for (const auto& v : ens.members)
        for (std::size_t k = 0; k < mean.size(); ++k) acc += (v[k] - mean[k]) * (v[k] - mean[k]);
    return std::sqrt(acc / (double(ens.size() - 1) * double(ens.dim())));
}

// -------------------------------------------------------- observation -----
std::vector<double> apply_operator(const ObsOperator& op, const std::vector<double>& state) {
    if (state.size() != op.state_dim) throw DimensionError("apply_operator: state dimension mismatch");
    std::vector<double> out;
    if (is_dense(op.kind)) {
        out = state;
    } else {
        out.reserve(op.indices.size());
        for (const std::size_t k : op.indices) out.push_back(state[k]);
    }
    if (is_arctan(op.kind))
        for (double& v : out) v = std::atan(v);
    return out;
}

// scatter pattern of the operator (for the arctan kinds: of its linearisation;
// the derivative factor 1/(1+x^2) is applied by likelihood_score)
std::vector<double> adjoint_scatter(const ObsOperator& op, const std::vector<double>& w) {
    if (w.size() != op.obs_dim()) throw DimensionError("adjoint_scatter: obs dimension mismatch");
    if (is_dense(op.kind)) return w;
    std::vector<double> out(op.state_dim, 0.0);
    for (std::size_t q = 0; q < op.indices.size(); ++q) out[op.indices[q]] += w[q];
    return out;
}

ObsOperator make_grid_operator(const GridSpec& grid, int thinning_stride) {
    ObsOperator op;
    op.state_dim = grid.grid_size();
    if (thinning_stride > 1) {
        op.kind = ObsOperatorKind::index_selection;
        for (std::size_t k = 0; k < op.state_dim; k += std::size_t(thinning_stride))
            op.indices.push_back(k);
    }
    return op;
}

ObsOperator make_arctan_operator(const GridSpec& grid, int thinning_stride) {
    ObsOperator op = make_grid_operator(grid, thinning_stride);
    op.kind = thinning_stride > 1 ? ObsOperatorKind::arctan_selection : ObsOperatorKind::arctan;
    return op;
}

std::vector<std::array<double, 2>> operator_locations(const GridSpec& grid, const ObsOperator& op) {
    const std::size_t plane = std::size_t(grid.ny) * std::size_t(grid.nx);
    const auto at = [&](std::size_t flat) {
        const std::size_t h = flat % plane;
        return std::array<double, 2>{double(h % std::size_t(grid.nx)),
                                     double(h / std::size_t(grid.nx))};
    };
    std::vector<std::array<double, 2>> out;
    if (is_dense(op.kind)) {
        out.reserve(op.state_dim);
        for (std::size_t k = 0; k < op.state_dim; ++k) out.push_back(at(k));
    } else {
        out.reserve(op.indices.size());
        for (const std::size_t k : op.indices) out.push_back(at(k));
    }
    return out;
}

Observation synthesize_observations(const std::vector<double>& truth, const GridSpec& grid,
                                    const ObsOperator& op, double r_variance, double time_hours,
                                    std::uint64_t seed, std::uint64_t cycle) {
    if (!(r_variance >= 0.0)) throw ConfigError("synthesize_observations: r must be >= 0");
    Observation obs;
    obs.op = op;
    obs.y = apply_operator(op, truth);
    obs.locations = operator_locations(grid, op);
    obs.time = time_hours;
    const double sd = std::sqrt(r_variance);
    RngStream noise(seed, StreamUse::obs_noise, cycle);
    for (double& v : obs.y) v += sd * noise.normal();
    obs.r_diag.assign(obs.y.size(), r_variance);
    return obs;
}

// --------------------------------------------------------------- ensf -----
namespace {

std::vector<double> pack(const Ensemble& e) {
    const std::size_t d = e.dim();
    std::vector<double> flat(std::size_t(e.size()) * d);
    for (int j = 0; j < e.size(); ++j)
        std::copy(e.members[size_t(j)].begin(), e.members[size_t(j)].end(),
                  flat.begin() + std::ptrdiff_t(size_t(j) * d));
    return flat;
}

std::vector<double> score_call(const std::vector<double>& z, double t, const Ensemble& forecast,
                               const std::vector<int>& batch, double eps, const Observation* obs,
                               double damping_t) {
    const std::vector<double> x = pack(forecast);
    std::vector<double> out(z.size());
    turbda_status st{};
    FlatObs fo;
    if (obs) fo = flatten_obs(*obs);
    const int rc = turbda_score(z.data(), int64_t(z.size()), t, x.data(), forecast.size(),
                                batch.empty() ? nullptr : batch.data(), int32_t(batch.size()), eps,
                                obs ? obs->y.data() : nullptr, obs ? obs->r_diag.data() : nullptr,
                                fo.idx.empty() ? nullptr : fo.idx.data(),
                                obs ? int64_t(obs->y.size()) : 0, fo.kind, damping_t, out.data(),
                                -1, &st);
    check(rc, st);
    return out;
}

}  // namespace

std::vector<double> prior_score(const std::vector<double>& z, double t, const Ensemble& forecast,
                                const std::vector<int>& batch, double eps) {
    if (t < eps) throw std::domain_error("prior_score: t below eps (beta -> 0)");
    if (t > 1.0) throw std::domain_error("prior_score: t > 1");
    forecast.validate(false);
    if (z.size() != forecast.dim()) throw DimensionError("prior_score: dimension mismatch");
    return score_call(z, t, forecast, batch, eps, nullptr, 0.0);
}

std::vector<double> likelihood_score(const std::vector<double>& z, const Observation& obs) {
    obs.validate();
    if (z.size() != obs.op.state_dim) throw DimensionError("likelihood_score: dimension mismatch");
    // on the device: turbda_likelihood_score (the {A, B} observation prep of
    // the analysis, duplicates adding as adjoint_scatter does)
    std::vector<int64_t> idx(obs.op.indices.begin(), obs.op.indices.end());
    std::vector<double> out(z.size());
    turbda_status st;
    const int rc = turbda_likelihood_score(z.data(), int64_t(z.size()), obs.y.data(),
                                           obs.r_diag.data(), is_dense(obs.op.kind) ? nullptr : idx.data(),
                                           int64_t(obs.y.size()), abi_kind(obs.op.kind), out.data(), -1,
                                           &st);
    check(rc, st);
    return out;
}

std::vector<double> posterior_score(const std::vector<double>& z, double t,
                                    const Ensemble& forecast, const Observation& obs,
                                    const EnsfConfig& cfg) {
    cfg.validate();
    if (t < cfg.eps) throw std::domain_error("prior_score: t below eps (beta -> 0)");
    if (t > 1.0) throw std::domain_error("prior_score: t > 1");
    forecast.validate(false);
    if (z.size() != forecast.dim()) throw DimensionError("prior_score: dimension mismatch");
    obs.validate();
    if (z.size() != obs.op.state_dim) throw DimensionError("likelihood_score: dimension mismatch");
    return score_call(z, t, forecast, {}, cfg.eps, &obs, cfg.damping_t);
}

void reverse_sde_step(std::vector<std::vector<double>>& particles, double t, double dt_pseudo,
                      const std::vector<std::vector<double>>& scores,
                      const std::vector<std::vector<double>>& noise) {
    if (dt_pseudo <= 0.0) throw ConfigError("reverse_sde_step: dt_pseudo > 0");
    if (scores.size() != particles.size() || noise.size() != particles.size())
        throw DimensionError("reverse_sde_step: array count mismatch");
    const size_t n = particles.size();
    const size_t d = n ? particles[0].size() : 0;
    for (size_t i = 0; i < n; ++i)
        if (particles[i].size() != d || scores[i].size() != d || noise[i].size() != d)
            throw DimensionError("reverse_sde_step: dimension mismatch");
    // on the device (turbda_reverse_sde_step): pack [n][d], one launch
    std::vector<double> z(n * d), sc(n * d), xi(n * d);
    for (size_t i = 0; i < n; ++i) {
        std::copy(particles[i].begin(), particles[i].end(), z.begin() + i * d);
        std::copy(scores[i].begin(), scores[i].end(), sc.begin() + i * d);
        std::copy(noise[i].begin(), noise[i].end(), xi.begin() + i * d);
    }
    turbda_status st;
    const int rc = turbda_reverse_sde_step(z.data(), int32_t(n), int64_t(d), t, dt_pseudo, sc.data(),
                                           xi.data(), -1, &st);
    if (rc != TURBDA_OK && rc != TURBDA_DIVERGED) check(rc, st);
    for (size_t i = 0; i < n; ++i)
        std::copy(z.begin() + i * d, z.begin() + (i + 1) * d, particles[i].begin());
    if (rc == TURBDA_DIVERGED) throw SamplerDivergedError(t);
}

Ensemble analyze(const Ensemble& forecast, const Observation& obs, const EnsfConfig& cfg,
                 std::uint64_t seed, std::uint64_t cycle, int /*workers: the GPU grid*/) {
    // validation order of proj/src/ensf.cpp:135-143
    forecast.validate(false);
    obs.validate();
    cfg.validate();
    if (std::fabs(forecast.valid_time - obs.time) > 1e-6)
        throw ConfigError("analyze: forecast/observation time mismatch");
    const std::size_t d = forecast.dim();
    if (obs.op.state_dim != d) throw DimensionError("analyze: observation operator dimension");
    for (const std::size_t k : obs.op.indices)
        if (!is_dense(obs.op.kind) && k >= d)
            throw DimensionError("analyze: observation index outside the state");

    turbda_ensf_params p;
    turbda_ensf_params_init(&p);
    p.d_total = int64_t(d);
    p.k0 = 0;
    p.d_local = int64_t(d);
    p.obs_dim = int64_t(obs.y.size());
    p.n_members = forecast.size();
    p.n_steps = cfg.n_steps;
    p.minibatch_j = cfg.minibatch_j;
    p.obs_kind = abi_kind(obs.op.kind);
    p.eps = cfg.eps;
    p.damping_t = cfg.damping_t;
    p.relax_factor = cfg.relax_factor;
    p.seed = seed;
    p.cycle = cycle;
    p.precision = int32_t(cfg.precision);
    p.device = cfg.device;
    p.device_count = std::max(1, cfg.device_count);

    Ensemble analysis;
    analysis.members.assign(size_t(forecast.size()), std::vector<double>(d));
    analysis.member_seeds = forecast.member_seeds;
    analysis.valid_time = forecast.valid_time;
    std::vector<const double*> in_rows(size_t(forecast.size()));
    std::vector<double*> out_rows(size_t(forecast.size()));
    for (int j = 0; j < forecast.size(); ++j) {
        in_rows[size_t(j)] = forecast.members[size_t(j)].data();
        out_rows[size_t(j)] = analysis.members[size_t(j)].data();
    }
    const FlatObs fo = flatten_obs(obs);
    turbda_status st{};
    const int rc = turbda_ensf_analyze_rows(&p, in_rows.data(), obs.y.data(), obs.r_diag.data(),
                                            fo.idx.empty() ? nullptr : fo.idx.data(),
                                            out_rows.data(), &st);
    check(rc, st);
    return analysis;
}

Ensemble relax_spread(const Ensemble& analysis, const Ensemble& forecast, double factor) {
    if (factor == 0.0) return analysis;
    analysis.validate(false);
    forecast.validate(false);
    if (analysis.size() != forecast.size() || analysis.dim() != forecast.dim())
        throw DimensionError("relax_spread: shape mismatch");
    if (analysis.size() < 2) return analysis;
    const std::vector<double> a = pack(analysis), f = pack(forecast);
    std::vector<double> o(a.size());
    turbda_status st{};
    check(turbda_relax_spread(a.data(), f.data(), analysis.size(), int64_t(analysis.dim()), factor,
                              o.data(), -1, 0u, nullptr, &st),
          st);
    Ensemble out = analysis;
    const std::size_t d = analysis.dim();
    for (int j = 0; j < out.size(); ++j)
        std::copy(o.begin() + std::ptrdiff_t(size_t(j) * d), o.begin() + std::ptrdiff_t(size_t(j + 1) * d),
                  out.members[size_t(j)].begin());
    return out;
}

// -------------------------------------------------------------- letkf -----
double gaspari_cohn(double r) {
    double v = 0.0;
    turbda_status st{};
    check(turbda_gaspari_cohn(r, &v, &st), st);
    return v;
}

Ensemble letkf_analyze(const Ensemble& forecast, const Observation& obs, const LetkfConfig& cfg,
                       const GridSpec& grid, int /*workers: the GPU grid*/) {
    // validation order of proj/src/letkf.cpp:57-69
    forecast.validate();
    obs.validate();
    cfg.validate();
    grid.validate();
    if (grid.nx != grid.ny || grid.lx != grid.ly)
        throw ConfigError("letkf_analyze: isotropic metric needs nx == ny");
    if (std::fabs(forecast.valid_time - obs.time) > 1e-6)
        throw ConfigError("letkf_analyze: forecast/observation time mismatch");
    const std::size_t d = forecast.dim();
    if (d != grid.grid_size() || obs.op.state_dim != d)
        throw DimensionError("letkf_analyze: state/grid size mismatch");

    turbda_letkf_params p;
    turbda_letkf_params_init(&p);
    p.nx = grid.nx;
    p.ny = grid.ny;
    p.n_members = forecast.size();
    p.obs_kind = abi_kind(obs.op.kind);
    p.obs_dim = int64_t(obs.y.size());
    p.cutoff_km = cfg.cutoff_km;
    p.domain_km = cfg.domain_km;
    p.rtps_alpha = cfg.rtps_alpha;
    const FlatObs fo = flatten_obs(obs);
    std::vector<double> locs(2 * obs.locations.size());
    for (std::size_t k = 0; k < obs.locations.size(); ++k) {
        locs[2 * k] = obs.locations[k][0];
        locs[2 * k + 1] = obs.locations[k][1];
    }
    const std::vector<double> x = pack(forecast);
    std::vector<double> o(x.size());
    turbda_status st{};
    check(turbda_letkf_analyze(&p, x.data(), obs.y.data(), obs.r_diag.data(),
                               fo.idx.empty() ? nullptr : fo.idx.data(),
                               locs.empty() ? nullptr : locs.data(), o.data(), nullptr, &st),
          st);
    Ensemble out = forecast;
    for (int j = 0; j < out.size(); ++j)
        std::copy(o.begin() + std::ptrdiff_t(size_t(j) * d), o.begin() + std::ptrdiff_t(size_t(j + 1) * d),
                  out.members[size_t(j)].begin());
    return out;
}

Ensemble rtps_inflate(const Ensemble& analysis, const Ensemble& background, double alpha) {
    if (alpha == 0.0) return analysis;
    analysis.validate(false);
    background.validate(false);
    if (analysis.size() != background.size() || analysis.dim() != background.dim())
        throw DimensionError("rtps_inflate: shape mismatch");
    if (analysis.size() < 2) return analysis;
    const std::vector<double> a = pack(analysis), b = pack(background);
    std::vector<double> o(a.size());
    turbda_status st{};
    check(turbda_rtps_inflate(a.data(), b.data(), analysis.size(), int64_t(analysis.dim()), alpha,
                              o.data(), -1, 0u, nullptr, &st),
          st);
    Ensemble out = analysis;
    const std::size_t d = analysis.dim();
    for (int j = 0; j < out.size(); ++j)
        std::copy(o.begin() + std::ptrdiff_t(size_t(j) * d), o.begin() + std::ptrdiff_t(size_t(j + 1) * d),
                  out.members[size_t(j)].begin());
    return out;
}

}  // namespace turbda
