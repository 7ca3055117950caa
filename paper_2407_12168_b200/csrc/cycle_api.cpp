// C++ host of the forecast / OSSE layer of the turbda API
// (include/turbda/{sqg,forecast,osse}.hpp) above the C-ABI: the SQG model
// steps on the GPU (turbda_sqg_*, turbda_nature_run), analyses run on the
// GPU (turbda::analyze, turbda::letkf_analyze); the cycle bookkeeping, model
// error draws and metrics follow the reference semantics
// (proj/src/forecast.cpp, proj/src/osse.cpp) on the host.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <numeric>
#include <string>
#include <vector>

#include "turbda/ensemble.hpp"
#include "turbda/forecast.hpp"
#include "turbda/observation.hpp"
#include "turbda/osse.hpp"
#include "turbda/rng.hpp"
#include "turbda_b200.h"

namespace turbda {

namespace {

turbda_sqg_params to_abi(const GridSpec& g, const SqgParams& p) {
    turbda_sqg_params a;
    turbda_sqg_params_init(&a);
    a.nx = g.nx;
    a.ny = g.ny;
    a.lx = g.lx;
    a.ly = g.ly;
    a.h = g.h;
    a.f = p.f;
    a.n = p.n;
    a.u0 = p.u0;
    a.hyper_order = p.hyper_order;
    a.hyper_efold = p.hyper_efold;
    a.dt = p.dt;
    a.drag_tau = p.drag_tau;
    return a;
}

[[noreturn]] void raise_sqg(int code, const turbda_status& st) {
    switch (code) {
        case TURBDA_CONFIG: throw ConfigError(st.msg);
        case TURBDA_DIMENSION: throw DimensionError(st.msg);
        case TURBDA_BLOWUP: throw BlowupError(st.diverged_t, st.diverged_particle);
        default: throw std::runtime_error(std::string("turbda_b200: ") + st.msg);
    }
}

bool whole_steps(double hours, double dt, long* steps) {
    const double q = hours / dt;
    *steps = std::lround(q);
    return hours >= 0.0 && std::fabs(q - double(*steps)) <= 1e-9;
}

}  // namespace

// ------------------------------------------------------------- SqgModel -----
SqgModel::SqgModel(const GridSpec& grid, const SqgParams& params, int batch, int device)
    : grid_(grid), params_(params), batch_(batch) {
    grid.validate();
    params.validate();
    if (batch < 1) throw ConfigError("sqg: batch >= 1");
    const turbda_sqg_params a = to_abi(grid, params);
    turbda_status st{};
    if (int rc = turbda_sqg_create(&a, batch, device, &handle_, &st)) raise_sqg(rc, st);
}

SqgModel::~SqgModel() {
    if (handle_) turbda_sqg_destroy(handle_);
}

void SqgModel::advance(double* states, double hours) {
    long steps = 0;
    if (!whole_steps(hours, params_.dt, &steps))
        throw ConfigError("advance: duration must be a multiple of dt");
    if (steps == 0) return;  // the exact identity
    double cfl = 0.0;
    turbda_status st{};
    const int rc = turbda_sqg_advance(handle_, states, hours, 0u, nullptr, &cfl, &st);
    max_cfl_ = std::max(max_cfl_, cfl);
    if (rc) raise_sqg(rc, st);
}

std::vector<KeBin> SqgModel::ke_spectrum(const double* state) {
    const int cap = grid_.nx + grid_.ny + 8;  // > number of shells
    std::vector<double> k(static_cast<size_t>(cap)), e(static_cast<size_t>(cap));
    int32_t n = 0;
    turbda_status st{};
    if (int rc = turbda_sqg_ke_spectrum(handle_, state, 0u, k.data(), e.data(), cap, &n, &st))
        raise_sqg(rc, st);
    std::vector<KeBin> bins(static_cast<size_t>(n));
    for (int s = 0; s < n; ++s) bins[size_t(s)] = {k[size_t(s)], e[size_t(s)]};
    return bins;
}

double fit_loglog_slope(const std::vector<KeBin>& spectrum, int lo_shell, int hi_shell) {
    std::vector<double> k, e;
    for (const KeBin& b : spectrum) {
        k.push_back(b.kappa);
        e.push_back(b.energy);
    }
    double slope = 0.0;
    turbda_status st{};
    if (int rc = turbda_fit_loglog_slope(k.data(), e.data(), int32_t(k.size()), lo_shell, hi_shell,
                                         &slope, &st))
        raise_sqg(rc, st);
    return slope;
}

// ------------------------------------------------------------- forecast -----
SqgStepper::SqgStepper(const GridSpec& grid, const SqgParams& params) : model_(grid, params) {}

void SqgStepper::advance(std::vector<double>& state, double hours) {
    if (state.size() != model_.grid().grid_size())
        throw DimensionError("advance: state size does not match grid");
    try {
        model_.advance(state.data(), hours);
    } catch (const BlowupError& e) {
        throw BlowupError(e.time_hours);  // a single state: no member index
    }
}

StepperFactory sqg_stepper_factory(const GridSpec& grid, const SqgParams& params) {
    return [grid, params]() { return std::make_unique<SqgStepper>(grid, params); };
}

void advance(std::vector<double>& state, double hours, Stepper& stepper) {
    stepper.advance(state, hours);
}

namespace {

// all members as one batched device model (SqgStepper factories)
Ensemble propagate_batched(const Ensemble& ens, double hours, SqgModel& model,
                           double* max_cfl_out) {
    const int m = ens.size();
    const std::size_t d = model.grid().grid_size();
    std::vector<double> flat(d * size_t(m));
    for (int j = 0; j < m; ++j) {
        if (ens.members[size_t(j)].size() != d)
            throw DimensionError("advance: state size does not match grid");
        std::copy(ens.members[size_t(j)].begin(), ens.members[size_t(j)].end(),
                  flat.begin() + std::ptrdiff_t(size_t(j) * d));
    }
    model.reset_cfl();
    model.advance(flat.data(), hours);  // BlowupError carries the member index
    Ensemble out = ens;
    for (int j = 0; j < m; ++j)
        std::copy(flat.begin() + std::ptrdiff_t(size_t(j) * d),
                  flat.begin() + std::ptrdiff_t(size_t(j + 1) * d), out.members[size_t(j)].begin());
    if (max_cfl_out) *max_cfl_out = model.max_cfl();
    out.valid_time = ens.valid_time + hours;
    return out;
}

}  // namespace

Ensemble propagate_ensemble(const Ensemble& ens, double hours, const StepperFactory& factory,
                            int workers, double* max_cfl_out) {
    ens.validate(false);
    if (workers < 1) throw ConfigError("propagate_ensemble: workers >= 1");
    std::unique_ptr<Stepper> probe = factory();
    if (auto* sqg = dynamic_cast<SqgStepper*>(probe.get())) {
        SqgModel batched(sqg->model().grid(), sqg->model().params(), ens.size());
        return propagate_batched(ens, hours, batched, max_cfl_out);
    }
    // a foreign Stepper: members in order through one instance
    Ensemble out = ens;
    for (int j = 0; j < ens.size(); ++j) {
        try {
            probe->advance(out.members[size_t(j)], hours);
        } catch (const BlowupError& e) {
            throw BlowupError(e.time_hours, j);
        }
    }
    if (max_cfl_out) *max_cfl_out = probe->max_cfl();
    out.valid_time = ens.valid_time + hours;
    return out;
}

Ensemble inject_model_error(const Ensemble& ens, const ModelErrorConfig& cfg, std::uint64_t cycle) {
    cfg.validate();
    if (!cfg.enabled) return ens;
    ens.validate(false);
    Ensemble out = ens;
    // cumulative category bounds, drawn in order from the member's stream
    std::vector<double> bound;
    double acc = 0.0;
    for (const auto& c : cfg.mixture) bound.push_back(acc += c.first);
    for (int j = 0; j < ens.size(); ++j) {
        RngStream rng(ens.member_seeds[size_t(j)], StreamUse::model_error, cycle);
        for (double& v : out.members[size_t(j)]) {
            const double u = rng.uniform();
            const auto hit = std::upper_bound(bound.begin(), bound.end(), u);
            if (hit != bound.end())
                v += cfg.mixture[size_t(hit - bound.begin())].second * cfg.base_amplitude * rng.normal();
        }
    }
    return out;
}

double climatological_amplitude(const std::vector<std::vector<double>>& trajectory) {
    if (trajectory.empty()) throw DimensionError("climatological_amplitude: empty trajectory");
    double ss = 0.0;
    std::size_t n = 0;
    for (const auto& s : trajectory) {
        ss = std::inner_product(s.begin(), s.end(), s.begin(), ss);
        n += s.size();
    }
    if (n == 0) throw DimensionError("climatological_amplitude: empty states");
    return std::sqrt(ss / double(n));
}

// ----------------------------------------------------------------- osse -----
std::string variant_name(Variant v) {
    static const char* names[] = {"free_run", "letkf", "ensf"};
    const int i = int(v);
    if (i < 0 || i > 2) throw ConfigError("unknown variant");
    return names[i];
}

Variant variant_from_name(const std::string& name) {
    for (Variant v : {Variant::free_run, Variant::letkf, Variant::ensf})
        if (variant_name(v) == name) return v;
    throw ConfigError("unknown variant '" + name + "'");
}

std::string quality_name(ModelQuality q) { return q == ModelQuality::perfect ? "perfect" : "imperfect"; }

ModelQuality quality_from_name(const std::string& name) {
    if (name == "perfect") return ModelQuality::perfect;
    if (name == "imperfect") return ModelQuality::imperfect;
    throw ConfigError("unknown model quality '" + name + "'");
}

void ExperimentConfig::validate() const {
    grid.validate();
    sqg.validate();
    ensf.validate();
    letkf.validate();
    model_error.validate();
    obs.validate();
    if (cycles < 1) throw ConfigError("cycles >= 1");
    if (!(obs_interval > 0.0)) throw ConfigError("obs_interval > 0");
    long steps = 0;
    if (!whole_steps(obs_interval, sqg.dt, &steps))
        throw ConfigError("obs_interval must be a multiple of dt");
    if (ensemble_size < 1) throw ConfigError("ensemble_size >= 1");
    if (spinup_hours < 0.0) throw ConfigError("spinup_hours >= 0");
    if (clim_hours < 0.0) throw ConfigError("clim_hours >= 0");
    if (ensemble_size > int(std::llround(clim_hours / obs_interval)) + 1)
        throw ConfigError("climatology too short for ensemble_size");
    if (fit_lo_shell < 1 || fit_hi_shell <= fit_lo_shell) throw ConfigError("fit shell range invalid");
}

namespace {

std::string num17(double x) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", x);
    return buf;
}

}  // namespace

std::string MetricsSeries::to_csv() const {
    std::string out = "time,forecast_rmse,analysis_rmse,spread\n";
    for (const CycleRecord& r : records)
        out += num17(r.time) + ',' + num17(r.forecast_rmse) + ',' + num17(r.analysis_rmse) + ',' +
               num17(r.analysis_spread) + '\n';
    return out;
}

std::vector<std::vector<double>> nature_run(const GridSpec& grid, const SqgParams& params,
                                            double spinup, double duration, double obs_interval,
                                            std::uint64_t seed) {
    grid.validate();
    params.validate();
    if (spinup < 0.0 || duration < 0.0) throw ConfigError("nature_run: negative duration");
    if (!(obs_interval > 0.0)) throw ConfigError("nature_run: obs_interval > 0");
    const int n_snap = int(std::llround(duration / obs_interval)) + 1;
    const std::size_t d = grid.grid_size();
    std::vector<double> flat(d * size_t(n_snap));
    const turbda_sqg_params a = to_abi(grid, params);
    int32_t got = 0;
    turbda_status st{};
    if (int rc = turbda_nature_run(&a, spinup, duration, obs_interval, seed, flat.data(), n_snap,
                                   &got, -1, &st))
        raise_sqg(rc, st);
    std::vector<std::vector<double>> snaps(static_cast<size_t>(got));
    for (int k = 0; k < got; ++k)
        snaps[size_t(k)].assign(flat.begin() + std::ptrdiff_t(size_t(k) * d),
                                flat.begin() + std::ptrdiff_t(size_t(k + 1) * d));
    return snaps;
}

TruthBundle make_truth_bundle(const ExperimentConfig& cfg) {
    cfg.validate();
    // climatology first, the verification trajectory one interval after its
    // last snapshot (proj/src/osse.cpp:137-153): the pools never overlap
    const double duration = cfg.clim_hours + cfg.obs_interval * double(cfg.cycles + 1);
    auto snaps = nature_run(cfg.grid, cfg.sqg, cfg.spinup_hours, duration, cfg.obs_interval, cfg.seed);
    const auto n_clim = std::ptrdiff_t(std::llround(cfg.clim_hours / cfg.obs_interval)) + 1;
    TruthBundle b;
    b.climatology.assign(std::make_move_iterator(snaps.begin()),
                         std::make_move_iterator(snaps.begin() + n_clim));
    b.truth.assign(std::make_move_iterator(snaps.begin() + n_clim),
                   std::make_move_iterator(snaps.end()));
    b.base_amplitude = climatological_amplitude(b.climatology);
    return b;
}

Ensemble initial_ensemble(const std::vector<std::vector<double>>& climatology, int m,
                          std::uint64_t seed) {
    const int n = int(climatology.size());
    if (m < 1) throw ConfigError("initial_ensemble: m >= 1");
    if (m > n) throw ConfigError("initial_ensemble: not enough snapshots");
    // the first m entries of a partial Fisher-Yates shuffle (init_select stream)
    std::vector<int> order(static_cast<size_t>(n));
    std::iota(order.begin(), order.end(), 0);
    RngStream pick(seed, StreamUse::init_select, 0);
    Ensemble e;
    e.valid_time = 0.0;
    for (int i = 0; i < m; ++i) {
        std::swap(order[size_t(i)], order[size_t(i) + size_t(pick.next_u64() % std::uint64_t(n - i))]);
        e.members.push_back(climatology[size_t(order[size_t(i)])]);
        e.member_seeds.push_back(RngStream(seed, StreamUse::member_seed, std::uint64_t(i)).next_u64());
    }
    return e;
}

MetricsSeries run_experiment(const ExperimentConfig& cfg, const TruthBundle* bundle,
                             const CycleCallback& on_cycle, int workers, double* max_cfl_out,
                             MetricsSeries* partial_out) {
    cfg.validate();
    TruthBundle own;
    if (!bundle) {
        own = make_truth_bundle(cfg);
        bundle = &own;
    }
    if (bundle->truth.size() < size_t(cfg.cycles) + 1)
        throw ConfigError("truth bundle shorter than experiment");
    ModelErrorConfig me = cfg.model_error;
    if (!(me.base_amplitude > 0.0)) me.base_amplitude = bundle->base_amplitude;
    const ObsOperator op = make_grid_operator(cfg.grid, cfg.obs.thinning_stride);

    Ensemble ens = initial_ensemble(bundle->climatology, cfg.ensemble_size, cfg.seed);
    SqgModel model(cfg.grid, cfg.sqg, cfg.ensemble_size);  // one batched model for all cycles
    MetricsSeries metrics;
    double max_cfl = 0.0;
    for (int k = 1; k <= cfg.cycles; ++k) {
        try {
            double cfl = 0.0;
            ens = propagate_batched(ens, cfg.obs_interval, model, &cfl);
            max_cfl = std::max(max_cfl, cfl);
            if (cfg.model_quality == ModelQuality::imperfect)
                ens = inject_model_error(ens, me, std::uint64_t(k));
            const std::vector<double>& truth = bundle->truth[size_t(k)];
            CycleRecord rec;
            rec.cycle = k;
            rec.time = double(k) * cfg.obs_interval;
            rec.forecast_rmse = rmse(ensemble_mean(ens), truth);
            rec.forecast_spread = spread(ens);
            if (cfg.variant == Variant::free_run) {
                rec.analysis_rmse = rec.forecast_rmse;
                rec.analysis_spread = rec.forecast_spread;
            } else {
                const Observation obs = synthesize_observations(truth, cfg.grid, op, cfg.obs.r,
                                                                rec.time, cfg.seed, std::uint64_t(k));
                ens = cfg.variant == Variant::letkf
                          ? letkf_analyze(ens, obs, cfg.letkf, cfg.grid, workers)
                          : analyze(ens, obs, cfg.ensf, cfg.seed, std::uint64_t(k), workers);
                rec.analysis_rmse = rmse(ensemble_mean(ens), truth);
                rec.analysis_spread = spread(ens);
            }
            metrics.records.push_back(rec);
            if (on_cycle) on_cycle(rec, ens);
        } catch (const RunAbortedError&) {
            throw;
        } catch (const std::exception& e) {
            if (partial_out) *partial_out = metrics;
            throw RunAbortedError(k, e.what());
        }
    }
    if (max_cfl_out) *max_cfl_out = max_cfl;
    if (partial_out) *partial_out = metrics;
    return metrics;
}

}  // namespace turbda
