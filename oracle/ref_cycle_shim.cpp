// TEST INFRASTRUCTURE ONLY - C-ABI over the reference's *unmodified* cycle
// driver and SQG model, built with cuFFTW in place of FFTW (oracle/Makefile
// `ref-cycle`, output oracle/_ref/libturbda_ref_cycle.so; needs a GPU at run
// time because cuFFTW runs on cuFFT).  Entry points:
//   refc_run_experiment -> turbda::run_experiment  proj/src/osse.cpp:182-253
//                          (JSON config: turbda::config_from_json, proj/src/config.cpp:64-131)
//   refc_sqg_advance    -> turbda::SqgStepper::advance proj/src/forecast.cpp:14-32
//   refc_nature_run     -> turbda::nature_run      proj/src/osse.cpp:101-135
//   refc_snapshot_write -> turbda::write_snapshot  proj/src/snapshot.cpp:12-30
//   refc_snapshot_read  -> turbda::read_snapshot   proj/src/snapshot.cpp:32-63
//   refc_letkf_analyze  -> turbda::letkf_analyze   (proj/src/letkf.cpp
//                          unmodified over the Eigen subset in
//                          oracle/ref_shadow/Eigen/Dense; the cycle driver's
//                          "letkf" variant calls the same function)
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "turbda/config.hpp"
#include "turbda/forecast.hpp"
#include "turbda/osse.hpp"
#include "turbda/snapshot.hpp"


using namespace turbda;

namespace {
void put(char* msg, int len, const char* what) {
    if (msg && len > 0) {
        std::strncpy(msg, what, size_t(len - 1));
        msg[len - 1] = 0;
    }
}
GridSpec grid_of(int nx, int ny, double lx, double ly, double h) {
    GridSpec g;
    g.nx = nx;
    g.ny = ny;
    g.lx = lx;
    g.ly = ly;
    g.h = h;
    return g;
}
}  // namespace

extern "C" {

// records: [max_records][6] = cycle, time, forecast_rmse, analysis_rmse,
// forecast_spread, analysis_spread
int refc_run_experiment(const char* config_json, int workers, double* records, int max_records,
                        int* n_records, char* msg, int msglen) {
    try {
        const ExperimentConfig cfg = config_from_json(nlohmann::json::parse(config_json));
        MetricsSeries partial;
        const MetricsSeries ms = run_experiment(cfg, nullptr, {}, workers, nullptr, &partial);
        int n = 0;
        for (const auto& r : ms.records) {
            if (n >= max_records) break;
            double* o = records + 6 * n;
            o[0] = r.cycle;
            o[1] = r.time;
            o[2] = r.forecast_rmse;
            o[3] = r.analysis_rmse;
            o[4] = r.forecast_spread;
            o[5] = r.analysis_spread;
            ++n;
        }
        *n_records = n;
        return 0;
    } catch (const std::exception& e) {
        put(msg, msglen, e.what());
        return 1;
    }
}

int refc_sqg_advance(int nx, int ny, double lx, double ly, double h, double dt, double hours,
                     const double* state, double* out, double* max_cfl, char* msg, int msglen) {
    try {
        SqgParams p;
        p.dt = dt;
        SqgStepper st(grid_of(nx, ny, lx, ly, h), p);
        std::vector<double> v(state, state + size_t(2) * nx * ny);
        st.advance(v, hours);
        std::memcpy(out, v.data(), v.size() * sizeof(double));
        if (max_cfl) *max_cfl = st.max_cfl();
        return 0;
    } catch (const std::exception& e) {
        put(msg, msglen, e.what());
        return 1;
    }
}

int refc_nature_run(int nx, int ny, double lx, double ly, double h, double spinup,
                    double duration, double interval, uint64_t seed, double* out, int max_snaps,
                    int* n_snaps, char* msg, int msglen) {
    try {
        const auto snaps =
            nature_run(grid_of(nx, ny, lx, ly, h), SqgParams{}, spinup, duration, interval, seed);
        int n = 0;
        for (const auto& s : snaps) {
            if (n >= max_snaps) break;
            std::memcpy(out + size_t(n) * s.size(), s.data(), s.size() * sizeof(double));
            ++n;
        }
        *n_snaps = n;
        return 0;
    } catch (const std::exception& e) {
        put(msg, msglen, e.what());
        return 1;
    }
}

int refc_snapshot_write(const char* path, const double* state, int nx, int ny, double time_hours,
                        char* msg, int msglen) {
    try {
        GridSpec g;
        g.nx = nx;
        g.ny = ny;
        write_snapshot(std::string(path), PhysicalField(g, std::vector<double>(state, state + g.grid_size())),
                       time_hours);
        return 0;
    } catch (const std::exception& e) {
        put(msg, msglen, e.what());
        return 1;
    }
}

// out: at least max_n doubles; *n = values read
int refc_snapshot_read(const char* path, double* out, long max_n, long* n, int* nx, int* ny,
                       double* time_hours, char* msg, int msglen) {
    try {
        const Snapshot s = read_snapshot(std::string(path));
        *nx = s.field.grid.nx;
        *ny = s.field.grid.ny;
        *time_hours = s.time_hours;
        *n = long(s.field.data.size());
        if (*n > max_n) throw IoError("buffer too small");
        std::memcpy(out, s.field.data.data(), sizeof(double) * s.field.data.size());
        return 0;
    } catch (const std::exception& e) {
        put(msg, msglen, e.what());
        return 1;
    }
}

// forecast / out: [m][2 nx ny]; idx == nullptr: identity operator
int refc_letkf_analyze(const double* forecast, int m, int nx, int ny, const double* y,
                       const double* r, const int64_t* idx, int64_t nobs, double cutoff_km,
                       double domain_km, double rtps_alpha, int workers, double* out, char* msg,
                       int msglen) {
    try {
        GridSpec g;
        g.nx = nx;
        g.ny = ny;
        g.lx = g.ly = 62.83185307179586 * (nx / 64.0);
        const size_t d = g.grid_size();
        Ensemble ens;
        ens.valid_time = 0.0;
        for (int j = 0; j < m; ++j) {
            ens.members.emplace_back(forecast + size_t(j) * d, forecast + size_t(j + 1) * d);
            ens.member_seeds.push_back(uint64_t(j) + 1);
        }
        Observation obs;
        if (idx) {
            obs.op = ObsOperator{ObsOperatorKind::index_selection, d,
                                 std::vector<std::size_t>(idx, idx + nobs)};
        } else {
            obs.op = ObsOperator{ObsOperatorKind::identity, d, {}};
        }
        obs.locations = operator_locations(g, obs.op);
        obs.y.assign(y, y + nobs);
        obs.r_diag.assign(r, r + nobs);
        obs.time = 0.0;
        LetkfConfig cfg;
        cfg.cutoff_km = cutoff_km;
        cfg.domain_km = domain_km;
        cfg.rtps_alpha = rtps_alpha;
        const Ensemble an = letkf_analyze(ens, obs, cfg, g, workers);
        for (int j = 0; j < m; ++j)
            std::memcpy(out + size_t(j) * d, an.members[size_t(j)].data(), sizeof(double) * d);
        return 0;
    } catch (const std::exception& e) {
        put(msg, msglen, e.what());
        return 1;
    }
}

}  // extern "C"
