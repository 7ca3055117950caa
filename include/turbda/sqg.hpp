// Two-boundary SQG forecast model of the turbda API on the GPU (reference:
// proj/include/turbda/sqg.hpp:17-37 for SqgParams).  SqgModel here is the
// forecast surface of the reference class (grid, params, CFL tracking) over
// a batch of states advanced together on the device (batched fp64 cuFFT,
// integrating-factor RK4 captured as a CUDA graph, csrc/sqg_gpu.cu via the
// C-ABI turbda_sqg_*), plus the kinetic-energy spectrum and its log-log
// slope fit (proj/src/sqg.cpp:306-357).  The reference's remaining spectral
// internals (forward_transform, tendency, ...) are not part of this build.
#pragma once

#include <cstdint>
#include <vector>

#include "turbda/errors.hpp"
#include "turbda/grid.hpp"

namespace turbda {

struct SqgParams {
    double f = 1.0;    // Coriolis
    double n = 10.0;   // buoyancy frequency
    double u0 = 0.1;   // shear velocity difference across the layer
    int hyper_order = 4;
    double hyper_efold = 5.0;  // e-folding time (hours) of the cutoff mode
    double dt = 0.25;          // hours
    double drag_tau = 200.0;   // Rayleigh drag timescale (hours); 0 = off
    double dealias_fraction = 2.0 / 3.0;

    void validate() const {
        if (f <= 0 || n <= 0 || u0 < 0 || hyper_efold <= 0 || dt <= 0)
            throw ConfigError("sqg: f, n, hyper_efold, dt must be positive");
        if (hyper_order < 1) throw ConfigError("sqg: hyper_order >= 1");
        if (drag_tau < 0) throw ConfigError("sqg: drag_tau >= 0");
        if (dealias_fraction != 2.0 / 3.0) throw ConfigError("sqg: dealias_fraction is fixed at 2/3");
    }

    bool operator==(const SqgParams&) const = default;
};

struct KeBin {
    double kappa;
    double energy;
};

// least-squares log-log slope over shells [lo_shell, hi_shell] (zero bins
// skipped); ConfigError when fewer than two usable bins remain
double fit_loglog_slope(const std::vector<KeBin>& spectrum, int lo_shell, int hi_shell);

class SqgModel {
public:
    // `batch` states of [2][ny][nx] advanced together on `device` (-1: current)
    SqgModel(const GridSpec& grid, const SqgParams& params, int batch = 1, int device = -1);
    ~SqgModel();
    SqgModel(const SqgModel&) = delete;
    SqgModel& operator=(const SqgModel&) = delete;

    // states: host [batch][2 ny nx], advanced in place by `hours` (a
    // non-negative multiple of dt; 0 is the exact identity).  ConfigError
    // for other durations; BlowupError(t, member) on a non-finite state.
    void advance(double* states, double hours);

    // shell-summed kinetic energy of ONE host state [2 ny nx] (bins at
    // kappa = s 2 pi / lx); ConfigError unless lx == ly
    std::vector<KeBin> ke_spectrum(const double* state);

    double max_cfl() const { return max_cfl_; }
    void reset_cfl() { max_cfl_ = 0.0; }
    const GridSpec& grid() const { return grid_; }
    const SqgParams& params() const { return params_; }
    int batch() const { return batch_; }

private:
    GridSpec grid_;
    SqgParams params_;
    int batch_ = 1;
    void* handle_ = nullptr;
    double max_cfl_ = 0.0;
};

}  // namespace turbda
