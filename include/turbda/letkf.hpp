// LETKF arm of the turbda API (reference: proj/include/turbda/letkf.hpp:11-56)
// without the Eigen types: gaspari_cohn, letkf_analyze and rtps_inflate keep
// the reference's names, arguments and exceptions and run on the GPU through
// turbda_letkf_analyze / turbda_rtps_inflate (include/turbda_b200.h).  The
// Eigen-typed helper etkf_local_analysis is not part of this build: the
// per-point transform lives inside the GPU kernel.
#pragma once

#include "turbda/ensemble.hpp"
#include "turbda/errors.hpp"
#include "turbda/grid.hpp"
#include "turbda/observation.hpp"

namespace turbda {

struct LetkfConfig {
    // working cutoff in grid units: cutoff_km / domain_km * nx
    double cutoff_km = 2000.0;
    double domain_km = 20000.0;
    double rtps_alpha = 0.3;
    int obs_thinning = 0;

    void validate() const {
        if (!(cutoff_km > 0.0) || !(domain_km > 0.0))
            throw ConfigError("letkf: cutoff_km, domain_km > 0");
        if (rtps_alpha < 0.0 || rtps_alpha > 1.0) throw ConfigError("letkf: rtps_alpha in [0, 1]");
        if (obs_thinning < 0) throw ConfigError("letkf: obs_thinning >= 0");
    }
};

// 5th-order Gaspari-Cohn correlation at normalized distance r, support [0, 2]
double gaspari_cohn(double r);

// localized ETKF per grid point (both levels share the transform), then
// RTPS; SingularAnalysisError(ix, iy) for a non-positive local eigenvalue.
// `workers` is accepted for signature compatibility (the GPU grid decides).
Ensemble letkf_analyze(const Ensemble& forecast, const Observation& obs, const LetkfConfig& cfg,
                       const GridSpec& grid, int workers = 0);

// deviations scaled per variable by 1 + alpha (sigma_b - sigma_a) / sigma_a
Ensemble rtps_inflate(const Ensemble& analysis, const Ensemble& background, double alpha);

}  // namespace turbda
