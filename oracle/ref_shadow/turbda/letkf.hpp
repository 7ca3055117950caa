// TEST INFRASTRUCTURE ONLY - stand-in for proj/include/turbda/letkf.hpp so
// the reference's cycle driver (proj/src/osse.cpp, proj/src/config.cpp)
// compiles without Eigen.  LetkfConfig matches the reference
// (proj/include/turbda/letkf.hpp:12-27); letkf_analyze / rtps_inflate /
// gaspari_cohn are the Eigen-free restatement in oracle/letkf_restated.cpp.
#pragma once
#include <cstdint>

#include "turbda/ensemble.hpp"
#include "turbda/grid.hpp"
#include "turbda/observation.hpp"

namespace turbda {

struct LetkfConfig {
    double cutoff_km = 2000.0;
    double domain_km = 20000.0;
    double rtps_alpha = 0.3;
    int obs_thinning = 0;

    void validate() const {
        if (!(cutoff_km > 0.0) || !(domain_km > 0.0))
            throw ConfigError("letkf: cutoff_km, domain_km > 0");
        if (rtps_alpha < 0.0 || rtps_alpha > 1.0)
            throw ConfigError("letkf: rtps_alpha in [0, 1]");
        if (obs_thinning < 0) throw ConfigError("letkf: obs_thinning >= 0");
    }
};

double gaspari_cohn(double r);
Ensemble letkf_analyze(const Ensemble& forecast, const Observation& obs,
                       const LetkfConfig& cfg, const GridSpec& grid, int workers = 0);
Ensemble rtps_inflate(const Ensemble& analysis, const Ensemble& background, double alpha);

}  // namespace turbda
