// TEST INFRASTRUCTURE ONLY - stand-in for proj/include/turbda/osse.hpp (see
// forecast.hpp in this directory): declares nature_run, which
// proj/tests/helpers.hpp references from an inline helper the hot-path tests
// never call.
#pragma once
#include <cstdint>
#include <vector>

#include "turbda/ensf.hpp"
#include "turbda/forecast.hpp"

namespace turbda {
std::vector<std::vector<double>> nature_run(const GridSpec& grid, const SqgParams& params,
                                            double spinup, double duration, double obs_interval,
                                            std::uint64_t seed);
}  // namespace turbda
