// TEST INFRASTRUCTURE ONLY - stand-in for proj/include/turbda/forecast.hpp so
// proj/tests/helpers.hpp compiles against the B200 headers.  The forecast
// model (SQG, FFTW) is out of scope; only the names helpers.hpp mentions
// exist, and nothing here is ever called by the hot-path tests.
#pragma once
#include <cstdint>
#include <vector>

#include "turbda/ensemble.hpp"
#include "turbda/grid.hpp"

namespace turbda {
struct SqgParams {
    double f = 1.0;
};
}  // namespace turbda
