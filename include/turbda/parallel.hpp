// Host worker utilities of the turbda API (reference: proj/include/turbda/parallel.hpp:9-18).
// The analysis itself runs on the GPU grid and ignores `workers`; these remain
// for callers that parallelise host work the way the reference does.
#pragma once

#include <cstddef>
#include <functional>

namespace turbda {

// TURBDA_WORKERS when set to >= 1, else the hardware thread count
int default_worker_count();

// static block partition of [0, n) over `workers` threads; the exception of
// the lowest failing index is rethrown on the caller
void parallel_for(std::size_t n, int workers, const std::function<void(std::size_t)>& fn);

}  // namespace turbda
