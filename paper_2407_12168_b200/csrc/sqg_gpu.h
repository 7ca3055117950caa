// Internal: batched GPU SQG model (sqg_gpu.cu) used by the C-ABI's
// turbda_sqg_* and turbda_run_experiment.
#pragma once
#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

namespace tb200 {

// proj/include/turbda/sqg.hpp:17-37 + the grid of proj/include/turbda/grid.hpp
struct SqgConfig {
    int nx = 64, ny = 64;
    double lx = 62.83185307179586, ly = 62.83185307179586, h = 0.3;
    double f = 1.0, n = 10.0, u0 = 0.1;
    int hyper_order = 4;
    double hyper_efold = 5.0, dt = 0.25, drag_tau = 200.0;
};

class SqgGpu {
public:
    struct Impl;
    SqgGpu();
    ~SqgGpu();
    // "" on success
    std::string init(const SqgConfig& cfg, int batch);
    int batch() const;
    size_t state_size() const;  // 2 * ny * nx
    // forward transform, 2/3 dealias, inverse (nature_run's IC filter)
    std::string dealias(double* states, cudaStream_t st);
    // states: device [batch][2][ny][nx], advanced in place by `hours` (a
    // multiple of dt).  "config:..." prefixes a ConfigError.  On a
    // non-finite state *blown_member / *blown_hours report the first one.
    std::string advance(double* states, double hours, cudaStream_t st, double* max_cfl,
                        int* blown_member, double* blown_hours);
    // shell-summed kinetic energy of one device state [2][ny][nx]
    std::string ke_spectrum(const double* state, cudaStream_t st, std::vector<double>* kappa,
                            std::vector<double>* energy);

private:
    std::unique_ptr<Impl> impl_;
};

}  // namespace tb200
