// C-ABI of the GPU forecast model and the GPU-resident cycle driver
// (SURVEY.md 8(f) ranks 1-2): turbda_sqg_* (SqgStepper / nature_run,
// proj/src/forecast.cpp, proj/src/osse.cpp:101-135) and
// turbda_run_experiment (run_experiment, proj/src/osse.cpp:182-253 with
// make_truth_bundle :137-153 and initial_ensemble :155-180).  Every cycle
// stays on the device: forecast (batched SQG), model error, observation
// synthesis, the EnSF analysis (turbda_ensf_analyze in device mode) and the
// rmse/spread diagnostics; only the six metrics per cycle come back.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "ensf_device.h"
#include "host_rng.h"
#include "philox.cuh"
#include "reduce.cuh"
#include "sqg_gpu.h"
#include "turbda_b200.h"

using namespace tb200;

namespace {

constexpr uint64_t kUseNatureIc = 1, kUseInitSelect = 2, kUseMemberSeed = 3,
                   kUseModelError = 4, kUseObsNoise = 5;

int fail(turbda_status* st, int code, const std::string& msg) {
    if (st) {
        st->code = code;
        std::snprintf(st->msg, sizeof(st->msg), "%s", msg.c_str());
    }
    return code;
}

void clear(turbda_status* st) {
    if (!st) return;
    std::memset(st, 0, sizeof(*st));
    st->diverged_particle = -1;
    st->diverged_step = -1;
    st->diverged_t = std::nan("");
}

#define CY_CUDA(call)                                                                  \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess)                                                         \
            return fail(st, TURBDA_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

SqgConfig to_cfg(const turbda_sqg_params* p) {
    SqgConfig c;
    c.nx = p->nx;
    c.ny = p->ny;
    c.lx = p->lx;
    c.ly = p->ly;
    c.h = p->h;
    c.f = p->f;
    c.n = p->n;
    c.u0 = p->u0;
    c.hyper_order = p->hyper_order;
    c.hyper_efold = p->hyper_efold;
    c.dt = p->dt;
    c.drag_tau = p->drag_tau;
    return c;
}

bool pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

// GridSpec::validate + SqgParams::validate (proj/include/turbda/grid.hpp:35-41,
// proj/include/turbda/sqg.hpp:27-35)
int validate_sqg(const turbda_sqg_params* p, turbda_status* st) {
    if (!pow2(p->nx) || !pow2(p->ny) || p->nx < 8 || p->ny < 8)
        return fail(st, TURBDA_CONFIG, "grid: nx, ny must be powers of two >= 8");
    if (!(p->lx > 0) || !(p->ly > 0) || !(p->h > 0))
        return fail(st, TURBDA_CONFIG, "grid: lx, ly, h must be positive");
    if (!(p->f > 0) || !(p->n > 0) || p->u0 < 0 || !(p->hyper_efold > 0) || !(p->dt > 0))
        return fail(st, TURBDA_CONFIG, "sqg: f, n, hyper_efold, dt must be positive");
    if (p->hyper_order < 1) return fail(st, TURBDA_CONFIG, "sqg: hyper_order >= 1");
    if (p->drag_tau < 0) return fail(st, TURBDA_CONFIG, "sqg: drag_tau >= 0");
    return TURBDA_OK;
}

int sqg_error(const std::string& e, turbda_status* st) {
    if (e.rfind("config:", 0) == 0) return fail(st, TURBDA_CONFIG, e.substr(7));
    return fail(st, TURBDA_CUDA, e);
}

// --- device helpers of the cycle -------------------------------------------

// y_q = h(truth[idx_q]) + sd * normal #q of RngStream(seed, obs_noise, cycle)
// (synthesize_observations, proj/src/observation.cpp:62-81)
__global__ void synth_obs_kernel(const double* __restrict__ truth, const int64_t* __restrict__ idx,
                                 int64_t nobs, int arctan, double sd, uint32_t k0, uint32_t k1,
                                 uint64_t cycle, double* __restrict__ y) {
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= nobs) return;
    double v = truth[idx ? idx[q] : q];
    if (arctan) v = atan(v);
    y[q] = v + sd * normal_f64(uint64_t(q), uint32_t(cycle), uint32_t(cycle >> 32), k0, k1);
}

// Sequential restatement of one RngStream (proj/src/rng.cpp:40-84) on the device.
struct DevStream {
    uint32_t k0, k1, e0, e1;
    uint64_t block = 0;
    uint32_t buf[4];
    int pos = 4;
    double spare = 0.0;
    bool has_spare = false;
    __device__ uint32_t u32() {
        if (pos >= 4) {
            const PhiloxOut w = philox_block(block, e0, e1, k0, k1);
            buf[0] = w.w0;
            buf[1] = w.w1;
            buf[2] = w.w2;
            buf[3] = w.w3;
            ++block;
            pos = 0;
        }
        return buf[pos++];
    }
    __device__ double uniform() {
        const uint64_t lo = u32();
        const uint64_t v = lo | (uint64_t(u32()) << 32);
        return (double(v >> 11) + 0.5) * 0x1.0p-53;
    }
    __device__ double normal() {
        if (has_spare) {
            has_spare = false;
            return spare;
        }
        const double u1 = uniform(), u2 = uniform();
        const double r = sqrt(-2.0 * log(u1));
        const double a = 2.0 * 3.14159265358979323846 * u2;
        double s, c;
        sincos(a, &s, &c);
        spare = r * s;
        has_spare = true;
        return r * c;
    }
};

// inject_model_error (proj/src/forecast.cpp:77-100): per member a sequential
// stream (the draw count depends on the categories hit), one thread each
__global__ void model_error_kernel(double* __restrict__ x, int m, int64_t d,
                                   const unsigned long long* __restrict__ member_keys,
                                   uint64_t cycle, int ncomp, const double* __restrict__ prob,
                                   const double* __restrict__ frac, double base) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    DevStream rs;
    rs.k0 = uint32_t(member_keys[j]);
    rs.k1 = uint32_t(member_keys[j] >> 32);
    rs.e0 = uint32_t(cycle);
    rs.e1 = uint32_t(cycle >> 32);
    double* row = x + size_t(j) * size_t(d);
    for (int64_t i = 0; i < d; ++i) {
        const double u = rs.uniform();
        double acc = 0.0;
        for (int c = 0; c < ncomp; ++c) {
            acc += prob[c];
            if (u < acc) {
                row[i] += frac[c] * base * rs.normal();
                break;
            }
        }
    }
}

// sum of squares of the climatology (model-error base amplitude,
// proj/src/forecast.cpp:77-100) in a fixed order: one partial per CTA of a
// fixed grid, summed in CTA order (reduce.cuh)
constexpr int kSumSqBlocks = 592;
__global__ void __launch_bounds__(256) sum_squares_kernel(const double* __restrict__ x, size_t n,
                                                          double* __restrict__ part) {
    double s = 0.0;
    for (size_t q = size_t(blockIdx.x) * blockDim.x + threadIdx.x; q < n; q += size_t(gridDim.x) * blockDim.x)
        s += x[q] * x[q];
    block_sum2_to(s, 0.0, part + 2 * blockIdx.x);
}

struct DeviceBuffer {
    void* p = nullptr;
    ~DeviceBuffer() { cudaFree(p); }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

// nature_run (proj/src/osse.cpp:101-135) into device snapshots [n_snap][d]
int nature_run_device(const turbda_sqg_params* p, double spinup, double duration,
                      double interval, uint64_t seed, DeviceBuffer& snaps, int* n_snap,
                      double* max_cfl, cudaStream_t s, turbda_status* st) {
    const SqgConfig c = to_cfg(p);
    const size_t d = size_t(2) * c.nx * c.ny;
    *n_snap = int(std::llround(duration / interval)) + 1;
    CY_CUDA(cudaMalloc(&snaps.p, sizeof(double) * d * size_t(*n_snap)));
    // small random IC (RngStream(seed, nature_ic, 0), 0.1 N(0,1)), dealiased
    std::vector<double> ic(d);
    {
        HostStream rs(seed, kUseNatureIc, 0);
        // RngStream::normal with cached pairs == normals #0, #1, ... of the stream
        for (size_t q = 0; q < d; q += 2) {
            const uint64_t a = rs.next_u64(), b = rs.next_u64();
            const double u1 = (double(a >> 11) + 0.5) * 0x1.0p-53;
            const double u2 = (double(b >> 11) + 0.5) * 0x1.0p-53;
            const double r = std::sqrt(-2.0 * std::log(u1));
            const double ang = 2.0 * 3.14159265358979323846 * u2;
            ic[q] = 0.1 * (r * std::cos(ang));
            if (q + 1 < d) ic[q + 1] = 0.1 * (r * std::sin(ang));
        }
    }
    SqgGpu model;
    std::string err = model.init(c, 1);
    if (!err.empty()) return sqg_error(err, st);
    double* state = snaps.as<double>();  // snapshot 0 doubles as the working state
    CY_CUDA(cudaMemcpyAsync(state, ic.data(), sizeof(double) * d, cudaMemcpyHostToDevice, s));
    // forward -> dealias -> inverse of the IC is one zero-length-free call:
    // advance by 0 is the identity in the reference, so dealias explicitly
    err = model.dealias(state, s);
    if (!err.empty()) return sqg_error(err, st);
    int blown = -1;
    double bh = 0.0, elapsed = 0.0;
    // BlowupError(t) of the single nature-run stepper, t = model hours since its start
    const auto blowup = [&]() {
        char buf[96];
        std::snprintf(buf, sizeof buf, "integration blowup (NaN/Inf) at t=%f h", elapsed + bh);
        if (st) st->diverged_t = elapsed + bh;
        return fail(st, TURBDA_BLOWUP, buf);
    };
    if (spinup > 0.0) {
        err = model.advance(state, spinup, s, max_cfl, &blown, &bh);
        if (!err.empty()) return sqg_error(err, st);
        if (blown >= 0) return blowup();
        elapsed += spinup;
    }
    for (int k = 1; k < *n_snap; ++k) {
        double* dst = state + size_t(k) * d;
        CY_CUDA(cudaMemcpyAsync(dst, dst - d, sizeof(double) * d, cudaMemcpyDeviceToDevice, s));
        err = model.advance(dst, interval, s, max_cfl, &blown, &bh);
        if (!err.empty()) return sqg_error(err, st);
        if (blown >= 0) return blowup();
        elapsed += interval;
    }
    return TURBDA_OK;
}

}  // namespace

extern "C" {

void turbda_sqg_params_init(turbda_sqg_params* p) {
    std::memset(p, 0, sizeof(*p));
    p->nx = 64;
    p->ny = 64;
    p->lx = 62.83185307179586;
    p->ly = 62.83185307179586;
    p->h = 0.3;
    p->f = 1.0;
    p->n = 10.0;
    p->u0 = 0.1;
    p->hyper_order = 4;
    p->hyper_efold = 5.0;
    p->dt = 0.25;
    p->drag_tau = 200.0;
}

int turbda_sqg_create(const turbda_sqg_params* p, int32_t batch, int32_t device, void** handle,
                      turbda_status* st) {
    clear(st);
    if (int rc = validate_sqg(p, st)) return rc;
    if (batch < 1) return fail(st, TURBDA_CONFIG, "sqg: batch >= 1");
    if (device >= 0) CY_CUDA(cudaSetDevice(device));
    auto* m = new SqgGpu();
    const std::string err = m->init(to_cfg(p), batch);
    if (!err.empty()) {
        delete m;
        return sqg_error(err, st);
    }
    *handle = m;
    return TURBDA_OK;
}

int turbda_sqg_advance(void* handle, double* states, double hours, uint32_t flags, void* stream,
                       double* max_cfl, turbda_status* st) {
    clear(st);
    auto* m = static_cast<SqgGpu*>(handle);
    if (!m) return fail(st, TURBDA_CONFIG, "sqg: null handle");
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
    const size_t bytes = sizeof(double) * m->state_size() * size_t(m->batch());
    double* dptr = states;
    DeviceBuffer tmp;
    if (!(flags & TURBDA_INPUTS_ON_DEVICE)) {
        CY_CUDA(cudaMalloc(&tmp.p, bytes));
        CY_CUDA(cudaMemcpyAsync(tmp.p, states, bytes, cudaMemcpyHostToDevice, s));
        dptr = tmp.as<double>();
    }
    int blown = -1;
    double bh = 0.0;
    const std::string err = m->advance(dptr, hours, s, max_cfl, &blown, &bh);
    if (!err.empty()) return sqg_error(err, st);
    if (!(flags & TURBDA_INPUTS_ON_DEVICE)) {
        CY_CUDA(cudaMemcpyAsync(states, dptr, bytes, cudaMemcpyDeviceToHost, s));
        CY_CUDA(cudaStreamSynchronize(s));
    }
    if (blown >= 0) {
        if (st) {
            st->diverged_particle = blown;
            st->diverged_t = bh;
        }
        char buf[128];
        std::snprintf(buf, sizeof buf, "integration blowup (NaN/Inf) at t=%f h in member %d", bh, blown);
        return fail(st, TURBDA_BLOWUP, buf);
    }
    return TURBDA_OK;
}

int turbda_sqg_ke_spectrum(void* handle, const double* state, uint32_t flags, double* kappa,
                           double* energy, int32_t max_bins, int32_t* n_bins, turbda_status* st) {
    clear(st);
    auto* m = static_cast<SqgGpu*>(handle);
    if (!m) return fail(st, TURBDA_CONFIG, "sqg: null handle");
    cudaStream_t s;
    CY_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct Guard {
        cudaStream_t s;
        ~Guard() { cudaStreamDestroy(s); }
    } guard{s};
    const double* dptr = state;
    DeviceBuffer tmp;
    if (!(flags & TURBDA_INPUTS_ON_DEVICE)) {
        const size_t bytes = sizeof(double) * m->state_size();
        CY_CUDA(cudaMalloc(&tmp.p, bytes));
        CY_CUDA(cudaMemcpyAsync(tmp.p, state, bytes, cudaMemcpyHostToDevice, s));
        dptr = tmp.as<double>();
    }
    std::vector<double> k, e;
    const std::string err = m->ke_spectrum(dptr, s, &k, &e);
    if (!err.empty()) return sqg_error(err, st);
    const int n = int(k.size());
    if (n_bins) *n_bins = n;
    for (int q = 0; q < std::min(n, int(max_bins)); ++q) {
        if (kappa) kappa[q] = k[size_t(q)];
        if (energy) energy[q] = e[size_t(q)];
    }
    return TURBDA_OK;
}

// least-squares log-log slope over shells [lo, hi] (proj/src/sqg.cpp:337-357)
int turbda_fit_loglog_slope(const double* kappa, const double* energy, int32_t n, int32_t lo,
                            int32_t hi, double* slope, turbda_status* st) {
    clear(st);
    double sx = 0.0, sy = 0.0, sxx = 0.0, sxy = 0.0;
    int used = 0;
    for (int b = std::max(lo, 0); b <= hi && b < n; ++b) {
        if (!(energy[b] > 0.0) || !(kappa[b] > 0.0)) continue;  // empty bins skipped
        const double lx = std::log(kappa[b]), ly = std::log(energy[b]);
        sx += lx;
        sy += ly;
        sxx += lx * lx;
        sxy += lx * ly;
        ++used;
    }
    if (used < 2) return fail(st, TURBDA_CONFIG, "slope fit needs at least two non-empty bins");
    if (slope) *slope = (used * sxy - sx * sy) / (used * sxx - sx * sx);
    return TURBDA_OK;
}

int turbda_sqg_destroy(void* handle) {
    delete static_cast<SqgGpu*>(handle);
    return TURBDA_OK;
}

int turbda_nature_run(const turbda_sqg_params* p, double spinup, double duration, double interval,
                      uint64_t seed, double* out, int32_t max_snaps, int32_t* n_snaps,
                      int32_t device, turbda_status* st) {
    clear(st);
    if (int rc = validate_sqg(p, st)) return rc;
    if (spinup < 0.0 || duration < 0.0) return fail(st, TURBDA_CONFIG, "nature_run: negative duration");
    if (!(interval > 0.0)) return fail(st, TURBDA_CONFIG, "nature_run: obs_interval > 0");
    if (device >= 0) CY_CUDA(cudaSetDevice(device));
    cudaStream_t s;
    CY_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    DeviceBuffer snaps;
    int n = 0;
    double cfl = 0.0;
    const int rc = nature_run_device(p, spinup, duration, interval, seed, snaps, &n, &cfl, s, st);
    if (rc == TURBDA_OK) {
        const size_t d = size_t(2) * p->nx * p->ny;
        const int k = std::min(n, int(max_snaps));
        cudaMemcpyAsync(out, snaps.p, sizeof(double) * d * size_t(k), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        *n_snaps = k;
    }
    cudaStreamDestroy(s);
    return rc;
}

void turbda_experiment_init(turbda_experiment* e) {
    std::memset(e, 0, sizeof(*e));
    turbda_sqg_params_init(&e->sqg);
    e->variant = TURBDA_VARIANT_ENSF;
    e->model_quality = 0;
    e->cycles = 300;
    e->obs_interval = 12.0;
    e->ensemble_size = 20;
    e->seed = 7;
    e->spinup_hours = 7200.0;
    e->clim_hours = 2880.0;
    e->obs_r = 1.0;
    e->obs_thinning = 0;
    e->obs_arctan = 0;
    e->n_steps = 100;
    e->eps = 0.01;
    e->minibatch_j = 0;
    e->damping_t = 1.0;
    e->relax_factor = 1.0;
    e->precision = TURBDA_FP32;
    e->score_mode = TURBDA_SCORE_COMPONENTWISE;
    e->me_enabled = 1;
    e->me_base_amplitude = 0.0;
    // ModelErrorConfig default mixture, proj/include/turbda/forecast.hpp:56-58
    const double prob[4] = {0.20, 0.15, 0.10, 0.05}, frac[4] = {0.2, 0.3, 0.4, 0.5};
    e->me_ncomp = 4;
    for (int c = 0; c < 4; ++c) {
        e->me_prob[c] = prob[c];
        e->me_frac[c] = frac[c];
    }
    // LetkfConfig defaults, proj/include/turbda/letkf.hpp:13-16
    e->letkf_cutoff_km = 2000.0;
    e->letkf_domain_km = 20000.0;
    e->letkf_rtps_alpha = 0.3;
    e->letkf_obs_thinning = 0;
}

int turbda_run_experiment(const turbda_experiment* e, int32_t device, double* records,
                          int32_t max_records, int32_t* n_records, double* max_cfl,
                          double* phase_seconds, turbda_status* st) {
    return turbda_run_experiment_probe(e, device, records, max_records, n_records, max_cfl,
                                       phase_seconds, nullptr, st);
}

int turbda_run_experiment_probe(const turbda_experiment* e, int32_t device, double* records,
                                int32_t max_records, int32_t* n_records, double* max_cfl,
                                double* phase_seconds, const turbda_probe* probe,
                                turbda_status* st) {
    clear(st);
    *n_records = 0;
    if (phase_seconds)
        for (int q = 0; q < 4; ++q) phase_seconds[q] = 0.0;
    // ExperimentConfig::validate, proj/src/osse.cpp:40-62
    if (int rc = validate_sqg(&e->sqg, st)) return rc;
    if (e->variant != TURBDA_VARIANT_ENSF && e->variant != TURBDA_VARIANT_FREE_RUN &&
        e->variant != TURBDA_VARIANT_LETKF)
        return fail(st, TURBDA_CONFIG, "run_experiment: unknown variant");
    // LetkfConfig::validate (called for every variant, proj/src/osse.cpp:43)
    if (!(e->letkf_cutoff_km > 0.0) || !(e->letkf_domain_km > 0.0))
        return fail(st, TURBDA_CONFIG, "letkf: cutoff_km, domain_km > 0");
    if (!(e->letkf_rtps_alpha >= 0.0 && e->letkf_rtps_alpha <= 1.0))
        return fail(st, TURBDA_CONFIG, "letkf: rtps_alpha in [0, 1]");
    if (e->letkf_obs_thinning < 0) return fail(st, TURBDA_CONFIG, "letkf: obs_thinning >= 0");
    if (!(e->eps > 0.0 && e->eps < 1.0)) return fail(st, TURBDA_CONFIG, "ensf: eps must lie in (0, 1)");
    if (e->n_steps < 10) return fail(st, TURBDA_CONFIG, "ensf: n_steps >= 10");
    if (e->minibatch_j < 0) return fail(st, TURBDA_CONFIG, "ensf: minibatch_j >= 0");
    if (e->relax_factor < 0.0 || e->relax_factor > 1.0)
        return fail(st, TURBDA_CONFIG, "ensf: relax_factor in [0, 1]");
    if (e->me_ncomp < 0 || e->me_ncomp > 8) return fail(st, TURBDA_CONFIG, "model error: up to 8 components");
    double psum = 0.0;
    for (int c = 0; c < e->me_ncomp; ++c) {
        if (e->me_prob[c] < 0.0) return fail(st, TURBDA_CONFIG, "model error: probability >= 0");
        if (!(e->me_frac[c] > 0.0)) return fail(st, TURBDA_CONFIG, "model error: fraction > 0");
        psum += e->me_prob[c];
    }
    if (psum > 1.0 + 1e-12) return fail(st, TURBDA_CONFIG, "model error: probabilities sum to <= 1");
    if (!(e->obs_r > 0.0)) return fail(st, TURBDA_CONFIG, "obs: r > 0");
    if (e->obs_thinning < 0) return fail(st, TURBDA_CONFIG, "obs: thinning >= 0");
    if (e->cycles < 1) return fail(st, TURBDA_CONFIG, "cycles >= 1");
    if (!(e->obs_interval > 0.0)) return fail(st, TURBDA_CONFIG, "obs_interval > 0");
    const double steps = e->obs_interval / e->sqg.dt;
    if (std::abs(steps - std::llround(steps)) > 1e-9)
        return fail(st, TURBDA_CONFIG, "obs_interval must be a multiple of dt");
    if (e->ensemble_size < 1) return fail(st, TURBDA_CONFIG, "ensemble_size >= 1");
    if (e->spinup_hours < 0.0) return fail(st, TURBDA_CONFIG, "spinup_hours >= 0");
    if (e->clim_hours < 0.0) return fail(st, TURBDA_CONFIG, "clim_hours >= 0");
    const int n_clim = int(std::llround(e->clim_hours / e->obs_interval)) + 1;
    if (e->ensemble_size > n_clim) return fail(st, TURBDA_CONFIG, "climatology too short for ensemble_size");
    if (probe && (probe->n_cycles < 0 || (probe->n_cycles > 0 && (!probe->cycles || !probe->forecast ||
                                                                 !probe->analysis)) ||
                  probe->k0 < 0 || probe->width < 0 ||
                  probe->k0 + probe->width > int64_t(2) * e->sqg.nx * e->sqg.ny))
        return fail(st, TURBDA_CONFIG, "probe: window outside the state");

    if (device >= 0) CY_CUDA(cudaSetDevice(device));
    int dev = 0;
    CY_CUDA(cudaGetDevice(&dev));
    cudaStream_t s;
    CY_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() { cudaStreamDestroy(s); }
    } guard{s};

    const SqgConfig cfg = to_cfg(&e->sqg);
    const int64_t d = int64_t(2) * cfg.nx * cfg.ny;
    const int m = e->ensemble_size;
    double cfl = 0.0;
    // phase timing with events on the driver stream
    cudaEvent_t ev_a, ev_b;
    CY_CUDA(cudaEventCreate(&ev_a));
    CY_CUDA(cudaEventCreate(&ev_b));
    struct EventGuard {
        cudaEvent_t a, b;
        ~EventGuard() {
            cudaEventDestroy(a);
            cudaEventDestroy(b);
        }
    } eguard{ev_a, ev_b};
    const auto tic = [&]() { cudaEventRecord(ev_a, s); };
    const auto toc = [&](int phase) {
        cudaEventRecord(ev_b, s);
        cudaEventSynchronize(ev_b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev_a, ev_b);
        if (phase_seconds) phase_seconds[phase] += 1e-3 * ms;
    };
    tic();

    // truth bundle (make_truth_bundle, proj/src/osse.cpp:137-153)
    const double duration = e->clim_hours + e->obs_interval * double(e->cycles + 1);
    DeviceBuffer snaps;
    int n_snap = 0;
    if (int rc = nature_run_device(&e->sqg, e->spinup_hours, duration, e->obs_interval, e->seed,
                                   snaps, &n_snap, &cfl, s, st))
        return rc;
    toc(0);
    const double* clim = snaps.as<double>();
    const double* truth = clim + size_t(n_clim) * size_t(d);  // truth[k], k = 0..cycles
    double base = e->me_base_amplitude;
    if (!(base > 0.0)) {
        DeviceBuffer acc;
        CY_CUDA(cudaMalloc(&acc.p, sizeof(double) * (2 + 2 * kSumSqBlocks)));
        sum_squares_kernel<<<kSumSqBlocks, 256, 0, s>>>(clim, size_t(n_clim) * size_t(d),
                                                        acc.as<double>() + 2);
        sum_partials_kernel<<<1, 32, 0, s>>>(acc.as<double>() + 2, kSumSqBlocks, acc.as<double>());
        double ss = 0.0;
        CY_CUDA(cudaMemcpyAsync(&ss, acc.p, sizeof ss, cudaMemcpyDeviceToHost, s));
        CY_CUDA(cudaStreamSynchronize(s));
        base = std::sqrt(ss / (double(n_clim) * double(d)));
    }

    // initial ensemble (proj/src/osse.cpp:155-180): partial Fisher-Yates over
    // the climatology snapshots, member seeds from the member_seed streams
    DeviceBuffer ens, ens_out;
    CY_CUDA(cudaMalloc(&ens.p, sizeof(double) * size_t(m) * size_t(d)));
    CY_CUDA(cudaMalloc(&ens_out.p, sizeof(double) * size_t(m) * size_t(d)));
    std::vector<unsigned long long> member_keys(static_cast<size_t>(m));
    {
        std::vector<int> idx(static_cast<size_t>(n_clim));
        std::iota(idx.begin(), idx.end(), 0);
        HostStream pick(e->seed, kUseInitSelect, 0);
        for (int i = 0; i < m; ++i) {
            const int j = i + int(pick.next_u64() % uint64_t(n_clim - i));
            std::swap(idx[size_t(i)], idx[size_t(j)]);
        }
        for (int i = 0; i < m; ++i) {
            CY_CUDA(cudaMemcpyAsync(ens.as<double>() + size_t(i) * size_t(d),
                                    clim + size_t(idx[size_t(i)]) * size_t(d), sizeof(double) * size_t(d),
                                    cudaMemcpyDeviceToDevice, s));
            const uint64_t member_seed = HostStream(e->seed, kUseMemberSeed, uint64_t(i)).next_u64();
            member_keys[size_t(i)] = stream_key(member_seed, kUseModelError);
        }
    }
    // observation operator (make_grid_operator) on the device
    std::vector<int64_t> obs_idx;
    if (e->obs_thinning > 1)
        for (int64_t k = 0; k < d; k += e->obs_thinning) obs_idx.push_back(k);
    const int64_t nobs = e->obs_thinning > 1 ? int64_t(obs_idx.size()) : d;
    DeviceBuffer dy, dr, didx, dkeys, dprob, dfrac, ddiag;
    CY_CUDA(cudaMalloc(&dy.p, sizeof(double) * size_t(nobs)));
    CY_CUDA(cudaMalloc(&dr.p, sizeof(double) * size_t(nobs)));
    {
        std::vector<double> rr(size_t(nobs), e->obs_r);
        CY_CUDA(cudaMemcpyAsync(dr.p, rr.data(), sizeof(double) * size_t(nobs), cudaMemcpyHostToDevice, s));
    }
    if (!obs_idx.empty()) {
        CY_CUDA(cudaMalloc(&didx.p, sizeof(int64_t) * obs_idx.size()));
        CY_CUDA(cudaMemcpyAsync(didx.p, obs_idx.data(), sizeof(int64_t) * obs_idx.size(),
                                cudaMemcpyHostToDevice, s));
    }
    CY_CUDA(cudaMalloc(&dkeys.p, sizeof(unsigned long long) * size_t(m)));
    CY_CUDA(cudaMemcpyAsync(dkeys.p, member_keys.data(), sizeof(unsigned long long) * size_t(m),
                            cudaMemcpyHostToDevice, s));
    CY_CUDA(cudaMalloc(&dprob.p, sizeof(double) * 8));
    CY_CUDA(cudaMalloc(&dfrac.p, sizeof(double) * 8));
    CY_CUDA(cudaMemcpyAsync(dprob.p, e->me_prob, sizeof(double) * 8, cudaMemcpyHostToDevice, s));
    CY_CUDA(cudaMemcpyAsync(dfrac.p, e->me_frac, sizeof(double) * 8, cudaMemcpyHostToDevice, s));
    CY_CUDA(cudaMalloc(&ddiag.p, sizeof(double) * diag_scratch_doubles()));

    SqgGpu model;
    {
        const std::string err = model.init(cfg, m);
        if (!err.empty()) return sqg_error(err, st);
    }
    const uint64_t obs_key = stream_key(e->seed, kUseObsNoise);
    const double sd = std::sqrt(e->obs_r);

    turbda_ensf_params ap;
    turbda_ensf_params_init(&ap);
    ap.d_total = d;
    ap.d_local = d;
    ap.obs_dim = nobs;
    ap.n_members = m;
    ap.n_steps = e->n_steps;
    ap.minibatch_j = e->minibatch_j;
    ap.obs_kind = (e->obs_thinning > 1 ? 1 : 0) + (e->obs_arctan ? 2 : 0);
    ap.eps = e->eps;
    ap.damping_t = e->damping_t;
    ap.relax_factor = e->relax_factor;
    ap.seed = e->seed;
    ap.precision = e->precision;
    ap.device = dev;
    ap.flags = TURBDA_INPUTS_ON_DEVICE;
    ap.score_mode = e->score_mode;

    turbda_letkf_params lp;
    turbda_letkf_params_init(&lp);
    lp.nx = cfg.nx;
    lp.ny = cfg.ny;
    lp.n_members = m;
    lp.obs_kind = ap.obs_kind;
    lp.obs_dim = nobs;
    lp.cutoff_km = e->letkf_cutoff_km;
    lp.domain_km = e->letkf_domain_km;
    lp.rtps_alpha = e->letkf_rtps_alpha;
    lp.device = dev;
    lp.flags = TURBDA_INPUTS_ON_DEVICE;

    const auto metrics = [&](const double* x, const double* tr, double* rmse_out,
                             double* spread_out) -> int {
        if (cudaError_t ce = launch_diag(x, m, d, tr, ddiag.as<double>(), s); ce != cudaSuccess)
            return fail(st, TURBDA_CUDA, cudaGetErrorString(ce));
        double h[2];
        CY_CUDA(cudaMemcpyAsync(h, ddiag.p, sizeof h, cudaMemcpyDeviceToHost, s));
        CY_CUDA(cudaStreamSynchronize(s));
        *rmse_out = std::sqrt(h[0] / double(d));
        *spread_out = m < 2 ? 0.0 : std::sqrt(h[1] / (double(m - 1) * double(d)));
        return TURBDA_OK;
    };
    const auto aborted = [&](int k, const std::string& what) {
        if (st) st->diverged_step = k;
        return fail(st, TURBDA_ABORTED, "cycle " + std::to_string(k) + ": " + what);
    };

    for (int k = 1; k <= e->cycles; ++k) {
        double* rec = records + 6 * size_t(k - 1);
        int blown = -1;
        double bh = 0.0;
        tic();
        const std::string err = model.advance(ens.as<double>(), e->obs_interval, s, &cfl, &blown, &bh);
        if (!err.empty()) return aborted(k, err);
        if (blown >= 0) {
            char buf[128];
            std::snprintf(buf, sizeof buf, "integration blowup (NaN/Inf) at t=%f h in member %d", bh, blown);
            return aborted(k, buf);
        }
        if (e->model_quality == 1 && e->me_enabled) {
            model_error_kernel<<<(m + 31) / 32, 32, 0, s>>>(ens.as<double>(), m, d, dkeys.as<unsigned long long>(),
                                                           uint64_t(k), e->me_ncomp, dprob.as<double>(),
                                                           dfrac.as<double>(), base);
            CY_CUDA(cudaGetLastError());
        }
        toc(1);
        const double* tk = truth + size_t(k) * size_t(d);
        double frm = 0, fsp = 0, arm = 0, asp = 0;
        tic();
        if (int rc = metrics(ens.as<double>(), tk, &frm, &fsp)) return rc;
        toc(3);
        if (e->variant == TURBDA_VARIANT_FREE_RUN) {
            arm = frm;
            asp = fsp;
        } else {
            tic();
            synth_obs_kernel<<<unsigned((nobs + 255) / 256), 256, 0, s>>>(
                tk, didx.as<int64_t>(), nobs, e->obs_arctan, sd, uint32_t(obs_key),
                uint32_t(obs_key >> 32), uint64_t(k), dy.as<double>());
            CY_CUDA(cudaGetLastError());
            ap.cycle = uint64_t(k);
            // open-loop probe: this cycle's forecast window and observations
            int slot = -1;
            if (probe)
                for (int q = 0; q < probe->n_cycles; ++q)
                    if (probe->cycles[q] == k) slot = q;
            const size_t pw = probe ? size_t(probe->width) : 0;
            if (slot >= 0) {
                CY_CUDA(cudaMemcpy2DAsync(probe->forecast + size_t(slot) * size_t(m) * pw,
                                          sizeof(double) * pw, ens.as<double>() + probe->k0,
                                          sizeof(double) * size_t(d), sizeof(double) * pw,
                                          size_t(m), cudaMemcpyDeviceToHost, s));
                if (probe->y)
                    CY_CUDA(cudaMemcpyAsync(probe->y + size_t(slot) * size_t(nobs), dy.p,
                                            sizeof(double) * size_t(nobs), cudaMemcpyDeviceToHost,
                                            s));
            }
            turbda_status ast{};
            const int rc =
                e->variant == TURBDA_VARIANT_LETKF
                    ? turbda_letkf_analyze(&lp, ens.as<double>(), dy.as<double>(), dr.as<double>(),
                                           didx.as<int64_t>(), nullptr, ens_out.as<double>(), s, &ast)
                    : turbda_ensf_analyze(&ap, ens.as<double>(), dy.as<double>(), dr.as<double>(),
                                          didx.as<int64_t>(), ens_out.as<double>(), s, &ast);
            if (rc != TURBDA_OK) return aborted(k, ast.msg);
            if (slot >= 0) {
                CY_CUDA(cudaMemcpy2DAsync(probe->analysis + size_t(slot) * size_t(m) * pw,
                                          sizeof(double) * pw, ens_out.as<double>() + probe->k0,
                                          sizeof(double) * size_t(d), sizeof(double) * pw,
                                          size_t(m), cudaMemcpyDeviceToHost, s));
                CY_CUDA(cudaStreamSynchronize(s));
            }
            toc(2);
            std::swap(ens.p, ens_out.p);
            tic();
            if (int rc2 = metrics(ens.as<double>(), tk, &arm, &asp)) return rc2;
            toc(3);
        }
        if (k <= max_records) {
            rec[0] = k;
            rec[1] = double(k) * e->obs_interval;
            rec[2] = frm;
            rec[3] = arm;
            rec[4] = fsp;
            rec[5] = asp;
            *n_records = k;
        }
    }
    if (max_cfl) *max_cfl = cfl;
    return TURBDA_OK;
}

}  // extern "C"
