// Batched two-boundary Eady SQG model on the GPU (fp64, cuFFT) - the
// forecast half of the cycled configs, a B200
// restatement of proj/src/sqg.cpp + proj/src/spectral.cpp +
// SqgStepper::advance (proj/src/forecast.cpp:14-32):
//   * state: boundary theta at z = 0, H; spectral [B][2][ny][nx/2+1]
//   * tendency (proj/src/sqg.cpp:189-260): invert theta -> psi, form
//     u, v, theta_x, theta_y on both levels (8 spectral planes per member),
//     one batched Z2D, the advective product in physical space (+ CFL),
//     one batched D2Z, 1/(nx ny) and the 2/3 dealias mask
//   * integrating-factor RK4 (proj/include/turbda/sqg.hpp:52-77) with the
//     exact hyperdiffusion / drag factors e^{-lambda dt}, e^{-lambda dt/2}
// All B members advance together (one FFT plan per batch), and one RK4 step
// (4 tendencies, ~24 launches) is captured once into a CUDA graph and
// replayed, so a long nature run is not launch-bound.
#include <cufft.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "ensf_device.h"
#include "sqg_gpu.h"

namespace tb200 {

namespace {

constexpr double kTwoPi = 6.283185307179586476925286766559;

__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
    // non-negative doubles order like their bit patterns
    atomicMax(reinterpret_cast<unsigned long long*>(addr),
              static_cast<unsigned long long>(__double_as_longlong(v)));
}

struct ModeTables {
    const double *kx, *ky, *mask, *i00, *i01, *i11, *ef, *eh;
};

// theta (masked) -> the 8 spectral planes u, v, theta_x, theta_y x 2 levels;
// plane index ((var * B + b) * 2 + lev)
__global__ void sqg_build_vars(const cufftDoubleComplex* __restrict__ th, ModeTables t, int nb,
                               int nmode, cufftDoubleComplex* __restrict__ cvar) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    if (i >= nmode) return;
    const double msk = t.mask[i], kx = t.kx[i], ky = t.ky[i];
    const cufftDoubleComplex a0 = th[(size_t(b) * 2 + 0) * nmode + i];
    const cufftDoubleComplex a1 = th[(size_t(b) * 2 + 1) * nmode + i];
    const double t0r = a0.x * msk, t0i = a0.y * msk, t1r = a1.x * msk, t1i = a1.y * msk;
    const double p0r = t.i00[i] * t0r + t.i01[i] * t1r, p0i = t.i00[i] * t0i + t.i01[i] * t1i;
    const double p1r = -t.i01[i] * t0r + t.i11[i] * t1r, p1i = -t.i01[i] * t0i + t.i11[i] * t1i;
    const size_t plane = size_t(nmode);
    const auto at = [&](int var, int lev) { return cvar + ((size_t(var) * nb + b) * 2 + lev) * plane + i; };
    // multiply by i k: (re, im) -> (-k im, k re)
    *at(0, 0) = make_cuDoubleComplex(ky * p0i, -ky * p0r);
    *at(0, 1) = make_cuDoubleComplex(ky * p1i, -ky * p1r);
    *at(1, 0) = make_cuDoubleComplex(-kx * p0i, kx * p0r);
    *at(1, 1) = make_cuDoubleComplex(-kx * p1i, kx * p1r);
    *at(2, 0) = make_cuDoubleComplex(-kx * t0i, kx * t0r);
    *at(2, 1) = make_cuDoubleComplex(-kx * t1i, kx * t1r);
    *at(3, 0) = make_cuDoubleComplex(-ky * t0i, ky * t0r);
    *at(3, 1) = make_cuDoubleComplex(-ky * t1i, ky * t1r);
}

// physical-space advection: t = -((u + U_lev) theta_x + v theta_y) + (u0/H) v.
// blockIdx.y = one (member, level) plane; each thread takes pixel pairs
// (16 B loads) in a block-stride loop and the CFL maximum is reduced per
// block, so the single global atomic is hit once per block instead of once
// per warp (that contention cost 3/4 of this kernel's time).
constexpr int kProdThreads = 256, kProdPairs = 4;  // pixel pairs per thread

__global__ void __launch_bounds__(kProdThreads) sqg_products(
    const double* __restrict__ gvar, int nb, int npix, double u0, double grad_bg, double inv_dx,
    double inv_dy, double dt, double* __restrict__ gten, double* __restrict__ cfl) {
    __shared__ double red[kProdThreads / 32];
    const int bl = blockIdx.y;  // b * 2 + lev
    const double ushift = (bl & 1) ? 0.5 * u0 : -0.5 * u0;
    const size_t plane = size_t(npix);
    const size_t stride_var = size_t(nb) * 2 * plane;
    const double2* u2 = reinterpret_cast<const double2*>(gvar + size_t(bl) * plane);
    const double2* v2 = reinterpret_cast<const double2*>(gvar + stride_var + size_t(bl) * plane);
    const double2* x2 = reinterpret_cast<const double2*>(gvar + 2 * stride_var + size_t(bl) * plane);
    const double2* y2 = reinterpret_cast<const double2*>(gvar + 3 * stride_var + size_t(bl) * plane);
    double2* t2 = reinterpret_cast<double2*>(gten + size_t(bl) * plane);
    double cmax = 0.0;
    const int npair = npix / 2;
    for (int q = blockIdx.x * kProdThreads + threadIdx.x; q < npair; q += gridDim.x * kProdThreads) {
        const double2 u = u2[q], v = v2[q], tx = x2[q], ty = y2[q];
        const double ua = u.x + ushift, ub = u.y + ushift;
        t2[q] = make_double2(-(ua * tx.x + v.x * ty.x) + grad_bg * v.x,
                             -(ub * tx.y + v.y * ty.y) + grad_bg * v.y);
        cmax = fmax(cmax, fmax(fmax(fabs(ua) * inv_dx, fabs(v.x) * inv_dy),
                               fmax(fabs(ub) * inv_dx, fabs(v.y) * inv_dy)));
    }
    cmax *= dt;
    for (int o = 16; o > 0; o >>= 1) cmax = fmax(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cmax;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kProdThreads / 32; ++w) cmax = fmax(cmax, red[w]);
        atomic_max_nonneg(cfl, cmax);
    }
}

// one of the four integrating-factor RK4 combinations
// (proj/include/turbda/sqg.hpp:63-76); k = cten * (1/(nx ny)) * mask
template <int kStage>
__global__ void sqg_rk4_combine(const cufftDoubleComplex* __restrict__ cten, ModeTables t,
                                int nmode, double scale, double dt,
                                cufftDoubleComplex* __restrict__ th,
                                cufftDoubleComplex* __restrict__ ks,  // [4][B*2*nmode]
                                cufftDoubleComplex* __restrict__ stage, size_t nstate,
                                unsigned long long* __restrict__ bad,
                                const unsigned int* __restrict__ step) {
    const size_t q = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= nstate) return;
    const int i = int(q % size_t(nmode));
    const double w = scale * t.mask[i];
    const cufftDoubleComplex c = cten[q];
    const double kr = c.x * w, ki = c.y * w;
    ks[(kStage - 1) * nstate + q] = make_cuDoubleComplex(kr, ki);
    const cufftDoubleComplex x = th[q];
    const double ef = t.ef[i], eh = t.eh[i];
    if (kStage == 1) {
        stage[q] = make_cuDoubleComplex(eh * (x.x + 0.5 * dt * kr), eh * (x.y + 0.5 * dt * ki));
    } else if (kStage == 2) {
        stage[q] = make_cuDoubleComplex(eh * x.x + 0.5 * dt * kr, eh * x.y + 0.5 * dt * ki);
    } else if (kStage == 3) {
        stage[q] = make_cuDoubleComplex(ef * x.x + dt * eh * kr, ef * x.y + dt * eh * ki);
    } else {
        const cufftDoubleComplex k1 = ks[q], k2 = ks[nstate + q], k3 = ks[2 * nstate + q];
        double nr = ef * x.x + dt / 6.0 * (ef * k1.x + 2.0 * eh * (k2.x + k3.x) + kr);
        double ni = ef * x.y + dt / 6.0 * (ef * k1.y + 2.0 * eh * (k2.y + k3.y) + ki);
        nr *= t.mask[i];
        ni *= t.mask[i];
        th[q] = make_cuDoubleComplex(nr, ni);
        if (!isfinite(nr) || !isfinite(ni)) {
            const unsigned long long member = q / (2 * size_t(nmode));
            atomicMin(bad, (member << 32) | *step);
        }
    }
}

__global__ void sqg_bump_step(unsigned int* step) { ++*step; }

// physical -> spectral scaling and dealias (forward transform + dealias())
__global__ void sqg_scale_mask(cufftDoubleComplex* __restrict__ th, const double* __restrict__ mask,
                               int nmode, size_t nstate, double scale, int apply_mask) {
    const size_t q = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= nstate) return;
    const double w = scale * (apply_mask ? mask[q % size_t(nmode)] : 1.0);
    th[q].x *= w;
    th[q].y *= w;
}

// per-mode kinetic energy of one state for ke_spectrum (proj/src/sqg.cpp:306-335):
// theta_hat (scaled forward transform, no dealias) -> psi -> 0.5 w |k p|^2 / nz,
// out [lev][mode]; the shell sums run on the host in the reference's order
__global__ void sqg_mode_energy(const cufftDoubleComplex* __restrict__ th, ModeTables t,
                                int nmode, int nkx, int nx, double scale,
                                double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nmode) return;
    const double t0r = th[i].x * scale, t0i = th[i].y * scale;
    const double t1r = th[nmode + i].x * scale, t1i = th[nmode + i].y * scale;
    const double pr[2] = {t.i00[i] * t0r + t.i01[i] * t1r, -t.i01[i] * t0r + t.i11[i] * t1r};
    const double pi[2] = {t.i00[i] * t0i + t.i01[i] * t1i, -t.i01[i] * t0i + t.i11[i] * t1i};
    const int jx = i % nkx;
    const double w = (jx == 0 || jx == nx / 2) ? 1.0 : 2.0;
    const double kx = t.kx[i], ky = t.ky[i];
    for (int lev = 0; lev < 2; ++lev) {
        const double ar = ky * pr[lev], ai = ky * pi[lev], br = kx * pr[lev], bi = kx * pi[lev];
        const double u2 = (ar * ar + ai * ai) + (br * br + bi * bi);
        out[size_t(lev) * nmode + i] = 0.5 * w * u2 / 2.0;
    }
}

}  // namespace

struct SqgGpu::Impl {
    SqgConfig cfg;
    int nb = 0, nmode = 0, npix = 0;
    size_t nstate = 0;  // nb * 2 * nmode
    cufftHandle c2r_vars = 0, r2c_ten = 0, r2c_state = 0, c2r_state = 0;
    double* tables = nullptr;  // 8 * nmode
    ModeTables t{};
    cufftDoubleComplex *th = nullptr, *ks = nullptr, *stage = nullptr, *cvar = nullptr,
                       *cten = nullptr, *cwork = nullptr;
    double *gvar = nullptr, *gten = nullptr, *cfl = nullptr;
    unsigned long long* bad = nullptr;
    unsigned int* step = nullptr;
    cudaStream_t own = nullptr;  // capture / replay stream (the legacy stream cannot be captured)
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    cudaGraphExec_t step_graph = nullptr;
    std::vector<double> hkx, hky;     // host copies of the wavenumber tables
    cufftHandle r2c_one = 0;          // one state (2 planes), ke_spectrum
};

static void free_all(SqgGpu::Impl* p) {
    if (p->step_graph) cudaGraphExecDestroy(p->step_graph);
    if (p->own) cudaStreamDestroy(p->own);
    if (p->ev_in) cudaEventDestroy(p->ev_in);
    if (p->ev_out) cudaEventDestroy(p->ev_out);
    if (p->c2r_vars) cufftDestroy(p->c2r_vars);
    if (p->r2c_ten) cufftDestroy(p->r2c_ten);
    if (p->r2c_state) cufftDestroy(p->r2c_state);
    if (p->c2r_state) cufftDestroy(p->c2r_state);
    if (p->r2c_one) cufftDestroy(p->r2c_one);
    cudaFree(p->tables);
    cudaFree(p->th);
    cudaFree(p->ks);
    cudaFree(p->stage);
    cudaFree(p->cvar);
    cudaFree(p->cten);
    cudaFree(p->cwork);
    cudaFree(p->gvar);
    cudaFree(p->gten);
    cudaFree(p->cfl);
    cudaFree(p->bad);
    cudaFree(p->step);
}

SqgGpu::SqgGpu() = default;
SqgGpu::~SqgGpu() {
    if (impl_) free_all(impl_.get());
}

// proj/src/sqg.cpp:47-130 (mode tables) restated; returns "" or an error text
std::string SqgGpu::init(const SqgConfig& c, int batch) {
    impl_ = std::make_unique<Impl>();
    Impl& p = *impl_;
    p.cfg = c;
    p.nb = batch;
    const int nx = c.nx, ny = c.ny, nkx = nx / 2 + 1;
    p.nmode = ny * nkx;
    p.npix = ny * nx;
    p.nstate = size_t(batch) * 2 * p.nmode;
    const int nmode = p.nmode;

    std::vector<double> h(size_t(8) * nmode);
    double* kx = h.data();
    double* ky = kx + nmode;
    double* mask = ky + nmode;
    double* i00 = mask + nmode;
    double* i01 = i00 + nmode;
    double* i11 = i01 + nmode;
    double* ef = i11 + nmode;
    double* eh = ef + nmode;
    const int cx = nx / 3, cy = ny / 3;
    const double kappa_cut = std::hypot(kTwoPi * cx / c.lx, kTwoPi * cy / c.ly);
    const double nu = 1.0 / (c.hyper_efold * std::pow(kappa_cut * kappa_cut, c.hyper_order));
    for (int jy = 0; jy < ny; ++jy) {
        const int jys = jy <= ny / 2 ? jy : jy - ny;
        for (int jx = 0; jx < nkx; ++jx) {
            const int i = jy * nkx + jx;
            kx[i] = kTwoPi * jx / c.lx;
            ky[i] = kTwoPi * jys / c.ly;
            mask[i] = (jx <= cx && jys <= cy && jys >= -cy) ? 1.0 : 0.0;
            const double kappa = std::hypot(kx[i], ky[i]);
            if (kappa > 0.0) {
                const double m = c.n * kappa / c.f;
                const double mu = m * c.h;
                i00[i] = -(1.0 / std::tanh(mu)) / m;
                i01[i] = (1.0 / std::sinh(mu)) / m;
                i11[i] = (1.0 / std::tanh(mu)) / m;
            } else {
                i00[i] = i01[i] = i11[i] = 0.0;
            }
            const double k2 = kx[i] * kx[i] + ky[i] * ky[i];
            double lambda = nu * std::pow(k2, c.hyper_order);
            if (kappa > 0.0 && c.drag_tau > 0.0) lambda += 1.0 / c.drag_tau;
            ef[i] = std::exp(-lambda * c.dt);
            eh[i] = std::exp(-0.5 * lambda * c.dt);
        }
    }
    if (cudaMalloc(&p.tables, sizeof(double) * h.size()) != cudaSuccess) return "cudaMalloc tables";
    cudaMemcpy(p.tables, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
    p.hkx.assign(kx, kx + nmode);
    p.hky.assign(ky, ky + nmode);
    p.t = ModeTables{p.tables, p.tables + nmode, p.tables + 2 * nmode, p.tables + 3 * nmode,
                     p.tables + 4 * nmode, p.tables + 5 * nmode, p.tables + 6 * nmode,
                     p.tables + 7 * nmode};

    const size_t cb = sizeof(cufftDoubleComplex);
    bool ok = cudaMalloc(&p.th, cb * p.nstate) == cudaSuccess &&
              cudaMalloc(&p.ks, cb * p.nstate * 4) == cudaSuccess &&
              cudaMalloc(&p.stage, cb * p.nstate) == cudaSuccess &&
              cudaMalloc(&p.cvar, cb * p.nstate * 4) == cudaSuccess &&
              cudaMalloc(&p.cten, cb * p.nstate) == cudaSuccess &&
              cudaMalloc(&p.cwork, cb * p.nstate) == cudaSuccess &&
              cudaMalloc(&p.gvar, sizeof(double) * size_t(batch) * 8 * p.npix) == cudaSuccess &&
              cudaMalloc(&p.gten, sizeof(double) * size_t(batch) * 2 * p.npix) == cudaSuccess &&
              cudaMalloc(&p.cfl, sizeof(double)) == cudaSuccess &&
              cudaMalloc(&p.bad, sizeof(unsigned long long)) == cudaSuccess &&
              cudaMalloc(&p.step, sizeof(unsigned int)) == cudaSuccess;
    if (!ok) return "cudaMalloc of SQG state";
    if (cudaStreamCreateWithFlags(&p.own, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&p.ev_in, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&p.ev_out, cudaEventDisableTiming) != cudaSuccess)
        return "SQG stream";
    int n2[2] = {ny, nx};
    if (cufftPlanMany(&p.c2r_vars, 2, n2, nullptr, 1, nmode, nullptr, 1, p.npix, CUFFT_Z2D,
                      8 * batch) != CUFFT_SUCCESS ||
        cufftPlanMany(&p.r2c_ten, 2, n2, nullptr, 1, p.npix, nullptr, 1, nmode, CUFFT_D2Z,
                      2 * batch) != CUFFT_SUCCESS ||
        cufftPlanMany(&p.r2c_state, 2, n2, nullptr, 1, p.npix, nullptr, 1, nmode, CUFFT_D2Z,
                      2 * batch) != CUFFT_SUCCESS ||
        cufftPlanMany(&p.c2r_state, 2, n2, nullptr, 1, nmode, nullptr, 1, p.npix, CUFFT_Z2D,
                      2 * batch) != CUFFT_SUCCESS)
        return "cufftPlanMany";
    return "";
}

int SqgGpu::batch() const { return impl_ ? impl_->nb : 0; }

// proj/src/sqg.cpp:306-335: shell-summed kinetic energy of ONE state
// [2][ny][nx] on the device; bins at kappa = s 2 pi / lx, s = round(|k| / dk)
std::string SqgGpu::ke_spectrum(const double* state, cudaStream_t st, std::vector<double>* kappa,
                                std::vector<double>* energy) {
    Impl& p = *impl_;
    const SqgConfig& c = p.cfg;
    if (c.lx != c.ly) return "config:ke_spectrum: requires lx == ly";
    if (!p.r2c_one) {
        int n2[2] = {c.ny, c.nx};
        if (cufftPlanMany(&p.r2c_one, 2, n2, nullptr, 1, p.npix, nullptr, 1, p.nmode, CUFFT_D2Z, 2) !=
            CUFFT_SUCCESS)
            return "cufftPlanMany";
    }
    cufftSetStream(p.r2c_one, st);
    if (cufftExecD2Z(p.r2c_one, const_cast<double*>(state), p.cwork) != CUFFT_SUCCESS)
        return "cufftExecD2Z";
    const int nkx = c.nx / 2 + 1;
    sqg_mode_energy<<<unsigned((p.nmode + 255) / 256), 256, 0, st>>>(
        p.cwork, p.t, p.nmode, nkx, c.nx, 1.0 / (double(c.nx) * c.ny), p.gten);
    if (cudaGetLastError() != cudaSuccess) return "sqg_mode_energy";
    std::vector<double> e(size_t(2) * p.nmode);
    if (cudaMemcpyAsync(e.data(), p.gten, sizeof(double) * e.size(), cudaMemcpyDeviceToHost, st) !=
            cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return "ke_spectrum copy";
    const double dk = kTwoPi / c.lx;
    const double kmax = std::hypot(kTwoPi * (c.nx / 2) / c.lx, kTwoPi * (c.ny / 2) / c.ly);
    const int nshell = int(std::lround(kmax / dk)) + 1;
    kappa->assign(size_t(nshell), 0.0);
    energy->assign(size_t(nshell), 0.0);
    for (int s = 0; s < nshell; ++s) (*kappa)[size_t(s)] = s * dk;
    for (int lev = 0; lev < 2; ++lev)  // the reference's summation order
        for (int i = 0; i < p.nmode; ++i) {
            const int s = int(std::lround(std::hypot(p.hkx[size_t(i)], p.hky[size_t(i)]) / dk));
            (*energy)[size_t(s)] += e[size_t(lev) * p.nmode + i];
        }
    return "";
}

size_t SqgGpu::state_size() const { return impl_ ? size_t(2) * impl_->npix : 0; }

std::string SqgGpu::dealias(double* states, cudaStream_t caller) {
    Impl& p = *impl_;
    cudaStream_t st = caller;
    cufftSetStream(p.r2c_state, st);
    cufftSetStream(p.c2r_state, st);
    if (cufftExecD2Z(p.r2c_state, states, p.th) != CUFFT_SUCCESS) return "cufftExecD2Z";
    sqg_scale_mask<<<unsigned((p.nstate + 255) / 256), 256, 0, st>>>(
        p.th, p.t.mask, p.nmode, p.nstate, 1.0 / (double(p.cfg.nx) * p.cfg.ny), 1);
    if (cufftExecZ2D(p.c2r_state, p.th, states) != CUFFT_SUCCESS) return "cufftExecZ2D";
    return cudaGetLastError() == cudaSuccess ? "" : "dealias";
}

// one tendency of `in` into ks[k-1] / the RK combination of stage k
static cudaError_t tendency_and_combine(SqgGpu::Impl& p, const cufftDoubleComplex* in, int k,
                                        cudaStream_t st) {
    const SqgConfig& c = p.cfg;
    cufftSetStream(p.c2r_vars, st);
    cufftSetStream(p.r2c_ten, st);
    sqg_build_vars<<<dim3(unsigned((p.nmode + 127) / 128), unsigned(p.nb)), 128, 0, st>>>(
        in, p.t, p.nb, p.nmode, p.cvar);
    if (cufftExecZ2D(p.c2r_vars, p.cvar, p.gvar) != CUFFT_SUCCESS) return cudaErrorUnknown;
    sqg_products<<<dim3(unsigned((p.npix / 2 + kProdThreads * kProdPairs - 1) /
                                 (kProdThreads * kProdPairs)),
                        unsigned(2 * p.nb)),
                   kProdThreads, 0, st>>>(
        p.gvar, p.nb, p.npix, c.u0, c.u0 / c.h, double(c.nx) / c.lx, double(c.ny) / c.ly, c.dt,
        p.gten, p.cfl);
    if (cufftExecD2Z(p.r2c_ten, p.gten, p.cten) != CUFFT_SUCCESS) return cudaErrorUnknown;
    const double scale = 1.0 / (double(c.nx) * c.ny);
    const unsigned g = unsigned((p.nstate + 255) / 256);
    switch (k) {
        case 1: sqg_rk4_combine<1><<<g, 256, 0, st>>>(p.cten, p.t, p.nmode, scale, c.dt, p.th, p.ks, p.stage, p.nstate, p.bad, p.step); break;
        case 2: sqg_rk4_combine<2><<<g, 256, 0, st>>>(p.cten, p.t, p.nmode, scale, c.dt, p.th, p.ks, p.stage, p.nstate, p.bad, p.step); break;
        case 3: sqg_rk4_combine<3><<<g, 256, 0, st>>>(p.cten, p.t, p.nmode, scale, c.dt, p.th, p.ks, p.stage, p.nstate, p.bad, p.step); break;
        default: sqg_rk4_combine<4><<<g, 256, 0, st>>>(p.cten, p.t, p.nmode, scale, c.dt, p.th, p.ks, p.stage, p.nstate, p.bad, p.step); break;
    }
    return cudaGetLastError();
}

static cudaError_t rk4_step(SqgGpu::Impl& p, cudaStream_t st) {
    cudaError_t e;
    if ((e = tendency_and_combine(p, p.th, 1, st)) != cudaSuccess) return e;
    if ((e = tendency_and_combine(p, p.stage, 2, st)) != cudaSuccess) return e;
    if ((e = tendency_and_combine(p, p.stage, 3, st)) != cudaSuccess) return e;
    if ((e = tendency_and_combine(p, p.stage, 4, st)) != cudaSuccess) return e;
    sqg_bump_step<<<1, 1, 0, st>>>(p.step);
    return cudaGetLastError();
}

std::string SqgGpu::advance(double* states, double hours, cudaStream_t caller, double* max_cfl,
                            int* blown_member, double* blown_hours) {
    Impl& p = *impl_;
    // run on the model's own stream, ordered after / before the caller's
    cudaStream_t st = p.own;
    cudaEventRecord(p.ev_in, caller);
    cudaStreamWaitEvent(st, p.ev_in, 0);
    const double steps_real = hours / p.cfg.dt;
    const long steps = std::lround(steps_real);
    if (hours < 0.0 || std::fabs(steps_real - double(steps)) > 1e-9)
        return "config:advance: duration must be a multiple of dt";
    if (blown_member) *blown_member = -1;
    if (steps == 0) return "";
    // forward transform + dealias (SqgStepper::advance, proj/src/forecast.cpp:24-26)
    cufftSetStream(p.r2c_state, st);
    cufftSetStream(p.c2r_state, st);
    if (cufftExecD2Z(p.r2c_state, states, p.th) != CUFFT_SUCCESS) return "cufftExecD2Z";
    const unsigned g = unsigned((p.nstate + 255) / 256);
    sqg_scale_mask<<<g, 256, 0, st>>>(p.th, p.t.mask, p.nmode, p.nstate,
                                      1.0 / (double(p.cfg.nx) * p.cfg.ny), 1);
    cudaMemsetAsync(p.cfl, 0, sizeof(double), st);
    cudaMemsetAsync(p.bad, 0xff, sizeof(unsigned long long), st);
    cudaMemsetAsync(p.step, 0, sizeof(unsigned int), st);
    // one RK4 step as a CUDA graph, replayed
    if (!p.step_graph) {
        cudaGraph_t graph;
        if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
            return "cudaStreamBeginCapture";
        const cudaError_t e = rk4_step(p, st);
        const cudaError_t e2 = cudaStreamEndCapture(st, &graph);
        if (e != cudaSuccess || e2 != cudaSuccess) return "capture of the SQG step";
        if (cudaGraphInstantiate(&p.step_graph, graph, 0) != cudaSuccess) return "cudaGraphInstantiate";
        cudaGraphDestroy(graph);
    }
    for (long s = 0; s < steps; ++s)
        if (cudaGraphLaunch(p.step_graph, st) != cudaSuccess) return "cudaGraphLaunch";
    // inverse transform (c2r destroys its input: work on a copy)
    cudaMemcpyAsync(p.cwork, p.th, sizeof(cufftDoubleComplex) * p.nstate, cudaMemcpyDeviceToDevice, st);
    if (cufftExecZ2D(p.c2r_state, p.cwork, states) != CUFFT_SUCCESS) return "cufftExecZ2D";
    unsigned long long bad = ~0ull;
    double cfl = 0.0;
    cudaMemcpyAsync(&bad, p.bad, sizeof bad, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&cfl, p.cfl, sizeof cfl, cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return "SQG advance";
    cudaEventRecord(p.ev_out, st);
    cudaStreamWaitEvent(caller, p.ev_out, 0);
    if (max_cfl) *max_cfl = std::max(*max_cfl, cfl);
    if (bad != ~0ull) {
        // BlowupError(t, member) of proj/src/sqg.cpp:296 / proj/src/forecast.cpp:63-67:
        // t = model time after the first non-finite step
        if (blown_member) *blown_member = int(bad >> 32);
        if (blown_hours) *blown_hours = double((bad & 0xffffffffu) + 1) * p.cfg.dt;
    }
    return "";
}

}  // namespace tb200
