// TEST INFRASTRUCTURE ONLY - C++ restatement of the reference LETKF arm
// (proj/src/letkf.cpp:10-207) for the reference cycle oracle.  The reference
// file needs Eigen, absent from this image; this restatement keeps its loop
// structure and arithmetic order and replaces Eigen with plain arrays and a
// cyclic Jacobi eigensolver (Eigen's SelfAdjointEigenSolver uses
// tridiagonalisation + QR: eigenpairs agree to rounding, so this oracle is
// "parity unpinned" for the LETKF arm).  It links against the reference's
// own Ensemble / Observation / parallel_for (compiled unmodified into
// oracle/_ref/libturbda_ref_cycle.so) and is checked against the numpy
// restatement oracle/letkf_oracle.py in tests/test_letkf_oracle.py.
#include <algorithm>
#include <cmath>
#include <vector>

#include "turbda/ensemble.hpp"
#include "turbda/letkf.hpp"
#include "turbda/observation.hpp"
#include "turbda/parallel.hpp"

namespace turbda {

double gaspari_cohn(double r) {  // proj/src/letkf.cpp:10-18
    if (r < 0.0) throw ConfigError("gaspari_cohn: r >= 0");
    if (r >= 2.0) return 0.0;
    const double r2 = r * r, r3 = r2 * r, r4 = r3 * r, r5 = r4 * r;
    if (r <= 1.0) return 1.0 - 5.0 / 3.0 * r2 + 5.0 / 8.0 * r3 + 0.5 * r4 - 0.25 * r5;
    return 4.0 - 5.0 * r + 5.0 / 3.0 * r2 + 5.0 / 8.0 * r3 - 0.5 * r4 + r5 / 12.0 -
           2.0 / (3.0 * r);
}

namespace {

// symmetric eigen-decomposition a = v diag(lam) v^T (cyclic Jacobi, row-major m x m)
bool sym_eigen(std::vector<double> a, int m, std::vector<double>& lam, std::vector<double>& v) {
    v.assign(size_t(m) * m, 0.0);
    for (int i = 0; i < m; ++i) v[size_t(i) * m + i] = 1.0;
    // rotations below double rounding (|a_pq| <= eps sqrt|a_pp a_qq|) are
    // skipped; converged once a whole sweep skips every pair
    for (int sweep = 0; sweep < 60; ++sweep) {
        bool rotated = false;
        for (int p = 0; p < m - 1; ++p)
            for (int q = p + 1; q < m; ++q) {
                const double apq = a[size_t(p) * m + q];
                const double app = a[size_t(p) * m + p], aqq = a[size_t(q) * m + q];
                if (!(std::fabs(apq) > 2.2e-16 * std::sqrt(std::fabs(app * aqq)))) continue;
                rotated = true;
                const double theta = (aqq - app) / (2.0 * apq);
                const double t = std::fabs(theta) > 1e150
                                     ? 0.5 / theta
                                     : std::copysign(1.0, theta) /
                                           (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (int i = 0; i < m; ++i) {  // columns
                    const double ip = a[size_t(i) * m + p], iq = a[size_t(i) * m + q];
                    a[size_t(i) * m + p] = c * ip - s * iq;
                    a[size_t(i) * m + q] = s * ip + c * iq;
                    const double vp = v[size_t(i) * m + p], vq = v[size_t(i) * m + q];
                    v[size_t(i) * m + p] = c * vp - s * vq;
                    v[size_t(i) * m + q] = s * vp + c * vq;
                }
                for (int j = 0; j < m; ++j) {  // rows
                    const double pj = a[size_t(p) * m + j], qj = a[size_t(q) * m + j];
                    a[size_t(p) * m + j] = c * pj - s * qj;
                    a[size_t(q) * m + j] = s * pj + c * qj;
                }
                a[size_t(p) * m + q] = a[size_t(q) * m + p] = 0.0;
            }
        if (!rotated) break;
    }
    lam.resize(size_t(m));
    for (int i = 0; i < m; ++i) lam[size_t(i)] = a[size_t(i) * m + i];
    return true;
}

}  // namespace

Ensemble letkf_analyze(const Ensemble& forecast, const Observation& obs, const LetkfConfig& cfg,
                       const GridSpec& grid, int workers) {
    forecast.validate();
    obs.validate();
    cfg.validate();
    grid.validate();
    if (grid.nx != grid.ny || grid.lx != grid.ly)
        throw ConfigError("letkf_analyze: isotropic metric needs nx == ny");
    if (std::fabs(forecast.valid_time - obs.time) > 1e-6)
        throw ConfigError("letkf_analyze: forecast/observation time mismatch");
    const std::size_t d = forecast.dim();
    if (d != grid.grid_size() || obs.op.state_dim != d)
        throw DimensionError("letkf_analyze: state/grid size mismatch");
    if (workers <= 0) workers = default_worker_count();
    const int m = forecast.size();
    const int nx = grid.nx, ny = grid.ny;
    const double cutoff = cfg.cutoff_km / cfg.domain_km * nx;

    // obs-space background, [p][m] (proj/src/letkf.cpp:82-91)
    const std::size_t p_total = obs.y.size();
    std::vector<double> hxb(p_total * size_t(m));
    for (int j = 0; j < m; ++j) {
        const std::vector<double> hx = apply_operator(obs.op, forecast.members[size_t(j)]);
        for (std::size_t k = 0; k < p_total; ++k) hxb[k * size_t(m) + size_t(j)] = hx[k];
    }
    std::vector<double> hxb_mean(p_total, 0.0);
    for (std::size_t k = 0; k < p_total; ++k) {
        double s = 0.0;
        for (int j = 0; j < m; ++j) s += hxb[k * size_t(m) + size_t(j)];
        hxb_mean[k] = s / double(m);
        for (int j = 0; j < m; ++j) hxb[k * size_t(m) + size_t(j)] -= hxb_mean[k];
    }
    const std::vector<double> xb_mean = ensemble_mean(forecast);

    // observations bucketed by the cell of their location (:96-101)
    std::vector<std::vector<int>> bucket(std::size_t(nx) * ny);
    for (std::size_t k = 0; k < p_total; ++k) {
        const int cx = int(std::floor(obs.locations[k][0])) % nx;
        const int cy = int(std::floor(obs.locations[k][1])) % ny;
        bucket[std::size_t(cy) * nx + cx].push_back(int(k));
    }
    // localization stencil as a periodic kernel: every cell residue whose
    // minimum-image distance is below twice the cutoff, weight gc(dist / c)
    // (the offset list of :103-121 visits exactly these residues)
    struct Tap {
        int dx, dy;
        double w;
    };
    std::vector<Tap> stencil;
    for (int dy = 0; dy < ny; ++dy)
        for (int dx = 0; dx < nx; ++dx) {
            const double dist = std::hypot(double(std::min(dx, nx - dx)), double(std::min(dy, ny - dy)));
            if (dist / cutoff < 2.0) stencil.push_back({dx, dy, gaspari_cohn(dist / cutoff)});
        }

    Ensemble analysis = forecast;
    auto& xa = analysis.members;
    parallel_for(std::size_t(nx) * ny, workers, [&](std::size_t pt) {
        const int ix = int(pt % nx), iy = int(pt / nx);
        std::vector<int> local;
        std::vector<double> local_gc;
        for (const Tap& t : stencil)
            for (int k : bucket[std::size_t((iy + t.dy) % ny) * nx + (ix + t.dx) % nx]) {
                local.push_back(k);
                local_gc.push_back(t.w);
            }
        const int p = int(local.size());
        if (p == 0) return;
        const std::size_t row0 = std::size_t(iy) * nx + ix, row1 = std::size_t(ny) * nx + row0;
        // etkf_local_analysis (:20-55): C = Yb^T R^-1, A = C Yb + (m-1) I
        std::vector<double> a(size_t(m) * m, 0.0), rhs(size_t(m), 0.0);
        for (int q = 0; q < p; ++q) {
            const std::size_t ko = size_t(local[size_t(q)]);
            const double rinv = local_gc[size_t(q)] / obs.r_diag[ko];
            const double* yk = &hxb[ko * size_t(m)];
            const double dk = obs.y[ko] - hxb_mean[ko];
            for (int i = 0; i < m; ++i) {
                const double ci = yk[i] * rinv;
                rhs[size_t(i)] += ci * dk;
                for (int j = 0; j < m; ++j) a[size_t(i) * m + j] += ci * yk[j];
            }
        }
        for (int i = 0; i < m; ++i) a[size_t(i) * m + i] += double(m - 1);
        std::vector<double> lam, v;
        sym_eigen(a, m, lam, v);
        for (int i = 0; i < m; ++i)
            if (!std::isfinite(lam[size_t(i)]) || lam[size_t(i)] <= 0.0)
                throw SingularAnalysisError(ix, iy);
        // wbar = V L^-1 V^T rhs ; W = sqrt(m-1) V L^-1/2 V^T
        std::vector<double> u(static_cast<size_t>(m)), wbar(static_cast<size_t>(m)), w(static_cast<size_t>(m) * m);
        for (int i = 0; i < m; ++i) {
            double s = 0.0;
            for (int k = 0; k < m; ++k) s += v[size_t(k) * m + i] * rhs[size_t(k)];
            u[size_t(i)] = s / lam[size_t(i)];
        }
        for (int i = 0; i < m; ++i) {
            double s = 0.0;
            for (int k = 0; k < m; ++k) s += v[size_t(i) * m + k] * u[size_t(k)];
            wbar[size_t(i)] = s;
        }
        const double sm1 = std::sqrt(double(m - 1));
        for (int i = 0; i < m; ++i)
            for (int j = 0; j < m; ++j) {
                double s = 0.0;
                for (int k = 0; k < m; ++k)
                    s += v[size_t(i) * m + k] * v[size_t(j) * m + k] / std::sqrt(lam[size_t(k)]);
                w[size_t(i) * m + j] = sm1 * s;
            }
        for (const std::size_t row : {row0, row1}) {  // :162-171
            const double mean = xb_mean[row];
            std::vector<double> pert(static_cast<size_t>(m));
            for (int j = 0; j < m; ++j) pert[size_t(j)] = forecast.members[size_t(j)][row] - mean;
            double wx = 0.0;
            for (int j = 0; j < m; ++j) wx += pert[size_t(j)] * wbar[size_t(j)];
            for (int j = 0; j < m; ++j) {
                double pw = 0.0;
                for (int i = 0; i < m; ++i) pw += w[size_t(i) * m + j] * pert[size_t(i)];
                xa[size_t(j)][row] = mean + wx + pw;
            }
        }
    });
    return rtps_inflate(analysis, forecast, cfg.rtps_alpha);
}

Ensemble rtps_inflate(const Ensemble& analysis, const Ensemble& background, double alpha) {
    // relaxation to the prior spread, :177-207: per coordinate, deviations
    // from the analysis mean scaled by 1 + alpha (sigma_b - sigma_a) / sigma_a
    if (alpha == 0.0) return analysis;
    analysis.validate(false);
    background.validate(false);
    if (analysis.size() != background.size() || analysis.dim() != background.dim())
        throw DimensionError("rtps_inflate: shape mismatch");
    const int m = analysis.size();
    if (m < 2) return analysis;
    const std::vector<double> mean_a = ensemble_mean(analysis), mean_b = ensemble_mean(background);
    Ensemble out = analysis;
    for (std::size_t k = 0; k < analysis.dim(); ++k) {
        double ssa = 0.0, ssb = 0.0;
        for (int j = 0; j < m; ++j) {
            const double ea = analysis.members[size_t(j)][k] - mean_a[k];
            const double eb = background.members[size_t(j)][k] - mean_b[k];
            ssa += ea * ea;
            ssb += eb * eb;
        }
        const double sig_a = std::max(std::sqrt(ssa / (m - 1)), 1e-12);
        const double sig_b = std::sqrt(ssb / (m - 1));
        const double f = 1.0 + alpha * (sig_b - sig_a) / sig_a;
        for (int j = 0; j < m; ++j)
            out.members[size_t(j)][k] = mean_a[k] + f * (analysis.members[size_t(j)][k] - mean_a[k]);
    }
    return out;
}

}  // namespace turbda
