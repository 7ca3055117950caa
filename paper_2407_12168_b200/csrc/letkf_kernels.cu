// LETKF analysis arm on the GPU: letkf_analyze,
// rtps_inflate and gaspari_cohn of proj/src/letkf.cpp:10-207, behind the
// C-ABI turbda_letkf_* (include/turbda_b200.h).
//
// The reference loops over grid points; each gathers the observations of
// every cell within twice the cutoff, weights R^-1 with Gaspari-Cohn, forms
// A = (M-1) I + Yb^T R^-1 Yb and solves a symmetric eigenproblem
// (proj/src/letkf.cpp:20-55,123-172).  Re-designed for the GPU:
//
//  1. obs kernel: h(x_j) for every observation, ensemble-mean removal
//     (Yb, member-major), innovation d = y - mean, 1/r, the observation's cell.
//  2. stable bucketing of observations by cell (cub radix sort + scan), so
//     per-cell sums run in observation order (deterministic).
//  3. per-cell fields S_c = sum_k y_k y_k^T / r_k (upper triangle), t_c =
//     sum_k y_k d_k / r_k and the observation count, one fp64 field each.
//  4. the localized sums A(pt) - (M-1) I = sum_o gc(|o|/c) S_{pt+o} and b(pt)
//     are a PERIODIC CONVOLUTION of those fields with the Gaspari-Cohn
//     stencil (every cell residue appears at most once in the reference's
//     offset list, proj/src/letkf.cpp:101-121): batched cuFFT D2Z, multiply
//     by the stencil's real spectrum, Z2D.  O(P log P) per field instead of
//     O(P x stencil) — the stencil holds ~8,000 cells at 256^2.
//  5. one CTA per grid point: parallel cyclic Jacobi eigensolver in shared
//     memory (round-robin pairs, all rotations of a round at once), then
//     wbar = V L^-1 V^T b and the transform of both levels with
//     W = sqrt(M-1) V L^-1/2 V^T applied as two mat-vecs.
//  6. RTPS inflation per coordinate.
//
// Everything is fp64.  Results agree with the reference formulation to
// rounding (a different summation order), not bit for bit.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <cub/cub.cuh>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cufft.h>

#include "ensf_device.h"
#include "turbda_b200.h"

namespace tb200 {
namespace {

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

#define LK_CUDA(call)                                                                        \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return fail(st, TURBDA_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define LK_FFT(call)                                                                    \
    do {                                                                                \
        cufftResult r_ = (call);                                                        \
        if (r_ != CUFFT_SUCCESS)                                                        \
            return fail(st, TURBDA_CUDA, std::string(#call) + ": cufft error " +        \
                                             std::to_string(int(r_)));                  \
    } while (0)

struct Buf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaError_t reserve(size_t b) {
        if (b <= bytes) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        cudaError_t e = cudaMalloc(&p, b);
        if (e == cudaSuccess) bytes = b;
        return e;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
    ~Buf() {
        if (p) cudaFree(p);
    }
};

// ---------------------------------------------------------------------------
// gaspari_cohn, proj/src/letkf.cpp:10-18 (host and device)
__host__ __device__ inline double gc_weight(double r) {
    if (r >= 2.0) return 0.0;
    const double r2 = r * r, r3 = r2 * r, r4 = r3 * r, r5 = r4 * r;
    if (r <= 1.0) return 1.0 - 5.0 / 3.0 * r2 + 5.0 / 8.0 * r3 + 0.5 * r4 - 0.25 * r5;
    return 4.0 - 5.0 * r + 5.0 / 3.0 * r2 + 5.0 / 8.0 * r3 - 0.5 * r4 + r5 / 12.0 -
           2.0 / (3.0 * r);
}

// upper-triangle (i <= j) row-major index
__host__ __device__ inline int tri(int i, int j, int m) { return i * m - (i * (i - 1)) / 2 + (j - i); }

// 1. observation space background.  Yb is member-major [m][p] (coalesced
// over observations); the mean is summed in member order and divided by m
// (Eigen rowwise().mean(), proj/src/letkf.cpp:85-90).
__global__ void letkf_obs_kernel(const double* __restrict__ x, int64_t d, int m,
                                 const int64_t* __restrict__ idx, int64_t p, int arctan,
                                 const double* __restrict__ y, const double* __restrict__ r,
                                 int64_t r_stride, const double* __restrict__ locs, int nx,
                                 int ny, double* __restrict__ yb, double* __restrict__ dinn,
                                 double* __restrict__ rinv, uint32_t* __restrict__ cell,
                                 uint32_t* __restrict__ order) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= p) return;
    const int64_t q = idx ? idx[k] : k;
    double s = 0.0;
    for (int j = 0; j < m; ++j) {
        double h = x[size_t(j) * size_t(d) + size_t(q)];
        if (arctan) h = atan(h);
        s += h;
    }
    const double mean = s / double(m);
    for (int j = 0; j < m; ++j) {
        double h = x[size_t(j) * size_t(d) + size_t(q)];
        if (arctan) h = atan(h);
        yb[size_t(j) * size_t(p) + size_t(k)] = h - mean;
    }
    dinn[k] = y[k] - mean;
    rinv[k] = 1.0 / r[k * r_stride];
    int cx, cy;
    if (locs) {
        // int(floor(loc)) % n of proj/src/letkf.cpp:98-99, kept non-negative
        cx = int(floor(locs[2 * k])) % nx;
        cy = int(floor(locs[2 * k + 1])) % ny;
        cx += cx < 0 ? nx : 0;
        cy += cy < 0 ? ny : 0;
    } else {
        // operator_locations (proj/src/observation.cpp:43-60): the cell of a
        // flat state index is its horizontal position
        const int64_t h = q % (int64_t(nx) * ny);
        cx = int(h % nx);
        cy = int(h / nx);
    }
    cell[k] = uint32_t(cy) * uint32_t(nx) + uint32_t(cx);
    order[k] = uint32_t(k);
}

__global__ void count_cells_kernel(const uint32_t* __restrict__ cell, int64_t p,
                                   int* __restrict__ count) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k < p) atomicAdd(&count[cell[k]], 1);
}

// 3. per-cell fields, field-major [f][P] with f < E: S entries, E..E+m-1: t,
// E+m: observation count.  A block covers 128 consecutive cells and a chunk
// of fields; each cell sums its observations in observation order.
constexpr int kFieldCells = 128;
constexpr int kFieldChunk = 16;

__global__ void __launch_bounds__(kFieldCells)
letkf_fields_kernel(const double* __restrict__ yb, const double* __restrict__ dinn,
                    const double* __restrict__ rinv, const uint32_t* __restrict__ sorted_obs,
                    const int* __restrict__ start, int64_t p, int m, int64_t P, int nf,
                    double* __restrict__ fields) {
    const int64_t c = int64_t(blockIdx.x) * kFieldCells + threadIdx.x;
    if (c >= P) return;
    const int E = m * (m + 1) / 2;
    const int lo = start[c], hi = start[c + 1];
    const int f0 = blockIdx.y * kFieldChunk;
    const int f1 = min(nf, f0 + kFieldChunk);
    // decode the first field's (i, j) once, then walk the triangle
    int i = 0, j = 0;
    if (f0 < E) {
        while (tri(i, m - 1, m) < f0) ++i;
        j = i + (f0 - tri(i, i, m));
    }
    for (int f = f0; f < f1; ++f) {
        double acc = 0.0;
        if (f < E) {
            for (int q = lo; q < hi; ++q) {
                const int64_t k = sorted_obs[q];
                acc += rinv[k] * yb[size_t(i) * p + k] * yb[size_t(j) * p + k];
            }
            if (++j == m) {
                ++i;
                j = i;
            }
        } else if (f < E + m) {
            const int a = f - E;
            for (int q = lo; q < hi; ++q) {
                const int64_t k = sorted_obs[q];
                acc += rinv[k] * yb[size_t(a) * p + k] * dinn[k];
            }
        } else {
            acc = double(hi - lo);
        }
        fields[size_t(f) * size_t(P) + size_t(c)] = acc;
    }
}

// 4. spectral multiply by the real stencil spectrum (scaled by 1/P); the
// observation-count field uses the stencil's indicator (r < 2) instead, so it
// counts the observations the reference gathers
__global__ void spectral_scale_kernel(cufftDoubleComplex* __restrict__ g,
                                      const double* __restrict__ khat, int64_t nh,
                                      int64_t total, int f0, int count_field) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= total) return;
    const int f = f0 + int(t / nh);
    const double k = khat[(f == count_field ? nh : 0) + t % nh];
    g[t].x *= k;
    g[t].y *= k;
}

// 5. per-point Jacobi ETKF.  Shared memory: A [m][ld], V [m][ld] (or V in
// global scratch for large m), rotations, vectors.
struct PointArgs {
    const double* fields;
    int64_t P;
    int m, nx, ny;
    int64_t d;
    const double* x;
    double* out;
    double* vscratch;       // global V slots (kVGlobal)
    unsigned long long* singular;  // min point index with a singular transform
    int max_sweeps;
    // Newton-Schulz points that did not converge are listed here and redone
    // by the Jacobi kernel, which then walks only this list
    int64_t* redo;                 // [P] point indices
    unsigned int* redo_n;          // entries in `redo`
    bool from_list;                // letkf_point_kernel: iterate redo[0 .. *redo_n)
};

template <bool kVGlobal>
__global__ void __launch_bounds__(256) letkf_point_kernel(PointArgs a) {
    extern __shared__ double sm[];
    const int m = a.m;
    const int ld = m + 1;
    const int mp = m + (m & 1);  // even pairing size (a dummy index when m is odd)
    const int npairs = mp / 2;
    const int nblk = npairs * (npairs + 1) / 2;
    double* A = sm;
    double* V = kVGlobal ? a.vscratch + size_t(blockIdx.x) * size_t(m) * ld : A + size_t(m) * ld;
    double* rot = kVGlobal ? A + size_t(m) * ld : V + size_t(m) * ld;  // [npairs][3] c, s, t
    double* vec = rot + 3 * npairs;                                     // 3 x m
    double* b = vec;
    double* u = vec + m;
    double* pert = vec + 2 * m;
    int* pr = reinterpret_cast<int*>(vec + 3 * m);   // [npairs][2] p, q of this round
    int* blk = pr + 2 * npairs;                      // [nblk] (k1 << 16 | k2), k1 <= k2
    int* rotated = blk + nblk;                       // any rotation this sweep
    const int tid = threadIdx.x, nt = blockDim.x;
    const int E = m * (m + 1) / 2;
    const double sm1 = sqrt(double(m - 1));
    // loop strides over (pair, row) items without integer division
    const int vi0 = tid % m, vk0 = tid / m, vdi = nt % m, vdk = nt / m;
    for (int t = tid; t < nblk; t += nt) {
        int k1 = 0, r = t;
        while (r >= npairs - k1) {
            r -= npairs - k1;
            ++k1;
        }
        blk[t] = (k1 << 16) | (k1 + r);
    }

    const int64_t n_pts = a.from_list ? int64_t(*a.redo_n) : a.P;
    for (int64_t it_pt = blockIdx.x; it_pt < n_pts; it_pt += gridDim.x) {
        const int64_t pt = a.from_list ? a.redo[it_pt] : it_pt;
        const double count = a.fields[size_t(E + m) * a.P + pt];
        const int64_t row0 = pt, row1 = a.P + pt;
        if (!(count > 0.5)) {
            // no observation within reach: the background is kept
            // (proj/src/letkf.cpp:141)
            for (int j = tid; j < m; j += nt) {
                a.out[size_t(j) * a.d + row0] = a.x[size_t(j) * a.d + row0];
                a.out[size_t(j) * a.d + row1] = a.x[size_t(j) * a.d + row1];
            }
            continue;
        }
        for (int t = tid; t < E; t += nt) {
            // upper-triangle field t -> (i, j), mirrored
            int i = 0, r = t;
            while (r >= m - i) {
                r -= m - i;
                ++i;
            }
            const int j = i + r;
            const double v = a.fields[size_t(t) * a.P + pt] + (i == j ? double(m - 1) : 0.0);
            A[i * ld + j] = v;
            A[j * ld + i] = v;
        }
        for (int t = tid; t < m * ld; t += nt) V[t] = 0.0;
        for (int t = tid; t < m; t += nt) b[t] = a.fields[size_t(E + t) * a.P + pt];
        __syncthreads();
        for (int t = tid; t < m; t += nt) V[t * ld + t] = 1.0;

        // cyclic Jacobi, round-robin ordering: pair 0 = (r, mp-1), pair k =
        // ((r+k) mod (mp-1), (r-k) mod (mp-1)); a round applies its mp/2
        // disjoint rotations at once as A <- J^T A J, one 2x2 block of A per
        // thread-item (upper blocks, mirrored), and V <- V J.  A rotation is
        // skipped when |a_pq| <= eps sqrt(|a_pp a_qq|) (below double
        // rounding); converged = a sweep without one.
        for (int sweep = 0; sweep < a.max_sweeps; ++sweep) {
            if (tid == 0) *rotated = 0;
            __syncthreads();
            for (int rnd = 0; rnd < mp - 1; ++rnd) {
                for (int k = tid; k < npairs; k += nt) {
                    int p, q;
                    if (k == 0) {
                        p = rnd;
                        q = mp - 1;
                    } else {
                        p = rnd + k;
                        p -= p >= mp - 1 ? mp - 1 : 0;
                        q = rnd - k;
                        q += q < 0 ? mp - 1 : 0;
                    }
                    if (p > q) {
                        const int t = p;
                        p = q;
                        q = t;
                    }
                    double c = 1.0, s = 0.0, tt = 0.0;
                    if (q < m) {
                        const double apq = A[p * ld + q];
                        const double app = A[p * ld + p], aqq = A[q * ld + q];
                        if (fabs(apq) > 2.2e-16 * sqrt(fabs(app * aqq))) {
                            *rotated = 1;
                            // t = tan(phi) = sign(h) g / (|h| + sqrt(h^2 + g^2)),
                            // h = a_qq - a_pp, g = 2 a_pq (the small root)
                            const double h = aqq - app, g = 2.0 * apq;
                            tt = (h < 0.0 ? -g : g) / (fabs(h) + sqrt(fma(h, h, g * g)));
                            c = rsqrt(fma(tt, tt, 1.0));
                            s = tt * c;
                        }
                    }
                    rot[3 * k] = c;
                    rot[3 * k + 1] = s;
                    rot[3 * k + 2] = tt;
                    pr[2 * k] = p;
                    pr[2 * k + 1] = q;
                }
                __syncthreads();
                // A <- J^T A J on 2x2 blocks (rows of pair k1, columns of pair k2)
                for (int t = tid; t < nblk; t += nt) {
                    const int k1 = blk[t] >> 16, k2 = blk[t] & 0xffff;
                    const double s1 = rot[3 * k1 + 1], s2 = rot[3 * k2 + 1];
                    if (s1 == 0.0 && s2 == 0.0) continue;
                    const int p1 = pr[2 * k1], q1 = pr[2 * k1 + 1];
                    const int p2 = pr[2 * k2], q2 = pr[2 * k2 + 1];
                    if (k1 == k2) {
                        // the annihilated pair: closed form (a_pq -> 0)
                        const double tt = rot[3 * k1 + 2], apq = A[p1 * ld + q1];
                        A[p1 * ld + p1] -= tt * apq;
                        A[q1 * ld + q1] += tt * apq;
                        A[p1 * ld + q1] = 0.0;
                        A[q1 * ld + p1] = 0.0;
                        continue;
                    }
                    const double c1 = rot[3 * k1], c2 = rot[3 * k2];
                    const bool r1 = q1 < m, r2 = q2 < m;
                    const double x11 = A[p1 * ld + p2];
                    const double x12 = r2 ? A[p1 * ld + q2] : 0.0;
                    const double x21 = r1 ? A[q1 * ld + p2] : 0.0;
                    const double x22 = (r1 && r2) ? A[q1 * ld + q2] : 0.0;
                    // columns (J2), then rows (J1^T)
                    const double y11 = c2 * x11 - s2 * x12, y12 = s2 * x11 + c2 * x12;
                    const double y21 = c2 * x21 - s2 * x22, y22 = s2 * x21 + c2 * x22;
                    const double z11 = c1 * y11 - s1 * y21, z21 = s1 * y11 + c1 * y21;
                    const double z12 = c1 * y12 - s1 * y22, z22 = s1 * y12 + c1 * y22;
                    A[p1 * ld + p2] = z11;
                    A[p2 * ld + p1] = z11;
                    if (r2) {
                        A[p1 * ld + q2] = z12;
                        A[q2 * ld + p1] = z12;
                    }
                    if (r1) {
                        A[q1 * ld + p2] = z21;
                        A[p2 * ld + q1] = z21;
                    }
                    if (r1 && r2) {
                        A[q1 * ld + q2] = z22;
                        A[q2 * ld + q1] = z22;
                    }
                }
                // V <- V J (rows i, columns p, q of every pair)
                for (int i = vi0, k = vk0; k < npairs;) {
                    const double s = rot[3 * k + 1];
                    const int q = pr[2 * k + 1];
                    if (s != 0.0 && q < m) {
                        const int p = pr[2 * k];
                        const double c = rot[3 * k];
                        const double vp = V[i * ld + p], vq = V[i * ld + q];
                        V[i * ld + p] = c * vp - s * vq;
                        V[i * ld + q] = s * vp + c * vq;
                    }
                    i += vdi;
                    k += vdk;
                    if (i >= m) {
                        i -= m;
                        ++k;
                    }
                }
                __syncthreads();
            }
            if (*rotated == 0) break;
            __syncthreads();
        }
        // eigenvalues on the diagonal; a non-positive or non-finite one is a
        // SingularAnalysisError (proj/src/letkf.cpp:40-44)
        bool bad = false;
        for (int i = tid; i < m; i += nt) {
            const double l = A[i * ld + i];
            if (!(l > 0.0) || !isfinite(l)) bad = true;
        }
        if (__syncthreads_or(bad)) {
            if (tid == 0) atomicMin(a.singular, (unsigned long long)pt);
            continue;
        }
        // wbar = V L^-1 V^T b  ->  u = L^-1 (V^T b) then wbar = V u
        for (int i = tid; i < m; i += nt) {
            double s = 0.0;
            for (int k = 0; k < m; ++k) s += V[k * ld + i] * b[k];
            u[i] = s / A[i * ld + i];
        }
        __syncthreads();
        for (int i = tid; i < m; i += nt) {
            double s = 0.0;
            for (int k = 0; k < m; ++k) s += V[i * ld + k] * u[k];
            pert[i] = s;  // wbar, parked
        }
        __syncthreads();
        for (int i = tid; i < m; i += nt) b[i] = pert[i];  // b <- wbar
        __syncthreads();
        // both levels with the same transform (proj/src/letkf.cpp:162-171)
        for (int lev = 0; lev < 2; ++lev) {
            const int64_t row = lev ? row1 : row0;
            // ensemble_mean: member-order sum times 1/m (proj/src/ensemble.cpp:7-16)
            double mean = 0.0;
            for (int j = 0; j < m; ++j) mean += a.x[size_t(j) * a.d + row];
            mean *= 1.0 / double(m);
            for (int j = tid; j < m; j += nt) pert[j] = a.x[size_t(j) * a.d + row] - mean;
            __syncthreads();
            // u = L^-1/2 V^T pert
            for (int i = tid; i < m; i += nt) {
                double s = 0.0;
                for (int k = 0; k < m; ++k) s += V[k * ld + i] * pert[k];
                u[i] = s / sqrt(A[i * ld + i]);
            }
            double wx = 0.0;
            for (int k = 0; k < m; ++k) wx += pert[k] * b[k];
            __syncthreads();
            for (int j = tid; j < m; j += nt) {
                double s = 0.0;
                for (int k = 0; k < m; ++k) s += V[j * ld + k] * u[k];
                a.out[size_t(j) * a.d + row] = mean + wx + sm1 * s;
            }
            __syncthreads();
        }
    }
}

// 5'. M <= 64: the transform without an eigendecomposition.  ETKF needs
// only A^-1 b and W = sqrt(M-1) A^-1/2 (proj/src/letkf.cpp:46-53): with
// B = A / c the coupled Newton-Schulz iteration
//     T = 3I - Z Y,   Y <- Y T / 2,   Z <- T Z / 2     (Y0 = B, Z0 = I)
// converges quadratically to Y = B^1/2, Z = B^-1/2 whenever the spectrum of
// B lies in (0, 2).  A >= (M-1) I and lambda_max <= ||A||_inf, so
// c = (M-1 + ||A||_inf) / 2 qualifies, and the iteration count follows from
// the scalar recurrence p <- p (3 - p)^2 / 4 at both spectrum ends.  Every
// product is a 64 x 64 x 64 fp64 GEMM on the FP64 tensor cores
// (DMMA.8x8x4): ~10 iterations x 3 GEMMs replace ~570 Jacobi rounds.
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// C = X Y for the Newton-Schulz iterates: warp w owns one block of 2 x 4
// tiles (8 x 8 each) of the output, accumulators in registers until the
// caller's barrier, so C may overwrite X or Y.  The full product is formed:
// the iterates are symmetric in exact arithmetic, but mirroring the upper
// triangle breaks the coupled iteration's self-correction and diverges for
// condition numbers >= 1e4 (measured on the numpy model of this kernel).
template <int NT8>
struct NsGemm {
    static constexpr int nbr = (NT8 + 1) / 2, nbc = (NT8 + 3) / 4;
    bool own;
    int br, bc;
    double acc[2][4][2];

    __device__ __forceinline__ void setup(int warp) {
        own = warp < nbr * nbc;
        br = own ? warp / nbc : 0;
        bc = own ? warp % nbc : 0;
    }

    __device__ __forceinline__ void compute(const double* X, const double* Y, int ld, int lane) {
        constexpr int mp = 8 * NT8;
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[r][q][0] = acc[r][q][1] = 0.0;
        if (!own) return;
        const int lr = lane >> 2, lk = lane & 3;
#pragma unroll 4
        for (int k0 = 0; k0 < mp; k0 += 4) {
            const int kk = k0 + lk;
            double av[2], bv[4];
#pragma unroll
            for (int r = 0; r < 2; ++r)
                av[r] = 2 * br + r < NT8 ? X[(16 * br + 8 * r + lr) * ld + kk] : 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                bv[q] = 4 * bc + q < NT8 ? Y[kk * ld + 32 * bc + 8 * q + lr] : 0.0;
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int q = 0; q < 4; ++q) dmma884(acc[r][q], av[r], bv[q]);
        }
    }

    // C = alpha acc + beta I; returns the local max |acc - I| (the
    // Newton-Schulz residual when X Y ~ I)
    __device__ __forceinline__ double store(double* C, int ld, int lane, double alpha,
                                            double beta) const {
        double res = 0.0;
        if (!own) return res;
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int tr = 2 * br + r, tc = 4 * bc + q;
                if (tr >= NT8 || tc >= NT8) continue;
                const int row = 8 * tr + (lane >> 2);
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int col = 8 * tc + 2 * (lane & 3) + e;
                    const double v = acc[r][q][e];
                    res = fmax(res, fabs(v - (row == col ? 1.0 : 0.0)));
                    C[row * ld + col] = alpha * v + (row == col ? beta : 0.0);
                }
            }
        return res;
    }
};

template <int NT8>
__global__ void __launch_bounds__(256) letkf_point_ns_kernel(PointArgs a) {
    extern __shared__ double sm[];
    const int m = a.m;
    constexpr int mp = 8 * NT8;
    const int ld = mp + 4;
    double* Y = sm;
    double* Z = Y + size_t(mp) * ld;
    double* T = Z + size_t(mp) * ld;
    double* vec = T + size_t(mp) * ld;  // b, u, pert, wbar [mp] each + reduction
    double* b = vec;
    double* u = vec + mp;
    double* pert = vec + 2 * mp;
    double* wbar = vec + 3 * mp;
    double* red = vec + 4 * mp;  // [8]
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    NsGemm<NT8> g;
    g.setup(warp);
    const int E = m * (m + 1) / 2;
    const double sm1 = sqrt(double(m - 1));

    for (int64_t pt = blockIdx.x; pt < a.P; pt += gridDim.x) {
        const double count = a.fields[size_t(E + m) * a.P + pt];
        const int64_t row0 = pt, row1 = a.P + pt;
        if (!(count > 0.5)) {
            for (int j = tid; j < m; j += nt) {
                a.out[size_t(j) * a.d + row0] = a.x[size_t(j) * a.d + row0];
                a.out[size_t(j) * a.d + row1] = a.x[size_t(j) * a.d + row1];
            }
            continue;
        }
        // A (mirrored upper fields) into T; padded rows/cols: identity
        for (int t = tid; t < mp * mp; t += nt) {
            const int i = t / mp, j = t - (t / mp) * mp;
            double v;
            if (i < m && j < m) {
                const int lo = min(i, j), hi = max(i, j);
                const int f = lo * m - (lo * (lo - 1)) / 2 + (hi - lo);
                v = a.fields[size_t(f) * a.P + pt] + (i == j ? double(m - 1) : 0.0);
            } else {
                v = i == j ? 1.0 : 0.0;
            }
            T[i * ld + j] = v;
        }
        for (int t = tid; t < mp; t += nt) b[t] = t < m ? a.fields[size_t(E + t) * a.P + pt] : 0.0;
        __syncthreads();
        // ||A||_inf (max absolute row sum)
        double rs = 0.0;
        for (int i = tid; i < m; i += nt) {
            double s = 0.0;
            for (int j = 0; j < m; ++j) s += fabs(T[i * ld + j]);
            rs = fmax(rs, s);
        }
        for (int o = 16; o; o >>= 1) rs = fmax(rs, __shfl_xor_sync(0xffffffffu, rs, o));
        if (lane == 0) red[warp] = rs;
        __syncthreads();
        double ainf = 0.0;
        for (int w = 0; w < nt / 32; ++w) ainf = fmax(ainf, red[w]);
        const double cs = 0.5 * (double(m - 1) + ainf);
        const double inv_c = 1.0 / cs;
        // Y0 = B = A / c (padding keeps eigenvalue 1), Z0 = I
        for (int t = tid; t < mp * mp; t += nt) {
            const int i = t / mp, j = t - (t / mp) * mp;
            const bool pad = i >= m || j >= m;
            Y[i * ld + j] = pad ? T[i * ld + j] : T[i * ld + j] * inv_c;
            Z[i * ld + j] = i == j ? 1.0 : 0.0;
        }
        const bool finite = isfinite(cs) && cs > 0.0;
        __syncthreads();
        // iterate until ||Z Y - I||_max <= 1e-10 (the next update squares the
        // error below double rounding), at most 60 times; the final
        // iteration skips the Y update nobody reads
        bool converged = false;
        for (int it = 0; finite && it < a.max_sweeps; ++it) {
            // T = 3I - Z Y, with the residual max |T - 2I| = max |Z Y - I|
            g.compute(Z, Y, ld, lane);
            double res = g.store(T, ld, lane, -1.0, 3.0);
            for (int o = 16; o; o >>= 1) res = fmax(res, __shfl_xor_sync(0xffffffffu, res, o));
            if (lane == 0) red[warp] = res;
            __syncthreads();
            res = 0.0;
            for (int w = 0; w < nt / 32; ++w) res = fmax(res, red[w]);
            const bool last = !(res > 1e-10);  // (fmax drops NaN: caught below)
            converged = last;
            if (!last) {
                // Y <- Y T / 2 (in place once every warp has read Y)
                g.compute(Y, T, ld, lane);
                __syncthreads();
                g.store(Y, ld, lane, 0.5, 0.0);
            }
            // Z <- T Z / 2
            g.compute(T, Z, ld, lane);
            __syncthreads();
            g.store(Z, ld, lane, 0.5, 0.0);
            __syncthreads();
            if (last) break;
        }
        // A^-1/2 = Z / sqrt(c); a non-finite transform is a
        // SingularAnalysisError (proj/src/letkf.cpp:40-44)
        bool bad = !finite;
        for (int t = tid; t < m * m && !bad; t += nt) {
            const int i = t / m, j = t - (t / m) * m;
            if (!isfinite(Z[i * ld + j])) bad = true;
        }
        if (__syncthreads_or(bad)) {
            if (tid == 0) atomicMin(a.singular, (unsigned long long)pt);
            continue;
        }
        if (!converged) {
            // still above the residual bound after 60 iterations (rounding-
            // limited or stalled): the Jacobi eigensolver redoes this point
            if (tid == 0) {
                const unsigned slot = atomicAdd(a.redo_n, 1u);
                TB_CHECK(int64_t(slot) < a.P);
                a.redo[slot] = pt;
            }
            continue;
        }
        const double isc = rsqrt(cs);
        // wbar = A^-1 b = (Z (Z b)) / c
        for (int i = tid; i < m; i += nt) {
            double s = 0.0;
            for (int k = 0; k < m; ++k) s += Z[i * ld + k] * b[k];
            u[i] = s;
        }
        __syncthreads();
        for (int i = tid; i < m; i += nt) {
            double s = 0.0;
            for (int k = 0; k < m; ++k) s += Z[i * ld + k] * u[k];
            wbar[i] = s * inv_c;
        }
        __syncthreads();
        // both levels with the same transform (proj/src/letkf.cpp:162-171)
        for (int lev = 0; lev < 2; ++lev) {
            const int64_t row = lev ? row1 : row0;
            for (int j = tid; j < m; j += nt) u[j] = a.x[size_t(j) * a.d + row];
            __syncthreads();
            // ensemble_mean: member-order sum times 1/m (proj/src/ensemble.cpp:7-16)
            double mean = 0.0;
            for (int j = 0; j < m; ++j) mean += u[j];
            mean *= 1.0 / double(m);
            for (int j = tid; j < m; j += nt) pert[j] = u[j] - mean;
            __syncthreads();
            double wx = 0.0;
            for (int k = 0; k < m; ++k) wx += pert[k] * wbar[k];
            for (int j = tid; j < m; j += nt) {
                double s = 0.0;
                for (int k = 0; k < m; ++k) s += Z[j * ld + k] * pert[k];
                a.out[size_t(j) * a.d + row] = mean + wx + sm1 * (s * isc);
            }
            __syncthreads();
        }
    }
}

// 6. RTPS, proj/src/letkf.cpp:177-207 (in place on the analysis)
__global__ void rtps_kernel(double* __restrict__ an, const double* __restrict__ bg, int m,
                            int64_t d, double alpha) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= d) return;
    const double inv = 1.0 / double(m);
    double ma = 0.0, mb = 0.0;
    for (int j = 0; j < m; ++j) {
        ma += an[size_t(j) * d + k];
        mb += bg[size_t(j) * d + k];
    }
    ma *= inv;
    mb *= inv;
    double va = 0.0, vb = 0.0;
    for (int j = 0; j < m; ++j) {
        const double da = an[size_t(j) * d + k] - ma;
        const double db = bg[size_t(j) * d + k] - mb;
        va += da * da;
        vb += db * db;
    }
    const double sa = fmax(sqrt(va / double(m - 1)), 1e-12);
    const double sb = sqrt(vb / double(m - 1));
    const double scale = 1.0 + alpha * (sb - sa) / sa;
    for (int j = 0; j < m; ++j) {
        double& v = an[size_t(j) * d + k];
        v = ma + scale * (v - ma);
    }
}

unsigned blocks_for(int64_t n, int t) { return unsigned((n + t - 1) / t); }

// ---------------------------------------------------------------------------
// host orchestration
struct SpectrumKey {
    int nx;
    double cutoff;
    bool operator<(const SpectrumKey& o) const {
        return nx != o.nx ? nx < o.nx : cutoff < o.cutoff;
    }
};

struct LetkfWorkspace {
    std::mutex mu;
    cudaStream_t stream = nullptr;
    Buf x, y, r, idx, locs, out;
    Buf yb, dinn, rinv, cell, cell_sorted, order, sorted_obs, count, start, cub_tmp;
    Buf fields, spec, vscratch, singular, redo;
    std::map<SpectrumKey, std::unique_ptr<Buf>> khat;
    int plan_nx = 0, plan_batch = 0;
    cufftHandle d2z = 0, z2d = 0;
    cudaStream_t plan_stream = nullptr;
};

LetkfWorkspace* workspace(int dev) {
    static std::mutex mu;
    static std::map<int, std::unique_ptr<LetkfWorkspace>> ws;
    std::lock_guard<std::mutex> lk(mu);
    auto& w = ws[dev];
    if (!w) w = std::make_unique<LetkfWorkspace>();
    return w.get();
}

constexpr int kFftBatchCap = 1 << 27;  // doubles per FFT batch (~1 GB of spectra)

int ensure_plans(LetkfWorkspace* w, int n, int batch, cudaStream_t s, turbda_status* st) {
    if (w->plan_nx != n || w->plan_batch != batch) {
        if (w->d2z) cufftDestroy(w->d2z);
        if (w->z2d) cufftDestroy(w->z2d);
        w->d2z = w->z2d = 0;
        int dims[2] = {n, n};
        const int nh = n * (n / 2 + 1);
        LK_FFT(cufftPlanMany(&w->d2z, 2, dims, nullptr, 1, n * n, nullptr, 1, nh, CUFFT_D2Z, batch));
        LK_FFT(cufftPlanMany(&w->z2d, 2, dims, nullptr, 1, nh, nullptr, 1, n * n, CUFFT_Z2D, batch));
        w->plan_nx = n;
        w->plan_batch = batch;
        w->plan_stream = nullptr;
    }
    if (w->plan_stream != s) {
        LK_FFT(cufftSetStream(w->d2z, s));
        LK_FFT(cufftSetStream(w->z2d, s));
        w->plan_stream = s;
    }
    return TURBDA_OK;
}

// real spectrum (scaled by 1/P) of the periodic Gaspari-Cohn stencil
int stencil_spectrum(LetkfWorkspace* w, int n, double cutoff, cudaStream_t s, const double** out,
                     turbda_status* st) {
    auto& slot = w->khat[SpectrumKey{n, cutoff}];
    if (!slot) {
        const int64_t P = int64_t(n) * n;
        const int64_t nh = int64_t(n) * (n / 2 + 1);
        // [0]: Gaspari-Cohn weights, [1]: support indicator (r < 2)
        std::vector<double> k(2 * size_t(P), 0.0);
        for (int oy = 0; oy < n; ++oy)
            for (int ox = 0; ox < n; ++ox) {
                const int ax = std::min(ox, n - ox), ay = std::min(oy, n - oy);
                const double rr = std::hypot(double(ax), double(ay)) / cutoff;
                k[size_t(oy) * n + ox] = rr < 2.0 ? gc_weight(rr) : 0.0;
                k[size_t(P) + size_t(oy) * n + ox] = rr < 2.0 ? 1.0 : 0.0;
            }
        Buf kd, kc;
        LK_CUDA(kd.reserve(sizeof(double) * 2 * size_t(P)));
        LK_CUDA(kc.reserve(sizeof(cufftDoubleComplex) * 2 * size_t(nh)));
        LK_CUDA(cudaMemcpyAsync(kd.p, k.data(), sizeof(double) * 2 * size_t(P),
                                cudaMemcpyHostToDevice, s));
        cufftHandle plan = 0;
        int dims[2] = {n, n};
        LK_FFT(cufftPlanMany(&plan, 2, dims, nullptr, 1, int(P), nullptr, 1, int(nh), CUFFT_D2Z, 2));
        cufftSetStream(plan, s);
        const cufftResult fr = cufftExecD2Z(plan, kd.as<double>(), kc.as<cufftDoubleComplex>());
        cufftDestroy(plan);
        if (fr != CUFFT_SUCCESS) return fail(st, TURBDA_CUDA, "letkf: stencil spectrum FFT failed");
        std::vector<cufftDoubleComplex> hc(2 * size_t(nh));
        LK_CUDA(cudaMemcpyAsync(hc.data(), kc.p, sizeof(cufftDoubleComplex) * 2 * size_t(nh),
                                cudaMemcpyDeviceToHost, s));
        LK_CUDA(cudaStreamSynchronize(s));
        // both stencils are even (K(o) = K(-o)), so their spectra are real
        std::vector<double> hr(2 * size_t(nh));
        for (size_t t = 0; t < hr.size(); ++t) hr[t] = hc[t].x / double(P);
        auto b = std::make_unique<Buf>();
        LK_CUDA(b->reserve(sizeof(double) * 2 * size_t(nh)));
        LK_CUDA(cudaMemcpyAsync(b->p, hr.data(), sizeof(double) * 2 * size_t(nh),
                                cudaMemcpyHostToDevice, s));
        LK_CUDA(cudaStreamSynchronize(s));
        slot = std::move(b);
    }
    *out = slot->as<double>();
    return TURBDA_OK;
}

bool pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

int validate(const turbda_letkf_params* p, turbda_status* st) {
    if (!p) return fail(st, TURBDA_CONFIG, "letkf: null params");
    // LetkfConfig::validate, proj/include/turbda/letkf.hpp:18-24
    if (!(p->cutoff_km > 0.0) || !(p->domain_km > 0.0))
        return fail(st, TURBDA_CONFIG, "letkf: cutoff_km, domain_km > 0");
    if (!(p->rtps_alpha >= 0.0 && p->rtps_alpha <= 1.0))
        return fail(st, TURBDA_CONFIG, "letkf: rtps_alpha in [0, 1]");
    // GridSpec::validate (proj/include/turbda/grid.hpp:32-38) + isotropy (letkf.cpp:62-63)
    if (!pow2(p->nx) || !pow2(p->ny) || p->nx < 8 || p->ny < 8)
        return fail(st, TURBDA_CONFIG, "grid: nx, ny must be powers of two >= 8");
    if (p->nx != p->ny)
        return fail(st, TURBDA_CONFIG, "letkf_analyze: isotropic metric needs nx == ny");
    if (p->n_members < 1) return fail(st, TURBDA_DIMENSION, "ensemble: empty");
    if (p->obs_kind < 0 || p->obs_kind > 3)
        return fail(st, TURBDA_CONFIG, "observation: unsupported operator kind");
    const int64_t d = 2 * int64_t(p->nx) * p->ny;
    if (p->obs_dim < 0) return fail(st, TURBDA_DIMENSION, "observation: negative obs_dim");
    if ((p->obs_kind == 0 || p->obs_kind == 2) && p->obs_dim != d)
        return fail(st, TURBDA_DIMENSION, "letkf_analyze: state/grid size mismatch");
    return TURBDA_OK;
}

}  // namespace
}  // namespace tb200

using namespace tb200;

extern "C" {

void turbda_letkf_params_init(turbda_letkf_params* p) {
    if (!p) return;
    std::memset(p, 0, sizeof(*p));
    p->nx = p->ny = 64;
    p->n_members = 20;
    p->obs_kind = 0;
    p->obs_dim = 2 * 64 * 64;
    // LetkfConfig defaults, proj/include/turbda/letkf.hpp:13-16
    p->cutoff_km = 2000.0;
    p->domain_km = 20000.0;
    p->rtps_alpha = 0.3;
    p->device = -1;
}

int turbda_gaspari_cohn(double r, double* out, turbda_status* st) {
    clear(st);
    if (r < 0.0 || std::isnan(r)) return fail(st, TURBDA_CONFIG, "gaspari_cohn: r >= 0");
    if (out) *out = gc_weight(r);
    return TURBDA_OK;
}

int turbda_letkf_analyze(const turbda_letkf_params* p, const double* forecast, const double* y,
                         const double* r_diag, const int64_t* obs_idx, const double* locations,
                         double* analysis_out, void* stream, turbda_status* st) {
    clear(st);
    if (int rc = validate(p, st)) return rc;
    const bool on_dev = (p->flags & TURBDA_INPUTS_ON_DEVICE) != 0;
    const bool r_uni = (p->flags & TURBDA_R_UNIFORM) != 0;
    const bool dense = p->obs_kind == 0 || p->obs_kind == 2;
    const int m = p->n_members, n = p->nx;
    const int64_t P = int64_t(n) * n, d = 2 * P, nobs = p->obs_dim;
    if (!forecast || !analysis_out || (nobs > 0 && (!y || !r_diag)) ||
        (!dense && nobs > 0 && !obs_idx))
        return fail(st, TURBDA_CONFIG, "letkf: null array");
    if (!on_dev) {
        // Observation::validate (positive variances, indices inside the state)
        const int64_t nr = r_uni ? std::min<int64_t>(nobs, 1) : nobs;
        for (int64_t q = 0; q < nr; ++q)
            if (!(r_diag[q] > 0.0)) return fail(st, TURBDA_CONFIG, "observation: r_diag > 0");
        if (!dense)
            for (int64_t q = 0; q < nobs; ++q)
                if (obs_idx[q] < 0 || obs_idx[q] >= d)
                    return fail(st, TURBDA_DIMENSION, "observation: index outside the state");
    }
    int dev = p->device;
    if (dev < 0) {
        if (cudaGetDevice(&dev) != cudaSuccess) return fail(st, TURBDA_CUDA, "no CUDA device");
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || dev >= ndev)
        return fail(st, TURBDA_CUDA, "no such CUDA device");
    LK_CUDA(cudaSetDevice(dev));
    LetkfWorkspace* w = workspace(dev);
    std::lock_guard<std::mutex> lk(w->mu);
    if (!w->stream) LK_CUDA(cudaStreamCreateWithFlags(&w->stream, cudaStreamNonBlocking));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : (on_dev ? cudaStreamLegacy : w->stream);

    const double *dx = forecast, *dy = y, *dr = r_diag, *dl = locations;
    const int64_t* didx = obs_idx;
    double* dout = analysis_out;
    const size_t md = size_t(m) * size_t(d);
    const int64_t nb = std::max<int64_t>(nobs, 1);
    if (!on_dev) {
        LK_CUDA(w->x.reserve(sizeof(double) * md));
        LK_CUDA(w->out.reserve(sizeof(double) * md));
        LK_CUDA(w->y.reserve(sizeof(double) * size_t(nb)));
        LK_CUDA(w->r.reserve(sizeof(double) * size_t(nb)));
        LK_CUDA(cudaMemcpyAsync(w->x.p, forecast, sizeof(double) * md, cudaMemcpyHostToDevice, s));
        if (nobs > 0) {
            LK_CUDA(cudaMemcpyAsync(w->y.p, y, sizeof(double) * size_t(nobs), cudaMemcpyHostToDevice, s));
            LK_CUDA(cudaMemcpyAsync(w->r.p, r_diag, sizeof(double) * size_t(r_uni ? 1 : nobs),
                                    cudaMemcpyHostToDevice, s));
        }
        if (!dense && nobs > 0) {
            LK_CUDA(w->idx.reserve(sizeof(int64_t) * size_t(nb)));
            LK_CUDA(cudaMemcpyAsync(w->idx.p, obs_idx, sizeof(int64_t) * size_t(nobs),
                                    cudaMemcpyHostToDevice, s));
            didx = w->idx.as<int64_t>();
        }
        if (locations && nobs > 0) {
            LK_CUDA(w->locs.reserve(sizeof(double) * 2 * size_t(nb)));
            LK_CUDA(cudaMemcpyAsync(w->locs.p, locations, sizeof(double) * 2 * size_t(nobs),
                                    cudaMemcpyHostToDevice, s));
            dl = w->locs.as<double>();
        }
        dx = w->x.as<double>();
        dy = w->y.as<double>();
        dr = w->r.as<double>();
        dout = w->out.as<double>();
    }
    if (dense) didx = nullptr;

    // 1-2. observation space + bucketing by cell
    const int E = m * (m + 1) / 2;
    const int nf = E + m + 1;
    LK_CUDA(w->yb.reserve(sizeof(double) * size_t(m) * size_t(nb)));
    LK_CUDA(w->dinn.reserve(sizeof(double) * size_t(nb)));
    LK_CUDA(w->rinv.reserve(sizeof(double) * size_t(nb)));
    LK_CUDA(w->cell.reserve(sizeof(uint32_t) * size_t(nb)));
    LK_CUDA(w->cell_sorted.reserve(sizeof(uint32_t) * size_t(nb)));
    LK_CUDA(w->order.reserve(sizeof(uint32_t) * size_t(nb)));
    LK_CUDA(w->sorted_obs.reserve(sizeof(uint32_t) * size_t(nb)));
    LK_CUDA(w->count.reserve(sizeof(int) * size_t(P + 1)));
    LK_CUDA(w->start.reserve(sizeof(int) * size_t(P + 1)));
    LK_CUDA(w->singular.reserve(sizeof(unsigned long long) + sizeof(unsigned int)));
    LK_CUDA(cudaMemsetAsync(w->singular.p, 0xff, sizeof(unsigned long long), s));
    unsigned int* redo_n = reinterpret_cast<unsigned int*>(w->singular.as<unsigned char>() + 8);
    LK_CUDA(cudaMemsetAsync(redo_n, 0, sizeof(unsigned int), s));
    LK_CUDA(w->redo.reserve(sizeof(int64_t) * size_t(std::max<int64_t>(P, 1))));
    LK_CUDA(cudaMemsetAsync(w->count.p, 0, sizeof(int) * size_t(P + 1), s));
    if (nobs > 0) {
        letkf_obs_kernel<<<blocks_for(nobs, 256), 256, 0, s>>>(
            dx, d, m, didx, nobs, (p->obs_kind >= 2) ? 1 : 0, dy, dr, r_uni ? 0 : 1, dl, n, n,
            w->yb.as<double>(), w->dinn.as<double>(), w->rinv.as<double>(),
            w->cell.as<uint32_t>(), w->order.as<uint32_t>());
        LK_CUDA(cudaGetLastError());
        add_launches(2);
        count_cells_kernel<<<blocks_for(nobs, 256), 256, 0, s>>>(w->cell.as<uint32_t>(), nobs,
                                                                  w->count.as<int>());
        LK_CUDA(cudaGetLastError());
        int bits = 1;
        while ((int64_t(1) << bits) < P) ++bits;
        size_t tmp_sort = 0, tmp_scan = 0;
        LK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_sort, w->cell.as<uint32_t>(),
                                                w->cell_sorted.as<uint32_t>(),
                                                w->order.as<uint32_t>(),
                                                w->sorted_obs.as<uint32_t>(), int(nobs), 0, bits, s));
        LK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_scan, w->count.as<int>(),
                                              w->start.as<int>(), int(P + 1), s));
        LK_CUDA(w->cub_tmp.reserve(std::max(tmp_sort, tmp_scan)));
        LK_CUDA(cub::DeviceRadixSort::SortPairs(w->cub_tmp.p, tmp_sort, w->cell.as<uint32_t>(),
                                                w->cell_sorted.as<uint32_t>(),
                                                w->order.as<uint32_t>(),
                                                w->sorted_obs.as<uint32_t>(), int(nobs), 0, bits, s));
        LK_CUDA(cub::DeviceScan::ExclusiveSum(w->cub_tmp.p, tmp_scan, w->count.as<int>(),
                                              w->start.as<int>(), int(P + 1), s));
    } else {
        LK_CUDA(cudaMemsetAsync(w->start.p, 0, sizeof(int) * size_t(P + 1), s));
    }

    // 3. per-cell fields (padded to whole FFT batches)
    const int cap = int(std::max<int64_t>(1, std::min<int64_t>(nf, kFftBatchCap / P)));
    const int nchunks = (nf + cap - 1) / cap;
    const int batch = (nf + nchunks - 1) / nchunks;
    const int nf_pad = nchunks * batch;
    const int64_t nh = int64_t(n) * (n / 2 + 1);
    LK_CUDA(w->fields.reserve(sizeof(double) * size_t(nf_pad) * size_t(P)));
    LK_CUDA(w->spec.reserve(sizeof(cufftDoubleComplex) * size_t(batch) * size_t(nh)));
    {
        dim3 grid(blocks_for(P, kFieldCells), unsigned((nf + kFieldChunk - 1) / kFieldChunk));
        letkf_fields_kernel<<<grid, kFieldCells, 0, s>>>(
            w->yb.as<double>(), w->dinn.as<double>(), w->rinv.as<double>(),
            w->sorted_obs.as<uint32_t>(), w->start.as<int>(), nobs, m, P, nf,
            w->fields.as<double>());
        LK_CUDA(cudaGetLastError());
        add_launches(1);
    }
    // 4. localization = periodic convolution with the Gaspari-Cohn stencil
    const double cutoff = p->cutoff_km / p->domain_km * double(n);
    const double* khat = nullptr;
    if (int rc = stencil_spectrum(w, n, cutoff, s, &khat, st)) return rc;
    if (int rc = ensure_plans(w, n, batch, s, st)) return rc;
    for (int f0 = 0; f0 < nf; f0 += batch) {
        double* fb = w->fields.as<double>() + size_t(f0) * size_t(P);
        auto* g = w->spec.as<cufftDoubleComplex>();
        LK_FFT(cufftExecD2Z(w->d2z, fb, g));
        const int64_t total = int64_t(batch) * nh;
        spectral_scale_kernel<<<blocks_for(total, 256), 256, 0, s>>>(g, khat, nh, total, f0,
                                                                      nf - 1);
        LK_CUDA(cudaGetLastError());
        add_launches(1);
        LK_FFT(cufftExecZ2D(w->z2d, g, fb));
    }
    // 5. per-point eigensolve + transform
    {
        const int threads = m > 32 ? 256 : 128;
        const int npairs = (m + (m & 1)) / 2;
        const size_t ld = size_t(m) + 1;
        const size_t mat = sizeof(double) * size_t(m) * ld;
        const size_t nblk = size_t(npairs) * (npairs + 1) / 2;
        const size_t extra = sizeof(double) * (3 * size_t(npairs) + 3 * size_t(m)) +
                             sizeof(int) * (2 * size_t(npairs) + nblk + 2);
        int dev_smem = 0, nsm = 0;
        LK_CUDA(cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        LK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        const bool ns = m <= 64;
        if (ns) {
            // tensor-core Newton-Schulz transform
            const int mp = (m + 7) & ~7;
            const size_t smem_ns = sizeof(double) * (3 * size_t(mp) * (mp + 4) + 4 * size_t(mp) + 8);
            PointArgs pn{};
            pn.fields = w->fields.as<double>();
            pn.P = P;
            pn.m = m;
            pn.nx = n;
            pn.ny = n;
            pn.d = d;
            pn.x = dx;
            pn.out = dout;
            pn.singular = w->singular.as<unsigned long long>();
            pn.redo = w->redo.as<int64_t>();
            pn.redo_n = redo_n;
            // iteration cap (60; TURBDA_LETKF_NS_ITERS lowers it in tests to
            // force the Jacobi redo of unconverged points)
            static const int ns_iters = [] {
                const char* e = std::getenv("TURBDA_LETKF_NS_ITERS");
                return e ? std::max(1, std::atoi(e)) : 60;
            }();
            pn.max_sweeps = ns_iters;
            void (*kern)(PointArgs) = nullptr;
            switch (mp / 8) {
                case 1: kern = letkf_point_ns_kernel<1>; break;
                case 2: kern = letkf_point_ns_kernel<2>; break;
                case 3: kern = letkf_point_ns_kernel<3>; break;
                case 4: kern = letkf_point_ns_kernel<4>; break;
                case 5: kern = letkf_point_ns_kernel<5>; break;
                case 6: kern = letkf_point_ns_kernel<6>; break;
                case 7: kern = letkf_point_ns_kernel<7>; break;
                default: kern = letkf_point_ns_kernel<8>; break;
            }
            LK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem_ns)));
            int per_sm_ns = 0;
            LK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_ns, kern, 256, smem_ns));
            const int64_t grid_ns = std::min<int64_t>(P, int64_t(std::max(per_sm_ns, 1)) * nsm);
            kern<<<unsigned(grid_ns), 256, smem_ns, s>>>(pn);
            LK_CUDA(cudaGetLastError());
            add_launches(1);
        }
        // parallel cyclic Jacobi: every point for M > 64; otherwise only the
        // points whose Newton-Schulz iteration did not converge (the kernel
        // reads their count on the device and exits when there are none)
        const bool vglobal = 2 * mat + extra + 64 > size_t(dev_smem);
        const size_t smem = (vglobal ? mat : 2 * mat) + extra + 64;
        if (smem > size_t(dev_smem))
            return fail(st, TURBDA_CONFIG, "letkf: ensemble too large for the per-point solver");
        PointArgs pa{};
        pa.fields = w->fields.as<double>();
        pa.P = P;
        pa.m = m;
        pa.nx = n;
        pa.ny = n;
        pa.d = d;
        pa.x = dx;
        pa.out = dout;
        pa.singular = w->singular.as<unsigned long long>();
        pa.max_sweeps = 40;
        pa.redo = w->redo.as<int64_t>();
        pa.redo_n = redo_n;
        pa.from_list = ns;
        int per_sm = 0;
        if (vglobal) {
            LK_CUDA(cudaFuncSetAttribute(letkf_point_kernel<true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            LK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, letkf_point_kernel<true>,
                                                                  threads, smem));
        } else {
            LK_CUDA(cudaFuncSetAttribute(letkf_point_kernel<false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            LK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, letkf_point_kernel<false>,
                                                                  threads, smem));
        }
        const int64_t grid = std::min<int64_t>(ns ? std::min<int64_t>(P, nsm) : P,
                                               int64_t(std::max(per_sm, 1)) * nsm);
        if (vglobal) {
            LK_CUDA(w->vscratch.reserve(mat * size_t(grid)));
            pa.vscratch = w->vscratch.as<double>();
            letkf_point_kernel<true><<<unsigned(grid), threads, smem, s>>>(pa);
        } else {
            letkf_point_kernel<false><<<unsigned(grid), threads, smem, s>>>(pa);
        }
        LK_CUDA(cudaGetLastError());
        add_launches(1);
    }
    // 6. RTPS (alpha == 0 or a single member: the analysis is returned as is)
    if (p->rtps_alpha != 0.0 && m >= 2) {
        rtps_kernel<<<blocks_for(d, 256), 256, 0, s>>>(dout, dx, m, d, p->rtps_alpha);
        LK_CUDA(cudaGetLastError());
        add_launches(1);
    }
    unsigned long long sing = 0;
    LK_CUDA(cudaMemcpyAsync(&sing, w->singular.p, sizeof(sing), cudaMemcpyDeviceToHost, s));
    if (!on_dev) LK_CUDA(cudaMemcpyAsync(analysis_out, dout, sizeof(double) * md, cudaMemcpyDeviceToHost, s));
    LK_CUDA(cudaStreamSynchronize(s));
    if (sing != ~0ull) {
        const int ix = int(sing % uint64_t(n)), iy = int(sing / uint64_t(n));
        if (st) {
            st->diverged_particle = ix;
            st->diverged_step = iy;
        }
        return fail(st, TURBDA_SINGULAR,
                    "singular local analysis at grid point (" + std::to_string(ix) + "," +
                        std::to_string(iy) + ")");
    }
    return TURBDA_OK;
}

int turbda_rtps_inflate(const double* analysis, const double* background, int32_t m, int64_t d,
                        double alpha, double* out, int32_t device, uint32_t flags, void* stream,
                        turbda_status* st) {
    clear(st);
    if (m < 1 || d < 0) return fail(st, TURBDA_DIMENSION, "rtps_inflate: shape mismatch");
    if (!(alpha >= 0.0 && alpha <= 1.0)) return fail(st, TURBDA_CONFIG, "letkf: rtps_alpha in [0, 1]");
    const bool on_dev = (flags & TURBDA_INPUTS_ON_DEVICE) != 0;
    const size_t md = size_t(m) * size_t(d);
    int dev = device;
    if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) return fail(st, TURBDA_CUDA, "no CUDA device");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || dev >= ndev)
        return fail(st, TURBDA_CUDA, "no such CUDA device");
    LK_CUDA(cudaSetDevice(dev));
    LetkfWorkspace* w = workspace(dev);
    std::lock_guard<std::mutex> lk(w->mu);
    if (!w->stream) LK_CUDA(cudaStreamCreateWithFlags(&w->stream, cudaStreamNonBlocking));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : (on_dev ? cudaStreamLegacy : w->stream);
    const double* bg = background;
    double* o = out;
    if (!on_dev) {
        LK_CUDA(w->x.reserve(sizeof(double) * std::max<size_t>(md, 1)));
        LK_CUDA(w->out.reserve(sizeof(double) * std::max<size_t>(md, 1)));
        LK_CUDA(cudaMemcpyAsync(w->x.p, background, sizeof(double) * md, cudaMemcpyHostToDevice, s));
        LK_CUDA(cudaMemcpyAsync(w->out.p, analysis, sizeof(double) * md, cudaMemcpyHostToDevice, s));
        bg = w->x.as<double>();
        o = w->out.as<double>();
    } else if (o != analysis) {
        LK_CUDA(cudaMemcpyAsync(o, analysis, sizeof(double) * md, cudaMemcpyDeviceToDevice, s));
    }
    if (alpha != 0.0 && m >= 2 && d > 0) {
        rtps_kernel<<<blocks_for(d, 256), 256, 0, s>>>(o, bg, m, d, alpha);
        LK_CUDA(cudaGetLastError());
        add_launches(1);
    }
    if (!on_dev) LK_CUDA(cudaMemcpyAsync(out, o, sizeof(double) * md, cudaMemcpyDeviceToHost, s));
    LK_CUDA(cudaStreamSynchronize(s));
    return TURBDA_OK;
}

}  // extern "C"
