// Joint-norm EnSF score (north_star extension; paper Eq. 15-16,
// /root/reference/PAPER.md:236-246) - the estimator the
// reference deliberately does NOT use (proj/src/ensf.cpp:27-32): one softmax
// per particle over the full-state squared distances
//     w_ij = softmax_j( -||z_i - alpha x_j||^2 / (2 beta^2) ),
//     s_i  = -(z_i - alpha sum_j w_ij x_j) / beta^2.
// Parity is UNPINNED (no reference implementation); the oracle is the C
// restatement oracle/ensf_oracle.c (orc_analyze_joint) with the weight line
// changed.
//
// Per pseudo-time step (the state dimension may be sharded over GPUs):
//   gram_partial   per coordinate chunk, the N x J Gram Z X^T and the norms
//                  ||z_i||^2, ||x_j||^2 (fp64, register-tiled DFMA GEMM)
//   reduce_chunks  fixed-order sum over chunks -> [G | nz | nx] (fp64)
//   (multi-GPU)    ONE ncclAllReduce(sum) of that N J + N + J buffer
//   joint_softmax  D_ij = nz_i + alpha^2 nx_j - 2 alpha G_ij, shifted by the
//                  row minimum, fast_exp_nonpos weights, normalised
//   joint_apply    xbar = W X (per coordinate), damped likelihood, Euler-
//                  Maruyama update with the particle noise, in place
// Every step streams Z and X through HBM (40 N d bytes at N = J): this mode
// is HBM / FP64-bound, not SFU-bound.
#include <cfloat>
#include <climits>
#include <cstdint>

#include "ensf_device.h"
#include "philox.cuh"

namespace tb200 {

namespace {

constexpr int kT = 64;   // output tile (particles x members) of the Gram
constexpr int kK = 16;   // coordinates per shared-memory stage

__device__ __forceinline__ double fast_exp_nonpos_j(double x) {
    constexpr double kInvLn2 = 1.4426950408889634074;
    constexpr double kLn2Hi = 6.93147180369123816490e-01;
    constexpr double kLn2Lo = 1.90821492927058770002e-10;
    constexpr double kMagic = 6755399441055744.0;
    const bool under = x < -708.0;
    if (under) x = 0.0;
    const double t = x * kInvLn2 + kMagic;
    const double nf = t - kMagic;
    const int32_t n = int32_t(uint32_t(__double_as_longlong(t)));
    double r = x - nf * kLn2Hi;
    r -= nf * kLn2Lo;
    double p = 1.0 / 479001600.0;
    p = p * r + 1.0 / 39916800.0;
    p = p * r + 1.0 / 3628800.0;
    p = p * r + 1.0 / 362880.0;
    p = p * r + 1.0 / 40320.0;
    p = p * r + 1.0 / 5040.0;
    p = p * r + 1.0 / 720.0;
    p = p * r + 1.0 / 120.0;
    p = p * r + 1.0 / 24.0;
    p = p * r + 1.0 / 6.0;
    p = p * r + 0.5;
    p = p * r + 1.0;
    p = p * r + 1.0;
    const long long pb = __double_as_longlong(p) + (static_cast<long long>(n) << 52);
    return under ? 0.0 : __longlong_as_double(pb);
}

// Z [n][dl] fp64 <- N(0, I) from the particle streams (normal #k, global k)
__global__ void joint_init_kernel(KernelArgs a, double* __restrict__ z) {
    const int64_t kl = 2 * (int64_t(blockIdx.x) * blockDim.x + threadIdx.x);
    const int i = blockIdx.y;
    if (kl >= a.dl) return;
    const double2 v = normal_pair_f64(uint64_t(a.k0 + kl), uint32_t(i), a.cycle_lo, a.key0, a.key1);
    double* row = z + size_t(i) * size_t(a.dl);
    row[kl] = v.x;
    if (kl + 1 < a.dl) row[kl + 1] = v.y;
}

// Partial Gram over coordinate chunk blockIdx.x for output tile blockIdx.y.
// 256 threads, 4 x 4 accumulators each; Z and X stages transposed in shared
// memory with a one-double pad (conflict-free column reads).
__global__ void __launch_bounds__(256) gram_partial_kernel(const double* __restrict__ z,
                                                           const double* __restrict__ x, int n,
                                                           int m, int64_t dl, int64_t chunk,
                                                           double* __restrict__ part) {
    __shared__ double zs[kK][kT + 1];
    __shared__ double xs[kK][kT + 1];
    const int ntj = (m + kT - 1) / kT;
    const int ti0 = (blockIdx.y / ntj) * kT, tj0 = (blockIdx.y % ntj) * kT;
    const int64_t c0 = int64_t(blockIdx.x) * chunk;
    const int64_t c1 = c0 + chunk < dl ? c0 + chunk : dl;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    double acc[4][4] = {};
    double nzv[4] = {}, nxv[4] = {};
    const bool do_nz = tj0 == 0 && tx == 0, do_nx = ti0 == 0 && ty == 0;

    for (int64_t kb = c0; kb < c1; kb += kK) {
        // stage kK coordinates of 64 particle rows and 64 member rows
        for (int q = threadIdx.x; q < kK * kT; q += 256) {
            const int r = q / kK, c = q % kK;
            const int64_t k = kb + c;
            const int iz = ti0 + r, jx = tj0 + r;
            zs[c][r] = (k < c1 && iz < n) ? z[size_t(iz) * size_t(dl) + size_t(k)] : 0.0;
            xs[c][r] = (k < c1 && jx < m) ? x[size_t(jx) * size_t(dl) + size_t(k)] : 0.0;
        }
        __syncthreads();
#pragma unroll 4
        for (int c = 0; c < kK; ++c) {
            double zi[4], xj[4];  // rows ty + 16u, columns tx + 16v: conflict-free
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                zi[u] = zs[c][ty + 16 * u];
                xj[u] = xs[c][tx + 16 * u];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = fma(zi[u], xj[v], acc[u][v]);
            if (do_nz)
#pragma unroll
                for (int u = 0; u < 4; ++u) nzv[u] = fma(zi[u], zi[u], nzv[u]);
            if (do_nx)
#pragma unroll
                for (int v = 0; v < 4; ++v) nxv[v] = fma(xj[v], xj[v], nxv[v]);
        }
        __syncthreads();
    }
    // part[chunk] = [G (n x m) | nz (n) | nx (m)]
    double* out = part + size_t(blockIdx.x) * (size_t(n) * m + n + m);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int i = ti0 + ty + 16 * u;
        if (i >= n) continue;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int j = tj0 + tx + 16 * v;
            if (j < m) out[size_t(i) * m + j] = acc[u][v];
        }
        if (do_nz) out[size_t(n) * m + i] = nzv[u];
    }
    if (do_nx)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int j = tj0 + tx + 16 * v;
            if (j < m) out[size_t(n) * m + n + j] = nxv[v];
        }
}

// red[q] = sum over chunks of part[chunk][q], in chunk order (deterministic)
__global__ void reduce_chunks_kernel(const double* __restrict__ part, int nchunk, size_t len,
                                     double* __restrict__ red) {
    const size_t q = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= len) return;
    double s = 0.0;
    for (int c = 0; c < nchunk; ++c) s += part[size_t(c) * len + q];
    red[q] = s;
}

// one warp per particle: D_ij, the row-minimum shift and normalised weights
__global__ void joint_softmax_kernel(const double* __restrict__ red, int n, int m, double alpha,
                                     double inv2b, double* __restrict__ wn) {
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    const double* g = red + size_t(i) * m;
    const double nz = red[size_t(n) * m + i];
    const double* nx = red + size_t(n) * m + n;
    double mn = __longlong_as_double(0x7ff0000000000000ll);
    for (int j = lane; j < m; j += 32) {
        const double dd = nz + alpha * alpha * nx[j] - 2.0 * alpha * g[j];
        mn = dd < mn ? dd : mn;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double t = __shfl_xor_sync(0xffffffffu, mn, o);
        mn = t < mn ? t : mn;
    }
    double den = 0.0;
    for (int j = lane; j < m; j += 32) {
        const double dd = nz + alpha * alpha * nx[j] - 2.0 * alpha * g[j];
        const double w = fast_exp_nonpos_j((mn - dd) * inv2b);
        wn[size_t(i) * m + j] = w;
        den += w;
    }
    for (int o = 16; o > 0; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
    const double inv = 1.0 / den;
    for (int j = lane; j < m; j += 32) wn[size_t(i) * m + j] *= inv;
}

// xbar_ik = sum_j w_ij x_jk; posterior score; Euler-Maruyama in place.
// CTA = 64 coordinates (lane = coordinate pair) x kJW warps x kJP particles
// per warp; member rows are staged through shared memory 64 at a time, so a
// loaded x pair feeds kJP particles.  kF32Noise: the particle normals come
// from the fp32 Box-Muller of the fast path (the update stays fp64).
constexpr int kJP = 8, kJW = 4, kJM = 64;

template <bool kF32Noise>
__global__ void __launch_bounds__(kJW * 32) joint_apply_kernel(
    KernelArgs a, const double* __restrict__ x, const double2* __restrict__ ab,
    const double* __restrict__ wn, StepF64 c, int step, double* __restrict__ z,
    unsigned long long* __restrict__ status) {
    __shared__ double2 xs[kJM][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t kl = int64_t(blockIdx.x) * 64 + 2 * lane;
    const int i0 = (blockIdx.y * kJW + warp) * kJP;
    const bool has_x = kl < a.dl, has_y = kl + 1 < a.dl;
    const bool aligned = (a.dl & 1) == 0;
    double sx[kJP], sy[kJP];
#pragma unroll
    for (int p = 0; p < kJP; ++p) sx[p] = sy[p] = 0.0;
    for (int j0 = 0; j0 < a.m; j0 += kJM) {
        const int jn = a.m - j0 < kJM ? a.m - j0 : kJM;
        __syncthreads();
        for (int q = threadIdx.x; q < jn * 32; q += kJW * 32) {
            const int jj = q >> 5, l = q & 31;
            const int64_t k = int64_t(blockIdx.x) * 64 + 2 * l;
            const double* row = x + size_t(j0 + jj) * size_t(a.dl);
            double2 v = make_double2(0.0, 0.0);
            if (k + 1 < a.dl)
                v = aligned ? __ldg(reinterpret_cast<const double2*>(row + k))
                            : make_double2(__ldg(row + k), __ldg(row + k + 1));
            else if (k < a.dl)
                v.x = __ldg(row + k);
            xs[jj][l] = v;
        }
        __syncthreads();
        for (int jj = 0; jj < jn; ++jj) {
            const double2 xv = xs[jj][lane];
#pragma unroll
            for (int p = 0; p < kJP; ++p) {
                const int i = i0 + p < a.m ? i0 + p : a.m - 1;
                const double w = __ldg(wn + size_t(i) * a.m + j0 + jj);  // warp-uniform
                sx[p] = fma(w, xv.x, sx[p]);
                sy[p] = fma(w, xv.y, sy[p]);
            }
        }
    }
    if (!has_x) return;
    const double2 o0 = ab[kl];
    const double2 o1 = has_y ? ab[kl + 1] : make_double2(0.0, 0.0);
    const uint64_t n0 = uint64_t(step + 1) * uint64_t(a.d_total) + uint64_t(a.k0 + kl);
#pragma unroll
    for (int p = 0; p < kJP; ++p) {
        const int i = i0 + p;
        if (i >= a.m) break;
        double* zr = z + size_t(i) * size_t(a.dl) + kl;
        double zx = zr[0], zy = has_y ? zr[1] : 0.0;
        double scx = -(zx - c.alpha * sx[p]) / c.beta2;
        double scy = -(zy - c.alpha * sy[p]) / c.beta2;
        if (a.obs_atan) {
            scx += c.damp * ((o0.y - o0.x * atan(zx)) / (1.0 + zx * zx));
            scy += c.damp * ((o1.y - o1.x * atan(zy)) / (1.0 + zy * zy));
        } else {
            scx += c.damp * (o0.y - o0.x * zx);
            scy += c.damp * (o1.y - o1.x * zy);
        }
        double2 xi;
        if (kF32Noise) {
            const float2 f = normal_pair_f32(n0, uint32_t(i), a.cycle_lo, a.key0, a.key1);
            xi = make_double2(f.x, f.y);
        } else {
            xi = normal_pair_f64(n0, uint32_t(i), a.cycle_lo, a.key0, a.key1);
        }
        zx += -(c.b * zx - c.s2 * scx) * c.dt + c.sig * xi.x;
        zy += -(c.b * zy - c.s2 * scy) * c.dt + c.sig * xi.y;
        zr[0] = zx;
        if (has_y) zr[1] = zy;
        if (!isfinite(zx) || (has_y && !isfinite(zy)))
            atomicMin(status, (uint64_t(i) << 32) | uint32_t(step));
    }
}

}  // namespace

JointPlan joint_plan(int n, int m, int64_t dl) {
    JointPlan pl;
    const int tiles = ((n + kT - 1) / kT) * ((m + kT - 1) / kT);
    pl.nchunk = (296 + tiles - 1) / tiles;  // ~2 CTAs per SM in total
    const int64_t want = (dl + pl.nchunk - 1) / pl.nchunk;
    pl.chunk = (want + kK - 1) / kK * kK;
    if (pl.chunk < kK) pl.chunk = kK;
    pl.nchunk = int((dl + pl.chunk - 1) / pl.chunk);
    if (pl.nchunk < 1) pl.nchunk = 1;
    pl.tiles = tiles;
    pl.red_len = size_t(n) * m + n + m;
    return pl;
}

cudaError_t launch_joint_init(const KernelArgs& a, double* z, cudaStream_t st) {
    if (a.dl <= 0) return cudaSuccess;
    const dim3 grid(unsigned((a.dl / 2 + 127) / 128 + 1), unsigned(a.m));
    joint_init_kernel<<<grid, 128, 0, st>>>(a, z);
    return cudaGetLastError();
}

cudaError_t launch_joint_gram(const KernelArgs& a, const JointPlan& pl, const double* z,
                              const double* x, double* part, double* red, cudaStream_t st) {
    if (a.dl > 0) {
        gram_partial_kernel<<<dim3(unsigned(pl.nchunk), unsigned(pl.tiles)), 256, 0, st>>>(
            z, x, a.m, a.m, a.dl, pl.chunk, part);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        reduce_chunks_kernel<<<unsigned((pl.red_len + 255) / 256), 256, 0, st>>>(part, pl.nchunk,
                                                                              pl.red_len, red);
    } else {
        cudaMemsetAsync(red, 0, sizeof(double) * pl.red_len, st);
    }
    return cudaGetLastError();
}

cudaError_t launch_joint_update(const KernelArgs& a, const double* x, const double2* ab,
                                const double* red, double* wn, const StepF64& c, int step,
                                double* z, unsigned long long* status, bool f32_noise,
                                cudaStream_t st) {
    joint_softmax_kernel<<<unsigned((a.m + 3) / 4), 128, 0, st>>>(red, a.m, a.m, c.alpha, c.inv2b,
                                                                  wn);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || a.dl <= 0) return e;
    const dim3 grid(unsigned((a.dl + 63) / 64), unsigned((a.m + kJP * kJW - 1) / (kJP * kJW)));
    if (f32_noise)
        joint_apply_kernel<true><<<grid, kJW * 32, 0, st>>>(a, x, ab, wn, c, step, z, status);
    else
        joint_apply_kernel<false><<<grid, kJW * 32, 0, st>>>(a, x, ab, wn, c, step, z, status);
    return cudaGetLastError();
}

}  // namespace tb200
