// sm_100a kernels for the EnSF analysis step (turbda::analyze,
// proj/src/ensf.cpp:132-223) and its epilogue relax_spread (:225-258).
//
// Layout and mapping:
//   * forecast X lives in HBM as the reference's [M][d] member-major fp64
//     array.  A CTA owns a tile of 64 consecutive coordinates; lane l owns the
//     coordinate pair (2l, 2l+1) of the tile, so every global access is a
//     coalesced 16 B (fp64) per lane and both Box-Muller outputs of a Philox
//     block land in the same thread.
//   * each warp owns P particles of the tile; the whole reverse SDE (all
//     n_steps pseudo-time steps) runs in registers: there is no per-step
//     HBM traffic at all.  The prior score is componentwise
//     (proj/src/ensf.cpp:27-64), so coordinates never talk to each other.
//   * fp32 fast kernel: the tile's members are converted once into shared
//     memory as float2 rows (lane-contiguous, conflict-free LDS.64); the
//     pair arithmetic is packed FFMA2/FMUL2/FADD2 on the coordinate pair and
//     the weights use MUFU.EX2 with a log2(e)-prescaled exponent.
//   * fp64 faithful kernel: same mapping, the reference's own arithmetic
//     (fast_exp_nonpos, num/den form, update order).
#include <cfloat>
#include <climits>
#include <cstdint>
#include <cstdlib>

#include "ensf_device.h"
#include "bulk_copy.cuh"
#include "philox.cuh"
#include "reduce.cuh"

#include <cub/device/device_radix_sort.cuh>

namespace tb200 {

namespace {

constexpr int kTile = 64;  // coordinates per CTA tile (32 lanes x 2)

__device__ __forceinline__ float ex2f(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

// num / den per coordinate.  kNewton (default): 1 / den on the FMA pipe -
// the 0x7EF311C3 seed (rel. error < 1/8) and three Newton steps
// r <- r (2 - den r) (rel. error < 1e-7), packed over the pair (config 3:
// 192.0 ms vs 195.1 ms with MUFU.RCP, profiles/r02_sweeps.md); otherwise
// MUFU.RCP (__fdividef).  den lies in [2^-60, J] (the redo guarantees the
// lower bound); a non-finite den only occurs in a diverged run.
template <bool kNewton>
__device__ __forceinline__ float2 recip_mul(float2 num, float2 den) {
    if (!kNewton) return make_float2(__fdividef(num.x, den.x), __fdividef(num.y, den.y));
    float2 r = make_float2(__uint_as_float(0x7EF311C3u - __float_as_uint(den.x)),
                           __uint_as_float(0x7EF311C3u - __float_as_uint(den.y)));
    const float2 nd = make_float2(-den.x, -den.y);
#pragma unroll
    for (int it = 0; it < 3; ++it) r = __fmul2_rn(r, __ffma2_rn(nd, r, f2(2.f)));
    return __fmul2_rn(num, r);
}

// one pseudo-step's coefficients: a warp-uniform 32 B read (L1 broadcast)
__device__ __forceinline__ StepF32 load_step(const StepF32* p) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p));
    const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
    return StepF32{a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
}

// proj/include/turbda/fastexp.hpp:13-50, restated for the device.
__device__ __forceinline__ double fast_exp_nonpos_dev(double x) {
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

// Loads X[j][k], X[j][k+1] (k local, even) with zero padding past dl.
__device__ __forceinline__ double2 load_pair(const double* __restrict__ row, int64_t k,
                                             int64_t dl, bool aligned) {
    if (k + 1 < dl) {
        if (aligned) return __ldg(reinterpret_cast<const double2*>(row + k));
        return make_double2(__ldg(row + k), __ldg(row + k + 1));
    }
    if (k < dl) return make_double2(__ldg(row + k), 0.0);
    return make_double2(0.0, 0.0);
}

// ---------------------------------------------------------------------------
// fp32 fast kernel
// ---------------------------------------------------------------------------

// 2^e (e <= ~0) on the FMA pipe, to offload part of the softmax from MUFU
// (FA4-style split): e is rounded to j by the 1.5*2^23 shifter, 2^(e-j) comes
// from a degree-5 minimax polynomial on [-1/2, 1/2] (max rel. error 2.2e-7,
// the accuracy class of MUFU.EX2) and j is added into the exponent field.
// e is clamped at -125 so the exponent never underflows (such weights are
// < 2^-125 of the largest one and vanish from every sum anyway).
__device__ __forceinline__ float2 ex2_poly2(float2 e) {
    e.x = fmaxf(e.x, -125.f);
    e.y = fmaxf(e.y, -125.f);
    const float2 t = __fadd2_rn(e, f2(12582912.f));                // 1.5 * 2^23 + j
    const float2 f = __fadd2_rn(e, __fadd2_rn(f2(12582912.f), make_float2(-t.x, -t.y)));
    float2 p = __ffma2_rn(f2(0.001330954604782164f), f, f2(0.009673058986663818f));
    p = __ffma2_rn(p, f, f2(0.055505912750959396f));
    p = __ffma2_rn(p, f, f2(0.24022164940834045f));
    p = __ffma2_rn(p, f, f2(0.6931470632553101f));
    p = __ffma2_rn(p, f, f2(1.0000001192092896f));
    return make_float2(__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23)),
                       __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23)));
}

// Smallest |u_j| = |fma(-alpha s, x_j, s z)| over sorted member columns:
// u_j falls with x_j (alpha > 0), so the nearest member sits where u changes
// sign.  All 2P searches of a thread (P particles x the coordinate pair)
// advance together, so each probe round issues 2P independent LDS and the
// shared-memory latency overlaps; ceil(log2 J) rounds replace a pass
// over all J members.
template <int P>
__device__ __forceinline__ void nearest_abs_u(const float* __restrict__ xsf, int lane, int j_n,
                                              int top, float nas, const float2 (&zs)[P],
                                              float2 (&mn)[P]) {
    int pos[P][2];
#pragma unroll
    for (int p = 0; p < P; ++p) pos[p][0] = pos[p][1] = 0;  // members with u > 0
    for (int st = top; st > 0; st >>= 1) {
#pragma unroll
        for (int p = 0; p < P; ++p) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int cand = pos[p][h] + st;
                const float xv = xsf[(min(cand, j_n) - 1) * 64 + 2 * lane + h];
                const float zc = h ? zs[p].y : zs[p].x;
                if (cand <= j_n && fmaf(nas, xv, zc) > 0.f) pos[p][h] = cand;
            }
        }
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
        float r[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int q = pos[p][h];
            const float zc = h ? zs[p].y : zs[p].x;
            const float lo = fabsf(fmaf(nas, xsf[max(q - 1, 0) * 64 + 2 * lane + h], zc));
            const float hi = fabsf(fmaf(nas, xsf[min(q, j_n - 1) * 64 + 2 * lane + h], zc));
            r[h] = fminf(q > 0 ? lo : FLT_MAX, q < j_n ? hi : FLT_MAX);
        }
        mn[p] = make_float2(r[0], r[1]);
    }
}

// NaN sorts last so every column stays a permutation of its members.
__device__ __forceinline__ float sort_key(float v) { return v != v ? __int_as_float(0x7f800000) : v; }

constexpr int kSortWarps = 8;  // warps that sort the fused tile's columns

// Fused prologue: the tile's forecast [m][64] (fp64, coalesced 512 B member
// rows) -> fp32 in shared memory, zero padded past dl; for kSorted every
// column sorted ascending (NaN last, ties by member index: the rank of
// (j, c) counts the members that order before it, so the column stays a
// permutation) by up to kSortWarps warps, one column at a time through a
// per-warp staging column.  The forecast statistics of relax_spread
// (ensemble_mean, proj/src/ensemble.cpp:7-16, then the sum of squared
// deviations, proj/src/ensf.cpp:225-258) in fp64 and member order, exactly
// as relax_kernel takes them.
template <bool kSorted>
__device__ __forceinline__ void fused_prologue(const KernelArgs& a, float* tile, int64_t tile0,
                                               double2* fstat) {
    const int m = a.m;
    // pairs of coordinates (16 B loads when the rows are 16-byte aligned),
    // unrolled so each thread keeps several loads in flight
    const bool vec = ((a.dl & 1) == 0) && ((reinterpret_cast<uintptr_t>(a.x64) & 15) == 0);
#pragma unroll 4
    for (int q = threadIdx.x; q < m * (kTile / 2); q += blockDim.x) {
        const int j = q >> 5, c = 2 * (q & 31);
        const int64_t k = tile0 + c;
        const double* src = a.x64 + size_t(j) * size_t(a.dl) + size_t(k);
        double2 v = make_double2(0.0, 0.0);
        if (k + 1 < a.dl) {
            v = vec ? __ldg(reinterpret_cast<const double2*>(src)) : make_double2(__ldg(src), __ldg(src + 1));
        } else if (k < a.dl) {
            v.x = __ldg(src);
        }
        TB_CHECK(sizeof(float) * size_t(j * kTile + c + 2) <= dyn_smem_bytes());
        *reinterpret_cast<float2*>(tile + j * kTile + c) = make_float2(float(v.x), float(v.y));
    }
    if (threadIdx.x < kTile) {
        const int64_t k = tile0 + threadIdx.x;
        double mb = 0.0, sb = 0.0;
        if (k < a.dl && a.relax != 0.0 && m >= 2) {
            // member-order sums; the loads are batched 8 ahead of the adds
            const double* col = a.x64 + size_t(k);
            const size_t ld = size_t(a.dl);
#pragma unroll 8
            for (int j = 0; j < m; ++j) mb += __ldg(col + size_t(j) * ld);
            mb *= 1.0 / m;
            double vb = 0.0;
#pragma unroll 8
            for (int j = 0; j < m; ++j) {
                const double db = __ldg(col + size_t(j) * ld) - mb;
                vb += db * db;
            }
            sb = sqrt(vb / (m - 1));
        }
        fstat[threadIdx.x] = make_double2(mb, sb);
    }
    __syncthreads();
    if (!kSorted) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sorters = min(int(blockDim.x >> 5), kSortWarps);
    float* stage = tile + size_t(m) * kTile + size_t(warp) * size_t(m);  // [m] per warp
    if (warp < sorters) {
        for (int c = warp; c < kTile; c += sorters) {
            TB_CHECK(sizeof(float) * (size_t(m) * kTile + size_t(warp + 1) * size_t(m)) <=
                     dyn_smem_bytes());
            for (int j = lane; j < m; j += 32) stage[j] = tile[j * kTile + c];
            __syncwarp();
            for (int j = lane; j < m; j += 32) {
                const float v = stage[j];
                const float kv = sort_key(v);
                int rank = 0;
                for (int i = 0; i < m; ++i) {
                    const float ki = sort_key(stage[i]);
                    rank += (ki < kv) || (ki == kv && i < j);
                }
                TB_CHECK(rank < m);
                tile[rank * kTile + c] = v;
            }
            __syncwarp();
        }
    }
    __syncthreads();
}

// Fused epilogue: relax_spread of the tile (proj/src/ensf.cpp:225-258).
// One CTA per tile (grid.y == 1): the particles go to shared memory (the
// member tile is dead by now).  Several CTAs per tile: each writes its
// particles to the fp32 scratch `zg` ([m][dl]) and takes a ticket; the last
// CTA of the tile to finish relaxes the whole tile from there (L2-resident)
// - no co-scheduling constraint, unlike a thread-block cluster, which
// measured 6 % slower at N = 128 (profiles/r02_sweeps.md).  Either way one
// thread per coordinate sums every particle in member order, so ma / va are
// the reference's sequential fp64 sums (bit-identical to relax_kernel), and
// the fp64 analysis is written once.  relax_factor 0 or one member: the
// analysis is the particles themselves.
template <int P>
__device__ __forceinline__ void fused_relax_epilogue(const KernelArgs& a, float* zs, float* zg,
                                                     int64_t tile0, int64_t kl, int i0,
                                                     const double2* fstat, const float2 (&z)[P]) {
    __shared__ double2 rstat[kTile];  // (ma, scale)
    __shared__ unsigned int ticket;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool relax = a.relax != 0.0 && a.m >= 2;
    const bool shared_path = gridDim.y == 1;
    const bool aligned = (a.dl & 1) == 0;
    __syncthreads();  // every warp is done with the member tile
    if (shared_path) {
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const int il = warp * P + p;
            TB_CHECK(sizeof(float) * size_t(il * kTile + 2 * lane + 2) <= dyn_smem_bytes());
            zs[il * kTile + 2 * lane] = z[p].x;
            zs[il * kTile + 2 * lane + 1] = z[p].y;
        }
    } else {
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const int i = i0 + p;
            if (i >= a.m) continue;
            float* row = zg + size_t(i) * size_t(a.dl);
            if (kl + 1 < a.dl) {
                if (aligned) {
                    *reinterpret_cast<float2*>(row + kl) = z[p];
                } else {
                    row[kl] = z[p].x;
                    row[kl + 1] = z[p].y;
                }
            } else if (kl < a.dl) {
                row[kl] = z[p].x;
            }
        }
        __threadfence();
        __syncthreads();
        TB_CHECK(a.tile_ticket != nullptr);
        if (threadIdx.x == 0) ticket = atomicAdd(a.tile_ticket + blockIdx.x, 1u);
        __syncthreads();
        TB_CHECK(ticket < gridDim.y);
        if (ticket != gridDim.y - 1) return;  // not the last CTA of this tile
        __threadfence();
        if (threadIdx.x == 0) a.tile_ticket[blockIdx.x] = 0u;  // ready for the next launch
    }
    __syncthreads();
    if (threadIdx.x < kTile) {
        const int c = threadIdx.x;
        const int64_t k = tile0 + c;
        double ma = 0.0, scale = 1.0;
        if (relax && (shared_path || k < a.dl)) {
            const float* col = shared_path ? zs + c : zg + size_t(k);
            const size_t ld = shared_path ? size_t(kTile) : size_t(a.dl);
#pragma unroll 8
            for (int j = 0; j < a.m; ++j) ma += double(col[size_t(j) * ld]);
            ma *= 1.0 / a.m;
            double va = 0.0;
#pragma unroll 8
            for (int j = 0; j < a.m; ++j) {
                const double da = double(col[size_t(j) * ld]) - ma;
                va += da * da;
            }
            const double sa = fmax(sqrt(va / (a.m - 1)), 1e-12);
            scale = (1.0 - a.relax) + a.relax * fstat[c].y / sa;
        }
        rstat[c] = make_double2(ma, scale);
    }
    __syncthreads();
    if (shared_path) {
        const double2 s0 = rstat[2 * lane], s1 = rstat[2 * lane + 1];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const int i = i0 + p;
            if (i >= a.m) continue;
            double* row = a.out64 + size_t(i) * size_t(a.dl);
            const double vx = relax ? s0.x + s0.y * (double(z[p].x) - s0.x) : double(z[p].x);
            const double vy = relax ? s1.x + s1.y * (double(z[p].y) - s1.x) : double(z[p].y);
            if (kl + 1 < a.dl) {
                if (aligned)
                    *reinterpret_cast<double2*>(row + kl) = make_double2(vx, vy);
                else {
                    row[kl] = vx;
                    row[kl + 1] = vy;
                }
            } else if (kl < a.dl) {
                row[kl] = vx;
            }
        }
        return;
    }
    // the last CTA writes the whole tile: member rows of 64 coordinates
    for (int q = threadIdx.x; q < a.m * kTile; q += blockDim.x) {
        const int j = q >> 6, c = q & (kTile - 1);
        const int64_t k = tile0 + c;
        if (k >= a.dl) continue;
        const double v = double(zg[size_t(j) * size_t(a.dl) + size_t(k)]);
        const double2 r = rstat[c];
        a.out64[size_t(j) * size_t(a.dl) + size_t(k)] = relax ? r.x + r.y * (v - r.x) : v;
    }
}

// kSorted: members of every coordinate are sorted once per analysis (the
// componentwise score only needs the multiset of member values per
// coordinate, proj/src/ensf.cpp:43-61), pass 1 becomes a binary search.
// kPolyEvery: every kPolyEvery-th (member, particle) slot of the unrolled
// member loop takes its two exponentials from ex2_poly2 instead of MUFU (the
// slot pattern depends on P: sorted tiles therefore always run P = 4).
// kFused: the whole analysis in one launch.  The prologue converts (and for
// kSorted rank-sorts) the tile's fp64 forecast columns straight into shared
// memory and takes the forecast statistics of relax_spread; the epilogue
// runs relax_spread (proj/src/ensf.cpp:225-258) on the tile (in shared
// memory, or - several CTAs per tile - by the tile's last CTA), so every
// coordinate's statistics are the reference's member-order fp64 sums
// (bit-identical to relax_kernel), and the fp64 analysis is written once.  No
// prep_tiles / relax launches.
template <int P, bool kMinibatch, bool kSorted, int kPolyEvery, int kMinBlocks = 1,
          bool kGlobalX = false, int kThreads = 256, bool kShiftFree = true, bool kFused = false,
          bool kNewtonRcp = true, int kJ = 0>
__global__ void __launch_bounds__(kThreads, kMinBlocks) ensf_f32_kernel(KernelArgs a, const float* __restrict__ xt,
                                                       const double2* __restrict__ ab,
                                                       const StepF32* __restrict__ steps,
                                                       const int32_t* __restrict__ batches,
                                                       float* __restrict__ z_out,
                                                       unsigned long long* __restrict__ status) {
    static_assert(!(kMinibatch && kSorted), "minibatches use the two-pass member loop");
    static_assert(!(kGlobalX && kSorted), "very large ensembles use the two-pass member loop");
    static_assert(!(kFused && (kGlobalX || kMinibatch)), "fused: shared-memory tiles, no minibatch");
    static_assert(kJ == 0 || !(kMinibatch || kSorted || kGlobalX), "compile-time J: unsorted tiles");
    constexpr int U = 4;  // member-loop unroll
    extern __shared__ float4 smem[];
    // the tile's members: shared memory, or (ensembles too large for it)
    // read straight from the fp32 tile in global memory through L1/L2
    const float2* xs = kGlobalX ? reinterpret_cast<const float2*>(
                                      xt + size_t(blockIdx.x) * size_t(a.m) * kTile)
                                : reinterpret_cast<const float2*>(smem);
    const float* xsf = reinterpret_cast<const float*>(xs);

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    const int64_t tile0 = int64_t(blockIdx.x) * kTile;
    const int64_t kl = tile0 + 2 * lane;  // local coordinate of this lane's pair
    const bool aligned = ((a.dl & 1) == 0);

    // the tile's members (fp32 [m][64], sorted per column when kSorted,
    // contiguous by prep_tiles_kernel) arrive by one TMA bulk copy issued by
    // one thread while the others set up their pairs.  The per-step
    // coefficients are read from global memory (warp-uniform, L1-resident),
    // so any n_steps fits.
    __shared__ uint64_t tile_bar;
    __shared__ double2 fstat[kTile];  // kFused: forecast (mean, sd) per coordinate
    if (kFused) {
        fused_prologue<kSorted>(a, reinterpret_cast<float*>(smem), tile0, fstat);
    } else if (!kGlobalX) {
        if (threadIdx.x == 0) mbar_init(&tile_bar, 1);
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t tile_bytes = uint32_t(sizeof(float)) * uint32_t(a.m) * kTile;
            mbar_arrive_expect_tx(&tile_bar, tile_bytes);
            bulk_copy_g2s(smem, xt + size_t(blockIdx.x) * size_t(a.m) * kTile, tile_bytes,
                          &tile_bar);
        }
    }
    // likelihood operator for this pair: B - A z with A = sum 1/r, B = sum y/r.
    // Fused launches are programmatic dependents of the observation prep
    // (the prologue above reads only the caller's forecast): wait for it
    // here.  A no-op for ordinary launches.
    if (kFused) asm volatile("griddepcontrol.wait;" ::: "memory");
    float2 A2 = f2(0.f), B2 = f2(0.f);
    if (kl < a.dl) {
        const double2 o = ab[kl];
        A2.x = float(o.x);
        B2.x = float(o.y);
    }
    if (kl + 1 < a.dl) {
        const double2 o = ab[kl + 1];
        A2.y = float(o.x);
        B2.y = float(o.y);
    }
    const float2 nA2 = make_float2(-A2.x, -A2.y);
    const bool has_y = kl + 1 < a.dl;  // the pair's second coordinate is real
    int top = 1;
    // probes top, top/2, .., 1 reach pos <= 2 top - 1 >= J - 1; pos = J - 1
    // when all J members have u > 0 still yields the right pair (J-2, J-1)
    while (top * 2 < a.j_batch) top *= 2;
    if (!kGlobalX && !kFused) mbar_wait(&tile_bar, 0);  // the member tile has landed

    const int i0 = (blockIdx.y * nwarps + warp) * P;
    const uint64_t kg = uint64_t(a.k0 + kl);  // global coordinate of the pair's first entry

    float2 z[P];
    // first non-finite (particle, step) of this thread: min over (p << 30 | s)
    // is the lowest particle and its first bad step (one register, not P)
    uint32_t bad = UINT_MAX;
#pragma unroll
    for (int p = 0; p < P; ++p) z[p] = normal_pair_f32(kg, uint32_t(i0 + p), a.cycle_lo, a.rk);

    for (int s = 0; s < a.n_steps; ++s) {
        const StepF32 c = load_step(steps + s);
        const float2 nas2 = f2(c.nas);
        const int32_t* bt = kMinibatch ? batches + size_t(s) * size_t(a.j_batch) : nullptr;
        const uint64_t n0 = uint64_t(s + 1) * uint64_t(a.d_total) + kg;
        // compile-time J: the step's noise is drawn first, in the same basic
        // block as the fully unrolled member loop, so ptxas interleaves the
        // Philox / Box-Muller chain with the exponentials (n0 even: the host
        // picks these kernels only for even d_total and k0)
        float2 xi_early[kJ > 0 ? P : 1];
        if constexpr (kJ > 0) {
#pragma unroll
            for (int p = 0; p < P; ++p)
                xi_early[p] = box_muller_f32(philox_block_rk(n0 >> 1, uint32_t(i0 + p), a.cycle_lo, a.rk));
        }

        // u_j = s (z - alpha x_j): one FFMA2 per member and coordinate pair
        float2 zs[P];
#pragma unroll
        for (int p = 0; p < P; ++p) zs[p] = __fmul2_rn(z[p], f2(c.s));

        // pass 2: w = 2^(c - u^2); den = sum w; num = sum w u,
        // proj/src/ensf.cpp:51-61 in the cancellation-free form of :62-63
        // (any shift c cancels in num / den)
        auto weight_pass = [&](const float2 (&m2)[P], float2 (&den)[P], float2 (&num)[P]) {
#pragma unroll
            for (int p = 0; p < P; ++p) {
                den[p] = f2(0.f);
                num[p] = f2(0.f);
            }
            if constexpr (kJ > 0) {
#pragma unroll
                for (int j = 0; j < kJ; ++j) {
                    const float2 xv = xs[j * 32 + lane];
#pragma unroll
                    for (int p = 0; p < P; ++p) {
                        const float2 u = __ffma2_rn(nas2, xv, zs[p]);
                        const float2 e = __ffma2_rn(make_float2(-u.x, -u.y), u, m2[p]);
                        const float2 w = make_float2(ex2f(e.x), ex2f(e.y));
                        den[p] = __fadd2_rn(den[p], w);
                        num[p] = __ffma2_rn(w, u, num[p]);
                    }
                }
                return;
            }
            int jj = 0;
            for (; jj + U <= a.j_batch; jj += U) {
#pragma unroll
                for (int uu = 0; uu < U; ++uu) {
                    const int j = kMinibatch ? __ldg(bt + jj + uu) : jj + uu;
                    TB_CHECK(j >= 0 && j < a.m);
                    TB_CHECK(kGlobalX || sizeof(float2) * size_t(j * 32 + lane + 1) <= dyn_smem_bytes());
                    const float2 xv = kGlobalX ? __ldg(xs + j * 32 + lane) : xs[j * 32 + lane];
#pragma unroll
                    for (int p = 0; p < P; ++p) {
                        const float2 u = __ffma2_rn(nas2, xv, zs[p]);
                        const float2 e = __ffma2_rn(make_float2(-u.x, -u.y), u, m2[p]);
                        float2 w;
                        if (kPolyEvery > 0 && (uu * P + p) % kPolyEvery == kPolyEvery - 1)
                            w = ex2_poly2(e);
                        else
                            w = make_float2(ex2f(e.x), ex2f(e.y));
                        den[p] = __fadd2_rn(den[p], w);
                        num[p] = __ffma2_rn(w, u, num[p]);
                    }
                }
            }
            for (; jj < a.j_batch; ++jj) {
                const int j = kMinibatch ? __ldg(bt + jj) : jj;
                const float2 xv = kGlobalX ? __ldg(xs + j * 32 + lane) : xs[j * 32 + lane];
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    const float2 u = __ffma2_rn(nas2, xv, zs[p]);
                    const float2 e = __ffma2_rn(make_float2(-u.x, -u.y), u, m2[p]);
                    const float2 w = make_float2(ex2f(e.x), ex2f(e.y));
                    den[p] = __fadd2_rn(den[p], w);
                    num[p] = __ffma2_rn(w, u, num[p]);
                }
            }
        };
        // pass 1: per-coordinate smallest |u| (the softmax shift of
        // proj/src/ensf.cpp:41-50, taken on |u| so no square is needed)
        auto nearest_pass = [&](float2 (&m2)[P]) {
            float2 mn[P];
#pragma unroll
            for (int p = 0; p < P; ++p) mn[p] = f2(FLT_MAX);
            if (kSorted) {
                nearest_abs_u<P>(xsf, lane, a.j_batch, top, c.nas, zs, mn);
            } else {
#pragma unroll 4
                for (int jj = 0; jj < a.j_batch; ++jj) {
                    const int j = kMinibatch ? __ldg(bt + jj) : jj;
                    const float2 xv = kGlobalX ? __ldg(xs + j * 32 + lane) : xs[j * 32 + lane];
#pragma unroll
                    for (int p = 0; p < P; ++p) {
                        const float2 u = __ffma2_rn(nas2, xv, zs[p]);
                        mn[p].x = fminf(mn[p].x, fabsf(u.x));
                        mn[p].y = fminf(mn[p].y, fabsf(u.y));
                    }
                }
            }
#pragma unroll
            for (int p = 0; p < P; ++p) m2[p] = __fmul2_rn(mn[p], mn[p]);
        };

        float2 m2[P], den[P], num[P];
        if (kShiftFree) {
            // shift c = 0: w = 2^(-u^2) is exact to fp32 rounding while the
            // nearest member has min u^2 <= 60 (then den >= 2^-min >= 2^-60
            // and nothing that matters reaches the 2^-126 flush).  Values with
            // den < 2^-60 (or NaN) are redone with the exact shift; the choice
            // is per value, so results do not depend on the warp's other lanes.
#pragma unroll
            for (int p = 0; p < P; ++p) m2[p] = f2(0.f);
            weight_pass(m2, den, num);
            unsigned redo = 0;
#pragma unroll
            for (int p = 0; p < P; ++p) {
                if (!(den[p].x >= 0x1.0p-60f)) redo |= 1u << (2 * p);
                if (!(den[p].y >= 0x1.0p-60f)) redo |= 2u << (2 * p);
            }
            if (__any_sync(0xffffffffu, redo != 0)) {
                // the other values keep c = 0 and recompute the same bits
                nearest_pass(m2);
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    if (!(redo & (1u << (2 * p)))) m2[p].x = 0.f;
                    if (!(redo & (2u << (2 * p)))) m2[p].y = 0.f;
                }
                weight_pass(m2, den, num);
            }
        } else {
            nearest_pass(m2);
            weight_pass(m2, den, num);
        }
        // posterior score + Euler-Maruyama, proj/src/ensf.cpp:197-214
#pragma unroll
        for (int p = 0; p < P; ++p) {
            // num / den per coordinate: a merged 1 / (den.x den.y) saves a
            // MUFU op but couples the pair's roundings, and a window edge can
            // split a pair, so results would depend on the sharding
            const float2 q = recip_mul<kNewtonRcp>(num[p], den[p]);
            float2 lik;
            if (a.obs_atan) {
                // h(z) = atan(z): H'^T R^-1 (y - h) = (B - A atan z) / (1 + z^2)
                lik.x = __fdividef(fmaf(nA2.x, atanf(z[p].x), B2.x), fmaf(z[p].x, z[p].x, 1.f));
                lik.y = __fdividef(fmaf(nA2.y, atanf(z[p].y), B2.y), fmaf(z[p].y, z[p].y, 1.f));
            } else {
                lik = __ffma2_rn(nA2, z[p], B2);
            }
            float2 xi;
            if constexpr (kJ > 0) xi = xi_early[p];
            else xi = normal_pair_f32(n0, uint32_t(i0 + p), a.cycle_lo, a.rk);
            float2 zn = __ffma2_rn(z[p], f2(c.nbdt), z[p]);
            zn = __ffma2_rn(f2(c.kp), q, zn);
            zn = __ffma2_rn(f2(c.kl), lik, zn);
            zn = __ffma2_rn(f2(c.sig), xi, zn);
            z[p] = zn;
            const bool fin = (fabsf(zn.x) <= FLT_MAX) && (fabsf(zn.y) <= FLT_MAX || !has_y);
            if (!fin) bad = min(bad, (uint32_t(p) << 30) | uint32_t(s));
        }
    }

    if (bad != UINT_MAX && kl < a.dl) {
        const int i = i0 + int(bad >> 30);  // particles past m are padding
        if (i < a.m) atomicMin(status, (uint64_t(i) << 32) | (bad & 0x3fffffffu));
    }
    if (kFused) {
        fused_relax_epilogue<P>(a, reinterpret_cast<float*>(smem), z_out, tile0, kl, i0, fstat, z);
        return;
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const int i = i0 + p;
        if (i >= a.m) continue;
        float* row = z_out + size_t(i) * size_t(a.dl);
        if (kl + 1 < a.dl) {
            if (aligned) {
                *reinterpret_cast<float2*>(row + kl) = z[p];
            } else {
                row[kl] = z[p].x;
                row[kl + 1] = z[p].y;
            }
        } else if (kl < a.dl) {
            row[kl] = z[p].x;
        }
    }
}


// fp64 forecast [m][dl] -> fp32 tiles [tile][m][64] (zero padded past dl).
// kSort: each of the 64 columns of a tile sorted ascending (NaN last, ties by
// member index) by rank counting; the rank of (j, c) is the number of members
// of column c that order before it, so the output is a permutation.
template <bool kSort>
__global__ void prep_tiles_kernel(const double* __restrict__ x, int m, int64_t dl,
                                  float* __restrict__ xt) {
    extern __shared__ float col[];  // [m][64] this tile's fp32 values
    const int64_t tile0 = int64_t(blockIdx.x) * kTile;
    float* out = xt + size_t(blockIdx.x) * size_t(m) * kTile;
    for (int q = threadIdx.x; q < m * kTile; q += blockDim.x) {
        const int j = q / kTile, c = q % kTile;
        const int64_t k = tile0 + c;
        const float v = k < dl ? float(x[size_t(j) * size_t(dl) + size_t(k)]) : 0.f;
        if (kSort)
            col[q] = v;
        else
            out[q] = v;
    }
    if (!kSort) return;
    __syncthreads();
    for (int q = threadIdx.x; q < m * kTile; q += blockDim.x) {
        const int j = q / kTile, c = q % kTile;
        const float v = col[q];
        const float kv = sort_key(v);
        int rank = 0;
        for (int i = 0; i < m; ++i) {
            const float ki = sort_key(col[i * kTile + c]);
            rank += (ki < kv) || (ki == kv && i < j);
        }
        out[rank * kTile + c] = v;
    }
}

// ---------------------------------------------------------------------------
// fp64 faithful kernel (reference arithmetic)
// ---------------------------------------------------------------------------
template <int P, bool kMinibatch, bool kSmemX>
__global__ void __launch_bounds__(128) ensf_f64_kernel(KernelArgs a, const double* __restrict__ x,
                                                       const double2* __restrict__ ab,
                                                       const StepF64* __restrict__ steps,
                                                       const int32_t* __restrict__ batches,
                                                       double* __restrict__ z_out,
                                                       unsigned long long* __restrict__ status) {
    extern __shared__ double2 smem2[];
    double2* xs = smem2;  // [m][32] when kSmemX; steps are read from global

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    const int64_t tile0 = int64_t(blockIdx.x) * kTile;
    const int64_t kl = tile0 + 2 * lane;
    const bool aligned = ((a.dl & 1) == 0);

    if (kSmemX) {
        for (int q = threadIdx.x; q < a.m * 32; q += blockDim.x) {
            const int j = q >> 5, l = q & 31;
            xs[q] = load_pair(x + size_t(j) * size_t(a.dl), tile0 + 2 * l, a.dl, aligned);
        }
    }
    double2 A = make_double2(0, 0), B = make_double2(0, 0);
    if (kl < a.dl) {
        const double2 o = ab[kl];
        A.x = o.x;
        B.x = o.y;
    }
    if (kl + 1 < a.dl) {
        const double2 o = ab[kl + 1];
        A.y = o.x;
        B.y = o.y;
    }
    __syncthreads();

    const int i0 = (blockIdx.y * nwarps + warp) * P;
    // warps past the last particle (N = 20 at P = 2: 10 groups in 3 CTAs of
    // 4 warps) leave instead of integrating padding particles; no barrier
    // follows
    if (i0 >= a.m) return;
    const uint64_t kg = uint64_t(a.k0 + kl);

    double zx[P], zy[P];
    int bad[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const double2 v = normal_pair_f64(kg, uint32_t(i0 + p), a.cycle_lo, a.key0, a.key1);
        zx[p] = v.x;
        zy[p] = v.y;
        bad[p] = INT_MAX;
    }

    for (int s = 0; s < a.n_steps; ++s) {
        const StepF64 c = steps[s];
        const int32_t* bt = kMinibatch ? batches + size_t(s) * size_t(a.j_batch) : nullptr;
        // weights w = fast_exp_nonpos((m - (z - alpha x_j)^2) / (2 beta^2)),
        // den = sum w, num = sum w x (proj/src/ensf.cpp:51-61)
        double nx[P], ny[P], ex[P], ey[P];
        auto weight_pass = [&](const double (&mx)[P], const double (&my)[P]) {
#pragma unroll
            for (int p = 0; p < P; ++p) nx[p] = ny[p] = ex[p] = ey[p] = 0.0;
            for (int jj = 0; jj < a.j_batch; ++jj) {
                const int j = kMinibatch ? __ldg(bt + jj) : jj;
                const double2 xv = kSmemX ? xs[j * 32 + lane]
                                          : load_pair(x + size_t(j) * size_t(a.dl), kl, a.dl, aligned);
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    const double dx = zx[p] - c.alpha * xv.x;
                    const double dy = zy[p] - c.alpha * xv.y;
                    const double wx = fast_exp_nonpos_dev((mx[p] - dx * dx) * c.inv2b);
                    const double wy = fast_exp_nonpos_dev((my[p] - dy * dy) * c.inv2b);
                    ex[p] += wx;
                    ey[p] += wy;
                    nx[p] += wx * xv.x;
                    ny[p] += wy * xv.y;
                }
            }
        };
        // Shift-free first: with shift 0 the weights differ from the
        // reference's min-shifted ones by one common factor, which cancels in
        // num / den, and only by exp rounding (1e-16) otherwise.  A value
        // whose weights all but vanish (den < 1e-280: every member beyond ~25
        // kernel widths, where the unshifted exp would underflow) is redone
        // with the reference's exact shift min_j (z - alpha x_j)^2
        // (proj/src/ensf.cpp:41-50); the choice is per value, so results do
        // not depend on which values share the warp.
        double mx[P], my[P];
#pragma unroll
        for (int p = 0; p < P; ++p) mx[p] = my[p] = 0.0;
        weight_pass(mx, my);
        unsigned redo = 0;
#pragma unroll
        for (int p = 0; p < P; ++p) {
            if (!(ex[p] >= 1e-280)) redo |= 1u << (2 * p);
            if (!(ey[p] >= 1e-280)) redo |= 2u << (2 * p);
        }
        if (__any_sync(0xffffffffu, redo != 0)) {
#pragma unroll
            for (int p = 0; p < P; ++p) mx[p] = my[p] = __longlong_as_double(0x7ff0000000000000ll);
            for (int jj = 0; jj < a.j_batch; ++jj) {
                const int j = kMinibatch ? __ldg(bt + jj) : jj;
                const double2 xv = kSmemX ? xs[j * 32 + lane]
                                          : load_pair(x + size_t(j) * size_t(a.dl), kl, a.dl, aligned);
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    const double dx = zx[p] - c.alpha * xv.x;
                    const double dy = zy[p] - c.alpha * xv.y;
                    const double d2x = dx * dx, d2y = dy * dy;
                    mx[p] = d2x < mx[p] ? d2x : mx[p];
                    my[p] = d2y < my[p] ? d2y : my[p];
                }
            }
#pragma unroll
            for (int p = 0; p < P; ++p) {
                if (!(redo & (1u << (2 * p)))) mx[p] = 0.0;
                if (!(redo & (2u << (2 * p)))) my[p] = 0.0;
            }
            weight_pass(mx, my);
        }
        const uint64_t n0 = uint64_t(s + 1) * uint64_t(a.d_total) + kg;
#pragma unroll
        for (int p = 0; p < P; ++p) {
            double scx = -(zx[p] - c.alpha * nx[p] / ex[p]) / c.beta2;
            double scy = -(zy[p] - c.alpha * ny[p] / ey[p]) / c.beta2;
            if (a.obs_atan) {
                scx += c.damp * ((B.x - A.x * atan(zx[p])) / (1.0 + zx[p] * zx[p]));
                scy += c.damp * ((B.y - A.y * atan(zy[p])) / (1.0 + zy[p] * zy[p]));
            } else {
                scx += c.damp * (B.x - A.x * zx[p]);
                scy += c.damp * (B.y - A.y * zy[p]);
            }
            const double2 xi = normal_pair_f64(n0, uint32_t(i0 + p), a.cycle_lo, a.key0, a.key1);
            zx[p] += -(c.b * zx[p] - c.s2 * scx) * c.dt + c.sig * xi.x;
            zy[p] += -(c.b * zy[p] - c.s2 * scy) * c.dt + c.sig * xi.y;
            const bool fin = isfinite(zx[p]) && (isfinite(zy[p]) || kl + 1 >= a.dl);
            if (!fin && bad[p] == INT_MAX) bad[p] = s;
        }
    }

#pragma unroll
    for (int p = 0; p < P; ++p) {
        const int i = i0 + p;
        if (i >= a.m || kl >= a.dl) continue;
        double* row = z_out + size_t(i) * size_t(a.dl);
        if (kl + 1 < a.dl) {
            if (aligned) {
                *reinterpret_cast<double2*>(row + kl) = make_double2(zx[p], zy[p]);
            } else {
                row[kl] = zx[p];
                row[kl + 1] = zy[p];
            }
        } else {
            row[kl] = zx[p];
        }
        if (bad[p] != INT_MAX) atomicMin(status, (uint64_t(i) << 32) | uint32_t(bad[p]));
    }
}

// ---------------------------------------------------------------------------
// relax_spread epilogue, proj/src/ensf.cpp:225-258 (+ ensemble_mean,
// proj/src/ensemble.cpp:7-16), fp64 statistics, one thread per coordinate.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void relax_kernel(const T* __restrict__ z, const double* __restrict__ x, int m,
                             int64_t dl, double factor, double* __restrict__ out) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= dl) return;
    if (factor == 0.0 || m < 2) {
        for (int j = 0; j < m; ++j) out[size_t(j) * dl + k] = double(z[size_t(j) * dl + k]);
        return;
    }
    double ma = 0.0, mb = 0.0;
    for (int j = 0; j < m; ++j) {
        ma += double(z[size_t(j) * dl + k]);
        mb += x[size_t(j) * dl + k];
    }
    const double inv = 1.0 / m;
    ma *= inv;
    mb *= inv;
    double va = 0.0, vb = 0.0;
    for (int j = 0; j < m; ++j) {
        const double da = double(z[size_t(j) * dl + k]) - ma;
        const double db = x[size_t(j) * dl + k] - mb;
        va += da * da;
        vb += db * db;
    }
    const double sa = fmax(sqrt(va / (m - 1)), 1e-12);
    const double sb = sqrt(vb / (m - 1));
    const double scale = (1.0 - factor) + factor * sb / sa;
    for (int j = 0; j < m; ++j)
        out[size_t(j) * dl + k] = ma + scale * (double(z[size_t(j) * dl + k]) - ma);
}

// obs -> per-coordinate {A, B}.  Identity: one entry per coordinate.
// r_stride 0: one error variance for every observation (TURBDA_R_UNIFORM)
__global__ void obs_identity_kernel(const double* __restrict__ y, const double* __restrict__ r,
                                    int64_t r_stride, int64_t dl, double2* __restrict__ ab) {
    // the fused analysis kernel may launch now (it waits for this grid's
    // results with griddepcontrol.wait before reading {A, B})
    asm volatile("griddepcontrol.launch_dependents;");
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k < dl) {
        const double inv = 1.0 / r[k * r_stride];
        ab[k] = make_double2(inv, y[k] * inv);
    }
}

// Selection, strictly increasing indices (every stride operator,
// make_grid_operator, proj/src/observation.cpp:29-41): at most one entry per
// coordinate, written directly.
__global__ void obs_select_unique_kernel(const double* __restrict__ y, const double* __restrict__ r,
                                         int64_t r_stride, const int64_t* __restrict__ idx,
                                         int64_t obs_dim, int64_t k0, int64_t dl,
                                         double2* __restrict__ ab) {
    // the fused analysis kernel may launch now (it waits for this grid's
    // results with griddepcontrol.wait before reading {A, B})
    asm volatile("griddepcontrol.launch_dependents;");
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= obs_dim) return;
    const int64_t k = idx[q] - k0;
    if (k < 0 || k >= dl) return;
    const double inv = 1.0 / r[q * r_stride];
    ab[k] = make_double2(inv, y[q] * inv);
}

// (window-local index, position) pairs to sort: an index outside the window
// [k0, k0 + dl) maps to the sentinel dl, so the keys span [0, dl] and the
// radix sort only runs over bitwidth(dl) bits
__global__ void window_keys_kernel(const int64_t* __restrict__ idx, int64_t n, int64_t k0,
                                   int64_t dl, uint32_t* __restrict__ keys,
                                   int32_t* __restrict__ pos) {
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int64_t k = idx[q] - k0;
    keys[q] = (k >= 0 && k < dl) ? uint32_t(k) : uint32_t(dl);
    pos[q] = int32_t(q);
}

// Selection, any index order (duplicates add, as adjoint_scatter does,
// proj/src/observation.cpp:18-27): (index, position) pairs stably sorted by
// index; the head of every run of equal indices sums its run in observation
// order.  No atomics: the sums are bitwise reproducible.
__global__ void obs_select_runs_kernel(const double* __restrict__ y, const double* __restrict__ r,
                                       int64_t r_stride, const uint32_t* __restrict__ keys,
                                       const int32_t* __restrict__ pos, int64_t obs_dim,
                                       int64_t dl, double2* __restrict__ ab) {
    // the fused analysis kernel may launch now (it waits for this grid's
    // results with griddepcontrol.wait before reading {A, B})
    asm volatile("griddepcontrol.launch_dependents;");
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= obs_dim) return;
    const uint32_t key = keys[t];
    if (t > 0 && keys[t - 1] == key) return;
    TB_CHECK(pos[t] >= 0 && pos[t] < obs_dim);
    const int64_t k = key;
    if (k >= dl) return;  // outside the window
    double A = 0.0, B = 0.0;
    for (int64_t u = t; u < obs_dim && keys[u] == key; ++u) {
        const int64_t q = pos[u];
        const double inv = 1.0 / r[q * r_stride];
        A += inv;
        B += y[q] * inv;
    }
    ab[k] = make_double2(A, B);
}

// likelihood_score, proj/src/ensf.cpp:84-94: B - A z (or the arctan chain
// rule) from the per-coordinate {A, B} of launch_obs_prep
__global__ void likelihood_kernel(const double* __restrict__ z, int64_t d,
                                  const double2* __restrict__ ab, int obs_atan,
                                  double* __restrict__ out) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= d) return;
    const double2 o = ab[k];
    out[k] = obs_atan ? (o.y - o.x * atan(z[k])) / (1.0 + z[k] * z[k]) : o.y - o.x * z[k];
}

// reverse_sde_step, proj/src/ensf.cpp:108-130, evaluated as :126 writes it;
// any non-finite result raises the flag
__global__ void sde_step_kernel(double* __restrict__ z, int64_t n, const double* __restrict__ sc,
                                const double* __restrict__ xi, double b, double s2, double dt,
                                double sig, unsigned int* __restrict__ bad) {
    const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= n) return;
    double v = z[q];
    v += -(b * v - s2 * sc[q]) * dt + sig * xi[q];
    z[q] = v;
    if (!isfinite(v)) *bad = 1u;
}

// single-vector componentwise score, proj/src/ensf.cpp:33-64,96-106
__global__ void score_kernel(const double* __restrict__ z, const double* __restrict__ x, int m,
                             int64_t d, const int32_t* __restrict__ batch, int nbatch,
                             double alpha, double beta2, const double2* __restrict__ ab,
                             double damp, int obs_atan, double* __restrict__ out) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= d) return;
    const double inv2b = 1.0 / (2.0 * beta2);
    const double zk = z[k];
    double mind2 = __longlong_as_double(0x7ff0000000000000ll);
    for (int jj = 0; jj < nbatch; ++jj) {
        const int j = batch ? batch[jj] : jj;
        const double diff = zk - alpha * x[size_t(j) * d + k];
        const double d2 = diff * diff;
        mind2 = d2 < mind2 ? d2 : mind2;
    }
    double num = 0.0, den = 0.0;
    for (int jj = 0; jj < nbatch; ++jj) {
        const int j = batch ? batch[jj] : jj;
        const double xv = x[size_t(j) * d + k];
        const double diff = zk - alpha * xv;
        const double w = fast_exp_nonpos_dev((mind2 - diff * diff) * inv2b);
        den += w;
        num += w * xv;
    }
    double s = -(zk - alpha * num / den) / beta2;
    if (ab)
        s += obs_atan ? damp * ((ab[k].y - ab[k].x * atan(zk)) / (1.0 + zk * zk))
                      : damp * (ab[k].y - ab[k].x * zk);
    out[k] = s;
}

// rmse/spread partial sums (proj/src/ensemble.cpp:18-43) in a fixed order:
// a fixed grid of kDiagBlocks CTAs, each thread strides the coordinates in a
// fixed sequence, the warp and block combine in a fixed tree, and one warp
// sums the block partials in block order.  No atomics: bitwise reproducible
// from run to run (the reference's byte-identical metrics contract,
// proj/tests/test_osse.cpp:163-179).
constexpr int kDiagBlocks = 592;  // 4 x 148 SMs

__global__ void __launch_bounds__(256) diag_kernel(const double* __restrict__ x, int m, int64_t d,
                                                   const double* __restrict__ truth,
                                                   double* __restrict__ part) {
    double e2 = 0.0, v2 = 0.0;
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < d;
         k += int64_t(gridDim.x) * blockDim.x) {
        double mean = 0.0;
        for (int j = 0; j < m; ++j) mean += x[size_t(j) * d + k];
        mean *= 1.0 / m;
        if (truth) {
            const double e = mean - truth[k];
            e2 += e * e;
        }
        for (int j = 0; j < m; ++j) {
            const double dv = x[size_t(j) * d + k] - mean;
            v2 += dv * dv;
        }
    }
    block_sum2_to(e2, v2, part + 2 * blockIdx.x);
}

int blocks_for(int64_t n, int t) { return int((n + t - 1) / t); }

// Ensembles whose fp32 tile ([m][64] floats) does not fit next to the step
// table in shared memory read their members from global memory (L1/L2).
bool f32_members_global(int m) { return sizeof(float) * 64 * size_t(m) > 200 * 1024; }

// Cross-check knobs read once per process (tests/ run both sides of each;
// the defaults are the measured best, profiles/r02_sweeps.md):
//   TURBDA_F32_POLY=0         every exponential on MUFU (default: the sorted
//                             kernels take one (member, particle) slot in 8
//                             from the FMA-pipe polynomial ex2_poly2)
//   TURBDA_F32_EXACT_SHIFT=1  always take the reference's exact softmax
//                             shift first (no shift-free pass)
//   TURBDA_F32_UNFUSED=1      prep_tiles -> ensf_f32 -> relax as three launches
//                             (the same arithmetic: bit-identical output)
//   TURBDA_F32_FUSE_ALL=1     the fused kernel also above 3 CTAs per tile
int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

template <class K>
cudaError_t launch_kernel(K kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                          const KernelArgs& a, const float* xt, const double2* ab,
                          const StepF32* steps, const int32_t* batches, float* z,
                          unsigned long long* status, bool dependent = false) {
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(smem));
        if (e != cudaSuccess) return e;
    }
    static const bool pdl = env_int("TURBDA_PDL", 1) != 0;
    if (!(dependent && pdl)) {
        kern<<<grid, block, smem, st>>>(a, xt, ab, steps, batches, z, status);
        return cudaGetLastError();
    }
    // programmatic dependent launch: the grid is scheduled while the
    // observation prep still runs, its prologue (forecast tile loads,
    // conversion, statistics) overlaps that kernel and the launch latency
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a, xt, ab, steps, batches, z, status);
}

// Kernel choice (sweeps in profiles/):
//  * sorted member tiles (N > 24), four tiles fit in shared memory: 8-warp
//    CTAs, 4 per SM (64 registers), 1/8 of the exponentials on the FMA-pipe
//    polynomial (config 2, config 5);
//  * sorted, one tile per SM (N >~ 440, config 4): one 32-warp CTA per SM
//    with the same 1/8 share;
//  * sorted, two or three tiles fit: 8-warp CTAs, 3 per SM, all MUFU;
//  * unsorted tiles (N <= 24, configs 1 and 3: brute-force redo shift):
//    CTAs of ceil(N/P) warps, 64 registers, all MUFU (the 1/8, 3/16 and 1/4
//    polynomial shares, 80-register and 32-48-register budgets, P = 1 / 2
//    and Box-Muller on the FMA pipe all measured slower or equal at config
//    3: the kernel sits at 86 % of the MUFU pipe, profiles/r02_sweeps.md);
//  * grids under a wave (config 1): P = 1 in 4-warp CTAs, and at N = 20 the
//    compile-time member loop with the noise drawn inside it;
//  * all of these fused: one launch per analysis;
//  * minibatches and ensembles whose tile exceeds shared memory: the
//    two-pass member loop, all MUFU, unfused.
constexpr int kPolySorted = 8;
constexpr int kPolyUnsorted = 0;

template <int P>
cudaError_t launch_f32_p(const KernelArgs& a, float* xt, const double2* ab,
                         const StepF32* steps, const int32_t* batches, float* z,
                         unsigned long long* status, cudaStream_t st, bool sorted) {
    static const int poly_env = env_int("TURBDA_F32_POLY", -1);
    static const bool exact = env_int("TURBDA_F32_EXACT_SHIFT", 0) != 0;
    static const bool unfused = env_int("TURBDA_F32_UNFUSED", 0) != 0;
    const int groups = (a.m + P - 1) / P;
    const bool global_x = f32_members_global(a.m);
    const size_t tile = sizeof(float) * kTile * size_t(a.m);
    const size_t smem_sm = size_t(227) * 1024;
    const bool wide = sorted && !exact && tile * 2 > smem_sm;  // one tile per SM
    // P = 1 (grids under a wave): 4-warp CTAs spread a tile's particles over
    // more SMs (config 1: 5 CTAs per tile, 4.3 per SM; 8-warp CTAs leave 60
    // SMs with 2 CTAs and 88 with 3)
    const int wmax = wide ? 32 : (P == 1 && !sorted) ? 4 : 8;
    // fewest CTAs per tile, warps spread evenly over them (N = 20 at P = 1:
    // 3 CTAs of 7 warps instead of 8 + 8 + 4 with 4 idle warps)
    const unsigned ny = unsigned((groups + wmax - 1) / wmax);
    const int nw = int((groups + ny - 1) / ny);
    // sorted tiles are fused when a tile spans at most 3 CTAs: measured
    // faster there (config 2: 2 CTAs, equal or better) and slower at 4
    // (config 5: 744 -> 756 ms, config 4: 5588 -> 5922 ms), where the
    // per-CTA prologue (fp64 loads, the O(N^2) tile sort) repeated by every
    // CTA of the tile and the last CTA's relax of N x 64 values outweigh the
    // two launches saved.  Unsorted tiles (N <= 24, no sort) are always
    // fused (config 3: 1 CTA, 190.3 -> 188.0 ms; config 1: 5 CTAs, 0.102
    // -> 0.093 ms)
    static const bool fuse_all = env_int("TURBDA_F32_FUSE_ALL", 0) != 0;
    const bool fused =
        !global_x && !a.minibatch && !exact && !unfused && (ny <= 3 || !sorted || fuse_all);
    // fused: + the sort staging columns, and room for the epilogue's
    // particles (nw P of them, which can exceed m by up to P - 1)
    const size_t smem =
        global_x ? 0
        : !fused ? tile
                 : std::max(tile + (sorted ? sizeof(float) * size_t(std::min(nw, kSortWarps)) *
                                                 size_t(a.m)
                                           : 0),
                            sizeof(float) * kTile * size_t(nw) * size_t(P));
    const unsigned tiles = unsigned((a.dl + kTile - 1) / kTile);
    const dim3 block(32 * nw);
    const dim3 grid(tiles, ny);
    if (!fused) {
        // fp64 forecast -> fp32 (sorted) tiles in global memory
        if (sorted) {
            if (tile > 48 * 1024) {
                cudaError_t e = cudaFuncSetAttribute(prep_tiles_kernel<true>,
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     int(tile));
                if (e != cudaSuccess) return e;
            }
            prep_tiles_kernel<true><<<tiles, 256, tile, st>>>(a.x64, a.m, a.dl, xt);
        } else {
            prep_tiles_kernel<false><<<tiles, 256, 0, st>>>(a.x64, a.m, a.dl, xt);
        }
        add_launches(1);
        if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) return e;
    }
    // fused over several CTAs: the tickets are zero (zeroed when the scratch
    // is allocated, reset by each tile's last CTA)
    auto go = [&](auto kern) {
        cudaError_t e = launch_kernel(kern, grid, block, smem, st, a, xt, ab, steps, batches, z,
                                      status, fused);
        add_launches(1);
        if (e != cudaSuccess || fused) return e;
        relax_kernel<float><<<blocks_for(a.dl, 256), 256, 0, st>>>(z, a.x64, a.m, a.dl, a.relax,
                                                                   a.out64);
        add_launches(1);
        return cudaGetLastError();
    };
    if (global_x)
        return a.minibatch ? go(ensf_f32_kernel<P, true, false, 0, 3, true>)
                           : go(ensf_f32_kernel<P, false, false, 0, 3, true>);
    if (a.minibatch) return go(ensf_f32_kernel<P, true, false, 0, 3>);
    if (!sorted) {
        if (exact) return go(ensf_f32_kernel<P, false, false, 0, 4, false, 256, false>);
        // grids under a wave with N = 20 (config 1): the member loop fully
        // unrolled at compile time with the step's noise drawn inside the same
        // basic block (ptxas interleaves the Philox / Box-Muller chain with the
        // exponentials), 4-warp CTAs, no register cap that matters at this
        // occupancy (with the 4-warp CTAs 0.102 -> 0.080 ms).  Same bits as the generic kernel
        // (same accumulation order); TURBDA_F32_J20=0 disables.  The even-n0
        // noise path needs even d_total and k0.
        static const bool j20 = env_int("TURBDA_F32_J20", 1) != 0;
        if constexpr (P == 1) {
            if (j20 && fused && a.j_batch == 20 && ((a.d_total | a.k0) & 1) == 0) {
                // 4-warp CTAs, 5 resident per SM (92 registers)
                return go(ensf_f32_kernel<1, false, false, 0, 5, false, 128, true, true, true, 20>);
            }
        }
        return fused ? go(ensf_f32_kernel<P, false, false, kPolyUnsorted, 4, false, 256, true, true>)
                     : go(ensf_f32_kernel<P, false, false, kPolyUnsorted, 4>);
    }
    // sorted member tiles always run P = 4 (launch_ensf_f32)
    if constexpr (P != 4) {
        return cudaErrorInvalidValue;
    } else {
    if (exact) return go(ensf_f32_kernel<P, false, true, 0, 3, false, 256, false>);
    if (wide)
        return fused ? go(ensf_f32_kernel<P, false, true, kPolySorted, 1, false, 1024, true, true>)
                     : go(ensf_f32_kernel<P, false, true, kPolySorted, 1, false, 1024>);
    if (smem * 4 <= smem_sm) {
        if (poly_env == 0)
            return fused ? go(ensf_f32_kernel<P, false, true, 0, 4, false, 256, true, true>)
                         : go(ensf_f32_kernel<P, false, true, 0, 4>);
        return fused ? go(ensf_f32_kernel<P, false, true, kPolySorted, 4, false, 256, true, true>)
                     : go(ensf_f32_kernel<P, false, true, kPolySorted, 4>);
    }
    return fused ? go(ensf_f32_kernel<P, false, true, 0, 3, false, 256, true, true>)
                 : go(ensf_f32_kernel<P, false, true, 0, 3>);
    }
}

template <int P, bool kSmemX>
cudaError_t launch_f64_p(const KernelArgs& a, const double* x, const double2* ab,
                         const StepF64* steps, const int32_t* batches, double* z,
                         unsigned long long* status, cudaStream_t st) {
    const int groups = (a.m + P - 1) / P;
    const int nw = groups < 4 ? groups : 4;
    const dim3 block(32 * nw);
    const dim3 grid(unsigned((a.dl + kTile - 1) / kTile), unsigned((groups + nw - 1) / nw));
    const size_t smem = kSmemX ? sizeof(double2) * 32 * size_t(a.m) : 0;
    // the register budget ptxas picks (114 at P = 2) beats capping it for
    // occupancy: config 3 1577 ms vs 1698 (80 regs) / 1747 ms (64 regs)
    auto kern = a.minibatch ? ensf_f64_kernel<P, true, kSmemX> : ensf_f64_kernel<P, false, kSmemX>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(smem));
        if (e != cudaSuccess) return e;
    }
    kern<<<grid, block, smem, st>>>(a, x, ab, steps, batches, z, status);
    return cudaGetLastError();
}

}  // namespace

size_t obs_prep_scratch_bytes(int64_t obs_dim) {
    if (obs_dim <= 0) return 0;
    size_t tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp, static_cast<const uint32_t*>(nullptr),
                                    static_cast<uint32_t*>(nullptr),
                                    static_cast<const int32_t*>(nullptr),
                                    static_cast<int32_t*>(nullptr), obs_dim);
    return 4 * align256(4 * size_t(obs_dim)) + align256(tmp);
}

cudaError_t launch_obs_prep(const double* y, const double* r, const int64_t* idx,
                            int64_t obs_dim, int obs_kind, int64_t k0, int64_t dl, double2* ab,
                            cudaStream_t st, int64_t r_stride, bool idx_increasing,
                            void* scratch, size_t scratch_bytes) {
    if (dl <= 0) return cudaSuccess;
    if (obs_dense(obs_kind)) {
        obs_identity_kernel<<<blocks_for(dl, 256), 256, 0, st>>>(y, r, r_stride, dl, ab);
        add_launches(1);
        return cudaGetLastError();
    }
    cudaError_t e = cudaMemsetAsync(ab, 0, sizeof(double2) * size_t(dl), st);
    if (e != cudaSuccess || obs_dim == 0) return e;
    if (obs_dim > INT32_MAX || dl >= int64_t(UINT32_MAX)) return cudaErrorInvalidValue;
    if (idx_increasing) {
        obs_select_unique_kernel<<<blocks_for(obs_dim, 256), 256, 0, st>>>(y, r, r_stride, idx,
                                                                          obs_dim, k0, dl, ab);
        add_launches(1);
        return cudaGetLastError();
    }
    if (!scratch || scratch_bytes < obs_prep_scratch_bytes(obs_dim)) return cudaErrorInvalidValue;
    const size_t seg = align256(4 * size_t(obs_dim));
    unsigned char* b = static_cast<unsigned char*>(scratch);
    uint32_t* keys_in = reinterpret_cast<uint32_t*>(b);
    uint32_t* keys = reinterpret_cast<uint32_t*>(b + seg);
    int32_t* pos_in = reinterpret_cast<int32_t*>(b + 2 * seg);
    int32_t* pos = reinterpret_cast<int32_t*>(b + 3 * seg);
    void* tmp = b + 4 * seg;
    size_t tmp_bytes = scratch_bytes - 4 * seg;
    window_keys_kernel<<<blocks_for(obs_dim, 256), 256, 0, st>>>(idx, obs_dim, k0, dl, keys_in,
                                                                pos_in);
    int end_bit = 1;
    while (end_bit < 32 && (uint64_t(1) << end_bit) <= uint64_t(dl)) ++end_bit;
    // LSD radix sort is stable: equal indices keep observation order
    e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys_in, keys, pos_in, pos, obs_dim, 0,
                                        end_bit, st);
    if (e != cudaSuccess) return e;
    obs_select_runs_kernel<<<blocks_for(obs_dim, 256), 256, 0, st>>>(y, r, r_stride, keys, pos,
                                                                    obs_dim, dl, ab);
    add_launches(3);
    return cudaGetLastError();
}

size_t ensf_f32_scratch_bytes(int m, int64_t dl) {
    return sizeof(float) * size_t(m) * size_t((dl + kTile - 1) / kTile) * kTile;
}

cudaError_t launch_ensf_f32(const KernelArgs& a, const double2* ab, const StepF32* steps,
                            const int32_t* batches, float* xt, float* z,
                            unsigned long long* status, cudaStream_t st, int64_t dl_concurrent) {
    if (a.dl <= 0) return cudaSuccess;
    // sorted tiles + binary-searched shift pay off past ~24 members; below,
    // the brute-force min pass is cheaper (measured, configs 1 and 3)
    const bool sorted = !a.minibatch && a.j_batch > 24 && !f32_members_global(a.m);
    // particles per warp: 4 when the grid still fills the GPU (a full wave
    // is 148 SMs x 24 warps), fewer for small windows so more warps exist
    const int64_t tiles_n = (std::max(a.dl, dl_concurrent) + kTile - 1) / kTile;
    const auto warps_for = [&](int pp) { return tiles_n * ((a.m + pp - 1) / pp); };
    const int64_t wave = 148 * 24;
    // (particles past m in the last warp are computed and discarded)
    // sorted tiles always take P = 4: their polynomial slots are a pattern
    // over (member, particle-in-warp), so one P for every window keeps
    // sharded results bit-identical to the whole-state call (tying the slot
    // to the member index instead measured 1.4-2.7 % slower, configs 2/4/5)
    if (sorted || ((a.m % 4 == 0 || a.m >= 32) && warps_for(4) >= wave))
        return launch_f32_p<4>(a, xt, ab, steps, batches, z, status, st, sorted);
    if ((a.m % 2 == 0 || a.m >= 16) && warps_for(2) >= wave / 2)
        return launch_f32_p<2>(a, xt, ab, steps, batches, z, status, st, sorted);
    return launch_f32_p<1>(a, xt, ab, steps, batches, z, status, st, sorted);
}

cudaError_t launch_ensf_f64(const KernelArgs& a, const double* x, const double2* ab,
                            const StepF64* steps, const int32_t* batches, double* z,
                            unsigned long long* status, cudaStream_t st) {
    if (a.dl <= 0) return cudaSuccess;
    const bool smem_x = a.m <= 160;
    if (a.m % 2 == 0)
        return smem_x ? launch_f64_p<2, true>(a, x, ab, steps, batches, z, status, st)
                      : launch_f64_p<2, false>(a, x, ab, steps, batches, z, status, st);
    return smem_x ? launch_f64_p<1, true>(a, x, ab, steps, batches, z, status, st)
                  : launch_f64_p<1, false>(a, x, ab, steps, batches, z, status, st);
}

cudaError_t launch_relax_f32(const float* z, const double* x, int m, int64_t dl, double factor,
                             double* out, cudaStream_t st) {
    if (dl <= 0) return cudaSuccess;
    relax_kernel<float><<<blocks_for(dl, 256), 256, 0, st>>>(z, x, m, dl, factor, out);
    return cudaGetLastError();
}

cudaError_t launch_relax_f64(const double* z, const double* x, int m, int64_t dl,
                             double factor, double* out, cudaStream_t st) {
    if (dl <= 0) return cudaSuccess;
    relax_kernel<double><<<blocks_for(dl, 256), 256, 0, st>>>(z, x, m, dl, factor, out);
    return cudaGetLastError();
}

cudaError_t launch_likelihood(const double* z, int64_t d, const double2* ab, int obs_atan,
                              double* out, cudaStream_t st) {
    if (d <= 0) return cudaSuccess;
    likelihood_kernel<<<blocks_for(d, 256), 256, 0, st>>>(z, d, ab, obs_atan, out);
    add_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_sde_step(double* z, int64_t n, const double* sc, const double* xi, double b,
                            double s2, double dt, double sig, unsigned int* bad,
                            cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    sde_step_kernel<<<blocks_for(n, 256), 256, 0, st>>>(z, n, sc, xi, b, s2, dt, sig, bad);
    add_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_score_f64(const double* z, const double* x, int m, int64_t d,
                             const int32_t* batch, int nbatch, double alpha, double beta2,
                             const double2* ab, double damp, int obs_atan, double* out,
                             cudaStream_t st) {
    if (d <= 0) return cudaSuccess;
    score_kernel<<<blocks_for(d, 128), 128, 0, st>>>(z, x, m, d, batch, nbatch, alpha, beta2, ab,
                                                      damp, obs_atan, out);
    return cudaGetLastError();
}

size_t diag_scratch_doubles() { return 2 + 2 * size_t(kDiagBlocks); }

cudaError_t launch_diag(const double* x, int m, int64_t d, const double* truth, double* out,
                        cudaStream_t st) {
    double* part = out + 2;
    diag_kernel<<<kDiagBlocks, 256, 0, st>>>(x, m, d, truth, part);
    sum_partials_kernel<<<1, 32, 0, st>>>(part, kDiagBlocks, out);
    add_launches(2);
    return cudaGetLastError();
}

}  // namespace tb200
