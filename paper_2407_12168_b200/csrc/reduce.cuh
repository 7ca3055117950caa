// Fixed-order fp64 reductions (no atomics): a kernel with a FIXED grid
// writes one partial per CTA (warp shuffle tree, then the CTA's warps in
// warp order), and sum_partials_kernel adds the partials in CTA order.  The
// result depends only on the input and the grid size, never on scheduling,
// so per-cycle metrics are bitwise reproducible (the reference's
// byte-identical metrics CSV contract, proj/tests/test_osse.cpp:163-179).
#pragma once
#include <cstddef>

namespace tb200 {

inline size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

// Sum of (a, b) over the CTA (blockDim.x a multiple of 32, <= 1024) into
// out[0], out[1]; thread 0 writes.
__device__ __forceinline__ void block_sum2_to(double a, double b, double* out) {
    __shared__ double sa[32], sb[32];
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        sa[warp] = a;
        sb[warp] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double ta = 0.0, tb = 0.0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) {
            ta += sa[w];
            tb += sb[w];
        }
        out[0] = ta;
        out[1] = tb;
    }
}

// out[c] = sum over n pairs part[2q + c], q in order (one warp; lane l
// takes q = l, l + 32, ..., then a fixed shuffle tree).
static __global__ void sum_partials_kernel(const double* __restrict__ part, int n,
                                    double* __restrict__ out) {
    double a = 0.0, b = 0.0;
    for (int q = threadIdx.x; q < n; q += 32) {
        a += part[2 * q];
        b += part[2 * q + 1];
    }
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if (threadIdx.x == 0) {
        out[0] = a;
        out[1] = b;
    }
}

}  // namespace tb200
