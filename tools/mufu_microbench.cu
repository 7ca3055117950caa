// What sustains MUFU.EX2 throughput on sm_100a?  Each variant reports
// MUFU.EX2 per clock per SM (one CTA of 512 threads per SM, many iterations).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float ex2nf(float x) { float y; asm volatile("ex2.approx.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

template <int V>
__global__ void k(float* out, long long* cyc, float seed, int iters) {
  float acc = 0.f;
  float2 st[8];
  for (int q = 0; q < 8; ++q) st[q] = make_float2(-1.0f - 0.01f * (threadIdx.x % 7) - q, -2.0f - q);
  const float2 k1 = f2(0.999f), k2 = f2(-0.001f);
  float2 den[8];
  for (int q = 0; q < 8; ++q) den[q] = f2(0.f);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (V == 0) {  // inputs from a packed FFMA2, outputs accumulated with FADD2 (pass-2 shape)
        const float2 e = __ffma2_rn(st[q], k1, k2);
        const float2 w = make_float2(ex2(e.x), ex2(e.y));
        den[q] = __fadd2_rn(den[q], w);
      } else if (V == 1) {  // same, inputs from two scalar FFMAs
        const float ex = fmaf(st[q].x, 0.999f, -0.001f), ey = fmaf(st[q].y, 0.998f, -0.002f);
        den[q].x += ex2(ex);
        den[q].y += ex2(ey);
      } else if (V == 2) {  // no-ftz variant
        const float2 e = __ffma2_rn(st[q], k1, k2);
        const float2 w = make_float2(ex2nf(e.x), ex2nf(e.y));
        den[q] = __fadd2_rn(den[q], w);
      } else if (V == 3) {  // one MUFU per FFMA2 pair (only .x)
        const float2 e = __ffma2_rn(st[q], k1, k2);
        den[q].x += ex2(e.x);
      } else if (V == 4) {  // exps of a large negative argument (typical weights)
        const float2 e = __ffma2_rn(st[q], f2(40.f), f2(-3.f));
        const float2 w = make_float2(ex2(e.x), ex2(e.y));
        den[q] = __fadd2_rn(den[q], w);
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) st[q] = __fadd2_rn(st[q], f2(1e-7f));
  }
  long long t1 = clock64();
  for (int q = 0; q < 8; ++q) acc += den[q].x + den[q].y;
  if (acc == 1.2345f) out[0] = acc;
  if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 32 + (threadIdx.x >> 5)] = t1 - t0;
}

template <int V>
void run(const char* name, int mufu_per_q) {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* d; long long* cyc; cudaMalloc(&d, 64); cudaMalloc(&cyc, sizeof(long long) * nsm * 32);
  const int iters = 2048;
  for (int threads : {256, 512, 1024}) {
    k<V><<<nsm, threads>>>(d, cyc, 1.f, iters);
    cudaDeviceSynchronize();
    long long h[148 * 32]; cudaMemcpy(h, cyc, sizeof(long long) * nsm * 32, cudaMemcpyDeviceToHost);
    long long mx = 0; for (int b = 0; b < nsm; ++b) for (int w = 0; w < threads / 32; ++w) mx = h[b * 32 + w] > mx ? h[b * 32 + w] : mx;
    const double mufu = double(threads) * iters * 8 * mufu_per_q;
    printf("%-32s threads/SM=%4d  MUFU.EX2 per clk per SM = %.2f (%s)\n", name, threads, mufu / mx,
           cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  run<0>("FFMA2 -> 2 ex2.ftz -> FADD2", 2);
  run<1>("2 FFMA -> 2 ex2.ftz -> 2 FADD", 2);
  run<2>("FFMA2 -> 2 ex2 (no ftz) -> FADD2", 2);
  run<3>("FFMA2 -> 1 ex2 -> FADD", 1);
  run<4>("FFMA2(large neg) -> 2 ex2 -> FADD2", 2);
  return 0;
}
