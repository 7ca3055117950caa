// Throughput of the EnSF pass-2 member loop alone (sm_100a): LDS.64 of a
// member pair + per particle FFMA2 (u), FFMA2 (e), 2x MUFU.EX2 (or the FMA
// polynomial), FADD2 (den), FFMA2 (num).  Reports pair-evals/clk/SM; the
// MUFU ceiling is 16.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float ex2f(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float2 ex2_poly2(float2 e) {
    e.x = fmaxf(e.x, -125.f); e.y = fmaxf(e.y, -125.f);
    const float2 t = __fadd2_rn(e, f2(12582912.f));
    const float2 f = __fadd2_rn(e, __fadd2_rn(f2(12582912.f), make_float2(-t.x, -t.y)));
    float2 p = __ffma2_rn(f2(0.001330954604782164f), f, f2(0.009673058986663818f));
    p = __ffma2_rn(p, f, f2(0.055505912750959396f));
    p = __ffma2_rn(p, f, f2(0.24022164940834045f));
    p = __ffma2_rn(p, f, f2(0.6931470632553101f));
    p = __ffma2_rn(p, f, f2(1.0000001192092896f));
    return make_float2(__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23)),
                       __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23)));
}

template <int P, int POLY, int MINB>
__global__ void __launch_bounds__(256, MINB) k(float* out, int J, int reps, float nas) {
  __shared__ float2 xs[64 * 32];
  const int lane = threadIdx.x & 31;
  for (int q = threadIdx.x; q < 64 * 32; q += blockDim.x) xs[q] = make_float2(0.01f * (q % 97) - 0.5f, 0.013f * (q % 89) - 0.6f);
  __syncthreads();
  float2 zs[P], m2[P], den[P], num[P];
  #pragma unroll
  for (int p = 0; p < P; ++p) { zs[p] = make_float2(0.1f * p + lane * 1e-3f, -0.2f * p); m2[p] = f2(0.f); den[p] = f2(0.f); num[p] = f2(0.f); }
  const float2 nas2 = f2(nas);
  for (int r = 0; r < reps; ++r) {
    for (int jj = 0; jj < J; jj += 4) {
      #pragma unroll
      for (int uu = 0; uu < 4; ++uu) {
        const float2 xv = xs[(jj + uu) * 32 + lane];
        #pragma unroll
        for (int p = 0; p < P; ++p) {
          const float2 u = __ffma2_rn(nas2, xv, zs[p]);
          const float2 e = __ffma2_rn(make_float2(-u.x, -u.y), u, m2[p]);
          float2 w;
          if (POLY > 0 && (uu * P + p) % POLY == POLY - 1) w = ex2_poly2(e);
          else w = make_float2(ex2f(e.x), ex2f(e.y));
          den[p] = __fadd2_rn(den[p], w);
          num[p] = __ffma2_rn(w, u, num[p]);
        }
      }
    }
    #pragma unroll
    for (int p = 0; p < P; ++p) { zs[p].x += 1e-7f * num[p].x; m2[p].y -= 1e-9f * den[p].y; }
  }
  float s = 0; for (int p = 0; p < P; ++p) s += den[p].x + den[p].y + num[p].x + num[p].y;
  if (s == 1.2345f) out[0] = s;
}

template <int P, int POLY, int MINB>
void run(const char* name) {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* d; cudaMalloc(&d, 64);
  const int J = 64, reps = 200;
  int bps = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k<P, POLY, MINB>, 256, 0);
  const int blocks = nsm * bps * 4;
  k<P, POLY, MINB><<<blocks, 256>>>(d, J, 2, -0.7f);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<P, POLY, MINB><<<blocks, 256>>>(d, J, reps, -0.7f);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k<P, POLY, MINB>);
  const double pairs = double(blocks) * 256 * reps * J * P * 2;
  printf("%-28s regs=%3d blocks/SM=%d  pair-evals/clk/SM = %.2f (at %d MHz)  %s\n", name, fa.numRegs, bps,
         pairs / (ms * 1e-3) / nsm / (clk * 1e3), clk / 1000, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<4, 0, 1>("P4 mufu");
  run<4, 0, 3>("P4 mufu minB3");
  run<2, 0, 4>("P2 mufu minB4");
  run<4, 4, 1>("P4 poly/4");
  run<4, 8, 1>("P4 poly/8");
  run<4, 8, 3>("P4 poly/8 minB3");
  run<4, 16, 3>("P4 poly/16 minB3");
  run<2, 8, 4>("P2 poly/8 minB4");
  run<8, 16, 2>("P8 poly/16 minB2");
  run<8, 0, 2>("P8 mufu minB2");
  return 0;
}
