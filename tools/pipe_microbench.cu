// Pipe-rate microbenchmark for the EnSF kernel design (sm_100a):
// MUFU.EX2 throughput, FFMA / FFMA2 (fma.rn.f32x2) throughput, DFMA throughput,
// IMAD.WIDE (Philox multiply) throughput.  Prints ops per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

__global__ void k_ex2(float* out, int iters, float seed) {
  float a[8];
  #pragma unroll
  for (int u = 0; u < 8; ++u) a[u] = seed * (threadIdx.x + u) * 1e-6f;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    #pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = ex2(a[u]) - 1.0f;   // ex2 + fadd
  }
  long long t1 = clock64();
  float s = 0; for (int u = 0; u < 8; ++u) s += a[u];
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0) out[1 + blockIdx.x] = float(t1 - t0);
}

__global__ void k_ffma(float* out, int iters, float seed) {
  float a[16];
  #pragma unroll
  for (int u = 0; u < 16; ++u) a[u] = seed + threadIdx.x + u;
  const float b = seed * 0.999f, c = seed * 1e-3f;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    #pragma unroll
    for (int u = 0; u < 16; ++u) a[u] = fmaf(a[u], b, c);
  }
  long long t1 = clock64();
  float s = 0; for (int u = 0; u < 16; ++u) s += a[u];
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0) out[1 + blockIdx.x] = float(t1 - t0);
}

__global__ void k_ffma2(float* out, int iters, float seed) {
  unsigned long long a[16];
  #pragma unroll
  for (int u = 0; u < 16; ++u) { float2 f = make_float2(seed + threadIdx.x + u, seed - u); a[u] = *reinterpret_cast<unsigned long long*>(&f); }
  float2 bf = make_float2(seed * 0.999f, seed * 0.998f), cf = make_float2(seed * 1e-3f, seed * 2e-3f);
  unsigned long long b = *reinterpret_cast<unsigned long long*>(&bf), c = *reinterpret_cast<unsigned long long*>(&cf);
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    #pragma unroll
    for (int u = 0; u < 16; ++u) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[u]) : "l"(b), "l"(c));
  }
  long long t1 = clock64();
  float s = 0; for (int u = 0; u < 16; ++u) { float2 f = *reinterpret_cast<float2*>(&a[u]); s += f.x + f.y; }
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0) out[1 + blockIdx.x] = float(t1 - t0);
}

__global__ void k_dfma(float* out, int iters, float seed) {
  double a[8];
  #pragma unroll
  for (int u = 0; u < 8; ++u) a[u] = seed + threadIdx.x + u;
  const double b = seed * 0.999, c = seed * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    #pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = fma(a[u], b, c);
  }
  long long t1 = clock64();
  double s = 0; for (int u = 0; u < 8; ++u) s += a[u];
  if (s == 12345.) out[0] = s;
  if (threadIdx.x == 0) out[1 + blockIdx.x] = float(t1 - t0);
}

__global__ void k_imadwide(float* out, int iters, unsigned seed) {
  unsigned a[8], b[8];
  #pragma unroll
  for (int u = 0; u < 8; ++u) { a[u] = seed + threadIdx.x + u; b[u] = seed ^ u; }
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    #pragma unroll
    for (int u = 0; u < 8; ++u) {
      unsigned long long p = (unsigned long long)a[u] * 0xD2511F53u;
      a[u] = (unsigned)(p >> 32) ^ b[u]; b[u] = (unsigned)p;
    }
  }
  long long t1 = clock64();
  unsigned s = 0; for (int u = 0; u < 8; ++u) s += a[u] + b[u];
  if (s == 12345u) out[0] = s;
  if (threadIdx.x == 0) out[1 + blockIdx.x] = float(t1 - t0);
}

template <typename K>
void run(const char* name, K kern, int ops_per_iter_per_thread, int threads, int iters) {
  int nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int blocks = nsm * (2048 / threads);
  float* d; cudaMalloc(&d, sizeof(float) * (blocks + 1));
  kern<<<blocks, threads>>>(d, 10, 1.0f);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(d, iters, 1.0f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  float* h = new float[blocks + 1]; cudaMemcpy(h, d, sizeof(float) * (blocks + 1), cudaMemcpyDeviceToHost);
  double cyc = 0; for (int b = 0; b < blocks; ++b) cyc = cyc > h[1 + b] ? cyc : h[1 + b];
  double ops = double(blocks) * threads * iters * ops_per_iter_per_thread;
  printf("%-10s ops/clk/SM (by clock64 max) = %7.2f   Gop/s = %9.1f   ms=%.3f  err=%s\n", name,
         ops / cyc / nsm * (2048.0 / threads) / (2048.0 / threads), ops / ms / 1e6, ms, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d); delete[] h;
}

int main() {
  int nsm, clk; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0); cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs=%d clock(kHz)=%d\n", nsm, clk);
  run("ex2", k_ex2, 8, 256, 4096);
  run("ffma", k_ffma, 16, 256, 4096);
  run("ffma2", k_ffma2, 32, 256, 4096);
  run("dfma", k_dfma, 8, 256, 1024);
  run("imadwide", k_imadwide, 8, 256, 4096);
  return 0;
}
