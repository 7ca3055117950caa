// Internal interface between the C-ABI layer (capi.cpp) and the sm_100a
// kernels (ensf_kernels.cu).  Not installed; the public surface is
// include/turbda_b200.h.
#pragma once
#include <cstdint>

#include <cuda_runtime.h>

#include "philox_keys.h"

// Checked builds (make CHECKED=1): device-side bounds assertions on every
// shared-memory tile / staging / scratch index and the global rows the
// kernels write - the stand-in for compute-sanitizer, which is closed on the
// GPU pool (profiles/r02_compute_sanitizer_closed.txt).  A failed check
// traps, so the call returns TURBDA_CUDA (cudaErrorAssert).
#ifdef TURBDA_CHECKED
#include <cassert>
#define TB_CHECK(cond) assert(cond)
#else
#define TB_CHECK(cond) ((void)0)
#endif

namespace tb200 {

#ifdef __CUDACC__
// bytes of dynamic shared memory of the running launch
__device__ __forceinline__ uint32_t dyn_smem_bytes() {
    uint32_t r;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
    return r;
}
#endif

// Per pseudo-time step coefficients of the fp32 fast kernel (32 B).  All are
// derived on the host in fp64 from the reference's time grid
// (proj/src/ensf.cpp:149,183-190) and rounded once.
// The kernel works with u = s (z - alpha x), s = sqrt(log2(e) / (2 beta^2)),
// so a softmax exponent is one FFMA2 away: log2 w = min u^2 - u^2.
struct StepF32 {
    float s;      // sqrt(log2(e) / (2 beta^2))
    float nas;    // -alpha(t) s
    float kp;     // -sigma^2 dt / (beta^2 s)   multiplies sum w u / sum w
    float kl;     // sigma^2 dt h(t)            multiplies B - A z (likelihood)
    float nbdt;   // -b(t) dt                   drift
    float sig;    // sqrt(sigma^2 dt)           noise amplitude
    float pad0, pad1;
};

// fp64 faithful kernel: the reference's own quantities, evaluated exactly as
// proj/src/ensf.cpp:183-190 does.
struct StepF64 {
    double alpha, beta2, inv2b, b, s2, damp, sig, dt;
};

struct KernelArgs {
    int64_t d_total;   // global state dimension (noise index stride)
    int64_t k0;        // global index of local coordinate 0
    int64_t dl;        // coordinates in this window
    int32_t m;         // ensemble members == particles
    int32_t n_steps;
    int32_t j_batch;   // members per step (== m unless minibatch)
    int32_t minibatch; // 1 when `batches` holds a [n_steps][j_batch] table
    uint32_t key0, key1;  // Philox key of the ensf_particles stream
    uint32_t cycle_lo;    // entity = (cycle << 32) | i  ->  hi word
    int32_t obs_atan;     // 1: h(x) = atan(x) (obs kinds 2, 3), 0: linear
    PhiloxKeys rk;        // round keys of (key0, key1)
    // fp32 analysis: the window's fp64 forecast [m][dl], the fp64 analysis
    // [m][dl] and relax_spread's factor (read by the fused kernel)
    const double* x64;
    double* out64;
    double relax;
    unsigned int* tile_ticket;  // fused, several CTAs per tile: [tiles] zeros
};

// observation operator kinds of the C-ABI (include/turbda_b200.h)
inline bool obs_dense(int kind) { return kind == 0 || kind == 2; }
inline bool obs_arctan(int kind) { return kind == 2 || kind == 3; }

// Divergence word: min over ((particle << 32) | step); ~0 = none.
constexpr unsigned long long kNoDivergence = ~0ull;

// obs (y, r, idx) -> per-coordinate {A = sum 1/r, B = sum y/r} over the
// window, summed in observation order without atomics.  Selection operators
// with strictly increasing indices (idx_increasing) write directly; any other
// index order is stably sorted first, in `scratch` (obs_prep_scratch_bytes).
size_t obs_prep_scratch_bytes(int64_t obs_dim);
cudaError_t launch_obs_prep(const double* y, const double* r, const int64_t* idx,
                            int64_t obs_dim, int obs_kind, int64_t k0, int64_t dl,
                            double2* ab, cudaStream_t st, int64_t r_stride,
                            bool idx_increasing, void* scratch, size_t scratch_bytes);

// fp32 analysis of a window: forecast a.x64 -> analysis a.out64 (fp64,
// [m][dl]) including relax_spread (a.relax).  Normally ONE fused launch
// (tile conversion/sort, all pseudo-steps, relax epilogue over a cluster of
// the tile's CTAs); minibatches, ensembles whose tile exceeds shared memory
// and the exact-shift cross-check run prep_tiles -> ensf_f32 -> relax with
// the fp32 tiles in `xt` (ensf_f32_scratch_bytes) and particles in `z`.
size_t ensf_f32_scratch_bytes(int m, int64_t dl);
inline size_t ensf_f32_ticket_bytes(int64_t dl) { return sizeof(unsigned int) * size_t((dl + 63) / 64 + 1); }
// dl_concurrent: coordinates analysed concurrently with this launch (the
// whole call when the host pipeline runs chunks side by side; 0 = a.dl),
// which sets the particles-per-warp choice.
cudaError_t launch_ensf_f32(const KernelArgs& a, const double2* ab, const StepF32* steps,
                            const int32_t* batches, float* xt, float* z,
                            unsigned long long* status, cudaStream_t st,
                            int64_t dl_concurrent = 0);
cudaError_t launch_ensf_f64(const KernelArgs& a, const double* x, const double2* ab,
                            const StepF64* steps, const int32_t* batches, double* z,
                            unsigned long long* status, cudaStream_t st);

// relax_spread epilogue (proj/src/ensf.cpp:225-258): z (T) + forecast -> out (fp64)
cudaError_t launch_relax_f32(const float* z, const double* x, int m, int64_t dl, double factor,
                             double* out, cudaStream_t st);
cudaError_t launch_relax_f64(const double* z, const double* x, int m, int64_t dl,
                             double factor, double* out, cudaStream_t st);

// likelihood_score / reverse_sde_step of the C++ API (host buffers staged)
cudaError_t launch_likelihood(const double* z, int64_t d, const double2* ab, int obs_atan,
                              double* out, cudaStream_t st);
cudaError_t launch_sde_step(double* z, int64_t n, const double* sc, const double* xi, double b,
                            double s2, double dt, double sig, unsigned int* bad,
                            cudaStream_t st);

// single-vector score (prior_score / posterior_score API), fp64 faithful
cudaError_t launch_score_f64(const double* z, const double* x, int m, int64_t d,
                             const int32_t* batch, int nbatch, double alpha, double beta2,
                             const double2* ab, double damp, int obs_atan, double* out,
                             cudaStream_t st);

// --- joint-norm mode (north_star extension, joint_kernels.cu) ----------------
struct JointPlan {
    int nchunk = 1;       // coordinate chunks of the Gram pass
    int64_t chunk = 16;   // coordinates per chunk
    int tiles = 1;        // 64 x 64 output tiles
    size_t red_len = 0;   // doubles in [G | nz | nx]
    size_t scratch = 0;   // doubles of `part` scratch launch_joint_gram needs
};
JointPlan joint_plan(int n, int m, int64_t dl);
cudaError_t launch_joint_init(const KernelArgs& a, double* z, cudaStream_t st);
// part: plan.scratch doubles; red: red_len doubles (the
// buffer a multi-GPU run allreduces)
cudaError_t launch_joint_gram(const KernelArgs& a, const JointPlan& pl, const double* z,
                              const double* x, double* part, double* red, cudaStream_t st);
// wn: m * m doubles of scratch; xbar: m * dl doubles of scratch (m > 64)
// f32_noise: particle normals from the fp32 Box-Muller (TURBDA_FP32)
cudaError_t launch_joint_update(const KernelArgs& a, const double* x, const double2* ab,
                                const double* red, double* wn, const StepF64& c, int step,
                                double* z, unsigned long long* status, bool f32_noise,
                                cudaStream_t st, double* xbar = nullptr);

// rmse / spread sums in a fixed order: out[0] = sum (mean - truth)^2,
// out[1] = sum dev^2; `out` holds diag_scratch_doubles() doubles (the
// per-CTA partials follow the two results)
size_t diag_scratch_doubles();
cudaError_t launch_diag(const double* x, int m, int64_t d, const double* truth, double* out,
                        cudaStream_t st);

// evidence counter behind turbda_launch_count() (kernels of this library)
void add_launches(uint64_t n);

}  // namespace tb200
