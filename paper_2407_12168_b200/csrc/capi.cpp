// C-ABI implementation (include/turbda_b200.h): validation, host-side
// precomputation of the pseudo-time grid and minibatch tables, per-device
// workspaces, H2D/D2H staging and the kernel sequence
//   obs_prep -> ensf_{f32,f64} (all pseudo-time steps fused) -> relax.
#include "turbda_b200.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <functional>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include "ensf_device.h"
#include "host_rng.h"

using namespace tb200;

namespace {

std::atomic<uint64_t> g_launches{0};

}  // namespace

void tb200::add_launches(uint64_t n) { g_launches += n; }

namespace {

// Optional live timing of the fused analysis kernel (bench.py's roofline):
// CUDA events recorded on the launching stream around each ensf launch.
std::atomic<int> g_profile{0};
std::mutex g_prof_mu;
struct ProfPair {
    cudaEvent_t a = nullptr, b = nullptr;
    int device = 0;
};
std::vector<ProfPair> g_prof_pending;
double g_prof_ms = 0.0;
uint64_t g_prof_n = 0;

int fail(turbda_status* st, int code, const std::string& msg) {
    if (st) {
        st->code = code;
        std::snprintf(st->msg, sizeof(st->msg), "%s", msg.c_str());
    }
    return code;
}

int cuda_fail(turbda_status* st, cudaError_t e, const char* where) {
    return fail(st, TURBDA_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define TB_CUDA(call)                                          \
    do {                                                       \
        cudaError_t e_ = (call);                               \
        if (e_ != cudaSuccess) return cuda_fail(st, e_, #call); \
    } while (0)

// Host copy pool for pageable buffers: the CUDA driver stages pageable
// memory through one internal pinned buffer on the calling thread (~9 GB/s
// measured on the B200 host); the analysis instead gathers each chunk into
// its own pinned slot with all pool threads and DMAs from there at the pinned
// rate, and scatters results (incl. first-touch page faults of a fresh
// output array) the same way.
class CopyPool {
public:
    static CopyPool& get() {
        // never destroyed: the detached workers wait on cv_ until the process
        // ends, and destroying a condition variable with waiters blocks exit
        static CopyPool* pool = new CopyPool;
        return *pool;
    }
    // fn(t) for t in [0, n), spread over the pool; returns when all are done
    void run(int64_t n, const std::function<void(int64_t)>& fn) {
        if (n <= 0) return;
        std::unique_lock<std::mutex> lk(run_mu_);  // one parallel region at a time
        {
            std::lock_guard<std::mutex> g(mu_);
            fn_ = &fn;
            n_ = n;
            next_ = 0;
            done_ = 0;
            ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> g(mu_);
        done_cv_.wait(g, [&] { return done_ == n_; });
        fn_ = nullptr;
    }

private:
    CopyPool() {
        const unsigned hw = std::thread::hardware_concurrency();
        const int nt = int(std::min<unsigned>(16, hw > 1 ? hw - 1 : 1));
        for (int t = 0; t < nt; ++t)
            std::thread([this] {
                uint64_t seen = 0;
                for (;;) {
                    {
                        std::unique_lock<std::mutex> g(mu_);
                        cv_.wait(g, [&] { return gen_ != seen; });
                        seen = gen_;
                    }
                    work();
                }
            }).detach();
    }
    void work() {
        for (;;) {
            int64_t t;
            const std::function<void(int64_t)>* fn;
            {
                std::lock_guard<std::mutex> g(mu_);
                if (!fn_ || next_ >= n_) return;
                t = next_++;
                fn = fn_;
            }
            (*fn)(t);
            std::lock_guard<std::mutex> g(mu_);
            if (++done_ == n_) done_cv_.notify_all();
        }
    }
    std::mutex run_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int64_t)>* fn_ = nullptr;
    int64_t n_ = 0, next_ = 0, done_ = 0;
    uint64_t gen_ = 0;
};

// m rows of `len` doubles between a row-pitched (or row-pointer) array and a
// contiguous [m][len] block, in ~1 MB pieces over the copy pool
void parallel_rows(int m, int64_t len, const std::function<void(int, int64_t, int64_t)>& piece) {
    const int64_t step = std::max<int64_t>(int64_t(1) << 17, 1);  // 1 MB of doubles
    const int64_t per_row = (len + step - 1) / step;
    CopyPool::get().run(int64_t(m) * per_row, [&](int64_t t) {
        const int j = int(t / per_row);
        const int64_t lo = (t % per_row) * step;
        piece(j, lo, std::min(len, lo + step) - lo);
    });
}

bool pageable(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return at.type == cudaMemoryTypeUnregistered;
}

// Pinned host buffer that only grows.
struct PinnedBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t reserve(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaHostAlloc(&p, bytes, cudaHostAllocDefault);
        if (e == cudaSuccess) cap = bytes;
        return e;
    }
    double* d() const { return static_cast<double*>(p); }
};

// Device buffer that only grows.
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t reserve(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        const size_t want = std::max<size_t>(bytes, 256);
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

// Per-device workspace, serialised by `mu` (calls are reentrant across devices).
struct Workspace {
    std::mutex mu;
    int device = -1;
    cudaStream_t stream = nullptr;
    DevBuf x, z, xt, ab, steps, batches, status, out, y, r, idx;
    DevBuf obs_tmp, diag;                       // obs sort scratch, diag partials
    DevBuf ticket;                              // fused fp32 kernel: per-tile tickets
    unsigned long long* status_host = nullptr;  // pinned
    void* comm = nullptr;                       // ncclComm_t (joint mode, sharded)
    int comm_world = 1;
    void* jsym = nullptr;                       // symmetric-window joint buffer
    void* jsym_win = nullptr;
    size_t jsym_bytes = 0;
    DevBuf jpart, jred, jw, jxbar;              // joint-mode scratch
    cudaGraphExec_t jgraph = nullptr;           // joint mode: captured pseudo-steps
    std::vector<cudaStream_t> cstreams;         // host-mode chunk pipeline
    std::vector<cudaEvent_t> ev_chunk;
    static constexpr int kSlots = 3;            // pageable staging ring
    PinnedBuf stage_in[kSlots], stage_out[kSlots];
    cudaEvent_t ev_out[kSlots] = {};
    cudaEvent_t ev_ready = nullptr;
    // the scratch above is shared by every call on this device: an
    // asynchronous call leaves its stream here and its completion in ev_done
    cudaStream_t pending = nullptr;
    cudaEvent_t ev_done = nullptr;
    // cached step table / batch table keys
    std::vector<unsigned char> steps_key, batch_key;
    // last analysis (for turbda_ensf_check)
    int last_m = 0, last_steps = 0;
    double last_eps = 0.0;
};

std::mutex g_ws_mu;
std::vector<std::unique_ptr<Workspace>> g_ws;

Workspace* workspace(int device) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    if (device < 0) return nullptr;
    if (size_t(device) >= g_ws.size()) g_ws.resize(size_t(device) + 1);
    if (!g_ws[size_t(device)]) {
        g_ws[size_t(device)] = std::make_unique<Workspace>();
        g_ws[size_t(device)]->device = device;
    }
    return g_ws[size_t(device)].get();
}

int ws_init(Workspace* w, turbda_status* st) {
    if (!w->stream) {
        TB_CUDA(cudaStreamCreateWithFlags(&w->stream, cudaStreamNonBlocking));
        TB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&w->status_host), 64));
        TB_CUDA(cudaEventCreateWithFlags(&w->ev_ready, cudaEventDisableTiming));
        TB_CUDA(cudaEventCreateWithFlags(&w->ev_done, cudaEventDisableTiming));
        for (cudaEvent_t& e : w->ev_out) TB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    return TURBDA_OK;
}

// A call on stream s may reuse the workspace only after an earlier
// asynchronous call (TURBDA_ASYNC) on another stream has finished with it.
cudaError_t ws_acquire(Workspace* w, cudaStream_t s) {
    if (w->pending && w->pending != s) return cudaStreamWaitEvent(s, w->ev_done, 0);
    return cudaSuccess;
}

// an asynchronous call hands the workspace over with its completion event;
// a synchronous one has drained it
cudaError_t ws_release(Workspace* w, cudaStream_t s, bool async) {
    if (!async) {
        w->pending = nullptr;
        return cudaSuccess;
    }
    w->pending = s;
    return cudaEventRecord(w->ev_done, s);
}

// proj/src/ensf.cpp:149,183-190 and proj/include/turbda/ensf.hpp:15-20
struct StepTimes {
    double t_ev, alpha, beta2, b, s2, damp, sig, dt;
};

std::vector<StepTimes> step_grid(int n_steps, double eps, double damping_t) {
    std::vector<StepTimes> g(static_cast<size_t>(n_steps));
    const double dt = (1.0 - eps) / n_steps;
    for (int s = 0; s < n_steps; ++s) {
        const double t_hi = 1.0 - s * dt;
        const double t = std::max(t_hi - dt, eps);
        StepTimes& q = g[size_t(s)];
        q.t_ev = t;
        q.alpha = 1.0 - t;
        q.beta2 = t;
        q.b = -1.0 / (1.0 - t);
        q.s2 = 1.0 + 2.0 * t / (1.0 - t);
        q.damp = damping_t - t;
        q.sig = std::sqrt(q.s2 * dt);
        q.dt = dt;
    }
    return g;
}

double step_time(int step, int n_steps, double eps) {
    const double dt = (1.0 - eps) / n_steps;
    return std::max(1.0 - step * dt - dt, eps);
}

// proj/src/ensf.cpp:151-168: partial Fisher-Yates per step
std::vector<int32_t> batch_table(uint64_t seed, uint64_t cycle, int m, int j, int n_steps) {
    std::vector<int32_t> t(size_t(n_steps) * size_t(j));
    std::vector<int32_t> pool(static_cast<size_t>(m));
    for (int s = 0; s < n_steps; ++s) {
        HostStream rs(seed, kUseEnsfBatch, (cycle << 20) + uint64_t(s));
        for (int q = 0; q < m; ++q) pool[size_t(q)] = q;
        for (int k = 0; k < j; ++k) {
            const int r = k + int(rs.next_u64() % uint64_t(m - k));
            std::swap(pool[size_t(k)], pool[size_t(r)]);
        }
        std::copy(pool.begin(), pool.begin() + j, t.begin() + size_t(s) * size_t(j));
    }
    return t;
}

template <class T>
std::vector<unsigned char> key_bytes(const T& v) {
    std::vector<unsigned char> k(sizeof(T));
    std::memcpy(k.data(), &v, sizeof(T));
    return k;
}

int validate(const turbda_ensf_params* p, turbda_status* st) {
    if (!p) return fail(st, TURBDA_CONFIG, "ensf: null params");
    // Ensemble::validate(false), include/turbda/ensemble.hpp:23-33
    if (p->n_members < 1) return fail(st, TURBDA_DIMENSION, "ensemble: empty");
    if (p->d_local < 0 || p->k0 < 0 || p->d_total < p->k0 + p->d_local)
        return fail(st, TURBDA_DIMENSION, "analyze: window outside the state");
    // Observation::validate length check, include/turbda/observation.hpp:49-55
    if (p->obs_kind < 0 || p->obs_kind > 3)
        return fail(st, TURBDA_CONFIG, "observation: unsupported operator kind");
    if (obs_dense(p->obs_kind) && p->obs_dim != p->d_local)
        return fail(st, TURBDA_DIMENSION, "observation: length mismatch");
    if (p->obs_dim < 0) return fail(st, TURBDA_DIMENSION, "observation: length mismatch");
    // EnsfConfig::validate, include/turbda/ensf.hpp:29-37
    if (!(p->eps > 0.0 && p->eps < 1.0)) return fail(st, TURBDA_CONFIG, "ensf: eps must lie in (0, 1)");
    if (p->n_steps < 10) return fail(st, TURBDA_CONFIG, "ensf: n_steps >= 10");
    if (p->minibatch_j < 0) return fail(st, TURBDA_CONFIG, "ensf: minibatch_j >= 0");
    if (p->relax_factor < 0.0 || p->relax_factor > 1.0)
        return fail(st, TURBDA_CONFIG, "ensf: relax_factor in [0, 1]");
    if (p->precision != TURBDA_FP32 && p->precision != TURBDA_FP64)
        return fail(st, TURBDA_CONFIG, "ensf: precision must be fp32 (0) or fp64 (1)");
    if (p->n_members > (1 << 24)) return fail(st, TURBDA_CONFIG, "ensf: too many members");
    if (p->score_mode != TURBDA_SCORE_COMPONENTWISE && p->score_mode != TURBDA_SCORE_JOINT)
        return fail(st, TURBDA_CONFIG, "ensf: unknown score_mode");
    if (p->score_mode == TURBDA_SCORE_JOINT && p->minibatch_j != 0 &&
        p->minibatch_j < p->n_members)
        return fail(st, TURBDA_CONFIG, "ensf: the joint score mode uses every member");
    return TURBDA_OK;
}

int validate_host_obs(const turbda_ensf_params* p, const double* r, const int64_t* idx,
                      turbda_status* st) {
    const int64_t nr = (p->flags & TURBDA_R_UNIFORM) ? std::min<int64_t>(p->obs_dim, 1) : p->obs_dim;
    for (int64_t q = 0; q < nr; ++q)
        if (!(r[q] > 0.0)) return fail(st, TURBDA_CONFIG, "observation: r_diag > 0");
    if (!obs_dense(p->obs_kind))
        for (int64_t q = 0; q < p->obs_dim; ++q)
            if (idx[q] < 0 || idx[q] >= p->d_total)
                return fail(st, TURBDA_DIMENSION, "observation: index outside the state");
    return TURBDA_OK;
}

// Selection indices in strictly increasing order (every stride operator):
// the observation prep writes them directly instead of sorting.
bool strictly_increasing(const int64_t* idx, int64_t n) {
    for (int64_t q = 1; q < n; ++q)
        if (idx[q] <= idx[q - 1]) return false;
    return true;
}

// {A, B} of a selection operator for the window [k0, k0 + dl) into ab.
int select_prep(Workspace* w, const double* dy, const double* dr, const int64_t* didx,
                const int64_t* host_idx, int64_t obs_dim, int obs_kind, int64_t k0, int64_t dl,
                double2* ab, int64_t r_stride, cudaStream_t s, turbda_status* st) {
    const bool inc = host_idx && strictly_increasing(host_idx, obs_dim);
    size_t bytes = 0;
    if (!inc) {
        bytes = obs_prep_scratch_bytes(obs_dim);
        TB_CUDA(w->obs_tmp.reserve(std::max<size_t>(bytes, 1)));
    }
    TB_CUDA(launch_obs_prep(dy, dr, didx, obs_dim, obs_kind, k0, dl, ab, s, r_stride, inc,
                            w->obs_tmp.p, bytes));
    return TURBDA_OK;
}

int diverged(const turbda_ensf_params* p, unsigned long long word, turbda_status* st) {
    if (word == kNoDivergence) return TURBDA_OK;
    const int particle = int(word >> 32);
    const int step = int(word & 0xffffffffu);
    const double t = step_time(step, p->n_steps, p->eps);
    if (st) {
        st->diverged_particle = particle;
        st->diverged_step = step;
        st->diverged_t = t;
    }
    // message text of SamplerDivergedError, include/turbda/errors.hpp:36-42
    return fail(st, TURBDA_DIVERGED, "reverse SDE diverged at pseudo-time t=" + std::to_string(t));
}

// Uploads the per-step coefficient table (cached by its defining parameters).
int upload_steps(Workspace* w, const turbda_ensf_params* p, cudaStream_t s, turbda_status* st) {
    struct Key {
        int32_t n_steps, precision;
        double eps, damping_t;
    } key{p->n_steps, p->precision, p->eps, p->damping_t};
    std::vector<unsigned char> kb = key_bytes(key);
    if (kb == w->steps_key && w->steps.p) return TURBDA_OK;
    const std::vector<StepTimes> g = step_grid(p->n_steps, p->eps, p->damping_t);
    if (p->precision == TURBDA_FP32) {
        std::vector<StepF32> h(g.size());
        const double log2e = 1.4426950408889634;
        for (size_t s2 = 0; s2 < g.size(); ++s2) {
            const StepTimes& q = g[s2];
            StepF32& o = h[s2];
            const double sc = std::sqrt(log2e / (2.0 * q.beta2));
            o.s = float(sc);
            o.nas = float(-q.alpha * sc);
            o.kp = float(-q.s2 * q.dt / (q.beta2 * sc));
            o.kl = float(q.s2 * q.dt * q.damp);
            o.nbdt = float(-q.b * q.dt);
            o.sig = float(q.sig);
            o.pad0 = o.pad1 = 0.f;
        }
        TB_CUDA(w->steps.reserve(sizeof(StepF32) * h.size()));
        TB_CUDA(cudaMemcpyAsync(w->steps.p, h.data(), sizeof(StepF32) * h.size(),
                                cudaMemcpyHostToDevice, s));
        TB_CUDA(cudaStreamSynchronize(s));
    } else {
        std::vector<StepF64> h(g.size());
        for (size_t s2 = 0; s2 < g.size(); ++s2) {
            const StepTimes& q = g[s2];
            h[s2] = StepF64{q.alpha, q.beta2, 1.0 / (2.0 * q.beta2), q.b, q.s2, q.damp, q.sig, q.dt};
        }
        TB_CUDA(w->steps.reserve(sizeof(StepF64) * h.size()));
        TB_CUDA(cudaMemcpyAsync(w->steps.p, h.data(), sizeof(StepF64) * h.size(),
                                cudaMemcpyHostToDevice, s));
        TB_CUDA(cudaStreamSynchronize(s));
    }
    w->steps_key = kb;
    return TURBDA_OK;
}

int upload_batches(Workspace* w, const turbda_ensf_params* p, int j_batch, cudaStream_t s,
                   turbda_status* st) {
    struct Key {
        uint64_t seed, cycle;
        int32_t m, j, n_steps;
    } key{p->seed, p->cycle, p->n_members, j_batch, p->n_steps};
    std::vector<unsigned char> kb = key_bytes(key);
    if (kb == w->batch_key && w->batches.p) return TURBDA_OK;
    const std::vector<int32_t> t = batch_table(p->seed, p->cycle, p->n_members, j_batch, p->n_steps);
    TB_CUDA(w->batches.reserve(sizeof(int32_t) * t.size()));
    TB_CUDA(cudaMemcpyAsync(w->batches.p, t.data(), sizeof(int32_t) * t.size(),
                            cudaMemcpyHostToDevice, s));
    TB_CUDA(cudaStreamSynchronize(s));
    w->batch_key = kb;
    return TURBDA_OK;
}

struct Window {
    int64_t k0_local;  // offset of this slice inside the enclosing window
    int64_t dl;        // coordinates in this slice
    int64_t off() const { return k0_local; }
};

constexpr int kMaxChunks = 32;  // >= 8 MB each: the exposed first H2D and last D2H shrink

int ws_streams(Workspace* w, int n, turbda_status* st) {
    while (int(w->cstreams.size()) < n) {
        cudaStream_t cs;
        cudaEvent_t ev;
        TB_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        TB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        w->cstreams.push_back(cs);
        w->ev_chunk.push_back(ev);
    }
    return TURBDA_OK;
}

int reduce_verdict_across_ranks(const turbda_ensf_params* p, Workspace* w,
                                unsigned long long* dstatus, cudaStream_t s, turbda_status* st);

// Runs one analysis slice on one device.  Host mode: `forecast`/`out` are the
// call's host arrays with row pitch p->d_local (or member rows); the slice
// starts at column win.k0_local.  The slice is cut into up to kMaxChunks (32)
// contiguous coordinate chunks, each on its own stream, so the H2D copy of
// chunk c+1, the kernels of chunk c and the D2H copy of chunk c-1 overlap
// (chunks are independent: the score is componentwise).  Device mode:
// pointers are device pointers of the whole window, one pass on the
// caller's stream.
int run_slice(const turbda_ensf_params* p, const Window& win, int device, const double* forecast,
              const double* const* frows, const double* y, const double* r, const int64_t* idx,
              double* out, double* const* orows, cudaStream_t user_stream, turbda_status* st) {
    const bool on_dev = (p->flags & TURBDA_INPUTS_ON_DEVICE) != 0;
    const bool r_uni = (p->flags & TURBDA_R_UNIFORM) != 0;
    const int64_t r_stride = r_uni ? 0 : 1;
    TB_CUDA(cudaSetDevice(device));
    Workspace* w = workspace(device);
    std::lock_guard<std::mutex> lk(w->mu);
    if (int rc = ws_init(w, st)) return rc;
    // device mode follows the caller's stream (NULL = the legacy default
    // stream, where the caller's buffers were most likely produced); host
    // mode runs on the workspace streams
    cudaStream_t s = user_stream ? user_stream : (on_dev ? cudaStreamLegacy : w->stream);
    TB_CUDA(ws_acquire(w, s));

    const int m = p->n_members;
    const int64_t dl = win.dl;
    const size_t md = size_t(m) * size_t(dl);
    const int j_batch = (p->minibatch_j == 0 || p->minibatch_j >= m) ? m : p->minibatch_j;
    const bool fp32 = p->precision == TURBDA_FP32;

    if (int rc = upload_steps(w, p, s, st)) return rc;
    if (j_batch != m)
        if (int rc = upload_batches(w, p, j_batch, s, st)) return rc;

    // chunking (host mode): >= 2 MB of forecast per chunk (at most
    // kMaxChunks), tile aligned; smaller chunks expose less of the first
    // H2D and the last D2H (config 2 e2e: 14.82 ms at 2 MB, 14.94 at 8 MB,
    // 16.80 unchunked; tools/sweep_chunks.sh)
    std::vector<Window> chunks;
    {
        const int64_t tiles = (dl + 63) / 64;
        int c = 1;
        if (!on_dev) {
            const int64_t bytes = int64_t(md) * int64_t(sizeof(double));
            static const int64_t chunk_bytes = [] {
                const char* e = std::getenv("TURBDA_CHUNK_MB");
                const int64_t mb = e ? std::atoll(e) : 0;
                return (mb > 0 ? mb : 2) << 20;
            }();
            c = int(std::min<int64_t>(kMaxChunks, std::max<int64_t>(1, bytes / chunk_bytes)));
            c = int(std::min<int64_t>(c, std::max<int64_t>(tiles, 1)));
        }
        int64_t start = 0;
        for (int q = 0; q < c; ++q) {
            const int64_t end = std::min<int64_t>(dl, (tiles * (q + 1) / c) * 64);
            chunks.push_back(Window{start, end - start});
            start = end;
        }
    }
    const int nc = int(chunks.size());
    if (int rc = ws_streams(w, nc, st)) return rc;
    // pageable host arrays above 32 MB go through the pinned staging ring
    constexpr int K = Workspace::kSlots;
    const bool staged =
        !on_dev && md * sizeof(double) >= (size_t(32) << 20) &&
        (pageable(frows ? static_cast<const void*>(frows[0]) : forecast) ||
         pageable(orows ? static_cast<const void*>(orows[0]) : out));
    if (staged) {
        size_t slot_bytes = 0;
        for (const Window& c : chunks) slot_bytes = std::max(slot_bytes, sizeof(double) * size_t(m) * size_t(c.dl));
        for (int q = 0; q < K; ++q) {
            TB_CUDA(w->stage_in[q].reserve(slot_bytes));
            TB_CUDA(w->stage_out[q].reserve(slot_bytes));
        }
    }
    // staged: results of chunk q leave the ring once its D2H has finished
    const auto drain = [&](int q) -> int {
        const Window& c = chunks[size_t(q)];
        if (c.dl <= 0 || m <= 0) return TURBDA_OK;
        TB_CUDA(cudaEventSynchronize(w->ev_out[q % K]));
        const double* src = w->stage_out[q % K].d();
        const int64_t col = win.k0_local + c.k0_local;
        parallel_rows(m, c.dl, [&](int j, int64_t lo, int64_t n) {
            double* dst = orows ? orows[j] + col : out + size_t(j) * size_t(p->d_local) + size_t(col);
            std::memcpy(dst + lo, src + size_t(j) * size_t(c.dl) + size_t(lo), sizeof(double) * size_t(n));
        });
        return TURBDA_OK;
    };

    // scratch: every chunk owns a disjoint region
    size_t xt_total = 0, tk_total = 0;
    std::vector<size_t> xt_off, tk_off;
    for (const Window& c : chunks) {
        xt_off.push_back(xt_total);
        tk_off.push_back(tk_total);
        xt_total += fp32 ? ensf_f32_scratch_bytes(m, c.dl) : 0;
        tk_total += fp32 ? ensf_f32_ticket_bytes(c.dl) : 0;
    }
    {
        // the fused kernel's per-tile tickets start at zero and each tile's
        // last CTA resets its own, so only a fresh allocation is cleared
        const void* before = w->ticket.p;
        TB_CUDA(w->ticket.reserve(std::max<size_t>(tk_total, 1)));
        if (w->ticket.p != before) TB_CUDA(cudaMemsetAsync(w->ticket.p, 0, w->ticket.cap, s));
    }
    TB_CUDA(w->z.reserve((fp32 ? sizeof(float) : sizeof(double)) * std::max<size_t>(md, 1)));
    TB_CUDA(w->xt.reserve(std::max<size_t>(xt_total, 1)));
    TB_CUDA(w->ab.reserve(sizeof(double2) * size_t(std::max<int64_t>(dl, 1))));
    TB_CUDA(w->status.reserve(64));
    unsigned long long* dstatus = w->status.as<unsigned long long>();
    TB_CUDA(cudaMemsetAsync(dstatus, 0xff, sizeof(unsigned long long), s));

    const double *dx0 = forecast, *dy = y, *dr = r;
    const int64_t* didx = idx;
    double* dout0 = out;
    if (!on_dev) {
        TB_CUDA(w->x.reserve(sizeof(double) * std::max<size_t>(md, 1)));
        TB_CUDA(w->out.reserve(sizeof(double) * std::max<size_t>(md, 1)));
        dx0 = w->x.as<double>();
        dout0 = w->out.as<double>();
        const size_t nb = size_t(std::max<int64_t>(obs_dense(p->obs_kind) ? dl : p->obs_dim, 1));
        TB_CUDA(w->y.reserve(sizeof(double) * nb));
        TB_CUDA(w->r.reserve(sizeof(double) * nb));
        dy = w->y.as<double>();
        dr = w->r.as<double>();
        if (r_uni && p->obs_dim > 0)
            TB_CUDA(cudaMemcpyAsync(w->r.p, r, sizeof(double), cudaMemcpyHostToDevice, s));
        if (!obs_dense(p->obs_kind)) {
            // selection entries are global: every chunk scans all of them
            TB_CUDA(w->idx.reserve(sizeof(int64_t) * nb));
            didx = w->idx.as<int64_t>();
            if (p->obs_dim > 0) {
                TB_CUDA(cudaMemcpyAsync(w->y.p, y, sizeof(double) * size_t(p->obs_dim),
                                        cudaMemcpyHostToDevice, s));
                if (!r_uni)
                    TB_CUDA(cudaMemcpyAsync(w->r.p, r, sizeof(double) * size_t(p->obs_dim),
                                            cudaMemcpyHostToDevice, s));
                TB_CUDA(cudaMemcpyAsync(w->idx.p, idx, sizeof(int64_t) * size_t(p->obs_dim),
                                        cudaMemcpyHostToDevice, s));
            }
        }
    }
    if (!obs_dense(p->obs_kind))
        if (int rc = select_prep(w, dy, dr, didx, on_dev ? nullptr : idx, p->obs_dim, p->obs_kind,
                                 p->k0 + win.k0_local, dl, w->ab.as<double2>(), r_stride, s, st))
            return rc;
    if (!on_dev) TB_CUDA(cudaEventRecord(w->ev_ready, s));

    KernelArgs a{};
    a.d_total = p->d_total;
    a.m = m;
    a.n_steps = p->n_steps;
    a.j_batch = j_batch;
    a.minibatch = j_batch != m;
    const uint64_t key = stream_key(p->seed, kUseEnsfParticles);
    a.key0 = uint32_t(key);
    a.key1 = uint32_t(key >> 32);
    a.cycle_lo = uint32_t(p->cycle);  // entity = (cycle << 32) | i
    a.obs_atan = obs_arctan(p->obs_kind) ? 1 : 0;
    a.rk = philox_round_keys(a.key0, a.key1);

    ProfPair prof;
    if (g_profile.load() && on_dev) {
        prof.device = device;
        TB_CUDA(cudaEventCreate(&prof.a));
        TB_CUDA(cudaEventCreate(&prof.b));
    }

    for (int q = 0; q < nc; ++q) {
        const Window& c = chunks[size_t(q)];
        cudaStream_t cs = on_dev ? s : w->cstreams[size_t(q)];
        const size_t moff = size_t(m) * size_t(c.off());
        const double* dx = on_dev ? forecast + 0 : dx0 + moff;
        double* dout = on_dev ? out : dout0 + moff;
        const int64_t col = win.k0_local + c.k0_local;  // column in the caller's arrays
        if (!on_dev) {
            TB_CUDA(cudaStreamWaitEvent(cs, w->ev_ready, 0));
            if (staged && c.dl > 0 && m > 0) {
                // the slot's previous chunk (q - K) must have left the ring
                if (q >= K)
                    if (int rc = drain(q - K)) return rc;
                double* slot = w->stage_in[q % K].d();
                parallel_rows(m, c.dl, [&](int j, int64_t lo, int64_t n) {
                    const double* src = frows ? frows[j] + col
                                              : forecast + size_t(j) * size_t(p->d_local) + size_t(col);
                    std::memcpy(slot + size_t(j) * size_t(c.dl) + size_t(lo), src + lo,
                                sizeof(double) * size_t(n));
                });
                TB_CUDA(cudaMemcpyAsync(w->x.as<double>() + moff, slot,
                                        sizeof(double) * size_t(m) * size_t(c.dl),
                                        cudaMemcpyHostToDevice, cs));
            } else if (c.dl > 0 && m > 0) {
                if (frows) {
                    for (int j = 0; j < m; ++j)
                        TB_CUDA(cudaMemcpyAsync(w->x.as<double>() + moff + size_t(j) * size_t(c.dl),
                                                frows[j] + col, sizeof(double) * size_t(c.dl),
                                                cudaMemcpyHostToDevice, cs));
                } else {
                    TB_CUDA(cudaMemcpy2DAsync(w->x.as<double>() + moff, sizeof(double) * size_t(c.dl),
                                              forecast + col, sizeof(double) * size_t(p->d_local),
                                              sizeof(double) * size_t(c.dl), size_t(m),
                                              cudaMemcpyHostToDevice, cs));
                }
            }
            if (obs_dense(p->obs_kind) && c.dl > 0) {
                TB_CUDA(cudaMemcpyAsync(w->y.as<double>() + c.k0_local, y + col,
                                        sizeof(double) * size_t(c.dl), cudaMemcpyHostToDevice, cs));
                if (!r_uni)
                    TB_CUDA(cudaMemcpyAsync(w->r.as<double>() + c.k0_local, r + col,
                                            sizeof(double) * size_t(c.dl), cudaMemcpyHostToDevice,
                                            cs));
            }
        }
        const int64_t k0c = p->k0 + col;
        double2* abc = w->ab.as<double2>() + c.k0_local;
        if (obs_dense(p->obs_kind))
            TB_CUDA(launch_obs_prep(dy + c.k0_local, r_uni ? dr : dr + c.k0_local, nullptr, c.dl,
                                    p->obs_kind, k0c, c.dl, abc, cs, r_stride, true, nullptr, 0));
        a.k0 = k0c;
        a.dl = c.dl;
        if (prof.a) TB_CUDA(cudaEventRecord(prof.a, cs));
        if (fp32) {
            // one fused launch: tiles, every pseudo-step, relax_spread
            a.x64 = dx;
            a.out64 = dout;
            a.relax = p->relax_factor;
            a.tile_ticket = reinterpret_cast<unsigned int*>(w->ticket.as<unsigned char>() +
                                                            tk_off[size_t(q)]);
            float* zc = w->z.as<float>() + moff;
            TB_CUDA(launch_ensf_f32(a, abc, w->steps.as<StepF32>(), w->batches.as<int32_t>(),
                                    reinterpret_cast<float*>(w->xt.as<unsigned char>() + xt_off[size_t(q)]),
                                    zc, dstatus, cs, dl));
            if (prof.b) TB_CUDA(cudaEventRecord(prof.b, cs));
        } else {
            double* zc = w->z.as<double>() + moff;
            TB_CUDA(launch_ensf_f64(a, dx, abc, w->steps.as<StepF64>(), w->batches.as<int32_t>(),
                                    zc, dstatus, cs));
            if (prof.b) TB_CUDA(cudaEventRecord(prof.b, cs));
            TB_CUDA(launch_relax_f64(zc, dx, m, c.dl, p->relax_factor, dout, cs));
        }
        if (staged && c.dl > 0 && m > 0) {
            TB_CUDA(cudaMemcpyAsync(w->stage_out[q % K].p, dout, sizeof(double) * size_t(m) * size_t(c.dl),
                                    cudaMemcpyDeviceToHost, cs));
            TB_CUDA(cudaEventRecord(w->ev_out[q % K], cs));
        }
        if (!fp32) g_launches += 2;  // (the fp32 path counts its own launches)
    }
    if (prof.a) {
        std::lock_guard<std::mutex> lk2(g_prof_mu);
        g_prof_pending.push_back(prof);
    }
    w->last_m = m;
    w->last_steps = p->n_steps;
    w->last_eps = p->eps;

    if (on_dev && (p->flags & TURBDA_ASYNC)) {
        if (int rc = reduce_verdict_across_ranks(p, w, dstatus, s, st)) return rc;
        TB_CUDA(ws_release(w, s, true));
        return TURBDA_OK;
    }

    if (staged)
        for (int q = std::max(0, nc - K); q < nc; ++q)
            if (int rc = drain(q)) return rc;
    if (!on_dev) {
        // results back per chunk, in chunk order (for pageable destinations
        // each copy returns once its chunk is done; later chunks keep running)
        for (int q = 0; q < nc && !staged; ++q) {
            const Window& c = chunks[size_t(q)];
            if (c.dl <= 0 || m <= 0) continue;
            cudaStream_t cs = w->cstreams[size_t(q)];
            const size_t moff = size_t(m) * size_t(c.off());
            const int64_t col = win.k0_local + c.k0_local;
            if (orows) {
                for (int j = 0; j < m; ++j)
                    TB_CUDA(cudaMemcpyAsync(orows[j] + col, dout0 + moff + size_t(j) * size_t(c.dl),
                                            sizeof(double) * size_t(c.dl), cudaMemcpyDeviceToHost, cs));
            } else {
                TB_CUDA(cudaMemcpy2DAsync(out + col, sizeof(double) * size_t(p->d_local),
                                          dout0 + moff, sizeof(double) * size_t(c.dl),
                                          sizeof(double) * size_t(c.dl), size_t(m),
                                          cudaMemcpyDeviceToHost, cs));
            }
        }
        for (int q = 0; q < nc; ++q) {
            TB_CUDA(cudaEventRecord(w->ev_chunk[size_t(q)], w->cstreams[size_t(q)]));
            TB_CUDA(cudaStreamWaitEvent(s, w->ev_chunk[size_t(q)], 0));
        }
    }
    // every chunk stream has been joined into s: the verdict is final here
    if (int rc = reduce_verdict_across_ranks(p, w, dstatus, s, st)) return rc;
    TB_CUDA(cudaMemcpyAsync(w->status_host, dstatus, sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, s));
    TB_CUDA(cudaStreamSynchronize(s));
    TB_CUDA(ws_release(w, s, false));
    return diverged(p, *w->status_host, st);
}

// --- NCCL, loaded on first use --------------------------------------------
struct NcclApi {
    bool tried = false, ok = false;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                               ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    // NCCL >= 2.27 symmetric memory (optional): ncclMemAlloc'd buffers
    // registered as a collective window let small allreduces take NCCL's
    // symmetric (NVLS / load-store) kernels
    ncclResult_t (*mem_alloc)(void**, size_t) = nullptr;
    ncclResult_t (*mem_free)(void*) = nullptr;
    ncclResult_t (*win_register)(ncclComm_t, void*, size_t, void**, int) = nullptr;
    ncclResult_t (*win_deregister)(ncclComm_t, void*) = nullptr;
};
std::mutex g_nccl_mu;
NcclApi g_nccl;

NcclApi* nccl_api() {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (!g_nccl.tried) {
        g_nccl.tried = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            g_nccl.get_unique_id = reinterpret_cast<decltype(g_nccl.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
            g_nccl.comm_init_rank = reinterpret_cast<decltype(g_nccl.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
            g_nccl.comm_init_all = reinterpret_cast<decltype(g_nccl.comm_init_all)>(dlsym(h, "ncclCommInitAll"));
            g_nccl.all_reduce = reinterpret_cast<decltype(g_nccl.all_reduce)>(dlsym(h, "ncclAllReduce"));
            g_nccl.comm_destroy = reinterpret_cast<decltype(g_nccl.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
            g_nccl.error_string = reinterpret_cast<decltype(g_nccl.error_string)>(dlsym(h, "ncclGetErrorString"));
            g_nccl.ok = g_nccl.get_unique_id && g_nccl.comm_init_rank && g_nccl.comm_init_all &&
                        g_nccl.all_reduce && g_nccl.comm_destroy && g_nccl.error_string;
            g_nccl.mem_alloc = reinterpret_cast<decltype(g_nccl.mem_alloc)>(dlsym(h, "ncclMemAlloc"));
            g_nccl.mem_free = reinterpret_cast<decltype(g_nccl.mem_free)>(dlsym(h, "ncclMemFree"));
            g_nccl.win_register =
                reinterpret_cast<decltype(g_nccl.win_register)>(dlsym(h, "ncclCommWindowRegister"));
            g_nccl.win_deregister =
                reinterpret_cast<decltype(g_nccl.win_deregister)>(dlsym(h, "ncclCommWindowDeregister"));
        }
    }
    return g_nccl.ok ? &g_nccl : nullptr;
}

int nccl_fail(turbda_status* st, NcclApi* api, ncclResult_t r, const char* where) {
    return fail(st, TURBDA_CUDA, std::string(where) + ": " + (api ? api->error_string(r) : "nccl"));
}

// collective, like the registration: every rank destroys its communicator
void release_symmetric(Workspace* w, NcclApi* api) {
    if (w->jsym_win && api->win_deregister)
        api->win_deregister(static_cast<ncclComm_t>(w->comm), w->jsym_win);
    if (w->jsym && api->mem_free) api->mem_free(w->jsym);
    w->jsym = nullptr;
    w->jsym_win = nullptr;
    w->jsym_bytes = 0;
}

// The joint mode's per-step [G | nz | nx] buffer for a sharded call: with
// NCCL symmetric memory, an ncclMemAlloc'd buffer registered once as a
// symmetric window of the communicator (collective - every rank reaches this
// point in the same call), else the plain workspace buffer.
// TURBDA_NCCL_SYMMETRIC=0 forces the plain buffer.
int joint_red_buffer(Workspace* w, NcclApi* api, void* comm, size_t bytes, turbda_status* st,
                     double** out) {
    static const bool sym_env = [] {
        const char* e = std::getenv("TURBDA_NCCL_SYMMETRIC");
        return !(e && std::atoi(e) == 0);
    }();
    const bool sym = sym_env && api && api->mem_alloc && api->mem_free && api->win_register &&
                     api->win_deregister && w->comm && comm == w->comm;
    if (!sym) {
        TB_CUDA(w->jred.reserve(bytes));
        *out = w->jred.as<double>();
        return TURBDA_OK;
    }
    if (bytes > w->jsym_bytes) {
        const ncclComm_t comm = static_cast<ncclComm_t>(w->comm);
        if (w->jsym_win) api->win_deregister(comm, w->jsym_win);
        if (w->jsym) api->mem_free(w->jsym);
        w->jsym = nullptr;
        w->jsym_win = nullptr;
        w->jsym_bytes = 0;
        const size_t want = (bytes + 4095) & ~size_t(4095);
        ncclResult_t r = api->mem_alloc(&w->jsym, want);
        if (r != ncclSuccess) return nccl_fail(st, api, r, "ncclMemAlloc");
        r = api->win_register(comm, w->jsym, want, &w->jsym_win, NCCL_WIN_COLL_SYMMETRIC);
        if (r != ncclSuccess) return nccl_fail(st, api, r, "ncclCommWindowRegister");
        w->jsym_bytes = want;
    }
    *out = static_cast<double*>(w->jsym);
    return TURBDA_OK;
}

// A window of a state sharded over ranks that share a communicator
// (turbda_comm_init): the divergence verdict is min-reduced over the ranks,
// so every rank reports the globally first (particle, step) - the error the
// unsharded reference run raises.
int reduce_verdict_across_ranks(const turbda_ensf_params* p, Workspace* w,
                                unsigned long long* dstatus, cudaStream_t s, turbda_status* st) {
    if (!(p->flags & TURBDA_SHARDED) || !w->comm || w->comm_world <= 1) return TURBDA_OK;
    NcclApi* api = nccl_api();
    if (!api) return fail(st, TURBDA_CUDA, "libnccl.so.2 not loadable");
    const ncclResult_t r = api->all_reduce(dstatus, dstatus, 1, ncclUint64, ncclMin,
                                           static_cast<ncclComm_t>(w->comm), s);
    if (r != ncclSuccess) return nccl_fail(st, api, r, "ncclAllReduce(verdict)");
    return TURBDA_OK;
}

// In-process cliques for device_count > 1 joint runs: comms[g] for device dev0 + g.
std::mutex g_clique_mu;
std::vector<std::pair<std::pair<int, int>, std::vector<ncclComm_t>>> g_cliques;

int clique(int dev0, int ndev, std::vector<ncclComm_t>* out, turbda_status* st) {
    std::lock_guard<std::mutex> lk(g_clique_mu);
    for (auto& c : g_cliques)
        if (c.first == std::make_pair(dev0, ndev)) {
            *out = c.second;
            return TURBDA_OK;
        }
    NcclApi* api = nccl_api();
    if (!api) return fail(st, TURBDA_CUDA, "libnccl.so.2 not loadable");
    std::vector<ncclComm_t> comms(static_cast<size_t>(ndev));
    std::vector<int> devs(static_cast<size_t>(ndev));
    for (int g = 0; g < ndev; ++g) devs[size_t(g)] = dev0 + g;
    ncclResult_t r = api->comm_init_all(comms.data(), ndev, devs.data());
    if (r != ncclSuccess) return nccl_fail(st, api, r, "ncclCommInitAll");
    g_cliques.push_back({{dev0, ndev}, comms});
    *out = comms;
    return TURBDA_OK;
}

// Joint-norm analysis of one window on one device (joint_kernels.cu).  Host
// mode copies X / obs in and the analysis out; `comm` (nullable) sums the
// per-step [G | nz | nx] buffer over the ranks that share the state.
int run_joint(const turbda_ensf_params* p, const Window& win, int device, const double* forecast,
              const double* const* frows, const double* y, const double* r, const int64_t* idx,
              double* out, double* const* orows, cudaStream_t user_stream, void* comm,
              turbda_status* st) {
    const bool on_dev = (p->flags & TURBDA_INPUTS_ON_DEVICE) != 0;
    const bool r_uni = (p->flags & TURBDA_R_UNIFORM) != 0;
    TB_CUDA(cudaSetDevice(device));
    Workspace* w = workspace(device);
    std::lock_guard<std::mutex> lk(w->mu);
    if (int rc = ws_init(w, st)) return rc;
    cudaStream_t s = user_stream ? user_stream : (on_dev ? cudaStreamLegacy : w->stream);
    TB_CUDA(ws_acquire(w, s));
    const int m = p->n_members;
    const int64_t dl = win.dl;
    const size_t md = size_t(m) * size_t(std::max<int64_t>(dl, 1));

    const double *dx = forecast, *dy = y, *dr = r;
    const int64_t* didx = idx;
    double* dout = out;
    const bool dense = obs_dense(p->obs_kind);
    if (!on_dev) {
        TB_CUDA(w->x.reserve(sizeof(double) * md));
        TB_CUDA(w->out.reserve(sizeof(double) * md));
        const size_t nb = size_t(std::max<int64_t>(dense ? dl : p->obs_dim, 1));
        TB_CUDA(w->y.reserve(sizeof(double) * nb));
        TB_CUDA(w->r.reserve(sizeof(double) * nb));
        TB_CUDA(w->idx.reserve(sizeof(int64_t) * nb));
        if (dl > 0) {
            if (frows) {
                for (int j = 0; j < m; ++j)
                    TB_CUDA(cudaMemcpyAsync(w->x.as<double>() + size_t(j) * size_t(dl),
                                            frows[j] + win.k0_local, sizeof(double) * size_t(dl),
                                            cudaMemcpyHostToDevice, s));
            } else {
                TB_CUDA(cudaMemcpy2DAsync(w->x.p, sizeof(double) * size_t(dl),
                                          forecast + win.k0_local, sizeof(double) * size_t(p->d_local),
                                          sizeof(double) * size_t(dl), size_t(m),
                                          cudaMemcpyHostToDevice, s));
            }
        }
        const int64_t nobs = dense ? dl : p->obs_dim;
        if (nobs > 0) {
            TB_CUDA(cudaMemcpyAsync(w->y.p, dense ? y + win.k0_local : y, sizeof(double) * size_t(nobs),
                                    cudaMemcpyHostToDevice, s));
            TB_CUDA(cudaMemcpyAsync(w->r.p, (dense && !r_uni) ? r + win.k0_local : r,
                                    sizeof(double) * size_t(r_uni ? 1 : nobs),
                                    cudaMemcpyHostToDevice, s));
            if (!dense)
                TB_CUDA(cudaMemcpyAsync(w->idx.p, idx, sizeof(int64_t) * size_t(nobs),
                                        cudaMemcpyHostToDevice, s));
        }
        dx = w->x.as<double>();
        dy = w->y.as<double>();
        dr = w->r.as<double>();
        didx = w->idx.as<int64_t>();
        dout = w->out.as<double>();
    }
    const JointPlan pl = joint_plan(m, m, std::max<int64_t>(dl, 1));
    TB_CUDA(w->z.reserve(sizeof(double) * md));
    TB_CUDA(w->ab.reserve(sizeof(double2) * size_t(std::max<int64_t>(dl, 1))));
    TB_CUDA(w->jpart.reserve(sizeof(double) * pl.scratch));
    double* red = nullptr;
    if (comm) {
        if (int rc = joint_red_buffer(w, nccl_api(), comm, sizeof(double) * pl.red_len, st, &red))
            return rc;
    } else {
        TB_CUDA(w->jred.reserve(sizeof(double) * pl.red_len));
        red = w->jred.as<double>();
    }
    TB_CUDA(w->jw.reserve(sizeof(double) * size_t(m) * size_t(m)));
    // N > 64: the weighted prior sums W X go through HBM ([N][d] fp64)
    double* jxbar = nullptr;
    if (m > 64) {
        TB_CUDA(w->jxbar.reserve(sizeof(double) * md));
        jxbar = w->jxbar.as<double>();
    }
    TB_CUDA(w->status.reserve(64));
    unsigned long long* dstatus = w->status.as<unsigned long long>();
    TB_CUDA(cudaMemsetAsync(dstatus, 0xff, sizeof(unsigned long long), s));

    const int64_t k0g = p->k0 + win.k0_local;
    if (dense)
        TB_CUDA(launch_obs_prep(dy, dr, nullptr, dl, p->obs_kind, k0g, dl, w->ab.as<double2>(), s,
                                r_uni ? 0 : 1, true, nullptr, 0));
    else if (int rc = select_prep(w, dy, dr, didx, on_dev ? nullptr : idx, p->obs_dim, p->obs_kind,
                                  k0g, dl, w->ab.as<double2>(), r_uni ? 0 : 1, s, st))
        return rc;
    KernelArgs a{};
    a.d_total = p->d_total;
    a.k0 = k0g;
    a.dl = dl;
    a.m = m;
    a.n_steps = p->n_steps;
    a.j_batch = m;
    const uint64_t key = stream_key(p->seed, kUseEnsfParticles);
    a.key0 = uint32_t(key);
    a.key1 = uint32_t(key >> 32);
    a.cycle_lo = uint32_t(p->cycle);
    a.obs_atan = obs_arctan(p->obs_kind) ? 1 : 0;
    a.rk = philox_round_keys(a.key0, a.key1);
    double* z = w->z.as<double>();
    TB_CUDA(launch_joint_init(a, z, s));
    ProfPair prof;
    if (g_profile.load() && on_dev) {
        prof.device = device;
        TB_CUDA(cudaEventCreate(&prof.a));
        TB_CUDA(cudaEventCreate(&prof.b));
        TB_CUDA(cudaEventRecord(prof.a, s));
    }
    const std::vector<StepTimes> grid = step_grid(p->n_steps, p->eps, p->damping_t);
    NcclApi* api = comm ? nccl_api() : nullptr;
    // the ~5 launches (+ the allreduce) of every pseudo-step are captured
    // into one CUDA graph and replayed: no per-launch host work and shorter
    // gaps on the device.  The executable graph is kept per workspace and
    // updated in place (cudaGraphExecUpdate) when only kernel arguments
    // change (the cycle, pointers).  Single-communicator-free calls only:
    // with the per-step NCCL allreduce inside, the graph measured slower
    // (2 GPUs: 18.6 vs 17.1 ms) and NCCL graph and eager collectives on one
    // communicator (an empty-window peer) do not mix.  Not on the legacy
    // default stream, which cannot be captured; TURBDA_JOINT_GRAPH=0
    // launches directly (1 GPU, config 2: 14.6 ms graph vs 15.5 ms direct).
    static const bool graph_env = [] {
        const char* e = std::getenv("TURBDA_JOINT_GRAPH");
        return !(e && std::atoi(e) == 0);
    }();
    const bool use_graph = graph_env && !comm && s != cudaStreamLegacy && s != nullptr;
    if (use_graph) TB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int step = 0; step < p->n_steps; ++step) {
        const StepTimes& q = grid[size_t(step)];
        const StepF64 c{q.alpha, q.beta2, 1.0 / (2.0 * q.beta2), q.b, q.s2, q.damp, q.sig, q.dt};
        cudaError_t ge = launch_joint_gram(a, pl, z, dx, w->jpart.as<double>(), red, s);
        if (ge == cudaSuccess && comm) {
            ncclResult_t rr = api->all_reduce(red, red, pl.red_len, ncclDouble, ncclSum,
                                              static_cast<ncclComm_t>(comm), s);
            if (rr != ncclSuccess) {
                if (use_graph) {
                    cudaGraph_t g = nullptr;
                    cudaStreamEndCapture(s, &g);
                    if (g) cudaGraphDestroy(g);
                }
                return nccl_fail(st, api, rr, "ncclAllReduce");
            }
        }
        if (ge == cudaSuccess)
            ge = launch_joint_update(a, dx, w->ab.as<double2>(), red, w->jw.as<double>(), c, step, z,
                                     dstatus, p->precision == TURBDA_FP32, s, jxbar);
        if (ge != cudaSuccess) {
            if (use_graph) {
                cudaGraph_t g = nullptr;
                cudaStreamEndCapture(s, &g);
                if (g) cudaGraphDestroy(g);
            }
            return cuda_fail(st, ge, "joint pseudo-step");
        }
    }
    if (use_graph) {
        cudaGraph_t g = nullptr;
        TB_CUDA(cudaStreamEndCapture(s, &g));
        bool updated = false;
        if (w->jgraph) {
            cudaGraphExecUpdateResultInfo info{};
            updated = cudaGraphExecUpdate(w->jgraph, g, &info) == cudaSuccess;
            if (!updated) {
                cudaGetLastError();
                cudaGraphExecDestroy(w->jgraph);
                w->jgraph = nullptr;
            }
        }
        if (!updated) {
            const cudaError_t ie = cudaGraphInstantiate(&w->jgraph, g, 0);
            if (ie != cudaSuccess) {
                cudaGraphDestroy(g);
                w->jgraph = nullptr;
                return cuda_fail(st, ie, "cudaGraphInstantiate(joint steps)");
            }
        }
        cudaGraphDestroy(g);
        TB_CUDA(cudaGraphLaunch(w->jgraph, s));
    }
    if (prof.a) {
        TB_CUDA(cudaEventRecord(prof.b, s));
        std::lock_guard<std::mutex> lk2(g_prof_mu);
        g_prof_pending.push_back(prof);
    }
    TB_CUDA(launch_relax_f64(z, dx, m, dl, p->relax_factor, dout, s));
    g_launches += 2 + 4 * uint64_t(p->n_steps);
    if (int rc = reduce_verdict_across_ranks(p, w, dstatus, s, st)) return rc;
    if (on_dev && (p->flags & TURBDA_ASYNC)) {
        TB_CUDA(ws_release(w, s, true));
        return TURBDA_OK;
    }
    TB_CUDA(cudaMemcpyAsync(w->status_host, dstatus, sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, s));
    if (!on_dev && dl > 0) {
        if (orows) {
            for (int j = 0; j < m; ++j)
                TB_CUDA(cudaMemcpyAsync(orows[j] + win.k0_local, dout + size_t(j) * size_t(dl),
                                        sizeof(double) * size_t(dl), cudaMemcpyDeviceToHost, s));
        } else {
            TB_CUDA(cudaMemcpy2DAsync(out + win.k0_local, sizeof(double) * size_t(p->d_local), dout,
                                      sizeof(double) * size_t(dl), sizeof(double) * size_t(dl),
                                      size_t(m), cudaMemcpyDeviceToHost, s));
        }
    }
    TB_CUDA(cudaStreamSynchronize(s));
    TB_CUDA(ws_release(w, s, false));
    return diverged(p, *w->status_host, st);
}

// An empty window (d_local == 0) of a state sharded over a communicator:
// nothing to analyse, but the peers' collectives must still complete, so the
// rank joins each of them with a neutral contribution - in joint mode one
// zero [G | nz | nx] buffer per pseudo-step, then the divergence verdict
// (kNoDivergence) - and reports the reduced verdict like its peers.
int join_empty_window(const turbda_ensf_params* p, int device, cudaStream_t user_stream,
                      turbda_status* st) {
    TB_CUDA(cudaSetDevice(device));
    Workspace* w = workspace(device);
    std::lock_guard<std::mutex> lk(w->mu);
    if (!(p->flags & TURBDA_SHARDED) || !w->comm || w->comm_world <= 1) return TURBDA_OK;
    if (int rc = ws_init(w, st)) return rc;
    const bool on_dev = (p->flags & TURBDA_INPUTS_ON_DEVICE) != 0;
    cudaStream_t s = user_stream ? user_stream : (on_dev ? cudaStreamLegacy : w->stream);
    TB_CUDA(ws_acquire(w, s));
    NcclApi* api = nccl_api();
    if (!api) return fail(st, TURBDA_CUDA, "libnccl.so.2 not loadable");
    const ncclComm_t comm = static_cast<ncclComm_t>(w->comm);
    if (p->score_mode == TURBDA_SCORE_JOINT) {
        const JointPlan pl = joint_plan(p->n_members, p->n_members, 1);
        double* red = nullptr;
        if (int rc = joint_red_buffer(w, api, w->comm, sizeof(double) * pl.red_len, st, &red))
            return rc;
        for (int step = 0; step < p->n_steps; ++step) {
            TB_CUDA(cudaMemsetAsync(red, 0, sizeof(double) * pl.red_len, s));
            const ncclResult_t r = api->all_reduce(red, red, pl.red_len, ncclDouble,
                                                   ncclSum, comm, s);
            if (r != ncclSuccess) return nccl_fail(st, api, r, "ncclAllReduce");
        }
    }
    TB_CUDA(w->status.reserve(64));
    unsigned long long* dstatus = w->status.as<unsigned long long>();
    TB_CUDA(cudaMemsetAsync(dstatus, 0xff, sizeof(unsigned long long), s));
    if (int rc = reduce_verdict_across_ranks(p, w, dstatus, s, st)) return rc;
    if (on_dev && (p->flags & TURBDA_ASYNC)) {
        TB_CUDA(ws_release(w, s, true));
        return TURBDA_OK;
    }
    TB_CUDA(cudaMemcpyAsync(w->status_host, dstatus, sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, s));
    TB_CUDA(cudaStreamSynchronize(s));
    TB_CUDA(ws_release(w, s, false));
    return diverged(p, *w->status_host, st);
}

int resolve_device(int requested, turbda_status* st, int* out) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        return fail(st, TURBDA_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    int dev = requested;
    if (dev < 0) TB_CUDA(cudaGetDevice(&dev));
    if (dev >= n) return fail(st, TURBDA_CUDA, "device ordinal out of range");
    *out = dev;
    return TURBDA_OK;
}

void clear(turbda_status* st) {
    if (!st) return;
    std::memset(st, 0, sizeof(*st));
    st->diverged_particle = -1;
    st->diverged_step = -1;
    st->diverged_t = std::nan("");
}

}  // namespace

extern "C" {

void turbda_ensf_params_init(turbda_ensf_params* p) {
    std::memset(p, 0, sizeof(*p));
    p->n_steps = 100;
    p->eps = 0.01;
    p->minibatch_j = 0;
    p->damping_t = 1.0;
    p->relax_factor = 1.0;
    p->seed = 7;
    p->cycle = 1;
    p->precision = TURBDA_FP32;
    p->device = -1;
    p->device_count = 1;
}

}  // extern "C"

namespace {

int analyze_impl(const turbda_ensf_params* p, const double* forecast, const double* const* frows,
                 const double* y, const double* r_diag, const int64_t* obs_idx,
                 double* analysis_out, double* const* orows, void* stream, turbda_status* st) {
    clear(st);
    if (int rc = validate(p, st)) return rc;
    const bool on_dev = (p->flags & TURBDA_INPUTS_ON_DEVICE) != 0;
    if (!on_dev) {
        if (int rc = validate_host_obs(p, r_diag, obs_idx, st)) return rc;
    }
    int dev0 = 0;
    if (int rc = resolve_device(p->device, st, &dev0)) return rc;
    int ndev = std::max(1, p->device_count);
    int avail = 0;
    cudaGetDeviceCount(&avail);
    if (dev0 + ndev > avail) return fail(st, TURBDA_CUDA, "device_count exceeds visible devices");
    if (on_dev && ndev > 1)
        return fail(st, TURBDA_CONFIG, "device_count > 1 needs host buffers");
    if (p->d_local == 0)
        return ndev == 1 ? join_empty_window(p, dev0, static_cast<cudaStream_t>(stream), st)
                         : TURBDA_OK;

    const bool joint = p->score_mode == TURBDA_SCORE_JOINT;
    if (ndev == 1) {
        if (joint) {
            // a window of a larger state shares the distances through the
            // device's communicator (turbda_comm_init)
            Workspace* w = workspace(dev0);
            const bool sharded = (p->flags & TURBDA_SHARDED) != 0;
            void* comm = (sharded && w->comm_world > 1) ? w->comm : nullptr;
            if (sharded && !comm)
                return fail(st, TURBDA_CONFIG, "TURBDA_SHARDED needs turbda_comm_init on this device");
            if (p->d_local < p->d_total && !comm)
                return fail(st, TURBDA_CONFIG,
                            "joint score mode on a window needs TURBDA_SHARDED and turbda_comm_init");
            return run_joint(p, Window{0, p->d_local}, dev0, forecast, frows, y, r_diag, obs_idx,
                             analysis_out, orows, static_cast<cudaStream_t>(stream), comm, st);
        }
        return run_slice(p, Window{0, p->d_local}, dev0, forecast, frows, y, r_diag, obs_idx,
                         analysis_out, orows, static_cast<cudaStream_t>(stream), st);
    }
    std::vector<ncclComm_t> comms;
    if (joint)
        if (int rc = clique(dev0, ndev, &comms, st)) return rc;

    // state-dimension sharding: contiguous slices aligned to the 64-coordinate tile
    std::vector<Window> wins;
    const int64_t tiles = (p->d_local + 63) / 64;
    int64_t start = 0;
    for (int g = 0; g < ndev; ++g) {
        const int64_t t_end = tiles * (g + 1) / ndev;
        const int64_t end = std::min<int64_t>(p->d_local, t_end * 64);
        wins.push_back(Window{start, end - start});
        start = end;
    }
    std::vector<turbda_status> sts(static_cast<size_t>(ndev));
    std::vector<int> rcs(static_cast<size_t>(ndev), 0);
    std::vector<std::thread> th;
    for (int g = 0; g < ndev; ++g) {
        clear(&sts[size_t(g)]);
        th.emplace_back([&, g] {
            rcs[size_t(g)] =
                joint ? run_joint(p, wins[size_t(g)], dev0 + g, forecast, frows, y, r_diag, obs_idx,
                                  analysis_out, orows, nullptr, comms[size_t(g)], &sts[size_t(g)])
                      : run_slice(p, wins[size_t(g)], dev0 + g, forecast, frows, y, r_diag,
                                  obs_idx, analysis_out, orows, nullptr, &sts[size_t(g)]);
        });
    }
    for (auto& t : th) t.join();
    // non-divergence failures first (first device wins), then the lowest
    // diverging particle / earliest step across shards
    for (int g = 0; g < ndev; ++g)
        if (rcs[size_t(g)] != TURBDA_OK && rcs[size_t(g)] != TURBDA_DIVERGED) {
            if (st) *st = sts[size_t(g)];
            return rcs[size_t(g)];
        }
    int best = -1;
    for (int g = 0; g < ndev; ++g) {
        if (rcs[size_t(g)] != TURBDA_DIVERGED) continue;
        const turbda_status& q = sts[size_t(g)];
        if (best < 0 || q.diverged_particle < sts[size_t(best)].diverged_particle ||
            (q.diverged_particle == sts[size_t(best)].diverged_particle &&
             q.diverged_step < sts[size_t(best)].diverged_step))
            best = g;
    }
    if (best >= 0) {
        if (st) *st = sts[size_t(best)];
        return TURBDA_DIVERGED;
    }
    return TURBDA_OK;
}

}  // namespace

extern "C" {

int turbda_ensf_analyze(const turbda_ensf_params* p, const double* forecast, const double* y,
                        const double* r_diag, const int64_t* obs_idx, double* analysis_out,
                        void* stream, turbda_status* st) {
    return analyze_impl(p, forecast, nullptr, y, r_diag, obs_idx, analysis_out, nullptr, stream,
                        st);
}

int turbda_ensf_analyze_rows(const turbda_ensf_params* p, const double* const* forecast_rows,
                             const double* y, const double* r_diag, const int64_t* obs_idx,
                             double* const* analysis_rows, turbda_status* st) {
    if (p && (p->flags & TURBDA_INPUTS_ON_DEVICE)) {
        clear(st);
        return fail(st, TURBDA_CONFIG, "turbda_ensf_analyze_rows takes host rows");
    }
    return analyze_impl(p, nullptr, forecast_rows, y, r_diag, obs_idx, nullptr, analysis_rows,
                        nullptr, st);
}

int turbda_ensf_check(int device, const turbda_ensf_params* p, turbda_status* st) {
    clear(st);
    int dev = 0;
    if (int rc = resolve_device(device, st, &dev)) return rc;
    TB_CUDA(cudaSetDevice(dev));
    Workspace* w = workspace(dev);
    std::lock_guard<std::mutex> lk(w->mu);
    if (!w->status.p) return TURBDA_OK;
    unsigned long long word = kNoDivergence;
    TB_CUDA(cudaMemcpy(&word, w->status.p, sizeof(word), cudaMemcpyDeviceToHost));
    return diverged(p, word, st);
}

int turbda_relax_spread(const double* analysis, const double* forecast, int32_t m, int64_t d,
                        double factor, double* out, int32_t device, uint32_t flags, void* stream,
                        turbda_status* st) {
    clear(st);
    if (m < 1) return fail(st, TURBDA_DIMENSION, "ensemble: empty");
    int dev = 0;
    if (int rc = resolve_device(device, st, &dev)) return rc;
    TB_CUDA(cudaSetDevice(dev));
    Workspace* w = workspace(dev);
    std::lock_guard<std::mutex> lk(w->mu);
    if (int rc = ws_init(w, st)) return rc;
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : w->stream;
    TB_CUDA(ws_acquire(w, s));
    const size_t md = size_t(m) * size_t(d);
    if (flags & TURBDA_INPUTS_ON_DEVICE) {
        TB_CUDA(launch_relax_f64(analysis, forecast, m, d, factor, out, s));
        ++g_launches;
        TB_CUDA(cudaStreamSynchronize(s));
        TB_CUDA(ws_release(w, s, false));
        return TURBDA_OK;
    }
    TB_CUDA(w->x.reserve(sizeof(double) * std::max<size_t>(md, 1)));
    TB_CUDA(w->z.reserve(sizeof(double) * std::max<size_t>(md, 1)));
    TB_CUDA(w->out.reserve(sizeof(double) * std::max<size_t>(md, 1)));
    TB_CUDA(cudaMemcpyAsync(w->z.p, analysis, sizeof(double) * md, cudaMemcpyHostToDevice, s));
    TB_CUDA(cudaMemcpyAsync(w->x.p, forecast, sizeof(double) * md, cudaMemcpyHostToDevice, s));
    TB_CUDA(launch_relax_f64(w->z.as<double>(), w->x.as<double>(), m, d, factor,
                             w->out.as<double>(), s));
    ++g_launches;
    TB_CUDA(cudaMemcpyAsync(out, w->out.p, sizeof(double) * md, cudaMemcpyDeviceToHost, s));
    TB_CUDA(cudaStreamSynchronize(s));
    TB_CUDA(ws_release(w, s, false));
    return TURBDA_OK;
}

int turbda_score(const double* z, int64_t d, double t, const double* forecast, int32_t m,
                 const int32_t* batch, int32_t n_batch, double eps, const double* y,
                 const double* r_diag, const int64_t* obs_idx, int64_t obs_dim, int32_t obs_kind,
                 double damping_t, double* out, int32_t device, turbda_status* st) {
    clear(st);
    // check_score_time, proj/src/ensf.cpp:15-19
    if (t < eps) return fail(st, TURBDA_DOMAIN, "prior_score: t below eps (beta -> 0)");
    if (t > 1.0) return fail(st, TURBDA_DOMAIN, "prior_score: t > 1");
    if (m < 1) return fail(st, TURBDA_DIMENSION, "ensemble: empty");
    const int nb = (batch && n_batch > 0) ? n_batch : m;
    if (batch)
        for (int q = 0; q < n_batch; ++q)
            if (batch[q] < 0 || batch[q] >= m)
                return fail(st, TURBDA_DIMENSION, "prior_score: batch index out of range");
    if (y) {
        if (obs_kind < 0 || obs_kind > 3)
            return fail(st, TURBDA_CONFIG, "observation: unsupported operator kind");
        if ((obs_dense(obs_kind) && obs_dim != d) || obs_dim < 0)
            return fail(st, TURBDA_DIMENSION, "likelihood_score: dimension mismatch");
        for (int64_t q = 0; q < obs_dim; ++q)
            if (!(r_diag[q] > 0.0)) return fail(st, TURBDA_CONFIG, "observation: r_diag > 0");
        if (!obs_dense(obs_kind))
            for (int64_t q = 0; q < obs_dim; ++q)
                if (obs_idx[q] < 0 || obs_idx[q] >= d)
                    return fail(st, TURBDA_DIMENSION, "observation: index outside the state");
    }
    int dev = 0;
    if (int rc = resolve_device(device, st, &dev)) return rc;
    TB_CUDA(cudaSetDevice(dev));
    Workspace* w = workspace(dev);
    std::lock_guard<std::mutex> lk(w->mu);
    if (int rc = ws_init(w, st)) return rc;
    cudaStream_t s = w->stream;
    TB_CUDA(ws_acquire(w, s));
    const size_t md = size_t(m) * size_t(d);
    const size_t d1 = size_t(std::max<int64_t>(d, 1));
    TB_CUDA(w->x.reserve(sizeof(double) * std::max<size_t>(md, 1)));
    TB_CUDA(w->z.reserve(sizeof(double) * d1));
    TB_CUDA(w->out.reserve(sizeof(double) * d1));
    TB_CUDA(w->batches.reserve(sizeof(int32_t) * size_t(std::max(nb, 1))));
    w->batch_key.clear();
    TB_CUDA(cudaMemcpyAsync(w->x.p, forecast, sizeof(double) * md, cudaMemcpyHostToDevice, s));
    TB_CUDA(cudaMemcpyAsync(w->z.p, z, sizeof(double) * size_t(d), cudaMemcpyHostToDevice, s));
    if (batch)
        TB_CUDA(cudaMemcpyAsync(w->batches.p, batch, sizeof(int32_t) * size_t(nb),
                                cudaMemcpyHostToDevice, s));
    const double2* dab = nullptr;
    double damp = 0.0;
    if (y) {
        const size_t nb2 = size_t(std::max<int64_t>(obs_dim, 1));
        TB_CUDA(w->y.reserve(sizeof(double) * nb2));
        TB_CUDA(w->r.reserve(sizeof(double) * nb2));
        TB_CUDA(w->idx.reserve(sizeof(int64_t) * nb2));
        TB_CUDA(w->ab.reserve(sizeof(double2) * d1));
        if (obs_dim > 0) {
            TB_CUDA(cudaMemcpyAsync(w->y.p, y, sizeof(double) * size_t(obs_dim), cudaMemcpyHostToDevice, s));
            TB_CUDA(cudaMemcpyAsync(w->r.p, r_diag, sizeof(double) * size_t(obs_dim), cudaMemcpyHostToDevice, s));
            if (!obs_dense(obs_kind))
                TB_CUDA(cudaMemcpyAsync(w->idx.p, obs_idx, sizeof(int64_t) * size_t(obs_dim),
                                        cudaMemcpyHostToDevice, s));
        }
        if (obs_dense(obs_kind))
            TB_CUDA(launch_obs_prep(w->y.as<double>(), w->r.as<double>(), nullptr, d, obs_kind, 0, d,
                                    w->ab.as<double2>(), s, 1, true, nullptr, 0));
        else if (int rc = select_prep(w, w->y.as<double>(), w->r.as<double>(), w->idx.as<int64_t>(),
                                      obs_idx, obs_dim, obs_kind, 0, d, w->ab.as<double2>(), 1, s, st))
            return rc;
        dab = w->ab.as<double2>();
        damp = damping_t - t;
    }
    // NoiseSchedule::alpha / beta2, include/turbda/ensf.hpp:15-20
    TB_CUDA(launch_score_f64(w->z.as<double>(), w->x.as<double>(), m, d,
                             batch ? w->batches.as<int32_t>() : nullptr, nb, 1.0 - t, t, dab, damp,
                             obs_arctan(obs_kind) ? 1 : 0, w->out.as<double>(), s));
    ++g_launches;
    TB_CUDA(cudaMemcpyAsync(out, w->out.p, sizeof(double) * size_t(d), cudaMemcpyDeviceToHost, s));
    TB_CUDA(cudaStreamSynchronize(s));
    TB_CUDA(ws_release(w, s, false));
    return TURBDA_OK;
}

int turbda_likelihood_score(const double* z, int64_t d, const double* y, const double* r_diag,
                            const int64_t* obs_idx, int64_t obs_dim, int32_t obs_kind, double* out,
                            int32_t device, turbda_status* st) {
    clear(st);
    if (obs_kind < 0 || obs_kind > 3) return fail(st, TURBDA_CONFIG, "observation: unsupported operator kind");
    if (d < 0 || obs_dim < 0 || (obs_dense(obs_kind) && obs_dim != d))
        return fail(st, TURBDA_DIMENSION, "likelihood_score: dimension mismatch");
    for (int64_t q = 0; q < obs_dim; ++q)
        if (!(r_diag[q] > 0.0)) return fail(st, TURBDA_CONFIG, "observation: r_diag > 0");
    if (!obs_dense(obs_kind))
        for (int64_t q = 0; q < obs_dim; ++q)
            if (obs_idx[q] < 0 || obs_idx[q] >= d)
                return fail(st, TURBDA_DIMENSION, "observation: index outside the state");
    int dev = 0;
    if (int rc = resolve_device(device, st, &dev)) return rc;
    TB_CUDA(cudaSetDevice(dev));
    Workspace* w = workspace(dev);
    std::lock_guard<std::mutex> lk(w->mu);
    if (int rc = ws_init(w, st)) return rc;
    cudaStream_t s = w->stream;
    TB_CUDA(ws_acquire(w, s));
    const size_t d1 = size_t(std::max<int64_t>(d, 1)), nb = size_t(std::max<int64_t>(obs_dim, 1));
    TB_CUDA(w->z.reserve(sizeof(double) * d1));
    TB_CUDA(w->out.reserve(sizeof(double) * d1));
    TB_CUDA(w->y.reserve(sizeof(double) * nb));
    TB_CUDA(w->r.reserve(sizeof(double) * nb));
    TB_CUDA(w->idx.reserve(sizeof(int64_t) * nb));
    TB_CUDA(w->ab.reserve(sizeof(double2) * d1));
    TB_CUDA(cudaMemcpyAsync(w->z.p, z, sizeof(double) * size_t(d), cudaMemcpyHostToDevice, s));
    if (obs_dim > 0) {
        TB_CUDA(cudaMemcpyAsync(w->y.p, y, sizeof(double) * size_t(obs_dim), cudaMemcpyHostToDevice, s));
        TB_CUDA(cudaMemcpyAsync(w->r.p, r_diag, sizeof(double) * size_t(obs_dim), cudaMemcpyHostToDevice, s));
        if (!obs_dense(obs_kind))
            TB_CUDA(cudaMemcpyAsync(w->idx.p, obs_idx, sizeof(int64_t) * size_t(obs_dim),
                                    cudaMemcpyHostToDevice, s));
    }
    if (obs_dense(obs_kind))
        TB_CUDA(launch_obs_prep(w->y.as<double>(), w->r.as<double>(), nullptr, d, obs_kind, 0, d,
                                w->ab.as<double2>(), s, 1, true, nullptr, 0));
    else if (int rc = select_prep(w, w->y.as<double>(), w->r.as<double>(), w->idx.as<int64_t>(),
                                  obs_idx, obs_dim, obs_kind, 0, d, w->ab.as<double2>(), 1, s, st))
        return rc;
    TB_CUDA(launch_likelihood(w->z.as<double>(), d, w->ab.as<double2>(), obs_arctan(obs_kind) ? 1 : 0,
                              w->out.as<double>(), s));
    TB_CUDA(cudaMemcpyAsync(out, w->out.p, sizeof(double) * size_t(d), cudaMemcpyDeviceToHost, s));
    TB_CUDA(cudaStreamSynchronize(s));
    TB_CUDA(ws_release(w, s, false));
    return TURBDA_OK;
}

int turbda_reverse_sde_step(double* particles, int32_t n, int64_t d, double t, double dt_pseudo,
                            const double* scores, const double* noise, int32_t device,
                            turbda_status* st) {
    clear(st);
    if (!(dt_pseudo > 0.0)) return fail(st, TURBDA_CONFIG, "reverse_sde_step: dt_pseudo > 0");
    if (n < 0 || d < 0) return fail(st, TURBDA_DIMENSION, "reverse_sde_step: dimension mismatch");
    int dev = 0;
    if (int rc = resolve_device(device, st, &dev)) return rc;
    TB_CUDA(cudaSetDevice(dev));
    Workspace* w = workspace(dev);
    std::lock_guard<std::mutex> lk(w->mu);
    if (int rc = ws_init(w, st)) return rc;
    cudaStream_t s = w->stream;
    TB_CUDA(ws_acquire(w, s));
    const size_t nd = size_t(n) * size_t(d), nd1 = std::max<size_t>(nd, 1);
    TB_CUDA(w->x.reserve(sizeof(double) * nd1));
    TB_CUDA(w->z.reserve(sizeof(double) * nd1));
    TB_CUDA(w->out.reserve(sizeof(double) * nd1));
    TB_CUDA(w->status.reserve(64));
    unsigned int* bad = reinterpret_cast<unsigned int*>(w->status.as<unsigned char>() + 32);
    TB_CUDA(cudaMemsetAsync(bad, 0, sizeof(unsigned int), s));
    TB_CUDA(cudaMemcpyAsync(w->z.p, particles, sizeof(double) * nd, cudaMemcpyHostToDevice, s));
    TB_CUDA(cudaMemcpyAsync(w->x.p, scores, sizeof(double) * nd, cudaMemcpyHostToDevice, s));
    TB_CUDA(cudaMemcpyAsync(w->out.p, noise, sizeof(double) * nd, cudaMemcpyHostToDevice, s));
    // NoiseSchedule, proj/include/turbda/ensf.hpp:15-20
    const double b = -1.0 / (1.0 - t);
    const double s2 = 1.0 + 2.0 * t / (1.0 - t);
    const double sig = std::sqrt(s2 * dt_pseudo);
    TB_CUDA(launch_sde_step(w->z.as<double>(), int64_t(nd), w->x.as<double>(), w->out.as<double>(),
                            b, s2, dt_pseudo, sig, bad, s));
    unsigned int h_bad = 0;
    TB_CUDA(cudaMemcpyAsync(particles, w->z.p, sizeof(double) * nd, cudaMemcpyDeviceToHost, s));
    TB_CUDA(cudaMemcpyAsync(&h_bad, bad, sizeof(unsigned int), cudaMemcpyDeviceToHost, s));
    TB_CUDA(cudaStreamSynchronize(s));
    TB_CUDA(ws_release(w, s, false));
    if (h_bad) {
        if (st) st->diverged_t = t;
        return fail(st, TURBDA_DIVERGED, "reverse SDE diverged at pseudo-time t=" + std::to_string(t));
    }
    return TURBDA_OK;
}

int turbda_diag(const double* members, int32_t m, int64_t d, const double* truth, double* out,
                int32_t device, uint32_t flags, void* stream, turbda_status* st) {
    clear(st);
    if (m < 1) return fail(st, TURBDA_DIMENSION, "ensemble: empty");
    int dev = 0;
    if (int rc = resolve_device(device, st, &dev)) return rc;
    TB_CUDA(cudaSetDevice(dev));
    Workspace* w = workspace(dev);
    std::lock_guard<std::mutex> lk(w->mu);
    if (int rc = ws_init(w, st)) return rc;
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : w->stream;
    TB_CUDA(ws_acquire(w, s));
    TB_CUDA(w->diag.reserve(sizeof(double) * diag_scratch_doubles()));
    double* dsum = w->diag.as<double>();
    const size_t md = size_t(m) * size_t(d);
    const double* dx = members;
    const double* dt = truth;
    if (!(flags & TURBDA_INPUTS_ON_DEVICE)) {
        TB_CUDA(w->x.reserve(sizeof(double) * std::max<size_t>(md, 1)));
        TB_CUDA(cudaMemcpyAsync(w->x.p, members, sizeof(double) * md, cudaMemcpyHostToDevice, s));
        dx = w->x.as<double>();
        if (truth) {
            TB_CUDA(w->y.reserve(sizeof(double) * size_t(std::max<int64_t>(d, 1))));
            TB_CUDA(cudaMemcpyAsync(w->y.p, truth, sizeof(double) * size_t(d), cudaMemcpyHostToDevice, s));
            dt = w->y.as<double>();
        }
    }
    TB_CUDA(launch_diag(dx, m, d, dt, dsum, s));
    if (flags & TURBDA_SHARDED) {
        // this rank's shard of a state split over the communicator's ranks
        if (!w->comm || w->comm_world <= 1)
            return fail(st, TURBDA_CONFIG, "TURBDA_SHARDED needs turbda_comm_init on this device");
        NcclApi* api = nccl_api();
        if (!api) return fail(st, TURBDA_CUDA, "libnccl.so.2 not loadable");
        const ncclResult_t r = api->all_reduce(dsum, dsum, 2, ncclDouble, ncclSum,
                                               static_cast<ncclComm_t>(w->comm), s);
        if (r != ncclSuccess) return nccl_fail(st, api, r, "ncclAllReduce(diag)");
    }
    TB_CUDA(cudaMemcpyAsync(out, dsum, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    TB_CUDA(cudaStreamSynchronize(s));
    TB_CUDA(ws_release(w, s, false));
    return TURBDA_OK;
}

int turbda_comm_unique_id(void* id128, turbda_status* st) {
    clear(st);
    NcclApi* api = nccl_api();
    if (!api) return fail(st, TURBDA_CUDA, "libnccl.so.2 not loadable");
    ncclUniqueId id;
    ncclResult_t r = api->get_unique_id(&id);
    if (r != ncclSuccess) return nccl_fail(st, api, r, "ncclGetUniqueId");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id128, &id, sizeof id);
    return TURBDA_OK;
}

int turbda_comm_init(int32_t device, int32_t rank, int32_t world, const void* id128,
                     turbda_status* st) {
    clear(st);
    int dev = 0;
    if (int rc = resolve_device(device, st, &dev)) return rc;
    NcclApi* api = nccl_api();
    if (!api) return fail(st, TURBDA_CUDA, "libnccl.so.2 not loadable");
    TB_CUDA(cudaSetDevice(dev));
    Workspace* w = workspace(dev);
    std::lock_guard<std::mutex> lk(w->mu);
    if (w->comm) {
        release_symmetric(w, api);
        api->comm_destroy(static_cast<ncclComm_t>(w->comm));
        w->comm = nullptr;
    }
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    ncclComm_t comm;
    ncclResult_t r = api->comm_init_rank(&comm, world, id, rank);
    if (r != ncclSuccess) return nccl_fail(st, api, r, "ncclCommInitRank");
    w->comm = comm;
    w->comm_world = world;
    return TURBDA_OK;
}

int turbda_comm_destroy(int32_t device) {
    if (device < 0 || cudaSetDevice(device) != cudaSuccess) return TURBDA_CUDA;
    Workspace* w = workspace(device);
    std::lock_guard<std::mutex> lk(w->mu);
    NcclApi* api = nccl_api();
    if (w->comm && api) {
        release_symmetric(w, api);
        api->comm_destroy(static_cast<ncclComm_t>(w->comm));
    }
    w->comm = nullptr;
    w->comm_world = 1;
    return TURBDA_OK;
}

int turbda_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int turbda_abi_version(void) { return TURBDA_B200_ABI_VERSION; }

const char* turbda_build_arch(void) { return "sm_100a"; }

uint64_t turbda_launch_count(void) { return g_launches.load(); }

void turbda_profile_enable(int on) {
    g_profile.store(on ? 1 : 0);
}

int turbda_profile_read(double* kernel_ms, uint64_t* launches) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (ProfPair& q : g_prof_pending) {
        cudaSetDevice(q.device);
        float ms = 0.f;
        if (cudaEventSynchronize(q.b) == cudaSuccess &&
            cudaEventElapsedTime(&ms, q.a, q.b) == cudaSuccess) {
            g_prof_ms += ms;
            ++g_prof_n;
        }
        cudaEventDestroy(q.a);
        cudaEventDestroy(q.b);
    }
    g_prof_pending.clear();
    if (kernel_ms) *kernel_ms = g_prof_ms;
    if (launches) *launches = g_prof_n;
    g_prof_ms = 0.0;
    g_prof_n = 0;
    return TURBDA_OK;
}

}  // extern "C"
