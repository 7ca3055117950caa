/*
 * turbda_b200.h - C-ABI of the B200-native EnSF analysis step.
 *
 * This is the drop-in boundary: plain pointers, sizes and PODs, no C++ or
 * torch types.  The C++ API in include/turbda/ (turbda::analyze & co., the
 * reference's own signatures) and the Python module
 * paper_2407_12168_b200._core are thin hosts above it.
 *
 * Reference interfaces replaced (all paths under /root/reference/proj):
 *   turbda_ensf_analyze   <- turbda::analyze          include/turbda/ensf.hpp:79-81,
 *                                                    src/ensf.cpp:132-223
 *                            (and its callers run_experiment src/osse.cpp:234-235,
 *                             _core.ensf_analyze python/bindings.cpp:140-155)
 *   turbda_relax_spread   <- turbda::relax_spread     include/turbda/ensf.hpp:85-86,
 *                                                    src/ensf.cpp:225-258
 *   turbda_score          <- turbda::prior_score / posterior_score
 *   turbda_likelihood_score <- turbda::likelihood_score  src/ensf.cpp:84-94
 *   turbda_reverse_sde_step <- turbda::reverse_sde_step  src/ensf.cpp:108-130
 *                                                    include/turbda/ensf.hpp:52-70,
 *                                                    src/ensf.cpp:68-82,96-106
 *   turbda_diag           <- turbda::rmse / spread    include/turbda/ensemble.hpp:32-38,
 *                                                    src/ensemble.cpp:18-43
 *   turbda_letkf_analyze  <- turbda::letkf_analyze    include/turbda/letkf.hpp:48-52,
 *                                                    src/letkf.cpp:57-175
 *   turbda_rtps_inflate   <- turbda::rtps_inflate     include/turbda/letkf.hpp:54-56,
 *                                                    src/letkf.cpp:177-207
 *   turbda_gaspari_cohn   <- turbda::gaspari_cohn     src/letkf.cpp:10-18
 *   turbda_snapshot_*     <- turbda::write_snapshot / read_snapshot
 *                                                    include/turbda/snapshot.hpp:12-23,
 *                                                    src/snapshot.cpp:12-63
 *
 * Error convention: every entry point returns a turbda_code and fills
 * *status (when non-NULL).  The C++ host maps TURBDA_CONFIG -> ConfigError,
 * TURBDA_DIMENSION -> DimensionError, TURBDA_DIVERGED ->
 * SamplerDivergedError(diverged_t), TURBDA_DOMAIN -> std::domain_error, as the
 * reference throws them (include/turbda/errors.hpp:9-57).
 *
 * There is no CPU fallback: without a CUDA device every compute entry point
 * returns TURBDA_CUDA.
 */
#ifndef TURBDA_B200_H
#define TURBDA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TURBDA_B200_ABI_VERSION 1

#if defined(__GNUC__)
#define TURBDA_API __attribute__((visibility("default")))
#else
#define TURBDA_API
#endif

typedef enum turbda_code {
    TURBDA_OK = 0,
    TURBDA_CONFIG = 1,     /* ConfigError                                  */
    TURBDA_DIMENSION = 2,  /* DimensionError                               */
    TURBDA_DIVERGED = 3,   /* SamplerDivergedError(pseudo_time)            */
    TURBDA_DOMAIN = 4,     /* std::domain_error (score time outside [eps,1]) */
    TURBDA_CUDA = 5,       /* no device / CUDA runtime failure             */
    TURBDA_INTERNAL = 6,
    TURBDA_BLOWUP = 7,     /* BlowupError(time, member): SQG state non-finite */
    TURBDA_ABORTED = 8,    /* RunAbortedError(cycle): status.diverged_step  */
    TURBDA_SINGULAR = 9,   /* SingularAnalysisError(ix, iy): LETKF, grid point */
                           /* in status.diverged_particle / diverged_step    */
    TURBDA_IO = 10         /* IoError (snapshot files)                      */
} turbda_code;

typedef enum turbda_precision {
    TURBDA_FP32 = 0,  /* fast path: fp32 registers, MUFU ex2, packed FFMA2 */
    TURBDA_FP64 = 1   /* faithful path: the reference's fp64 arithmetic    */
} turbda_precision;

/* flags */
#define TURBDA_INPUTS_ON_DEVICE 0x1u /* every array pointer is a device pointer  */
#define TURBDA_ASYNC 0x2u            /* device mode only: do not synchronize;     */
                                     /* fetch the divergence verdict later with   */
                                     /* turbda_ensf_check().  A later call on     */
                                     /* another stream of the same device waits   */
                                     /* for it (the scratch is per device)        */
#define TURBDA_R_UNIFORM 0x4u        /* r_diag points to ONE error variance used  */
                                     /* for every observation (the scalar `r` of  */
                                     /* the Python binding, bindings/python/      */
                                     /* core.cpp); host or device pointer as the  */
                                     /* other arrays                              */
#define TURBDA_SHARDED 0x8u          /* the call is this rank's window / shard of  */
                                     /* a state split over the ranks of           */
                                     /* turbda_comm_init, and every rank makes    */
                                     /* the same call: the analysis min-reduces   */
                                     /* its divergence verdict (the joint mode    */
                                     /* also allreduces its per-step distances),  */
                                     /* turbda_diag its partial sums.  Without    */
                                     /* it a call is local even when a            */
                                     /* communicator exists                       */

typedef struct turbda_status {
    int32_t code;              /* turbda_code                                   */
    int32_t diverged_particle; /* lowest particle index that went non-finite    */
    int32_t diverged_step;     /* its first non-finite pseudo-time step         */
    int32_t reserved;
    double diverged_t;         /* pseudo-time of that step (t_ev)               */
    char msg[256];
} turbda_status;

/*
 * One EnSF analysis (turbda::analyze) on the coordinate window
 * [k0, k0 + d_local) of a state of global dimension d_total.  A whole-state
 * call has k0 = 0, d_local = d_total.  Because the reference's prior score is
 * componentwise, every window reproduces exactly the coordinates a
 * whole-state call would produce (the particle noise is keyed by the global
 * coordinate), which is how the state dimension shards across GPUs.
 */
typedef struct turbda_ensf_params {
    int64_t d_total;      /* global state dimension                              */
    int64_t k0;           /* first global coordinate of the window               */
    int64_t d_local;      /* coordinates in the window                           */
    int64_t obs_dim;      /* entries of y / r_diag (/ obs_idx)                   */
    int32_t n_members;    /* M: forecast members == analysis particles           */
    int32_t n_steps;      /* EnsfConfig::n_steps (>= 10)                          */
    int32_t minibatch_j;  /* EnsfConfig::minibatch_j (0 = all members)           */
    int32_t obs_kind;     /* 0 identity (obs_dim == d_local), 1 index_selection, */
                          /* 2 arctan of the full state, 3 arctan of selected   */
                          /* indices (2/3: h(x) = atan(x), a north-star          */
                          /* extension without a reference implementation)      */
    double eps;           /* EnsfConfig::eps in (0, 1)                            */
    double damping_t;     /* EnsfConfig::damping_t: h(t) = damping_t - t          */
    double relax_factor;  /* EnsfConfig::relax_factor in [0, 1]                   */
    uint64_t seed;
    uint64_t cycle;
    int32_t precision;    /* turbda_precision                                    */
    int32_t device;       /* first CUDA device; -1 = current device              */
    int32_t device_count; /* >1 (host buffers only): split the window over       */
                          /* devices device .. device + device_count - 1         */
    uint32_t flags;       /* TURBDA_INPUTS_ON_DEVICE | TURBDA_ASYNC |            */
                          /* TURBDA_R_UNIFORM                                     */
    int32_t score_mode;   /* TURBDA_SCORE_COMPONENTWISE (the reference) or        */
                          /* TURBDA_SCORE_JOINT (north-star extension, fp64)      */
    int32_t reserved;
} turbda_ensf_params;

/* score_mode */
#define TURBDA_SCORE_COMPONENTWISE 0 /* proj/src/ensf.cpp:27-64: a softmax per coordinate */
#define TURBDA_SCORE_JOINT 1         /* paper Eq. 15-16: one softmax per particle over   */
                                     /* full-state distances; per pseudo-step one Gram   */
                                     /* pass and, with a communicator, ONE allreduce of  */
                                     /* the N x N (+2N) partial distances. Distances and */
                                     /* the update in fp64; TURBDA_FP32 only switches    */
                                     /* the particle noise to the fp32 Box-Muller. No    */
                                     /* minibatches. Parity unpinned (no reference).     */

/* Fills *p with the reference defaults (include/turbda/ensf.hpp:22-27):
 * n_steps 100, eps 0.01, minibatch 0, damping_t 1, relax 1, fp32, device -1. */
TURBDA_API void turbda_ensf_params_init(turbda_ensf_params* p);

/*
 * forecast     [n_members][d_local] row-major fp64 (member-major, like the
 *              reference's Ensemble::members and the Python (M, d) array)
 * y, r_diag    [obs_dim] fp64
 * obs_idx      [obs_dim] global state indices (index_selection); NULL for identity
 * analysis_out [n_members][d_local] fp64
 * stream       cudaStream_t to run on; NULL = the legacy default stream in
 *              device mode, an internal per-device stream in host mode
 */
TURBDA_API int turbda_ensf_analyze(const turbda_ensf_params* p, const double* forecast, const double* y,
                        const double* r_diag, const int64_t* obs_idx, double* analysis_out,
                        void* stream, turbda_status* status);

/* Same analysis with the members kept as separate host rows (the
 * reference's Ensemble::members layout): forecast_rows[j] and
 * analysis_rows[j] point at d_local doubles each.  Host buffers only; saves
 * the caller packing a contiguous [M][d] copy. */
TURBDA_API int turbda_ensf_analyze_rows(const turbda_ensf_params* p, const double* const* forecast_rows,
                             const double* y, const double* r_diag, const int64_t* obs_idx,
                             double* const* analysis_rows, turbda_status* status);

/* After a TURBDA_ASYNC call and a synchronize of its stream: verdict of the
 * most recent analysis on `device`. */
TURBDA_API int turbda_ensf_check(int device, const turbda_ensf_params* p, turbda_status* status);

/* relax_spread on the device; host or device buffers per `flags`. */
TURBDA_API int turbda_relax_spread(const double* analysis, const double* forecast, int32_t n_members,
                        int64_t d, double factor, double* out, int32_t device, uint32_t flags,
                        void* stream, turbda_status* status);

/*
 * Componentwise prior score at pseudo-time t (prior_score), plus the damped
 * likelihood when y != NULL (posterior_score), fp64, host buffers.
 * batch: member indices or NULL (all members).
 */
TURBDA_API int turbda_score(const double* z, int64_t d, double t, const double* forecast, int32_t n_members,
                 const int32_t* batch, int32_t n_batch, double eps, const double* y,
                 const double* r_diag, const int64_t* obs_idx, int64_t obs_dim, int32_t obs_kind,
                 double damping_t, double* out, int32_t device, turbda_status* status);

/* likelihood_score (proj/src/ensf.cpp:84-94): H'^T R^-1 (y - h(z)) for the
 * identity / index-selection (and arctan) operators, duplicates adding as
 * adjoint_scatter does; host buffers, computed on the device. */
TURBDA_API int turbda_likelihood_score(const double* z, int64_t d, const double* y,
                            const double* r_diag, const int64_t* obs_idx, int64_t obs_dim,
                            int32_t obs_kind, double* out, int32_t device,
                            turbda_status* status);

/* reverse_sde_step (proj/src/ensf.cpp:108-130): one Euler-Maruyama step of
 * n particles [n][d] in place, z += -(b z - sigma^2 score) dt + sqrt(sigma^2
 * dt) noise at pseudo-time t; host buffers, computed on the device.  A
 * non-finite result returns TURBDA_DIVERGED (SamplerDivergedError(t)). */
TURBDA_API int turbda_reverse_sde_step(double* particles, int32_t n, int64_t d, double t,
                            double dt_pseudo, const double* scores, const double* noise,
                            int32_t device, turbda_status* status);

/* out[0] = sum_k (mean_k - truth_k)^2 (0 when truth == NULL),
 * out[1] = sum_{j,k} (x_jk - mean_k)^2.  members / truth are host or device
 * buffers per flags; out is always a host double[2].  The sums are taken in
 * a fixed order (fixed grid, two-stage reduction): bitwise reproducible.
 * With TURBDA_SHARDED (and a communicator on `device`) they are summed over
 * the communicator's ranks; without it the call is local even when a
 * communicator exists. */
TURBDA_API int turbda_diag(const double* members, int32_t n_members, int64_t d, const double* truth,
                double* out, int32_t device, uint32_t flags, void* stream,
                turbda_status* status);

/*
 * NCCL communicator for state-dimension sharding across processes (one rank
 * per GPU).  Calls flagged TURBDA_SHARDED use it: the joint score mode
 * exchanges the per-step distances through it; the componentwise mode needs
 * none, but a sharded window min-reduces its divergence verdict, so every
 * rank reports the unsharded run's SamplerDivergedError, and turbda_diag
 * sums its partials over the ranks.  A rank whose window is empty
 * (d_local == 0) still joins every collective of the call, so its peers
 * never wait on it.  NCCL is loaded on first use
 * (dlopen("libnccl.so.2"), the copy torch already loaded when present).
 *   rank 0: turbda_comm_unique_id(id) -> broadcast the 128 bytes -> every
 *   rank: turbda_comm_init(device, rank, world, id).
 */
TURBDA_API int turbda_comm_unique_id(void* id128, turbda_status* status);
TURBDA_API int turbda_comm_init(int32_t device, int32_t rank, int32_t world, const void* id128,
                     turbda_status* status);
TURBDA_API int turbda_comm_destroy(int32_t device);

/* ---------------------------------------------------------------------------
 * Forecast model and cycle driver (the callers either side of the analysis,
 * SURVEY.md 8(f)): a batched GPU two-boundary SQG model (fp64, cuFFT)
 * replacing SqgStepper / nature_run (proj/src/forecast.cpp:14-75,
 * proj/src/osse.cpp:101-135), and the GPU-resident twin experiment
 * run_experiment (proj/src/osse.cpp:182-253).
 * ------------------------------------------------------------------------- */
typedef struct turbda_sqg_params { /* GridSpec + SqgParams (nz = 2)         */
    int32_t nx, ny;
    double lx, ly, h;
    double f, n, u0;
    int32_t hyper_order, reserved;
    double hyper_efold, dt, drag_tau;
} turbda_sqg_params;

/* reference defaults: 64 x 64, lx = ly = 20 pi, h 0.3, f 1, N 10, u0 0.1,
 * order 4, e-fold 5 h, dt 0.25 h, drag 200 h */
TURBDA_API void turbda_sqg_params_init(turbda_sqg_params* p);
/* a model advancing `batch` states [batch][2][ny][nx] together */
TURBDA_API int turbda_sqg_create(const turbda_sqg_params* p, int32_t batch, int32_t device, void** handle,
                      turbda_status* status);
/* states (host, or device with TURBDA_INPUTS_ON_DEVICE) advanced in place by
 * `hours` (a multiple of dt); TURBDA_BLOWUP names the first non-finite member
 * (status.diverged_particle) and its model time (status.diverged_t) */
TURBDA_API int turbda_sqg_advance(void* handle, double* states, double hours, uint32_t flags, void* stream,
                       double* max_cfl, turbda_status* status);
TURBDA_API int turbda_sqg_destroy(void* handle);
/* shell-summed kinetic energy of ONE state [2][ny][nx] (host, or device with
 * TURBDA_INPUTS_ON_DEVICE): bins kappa = s 2 pi / lx (SqgModel::ke_spectrum,
 * proj/src/sqg.cpp:306-335); *n_bins = shells, up to max_bins written */
TURBDA_API int turbda_sqg_ke_spectrum(void* handle, const double* state, uint32_t flags,
                                      double* kappa, double* energy, int32_t max_bins,
                                      int32_t* n_bins, turbda_status* status);
/* log-log least-squares slope over shells [lo, hi], empty bins skipped
 * (fit_loglog_slope, proj/src/sqg.cpp:337-357); TURBDA_CONFIG with < 2 bins */
TURBDA_API int turbda_fit_loglog_slope(const double* kappa, const double* energy, int32_t n,
                                       int32_t lo_shell, int32_t hi_shell, double* slope,
                                       turbda_status* status);
/* nature_run: snapshots [n][2][ny][nx] into host memory */
TURBDA_API int turbda_nature_run(const turbda_sqg_params* p, double spinup, double duration,
                      double interval, uint64_t seed, double* snapshots, int32_t max_snaps,
                      int32_t* n_snaps, int32_t device, turbda_status* status);

#define TURBDA_VARIANT_FREE_RUN 0
#define TURBDA_VARIANT_LETKF 1 /* turbda_letkf_analyze on the device each cycle */
#define TURBDA_VARIANT_ENSF 2

typedef struct turbda_experiment { /* ExperimentConfig, proj/include/turbda/osse.hpp:30-50 */
    turbda_sqg_params sqg;
    int32_t variant;        /* TURBDA_VARIANT_*                                   */
    int32_t model_quality;  /* 0 perfect, 1 imperfect (inject_model_error)        */
    int32_t cycles, ensemble_size;
    double obs_interval, spinup_hours, clim_hours;
    uint64_t seed;
    double obs_r;
    int32_t obs_thinning, obs_arctan;
    int32_t n_steps, minibatch_j;  /* EnsfConfig                                */
    double eps, damping_t, relax_factor;
    int32_t precision, score_mode; /* B200 extensions (turbda_ensf_params)      */
    int32_t me_enabled, me_ncomp;  /* ModelErrorConfig                          */
    double me_base_amplitude;      /* <= 0: climatological RMS of the nature run */
    double me_prob[8], me_frac[8];
    double letkf_cutoff_km, letkf_domain_km, letkf_rtps_alpha; /* LetkfConfig */
    int32_t letkf_obs_thinning, reserved;
} turbda_experiment;

TURBDA_API void turbda_experiment_init(turbda_experiment* e);
/* records: [cycles][6] = cycle, time, forecast_rmse, analysis_rmse,
 * forecast_spread, analysis_spread (CycleRecord, proj/include/turbda/osse.hpp:52-59).
 * On TURBDA_ABORTED the records of the completed cycles are valid
 * (*n_records of them), as run_experiment's partial_out.
 * phase_seconds (optional, [4]): device time of the nature run + truth bundle,
 * all ensemble forecasts (+ model error), all analyses (+ observation
 * synthesis), all diagnostics. */
TURBDA_API int turbda_run_experiment(const turbda_experiment* e, int32_t device, double* records,
                          int32_t max_records, int32_t* n_records, double* max_cfl,
                          double* phase_seconds, turbda_status* status);

/* Open-loop probe of a cycled run: the same experiment, and at each listed
 * cycle a copy of what that cycle's analysis saw and produced over the
 * coordinate window [k0, k0 + width): the forecast ensemble, the analysis
 * ensemble (both [n_cycles][m][width]) and the whole observation vector
 * ([n_cycles][obs_dim]).  Lets a test recompute one cycle's analysis of the
 * window with the CPU oracle and compare (open-loop per-cycle parity). */
typedef struct turbda_probe {
    int32_t n_cycles;
    const int32_t* cycles;  /* ascending cycle numbers (1-based)              */
    int64_t k0, width;      /* coordinate window                              */
    double* forecast;       /* host, [n_cycles][ensemble_size][width]         */
    double* analysis;       /* host, [n_cycles][ensemble_size][width]         */
    double* y;              /* host, [n_cycles][obs_dim] (NULL: not copied)   */
} turbda_probe;

TURBDA_API int turbda_run_experiment_probe(const turbda_experiment* e, int32_t device,
                                double* records, int32_t max_records, int32_t* n_records,
                                double* max_cfl, double* phase_seconds,
                                const turbda_probe* probe, turbda_status* status);

/* -------------------------------------------------------------------------
 * LETKF arm: letkf_analyze / rtps_inflate /
 * gaspari_cohn, proj/include/turbda/letkf.hpp:11-56, proj/src/letkf.cpp:10-207.
 * Grid operators only (identity / index selection, optional arctan), the
 * observations located on the grid (operator_locations,
 * proj/src/observation.cpp:43-60) unless `locations` ([obs_dim][2]) is given.
 * fp64; agrees with the reference formulation to rounding.
 * ------------------------------------------------------------------------- */
typedef struct turbda_letkf_params { /* LetkfConfig + GridSpec + Observation shape */
    int32_t nx, ny;         /* grid (nz = 2), nx == ny (isotropic metric)        */
    int32_t n_members;      /* M                                                 */
    int32_t obs_kind;       /* as turbda_ensf_params.obs_kind                    */
    int64_t obs_dim;
    double cutoff_km;       /* LetkfConfig::cutoff_km (default 2000)             */
    double domain_km;       /* LetkfConfig::domain_km (default 20000)            */
    double rtps_alpha;      /* LetkfConfig::rtps_alpha in [0, 1] (default 0.3)   */
    int32_t device;         /* -1 = current device                               */
    uint32_t flags;         /* TURBDA_INPUTS_ON_DEVICE | TURBDA_R_UNIFORM        */
} turbda_letkf_params;

TURBDA_API void turbda_letkf_params_init(turbda_letkf_params* p);
/* forecast / analysis_out: [M][2 nx ny] fp64; y, r_diag [obs_dim];
 * obs_idx [obs_dim] for kinds 1/3; locations optional.  TURBDA_SINGULAR when a
 * local transform has a non-positive eigenvalue. */
TURBDA_API int turbda_letkf_analyze(const turbda_letkf_params* p, const double* forecast,
                                    const double* y, const double* r_diag,
                                    const int64_t* obs_idx, const double* locations,
                                    double* analysis_out, void* stream, turbda_status* status);
/* RTPS inflation of an [M][d] analysis towards the background spread */
TURBDA_API int turbda_rtps_inflate(const double* analysis, const double* background, int32_t m,
                                   int64_t d, double alpha, double* out, int32_t device,
                                   uint32_t flags, void* stream, turbda_status* status);
/* Gaspari-Cohn correlation at normalized distance r (TURBDA_CONFIG for r < 0) */
TURBDA_API int turbda_gaspari_cohn(double r, double* out, turbda_status* status);

/* SQGSNAP v1 snapshot / ensemble checkpoint files (write_snapshot /
 * read_snapshot, proj/src/snapshot.cpp:12-63): `count` consecutive
 * [2][ny][nx] fp64 states, one header each; host or device buffers
 * (TURBDA_INPUTS_ON_DEVICE).  read: up to max_count snapshots; states NULL
 * only queries count / nx / ny / time. */
TURBDA_API int turbda_snapshot_write(const char* path, const double* states, int32_t count,
                                     int32_t nx, int32_t ny, double time_hours, uint32_t flags,
                                     turbda_status* status);
TURBDA_API int turbda_snapshot_read(const char* path, double* states, int32_t max_count,
                                    int32_t* count, int32_t* nx, int32_t* ny, double* time_hours,
                                    uint32_t flags, turbda_status* status);

/* Number of CUDA devices (0 when none), library ABI version, and the name of
 * the kernel family compiled in ("sm_100a"). */
TURBDA_API int turbda_device_count(void);
TURBDA_API int turbda_abi_version(void);
TURBDA_API const char* turbda_build_arch(void);

/* Kernel launches issued by this process since load (evidence counter). */
TURBDA_API uint64_t turbda_launch_count(void);

/* Live timing of the fused analysis kernel: when enabled, every analysis
 * records CUDA events on its launching stream around the ensf kernel.
 * turbda_profile_read() returns (and resets) the summed kernel milliseconds
 * and the number of timed launches since the previous read. */
TURBDA_API void turbda_profile_enable(int on);
TURBDA_API int turbda_profile_read(double* kernel_ms, uint64_t* launches);

#ifdef __cplusplus
}
#endif

#endif /* TURBDA_B200_H */
