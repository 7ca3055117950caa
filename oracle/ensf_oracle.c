/*
 * TEST INFRASTRUCTURE ONLY - the CPU oracle ("port") for the EnSF analysis
 * step.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * may load this; the product path never does.
 *
 * A plain-C restatement of the reference hot path, function by function:
 *
 *   orc_splitmix64      proj/src/rng.cpp:33-38
 *   orc_philox4x32      proj/src/rng.cpp:8-31   (Philox4x32-10)
 *   stream key          proj/src/rng.cpp:40-45  (splitmix64(seed ^ splitmix64(use)))
 *   orc_stream_normal   proj/src/rng.cpp:61-84  closed-form: normal #n of a stream
 *                       is half of the Box-Muller pair built from Philox block n>>1
 *                       (verified against RngStream)
 *   orc_fast_exp_nonpos proj/include/turbda/fastexp.hpp:13-50
 *   mixture score       proj/src/ensf.cpp:33-64 (two passes: min shift, accumulate)
 *   likelihood          proj/src/ensf.cpp:197-206
 *   Euler-Maruyama      proj/src/ensf.cpp:208-214
 *   time grid           proj/src/ensf.cpp:149,183-190, proj/include/turbda/ensf.hpp:15-20
 *   minibatch tables    proj/src/ensf.cpp:146-168
 *   orc_relax_spread    proj/src/ensf.cpp:225-258 (+ ensemble_mean proj/src/ensemble.cpp:7-16)
 *
 * Extension over the reference: the analysis may run on a window
 * [k0, k0 + dl) of a state of global dimension d_total (state-dimension
 * sharding).  Because the reference's prior score is componentwise, a window
 * reproduces exactly the reference's values for those coordinates; the noise
 * index uses the global coordinate, n = (s + 1) * d_total + k.
 *
 * Extension (parity UNPINNED - the reference has no such operator,
 * proj/include/turbda/observation.hpp:12): obs_kind 2 / 3 apply
 * h(x) = atan(x) to the full state / selected indices (BASELINE north_star,
 * configs 1 and 5).  The likelihood line of proj/src/ensf.cpp:197-206 then
 * reads sc[k] += damp * ((y - atan(z_k)) / r) / (1 + z_k^2) - the gradient
 * H'(z)^T R^-1 (y - h(z)); everything else is unchanged.
 *
 * Extension (parity UNPINNED; paper Eq. 15-16, the estimator the reference
 * rejects at proj/src/ensf.cpp:27-32): joint = 1 replaces the componentwise
 * weights of mixture_score by one softmax per particle over the full-state
 * squared distances, w_j = softmax_j(-sum_k (z_k - alpha x_jk)^2 / (2 beta^2))
 * (row-minimum shift, fast_exp_nonpos), used for every coordinate.  On a
 * window the distances must span the whole state, so joint runs take the
 * whole state only (k0 = 0, dl = d_total).
 *
 * Status codes follow include/turbda_b200.h: 0 ok, 1 config, 2 dimension,
 * 3 sampler diverged.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_USE_ENSF_PARTICLES 6u
#define ORC_USE_ENSF_BATCH 7u

uint64_t orc_splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

void orc_philox4x32(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        c1 = (uint32_t)p1;
        c3 = (uint32_t)p0;
        c0 = n0;
        c2 = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

uint64_t orc_stream_key(uint64_t seed, uint64_t use) {
    return orc_splitmix64(seed ^ orc_splitmix64(use));
}

static void block_words(uint64_t key, uint64_t entity, uint64_t q, uint32_t w[4]) {
    const uint32_t ctr[4] = {(uint32_t)q, (uint32_t)(q >> 32), (uint32_t)entity,
                             (uint32_t)(entity >> 32)};
    const uint32_t k[2] = {(uint32_t)key, (uint32_t)(key >> 32)};
    orc_philox4x32(ctr, k, w);
}

static double u53(uint32_t lo, uint32_t hi) {
    const uint64_t v = (uint64_t)lo | ((uint64_t)hi << 32);
    return ((double)(v >> 11) + 0.5) * 0x1.0p-53;
}

/* normal #n of the stream (key, entity); RngStream::normal() caches the sin
 * half of each Box-Muller pair, so even n -> cos, odd n -> sin of block n>>1 */
double orc_stream_normal(uint64_t key, uint64_t entity, uint64_t n) {
    uint32_t w[4];
    block_words(key, entity, n >> 1, w);
    const double u1 = u53(w[0], w[1]);
    const double u2 = u53(w[2], w[3]);
    const double r = sqrt(-2.0 * log(u1));
    const double a = 2.0 * 3.14159265358979323846 * u2;
    return (n & 1u) ? r * sin(a) : r * cos(a);
}

/* next_u64 #n of a stream: words 2n, 2n+1 of the word sequence */
uint64_t orc_stream_u64(uint64_t key, uint64_t entity, uint64_t n) {
    uint32_t w[4];
    const uint64_t word = 2 * n;
    block_words(key, entity, word >> 2, w);
    const unsigned o = (unsigned)(word & 3u);
    return (uint64_t)w[o] | ((uint64_t)w[o + 1] << 32);
}

void orc_stream_normals(uint64_t seed, uint64_t use, uint64_t entity, int64_t n0,
                        int64_t count, double* out) {
    const uint64_t key = orc_stream_key(seed, use);
    for (int64_t q = 0; q < count; ++q) out[q] = orc_stream_normal(key, entity, (uint64_t)(n0 + q));
}

double orc_fast_exp_nonpos(double x) {
    const double inv_ln2 = 1.4426950408889634074;
    const double ln2_hi = 6.93147180369123816490e-01;
    const double ln2_lo = 1.90821492927058770002e-10;
    const double magic = 6755399441055744.0; /* 1.5 * 2^52 */
    const int under = x < -708.0;
    if (under) x = 0.0;
    const double t = x * inv_ln2 + magic;
    const double nf = t - magic;
    uint64_t tb;
    memcpy(&tb, &t, 8);
    const int32_t n = (int32_t)(tb & 0xffffffffu);
    double r = x - nf * ln2_hi;
    r -= nf * ln2_lo;
    /* Taylor series of e^r to degree 13, Horner from the top coefficient */
    static const double inv_fact[14] = {
        1.0, 1.0, 0.5, 1.0 / 6.0, 1.0 / 24.0, 1.0 / 120.0, 1.0 / 720.0,
        1.0 / 5040.0, 1.0 / 40320.0, 1.0 / 362880.0, 1.0 / 3628800.0,
        1.0 / 39916800.0, 1.0 / 479001600.0, 0.0};
    double p = inv_fact[12];
    for (int q = 11; q >= 0; --q) p = p * r + inv_fact[q];
    uint64_t pb;
    memcpy(&pb, &p, 8);
    pb += (uint64_t)((int64_t)n) << 52;
    memcpy(&p, &pb, 8);
    return under ? 0.0 : p;
}

typedef struct {
    /* inputs */
    const double* x;      /* [m][dl] window of the forecast */
    int m;
    int64_t dl, k0, d_total;
    const double* y;      /* identity: [dl]; selection: [obs_dim] */
    const double* r;
    const int64_t* idx;   /* selection: global indices (must lie in the window) */
    int64_t obs_dim;
    int obs_kind;
    int n_steps;
    double eps, damping_t;
    uint64_t seed, cycle;
    int j_batch;
    int joint;            /* 1: joint-norm weights (extension) */
    const int* batches;   /* [n_steps][j_batch] or NULL for full batch */
    double* z;            /* [m][dl] particles */
    int* bad_step;        /* [m], -1 = finite throughout */
    int next;             /* shared work counter */
    pthread_mutex_t lock;
} orc_job;

static void run_particle(orc_job* jb, int i) {
    const int64_t dl = jb->dl;
    double* z = jb->z + (size_t)i * (size_t)dl;
    double* mind2 = malloc(sizeof(double) * (size_t)dl);
    double* num = malloc(sizeof(double) * (size_t)dl);
    double* den = malloc(sizeof(double) * (size_t)dl);
    double* sc = malloc(sizeof(double) * (size_t)dl);
    const uint64_t key = orc_stream_key(jb->seed, ORC_USE_ENSF_PARTICLES);
    const uint64_t entity = (jb->cycle << 32) | (uint64_t)i;
    const double dt = (1.0 - jb->eps) / jb->n_steps;
    int* full = NULL;
    if (!jb->batches) {
        full = malloc(sizeof(int) * (size_t)jb->m);
        for (int q = 0; q < jb->m; ++q) full[q] = q;
    }
    jb->bad_step[i] = -1;

    for (int64_t k = 0; k < dl; ++k)
        z[k] = orc_stream_normal(key, entity, (uint64_t)(jb->k0 + k));

    for (int s = 0; s < jb->n_steps; ++s) {
        const double t_hi = 1.0 - s * dt;
        const double t_ev = fmax(t_hi - dt, jb->eps);
        const double alpha = 1.0 - t_ev;
        const double beta2 = t_ev;
        const double b = -1.0 / (1.0 - t_ev);
        const double s2 = 1.0 + 2.0 * t_ev / (1.0 - t_ev);
        const double damp = jb->damping_t - t_ev;
        const double sig = sqrt(s2 * dt);
        const double inv2b = 1.0 / (2.0 * beta2);
        const int* batch = jb->batches ? jb->batches + (size_t)s * (size_t)jb->j_batch : full;

        if (jb->joint) {
            /* one weight per member from the full-state distance */
            double dmin = INFINITY;
            double* dist = num; /* scratch: j_batch <= dl is not guaranteed, use a heap array */
            double* dj = malloc(sizeof(double) * (size_t)jb->j_batch);
            for (int jj = 0; jj < jb->j_batch; ++jj) {
                const double* xm = jb->x + (size_t)batch[jj] * (size_t)dl;
                double acc = 0.0;
                for (int64_t k = 0; k < dl; ++k) {
                    const double diff = z[k] - alpha * xm[k];
                    acc += diff * diff;
                }
                dj[jj] = acc;
                dmin = acc < dmin ? acc : dmin;
            }
            (void)dist;
            double dsum = 0.0;
            for (int jj = 0; jj < jb->j_batch; ++jj) {
                dj[jj] = orc_fast_exp_nonpos((dmin - dj[jj]) * inv2b);
                dsum += dj[jj];
            }
            for (int64_t k = 0; k < dl; ++k) num[k] = 0.0;
            for (int jj = 0; jj < jb->j_batch; ++jj) {
                const double* xm = jb->x + (size_t)batch[jj] * (size_t)dl;
                for (int64_t k = 0; k < dl; ++k) num[k] += dj[jj] * xm[k];
            }
            for (int64_t k = 0; k < dl; ++k) sc[k] = -(z[k] - alpha * num[k] / dsum) / beta2;
            free(dj);
        } else {
        for (int64_t k = 0; k < dl; ++k) mind2[k] = INFINITY;
        for (int jj = 0; jj < jb->j_batch; ++jj) {
            const double* xm = jb->x + (size_t)batch[jj] * (size_t)dl;
            for (int64_t k = 0; k < dl; ++k) {
                const double diff = z[k] - alpha * xm[k];
                const double d2 = diff * diff;
                mind2[k] = d2 < mind2[k] ? d2 : mind2[k];
            }
        }
        for (int64_t k = 0; k < dl; ++k) { num[k] = 0.0; den[k] = 0.0; }
        for (int jj = 0; jj < jb->j_batch; ++jj) {
            const double* xm = jb->x + (size_t)batch[jj] * (size_t)dl;
            for (int64_t k = 0; k < dl; ++k) {
                const double diff = z[k] - alpha * xm[k];
                const double w = orc_fast_exp_nonpos((mind2[k] - diff * diff) * inv2b);
                den[k] += w;
                num[k] += w * xm[k];
            }
        }
        for (int64_t k = 0; k < dl; ++k) sc[k] = -(z[k] - alpha * num[k] / den[k]) / beta2;
        }

        if (jb->obs_kind == 0) {
            for (int64_t k = 0; k < dl; ++k) sc[k] += damp * ((jb->y[k] - z[k]) / jb->r[k]);
        } else if (jb->obs_kind == 1) {
            for (int64_t q = 0; q < jb->obs_dim; ++q) {
                const int64_t k = jb->idx[q] - jb->k0;
                sc[k] += damp * ((jb->y[q] - z[k]) / jb->r[q]);
            }
        } else if (jb->obs_kind == 2) { /* extension: h = atan on every entry */
            for (int64_t k = 0; k < dl; ++k)
                sc[k] += damp * (((jb->y[k] - atan(z[k])) / jb->r[k]) / (1.0 + z[k] * z[k]));
        } else { /* extension: h = atan on selected entries */
            for (int64_t q = 0; q < jb->obs_dim; ++q) {
                const int64_t k = jb->idx[q] - jb->k0;
                sc[k] += damp * (((jb->y[q] - atan(z[k])) / jb->r[q]) / (1.0 + z[k] * z[k]));
            }
        }

        int ok = 1;
        const uint64_t n0 = (uint64_t)(s + 1) * (uint64_t)jb->d_total + (uint64_t)jb->k0;
        for (int64_t k = 0; k < dl; ++k) {
            const double xi = orc_stream_normal(key, entity, n0 + (uint64_t)k);
            z[k] += -(b * z[k] - s2 * sc[k]) * dt + sig * xi;
            if (!isfinite(z[k])) ok = 0;
        }
        if (!ok) { jb->bad_step[i] = s; break; }
    }
    free(full); free(mind2); free(num); free(den); free(sc);
}

static void* worker(void* arg) {
    orc_job* jb = (orc_job*)arg;
    for (;;) {
        pthread_mutex_lock(&jb->lock);
        const int i = jb->next++;
        pthread_mutex_unlock(&jb->lock);
        if (i >= jb->m) break;
        run_particle(jb, i);
    }
    return NULL;
}

/* per-step member subsets, proj/src/ensf.cpp:156-167 */
void orc_batch_table(uint64_t seed, uint64_t cycle, int m, int j_batch, int n_steps, int* out) {
    const uint64_t key = orc_stream_key(seed, ORC_USE_ENSF_BATCH);
    int* pool = malloc(sizeof(int) * (size_t)m);
    for (int s = 0; s < n_steps; ++s) {
        const uint64_t entity = (cycle << 20) + (uint64_t)s;
        for (int q = 0; q < m; ++q) pool[q] = q;
        for (int k = 0; k < j_batch; ++k) {
            const uint64_t u = orc_stream_u64(key, entity, (uint64_t)k);
            const int rr = k + (int)(u % (uint64_t)(m - k));
            const int tmp = pool[k]; pool[k] = pool[rr]; pool[rr] = tmp;
        }
        memcpy(out + (size_t)s * (size_t)j_batch, pool, sizeof(int) * (size_t)j_batch);
    }
    free(pool);
}

int orc_relax_spread(const double* a, const double* f, int m, int64_t d, double factor,
                     double* out) {
    memcpy(out, a, sizeof(double) * (size_t)m * (size_t)d);
    if (factor == 0.0 || m < 2) return 0;
    for (int64_t k = 0; k < d; ++k) {
        double ma = 0.0, mb = 0.0, va = 0.0, vb = 0.0;
        for (int j = 0; j < m; ++j) { ma += a[(size_t)j * d + k]; mb += f[(size_t)j * d + k]; }
        ma *= 1.0 / m;
        mb *= 1.0 / m;
        for (int j = 0; j < m; ++j) {
            const double da = a[(size_t)j * d + k] - ma, db = f[(size_t)j * d + k] - mb;
            va += da * da;
            vb += db * db;
        }
        const double sa = fmax(sqrt(va / (m - 1)), 1e-12);
        const double sb = sqrt(vb / (m - 1));
        const double scale = (1.0 - factor) + factor * sb / sa;
        for (int j = 0; j < m; ++j)
            out[(size_t)j * d + k] = ma + scale * (a[(size_t)j * d + k] - ma);
    }
    return 0;
}

/*
 * Full analysis on the coordinate window [k0, k0 + dl) of a state of global
 * dimension d_total.  x: [m][dl]; out: [m][dl].  Returns 0, 1 (config),
 * 2 (dimension) or 3 (diverged; *diverged_t = pseudo-time of the first
 * non-finite step of the lowest diverging particle).
 */
int orc_analyze(const double* x, int m, int64_t dl, int64_t k0, int64_t d_total,
                const double* y, const double* r, const int64_t* idx, int64_t obs_dim,
                int obs_kind, int n_steps, double eps, int minibatch_j, double damping_t,
                double relax_factor, uint64_t seed, uint64_t cycle, int workers,
                double* out, double* diverged_t, int joint) {
    if (!(eps > 0.0 && eps < 1.0) || n_steps < 10 || minibatch_j < 0 ||
        relax_factor < 0.0 || relax_factor > 1.0)
        return 1;
    if (m < 1 || dl < 0 || k0 < 0 || k0 + dl > d_total) return 2;
    if (joint && (k0 != 0 || dl != d_total)) return 2;
    if (joint && minibatch_j != 0 && minibatch_j < m) return 1;
    for (int64_t q = 0; q < obs_dim; ++q) if (!(r[q] > 0.0)) return 1;
    if (obs_kind < 0 || obs_kind > 3) return 1;
    if ((obs_kind == 0 || obs_kind == 2) && obs_dim != dl) return 2;
    if (obs_kind == 1 || obs_kind == 3)
        for (int64_t q = 0; q < obs_dim; ++q)
            if (idx[q] < k0 || idx[q] >= k0 + dl) return 2;

    orc_job jb;
    memset(&jb, 0, sizeof jb);
    jb.x = x; jb.m = m; jb.dl = dl; jb.k0 = k0; jb.d_total = d_total;
    jb.y = y; jb.r = r; jb.idx = idx; jb.obs_dim = obs_dim; jb.obs_kind = obs_kind;
    jb.n_steps = n_steps; jb.eps = eps; jb.damping_t = damping_t;
    jb.seed = seed; jb.cycle = cycle; jb.joint = joint;
    jb.j_batch = (minibatch_j == 0 || minibatch_j >= m) ? m : minibatch_j;
    int* table = NULL;
    if (jb.j_batch != m) {
        table = malloc(sizeof(int) * (size_t)n_steps * (size_t)jb.j_batch);
        orc_batch_table(seed, cycle, m, jb.j_batch, n_steps, table);
    }
    jb.batches = table;
    double* z = malloc(sizeof(double) * (size_t)m * (size_t)(dl > 0 ? dl : 1));
    int* bad = malloc(sizeof(int) * (size_t)m);
    jb.z = z; jb.bad_step = bad;
    pthread_mutex_init(&jb.lock, NULL);
    if (workers < 1) workers = 1;
    if (workers > m) workers = m;
    pthread_t* th = malloc(sizeof(pthread_t) * (size_t)workers);
    for (int q = 0; q < workers; ++q) pthread_create(&th[q], NULL, worker, &jb);
    for (int q = 0; q < workers; ++q) pthread_join(th[q], NULL);
    free(th);
    pthread_mutex_destroy(&jb.lock);

    int status = 0;
    for (int i = 0; i < m; ++i) {
        if (bad[i] >= 0) {
            const double dt = (1.0 - eps) / n_steps;
            const double t_ev = fmax(1.0 - bad[i] * dt - dt, eps);
            if (diverged_t) *diverged_t = t_ev;
            status = 3;
            break;
        }
    }
    if (status == 0) orc_relax_spread(z, x, m, dl, relax_factor, out);
    free(z); free(bad); free(table);
    return status;
}
