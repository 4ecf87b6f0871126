/*
 * oscim_oracle.c -- CPU restatement of the reference hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * This file is the parity oracle for the B200 solver.  It is NOT part of the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  The product path (paper_2505_22631_b200/) never calls into it.
 *
 * It restates, in plain C, the algorithm of the reference package `oscim` 0.1.0
 * (paths relative to /root/reference/pkg/src/oscim/):
 *
 *   osc_philox4x64_10        numpy.random.Philox block function (third-party: numpy 2.3.5,
 *                            Philox4x64-10, Salmon et al. SC'11); call sites dynamics.py:113-114
 *   osc_initial_phases       NoiseSource.initial_phases          dynamics.py:127-129
 *   osc_normal_chunk         NoiseSource.normal_chunk            dynamics.py:116-119
 *                            (Ziggurat draw = numpy's own random_standard_normal_fill, linked
 *                             from numpy's shipped static library numpy/random/lib/libnpyrandom.a,
 *                             so the stream is numpy's bit for bit)
 *   osc_ks_value             KsSchedule.value                    dynamics.py:83-88
 *   osc_step                 trig precompute + _step_serial/_step_parallel
 *                                                                dynamics.py:393-395, 155-190
 *   osc_score                _score_kernel                       dynamics.py:193-223
 *   osc_continuous_energy    sample() energy                     dynamics.py:380
 *   osc_simulate             _simulate                           dynamics.py:333-431
 *
 * Parity status: PINNED.  tests/test_oracle_golden.py checks every function against golden
 * vectors generated from the unmodified reference (tests/golden/make_golden.py, run in the
 * build container where /root/reference is mounted) and against the reference's own
 * known-answer tests (test_dynamics.py:52-58, 110-127, 143-173, 402-418; test_model.py:157-166).
 *
 * Floating point: same operation order as the reference kernels (CSR order, sequential fp64
 * accumulation, x - floor(x) wrap).  sin/cos come from libm where the reference uses numpy's
 * SIMD ufuncs; those agree to <= 1 ulp, which is why trajectory parity is stated with a
 * tolerance (1e-12 per step) rather than bit-exact.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OSC_NOISE_CHUNK 256
static const double OSC_TWO_PI = 6.283185307179586476925286766559;

/* ---- numpy bitgen ABI (numpy/_core/include/numpy/random/bitgen.h) ------------------- */
typedef struct osc_bitgen {
    void *state;
    uint64_t (*next_uint64)(void *st);
    uint32_t (*next_uint32)(void *st);
    double (*next_double)(void *st);
    uint64_t (*next_raw)(void *st);
} osc_bitgen_t;
/* from libnpyrandom.a (numpy/random/src/distributions/distributions.c) */
extern void random_standard_normal_fill(osc_bitgen_t *bitgen, intptr_t cnt, double *out);

/* ---- Philox4x64-10, numpy conventions ------------------------------------------------
 * key = [seed, 0]; 256-bit counter as 4 little-endian u64 words; the counter is incremented
 * BEFORE each block is produced; the 4 outputs are handed out in order. */
typedef struct {
    uint64_t ctr[4];
    uint64_t key[2];
    uint64_t buf[4];
    int pos;
    int has32;
    uint32_t saved32;
} osc_philox_t;

static inline void mulhilo64(uint64_t a, uint64_t b, uint64_t *hi, uint64_t *lo)
{
    __uint128_t p = (__uint128_t)a * b;
    *hi = (uint64_t)(p >> 64);
    *lo = (uint64_t)p;
}

void osc_philox4x64_10(const uint64_t ctr[4], const uint64_t key[2], uint64_t out[4])
{
    uint64_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint64_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        uint64_t hi0, lo0, hi1, lo1;
        mulhilo64(0xD2E7470EE14C6C93ULL, c0, &hi0, &lo0);
        mulhilo64(0xCA5A826395121157ULL, c2, &hi1, &lo1);
        uint64_t n0 = hi1 ^ c1 ^ k0;
        uint64_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B97F4A7C15ULL;
        k1 += 0xBB67AE8584CAA73BULL;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static uint64_t philox_next64(void *st)
{
    osc_philox_t *s = (osc_philox_t *)st;
    if (s->pos < 4)
        return s->buf[s->pos++];
    for (int i = 0; i < 4; ++i)
        if (++s->ctr[i] != 0)
            break;
    osc_philox4x64_10(s->ctr, s->key, s->buf);
    s->pos = 1;
    return s->buf[0];
}
static uint32_t philox_next32(void *st)
{
    osc_philox_t *s = (osc_philox_t *)st;
    if (s->has32) {
        s->has32 = 0;
        return s->saved32;
    }
    uint64_t v = philox_next64(st);
    s->has32 = 1;
    s->saved32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
}
static double philox_next_double(void *st)
{
    return (double)(philox_next64(st) >> 11) * (1.0 / 9007199254740992.0);
}

static void philox_seed(osc_philox_t *s, uint64_t seed, const uint64_t counter[4])
{
    memset(s, 0, sizeof(*s));
    s->key[0] = seed;
    memcpy(s->ctr, counter, sizeof(s->ctr));
    s->pos = 4; /* empty buffer */
}

/* dynamics.py:127-129 -- Philox(key=seed, counter=1<<192).random(n) */
void osc_initial_phases(uint64_t seed, int64_t n, double *out)
{
    osc_philox_t s;
    const uint64_t ctr[4] = {0, 0, 0, 1};
    philox_seed(&s, seed, ctr);
    for (int64_t i = 0; i < n; ++i)
        out[i] = philox_next_double(&s);
}

/* dynamics.py:116-119 -- Philox(key=seed, counter=(chunk*256)<<64).standard_normal((256, n)) */
void osc_normal_chunk(uint64_t seed, int64_t chunk_index, int64_t n, double *out)
{
    osc_philox_t s;
    const uint64_t ctr[4] = {0, (uint64_t)chunk_index * OSC_NOISE_CHUNK, 0, 0};
    philox_seed(&s, seed, ctr);
    osc_bitgen_t bg = {&s, philox_next64, philox_next32, philox_next_double, philox_next64};
    random_standard_normal_fill(&bg, (intptr_t)(OSC_NOISE_CHUNK * n), out);
}

/* dynamics.py:83-88 (Python float %, operands >= 0 => fmod) */
double osc_ks_value(double ks_max, double period, double t)
{
    double tm = fmod(t, period);
    if (tm < 0.0)
        tm += period;
    double half = 0.5 * period;
    if (tm <= half)
        return ks_max * (tm / half);
    return ks_max * (2.0 - tm / half);
}

/* dynamics.py:393-395 then dynamics.py:182-190.  phi, noise, out: [R, n] row-major.
 * noise may be NULL (treated as zeros, i.e. kn_sqrt_h * 0).  scratch: 3*R*n doubles. */
void osc_step(const int64_t *indptr, const int64_t *indices, const double *data,
              int64_t R, int64_t n, const double *phi, const double *noise,
              double K, double ks, double h, double kn_sqrt_h, int64_t n_states,
              double *out, double *scratch, int threads)
{
    const int64_t total = R * n;
    double *sin_p = scratch, *cos_p = scratch + total, *shil = scratch + 2 * total;
    const double w1 = OSC_TWO_PI, wN = OSC_TWO_PI * (double)n_states;
    (void)threads;
#pragma omp parallel num_threads(threads > 0 ? threads : 1)
    {
#pragma omp for schedule(static)
        for (int64_t q = 0; q < total; ++q) {
            double a = w1 * phi[q];
            sin_p[q] = sin(a);
            cos_p[q] = cos(a);
            shil[q] = sin(wN * phi[q]);
        }
#pragma omp for schedule(static)
        for (int64_t q = 0; q < total; ++q) {
            const int64_t r = q / n, i = q - r * n;
            const double *sr = sin_p + r * n, *cr = cos_p + r * n;
            const double si = sr[i], ci = cr[i];
            double acc = 0.0;
            for (int64_t kk = indptr[i]; kk < indptr[i + 1]; ++kk) {
                const int64_t j = indices[kk];
                acc += data[kk] * (si * cr[j] - ci * sr[j]);
            }
            double kick = noise ? kn_sqrt_h * noise[q] : kn_sqrt_h * 0.0;
            double x = phi[q] + h * (K * acc - ks * shil[q]) + kick;
            out[q] = x - floor(x);
        }
    }
}

/* dynamics.py:193-223.  states: int64 [R, n]; obj: [R]. */
void osc_score(const double *phi, int64_t R, int64_t n, int64_t n_states,
               const int64_t *iu, const int64_t *jv, const double *w, int64_t m,
               int maximize, int64_t *states, double *obj, int threads)
{
    (void)threads;
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
    for (int64_t r = 0; r < R; ++r) {
        int64_t *st = states + r * n;
        for (int64_t i = 0; i < n; ++i) {
            double p = phi[r * n + i];
            int64_t best_k = 0;
            double best_d = 2.0;
            for (int64_t k = 0; k < n_states; ++k) {
                double d = fabs(p - (double)k / (double)n_states);
                if (1.0 - d < d)
                    d = 1.0 - d;
                if (d < best_d) {
                    best_d = d;
                    best_k = k;
                }
            }
            st[i] = best_k;
        }
        double acc = 0.0;
        if (maximize) {
            for (int64_t e = 0; e < m; ++e)
                if (st[iu[e]] != st[jv[e]])
                    acc += w[e];
        } else {
            for (int64_t e = 0; e < m; ++e)
                if (st[iu[e]] == st[jv[e]])
                    acc += 1.0;
        }
        obj[r] = acc;
    }
}

/* dynamics.py:380 -- sum_e w_e cos(2 pi (phi_iu - phi_jv)) for one replica row */
double osc_continuous_energy(const double *phi_row, const int64_t *iu, const int64_t *jv,
                             const double *w, int64_t m)
{
    double acc = 0.0;
    for (int64_t e = 0; e < m; ++e)
        acc += w[e] * cos(OSC_TWO_PI * (phi_row[iu[e]] - phi_row[jv[e]]));
    return acc;
}

/* dynamics.py:317-322 */
static double objective_from_states(const int64_t *st, const int64_t *iu, const int64_t *jv,
                                    const double *w, int64_t m, int maximize)
{
    double acc = 0.0;
    for (int64_t e = 0; e < m; ++e) {
        if (maximize)
            acc += w[e] * (double)(st[iu[e]] != st[jv[e]]);
        else
            acc += (double)(st[iu[e]] == st[jv[e]]);
    }
    return acc;
}

/* dynamics.py:325-330; Python round() is round-half-even == rint() in the default mode */
int64_t osc_objective_cadence(int64_t n, int64_t pair_count)
{
    double q = rint((double)pair_count / (double)(n > 1 ? n : 1));
    int64_t c = (int64_t)q;
    if (c > 10) c = 10;
    if (c < 1) c = 1;
    return c;
}

/*
 * dynamics.py:333-431 -- advance R replicas (seeds[r]) together.
 *
 * Inputs : CSR (indptr/indices/data), canonical pairs (iu<jv, w), parameters, seeds.
 *          phi0 (may be NULL) overrides the Philox initial phases; noise_scale 0 skips the
 *          Ziggurat draw entirely (kn == 0 runs need no stream).
 * Outputs: final_phases [R,n]; best_states int64 [R,n]; best_obj [R] (recomputed from the
 *          states, dynamics.py:421); trace_t/trace_ks [max_samples]; energy/best_trace
 *          [R,max_samples]; *n_samples; on a non-finite phase returns 3 and fills
 *          nonfinite[3] = {replica row, oscillator, step} (dynamics.py:276-283).
 * Returns 0 ok, 1 bad argument, 2 trace buffer too small, 3 non-finite.
 */
int osc_simulate(const int64_t *indptr, const int64_t *indices, const double *data,
                 int64_t n, const int64_t *iu, const int64_t *jv, const double *w, int64_t m,
                 double K, double ks_max, double ks_period, double kn, double h, double t_stop,
                 int64_t n_states, const uint64_t *seeds, int64_t R, int maximize,
                 double trace_stride, const double *phi0, int threads,
                 double *final_phases, int64_t *best_states, double *best_obj,
                 double *trace_t, double *trace_ks, double *energy, double *best_trace,
                 int64_t max_samples, int64_t *n_samples, int64_t *steps_out,
                 int64_t *nonfinite)
{
    if (n < 1 || R < 1 || !(h > 0.0) || !(t_stop > 0.0))
        return 1;
    const double stride = trace_stride > 0.0 ? trace_stride : ks_period / 2.0;
    const int64_t steps = (int64_t)ceil(t_stop / h);
    const int64_t total = R * n;
    const int64_t cadence = osc_objective_cadence(n, m);
    const double kn_sqrt_h = kn * sqrt(h);
    int rc = 0;
    int64_t ns = 0;

    double *phi = (double *)malloc(sizeof(double) * total);
    double *out = (double *)malloc(sizeof(double) * total);
    double *scratch = (double *)malloc(sizeof(double) * 3 * total);
    double *noise_block = kn != 0.0 ? (double *)malloc(sizeof(double) * OSC_NOISE_CHUNK * total) : NULL;
    int64_t *states_tmp = (int64_t *)calloc((size_t)total, sizeof(int64_t));
    double *obj_tmp = (double *)calloc((size_t)R, sizeof(double));
    double *best_run = (double *)malloc(sizeof(double) * R);
    if (!phi || !out || !scratch || !states_tmp || !obj_tmp || !best_run || (kn != 0.0 && !noise_block)) {
        rc = 1;
        goto done;
    }

    if (phi0)
        memcpy(phi, phi0, sizeof(double) * total);
    else {
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
        for (int64_t r = 0; r < R; ++r)
            osc_initial_phases(seeds[r], n, phi + r * n);
    }
    for (int64_t r = 0; r < R; ++r)
        best_run[r] = maximize ? -INFINITY : INFINITY;
    memset(best_states, 0, sizeof(int64_t) * total);

#define OSC_SCORE()                                                                        \
    do {                                                                                   \
        osc_score(phi, R, n, n_states, iu, jv, w, m, maximize, states_tmp, obj_tmp, threads); \
        for (int64_t r_ = 0; r_ < R; ++r_) {                                               \
            int better = maximize ? (obj_tmp[r_] > best_run[r_]) : (obj_tmp[r_] < best_run[r_]); \
            if (better) {                                                                  \
                best_run[r_] = obj_tmp[r_];                                                \
                memcpy(best_states + r_ * n, states_tmp + r_ * n, sizeof(int64_t) * n);    \
            }                                                                              \
        }                                                                                  \
    } while (0)
#define OSC_SAMPLE(T_NOW, KS_NOW)                                                          \
    do {                                                                                   \
        OSC_SCORE();                                                                       \
        if (ns >= max_samples) { rc = 2; goto done; }                                      \
        trace_t[ns] = (T_NOW);                                                             \
        trace_ks[ns] = (KS_NOW);                                                           \
        for (int64_t r_ = 0; r_ < R; ++r_) {                                               \
            energy[r_ * max_samples + ns] = osc_continuous_energy(phi + r_ * n, iu, jv, w, m); \
            best_trace[r_ * max_samples + ns] = best_run[r_];                              \
        }                                                                                  \
        ++ns;                                                                              \
    } while (0)

    OSC_SAMPLE(0.0, osc_ks_value(ks_max, ks_period, 0.0));
    double next_sample = stride;
    for (int64_t step = 0; step < steps; ++step) {
        const double t = (double)step * h;
        if (noise_block && step % OSC_NOISE_CHUNK == 0) {
            /* layout [256, R, n] like np.stack(..., axis=1) (dynamics.py:390-392) */
            const int64_t chunk = step / OSC_NOISE_CHUNK;
#pragma omp parallel num_threads(threads > 0 ? threads : 1)
            {
                double *tmp = (double *)malloc(sizeof(double) * OSC_NOISE_CHUNK * n);
#pragma omp for schedule(dynamic, 1)
                for (int64_t r = 0; r < R; ++r) {
                    osc_normal_chunk(seeds[r], chunk, n, tmp);
                    for (int64_t s = 0; s < OSC_NOISE_CHUNK; ++s)
                        memcpy(noise_block + (s * R + r) * n, tmp + s * n, sizeof(double) * n);
                }
                free(tmp);
            }
        }
        const double *kick = noise_block ? noise_block + (step % OSC_NOISE_CHUNK) * total : NULL;
        osc_step(indptr, indices, data, R, n, phi, kick, K,
                 osc_ks_value(ks_max, ks_period, t), h, kn_sqrt_h, n_states, out, scratch, threads);
        double *sw = phi; phi = out; out = sw;
        for (int64_t q = 0; q < total; ++q) {
            if (!isfinite(phi[q])) {
                nonfinite[0] = q / n;
                nonfinite[1] = q % n;
                nonfinite[2] = step;
                rc = 3;
                goto done;
            }
        }
        const double t_next = (double)(step + 1) * h;
        if (t_next >= next_sample || step == steps - 1) {
            while (next_sample <= t_next)
                next_sample += stride;
            OSC_SAMPLE(t_next, osc_ks_value(ks_max, ks_period, t_next));
        } else if (step % cadence == 0) {
            OSC_SCORE();
        }
    }
    memcpy(final_phases, phi, sizeof(double) * total);
    for (int64_t r = 0; r < R; ++r)
        best_obj[r] = objective_from_states(best_states + r * n, iu, jv, w, m, maximize);
    *steps_out = steps;
done:
    *n_samples = ns;
    free(phi); free(out); free(scratch); free(noise_block);
    free(states_tmp); free(obj_tmp); free(best_run);
    return rc;
}

int osc_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
