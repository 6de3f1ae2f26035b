/* bhgen.c — seeded, counter-based synthetic event generator.
 *
 * Shared by the oracle and the CUDA path as the ONLY common module: it produces
 * input bytes (event coordinates, weights, variable-axis edges) and contains none
 * of the histogramming arithmetic (no FindBin, no bin sums, no statistics).
 *
 * Every value is a pure function of (seed, index):
 *   splitmix64(z)   : Steele/Lea/Flood SplitMix64 finaliser
 *   u(s, i)         = (splitmix64(s ^ splitmix64(i)) >> 11) * 2^-53  in [0, 1)
 *                     (53-bit mantissa mapping of SPEC.md D15)
 * so any chunking of an index range reproduces the same stream and 1e9-event
 * columns never have to exist in memory at once.  Transforms use glibc libm on
 * the host; the GPU consumes exactly these bytes (copied H2D), never a
 * re-generation, so libm differences cannot reach a parity test.
 */
#include <math.h>
#include <stdint.h>
#include <pthread.h>
#include <string.h>

static inline uint64_t splitmix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

static inline double u01(uint64_t seed, uint64_t i) {
    return (double)(splitmix64(seed ^ splitmix64(i)) >> 11) * 0x1.0p-53;
}

enum { BG_UNIFORM = 0, BG_GAUSS = 1, BG_CAUCHY = 2, BG_EXP = 3 };

/* value of distribution `kind` at global event index i (p0, p1 = parameters):
 *   UNIFORM : p0 + (p1 - p0) * u                     (U[p0, p1))
 *   GAUSS   : p0 + p1 * z, z from Box-Muller on the pair k = i/2 with
 *             u1 = 1 - u(s, 2k) in (0, 1], u2 = u(s, 2k+1); even i -> cos, odd i -> sin
 *   CAUCHY  : p0 + p1 * tan(pi * (u - 1/2))          (location p0, scale p1)
 *   EXP     : -log(1 - u) / p0                        (rate p0)
 */
static inline double sample(int kind, uint64_t seed, uint64_t i, double p0, double p1) {
    switch (kind) {
    case BG_UNIFORM: return p0 + (p1 - p0) * u01(seed, i);
    case BG_GAUSS: {
        uint64_t k = i >> 1;
        double u1 = 1.0 - u01(seed, 2 * k), u2 = u01(seed, 2 * k + 1);
        double r = sqrt(-2.0 * log(u1));
        double t = 6.283185307179586 * u2;
        return p0 + p1 * ((i & 1) ? r * sin(t) : r * cos(t));
    }
    case BG_CAUCHY: return p0 + p1 * tan(3.141592653589793 * (u01(seed, i) - 0.5));
    case BG_EXP: return -log(1.0 - u01(seed, i)) / p0;
    }
    return 0.0;
}

typedef struct { int kind; uint64_t seed, start; int64_t n; double p0, p1; double *out; } job_t;

static void *run_job(void *arg) {
    job_t *j = (job_t *)arg;
    for (int64_t t = 0; t < j->n; ++t) j->out[t] = sample(j->kind, j->seed, j->start + (uint64_t)t, j->p0, j->p1);
    return NULL;
}

/* Fill out[0..n) with events start..start+n-1 of the (kind, seed, p0, p1) stream,
 * using up to nthreads host threads. Returns 0, or -1 on bad arguments. */
int bg_fill(int kind, uint64_t seed, uint64_t start, int64_t n, double p0, double p1,
            double *out, int nthreads) {
    if (n < 0 || (n > 0 && !out) || kind < 0 || kind > 3) return -1;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if (n < 65536) nthreads = 1;
    pthread_t th[256];
    int ok[256];
    job_t jobs[256];
    int64_t per = (n + nthreads - 1) / nthreads;
    int nj = 0;
    for (int64_t b = 0; b < n; b += per, ++nj) {
        int64_t e = b + per < n ? b + per : n;
        jobs[nj] = (job_t){kind, seed, start + (uint64_t)b, e - b, p0, p1, out + b};
    }
    for (int t = 1; t < nj; ++t) ok[t] = pthread_create(&th[t], NULL, run_job, &jobs[t]) == 0;
    if (nj > 0) run_job(&jobs[0]);
    for (int t = 1; t < nj; ++t) {
        if (ok[t]) pthread_join(th[t], NULL);
        else run_job(&jobs[t]);
    }
    return 0;
}

/* Variable-axis edges of SURVEY §8(d) C2: e_i = S_i / S_n with
 * S_i = sum_{j<i} (0.5 + u(seed, j)), so e_0 = 0 and e_n = 1 exactly.
 * Widths vary by up to 3x. out has n+1 entries. Returns 0 / -1. */
int bg_edges_random_widths(uint64_t seed, int32_t n, double *out) {
    if (n < 1 || !out) return -1;
    double s = 0.0;
    out[0] = 0.0;
    for (int32_t i = 1; i <= n; ++i) { s += 0.5 + u01(seed, (uint64_t)(i - 1)); out[i] = s; }
    for (int32_t i = 1; i < n; ++i) out[i] = out[i] / s;
    out[n] = 1.0;
    return 0;
}

/* Log-spaced edges on [lo, hi]: e_i = lo * (hi/lo)^(i/n), e_0 = lo, e_n = hi exactly.
 * (C5 H3.) Returns 0 / -1 (needs 0 < lo < hi). */
int bg_edges_log(double lo, double hi, int32_t n, double *out) {
    if (n < 1 || !out || !(lo > 0) || !(hi > lo)) return -1;
    double r = log(hi / lo);
    out[0] = lo;
    for (int32_t i = 1; i < n; ++i) out[i] = lo * exp(r * ((double)i / n));
    out[n] = hi;
    return 0;
}

uint64_t bg_splitmix64(uint64_t z) { return splitmix64(z); }
double bg_u01(uint64_t seed, uint64_t i) { return u01(seed, i); }
