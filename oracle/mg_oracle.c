/*
 * mg_oracle.c -- CPU restatement of the M-Gaussian block-rendering kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library,
 * and only as the checker or the CPU baseline -- never as the product path.
 *
 * Restates, in plain C99 float64, the algorithm of
 *   /root/reference/pkg/src/mgauss/spatial.py:18-66   (cell_index, build)
 *   /root/reference/pkg/src/mgauss/_kernels.py:24-70  (block_forward)
 *   /root/reference/pkg/src/mgauss/_kernels.py:73-144 (block_backward)
 *   /root/reference/pkg/src/mgauss/_kernels.py:147-162 (dense_forward)
 *   /root/reference/pkg/src/mgauss/render.py:60-77,299-317 (chunked threads,
 *     per-thread gradient buffers reduced in fixed thread order)
 * Parity is pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py) -- see tests/test_oracle_golden.py.
 *
 * Compiled with -ffp-contract=off so the transform and cell-key expressions
 * round exactly like numpy's element-wise evaluation.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define MG_EXP_CUTOFF 64.0 /* _kernels.py:21 */

static inline int64_t clamp_i64(int64_t v, int64_t lo, int64_t hi) {
    return v < lo ? lo : (v > hi ? hi : v);
}

/* spatial.py:18-27 -- floor((mu + 1) * (G / 2)), clamped to [0, G-1]. */
static inline int64_t cell_of(double v, int64_t g) {
    double half = (double)g / 2.0;
    return clamp_i64((int64_t)floor((v + 1.0) * half), 0, g - 1);
}

void mgo_cell_index(const double *mu, int64_t n, int64_t g, int64_t *out) {
    for (int64_t i = 0; i < 3 * n; ++i) out[i] = cell_of(mu[i], g);
}

/* spatial.py:46-66 -- stable counting sort by flat key (i*G + j)*G + k. */
void mgo_build(const double *positions, int64_t n, int64_t g,
               int64_t *cell_starts /* g^3 + 1 */, int64_t *cell_indices /* n */) {
    int64_t ncell = g * g * g;
    int64_t *key = (int64_t *)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    memset(cell_starts, 0, sizeof(int64_t) * (ncell + 1));
    for (int64_t p = 0; p < n; ++p) {
        int64_t ci = cell_of(positions[3 * p + 0], g);
        int64_t cj = cell_of(positions[3 * p + 1], g);
        int64_t ck = cell_of(positions[3 * p + 2], g);
        key[p] = (ci * g + cj) * g + ck;
        cell_starts[key[p] + 1] += 1;
    }
    for (int64_t c = 0; c < ncell; ++c) cell_starts[c + 1] += cell_starts[c];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (ncell > 0 ? ncell : 1));
    memcpy(fill, cell_starts, sizeof(int64_t) * ncell);
    for (int64_t p = 0; p < n; ++p) cell_indices[fill[key[p]]++] = p; /* stable */
    free(fill);
    free(key);
}

/* The per-point rigid map of _kernels.py:31-41: x = R_s p + t_s (s >= 0). */
static inline void transform_point(const double *pt, int64_t s, const double *rot,
                                   const double *trans, double *x) {
    if (s >= 0) {
        const double *r = rot + 9 * s;
        const double *t = trans + 3 * s;
        for (int a = 0; a < 3; ++a)
            x[a] = r[3 * a + 0] * pt[0] + r[3 * a + 1] * pt[1] + r[3 * a + 2] * pt[2] + t[a];
    } else {
        x[0] = pt[0]; x[1] = pt[1]; x[2] = pt[2];
    }
}

/* _kernels.py:24-70, one contiguous chunk of points. */
static void forward_chunk(int64_t lo, int64_t hi, const double *points,
                          const int64_t *sids, const double *rot, const double *trans,
                          const double *mu, const double *prec6, const double *alpha,
                          const int64_t *cs, const int64_t *ci_idx, int64_t g,
                          int64_t r, double *out_i, int64_t *out_cnt, double *out_x) {
    for (int64_t b = lo; b < hi; ++b) {
        double x[3];
        transform_point(points + 3 * b, sids[b], rot, trans, x);
        out_x[3 * b + 0] = x[0]; out_x[3 * b + 1] = x[1]; out_x[3 * b + 2] = x[2];
        int64_t c0 = cell_of(x[0], g), c1 = cell_of(x[1], g), c2 = cell_of(x[2], g);
        int64_t klo = c2 - r > 0 ? c2 - r : 0, khi = c2 + r < g - 1 ? c2 + r : g - 1;
        int64_t ilo = c0 - r > 0 ? c0 - r : 0, ihi = c0 + r < g - 1 ? c0 + r : g - 1;
        int64_t jlo = c1 - r > 0 ? c1 - r : 0, jhi = c1 + r < g - 1 ? c1 + r : g - 1;
        double acc = 0.0;
        int64_t cnt = 0;
        for (int64_t ii = ilo; ii <= ihi; ++ii) {
            for (int64_t jj = jlo; jj <= jhi; ++jj) {
                int64_t base = (ii * g + jj) * g;
                for (int64_t p = cs[base + klo]; p < cs[base + khi + 1]; ++p) {
                    int64_t i = ci_idx[p];
                    const double *P = prec6 + 6 * i;
                    double dx = x[0] - mu[3 * i], dy = x[1] - mu[3 * i + 1], dz = x[2] - mu[3 * i + 2];
                    double m = P[0] * dx * dx + P[3] * dy * dy + P[5] * dz * dz +
                               2.0 * (P[1] * dx * dy + P[2] * dx * dz + P[4] * dy * dz);
                    ++cnt;
                    if (m <= MG_EXP_CUTOFF) acc += alpha[i] * exp(-0.5 * m);
                }
            }
        }
        out_i[b] = acc;
        out_cnt[b] = cnt;
    }
}

/* _kernels.py:73-144, one chunk; accumulates into the given buffers. */
static void backward_chunk(int64_t lo, int64_t hi, const double *points,
                           const int64_t *sids, const double *rot, const double *trans,
                           const double *mu, const double *prec6, const double *alpha,
                           const int64_t *cs, const int64_t *ci_idx, int64_t g, int64_t r,
                           const double *upstream, double *d_mu, double *d_abar6,
                           double *d_alpha, double *out_dp) {
    for (int64_t b = lo; b < hi; ++b) {
        double x[3];
        transform_point(points + 3 * b, sids[b], rot, trans, x);
        int64_t c0 = cell_of(x[0], g), c1 = cell_of(x[1], g), c2 = cell_of(x[2], g);
        int64_t klo = c2 - r > 0 ? c2 - r : 0, khi = c2 + r < g - 1 ? c2 + r : g - 1;
        int64_t ilo = c0 - r > 0 ? c0 - r : 0, ihi = c0 + r < g - 1 ? c0 + r : g - 1;
        int64_t jlo = c1 - r > 0 ? c1 - r : 0, jhi = c1 + r < g - 1 ? c1 + r : g - 1;
        double u = upstream[b];
        double h[3] = {0.0, 0.0, 0.0};
        for (int64_t ii = ilo; ii <= ihi; ++ii) {
            for (int64_t jj = jlo; jj <= jhi; ++jj) {
                int64_t base = (ii * g + jj) * g;
                for (int64_t p = cs[base + klo]; p < cs[base + khi + 1]; ++p) {
                    int64_t i = ci_idx[p];
                    const double *P = prec6 + 6 * i;
                    double d[3] = {x[0] - mu[3 * i], x[1] - mu[3 * i + 1], x[2] - mu[3 * i + 2]};
                    double pd[3] = {P[0] * d[0] + P[1] * d[1] + P[2] * d[2],
                                    P[1] * d[0] + P[3] * d[1] + P[4] * d[2],
                                    P[2] * d[0] + P[4] * d[1] + P[5] * d[2]};
                    double m = d[0] * pd[0] + d[1] * pd[1] + d[2] * pd[2];
                    if (m > MG_EXP_CUTOFF) continue;
                    double gv = exp(-0.5 * m);
                    d_alpha[i] += u * gv;
                    double coef = u * alpha[i] * gv;
                    for (int a = 0; a < 3; ++a) {
                        d_mu[3 * i + a] += coef * pd[a];
                        h[a] -= coef * pd[a];
                    }
                    double w = -0.5 * coef;
                    double *A = d_abar6 + 6 * i;
                    A[0] += w * d[0] * d[0]; A[1] += w * d[0] * d[1]; A[2] += w * d[0] * d[2];
                    A[3] += w * d[1] * d[1]; A[4] += w * d[1] * d[2]; A[5] += w * d[2] * d[2];
                }
            }
        }
        out_dp[3 * b + 0] = h[0]; out_dp[3 * b + 1] = h[1]; out_dp[3 * b + 2] = h[2];
    }
}

/* render.py:60-63 -- at most `threads` chunks of >= 1024 points, linspace edges. */
static int64_t chunk_edges(int64_t n, int threads, int64_t *edges) {
    int64_t t = n / 1024;
    if (t < 1) t = 1;
    if (t > threads) t = threads;
    for (int64_t k = 0; k <= t; ++k) edges[k] = (int64_t)((double)n * (double)k / (double)t);
    return t;
}

typedef struct {
    int64_t lo, hi;
    const double *points; const int64_t *sids; const double *rot; const double *trans;
    const double *mu; const double *prec6; const double *alpha;
    const int64_t *cs; const int64_t *ci_idx; int64_t g, r;
    double *out_i; int64_t *out_cnt; double *out_x;
    const double *upstream; double *d_mu, *d_abar6, *d_alpha, *out_dp;
    int backward;
} chunk_job;

static void *run_chunk(void *arg) {
    chunk_job *j = (chunk_job *)arg;
    if (j->backward)
        backward_chunk(j->lo, j->hi, j->points, j->sids, j->rot, j->trans, j->mu, j->prec6,
                       j->alpha, j->cs, j->ci_idx, j->g, j->r, j->upstream, j->d_mu,
                       j->d_abar6, j->d_alpha, j->out_dp);
    else
        forward_chunk(j->lo, j->hi, j->points, j->sids, j->rot, j->trans, j->mu, j->prec6,
                      j->alpha, j->cs, j->ci_idx, j->g, j->r, j->out_i, j->out_cnt, j->out_x);
    return NULL;
}

/* render.py:66-77 -- one thread per chunk; chunk 0 runs on the caller. */
static void run_jobs(chunk_job *jobs, int64_t t) {
    pthread_t th[256];
    for (int64_t k = 1; k < t; ++k) pthread_create(&th[k], NULL, run_chunk, &jobs[k]);
    run_chunk(&jobs[0]);
    for (int64_t k = 1; k < t; ++k) pthread_join(th[k], NULL);
}

void mgo_block_forward(const double *points, const int64_t *sids, int64_t b,
                       const double *rot, const double *trans, const double *mu,
                       const double *prec6, const double *alpha, const int64_t *cs,
                       const int64_t *ci_idx, int64_t g, int64_t r, double *out_i,
                       int64_t *out_cnt, double *out_x, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    int64_t edges[257];
    int64_t t = chunk_edges(b, threads, edges);
    chunk_job jobs[256];
    for (int64_t k = 0; k < t; ++k) {
        chunk_job j = {edges[k], edges[k + 1], points, sids, rot, trans, mu, prec6, alpha,
                       cs, ci_idx, g, r, out_i, out_cnt, out_x, NULL, NULL, NULL, NULL, NULL, 0};
        jobs[k] = j;
    }
    run_jobs(jobs, t);
}

void mgo_block_backward(const double *points, const int64_t *sids, int64_t b,
                        const double *rot, const double *trans, const double *mu,
                        const double *prec6, const double *alpha, int64_t n,
                        const int64_t *cs, const int64_t *ci_idx, int64_t g, int64_t r,
                        const double *upstream, double *d_mu, double *d_abar6,
                        double *d_alpha, double *out_dp, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    int64_t edges[257];
    int64_t t = chunk_edges(b, threads, edges);
    if (t == 1) {
        backward_chunk(0, b, points, sids, rot, trans, mu, prec6, alpha, cs, ci_idx, g, r,
                       upstream, d_mu, d_abar6, d_alpha, out_dp);
        return;
    }
    /* per-thread buffers (render.py:299-302); buffer 0 is the caller's */
    double *bufs = (double *)calloc((size_t)(t - 1) * (size_t)n * 10, sizeof(double));
    chunk_job jobs[256];
    for (int64_t k = 0; k < t; ++k) {
        double *bm = k == 0 ? d_mu : bufs + (size_t)(k - 1) * n * 10;
        double *ba = k == 0 ? d_abar6 : bm + 3 * n;
        double *bl = k == 0 ? d_alpha : bm + 9 * n;
        chunk_job j = {edges[k], edges[k + 1], points, sids, rot, trans, mu, prec6, alpha,
                       cs, ci_idx, g, r, NULL, NULL, NULL, upstream, bm, ba, bl, out_dp, 1};
        jobs[k] = j;
    }
    run_jobs(jobs, t);
    /* fixed-order reduction (render.py:313-317) */
    for (int64_t k = 1; k < t; ++k) {
        const double *bm = bufs + (size_t)(k - 1) * n * 10;
        for (int64_t i = 0; i < 3 * n; ++i) d_mu[i] += bm[i];
        for (int64_t i = 0; i < 6 * n; ++i) d_abar6[i] += bm[3 * n + i];
        for (int64_t i = 0; i < n; ++i) d_alpha[i] += bm[9 * n + i];
    }
    free(bufs);
}

/* _kernels.py:147-162 -- all-pairs reference with the same cutoff. */
void mgo_dense_forward(const double *points, int64_t b, const double *mu,
                       const double *prec6, const double *alpha, int64_t n, double *out) {
    for (int64_t q = 0; q < b; ++q) {
        double acc = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            const double *P = prec6 + 6 * i;
            double dx = points[3 * q] - mu[3 * i], dy = points[3 * q + 1] - mu[3 * i + 1],
                   dz = points[3 * q + 2] - mu[3 * i + 2];
            double m = P[0] * dx * dx + P[3] * dy * dy + P[5] * dz * dz +
                       2.0 * (P[1] * dx * dy + P[2] * dx * dz + P[4] * dy * dz);
            if (m <= MG_EXP_CUTOFF) acc += alpha[i] * exp(-0.5 * m);
        }
        out[q] = acc;
    }
}

int mgo_max_threads(void) { return (int)sysconf(_SC_NPROCESSORS_ONLN); }
