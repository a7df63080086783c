/*
 * CPU ORACLE — test infrastructure only.
 *
 * Plain-C restatement of the reference's compiled OMP inner loops
 * (/root/reference/pkg/src/sparsedict/_kernels.py). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library; the product path (paper_1403_4781_b200) never does.
 *
 * Bit-exactness: the reference kernels are Numba @njit without fastmath, so
 * LLVM neither contracts a*b+c into an FMA nor reassociates reductions. This
 * file must therefore be compiled with -ffp-contract=off and without
 * -ffast-math (see oracle/Makefile); every loop below keeps the reference's
 * iteration order so results are bitwise identical to the Numba kernels
 * (pinned by tests/test_oracle_golden.py against vectors produced by the
 * reference itself, tests/golden/make_golden.py).
 *
 * Layouts (same as the reference's Fortran-ordered arrays):
 *   D  : m x K, column-major  -> D[t + j*m]
 *   Y  : m x N, column-major  -> Y[t + i*m]
 *   G  : K x K (symmetric)     -> G[i*K + j]
 *   idx_out / val_out : N x cap, row-major (row i = signal i)
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_STATUS_OK 0
#define ORC_STATUS_SINGULAR 2
#define ORC_STATUS_STALLED 3

/* _kernels.py:18,20 */
static const double kDiagGuard = 1e-12;
static const double kTieRel = 1e-12;

/* _kernels.py:23-35 — G = D^T D, upper triangle by a scalar loop, mirrored. */
void orc_gram_matrix(const double *D, int64_t m, int64_t K, double *G) {
    for (int64_t i = 0; i < K; ++i) {
        const double *di = D + i * m;
        for (int64_t j = i; j < K; ++j) {
            const double *dj = D + j * m;
            double acc = 0.0;
            for (int64_t t = 0; t < m; ++t) acc += di[t] * dj[t];
            G[i * K + j] = acc;
            G[j * K + i] = acc;
        }
    }
}

/* Per-call scratch for orc_omp_single (the reference allocates these with
 * np.empty/np.zeros inside omp_single, _kernels.py:54,69-74). */
typedef struct {
    double *c0, *corr, *L, *x, *tmp, *r;
    unsigned char *selected;
    int64_t K, m, s_max;
} orc_scratch;

static int scratch_init(orc_scratch *w, int64_t m, int64_t K, int64_t s_max) {
    w->K = K; w->m = m; w->s_max = s_max;
    w->c0 = (double *)malloc(sizeof(double) * (size_t)(K > 0 ? K : 1));
    w->corr = (double *)malloc(sizeof(double) * (size_t)(K > 0 ? K : 1));
    w->L = (double *)malloc(sizeof(double) * (size_t)(s_max * s_max > 0 ? s_max * s_max : 1));
    w->x = (double *)malloc(sizeof(double) * (size_t)(s_max > 0 ? s_max : 1));
    w->tmp = (double *)malloc(sizeof(double) * (size_t)(s_max > 0 ? s_max : 1));
    w->r = (double *)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    w->selected = (unsigned char *)malloc((size_t)(K > 0 ? K : 1));
    return (w->c0 && w->corr && w->L && w->x && w->tmp && w->r && w->selected) ? 0 : -1;
}

static void scratch_free(orc_scratch *w) {
    free(w->c0); free(w->corr); free(w->L); free(w->x); free(w->tmp); free(w->r);
    free(w->selected);
}

/*
 * _kernels.py:38-158 — greedy OMP on one signal with a progressive Cholesky
 * factor of G[S,S]. Writes the support (selection order) into out_idx and the
 * coefficients into out_val; returns n, *status and *rnorm.
 */
static int64_t omp_single_ws(orc_scratch *w, const double *D, const double *G,
                             const double *y, int64_t s_max, double eps,
                             int64_t *out_idx, double *out_val, int64_t *status,
                             double *rnorm_out) {
    const int64_t m = w->m, K = w->K;
    double *c0 = w->c0, *corr = w->corr, *L = w->L, *x = w->x, *tmp = w->tmp, *r = w->r;
    unsigned char *selected = w->selected;

    /* :54-59  c0 = D^T y */
    for (int64_t j = 0; j < K; ++j) {
        const double *dj = D + j * m;
        double acc = 0.0;
        for (int64_t t = 0; t < m; ++t) acc += dj[t] * y[t];
        c0[j] = acc;
    }
    /* :61-67 */
    double ysq = 0.0;
    for (int64_t t = 0; t < m; ++t) ysq += y[t] * y[t];
    double rnorm = sqrt(ysq);
    if (rnorm <= eps || rnorm == 0.0) {
        *status = ORC_STATUS_OK;
        *rnorm_out = rnorm;
        return 0;
    }
    memset(L, 0, sizeof(double) * (size_t)(s_max * s_max));
    memset(x, 0, sizeof(double) * (size_t)s_max);
    memset(selected, 0, (size_t)K);
    int64_t n = 0;
    int64_t st = ORC_STATUS_OK;

    for (int64_t step = 0; step < s_max; ++step) {
        /* :81-87  corr = c0 - sum_t G[idx_t, :] x_t */
        for (int64_t j = 0; j < K; ++j) corr[j] = c0[j];
        for (int64_t t = 0; t < n; ++t) {
            const double coef = x[t];
            const double *grow = G + out_idx[t] * K;
            for (int64_t j = 0; j < K; ++j) corr[j] -= grow[j] * coef;
        }
        /* :88-96  abs, exclusion of the support, max */
        double cmax = -1.0;
        for (int64_t j = 0; j < K; ++j) {
            if (selected[j]) { corr[j] = 0.0; continue; }
            const double a = fabs(corr[j]);
            corr[j] = a;
            if (a > cmax) cmax = a;
        }
        /* :97-100  stall */
        if (cmax <= 1e-13 * rnorm) { st = ORC_STATUS_STALLED; break; }
        /* :101-107  lowest index inside the tie window */
        int64_t best = -1;
        const double thresh = cmax - kTieRel * cmax;
        for (int64_t j = 0; j < K; ++j) {
            if (!selected[j] && corr[j] >= thresh) { best = j; break; }
        }
        /* :109-127  append a Cholesky row with the diagonal guard */
        double dsq = G[best * K + best];
        for (int64_t t = 0; t < n; ++t) {
            double acc = G[out_idx[t] * K + best];
            for (int64_t u = 0; u < t; ++u) acc -= L[t * s_max + u] * L[n * s_max + u];
            const double wv = acc / L[t * s_max + t];
            L[n * s_max + t] = wv;
            dsq -= wv * wv;
        }
        if (dsq <= kDiagGuard) { st = ORC_STATUS_SINGULAR; break; }
        L[n * s_max + n] = sqrt(dsq);
        out_idx[n] = best;
        selected[best] = 1;
        n += 1;
        /* :129-139  L L^T x = c0[S] */
        for (int64_t t = 0; t < n; ++t) {
            double acc = c0[out_idx[t]];
            for (int64_t u = 0; u < t; ++u) acc -= L[t * s_max + u] * tmp[u];
            tmp[t] = acc / L[t * s_max + t];
        }
        for (int64_t t = n - 1; t >= 0; --t) {
            double acc = tmp[t];
            for (int64_t u = t + 1; u < n; ++u) acc -= L[u * s_max + t] * x[u];
            x[t] = acc / L[t * s_max + t];
        }
        /* :141-154  explicit residual */
        for (int64_t i = 0; i < m; ++i) r[i] = y[i];
        for (int64_t t = 0; t < n; ++t) {
            const double coef = x[t];
            const double *dc = D + out_idx[t] * m;
            for (int64_t i = 0; i < m; ++i) r[i] -= dc[i] * coef;
        }
        double rsq = 0.0;
        for (int64_t i = 0; i < m; ++i) rsq += r[i] * r[i];
        rnorm = sqrt(rsq);
        if (rnorm <= eps) break;
    }
    for (int64_t t = 0; t < n; ++t) out_val[t] = x[t];
    *status = st;
    *rnorm_out = rnorm;
    return n;
}

/* Single-signal entry (mirrors _kernels.omp_single's contract). */
int64_t orc_omp_single(const double *D, const double *G, const double *y, int64_t m,
                       int64_t K, int64_t s_max, double eps, int64_t *out_idx,
                       double *out_val, int64_t *status, double *rnorm) {
    orc_scratch w;
    if (scratch_init(&w, m, K, s_max) != 0) { scratch_free(&w); return -1; }
    int64_t n = omp_single_ws(&w, D, G, y, s_max, eps, out_idx, out_val, status, rnorm);
    scratch_free(&w);
    return n;
}

/* _kernels.py:161-173 — columns lo..hi-1 of Y. Returns 0, or -1 on OOM. */
int orc_omp_batch_range(const double *D, const double *G, const double *Y, int64_t m,
                        int64_t K, int64_t s_max, double eps, int64_t lo, int64_t hi,
                        int64_t *idx_out, double *val_out, int64_t *counts,
                        int64_t *status_out, double *rnorm_out) {
    orc_scratch w;
    if (scratch_init(&w, m, K, s_max) != 0) { scratch_free(&w); return -1; }
    for (int64_t i = lo; i < hi; ++i) {
        int64_t st = 0;
        double rn = 0.0;
        /* the reference copies column i into a contiguous y; Y is F-ordered so
         * the column already is contiguous */
        int64_t n = omp_single_ws(&w, D, G, Y + i * m, s_max, eps, idx_out + i * s_max,
                                  val_out + i * s_max, &st, &rn);
        counts[i] = n;
        status_out[i] = st;
        rnorm_out[i] = rn;
    }
    scratch_free(&w);
    return 0;
}

/* Thread-parallel batch (the reference's ThreadPoolExecutor split,
 * sparse_coding.py:276-292): disjoint column ranges, identical results. */
typedef struct {
    const double *D, *G, *Y;
    int64_t m, K, s_max, lo, hi;
    double eps;
    int64_t *idx_out, *counts, *status_out;
    double *val_out, *rnorm_out;
    int rc;
} orc_job;

static void *orc_job_run(void *arg) {
    orc_job *j = (orc_job *)arg;
    j->rc = orc_omp_batch_range(j->D, j->G, j->Y, j->m, j->K, j->s_max, j->eps, j->lo, j->hi,
                                j->idx_out, j->val_out, j->counts, j->status_out, j->rnorm_out);
    return NULL;
}

int orc_omp_batch_threads(const double *D, const double *G, const double *Y, int64_t m,
                          int64_t K, int64_t N, int64_t s_max, double eps, int threads,
                          int64_t *idx_out, double *val_out, int64_t *counts,
                          int64_t *status_out, double *rnorm_out) {
    if (threads < 1) threads = 1;
    if (threads == 1 || N < 2 * threads)
        return orc_omp_batch_range(D, G, Y, m, K, s_max, eps, 0, N, idx_out, val_out, counts,
                                   status_out, rnorm_out);
    pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)threads);
    orc_job *jobs = (orc_job *)malloc(sizeof(orc_job) * (size_t)threads);
    if (!tid || !jobs) { free(tid); free(jobs); return -1; }
    for (int t = 0; t < threads; ++t) {
        orc_job *j = &jobs[t];
        j->D = D; j->G = G; j->Y = Y; j->m = m; j->K = K; j->s_max = s_max; j->eps = eps;
        j->lo = (N * t) / threads;
        j->hi = (N * (t + 1)) / threads;
        j->idx_out = idx_out; j->val_out = val_out; j->counts = counts;
        j->status_out = status_out; j->rnorm_out = rnorm_out; j->rc = 0;
        pthread_create(&tid[t], NULL, orc_job_run, j);
    }
    int rc = 0;
    for (int t = 0; t < threads; ++t) {
        pthread_join(tid[t], NULL);
        if (jobs[t].rc != 0) rc = jobs[t].rc;
    }
    free(tid);
    free(jobs);
    return rc;
}
