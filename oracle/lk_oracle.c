/*
 * lk_oracle.c -- CPU fp64 restatement of the reference's exact Lloyd path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path links or calls this
 * file; it is the checker that tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py compare the CUDA path against.
 *
 * It restates, bit for bit, what the reference computes in numpy:
 *
 *   dist_matrix   /root/reference/pkg/src/lloydkit/core.py:98-108
 *       diff = x - c (fp64), sq = diff*diff, numpy pairwise summation over d,
 *       sqrt.  The pairwise order (8 accumulators, blocks of <=128, recursive
 *       halving rounded down to a multiple of 8) is numpy's pairwise_sum for
 *       a contiguous reduction axis; pinned against the reference itself by
 *       tests/test_oracle.py.
 *   assign_full   lloyd.py:69-75       argmin keeps the FIRST minimum.
 *   refine_full   lloyd.py:78-97       np.bincount(weights=...) per dim is a
 *       sequential row-order fp64 accumulation; empty clusters keep the
 *       previous centroid.
 *   sse           core.py:172-179      np.sum over the flattened (n,d)
 *       residual matrix -- pairwise over n*d in C order.
 *   run_lloyd     lloyd.py:145-182     changed vs the previous labels (all -1
 *       initially), stop after the first iteration with changed == 0.
 *
 * Compiled with -ffp-contract=off: numpy never fuses the multiply into the
 * add, so neither may we.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define PW_BLOCKSIZE 128

/* numpy pairwise_sum for a contiguous double array (numpy/_core/src/umath/
 * loops_utils.h.src).  Restated, not copied: same association order. */
double lko_pairwise_sum(const double *a, int64_t n)
{
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; i++) res += a[i];
        return res;
    }
    if (n <= PW_BLOCKSIZE) {
        double r[8];
        for (int j = 0; j < 8; j++) r[j] = a[j];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return lko_pairwise_sum(a, n2) + lko_pairwise_sum(a + n2, n - n2);
}

/* One row of dist_matrix: out[j] = sqrt(pairwise(sq(x - C[j]))). */
void lko_dist_row(const double *x, const double *C, int32_t k, int32_t d,
                  double *out, double *scratch)
{
    for (int32_t j = 0; j < k; j++) {
        const double *c = C + (int64_t)j * d;
        for (int32_t z = 0; z < d; z++) {
            double t = x[z] - c[z];
            scratch[z] = t * t;
        }
        out[j] = sqrt(lko_pairwise_sum(scratch, d));
    }
}

/* argmin (first minimum) + the smallest and second-smallest distances,
 * the latter as np.partition(d, 1)[:, :2] would give them (inf if k == 1). */
static void row_top2(const double *dist, int32_t k, int64_t *lab, double *d1, double *d2)
{
    int32_t best = 0;
    double b = dist[0];
    for (int32_t j = 1; j < k; j++)
        if (dist[j] < b) { b = dist[j]; best = j; }
    double s = INFINITY;
    for (int32_t j = 0; j < k; j++)
        if (j != best && dist[j] < s) s = dist[j];
    *lab = best;
    if (d1) *d1 = b;
    if (d2) *d2 = s;
}

typedef struct {
    const double *X;
    const double *C;
    int64_t r0, r1;
    int32_t d, k;
    int64_t *labels;
    double *d1, *d2;
} assign_job;

static void *assign_worker(void *arg)
{
    assign_job *jb = (assign_job *)arg;
    double *dist = (double *)malloc(sizeof(double) * (size_t)jb->k);
    double *scr = (double *)malloc(sizeof(double) * (size_t)(jb->d > 0 ? jb->d : 1));
    for (int64_t i = jb->r0; i < jb->r1; i++) {
        lko_dist_row(jb->X + i * jb->d, jb->C, jb->k, jb->d, dist, scr);
        row_top2(dist, jb->k, jb->labels + i, jb->d1 ? jb->d1 + i : NULL,
                 jb->d2 ? jb->d2 + i : NULL);
    }
    free(dist);
    free(scr);
    return NULL;
}

/* assign_full over rows [0, n), split across nthreads pthreads. d1/d2 may be NULL. */
void lko_assign_full(const double *X, int64_t n, int32_t d, const double *C, int32_t k,
                     int64_t *labels, double *d1, double *d2, int32_t nthreads)
{
    if (nthreads < 1) nthreads = 1;
    if ((int64_t)nthreads > n) nthreads = (int32_t)(n > 0 ? n : 1);
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    assign_job *jobs = (assign_job *)malloc(sizeof(assign_job) * (size_t)nthreads);
    for (int32_t t = 0; t < nthreads; t++) {
        jobs[t].X = X; jobs[t].C = C; jobs[t].d = d; jobs[t].k = k;
        jobs[t].r0 = n * t / nthreads; jobs[t].r1 = n * (t + 1) / nthreads;
        jobs[t].labels = labels; jobs[t].d1 = d1; jobs[t].d2 = d2;
        if (nthreads == 1) assign_worker(&jobs[t]);
        else pthread_create(&th[t], NULL, assign_worker, &jobs[t]);
    }
    if (nthreads > 1)
        for (int32_t t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    free(th);
    free(jobs);
}

/* refine_full: sequential row-order sums (np.bincount with weights), then
 * sums / counts for non-empty clusters, previous centroid otherwise. */
void lko_refine_full(const double *X, int64_t n, int32_t d, const int64_t *labels,
                     int32_t k, const double *prev, double *out, int64_t *counts_out)
{
    double *sums = (double *)calloc((size_t)k * (size_t)d, sizeof(double));
    int64_t *cnt = (int64_t *)calloc((size_t)k, sizeof(int64_t));
    /* bincount is per dimension over all rows; the per-(cluster,dim) addition
     * order is row order either way, so one pass over rows is identical. */
    for (int64_t i = 0; i < n; i++) {
        int64_t a = labels[i];
        cnt[a]++;
        const double *x = X + i * d;
        double *s = sums + a * d;
        for (int32_t z = 0; z < d; z++) s[z] += x[z];
    }
    for (int32_t j = 0; j < k; j++) {
        for (int32_t z = 0; z < d; z++) {
            out[(int64_t)j * d + z] = cnt[j] > 0 ? sums[(int64_t)j * d + z] / (double)cnt[j]
                                                 : prev[(int64_t)j * d + z];
        }
        if (counts_out) counts_out[j] = cnt[j];
    }
    free(sums);
    free(cnt);
}

/* sse: np.sum(diff * diff) over the flattened C-order (n, d) matrix. */
double lko_sse(const double *X, int64_t n, int32_t d, const double *C, const int64_t *labels)
{
    int64_t m = n * (int64_t)d;
    double *sq = (double *)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    for (int64_t i = 0; i < n; i++) {
        const double *x = X + i * d;
        const double *c = C + labels[i] * d;
        for (int32_t z = 0; z < d; z++) {
            double t = x[z] - c[z];
            sq[i * d + z] = t * t;
        }
    }
    double s = lko_pairwise_sum(sq, m);
    free(sq);
    return s;
}

/* run_lloyd with a given init.  history: [t_max, n] int64 (may be NULL),
 * changed/sse: [t_max].  Returns the number of iterations run; *converged set. */
int32_t lko_run_lloyd(const double *X, int64_t n, int32_t d, int32_t k, const double *init,
                      int32_t t_max, int32_t nthreads, int64_t *history, double *centroids_out,
                      int64_t *labels_out, int64_t *changed_out, double *sse_out,
                      int32_t *converged)
{
    size_t kd = (size_t)k * (size_t)d;
    double *C = (double *)malloc(sizeof(double) * kd);
    double *Cn = (double *)malloc(sizeof(double) * kd);
    int64_t *prev = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    memcpy(C, init, sizeof(double) * kd);
    for (int64_t i = 0; i < n; i++) prev[i] = -1;
    *converged = 0;
    int32_t it = 0;
    while (it < t_max) {
        lko_assign_full(X, n, d, C, k, cur, NULL, NULL, nthreads);
        int64_t ch = 0;
        for (int64_t i = 0; i < n; i++) ch += (cur[i] != prev[i]);
        lko_refine_full(X, n, d, cur, k, C, Cn, NULL);
        memcpy(C, Cn, sizeof(double) * kd);
        if (history) memcpy(history + (int64_t)it * n, cur, sizeof(int64_t) * (size_t)n);
        if (changed_out) changed_out[it] = ch;
        if (sse_out) sse_out[it] = lko_sse(X, n, d, C, cur);
        memcpy(prev, cur, sizeof(int64_t) * (size_t)n);
        it++;
        if (ch == 0) { *converged = 1; break; }
    }
    memcpy(centroids_out, C, sizeof(double) * kd);
    if (labels_out) memcpy(labels_out, prev, sizeof(int64_t) * (size_t)n);
    free(C); free(Cn); free(prev); free(cur);
    return it;
}

/* ------------------------------------------------------------------------
 * Hamerly (pruners.py:222-264 + run_pruner :862-923) in fp64: the reference's
 * bounded strategy, restated for the CPU baseline.  Pruning uses the bounds
 * with a 1e-10 relative safety margin, and every rescanned row uses the exact
 * numpy-order distances, so labels are identical to lko_run_lloyd.
 */
typedef struct {
    const double *X, *C;
    const double *s, *drift;
    double dmax1, dmax2;
    int32_t amax;
    int64_t r0, r1;
    int32_t d, k, first;
    int64_t *lab;
    double *ub, *lb;
    int64_t dist;     /* distances evaluated (reference accounting) */
} ham_job;

static void *ham_worker(void *arg)
{
    ham_job *jb = (ham_job *)arg;
    const int32_t d = jb->d, k = jb->k;
    double *dist = (double *)malloc(sizeof(double) * (size_t)k);
    double *scr = (double *)malloc(sizeof(double) * (size_t)(d > 0 ? d : 1));
    int64_t nd = 0;
    for (int64_t i = jb->r0; i < jb->r1; i++) {
        const double *x = jb->X + i * d;
        if (!jb->first) {
            int64_t a = jb->lab[i];
            double u = jb->ub[i] + jb->drift[a];
            double l = jb->lb[i] - (a == jb->amax ? jb->dmax2 : jb->dmax1);
            double gate = l > jb->s[a] ? l : jb->s[a];
            jb->ub[i] = u;
            jb->lb[i] = l;
            if (gate > u * (1.0 + 1e-10)) continue;
            lko_dist_row(x, jb->C + a * d, 1, d, &u, scr);
            nd += 1;
            jb->ub[i] = u;
            if (gate > u * (1.0 + 1e-10)) continue;
            nd += k - 1;
        } else {
            nd += k;
        }
        lko_dist_row(x, jb->C, k, d, dist, scr);
        double b1, b2;
        row_top2(dist, k, jb->lab + i, &b1, &b2);
        jb->ub[i] = b1;
        jb->lb[i] = b2;
    }
    jb->dist = nd;
    free(dist);
    free(scr);
    return NULL;
}

int32_t lko_run_hamerly(const double *X, int64_t n, int32_t d, int32_t k, const double *init,
                        int32_t t_max, int32_t nthreads, int64_t *history, double *centroids_out,
                        int64_t *labels_out, int64_t *changed_out, int64_t *dist_out,
                        int32_t *converged)
{
    size_t kd = (size_t)k * (size_t)d;
    double *C = (double *)malloc(sizeof(double) * kd);
    double *Cn = (double *)malloc(sizeof(double) * kd);
    double *s = (double *)malloc(sizeof(double) * (size_t)k);
    double *drift = (double *)calloc((size_t)k, sizeof(double));
    double *tmp = (double *)malloc(sizeof(double) * (size_t)k);
    double *scr = (double *)malloc(sizeof(double) * (size_t)(d > 0 ? d : 1));
    int64_t *prev = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    double *ub = (double *)malloc(sizeof(double) * (size_t)n);
    double *lb = (double *)malloc(sizeof(double) * (size_t)n);
    memcpy(C, init, sizeof(double) * kd);
    for (int64_t i = 0; i < n; i++) prev[i] = -1;
    if (nthreads < 1) nthreads = 1;
    if ((int64_t)nthreads > n) nthreads = (int32_t)(n > 0 ? n : 1);
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    ham_job *jobs = (ham_job *)malloc(sizeof(ham_job) * (size_t)nthreads);
    *converged = 0;
    int32_t it = 0;
    double dmax1 = 0, dmax2 = 0;
    int32_t amax = -1;
    while (it < t_max) {
        if (it > 0) {
            /* s_j = 1/2 min_{j' != j} |c_j - c_j'| (bounds.py:38-47) */
            for (int32_t j = 0; j < k; j++) {
                lko_dist_row(C + (int64_t)j * d, C, k, d, tmp, scr);
                double m = INFINITY;
                for (int32_t jj = 0; jj < k; jj++)
                    if (jj != j && tmp[jj] < m) m = tmp[jj];
                s[j] = 0.5 * m * (1.0 - 1e-10);
            }
        }
        if (it > 0) memcpy(cur, prev, sizeof(int64_t) * (size_t)n);
        for (int32_t t = 0; t < nthreads; t++) {
            ham_job *jb = &jobs[t];
            jb->X = X; jb->C = C; jb->s = s; jb->drift = drift;
            jb->dmax1 = dmax1; jb->dmax2 = dmax2; jb->amax = amax;
            jb->r0 = n * t / nthreads; jb->r1 = n * (t + 1) / nthreads;
            jb->d = d; jb->k = k; jb->first = (it == 0);
            jb->lab = cur; jb->ub = ub; jb->lb = lb; jb->dist = 0;
            if (nthreads == 1) ham_worker(jb);
            else pthread_create(&th[t], NULL, ham_worker, jb);
        }
        int64_t nd = 0;
        for (int32_t t = 0; t < nthreads; t++) {
            if (nthreads > 1) pthread_join(th[t], NULL);
            nd += jobs[t].dist;
        }
        int64_t ch = 0;
        for (int64_t i = 0; i < n; i++) ch += (cur[i] != prev[i]);
        lko_refine_full(X, n, d, cur, k, C, Cn, NULL);
        /* drifts (bounds.py:31-35), top-2 for _max_other (pruners.py:58-67) */
        dmax1 = 0; dmax2 = 0; amax = -1;
        for (int32_t j = 0; j < k; j++) {
            lko_dist_row(Cn + (int64_t)j * d, C + (int64_t)j * d, 1, d, &drift[j], scr);
            drift[j] *= (1.0 + 1e-10);
            if (drift[j] > dmax1) { dmax2 = dmax1; dmax1 = drift[j]; amax = j; }
            else if (drift[j] > dmax2) dmax2 = drift[j];
        }
        memcpy(C, Cn, sizeof(double) * kd);
        if (history) memcpy(history + (int64_t)it * n, cur, sizeof(int64_t) * (size_t)n);
        if (changed_out) changed_out[it] = ch;
        if (dist_out) dist_out[it] = nd;
        memcpy(prev, cur, sizeof(int64_t) * (size_t)n);
        it++;
        if (ch == 0) { *converged = 1; break; }
    }
    memcpy(centroids_out, C, sizeof(double) * kd);
    if (labels_out) memcpy(labels_out, prev, sizeof(int64_t) * (size_t)n);
    free(C); free(Cn); free(s); free(drift); free(tmp); free(scr); free(prev); free(cur);
    free(ub); free(lb); free(th); free(jobs);
    return it;
}
