/*
 * oracle/attention_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct fp64 attention used to check the CUDA path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library.  It shares no code, header, table or
 * constant with paper_2511_12056_b200/ (the product), and the product never
 * calls it.
 *
 * What it computes -- the plain definition of the method's result:
 *   PipeSP is exact attention, resharded ("Psi T^mod = T^orig",
 *   PAPER.md:736 "the generated videos are identical"); the per-head operation
 *   is Alg. 1 line 3 `attention(Q[:,j],K[:,j],V[:,j])`, i.e.
 *   softmax(Q K^T / sqrt(D)) V with the 1/sqrt(D) scale fixed by BASELINE.json
 *   north_star (the paper never states it; reading R1).
 *
 * For one head and one query row q (length D) against keys K[S][D], values V[S][D]:
 *   z[t]   = ( sum_{d ascending} q[d]*K[t][d] ) / sqrt(D)
 *   m      = max_t z[t]
 *   e[t]   = exp(z[t] - m)
 *   l      = sum_{t ascending} e[t]
 *   O[d]   = sum_{t ascending} (e[t] / l) * V[t][d]
 * All in IEEE fp64, no reassociation (compile WITHOUT -ffast-math), so the
 * result is a pure function of (q, K, V): identical inputs give identical bits
 * no matter which rank / stage / thread evaluated the row.
 *
 * Threads (pthreads) only split independent query rows; each row is computed
 * start to finish by one thread in the order above.
 */
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/*
 * Softmax weights w[t] = e[t]/l of one row.  key_valid (NULL = every key valid) is the key-padding
 * mask of Alg. 1's `attention(Q[:,j], K[:,j], V[:,j], attention_mask[:,j])` (the
 * paper never defines it -- DESIGN.md reading R2/R20): a masked key takes no part in the softmax,
 * i.e. z[t] = -inf, e[t] = 0.  A row with no valid key gets w = 0 everywhere (its output is 0).
 */
static int softmax_weights_lse(const double *q, const double *K, long S, long D, const unsigned char *key_valid,
                               double *w, double *lse_out);

int oracle_softmax_weights_masked(const double *q, const double *K, long S, long D, const unsigned char *key_valid,
                                  double *w)
{
    return softmax_weights_lse(q, K, S, D, key_valid, w, NULL);
}

/* ... and lse = ln sum_t exp(z[t]) = m + ln l over the valid keys (-inf if none): the quantity two partial
 * softmaxes over disjoint key blocks are combined with (ring attention, R21). */
static int softmax_weights_lse(const double *q, const double *K, long S, long D, const unsigned char *key_valid,
                               double *w, double *lse_out)
{
    if (!q || !K || !w || S <= 0 || D <= 0) return 1;
    double sqrt_d = sqrt((double)D);
    double m = -INFINITY;
    for (long t = 0; t < S; ++t) {
        if (key_valid && !key_valid[t]) { w[t] = -INFINITY; continue; }
        double acc = 0.0;
        for (long d = 0; d < D; ++d) acc += q[d] * K[t * D + d];
        w[t] = acc / sqrt_d;
        if (w[t] > m) m = w[t];
    }
    if (m == -INFINITY) {           /* no valid key */
        for (long t = 0; t < S; ++t) w[t] = 0.0;
        if (lse_out) *lse_out = -INFINITY;
        return 0;
    }
    double l = 0.0;
    for (long t = 0; t < S; ++t) {
        w[t] = (w[t] == -INFINITY) ? 0.0 : exp(w[t] - m);
        l += w[t];
    }
    for (long t = 0; t < S; ++t) w[t] = w[t] / l;
    if (lse_out) *lse_out = m + log(l);
    return 0;
}

int oracle_softmax_weights(const double *q, const double *K, long S, long D, double *w)
{
    return oracle_softmax_weights_masked(q, K, S, D, NULL, w);
}

/* One output row: out[D] = sum_t w[t] V[t,:] (t ascending). scratch has S doubles. */
static void attention_one_row(const double *q, const double *K, const double *V, long S, long D,
                              const unsigned char *key_valid, double *out, double *lse, double *scratch)
{
    softmax_weights_lse(q, K, S, D, key_valid, scratch, lse);
    for (long d = 0; d < D; ++d) out[d] = 0.0;
    for (long t = 0; t < S; ++t) {
        double wt = scratch[t];
        const double *vt = V + t * D;
        for (long d = 0; d < D; ++d) out[d] += wt * vt[d];
    }
}

typedef struct {
    const double *Q, *K, *V;
    const unsigned char *key_valid;
    double *O;
    double *lse;     /* optional [nq] */
    long nq, S, D;
    long q_stride, o_stride; /* elements between consecutive query / output rows */
    int tid, nthreads;
    int err;
} rows_job;

static void *rows_worker(void *arg)
{
    rows_job *j = (rows_job *)arg;
    double *scratch = (double *)malloc(sizeof(double) * (size_t)j->S);
    if (!scratch) { j->err = 2; return NULL; }
    for (long r = j->tid; r < j->nq; r += j->nthreads)
        attention_one_row(j->Q + r * j->q_stride, j->K, j->V, j->S, j->D, j->key_valid, j->O + r * j->o_stride,
                          j->lse ? j->lse + r : NULL, scratch);
    free(scratch);
    return NULL;
}

/*
 * out[r][:] = attention(Q[r][:], K, V) for r < nq, over the keys with key_valid[t] != 0
 * (key_valid NULL = all keys).  Q rows at stride q_stride, out rows at o_stride; K, V dense [S][D].
 * nthreads <= 0 -> 1.  Returns 0 on success.
 */
int oracle_attention_rows_lse(const double *Q, long nq, long q_stride, const double *K, const double *V,
                              long S, long D, const unsigned char *key_valid, double *out, long o_stride,
                              double *lse, int nthreads);

int oracle_attention_rows_masked(const double *Q, long nq, long q_stride, const double *K, const double *V,
                                 long S, long D, const unsigned char *key_valid, double *out, long o_stride,
                                 int nthreads)
{
    return oracle_attention_rows_lse(Q, nq, q_stride, K, V, S, D, key_valid, out, o_stride, NULL, nthreads);
}

/* As above, and lse[r] = ln sum_t exp(z[r][t]) over the valid keys (lse may be NULL). */
int oracle_attention_rows_lse(const double *Q, long nq, long q_stride, const double *K, const double *V,
                              long S, long D, const unsigned char *key_valid, double *out, long o_stride,
                              double *lse, int nthreads)
{
    if (!Q || !K || !V || !out || S <= 0 || D <= 0 || nq < 0) return 1;
    if (nthreads <= 0) nthreads = 1;
    if (nthreads > nq) nthreads = nq > 0 ? (int)nq : 1;
    rows_job *jobs = (rows_job *)calloc((size_t)nthreads, sizeof(rows_job));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    if (!jobs || !th) { free(jobs); free(th); return 2; }
    for (int i = 0; i < nthreads; ++i) {
        jobs[i] = (rows_job){Q, K, V, key_valid, out, lse, nq, S, D, q_stride, o_stride, i, nthreads, 0};
        if (nthreads == 1) rows_worker(&jobs[i]);
        else pthread_create(&th[i], NULL, rows_worker, &jobs[i]);
    }
    int err = 0;
    for (int i = 0; i < nthreads; ++i) {
        if (nthreads > 1) pthread_join(th[i], NULL);
        if (jobs[i].err) err = jobs[i].err;
    }
    free(jobs);
    free(th);
    return err;
}

int oracle_attention_rows(const double *Q, long nq, long q_stride, const double *K, const double *V,
                          long S, long D, double *out, long o_stride, int nthreads)
{
    return oracle_attention_rows_masked(Q, nq, q_stride, K, V, S, D, NULL, out, o_stride, nthreads);
}
