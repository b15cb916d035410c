/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_2506_03296_b200/) never links, imports or calls it, and this file
 * shares no code, header or constant with the CUDA path.
 *
 * Plain float64 decode-phase attention over a LOGICAL, contiguous KV cache
 * (no block tables: paging bugs on the GPU side show up as mismatches).
 *
 * What it computes (the definition; DESIGN.md "Readings" c1-c5):
 *   PAPER.md P:49-53 (§2.1): decode = one new token per step; each layer caches
 *     one K and one V vector per token; attention of the new token's query
 *     against the cache.  P:51: GQA shares K/V projections across query heads.
 *   The formula softmax(q.K^T/sqrt(d)).V is stated by BASELINE.json north_star
 *   (PAPER.md never writes it).  For request b, q-head h,
 *   kv-head g(h) = floor(h / (Hq/Hkv)), context n_b >= 1:
 *       s_t   = scale * sum_d q[b,h,d] * K[b,g,t,d]          t = 0..n_b-1
 *       m     = max_t s_t
 *       w_t   = exp(s_t - m) / sum_u exp(s_u - m)
 *       out_d = sum_t w_t * V[b,g,t,d]
 *   Inputs are exact fp32/fp16/bf16 values widened to double by the decoders
 *   below (written from the IEEE-754 / bfloat16 field definitions); the output
 *   stays double.  Plain scalar loops, no fast-math, no blocking or reordering.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { OR_F32 = 0, OR_F16 = 1, OR_BF16 = 2, OR_F64 = 3 };

/* bfloat16 = upper 16 bits of an IEEE binary32 */
static double dec_bf16(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return (double)f;
}

/* IEEE binary16: sign | 5-bit exponent (bias 15) | 10-bit fraction */
static double dec_f16(uint16_t h) {
    int sign = h >> 15, e = (h >> 10) & 0x1f, m = h & 0x3ff;
    double v;
    if (e == 0)
        v = ldexp((double)m, -24);               /* subnormal: m * 2^-24 */
    else if (e == 31)
        v = m ? NAN : INFINITY;
    else
        v = ldexp((double)(1024 + m), e - 25);   /* (1 + m/2^10) * 2^(e-15) */
    return sign ? -v : v;
}

static double load(const void *p, int dtype, size_t i) {
    switch (dtype) {
    case OR_F32: return (double)((const float *)p)[i];
    case OR_F16: return dec_f16(((const uint16_t *)p)[i]);
    case OR_BF16: return dec_bf16(((const uint16_t *)p)[i]);
    default: return ((const double *)p)[i];
    }
}

/* softmax weights w[0..n) of one (request, q-head) row; returns 0 */
static void row_weights(int dtype, const void *q, size_t q_off, const void *k, int64_t n,
                        int Hkv, int g, int D, double scale, double *w) {
    for (int64_t t = 0; t < n; ++t) {
        double dot = 0.0;
        for (int d = 0; d < D; ++d)
            dot += load(q, dtype, q_off + d) * load(k, dtype, ((size_t)t * Hkv + g) * D + d);
        w[t] = scale * dot;                                   /* s_t */
    }
    double m = -INFINITY;
    for (int64_t t = 0; t < n; ++t)
        if (w[t] > m) m = w[t];                               /* m = max_t s_t */
    double z = 0.0;
    for (int64_t t = 0; t < n; ++t) {
        w[t] = exp(w[t] - m);
        z += w[t];                                            /* sum_u exp(s_u - m) */
    }
    for (int64_t t = 0; t < n; ++t) w[t] /= z;                /* w_t */
}

static void attend_row(int dtype, const void *q, size_t q_off, const void *k, const void *v,
                       int64_t n, int Hkv, int g, int D, double scale, double *w, double *out) {
    row_weights(dtype, q, q_off, k, n, Hkv, g, D, scale, w);
    for (int d = 0; d < D; ++d) out[d] = 0.0;
    for (int64_t t = 0; t < n; ++t)
        for (int d = 0; d < D; ++d)
            out[d] += w[t] * load(v, dtype, ((size_t)t * Hkv + g) * D + d);  /* sum_t w_t V_t */
}

typedef struct {
    int dtype;
    const void *q;
    const void *const *k;
    const void *const *v;
    const int64_t *n;
    int Hq, Hkv, D;
    double scale;
    const int64_t *rows;
    int64_t r0, r1;
    double *out;
    int status;
} job_t;

static void *worker(void *arg) {
    job_t *j = (job_t *)arg;
    int64_t nmax = 1;
    for (int64_t r = j->r0; r < j->r1; ++r) {
        int64_t row = j->rows ? j->rows[r] : r;
        int64_t nb = j->n[row / j->Hq];
        if (nb > nmax) nmax = nb;
    }
    double *w = (double *)malloc(sizeof(double) * (size_t)nmax);
    if (!w) { j->status = -2; return NULL; }
    int group = j->Hq / j->Hkv;
    for (int64_t r = j->r0; r < j->r1; ++r) {
        int64_t row = j->rows ? j->rows[r] : r;
        int64_t b = row / j->Hq;
        int h = (int)(row % j->Hq);
        attend_row(j->dtype, j->q, (size_t)row * j->D, j->k[b], j->v[b], j->n[b], j->Hkv,
                   h / group, j->D, j->scale, w, j->out + (size_t)r * j->D);
    }
    free(w);
    return NULL;
}

/*
 * q:    [B][Hq][D] in `dtype`;  k[b], v[b]: [n[b]][Hkv][D] in `dtype` (logical order)
 * rows: optional list of row ids b*Hq+h (NULL = all B*Hq rows, in order)
 * out:  [n_rows][D] float64
 * Returns 0, -1 on invalid arguments, -2 on allocation failure.
 */
int oracle_decode_attention(int dtype, const void *q, const void *const *k, const void *const *v,
                            const int64_t *n, int B, int Hq, int Hkv, int D, double scale,
                            const int64_t *rows, int64_t n_rows, double *out, int nthreads) {
    if (B < 0 || Hq <= 0 || Hkv <= 0 || D <= 0 || Hq % Hkv != 0 || dtype < 0 || dtype > 3)
        return -1;
    if (!rows) n_rows = (int64_t)B * Hq;
    for (int64_t r = 0; r < n_rows; ++r) {
        int64_t row = rows ? rows[r] : r;
        if (row < 0 || row >= (int64_t)B * Hq || n[row / Hq] < 1) return -1;   /* ctx >= 1 (c4) */
    }
    if (nthreads < 1) nthreads = 1;
    if (nthreads > n_rows) nthreads = n_rows > 0 ? (int)n_rows : 1;
    job_t *jobs = (job_t *)calloc((size_t)nthreads, sizeof(job_t));
    pthread_t *tid = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    if (!jobs || !tid) { free(jobs); free(tid); return -2; }
    for (int i = 0; i < nthreads; ++i) {
        job_t j = {dtype, q, k, v, n, Hq, Hkv, D, scale, rows,
                   n_rows * i / nthreads, n_rows * (i + 1) / nthreads, out, 0};
        jobs[i] = j;
    }
    for (int i = 1; i < nthreads; ++i) pthread_create(&tid[i], NULL, worker, &jobs[i]);
    worker(&jobs[0]);
    int status = jobs[0].status;
    for (int i = 1; i < nthreads; ++i) {
        pthread_join(tid[i], NULL);
        if (jobs[i].status) status = jobs[i].status;
    }
    free(jobs);
    free(tid);
    return status;
}

/* softmax weights of one row (for the "weights sum to 1" pin); w: [n] */
int oracle_attention_weights(int dtype, const void *q_row, const void *k, int64_t n, int Hkv,
                             int g, int D, double scale, double *w) {
    if (n < 1 || g < 0 || g >= Hkv) return -1;
    row_weights(dtype, q_row, 0, k, n, Hkv, g, D, scale, w);
    return 0;
}

/* element decoders exposed for the dtype pins (tests/test_oracle.py) */
double oracle_decode_f16(uint16_t h) { return dec_f16(h); }
double oracle_decode_bf16(uint16_t h) { return dec_bf16(h); }
