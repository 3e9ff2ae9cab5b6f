/* cpu_multisplit.c -- parallel CPU baseline for bench.py (not the oracle, not
 * the product): the paper's {local, global, local} structure on
 * host threads.  Thread t owns a contiguous chunk; (1) it counts its chunk's
 * bucket histogram, (2) one exclusive scan over (bucket, thread) gives every
 * thread the start of its part of each bucket (Eq.2 with threads as
 * subproblems), (3) every thread scatters its chunk stably.  Bucket function:
 * DELTA min(u / delta, m - 1) or RADIX (u >> shift) & (2^bits - 1).
 * Build: gcc -O3 -march=native -shared -fPIC -pthread. */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  const uint32_t *k, *v;
  uint32_t *ko, *vo;
  uint64_t lo, hi;
  uint32_t m, kind, delta, shift, mask;
  uint64_t *cnt; /* [m] counts, then starts */
} job_t;

static inline uint32_t bkt(const job_t *j, uint32_t u) {
  if (j->kind == 2) return (u >> j->shift) & j->mask;
  uint32_t q = u / j->delta;
  return q < j->m - 1 ? q : j->m - 1;
}

static void *count_fn(void *p) {
  job_t *j = (job_t *)p;
  memset(j->cnt, 0, sizeof(uint64_t) * j->m);
  for (uint64_t i = j->lo; i < j->hi; ++i) j->cnt[bkt(j, j->k[i])]++;
  return NULL;
}

static void *scatter_fn(void *p) {
  job_t *j = (job_t *)p;
  for (uint64_t i = j->lo; i < j->hi; ++i) {
    const uint64_t d = j->cnt[bkt(j, j->k[i])]++;
    j->ko[d] = j->k[i];
    if (j->v) j->vo[d] = j->v[i];
  }
  return NULL;
}

/* kind: 1 = DELTA (delta), 2 = RADIX (shift, bits).  Returns 0 on success. */
int cpu_multisplit(const uint32_t *keys, const uint32_t *vals, uint32_t *keys_out, uint32_t *vals_out,
                   uint64_t n, uint32_t m, uint32_t kind, uint32_t delta, uint32_t shift, uint32_t bits,
                   int nthreads) {
  if (nthreads < 1 || m < 1) return 1;
  job_t *jobs = calloc(nthreads, sizeof(job_t));
  pthread_t *th = calloc(nthreads, sizeof(pthread_t));
  uint64_t *cnt = calloc((size_t)nthreads * m, sizeof(uint64_t));
  if (!jobs || !th || !cnt) return 2;
  for (int t = 0; t < nthreads; ++t) {
    job_t *j = &jobs[t];
    j->k = keys; j->v = vals; j->ko = keys_out; j->vo = vals_out;
    j->lo = n * t / nthreads; j->hi = n * (t + 1) / nthreads;
    j->m = m; j->kind = kind; j->delta = delta ? delta : 1; j->shift = shift;
    j->mask = bits >= 32 ? 0xFFFFFFFFu : ((1u << bits) - 1u);
    j->cnt = cnt + (size_t)t * m;
    pthread_create(&th[t], NULL, count_fn, j);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  uint64_t run = 0; /* exclusive scan in (bucket, thread) order */
  for (uint32_t b = 0; b < m; ++b)
    for (int t = 0; t < nthreads; ++t) {
      const uint64_t c = cnt[(size_t)t * m + b];
      cnt[(size_t)t * m + b] = run;
      run += c;
    }
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, scatter_fn, &jobs[t]);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(jobs); free(th); free(cnt);
  return 0;
}

/* LSD radix sort with r-bit digits built on cpu_multisplit (ping-pong). */
int cpu_radix_sort(const uint32_t *keys, const uint32_t *vals, uint32_t *keys_out, uint32_t *vals_out,
                   uint64_t n, uint32_t r, int nthreads) {
  uint32_t *tk = malloc(n * 4), *tv = vals ? malloc(n * 4) : NULL;
  if (!tk || (vals && !tv)) return 2;
  const int passes = (32 + r - 1) / r;
  const uint32_t *sk = keys, *sv = vals;
  for (int p = 0; p < passes; ++p) {
    const int to_out = ((passes - 1 - p) % 2) == 0;
    uint32_t *dk = to_out ? keys_out : tk, *dv = to_out ? vals_out : tv;
    const uint32_t b = (32 - p * r) < r ? (32 - p * r) : r;
    cpu_multisplit(sk, sv, dk, dv, n, 1u << b, 2, 0, p * r, b, nthreads);
    sk = dk; sv = dv;
  }
  free(tk); free(tv);
  return 0;
}
