/*
 * multisplit_oracle.c -- plain, slow, obviously-correct CPU oracle for the
 * stable multisplit of arXiv 1701.01189 ("GPU Multisplit: an extended study of
 * a parallel algorithm", Ashkiani, Davidson, Meyer, Owens).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_1701_01189_b200/csrc); neither side includes or links the other.
 *
 * Citations: "P:nnn" = line of /root/reference/PAPER.md (LaTeX source).
 *
 *   orc_bucket          bucket identifiers: delta f(u)=floor(u/Delta)
 *                       (Sec.6 "Bucket identification"), identity
 *                       f(u)=u, radix digit
 *                       f_k(u)=(u>>kr)&(2^r-1) (Sec.7.1).
 *                       Delta clamps to m-1 (reading R7);
 *                       identity with u>=m is a domain error (reading R8).
 *                       Splitter buckets (Sec.6 "Bucket
 *                       identification"): f(u) = the j with s_j <= u <
 *                       s_{j+1}, where the caller gives the m-1 interior
 *                       splitters s_1 < ... < s_{m-1} and s_0 = 0, s_m = 2^32
 *                       are the ends of the uint32 key domain (DESIGN.md
 *                       reading R27), found by a textbook upper-bound
 *                       binary search (the search P:1110 names).
 *   orc_multisplit      stable multisplit = Eq.(1) (Sec.4.2):
 *                       p(i) = sum_{k<j} h_k + |{u_r in B_j : r < i}|,
 *                       computed as count -> exclusive scan -> stable
 *                       ascending scatter.  bucket_offsets has m+1 entries
 *                       (reading R2).  m <= 256 (the paper's scope).
 *   orc_multisplit_ex   the same Eq.(1) for every bucket kind including
 *                       splitters, and for m up to 65536 buckets (the m > 256
 *                       regime of Sec.6.3): the definition does
 *                       not depend on m, only the histogram array grows.
 *   orc_tile_histogram  the matrix H=[h_{j,l}] of Eq.(2) (Sec.4.3)
 *                       for L contiguous subproblems of T elements (last one
 *                       ragged), stored tile-major H[l*m + j].
 *   orc_global_scan     G = exclusive scan of row-vectorized H (P:291, P:777,
 *                       Alg.1 P:804-812 with the index typo read as i*L+j,
 *                       reading R3), returned in the same tile-major storage.
 *   orc_histogram_even  device-wide histogram, Even scenario (Sec.7.3,
 *                       P:1890): m buckets of width Delta = (s_m - s_0) / m
 *                       between s_0 and s_m; bucket of x = floor((x - s_0) /
 *                       Delta), all in IEEE binary32 round-to-nearest
 *                       (reading R25); x outside [s_0, s_m) or NaN is not
 *                       counted, a quotient of m (rounding at the top edge)
 *                       is clamped to m-1 (reading R26).
 *   orc_histogram_range device-wide histogram, Range scenario (Sec.7.3,
 *                       P:1891): splitters s_0 < ... < s_m; bucket of x = the
 *                       j with s_j <= x < s_{j+1}, found by the upper-bound
 *                       search the paper names, written here as a linear
 *                       count of splitters <= x (reading R26).
 *   orc_sssp            single-source shortest paths (Sec.7.2):
 *                       the minimum-cost path from the source to every
 *                       vertex, computed by Dijkstra's algorithm (P:1805,
 *                       a single priority queue, vertices settled from the
 *                       lowest to the highest distance) with a textbook binary
 *                       heap and lazy deletion; distances of unreachable
 *                       vertices are 0xFFFFFFFF; a reachable distance >=
 *                       2^32-1 is not representable (ORC_ERR_UNSUPPORTED).
 *   orc_radix_sort      the result of multisplit-sort (Sec.7.1):
 *                       a stable sort of (keys,values) by the key bits
 *                       [begin_bit, end_bit) as unsigned integers, written as
 *                       a plain stable merge sort (the plain definition of
 *                       what LSD stable passes produce, reading R10).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { ORC_OK = 0, ORC_ERR_INVALID = 1, ORC_ERR_UNSUPPORTED = 2,
       ORC_ERR_KEY_DOMAIN = 5 };
enum { ORC_IDENTITY = 0, ORC_DELTA = 1, ORC_RADIX = 2, ORC_SPLITTERS = 3 };
enum { ORC_MAX_M = 65536 };

/* Validation rules of the bucket function. */
int orc_validate(uint32_t kind, uint32_t m, uint64_t delta, uint32_t shift,
                 uint32_t bits) {
  if (m < 1 || m > 256) return ORC_ERR_UNSUPPORTED;  /* paper scope m<=256 */
  if (kind == ORC_IDENTITY) return ORC_OK;
  if (kind == ORC_DELTA) return delta >= 1 ? ORC_OK : ORC_ERR_INVALID;
  if (kind == ORC_RADIX) {
    if (bits < 1 || bits > 8) return ORC_ERR_INVALID;
    if ((uint64_t)shift + bits > 32) return ORC_ERR_INVALID;
    if (m != (1u << bits)) return ORC_ERR_INVALID;
    return ORC_OK;
  }
  return ORC_ERR_INVALID;
}

/* Bucket identifier f(u).  Returns ORC_OK and *b in [0,m), or
 * ORC_ERR_KEY_DOMAIN for an identity key outside [0,m). */
int orc_bucket(uint32_t kind, uint32_t m, uint64_t delta, uint32_t shift,
               uint32_t bits, uint32_t u, uint32_t *b) {
  if (kind == ORC_IDENTITY) {             /* f(u) = u */
    if (u >= m) return ORC_ERR_KEY_DOMAIN;
    *b = u;
    return ORC_OK;
  }
  if (kind == ORC_DELTA) {                /* f(u) = floor(u/D) */
    uint64_t q = (uint64_t)u / delta;     /* exact 64-bit integer division */
    *b = q < (uint64_t)(m - 1) ? (uint32_t)q : m - 1;
    return ORC_OK;
  }
  /* f_k(u) = (u >> kr) & (2^r - 1) */
  *b = (uint32_t)(((uint64_t)u >> shift) & ((1u << bits) - 1u));
  return ORC_OK;
}

/* Eq.(1): count, exclusive scan, stable scatter.  vals_in / vals_out may be
 * NULL (key-only).  offsets (m+1 entries) may be NULL. */
int orc_multisplit(const uint32_t *keys_in, const uint32_t *vals_in,
                   uint32_t *keys_out, uint32_t *vals_out, uint64_t n,
                   uint32_t kind, uint32_t m, uint64_t delta, uint32_t shift,
                   uint32_t bits, uint32_t *offsets) {
  int st = orc_validate(kind, m, delta, shift, bits);
  if (st) return st;
  uint64_t h[256], cur[256];
  memset(h, 0, sizeof h);
  /* histogram h_k: reduction of each bucket's membership */
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t b;
    st = orc_bucket(kind, m, delta, shift, bits, keys_in[i], &b);
    if (st) return st;
    h[b] += 1;
  }
  /* global offset: sum_{k<j} h_k (first term of Eq.1) */
  uint64_t run = 0;
  for (uint32_t j = 0; j < m; ++j) {
    if (offsets) offsets[j] = (uint32_t)run;
    cur[j] = run;
    run += h[j];
  }
  if (offsets) offsets[m] = (uint32_t)run;
  /* local offset: |{u_r in B_j : r < i}| (second term of Eq.1), obtained by
   * visiting i in ascending order */
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t b;
    orc_bucket(kind, m, delta, shift, bits, keys_in[i], &b);
    uint64_t p = cur[b]++;
    keys_out[p] = keys_in[i];
    if (vals_in && vals_out) vals_out[p] = vals_in[i];
  }
  return ORC_OK;
}

/* ------------------------------------------------------------- extended
 * Every bucket kind (splitters included) and 1 <= m <= 65536.  RADIX digits
 * may then be up to 16 bits wide.  spl: the m-1 interior splitters (may be
 * NULL when m = 1 or the kind is not ORC_SPLITTERS). */
int orc_validate_ex(uint32_t kind, uint32_t m, uint64_t delta, uint32_t shift,
                    uint32_t bits, const uint32_t *spl) {
  if (m < 1 || m > ORC_MAX_M) return ORC_ERR_UNSUPPORTED;
  if (kind == ORC_IDENTITY) return ORC_OK;
  if (kind == ORC_DELTA) return delta >= 1 ? ORC_OK : ORC_ERR_INVALID;
  if (kind == ORC_RADIX) {
    if (bits < 1 || bits > 16) return ORC_ERR_INVALID;
    if ((uint64_t)shift + bits > 32) return ORC_ERR_INVALID;
    if (m != (1u << bits)) return ORC_ERR_INVALID;
    return ORC_OK;
  }
  if (kind == ORC_SPLITTERS) {
    if (m > 1 && !spl) return ORC_ERR_INVALID;
    for (uint32_t j = 1; j + 1 < m; ++j)  /* s_1 < s_2 < ... < s_{m-1} */
      if (!(spl[j - 1] < spl[j])) return ORC_ERR_INVALID;
    return ORC_OK;
  }
  return ORC_ERR_INVALID;
}

/* Splitter bucket: the number of interior splitters <= u (upper bound over
 * s_1..s_{m-1}), i.e. the j with s_j <= u < s_{j+1} (reading R27). */
static uint32_t orc_splitter_bucket(const uint32_t *spl, uint32_t m, uint32_t u) {
  uint32_t lo = 0, hi = m - 1;  /* answer in [lo, hi]: count of spl[0..m-2] <= u */
  while (lo < hi) {
    uint32_t mid = lo + (hi - lo) / 2;  /* spl[mid] is s_{mid+1} */
    if (spl[mid] <= u)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

int orc_bucket_ex(uint32_t kind, uint32_t m, uint64_t delta, uint32_t shift,
                  uint32_t bits, const uint32_t *spl, uint32_t u, uint32_t *b) {
  if (kind == ORC_SPLITTERS) {
    *b = orc_splitter_bucket(spl, m, u);
    return ORC_OK;
  }
  if (kind == ORC_RADIX) {
    *b = (uint32_t)(((uint64_t)u >> shift) & ((1ull << bits) - 1ull));
    return ORC_OK;
  }
  return orc_bucket(kind, m, delta, shift, bits, u, b);
}

int orc_multisplit_ex(const uint32_t *keys_in, const uint32_t *vals_in,
                      uint32_t *keys_out, uint32_t *vals_out, uint64_t n,
                      uint32_t kind, uint32_t m, uint64_t delta, uint32_t shift,
                      uint32_t bits, const uint32_t *spl, uint32_t *offsets) {
  int st = orc_validate_ex(kind, m, delta, shift, bits, spl);
  if (st) return st;
  uint64_t *h = (uint64_t *)calloc(m, sizeof(uint64_t));
  uint64_t *cur = (uint64_t *)calloc(m, sizeof(uint64_t));
  if (!h || !cur) { free(h); free(cur); return ORC_ERR_INVALID; }
  for (uint64_t i = 0; i < n; ++i) {  /* h_k */
    uint32_t b;
    st = orc_bucket_ex(kind, m, delta, shift, bits, spl, keys_in[i], &b);
    if (st) { free(h); free(cur); return st; }
    h[b] += 1;
  }
  uint64_t run = 0;                   /* sum_{k<j} h_k */
  for (uint32_t j = 0; j < m; ++j) {
    if (offsets) offsets[j] = (uint32_t)run;
    cur[j] = run;
    run += h[j];
  }
  if (offsets) offsets[m] = (uint32_t)run;
  for (uint64_t i = 0; i < n; ++i) {  /* ascending i: |{u_r in B_j : r < i}| */
    uint32_t b;
    orc_bucket_ex(kind, m, delta, shift, bits, spl, keys_in[i], &b);
    uint64_t p = cur[b]++;
    keys_out[p] = keys_in[i];
    if (vals_in && vals_out) vals_out[p] = vals_in[i];
  }
  free(h);
  free(cur);
  return ORC_OK;
}

/* H = [h_{j,l}] of Eq.(2): per-subproblem bucket counts for L = ceil(n/T)
 * contiguous subproblems of T elements, stored tile-major H[l*m + j]. */
int orc_tile_histogram(const uint32_t *keys, uint64_t n, uint64_t T,
                       uint32_t kind, uint32_t m, uint64_t delta,
                       uint32_t shift, uint32_t bits, uint32_t *H) {
  int st = orc_validate(kind, m, delta, shift, bits);
  if (st) return st;
  if (T == 0) return ORC_ERR_INVALID;
  uint64_t L = (n + T - 1) / T;
  memset(H, 0, (size_t)(L * m) * sizeof(uint32_t));
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t b;
    st = orc_bucket(kind, m, delta, shift, bits, keys[i], &b);
    if (st) return st;
    H[(i / T) * m + b] += 1;
  }
  return ORC_OK;
}

/* G = exclusive scan of the row-vectorized H (rows = buckets):
 * H_row = [H[0][0:L-1], H[1][0:L-1], ...]; G_row = exclusive_scan(H_row).
 * Input/output in tile-major storage X[l*m + j] = X_{j,l}. */
void orc_global_scan(const uint32_t *H, uint64_t L, uint32_t m, uint32_t *G) {
  uint64_t run = 0;
  for (uint32_t j = 0; j < m; ++j)          /* row j = bucket j */
    for (uint64_t l = 0; l < L; ++l) {      /* column l = subproblem l */
      G[l * m + j] = (uint32_t)run;
      run += H[l * m + j];
    }
}

/* Stable sort of indices by digit d(i) = (keys[i] >> begin) & mask:
 * a textbook top-down merge sort (ties keep input order). */
static uint32_t orc_digit(uint32_t u, uint32_t begin, uint32_t end) {
  uint32_t w = end - begin;
  uint64_t mask = (w >= 32) ? 0xFFFFFFFFull : ((1ull << w) - 1ull);
  return (uint32_t)(((uint64_t)u >> begin) & mask);
}

static void orc_merge_sort(uint32_t *idx, uint32_t *tmp, uint64_t lo,
                           uint64_t hi, const uint32_t *keys, uint32_t begin,
                           uint32_t end) {
  if (hi - lo < 2) return;
  uint64_t mid = lo + (hi - lo) / 2;
  orc_merge_sort(idx, tmp, lo, mid, keys, begin, end);
  orc_merge_sort(idx, tmp, mid, hi, keys, begin, end);
  uint64_t a = lo, b = mid, o = lo;
  while (a < mid && b < hi) {
    /* take from the left run unless the right element is strictly smaller:
     * this is what keeps equal digits in input order (stability) */
    if (orc_digit(keys[idx[b]], begin, end) < orc_digit(keys[idx[a]], begin, end))
      tmp[o++] = idx[b++];
    else
      tmp[o++] = idx[a++];
  }
  while (a < mid) tmp[o++] = idx[a++];
  while (b < hi) tmp[o++] = idx[b++];
  memcpy(idx + lo, tmp + lo, (size_t)(hi - lo) * sizeof(uint32_t));
}

int orc_radix_sort(const uint32_t *keys_in, const uint32_t *vals_in,
                   uint32_t *keys_out, uint32_t *vals_out, uint64_t n,
                   uint32_t begin_bit, uint32_t end_bit) {
  if (begin_bit >= end_bit || end_bit > 32) return ORC_ERR_INVALID;
  if (n >= (1ull << 32)) return ORC_ERR_UNSUPPORTED;
  uint32_t *idx = (uint32_t *)malloc((size_t)(n ? n : 1) * sizeof(uint32_t));
  uint32_t *tmp = (uint32_t *)malloc((size_t)(n ? n : 1) * sizeof(uint32_t));
  if (!idx || !tmp) { free(idx); free(tmp); return ORC_ERR_INVALID; }
  for (uint64_t i = 0; i < n; ++i) idx[i] = (uint32_t)i;
  orc_merge_sort(idx, tmp, 0, n, keys_in, begin_bit, end_bit);
  for (uint64_t i = 0; i < n; ++i) {
    keys_out[i] = keys_in[idx[i]];
    if (vals_in && vals_out) vals_out[i] = vals_in[idx[i]];
  }
  free(idx);
  free(tmp);
  return ORC_OK;
}

/* ---------------------------------------------------------------- histogram
 * Sec.7.3.  counts[0..m) are overwritten.  Returns
 * ORC_ERR_UNSUPPORTED for m outside 1..256 (the paper's scope), ORC_ERR_INVALID
 * for empty or unordered bounds / splitters. */
int orc_histogram_even(const float *x, uint64_t n, uint32_t m, float lower, float upper,
                       uint32_t *counts) {
  if (m < 1 || m > 256) return ORC_ERR_UNSUPPORTED;
  if (!(lower < upper)) return ORC_ERR_INVALID;
  volatile float delta = (upper - lower) / (float)m; /* binary32, round to nearest */
  for (uint32_t j = 0; j < m; ++j) counts[j] = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const float v = x[i];
    if (!(v >= lower && v < upper)) continue; /* outside [s_0, s_m) or NaN */
    volatile float d = v - lower;
    volatile float q = d / delta;
    uint32_t b = (uint32_t)floorf(q);
    if (b > m - 1) b = m - 1;
    counts[b]++;
  }
  return ORC_OK;
}

int orc_histogram_range(const float *x, uint64_t n, uint32_t m, const float *s,
                        uint32_t *counts) {
  if (m < 1 || m > 256) return ORC_ERR_UNSUPPORTED;
  for (uint32_t j = 0; j < m; ++j)
    if (!(s[j] < s[j + 1])) return ORC_ERR_INVALID;
  for (uint32_t j = 0; j < m; ++j) counts[j] = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const float v = x[i];
    if (!(v >= s[0] && v < s[m])) continue;
    uint32_t le = 0; /* number of splitters <= v: upper_bound(s, s+m+1, v) - s */
    for (uint32_t j = 0; j <= m; ++j) le += s[j] <= v;
    counts[le - 1]++;
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------- SSSP
 * Sec.7.2.  CSR graph: row_ptr[V+1], col[E], w[E] (weights >= 0).
 * dist[V] receives the shortest distances from `source`. */
typedef struct { uint64_t d; uint32_t v; } orc_heap_item;

static void orc_heap_push(orc_heap_item *h, uint64_t *size, orc_heap_item x) {
  uint64_t i = (*size)++;
  h[i] = x;
  while (i > 0) {                          /* sift up */
    uint64_t p = (i - 1) / 2;
    if (h[p].d <= h[i].d) break;
    orc_heap_item t = h[p]; h[p] = h[i]; h[i] = t;
    i = p;
  }
}

static orc_heap_item orc_heap_pop(orc_heap_item *h, uint64_t *size) {
  orc_heap_item top = h[0];
  h[0] = h[--(*size)];
  uint64_t i = 0;
  for (;;) {                               /* sift down */
    uint64_t l = 2 * i + 1, r = l + 1, s = i;
    if (l < *size && h[l].d < h[s].d) s = l;
    if (r < *size && h[r].d < h[s].d) s = r;
    if (s == i) break;
    orc_heap_item t = h[s]; h[s] = h[i]; h[i] = t;
    i = s;
  }
  return top;
}

int orc_sssp(const uint32_t *row_ptr, const uint32_t *col, const uint32_t *w, uint32_t V,
             uint32_t source, uint32_t *dist) {
  if (V == 0 || source >= V) return ORC_ERR_INVALID;
  const uint64_t E = row_ptr[V];
  uint64_t *d = (uint64_t *)malloc((size_t)V * sizeof(uint64_t));
  unsigned char *done = (unsigned char *)calloc(V, 1);
  orc_heap_item *h = (orc_heap_item *)malloc((size_t)(E + 1) * sizeof(orc_heap_item));
  if (!d || !done || !h) { free(d); free(done); free(h); return ORC_ERR_INVALID; }
  for (uint32_t v = 0; v < V; ++v) d[v] = UINT64_MAX;
  uint64_t size = 0;
  d[source] = 0;
  orc_heap_push(h, &size, (orc_heap_item){0, source});
  while (size > 0) {
    orc_heap_item it = orc_heap_pop(h, &size);
    if (done[it.v] || it.d != d[it.v]) continue;   /* a stale queue entry */
    done[it.v] = 1;                                /* settled: lowest distance first */
    for (uint64_t e = row_ptr[it.v]; e < row_ptr[it.v + 1]; ++e) {
      const uint32_t u = col[e];
      const uint64_t nd = it.d + w[e];
      if (nd < d[u]) {                             /* relaxation */
        d[u] = nd;
        orc_heap_push(h, &size, (orc_heap_item){nd, u});
      }
    }
  }
  int st = ORC_OK;
  for (uint32_t v = 0; v < V; ++v) {
    if (d[v] == UINT64_MAX) dist[v] = 0xFFFFFFFFu;
    else if (d[v] >= 0xFFFFFFFFull) st = ORC_ERR_UNSUPPORTED;
    else dist[v] = (uint32_t)d[v];
  }
  free(d); free(done); free(h);
  return st;
}
