// ms_capi.cu -- the extern "C" boundary of libms (include/multisplit.h):
// argument validation, workspace carving, strategy dispatch and the LSD
// radix-sort pass driver.  All launches are stream-ordered; nothing here
// synchronizes except ms_device_status.
#include <atomic>
#include <cstdlib>
#include <cstring>

#include "../../include/multisplit.h"
#include "ms_dispatch.cuh"
#include "ms_scan.cuh"

namespace ms {
template <int KIND>
cudaError_t launch_prescan(int, int, const uint32_t *, uint32_t, const BucketParams &,
                           uint32_t *, unsigned long long *, uint32_t, uint32_t *, cudaStream_t);
template <int KIND>
cudaError_t launch_postscan(int, int, bool, const KsArgs &, const BucketParams &, uint32_t,
                            cudaStream_t);
}  // namespace ms

using namespace ms;

namespace {

thread_local void *const *g_stage_events = nullptr;
std::atomic<unsigned long long> g_launches{0};

void stage_event(int i, cudaStream_t s) {
  if (g_stage_events) cudaEventRecord((cudaEvent_t)g_stage_events[i], s);
}

cudaError_t counted(cudaError_t e, unsigned k = 1) {
  if (e == cudaSuccess) g_launches.fetch_add(k, std::memory_order_relaxed);
  return e;
}

constexpr size_t kAlign = 256;
constexpr size_t kHdrBytes = 256;   // [0] error flag, [1] scan ticket
constexpr size_t kBaseBytes = 1280; // m+1 <= 257 words

size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

uint32_t ceil_log2(uint32_t m) {
  uint32_t l = 0;
  while ((1u << l) < m) ++l;
  return l;
}

// tiles per look-back chunk: ~4096 H words per scan CTA
uint32_t scan_chunk_tiles(uint32_t m) {
  uint32_t c = 4096u / m;
  return c < 1 ? 1 : c;
}

struct Layout {
  size_t base, H, status, total;
  uint32_t L, nchunks, C;
};

Layout layout_for(uint64_t n, uint32_t m) {
  Layout lo{};
  lo.base = kHdrBytes;
  if (n <= (uint64_t)kTile) {  // single-CTA path: header only
    lo.H = lo.status = lo.total = kHdrBytes + kBaseBytes;
    lo.L = n ? 1 : 0;
    lo.nchunks = 0;
    lo.C = 0;
    return lo;
  }
  lo.L = (uint32_t)((n + kTile - 1) / kTile);
  lo.C = scan_chunk_tiles(m);
  lo.nchunks = (lo.L + lo.C - 1) / lo.C;
  lo.H = kHdrBytes + kBaseBytes;
  lo.status = lo.H + align_up((size_t)lo.L * m * 4u);
  lo.total = lo.status + align_up((size_t)lo.nchunks * m * 8u);
  return lo;
}

ms_status validate_fn(const ms_bucket_fn *fn) {
  if (!fn) return MS_ERR_INVALID_VALUE;
  const uint32_t m = fn->num_buckets;
  if (m < 1 || m > 256) return MS_ERR_UNSUPPORTED;
  switch (fn->kind) {
    case MS_BUCKET_IDENTITY: return MS_SUCCESS;
    case MS_BUCKET_DELTA: return fn->delta >= 1 ? MS_SUCCESS : MS_ERR_INVALID_VALUE;
    case MS_BUCKET_RADIX:
      if (fn->bits < 1 || fn->bits > 8) return MS_ERR_INVALID_VALUE;
      if ((uint64_t)fn->shift + fn->bits > 32) return MS_ERR_INVALID_VALUE;
      if (m != (1u << fn->bits)) return MS_ERR_INVALID_VALUE;
      return MS_SUCCESS;
    default: return MS_ERR_INVALID_VALUE;
  }
}

BucketParams make_params(const ms_bucket_fn *fn) {
  BucketParams p{};
  p.m = fn->num_buckets;
  p.m1 = fn->num_buckets - 1;
  p.shift = fn->shift;
  p.mask = fn->kind == MS_BUCKET_RADIX ? ((1u << fn->bits) - 1u) : 0u;
  if (fn->kind == MS_BUCKET_DELTA) {
    p.delta_is_one = fn->delta == 1;
    if (!p.delta_is_one) {
      // M = ceil(2^64 / delta) = floor((2^64 - 1) / delta) + 1  (delta >= 2)
      const unsigned long long M = ~0ull / fn->delta + 1ull;
      p.magic_hi = (uint32_t)(M >> 32);
      p.magic_lo = (uint32_t)M;
    }
  }
  return p;
}

int env_strategy(const char *name, int dflt) {
  const char *v = std::getenv(name);
  if (!v || !*v) return dflt;
  if (!std::strcmp(v, "count1")) return kCount1;
  if (!std::strcmp(v, "peers") || !std::strcmp(v, "ballot")) return kPeers;
  if (!std::strcmp(v, "match")) return kMatch;
  if (!std::strcmp(v, "atomic")) return kAtomic;
  return dflt;
}

// Per-m strategy table; env overrides for the bench only.
int hist_strategy(uint32_t m) {
  int s = env_strategy("MS_HIST", m <= 2 ? kCount1 : kPeers);
  if (s == kCount1 && m > 2) s = kPeers;
  return s;
}
int rank_strategy(uint32_t m) {
  int s = env_strategy("MS_RANK", m <= 2 ? kCount1 : kPeers);
  if (s == kCount1 && m > 2) s = kPeers;
  if (s == kAtomic) s = kPeers;
  return s;
}

bool overlaps(const void *a, const void *b, uint64_t n) {
  if (!a || !b || n == 0) return false;
  const char *pa = (const char *)a, *pb = (const char *)b;
  const uint64_t bytes = n * 4u;
  return pa < pb + bytes && pb < pa + bytes;
}

cudaError_t prescan_dispatch(uint32_t kind, int strat, int logm, const uint32_t *keys, uint32_t n,
                             const BucketParams &bp, uint32_t *H, unsigned long long *zs,
                             uint32_t zw, uint32_t *hdr, cudaStream_t s) {
  switch (kind) {
    case MS_BUCKET_IDENTITY:
      return launch_prescan<kIdentity>(strat, logm, keys, n, bp, H, zs, zw, hdr, s);
    case MS_BUCKET_DELTA:
      return launch_prescan<kDelta>(strat, logm, keys, n, bp, H, zs, zw, hdr, s);
    default: return launch_prescan<kRadix>(strat, logm, keys, n, bp, H, zs, zw, hdr, s);
  }
}

cudaError_t postscan_dispatch(uint32_t kind, int strat, int logm, bool pairs, const KsArgs &a,
                              const BucketParams &bp, uint32_t grid, cudaStream_t s) {
  switch (kind) {
    case MS_BUCKET_IDENTITY: return launch_postscan<kIdentity>(strat, logm, pairs, a, bp, grid, s);
    case MS_BUCKET_DELTA: return launch_postscan<kDelta>(strat, logm, pairs, a, bp, grid, s);
    default: return launch_postscan<kRadix>(strat, logm, pairs, a, bp, grid, s);
  }
}

ms_status multisplit_impl(const uint32_t *keys_in, const uint32_t *vals_in, uint32_t *keys_out,
                          uint32_t *vals_out, uint64_t n, const ms_bucket_fn *fn,
                          uint32_t *bucket_offsets, void *ws, size_t ws_bytes, void *stream,
                          bool pairs) {
  ms_status st = validate_fn(fn);
  if (st != MS_SUCCESS) return st;
  if (n >= (1ull << 32)) return MS_ERR_UNSUPPORTED;
  const uint32_t m = fn->num_buckets;
  if (!ws) return MS_ERR_INVALID_VALUE;
  if (n > 0) {
    if (!keys_in || !keys_out) return MS_ERR_INVALID_VALUE;
    if (pairs && (!vals_in || !vals_out)) return MS_ERR_INVALID_VALUE;
    if (overlaps(keys_in, keys_out, n)) return MS_ERR_INVALID_VALUE;
    if (pairs && (overlaps(vals_in, vals_out, n) || overlaps(keys_in, vals_out, n) ||
                  overlaps(vals_in, keys_out, n) || overlaps(keys_out, vals_out, n)))
      return MS_ERR_INVALID_VALUE;
  }
  const Layout lo = layout_for(n, m);
  if (ws_bytes < lo.total) return MS_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  char *w = (char *)ws;
  uint32_t *hdr = (uint32_t *)w;

  if (n == 0) {
    if (cudaMemsetAsync(hdr, 0, 8, s) != cudaSuccess) return MS_ERR_CUDA;
    if (bucket_offsets && cudaMemsetAsync(bucket_offsets, 0, (m + 1) * 4u, s) != cudaSuccess)
      return MS_ERR_CUDA;
    return MS_SUCCESS;
  }

  const BucketParams bp = make_params(fn);
  const int logm = m <= 2 ? 1 : (int)ceil_log2(m);
  const int hs = hist_strategy(m), rs = rank_strategy(m);
  KsArgs a{};
  a.keys_in = keys_in;
  a.vals_in = pairs ? vals_in : nullptr;
  a.keys_out = keys_out;
  a.vals_out = pairs ? vals_out : nullptr;
  a.n = (uint32_t)n;
  a.hdr = hdr;
  a.bucket_offsets = bucket_offsets;
  a.use_tma = (((uintptr_t)keys_in & 15u) == 0) && (!pairs || (((uintptr_t)vals_in & 15u) == 0));

  if (n <= (uint64_t)kTile) {  // one subproblem: a single fused launch
    a.single = 1;
    stage_event(0, s);
    stage_event(1, s);
    stage_event(2, s);
    const cudaError_t e = counted(postscan_dispatch(fn->kind, rs, logm, pairs, a, bp, 1, s));
    stage_event(3, s);
    return e == cudaSuccess ? MS_SUCCESS : MS_ERR_CUDA;
  }

  uint32_t *base = (uint32_t *)(w + lo.base);
  uint32_t *H = (uint32_t *)(w + lo.H);
  unsigned long long *status = (unsigned long long *)(w + lo.status);
  stage_event(0, s);
  if (counted(prescan_dispatch(fn->kind, hs, logm, keys_in, (uint32_t)n, bp, H, status,
                               lo.nchunks * m, hdr, s)) != cudaSuccess)
    return MS_ERR_CUDA;
  stage_event(1, s);
  kg_scan<<<lo.nchunks, kScanThreads, 0, s>>>(H, H, lo.L, m, lo.C, lo.nchunks, status, hdr + 1,
                                               base, bucket_offsets);
  if (counted(cudaGetLastError()) != cudaSuccess) return MS_ERR_CUDA;
  stage_event(2, s);
  a.single = 0;
  a.G = H;
  a.base = base;
  const cudaError_t e = counted(postscan_dispatch(fn->kind, rs, logm, pairs, a, bp, lo.L, s));
  stage_event(3, s);
  return e == cudaSuccess ? MS_SUCCESS : MS_ERR_CUDA;
}

ms_status radix_impl(const uint32_t *keys_in, const uint32_t *vals_in, uint32_t *keys_out,
                     uint32_t *vals_out, uint64_t n, uint32_t begin_bit, uint32_t end_bit,
                     uint32_t r, void *ws, size_t ws_bytes, void *stream, bool pairs) {
  uint32_t shifts[32], bits[32];
  const int passes = ms_radix_pass_schedule(begin_bit, end_bit, r, shifts, bits, 32);
  if (passes < 0) return MS_ERR_INVALID_VALUE;
  if (n >= (1ull << 32)) return MS_ERR_UNSUPPORTED;
  if (!ws) return MS_ERR_INVALID_VALUE;
  if (n == 0) return MS_SUCCESS;
  if (!keys_in || !keys_out || (pairs && (!vals_in || !vals_out))) return MS_ERR_INVALID_VALUE;
  if (overlaps(keys_in, keys_out, n)) return MS_ERR_INVALID_VALUE;
  if (pairs && (overlaps(vals_in, vals_out, n) || overlaps(keys_out, vals_out, n) ||
                overlaps(keys_in, vals_out, n) || overlaps(vals_in, keys_out, n)))
    return MS_ERR_INVALID_VALUE;
  if (ws_bytes < ms_radix_sort_workspace_size(n, pairs)) return MS_ERR_WORKSPACE;
  const size_t ms_bytes = ms_multisplit_workspace_size(n, 1u << r, pairs);
  char *w = (char *)ws;
  uint32_t *alt_k = (uint32_t *)(w + align_up(ms_bytes));
  uint32_t *alt_v = pairs ? (uint32_t *)((char *)alt_k + align_up(n * 4u)) : nullptr;
  // ping-pong so that the last pass lands in the output: ... alt -> out
  const uint32_t *src_k = keys_in, *src_v = vals_in;
  for (int p = 0; p < passes; ++p) {
    const bool to_out = ((passes - 1 - p) % 2) == 0;
    uint32_t *dk = to_out ? keys_out : alt_k;
    uint32_t *dv = to_out ? vals_out : alt_v;
    ms_bucket_fn fn{MS_BUCKET_RADIX, 1u << bits[p], 0u, shifts[p], bits[p]};
    ms_status st = multisplit_impl(src_k, src_v, dk, dv, n, &fn, nullptr, w, ms_bytes, stream,
                                   pairs);
    if (st != MS_SUCCESS) return st;
    src_k = dk;
    src_v = dv;
  }
  return MS_SUCCESS;
}

}  // namespace

extern "C" {

const char *ms_status_string(ms_status s) {
  switch (s) {
    case MS_SUCCESS: return "MS_SUCCESS";
    case MS_ERR_INVALID_VALUE: return "MS_ERR_INVALID_VALUE";
    case MS_ERR_UNSUPPORTED: return "MS_ERR_UNSUPPORTED";
    case MS_ERR_WORKSPACE: return "MS_ERR_WORKSPACE";
    case MS_ERR_CUDA: return "MS_ERR_CUDA";
    case MS_ERR_KEY_DOMAIN: return "MS_ERR_KEY_DOMAIN";
    case MS_ERR_NCCL: return "MS_ERR_NCCL";
  }
  return "MS_UNKNOWN";
}

const char *ms_version(void) { return "0.1.0"; }

ms_status ms_bucket_delta_default(uint32_t m, ms_bucket_fn *out) {
  if (!out) return MS_ERR_INVALID_VALUE;
  if (m < 1 || m > 256) return MS_ERR_UNSUPPORTED;
  const unsigned long long d = ((1ull << 32) + m - 1) / m;
  *out = ms_bucket_fn{MS_BUCKET_DELTA, m, (uint32_t)(d > 0xFFFFFFFFull ? 0xFFFFFFFFull : d), 0, 0};
  return MS_SUCCESS;
}

ms_status ms_bucket_identity(uint32_t m, ms_bucket_fn *out) {
  if (!out) return MS_ERR_INVALID_VALUE;
  if (m < 1 || m > 256) return MS_ERR_UNSUPPORTED;
  *out = ms_bucket_fn{MS_BUCKET_IDENTITY, m, 0, 0, 0};
  return MS_SUCCESS;
}

ms_status ms_bucket_radix(uint32_t shift, uint32_t bits, ms_bucket_fn *out) {
  if (!out) return MS_ERR_INVALID_VALUE;
  if (bits < 1 || bits > 8 || (uint64_t)shift + bits > 32) return MS_ERR_INVALID_VALUE;
  *out = ms_bucket_fn{MS_BUCKET_RADIX, 1u << bits, 0, shift, bits};
  return MS_SUCCESS;
}

ms_status ms_bucket_validate(const ms_bucket_fn *fn) { return validate_fn(fn); }

size_t ms_multisplit_workspace_size(uint64_t n, uint32_t m, int with_values) {
  (void)with_values;
  if (m < 1) m = 1;
  if (m > 256) m = 256;
  return layout_for(n, m).total;
}

ms_status ms_multisplit_keys(const uint32_t *keys_in, uint32_t *keys_out, uint64_t n,
                             const ms_bucket_fn *fn, uint32_t *bucket_offsets, void *ws,
                             size_t ws_bytes, void *stream) {
  return multisplit_impl(keys_in, nullptr, keys_out, nullptr, n, fn, bucket_offsets, ws, ws_bytes,
                         stream, false);
}

ms_status ms_multisplit_pairs(const uint32_t *keys_in, const uint32_t *vals_in,
                              uint32_t *keys_out, uint32_t *vals_out, uint64_t n,
                              const ms_bucket_fn *fn, uint32_t *bucket_offsets, void *ws,
                              size_t ws_bytes, void *stream) {
  return multisplit_impl(keys_in, vals_in, keys_out, vals_out, n, fn, bucket_offsets, ws,
                         ws_bytes, stream, true);
}

int ms_radix_pass_schedule(uint32_t begin_bit, uint32_t end_bit, uint32_t r, uint32_t *shifts,
                           uint32_t *bits, int cap) {
  if (r < 1 || r > 8 || begin_bit >= end_bit || end_bit > 32) return -1;
  int p = 0;
  for (uint32_t s = begin_bit; s < end_bit; s += r, ++p) {
    if (p < cap) {
      if (shifts) shifts[p] = s;
      if (bits) bits[p] = (end_bit - s) < r ? (end_bit - s) : r;
    }
  }
  return p;
}

size_t ms_radix_sort_workspace_size(uint64_t n, int with_values) {
  return align_up(ms_multisplit_workspace_size(n, 256, with_values)) + align_up(n * 4u) +
         (with_values ? align_up(n * 4u) : 0u);
}

ms_status ms_radix_sort_keys(const uint32_t *keys_in, uint32_t *keys_out, uint64_t n,
                             uint32_t begin_bit, uint32_t end_bit, uint32_t bits_per_pass,
                             void *ws, size_t ws_bytes, void *stream) {
  return radix_impl(keys_in, nullptr, keys_out, nullptr, n, begin_bit, end_bit, bits_per_pass, ws,
                    ws_bytes, stream, false);
}

ms_status ms_radix_sort_pairs(const uint32_t *keys_in, const uint32_t *vals_in,
                              uint32_t *keys_out, uint32_t *vals_out, uint64_t n,
                              uint32_t begin_bit, uint32_t end_bit, uint32_t bits_per_pass,
                              void *ws, size_t ws_bytes, void *stream) {
  return radix_impl(keys_in, vals_in, keys_out, vals_out, n, begin_bit, end_bit, bits_per_pass,
                    ws, ws_bytes, stream, true);
}

ms_status ms_device_status(const void *ws, void *stream) {
  if (!ws) return MS_ERR_INVALID_VALUE;
  uint32_t flag = 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemcpyAsync(&flag, ws, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess) return MS_ERR_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return MS_ERR_CUDA;
  return flag ? MS_ERR_KEY_DOMAIN : MS_SUCCESS;
}

uint32_t ms_multisplit_tile_size(uint32_t m, int with_values) {
  (void)m;
  (void)with_values;
  return (uint32_t)kTile;
}

ms_status ms_stage_prescan(const uint32_t *keys_in, uint64_t n, const ms_bucket_fn *fn,
                           uint32_t *H, uint32_t tile, void *stream) {
  ms_status st = validate_fn(fn);
  if (st != MS_SUCCESS) return st;
  if (tile != (uint32_t)kTile) return MS_ERR_INVALID_VALUE;
  if (n >= (1ull << 32)) return MS_ERR_UNSUPPORTED;
  if (n == 0) return MS_SUCCESS;
  if (!keys_in || !H) return MS_ERR_INVALID_VALUE;
  const uint32_t m = fn->num_buckets;
  const BucketParams bp = make_params(fn);
  const int logm = m <= 2 ? 1 : (int)ceil_log2(m);
  return counted(prescan_dispatch(fn->kind, hist_strategy(m), logm, keys_in, (uint32_t)n, bp, H,
                                  nullptr, 0, nullptr, (cudaStream_t)stream)) == cudaSuccess
             ? MS_SUCCESS
             : MS_ERR_CUDA;
}

size_t ms_stage_scan_workspace_size(uint64_t L, uint32_t m) {
  if (m < 1) m = 1;
  if (m > 256) m = 256;
  const uint64_t nchunks = (L + scan_chunk_tiles(m) - 1) / scan_chunk_tiles(m);
  return kHdrBytes + kBaseBytes + align_up((size_t)nchunks * m * 8u);
}

ms_status ms_stage_scan(const uint32_t *H, uint32_t *G, uint64_t L, uint32_t m,
                        uint32_t *bucket_offsets, void *ws, size_t ws_bytes, void *stream) {
  if (m < 1 || m > 256) return MS_ERR_UNSUPPORTED;
  if (L == 0) return MS_SUCCESS;
  if (!H || !G || !ws) return MS_ERR_INVALID_VALUE;
  if (L * m >= (1ull << 32)) return MS_ERR_UNSUPPORTED;
  if (ws_bytes < ms_stage_scan_workspace_size(L, m)) return MS_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  char *w = (char *)ws;
  uint32_t *hdr = (uint32_t *)w;
  uint32_t *base = (uint32_t *)(w + kHdrBytes);
  unsigned long long *status = (unsigned long long *)(w + kHdrBytes + kBaseBytes);
  const uint32_t C = scan_chunk_tiles(m);
  const uint32_t nchunks = (uint32_t)((L + C - 1) / C);
  zero_words_kernel<<<64, 256, 0, s>>>(status, nchunks * m, hdr);
  kg_scan<<<nchunks, kScanThreads, 0, s>>>(H, G, (uint32_t)L, m, C, nchunks, status, hdr + 1, base,
                                           bucket_offsets);
  kg_add_base<<<296, 256, 0, s>>>(G, L * m, m, base);
  return counted(cudaGetLastError(), 3) == cudaSuccess ? MS_SUCCESS : MS_ERR_CUDA;
}

void ms_set_stage_events(void *const *events) { g_stage_events = events; }

uint64_t ms_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

}  // extern "C"
