// ms_capi.cu -- the extern "C" boundary of libms (include/multisplit.h):
// argument validation, workspace carving, strategy dispatch and the LSD
// radix-sort pass driver.  All launches are stream-ordered; nothing here
// synchronizes except ms_device_status.
#include <atomic>
#include <mutex>
#include <cmath>
#include <vector>
#include <cstdlib>
#include <cstring>

#include "../../include/multisplit.h"
#include "ms_dispatch.cuh"
#include "ms_hist.cuh"
#include "ms_scan.cuh"

using namespace ms;

namespace ms {
// Reading R23 probe per device (k_probe_lane_ordered_inc, ms_meta.cuh): -1 not
// yet run, 0 failed, 1 held.  Run only by ms_device_init / ms_lane_ordered_increment
// (synchronous, on a private stream); a multisplit on a device that has not
// been probed ranks with the deterministic peer masks.
constexpr int kMaxDevices = 64;
std::atomic<int> g_probe[kMaxDevices];
std::mutex g_probe_mu;
std::atomic<int> g_opt[3] = {{MS_RANK_AUTO}, {1}, {MS_PIPELINE_LEVEL0}};

int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) return -1;
  return d;
}

int run_probe() {
  int sms = 0, dev = current_device();
  if (dev < 0 || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return 0;
  const size_t smem = kfm_smem_bytes(32, false);  // the postscan's footprint: 2 CTAs per SM
  if (cudaFuncSetAttribute(k_probe_lane_ordered_inc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return 0;
  uint32_t *d = nullptr, h = 0, one = 1;
  cudaStream_t st = nullptr;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return 0;
  bool r = false;
  if (cudaMallocAsync((void **)&d, 4, st) == cudaSuccess) {
    r = cudaMemcpyAsync(d, &one, 4, cudaMemcpyHostToDevice, st) == cudaSuccess;
    if (r) {
      k_probe_lane_ordered_inc<<<2 * sms, kThreads, smem, st>>>(d, 64u);
      r = cudaGetLastError() == cudaSuccess &&
          cudaMemcpyAsync(&h, d, 4, cudaMemcpyDeviceToHost, st) == cudaSuccess;
    }
    r = cudaFreeAsync(d, st) == cudaSuccess && cudaStreamSynchronize(st) == cudaSuccess && r &&
        h == 1u;
  }
  cudaStreamDestroy(st);
  return r ? 1 : 0;
}

// the probe result of the current device, running it if `run` and not yet done
int lane_ordered_inc(bool run) {
  const int dev = current_device();
  if (dev < 0) return 0;
  int v = g_probe[dev].load(std::memory_order_acquire);
  if (v >= 0 || !run) return v;
  std::lock_guard<std::mutex> lk(g_probe_mu);
  v = g_probe[dev].load(std::memory_order_acquire);
  if (v < 0) {
    v = run_probe();
    g_probe[dev].store(v, std::memory_order_release);
  }
  return v;
}

struct ProbeInit {
  ProbeInit() {
    for (auto &p : g_probe) p.store(-1);
  }
} g_probe_init;
}  // namespace ms

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

// tiles per look-back chunk: ~4096 H words per scan CTA
uint32_t scan_chunk_tiles(uint32_t m) {
  uint32_t c = 4096u / m;
  return c < 1 ? 1 : c;
}

uint32_t tile_elems(uint32_t m, bool pairs) { return kf_tile(pairs, kf_class(m)); }
uint32_t ctas_per_sm(uint32_t m, bool pairs) {
  return (uint32_t)kf_shape(pairs, kf_class(m)).ctas_per_sm;
}

// Workspace: [hdr 256 B][base 1280 B][R or H: L*m words][KG status: nchunks*m u64]
// (the level-0 histogram R needs G <= L rows; the three-launch mode needs L rows of H).
struct Layout {
  size_t base, H, status, meta, total;
  uint32_t T, L, nchunks, C, MS;
};


Layout layout_for(uint64_t n, uint32_t m, bool pairs) {
  Layout lo{};
  lo.T = tile_elems(m, pairs);
  lo.base = kHdrBytes;
  lo.H = kHdrBytes + kBaseBytes;
  if (n <= lo.T) {  // single-CTA path: header only
    lo.status = lo.total = lo.H;
    lo.L = n ? 1 : 0;
    return lo;
  }
  lo.L = (uint32_t)((n + lo.T - 1) / lo.T);
  lo.C = scan_chunk_tiles(m);
  lo.nchunks = (lo.L + lo.C - 1) / lo.C;
  lo.status = lo.H + align_up((size_t)lo.L * m * 8u);  // H (or R and its prefixes P)
  lo.total = lo.status + align_up((size_t)lo.nchunks * m * 8u);
  lo.meta = lo.total;
  if (m <= 32) {  // tile meta records (ms_meta.cuh)
    lo.MS = meta_stride(meta_ms(m), kWarps);
    lo.total = lo.meta + align_up((size_t)lo.L * lo.MS * 4u);
  }
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

// Device kind + parameters.  DELTA with delta = 2^s becomes a shift (kDeltaShift).
struct Plan {
  int kind;
  BucketParams bp;
};

Plan make_plan(const ms_bucket_fn *fn) {
  Plan pl{};
  BucketParams &p = pl.bp;
  p.m = fn->num_buckets;
  p.m1 = fn->num_buckets - 1;
  switch (fn->kind) {
    case MS_BUCKET_IDENTITY: pl.kind = kIdentity; break;
    case MS_BUCKET_RADIX:
      pl.kind = fn->shift + fn->bits == 32 ? kTopBits : kRadix;
      p.shift = fn->shift;
      p.mask = (1u << fn->bits) - 1u;
      break;
    default: {
      const uint32_t d = fn->delta;
      if ((d & (d - 1u)) == 0u) {  // power of two, including delta = 1
        p.shift = (uint32_t)__builtin_ctz(d);
        // m * delta >= 2^32: u >> shift < m already, no clamp needed
        pl.kind = ((uint64_t)p.m << p.shift) >= (1ull << 32) ? kTopBits : kDeltaShift;
      } else {
        pl.kind = kDelta;
        // M = ceil(2^64 / delta) = floor((2^64 - 1) / delta) + 1   (delta >= 3 here)
        const unsigned long long M = ~0ull / d + 1ull;
        p.magic_hi = (uint32_t)(M >> 32);
        p.magic_lo = (uint32_t)M;
      }
    }
  }
  return pl;
}

int sm_count() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
    return 148;
  return n;
}


cudaError_t launch_level0_scan(const uint32_t *R, uint32_t *P, uint32_t *Tot, uint32_t G,
                               uint32_t m, cudaStream_t s) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((m + 31) / 32);
  cfg.blockDim = dim3(kThreads);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kr_level0_scan, R, P, Tot, G, m);
}

bool overlaps(const void *a, const void *b, uint64_t n) {
  if (!a || !b || n == 0) return false;
  const char *pa = (const char *)a, *pb = (const char *)b;
  const uint64_t bytes = n * 4u;
  return pa < pb + bytes && pb < pa + bytes;
}

cudaError_t range_hist(const Plan &pl, const uint32_t *keys, uint32_t n, uint32_t per,
                       uint32_t grid, uint32_t *R, uint32_t *hdr, cudaStream_t s) {
  switch (pl.kind) {
    case kIdentity: return Launch<kIdentity>::range_hist(keys, n, per, grid, pl.bp, R, hdr, s);
    case kDelta: return Launch<kDelta>::range_hist(keys, n, per, grid, pl.bp, R, hdr, s);
    case kRadix: return Launch<kRadix>::range_hist(keys, n, per, grid, pl.bp, R, hdr, s);
    case kTopBits: return Launch<kTopBits>::range_hist(keys, n, per, grid, pl.bp, R, hdr, s);
    default: return Launch<kDeltaShift>::range_hist(keys, n, per, grid, pl.bp, R, hdr, s);
  }
}

cudaError_t tile_hist(const Plan &pl, const uint32_t *keys, uint32_t n, uint32_t tile,
                      uint32_t grid, uint32_t *H, uint32_t *hdr, cudaStream_t s) {
  switch (pl.kind) {
    case kIdentity: return Launch<kIdentity>::tile_hist(keys, n, tile, grid, pl.bp, H, hdr, s);
    case kDelta: return Launch<kDelta>::tile_hist(keys, n, tile, grid, pl.bp, H, hdr, s);
    case kRadix: return Launch<kRadix>::tile_hist(keys, n, tile, grid, pl.bp, H, hdr, s);
    case kTopBits: return Launch<kTopBits>::tile_hist(keys, n, tile, grid, pl.bp, H, hdr, s);
    default: return Launch<kDeltaShift>::tile_hist(keys, n, tile, grid, pl.bp, H, hdr, s);
  }
}

cudaError_t tile_meta(const Plan &pl, bool pairs, const uint32_t *keys, uint32_t n, uint32_t L,
                      uint32_t K, uint32_t grid, uint32_t *meta, uint32_t *R, uint32_t *hdr,
                      cudaStream_t s) {
  switch (pl.kind) {
    case kIdentity: return Launch<kIdentity>::tile_meta(pairs, keys, n, L, K, grid, pl.bp, meta, R, hdr, s);
    case kDelta: return Launch<kDelta>::tile_meta(pairs, keys, n, L, K, grid, pl.bp, meta, R, hdr, s);
    case kRadix: return Launch<kRadix>::tile_meta(pairs, keys, n, L, K, grid, pl.bp, meta, R, hdr, s);
    case kTopBits: return Launch<kTopBits>::tile_meta(pairs, keys, n, L, K, grid, pl.bp, meta, R, hdr, s);
    default: return Launch<kDeltaShift>::tile_meta(pairs, keys, n, L, K, grid, pl.bp, meta, R, hdr, s);
  }
}

cudaError_t fused_meta(const Plan &pl, bool pairs, const KfArgs &a, uint32_t grid, cudaStream_t s) {
  switch (pl.kind) {
    case kIdentity: return Launch<kIdentity>::fused_meta(pairs, a, pl.bp, grid, s);
    case kDelta: return Launch<kDelta>::fused_meta(pairs, a, pl.bp, grid, s);
    case kRadix: return Launch<kRadix>::fused_meta(pairs, a, pl.bp, grid, s);
    case kTopBits: return Launch<kTopBits>::fused_meta(pairs, a, pl.bp, grid, s);
    default: return Launch<kDeltaShift>::fused_meta(pairs, a, pl.bp, grid, s);
  }
}

cudaError_t fused(const Plan &pl, bool pairs, const KfArgs &a, uint32_t grid, cudaStream_t s) {
  switch (pl.kind) {
    case kIdentity: return Launch<kIdentity>::fused(pairs, a, pl.bp, grid, s);
    case kDelta: return Launch<kDelta>::fused(pairs, a, pl.bp, grid, s);
    case kRadix: return Launch<kRadix>::fused(pairs, a, pl.bp, grid, s);
    case kTopBits: return Launch<kTopBits>::fused(pairs, a, pl.bp, grid, s);
    default: return Launch<kDeltaShift>::fused(pairs, a, pl.bp, grid, s);
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
  if (!ws || ((uintptr_t)ws & (kAlign - 1))) return MS_ERR_INVALID_VALUE;
  if (n > 0) {
    if (!keys_in || !keys_out) return MS_ERR_INVALID_VALUE;
    if (pairs && (!vals_in || !vals_out)) return MS_ERR_INVALID_VALUE;
    if (overlaps(keys_in, keys_out, n)) return MS_ERR_INVALID_VALUE;
    if (pairs && (overlaps(vals_in, vals_out, n) || overlaps(keys_in, vals_out, n) ||
                  overlaps(vals_in, keys_out, n) || overlaps(keys_out, vals_out, n)))
      return MS_ERR_INVALID_VALUE;
  }
  const Layout lo = layout_for(n, m, pairs);
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

  const Plan pl = make_plan(fn);
  KfArgs a{};
  a.keys_in = keys_in;
  a.vals_in = pairs ? vals_in : nullptr;
  a.keys_out = keys_out;
  a.vals_out = pairs ? vals_out : nullptr;
  a.n = (uint32_t)n;
  a.hdr = hdr;
  a.bucket_offsets = bucket_offsets;
  a.use_tma = (((uintptr_t)keys_in & 15u) == 0) && (!pairs || (((uintptr_t)vals_in & 15u) == 0));
  // whole-run TMA bulk stores pay off when the average bucket run of a tile is
  // >= 256 elements (measured: profiles/r01/); shorter runs use per-element stores
  a.store_runs = m <= 64 && lo.T / m >= 256u && (((uintptr_t)keys_out & 15u) == 0) &&
                 (!pairs || (((uintptr_t)vals_out & 15u) == 0)) &&
                 g_opt[MS_OPT_RUN_STORES].load(std::memory_order_relaxed) != 0;
  // Eq.4 term 1 by lane-ordered increments (reading R23) only on a device whose
  // probe passed and unless deterministic peer masks are requested; measured
  // (profiles/r01/s2_summary.md): increments win for keys and for m <= 32
  a.rank_inc = m > 2 && (!pairs || m <= 32) &&
               g_opt[MS_OPT_RANK].load(std::memory_order_relaxed) == MS_RANK_AUTO &&
               ms::lane_ordered_inc(false) == 1;

  if (n <= lo.T) {  // one subproblem: a single launch
    a.mode = kModeSingle;
    a.num_tiles = 1;
    a.tiles_per_cta = 1;
    stage_event(0, s);
    stage_event(1, s);
    stage_event(2, s);
    const cudaError_t e = counted(fused(pl, pairs, a, 1, s));
    stage_event(3, s);
    return e == cudaSuccess ? MS_SUCCESS : MS_ERR_CUDA;
  }

  uint32_t *base = (uint32_t *)(w + lo.base);
  uint32_t *H = (uint32_t *)(w + lo.H);
  a.num_tiles = lo.L;

  if (g_opt[MS_OPT_PIPELINE].load(std::memory_order_relaxed) == MS_PIPELINE_TILE) {
    // paper-faithful {local, global, local}: tile histograms H -> scan -> postscan
    unsigned long long *status = (unsigned long long *)(w + lo.status);
    stage_event(0, s);
    if (counted(tile_hist(pl, keys_in, (uint32_t)n, lo.T, lo.L, H, hdr, s)) != cudaSuccess)
      return MS_ERR_CUDA;
    stage_event(1, s);
    zero_words_kernel<<<64, 256, 0, s>>>(status, lo.nchunks * m, hdr + 1);
    kg_scan<<<lo.nchunks, kScanThreads, 0, s>>>(H, H, lo.L, m, lo.C, lo.nchunks, status,
                                                 hdr + 1, base, bucket_offsets);
    if (counted(cudaGetLastError(), 2) != cudaSuccess) return MS_ERR_CUDA;
    stage_event(2, s);
    a.mode = kModeTileG;
    a.Gt = H;
    a.base = base;
    a.tiles_per_cta = 1;
    a.num_ranges = lo.L;
    const cudaError_t e = counted(fused(pl, pairs, a, lo.L, s));
    stage_event(3, s);
    return e == cudaSuccess ? MS_SUCCESS : MS_ERR_CUDA;
  }

  // level-0 localization (Eq.3 with L_0 = G): G ranges of K consecutive tiles,
  // one CTA each.  KU: range histograms R (m x G); KR: column scan P of R and
  // the bucket totals; KF: bucket bases from the totals, then per range, tiles
  // in order with running per-bucket offsets.  KR and KF are programmatic
  // dependent launches.
  const uint32_t target = (uint32_t)sm_count() * ctas_per_sm(m, pairs);
  const uint32_t K = (lo.L + target - 1) / target;
  const uint32_t G = (lo.L + K - 1) / K;
  const bool meta_mode = m <= 32;
  uint32_t *meta = (uint32_t *)(w + lo.meta);
  stage_event(0, s);
  if (meta_mode) {
    if (counted(tile_meta(pl, pairs, keys_in, (uint32_t)n, lo.L, K, G, meta, H, hdr, s)) !=
        cudaSuccess)
      return MS_ERR_CUDA;
  } else if (counted(range_hist(pl, keys_in, (uint32_t)n, K * lo.T, G, H, hdr, s)) != cudaSuccess) {
    return MS_ERR_CUDA;
  }
  stage_event(1, s);
  uint32_t *P = H + (size_t)G * m;  // prefixes (the layout holds 2 L m words)
  if (meta_mode) {  // KF reduces the range histograms itself (no KR)
    stage_event(2, s);
    a.mode = kModeRange;
    a.R = H;
    a.tiles_per_cta = K;
    a.num_ranges = G;
    a.meta = meta;
    const cudaError_t e = counted(fused_meta(pl, pairs, a, G, s));
    stage_event(3, s);
    return e == cudaSuccess ? MS_SUCCESS : MS_ERR_CUDA;
  }
  if (counted(launch_level0_scan(H, P, base, G, m, s)) != cudaSuccess) return MS_ERR_CUDA;
  stage_event(2, s);
  a.mode = kModeRange;
  a.R = P;
  a.Tot = base;
  a.tiles_per_cta = K;
  a.num_ranges = G;
  const cudaError_t e = counted(fused(pl, pairs, a, G, s));
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
  if (!ws || ((uintptr_t)ws & (kAlign - 1))) return MS_ERR_INVALID_VALUE;
  if (n == 0) return MS_SUCCESS;
  if (!keys_in || !keys_out || (pairs && (!vals_in || !vals_out))) return MS_ERR_INVALID_VALUE;
  if (overlaps(keys_in, keys_out, n)) return MS_ERR_INVALID_VALUE;
  if (pairs && (overlaps(vals_in, vals_out, n) || overlaps(keys_out, vals_out, n) ||
                overlaps(keys_in, vals_out, n) || overlaps(vals_in, keys_out, n)))
    return MS_ERR_INVALID_VALUE;
  if (ws_bytes < ms_radix_sort_workspace_size(n, pairs)) return MS_ERR_WORKSPACE;
  size_t ms_bytes = 0;  // widest multisplit workspace over the passes
  for (int p = 0; p < passes; ++p) {
    const size_t x = ms_multisplit_workspace_size(n, 1u << bits[p], pairs);
    ms_bytes = x > ms_bytes ? x : ms_bytes;
  }
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

int ms_lane_ordered_increment(void) { return ms::lane_ordered_inc(true) == 1 ? 1 : 0; }

ms_status ms_device_init(int device) {
  int prev = 0;
  if (cudaGetDevice(&prev) != cudaSuccess) return MS_ERR_CUDA;
  if (device >= 0 && device != prev && cudaSetDevice(device) != cudaSuccess) return MS_ERR_CUDA;
  const int r = ms::lane_ordered_inc(true);
  if (device >= 0 && device != prev) cudaSetDevice(prev);
  return r < 0 ? MS_ERR_CUDA : MS_SUCCESS;
}

ms_status ms_set_option(int option, int value) {
  switch (option) {
    case MS_OPT_RANK:
      if (value != MS_RANK_AUTO && value != MS_RANK_PEER_MASKS) return MS_ERR_INVALID_VALUE;
      break;
    case MS_OPT_RUN_STORES:
      if (value != 0 && value != 1) return MS_ERR_INVALID_VALUE;
      break;
    case MS_OPT_PIPELINE:
      if (value != MS_PIPELINE_LEVEL0 && value != MS_PIPELINE_TILE) return MS_ERR_INVALID_VALUE;
      break;
    default: return MS_ERR_INVALID_VALUE;
  }
  ms::g_opt[option].store(value, std::memory_order_relaxed);
  return MS_SUCCESS;
}

int ms_get_option(int option) {
  return option >= 0 && option < 3 ? ms::g_opt[option].load(std::memory_order_relaxed) : -1;
}

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
  if (m < 1) m = 1;
  if (m > 256) m = 256;
  return layout_for(n, m, with_values != 0).total;
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

// ---------------------------------------------------------------- histogram (Sec.7.3)
static ms_status histogram_impl(const float *x, uint64_t n, uint32_t m, float lower, float upper,
                                const float *splitters, uint32_t *counts, void *stream,
                                bool range) {
  if (m < 1 || m > 256) return MS_ERR_UNSUPPORTED;
  if (n >= (1ull << 32)) return MS_ERR_UNSUPPORTED;
  if (!counts || (n > 0 && !x) || (range && !splitters)) return MS_ERR_INVALID_VALUE;
  if (!range && !(lower < upper)) return MS_ERR_INVALID_VALUE;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(counts, 0, (size_t)m * 4u, s) != cudaSuccess) return MS_ERR_CUDA;
  if (n == 0) return MS_SUCCESS;
  volatile float delta = (upper - lower) / (float)m;  // binary32, round to nearest (R25)
  const uint32_t target = (uint32_t)sm_count() * 2u;
  uint32_t per = (uint32_t)((n + target - 1) / target);
  per = (per + 4095u) & ~4095u;  // whole 16-byte vectors per CTA, >= 4096 samples
  const uint32_t grid = (uint32_t)((n + per - 1) / per);
  const size_t smem = ((size_t)kWarps * m + m + 1) * 4u;
  int ex = 0;
  const bool pow2 = std::frexp((float)delta, &ex) == 0.5f && std::isnormal((float)delta) &&
                    std::isnormal(1.0f / (float)delta);
  if (range)
    kh_histogram<true, false><<<grid, kThreads, smem, s>>>(x, (uint32_t)n, per, m, 0.f, 0.f, 0.f,
                                                           splitters, counts);
  else if (pow2)  // exact: multiply by the power-of-two reciprocal
    kh_histogram<false, true><<<grid, kThreads, smem, s>>>(x, (uint32_t)n, per, m, lower, upper,
                                                           1.0f / (float)delta, nullptr, counts);
  else
    kh_histogram<false, false><<<grid, kThreads, smem, s>>>(x, (uint32_t)n, per, m, lower, upper,
                                                            delta, nullptr, counts);
  return counted(cudaGetLastError()) == cudaSuccess ? MS_SUCCESS : MS_ERR_CUDA;
}

ms_status ms_histogram_even(const float *samples, uint64_t n, uint32_t m, float lower,
                            float upper, uint32_t *counts, void *stream) {
  return histogram_impl(samples, n, m, lower, upper, nullptr, counts, stream, false);
}

ms_status ms_histogram_range(const float *samples, uint64_t n, uint32_t m,
                             const float *splitters, uint32_t *counts, void *stream) {
  return histogram_impl(samples, n, m, 0.f, 0.f, splitters, counts, stream, true);
}

int ms_radix_pass_schedule(uint32_t begin_bit, uint32_t end_bit, uint32_t r, uint32_t *shifts,
                           uint32_t *bits, int cap) {
  if (r == 0) r = 5;  // library choice: digits that use the m <= 32 pipeline
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
  // the multisplit workspace of the widest pass over every digit width r = 1..8
  size_t ms_ws = 0;
  for (uint32_t r = 1; r <= 8; ++r) {
    const size_t x = ms_multisplit_workspace_size(n, 1u << r, with_values);
    ms_ws = x > ms_ws ? x : ms_ws;
  }
  return align_up(ms_ws) + align_up(n * 4u) +
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
  return tile_elems(m, with_values != 0);
}

ms_status ms_stage_prescan(const uint32_t *keys_in, uint64_t n, const ms_bucket_fn *fn,
                           uint32_t *H, uint32_t tile, void *stream) {
  ms_status st = validate_fn(fn);
  if (st != MS_SUCCESS) return st;
  if (tile == 0) return MS_ERR_INVALID_VALUE;
  if (n >= (1ull << 32)) return MS_ERR_UNSUPPORTED;
  if (n == 0) return MS_SUCCESS;
  if (!keys_in || !H) return MS_ERR_INVALID_VALUE;
  const Plan pl = make_plan(fn);
  const uint32_t L = (uint32_t)((n + tile - 1) / tile);
  return counted(tile_hist(pl, keys_in, (uint32_t)n, tile, L, H, nullptr,
                           (cudaStream_t)stream)) == cudaSuccess
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

ms_status ms_shard_plan(const uint64_t *C, uint32_t G, uint32_t m, uint32_t r,
                        uint64_t *send_counts, uint64_t *send_displs, uint64_t *recv_counts,
                        uint64_t *recv_displs, uint32_t *merge_offsets,
                        uint64_t *global_bucket_offsets) {
  if (!C || G == 0 || r >= G || m < 1 || m > 256) return MS_ERR_INVALID_VALUE;
  if (!send_counts || !send_displs || !recv_counts || !recv_displs || !merge_offsets)
    return MS_ERR_INVALID_VALUE;
  std::vector<uint64_t> n(G, 0), N0(G + 1, 0), A(m + 1, 0), colpre((size_t)G * m, 0);
  for (uint32_t s = 0; s < G; ++s) {
    for (uint32_t j = 0; j < m; ++j) n[s] += C[(size_t)s * m + j];
    if (n[s] >= (1ull << 32)) return MS_ERR_UNSUPPORTED;
    N0[s + 1] = N0[s] + n[s];  // output shard s = global [N0[s], N0[s+1])
  }
  for (uint32_t j = 0; j < m; ++j) {  // Eq.3 term 1 (A) and term 2 (colpre = B_{j,s})
    uint64_t run = 0;
    for (uint32_t s = 0; s < G; ++s) {
      colpre[(size_t)s * m + j] = run;
      run += C[(size_t)s * m + j];
    }
    A[j + 1] = A[j] + run;
  }
  if (global_bucket_offsets)
    for (uint32_t j = 0; j <= m; ++j) global_bucket_offsets[j] = A[j];
  // number of shard-s elements whose global position is < x: global position is
  // monotone along s's local (bucket-major) order, so this is a prefix of it
  auto below = [&](uint32_t s, uint64_t x) {
    uint64_t cnt = 0;
    for (uint32_t j = 0; j < m; ++j) {
      const uint64_t g = A[j] + colpre[(size_t)s * m + j], c = C[(size_t)s * m + j];
      cnt += x <= g ? 0 : (x - g < c ? x - g : c);
    }
    return cnt;
  };
  for (uint32_t d = 0; d < G; ++d) {  // what r sends to d: one range of r's local order
    const uint64_t lo = below(r, N0[d]), hi = below(r, N0[d + 1]);
    send_displs[d] = lo;
    send_counts[d] = hi - lo;
  }
  uint64_t packed = 0;
  for (uint32_t s = 0; s < G; ++s) {  // what r receives from s, packed in source order
    const uint64_t lo = below(s, N0[r]), hi = below(s, N0[r + 1]);
    recv_counts[s] = hi - lo;
    recv_displs[s] = packed;
    // element e of the receive buffer from s is s's local index q = lo + (e - packed);
    // bucket j: global = A_j + B_{j,s} + (q - localbase_{s,j}); output index = global - N0[r]
    uint64_t lb = 0;
    for (uint32_t j = 0; j < m; ++j) {
      const uint64_t g = A[j] + colpre[(size_t)s * m + j];
      merge_offsets[(size_t)s * m + j] = (uint32_t)(g - lb + lo - N0[r] - packed);
      lb += C[(size_t)s * m + j];
    }
    packed += hi - lo;
  }
  return MS_SUCCESS;
}

static ms_status shard_merge(const uint32_t *keys_recv, const uint32_t *vals_recv, uint64_t n_recv,
                             const ms_bucket_fn *fn, const uint32_t *recv_starts,
                             const uint32_t *merge_offsets, uint32_t G, uint32_t *keys_out,
                             uint32_t *vals_out, void *stream, bool pairs) {
  ms_status st = validate_fn(fn);
  if (st != MS_SUCCESS) return st;
  if (n_recv >= (1ull << 32)) return MS_ERR_UNSUPPORTED;
  if (n_recv == 0) return MS_SUCCESS;
  if (!keys_recv || !keys_out || !recv_starts || !merge_offsets || G == 0 ||
      (pairs && (!vals_recv || !vals_out)))
    return MS_ERR_INVALID_VALUE;
  const Plan pl = make_plan(fn);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  switch (pl.kind) {
    case kIdentity:
      e = Launch<kIdentity>::merge(pairs, keys_recv, vals_recv, (uint32_t)n_recv, pl.bp,
                                   recv_starts, merge_offsets, G, keys_out, vals_out, s);
      break;
    case kDelta:
      e = Launch<kDelta>::merge(pairs, keys_recv, vals_recv, (uint32_t)n_recv, pl.bp, recv_starts,
                                merge_offsets, G, keys_out, vals_out, s);
      break;
    case kRadix:
      e = Launch<kRadix>::merge(pairs, keys_recv, vals_recv, (uint32_t)n_recv, pl.bp, recv_starts,
                                merge_offsets, G, keys_out, vals_out, s);
      break;
    case kTopBits:
      e = Launch<kTopBits>::merge(pairs, keys_recv, vals_recv, (uint32_t)n_recv, pl.bp,
                                  recv_starts, merge_offsets, G, keys_out, vals_out, s);
      break;
    default:
      e = Launch<kDeltaShift>::merge(pairs, keys_recv, vals_recv, (uint32_t)n_recv, pl.bp,
                                     recv_starts, merge_offsets, G, keys_out, vals_out, s);
  }
  return counted(e) == cudaSuccess ? MS_SUCCESS : MS_ERR_CUDA;
}

ms_status ms_shard_merge_keys(const uint32_t *keys_recv, uint64_t n_recv, const ms_bucket_fn *fn,
                              const uint32_t *recv_starts, const uint32_t *merge_offsets,
                              uint32_t G, uint32_t *keys_out, void *stream) {
  return shard_merge(keys_recv, nullptr, n_recv, fn, recv_starts, merge_offsets, G, keys_out,
                     nullptr, stream, false);
}

ms_status ms_shard_merge_pairs(const uint32_t *keys_recv, const uint32_t *vals_recv,
                               uint64_t n_recv, const ms_bucket_fn *fn,
                               const uint32_t *recv_starts, const uint32_t *merge_offsets,
                               uint32_t G, uint32_t *keys_out, uint32_t *vals_out, void *stream) {
  return shard_merge(keys_recv, vals_recv, n_recv, fn, recv_starts, merge_offsets, G, keys_out,
                     vals_out, stream, true);
}

void ms_set_stage_events(void *const *events) { g_stage_events = events; }

uint64_t ms_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

}  // extern "C"
