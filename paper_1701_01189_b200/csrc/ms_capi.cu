// ms_capi.cu -- the extern "C" boundary of libms (include/multisplit.h):
// argument validation, workspace carving, strategy dispatch and the LSD
// radix-sort pass driver.  All launches are stream-ordered; nothing here
// synchronizes except ms_device_status.
#include <algorithm>
#include <type_traits>
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
#include "ms_nccl.cuh"

#include <cuda.h>

using namespace ms;

namespace ms {
// Reading R23 probe per device (k_probe_lane_ordered_inc, ms_meta.cuh): -1 not
// yet run, 0 failed, 1 held.  Run only by ms_device_init / ms_lane_ordered_increment
// (synchronous, on a private stream); a multisplit on a device that has not
// been probed ranks with the deterministic peer masks.
constexpr int kMaxDevices = 64;
std::atomic<int> g_probe[kMaxDevices];
std::mutex g_probe_mu;
constexpr int kNumOpts = 4;
std::atomic<int> g_opt[kNumOpts] = {{MS_RANK_AUTO}, {1}, {MS_PIPELINE_AUTO}, {MS_SORT_AUTO}};

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
  size_t base, H, status, meta, wmeta, total;
  uint32_t T, L, nchunks, C, MS;
  uint32_t LW, NB;  // m > 32: tiles and buckets per lane of the wide pipeline (ms_wide.cuh)
};
constexpr uint32_t kMaxRanges = 4096;  // level-0 ranges (CTAs) of the persistent kernels


// ranges: always lay out the level-0 range pipeline (the sharded path has no
// single-CTA shortcut)
Layout layout_for(uint64_t n, uint32_t m, bool pairs, bool ranges = false) {
  Layout lo{};
  lo.T = tile_elems(m, pairs);
  lo.base = kHdrBytes;
  lo.H = kHdrBytes + kBaseBytes;
  if (n == 0 || (n <= lo.T && !ranges)) {  // single-CTA path: header only
    lo.status = lo.total = lo.H;
    lo.L = n ? 1 : 0;
    return lo;
  }
  lo.L = (uint32_t)((n + lo.T - 1) / lo.T);
  lo.C = scan_chunk_tiles(m);
  lo.nchunks = (lo.L + lo.C - 1) / lo.C;
  size_t hwords = (size_t)lo.L * m * 2u;  // H (or R and its prefixes P)
  if (m > 32) {
    lo.NB = wide_nb(m);
    lo.LW = (uint32_t)((n + wide_tile(pairs) - 1) / wide_tile(pairs));
    const size_t rw = 2u * (size_t)std::min(lo.LW, kMaxRanges) * 32u * lo.NB;
    hwords = std::max(hwords, rw);
  }
  lo.status = lo.H + align_up(hwords * 4u);
  lo.total = lo.status + align_up((size_t)lo.nchunks * m * 8u);
  lo.meta = lo.wmeta = lo.total;
  if (m <= 32) {  // tile meta records (ms_meta.cuh)
    lo.MS = meta_stride(meta_ms(m), kWarps);
    lo.total = lo.meta + align_up((size_t)lo.L * lo.MS * 4u);
  } else {  // wide records (ms_wide.cuh)
    lo.total = lo.wmeta + align_up((size_t)lo.LW * wide_rec_words(pairs, lo.NB) * 4u);
  }
  return lo;
}

constexpr uint32_t kMaxLargeM = 65536;  // m > 256: two LSD digit passes of the bucket id

// large: the multisplit entry points also take 256 < m <= 65536 (RADIX digits
// up to 16 bits); the stage, merge and sharded calls keep the paper's m <= 256
ms_status validate_fn(const ms_bucket_fn *fn, bool large = false) {
  if (!fn) return MS_ERR_INVALID_VALUE;
  const uint32_t m = fn->num_buckets;
  if (m < 1 || m > (large ? kMaxLargeM : 256u)) return MS_ERR_UNSUPPORTED;
  switch (fn->kind) {
    case MS_BUCKET_IDENTITY: return MS_SUCCESS;
    case MS_BUCKET_DELTA: return fn->delta >= 1 ? MS_SUCCESS : MS_ERR_INVALID_VALUE;
    case MS_BUCKET_RADIX:
      if (fn->bits < 1 || fn->bits > (large ? 16u : 8u)) return MS_ERR_INVALID_VALUE;
      if ((uint64_t)fn->shift + fn->bits > 32) return MS_ERR_INVALID_VALUE;
      if (m != (1u << fn->bits)) return MS_ERR_INVALID_VALUE;
      return MS_SUCCESS;
    case MS_BUCKET_SPLITTERS:
      return (m == 1 || fn->splitters) ? MS_SUCCESS : MS_ERR_INVALID_VALUE;
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
    case MS_BUCKET_SPLITTERS: {
      pl.kind = kSplitters;
      p.spl = fn->splitters;
      uint32_t pw = 1;
      while (pw < p.m) pw <<= 1;
      p.spl_pow = pw;
      break;
    }
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

// Calls f(std::integral_constant<int, K>) with the plan's compile-time bucket kind K.
template <typename F>
cudaError_t by_kind(int kind, F &&f) {
  switch (kind) {
    case kIdentity: return f(std::integral_constant<int, kIdentity>{});
    case kDelta: return f(std::integral_constant<int, kDelta>{});
    case kRadix: return f(std::integral_constant<int, kRadix>{});
    case kTopBits: return f(std::integral_constant<int, kTopBits>{});
    case kSplitters: return f(std::integral_constant<int, kSplitters>{});
    default: return f(std::integral_constant<int, kDeltaShift>{});
  }
}
#define MS_LAUNCH(fn_, ...) \
  by_kind(pl.kind, [&](auto k_) { return Launch<decltype(k_)::value>::fn_(__VA_ARGS__); })

cudaError_t range_hist(const Plan &pl, const uint32_t *keys, uint32_t n, uint32_t per,
                       uint32_t grid, uint32_t *R, uint32_t *hdr, cudaStream_t s) {
  return MS_LAUNCH(range_hist, keys, n, per, grid, pl.bp, R, hdr, s);
}

cudaError_t tile_hist(const Plan &pl, const uint32_t *keys, uint32_t n, uint32_t tile,
                      uint32_t grid, uint32_t *H, uint32_t *hdr, cudaStream_t s) {
  return MS_LAUNCH(tile_hist, keys, n, tile, grid, pl.bp, H, hdr, s);
}

cudaError_t tile_meta(const Plan &pl, bool pairs, const uint32_t *keys, uint32_t n, uint32_t L,
                      uint32_t K, uint32_t grid, uint32_t *meta, uint32_t *R, uint32_t *hdr,
                      cudaStream_t s) {
  return MS_LAUNCH(tile_meta, pairs, keys, n, L, K, grid, pl.bp, meta, R, hdr, s);
}

cudaError_t fused_meta(const Plan &pl, bool pairs, const KfArgs &a, uint32_t grid, cudaStream_t s) {
  return MS_LAUNCH(fused_meta, pairs, a, pl.bp, grid, s);
}

cudaError_t tile_meta_wide(const Plan &pl, bool pairs, const uint32_t *keys, uint32_t n, uint32_t LM,
                           uint32_t per, uint32_t grid, uint32_t *meta, uint32_t nkf, uint32_t *R,
                           uint32_t *hdr, cudaStream_t s) {
  return MS_LAUNCH(tile_meta_wide, pairs, keys, n, LM, per, grid, pl.bp, meta, nkf, R, hdr, s);
}

cudaError_t fused_meta_wide(const Plan &pl, bool pairs, const KfArgs &a, uint32_t grid, cudaStream_t s) {
  return MS_LAUNCH(fused_meta_wide, pairs, a, pl.bp, grid, s);
}

cudaError_t fused(const Plan &pl, bool pairs, const KfArgs &a, uint32_t grid, cudaStream_t s) {
  return MS_LAUNCH(fused, pairs, a, pl.bp, grid, s);
}

// Level-0 pipelines with prescan records: m <= 32 KM -> kf_meta (ms_meta.cuh),
// 32 < m <= 256 KMW -> KR -> kf_meta_wide (ms_wide.cuh; increments only).
struct L0 {
  bool wide;
  uint32_t G, K, mP, num_tiles;
  uint32_t GM, KM;  // prescan CTAs and their tiles: KM = K, or K / 2 (two per range)
  uint32_t *R, *P, *Tot, *meta;
};

// the ranges and buffers of a call (pure host arithmetic: the sharded scatter
// recomputes what its prescan used)
L0 l0_setup(uint32_t m, bool pairs, const Layout &lo, char *w) {
  L0 st{};
  uint32_t *H = (uint32_t *)(w + lo.H);
  st.Tot = (uint32_t *)(w + lo.base);
  st.wide = m > 32;
  if (!st.wide) {
    const uint32_t target = std::min((uint32_t)sm_count() * ctas_per_sm(m, pairs), kMaxRanges);
    st.K = (lo.L + target - 1) / target;
    st.G = (lo.L + st.K - 1) / st.K;
    st.mP = m;
    st.num_tiles = lo.L;
    st.R = H;
    st.P = H + (size_t)st.G * m;
    st.meta = (uint32_t *)(w + lo.meta);
    return st;
  }
  // the KM tile is the KF tile (ms_wide.cuh); one range per postscan CTA,
  // one postscan CTA per SM, two prescan CTAs per SM and range (each half of
  // it, K even): R and its column prefix P have a row per prescan CTA and
  // range c starts at row 2c
  st.mP = 32u * lo.NB;
  const uint32_t target = std::min((uint32_t)sm_count() * wide_ctas_per_sm(pairs), kMaxRanges);
  st.K = (lo.LW + target - 1) / target;
  if (st.K & 1u) ++st.K;
  st.G = (lo.LW + st.K - 1) / st.K;
  st.KM = st.K / 2u;
  st.GM = (lo.LW + st.KM - 1) / st.KM;
  st.num_tiles = lo.LW;
  st.R = H;
  st.P = H + (size_t)st.GM * st.mP;
  st.meta = (uint32_t *)(w + lo.wmeta);
  return st;
}

// with_totals: also the bucket totals Tot (m <= 32: an extra KR launch; the
// wide pipeline always has them)
cudaError_t l0_prescan(const Plan &pl, bool pairs, const uint32_t *keys, uint32_t n, const Layout &lo,
                       char *w, bool with_totals, L0 &st, cudaStream_t s) {
  const uint32_t m = pl.bp.m;
  uint32_t *hdr = (uint32_t *)w;
  st = l0_setup(m, pairs, lo, w);
  if (!st.wide) {
    cudaError_t e = counted(tile_meta(pl, pairs, keys, n, lo.L, st.K, st.G, st.meta, st.R, hdr, s));
    if (e == cudaSuccess && with_totals)
      e = counted(launch_level0_scan(st.R, st.P, st.Tot, st.G, m, s));
    return e;
  }
  cudaError_t e = counted(tile_meta_wide(pl, pairs, keys, n, lo.LW, st.KM, st.GM, st.meta, lo.LW, st.R, hdr, s));
  if (e == cudaSuccess && with_totals)  // the postscan reduces R itself; KR only for the sharded counts
    e = counted(launch_level0_scan(st.R, st.P, st.Tot, st.GM, st.mP, s));
  return e;
}

cudaError_t l0_postscan(const Plan &pl, bool pairs, KfArgs &a, const L0 &st, cudaStream_t s) {
  a.mode = kModeRange;
  a.meta = st.meta;
  a.num_tiles = st.num_tiles;
  a.tiles_per_cta = st.K;
  a.num_ranges = st.G;
  if (!st.wide) {
    a.R = st.R;  // kf_meta reduces the range histograms itself
    return counted(fused_meta(pl, pairs, a, st.G, s));
  }
  a.R = st.R;  // kf_meta_wide reduces the range histograms itself
  a.r_rows = st.GM;
  a.prefix_step = st.KM == st.K ? 1u : 2u;
  return counted(fused_meta_wide(pl, pairs, a, st.G, s));
}

// ---------------------------------------------------------------- one pass (f1)
// ms_onesweep.cuh.  Workspace: [hdr 256 B][gh: nbins words][tickets: P words]
// [status: P x L x 256 words]; everything up to the end of the status words is
// zeroed by one memset at the start of the call.
struct OsLayout {
  size_t gh, tickets, status, total;
  uint32_t L;
};
OsLayout os_layout(uint64_t n, uint32_t passes, bool pairs) {
  OsLayout lo{};
  lo.L = (uint32_t)((n + ko_tile(pairs) - 1) / ko_tile(pairs));
  lo.gh = kHdrBytes;
  lo.tickets = lo.gh + align_up((size_t)kKoMaxBins * 4u);
  lo.status = lo.tickets + align_up((size_t)kKoMaxPasses * 4u);
  lo.total = lo.status + align_up((size_t)passes * lo.L * kKoBins * 4u);
  return lo;
}

// the one-pass pipeline ranks with lane-ordered increments (reading R23): only
// where the device's probe held and deterministic ranks were not requested
bool onesweep_ok(uint64_t n) {
  return n > 0 && n < kKoMaxN && g_opt[MS_OPT_RANK].load(std::memory_order_relaxed) == MS_RANK_AUTO &&
         ms::lane_ordered_inc(false) == 1;
}

cudaError_t os_pass(const Plan &pl, bool pairs, const uint32_t *ki, const uint32_t *vi, uint32_t *ko,
                    uint32_t *vo, uint32_t n, const OsLayout &lo, char *w, uint32_t p, uint32_t bin0,
                    uint32_t *bucket_offsets, cudaStream_t s) {
  KoArgs a{};
  a.keys_in = ki;
  a.vals_in = pairs ? vi : nullptr;
  a.keys_out = ko;
  a.vals_out = pairs ? vo : nullptr;
  a.n = n;
  a.num_tiles = lo.L;
  a.gh = (const uint32_t *)(w + lo.gh) + bin0;
  a.status = (uint32_t *)(w + lo.status) + (size_t)p * lo.L * kKoBins;
  a.ticket = (uint32_t *)(w + lo.tickets) + p;
  a.hdr = (uint32_t *)w;
  a.bucket_offsets = bucket_offsets;
  a.use_tma = (((uintptr_t)ki & 15u) == 0) && (!pairs || (((uintptr_t)vi & 15u) == 0));
  const uint32_t grid = std::min((uint32_t)sm_count(), lo.L);
  return counted(MS_LAUNCH(onesweep, pairs, a, pl.bp, grid, s));
}

// one-pass multisplit: KOH (the bucket counts) -> KO
ms_status onesweep_multisplit(const Plan &pl, bool pairs, const uint32_t *ki, const uint32_t *vi,
                              uint32_t *ko, uint32_t *vo, uint32_t n, uint32_t *bucket_offsets,
                              char *w, cudaStream_t s) {
  const OsLayout lo = os_layout(n, 1, pairs);
  stage_event(0, s);
  if (cudaMemsetAsync(w, 0, lo.total, s) != cudaSuccess) return MS_ERR_CUDA;
  KoHistArgs h{};
  h.keys = ki;
  h.n = n;
  h.npass = 1;
  h.shift[0] = pl.bp.shift;
  h.mask[0] = pl.bp.mask;
  h.nbins = pl.bp.m;
  h.gh = (uint32_t *)(w + lo.gh);
  h.hdr = (uint32_t *)w;
  if (counted(MS_LAUNCH(ko_hist, h, pl.bp, (uint32_t)sm_count(), s)) != cudaSuccess) return MS_ERR_CUDA;
  stage_event(1, s);
  stage_event(2, s);
  const cudaError_t e = os_pass(pl, pairs, ki, vi, ko, vo, n, lo, w, 0, 0, bucket_offsets, s);
  stage_event(3, s);
  return e == cudaSuccess ? MS_SUCCESS : MS_ERR_CUDA;
}

// ---------------------------------------------------------------- m > 256
// Sec.6.3: iterated multisplits over <= 256 buckets, here LSD over
// the 8-bit digits of the bucket id (ms_large.cuh).  RADIX digits wider than 8
// bits are two radix passes over the keys themselves.
// Workspace: [hdr][inner multisplit / radix-sort ws][non-RADIX: b0 p0 b1 p1 b2
//             (+p2 for pairs), n words each]
struct LargeLayout {
  size_t inner, inner_bytes, x[6], total;
};
LargeLayout large_layout(uint64_t n, uint32_t kind, bool pairs) {
  LargeLayout lo{};
  // RADIX and IDENTITY: two key passes (top-bit DELTA uses the DELTA layout, a superset)
  const bool radix = kind == MS_BUCKET_RADIX || kind == MS_BUCKET_IDENTITY;
  lo.inner = kHdrBytes;
  lo.inner_bytes = std::max(ms_multisplit_workspace_size(n, 256, 0), ms_multisplit_workspace_size(n, 256, 1));
  // radix digits (and top-bit delta buckets) of the key itself: an LSD radix sort
  // over the digit's bits (the one-pass pipeline where it applies)
  lo.inner_bytes = std::max(lo.inner_bytes, ms_radix_sort_workspace_size(n, 1));
  size_t off = lo.inner + align_up(lo.inner_bytes);
  const int arrays = radix ? 0 : (pairs ? 6 : 5);  // the radix passes keep their own ping-pong buffer
  for (int i = 0; i < arrays; ++i) {
    lo.x[i] = off;
    off += align_up(n * 4u);
  }
  lo.total = off;
  return lo;
}

ms_status multisplit_impl(const uint32_t *keys_in, const uint32_t *vals_in, uint32_t *keys_out,
                          uint32_t *vals_out, uint64_t n, const ms_bucket_fn *fn,
                          uint32_t *bucket_offsets, void *ws, size_t ws_bytes, void *stream,
                          bool pairs);

ms_status radix_impl(const uint32_t *keys_in, const uint32_t *vals_in, uint32_t *keys_out,
                     uint32_t *vals_out, uint64_t n, uint32_t begin_bit, uint32_t end_bit,
                     uint32_t r, void *ws, size_t ws_bytes, void *stream, bool pairs);

ms_status large_impl(const uint32_t *keys_in, const uint32_t *vals_in, uint32_t *keys_out,
                     uint32_t *vals_out, uint64_t n, const ms_bucket_fn *fn,
                     uint32_t *bucket_offsets, char *w, cudaStream_t s, bool pairs) {
  const uint32_t m = fn->num_buckets;
  const LargeLayout lo = large_layout(n, fn->kind, pairs);
  void *const *hooks = g_stage_events;
  g_stage_events = nullptr;  // the inner multisplits record nothing
  auto ev = [&](int i) {
    if (hooks) cudaEventRecord((cudaEvent_t)hooks[i], s);
  };
  auto done = [&](ms_status st) {
    g_stage_events = hooks;
    return st;
  };
  char *inner = w + lo.inner;
  uint32_t *hdr = (uint32_t *)w;
  ev(0);
  if (cudaMemsetAsync(hdr, 0, 8, s) != cudaSuccess) return done(MS_ERR_CUDA);
  // RADIX digits, and DELTA buckets that are the top bits of the key (Delta a
  // power of two with m * Delta >= 2^32: f(u) = u >> s), are radix passes over
  // the keys themselves: no bucket-id pass, no gather
  // Identity buckets are the key's low bits (keys >= m are domain errors,
  // flagged by one check pass; their output is unspecified but in bounds).
  const Plan tp = make_plan(fn);
  const bool top = tp.kind == kTopBits, ident = fn->kind == MS_BUCKET_IDENTITY;
  if (fn->kind == MS_BUCKET_RADIX || top || ident) {
    uint32_t hb = 0;
    while ((1u << hb) < m) ++hb;
    const uint32_t sh = top ? tp.bp.shift : (ident ? 0u : fn->shift);
    const uint32_t bits = top ? 32u - tp.bp.shift : (ident ? hb : fn->bits);
    if (ident) {
      k_domain_check<<<min((uint32_t)((n + 255u) / 256u), 148u * 8u), 256, 0, s>>>(keys_in, (uint32_t)n, m, hdr);
      if (counted(cudaGetLastError()) != cudaSuccess) return done(MS_ERR_CUDA);
    }
    // two stable passes, the low 8 bits of the digit first (Sec.6.3 as an LSD sort
    // by the bucket id, R30): the radix sort over bits [sh, sh + bits)
    ev(1);
    ev(2);
    const ms_status st = radix_impl(keys_in, vals_in, keys_out, vals_out, n, sh, sh + bits, 8u, inner,
                                    lo.inner_bytes, s, pairs);
    if (st != MS_SUCCESS) return done(st);
    if (bucket_offsets) {
      k_offsets_sorted<<<min((uint32_t)((n + 256u) / 256u), 148u * 8u), 256, 0, s>>>(
          keys_out, (uint32_t)n, sh, (uint32_t)((1ull << bits) - 1u), m, bucket_offsets);
      if (counted(cudaGetLastError()) != cudaSuccess) return done(MS_ERR_CUDA);
    }
    ev(3);
    return done(MS_SUCCESS);
  }
  uint32_t *b0 = (uint32_t *)(w + lo.x[0]), *p0 = (uint32_t *)(w + lo.x[1]);
  uint32_t *b1 = (uint32_t *)(w + lo.x[2]), *p1 = (uint32_t *)(w + lo.x[3]);
  uint32_t *b2 = (uint32_t *)(w + lo.x[4]);
  uint32_t *p2 = pairs ? (uint32_t *)(w + lo.x[5]) : keys_out;
  const Plan pl = make_plan(fn);
  if (counted(MS_LAUNCH(bucket_ids, keys_in, (uint32_t)n, pl.bp, pairs, b0, p0, hdr, s)) != cudaSuccess)
    return done(MS_ERR_CUDA);
  ev(1);
  uint32_t hb = 0;
  while ((1u << hb) < m) ++hb;  // bits of the bucket id
  const ms_bucket_fn a{MS_BUCKET_RADIX, 256u, 0u, 0u, 8u, nullptr};
  const ms_bucket_fn b{MS_BUCKET_RADIX, 1u << (hb - 8u), 0u, 8u, hb - 8u, nullptr};
  ms_status st = multisplit_impl(b0, p0, b1, p1, n, &a, nullptr, inner, lo.inner_bytes, s, true);
  if (st != MS_SUCCESS) return done(st);
  ev(2);
  st = multisplit_impl(b1, p1, b2, p2, n, &b, nullptr, inner, lo.inner_bytes, s, true);
  if (st != MS_SUCCESS) return done(st);
  const uint32_t grid = min((uint32_t)((n + 256u) / 256u), 148u * 8u);
  if (bucket_offsets) {
    k_offsets_sorted<<<grid, 256, 0, s>>>(b2, (uint32_t)n, 0u, 0xFFFFFFFFu, m, bucket_offsets);
    if (counted(cudaGetLastError()) != cudaSuccess) return done(MS_ERR_CUDA);
  }
  if (pairs) {
    k_gather_pairs<<<grid, 256, 0, s>>>(p2, (uint32_t)n, keys_in, vals_in, keys_out, vals_out);
    if (counted(cudaGetLastError()) != cudaSuccess) return done(MS_ERR_CUDA);
  }
  ev(3);
  return done(MS_SUCCESS);
}

ms_status multisplit_impl(const uint32_t *keys_in, const uint32_t *vals_in, uint32_t *keys_out,
                          uint32_t *vals_out, uint64_t n, const ms_bucket_fn *fn,
                          uint32_t *bucket_offsets, void *ws, size_t ws_bytes, void *stream,
                          bool pairs) {
  ms_status st = validate_fn(fn, true);
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
  if (ws_bytes < ms_multisplit_workspace_size(n, m, pairs)) return MS_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  char *w = (char *)ws;
  uint32_t *hdr = (uint32_t *)w;

  if (n == 0) {
    if (cudaMemsetAsync(hdr, 0, 8, s) != cudaSuccess) return MS_ERR_CUDA;
    if (bucket_offsets && cudaMemsetAsync(bucket_offsets, 0, ((size_t)m + 1) * 4u, s) != cudaSuccess)
      return MS_ERR_CUDA;
    return MS_SUCCESS;
  }
  if (m > 256)
    return large_impl(keys_in, vals_in, keys_out, vals_out, n, fn, bucket_offsets, w, s, pairs);
  const Layout lo = layout_for(n, m, pairs);

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
  const bool inc_ok = m > 2 && g_opt[MS_OPT_RANK].load(std::memory_order_relaxed) == MS_RANK_AUTO &&
                      ms::lane_ordered_inc(false) == 1;
  a.rank_inc = inc_ok && (!pairs || m <= 32);

  if (n <= kSmallMax && ms::lane_ordered_inc(false) == 1 &&
      g_opt[MS_OPT_RANK].load(std::memory_order_relaxed) == MS_RANK_AUTO) {
    // latency-bound sizes: one CTA, one pass (k_small, ms_large.cuh)
    a.mode = kModeSingle;
    stage_event(0, s);
    stage_event(1, s);
    stage_event(2, s);
    const cudaError_t e = counted(MS_LAUNCH(small, pairs, a, pl.bp, s));
    stage_event(3, s);
    return e == cudaSuccess ? MS_SUCCESS : MS_ERR_CUDA;
  }
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

  // one pass (f1): on request, or (AUTO) for pairs with m > 128, where it was
  // measured faster than the level-0 pipeline (2^25 pairs m = 256: 195 vs 159
  // Gpairs/s; m = 128: 201 vs 208; keys m = 256: 267 vs 288)
  const int pipe = g_opt[MS_OPT_PIPELINE].load(std::memory_order_relaxed);
  if ((pipe == MS_PIPELINE_ONESWEEP || (pipe == MS_PIPELINE_AUTO && pairs && m > 128)) && onesweep_ok(n))
    return onesweep_multisplit(pl, pairs, keys_in, vals_in, keys_out, vals_out, (uint32_t)n,
                               bucket_offsets, w, s);
  if (pipe == MS_PIPELINE_TILE) {
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
  // one CTA each, tiles in order with running per-bucket offsets
  if (m <= 32 || inc_ok) {  // prescan records + rank/reorder postscan (ms_meta / ms_wide)
    L0 st{};
    stage_event(0, s);
    if (l0_prescan(pl, pairs, keys_in, (uint32_t)n, lo, w, false, st, s) != cudaSuccess)
      return MS_ERR_CUDA;
    stage_event(1, s);
    stage_event(2, s);
    const cudaError_t e = l0_postscan(pl, pairs, a, st, s);
    stage_event(3, s);
    return e == cudaSuccess ? MS_SUCCESS : MS_ERR_CUDA;
  }
  // m > 32 with deterministic ranks: KU range histograms R (m x G) -> KR column
  // scan P of R and the bucket totals -> KF (kf_fused) counts, scans and ranks
  // each tile itself.  KR and KF are programmatic dependent launches.
  const uint32_t target = (uint32_t)sm_count() * ctas_per_sm(m, pairs);
  const uint32_t K = (lo.L + target - 1) / target;
  const uint32_t G = (lo.L + K - 1) / K;
  stage_event(0, s);
  if (counted(range_hist(pl, keys_in, (uint32_t)n, K * lo.T, G, H, hdr, s)) != cudaSuccess)
    return MS_ERR_CUDA;
  stage_event(1, s);
  uint32_t *P = H + (size_t)G * m;  // prefixes (the layout holds 2 L m words)
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
  uint32_t nbins = 0, min_bits = 32;
  for (int p = 0; p < passes; ++p) {
    nbins += 1u << bits[p];
    min_bits = bits[p] < min_bits ? bits[p] : min_bits;
  }
  // the one-pass kernel's per-tile cost is that of 256 buckets and its ranks
  // serialize on shared counters when few buckets take all the keys: it wins
  // only when every digit has >= 7 bits (measured: 4 x 8 bits 88 -> 92 Gkeys/s,
  // but 6 x 5 + 2 bits 66 -> 54, and 8 + 2 bits (m = 1024 top-bit buckets)
  // 130 -> 111)
  if (onesweep_ok(n) && min_bits >= 7u && passes <= (int)kKoMaxPasses && nbins <= kKoMaxBins &&
      g_opt[MS_OPT_SORT].load(std::memory_order_relaxed) == MS_SORT_AUTO) {
    // f1: every digit histogram in one read (KOH), then one KO pass per digit
    cudaStream_t s = (cudaStream_t)stream;
    const OsLayout lo = os_layout(n, (uint32_t)passes, pairs);
    uint32_t *alt_k = (uint32_t *)(w + align_up(lo.total));
    uint32_t *alt_v = pairs ? (uint32_t *)((char *)alt_k + align_up(n * 4u)) : nullptr;
    if (cudaMemsetAsync(w, 0, lo.total, s) != cudaSuccess) return MS_ERR_CUDA;
    KoHistArgs h{};
    h.keys = keys_in;
    h.n = (uint32_t)n;
    h.npass = (uint32_t)passes;
    uint32_t bin0[kKoMaxPasses];
    for (int p = 0, b = 0; p < passes; b += 1 << bits[p], ++p) {
      h.shift[p] = shifts[p];
      h.mask[p] = (1u << bits[p]) - 1u;
      h.bin0[p] = bin0[p] = (uint32_t)b;
    }
    h.nbins = nbins;
    h.gh = (uint32_t *)(w + lo.gh);
    h.hdr = (uint32_t *)w;
    BucketParams none{};
    none.m = 256;
    none.m1 = 255;
    if (counted(Launch<kRadix>::ko_hist(h, none, (uint32_t)sm_count(), s)) != cudaSuccess) return MS_ERR_CUDA;
    const uint32_t *src_k = keys_in, *src_v = vals_in;
    for (int p = 0; p < passes; ++p) {
      const bool to_out = ((passes - 1 - p) % 2) == 0;
      uint32_t *dk = to_out ? keys_out : alt_k;
      uint32_t *dv = to_out ? vals_out : alt_v;
      const ms_bucket_fn fn{MS_BUCKET_RADIX, 1u << bits[p], 0u, shifts[p], bits[p]};
      if (os_pass(make_plan(&fn), pairs, src_k, src_v, dk, dv, (uint32_t)n, lo, w, (uint32_t)p, bin0[p],
                  nullptr, s) != cudaSuccess)
        return MS_ERR_CUDA;
      src_k = dk;
      src_v = dv;
    }
    return MS_SUCCESS;
  }
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
      if (value != MS_PIPELINE_LEVEL0 && value != MS_PIPELINE_TILE && value != MS_PIPELINE_ONESWEEP &&
          value != MS_PIPELINE_AUTO)
        return MS_ERR_INVALID_VALUE;
      break;
    case MS_OPT_SORT:
      if (value != MS_SORT_AUTO && value != MS_SORT_PASSES) return MS_ERR_INVALID_VALUE;
      break;
    default: return MS_ERR_INVALID_VALUE;
  }
  ms::g_opt[option].store(value, std::memory_order_relaxed);
  return MS_SUCCESS;
}

int ms_get_option(int option) {
  return option >= 0 && option < ms::kNumOpts ? ms::g_opt[option].load(std::memory_order_relaxed) : -1;
}

ms_status ms_bucket_delta_default(uint32_t m, ms_bucket_fn *out) {
  if (!out) return MS_ERR_INVALID_VALUE;
  if (m < 1 || m > kMaxLargeM) return MS_ERR_UNSUPPORTED;
  const unsigned long long d = ((1ull << 32) + m - 1) / m;
  *out = ms_bucket_fn{MS_BUCKET_DELTA, m, (uint32_t)(d > 0xFFFFFFFFull ? 0xFFFFFFFFull : d), 0, 0, nullptr};
  return MS_SUCCESS;
}

ms_status ms_bucket_identity(uint32_t m, ms_bucket_fn *out) {
  if (!out) return MS_ERR_INVALID_VALUE;
  if (m < 1 || m > kMaxLargeM) return MS_ERR_UNSUPPORTED;
  *out = ms_bucket_fn{MS_BUCKET_IDENTITY, m, 0, 0, 0};
  return MS_SUCCESS;
}

ms_status ms_bucket_radix(uint32_t shift, uint32_t bits, ms_bucket_fn *out) {
  if (!out) return MS_ERR_INVALID_VALUE;
  if (bits < 1 || bits > 16 || (uint64_t)shift + bits > 32) return MS_ERR_INVALID_VALUE;
  *out = ms_bucket_fn{MS_BUCKET_RADIX, 1u << bits, 0, shift, bits};
  return MS_SUCCESS;
}

ms_status ms_bucket_validate(const ms_bucket_fn *fn) { return validate_fn(fn, true); }

size_t ms_multisplit_workspace_size(uint64_t n, uint32_t m, int with_values) {
  if (m < 1) m = 1;
  if (m > 256) {  // the m > 256 path (either identifier layout: the larger one)
    const size_t a = large_layout(n, MS_BUCKET_DELTA, with_values != 0).total;
    const size_t b = large_layout(n, MS_BUCKET_RADIX, with_values != 0).total;
    return a > b ? a : b;
  }
  const size_t t = layout_for(n, m, with_values != 0).total;
  // the one-pass pipeline (MS_PIPELINE_ONESWEEP) on the same workspace
  const size_t o = n < kKoMaxN ? os_layout(n, 1, with_values != 0).total : 0u;
  return t > o ? t : o;
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
  const size_t smem = ((size_t)kWarps * m + m + 1 + (range ? kHistCells : 0u)) * 4u;
  int ex = 0;
  const bool pow2 = std::frexp((float)delta, &ex) == 0.5f && std::isnormal((float)delta) &&
                    std::isnormal(1.0f / (float)delta);
  if (range)  // the kernel derives the cell scale cells / (s_m - s_0) itself (delta < 0: unset)
    kh_histogram<true, false><<<grid, kThreads, smem, s>>>(x, (uint32_t)n, per, m, 0.f, 0.f, -1.f,
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
  if (r == 0) r = 8;  // library choice: 8-bit digits (4 passes through the wide pipeline, measured fastest)
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
  // or the one-pass sort (f1): up to kKoMaxPasses status blocks
  if (n < kKoMaxN) {
    const size_t o = os_layout(n, kKoMaxPasses, with_values != 0).total;
    ms_ws = o > ms_ws ? o : ms_ws;
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
  e = MS_LAUNCH(merge, pairs, keys_recv, vals_recv, (uint32_t)n_recv, pl.bp, recv_starts,
                merge_offsets, G, keys_out, vals_out, s);
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

// ---------------------------------------------------------------- sharded (Eq.3, GPUs as level 0)
}  // extern "C"

// KPP: the rank's global bucket bases (Eq.3 terms 1-2 with L_0 = G ranks)
//   gb[b] = sum_{b'<b} sum_s C[s][b'] + sum_{s<r} C[s][b],
// the output shard starts pstart[s] = sum_{s'<s} n_s' (n_s = sum_b C[s][b],
// pstart[G] = n_total) and the global bucket offsets gofs[0..m].  One CTA.
static __global__ void __launch_bounds__(256)
    k_shard_plan(const uint32_t *__restrict__ C, uint32_t G, uint32_t r, uint32_t m,
                 uint32_t *__restrict__ gb, uint32_t *__restrict__ pstart,
                 unsigned long long *__restrict__ gofs) {
  __shared__ uint32_t s_w[8];
  __shared__ uint32_t s_n[kMaxPeers];
  const uint32_t b = threadIdx.x, lane = b & 31u, warp = b >> 5;
  uint32_t col = 0, below = 0;
  for (uint32_t sr = 0; sr < G; ++sr) {
    const uint32_t c = b < m ? C[(size_t)sr * m + b] : 0u;
    col += c;
    below += sr < r ? c : 0u;
    uint32_t t = c;  // n_s: block reduction of row s
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xFFFFFFFFu, t, o);
    if (lane == 0) s_w[warp] = t;
    __syncthreads();
    if (b == 0) {
      uint32_t x = 0;
      for (int w = 0; w < 8; ++w) x += s_w[w];
      s_n[sr] = x;
    }
    __syncthreads();
  }
  uint32_t incl = col;  // exclusive scan of the column sums over the buckets
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= (uint32_t)o) incl += y;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  uint32_t wpre = 0;
  for (uint32_t w = 0; w < warp; ++w) wpre += s_w[w];
  const uint32_t A = wpre + incl - col;
  if (b < m) {
    gb[b] = A + below;
    if (gofs) {
      gofs[b] = A;
      if (b == m - 1) gofs[m] = A + col;
    }
  }
  if (b == 0) {
    uint32_t x = 0;
    for (uint32_t sr = 0; sr < G; ++sr) {
      pstart[sr] = x;
      x += s_n[sr];
    }
    pstart[G] = x;
  }
}

struct ms_comm {
  int nranks = 0, rank = 0, device = 0;
  ncclComm_t nccl = nullptr;
  uint32_t *d_scratch = nullptr;  // handle exchange + barrier word
  // registered output windows (KP)
  uint32_t *win_k = nullptr, *win_v = nullptr;
  uint64_t win_n = 0;
  uint32_t *peer_k[kMaxPeers] = {}, *peer_v[kMaxPeers] = {};
  void *opened[2 * kMaxPeers] = {};
  int nopened = 0;
  // NCCL path: pinned host buffers of the plan, and the event of their last H2D
  uint32_t *h_offs = nullptr;
  unsigned char *h_plan = nullptr;
  cudaEvent_t plan_done = nullptr;
};

namespace {

constexpr size_t kShardScratch = 4096;
constexpr size_t kPlanBytes = (size_t)kMaxPeers * 256 * 4 + (kMaxPeers + 1) * 4 + 257 * 8 + 256;

// the KP state after the level-0 layout of the local shard: [C_all G x m][gb m][pstart G+1]
struct ShardLayout {
  Layout lo;
  size_t C, gb, pstart, total;
};
ShardLayout shard_layout(uint64_t n, uint32_t m, uint32_t G, bool pairs) {
  ShardLayout sl{};
  sl.lo = layout_for(n, m, pairs, true);
  sl.C = align_up(sl.lo.total);
  sl.gb = sl.C + align_up((size_t)G * m * 4u);
  sl.pstart = sl.gb + align_up((size_t)m * 4u);
  sl.total = sl.pstart + align_up((size_t)(G + 1) * 4u);
  return sl;
}

bool kp_supported(uint32_t m) {
  return m <= 32 || (g_opt[MS_OPT_RANK].load(std::memory_order_relaxed) == MS_RANK_AUTO &&
                     ms::lane_ordered_inc(false) == 1);
}

ms_status shard_check(const uint32_t *keys_in, uint64_t n, const ms_bucket_fn *fn, void *ws) {
  ms_status st = validate_fn(fn);
  if (st != MS_SUCCESS) return st;
  if (n >= (1ull << 32)) return MS_ERR_UNSUPPORTED;
  if (!ws || ((uintptr_t)ws & (kAlign - 1))) return MS_ERR_INVALID_VALUE;
  if (n > 0 && !keys_in) return MS_ERR_INVALID_VALUE;
  return MS_SUCCESS;
}

ms_status shard_prescan_impl(const uint32_t *keys_in, uint64_t n, const ms_bucket_fn *fn, bool pairs,
                             uint32_t G, uint32_t *counts, void *ws, size_t ws_bytes,
                             cudaStream_t s) {
  ms_status st = shard_check(keys_in, n, fn, ws);
  if (st != MS_SUCCESS) return st;
  const uint32_t m = fn->num_buckets;
  if (!kp_supported(m)) return MS_ERR_UNSUPPORTED;
  const ShardLayout sl = shard_layout(n, m, G, pairs);
  if (ws_bytes < sl.total) return MS_ERR_WORKSPACE;
  char *w = (char *)ws;
  if (n == 0) {
    if (cudaMemsetAsync(w, 0, 8, s) != cudaSuccess) return MS_ERR_CUDA;
    if (counts && cudaMemsetAsync(counts, 0, (size_t)m * 4u, s) != cudaSuccess) return MS_ERR_CUDA;
    return MS_SUCCESS;
  }
  const Plan pl = make_plan(fn);
  L0 l0{};
  if (l0_prescan(pl, pairs, keys_in, (uint32_t)n, sl.lo, w, true, l0, s) != cudaSuccess)
    return MS_ERR_CUDA;
  if (counts && cudaMemcpyAsync(counts, l0.Tot, (size_t)m * 4u, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return MS_ERR_CUDA;
  return MS_SUCCESS;
}

ms_status shard_scatter_impl(const uint32_t *keys_in, const uint32_t *vals_in, uint64_t n,
                             const ms_bucket_fn *fn, const uint32_t *C, uint32_t G, uint32_t r,
                             uint32_t *const *peer_k, uint32_t *const *peer_v,
                             uint64_t *gofs, void *ws, size_t ws_bytes, cudaStream_t s,
                             bool pairs) {
  ms_status st = shard_check(keys_in, n, fn, ws);
  if (st != MS_SUCCESS) return st;
  const uint32_t m = fn->num_buckets;
  if (!kp_supported(m)) return MS_ERR_UNSUPPORTED;
  if (G == 0 || G > kMaxPeers || r >= G || !C || !peer_k) return MS_ERR_INVALID_VALUE;
  if (pairs && (!peer_v || (n > 0 && !vals_in))) return MS_ERR_INVALID_VALUE;
  // peer windows may be NULL only for ranks whose shard is empty (nothing is
  // stored there); this rank's own window must exist when it holds elements
  if (n > 0 && (!peer_k[r] || (pairs && !peer_v[r]))) return MS_ERR_INVALID_VALUE;
  const ShardLayout sl = shard_layout(n, m, G, pairs);
  if (ws_bytes < sl.total) return MS_ERR_WORKSPACE;
  char *w = (char *)ws;
  uint32_t *gb = (uint32_t *)(w + sl.gb), *pstart = (uint32_t *)(w + sl.pstart);
  k_shard_plan<<<1, 256, 0, s>>>(C, G, r, m, gb, pstart, (unsigned long long *)gofs);
  if (counted(cudaGetLastError()) != cudaSuccess) return MS_ERR_CUDA;
  if (n == 0) return MS_SUCCESS;
  const Plan pl = make_plan(fn);
  L0 l0 = l0_setup(m, pairs, sl.lo, w);
  KfArgs a{};
  a.keys_in = keys_in;
  a.vals_in = pairs ? vals_in : nullptr;
  a.keys_out = peer_k[r];
  a.vals_out = pairs ? peer_v[r] : nullptr;
  a.n = (uint32_t)n;
  a.hdr = (uint32_t *)w;
  a.bucket_offsets = nullptr;
  a.use_tma = (((uintptr_t)keys_in & 15u) == 0) && (!pairs || (((uintptr_t)vals_in & 15u) == 0));
  a.store_runs = 0;  // per-element stores into the owners' windows
  a.rank_inc = m > 2 && g_opt[MS_OPT_RANK].load(std::memory_order_relaxed) == MS_RANK_AUTO &&
               ms::lane_ordered_inc(false) == 1;
  a.gbase_ovr = gb;
  a.peer_start = pstart;
  a.npeers = G;
  for (uint32_t d = 0; d < G; ++d) {
    a.peer_k[d] = peer_k[d];
    a.peer_v[d] = pairs ? peer_v[d] : nullptr;
  }
  return l0_postscan(pl, pairs, a, l0, s) == cudaSuccess ? MS_SUCCESS : MS_ERR_CUDA;
}

// NCCL path workspace: [local multisplit ws][stage k, v][recv k, v][offs G x (m+1)][merge G x m][starts G+1]
struct NcclLayout {
  size_t ms, stage_k, stage_v, recv_k, recv_v, offs, merge, starts, total;
};
NcclLayout nccl_layout(uint64_t n, uint32_t m, uint32_t G, bool pairs) {
  NcclLayout L{};
  L.ms = 0;
  const size_t nb = align_up(n * 4u);
  L.stage_k = align_up(ms_multisplit_workspace_size(n, m, pairs));  // the local multisplit's workspace
  L.stage_v = L.stage_k + nb;
  L.recv_k = L.stage_v + (pairs ? nb : 0);
  L.recv_v = L.recv_k + nb;
  L.offs = L.recv_v + (pairs ? nb : 0);
  L.merge = L.offs + align_up((size_t)G * (m + 1) * 4u);
  L.starts = L.merge + align_up((size_t)G * m * 4u);
  L.total = L.starts + align_up((size_t)(G + 1) * 4u);
  return L;
}

ms_status nccl_status(ncclResult_t r) { return r == ncclSuccess ? MS_SUCCESS : MS_ERR_NCCL; }

ms_status sharded_impl(ms_comm *c, const uint32_t *keys_in, const uint32_t *vals_in,
                       uint32_t *keys_out, uint32_t *vals_out, uint64_t n, const ms_bucket_fn *fn,
                       uint64_t *gofs, void *ws, size_t ws_bytes, void *stream, bool pairs) {
  if (!c) return MS_ERR_INVALID_VALUE;
  ms_status st = shard_check(keys_in, n, fn, ws);
  if (st != MS_SUCCESS) return st;
  if (n > 0 && (!keys_out || (pairs && (!vals_in || !vals_out)))) return MS_ERR_INVALID_VALUE;
  if (ws_bytes < ms_sharded_workspace_size(c, n, fn->num_buckets, pairs)) return MS_ERR_WORKSPACE;
  const NcclApi &nc = nccl();
  if (!nc.ok) return MS_ERR_NCCL;
  const uint32_t m = fn->num_buckets, G = (uint32_t)c->nranks, r = (uint32_t)c->rank;
  cudaStream_t s = (cudaStream_t)stream;
  char *w = (char *)ws;
  const bool kp = c->win_k == keys_out && c->win_n == n && (!pairs || c->win_v == vals_out) &&
                  kp_supported(m);
  if (kp) {
    // KP: prescan -> all-gather of the G x m counts -> plan + fused scatter into
    // the owners' windows -> all-reduce of one word as the completion barrier
    const ShardLayout sl = shard_layout(n, m, G, pairs);
    uint32_t *C = (uint32_t *)(w + sl.C);
    st = shard_prescan_impl(keys_in, n, fn, pairs, G, C + (size_t)r * m, ws, ws_bytes, s);
    if (st != MS_SUCCESS) return st;
    if (nc.AllGather(C + (size_t)r * m, C, m, ncclUint32, c->nccl, s) != ncclSuccess) return MS_ERR_NCCL;
    st = shard_scatter_impl(keys_in, vals_in, n, fn, C, G, r, c->peer_k, c->peer_v, gofs, ws, ws_bytes,
                            s, pairs);
    if (st != MS_SUCCESS) return st;
    return nccl_status(nc.AllReduce(c->d_scratch, c->d_scratch, 1, ncclUint32, ncclSum, c->nccl, s));
  }
  // NCCL path: local multisplit -> all-gather of the bucket offsets -> host
  // plan (one D2H + stream sync) -> send / receive of contiguous ranges -> KX merge
  const NcclLayout L = nccl_layout(n, m, G, pairs);
  uint32_t *sk = (uint32_t *)(w + L.stage_k), *sv = (uint32_t *)(w + L.stage_v);
  uint32_t *rk = (uint32_t *)(w + L.recv_k), *rv = (uint32_t *)(w + L.recv_v);
  uint32_t *offs = (uint32_t *)(w + L.offs), *merge = (uint32_t *)(w + L.merge);
  uint32_t *starts = (uint32_t *)(w + L.starts);
  st = multisplit_impl(keys_in, pairs ? vals_in : nullptr, sk, pairs ? sv : nullptr, n, fn,
                       offs + (size_t)r * (m + 1), ws, L.stage_k, stream, pairs);
  if (st != MS_SUCCESS) return st;
  if (nc.AllGather(offs + (size_t)r * (m + 1), offs, m + 1, ncclUint32, c->nccl, s) != ncclSuccess)
    return MS_ERR_NCCL;
  if (c->plan_done && cudaEventSynchronize(c->plan_done) != cudaSuccess) return MS_ERR_CUDA;
  if (cudaMemcpyAsync(c->h_offs, offs, (size_t)G * (m + 1) * 4u, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return MS_ERR_CUDA;
  std::vector<uint64_t> Ch((size_t)G * m), sc(G), sd(G), rc(G), rd(G), go(m + 1);
  for (uint32_t q = 0; q < G; ++q)
    for (uint32_t j = 0; j < m; ++j)
      Ch[(size_t)q * m + j] = c->h_offs[(size_t)q * (m + 1) + j + 1] - c->h_offs[(size_t)q * (m + 1) + j];
  uint32_t *h_merge = (uint32_t *)c->h_plan;
  uint32_t *h_starts = h_merge + (size_t)G * m;
  uint64_t *h_gofs = (uint64_t *)(c->h_plan + align_up(((size_t)G * m + G + 1) * 4u));
  st = ms_shard_plan(Ch.data(), G, m, r, sc.data(), sd.data(), rc.data(), rd.data(), h_merge, h_gofs);
  if (st != MS_SUCCESS) return st;
  uint64_t nrecv = 0;
  for (uint32_t q = 0; q < G; ++q) {
    h_starts[q] = (uint32_t)rd[q];
    nrecv += rc[q];
  }
  h_starts[G] = (uint32_t)nrecv;
  if (cudaMemcpyAsync(merge, h_merge, ((size_t)G * m + G + 1) * 4u, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return MS_ERR_CUDA;
  if (gofs && cudaMemcpyAsync(gofs, h_gofs, (m + 1) * 8u, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return MS_ERR_CUDA;
  if (cudaEventRecord(c->plan_done, s) != cudaSuccess) return MS_ERR_CUDA;
  if (nc.GroupStart() != ncclSuccess) return MS_ERR_NCCL;
  for (uint32_t d = 0; d < G; ++d) {
    if (d == r) continue;
    if (sc[d]) {
      nc.Send(sk + sd[d], sc[d], ncclUint32, (int)d, c->nccl, s);
      if (pairs) nc.Send(sv + sd[d], sc[d], ncclUint32, (int)d, c->nccl, s);
    }
    if (rc[d]) {
      nc.Recv(rk + rd[d], rc[d], ncclUint32, (int)d, c->nccl, s);
      if (pairs) nc.Recv(rv + rd[d], rc[d], ncclUint32, (int)d, c->nccl, s);
    }
  }
  if (nc.GroupEnd() != ncclSuccess) return MS_ERR_NCCL;
  if (sc[r]) {  // this rank's own part: a device copy
    if (cudaMemcpyAsync(rk + rd[r], sk + sd[r], sc[r] * 4u, cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
        (pairs && cudaMemcpyAsync(rv + rd[r], sv + sd[r], sc[r] * 4u, cudaMemcpyDeviceToDevice, s) != cudaSuccess))
      return MS_ERR_CUDA;
  }
  return pairs ? ms_shard_merge_pairs(rk, rv, nrecv, fn, starts, merge, G, keys_out, vals_out, stream)
               : ms_shard_merge_keys(rk, nrecv, fn, starts, merge, G, keys_out, stream);
}

}  // namespace

extern "C" {

size_t ms_shard_workspace_size(uint64_t n_local, uint32_t m, uint32_t G, int with_values) {
  if (m < 1) m = 1;
  if (m > 256) m = 256;
  if (G < 1) G = 1;
  return shard_layout(n_local, m, G, with_values != 0).total;
}

ms_status ms_shard_prescan(const uint32_t *keys_in, uint64_t n_local, const ms_bucket_fn *fn,
                           int with_values, uint32_t G, uint32_t *counts, void *ws, size_t ws_bytes,
                           void *stream) {
  return shard_prescan_impl(keys_in, n_local, fn, with_values != 0, G, counts, ws, ws_bytes,
                            (cudaStream_t)stream);
}

ms_status ms_shard_scatter(const uint32_t *keys_in, const uint32_t *vals_in, uint64_t n_local,
                           const ms_bucket_fn *fn, const uint32_t *C, uint32_t G, uint32_t rank,
                           uint32_t *const *peer_keys, uint32_t *const *peer_vals,
                           uint64_t *global_bucket_offsets, void *ws, size_t ws_bytes, void *stream) {
  return shard_scatter_impl(keys_in, vals_in, n_local, fn, C, G, rank, peer_keys, peer_vals,
                            global_bucket_offsets, ws, ws_bytes, (cudaStream_t)stream,
                            peer_vals != nullptr);
}

ms_status ms_comm_unique_id(void *out128) {
  if (!out128) return MS_ERR_INVALID_VALUE;
  const NcclApi &nc = nccl();
  if (!nc.ok) return MS_ERR_NCCL;
  ncclUniqueId id;
  if (nc.GetUniqueId(&id) != ncclSuccess) return MS_ERR_NCCL;
  std::memcpy(out128, &id, sizeof(id));
  return MS_SUCCESS;
}

ms_status ms_comm_init(ms_comm **out, int nranks, int rank, const void *id128, int cuda_device) {
  if (!out || !id128 || nranks < 1 || nranks > (int)kMaxPeers || rank < 0 || rank >= nranks)
    return MS_ERR_INVALID_VALUE;
  const NcclApi &nc = nccl();
  if (!nc.ok) return MS_ERR_NCCL;
  if (cudaSetDevice(cuda_device) != cudaSuccess) return MS_ERR_CUDA;
  ms_comm *c = new ms_comm();
  c->nranks = nranks;
  c->rank = rank;
  c->device = cuda_device;
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ms_status st = MS_SUCCESS;
  if (nc.CommInitRank(&c->nccl, nranks, id, rank) != ncclSuccess) st = MS_ERR_NCCL;
  if (st == MS_SUCCESS && (cudaMalloc((void **)&c->d_scratch, kShardScratch) != cudaSuccess ||
                           cudaMemset(c->d_scratch, 0, kShardScratch) != cudaSuccess ||
                           cudaMallocHost((void **)&c->h_offs, (size_t)kMaxPeers * 257 * 4) != cudaSuccess ||
                           cudaMallocHost((void **)&c->h_plan, kPlanBytes) != cudaSuccess ||
                           cudaEventCreateWithFlags(&c->plan_done, cudaEventDisableTiming) != cudaSuccess))
    st = MS_ERR_CUDA;
  if (st != MS_SUCCESS) {
    ms_comm_destroy(c);
    return st;
  }
  *out = c;
  return MS_SUCCESS;
}

ms_status ms_comm_check(ms_comm *c) {
  if (!c) return MS_ERR_INVALID_VALUE;
  const NcclApi &nc = nccl();
  if (!nc.ok || !c->nccl) return MS_ERR_NCCL;
  if (!nc.CommGetAsyncError) return MS_SUCCESS;
  ncclResult_t r = ncclSuccess;
  if (nc.CommGetAsyncError(c->nccl, &r) != ncclSuccess) return MS_ERR_NCCL;
  return (r == ncclSuccess || r == ncclInProgress) ? MS_SUCCESS : MS_ERR_NCCL;
}

ms_status ms_comm_abort(ms_comm *c) {
  if (!c) return MS_ERR_INVALID_VALUE;
  const NcclApi &nc = nccl();
  if (c->nccl && nc.CommAbort) {
    nc.CommAbort(c->nccl);
    c->nccl = nullptr;  // ms_comm_destroy still releases the rest
  }
  return MS_SUCCESS;
}

ms_status ms_comm_destroy(ms_comm *c) {
  if (!c) return MS_ERR_INVALID_VALUE;
  for (int i = 0; i < c->nopened; ++i) cudaIpcCloseMemHandle(c->opened[i]);
  if (c->nccl) nccl().CommDestroy(c->nccl);
  if (c->d_scratch) cudaFree(c->d_scratch);
  if (c->h_offs) cudaFreeHost(c->h_offs);
  if (c->h_plan) cudaFreeHost(c->h_plan);
  if (c->plan_done) cudaEventDestroy(c->plan_done);
  delete c;
  return MS_SUCCESS;
}

ms_status ms_comm_register_output(ms_comm *c, uint32_t *keys_out, uint32_t *vals_out,
                                  uint64_t n_local) {
  if (!c || !keys_out) return MS_ERR_INVALID_VALUE;
  const NcclApi &nc = nccl();
  if (!nc.ok) return MS_ERR_NCCL;
  for (int i = 0; i < c->nopened; ++i) cudaIpcCloseMemHandle(c->opened[i]);
  c->nopened = 0;
  c->win_k = c->win_v = nullptr;
  // per rank: {keys handle, keys offset, values handle, values offset, has values}
  struct Rec {
    cudaIpcMemHandle_t hk, hv;
    unsigned long long ok, ov, has_v, pad;
  };
  static_assert(sizeof(Rec) % 16 == 0, "record size");
  Rec mine{};
  // the allocation that holds p (driver entry point: libms does not link libcuda)
  using GetRange = CUresult (*)(CUdeviceptr *, size_t *, CUdeviceptr);
  static GetRange get_range = [] {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<GetRange>(fn);
  }();
  if (!get_range) return MS_ERR_CUDA;
  auto handle = [](void *p, cudaIpcMemHandle_t *h, unsigned long long *off) {
    CUdeviceptr base = 0;
    size_t size = 0;
    if (get_range(&base, &size, (CUdeviceptr)p) != CUDA_SUCCESS) return false;
    *off = (unsigned long long)((CUdeviceptr)p - base);
    return cudaIpcGetMemHandle(h, (void *)base) == cudaSuccess;
  };
  if (c->nranks > 1) {
    if (!handle(keys_out, &mine.hk, &mine.ok)) return MS_ERR_CUDA;
    if (vals_out && !handle(vals_out, &mine.hv, &mine.ov)) return MS_ERR_CUDA;
  }
  mine.has_v = vals_out ? 1u : 0u;
  const size_t rb = sizeof(Rec);
  if (rb * (size_t)c->nranks > kShardScratch) return MS_ERR_UNSUPPORTED;
  unsigned char *d = (unsigned char *)c->d_scratch;
  std::vector<Rec> all(c->nranks);
  if (cudaMemcpy(d + rb * c->rank, &mine, rb, cudaMemcpyHostToDevice) != cudaSuccess) return MS_ERR_CUDA;
  if (nc.AllGather(d + rb * c->rank, d, rb, ncclUint8, c->nccl, nullptr) != ncclSuccess) return MS_ERR_NCCL;
  if (cudaMemcpy(all.data(), d, rb * c->nranks, cudaMemcpyDeviceToHost) != cudaSuccess) return MS_ERR_CUDA;
  if (cudaMemset(c->d_scratch, 0, kShardScratch) != cudaSuccess) return MS_ERR_CUDA;
  for (int q = 0; q < c->nranks; ++q) {
    if (q == c->rank) {
      c->peer_k[q] = keys_out;
      c->peer_v[q] = vals_out;
      continue;
    }
    void *pk = nullptr, *pv = nullptr;
    if (cudaIpcOpenMemHandle(&pk, all[q].hk, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
      return MS_ERR_CUDA;
    c->opened[c->nopened++] = pk;
    c->peer_k[q] = (uint32_t *)((char *)pk + all[q].ok);
    c->peer_v[q] = nullptr;
    if (all[q].has_v) {
      if (std::memcmp(&all[q].hv, &all[q].hk, sizeof(cudaIpcMemHandle_t)) == 0) {
        pv = pk;  // values in the same allocation as the keys
      } else {
        if (cudaIpcOpenMemHandle(&pv, all[q].hv, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
          return MS_ERR_CUDA;
        c->opened[c->nopened++] = pv;
      }
      c->peer_v[q] = (uint32_t *)((char *)pv + all[q].ov);
    }
  }
  c->win_k = keys_out;
  c->win_v = vals_out;
  c->win_n = n_local;
  return MS_SUCCESS;
}

size_t ms_sharded_workspace_size(const ms_comm *c, uint64_t n_local, uint32_t m, int with_values) {
  if (m < 1) m = 1;
  if (m > 256) m = 256;
  const uint32_t G = c ? (uint32_t)c->nranks : 1u;
  const size_t kp = shard_layout(n_local, m, G, with_values != 0).total;
  const size_t nccl_path = nccl_layout(n_local, m, G, with_values != 0).total;
  return kp > nccl_path ? kp : nccl_path;
}

ms_status ms_multisplit_keys_sharded(ms_comm *c, const uint32_t *keys_in, uint32_t *keys_out,
                                     uint64_t n_local, const ms_bucket_fn *fn,
                                     uint64_t *global_bucket_offsets, void *ws, size_t ws_bytes,
                                     void *stream) {
  return sharded_impl(c, keys_in, nullptr, keys_out, nullptr, n_local, fn, global_bucket_offsets, ws,
                      ws_bytes, stream, false);
}

ms_status ms_multisplit_pairs_sharded(ms_comm *c, const uint32_t *keys_in, const uint32_t *vals_in,
                                      uint32_t *keys_out, uint32_t *vals_out, uint64_t n_local,
                                      const ms_bucket_fn *fn, uint64_t *global_bucket_offsets,
                                      void *ws, size_t ws_bytes, void *stream) {
  return sharded_impl(c, keys_in, vals_in, keys_out, vals_out, n_local, fn, global_bucket_offsets, ws,
                      ws_bytes, stream, true);
}

void ms_set_stage_events(void *const *events) { g_stage_events = events; }

uint64_t ms_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

}  // extern "C"
