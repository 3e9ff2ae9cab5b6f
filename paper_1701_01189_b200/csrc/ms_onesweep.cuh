// ms_onesweep.cuh -- SURVEY §8(f) f1: the one-pass fused scan + scatter
// ("Onesweep"), and for the radix sort all digit histograms in one read.
//
// The paper's skeleton is {local count, global scan, local recount + scatter}
// (P:529-540), and its radix sort runs that skeleton once per digit
// (P:1613-1616), i.e. three passes over the keys per digit (48 B/key for four
// 8-bit digits).  P:1617-1619 notes that the same structure is an up-sweep /
// scan / down-sweep; here the scan is folded into the down-sweep:
//
//   KOH ko_hist: one read of the keys computes the global bucket histogram of
//       every pass at once (P passes, all digits of the sort: P:1614 f_k), and
//       the exclusive scan of each is done by the consumer (Eq.2 term 1).
//   KO  ko_onesweep: persistent CTAs take tiles by an atomic ticket (tile
//       order = scheduling order, so every tile a CTA waits on is owned by a
//       running CTA).  Per tile: rank each key inside its warp's slice by
//       lane-ordered increments of warp-private counters (Eq.4 term 1, reading
//       R23), which leave the warp's bucket counts behind (Alg.1's per-
//       subproblem histogram); one scan of the W x 256 counters
//       gives the tile's bucket counts and the slot bases (Eq.4 terms 2-3);
//       the tile publishes its counts and looks back over its predecessors'
//       (decoupled look-back: Eq.2 term 2, sum over l' < l of h_{j,l'});
//       the keys are placed in shared memory in bucket order and written with
//       coalesced runs (Sec.4.7).
//
// Traffic: the sort reads the keys once for the histograms (4 B) and each pass
// reads and writes them once (8 B): 4 + 4 x 8 = 36 B/key for four 8-bit
// digits instead of 48 (pairs: 4 + 4 x 16 = 68 B/pair instead of 80).  A
// one-pass multisplit is 12 B/key, like the two-kernel pipeline.
//
// Look-back status: one 32-bit word per (tile, bucket), flag in bits 31:30
// (01 = tile count only, 10 = inclusive prefix), value in bits 29:0, so
// n < 2^30 (the callers keep larger inputs on the two-kernel pipeline).
#pragma once
#include "ms_wide.cuh"

namespace ms {

constexpr uint32_t kKoBins = 256;               // buckets per pass (m <= 256)
constexpr uint32_t kKoMaxPasses = 8;            // histogram passes of one KOH launch
constexpr uint32_t kKoMaxBins = 1024;           // sum of the passes' bucket counts
constexpr uint32_t kKoFlagAgg = 1u << 30;
constexpr uint32_t kKoFlagInc = 2u << 30;
constexpr uint32_t kKoValMask = (1u << 30) - 1u;
constexpr uint32_t kKoMaxN = 1u << 30;

// KO CTA shape: W compute warps x 16 windows (tile T = 512 W) and LBW look-
// back warps: keys 24 + 8 warps (12288 keys, 64 registers), pairs 16 + 8
// warps (8192 pairs, 80 registers); one CTA per SM, three tile stages.  (The
// inline look-back, LBW = 0, stays compilable for measurements.)
#ifndef KO_KEYS_W
#define KO_KEYS_W 24
#endif
#ifndef KO_KEYS_LBW
#define KO_KEYS_LBW 8
#endif
#ifndef KO_PAIRS_W
#define KO_PAIRS_W 16
#endif
#ifndef KO_PAIRS_LBW
#define KO_PAIRS_LBW 8
#endif
__host__ __device__ constexpr uint32_t ko_warps(bool pairs) { return pairs ? KO_PAIRS_W : KO_KEYS_W; }
__host__ __device__ constexpr uint32_t ko_lb_warps(bool pairs) { return pairs ? KO_PAIRS_LBW : KO_KEYS_LBW; }
__host__ __device__ constexpr uint32_t ko_threads(bool pairs) { return 32u * (ko_warps(pairs) + ko_lb_warps(pairs)); }
__host__ __device__ constexpr uint32_t ko_tile(bool pairs) { return 512u * ko_warps(pairs); }
// stages [3][T (+T values)] | counters [W][256] | s_tab [2][256] | (LBW) s_tot,
// s_tb [2][256], s_gb [256]   (keys 175 KB, pairs 219 KB)
__host__ __device__ inline size_t ko_smem_bytes(bool pairs) {
  const uint32_t T = ko_tile(pairs);
  return (3u * T * (pairs ? 2u : 1u) + ko_warps(pairs) * kKoBins + (ko_lb_warps(pairs) ? 7u : 2u) * kKoBins) * 4u;
}

struct KoHistArgs {
  const uint32_t *keys;
  uint32_t n;
  uint32_t npass;
  uint32_t shift[kKoMaxPasses];  // RADIX passes: bucket (u >> shift) & mask
  uint32_t mask[kKoMaxPasses];
  uint32_t bin0[kKoMaxPasses];   // first bin of pass p in gh
  uint32_t nbins;                // sum of the passes' bucket counts
  uint32_t *gh;                  // [nbins] global counts (zeroed by the caller)
  uint32_t *hdr;                 // [0] key-domain error flag
};

__device__ __forceinline__ void red_shared_inc(uint32_t saddr) {
  asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(saddr) : "memory");
}

// ============================================================================
// KOH.  Counters are lane columns, cnt[bin][lane] at bin * 32 + lane: a warp's
// increments hit 32 distinct banks whatever the keys (no conflicts, no
// same-address serialization under skew); warps share the columns through
// shared-memory reductions.  Each thread holds 16 keys (four 16-byte loads in
// flight) and counts them pass by pass, so the per-pass parameters are loaded
// once per 16 keys.  Non-RADIX kinds (the one-pass multisplit) have one pass,
// f = bucket_of<KIND>.
// ============================================================================
template <int KIND, bool BYTES>
__global__ void __launch_bounds__(1024, 1) ko_hist(KoHistArgs a, BucketParams bp) {
  MS_STAGE_SPLITTERS(bp, kMaxBuckets);
  extern __shared__ __align__(16) uint32_t koh_cnt[];  // [nbins][32]
  const uint32_t tid = threadIdx.x, lane = tid & 31u;
  for (uint32_t i = tid; i < a.nbins * 32u; i += blockDim.x) koh_cnt[i] = 0u;
  __syncthreads();
  const uint32_t cbase = smem_u32(koh_cnt) + lane * 4u;
  bool derr = false;
  auto count = [&](const uint32_t *u, int cnt) {
    if constexpr (KIND == kRadix && BYTES) {
      // the 4 x 8-bit sort: digit p is byte p (one PRMT), bins of pass p at
      // the constant offset p * 256 * 32 words (an immediate of the reduction)
#pragma unroll
      for (uint32_t p = 0; p < 4; ++p)
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (j < cnt) red_shared_inc(cbase + (__byte_perm(u[j], 0u, 0x4440u + p) << 7) + p * 256u * 128u);
    } else if constexpr (KIND == kRadix) {
#pragma unroll 1
      for (uint32_t p = 0; p < a.npass; ++p) {
        const uint32_t sh = a.shift[p], mk = a.mask[p], b0 = cbase + (a.bin0[p] << 7);
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (j < cnt) red_shared_inc(b0 + (((u[j] >> sh) & mk) << 7));
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < cnt) {
          if constexpr (KIND == kIdentity) derr |= key_domain_error<KIND>(u[j], bp);
          red_shared_inc(cbase + (bucket_of<KIND>(u[j], bp) << 7));
        }
    }
  };
  const bool aligned = (reinterpret_cast<uintptr_t>(a.keys) & 15u) == 0;
  const uint32_t nv = aligned ? a.n / 4u : 0u;  // 16-byte vectors
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint4 *v = reinterpret_cast<const uint4 *>(a.keys);
  uint32_t i = blockIdx.x * blockDim.x + tid;
  uint32_t u[16];
  for (; i + 3u * stride < nv; i += 4u * stride) {  // four vectors in flight per thread
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint4 q = ldg_stream_v4(v + i + (uint32_t)j * stride);
      u[4 * j] = q.x;
      u[4 * j + 1] = q.y;
      u[4 * j + 2] = q.z;
      u[4 * j + 3] = q.w;
    }
    count(u, 16);
  }
  for (; i < nv; i += stride) {
    const uint4 q = ldg_stream_v4(v + i);
    u[0] = q.x;
    u[1] = q.y;
    u[2] = q.z;
    u[3] = q.w;
    count(u, 4);
  }
  for (uint32_t e = nv * 4u + blockIdx.x * blockDim.x + tid; e < a.n; e += stride) {
    u[0] = __ldg(a.keys + e);
    count(u, 1);
  }
  if constexpr (KIND == kIdentity) {
    if (__any_sync(0xFFFFFFFFu, derr) && lane == 0) atomicOr(a.hdr, 1u);
  }
  __syncthreads();
  for (uint32_t b = tid; b < a.nbins; b += blockDim.x) {
    uint32_t s = 0;
#pragma unroll 8
    for (uint32_t j = 0; j < 32u; ++j) s += koh_cnt[(b << 5) + ((j + b) & 31u)];  // rotated: no conflicts
    if (s) atomicAdd(a.gh + b, s);
  }
}

struct KoArgs {
  const uint32_t *keys_in;
  const uint32_t *vals_in;
  uint32_t *keys_out;
  uint32_t *vals_out;
  uint32_t n;
  uint32_t num_tiles;
  const uint32_t *gh;      // [256] this pass's global bucket counts (KOH)
  uint32_t *status;        // [num_tiles][256] look-back words (zeroed by the caller)
  uint32_t *ticket;        // tile ticket counter (zeroed by the caller)
  uint32_t *hdr;           // [0] key-domain error flag
  uint32_t *bucket_offsets;  // m + 1 words, or null
  int use_tma;             // inputs 16-byte aligned: tiles by TMA bulk copies
};

__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// eight consecutive status words (one 32-byte sector, 32-byte aligned)
__device__ __forceinline__ void ld_relaxed_v8(const uint32_t *p, uint32_t (&v)[8]) {
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "l"(p) : "memory");
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]) : "l"(p + 4) : "memory");
}
__device__ __forceinline__ void st_relaxed_u32(uint32_t *p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ============================================================================
// KO: persistent, one CTA per SM, three tile stages.  A tile's stage holds its
// keys (+ values), then the same tile in bucket order.  The scatter of a tile
// is deferred by one iteration, so its look-back (the only wait on other CTAs)
// overlaps the next tile's work.  Iteration k (tile t_k in stage k % 3) of the
// W compute warps:
//   load the warp's 16 windows into registers (TMA'd stage, or global loads
//   for a ragged / unaligned tile); rank into the warp's counter row;
//   B1; 256 threads (one per bucket) total the W x 256 counts, publish the
//       tile count, scan the counts over the buckets (B2 among those 256) and
//       turn the counters into slot bases (tile base + earlier warps' counts);
//   B3; each warp places its keys (slot = base + rank) and zeroes its own row
//       (no other warp reads it before the next B1);
//   every warp scatters tile k-1.
// The look-back of tile k walks its predecessors' status words, R rows per
// round trip, publishes the inclusive prefix of tile k and of the first
// window's rows that held only tile counts (the same values whoever writes
// them: later walkers stop sooner), and writes the scatter offsets.  With
// LBW = 8 (keys) it runs in eight dedicated look-back warps, one bucket per
// thread, handed the tile through an mbarrier, so no compute warp waits on it
// (keys and pairs); with LBW = 0 the 256 scan threads run it after placing the
// tile (measured slower: 2^28-pair pass 1287 vs 1040 us).
// ============================================================================
__host__ __device__ constexpr uint32_t ko_stages() { return 3u; }

// Phase timing for the standalone harness (scripts/ko_harness.cu): compiled
// out of the library.  Lane 0 of warps 0 (a scan warp) and W-1 accumulate
// clock() deltas per phase into ko_timing[block][2][kKoPhases].
constexpr int kKoPhases = 8;
#ifdef MS_KO_TIMING
__device__ unsigned long long ko_timing[1024][2][kKoPhases];
__device__ unsigned long long ko_lbstat[4];  // windows, spins, -, -
#define KO_LB(i, v) do { if (lb == 0) atomicAdd(&ko_lbstat[i], (unsigned long long)(v)); } while (0)
#define KO_T0() uint32_t ko_last_ = (uint32_t)clock(); uint32_t ko_acc_[kKoPhases] = {0, 0, 0, 0, 0, 0, 0, 0}
#define KO_T(i) do { const uint32_t c_ = (uint32_t)clock(); ko_acc_[i] += c_ - ko_last_; ko_last_ = c_; } while (0)
#define KO_TDONE() do { if (lane == 0 && (warp == 0 || warp == W - 1)) { \
    for (int q_ = 0; q_ < kKoPhases; ++q_) ko_timing[blockIdx.x][warp == 0 ? 0 : 1][q_] += ko_acc_[q_]; } } while (0)
#else
#define KO_LB(i, v) do { } while (0)
#define KO_T0() do { } while (0)
#define KO_T(i) do { } while (0)
#define KO_TDONE() do { } while (0)
#endif
#ifndef KO_R
#define KO_R 2  // look-back rows per round trip, scan threads (measured: 2-3 > 4 > 8; 1 is slower)
#endif
#ifndef KO_CH
#define KO_CH 4  // scatter chunk, slots per thread per round (measured: 4 > 2, 8 > 1, 16)
#endif
#ifndef KO_RL
#define KO_RL 2  // look-back rows per round trip, dedicated look-back warps
#endif
#ifndef KO_SLEEP
#define KO_SLEEP 1
#endif
#if KO_SLEEP
#define KO_WAIT(b, p) mbar_wait_sleep(b, p)
#else
#define KO_WAIT(b, p) mbar_wait(b, p)
#endif

// Look-back of tile t for bucket b (Eq.2 term 2): returns sum_{l < t} h_{b,l}
// and publishes the inclusive prefix of t (tot = h_{b,t}).  v: the status words
// of tiles t-1 .. t-R, possibly loaded earlier (a zero flag is re-read).
template <uint32_t R>
__device__ __forceinline__ uint32_t ko_lookback(uint32_t *status, uint32_t t, uint32_t b, uint32_t tot,
                                                uint32_t (&v)[R], uint32_t lb) {
  constexpr uint32_t NB = kKoBins;
  if (t == 0) return 0u;
  uint32_t excl = 0, pre[R];  // pre[q]: sum of the first window's rows nearer than row t-1-q
#ifdef MS_KO_TIMING
  uint32_t nwin = 1, spins = 0;
#endif
  bool done = false;
  auto take_row = [&](uint32_t row, uint32_t x) {
    while ((x & ~kKoValMask) == 0u) {
#ifdef MS_KO_TIMING
      ++spins;
#endif
      x = ld_relaxed_u32(status + (size_t)row * NB + b);
    }
    excl += x & kKoValMask;
    done = (x & kKoFlagInc) != 0u;
    return x;
  };
#pragma unroll
  for (uint32_t q = 0; q < R; ++q) {
    pre[q] = excl;
    if (!done && q < t)
      v[q] = take_row(t - 1u - q, v[q]);
    else
      v[q] = kKoFlagInc;  // not walked: no fix-up
  }
  for (uint32_t p = t > R ? t - R : 0u; !done;) {  // further windows: rows p-1, p-2, ...
#ifdef MS_KO_TIMING
    ++nwin;
#endif
    uint32_t u[R];
#pragma unroll
    for (uint32_t q = 0; q < R; ++q) u[q] = q < p ? ld_relaxed_u32(status + (size_t)(p - 1u - q) * NB + b) : 0u;
#pragma unroll
    for (uint32_t q = 0; q < R; ++q)
      if (!done && q < p) take_row(p - 1u - q, u[q]);
    p = p > R ? p - R : 0u;
  }
  st_relaxed_u32(status + (size_t)t * NB + b, kKoFlagInc | (excl + tot));
#pragma unroll
  for (uint32_t q = 0; q < R; ++q)
    if (!(v[q] & kKoFlagInc)) st_relaxed_u32(status + (size_t)(t - 1u - q) * NB + b, kKoFlagInc | (excl - pre[q]));
#ifdef MS_KO_TIMING
  KO_LB(0, nwin);
  KO_LB(1, spins);
#endif
  return excl;
}

template <int KIND, bool PAIRS>
__global__ void __launch_bounds__((ko_warps(PAIRS) + ko_lb_warps(PAIRS)) * 32, 1)
    ko_onesweep(KoArgs a, BucketParams bp) {
  MS_STAGE_SPLITTERS(bp, kMaxBuckets);  // 1 KB of splitters + the 4 KB cell table
  constexpr uint32_t W = ko_warps(PAIRS), NC = W * 32u, ITEMS = 16u, T = NC * ITEMS;
  constexpr uint32_t LBW = ko_lb_warps(PAIRS);
  constexpr uint32_t SWD = T * (PAIRS ? 2u : 1u);  // words per stage
  constexpr uint32_t NB = kKoBins, NS = ko_stages(), R = KO_R;
  constexpr uint32_t kBarC = 1, kBarS = 2;  // named barriers: compute warps, 256 scan threads
  static_assert(LBW == 0 || LBW * 32u == NB, "one look-back thread per bucket");
  extern __shared__ __align__(128) uint32_t ko_smem[];
  uint32_t *stage0 = ko_smem;
  uint32_t *cnt = stage0 + NS * SWD;  // [W][NB] warp-private counters, then slot bases
  uint32_t *s_tab = cnt + W * NB;     // [2][NB] global position minus tile slot, by iteration parity
  uint32_t *s_tot = s_tab + 2u * NB;  // LBW: [2][NB] tile counts, [2][NB] tile bases, [NB] bucket bases
  uint32_t *s_tb = s_tot + 2u * NB;
  uint32_t *s_gb = s_tb + 2u * NB;
  __shared__ __align__(8) uint64_t full[NS];
  __shared__ __align__(8) uint64_t aggb[2];  // LBW: tile handed to the look-back warps
  __shared__ __align__(8) uint64_t tabr[2];  // LBW: its scatter offsets are ready
  __shared__ uint32_t s_tile[NS];
  __shared__ uint32_t s_lbt[2];  // LBW: tile of the hand-off, ~0u: no more tiles
  __shared__ uint32_t s_wsum[NB / 32u];
  __shared__ uint32_t s_hot;
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
  constexpr uint32_t kProducer = NC - 32u;  // outside the scan threads
  auto tile_n = [&](uint32_t t) { return min(T, a.n - t * T); };
  auto via_tma = [&](uint32_t t) { return a.use_tma && tile_n(t) == T; };
  auto issue = [&](uint32_t st, uint32_t t) {  // producer: tile t into stage st
    s_tile[st] = t;
    if (t < a.num_tiles && via_tma(t)) {
      uint32_t *dst = stage0 + st * SWD;
      const uint64_t pol = policy_evict_first();
      mbar_arrive_expect_tx(&full[st], T * 4u * (PAIRS ? 2u : 1u));
      tma_load_1d(dst, a.keys_in + (size_t)t * T, T * 4u, &full[st], pol);
      if constexpr (PAIRS) tma_load_1d(dst + T, a.vals_in + (size_t)t * T, T * 4u, &full[st], pol);
    }
  };
  if (tid == kProducer) {
    for (uint32_t i = 0; i < NS; ++i) mbar_init(&full[i], 1);
    for (uint32_t i = 0; i < 2; ++i) {
      mbar_init(&aggb[i], NB);
      mbar_init(&tabr[i], NB);
    }
    issue(0, atomicAdd(a.ticket, 1u));
    issue(1, atomicAdd(a.ticket, 1u));
  }
  for (uint32_t i = tid; i < W * NB; i += blockDim.x) cnt[i] = 0u;
  // bucket bases (Eq.2 term 1): exclusive scan of the global counts; the hot
  // bucket (more than 1/16 of all keys) ranks by ballots (same-address
  // increments with a return value serialize)
  uint32_t gbase = 0;
  if (tid < NB) {
    const uint32_t c = tid < bp.m ? __ldg(a.gh + tid) : 0u;
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= (uint32_t)o) incl += y;
    }
    if (lane == 31) s_wsum[warp] = incl;
    gbase = incl - c;
    const uint32_t top = __reduce_max_sync(0xFFFFFFFFu, c);
    if (tid == 0) s_hot = 0u;
    if (lane == 0) s_tab[warp] = top;  // scratch: per-warp maxima
  }
  __syncthreads();
  if (tid < NB) {
    uint32_t top = 0;
#pragma unroll
    for (uint32_t j = 0; j < NB / 32u; ++j) {
      gbase += j < warp ? s_wsum[j] : 0u;
      top = max(top, s_tab[j]);
    }
    const uint32_t c = tid < bp.m ? __ldg(a.gh + tid) : 0u;
    if (blockIdx.x == 0 && a.bucket_offsets && tid < bp.m) {
      a.bucket_offsets[tid] = gbase;
      if (tid + 1u == bp.m) a.bucket_offsets[bp.m] = gbase + c;
    }
    if constexpr (LBW > 0) s_gb[tid] = gbase;
    // the lowest bucket holding the maximum count, if it is hot
    const uint32_t who = __ballot_sync(0xFFFFFFFFu, c == top && top > a.n / 16u);
    if (who && lane == __ffs(who) - 1) atomicMax(&s_hot, 0x80000000u | (NB - 1u - tid));
  }
  __syncthreads();

  if constexpr (LBW > 0) {
    if (warp >= W) {
      // ========================= look-back warps ==============================
      const uint32_t lb = tid - NC;  // this thread's bucket
      const uint32_t gb = s_gb[lb];
      for (uint32_t i = 0;; ++i) {
        const uint32_t par = i & 1u;
        KO_WAIT(&aggb[par], (i >> 1) & 1u);
        const uint32_t t = s_lbt[par];
        if (t == ~0u) break;
        constexpr uint32_t RL = KO_RL;
        uint32_t v[RL];
#pragma unroll
        for (uint32_t q = 0; q < RL; ++q) v[q] = q < t ? ld_relaxed_u32(a.status + (size_t)(t - 1u - q) * NB + lb) : 0u;
        const uint32_t excl = ko_lookback<RL>(a.status, t, lb, s_tot[par * NB + lb], v, lb);
        s_tab[par * NB + lb] = gb + excl - s_tb[par * NB + lb];
        mbar_arrive(&tabr[par]);
      }
      return;
    }
  }

  // ============================== compute warps ===============================
  const uint32_t hot = s_hot ? NB - 1u - (s_hot & 0x7FFFFFFFu) : ~0u;
  KO_T0();
  auto csync = [&]() {
    if constexpr (LBW > 0)
      named_barrier_sync(kBarC, NC);
    else
      __syncthreads();
  };
  // ---- coalesced scatter of a placed tile: slot s of bucket b -> tab[b] + s
  auto scatter = [&](uint32_t t, uint32_t it) {  // tile t of iteration it
    if constexpr (LBW > 0) KO_WAIT(&tabr[it & 1u], (it >> 1) & 1u);
    const uint32_t *s_stage = stage0 + (it % NS) * SWD;
    const uint32_t *tab = s_tab + (it & 1u) * NB;
    const uint32_t tn = tile_n(t);
    const uint32_t s0 = warp * (ITEMS * 32u) + lane;
    constexpr uint32_t CH = KO_CH;
#pragma unroll
    for (uint32_t c = 0; c < ITEMS; c += CH) {
      uint32_t kk[CH], vv[PAIRS ? CH : 1], pos[CH];
#pragma unroll
      for (uint32_t i = 0; i < CH; ++i) {
        if constexpr (PAIRS) {
          const uint2 kv = reinterpret_cast<const uint2 *>(s_stage)[s0 + 32u * (c + i)];
          kk[i] = kv.x;
          vv[i] = kv.y;
        } else {
          kk[i] = s_stage[s0 + 32u * (c + i)];
        }
      }
#pragma unroll
      for (uint32_t i = 0; i < CH; ++i) pos[i] = tab[bucket_of<KIND>(kk[i], bp)] + s0 + 32u * (c + i);
      if (tn == T) {
#pragma unroll
        for (uint32_t i = 0; i < CH; ++i) a.keys_out[pos[i]] = kk[i];
        if constexpr (PAIRS) {
#pragma unroll
          for (uint32_t i = 0; i < CH; ++i) a.vals_out[pos[i]] = vv[i];
        }
      } else {
#pragma unroll
        for (uint32_t i = 0; i < CH; ++i)
          if (s0 + 32u * (c + i) < tn) {
            a.keys_out[pos[i]] = kk[i];
            if constexpr (PAIRS) a.vals_out[pos[i]] = vv[i];
          }
      }
    }
  };

  uint32_t key[ITEMS];
  uint32_t val[PAIRS ? ITEMS : 1];
  uint32_t br[ITEMS];  // (bucket << 16) | rank inside the warp's slice
  const uint32_t wbase = warp * (ITEMS * 32u);
  uint32_t *crow = cnt + warp * NB;
  uint32_t phase = 0;  // mbarrier parity bit per stage
  uint32_t tprev = 0;  // tile of the previous iteration (scattered in this one)
  bool derr = false;
  uint32_t k = 0;
  for (;; ++k) {
    const uint32_t st = k % NS;
    const uint32_t t = s_tile[st];
    if (t >= a.num_tiles) break;
    uint32_t *s_stage = stage0 + st * SWD;
    const uint32_t tn = tile_n(t);
    // ---- load the warp's windows
    if (via_tma(t)) {
      mbar_wait(&full[st], (phase >> st) & 1u);
      phase ^= 1u << st;
      KO_T(0);
#pragma unroll
      for (uint32_t i = 0; i < ITEMS; ++i) key[i] = s_stage[wbase + 32u * i + lane];
      if constexpr (PAIRS) {
#pragma unroll
        for (uint32_t i = 0; i < ITEMS; ++i) val[i] = s_stage[T + wbase + 32u * i + lane];
      }
    } else {
      const size_t g = (size_t)t * T;
#pragma unroll
      for (uint32_t i = 0; i < ITEMS; ++i) {
        const uint32_t e = wbase + 32u * i + lane;
        key[i] = e < tn ? __ldg(a.keys_in + g + e) : 0u;
        if constexpr (PAIRS) val[i] = e < tn ? __ldg(a.vals_in + g + e) : 0u;
      }
    }
    // ---- rank (Eq.4 term 1): lane-ordered increments of the warp's counters
    if (tn == T) {
      if (hot != ~0u) {
        const uint32_t lt = lanemask_lt();
        uint32_t hc = 0;
#pragma unroll
        for (uint32_t i = 0; i < ITEMS; ++i) {
          const uint32_t b = bucket_of<KIND>(key[i], bp);
          if constexpr (KIND == kIdentity) derr |= key_domain_error<KIND>(key[i], bp);
          const uint32_t hm = __ballot_sync(0xFFFFFFFFu, b == hot);
          const uint32_t r = b == hot ? hc + __popc(hm & lt) : atomicAdd(crow + b, 1u);
          hc += __popc(hm);
          br[i] = (b << 16) | r;
        }
        if (lane == 0) crow[hot] = hc;  // the hot bucket's counter is this warp's alone
      } else {
        uint32_t bk[ITEMS];
#pragma unroll
        for (uint32_t i = 0; i < ITEMS; ++i) bk[i] = bucket_of<KIND>(key[i], bp);
#pragma unroll
        for (uint32_t i = 0; i < ITEMS; ++i) {
          if constexpr (KIND == kIdentity) derr |= key_domain_error<KIND>(key[i], bp);
          br[i] = (bk[i] << 16) | atomicAdd(crow + bk[i], 1u);
        }
      }
    } else {
#pragma unroll
      for (uint32_t i = 0; i < ITEMS; ++i) {
        br[i] = 0u;
        if (wbase + 32u * i + lane < tn) {
          const uint32_t b = bucket_of<KIND>(key[i], bp);
          if constexpr (KIND == kIdentity) derr |= key_domain_error<KIND>(key[i], bp);
          br[i] = (b << 16) | atomicAdd(crow + b, 1u);
        }
      }
    }
    KO_T(1);
    csync();  // B1: counts complete; every stage read and the scatter of tile k-2 done
    KO_T(2);
    if (tid == kProducer && k > 0) {
      fence_proxy_async_smem();
      issue((k + 1u) % NS, atomicAdd(a.ticket, 1u));
    }
    // ---- per bucket: tile count (publish), first look-back window, scan
    // (two threads per bucket, each half of the rows, measured slower: the
    // pair shares the bucket's bank)
    uint32_t tot = 0, tb = 0;
    uint32_t v[R];  // status words of tiles t-1 .. t-R (thread b's bucket)
    if (tid < NB) {
#pragma unroll 8
      for (uint32_t w = 0; w < W; ++w) tot += cnt[w * NB + tid];
      st_relaxed_u32(a.status + (size_t)t * NB + tid, (t == 0 ? kKoFlagInc : kKoFlagAgg) | tot);
      if constexpr (LBW == 0) {
#pragma unroll
        for (uint32_t q = 0; q < R; ++q)
          v[q] = q < t ? ld_relaxed_u32(a.status + (size_t)(t - 1u - q) * NB + tid) : 0u;
      }
      uint32_t incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= (uint32_t)o) incl += y;
      }
      if (lane == 31) s_wsum[warp] = incl;
      tb = incl - tot;
      named_barrier_sync(kBarS, NB);  // B2
#pragma unroll
      for (uint32_t j = 0; j < NB / 32u; ++j) tb += j < warp ? s_wsum[j] : 0u;
      uint32_t run = tb;  // slot base of warp w's bucket-tid keys: tb + sum_{w'<w} c_{w'}
#pragma unroll 8
      for (uint32_t w = 0; w < W; ++w) {
        const uint32_t c = cnt[w * NB + tid];
        cnt[w * NB + tid] = run;
        run += c;
      }
      if constexpr (LBW > 0) {  // hand the tile to the look-back warps
        s_tot[(k & 1u) * NB + tid] = tot;
        s_tb[(k & 1u) * NB + tid] = tb;
        if (tid == 0) s_lbt[k & 1u] = t;
        mbar_arrive(&aggb[k & 1u]);
      }
    }
    KO_T(3);
    csync();  // B3
    KO_T(5);
    // ---- place in bucket order (in place: every warp holds its windows)
#pragma unroll
    for (uint32_t i = 0; i < ITEMS; ++i) {
      if (tn == T || wbase + 32u * i + lane < tn) {
        const uint32_t slot = crow[br[i] >> 16] + (br[i] & 0xFFFFu);
        if constexpr (PAIRS)
          reinterpret_cast<uint2 *>(s_stage)[slot] = make_uint2(key[i], val[i]);
        else
          s_stage[slot] = key[i];
      }
    }
    __syncwarp();
#pragma unroll
    for (uint32_t j = 0; j < NB / 128u; ++j)  // this warp's row, for its next tile
      reinterpret_cast<uint4 *>(crow)[lane + 32u * j] = make_uint4(0u, 0u, 0u, 0u);
    KO_T(6);
    if constexpr (LBW == 0) {  // the look-back of tile k, here by the scan threads
      if (tid < NB) {
        const uint32_t lb = tid;
        const uint32_t excl = ko_lookback<R>(a.status, t, lb, tot, v, lb);
        s_tab[(k & 1u) * NB + tid] = gbase + excl - tb;
      }
    }
    KO_T(7);
    // ---- the previous tile
    if (k > 0) scatter(tprev, k - 1u);
    KO_T(4);
    tprev = t;
  }
  if constexpr (LBW > 0) {  // no more tiles: release the look-back warps
    if (tid < NB) {
      if (tid == 0) s_lbt[k & 1u] = ~0u;
      mbar_arrive(&aggb[k & 1u]);
    }
  }
  if (k > 0) {
    csync();  // the last tile placed (and, LBW = 0, looked back)
    scatter(tprev, k - 1u);
  }
  KO_TDONE();
  if constexpr (KIND == kIdentity) {
    if (__any_sync(0xFFFFFFFFu, derr) && lane == 0) atomicOr(a.hdr, 1u);
  }
}

}  // namespace ms
