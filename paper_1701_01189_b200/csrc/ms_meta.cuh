// ms_meta.cuh -- the m <= 32 pipeline with warp-level offsets computed in the
// prescan (KM) instead of the postscan (KF):
//
//   KM  km_tile_meta (P:534-535 prescan, extended): for every tile l of its
//       level-0 range and every warp slice w of the tile, the per-warp bucket
//       counts c_{l,w}[j], then the tile-local exclusive scan in (bucket, warp)
//       order S_l[j][w] = sum_{j'<j} h_{l}[j'] + sum_{w'<w} c_{l,w'}[j]
//       (Eq.4 terms 2-3).  It writes them as one "tile meta" record
//       per tile, and the range histogram R[c][j] for the level-0 scan (KR).
//       KF accumulates the range-running prefix sum_{l'<l} h_{l'}[j] (Eq.3
//       term 3) itself from the records' tile counts.
//   KF  kf_meta: per tile, each warp reads its m slot bases from the meta
//       record (TMA'd with the tile), ranks its windows (Eq.4 term 1) and
//       places the keys in shared memory in place; one CTA barrier per tile,
//       then the coalesced scatter of the bucket runs.
//
// Why (B200, measured in profiles/r01/s2_summary.md): the postscan is
// issue-bound (43 thread-instructions per key, 52 % issue utilisation, 27 % of
// warp samples parked at the post-count barrier) while the prescan streams at
// ~5.5 TB/s with 77 % of its issue slots idle.  The count pass and the
// redundant per-warp scan (16.5 instructions per key) move to the prescan;
// the price is one meta record per tile, 16 m words, i.e. 0.25 B/key
// written and read again at m = 32 (the paper recomputes instead, P:778
// footnote, which was the right trade on a GPU whose postscan was not
// issue-bound).
#pragma once
#include <type_traits>

#include "ms_kernels.cuh"

namespace ms {

// meta record: [S: W x mS words, warp-major: S[w][j] at w*mS + j][pad to 16 B]; the
// range-running prefix (Eq.3 term 3) is accumulated by KF from the tile counts
__host__ __device__ constexpr uint32_t meta_stride(uint32_t mS, uint32_t W) {
  return (mS * W + 3u) & ~3u;
}
__host__ __device__ constexpr uint32_t meta_ms(uint32_t m) { return m < 2 ? 2u : m; }

// ============================================================================
// KM: per-tile warp-slice counts -> tile meta records + range histogram.
// CTA c handles tiles [c*K, min(L, (c+1)*K)) -- the same partition as KF.
// Warp w of the CTA counts slice w of each tile: keys [l*T + w*SL, +SL).
// ============================================================================
// KM: keys-only tiles of T = 512 ITEMS words in a TMA ring of KS stages.
// 16 counting warps (one slice of each tile each) and one scan warp that owns
// the TMA ring and turns each tile's W x m counts into its meta record; the
// two roles hand over through mbarriers (count buffers double-buffered by tile
// parity), so no counting warp ever waits at a CTA barrier.
__host__ __device__ constexpr uint32_t km_stages(int items) { return items >= 16 ? 3u : 5u; }
__host__ __device__ inline size_t km_smem_bytes(uint32_t m, bool pairs) {
  const int items = pairs ? 8 : 16;
  return ((size_t)km_stages(items) * kThreads * items + 2u * kWarps * meta_ms(m)) * 4u;
}

template <int KIND, bool SMALLM, int ITEMS>
__global__ void __launch_bounds__(kThreads + 32, 2)
    km_tile_meta(const uint32_t *__restrict__ keys, uint32_t n, uint32_t num_tiles,
                 uint32_t tiles_per_cta, BucketParams bp, uint32_t *__restrict__ meta,
                 uint32_t *__restrict__ R, uint32_t *__restrict__ hdr) {
  MS_STAGE_SPLITTERS(bp, 32);
  constexpr uint32_t W = kWarps;
  constexpr uint32_t SL = 32u * ITEMS;  // keys per warp slice
  constexpr uint32_t T = W * SL;
  constexpr int NV = ITEMS / 4;         // uint4 per lane per slice
  constexpr uint32_t KS = km_stages(ITEMS);
  extern __shared__ __align__(128) uint32_t km_smem[];  // stages [KS][T] | cnt[2][W][mS]
  __shared__ __align__(8) uint64_t full[KS];
  __shared__ __align__(8) uint64_t cfull[2];   // counts of a tile complete (512 arrivals)
  __shared__ __align__(8) uint64_t cempty[2];  // counts consumed and zeroed (32 arrivals)
  griddep_launch_dependents();  // KF may start its prologue (it waits for our completion)
  const uint32_t m = bp.m, mS = SMALLM ? 2u : m;
  const uint32_t MS = meta_stride(mS, W);
  uint32_t *cnt = km_smem + KS * T;
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (blockIdx.x == 0 && tid == 0) hdr[0] = 0u;  // key-domain flag of this call (KF sets it)
  for (uint32_t i = tid; i < 2 * W * mS; i += blockDim.x) cnt[i] = 0u;
  const uint32_t t0 = blockIdx.x * tiles_per_cta;
  const uint32_t t1 = min(num_tiles, t0 + tiles_per_cta);
  const bool aligned = ((reinterpret_cast<uintptr_t>(keys) & 15u) == 0);
  auto via_tma = [&](uint32_t t) { return aligned && (uint64_t)(t + 1) * T <= n; };
  if (tid == 0) {
    for (uint32_t i = 0; i < KS; ++i) mbar_init(&full[i], 1);
    for (uint32_t i = 0; i < 2; ++i) {
      mbar_init(&cfull[i], kThreads);
      mbar_init(&cempty[i], 32);
    }
  }
  __syncthreads();

  if (warp == W) {
    // ============================ scan warp ===================================
    auto issue = [&](uint32_t t, uint32_t st) {
      if (lane == 0 && t < t1 && via_tma(t)) {
        mbar_arrive_expect_tx(&full[st], T * 4u);
        tma_load_1d(km_smem + st * T, keys + (size_t)t * T, T * 4u, &full[st], policy_evict_first());
      }
    };
    for (uint32_t i = 0; i < KS; ++i) issue(t0 + i, i);
    uint32_t running = 0;  // range count of bucket lane
    uint32_t k = 0;
    for (uint32_t t = t0; t < t1; ++t, ++k) {
      const uint32_t p = k & 1u;
      mbar_wait(&cfull[p], (k >> 1) & 1u);
      // every counting warp has read its slice of stage k % KS: refill it
      if (lane == 0) fence_proxy_async_smem();
      issue(t + KS, k % KS);
      // column of bucket lane: exclusive prefix over the warps, tile count h
      uint32_t *c = cnt + p * W * mS;
      uint32_t col[W];
      uint32_t h = 0;
#pragma unroll
      for (uint32_t w = 0; w < W; ++w) {
        const uint32_t x = lane < mS ? c[w * mS + lane] : 0u;
        col[w] = h;
        h += x;
      }
#pragma unroll
      for (uint32_t w = 0; w < W; ++w)
        if (lane < mS) c[w * mS + lane] = 0u;
      uint32_t incl = h;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= (uint32_t)o) incl += y;
      }
      const uint32_t tb = incl - h;  // tile base of bucket lane
      if (lane < mS) {
        uint32_t *rec = meta + (size_t)t * MS;
#pragma unroll
        for (uint32_t w = 0; w < W; ++w) rec[w * mS + lane] = tb + col[w];
      }
      running += h;
      __syncwarp();
      mbar_arrive(&cempty[p]);
    }
    if (lane < m) R[(size_t)blockIdx.x * m + lane] = running;
    return;
  }

  // ============================ counting warps ================================
  uint32_t k = 0;
  for (uint32_t t = t0; t < t1; ++t, ++k) {
    const uint32_t p = k & 1u, st = k % KS;
    if (k >= 2) mbar_wait(&cempty[p], ((k - 2) >> 1) & 1u);  // count buffer p is free again
    uint32_t ones = 0, nvalid = SL;
    uint32_t *row = cnt + (p * W + warp) * mS;
    if (via_tma(t)) {
      mbar_wait(&full[st], (k / KS) & 1u);
      const uint4 *v = reinterpret_cast<const uint4 *>(km_smem + st * T + warp * SL);
      uint4 q[NV];
#pragma unroll
      for (int u = 0; u < NV; ++u) q[u] = v[lane + 32u * (uint32_t)u];
      // every bucket id first, then the increments: the compiler cannot move a
      // shared-memory load (the splitter search) above an atomic on the
      // counters, so interleaving them serialized the searches
      uint32_t bk[4 * NV];
#pragma unroll
      for (int u = 0; u < NV; ++u) {
        bk[4 * u] = bucket_of<KIND>(q[u].x, bp);
        bk[4 * u + 1] = bucket_of<KIND>(q[u].y, bp);
        bk[4 * u + 2] = bucket_of<KIND>(q[u].z, bp);
        bk[4 * u + 3] = bucket_of<KIND>(q[u].w, bp);
      }
#pragma unroll
      for (int e = 0; e < 4 * NV; ++e) {
        if constexpr (SMALLM) ones += bk[e]; else atomicAdd(row + bk[e], 1u);
      }
    } else {  // ragged last tile / unaligned input
      const uint64_t lo = (uint64_t)t * T + warp * SL;
      const uint32_t hi = (uint32_t)min((uint64_t)n, lo + SL);
      nvalid = hi > lo ? hi - (uint32_t)lo : 0u;
      for (uint32_t i = (uint32_t)lo + lane; i < hi; i += 32u) {
        const uint32_t b = bucket_of<KIND>(__ldg(keys + i), bp);
        if constexpr (SMALLM) ones += b; else atomicAdd(row + b, 1u);
      }
    }
    if constexpr (SMALLM) {
      ones = __reduce_add_sync(0xFFFFFFFFu, ones);
      if (lane == 0) {
        row[0] = nvalid - ones;
        row[1] = ones;
      }
    }
    mbar_arrive(&cfull[p]);
  }
}

// ============================================================================
// Probe of reading R23: the old values that one warp-wide
// shared-memory atomicAdd(p, 1) returns to the lanes sharing an address are
// consecutive in lane order, and consecutive such instructions of a warp are
// applied in program order.  Run in the postscan's own launch shape (512
// threads, two CTAs per SM over the whole grid, every warp hammering its own
// row of up to 256 counters with runs, random and skewed bucket patterns, 16
// instructions back to back as in the rank loop; plain and packed 16-bit
// counters as in ms_wide.cuh); lane 0 of each warp replays
// the same increments sequentially with plain loads and stores, and every
// returned value must equal the replay.  *flag is cleared if any differs.
// ============================================================================
constexpr uint32_t kProbeWords = 1024u;  // per warp: row[256] | shadow[256] | bucket/expect[512]
static __global__ void __launch_bounds__(kThreads, 2)
    k_probe_lane_ordered_inc(uint32_t *flag, uint32_t patterns) {
  extern __shared__ uint32_t pr_smem[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  uint32_t *row = pr_smem + warp * kProbeWords, *shadow = row + 256, *ex = row + 512;
  bool ok = true;
  for (uint32_t pat = 0; pat < patterns; ++pat) {
    const uint32_t salt = (blockIdx.x * 131u + warp) * 0x9E3779B9u + pat * 0x85EBCA6Bu;
    const uint32_t mb = 1u + ((salt >> 7) & 255u);  // buckets in play: 1 .. 256
    const uint32_t kind = pat & 3u;                  // random / runs / 90 % hot / two values
    const bool packed = (pat & 4u) != 0u;            // two 16-bit counters per word (ms_wide.cuh)
    for (uint32_t j = lane; j < 256u; j += 32u) row[j] = shadow[j] = (salt ^ j) & 0x7FFF7FFFu;
    uint32_t b[16], got[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      uint32_t h = salt ^ (lane * 0x2C1B3C6Du) ^ ((uint32_t)i * 0x297A2D39u);
      h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12; h *= 0x297A2D39u; h ^= h >> 15;
      uint32_t v = h % mb;
      if (kind == 1u) v = ((lane + 32u * (uint32_t)i) * mb) >> 9;      // sorted runs
      if (kind == 2u && (h >> 24) < 230u) v = salt % mb;               // 90 % one bucket
      if (kind == 3u) v = (h >> 31) ? 0u : mb - 1u;                     // two buckets
      b[i] = v;
      ex[i * 32 + lane] = v;
    }
    __syncwarp();
    if (packed) {
#pragma unroll
      for (int i = 0; i < 16; ++i) got[i] = atomicAdd(row + (b[i] >> 1), 1u << ((b[i] & 1u) << 4));
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) got[i] = atomicAdd(row + b[i], 1u);
    }
    __syncwarp();
    if (lane == 0) {  // sequential replay in (instruction, lane) order
      for (uint32_t e = 0; e < 512u; ++e) {
        const uint32_t v = ex[e];
        const uint32_t w = packed ? v >> 1 : v;
        const uint32_t old = shadow[w];
        shadow[w] = old + (packed ? 1u << ((v & 1u) << 4) : 1u);
        ex[e] = old;
      }
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 16; ++i) ok &= got[i] == ex[i * 32 + lane];
    __syncwarp();
  }
  if (!__all_sync(0xFFFFFFFFu, ok) && lane == 0) atomicAnd(flag, 0u);
}

// Shared memory of kf_meta: 3 stages of [keys OS | values OS | meta MS] words,
// rank rows [3][W][32], run tables [3][3][32] (or deltas [3][32]).
__host__ __device__ inline size_t kfm_smem_bytes(uint32_t m, bool pairs) {
  const uint32_t T = kThreads * (pairs ? 8u : 16u);
  const size_t SW = (size_t)kf_out_slots(T, m) * (pairs ? 2u : 1u) + meta_stride(meta_ms(m), kWarps);
  return (3 * SW + 3 * kWarps * 32 + 3 * 3 * 32) * 4;
}

// Rank modes of kf_meta (m > 2; m <= 2 always ranks with one ballot per window):
//   kRankInc   Eq.4 term 1 as the value a lane-ordered shared-memory increment
//              of the warp's running slot returns (reading R23; used only on a
//              device where the full-occupancy probe above passed);
//   kRankMasks deterministic: peer masks by a shared-memory OR of the lane bit,
//              taken and cleared by one atomic exchange per bucket lane, two
//              windows in flight (Alg.3's peer masks).
//   kRankVote2 deterministic, for 2 < m <= 4: Alg.3's ballots
//              (P:909-930), one __ballot_sync per bit of the bucket id; the
//              peer mask of a key is the AND of the (possibly inverted)
//              ballots, and lane j forms bucket j's mask the same way to
//              advance the warp's running slot.  No shared-memory atomics: at
//              m = 4 eight lanes share each counter and the increments
//              serialize in the atomic unit (profiles/r02; measured 337 -> 396
//              Gkeys/s at m = 4; three ballots at m = 8 were slower than
//              increments, 335 vs 371).
enum : int { kRankBallot = 0, kRankVote2 = 2, kRankMasks = 7, kRankInc = 8 };

// ============================================================================
// KF (meta mode): persistent CTA per level-0 range, tiles in order; 16
// consumer warps rank and place, and (PROD) one producer warp does all TMA.
//   consumer iteration k (tile t): per-warp setup from the tile meta; rank and
//   place the keys held in registers into the stage, in place; load tile t+1's
//   keys into registers; ONE barrier among the consumers.  All consumer warps
//   load tile t+1's keys before that barrier, so the in-place placement of
//   tile t+1 never overwrites a key that is still unread.
//   PROD (whole-run TMA bulk stores): the consumers arrive on placed[k % 3];
//   the producer warp waits for it, issues tile t's run stores, and refills
//   the stage of tile t-1 (read by now) with tile t+2 -- the consumers never
//   wait for a store or issue one.  A tile that is not TMA-loaded (ragged last
//   tile, unaligned input) is placed only after the producer has signalled
//   empty[stage]: the bulk stores of the stage's previous tile have read it.
//   !PROD: after the barrier the last warp issues tile t's run stores (TMA
//   bulk) and every thread stores run heads / tails, or (no run stores) every
//   thread scatters its slots; then the stage of tile t-1 gets tile t+2.
// Meta records of tiles that are not TMA-loaded are read from global memory.
// ============================================================================
template <int KIND, bool PAIRS, bool SMALLM, int ITEMS, int RANK, bool PROD>
__global__ void __launch_bounds__(PROD ? kThreads + 32 : kThreads, 2) kf_meta(KfArgs a, BucketParams bp) {
  MS_STAGE_SPLITTERS(bp, 32);
  constexpr uint32_t W = kWarps, NT = kThreads;  // consumer warps / threads
  constexpr uint32_t T = NT * ITEMS;
  constexpr uint32_t kStages = 3;
  constexpr uint32_t kPrefetch = 2;  // L2 prefetch distance beyond the ring (measured, profiles/r01)
  extern __shared__ __align__(128) uint8_t kf_smem[];
  __shared__ __align__(8) uint64_t bar[kStages];
  __shared__ __align__(8) uint64_t placed[kStages];  // PROD: tile placed, 512 arrivals
  __shared__ __align__(8) uint64_t empty[kStages];   // PROD: stage free for a non-TMA tile
  __shared__ uint32_t s_ps[kMaxPeers + 1];           // sharded: output shard starts
  const uint32_t m = bp.m, mS = SMALLM ? 2u : m;
  const uint32_t OS = kf_out_slots(T, m);
  const uint32_t MS = meta_stride(mS, W);
  const uint32_t MO = OS * (PAIRS ? 2u : 1u);  // meta offset inside a stage
  const uint32_t SW = MO + MS;                 // words per stage
  uint32_t *stage0 = reinterpret_cast<uint32_t *>(kf_smem);
  uint32_t *s_mask = stage0 + kStages * SW;  // [3][W][32]
  uint32_t *s_tab = s_mask + 3 * W * 32;     // [3][3][32] run tables / deltas per stage
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t lt = lanemask_lt(), lanebit = 1u << lane;
  // the thread that issues the TMA loads: lane 0 of the producer warp (PROD) or
  // of the last consumer warp
  constexpr uint32_t kProducer = PROD ? NT : NT - 32;

  const uint32_t t0 = blockIdx.x * a.tiles_per_cta;
  const uint32_t t1 = min(a.num_tiles, t0 + a.tiles_per_cta);
  if (t0 >= t1) return;
  const uint32_t nt = t1 - t0;
  auto tile = [&](uint32_t k) { return k >= nt ? t1 : t0 + k; };
  auto tile_n = [&](uint32_t t) { return min(T, a.n - t * T); };
  auto via_tma = [&](uint32_t t) { return a.use_tma && tile_n(t) == T; };
  // one elected thread starts the TMA bulk copies of a tile: the input data
  // (may run before griddep_wait: the inputs predate KM) and the meta record
  // (written by KM: only after griddep_wait); one mbarrier transaction count
  auto issue_data = [&](uint32_t t, uint32_t st) {
    if (tid == kProducer && t < t1 && via_tma(t)) {
      uint32_t *dst = stage0 + st * SW;
      const uint64_t pol = policy_evict_first();
      mbar_arrive_expect_tx(&bar[st], T * 4u * (PAIRS ? 2u : 1u) + MS * 4u);
      tma_load_1d(dst, a.keys_in + (size_t)t * T, T * 4u, &bar[st], pol);
      if constexpr (PAIRS) tma_load_1d(dst + OS, a.vals_in + (size_t)t * T, T * 4u, &bar[st], pol);
    }
  };
  auto issue_meta = [&](uint32_t t, uint32_t st) {
    if (tid == kProducer && t < t1 && via_tma(t))
      tma_load_1d(stage0 + st * SW + MO, a.meta + (size_t)t * MS, MS * 4u, &bar[st],
                  policy_evict_first());
  };
  // the TMA ring holds only three tiles; tiles further ahead are prefetched
  // into L2 (evict_last, so that the streaming output does not evict them
  // before their TMA load: measured +1-3.5 %)
  auto prefetch = [&](uint32_t t) {
    if (tid == kProducer && t < t1 && via_tma(t)) {
      const uint64_t pol = policy_evict_last();
      prefetch_l2_bulk_hint(a.keys_in + (size_t)t * T, T * 4u, pol);
      if constexpr (PAIRS) prefetch_l2_bulk_hint(a.vals_in + (size_t)t * T, T * 4u, pol);
      prefetch_l2_bulk_hint(a.meta + (size_t)t * MS, MS * 4u, pol);
    }
  };
  auto issue = [&](uint32_t k, uint32_t st) {
    issue_data(tile(k), st);
    issue_meta(tile(k), st);
    prefetch(tile(k + kPrefetch));
  };
  if (tid == 0) {
    for (uint32_t i = 0; i < kStages; ++i) mbar_init(&bar[i], 1);
    if constexpr (PROD)
      for (uint32_t i = 0; i < kStages; ++i) {
        mbar_init(&placed[i], NT);
        mbar_init(&empty[i], 1);
      }
  }
  __syncthreads();
  issue_data(tile(0), 0);
  issue_data(tile(1), 1);
  if constexpr (PROD) {
    if (warp == W) {
      // ======================= producer warp =================================
      griddep_wait();  // meta records are complete
      issue_meta(tile(0), 0);
      issue_meta(tile(1), 1);
      for (uint32_t j = 2; j < 2 + kPrefetch; ++j) prefetch(tile(j));
      for (uint32_t k = 0; k < nt; ++k) {
        const uint32_t st = k % kStages;
        uint32_t *s_stage = stage0 + st * SW;
        const uint32_t *tab = s_tab + st * 96u;
        // refill the stage of tile t-1 with tile t+2 as soon as tile t-1's bulk
        // stores have read it, before tile t's stores are queued behind it; a
        // tile that is not TMA-loaded gets the stage through empty[]
        bulk_wait_read();
        __syncwarp();
        if (lane == 0) fence_proxy_async_smem();
        issue(k + 2, (k + 2) % kStages);
        if (lane == 0 && k + 2 < nt && !via_tma(tile(k + 2))) mbar_arrive(&empty[(k + 2) % kStages]);
        mbar_wait(&placed[st], (k / kStages) & 1u);
        // one TMA bulk store per bucket run body (16-byte aligned), then the
        // <= 3 leading / trailing elements of every run with plain stores
        if (lane < m) {
          const uint32_t len = tab[64 + lane], gs = tab[32 + lane], st0 = tab[lane];
          const uint32_t head = min(len, (4u - (gs & 3u)) & 3u);
          const uint32_t body = (len - head) & ~3u;
          if (body) {
            fence_proxy_async_smem();
            tma_store_1d(a.keys_out + gs + head, s_stage + st0 + head, body * 4u);
            if constexpr (PAIRS) tma_store_1d(a.vals_out + gs + head, s_stage + OS + st0 + head, body * 4u);
          }
        }
        bulk_commit();
        for (uint32_t x = lane; x < 8u * m; x += 32u) {
          const uint32_t b = x >> 3, j = x & 7u;
          const uint32_t len = tab[64 + b], gs = tab[32 + b];
          const uint32_t head = min(len, (4u - (gs & 3u)) & 3u);
          const uint32_t tail = (len - head) & 3u;
          uint32_t e = 0xFFFFFFFFu;
          if (j < 4u) {
            if (j < head) e = j;
          } else if (j - 4u < tail) {
            e = len - tail + (j - 4u);
          }
          if (e != 0xFFFFFFFFu) {
            const uint32_t sidx = tab[b] + e;
            a.keys_out[gs + e] = s_stage[sidx];
            if constexpr (PAIRS) a.vals_out[gs + e] = s_stage[OS + sidx];
          }
        }
      }
      bulk_wait_all();  // run stores complete before smem is released
      return;
    }
  }

  // keys (values) of one tile -> registers: lane l of warp w holds element
  // w*32*ITEMS + 32 i + l.  TMA tiles come from the stage, others from global.
  uint32_t key[ITEMS];
  uint32_t val[PAIRS ? ITEMS : 1];
  const uint32_t wbase = warp * (ITEMS * 32);
  auto load_tile = [&](uint32_t t, uint32_t k) {
    const uint32_t st = k % kStages;
    uint32_t *s = stage0 + st * SW;
    const uint32_t tn = tile_n(t);
    if (via_tma(t)) {
      mbar_wait(&bar[st], (k / kStages) & 1u);
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) key[i] = s[wbase + 32 * i + lane];
      if constexpr (PAIRS) {
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) val[i] = s[OS + wbase + 32 * i + lane];
      }
    } else {
      const size_t g = (size_t)t * T;
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const uint32_t e = wbase + 32 * i + lane;
        key[i] = e < tn ? __ldg(a.keys_in + g + e) : 0u;
        if constexpr (PAIRS) val[i] = e < tn ? __ldg(a.vals_in + g + e) : 0u;
      }
    }
  };

  // ---- level-0 offsets (Eq.3 terms 1-2 with L_0 = G), no separate scan
  // kernel: the CTA reduces the G x m range histograms R (written by KM) to
  // its prefix P[c][b] = sum_{c'<c} R[c'][b] and the totals Tot[b]; every warp
  // then forms base[b] + P[c][b] for its bucket lanes.  R is G m words, read
  // from L2 (11 MB in all at m = 32, G = 296).
  griddep_wait();  // KM complete: meta records and range histograms
  if (a.npeers && tid <= a.npeers) s_ps[tid] = __ldcg(a.peer_start + tid);
  issue_meta(tile(0), 0);
  issue_meta(tile(1), 1);
  for (uint32_t j = 2; j < 2 + kPrefetch; ++j) prefetch(tile(j));
  uint32_t gbase = 0, grun = 0;
  {
    uint32_t *red = s_mask;  // [2][16][32] scratch (the mask rows are zeroed per tile)
    const uint32_t G = a.num_ranges, c = blockIdx.x;
    uint32_t pre = 0, tot = 0;
    if (lane < m) {
      // batches of 20 independent loads (rows warp, warp + W, ...): one batch
      // covers G <= 320 ranges (2 CTAs on 148 SMs: G = 296)
      for (uint32_t r0 = warp; r0 < G; r0 += 20 * W) {
        uint32_t v[20];
#pragma unroll
        for (int j = 0; j < 20; ++j) {
          const uint32_t r = r0 + j * W;
          v[j] = r < G ? __ldcg(a.R + (size_t)r * m + lane) : 0u;
        }
#pragma unroll
        for (int j = 0; j < 20; ++j) {
          tot += v[j];
          pre += r0 + j * W < c ? v[j] : 0u;
        }
      }
    }
    red[warp * 32 + lane] = pre;
    red[(W + warp) * 32 + lane] = tot;
    named_barrier_sync(1, NT);
    pre = 0;
    tot = 0;
#pragma unroll
    for (uint32_t g = 0; g < W; ++g) {
      pre += red[g * 32 + lane];
      tot += red[(W + g) * 32 + lane];
    }
    uint32_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= (uint32_t)o) incl += y;
    }
    if (lane < m) {
      gbase = (a.gbase_ovr ? __ldcg(a.gbase_ovr + lane) : incl - tot) + pre;
      if (c == 0 && warp == 0 && a.bucket_offsets) {
        a.bucket_offsets[lane] = incl - tot;
        if (lane == m - 1) a.bucket_offsets[m] = incl;
      }
    }
  }
  load_tile(tile(0), 0);
  named_barrier_sync(1, NT);

  uint32_t *mrow0 = s_mask + warp * 32, *mrow1 = s_mask + (W + warp) * 32;
  for (uint32_t k = 0; k < nt; ++k) {
    const uint32_t t = tile(k);
    const uint32_t st = k % kStages;
    uint32_t *s_stage = stage0 + st * SW;
    const bool tma_tile = via_tma(t);
    const uint32_t *rec = tma_tile ? s_stage + MO : a.meta + (size_t)t * MS;
    const uint32_t tn = tile_n(t);
    const bool full = tn == T;
    uint32_t *tab = s_tab + st * 96u;
    if constexpr (PROD) {
      // a tile that is not TMA-loaded: the producer has finished the previous
      // tile of this stage (its run table and its bulk stores' reads of the
      // stage) before this tile's run table and placement overwrite them
      if (!tma_tile && k >= 2) mbar_wait(&empty[st], a.use_tma ? 0u : ((k - 2) / kStages) & 1u);
    }

    // ---- per-warp setup from the meta record (lane b = bucket b) -------------
    // slot of this warp's first bucket-b key = S[b][warp] (+ run padding adj[b]
    // so that the run starts congruent mod 4 with its global destination)
    uint32_t wrun = 0;
    if (lane < m) {
      // records of tiles that are not TMA-loaded come from global memory,
      // written by KM: read through L2 (a programmatic dependent launch may
      // start before KM completes, and its L1 can hold lines of an earlier
      // use of the workspace -- measured: stale reads without .cg)
      auto rd = [&](uint32_t i) { return tma_tile ? rec[i] : __ldcg(rec + i); };
      const uint32_t sbw = rd(warp * mS + lane);
      const uint32_t tb = rd(lane);
      const uint32_t te = lane + 1 < m ? rd(lane + 1) : tn;
      const uint32_t gs = gbase + grun;  // + Eq.3 term 3: the range's tiles before this one
      grun += te - tb;
      const uint32_t adj = a.store_runs ? 4u * lane + ((gs - tb) & 3u) : 0u;
      wrun = sbw + adj;
      if (warp == W - 1) {
        if (a.store_runs) {
          tab[lane] = tb + adj;
          tab[32 + lane] = gs;
          tab[64 + lane] = te - tb;
        } else {
          tab[lane] = gs - tb;
        }
      }
    }
    if constexpr (!SMALLM && RANK == kRankMasks) {
      mrow0[lane] = 0u;
      mrow1[lane] = 0u;
    }
    __syncwarp();

    // ---- rank and place (Eq.4 term 1 + this warp's running slot) -------------
    bool derr = false;
    auto place = [&](auto full_c) {
      constexpr bool FULL = decltype(full_c)::value;
      if constexpr (RANK == kRankInc && !SMALLM) {
        // rank by the shared-memory atomic increment of this warp's running
        // slot of the bucket (reading R23)
        uint32_t *brow = mrow0;
        if (lane < m) brow[lane] = wrun;
        __syncwarp();
        // (one increment, then its placement: issuing all increments first was
        // measured slower at m = 8 / 16, where more lanes share a counter)
        uint32_t bk[ITEMS];  // bucket ids first (see KM): the searches interleave
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) bk[i] = bucket_of<KIND>(key[i], bp);
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          const bool valid = FULL || wbase + (uint32_t)i * 32u + lane < tn;
          if (!FULL && wbase + (uint32_t)i * 32u >= tn) continue;
          const uint32_t b = bk[i];
          if constexpr (KIND == kIdentity) derr |= valid && key_domain_error<KIND>(key[i], bp);
          if (valid) {
            const uint32_t slot = atomicAdd(brow + b, 1u);
            s_stage[slot] = key[i];
            if constexpr (PAIRS) s_stage[OS + slot] = val[i];
          }
        }
        return;
      }
      if constexpr (RANK == kRankMasks && FULL && !SMALLM && (ITEMS % 2 == 0)) {
        // two windows at a time: both windows' shared-memory round trips
        // (OR of the lane bit, exchange of the bucket lane's mask) are in
        // flight together; only the cheap running-slot update is serial
#pragma unroll
        for (int i = 0; i < ITEMS; i += 2) {
          const uint32_t b0 = bucket_of<KIND>(key[i], bp), b1 = bucket_of<KIND>(key[i + 1], bp);
          if constexpr (KIND == kIdentity)
            derr |= key_domain_error<KIND>(key[i], bp) || key_domain_error<KIND>(key[i + 1], bp);
          atomicOr(mrow0 + b0, lanebit);
          atomicOr(mrow1 + b1, lanebit);
          __syncwarp();
          const uint32_t mine0 = atomicExch(mrow0 + lane, 0u);
          const uint32_t mine1 = atomicExch(mrow1 + lane, 0u);
          const uint32_t peers0 = __shfl_sync(0xFFFFFFFFu, mine0, b0);
          const uint32_t peers1 = __shfl_sync(0xFFFFFFFFu, mine1, b1);
          const uint32_t w1 = wrun + __popc(mine0);
          const uint32_t slot0 = __shfl_sync(0xFFFFFFFFu, wrun, b0) + __popc(peers0 & lt);
          const uint32_t slot1 = __shfl_sync(0xFFFFFFFFu, w1, b1) + __popc(peers1 & lt);
          wrun = w1 + __popc(mine1);
          __syncwarp();  // both rows are clear before the next pair's ORs
          s_stage[slot0] = key[i];
          s_stage[slot1] = key[i + 1];
          if constexpr (PAIRS) {
            s_stage[OS + slot0] = val[i];
            s_stage[OS + slot1] = val[i + 1];
          }
        }
        return;
      }
      if constexpr (RANK == kRankVote2) {
        constexpr int LOGM = 2;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
          const bool valid = FULL || wbase + (uint32_t)i * 32u + lane < tn;
          if (!FULL && wbase + (uint32_t)i * 32u >= tn) continue;  // warp-uniform
          const uint32_t b = bucket_of<KIND>(key[i], bp);
          if constexpr (KIND == kIdentity) derr |= valid && key_domain_error<KIND>(key[i], bp);
          const uint32_t vm = FULL ? 0xFFFFFFFFu : __ballot_sync(0xFFFFFFFFu, valid);
          uint32_t peers = vm, mine = vm;
#pragma unroll
          for (int q = 0; q < LOGM; ++q) {
            const uint32_t bq = __ballot_sync(0xFFFFFFFFu, valid && ((b >> q) & 1u));
            peers &= ((b >> q) & 1u) ? bq : ~bq;
            mine &= ((lane >> q) & 1u) ? bq : ~bq;
          }
          const uint32_t slot = __shfl_sync(0xFFFFFFFFu, wrun, b) + __popc(peers & lt);
          wrun += __popc(mine);  // lanes >= m: buckets that never occur
          if (valid) {
            s_stage[slot] = key[i];
            if constexpr (PAIRS) s_stage[OS + slot] = val[i];
          }
        }
        return;
      }
      uint32_t base0 = 0, base1 = 0, c0 = 0, c1 = 0;
      if constexpr (SMALLM) {
        base0 = __shfl_sync(0xFFFFFFFFu, wrun, 0);
        base1 = __shfl_sync(0xFFFFFFFFu, wrun, 1);
      }
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const bool valid = FULL || wbase + (uint32_t)i * 32u + lane < tn;
        if (!FULL && wbase + (uint32_t)i * 32u >= tn) continue;  // warp-uniform: past the tail
        const uint32_t b = bucket_of<KIND>(key[i], bp);
        if constexpr (KIND == kIdentity) derr |= valid && key_domain_error<KIND>(key[i], bp);
        uint32_t slot;
        if constexpr (SMALLM) {
          // m <= 2: one ballot gives every peer mask (Alg.2/3 with log2 m = 1)
          const uint32_t ones = __ballot_sync(0xFFFFFFFFu, valid && b != 0u);
          const uint32_t ones_below = __popc(ones & lt);
          const uint32_t nones = __popc(ones);
          if (FULL) {
            slot = b ? base1 + c1 + ones_below : base0 + c0 + lane - ones_below;
            c0 += 32u - nones;
          } else {
            const uint32_t vm = __ballot_sync(0xFFFFFFFFu, valid);
            slot = b ? base1 + c1 + ones_below : base0 + c0 + __popc(vm & ~ones & lt);
            c0 += __popc(vm) - nones;
          }
          c1 += nones;
        } else {
          // one window at a time (partial tiles of kRankMasks): peer masks by
          // one shared-memory OR of the lane bit; lane j takes bucket j's mask
          // and clears it with one atomic exchange, the key of bucket b gets
          // its peers and running slot from lane b by shuffles.  Two rows
          // alternate, one __syncwarp each.
          uint32_t *mrow = (i & 1) ? mrow1 : mrow0;
          if (valid) atomicOr(mrow + b, lanebit);
          __syncwarp();
          const uint32_t mine = atomicExch(mrow + lane, 0u);  // lanes >= m: an unused, zero word
          const uint32_t peers = __shfl_sync(0xFFFFFFFFu, mine, b);
          slot = __shfl_sync(0xFFFFFFFFu, wrun, b) + __popc(peers & lt);
          wrun += __popc(mine);
        }
        if (valid) {
          s_stage[slot] = key[i];
          if constexpr (PAIRS) s_stage[OS + slot] = val[i];
        }
      }
    };
    if (full)
      place(std::true_type{});
    else
      place(std::false_type{});
    if constexpr (KIND == kIdentity) {
      if (__any_sync(0xFFFFFFFFu, derr) && lane == 0) atomicOr(a.hdr, 1u);
    }
    if constexpr (PROD) {
      mbar_arrive(&placed[st]);  // tile t placed: the producer may store it
      if (k + 1 < nt) load_tile(tile(k + 1), k + 1);
      named_barrier_sync(1, NT);
    } else if (a.store_runs) {
      // ---- next tile's keys into registers before the barrier -----------------
      if (k + 1 < nt) load_tile(tile(k + 1), k + 1);
      named_barrier_sync(1, NT);
      // ---- refill the stage of tile t-1 with tile t+2 as soon as tile t-1's
      // bulk stores (issued a whole iteration ago) have read it, before this
      // tile's stores are queued
      if (warp == W - 1) {
        bulk_wait_read();
        __syncwarp();
        if (lane == 0) fence_proxy_async_smem();
        issue(k + 2, (k + 2) % kStages);
      }
      // ---- run stores of tile t: one TMA bulk store per run body by the last
      // warp, the <= 3 leading / trailing elements by threads 8b .. 8b+7
      if (warp == W - 1) {
        if (lane < m) {
          const uint32_t len = tab[64 + lane], gs = tab[32 + lane], st0 = tab[lane];
          const uint32_t head = min(len, (4u - (gs & 3u)) & 3u);
          const uint32_t body = (len - head) & ~3u;
          if (body) {
            fence_proxy_async_smem();
            tma_store_1d(a.keys_out + gs + head, s_stage + st0 + head, body * 4u);
            if constexpr (PAIRS) tma_store_1d(a.vals_out + gs + head, s_stage + OS + st0 + head, body * 4u);
          }
        }
        bulk_commit();
      }
      if (tid < 8u * m) {
        const uint32_t b = tid >> 3, j = tid & 7u;
        const uint32_t len = tab[64 + b], gs = tab[32 + b];
        const uint32_t head = min(len, (4u - (gs & 3u)) & 3u);
        const uint32_t tail = (len - head) & 3u;
        uint32_t e = 0xFFFFFFFFu;
        if (j < 4u) {
          if (j < head) e = j;
        } else if (j - 4u < tail) {
          e = len - tail + (j - 4u);
        }
        if (e != 0xFFFFFFFFu) {
          const uint32_t sidx = tab[b] + e;
          a.keys_out[gs + e] = s_stage[sidx];
          if constexpr (PAIRS) a.vals_out[gs + e] = s_stage[OS + sidx];
        }
      }
    } else {
      // ---- next tile's keys into registers before the barrier -----------------
      if (k + 1 < nt) load_tile(tile(k + 1), k + 1);
      named_barrier_sync(1, NT);
      // ---- refill the stage of tile t-1 with tile t+2 (every warp finished
      // tile t-1's scatter before this barrier): a whole scatter earlier
      if (tid == kProducer) {
        fence_proxy_async_smem();
        issue(k + 2, (k + 2) % kStages);
      }
      // ---- coalesced scatter of tile t: slot s of bucket b -> delta[b] + s ----
      const uint32_t s0 = wbase + lane;
      uint32_t kk[ITEMS], pos[ITEMS];
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) kk[i] = s_stage[s0 + 32 * i];
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) pos[i] = tab[bucket_of<KIND>(kk[i], bp)] + s0 + 32 * i;
      if (a.npeers) {  // sharded: into the owning rank's window (KP)
#pragma unroll
        for (int i = 0; i < ITEMS; ++i)
          if (full || s0 + 32 * i < tn)
            kp_store<PAIRS>(a, s_ps, pos[i], kk[i], PAIRS ? s_stage[OS + s0 + 32 * i] : 0u);
      } else {
#pragma unroll
      for (int i = 0; i < ITEMS; ++i)
        if (full || s0 + 32 * i < tn) a.keys_out[pos[i]] = kk[i];
      if constexpr (PAIRS) {
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) kk[i] = s_stage[OS + s0 + 32 * i];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i)
          if (full || s0 + 32 * i < tn) a.vals_out[pos[i]] = kk[i];
      }
      }
    }
  }
  if constexpr (!PROD) {
    if (a.store_runs) bulk_wait_all();  // run stores complete before smem is released
  }
}

}  // namespace ms
