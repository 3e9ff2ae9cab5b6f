// ms_kernels.cuh -- the multisplit on sm_100a as the paper's lambda-level
// localization (Sec.4.4, Eq.3) mapped onto B200:
//
//   level 0: G CTA ranges of K consecutive tiles      -> H = [h_{j,l0}] is m x G
//   level 1: tiles of T elements inside a range        -> running per-bucket offsets
//   level 2: warps inside a tile, level 3: 32-wide windows inside a warp (Eq.4)
//
//   KU  prescan:   range histogram R[c][j] = h_{j,c} (level-0 column of H)
//   KF  scan + postscan: each CTA scans the small m x G matrix R
//       (Eq.3 terms 1-2), then for every tile of its range, in order: stable
//       tile-local rank (Eq.4), tile-local reorder in shared memory
//       (Sec.5.6.2), coalesced scatter of each bucket run.
//
// Also here: KH, the tile-granular prescan H[l][j] of Eq.(2) used by the
// stage API and by the paper-faithful three-launch mode (KH -> KG -> KF).
//
// Citations "P:nnn" are lines of the paper's LaTeX source.
#pragma once
#include "ms_device.cuh"

namespace ms {

// ============================================================================
// Shared histogram helpers.  m <= 2 counts ones in registers; otherwise each
// warp owns a private row of m counters in shared memory (warp-level
// privatization) updated with shared-memory atomics (measured
// cheapest on B200, profiles/r01/v0_summary.md).
// ============================================================================
template <int KIND, bool SMALLM>
__device__ __forceinline__ void hist_add(uint32_t key, const BucketParams &bp, uint32_t *row,
                                         uint32_t &ones) {
  const uint32_t b = bucket_of<KIND>(key, bp);
  if constexpr (SMALLM) {
    ones += b;
  } else {
    atomicAdd(row + b, 1u);
  }
}

// Count keys[lo, hi) into the CTA's counters (vector loads when aligned).
template <int KIND, bool SMALLM>
__device__ __forceinline__ void hist_range(const uint32_t *__restrict__ keys, uint32_t lo,
                                           uint32_t hi, const BucketParams &bp, uint32_t *row,
                                           uint32_t &ones) {
  const uint32_t tid = threadIdx.x;
  const bool aligned = ((reinterpret_cast<uintptr_t>(keys + lo) & 15u) == 0);
  uint32_t i = lo;
  if (aligned) {
    const uint4 *v = reinterpret_cast<const uint4 *>(keys + lo);
    const uint32_t nv = (hi - lo) >> 2;
    uint32_t j = tid;
    for (; j + 7u * kThreads < nv; j += 8u * kThreads) {  // 8 x 16 B in flight per thread
      uint4 q[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) q[u] = ldg_stream_v4(v + j + (uint32_t)u * kThreads);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        hist_add<KIND, SMALLM>(q[u].x, bp, row, ones);
        hist_add<KIND, SMALLM>(q[u].y, bp, row, ones);
        hist_add<KIND, SMALLM>(q[u].z, bp, row, ones);
        hist_add<KIND, SMALLM>(q[u].w, bp, row, ones);
      }
    }
    for (; j < nv; j += kThreads) {
      const uint4 q = ldg_stream_v4(v + j);
      hist_add<KIND, SMALLM>(q.x, bp, row, ones);
      hist_add<KIND, SMALLM>(q.y, bp, row, ones);
      hist_add<KIND, SMALLM>(q.z, bp, row, ones);
      hist_add<KIND, SMALLM>(q.w, bp, row, ones);
    }
    i = lo + (nv << 2);
  }
  for (i += tid; i < hi; i += kThreads) hist_add<KIND, SMALLM>(__ldg(keys + i), bp, row, ones);
}

// Sum the CTA's counters and write m words to out[0..m).  `total` = elements counted.
template <bool SMALLM>
__device__ __forceinline__ void hist_flush(uint32_t *cnt, uint32_t m, uint32_t ones,
                                           uint32_t total, uint32_t *__restrict__ out,
                                           uint32_t *s_red) {
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if constexpr (SMALLM) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ones += __shfl_xor_sync(0xFFFFFFFFu, ones, o);
    if (lane == 0) s_red[warp] = ones;
    __syncthreads();
    if (tid == 0) {
      uint32_t o = 0;
      for (int w = 0; w < kWarps; ++w) o += s_red[w];
      if (m == 1) {
        out[0] = total;
      } else {
        out[0] = total - o;
        out[1] = o;
      }
    }
  } else {
    __syncthreads();
    for (uint32_t j = tid; j < m; j += kThreads) {
      uint32_t s = 0;
#pragma unroll 4
      for (int w = 0; w < kWarps; ++w) s += cnt[w * m + j];
      out[j] = s;
    }
  }
}

// ============================================================================
// Level-0 column scan (Eq.3 terms 1-2 with L_0 = G) of the G x m matrix R of
// range histograms: P[c][b] = sum_{c'<c} R[c'][b] and Tot[b] = sum_c R[c][b].
// CTA j owns buckets [32j, 32j + 32); thread (b, p) sums a block of rows of
// column b (P_ row blocks), the blocks are scanned in shared memory, then each
// thread writes its rows' prefixes.  The bucket bases (exclusive scan of Tot)
// are formed by every KF CTA from the m totals.
// ============================================================================
static __global__ void __launch_bounds__(kThreads)
    kr_level0_scan(const uint32_t *__restrict__ R, uint32_t *__restrict__ P, uint32_t *__restrict__ Tot,
                   uint32_t G, uint32_t m) {
  __shared__ uint32_t s_part[kThreads];
  griddep_launch_dependents();  // KF may start its prologue (TMA of its first tiles)
  griddep_wait();               // KU's range histograms are complete
  const uint32_t tid = threadIdx.x;
  const uint32_t wb = min(32u, m - blockIdx.x * 32u);  // buckets of this CTA
  const uint32_t NP = kThreads / wb;                   // row blocks
  const uint32_t bl = tid % wb, p = tid / wb, b = blockIdx.x * 32u + bl;
  const uint32_t S = (G + NP - 1) / NP;
  const uint32_t r0 = min(G, p * S), r1 = min(G, r0 + S);
  constexpr uint32_t kMaxS = 32;  // rows held in registers (one batch of loads in flight)
  uint32_t v[kMaxS];
  uint32_t sum = 0;
  if (p < NP) {
    if (S <= kMaxS) {
#pragma unroll
      for (uint32_t i = 0; i < kMaxS; ++i) v[i] = r0 + i < r1 ? __ldcg(R + (size_t)(r0 + i) * m + b) : 0u;
#pragma unroll
      for (uint32_t i = 0; i < kMaxS; ++i) sum += v[i];
    } else {
#pragma unroll 8
      for (uint32_t r = r0; r < r1; ++r) sum += __ldcg(R + (size_t)r * m + b);
    }
    s_part[p * wb + bl] = sum;
  }
  __syncthreads();
  if (p < NP) {
    uint32_t pre = 0, tot = 0;
    for (uint32_t q = 0; q < NP; ++q) {
      const uint32_t x = s_part[q * wb + bl];
      pre += q < p ? x : 0u;
      tot += x;
    }
    if (p == 0) Tot[b] = tot;
    uint32_t run = pre;
    if (S <= kMaxS) {
#pragma unroll
      for (uint32_t i = 0; i < kMaxS; ++i) {
        if (r0 + i < r1) P[(size_t)(r0 + i) * m + b] = run;
        run += v[i];
      }
    } else {
#pragma unroll 8
      for (uint32_t r = r0; r < r1; ++r) {
        const uint32_t x = __ldcg(R + (size_t)r * m + b);
        P[(size_t)r * m + b] = run;
        run += x;
      }
    }
  }
}

// ============================================================================
// KU: range histogram (level-0 prescan).  CTA c counts keys
// [c*E, min(n, (c+1)*E)) where E = K tiles, and writes R[c][0..m).
// ============================================================================
template <int KIND, bool SMALLM>
__global__ void __launch_bounds__(kThreads)
    ku_range_hist(const uint32_t *__restrict__ keys, uint32_t n, uint32_t elems_per_cta,
                  BucketParams bp, uint32_t *__restrict__ R, uint32_t *__restrict__ hdr) {
  MS_STAGE_SPLITTERS(bp, kMaxBuckets);
  extern __shared__ uint32_t ku_smem[];  // [kWarps][m]
  __shared__ uint32_t s_red[kWarps];
  griddep_launch_dependents();  // let KR (programmatic launch) get scheduled early
  const uint32_t m = bp.m, tid = threadIdx.x;
  const uint32_t lo = blockIdx.x * elems_per_cta;
  const uint32_t hi = (uint32_t)min((uint64_t)n, (uint64_t)lo + elems_per_cta);
  if (blockIdx.x == 0 && tid == 0) hdr[0] = 0u;  // key-domain error flag of this call (KF sets it)
  if constexpr (!SMALLM) {
    for (uint32_t i = tid; i < kWarps * m; i += kThreads) ku_smem[i] = 0u;
    __syncthreads();
  }
  uint32_t ones = 0;
  hist_range<KIND, SMALLM>(keys, lo, hi, bp, ku_smem + (tid >> 5) * m, ones);
  hist_flush<SMALLM>(ku_smem, m, ones, hi - lo, R + (size_t)blockIdx.x * m, s_red);
}

// ============================================================================
// KH: tile-granular prescan (stage API and three-launch mode).  CTA l counts
// tile [l*T, min(n, (l+1)*T)) into H[l][0..m)  (Eq.2's h_{j,l}, Alg.1).
// ============================================================================
template <int KIND, bool SMALLM>
__global__ void __launch_bounds__(kThreads)
    kh_tile_hist(const uint32_t *__restrict__ keys, uint32_t n, uint32_t tile, BucketParams bp,
                 uint32_t *__restrict__ H, uint32_t *__restrict__ hdr) {
  MS_STAGE_SPLITTERS(bp, kMaxBuckets);
  extern __shared__ uint32_t kh_smem[];
  __shared__ uint32_t s_red[kWarps];
  const uint32_t m = bp.m, tid = threadIdx.x;
  const uint32_t lo = blockIdx.x * tile;
  const uint32_t hi = (uint32_t)min((uint64_t)n, (uint64_t)lo + tile);
  if (hdr && blockIdx.x == 0 && tid == 0) hdr[0] = 0u;
  if constexpr (!SMALLM) {
    for (uint32_t i = tid; i < kWarps * m; i += kThreads) kh_smem[i] = 0u;
    __syncthreads();
  }
  uint32_t ones = 0;
  hist_range<KIND, SMALLM>(keys, lo, hi, bp, kh_smem + (tid >> 5) * m, ones);
  hist_flush<SMALLM>(kh_smem, m, ones, hi - lo, H + (size_t)blockIdx.x * m, s_red);
}

// ============================================================================
// KF: scan + postscan.
// ============================================================================
constexpr uint32_t kMaxPeers = 8;  // ranks of one node (sharded fused scatter)

enum KfMode : int {
  kModeRange = 0,   // offsets from the range histograms R (two launches: KU, KF)
  kModeTileG = 1,   // offsets G[l][j] given per tile (three launches: KH, KG, KF)
  kModeSingle = 2,  // n <= T: one tile, one launch; the tile histogram is global
};

struct KfArgs {
  const uint32_t *keys_in;
  const uint32_t *vals_in;
  uint32_t *keys_out;
  uint32_t *vals_out;
  uint32_t n;
  uint32_t num_tiles;
  uint32_t tiles_per_cta;
  uint32_t num_ranges;
  const uint32_t *R;     // [num_ranges][m] column exclusive prefix of the range histograms (kModeRange)
  const uint32_t *Tot;   // [m] bucket totals (kModeRange)
  const uint32_t *Gt;    // [num_tiles][m] column part of Eq.2 offsets (kModeTileG)
  const uint32_t *base;  // [m] bucket bases, first term of Eq.2 (kModeTileG)
  const uint32_t *meta;  // [num_tiles][meta_stride] tile meta records from KM (kf_meta)
  uint32_t *hdr;         // [0] key-domain error flag
  uint32_t *bucket_offsets;
  int mode;
  int use_tma;     // TMA bulk loads of input tiles (inputs 16-byte aligned)
  int store_runs;  // TMA bulk stores of whole bucket runs (m <= 64, outputs 16-byte aligned)
  int rank_inc;    // rank by lane-ordered shared-memory increments (reading R23, probed per device)
  uint32_t prefix_step;  // kf_meta_wide: first row of range c in the range histograms = c * prefix_step
  uint32_t r_rows;       // kf_meta_wide: rows of the range histograms R (prescan CTAs)
  // sharded fused scatter (KP, Eq.3 with the GPUs as level 0): the bucket bases
  // are the global A_b + B_{b,r} and every element goes to the output window of
  // the rank that owns its global position (kf_meta / kf_meta_wide only)
  const uint32_t *gbase_ovr;   // [m] global bucket bases of this rank, or null (local)
  const uint32_t *peer_start;  // [npeers + 1] first global position of each output shard
  uint32_t npeers;             // 0: local outputs keys_out / vals_out
  uint32_t *peer_k[kMaxPeers];
  uint32_t *peer_v[kMaxPeers];
};

// store of a scattered element at global position p: local, or (sharded) into
// the window of the rank owning p (s_ps: the npeers + 1 shard starts in smem)
template <bool PAIRS>
__device__ __forceinline__ void kp_store(const KfArgs &a, const uint32_t *s_ps, uint32_t p,
                                         uint32_t k, uint32_t v) {
  uint32_t d = 0;
#pragma unroll
  for (uint32_t g = 1; g < kMaxPeers; ++g) d += (g < a.npeers && p >= s_ps[g]) ? 1u : 0u;
  const uint32_t o = p - s_ps[d];
  a.peer_k[d][o] = k;
  if constexpr (PAIRS) a.peer_v[d][o] = v;
}

// CTA shapes by bucket class (warps W, windows per warp ITEMS; tile T = 32 W ITEMS),
// chosen so that two (m <= 32, pairs) or three (keys, m > 32) CTAs fit in an SM's 228 KB:
//   class 0, m <= 32 : keys 16 x 16 (T 8192), pairs 16 x 16 (T 4096), warp scan, 1 bucket/lane
//   class 1, m <= 64 : keys  8 x 16 (T 4096), pairs  8 x 16 (T 4096), warp scan, 2 buckets/lane
//   class 2, m >  64 : keys  8 x 16 (T 4096), pairs  8 x 16 (T 4096), block scan
// (pairs: 4096-pair tiles measured faster than 2048 at m = 256: bucket runs of
// 16 instead of 8 elements, fewer partially written sectors)
__host__ __device__ constexpr int kf_class(uint32_t m) { return m <= 32 ? 0 : (m <= 64 ? 1 : 2); }
struct KfShape {
  int warps, items, ctas_per_sm;
};
__host__ __device__ constexpr KfShape kf_shape(bool pairs, int cls) {
  // classes 1-2, pairs: 4096-pair tiles (bucket runs of 16 at m = 256), 2 CTAs / SM
  return cls == 0 ? KfShape{16, pairs ? 8 : 16, 2} : (pairs ? KfShape{8, 16, 2} : KfShape{8, 16, 3});
}
__host__ __device__ constexpr uint32_t kf_tile(bool pairs, int cls) {
  return 32u * (uint32_t)kf_shape(pairs, cls).warps * (uint32_t)kf_shape(pairs, cls).items;
}

// Reordered-tile capacity: T slots plus up to 4m+4 of padding, so that every
// bucket run can start at the same offset mod 4 as its global destination
// (16-byte aligned TMA bulk stores of the run body; m <= 64 only).
__host__ __device__ constexpr uint32_t kf_out_slots(uint32_t T, uint32_t m) {
  return m > 64 ? T : T + 4u * (m < 2 ? 2u : m) + 4u;
}
// Shared memory (bytes): 3 tile stages (each padded to kf_out_slots, keys then values)
// | peer masks [2 or 3][W][m]
// | per-warp counts [W][m] | per-warp running slots [W][m] (m <= 64) | delta[m]
// | run table [3][m] (m <= 64)
// (inc: ranking by lane-ordered increments, no peer-mask rows)
__host__ __device__ inline size_t kf_smem_bytes(uint32_t m, bool pairs, bool inc = false) {
  const int cls = kf_class(m);
  const size_t T = kf_tile(pairs, cls), W = (size_t)kf_shape(pairs, cls).warps;
  const size_t k = pairs ? 2u : 1u;
  const size_t mm = m < 2 ? 2 : m;
  const size_t mrows = inc ? 0 : (cls == 0 ? 3 : 2);
  const size_t rows = mrows + (cls == 2 ? 1 : 2);  // masks + counts (+ slots)
  const size_t tables = cls == 2 ? 1 : 4;
  return 3 * (size_t)kf_out_slots((uint32_t)T, m) * k * 4 + rows * W * mm * 4 + tables * mm * 4;
}

// SCAN = 1 (m <= 32) / 2 (m <= 64): every warp scans the m x W tile counts
// itself, holding SCAN buckets per lane, so a tile needs two CTA barriers
// (after ranking, after reordering); SCAN = 0: block-wide scan.
// running[k] = next global position of bucket lane + 32k (SCAN > 0) or of
// bucket tid (block scan).
template <int KIND, bool PAIRS, bool SMALLM, int W, int ITEMS, int SCAN, bool FULL>
__device__ __forceinline__ void kf_do_tile(const KfArgs &a, const BucketParams &bp, uint32_t tile,
                                           uint32_t tn, uint32_t *s_stage, uint32_t OS,
                                           uint32_t *s_mask, uint32_t *s_cnt,
                                           uint32_t *s_base, uint32_t *s_delta, uint32_t *s_run,
                                           uint32_t *s_wsum, uint32_t (&running)[2]) {
  constexpr uint32_t NT = W * 32;
  constexpr uint32_t T = NT * ITEMS;
  constexpr bool WSCAN = SCAN != 0;
  constexpr int NBL = SCAN == 2 ? 2 : 1;  // buckets per lane in the warp scan
  const uint32_t m = bp.m;
  const uint32_t re = SMALLM ? 2u : m;  // counters per warp row
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t lt = lanemask_lt(), lanebit = 1u << lane;
  const uint32_t wbase = warp * (ITEMS * 32);
  uint32_t *crow = s_cnt + warp * re;
  uint32_t *mrow0 = s_mask + warp * re;        // window parity 0
  uint32_t *mrow1 = s_mask + (W + warp) * re;  // window parity 1
  uint32_t *mrow2 = s_mask + (2 * W + warp) * re;  // m <= 32: windows i mod 3
  // the tile is reordered in place: keys arrive in stage[0, T) (values in
  // stage[OS, OS + T)), every lane holds its elements in registers from the count
  // pass on, and the reordered tile is written back into the same stage
  const uint32_t *in_k = s_stage + wbase + lane;  // element i of this lane: in_k[32 i]
  const uint32_t *in_v = s_stage + OS + wbase + lane;
  uint32_t *out_k = s_stage;
  uint32_t *out_v = s_stage + OS;
  auto valid_at = [&](int i) { return FULL || wbase + (uint32_t)i * 32u + lane < tn; };

  // ---- 1. count pass: each warp's bucket counts (Eq.4 terms 2-3 need them
  //         before any element can be placed) -----------------------------------
  if constexpr (!SMALLM) {
    if (a.rank_inc) {
      for (uint32_t j = lane; j < m; j += 32) crow[j] = 0u;
    } else {
      for (uint32_t j = lane; j < m; j += 32) {
        mrow0[j] = 0u;
        mrow1[j] = 0u;
        if constexpr (SCAN == 1) mrow2[j] = 0u;
        crow[j] = 0u;
      }
    }
    __syncwarp();
  }
  bool derr = false;
  uint32_t key[ITEMS];
  uint32_t val[PAIRS ? ITEMS : 1];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) key[i] = valid_at(i) ? in_k[32 * i] : 0u;
  if constexpr (PAIRS) {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) val[i] = valid_at(i) ? in_v[32 * i] : 0u;
  }
  {
    uint32_t c0 = 0, c1 = 0;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const bool valid = valid_at(i);
      const uint32_t b = bucket_of<KIND>(key[i], bp);
      if constexpr (KIND == kIdentity) derr |= valid && key_domain_error<KIND>(key[i], bp);
      if constexpr (SMALLM) {
        const uint32_t ones = __ballot_sync(0xFFFFFFFFu, valid && b != 0u);
        const uint32_t vm = FULL ? 0xFFFFFFFFu : __ballot_sync(0xFFFFFFFFu, valid);
        c1 += __popc(ones);
        c0 += __popc(vm & ~ones);
      } else {
        if (valid) atomicAdd(crow + b, 1u);
      }
    }
    if constexpr (SMALLM) {
      if (lane == 0) {
        crow[0] = c0;
        crow[1] = c1;
      }
    }
  }
  if constexpr (KIND == kIdentity) {
    if (__any_sync(0xFFFFFFFFu, derr) && lane == 0) atomicOr(a.hdr, 1u);
  }
  __syncthreads();  // every element is in registers: the stage may be overwritten

  uint32_t *brow = WSCAN ? s_base + warp * re : crow;  // this warp's running slot per bucket
  uint32_t wrun = 0;  // SCAN == 1: lane b's running slot of bucket b
  if constexpr (WSCAN) {
    // ---- 2'. per-warp scan: this warp's first slot for bucket b is the tile
    //   base tb[b] (buckets before b) + counts of b in warps before this one
    //   (Eq.4 terms 2-3), plus the run padding adj[b] (run stores).
    uint32_t colp[2] = {0u, 0u}, tot[2] = {0u, 0u};
#pragma unroll
    for (int k = 0; k < NBL; ++k) {
      const uint32_t b = lane + 32u * (uint32_t)k;
      if (b < m) {
#pragma unroll
        for (int w = 0; w < W; ++w) {
          const uint32_t c = s_cnt[w * re + b];
          tot[k] += c;
          colp[k] += ((uint32_t)w < warp) ? c : 0u;
        }
      }
    }
    uint32_t incl[2] = {tot[0], tot[1]};
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
      for (int k = 0; k < NBL; ++k) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl[k], o);
        if (lane >= (uint32_t)o) incl[k] += t;
      }
    }
    const uint32_t sum0 = NBL == 2 ? __shfl_sync(0xFFFFFFFFu, incl[0], 31) : 0u;
#pragma unroll
    for (int k = 0; k < NBL; ++k) {
      const uint32_t b = lane + 32u * (uint32_t)k;
      if (b < m) {
        const uint32_t tb = incl[k] - tot[k] + (k ? sum0 : 0u);
        uint32_t gs;
        if (a.mode == kModeSingle) {
          gs = tb;
          if (warp == 0 && a.bucket_offsets) {
            a.bucket_offsets[b] = tb;
            if (b == m - 1) a.bucket_offsets[m] = tn;
          }
        } else if (a.mode == kModeTileG) {
          gs = a.Gt[(size_t)tile * m + b] + a.base[b];
        } else {
          gs = running[k];
          running[k] += tot[k];
        }
        const uint32_t adj = a.store_runs ? 4u * b + ((gs - tb) & 3u) : 0u;
        brow[b] = tb + colp[k] + adj;
        if (k == 0) wrun = tb + colp[k] + adj;
        if (warp == 0) {
          if (a.store_runs) {
            s_run[b] = tb + adj;
            s_run[m + b] = gs;
            s_run[2 * m + b] = tot[k];
          } else {
            s_delta[b] = gs - tb;
          }
        }
      }
    }
    __syncwarp();
  } else {
  // ---- 2. tile exclusive scan of the counts in (bucket, warp) order ----------
  // (Eq.4 term 3 plus the tile's bucket bases: a stable local multisplit of
  // the tile, Sec.4.7 / Sec.5.6.2).  Entry q = b*W + w lives at s_cnt[w*re + b].
  {
    const uint32_t total = m * W;
    const uint32_t per = (total + NT - 1) / NT;
    const uint32_t q0 = tid * per, q1 = min(total, q0 + per);
    uint32_t s = 0;
    for (uint32_t q = q0; q < q1; ++q) s += s_cnt[(q % W) * re + q / W];
    uint32_t incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= (uint32_t)o) incl += t;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const uint32_t x = lane < (uint32_t)W ? s_wsum[lane] : 0u;
      uint32_t xi = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, xi, o);
        if (lane >= (uint32_t)o) xi += t;
      }
      if (lane < (uint32_t)W) s_wsum[lane] = xi - x;
    }
    __syncthreads();
    uint32_t run = s_wsum[warp] + incl - s;
    for (uint32_t q = q0; q < q1; ++q) {
      uint32_t *c = s_cnt + (q % W) * re + q / W;
      const uint32_t v = *c;
      *c = run;
      run += v;
    }
  }
  __syncthreads();

  // ---- 3. per bucket: global start gs of this tile's run (Eq.2/3 terms 1-2) --
  // With run stores, bucket b's run is placed at smem offset tb + adj with
  // adj = 4b + ((gs - tb) mod 4), congruent to gs mod 4 (runs cannot overlap).
  const uint32_t mw = (m + 31u) & ~31u;       // warps holding the m bucket threads
  if (tid < mw) {
    uint32_t tb = 0, te = 0, gs = 0;
    if (tid < m) {
      tb = s_cnt[tid];  // warp 0 row = tile bucket base
      te = tid + 1 < m ? s_cnt[tid + 1] : tn;
      if (a.mode == kModeSingle) {
        gs = tb;
        if (a.bucket_offsets) {
          a.bucket_offsets[tid] = tb;
          if (tid == m - 1) a.bucket_offsets[m] = tn;
        }
      } else if (a.mode == kModeTileG) {
        gs = a.Gt[(size_t)tile * m + tid] + a.base[tid];
      } else {
        gs = running[0];
        running[0] += te - tb;
      }
    }
    if (a.store_runs) {
      // every bucket thread has read its neighbour's base before any is shifted
      if (mw > 32) named_barrier_sync(1, mw); else __syncwarp();
      if (tid < m) {
        const uint32_t adj = 4u * tid + ((gs - tb) & 3u);
        s_run[tid] = tb + adj;
        s_run[m + tid] = gs;
        s_run[2 * m + tid] = te - tb;
        if (adj)
          for (uint32_t w = 0; w < (uint32_t)W; ++w) s_cnt[w * re + tid] += adj;
      }
    } else if (tid < m) {
      s_delta[tid] = gs - tb;
    }
  }
  __syncthreads();  // bucket threads have read warp 0's bases before it starts placing
  }  // block scan


  // ---- 3'. rank and place by lane-ordered increments of this warp's running
  //          slot per bucket (one shared-memory atomic per key; m > 2)
  if (!SMALLM && a.rank_inc) {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const bool valid = valid_at(i);
      if (!FULL && wbase + (uint32_t)i * 32u >= tn) continue;
      if (valid) {
        const uint32_t slot = atomicAdd(brow + bucket_of<KIND>(key[i], bp), 1u);
        out_k[slot] = key[i];
        if constexpr (PAIRS) out_v[slot] = val[i];
      }
    }
  } else
  // ---- 3. rank and place, window by window (Eq.4 term 1 + the running slot) --
  // Peer masks come from one shared-memory OR of the lane bit per key (the
  // ballot-based voting of Alg.3, in one instruction); masks are
  // double-buffered by window parity.  slot = this warp's running slot of the
  // bucket + same-bucket lanes below; the key (and value) is stored there.
  {
    uint32_t base0 = 0, base1 = 0, c0 = 0, c1 = 0;
    if constexpr (SMALLM) {
      base0 = brow[0];
      base1 = brow[1];
    }
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const bool valid = valid_at(i);
      if (!FULL && wbase + (uint32_t)i * 32u >= tn) continue;  // warp-uniform: past the tail
      const uint32_t b = bucket_of<KIND>(key[i], bp);
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
      } else if constexpr (SCAN == 1) {
        // m <= 32: lane j keeps bucket j's running slot in a register and reads
        // bucket j's mask to advance it; masks rotate over three rows so that one
        // __syncwarp per window orders the ORs, the reads and the clears
        uint32_t *mrow = (i % 3 == 0) ? mrow0 : ((i % 3 == 1) ? mrow1 : mrow2);
        uint32_t *mprev = (i % 3 == 0) ? mrow2 : ((i % 3 == 1) ? mrow0 : mrow1);
        if (valid) atomicOr(mrow + b, lanebit);
        __syncwarp();
        const uint32_t peers = valid ? mrow[b] : 0u;
        const uint32_t mine = lane < m ? mrow[lane] : 0u;
        slot = __shfl_sync(0xFFFFFFFFu, wrun, b) + __popc(peers & lt);
        if (i > 0 && lane < m) mprev[lane] = 0u;  // every lane read the previous row last window
        wrun += __popc(mine);
      } else {
        uint32_t *mrow = (i & 1) ? mrow1 : mrow0;
        if (valid) atomicOr(mrow + b, lanebit);
        __syncwarp();
        const uint32_t peers = valid ? mrow[b] : 0u;
        const uint32_t first = valid ? brow[b] : 0u;
        const uint32_t below = peers & lt;
        slot = first + __popc(below);
        __syncwarp();                // every lane has read before the leader writes
        if (valid && below == 0u) {  // group leader: clear this parity's mask, advance the slot
          mrow[b] = 0u;
          brow[b] = first + __popc(peers);
        }
      }
      if (valid) {
        out_k[slot] = key[i];
        if constexpr (PAIRS) out_v[slot] = val[i];
      }
    }
  }
  __syncthreads();

  if (a.store_runs) {
    // ---- 5a. one TMA bulk store per bucket run: the 16-byte aligned body by
    //          thread b, the <= 3 leading / trailing elements by threads 8b..8b+7
    // run bodies: one TMA bulk store per bucket, issued by the producer warp
    // (lane b, b + 32); every lane commits one bulk group per tile so that the
    // producer can later wait for all but the newest before refilling a stage
    if (warp == W - 1) {
      bool fenced = false;
      for (uint32_t b = lane; b < m; b += 32) {
        const uint32_t len = s_run[2 * m + b];
        const uint32_t gs = s_run[m + b];
        const uint32_t st = s_run[b];
        const uint32_t head = min(len, (4u - (gs & 3u)) & 3u);
        const uint32_t body = (len - head) & ~3u;
        if (body) {
          if (!fenced) fence_proxy_async_smem();  // generic smem writes -> async proxy
          fenced = true;
          tma_store_1d(a.keys_out + gs + head, out_k + st + head, body * 4u);
          if constexpr (PAIRS) tma_store_1d(a.vals_out + gs + head, out_v + st + head, body * 4u);
        }
      }
      bulk_commit();
    }
    for (uint32_t t8 = tid; t8 < 8u * m; t8 += NT) {
      const uint32_t b = t8 >> 3, j = t8 & 7u;
      const uint32_t len = s_run[2 * m + b];
      const uint32_t gs = s_run[m + b];
      const uint32_t head = min(len, (4u - (gs & 3u)) & 3u);
      const uint32_t tail = (len - head) & 3u;
      uint32_t e = 0xFFFFFFFFu;  // run-relative element this thread stores, if any
      if (j < 4u) {
        if (j < head) e = j;
      } else if (j - 4u < tail) {
        e = len - tail + (j - 4u);
      }
      if (e != 0xFFFFFFFFu) {
        const uint32_t st = s_run[b] + e;
        a.keys_out[gs + e] = out_k[st];
        if constexpr (PAIRS) a.vals_out[gs + e] = out_v[st];
      }
    }
    return;
  }

  // ---- 5. coalesced scatter: slot s of bucket b -> delta[b] + s --------------
  {
    const uint32_t s0 = wbase + lane;
    uint32_t key[ITEMS], pos[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) key[i] = out_k[s0 + 32 * i];
    {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) pos[i] = s_delta[bucket_of<KIND>(key[i], bp)] + s0 + 32 * i;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i)
      if (valid_at(i)) a.keys_out[pos[i]] = key[i];
    if constexpr (PAIRS) {
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) key[i] = out_v[s0 + 32 * i];
#pragma unroll
      for (int i = 0; i < ITEMS; ++i)
        if (valid_at(i)) a.vals_out[pos[i]] = key[i];
    }
    }
  }
}

template <int KIND, bool PAIRS, bool SMALLM, int W, int ITEMS, int MINB, int SCAN>
__global__ void __launch_bounds__(W * 32, MINB) kf_fused(KfArgs a, BucketParams bp) {
  MS_STAGE_SPLITTERS(bp, kMaxBuckets);
  constexpr bool WSCAN = SCAN != 0;
  constexpr uint32_t NT = W * 32;
  constexpr uint32_t T = NT * ITEMS;
  constexpr uint32_t kStages = 3;  // tile k lives in stage k % 3 from its TMA load to its stores
  extern __shared__ __align__(128) uint8_t kf_smem[];
  __shared__ __align__(8) uint64_t bar[kStages];
  __shared__ uint32_t s_wsum[32];
  const uint32_t m = bp.m;
  const uint32_t mm = m < 2 ? 2 : m;
  const uint32_t OS = kf_out_slots(T, m);         // words per stage region (keys; values after)
  const uint32_t SW = OS * (PAIRS ? 2u : 1u);     // words per stage
  uint32_t *stage0 = reinterpret_cast<uint32_t *>(kf_smem);
  uint32_t *s_mask = stage0 + kStages * SW;
  constexpr uint32_t kMaskRows = SCAN == 1 ? 3 : 2;  // m <= 32: triple-buffered masks
  uint32_t *s_cnt = s_mask + (a.rank_inc ? 0u : kMaskRows) * W * mm;  // no masks when ranking by increments
  uint32_t *s_base = s_cnt + W * mm;  // WSCAN only
  uint32_t *s_delta = WSCAN ? s_base + W * mm : s_base;
  uint32_t *s_run = s_delta + mm;
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr uint32_t kProducer = NT - 32;  // lane 0 of the last warp issues the TMA loads

  uint32_t t0 = 0, t1 = 1;
  if (a.mode != kModeSingle) {
    t0 = blockIdx.x * a.tiles_per_cta;
    t1 = min(a.num_tiles, t0 + a.tiles_per_cta);
    if (t0 >= t1) return;
  }
  auto tile_n = [&](uint32_t t) { return min(T, a.n - t * T); };
  auto issue = [&](uint32_t t, uint32_t st) {  // one elected thread starts the TMA bulk copy
    if (tid == kProducer && t < t1 && a.use_tma && tile_n(t) == T) {
      uint32_t *dst = stage0 + st * SW;
      const uint64_t pol = policy_evict_first();
      mbar_arrive_expect_tx(&bar[st], T * 4u * (PAIRS ? 2u : 1u));
      tma_load_1d(dst, a.keys_in + (size_t)t * T, T * 4u, &bar[st], pol);
      if constexpr (PAIRS) tma_load_1d(dst + OS, a.vals_in + (size_t)t * T, T * 4u, &bar[st], pol);
      // tiles beyond the three-stage ring: into L2 (evict_last) ahead of their TMA loads
      const uint32_t tp = t + 2;
      if (a.mode == kModeRange && tp < t1 && tile_n(tp) == T) {
        const uint64_t kp = policy_evict_last();
        prefetch_l2_bulk_hint(a.keys_in + (size_t)tp * T, T * 4u, kp);
        if constexpr (PAIRS) prefetch_l2_bulk_hint(a.vals_in + (size_t)tp * T, T * 4u, kp);
      }
    }
  };
  if (tid == 0) {
    for (uint32_t i = 0; i < kStages; ++i) mbar_init(&bar[i], 1);
    if (a.mode == kModeSingle) a.hdr[0] = 0u;
  }
  __syncthreads();
  issue(t0, 0);
  issue(t0 + 1, 1);

  // ---- level-0 offsets (Eq.3 terms 1-2): KG has scanned the m x G matrix of
  // range histograms, R[c][b] = sum_{c'<c} h_{b,c'}, base[b] = sum_{b'<b} total_{b'}
  uint32_t running[2] = {0u, 0u};
  griddep_wait();  // programmatic launch: KR's scan (and everything before it) is complete
  if (a.mode == kModeRange) {
    // bucket bases = exclusive scan of the totals (block scan; thread b holds bucket b)
    const uint32_t lane = tid & 31, warp = tid >> 5;
    const uint32_t t = tid < m ? __ldcg(a.Tot + tid) : 0u;
    uint32_t incl = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= (uint32_t)o) incl += x;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const uint32_t x = lane < (uint32_t)W ? s_wsum[lane] : 0u;
      uint32_t xi = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, xi, o);
        if (lane >= (uint32_t)o) xi += y;
      }
      if (lane < (uint32_t)W) s_wsum[lane] = xi - x;
    }
    __syncthreads();
    if (tid < m) {
      const uint32_t gbase = s_wsum[warp] + incl - t;
      s_delta[tid] = gbase + __ldcg(a.R + (size_t)blockIdx.x * m + tid);
      if (blockIdx.x == 0 && a.bucket_offsets) {
        a.bucket_offsets[tid] = gbase;
        if (tid == m - 1) a.bucket_offsets[m] = gbase + t;
      }
    }
    __syncthreads();
    if constexpr (WSCAN) {  // every warp keeps the offsets of buckets lane, lane + 32
      if (lane < m) running[0] = s_delta[lane];
      if (lane + 32 < m) running[1] = s_delta[lane + 32];
    } else if (tid < m) {
      running[0] = s_delta[tid];
    }
  }

  // ---- tiles of this range, in order; three stages rotate through
  //      TMA load -> count/place in place -> stores ----------------------------
  uint32_t k = 0;
  for (uint32_t t = t0; t < t1; ++t, ++k) {
    const uint32_t st = k % kStages;
    uint32_t *s_stage = stage0 + st * SW;
    const uint32_t tn = tile_n(t);
    if (a.use_tma && tn == T) {
      mbar_wait(&bar[st], (k / kStages) & 1u);
    } else {  // ragged last tile / unaligned input: plain loads
      for (uint32_t i = tid; i < tn; i += NT) {
        s_stage[i] = __ldg(a.keys_in + (size_t)t * T + i);
        if constexpr (PAIRS) s_stage[OS + i] = __ldg(a.vals_in + (size_t)t * T + i);
      }
      __syncthreads();
    }
    if (tn == T)
      kf_do_tile<KIND, PAIRS, SMALLM, W, ITEMS, SCAN, true>(a, bp, t, tn, s_stage, OS, s_mask,
                                                            s_cnt, s_base, s_delta, s_run, s_wsum,
                                                            running);
    else
      kf_do_tile<KIND, PAIRS, SMALLM, W, ITEMS, SCAN, false>(a, bp, t, tn, s_stage, OS, s_mask,
                                                             s_cnt, s_base, s_delta, s_run, s_wsum,
                                                             running);
    // refill stage (k+2) % 3 with tile t+2: its last user, tile t-1, was stored
    // from it; the producer warp waits until those bulk stores have read it (all
    // but its newest bulk group).  Plain loads/stores of tile t-1 from that stage
    // finished before this tile's first barrier.
    if (warp == W - 1) {
      if (a.store_runs) bulk_wait_read_newest_pending();
      __syncwarp();
      if (lane == 0) fence_proxy_async_smem();
      issue(t + 2, (k + 2) % kStages);
    }
  }
  if (a.store_runs) bulk_wait_all();  // run stores complete before smem is released
}

// ============================================================================
// KX: receiver merge of the sharded multisplit.  Element e of the packed
// receive buffer comes from source s (recv_starts[s] <= e < recv_starts[s+1])
// and goes to out[merge_offsets[s][f(key)] + e].  Runs of one (source, bucket)
// are consecutive in e, so stores are coalesced within each run.
// ============================================================================
template <int KIND, bool PAIRS>
__global__ void __launch_bounds__(256)
    kx_shard_merge(const uint32_t *__restrict__ keys, const uint32_t *__restrict__ vals,
                   uint32_t n, BucketParams bp, const uint32_t *__restrict__ starts,
                   const uint32_t *__restrict__ offs, uint32_t G, uint32_t *__restrict__ keys_out,
                   uint32_t *__restrict__ vals_out) {
  MS_STAGE_SPLITTERS(bp, kMaxBuckets);
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    uint32_t s = 0;
    while (s + 1 < G && __ldg(starts + s + 1) <= e) ++s;
    const uint32_t k = keys[e];
    const uint32_t p = __ldg(offs + (size_t)s * bp.m + bucket_of<KIND>(k, bp)) + e;
    keys_out[p] = k;
    if constexpr (PAIRS) vals_out[p] = vals[e];
  }
}

}  // namespace ms
