// ms_kernels.cuh -- the three stages of the multisplit on sm_100a.
//
//   KH  prescan  : per-tile bucket histogram H[l][j]          (Alg.1)
//   KG  scan     : decoupled-lookback exclusive scan of the
//                  row-vectorized H -> G, bucket bases        (Alg.1)
//   KS  postscan : tile-local stable rank + reorder in smem,
//                  coalesced scatter                          (Eq.4, Sec.5.6.2)
//
// Layout in HBM: H/G tile-major (H[l*m + j]) so that every tile writes and
// reads m contiguous words.  G holds only the column part sum_{l'<l} h_{j,l'}
// of Eq.(2); the bucket bases sum_{j'<j} sum_l h_{j',l} live in a separate
// (m+1)-word array written by the last scan CTA, and the postscan adds them.
#pragma once
#include "ms_device.cuh"

namespace ms {

// Histogram / rank strategies (picked per m by the host dispatcher).
enum Strategy : int {
  kCount1 = 0,  // m <= 2: per-thread count of bucket 1 (KH) / one ballot per window (KS)
  kPeers = 1,   // ceil(log2 m) ballots -> peer mask, leader update (Alg.2/3)
  kMatch = 2,   // __match_any_sync peer mask, leader update
  kAtomic = 3,  // KH only: one shared-memory atomic per key into warp-private counters
};

// Status word of the decoupled look-back: high 32 bits = flag, low = value.
constexpr unsigned long long kFlagAggregate = 1ull << 32;
constexpr unsigned long long kFlagInclusive = 2ull << 32;

// ============================================================================
// KH: prescan.  One CTA per tile of kTile keys.  Keys are read with 128-bit
// streaming loads (order is irrelevant for a histogram).  Per-warp counters
// live in shared memory (warp-level privatization); the tile
// column of H is their sum.  CTA b also zeroes slice b of the look-back
// status array (and CTA 0 the ticket / error words) for the following KG.
// ============================================================================
template <int KIND, int STRAT, int LOGM>
__global__ void __launch_bounds__(kThreads, 2)
    kh_prescan(const uint32_t *__restrict__ keys, uint32_t n, BucketParams bp,
               uint32_t *__restrict__ H, unsigned long long *__restrict__ zero_status,
               uint32_t zero_words, uint32_t *__restrict__ hdr) {
  extern __shared__ uint32_t kh_smem[];  // [kWarps][m]
  const uint32_t m = bp.m;
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t tile = blockIdx.x;
  const uint32_t tile_start = tile * (uint32_t)kTile;
  const uint32_t tile_n = min((uint32_t)kTile, n - tile_start);

  // zero this CTA's slice of the look-back status array (consumed by KG)
  if (zero_status) {
    const uint32_t per = (zero_words + gridDim.x - 1) / gridDim.x;
    const uint32_t lo = tile * per, hi = min(zero_words, lo + per);
    for (uint32_t i = lo + tid; i < hi; i += kThreads) zero_status[i] = 0ull;
    if (tile == 0 && tid < 2) hdr[tid] = 0u;  // [0] error flag, [1] scan ticket
  }

  uint32_t *cnt = kh_smem + warp * m;
  if constexpr (STRAT != kCount1) {
    for (uint32_t i = tid; i < kWarps * m; i += kThreads) kh_smem[i] = 0u;
    __syncthreads();
  }

  // each warp owns a contiguous quarter... of the tile: 4 x 128-bit loads / lane
  constexpr int kVec = kItems / 4;
  const uint32_t wbase = warp * (kItems * 32);
  uint32_t ones = 0, valid_cnt = 0;
  const bool full = (tile_n == (uint32_t)kTile);
  const bool aligned = ((reinterpret_cast<uintptr_t>(keys) & 15u) == 0);

#pragma unroll
  for (int v = 0; v < kVec; ++v) {
    const uint32_t e0 = wbase + (uint32_t)v * 128u + lane * 4u;  // first element of this lane
    uint32_t k4[4];
    bool ok4[4];
    if (full && aligned) {
      uint4 q = ldg_stream_v4(reinterpret_cast<const uint4 *>(keys + tile_start + e0));
      k4[0] = q.x; k4[1] = q.y; k4[2] = q.z; k4[3] = q.w;
#pragma unroll
      for (int c = 0; c < 4; ++c) ok4[c] = true;
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        ok4[c] = (e0 + c) < tile_n;
        k4[c] = ok4[c] ? __ldg(keys + tile_start + e0 + c) : 0u;
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint32_t b = bucket_of<KIND>(k4[c], bp);
      if constexpr (STRAT == kCount1) {
        ones += ok4[c] ? b : 0u;
        valid_cnt += ok4[c] ? 1u : 0u;
      } else if constexpr (STRAT == kAtomic) {
        if (ok4[c]) atomicAdd(cnt + b, 1u);
      } else {
        const uint32_t active = __ballot_sync(0xFFFFFFFFu, ok4[c]);
        uint32_t peers;
        if constexpr (STRAT == kMatch) {
          peers = __match_any_sync(0xFFFFFFFFu, ok4[c] ? b : 0xFFFFFFFFu) & active;
        } else {
          peers = peer_mask_ballot<LOGM>(b, active, ok4[c]);
        }
        const bool leader = ok4[c] && ((peers & lanemask_lt()) == 0u);
        if (leader) atomicAdd(cnt + b, (uint32_t)__popc(peers));
      }
    }
  }

  if constexpr (STRAT == kCount1) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ones += __shfl_xor_sync(0xFFFFFFFFu, ones, o);
      valid_cnt += __shfl_xor_sync(0xFFFFFFFFu, valid_cnt, o);
    }
    __shared__ uint32_t w1[kWarps], wv[kWarps];
    if (lane == 0) { w1[warp] = ones; wv[warp] = valid_cnt; }
    __syncthreads();
    if (tid == 0) {
      uint32_t o = 0, v = 0;
      for (int w = 0; w < kWarps; ++w) { o += w1[w]; v += wv[w]; }
      if (m == 1) {
        H[tile] = v;
      } else {
        H[tile * 2 + 0] = v - o;
        H[tile * 2 + 1] = o;
      }
    }
  } else {
    __syncthreads();
    for (uint32_t j = tid; j < m; j += kThreads) {
      uint32_t s = 0;
#pragma unroll 4
      for (int w = 0; w < kWarps; ++w) s += kh_smem[w * m + j];
      H[tile * m + j] = s;
    }
  }
}

// ============================================================================
// KS: postscan.  One CTA per tile.
//  1. TMA bulk copy of the tile's keys (and values) into shared memory.
//  2. Each warp ranks its contiguous kItems*32 elements window by window
//     (lane i holds element i of the window): rank = warp-private
//     running count of the bucket + same-bucket lanes below (Eq.4 terms 1-2).
//  3. Block exclusive scan of the warp counts in (bucket, warp) order gives
//     the tile's stable local multisplit slot (Eq.4 term 3 + tile bucket base,
//     block-level reordering Sec.5.6.2).
//  4. Keys (then values) are written to their slots in shared memory.
//  5. Slot s of bucket b goes to out[G[l][b] + base[b] + s - tilebase[b]]:
//     consecutive threads write consecutive addresses inside each bucket run.
// SINGLE (n <= kTile): G = 0 and base = tile bases; writes bucket_offsets.
// ============================================================================
struct KsArgs {
  const uint32_t *keys_in;
  const uint32_t *vals_in;
  uint32_t *keys_out;
  uint32_t *vals_out;
  uint32_t n;
  const uint32_t *G;     // [L][m] column prefix (multi-tile)
  const uint32_t *base;  // [m+1] bucket bases (multi-tile)
  uint32_t *hdr;         // [0] error flag
  uint32_t *bucket_offsets;
  int single;
  int use_tma;
};

__host__ __device__ constexpr uint32_t ks_cnt_stride(uint32_t m) { return m + 1; }

__host__ __device__ inline size_t ks_smem_bytes(uint32_t m, bool pairs) {
  // keys tile (+ values tile) + counters [kWarps][m+1] + delta[m] + scratch
  return (size_t)kTile * 4u * (pairs ? 2u : 1u) + (size_t)kWarps * ks_cnt_stride(m) * 4u +
         (size_t)m * 4u + 64u * 4u;
}

template <int KIND, bool PAIRS, int STRAT, int LOGM>
__global__ void __launch_bounds__(kThreads, 2) ks_postscan(KsArgs a, BucketParams bp) {
  extern __shared__ __align__(128) uint32_t ks_smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t s_wsum[kWarps];
  const uint32_t m = bp.m;
  uint32_t *s_keys = ks_smem;
  uint32_t *s_vals = ks_smem + kTile;
  uint32_t *s_cnt = ks_smem + kTile * (PAIRS ? 2 : 1);  // [kWarps][m+1], warp-major
  uint32_t *s_delta = s_cnt + kWarps * ks_cnt_stride(m);
  const uint32_t stride = ks_cnt_stride(m);

  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t tile = blockIdx.x;
  const uint32_t tile_start = tile * (uint32_t)kTile;
  const uint32_t tile_n = min((uint32_t)kTile, a.n - tile_start);

  // ---- 1. load the tile into shared memory -------------------------------
  const uint32_t bulk_elems = a.use_tma ? (tile_n & ~3u) : 0u;  // 16-byte multiple
  if (tid == 0 && a.use_tma) mbar_init(&bar, 1);
  for (uint32_t i = bulk_elems + tid; i < tile_n; i += kThreads) {  // ragged tail / no-TMA
    s_keys[i] = __ldg(a.keys_in + tile_start + i);
    if constexpr (PAIRS) s_vals[i] = __ldg(a.vals_in + tile_start + i);
  }
  for (uint32_t i = tid; i < kWarps * stride; i += kThreads) s_cnt[i] = 0u;
  if (a.single && tid == 0) a.hdr[0] = 0u;
  __syncthreads();
  if (a.use_tma) {
    if (tid == 0 && bulk_elems > 0) {
      const uint64_t pol = policy_evict_first();
      mbar_arrive_expect_tx(&bar, bulk_elems * 4u * (PAIRS ? 2u : 1u));
      tma_load_1d(s_keys, a.keys_in + tile_start, bulk_elems * 4u, &bar, pol);
      if constexpr (PAIRS) tma_load_1d(s_vals, a.vals_in + tile_start, bulk_elems * 4u, &bar, pol);
    }
    if (bulk_elems > 0) mbar_wait(&bar, 0);
  }

  // ---- 2. warp-level ranking ---------------------------------------------
  const uint32_t wbase = warp * (kItems * 32);
  uint32_t key[kItems];
  uint32_t packed[kItems];  // (bucket << 16) | rank within warp
  const uint32_t lt = lanemask_lt();
  bool dom_err = false;
  uint32_t c0 = 0, c1 = 0;  // kCount1 running counts (warp-uniform)
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint32_t idx = wbase + (uint32_t)i * 32u + lane;
    const bool valid = idx < tile_n;
    key[i] = valid ? s_keys[idx] : 0u;
    const uint32_t b = bucket_of<KIND>(key[i], bp);
    dom_err |= valid && key_domain_error<KIND>(key[i], bp);
    if (wbase + (uint32_t)i * 32u >= tile_n) {  // window entirely past the tail
      packed[i] = 0u;
      continue;
    }
    if constexpr (STRAT == kCount1) {
      const uint32_t vmask = __ballot_sync(0xFFFFFFFFu, valid);
      const uint32_t ones = __ballot_sync(0xFFFFFFFFu, valid && b == 1u);
      const uint32_t zeros = vmask & ~ones;
      const uint32_t r = b ? c1 + __popc(ones & lt) : c0 + __popc(zeros & lt);
      packed[i] = (b << 16) | r;
      c1 += __popc(ones);
      c0 += __popc(zeros);
    } else {
      const uint32_t active = __ballot_sync(0xFFFFFFFFu, valid);
      uint32_t peers;
      if constexpr (STRAT == kMatch) {
        peers = __match_any_sync(0xFFFFFFFFu, valid ? b : 0xFFFFFFFFu) & active;
      } else {
        peers = peer_mask_ballot<LOGM>(b, active, valid);
      }
      const uint32_t below = peers & lt;
      uint32_t *ctr = s_cnt + warp * stride + b;
      const uint32_t old = valid ? *ctr : 0u;
      __syncwarp();
      if (valid && below == 0u) *ctr = old + (uint32_t)__popc(peers);
      __syncwarp();
      packed[i] = (b << 16) | (old + (uint32_t)__popc(below));
    }
  }
  if constexpr (STRAT == kCount1) {
    if (lane == 0) {
      s_cnt[warp * stride + 0] = c0;
      if (m > 1) s_cnt[warp * stride + 1] = c1;
    }
  }
  if constexpr (KIND == kIdentity) {
    if (__any_sync(0xFFFFFFFFu, dom_err) && lane == 0) atomicOr(a.hdr, 1u);
  }
  __syncthreads();

  // ---- 3. block exclusive scan of counts in (bucket, warp) order ---------
  {
    const uint32_t total = m * kWarps;
    const uint32_t per = (total + kThreads - 1) / kThreads;  // <= 8
    const uint32_t q0 = tid * per;
    uint32_t v[8];
    uint32_t s = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t q = q0 + e;
      v[e] = 0;
      if (e < (int)per && q < total) {
        const uint32_t b = q / kWarps, w = q % kWarps;
        v[e] = s_cnt[w * stride + b];
      }
      s += v[e];
    }
    uint32_t incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= (uint32_t)o) incl += t;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      uint32_t x = lane < (uint32_t)kWarps ? s_wsum[lane] : 0u;
      uint32_t xi = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, xi, o);
        if (lane >= (uint32_t)o) xi += t;
      }
      if (lane < (uint32_t)kWarps) s_wsum[lane] = xi - x;
    }
    __syncthreads();
    uint32_t run = s_wsum[warp] + incl - s;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t q = q0 + e;
      if (e < (int)per && q < total) {
        const uint32_t b = q / kWarps, w = q % kWarps;
        s_cnt[w * stride + b] = run;
        run += v[e];
      }
    }
  }
  __syncthreads();
  // tile bucket base = scanned (b, warp 0); delta[b] = global start - tile base
  for (uint32_t b = tid; b < m; b += kThreads) {
    const uint32_t tb = s_cnt[b];  // warp 0 row
    if (a.single) {
      s_delta[b] = 0u;
      if (a.bucket_offsets) a.bucket_offsets[b] = tb;
    } else {
      s_delta[b] = a.G[(size_t)tile * m + b] + a.base[b] - tb;
    }
  }
  if (a.single && tid == 0 && a.bucket_offsets) a.bucket_offsets[m] = tile_n;

  // ---- 4. reorder into shared memory --------------------------------------
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint32_t idx = wbase + (uint32_t)i * 32u + lane;
    if (idx < tile_n) {
      const uint32_t b = packed[i] >> 16;
      const uint32_t slot = s_cnt[warp * stride + b] + (packed[i] & 0xFFFFu);
      packed[i] = slot;
      s_keys[slot] = key[i];
    }
  }
  if constexpr (PAIRS) {
    uint32_t val[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const uint32_t idx = wbase + (uint32_t)i * 32u + lane;
      val[i] = idx < tile_n ? s_vals[idx] : 0u;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const uint32_t idx = wbase + (uint32_t)i * 32u + lane;
      if (idx < tile_n) s_vals[packed[i]] = val[i];
    }
  }
  __syncthreads();

  // ---- 5. coalesced scatter of bucket runs --------------------------------
#pragma unroll 4
  for (uint32_t s = tid; s < tile_n; s += kThreads) {
    const uint32_t k = s_keys[s];
    const uint32_t b = bucket_of<KIND>(k, bp);
    const uint32_t p = s_delta[b] + s;
    a.keys_out[p] = k;
    if constexpr (PAIRS) a.vals_out[p] = s_vals[s];
  }
}

}  // namespace ms
