// ms_wide.cuh -- the two-kernel pipeline of ms_meta.cuh widened to 32 < m <= 256
// buckets (the m = 64/128/256 multisplits of configs[2] and every 8-bit pass of
// the radix sort, configs[3]).
//
//   KMW km_meta_wide (prescan, P:534-535 extended): 16 counting warps count one
//       512-key slice each of every 8192-key tile into warp-private counters
//       (32-bit: same-address increments of one value merge in the shared-
//       memory atomic unit, so a 90 % hot bucket costs nothing); one scan warp turns them into tile meta records
//       S[w][b] = sum_{b'<b} h_b' + sum_{w'<w} c_{w',b}  (Eq.4 terms 2-3,
//       P:952-955), stored as 16-bit slot bases, and accumulates the range
//       histograms R[c][b] (the level-0 column of Eq.3).  The KM tile is the
//       KF tile (8192 keys or pairs, 16 warp slices of 512).
//   KR  kr_level0_scan (ms_kernels.cuh): P[c][b] = sum_{c'<c} R[c'][b], totals.
//   KFW kf_meta_wide (postscan): persistent CTA per level-0 range,
//       tiles in order; each warp takes its slot bases from its record row,
//       ranks its keys (Eq.4 term 1) by lane-ordered increments of packed
//       16-bit running slots (reading R23), places them in shared memory in
//       place, one barrier, then the coalesced per-element scatter.
//
// Why (profiles/r02/dram0_*, smem_ubench): at m = 256 the single-kernel
// postscan (kf_fused: count pass + block scan of the m x W counts + rank +
// reorder) spends 16.8 shared-memory wavefronts per 32 keys and reaches
// 2.2-2.6 TB/s; moving the count pass and the scan into the prescan (whose
// shared-memory pipe is idle while it streams the keys) leaves the postscan
// one atomic, one store and two loads per key.  The price is the records:
// 2 B per key written and read at m = 256 keys (1 B per pair), which the
// paper's recompute-instead-of-store choice (P:778 footnote) avoided on a GPU
// whose postscan was not the bottleneck.
//
// Buckets are laid out blocked: lane l owns buckets NB*l .. NB*l+NB-1, and the
// records, counters and range histograms use the padded width mP = 32 NB
// (buckets >= m are empty).
#pragma once
#include "ms_meta.cuh"

namespace ms {

__host__ __device__ constexpr uint32_t wide_nb(uint32_t m) {
  return m <= 64 ? 2u : (m <= 128 ? 4u : 8u);
}
// KF tile and its warp count: W warps x 16 windows, W = 32 for keys (16384
// keys, 1024 threads) and 16 for pairs (8192 pairs, 128 registers); one CTA
// per SM, 3 stages of 64 KB.  Measured, the postscan's DRAM efficiency follows
// the length of the bucket runs a tile writes (T/m elements): 4096-pair tiles
// (runs of 16 at m = 256) reached 2.3 TB/s, runs of 32 3.1 TB/s (profiles/r02).
// The KM tile is the KF tile, counted by W warps.
__host__ __device__ constexpr uint32_t wide_kw(bool pairs) { return pairs ? 16u : 32u; }
__host__ __device__ constexpr uint32_t wide_ctas_per_sm(bool) { return 1u; }
__host__ __device__ constexpr uint32_t wide_tile(bool pairs) { return 32u * 16u * wide_kw(pairs); }
// record: KW rows of mP 16-bit slot bases
__host__ __device__ constexpr uint32_t wide_rec_words(bool pairs, uint32_t nb) {
  return wide_kw(pairs) * 32u * nb / 2u;
}
// KMW shared memory <= 96 KB (two CTAs per SM): 32-bit warp counters, two
// buffers of W rows of 32 NB words, and as many TMA units of 8192 keys (32 KB)
// as fit, at most 3 (keys at m > 128: 64 KB of counters, one unit)
// counter buffers: two (the counting warps run a tile ahead of the scan warp),
// one where two would take more than 32 KB (keys at m > 128: the ring keeps two
// units, measured faster than two counter buffers and one unit)
__host__ __device__ constexpr uint32_t kmw_cnt_bufs(uint32_t nb, bool pairs) {
  return wide_kw(pairs) * 32u * nb * 2u <= 8192u ? 2u : 1u;
}
__host__ __device__ constexpr uint32_t kmw_cnt_words(uint32_t nb, bool pairs) {
  return kmw_cnt_bufs(nb, pairs) * wide_kw(pairs) * 32u * nb;
}
__host__ __device__ constexpr uint32_t kmw_stages(uint32_t nb, bool pairs) {
  return (24576u - kmw_cnt_words(nb, pairs)) / 8192u > 3u ? 3u : (24576u - kmw_cnt_words(nb, pairs)) / 8192u;
}
__host__ __device__ inline size_t kmw_smem_bytes(uint32_t nb, bool pairs) {
  return ((size_t)kmw_stages(nb, pairs) * 8192u + kmw_cnt_words(nb, pairs)) * 4u;
}
__host__ __device__ inline size_t kfw_smem_bytes(bool pairs, uint32_t nb) {
  const uint32_t T = wide_tile(pairs);
  // 3 stages of [keys | values | record row 0], rank rows, 2 run tables, running offsets
  return (3u * (T * (pairs ? 2u : 1u) + 16u * nb) + wide_kw(pairs) * 16u * nb + 2u * 32u * nb + 32u * nb) * 4u;
}

template <int NB>
struct WideVec;  // NB/2 packed words
template <> struct WideVec<2> { using T = uint32_t; };
template <> struct WideVec<4> { using T = uint2; };
template <> struct WideVec<8> { using T = uint4; };

// NB consecutive 32-bit words of shared memory (16-byte vector accesses)
template <int NB>
__device__ __forceinline__ void ld_words(const uint32_t *p, uint32_t (&u)[NB]) {
  if constexpr (NB == 2) {
    const uint2 v = *reinterpret_cast<const uint2 *>(p);
    u[0] = v.x;
    u[1] = v.y;
  } else {
#pragma unroll
    for (int q = 0; q < NB / 4; ++q) {
      const uint4 v = reinterpret_cast<const uint4 *>(p)[q];
      u[4 * q] = v.x;
      u[4 * q + 1] = v.y;
      u[4 * q + 2] = v.z;
      u[4 * q + 3] = v.w;
    }
  }
}
template <int NB>
__device__ __forceinline__ void st_zero_words(uint32_t *p) {
  if constexpr (NB == 2) {
    *reinterpret_cast<uint2 *>(p) = make_uint2(0u, 0u);
  } else {
#pragma unroll
    for (int q = 0; q < NB / 4; ++q) reinterpret_cast<uint4 *>(p)[q] = make_uint4(0u, 0u, 0u, 0u);
  }
}

template <int NB>
__device__ __forceinline__ void wide_unpack(const typename WideVec<NB>::T &v, uint32_t (&w)[NB / 2]) {
  if constexpr (NB == 2) {
    w[0] = v;
  } else if constexpr (NB == 4) {
    w[0] = v.x;
    w[1] = v.y;
  } else {
    w[0] = v.x;
    w[1] = v.y;
    w[2] = v.z;
    w[3] = v.w;
  }
}
template <int NB>
__device__ __forceinline__ typename WideVec<NB>::T wide_pack(const uint32_t (&w)[NB / 2]) {
  if constexpr (NB == 2) {
    return w[0];
  } else if constexpr (NB == 4) {
    return make_uint2(w[0], w[1]);
  } else {
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// ============================================================================
// KMW.  CTA c handles KF tiles [c*K, min(LM, (c+1)*K)); a tile has W slices of
// 512 keys (W = 32 keys / 16 pairs), each a record row.  The TMA unit is a
// half tile of 8192 keys (32 KB; H = W / 16 units per tile) in a ring of KS
// units; the 16 counting warps count slice w of every unit into row
// (h * 16 + w) of the tile's 32-bit counters (kmw_cnt_bufs buffers; a
// constant +1 compiles to ATOMS.POPC.INC, which merges a warp's same-address
// increments: packed 16-bit counters made the 90 %-skewed C3 prescan 4x
// slower), then arrive on the unit's sfree barrier.  The scan warp refills a
// stage as soon as its unit is counted and, once every unit of a tile is,
// turns the counters into the record and zeroes them.  <= 96 KB of shared
// memory: two CTAs per SM.
// ============================================================================
__host__ __device__ constexpr uint32_t kmw_unit() { return 8192u; }

// Scan warps: two at m > 128 (each owns half the buckets; the one scan warp
// was the prescan's bottleneck there, measured: the counting warps waited on
// the counter buffer for 60 % of their samples), else one.
__host__ __device__ constexpr uint32_t kmw_scan_warps(uint32_t nb) { return nb == 8 ? 2u : 1u; }

template <int KIND, int NB, bool PAIRS>
__global__ void __launch_bounds__(kThreads + 64, 2)
    km_meta_wide(const uint32_t *__restrict__ keys, uint32_t n, uint32_t num_tiles,
                 uint32_t tiles_per_cta, BucketParams bp, uint32_t *__restrict__ meta,
                 uint32_t num_kf_tiles, uint32_t *__restrict__ R, uint32_t *__restrict__ hdr) {
  MS_STAGE_SPLITTERS(bp, kMaxBuckets);
  constexpr uint32_t W = wide_kw(PAIRS), CW = kWarps, SL = 512, T = W * SL, U = CW * SL;
  constexpr uint32_t H = W / CW;                  // TMA units per tile
  constexpr uint32_t KS = kmw_stages(NB, PAIRS);  // units in the ring
  constexpr uint32_t CB = kmw_cnt_bufs(NB, PAIRS);  // counter buffers
  constexpr uint32_t SW = kmw_scan_warps(NB);     // scan warps
  constexpr int LB = NB / SW;                     // buckets per scan lane
  constexpr uint32_t HL = LB / 2;                 // packed record words per scan lane per row
  constexpr uint32_t RW = 16u * NB;               // packed record words per row (mP / 2)
  constexpr uint32_t MP = 32u * NB;               // counters per row
  constexpr uint32_t REC = wide_rec_words(PAIRS, NB);
  using VL = typename WideVec<LB>::T;
  extern __shared__ __align__(128) uint32_t kmw_smem[];  // stages [KS][U] | cnt[CB][W][MP]
  __shared__ __align__(8) uint64_t full[KS];
  __shared__ __align__(8) uint64_t sfree[KS];
  __shared__ __align__(8) uint64_t cempty[2];
  __shared__ uint32_t s_carry[2];  // SW = 2: the first scan warp's bucket total, by tile parity
  griddep_launch_dependents();
  uint32_t *cnt = kmw_smem + KS * U;
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (blockIdx.x == 0 && tid == 0) hdr[0] = 0u;
  for (uint32_t i = tid; i < CB * W * MP; i += blockDim.x) cnt[i] = 0u;
  const uint32_t t0 = blockIdx.x * tiles_per_cta;
  const uint32_t t1 = min(num_tiles, t0 + tiles_per_cta);
  const uint32_t nu = t1 > t0 ? (t1 - t0) * H : 0u;  // units of this CTA
  const bool aligned = ((reinterpret_cast<uintptr_t>(keys) & 15u) == 0);
  auto unit_start = [&](uint32_t u) { return (uint64_t)t0 * T + (uint64_t)u * U; };
  auto via_tma = [&](uint32_t u) { return aligned && unit_start(u) + U <= n; };
  if (tid == 0) {
    for (uint32_t i = 0; i < KS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&sfree[i], CW * 32u);
    }
    for (uint32_t i = 0; i < 2; ++i) mbar_init(&cempty[i], 32u * SW);
  }
  __syncthreads();

  if (warp >= CW) {
    // ============================ scan warps ==================================
    const uint32_t sidx = warp - CW, blk = sidx * 32u + lane;  // this lane's bucket block
    auto issue = [&](uint32_t u) {
      if (sidx == 0 && lane == 0 && u < nu && via_tma(u)) {
        const uint32_t st = u % KS;
        mbar_arrive_expect_tx(&full[st], U * 4u);
        tma_load_1d(kmw_smem + st * U, keys + unit_start(u), U * 4u, &full[st], policy_evict_first());
      }
    };
    for (uint32_t u = 0; u < KS; ++u) issue(u);
    uint32_t running[LB];
#pragma unroll
    for (int j = 0; j < LB; ++j) running[j] = 0u;
    uint32_t k = 0;
    for (uint32_t t = t0; t < t1; ++t, ++k) {
      const uint32_t p = k % CB;
#pragma unroll
      for (uint32_t h = 0; h < H; ++h) {  // every unit of the tile counted; refill its stage
        const uint32_t u = k * H + h;
        mbar_wait(&sfree[u % KS], (u / KS) & 1u);
        if (lane == 0) fence_proxy_async_smem();
        issue(u + KS);
      }
      uint32_t *c = cnt + p * W * MP;
      // pass 1: tile count h of this lane's buckets
      uint32_t hc[LB];
#pragma unroll
      for (int j = 0; j < LB; ++j) hc[j] = 0u;
#pragma unroll 4
      for (uint32_t w = 0; w < W; ++w) {
        uint32_t x[LB];
        ld_words<LB>(c + w * MP + blk * LB, x);
#pragma unroll
        for (int j = 0; j < LB; ++j) hc[j] += x[j];
      }
      // exclusive scan over the buckets (in-lane prefix, warp scan of lane sums,
      // and the first scan warp's total for the second)
      uint32_t tb[LB], s = 0;
#pragma unroll
      for (int j = 0; j < LB; ++j) {
        tb[j] = s;
        s += hc[j];
      }
      uint32_t incl = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= (uint32_t)o) incl += y;
      }
      uint32_t carry = 0;
      if constexpr (SW == 2) {
        if (sidx == 0 && lane == 31) s_carry[k & 1u] = incl;
        named_barrier_sync(1, 64);
        if (sidx == 1) carry = s_carry[k & 1u];
      }
#pragma unroll
      for (int j = 0; j < LB; ++j) {
        tb[j] += incl - s + carry;
        running[j] += hc[j];
      }
      // pass 2: S[w][b] = tb[b] + sum_{w'<w} c_{w',b} (16-bit); zero the counters
      uint32_t *rec = meta + (size_t)t * REC;
#pragma unroll 2
      for (uint32_t w = 0; w < W; ++w) {
        uint32_t *cw = c + w * MP + blk * LB;
        uint32_t x[LB], o[HL];
        ld_words<LB>(cw, x);
#pragma unroll
        for (int i = 0; i < (int)HL; ++i) {
          o[i] = (tb[2 * i] & 0xFFFFu) | (tb[2 * i + 1] << 16);
          tb[2 * i] += x[2 * i];
          tb[2 * i + 1] += x[2 * i + 1];
        }
        st_zero_words<LB>(cw);
        if (t < num_kf_tiles) reinterpret_cast<VL *>(rec + w * RW)[blk] = wide_pack<LB>(o);
      }
      __syncwarp();
      mbar_arrive(&cempty[p]);
    }
    uint32_t *r = R + (size_t)blockIdx.x * MP + blk * LB;
#pragma unroll
    for (int j = 0; j < LB; ++j) r[j] = running[j];
    return;
  }

  // ============================ counting warps ================================
  for (uint32_t u = 0; u < nu; ++u) {
    const uint32_t k = u / H, h = u % H, p = k % CB, st = u % KS;
    if (h == 0 && k >= CB) mbar_wait(&cempty[p], ((k - CB) / CB) & 1u);  // buffer p scanned and zeroed
    uint32_t *row = cnt + (p * W + h * CW + warp) * MP;
    if (via_tma(u)) {
      mbar_wait(&full[st], (u / KS) & 1u);
      const uint4 *v = reinterpret_cast<const uint4 *>(kmw_smem + st * U + warp * SL);
      uint4 q[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) q[i] = v[lane + 32u * (uint32_t)i];
      uint32_t bk[16];  // bucket ids first, then the increments (see km_tile_meta)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        bk[4 * i] = bucket_of<KIND>(q[i].x, bp);
        bk[4 * i + 1] = bucket_of<KIND>(q[i].y, bp);
        bk[4 * i + 2] = bucket_of<KIND>(q[i].z, bp);
        bk[4 * i + 3] = bucket_of<KIND>(q[i].w, bp);
      }
#pragma unroll
      for (int e = 0; e < 16; ++e) atomicAdd(row + bk[e], 1u);
    } else {  // ragged last unit / unaligned input
      const uint64_t lo = unit_start(u) + warp * SL;
      const uint32_t hi = (uint32_t)min((uint64_t)n, lo + SL);
      for (uint32_t i = (uint32_t)lo + lane; i < hi; i += 32u) {
        atomicAdd(row + bucket_of<KIND>(__ldg(keys + i), bp), 1u);
      }
    }
    mbar_arrive(&sfree[st]);
  }
}

// ============================================================================
// KFW: persistent CTA per level-0 range (KF tiles [c K, (c+1) K)), KW warps.
//   iteration k (tile t): per-warp setup from the record row (loaded into
//   registers with the tile's keys); rank + place in place; load tile t+1
//   into registers; one barrier; per-element coalesced scatter of tile t;
//   the last warp refills the stage of tile t-1 with tile t+2.
// ============================================================================
template <int KIND, bool PAIRS, int NB>
__global__ void __launch_bounds__(wide_kw(PAIRS) * 32, wide_ctas_per_sm(PAIRS)) kf_meta_wide(KfArgs a, BucketParams bp) {
  MS_STAGE_SPLITTERS(bp, kMaxBuckets);
  constexpr uint32_t W = wide_kw(PAIRS), NT = W * 32, ITEMS = 16;
  constexpr uint32_t T = NT * ITEMS;
  constexpr uint32_t kStages = 3, kPrefetch = 2;
  constexpr uint32_t HW = NB / 2, RW = 16u * NB, MP = 32u * NB;
  constexpr uint32_t REC = wide_rec_words(PAIRS, NB);
  constexpr uint32_t SWD = T * (PAIRS ? 2u : 1u) + RW;  // words per stage: keys | values | record row 0
  constexpr uint32_t R0 = T * (PAIRS ? 2u : 1u);        // offset of record row 0 in a stage
  using V = typename WideVec<NB>::T;
  extern __shared__ __align__(128) uint8_t kfw_raw[];
  __shared__ __align__(8) uint64_t bar[kStages];
  __shared__ uint32_t s_ps[kMaxPeers + 1];  // sharded: output shard starts
  __shared__ uint32_t s_hot[2];             // per tile parity: the hot bucket, or ~0u
  uint32_t *stage0 = reinterpret_cast<uint32_t *>(kfw_raw);
  uint32_t *s_row = stage0 + kStages * SWD;  // [W][RW] packed running slots
  uint32_t *s_tab = s_row + W * RW;          // [2][MP] global minus tile offsets
  uint32_t *s_grun = s_tab + 2u * MP;        // [MP] next global position of each bucket in this range
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr uint32_t kProducer = NT - 32;

  const uint32_t t0 = blockIdx.x * a.tiles_per_cta;
  const uint32_t t1 = min(a.num_tiles, t0 + a.tiles_per_cta);
  if (t0 >= t1) return;
  const uint32_t nt = t1 - t0;
  auto tile_n = [&](uint32_t t) { return min(T, a.n - t * T); };
  auto via_tma = [&](uint32_t t) { return a.use_tma && tile_n(t) == T; };
  // one elected thread starts the TMA copies of a tile: the input (may run
  // before griddep_wait: it predates KMW) and record row 0 (written by KMW:
  // only after griddep_wait); one mbarrier transaction count for both
  auto issue_data = [&](uint32_t t, uint32_t st) {
    if (tid == kProducer && t < t1 && via_tma(t)) {
      uint32_t *dst = stage0 + st * SWD;
      const uint64_t pol = policy_evict_first();
      mbar_arrive_expect_tx(&bar[st], T * 4u * (PAIRS ? 2u : 1u) + RW * 4u);
      tma_load_1d(dst, a.keys_in + (size_t)t * T, T * 4u, &bar[st], pol);
      if constexpr (PAIRS) tma_load_1d(dst + T, a.vals_in + (size_t)t * T, T * 4u, &bar[st], pol);
    }
  };
  auto issue_rec = [&](uint32_t t, uint32_t st) {
    if (tid == kProducer && t < t1 && via_tma(t))
      tma_load_1d(stage0 + st * SWD + R0, a.meta + (size_t)t * REC, RW * 4u, &bar[st], policy_evict_first());
  };
  auto issue = [&](uint32_t t, uint32_t st) {
    issue_data(t, st);
    issue_rec(t, st);
  };
  auto prefetch = [&](uint32_t t, bool meta) {
    if (tid == kProducer && t < t1) {
      const uint64_t pol = policy_evict_last();
      if (via_tma(t)) {
        prefetch_l2_bulk_hint(a.keys_in + (size_t)t * T, T * 4u, pol);
        if constexpr (PAIRS) prefetch_l2_bulk_hint(a.vals_in + (size_t)t * T, T * 4u, pol);
      }
      if (meta) prefetch_l2_bulk_hint(a.meta + (size_t)t * REC, REC * 4u, pol);
    }
  };
  if (tid == 0)
    for (uint32_t i = 0; i < kStages; ++i) mbar_init(&bar[i], 1);
  __syncthreads();
  issue_data(t0, 0);
  issue_data(t0 + 1, 1);
  for (uint32_t j = 2; j < 2 + kPrefetch; ++j) prefetch(t0 + j, false);

  uint32_t key[ITEMS];
  uint32_t val[PAIRS ? ITEMS : 1];
  uint32_t mrow[HW];  // this warp's record row (packed 16-bit)
  const uint32_t wbase = warp * (ITEMS * 32);
  auto load_tile = [&](uint32_t t, uint32_t k) {
    const uint32_t st = k % kStages;
    const uint32_t *s = stage0 + st * SWD;
    const uint32_t tn = tile_n(t);
    const uint32_t *rec = a.meta + (size_t)t * REC;
    wide_unpack<NB>(__ldcg(reinterpret_cast<const V *>(rec + warp * RW) + lane), mrow);
    if (via_tma(t)) {
      mbar_wait(&bar[st], (k / kStages) & 1u);
#pragma unroll
      for (int i = 0; i < (int)ITEMS; ++i) key[i] = s[wbase + 32 * i + lane];
      if constexpr (PAIRS) {
#pragma unroll
        for (int i = 0; i < (int)ITEMS; ++i) val[i] = s[T + wbase + 32 * i + lane];
      }
    } else {
      const size_t g = (size_t)t * T;
#pragma unroll
      for (int i = 0; i < (int)ITEMS; ++i) {
        const uint32_t e = wbase + 32 * i + lane;
        key[i] = e < tn ? __ldg(a.keys_in + g + e) : 0u;
        if constexpr (PAIRS) val[i] = e < tn ? __ldg(a.vals_in + g + e) : 0u;
      }
    }
  };

  // ---- level-0 offsets (Eq.3 terms 1-2): KR's column prefix P[c][b] and the
  // bucket totals; base[b] = exclusive scan of the totals
  griddep_wait();  // KM and KR complete
  if (a.npeers && tid <= a.npeers) s_ps[tid] = __ldcg(a.peer_start + tid);
  issue_rec(t0, 0);
  issue_rec(t0 + 1, 1);
  for (uint32_t j = 2; j < 2 + kPrefetch; ++j) prefetch(t0 + j, true);
  // level-0 offsets without a scan kernel: the CTA reduces the range
  // histograms R (a.r_rows rows of KMW, L2-resident) to the bucket totals and
  // this range's column prefix (rows < c * prefix_step); stage 2 is scratch
  // until the first refill
  {
    constexpr uint32_t NG = NT / MP;
    uint32_t *red = stage0 + 2u * SWD;
    const uint32_t b = tid % MP, g = tid / MP, cp = blockIdx.x * a.prefix_step;
    uint32_t tp = 0, pp = 0;
#pragma unroll 8
    for (uint32_t r = g; r < a.r_rows; r += NG) {
      const uint32_t x = __ldcg(a.R + (size_t)r * MP + b);
      tp += x;
      pp += r < cp ? x : 0u;
    }
    red[g * MP + b] = tp;
    red[(NG + g) * MP + b] = pp;
  }
  __syncthreads();
  if (warp == W - 1) {  // the running offsets live in shared memory, kept by the last warp
    constexpr uint32_t NG = NT / MP;
    const uint32_t *red = stage0 + 2u * SWD;
    uint32_t grun[NB], tot[NB], pre[NB], s = 0;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const uint32_t b = lane * NB + j;
      tot[j] = pre[j] = 0u;
#pragma unroll
      for (uint32_t g = 0; g < NG; ++g) {
        tot[j] += red[g * MP + b];
        pre[j] += red[(NG + g) * MP + b];
      }
      grun[j] = s;
      s += tot[j];
    }
    uint32_t incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= (uint32_t)o) incl += y;
    }
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      grun[j] += incl - s;
      const uint32_t b = lane * NB + j;
      if (a.gbase_ovr) grun[j] = b < bp.m ? __ldcg(a.gbase_ovr + b) : 0u;
      if (blockIdx.x == 0 && a.bucket_offsets) {
        if (b < bp.m) a.bucket_offsets[b] = grun[j];
        if (b + 1 == bp.m) a.bucket_offsets[bp.m] = grun[j] + tot[j];
      }
      s_grun[b] = grun[j] + pre[j];
    }
  }
  __syncthreads();  // stage 2 scratch read before any refill
  // a tile whose largest bucket holds more than T/16 elements ranks that bucket
  // by ballots: lanes of one bucket in one increment instruction serialize in
  // the shared-memory atomic unit (90 % skew, C3).  The last warp finds it from
  // the tile's record row 0 (bucket bases) after loading the tile, before the
  // barrier that precedes the tile's ranking.
  auto find_hot = [&](uint32_t t, uint32_t k) {
    const uint32_t *r0 = via_tma(t) ? stage0 + (k % kStages) * SWD + R0 : a.meta + (size_t)t * REC;
    uint32_t m0[HW], tb[NB];
    wide_unpack<NB>(via_tma(t) ? reinterpret_cast<const V *>(r0)[lane]
                               : __ldcg(reinterpret_cast<const V *>(r0) + lane), m0);
#pragma unroll
    for (int j = 0; j < NB; ++j) tb[j] = (m0[j >> 1] >> ((j & 1) * 16)) & 0xFFFFu;
    const uint32_t nxt = __shfl_down_sync(0xFFFFFFFFu, tb[0], 1);
    uint32_t best = 0, bb = 0;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const uint32_t te = j + 1 < NB ? tb[j + 1] : (lane < 31 ? nxt : tile_n(t));
      if (te - tb[j] > best) {
        best = te - tb[j];
        bb = lane * NB + j;
      }
    }
    const uint32_t top = __reduce_max_sync(0xFFFFFFFFu, best);
    const uint32_t who = __ballot_sync(0xFFFFFFFFu, best == top);
    const uint32_t hot = __shfl_sync(0xFFFFFFFFu, bb, __ffs(who) - 1);
    if (lane == 0) s_hot[k & 1u] = top > T / 16u ? hot : ~0u;
  };
  load_tile(t0, 0);
  if (warp == W - 1) find_hot(t0, 0);
  __syncthreads();  // every warp holds tile t0 in registers before any places into its stage

  uint32_t *brow = s_row + warp * RW;
  // placement into the stage: keys alone, or (key, value) as one 64-bit word
  // (pairs: one store here and one load in the scatter instead of two each;
  // the stage's raw data is dead once every warp holds the tile in registers)
  auto place = [&](uint32_t *st, uint32_t slot, uint32_t k_, uint32_t v_) {
    if constexpr (PAIRS)
      reinterpret_cast<uint2 *>(st)[slot] = make_uint2(k_, v_);
    else
      st[slot] = k_;
  };
  for (uint32_t k = 0; k < nt; ++k) {
    const uint32_t t = t0 + k;
    const uint32_t st = k % kStages;
    uint32_t *s_stage = stage0 + st * SWD;
    const uint32_t tn = tile_n(t);
    uint32_t *tab = s_tab + (k & 1u) * MP;

    // ---- per-warp setup: running slots of this warp's buckets; the tile's
    // global offsets (Eq.3 term 3: grun accumulates the range's earlier tiles)
    if (warp == W - 1) {
      // record row 0 = the tile's bucket bases: from the stage (TMA) or global
      const uint32_t *r0 = via_tma(t) ? s_stage + R0 : a.meta + (size_t)t * REC;
      uint32_t mrow0[HW], tb[NB], g[NB];
      wide_unpack<NB>(via_tma(t) ? reinterpret_cast<const V *>(r0)[lane]
                                 : __ldcg(reinterpret_cast<const V *>(r0) + lane), mrow0);
#pragma unroll
      for (int j = 0; j < NB; ++j) tb[j] = (mrow0[j >> 1] >> ((j & 1) * 16)) & 0xFFFFu;
      ld_words<NB>(s_grun + lane * NB, g);
      const uint32_t nxt = __shfl_down_sync(0xFFFFFFFFu, tb[0], 1);
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const uint32_t te = j + 1 < NB ? tb[j + 1] : (lane < 31 ? nxt : tn);
        tab[lane * NB + j] = g[j] - tb[j];
        g[j] += te - tb[j];
      }
#pragma unroll
      for (int j = 0; j < NB; ++j) s_grun[lane * NB + j] = g[j];
    }
    reinterpret_cast<V *>(brow)[lane] = wide_pack<NB>(mrow);
    __syncwarp();

    // ---- rank and place: slot = lane-ordered increment of the packed 16-bit
    // running slot of the key's bucket (Eq.4 term 1, reading R23)
    // all increments of the warp first, then the placements: the increments
    // are in flight together (the probe checks exactly this back-to-back form)
    bool derr = false;
    const uint32_t hot = s_hot[k & 1u];
    if (tn == T && hot != ~0u) {
      // the hot bucket's keys take their slots from one ballot per window
      // (Alg.3 with the peer mask of a single bucket); the others increment
      uint32_t hbase = (brow[hot >> 1] >> ((hot & 1u) << 4)) & 0xFFFFu;
      const uint32_t lt = lanemask_lt();
#pragma unroll
      for (int i = 0; i < (int)ITEMS; ++i) {
        const uint32_t b = bucket_of<KIND>(key[i], bp);
        if constexpr (KIND == kIdentity) derr |= key_domain_error<KIND>(key[i], bp);
        const bool ish = b == hot;
        const uint32_t hm = __ballot_sync(0xFFFFFFFFu, ish);
        uint32_t slot;
        if (ish) {
          slot = hbase + __popc(hm & lt);
        } else {
          slot = atomicAdd(brow + (b >> 1), 1u << ((b & 1u) << 4));
          slot = (slot >> ((b & 1u) << 4)) & 0xFFFFu;
        }
        hbase += __popc(hm);
        place(s_stage, slot, key[i], PAIRS ? val[i] : 0u);
      }
    } else if (tn == T) {
      uint32_t slot[ITEMS], bk[ITEMS];
#pragma unroll
      for (int i = 0; i < (int)ITEMS; ++i) bk[i] = bucket_of<KIND>(key[i], bp);  // searches interleave
#pragma unroll
      for (int i = 0; i < (int)ITEMS; ++i) {
        const uint32_t b = bk[i];
        if constexpr (KIND == kIdentity) derr |= key_domain_error<KIND>(key[i], bp);
        slot[i] = atomicAdd(brow + (b >> 1), 1u << ((b & 1u) << 4));
        slot[i] = (slot[i] >> ((b & 1u) << 4)) & 0xFFFFu;
      }
#pragma unroll
      for (int i = 0; i < (int)ITEMS; ++i) place(s_stage, slot[i], key[i], PAIRS ? val[i] : 0u);
    } else {
#pragma unroll
      for (int i = 0; i < (int)ITEMS; ++i) {
        if (wbase + (uint32_t)i * 32u >= tn) break;  // warp-uniform: past the tail
        const bool valid = wbase + (uint32_t)i * 32u + lane < tn;
        const uint32_t b = bucket_of<KIND>(key[i], bp);
        if constexpr (KIND == kIdentity) derr |= valid && key_domain_error<KIND>(key[i], bp);
        if (valid) {
          const uint32_t sh = (b & 1u) << 4;
          const uint32_t slot = (atomicAdd(brow + (b >> 1), 1u << sh) >> sh) & 0xFFFFu;
          place(s_stage, slot, key[i], PAIRS ? val[i] : 0u);
        }
      }
    }
    if constexpr (KIND == kIdentity) {
      if (__any_sync(0xFFFFFFFFu, derr) && lane == 0) atomicOr(a.hdr, 1u);
    }
    if (k + 1 < nt) {
      load_tile(t + 1, k + 1);
      if (warp == W - 1) find_hot(t + 1, k + 1);
    }
    __syncthreads();
    // ---- refill the stage of tile t-1 with tile t+2: every warp finished tile
    // t-1's scatter before this barrier, so the copy starts a whole scatter
    // earlier than after this tile's
    if (tid == kProducer) {
      fence_proxy_async_smem();
      issue(t + 2, (k + 2) % kStages);
      prefetch(t + 2 + kPrefetch, true);
    }

    // ---- coalesced scatter of tile t: slot s of bucket b -> tab[b] + s, in
    // chunks of 4 slots per thread (measured: 4 beats 8 by 1.5-2 %, as in KO)
    {
      const uint32_t s0 = wbase + lane;
      constexpr uint32_t CH = 4;
#pragma unroll
      for (uint32_t c = 0; c < ITEMS; c += CH) {
        uint32_t kk[CH], vv[PAIRS ? CH : 1], pos[CH];
#pragma unroll
        for (uint32_t i = 0; i < CH; ++i) {
          if constexpr (PAIRS) {
            const uint2 kv = reinterpret_cast<const uint2 *>(s_stage)[s0 + 32 * (c + i)];
            kk[i] = kv.x;
            vv[i] = kv.y;
          } else {
            kk[i] = s_stage[s0 + 32 * (c + i)];
          }
        }
#pragma unroll
        for (uint32_t i = 0; i < CH; ++i) pos[i] = tab[bucket_of<KIND>(kk[i], bp)] + s0 + 32 * (c + i);
        if (a.npeers) {  // sharded: into the owning rank's window (KP)
#pragma unroll
          for (uint32_t i = 0; i < CH; ++i)
            if (s0 + 32 * (c + i) < tn) kp_store<PAIRS>(a, s_ps, pos[i], kk[i], PAIRS ? vv[i] : 0u);
        } else if (tn == T) {  // full tile: no per-element predicates
          uint32_t *__restrict__ ko = a.keys_out;
#pragma unroll
          for (uint32_t i = 0; i < CH; ++i) ko[pos[i]] = kk[i];
          if constexpr (PAIRS) {
            uint32_t *__restrict__ vo = a.vals_out;
#pragma unroll
            for (uint32_t i = 0; i < CH; ++i) vo[pos[i]] = vv[i];
          }
        } else {
#pragma unroll
          for (uint32_t i = 0; i < CH; ++i)
            if (s0 + 32 * (c + i) < tn) {
              a.keys_out[pos[i]] = kk[i];
              if constexpr (PAIRS) a.vals_out[pos[i]] = vv[i];
            }
        }
      }
    }
  }
}

}  // namespace ms
