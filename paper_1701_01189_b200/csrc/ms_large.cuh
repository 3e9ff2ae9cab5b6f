// ms_large.cuh -- kernels of the m > 256 path (Sec.6.3 "Performance for more
// than 256 buckets").  The paper iterates multisplits over at most
// 256 (super-)buckets; here the iteration is LSD over the 8-bit digits of the
// bucket id itself, which works for every bucket identifier (not only for
// those that admit super-buckets):
//   KB  k_bucket_ids: b_i = f(u_i) and the payload p_i (the key, or the index i
//       for pairs) -- one read of the keys, two words written;
//   two stable multisplits of the (b, p) pairs with radix-digit buckets
//       (b & 255, then b >> 8): a stable sort by b, i.e. the stable multisplit;
//   KO  k_offsets_sorted: bucket_offsets from the sorted bucket ids;
//   KGA k_gather_pairs (pairs only): keys_out[j] = keys[p_j], vals_out[j] = vals[p_j].
#pragma once
#include "ms_device.cuh"
#include "ms_kernels.cuh"

namespace ms {

template <int KIND>
__global__ void __launch_bounds__(256)
    k_bucket_ids(const uint32_t *__restrict__ keys, uint32_t n, BucketParams bp, int payload_index,
                 uint32_t *__restrict__ b, uint32_t *__restrict__ p, uint32_t *__restrict__ hdr) {
  bool derr = false;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t u = __ldg(keys + i);
    derr |= key_domain_error<KIND>(u, bp);
    if constexpr (KIND == kSplitters)  // the table stays in global memory (up to 65535 entries)
      b[i] = splitter_bucket<16>(u, bp);
    else
      b[i] = bucket_of<KIND>(u, bp);
    p[i] = payload_index ? i : u;
  }
  if (KIND == kIdentity && __any_sync(0xFFFFFFFFu, derr) && (threadIdx.x & 31u) == 0) atomicOr(hdr, 1u);
}

// identity buckets with m > 256 run as radix passes over the keys: the
// key-domain check (u < m, reading R8) is this separate read
static __global__ void __launch_bounds__(256)
    k_domain_check(const uint32_t *__restrict__ keys, uint32_t n, uint32_t m, uint32_t *__restrict__ hdr) {
  bool bad = false;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    bad |= __ldg(keys + i) >= m;
  if (__any_sync(0xFFFFFFFFu, bad) && (threadIdx.x & 31u) == 0) atomicOr(hdr, 1u);
}

// src sorted by d(x) = (x >> shift) & mask: off[j] = first index with d >= j, off[m] = n.
static __global__ void __launch_bounds__(256)
    k_offsets_sorted(const uint32_t *__restrict__ src, uint32_t n, uint32_t shift, uint32_t mask,
                     uint32_t m, uint32_t *__restrict__ off) {
  for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t lo = i == 0 ? 0u : ((__ldg(src + i - 1) >> shift) & mask) + 1u;
    const uint32_t hi = i == n ? m : (__ldg(src + i) >> shift) & mask;
    for (uint32_t j = lo; j <= hi; ++j) off[j] = (uint32_t)i;
  }
}

static __global__ void __launch_bounds__(256)
    k_gather_pairs(const uint32_t *__restrict__ idx, uint32_t n, const uint32_t *__restrict__ keys,
                   const uint32_t *__restrict__ vals, uint32_t *__restrict__ keys_out,
                   uint32_t *__restrict__ vals_out) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const uint32_t i = __ldg(idx + j);
    keys_out[j] = __ldg(keys + i);
    vals_out[j] = __ldg(vals + i);
  }
}

}  // namespace ms

namespace ms {

// ============================================================================
// KT k_small: the whole multisplit of n <= 4096 elements in one CTA of 16
// warps, for the latency-bound regime (configs[0], n = 2^10; Multisplit-SSSP's
// small work lists).  Warp w owns elements [256 w, 256 w + 256) as 8
// windows in input order.  One pass: per-warp ranks by lane-ordered increments
// (reading R23; only on a device whose probe held), which also leave the
// (warp, bucket) counts; a column scan over the warps and a scan over the
// buckets (Eq.2 with the warps as subproblems); every element is then stored
// at base[b] + (earlier warps' count of b) + rank.  Three barriers, no TMA.
// ============================================================================
constexpr uint32_t kSmallMax = 4096;

template <int KIND, bool PAIRS>
__global__ void __launch_bounds__(kThreads) k_small(KfArgs a, BucketParams bp) {
  MS_STAGE_SPLITTERS3(bp, kMaxBuckets, false);
  constexpr uint32_t W = kWarps, PER = kSmallMax / W, ITEMS = PER / 32;
  __shared__ uint32_t cnt[W][kMaxBuckets];
  __shared__ uint32_t s_base[kMaxBuckets];
  __shared__ uint32_t s_wsum[W];
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u, m = bp.m;
  for (uint32_t i = tid; i < W * kMaxBuckets; i += blockDim.x) (&cnt[0][0])[i] = 0u;
  if (tid == 0) a.hdr[0] = 0u;  // the key-domain flag of this call (set after the barrier)
  __syncthreads();
  uint32_t key[ITEMS], b[ITEMS], r[ITEMS], val[PAIRS ? ITEMS : 1];
  bool derr = false;
#pragma unroll
  for (uint32_t i = 0; i < ITEMS; ++i) {
    const uint32_t e = warp * PER + 32u * i + lane;
    const bool valid = e < a.n;
    key[i] = valid ? __ldg(a.keys_in + e) : 0u;
    if constexpr (PAIRS) val[i] = valid ? __ldg(a.vals_in + e) : 0u;
    b[i] = bucket_of<KIND>(key[i], bp);
    if constexpr (KIND == kIdentity) derr |= valid && key_domain_error<KIND>(key[i], bp);
    r[i] = valid ? atomicAdd(&cnt[warp][b[i]], 1u) : 0u;
  }
  if constexpr (KIND == kIdentity) {
    if (__any_sync(0xFFFFFFFFu, derr) && lane == 0) atomicOr(a.hdr, 1u);
  }
  __syncthreads();
  // column scan over the warps (thread j < m owns bucket j), then the buckets
  uint32_t tot = 0;
  if (tid < m) {
#pragma unroll
    for (uint32_t w = 0; w < W; ++w) {
      const uint32_t c = cnt[w][tid];
      cnt[w][tid] = tot;
      tot += c;
    }
  }
  uint32_t incl = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= (uint32_t)o) incl += y;
  }
  if (lane == 31) s_wsum[warp] = incl;
  __syncthreads();
  if (tid < m) {
    uint32_t pre = 0;
    for (uint32_t w = 0; w < warp; ++w) pre += s_wsum[w];
    const uint32_t base = pre + incl - tot;
    s_base[tid] = base;
    if (a.bucket_offsets) {
      a.bucket_offsets[tid] = base;
      if (tid == m - 1) a.bucket_offsets[m] = base + tot;
    }
  }
  __syncthreads();
#pragma unroll
  for (uint32_t i = 0; i < ITEMS; ++i) {
    const uint32_t e = warp * PER + 32u * i + lane;
    if (e < a.n) {
      const uint32_t p = s_base[b[i]] + cnt[warp][b[i]] + r[i];
      a.keys_out[p] = key[i];
      if constexpr (PAIRS) a.vals_out[p] = val[i];
    }
  }
}

}  // namespace ms
