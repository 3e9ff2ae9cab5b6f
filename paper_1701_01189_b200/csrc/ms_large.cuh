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

namespace ms {

template <int KIND>
__global__ void __launch_bounds__(256)
    k_bucket_ids(const uint32_t *__restrict__ keys, uint32_t n, BucketParams bp, int payload_index,
                 uint32_t *__restrict__ b, uint32_t *__restrict__ p, uint32_t *__restrict__ hdr) {
  bool derr = false;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t u = __ldg(keys + i);
    derr |= key_domain_error<KIND>(u, bp);
    b[i] = bucket_of<KIND>(u, bp);  // SPLITTERS: the table stays in global memory (m-1 > smem)
    p[i] = payload_index ? i : u;
  }
  if (KIND == kIdentity && __any_sync(0xFFFFFFFFu, derr) && (threadIdx.x & 31u) == 0) atomicOr(hdr, 1u);
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
