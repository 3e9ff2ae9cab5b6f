// ms_scan.cuh -- KG, the global stage (Alg.1), plus
// the small helper kernels of the stage API.  Included by ms_capi.cu only.
#pragma once
#include "ms_kernels.cuh"

namespace ms {

// Status word of the decoupled look-back: high 32 bits = flag, low = value.
constexpr unsigned long long kFlagAggregate = 1ull << 32;
constexpr unsigned long long kFlagInclusive = 2ull << 32;

// ============================================================================
// KG: decoupled look-back scan over the tile-major H.  CTA (ticket c) owns
// tiles [c*C, (c+1)*C) x all m buckets.  Threads are (group g, bucket j)
// pairs; each group scans a contiguous sub-range of the chunk's tiles for its
// bucket.  Per bucket, the chunk aggregate is published, then the exclusive
// prefix is found by looking back over predecessors (inclusive prefixes end
// the walk).  Writes G[l][j] = sum_{l'<l} h_{j,l'} (may alias H).  The last
// chunk turns the column totals into the bucket bases (first term of Eq.2)
// base[j] = sum_{j'<j} total_{j'}, base[m] = n_total.
// ============================================================================
constexpr int kScanThreads = 256;

__global__ void __launch_bounds__(kScanThreads)
    kg_scan(const uint32_t *H, uint32_t *G, uint32_t L, uint32_t m, uint32_t C,
            uint32_t nchunks, unsigned long long *__restrict__ status,
            uint32_t *__restrict__ ticket, uint32_t *__restrict__ base,
            uint32_t *__restrict__ bucket_offsets) {
  __shared__ uint32_t s_part[kScanThreads];  // [group][bucket] partial sums -> prefixes
  __shared__ uint32_t s_excl[kMaxBuckets];
  __shared__ uint32_t s_chunk;
  __shared__ uint32_t s_scan[kMaxBuckets];
  const uint32_t tid = threadIdx.x;
  if (tid == 0) s_chunk = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t c = s_chunk;
  const uint32_t P = kScanThreads / m;       // groups (>= 1)
  const uint32_t g = tid / m, j = tid % m;
  const uint32_t c0 = c * C, c1 = min(L, c0 + C);
  const uint32_t S = (C + P - 1) / P;        // tiles per group
  const bool active = g < P;
  const uint32_t l0 = min(c1, c0 + g * S), l1 = min(c1, l0 + S);

  uint32_t sum = 0;
  if (active)
#pragma unroll 8
    for (uint32_t l = l0; l < l1; ++l) sum += H[(size_t)l * m + j];
  if (active) s_part[g * m + j] = sum;
  __syncthreads();

  if (tid < m) {
    uint32_t run = 0;
    for (uint32_t gg = 0; gg < P; ++gg) {
      const uint32_t v = s_part[gg * m + tid];
      s_part[gg * m + tid] = run;
      run += v;
    }
    const uint32_t agg = run;
    unsigned long long *my = status + (size_t)c * m + tid;
    if (c == 0) {
      st_release_u64(my, kFlagInclusive | agg);
      s_excl[tid] = 0;
    } else {
      st_release_u64(my, kFlagAggregate | agg);
      uint32_t excl = 0;
      for (int p = (int)c - 1; p >= 0; --p) {
        unsigned long long w;
        do {
          w = ld_acquire_u64(status + (size_t)p * m + tid);
        } while ((w >> 32) == 0ull);
        excl += (uint32_t)w;
        if ((w >> 32) == (kFlagInclusive >> 32)) break;
      }
      st_release_u64(my, kFlagInclusive | (unsigned long long)(excl + agg));
      s_excl[tid] = excl;
    }
    s_scan[tid] = s_excl[tid] + agg;  // inclusive column total through this chunk
  }
  __syncthreads();

  if (active) {
    uint32_t run = s_excl[j] + s_part[g * m + j];
    for (uint32_t l = l0; l < l1; ++l) {
      const uint32_t h = H[(size_t)l * m + j];
      G[(size_t)l * m + j] = run;
      run += h;
    }
  }

  if (c == nchunks - 1) {  // totals are complete: bucket bases (block scan over j)
    if (tid == 0) {
      uint32_t run = 0;
      for (uint32_t jj = 0; jj < m; ++jj) {
        const uint32_t t = s_scan[jj];
        base[jj] = run;
        if (bucket_offsets) bucket_offsets[jj] = run;
        run += t;
      }
      base[m] = run;
      if (bucket_offsets) bucket_offsets[m] = run;
    }
  }
}

// Stage-API epilogue: G_full[l][j] = G[l][j] + base[j].
__global__ void kg_add_base(uint32_t *G, uint64_t total, uint32_t m, const uint32_t *base) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x)
    G[i] += base[i % m];
}

__global__ void zero_words_kernel(unsigned long long *p, uint32_t words, uint32_t *hdr) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < words; i += gridDim.x * blockDim.x)
    p[i] = 0ull;
  if (blockIdx.x == 0 && threadIdx.x < 2) hdr[threadIdx.x] = 0u;
}

}  // namespace ms
