// ms_hist.cuh -- device-wide histogram (Sec.7.3 "GPU Histogram"):
// the multisplit's prescan with the per-subproblem histograms summed into one
// global histogram instead of stored for a scan.  As the paper chose (option
// 2): each CTA (a contiguous range of samples, one per SM slot)
// counts into warp-private shared-memory rows (the warp-level privatization
// of P:1941-1943, here with shared-memory increments, measured cheapest on
// B200 for the multisplit prescan) and adds its m totals to the global
// histogram with one atomicAdd per bucket.
//
//   Even: b = floor((x - s_0) / Delta), Delta = (s_m - s_0) / m,
//                   binary32 round-to-nearest (reading R25), a
//                   quotient of m clamped to m-1, x outside [s_0, s_m) or NaN
//                   not counted (reading R26).
//   Range: splitters s_0 < ... < s_m staged in shared memory (P:1960-
//                   1962); b = upper_bound(s, x) - 1.  A cell table over
//                   [s_0, s_m) (1024 cells, cell(x) = floor((x - s_0) * inv),
//                   monotone in x) gives the splitters inside x's cell, so a
//                   sample costs one table load and at most two compares; a
//                   crowded cell takes the branch-free binary search.
#pragma once
#include "ms_device.cuh"

namespace ms {

// POW2 (Even, Delta a power of two): x / Delta and x * (1 / Delta) are the same
// correctly rounded binary32 value, so the division becomes a multiply.
constexpr uint32_t kHistCells = 1024;

// the Range cell of v (v in [s_0, s_m)): monotone non-decreasing in v, so a
// splitter in a lower cell is < v and one in a higher cell is > v
__device__ __forceinline__ uint32_t hist_cell(float v, float s0, float inv) {
  const float q = __fmul_rn(__fsub_rn(v, s0), inv);
  return q < (float)(kHistCells - 1) ? (uint32_t)q : kHistCells - 1;  // q >= 0
}

// crowded cell: the branch-free binary search (out of line: the common path
// stays free of its predicated steps)
__device__ __noinline__ uint32_t hist_range_search(float v, uint32_t m, const float *spl) {
  uint32_t j = 0;  // largest j with spl[j] <= v (spl[0] <= v < spl[m])
#pragma unroll
  for (uint32_t step = 128; step >= 1; step >>= 1)
    if (j + step < m && spl[j + step] <= v) j += step;
  return j;
}

template <bool RANGE, bool POW2 = false>
__device__ __forceinline__ void hist_sample(float v, uint32_t m, float lower, float upper,
                                            float delta, const float *spl, uint32_t *row,
                                            const uint32_t *cell = nullptr) {
  uint32_t b;
  if constexpr (RANGE) {
    if (!(v >= lower && v < upper)) return;  // Range: lower = s_0, upper = s_m (registers)
    // cell c = [A | B << 16]: the interior splitters s_{A+1} .. s_B lie in c
    const uint32_t x = cell ? cell[hist_cell(v, lower, delta)] : 0xFFFF0000u;
    const uint32_t j = x & 0xFFFFu, e = x >> 16;
    if (e - j > 2u) {
      b = hist_range_search(v, m, spl);
    } else {
      b = j;
      if (j < e && spl[j + 1] <= v) {
        b = j + 1u;
        if (j + 1u < e && spl[j + 2] <= v) b = j + 2u;
      }
    }
  } else {
    if (!(v >= lower && v < upper)) return;
    const float q = POW2 ? __fmul_rn(__fsub_rn(v, lower), delta) : __fdiv_rn(__fsub_rn(v, lower), delta);
    b = (uint32_t)floorf(q);
    b = b < m - 1 ? b : m - 1;
  }
  atomicAdd(row + b, 1u);
}

template <bool RANGE, bool POW2>
__global__ void __launch_bounds__(kThreads, 2)
    kh_histogram(const float *__restrict__ x, uint32_t n, uint32_t elems_per_cta, uint32_t m,
                 float lower, float upper, float delta, const float *__restrict__ splitters,
                 uint32_t *__restrict__ counts) {
  extern __shared__ uint32_t hg_smem[];  // cnt[kWarps][m] | splitters[m+1] | (Range) cells
  uint32_t *cnt = hg_smem;
  float *spl = reinterpret_cast<float *>(hg_smem + kWarps * m);
  uint32_t *cell = hg_smem + kWarps * m + m + 1;
  const uint32_t tid = threadIdx.x;
  for (uint32_t i = tid; i < kWarps * m; i += kThreads) cnt[i] = 0u;
  if constexpr (RANGE)
    for (uint32_t i = tid; i <= m; i += kThreads) spl[i] = __ldg(splitters + i);
  __syncthreads();
  if constexpr (RANGE) {
    // delta becomes inv = cells / (s_m - s_0) (a finite positive span; else no
    // table: every sample takes the search); A_c = #{interior s_j : cell(s_j) < c}
    // (a lower bound over the sorted splitters: cell() is monotone)
    lower = spl[0];  // the range ends, kept in registers
    upper = spl[m];
    const float span = __fsub_rn(upper, lower);
    if (!(span > 0.f && span <= 3.402823466e38f)) cell = nullptr;
    delta = __fdiv_rn((float)kHistCells, span);
    for (uint32_t c = tid; cell && c < kHistCells; c += kThreads) {
      uint32_t a = 0, bb = 0;
#pragma unroll
      for (int k = 7; k >= 0; --k) {
        const uint32_t ta = a + (1u << k), tb = bb + (1u << k);
        if (ta < m && hist_cell(spl[ta], spl[0], delta) < c) a = ta;
        if (tb < m && hist_cell(spl[tb], spl[0], delta) <= c) bb = tb;
      }
      cell[c] = a | (bb << 16);
    }
    __syncthreads();
  }
  uint32_t *row = cnt + (tid >> 5) * m;
  const uint32_t lo = blockIdx.x * elems_per_cta;
  const uint32_t hi = (uint32_t)min((uint64_t)n, (uint64_t)lo + elems_per_cta);
  uint32_t i = lo;
  if ((reinterpret_cast<uintptr_t>(x + lo) & 15u) == 0) {
    const uint4 *v = reinterpret_cast<const uint4 *>(x + lo);
    const uint32_t nv = (hi - lo) >> 2;
    uint32_t j = tid;
    for (; j + 7u * kThreads < nv; j += 8u * kThreads) {  // 8 x 16 B in flight per thread
      uint4 q[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) q[u] = ldg_stream_v4(v + j + (uint32_t)u * kThreads);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        hist_sample<RANGE, POW2>(__uint_as_float(q[u].x), m, lower, upper, delta, spl, row, cell);
        hist_sample<RANGE, POW2>(__uint_as_float(q[u].y), m, lower, upper, delta, spl, row, cell);
        hist_sample<RANGE, POW2>(__uint_as_float(q[u].z), m, lower, upper, delta, spl, row, cell);
        hist_sample<RANGE, POW2>(__uint_as_float(q[u].w), m, lower, upper, delta, spl, row, cell);
      }
    }
    for (; j < nv; j += kThreads) {
      const uint4 q = ldg_stream_v4(v + j);
      hist_sample<RANGE, POW2>(__uint_as_float(q.x), m, lower, upper, delta, spl, row, cell);
      hist_sample<RANGE, POW2>(__uint_as_float(q.y), m, lower, upper, delta, spl, row, cell);
      hist_sample<RANGE, POW2>(__uint_as_float(q.z), m, lower, upper, delta, spl, row, cell);
      hist_sample<RANGE, POW2>(__uint_as_float(q.w), m, lower, upper, delta, spl, row, cell);
    }
    i = lo + (nv << 2);
  }
  for (i += tid; i < hi; i += kThreads) hist_sample<RANGE, POW2>(__ldg(x + i), m, lower, upper, delta, spl, row, cell);
  __syncthreads();
  for (uint32_t b = tid; b < m; b += kThreads) {
    uint32_t s = 0;
#pragma unroll 4
    for (int w = 0; w < kWarps; ++w) s += cnt[w * m + b];
    if (s) atomicAdd(counts + b, s);
  }
}

}  // namespace ms
