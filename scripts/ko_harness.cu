// Standalone harness for the one-pass kernels (csrc/ms_onesweep.cuh): times
// KOH and KO on a uniform 8-bit-digit multisplit, checks the result against a
// host stable counting sort, and (built with -DMS_KO_TIMING) prints the
// per-phase cycles of KO's compute warps.  Development tool, not the product:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        -I paper_1701_01189_b200/csrc scripts/ko_harness.cu -o /tmp/koh
//   /tmp/koh [log2 n] [pairs] [reps] [max grid] [n]
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ms_onesweep.cuh"

using namespace ms;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1); } } while (0)

__global__ void fill(uint32_t *k, uint32_t *v, uint32_t n, uint32_t seed) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint64_t z = (uint64_t)i * 0x9E3779B97F4A7C15ull + seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    k[i] = (uint32_t)((z ^ (z >> 31)) >> 32);
    if (v) v[i] = i;
  }
}

template <bool PAIRS>
int run(uint32_t n, int reps, uint32_t max_grid) {
  uint32_t *k, *v = nullptr, *ko, *vo = nullptr, *ws;
  const uint32_t T = ko_tile(PAIRS), L = (n + T - 1) / T;
  const uint32_t Lpad = (L + 7u) & ~7u;
  const size_t wsw = 256 + 1024 + 64 + (size_t)Lpad * 256;
  CK(cudaMalloc(&k, n * 4ull));
  CK(cudaMalloc(&ko, n * 4ull));
  if (PAIRS) {
    CK(cudaMalloc(&v, n * 4ull));
    CK(cudaMalloc(&vo, n * 4ull));
  }
  CK(cudaMalloc(&ws, wsw * 4));
  fill<<<1024, 256>>>(k, v, n, 12345);
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  BucketParams bp{};
  bp.m = 256;
  bp.m1 = 255;
  bp.shift = 0;
  bp.mask = 255;
  KoHistArgs h{};
  h.keys = k;
  h.n = n;
  h.npass = 1;
  h.shift[0] = 0;
  h.mask[0] = 255;
  h.nbins = 256;
  h.gh = ws + 256;
  h.hdr = ws;
  KoArgs a{};
  a.keys_in = k;
  a.vals_in = v;
  a.keys_out = ko;
  a.vals_out = vo;
  a.n = n;
  a.num_tiles = L;
  a.gh = ws + 256;
  a.ticket = ws + 256 + 1024;
  a.status = ws + 256 + 1024 + 64;
  a.hdr = ws;
  a.use_tma = 1;
  auto kh = ko_hist<kRadix, false>;
  auto kh4 = ko_hist<kRadix, true>;
  auto kk = ko_onesweep<kRadix, PAIRS>;
  CK(cudaFuncSetAttribute(kh, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 * 32 * 4));
  CK(cudaFuncSetAttribute(kh4, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 * 32 * 4));
  CK(cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ko_smem_bytes(PAIRS)));
  cudaEvent_t e0, e1, e2;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventCreate(&e2));
  {  // the 4 x 8-bit sort's histogram: generic vs byte kernel
    KoHistArgs h4 = h;
    uint32_t *gh4;
    CK(cudaMalloc(&gh4, 1024 * 4));
    h4.npass = 4;
    h4.nbins = 1024;
    h4.gh = gh4;
    for (int p = 0; p < 4; ++p) {
      h4.shift[p] = 8 * p;
      h4.mask[p] = 255;
      h4.bin0[p] = 256 * p;
    }
    std::vector<uint32_t> r0(1024), r1(1024);
    float tg = 0, tb = 0;
    for (int r = 0; r < 4; ++r) {
      CK(cudaMemset(gh4, 0, 4096));
      CK(cudaEventRecord(e0));
      kh<<<sms, 1024, 1024 * 32 * 4>>>(h4, bp);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaMemcpy(r0.data(), gh4, 4096, cudaMemcpyDeviceToHost));
      CK(cudaMemset(gh4, 0, 4096));
      CK(cudaEventRecord(e1));
      kh4<<<sms, 1024, 1024 * 32 * 4>>>(h4, bp);
      CK(cudaEventRecord(e2));
      CK(cudaEventSynchronize(e2));
      CK(cudaMemcpy(r1.data(), gh4, 4096, cudaMemcpyDeviceToHost));
      float x, y;
      CK(cudaEventElapsedTime(&x, e0, e1));
      CK(cudaEventElapsedTime(&y, e1, e2));
      if (r) {
        tg += x;
        tb += y;
      }
    }
    printf("KOH 4 x 8-bit: generic %.1f us, byte kernel %.1f us, %s\n", tg / 3 * 1e3, tb / 3 * 1e3,
           r0 == r1 ? "equal counts" : "COUNTS DIFFER");
    CK(cudaFree(gh4));
  }
  uint32_t grid = L < (uint32_t)sms ? L : (uint32_t)sms;
  if (max_grid && grid > max_grid) grid = max_grid;  // several tiles per CTA at small n (sanitizers)
  float th = 0, tk = 0;
#ifdef MS_KO_TIMING
  {
    static unsigned long long zero[1024][2][kKoPhases] = {};
    CK(cudaMemcpyToSymbol(ko_timing, zero, sizeof(zero)));
    unsigned long long z4[4] = {0, 0, 0, 0};
    CK(cudaMemcpyToSymbol(ko_lbstat, z4, sizeof(z4)));
  }
#endif
  for (int r = 0; r < reps + 1; ++r) {
    CK(cudaMemsetAsync(ws, 0, wsw * 4));
    CK(cudaEventRecord(e0));
    kh<<<sms, 1024, 256 * 32 * 4>>>(h, bp);
    CK(cudaEventRecord(e1));
    kk<<<grid, ko_threads(PAIRS), ko_smem_bytes(PAIRS)>>>(a, bp);
    CK(cudaEventRecord(e2));
    CK(cudaGetLastError());
    CK(cudaEventSynchronize(e2));
    float x, y;
    CK(cudaEventElapsedTime(&x, e0, e1));
    CK(cudaEventElapsedTime(&y, e1, e2));
    if (r > 0) {
      th += x;
      tk += y;
    }
  }
  th /= reps;
  tk /= reps;
  const double bytes = (double)n * (PAIRS ? 16 : 8);
  printf("n=%u pairs=%d T=%u L=%u grid=%u: KOH %.1f us (%.0f GB/s)  KO %.1f us (%.0f GB/s, %.3f of 6535)\n", n,
         (int)PAIRS, T, L, grid, th * 1e3, n * 4.0 / th / 1e6, tk * 1e3, bytes / tk / 1e6, bytes / tk / 1e6 / 6535);
  // check: stable counting sort by the low 8 bits
  std::vector<uint32_t> hk(n), hko(n), hv(PAIRS ? n : 0), hvo(PAIRS ? n : 0);
  CK(cudaMemcpy(hk.data(), k, n * 4ull, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hko.data(), ko, n * 4ull, cudaMemcpyDeviceToHost));
  if (PAIRS) CK(cudaMemcpy(hvo.data(), vo, n * 4ull, cudaMemcpyDeviceToHost));
  std::vector<uint32_t> off(257, 0);
  for (uint32_t i = 0; i < n; ++i) off[(hk[i] & 255) + 1]++;
  for (int b = 0; b < 256; ++b) off[b + 1] += off[b];
  size_t bad = 0;
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t p = off[hk[i] & 255]++;
    if (hko[p] != hk[i] || (PAIRS && hvo[p] != i)) ++bad;
  }
  printf("  check: %zu mismatches\n", bad);
#ifdef MS_KO_TIMING
  static unsigned long long tm[1024][2][kKoPhases];
  CK(cudaMemcpyFromSymbol(tm, ko_timing, sizeof(tm)));
  const char *names[kKoPhases] = {"tma-wait", "load+rank", "B1", "scan+B2", "scatter", "B3", "place", "lookback"};
  for (int w = 0; w < 2; ++w) {
    printf("  warp %s cycles per tile:", w ? "W-1" : "0  ");
    double tot = 0;
    for (int q = 0; q < kKoPhases; ++q) {
      unsigned long long s = 0;
      for (uint32_t b = 0; b < grid; ++b) s += tm[b][w][q];
      const double c = (double)s / (reps + 1) / L;
      tot += c;
      printf(" %s %.0f", names[q], c);
    }
    printf(" | total %.0f\n", tot);
  }
  unsigned long long lb[4];
  CK(cudaMemcpyFromSymbol(lb, ko_lbstat, sizeof(lb)));
  const double nt = (double)L * (reps + 1);
  printf("  look-back per tile (thread 0): windows %.2f first-window spins %.2f\n", lb[0] / nt, lb[1] / nt);
#endif
  return bad ? 1 : 0;
}

int main(int argc, char **argv) {
  const int lg = argc > 1 ? atoi(argv[1]) : 25;
  const int pairs = argc > 2 ? atoi(argv[2]) : 0;
  const int reps = argc > 3 ? atoi(argv[3]) : 10;
  const uint32_t max_grid = argc > 4 ? (uint32_t)atoi(argv[4]) : 0u;
  const uint32_t n = argc > 5 ? (uint32_t)atoi(argv[5]) : (1u << lg);  // explicit n (ragged tails)
  return pairs ? run<true>(n, reps, max_grid) : run<false>(n, reps, max_grid);
}
