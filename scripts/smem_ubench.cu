// smem_ubench.cu -- shared-memory operation costs on B200 for the postscan
// design (not part of the product): cycles per warp-instruction per SM for
// bucket-indexed atomics / loads / stores with m buckets per warp row, at
// full occupancy.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// Each CTA: NW warps; each warp owns a row of m words; every lane draws a
// random bucket per iteration (hash), does OP, accumulates a checksum.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int OP>
__global__ void kbench(uint32_t *out, int iters, int m, int skew) {
  extern __shared__ uint32_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t *row = sm + warp * 512;
  for (int j = lane; j < 512; j += 32) row[j] = j;
  __syncwarp();
  uint32_t acc = 0, h = hsh(threadIdx.x * 977 + blockIdx.x);
  unsigned long long *row64 = reinterpret_cast<unsigned long long *>(sm) + warp * 256;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      h = h * 1664525u + 1013904223u;
      uint32_t b = (h >> 8) & (m - 1);
      if (skew && (h & 15) < 14) b = 7;
      if constexpr (OP == 0) acc += atomicAdd(row + b, 1u);          // ATOMS.ADD with return
      else if constexpr (OP == 1) atomicAdd(row + b, 1u);            // RED (no return)
      else if constexpr (OP == 2) acc += row[b];                      // LDS random
      else if constexpr (OP == 3) row[b] = h;                         // STS random
      else if constexpr (OP == 4) acc += (uint32_t)row64[b & 255];    // LDS.64 random
      else if constexpr (OP == 5) acc += __match_any_sync(0xffffffffu, b);  // MATCH.ANY
      else if constexpr (OP == 6) acc += row[(lane + u * 32) & 511];  // LDS conflict-free
      else if constexpr (OP == 7) acc += (uint32_t)atomicAdd(row64 + (b & 255), 0x100000001ull);  // ATOMS.64
      else if constexpr (OP == 8) acc += __ballot_sync(0xffffffffu, b & 1);  // ballot
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
  if (OP == 3 && lane == 0) out[1 + blockIdx.x] = row[lane];
}

template <int OP>
void run(const char *name, int m, int nw, int ctas_per_sm, int skew) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t *out;
  cudaMalloc(&out, 4 * (1 + sms * 8));
  size_t smem = (size_t)nw * 512 * 4;
  cudaFuncSetAttribute(kbench<OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  const int iters = 256;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kbench<OP><<<sms * ctas_per_sm, nw * 32, smem>>>(out, 8, m, skew);
  cudaEventRecord(a);
  kbench<OP><<<sms * ctas_per_sm, nw * 32, smem>>>(out, iters, m, skew);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double cycles = ms * 1e-3 * clk * 1e3;  // at max clock
  double winst_per_sm = (double)ctas_per_sm * nw * iters * 16;
  printf("%-10s m=%3d warps/SM=%3d skew=%d : %.2f cycles per warp-op per SM (%.3f ms) %s\n", name, m,
         nw * ctas_per_sm, skew, cycles / winst_per_sm, ms, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  for (int m : {32, 256}) {
    for (int w : {16, 32}) {
      run<0>("atom_ret", m, w / 2, 2, 0);
      run<1>("red", m, w / 2, 2, 0);
      run<2>("lds_rand", m, w / 2, 2, 0);
      run<3>("sts_rand", m, w / 2, 2, 0);
      run<4>("lds64", m, w / 2, 2, 0);
      run<7>("atom64", m, w / 2, 2, 0);
      run<5>("match", m, w / 2, 2, 0);
    }
  }
  run<6>("lds_cf", 256, 16, 2, 0);
  run<8>("ballot", 256, 16, 2, 0);
  run<0>("atom_ret", 256, 16, 2, 1);
  run<1>("red", 256, 16, 2, 1);
  run<5>("match", 256, 16, 2, 1);
  return 0;
}
