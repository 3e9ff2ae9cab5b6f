// gen.cu -- device copy of the counter-based input generator of gen/inputs.py
// (same recipe, byte-identical output; checked by tests/test_gpu_gen.py).
// It holds no multisplit arithmetic.  Built into gen/libmsgen.so.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t h64(uint64_t seed, uint64_t stream, uint64_t i) {
  return mix64(seed ^ (stream * 0xD1B54A32D192ED03ull) ^ i);
}
__device__ __forceinline__ uint32_t rnd32(uint64_t seed, uint64_t stream, uint64_t i) {
  return (uint32_t)(h64(seed, stream, i) >> 32);
}
__device__ __forceinline__ uint32_t below(uint32_t x, uint64_t w) {
  return (uint32_t)(((uint64_t)x * w) >> 32);
}

struct GenArgs {
  uint32_t *out;
  uint64_t n, seed, alpha32;
  uint32_t kind, m, delta, shift, bits, dist;
};

__global__ void gen_keys_kernel(GenArgs a) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < a.n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (a.dist == 0 && a.kind != 0) {  // uniform keys
      a.out[i] = rnd32(a.seed, 0, i);
      continue;
    }
    uint32_t b;
    if (a.dist == 0) {
      b = below(rnd32(a.seed, 1, i), a.m);
    } else if (a.dist == 1) {
      const uint32_t hot = below(rnd32(a.seed, 2, 0), a.m);
      b = ((uint64_t)rnd32(a.seed, 3, i) < a.alpha32) ? below(rnd32(a.seed, 1, i), a.m) : hot;
    } else {
      int nbits = (int)a.m - 1;
      b = 0;
      for (int w = 0; w < 4 && nbits > 0; ++w) {
        const int take = nbits < 64 ? nbits : 64;
        const uint64_t mask = take == 64 ? ~0ull : ((1ull << take) - 1ull);
        b += __popcll(h64(a.seed, 4 + w, i) & mask);
        nbits -= take;
      }
    }
    uint32_t key;
    if (a.kind == 0) {
      key = b;
    } else if (a.kind == 2) {
      const uint32_t mask = ((1u << a.bits) - 1u) << a.shift;
      key = (rnd32(a.seed, 0, i) & ~mask) | (b << a.shift);
    } else {
      const uint64_t lo = (uint64_t)b * a.delta;
      uint64_t hi = lo + a.delta;
      if (hi > (1ull << 32)) hi = 1ull << 32;
      if (b == a.m - 1) hi = 1ull << 32;
      key = (uint32_t)(lo + below(rnd32(a.seed, 0, i), hi - lo));
    }
    a.out[i] = key;
  }
}

__global__ void gen_values_kernel(uint32_t *out, uint64_t n, uint64_t seed, int parity) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = parity ? (uint32_t)i : rnd32(seed, 8, i);
}

}  // namespace

extern "C" {

// dist: 0 uniform, 1 alpha-uniform skew (alpha32 = floor(alpha * 2^32)), 2 binomial B(m-1, 1/2)
int msgen_keys(uint32_t *out, uint64_t n, uint64_t seed, uint32_t kind, uint32_t m,
               uint32_t delta, uint32_t shift, uint32_t bits, uint32_t dist, uint64_t alpha32,
               void *stream) {
  if (n == 0) return 0;
  GenArgs a{out, n, seed, alpha32, kind, m, delta, shift, bits, dist};
  gen_keys_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(a);
  return (int)cudaGetLastError();
}

int msgen_values(uint32_t *out, uint64_t n, uint64_t seed, int parity, void *stream) {
  if (n == 0) return 0;
  gen_values_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(out, n, seed, parity);
  return (int)cudaGetLastError();
}

// L2 flush helper for the bench: overwrite `bytes` of scratch (> L2 size).
__global__ void flush_kernel(uint4 *p, uint64_t n16, uint32_t v) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16;
       i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(v, v, v, v);
}

int msgen_flush(void *scratch, uint64_t bytes, uint32_t v, void *stream) {
  flush_kernel<<<148 * 4, 512, 0, (cudaStream_t)stream>>>((uint4 *)scratch, bytes / 16, v);
  return (int)cudaGetLastError();
}

}  // extern "C"
