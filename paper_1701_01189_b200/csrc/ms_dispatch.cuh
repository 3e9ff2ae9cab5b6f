// ms_dispatch.cuh -- host-side launchers that map runtime (strategy, log2 m,
// pairs) onto the kernel template instantiations.  Each bucket kind is
// instantiated in its own translation unit (ms_inst_*.cu) to keep nvcc
// parallel.
#pragma once
#include "ms_kernels.cuh"

namespace ms {

template <int KIND>
cudaError_t launch_prescan(int strat, int logm, const uint32_t *keys, uint32_t n,
                           const BucketParams &bp, uint32_t *H, unsigned long long *zs,
                           uint32_t zw, uint32_t *hdr, cudaStream_t s);

template <int KIND>
cudaError_t launch_postscan(int strat, int logm, bool pairs, const KsArgs &a,
                            const BucketParams &bp, uint32_t grid, cudaStream_t s);

#define MS_LOGM_SWITCH(logm, BODY)          \
  switch (logm) {                           \
    case 1: { constexpr int L_ = 1; BODY; } break; \
    case 2: { constexpr int L_ = 2; BODY; } break; \
    case 3: { constexpr int L_ = 3; BODY; } break; \
    case 4: { constexpr int L_ = 4; BODY; } break; \
    case 5: { constexpr int L_ = 5; BODY; } break; \
    case 6: { constexpr int L_ = 6; BODY; } break; \
    case 7: { constexpr int L_ = 7; BODY; } break; \
    default: { constexpr int L_ = 8; BODY; } break; \
  }

template <int KIND, int STRAT, int LOGM>
static cudaError_t kh_go(const uint32_t *keys, uint32_t n, const BucketParams &bp, uint32_t *H,
                         unsigned long long *zs, uint32_t zw, uint32_t *hdr, cudaStream_t s) {
  const uint32_t grid = (n + kTile - 1) / kTile;
  const size_t smem = (STRAT == kCount1) ? 0 : (size_t)kWarps * bp.m * 4u;
  kh_prescan<KIND, STRAT, LOGM><<<grid, kThreads, smem, s>>>(keys, n, bp, H, zs, zw, hdr);
  return cudaGetLastError();
}

template <int KIND, bool PAIRS, int STRAT, int LOGM>
static cudaError_t ks_go(const KsArgs &a, const BucketParams &bp, uint32_t grid, cudaStream_t s) {
  const size_t smem = ks_smem_bytes(bp.m, PAIRS);
  auto kern = ks_postscan<KIND, PAIRS, STRAT, LOGM>;
  static thread_local bool configured = false;  // per instantiation
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)ks_smem_bytes(kMaxBuckets, true));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  kern<<<grid, kThreads, smem, s>>>(a, bp);
  return cudaGetLastError();
}

template <int KIND>
cudaError_t launch_prescan(int strat, int logm, const uint32_t *keys, uint32_t n,
                           const BucketParams &bp, uint32_t *H, unsigned long long *zs,
                           uint32_t zw, uint32_t *hdr, cudaStream_t s) {
  switch (strat) {
    case kCount1: return kh_go<KIND, kCount1, 0>(keys, n, bp, H, zs, zw, hdr, s);
    case kMatch: return kh_go<KIND, kMatch, 0>(keys, n, bp, H, zs, zw, hdr, s);
    case kAtomic: return kh_go<KIND, kAtomic, 0>(keys, n, bp, H, zs, zw, hdr, s);
    default: MS_LOGM_SWITCH(logm, return (kh_go<KIND, kPeers, L_>(keys, n, bp, H, zs, zw, hdr, s)));
  }
  return cudaErrorInvalidValue;
}

template <int KIND>
cudaError_t launch_postscan(int strat, int logm, bool pairs, const KsArgs &a,
                            const BucketParams &bp, uint32_t grid, cudaStream_t s) {
  if (pairs) {
    switch (strat) {
      case kCount1: return ks_go<KIND, true, kCount1, 0>(a, bp, grid, s);
      case kMatch: return ks_go<KIND, true, kMatch, 0>(a, bp, grid, s);
      default: MS_LOGM_SWITCH(logm, return (ks_go<KIND, true, kPeers, L_>(a, bp, grid, s)));
    }
  } else {
    switch (strat) {
      case kCount1: return ks_go<KIND, false, kCount1, 0>(a, bp, grid, s);
      case kMatch: return ks_go<KIND, false, kMatch, 0>(a, bp, grid, s);
      default: MS_LOGM_SWITCH(logm, return (ks_go<KIND, false, kPeers, L_>(a, bp, grid, s)));
    }
  }
  return cudaErrorInvalidValue;
}

#define MS_INSTANTIATE_KIND(KIND)                                                              \
  template cudaError_t launch_prescan<KIND>(int, int, const uint32_t *, uint32_t,             \
                                            const BucketParams &, uint32_t *,                   \
                                            unsigned long long *, uint32_t, uint32_t *,         \
                                            cudaStream_t);                                      \
  template cudaError_t launch_postscan<KIND>(int, int, bool, const KsArgs &,                  \
                                             const BucketParams &, uint32_t, cudaStream_t);

}  // namespace ms
