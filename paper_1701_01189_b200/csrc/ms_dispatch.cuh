// ms_dispatch.cuh -- host-side launchers mapping the runtime (bucket kind,
// m <= 2, pairs) onto kernel template instantiations.  Each bucket kind is
// instantiated in its own translation unit (ms_inst_*.cu) so nvcc runs them
// in parallel.
#pragma once
#include "ms_kernels.cuh"

namespace ms {

template <int KIND>
struct Launch {
  static cudaError_t range_hist(const uint32_t *keys, uint32_t n, uint32_t elems_per_cta,
                                uint32_t grid, const BucketParams &bp, uint32_t *R, uint32_t *hdr,
                                cudaStream_t s);
  static cudaError_t tile_hist(const uint32_t *keys, uint32_t n, uint32_t tile, uint32_t grid,
                               const BucketParams &bp, uint32_t *H, uint32_t *hdr,
                               cudaStream_t s);
  static cudaError_t fused(bool pairs, const KfArgs &a, const BucketParams &bp, uint32_t grid,
                           cudaStream_t s);
  static cudaError_t merge(bool pairs, const uint32_t *keys, const uint32_t *vals, uint32_t n,
                           const BucketParams &bp, const uint32_t *starts, const uint32_t *offs,
                           uint32_t G, uint32_t *keys_out, uint32_t *vals_out, cudaStream_t s);
};

template <int KIND>
cudaError_t Launch<KIND>::merge(bool pairs, const uint32_t *keys, const uint32_t *vals, uint32_t n,
                                const BucketParams &bp, const uint32_t *starts,
                                const uint32_t *offs, uint32_t G, uint32_t *keys_out,
                                uint32_t *vals_out, cudaStream_t s) {
  const uint32_t grid = min((n + 255u) / 256u, 148u * 16u);
  if (pairs)
    kx_shard_merge<KIND, true><<<grid, 256, 0, s>>>(keys, vals, n, bp, starts, offs, G, keys_out,
                                                    vals_out);
  else
    kx_shard_merge<KIND, false><<<grid, 256, 0, s>>>(keys, vals, n, bp, starts, offs, G, keys_out,
                                                     vals_out);
  return cudaGetLastError();
}

template <int KIND>
cudaError_t Launch<KIND>::range_hist(const uint32_t *keys, uint32_t n, uint32_t elems_per_cta,
                                     uint32_t grid, const BucketParams &bp, uint32_t *R,
                                     uint32_t *hdr, cudaStream_t s) {
  if (bp.m <= 2)
    ku_range_hist<KIND, true><<<grid, kThreads, 0, s>>>(keys, n, elems_per_cta, bp, R, hdr);
  else
    ku_range_hist<KIND, false><<<grid, kThreads, (size_t)kWarps * bp.m * 4u, s>>>(
        keys, n, elems_per_cta, bp, R, hdr);
  return cudaGetLastError();
}

template <int KIND>
cudaError_t Launch<KIND>::tile_hist(const uint32_t *keys, uint32_t n, uint32_t tile,
                                    uint32_t grid, const BucketParams &bp, uint32_t *H,
                                    uint32_t *hdr, cudaStream_t s) {
  if (bp.m <= 2)
    kh_tile_hist<KIND, true><<<grid, kThreads, 0, s>>>(keys, n, tile, bp, H, hdr);
  else
    kh_tile_hist<KIND, false><<<grid, kThreads, (size_t)kWarps * bp.m * 4u, s>>>(keys, n, tile,
                                                                                 bp, H, hdr);
  return cudaGetLastError();
}

template <int KIND, bool PAIRS, bool SMALLM, int CLS, int SCAN>
static cudaError_t kf_go(const KfArgs &a, const BucketParams &bp, uint32_t grid, cudaStream_t s) {
  constexpr KfShape sh = kf_shape(PAIRS, CLS);
  auto kern = kf_fused<KIND, PAIRS, SMALLM, sh.warps, sh.items, sh.ctas_per_sm, SCAN>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kf_smem_bytes(CLS == 0 ? 32 : (CLS == 1 ? 64 : kMaxBuckets), PAIRS));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  // programmatic dependent launch: the prologue (barrier init, TMA of the first
  // tiles) overlaps the tail of the previous kernel; griddep_wait() orders the rest
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(sh.warps * 32);
  cfg.dynamicSmemBytes = kf_smem_bytes(bp.m, PAIRS);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  // only after our own KR: a user kernel producing the input must complete first
  cfg.numAttrs = a.mode == kModeRange ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, a, bp);
}

template <int KIND>
cudaError_t Launch<KIND>::fused(bool pairs, const KfArgs &a, const BucketParams &bp,
                                uint32_t grid, cudaStream_t s) {
  if (bp.m <= 2)
    return pairs ? kf_go<KIND, true, true, 0, 1>(a, bp, grid, s)
                 : kf_go<KIND, false, true, 0, 1>(a, bp, grid, s);
  if (bp.m <= 32)
    return pairs ? kf_go<KIND, true, false, 0, 1>(a, bp, grid, s)
                 : kf_go<KIND, false, false, 0, 1>(a, bp, grid, s);
  if (bp.m <= 64)
    return pairs ? kf_go<KIND, true, false, 1, 2>(a, bp, grid, s)
                 : kf_go<KIND, false, false, 1, 2>(a, bp, grid, s);
  return pairs ? kf_go<KIND, true, false, 2, 0>(a, bp, grid, s)
               : kf_go<KIND, false, false, 2, 0>(a, bp, grid, s);
}

}  // namespace ms
