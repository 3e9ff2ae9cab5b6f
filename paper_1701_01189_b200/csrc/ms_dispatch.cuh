// ms_dispatch.cuh -- host-side launchers mapping the runtime (bucket kind,
// m <= 2, pairs) onto kernel template instantiations.  Each bucket kind is
// instantiated in its own translation unit (ms_inst_*.cu) so nvcc runs them
// in parallel.
#pragma once
#include <cstdlib>
#include <cstring>

#include "ms_meta.cuh"

namespace ms {

// L2 prefetch distance (tiles) of KM beyond its TMA ring (MS_KM_PREFETCH; default 0:
// 2 and 4 measured slower)
inline uint32_t km_prefetch() {
  static const uint32_t v = [] {
    const char *e = std::getenv("MS_KM_PREFETCH");
    return e ? (uint32_t)std::atoi(e) : 0u;
  }();
  return v;
}

// MS_META_RANK=atomic selects the shared-memory atomicOr peer masks in kf_meta
// Tiles at the end of each KM range loaded with an L2 evict_last policy, for
// KF's reverse tile order (MS_KM_KEEP, default 0; with MS_KF_REVERSE=1)
inline uint32_t km_keep_last() {
  static const uint32_t v = [] {
    const char *e = std::getenv("MS_KM_KEEP");
    return e ? (uint32_t)std::atoi(e) : 0u;
  }();
  return v;
}

// Whether this GPU returns same-address shared-memory increments in lane order
// (RANK 8); probed once per process on a private stream (ms_capi.cu).
bool lane_ordered_inc();

// kf_meta's RANK for m buckets: MS_META_RANK = atomic | ballot | mix3 | mix2 |
// xatomic | xmix3 | xmix2 overrides; by default the choice measured best per
// number of bucket bits (profiles/r01/s2_rank_modes.md)
inline int meta_rank_mode(uint32_t m) {
  static const int forced = [] {
    const char *e = std::getenv("MS_META_RANK");
    if (!e) return -1;
    const char *names[] = {"atomic", "ballot", "mix3", "mix2", "xatomic", "xmix3", "xmix2", "xpair", "inc"};
    for (int i = 0; i < 9; ++i)
      if (!std::strcmp(e, names[i])) return i;
    return -1;
  }();
  if (forced >= 0) return forced;
  if (lane_ordered_inc()) return 8;
  return m <= 8 ? 6 : (m <= 16 ? 5 : 7);
}

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
  // m <= 32 pipeline with warp offsets from the prescan (ms_meta.cuh)
  static cudaError_t tile_meta(bool pairs, const uint32_t *keys, uint32_t n, uint32_t num_tiles,
                               uint32_t tiles_per_cta, uint32_t grid, const BucketParams &bp,
                               uint32_t *meta, uint32_t *R, uint32_t *hdr, cudaStream_t s);
  static cudaError_t fused_meta(bool pairs, const KfArgs &a, const BucketParams &bp,
                                uint32_t grid, cudaStream_t s);
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
                                         (int)kf_smem_bytes(CLS == 0 ? 32 : (CLS == 1 ? 64 : kMaxBuckets), PAIRS, false, true));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  // programmatic dependent launch: the prologue (barrier init, TMA of the first
  // tiles) overlaps the tail of the previous kernel; griddep_wait() orders the rest
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(sh.warps * 32);
  cfg.dynamicSmemBytes = kf_smem_bytes(bp.m, PAIRS, a.rank_inc != 0, a.carry != 0);
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
cudaError_t Launch<KIND>::tile_meta(bool pairs, const uint32_t *keys, uint32_t n,
                                    uint32_t num_tiles, uint32_t tiles_per_cta, uint32_t grid,
                                    const BucketParams &bp, uint32_t *meta, uint32_t *R,
                                    uint32_t *hdr, cudaStream_t s) {
  const size_t smem = km_smem_bytes(bp.m, pairs);
  static bool configured = false;
  if (!configured) {
    for (auto kern : {km_tile_meta<KIND, true, 8>, km_tile_meta<KIND, false, 8>,
                      km_tile_meta<KIND, true, 16>, km_tile_meta<KIND, false, 16>}) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)(km_smem_bytes(32, false) > km_smem_bytes(32, true) ? km_smem_bytes(32, false) : km_smem_bytes(32, true)));
      if (e != cudaSuccess) return e;
    }
    configured = true;
  }
  if (bp.m <= 2) {
    if (pairs)
      km_tile_meta<KIND, true, 8><<<grid, kThreads + 32, smem, s>>>(keys, n, num_tiles, tiles_per_cta, bp, meta, R, hdr, km_prefetch(), km_keep_last());
    else
      km_tile_meta<KIND, true, 16><<<grid, kThreads + 32, smem, s>>>(keys, n, num_tiles, tiles_per_cta, bp, meta, R, hdr, km_prefetch(), km_keep_last());
  } else {
    if (pairs)
      km_tile_meta<KIND, false, 8><<<grid, kThreads + 32, smem, s>>>(keys, n, num_tiles, tiles_per_cta, bp, meta, R, hdr, km_prefetch(), km_keep_last());
    else
      km_tile_meta<KIND, false, 16><<<grid, kThreads + 32, smem, s>>>(keys, n, num_tiles, tiles_per_cta, bp, meta, R, hdr, km_prefetch(), km_keep_last());
  }
  return cudaGetLastError();
}

template <int KIND, bool PAIRS, bool SMALLM, int RANK, bool PROD>
static cudaError_t kfm_go2(const KfArgs &a, const BucketParams &bp, uint32_t grid, cudaStream_t s) {
  auto kern = kf_meta<KIND, PAIRS, SMALLM, PAIRS ? 8 : 16, RANK, PROD>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kfm_smem_bytes(32, PAIRS));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(PROD ? kThreads + 32 : kThreads);
  cfg.dynamicSmemBytes = kfm_smem_bytes(bp.m, PAIRS);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;  // always right after our own KM
  return cudaLaunchKernelEx(&cfg, kern, a, bp);
}

// whole-run TMA bulk stores -> producer-warp variant; per-element scatter otherwise
template <int KIND, bool PAIRS, bool SMALLM, int RANK>
static cudaError_t kfm_go(const KfArgs &a, const BucketParams &bp, uint32_t grid, cudaStream_t s) {
  // producer warp: measured faster for m <= 16, slower at m = 32 (profiles/r01/)
  static const int prod_env = [] {
    const char *e = std::getenv("MS_META_PROD");
    return e ? std::atoi(e) : -1;
  }();
  const bool prod = a.store_runs && (prod_env >= 0 ? prod_env != 0 : bp.m <= 16);
  return prod ? kfm_go2<KIND, PAIRS, SMALLM, RANK, true>(a, bp, grid, s)
              : kfm_go2<KIND, PAIRS, SMALLM, RANK, false>(a, bp, grid, s);
}

template <int KIND>
cudaError_t Launch<KIND>::fused_meta(bool pairs, const KfArgs &a, const BucketParams &bp,
                                     uint32_t grid, cudaStream_t s) {
  if (bp.m <= 2)
    return pairs ? kfm_go<KIND, true, true, 0>(a, bp, grid, s) : kfm_go<KIND, false, true, 0>(a, bp, grid, s);
#define MS_KFM_CASE(R) \
  case R: return pairs ? kfm_go<KIND, true, false, R>(a, bp, grid, s) : kfm_go<KIND, false, false, R>(a, bp, grid, s)
  switch (meta_rank_mode(bp.m)) {
    MS_KFM_CASE(0);
    MS_KFM_CASE(1);
    MS_KFM_CASE(3);
    MS_KFM_CASE(4);
    MS_KFM_CASE(5);
    MS_KFM_CASE(6);
    MS_KFM_CASE(7);
    MS_KFM_CASE(8);
    default: return pairs ? kfm_go<KIND, true, false, 2>(a, bp, grid, s) : kfm_go<KIND, false, false, 2>(a, bp, grid, s);
  }
#undef MS_KFM_CASE
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
