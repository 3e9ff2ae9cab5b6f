// ms_dispatch.cuh -- host-side launchers mapping the runtime (bucket kind,
// m <= 2, pairs) onto kernel template instantiations.  Each bucket kind is
// instantiated in its own translation unit (ms_inst_*.cu) so nvcc runs them
// in parallel.
#pragma once
#include <cstdlib>
#include <cstring>

#include "ms_wide.cuh"
#include "ms_large.cuh"
#include "ms_onesweep.cuh"

#include <atomic>

namespace ms {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) applies to the current
// device only: each kernel instantiation keeps one bit per device (thread-safe;
// setting the attribute twice is harmless).
template <typename K>
inline cudaError_t set_max_smem(K kern, size_t bytes, std::atomic<unsigned long long> &done) {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) d = 0;
  const unsigned long long bit = 1ull << (d & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  const cudaError_t e =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
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
  // 32 < m <= 256 with warp offsets from the prescan (ms_wide.cuh)
  static cudaError_t tile_meta_wide(bool pairs, const uint32_t *keys, uint32_t n, uint32_t num_tiles,
                                    uint32_t tiles_per_cta, uint32_t grid, const BucketParams &bp,
                                    uint32_t *meta, uint32_t num_kf_tiles, uint32_t *R, uint32_t *hdr,
                                    cudaStream_t s);
  static cudaError_t fused_meta_wide(bool pairs, const KfArgs &a, const BucketParams &bp,
                                     uint32_t grid, cudaStream_t s);
  // m > 256 (ms_large.cuh): bucket ids and payloads of every key
  static cudaError_t bucket_ids(const uint32_t *keys, uint32_t n, const BucketParams &bp,
                                bool payload_index, uint32_t *b, uint32_t *p, uint32_t *hdr,
                                cudaStream_t s) {
    const uint32_t grid = min((n + 255u) / 256u, 148u * 8u);
    k_bucket_ids<KIND><<<grid ? grid : 1u, 256, 0, s>>>(keys, n, bp, payload_index ? 1 : 0, b, p, hdr);
    return cudaGetLastError();
  }
  // n <= kSmallMax in one CTA (ms_large.cuh)
  static cudaError_t small(bool pairs, const KfArgs &a, const BucketParams &bp, cudaStream_t s) {
    if (pairs)
      k_small<KIND, true><<<1, kThreads, 0, s>>>(a, bp);
    else
      k_small<KIND, false><<<1, kThreads, 0, s>>>(a, bp);
    return cudaGetLastError();
  }
  static cudaError_t merge(bool pairs, const uint32_t *keys, const uint32_t *vals, uint32_t n,
                           const BucketParams &bp, const uint32_t *starts, const uint32_t *offs,
                           uint32_t G, uint32_t *keys_out, uint32_t *vals_out, cudaStream_t s);
  // one-pass pipeline (ms_onesweep.cuh): bucket histograms of every pass in one
  // read, then one fused rank / look-back / scatter kernel per pass
  static cudaError_t ko_hist(const KoHistArgs &a, const BucketParams &bp, uint32_t grid, cudaStream_t s) {
    // the 4 x 8-bit sort (digits = the key's bytes) has its own unrolled kernel
    bool bytes = KIND == kRadix && a.npass == 4u;
    for (uint32_t p = 0; p < a.npass && bytes; ++p)
      bytes = a.shift[p] == 8u * p && a.mask[p] == 255u && a.bin0[p] == 256u * p;
    auto go = [&](auto kern, std::atomic<unsigned long long> &done) {
      const cudaError_t e = set_max_smem(kern, (size_t)kKoMaxBins * 32u * 4u, done);
      if (e != cudaSuccess) return e;
      kern<<<grid, 1024, (size_t)a.nbins * 32u * 4u, s>>>(a, bp);
      return cudaGetLastError();
    };
    static std::atomic<unsigned long long> done[2];
    return bytes ? go(ms::ko_hist<KIND, true>, done[0]) : go(ms::ko_hist<KIND, false>, done[1]);
  }
  static cudaError_t onesweep(bool pairs, const KoArgs &a, const BucketParams &bp, uint32_t grid,
                              cudaStream_t s) {
    auto go = [&](auto kern, bool pr, std::atomic<unsigned long long> &done) {
      const cudaError_t e = set_max_smem(kern, ko_smem_bytes(pr), done);
      if (e != cudaSuccess) return e;
      kern<<<grid, ko_threads(pr), ko_smem_bytes(pr), s>>>(a, bp);
      return cudaGetLastError();
    };
    static std::atomic<unsigned long long> done[2];
    return pairs ? go(ko_onesweep<KIND, true>, true, done[0]) : go(ko_onesweep<KIND, false>, false, done[1]);
  }
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
  static std::atomic<unsigned long long> done{0};
  const cudaError_t e0 =
      set_max_smem(kern, kf_smem_bytes(CLS == 0 ? 32 : (CLS == 1 ? 64 : kMaxBuckets), PAIRS, false), done);
  if (e0 != cudaSuccess) return e0;
  // programmatic dependent launch: the prologue (barrier init, TMA of the first
  // tiles) overlaps the tail of the previous kernel; griddep_wait() orders the rest
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(sh.warps * 32);
  cfg.dynamicSmemBytes = kf_smem_bytes(bp.m, PAIRS, a.rank_inc != 0);
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
  const size_t smax = km_smem_bytes(32, false) > km_smem_bytes(32, true) ? km_smem_bytes(32, false)
                                                                          : km_smem_bytes(32, true);
  static std::atomic<unsigned long long> done[4];
  auto go = [&](auto kern, int i) {
    const cudaError_t e = set_max_smem(kern, smax, done[i]);
    if (e != cudaSuccess) return e;
    kern<<<grid, kThreads + 32, smem, s>>>(keys, n, num_tiles, tiles_per_cta, bp, meta, R, hdr);
    return cudaGetLastError();
  };
  if (bp.m <= 2)
    return pairs ? go(km_tile_meta<KIND, true, 8>, 0) : go(km_tile_meta<KIND, true, 16>, 1);
  return pairs ? go(km_tile_meta<KIND, false, 8>, 2) : go(km_tile_meta<KIND, false, 16>, 3);
}

template <int KIND, bool PAIRS, bool SMALLM, int RANK, bool PROD>
static cudaError_t kfm_go2(const KfArgs &a, const BucketParams &bp, uint32_t grid, cudaStream_t s) {
  auto kern = kf_meta<KIND, PAIRS, SMALLM, PAIRS ? 8 : 16, RANK, PROD>;
  static std::atomic<unsigned long long> done{0};
  const cudaError_t e = set_max_smem(kern, kfm_smem_bytes(32, PAIRS), done);
  if (e != cudaSuccess) return e;
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

// whole-run TMA bulk stores with a producer warp: measured faster for m <= 16,
// slower at m = 32 (profiles/r01/); per-element scatter otherwise
template <int KIND, bool PAIRS, bool SMALLM, int RANK>
static cudaError_t kfm_go(const KfArgs &a, const BucketParams &bp, uint32_t grid, cudaStream_t s) {
  const bool prod = a.store_runs && bp.m <= 16;
  return prod ? kfm_go2<KIND, PAIRS, SMALLM, RANK, true>(a, bp, grid, s)
              : kfm_go2<KIND, PAIRS, SMALLM, RANK, false>(a, bp, grid, s);
}

template <int KIND>
cudaError_t Launch<KIND>::fused_meta(bool pairs, const KfArgs &a, const BucketParams &bp,
                                     uint32_t grid, cudaStream_t s) {
  if (bp.m <= 2)
    return pairs ? kfm_go<KIND, true, true, kRankBallot>(a, bp, grid, s)
                 : kfm_go<KIND, false, true, kRankBallot>(a, bp, grid, s);
  // m <= 4: ballots (measured faster than increments, which serialize on
  // eight lanes per counter); otherwise increments where the probe held
  if (bp.m <= 4)
    return pairs ? kfm_go<KIND, true, false, kRankVote2>(a, bp, grid, s)
                 : kfm_go<KIND, false, false, kRankVote2>(a, bp, grid, s);
  if (a.rank_inc)
    return pairs ? kfm_go<KIND, true, false, kRankInc>(a, bp, grid, s)
                 : kfm_go<KIND, false, false, kRankInc>(a, bp, grid, s);
  return pairs ? kfm_go<KIND, true, false, kRankMasks>(a, bp, grid, s)
               : kfm_go<KIND, false, false, kRankMasks>(a, bp, grid, s);
}

template <int KIND, int NB, bool PAIRS>
static cudaError_t kmw_go(const uint32_t *keys, uint32_t n, uint32_t num_tiles, uint32_t per,
                          uint32_t grid, const BucketParams &bp, uint32_t *meta, uint32_t nkf,
                          uint32_t *R, uint32_t *hdr, cudaStream_t s) {
  auto kern = km_meta_wide<KIND, NB, PAIRS>;
  static std::atomic<unsigned long long> done{0};
  const cudaError_t e = set_max_smem(kern, kmw_smem_bytes(NB, PAIRS), done);
  if (e != cudaSuccess) return e;
  kern<<<grid, kThreads + 32 * kmw_scan_warps(NB), kmw_smem_bytes(NB, PAIRS), s>>>(keys, n, num_tiles, per, bp, meta,
                                                                       nkf, R, hdr);
  return cudaGetLastError();
}

template <int KIND>
cudaError_t Launch<KIND>::tile_meta_wide(bool pairs, const uint32_t *keys, uint32_t n,
                                         uint32_t num_tiles, uint32_t per, uint32_t grid,
                                         const BucketParams &bp, uint32_t *meta, uint32_t nkf,
                                         uint32_t *R, uint32_t *hdr, cudaStream_t s) {
  const uint32_t nb = wide_nb(bp.m);
#define MS_KMW(NB_) \
  return pairs ? kmw_go<KIND, NB_, true>(keys, n, num_tiles, per, grid, bp, meta, nkf, R, hdr, s) \
               : kmw_go<KIND, NB_, false>(keys, n, num_tiles, per, grid, bp, meta, nkf, R, hdr, s)
  if (nb == 2) { MS_KMW(2); }
  if (nb == 4) { MS_KMW(4); }
  MS_KMW(8);
#undef MS_KMW
}

template <int KIND, bool PAIRS, int NB>
static cudaError_t kfw_go(const KfArgs &a, const BucketParams &bp, uint32_t grid, cudaStream_t s) {
  auto kern = kf_meta_wide<KIND, PAIRS, NB>;
  static std::atomic<unsigned long long> done{0};
  const cudaError_t e = set_max_smem(kern, kfw_smem_bytes(PAIRS, NB), done);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(wide_kw(PAIRS) * 32);
  cfg.dynamicSmemBytes = kfw_smem_bytes(PAIRS, NB);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;  // right after our own KR
  return cudaLaunchKernelEx(&cfg, kern, a, bp);
}

template <int KIND>
cudaError_t Launch<KIND>::fused_meta_wide(bool pairs, const KfArgs &a, const BucketParams &bp,
                                          uint32_t grid, cudaStream_t s) {
  const uint32_t nb = wide_nb(bp.m);
  if (nb == 2) return pairs ? kfw_go<KIND, true, 2>(a, bp, grid, s) : kfw_go<KIND, false, 2>(a, bp, grid, s);
  if (nb == 4) return pairs ? kfw_go<KIND, true, 4>(a, bp, grid, s) : kfw_go<KIND, false, 4>(a, bp, grid, s);
  return pairs ? kfw_go<KIND, true, 8>(a, bp, grid, s) : kfw_go<KIND, false, 8>(a, bp, grid, s);
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
