// ms_device.cuh -- device-side building blocks for the sm_100a multisplit:
// bucket identifiers, warp-level ranking helpers and the PTX wrappers for the
// TMA bulk-copy engine (cp.async.bulk + mbarrier) and release/acquire flags.
//
// Citations "P:nnn" are lines of the paper's LaTeX source.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ms {

// ---------------------------------------------------------------- tunables
constexpr int kWarp = 32;
// Histogram kernels use 16-warp CTAs; the postscan CTA shapes are in
// ms_kernels.cuh (kf_shape).
constexpr int kThreads = 512;
constexpr int kWarps = kThreads / kWarp;
constexpr int kMaxBuckets = 256;

// Internal forms: kDeltaShift is DELTA with delta = 2^shift (floor(u/delta) is a
// shift, then the clamp to m-1); kTopBits is f(u) = u >> shift with no clamp or
// mask, used when the digit is the key's top bits: DELTA with m * 2^shift =
// 2^32 (the bench's equal-width buckets of P:1107 with m = 2^k) and RADIX
// with shift + bits = 32 (the last LSD pass).
enum BucketKind : uint32_t {
  kIdentity = 0,
  kDelta = 1,
  kRadix = 2,
  kDeltaShift = 3,
  kTopBits = 4,
  kSplitters = 5
};

// Bucket identifier parameters, precomputed on the host.
struct BucketParams {
  uint32_t m;        // number of buckets
  uint32_t m1;       // m - 1
  uint32_t shift;    // RADIX
  uint32_t mask;     // RADIX: 2^bits - 1
  uint32_t magic_hi; // DELTA: M = ceil(2^64 / delta) split in two words
  uint32_t magic_lo;
  uint32_t delta_is_one;
  uint32_t spl_pow;          // SPLITTERS: smallest power of two >= m
  const uint32_t *spl;       // SPLITTERS: the m-1 interior splitters s_1 < ... < s_{m-1}
                             // (global on entry; kernels re-point it at a shared copy)
  const uint32_t *cell;      // SPLITTERS, staged: cell table over the key's top bits, or null
  uint32_t cell_shift;       // 32 - log2(cells)
  uint32_t spl_s, cell_s;    // the staged tables' shared-window addresses (ld.shared: a generic
                             // pointer into shared memory costs a generic load per probe)
};

// volatile: a plain asm statement may be speculated out of its guard (a kernel
// whose table is not staged then loads from a garbage shared address)
__device__ __forceinline__ uint32_t lds_u32(uint32_t saddr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr));
  return v;
}

// SPLITTERS (reading R27): f(u) = the j with s_j <= u <
// s_{j+1}, s_0 = 0 and s_m = 2^32 the ends of the key domain, i.e. the number
// of interior splitters <= u.  Branch-free upper-bound search with
// power-of-two steps (log2 spl_pow probes of the table).
// DEPTH = log2 of the largest table (8: m <= 256); the probes are unrolled so
// that the searches of a thread's keys interleave (a runtime-bounded loop
// serialized them: measured 136 Gkeys/s at m = 32)
// crowded cell (more than two splitters): the branch-free search over the
// staged table, out of line so that the common path is not if-converted into it
template <int DEPTH>
__device__ __noinline__ uint32_t splitter_search_staged(uint32_t u, uint32_t spl_s, uint32_t m1) {
  uint32_t k = 0;
#pragma unroll
  for (int q = DEPTH - 1; q >= 0; --q) {
    const uint32_t t = k + (1u << q);
    if (t <= m1 && lds_u32(spl_s + ((t - 1u) << 2)) <= u) k = t;
  }
  return k;
}

template <int DEPTH = 8>
__device__ __forceinline__ uint32_t splitter_bucket(uint32_t u, const BucketParams &p) {
  if (p.cell_shift) {  // staged (a shared-window address may be 0)
    // the cell of u's top bits holds the splitter indices [A, B): those of the
    // splitters inside the cell (A = the number below it).  For splitters spread
    // over the key domain a cell holds none or one (m = 256: 0.25 on average
    // with 1024 cells), so the bucket costs one table load and at most a
    // compare or two.
    const uint32_t x = lds_u32(p.cell_s + ((u >> p.cell_shift) << 2));
    const uint32_t j = x & 0xFFFFu, e = x >> 16;
    if (e - j > 2u) return splitter_search_staged<DEPTH>(u, p.spl_s, p.m1);
    uint32_t r = j;
    if (j < e && lds_u32(p.spl_s + (j << 2)) <= u) {
      r = j + 1u;
      if (j + 1u < e && lds_u32(p.spl_s + ((j + 1u) << 2)) <= u) r = j + 2u;
    }
    return r;
  }
  uint32_t j = 0;
#pragma unroll
  for (int k = DEPTH - 1; k >= 0; --k) {
    const uint32_t t = j + (1u << k);  // are the first t splitters all <= u?
    if (t <= p.m1 && p.spl[t - 1] <= u) j = t;
  }
  return j;
}

// Every kernel templated on the bucket kind starts with this: for SPLITTERS it
// copies the table into shared memory (CAP >= m-1 entries) and re-points
// bp.spl at the copy, so that the per-key search probes shared memory.
// It also builds the cell table: CAP >= 256 (m <= 256) 1024 cells of the top 10
// bits (4 KB), smaller tables 128 cells (512 B); cell c = [A_c | A_{c+1} << 16]
// with A_c = the number of splitters below c << cell_shift (A_cells = m - 1).
#define MS_STAGE_SPLITTERS(bp_, CAP) MS_STAGE_SPLITTERS3(bp_, CAP, true)
// CELLS = false: no cell table (a one-tile, latency-bound kernel: the table's
// build would cost more than the searches it saves)
#define MS_STAGE_SPLITTERS3(bp_, CAP, CELLS)                                    \
  if constexpr (KIND == kSplitters) {                                           \
    constexpr uint32_t ms_cb_ = (CAP) >= 256 ? 10u : 7u;                        \
    __shared__ uint32_t ms_s_spl[CAP];                                          \
    __shared__ uint32_t ms_s_cell[1u << ms_cb_];                                \
    for (uint32_t i_ = threadIdx.x; i_ < (bp_).m1 && i_ < (CAP); i_ += blockDim.x) \
      ms_s_spl[i_] = __ldg((bp_).spl + i_);                                     \
    __syncthreads();                                                            \
    if ((CELLS) && (bp_).m1 <= (CAP)) {                                         \
      for (uint32_t c_ = threadIdx.x; c_ < (1u << ms_cb_); c_ += blockDim.x) {  \
        const uint64_t lo_ = (uint64_t)c_ << (32u - ms_cb_);                    \
        const uint64_t hi_ = (uint64_t)(c_ + 1u) << (32u - ms_cb_);             \
        uint32_t a_ = 0, b_ = 0; /* splitters below lo_ / hi_ (lower bounds) */ \
        for (int k_ = 7; k_ >= 0; --k_) {                                       \
          const uint32_t ta_ = a_ + (1u << k_), tb_ = b_ + (1u << k_);          \
          if (ta_ <= (bp_).m1 && ms_s_spl[ta_ - 1u] < lo_) a_ = ta_;            \
          if (tb_ <= (bp_).m1 && ms_s_spl[tb_ - 1u] < hi_) b_ = tb_;            \
        }                                                                       \
        ms_s_cell[c_] = a_ | (b_ << 16);                                        \
      }                                                                         \
      __syncthreads();                                                          \
      (bp_).cell = ms_s_cell;                                                   \
      (bp_).cell_shift = 32u - ms_cb_;                                          \
      (bp_).cell_s = smem_u32(ms_s_cell);                                       \
      (bp_).spl_s = smem_u32(ms_s_spl);                                         \
    }                                                                           \
    (bp_).spl = ms_s_spl;                                                       \
  }

// f(u) for the three identifiers.  DELTA computes
// floor(u / delta) exactly as the high 64 bits of u * ceil(2^64/delta): the
// rounding error u*e/(delta*2^64) < 2^-32 <= 1/delta never crosses an integer
// for u, delta < 2^32.  IDENTITY clamps keys
// >= m into m-1 (the domain error itself is flagged by the caller).
template <int KIND>
__device__ __forceinline__ uint32_t bucket_of(uint32_t u, const BucketParams &p) {
  if constexpr (KIND == kRadix) {
    return (u >> p.shift) & p.mask;
  } else if constexpr (KIND == kTopBits) {
    return u >> p.shift;
  } else if constexpr (KIND == kDeltaShift) {
    const uint32_t q = u >> p.shift;
    return q < p.m1 ? q : p.m1;
  } else if constexpr (KIND == kIdentity) {
    return u < p.m1 ? u : p.m1;
  } else if constexpr (KIND == kSplitters) {
    return splitter_bucket<8>(u, p);
  } else {
    uint32_t q;
    if (p.delta_is_one) {
      q = u;
    } else {
      uint64_t t = (uint64_t)u * p.magic_hi + __umulhi(u, p.magic_lo);
      q = (uint32_t)(t >> 32);
    }
    return q < p.m1 ? q : p.m1;
  }
}

template <int KIND>
__device__ __forceinline__ bool key_domain_error(uint32_t u, const BucketParams &p) {
  if constexpr (KIND == kIdentity) return u >= p.m;
  return false;
}

// ---------------------------------------------------------------- warp helpers
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// Peer mask of Alg.3 (reading R4): the lanes of `active` whose
// bucket equals mine, from ceil(log2 m) binary ballots of the bucket bits
// (ballot-based voting).
template <int LOGM>
__device__ __forceinline__ uint32_t peer_mask_ballot(uint32_t b, uint32_t active, bool valid) {
  uint32_t peers = active;
#pragma unroll
  for (int k = 0; k < LOGM; ++k) {
    const bool bit = (b >> k) & 1u;
    const uint32_t vote = __ballot_sync(0xFFFFFFFFu, valid && bit);
    peers &= bit ? vote : ~vote;
  }
  return peers;
}

// ---------------------------------------------------------------- programmatic dependent launch
// griddepcontrol: a kernel launched with programmatic stream serialization may
// start before its predecessor finishes; griddep_wait() blocks until the
// predecessor grid has completed and its memory is visible.  Both are no-ops
// for a normal launch.
__device__ __forceinline__ void griddep_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------- PTX: smem address
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// bar.sync on a named barrier among the first `count` threads (multiple of 32)
__device__ __forceinline__ void named_barrier_sync(uint32_t id, uint32_t count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- PTX: mbarrier + TMA bulk copy
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// the same, with a suspend-time hint: a waiting thread may sleep (up to the hint,
// in ns) until the phase completes instead of re-polling (long waits of idle warps)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(0x100000u)
        : "memory");
  } while (!ok);
}

// 1-D bulk copy global -> shared through the TMA engine (SASS UBLKCP); bytes
// and both addresses must be multiples of 16.  Completion is signalled on
// `bar` as transaction bytes.  L2 policy: evict_first for streamed input.
__device__ __forceinline__ void tma_load_1d(void *smem_dst, const void *gmem_src, uint32_t bytes,
                                            uint64_t *bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// bulk prefetch global -> L2 (no shared memory, no completion tracking)
__device__ __forceinline__ void prefetch_l2_bulk(const void *gmem, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(gmem), "r"(bytes) : "memory");
}
// the same with an L2 cache policy (e.g. evict_last: keep the lines until their
// TMA load, ahead of the streaming output)
__device__ __forceinline__ void prefetch_l2_bulk_hint(const void *gmem, uint32_t bytes,
                                                      uint64_t policy) {
  asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(gmem),
               "r"(bytes), "l"(policy)
               : "memory");
}

// 1-D bulk copy shared -> global (TMA store, SASS UBLKCP).  Addresses and size
// must be multiples of 16 bytes; completion is tracked with bulk groups.
__device__ __forceinline__ void tma_store_1d(void *gmem_dst, const void *smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem_dst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// wait until every committed bulk store has finished READING shared memory
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// wait until all but the most recently committed bulk group have finished
// READING shared memory
__device__ __forceinline__ void bulk_wait_read_newest_pending() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
// wait until every committed bulk store has completed (writes performed)
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ---------------------------------------------------------------- PTX: global loads / flags
__device__ __forceinline__ uint4 ldg_stream_v4(const uint4 *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_release_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

}  // namespace ms
