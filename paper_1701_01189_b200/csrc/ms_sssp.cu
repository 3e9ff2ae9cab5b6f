// ms_sssp.cu -- Multisplit-SSSP (Sec.7.2): delta-stepping with the
// Bucketing strategy of Davidson et al., whose bucketing step --
// a radix sort in the original -- is this library's stable multisplit with
// splitter buckets.
//
// Per iteration (host loop; one small device-to-host read per iteration):
//   1. splitters s_j = B + j*Delta (j = 1 .. K-1), B = the smallest tentative
//      distance in the work list: bucket 0 = [0, B + Delta) is the near-most
//      bucket of delta-stepping (Meyer & Sanders), K-1 = everything beyond;
//   2. ms_multisplit_pairs of the work list (key = tentative distance when the
//      item was pushed, value = vertex) into the K buckets;
//   3. KRX k_sssp_relax: items of bucket 0 whose key still equals dist[v] relax
//      their out-edges (atomicMin on dist); every improvement pushes (nd, u)
//      to the next work list behind the items of buckets 1..K-1, which are
//      carried over as they are; the minimum key of the next list is reduced
//      on the fly.
// The work list is label-correcting: the loop ends when it is empty, and the
// distances are then the shortest ones whatever the processing order.
#include <algorithm>
#include <cstdint>

#include "../../include/multisplit.h"
#include "ms_device.cuh"

namespace {

using namespace ms;

constexpr uint32_t kInf = 0xFFFFFFFFu;

struct SsspCtl {
  uint32_t push, minkey, overflow, nrem;
  uint32_t relax_attempts, pad[3];
};

__global__ void __launch_bounds__(256)
    k_sssp_init(uint32_t *__restrict__ dist, uint32_t V, uint32_t source, uint32_t *__restrict__ wk,
                uint32_t *__restrict__ wv, SsspCtl *ctl) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x)
    dist[v] = v == source ? 0u : kInf;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    wk[0] = 0u;
    wv[0] = source;
    ctl->overflow = 0u;
  }
}

// splitters s_1..s_{K-1} of this iteration and the reset of the per-iteration counters
__global__ void __launch_bounds__(256)
    k_sssp_splitters(uint32_t *__restrict__ spl, uint32_t k1, uint32_t base, uint32_t delta, SsspCtl *ctl) {
  for (uint32_t j = threadIdx.x; j < k1; j += blockDim.x) spl[j] = base + (j + 1u) * delta;
  if (threadIdx.x == 0) {
    ctl->push = 0u;
    ctl->minkey = kInf;
    ctl->relax_attempts = 0u;
  }
}

// A warp relaxes one edge per lane (valid lanes); improvements are pushed with
// one warp-aggregated atomic on the push counter.
__device__ __forceinline__ void relax_edge(bool valid, uint32_t e, uint32_t d, uint32_t *__restrict__ dist,
                                           const uint32_t *__restrict__ col, const uint32_t *__restrict__ w,
                                           uint32_t *__restrict__ nk, uint32_t *__restrict__ nv, uint32_t nrem,
                                           uint32_t cap, SsspCtl *ctl, uint32_t &mymin, uint32_t lane) {
  bool push = false;
  uint32_t u = 0, nd = 0;
  if (valid) {
    u = __ldg(col + e);
    const uint64_t t = (uint64_t)d + __ldg(w + e);
    if (t < kInf) {
      nd = (uint32_t)t;
      if (nd < __ldcg(dist + u)) push = nd < atomicMin(dist + u, nd);
    }
  }
  const uint32_t pm = __ballot_sync(0xFFFFFFFFu, push);
  if (pm) {
    const uint32_t leader = __ffs(pm) - 1u;
    uint32_t b = 0;
    if (lane == leader) b = atomicAdd(&ctl->push, (uint32_t)__popc(pm));
    b = __shfl_sync(0xFFFFFFFFu, b, leader);
    if (push) {
      const uint64_t slot = (uint64_t)nrem + b + __popc(pm & lanemask_lt());
      if (slot < cap) {
        nk[slot] = nd;
        nv[slot] = u;
        mymin = min(mymin, nd);
      } else {
        ctl->overflow = 1u;
      }
    }
  }
}

__global__ void __launch_bounds__(256)
    k_sssp_relax(const uint32_t *__restrict__ ok, const uint32_t *__restrict__ ov, uint32_t n,
                 const uint32_t *__restrict__ off, uint32_t *__restrict__ dist,
                 const uint32_t *__restrict__ rp, const uint32_t *__restrict__ col,
                 const uint32_t *__restrict__ w, uint32_t *__restrict__ nk, uint32_t *__restrict__ nv,
                 uint32_t cap, SsspCtl *ctl) {
  const uint32_t hi = __ldcg(off + 1);  // bucket 0 = items [0, hi)
  const uint32_t nrem = n - hi;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x, gsz = gridDim.x * blockDim.x;
  if (gtid == 0) ctl->nrem = nrem;
  uint32_t mymin = kInf;
  // buckets 1..K-1 carry over to the front of the next work list
  for (uint32_t i = gtid; i < nrem; i += gsz) {
    const uint32_t k = __ldg(ok + hi + i);
    nk[i] = k;
    nv[i] = __ldg(ov + hi + i);
    mymin = min(mymin, k);
  }
  // bucket 0: warps take 32 items at a time and flatten their edge lists: the
  // warp's edges are numbered by an exclusive scan of the lanes' degrees and
  // lane j relaxes edge g = 32 c + j of chunk c, found by a binary search over
  // the scan (all lanes busy whatever the degree mix; the loads of a chunk are
  // independent, unlike a per-lane walk of a vertex's list)
  // Each warp takes a contiguous segment of ceil(hi / warps) items (usually a
  // handful: frontiers are small next to the grid), so every warp of the grid
  // has edges in flight, not only hi / 32 of them.
  const uint32_t wid = gtid >> 5, nw = gsz >> 5;
  const uint32_t S = max(1u, (hi + nw - 1u) / nw);
  for (uint32_t s0 = wid * S; s0 < hi; s0 += nw * S)
  for (uint32_t b0 = s0, s1 = min(hi, s0 + S); b0 < s1; b0 += 32u) {
    const uint32_t i = b0 + lane;
    uint32_t d = 0, e0 = 0, deg = 0;
    if (i < s1) {
      const uint32_t v = __ldg(ov + i);
      d = __ldg(ok + i);
      if (d == __ldcg(dist + v)) {  // else a stale item: a shorter path has been pushed
        e0 = __ldg(rp + v);
        deg = __ldg(rp + v + 1) - e0;
      }
    }
    uint32_t incl = deg;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= (uint32_t)o) incl += y;
    }
    const uint32_t excl = incl - deg;
    const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    for (uint32_t c = 0; c < total; c += 32u) {
      const uint32_t g = c + lane;
      uint32_t s = 0;  // the last lane whose first edge is <= g
#pragma unroll
      for (uint32_t step = 16; step != 0; step >>= 1) {
        const uint32_t ex = __shfl_sync(0xFFFFFFFFu, excl, s + step);
        if (ex <= g) s += step;
      }
      const uint32_t sd = __shfl_sync(0xFFFFFFFFu, d, s);
      const uint32_t se = __shfl_sync(0xFFFFFFFFu, e0, s) + (g - __shfl_sync(0xFFFFFFFFu, excl, s));
      relax_edge(g < total, se, sd, dist, col, w, nk, nv, nrem, cap, ctl, mymin, lane);
    }
  }
  mymin = __reduce_min_sync(0xFFFFFFFFu, mymin);
  if (lane == 0 && mymin != kInf) atomicMin(&ctl->minkey, mymin);
}

constexpr size_t kAl = 256;
size_t al(size_t x) { return (x + kAl - 1) / kAl * kAl; }

struct SsspLayout {
  size_t ctl, off, spl, wk0, wv0, wk1, wv1, ms, ms_bytes, total;
  uint64_t cap;
};

SsspLayout sssp_layout(uint32_t V, uint64_t E, uint32_t K) {
  SsspLayout l{};
  l.cap = std::min<uint64_t>(2ull * E + V + 1024ull, 0xFFFFFFFFull);
  size_t o = 0;
  l.ctl = o; o += al(sizeof(SsspCtl));
  l.off = o; o += al((size_t)(K + 1) * 4u);
  l.spl = o; o += al((size_t)K * 4u);
  l.wk0 = o; o += al(l.cap * 4u);
  l.wv0 = o; o += al(l.cap * 4u);
  l.wk1 = o; o += al(l.cap * 4u);
  l.wv1 = o; o += al(l.cap * 4u);
  l.ms = o;
  l.ms_bytes = ms_multisplit_workspace_size(l.cap, K, 1);
  o += al(l.ms_bytes);
  l.total = o;
  return l;
}

}  // namespace

extern "C" {

size_t ms_sssp_workspace_size(uint32_t V, uint64_t E, uint32_t K) {
  if (K < 1) K = 1;
  if (K > 256) K = 256;
  return sssp_layout(V, E, K).total;
}

ms_status ms_sssp(const uint32_t *row_ptr, const uint32_t *col, const uint32_t *w, uint32_t V,
                  uint64_t E, uint32_t source, uint32_t delta, uint32_t K, uint32_t *dist, void *ws,
                  size_t ws_bytes, void *stream, ms_sssp_stats *stats) {
  if (V == 0 || source >= V || delta == 0) return MS_ERR_INVALID_VALUE;
  if (K < 1 || K > 256 || E >= (1ull << 32) || 2ull * E + V + 1024ull > 0xFFFFFFFFull)
    return MS_ERR_UNSUPPORTED;
  if (!row_ptr || !dist || !ws || (E > 0 && (!col || !w)) || ((uintptr_t)ws & (kAl - 1)))
    return MS_ERR_INVALID_VALUE;
  const SsspLayout lo = sssp_layout(V, E, K);
  if (ws_bytes < lo.total) return MS_ERR_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  char *p = (char *)ws;
  SsspCtl *ctl = (SsspCtl *)(p + lo.ctl);
  uint32_t *off = (uint32_t *)(p + lo.off), *spl = (uint32_t *)(p + lo.spl);
  uint32_t *wk = (uint32_t *)(p + lo.wk0), *wv = (uint32_t *)(p + lo.wv0);
  uint32_t *ok = (uint32_t *)(p + lo.wk1), *ov = (uint32_t *)(p + lo.wv1);
  ms_sssp_stats st{};
  k_sssp_init<<<std::min((V + 255u) / 256u, 148u * 8u), 256, 0, s>>>(dist, V, source, wk, wv, ctl);
  if (cudaGetLastError() != cudaSuccess) return MS_ERR_CUDA;
  uint64_t n = 1;
  uint32_t base = 0;
  while (n > 0) {
    // K buckets of width delta from the smallest tentative distance, as many as fit below 2^32
    const uint64_t room = (0xFFFFFFFFull - base) / delta;
    const uint32_t keff = (uint32_t)std::min<uint64_t>(K, room + 1u);
    k_sssp_splitters<<<1, 256, 0, s>>>(spl, keff - 1u, base, delta, ctl);
    if (cudaGetLastError() != cudaSuccess) return MS_ERR_CUDA;
    const ms_bucket_fn fn{MS_BUCKET_SPLITTERS, keff, 0u, 0u, 0u, keff > 1 ? spl : nullptr};
    ms_status r = ms_multisplit_pairs(wk, wv, ok, ov, n, &fn, off, p + lo.ms, lo.ms_bytes, stream);
    if (r != MS_SUCCESS) return r;
    const uint32_t grid = (uint32_t)std::max<uint64_t>(1u, std::min<uint64_t>((n + 255u) / 256u, 148u * 8u));
    k_sssp_relax<<<grid, 256, 0, s>>>(ok, ov, (uint32_t)n, off, dist, row_ptr, col, w, wk, wv,
                                       (uint32_t)lo.cap, ctl);
    if (cudaGetLastError() != cudaSuccess) return MS_ERR_CUDA;
    SsspCtl h{};
    if (cudaMemcpyAsync(&h, ctl, sizeof h, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return MS_ERR_CUDA;
    if (h.overflow) return MS_ERR_WORKSPACE;
    st.iterations += 1;
    st.items += n;
    st.frontier += n - h.nrem;
    st.pushes += h.push;
    n = (uint64_t)h.nrem + h.push;
    base = h.minkey;
  }
  if (stats) *stats = st;
  return MS_SUCCESS;
}

}  // extern "C"
