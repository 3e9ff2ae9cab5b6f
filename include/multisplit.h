/*
 * multisplit.h -- C ABI of libms, a B200 (sm_100a) implementation of the
 * stable multisplit and multisplit radix sort of arXiv 1701.01189
 * ("GPU Multisplit: an extended study of a parallel algorithm").
 *
 * Citations "P:nnn" are lines of the paper's LaTeX source.
 *
 * Conventions (all entry points):
 *  - Data pointers are DEVICE pointers unless stated; keys and values are
 *    32-bit words (keys unsigned, values opaque payload).
 *  - Calls are asynchronous and stream-ordered on `stream` (a cudaStream_t
 *    passed as void*; NULL = legacy default stream).  No call allocates
 *    memory, synchronizes, or copies to the host, except ms_device_init /
 *    ms_lane_ordered_increment (one-time probe), ms_device_status, and the
 *    NCCL path of the sharded calls (documented there).  Every multisplit /
 *    sort call can be captured in a CUDA graph.
 *  - The caller owns every buffer.  Workspace is queried with the matching
 *    *_workspace_size function (pure host arithmetic) and passed in; it must
 *    be 256-byte aligned (else MS_ERR_INVALID_VALUE; cudaMalloc and torch
 *    allocations are); one workspace serves one in-flight call.  Inputs are never modified.  Outputs must not alias
 *    inputs (P:785-787 key_in / key_out are distinct).
 *  - Host-detectable argument errors return before anything is launched.
 *    Device-detected key-domain errors (identity bucket with key >= m) set
 *    a flag in the workspace that ms_device_status reports; the output of
 *    that call is then unspecified (no out-of-bounds write happens).
 *  - n < 2^32 (offsets are 32-bit).  1 <= m <= 256 (paper scope) for
 *    every call; the multisplit calls also take 256 < m <= 65536 (below).
 */
#ifndef MULTISPLIT_H_
#define MULTISPLIT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MS_SUCCESS = 0,
  MS_ERR_INVALID_VALUE = 1, /* null pointer, aliasing, bad bucket parameters */
  MS_ERR_UNSUPPORTED = 2,   /* m outside [1,256], n >= 2^32 */
  MS_ERR_WORKSPACE = 3,     /* ws_bytes smaller than the *_workspace_size value */
  MS_ERR_CUDA = 4,          /* a CUDA launch / runtime error */
  MS_ERR_KEY_DOMAIN = 5,    /* device-detected: identity key >= m */
  MS_ERR_NCCL = 6           /* NCCL missing or an NCCL call failed (sharded calls) */
} ms_status;

/* Bucket identifiers f(u). */
typedef enum {
  MS_BUCKET_IDENTITY = 0, /* f(u) = u; requires u < m                     */
  MS_BUCKET_DELTA = 1,    /* f(u) = min(floor(u / delta), m-1), delta >= 1 */
  MS_BUCKET_RADIX = 2,    /* f(u) = (u >> shift) & (2^bits - 1), m = 2^bits */
  MS_BUCKET_SPLITTERS = 3 /* f(u) = j with s_j <= u < s_{j+1}: `splitters` holds
                             the m-1 interior splitters s_1 < ... < s_{m-1} (device memory,
                             strictly increasing -- not checked; an unordered table gives an
                             unspecified permutation, never an out-of-bounds write); s_0 = 0
                             and s_m = 2^32 are the ends of the key domain (R27) */
} ms_bucket_kind;

typedef struct {
  uint32_t kind;        /* ms_bucket_kind */
  uint32_t num_buckets; /* m: 1..256, or up to 65536 for the m > 256 path (see below) */
  uint32_t delta;       /* DELTA only: bucket width, >= 1 */
  uint32_t shift;       /* RADIX only: first bit of the digit */
  uint32_t bits;        /* RADIX only: digit width 1..8 (1..16 when m > 256), shift + bits <= 32 */
  const uint32_t *splitters; /* SPLITTERS only: m-1 device words (may be NULL when m = 1) */
} ms_bucket_fn;

/* Human-readable name of a status code (static storage). */
const char *ms_status_string(ms_status s);

/* Library version, e.g. "0.1.0". */
const char *ms_version(void);

/* One-time, per-device initialisation (synchronous; call it once per device
 * before use and outside any CUDA graph capture; idempotent and thread-safe;
 * device < 0 = the current device).  It runs the probe of reading R23
 * (DESIGN.md): whether the GPU returns the old values of one warp
 * instruction's same-address shared-memory increments in lane order, and
 * applies consecutive increments of a warp in program order -- checked over
 * the whole grid in the postscan's own launch shape (512 threads, two CTAs per
 * SM) with random, sorted-run, 90 %-skewed and two-bucket patterns over up to
 * 256 counters.  Where the probe held, the postscan ranks a window's keys with
 * such increments of the warp's running slot (Eq.4 term 1); on a
 * device that has not been initialised, or where the probe failed, it ranks
 * with deterministic peer masks (Alg.3's peer masks).  Results are
 * identical either way; only speed differs.  MS_ERR_CUDA on a CUDA failure. */
ms_status ms_device_init(int device);

/* The probe result for the current device (runs the probe if needed, as
 * ms_device_init does): 1 = lane-ordered, 0 = not (or a CUDA failure). */
int ms_lane_ordered_increment(void);

/* Process-wide options (thread-safe; they apply to calls issued afterwards).
 *   MS_OPT_RANK:       MS_RANK_AUTO (default: increments where the device's
 *                      probe held) or MS_RANK_PEER_MASKS (always the
 *                      deterministic peer masks).
 *   MS_OPT_RUN_STORES: 1 (default: whole-run TMA bulk stores where runs are
 *                      long) or 0 (per-element coalesced stores only).
 *   MS_OPT_PIPELINE:   MS_PIPELINE_AUTO (default: LEVEL0, except key-value
 *                      pairs with m > 128, which take ONESWEEP -- measured
 *                      faster there: 2^27 pairs, m = 256, 216 vs 170 Gpairs/s),
 *                      MS_PIPELINE_LEVEL0 (Eq.3 with the CTA ranges
 *                      as level 0, two launches) or MS_PIPELINE_TILE (the
 *                      paper's {tile histograms H, scan of H, postscan},
 *                      P:529-540, three launches) or MS_PIPELINE_ONESWEEP
 *                      (bucket counts in one read, then one
 *                      fused rank / decoupled look-back / scatter kernel;
 *                      n < 2^30 on a device whose probe held, else LEVEL0).
 *   MS_OPT_SORT:       MS_SORT_AUTO (default: the radix sort computes every
 *                      digit histogram in one read and runs one fused
 *                      look-back pass per digit, 36 B/key for 4 x 8 bits;
 *                      where n < 2^30, the probe held, every digit has
 *                      >= 7 bits) or
 *                      MS_SORT_PASSES (every pass a full multisplit,
 *                      P:1613-1616, 48 B/key).
 * ms_set_option returns MS_ERR_INVALID_VALUE for an unknown option / value;
 * ms_get_option returns the value, or -1 for an unknown option. */
enum { MS_OPT_RANK = 0, MS_OPT_RUN_STORES = 1, MS_OPT_PIPELINE = 2, MS_OPT_SORT = 3 };
enum { MS_RANK_AUTO = 0, MS_RANK_PEER_MASKS = 1 };
enum { MS_PIPELINE_LEVEL0 = 0, MS_PIPELINE_TILE = 1, MS_PIPELINE_ONESWEEP = 2, MS_PIPELINE_AUTO = 3 };
enum { MS_SORT_AUTO = 0, MS_SORT_PASSES = 1 };
ms_status ms_set_option(int option, int value);
int ms_get_option(int option);

/* Fill *out with delta buckets of width ceil(2^32 / m) (2^32-1 for m = 1),
 * the equal-width partition of the key domain of P:1107. */
ms_status ms_bucket_delta_default(uint32_t m, ms_bucket_fn *out);
ms_status ms_bucket_identity(uint32_t m, ms_bucket_fn *out);
ms_status ms_bucket_radix(uint32_t shift, uint32_t bits, ms_bucket_fn *out);

/* Check a bucket function (host only): MS_SUCCESS, MS_ERR_INVALID_VALUE or
 * MS_ERR_UNSUPPORTED. */
ms_status ms_bucket_validate(const ms_bucket_fn *fn);

/* ------------------------------------------------------------------------
 * Stable multisplit (Eq.(1)): permute n keys (and
 * values) so that buckets B_0..B_{m-1} are contiguous in ascending bucket
 * order and input order is preserved inside each bucket.
 *
 *   keys_in, vals_in     n words each (device).  vals_* may be NULL only in
 *                        the _keys variant.
 *   keys_out, vals_out   n words each (device), must not overlap the inputs.
 *   bucket_offsets       NULL, or m+1 words (device): start of each bucket in
 *                        the output, bucket_offsets[m] = n (reading R2).
 *   ws, ws_bytes         device workspace of at least
 *                        ms_multisplit_workspace_size(n, m, with_values) bytes.
 *
 * Pipeline (Alg.1): per-tile histogram -> global
 * exclusive scan of the bucket x tile matrix (Eq.2) -> tile-local stable
 * reorder in shared memory + coalesced scatter.  n <= one tile runs as a
 * single launch.
 *
 * m > 256 (Sec.6.3; DELTA / IDENTITY / SPLITTERS up to 65536
 * buckets, RADIX digits of 9..16 bits): the paper iterates multisplits over at
 * most 256 buckets; here the iteration is LSD over the 8-bit digits of the
 * bucket id, which needs no property of f: one pass writes the bucket ids b_i
 * and payloads (the key, or the index for pairs), two stable radix-digit
 * multisplits of the (b, payload) pairs sort them by b, the offsets come from
 * the sorted ids, and pairs are gathered by index.  RADIX digits wider than 8
 * bits are two radix passes over the keys.  The workspace query covers it.
 * --------------------------------------------------------------------- */
size_t ms_multisplit_workspace_size(uint64_t n, uint32_t m, int with_values);

ms_status ms_multisplit_keys(const uint32_t *keys_in, uint32_t *keys_out, uint64_t n,
                             const ms_bucket_fn *fn, uint32_t *bucket_offsets, void *ws,
                             size_t ws_bytes, void *stream);

ms_status ms_multisplit_pairs(const uint32_t *keys_in, const uint32_t *vals_in,
                              uint32_t *keys_out, uint32_t *vals_out, uint64_t n,
                              const ms_bucket_fn *fn, uint32_t *bucket_offsets, void *ws,
                              size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------
 * Multisplit radix sort (Sec.7.1): ceil((end_bit-begin_bit) /
 * bits_per_pass) LSD passes of stable multisplit with radix-digit buckets,
 * the last pass narrower.  Result: keys ascending by the digit of
 * bits [begin_bit, end_bit) as unsigned integers; pairs stably ordered.
 *   0 <= begin_bit < end_bit <= 32, 1 <= bits_per_pass <= 8, or
 *   bits_per_pass = 0: the library's choice, 8 bits (measured on B200 at 2^28
 *   keys: 4 x 8-bit passes 88 Gkeys/s vs 7 x 5-bit 66 Gkeys/s, pairs 43 vs 38).
 * --------------------------------------------------------------------- */
size_t ms_radix_sort_workspace_size(uint64_t n, int with_values);

ms_status ms_radix_sort_keys(const uint32_t *keys_in, uint32_t *keys_out, uint64_t n,
                             uint32_t begin_bit, uint32_t end_bit, uint32_t bits_per_pass,
                             void *ws, size_t ws_bytes, void *stream);

ms_status ms_radix_sort_pairs(const uint32_t *keys_in, const uint32_t *vals_in,
                              uint32_t *keys_out, uint32_t *vals_out, uint64_t n,
                              uint32_t begin_bit, uint32_t end_bit, uint32_t bits_per_pass,
                              void *ws, size_t ws_bytes, void *stream);

/* Host-only: the LSD pass schedule (digit shifts and widths) used by
 * ms_radix_sort_* (bits_per_pass = 0: the library's choice, as above).
 * Writes at most `cap` entries; returns the pass count, or -1 on invalid
 * arguments. */
int ms_radix_pass_schedule(uint32_t begin_bit, uint32_t end_bit, uint32_t bits_per_pass,
                           uint32_t *shifts, uint32_t *bits, int cap);

/* ------------------------------------------------------------------------
 * Device-wide histogram (Sec.7.3 "GPU Histogram"): counts[j] =
 * number of samples in bucket j, j < m, m in 1..256.  `samples` (n binary32
 * values) and `counts` (m words, overwritten) are device pointers; stream-
 * ordered, no allocation, no synchronization.
 *   ms_histogram_even:  m buckets of width Delta = (upper - lower) / m between
 *     s_0 = lower and s_m = upper; bucket of x = floor((x - lower) /
 *     Delta) in binary32 round-to-nearest, clamped to m-1; samples outside
 *     [lower, upper) and NaN are not counted (readings R25-R26).
 *     MS_ERR_INVALID_VALUE unless lower < upper.
 *   ms_histogram_range: m+1 device splitters s_0 < s_1 < ... < s_m (strictly
 *     increasing; not checked); bucket of x = j with s_j <= x < s_{j+1}
 *     (upper-bound search); samples outside [s_0, s_m) not counted.
 * Errors: MS_ERR_UNSUPPORTED for m outside 1..256 or n >= 2^32,
 * MS_ERR_INVALID_VALUE for NULL pointers (samples may be NULL when n = 0).
 * --------------------------------------------------------------------- */
ms_status ms_histogram_even(const float *samples, uint64_t n, uint32_t m, float lower,
                            float upper, uint32_t *counts, void *stream);
ms_status ms_histogram_range(const float *samples, uint64_t n, uint32_t m,
                             const float *splitters, uint32_t *counts, void *stream);

/* Synchronizes `stream` and returns MS_ERR_KEY_DOMAIN if the most recent
 * multisplit that used `ws` saw an identity key >= m, else MS_SUCCESS. */
ms_status ms_device_status(const void *ws, void *stream);

/* ------------------------------------------------------------------------
 * Stage entry points (the three steps of P:529-540, exposed for per-stage
 * tests and timing).
 * --------------------------------------------------------------------- */

/* Elements per tile T (the subproblem reordered in shared memory) used by
 * the product path: 8192 for keys, 4096 for pairs. */
uint32_t ms_multisplit_tile_size(uint32_t m, int with_values);

/* Prescan (Alg.1): H[l*m + j] = |{i in tile l : f(u_i) = j}|
 * for the L = ceil(n/tile) subproblems of `tile` (>= 1) consecutive elements
 * (H is L*m words, device, tile-major). */
ms_status ms_stage_prescan(const uint32_t *keys_in, uint64_t n, const ms_bucket_fn *fn,
                           uint32_t *H, uint32_t tile, void *stream);

/* Scan (Alg.1): G = exclusive scan of the
 * row-vectorized (bucket-major) H, written tile-major like H (G may equal H).
 * bucket_offsets (m+1 words or NULL) receives the bucket starts and n_total.
 * ws: ms_stage_scan_workspace_size(L, m) bytes. */
size_t ms_stage_scan_workspace_size(uint64_t L, uint32_t m);
ms_status ms_stage_scan(const uint32_t *H, uint32_t *G, uint64_t L, uint32_t m,
                        uint32_t *bucket_offsets, void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------
 * Sharded multisplit (Eq.(3) P:408-427 with the GPUs as the first level of
 * localization, L_0 = G ranks).  Rank s holds input shard s (global elements
 * N_<s .. N_<s + n_s - 1) and receives output shard s (the same global index
 * range of the stable multisplit of the rank-order concatenation).  Per rank:
 *   1. local stable multisplit of the shard (ms_multisplit_*): local bucket
 *      order, bucket_offsets give the shard's counts C[s][j];
 *   2. all-gather of the counts C (G x m) over the process group;
 *   3. ms_shard_plan (host): all-to-all-v counts/displacements and the
 *      receiver's merge offsets;
 *   4. all-to-all-v of keys (and values): what rank s sends to rank d is one
 *      contiguous range of its local order (global positions are monotone in
 *      it);
 *   5. ms_shard_merge_* (device): each received element goes to
 *      merge_offsets[src][f(key)] + its index in the receive buffer.
 * --------------------------------------------------------------------- */

/* Host only.  C: G*m counts, row s = bucket counts of shard s.  For rank r:
 * send_counts/displs[d] (elements of r's local order sent to d, as a range),
 * recv_counts/displs[s] (elements received from s, packed in source order),
 * merge_offsets[s*m + j] (uint32, modulo 2^32) such that a received element e
 * (index in the packed receive buffer) from source s with bucket j lands at
 * output index merge_offsets[s*m + j] + e of rank r's output shard, and
 * global_bucket_offsets[0..m] (start of each bucket in the global output; may
 * be NULL).  Returns MS_SUCCESS or MS_ERR_INVALID_VALUE / MS_ERR_UNSUPPORTED
 * (a rank's shard >= 2^32 elements). */
ms_status ms_shard_plan(const uint64_t *C, uint32_t G, uint32_t m, uint32_t r,
                        uint64_t *send_counts, uint64_t *send_displs, uint64_t *recv_counts,
                        uint64_t *recv_displs, uint32_t *merge_offsets,
                        uint64_t *global_bucket_offsets);

/* Device merge (step 5): keys_recv/vals_recv (n_recv words, device) are the
 * packed receive buffers; recv_starts (G+1 uint32, device) the start of each
 * source's chunk (recv_starts[G] = n_recv); merge_offsets (G*m, device).
 * Writes keys_out/vals_out (n_recv words, the rank's output shard). */
ms_status ms_shard_merge_keys(const uint32_t *keys_recv, uint64_t n_recv, const ms_bucket_fn *fn,
                              const uint32_t *recv_starts, const uint32_t *merge_offsets,
                              uint32_t G, uint32_t *keys_out, void *stream);
ms_status ms_shard_merge_pairs(const uint32_t *keys_recv, const uint32_t *vals_recv,
                               uint64_t n_recv, const ms_bucket_fn *fn,
                               const uint32_t *recv_starts, const uint32_t *merge_offsets,
                               uint32_t G, uint32_t *keys_out, uint32_t *vals_out, void *stream);

/* ------------------------------------------------------------------------
 * Sharded multisplit as the library's own call (Eq.(3), with the
 * G ranks of one node as the first level of localization).  One process per
 * GPU; rank s holds input shard s (n_s elements, global indices N_<s ..
 * N_<s + n_s - 1 of the rank-order concatenation) and receives output shard s
 * (the same global index range of the stable multisplit of that
 * concatenation, so n_s elements too).  sum_s n_s must be < 2^32.
 *
 * NCCL is bound at run time (dlopen of libnccl.so.2: the process's copy, e.g.
 * PyTorch's); without it every call below returns MS_ERR_NCCL.
 *
 *   ms_comm_unique_id  rank 0 only: 128 opaque bytes the caller broadcasts
 *                      (e.g. over a torch.distributed process group).
 *   ms_comm_init       collective over the G ranks (G <= 8): binds the
 *                      current process to `cuda_device` and creates the NCCL
 *                      communicator.  ms_comm_destroy releases everything.
 *   ms_comm_register_output
 *                      collective, synchronous: registers this rank's output
 *                      buffers (n_local words each; vals_out may be NULL) as
 *                      windows the other ranks map through CUDA IPC (buffers
 *                      from cudaMalloc or a caching allocator on top of it).
 *   ms_multisplit_{keys,pairs}_sharded
 *                      collective, stream-ordered on `stream`.  When keys_out
 *                      (and vals_out) are the registered windows and n_local
 *                      their size, the fused path KP runs: local prescan ->
 *                      NCCL all-gather of the G x m bucket counts -> plan
 *                      kernel (Eq.3 terms 1-2 per bucket) -> postscan that
 *                      stores every element straight into the window of the
 *                      rank owning its global position (NVLink peer stores;
 *                      no staging, no merge, no host synchronization) -> an
 *                      NCCL all-reduce of one word as the completion barrier.
 *                      Otherwise the NCCL path runs: local multisplit into the
 *                      workspace -> all-gather of the offsets -> one D2H copy +
 *                      stream synchronization -> host plan (ms_shard_plan) ->
 *                      ncclSend / ncclRecv of contiguous ranges -> KX merge.
 *                      KP needs m <= 32, or the device's lane-order probe
 *                      (ms_device_init) for m > 32; else the NCCL path runs.
 *                      global_bucket_offsets: NULL or m+1 device uint64 words
 *                      (start of each bucket in the global output, [m] = n_total).
 *   ms_sharded_workspace_size: bytes of `ws` (256-byte aligned) for either path.
 * --------------------------------------------------------------------- */
typedef struct ms_comm ms_comm;
ms_status ms_comm_unique_id(void *out128);
ms_status ms_comm_init(ms_comm **comm, int nranks, int rank, const void *id128, int cuda_device);
ms_status ms_comm_destroy(ms_comm *comm);
/* Failure detection: ms_comm_check returns MS_ERR_NCCL if the
 * communicator reported an asynchronous error (ncclCommGetAsyncError), e.g. a
 * peer that died; ms_comm_abort then aborts the NCCL communicator
 * (ncclCommAbort) so that no collective blocks forever -- the caller still
 * calls ms_comm_destroy.  Both are host-only and do not synchronize. */
ms_status ms_comm_check(ms_comm *comm);
ms_status ms_comm_abort(ms_comm *comm);
ms_status ms_comm_register_output(ms_comm *comm, uint32_t *keys_out, uint32_t *vals_out,
                                  uint64_t n_local);
size_t ms_sharded_workspace_size(const ms_comm *comm, uint64_t n_local, uint32_t m, int with_values);
ms_status ms_multisplit_keys_sharded(ms_comm *comm, const uint32_t *keys_in, uint32_t *keys_out,
                                     uint64_t n_local, const ms_bucket_fn *fn,
                                     uint64_t *global_bucket_offsets, void *ws, size_t ws_bytes,
                                     void *stream);
ms_status ms_multisplit_pairs_sharded(ms_comm *comm, const uint32_t *keys_in, const uint32_t *vals_in,
                                      uint32_t *keys_out, uint32_t *vals_out, uint64_t n_local,
                                      const ms_bucket_fn *fn, uint64_t *global_bucket_offsets,
                                      void *ws, size_t ws_bytes, void *stream);

/* The two steps of the fused path KP without the collectives, so that G
 * "virtual ranks" can run on one GPU (the collectives become copies):
 *   ms_shard_prescan: prescan of this rank's shard into `ws` (which must then
 *     be passed unchanged to ms_shard_scatter); counts (m device words, may be
 *     NULL) receives the shard's bucket counts C[r][0..m).
 *   ms_shard_scatter: C = the G x m gathered counts (device, row s = rank s);
 *     peer_keys / peer_vals = host arrays of G device pointers, the output
 *     shard of every rank (peer_vals NULL: keys only; an entry may be NULL
 *     for a rank whose shard is empty); writes this rank's
 *     elements into the owners' shards and, if global_bucket_offsets is not
 *     NULL, the m+1 global bucket starts (uint64, device).
 * ws: ms_shard_workspace_size(n_local, m, G, with_values) bytes.  Errors as
 * for ms_multisplit_*, and MS_ERR_UNSUPPORTED for m > 32 on a device whose
 * lane-order probe has not passed. */
size_t ms_shard_workspace_size(uint64_t n_local, uint32_t m, uint32_t G, int with_values);
ms_status ms_shard_prescan(const uint32_t *keys_in, uint64_t n_local, const ms_bucket_fn *fn,
                           int with_values, uint32_t G, uint32_t *counts, void *ws, size_t ws_bytes,
                           void *stream);
ms_status ms_shard_scatter(const uint32_t *keys_in, const uint32_t *vals_in, uint64_t n_local,
                           const ms_bucket_fn *fn, const uint32_t *C, uint32_t G, uint32_t rank,
                           uint32_t *const *peer_keys, uint32_t *const *peer_vals,
                           uint64_t *global_bucket_offsets, void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------
 * Multisplit-SSSP (Sec.7.2): single-source shortest paths by
 * delta-stepping with the Bucketing strategy, the bucketing
 * step being ms_multisplit_pairs with splitter buckets.  Each
 * iteration splits the work list (key = tentative distance, value = vertex)
 * into K buckets of width `delta` starting at the smallest tentative distance
 * (the last bucket takes everything beyond), relaxes the out-edges of bucket
 * 0's up-to-date items (atomicMin on dist) and appends every improvement to
 * the carried-over buckets 1..K-1.  The loop ends when the work list is empty.
 *
 *   row_ptr (V+1), col (E), w (E)   CSR graph in device memory, weights >= 0;
 *                                   E < 2^32; parallel edges and self loops
 *                                   are allowed.
 *   source < V, delta >= 1, 1 <= K <= 256 (the paper's best K is 10).
 *   dist (V words, device)          shortest distances; 0xFFFFFFFF =
 *                                   unreachable.  Every shortest distance must
 *                                   be < 2^32 - 1 (sums are saturated).
 *   ws                              ms_sssp_workspace_size(V, E, K) bytes,
 *                                   256-byte aligned (the work lists hold
 *                                   2E + V + 1024 items; MS_ERR_WORKSPACE if a
 *                                   graph ever needs more).
 *   stats                           NULL or host struct: iterations, work-list
 *                                   items multisplit, frontier items, pushes.
 * SYNCHRONIZES `stream` once per iteration (the work-list length is read back),
 * so it cannot be captured in a CUDA graph.
 * --------------------------------------------------------------------- */
typedef struct {
  uint64_t iterations, items, frontier, pushes;
} ms_sssp_stats;
size_t ms_sssp_workspace_size(uint32_t V, uint64_t E, uint32_t K);
ms_status ms_sssp(const uint32_t *row_ptr, const uint32_t *col, const uint32_t *w, uint32_t V,
                  uint64_t E, uint32_t source, uint32_t delta, uint32_t K, uint32_t *dist, void *ws,
                  size_t ws_bytes, void *stream, ms_sssp_stats *stats);

/* ------------------------------------------------------------------------
 * Instrumentation (host only, thread-local, zero cost when unset).
 * --------------------------------------------------------------------- */

/* Stage timing hooks: `events` is NULL (off) or points to 4 cudaEvent_t
 * handles (passed as void*) that every subsequent multisplit call made by
 * this host thread records on its stream: [0] before the prescan, [1] before
 * the scan, [2] before the postscan, [3] after the postscan.  The single-CTA
 * path (n <= tile) records [0]=[1]=[2] before and [3] after its one launch.
 * The array must stay valid until hooks are cleared. */
void ms_set_stage_events(void *const *events);

/* Number of kernels this library has launched since load (all threads). */
uint64_t ms_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* MULTISPLIT_H_ */
