// gi_internal.cuh — shared internals of the CUDA library (not part of the ABI).
//
// Data layout in HBM. All internal arrays use the library's
// vertex numbering: by default vertices are relabelled by out-degree
// (descending, ties by input id) so that the hottest sources form a dense
// prefix; `perm[new] = input id`, `inv[input id] = new`. Results are always
// reported in input ids.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <utility>
#include <vector>

#include "gi.h"

namespace gi {

// ------------------------------------------------------------------ errors
void set_error(const std::string& msg);
gi_status fail(gi_status s, const std::string& msg);
gi_status cuda_fail(cudaError_t e, const char* what, const char* file, int line);

#define GI_CUDA(call)                                                        \
  do {                                                                       \
    cudaError_t e__ = (call);                                                \
    if (e__ != cudaSuccess) return ::gi::cuda_fail(e__, #call, __FILE__, __LINE__); \
  } while (0)

#define GI_TRY(call)                    \
  do {                                  \
    gi_status s__ = (call);             \
    if (s__ != GI_OK) return s__;       \
  } while (0)

// ------------------------------------------------------------------ device buffer
// RAII device allocation (cudaMalloc; freed on destruction).
// Allocations of up to kPoolMaxBlock bytes inside a library call are
// stream-ordered on the context's stream (cudaMallocAsync / cudaFreeAsync from
// the device's pool, which keeps up to kPoolKeep bytes cached), so the temporaries of a graph build or a layout
// build, and a graph's buffers after gi_graph_destroy, are reused instead of
// going back to cudaMalloc / cudaFree. AllocScope sets the stream for the
// calling thread; outside a scope (or with GI_POOL=0) DevBuf uses cudaMalloc.
constexpr uint64_t kPoolKeepDefault = 16ull << 30;
inline uint64_t pool_keep() {  // GI_POOL_KEEP_GB overrides (A/B runs)
  static const uint64_t v = getenv("GI_POOL_KEEP_GB") ? (uint64_t)atoll(getenv("GI_POOL_KEEP_GB")) << 30 : kPoolKeepDefault;
  return v;
}
// larger buffers go through the per-process cache of cudaMalloc'd blocks below:
// in steady state (the same sizes call after call) no allocation reaches the
// driver. Pool growth alone measured 10-700 ms per cudaMallocAsync on config 4's
// end-to-end steps (even for 24 MB, whatever the release threshold), and the
// pool re-maps multi-GB blocks around synchronisations
constexpr size_t kPoolMaxBlockDefault = 8ull << 20;
inline size_t pool_max_block() {  // GI_POOL_MAX_MB overrides (A/B runs)
  static const size_t v = getenv("GI_POOL_MAX_MB") ? (size_t)atoll(getenv("GI_POOL_MAX_MB")) << 20 : kPoolMaxBlockDefault;
  return v;
}
inline cudaStream_t& tl_alloc_stream() {
  static thread_local cudaStream_t s = nullptr;
  return s;
}
inline bool pool_enabled() {
  static const bool on = !getenv("GI_POOL") || atoi(getenv("GI_POOL")) != 0;
  return on;
}
struct AllocScope {
  cudaStream_t prev;
  explicit AllocScope(cudaStream_t s) : prev(tl_alloc_stream()) { tl_alloc_stream() = s; }
  ~AllocScope() { tl_alloc_stream() = prev; }
  AllocScope(const AllocScope&) = delete;
  AllocScope& operator=(const AllocScope&) = delete;
};

// Large buffers (above the pool's block limit: the temporaries of a
// billion-edge build or layout build) are cudaMalloc'd; freeing one returns it
// to a per-process cache keyed by (device, stream) instead of cudaFree, and an
// allocation on the same stream reuses a cached block of 1 to 2x its size.
// Reuse is stream-ordered (every user of a block is on the same stream), so no
// synchronisation is needed; cudaMalloc / cudaFree of multi-GB blocks cost
// 10-400 ms each and stall the device (DESIGN §6 e2e). The cache holds at most
// GI_BIGCACHE_GB (default 120) GB and never leaves less than 24 GB of the device
// free (other allocators), frees its oldest blocks one by one while an allocation fails, and the blocks
// of a stream are freed when its context is destroyed.
void* big_cache_get(size_t nbytes, cudaStream_t s, size_t* got);
void big_cache_put(void* p, size_t bytes, cudaStream_t s);
void big_cache_flush(cudaStream_t s);  // s = nullptr: every stream of the current device
void big_cache_note_malloc();          // a large block was cudaMalloc'd (the cache re-checks free memory)
bool big_cache_evict_one();            // frees the oldest cached block of the device (false: none left)
// diagnostics: GI_DEBUG_SLOW_MS=t prints every allocation / free that takes longer than t ms
double slow_ms();
void slow_report(const char* what, size_t bytes, std::chrono::steady_clock::time_point t0);

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;  // stream of a pooled / cached allocation (freed on / returned for it)
  bool pooled = false;
  bool cached = false;       // a large block owned by the big-buffer cache protocol
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { reset(); }
  void reset() {
    if (p) {
      const auto t0 = std::chrono::steady_clock::now();
      if (pooled) cudaFreeAsync(p, s);
      else if (cached) big_cache_put(p, cap, s);
      else cudaFree(p);
      if (slow_ms() > 0) slow_report(pooled ? "cudaFreeAsync" : cached ? "big_cache_put" : "cudaFree", cap, t0);
    }
    p = nullptr;
    bytes = 0;
    cap = 0;
    pooled = false;
    cached = false;
  }
  // plain = true: always cudaMalloc (memory that is exported to peers by CUDA IPC)
  gi_status alloc(size_t nbytes, bool plain = false) {
    reset();
    if (nbytes == 0) nbytes = 16;
    const cudaStream_t st = tl_alloc_stream();
    cudaError_t e = cudaSuccess;
    const auto t0 = std::chrono::steady_clock::now();
    if (!plain && st && pool_enabled() && nbytes <= pool_max_block()) {
      e = cudaMallocAsync(&p, nbytes, st);
      pooled = e == cudaSuccess;
      s = st;
    } else if (!plain && st && pool_enabled()) {
      size_t got = 0;
      p = big_cache_get(nbytes, st, &got);
      if (!p) {
        e = cudaMalloc(&p, nbytes);
        while (e != cudaSuccess && big_cache_evict_one()) {  // memory held by the cache: free the
          cudaGetLastError();                                // oldest blocks until the allocation fits
          e = cudaMalloc(&p, nbytes);
        }
        got = nbytes;
        if (e == cudaSuccess) big_cache_note_malloc();
      }
      if (e == cudaSuccess) {
        cached = true;
        cap = got;
        s = st;
      }
    } else {
      e = cudaMalloc(&p, nbytes);
    }
    if (e != cudaSuccess) {
      p = nullptr;
      pooled = false;
      cached = false;
      cudaGetLastError();
      return fail(GI_ERR_OUT_OF_MEMORY, "cudaMalloc of " + std::to_string(nbytes) + " bytes failed: " +
                                            cudaGetErrorString(e));
    }
    bytes = nbytes;
    if (!cached) cap = nbytes;
    if (slow_ms() > 0) slow_report(pooled ? "cudaMallocAsync" : cached ? "big alloc" : "cudaMalloc", nbytes, t0);
    return GI_OK;
  }
  size_t cap = 0;  // bytes of the underlying block (>= bytes for a reused cached block)
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

}  // namespace gi

// ------------------------------------------------------------------ context / graph
struct NcclApi;  // dynamically loaded NCCL entry points (nccl_dyn.cu)
namespace gi {
struct Comm;  // comm.cuh
}

struct gi_context_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int rank = 0, nranks = 1;
  void* nccl_comm = nullptr;  // ncclComm_t when nranks > 1 (NCCL contexts)
  gi::Comm* comm = nullptr;   // exchange layer when nranks > 1 (NCCL or in-process local group)
  int num_sms = 148;
  // pinned host scratch for small D2H reads (counters)
  int64_t* h_scratch = nullptr;
  int64_t* h_batch = nullptr;  // pinned per-source state slots of gi_bfs_multi
  int64_t h_batch_len = 0;
  int live_graphs = 0;  // graphs created on this context and not yet destroyed
  cudaStream_t copy_stream = nullptr;  // host-edge H2D chunks of gi_graph_create (created on first use)
};

// Pull-PageRank tiling (merge-path over CSC rows + edges).
constexpr int kPullThreads = 256;
constexpr int kPullItemsPerThread = 8;
constexpr int kPullTile = kPullThreads * kPullItemsPerThread;  // merge items per tile

struct gi_graph_s {
  gi_context ctx = nullptr;
  int64_t n = 0;       // vertices (global)
  int64_t m = 0;       // directed edges after cleanup (global)
  // 1-D destination partition; single GPU: r0 = 0, nr = n, ml = m.
  // CSC rows = owned destinations [r0, r0 + nr) (local row = id - r0); the CSR
  // rows are all n sources but hold only the edges into the owned range.
  int64_t r0 = 0, nr = 0, ml = 0;
  std::vector<int64_t> bounds;  // nranks + 1 owner boundaries (multiples of 32)
  bool off64 = false;  // offsets stored as int64 (m >= 2^31) else int32
  bool relabeled = false;
  // vertex relabelling (n each; empty when !relabeled)
  gi::DevBuf perm, inv;
  // CSR (out-edges) and CSC (in-edges) in internal ids
  gi::DevBuf csr_off, csr_idx, csc_off, csc_idx;
  gi::DevBuf outdeg;  // int32[n], internal ids
  // pull tiling: first/last row of each merge-path tile (int32 pairs)
  int64_t ntiles = 0;
  int max_indeg = -1;  // longest CSC row (owned rows), computed on first use
  gi::DevBuf tile_rows;
  // PageRank workspace
  gi::DevBuf contrib[2];  // float[n]
  gi::DevBuf dbuf;        // double[4]: dangling-mass ring
  gi::DevBuf split_acc;   // double[n]: partial sums of rows split across tiles
  gi::DevBuf split_cnt;   // int32[n]: arrival counters for split rows
  gi::DevBuf push_sum;    // double[n]: push-form accumulator
  // segmented pull (pr_segmented.cu); seg_Z == 0 until built
  int seg_Z = 0, seg_S = 0, seg_U = 0, seg_ctas = 0;  // segment size, segments, units, CTAs
  int64_t seg_DB = 0, seg_P = 0, seg_C = 0;          // rows per destination block, pieces, records
  gi::DevBuf seg_rec;      // records: long (lane-aligned) and short (lane-per-piece), pr_segmented.cu
  gi::DevBuf seg_unit_c0;  // int32[U+1]: first record of each (block, segment) unit
  gi::DevBuf seg_cta;      // int32[CTAs+1]: cost-balanced record range of each CTA
  std::vector<int32_t> seg_h_cta;  // host copy of seg_cta's record starts
  std::vector<int32_t> seg_h_uc;   // host copy of seg_unit_c0
  std::vector<int64_t> seg_h_model;  // prefix of the per-record cost model (C + 1)
  gi::DevBuf seg_time;     // uint64[4*CTAs]: per-CTA timings of the last calibrated launch
  gi::DevBuf seg_ht;       // uint64[CTAs]: {tail, head} of each CTA's remaining record range (work stealing)
  int seg_calib = 0;       // edge passes left that re-balance the CTA ranges from measured timings
  int seg_steal = 0;       // CTAs steal records from each other's ranges (large layouts)
  gi::DevBuf seg_acc;      // float[2][seg_acc_stride]: per-row sums (ping-pong), L2-resident
  int64_t seg_acc_stride = 0;
  int seg_acc_cur = 0;     // buffer the next edge pass reduces into (all zero)
  // source-partitioned pull (pagerank.cu; the paper's cache partitioning):
  // the CSC's edges grouped by source range [p << sp_shift, (p+1) << sp_shift),
  // each group a CSC of its own (offsets sp_off + p * (nr+1), edges sp_idx +
  // sp_base[p], merge-path tiles sp_tiles + 2 * sp_tile0[p]); sp_P == 0 until built
  int sp_P = 0, sp_shift = 0;
  bool sp_off64 = false;
  std::vector<int64_t> sp_m, sp_base, sp_ntiles, sp_tile0;
  gi::DevBuf sp_idx, sp_off, sp_tiles, sp_acc;
  int pr_auto = -1;       // auto-selected pull kernel, decided on first use
  // propagation-blocked pull (pr_blocked.cu); pb_Ks == 0 until built
  int pb_Ks = 0, pb_Kd = 0, pb_nitems = 0;
  int64_t pb_mp = 0;
  double pb_epp = 0.0;    // edges per segmented-pull piece (the auto choice's statistic)
  gi::DevBuf pb_rb, pb_tstart, pb_src, pb_dst, pb_vals, pb_items;
  // multi-GPU PageRank with peer stores: every rank's
  // contrib[k] replica as seen from this rank (index = rank; own entry = local)
  int peer_state = 0;                 // 0 unknown, 1 mapped, -1 unavailable (allgather path)
  std::vector<void*> peer_c[2];
  std::vector<void*> peer_opened;     // CUDA IPC mappings to close on destroy
  // multi-GPU BFS with peer stores: a ring of 3 frontier bitmaps (cudaMalloc, IPC-exported)
  // and every rank's replicas of them
  int bfs_peer_state = 0;             // 0 unknown, 1 mapped, -1 unavailable (allgather path)
  gi::DevBuf bfs_ring[3];
  std::vector<void*> bfs_peer_bm[3];
  std::vector<void*> bfs_peer_opened;
  gi::DevBuf out_stage;   // float/int32[n]: output staging in input ids
  // BFS workspace
  gi::DevBuf parent;      // int32[n], internal ids
  gi::DevBuf queue[2];    // int32[n]
  gi::DevBuf bitmap[2];   // uint32[ceil(n/32)]
  gi::DevBuf counters;    // int64 slots, see bfs.cu
  gi::DevBuf bfs_pre;     // int64[n+1]: scan of frontier degrees (balanced push)
  gi::DevBuf bfs_scan_tmp;
  gi::DevBuf bfs_cand;    // uint64[n]: (epoch << 32 | parent candidate), stamp + collect push
  struct {                // fused cooperative BFS (bfs_fused.cu)
    bool ready = false;
    bool cluster = false;  // the small grid runs as one thread-block cluster
    int dyn = 0, grid = 0;
    gi::DevBuf stamp, q[2], bm[3], cnt, pre, ctot;  // stamp[v] == epoch: visited by the current source
    gi::DevBuf vinfo;                                // int2 {input id, out-degree} per internal id
    gi::DevBuf msrc, mstates, mstage;                // gi_bfs_multi: sources, final states, host-output staging
    uint32_t epoch = 0;
  } fused;
  unsigned bfs_epoch = 0;
  struct {  // bit-parallel multi-source BFS (msbfs.cu)
    gi::DevBuf seen, fr[2], act[2], cnt, src, heavy, par, par8, hidx, csc_in;
    gi::DevBuf fc;       // the frontier masks narrowed to 16 / 32 bits for the pull gathers (k <= 32)
    gi::DevBuf fc32, acc32, rlist;  // segmented OR pull: 32-bit masks, OR accumulator, heavy rows to resolve
    gi::DevBuf fc32hi, acc32hi;      // segmented OR pull, k > 32: the masks' upper halves and their OR
    gi::DevBuf hlist;                // sparse row pulls: the heavy chunks of rows still missing a source
    gi::DevBuf tsum;                 // push levels: tile sums of the out-degree prefix
    int64_t nheavy = 0;  // rows with in-degree >= 32 (pulled by whole warps)
    gi::DevBuf hch;      // their chunks: int2 (row, first in-edge offset)
    int64_t nhch = 0;
    gi::DevBuf chunks[2], scan_tmp;  // push: chunk counts / inclusive prefix, cub scan scratch
    size_t scan_bytes = 0;
  } ms;
  struct {  // connected components / SSSP (cc.cu): labels or distances, frontier bitmaps, edge weights
    gi::DevBuf ids, bm[2], wcsr, wcsc, acc;
    bool w_ready = false;
    uint64_t w_seed = 0;
  } ccs;
};

namespace gi {
// host-side partition of [0, n) into nranks ranges of ~equal weight, cut at
// multiples of 32 (bitmap words); prefix(i) = sum of weights of vertices < i.
void partition_ranges(int64_t n, int nranks, int64_t (*prefix)(void*, int64_t), void* ctx, int64_t* bounds);
// build.cu
gi_status build_graph_dist(gi_context ctx, int64_t n, int64_t m0, const int32_t* d_src,
                           const int32_t* d_dst, uint32_t flags, gi_graph g);
gi_status build_graph(gi_context ctx, int64_t n, int64_t m0, const int32_t* d_src,
                      const int32_t* d_dst, uint32_t flags, gi_graph g);
// host edges (pinned for overlap): the H2D copy in chunks on the context's copy
// stream, overlapped with the histogram, key making and per-chunk sorts
gi_status build_graph_host(gi_context ctx, int64_t n, int64_t m0, const int32_t* h_src, const int32_t* h_dst,
                           uint32_t flags, gi_graph g);
bool build_host_pipelined(gi_context ctx, int64_t m0, uint32_t flags);
// pagerank.cu
gi_status pagerank_run(gi_graph g, int32_t iters, double damping, const gi_pr_opts& o,
                       float* d_out_input_ids, gi_pr_stats* stats);
// pr_segmented.cu
struct PrArgs;
// the segment size the segmented pull uses on this device
gi_status seg_default_Z(gi_graph g, int* Z);
// pr_blocked.cu: propagation-blocked pull (layout once per graph; one iteration = 2 launches)
gi_status pb_build(gi_graph g);
gi_status pb_count_pieces(gi_graph g, int Z, int64_t* pieces);
// mid: recorded between the scatter and the gather (profiling; may be null)
gi_status pb_iteration(gi_graph g, const PrArgs& A, cudaEvent_t mid);
// segment_size / block_rows: 0 = automatic (tests pass small values)
gi_status seg_build(gi_graph g, int segment_size, int64_t block_rows);
// merge-path tile rows of a CSC (build.cu); rows: int32[2 * ntiles]
gi_status tile_rows_launch(const void* off, bool off64, int64_t n, int64_t m, int64_t ntiles, int32_t* rows,
                           cudaStream_t st, int sms);
// seg_acc_buf(g, cur)[v] = sum of cin over v's in-edges (the buffer is zero before the pass)
gi_status seg_edge_pass(gi_graph g, const float* cin);
int64_t seg_record_bytes();  // bytes per record of the segmented layout
// a min pass over the segmented layout: acc[v] = min(acc[v], labels[u] over in-edges (u, v)) (CC, cc.cu)
gi_status seg_min_pass(gi_graph g, const int32_t* labels, int32_t* acc);
gi_status seg_or_pass(gi_graph g, const uint32_t* masks, uint32_t* acc);
// bit-parallel BFS / CC shared state (g->ms): masks, active lists, heavy-row chunks
gi_status ms_prepare(gi_graph g);
// out-degree of an active vertex, as a scan input (the push levels' degree prefix
// is one cub scan over the active list through this functor: no separate pass)
struct OutdegOf {
  const int32_t* outdeg;
  __host__ __device__ __forceinline__ long long operator()(int32_t v) const { return (long long)outdeg[v]; }
};
gi_status cc_run(gi_graph g, const gi_cc_opts& o, int32_t* d_out, gi_cc_stats* stats);  // cc.cu
// SSSP weights: synthetic from `seed` (R24), or w_user != nullptr: device int32[m]
// in the edge order of csr_input_ids / gi_graph_csr
gi_status sssp_run(gi_graph g, int32_t source, uint64_t seed, const int32_t* w_user, const gi_cc_opts& o,
                   int32_t* d_out, gi_cc_stats* stats);  // cc.cu
// the cleaned CSR in input ids on the device (gi_api.cu)
gi_status csr_input_ids(gi_graph g, DevBuf& doff, DevBuf& didx);
// the two accumulators: cur holds the sums of the last edge pass; the other is zero
inline float* seg_acc_buf(gi_graph g, int which) { return g->seg_acc.as<float>() + which * g->seg_acc_stride; }
// vertex update from the current accumulator; zeroes the other one (never a
// load and a store to the same line: that stalls on L2 misses) and flips them
gi_status seg_vertex_pass(gi_graph g, const PrArgs& A);
// prdelta.cu
gi_status prdelta_run(gi_graph g, int32_t iters, double damping, double eps, const gi_prdelta_opts& o, float* d_out,
                      gi_prdelta_stats* stats);
// bfs.cu / bfs_fused.cu
gi_status bfs_fused(gi_graph g, int32_t source_input_id, const gi_bfs_opts& o, int32_t* d_parent_input_ids,
                    gi_bfs_stats* stats);
// k sources in one launch (single GPU); d_out: device rows out_stride apart
gi_status bfs_fused_multi(gi_graph g, int32_t k, const int32_t* sources, const gi_bfs_opts& o, int32_t* d_out,
                          int64_t out_stride, gi_bfs_stats* stats);
// msbfs.cu: k sources, 64 per bit-parallel pass; d_out: k device rows of n
gi_status msbfs_run(gi_graph g, int32_t k, const int32_t* sources, const gi_bfs_opts& o, int32_t* d_out,
                    gi_bfs_stats* stats);
gi_status bfs_finish_output(gi_graph g, const int32_t* parent_internal, int32_t* d_out, int64_t* reached,
                            int64_t* edges);
gi_status bfs_run(gi_graph g, int32_t source_input_id, const gi_bfs_opts& o,
                  int32_t* d_parent_input_ids, gi_bfs_stats* stats);
// Low-latency wait for the stream: spin on cudaStreamQuery instead of a
// blocking synchronise (which may yield the thread and add tens of µs of
// wake-up latency to every BFS level's host round trip).
inline cudaError_t stream_wait(cudaStream_t st) {
  cudaError_t e;
  while ((e = cudaStreamQuery(st)) == cudaErrorNotReady) {
  }
  return e;
}
// util
inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
// launch with programmatic stream serialization (the kernel calls griddepcontrol.wait
// before touching its predecessor's data); GI_PDL=0 turns it off for A/B runs
template <typename... KArgs, typename... Args>
inline gi_status launch_pdl(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t st,
                            Args&&... args) {
  static const bool on = !getenv("GI_PDL") || atoi(getenv("GI_PDL")) != 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = on ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  GI_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
  return GI_OK;
}

inline int grid_for(int64_t work, int threads, int num_sms, int per_sm = 8) {
  int64_t g = ceil_div(work, threads);
  int64_t cap = (int64_t)num_sms * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}
}  // namespace gi
