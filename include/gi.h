/*
 * gi.h — C ABI of the B200-native edgeset.apply library (GraphIt hot path).
 *
 * The library implements the paper's edge-traversal operator
 *     edges.from(frontier).to(filter).apply(f)
 * in its pull (DensePull, CSC gather), push (SparsePush / DensePush, CSR
 * scatter with atomics) and direction-optimising hybrid (DensePull-SparsePush,
 * P:661-675) forms, instantiated for fixed-iteration PageRank (P:855-856,
 * P:2286, vertex update P:3242-3253 [draft]) and BFS (parent vector
 * initialised to -1; applyModified without dedup).
 *
 * Conventions for every function:
 *   - returns gi_status; never throws, never exits, never prints;
 *   - on error, a thread-local message is available from gi_last_error()
 *     until the next call from the same thread; outputs are unspecified and
 *     any graph passed in stays valid;
 *   - calls are stream-ordered on the context's CUDA stream and RETURN AFTER
 *     COMPLETION (the stream is synchronised before returning); asynchronous
 *     CUDA faults surface at that synchronisation as GI_ERR_CUDA;
 *   - pointer arguments may be host or device memory unless stated; the
 *     library detects which with cudaPointerGetAttributes and copies as needed;
 *   - input arrays are borrowed for the duration of the call (copied);
 *     outputs are caller-allocated with the stated length.
 * There is no CPU fallback: without a usable CUDA device every call that
 * needs one fails with GI_ERR_CUDA.
 */
#ifndef GI_H_
#define GI_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GI_ABI_VERSION 3

#if defined(__GNUC__)
#define GI_API __attribute__((visibility("default")))
#else
#define GI_API
#endif

typedef enum {
  GI_OK = 0,
  GI_ERR_INVALID_ARGUMENT = 1,  /* null pointer, negative size, bad flag/option */
  GI_ERR_VERTEX_OUT_OF_RANGE = 2, /* an endpoint or source not in [0, n) */
  GI_ERR_OUT_OF_MEMORY = 3,     /* device or host allocation failed */
  GI_ERR_CUDA = 4,              /* CUDA runtime error (incl. async faults) */
  GI_ERR_NCCL = 5,              /* NCCL missing or a collective failed */
  GI_ERR_UNSUPPORTED = 6,       /* valid request this build cannot serve */
  GI_ERR_INTERNAL = 7           /* invariant violated inside the library */
} gi_status;

typedef struct gi_context_s* gi_context; /* device, CUDA stream, optional NCCL comm */
typedef struct gi_local_group_s* gi_local_group; /* in-process simulated ranks (tests) */
typedef struct gi_graph_s* gi_graph;     /* device CSR + CSC + degrees (+ partition) */

/* ---------------------------------------------------------------- context */

/* device: CUDA ordinal. cuda_stream: a cudaStream_t to order all work on, or
 * NULL for a stream owned by the context. */
GI_API gi_status gi_context_create(int device, void* cuda_stream, gi_context* out);

/* Multi-GPU (one process per GPU): rank 0 calls
 * gi_nccl_unique_id, broadcasts the 128 bytes (e.g. with torch.distributed),
 * then every rank calls gi_context_create_dist. NCCL is loaded at run time
 * (dlopen "libnccl.so.2"); GI_ERR_NCCL if it cannot be.
 * PageRank exchanges contrib slices with an NCCL allgatherv every iteration.
 * With GI_PR_PEER=1 it instead maps every rank's contrib replicas once per
 * graph (CUDA IPC) and stores new contrib values straight into them from the
 * vertex update (no per-iteration allgather); the ranks
 * agree on the choice (an allreduce: peer stores only if every rank asks for
 * them and every rank can map), else all use the allgatherv. Peer stores are
 * tested across processes sharing one GPU (gi_context_create_hostcomm) and
 * with in-process ranks, NOT across GPUs over NVLink (no multi-GPU box here).
 * gi_graph_destroy is then collective: every rank closes its mappings, then
 * all ranks meet at a barrier before any frees the mapped buffers. */
GI_API gi_status gi_nccl_unique_id(unsigned char id[128]);
GI_API gi_status gi_context_create_dist(int device, void* cuda_stream, int rank, int nranks,
                                 const unsigned char id[128], gi_context* out);
GI_API gi_status gi_context_destroy(gi_context ctx);
GI_API gi_status gi_context_rank(gi_context ctx, int* rank, int* nranks);

/* Multi-process contexts over ANY transport: the multi-GPU path's collectives
 * (allreduce of degree histograms and scalars, allgatherv of
 * contrib / bitmap / parent slices, alltoallv of the build's owner shuffle)
 * staged through host memory and performed by the caller's callbacks, e.g.
 * torch.distributed over gloo. Each callback returns 0 on success; it is
 * called on the thread making the library call, with host buffers valid for
 * the duration of the callback:
 *   allreduce(user, buf, count, dtype): in-place element-wise SUM over ranks of
 *     `count` elements, dtype GI_DT_INT32 / GI_DT_INT64 / GI_DT_F64;
 *   allgatherv(user, buf, off, nranks): `buf` holds off[nranks] bytes; on
 *     return bytes [off[q], off[q+1]) must hold rank q's bytes (this rank's
 *     own range is filled on entry);
 *   alltoallv(user, send, soff, recv, roff, nranks): send bytes
 *     [soff[q], soff[q+1]) to rank q; receive rank q's bytes into
 *     recv + [roff[q], roff[q+1]) (counts agree pairwise).
 * Ranks may share a device (no kernel waits on another rank: every collective
 * synchronises the stream first). PageRank peer stores (CUDA IPC, handles
 * exchanged through allgatherv) are used only with GI_PR_PEER=1 on every rank.
 * The struct is copied; `user` must stay valid until gi_context_destroy. */
enum { GI_DT_INT32 = 0, GI_DT_INT64 = 1, GI_DT_F64 = 2 };
typedef struct {
  void* user;
  int (*allreduce)(void* user, void* buf, int64_t count, int32_t dtype);
  int (*allgatherv)(void* user, void* buf, const int64_t* off, int32_t nranks);
  int (*alltoallv)(void* user, const void* send, const int64_t* soff, void* recv, const int64_t* roff,
                   int32_t nranks);
} gi_host_comm;
GI_API gi_status gi_context_create_hostcomm(int device, void* cuda_stream, int rank, int nranks,
                                            const gi_host_comm* comm, gi_context* out);

/* Test hook for the partitioned path on ONE GPU: nranks simulated ranks,
 * each driven by its own host thread with its own context created by
 * gi_context_create_local(device, stream, group, rank). Every collective of the
 * multi-GPU path (allreduce, allgatherv, alltoallv) is performed by device
 * copies between the ranks' buffers plus a host barrier; no kernel waits on
 * another rank. All ranks must make the same calls in the same order, as with
 * NCCL. Destroy the group after every context of it. */
GI_API gi_status gi_local_group_create(int nranks, gi_local_group* out);
GI_API gi_status gi_local_group_destroy(gi_local_group grp);
GI_API gi_status gi_context_create_local(int device, void* cuda_stream, gi_local_group grp, int rank,
                                  gi_context* out);

/* Host-only helper (no device): the 1-D destination partition the multi-GPU
 * build uses: bounds[0] = 0 <= bounds[1] <= ... <= bounds[nranks] = n,
 * inner bounds multiples of 32 (whole frontier-bitmap words), each range
 * holding ~1/nranks of the total weight; weight_prefix[i] = sum of the weights
 * of vertices < i (length n+1, host memory; the build uses in-degree + 1). */
GI_API gi_status gi_partition_ranges(int64_t n, int nranks, const int64_t* weight_prefix, int64_t* bounds);

/* ---------------------------------------------------------------- graph */

/* flags for gi_graph_create */
enum {
  GI_EDGES_ON_DEVICE = 1u << 0,   /* hint: src/dst are device pointers (checked) */
  GI_REMOVE_SELF_LOOPS = 1u << 1, /* drop (u,u) pairs (reading R5) */
  GI_DEDUP = 1u << 2,             /* keep one copy of repeated (u,v) (R5) */
  GI_SYMMETRIZE = 1u << 3,        /* add (v,u) for every (u,v): "an undirected
                                     graph would be represented by duplicating
                                     the directed edges" P:3183 [draft] */
  GI_NO_RELABEL = 1u << 4,        /* keep input vertex order internally (the
                                     default relabels by out-degree when the
                                     degrees are skewed: max > 32 x mean, on one
                                     GPU; results are always in input ids) */
  GI_OFFSETS64 = 1u << 5          /* store CSR/CSC row offsets as int64 even when
                                     m < 2^31 (they are int64 anyway from 2^31
                                     edges on, e.g. config 5): runs
                                     the wide-offset kernels on small graphs */
};

/* Builds the edgeset from an edge list ("edges = load(...)"):
 *   num_vertices n: V = {0..n-1}; isolated ids are vertices (reading R4);
 *                   0 <= n <= 2^31-1.
 *   num_edges m0:   length of src/dst (int32 vertex ids), 0 <= m0 < 2^40.
 *   flags:          GI_* above; unknown bits -> GI_ERR_INVALID_ARGUMENT.
 * Any endpoint outside [0, n) -> GI_ERR_VERTEX_OUT_OF_RANGE.
 * Device work: validate, clean (self-loops, symmetrise, dedup) by radix sort
 * of 64-bit keys, CSR by source, CSC by destination, out-degrees, pull-kernel
 * tiling metadata.
 * Multi-GPU context: every rank passes ANY share of the edge list; the graph
 * is the union. The graph owns its device memory until gi_graph_destroy. */
GI_API gi_status gi_graph_create(gi_context ctx, int64_t num_vertices, int64_t num_edges,
                          const int32_t* src, const int32_t* dst, uint32_t flags,
                          gi_graph* out);
GI_API gi_status gi_graph_destroy(gi_graph g);
GI_API gi_status gi_graph_num_vertices(gi_graph g, int64_t* n);
GI_API gi_status gi_graph_num_edges(gi_graph g, int64_t* m); /* global m after cleanup */

/* Owned destination range [*lo, *hi) of this rank (input ids are not ranges:
 * this is in the library's internal vertex order; single GPU: [0, n)). */
GI_API gi_status gi_graph_partition(gi_graph g, int64_t* lo, int64_t* hi, int64_t* local_edges);

/* Test hooks (length n, input ids; host or device pointers). */
GI_API gi_status gi_graph_out_degrees(gi_graph g, int32_t* outdeg);
GI_API gi_status gi_graph_in_degrees(gi_graph g, int32_t* indeg);
/* Cleaned CSR in input ids: off[n+1] (int64), idx[m] (int32, ascending per row).
 * Single-GPU graphs only. */
GI_API gi_status gi_graph_csr(gi_graph g, int64_t* off, int32_t* idx);

/* ---------------------------------------------------------------- PageRank */

/* Fixed-iteration Jacobi PageRank, fp32 storage (reading R10):
 *   r_0[v] = 1/n                                                  (R2)
 *   r_{k+1}[v] = (1-d)/n + d * ( sum_{(u,v) in E} r_k[u]/outdeg(u) + D_k/n )
 *   D_k = sum over dangling u (outdeg 0) of r_k[u]      (uniform rule, R3)
 * P:3242-3253 [draft], base score P:856, fixed MaxIter P:514-517.
 *   iters >= 0 (iters = 0 gives 1/n), damping in [0, 1].
 *   out: float[n] in input ids (host or device).
 * n = 0 -> GI_OK, nothing written. */
GI_API gi_status gi_pagerank(gi_graph g, int32_t iters, double damping, float* out);

enum { GI_PR_PULL = 0, GI_PR_PUSH = 1, GI_PR_PULL_DIRECT = 2, GI_PR_PULL_SEGMENTED = 3, GI_PR_PULL_PARTITIONED = 4,
       GI_PR_PULL_BLOCKED = 5 };
enum { GI_DANGLING_UNIFORM = 0, GI_DANGLING_DROP = 1 };
typedef struct {
  int32_t direction; /* GI_PR_PULL (auto-selected pull kernel), GI_PR_PUSH
                        (DensePush with atomics, the parity form),
                        GI_PR_PULL_DIRECT (CSC gather via L1/L2),
                        GI_PR_PULL_SEGMENTED (shared-memory source segments),
                        GI_PR_PULL_PARTITIONED (the CSC split by source
                        range into L2-sized partitions, one gather pass per
                        partition: the paper's cache partitioning),
                        GI_PR_PULL_BLOCKED (propagation blocking, the
                        write-side counterpart the paper cites at P:755:
                        contributions binned by (source chunk, destination
                        block) in a streaming pass, summed per block in
                        shared memory in a second; chosen by GI_PR_PULL when
                        the segmented pull's pieces hold < 2.5 edges and
                        contrib exceeds 64 MB, e.g. config 5; up to
                        2048 x 49152 vertices, GI_ERR_UNSUPPORTED beyond) */
  int32_t dangling;  /* GI_DANGLING_UNIFORM (default) or GI_DANGLING_DROP
                        (paper-literal: no D term) */
  int32_t profile;   /* 1: fill gi_pr_stats kernel timings (CUDA events on the
                        context stream around every edge-pass launch) */
  int32_t segment_size; /* GI_PR_PULL_SEGMENTED: sources per shared-memory
                        segment; 0 = as many as fit in one CTA's shared memory
                        (smaller values exercise many segments in tests).
                        GI_PR_PULL_PARTITIONED: sources per partition, rounded
                        up to a power of two; 0 = sized to the L2 cache */
  int32_t dst_block;    /* GI_PR_PULL_SEGMENTED: destination rows per block
                        (the per-row accumulator of one block stays in L2);
                        0 = automatic */
} gi_pr_opts;

typedef struct {
  int32_t edge_launches;   /* edge-pass kernel launches (one per iteration) */
  int32_t aux_launches;    /* other kernel launches in the call */
  float edge_ms;           /* sum of edge-pass kernel durations (profile=1) */
  float total_ms;          /* whole call on the stream (profile=1) */
  int32_t kernel;          /* GI_PR_* kernel actually used */
  float vertex_ms;         /* segmented pull: part of edge_ms spent in the
                              vertex-update kernel (profile=1) */
  int64_t bytes_alg_per_iter; /* 4m + (o+12)n for pull (this rank's rows) */
  int32_t exchange;        /* multi-GPU contrib exchange: 0 none (one rank),
                              1 allgatherv per iteration, 2 peer stores */
  float exchange_ms;       /* profile=1: device time of the per-iteration
                              collectives (dangling allreduce + allgatherv) */
  int64_t reductions_per_iter; /* segmented pull: global reductions (RED.ADD.F32)
                              per edge pass = the layout's pieces, one per
                              (source segment, destination row) pair with an
                              edge; 0 for the other kernels */
  int64_t stream_bytes_per_iter; /* segmented pull: record bytes streamed per
                              edge pass; 0 for the other kernels */
} gi_pr_stats;

GI_API gi_status gi_pagerank_ex(gi_graph g, int32_t iters, double damping, const gi_pr_opts* opts,
                         float* out, gi_pr_stats* stats /* may be NULL */);

/* ---------------------------------------------------------------- PageRankDelta */

/* PageRankDelta (the paper's running example: Alg.
 * PageRankDelta P:426-456, GraphIt program P:849-893): Rank = 0, Delta = 1/V,
 * Frontier = V; each round DeltaSum[dst] += Delta[src]/outdeg(src) over edges
 * from the frontier, round 1: Delta = d*DeltaSum + (1-d)/V, Rank += Delta,
 * Delta -= 1/V; later: Delta = d*DeltaSum, Rank += Delta; the next frontier
 * is {v : |Delta[v]| > epsilon * Rank[v]} (readings R17, R18). The edge pass
 * is DensePull-SparsePush: pull iff |F| + sum outdeg(F) > m / threshold_div.
 *   iters >= 0 rounds (stops early if the frontier empties), damping in [0,1],
 *   epsilon >= 0; out: float[n] Rank in input ids. Single-GPU graphs only. */
enum { GI_PRD_AUTO = 0, GI_PRD_PUSH_ONLY = 1, GI_PRD_PULL_ONLY = 2 };
typedef struct {
  int32_t policy;        /* GI_PRD_AUTO / PUSH_ONLY / PULL_ONLY */
  int32_t threshold_div; /* 0 -> 20 */
  int32_t profile;       /* 1: total_ms */
  int32_t reserved;
} gi_prdelta_opts;

typedef struct {
  int32_t rounds;       /* rounds executed */
  int32_t pull_rounds;  /* rounds whose edge pass ran in the pull direction */
  int64_t active_total; /* sum over rounds of the frontier size */
  float total_ms;       /* profile=1 */
  int32_t launches;
  int32_t reserved;
} gi_prdelta_stats;

GI_API gi_status gi_pagerank_delta(gi_graph g, int32_t iters, double damping, double epsilon,
                                   const gi_prdelta_opts* opts, float* out, gi_prdelta_stats* stats);

/* ---------------------------------------------------------------- BFS */

/* Breadth-first search from `source` along out-edges (R9), direction-
 * optimising by default: pull (DensePull + bitmap frontier + early exit) iff
 * |F| + sum_{v in F} outdeg(v) > m / threshold_div, else push (SparsePush +
 * queue frontier + CAS claim) (Ligra's m/20 P:3074 [punt], R7).
 *   parent_out: int32[n] in input ids; parent[source] = source, parent[v] = -1
 *   when unreachable, otherwise an in-neighbour one level closer to the source
 *   (any valid one, R8). */
GI_API gi_status gi_bfs(gi_graph g, int32_t source, int32_t* parent_out);

enum { GI_BFS_AUTO = 0, GI_BFS_PUSH_ONLY = 1, GI_BFS_PULL_ONLY = 2 };
typedef struct {
  int32_t policy;        /* GI_BFS_AUTO / PUSH_ONLY / PULL_ONLY (pull-only runs
                            the first level as push: a 1-vertex frontier) */
  int32_t threshold_div; /* 0 -> 20 */
  int32_t profile;       /* 1: fill timing fields of gi_bfs_stats */
  int32_t batch;         /* gi_bfs_multi only: GI_BFS_BATCH_AUTO (0),
                            GI_BFS_BATCH_PER_SOURCE (one direction-optimising
                            traversal per source) or GI_BFS_BATCH_BITPARALLEL
                            (up to 64 sources per traversal, one bit each) */
  int32_t pull_kernel;   /* bit-parallel passes only, their pull levels:
                            GI_MS_PULL_AUTO (0), GI_MS_PULL_ROWS (each row scans
                            its in-edges, gathering frontier masks, until it holds
                            every source) or GI_MS_PULL_SEGMENTED (one OR pass of
                            the PageRank edge kernel over the segmented layout —
                            frontier masks staged per source segment in shared
                            memory — then each new bit's parent by a row scan
                            that stops once every new bit has one; one GPU;
                            32-bit OR passes: two when k > 32; builds the
                            layout if the graph has none). AUTO takes the
                            OR pass when the graph already has the layout and
                            the rows still missing a source hold > 0.7 m
                            (k <= 16) / 0.25 m (k > 16) in-edges */
} gi_bfs_opts;
enum { GI_BFS_BATCH_AUTO = 0, GI_BFS_BATCH_PER_SOURCE = 1, GI_BFS_BATCH_BITPARALLEL = 2 };
enum { GI_MS_PULL_AUTO = 0, GI_MS_PULL_ROWS = 1, GI_MS_PULL_SEGMENTED = 2 };

typedef struct {
  int32_t levels;          /* frontier rounds executed */
  int32_t pull_levels;     /* rounds run in the pull direction */
  int64_t reached;         /* vertices with parent != -1 */
  int64_t edges_traversed; /* R16: sum of outdeg over reached vertices */
  float total_ms;          /* profile=1 */
  int32_t launches;        /* kernel launches in the call */
  float pull_ms;           /* profile=1, bit-parallel passes: device time of the
                              pull-level kernels (0 for per-source traversals,
                              whose pulls run inside the fused kernel) */
  int64_t edges_examined;  /* edge reads of the traversal: push levels every
                              out-edge of the frontier, pull levels the in-edges
                              probed before the early exit (single GPU; 0 else) */
  int64_t pull_vertices;   /* vertex checks of the pull levels (n per level) */
  int64_t pull_edges_examined; /* the part of edges_examined read by pull levels
                                  (bit-parallel passes; 0 for per-source) */
  int32_t pull_or_levels;  /* bit-parallel passes: pull levels run as a segmented
                              OR pass (GI_MS_PULL_SEGMENTED); their edge reads
                              count every in-edge */
  int32_t pull_sparse_levels; /* bit-parallel passes: row-pull levels that pulled
                                 only the listed rows still missing a source
                                 (those rows' in-edges < m/64; not with ROWS) */
} gi_bfs_stats;
/* A bit-parallel pass serves up to 64 sources at once: its shared quantities
 * (total_ms, pull_ms, edges_examined, pull_vertices, pull_edges_examined) are
 * reported divided by the pass's source count, so summing over the sources of
 * a call gives the call's totals. */

GI_API gi_status gi_bfs_ex(gi_graph g, int32_t source, const gi_bfs_opts* opts, int32_t* parent_out,
                    gi_bfs_stats* stats /* may be NULL */);

/* k independent BFS runs (the multi-source workloads of BASELINE configs
 * 2/4/5), each a valid BFS tree of its source as k gi_bfs_ex calls give
 * (depths identical; a vertex may get another, equally valid parent, R8):
 *   sources:     int32[k] in input ids, HOST memory;
 *   parents_out: int32[k][n] (row i = parents of sources[i], layout as
 *                gi_bfs), host or device;
 *   stats:       gi_bfs_stats[k] or NULL (with profile=1, total_ms is the
 *                batch time divided by k).
 * On one GPU, opts->batch selects per-source traversals (all sources in one
 * cooperative launch) or the bit-parallel traversal (edgeset.apply over a
 * 64-bit frontier mask per vertex: one pass over an edge serves 64 sources);
 * AUTO takes the bit-parallel form for k >= 8. With BITPARALLEL, stats report
 * the shared quantities divided by the sources of the pass. Bit-parallel
 * scratch: 8 bytes x 3 + 4 x 3 + 4 x round8(min(k, 64)) bytes per vertex, kept
 * with the graph.
 * On several GPUs this is a loop of gi_bfs_ex.
 * Errors as gi_bfs_ex (checked for every source before any run); k = 0 -> GI_OK. */
GI_API gi_status gi_bfs_multi(gi_graph g, int32_t k, const int32_t* sources, const gi_bfs_opts* opts,
                              int32_t* parents_out, gi_bfs_stats* stats /* may be NULL */);

/* ---------------------------------------------------------------- connected components (NEXT #4)
 * Label propagation, the paper's CC (P:3440-3472 [punt], P:3600-3615;
 * "synchronous label propagation" P:2237): IDs[v] = v, frontier = every
 * vertex, then rounds of
 *   frontier = edges.from(frontier).apply(IDs[dst] min= IDs[src]).modified(IDs)
 * until the frontier is empty; each round runs pull (DensePull over the frontier
 * bitmap) iff |F| + sum outdeg(F) > m / threshold_div, else push (SparsePush with
 * atomicMin), as BFS (R7).
 *   labels_out: int32[n], host or device; labels_out[v] = the fixed point
 *     min{ u : u = v or a directed path u ->* v } in input ids (reading R22);
 *     on a graph built with GI_SYMMETRIZE that is the smallest vertex id of v's
 *     connected component.
 * Errors: GI_ERR_INVALID_ARGUMENT (NULL graph/output, bad options),
 * GI_ERR_UNSUPPORTED on a multi-GPU context. n = 0 -> GI_OK. */
typedef struct {
  int32_t policy;        /* GI_BFS_AUTO / GI_BFS_PUSH_ONLY / GI_BFS_PULL_ONLY */
  int32_t threshold_div; /* 0 -> 20 */
  int32_t profile;       /* 1: fill total_ms */
  int32_t reserved;
} gi_cc_opts;
typedef struct {
  int32_t rounds;          /* label-propagation rounds (the last one changes nothing) */
  int32_t pull_rounds;     /* rounds run in the pull direction */
  int64_t edges_examined;  /* in-edges read by pull rounds + out-edges by push rounds */
  float total_ms;          /* profile = 1 */
  int32_t launches;        /* kernel launches in the call */
} gi_cc_stats;
GI_API gi_status gi_cc(gi_graph g, int32_t* labels_out);
GI_API gi_status gi_cc_ex(gi_graph g, const gi_cc_opts* opts, int32_t* labels_out, gi_cc_stats* stats);

/* ---------------------------------------------------------------- SSSP (NEXT #4)
 * Single-source shortest paths, the paper's frontier-based Bellman-Ford
 * (P:2246-2247 [punt]): dist[source] = 0, frontier = {source},
 * rounds of edges.from(frontier).apply(dist[dst] min= dist[src] + w).modified(dist)
 * until the frontier is empty, each round pull or push by the BFS rule (R7).
 * Edge weights are synthetic (the graph carries none, reading R24): the weight
 * of directed edge (u, v), input ids, is 1 + mix64(mix64(weight_seed) +
 * (u << 32 | v)) % 255 (graphgen.edge_weights draws the same values; mix64 =
 * the splitmix64 finaliser). Weights are computed on the device once per
 * (graph, seed) and kept with the graph (8 bytes per edge).
 *   dist_out: int32[n], host or device: the shortest-path distance from
 *     `source` along out-edges (exact integers), -1 when unreachable.
 * Errors: as gi_bfs_ex (source out of range: GI_ERR_VERTEX_OUT_OF_RANGE);
 * GI_ERR_UNSUPPORTED on a multi-GPU context. */
typedef gi_cc_opts gi_sssp_opts;   /* policy, threshold_div (0 -> 20), profile */
typedef gi_cc_stats gi_sssp_stats; /* rounds, pull_rounds, edges_examined, total_ms, launches */
GI_API gi_status gi_sssp(gi_graph g, int32_t source, uint64_t weight_seed, int32_t* dist_out);
/* SSSP over the caller's edge weights (the paper runs SSSP on weighted
 * datasets):
 *   weights: int32[m], host or device, one per edge of the CLEANED graph in
 *     gi_graph_csr's order (input ids: rows by source ascending, neighbours
 *     ascending within a row); every weight >= 0 (GI_ERR_INVALID_ARGUMENT
 *     otherwise); every shortest-path length must be < 2^31 - 1.
 *   dist_out: int32[n] as gi_sssp.
 * The weights are moved into the library's CSR and CSC order on every call
 * (one binary search per edge) and replace any cached synthetic weights. */
GI_API gi_status gi_sssp_weighted(gi_graph g, int32_t source, const int32_t* weights, const gi_sssp_opts* opts,
                                  int32_t* dist_out, gi_sssp_stats* stats);
GI_API gi_status gi_sssp_ex(gi_graph g, int32_t source, uint64_t weight_seed, const gi_sssp_opts* opts,
                            int32_t* dist_out, gi_sssp_stats* stats);

/* ---------------------------------------------------------------- misc */
GI_API const char* gi_status_string(gi_status s);
GI_API const char* gi_last_error(void); /* thread-local; valid until the next call */
GI_API int gi_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GI_H_ */
