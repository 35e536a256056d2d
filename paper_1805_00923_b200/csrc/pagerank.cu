// pagerank.cu — fixed-iteration PageRank through edgeset.apply (SURVEY §8(a)
// rows a3-a5, §2.7 K4/K5).
//
// Math (PAPER.md P:3242-3253 [draft] edge/vertex update, base score P:856,
// DESIGN.md readings R1-R3, R10):
//   contrib_k[u] = r_k[u] / outdeg(u)   (0 for dangling u)
//   r_{k+1}[v]   = (1-d)/n + d * ( sum_{u in in(v)} contrib_k[u] + D_k/n )
//   D_k          = sum_{outdeg(u)=0} r_k[u]      (uniform rule; drop rule: no D)
//
// Pull (DensePull): one launch per iteration, the
// merge-path tile kernel k_pr_pull below; no atomics on the row sums except
// for rows split across tiles (last-arriver fix-up), which is the only
// cross-CTA dependence ("pull needs no atomics").
// Push (DensePush with an all-active frontier): red.global.add.f32
// per edge into an accumulator + a vertex kernel — the parity form.
#include "gi_internal.cuh"
#include "pr_common.cuh"
#include "comm.cuh"

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstring>
#include <cub/device/device_scan.cuh>

namespace gi {
namespace {

// auto choice of the propagation-blocked pull: fewer edges per segmented-pull
// piece than this, and a contrib vector larger than this (bytes)
constexpr double kBlockedEpp = 2.5;
constexpr int64_t kBlockedMinContrib = 64ll << 20;

// ---------------------------------------------------------------- pull, direct gather (K4)
// Tile b covers merge positions [bT, (b+1)T) of the CSC item sequence
// (pr_common.cuh). Phase A stages the tile's row offsets and gathers
// contrib[idx[e]] for its edges with coalesced index loads (the random reads
// of P:598-599, through L1/L2); phase B is the merge-path walk with the fused
// vertex update; rows that cross tiles add a double partial and an arrival
// count, and the last arriving tile finishes them (pieces = tiles touched).
// Row r's sum s over this pass's edges: the whole in-row (pmode 0), or the
// part from one source partition (cache partitioning):
// partial sums merge in pacc and the last partition's pass finishes the row.
__device__ __forceinline__ void pr_part_finish(const PrArgs& A, int64_t r, float s, float dn, double& dpart) {
  if (A.pmode == 0) pr_epilogue(A, r, s, dn, dpart);
  else if (A.pmode == 1) A.pacc[r] = s;
  else if (A.pmode == 2) A.pacc[r] += s;
  else pr_epilogue(A, r, A.pacc[r] + s, dn, dpart);
}

template <typename OffT>
__global__ void __launch_bounds__(kPullThreads) k_pr_pull(PrArgs A) {
  constexpr int NT = kPullThreads, IPT = kPullItemsPerThread, T = kPullTile;
  __shared__ int loff[T + 2];
  __shared__ float sval[T];
  __shared__ KeyVal scratch[NT / 32];
  __shared__ double sred[32];

  const OffT* __restrict__ off = static_cast<const OffT*>(A.off);
  const int tid = threadIdx.x;
  const int64_t b = blockIdx.x;
  const int64_t p0 = b * (int64_t)T;
  const int64_t p1 = min(p0 + (int64_t)T, A.n + A.m);
  const int64_t r0 = A.tile_rows[2 * b], r1 = A.tile_rows[2 * b + 1];
  const int R = (int)(r1 - r0 + 1);
  const int items = (int)(p1 - p0);
  const int64_t eb = p0 - r0;  // the tile's first edge

  if (b == 0 && tid == 0) A.dbuf[(A.it + 2) % 3] = 0.0;
  const double D = A.uniform ? A.dbuf[A.it % 3] : 0.0;
  const float dn = (float)(D * A.inv_n);

  for (int i = tid; i <= R; i += NT) {
    const int64_t v = (int64_t)off[r0 + i] - eb;
    loff[i] = (int)max((int64_t)-1, min(v, (int64_t)items + 1));
  }
  __syncthreads();
  const int ne = min(loff[R], items - (R - 1));
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const int j = tid + k * NT;
    if (j < ne) sval[j] = __ldg(&A.cin[__ldg(&A.idx[eb + j])]);
  }
  __syncthreads();

  double dpart = 0.0;
  tile_walk<NT, IPT>(
      loff, R, items, sval, scratch, [&](int i, float v) { pr_part_finish(A, r0 + i, v, dn, dpart); },
      [&](int i, float v) {
        const int64_t r = r0 + i;
        const int64_t sp = r + (int64_t)off[r], ep = r + (int64_t)off[r + 1];
        const int pieces = (int)(ep / T - sp / T + 1);
        atomicAdd(&A.split_acc[r], (double)v);
        __threadfence();
        const int prev = atomicAdd(&A.split_cnt[r], 1);
        if (prev == pieces - 1) {
          __threadfence();
          const double tot = atomicAdd(&A.split_acc[r], 0.0);
          pr_part_finish(A, r, (float)tot, dn, dpart);
          A.split_acc[r] = 0.0;
          A.split_cnt[r] = 0;
        }
      });
  if (A.npeer) __threadfence_system();  // peer stores ordered before the next collective
  const double bs = block_sum(dpart, sred);
  if (tid == 0 && bs != 0.0) atomicAdd(&A.dbuf[(A.it + 1) % 3], bs);
}

// ---------------------------------------------------------------- pull, thread per row (flat graphs)
// Graphs whose rows are all short (max in-degree <= kRowsMaxDeg: a road grid)
// need no merge-path balancing: every thread sums kRowsPT rows spaced a block
// apart (independent offset -> index -> contrib chains in flight), the
// gathers stay local in input order, and the vertex update is fused.
#ifndef GI_ROWS_PT
#define GI_ROWS_PT 4
#endif
constexpr int kRowsPT = GI_ROWS_PT;
constexpr int kRowsMaxDeg = 64;

template <typename OffT>
#ifndef GI_ROWS_MINB
#define GI_ROWS_MINB 4  // 64 registers: 4 CTAs per SM (96 registers, 2 CTAs: config 3 0.18-0.27 ms; 4: 0.150)
#endif
__global__ void __launch_bounds__(256, GI_ROWS_MINB) k_pr_rows(PrArgs A) {
  __shared__ double sred[32];
  const OffT* __restrict__ off = static_cast<const OffT*>(A.off);
  if (blockIdx.x == 0 && threadIdx.x == 0) A.dbuf[(A.it + 2) % 3] = 0.0;
  const double D = A.uniform ? A.dbuf[A.it % 3] : 0.0;
  const float dn = (float)(D * A.inv_n);
  double dpart = 0.0;
  const int64_t span = (int64_t)blockDim.x * kRowsPT;
  for (int64_t base = blockIdx.x * span; base < A.n; base += (int64_t)gridDim.x * span) {
    int64_t a[kRowsPT], b[kRowsPT];
#pragma unroll
    for (int k = 0; k < kRowsPT; ++k) {
      const int64_t r = base + threadIdx.x + (int64_t)k * blockDim.x;
      a[k] = b[k] = 0;
      if (r < A.n) {
        a[k] = (int64_t)off[r];
        b[k] = (int64_t)off[r + 1];
      }
    }
    // 4 edges of each of the kRowsPT rows per step: 16 independent index loads,
    // then 16 independent gathers
    float s[kRowsPT];
    int64_t len = 0;
#pragma unroll
    for (int k = 0; k < kRowsPT; ++k) {
      s[k] = 0.f;
      len = max(len, b[k] - a[k]);
    }
    for (int64_t j = 0; j < len; j += 4) {
      int32_t u[kRowsPT][4];
#pragma unroll
      for (int k = 0; k < kRowsPT; ++k)
#pragma unroll
        for (int q = 0; q < 4; ++q) u[k][q] = a[k] + j + q < b[k] ? __ldg(&A.idx[a[k] + j + q]) : -1;
#pragma unroll
      for (int k = 0; k < kRowsPT; ++k)
#pragma unroll
        for (int q = 0; q < 4; ++q) s[k] += u[k][q] >= 0 ? __ldg(&A.cin[u[k][q]]) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < kRowsPT; ++k) {
      const int64_t r = base + threadIdx.x + (int64_t)k * blockDim.x;
      if (r < A.n) pr_epilogue(A, r, s[k], dn, dpart);
    }
  }
  if (A.npeer) __threadfence_system();  // peer stores ordered before the next collective
  const double bs = block_sum(dpart, sred);
  if (threadIdx.x == 0 && bs != 0.0) atomicAdd(&A.dbuf[(A.it + 1) % 3], bs);
}

template <typename OffT>
__global__ void k_max_rowlen(const OffT* __restrict__ off, int64_t n, int* __restrict__ out) {
  int mx = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    mx = max(mx, (int)min((int64_t)INT32_MAX, (int64_t)off[r + 1] - (int64_t)off[r]));
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(out, mx);
}

// ---------------------------------------------------------------- push (K5)
template <typename OffT>
__global__ void __launch_bounds__(256) k_pr_push(int64_t n, int64_t row0, const OffT* __restrict__ off,
                                                 const int32_t* __restrict__ idx, const float* __restrict__ cin,
                                                 double* __restrict__ acc) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = warp; u < n; u += nwarps) {
    const float c = __ldg(&cin[u]);
    if (c == 0.f) continue;
    for (int64_t j = (int64_t)off[u] + lane; j < (int64_t)off[u + 1]; j += 32)
      atomicAdd(&acc[__ldg(&idx[j]) - row0], (double)c);  // result unused -> RED.E.ADD.F64 (fp64: hub rows sum
                                                    // 1e5+ terms; fp32 atomics drift past 1e-4)
  }
}

__global__ void __launch_bounds__(256) k_pr_vertex(PrArgs A, double* __restrict__ acc) {
  __shared__ double sred[8];
  if (blockIdx.x == 0 && threadIdx.x == 0) A.dbuf[(A.it + 2) % 3] = 0.0;
  const double D = A.uniform ? A.dbuf[A.it % 3] : 0.0;
  const float dn = (float)(D * A.inv_n);
  double dpart = 0.0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < A.n; v += (int64_t)gridDim.x * blockDim.x) {
    const float s = (float)acc[v];
    acc[v] = 0.0;
    pr_epilogue(A, v, s, dn, dpart);
  }
  if (A.npeer) __threadfence_system();  // peer stores ordered before the next collective
  const double bs = block_sum(dpart, sred);
  if (threadIdx.x == 0 && bs != 0.0) atomicAdd(&A.dbuf[(A.it + 1) % 3], bs);
}

// r_0 = 1/n: contrib_0 and D_0
__global__ void __launch_bounds__(256) k_pr_init(int64_t n, const int32_t* __restrict__ outdeg, float* __restrict__ c0,
                                                 double* __restrict__ dbuf, float r0) {
  __shared__ double sred[8];
  double dpart = 0.0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int od = outdeg[v];
    c0[v] = od > 0 ? r0 / (float)od : 0.f;
    if (od == 0) dpart += (double)r0;
  }
  const double bs = block_sum(dpart, sred);
  if (threadIdx.x == 0 && bs != 0.0) atomicAdd(&dbuf[0], bs);
}

// out[perm[v]] = in[v] (internal ids -> input ids)
__global__ void k_permute_out(const float* __restrict__ in, const int32_t* __restrict__ perm, int64_t n,
                              float* __restrict__ out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    out[perm ? perm[v] : v] = in[v];
}

__global__ void k_fill(float* __restrict__ out, int64_t n, float v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = v;
}

// ---------------------------------------------------------------- source-partitioned CSC (cache partitioning)
// "incoming edges (src, dst) are assigned to SSG_i if src
// in V_i, and sorted by dst"; V_i = [i << shift, (i+1) << shift). A warp per
// CSC row counts its edges per partition (k_sp_count), then places them
// (k_sp_fill) keeping their order inside the row: lanes of one step holding
// the same partition take consecutive slots by rank (__match_any_sync).
constexpr int kSpMax = 32;  // partitions at most (one histogram bin per lane)

template <typename OffT>
__global__ void __launch_bounds__(256) k_sp_count(const OffT* __restrict__ off, const int32_t* __restrict__ idx,
                                                  int64_t nr, int shift, int P, int64_t* __restrict__ cnt) {
  __shared__ int hist[8][kSpMax];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  for (int64_t w = blockIdx.x * 8ll + wp; w < nr; w += gridDim.x * 8ll) {
    hist[wp][lane] = 0;
    __syncwarp();
    for (int64_t e = (int64_t)off[w] + lane; e < (int64_t)off[w + 1]; e += 32) atomicAdd(&hist[wp][idx[e] >> shift], 1);
    __syncwarp();
    if (lane < P) cnt[lane * (nr + 1) + w] = hist[wp][lane];
    __syncwarp();
  }
}

template <typename OffT>
__global__ void __launch_bounds__(256) k_sp_fill(const OffT* __restrict__ off, const int32_t* __restrict__ idx,
                                                 int64_t nr, int shift, const int64_t* __restrict__ poff,
                                                 const int64_t* __restrict__ base, int32_t* __restrict__ out) {
  __shared__ int cur[8][kSpMax + 1];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  for (int64_t w = blockIdx.x * 8ll + wp; w < nr; w += gridDim.x * 8ll) {
    cur[wp][lane] = 0;
    __syncwarp();
    const int64_t e0 = (int64_t)off[w], e1 = (int64_t)off[w + 1];
    for (int64_t b = e0; b < e1; b += 32) {
      const int64_t e = b + lane;
      const int32_t v = e < e1 ? idx[e] : -1;
      const int p = v >= 0 ? v >> shift : kSpMax;
      const unsigned peers = __match_any_sync(0xffffffffu, p);
      const int rank = __popc(peers & ((1u << lane) - 1u));
      const int c = cur[wp][p];
      if (v >= 0) out[base[p] + poff[p * (nr + 1) + w] + c + rank] = v;
      __syncwarp();
      if (rank == 0) cur[wp][p] = c + __popc(peers);
      __syncwarp();
    }
  }
}

__global__ void k_narrow_off(const int64_t* __restrict__ in, int64_t n, int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)in[i];
}

}  // namespace

// Builds the source-partitioned CSC once per graph (single GPU).
static gi_status sp_build(gi_graph g, int sources_per_part) {
  gi_context ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  const int64_t n = g->n, nr = g->nr, m = g->ml;
  int64_t z = sources_per_part;
  if (z <= 0) {  // a partition's contrib slice: ~3/8 of L2 (the record stream and the row sums share it)
    int l2 = 0;
    GI_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ctx->device));
    z = std::max<int64_t>((int64_t)l2 * 3 / 8 / 4, 1024);
  }
  int shift = 0;
  if (sources_per_part > 0)
    while ((1ll << shift) < z) ++shift;  // round up
  else
    while ((2ll << shift) <= z) ++shift;  // round down
  while (((n + (1ll << shift) - 1) >> shift) > kSpMax) ++shift;
  const int P = (int)std::max<int64_t>(1, (n + (1ll << shift) - 1) >> shift);
  if (g->sp_P == P && g->sp_shift == shift) return GI_OK;
  g->sp_P = 0;
  const int64_t stride = nr + 1;
  DevBuf cnt, poff, dbase, tmp;
  GI_TRY(cnt.alloc((size_t)P * stride * sizeof(int64_t)));
  GI_TRY(poff.alloc((size_t)P * stride * sizeof(int64_t)));
  GI_CUDA(cudaMemsetAsync(cnt.p, 0, (size_t)P * stride * sizeof(int64_t), st));
  const int grid = grid_for(ceil_div(nr, 8), 256, sms, 8);
  if (nr > 0) {
    if (g->off64) k_sp_count<int64_t><<<grid, 256, 0, st>>>(g->csc_off.as<int64_t>(), g->csc_idx.as<int32_t>(), nr, shift, P, cnt.as<int64_t>());
    else k_sp_count<int32_t><<<grid, 256, 0, st>>>(g->csc_off.as<int32_t>(), g->csc_idx.as<int32_t>(), nr, shift, P, cnt.as<int64_t>());
    GI_CUDA(cudaGetLastError());
  }
  size_t tb = 0;
  GI_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.as<int64_t>(), poff.as<int64_t>(), stride, st));
  GI_TRY(tmp.alloc(tb));
  for (int p = 0; p < P; ++p)
    GI_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.as<int64_t>() + p * stride, poff.as<int64_t>() + p * stride,
                                          stride, st));
  std::vector<int64_t> mp(P);
  for (int p = 0; p < P; ++p)
    GI_CUDA(cudaMemcpyAsync(&mp[p], poff.as<int64_t>() + p * stride + nr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  g->sp_m = mp;
  g->sp_base.assign(P + 1, 0);
  g->sp_ntiles.assign(P, 0);
  g->sp_tile0.assign(P + 1, 0);
  bool wide = false;
  for (int p = 0; p < P; ++p) {
    g->sp_base[p + 1] = g->sp_base[p] + mp[p];
    wide = wide || mp[p] > INT32_MAX - 1;
    g->sp_ntiles[p] = nr > 0 ? ceil_div(nr + mp[p], kPullTile) : 0;
    g->sp_tile0[p + 1] = g->sp_tile0[p] + g->sp_ntiles[p];
  }
  if (g->sp_base[P] != m) return fail(GI_ERR_INTERNAL, "source partitions do not cover the CSC");
  GI_TRY(dbase.alloc(P * sizeof(int64_t)));
  GI_CUDA(cudaMemcpyAsync(dbase.p, g->sp_base.data(), P * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  GI_TRY(g->sp_idx.alloc(std::max<int64_t>(m, 1) * sizeof(int32_t)));
  if (nr > 0) {
    if (g->off64)
      k_sp_fill<int64_t><<<grid, 256, 0, st>>>(g->csc_off.as<int64_t>(), g->csc_idx.as<int32_t>(), nr, shift,
                                               poff.as<int64_t>(), dbase.as<int64_t>(), g->sp_idx.as<int32_t>());
    else
      k_sp_fill<int32_t><<<grid, 256, 0, st>>>(g->csc_off.as<int32_t>(), g->csc_idx.as<int32_t>(), nr, shift,
                                               poff.as<int64_t>(), dbase.as<int64_t>(), g->sp_idx.as<int32_t>());
    GI_CUDA(cudaGetLastError());
  }
  g->sp_off64 = wide;
  if (wide) {
    GI_TRY(g->sp_off.alloc((size_t)P * stride * sizeof(int64_t)));
    GI_CUDA(cudaMemcpyAsync(g->sp_off.p, poff.p, (size_t)P * stride * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  } else {
    GI_TRY(g->sp_off.alloc((size_t)P * stride * sizeof(int32_t)));
    k_narrow_off<<<grid_for(P * stride, 256, sms), 256, 0, st>>>(poff.as<int64_t>(), P * stride, g->sp_off.as<int32_t>());
    GI_CUDA(cudaGetLastError());
  }
  GI_TRY(g->sp_tiles.alloc(2 * std::max<int64_t>(g->sp_tile0[P], 1) * sizeof(int32_t)));
  const size_t osz = wide ? 8 : 4;
  for (int p = 0; p < P; ++p)
    GI_TRY(tile_rows_launch(static_cast<const char*>(g->sp_off.p) + (size_t)p * stride * osz, wide, nr, mp[p],
                            g->sp_ntiles[p], g->sp_tiles.as<int32_t>() + 2 * g->sp_tile0[p], st, sms));
  GI_TRY(g->sp_acc.alloc(std::max<int64_t>(nr, 1) * sizeof(float)));
  GI_CUDA(cudaStreamSynchronize(st));
  g->sp_P = P;
  g->sp_shift = shift;
  return GI_OK;
}

gi_status pagerank_run(gi_graph g, int32_t iters, double damping, const gi_pr_opts& o, float* d_out,
                       gi_pr_stats* stats) {
  gi_context ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  const int64_t n = g->n;                 // global vertices
  const int64_t nr = g->nr, ml = g->ml;   // rows and edges held by this rank
  const bool dist = ctx->nranks > 1;
  gi_pr_stats S{};
  int kernel = o.direction;
  // auto pull kernel: shared-memory segments for skewed (relabelled) graphs, whose
  // hubs concentrate the gathers; the direct L2 gather keeps the input order's
  // locality on flat-degree graphs (a grid's in-neighbours are +-1, +-width)
  // auto pull: segmented on relabelled graphs, else direct (decided once per graph).
  // The source-partitioned pull (cache partitioning) is explicit only: on B200 a
  // random 4-byte gather costs the same whether its sector hits L2 or HBM
  // (DESIGN.md §5), so partitions sized to L2 measured no faster than the
  // direct gather on configs 2, 4 and 5.
  if (kernel == GI_PR_PULL && g->pr_auto >= 0 && !dist) kernel = g->pr_auto;
  if (kernel == GI_PR_PULL) {
    // skewed (relabelled) graphs: the segmented pull, unless its (row, segment)
    // pieces hold so few edges that its one RED per piece dominates (config 5's
    // flat, symmetrised RMAT: ~1.6 edges per piece) and contrib exceeds what L2
    // keeps: then the propagation-blocked pull (pr_blocked.cu). Decided from
    // global counts, so every rank picks the same family.
    kernel = GI_PR_PULL_DIRECT;
    if (g->relabeled && o.segment_size == 0) {
      int Z = 0;
      int64_t cnt[2] = {0, 0};  // pieces, edges
      if (nr > 0 && ml > 0 && seg_default_Z(g, &Z) == GI_OK) {
        GI_TRY(pb_count_pieces(g, Z, &cnt[0]));
        cnt[1] = ml;
      }
      if (dist) {
        DevBuf cb2;
        GI_TRY(cb2.alloc(sizeof cnt));
        GI_CUDA(cudaMemcpyAsync(cb2.p, cnt, sizeof cnt, cudaMemcpyHostToDevice, st));
        GI_TRY(ctx->comm->allreduce_i64(cb2.as<int64_t>(), 2, st));
        GI_CUDA(cudaMemcpyAsync(cnt, cb2.p, sizeof cnt, cudaMemcpyDeviceToHost, st));
        GI_CUDA(cudaStreamSynchronize(st));
      }
      static const double epp_min = getenv("GI_PB_EPP") ? atof(getenv("GI_PB_EPP")) : kBlockedEpp;
      const double epp = cnt[0] > 0 ? (double)cnt[1] / (double)cnt[0] : 1e30;
      g->pb_epp = epp;
      if (const char* dbg = getenv("GI_DEBUG_SEG_LAYOUT"))
        if (FILE* f = fopen(dbg, "a")) {
          fprintf(f, "auto pull: Z=%d pieces=%lld edges=%lld edges/piece=%.3f\n", Z, (long long)cnt[0],
                  (long long)cnt[1], epp);
          fclose(f);
        }
      if (epp < epp_min && (int64_t)n * 4 > kBlockedMinContrib && nr > 0 && ml > 0 && pb_build(g) == GI_OK)
        kernel = GI_PR_PULL_BLOCKED;
    }
    if (kernel == GI_PR_PULL_DIRECT && nr > 0 && ml > 0 && g->relabeled &&
        seg_build(g, o.segment_size, o.dst_block) == GI_OK)
      kernel = GI_PR_PULL_SEGMENTED;
    if (!dist) g->pr_auto = kernel;
  }
  if (kernel == GI_PR_PULL_BLOCKED) {
    if (nr > 0 && ml > 0) GI_TRY(pb_build(g));
    else kernel = GI_PR_PULL_DIRECT;
  }
  if (kernel == GI_PR_PULL_PARTITIONED) {
    if (dist || nr == 0 || ml == 0) kernel = GI_PR_PULL_DIRECT;
    else GI_TRY(sp_build(g, o.segment_size));
  } else if (kernel == GI_PR_PULL_SEGMENTED) {
    if (nr > 0 && ml > 0) GI_TRY(seg_build(g, o.segment_size, o.dst_block));
    else kernel = GI_PR_PULL_DIRECT;
  }
  // multi-GPU peer stores: asked for by GI_PR_PEER=1
  // (=0 forbids them; unset: the comm's default, on only for in-process ranks)
  const char* peer_env = getenv("GI_PR_PEER");
  const bool ask_peer = dist && ctx->nranks <= 8 &&
                        (peer_env ? strcmp(peer_env, "0") != 0 : ctx->comm->peer_stores_default());
  bool want_peer = false;
  if (dist) {  // every rank must run the same kernel family and exchange (collective call sequence)
    DevBuf kk;
    GI_TRY(kk.alloc(3 * sizeof(int32_t)));
    int32_t mine[3] = {kernel == GI_PR_PULL_SEGMENTED ? 1 : 0, ask_peer ? 1 : 0, kernel == GI_PR_PULL_BLOCKED ? 1 : 0};
    GI_CUDA(cudaMemcpyAsync(kk.p, mine, sizeof mine, cudaMemcpyHostToDevice, st));
    GI_TRY(ctx->comm->allreduce_i32(kk.as<int32_t>(), 3, st));
    int32_t all[3] = {0, 0, 0};
    GI_CUDA(cudaMemcpyAsync(all, kk.p, sizeof all, cudaMemcpyDeviceToHost, st));
    GI_CUDA(cudaStreamSynchronize(st));
    const bool mixed = (all[0] != 0 && all[0] != ctx->nranks) || (all[2] != 0 && all[2] != ctx->nranks);
    if (o.direction == GI_PR_PULL && mixed) kernel = GI_PR_PULL_DIRECT;
    want_peer = all[1] == ctx->nranks;  // every rank asked
  }
  S.kernel = kernel;
  // direct pull: thread-per-row kernel when every row is short, else merge-path tiles
  if (kernel == GI_PR_PULL_DIRECT && g->max_indeg < 0) {
    DevBuf mx;
    GI_TRY(mx.alloc(sizeof(int)));
    GI_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(int), st));
    if (g->off64) k_max_rowlen<int64_t><<<grid_for(nr, 256, sms), 256, 0, st>>>(g->csc_off.as<int64_t>(), nr, mx.as<int>());
    else k_max_rowlen<int32_t><<<grid_for(nr, 256, sms), 256, 0, st>>>(g->csc_off.as<int32_t>(), nr, mx.as<int>());
    int h = 0;
    GI_CUDA(cudaMemcpyAsync(&h, mx.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    GI_CUDA(cudaStreamSynchronize(st));
    g->max_indeg = h;
  }
  const bool rows_kernel = kernel == GI_PR_PULL_DIRECT && g->max_indeg <= kRowsMaxDeg;
  const int osz = g->off64 ? 8 : 4;
  S.bytes_alg_per_iter = 4 * ml + (int64_t)(osz + 12) * nr;
  if (n == 0) {
    if (stats) *stats = S;
    return GI_OK;
  }
  if (iters == 0) {
    k_fill<<<grid_for(n, 256, sms), 256, 0, st>>>(d_out, n, (float)(1.0 / (double)n));
    GI_CUDA(cudaGetLastError());
    S.aux_launches = 1;
    if (stats) *stats = S;
    return GI_OK;
  }
  // workspace (lazily allocated, reused across calls)
  for (int k = 0; k < 2; ++k)
    if (!g->contrib[k].p) GI_TRY(g->contrib[k].alloc((n + 16) * sizeof(float), /*plain=*/dist));
  if (!g->dbuf.p) GI_TRY(g->dbuf.alloc(4 * sizeof(double)));
  if (kernel == GI_PR_PUSH) {
    if (!g->push_sum.p) {
      GI_TRY(g->push_sum.alloc((nr + 1) * sizeof(double)));
      GI_CUDA(cudaMemsetAsync(g->push_sum.p, 0, (nr + 1) * sizeof(double), st));
    }
  } else if (!g->split_acc.p) {
    GI_TRY(g->split_acc.alloc((nr + 1) * sizeof(double)));
    GI_TRY(g->split_cnt.alloc((nr + 1) * sizeof(int32_t)));
    GI_CUDA(cudaMemsetAsync(g->split_acc.p, 0, (nr + 1) * sizeof(double), st));
    GI_CUDA(cudaMemsetAsync(g->split_cnt.p, 0, (nr + 1) * sizeof(int32_t), st));
  }
  // multi-GPU: contrib slices exchanged every iteration; the final ranks
  // gathered in internal order, then permuted to input ids
  std::vector<int64_t> cb;
  DevBuf rank_int;
  if (dist) {
    cb.resize(g->bounds.size());
    for (size_t i = 0; i < cb.size(); ++i) cb[i] = g->bounds[i] * (int64_t)sizeof(float);
    GI_TRY(rank_int.alloc(n * sizeof(float)));
  }

  // multi-GPU: map every rank's contrib replicas once per graph; the vertex
  // update then stores each owned row's new contrib into all replicas over
  // NVLink, and the per-iteration allgather goes away.
  // The dangling-mass allreduce that follows every vertex pass orders those
  // stores before any rank's next edge pass. GI_PR_PEER=0: allgather path.
  if (want_peer && g->peer_state == 0) {
    // both maps always run on every rank (a failed map is agreed on inside)
    gi_status e0 = ctx->comm->peer_map(g->contrib[0].p, g->peer_c[0], g->peer_opened, st);
    gi_status e1 = ctx->comm->peer_map(g->contrib[1].p, g->peer_c[1], g->peer_opened, st);
    g->peer_state = (e0 == GI_OK && e1 == GI_OK) ? 1 : -1;
    if (g->peer_state != 1) {
      peer_unmap(g->peer_opened);
      set_error("");  // the allgather fallback serves the call: no stale message
    }
  }
  const bool peer = want_peer && g->peer_state == 1;
  S.exchange = dist ? (peer ? 2 : 1) : 0;
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr}, tot[2] = {nullptr, nullptr}, xev[2] = {nullptr, nullptr};
  if (o.profile) {
    for (int k = 0; k < 3; ++k) GI_CUDA(cudaEventCreate(&ev[k]));
    for (int k = 0; k < 2; ++k) GI_CUDA(cudaEventCreate(&tot[k]));
    for (int k = 0; k < 2; ++k) GI_CUDA(cudaEventCreate(&xev[k]));
    GI_CUDA(cudaEventRecord(tot[0], st));
  }
  GI_CUDA(cudaMemsetAsync(g->dbuf.p, 0, 4 * sizeof(double), st));
  k_pr_init<<<grid_for(n, 256, sms), 256, 0, st>>>(n, g->outdeg.as<int32_t>(), g->contrib[0].as<float>(),
                                                   g->dbuf.as<double>(), (float)(1.0 / (double)n));
  S.aux_launches = 1;

  PrArgs A{};
  A.n = nr;
  A.m = ml;
  A.row0 = g->r0;
  A.outdeg = g->outdeg.as<int32_t>();
  A.dbuf = g->dbuf.as<double>();
  A.base = (float)((1.0 - damping) / (double)n);
  A.damp = (float)damping;
  A.inv_n = 1.0 / (double)n;
  A.uniform = o.dangling == GI_DANGLING_UNIFORM;
  A.split_acc = g->split_acc.as<double>();
  A.split_cnt = g->split_cnt.as<int32_t>();
  A.perm = (g->relabeled && !dist) ? g->perm.as<int32_t>() : nullptr;
  float edge_ms = 0.f, vertex_ms = 0.f;
  for (int it = 0; it < iters; ++it) {
    A.it = it;
    A.cin = g->contrib[it & 1].as<float>();
    A.cout = g->contrib[(it + 1) & 1].as<float>();
    A.rank_out = (it == iters - 1) ? (dist ? rank_int.as<float>() : d_out) : nullptr;
    A.npeer = 0;
    if (peer)
      for (int q = 0; q < ctx->nranks; ++q)
        if (q != ctx->rank) A.peer[A.npeer++] = static_cast<float*>(g->peer_c[(it + 1) & 1][q]);
    if (o.profile) GI_CUDA(cudaEventRecord(ev[0], st));
    if (dist) GI_CUDA(cudaMemsetAsync(A.dbuf + (it + 1) % 3, 0, sizeof(double), st));  // ranks without rows
    if (kernel == GI_PR_PUSH) {
      const int grid = grid_for(n * 32, 256, sms, 16);
      if (g->off64)
        k_pr_push<int64_t><<<grid, 256, 0, st>>>(n, g->r0, g->csr_off.as<int64_t>(), g->csr_idx.as<int32_t>(), A.cin,
                                                 g->push_sum.as<double>());
      else
        k_pr_push<int32_t><<<grid, 256, 0, st>>>(n, g->r0, g->csr_off.as<int32_t>(), g->csr_idx.as<int32_t>(), A.cin,
                                                 g->push_sum.as<double>());
      if (o.profile) GI_CUDA(cudaEventRecord(ev[1], st));
      k_pr_vertex<<<grid_for(nr, 256, sms), 256, 0, st>>>(A, g->push_sum.as<double>());
      S.aux_launches++;
    } else if (kernel == GI_PR_PULL_BLOCKED) {  // scatter to bins + gather with fused vertex update
      GI_TRY(pb_iteration(g, A, o.profile ? ev[2] : nullptr));
      S.aux_launches++;
      if (o.profile) GI_CUDA(cudaEventRecord(ev[1], st));
    } else if (kernel == GI_PR_PULL_SEGMENTED) {
      GI_TRY(seg_edge_pass(g, A.cin));
      if (o.profile) GI_CUDA(cudaEventRecord(ev[2], st));
      GI_TRY(seg_vertex_pass(g, A));
      S.aux_launches++;
      if (o.profile) GI_CUDA(cudaEventRecord(ev[1], st));
    } else if (kernel == GI_PR_PULL_PARTITIONED) {  // one merge-path pass per source partition
      const int P = g->sp_P;
      A.pacc = g->sp_acc.as<float>();
      for (int p = 0; p < P; ++p) {
        A.pmode = P == 1 ? 0 : p == 0 ? 1 : p == P - 1 ? 3 : 2;
        A.m = g->sp_m[p];
        A.idx = g->sp_idx.as<int32_t>() + g->sp_base[p];
        A.tile_rows = g->sp_tiles.as<int32_t>() + 2 * g->sp_tile0[p];
        if (g->sp_ntiles[p] == 0) continue;
        if (g->sp_off64) {
          A.off = g->sp_off.as<int64_t>() + p * (nr + 1);
          k_pr_pull<int64_t><<<(unsigned)g->sp_ntiles[p], kPullThreads, 0, st>>>(A);
        } else {
          A.off = g->sp_off.as<int32_t>() + p * (nr + 1);
          k_pr_pull<int32_t><<<(unsigned)g->sp_ntiles[p], kPullThreads, 0, st>>>(A);
        }
      }
      A.pmode = 0;
      A.m = ml;
      if (o.profile) GI_CUDA(cudaEventRecord(ev[1], st));
    } else {
      A.tile_rows = g->tile_rows.as<int32_t>();
      A.idx = g->csc_idx.as<int32_t>();
      const int rgrid = grid_for(ceil_div(nr, kRowsPT), 256, sms, 8);
      if (g->off64) {
        A.off = g->csc_off.as<int64_t>();
        if (rows_kernel) k_pr_rows<int64_t><<<rgrid, 256, 0, st>>>(A);
        else if (g->ntiles > 0) k_pr_pull<int64_t><<<(unsigned)g->ntiles, kPullThreads, 0, st>>>(A);
      } else {
        A.off = g->csc_off.as<int32_t>();
        if (rows_kernel) k_pr_rows<int32_t><<<rgrid, 256, 0, st>>>(A);
        else if (g->ntiles > 0) k_pr_pull<int32_t><<<(unsigned)g->ntiles, kPullThreads, 0, st>>>(A);
      }
      if (o.profile) GI_CUDA(cudaEventRecord(ev[1], st));
    }
    GI_CUDA(cudaGetLastError());
    S.edge_launches++;
    if (dist) {  // dangling partials (allreduce) + contrib slices (allgatherv)
      if (o.profile) GI_CUDA(cudaEventRecord(xev[0], st));
      GI_TRY(ctx->comm->allreduce_f64(A.dbuf + (it + 1) % 3, 1, st));
      if (!peer) GI_TRY(ctx->comm->allgatherv(A.cout, cb, st));
      if (o.profile) {
        GI_CUDA(cudaEventRecord(xev[1], st));
        GI_CUDA(cudaEventSynchronize(xev[1]));
        float xm = 0.f;
        GI_CUDA(cudaEventElapsedTime(&xm, xev[0], xev[1]));
        S.exchange_ms += xm;
      }
      if (it == iters - 1) {
        std::vector<int64_t> rb = cb;
        GI_TRY(ctx->comm->allgatherv(rank_int.p, rb, st));
        k_permute_out<<<grid_for(n, 256, sms), 256, 0, st>>>(rank_int.as<float>(),
                                                             g->relabeled ? g->perm.as<int32_t>() : nullptr, n, d_out);
        S.aux_launches++;
      }
    }
    if (o.profile) {
      GI_CUDA(cudaEventSynchronize(ev[1]));
      float ms = 0.f;
      GI_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
      edge_ms += ms;
      if (kernel == GI_PR_PULL_SEGMENTED || kernel == GI_PR_PULL_BLOCKED) {
        GI_CUDA(cudaEventElapsedTime(&ms, ev[2], ev[1]));
        vertex_ms += ms;
      }
    }
  }
  if (o.profile) {
    GI_CUDA(cudaEventRecord(tot[1], st));
    GI_CUDA(cudaEventSynchronize(tot[1]));
    GI_CUDA(cudaEventElapsedTime(&S.total_ms, tot[0], tot[1]));
    S.edge_ms = edge_ms;
    S.vertex_ms = vertex_ms;
    for (int k = 0; k < 3; ++k) cudaEventDestroy(ev[k]);
    for (int k = 0; k < 2; ++k) cudaEventDestroy(tot[k]);
    for (int k = 0; k < 2; ++k) cudaEventDestroy(xev[k]);
  }
  if (kernel == GI_PR_PULL_SEGMENTED) {  // the segmented pass's per-iteration work (layout counts)
    S.reductions_per_iter = g->seg_P;
    S.stream_bytes_per_iter = g->seg_C * seg_record_bytes();
  }
  if (stats) *stats = S;
  return GI_OK;
}

}  // namespace gi
