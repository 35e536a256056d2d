// cc.cu — connected components by label propagation and SSSP by frontier
// Bellman-Ford: one min-propagation engine.
//
// The paper's CC (P:3440-3472 [punt]; "synchronous label
// propagation" P:2237): IDs[v] = v, frontier = every vertex, then rounds of
//   frontier = edges.from(frontier).apply(IDs[dst] min= IDs[src]).modified(IDs)
// until the frontier is empty — the same edgeset.apply as BFS with a min
// reduction on the destination and the "modified" filter building the next
// frontier (the vertices whose label dropped, each once). The labels reach the
// fixed point IDs[v] = min{u : u = v or u ->* v} (reading R22; on a symmetric
// graph the smallest vertex id of v's component). Labels are INPUT ids, so the
// result does not depend on the internal relabelling.
//
// Per round, direction by the BFS rule (R7): pull iff |F| + sum outdeg F > m/20.
//   pull (DensePull), CC on a graph with the segmented layout: one pass of the
//     PageRank edge kernel with an int32-min reduction (seg_min_pass) over every
//     in-neighbour's label, then k_cc_apply lowers the labels and builds the
//     next frontier; otherwise (and for SSSP) every row takes the min over its
//     in-neighbours in F (frontier bitmap): light rows (in-degree < 32) a thread
//     each, heavy rows in chunks of <= 1024 in-edges a warp each (chunks of one
//     row race through atomicMin; the one whose atomicMin lowered the label
//     marks the row);
//   push (SparsePush): the frontier's out-edges, concatenated by an inclusive
//     prefix of their out-degrees and walked 32 at a time, a lane per edge:
//     atomicMin on the destination's label; a lowered label sets the row's bit
//     in the next bitmap, and the claim that sets it appends the row.
// Labels change in place (a round may carry a label further than one hop);
// every lowered label enters the next frontier, so the fixed point is the same.
#include <algorithm>
#include <climits>
#include <cub/cub.cuh>

#include "gi_internal.cuh"

namespace gi {
namespace {

constexpr int kCT = 256;
constexpr int kCcHeavy = 32;      // rows of at least this many in-edges: the heavy kernel (ms_prepare's chunks)
constexpr int kCcHChunk = 1024;   // in-edges per heavy chunk (as ms_prepare cuts them)
// direction rule: BFS's (R7), pull iff |F| + sum outdeg F > m / 20. A CC pull
// row has no early exit, but the pull streams the CSC while the push scatters
// atomics: m/3 and m/8 measured slower or equal on RMAT and the grid
constexpr int kCcPullDiv = 20;

struct CcArgs {
  int64_t n;
  const void* csr_off;
  const int32_t* __restrict__ csr_idx;
  const void* csc_off;
  const int32_t* __restrict__ csc_idx;
  const int32_t* __restrict__ outdeg;
  int32_t* ids;                         // labels (input ids), internal order
  const uint32_t* __restrict__ bcur;    // frontier bitmap
  uint32_t* bnext;                      // next frontier bitmap (zeroed before the round)
  const int32_t* __restrict__ qcur;     // frontier queue (push rounds)
  int32_t* qnext;                       // next frontier queue
  unsigned long long* cnt;              // [0] |F'|, [1] sum outdeg F', [2] edges examined
  int64_t nf;                           // |F| (push)
  const int32_t* __restrict__ wcsr;     // SSSP: edge weights in CSR / CSC order
  const int32_t* __restrict__ wcsc;
};

__device__ __forceinline__ int32_t vload(const int32_t* p) { return *(volatile const int32_t*)p; }

// append the rows whose bit this warp set (+ their degrees) through a per-warp
// shared-memory buffer: one atomicAdd on the queue tail per 32 rows (a tail
// shared by every warp is a serialisation point)
__device__ __forceinline__ void cc_flush(const CcArgs& A, int32_t* buf, int cnt) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  unsigned long long pos = 0;
  if (lane == 0) pos = atomicAdd(&A.cnt[0], (unsigned long long)cnt);
  pos = __shfl_sync(0xffffffffu, pos, 0);
  if (lane < cnt) A.qnext[pos + lane] = buf[lane];
  __syncwarp();
}
__device__ __forceinline__ void cc_append(const CcArgs& A, bool add, int32_t w, unsigned long long& deg,
                                          int32_t* buf, int& nbuf) {
  const int lane = threadIdx.x & 31;
  const unsigned am = __ballot_sync(0xffffffffu, add);
  if (!am) return;
  if (add) {
    buf[nbuf + __popc(am & ((1u << lane) - 1u))] = w;
    deg += (unsigned long long)__ldg(&A.outdeg[w]);
  }
  nbuf += __popc(am);
  if (nbuf >= 32) {
    cc_flush(A, buf, 32);
    nbuf -= 32;
    if (lane < nbuf) buf[lane] = buf[32 + lane];
    __syncwarp();
  }
}

__device__ __forceinline__ void cc_counters(const CcArgs& A, unsigned long long deg, unsigned long long exam) {
  for (int o = 16; o > 0; o >>= 1) {
    deg += __shfl_xor_sync(0xffffffffu, deg, o);
    exam += __shfl_xor_sync(0xffffffffu, exam, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (deg) atomicAdd(&A.cnt[1], deg);
    if (exam) atomicAdd(&A.cnt[2], exam);
  }
}

// IDs[v] = input id of v; frontier = every vertex (bitmap) and, for a push
// first round, the queue 0..n-1
__global__ void k_cc_init(int32_t* __restrict__ ids, const int32_t* __restrict__ perm, int64_t n,
                          uint32_t* __restrict__ bm, int32_t* __restrict__ q, int fill_queue) {
  const int64_t words = (n + 31) >> 5;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n || i < words;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n) {
      ids[i] = perm ? __ldg(&perm[i]) : (int32_t)i;
      if (fill_queue) q[i] = (int32_t)i;
    }
    if (i < words) bm[i] = i + 1 < words || (n & 31) == 0 ? 0xffffffffu : ((1u << (n & 31)) - 1u);
  }
}

// pull over the light rows: a thread per row, a warp per 32 consecutive rows
// (one atomicOr sets their bits in the next bitmap)
// W (SSSP): the value a frontier in-neighbour u offers over edge e is
// dist[u] + w(e); otherwise (CC) its label
template <typename OffT, bool W>
__global__ void __launch_bounds__(kCT) k_cc_pull(CcArgs A) {
  __shared__ int32_t s_buf[kCT / 32][64];
  const OffT* __restrict__ off = static_cast<const OffT*>(A.csc_off);
  const int lane = threadIdx.x & 31;
  int32_t* buf = s_buf[threadIdx.x >> 5];
  int nbuf = 0;
  unsigned long long deg = 0, exam = 0;
  for (int64_t b = (blockIdx.x * (int64_t)kCT + threadIdx.x) & ~31ll; b < A.n; b += (int64_t)gridDim.x * kCT) {
    const int64_t w = b + lane;
    bool changed = false;
    if (w < A.n) {
      const int64_t e0 = (int64_t)off[w], e1 = (int64_t)off[w + 1];
      if (e1 - e0 < kCcHeavy && e1 > e0) {
        int32_t best = INT_MAX;
        for (int64_t e = e0; e < e1; e += 4) {
          int32_t u[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) u[j] = e + j < e1 ? __ldg(&A.csc_idx[e + j]) : -1;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (u[j] >= 0 && ((__ldg(&A.bcur[u[j] >> 5]) >> (u[j] & 31)) & 1u))
              best = min(best, vload(&A.ids[u[j]]) + (W ? __ldg(&A.wcsc[e + j]) : 0));
        }
        exam += (unsigned long long)(e1 - e0);
        if (best < vload(&A.ids[w])) {  // the only writer of a light row in a pull round
          A.ids[w] = best;
          changed = true;
        }
      }
    }
    const unsigned word = __ballot_sync(0xffffffffu, changed);
    if (word && lane == 0) atomicOr(&A.bnext[b >> 5], word);  // (b is a multiple of 32)
    cc_append(A, changed, (int32_t)w, deg, buf, nbuf);
  }
  if (nbuf > 0) cc_flush(A, buf, nbuf);
  cc_counters(A, deg, exam);
}

// pull over the heavy rows: a warp per chunk (row, first in-edge)
template <typename OffT, bool W>
__global__ void __launch_bounds__(kCT) k_cc_pull_heavy(CcArgs A, const int2* __restrict__ hch, int64_t C) {
  __shared__ int32_t s_buf[kCT / 32][64];
  const OffT* __restrict__ off = static_cast<const OffT*>(A.csc_off);
  const int lane = threadIdx.x & 31;
  int32_t* buf = s_buf[threadIdx.x >> 5];
  int nbuf = 0;
  const int64_t nw = (int64_t)gridDim.x * (kCT / 32);
  unsigned long long deg = 0, exam = 0;
  for (int64_t c = blockIdx.x * (int64_t)(kCT / 32) + (threadIdx.x >> 5); c < C; c += nw) {
    const int2 ch = __ldg(&hch[c]);
    const int32_t w = ch.x;
    const int64_t e0 = (int64_t)off[w] + ch.y, e1 = min((int64_t)off[w + 1], e0 + kCcHChunk);
    int32_t best = INT_MAX;
    for (int64_t b = e0; b < e1; b += 32 * 4) {
      int32_t u[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t e = b + 32 * j + lane;
        u[j] = e < e1 ? __ldg(&A.csc_idx[e]) : -1;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (u[j] >= 0 && ((__ldg(&A.bcur[u[j] >> 5]) >> (u[j] & 31)) & 1u))
          best = min(best, vload(&A.ids[u[j]]) + (W ? __ldg(&A.wcsc[b + 32 * j + lane]) : 0));
    }
    if (lane == 0) exam += (unsigned long long)(e1 - e0);
    best = __reduce_min_sync(0xffffffffu, best);
    bool add = false;
    if (lane == 0 && best < vload(&A.ids[w]) && best < atomicMin(&A.ids[w], best)) {  // this chunk lowered it
      const uint32_t bit = 1u << (w & 31);
      add = !(atomicOr(&A.bnext[w >> 5], bit) & bit);
    }
    cc_append(A, add, w, deg, buf, nbuf);
  }
  if (nbuf > 0) cc_flush(A, buf, nbuf);
  cc_counters(A, deg, exam);
}


// push: the frontier's out-edges (dp = inclusive prefix of their out-degrees)
// split evenly over the warps, 32 per step; a lane finds its edge's vertex in
// a window of 32 prefix entries by a 5-step shuffle search
template <typename OffT, bool W>
__global__ void __launch_bounds__(kCT) k_cc_push(CcArgs A, const long long* __restrict__ dp) {
  __shared__ int32_t s_buf[kCT / 32][64];
  const OffT* __restrict__ off = static_cast<const OffT*>(A.csr_off);
  const int lane = threadIdx.x & 31;
  int32_t* buf = s_buf[threadIdx.x >> 5];
  int nbuf = 0;
  const int64_t nw = (int64_t)gridDim.x * (kCT / 32);
  const int64_t gw = blockIdx.x * (int64_t)(kCT / 32) + (threadIdx.x >> 5);
  unsigned long long deg = 0, exam = 0;
  const long long E = A.nf > 0 ? __ldg(&dp[A.nf - 1]) : 0;
  const long long per = (E + nw - 1) / nw;
  long long e = gw * per;
  const long long eend = min(E, e + per);
  if (e < eend) {
    int64_t i0 = 0, hi = A.nf;
    while (i0 < hi) {
      const int64_t mid = (i0 + hi) >> 1;
      if (__ldg(&dp[mid]) <= e) i0 = mid + 1;
      else hi = mid;
    }
    while (e < eend) {
      const long long P = i0 + lane < A.nf ? __ldg(&dp[i0 + lane]) : LLONG_MAX;
      const long long Pprev = i0 > 0 ? __ldg(&dp[i0 - 1]) : 0;
      const long long stop = min(eend, min(e + 32, (long long)__shfl_sync(0xffffffffu, P, 31)));
      const long long my = e + lane;
      int pos = 0;
#pragma unroll
      for (int s = 16; s > 0; s >>= 1)
        if (__shfl_sync(0xffffffffu, P, pos + s - 1) <= my) pos += s;
      const long long pl = __shfl_sync(0xffffffffu, P, pos > 0 ? pos - 1 : 0);
      const long long start = pos ? pl : Pprev;
      bool add = false;
      int32_t w = 0;
      if (my < stop) {
        const int32_t u = __ldg(&A.qcur[i0 + pos]);
        const int64_t ei = (int64_t)off[u] + (my - start);
        w = __ldg(&A.csr_idx[ei]);
        ++exam;
        const int32_t lu = vload(&A.ids[u]) + (W ? __ldg(&A.wcsr[ei]) : 0);
        if (lu < vload(&A.ids[w]) && lu < atomicMin(&A.ids[w], lu)) {  // this edge lowered w's label
          const uint32_t bit = 1u << (w & 31);
          add = !(atomicOr(&A.bnext[w >> 5], bit) & bit);
        }
      }
      cc_append(A, add, w, deg, buf, nbuf);
      i0 += __popc(__ballot_sync(0xffffffffu, P <= stop));
      e = stop;
    }
  }
  if (nbuf > 0) cc_flush(A, buf, nbuf);
  cc_counters(A, deg, exam);
}

// after a segmented min pass (every in-neighbour, not only F's: the labels only
// fall, so the fixed point is the same): IDs[v] = min(IDs[v], acc[v]); a row
// whose label dropped joins the next frontier
__global__ void __launch_bounds__(kCT) k_cc_apply(CcArgs A, const int32_t* __restrict__ acc) {
  __shared__ int32_t s_buf[kCT / 32][64];
  const int lane = threadIdx.x & 31;
  int32_t* buf = s_buf[threadIdx.x >> 5];
  int nbuf = 0;
  unsigned long long deg = 0;
  for (int64_t b = (blockIdx.x * (int64_t)kCT + threadIdx.x) & ~31ll; b < A.n; b += (int64_t)gridDim.x * kCT) {
    const int64_t w = b + lane;
    bool changed = false;
    if (w < A.n) {
      const int32_t a = acc[w];
      if (a < A.ids[w]) {
        A.ids[w] = a;
        changed = true;
      }
    }
    const unsigned word = __ballot_sync(0xffffffffu, changed);
    if (word && lane == 0) A.bnext[b >> 5] = word;
    cc_append(A, changed, (int32_t)w, deg, buf, nbuf);
  }
  if (nbuf > 0) cc_flush(A, buf, nbuf);
  cc_counters(A, deg, 0);
}

// out[input id of v] = IDs[v]
__global__ void k_cc_out(const int32_t* __restrict__ ids, const int32_t* __restrict__ perm, int64_t n,
                         int32_t* __restrict__ out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    out[perm ? __ldg(&perm[v]) : v] = ids[v];
}

// SSSP: out[input id of v] = dist[v], -1 when unreachable
__global__ void k_sssp_out(const int32_t* __restrict__ dist, const int32_t* __restrict__ perm, int64_t n,
                           int32_t* __restrict__ out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t d = dist[v];
    out[perm ? __ldg(&perm[v]) : v] = d == INT_MAX ? -1 : d;
  }
}

// SSSP: dist = "infinity" except the source; frontier {source}
__global__ void k_sssp_init(int32_t* __restrict__ dist, int64_t n, int32_t s, uint32_t* __restrict__ bm,
                            int32_t* __restrict__ q) {
  const int64_t words = (n + 31) >> 5;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n || i < words;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n) dist[i] = i == s ? 0 : INT_MAX;
    if (i < words) bm[i] = i == (s >> 5) ? 1u << (s & 31) : 0u;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) q[0] = s;
}

// The synthetic weight of edge (u, v), input ids: the library's copy of
// graphgen's counter-based generator (R24), 1 + mix64(mix64(seed) + (u << 32 | v)) % 255
__device__ __forceinline__ uint64_t w_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ int32_t edge_weight(uint64_t key, int32_t u, int32_t v) {
  return 1 + (int32_t)(w_mix64(key + (((uint64_t)(uint32_t)u << 32) | (uint32_t)v)) % 255u);
}

// weights of every edge of a CSR (src_is_row) or CSC layout, a warp per row
template <typename OffT>
__global__ void k_edge_weights(const OffT* __restrict__ off, const int32_t* __restrict__ idx, int64_t n,
                               const int32_t* __restrict__ perm, uint64_t key, bool src_is_row,
                               int32_t* __restrict__ w) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
    const int32_t ri = perm ? __ldg(&perm[r]) : (int32_t)r;
    for (int64_t e = (int64_t)off[r] + lane; e < (int64_t)off[r + 1]; e += 32) {
      const int32_t x = __ldg(&idx[e]);
      const int32_t xi = perm ? __ldg(&perm[x]) : x;
      w[e] = src_is_row ? edge_weight(key, ri, xi) : edge_weight(key, xi, ri);
    }
  }
}

// caller weights (w_user: int32[m] in the input-id CSR order, rows ascending,
// neighbours ascending) moved to the internal CSR (src_is_row) or CSC layout: a
// warp per internal row, each edge's input-id CSR position by binary search
template <typename OffT>
__global__ void k_map_weights(const OffT* __restrict__ off, const int32_t* __restrict__ idx, int64_t n,
                              const int32_t* __restrict__ perm, const int64_t* __restrict__ ioff,
                              const int32_t* __restrict__ iidx, const int32_t* __restrict__ w_user, bool src_is_row,
                              int32_t* __restrict__ w) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
    const int32_t ri = perm ? __ldg(&perm[r]) : (int32_t)r;
    for (int64_t e = (int64_t)off[r] + lane; e < (int64_t)off[r + 1]; e += 32) {
      const int32_t x = __ldg(&idx[e]);
      const int32_t xi = perm ? __ldg(&perm[x]) : x;
      const int32_t u = src_is_row ? ri : xi, v = src_is_row ? xi : ri;
      int64_t lo = ioff[u], hi = ioff[u + 1];
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(&iidx[mid]) < v) lo = mid + 1;
        else hi = mid;
      }
      w[e] = __ldg(&w_user[lo]);
    }
  }
}

// host side of graphgen's key: mix64(seed)
static uint64_t h_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// CC (W = false) or SSSP from `source` (W = true, weights drawn with `seed`)
template <typename OffT, bool W>
gi_status cc_t(gi_graph g, const gi_cc_opts& o, int32_t source, uint64_t seed, int32_t* d_out, gi_cc_stats* stats,
               const int32_t* w_user = nullptr) {
  gi_context ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  const int64_t n = g->n, words = (n + 31) >> 5;
  auto& M = g->ms;
  GI_TRY(ms_prepare(g));
  auto& K = g->ccs;
  if (!K.ids.p) {
    GI_TRY(K.ids.alloc((n + 1) * 4));
    for (int c = 0; c < 2; ++c) GI_TRY(K.bm[c].alloc((words + 1) * 4));
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (o.profile) {
    GI_CUDA(cudaEventCreate(&e0));
    GI_CUDA(cudaEventCreate(&e1));
    GI_CUDA(cudaEventRecord(e0, st));
  }
  const int64_t mdiv = g->m / (o.threshold_div > 0 ? o.threshold_div : kCcPullDiv);
  const int32_t* perm = g->relabeled ? g->perm.as<int32_t>() : nullptr;
  unsigned long long* cnt = M.cnt.as<unsigned long long>();
  int64_t* h = ctx->h_scratch;
  int launches = 1, rounds = 0, pulls = 0;
  int64_t nf = n, sdeg = g->m, examined = 0;
  // CC pull rounds use the segmented layout when the graph has one (skewed,
  // relabelled graphs; built on first use, shared with PageRank)
  static const bool seg_env = !getenv("GI_CC_SEG") || atoi(getenv("GI_CC_SEG")) != 0;
  bool seg = false;
  if (!W && seg_env && g->relabeled && g->ctx->nranks == 1 && g->ml > 0 && seg_build(g, 0, 0) == GI_OK) {
    seg = true;
    if (!K.acc.p) GI_TRY(K.acc.alloc((n + 64) * 4));
  }
  if (W) {  // weights of this seed (cached with the graph) or the caller's, dist, frontier {source}
    if (w_user) {  // explicit weights in input-id CSR order -> internal CSR and CSC order
      if (!K.wcsr.p) {
        GI_TRY(K.wcsr.alloc((g->m + 1) * 4));
        GI_TRY(K.wcsc.alloc((g->m + 1) * 4));
      }
      DevBuf ioff, iidx;
      GI_TRY(csr_input_ids(g, ioff, iidx));
      k_map_weights<OffT><<<grid_for(n * 32, 256, sms, 16), 256, 0, st>>>(
          g->csr_off.as<OffT>(), g->csr_idx.as<int32_t>(), n, perm, ioff.as<int64_t>(), iidx.as<int32_t>(), w_user,
          true, K.wcsr.as<int32_t>());
      k_map_weights<OffT><<<grid_for(n * 32, 256, sms, 16), 256, 0, st>>>(
          g->csc_off.as<OffT>(), g->csc_idx.as<int32_t>(), n, perm, ioff.as<int64_t>(), iidx.as<int32_t>(), w_user,
          false, K.wcsc.as<int32_t>());
      GI_CUDA(cudaStreamSynchronize(st));  // ioff / iidx are released below
      launches += 2;
      K.w_ready = false;  // the cache no longer holds a seed's weights
    } else if (!K.w_ready || K.w_seed != seed) {
      if (!K.wcsr.p) {
        GI_TRY(K.wcsr.alloc((g->m + 1) * 4));
        GI_TRY(K.wcsc.alloc((g->m + 1) * 4));
      }
      const uint64_t key = h_mix64(seed);
      k_edge_weights<OffT><<<grid_for(n * 32, 256, sms, 16), 256, 0, st>>>(
          g->csr_off.as<OffT>(), g->csr_idx.as<int32_t>(), n, perm, key, true, K.wcsr.as<int32_t>());
      k_edge_weights<OffT><<<grid_for(n * 32, 256, sms, 16), 256, 0, st>>>(
          g->csc_off.as<OffT>(), g->csc_idx.as<int32_t>(), n, perm, key, false, K.wcsc.as<int32_t>());
      launches += 2;
      K.w_ready = true;
      K.w_seed = seed;
    }
    int32_t s = source;  // internal id of the source
    if (g->relabeled) {
      GI_CUDA(cudaMemcpyAsync(&s, g->inv.as<int32_t>() + source, 4, cudaMemcpyDeviceToHost, st));
      GI_CUDA(cudaStreamSynchronize(st));
    }
    k_sssp_init<<<grid_for(std::max(n, words), 256, sms), 256, 0, st>>>(K.ids.as<int32_t>(), n, s,
                                                                       K.bm[0].as<uint32_t>(), M.act[0].as<int32_t>());
    int32_t od = 0;
    GI_CUDA(cudaMemcpyAsync(&od, g->outdeg.as<int32_t>() + s, 4, cudaMemcpyDeviceToHost, st));
    GI_CUDA(cudaStreamSynchronize(st));
    nf = 1;
    sdeg = od;
  } else {  // CC round 0: every vertex in the frontier (|F| = n, sum outdeg = m)
    const bool first_push = o.policy == GI_BFS_PUSH_ONLY;
    k_cc_init<<<grid_for(std::max(n, words), 256, sms), 256, 0, st>>>(K.ids.as<int32_t>(), perm, n,
                                                                    K.bm[0].as<uint32_t>(), M.act[0].as<int32_t>(),
                                                                    first_push ? 1 : 0);
  }
  CcArgs A{};
  A.n = n;
  A.csr_off = g->csr_off.p;
  A.csr_idx = g->csr_idx.as<int32_t>();
  A.csc_off = g->csc_off.p;
  A.csc_idx = g->csc_idx.as<int32_t>();
  A.outdeg = g->outdeg.as<int32_t>();
  A.ids = K.ids.as<int32_t>();
  A.cnt = cnt;
  A.wcsr = W ? K.wcsr.as<int32_t>() : nullptr;
  A.wcsc = W ? K.wcsc.as<int32_t>() : nullptr;
  for (int r = 0; nf > 0; ++r) {
    const int c = r & 1;
    A.bcur = K.bm[c].as<uint32_t>();
    A.bnext = K.bm[c ^ 1].as<uint32_t>();
    A.qcur = M.act[c].as<int32_t>();
    A.qnext = M.act[c ^ 1].as<int32_t>();
    A.nf = nf;
    GI_CUDA(cudaMemsetAsync(A.bnext, 0, words * 4, st));
    GI_CUDA(cudaMemsetAsync(cnt, 0, 3 * 8, st));
    const bool pull = (o.policy == GI_BFS_PULL_ONLY && (r > 0 || !W)) || (o.policy == GI_BFS_AUTO && nf + sdeg > mdiv);
    if (pull && seg) {  // CC: a min pass over the segmented layout, then the label update
      GI_CUDA(cudaMemsetAsync(K.acc.p, 0x7F, (n + 64) * 4, st));  // 0x7F7F7F7F exceeds every label
      GI_TRY(seg_min_pass(g, K.ids.as<int32_t>(), K.acc.as<int32_t>()));
      k_cc_apply<<<grid_for(n, kCT, sms, 16), kCT, 0, st>>>(A, K.acc.as<int32_t>());
      launches += 2;
      examined += g->m;
      ++pulls;
    } else if (pull) {
      k_cc_pull<OffT, W><<<grid_for(n, kCT, sms, 16), kCT, 0, st>>>(A);
      ++launches;
      if (M.nhch > 0) {
        k_cc_pull_heavy<OffT, W><<<grid_for(M.nhch * 32, kCT, sms, 16), kCT, 0, st>>>(A, M.hch.as<int2>(), M.nhch);
        ++launches;
      }
      ++pulls;
    } else {
      long long* dp = M.chunks[1].as<long long>();
      size_t tb = M.scan_bytes;
      GI_CUDA(cub::DeviceScan::InclusiveSum(
          M.scan_tmp.p, tb, cub::TransformInputIterator<long long, OutdegOf, const int32_t*>(A.qcur, OutdegOf{A.outdeg}),
          dp, (int)nf, st));
      k_cc_push<OffT, W><<<grid_for((sdeg + 255) / 256 * 32, kCT, sms, 8), kCT, 0, st>>>(A, dp);
      launches += 3;  // scan (2) + push
    }
    GI_CUDA(cudaGetLastError());
    GI_CUDA(cudaMemcpyAsync(h, cnt, 3 * 8, cudaMemcpyDeviceToHost, st));
    GI_CUDA(stream_wait(st));
    nf = h[0];
    sdeg = h[1];
    examined += h[2];
    ++rounds;
  }
  if (W) k_sssp_out<<<grid_for(n, 256, sms), 256, 0, st>>>(K.ids.as<int32_t>(), perm, n, d_out);
  else k_cc_out<<<grid_for(n, 256, sms), 256, 0, st>>>(K.ids.as<int32_t>(), perm, n, d_out);
  ++launches;
  GI_CUDA(cudaGetLastError());
  float ms = 0.f;
  if (o.profile) {
    GI_CUDA(cudaEventRecord(e1, st));
    GI_CUDA(cudaEventSynchronize(e1));
    GI_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  if (stats) {
    gi_cc_stats s{};
    s.rounds = rounds;
    s.pull_rounds = pulls;
    s.edges_examined = examined;
    s.total_ms = ms;
    s.launches = launches;
    *stats = s;
  }
  return GI_OK;
}

}  // namespace

gi_status cc_run(gi_graph g, const gi_cc_opts& o, int32_t* d_out, gi_cc_stats* stats) {
  if (g->n == 0) {
    if (stats) *stats = gi_cc_stats{};
    return GI_OK;
  }
  return g->off64 ? cc_t<int64_t, false>(g, o, 0, 0, d_out, stats) : cc_t<int32_t, false>(g, o, 0, 0, d_out, stats);
}

gi_status sssp_run(gi_graph g, int32_t source, uint64_t seed, const int32_t* w_user, const gi_cc_opts& o,
                   int32_t* d_out, gi_cc_stats* stats) {
  return g->off64 ? cc_t<int64_t, true>(g, o, source, seed, d_out, stats, w_user)
                  : cc_t<int32_t, true>(g, o, source, seed, d_out, stats, w_user);
}

}  // namespace gi
