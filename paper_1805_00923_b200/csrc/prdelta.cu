// prdelta.cu — PageRankDelta through edgeset.apply (the
// paper's running example, PAPER.md Alg. PageRankDelta P:426-456 and the
// GraphIt program P:849-893).
//
//   Rank = 0, DeltaSum = 0, Delta = 1/V, Frontier = V
//   round r: DeltaSum[dst] += Delta[src] / OutDegree[src]  for src in Frontier
//            (edges.from(frontier).apply(updateEdge))
//            round 1: Delta = d*DeltaSum + (1-d)/V; Rank += Delta; Delta -= 1/V
//            later:   Delta = d*DeltaSum; Rank += Delta         (R17)
//            next Frontier = {v : |Delta[v]| > eps * Rank[v]}  (R18)
//
// The edge pass is DensePull-SparsePush: pull iff
// |F| + sum outdeg(F) > m / threshold_div. Pull reuses the segmented
// shared-memory kernel (pr_segmented.cu) with contrib[u] = Delta[u]/outdeg(u)
// for frontier members and 0 otherwise (the from(frontier) filter folded into
// the gathered value); push scatters Delta[u]/outdeg(u) from the frontier
// queue with fp64 red.global.add. One vertex kernel then applies the update,
// writes the next contrib, and appends the next frontier to a queue (one
// atomic per CTA) with its size and out-degree sum for the next direction
// decision.
#include <algorithm>
#include <cub/cub.cuh>

#include "gi_internal.cuh"
#include "pr_common.cuh"

namespace gi {
namespace {

constexpr int kVT = 256;

template <typename OffT>
struct PrdVertexArgs {
  int64_t n;
  const float* __restrict__ pacc;      // pull: per-vertex sums of the segmented pass
  float* __restrict__ pzero;           // pull: the other accumulator, zeroed here
  double* __restrict__ acc;            // push: per-vertex accumulator (zeroed here)
  const int32_t* __restrict__ outdeg;
  double* __restrict__ rank;           // fp64 like the paper's vectors: the frontier
                                       // test |Delta| > eps*Rank is decided in the paper's precision
  float* __restrict__ cnext;           // next round's contrib (0 outside the frontier)
  int32_t* __restrict__ qnext;         // next frontier queue
  unsigned long long* __restrict__ cn; // {|F'|, sum outdeg F'}
  double damp, base, inv_v, eps;
  int first;                           // round 1
};

template <typename OffT>
__global__ void __launch_bounds__(kVT) k_prd_vertex(PrdVertexArgs<OffT> A) {
  using Scan = cub::BlockScan<int, kVT>;
  using Red = cub::BlockReduce<long long, kVT>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ typename Red::TempStorage red_tmp;
  __shared__ long long s_base;
  for (int64_t b = blockIdx.x * (int64_t)kVT; b < A.n; b += (int64_t)gridDim.x * kVT) {
    const int64_t v = b + threadIdx.x;
    bool in = false;
    long long od = 0;
    if (v < A.n) {
      double ds;
      if (A.acc) {
        ds = A.acc[v];
        A.acc[v] = 0.0;
      } else {
        ds = (double)A.pacc[v];
        A.pzero[v] = 0.f;
      }
      double delta;
      if (A.first) {
        delta = A.damp * ds + A.base;
        A.rank[v] += delta;
        delta -= A.inv_v;
      } else {
        delta = ds * A.damp;
        A.rank[v] += delta;
      }
      in = fabs(delta) > A.eps * A.rank[v];
      const int d = __ldg(&A.outdeg[v]);
      A.cnext[v] = (in && d > 0) ? (float)(delta / (double)d) : 0.f;
      od = in ? d : 0;
    }
    int pos, tot;
    Scan(scan_tmp).ExclusiveSum((int)in, pos, tot);
    const long long dsum = Red(red_tmp).Sum(od);
    if (threadIdx.x == 0) {
      s_base = tot ? (long long)atomicAdd(&A.cn[0], (unsigned long long)tot) : 0;
      if (dsum) atomicAdd(&A.cn[1], (unsigned long long)dsum);
    }
    __syncthreads();
    if (in) A.qnext[s_base + pos] = (int32_t)v;
    __syncthreads();
  }
}

// SparsePush: every frontier vertex scatters its contribution along its out-edges
template <typename OffT>
__global__ void __launch_bounds__(256) k_prd_push(const int32_t* __restrict__ q, int64_t nf,
                                                  const OffT* __restrict__ off, const int32_t* __restrict__ idx,
                                                  const float* __restrict__ cin, double* __restrict__ acc) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < nf; i += nw) {
    const int32_t u = __ldg(&q[i]);
    const float c = __ldg(&cin[u]);
    if (c == 0.f) continue;
    for (int64_t j = (int64_t)off[u] + lane; j < (int64_t)off[u + 1]; j += 32)
      atomicAdd(&acc[__ldg(&idx[j])], (double)c);  // RED.E.ADD.F64
  }
}

__global__ void k_prd_init(int64_t n, const int32_t* __restrict__ outdeg, double* __restrict__ rank,
                           float* __restrict__ c0, int32_t* __restrict__ q, double inv_v) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    rank[v] = 0.0;
    const int d = outdeg[v];
    c0[v] = d > 0 ? (float)(inv_v / d) : 0.f;
    q[v] = (int32_t)v;  // round 1: Frontier = V
  }
}

__global__ void k_prd_out(const double* __restrict__ rank, const int32_t* __restrict__ perm, int64_t n,
                          float* __restrict__ out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    out[perm ? perm[v] : v] = (float)rank[v];
}

}  // namespace

template <typename OffT>
static gi_status prdelta_t(gi_graph g, int32_t iters, double damping, double eps, const gi_prdelta_opts& o,
                           float* d_out, gi_prdelta_stats* stats) {
  gi_context ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  const int64_t n = g->n, m = g->m;
  gi_prdelta_stats S{};
  const bool can_pull = o.policy != GI_PRD_PUSH_ONLY && seg_build(g, 0, 0) == GI_OK;
  if (o.policy == GI_PRD_PULL_ONLY && !can_pull)
    return fail(GI_ERR_UNSUPPORTED, "gi_pagerank_delta: pull needs the segmented layout (non-empty graph)");
  DevBuf rank, cbuf[2], q[2], acc, cnt;
  GI_TRY(rank.alloc(n * sizeof(double)));
  for (int k = 0; k < 2; ++k) {
    GI_TRY(cbuf[k].alloc((n + 16) * sizeof(float)));
    GI_TRY(q[k].alloc(n * sizeof(int32_t)));
  }
  GI_TRY(acc.alloc(n * sizeof(double)));
  GI_TRY(cnt.alloc(4 * sizeof(unsigned long long)));
  GI_CUDA(cudaMemsetAsync(acc.p, 0, n * sizeof(double), st));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (o.profile) {
    GI_CUDA(cudaEventCreate(&e0));
    GI_CUDA(cudaEventCreate(&e1));
    GI_CUDA(cudaEventRecord(e0, st));
  }
  const double inv_v = 1.0 / (double)n;
  k_prd_init<<<grid_for(n, 256, sms), 256, 0, st>>>(n, g->outdeg.as<int32_t>(), rank.as<double>(), cbuf[0].as<float>(),
                                                    q[0].as<int32_t>(), inv_v);
  S.launches++;
  int64_t nf = n, sdeg = m;
  const int div = o.threshold_div > 0 ? o.threshold_div : 20;
  unsigned long long* cn = cnt.as<unsigned long long>();
  int64_t* h = ctx->h_scratch;
  for (int r = 1; r <= iters && nf > 0; ++r) {
    const int cur = (r - 1) & 1, nxt = r & 1;
    bool pull = o.policy == GI_PRD_PULL_ONLY || (o.policy == GI_PRD_AUTO && can_pull && nf + sdeg > m / div);
    PrdVertexArgs<OffT> V{};
    V.n = n;
    V.outdeg = g->outdeg.as<int32_t>();
    V.rank = rank.as<double>();
    V.cnext = cbuf[nxt].as<float>();
    V.qnext = q[nxt].as<int32_t>();
    V.cn = cn;
    V.damp = damping;
    V.base = (1.0 - damping) / (double)n;
    V.inv_v = inv_v;
    V.eps = eps;
    V.first = r == 1;
    GI_CUDA(cudaMemsetAsync(cn, 0, 2 * sizeof(unsigned long long), st));
    if (pull) {
      GI_TRY(seg_edge_pass(g, cbuf[cur].as<float>()));  // seg_acc[v] = sum of contrib over in(v)
      V.pacc = seg_acc_buf(g, g->seg_acc_cur);
      V.pzero = seg_acc_buf(g, g->seg_acc_cur ^ 1);
      g->seg_acc_cur ^= 1;
      S.pull_rounds++;
      S.launches += 2;
    } else {
      if (sdeg > 0)
        k_prd_push<OffT><<<grid_for(nf * 32, 256, sms, 16), 256, 0, st>>>(
            q[cur].as<int32_t>(), nf, g->csr_off.as<OffT>(), g->csr_idx.as<int32_t>(), cbuf[cur].as<float>(),
            acc.as<double>());
      V.acc = acc.as<double>();
      S.launches++;
    }
    k_prd_vertex<OffT><<<grid_for(n, kVT, sms, 8), kVT, 0, st>>>(V);
    GI_CUDA(cudaGetLastError());
    S.launches++;
    S.rounds++;
    S.active_total += nf;
    GI_CUDA(cudaMemcpyAsync(h, cn, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    GI_CUDA(stream_wait(st));
    nf = h[0];
    sdeg = h[1];
  }
  k_prd_out<<<grid_for(n, 256, sms), 256, 0, st>>>(rank.as<double>(), g->relabeled ? g->perm.as<int32_t>() : nullptr, n,
                                                   d_out);
  S.launches++;
  GI_CUDA(cudaGetLastError());
  if (o.profile) {
    GI_CUDA(cudaEventRecord(e1, st));
    GI_CUDA(cudaEventSynchronize(e1));
    GI_CUDA(cudaEventElapsedTime(&S.total_ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  GI_CUDA(stream_wait(st));
  if (stats) *stats = S;
  return GI_OK;
}

gi_status prdelta_run(gi_graph g, int32_t iters, double damping, double eps, const gi_prdelta_opts& o, float* d_out,
                      gi_prdelta_stats* stats) {
  if (g->ctx->nranks > 1) return fail(GI_ERR_UNSUPPORTED, "gi_pagerank_delta: single-GPU graphs only");
  if (g->off64) return prdelta_t<int64_t>(g, iters, damping, eps, o, d_out, stats);
  return prdelta_t<int32_t>(g, iters, damping, eps, o, d_out, stats);
}

}  // namespace gi
