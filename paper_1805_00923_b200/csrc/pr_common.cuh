// pr_common.cuh — device pieces shared by the pull-PageRank kernels.
//
// Merge-path tile reduction (the paper's edge-aware
// vertex chunking, at thread granularity): a CSR-like
// sequence of rows r (CSC rows, or (segment, row) pieces) is laid out as
// items — each row's edges followed by one end marker — so row r occupies
// merge positions [r + off[r], r + off[r+1]]. A tile is a fixed range of
// positions [p0, p1); each thread walks IPT consecutive positions. Rows that
// cross thread boundaries are joined with a block-wide segmented scan of the
// threads' carry-outs (no atomics); rows that cross the tile boundary are
// reported to the caller once per tile (`split`).
#pragma once
#include "gi_internal.cuh"

namespace gi {

struct PrArgs {
  int64_t n, m;     // CSC rows and edges held here (single GPU: all)
  int64_t row0;     // global id of local row 0 (destination partition)
  const void* off;
  const int32_t* __restrict__ idx;
  const int32_t* __restrict__ tile_rows;
  const float* __restrict__ cin;
  float* __restrict__ cout;
  const int32_t* __restrict__ outdeg;
  double* dbuf;  // dangling-mass ring (3 slots)
  int it;
  float base, damp;
  double inv_n;
  int uniform;
  double* split_acc;
  int32_t* split_cnt;
  float* rank_out;  // non-null on the final iteration (input ids)
  const int32_t* __restrict__ perm;
  // source-partitioned pull: pmode 0 = one pass (finish every row), 1 = first
  // partition (pacc = s), 2 = middle (pacc += s), 3 = last (finish with pacc + s)
  float* pacc;
  int pmode;
  // multi-GPU peer stores: the new contrib of an owned row is also written
  // into the other ranks' replicas (replaces the per-iteration allgather)
  float* peer[7];
  int npeer;
};

// vertex update (a3): r' = base + d (s + D/n); contrib' = r'/outdeg; dangling partial
// (r is a local row; outdeg, contrib and perm are indexed by global id row0 + r)
__device__ __forceinline__ void pr_epilogue(const PrArgs& A, int64_t r, float s, float dn, double& dpart) {
  const int64_t v = A.row0 + r;
  const float rn = A.base + A.damp * (s + dn);
  const int od = __ldg(&A.outdeg[v]);
  const float c = od > 0 ? rn / (float)od : 0.f;
  A.cout[v] = c;
  for (int q = 0; q < A.npeer; ++q) A.peer[q][v] = c;
  if (od == 0) dpart += (double)rn;
  if (A.rank_out) A.rank_out[A.perm ? __ldg(&A.perm[v]) : v] = rn;
}

// Block sum of a double; result valid in thread 0. sred: >= 32 doubles.
__device__ __forceinline__ double block_sum(double v, double* sred) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sred[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < (blockDim.x >> 5) ? sred[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  return t;
}

struct KeyVal {
  int key;
  float val;
};

// combine(a, b) for b following a in thread order: same key -> sum, else b.
__device__ __forceinline__ KeyVal kv_combine(KeyVal a, KeyVal b) {
  return KeyVal{b.key, b.key == a.key ? a.val + b.val : b.val};
}

// Block-wide segmented scan over (key, val) in thread order; keys are
// non-decreasing across threads. Returns the exclusive prefix (the running
// sum of the run of equal keys ending at thread t-1; key -1 for thread 0) and
// writes the inclusive value. scratch: NT/32 KeyVal in smem.
template <int NT>
__device__ __forceinline__ KeyVal seg_scan(KeyVal x, KeyVal& incl, KeyVal* scratch) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  KeyVal run = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    KeyVal up;
    up.key = __shfl_up_sync(0xffffffffu, run.key, o);
    up.val = __shfl_up_sync(0xffffffffu, run.val, o);
    if (lane >= o) run = kv_combine(up, run);
  }
  if (lane == 31) scratch[w] = run;
  __syncthreads();
  if (w == 0) {
    KeyVal t = lane < NT / 32 ? scratch[lane] : KeyVal{0x7fffffff, 0.f};
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      KeyVal up;
      up.key = __shfl_up_sync(0xffffffffu, t.key, o);
      up.val = __shfl_up_sync(0xffffffffu, t.val, o);
      if (lane >= o) t = kv_combine(up, t);
    }
    if (lane < NT / 32) scratch[lane] = t;  // inclusive prefix over warps
  }
  __syncthreads();
  KeyVal wpre = w > 0 ? scratch[w - 1] : KeyVal{-1, 0.f};
  incl = kv_combine(wpre, run);
  KeyVal ex;
  ex.key = __shfl_up_sync(0xffffffffu, run.key, 1);
  ex.val = __shfl_up_sync(0xffffffffu, run.val, 1);
  if (lane == 0) ex = wpre;
  else ex = kv_combine(wpre, ex);
  return ex;
}

// One tile of the merge-path reduction, in tile-local 32-bit coordinates.
//   loff[i], i in [0, R]: first edge of row i relative to the tile's first
//     edge, clamped to [-1, items + 1] (only row 0 can start before the tile,
//     only row R-1 can end after it); row i occupies local items
//     [i + loff[i], i + loff[i+1]] (its edges, then its end marker)
//   sval[e]: value of the tile's local edge e
//   complete(i, v): row i starts and ends inside the tile; v is its sum
//   split(i, v):    row i crosses the tile boundary; v is this tile's part
//                   (called exactly once per such row per tile)
// Must be called by all NT threads (contains __syncthreads).
template <int NT, int IPT, typename Complete, typename Split>
__device__ __forceinline__ void tile_walk(const int* loff, int R, int items, const float* sval, KeyVal* scratch,
                                          Complete&& complete, Split&& split) {
  const int q0 = threadIdx.x * IPT;
  const int q1 = min(q0 + IPT, items);
  const bool active = q0 < items;
  int i = R;  // current row
  float acc = 0.f, head_val = 0.f;
  int head = -1;  // row completed in this window that started before it
  if (active) {
    int lo = 0, hi = R - 1;  // row containing q0: min i with i + loff[i+1] >= q0
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (mid + loff[mid + 1] >= q0) hi = mid;
      else lo = mid + 1;
    }
    i = lo;
    int e = q0 - i;
    bool own = i + loff[i] >= q0;
    int pe = i + loff[i + 1];
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      const int q = q0 + k;
      if (q < q1) {
        if (q < pe) {
          acc += sval[e];
          ++e;
        } else {
          if (own) complete(i, acc);
          else {
            head = i;
            head_val = acc;
          }
          acc = 0.f;
          ++i;
          own = true;
          pe = i < R ? i + loff[i + 1] : 0x7fffffff;
        }
      }
    }
  }
  // carry-out: (row open at q1, its partial inside [q0, q1))
  KeyVal incl;
  const KeyVal ex = seg_scan<NT>(KeyVal{active ? i : 0x7fffffff, active ? acc : 0.f}, incl, scratch);
  if (head >= 0) {
    const float tot = head_val + (ex.key == head ? ex.val : 0.f);
    if (head + loff[head] >= 0) complete(head, tot);
    else split(head, tot);
  }
  // the last active thread reports the row still open at the tile end, if the tile holds part of it
  if (active && q1 == items && i < R && i + loff[i] < items) split(i, incl.val);
}

}  // namespace gi
