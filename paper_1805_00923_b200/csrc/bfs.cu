// bfs.cu — direction-optimising BFS through edgeset.apply (SURVEY §8(a) rows
// a6-a9, §2.7 K6-K9).
//
//  push level (SparsePush + to(unvisited) + applyModified without dedup,
//    PAPER.md P:1779-1808): for u in the sparse queue, for
//    v in out(u): if parent[v] == -1 and CAS(parent[v], -1, u) wins, append v.
//    The CAS is the claim that makes "each vertex inserted once" hold without
//    a dedup pass. Load balance: per-CTA exclusive scan of frontier degrees,
//    then the CTA walks the flattened edge list (the paper's edge-aware
//    chunking, at CTA granularity).
//  pull level (DensePull + bitvector frontier + early exit, P:600-601,
//    P:1812-1817): each warp owns 32 consecutive vertices = one
//    bitmap word; an unvisited vertex scans its in-edges until it finds a
//    frontier member; the next-frontier word is the warp ballot (no atomics).
//  direction (DensePull-SparsePush): pull iff
//    |F| + sum_{v in F} outdeg(v) > m / threshold_div (Ligra's m/20,
//    P:3074 [punt]; reading R7). Both counts are produced by the level
//    kernels themselves (warp-aggregated atomics), so the only host read per
//    level is two int64.
//  conversion: queue -> bitmap (atomicOr per id);
//    bitmap -> queue (popc + warp scan + one atomicAdd per warp).
#include <algorithm>
#include <climits>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cooperative_groups.h>
#include <cub/cub.cuh>

namespace cg = cooperative_groups;

#include "gi_internal.cuh"
#include "comm.cuh"

namespace gi {
namespace {

constexpr int kRing = 4;  // counter slots ring: slot(l) = cnt + 2*(l % kRing): {|F_l|, sum outdeg F_l}
constexpr int64_t kBalancedMin = 1 << 17;  // push levels with more frontier edges use k_bfs_push_bal
constexpr int64_t kPersistMax = 1 << 15;
constexpr int64_t kStampMin = 1 << 18;      // push levels with more frontier edges use stamp + collect   // push levels with fewer frontier edges run in k_bfs_persist

__global__ void k_bfs_init(int32_t s_in, const int32_t* __restrict__ inv, const int32_t* __restrict__ outdeg,
                           int32_t* __restrict__ parent, int32_t* __restrict__ q, int64_t* __restrict__ cnt) {
  const int32_t s = inv ? inv[s_in] : s_in;
  parent[s] = s;
  q[0] = s;
  cnt[0] = 1;
  cnt[1] = outdeg[s];
}

struct PushSmem {
  cub::BlockScan<long long, 256>::TempStorage scan;
  long long pre[257];
  long long beg[256];
  int32_t u[256];
};

// One push level over queue q[0, qlen) by this CTA's share of 256-vertex
// chunks (CTA-wide scan of degrees, then a balanced walk of the chunk's edges).
template <typename OffT>
__device__ __forceinline__ void push_chunks(const int32_t* __restrict__ q, int64_t qlen, const OffT* __restrict__ off,
                                            const int32_t* __restrict__ idx, const int32_t* __restrict__ outdeg,
                                            int32_t* parent, int32_t* __restrict__ qnext, int64_t* cnext,
                                            PushSmem& sm) {
  constexpr int NT = 256;
  using Scan = cub::BlockScan<long long, NT>;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int64_t c0 = (int64_t)blockIdx.x * NT; c0 < qlen; c0 += (int64_t)gridDim.x * NT) {
    const int64_t i = c0 + tid;
    long long deg = 0, beg = 0;
    int32_t u = -1;
    if (i < qlen) {
      u = q[i];
      beg = (long long)off[u];
      deg = (long long)off[u + 1] - beg;
    }
    long long pre, total;
    Scan(sm.scan).ExclusiveSum(deg, pre, total);
    sm.pre[tid] = pre;
    sm.beg[tid] = beg;
    sm.u[tid] = u;
    __syncthreads();
    for (long long base = 0; base < total; base += NT) {
      const long long f = base + tid;
      bool won = false;
      int32_t v = 0;
      if (f < total) {
        int lo = 0, hi = NT - 1;  // owner = last k with pre[k] <= f
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (sm.pre[mid] <= f) lo = mid;
          else hi = mid - 1;
        }
        const int32_t uu = sm.u[lo];
        v = __ldg(&idx[sm.beg[lo] + (f - sm.pre[lo])]);
        if (*(volatile int32_t*)&parent[v] == -1) won = atomicCAS(&parent[v], -1, uu) == -1;
      }
      const unsigned mask = __ballot_sync(0xffffffffu, won);
      if (mask) {
        long long od = won ? (long long)__ldg(&outdeg[v]) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) od += __shfl_xor_sync(0xffffffffu, od, o);
        long long pos = 0;
        if (lane == 0) {
          pos = atomicAdd((unsigned long long*)&cnext[0], (unsigned long long)__popc(mask));
          atomicAdd((unsigned long long*)&cnext[1], (unsigned long long)od);
        }
        pos = __shfl_sync(0xffffffffu, pos, 0);
        if (won) qnext[pos + __popc(mask & ((1u << lane) - 1))] = v;
      }
    }
    __syncthreads();
  }
}

// Small frontiers (nf <= kSmallF): every CTA of the grid scans the whole
// frontier's degrees in shared memory (cheap, redundant) and then walks an
// equal slice of the flattened edge list, so a frontier of a few hubs is
// spread over the whole grid instead of landing on one CTA.
constexpr int kSmallF = 4096;
struct SmallSmem {
  cub::BlockScan<int, 256>::TempStorage scan;
  int pre[kSmallF + 1];  // inclusive scan of degrees, pre[0] = 0
  int32_t u[kSmallF];
};

template <typename OffT>
__device__ __forceinline__ void push_small(const int32_t* __restrict__ q, int nf, const OffT* __restrict__ off,
                                           const int32_t* __restrict__ idx, const int32_t* __restrict__ outdeg,
                                           int32_t* parent, int32_t* __restrict__ qnext, int64_t* cnext,
                                           SmallSmem& sm) {
  constexpr int NT = 256, PT = kSmallF / NT;  // 16 frontier entries per thread
  const int tid = threadIdx.x, lane = tid & 31;
  int d[PT];
  int run = 0;
#pragma unroll
  for (int k = 0; k < PT; ++k) {  // thread t owns entries [t*PT, (t+1)*PT)
    const int i = tid * PT + k;
    d[k] = 0;
    if (i < nf) {
      const int32_t u = q[i];
      sm.u[i] = u;
      d[k] = (int)(off[u + 1] - off[u]);
    }
    run += d[k];
  }
  int excl, total;
  cub::BlockScan<int, NT>(sm.scan).ExclusiveSum(run, excl, total);
#pragma unroll
  for (int k = 0; k < PT; ++k) {
    const int i = tid * PT + k;
    if (i < nf) sm.pre[i] = excl;
    excl += d[k];
  }
  if (tid == 0) sm.pre[nf] = total;
  __syncthreads();
  const long long E = total;
  const long long lo = E * blockIdx.x / gridDim.x, hi = E * (blockIdx.x + 1) / gridDim.x;
  for (long long base = lo; base < hi; base += NT) {
    const long long f = base + tid;
    bool won = false;
    int32_t v = 0;
    if (f < hi) {
      int a = 0, b = nf - 1;  // owner = last i with pre[i] <= f
      while (a < b) {
        const int mid = (a + b + 1) >> 1;
        if (sm.pre[mid] <= f) a = mid;
        else b = mid - 1;
      }
      const int32_t uu = sm.u[a];
      v = __ldg(&idx[(long long)off[uu] + (f - sm.pre[a])]);
      if (*(volatile int32_t*)&parent[v] == -1) won = atomicCAS(&parent[v], -1, uu) == -1;
    }
    const unsigned mask = __ballot_sync(0xffffffffu, won);
    if (mask) {
      long long od = won ? (long long)__ldg(&outdeg[v]) : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) od += __shfl_xor_sync(0xffffffffu, od, o);
      long long pos = 0;
      if (lane == 0) {
        pos = atomicAdd((unsigned long long*)&cnext[0], (unsigned long long)__popc(mask));
        atomicAdd((unsigned long long*)&cnext[1], (unsigned long long)od);
      }
      pos = __shfl_sync(0xffffffffu, pos, 0);
      if (won) qnext[pos + __popc(mask & ((1u << lane) - 1))] = v;
    }
  }
  __syncthreads();
}

template <typename OffT>
__global__ void __launch_bounds__(256) k_bfs_push(const int32_t* __restrict__ q, int64_t qlen,
                                                  const OffT* __restrict__ off, const int32_t* __restrict__ idx,
                                                  const int32_t* __restrict__ outdeg, int32_t* parent,
                                                  int32_t* __restrict__ qnext, int64_t* __restrict__ cnext, int small) {
  __shared__ union {
    PushSmem chunks;
    SmallSmem small;
  } sm;
  if (small) push_small<OffT>(q, (int)qlen, off, idx, outdeg, parent, qnext, cnext, sm.small);
  else push_chunks<OffT>(q, qlen, off, idx, outdeg, parent, qnext, cnext, sm.chunks);
}

// Persistent small-frontier BFS (cooperative launch): runs consecutive push
// levels with a grid-wide barrier instead of a host round trip per level,
// until the frontier empties, the direction rule picks pull, or the frontier's
// edge count exceeds `small_max` (then the host continues with the level
// kernels). High-diameter graphs (config 3: thousands of tiny levels)
// spend their whole traversal here. state[0] = level, state[1] = current queue.
template <typename OffT>
__global__ void __launch_bounds__(256) k_bfs_persist(const OffT* __restrict__ off, const int32_t* __restrict__ idx,
                                                     const int32_t* __restrict__ outdeg, int32_t* parent,
                                                     int32_t* q0, int32_t* q1, int64_t* cnt, int64_t* state,
                                                     int64_t m_div, int64_t small_max, int policy) {
  __shared__ union {
    PushSmem chunks;
    SmallSmem small;
  } sm;
  cg::grid_group grid = cg::this_grid();
  int64_t level = state[0];
  int qc = (int)state[1];
  for (;;) {
    const int64_t* cur = cnt + 2 * (level % kRing);
    const int64_t nf = *(volatile const int64_t*)&cur[0];
    const int64_t sdeg = *(volatile const int64_t*)&cur[1];
    if (nf == 0) break;
    const bool pull = policy == GI_BFS_PULL_ONLY ? level > 0 : (policy == GI_BFS_AUTO && nf + sdeg > m_div);
    if (pull || sdeg > small_max) break;
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // slot for level + 2 (its old contents are two levels stale)
      int64_t* z = cnt + 2 * ((level + 2) % kRing);
      z[0] = 0;
      z[1] = 0;
    }
    if (nf <= kSmallF && sdeg < INT32_MAX)
      push_small<OffT>(qc ? q1 : q0, (int)nf, off, idx, outdeg, parent, qc ? q0 : q1, cnt + 2 * ((level + 1) % kRing),
                       sm.small);
    else
      push_chunks<OffT>(qc ? q1 : q0, nf, off, idx, outdeg, parent, qc ? q0 : q1, cnt + 2 * ((level + 1) % kRing),
                        sm.chunks);
    grid.sync();
    ++level;
    qc ^= 1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    state[0] = level;
    state[1] = qc;
  }
}

template <typename OffT>
__global__ void __launch_bounds__(256) k_bfs_pull(const uint32_t* __restrict__ fcur, uint32_t* __restrict__ fnext,
                                                  int32_t* __restrict__ parent, const OffT* __restrict__ off,
                                                  const int32_t* __restrict__ idx, const int32_t* __restrict__ outdeg,
                                                  int64_t n, int64_t* __restrict__ cnext) {
  const int lane = threadIdx.x & 31;
  const int64_t words = (n + 31) >> 5;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  long long cnt = 0, sdeg = 0;
  for (int64_t w = warp; w < words; w += nwarps) {
    const int64_t v = (w << 5) + lane;
    bool found = false;
    if (v < n && parent[v] == -1) {
      const int64_t e1 = (int64_t)off[v + 1];
      for (int64_t e = (int64_t)off[v]; e < e1; ++e) {
        const int32_t u = __ldg(&idx[e]);
        if ((__ldg(&fcur[u >> 5]) >> (u & 31)) & 1u) {
          parent[v] = u;
          found = true;
          break;
        }
      }
    }
    const unsigned mask = __ballot_sync(0xffffffffu, found);
    if (lane == 0) fnext[w] = mask;
    if (found) {
      cnt += 1;
      sdeg += __ldg(&outdeg[v]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    sdeg += __shfl_xor_sync(0xffffffffu, sdeg, o);
  }
  if (lane == 0 && cnt) {
    atomicAdd((unsigned long long*)&cnext[0], (unsigned long long)cnt);
    atomicAdd((unsigned long long*)&cnext[1], (unsigned long long)sdeg);
  }
}

// Multi-GPU BFS with peer stores (SURVEY §8(f) NEXT #3 for the frontier): the
// next-frontier words a rank produces for its owned range are also written into
// every other rank's replica of the bitmap (mapped through CUDA IPC), so no
// per-level allgather is needed. np = 0: local bitmap only.
struct PeerBits {
  uint32_t* p[7];
  int np;
};

// Pull level with the hot prefix of the frontier bitmap staged in shared
// memory (the north_star's "bitmap staged in shared memory"): vertices are
// relabelled hottest-first, so the first `sw` words (up to ~1.8 M vertices)
// answer almost every in-neighbour membership test from smem (~7 random
// reads / SM-clock measured) instead of L2 (~1). Two CTAs per SM, grid-stride
// over output words; each warp owns one word (32 vertices, ballot write).
template <typename OffT>
__global__ void __launch_bounds__(1024, 2) k_bfs_pull_smem(const uint32_t* __restrict__ fcur,
                                                           uint32_t* __restrict__ fnext, int32_t* __restrict__ parent,
                                                           const OffT* __restrict__ off,
                                                           const int32_t* __restrict__ idx,
                                                           const int32_t* __restrict__ outdeg, int64_t n, int sw,
                                                           int64_t* __restrict__ cnext, int64_t r0,
                                                           PeerBits peers) {
  // n = CSC rows held here, r0 = global id of row 0 (a multiple of 32);
  // parent is indexed by local row, fnext / outdeg by global id
  extern __shared__ uint32_t sbits[];
  for (int i = threadIdx.x; i < sw; i += blockDim.x) sbits[i] = __ldg(&fcur[i]);
  __syncthreads();
  const uint32_t lim = (uint32_t)sw * 32u;
  const int lane = threadIdx.x & 31;
  const int64_t words = (n + 31) >> 5;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  long long cnt = 0, sdeg = 0;
  for (int64_t w = warp; w < words; w += nwarps) {
    const int64_t v = (w << 5) + lane;
    bool found = false;
    if (v < n && parent[v] == -1) {
      // probe 4 in-edges per step (independent loads; rows are sorted by
      // source id = hottest first, so most vertices stop in the first step)
      const int64_t e1 = (int64_t)off[v + 1];
      for (int64_t e = (int64_t)off[v]; e < e1 && !found; e += 4) {
        uint32_t u[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) u[k] = e + k < e1 ? (uint32_t)__ldg(&idx[e + k]) : 0xffffffffu;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (!found && u[k] != 0xffffffffu) {
            const uint32_t word = u[k] < lim ? sbits[u[k] >> 5] : __ldg(&fcur[u[k] >> 5]);
            if ((word >> (u[k] & 31)) & 1u) {
              parent[v] = (int32_t)u[k];
              found = true;
            }
          }
        }
      }
    }
    const unsigned mask = __ballot_sync(0xffffffffu, found);
    if (lane < 1 + peers.np) (lane == 0 ? fnext : peers.p[lane - 1])[(r0 >> 5) + w] = mask;
    if (found) {
      cnt += 1;
      sdeg += __ldg(&outdeg[r0 + v]);
    }
  }
  if (peers.np) __threadfence_system();  // peer stores ordered before the level's allreduce
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    sdeg += __shfl_xor_sync(0xffffffffu, sdeg, o);
  }
  if (lane == 0 && cnt) {
    atomicAdd((unsigned long long*)&cnext[0], (unsigned long long)cnt);
    atomicAdd((unsigned long long*)&cnext[1], (unsigned long long)sdeg);
  }
}

// Edge-balanced push level (the paper's edge-parallel strategy):
// pre = exclusive scan of the frontier's out-degrees, E = their sum. Thread
// g owns flattened edges [g*EPT, (g+1)*EPT): one binary search for its first
// owner, then a forward walk, so a hub's edges spread over the whole grid.
struct FrontierDegree {
  const int32_t* __restrict__ outdeg;
  const int32_t* __restrict__ q;
  __host__ __device__ long long operator()(const int64_t& i) const { return (long long)outdeg[q[i]]; }
};

// Flattened-edge walk shared by the edge-balanced push kernels. Each CTA step
// takes kFlatCH consecutive edges of the frontier's flattened edge list; thread
// 0 finds the step's first owner once (binary search in `pre`), the CTA stages
// the next kFlatW owners' prefix values and ids in shared memory, and every
// edge finds its owner there (an owner beyond the window — only possible with
// many zero-degree frontier vertices — falls back to a global search).
constexpr int kFlatCH = 2048;
constexpr int kFlatW = kFlatCH + 1;
struct FlatSmem {
  long long pre[kFlatW + 1];
  int32_t u[kFlatW];
  long long o0;
};

template <typename OffT, typename Visit>
__device__ __forceinline__ void flat_edges(const int32_t* __restrict__ q, int64_t nf, const long long* __restrict__ pre,
                                           long long E, const OffT* __restrict__ off,
                                           const int32_t* __restrict__ idx, FlatSmem& sm, Visit&& visit) {
  const int tid = threadIdx.x;
  auto global_owner = [&](long long f) {  // last i with pre[i] <= f
    int64_t lo = 0, hi = nf - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (__ldg(&pre[mid]) <= f) lo = mid;
      else hi = mid - 1;
    }
    return lo;
  };
  for (long long lo = (long long)blockIdx.x * kFlatCH; lo < E; lo += (long long)gridDim.x * kFlatCH) {
    const long long hi = min(lo + (long long)kFlatCH, E);
    if (tid == 0) sm.o0 = global_owner(lo);
    __syncthreads();
    const int64_t o0 = sm.o0;
    for (int i = tid; i <= kFlatW; i += blockDim.x) {
      const int64_t o = o0 + i;
      sm.pre[i] = o < nf ? __ldg(&pre[o]) : LLONG_MAX;
      if (i < kFlatW) sm.u[i] = o < nf ? __ldg(&q[o]) : -1;
    }
    __syncthreads();
    for (long long base = lo; base < hi; base += blockDim.x) {
      const long long f = base + tid;
      const bool valid = f < hi;
      int32_t u = -1, v = -1;
      if (valid) {
        long long pf;
        if (sm.pre[kFlatW] <= f) {  // owner outside the staged window
          const int64_t o = global_owner(f);
          u = __ldg(&q[o]);
          pf = __ldg(&pre[o]);
        } else {
          int a = 0, b = kFlatW - 1;
          while (a < b) {
            const int mid = (a + b + 1) >> 1;
            if (sm.pre[mid] <= f) a = mid;
            else b = mid - 1;
          }
          u = sm.u[a];
          pf = sm.pre[a];
        }
        v = __ldg(&idx[(long long)off[u] + (f - pf)]);
      }
      visit(valid, u, v);
    }
    __syncthreads();
  }
}

// Edge-balanced push level with CAS claims (mid-size levels).
template <typename OffT>
__global__ void __launch_bounds__(256) k_bfs_push_bal(const int32_t* __restrict__ q, int64_t nf,
                                                      const long long* __restrict__ pre, long long E,
                                                      const OffT* __restrict__ off, const int32_t* __restrict__ idx,
                                                      const int32_t* __restrict__ outdeg, int32_t* parent,
                                                      int32_t* __restrict__ qnext, int64_t* __restrict__ cnext) {
  __shared__ FlatSmem sm;
  const int lane = threadIdx.x & 31;
  flat_edges<OffT>(q, nf, pre, E, off, idx, sm, [&](bool valid, int32_t u, int32_t v) {
    bool won = false;
    if (valid && *(volatile int32_t*)&parent[v] == -1) won = atomicCAS(&parent[v], -1, u) == -1;
    const unsigned mask = __ballot_sync(0xffffffffu, won);
    if (mask) {
      long long od = won ? (long long)__ldg(&outdeg[v]) : 0;
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) od += __shfl_xor_sync(0xffffffffu, od, s);
      long long pos = 0;
      if (lane == 0) {
        pos = atomicAdd((unsigned long long*)&cnext[0], (unsigned long long)__popc(mask));
        atomicAdd((unsigned long long*)&cnext[1], (unsigned long long)od);
      }
      pos = __shfl_sync(0xffffffffu, pos, 0);
      if (won) qnext[pos + __popc(mask & ((1u << lane) - 1))] = v;
    }
  });
}

// Large push levels, two phases, no atomics on the vertex data (the dedup of
// applyModified, done by a stamp instead of a CAS: thousands of
// frontier edges that reach the same hub would otherwise serialise on one
// L2 atomic unit).
//  phase 1 (k_bfs_push_stamp, edge-balanced): for frontier edge (u, v) with
//    parent[v] == -1, stamp cand[v] = (epoch << 32 | u) with a plain store
//    unless already stamped this epoch — racing writers all write a valid
//    parent (same level), the last one wins;
//  phase 2 (k_bfs_collect, vertex order): every v stamped this epoch and still
//    unvisited takes parent[v] = u and is appended to the next queue.
template <typename OffT>
__global__ void __launch_bounds__(256) k_bfs_push_stamp(const int32_t* __restrict__ q, int64_t nf,
                                                        const long long* __restrict__ pre, long long E,
                                                        const OffT* __restrict__ off, const int32_t* __restrict__ idx,
                                                        const int32_t* __restrict__ parent,
                                                        unsigned long long* cand, unsigned epoch) {
  __shared__ FlatSmem sm;
  flat_edges<OffT>(q, nf, pre, E, off, idx, sm, [&](bool valid, int32_t u, int32_t v) {
    if (valid && parent[v] == -1 && (unsigned)(cand[v] >> 32) != epoch)
      cand[v] = ((unsigned long long)epoch << 32) | (uint32_t)u;
  });
}

// Phase 2 of the stamped push: vertex order, CTA chunks of 2048 vertices.
// Winners are appended with ONE atomic per chunk (block scan of per-thread
// counts; per-warp atomics on a single counter serialised at L2), and the next
// frontier's bitmap words are written directly from the warp ballots, so a
// following pull level needs no queue -> bitmap conversion.
__global__ void __launch_bounds__(256) k_bfs_collect(const unsigned long long* __restrict__ cand, unsigned epoch,
                                                     int32_t* __restrict__ parent, const int32_t* __restrict__ outdeg,
                                                     int64_t n, int32_t* __restrict__ qnext,
                                                     uint32_t* __restrict__ bnext, int64_t* __restrict__ cnext) {
  constexpr int NT = 256, K = 8, CH = NT * K;
  using Scan = cub::BlockScan<int, NT>;
  using Red = cub::BlockReduce<long long, NT>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ typename Red::TempStorage red_tmp;
  __shared__ long long s_base;
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t nchunks = (n + CH - 1) / CH;
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    unsigned won = 0;  // bit k: vertex ch*CH + k*NT + tid claimed
    int32_t par[K];
    long long od = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int64_t v = ch * CH + (int64_t)k * NT + tid;
      bool w = false;
      par[k] = -1;
      if (v < n) {
        const unsigned long long c = cand[v];
        if ((unsigned)(c >> 32) == epoch && parent[v] == -1) {
          w = true;
          par[k] = (int32_t)(uint32_t)c;
          parent[v] = par[k];
          od += __ldg(&outdeg[v]);
        }
      }
      const unsigned mask = __ballot_sync(0xffffffffu, w);
      if (lane == 0 && ((ch * CH + (int64_t)k * NT + tid) >> 5) < ((n + 31) >> 5))
        bnext[(ch * CH + (int64_t)k * NT + tid) >> 5] = mask;
      won |= (unsigned)w << k;
    }
    int cnt = __popc(won), pre = 0, total = 0;
    Scan(scan_tmp).ExclusiveSum(cnt, pre, total);
    const long long dsum = Red(red_tmp).Sum(od);
    if (tid == 0) {
      s_base = total ? (long long)atomicAdd((unsigned long long*)&cnext[0], (unsigned long long)total) : 0;
      if (dsum) atomicAdd((unsigned long long*)&cnext[1], (unsigned long long)dsum);
    }
    __syncthreads();
    long long pos = s_base + pre;
#pragma unroll
    for (int k = 0; k < K; ++k)
      if ((won >> k) & 1u) qnext[pos++] = (int32_t)(ch * CH + (int64_t)k * NT + tid);
    __syncthreads();
  }
}

__global__ void k_q2b(const int32_t* __restrict__ q, int64_t qlen, uint32_t* __restrict__ bm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < qlen; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = q[i];
    atomicOr(&bm[u >> 5], 1u << (u & 31));
  }
}

__global__ void k_b2q(const uint32_t* __restrict__ bm, int64_t words, int32_t* __restrict__ q,
                      unsigned long long* __restrict__ tail) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;  // multiple of 32: warps stay aligned
  for (int64_t wb = blockIdx.x * (int64_t)blockDim.x + threadIdx.x - lane; wb < words; wb += stride) {
    const int64_t w = wb + lane;
    uint32_t bits = w < words ? bm[w] : 0u;
    int c = __popc(bits), inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const int total = __shfl_sync(0xffffffffu, inc, 31);
    unsigned long long base = 0;
    if (lane == 0 && total) base = atomicAdd(tail, (unsigned long long)total);
    base = __shfl_sync(0xffffffffu, base, 0);
    long long pos = (long long)base + inc - c;
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      q[pos++] = (int32_t)((w << 5) + b);
    }
  }
}

__global__ void __launch_bounds__(256) k_bfs_finish(const int32_t* __restrict__ parent, int64_t n,
                                                    const int32_t* __restrict__ perm, const int32_t* __restrict__ outdeg,
                                                    int32_t* __restrict__ out, unsigned long long* __restrict__ red) {
  using Red = cub::BlockReduce<long long, 256>;
  __shared__ typename Red::TempStorage t0, t1;
  long long reached = 0, edges = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = parent[v];
    const int32_t vin = perm ? perm[v] : (int32_t)v;
    out[vin] = p < 0 ? -1 : (perm ? perm[p] : p);
    if (p >= 0) {
      reached += 1;
      edges += outdeg[v];
    }
  }
  // one atomic pair per CTA (per-warp atomics on two addresses serialise at L2)
  reached = Red(t0).Sum(reached);
  edges = Red(t1).Sum(edges);
  if (threadIdx.x == 0 && reached) {
    atomicAdd(&red[0], (unsigned long long)reached);
    atomicAdd(&red[1], (unsigned long long)edges);
  }
}

}  // namespace

template <typename OffT>
static gi_status bfs_impl(gi_graph g, int32_t source, const gi_bfs_opts& o, int32_t* d_out, gi_bfs_stats* stats) {
  gi_context ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  const int64_t n = g->n, m = g->m;
  const int64_t words = (n + 31) >> 5;
  const int div = o.threshold_div > 0 ? o.threshold_div : 20;
  if (!g->parent.p) {
    GI_TRY(g->parent.alloc(n * sizeof(int32_t)));
    for (int k = 0; k < 2; ++k) {
      GI_TRY(g->queue[k].alloc(n * sizeof(int32_t)));
      GI_TRY(g->bitmap[k].alloc(words * sizeof(uint32_t)));
    }
    GI_TRY(g->counters.alloc((2 * kRing + 8) * sizeof(int64_t)));
    GI_TRY(g->bfs_pre.alloc((n + 1) * sizeof(long long)));
    size_t tb = 0;
    cub::TransformInputIterator<long long, FrontierDegree, cub::CountingInputIterator<int64_t>> it(
        cub::CountingInputIterator<int64_t>(0), FrontierDegree{g->outdeg.as<int32_t>(), g->queue[0].as<int32_t>()});
    GI_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, it, g->bfs_pre.as<long long>(), n, st));
    GI_TRY(g->bfs_scan_tmp.alloc(tb));
  }
  int64_t* cnt = g->counters.as<int64_t>();
  unsigned long long* aux = reinterpret_cast<unsigned long long*>(cnt + 2 * kRing);  // [0]=tail [1..2]=finish
  int64_t* h = ctx->h_scratch;
  int32_t* parent = g->parent.as<int32_t>();
  const OffT* csr_off = g->csr_off.as<OffT>();
  const OffT* csc_off = g->csc_off.as<OffT>();
  const int32_t* outdeg = g->outdeg.as<int32_t>();
  gi_bfs_stats S{};

  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (o.profile) {
    GI_CUDA(cudaEventCreate(&e0));
    GI_CUDA(cudaEventCreate(&e1));
    GI_CUDA(cudaEventRecord(e0, st));
  }
  GI_CUDA(cudaMemsetAsync(parent, 0xFF, n * sizeof(int32_t), st));
  GI_CUDA(cudaMemsetAsync(cnt, 0, (2 * kRing + 8) * sizeof(int64_t), st));
  k_bfs_init<<<1, 1, 0, st>>>(source, g->relabeled ? g->inv.as<int32_t>() : nullptr, outdeg, parent,
                              g->queue[0].as<int32_t>(), cnt);
  S.launches = 1;
  int qc = 0, bc = 0;     // current queue / bitmap buffers
  bool in_bitmap = false;  // representation of the current frontier
  bool bitmap_ready = false;  // bitmap[bc] also holds the current frontier (written by k_bfs_collect)
  int64_t* state = cnt + 2 * kRing + 4;  // [level, current queue] for k_bfs_persist
  static int persist_grid[2] = {0, 0};
  const int pk = sizeof(OffT) == 8;
  if (!persist_grid[pk]) {
    int bpm = 0;
    GI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpm, k_bfs_persist<OffT>, 256, 0));
    persist_grid[pk] = bpm > 0 ? std::min(sms, 64) : -1;  // few CTAs: cheap grid barrier
  }
  static const char* dbg = getenv("GI_DEBUG_BFS");  // diagnostics: per-level host timeline
  FILE* dbgf = dbg ? fopen(dbg, "a") : nullptr;
  auto now_us = [] {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  const double t_begin = now_us();
  for (int64_t level = 0;;) {
    int64_t* cur = cnt + 2 * (level % kRing);
    int64_t* nxt = cnt + 2 * ((level + 1) % kRing);
    GI_CUDA(cudaMemcpyAsync(h, cur, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    GI_CUDA(stream_wait(st));
    const int64_t nf = h[0], sdeg = h[1];
    if (dbgf) fprintf(dbgf, "src=%d level=%lld nf=%lld sdeg=%lld t=%.1f\n", source, (long long)level, (long long)nf,
                      (long long)sdeg, now_us() - t_begin);
    if (nf == 0) break;
    bool pull;
    if (o.policy == GI_BFS_PUSH_ONLY) pull = false;
    else if (o.policy == GI_BFS_PULL_ONLY) pull = level > 0;
    else pull = (nf + sdeg) > m / div;
    GI_CUDA(cudaMemsetAsync(nxt, 0, 2 * sizeof(int64_t), st));
    if (!pull && !in_bitmap && sdeg <= kPersistMax && persist_grid[pk] > 0) {
      // run as many small push levels as possible on the device
      h[2] = level;
      h[3] = qc;
      GI_CUDA(cudaMemcpyAsync(state, h + 2, 2 * sizeof(int64_t), cudaMemcpyHostToDevice, st));
      const int32_t* cidx = g->csr_idx.as<int32_t>();
      int32_t* q0p = g->queue[0].as<int32_t>();
      int32_t* q1p = g->queue[1].as<int32_t>();
      int64_t mdiv = m / div, smax = kPersistMax;
      int pol = o.policy;
      void* args[] = {(void*)&csr_off, (void*)&cidx, (void*)&outdeg, (void*)&parent, (void*)&q0p, (void*)&q1p,
                      (void*)&cnt, (void*)&state, (void*)&mdiv, (void*)&smax, (void*)&pol};
      GI_CUDA(cudaLaunchCooperativeKernel((void*)k_bfs_persist<OffT>, dim3(persist_grid[pk]), dim3(256), args, 0, st));
      GI_CUDA(cudaMemcpyAsync(h + 2, state, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      GI_CUDA(stream_wait(st));
      S.levels += (int32_t)(h[2] - level);
      S.launches++;
      level = h[2];
      qc = (int)h[3];
      bitmap_ready = false;
      continue;
    }
    bool next_bitmap_ready = false;
    if (pull) {
      if (!in_bitmap && !bitmap_ready) {
        GI_CUDA(cudaMemsetAsync(g->bitmap[bc].p, 0, words * sizeof(uint32_t), st));
        k_q2b<<<grid_for(nf, 256, sms), 256, 0, st>>>(g->queue[qc].as<int32_t>(), nf, g->bitmap[bc].as<uint32_t>());
        S.launches++;
      }
      {
        static int smem_words = -1;  // frontier-bitmap words staged per CTA
        if (smem_words < 0) {
          int optin = 0;
          GI_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
          int per_sm = 0;
          GI_CUDA(cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, ctx->device));
          smem_words = std::min(optin - 2048, per_sm / 2 - 2048) / 4;  // two CTAs per SM
          GI_CUDA(cudaFuncSetAttribute(k_bfs_pull_smem<int32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       smem_words * 4));
          GI_CUDA(cudaFuncSetAttribute(k_bfs_pull_smem<int64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       smem_words * 4));
        }
        const int sw = (int)std::min<int64_t>(words, smem_words);
        k_bfs_pull_smem<OffT><<<2 * sms, 1024, (size_t)sw * 4, st>>>(g->bitmap[bc].as<uint32_t>(),
                                                                 g->bitmap[bc ^ 1].as<uint32_t>(), parent, csc_off,
                                                                 g->csc_idx.as<int32_t>(), outdeg, n, sw, nxt, 0,
                                                                 PeerBits{});
      }
      bc ^= 1;
      in_bitmap = true;
      S.pull_levels++;
    } else {
      if (in_bitmap) {
        GI_CUDA(cudaMemsetAsync(aux, 0, sizeof(unsigned long long), st));
        k_b2q<<<grid_for(words, 256, sms), 256, 0, st>>>(g->bitmap[bc].as<uint32_t>(), words,
                                                         g->queue[qc].as<int32_t>(), aux);
        S.launches++;
      }
      if (sdeg >= kBalancedMin) {  // edge-balanced: a hub's edges spread over the grid
        cub::TransformInputIterator<long long, FrontierDegree, cub::CountingInputIterator<int64_t>> it(
            cub::CountingInputIterator<int64_t>(0), FrontierDegree{outdeg, g->queue[qc].as<int32_t>()});
        size_t tb = g->bfs_scan_tmp.bytes;
        GI_CUDA(cub::DeviceScan::ExclusiveSum(g->bfs_scan_tmp.p, tb, it, g->bfs_pre.as<long long>(), nf, st));
        const int grid = (int)std::min<int64_t>(ceil_div(sdeg, kFlatCH), (int64_t)sms * 8);
        static const int64_t stamp_min = getenv("GI_BFS_STAMP_MIN") ? atoll(getenv("GI_BFS_STAMP_MIN")) : kStampMin;
        if (sdeg >= stamp_min) {  // two-phase stamp + collect (no atomics on hub destinations)
          if (!g->bfs_cand.p || ++g->bfs_epoch == 0) {
            if (!g->bfs_cand.p) GI_TRY(g->bfs_cand.alloc(n * sizeof(unsigned long long)));
            GI_CUDA(cudaMemsetAsync(g->bfs_cand.p, 0, n * sizeof(unsigned long long), st));
            g->bfs_epoch = 1;
          }
          k_bfs_push_stamp<OffT><<<grid, 256, 0, st>>>(g->queue[qc].as<int32_t>(), nf,
                                                            g->bfs_pre.as<long long>(), sdeg, csr_off,
                                                            g->csr_idx.as<int32_t>(), parent,
                                                            g->bfs_cand.as<unsigned long long>(), g->bfs_epoch);
          k_bfs_collect<<<grid_for(ceil_div(n, 2048), 1, sms, 8), 256, 0, st>>>(
              g->bfs_cand.as<unsigned long long>(), g->bfs_epoch, parent, outdeg, n, g->queue[qc ^ 1].as<int32_t>(),
              g->bitmap[bc].as<uint32_t>(), nxt);
          next_bitmap_ready = true;  // bitmap[bc] now holds the next frontier too
          S.launches += 2;
        } else {
          k_bfs_push_bal<OffT><<<grid, 256, 0, st>>>(g->queue[qc].as<int32_t>(), nf, g->bfs_pre.as<long long>(),
                                                          sdeg, csr_off, g->csr_idx.as<int32_t>(), outdeg, parent,
                                                          g->queue[qc ^ 1].as<int32_t>(), nxt);
          S.launches++;
        }
      } else {
        const int small = nf <= kSmallF && sdeg < INT32_MAX;
        const int grid = small ? (int)std::min<int64_t>(std::max<int64_t>(ceil_div(sdeg, 1024), 1), (int64_t)sms * 4)
                                       : (int)std::min<int64_t>(ceil_div(nf, 256), (int64_t)sms * 8);
        k_bfs_push<OffT><<<grid, 256, 0, st>>>(g->queue[qc].as<int32_t>(), nf, csr_off, g->csr_idx.as<int32_t>(),
                                               outdeg, parent, g->queue[qc ^ 1].as<int32_t>(), nxt, small);
      }
      qc ^= 1;
      in_bitmap = false;
    }
    GI_CUDA(cudaGetLastError());
    S.launches++;
    S.levels++;
    ++level;
    bitmap_ready = next_bitmap_ready;
  }
  if (dbgf) fclose(dbgf);
  GI_CUDA(cudaMemsetAsync(aux + 1, 0, 2 * sizeof(unsigned long long), st));
  k_bfs_finish<<<grid_for(n, 256, sms), 256, 0, st>>>(parent, n, g->relabeled ? g->perm.as<int32_t>() : nullptr,
                                                      outdeg, d_out, aux + 1);
  S.launches++;
  GI_CUDA(cudaGetLastError());
  GI_CUDA(cudaMemcpyAsync(h, aux + 1, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  if (o.profile) GI_CUDA(cudaEventRecord(e1, st));
  GI_CUDA(cudaStreamSynchronize(st));
  S.reached = h[0];
  S.edges_traversed = h[1];
  if (o.profile) {
    GI_CUDA(cudaEventElapsedTime(&S.total_ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  if (stats) *stats = S;
  return GI_OK;
}

// ---------------------------------------------------------------------------------------------
// Multi-GPU BFS: each rank owns the destinations [r0, r0 + nr)
// and their parents; the frontier is a replicated bitmap. Per level:
//   pull: owned unvisited rows scan their in-edges against the replicated
//         bitmap (k_bfs_pull_smem with a row offset);
//   push: every rank turns the replicated bitmap into the same queue and
//         expands only the edges into its range (local CSR by source),
//         claiming with CAS and setting bits of its own bitmap words;
//   exchange: allgatherv of the owned bitmap words + allreduce of
//         (|F|, sum outdeg F); the direction decision is identical everywhere.
// The owned parent slices are allgathered once at the end.
namespace {

template <typename OffT>
struct LocalFrontierDegree {
  const OffT* __restrict__ off;
  const int32_t* __restrict__ q;
  int64_t nf;
  __host__ __device__ long long operator()(const int64_t& i) const {
    return i < nf ? (long long)(off[q[i] + 1] - off[q[i]]) : 0;
  }
};

template <typename OffT>
__global__ void __launch_bounds__(256) k_dist_push(const int32_t* __restrict__ q, int64_t nf,
                                                   const long long* __restrict__ pre, long long E,
                                                   const OffT* __restrict__ off, const int32_t* __restrict__ idx,
                                                   const int32_t* __restrict__ outdeg, int32_t* parent, int64_t r0,
                                                   uint32_t* __restrict__ fnext, int64_t* __restrict__ cnext,
                                                   PeerBits peers) {
  __shared__ FlatSmem sm;
  long long cnt = 0, sdeg = 0;
  flat_edges<OffT>(q, nf, pre, E, off, idx, sm, [&](bool valid, int32_t u, int32_t v) {
    if (valid) {
      int32_t* p = &parent[v - r0];
      if (*(volatile int32_t*)p == -1 && atomicCAS(p, -1, u) == -1) {
        atomicOr(&fnext[v >> 5], 1u << (v & 31));
        for (int k = 0; k < peers.np; ++k) atomicOr_system(&peers.p[k][v >> 5], 1u << (v & 31));
        cnt += 1;
        sdeg += __ldg(&outdeg[v]);
      }
    }
  });
  if (peers.np) __threadfence_system();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    sdeg += __shfl_xor_sync(0xffffffffu, sdeg, o);
  }
  if ((threadIdx.x & 31) == 0 && cnt) {
    atomicAdd((unsigned long long*)&cnext[0], (unsigned long long)cnt);
    atomicAdd((unsigned long long*)&cnext[1], (unsigned long long)sdeg);
  }
}

__global__ void k_dist_init(int32_t s_in, const int32_t* __restrict__ inv, const int32_t* __restrict__ outdeg,
                            int64_t r0, int64_t nr, int32_t* __restrict__ parent, uint32_t* __restrict__ bm,
                            int64_t* __restrict__ h2) {
  const int32_t s = inv ? inv[s_in] : s_in;
  bm[s >> 5] = 1u << (s & 31);
  if (s >= r0 && s < r0 + nr) parent[s - r0] = s;
  h2[0] = 1;
  h2[1] = outdeg[s];
}

}  // namespace

static bool all_peer_ok(gi_graph g, int P, bool ask) { return ask && P > 1 && g->bfs_peer_state == 1; }

template <typename OffT>
static gi_status bfs_dist_impl(gi_graph g, int32_t source, const gi_bfs_opts& o, int32_t* d_out, gi_bfs_stats* stats) {
  gi_context ctx = g->ctx;
  Comm* C = ctx->comm;
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  const int64_t n = g->n, nr = g->nr, r0 = g->r0, m = g->m;
  const int64_t words = (n + 31) >> 5;
  const int div = o.threshold_div > 0 ? o.threshold_div : 20;
  if (!g->parent.p) {
    GI_TRY(g->parent.alloc((n + 1) * sizeof(int32_t)));  // owned slice first, then the gathered full vector
    GI_TRY(g->queue[0].alloc((n + 1) * sizeof(int32_t)));
    for (int k = 0; k < 2; ++k) GI_TRY(g->bitmap[k].alloc((words + 1) * sizeof(uint32_t)));
    GI_TRY(g->counters.alloc(8 * sizeof(int64_t)));
    GI_TRY(g->bfs_pre.alloc((n + 2) * sizeof(long long)));
    size_t tb = 0;
    cub::TransformInputIterator<long long, LocalFrontierDegree<OffT>, cub::CountingInputIterator<int64_t>> it(
        cub::CountingInputIterator<int64_t>(0), LocalFrontierDegree<OffT>{g->csr_off.as<OffT>(), g->queue[0].as<int32_t>(), 0});
    GI_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, it, g->bfs_pre.as<long long>(), n + 1, st));
    GI_TRY(g->bfs_scan_tmp.alloc(tb));
  }
  DevBuf parent_full;
  GI_TRY(parent_full.alloc((n + 1) * sizeof(int32_t)));
  int32_t* parent = g->parent.as<int32_t>();
  int64_t* cnt = g->counters.as<int64_t>();
  unsigned long long* aux = reinterpret_cast<unsigned long long*>(cnt + 4);
  int64_t* h = ctx->h_scratch;
  const OffT* csr_off = g->csr_off.as<OffT>();
  const OffT* csc_off = g->csc_off.as<OffT>();
  const int32_t* outdeg = g->outdeg.as<int32_t>();
  const int P = C->nranks;
  std::vector<int64_t> wslice(P + 1), pslice(P + 1);
  for (int p = 0; p <= P; ++p) {
    wslice[p] = std::min<int64_t>((g->bounds[p] + 31) >> 5, words) * 4;
    pslice[p] = g->bounds[p] * 4;
  }
  gi_bfs_stats S{};
  cudaEvent_t pe[2] = {nullptr, nullptr};
  if (o.profile) {
    for (int k = 0; k < 2; ++k) GI_CUDA(cudaEventCreate(&pe[k]));
    GI_CUDA(cudaEventRecord(pe[0], st));
  }
  // peer stores of the next-frontier words (GI_BFS_PEER=1, or the comm's default;
  // every rank must ask and every rank must map, agreed by allreduce): a ring of
  // three bitmaps, so the one a level writes into on every replica was zeroed
  // by its owner a level earlier, before that level's allreduce (which no rank
  // passes before every rank has reached it)
  const char* peer_env = getenv("GI_BFS_PEER");
  const bool ask = P <= 8 && (peer_env ? strcmp(peer_env, "0") != 0 : C->peer_stores_default());
  {
    int64_t mine = ask ? 1 : 0;
    GI_CUDA(cudaMemcpyAsync(cnt + 2, &mine, sizeof mine, cudaMemcpyHostToDevice, st));
    GI_TRY(C->allreduce_i64(cnt + 2, 1, st));
    int64_t all = 0;
    GI_CUDA(cudaMemcpyAsync(&all, cnt + 2, sizeof all, cudaMemcpyDeviceToHost, st));
    GI_CUDA(cudaStreamSynchronize(st));
    if (all == P && g->bfs_peer_state == 0) {
      bool ok = true;
      for (int k = 0; k < 3 && ok; ++k) ok = g->bfs_ring[k].alloc((words + 1) * sizeof(uint32_t), /*plain=*/true) == GI_OK;
      int32_t bad = ok ? 0 : 1;  // every rank reaches the maps' collectives
      GI_CUDA(cudaMemcpyAsync(cnt + 2, &bad, sizeof bad, cudaMemcpyHostToDevice, st));
      GI_TRY(C->allreduce_i32(reinterpret_cast<int32_t*>(cnt + 2), 1, st));
      GI_CUDA(cudaMemcpyAsync(&bad, cnt + 2, sizeof bad, cudaMemcpyDeviceToHost, st));
      GI_CUDA(cudaStreamSynchronize(st));
      bool mapped = bad == 0;
      for (int k = 0; k < 3 && mapped; ++k)
        mapped = C->peer_map(g->bfs_ring[k].p, g->bfs_peer_bm[k], g->bfs_peer_opened, st) == GI_OK;
      g->bfs_peer_state = mapped ? 1 : -1;
      if (!mapped) {
        peer_unmap(g->bfs_peer_opened);
        set_error("");  // the allgather serves the call
      }
    }
  }
  const bool peer = all_peer_ok(g, P, ask);
  GI_CUDA(cudaMemsetAsync(parent, 0xFF, (nr + 1) * sizeof(int32_t), st));
  uint32_t* ring[3] = {g->bitmap[0].as<uint32_t>(), g->bitmap[1].as<uint32_t>(), nullptr};
  if (peer) {
    for (int k = 0; k < 3; ++k) {
      ring[k] = g->bfs_ring[k].as<uint32_t>();
      GI_CUDA(cudaMemsetAsync(ring[k], 0, words * sizeof(uint32_t), st));
    }
    GI_TRY(C->barrier(st));  // every replica zeroed before any rank's level-0 stores
  } else {
    GI_CUDA(cudaMemsetAsync(ring[0], 0, words * sizeof(uint32_t), st));
  }
  k_dist_init<<<1, 1, 0, st>>>(source, g->relabeled ? g->inv.as<int32_t>() : nullptr, outdeg, r0, nr, parent,
                               ring[0], cnt);
  S.launches++;
  static int smem_words = -1;
  if (smem_words < 0) {
    int optin = 0, per_sm = 0;
    GI_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
    GI_CUDA(cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, ctx->device));
    smem_words = std::min(optin - 2048, per_sm / 2 - 2048) / 4;
    GI_CUDA(cudaFuncSetAttribute(k_bfs_pull_smem<OffT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_words * 4));
  }
  for (int64_t level = 0;; ++level) {
    GI_CUDA(cudaMemcpyAsync(h, cnt, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    GI_CUDA(stream_wait(st));
    const int64_t nf = h[0], sdeg = h[1];
    if (nf == 0) break;
    bool pull;
    if (o.policy == GI_BFS_PUSH_ONLY) pull = false;
    else if (o.policy == GI_BFS_PULL_ONLY) pull = level > 0;
    else pull = (nf + sdeg) > m / div;
    uint32_t* fcur = peer ? ring[level % 3] : ring[level & 1];
    uint32_t* fnext = peer ? ring[(level + 1) % 3] : ring[(level + 1) & 1];
    PeerBits pb{};
    if (peer) {
      for (int q = 0; q < P; ++q)
        if (q != C->rank) pb.p[pb.np++] = static_cast<uint32_t*>(g->bfs_peer_bm[(level + 1) % 3][q]);
      // the bitmap peers write into two levels from now (see above)
      GI_CUDA(cudaMemsetAsync(ring[(level + 2) % 3], 0, words * sizeof(uint32_t), st));
    } else {
      GI_CUDA(cudaMemsetAsync(fnext, 0, words * sizeof(uint32_t), st));
    }
    GI_CUDA(cudaMemsetAsync(cnt, 0, 2 * sizeof(int64_t), st));
    if (pull) {
      const int sw = (int)std::min<int64_t>(words, smem_words);
      if (nr > 0)
        k_bfs_pull_smem<OffT><<<2 * sms, 1024, (size_t)sw * 4, st>>>(fcur, fnext, parent, csc_off,
                                                                     g->csc_idx.as<int32_t>(), outdeg, nr, sw, cnt, r0,
                                                                     pb);
      S.pull_levels++;
    } else {
      GI_CUDA(cudaMemsetAsync(aux, 0, sizeof(unsigned long long), st));
      k_b2q<<<grid_for(words, 256, sms), 256, 0, st>>>(fcur, words, g->queue[0].as<int32_t>(), aux);
      cub::TransformInputIterator<long long, LocalFrontierDegree<OffT>, cub::CountingInputIterator<int64_t>> it(
          cub::CountingInputIterator<int64_t>(0), LocalFrontierDegree<OffT>{csr_off, g->queue[0].as<int32_t>(), nf});
      size_t tb = g->bfs_scan_tmp.bytes;
      GI_CUDA(cub::DeviceScan::ExclusiveSum(g->bfs_scan_tmp.p, tb, it, g->bfs_pre.as<long long>(), nf + 1, st));
      GI_CUDA(cudaMemcpyAsync(h + 2, g->bfs_pre.as<long long>() + nf, sizeof(long long), cudaMemcpyDeviceToHost, st));
      GI_CUDA(stream_wait(st));
      const long long E = h[2];
      if (E > 0) {
        const int grid = (int)std::min<int64_t>(ceil_div(E, kFlatCH), (int64_t)sms * 8);
        k_dist_push<OffT><<<grid, 256, 0, st>>>(g->queue[0].as<int32_t>(), nf, g->bfs_pre.as<long long>(), E, csr_off,
                                                g->csr_idx.as<int32_t>(), outdeg, parent, r0, fnext, cnt, pb);
      }
      S.launches += 2;
    }
    GI_CUDA(cudaGetLastError());
    if (!peer) GI_TRY(C->allgatherv(fnext, wslice, st));
    GI_TRY(C->allreduce_i64(cnt, 2, st));
    S.launches++;
    S.levels++;
  }
  // gather the owned parent slices, then translate to input ids
  GI_CUDA(cudaMemcpyAsync(parent_full.as<int32_t>() + r0, parent, nr * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
  GI_TRY(C->allgatherv(parent_full.p, pslice, st));
  GI_CUDA(cudaMemsetAsync(aux + 1, 0, 2 * sizeof(unsigned long long), st));
  k_bfs_finish<<<grid_for(n, 256, sms), 256, 0, st>>>(parent_full.as<int32_t>(), n,
                                                      g->relabeled ? g->perm.as<int32_t>() : nullptr, outdeg, d_out,
                                                      aux + 1);
  S.launches++;
  GI_CUDA(cudaGetLastError());
  GI_CUDA(cudaMemcpyAsync(h, aux + 1, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GI_CUDA(stream_wait(st));
  S.reached = h[0];
  S.edges_traversed = h[1];
  if (o.profile) {
    GI_CUDA(cudaEventRecord(pe[1], st));
    GI_CUDA(cudaEventSynchronize(pe[1]));
    GI_CUDA(cudaEventElapsedTime(&S.total_ms, pe[0], pe[1]));
    for (int k = 0; k < 2; ++k) cudaEventDestroy(pe[k]);
  }
  if (stats) *stats = S;
  return GI_OK;
}

// parent (internal ids, full n) -> input ids; reached vertices and their out-edges
gi_status bfs_finish_output(gi_graph g, const int32_t* parent, int32_t* d_out, int64_t* reached, int64_t* edges) {
  gi_context ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  if (!g->counters.p) GI_TRY(g->counters.alloc((2 * kRing + 8) * sizeof(int64_t)));
  unsigned long long* red = reinterpret_cast<unsigned long long*>(g->counters.as<int64_t>() + 2 * kRing + 6);
  GI_CUDA(cudaMemsetAsync(red, 0, 2 * sizeof(unsigned long long), st));
  k_bfs_finish<<<grid_for(g->n, 256, ctx->num_sms), 256, 0, st>>>(parent, g->n,
                                                                 g->relabeled ? g->perm.as<int32_t>() : nullptr,
                                                                 g->outdeg.as<int32_t>(), d_out, red);
  GI_CUDA(cudaGetLastError());
  int64_t* h = ctx->h_scratch;
  GI_CUDA(cudaMemcpyAsync(h + 8, red, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GI_CUDA(stream_wait(st));
  *reached = h[8];
  *edges = h[9];
  return GI_OK;
}

gi_status bfs_run(gi_graph g, int32_t source, const gi_bfs_opts& o, int32_t* d_out, gi_bfs_stats* stats) {
  static const char* impl = getenv("GI_BFS_IMPL");  // "host": the host-driven level loop (A/B comparisons)
  if (g->ctx->nranks == 1 && !(impl && strcmp(impl, "host") == 0)) return bfs_fused(g, source, o, d_out, stats);
  if (g->ctx->nranks > 1) {
    if (g->off64) return bfs_dist_impl<int64_t>(g, source, o, d_out, stats);
    return bfs_dist_impl<int32_t>(g, source, o, d_out, stats);
  }
  if (g->off64) return bfs_impl<int64_t>(g, source, o, d_out, stats);
  return bfs_impl<int32_t>(g, source, o, d_out, stats);
}

}  // namespace gi
