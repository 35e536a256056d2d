// bfs_fused.cu — the whole direction-optimising BFS as ONE cooperative,
// persistent kernel (single GPU).
//
// Every level of the host-driven loop in bfs.cu costs a device->host read of
// two counters (|F|, sum outdeg F) before the direction (PAPER.md P:661-675,
// R7) can be chosen: ~15-20 µs of round trip per level, a third of a config-2
// BFS. Here every CTA reads the same counters after a grid barrier and takes
// the same decision, so the host launches once per source.
//
// Data written by other CTAs in earlier levels (parent, bitmaps, queues) is
// read with ld.global.cg (L2) so no stale L1 line survives a grid barrier.
//
// Per level l (frontier F_l held as bitmap bm[l%3] and, after push levels, as
// queue q[l&1]; counters ring cnt[l%4]):
//   pull (DensePull + bitvector + early exit): each
//     warp owns one 32-vertex word; unvisited vertices probe in-edges (4 per
//     step) against the frontier bitmap, whose hot prefix is staged in shared
//     memory; the next bitmap word is the ballot (no atomics);
//   push (SparsePush + CAS claim): if the frontier
//     is only a bitmap it is compacted to a queue first (CTA-aggregated); then
//     small frontiers (<= kFSmall vertices) are expanded by every CTA over an
//     equal slice of their flattened edge list (each CTA scans the frontier's
//     degrees itself), large ones by a grid-wide scan of degrees (two extra
//     barriers) and the same flattened walk; claims append to the next queue
//     with one atomic per CTA step (per warp for low-degree frontiers);
//   push levels leave only a queue: a pull level after them first rebuilds the
//   frontier bitmap; cnt[(l+2)%4] is cleared during level l (unused then).
#include <cooperative_groups.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cub/cub.cuh>

#include "gi_internal.cuh"

namespace cg = cooperative_groups;

namespace gi {
namespace {

constexpr int kFT = 1024;        // threads per CTA (one CTA per SM: 64 registers)
constexpr int kFW = kFT / 32;    // warps per CTA
constexpr int kFSmall = 8 * kFT; // frontier size expanded by the per-CTA scan
constexpr int kFChunk = kFT;     // frontier entries per scan chunk (large frontiers)
constexpr int kStreak = 16;      // consecutive small push levels before handing over to the small grid
constexpr int kSmallGrid = 16;   // CTAs of the small-grid launch
constexpr int64_t kBitmapPush = 1 << 16;  // push levels expanding more edges emit a bitmap frontier
constexpr uint32_t kNever = 0xFFFFFFFFu;   // stamp of vertices without in-edges: no BFS reaches them
#ifndef GI_BFS_VINFO
#define GI_BFS_VINFO 1  // claims read {input id, out-degree} with one 8-byte gather
#endif
#ifndef GI_BFS_KPW
#define GI_BFS_KPW 4    // 32-vertex words per warp and pull step
#endif
#ifndef GI_BFS_SMEM_DIV
#define GI_BFS_SMEM_DIV 4  // dynamic shared memory = 1/GI_BFS_SMEM_DIV of the SM's (the rest is L1)
#endif

template <typename OffT>
struct FusedArgs {
  const OffT* __restrict__ csr_off;
  const int32_t* __restrict__ csr_idx;
  const OffT* __restrict__ csc_off;
  const int32_t* __restrict__ csc_idx;
  const int32_t* __restrict__ outdeg;
  uint32_t* stamp;                 // visited: stamp[v] == epoch (never cleared between sources)
  uint32_t epoch;
  int32_t source_in;               // input id of the source
  const int32_t* __restrict__ inv; // input -> internal id (null: not relabelled)
  int fresh;                       // first launch of a source: reset the frontier state in the kernel prologue
  int nsrc;                        // sources run one after another in this launch (epoch + i, out + i*stride)
  const int32_t* __restrict__ sources;  // device, nsrc input ids (null: source_in)
  int64_t out_stride;
  int64_t* states;                 // nsrc x 16 final states (null: none)
  int32_t* out;                    // parents in input ids (written at claim time; -1 preset)
  const int32_t* __restrict__ perm;  // internal -> input id (null: not relabelled)
  const int2* __restrict__ vinfo;    // {input id, out-degree} per internal id
  int32_t* q[2];
  uint32_t* bm[3];
  int64_t* cnt;        // 4-level ring of {|F|, sum outdeg F}
  long long* tail;     // 4-level ring of queue tails (bitmap -> queue compaction)
  long long* pre;      // per-entry exclusive prefix of degrees within its chunk
  long long* ctot;     // chunk totals -> exclusive chunk offsets; ctot[nchunks] = E
  int64_t* state;      // [level, queue valid, bitmap valid, pull levels, done, reached, edges, examined,
                       //  pull-checked vertices] across launches
  int64_t n, mdiv;
  int64_t small_max;   // a push level with sum outdeg F <= small_max is "small"
  int mode;            // 0: full grid, hands over after kStreak small levels; 1: small grid, hands back
                       //    as soon as a level is not small (high-diameter graphs: cheaper barriers)
  int clustered;       // the launch is one thread-block cluster: barriers are cluster barriers (hardware)
  int policy, sw;
  unsigned long long* times;  // optional (GI_DEBUG_BFS_FUSED): per level [start, work done, barrier done]
  unsigned long long* ctimes; // optional: per level < 16 and CTA, the CTA's work-done time
  int max_times;
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct FSmem {  // carved from dynamic shared memory, phase by phase
  union {
    struct {
      int pre[kFSmall + 1];
      int32_t u[kFSmall];
    } small;
    struct {
      long long pre[kFChunk + 2];
      int32_t u[kFChunk + 1];
    } win;
  };
};

__device__ __forceinline__ long long vload(const long long* p) { return *(volatile const long long*)p; }
__device__ __forceinline__ int64_t vload(const int64_t* p) { return *(volatile const int64_t*)p; }

// CTA-aggregated append of the lanes with `want` set: one atomic per CTA step.
// Must be called by all threads of the CTA.
__device__ __forceinline__ void cta_append(bool want, int32_t v, int32_t* __restrict__ q,
                                           unsigned long long* __restrict__ tail, int* s_warp, long long* s_base) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned mask = __ballot_sync(0xffffffffu, want);
  if (lane == 0) s_warp[w] = __popc(mask);
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int i = 0; i < kFW; ++i) {
      const int c = s_warp[i];
      s_warp[i] = tot;
      tot += c;
    }
    *s_base = tot ? (long long)atomicAdd(tail, (unsigned long long)tot) : 0;
  }
  __syncthreads();
  if (want) q[*s_base + s_warp[w] + __popc(mask & ((1u << lane) - 1))] = v;
  __syncthreads();
}

template <typename OffT>
__global__ void __launch_bounds__(kFT, 1) k_bfs_fused(FusedArgs<OffT> A) {
  extern __shared__ __align__(16) unsigned char fsmem[];
  FSmem& sm = *reinterpret_cast<FSmem*>(fsmem);
  uint32_t* sbits = reinterpret_cast<uint32_t*>(fsmem);  // pull phase: staged bitmap prefix
  __shared__ int s_warp[kFW];
  __shared__ long long s_base;
  __shared__ long long s_red[3][kFW];
  __shared__ union {
    typename cub::BlockScan<int, kFT>::TempStorage i;
    typename cub::BlockScan<long long, kFT>::TempStorage l;
  } scan_tmp;
  cg::grid_group grid = cg::this_grid();
  // the barrier between phases: the grid's (cooperative launch) or, for the
  // small grid launched as one cluster, the cluster's hardware barrier
  auto gsync = [&]() {
    if (A.clustered) cg::this_cluster().sync();
    else grid.sync();
  };
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t G = gridDim.x;
  const int64_t words = (A.n + 31) >> 5;
  for (int si = 0; si < A.nsrc; ++si) {  // several sources per launch (gi_bfs_multi): no launch gap
  const uint32_t epoch = A.epoch + (uint32_t)si;
  int32_t* const out = A.out + si * A.out_stride;
  const int32_t source_in = A.sources ? A.sources[si] : A.source_in;
  // claim v for this source: the first thread to move its stamp to `epoch` wins
  auto claim = [&](int32_t v) {
    const uint32_t s = *(volatile uint32_t*)&A.stamp[v];
    return s != epoch && atomicCAS(&A.stamp[v], s, epoch) == s;
  };
  if (A.fresh) {  // new source: output -1 everywhere, empty level-0 bitmap, then the source itself
    // the stamps are read at random by every level: pull them into L2 (32 lines per thread pass)
    for (int64_t i = (blockIdx.x * (int64_t)kFT + tid) * 32; i < A.n; i += G * kFT * 32)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(A.stamp + i));
    for (int64_t i = blockIdx.x * (int64_t)kFT + tid; i < A.n; i += G * kFT) out[i] = -1;
    for (int64_t i = blockIdx.x * (int64_t)kFT + tid; i < words; i += G * kFT) A.bm[0][i] = 0u;
    gsync();
    if (blockIdx.x == 0 && tid == 0) {
      const int32_t s = A.inv ? A.inv[source_in] : source_in;
      A.stamp[s] = epoch;
      out[source_in] = source_in;
      A.q[0][0] = s;
      A.bm[0][s >> 5] = 1u << (s & 31);
      for (int i = 0; i < 8; ++i) A.cnt[i] = 0;
      for (int i = 0; i < 4; ++i) A.tail[i] = 0;
      A.cnt[0] = 1;
      A.cnt[1] = __ldg(&A.outdeg[s]);
      for (int i = 0; i < 11; ++i) A.state[i] = 0;
      A.state[1] = 1;  // frontier valid as a queue
      A.state[2] = 1;  // ... and as a bitmap
      A.state[9] = (int64_t)gtimer();
    }
    gsync();
  }
  int64_t level = A.state[0], pulls = A.state[3];
  bool qvalid = A.state[1] != 0;  // the current frontier is available as a queue ...
  bool bvalid = A.state[2] != 0;  // ... and as a bitmap (level 0: both)
  bool done = false;
  int streak = 0;
  // a claimed vertex: its parent goes to the output vector in input ids; returns its out-degree
  auto emit = [&](int64_t v, int32_t u) -> int {
#if GI_BFS_VINFO
    const int2 iv = __ldg(&A.vinfo[v]);  // {input id, out-degree}: one gather
    out[iv.x] = A.perm ? __ldg(&A.perm[u]) : u;
    return iv.y;
#else
    if (A.perm) out[__ldg(&A.perm[v])] = __ldg(&A.perm[u]);
    else out[v] = u;
    return __ldg(&A.outdeg[v]);
#endif
  };
  for (;;) {
    const int64_t* c = A.cnt + 2 * (level % 4);
    const int64_t nf = vload(c), sdeg = vload(c + 1);

    const bool timed = A.times && blockIdx.x == 0 && tid == 0 && level < A.max_times;
    if (timed) A.times[3 * level] = gtimer();
    if (nf == 0) {
      done = true;
      break;
    }
    const bool pull = A.policy == GI_BFS_PULL_ONLY ? level > 0
                                                   : (A.policy == GI_BFS_AUTO && nf + sdeg > A.mdiv);
    const bool small = !pull && sdeg <= A.small_max;
    if (A.mode == 1 && !small) break;                  // back to the full grid
    streak = small ? streak + 1 : 0;
    if (A.mode == 0 && A.small_max > 0 && streak > kStreak) break;  // hand over to the small grid
    if (blockIdx.x == 0 && tid == 0) {  // reached vertices and their out-edges (R16), summed over levels
      A.state[5] += nf;
      A.state[6] += sdeg;
      if (!pull) atomicAdd((unsigned long long*)&A.state[7], (unsigned long long)sdeg);  // push: every out-edge of F
      if (pull) atomicAdd((unsigned long long*)&A.state[8], (unsigned long long)A.n);   // pull: every vertex checked
    }
    uint32_t* bcur = A.bm[level % 3];
    uint32_t* bnext = A.bm[(level + 1) % 3];
    int32_t* qcur = A.q[level & 1];
    int32_t* qnext = A.q[(level + 1) & 1];
    int64_t* cn = A.cnt + 2 * ((level + 1) % 4);
    if (blockIdx.x == 0 && tid == 0) {
      A.cnt[2 * ((level + 2) % 4)] = 0;
      A.cnt[2 * ((level + 2) % 4) + 1] = 0;
      A.tail[(level + 2) % 4] = 0;
    }
    long long fcnt = 0, fdeg = 0;  // this thread's share of |F_{l+1}| and its out-degrees
    long long fexam = 0;           // in-edges this thread probed (pull levels)

    if (pull) {
      ++pulls;
      if (!bvalid) {  // frontier only as a queue (after push levels): build its bitmap
        for (int64_t i = blockIdx.x * (int64_t)kFT + tid; i < words; i += G * kFT) bcur[i] = 0u;
        gsync();
        for (int64_t i = blockIdx.x * (int64_t)kFT + tid; i < nf; i += G * kFT) {
          const int32_t u = __ldcg(&qcur[i]);
          atomicOr(&bcur[u >> 5], 1u << (u & 31));
        }
        gsync();
      }
      for (int i = tid; i < A.sw; i += kFT) sbits[i] = __ldcg(&bcur[i]);
      __syncthreads();
      const uint32_t lim = (uint32_t)A.sw * 32u;
      auto in_frontier = [&](uint32_t u) {
        const uint32_t word = u < lim ? sbits[u >> 5] : __ldcg(&bcur[u >> 5]);
        return ((word >> (u & 31)) & 1u) != 0u;
      };
      // each warp owns kPW words per step (lane l: vertex l of each), so every
      // lane has kPW independent parent / offset / first-edge chains in flight;
      // vertices not settled by their first 4 in-edges continue one by one
      constexpr int kPW = GI_BFS_KPW;
      for (int64_t wd0 = (blockIdx.x * (int64_t)kFW + w) * kPW; wd0 < words; wd0 += G * kFW * kPW) {
        int64_t v[kPW], e[kPW], e1[kPW];
        bool open[kPW], found[kPW];
#pragma unroll
        for (int j = 0; j < kPW; ++j) {
          v[j] = ((wd0 + j) << 5) + lane;
          if (wd0 + j < words && v[j] < A.n) {
            const uint32_t s = __ldcg(&A.stamp[v[j]]);
            open[j] = s != epoch && s != kNever;
          } else {
            open[j] = false;
          }
          found[j] = false;
          e[j] = e1[j] = 0;
        }
#pragma unroll
        for (int j = 0; j < kPW; ++j)
          if (open[j]) {
            e[j] = (int64_t)A.csc_off[v[j]];
            e1[j] = (int64_t)A.csc_off[v[j] + 1];
          }
        uint32_t u[kPW][4];
#pragma unroll
        for (int j = 0; j < kPW; ++j)
#pragma unroll
          for (int k = 0; k < 4; ++k) u[j][k] = e[j] + k < e1[j] ? (uint32_t)__ldg(&A.csc_idx[e[j] + k]) : 0xffffffffu;
#pragma unroll
        for (int j = 0; j < kPW; ++j) fexam += min((int64_t)4, e1[j] - e[j]);
#pragma unroll
        for (int j = 0; j < kPW; ++j) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (!found[j] && u[j][k] != 0xffffffffu && in_frontier(u[j][k])) {
              A.stamp[v[j]] = epoch;
              fdeg += emit(v[j], (int32_t)u[j][k]);
              found[j] = true;
            }
          for (int64_t ee = e[j] + 4; ee < e1[j] && !found[j]; ee += 4) {
            uint32_t x[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) x[k] = ee + k < e1[j] ? (uint32_t)__ldg(&A.csc_idx[ee + k]) : 0xffffffffu;
            fexam += min((int64_t)4, e1[j] - ee);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if (!found[j] && x[k] != 0xffffffffu && in_frontier(x[k])) {
                A.stamp[v[j]] = epoch;
                fdeg += emit(v[j], (int32_t)x[k]);
                found[j] = true;
              }
          }
        }
#pragma unroll
        for (int j = 0; j < kPW; ++j) {
          const unsigned mask = __ballot_sync(0xffffffffu, found[j]);
          if (lane == 0 && wd0 + j < words) bnext[wd0 + j] = mask;
          if (found[j]) fcnt += 1;
        }
      }
      qvalid = false;
      bvalid = true;
    } else {
      if (!qvalid) {  // bitmap -> queue, one atomic per CTA word block
        unsigned long long* t = reinterpret_cast<unsigned long long*>(A.tail + level % 4);
        const int64_t per = (words + G - 1) / G;
        const int64_t w0 = blockIdx.x * per, w1 = min(words, w0 + per);
        for (int64_t b = w0; b < w1; b += kFT) {
          const int64_t wd = b + tid;
          uint32_t bits = wd < w1 ? __ldcg(&bcur[wd]) : 0u;
          int pos, tot;
          cub::BlockScan<int, kFT>(scan_tmp.i).ExclusiveSum(__popc(bits), pos, tot);
          if (tid == 0) s_base = tot ? (long long)atomicAdd(t, (unsigned long long)tot) : 0;
          __syncthreads();
          long long p = s_base + pos;
          while (bits) {
            const int k = __ffs(bits) - 1;
            bits &= bits - 1;
            qcur[p++] = (int32_t)((wd << 5) + k);
          }
          __syncthreads();
        }
        gsync();
      }
      unsigned long long* tn = reinterpret_cast<unsigned long long*>(cn);
      // Big push levels (the hub levels of social graphs) emit the next
      // frontier as a bitmap (one atomicOr per claim, no queue appends and
      // their CTA barriers); the pull level that usually follows reads it
      // directly, and a push level converts it back to a queue.
      const bool to_bm = sdeg > kBitmapPush && sdeg > 4 * nf;
      if (to_bm) {
        for (int64_t i = blockIdx.x * (int64_t)kFT + tid; i < words; i += G * kFT) bnext[i] = 0u;
        gsync();
      }
      // visit one flattened edge (u -> v): claim v, then append it (or set its bit)
      auto claim_step = [&](bool valid, int32_t u, int32_t v) {
        bool won = false;
        if (valid) won = claim(v);
        if (won) {
          fdeg += emit(v, u);
        }
        if (to_bm) {
          if (won) {
            atomicOr(&bnext[v >> 5], 1u << (v & 31));
            fcnt += 1;
          }
        } else {
          cta_append(won, v, qnext, tn, s_warp, &s_base);
        }
      };
      if (sdeg <= 4 * nf) {
        // low-degree frontier (road/grid-like levels): thread per frontier vertex,
        // no scan; every thread steps through the same number of rounds so the
        // CTA-aggregated append stays collective
        const int64_t per = (nf + G - 1) / G;
        const int64_t i0 = blockIdx.x * per, i1 = min(nf, i0 + per);
        for (int64_t b = i0; b < i1; b += kFT) {
          const int64_t i = b + tid;
          int32_t u = -1;
          int64_t e = 0, e1 = 0;
          if (i < i1) {
            u = __ldcg(&qcur[i]);
            e = (int64_t)A.csr_off[u];
            e1 = (int64_t)A.csr_off[u + 1];
          }
          // 4 neighbours per step with independent loads / CAS (one dependent chain per
          // step instead of per edge), then one warp-aggregated append of all wins
          int rounds = (int)min((e1 - e + 3) / 4, (int64_t)INT_MAX);
          for (int o = 16; o > 0; o >>= 1) rounds = max(rounds, __shfl_xor_sync(0xffffffffu, rounds, o));
          for (int k = 0; k < rounds; ++k) {
            int32_t v[4];
            unsigned wmask = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = e + 4 * k + j < e1 ? __ldg(&A.csr_idx[e + 4 * k + j]) : -1;
            uint32_t pv[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) pv[j] = v[j] >= 0 ? *(volatile uint32_t*)&A.stamp[v[j]] : epoch;
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (pv[j] != epoch && atomicCAS(&A.stamp[v[j]], pv[j], epoch) == pv[j]) {
                wmask |= 1u << j;
                fdeg += emit(v[j], u);
              }
            const int mine = __popc(wmask);
            int incl = mine;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int t = __shfl_up_sync(0xffffffffu, incl, o);
              if (lane >= o) incl += t;
            }
            const int wtot = __shfl_sync(0xffffffffu, incl, 31);
            if (wtot) {
              long long pos = 0;
              if (lane == 0) pos = (long long)atomicAdd(tn, (unsigned long long)wtot);
              pos = __shfl_sync(0xffffffffu, pos, 0) + incl - mine;
#pragma unroll
              for (int j = 0; j < 4; ++j)
                if ((wmask >> j) & 1u) {
                  qnext[pos++] = v[j];
                }
            }
          }
        }
      } else if (nf <= kFSmall && sdeg < INT_MAX) {
        // every CTA scans the whole (small) frontier's degrees, then walks 1/G of the edges
        constexpr int PT = kFSmall / kFT;
        int d[PT], run = 0;
#pragma unroll
        for (int k = 0; k < PT; ++k) {
          const int i = tid * PT + k;
          d[k] = 0;
          if (i < nf) {
            const int32_t u = __ldcg(&qcur[i]);
            sm.small.u[i] = u;
            d[k] = (int)(A.csr_off[u + 1] - A.csr_off[u]);
          }
          run += d[k];
        }
        int excl, total;
        cub::BlockScan<int, kFT>(scan_tmp.i).ExclusiveSum(run, excl, total);
#pragma unroll
        for (int k = 0; k < PT; ++k) {
          const int i = tid * PT + k;
          if (i < nf) sm.small.pre[i] = excl;
          excl += d[k];
        }
        __syncthreads();
        const long long E = total;
        const long long lo = E * blockIdx.x / G, hi = E * (blockIdx.x + 1) / G;
        for (long long base = lo; base < hi; base += kFT) {
          const long long f = base + tid;
          int32_t u = -1, v = -1;
          if (f < hi) {
            int a = 0, b = (int)nf - 1;
            while (a < b) {
              const int mid = (a + b + 1) >> 1;
              if (sm.small.pre[mid] <= f) a = mid;
              else b = mid - 1;
            }
            u = sm.small.u[a];
            v = __ldg(&A.csr_idx[(long long)A.csr_off[u] + (f - sm.small.pre[a])]);
          }
          claim_step(f < hi, u, v);
        }
        if (!to_bm) fcnt = 0;  // counted through the tail below
      } else {
        // grid-wide scan of the frontier's degrees: chunk prefixes, then chunk offsets
        const int64_t nch = (nf + kFChunk - 1) / kFChunk;
        for (int64_t ch = blockIdx.x; ch < nch; ch += G) {
          const int64_t i = ch * kFChunk + tid;
          long long dg = 0;
          if (i < nf) {
            const int32_t u = __ldcg(&qcur[i]);
            dg = (long long)(A.csr_off[u + 1] - A.csr_off[u]);
          }
          long long ex, tot;
          cub::BlockScan<long long, kFT>(scan_tmp.l).ExclusiveSum(dg, ex, tot);
          if (i < nf) A.pre[i] = ex;
          if (tid == 0) A.ctot[ch] = tot;
          __syncthreads();
        }
        gsync();
        if (blockIdx.x == 0) {
          long long carry = 0;
          for (int64_t b = 0; b < nch; b += kFT) {
            const int64_t i = b + tid;
            const long long x = i < nch ? A.ctot[i] : 0;
            long long ex, tot;
            cub::BlockScan<long long, kFT>(scan_tmp.l).ExclusiveSum(x, ex, tot);
            if (i < nch) A.ctot[i] = carry + ex;
            carry += tot;
            __syncthreads();
          }
          if (tid == 0) A.ctot[nch] = carry;
        }
        gsync();
        const long long E = vload(A.ctot + nch);
        auto gpre = [&](int64_t i) { return vload(A.ctot + i / kFChunk) + vload(A.pre + i); };
        auto owner = [&](long long f) {  // last i with gpre(i) <= f
          int64_t a = 0, b = nf - 1;
          while (a < b) {
            const int64_t mid = (a + b + 1) >> 1;
            if (gpre(mid) <= f) a = mid;
            else b = mid - 1;
          }
          return a;
        };
        for (long long lo = (long long)blockIdx.x * kFChunk; lo < E; lo += G * kFChunk) {
          const long long hi = min(lo + (long long)kFChunk, E);
          if (tid == 0) s_base = owner(lo);
          __syncthreads();
          const int64_t o0 = s_base;
          for (int i = tid; i <= kFChunk + 1; i += kFT) {
            const int64_t o = o0 + i;
            sm.win.pre[i] = o < nf ? gpre(o) : LLONG_MAX;
            if (i <= kFChunk) sm.win.u[i] = o < nf ? __ldcg(&qcur[o]) : -1;
          }
          __syncthreads();
          const long long f = lo + tid;
          int32_t u = -1, v = -1;
          if (f < hi) {
            long long pf;
            if (sm.win.pre[kFChunk + 1] <= f) {
              const int64_t o = owner(f);
              u = __ldcg(&qcur[o]);
              pf = gpre(o);
            } else {
              int a = 0, b = kFChunk;
              while (a < b) {
                const int mid = (a + b + 1) >> 1;
                if (sm.win.pre[mid] <= f) a = mid;
                else b = mid - 1;
              }
              u = sm.win.u[a];
              pf = sm.win.pre[a];
            }
            v = __ldg(&A.csr_idx[(long long)A.csr_off[u] + (f - pf)]);
          }
          claim_step(f < hi, u, v);
        }
        if (!to_bm) fcnt = 0;
      }
      qvalid = !to_bm;  // push levels produce the queue or (big ones) the bitmap
      bvalid = to_bm;
    }
    // |F_{l+1}| and sum of its out-degrees: one atomic pair per CTA
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      fcnt += __shfl_xor_sync(0xffffffffu, fcnt, o);
      fdeg += __shfl_xor_sync(0xffffffffu, fdeg, o);
      fexam += __shfl_xor_sync(0xffffffffu, fexam, o);
    }
    if (lane == 0) {
      s_red[0][w] = fcnt;
      s_red[1][w] = fdeg;
      s_red[2][w] = fexam;
    }
    __syncthreads();
    if (tid == 0) {
      long long a = 0, b = 0, x = 0;
      for (int i = 0; i < kFW; ++i) {
        a += s_red[0][i];
        b += s_red[1][i];
        x += s_red[2][i];
      }
      if (a) atomicAdd((unsigned long long*)&cn[0], (unsigned long long)a);
      if (b) atomicAdd((unsigned long long*)&cn[1], (unsigned long long)b);
      if (x) atomicAdd((unsigned long long*)&A.state[7], (unsigned long long)x);
    }
    if (timed) A.times[3 * level + 1] = gtimer();
    if (A.ctimes && tid == 0 && level < 16) A.ctimes[level * G + blockIdx.x] = gtimer();
    gsync();
    if (timed) A.times[3 * level + 2] = gtimer();
    ++level;
  }
  if (blockIdx.x == 0 && tid == 0) {
    A.state[10] = (int64_t)gtimer();  // last exit
    A.state[0] = level;
    A.state[1] = qvalid;
    A.state[2] = bvalid;
    A.state[3] = pulls;
    A.state[4] = done;
    if (A.states)
      for (int i = 0; i < 11; ++i) A.states[16 * si + i] = A.state[i];
  }
  if (si + 1 < A.nsrc) gsync();  // the next prologue rewrites what this source's last level read
  }  // sources
}


}  // namespace

// stamps at setup (and after an epoch wrap): kNever for vertices no edge
// enters (the pull levels skip them after one coalesced load), else 0
template <typename OffT>
__global__ void k_stamp_init(const OffT* __restrict__ csc_off, int64_t n, uint32_t* __restrict__ stamp) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    stamp[v] = csc_off[v + 1] == csc_off[v] ? kNever : 0u;
}

__global__ void k_vinfo(const int32_t* __restrict__ perm, const int32_t* __restrict__ outdeg, int64_t n,
                        int2* __restrict__ vinfo) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    vinfo[v] = make_int2(perm ? perm[v] : (int32_t)v, outdeg[v]);
}

// one-time per graph: buffers, dynamic shared memory, co-resident grid size
template <typename OffT>
static gi_status fused_setup(gi_graph g) {
  gi_context ctx = g->ctx;
  const int64_t n = g->n, words = (n + 31) >> 5;
  auto& F = g->fused;
  if (F.ready) return GI_OK;
  GI_TRY(F.stamp.alloc((n + 1) * sizeof(uint32_t)));
  k_stamp_init<OffT><<<grid_for(n, 256, ctx->num_sms), 256, 0, ctx->stream>>>(g->csc_off.as<OffT>(), n,
                                                                              F.stamp.as<uint32_t>());
  GI_TRY(F.vinfo.alloc((n + 1) * sizeof(int2)));
  k_vinfo<<<grid_for(n, 256, ctx->num_sms), 256, 0, ctx->stream>>>(g->relabeled ? g->perm.as<int32_t>() : nullptr,
                                                                  g->outdeg.as<int32_t>(), n, F.vinfo.as<int2>());
  GI_CUDA(cudaGetLastError());
  F.epoch = 0;
  for (int k = 0; k < 2; ++k) GI_TRY(F.q[k].alloc((n + 1) * sizeof(int32_t)));
  for (int k = 0; k < 3; ++k) GI_TRY(F.bm[k].alloc((words + 1) * sizeof(uint32_t)));
  GI_TRY(F.cnt.alloc(32 * sizeof(int64_t)));
  GI_TRY(F.pre.alloc((n + 1) * sizeof(long long)));
  GI_TRY(F.ctot.alloc((n / kFChunk + 2) * sizeof(long long)));
  int optin = 0, per_sm = 0;
  GI_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  GI_CUDA(cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, ctx->device));
  cudaFuncAttributes fa{};
  GI_CUDA(cudaFuncGetAttributes(&fa, k_bfs_fused<OffT>));
  // shared memory vs L1: the rest of the 256 KB stays L1, which the random
  // gathers (offsets, vinfo, register spills) of every level lean on
  int dyn = std::min(optin, per_sm / GI_BFS_SMEM_DIV) - (int)fa.sharedSizeBytes - 2048;
  dyn = std::max(dyn, (int)sizeof(FSmem)) & ~15;
  GI_CUDA(cudaFuncSetAttribute(k_bfs_fused<OffT>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
  int bpm = 0;
  GI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpm, k_bfs_fused<OffT>, kFT, dyn));
  if (bpm < 1) return fail(GI_ERR_UNSUPPORTED, "fused BFS kernel cannot be co-resident");
  F.dyn = dyn;
  F.grid = bpm * ctx->num_sms;
  // the small grid as one cluster of kSmallGrid CTAs (non-portable size), if the device can hold one
  F.cluster = false;
  static const bool cl_env = !getenv("GI_BFS_CLUSTER") || atoi(getenv("GI_BFS_CLUSTER")) != 0;
  if (cl_env && cudaFuncSetAttribute(k_bfs_fused<OffT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
                    cudaSuccess) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(kSmallGrid);
    cfg.blockDim = dim3(kFT);
    cfg.dynamicSmemBytes = (size_t)dyn;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kSmallGrid;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, k_bfs_fused<OffT>, &cfg) == cudaSuccess && nc >= 1) F.cluster = true;
  }
  cudaGetLastError();
  F.ready = true;
  return GI_OK;
}

template <typename OffT>
static FusedArgs<OffT> fused_args(gi_graph g, const gi_bfs_opts& o, int32_t* d_out) {
  auto& F = g->fused;
  const int64_t words = (g->n + 31) >> 5;
  int64_t* cnt = F.cnt.as<int64_t>();
  FusedArgs<OffT> A;
  A.csr_off = g->csr_off.as<OffT>();
  A.csr_idx = g->csr_idx.as<int32_t>();
  A.csc_off = g->csc_off.as<OffT>();
  A.csc_idx = g->csc_idx.as<int32_t>();
  A.outdeg = g->outdeg.as<int32_t>();
  A.stamp = F.stamp.as<uint32_t>();
  A.inv = g->relabeled ? g->inv.as<int32_t>() : nullptr;
  A.vinfo = F.vinfo.as<int2>();
  A.fresh = 0;
  A.nsrc = 1;
  A.sources = nullptr;
  A.out_stride = 0;
  A.states = nullptr;
  A.out = d_out;
  A.perm = g->relabeled ? g->perm.as<int32_t>() : nullptr;
  A.q[0] = F.q[0].as<int32_t>();
  A.q[1] = F.q[1].as<int32_t>();
  for (int k = 0; k < 3; ++k) A.bm[k] = F.bm[k].as<uint32_t>();
  A.cnt = cnt;
  A.tail = reinterpret_cast<long long*>(cnt + 8);
  A.pre = F.pre.as<long long>();
  A.ctot = F.ctot.as<long long>();
  A.state = cnt + 8 + 4;  // state[7] after the tail ring
  A.small_max = 1 << 16;
  A.mode = 0;
  A.clustered = 0;
  A.n = g->n;
  A.mdiv = g->m / (o.threshold_div > 0 ? o.threshold_div : 20);
  A.policy = o.policy;
  A.sw = (int)std::min<int64_t>(words, (int64_t)((F.dyn) / 4));
  A.times = nullptr;
  A.ctimes = nullptr;
  A.max_times = 0;
  return A;
}

// start a source: a fresh epoch (the visited stamps of earlier sources become
// stale, no clearing), then one full-grid launch whose prologue resets the
// output, the level-0 bitmap and the counters
template <typename OffT>
static gi_status fused_start(gi_graph g, int32_t source, FusedArgs<OffT>& A) {
  gi_context ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  auto& F = g->fused;
  if (++F.epoch == kNever) {  // epochs exhausted (2^32 - 1 sources): reset the stamps once
    k_stamp_init<OffT><<<grid_for(g->n, 256, ctx->num_sms), 256, 0, st>>>(g->csc_off.as<OffT>(), g->n,
                                                                        F.stamp.as<uint32_t>());
    GI_CUDA(cudaGetLastError());
    F.epoch = 1;
  }
  A.epoch = F.epoch;
  A.source_in = source;
  A.fresh = 1;
  A.mode = 0;
  A.clustered = 0;
  void* args[] = {&A};
  GI_CUDA(cudaLaunchCooperativeKernel((void*)k_bfs_fused<OffT>, dim3(F.grid), dim3(kFT), args, (size_t)F.dyn, st));
  GI_CUDA(cudaGetLastError());
  A.fresh = 0;
  return GI_OK;
}

template <typename OffT>
static gi_status bfs_fused_t(gi_graph g, int32_t source, const gi_bfs_opts& o, int32_t* d_out, gi_bfs_stats* stats) {
  gi_context ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  GI_TRY(fused_setup<OffT>(g));
  auto& F = g->fused;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (o.profile) {
    GI_CUDA(cudaEventCreate(&e0));
    GI_CUDA(cudaEventCreate(&e1));
    GI_CUDA(cudaEventRecord(e0, st));
  }
  FusedArgs<OffT> A = fused_args<OffT>(g, o, d_out);
  static const char* dbg = getenv("GI_DEBUG_BFS_FUSED");  // diagnostics: per-level timeline file
  DevBuf tbuf, cbuf;
  if (dbg) {
    A.max_times = 1 << 16;
    GI_TRY(tbuf.alloc((size_t)3 * A.max_times * sizeof(unsigned long long)));
    GI_CUDA(cudaMemsetAsync(tbuf.p, 0, (size_t)3 * A.max_times * sizeof(unsigned long long), st));
    A.times = tbuf.as<unsigned long long>();
    GI_TRY(cbuf.alloc((size_t)16 * F.grid * sizeof(unsigned long long)));
    GI_CUDA(cudaMemsetAsync(cbuf.p, 0, (size_t)16 * F.grid * sizeof(unsigned long long), st));
    A.ctimes = cbuf.as<unsigned long long>();
  }
  GI_TRY(fused_start<OffT>(g, source, A));
  // full grid; high-diameter stretches continue on a small grid (cheaper grid barriers)
  int64_t* h = ctx->h_scratch;
  int launches = 2;
  for (int mode = 1;; mode ^= 1) {
    GI_CUDA(cudaMemcpyAsync(h + 16, A.state, 9 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    GI_CUDA(stream_wait(st));
    if (h[16 + 4]) break;
    A.mode = mode;
    A.clustered = mode == 1 && F.cluster;
    void* args[] = {&A};
    const int grid = mode == 0 ? F.grid : std::min(F.grid, kSmallGrid);
    if (A.clustered) {  // one cluster: hardware barriers between the phases of a level
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(kSmallGrid);
      cfg.blockDim = dim3(kFT);
      cfg.dynamicSmemBytes = (size_t)F.dyn;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = kSmallGrid;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      GI_CUDA(cudaLaunchKernelEx(&cfg, k_bfs_fused<OffT>, A));
    } else {
      GI_CUDA(cudaLaunchCooperativeKernel((void*)k_bfs_fused<OffT>, dim3(grid), dim3(kFT), args, (size_t)F.dyn, st));
    }
    GI_CUDA(cudaGetLastError());
    ++launches;
  }
  const int64_t lv[2] = {h[16], h[16 + 3]};
  const int64_t reached = h[16 + 5], edges = h[16 + 6];
  if (dbg) {
    std::vector<unsigned long long> ht((size_t)3 * A.max_times);
    GI_CUDA(cudaMemcpy(ht.data(), tbuf.p, ht.size() * 8, cudaMemcpyDeviceToHost));
    std::vector<unsigned long long> hc((size_t)16 * F.grid);
    GI_CUDA(cudaMemcpy(hc.data(), cbuf.p, hc.size() * 8, cudaMemcpyDeviceToHost));
    if (FILE* f = fopen(dbg, "a")) {
      for (int l = 0; l < A.max_times && ht[3 * l]; ++l) {
        fprintf(f, "src=%d level=%d work_us=%.2f barrier_us=%.2f", source, l,
                ht[3 * l + 1] ? (ht[3 * l + 1] - ht[3 * l]) / 1e3 : 0.0,
                ht[3 * l + 2] ? (ht[3 * l + 2] - ht[3 * l + 1]) / 1e3 : 0.0);
        if (l < 16 && ht[3 * l + 1]) {  // per-CTA work time: min / median / max
          std::vector<double> w;
          for (int c = 0; c < F.grid; ++c)
            if (hc[(size_t)l * F.grid + c]) w.push_back((hc[(size_t)l * F.grid + c] - ht[3 * l]) / 1e3);
          std::sort(w.begin(), w.end());
          if (!w.empty()) fprintf(f, " cta_work_us min=%.2f med=%.2f max=%.2f", w.front(), w[w.size() / 2], w.back());
        }
        fprintf(f, "\n");
      }
      fclose(f);
    }
  }
  float ms = 0.f;
  if (o.profile) {
    GI_CUDA(cudaEventRecord(e1, st));
    GI_CUDA(cudaEventSynchronize(e1));
    GI_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  if (stats) {
    stats->total_ms = ms;
    stats->levels = (int32_t)lv[0];
    stats->pull_levels = (int32_t)lv[1];
    stats->reached = reached;
    stats->edges_traversed = edges;
    stats->edges_examined = h[16 + 7];
    stats->pull_vertices = h[16 + 8];
    stats->launches = launches + 3;
  }
  return GI_OK;
}

// k sources back to back in ONE cooperative launch: the kernel loops over the
// sources (epochs F.epoch+1 .. F.epoch+k, output rows out + i*stride) with a
// grid barrier in between, and leaves every source's final state in `states`.
// A source that reaches a long run of small levels (a high-diameter graph)
// stops there and is rerun alone with the small-grid handover.
template <typename OffT>
static gi_status bfs_fused_multi_t(gi_graph g, int32_t k, const int32_t* sources, const gi_bfs_opts& o,
                                   int32_t* d_out, int64_t out_stride, gi_bfs_stats* stats) {
  gi_context ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  GI_TRY(fused_setup<OffT>(g));
  auto& F = g->fused;
  if (ctx->h_batch_len < (int64_t)k * 16) {
    if (ctx->h_batch) cudaFreeHost(ctx->h_batch);
    ctx->h_batch = nullptr;
    ctx->h_batch_len = 0;
    GI_CUDA(cudaMallocHost(&ctx->h_batch, (size_t)k * 16 * sizeof(int64_t)));
    ctx->h_batch_len = (int64_t)k * 16;
  }
  int64_t* hb = ctx->h_batch;
  if (F.msrc.bytes < (size_t)k * sizeof(int32_t)) GI_TRY(F.msrc.alloc((size_t)k * sizeof(int32_t)));
  if (F.mstates.bytes < (size_t)k * 16 * sizeof(int64_t)) GI_TRY(F.mstates.alloc((size_t)k * 16 * sizeof(int64_t)));
  GI_CUDA(cudaMemcpyAsync(F.msrc.p, sources, (size_t)k * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  if ((uint64_t)F.epoch + (uint64_t)k >= (uint64_t)kNever) {  // epochs would run out: reset the stamps
    k_stamp_init<OffT><<<grid_for(g->n, 256, ctx->num_sms), 256, 0, st>>>(g->csc_off.as<OffT>(), g->n,
                                                                        F.stamp.as<uint32_t>());
    GI_CUDA(cudaGetLastError());
    F.epoch = 0;
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (o.profile) {
    GI_CUDA(cudaEventCreate(&e0));
    GI_CUDA(cudaEventCreate(&e1));
    GI_CUDA(cudaEventRecord(e0, st));
  }
  FusedArgs<OffT> A = fused_args<OffT>(g, o, d_out);
  A.epoch = F.epoch + 1;
  F.epoch += (uint32_t)k;
  A.nsrc = k;
  A.sources = F.msrc.as<int32_t>();
  A.out_stride = out_stride;
  A.states = F.mstates.as<int64_t>();
  A.fresh = 1;
  A.mode = 0;
  A.clustered = 0;
  void* args[] = {&A};
  GI_CUDA(cudaLaunchCooperativeKernel((void*)k_bfs_fused<OffT>, dim3(F.grid), dim3(kFT), args, (size_t)F.dyn, st));
  GI_CUDA(cudaGetLastError());
  GI_CUDA(cudaMemcpyAsync(hb, F.mstates.p, (size_t)k * 16 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  float ms = 0.f;
  if (o.profile) GI_CUDA(cudaEventRecord(e1, st));
  GI_CUDA(stream_wait(st));
  if (o.profile) {
    GI_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  if (const char* dbg = getenv("GI_DEBUG_BFS_MULTI")) {  // diagnostics: per-source kernel span
    if (FILE* f = fopen(dbg, "a")) {
      for (int32_t i = 0; i < k; ++i)
        fprintf(f, "src=%d span_us=%.2f\n", sources[i], (hb[16 * i + 10] - hb[16 * i + 9]) / 1e3);
      fclose(f);
    }
  }
  for (int32_t i = 0; i < k; ++i) {
    if (!hb[16 * i + 4]) {  // stopped before a long run of small levels: rerun it with the handover
      gi_bfs_stats s{};
      GI_TRY(bfs_fused_t<OffT>(g, sources[i], o, d_out + (int64_t)i * out_stride, &s));
      if (stats) stats[i] = s;
      continue;
    }
    if (!stats) continue;
    gi_bfs_stats s{};
    s.levels = (int32_t)hb[16 * i];
    s.pull_levels = (int32_t)hb[16 * i + 3];
    s.reached = hb[16 * i + 5];
    s.edges_traversed = hb[16 * i + 6];
    s.edges_examined = hb[16 * i + 7];
    s.pull_vertices = hb[16 * i + 8];
    s.launches = i == 0 ? 1 : 0;
    s.total_ms = ms / (float)k;
    stats[i] = s;
  }
  return GI_OK;
}

gi_status bfs_fused(gi_graph g, int32_t source, const gi_bfs_opts& o, int32_t* d_out, gi_bfs_stats* stats) {
  if (g->off64) return bfs_fused_t<int64_t>(g, source, o, d_out, stats);
  return bfs_fused_t<int32_t>(g, source, o, d_out, stats);
}

gi_status bfs_fused_multi(gi_graph g, int32_t k, const int32_t* sources, const gi_bfs_opts& o, int32_t* d_out,
                          int64_t out_stride, gi_bfs_stats* stats) {
  if (g->off64) return bfs_fused_multi_t<int64_t>(g, k, sources, o, d_out, out_stride, stats);
  return bfs_fused_multi_t<int32_t>(g, k, sources, o, d_out, out_stride, stats);
}

}  // namespace gi
