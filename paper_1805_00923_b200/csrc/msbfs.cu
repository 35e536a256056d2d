// msbfs.cu — bit-parallel multi-source BFS: up to 64 sources in one traversal.
//
// The batched form of edgeset.apply for the multi-source BFS workloads of
// BASELINE configs 2/4/5 ("BFS from 64 seeded random sources"): the vertex
// payload of the BFS frontier (Table 2's
// edges.from(frontier).to(filter).apply) becomes a 64-bit mask, bit i = "in
// source i's frontier", so one pass over an edge serves every source. Each
// source's result is exactly a BFS tree of its own (every bit follows the
// level-synchronous BFS of its source; parents are in-neighbours one level
// closer, reading R8). The direction choice per level is the single-source
// rule (R7) over the union frontier.
//
//   seen[v]    bits of the sources that have reached v (levels <= current)
//   fr[c][v]   bits of the sources whose current frontier holds v
//   act[c]     the vertices with fr[c][v] != 0 (push levels read it)
// Per level (direction: pull iff |F| + sum outdeg F > m / 8 — a pull rarely
// exits early here, since a vertex stops only once it has all k sources):
//   pull (DensePull + early exit): light rows (in-degree < 32) a thread each;
//     heavy rows cut into chunks of <= 1024 in-edges, a warp per chunk (chunks
//     of one row race through atomicOr on seen / fr_next, R8 parents either
//     way); a row ORs the frontier masks of its in-neighbours into the bits it
//     misses, recording for every new bit an in-neighbour that brought it, and
//     stops once it has every source;
//   push (SparsePush): the active vertices' out-edges, concatenated by an
//     inclusive prefix of their out-degrees and walked 32 at a time, a lane per
//     edge; an edge claims new bits with atomicOr on seen (the returned old
//     value says which bits this edge won) and adds them to the next frontier.
//     Sinks (out-degree 0) never enter the active list.
// Parents are staged vertex-major (par[v][i], rows of k rounded up to a power of two >= 8) so a
// vertex's bits land in one 256-byte row; the epilogue (registers, a lane per
// vertex) writes them into the k output rows (int32[k][n], input ids; -1 where
// source i never reached v) and counts, per source, the vertices reached and
// their out-degrees.
#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include <cub/cub.cuh>

#include "gi_internal.cuh"
#include "pr_common.cuh"

namespace gi {
namespace {

#ifndef GI_MS_OUT
#define GI_MS_OUT 1  // diagnostics: 0 drops the parent writes
#endif
#ifndef GI_MS_CS
#define GI_MS_CS 0
#endif
constexpr int kMsT = 256;
#ifndef GI_MS_LMINB
#define GI_MS_LMINB 4  // min resident CTAs per SM requested from ptxas (register cap: 64) for the light pull
#endif
#ifndef GI_MS_OMINB
#define GI_MS_OMINB 6  // min resident CTAs per SM for the OR level's vertex kernel (0: no cap; 6: 40 registers, config 4 1.105 -> 1.005 ms)
#endif
#ifndef GI_MS_HMINB
#define GI_MS_HMINB 6  // ... and for the heavy pull (40 registers: 6 CTAs per SM hide the L2 gather latency;
                       // 13.6 vs 14.1-16.4 ms for config 4's 16-source pass)
#endif
#ifndef GI_MS_HEAVY
#define GI_MS_HEAVY 32
#endif
constexpr int64_t kHeavy = GI_MS_HEAVY;  // rows with at least this many in-edges are pulled by whole warps
constexpr int kMsPullDiv = 8;     // bit-parallel direction rule: pull iff |F| + sum outdeg F > m / 8 (R21)
constexpr int kMsPullDivBig = 12; // ... m / 12 when the vertex state the push hits at random exceeds L2
// segmented OR pull iff the rows still missing a source hold > this fraction of
// the in-edges: a row pull scans those rows to the end. With 16-bit masks the row
// pull is cheap enough to win below ~0.6 m (config 4, 16 sources: level 2 at m
// 3.95 vs 6.17 ms, level 3 at 0.56 m 3.8 vs 3.3 ms); 32-bit rows win nowhere
// measured (config 2, 32 sources: every pull level faster as OR)
constexpr double kSegOrFrac16 = 0.7, kSegOrFrac32 = 0.25;
// row pull over the listed incomplete rows below this fraction of m: config 4's
// third pull level (0.0006 m) 1.06 -> 0.67 ms; at 0.23 m (its second) listing
// cost more than it saved (3.0 -> 3.4 ms), at 0.036 m on config 2 too (0.21 -> 0.26)
constexpr double kSparseFrac = 1.0 / 64;
constexpr int kPushChunk = 256;   // push: out-edges per warp at least
#ifndef GI_MS_BATCH
#define GI_MS_BATCH 2
#endif
constexpr int kPullBatch = GI_MS_BATCH;  // in-edge gathers in flight per pull step
#ifndef GI_MS_OR_BATCH
#define GI_MS_OR_BATCH 2
#endif
constexpr int kOrBatch = GI_MS_OR_BATCH;  // ... per step of a light row's parent scan (OR levels)
#ifndef GI_MS_HCHUNK
#define GI_MS_HCHUNK 1024
#endif
constexpr int kHChunk = GI_MS_HCHUNK;  // heavy-row in-edges per pull work item
#ifndef GI_MS_HPER
#define GI_MS_HPER 16
#endif
constexpr int kHeavyPer = GI_MS_HPER;  // heavy chunks per warp
#ifndef GI_MS_LPERSM
#define GI_MS_LPERSM 16
#endif
constexpr int kLightPerSM = GI_MS_LPERSM;  // light-row pull CTAs per SM (grid-stride beyond)

struct MsArgs {
  int64_t n;
  const void* csr_off;
  const int32_t* __restrict__ csr_idx;
  const void* csc_off;
  const int32_t* __restrict__ csc_idx;
  const int32_t* __restrict__ outdeg;
  const int32_t* __restrict__ perm;  // internal -> input id (null: not relabelled)
  const int32_t* __restrict__ inv;   // input -> internal id
  unsigned long long* seen;
  const unsigned long long* __restrict__ fcur;
  const void* fc;                    // the frontier masks the pull levels gather: fcur itself, or a copy
                                     //   narrowed to 16 / 32 bits when k <= 16 / 32 (4x / 2x smaller, so a
                                     //   billion-edge graph's gathered array stays in L2)
  unsigned long long* fnext;
  const int32_t* __restrict__ acur;  // active vertices of the current level (push)
  int32_t* anext;                    // active vertices of the next level
  unsigned long long* cnt;           // [0] |active next|, [1] sum outdeg, [2] OR of new bits, [3] edges examined,
                                     // [4] in-edges of the rows that got every source this level, [5] |rlist|
  int32_t* par;                      // heavy rows' parents (input ids): par[hidx[v] * kp + source bit]
  int kp;                            // par row stride: k rounded up to a power of two >= 8
  uint8_t* par8;                     // light rows: par8[v * 64 + source bit] = index of the parent in v's
                                     //   in-edge list (< 32), 0xFF = v is that source itself
  const int32_t* __restrict__ hidx;  // heavy row -> its par row, -1 for a light row
  int par_all;                       // k <= 16: every row keeps int32 parents, par[v * kp + source bit]
                                     //   (64 bytes per row, the size of a byte row): no byte rows, no
                                     //   read-merge-write, no in-edge scans in the push
  int64_t nact;
  unsigned long long all;            // mask of the k sources
  const uint32_t* acc32;             // segmented OR pull: OR of each row's in-neighbours' frontier masks
  const uint32_t* acc32hi;           //   ... of their upper 32 bits (k > 32; else null)
  int32_t* rlist;                    // segmented OR pull: heavy rows with new bits (parents resolved by warps);
                                     //   sparse row pulls: the light rows still missing a source
  int64_t nlist;                     // sparse row pulls: rows in rlist
};

__device__ __forceinline__ int32_t in_id(const MsArgs& A, int32_t v) { return A.perm ? __ldg(&A.perm[v]) : v; }

// edge-index streams are read once per level: evict-first (ld.global.cs) keeps
// the frontier masks, seen and the parent rows in L2
__device__ __forceinline__ int32_t ms_idx(const int32_t* p) {
#if GI_MS_CS
  return __ldcs(p);
#else
  return __ldg(p);
#endif
}

// heavy row (several writers may claim bits of it concurrently): entries of
// the bits in m := val; a sector whose 8 bits are all in m is stored whole
// with one 256-bit store, other bits one entry at a time
__device__ __forceinline__ void par_put(int32_t* row, unsigned long long m, int32_t val) {
  while (m) {
    const int g = (__ffsll((long long)m) - 1) >> 3;
    const unsigned nm = (unsigned)(m >> (8 * g)) & 0xFFu;
    if (nm == 0xFFu) {
      asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(row + 8 * g), "r"(val) : "memory");
    } else {
      for (unsigned q = nm; q; q &= q - 1) row[8 * g + __ffs(q) - 1] = val;
    }
    m &= ~(0xFFull << (8 * g));
  }
}

// the par row of vertex w: its own in par_all mode, else its heavy row (-1: a byte row)
__device__ __forceinline__ int64_t par_row(const MsArgs& A, int32_t w) {
  return A.par_all ? (int64_t)w : (int64_t)__ldg(&A.hidx[w]);
}

// int32 parents of a row whose only writer is this thread (a pull): a sector
// none of whose bits was known before (old) is written whole — the other
// entries get placeholders, masked by seen at the end — so no sector is
// partially written; other sectors one entry per new bit
__device__ __forceinline__ void par_put_owner(int32_t* row, unsigned long long m, unsigned long long old,
                                              int32_t val) {
  while (m) {
    const int g = (__ffsll((long long)m) - 1) >> 3;
    const unsigned nm = (unsigned)(m >> (8 * g)) & 0xFFu;
    if (((old >> (8 * g)) & 0xFFull) == 0ull) {
      asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(row + 8 * g), "r"(val) : "memory");
    } else {
      for (unsigned q = nm; q; q &= q - 1) row[8 * g + __ffs(q) - 1] = val;
    }
    old |= (unsigned long long)nm << (8 * g);
    m &= ~(0xFFull << (8 * g));
  }
}

// light row: byte entries of the bits in m := idx, read-merge-write per 32-byte
// sector (32 sources); the pull thread is the row's only writer in its launch
__device__ __forceinline__ void par8_put(uint8_t* row, unsigned long long m, uint32_t idx) {
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    const unsigned nm = (unsigned)(m >> (32 * g));
    if (!nm) continue;
    uint32_t x[8];
    asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7])
                 : "l"(row + 32 * g));
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const unsigned q = (nm >> (4 * j)) & 0xFu;
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if ((q >> b) & 1u) x[j] = (x[j] & ~(0xFFu << (8 * b))) | (idx << (8 * b));
    }
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(row + 32 * g), "r"(x[0]), "r"(x[1]),
                 "r"(x[2]), "r"(x[3]), "r"(x[4]), "r"(x[5]), "r"(x[6]), "r"(x[7])
                 : "memory");
  }
}

// warp-level append through a shared-memory buffer: one tail atomic per 32
// appended rows, no block barrier (the rows of a CTA round finish unevenly)
__device__ __forceinline__ void ms_warp_flush(const MsArgs& A, int32_t* buf, int cnt) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  unsigned long long pos = 0;
  if (lane == 0) pos = atomicAdd(&A.cnt[0], (unsigned long long)cnt);
  pos = __shfl_sync(0xffffffffu, pos, 0);
  if (lane < cnt) A.anext[pos + lane] = buf[lane];
  __syncwarp();
}
__device__ __forceinline__ void ms_warp_append(const MsArgs& A, bool act, int32_t v, int32_t* buf, int& nbuf) {
  const int lane = threadIdx.x & 31;
  const unsigned am = __ballot_sync(0xffffffffu, act);
  if (!am) return;
  if (act) buf[nbuf + __popc(am & ((1u << lane) - 1u))] = v;
  nbuf += __popc(am);
  if (nbuf >= 32) {
    ms_warp_flush(A, buf, 32);
    nbuf -= 32;
    if (lane < nbuf) buf[lane] = buf[32 + lane];
    __syncwarp();
  }
}

// the level's counters (cnt[1..3]), reduced over the CTA once at kernel end;
// every thread of the CTA calls it
__device__ __forceinline__ void ms_counters(const MsArgs& A, long long deg, unsigned long long bits, long long exam,
                                            long long done) {
  __shared__ unsigned long long s_red[4 * (kMsT / 32)];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    deg += __shfl_xor_sync(0xffffffffu, deg, o);
    bits |= __shfl_xor_sync(0xffffffffu, bits, o);
    exam += __shfl_xor_sync(0xffffffffu, exam, o);
    done += __shfl_xor_sync(0xffffffffu, done, o);
  }
  if (lane == 0) {
    s_red[4 * w] = (unsigned long long)deg;
    s_red[4 * w + 1] = bits;
    s_red[4 * w + 2] = (unsigned long long)exam;
    s_red[4 * w + 3] = (unsigned long long)done;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long d = 0, b = 0, x = 0, c = 0;
    for (int i = 0; i < kMsT / 32; ++i) {
      d += s_red[4 * i];
      b |= s_red[4 * i + 1];
      x += s_red[4 * i + 2];
      c += s_red[4 * i + 3];
    }
    if (d) atomicAdd(&A.cnt[1], d);
    if (b) atomicOr(&A.cnt[2], b);
    if (x) atomicAdd(&A.cnt[3], x);
    if (c) atomicAdd(&A.cnt[4], c);
  }
}

// narrowed frontier masks for the pull gathers (k <= 8 * sizeof(FM) sources)
template <typename FM>
__global__ void k_ms_narrow(const unsigned long long* __restrict__ f, int64_t n, FM* __restrict__ out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    out[v] = (FM)f[v];
}
template <typename FM>
__device__ __forceinline__ unsigned long long ms_fget(const MsArgs& A, int32_t v) {
  return (unsigned long long)reinterpret_cast<const FM*>(A.fc)[v];
}

// LIST: the level's rows are A.rlist[0, A.nlist) (the light rows still missing a
// source, sparse pull levels) and fnext is zeroed beforehand; else every row
template <typename OffT, typename FM, bool LIST = false>
__global__ void __launch_bounds__(kMsT, GI_MS_LMINB) k_ms_pull(MsArgs A) {
  __shared__ int32_t s_buf[kMsT / 32][64];  // per-warp staging of the rows joining the next frontier
  int32_t* wbuf = s_buf[threadIdx.x >> 5];
  int nbuf = 0;
  const OffT* __restrict__ off = static_cast<const OffT*>(A.csc_off);
  long long tdeg = 0, exam = 0, tdone = 0;
  unsigned long long tbits = 0;
  const int64_t N = LIST ? A.nlist : A.n;
  for (int64_t b = blockIdx.x * (int64_t)kMsT; b < N; b += (int64_t)gridDim.x * kMsT) {
    const int64_t i = b + threadIdx.x;
    const int32_t w = LIST ? (i < N ? __ldg(&A.rlist[i]) : 0) : (int32_t)i;
    bool act = false;
    unsigned long long found = 0;
    if (i < N) {
      const int64_t e0 = (int64_t)off[w], e1 = (int64_t)off[w + 1];
      const unsigned long long s = e1 - e0 >= kHeavy ? A.all : A.seen[w];  // heavy rows: k_ms_pull_heavy
      if (s != A.all) {
        for (int64_t e = e0; e < e1; e += kPullBatch) {  // kPullBatch independent gathers per step
          int32_t v[kPullBatch];
          unsigned long long f[kPullBatch];
#pragma unroll
          for (int j = 0; j < kPullBatch; ++j) v[j] = e + j < e1 ? ms_idx(&A.csc_idx[e + j]) : -1;
#pragma unroll
          for (int j = 0; j < kPullBatch; ++j) f[j] = v[j] >= 0 ? ms_fget<FM>(A, v[j]) : 0ull;
          exam += min((int64_t)kPullBatch, e1 - e);
#pragma unroll
          for (int j = 0; j < kPullBatch; ++j) {
            const unsigned long long m = f[j] & ~s & ~found;
            if (m) {  // the parent of these bits: in-edge e + j - e0 of the row
              if (GI_MS_OUT) {
                if (A.par_all) par_put_owner(A.par + (int64_t)w * A.kp, m, s | found, in_id(A, v[j]));
                else par8_put(A.par8 + (int64_t)w * 64, m, (uint32_t)(e + j - e0));
              }
              found |= m;
            }
          }
          if ((s | found) == A.all) break;
        }
        if (found) {
          A.seen[w] = s | found;
          if ((s | found) == A.all) tdone += e1 - e0;
          const int32_t deg = __ldg(&A.outdeg[w]);
          act = deg > 0;  // a sink never pushes: it stays out of the active list
          tdeg += deg;
          tbits |= found;
        }
      }
      if (!LIST || found) A.fnext[w] = found;  // heavy rows: 0 here, k_ms_pull_heavy ORs into it
    }
    ms_warp_append(A, act, w, wbuf, nbuf);
  }
  if (nbuf > 0) ms_warp_flush(A, wbuf, nbuf);
  ms_counters(A, tdeg, tbits, exam, tdone);
}

// pull for the heavy rows (in-degree >= kHeavy), edge-balanced: the rows are
// cut into chunks of kHChunk in-edges (built once per graph; a row of at most
// kHChunk in-edges is one chunk) and every warp takes a contiguous run of
// chunks, kPullBatch x 32 gathers in flight per step. Chunks of one row may run
// concurrently: each ORs what it found into seen / fnext with atomics, and the
// chunk whose atomicOr on fnext returns 0 appends the row to the next frontier.
// A chunk stops early once seen (as of its start) plus its own finds hold
// every source. A new bit's parent is the lowest lane bringing it in its step;
// lane L holds the parents of sources L and 32 + L, so a row's parents leave
// in two coalesced stores at the end of the chunk (chunks of a split row race
// on a bit found by both; either store is a valid parent).
// 32x32 bit-matrix transpose across a warp: on return bit l of lane L's word
// is bit L of lane l's input word
__device__ __forceinline__ unsigned warp_transpose32(unsigned x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 16, i = 0; j > 0; j >>= 1, ++i) {
    const unsigned mk = i == 0 ? 0x0000FFFFu : i == 1 ? 0x00FF00FFu : i == 2 ? 0x0F0F0F0Fu : i == 3 ? 0x33333333u : 0x55555555u;
    const unsigned y = __shfl_xor_sync(0xffffffffu, x, j);
    x = (lane & j) ? (x & ~mk) | ((y >> j) & mk) : (x & mk) | ((y << j) & ~mk);
  }
  return x;
}

template <typename OffT, typename FM>
__global__ void __launch_bounds__(kMsT, GI_MS_HMINB) k_ms_pull_heavy(MsArgs A, const int2* __restrict__ hch, int64_t C) {
  __shared__ int32_t s_buf[kMsT / 32][32];  // per-warp staging of the rows joining the next frontier
  const OffT* __restrict__ off = static_cast<const OffT*>(A.csc_off);
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int64_t nw = (int64_t)gridDim.x * (kMsT / 32);
  const int64_t gw = blockIdx.x * (int64_t)(kMsT / 32) + wp;
  const int64_t per = (C + nw - 1) / nw;
  const int64_t c1 = min(C, (gw + 1) * per);
  long long tdeg = 0, exam = 0, tdone = 0;
  unsigned long long tbits = 0;
  int nbuf = 0;
  for (int64_t c = gw * per; c < c1; ++c) {
    const int2 ch = __ldg(&hch[c]);
    const int32_t w = ch.x;
    const unsigned long long s = *(volatile unsigned long long*)&A.seen[w];
    bool newact = false;
    if (s != A.all) {
      const int64_t rb = (int64_t)off[w], re = (int64_t)off[w + 1];
      const int64_t e0 = rb + ch.y, e1 = min(re, e0 + kHChunk);
      const bool whole = re - rb <= kHChunk;  // the warp is the row's only writer this launch
      int32_t* prow = A.par + par_row(A, w) * A.kp;
      // lane L keeps the parents of sources L (plo) and 32 + L (phi)
      int32_t plo = 0, phi = 0;
      unsigned long long found = 0;
      for (int64_t b = e0; b < e1; b += 32 * kPullBatch) {
        int32_t v[kPullBatch];
        unsigned long long f[kPullBatch];
#pragma unroll
        for (int j = 0; j < kPullBatch; ++j) {
          const int64_t e = b + 32 * j + lane;
          v[j] = e < e1 ? ms_idx(&A.csc_idx[e]) : -1;
        }
#pragma unroll
        for (int j = 0; j < kPullBatch; ++j) f[j] = v[j] >= 0 ? ms_fget<FM>(A, v[j]) : 0ull;
        if (lane == 0) exam += min((int64_t)32 * kPullBatch, e1 - b);
#pragma unroll
        for (int j = 0; j < kPullBatch; ++j) {
          const unsigned long long mj = f[j] & ~s & ~found;
          const unsigned lo = __reduce_or_sync(0xffffffffu, (unsigned)mj);
          // masks of <= 32 bits (k <= 32) have no upper half: one reduction per slot
          const unsigned hi = sizeof(FM) > 4 ? __reduce_or_sync(0xffffffffu, (unsigned)(mj >> 32)) : 0u;
          if ((lo | hi) == 0u) continue;  // warp-uniform: nothing new from this batch slot
          const int32_t vin = mj ? in_id(A, v[j]) : 0;
          // each new bit's parent: the lowest lane bringing it (bit-matrix transpose of the lanes' masks)
          if (lo) {
            const unsigned tl = warp_transpose32((unsigned)mj);
            const int32_t p = __shfl_sync(0xffffffffu, vin, tl ? __ffs(tl) - 1 : 0);
            if (tl) plo = p;
          }
          if (hi) {
            const unsigned th = warp_transpose32((unsigned)(mj >> 32));
            const int32_t p = __shfl_sync(0xffffffffu, vin, th ? __ffs(th) - 1 : 0);
            if (th) phi = p;
          }
          found |= ((unsigned long long)hi << 32) | lo;
        }
        if ((s | found) == A.all) break;
      }
      if (GI_MS_OUT && found) {
        // whole row: a sector without known bits is written in full (placeholders
        // for its unfound sources), else only the new entries; split rows: new entries
        const unsigned kl = (unsigned)s, kh = (unsigned)(s >> 32);
        const unsigned nl = (unsigned)found, nh = (unsigned)(found >> 32);
        const int sh = lane & ~7;
        const bool wl = (nl >> lane) & 1u || (whole && ((nl >> sh) & 0xFFu) && !((kl >> sh) & 0xFFu));
        const bool wh = (nh >> lane) & 1u || (whole && ((nh >> sh) & 0xFFu) && !((kh >> sh) & 0xFFu));
        if (wl && lane < A.kp) prow[lane] = plo;
        if (wh && 32 + lane < A.kp) prow[32 + lane] = phi;
      }
      if (found && lane == 0) {
        const unsigned long long old = atomicOr(&A.seen[w], found);
        if (old != A.all && (old | found) == A.all) tdone += re - rb;  // this chunk completed the row
        tbits |= found;
        if (atomicOr(&A.fnext[w], found) == 0ull) {  // the row's first bits this level
          const int32_t d = __ldg(&A.outdeg[w]);
          tdeg += d;
          newact = d > 0;
        }
      }
    }
    if (__shfl_sync(0xffffffffu, newact, 0)) {
      if (lane == 0) s_buf[wp][nbuf] = w;
      if (++nbuf == 32) {  // one atomic per 32 appended rows
        __syncwarp();
        unsigned long long pos = 0;
        if (lane == 0) pos = atomicAdd(&A.cnt[0], 32ull);
        pos = __shfl_sync(0xffffffffu, pos, 0);
        A.anext[pos + lane] = s_buf[wp][lane];
        __syncwarp();
        nbuf = 0;
      }
    }
  }
  __syncwarp();
  if (nbuf > 0) {
    unsigned long long pos = 0;
    if (lane == 0) pos = atomicAdd(&A.cnt[0], (unsigned long long)nbuf);
    pos = __shfl_sync(0xffffffffu, pos, 0);
    if (lane < nbuf) A.anext[pos + lane] = s_buf[wp][lane];
  }
  ms_counters(A, tdeg, tbits, exam, tdone);
}

__global__ void k_ms_csc_in(const int32_t* __restrict__ idx, int64_t m, const int32_t* __restrict__ perm,
                            int32_t* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = perm ? __ldg(&perm[idx[e]]) : idx[e];
}

__global__ void k_ms_hidx(const int32_t* __restrict__ heavy, int64_t nh, int32_t* __restrict__ hidx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nh; i += (int64_t)gridDim.x * blockDim.x)
    hidx[heavy[i]] = (int32_t)i;
}

// heavy-row chunks: cc[i] = chunks of heavy row i; then (row, first in-edge offset) per chunk
template <typename OffT>
__global__ void k_ms_hchunk_count(const OffT* __restrict__ off, const int32_t* __restrict__ heavy, int64_t nh,
                                  int32_t* __restrict__ cc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nh; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t w = heavy[i];
    cc[i] = (int32_t)(((int64_t)off[w + 1] - (int64_t)off[w] + kHChunk - 1) / kHChunk);
  }
}
__global__ void k_ms_hchunk_fill(const int32_t* __restrict__ heavy, int64_t nh, const int32_t* __restrict__ cc,
                                 const int32_t* __restrict__ cp, int2* __restrict__ hch) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nh; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t w = heavy[i], c = cc[i], base = cp[i] - c;
    for (int32_t j = 0; j < c; ++j) hch[base + j] = make_int2(w, j * kHChunk);
  }
}

// the heavy rows (in-degree >= kHeavy), appended in any order
template <typename OffT>
__global__ void k_ms_heavy_list(const OffT* __restrict__ off, int64_t n, int32_t* __restrict__ list,
                                unsigned long long* __restrict__ cnt) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    if ((int64_t)off[v + 1] - (int64_t)off[v] >= kHeavy) list[atomicAdd(cnt, 1ull)] = (int32_t)v;
}


// push, edge-parallel: the active vertices' out-edges, concatenated (dp =
// inclusive prefix of their out-degrees), are split evenly over the warps and
// walked 32 at a time, a lane per edge. A warp keeps a window of 32 prefix
// entries; each lane finds its edge's vertex in it by a 5-step search over
// shuffles, so low-degree vertices share a step and a hub spreads over many
// warps.
template <typename OffT>
__global__ void __launch_bounds__(kMsT) k_ms_push(MsArgs A, const long long* __restrict__ dp) {
  __shared__ int32_t s_buf[kMsT / 32][64];  // per-warp staging of the vertices joining the next frontier
  const OffT* __restrict__ off = static_cast<const OffT*>(A.csr_off);
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  int nbuf = 0;
  const int64_t nw = (int64_t)gridDim.x * (kMsT / 32);
  const int64_t gw = blockIdx.x * (int64_t)(kMsT / 32) + wp;
  long long deg = 0, exam = 0, done = 0;
  unsigned long long bits = 0;
  const long long E = A.nact > 0 ? __ldg(&dp[A.nact - 1]) : 0;
  const long long per = (E + nw - 1) / nw;
  long long e = gw * per;
  const long long eend = min(E, e + per);
  if (e < eend) {
    int64_t i0 = 0, hi = A.nact;  // the active vertex holding edge e: first i with dp[i] > e
    while (i0 < hi) {
      const int64_t mid = (i0 + hi) >> 1;
      if (__ldg(&dp[mid]) <= e) i0 = mid + 1;
      else hi = mid;
    }
    while (e < eend) {  // warp-uniform
      const long long P = i0 + lane < A.nact ? __ldg(&dp[i0 + lane]) : LLONG_MAX;
      const long long Pprev = i0 > 0 ? __ldg(&dp[i0 - 1]) : 0;
      const long long stop = min(eend, min(e + 32, (long long)__shfl_sync(0xffffffffu, P, 31)));
      const long long my = e + lane;
      int pos = 0;  // my edge's vertex: i0 + #{l : P_l <= my}
#pragma unroll
      for (int s = 16; s > 0; s >>= 1)
        if (__shfl_sync(0xffffffffu, P, pos + s - 1) <= my) pos += s;
      const long long pl = __shfl_sync(0xffffffffu, P, pos > 0 ? pos - 1 : 0);  // every lane takes part
      const long long start = pos ? pl : Pprev;
      bool newact = false;
      int32_t w = 0;
      if (my < stop) {
        const int32_t u = __ldg(&A.acur[i0 + pos]);
        w = ms_idx(&A.csr_idx[(int64_t)off[u] + (my - start)]);
        ++exam;
        const unsigned long long m = A.fcur[u] & ~*(volatile unsigned long long*)&A.seen[w];
        if (m) {
          const unsigned long long old = atomicOr(&A.seen[w], m);
          const unsigned long long got = m & ~old;  // the bits this edge claims
          if (got) {
            if ((old | got) == A.all) {  // this claim completed w: its in-edges leave the pull's scan mass
              const OffT* __restrict__ coff = static_cast<const OffT*>(A.csc_off);
              done += (long long)(coff[w + 1] - coff[w]);
            }
            if (GI_MS_OUT) {
              const int64_t h = par_row(A, w);
              if (h >= 0) {
                par_put(A.par + h * A.kp, got, in_id(A, u));
              } else {  // light row: u's position in w's in-edge list (< 32 entries, scanned 8 at a time)
                const OffT* __restrict__ coff = static_cast<const OffT*>(A.csc_off);
                const int64_t lo = (int64_t)coff[w], hi = (int64_t)coff[w + 1];
                int pos = 0;
                for (int64_t e = lo; e < hi; e += 8) {
                  int32_t x[8];
#pragma unroll
                  for (int j = 0; j < 8; ++j) x[j] = e + j < hi ? __ldg(&A.csc_idx[e + j]) : -1;
#pragma unroll
                  for (int j = 0; j < 8; ++j)
                    if (x[j] == u) pos = (int)(e + j - lo);
                }
                for (unsigned long long x = got; x; x &= x - 1)
                  A.par8[(int64_t)w * 64 + __ffsll((long long)x) - 1] = (uint8_t)pos;
              }
            }
            bits |= got;
            if (atomicOr(&A.fnext[w], got) == 0ull) {  // w's first bits this level: it joins the next frontier
              const int32_t dw = __ldg(&A.outdeg[w]);
              newact = dw > 0;  // sinks stay out of the active list
              deg += dw;
            }
          }
        }
      }
      const unsigned am = __ballot_sync(0xffffffffu, newact);
      if (am) {
        if (newact) s_buf[wp][nbuf + __popc(am & ((1u << lane) - 1u))] = w;
        nbuf += __popc(am);
        if (nbuf >= 32) {  // one atomic per 32 appended vertices
          __syncwarp();
          unsigned long long pos2 = 0;
          if (lane == 0) pos2 = atomicAdd(&A.cnt[0], 32ull);
          pos2 = __shfl_sync(0xffffffffu, pos2, 0);
          A.anext[pos2 + lane] = s_buf[wp][lane];
          __syncwarp();
          nbuf -= 32;
          if (lane < nbuf) s_buf[wp][lane] = s_buf[wp][32 + lane];
          __syncwarp();
        }
      }
      i0 += __popc(__ballot_sync(0xffffffffu, P <= stop));
      e = stop;
    }
  }
  __syncwarp();
  if (nbuf > 0) {
    unsigned long long pos = 0;
    if (lane == 0) pos = atomicAdd(&A.cnt[0], (unsigned long long)nbuf);
    pos = __shfl_sync(0xffffffffu, pos, 0);
    if (lane < nbuf) A.anext[pos + lane] = s_buf[wp][lane];
  }
  ms_counters(A, deg, bits, exam, done);
}

// ---- sparse row pulls: only the rows still missing a source ----
// Late pull levels find few rows without every source (config 4: 0.9 M in-edges
// of them at its third pull level) but a full row pull still reads every row's
// offsets and seen word and writes its next-frontier word (1.1 ms). When the
// rows missing a source hold < m / 64 in-edges the level zeroes the next frontier,
// lists those rows (light ones; heavy ones by their chunks) and pulls only them.
// warp-buffered list append: one atomic per 32 listed entries (buf: 64 per warp)
template <typename T>
__device__ __forceinline__ void list_append(bool in, T v, T* list, unsigned long long* cnt, T* buf, int& nbuf) {
  const int lane = threadIdx.x & 31;
  const unsigned m = __ballot_sync(0xffffffffu, in);
  if (in) buf[nbuf + __popc(m & ((1u << lane) - 1u))] = v;
  nbuf += __popc(m);
  if (nbuf >= 32) {
    __syncwarp();
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(cnt, 32ull);
    base = __shfl_sync(0xffffffffu, base, 0);
    list[base + lane] = buf[lane];
    __syncwarp();
    nbuf -= 32;
    if (lane < nbuf) buf[lane] = buf[32 + lane];
    __syncwarp();
  }
}
template <typename T>
__device__ __forceinline__ void list_flush(T* list, unsigned long long* cnt, T* buf, int nbuf) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  if (nbuf == 0) return;
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(cnt, (unsigned long long)nbuf);
  base = __shfl_sync(0xffffffffu, base, 0);
  if (lane < nbuf) list[base + lane] = buf[lane];
}

template <typename OffT>
__global__ void __launch_bounds__(256) k_ms_list_light(const OffT* __restrict__ off,
                                                      const unsigned long long* __restrict__ seen, int64_t n,
                                                      unsigned long long all, int32_t* __restrict__ list,
                                                      unsigned long long* cnt) {
  __shared__ int32_t s_buf[8][64];
  int nbuf = 0;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x; b < n; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = b + threadIdx.x;  // warp-uniform loop: blockDim is a multiple of 32
    bool in = false;
    if (w < n && seen[w] != all) {
      const int64_t d = (int64_t)off[w + 1] - (int64_t)off[w];
      in = d > 0 && d < kHeavy;
    }
    list_append(in, (int32_t)w, list, cnt, s_buf[threadIdx.x >> 5], nbuf);
  }
  list_flush(list, cnt, s_buf[threadIdx.x >> 5], nbuf);
}
__global__ void __launch_bounds__(256) k_ms_list_chunks(const int2* __restrict__ hch, int64_t C,
                                                       const unsigned long long* __restrict__ seen,
                                                       unsigned long long all, int2* __restrict__ list,
                                                       unsigned long long* cnt) {
  __shared__ int2 s_buf[8][64];
  int nbuf = 0;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x; b < C; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = b + threadIdx.x;
    int2 ch = make_int2(0, 0);
    bool in = false;
    if (c < C) {
      ch = __ldg(&hch[c]);
      in = seen[ch.x] != all;
    }
    list_append(in, ch, list, cnt, s_buf[threadIdx.x >> 5], nbuf);
  }
  list_flush(list, cnt, s_buf[threadIdx.x >> 5], nbuf);
}

// ---- segmented OR pull (dense pull levels; 32-bit OR passes: one for k <= 32, two for k <= 64) ----
// A pull level whose rows would mostly scan to the end (rows stop early only
// once they hold every source) runs as one pass of the PageRank edge kernel over
// the segmented layout with the reduction swapped for OR (pr_segmented.cu,
// seg_or_pass): acc32[v] = OR over v's in-edges of the 32-bit frontier masks,
// staged per source segment in shared memory, so every edge costs a shared-memory
// gather instead of an L2 gather. The level's new bits are then acc32 & ~seen,
// exactly the pull's result; each new bit's parent is found by scanning the row's
// in-edges only until every NEW bit has a frontier in-neighbour (light rows a
// thread each in k_ms_or_vertex, heavy rows a warp each in k_ms_resolve_heavy).

// the frontier masks of an OR level: 32-bit words (staged by the OR pass) and,
// k <= 16, the 16-bit copy the parent resolution gathers
__global__ void k_ms_narrow_or(const unsigned long long* __restrict__ f, int64_t n, uint32_t* __restrict__ o32,
                               uint16_t* __restrict__ o16, uint32_t* __restrict__ o32hi) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long x = f[v];
    o32[v] = (uint32_t)x;
    if (o16) o16[v] = (uint16_t)x;
    if (o32hi) o32hi[v] = (uint32_t)(x >> 32);
  }
}

// the level's vertex pass: new = acc32 & ~seen; seen, next frontier, active list,
// counters; a light row's parents found by its thread, a heavy row queued in rlist
template <typename OffT, typename FM>
#if GI_MS_OMINB
__global__ void __launch_bounds__(kMsT, GI_MS_OMINB) k_ms_or_vertex(MsArgs A) {
#else
__global__ void __launch_bounds__(kMsT) k_ms_or_vertex(MsArgs A) {
#endif
  __shared__ int32_t s_buf[kMsT / 32][64], s_hbuf[kMsT / 32][64];
  int32_t* wbuf = s_buf[threadIdx.x >> 5];
  int32_t* hbuf = s_hbuf[threadIdx.x >> 5];
  int nbuf = 0, nhbuf = 0;
  const int lane = threadIdx.x & 31;
  const OffT* __restrict__ off = static_cast<const OffT*>(A.csc_off);
  long long tdeg = 0, exam = 0, tdone = 0;
  unsigned long long tbits = 0;
  for (int64_t b = blockIdx.x * (int64_t)kMsT; b < A.n; b += (int64_t)gridDim.x * kMsT) {
    const int32_t w = (int32_t)(b + threadIdx.x);
    bool act = false, heavy = false;
    if (w < A.n) {
      const unsigned long long s = A.seen[w];
      unsigned long long a = (unsigned long long)__ldcs(&A.acc32[w]);
      if (A.acc32hi) a |= (unsigned long long)__ldcs(&A.acc32hi[w]) << 32;  // k > 32: the second OR pass
      const unsigned long long nb = a & ~s & A.all;
      A.fnext[w] = nb;
      if (nb) {
        A.seen[w] = s | nb;
        const int64_t e0 = (int64_t)off[w], e1 = (int64_t)off[w + 1];
        if ((s | nb) == A.all) tdone += e1 - e0;
        const int32_t deg = __ldg(&A.outdeg[w]);
        act = deg > 0;
        tdeg += deg;
        tbits |= nb;
        if (e1 - e0 >= kHeavy) {
          heavy = true;
        } else {  // the parents of the new bits: the first frontier in-neighbour bringing each
          unsigned long long rem = nb, known = s;
          for (int64_t e = e0; rem && e < e1; e += kOrBatch) {
            int32_t v[kOrBatch];
            unsigned long long f[kOrBatch];
#pragma unroll
            for (int j = 0; j < kOrBatch; ++j) v[j] = e + j < e1 ? ms_idx(&A.csc_idx[e + j]) : -1;
#pragma unroll
            for (int j = 0; j < kOrBatch; ++j) f[j] = v[j] >= 0 ? ms_fget<FM>(A, v[j]) : 0ull;
            exam += min((int64_t)kOrBatch, e1 - e);
#pragma unroll
            for (int j = 0; j < kOrBatch; ++j) {
              const unsigned long long m = f[j] & rem;
              if (m) {
                if (GI_MS_OUT) {
                  if (A.par_all) par_put_owner(A.par + (int64_t)w * A.kp, m, known, in_id(A, v[j]));
                  else par8_put(A.par8 + (int64_t)w * 64, m, (uint32_t)(e + j - e0));
                }
                known |= m;
                rem &= ~m;
              }
            }
          }
        }
      }
    }
    list_append(heavy, w, A.rlist, &A.cnt[5], hbuf, nhbuf);  // heavy rows: one atomic per 32
    ms_warp_append(A, act, w, wbuf, nbuf);
  }
  list_flush(A.rlist, &A.cnt[5], hbuf, nhbuf);
  if (nbuf > 0) ms_warp_flush(A, wbuf, nbuf);
  ms_counters(A, tdeg, tbits, exam, tdone);
}

// heavy rows with new bits (rlist, cnt[5] of them), a warp per row: 32 x
// kPullBatch in-edges per step until every new bit has a parent (the lowest lane
// bringing it: bit-matrix transpose, lane L ends up with source L's parent)
template <typename OffT, typename FM>
__global__ void __launch_bounds__(kMsT) k_ms_resolve_heavy(MsArgs A) {
  const OffT* __restrict__ off = static_cast<const OffT*>(A.csc_off);
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (kMsT / 32);
  const int64_t R = (int64_t)*(volatile unsigned long long*)&A.cnt[5];
  long long exam = 0;
  for (int64_t i = blockIdx.x * (int64_t)(kMsT / 32) + (threadIdx.x >> 5); i < R; i += nw) {
    const int32_t w = __ldg(&A.rlist[i]);
    const unsigned long long nb = A.fnext[w];          // this level's new bits (k_ms_or_vertex)
    const unsigned long long known = A.seen[w] & ~nb;  // bits of earlier levels
    const int64_t e0 = (int64_t)off[w], e1 = (int64_t)off[w + 1];
    using RemT = typename std::conditional<(sizeof(FM) > 4), unsigned long long, unsigned>::type;
    RemT rem = (RemT)nb;  // k <= 32: 32-bit state (fewer registers, more resident warps)
    int32_t plo = 0, phi = 0;  // lane L: the parents of sources L and 32 + L
    for (int64_t b = e0; rem && b < e1; b += 32 * kPullBatch) {
      int32_t v[kPullBatch];
      RemT f[kPullBatch];
#pragma unroll
      for (int j = 0; j < kPullBatch; ++j) {
        const int64_t e = b + 32 * j + lane;
        v[j] = e < e1 ? ms_idx(&A.csc_idx[e]) : -1;
      }
#pragma unroll
      for (int j = 0; j < kPullBatch; ++j) f[j] = v[j] >= 0 ? (RemT)ms_fget<FM>(A, v[j]) : (RemT)0;
      if (lane == 0) exam += min((int64_t)32 * kPullBatch, e1 - b);
#pragma unroll
      for (int j = 0; j < kPullBatch; ++j) {
        const RemT mj = f[j] & rem;
        const unsigned lo = __reduce_or_sync(0xffffffffu, (unsigned)mj);
        unsigned hi = 0u;
        if constexpr (sizeof(FM) > 4) hi = __reduce_or_sync(0xffffffffu, (unsigned)((unsigned long long)mj >> 32));
        if ((lo | hi) == 0u) continue;
        const int32_t vin = mj ? in_id(A, v[j]) : 0;
        if (lo) {
          const unsigned tl = warp_transpose32((unsigned)mj);
          const int32_t p = __shfl_sync(0xffffffffu, vin, tl ? __ffs(tl) - 1 : 0);
          if (tl) plo = p;
        }
        if constexpr (sizeof(FM) > 4) {
          if (hi) {
            const unsigned th = warp_transpose32((unsigned)((unsigned long long)mj >> 32));
            const int32_t p = __shfl_sync(0xffffffffu, vin, th ? __ffs(th) - 1 : 0);
            if (th) phi = p;
          }
          rem &= ~(((unsigned long long)hi << 32) | lo);
        } else {
          rem &= ~lo;
        }
      }
    }
    if (GI_MS_OUT) {  // a sector without earlier bits is written whole (placeholders), else the new entries
      int32_t* prow = A.par + par_row(A, w) * A.kp;
      const unsigned kl = (unsigned)known, nl = (unsigned)nb;
      const int sh = lane & ~7;
      const bool wl = ((nl >> lane) & 1u) || (((nl >> sh) & 0xFFu) && !((kl >> sh) & 0xFFu));
      if (wl && lane < A.kp) prow[lane] = plo;
      if constexpr (sizeof(FM) > 4) {
        const unsigned kh = (unsigned)(known >> 32), nh = (unsigned)(nb >> 32);
        const bool wh = ((nh >> lane) & 1u) || (((nh >> sh) & 0xFFu) && !((kh >> sh) & 0xFFu));
        if (wh && 32 + lane < A.kp) prow[32 + lane] = phi;
      }
    }
  }
  ms_counters(A, 0, 0ull, exam, 0);
}

// ---- the push levels' edge prefix: dp[i] = sum of outdeg over act[0..i] (inclusive),
// in three passes over tiles of kScanTile active vertices: tile sums, one block
// scanning the tile sums, then each tile's scan plus its offset
constexpr int kScanT = 256, kScanVT = 8, kScanTile = kScanT * kScanVT;
// block-wide exclusive scan of one value per thread (warp shuffles + one smem round)
__device__ __forceinline__ long long block_excl_scan(long long x, long long* total) {
  __shared__ long long s_w[32];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5, nwp = blockDim.x >> 5;
  long long incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_w[wp] = incl;
  __syncthreads();
  if (wp == 0) {
    long long w = lane < nwp ? s_w[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nwp) s_w[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  const long long before = (wp > 0 ? s_w[wp - 1] : 0) + incl - x;
  *total = s_w[nwp - 1];
  __syncthreads();
  return before;
}
__global__ void __launch_bounds__(kScanT) k_deg_tile_sums(const int32_t* __restrict__ act, const int32_t* __restrict__ od,
                                                         int64_t nact, long long* __restrict__ tsum) {
  const int64_t base = blockIdx.x * (int64_t)kScanTile + threadIdx.x * kScanVT;
  long long x = 0;
#pragma unroll
  for (int j = 0; j < kScanVT; ++j)
    if (base + j < nact) x += __ldg(&od[__ldg(&act[base + j])]);
  long long t;
  block_excl_scan(x, &t);
  if (threadIdx.x == 0) tsum[blockIdx.x] = t;
}
__global__ void __launch_bounds__(1024) k_scan_tile_sums(long long* __restrict__ tsum, int64_t nt) {
  // one block: thread t scans its run of ceil(nt / 1024) tile sums; exclusive result in place
  const int64_t per = (nt + 1023) / 1024, b0 = threadIdx.x * per, b1 = min(nt, b0 + per);
  long long x = 0;
  for (int64_t i = b0; i < b1; ++i) x += tsum[i];
  long long t;
  long long run = block_excl_scan(x, &t);
  for (int64_t i = b0; i < b1; ++i) {
    const long long v = tsum[i];
    tsum[i] = run;
    run += v;
  }
}
__global__ void __launch_bounds__(kScanT) k_deg_scan(const int32_t* __restrict__ act, const int32_t* __restrict__ od,
                                                    int64_t nact, const long long* __restrict__ toff,
                                                    long long* __restrict__ dp) {
  const int64_t base = blockIdx.x * (int64_t)kScanTile + threadIdx.x * kScanVT;
  long long d[kScanVT], x = 0;
#pragma unroll
  for (int j = 0; j < kScanVT; ++j) {
    d[j] = base + j < nact ? (long long)__ldg(&od[__ldg(&act[base + j])]) : 0;
    x += d[j];
  }
  long long t;
  long long run = block_excl_scan(x, &t) + toff[blockIdx.x];
#pragma unroll
  for (int j = 0; j < kScanVT; ++j) {
    run += d[j];
    if (base + j < nact) dp[base + j] = run;
  }
}

// sources: bit i at source i (internal id), its own parent in row i, active list
__global__ void k_ms_init(const int32_t* __restrict__ src_in, int k, const int32_t* __restrict__ inv, int64_t n,
                          const int32_t* __restrict__ outdeg, unsigned long long* seen, unsigned long long* f0,
                          int32_t* act, unsigned long long* cnt, int32_t* par, int kp, uint8_t* par8,
                          const int32_t* __restrict__ hidx, int par_all) {
  const int i = threadIdx.x;
  if (i >= k) return;
  const int32_t si = src_in[i];
  const int32_t s = inv ? inv[si] : si;
  atomicOr(&seen[s], 1ull << i);
  const int64_t h = par_all ? (int64_t)s : (int64_t)hidx[s];
  if (h >= 0) par[h * kp + i] = si;
  else par8[(int64_t)s * 64 + i] = 0xFF;  // the source is its own parent
  if (atomicOr(&f0[s], 1ull << i) == 0ull) {
    act[atomicAdd(&cnt[0], 1ull)] = s;
    atomicAdd(&cnt[1], (unsigned long long)outdeg[s]);
  }
}

// The pass's epilogue: out[i][v] (input ids) = source i's parent of v, or -1
// when i never reached v, and per source the vertices reached and the sum of
// their out-degrees (R16). A warp per 32 consecutive input ids, lane l owns
// vertex v0 + l. The lane reads its vertex's parent row (whole 32-byte sectors,
// 16 sources per pass) into registers; then for each source b the warp stores
// out[b][v0 .. v0+31] — lane l's register b — as one coalesced 128-byte row
// segment. No shared-memory transpose, no block barrier.
template <typename OffT, int KP>
__global__ void __launch_bounds__(256) k_ms_finish_reg(const int32_t* __restrict__ par,
                                                      const uint8_t* __restrict__ par8,
                                                      const int32_t* __restrict__ hidx,
                                                      const OffT* __restrict__ csc_off,
                                                      const int32_t* __restrict__ csc_in,
                                                      const unsigned long long* __restrict__ seen,
                                                      const int32_t* __restrict__ inv,
                                                      const int32_t* __restrict__ outdeg, int64_t n, int k,
                                                      int32_t* __restrict__ out,
                                                      unsigned long long* __restrict__ reached,
                                                      unsigned long long* __restrict__ edges, int par_all) {
  __shared__ unsigned long long r[64], d[64];
  __shared__ int32_t nbr[8][32][33];  // per warp and lane: a light row's in-neighbours in input ids
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64; i += blockDim.x) r[i] = d[i] = 0;
  __syncthreads();
  unsigned long long r0 = 0, r1 = 0, d0 = 0, d1 = 0;
  int32_t* my = nbr[wp][lane];
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t * 32 < n; t += nw) {
    const int64_t v = t * 32 + lane;
    const bool in = v < n;
    const int32_t w = in ? (inv ? __ldg(&inv[v]) : (int32_t)v) : 0;
    const unsigned long long sv = in ? seen[w] : 0ull;
    const unsigned long long ov = in ? (unsigned long long)__ldg(&outdeg[w]) : 0ull;
    const int32_t h = sv ? (par_all ? w : __ldg(&hidx[w])) : -1;
    const bool light = sv && h < 0;
    uint4 p8[4] = {};
    if (light) {  // byte row (parent = an in-edge index) and the row's in-neighbours' input ids
      const uint4* r8 = reinterpret_cast<const uint4*>(par8 + (int64_t)w * 64);
#pragma unroll
      for (int j = 0; j < 4; ++j) p8[j] = __ldg(&r8[j]);
      const int64_t e0 = (int64_t)csc_off[w];
      const int deg = (int)((int64_t)csc_off[w + 1] - e0);
      for (int j0 = 0; j0 < deg; j0 += 8) {  // csc_in: the CSC's sources already in input ids
        int32_t u[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) u[j] = j0 + j < deg ? __ldg(&csc_in[e0 + j0 + j]) : 0;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j0 + j < deg) my[j0 + j] = u[j];
      }
    }
    const int4* row = reinterpret_cast<const int4*>(par + (int64_t)(h < 0 ? 0 : h) * KP);
    const uint32_t* b8 = reinterpret_cast<const uint32_t*>(p8);
#pragma unroll
    for (int b0 = 0; b0 < KP; b0 += 16) {
      if (b0 >= k) break;
      int32_t x[16];
      if (light) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint32_t byte = (b8[(b0 + j) >> 2] >> (8 * ((b0 + j) & 3))) & 0xFFu;
          x[j] = byte == 0xFFu ? (int32_t)v : my[byte & 31u];
        }
      } else {
        int4 q[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)  // unreached vertices' rows are never read
          q[j] = sv ? __ldg(&row[b0 / 4 + j]) : make_int4(-1, -1, -1, -1);
        const int32_t y[16] = {q[0].x, q[0].y, q[0].z, q[0].w, q[1].x, q[1].y, q[1].z, q[1].w,
                               q[2].x, q[2].y, q[2].z, q[2].w, q[3].x, q[3].y, q[3].z, q[3].w};
#pragma unroll
        for (int j = 0; j < 16; ++j) x[j] = y[j];
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int b = b0 + j;
        if (b < k && in) out[(int64_t)b * n + v] = (sv >> b) & 1ull ? x[j] : -1;
      }
    }
    if (__ballot_sync(0xffffffffu, sv != 0) == 0) continue;
    if (KP <= 32) {  // k <= 32: per source one vote and two warp sums (lane b keeps source b's counts)
#pragma unroll
      for (int b = 0; b < KP; ++b) {
        if (b >= k) break;
        const bool has = (sv >> b) & 1ull;
        const unsigned c = __popc(__ballot_sync(0xffffffffu, has));
        const unsigned hi = __reduce_add_sync(0xffffffffu, has ? (unsigned)(ov >> 16) : 0u);  // < 2^20 each
        const unsigned lo = __reduce_add_sync(0xffffffffu, has ? (unsigned)(ov & 0xFFFFu) : 0u);
        if (lane == b) {
          r0 += c;
          d0 += ((unsigned long long)hi << 16) + lo;
        }
      }
      continue;
    }
#pragma unroll 4
    for (int j = 0; j < 32; ++j) {
      const unsigned long long s = __shfl_sync(0xffffffffu, sv, j);
      const unsigned long long od = __shfl_sync(0xffffffffu, ov, j);
      const unsigned long long bb0 = (s >> lane) & 1ull, bb1 = (s >> (lane + 32)) & 1ull;
      r0 += bb0;
      r1 += bb1;
      d0 += bb0 * od;
      d1 += bb1 * od;
    }
  }
  if (r0) { atomicAdd(&r[lane], r0); atomicAdd(&d[lane], d0); }
  if (r1) { atomicAdd(&r[lane + 32], r1); atomicAdd(&d[lane + 32], d1); }
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    if (r[i]) atomicAdd(&reached[i], r[i]);
    if (d[i]) atomicAdd(&edges[i], d[i]);
  }
}

// The traversal state shared by the bit-parallel BFS and CC (cc.cu), allocated
// once per graph: masks, active lists, degree-prefix scratch and the heavy-row
// chunks of the CSC (rows of >= kHeavy in-edges cut into <= kHChunk pieces).
template <typename OffT>
static gi_status ms_prepare_t(gi_graph g) {
  auto& M = g->ms;
  cudaStream_t st = g->ctx->stream;
  const int sms = g->ctx->num_sms;
  const int64_t n = g->n;
  if (!M.seen.p) {
    GI_TRY(M.seen.alloc((n + 1) * 8));
    for (int c = 0; c < 2; ++c) {
      GI_TRY(M.fr[c].alloc((n + 1) * 8));
      GI_TRY(M.act[c].alloc((n + 1) * 4));
    }
    GI_TRY(M.cnt.alloc(8 * 8 + 2 * 64 * 8));
    GI_TRY(M.src.alloc(64 * 4));
    GI_TRY(M.heavy.alloc((n + 1) * 4));
    GI_TRY(M.chunks[0].alloc((n + 1) * 8));
    GI_TRY(M.chunks[1].alloc((n + 1) * 8));
    size_t tb = 0, tb64 = 0;
    GI_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, M.chunks[0].as<int32_t>(), M.chunks[1].as<int32_t>(), (int)n, st));
    GI_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb64, M.chunks[0].as<long long>(), M.chunks[1].as<long long>(),
                                          (int)n, st));
    size_t tbt = 0;  // the degree-prefix scan reads the active list through OutdegOf
    GI_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tbt,
                                          cub::TransformInputIterator<long long, OutdegOf, const int32_t*>(
                                              M.act[0].as<int32_t>(), OutdegOf{g->outdeg.as<int32_t>()}),
                                          M.chunks[1].as<long long>(), (int)n, st));
    tb = std::max(std::max(tb, tb64), tbt);
    GI_TRY(M.scan_tmp.alloc(tb + 16));
    M.scan_bytes = tb;
    GI_CUDA(cudaMemsetAsync(M.cnt.p, 0, 8, st));
    k_ms_heavy_list<OffT><<<grid_for(n, 256, sms), 256, 0, st>>>(g->csc_off.as<OffT>(), n, M.heavy.as<int32_t>(),
                                                                 M.cnt.as<unsigned long long>());
    int64_t hn = 0;
    GI_CUDA(cudaMemcpyAsync(&hn, M.cnt.p, 8, cudaMemcpyDeviceToHost, st));
    GI_CUDA(cudaStreamSynchronize(st));
    M.nheavy = hn;
    // heavy rows' compact index into the int32 parent rows; light rows (< kHeavy in-edges)
    // stage their parents as 1-byte in-edge indices
    GI_TRY(M.hidx.alloc((n + 1) * 4));
    GI_CUDA(cudaMemsetAsync(M.hidx.p, 0xFF, (n + 1) * 4, st));
    if (hn > 0) k_ms_hidx<<<grid_for(hn, 256, sms), 256, 0, st>>>(M.heavy.as<int32_t>(), hn, M.hidx.as<int32_t>());
    GI_TRY(M.par8.alloc((size_t)n * 64 + 64));
    M.nhch = 0;
    if (hn > 0) {
      int32_t* cc = M.chunks[0].as<int32_t>();
      int32_t* cp = M.chunks[1].as<int32_t>();
      k_ms_hchunk_count<OffT><<<grid_for(hn, 256, sms), 256, 0, st>>>(g->csc_off.as<OffT>(), M.heavy.as<int32_t>(), hn, cc);
      size_t tb2 = M.scan_bytes;
      GI_CUDA(cub::DeviceScan::InclusiveSum(M.scan_tmp.p, tb2, cc, cp, (int)hn, st));
      int32_t hc = 0;
      GI_CUDA(cudaMemcpyAsync(&hc, cp + hn - 1, 4, cudaMemcpyDeviceToHost, st));
      GI_CUDA(cudaStreamSynchronize(st));
      GI_TRY(M.hch.alloc((size_t)hc * 8));
      k_ms_hchunk_fill<<<grid_for(hn, 256, sms), 256, 0, st>>>(M.heavy.as<int32_t>(), hn, cc, cp, M.hch.as<int2>());
      M.nhch = hc;
    }
  }
  return GI_OK;
}

}  // namespace

gi_status ms_prepare(gi_graph g) { return g->off64 ? ms_prepare_t<int64_t>(g) : ms_prepare_t<int32_t>(g); }

namespace {

template <typename OffT>
gi_status msbfs_t(gi_graph g, int32_t k, const int32_t* sources, const gi_bfs_opts& o, int32_t* d_out,
                  gi_bfs_stats* stats) {
  gi_context ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  const int64_t n = g->n;
  auto& M = g->ms;
  GI_TRY(ms_prepare(g));
  int lkp = 3;  // par row: kp = 2^lkp >= k ints (whole 32-byte sectors, power-of-two tiles in the epilogue)
  while ((1 << lkp) < k) ++lkp;
  const int kp = 1 << lkp;
  // k <= 16: int32 parents for every row (64 bytes per row, like a byte row);
  // GI_MS_PAR_ALL=0 keeps byte rows for the light rows (A/B)
  static const bool par_all_env = !getenv("GI_MS_PAR_ALL") || atoi(getenv("GI_MS_PAR_ALL")) != 0;
  const bool par_all = par_all_env && kp <= 16;
  const int64_t par_rows = par_all ? n + 1 : M.nheavy + 1;
  if (!par_all && !M.csc_in.p) {  // byte rows: the CSC's sources in input ids (the epilogue resolves
                                  // light rows' parent indices through it), built on first need
    GI_TRY(M.csc_in.alloc((size_t)(g->ml + 1) * 4));
    k_ms_csc_in<<<grid_for(g->ml, 256, sms), 256, 0, st>>>(g->csc_idx.as<int32_t>(), g->ml,
                                                          g->relabeled ? g->perm.as<int32_t>() : nullptr,
                                                          M.csc_in.as<int32_t>());
  }
  if (M.par.bytes < (size_t)par_rows * kp * 4) GI_TRY(M.par.alloc((size_t)par_rows * kp * 4));
  if (k <= 32 && M.fc.bytes < (size_t)(n + 1) * (k <= 16 ? 2 : 4)) GI_TRY(M.fc.alloc((size_t)(n + 1) * (k <= 16 ? 2 : 4)));
  cudaEvent_t e0 = nullptr, e1 = nullptr, pe0 = nullptr, pe1 = nullptr;
  int64_t pull_examined = 0;
  float pull_ms = 0.f;
  if (o.profile) {
    GI_CUDA(cudaEventCreate(&e0));
    GI_CUDA(cudaEventCreate(&e1));
    GI_CUDA(cudaEventCreate(&pe0));
    GI_CUDA(cudaEventCreate(&pe1));
    GI_CUDA(cudaEventRecord(e0, st));
  }
  unsigned long long* cnt = M.cnt.as<unsigned long long>();
  int64_t* h = ctx->h_scratch;
  // R21's m/8, or m/12 when the push's random atomics on seen / fr_next (16 bytes
  // per vertex) miss L2: config 5 45 ms at m/12 against 49 at m/8, config 4 neutral,
  // config 2 (in L2) 2.44 ms at m/8 against 2.86 at m/12
  int l2 = 0;
  if (cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ctx->device) != cudaSuccess) l2 = 0;
  const int div_auto = (double)n * 16.0 > (double)l2 ? kMsPullDivBig : kMsPullDiv;
  const int64_t mdiv = g->m / (o.threshold_div > 0 ? o.threshold_div : div_auto);
  std::vector<int32_t> levels(k, 1);
  int64_t examined = 0;
  int launches = 0;
  GI_CUDA(cudaMemsetAsync(M.seen.p, 0, n * 8, st));
  GI_CUDA(cudaMemsetAsync(M.fr[0].p, 0, n * 8, st));
  GI_CUDA(cudaMemsetAsync(cnt, 0, 8 * 8 + 2 * 64 * 8, st));
  GI_CUDA(cudaMemcpyAsync(M.src.p, sources, k * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  k_ms_init<<<1, 64, 0, st>>>(M.src.as<int32_t>(), k, g->relabeled ? g->inv.as<int32_t>() : nullptr, n,
                              g->outdeg.as<int32_t>(), M.seen.as<unsigned long long>(), M.fr[0].as<unsigned long long>(),
                              M.act[0].as<int32_t>(), cnt, M.par.as<int32_t>(), kp, M.par8.as<uint8_t>(),
                              M.hidx.as<int32_t>(), par_all ? 1 : 0);
  launches += 1;
  GI_CUDA(cudaMemcpyAsync(h, cnt, 4 * 8, cudaMemcpyDeviceToHost, st));
  GI_CUDA(stream_wait(st));
  int64_t nact = h[0], sdeg = h[1];
  int pulls = 0;
  MsArgs A{};
  A.n = n;
  A.csr_off = g->csr_off.p;
  A.csr_idx = g->csr_idx.as<int32_t>();
  A.csc_off = g->csc_off.p;
  A.csc_idx = g->csc_idx.as<int32_t>();
  A.outdeg = g->outdeg.as<int32_t>();
  A.perm = g->relabeled ? g->perm.as<int32_t>() : nullptr;
  A.inv = g->relabeled ? g->inv.as<int32_t>() : nullptr;
  A.seen = M.seen.as<unsigned long long>();
  A.cnt = cnt;
  A.par = M.par.as<int32_t>();
  A.par8 = M.par8.as<uint8_t>();
  A.hidx = M.hidx.as<int32_t>();
  A.kp = kp;
  A.par_all = par_all ? 1 : 0;
  A.all = k == 64 ? ~0ull : ((1ull << k) - 1ull);
  // segmented OR pull (one GPU, a graph with the segmented layout; k > 32: two OR passes):
  // AUTO takes it for a pull level while the rows still missing sources hold more
  // than segor_frac x m in-edges; GI_MS_PULL_SEGMENTED takes it for every pull
  // level, building the layout if needed
  static const char* frac_env = getenv("GI_MS_SEGOR_FRAC");
  const double segor_frac = frac_env ? atof(frac_env) : k <= 16 ? kSegOrFrac16 : kSegOrFrac32;  // k > 32 as k <= 32
  const bool segor_ok = o.pull_kernel != GI_MS_PULL_ROWS && ctx->nranks == 1 && g->ml > 0;
  bool segor_ready = segor_ok && g->seg_Z != 0;
  if (segor_ok && !segor_ready && o.pull_kernel == GI_MS_PULL_SEGMENTED) {
    GI_TRY(seg_build(g, 0, 0));
    segor_ready = true;
  }
  if (segor_ready) {
    if (M.fc32.bytes < (size_t)(n + 16) * 4) GI_TRY(M.fc32.alloc((size_t)(n + 16) * 4));
    if (M.acc32.bytes < (size_t)(n + 16) * 4) GI_TRY(M.acc32.alloc((size_t)(n + 16) * 4));
    if (M.rlist.bytes < (size_t)(n + 1) * 4) GI_TRY(M.rlist.alloc((size_t)(n + 1) * 4));
    if (k > 32) {  // the upper halves: a second 32-bit OR pass
      if (M.fc32hi.bytes < (size_t)(n + 16) * 4) GI_TRY(M.fc32hi.alloc((size_t)(n + 16) * 4));
      if (M.acc32hi.bytes < (size_t)(n + 16) * 4) GI_TRY(M.acc32hi.alloc((size_t)(n + 16) * 4));
    }
  }
  int64_t inc = g->ml;  // in-edges of the rows still missing a source
  int segor_levels = 0, sparse_levels = 0;
  static const double sparse_frac = getenv("GI_MS_SPARSE_FRAC") ? atof(getenv("GI_MS_SPARSE_FRAC")) : kSparseFrac;
  static const char* dbg = getenv("GI_DEBUG_MSBFS");  // diagnostics: per-level direction, size, time
  FILE* df = dbg ? fopen(dbg, "a") : nullptr;
  for (int level = 0; nact > 0; ++level) {
    const auto tl0 = df ? std::chrono::steady_clock::now() : std::chrono::steady_clock::time_point{};
    const int c = level & 1;
    A.fcur = M.fr[c].as<unsigned long long>();
    A.fnext = M.fr[c ^ 1].as<unsigned long long>();
    A.acur = M.act[c].as<int32_t>();
    A.anext = M.act[c ^ 1].as<int32_t>();
    A.nact = nact;
    GI_CUDA(cudaMemsetAsync(cnt, 0, 6 * 8, st));
    // R21, plus: a listed-row pull (the rows still missing a source hold < m/64
    // in-edges) replaces a push whose frontier's out-edges outweigh the listing
    // (a pass over the n rows) and the listed in-edges: config 5's fifth level,
    // 214 M out-edges against 0.34 M listed in-edges, 4.3 ms as a push
    const bool sparse_pull = o.pull_kernel != GI_MS_PULL_ROWS && level > 0 &&
                             (double)inc < sparse_frac * (double)g->ml && sdeg > n / 2 + 2 * inc;
    const bool pull = o.policy == GI_BFS_PULL_ONLY ? level > 0
                                                   : (o.policy == GI_BFS_AUTO && (nact + sdeg > mdiv || sparse_pull));
    const bool segor = pull && segor_ready &&
                       (o.pull_kernel == GI_MS_PULL_SEGMENTED || (double)inc > segor_frac * (double)g->ml);
    bool sparse_used = false;
    if (pull && o.profile) GI_CUDA(cudaEventRecord(pe0, st));
    if (segor) {
      const bool f16 = k <= 16, wide = k > 32;
      k_ms_narrow_or<<<grid_for(n, 256, sms, 8), 256, 0, st>>>(A.fcur, n, M.fc32.as<uint32_t>(),
                                                              f16 ? M.fc.as<uint16_t>() : nullptr,
                                                              wide ? M.fc32hi.as<uint32_t>() : nullptr);
      GI_CUDA(cudaMemsetAsync(M.acc32.p, 0, (size_t)(n + 1) * 4, st));
      GI_TRY(seg_or_pass(g, M.fc32.as<uint32_t>(), M.acc32.as<uint32_t>()));
      A.acc32 = M.acc32.as<uint32_t>();
      A.acc32hi = nullptr;
      if (wide) {
        GI_CUDA(cudaMemsetAsync(M.acc32hi.p, 0, (size_t)(n + 1) * 4, st));
        GI_TRY(seg_or_pass(g, M.fc32hi.as<uint32_t>(), M.acc32hi.as<uint32_t>()));
        A.acc32hi = M.acc32hi.as<uint32_t>();
        launches += 1;
      }
      A.rlist = M.rlist.as<int32_t>();
      const int lg = grid_for(n, kMsT, sms, kLightPerSM);
      const unsigned rg = (unsigned)(sms * 8);
      if (f16) {
        A.fc = M.fc.p;
        k_ms_or_vertex<OffT, uint16_t><<<lg, kMsT, 0, st>>>(A);
        k_ms_resolve_heavy<OffT, uint16_t><<<rg, kMsT, 0, st>>>(A);
      } else if (wide) {  // parent scans gather the 64-bit masks
        A.fc = A.fcur;
        k_ms_or_vertex<OffT, unsigned long long><<<lg, kMsT, 0, st>>>(A);
        k_ms_resolve_heavy<OffT, unsigned long long><<<rg, kMsT, 0, st>>>(A);
      } else {
        A.fc = M.fc32.p;
        k_ms_or_vertex<OffT, uint32_t><<<lg, kMsT, 0, st>>>(A);
        k_ms_resolve_heavy<OffT, uint32_t><<<rg, kMsT, 0, st>>>(A);
      }
      launches += 4;
      if (o.profile) GI_CUDA(cudaEventRecord(pe1, st));
      ++pulls;
      ++segor_levels;
    } else if (pull) {
      const int fw = k <= 16 ? 2 : k <= 32 ? 4 : 8;  // bytes per gathered frontier mask
      // sparse level: only the rows still missing a source (listed; fnext zeroed)
      const bool sparse = o.pull_kernel != GI_MS_PULL_ROWS && level > 0 && (double)inc < sparse_frac * (double)g->ml;
      int64_t nlight = n, nchunks = M.nhch;
      const int2* chunks = M.hch.as<int2>();
      if (sparse) {
        if (M.rlist.bytes < (size_t)(n + 1) * 4) GI_TRY(M.rlist.alloc((size_t)(n + 1) * 4));
        if (M.hlist.bytes < (size_t)(M.nhch + 1) * 8) GI_TRY(M.hlist.alloc((size_t)(M.nhch + 1) * 8));
        GI_CUDA(cudaMemsetAsync(A.fnext, 0, n * 8, st));
        GI_CUDA(cudaMemsetAsync(cnt + 6, 0, 2 * 8, st));
        k_ms_list_light<OffT><<<grid_for(n, 256, sms, 8), 256, 0, st>>>(g->csc_off.as<OffT>(), A.seen, n, A.all,
                                                                        M.rlist.as<int32_t>(), cnt + 6);
        if (M.nhch > 0)
          k_ms_list_chunks<<<grid_for(M.nhch, 256, sms, 8), 256, 0, st>>>(M.hch.as<int2>(), M.nhch, A.seen, A.all,
                                                                         M.hlist.as<int2>(), cnt + 7);
        GI_CUDA(cudaMemcpyAsync(h + 6, cnt + 6, 2 * 8, cudaMemcpyDeviceToHost, st));
        GI_CUDA(stream_wait(st));
        nlight = h[6];
        nchunks = h[7];
        chunks = M.hlist.as<int2>();
        A.rlist = M.rlist.as<int32_t>();
        A.nlist = nlight;
        launches += 2;
        ++sparse_levels;
        sparse_used = true;
      }
      const int lg = grid_for(std::max<int64_t>(nlight, 1), kMsT, sms, kLightPerSM);
      const int64_t hw = (nchunks + kHeavyPer - 1) / kHeavyPer;
      const unsigned hg = (unsigned)std::max<int64_t>(1, (hw + kMsT / 32 - 1) / (kMsT / 32));
      // a few chunks per warp and many CTAs: the block scheduler balances the uneven chunks
      if (fw == 8) {
        A.fc = A.fcur;
        if (sparse) { if (nlight > 0) k_ms_pull<OffT, unsigned long long, true><<<lg, kMsT, 0, st>>>(A); }
        else k_ms_pull<OffT, unsigned long long><<<lg, kMsT, 0, st>>>(A);
        if (nchunks > 0) k_ms_pull_heavy<OffT, unsigned long long><<<hg, kMsT, 0, st>>>(A, chunks, nchunks);
      } else if (fw == 4) {
        k_ms_narrow<uint32_t><<<grid_for(n, 256, sms, 8), 256, 0, st>>>(A.fcur, n, M.fc.as<uint32_t>());
        A.fc = M.fc.p;
        if (sparse) { if (nlight > 0) k_ms_pull<OffT, uint32_t, true><<<lg, kMsT, 0, st>>>(A); }
        else k_ms_pull<OffT, uint32_t><<<lg, kMsT, 0, st>>>(A);
        if (nchunks > 0) k_ms_pull_heavy<OffT, uint32_t><<<hg, kMsT, 0, st>>>(A, chunks, nchunks);
        ++launches;
      } else {
        k_ms_narrow<uint16_t><<<grid_for(n, 256, sms, 8), 256, 0, st>>>(A.fcur, n, M.fc.as<uint16_t>());
        A.fc = M.fc.p;
        if (sparse) { if (nlight > 0) k_ms_pull<OffT, uint16_t, true><<<lg, kMsT, 0, st>>>(A); }
        else k_ms_pull<OffT, uint16_t><<<lg, kMsT, 0, st>>>(A);
        if (nchunks > 0) k_ms_pull_heavy<OffT, uint16_t><<<hg, kMsT, 0, st>>>(A, chunks, nchunks);
        ++launches;
      }
      if (nchunks > 0) ++launches;
      if (o.profile) GI_CUDA(cudaEventRecord(pe1, st));
      ++pulls;
    } else {
      GI_CUDA(cudaMemsetAsync(A.fnext, 0, n * 8, st));
      long long* dp = M.chunks[1].as<long long>();

      const int64_t nt = (nact + kScanTile - 1) / kScanTile;
      if (M.tsum.bytes < (size_t)(nt + 1) * 8) GI_TRY(M.tsum.alloc((size_t)(nt + 1) * 8));
      long long* ts = M.tsum.as<long long>();
      k_deg_tile_sums<<<(unsigned)nt, kScanT, 0, st>>>(A.acur, A.outdeg, nact, ts);
      k_scan_tile_sums<<<1, 1024, 0, st>>>(ts, nt);
      k_deg_scan<<<(unsigned)nt, kScanT, 0, st>>>(A.acur, A.outdeg, nact, ts, dp);
      launches += 3;
      k_ms_push<OffT><<<grid_for((sdeg + kPushChunk - 1) / kPushChunk * 32, kMsT, sms, 8), kMsT, 0, st>>>(A, dp);
    }
    GI_CUDA(cudaGetLastError());
    ++launches;
    GI_CUDA(cudaMemcpyAsync(h, cnt, 6 * 8, cudaMemcpyDeviceToHost, st));
    GI_CUDA(stream_wait(st));
    if (segor) h[3] += g->ml;  // the OR pass reads every in-edge (+ the parent scans)
    if (df)
      fprintf(df, "level=%d %s nact=%lld sdeg=%lld inc=%lld -> next=%lld examined=%lld us=%.1f\n", level,
              segor ? "pull-or" : sparse_used ? "pull-sparse" : pull ? "pull" : "push", (long long)nact, (long long)sdeg, (long long)inc,
              (long long)h[0], (long long)h[3],
              std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tl0).count());
    nact = h[0];
    sdeg = h[1];
    inc -= h[4];
    examined += h[3];
    if (pull) {
      pull_examined += h[3];
      if (o.profile) {
        float pm = 0.f;
        GI_CUDA(cudaEventElapsedTime(&pm, pe0, pe1));
        pull_ms += pm;
      }
    }
    for (int i = 0; i < k; ++i)
      if ((h[2] >> i) & 1) levels[i] = level + 2;  // source i still found vertices at this level
  }
  if (df) fclose(df);
  unsigned long long* hr = cnt + 8;
  GI_CUDA(cudaMemsetAsync(hr, 0, 2 * 64 * 8, st));
  {  // epilogue: the k output rows + per-source counts (R16)
    auto* fk = kp == 8 ? k_ms_finish_reg<OffT, 8> : kp == 16 ? k_ms_finish_reg<OffT, 16>
             : kp == 32 ? k_ms_finish_reg<OffT, 32> : k_ms_finish_reg<OffT, 64>;
    fk<<<grid_for(n, 256, sms, 8), 256, 0, st>>>(
        M.par.as<int32_t>(), M.par8.as<uint8_t>(), M.hidx.as<int32_t>(), g->csc_off.as<OffT>(),
        M.csc_in.as<int32_t>(), M.seen.as<unsigned long long>(),
        A.inv, g->outdeg.as<int32_t>(), n, k, d_out, hr, hr + 64, A.par_all);
  }
  ++launches;
  std::vector<unsigned long long> hs(128);
  GI_CUDA(cudaMemcpyAsync(hs.data(), hr, 128 * 8, cudaMemcpyDeviceToHost, st));
  float ms = 0.f;
  if (o.profile) GI_CUDA(cudaEventRecord(e1, st));
  GI_CUDA(stream_wait(st));
  if (o.profile) {
    GI_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(pe0);
    cudaEventDestroy(pe1);
  }
  if (stats)
    for (int i = 0; i < k; ++i) {
      gi_bfs_stats s{};
      s.levels = levels[i];
      s.pull_levels = pulls;
      s.reached = (int64_t)hs[i];
      s.edges_traversed = (int64_t)hs[64 + i];
      s.edges_examined = examined / k;  // shared by the k sources of the pass
      s.pull_vertices = (int64_t)pulls * n / k;
      s.total_ms = ms / (float)k;
      s.pull_ms = pull_ms / (float)k;
      s.pull_edges_examined = pull_examined / k;
      s.pull_or_levels = segor_levels;
      s.pull_sparse_levels = sparse_levels;
      s.launches = i == 0 ? launches : 0;
      stats[i] = s;
    }
  return GI_OK;
}

}  // namespace

// up to 64 sources per pass; longer batches run in passes of 64
gi_status msbfs_run(gi_graph g, int32_t k, const int32_t* sources, const gi_bfs_opts& o, int32_t* d_out,
                    gi_bfs_stats* stats) {
  for (int32_t i0 = 0; i0 < k; i0 += 64) {
    const int32_t kk = std::min<int32_t>(64, k - i0);
    gi_status s = g->off64 ? msbfs_t<int64_t>(g, kk, sources + i0, o, d_out + (int64_t)i0 * g->n, stats ? stats + i0 : nullptr)
                           : msbfs_t<int32_t>(g, kk, sources + i0, o, d_out + (int64_t)i0 * g->n, stats ? stats + i0 : nullptr);
    if (s != GI_OK) return s;
  }
  return GI_OK;
}

}  // namespace gi
