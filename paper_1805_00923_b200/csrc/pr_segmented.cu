// pr_segmented.cu — pull PageRank over shared-memory source segments.
//
// The paper's cache optimisation ("Segmented Subgraphs", PAPER.md P:741-757,
// partition the source range so each segment's
// random reads hit cache, then merge the per-segment partial sums) retargeted
// at the B200's 227 KB of shared memory per CTA. Measured on this part
// (tools/microbench/, profiles/): random 4-byte gathers run at ~1.0 per
// SM-clock from L2 but ~7 per SM-clock from shared memory, so the pull edge
// pass (a4) gathers contrib from a staged segment instead of from L2. A
// segment holds Z <= 65535 sources, so in-segment source ids are 16-bit and
// the index stream is 2 bytes per edge.
//
// Layout (built once per graph):
//   unit u  = (destination block b, source segment s), u = b*S + s: the edges
//             (v, w) with v in rows [b*DB, (b+1)*DB) and w in sources
//             [s*Z, (s+1)*Z). One block (DB = all rows) unless the per-row
//             accumulator would not fit in L2.
//   piece   = (unit, destination) run: the partial sum the paper's segmented
//             subgraphs merge ("SSG" partials).
//   record  = kRecBytes: a 16-byte header {type, L, groups} and one of
//     long  (type 1): 512 edge slots of pieces with >= kLongPiece edges, each
//           piece padded to whole 16-slot lanes (so a lane never holds two
//           pieces): uint16 idx[512] | int32 dst[33] | uint32 mask.
//           mask bit l: lane l starts a piece; dst[0]: the piece holding lane
//           0, dst[q]: the q-th piece starting at lanes 1..31.
//     short (type 2): pieces of exactly L < kLongPiece edges, 32 per group
//           (one lane each), R_L groups: per group uint16 idx[L][32] |
//           int32 dst[32]. Unused lanes read the zero slot and add into a
//           trash row.
//   A unit's records are its long records, then its short records by L.
// Per iteration:
//   k_pr_seg  persistent, one CTA per SM over a cost-balanced range of
//             records. A producer warp streams records into a kStages-deep
//             shared-memory ring with bulk copies (TMA); the unit's contrib
//             segment is staged with one more bulk copy. Each of kConsumers
//             warps takes one record per stage: long: every lane sums its 16
//             gathers, a warp segmented scan over lanes (resets from the
//             mask) leaves each piece's sum in its last lane; short: every
//             lane sums its piece's L gathers. The sums go into acc[v] with
//             red.global.add.f32 — acc (4 B per row of the block) stays in
//             L2, so no partials reach HBM and no merge pass is needed.
//   k_pr_acc  r'[v] = (1-d)/n + d (acc[v] + D/n), contrib', dangling mass
//             (fused vertex update a3); zeroes the other (ping-pong) accumulator.
#include <algorithm>
#include <climits>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cub/cub.cuh>
#include <memory>
#include <string>
#include <vector>

#include "gi_internal.cuh"
#include "pr_common.cuh"

namespace gi {
namespace {

#ifndef GI_SEG_CONSUMERS
#define GI_SEG_CONSUMERS 30
#endif
#ifndef GI_SEG_STAGES
#define GI_SEG_STAGES 2
#endif
constexpr int kConsumers = GI_SEG_CONSUMERS;        // consumer warps (one record each per stage)
constexpr int kSegThreads = 32 * (kConsumers + 1);  // + one producer warp (TMA)
constexpr int kLaneE = 16;                          // edge slots per lane (long records)
constexpr int kChunkE = 32 * kLaneE;                // edge slots per long record
constexpr int kLongPiece = 16;                      // pieces of >= 16 edges go to long records
constexpr int kADst = 33;
constexpr int kRecHdr = 16;
constexpr int kRecPayload = 1168;
constexpr int kRecBytes = kRecHdr + kRecPayload;    // 1184, a multiple of the 16-byte bulk-copy granule
constexpr int kLDst = kRecHdr + 2 * kChunkE;        // long: dst[33]
constexpr int kLMask = kLDst + 4 * kADst;           // long: mask
static_assert(kLMask + 4 <= kRecBytes, "long record overflows");
// short groups: wide (type 2: int32 destination per lane) or compact (type 3: a
// 16-bit offset per lane from an int32 group base, 0xFFFF = the trash row),
// used when the group's 32 destinations (sorted) span < 65535 rows
__host__ __device__ constexpr int short_group_bytes(int L, bool compact = false) {
  return compact ? 64 * L + 80 : 64 * L + 128;
}
__host__ __device__ constexpr int short_groups(int L, bool compact = false) {
  return kRecPayload / short_group_bytes(L, compact);
}
constexpr int kStages = GI_SEG_STAGES;              // ring depth (stages in flight per CTA)
constexpr int kStageBytes = kConsumers * kRecBytes;
// CTA balance: an initial cost model (in gather slots), then refined from
// measured per-CTA times over the first kCalibPasses edge passes (seg_rebalance)
constexpr int kPieceCost = 4;
#ifndef GI_ACC_LDCS
#define GI_ACC_LDCS 1
#endif
#ifndef GI_SEG_RED_EVICT_LAST
#define GI_SEG_RED_EVICT_LAST 1  // config 4: 1.67-1.68 vs 1.70 ms per iteration
#endif
#ifndef GI_SEG_EVICT_FIRST
#define GI_SEG_EVICT_FIRST 1  // the record stream carries an L2 evict_first hint (keeps acc and contrib in L2)
#endif
#ifndef GI_ACC_PER_SM
#define GI_ACC_PER_SM 4  // vertex-pass CTAs per SM
#endif
#ifndef GI_SEG_DIRECT
#define GI_SEG_DIRECT 16
#endif
constexpr int kDirectRecs = GI_SEG_DIRECT;  // units with fewer records gather from global memory (no staging)
constexpr int kDirectCost = 5;              // cost factor of a record of such a unit (L2 vs shared-memory gathers)
constexpr int64_t kUnitCost = 40 * kChunkE;         // a unit start: segment staging + pipeline refill
constexpr int64_t kDefaultBlockRows = 16 << 20;     // 64 MB accumulator per destination block (8 M: config 4 1.89-1.95 ms, 16-32 M: 1.78)
constexpr int64_t kBlockEdges = (1ll << 31) - (1ll << 20);  // and fewer edges than the build's 32-bit sorts take
#ifndef GI_SEG_CALIB
#define GI_SEG_CALIB 8
#endif
#ifndef GI_SEG_DAMP
#define GI_SEG_DAMP 1.0  // fraction of the way each re-balance moves a boundary
#endif
constexpr int kCalibPasses = GI_SEG_CALIB;
#ifndef GI_ACC_UNROLL
#define GI_ACC_UNROLL 2  // config 4 vertex pass 0.113 -> 0.109 ms (1: one quad per step; 4: 0.119)
#endif
constexpr int kAccUnroll = GI_ACC_UNROLL;  // vertex pass: quads in flight per thread


struct SegArgs {
  const uint8_t* __restrict__ rec;     // kRecBytes per record
  const int32_t* __restrict__ unit_c0; // U + 1: first record of each unit
  const int32_t* __restrict__ cta_c0;  // grid + 1: first record of each CTA
  const int32_t* __restrict__ cta_u;   // grid: unit of each CTA's first record
  const float* __restrict__ cin;       // contrib, global ids, padded by >= 16 floats
  float* __restrict__ acc;             // per local row (+ trash row at nr)
  int64_t n;
  int Z, S, U;
  unsigned long long* timing;  // per CTA [start, end, staging ns, units] (balance calibration, diagnostics)
  unsigned long long* ht;      // per CTA {tail << 32 | head}: its remaining record range (work stealing)
  int trash;                   // accumulator row of padding lanes (the owned rows' count)
  int steal;                   // 1: CTAs that finish their range steal half of the largest remaining one
};

// programmatic dependent launch (the edge and vertex passes of consecutive
// iterations are launched with cudaLaunchAttributeProgrammaticStreamSerialization):
// a kernel lets its successor be scheduled as soon as all its CTAs run, and
// waits for its predecessor's completion and memory before touching its data
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// 1-D TMA bulk copy global -> shared, completion counted on `bar` (UBLKCP in SASS)
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// the same bulk copy with an L2 eviction-priority hint (the streamed records
// are read once per pass: evict_first keeps the accumulator and contrib in L2)
__device__ __forceinline__ void tma_load_1d_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                                 uint64_t policy) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// The reduction a pass folds over a destination's in-edges: PageRank's sum of
// fp32 contributions (RED.ADD.F32), or connected components' min of int32
// labels (RED.MIN.S32) — the same records, gathers and piece structure.
struct OpSum {
  using T = float;
  static __device__ __forceinline__ T id() { return 0.f; }
  static __device__ __forceinline__ T op(T a, T b) { return a + b; }
  static __device__ __forceinline__ void red(T* p, T v) {
#if GI_SEG_RED_EVICT_LAST  // keep the accumulator's lines in L2 past the streamed records
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("red.global.add.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
#else
    atomicAdd(p, v);
#endif
  }
};
struct OpMin {
  using T = int32_t;
  static __device__ __forceinline__ T id() { return INT_MAX; }
  static __device__ __forceinline__ T op(T a, T b) { return min(a, b); }
  static __device__ __forceinline__ void red(T* p, T v) { atomicMin(p, v); }
};
// the bit-parallel BFS's dense pull levels (msbfs.cu): the OR of the in-neighbours'
// 32-bit frontier masks (RED.OR.B32)
struct OpOr {
  using T = uint32_t;
  static __device__ __forceinline__ T id() { return 0u; }
  static __device__ __forceinline__ T op(T a, T b) { return a | b; }
  static __device__ __forceinline__ void red(T* p, T v) {
    if (v) atomicOr(p, v);  // a piece that brings no frontier bit needs no atomic
  }
};

// a value of the unit's segment: from the staged copy in shared memory, or (G:
// a sparse unit, not staged) straight from global memory; offset Z is the
// identity slot that padding slots point at
template <bool G, class OP>
__device__ __forceinline__ typename OP::T seg_val(const typename OP::T* sc, uint32_t o, uint32_t Z) {
  if (G) return o < Z ? __ldg(sc + o) : OP::id();
  return sc[o];
}

// Long record: every lane's 16 slots belong to one piece, so a lane sums its
// gathers; a warp segmented scan over lanes (reset where the mask marks a
// piece start) leaves each piece's sum in its last lane, which folds it into acc.
template <int MODE, bool G, class OP>
__device__ __forceinline__ void reduce_long(const SegArgs& A, const uint8_t* r, const typename OP::T* sc, int lane,
                                            uint64_t* empty) {
  using T = typename OP::T;
  const uint4 qa = *reinterpret_cast<const uint4*>(r + kRecHdr + 32 * lane);
  const uint4 qb = *reinterpret_cast<const uint4*>(r + kRecHdr + 32 * lane + 16);
  const uint32_t mask = *reinterpret_cast<const uint32_t*>(r + kLMask);
  const int q = __popc(mask & ((2u << lane) - 1u) & ~1u);
  const int dst = *reinterpret_cast<const int32_t*>(r + kLDst + 4 * q);
  __syncwarp();
  if (lane == 0) mbar_arrive(empty);  // the record may be overwritten now
  const uint32_t w[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
  T v[kLaneE];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (MODE == 3) {  // diagnostics: the same gathers made bank-conflict free (wrong sums)
      v[2 * j] = seg_val<G, OP>(sc, min(((w[j] & 0xFFFFu) & ~31u) | (uint32_t)lane, (uint32_t)A.Z), A.Z);
      v[2 * j + 1] = seg_val<G, OP>(sc, min(((w[j] >> 16) & ~31u) | (uint32_t)lane, (uint32_t)A.Z), A.Z);
    } else {
      v[2 * j] = seg_val<G, OP>(sc, w[j] & 0xFFFFu, A.Z);
      v[2 * j + 1] = seg_val<G, OP>(sc, w[j] >> 16, A.Z);
    }
  }
#pragma unroll
  for (int s = 1; s < kLaneE; s <<= 1)
#pragma unroll
    for (int k = 0; k < kLaneE; k += 2 * s) v[k] = OP::op(v[k], v[k + s]);
  T X = v[0];
  if (MODE == 1) {  // diagnostics: stream + gathers only
    if (X == (T)-1) A.acc[lane] += (float)X;
    return;
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, X, o);
    if (lane >= o && ((mask >> (lane - o + 1)) & ((1u << o) - 1u)) == 0u) X = OP::op(y, X);
  }
  const bool last = lane == 31 || ((mask >> (lane + 1)) & 1u);
  if (last) OP::red(reinterpret_cast<T*>(A.acc) + dst, X);  // RED.E.ADD.F32 / RED.E.MIN.S32
}

// Short record of pieces with exactly L edges: lane l of group g owns one
// piece: L gathers, one RED.
template <int MODE, bool G, class OP>
__device__ __forceinline__ void reduce_short(const SegArgs& A, const uint8_t* r, const typename OP::T* sc, int lane,
                                             uint64_t* empty) {
  using T = typename OP::T;
  const bool compact = *reinterpret_cast<const int32_t*>(r) == 3;
  const int L = *reinterpret_cast<const int32_t*>(r + 4);
  const int ng = *reinterpret_cast<const int32_t*>(r + 8);
  const int gb = short_group_bytes(L, compact);
  for (int g = 0; g < ng; ++g) {
    const uint8_t* b = r + kRecHdr + g * gb + 2 * lane;
    int d;
    if (compact) {
      const uint32_t off = *reinterpret_cast<const uint16_t*>(r + kRecHdr + g * gb + 64 * L + 2 * lane);
      d = off == 0xFFFFu ? A.trash : *reinterpret_cast<const int32_t*>(r + kRecHdr + g * gb + 64 * L + 64) + (int)off;
    } else {
      d = *reinterpret_cast<const int32_t*>(r + kRecHdr + g * gb + 64 * L + 4 * lane);
    }
    T s = OP::id();
#pragma unroll 4
    for (int k = 0; k < L; ++k) {
      uint32_t o = *reinterpret_cast<const uint16_t*>(b + 64 * k);
      if (MODE == 3) o = min((o & ~31u) | (uint32_t)lane, (uint32_t)A.Z);  // diagnostics: conflict-free
      s = OP::op(s, seg_val<G, OP>(sc, o, A.Z));
    }
    if (MODE == 1) {
      if (s == (T)-1) A.acc[lane] += (float)s;
    } else {
      OP::red(reinterpret_cast<T*>(A.acc) + d, s);  // RED.E.ADD.F32 / RED.E.MIN.S32
    }
  }
  __syncwarp();
  if (lane == 0) mbar_arrive(empty);
}

template <int MODE, bool G, class OP>
__device__ __forceinline__ void reduce_record(const SegArgs& A, const uint8_t* r, const typename OP::T* sc, int lane,
                                              uint64_t* empty) {
  const int type = *reinterpret_cast<const int32_t*>(r);
  if (MODE == 2) {  // diagnostics: record stream only
    __syncwarp();
    if (lane == 0) mbar_arrive(empty);
    if (type == 7) A.acc[lane] += 1.f;
    return;
  }
  if (type == 1) reduce_long<MODE, G, OP>(A, r, sc, lane, empty);
  else reduce_short<MODE, G, OP>(A, r, sc, lane, empty);
}

// Persistent CTA per SM over records [cta_c0[b], cta_c0[b+1]), unit by unit.
// Warp kConsumers is the producer: one lane claims records and streams them
// into a kStages-deep shared-memory ring with bulk copies (full[s]: bytes
// landed; empty[s]: every consumer warp has taken its record out of slot s),
// writing a descriptor per stage (first record, count, sparse-unit flag,
// restage flag). Consumer warp w reduces record w of every stage. A unit's
// contrib segment is staged with one more bulk copy once every consumer has
// left the previous segment (seg_free) and has been told by the descriptor to
// wait for the new one (seg_bar).
// Work stealing: a CTA's remaining range is one 64-bit word {tail, head}; the
// owner claims a stage by adding to head, and a CTA that has exhausted its range
// takes the upper half of the largest remaining range by lowering that range's
// tail (CAS on the same word: a concurrent claim makes it retry). Ranges stay
// contiguous, so records keep their RED and DRAM locality; the static cuts only
// set where CTAs start. MODE (GI_SEG_MODE diagnostics): 0 full, 1 no REDs,
// 2 record stream only.
constexpr int kMinSteal = 256;  // records: below this, a steal does not pay for its segment staging
constexpr int kClaim = 8 * kConsumers;  // records an owner claims from its range per atomic
constexpr int kStealMinPerCta = 8192;   // records per CTA from which stealing pays (configs 4/5, not 2)
template <int MODE, class OP>
__global__ void __launch_bounds__(kSegThreads, 1) k_pr_seg(SegArgs A) {
  using T = typename OP::T;
  extern __shared__ __align__(128) uint8_t smem[];  // [kStages][kStageBytes] ring | Z + 4 floats of segment
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages], seg_bar, seg_free;
  __shared__ int4 desc[kStages];  // first record, count (-1: end of work), sparse unit, restage
  __shared__ unsigned long long s_units;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint8_t* ring = smem;
  T* scontrib = reinterpret_cast<T*>(smem + kStages * kStageBytes);
  const int b = blockIdx.x;
  unsigned long long t_start = 0, n_units = 0;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers);
    }
    mbar_init(&seg_bar, 1);
    mbar_init(&seg_free, kConsumers);
  }
  pdl_launch_dependents();
  __syncthreads();
  pdl_wait();  // the previous vertex pass wrote cin and cleared acc
  if (A.timing && tid == 0) t_start = globaltimer();
  if (warp == kConsumers) {
    if (lane == 0) {  // producer
#if GI_SEG_EVICT_FIRST
      uint64_t rec_policy;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(rec_policy));
#endif
      const int c1 = __ldg(&A.cta_c0[b + 1]);
      int h = __ldg(&A.cta_c0[b]);  // next record to issue
      int ce = A.steal ? h : c1;    // end of the block of records claimed so far
      if (A.steal) atomicExch(&A.ht[b], ((unsigned long long)(uint32_t)c1 << 32) | (uint32_t)h);
      int u = __ldg(&A.cta_u[b]);  // unit of h
      uint32_t it = 0, nrestage = 0;
      int staged_seg = -1;
      int span_u = -1, span_ce = -1, uend = 0, ulast = 0;
      bool direct = false;
      auto wait_slot = [&](uint32_t i) {
        if (i >= kStages) mbar_wait(&empty[i % kStages], ((i / kStages) & 1u) ^ 1u);
      };
      for (;;) {
        if (h >= ce) {
          if (!A.steal) break;
          // claim the next block of kClaim records of the own range (one atomic per
          // kClaim / kConsumers stages); a thief may have lowered the tail meanwhile
          const unsigned long long old = atomicAdd(&A.ht[b], (unsigned long long)kClaim);
          const int oh = (int)(uint32_t)old, ot = (int)(old >> 32);
          if (oh < ot) {
            h = oh;
            ce = min(oh + kClaim, ot);
          } else {  // own range exhausted: steal the upper half of the largest remaining range
            bool got = false;
            for (int tries = 0; tries < 8 && !got; ++tries) {
              int vbest = -1, rbest = kMinSteal - 1;
              unsigned long long wbest = 0;
              for (int v = 0; v < (int)gridDim.x; ++v) {
                const unsigned long long w = *reinterpret_cast<volatile unsigned long long*>(&A.ht[v]);
                const int rem = (int)(w >> 32) - (int)(uint32_t)w;
                if (rem > rbest) {
                  rbest = rem;
                  vbest = v;
                  wbest = w;
                }
              }
              if (vbest < 0) break;
              const int vh = (int)(uint32_t)wbest, vt = (int)(wbest >> 32);
              const int nt = vh + (vt - vh) / 2;
              const unsigned long long nw = ((unsigned long long)(uint32_t)nt << 32) | (uint32_t)vh;
              if (atomicCAS(&A.ht[vbest], wbest, nw) == wbest) {  // [nt, vt) is ours now
                atomicExch(&A.ht[b], ((unsigned long long)(uint32_t)vt << 32) | (uint32_t)nt);
                h = ce = nt;  // the next pass claims from it
                int lo = 0, hi = A.U - 1;  // the unit of nt: last u with unit_c0[u] <= nt
                while (lo < hi) {
                  const int mid = (lo + hi + 1) >> 1;
                  if (__ldg(&A.unit_c0[mid]) <= nt) lo = mid;
                  else hi = mid - 1;
                }
                u = lo;
                got = true;
              }
            }
            if (!got) break;
          }
          continue;
        }
        // the span of the unit holding h (a run of consecutive sparse units is one span:
        // their records carry their segment), looked up once per unit (and after a steal)
        if (u != span_u || ce != span_ce) {
          span_u = u;
          span_ce = ce;
          uend = __ldg(&A.unit_c0[u + 1]);
          direct = uend - __ldg(&A.unit_c0[u]) < kDirectRecs;
          ulast = u;
          if (direct)
            while (uend < ce && ulast + 1 < A.U && __ldg(&A.unit_c0[ulast + 2]) - uend < kDirectRecs)
              uend = __ldg(&A.unit_c0[++ulast + 1]);
        }
        const int seg = u % A.S;
        const int cnt = min(kConsumers, min(uend, ce) - h);
        const bool restage = !direct && seg != staged_seg;
        wait_slot(it);
        const uint32_t sl = it % kStages;
        desc[sl] = make_int4(h, cnt, direct ? 1 : 0, restage ? 1 : 0);
#if GI_SEG_EVICT_FIRST
        tma_load_1d_hint(ring + sl * kStageBytes, A.rec + (int64_t)h * kRecBytes, (uint32_t)(cnt * kRecBytes),
                         &full[sl], rec_policy);
#else
        tma_load_1d(ring + sl * kStageBytes, A.rec + (int64_t)h * kRecBytes, (uint32_t)(cnt * kRecBytes), &full[sl]);
#endif
        ++it;
        if (restage) {  // every consumer has left the old segment (it reached this stage): load the new one
          mbar_wait(&seg_free, nrestage & 1u);
          ++nrestage;
          const int64_t base = (int64_t)seg * A.Z;
          const int64_t zlen = min((int64_t)A.Z, A.n - base);
          scontrib[A.Z] = OP::id();
          tma_load_1d(scontrib, A.cin + base, (uint32_t)(((zlen * 4) + 15) & ~15ll), &seg_bar);
          staged_seg = seg;
        }
        h += cnt;
        if (h >= uend) {
          u = ulast + 1;
          ++n_units;
        }
      }
      // end of work: one more descriptor, completed by a plain arrive
      wait_slot(it);
      const uint32_t sl = it % kStages;
      desc[sl] = make_int4(0, -1, 0, 0);
      s_units = n_units;
      mbar_arrive(&full[sl]);
    }
  } else {
    uint32_t it = 0, seg_phase = 0;
    for (;; ++it) {
      const uint32_t sl = it % kStages, ph = (it / kStages) & 1u;
      mbar_wait(&full[sl], ph);
      const int4 d = desc[sl];
      if (d.y < 0) break;
      if (d.w) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&seg_free);  // done with the previous segment
        mbar_wait(&seg_bar, seg_phase);
        seg_phase ^= 1u;
      }
      const uint8_t* r = ring + sl * kStageBytes + warp * kRecBytes;
      if (warp < d.y) {
        if (d.z)
          reduce_record<MODE, true, OP>(
              A, r, reinterpret_cast<const T*>(A.cin) + (int64_t)*reinterpret_cast<const int32_t*>(r + 12) * A.Z,
              lane, &empty[sl]);
        else reduce_record<MODE, false, OP>(A, r, scontrib, lane, &empty[sl]);
      } else if (lane == 0) {
        mbar_arrive(&empty[sl]);  // nothing to take from this slot
      }
    }
  }
  if (A.timing) {
    __syncthreads();
    if (tid == 0) {
      unsigned long long* Tm = A.timing + 4 * blockIdx.x;
      Tm[0] = t_start;
      Tm[1] = globaltimer();
      Tm[2] = 0;
      Tm[3] = s_units;
    }
  }
}

// Vertex update over local rows, 4 per thread (vector loads): s = acc[v],
// then pr_epilogue's arithmetic; zero[v] = 0 readies the other accumulator.
__global__ void __launch_bounds__(256) k_pr_acc(PrArgs A, const float* __restrict__ acc, float* __restrict__ zero) {
  __shared__ double sred[32];
  pdl_launch_dependents();
  pdl_wait();  // the edge pass's accumulator
  if (blockIdx.x == 0 && threadIdx.x == 0) A.dbuf[(A.it + 2) % 3] = 0.0;
  const double D = A.uniform ? A.dbuf[A.it % 3] : 0.0;
  const float dn = (float)(D * A.inv_n);
  double dpart = 0.0;
  const int64_t nq = A.n / 4;
  const float4* acc4 = reinterpret_cast<const float4*>(acc);
  const bool vec = (A.row0 & 3) == 0;
  auto update4 = [&](int64_t q, float4 s4, int4 od4) {
    reinterpret_cast<float4*>(zero)[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int64_t v0 = A.row0 + 4 * q;
    const float s[4] = {s4.x, s4.y, s4.z, s4.w};
    const int od[4] = {od4.x, od4.y, od4.z, od4.w};
    float c[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float rn = A.base + A.damp * (s[k] + dn);
      c[k] = od[k] > 0 ? rn / (float)od[k] : 0.f;
      if (od[k] == 0) dpart += (double)rn;
      if (A.rank_out) A.rank_out[A.perm ? __ldg(&A.perm[v0 + k]) : v0 + k] = rn;
    }
    *reinterpret_cast<float4*>(A.cout + v0) = make_float4(c[0], c[1], c[2], c[3]);
    for (int p = 0; p < A.npeer; ++p) *reinterpret_cast<float4*>(A.peer[p] + v0) = make_float4(c[0], c[1], c[2], c[3]);
  };
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // kAccUnroll quads per thread per step, all loads issued before the first store
  for (int64_t q0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q0 < (vec ? nq : 0); q0 += kAccUnroll * stride) {
    float4 s4[kAccUnroll];
    int4 od4[kAccUnroll];
#pragma unroll
    for (int j = 0; j < kAccUnroll; ++j) {
      const int64_t q = q0 + j * stride;
      if (q < nq) {
#if GI_ACC_LDCS
        s4[j] = __ldcs(acc4 + q);  // read once: evict-first, the zeroed buffer and contrib stay
#else
        s4[j] = acc4[q];
#endif
        od4[j] = __ldg(reinterpret_cast<const int4*>(A.outdeg + A.row0 + 4 * q));
      }
    }
#pragma unroll
    for (int j = 0; j < kAccUnroll; ++j)
      if (q0 + j * stride < nq) update4(q0 + j * stride, s4[j], od4[j]);
  }
  for (int64_t r = (vec ? 4 * nq : 0) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < A.n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const float s = acc[r];
    zero[r] = 0.f;
    pr_epilogue(A, r, s, dn, dpart);
  }
  if (A.npeer) __threadfence_system();  // peer stores ordered before the next collective
  const double bs = block_sum(dpart, sred);
  if (threadIdx.x == 0 && bs != 0.0) atomicAdd(&A.dbuf[(A.it + 1) % 3], bs);
}



// ---------------------------------------------------------------- layout build
// out[i] = a[ix[i]]
__global__ void k_gather_i64(const int64_t* __restrict__ a, const int64_t* __restrict__ ix, int64_t n,
                             int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a[ix[i]];
}

// row of every CSC edge (warp per row)
template <typename OffT>
// (rows [r0, r0 + n) of the CSC, whose edges start at e0: row[e - e0] = r0 + v)
__global__ void k_edge_rows(const OffT* __restrict__ off, int64_t n, int64_t e0, int64_t r0,
                            int32_t* __restrict__ row) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = w0; v < n; v += nw)
    for (int64_t e = (int64_t)off[v] + lane; e < (int64_t)off[v + 1]; e += 32) row[e - e0] = (int32_t)(r0 + v);
}

// unit key of every edge and its position (the sort payload)
template <typename OffT>
__global__ void k_unit_keys(const int32_t* __restrict__ idx, const int32_t* __restrict__ row, int64_t m, int Z, int S,
                            int64_t DB, uint32_t* __restrict__ key, OffT* __restrict__ eid) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    key[e] = (uint32_t)((row[e] / DB) * S + idx[e] / Z);
    eid[e] = (OffT)e;
  }
}

// piece heads over the sorted edges: a new (unit, destination) run
template <typename OffT>
__global__ void k_sorted_heads(const uint32_t* __restrict__ skey, const OffT* __restrict__ order,
                               const int32_t* __restrict__ row, int64_t m, int32_t* __restrict__ h) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    h[i] = i == 0 || skey[i] != skey[i - 1] || row[(int64_t)order[i]] != row[(int64_t)order[i - 1]];
}

// per piece p (pid = inclusive head count): first sorted edge, unit, destination
template <typename OffT>
__global__ void k_piece_info(const int32_t* __restrict__ h, const int32_t* __restrict__ pid,
                             const uint32_t* __restrict__ skey, const OffT* __restrict__ order,
                             const int32_t* __restrict__ row, int64_t m, int64_t* __restrict__ pstart,
                             int32_t* __restrict__ punit, int32_t* __restrict__ pdst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    if (h[i]) {
      const int32_t p = pid[i] - 1;
      pstart[p] = i;
      punit[p] = (int32_t)skey[i];
      pdst[p] = row[(int64_t)order[i]];
    }
}

// long pieces: slots padded to whole lanes (else 0); short pieces: class key
// u*16 + L (long: past every class), for the stable class sort
__global__ void k_piece_class(const int64_t* __restrict__ pstart, const int32_t* __restrict__ punit, int64_t P,
                              int64_t m, int64_t* __restrict__ asz, uint32_t* __restrict__ ckey,
                              int32_t* __restrict__ pids, uint32_t sentinel) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t len = (p + 1 < P ? pstart[p + 1] : m) - pstart[p];
    const bool lg = len >= kLongPiece;
    asz[p] = lg ? (len + kLaneE - 1) / kLaneE * kLaneE : 0;
    ckey[p] = lg ? sentinel : (uint32_t)punit[p] * 16u + (uint32_t)len;
    pids[p] = (int32_t)p;
  }
}

// lower bound of each value in a sorted array
template <typename K>
__global__ void k_lower_bounds(const K* __restrict__ a, int64_t n, int64_t nq, int64_t* __restrict__ out) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)a[mid] < q) lo = mid + 1;
      else hi = mid;
    }
    out[q] = lo;
  }
}

// long record of each long piece's first slot, and the edges' index slots
template <typename OffT>
__global__ void k_place_long(const int64_t* __restrict__ asz, const int64_t* __restrict__ aoff,
                             const int32_t* __restrict__ punit, const int64_t* __restrict__ unit_p0,
                             const int32_t* __restrict__ unit_c0, const int64_t* __restrict__ pstart,
                             const uint32_t* __restrict__ skey, const OffT* __restrict__ order,
                             const int32_t* __restrict__ idx, const int32_t* __restrict__ pdst, int64_t P, int64_t m,
                             int Z, int S, const int32_t* __restrict__ lpid, int64_t NL, uint8_t* __restrict__ rec) {
  // a warp per long piece (lpid: the long pieces' ids, the tail of the class
  // order), its lanes striding over the piece's edges (a hub's piece holds up to
  // ~10^5 edges: one thread per piece serialised the build on them)
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; q < NL; q += nw) {
    const int64_t p = __ldg(&lpid[q]);
    if (asz[p] == 0) continue;
    const int u = punit[p];
    const int64_t s0 = (int64_t)unit_c0[u] * kChunkE + (aoff[p] - aoff[unit_p0[u]]);  // slot in record units
    const int64_t len = (p + 1 < P ? pstart[p + 1] : m) - pstart[p];
    const int64_t base = (int64_t)(skey[pstart[p]] % (uint32_t)S) * Z;
    for (int64_t o = lane; o < len; o += 32) {
      const int64_t s = s0 + o;
      *reinterpret_cast<uint16_t*>(rec + (s / kChunkE) * kRecBytes + kRecHdr + 2 * (s % kChunkE)) =
          (uint16_t)(idx[(int64_t)order[pstart[p] + o]] - base);
    }
    if (lane == 0) {
      const int l0 = (int)((s0 % kChunkE) / kLaneE);
      atomicOr(reinterpret_cast<uint32_t*>(rec + (s0 / kChunkE) * kRecBytes + kLMask), 1u << l0);
    }
  }
}

// dst table of the long records (after every mask is complete)
__global__ void k_long_dst(const int64_t* __restrict__ asz, const int64_t* __restrict__ aoff,
                           const int32_t* __restrict__ punit, const int64_t* __restrict__ unit_p0,
                           const int32_t* __restrict__ unit_c0, const int32_t* __restrict__ pdst,
                           const int32_t* __restrict__ lpid, int64_t NL, uint8_t* __restrict__ rec) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < NL; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = __ldg(&lpid[q]);
    if (asz[p] == 0) continue;
    const int u = punit[p];
    const int64_t s0 = (int64_t)unit_c0[u] * kChunkE + (aoff[p] - aoff[unit_p0[u]]), s1 = s0 + asz[p];
    for (int64_t c = s0 / kChunkE; c * kChunkE < s1; ++c) {
      uint8_t* r = rec + c * kRecBytes;
      const int l = c * kChunkE >= s0 ? 0 : (int)((s0 % kChunkE) / kLaneE);
      const uint32_t mask = *reinterpret_cast<const uint32_t*>(r + kLMask);
      const int q = l == 0 ? 0 : __popc(mask & ((2u << l) - 1u) & ~1u);
      *reinterpret_cast<int32_t*>(r + kLDst + 4 * q) = pdst[p];
    }
  }
}

// every word of every record (a warp per record, coalesced stores; no memset
// first): headers; long records' index padding (overwritten by the real slots)
// and zero destinations / mask; short records' padding lanes (index Z, trash
// row) in their groups, zeros past them
__global__ void k_record_headers(const int32_t* __restrict__ rtype, const int32_t* __restrict__ rL,
                                 const int32_t* __restrict__ rng, int64_t C, int Z, int trash,
                                 const int32_t* __restrict__ unit_c0, int U, int S, uint8_t* __restrict__ rec) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t zz = (uint32_t)Z | ((uint32_t)Z << 16);
  for (int64_t c = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; c < C; c += nw) {
    const int type = __ldg(&rtype[c]), L = __ldg(&rL[c]), ng = __ldg(&rng[c]);
    uint32_t seg = 0;
    if (lane == 3) {  // the record's source segment (read when its unit is gathered unstaged)
      int lo = 0, hi = U - 1;  // last unit u with unit_c0[u] <= c
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(&unit_c0[mid]) <= c) lo = mid;
        else hi = mid - 1;
      }
      seg = (uint32_t)(lo % S);
    }
    const bool compact = type == 3;
    const int gb = type == 1 ? 1 : short_group_bytes(L, compact);
    uint32_t* r = reinterpret_cast<uint32_t*>(rec + c * kRecBytes);
    for (int wi = lane; wi < kRecBytes / 4; wi += 32) {
      const int o = 4 * wi;
      uint32_t v = 0u;
      if (o < kRecHdr) {
        v = o == 0 ? (uint32_t)type : o == 4 ? (uint32_t)L : o == 8 ? (uint32_t)ng : seg;
      } else if (type == 1) {
        if (o < kLDst) v = zz;
      } else {
        const int g = (o - kRecHdr) / gb, go = (o - kRecHdr) - g * gb;
        if (g < ng) {
          if (go < 64 * L) v = zz;                          // idx padding (the identity slot)
          else if (!compact) v = (uint32_t)trash;           // wide: trash destination
          else if (go < 64 * L + 64) v = 0xFFFFFFFFu;       // compact: trash offsets
          // compact: base 0 (set by placement)
        }
      }
      r[wi] = v;
    }
  }
}

// the largest destination span of any 32-piece group of each short class (pieces
// are in ascending destination order inside a class): compact groups need < 65535.
// A thread per short piece in class order; the first piece of each group folds its
// group's span into span[class] (zeroed) — one class can hold millions of groups
// (the hub segments), so a thread per class would serialise them
__global__ void k_class_span(const uint32_t* __restrict__ sckey, int64_t NS, const int64_t* __restrict__ cstart,
                             const int32_t* __restrict__ spid, const int32_t* __restrict__ pdst,
                             int32_t* __restrict__ span) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < NS; j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = sckey[j];
    const int64_t c0 = cstart[k];
    if ((j - c0) & 31) continue;
    const int64_t ql = min(j + 31, cstart[k + 1] - 1);
    const int32_t d = pdst[spid[ql]] - pdst[spid[j]];
    if (d > 0) atomicMax(&span[k], d);
  }
}

// short pieces in class order: piece at class rank q -> record, group, lane
template <typename OffT>
__global__ void k_place_short(const uint32_t* __restrict__ sckey, const int32_t* __restrict__ spid, int64_t NS,
                              const int64_t* __restrict__ cstart, const int32_t* __restrict__ crec0,
                              const int64_t* __restrict__ pstart, const uint32_t* __restrict__ skey,
                              const OffT* __restrict__ order, const int32_t* __restrict__ idx,
                              const int32_t* __restrict__ pdst, int Z, int S, uint8_t* __restrict__ rec) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < NS; j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = sckey[j];
    const int L = (int)(k % 16u);
    const int64_t q = j - cstart[k];
    const int64_t grp = q / 32;
    const bool compact = *reinterpret_cast<const int32_t*>(rec + (int64_t)crec0[k] * kRecBytes) == 3;
    const int lane = (int)(q % 32), R = short_groups(L, compact);
    uint8_t* b = rec + (int64_t)(crec0[k] + grp / R) * kRecBytes + kRecHdr + (grp % R) * short_group_bytes(L, compact);
    const int32_t p = spid[j];
    const int64_t base = (int64_t)(skey[pstart[p]] % (uint32_t)S) * Z;
    for (int e = 0; e < L; ++e)
      *reinterpret_cast<uint16_t*>(b + 64 * e + 2 * lane) = (uint16_t)(idx[(int64_t)order[pstart[p] + e]] - base);
    if (compact) {  // offset from the group's first (smallest) destination
      const int32_t d0 = pdst[spid[cstart[k] + grp * 32]];
      *reinterpret_cast<uint16_t*>(b + 64 * L + 2 * lane) = (uint16_t)(pdst[p] - d0);
      if (lane == 0) *reinterpret_cast<int32_t*>(b + 64 * L + 64) = d0;
    } else {
      *reinterpret_cast<int32_t*>(b + 64 * L + 4 * lane) = pdst[p];
    }
  }
}

template <typename T>
static gi_status exclusive_scan(const T* in, T* out, int64_t n, DevBuf& tmp, cudaStream_t st) {
  size_t tb = 0;
  GI_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, st));
  if (tmp.bytes < tb) GI_TRY(tmp.alloc(tb));
  GI_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, n, st));
  return GI_OK;
}

template <typename T>
static gi_status inclusive_scan(const T* in, T* out, int64_t n, DevBuf& tmp, cudaStream_t st) {
  size_t tb = 0;
  GI_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, in, out, n, st));
  if (tmp.bytes < tb) GI_TRY(tmp.alloc(tb));
  GI_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tb, in, out, n, st));
  return GI_OK;
}

template <typename K, typename V>
static gi_status sort_pairs(const K* ki, K* ko, const V* vi, V* vo, int64_t n, int bits, DevBuf& tmp,
                            cudaStream_t st) {
  size_t tb = 0;  // stable LSD radix sort
  GI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, ki, ko, vi, vo, n, 0, bits, st));
  if (tmp.bytes < tb) GI_TRY(tmp.alloc(tb));
  GI_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, ki, ko, vi, vo, n, 0, bits, st));
  return GI_OK;
}

}  // namespace

static gi_status seg_upload_ctas(gi_graph g);

// a grow-only pinned host array, kept per thread across layout builds (its
// previous upload has completed: every block build ends synchronised)
struct PinnedI32 {
  int32_t* p = nullptr;
  size_t cap = 0;
  gi_status resize(size_t n) {
    if (n <= cap) return GI_OK;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    const size_t want = n + n / 4;
    GI_CUDA(cudaMallocHost(&p, want * sizeof(int32_t)));
    cap = want;
    return GI_OK;
  }
};

// the records of one destination block (CSC rows [r0, r1), fewer than 2^31
// edges): units (block, segment) for every segment, in segment order
struct SegBlock {
  DevBuf rec;                   // C records
  std::vector<int32_t> uc;      // S + 1: first record of each unit (block-local)
  std::vector<int64_t> cost;    // per record, for the CTA balance
  int64_t C = 0, CL = 0, NS = 0, P = 0;
};

template <typename OffT>
static gi_status seg_build_block(gi_graph g, int Z, int S, int64_t r0, int64_t r1, SegBlock& out) {
  gi_context ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  const int64_t nb = r1 - r0;
  int64_t e0 = 0, e1 = 0;
  GI_CUDA(cudaMemcpyAsync(&e0, g->csc_off.as<OffT>() + r0, sizeof(OffT), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaMemcpyAsync(&e1, g->csc_off.as<OffT>() + r1, sizeof(OffT), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  if (sizeof(OffT) == 4) {  // the copies filled the low halves
    e0 = (int64_t)(int32_t)e0;
    e1 = (int64_t)(int32_t)e1;
  }
  const int64_t m = e1 - e0;
  if (m >= INT32_MAX) return fail(GI_ERR_INTERNAL, "segmented pull: block of 2^31 edges");
  // diagnostics (GI_DEBUG_SEG_LAYOUT): synchronised phase times of this block's build
  static const char* ldbg = getenv("GI_DEBUG_SEG_LAYOUT");
  auto tp = std::chrono::steady_clock::now();
  std::string phases;
  auto mark = [&](const char* name) {
    if (!ldbg) return;
    cudaStreamSynchronize(st);
    const auto t2 = std::chrono::steady_clock::now();
    char b[64];
    snprintf(b, sizeof(b), " %s=%.1f", name, std::chrono::duration<double, std::milli>(t2 - tp).count());
    phases += b;
    tp = t2;
  };
  const OffT* off = g->csc_off.as<OffT>() + r0;
  const int32_t* idx = g->csc_idx.as<int32_t>() + e0;
  const int U = S;  // this block's units
  const int64_t DB = INT64_MAX;  // one block: the unit key is the segment
  out.rec.reset();
  out.uc.clear();
  out.cost.clear();
  out.C = out.CL = out.NS = out.P = 0;
  if (m == 0) {
    out.uc.assign(S + 1, 0);
    return GI_OK;
  }
  DevBuf row, key, skey, eid, order, tmp;
  GI_TRY(row.alloc(m * sizeof(int32_t)));
  k_edge_rows<OffT><<<grid_for(nb * 32, 256, sms, 16), 256, 0, st>>>(off, nb, e0, r0, row.as<int32_t>());
  GI_TRY(key.alloc(m * sizeof(uint32_t)));
  GI_TRY(skey.alloc(m * sizeof(uint32_t)));
  GI_TRY(eid.alloc(m * sizeof(OffT)));
  GI_TRY(order.alloc(m * sizeof(OffT)));
  k_unit_keys<OffT><<<grid_for(m, 256, sms), 256, 0, st>>>(idx, row.as<int32_t>(), m, Z, S, DB, key.as<uint32_t>(),
                                                          eid.as<OffT>());
  mark("keys");
  int kbits = 1;
  while ((1ll << kbits) < U) ++kbits;
  // stable: (v, w) order is kept inside each unit
  GI_TRY(sort_pairs(key.as<uint32_t>(), skey.as<uint32_t>(), eid.as<OffT>(), order.as<OffT>(), m, kbits, tmp, st));
  mark("sort1");
  key.reset();
  eid.reset();
  // ---- pieces: (unit, destination) runs of the sorted edges
  DevBuf h, pid, pstart, punit, pdst, asz, aoff, ckey, pids, sckey, spid, unit_p0;
  GI_TRY(h.alloc(m * sizeof(int32_t)));
  GI_TRY(pid.alloc(m * sizeof(int32_t)));
  k_sorted_heads<OffT><<<grid_for(m, 256, sms), 256, 0, st>>>(skey.as<uint32_t>(), order.as<OffT>(), row.as<int32_t>(),
                                                              m, h.as<int32_t>());
  GI_TRY(inclusive_scan(h.as<int32_t>(), pid.as<int32_t>(), m, tmp, st));
  int32_t Pi = 0;
  GI_CUDA(cudaMemcpyAsync(&Pi, pid.as<int32_t>() + m - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  const int64_t P = Pi;
  GI_TRY(pstart.alloc((P + 1) * sizeof(int64_t)));
  GI_TRY(punit.alloc((P + 1) * sizeof(int32_t)));
  GI_TRY(pdst.alloc((P + 1) * sizeof(int32_t)));
  k_piece_info<OffT><<<grid_for(m, 256, sms), 256, 0, st>>>(h.as<int32_t>(), pid.as<int32_t>(), skey.as<uint32_t>(),
                                                            order.as<OffT>(), row.as<int32_t>(), m,
                                                            pstart.as<int64_t>(), punit.as<int32_t>(),
                                                            pdst.as<int32_t>());
  mark("pieces");
  h.reset();
  pid.reset();
  row.reset();
  // ---- classes: long pieces (lane-aligned records) and short pieces by (unit, L)
  const uint32_t sentinel = (uint32_t)U * 16u;
  GI_TRY(asz.alloc((P + 1) * sizeof(int64_t)));
  GI_TRY(aoff.alloc((P + 1) * sizeof(int64_t)));
  GI_TRY(ckey.alloc((P + 1) * sizeof(uint32_t)));
  GI_TRY(pids.alloc((P + 1) * sizeof(int32_t)));
  GI_TRY(sckey.alloc((P + 1) * sizeof(uint32_t)));
  GI_TRY(spid.alloc((P + 1) * sizeof(int32_t)));
  k_piece_class<<<grid_for(P, 256, sms), 256, 0, st>>>(pstart.as<int64_t>(), punit.as<int32_t>(), P, m,
                                                       asz.as<int64_t>(), ckey.as<uint32_t>(), pids.as<int32_t>(),
                                                       sentinel);
  GI_CUDA(cudaMemsetAsync(asz.as<int64_t>() + P, 0, sizeof(int64_t), st));
  GI_TRY(exclusive_scan(asz.as<int64_t>(), aoff.as<int64_t>(), P + 1, tmp, st));
  int cbits = 1;
  while ((1ll << cbits) <= (int64_t)sentinel) ++cbits;
  GI_TRY(sort_pairs(ckey.as<uint32_t>(), sckey.as<uint32_t>(), pids.as<int32_t>(), spid.as<int32_t>(), P, cbits, tmp,
                    st));
  mark("classes");
  ckey.reset();
  pids.reset();
  const int64_t NC = (int64_t)U * 16;  // short classes (L = 0 unused)
  DevBuf cstart;
  GI_TRY(cstart.alloc((NC + 1) * sizeof(int64_t)));
  GI_TRY(unit_p0.alloc((U + 1) * sizeof(int64_t)));
  k_lower_bounds<uint32_t><<<grid_for(NC + 1, 256, sms), 256, 0, st>>>(sckey.as<uint32_t>(), P, NC + 1,
                                                                      cstart.as<int64_t>());
  k_lower_bounds<int32_t><<<grid_for(U + 1, 256, sms), 256, 0, st>>>(punit.as<int32_t>(), P, U + 1,
                                                                    unit_p0.as<int64_t>());
  std::vector<int64_t> h_cs(NC + 1), h_up0(U + 1), h_ao(U + 1);
  GI_CUDA(cudaMemcpyAsync(h_cs.data(), cstart.p, (NC + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaMemcpyAsync(h_up0.data(), unit_p0.p, (U + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  {  // h_ao[u] = aoff[unit_p0[u]]: one gather, one copy
    DevBuf ao;
    GI_TRY(ao.alloc((U + 1) * sizeof(int64_t)));
    k_gather_i64<<<grid_for(U + 1, 256, sms), 256, 0, st>>>(aoff.as<int64_t>(), unit_p0.as<int64_t>(), U + 1,
                                                           ao.as<int64_t>());
    GI_CUDA(cudaMemcpyAsync(h_ao.data(), ao.p, (U + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    GI_CUDA(cudaStreamSynchronize(st));
  }
  // the largest destination span of a group of each short class: compact groups where it fits 16 bits
  std::vector<int32_t> h_span(NC, 0);
  {
    DevBuf span;
    GI_TRY(span.alloc(std::max<int64_t>(NC, 1) * sizeof(int32_t)));
    GI_CUDA(cudaMemsetAsync(span.p, 0, std::max<int64_t>(NC, 1) * sizeof(int32_t), st));
    const int64_t NSc = h_cs[NC];  // the short pieces: class keys below the long pieces' sentinel sort first
    if (NSc > 0)
      k_class_span<<<grid_for(NSc, 256, sms, 8), 256, 0, st>>>(sckey.as<uint32_t>(), NSc, cstart.as<int64_t>(),
                                                               spid.as<int32_t>(), pdst.as<int32_t>(),
                                                               span.as<int32_t>());
    GI_CUDA(cudaMemcpyAsync(h_span.data(), span.p, NC * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    GI_CUDA(cudaStreamSynchronize(st));
  }
  static const bool compact_on = !getenv("GI_SEG_COMPACT") || atoi(getenv("GI_SEG_COMPACT")) != 0;
  auto compact_k = [&](int64_t k) { return compact_on && h_span[k] < 65535; };
  mark("bounds");
  int64_t hist_L[16] = {};  // short pieces by length (layout diagnostics)
  // ---- record layout: per unit, long records then short records by L. Counts
  // first (the first record of every unit and class), then each class's run of
  // records filled at once (millions of records: no per-record push_back)
  // (the per-record staging vectors are kept per thread: tens of MB, first-touch
  // page faults on every build otherwise)
  static thread_local PinnedI32 h_type, h_L, h_ng;  // pinned: the uploads below run at full PCIe rate
  std::vector<int32_t> h_uc(U + 1), h_crec0(NC, 0);
  std::vector<int64_t>& h_cost = out.cost;  // per record, for the CTA balance (capacity kept across builds)
  int64_t C = 0, CL = 0, NS = 0;
  for (int u = 0; u < U; ++u) {
    h_uc[u] = (int32_t)C;
    const int64_t nl = ceil_div(h_ao[u + 1] - h_ao[u], kChunkE);
    C += nl;
    CL += nl;
    for (int L = 1; L < 16; ++L) {
      const int64_t k = (int64_t)u * 16 + L;
      const int64_t cnt = h_cs[k + 1] - h_cs[k];
      NS += cnt;
      hist_L[L] += cnt;
      h_crec0[k] = (int32_t)C;
      C += ceil_div(ceil_div(cnt, 32), short_groups(L, compact_k(k)));
    }
    if (C >= INT32_MAX) return fail(GI_ERR_UNSUPPORTED, "segmented pull: more than 2^31 records");
  }
  GI_TRY(h_type.resize(C));
  GI_TRY(h_L.resize(C));
  GI_TRY(h_ng.resize(C));
  h_cost.resize(C);
  for (int u = 0; u < U; ++u) {
    const int64_t c0 = h_uc[u], nl = ceil_div(h_ao[u + 1] - h_ao[u], kChunkE);
    std::fill_n(h_type.p + c0, nl, 1);
    std::fill_n(h_L.p + c0, nl, 0);
    std::fill_n(h_ng.p + c0, nl, 0);
    std::fill_n(h_cost.begin() + c0, nl, (int64_t)(kChunkE + 2 * kPieceCost));
    for (int L = 1; L < 16; ++L) {
      const int64_t k = (int64_t)u * 16 + L;
      const int64_t groups = ceil_div(h_cs[k + 1] - h_cs[k], 32);
      if (groups == 0) continue;
      const bool cmp = compact_k(k);
      const int64_t R = short_groups(L, cmp), nr = ceil_div(groups, R), c = h_crec0[k];
      const int ngl = (int)(groups - (nr - 1) * R);  // the last record's groups
      std::fill_n(h_type.p + c, nr, cmp ? 3 : 2);
      std::fill_n(h_L.p + c, nr, L);
      std::fill_n(h_ng.p + c, nr - 1, (int32_t)R);
      h_ng.p[c + nr - 1] = ngl;
      std::fill_n(h_cost.begin() + c, nr - 1, R * 32 * (L + kPieceCost));
      h_cost[c + nr - 1] = (int64_t)ngl * 32 * (L + kPieceCost);
    }
  }
  h_uc[U] = (int32_t)C;
  mark("host_layout");
  DevBuf unit_c0, crec0, rtype, rL, rng;
  GI_TRY(unit_c0.alloc((U + 1) * sizeof(int32_t)));
  GI_TRY(crec0.alloc((NC + 1) * sizeof(int32_t)));
  GI_TRY(rtype.alloc((C + 1) * sizeof(int32_t)));
  GI_TRY(rL.alloc((C + 1) * sizeof(int32_t)));
  GI_TRY(rng.alloc((C + 1) * sizeof(int32_t)));
  GI_CUDA(cudaMemcpyAsync(unit_c0.p, h_uc.data(), (U + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  GI_CUDA(cudaMemcpyAsync(crec0.p, h_crec0.data(), NC * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  if (C > 0) {
    GI_CUDA(cudaMemcpyAsync(rtype.p, h_type.p, C * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    GI_CUDA(cudaMemcpyAsync(rL.p, h_L.p, C * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    GI_CUDA(cudaMemcpyAsync(rng.p, h_ng.p, C * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  }
  GI_TRY(out.rec.alloc(C * kRecBytes + 16));
  GI_CUDA(cudaMemsetAsync(out.rec.as<uint8_t>() + C * kRecBytes, 0, 16, st));  // k_record_headers writes the rest
  const int trash = (int)g->nr;  // accumulator row past the owned rows
  k_record_headers<<<grid_for(C * 32, 256, sms, 8), 256, 0, st>>>(
      rtype.as<int32_t>(), rL.as<int32_t>(), rng.as<int32_t>(), C, Z, trash, unit_c0.as<int32_t>(), (int)U, S,
      out.rec.as<uint8_t>());
  mark("headers");
  const int64_t NL = P - NS;  // long pieces: the tail of the class order (sentinel key)
  if (NL > 0)
    k_place_long<OffT><<<grid_for(NL * 32, 256, sms, 16), 256, 0, st>>>(
        asz.as<int64_t>(), aoff.as<int64_t>(), punit.as<int32_t>(), unit_p0.as<int64_t>(), unit_c0.as<int32_t>(),
        pstart.as<int64_t>(), skey.as<uint32_t>(), order.as<OffT>(), idx, pdst.as<int32_t>(), P, m, Z, S,
        spid.as<int32_t>() + NS, NL, out.rec.as<uint8_t>());
  mark("place_long");
  if (NL > 0)
    k_long_dst<<<grid_for(NL, 256, sms), 256, 0, st>>>(asz.as<int64_t>(), aoff.as<int64_t>(), punit.as<int32_t>(),
                                                       unit_p0.as<int64_t>(), unit_c0.as<int32_t>(), pdst.as<int32_t>(),
                                                       spid.as<int32_t>() + NS, NL, out.rec.as<uint8_t>());
  if (NS > 0)
    k_place_short<OffT><<<grid_for(NS, 256, sms), 256, 0, st>>>(
        sckey.as<uint32_t>(), spid.as<int32_t>(), NS, cstart.as<int64_t>(), crec0.as<int32_t>(), pstart.as<int64_t>(),
        skey.as<uint32_t>(), order.as<OffT>(), idx, pdst.as<int32_t>(), Z, S, out.rec.as<uint8_t>());
  mark("long_dst+short");
  if (ldbg && !phases.empty())
    if (FILE* f = fopen(ldbg, "a")) {
      fprintf(f, "block rows [%lld, %lld) edges %lld:%s\n  short pieces by L:", (long long)r0, (long long)r1,
              (long long)m, phases.c_str());
      for (int L = 1; L < 16; ++L) fprintf(f, " %d:%lld", L, (long long)hist_L[L]);
      int64_t ncmp = 0, nshort = 0;
      for (int64_t c = 0; c < C; ++c) {
        ncmp += h_type.p[c] == 3;
        nshort += h_type.p[c] != 1;
      }
      fprintf(f, "\n  short records %lld (compact %lld)\n", (long long)nshort, (long long)ncmp);
      fclose(f);
    }
  GI_CUDA(cudaGetLastError());
  GI_CUDA(cudaStreamSynchronize(st));  // the temporaries are freed on return
  out.uc = std::move(h_uc);
  out.C = C;
  out.CL = CL;
  out.NS = NS;
  out.P = P;
  return GI_OK;
}

// GI_SEG_STEAL: 0 static ranges only, 1 (default) stealing on large layouts, 2 stealing on
// every layout (tests); read at each layout build
static int seg_steal() { return getenv("GI_SEG_STEAL") ? atoi(getenv("GI_SEG_STEAL")) : 1; }

template <typename OffT>
static gi_status seg_build_t(gi_graph g, int Z, int64_t DB) {
  gi_context ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  const int64_t n = g->nr, m = g->ml;  // CSC rows (owned destinations) and local edges
  const int S = (int)ceil_div(g->n, Z);  // segments over all sources
  if ((int64_t)S * 16 >= INT32_MAX / 2) return fail(GI_ERR_UNSUPPORTED, "segmented pull: too many units");
  const auto tb0 = std::chrono::steady_clock::now();
  // destination blocks: at most DB rows (the accumulator range kept in L2) and
  // fewer than 2^31 edges each (the build's sorts and piece ids are 32-bit)
  // (only the offsets at candidate block ends are read back; a block over emax
  // edges reads its rows' offsets to cut it)
  auto off_at = [&](int64_t r, int64_t* v) -> gi_status {
    OffT x = 0;
    GI_CUDA(cudaMemcpyAsync(&x, g->csc_off.as<OffT>() + r, sizeof(OffT), cudaMemcpyDeviceToHost, st));
    GI_CUDA(cudaStreamSynchronize(st));
    *v = (int64_t)x;
    return GI_OK;
  };
  const auto tb_hoff = std::chrono::steady_clock::now();
  std::vector<int64_t> br{0};
  {
    static const int64_t emax = getenv("GI_SEG_BLOCK_EDGES") ? atoll(getenv("GI_SEG_BLOCK_EDGES")) : kBlockEdges;
    int64_t r = 0;
    while (r < n) {
      int64_t r1 = std::min<int64_t>(n, r + DB);
      int64_t er = 0, er1 = 0;
      GI_TRY(off_at(r, &er));
      GI_TRY(off_at(r1, &er1));
      if (er1 - er > emax) {  // last row keeping the block under emax edges
        std::vector<OffT> hoff(r1 - r + 1);
        GI_CUDA(cudaMemcpyAsync(hoff.data(), g->csc_off.as<OffT>() + r, (r1 - r + 1) * sizeof(OffT),
                                cudaMemcpyDeviceToHost, st));
        GI_CUDA(cudaStreamSynchronize(st));
        r1 = r + std::max<int64_t>(1, (int64_t)(std::upper_bound(hoff.begin(), hoff.end(), (OffT)(er + emax)) -
                                                hoff.begin()) - 1);
      }
      br.push_back(r1);
      r = r1;
    }
    if (n == 0) br.push_back(0);
  }
  const int B = (int)br.size() - 1;
  if ((int64_t)B * S >= INT32_MAX / 2) return fail(GI_ERR_UNSUPPORTED, "segmented pull: too many units");
  const int U = B * S;
  // the blocks (their host vectors keep their capacity across layout builds on
  // this thread: tens of MB, first-touch page faults on every build otherwise)
  static thread_local std::vector<std::unique_ptr<SegBlock>> tl_blocks;
  while ((int)tl_blocks.size() < B) tl_blocks.emplace_back(new SegBlock());
  struct Release {  // the blocks' device records go back to the cache on every return
    std::vector<std::unique_ptr<SegBlock>>& v;
    int b;
    ~Release() {
      for (int i = 0; i < b; ++i) v[i]->rec.reset();
    }
  } release_{tl_blocks, B};
  auto blocks = [&](int b) -> SegBlock& { return *tl_blocks[b]; };
  int64_t C = 0, CL = 0, NS = 0, P = 0;
  std::vector<double> tblk;
  for (int b = 0; b < B; ++b) {
    const auto tq = std::chrono::steady_clock::now();
    GI_TRY(seg_build_block<OffT>(g, Z, S, br[b], br[b + 1], blocks(b)));
    tblk.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tq).count());
    C += blocks(b).C;
    CL += blocks(b).CL;
    NS += blocks(b).NS;
    P += blocks(b).P;
    if (C >= INT32_MAX) return fail(GI_ERR_UNSUPPORTED, "segmented pull: more than 2^31 records");
  }
  // concatenate the blocks' records; unit u = b * S + segment
  std::vector<int32_t> h_uc(U + 1);
  GI_TRY(g->seg_rec.alloc(C * kRecBytes + 16));
  GI_CUDA(cudaMemsetAsync(g->seg_rec.as<uint8_t>() + C * kRecBytes, 0, 16, st));
  int64_t cb = 0;
  for (int b = 0; b < B; ++b) {
    SegBlock& k = blocks(b);
    for (int s = 0; s < S; ++s) h_uc[b * S + s] = (int32_t)(cb + k.uc[s]);
    if (k.C > 0)
      GI_CUDA(cudaMemcpyAsync(g->seg_rec.as<uint8_t>() + cb * kRecBytes, k.rec.p, k.C * kRecBytes,
                              cudaMemcpyDeviceToDevice, st));
    cb += k.C;
  }
  h_uc[U] = (int32_t)C;
  GI_CUDA(cudaStreamSynchronize(st));
  for (int b = 0; b < B; ++b) blocks(b).rec.reset();
  const auto tb1 = std::chrono::steady_clock::now();
  // ---- cost-balanced CTA ranges (every staged unit start adds kUnitCost)
  const int ctas = sms;
  std::vector<int32_t> h_cta(ctas + 1, (int32_t)C);
  {
    std::vector<int64_t> pre(C + 1, 0);
    int u = 0, kb = 0;
    int64_t kc0 = 0;  // first record of block kb
    for (int64_t c = 0; c < C; ++c) {
      while (c - kc0 >= blocks(kb).C) kc0 += blocks(kb++).C;
      int64_t cost = blocks(kb).cost[c - kc0];
      while (u + 1 < U && h_uc[u + 1] <= c) ++u;  // u: the unit holding record c
      if (h_uc[u + 1] - h_uc[u] < kDirectRecs) cost *= kDirectCost;  // unstaged: L2 gathers
      else if (h_uc[u] == c) cost += kUnitCost;
      pre[c + 1] = pre[c] + cost;
    }
    int64_t c = 0;
    h_cta[0] = 0;
    for (int k = 1; k < ctas; ++k) {
      const int64_t target = pre[C] * k / ctas;
      while (c < C && pre[c] < target) ++c;
      h_cta[k] = (int32_t)c;
    }
    h_cta[ctas] = (int32_t)C;
    g->seg_h_model.swap(pre);  // the model's prefix: the shape of cost inside a range when re-balancing
  }
  GI_TRY(g->seg_unit_c0.alloc((U + 1) * sizeof(int32_t)));
  GI_CUDA(cudaMemcpyAsync(g->seg_unit_c0.p, h_uc.data(), (U + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  GI_TRY(g->seg_cta.alloc((2 * ctas + 1) * sizeof(int32_t)));
  g->seg_h_cta = h_cta;
  g->seg_h_uc = h_uc;
  GI_TRY(seg_upload_ctas(g));
  GI_TRY(g->seg_time.alloc(4 * ctas * sizeof(unsigned long long)));
  GI_TRY(g->seg_ht.alloc(ctas * sizeof(unsigned long long)));
  GI_CUDA(cudaMemsetAsync(g->seg_ht.p, 0, ctas * sizeof(unsigned long long), st));  // every range empty
  // work stealing where each CTA holds many records (a large graph), on top of the
  // measured-time re-balancing of the static cuts (stealing only evens out the rest:
  // a steal costs a segment staging and breaks the thief's contiguity)
  const int steal_mode = seg_steal();
  g->seg_steal = steal_mode == 2 || (steal_mode == 1 && C >= (int64_t)ctas * kStealMinPerCta);
  g->seg_calib = getenv("GI_SEG_NO_CALIB") ? 0 : getenv("GI_SEG_CALIB") ? atoi(getenv("GI_SEG_CALIB")) : kCalibPasses;
  g->seg_acc_stride = (n + 64) & ~31ll;  // >= n + 1: row n is the trash row of padding lanes
  GI_TRY(g->seg_acc.alloc(2 * g->seg_acc_stride * sizeof(float)));
  GI_CUDA(cudaMemsetAsync(g->seg_acc.p, 0, 2 * g->seg_acc_stride * sizeof(float), st));
  g->seg_acc_cur = 0;
  GI_CUDA(cudaGetLastError());
  GI_CUDA(cudaStreamSynchronize(st));
  if (const char* dbg = getenv("GI_DEBUG_SEG_LAYOUT")) {
    if (FILE* f = fopen(dbg, "a")) {
      const auto tb2 = std::chrono::steady_clock::now();
      fprintf(f, "  hoff %.1f ms, per-block builds", std::chrono::duration<double, std::milli>(tb_hoff - tb0).count());
      for (double x : tblk) fprintf(f, " %.1f", x);
      fprintf(f, " ms\n");
      fprintf(f, "n=%lld m=%lld Z=%d S=%d B=%d U=%d records=%lld (long %lld, short %lld) bytes=%lld P=%lld "
              "(short %lld) build %.1f ms (blocks %.1f, ranges + upload %.1f)\n", (long long)n, (long long)m, Z, S, B,
              U, (long long)C, (long long)CL, (long long)(C - CL), (long long)(C * kRecBytes), (long long)P,
              (long long)NS, std::chrono::duration<double, std::milli>(tb2 - tb0).count(),
              std::chrono::duration<double, std::milli>(tb1 - tb0).count(),
              std::chrono::duration<double, std::milli>(tb2 - tb1).count());
      fclose(f);
    }
  }
  g->seg_Z = Z;
  g->seg_S = S;
  g->seg_U = U;
  g->seg_DB = DB;
  g->seg_P = P;
  g->seg_C = C;
  g->seg_ctas = ctas;
  return GI_OK;
}

// Re-balance the CTA record ranges from one launch's measured per-CTA busy
// times: every CTA's time is spread uniformly over its records, and the new
// boundaries cut the resulting cumulative cost into equal shares.
static gi_status seg_rebalance(gi_graph g, const std::vector<unsigned long long>& ht) {
  const int ctas = g->seg_ctas;
  std::vector<int32_t>& hc = g->seg_h_cta;
  std::vector<double> T(ctas, 0.0);
  double total = 0.0;
  for (int k = 0; k < ctas; ++k) {
    if (hc[k + 1] > hc[k] && ht[4 * k + 1] > ht[4 * k]) T[k] = (double)(ht[4 * k + 1] - ht[4 * k]);
    total += T[k];
  }
  if (total <= 0.0) return GI_OK;
  std::vector<int32_t> nc(ctas + 1);
  nc[0] = 0;
  nc[ctas] = hc[ctas];
  // inside CTA k's range the measured time T[k] is spread over the records in
  // proportion to the build's cost model (dense staged records, sparse unstaged
  // ones and segment stagings cost very differently)
  const std::vector<int64_t>& pm = g->seg_h_model;
  int k = 0;
  double before = 0.0;  // cost of CTA ranges < k
  for (int j = 1; j < ctas; ++j) {
    const double target = total * j / ctas;
    while (k < ctas - 1 && before + T[k] < target) before += T[k++];
    const double frac = T[k] > 0.0 ? (target - before) / T[k] : 0.0;
    const double mk = (double)(pm[hc[k + 1]] - pm[hc[k]]);
    const int64_t want = pm[hc[k]] + (int64_t)(frac * mk);  // model position of the cut
    const int32_t cut = (int32_t)(std::lower_bound(pm.begin() + hc[k], pm.begin() + hc[k + 1], want) - pm.begin());
    nc[j] = std::max(nc[j - 1], std::min(hc[k + 1], cut));
  }
  static const double damp = getenv("GI_SEG_DAMP") ? atof(getenv("GI_SEG_DAMP")) : GI_SEG_DAMP;
  for (int j = 1; j < ctas; ++j)  // damped move from the old boundary
    nc[j] = std::max(nc[j - 1], (int32_t)(hc[j] + damp * (nc[j] - hc[j]) + 0.5));
  hc = nc;
  return seg_upload_ctas(g);
}

// seg_cta = [record start of each CTA (ctas + 1)] ++ [unit of each CTA's first record (ctas)]
static gi_status seg_upload_ctas(gi_graph g) {
  const std::vector<int32_t>& hc = g->seg_h_cta;
  const std::vector<int32_t>& uc = g->seg_h_uc;
  const int ctas = (int)hc.size() - 1;
  std::vector<int32_t> buf(hc);
  buf.resize(2 * ctas + 1);
  for (int c = 0; c < ctas; ++c)  // last unit u with unit_c0[u] <= hc[c]
    buf[ctas + 1 + c] = std::max<int32_t>(0, (int32_t)(std::upper_bound(uc.begin(), uc.end() - 1, hc[c]) - uc.begin()) - 1);
  // pageable source: the call returns once buf has been staged
  GI_CUDA(cudaMemcpyAsync(g->seg_cta.p, buf.data(), buf.size() * sizeof(int32_t), cudaMemcpyHostToDevice,
                          g->ctx->stream));
  return GI_OK;
}

static size_t seg_dyn_smem(int Z) { return (size_t)kStages * kStageBytes + ((size_t)Z + 4) * sizeof(float); }

gi_status seg_default_Z(gi_graph g, int* Zout) {
  int optin = 0;
  GI_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, g->ctx->device));
  cudaFuncAttributes a{};
  GI_CUDA(cudaFuncGetAttributes(&a, k_pr_seg<0, OpSum>));
  int Z = (optin - (int)a.sharedSizeBytes - 64 - (int)seg_dyn_smem(0)) / 4;
  Z = std::min(Z, 65535) & ~31;
  if (Z < 1024) return fail(GI_ERR_UNSUPPORTED, "segmented pull: not enough shared memory");
  *Zout = Z;
  return GI_OK;
}

gi_status seg_build(gi_graph g, int segment_size, int64_t block_rows) {
  if (segment_size < 0 || block_rows < 0) return fail(GI_ERR_INVALID_ARGUMENT, "segment_size / dst_block < 0");
  int Z = 0;
  GI_TRY(seg_default_Z(g, &Z));
  if (segment_size > 0) Z = std::max(32, std::min(Z, segment_size) & ~3);
  int64_t DB = block_rows > 0 ? block_rows : kDefaultBlockRows;
  DB = std::max<int64_t>(1, std::min<int64_t>(DB, std::max<int64_t>(g->nr, 1)));
  if (g->seg_Z == Z && g->seg_DB == DB) return GI_OK;
  g->seg_Z = 0;
  if (g->ml == 0 || g->nr == 0) return fail(GI_ERR_UNSUPPORTED, "segmented pull: empty graph");
  if (g->off64) return seg_build_t<int64_t>(g, Z, DB);
  return seg_build_t<int32_t>(g, Z, DB);
}

// One min pass over the segmented layout (connected components, cc.cu):
// acc[v] = min over v's in-edges (u, v) of labels[u]; acc must hold the
// identity-or-larger (INT_MAX-ish) values for rows 0..n (row n: padding lanes).
gi_status seg_min_pass(gi_graph g, const int32_t* labels, int32_t* acc) {
  cudaStream_t st = g->ctx->stream;
  SegArgs S;
  S.rec = g->seg_rec.as<uint8_t>();
  S.unit_c0 = g->seg_unit_c0.as<int32_t>();
  S.cta_c0 = g->seg_cta.as<int32_t>();
  S.cta_u = g->seg_cta.as<int32_t>() + g->seg_ctas + 1;
  S.cin = reinterpret_cast<const float*>(labels);  // raw 4-byte words: the kernel reads them as int32
  S.acc = reinterpret_cast<float*>(acc);
  S.n = g->n;
  S.Z = g->seg_Z;
  S.S = g->seg_S;
  S.U = g->seg_U;
  S.timing = nullptr;
  S.ht = g->seg_ht.as<unsigned long long>();
  S.trash = (int)g->nr;
  S.steal = g->seg_steal;
  const size_t dyn = seg_dyn_smem(g->seg_Z);
  static size_t attr_min[64] = {};
  const int dev = g->ctx->device & 63;
  if (attr_min[dev] < dyn) {
    GI_CUDA(cudaFuncSetAttribute(k_pr_seg<0, OpMin>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    attr_min[dev] = dyn;
  }
  GI_TRY(launch_pdl(k_pr_seg<0, OpMin>, g->seg_ctas, kSegThreads, dyn, st, S));
  return GI_OK;
}

// One OR pass over the segmented layout (the bit-parallel BFS's dense pull
// levels, msbfs.cu): acc[v] |= OR over v's in-edges (u, v) of masks[u]; masks
// padded by >= 16 words, acc zeroed for rows 0..n (row n: padding lanes).
gi_status seg_or_pass(gi_graph g, const uint32_t* masks, uint32_t* acc) {
  cudaStream_t st = g->ctx->stream;
  SegArgs S;
  S.rec = g->seg_rec.as<uint8_t>();
  S.unit_c0 = g->seg_unit_c0.as<int32_t>();
  S.cta_c0 = g->seg_cta.as<int32_t>();
  S.cta_u = g->seg_cta.as<int32_t>() + g->seg_ctas + 1;
  S.cin = reinterpret_cast<const float*>(masks);  // raw 4-byte words: the kernel reads them as uint32
  S.acc = reinterpret_cast<float*>(acc);
  S.n = g->n;
  S.Z = g->seg_Z;
  S.S = g->seg_S;
  S.U = g->seg_U;
  S.timing = nullptr;
  S.ht = g->seg_ht.as<unsigned long long>();
  S.trash = (int)g->nr;
  S.steal = g->seg_steal;
  const size_t dyn = seg_dyn_smem(g->seg_Z);
  static size_t attr_or[64] = {};
  const int dev = g->ctx->device & 63;
  if (attr_or[dev] < dyn) {
    GI_CUDA(cudaFuncSetAttribute(k_pr_seg<0, OpOr>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    attr_or[dev] = dyn;
  }
  GI_TRY(launch_pdl(k_pr_seg<0, OpOr>, g->seg_ctas, kSegThreads, dyn, st, S));
  return GI_OK;
}

int64_t seg_record_bytes() { return kRecBytes; }

gi_status seg_edge_pass(gi_graph g, const float* cin) {
  cudaStream_t st = g->ctx->stream;
  SegArgs S;
  S.rec = g->seg_rec.as<uint8_t>();
  S.unit_c0 = g->seg_unit_c0.as<int32_t>();
  S.cta_c0 = g->seg_cta.as<int32_t>();
  S.cta_u = g->seg_cta.as<int32_t>() + g->seg_ctas + 1;
  S.cin = cin;
  S.acc = seg_acc_buf(g, g->seg_acc_cur);
  S.n = g->n;
  S.Z = g->seg_Z;
  S.S = g->seg_S;
  S.U = g->seg_U;
  S.ht = g->seg_ht.as<unsigned long long>();
  S.trash = (int)g->nr;
  S.steal = g->seg_steal;
  static const int mode = getenv("GI_SEG_MODE") ? atoi(getenv("GI_SEG_MODE")) : 0;
  void (*kern)(SegArgs) = mode == 1 ? k_pr_seg<1, OpSum> : mode == 2 ? k_pr_seg<2, OpSum>
                        : mode == 3 ? k_pr_seg<3, OpSum> : k_pr_seg<0, OpSum>;
  const size_t dyn = seg_dyn_smem(g->seg_Z);
  static size_t attr_set[64] = {};  // per device: largest dynamic smem size configured so far
  const int dev = g->ctx->device & 63;
  if (attr_set[dev] < dyn) {
    GI_CUDA(cudaFuncSetAttribute(k_pr_seg<0, OpSum>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    GI_CUDA(cudaFuncSetAttribute(k_pr_seg<1, OpSum>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    GI_CUDA(cudaFuncSetAttribute(k_pr_seg<2, OpSum>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    GI_CUDA(cudaFuncSetAttribute(k_pr_seg<3, OpSum>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    attr_set[dev] = dyn;
  }
  static const char* dbg = getenv("GI_DEBUG_SEG_TIMING");  // diagnostics: file to append per-CTA timings to
  const bool timed = dbg || g->seg_calib > 0;
  const int ctas = g->seg_ctas;
  S.timing = nullptr;
  if (timed) {
    GI_CUDA(cudaMemsetAsync(g->seg_time.p, 0, 4 * ctas * sizeof(unsigned long long), st));
    S.timing = g->seg_time.as<unsigned long long>();
  }
  GI_TRY(launch_pdl(kern, ctas, kSegThreads, dyn, st, S));
  if (!timed) return GI_OK;
  std::vector<unsigned long long> ht(4 * ctas);
  GI_CUDA(cudaMemcpyAsync(ht.data(), g->seg_time.p, ht.size() * 8, cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  const std::vector<int32_t>& hc = g->seg_h_cta;
  if (dbg) {
    if (FILE* f = fopen(dbg, "a")) {
      const std::vector<int32_t>& uc = g->seg_h_uc;
      for (int c = 0; c < ctas; ++c) {
        // + records in unstaged (sparse) units, staged units touched, first unit, last unit
        int u = std::max<int>(0, (int)(std::upper_bound(uc.begin(), uc.end() - 1, hc[c]) - uc.begin()) - 1);
        const int ufirst = u;
        long long drec = 0, su = 0;
        for (int32_t r = hc[c]; r < hc[c + 1]; ++r) {
          while (u + 1 < (int)uc.size() - 1 && uc[u + 1] <= r) ++u;
          const bool direct = uc[u + 1] - uc[u] < kDirectRecs;
          if (direct) ++drec;
          else if (r == hc[c] || uc[u] == r) ++su;
        }
        fprintf(f, "%d,%d,%d,%llu,%llu,%llu,%llu,%lld,%lld,%d,%d\n", c, hc[c], hc[c + 1], ht[4 * c], ht[4 * c + 1],
                ht[4 * c + 2], ht[4 * c + 3], drec, su, ufirst, u);
      }
      fclose(f);
    }
  }
  if (g->seg_calib > 0) {
    --g->seg_calib;
    GI_TRY(seg_rebalance(g, ht));
  }
  return GI_OK;
}

gi_status seg_vertex_pass(gi_graph g, const PrArgs& A) {
  cudaStream_t st = g->ctx->stream;
  GI_TRY(launch_pdl(k_pr_acc, grid_for(ceil_div(g->nr, 4), 256, g->ctx->num_sms, GI_ACC_PER_SM), 256, 0, st, A,
                    (const float*)seg_acc_buf(g, g->seg_acc_cur), seg_acc_buf(g, g->seg_acc_cur ^ 1)));
  g->seg_acc_cur ^= 1;
  return GI_OK;
}

}  // namespace gi
