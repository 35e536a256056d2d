// pr_segmented.cu — pull PageRank over shared-memory source segments.
//
// The paper's cache optimisation ("Segmented Subgraphs", PAPER.md P:741-757,
// partition the source range so each segment's
// random reads hit cache, then merge the per-segment partial sums) retargeted
// at the B200's 227 KB of shared memory per CTA. Measured on this part
// (tools/microbench/, profiles/r01_gather_rates.txt, r01_red_rates.txt):
// random 4-byte gathers run at ~1.0 per SM-clock from L2 but ~7 per SM-clock
// from shared memory, so the pull edge pass (a4) gathers contrib from a staged
// segment instead of from L2. A segment holds Z <= 65535 sources, so in-segment
// source ids are 16-bit and the index stream is 2 bytes per edge.
//
// Layout (built once per graph):
//   unit u = (destination block b, source segment s), u = b*S + s, holding the
//            edges (v, w) with v in block b (rows [b*DB, (b+1)*DB)) and w in
//            segment s (sources [s*Z, (s+1)*Z)), in (v, w) order. One block
//            (DB = all rows) unless the accumulator would not fit in L2.
//   piece    = (unit, destination) run: the partial sum the paper's segmented
//              subgraphs merge ("SSG" partials).
//   chunk    = 512 consecutive edge slots of one unit (32 lanes x 16); every
//              unit is padded to whole chunks with the index Z (a shared-memory
//              zero), so a chunk never spans two units.
//   idx[]    uint16 per slot: w - s*Z
//   head[]   1 bit per slot: the slot starts a piece
//   cbase[c] piece index of chunk c's first slot
//   pdst[p]  destination (local row) of piece p
// Per iteration:
//   k_pr_seg  persistent, one 512-thread CTA per SM over a cost-balanced
//             range of chunks: stage the unit's contrib segment in shared
//             memory (TMA bulk copy), then every warp reduces whole chunks on
//             its own — 16 shared-memory gathers per lane, a warp segmented
//             scan whose reset flags come from one ballot — and folds every
//             piece that ends in the chunk (and the one still open at its end)
//             into acc[v] with red.global.add.f32. acc (4 B per row of the
//             block) stays in L2, so no partials go to HBM and no merge pass
//             is needed; pieces cut by chunk boundaries need no carries.
//   k_pr_acc  r'[v] = (1-d)/n + d (acc[v] + D/n), contrib', dangling mass
//             (fused vertex update a3); acc[v] reset to 0.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cub/cub.cuh>
#include <vector>

#include "gi_internal.cuh"
#include "pr_common.cuh"

namespace gi {
namespace {

constexpr int kConsumers = 16;                // consumer warps (one chunk each per stage)
constexpr int kSegThreads = 32 * (kConsumers + 1);  // + one producer warp (TMA)
constexpr int kLaneE = 16;                    // edge slots per lane per chunk
constexpr int kChunkE = 32 * kLaneE;          // edge slots per chunk (one warp)
constexpr int kChunkW = kChunkE / 32;         // head words per chunk
// chunk record (interleaved so one bulk copy moves a run of chunks):
//   uint16 idx[512] | uint32 head[16] | uint16 j0[32] | int32 cbase | pad
// j0[l] = pieces closed in lanes < l (chunk-relative index of the piece open
// at lane l's first slot)
constexpr int kRecHead = 2 * kChunkE;         // byte offset of the head words
constexpr int kRecJ0 = kRecHead + 4 * kChunkW;
constexpr int kRecBase = kRecJ0 + 2 * 32;
constexpr int kRecBytes = kRecBase + 16;      // 1168, a multiple of 16 (bulk-copy granule)
constexpr int kStages = 4;                    // ring depth (stages in flight per CTA)
constexpr int kStageBytes = kConsumers * kRecBytes;
constexpr int kScratch = kChunkE + 32;        // floats of piece scratch per consumer warp
constexpr int kChunkCost = 2 * kChunkE;       // CTA balance: a chunk costs 2 per slot ...
constexpr int kPieceCost = 3;                 // ... plus 3 per piece (fitted from per-CTA timings)
constexpr int64_t kStageCost = 99 * kChunkCost;  // a unit start ~ 99 chunks (staging + pipeline refill)
constexpr int64_t kDefaultBlockRows = 8 << 20;  // 32 MB accumulator per destination block

struct SegArgs {
  const uint8_t* __restrict__ rec;     // kRecBytes per chunk
  const int32_t* __restrict__ cbase;   // C + 1 (consumers prefetch piece destinations ahead)
  const int32_t* __restrict__ pdst;    // P (+ padding)
  const int32_t* __restrict__ unit_c0; // U + 1: first chunk of each unit
  const int32_t* __restrict__ cta_c0;  // grid + 1: first chunk of each CTA
  const float* __restrict__ cin;       // contrib, global ids, padded by >= 16 floats
  float* __restrict__ acc;             // per local row
  int64_t n;
  int Z, S, U;
  // diagnostics (GI_SEG_MODE, template MODE): 0 full, 1 no REDs, 2 gathers only, 3 stream only
  unsigned long long* timing;  // diagnostics (GI_DEBUG_SEG_TIMING): per CTA [start, end, staging ns, units]
};

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

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Reduce one chunk whose record sits in shared memory at `r`. SMEM: gather
// from the staged segment `sc`; else from global `gsrc` (= cin + s*Z; the
// padding index Z reads as 0). `sv` is this warp's scratch: the value of the
// chunk's j-th piece (piece cbase + j) lands in sv[j], then the warp folds
// them into acc with dense, coalesced REDs (a chunk's pieces have increasing
// destinations). `empty`: the stage barrier to release once the record is
// in registers.
template <int MODE, bool SMEM>
__device__ __forceinline__ void chunk_reduce(const SegArgs& A, const uint8_t* r, const float* sc, const float* gsrc,
                                             float* sv, int lane, int Z, uint64_t* empty, int pd0, int pd1) {
  const uint4 qa = *reinterpret_cast<const uint4*>(r + 32 * lane);
  const uint4 qb = *reinterpret_cast<const uint4*>(r + 32 * lane + 16);
  const uint32_t hw = *reinterpret_cast<const uint32_t*>(r + kRecHead + 4 * (lane >> 1));
  const int cb = *reinterpret_cast<const int32_t*>(r + kRecBase);
  const int j0 = *reinterpret_cast<const uint16_t*>(r + kRecJ0 + 2 * lane);
  __syncwarp();
  if (lane == 0) mbar_arrive(empty);  // the record may be overwritten now
  const uint32_t w[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
  if (MODE == 3) {  // diagnostics: stream only
    if ((qa.x ^ qa.y ^ qa.z ^ qa.w ^ qb.x ^ qb.y ^ qb.z ^ qb.w ^ hw ^ pd0 ^ pd1) == 0x9e3779b9u) A.acc[lane] += 1.f;
    return;
  }
  float v[kLaneE];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t i0 = w[j] & 0xFFFFu, i1 = w[j] >> 16;
    if (SMEM) {
      v[2 * j] = sc[i0];
      v[2 * j + 1] = sc[i1];
    } else {
      v[2 * j] = i0 == (uint32_t)Z ? 0.f : __ldg(gsrc + i0);
      v[2 * j + 1] = i1 == (uint32_t)Z ? 0.f : __ldg(gsrc + i1);
    }
  }
  if (MODE == 2) {  // diagnostics: stream + gathers, no segmentation
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < kLaneE; ++k) s += v[k];
    if (s == -1.f) A.acc[lane + pd0 + pd1] += s;
    return;
  }
  const uint32_t hb = (hw >> ((lane & 1) * 16)) & 0xFFFFu;  // bit k: slot lane*16+k starts a piece
  // every head closes the piece before it, except at chunk position 0 (that
  // piece has no slot in this chunk)
  const uint32_t cl = lane == 0 ? (hb & ~1u) : hb;
  const int cnt = __popc(cl);
  // branch-free pass over the slots, as two independent halves: a closing
  // stores the run it ends at sv[j] (j = chunk-relative index of the piece
  // open at that slot) and restarts it. The lane's first closing ends the
  // piece that began in an earlier lane: the scan's carry is added to it
  // below. Half 1 starts as if no piece were open (run 0); if it has a
  // closing, its first one is completed with half 0's open run.
  constexpr int H = kLaneE / 2;
  const uint32_t cl0 = cl & ((1u << H) - 1u), cl1 = cl >> H;
  float run0 = 0.f, run1 = 0.f;
  float* sp0 = sv + j0;
  float* sp1 = sv + j0 + __popc(cl0);
  float* first1 = sp1;
#pragma unroll
  for (int k = 0; k < H; ++k) {
    const bool c0 = (cl0 >> k) & 1u, c1 = (cl1 >> k) & 1u;
    if (c0) *sp0 = run0;
    if (c1) *sp1 = run1;
    sp0 += c0 ? 1 : 0;
    sp1 += c1 ? 1 : 0;
    run0 = (c0 ? 0.f : run0) + v[k];
    run1 = (c1 ? 0.f : run1) + v[H + k];
  }
  float run;
  if (cl1) {
    *first1 += run0;  // half 1's first closing ends the run open at the end of half 0
    run = run1;
  } else {
    run = run0 + run1;
  }
  // warp segmented inclusive scan of the runs open at each lane's end (`run`:
  // after the lane's last head, or the whole lane); a lane with a head resets
  // it (flags from one ballot)
  const unsigned hm = __ballot_sync(0xffffffffu, hb != 0);
  float X = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float y = __shfl_up_sync(0xffffffffu, X, o);
    if (lane >= o && ((hm >> (lane - o + 1)) & ((1u << o) - 1u)) == 0u) X = y + X;
  }
  float carry = __shfl_up_sync(0xffffffffu, X, 1);  // run open at this lane's start
  if (lane == 0) carry = 0.f;
  if (cnt > 0) sv[j0] += carry;
  const int np = __shfl_sync(0xffffffffu, j0 + cnt, 31);  // closed pieces; piece np is open at the end
  if (lane == 31) sv[np] = X;
  __syncwarp();
  if (MODE == 1) {  // diagnostics: no REDs
    if (sv[lane] == -1.f) A.acc[lane] += 1.f;
    __syncwarp();
    return;
  }
  // dense REDs: lane q folds piece cb + q (destinations of the first 64 in registers)
  float* acc = A.acc;
  if (lane <= np) atomicAdd(acc + pd0, sv[lane]);  // RED.E.ADD.F32
  if (np >= 32) {
    if (lane + 32 <= np) atomicAdd(acc + pd1, sv[lane + 32]);
    for (int q = lane + 64; q <= np; q += 32) atomicAdd(acc + __ldg(&A.pdst[cb + q]), sv[q]);
  }
  __syncwarp();
}

// Persistent CTA per SM over chunks [cta_c0[b], cta_c0[b+1]), unit by unit.
// Warp kConsumers is the producer: one lane streams chunk records into a
// kStages-deep shared-memory ring with bulk copies (full[s]: bytes landed;
// empty[s]: all consumer warps have taken their record). Consumer warp w
// reduces record w of every stage. The unit's contrib segment is staged
// with one more bulk copy when the unit is large enough to repay it.
template <int MODE>
__global__ void __launch_bounds__(kSegThreads, 1) k_pr_seg(SegArgs A) {
  extern __shared__ __align__(128) uint8_t smem[];
  // [kStages][kStageBytes] ring | [kConsumers][kScratch] floats | Z + 4 floats of segment
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages], seg_bar;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint8_t* ring = smem;
  float* scontrib = reinterpret_cast<float*>(smem + kStages * kStageBytes + kConsumers * kScratch * 4);
  int c0 = A.cta_c0[blockIdx.x];
  const int c1 = A.cta_c0[blockIdx.x + 1];
  if (c0 >= c1) return;
  unsigned long long t_start = 0, t_stage = 0, n_units = 0;
  if (A.timing && tid == 0) t_start = globaltimer();
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers);
    }
    mbar_init(&seg_bar, 1);
  }
  __syncthreads();
  int u;  // unit of c0: last u with unit_c0[u] <= c0
  {
    int lo = 0, hi = A.U - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (__ldg(&A.unit_c0[mid]) <= c0) lo = mid;
      else hi = mid - 1;
    }
    u = lo;
  }
  // ring position: stage index and phase, advanced identically by producer and consumers
  uint32_t it = 0;  // stages issued (producer) / consumed (consumers) so far, over all units
  uint32_t seg_phase = 0;
  int staged_seg = -1;
  while (c0 < c1) {
    const int ue = min(c1, __ldg(&A.unit_c0[u + 1]));
    const int seg = u % A.S;
    const bool stage_seg = (int64_t)(ue - c0) * kChunkE * 8 >= A.Z;
    const int nst = (ue - c0 + kConsumers - 1) / kConsumers;  // stages in this unit
    const bool restage = stage_seg && seg != staged_seg;
    if (restage) {
      __syncthreads();  // every consumer is done with the previous segment
      if (tid == 0) {
        const int64_t base = (int64_t)seg * A.Z;
        const int64_t zlen = min((int64_t)A.Z, A.n - base);
        scontrib[A.Z] = 0.f;
        tma_load_1d(scontrib, A.cin + base, (uint32_t)(((zlen * 4) + 15) & ~15ll), &seg_bar);
      }
      staged_seg = seg;
    }
    if (warp == kConsumers) {
      if (lane == 0) {  // producer
        for (int k = 0; k < nst; ++k, ++it) {
          const uint32_t s = it % kStages, ph = (it / kStages) & 1u;
          if (it >= kStages) mbar_wait(&empty[s], ph ^ 1u);  // consumers released this slot's last use
          const int cs = c0 + k * kConsumers;
          const int nc = min(kConsumers, ue - cs);
          tma_load_1d(ring + s * kStageBytes, A.rec + (int64_t)cs * kRecBytes, (uint32_t)(nc * kRecBytes), &full[s]);
        }
      }
      it = __shfl_sync(0xffffffffu, it, 0);
    } else {
      if (restage) {
        const unsigned long long t0 = A.timing && tid == 0 ? globaltimer() : 0;
        mbar_wait(&seg_bar, seg_phase);
        if (A.timing && tid == 0) t_stage += globaltimer() - t0;
      }
      const float* gsrc = A.cin + (int64_t)seg * A.Z;
      float* sv = reinterpret_cast<float*>(smem + kStages * kStageBytes) + warp * kScratch;
      // destinations of the first 64 pieces of this warp's chunks, loaded into
      // registers one chunk ahead (their piece base cbase two chunks ahead);
      // further lines of the next chunk's destinations prefetched into L2
      auto cbase_of = [&](int k) { const int c = c0 + k * kConsumers + warp; return c < ue ? __ldg(&A.cbase[c]) : -1; };
      int pd0 = 0, pd1 = 0;
      {
        const int cb = cbase_of(0);
        if (cb >= 0) {
          pd0 = __ldg(&A.pdst[cb + lane]);  // pdst is padded: always in bounds
          pd1 = __ldg(&A.pdst[cb + 32 + lane]);
        }
      }
      int cb_next = cbase_of(1);
      for (int k = 0; k < nst; ++k, ++it) {
        const uint32_t s = it % kStages, ph = (it / kStages) & 1u;
        int npd0 = 0, npd1 = 0;
        if (cb_next >= 0) {
          npd0 = __ldg(&A.pdst[cb_next + lane]);
          npd1 = __ldg(&A.pdst[cb_next + 32 + lane]);
          if (lane >= 2 && lane < 16) prefetch_l2(A.pdst + cb_next + 32 * lane);
        }
        const int cb_nn = cbase_of(k + 2);
        mbar_wait(&full[s], ph);
        const int c = c0 + k * kConsumers + warp;
        const uint8_t* r = ring + s * kStageBytes + warp * kRecBytes;
        if (c < ue) {
          if (stage_seg) chunk_reduce<MODE, true>(A, r, scontrib, gsrc, sv, lane, A.Z, &empty[s], pd0, pd1);
          else chunk_reduce<MODE, false>(A, r, scontrib, gsrc, sv, lane, A.Z, &empty[s], pd0, pd1);
        } else if (lane == 0) {
          mbar_arrive(&empty[s]);  // nothing to take from this slot
        }
        pd0 = npd0;
        pd1 = npd1;
        cb_next = cb_nn;
      }
    }
    if (restage) seg_phase ^= 1u;
    c0 = ue;
    ++u;
    ++n_units;
  }
  if (A.timing && tid == 0) {
    unsigned long long* T = A.timing + 4 * blockIdx.x;
    T[0] = t_start;
    T[1] = globaltimer();
    T[2] = t_stage;
    T[3] = n_units;
  }
}

// Vertex update over local rows, 4 per thread (vector loads): s = acc[v],
// then pr_epilogue's arithmetic; zero[v] = 0 readies the other accumulator.
__global__ void __launch_bounds__(256) k_pr_acc(PrArgs A, const float* __restrict__ acc, float* __restrict__ zero) {
  __shared__ double sred[32];
  if (blockIdx.x == 0 && threadIdx.x == 0) A.dbuf[(A.it + 2) % 3] = 0.0;
  const double D = A.uniform ? A.dbuf[A.it % 3] : 0.0;
  const float dn = (float)(D * A.inv_n);
  double dpart = 0.0;
  const int64_t nq = A.n / 4;
  const float4* acc4 = reinterpret_cast<const float4*>(acc);
  const bool vec = (A.row0 & 3) == 0;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < (vec ? nq : 0);
       q += (int64_t)gridDim.x * blockDim.x) {
    const float4 s4 = acc4[q];
    reinterpret_cast<float4*>(zero)[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int64_t v0 = A.row0 + 4 * q;
    const int4 od4 = __ldg(reinterpret_cast<const int4*>(A.outdeg + v0));
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
  }
  for (int64_t r = (vec ? 4 * nq : 0) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < A.n;
       r += (int64_t)gridDim.x * blockDim.x) {
    const float s = acc[r];
    zero[r] = 0.f;
    pr_epilogue(A, r, s, dn, dpart);
  }
  const double bs = block_sum(dpart, sred);
  if (threadIdx.x == 0 && bs != 0.0) atomicAdd(&A.dbuf[(A.it + 1) % 3], bs);
}

// ---------------------------------------------------------------- layout build
// interleave idx / head / cbase into chunk records (kRecBytes each)
__global__ void k_pack_records(const uint16_t* __restrict__ idx, const uint32_t* __restrict__ head,
                               const int32_t* __restrict__ cbase, const int32_t* __restrict__ hc, int64_t C,
                               uint8_t* __restrict__ rec) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < C * (kRecBytes / 4);
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / (kRecBytes / 4);
    const int o = (int)(i % (kRecBytes / 4)) * 4;  // byte offset in the record
    uint32_t w;
    if (o < kRecHead) w = reinterpret_cast<const uint32_t*>(idx + c * kChunkE)[o / 4];
    else if (o < kRecJ0) w = head[c * kChunkW + (o - kRecHead) / 4];
    else if (o < kRecBase) {  // two lanes' j0: heads at chunk positions [1, 16 l)
      const int l = (o - kRecJ0) / 2;
      const int64_t p0 = c * kChunkE;
      const uint32_t a = l == 0 ? 0u : (uint32_t)(hc[p0 + kLaneE * l - 1] - hc[p0]);
      const uint32_t b = (uint32_t)(hc[p0 + kLaneE * (l + 1) - 1] - hc[p0]);
      w = a | (b << 16);
    }
    else if (o == kRecBase) w = (uint32_t)cbase[c];
    else w = 0;
    reinterpret_cast<uint32_t*>(rec + c * kRecBytes)[o / 4] = w;
  }
}

__global__ void k_fill_u16(uint16_t* __restrict__ p, int64_t n, uint16_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

// row of every CSC edge (warp per row)
template <typename OffT>
__global__ void k_edge_rows(const OffT* __restrict__ off, int64_t n, int32_t* __restrict__ row) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = w0; v < n; v += nw)
    for (int64_t e = (int64_t)off[v] + lane; e < (int64_t)off[v + 1]; e += 32) row[e] = (int32_t)v;
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

// unit_e[u] = first sorted position of unit u (lower bound of u in the sorted keys)
__global__ void k_unit_starts(const uint32_t* __restrict__ skey, int64_t m, int U, int64_t* __restrict__ unit_e) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u <= U; u += gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = m;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (skey[mid] < (uint32_t)u) lo = mid + 1;
      else hi = mid;
    }
    unit_e[u] = lo;
  }
}

// place sorted edge i at its padded slot: index, head flag, destination
template <typename OffT>
__global__ void k_place(const uint32_t* __restrict__ skey, const OffT* __restrict__ order, int64_t m,
                        const int32_t* __restrict__ idx, const int32_t* __restrict__ row,
                        const int64_t* __restrict__ unit_e, const int32_t* __restrict__ unit_c0, int Z, int S,
                        uint16_t* __restrict__ sidx, int32_t* __restrict__ hflag, int32_t* __restrict__ srow) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t u = skey[i];
    const int64_t e = (int64_t)order[i];
    const int64_t pos = (int64_t)unit_c0[u] * kChunkE + (i - unit_e[u]);
    const int32_t v = row[e];
    const bool h = i == unit_e[u] || v != row[(int64_t)order[i - 1]];
    sidx[pos] = (uint16_t)(idx[e] - (int64_t)(u % S) * Z);
    hflag[pos] = h;
    srow[pos] = v;
  }
}

// pack head flags into bits (one warp per 32 slots)
__global__ void k_pack_heads(const int32_t* __restrict__ hflag, int64_t E, uint32_t* __restrict__ head) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i - lane < E; i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned b = __ballot_sync(0xffffffffu, i < E && hflag[i] != 0);
    if (lane == 0) head[i >> 5] = b;
  }
}

// hc = inclusive count of heads: pdst[hc-1] at heads, cbase[c] = hc[c*kChunkE] - 1
__global__ void k_pieces(const int32_t* __restrict__ hflag, const int32_t* __restrict__ hc,
                         const int32_t* __restrict__ srow, int64_t E, int32_t* __restrict__ pdst,
                         int32_t* __restrict__ cbase) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < E; q += (int64_t)gridDim.x * blockDim.x) {
    if (hflag[q]) pdst[hc[q] - 1] = srow[q];
    if ((q % kChunkE) == 0) cbase[q / kChunkE] = hc[q] - 1;
  }
}

}  // namespace

template <typename OffT>
static gi_status seg_build_t(gi_graph g, int Z, int64_t DB) {
  gi_context ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  const int64_t n = g->nr, m = g->ml;  // CSC rows (owned destinations) and local edges
  const OffT* off = g->csc_off.as<OffT>();
  const int32_t* idx = g->csc_idx.as<int32_t>();
  const int S = (int)ceil_div(g->n, Z);         // segments over all sources
  const int B = (int)ceil_div(n, DB);           // destination blocks
  if ((int64_t)B * S >= INT32_MAX / 2) return fail(GI_ERR_UNSUPPORTED, "segmented pull: too many units");
  const int U = B * S;
  DevBuf row, key, skey, eid, order, unit_e, tmp;
  GI_TRY(row.alloc(m * sizeof(int32_t)));
  k_edge_rows<OffT><<<grid_for(n * 32, 256, sms, 16), 256, 0, st>>>(off, n, row.as<int32_t>());
  GI_TRY(key.alloc(m * sizeof(uint32_t)));
  GI_TRY(skey.alloc(m * sizeof(uint32_t)));
  GI_TRY(eid.alloc(m * sizeof(OffT)));
  GI_TRY(order.alloc(m * sizeof(OffT)));
  k_unit_keys<OffT><<<grid_for(m, 256, sms), 256, 0, st>>>(idx, row.as<int32_t>(), m, Z, S, DB, key.as<uint32_t>(),
                                                          eid.as<OffT>());
  int kbits = 1;
  while ((1ll << kbits) < U) ++kbits;
  size_t tb = 0;  // stable LSD radix sort: (v, w) order is kept inside each unit
  GI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.as<uint32_t>(), skey.as<uint32_t>(), eid.as<OffT>(),
                                          order.as<OffT>(), m, 0, kbits, st));
  GI_TRY(tmp.alloc(tb));
  GI_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, key.as<uint32_t>(), skey.as<uint32_t>(), eid.as<OffT>(),
                                          order.as<OffT>(), m, 0, kbits, st));
  key.reset();
  eid.reset();
  GI_TRY(unit_e.alloc((U + 1) * sizeof(int64_t)));
  k_unit_starts<<<grid_for(U + 1, 256, sms), 256, 0, st>>>(skey.as<uint32_t>(), m, U, unit_e.as<int64_t>());
  std::vector<int64_t> h_ue(U + 1);
  GI_CUDA(cudaMemcpyAsync(h_ue.data(), unit_e.p, (U + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  std::vector<int32_t> h_uc(U + 1);
  int64_t C = 0;
  for (int u = 0; u < U; ++u) {
    h_uc[u] = (int32_t)C;
    C += ceil_div(h_ue[u + 1] - h_ue[u], kChunkE);
    if (C >= INT32_MAX) return fail(GI_ERR_UNSUPPORTED, "segmented pull: more than 2^31 chunks");
  }
  h_uc[U] = (int32_t)C;
  const int64_t E = C * kChunkE;
  DevBuf unit_c0, hflag, hc, srow;
  GI_TRY(unit_c0.alloc((U + 1) * sizeof(int32_t)));
  GI_CUDA(cudaMemcpyAsync(unit_c0.p, h_uc.data(), (U + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  GI_TRY(g->seg_idx.alloc(E * sizeof(uint16_t) + 16));
  GI_TRY(hflag.alloc(E * sizeof(int32_t)));
  GI_TRY(srow.alloc(E * sizeof(int32_t)));
  // padding: index Z (reads 0), no head (joins the unit's last piece)
  k_fill_u16<<<grid_for(E, 256, sms), 256, 0, st>>>(g->seg_idx.as<uint16_t>(), E, (uint16_t)Z);
  GI_CUDA(cudaMemsetAsync(hflag.p, 0, E * sizeof(int32_t), st));
  GI_CUDA(cudaMemsetAsync(srow.p, 0, E * sizeof(int32_t), st));
  k_place<OffT><<<grid_for(m, 256, sms), 256, 0, st>>>(skey.as<uint32_t>(), order.as<OffT>(), m, idx,
                                                       row.as<int32_t>(), unit_e.as<int64_t>(),
                                                       unit_c0.as<int32_t>(), Z, S, g->seg_idx.as<uint16_t>(),
                                                       hflag.as<int32_t>(), srow.as<int32_t>());
  skey.reset();
  order.reset();
  row.reset();
  GI_TRY(g->seg_head.alloc((E / 32) * sizeof(uint32_t) + 16));
  k_pack_heads<<<grid_for(E, 256, sms), 256, 0, st>>>(hflag.as<int32_t>(), E, g->seg_head.as<uint32_t>());
  GI_TRY(hc.alloc(E * sizeof(int32_t)));
  tb = 0;
  GI_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, hflag.as<int32_t>(), hc.as<int32_t>(), E, st));
  GI_TRY(tmp.alloc(tb));
  GI_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tb, hflag.as<int32_t>(), hc.as<int32_t>(), E, st));
  int32_t P = 0;
  GI_CUDA(cudaMemcpyAsync(&P, hc.as<int32_t>() + E - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  GI_TRY(g->seg_pdst.alloc(((int64_t)P + 32 * 32) * sizeof(int32_t)));
  GI_CUDA(cudaMemsetAsync(g->seg_pdst.p, 0, ((int64_t)P + 32 * 32) * sizeof(int32_t), st));
  GI_TRY(g->seg_cbase.alloc((C + 1) * sizeof(int32_t)));
  k_pieces<<<grid_for(E, 256, sms), 256, 0, st>>>(hflag.as<int32_t>(), hc.as<int32_t>(), srow.as<int32_t>(), E,
                                                  g->seg_pdst.as<int32_t>(), g->seg_cbase.as<int32_t>());
  GI_CUDA(cudaMemcpyAsync(g->seg_cbase.as<int32_t>() + C, &P, sizeof(int32_t), cudaMemcpyHostToDevice, st));
  GI_TRY(g->seg_rec.alloc(C * kRecBytes + 16));
  k_pack_records<<<grid_for(C * (kRecBytes / 4), 256, sms), 256, 0, st>>>(
      g->seg_idx.as<uint16_t>(), g->seg_head.as<uint32_t>(), g->seg_cbase.as<int32_t>(), hc.as<int32_t>(), C,
      g->seg_rec.as<uint8_t>());
  // cost-balanced CTA ranges: a chunk costs its slots plus kPieceCost per
  // piece ending in it; every unit start adds the cost of staging a segment
  std::vector<int32_t> h_cb(C + 1);
  GI_CUDA(cudaMemcpyAsync(h_cb.data(), g->seg_cbase.p, (C + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  const int ctas = sms;
  std::vector<int32_t> h_cta(ctas + 1, (int32_t)C);
  {
    std::vector<int64_t> pre(C + 1, 0);
    int u = 0;
    for (int64_t c = 0; c < C; ++c) {
      int64_t cost = kChunkCost + (int64_t)kPieceCost * (h_cb[c + 1] - h_cb[c]);
      while (u < U && h_uc[u] < c) ++u;
      if (u < U && h_uc[u] == c) cost += kStageCost;
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
  }
  GI_TRY(g->seg_unit_c0.alloc((U + 1) * sizeof(int32_t)));
  GI_CUDA(cudaMemcpyAsync(g->seg_unit_c0.p, h_uc.data(), (U + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  GI_TRY(g->seg_cta.alloc((ctas + 1) * sizeof(int32_t)));
  GI_CUDA(cudaMemcpyAsync(g->seg_cta.p, h_cta.data(), (ctas + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  g->seg_acc_stride = (n + 64) & ~31ll;
  GI_TRY(g->seg_acc.alloc(2 * g->seg_acc_stride * sizeof(float)));
  GI_CUDA(cudaMemsetAsync(g->seg_acc.p, 0, 2 * g->seg_acc_stride * sizeof(float), st));
  g->seg_acc_cur = 0;
  GI_CUDA(cudaGetLastError());
  GI_CUDA(cudaStreamSynchronize(st));
  g->seg_idx.reset();
  g->seg_head.reset();
  if (const char* dbg = getenv("GI_DEBUG_SEG_LAYOUT")) {
    if (FILE* f = fopen(dbg, "a")) {
      fprintf(f, "n=%lld m=%lld Z=%d S=%d B=%d U=%d C=%lld E=%lld P=%d pad=%.3f\n", (long long)n, (long long)m, Z, S,
              B, U, (long long)C, (long long)E, P, m ? (double)E / (double)m - 1.0 : 0.0);
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

static size_t seg_dyn_smem(int Z) {
  return (size_t)kStages * kStageBytes + (size_t)kConsumers * kScratch * sizeof(float) + ((size_t)Z + 4) * sizeof(float);
}

gi_status seg_build(gi_graph g, int segment_size, int64_t block_rows) {
  if (segment_size < 0 || block_rows < 0) return fail(GI_ERR_INVALID_ARGUMENT, "segment_size / dst_block < 0");
  int optin = 0;
  GI_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, g->ctx->device));
  cudaFuncAttributes a{};
  GI_CUDA(cudaFuncGetAttributes(&a, k_pr_seg<0>));
  int Z = (optin - (int)a.sharedSizeBytes - 64 - (int)seg_dyn_smem(0)) / 4;
  Z = std::min(Z, 65535) & ~31;
  if (Z < 1024) return fail(GI_ERR_UNSUPPORTED, "segmented pull: not enough shared memory");
  if (segment_size > 0) Z = std::max(32, std::min(Z, segment_size) & ~3);
  int64_t DB = block_rows > 0 ? block_rows : kDefaultBlockRows;
  DB = std::max<int64_t>(1, std::min<int64_t>(DB, std::max<int64_t>(g->nr, 1)));
  if (g->seg_Z == Z && g->seg_DB == DB) return GI_OK;
  g->seg_Z = 0;
  if (g->ml == 0 || g->nr == 0) return fail(GI_ERR_UNSUPPORTED, "segmented pull: empty graph");
  if (g->off64) return seg_build_t<int64_t>(g, Z, DB);
  return seg_build_t<int32_t>(g, Z, DB);
}

gi_status seg_edge_pass(gi_graph g, const float* cin) {
  cudaStream_t st = g->ctx->stream;
  SegArgs S;
  S.rec = g->seg_rec.as<uint8_t>();
  S.cbase = g->seg_cbase.as<int32_t>();
  S.pdst = g->seg_pdst.as<int32_t>();
  S.unit_c0 = g->seg_unit_c0.as<int32_t>();
  S.cta_c0 = g->seg_cta.as<int32_t>();
  S.cin = cin;
  S.acc = seg_acc_buf(g, g->seg_acc_cur);
  S.n = g->n;
  S.Z = g->seg_Z;
  S.S = g->seg_S;
  S.U = g->seg_U;
  static const int mode = getenv("GI_SEG_MODE") ? atoi(getenv("GI_SEG_MODE")) : 0;
  void (*kern)(SegArgs) = mode == 1 ? k_pr_seg<1> : mode == 2 ? k_pr_seg<2> : mode == 3 ? k_pr_seg<3> : k_pr_seg<0>;
  const size_t dyn = seg_dyn_smem(g->seg_Z);
  static size_t attr_set = 0;  // largest dynamic smem size configured so far
  if (attr_set < dyn) {
    GI_CUDA(cudaFuncSetAttribute(k_pr_seg<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    GI_CUDA(cudaFuncSetAttribute(k_pr_seg<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    GI_CUDA(cudaFuncSetAttribute(k_pr_seg<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    GI_CUDA(cudaFuncSetAttribute(k_pr_seg<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    attr_set = dyn;
  }
  static const char* dbg = getenv("GI_DEBUG_SEG_TIMING");  // diagnostics: file to append per-CTA timings to
  DevBuf tbuf;
  S.timing = nullptr;
  if (dbg) {
    GI_TRY(tbuf.alloc(4 * g->seg_ctas * sizeof(unsigned long long)));
    GI_CUDA(cudaMemsetAsync(tbuf.p, 0, 4 * g->seg_ctas * sizeof(unsigned long long), st));
    S.timing = tbuf.as<unsigned long long>();
  }
  kern<<<g->seg_ctas, kSegThreads, dyn, st>>>(S);
  GI_CUDA(cudaGetLastError());
  if (dbg) {
    std::vector<unsigned long long> ht(4 * g->seg_ctas);
    std::vector<int32_t> hc(g->seg_ctas + 1);
    GI_CUDA(cudaMemcpyAsync(ht.data(), tbuf.p, ht.size() * 8, cudaMemcpyDeviceToHost, st));
    GI_CUDA(cudaMemcpyAsync(hc.data(), g->seg_cta.p, hc.size() * 4, cudaMemcpyDeviceToHost, st));
    GI_CUDA(cudaStreamSynchronize(st));
    std::vector<int32_t> pc(g->seg_ctas + 1);  // piece index at each CTA boundary
    for (int c = 0; c <= g->seg_ctas; ++c)
      GI_CUDA(cudaMemcpyAsync(&pc[c], g->seg_cbase.as<int32_t>() + hc[c], 4, cudaMemcpyDeviceToHost, st));
    GI_CUDA(cudaStreamSynchronize(st));
    if (FILE* f = fopen(dbg, "a")) {
      for (int c = 0; c < g->seg_ctas; ++c)
        fprintf(f, "%d,%d,%d,%llu,%llu,%llu,%llu,%d\n", c, hc[c], hc[c + 1], ht[4 * c], ht[4 * c + 1], ht[4 * c + 2],
                ht[4 * c + 3], pc[c + 1] - pc[c]);
      fclose(f);
    }
  }
  return GI_OK;
}

gi_status seg_vertex_pass(gi_graph g, const PrArgs& A) {
  cudaStream_t st = g->ctx->stream;
  k_pr_acc<<<grid_for(ceil_div(g->nr, 4), 256, g->ctx->num_sms, 4), 256, 0, st>>>(
      A, seg_acc_buf(g, g->seg_acc_cur), seg_acc_buf(g, g->seg_acc_cur ^ 1));
  GI_CUDA(cudaGetLastError());
  g->seg_acc_cur ^= 1;
  return GI_OK;
}

}  // namespace gi
