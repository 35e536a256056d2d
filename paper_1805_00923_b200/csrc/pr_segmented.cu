// pr_segmented.cu — pull PageRank over shared-memory source segments.
//
// The paper's cache optimisation ("Segmented Subgraphs", PAPER.md P:741-757,
// partition the source range so each segment's
// random reads hit cache, merge the per-segment partial sums) retargeted at
// the B200's 227 KB of shared memory per CTA. Measured on this part
// (tools/microbench/gather_rates.cu, profiles/): random 4-byte gathers run at
// ~1.0 per SM-clock from L2 via LDG but ~7 per SM-clock from shared memory,
// so the pull edge pass (a4) gathers contrib from a staged segment instead of
// from L2. Because a segment holds <= 65536 sources, in-segment source ids are
// 16-bit: the index stream halves from 4 to 2 bytes per edge.
//
// Layout (built once per graph):
//   segment s = sources [s*Z, (s+1)*Z) (internal ids, hottest first)
//   piece     = (segment s, destination v) with >= 1 edge
//   seg_idx16 = edges in (s, v, u) order, u - s*Z as uint16
//   pc_off    = piece offsets into seg_idx16 (segment-major piece order)
//   pc_slot   = the piece's index in destination-major order
//   pstart[v] = first destination-major piece of v
// Per iteration:
//   k_pr_seg   (persistent, one CTA per SM): stage contrib segment in smem,
//              merge-path walk over pieces, write one fp32 partial per piece;
//   k_pr_merge r'[v] = (1-d)/n + d (sum of v's partials + D/n), contrib',
//              dangling mass (fused vertex update, a3).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cub/cub.cuh>
#include <vector>

#include "gi_internal.cuh"
#include "pr_common.cuh"

namespace gi {
namespace {

constexpr int kSegThreads = 512;

// ---------------------------------------------------------------- chunked segment kernel
// Chunked layout (built below from the piece layout): every piece is cut into
// chunks of kChunkE = 4 edges, the last chunk padded with the index Z (a
// shared-memory zero). chunk c holds 4 uint16 source ids (8 bytes) and
// cslot[c] = the piece's destination-major slot, bit 31 set on the piece's
// last chunk. Each segment's chunk list is padded to whole tiles (kTileCh
// chunks), so every tile lies in one segment. CTA c processes the contiguous
// tile range [cta_tiles[c], cta_tiles[c+1]), cut so that every CTA carries the
// same modelled cost (chunks + kTailCost x pieces ending in its tiles).
constexpr int kChunkE = 4;
constexpr int kCPT = 4;                          // chunks per thread per tile
constexpr int kTileCh = kSegThreads * kCPT;      // chunks per tile
constexpr float kTailCost = 0.45f;               // cost of a piece completion, in chunks (fitted from per-CTA timings)

struct SegArgs {
  const uint4* __restrict__ cidx;   // 2 chunks per uint4
  const int4* __restrict__ cslot;   // 4 chunks per int4
  const int32_t* __restrict__ tile_seg;
  const int32_t* __restrict__ cta_tiles;  // CTA c: tiles [cta_tiles[c], cta_tiles[c+1])
  const float* __restrict__ cin;    // padded to a multiple of 4 floats
  float* __restrict__ partial;
  int32_t* __restrict__ carry_slot; // per CTA: piece still open at the CTA's end (-1: none)
  float* __restrict__ carry_val;
  int64_t n;
  int Z;
  unsigned long long* timing;  // optional (GI_DEBUG_SEG_TIMING): per CTA [start, end] globaltimer
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

// Sum of one chunk's 4 staged contributions; padding entries (index Z) are
// skipped (predicated loads: fewer active lanes per shared-memory wavefront).
__device__ __forceinline__ float chunk_sum(const float* sc, uint32_t lo, uint32_t hi, uint32_t Z) {
  const uint32_t i0 = lo & 0xFFFFu, i1 = lo >> 16, i2 = hi & 0xFFFFu, i3 = hi >> 16;
  const float a = sc[i0];
  const float b = i1 != Z ? sc[i1] : 0.f;
  const float c = i2 != Z ? sc[i2] : 0.f;
  const float d = i3 != Z ? sc[i3] : 0.f;
  return (a + b) + (c + d);
}

// Per tile: thread t owns chunks [t*kCPT, (t+1)*kCPT) (32 B of indices, 16 B
// of slots, one vector load each, prefetched one tile ahead). It sums its
// chunks from the staged segment, stores every piece that ends inside its
// window and starts inside it, and hands (slot of its last piece, open
// partial) to a block segmented scan; the first piece that ends in its window
// adds the scan's exclusive prefix. The open piece at the tile end is carried
// to the next tile; at the CTA end it is exported for k_fold_carries.
__global__ void __launch_bounds__(kSegThreads, 1) k_pr_seg(SegArgs A) {
  constexpr int NT = kSegThreads;
  extern __shared__ __align__(128) float scontrib[];  // Z + 4 floats; scontrib[Z] = 0 (chunk padding)
  __shared__ KeyVal scratch[NT / 32];
  __shared__ int s_carry_key;
  __shared__ float s_carry_val;
  __shared__ __align__(8) uint64_t s_bar;
  const int tid = threadIdx.x;
  const uint32_t zpad = (uint32_t)A.Z;
  const int64_t ta = A.cta_tiles[blockIdx.x], tb = A.cta_tiles[blockIdx.x + 1];
  if (ta >= tb) {
    if (tid == 0) A.carry_slot[blockIdx.x] = -1;
    return;
  }
  if (tid == 0 && A.timing) A.timing[2 * blockIdx.x] = globaltimer();
  if (tid == 0) {
    mbar_init(&s_bar, 1);
    scontrib[A.Z] = 0.f;
    s_carry_key = -1;
    s_carry_val = 0.f;
  }
  __syncthreads();
  auto load_segment = [&](int seg) {  // thread 0
    const int64_t base = (int64_t)seg * A.Z;
    const int64_t zlen = min((int64_t)A.Z, A.n - base);
    tma_load_1d(scontrib, A.cin + base, (uint32_t)(((zlen * 4) + 15) & ~15ll), &s_bar);
  };
  int cur_seg = __ldg(&A.tile_seg[ta]);
  if (tid == 0) load_segment(cur_seg);
  uint32_t parity = 0;
  bool pending = true;
  // Register prefetch two tiles ahead (two register sets, the loop unrolled by
  // two so each set stays in place): 4 chunks = 2 x uint4 indices + 1 x int4 slots.
  auto fetch = [&](int64_t t, uint4& a, uint4& b, int4& sl) {
    if (t < tb) {
      const int64_t c = t * kTileCh + (int64_t)tid * kCPT;
      a = __ldg(&A.cidx[c / 2]);
      b = __ldg(&A.cidx[c / 2 + 1]);
      sl = __ldg(&A.cslot[c / 4]);
    }
  };
  auto tile = [&](int64_t t, uint4& pa, uint4& pb, int4& ps) {
    const uint4 ia = pa, ib = pb;
    const int4 sl = ps;
    fetch(t + 2, pa, pb, ps);  // in flight during the next two tiles
    const int next_seg = t + 1 < tb ? __ldg(&A.tile_seg[t + 1]) : cur_seg;
    if (pending) {
      mbar_wait(&s_bar, parity);
      parity ^= 1u;
      pending = false;
    }
    float v[kCPT];
    v[0] = chunk_sum(scontrib, ia.x, ia.y, zpad);
    v[1] = chunk_sum(scontrib, ia.z, ia.w, zpad);
    v[2] = chunk_sum(scontrib, ib.x, ib.y, zpad);
    v[3] = chunk_sum(scontrib, ib.z, ib.w, zpad);
    const int s[kCPT] = {sl.x, sl.y, sl.z, sl.w};
    __syncthreads();  // every read of scontrib for this tile is done
    if (next_seg != cur_seg) {
      cur_seg = next_seg;
      if (tid == 0) load_segment(cur_seg);  // overlaps the rest of this tile
      pending = true;
    }
    const int carry_key = s_carry_key;
    const float carry_val = s_carry_val;
    float acc = 0.f, head_val = 0.f;
    int head = -1;
#pragma unroll
    for (int k = 0; k < kCPT; ++k) {
      acc += v[k];
      if (s[k] < 0) {  // last chunk of its piece
        const int slot = s[k] & 0x7fffffff;
        if (head < 0) {
          head = slot;
          head_val = acc;
        } else {
          A.partial[slot] = acc;
        }
        acc = 0.f;
      }
    }
    const int last_key = s[kCPT - 1] & 0x7fffffff;
    if (tid == 0) {  // fold the carry from the previous tile into the first run
      if (head >= 0) head_val += head == carry_key ? carry_val : 0.f;
      else if (last_key == carry_key) acc += carry_val;
    }
    KeyVal incl;
    const KeyVal ex = seg_scan<NT>(KeyVal{last_key, acc}, incl, scratch);
    if (head >= 0) A.partial[head] = head_val + (tid > 0 && ex.key == head ? ex.val : 0.f);
    if (tid == NT - 1) {
      const bool open = s[kCPT - 1] >= 0;
      s_carry_key = open ? last_key : -1;
      s_carry_val = open ? incl.val : 0.f;
      if (t + 1 == tb) {
        A.carry_slot[blockIdx.x] = open ? last_key : -1;
        A.carry_val[blockIdx.x] = open ? incl.val : 0.f;
      }
    }
  };
  uint4 a0 = make_uint4(0, 0, 0, 0), b0 = a0, a1 = a0, b1 = a0;
  int4 s0 = make_int4(0, 0, 0, 0), s1 = s0;
  fetch(ta, a0, b0, s0);
  fetch(ta + 1, a1, b1, s1);
  for (int64_t t = ta; t < tb; t += 2) {
    tile(t, a0, b0, s0);
    if (t + 1 < tb) tile(t + 1, a1, b1, s1);
  }
  if (tid == 0 && A.timing) A.timing[2 * blockIdx.x + 1] = globaltimer();
}

// partial[carry_slot[c]] += carry_val[c]: pieces cut by CTA boundaries
__global__ void k_fold_carries(const int32_t* __restrict__ slot, const float* __restrict__ val, int C,
                               float* __restrict__ partial) {
  for (int c = threadIdx.x; c < C; c += blockDim.x)
    if (slot[c] >= 0) atomicAdd(&partial[slot[c]], val[c]);
}

template <typename OffT>
__global__ void __launch_bounds__(256) k_pr_merge(PrArgs A, const OffT* __restrict__ pstart,
                                                  const float* __restrict__ partial) {
  // Each thread finishes kV vertices spaced blockDim apart, issuing all their
  // loads before consuming any (independent chains: pstart -> partial, outdeg).
  constexpr int kV = 4;
  __shared__ double sred[32];
  if (blockIdx.x == 0 && threadIdx.x == 0) A.dbuf[(A.it + 2) % 3] = 0.0;
  const double D = A.uniform ? A.dbuf[A.it % 3] : 0.0;
  const float dn = (float)(D * A.inv_n);
  double dpart = 0.0;
  const int64_t span = (int64_t)blockDim.x * kV;
  for (int64_t base = (int64_t)blockIdx.x * span; base < A.n; base += (int64_t)gridDim.x * span) {
    int64_t a[kV], b[kV];
    int od[kV];
#pragma unroll
    for (int k = 0; k < kV; ++k) {
      const int64_t v = base + threadIdx.x + (int64_t)k * blockDim.x;
      a[k] = b[k] = 0;
      od[k] = 0;
      if (v < A.n) {
        a[k] = (int64_t)__ldg(&pstart[v]);
        b[k] = (int64_t)__ldg(&pstart[v + 1]);
        od[k] = __ldg(&A.outdeg[A.row0 + v]);
      }
    }
    float s[kV];
#pragma unroll
    for (int k = 0; k < kV; ++k) s[k] = b[k] > a[k] ? __ldg(&partial[a[k]]) : 0.f;
#pragma unroll
    for (int k = 0; k < kV; ++k) {
      if (b[k] - a[k] > 1) {
        double ds = (double)s[k];
        for (int64_t j = a[k] + 1; j < b[k]; ++j) ds += (double)__ldg(&partial[j]);
        s[k] = (float)ds;
      }
    }
#pragma unroll
    for (int k = 0; k < kV; ++k) {
      const int64_t v = base + threadIdx.x + (int64_t)k * blockDim.x;
      if (v < A.n) {
        const int64_t gv = A.row0 + v;
        const float rn = A.base + A.damp * (s[k] + dn);
        A.cout[gv] = od[k] > 0 ? rn / (float)od[k] : 0.f;
        if (od[k] == 0) dpart += (double)rn;
        if (A.rank_out) A.rank_out[A.perm ? __ldg(&A.perm[gv]) : gv] = rn;
      }
    }
  }
  const double bs = block_sum(dpart, sred);
  if (threadIdx.x == 0 && bs != 0.0) atomicAdd(&A.dbuf[(A.it + 1) % 3], bs);
}

// ---------------------------------------------------------------- layout build
__global__ void k_piece_flags(const int32_t* __restrict__ idx, int64_t m, int Z, int32_t* __restrict__ flag) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e <= m; e += (int64_t)gridDim.x * blockDim.x)
    flag[e] = e == m ? 0 : (e == 0 ? 1 : (idx[e] / Z != idx[e - 1] / Z));
}

template <typename OffT>
__global__ void k_row_start_flags(const OffT* __restrict__ off, int64_t n, int32_t* __restrict__ flag) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    if (off[v] < off[v + 1]) flag[off[v]] = 1;
}

template <typename OffT>
__global__ void k_piece_dm(const int32_t* __restrict__ flag, const OffT* __restrict__ ex, int64_t m,
                           const int32_t* __restrict__ idx, int Z, OffT* __restrict__ pdm, uint32_t* __restrict__ seg,
                           OffT* __restrict__ eid) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    pdm[e] = ex[e] + flag[e] - 1;
    seg[e] = (uint32_t)(idx[e] / Z);
    eid[e] = (OffT)e;
  }
}

template <typename OffT>
__global__ void k_pstart(const OffT* __restrict__ off, const OffT* __restrict__ ex, int64_t n, OffT* __restrict__ pstart) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= n; v += (int64_t)gridDim.x * blockDim.x)
    pstart[v] = ex[off[v]];
}

template <typename OffT>
__global__ void k_seg_gather(const OffT* __restrict__ order, const uint32_t* __restrict__ sseg, int64_t m,
                             const int32_t* __restrict__ idx, const OffT* __restrict__ pdm, int Z,
                             uint16_t* __restrict__ idx16, OffT* __restrict__ spdm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const OffT e = order[i];
    idx16[i] = (uint16_t)(idx[e] - (int64_t)sseg[i] * Z);
    spdm[i] = pdm[e];
  }
}

template <typename OffT>
__global__ void k_piece_start_flags(const OffT* __restrict__ spdm, int64_t m, int32_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = (i == 0) || (spdm[i] != spdm[i - 1]);
}

template <typename OffT>
__global__ void k_piece_slot(const OffT* __restrict__ pc_off, int64_t P, const OffT* __restrict__ spdm,
                             int32_t* __restrict__ slot) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x)
    slot[p] = (int32_t)spdm[pc_off[p]];
}

// seg_e[s] = first position of segment s in the segment-sorted edge array
__global__ void k_seg_starts(const uint32_t* __restrict__ sseg, int64_t m, int S, int64_t* __restrict__ seg_e) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s <= S; s += gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = m;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (sseg[mid] < (uint32_t)s) lo = mid + 1;
      else hi = mid;
    }
    seg_e[s] = lo;
  }
}

template <typename OffT>
__global__ void k_piece_nch(const OffT* __restrict__ pc_off, int64_t P, int64_t* __restrict__ nch) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p <= P; p += (int64_t)gridDim.x * blockDim.x)
    nch[p] = p < P ? ((int64_t)pc_off[p + 1] - (int64_t)pc_off[p] + kChunkE - 1) / kChunkE : 0;
}

// seg_p[s] = first piece of segment s (lower bound of seg_e[s] in pc_off)
template <typename OffT>
__global__ void k_seg_piece_starts(const OffT* __restrict__ pc_off, int64_t P, const int64_t* __restrict__ seg_e,
                                   int S, int64_t* __restrict__ seg_p) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s <= S; s += gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = P;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)pc_off[mid] < seg_e[s]) lo = mid + 1;
      else hi = mid;
    }
    seg_p[s] = lo;
  }
}

__global__ void k_gather_i64(const int64_t* __restrict__ src, const int64_t* __restrict__ at, int k,
                             int64_t* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) out[i] = src[at[i]];
}

// tails[t] = number of pieces ending in tile t (chunks with bit 31 set)
__global__ void __launch_bounds__(256) k_tile_tails(const int32_t* __restrict__ cslot, int32_t* __restrict__ tails) {
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  int c = 0;
  for (int i = threadIdx.x; i < kTileCh; i += blockDim.x) c += cslot[(int64_t)blockIdx.x * kTileCh + i] < 0;
  atomicAdd(&cnt, c);
  __syncthreads();
  if (threadIdx.x == 0) tails[blockIdx.x] = cnt;
}

__global__ void k_fill_pad(uint16_t* __restrict__ cidx, int32_t* __restrict__ cslot, int64_t C, uint16_t pad_idx,
                           int32_t pad_slot) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C; c += (int64_t)gridDim.x * blockDim.x) {
    for (int k = 0; k < kChunkE; ++k) cidx[c * kChunkE + k] = pad_idx;
    cslot[c] = pad_slot;
  }
}

template <typename OffT>
__global__ void k_fill_chunks(const OffT* __restrict__ pc_off, const int32_t* __restrict__ pc_slot,
                              const uint16_t* __restrict__ idx16, int64_t P, const int64_t* __restrict__ cp,
                              const int64_t* __restrict__ seg_p, const int64_t* __restrict__ seg_base, int S, int Z,
                              uint16_t* __restrict__ cidx, int32_t* __restrict__ cslot) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = S - 1;  // segment of p: last s with seg_p[s] <= p
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (seg_p[mid] <= p) lo = mid;
      else hi = mid - 1;
    }
    const int64_t c0 = seg_base[lo] + (cp[p] - cp[seg_p[lo]]);
    const int64_t e0 = pc_off[p], len = (int64_t)pc_off[p + 1] - e0;
    const int64_t nch = (len + kChunkE - 1) / kChunkE;
    const int32_t slot = pc_slot[p];
    for (int64_t j = 0; j < nch; ++j) {
      const int64_t c = c0 + j;
      for (int k = 0; k < kChunkE; ++k) {
        const int64_t e = j * kChunkE + k;
        cidx[c * kChunkE + k] = e < len ? idx16[e0 + e] : (uint16_t)Z;
      }
      cslot[c] = j == nch - 1 ? (int32_t)(slot | 0x80000000u) : slot;
    }
  }
}

}  // namespace

template <typename OffT>
static gi_status seg_build_t(gi_graph g, int Z) {
  gi_context ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  const int64_t n = g->nr, m = g->ml;  // CSC rows (owned destinations) and local edges
  const OffT* off = g->csc_off.as<OffT>();
  const int32_t* idx = g->csc_idx.as<int32_t>();
  const int S = (int)ceil_div(g->n, Z);  // segments over all sources
  // ---- piece layout: (segment, destination) runs of the CSC
  DevBuf flag, ex, pdm, seg, seg2, eid, order, spdm, tmp, nsel, seg_e, pc_off, pc_slot, idx16;
  GI_TRY(flag.alloc((m + 1) * sizeof(int32_t)));
  GI_TRY(ex.alloc((m + 1) * sizeof(OffT)));
  k_piece_flags<<<grid_for(m + 1, 256, sms), 256, 0, st>>>(idx, m, Z, flag.as<int32_t>());
  k_row_start_flags<OffT><<<grid_for(n, 256, sms), 256, 0, st>>>(off, n, flag.as<int32_t>());
  size_t tb = 0;
  GI_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, flag.as<int32_t>(), ex.as<OffT>(), m + 1, st));
  GI_TRY(tmp.alloc(tb));
  GI_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, flag.as<int32_t>(), ex.as<OffT>(), m + 1, st));
  OffT Pt = 0;
  GI_CUDA(cudaMemcpyAsync(&Pt, ex.as<OffT>() + m, sizeof(OffT), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  const int64_t P = (int64_t)Pt;
  if (P >= INT32_MAX) return fail(GI_ERR_UNSUPPORTED, "segmented pull: more than 2^31 pieces");
  GI_TRY(g->seg_pstart.alloc((n + 1) * sizeof(OffT)));
  k_pstart<OffT><<<grid_for(n + 1, 256, sms), 256, 0, st>>>(off, ex.as<OffT>(), n, g->seg_pstart.as<OffT>());
  GI_TRY(pdm.alloc(m * sizeof(OffT)));
  GI_TRY(seg.alloc(m * sizeof(uint32_t)));
  GI_TRY(seg2.alloc(m * sizeof(uint32_t)));
  GI_TRY(eid.alloc(m * sizeof(OffT)));
  GI_TRY(order.alloc(m * sizeof(OffT)));
  k_piece_dm<OffT><<<grid_for(m, 256, sms), 256, 0, st>>>(flag.as<int32_t>(), ex.as<OffT>(), m, idx, Z, pdm.as<OffT>(),
                                                          seg.as<uint32_t>(), eid.as<OffT>());
  ex.reset();
  int sbits = 1;
  while ((1ll << sbits) < S) ++sbits;
  tb = 0;
  GI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, seg.as<uint32_t>(), seg2.as<uint32_t>(), eid.as<OffT>(),
                                          order.as<OffT>(), m, 0, sbits, st));
  GI_TRY(tmp.alloc(tb));
  GI_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, seg.as<uint32_t>(), seg2.as<uint32_t>(), eid.as<OffT>(),
                                          order.as<OffT>(), m, 0, sbits, st));
  eid.reset();
  seg.reset();
  GI_TRY(idx16.alloc((m + 64) * sizeof(uint16_t)));
  GI_TRY(spdm.alloc(m * sizeof(OffT)));
  k_seg_gather<OffT><<<grid_for(m, 256, sms), 256, 0, st>>>(order.as<OffT>(), seg2.as<uint32_t>(), m, idx,
                                                            pdm.as<OffT>(), Z, idx16.as<uint16_t>(), spdm.as<OffT>());
  order.reset();
  pdm.reset();
  k_piece_start_flags<OffT><<<grid_for(m, 256, sms), 256, 0, st>>>(spdm.as<OffT>(), m, flag.as<int32_t>());
  GI_TRY(pc_off.alloc((P + 2) * sizeof(OffT)));
  GI_TRY(nsel.alloc(sizeof(int64_t)));
  cub::CountingInputIterator<OffT> cnt(0);
  tb = 0;
  GI_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, cnt, flag.as<int32_t>(), pc_off.as<OffT>(), nsel.as<int64_t>(), m, st));
  GI_TRY(tmp.alloc(tb));
  GI_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, cnt, flag.as<int32_t>(), pc_off.as<OffT>(), nsel.as<int64_t>(), m, st));
  const OffT mm = (OffT)m;
  GI_CUDA(cudaMemcpyAsync(pc_off.as<OffT>() + P, &mm, sizeof(OffT), cudaMemcpyHostToDevice, st));
  GI_TRY(pc_slot.alloc((P + 1) * sizeof(int32_t)));
  k_piece_slot<OffT><<<grid_for(P, 256, sms), 256, 0, st>>>(pc_off.as<OffT>(), P, spdm.as<OffT>(), pc_slot.as<int32_t>());
  GI_TRY(seg_e.alloc((S + 1) * sizeof(int64_t)));
  k_seg_starts<<<grid_for(S + 1, 256, sms), 256, 0, st>>>(seg2.as<uint32_t>(), m, S, seg_e.as<int64_t>());
  spdm.reset();
  seg2.reset();
  flag.reset();

  // ---- chunked layout
  DevBuf nch, cp, seg_p, cp_at, seg_base;
  GI_TRY(nch.alloc((P + 1) * sizeof(int64_t)));
  GI_TRY(cp.alloc((P + 1) * sizeof(int64_t)));
  k_piece_nch<OffT><<<grid_for(P + 1, 256, sms), 256, 0, st>>>(pc_off.as<OffT>(), P, nch.as<int64_t>());
  tb = 0;
  GI_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, nch.as<int64_t>(), cp.as<int64_t>(), P + 1, st));
  GI_TRY(tmp.alloc(tb));
  GI_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, nch.as<int64_t>(), cp.as<int64_t>(), P + 1, st));
  GI_TRY(seg_p.alloc((S + 1) * sizeof(int64_t)));
  GI_TRY(cp_at.alloc((S + 1) * sizeof(int64_t)));
  k_seg_piece_starts<OffT><<<grid_for(S + 1, 256, sms), 256, 0, st>>>(pc_off.as<OffT>(), P, seg_e.as<int64_t>(), S,
                                                                      seg_p.as<int64_t>());
  k_gather_i64<<<grid_for(S + 1, 256, sms), 256, 0, st>>>(cp.as<int64_t>(), seg_p.as<int64_t>(), S + 1,
                                                          cp_at.as<int64_t>());
  std::vector<int64_t> h_cp_at(S + 1);
  GI_CUDA(cudaMemcpyAsync(h_cp_at.data(), cp_at.p, (S + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  std::vector<int64_t> h_base(S + 1);
  std::vector<int32_t> h_tile_seg;
  int64_t C = 0;
  for (int s = 0; s < S; ++s) {
    h_base[s] = C;
    const int64_t raw = h_cp_at[s + 1] - h_cp_at[s];
    const int64_t tiles = ceil_div(raw, kTileCh);
    for (int64_t t = 0; t < tiles; ++t) h_tile_seg.push_back(s);
    C += tiles * kTileCh;
  }
  h_base[S] = C;
  const int64_t T = (int64_t)h_tile_seg.size();
  GI_TRY(seg_base.alloc((S + 1) * sizeof(int64_t)));
  GI_CUDA(cudaMemcpyAsync(seg_base.p, h_base.data(), (S + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  GI_TRY(g->seg_cidx.alloc((C > 0 ? C : 1) * kChunkE * sizeof(uint16_t)));
  GI_TRY(g->seg_cslot.alloc((C > 0 ? C : 1) * sizeof(int32_t)));
  GI_TRY(g->seg_tiles.alloc((T > 0 ? T : 1) * sizeof(int32_t)));
  if (T > 0)
    GI_CUDA(cudaMemcpyAsync(g->seg_tiles.p, h_tile_seg.data(), T * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  k_fill_pad<<<grid_for(C, 256, sms), 256, 0, st>>>(g->seg_cidx.as<uint16_t>(), g->seg_cslot.as<int32_t>(), C,
                                                    (uint16_t)Z, (int32_t)((uint32_t)P | 0x80000000u));
  k_fill_chunks<OffT><<<grid_for(P, 256, sms), 256, 0, st>>>(
      pc_off.as<OffT>(), pc_slot.as<int32_t>(), idx16.as<uint16_t>(), P, cp.as<int64_t>(), seg_p.as<int64_t>(),
      seg_base.as<int64_t>(), S, Z, g->seg_cidx.as<uint16_t>(), g->seg_cslot.as<int32_t>());
  // cost-balanced CTA ranges over tiles
  std::vector<int32_t> h_tails(T > 0 ? T : 1, 0);
  if (T > 0) {
    DevBuf tails;
    GI_TRY(tails.alloc(T * sizeof(int32_t)));
    k_tile_tails<<<(unsigned)T, 256, 0, st>>>(g->seg_cslot.as<int32_t>(), tails.as<int32_t>());
    GI_CUDA(cudaMemcpyAsync(h_tails.data(), tails.p, T * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    GI_CUDA(cudaStreamSynchronize(st));
  }
  if (const char* dbg = getenv("GI_DEBUG_SEG_TILES")) {  // diagnostics: per-tile segment and piece ends
    if (FILE* f = fopen(dbg, "w")) {
      for (int64_t t = 0; t < T; ++t) fprintf(f, "%lld,%d,%d\n", (long long)t, h_tile_seg[t], h_tails[t]);
      fclose(f);
    }
  }
  std::vector<int32_t> h_cta(sms + 1, 0);
  {
    double total = 0;
    for (int64_t t = 0; t < T; ++t) total += kTileCh + (double)kTailCost * h_tails[t];
    double acc = 0;
    int c = 1;
    for (int64_t t = 0; t < T && c < sms; ++t) {
      acc += kTileCh + (double)kTailCost * h_tails[t];
      while (c < sms && acc >= total * c / sms) h_cta[c++] = (int32_t)(t + 1);
    }
    for (; c <= sms; ++c) h_cta[c] = (int32_t)T;
  }
  GI_TRY(g->seg_cta_tiles.alloc((sms + 1) * sizeof(int32_t)));
  GI_CUDA(cudaMemcpyAsync(g->seg_cta_tiles.p, h_cta.data(), (sms + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  GI_TRY(g->seg_partial.alloc((P + 1) * sizeof(float)));
  GI_TRY(g->seg_carry_slot.alloc(sms * sizeof(int32_t)));
  GI_TRY(g->seg_carry_val.alloc(sms * sizeof(float)));
  GI_CUDA(cudaGetLastError());
  GI_CUDA(cudaStreamSynchronize(st));
  g->seg_Z = Z;
  g->seg_S = S;
  g->seg_P = P;
  g->seg_C = C;
  g->seg_T = T;
  g->seg_ctas = sms;
  return GI_OK;
}

gi_status seg_build(gi_graph g, int segment_size) {
  if (segment_size < 0) return fail(GI_ERR_INVALID_ARGUMENT, "segment_size < 0");
  int optin = 0;
  GI_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, g->ctx->device));
  cudaFuncAttributes a{};
  GI_CUDA(cudaFuncGetAttributes(&a, k_pr_seg));
  int Z = (optin - (int)a.sharedSizeBytes - 64) / 4 - 4;
  Z = std::min(Z, 65535) & ~31;
  if (Z < 1024) return fail(GI_ERR_UNSUPPORTED, "segmented pull: not enough shared memory");
  if (segment_size > 0) Z = std::max(32, std::min(Z, segment_size) & ~3);
  if (g->seg_Z == Z) return GI_OK;
  g->seg_Z = 0;
  if (g->ml == 0 || g->nr == 0) return fail(GI_ERR_UNSUPPORTED, "segmented pull: empty graph");
  if (g->off64) return seg_build_t<int64_t>(g, Z);
  return seg_build_t<int32_t>(g, Z);
}

gi_status seg_edge_pass(gi_graph g, const PrArgs& A) {
  cudaStream_t st = g->ctx->stream;
  SegArgs S;
  S.cidx = g->seg_cidx.as<uint4>();
  S.cslot = g->seg_cslot.as<int4>();
  S.tile_seg = g->seg_tiles.as<int32_t>();
  S.cta_tiles = g->seg_cta_tiles.as<int32_t>();
  S.cin = A.cin;
  S.partial = g->seg_partial.as<float>();
  S.carry_slot = g->seg_carry_slot.as<int32_t>();
  S.carry_val = g->seg_carry_val.as<float>();
  S.n = g->n;
  S.Z = g->seg_Z;
  const size_t dyn = ((size_t)g->seg_Z + 4) * sizeof(float);
  static size_t attr_set = 0;  // largest dynamic smem size configured so far
  if (attr_set < dyn) {
    GI_CUDA(cudaFuncSetAttribute(k_pr_seg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    attr_set = dyn;
  }
  static const char* dbg = getenv("GI_DEBUG_SEG_TIMING");  // diagnostics: file to append per-CTA timings to
  DevBuf tbuf;
  S.timing = nullptr;
  if (dbg) {
    GI_TRY(tbuf.alloc(2 * g->seg_ctas * sizeof(unsigned long long)));
    S.timing = tbuf.as<unsigned long long>();
  }
  k_pr_seg<<<g->seg_ctas, kSegThreads, dyn, st>>>(S);
  if (dbg) {
    std::vector<unsigned long long> ht(2 * g->seg_ctas);
    std::vector<int32_t> hc(g->seg_ctas + 1);
    GI_CUDA(cudaMemcpyAsync(ht.data(), tbuf.p, ht.size() * 8, cudaMemcpyDeviceToHost, st));
    GI_CUDA(cudaMemcpyAsync(hc.data(), g->seg_cta_tiles.p, hc.size() * 4, cudaMemcpyDeviceToHost, st));
    GI_CUDA(cudaStreamSynchronize(st));
    if (FILE* f = fopen(dbg, "a")) {
      for (int c = 0; c < g->seg_ctas; ++c)
        fprintf(f, "%d,%d,%d,%llu,%llu\n", c, hc[c], hc[c + 1], ht[2 * c], ht[2 * c + 1]);
      fclose(f);
    }
  }
  k_fold_carries<<<1, 256, 0, st>>>(S.carry_slot, S.carry_val, g->seg_ctas, S.partial);
  GI_CUDA(cudaGetLastError());
  return GI_OK;
}

gi_status seg_vertex_pass(gi_graph g, const PrArgs& A) {
  cudaStream_t st = g->ctx->stream;
  if (g->off64)
    k_pr_merge<int64_t><<<grid_for(ceil_div(g->nr, 4), 256, g->ctx->num_sms, 8), 256, 0, st>>>(A, g->seg_pstart.as<int64_t>(),
                                                                                   g->seg_partial.as<float>());
  else
    k_pr_merge<int32_t><<<grid_for(ceil_div(g->nr, 4), 256, g->ctx->num_sms, 8), 256, 0, st>>>(A, g->seg_pstart.as<int32_t>(),
                                                                                   g->seg_partial.as<float>());
  GI_CUDA(cudaGetLastError());
  return GI_OK;
}

}  // namespace gi
