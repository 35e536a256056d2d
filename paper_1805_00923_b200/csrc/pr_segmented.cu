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
#include <cub/cub.cuh>
#include <vector>

#include "gi_internal.cuh"
#include "pr_common.cuh"

namespace gi {
namespace {

constexpr int kSegThreads = 512;
constexpr int kSegIPT = 16;
constexpr int kSegTile = kSegThreads * kSegIPT;  // merge items per tile
constexpr int kSegRows = kSegTile / 2 + 2;       // max pieces touching a tile (>= 2 items each)

struct SegTile {
  int64_t pos;  // first merge position
  int32_t r0;   // piece containing pos
  int32_t r1;   // piece containing the tile's last position
  int32_t seg;
  int32_t pad;
};

// dynamic smem besides the contrib segment: loff | sval | spart
__host__ __device__ constexpr int seg_loff_bytes() { return ((kSegRows + 1) * 4 + 15) / 16 * 16; }
constexpr int seg_fixed_dyn_bytes() { return seg_loff_bytes() + kSegTile * 4 + ((kSegRows * 4 + 15) / 16 * 16); }

template <typename OffT>
struct SegArgs {
  const SegTile* __restrict__ tiles;
  const int32_t* __restrict__ cta_tiles;
  const OffT* __restrict__ pc_off;
  const int32_t* __restrict__ pc_slot;
  const uint16_t* __restrict__ idx16;
  const float* __restrict__ cin;  // padded to a multiple of 4 floats
  float* __restrict__ partial;
  int64_t n, m;
  int Z;
};

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

// Persistent: CTA c processes tiles [cta_tiles[c], cta_tiles[c+1]) in order.
// Software pipeline per tile t:
//   regs(t) -> smem offsets | sync | issue loads of tile t+1 into regs |
//   gather sval from the staged segment | sync | TMA next segment if it
//   changes (overlaps the walk) | merge-path walk -> spart | sync | write
//   the tile's completed piece partials (slot list held in registers).
template <typename OffT>
__global__ void __launch_bounds__(kSegThreads, 1) k_pr_seg(SegArgs<OffT> A) {
  constexpr int NT = kSegThreads, IPT = kSegIPT, TT = kSegTile;
  constexpr int RPT = (kSegRows + 1 + NT - 1) / NT;  // piece entries per thread
  extern __shared__ __align__(128) unsigned char dyn_smem[];
  int* loff = reinterpret_cast<int*>(dyn_smem);
  float* sval = reinterpret_cast<float*>(dyn_smem + seg_loff_bytes());
  float* spart = sval + TT;
  float* scontrib = reinterpret_cast<float*>(dyn_smem + seg_fixed_dyn_bytes());
  __shared__ KeyVal scratch[NT / 32];
  __shared__ float s_carry;
  __shared__ __align__(8) uint64_t s_bar;
  const int tid = threadIdx.x;
  const int t0 = A.cta_tiles[blockIdx.x], t1 = A.cta_tiles[blockIdx.x + 1];
  if (t0 >= t1) return;
  if (tid == 0) mbar_init(&s_bar, 1);
  __syncthreads();

  auto load_segment = [&](int seg) {  // thread 0
    const int64_t base = (int64_t)seg * A.Z;
    const int64_t zlen = min((int64_t)A.Z, A.n - base);
    tma_load_1d(scontrib, A.cin + base, (uint32_t)(((zlen * 4) + 15) & ~15ll), &s_bar);
  };
  uint16_t pidx[IPT];
  int poff[RPT];
  int32_t pslot[RPT];
  auto prefetch = [&](const SegTile& T, int items) {
    const int64_t r0 = T.r0;
    const int R = T.r1 - T.r0 + 1;
    const int64_t eb = T.pos - r0;
    const int lim = (int)min((int64_t)items, A.m - eb);
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      const int i = tid + k * NT;
      const int64_t v = i <= R ? (int64_t)__ldg(&A.pc_off[r0 + i]) - eb : 0;
      poff[k] = (int)max((int64_t)-1, min(v, (int64_t)items + 1));
      pslot[k] = i < R ? __ldg(&A.pc_slot[r0 + i]) : 0;
    }
    const uint16_t* src = A.idx16 + eb;
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      const int j = tid + k * NT;
      pidx[k] = j < lim ? __ldg(&src[j]) : (uint16_t)0;
    }
  };

  SegTile Tn = A.tiles[t0];
  int items_n = (int)(A.tiles[t0 + 1].pos - Tn.pos);
  int cur_seg = Tn.seg;
  if (tid == 0) load_segment(cur_seg);
  bool seg_pending = true;
  uint32_t parity = 0;
  prefetch(Tn, items_n);

  for (int t = t0; t < t1; ++t) {
    const SegTile T = Tn;
    const int items = items_n;
    const int R = T.r1 - T.r0 + 1;
    if (t + 1 < t1) {
      Tn = A.tiles[t + 1];
      items_n = (int)(A.tiles[t + 2].pos - Tn.pos);
    }
    uint16_t cidx[IPT];
    int32_t cslot[RPT];
#pragma unroll
    for (int k = 0; k < IPT; ++k) cidx[k] = pidx[k];
#pragma unroll
    for (int k = 0; k < RPT; ++k) cslot[k] = pslot[k];
    __syncthreads();  // the previous tile's write-out is done with loff
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      const int i = tid + k * NT;
      if (i <= R) loff[i] = poff[k];
    }
    const float carry_in = s_carry;
    __syncthreads();  // loff visible
    const int ne = min(loff[R], items - (R - 1));
    if (t + 1 < t1) prefetch(Tn, items_n);  // in flight during this tile
    if (seg_pending) {
      mbar_wait(&s_bar, parity);
      parity ^= 1u;
      seg_pending = false;
    }
#pragma unroll
    for (int k = 0; k < IPT; ++k) {
      const int j = tid + k * NT;
      if (j < ne) sval[j] = scontrib[cidx[k]];
    }
    __syncthreads();  // sval ready; every read of scontrib for this tile is done
    if (t + 1 < t1 && Tn.seg != cur_seg) {
      cur_seg = Tn.seg;
      if (tid == 0) load_segment(cur_seg);  // overlaps the walk below
      seg_pending = true;
    }
    tile_walk<NT, IPT>(
        loff, R, items, sval, scratch, [&](int i, float v) { spart[i] = v; },
        [&](int i, float v) {
          const float tot = v + (loff[i] < 0 ? carry_in : 0.f);
          if (i + loff[i + 1] < items) spart[i] = tot;
          else s_carry = tot;  // piece continues in this CTA's next tile
        });
    __syncthreads();  // spart ready
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
      const int i = tid + k * NT;
      if (i < R && i + loff[i + 1] < items) A.partial[cslot[k]] = spart[i];
    }
  }
}

template <typename OffT>
__global__ void __launch_bounds__(256) k_pr_merge(PrArgs A, const OffT* __restrict__ pstart,
                                                  const float* __restrict__ partial) {
  __shared__ double sred[32];
  if (blockIdx.x == 0 && threadIdx.x == 0) A.dbuf[(A.it + 2) % 3] = 0.0;
  const double D = A.uniform ? A.dbuf[A.it % 3] : 0.0;
  const float dn = (float)(D * A.inv_n);
  double dpart = 0.0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < A.n; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = pstart[v], b = pstart[v + 1];
    float s = 0.f;
    if (b - a == 1) {
      s = __ldg(&partial[a]);
    } else {
      double ds = 0.0;
      for (int64_t j = a; j < b; ++j) ds += (double)__ldg(&partial[j]);
      s = (float)ds;
    }
    pr_epilogue(A, v, s, dn, dpart);
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

}  // namespace

template <typename OffT>
static gi_status seg_build_t(gi_graph g, int Z) {
  gi_context ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  const int64_t n = g->n, m = g->m;
  const OffT* off = g->csc_off.as<OffT>();
  const int32_t* idx = g->csc_idx.as<int32_t>();
  const int S = (int)ceil_div(n, Z);
  DevBuf flag, ex, pdm, seg, seg2, eid, order, spdm, tmp, nsel, seg_e;
  GI_TRY(flag.alloc((m + 1) * sizeof(int32_t)));
  GI_TRY(ex.alloc((m + 1) * sizeof(OffT)));
  k_piece_flags<<<grid_for(m + 1, 256, sms), 256, 0, st>>>(idx, m, Z, flag.as<int32_t>());
  k_row_start_flags<OffT><<<grid_for(n, 256, sms), 256, 0, st>>>(off, n, flag.as<int32_t>());
  size_t tb = 0;
  GI_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, flag.as<int32_t>(), ex.as<OffT>(), m + 1, st));
  GI_TRY(tmp.alloc(tb));
  GI_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, flag.as<int32_t>(), ex.as<OffT>(), m + 1, st));
  OffT P = 0;
  GI_CUDA(cudaMemcpyAsync(&P, ex.as<OffT>() + m, sizeof(OffT), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  GI_TRY(g->seg_pstart.alloc((n + 1) * sizeof(OffT)));
  k_pstart<OffT><<<grid_for(n + 1, 256, sms), 256, 0, st>>>(off, ex.as<OffT>(), n, g->seg_pstart.as<OffT>());
  GI_TRY(pdm.alloc(m * sizeof(OffT)));
  GI_TRY(seg.alloc(m * sizeof(uint32_t)));
  GI_TRY(seg2.alloc(m * sizeof(uint32_t)));
  GI_TRY(eid.alloc(m * sizeof(OffT)));
  GI_TRY(order.alloc(m * sizeof(OffT)));
  k_piece_dm<OffT><<<grid_for(m, 256, sms), 256, 0, st>>>(flag.as<int32_t>(), ex.as<OffT>(), m, idx, Z, pdm.as<OffT>(),
                                                          seg.as<uint32_t>(), eid.as<OffT>());
  int sbits = 1;
  while ((1ll << sbits) < S) ++sbits;
  tb = 0;
  GI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, seg.as<uint32_t>(), seg2.as<uint32_t>(), eid.as<OffT>(),
                                          order.as<OffT>(), m, 0, sbits, st));
  GI_TRY(tmp.alloc(tb));
  GI_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, seg.as<uint32_t>(), seg2.as<uint32_t>(), eid.as<OffT>(),
                                          order.as<OffT>(), m, 0, sbits, st));
  GI_TRY(g->seg_idx16.alloc((m + 64) * sizeof(uint16_t)));
  GI_TRY(spdm.alloc(m * sizeof(OffT)));
  k_seg_gather<OffT><<<grid_for(m, 256, sms), 256, 0, st>>>(order.as<OffT>(), seg2.as<uint32_t>(), m, idx,
                                                            pdm.as<OffT>(), Z, g->seg_idx16.as<uint16_t>(),
                                                            spdm.as<OffT>());
  // piece starts in segment-major order
  k_piece_start_flags<OffT><<<grid_for(m, 256, sms), 256, 0, st>>>(spdm.as<OffT>(), m, flag.as<int32_t>());
  GI_TRY(g->seg_pc_off.alloc(((int64_t)P + 2) * sizeof(OffT)));
  GI_TRY(nsel.alloc(sizeof(int64_t)));
  cub::CountingInputIterator<OffT> cnt(0);
  tb = 0;
  GI_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, cnt, flag.as<int32_t>(), g->seg_pc_off.as<OffT>(), nsel.as<int64_t>(),
                                     m, st));
  GI_TRY(tmp.alloc(tb));
  GI_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, cnt, flag.as<int32_t>(), g->seg_pc_off.as<OffT>(), nsel.as<int64_t>(),
                                     m, st));
  const OffT mm = (OffT)m;
  GI_CUDA(cudaMemcpyAsync(g->seg_pc_off.as<OffT>() + P, &mm, sizeof(OffT), cudaMemcpyHostToDevice, st));
  GI_TRY(g->seg_pc_slot.alloc(((int64_t)P + 1) * sizeof(int32_t)));
  k_piece_slot<OffT><<<grid_for(P, 256, sms), 256, 0, st>>>(g->seg_pc_off.as<OffT>(), P, spdm.as<OffT>(),
                                                            g->seg_pc_slot.as<int32_t>());
  GI_TRY(seg_e.alloc((S + 1) * sizeof(int64_t)));
  k_seg_starts<<<grid_for(S + 1, 256, sms), 256, 0, st>>>(seg2.as<uint32_t>(), m, S, seg_e.as<int64_t>());
  GI_CUDA(cudaGetLastError());

  // ---- host tile planning (native runtime: merge-path cuts, one CTA per SM)
  std::vector<OffT> h_off((size_t)P + 1);
  std::vector<int64_t> h_seg_e(S + 1);
  GI_CUDA(cudaMemcpyAsync(h_off.data(), g->seg_pc_off.p, ((size_t)P + 1) * sizeof(OffT), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaMemcpyAsync(h_seg_e.data(), seg_e.p, (S + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  const int64_t PP = (int64_t)P;
  const int64_t I = PP + m;
  auto pe = [&](int64_t p) { return p + (int64_t)h_off[p + 1]; };
  auto ps = [&](int64_t p) { return p + (int64_t)h_off[p]; };
  auto piece_at = [&](int64_t x) {  // min p with pe(p) >= x
    int64_t lo = 0, hi = PP - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (pe(mid) >= x) hi = mid;
      else lo = mid + 1;
    }
    return lo;
  };
  std::vector<int64_t> seg_p(S + 1);  // first piece of each segment
  for (int s = 0; s <= S; ++s) {
    int64_t lo = 0, hi = PP;  // lower_bound(h_off[0..P), seg_e[s])
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)h_off[mid] < h_seg_e[s]) lo = mid + 1;
      else hi = mid;
    }
    seg_p[s] = lo;
  }
  const int C = sms;
  std::vector<int64_t> cuts(C + 1, 0);
  cuts[C] = I;
  for (int c = 1; c < C; ++c) {
    const int64_t target = (int64_t)((__int128)I * c / C);
    int64_t cut = PP > 0 ? pe(piece_at(target)) + 1 : 0;
    cut = std::min(std::max(cut, cuts[c - 1]), I);
    cuts[c] = cut;
  }
  std::vector<SegTile> tiles;
  std::vector<int32_t> cta_tiles(C + 1);
  tiles.reserve((size_t)(I / kSegTile + 2 * (S + C) + 2));
  int seg_cur = 0;
  for (int c = 0; c < C; ++c) {
    cta_tiles[c] = (int32_t)tiles.size();
    int64_t pos = cuts[c];
    while (pos < cuts[c + 1]) {
      const int64_t p = piece_at(pos);
      while (seg_cur + 1 <= S && seg_p[seg_cur + 1] <= p) ++seg_cur;
      const int64_t seg_end = seg_p[seg_cur + 1] >= PP ? I : ps(seg_p[seg_cur + 1]);
      const int64_t end = std::min(std::min(pos + (int64_t)kSegTile, cuts[c + 1]), seg_end);
      SegTile T;
      T.pos = pos;
      T.r0 = (int32_t)p;
      T.r1 = (int32_t)piece_at(end - 1);
      T.seg = seg_cur;
      T.pad = 0;
      tiles.push_back(T);
      pos = end;
    }
  }
  cta_tiles[C] = (int32_t)tiles.size();
  tiles.push_back(SegTile{I, 0, 0, 0, 0});
  GI_TRY(g->seg_tiles.alloc(tiles.size() * sizeof(SegTile)));
  GI_TRY(g->seg_cta_tiles.alloc((C + 1) * sizeof(int32_t)));
  GI_CUDA(cudaMemcpyAsync(g->seg_tiles.p, tiles.data(), tiles.size() * sizeof(SegTile), cudaMemcpyHostToDevice, st));
  GI_CUDA(cudaMemcpyAsync(g->seg_cta_tiles.p, cta_tiles.data(), (C + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  GI_TRY(g->seg_partial.alloc(((int64_t)P + 1) * sizeof(float)));
  GI_CUDA(cudaStreamSynchronize(st));
  g->seg_Z = Z;
  g->seg_S = S;
  g->seg_P = PP;
  g->seg_ctas = C;
  return GI_OK;
}

static int seg_static_smem() {
  cudaFuncAttributes a{};
  cudaFuncGetAttributes(&a, k_pr_seg<int32_t>);
  cudaFuncAttributes b{};
  cudaFuncGetAttributes(&b, k_pr_seg<int64_t>);
  return (int)std::max(a.sharedSizeBytes, b.sharedSizeBytes) + seg_fixed_dyn_bytes();
}

gi_status seg_build(gi_graph g, int segment_size) {
  if (segment_size < 0) return fail(GI_ERR_INVALID_ARGUMENT, "segment_size < 0");
  int optin = 0;
  GI_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, g->ctx->device));
  int Z = (optin - seg_static_smem() - 1024) / 4;
  Z = std::min(Z, 65536) & ~31;
  if (Z < 1024) return fail(GI_ERR_UNSUPPORTED, "segmented pull: not enough shared memory");
  if (segment_size > 0) Z = std::min(Z, segment_size);
  if (g->seg_Z == Z) return GI_OK;
  g->seg_Z = 0;
  if (g->m == 0 || g->n == 0) return fail(GI_ERR_UNSUPPORTED, "segmented pull: empty graph");
  if (g->off64) return seg_build_t<int64_t>(g, Z);
  return seg_build_t<int32_t>(g, Z);
}

template <typename OffT>
static gi_status seg_iter_t(gi_graph g, const PrArgs& A) {
  cudaStream_t st = g->ctx->stream;
  SegArgs<OffT> S;
  S.tiles = g->seg_tiles.as<SegTile>();
  S.cta_tiles = g->seg_cta_tiles.as<int32_t>();
  S.pc_off = g->seg_pc_off.as<OffT>();
  S.pc_slot = g->seg_pc_slot.as<int32_t>();
  S.idx16 = g->seg_idx16.as<uint16_t>();
  S.cin = A.cin;
  S.partial = g->seg_partial.as<float>();
  S.n = g->n;
  S.m = g->m;
  S.Z = g->seg_Z;
  const size_t dyn = (size_t)g->seg_Z * sizeof(float) + seg_fixed_dyn_bytes();
  static size_t attr_set[2] = {0, 0};  // largest dynamic smem size configured so far
  const int k = sizeof(OffT) == 8;
  if (attr_set[k] < dyn) {
    GI_CUDA(cudaFuncSetAttribute(k_pr_seg<OffT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    attr_set[k] = dyn;
  }
  k_pr_seg<OffT><<<g->seg_ctas, kSegThreads, dyn, st>>>(S);
  GI_CUDA(cudaGetLastError());
  return GI_OK;
}

template <typename OffT>
static gi_status seg_merge_t(gi_graph g, const PrArgs& A) {
  cudaStream_t st = g->ctx->stream;
  k_pr_merge<OffT><<<grid_for(g->n, 256, g->ctx->num_sms, 16), 256, 0, st>>>(A, g->seg_pstart.as<OffT>(),
                                                                              g->seg_partial.as<float>());
  GI_CUDA(cudaGetLastError());
  return GI_OK;
}

gi_status seg_edge_pass(gi_graph g, const PrArgs& A) {
  if (g->off64) return seg_iter_t<int64_t>(g, A);
  return seg_iter_t<int32_t>(g, A);
}

gi_status seg_vertex_pass(gi_graph g, const PrArgs& A) {
  if (g->off64) return seg_merge_t<int64_t>(g, A);
  return seg_merge_t<int32_t>(g, A);
}

}  // namespace gi
