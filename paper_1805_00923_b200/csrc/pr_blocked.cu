// pr_blocked.cu — pull PageRank by propagation blocking, for graphs whose
// in-edges do not cluster by source (the low-locality
// regime of config 5, RMAT a = 0.45 symmetrised).
//
// The paper's cache optimisation partitions the source range so each
// segment's random reads hit cache and then merges the per-segment partial
// sums; it cites propagation blocking
// (Beamer et al. 2017) as the write-side counterpart. On B200 the
// segmented pull (pr_segmented.cu) folds each (segment, destination) piece into
// an L2-resident accumulator with one RED; when a piece holds ~1.6 edges (config
// 5) that is one random RED per edge and the pass runs at ~0.09 of the HBM
// roofline. Here the edges are binned twice instead, and every HBM access is a
// stream:
//
//   tile (s, d) = the in-edges whose source lies in chunk s (C consecutive
//   sources, staged in shared memory) and whose destination lies in row block
//   d (at most B rows, at most ~2 m / (rows / B) edges: blocks are cut by edge
//   count too, so hub rows do not make one block the whole pass). Tiles are laid
//   out chunk-major, [s][d], each padded to a multiple of 8 edges:
//     src16[e]  = source - s*C (16 bits; C for padding: the zero slot)
//     dst16[e]  = row - rb[d]  (16 bits; the block's trash row for padding)
//   Per iteration:
//   k_pb_scatter  work item (s, e0, e1) (a chunk's tiles, split into ranges of
//                 ~W edges): stage contrib[chunk] in shared memory, then
//                 vals[e] = contrib[s*C + src16[e]] for e in [e0, e1) — a pure
//                 streaming map (2 B read + 4 B written per edge).
//   k_pb_gather   CTA per row block d: acc[rows] in shared memory; the block's
//                 runs (s, d) over all s, flattened into one group space split
//                 evenly over the warps (4 B + 2 B read per edge), runs of one
//                 destination summed in registers and across lanes, then added
//                 as 64-bit fixed point with native 32-bit shared atomics (low
//                 word + carry into the high word: exact integer sums, where
//                 an fp32 shared atomic add is a CAS loop); then the fused
//                 vertex update a3 (pr_epilogue) for the block's rows.
// 12 bytes per edge of HBM traffic, all sequential, instead of one random
// 32-byte sector (gather) or one random RED (segmented) per edge.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cub/device/device_scan.cuh>
#include <vector>

#include "gi_internal.cuh"
#include "pr_common.cuh"

namespace gi {
namespace {

constexpr int kPbThreads = 1024;
constexpr int kPbC = 49152;          // sources per chunk (16-bit local ids; 192 KB of staged contrib)
constexpr int kPbB = 24576;          // rows per block (two 32-bit accumulator words per row: 192 KB)
constexpr int kPbMaxChunks = 2048;   // k_pb_gather keeps one run start + prefix per chunk in smem
constexpr int kPbGroup = 8;          // edges per group (one 16-byte index load, two 16-byte value stores)

struct PbArgs {
  const uint16_t* __restrict__ src16;
  const uint16_t* __restrict__ dst16;
  float* __restrict__ vals;
  const int64_t* __restrict__ tstart;  // Ks * Kd + 1 tile starts ([s][d] order), multiples of 8
  const int64_t* __restrict__ items;   // 3 per scatter work item: chunk, first edge, end edge
  const int64_t* __restrict__ rb;      // Kd + 1 row-block bounds (local rows)
  const float* __restrict__ cin;       // contrib by global source id
  int64_t n;                           // global sources
  int Ks, Kd;
};

// streamed once per pass: cache-streaming loads (ld.global.cs)
__device__ __forceinline__ uint4 ld_stream16(const void* p) { return __ldcs(reinterpret_cast<const uint4*>(p)); }
__device__ __forceinline__ float4 ld_stream16f(const void* p) { return __ldcs(reinterpret_cast<const float4*>(p)); }

// phase 1: vals[e] = contrib[chunk base + src16[e]] over a work item's edges
__global__ void __launch_bounds__(kPbThreads, 1) k_pb_scatter(PbArgs P) {
  extern __shared__ __align__(16) float sc[];  // kPbC + 4
  const int64_t s = P.items[3 * blockIdx.x];
  const int64_t e0 = P.items[3 * blockIdx.x + 1], e1 = P.items[3 * blockIdx.x + 2];
  const int64_t base = s * kPbC;
  const int64_t len = min((int64_t)kPbC, P.n - base);
  for (int64_t i = threadIdx.x; i < len; i += blockDim.x) sc[i] = __ldg(&P.cin[base + i]);
  if (threadIdx.x == 0) sc[kPbC] = 0.f;  // padding slots read the zero slot
  __syncthreads();
  const int64_t ng = (e1 - e0) / kPbGroup;
  const uint16_t* src = P.src16 + e0;
  float* out = P.vals + e0;
#ifndef GI_PB_U
#define GI_PB_U 2
#endif
  constexpr int U = GI_PB_U;  // groups per thread in flight
  int64_t g = threadIdx.x;
  for (; g + (U - 1) * kPbThreads < ng; g += U * kPbThreads) {
    uint4 q[U];
#pragma unroll
    for (int k = 0; k < U; ++k) q[k] = ld_stream16(src + 8 * (g + k * kPbThreads));
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const float4 a = make_float4(sc[q[k].x & 0xFFFFu], sc[q[k].x >> 16], sc[q[k].y & 0xFFFFu], sc[q[k].y >> 16]);
      const float4 b = make_float4(sc[q[k].z & 0xFFFFu], sc[q[k].z >> 16], sc[q[k].w & 0xFFFFu], sc[q[k].w >> 16]);
      float4* o = reinterpret_cast<float4*>(out + 8 * (g + k * kPbThreads));
      __stcs(o, a);
      __stcs(o + 1, b);
    }
  }
  for (; g < ng; g += kPbThreads) {
    const uint4 q = ld_stream16(src + 8 * g);
    float4* o = reinterpret_cast<float4*>(out + 8 * g);
    __stcs(o, make_float4(sc[q.x & 0xFFFFu], sc[q.x >> 16], sc[q.y & 0xFFFFu], sc[q.y >> 16]));
    __stcs(o + 1, make_float4(sc[q.z & 0xFFFFu], sc[q.z >> 16], sc[q.w & 0xFFFFu], sc[q.w >> 16]));
  }
}

// phase 2: CTA per row block; acc in smem, runs (s, d) flattened over the warps,
// then the fused vertex update of the block's rows
__global__ void __launch_bounds__(kPbThreads, 1) k_pb_gather(PbArgs P, PrArgs A) {
  // row sums as 64-bit fixed point (2^-62 units, exact integer adds) in two 32-bit words:
  // shared memory has a native 32-bit atomic add but none for fp32 (a CAS loop)
  extern __shared__ __align__(16) uint32_t lo[];  // kPbB + 4 low words | kPbB + 4 high words | prefix | starts
  __shared__ double sred[32];
  uint32_t* hi = lo + kPbB + 4;
  int32_t* pre = reinterpret_cast<int32_t*>(hi + kPbB + 4);
  int64_t* rs = reinterpret_cast<int64_t*>(pre + ((P.Ks + 2) & ~1));
  const int d = blockIdx.x;
  const int64_t r0 = P.rb[d], nrow = P.rb[d + 1] - r0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i <= kPbB; i += kPbThreads) {
    lo[i] = 0u;
    hi[i] = 0u;
  }
  // add X >= 0 (X * 2^62 < 2^64: a row's sum never exceeds the total rank mass 1)
  auto add = [&](uint32_t k, float X) {
    const unsigned long long x = __float2ull_rn(X * 0x1p62f);
    const uint32_t l = (uint32_t)x, h = (uint32_t)(x >> 32);
    const uint32_t old = atomicAdd(&lo[k], l);
    const uint32_t c = (uint32_t)(old + l < old);  // carry out of the low word
    if (h + c) atomicAdd(&hi[k], h + c);
  };
  // group counts of the block's runs, then an exclusive prefix (one warp)
  for (int s = tid; s < P.Ks; s += kPbThreads) {
    const int64_t a = P.tstart[(int64_t)s * P.Kd + d], b = P.tstart[(int64_t)s * P.Kd + d + 1];
    rs[s] = a;
    pre[s + 1] = (int32_t)((b - a) / kPbGroup);
  }
  __syncthreads();
  if (warp == 0) {
    int32_t run = 0;
    for (int s0 = 0; s0 < P.Ks; s0 += 32) {
      const int s = s0 + lane;
      int32_t v = s < P.Ks ? pre[s + 1] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      if (s < P.Ks) pre[s + 1] = run + v;
      run += __shfl_sync(0xffffffffu, v, 31);
    }
    if (lane == 0) pre[0] = 0;
  }
  __syncthreads();
  const int32_t G = pre[P.Ks];
  const int nw = kPbThreads / 32;
  const int32_t g0 = (int32_t)((int64_t)G * warp / nw), g1 = (int32_t)((int64_t)G * (warp + 1) / nw);
  // the run of the warp's first group (binary search over the prefix)
  int s = 0;
  {
    int lo = 0, hi = P.Ks;  // largest s with pre[s] <= g0
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (pre[mid] <= g0) lo = mid;
      else hi = mid;
    }
    s = lo;
  }
  // the next group's loads are issued before this group's shared-memory atomics
  auto locate = [&](int32_t g) -> int64_t {
    while (pre[s + 1] <= g) ++s;  // the run (s, d) holding group g (monotone within the lane)
    return rs[s] + (int64_t)(g - pre[s]) * kPbGroup;
  };
  uint4 q = make_uint4(0, 0, 0, 0);
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
  if (g0 + lane < g1) {
    const int64_t e = locate(g0 + lane);
    q = ld_stream16(P.dst16 + e);
    a = ld_stream16f(P.vals + e);
    b = ld_stream16f(P.vals + e + 4);
  }
  for (int32_t gb = g0; gb < g1; gb += 32) {
    const bool mine = gb + lane < g1;
    const uint4 qc = q;
    const float4 ac = a, bc = b;
    if (gb + 32 + lane < g1) {  // prefetch the lane's next group
      const int64_t e = locate(gb + 32 + lane);
      q = ld_stream16(P.dst16 + e);
      a = ld_stream16f(P.vals + e);
      b = ld_stream16f(P.vals + e + 4);
    }
    uint32_t key = 0xFFFFFFFFu;  // the destination of this lane's last run (none: unique sentinel)
    float X = 0.f;
    if (mine) {
      const uint32_t k8[8] = {qc.x & 0xFFFFu, qc.x >> 16, qc.y & 0xFFFFu, qc.y >> 16,
                              qc.z & 0xFFFFu, qc.z >> 16, qc.w & 0xFFFFu, qc.w >> 16};
      const float v8[8] = {ac.x, ac.y, ac.z, ac.w, bc.x, bc.y, bc.z, bc.w};
      // tiles are sorted by destination: runs of equal keys are summed in registers;
      // every run but the last is added now
      key = k8[0];
      X = v8[0];
#pragma unroll
      for (int k = 1; k < 8; ++k) {
        if (k8[k] == key) {
          X += v8[k];
        } else {
          add(key, X);
          key = k8[k];
          X = v8[k];
        }
      }
    }
    // the lanes' last runs: equal keys on consecutive lanes (a hub row's groups) are
    // summed by a segmented scan; the segment's last lane adds the total
    const uint32_t kprev = __shfl_up_sync(0xffffffffu, key, 1);
    const uint32_t heads = __ballot_sync(0xffffffffu, lane == 0 || kprev != key);
    if (heads != 0xFFFFFFFFu) {  // some lanes continue their left neighbour's run: merge (warp-uniform)
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, X, o);
        if (lane >= o && ((heads >> (lane - o + 1)) & ((1u << o) - 1u)) == 0u) X += y;
      }
    }
    const bool last = lane == 31 || ((heads >> (lane + 1)) & 1u);
    if (last && key != 0xFFFFFFFFu) add(key, X);
  }
  __syncthreads();
  // vertex update (a3) of rows [r0, r0 + nrow)
  if (blockIdx.x == 0 && tid == 0) A.dbuf[(A.it + 2) % 3] = 0.0;
  const double D = A.uniform ? A.dbuf[A.it % 3] : 0.0;
  const float dn = (float)(D * A.inv_n);
  double dpart = 0.0;
  for (int64_t i = tid; i < nrow; i += kPbThreads)
    pr_epilogue(A, r0 + i, (float)(((double)hi[i] * 4294967296.0 + (double)lo[i]) * 0x1p-62), dn, dpart);
  if (A.npeer) __threadfence_system();  // peer stores ordered before the next collective
  const double bs = block_sum(dpart, sred);
  if (tid == 0 && bs != 0.0) atomicAdd(&A.dbuf[(A.it + 1) % 3], bs);
}

// row -> row block
__global__ void k_pb_rowblock(const int64_t* __restrict__ rb, int Kd, int32_t* __restrict__ blk) {
  for (int d = blockIdx.x; d < Kd; d += gridDim.x)
    for (int64_t r = rb[d] + threadIdx.x; r < rb[d + 1]; r += blockDim.x) blk[r] = d;
}

// count the edges of every tile: a warp per CSC row, lanes of one step with the
// same tile aggregated (__match_any_sync: rows are sorted by source)
template <typename OffT>
__global__ void k_pb_count(const OffT* __restrict__ off, const int32_t* __restrict__ idx, int64_t nr,
                           const int32_t* __restrict__ blk, int Kd, unsigned long long* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < nr; v += nw) {
    const int d = blk[v];
    const int64_t b = (int64_t)off[v], e = (int64_t)off[v + 1];
    for (int64_t j0 = b; j0 < e; j0 += 32) {
      const int64_t j = j0 + lane;
      const bool on = j < e;
      const unsigned act = __ballot_sync(0xffffffffu, on);
      if (!on) continue;
      const int64_t t = (int64_t)(__ldg(&idx[j]) / kPbC) * Kd + d;
      const unsigned peers = __match_any_sync(act, (unsigned long long)t);
      if (lane == __ffs(peers) - 1) atomicAdd(&cnt[t], (unsigned long long)__popc(peers));
    }
  }
}

// place the edges: one warp per row block walks its rows in ascending order,
// keeping the fill of each of the block's tiles in shared memory, so every tile
// comes out sorted by destination (then source) — deterministic, and a group of 8
// edges of a hub row shares one destination (k_pb_gather merges such runs)
template <typename OffT>
__global__ void __launch_bounds__(32) k_pb_place(const OffT* __restrict__ off, const int32_t* __restrict__ idx,
                                                 const int64_t* __restrict__ rb, int Ks, int Kd,
                                                 const int64_t* __restrict__ tstart, uint16_t* __restrict__ src16,
                                                 uint16_t* __restrict__ dst16) {
  extern __shared__ int32_t fill[];  // Ks
  const int lane = threadIdx.x;
  const int d = blockIdx.x;
  for (int s = lane; s < Ks; s += 32) fill[s] = 0;
  __syncwarp();
  for (int64_t v = rb[d]; v < rb[d + 1]; ++v) {
    const int64_t b = (int64_t)off[v], e = (int64_t)off[v + 1];
    for (int64_t j0 = b; j0 < e; j0 += 32) {
      const int64_t j = j0 + lane;
      const bool on = j < e;
      const unsigned act = __ballot_sync(0xffffffffu, on);
      int32_t u = 0, sidx = 0, base = 0;
      unsigned peers = 0;
      if (on) {
        u = __ldg(&idx[j]);
        sidx = u / kPbC;
        peers = __match_any_sync(act, sidx);
        if (lane == __ffs(peers) - 1) {
          base = fill[sidx];
          fill[sidx] = base + __popc(peers);
        }
      }
      __syncwarp();
      if (on) {
        base = __shfl_sync(peers, base, __ffs(peers) - 1);
        const int64_t pos = tstart[(int64_t)sidx * Kd + d] + base + __popc(peers & ((1u << lane) - 1u));
        src16[pos] = (uint16_t)(u - sidx * kPbC);
        dst16[pos] = (uint16_t)(v - rb[d]);
      }
      __syncwarp();
    }
  }
}

__global__ void k_pb_pad(const unsigned long long* __restrict__ cnt, int64_t T, int64_t* __restrict__ pc) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x)
    pc[t] = (int64_t)((cnt[t] + kPbGroup - 1) / kPbGroup * kPbGroup);
}

__global__ void k_pb_fill(uint16_t* __restrict__ a, int64_t n, uint16_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = v;
}

// (row, source segment of Z) pairs holding an edge — the segmented pull's pieces —
// counted edge-parallel (rows are sorted by source): with s_j = idx[j] / Z,
//   pieces = #{j >= 1 : s_j != s_(j-1)} + #{non-empty rows starting at b : b == 0 or s_b == s_(b-1)}
// (every segment change inside a row starts a piece; a row's first edge starts
// one, which the global change count already holds unless its segment equals the
// previous row's last). Was a warp per row (15 ms on config 4).
__device__ __forceinline__ void count_add(unsigned long long c, unsigned long long* out) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}
__global__ void k_count_changes(const int32_t* __restrict__ idx, int64_t m, int Z, unsigned long long* __restrict__ out) {
  unsigned long long c = 0;
  const uint32_t z = (uint32_t)Z;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x + 1; j < m; j += (int64_t)gridDim.x * blockDim.x)
    c += (uint32_t)__ldg(&idx[j]) / z != (uint32_t)__ldg(&idx[j - 1]) / z;
  count_add(c, out);
}
template <typename OffT>
__global__ void k_count_row_starts(const OffT* __restrict__ off, const int32_t* __restrict__ idx, int64_t nr, int Z,
                                   unsigned long long* __restrict__ out) {
  unsigned long long c = 0;
  const uint32_t z = (uint32_t)Z;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nr; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = (int64_t)off[v], e = (int64_t)off[v + 1];
    if (e > b) c += b == 0 || (uint32_t)__ldg(&idx[b]) / z == (uint32_t)__ldg(&idx[b - 1]) / z;
  }
  count_add(c, out);
}

template <typename OffT>
gi_status pb_build_t(gi_graph g) {
  gi_context ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  const int64_t nr = g->nr, m = g->ml, n = g->n;
  const int Ks = (int)ceil_div(n, kPbC);
  if (Ks > kPbMaxChunks) return fail(GI_ERR_UNSUPPORTED, "blocked pull: too many source chunks");
  // row blocks: <= kPbB rows and <= W2 edges (a block of one row may hold more)
  std::vector<OffT> hoff(nr + 1);
  GI_CUDA(cudaMemcpyAsync(hoff.data(), g->csc_off.p, (nr + 1) * sizeof(OffT), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  const int64_t W2 = std::max<int64_t>(2 * m / std::max<int64_t>(ceil_div(nr, kPbB), 1), 1 << 16);
  std::vector<int64_t> rb{0};
  for (int64_t r = 0; r < nr;) {
    int64_t r1 = std::min<int64_t>(nr, r + kPbB);
    if ((int64_t)hoff[r1] - (int64_t)hoff[r] > W2)
      r1 = std::max<int64_t>(r + 1, (int64_t)(std::upper_bound(hoff.begin() + r, hoff.begin() + r1 + 1,
                                                                (OffT)((int64_t)hoff[r] + W2)) - hoff.begin()) - 1);
    rb.push_back(r1);
    r = r1;
  }
  if (nr == 0) rb.push_back(0);
  const int Kd = (int)rb.size() - 1;
  const int64_t T = (int64_t)Ks * Kd;
  GI_TRY(g->pb_rb.alloc((Kd + 1) * sizeof(int64_t)));
  GI_CUDA(cudaMemcpyAsync(g->pb_rb.p, rb.data(), (Kd + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  DevBuf blk, cnt, pc, tmp;
  GI_TRY(blk.alloc(std::max<int64_t>(nr, 1) * sizeof(int32_t)));
  k_pb_rowblock<<<std::min(Kd, 65535), 256, 0, st>>>(g->pb_rb.as<int64_t>(), Kd, blk.as<int32_t>());
  GI_TRY(cnt.alloc((T + 1) * sizeof(unsigned long long)));
  GI_CUDA(cudaMemsetAsync(cnt.p, 0, (T + 1) * sizeof(unsigned long long), st));
  const int gb = grid_for(nr * 32, 256, sms, 16);
  k_pb_count<OffT><<<gb, 256, 0, st>>>(g->csc_off.as<OffT>(), g->csc_idx.as<int32_t>(), nr, blk.as<int32_t>(), Kd,
                                       cnt.as<unsigned long long>());
  GI_TRY(pc.alloc((T + 1) * sizeof(int64_t)));
  k_pb_pad<<<grid_for(T + 1, 256, sms), 256, 0, st>>>(cnt.as<unsigned long long>(), T + 1, pc.as<int64_t>());
  GI_TRY(g->pb_tstart.alloc((T + 1) * sizeof(int64_t)));
  size_t tb = 0;
  GI_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, pc.as<int64_t>(), g->pb_tstart.as<int64_t>(), T + 1, st));
  GI_TRY(tmp.alloc(tb));
  GI_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, pc.as<int64_t>(), g->pb_tstart.as<int64_t>(), T + 1, st));
  std::vector<int64_t> hts(T + 1);
  GI_CUDA(cudaMemcpyAsync(hts.data(), g->pb_tstart.p, (T + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  const int64_t mp = hts[T];
  GI_TRY(g->pb_src.alloc((mp + 8) * sizeof(uint16_t)));
  GI_TRY(g->pb_dst.alloc((mp + 8) * sizeof(uint16_t)));
  GI_TRY(g->pb_vals.alloc((mp + 8) * sizeof(float)));
  k_pb_fill<<<grid_for(mp + 8, 256, sms, 16), 256, 0, st>>>(g->pb_src.as<uint16_t>(), mp + 8, (uint16_t)kPbC);
  k_pb_fill<<<grid_for(mp + 8, 256, sms, 16), 256, 0, st>>>(g->pb_dst.as<uint16_t>(), mp + 8, (uint16_t)kPbB);
  k_pb_place<OffT><<<Kd, 32, (size_t)Ks * sizeof(int32_t), st>>>(g->csc_off.as<OffT>(), g->csc_idx.as<int32_t>(),
                                                                 g->pb_rb.as<int64_t>(), Ks, Kd,
                                                                 g->pb_tstart.as<int64_t>(), g->pb_src.as<uint16_t>(),
                                                                 g->pb_dst.as<uint16_t>());
  GI_CUDA(cudaGetLastError());
  // scatter work items: each chunk's edge range cut into pieces of <= W1 edges
  const int64_t W1 = std::max<int64_t>(ceil_div(mp, 4 * (int64_t)sms) / kPbGroup * kPbGroup, 1 << 16);
  std::vector<int64_t> items;
  for (int s = 0; s < Ks; ++s) {
    const int64_t a = hts[(int64_t)s * Kd], b = hts[(int64_t)(s + 1) * Kd];
    for (int64_t e = a; e < b; e += W1) {
      items.push_back(s);
      items.push_back(e);
      items.push_back(std::min(b, e + W1));
    }
  }
  g->pb_nitems = (int)(items.size() / 3);
  GI_TRY(g->pb_items.alloc(std::max<size_t>(items.size(), 3) * sizeof(int64_t)));
  if (!items.empty())
    GI_CUDA(cudaMemcpyAsync(g->pb_items.p, items.data(), items.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  GI_CUDA(cudaStreamSynchronize(st));
  g->pb_Ks = Ks;
  g->pb_Kd = Kd;
  g->pb_mp = mp;
  if (const char* dbg = getenv("GI_DEBUG_SEG_LAYOUT")) {
    if (FILE* f = fopen(dbg, "a")) {
      fprintf(f, "blocked: n=%lld m=%lld Ks=%d Kd=%d tiles=%lld padded edges=%lld items=%d\n", (long long)nr,
              (long long)m, Ks, Kd, (long long)T, (long long)mp, g->pb_nitems);
      fclose(f);
    }
  }
  return GI_OK;
}

size_t pb_gather_smem(int Ks) { return 2 * (kPbB + 4) * sizeof(uint32_t) + ((Ks + 2) & ~1) * 4 + (size_t)Ks * 8; }

}  // namespace

gi_status pb_build(gi_graph g) {
  if (g->pb_Ks > 0) return GI_OK;
  if (g->ml == 0 || g->nr == 0) return fail(GI_ERR_UNSUPPORTED, "blocked pull: empty graph");
  int optin = 0;
  GI_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, g->ctx->device));
  if ((size_t)optin < pb_gather_smem(kPbMaxChunks) + 512) return fail(GI_ERR_UNSUPPORTED, "blocked pull: smem");
  return g->off64 ? pb_build_t<int64_t>(g) : pb_build_t<int32_t>(g);
}

// pieces of the segmented pull for segments of Z sources, i.e. (row, segment) pairs with an
// edge (the auto choice between the segmented pull and this one: a piece costs one RED there)
gi_status pb_count_pieces(gi_graph g, int Z, int64_t* pieces) {
  cudaStream_t st = g->ctx->stream;
  DevBuf c;
  GI_TRY(c.alloc(sizeof(unsigned long long)));
  GI_CUDA(cudaMemsetAsync(c.p, 0, sizeof(unsigned long long), st));
  const int sms = g->ctx->num_sms;
  if (g->ml > 1)
    k_count_changes<<<grid_for(g->ml, 256, sms, 8), 256, 0, st>>>(g->csc_idx.as<int32_t>(), g->ml, Z,
                                                                  c.as<unsigned long long>());
  if (g->off64)
    k_count_row_starts<int64_t><<<grid_for(g->nr, 256, sms, 8), 256, 0, st>>>(
        g->csc_off.as<int64_t>(), g->csc_idx.as<int32_t>(), g->nr, Z, c.as<unsigned long long>());
  else
    k_count_row_starts<int32_t><<<grid_for(g->nr, 256, sms, 8), 256, 0, st>>>(
        g->csc_off.as<int32_t>(), g->csc_idx.as<int32_t>(), g->nr, Z, c.as<unsigned long long>());
  unsigned long long h = 0;
  GI_CUDA(cudaMemcpyAsync(&h, c.p, sizeof h, cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  *pieces = (int64_t)h;
  return GI_OK;
}

// one iteration's edge pass + vertex update (A: the PrArgs of the iteration)
gi_status pb_iteration(gi_graph g, const PrArgs& A, cudaEvent_t mid) {
  cudaStream_t st = g->ctx->stream;
  PbArgs P;
  P.src16 = g->pb_src.as<uint16_t>();
  P.dst16 = g->pb_dst.as<uint16_t>();
  P.vals = g->pb_vals.as<float>();
  P.tstart = g->pb_tstart.as<int64_t>();
  P.items = g->pb_items.as<int64_t>();
  P.rb = g->pb_rb.as<int64_t>();
  P.cin = A.cin;
  P.n = g->n;
  P.Ks = g->pb_Ks;
  P.Kd = g->pb_Kd;
  const size_t s1 = (kPbC + 4) * sizeof(float), s2 = pb_gather_smem(g->pb_Ks);
  static size_t attr[64][2] = {};
  const int dev = g->ctx->device & 63;
  if (attr[dev][0] < s1) {
    GI_CUDA(cudaFuncSetAttribute(k_pb_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1));
    attr[dev][0] = s1;
  }
  if (attr[dev][1] < s2) {
    GI_CUDA(cudaFuncSetAttribute(k_pb_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2));
    attr[dev][1] = s2;
  }
  if (g->pb_nitems > 0) k_pb_scatter<<<g->pb_nitems, kPbThreads, s1, st>>>(P);
  if (mid) GI_CUDA(cudaEventRecord(mid, st));
  k_pb_gather<<<g->pb_Kd, kPbThreads, s2, st>>>(P, A);
  GI_CUDA(cudaGetLastError());
  return GI_OK;
}

}  // namespace gi
