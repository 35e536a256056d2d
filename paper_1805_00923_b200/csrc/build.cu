// build.cu — device graph builder.
//
// edge list (int32 src, dst) -> validate -> out-degree histogram (before dedup)
// -> relabel by it (descending, stable) when skewed -> 64-bit keys (u' << b | v')
// in internal ids, self-loops dropped, optional symmetrisation ("an undirected
// graph would be represented by duplicating the directed edges", PAPER.md
// P:3183 [draft]) -> radix sort -> unique (dedup) -> CSR (offsets by binary
// search per vertex) and exact out-degrees -> transposed keys -> radix sort ->
// CSC -> merge-path tile metadata for the pull kernel.
//
// The sort and select primitives are CUB (CUDA toolkit, header-only): library
// primitives in the sense of a cuBLAS call; every graph-specific step is a
// kernel below.
#include <cub/cub.cuh>

#include <chrono>
#include <cstdio>
#include <string>

#include "gi_internal.cuh"
#include "comm.cuh"

namespace gi {
namespace {

constexpr uint64_t kSentinel = ~0ull;
constexpr double kSkewRatio = 32.0;  // relabel when max out-degree > kSkewRatio x mean out-degree

__global__ void k_validate(const int32_t* __restrict__ src, const int32_t* __restrict__ dst, int64_t m0,
                           int64_t n, int* __restrict__ bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m0; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t u = src[i], v = dst[i];
    if (u < 0 || u >= n || v < 0 || v >= n) atomicExch(bad, 1);
  }
}

// keys of the pairs in internal ids (inv: input -> internal id, null = identity)
// (bad != null: the endpoints are validated here — an edge outside [0, n) sets
// *bad and becomes a sentinel — for the pipelined host-edge build)
__global__ void k_make_keys(const int32_t* __restrict__ src, const int32_t* __restrict__ dst, int64_t m0,
                            int bits, int rm_self, int sym, uint64_t* __restrict__ keys,
                            const int32_t* __restrict__ inv = nullptr, int64_t n = 0, int* __restrict__ bad = nullptr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m0; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t u = (uint32_t)src[i], v = (uint32_t)dst[i];
    bool drop = rm_self && u == v;
    if (bad && (u >= (uint64_t)n || v >= (uint64_t)n)) {
      atomicExch(bad, 1);
      u = v = 0;
      drop = true;
    }
    if (inv) {
      u = (uint32_t)__ldg(&inv[u]);
      v = (uint32_t)__ldg(&inv[v]);
    }
    if (sym) {
      keys[2 * i] = drop ? kSentinel : (u << bits) | v;
      keys[2 * i + 1] = drop ? kSentinel : (v << bits) | u;
    } else {
      keys[i] = drop ? kSentinel : (u << bits) | v;
    }
  }
}

// out-degrees before dedup (the relabelling's order and skew test; exact degrees come
// from the CSR): one count per kept pair, both directions when symmetrising
// the relabelling's degree: edge-list entries per source (self-loops and
// duplicates included; with symmetrisation also per destination). A heuristic
// order only — any internal order gives the same results in input ids — counted
// from src alone so the pipelined host-edge build can count before dst arrives
// (dst = null; bad != null: sources outside [0, n) set *bad and are skipped)
__global__ void k_hist_src(const int32_t* __restrict__ src, const int32_t* __restrict__ dst, int64_t m0, int sym,
                           int32_t* __restrict__ deg, int64_t n = 0, int* __restrict__ bad = nullptr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m0; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = src[i];
    if (bad && (u < 0 || u >= n)) {
      atomicExch(bad, 1);
      continue;
    }
    atomicAdd(&deg[u], 1);
    if (sym) atomicAdd(&deg[dst[i]], 1);
  }
}

// merge path (pairwise merge of sorted runs of 64-bit keys, the pipelined
// build's per-chunk sorts): split[t] = elements of A among the first t * kMergeTile
// outputs; a CTA merges one tile through shared memory
constexpr int kMergeThreads = 256, kMergeVT = 16, kMergeTile = kMergeThreads * kMergeVT;
__device__ __forceinline__ int64_t merge_path(const uint64_t* a, int64_t na, const uint64_t* b, int64_t nb,
                                              int64_t diag) {
  int64_t lo = diag > nb ? diag - nb : 0, hi = diag < na ? diag : na;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] <= b[diag - 1 - mid]) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
__global__ void k_merge_split(const uint64_t* __restrict__ a, int64_t na, const uint64_t* __restrict__ b, int64_t nb,
                              int64_t tiles, int64_t* __restrict__ split) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= tiles; t += (int64_t)gridDim.x * blockDim.x)
    split[t] = merge_path(a, na, b, nb, t * kMergeTile < na + nb ? t * kMergeTile : na + nb);
}
__global__ void __launch_bounds__(kMergeThreads) k_merge(const uint64_t* __restrict__ a, int64_t na,
                                                        const uint64_t* __restrict__ b, int64_t nb,
                                                        const int64_t* __restrict__ split, uint64_t* __restrict__ out) {
  __shared__ uint64_t s[kMergeTile];
  const int64_t tot = na + nb, d0 = blockIdx.x * (int64_t)kMergeTile;
  const int64_t d1 = d0 + kMergeTile < tot ? d0 + kMergeTile : tot;
  const int64_t a0 = split[blockIdx.x], a1 = split[blockIdx.x + 1], b0 = d0 - a0, b1 = d1 - a1;
  const int ta = (int)(a1 - a0), tn = (int)(d1 - d0);
  for (int i = threadIdx.x; i < tn; i += kMergeThreads) s[i] = i < ta ? a[a0 + i] : b[b0 + i - ta];
  __syncthreads();
  const int diag = min((int)threadIdx.x * kMergeVT, tn);
  int ia = (int)merge_path(s, ta, s + ta, tn - ta, diag), ib = diag - ia;
  uint64_t r[kMergeVT];
#pragma unroll
  for (int k = 0; k < kMergeVT; ++k) {
    if (diag + k < tn) {
      const bool takea = ib >= tn - ta || (ia < ta && s[ia] <= s[ta + ib]);
      r[k] = takea ? s[ia] : s[ta + ib];
      if (takea) ++ia;
      else ++ib;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kMergeVT; ++k)
    if (diag + k < tn) s[diag + k] = r[k];
  __syncthreads();
  for (int i = threadIdx.x; i < tn; i += kMergeThreads) out[d0 + i] = s[i];
}

// first index of a sentinel in sorted keys (the sentinels sort last)
__global__ void k_count_valid(const uint64_t* __restrict__ keys, int64_t m, int64_t* __restrict__ out) {
  int64_t lo = 0, hi = m;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (keys[mid] != kSentinel) lo = mid + 1;
    else hi = mid;
  }
  *out = lo;
}

struct NotSentinel {
  __host__ __device__ bool operator()(const uint64_t& k) const { return k != kSentinel; }
};

// off[u] = first position of row u in the sorted key array (lower bound of u << bits).
template <typename OffT>
__global__ void k_offsets(const uint64_t* __restrict__ keys, int64_t m, int64_t n, int bits, OffT* __restrict__ off) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u <= n; u += (int64_t)gridDim.x * blockDim.x) {
    uint64_t target = (uint64_t)u << bits;
    int64_t lo = 0, hi = m;
    while (lo < hi) {
      int64_t mid = lo + ((hi - lo) >> 1);
      if (keys[mid] < target) lo = mid + 1;
      else hi = mid;
    }
    off[u] = (OffT)lo;
  }
}

template <typename OffT>
__global__ void k_degrees(const OffT* __restrict__ off, int64_t n, int32_t* __restrict__ deg) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
    deg[u] = (int32_t)(off[u + 1] - off[u]);
}

__global__ void k_low_bits(const uint64_t* __restrict__ keys, int64_t m, int bits, int32_t* __restrict__ idx) {
  const uint64_t mask = (1ull << bits) - 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    idx[i] = (int32_t)(keys[i] & mask);
}

// sort key for relabelling: descending out-degree, stable on input id
__global__ void k_relabel_keys(const int32_t* __restrict__ deg, int64_t n, uint32_t* __restrict__ k,
                               int32_t* __restrict__ ids) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
    k[u] = 0x7FFFFFFFu - (uint32_t)deg[u];
    ids[u] = (int32_t)u;
  }
}

__global__ void k_invert(const int32_t* __restrict__ perm, int64_t n, int32_t* __restrict__ inv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    inv[perm[i]] = (int32_t)i;
}

// re-key sorted input-id edges (u << b | v) into internal ids; transpose => (v', u')
__global__ void k_rekey(const uint64_t* __restrict__ in, int64_t m, int bits, const int32_t* __restrict__ inv,
                        int transpose, uint64_t* __restrict__ out) {
  const uint64_t mask = (1ull << bits) - 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t u = in[i] >> bits, v = in[i] & mask;
    if (inv) {
      u = (uint32_t)inv[u];
      v = (uint32_t)inv[v];
    }
    out[i] = transpose ? ((v << bits) | u) : ((u << bits) | v);
  }
}

// Merge-path tiling of the CSC (items = rows' end markers + edges, n + m in
// total; row r occupies merge positions [r + off[r], r + off[r+1]]).
// rows[2b] = row containing position b*T, rows[2b+1] = row containing the
// tile's last position. "Row containing p" = min r with r + off[r+1] >= p.
template <typename OffT>
__global__ void k_tile_rows(const OffT* __restrict__ off, int64_t n, int64_t m, int64_t ntiles, int T,
                            int32_t* __restrict__ rows) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < 2 * ntiles;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = t >> 1;
    int64_t p = (t & 1) ? min((b + 1) * (int64_t)T, n + m) - 1 : b * (int64_t)T;
    int64_t lo = 0, hi = n - 1;
    while (lo < hi) {
      int64_t mid = lo + ((hi - lo) >> 1);
      if (mid + (int64_t)off[mid + 1] >= p) hi = mid;
      else lo = mid + 1;
    }
    rows[t] = (int32_t)lo;
  }
}

// CSR keys (u << bits | v) -> the pair (v, u) as two 32-bit arrays (the CSC's row key and value)
__global__ void k_split_keys(const uint64_t* __restrict__ keys, int64_t m, int bits, uint32_t* __restrict__ vk,
                             int32_t* __restrict__ uv) {
  const uint64_t mask = (1ull << bits) - 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    vk[i] = (uint32_t)(keys[i] & mask);
    uv[i] = (int32_t)(keys[i] >> bits);
  }
}

// off[r] = first position of row r in sorted 32-bit row keys
template <typename OffT>
__global__ void k_offsets32(const uint32_t* __restrict__ keys, int64_t m, int64_t n, OffT* __restrict__ off) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= n; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = m;
    while (lo < hi) {
      const int64_t mid = lo + ((hi - lo) >> 1);
      if ((int64_t)keys[mid] < r) lo = mid + 1;
      else hi = mid;
    }
    off[r] = (OffT)lo;
  }
}

int bits_for(int64_t n) {
  int b = 1;
  while ((1ll << b) < n) ++b;
  return b;
}

// diagnostics (GI_DEBUG_BUILD=file): synchronised phase times
struct BuildDbg {
  const char* file = getenv("GI_DEBUG_BUILD");
  cudaStream_t st;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  std::string s;
  explicit BuildDbg(cudaStream_t st_) : st(st_) {}
  void mark(const char* name) {
    if (!file) return;
    cudaStreamSynchronize(st);
    const auto t2 = std::chrono::steady_clock::now();
    char b[64];
    snprintf(b, sizeof(b), " %s=%.1f", name, std::chrono::duration<double, std::milli>(t2 - t).count());
    s += b;
    t = t2;
  }
  void flush(const char* what, int64_t n, int64_t m0, int64_t m) {
    if (!file) return;
    if (FILE* f = fopen(file, "a")) {
      fprintf(f, "%s n=%lld m0=%lld m=%lld:%s\n", what, (long long)n, (long long)m0, (long long)m, s.c_str());
      fclose(f);
    }
  }
};

struct Temp {
  DevBuf buf;
  gi_status ensure(size_t bytes) {
    if (buf.bytes >= bytes && buf.p) return GI_OK;
    return buf.alloc(bytes);
  }
};

}  // namespace

// rows + 1 offsets (lower bounds of r << bits) and the low-bit column ids
template <typename OffT>
static gi_status csr_from_sorted(gi_graph g, const uint64_t* keys, int64_t m, int bits, int64_t rows, DevBuf& off,
                                 DevBuf& idx) {
  cudaStream_t st = g->ctx->stream;
  const int sms = g->ctx->num_sms;
  GI_TRY(off.alloc((rows + 1) * sizeof(OffT)));
  GI_TRY(idx.alloc(m * sizeof(int32_t)));
  k_offsets<OffT><<<grid_for(rows + 1, 256, sms), 256, 0, st>>>(keys, m, rows, bits, off.as<OffT>());
  k_low_bits<<<grid_for(m, 256, sms), 256, 0, st>>>(keys, m, bits, idx.as<int32_t>());
  GI_CUDA(cudaGetLastError());
  return GI_OK;
}

static gi_status build_tail(gi_graph g, uint32_t flags, int64_t n, int64_t m, int bits, DevBuf* cur, DevBuf* alt,
                            Temp& tmp, BuildDbg& dbg);
static gi_status relabel_from_degrees(gi_graph g, int64_t n, Temp& tmp, const int32_t** inv);

gi_status build_graph(gi_context ctx, int64_t n, int64_t m0, const int32_t* d_src, const int32_t* d_dst,
                      uint32_t flags, gi_graph g) {
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  g->ctx = ctx;
  g->n = n;
  const bool rm_self = flags & GI_REMOVE_SELF_LOOPS;
  const bool dedup = flags & GI_DEDUP;
  const bool sym = flags & GI_SYMMETRIZE;
  g->relabeled = !(flags & GI_NO_RELABEL) && n > 1;

  BuildDbg dbg(st);
  // 1. validate endpoints
  DevBuf bad;
  GI_TRY(bad.alloc(sizeof(int)));
  GI_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
  if (m0 > 0) k_validate<<<grid_for(m0, 256, sms), 256, 0, st>>>(d_src, d_dst, m0, n, bad.as<int>());
  int h_bad = 0;
  GI_CUDA(cudaMemcpyAsync(&h_bad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  if (h_bad) return fail(GI_ERR_VERTEX_OUT_OF_RANGE, "gi_graph_create: an edge endpoint is outside [0, n)");

  // 2. relabel by out-degree (descending, stable) when the degrees are skewed:
  // hub sources then form a dense prefix (segment 0 of the segmented pull, the
  // staged bitmap prefix of the BFS pull). A flat degree distribution (a road
  // grid) keeps its input order and with it its locality. The order and the
  // skew test use the degrees before dedup (one histogram pass), so the keys are
  // made in internal ids directly and sorted twice in all (CSR, CSC); any
  // internal order is valid: results are reported in input ids.
  const int bits = bits_for(n > 1 ? n : 2);
  const int64_t mk = sym ? 2 * m0 : m0;
  Temp tmp;
  GI_TRY(g->outdeg.alloc(n * sizeof(int32_t)));
  const int32_t* inv = nullptr;
  if (g->relabeled && m0 > 0) {
    GI_CUDA(cudaMemsetAsync(g->outdeg.p, 0, n * sizeof(int32_t), st));
    k_hist_src<<<grid_for(m0, 256, sms, 16), 256, 0, st>>>(d_src, d_dst, m0, sym, g->outdeg.as<int32_t>());
    GI_TRY(relabel_from_degrees(g, n, tmp, &inv));
  } else {
    g->relabeled = false;
  }
  dbg.mark("validate+relabel");
  // 3. keys (u' << b | v') in internal ids, 4. select non-sentinel, 5. sort, 6. unique
  DevBuf kA, kB, nsel;
  GI_TRY(kA.alloc(mk * sizeof(uint64_t)));
  GI_TRY(kB.alloc(mk * sizeof(uint64_t)));
  GI_TRY(nsel.alloc(sizeof(int64_t)));
  size_t tb = 0;
  int64_t m = 0;
  if (mk > 0) {
    k_make_keys<<<grid_for(m0, 256, sms), 256, 0, st>>>(d_src, d_dst, m0, bits, rm_self, sym, kA.as<uint64_t>(), inv);
    GI_CUDA(cub::DeviceSelect::If(nullptr, tb, kA.as<uint64_t>(), kB.as<uint64_t>(), nsel.as<int64_t>(), mk,
                                  NotSentinel(), st));
    GI_TRY(tmp.ensure(tb));
    GI_CUDA(cub::DeviceSelect::If(tmp.buf.p, tb, kA.as<uint64_t>(), kB.as<uint64_t>(), nsel.as<int64_t>(), mk,
                                  NotSentinel(), st));
    GI_CUDA(cudaMemcpyAsync(&m, nsel.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    GI_CUDA(cudaStreamSynchronize(st));
  }
  // sorted keys end up in `cur`
  DevBuf* cur = &kB;
  DevBuf* alt = &kA;
  auto sort_keys = [&](int64_t count) -> gi_status {
    if (count <= 1) return GI_OK;
    cub::DoubleBuffer<uint64_t> db(cur->as<uint64_t>(), alt->as<uint64_t>());
    size_t b = 0;
    GI_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, b, db, count, 0, 2 * bits, st));
    GI_TRY(tmp.ensure(b));
    GI_CUDA(cub::DeviceRadixSort::SortKeys(tmp.buf.p, b, db, count, 0, 2 * bits, st));
    if (db.Current() != cur->as<uint64_t>()) std::swap(cur, alt);
    return GI_OK;
  };
  dbg.mark("keys");
  GI_TRY(sort_keys(m));
  dbg.mark("sort1");
  GI_TRY(build_tail(g, flags, n, m, bits, cur, alt, tmp, dbg));
  dbg.flush("build", n, m0, g->m);
  return GI_OK;
}

// from the sorted keys (in *cur, m of them, sentinels removed): unique (dedup),
// CSR and exact out-degrees, CSC, pull tiles
static gi_status build_tail(gi_graph g, uint32_t flags, int64_t n, int64_t m, int bits, DevBuf* cur, DevBuf* alt,
                            Temp& tmp, BuildDbg& dbg) {
  cudaStream_t st = g->ctx->stream;
  const int sms = g->ctx->num_sms;
  const bool dedup = flags & GI_DEDUP;
  DevBuf nsel;
  GI_TRY(nsel.alloc(sizeof(int64_t)));
  if (dedup && m > 1) {
    size_t b = 0;
    GI_CUDA(cub::DeviceSelect::Unique(nullptr, b, cur->as<uint64_t>(), alt->as<uint64_t>(), nsel.as<int64_t>(), m, st));
    GI_TRY(tmp.ensure(b));
    GI_CUDA(cub::DeviceSelect::Unique(tmp.buf.p, b, cur->as<uint64_t>(), alt->as<uint64_t>(), nsel.as<int64_t>(), m,
                                      st));
    GI_CUDA(cudaMemcpyAsync(&m, nsel.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    GI_CUDA(cudaStreamSynchronize(st));
    std::swap(cur, alt);
  }
  g->m = m;
  g->ml = m;
  g->r0 = 0;
  g->nr = n;
  g->off64 = m >= (int64_t)INT32_MAX || (flags & GI_OFFSETS64);

  dbg.mark("unique");
  // 7. CSR in internal ids and the exact out-degrees
  if (g->off64) GI_TRY(csr_from_sorted<int64_t>(g, cur->as<uint64_t>(), m, bits, n, g->csr_off, g->csr_idx));
  else GI_TRY(csr_from_sorted<int32_t>(g, cur->as<uint64_t>(), m, bits, n, g->csr_off, g->csr_idx));
  if (n > 0) {
    if (g->off64) k_degrees<int64_t><<<grid_for(n, 256, sms), 256, 0, st>>>(g->csr_off.as<int64_t>(), n, g->outdeg.as<int32_t>());
    else k_degrees<int32_t><<<grid_for(n, 256, sms), 256, 0, st>>>(g->csr_off.as<int32_t>(), n, g->outdeg.as<int32_t>());
  }

  dbg.mark("csr");
  // 8. CSC in internal ids: a stable sort of the CSR's (v, u) pairs by v alone
  // (`bits`-bit 32-bit keys, half the passes and bytes of re-sorting 64-bit
  // transposed keys): the CSR order already has u ascending inside each v
  GI_TRY(g->csc_idx.alloc(std::max<int64_t>(m, 1) * sizeof(int32_t)));
  const uint32_t* vsorted = nullptr;
  if (m > 0) {
    uint32_t* vk = alt->as<uint32_t>();  // alt holds 8 x mk >= 8m bytes: two 4m-byte arrays
    int32_t* uv = reinterpret_cast<int32_t*>(vk + m);
    k_split_keys<<<grid_for(m, 256, sms), 256, 0, st>>>(cur->as<uint64_t>(), m, bits, vk, uv);
    uint32_t* vk2 = cur->as<uint32_t>();  // the CSR keys are consumed: cur is scratch now
    cub::DoubleBuffer<uint32_t> dk(vk, vk2);
    cub::DoubleBuffer<int32_t> dv(uv, g->csc_idx.as<int32_t>());
    size_t b = 0;
    GI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b, dk, dv, m, 0, bits, st));
    GI_TRY(tmp.ensure(b));
    GI_CUDA(cub::DeviceRadixSort::SortPairs(tmp.buf.p, b, dk, dv, m, 0, bits, st));
    if (dv.Current() != g->csc_idx.as<int32_t>())
      GI_CUDA(cudaMemcpyAsync(g->csc_idx.p, dv.Current(), m * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    vsorted = dk.Current();
  }
  dbg.mark("sort2");
  GI_TRY(g->csc_off.alloc((n + 1) * (g->off64 ? sizeof(int64_t) : sizeof(int32_t))));
  if (g->off64)
    k_offsets32<int64_t><<<grid_for(n + 1, 256, sms), 256, 0, st>>>(vsorted, m, n, g->csc_off.as<int64_t>());
  else
    k_offsets32<int32_t><<<grid_for(n + 1, 256, sms), 256, 0, st>>>(vsorted, m, n, g->csc_off.as<int32_t>());
  GI_CUDA(cudaGetLastError());

  // 10. pull tiling metadata
  g->ntiles = n > 0 ? ceil_div(n + m, kPullTile) : 0;
  GI_TRY(g->tile_rows.alloc(2 * (g->ntiles > 0 ? g->ntiles : 1) * sizeof(int32_t)));
  if (g->ntiles > 0) {
    if (g->off64)
      k_tile_rows<int64_t><<<grid_for(2 * g->ntiles, 256, sms), 256, 0, st>>>(g->csc_off.as<int64_t>(), n, m, g->ntiles,
                                                                            kPullTile, g->tile_rows.as<int32_t>());
    else
      k_tile_rows<int32_t><<<grid_for(2 * g->ntiles, 256, sms), 256, 0, st>>>(g->csc_off.as<int32_t>(), n, m, g->ntiles,
                                                                            kPullTile, g->tile_rows.as<int32_t>());
  }
  GI_CUDA(cudaGetLastError());
  GI_CUDA(cudaStreamSynchronize(st));
  dbg.mark("csc+tiles");
  return GI_OK;
}


// skew test on the relabelling degrees (g->outdeg, filled by k_hist_src) and, when
// skewed, the order by them (descending, stable): perm (internal -> input), inv
static gi_status relabel_from_degrees(gi_graph g, int64_t n, Temp& tmp, const int32_t** inv) {
  cudaStream_t st = g->ctx->stream;
  const int sms = g->ctx->num_sms;
  DevBuf mx, tot;
  GI_TRY(mx.alloc(sizeof(int32_t)));
  GI_TRY(tot.alloc(sizeof(int64_t)));
  size_t b = 0;
  GI_CUDA(cub::DeviceReduce::Max(nullptr, b, g->outdeg.as<int32_t>(), mx.as<int32_t>(), n, st));
  GI_TRY(tmp.ensure(b));
  GI_CUDA(cub::DeviceReduce::Max(tmp.buf.p, b, g->outdeg.as<int32_t>(), mx.as<int32_t>(), n, st));
  b = 0;
  GI_CUDA(cub::DeviceReduce::Sum(nullptr, b, g->outdeg.as<int32_t>(), tot.as<int64_t>(), n, st));
  GI_TRY(tmp.ensure(b));
  GI_CUDA(cub::DeviceReduce::Sum(tmp.buf.p, b, g->outdeg.as<int32_t>(), tot.as<int64_t>(), n, st));
  int32_t hmax = 0;
  int64_t htot = 0;
  GI_CUDA(cudaMemcpyAsync(&hmax, mx.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaMemcpyAsync(&htot, tot.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  const double mean = n > 0 ? (double)htot / (double)n : 0.0;
  g->relabeled = (double)hmax > kSkewRatio * std::max(1.0, mean);
  if (!g->relabeled) return GI_OK;
  DevBuf rk, rk2, ids;
  GI_TRY(rk.alloc(n * sizeof(uint32_t)));
  GI_TRY(rk2.alloc(n * sizeof(uint32_t)));
  GI_TRY(ids.alloc(n * sizeof(int32_t)));
  GI_TRY(g->perm.alloc(n * sizeof(int32_t)));
  GI_TRY(g->inv.alloc(n * sizeof(int32_t)));
  k_relabel_keys<<<grid_for(n, 256, sms), 256, 0, st>>>(g->outdeg.as<int32_t>(), n, rk.as<uint32_t>(), ids.as<int32_t>());
  b = 0;
  GI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b, rk.as<uint32_t>(), rk2.as<uint32_t>(), ids.as<int32_t>(),
                                          g->perm.as<int32_t>(), n, 0, 32, st));
  GI_TRY(tmp.ensure(b));
  GI_CUDA(cub::DeviceRadixSort::SortPairs(tmp.buf.p, b, rk.as<uint32_t>(), rk2.as<uint32_t>(), ids.as<int32_t>(),
                                          g->perm.as<int32_t>(), n, 0, 32, st));
  k_invert<<<grid_for(n, 256, sms), 256, 0, st>>>(g->perm.as<int32_t>(), n, g->inv.as<int32_t>());
  GI_CUDA(cudaGetLastError());
  *inv = g->inv.as<int32_t>();
  return GI_OK;
}

// ---- host edges: the H2D copy overlapped with the build (gi_graph_create's
// host-pointer path; pinned memory makes the copies asynchronous). The copy
// stream moves src in kSrcChunks chunks, then dst in kDstChunks; the build stream
// counts each src chunk's relabelling degrees as it lands (validating sources),
// orders the vertices once src is complete (exactly as from device edges), then
// per dst chunk makes its keys (validating destinations) and radix-sorts them
// while the next chunk is in flight; pairwise merge-path rounds join the sorted
// chunks, and the rest (dedup, CSR, CSC) is build_tail. Config 4: the 12.9 GB
// H2D (~220 ms) used to precede a ~235 ms build.
constexpr int kSrcChunks = 8, kDstChunks = 4;
constexpr int64_t kPipeMinEdges = 1ll << 24;

}  // namespace gi

bool gi::build_host_pipelined(gi_context ctx, int64_t m0, uint32_t flags) {
  static const bool on = !getenv("GI_BUILD_PIPELINE") || atoi(getenv("GI_BUILD_PIPELINE")) != 0;
  return on && ctx->nranks == 1 && m0 >= kPipeMinEdges && !(flags & GI_SYMMETRIZE);
}

gi_status gi::build_graph_host(gi_context ctx, int64_t n, int64_t m0, const int32_t* h_src, const int32_t* h_dst,
                               uint32_t flags, gi_graph g) {
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  g->ctx = ctx;
  g->n = n;
  const bool rm_self = flags & GI_REMOVE_SELF_LOOPS;
  g->relabeled = !(flags & GI_NO_RELABEL) && n > 1;
  BuildDbg dbg(st);
  if (!ctx->copy_stream) GI_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  cudaStream_t cs = ctx->copy_stream;
  DevBuf ds, dd, bad;
  GI_TRY(ds.alloc(m0 * sizeof(int32_t)));
  GI_TRY(dd.alloc(m0 * sizeof(int32_t)));
  GI_TRY(bad.alloc(sizeof(int)));
  GI_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
  const int bits = bits_for(n > 1 ? n : 2);
  Temp tmp;
  GI_TRY(g->outdeg.alloc(n * sizeof(int32_t)));
  GI_CUDA(cudaMemsetAsync(g->outdeg.p, 0, n * sizeof(int32_t), st));
  DevBuf kA, kB, nsel;
  GI_TRY(kA.alloc(m0 * sizeof(uint64_t)));
  GI_TRY(kB.alloc(m0 * sizeof(uint64_t)));
  GI_TRY(nsel.alloc(sizeof(int64_t)));
  // the copy stream starts once the buffers are ready on the build stream
  cudaEvent_t ready, ev[kSrcChunks + kDstChunks];
  GI_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  for (auto& e : ev) GI_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  struct Events {  // on every return: the copies are complete before ds / dd are freed
    cudaEvent_t* e;
    int k;
    cudaEvent_t r;
    cudaStream_t cs;
    ~Events() {
      cudaStreamSynchronize(cs);
      for (int i = 0; i < k; ++i) cudaEventDestroy(e[i]);
      cudaEventDestroy(r);
    }
  } evs{ev, kSrcChunks + kDstChunks, ready, cs};
  GI_CUDA(cudaEventRecord(ready, st));
  GI_CUDA(cudaStreamWaitEvent(cs, ready, 0));
  auto cut = [&](int i, int k) { return m0 * i / k; };
  for (int i = 0; i < kSrcChunks; ++i) {
    const int64_t a = cut(i, kSrcChunks), b = cut(i + 1, kSrcChunks);
    GI_CUDA(cudaMemcpyAsync(ds.as<int32_t>() + a, h_src + a, (b - a) * sizeof(int32_t), cudaMemcpyHostToDevice, cs));
    GI_CUDA(cudaEventRecord(ev[i], cs));
  }
  for (int i = 0; i < kDstChunks; ++i) {
    const int64_t a = cut(i, kDstChunks), b = cut(i + 1, kDstChunks);
    GI_CUDA(cudaMemcpyAsync(dd.as<int32_t>() + a, h_dst + a, (b - a) * sizeof(int32_t), cudaMemcpyHostToDevice, cs));
    GI_CUDA(cudaEventRecord(ev[kSrcChunks + i], cs));
  }
  // relabelling degrees per src chunk, then the order
  const int32_t* inv = nullptr;
  for (int i = 0; i < kSrcChunks; ++i) {
    const int64_t a = cut(i, kSrcChunks), b = cut(i + 1, kSrcChunks);
    GI_CUDA(cudaStreamWaitEvent(st, ev[i], 0));
    if (g->relabeled && b > a)
      k_hist_src<<<grid_for(b - a, 256, sms, 16), 256, 0, st>>>(ds.as<int32_t>() + a, nullptr, b - a, 0,
                                                               g->outdeg.as<int32_t>(), n, bad.as<int>());
  }
  if (g->relabeled) GI_TRY(relabel_from_degrees(g, n, tmp, &inv));
  dbg.mark("src+relabel");
  // keys and a sort per dst chunk (validating every endpoint: an invalid edge is a
  // sentinel and raises the flag, checked before the result is used)
  std::vector<int64_t> run{0};
  bool in_b = false;
  for (int i = 0; i < kDstChunks; ++i) {
    const int64_t a = cut(i, kDstChunks), b = cut(i + 1, kDstChunks);
    GI_CUDA(cudaStreamWaitEvent(st, ev[kSrcChunks + i], 0));
    if (b > a) {
      k_make_keys<<<grid_for(b - a, 256, sms), 256, 0, st>>>(ds.as<int32_t>() + a, dd.as<int32_t>() + a, b - a, bits,
                                                            rm_self, 0, kA.as<uint64_t>() + a, inv, n, bad.as<int>());
      // bit 2 * bits separates the sentinels (all ones) from every key
      cub::DoubleBuffer<uint64_t> db(kA.as<uint64_t>() + a, kB.as<uint64_t>() + a);
      size_t tb = 0;
      GI_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, b - a, 0, 2 * bits + 1, st));
      GI_TRY(tmp.ensure(tb));
      GI_CUDA(cub::DeviceRadixSort::SortKeys(tmp.buf.p, tb, db, b - a, 0, 2 * bits + 1, st));
      in_b = db.Current() != kA.as<uint64_t>() + a;  // the same pass count for every chunk
    }
    run.push_back(b);
  }
  dbg.mark("dst+keys+chunk sorts");
  int h_bad = 0;
  GI_CUDA(cudaMemcpyAsync(&h_bad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  if (h_bad) return fail(GI_ERR_VERTEX_OUT_OF_RANGE, "gi_graph_create: an edge endpoint is outside [0, n)");
  ds.reset();
  dd.reset();
  // pairwise merge rounds until one run is left
  DevBuf* cur = in_b ? &kB : &kA;
  DevBuf* alt = in_b ? &kA : &kB;
  DevBuf split;
  while (run.size() > 2) {
    std::vector<int64_t> next{0};
    for (size_t r = 0; r + 1 < run.size(); r += 2) {
      const int64_t a0 = run[r], a1 = run[r + 1];
      if (r + 2 >= run.size()) {  // odd run out: copied
        GI_CUDA(cudaMemcpyAsync(alt->as<uint64_t>() + a0, cur->as<uint64_t>() + a0, (a1 - a0) * 8,
                                cudaMemcpyDeviceToDevice, st));
        next.push_back(a1);
        continue;
      }
      const int64_t b1 = run[r + 2], na = a1 - a0, nb = b1 - a1;
      const int64_t tiles = ceil_div(na + nb, kMergeTile);
      if (split.bytes < (size_t)(tiles + 1) * 8) GI_TRY(split.alloc((tiles + 1) * 8));
      k_merge_split<<<grid_for(tiles + 1, 256, sms), 256, 0, st>>>(cur->as<uint64_t>() + a0, na,
                                                                 cur->as<uint64_t>() + a1, nb, tiles,
                                                                 split.as<int64_t>());
      k_merge<<<(unsigned)tiles, kMergeThreads, 0, st>>>(cur->as<uint64_t>() + a0, na, cur->as<uint64_t>() + a1, nb,
                                                         split.as<int64_t>(), alt->as<uint64_t>() + a0);
      next.push_back(b1);
    }
    run.swap(next);
    std::swap(cur, alt);
  }
  GI_CUDA(cudaGetLastError());
  // the sentinels (self-loops) sort last: m = the first sentinel's index
  int64_t m = 0;
  k_count_valid<<<1, 1, 0, st>>>(cur->as<uint64_t>(), m0, nsel.as<int64_t>());
  GI_CUDA(cudaMemcpyAsync(&m, nsel.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  dbg.mark("merge");
  GI_TRY(build_tail(g, flags, n, m, bits, cur, alt, tmp, dbg));
  dbg.flush("build (host edges, pipelined)", n, m0, g->m);
  return GI_OK;
}

namespace gi {

// ---------------------------------------------------------------------------------------------
// Multi-GPU build: 1-D destination-range partition. Every rank
// passes any share of the edge list; the graph is the union.
//   1. validate (allreduce of an error flag: every rank fails alike)
//   2. local keys (u << 32 | v), self-loops dropped, optional symmetrisation
//   3. approximate degree histograms (before dedup) -> allreduce
//   4. relabel by approximate out-degree (identical on every rank: same input,
//      same deterministic radix sort); only the internal order depends on it
//   5. owner ranges: in-degree + 1 weights, equal shares cut at whole bitmap
//      words (partition_ranges)
//   6. owner shuffle: sort keys by owner, alltoallv (NCCL grouped send/recv)
//   7. local sort + dedup (duplicates share an owner), CSR by source over all
//      n sources (edges into the owned range), CSC of the owned rows, exact
//      out-degrees by allreduce, global m by allreduce
namespace {

__global__ void k_key_hist(const uint64_t* __restrict__ keys, int64_t k, int32_t* __restrict__ od,
                           int32_t* __restrict__ id) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
    atomicAdd(&od[keys[i] >> 32], 1);
    atomicAdd(&id[keys[i] & 0xFFFFFFFFull], 1);
  }
}

__global__ void k_weights(const int32_t* __restrict__ perm, const int32_t* __restrict__ indeg, int64_t n,
                          int64_t* __restrict__ w) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x)
    w[i] = i < n ? (int64_t)indeg[perm ? perm[i] : i] + 1 : 0;
}

__global__ void k_dist_owner(const uint64_t* __restrict__ keys, int64_t k, const int32_t* __restrict__ inv,
                             const int64_t* __restrict__ bounds, int P, uint32_t* __restrict__ owner,
                             uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t u = keys[i] >> 32, v = keys[i] & 0xFFFFFFFFull;
    if (inv) {
      u = (uint32_t)inv[u];
      v = (uint32_t)inv[v];
    }
    int lo = 0, hi = P - 1;  // last p with bounds[p] <= v
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (bounds[mid] <= (int64_t)v) lo = mid;
      else hi = mid - 1;
    }
    owner[i] = (uint32_t)lo;
    out[i] = (u << 32) | v;
  }
}

__global__ void k_owner_starts(const uint32_t* __restrict__ owner, int64_t k, int P, int64_t* __restrict__ starts) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p <= P; p += gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = k;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (owner[mid] < (uint32_t)p) lo = mid + 1;
      else hi = mid;
    }
    starts[p] = lo;
  }
}

// (u << 32 | v) -> (u << b | v)  or, transposed for the local CSC, ((v - r0) << b | u)
__global__ void k_pack_local(const uint64_t* __restrict__ in, int64_t k, int bits, int64_t r0, int transpose,
                             uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t u = in[i] >> 32, v = in[i] & 0xFFFFFFFFull;
    out[i] = transpose ? (((v - (uint64_t)r0) << bits) | u) : ((u << bits) | v);
  }
}

// (u << b | v) -> ((v - r0) << b | u)
__global__ void k_repack_transpose(const uint64_t* __restrict__ in, int64_t k, int bits, int64_t r0,
                                   uint64_t* __restrict__ out) {
  const uint64_t mask = (1ull << bits) - 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t u = in[i] >> bits, v = in[i] & mask;
    out[i] = ((v - (uint64_t)r0) << bits) | u;
  }
}

struct DevPrefix {
  const int64_t* d;
};
int64_t dev_prefix(void* ctx, int64_t i) {
  int64_t v = 0;
  cudaMemcpy(&v, static_cast<DevPrefix*>(ctx)->d + i, sizeof(int64_t), cudaMemcpyDeviceToHost);
  return v;
}

}  // namespace

gi_status build_graph_dist(gi_context ctx, int64_t n, int64_t m0, const int32_t* d_src, const int32_t* d_dst,
                           uint32_t flags, gi_graph g) {
  Comm* C = ctx->comm;
  if (!C) return fail(GI_ERR_INTERNAL, "multi-GPU context without a comm layer");
  cudaStream_t st = ctx->stream;
  const int sms = ctx->num_sms;
  const int P = C->nranks, R = C->rank;
  g->ctx = ctx;
  g->n = n;
  const bool rm_self = flags & GI_REMOVE_SELF_LOOPS;
  const bool dedup = flags & GI_DEDUP;
  const bool sym = flags & GI_SYMMETRIZE;
  g->relabeled = !(flags & GI_NO_RELABEL) && n > 1;

  // 1. validate
  DevBuf bad;
  GI_TRY(bad.alloc(sizeof(int32_t)));
  GI_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int32_t), st));
  if (m0 > 0) k_validate<<<grid_for(m0, 256, sms), 256, 0, st>>>(d_src, d_dst, m0, n, bad.as<int>());
  GI_TRY(C->allreduce_i32(bad.as<int32_t>(), 1, st));
  int32_t h_bad = 0;
  GI_CUDA(cudaMemcpyAsync(&h_bad, bad.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  if (h_bad) return fail(GI_ERR_VERTEX_OUT_OF_RANGE, "gi_graph_create: an edge endpoint is outside [0, n) on some rank");

  // 2. local keys in input ids (u << 32 | v)
  const int64_t mk = sym ? 2 * m0 : m0;
  DevBuf kA, kB, nsel, tmp;
  GI_TRY(kA.alloc(mk * sizeof(uint64_t)));
  GI_TRY(kB.alloc(mk * sizeof(uint64_t)));
  GI_TRY(nsel.alloc(sizeof(int64_t)));
  int64_t k = 0;
  size_t tb = 0;
  if (mk > 0) {
    k_make_keys<<<grid_for(m0, 256, sms), 256, 0, st>>>(d_src, d_dst, m0, 32, rm_self, sym, kA.as<uint64_t>());
    GI_CUDA(cub::DeviceSelect::If(nullptr, tb, kA.as<uint64_t>(), kB.as<uint64_t>(), nsel.as<int64_t>(), mk,
                                  NotSentinel(), st));
    GI_TRY(tmp.alloc(tb));
    GI_CUDA(cub::DeviceSelect::If(tmp.p, tb, kA.as<uint64_t>(), kB.as<uint64_t>(), nsel.as<int64_t>(), mk,
                                  NotSentinel(), st));
    GI_CUDA(cudaMemcpyAsync(&k, nsel.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    GI_CUDA(cudaStreamSynchronize(st));
  }
  // 3. approximate degree histograms (duplicates counted), summed over ranks
  DevBuf hod, hid;
  GI_TRY(hod.alloc(n * sizeof(int32_t)));
  GI_TRY(hid.alloc(n * sizeof(int32_t)));
  GI_CUDA(cudaMemsetAsync(hod.p, 0, n * sizeof(int32_t), st));
  GI_CUDA(cudaMemsetAsync(hid.p, 0, n * sizeof(int32_t), st));
  if (k > 0) k_key_hist<<<grid_for(k, 256, sms), 256, 0, st>>>(kB.as<uint64_t>(), k, hod.as<int32_t>(), hid.as<int32_t>());
  GI_TRY(C->allreduce_i32(hod.as<int32_t>(), n, st));
  GI_TRY(C->allreduce_i32(hid.as<int32_t>(), n, st));
  // 4. relabel (same permutation on every rank)
  const int32_t* inv = nullptr;
  if (g->relabeled) {
    DevBuf rk, rk2, ids;
    GI_TRY(rk.alloc(n * sizeof(uint32_t)));
    GI_TRY(rk2.alloc(n * sizeof(uint32_t)));
    GI_TRY(ids.alloc(n * sizeof(int32_t)));
    GI_TRY(g->perm.alloc(n * sizeof(int32_t)));
    GI_TRY(g->inv.alloc(n * sizeof(int32_t)));
    k_relabel_keys<<<grid_for(n, 256, sms), 256, 0, st>>>(hod.as<int32_t>(), n, rk.as<uint32_t>(), ids.as<int32_t>());
    tb = 0;
    GI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, rk.as<uint32_t>(), rk2.as<uint32_t>(), ids.as<int32_t>(),
                                            g->perm.as<int32_t>(), n, 0, 32, st));
    GI_TRY(tmp.alloc(tb));
    GI_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, rk.as<uint32_t>(), rk2.as<uint32_t>(), ids.as<int32_t>(),
                                            g->perm.as<int32_t>(), n, 0, 32, st));
    k_invert<<<grid_for(n, 256, sms), 256, 0, st>>>(g->perm.as<int32_t>(), n, g->inv.as<int32_t>());
    inv = g->inv.as<int32_t>();
  }
  // 5. owner ranges over internal ids
  {
    DevBuf w, pre;
    GI_TRY(w.alloc((n + 1) * sizeof(int64_t)));
    GI_TRY(pre.alloc((n + 1) * sizeof(int64_t)));
    k_weights<<<grid_for(n + 1, 256, sms), 256, 0, st>>>(g->relabeled ? g->perm.as<int32_t>() : nullptr,
                                                         hid.as<int32_t>(), n, w.as<int64_t>());
    tb = 0;
    GI_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, w.as<int64_t>(), pre.as<int64_t>(), n + 1, st));
    GI_TRY(tmp.alloc(tb));
    GI_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, w.as<int64_t>(), pre.as<int64_t>(), n + 1, st));
    GI_CUDA(cudaStreamSynchronize(st));
    g->bounds.assign(P + 1, 0);
    DevPrefix dp{pre.as<int64_t>()};
    partition_ranges(n, P, dev_prefix, &dp, g->bounds.data());
  }
  g->r0 = g->bounds[R];
  g->nr = g->bounds[R + 1] - g->bounds[R];
  // 6. owner shuffle
  DevBuf owner, owner2, dbounds, starts;
  GI_TRY(owner.alloc(k * sizeof(uint32_t)));
  GI_TRY(owner2.alloc(k * sizeof(uint32_t)));
  GI_TRY(dbounds.alloc((P + 1) * sizeof(int64_t)));
  GI_TRY(starts.alloc((P + 1) * sizeof(int64_t)));
  GI_CUDA(cudaMemcpyAsync(dbounds.p, g->bounds.data(), (P + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  if (k > 0) {
    k_dist_owner<<<grid_for(k, 256, sms), 256, 0, st>>>(kB.as<uint64_t>(), k, inv, dbounds.as<int64_t>(), P,
                                                       owner.as<uint32_t>(), kA.as<uint64_t>());
    int obits = 1;
    while ((1 << obits) < P) ++obits;
    tb = 0;
    GI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, owner.as<uint32_t>(), owner2.as<uint32_t>(),
                                            kA.as<uint64_t>(), kB.as<uint64_t>(), k, 0, obits, st));
    GI_TRY(tmp.alloc(tb));
    GI_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, owner.as<uint32_t>(), owner2.as<uint32_t>(),
                                            kA.as<uint64_t>(), kB.as<uint64_t>(), k, 0, obits, st));
  }
  k_owner_starts<<<1, 64, 0, st>>>(owner2.as<uint32_t>(), k, P, starts.as<int64_t>());
  std::vector<int64_t> h_starts(P + 1);
  GI_CUDA(cudaMemcpyAsync(h_starts.data(), starts.p, (P + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  // exchange the count matrix: row R = what this rank sends to each owner
  DevBuf mat;
  GI_TRY(mat.alloc((size_t)P * P * sizeof(int64_t)));
  GI_CUDA(cudaMemsetAsync(mat.p, 0, (size_t)P * P * sizeof(int64_t), st));
  std::vector<int64_t> row(P);
  for (int p = 0; p < P; ++p) row[p] = h_starts[p + 1] - h_starts[p];
  GI_CUDA(cudaMemcpyAsync(mat.as<int64_t>() + (size_t)R * P, row.data(), P * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  GI_TRY(C->allreduce_i64(mat.as<int64_t>(), (int64_t)P * P, st));
  std::vector<int64_t> h_mat((size_t)P * P);
  GI_CUDA(cudaMemcpyAsync(h_mat.data(), mat.p, (size_t)P * P * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  std::vector<int64_t> soff(P + 1), roff(P + 1);
  soff[0] = roff[0] = 0;
  for (int p = 0; p < P; ++p) {
    soff[p + 1] = soff[p] + row[p] * 8;
    roff[p + 1] = roff[p] + h_mat[(size_t)p * P + R] * 8;
  }
  const int64_t kr = roff[P] / 8;  // edges received (owned destinations)
  DevBuf recv;
  GI_TRY(recv.alloc(kr * sizeof(uint64_t)));
  GI_TRY(C->alltoallv(kB.p, soff, recv.p, roff, st));
  kA.reset();
  kB.reset();
  owner.reset();
  owner2.reset();

  // 7. local graph: CSR by source (edges into the owned range) and CSC of owned rows
  const int bits = bits_for(n > 1 ? n : 2);
  DevBuf cur, alt;
  GI_TRY(cur.alloc(kr * sizeof(uint64_t)));
  GI_TRY(alt.alloc(kr * sizeof(uint64_t)));
  if (kr > 0) k_pack_local<<<grid_for(kr, 256, sms), 256, 0, st>>>(recv.as<uint64_t>(), kr, bits, 0, 0, cur.as<uint64_t>());
  DevBuf* pc = &cur;
  DevBuf* pa = &alt;
  auto sort_keys = [&](int64_t count) -> gi_status {
    if (count <= 1) return GI_OK;
    cub::DoubleBuffer<uint64_t> db(pc->as<uint64_t>(), pa->as<uint64_t>());
    size_t b = 0;
    GI_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, b, db, count, 0, 2 * bits, st));
    GI_TRY(tmp.alloc(b));
    GI_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, b, db, count, 0, 2 * bits, st));
    if (db.Current() != pc->as<uint64_t>()) std::swap(pc, pa);
    return GI_OK;
  };
  GI_TRY(sort_keys(kr));
  int64_t ml = kr;
  if (dedup && kr > 1) {
    size_t b = 0;
    GI_CUDA(cub::DeviceSelect::Unique(nullptr, b, pc->as<uint64_t>(), pa->as<uint64_t>(), nsel.as<int64_t>(), kr, st));
    GI_TRY(tmp.alloc(b));
    GI_CUDA(cub::DeviceSelect::Unique(tmp.p, b, pc->as<uint64_t>(), pa->as<uint64_t>(), nsel.as<int64_t>(), kr, st));
    GI_CUDA(cudaMemcpyAsync(&ml, nsel.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    GI_CUDA(cudaStreamSynchronize(st));
    std::swap(pc, pa);
  }
  g->ml = ml;
  g->off64 = ml >= (int64_t)INT32_MAX || (flags & GI_OFFSETS64);
  if (g->off64) GI_TRY(csr_from_sorted<int64_t>(g, pc->as<uint64_t>(), ml, bits, n, g->csr_off, g->csr_idx));
  else GI_TRY(csr_from_sorted<int32_t>(g, pc->as<uint64_t>(), ml, bits, n, g->csr_off, g->csr_idx));
  // exact out-degrees: local row lengths summed over ranks
  GI_TRY(g->outdeg.alloc(n * sizeof(int32_t)));
  if (g->off64) k_degrees<int64_t><<<grid_for(n, 256, sms), 256, 0, st>>>(g->csr_off.as<int64_t>(), n, g->outdeg.as<int32_t>());
  else k_degrees<int32_t><<<grid_for(n, 256, sms), 256, 0, st>>>(g->csr_off.as<int32_t>(), n, g->outdeg.as<int32_t>());
  GI_TRY(C->allreduce_i32(g->outdeg.as<int32_t>(), n, st));
  DevBuf msum;
  GI_TRY(msum.alloc(sizeof(int64_t)));
  GI_CUDA(cudaMemcpyAsync(msum.p, &ml, sizeof(int64_t), cudaMemcpyHostToDevice, st));
  GI_TRY(C->allreduce_i64(msum.as<int64_t>(), 1, st));
  int64_t mg = 0;
  GI_CUDA(cudaMemcpyAsync(&mg, msum.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  g->m = mg;
  // CSC of the owned rows: ((v - r0) << b | u), sorted
  if (ml > 0)
    k_repack_transpose<<<grid_for(ml, 256, sms), 256, 0, st>>>(pc->as<uint64_t>(), ml, bits, g->r0, pa->as<uint64_t>());
  std::swap(pc, pa);
  GI_TRY(sort_keys(ml));
  if (g->off64) GI_TRY(csr_from_sorted<int64_t>(g, pc->as<uint64_t>(), ml, bits, g->nr, g->csc_off, g->csc_idx));
  else GI_TRY(csr_from_sorted<int32_t>(g, pc->as<uint64_t>(), ml, bits, g->nr, g->csc_off, g->csc_idx));
  // pull tiling over the owned rows
  g->ntiles = g->nr > 0 ? ceil_div(g->nr + ml, kPullTile) : 0;
  GI_TRY(g->tile_rows.alloc(2 * (g->ntiles > 0 ? g->ntiles : 1) * sizeof(int32_t)));
  if (g->ntiles > 0) {
    if (g->off64)
      k_tile_rows<int64_t><<<grid_for(2 * g->ntiles, 256, sms), 256, 0, st>>>(g->csc_off.as<int64_t>(), g->nr, ml,
                                                                            g->ntiles, kPullTile, g->tile_rows.as<int32_t>());
    else
      k_tile_rows<int32_t><<<grid_for(2 * g->ntiles, 256, sms), 256, 0, st>>>(g->csc_off.as<int32_t>(), g->nr, ml,
                                                                            g->ntiles, kPullTile, g->tile_rows.as<int32_t>());
  }
  GI_CUDA(cudaGetLastError());
  GI_CUDA(cudaStreamSynchronize(st));
  return GI_OK;
}

gi_status tile_rows_launch(const void* off, bool off64, int64_t n, int64_t m, int64_t ntiles, int32_t* rows,
                           cudaStream_t st, int sms) {
  if (ntiles <= 0) return GI_OK;
  if (off64)
    k_tile_rows<int64_t><<<grid_for(2 * ntiles, 256, sms), 256, 0, st>>>(static_cast<const int64_t*>(off), n, m, ntiles,
                                                                        kPullTile, rows);
  else
    k_tile_rows<int32_t><<<grid_for(2 * ntiles, 256, sms), 256, 0, st>>>(static_cast<const int32_t*>(off), n, m, ntiles,
                                                                        kPullTile, rows);
  GI_CUDA(cudaGetLastError());
  return GI_OK;
}

}  // namespace gi
