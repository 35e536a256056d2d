// gi_api.cu — the extern "C" boundary declared in include/gi.h: argument
// validation, host/device pointer handling, error reporting, orchestration.
#include <dlfcn.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>

#include "gi_internal.cuh"
#include "nccl_dyn.cuh"
#include "comm.cuh"

namespace gi {

static thread_local std::string t_last_error;

void set_error(const std::string& msg) { t_last_error = msg; }

gi_status fail(gi_status s, const std::string& msg) {
  t_last_error = msg;
  return s;
}

gi_status cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  char buf[512];
  snprintf(buf, sizeof buf, "CUDA error %s (%d) in %s at %s:%d", cudaGetErrorString(e), (int)e, what, file, line);
  t_last_error = buf;
  if (e == cudaErrorMemoryAllocation) return GI_ERR_OUT_OF_MEMORY;
  return GI_ERR_CUDA;
}

// ---------------------------------------------------------------- big-buffer cache (gi_internal.cuh)
namespace {
struct BigEntry {
  void* p;
  size_t bytes;
  cudaStream_t s;
  int dev;
};
std::mutex g_big_mu;
std::vector<BigEntry> g_big;
size_t g_big_total = 0;
uint64_t g_big_mallocs = 0;  // cudaMalloc / cudaFree events of large blocks (free-memory checks)
// GI_DEBUG_BIGCACHE=1: one stderr line per miss / eviction (diagnostics)
bool big_debug() {
  static const bool v = getenv("GI_DEBUG_BIGCACHE") && atoi(getenv("GI_DEBUG_BIGCACHE")) != 0;
  return v;
}
size_t big_cap() {
  static const size_t v = (getenv("GI_BIGCACHE_GB") ? (size_t)atoll(getenv("GI_BIGCACHE_GB")) : 120) << 30;
  return v;
}
}  // namespace

void* big_cache_get(size_t nbytes, cudaStream_t s, size_t* got) {
  int dev = -1;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_big_mu);
  int best = -1;
  for (int i = 0; i < (int)g_big.size(); ++i) {
    const BigEntry& e = g_big[i];
    if (e.s == s && e.dev == dev && e.bytes >= nbytes && e.bytes <= 2 * nbytes &&
        (best < 0 || e.bytes < g_big[best].bytes))
      best = i;
  }
  if (best < 0) {
    if (big_debug()) fprintf(stderr, "bigcache miss %.2f GB (cached %.2f GB in %zu)\n", nbytes / 1e9, g_big_total / 1e9, g_big.size());
    return nullptr;
  }
  void* p = g_big[best].p;
  *got = g_big[best].bytes;
  g_big_total -= g_big[best].bytes;
  g_big.erase(g_big.begin() + best);
  return p;
}

void big_cache_put(void* p, size_t bytes, cudaStream_t s) {
  int dev = -1;
  cudaGetDevice(&dev);
  // the device must keep kBigMinFree bytes free for everybody else (torch's allocator,
  // other contexts): cached blocks count as used. cudaMemGetInfo can take tens of ms,
  // so it is asked only when a block was cudaMalloc'd since the last answer (a block
  // moving between use and the cache does not change the device's free memory)
  constexpr size_t kBigMinFree = 24ull << 30;
  std::vector<void*> drop;
  {
    std::lock_guard<std::mutex> lk(g_big_mu);
    static uint64_t checked = ~0ull;
    static size_t fr_seen = 0;
    if (checked != g_big_mallocs) {
      size_t f = 0, tot = 0;
      if (cudaMemGetInfo(&f, &tot) != cudaSuccess) {
        cudaGetLastError();
        f = 0;
      }
      fr_seen = f;
      checked = g_big_mallocs;
    }
    size_t fr = fr_seen;
    if (bytes > big_cap()) {
      drop.push_back(p);
    } else {
      while ((g_big_total + bytes > big_cap() || fr < kBigMinFree) && !g_big.empty()) {  // oldest first
        drop.push_back(g_big.front().p);
        fr += g_big.front().bytes;
        g_big_total -= g_big.front().bytes;
        g_big.erase(g_big.begin());
      }
      if (fr < kBigMinFree) {
        drop.push_back(p);
      } else {
        g_big.push_back(BigEntry{p, bytes, s, dev});
        g_big_total += bytes;
      }
    }
  }
  {
    std::lock_guard<std::mutex> lk(g_big_mu);
    for (size_t i = 0; i < drop.size(); ++i) ++g_big_mallocs;  // frees change the device's free memory too
  }
  if (big_debug() && !drop.empty())
    fprintf(stderr, "bigcache put %.2f GB: %zu blocks freed\n", bytes / 1e9, drop.size());
  for (void* q : drop) cudaFree(q);
}

double slow_ms() {
  static const double v = getenv("GI_DEBUG_SLOW_MS") ? atof(getenv("GI_DEBUG_SLOW_MS")) : 0.0;
  return v;
}

void slow_report(const char* what, size_t bytes, std::chrono::steady_clock::time_point t0) {
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (ms > slow_ms()) fprintf(stderr, "slow %s %.3f GB: %.1f ms\n", what, bytes / 1e9, ms);
}

void big_cache_note_malloc() {
  std::lock_guard<std::mutex> lk(g_big_mu);
  ++g_big_mallocs;
}

// frees the oldest cached block of the current device (an allocation failed):
// false when the cache holds none; the caller retries its allocation
bool big_cache_evict_one() {
  int dev = -1;
  cudaGetDevice(&dev);
  void* p = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_big_mu);
    for (size_t i = 0; i < g_big.size(); ++i)
      if (g_big[i].dev == dev) {
        p = g_big[i].p;
        g_big_total -= g_big[i].bytes;
        g_big.erase(g_big.begin() + i);
        ++g_big_mallocs;
        break;
      }
  }
  if (!p) return false;
  cudaDeviceSynchronize();  // a block of another stream may still be in use
  cudaFree(p);
  return true;
}

void big_cache_flush(cudaStream_t s) {
  int dev = -1;
  cudaGetDevice(&dev);
  std::vector<void*> drop;
  {
    std::lock_guard<std::mutex> lk(g_big_mu);
    for (int i = (int)g_big.size() - 1; i >= 0; --i)
      if (g_big[i].dev == dev && (!s || g_big[i].s == s)) {
        drop.push_back(g_big[i].p);
        g_big_total -= g_big[i].bytes;
        g_big.erase(g_big.begin() + i);
      }
  }
  if (!drop.empty()) cudaDeviceSynchronize();  // blocks of other streams may still be in use
  for (void* q : drop) cudaFree(q);
}

static bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Makes `p` (n elements of T, host or device) available on the device.
template <typename T>
static gi_status to_device(gi_context ctx, const T* p, int64_t n, DevBuf& hold, const T** out) {
  if (n == 0 || is_device_ptr(p)) {
    *out = p;
    return GI_OK;
  }
  GI_TRY(hold.alloc(n * sizeof(T)));
  GI_CUDA(cudaMemcpyAsync(hold.p, p, n * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
  *out = hold.as<T>();
  return GI_OK;
}

// Output helper: device pointer -> write in place; host pointer -> stage + D2H copy.
template <typename T>
struct OutBuf {
  T* user;
  int64_t n;
  bool dev;
  DevBuf* stage;
  gi_status prepare(gi_graph g, T** d) {
    dev = is_device_ptr(user);
    if (dev) {
      *d = user;
      return GI_OK;
    }
    if (!stage->p || stage->bytes < (size_t)n * sizeof(T)) GI_TRY(stage->alloc(n * sizeof(T)));
    *d = stage->as<T>();
    return GI_OK;
  }
  gi_status finish(gi_context ctx) {
    if (!dev && n > 0) GI_CUDA(cudaMemcpyAsync(user, stage->p, n * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
    return GI_OK;
  }
};

static gi_status sync(gi_context ctx) {
  GI_CUDA(stream_wait(ctx->stream));
  GI_CUDA(cudaGetLastError());
  return GI_OK;
}

}  // namespace gi

using namespace gi;

#define GI_GUARD_BEGIN try {
#define GI_GUARD_END                                                    \
  }                                                                     \
  catch (const std::bad_alloc&) {                                       \
    return fail(GI_ERR_OUT_OF_MEMORY, "host allocation failed");        \
  }                                                                     \
  catch (...) {                                                         \
    return fail(GI_ERR_INTERNAL, "unexpected C++ exception");           \
  }

extern "C" {

int gi_abi_version(void) { return GI_ABI_VERSION; }

const char* gi_status_string(gi_status s) {
  switch (s) {
    case GI_OK: return "GI_OK";
    case GI_ERR_INVALID_ARGUMENT: return "GI_ERR_INVALID_ARGUMENT";
    case GI_ERR_VERTEX_OUT_OF_RANGE: return "GI_ERR_VERTEX_OUT_OF_RANGE";
    case GI_ERR_OUT_OF_MEMORY: return "GI_ERR_OUT_OF_MEMORY";
    case GI_ERR_CUDA: return "GI_ERR_CUDA";
    case GI_ERR_NCCL: return "GI_ERR_NCCL";
    case GI_ERR_UNSUPPORTED: return "GI_ERR_UNSUPPORTED";
    case GI_ERR_INTERNAL: return "GI_ERR_INTERNAL";
  }
  return "GI_ERR_UNKNOWN";
}

const char* gi_last_error(void) { return t_last_error.c_str(); }

gi_status gi_context_create(int device, void* cuda_stream, gi_context* out) {
  GI_GUARD_BEGIN
  if (!out) return fail(GI_ERR_INVALID_ARGUMENT, "gi_context_create: out is NULL");
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(GI_ERR_CUDA, std::string("gi_context_create: no CUDA device (") + cudaGetErrorString(e) + ")");
  }
  if (device < 0 || device >= ndev) return fail(GI_ERR_INVALID_ARGUMENT, "gi_context_create: bad device ordinal");
  GI_CUDA(cudaSetDevice(device));
  gi_context c = new gi_context_s();
  c->device = device;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (cuda_stream) {
    c->stream = static_cast<cudaStream_t>(cuda_stream);
  } else {
    cudaError_t se = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (se != cudaSuccess) {
      delete c;
      return cuda_fail(se, "cudaStreamCreate", __FILE__, __LINE__);
    }
    c->own_stream = true;
  }
  if (pool_enabled()) {  // keep freed blocks cached (up to kPoolKeep) for the next graph or layout build
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = pool_keep();
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
  }
  cudaError_t he = cudaMallocHost(&c->h_scratch, 64 * sizeof(int64_t));
  if (he != cudaSuccess) {
    if (c->own_stream) cudaStreamDestroy(c->stream);
    delete c;
    return cuda_fail(he, "cudaMallocHost", __FILE__, __LINE__);
  }
  *out = c;
  return GI_OK;
  GI_GUARD_END
}

gi_status gi_context_destroy(gi_context ctx) {
  if (!ctx) return fail(GI_ERR_INVALID_ARGUMENT, "gi_context_destroy: NULL context");
  if (ctx->live_graphs > 0)
    return fail(GI_ERR_INVALID_ARGUMENT, "gi_context_destroy: destroy the context's graphs first");
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  big_cache_flush(ctx->stream);  // the stream's cached blocks (the stream may be destroyed below)
  delete ctx->comm;
  ctx->comm = nullptr;
  if (ctx->nccl_comm) {
    const NcclApi* a = nccl_api();
    if (a) a->commDestroy(static_cast<ncclComm_t>(ctx->nccl_comm));
    ctx->nccl_comm = nullptr;
  }
  if (ctx->h_scratch) cudaFreeHost(ctx->h_scratch);
  if (ctx->h_batch) cudaFreeHost(ctx->h_batch);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  delete ctx;
  return GI_OK;
}

gi_status gi_context_rank(gi_context ctx, int* rank, int* nranks) {
  if (!ctx || !rank || !nranks) return fail(GI_ERR_INVALID_ARGUMENT, "gi_context_rank: NULL argument");
  *rank = ctx->rank;
  *nranks = ctx->nranks;
  return GI_OK;
}

gi_status gi_graph_create(gi_context ctx, int64_t n, int64_t m0, const int32_t* src, const int32_t* dst,
                          uint32_t flags, gi_graph* out) {
  GI_GUARD_BEGIN
  if (!out) return fail(GI_ERR_INVALID_ARGUMENT, "gi_graph_create: out is NULL");
  *out = nullptr;
  if (!ctx) return fail(GI_ERR_INVALID_ARGUMENT, "gi_graph_create: NULL context");
  if (n < 0 || n > INT32_MAX) return fail(GI_ERR_INVALID_ARGUMENT, "gi_graph_create: n must be in [0, 2^31-1]");
  if (m0 < 0 || m0 >= (1ll << 40)) return fail(GI_ERR_INVALID_ARGUMENT, "gi_graph_create: bad edge count");
  if (m0 > 0 && (!src || !dst)) return fail(GI_ERR_INVALID_ARGUMENT, "gi_graph_create: NULL edge array");
  const uint32_t known = GI_EDGES_ON_DEVICE | GI_REMOVE_SELF_LOOPS | GI_DEDUP | GI_SYMMETRIZE | GI_NO_RELABEL | GI_OFFSETS64;
  if (flags & ~known) return fail(GI_ERR_INVALID_ARGUMENT, "gi_graph_create: unknown flag bits");
  if (n == 0 && m0 > 0) return fail(GI_ERR_VERTEX_OUT_OF_RANGE, "gi_graph_create: edges given but n = 0");
  GI_CUDA(cudaSetDevice(ctx->device));
  AllocScope as_(ctx->stream);
  if ((flags & GI_EDGES_ON_DEVICE) && m0 > 0 && !(is_device_ptr(src) && is_device_ptr(dst)))
    return fail(GI_ERR_INVALID_ARGUMENT, "gi_graph_create: GI_EDGES_ON_DEVICE but edges are host memory");
  gi_graph g = new gi_graph_s();
  gi_status s;
  if (m0 > 0 && !is_device_ptr(src) && !is_device_ptr(dst) && build_host_pipelined(ctx, m0, flags)) {
    s = build_graph_host(ctx, n, m0, src, dst, flags, g);  // H2D overlapped with the build
  } else {
    DevBuf hs, hd;
    const int32_t *ds = nullptr, *dd = nullptr;
    s = to_device(ctx, src, m0, hs, &ds);
    if (s == GI_OK) s = to_device(ctx, dst, m0, hd, &dd);
    if (s == GI_OK)
      s = ctx->nranks > 1 ? build_graph_dist(ctx, n, m0, ds, dd, flags, g) : build_graph(ctx, n, m0, ds, dd, flags, g);
  }
  if (s == GI_OK) s = sync(ctx);
  if (s != GI_OK) {
    delete g;
    return s;
  }
  ctx->live_graphs++;
  *out = g;
  return GI_OK;
  GI_GUARD_END
}

gi_status gi_graph_destroy(gi_graph g) {
  if (!g) return fail(GI_ERR_INVALID_ARGUMENT, "gi_graph_destroy: NULL graph");
  cudaSetDevice(g->ctx->device);
  cudaStreamSynchronize(g->ctx->stream);
  g->ctx->live_graphs--;
  gi_status s = GI_OK;
  if ((g->peer_state == 1 || g->bfs_peer_state == 1) && g->ctx->comm) {
    // other ranks store into (and map) this rank's contrib / frontier buffers:
    // every rank closes its mappings, and no rank frees before all have (collective)
    peer_unmap(g->peer_opened);
    peer_unmap(g->bfs_peer_opened);
    AllocScope as_(g->ctx->stream);
    s = g->ctx->comm->barrier(g->ctx->stream);
  }
  peer_unmap(g->peer_opened);
  peer_unmap(g->bfs_peer_opened);
  delete g;  // pooled buffers go back to the pool (stream-ordered frees)
  return s;
}

gi_status gi_graph_num_vertices(gi_graph g, int64_t* n) {
  if (!g || !n) return fail(GI_ERR_INVALID_ARGUMENT, "gi_graph_num_vertices: NULL argument");
  *n = g->n;
  return GI_OK;
}

gi_status gi_graph_num_edges(gi_graph g, int64_t* m) {
  if (!g || !m) return fail(GI_ERR_INVALID_ARGUMENT, "gi_graph_num_edges: NULL argument");
  *m = g->m;
  return GI_OK;
}

}  // extern "C"

namespace gi {
namespace {
__global__ void k_degree_out(const int32_t* __restrict__ deg_int, const int32_t* __restrict__ perm, int64_t n,
                             int32_t* __restrict__ out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    out[perm ? perm[v] : v] = deg_int[v];
}

template <typename OffT>
__global__ void k_indeg(const OffT* __restrict__ off, const int32_t* __restrict__ perm, int64_t n,
                        int32_t* __restrict__ out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    out[perm ? perm[v] : v] = (int32_t)(off[v + 1] - off[v]);
}

// CSR in input ids: row lengths first (scan on host side of the caller), then
// *out = min(*out, a[0..n)) (the caller initialises *out)
__global__ void k_min_i32(const int32_t* __restrict__ a, int64_t n, int32_t* __restrict__ out) {
  int32_t v = INT32_MAX;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v = min(v, a[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0 && v != INT32_MAX) atomicMin(out, v);
}
// rows copied with ids mapped back and sorted per row.
template <typename OffT>
__global__ void k_csr_export(const OffT* __restrict__ off, const int32_t* __restrict__ idx,
                             const int32_t* __restrict__ perm, const int32_t* __restrict__ inv, int64_t n,
                             const int64_t* __restrict__ out_off, int32_t* __restrict__ out_idx) {
  // one warp per input-id row
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u_in = warp; u_in < n; u_in += nw) {
    const int64_t u = inv ? inv[u_in] : u_in;
    const int64_t b = off[u], e = off[u + 1], o = out_off[u_in];
    for (int64_t j = b + lane; j < e; j += 32) out_idx[o + (j - b)] = perm ? perm[idx[j]] : idx[j];
  }
}
}  // namespace
}  // namespace gi


#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_radix_sort.cuh>

namespace gi {
// The cleaned CSR in input ids (rows ascending, neighbours ascending):
// off int64[n+1], idx int32[m], device buffers (gi_graph_csr, explicit SSSP weights).
gi_status csr_input_ids(gi_graph g, DevBuf& doff, DevBuf& didx) {
  gi_context ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  const int64_t n = g->n, m = g->m;
  const int sms = ctx->num_sms;
  DevBuf deg, didx2, tmp;
  GI_TRY(deg.alloc((n + 1) * sizeof(int32_t)));
  GI_TRY(doff.alloc((n + 1) * sizeof(int64_t)));
  GI_TRY(didx.alloc(m * sizeof(int32_t)));
  GI_TRY(didx2.alloc(m * sizeof(int32_t)));
  const int32_t* perm = g->relabeled ? g->perm.as<int32_t>() : nullptr;
  const int32_t* inv = g->relabeled ? g->inv.as<int32_t>() : nullptr;
  GI_CUDA(cudaMemsetAsync(deg.p, 0, (n + 1) * sizeof(int32_t), st));
  if (n > 0)
    k_degree_out<<<grid_for(n, 256, sms), 256, 0, st>>>(g->outdeg.as<int32_t>(), perm, n, deg.as<int32_t>());
  size_t tb = 0;
  GI_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, deg.as<int32_t>(), doff.as<int64_t>(), n + 1, st));
  GI_TRY(tmp.alloc(tb));
  GI_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, deg.as<int32_t>(), doff.as<int64_t>(), n + 1, st));
  if (n > 0 && m > 0) {
    if (g->off64)
      k_csr_export<int64_t><<<grid_for(n * 32, 256, sms), 256, 0, st>>>(g->csr_off.as<int64_t>(), g->csr_idx.as<int32_t>(),
                                                                     perm, inv, n, doff.as<int64_t>(), didx.as<int32_t>());
    else
      k_csr_export<int32_t><<<grid_for(n * 32, 256, sms), 256, 0, st>>>(g->csr_off.as<int32_t>(), g->csr_idx.as<int32_t>(),
                                                                     perm, inv, n, doff.as<int64_t>(), didx.as<int32_t>());
    if (perm) {  // rows must be ascending in input ids
      size_t sb = 0;
      GI_CUDA(cub::DeviceSegmentedRadixSort::SortKeys(nullptr, sb, didx.as<int32_t>(), didx2.as<int32_t>(), m, n,
                                                      doff.as<int64_t>(), doff.as<int64_t>() + 1, 0, 32, st));
      DevBuf tmp2;
      GI_TRY(tmp2.alloc(sb));
      GI_CUDA(cub::DeviceSegmentedRadixSort::SortKeys(tmp2.p, sb, didx.as<int32_t>(), didx2.as<int32_t>(), m, n,
                                                      doff.as<int64_t>(), doff.as<int64_t>() + 1, 0, 32, st));
      GI_CUDA(cudaStreamSynchronize(st));
      std::swap(didx.p, didx2.p);
      std::swap(didx.bytes, didx2.bytes);
      std::swap(didx.cap, didx2.cap);
      std::swap(didx.pooled, didx2.pooled);
      std::swap(didx.cached, didx2.cached);
      std::swap(didx.s, didx2.s);
    }
  }
  GI_CUDA(cudaGetLastError());
  return GI_OK;
}
}  // namespace gi

extern "C" {

gi_status gi_graph_out_degrees(gi_graph g, int32_t* outdeg) {
  GI_GUARD_BEGIN
  if (!g || (!outdeg && g->n > 0)) return fail(GI_ERR_INVALID_ARGUMENT, "gi_graph_out_degrees: NULL argument");
  gi_context ctx = g->ctx;
  GI_CUDA(cudaSetDevice(ctx->device));
  AllocScope as_(ctx->stream);
  if (g->n == 0) return GI_OK;
  OutBuf<int32_t> ob{outdeg, g->n, false, &g->out_stage};
  int32_t* d = nullptr;
  GI_TRY(ob.prepare(g, &d));
  k_degree_out<<<grid_for(g->n, 256, ctx->num_sms), 256, 0, ctx->stream>>>(
      g->outdeg.as<int32_t>(), g->relabeled ? g->perm.as<int32_t>() : nullptr, g->n, d);
  GI_CUDA(cudaGetLastError());
  GI_TRY(ob.finish(ctx));
  return sync(ctx);
  GI_GUARD_END
}

gi_status gi_graph_in_degrees(gi_graph g, int32_t* indeg) {
  GI_GUARD_BEGIN
  if (!g || (!indeg && g->n > 0)) return fail(GI_ERR_INVALID_ARGUMENT, "gi_graph_in_degrees: NULL argument");
  if (g->ctx->nranks > 1) return fail(GI_ERR_UNSUPPORTED, "gi_graph_in_degrees: single-GPU graphs only");
  gi_context ctx = g->ctx;
  GI_CUDA(cudaSetDevice(ctx->device));
  AllocScope as_(ctx->stream);
  if (g->n == 0) return GI_OK;
  OutBuf<int32_t> ob{indeg, g->n, false, &g->out_stage};
  int32_t* d = nullptr;
  GI_TRY(ob.prepare(g, &d));
  const int32_t* perm = g->relabeled ? g->perm.as<int32_t>() : nullptr;
  if (g->off64)
    k_indeg<int64_t><<<grid_for(g->n, 256, ctx->num_sms), 256, 0, ctx->stream>>>(g->csc_off.as<int64_t>(), perm, g->n, d);
  else
    k_indeg<int32_t><<<grid_for(g->n, 256, ctx->num_sms), 256, 0, ctx->stream>>>(g->csc_off.as<int32_t>(), perm, g->n, d);
  GI_CUDA(cudaGetLastError());
  GI_TRY(ob.finish(ctx));
  return sync(ctx);
  GI_GUARD_END
}

gi_status gi_graph_csr(gi_graph g, int64_t* off, int32_t* idx) {
  GI_GUARD_BEGIN
  if (!g || !off || (!idx && g->m > 0)) return fail(GI_ERR_INVALID_ARGUMENT, "gi_graph_csr: NULL argument");
  if (g->ctx->nranks > 1) return fail(GI_ERR_UNSUPPORTED, "gi_graph_csr: single-GPU graphs only");
  gi_context ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  GI_CUDA(cudaSetDevice(ctx->device));
  AllocScope as_(ctx->stream);
  const int64_t n = g->n, m = g->m;
  DevBuf doff, didx;
  GI_TRY(csr_input_ids(g, doff, didx));
  GI_CUDA(cudaMemcpyAsync(off, doff.p, (n + 1) * sizeof(int64_t), is_device_ptr(off) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
  if (m > 0)
    GI_CUDA(cudaMemcpyAsync(idx, didx.p, m * sizeof(int32_t), is_device_ptr(idx) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
  return sync(ctx);
  GI_GUARD_END
}

gi_status gi_pagerank_ex(gi_graph g, int32_t iters, double damping, const gi_pr_opts* opts, float* out,
                         gi_pr_stats* stats) {
  GI_GUARD_BEGIN
  if (!g) return fail(GI_ERR_INVALID_ARGUMENT, "gi_pagerank: NULL graph");
  if (!out && g->n > 0) return fail(GI_ERR_INVALID_ARGUMENT, "gi_pagerank: NULL output");
  if (iters < 0) return fail(GI_ERR_INVALID_ARGUMENT, "gi_pagerank: iters < 0");
  if (!(damping >= 0.0 && damping <= 1.0)) return fail(GI_ERR_INVALID_ARGUMENT, "gi_pagerank: damping not in [0,1]");
  gi_pr_opts o{};
  if (opts) o = *opts;
  if (o.direction < GI_PR_PULL || o.direction > GI_PR_PULL_BLOCKED)
    return fail(GI_ERR_INVALID_ARGUMENT, "gi_pagerank: bad direction");
  if (o.dangling != GI_DANGLING_UNIFORM && o.dangling != GI_DANGLING_DROP)
    return fail(GI_ERR_INVALID_ARGUMENT, "gi_pagerank: bad dangling rule");
  if (o.segment_size < 0 || o.dst_block < 0)
    return fail(GI_ERR_INVALID_ARGUMENT, "gi_pagerank: segment_size / dst_block < 0");
  gi_context ctx = g->ctx;
  GI_CUDA(cudaSetDevice(ctx->device));
  AllocScope as_(ctx->stream);
  OutBuf<float> ob{out, g->n, false, &g->out_stage};
  float* d = nullptr;
  if (g->n > 0) GI_TRY(ob.prepare(g, &d));
  GI_TRY(pagerank_run(g, iters, damping, o, d, stats));
  GI_TRY(ob.finish(ctx));
  return sync(ctx);
  GI_GUARD_END
}

gi_status gi_pagerank_delta(gi_graph g, int32_t iters, double damping, double epsilon, const gi_prdelta_opts* opts,
                            float* out, gi_prdelta_stats* stats) {
  GI_GUARD_BEGIN
  if (!g) return fail(GI_ERR_INVALID_ARGUMENT, "gi_pagerank_delta: NULL graph");
  if (!out && g->n > 0) return fail(GI_ERR_INVALID_ARGUMENT, "gi_pagerank_delta: NULL output");
  if (iters < 0) return fail(GI_ERR_INVALID_ARGUMENT, "gi_pagerank_delta: iters < 0");
  if (!(damping >= 0.0 && damping <= 1.0)) return fail(GI_ERR_INVALID_ARGUMENT, "gi_pagerank_delta: damping not in [0,1]");
  if (!(epsilon >= 0.0)) return fail(GI_ERR_INVALID_ARGUMENT, "gi_pagerank_delta: epsilon < 0");
  gi_prdelta_opts o{};
  if (opts) o = *opts;
  if (o.policy < GI_PRD_AUTO || o.policy > GI_PRD_PULL_ONLY || o.threshold_div < 0)
    return fail(GI_ERR_INVALID_ARGUMENT, "gi_pagerank_delta: bad options");
  gi_context ctx = g->ctx;
  GI_CUDA(cudaSetDevice(ctx->device));
  AllocScope as_(ctx->stream);
  if (g->n == 0) {
    if (stats) *stats = gi_prdelta_stats{};
    return GI_OK;
  }
  OutBuf<float> ob{out, g->n, false, &g->out_stage};
  float* d = nullptr;
  GI_TRY(ob.prepare(g, &d));
  GI_TRY(prdelta_run(g, iters, damping, epsilon, o, d, stats));
  GI_TRY(ob.finish(ctx));
  return sync(ctx);
  GI_GUARD_END
}

gi_status gi_pagerank(gi_graph g, int32_t iters, double damping, float* out) {
  return gi_pagerank_ex(g, iters, damping, nullptr, out, nullptr);
}

gi_status gi_cc_ex(gi_graph g, const gi_cc_opts* opts, int32_t* labels_out, gi_cc_stats* stats) {
  GI_GUARD_BEGIN
  if (!g) return fail(GI_ERR_INVALID_ARGUMENT, "gi_cc: NULL graph");
  if (!labels_out && g->n > 0) return fail(GI_ERR_INVALID_ARGUMENT, "gi_cc: NULL output");
  gi_cc_opts o{};
  if (opts) o = *opts;
  if (o.policy < GI_BFS_AUTO || o.policy > GI_BFS_PULL_ONLY || o.threshold_div < 0)
    return fail(GI_ERR_INVALID_ARGUMENT, "gi_cc: bad options");
  gi_context ctx = g->ctx;
  if (ctx->nranks > 1) return fail(GI_ERR_UNSUPPORTED, "gi_cc: single-GPU contexts only");
  if (g->n == 0) {
    if (stats) *stats = gi_cc_stats{};
    return GI_OK;
  }
  GI_CUDA(cudaSetDevice(ctx->device));
  AllocScope as_(ctx->stream);
  OutBuf<int32_t> ob{labels_out, g->n, false, &g->out_stage};
  int32_t* d = nullptr;
  GI_TRY(ob.prepare(g, &d));
  GI_TRY(cc_run(g, o, d, stats));
  GI_TRY(ob.finish(ctx));
  return sync(ctx);
  GI_GUARD_END
}

gi_status gi_cc(gi_graph g, int32_t* labels_out) { return gi_cc_ex(g, nullptr, labels_out, nullptr); }

gi_status gi_sssp_ex(gi_graph g, int32_t source, uint64_t weight_seed, const gi_sssp_opts* opts, int32_t* dist_out,
                     gi_sssp_stats* stats) {
  GI_GUARD_BEGIN
  if (!g) return fail(GI_ERR_INVALID_ARGUMENT, "gi_sssp: NULL graph");
  if (!dist_out) return fail(GI_ERR_INVALID_ARGUMENT, "gi_sssp: NULL output");
  if (source < 0 || source >= g->n) return fail(GI_ERR_VERTEX_OUT_OF_RANGE, "gi_sssp: source not in [0, n)");
  gi_sssp_opts o{};
  if (opts) o = *opts;
  if (o.policy < GI_BFS_AUTO || o.policy > GI_BFS_PULL_ONLY || o.threshold_div < 0)
    return fail(GI_ERR_INVALID_ARGUMENT, "gi_sssp: bad options");
  gi_context ctx = g->ctx;
  if (ctx->nranks > 1) return fail(GI_ERR_UNSUPPORTED, "gi_sssp: single-GPU contexts only");
  GI_CUDA(cudaSetDevice(ctx->device));
  AllocScope as_(ctx->stream);
  OutBuf<int32_t> ob{dist_out, g->n, false, &g->out_stage};
  int32_t* d = nullptr;
  GI_TRY(ob.prepare(g, &d));
  GI_TRY(sssp_run(g, source, weight_seed, nullptr, o, d, stats));
  GI_TRY(ob.finish(ctx));
  return sync(ctx);
  GI_GUARD_END
}

gi_status gi_sssp_weighted(gi_graph g, int32_t source, const int32_t* weights, const gi_sssp_opts* opts,
                           int32_t* dist_out, gi_sssp_stats* stats) {
  GI_GUARD_BEGIN
  if (!g) return fail(GI_ERR_INVALID_ARGUMENT, "gi_sssp_weighted: NULL graph");
  if (!dist_out) return fail(GI_ERR_INVALID_ARGUMENT, "gi_sssp_weighted: NULL output");
  if (!weights && g->m > 0) return fail(GI_ERR_INVALID_ARGUMENT, "gi_sssp_weighted: NULL weights");
  if (source < 0 || source >= g->n) return fail(GI_ERR_VERTEX_OUT_OF_RANGE, "gi_sssp_weighted: source not in [0, n)");
  gi_sssp_opts o{};
  if (opts) o = *opts;
  if (o.policy < GI_BFS_AUTO || o.policy > GI_BFS_PULL_ONLY || o.threshold_div < 0)
    return fail(GI_ERR_INVALID_ARGUMENT, "gi_sssp_weighted: bad options");
  gi_context ctx = g->ctx;
  if (ctx->nranks > 1) return fail(GI_ERR_UNSUPPORTED, "gi_sssp_weighted: single-GPU contexts only");
  GI_CUDA(cudaSetDevice(ctx->device));
  AllocScope as_(ctx->stream);
  DevBuf hold, mn;
  const int32_t* dw = nullptr;
  GI_TRY(to_device(ctx, weights, g->m, hold, &dw));
  if (g->m > 0) {  // weights must be >= 0 (the frontier Bellman-Ford's fixed point is then the shortest paths)
    GI_TRY(mn.alloc(sizeof(int32_t)));
    GI_CUDA(cudaMemsetAsync(mn.p, 0x7F, sizeof(int32_t), ctx->stream));
    k_min_i32<<<grid_for(g->m, 256, ctx->num_sms), 256, 0, ctx->stream>>>(dw, g->m, mn.as<int32_t>());
    int32_t hmin = 0;
    GI_CUDA(cudaMemcpyAsync(&hmin, mn.p, sizeof hmin, cudaMemcpyDeviceToHost, ctx->stream));
    GI_CUDA(cudaStreamSynchronize(ctx->stream));
    if (hmin < 0) return fail(GI_ERR_INVALID_ARGUMENT, "gi_sssp_weighted: negative edge weight");
  }
  OutBuf<int32_t> ob{dist_out, g->n, false, &g->out_stage};
  int32_t* d = nullptr;
  GI_TRY(ob.prepare(g, &d));
  GI_TRY(sssp_run(g, source, 0, dw, o, d, stats));
  GI_TRY(ob.finish(ctx));
  return sync(ctx);
  GI_GUARD_END
}

gi_status gi_sssp(gi_graph g, int32_t source, uint64_t weight_seed, int32_t* dist_out) {
  return gi_sssp_ex(g, source, weight_seed, nullptr, dist_out, nullptr);
}

gi_status gi_bfs_ex(gi_graph g, int32_t source, const gi_bfs_opts* opts, int32_t* parent_out, gi_bfs_stats* stats) {
  GI_GUARD_BEGIN
  if (!g) return fail(GI_ERR_INVALID_ARGUMENT, "gi_bfs: NULL graph");
  if (!parent_out) return fail(GI_ERR_INVALID_ARGUMENT, "gi_bfs: NULL output");
  if (source < 0 || source >= g->n) return fail(GI_ERR_VERTEX_OUT_OF_RANGE, "gi_bfs: source not in [0, n)");
  gi_bfs_opts o{};
  if (opts) o = *opts;
  if (o.policy < GI_BFS_AUTO || o.policy > GI_BFS_PULL_ONLY || o.threshold_div < 0)
    return fail(GI_ERR_INVALID_ARGUMENT, "gi_bfs: bad options");
  gi_context ctx = g->ctx;
  GI_CUDA(cudaSetDevice(ctx->device));
  AllocScope as_(ctx->stream);
  OutBuf<int32_t> ob{parent_out, g->n, false, &g->out_stage};
  int32_t* d = nullptr;
  GI_TRY(ob.prepare(g, &d));
  GI_TRY(bfs_run(g, source, o, d, stats));
  GI_TRY(ob.finish(ctx));
  return sync(ctx);
  GI_GUARD_END
}

gi_status gi_bfs(gi_graph g, int32_t source, int32_t* parent_out) {
  return gi_bfs_ex(g, source, nullptr, parent_out, nullptr);
}

gi_status gi_bfs_multi(gi_graph g, int32_t k, const int32_t* sources, const gi_bfs_opts* opts, int32_t* parents_out,
                       gi_bfs_stats* stats) {
  GI_GUARD_BEGIN
  if (!g) return fail(GI_ERR_INVALID_ARGUMENT, "gi_bfs_multi: NULL graph");
  if (k < 0) return fail(GI_ERR_INVALID_ARGUMENT, "gi_bfs_multi: k < 0");
  if (k == 0) return GI_OK;
  if (!sources || !parents_out) return fail(GI_ERR_INVALID_ARGUMENT, "gi_bfs_multi: NULL sources / output");
  if (is_device_ptr(sources)) return fail(GI_ERR_INVALID_ARGUMENT, "gi_bfs_multi: sources must be host memory");
  for (int32_t i = 0; i < k; ++i)
    if (sources[i] < 0 || sources[i] >= g->n)
      return fail(GI_ERR_VERTEX_OUT_OF_RANGE, "gi_bfs_multi: a source is not in [0, n)");
  gi_bfs_opts o{};
  if (opts) o = *opts;
  if (o.policy < GI_BFS_AUTO || o.policy > GI_BFS_PULL_ONLY || o.threshold_div < 0 ||
      o.batch < GI_BFS_BATCH_AUTO || o.batch > GI_BFS_BATCH_BITPARALLEL || o.pull_kernel < GI_MS_PULL_AUTO ||
      o.pull_kernel > GI_MS_PULL_SEGMENTED)
    return fail(GI_ERR_INVALID_ARGUMENT, "gi_bfs_multi: bad options");
  const bool bitpar = o.batch == GI_BFS_BATCH_BITPARALLEL || (o.batch == GI_BFS_BATCH_AUTO && k >= 8);
  gi_context ctx = g->ctx;
  GI_CUDA(cudaSetDevice(ctx->device));
  AllocScope as_(ctx->stream);
  static const char* impl = getenv("GI_BFS_IMPL");
  if (ctx->nranks > 1 || (impl && strcmp(impl, "host") == 0)) {  // one call per source
    for (int32_t i = 0; i < k; ++i) {
      OutBuf<int32_t> ob{parents_out + (int64_t)i * g->n, g->n, false, &g->out_stage};
      int32_t* d = nullptr;
      GI_TRY(ob.prepare(g, &d));
      GI_TRY(bfs_run(g, sources[i], o, d, stats ? stats + i : nullptr));
      GI_TRY(ob.finish(ctx));
      GI_TRY(sync(ctx));
    }
    return GI_OK;
  }
  auto run = [&](int32_t* rows) {
    return bitpar ? msbfs_run(g, k, sources, o, rows, stats) : bfs_fused_multi(g, k, sources, o, rows, g->n, stats);
  };
  if (is_device_ptr(parents_out)) {
    GI_TRY(run(parents_out));
  } else {  // host output: stage all k rows on the device, one copy back
    DevBuf& stage = g->fused.mstage;
    const size_t bytes = (size_t)k * g->n * sizeof(int32_t);
    if (stage.bytes < bytes) GI_TRY(stage.alloc(bytes));
    GI_TRY(run(stage.as<int32_t>()));
    GI_CUDA(cudaMemcpyAsync(parents_out, stage.p, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  }
  return sync(ctx);
  GI_GUARD_END
}

}  // extern "C"

namespace gi {

void partition_ranges(int64_t n, int nranks, int64_t (*prefix)(void*, int64_t), void* ctx, int64_t* bounds) {
  bounds[0] = 0;
  bounds[nranks] = n;
  const int64_t total = prefix(ctx, n);
  for (int r = 1; r < nranks; ++r) {
    const long double target = (long double)total * r / nranks;
    int64_t lo = 0, hi = n;  // first i with prefix(i) >= target
    while (lo < hi) {
      const int64_t mid = lo + (hi - lo) / 2;
      if ((long double)prefix(ctx, mid) >= target) hi = mid;
      else lo = mid + 1;
    }
    int64_t b = (lo + 31) / 32 * 32;  // whole bitmap words per rank
    b = std::min(std::max(b, bounds[r - 1]), n);
    bounds[r] = b;
  }
}

}  // namespace gi

static int64_t host_prefix(void* ctx, int64_t i) { return static_cast<const int64_t*>(ctx)[i]; }

extern "C" {

gi_status gi_partition_ranges(int64_t n, int nranks, const int64_t* weight_prefix, int64_t* bounds) {
  if (n < 0 || nranks < 1 || !weight_prefix || !bounds)
    return fail(GI_ERR_INVALID_ARGUMENT, "gi_partition_ranges: bad argument");
  partition_ranges(n, nranks, host_prefix, const_cast<int64_t*>(weight_prefix), bounds);
  return GI_OK;
}

gi_status gi_local_group_create(int nranks, gi_local_group* out) {
  GI_GUARD_BEGIN
  if (!out || nranks < 1) return fail(GI_ERR_INVALID_ARGUMENT, "gi_local_group_create: bad argument");
  gi_local_group grp = new gi_local_group_s();
  grp->g.n = nranks;
  grp->g.ptr.assign(nranks, nullptr);
  grp->g.offs.assign(nranks, {});
  grp->g.dev.assign(nranks, -1);
  grp->g.flag.assign(nranks, 0);
  *out = grp;
  return GI_OK;
  GI_GUARD_END
}

gi_status gi_local_group_destroy(gi_local_group grp) {
  if (!grp) return fail(GI_ERR_INVALID_ARGUMENT, "gi_local_group_destroy: NULL group");
  delete grp;
  return GI_OK;
}

gi_status gi_context_create_local(int device, void* cuda_stream, gi_local_group grp, int rank, gi_context* out) {
  GI_GUARD_BEGIN
  if (!out || !grp || rank < 0 || rank >= grp->g.n)
    return fail(GI_ERR_INVALID_ARGUMENT, "gi_context_create_local: bad argument");
  *out = nullptr;
  gi_context c = nullptr;
  GI_TRY(gi_context_create(device, cuda_stream, &c));
  c->rank = rank;
  c->nranks = grp->g.n;
  if (c->nranks > 1) c->comm = make_local_comm(&grp->g, rank);
  *out = c;
  return GI_OK;
  GI_GUARD_END
}

gi_status gi_context_create_hostcomm(int device, void* cuda_stream, int rank, int nranks, const gi_host_comm* comm,
                                     gi_context* out) {
  GI_GUARD_BEGIN
  if (!out || !comm || !comm->allreduce || !comm->allgatherv || !comm->alltoallv)
    return fail(GI_ERR_INVALID_ARGUMENT, "gi_context_create_hostcomm: NULL argument or callback");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return fail(GI_ERR_INVALID_ARGUMENT, "gi_context_create_hostcomm: bad rank / nranks");
  gi_context c = nullptr;
  GI_TRY(gi_context_create(device, cuda_stream, &c));
  c->rank = rank;
  c->nranks = nranks;
  if (nranks > 1) c->comm = make_host_comm(*comm, rank, nranks);
  *out = c;
  return GI_OK;
  GI_GUARD_END
}

gi_status gi_graph_partition(gi_graph g, int64_t* lo, int64_t* hi, int64_t* local_edges) {
  if (!g || !lo || !hi || !local_edges) return fail(GI_ERR_INVALID_ARGUMENT, "gi_graph_partition: NULL argument");
  *lo = g->r0;
  *hi = g->r0 + g->nr;
  *local_edges = g->ml;
  return GI_OK;
}

}  // extern "C"
