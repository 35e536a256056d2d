// comm.cu — NcclComm and LocalComm (see comm.cuh).
#include <nccl.h>

#include <algorithm>
#include <cstring>

#include "comm.cuh"
#include "nccl_dyn.cuh"

namespace gi {

gi_status Comm::peer_map(void* local, std::vector<void*>& peers, std::vector<void*>& opened, cudaStream_t st) {
  const int64_t hs = (int64_t)sizeof(cudaIpcMemHandle_t);
  std::vector<cudaIpcMemHandle_t> h(nranks);
  memset(h.data(), 0, nranks * hs);
  // local failures only raise `bad`: every rank always reaches both collectives
  int32_t bad = cudaIpcGetMemHandle(&h[rank], local) != cudaSuccess;
  cudaGetLastError();
  DevBuf hb, flag;
  GI_TRY(hb.alloc(nranks * hs));
  GI_TRY(flag.alloc(sizeof(int32_t)));
  GI_CUDA(cudaMemcpyAsync(hb.as<char>() + rank * hs, &h[rank], hs, cudaMemcpyHostToDevice, st));
  std::vector<int64_t> off(nranks + 1);
  for (int q = 0; q <= nranks; ++q) off[q] = q * hs;
  GI_TRY(allgatherv(hb.p, off, st));
  GI_CUDA(cudaMemcpyAsync(h.data(), hb.p, nranks * hs, cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  peers.assign(nranks, nullptr);
  peers[rank] = local;
  for (int q = 0; q < nranks && !bad; ++q) {
    if (q == rank) continue;
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, h[q], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      bad = 1;
      break;
    }
    peers[q] = p;
    opened.push_back(p);
  }
  GI_CUDA(cudaMemcpyAsync(flag.p, &bad, sizeof(int32_t), cudaMemcpyHostToDevice, st));
  GI_TRY(allreduce_i32(flag.as<int32_t>(), 1, st));
  int32_t any = 0;
  GI_CUDA(cudaMemcpyAsync(&any, flag.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  GI_CUDA(cudaStreamSynchronize(st));
  if (any) {
    peer_unmap(opened);
    return fail(GI_ERR_CUDA, "peer_map: CUDA IPC mapping unavailable on some rank");
  }
  return GI_OK;
}

gi_status Comm::barrier(cudaStream_t st) {
  DevBuf one;
  GI_TRY(one.alloc(sizeof(int32_t)));
  GI_CUDA(cudaMemsetAsync(one.p, 0, sizeof(int32_t), st));
  GI_TRY(allreduce_i32(one.as<int32_t>(), 1, st));
  GI_CUDA(cudaStreamSynchronize(st));
  return GI_OK;
}

void LocalGroup::barrier() {
  std::unique_lock<std::mutex> lk(mu);
  const int64_t g = gen;
  if (++arrived == n) {
    arrived = 0;
    ++gen;
    cv.notify_all();
  } else {
    cv.wait(lk, [&] { return gen != g; });
  }
}

namespace {

class NcclComm : public Comm {
 public:
  NcclComm(ncclComm_t c, int r, int p) : comm_(c) {
    rank = r;
    nranks = p;
  }
  gi_status allreduce_i32(int32_t* d, int64_t count, cudaStream_t st) override {
    return red(d, count, ncclInt32, st);
  }
  gi_status allreduce_i64(int64_t* d, int64_t count, cudaStream_t st) override {
    return red(d, count, ncclInt64, st);
  }
  gi_status allreduce_f64(double* d, int64_t count, cudaStream_t st) override {
    return red(d, count, ncclFloat64, st);
  }
  gi_status allgatherv(void* buf, const std::vector<int64_t>& off, cudaStream_t st) override {
    const NcclApi* a = nccl_api();
    if (!a) return GI_ERR_NCCL;
    char* b = static_cast<char*>(buf);
    GI_TRY(nccl_check(a->groupStart(), "ncclGroupStart"));
    for (int p = 0; p < nranks; ++p) {
      const size_t len = (size_t)(off[p + 1] - off[p]);
      if (len == 0) continue;
      GI_TRY(nccl_check(a->broadcast(b + off[p], b + off[p], len, ncclUint8, p, comm_, st), "ncclBroadcast"));
    }
    return nccl_check(a->groupEnd(), "ncclGroupEnd");
  }
  gi_status alltoallv(const void* send, const std::vector<int64_t>& soff, void* recv,
                      const std::vector<int64_t>& roff, cudaStream_t st) override {
    const NcclApi* a = nccl_api();
    if (!a) return GI_ERR_NCCL;
    const char* s = static_cast<const char*>(send);
    char* r = static_cast<char*>(recv);
    GI_TRY(nccl_check(a->groupStart(), "ncclGroupStart"));
    for (int p = 0; p < nranks; ++p) {
      const size_t sl = (size_t)(soff[p + 1] - soff[p]), rl = (size_t)(roff[p + 1] - roff[p]);
      if (sl) GI_TRY(nccl_check(a->send(s + soff[p], sl, ncclUint8, p, comm_, st), "ncclSend"));
      if (rl) GI_TRY(nccl_check(a->recv(r + roff[p], rl, ncclUint8, p, comm_, st), "ncclRecv"));
    }
    return nccl_check(a->groupEnd(), "ncclGroupEnd");
  }

 private:
  gi_status red(void* d, int64_t count, ncclDataType_t t, cudaStream_t st) {
    const NcclApi* a = nccl_api();
    if (!a) return GI_ERR_NCCL;
    if (count == 0) return GI_OK;
    return nccl_check(a->allReduce(d, d, (size_t)count, t, ncclSum, comm_, st), "ncclAllReduce");
  }
  ncclComm_t comm_;
};

class LocalComm : public Comm {
 public:
  LocalComm(LocalGroup* g, int r) : g_(g) {
    rank = r;
    nranks = g->n;
  }
  gi_status allreduce_i32(int32_t* d, int64_t count, cudaStream_t st) override { return red<int32_t>(d, count, st); }
  gi_status allreduce_i64(int64_t* d, int64_t count, cudaStream_t st) override { return red<int64_t>(d, count, st); }
  gi_status allreduce_f64(double* d, int64_t count, cudaStream_t st) override { return red<double>(d, count, st); }
  // in-process ranks: the buffers are directly addressable when every rank
  // runs on the same device (or peer access between the devices is enabled)
  gi_status peer_map(void* local, std::vector<void*>& peers, std::vector<void*>&, cudaStream_t st) override {
    GI_CUDA(cudaStreamSynchronize(st));
    int dev = -1;
    GI_CUDA(cudaGetDevice(&dev));
    g_->ptr[rank] = local;
    g_->dev[rank] = dev;
    g_->barrier();
    bool ok = true;
    for (int q = 0; q < nranks; ++q) {
      if (g_->dev[q] == dev) continue;
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, dev, g_->dev[q]) != cudaSuccess || !can) {
        ok = false;
        continue;
      }
      cudaError_t e = cudaDeviceEnablePeerAccess(g_->dev[q], 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ok = false;
    }
    cudaGetLastError();
    g_->flag[rank] = ok ? 0 : 1;
    g_->barrier();
    int any = 0;
    for (int q = 0; q < nranks; ++q) any |= g_->flag[q];
    peers.assign(nranks, nullptr);
    for (int q = 0; q < nranks; ++q) peers[q] = const_cast<void*>(g_->ptr[q]);
    g_->barrier();
    if (any) return fail(GI_ERR_CUDA, "peer_map: ranks on devices without peer access");
    return GI_OK;
  }
  gi_status barrier(cudaStream_t st) override {
    GI_CUDA(cudaStreamSynchronize(st));
    g_->barrier();
    return GI_OK;
  }
  bool peer_stores_default() const override { return true; }
  gi_status allgatherv(void* buf, const std::vector<int64_t>& off, cudaStream_t st) override {
    GI_CUDA(cudaStreamSynchronize(st));
    g_->ptr[rank] = buf;
    g_->barrier();
    char* b = static_cast<char*>(buf);
    for (int p = 0; p < nranks; ++p) {
      const int64_t len = off[p + 1] - off[p];
      if (p == rank || len == 0) continue;
      GI_CUDA(cudaMemcpyAsync(b + off[p], static_cast<const char*>(g_->ptr[p]) + off[p], len,
                              cudaMemcpyDeviceToDevice, st));
    }
    GI_CUDA(cudaStreamSynchronize(st));
    g_->barrier();
    return GI_OK;
  }
  gi_status alltoallv(const void* send, const std::vector<int64_t>& soff, void* recv,
                      const std::vector<int64_t>& roff, cudaStream_t st) override {
    GI_CUDA(cudaStreamSynchronize(st));
    g_->ptr[rank] = send;
    g_->offs[rank] = soff;
    g_->barrier();
    for (int p = 0; p < nranks; ++p) {
      const int64_t a = g_->offs[p][rank], b = g_->offs[p][rank + 1];
      if (b - a != roff[p + 1] - roff[p]) return fail(GI_ERR_INTERNAL, "alltoallv: count mismatch");
      if (b > a)
        GI_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + roff[p], static_cast<const char*>(g_->ptr[p]) + a, b - a,
                                cudaMemcpyDeviceToDevice, st));
    }
    GI_CUDA(cudaStreamSynchronize(st));
    g_->barrier();
    return GI_OK;
  }

 private:
  template <typename T>
  gi_status red(T* d, int64_t count, cudaStream_t st) {
    GI_CUDA(cudaStreamSynchronize(st));
    g_->ptr[rank] = d;
    g_->barrier();
    std::vector<T> acc((size_t)count, T(0)), tmp((size_t)count);
    for (int p = 0; p < nranks; ++p) {  // same order on every rank: identical sums
      GI_CUDA(cudaMemcpy(tmp.data(), g_->ptr[p], count * sizeof(T), cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < count; ++i) acc[i] += tmp[i];
    }
    g_->barrier();  // everyone has read every buffer before anyone overwrites its own
    GI_CUDA(cudaMemcpy(d, acc.data(), count * sizeof(T), cudaMemcpyHostToDevice));
    g_->barrier();
    return GI_OK;
  }
  LocalGroup* g_;
};

// Host-staged collectives through caller callbacks (gi_context_create_hostcomm).
// Every collective synchronises the stream, copies the device bytes to host
// memory, calls the callback, and copies the result back: no kernel ever
// waits on another rank.
class HostComm : public Comm {
 public:
  HostComm(const gi_host_comm& cb, int r, int p) : cb_(cb) {
    rank = r;
    nranks = p;
  }
  gi_status allreduce_i32(int32_t* d, int64_t count, cudaStream_t st) override { return red(d, count, 4, 0, st); }
  gi_status allreduce_i64(int64_t* d, int64_t count, cudaStream_t st) override { return red(d, count, 8, 1, st); }
  gi_status allreduce_f64(double* d, int64_t count, cudaStream_t st) override { return red(d, count, 8, 2, st); }
  gi_status allgatherv(void* buf, const std::vector<int64_t>& off, cudaStream_t st) override {
    const int64_t total = off[nranks];
    std::vector<char> h((size_t)std::max<int64_t>(total, 1));
    const int64_t a = off[rank], b = off[rank + 1];
    if (b > a) GI_CUDA(cudaMemcpyAsync(h.data() + a, static_cast<char*>(buf) + a, b - a, cudaMemcpyDeviceToHost, st));
    GI_CUDA(cudaStreamSynchronize(st));
    if (cb_.allgatherv(cb_.user, h.data(), off.data(), nranks) != 0)
      return fail(GI_ERR_NCCL, "host comm: allgatherv callback failed");
    if (total > 0) GI_CUDA(cudaMemcpyAsync(buf, h.data(), total, cudaMemcpyHostToDevice, st));
    GI_CUDA(cudaStreamSynchronize(st));
    return GI_OK;
  }
  gi_status alltoallv(const void* send, const std::vector<int64_t>& soff, void* recv,
                      const std::vector<int64_t>& roff, cudaStream_t st) override {
    std::vector<char> hs((size_t)std::max<int64_t>(soff[nranks], 1)), hr((size_t)std::max<int64_t>(roff[nranks], 1));
    if (soff[nranks] > 0) GI_CUDA(cudaMemcpyAsync(hs.data(), send, soff[nranks], cudaMemcpyDeviceToHost, st));
    GI_CUDA(cudaStreamSynchronize(st));
    if (cb_.alltoallv(cb_.user, hs.data(), soff.data(), hr.data(), roff.data(), nranks) != 0)
      return fail(GI_ERR_NCCL, "host comm: alltoallv callback failed");
    if (roff[nranks] > 0) GI_CUDA(cudaMemcpyAsync(recv, hr.data(), roff[nranks], cudaMemcpyHostToDevice, st));
    GI_CUDA(cudaStreamSynchronize(st));
    return GI_OK;
  }

 private:
  gi_status red(void* d, int64_t count, int esz, int dtype, cudaStream_t st) {
    if (count == 0) return GI_OK;
    std::vector<char> h((size_t)(count * esz));
    GI_CUDA(cudaMemcpyAsync(h.data(), d, count * esz, cudaMemcpyDeviceToHost, st));
    GI_CUDA(cudaStreamSynchronize(st));
    if (cb_.allreduce(cb_.user, h.data(), count, dtype) != 0)
      return fail(GI_ERR_NCCL, "host comm: allreduce callback failed");
    GI_CUDA(cudaMemcpyAsync(d, h.data(), count * esz, cudaMemcpyHostToDevice, st));
    GI_CUDA(cudaStreamSynchronize(st));
    return GI_OK;
  }
  gi_host_comm cb_;
};

}  // namespace

Comm* make_host_comm(const gi_host_comm& cb, int rank, int nranks) { return new HostComm(cb, rank, nranks); }

Comm* make_nccl_comm(void* nccl_comm, int rank, int nranks) {
  return new NcclComm(static_cast<ncclComm_t>(nccl_comm), rank, nranks);
}

Comm* make_local_comm(LocalGroup* g, int rank) { return new LocalComm(g, rank); }

void peer_unmap(std::vector<void*>& opened) {
  for (void* p : opened) cudaIpcCloseMemHandle(p);
  opened.clear();
}

}  // namespace gi
