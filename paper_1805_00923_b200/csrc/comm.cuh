// comm.cuh — the exchange layer of the destination-partitioned multi-GPU path
// (SURVEY §8(e), §2.7 K10-K12).
//
// Three implementations behind one interface:
//   NcclComm  — one process per GPU, NCCL over NVLink/NVSwitch: allreduce for
//               scalars and degree histograms, allgatherv (grouped in-place
//               broadcasts) for contrib / bitmap / parent slices, alltoallv
//               (grouped send/recv) for the build's owner shuffle;
//   HostComm  — the same collectives staged through host memory and performed
//               by caller-supplied callbacks (gi_context_create_hostcomm; e.g.
//               torch.distributed over gloo): any transport, any process layout,
//               including several processes sharing one GPU in tests;
//   LocalComm — P ranks as host threads of one process sharing one device
//               (tests only, gi_local_group_create): the same collectives done
//               with device-to-device copies between the ranks' buffers and a
//               host barrier. No kernel ever waits on another rank's kernel.
#pragma once
#include <condition_variable>
#include <mutex>
#include <vector>

#include "gi_internal.cuh"

namespace gi {

struct Comm {
  int rank = 0, nranks = 1;
  virtual ~Comm() {}
  // in-place sums over ranks of device arrays
  virtual gi_status allreduce_i32(int32_t* d, int64_t count, cudaStream_t st) = 0;
  virtual gi_status allreduce_i64(int64_t* d, int64_t count, cudaStream_t st) = 0;
  virtual gi_status allreduce_f64(double* d, int64_t count, cudaStream_t st) = 0;
  // in-place allgatherv: every rank ends with rank r's bytes [off[r], off[r+1]) of buf
  virtual gi_status allgatherv(void* buf, const std::vector<int64_t>& off, cudaStream_t st) = 0;
  // send bytes [soff[p], soff[p+1]) of `send` to rank p; receive rank p's bytes into
  // recv + roff[p] (counts must agree pairwise)
  virtual gi_status alltoallv(const void* send, const std::vector<int64_t>& soff, void* recv,
                              const std::vector<int64_t>& roff, cudaStream_t st) = 0;
  // Collective: every rank passes a buffer of the same size (cudaMalloc'd);
  // on GI_OK peers[q] is rank q's buffer addressable from this device
  // (peers[rank] = local) and `opened` lists mappings to release with
  // peer_unmap. Any rank failing makes every rank return GI_ERR_CUDA (the
  // collectives inside are always all executed, failure or not).
  // Default: CUDA IPC handles exchanged with allgatherv, opened with lazy peer
  // access, the outcome agreed with an allreduce.
  virtual gi_status peer_map(void* local, std::vector<void*>& peers, std::vector<void*>& opened,
                             cudaStream_t st);
  // Collective: returns on every rank after every rank has called it (and the
  // stream's earlier work has completed).
  virtual gi_status barrier(cudaStream_t st);
  // whether PageRank stores contrib into the peers' replicas unless
  // GI_PR_PEER says otherwise (the ranks agree on the final choice)
  virtual bool peer_stores_default() const { return false; }
};
void peer_unmap(std::vector<void*>& opened);

// Shared state of an in-process group of simulated ranks.
struct LocalGroup {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t gen = 0;
  std::vector<const void*> ptr;
  std::vector<int> dev, flag;
  std::vector<std::vector<int64_t>> offs;
  void barrier();
};

Comm* make_nccl_comm(void* nccl_comm, int rank, int nranks);
Comm* make_host_comm(const gi_host_comm& cb, int rank, int nranks);
Comm* make_local_comm(LocalGroup* g, int rank);

}  // namespace gi

struct gi_local_group_s {
  gi::LocalGroup g;
};
