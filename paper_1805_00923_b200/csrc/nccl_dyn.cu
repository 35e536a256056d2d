// nccl_dyn.cu — NCCL loaded at run time (dlopen "libnccl.so.2").
//
// The library does not link NCCL: when torch has already loaded its NCCL the
// dlopen returns that same image, otherwise the system one is used. Only the
// handful of entry points the multi-GPU path needs are resolved
// (allgather of contrib / bitmap slices, allreduce of
// scalars, grouped send/recv for the build shuffle).
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>

#include "gi_internal.cuh"
#include "nccl_dyn.cuh"
#include "comm.cuh"

namespace gi {

static NcclApi g_api;
static std::once_flag g_once;
static std::string g_err;

static void load() {
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  for (const char* nm : names) {
    h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (h) break;
  }
  if (!h) {
    g_err = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
    return;
  }
#define GI_SYM(field, name)                                                 \
  g_api.field = reinterpret_cast<decltype(g_api.field)>(dlsym(h, name));    \
  if (!g_api.field) {                                                       \
    g_err = std::string("NCCL symbol missing: ") + name;                    \
    return;                                                                 \
  }
  GI_SYM(getUniqueId, "ncclGetUniqueId");
  GI_SYM(commInitRank, "ncclCommInitRank");
  GI_SYM(commDestroy, "ncclCommDestroy");
  GI_SYM(allGather, "ncclAllGather");
  GI_SYM(allReduce, "ncclAllReduce");
  GI_SYM(broadcast, "ncclBroadcast");
  GI_SYM(send, "ncclSend");
  GI_SYM(recv, "ncclRecv");
  GI_SYM(groupStart, "ncclGroupStart");
  GI_SYM(groupEnd, "ncclGroupEnd");
  GI_SYM(getErrorString, "ncclGetErrorString");
#undef GI_SYM
  g_api.ok = true;
}

const NcclApi* nccl_api() {
  std::call_once(g_once, load);
  if (!g_api.ok) {
    fail(GI_ERR_NCCL, g_err);
    return nullptr;
  }
  return &g_api;
}

gi_status nccl_check(int r, const char* what) {
  if (r == 0) return GI_OK;
  const NcclApi* a = nccl_api();
  std::string msg = std::string(what) + ": " + (a ? a->getErrorString((ncclResult_t)r) : "NCCL error");
  return fail(GI_ERR_NCCL, msg);
}

}  // namespace gi

using namespace gi;

extern "C" {

gi_status gi_nccl_unique_id(unsigned char id[128]) {
  if (!id) return fail(GI_ERR_INVALID_ARGUMENT, "gi_nccl_unique_id: NULL id");
  const NcclApi* a = nccl_api();
  if (!a) return GI_ERR_NCCL;
  ncclUniqueId u;
  GI_TRY(nccl_check(a->getUniqueId(&u), "ncclGetUniqueId"));
  static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
  memcpy(id, &u, 128);
  return GI_OK;
}

gi_status gi_context_create_dist(int device, void* cuda_stream, int rank, int nranks, const unsigned char id[128],
                                 gi_context* out) {
  if (!out || !id) return fail(GI_ERR_INVALID_ARGUMENT, "gi_context_create_dist: NULL argument");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return fail(GI_ERR_INVALID_ARGUMENT, "gi_context_create_dist: bad rank / nranks");
  gi_context c = nullptr;
  GI_TRY(gi_context_create(device, cuda_stream, &c));
  c->rank = rank;
  c->nranks = nranks;
  if (nranks > 1) {
    const NcclApi* a = nccl_api();
    if (!a) {
      gi_context_destroy(c);
      return GI_ERR_NCCL;
    }
    ncclUniqueId u;
    memcpy(&u, id, 128);
    ncclComm_t comm = nullptr;
    gi_status s = nccl_check(a->commInitRank(&comm, nranks, u, rank), "ncclCommInitRank");
    if (s != GI_OK) {
      gi_context_destroy(c);
      return s;
    }
    c->nccl_comm = comm;
    c->comm = make_nccl_comm(comm, rank, nranks);
  }
  *out = c;
  return GI_OK;
}

}  // extern "C"
