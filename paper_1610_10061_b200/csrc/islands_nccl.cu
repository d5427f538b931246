// K4 native exchange: the island allgather of pm_run_ga_islands over NCCL
// (one communicator per rank/GPU), for C/C++ hosts that do not run
// torch.distributed.  Replaces the reference's in-process worker pool merge
// (ga.cpp:253-282): every rank receives all block-best records and computes
// the same global best.
//
// NCCL is bound at run time (dlopen on first use), not linked: a process that
// loads this library before PyTorch would otherwise pin the system libnccl.so.2
// and torch's own (newer) NCCL could no longer resolve its symbols.  If a
// libnccl.so.2 is already loaded (e.g. torch's), that one is used.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "../../include/pmedian_b200.h"

struct pm_nccl {
  ncclComm_t comm = nullptr;
  cudaStream_t stream = nullptr;
  unsigned char* dbuf = nullptr;  // world * bytes
  size_t cap = 0;
  int rank = 0, world = 1, device = 0;
};

static_assert(PM_NCCL_ID_BYTES == NCCL_UNIQUE_ID_BYTES, "NCCL unique id size");

namespace {

struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_gather;
  });
  return api;
}

}  // namespace

extern "C" {

int pm_nccl_unique_id(char id[PM_NCCL_ID_BYTES]) {
  if (!nccl().ok) return PM_NCCL;
  ncclUniqueId u;
  if (nccl().get_unique_id(&u) != ncclSuccess) return PM_NCCL;
  std::memcpy(id, u.internal, PM_NCCL_ID_BYTES);
  return PM_OK;
}

int pm_nccl_create(const char id[PM_NCCL_ID_BYTES], int rank, int world, int device, pm_nccl** out) {
  if (!out || world < 1 || rank < 0 || rank >= world) return PM_DOMAIN;
  *out = nullptr;
  if (!nccl().ok) return PM_NCCL;
  if (cudaSetDevice(device) != cudaSuccess) return PM_CUDA;
  pm_nccl* c = new pm_nccl;
  c->rank = rank;
  c->world = world;
  c->device = device;
  ncclUniqueId u;
  std::memcpy(u.internal, id, PM_NCCL_ID_BYTES);
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return PM_CUDA;
  }
  if (nccl().comm_init_rank(&c->comm, world, u, rank) != ncclSuccess) {
    cudaStreamDestroy(c->stream);
    delete c;
    return PM_NCCL;
  }
  *out = c;
  return PM_OK;
}

void pm_nccl_destroy(pm_nccl* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->comm) nccl().comm_destroy(c->comm);
  if (c->dbuf) cudaFree(c->dbuf);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

int pm_nccl_allgather(const void* send, size_t bytes, void* recv, void* user) {
  pm_nccl* c = static_cast<pm_nccl*>(user);
  if (!c || (!send && bytes)) return PM_NCCL;
  if (cudaSetDevice(c->device) != cudaSuccess) return PM_CUDA;
  const size_t need = bytes * (size_t)c->world;
  if (need > c->cap) {
    if (c->dbuf) cudaFree(c->dbuf);
    c->dbuf = nullptr;
    c->cap = 0;
    if (cudaMalloc(&c->dbuf, need) != cudaSuccess) return PM_CUDA;
    c->cap = need;
  }
  unsigned char* mine = c->dbuf + bytes * (size_t)c->rank;  // in-place allgather
  if (cudaMemcpyAsync(mine, send, bytes, cudaMemcpyHostToDevice, c->stream) != cudaSuccess) return PM_CUDA;
  if (nccl().all_gather(mine, c->dbuf, bytes, ncclUint8, c->comm, c->stream) != ncclSuccess) return PM_NCCL;
  if (cudaMemcpyAsync(recv, c->dbuf, need, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess) return PM_CUDA;
  return cudaStreamSynchronize(c->stream) == cudaSuccess ? PM_OK : PM_CUDA;
}

int pm_nccl_allgather_device(const void* send_device, size_t bytes, void* recv_device, void* stream, void* user) {
  pm_nccl* c = static_cast<pm_nccl*>(user);
  if (!c || (!send_device && bytes) || !recv_device) return PM_NCCL;
  if (nccl().all_gather(send_device, recv_device, bytes, ncclUint8, c->comm, static_cast<cudaStream_t>(stream)) !=
      ncclSuccess)
    return PM_NCCL;
  return PM_OK;
}

int pm_nccl_rank(const pm_nccl* c, int* rank, int* world) {
  if (!c) return PM_STRUCTURAL;
  if (rank) *rank = c->rank;
  if (world) *world = c->world;
  return PM_OK;
}

}  // extern "C"
