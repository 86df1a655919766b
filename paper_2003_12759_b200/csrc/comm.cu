// Native multi-GPU exchange (K6): an NCCL communicator owned by
// libmpg.so and an all-gather on the library's own stream, so the sharded
// IRKA (irka.cu irka_run, world > 1) exchanges its solved V/W columns device
// to device over NVLink with no staging through another framework.
//
// NCCL is bound at run time (dlopen of libnccl.so.2: the copy already mapped
// into the process, e.g. torch's, is reused; otherwise the system one), so
// libmpg.so carries no link-time NCCL dependency and a process that never
// creates a communicator never loads it. Only the unique id travels through
// the caller's rendezvous (torch.distributed broadcast in dist.py).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "irka.hpp"
#include "runtime.cuh"

namespace mpg {
namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      err = std::string("NCCL is not available: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p) err = std::string("NCCL symbol missing: ") + name;
      return p;
    };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    api.get_version = reinterpret_cast<decltype(api.get_version)>(sym("ncclGetVersion"));
  });
  if (!err.empty()) throw CudaError(err);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw CudaError(std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace
}  // namespace mpg

struct mpg_comm {
  int device = 0, rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  long long calls = 0;
  double bytes = 0.0;
};

namespace mpg {
int comm_unique_id(char* out, int len) {
  if (len < int(sizeof(ncclUniqueId))) throw std::invalid_argument("comm: id buffer smaller than NCCL_UNIQUE_ID_BYTES");
  ncclUniqueId id;
  nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof id);
  return int(sizeof id);
}

mpg_comm* comm_create(int device, int rank, int world, const char* id_bytes) {
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("comm: bad rank/world");
  DeviceGuard guard(device);
  (void)ctx(device);
  ncclUniqueId id;
  std::memcpy(&id, id_bytes, sizeof id);
  auto* c = new mpg_comm;
  c->device = device;
  c->rank = rank;
  c->world = world;
  const ncclResult_t r = nccl().comm_init_rank(&c->comm, world, id, rank);
  if (r != ncclSuccess) {
    delete c;
    nccl_check(r, "ncclCommInitRank");
  }
  return c;
}

void comm_destroy(mpg_comm* c) {
  if (!c) return;
  if (c->comm) {
    DeviceGuard guard(c->device);
    nccl().comm_destroy(c->comm);
  }
  delete c;
}

// mpg_allgather_fn over the communicator: rank k's `bytes` land at
// recv + k * bytes, enqueued on the library stream of the communicator's device
// (the stream irka_run's copies are ordered on), so no host synchronisation is
// needed around it.
int comm_allgather(mpg_comm* c, const void* send, void* recv, int64_t bytes) {
  if (!c || bytes < 0) return 1;
  try {
    DeviceGuard guard(c->device);
    nccl_check(nccl().all_gather(send, recv, size_t(bytes), ncclChar, c->comm, ctx(c->device).stream), "ncclAllGather");
    ++c->calls;
    c->bytes += double(bytes) * c->world;
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

void comm_stats(const mpg_comm* c, long long* calls, double* bytes) {
  if (calls) *calls = c ? c->calls : 0;
  if (bytes) *bytes = c ? c->bytes : 0.0;
}

int nccl_version() {
  int v = 0;
  nccl().get_version(&v);
  return v;
}
}  // namespace mpg
