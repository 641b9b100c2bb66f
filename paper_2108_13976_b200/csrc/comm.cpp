// comm.cpp — the NCCL side of the multi-GPU path: envs shard
// across GPUs with no data-path exchange, and the only collective is the
// episode-statistics all-reduce (EpisodeTracker sums, trainer.cpp:221-258;
// sum of integer-valued doubles, so exact and order-independent).
//
// libnccl is resolved at run time (dlopen + dlsym), not linked: in a process
// that already loaded NCCL (PyTorch's bundled libnccl.so.2) the loaded copy is
// used, so a communicator created there (ProcessGroupNCCL._comm_ptr) can be
// wrapped; otherwise the system libnccl.so.2. nccl.h is used for its types only.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "facade.hpp"

namespace wdg {
namespace {

struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*comm_count)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*comm_user_rank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's copy, if loaded
    if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) return;
    auto sym = [&](auto& fn, const char* name) { fn = reinterpret_cast<std::decay_t<decltype(fn)>>(dlsym(h, name)); };
    sym(api.get_version, "ncclGetVersion");
    sym(api.get_unique_id, "ncclGetUniqueId");
    sym(api.comm_init_rank, "ncclCommInitRank");
    sym(api.comm_destroy, "ncclCommDestroy");
    sym(api.comm_count, "ncclCommCount");
    sym(api.comm_user_rank, "ncclCommUserRank");
    sym(api.all_reduce, "ncclAllReduce");
    sym(api.error_string, "ncclGetErrorString");
    if (api.get_version && api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.comm_count &&
        api.comm_user_rank && api.all_reduce && api.error_string) {
      api.handle = h;
    }
  });
  if (api.handle == nullptr) raise(Errc::state_error, "NCCL: libnccl.so.2 could not be loaded");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) raise(Errc::cuda, std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace

int32_t comm_nccl_version() {
  int v = 0;
  nccl_check(nccl().get_version(&v), "ncclGetVersion");
  return v;
}

void comm_unique_id(uint8_t* out, int64_t bytes) {
  if (out == nullptr || bytes < NCCL_UNIQUE_ID_BYTES) {
    raise(Errc::invalid_argument, "comm_unique_id: need a 128-byte buffer");
  }
  ncclUniqueId id;
  nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
}

Comm* comm_init(int32_t world, int32_t rank, const uint8_t* id, int64_t bytes) {
  if (world < 1 || rank < 0 || rank >= world) raise(Errc::invalid_argument, "comm_init: bad world/rank");
  if (id == nullptr || bytes < NCCL_UNIQUE_ID_BYTES) raise(Errc::invalid_argument, "comm_init: need the 128-byte id");
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t c = nullptr;
  nccl_check(nccl().comm_init_rank(&c, world, uid, rank), "ncclCommInitRank");
  return new Comm{c, true, world, rank};
}

Comm* comm_wrap(void* nccl_comm) {
  if (nccl_comm == nullptr) raise(Errc::invalid_argument, "comm_wrap: null communicator");
  auto c = static_cast<ncclComm_t>(nccl_comm);
  int world = 0, rank = 0;
  nccl_check(nccl().comm_count(c, &world), "ncclCommCount");
  nccl_check(nccl().comm_user_rank(c, &rank), "ncclCommUserRank");
  return new Comm{nccl_comm, false, world, rank};
}

void comm_destroy(Comm* c) {
  if (c == nullptr) return;
  if (c->owned && c->nccl != nullptr) nccl().comm_destroy(static_cast<ncclComm_t>(c->nccl));
  delete c;
}

void comm_allreduce_sum_f64(Comm* c, double* buf, int64_t count, cudaStream_t st) {
  if (c == nullptr || buf == nullptr || count < 0) raise(Errc::invalid_argument, "allreduce: bad arguments");
  nccl_check(nccl().all_reduce(buf, buf, static_cast<size_t>(count), ncclFloat64, ncclSum,
                               static_cast<ncclComm_t>(c->nccl), st),
             "ncclAllReduce");
}

// The stats all-reduce: this shard's tracker slots reduced on device into
// device_out (double[WDG_STAT_COUNT]), then summed over the communicator in
// place, all on the store's stream (no host round trip).
void stats_allreduce(Rollout& r, Comm* c, double* device_out) {
  r.reduce_stats_into(device_out);
  comm_allreduce_sum_f64(c, device_out, WDG_STAT_COUNT, r.stream());
}

}  // namespace wdg
