// store.cpp — device-resident DataStore (proj/include/warp/data_store.hpp,
// proj/src/data_store.cpp). Registration, lock and validation rules are the
// reference's (same error codes and messages); storage is one cudaMalloc per
// array in the reference's dense row-major layout (env outermost)
// plus a device snapshot copy for snapshot_on_reset arrays.
#include <cstring>

#include "facade.hpp"
#include "kernels.hpp"

namespace wdg {

[[noreturn]] void raise(Errc code, const std::string& what) { throw Error(code, what); }

void cuda_check(cudaError_t err, const char* what) {
  if (err != cudaSuccess) {
    raise(Errc::cuda, std::string(what) + ": " + cudaGetErrorName(err) + " (" +
                          cudaGetErrorString(err) + ")");
  }
}

DataStore::DataStore(int64_t num_envs, int64_t num_agents)
    : num_envs_(num_envs), num_agents_(num_agents) {
  // data_store.cpp:7-12
  if (num_envs < 1 || num_agents < 1) {
    raise(Errc::invalid_argument, "DataStore requires num_envs >= 1 and num_agents >= 1");
  }
  int dev_count = 0;
  if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count < 1) {
    cudaGetLastError();
    raise(Errc::cuda, "DataStore: no CUDA device visible (the B200 path has no CPU fallback)");
  }
}

DataStore::~DataStore() {
  for (Entry& e : arrays_) {
    if (e.dev) cudaFree(e.dev);
    if (e.snap) cudaFree(e.snap);
  }
  if (mask_) cudaFree(mask_);
  if (ids_) cudaFree(ids_);
  if (descs_) cudaFree(descs_);
  if (pdl_flags_) cudaFree(pdl_flags_);
}

uint32_t* DataStore::pdl_flags() {
  if (pdl_flags_ == nullptr) {
    const size_t bytes = static_cast<size_t>(num_envs_) * sizeof(uint32_t);
    cuda_check(cudaMalloc(&pdl_flags_, bytes), "cudaMalloc(pdl flags)");
    cuda_check(cudaMemset(pdl_flags_, 0, bytes), "memset(pdl flags)");  // before any stream uses them
    pdl_seq_ = 0;
  }
  return pdl_flags_;
}

void DataStore::reset_pdl() {
  // Only after a synchronize (no launch in flight): every flag back to 0 and
  // the next launch waits for sequence 0, which every env now shows.
  if (pdl_flags_ != nullptr) {
    cuda_check(cudaMemset(pdl_flags_, 0, static_cast<size_t>(num_envs_) * sizeof(uint32_t)),
               "memset(pdl flags)");
  }
  pdl_seq_ = 0;
  pdl_open_ = false;
}

void DataStore::set_env_offset(int64_t off) {
  if (off < 0) raise(Errc::invalid_argument, "set_env_offset: offset must be >= 0");
  env_offset_ = off;
}

int32_t DataStore::register_array(const ArraySpec& spec, const void* initial, int64_t count) {
  // data_store.cpp:14-55
  if (locked_) raise(Errc::store_locked, "register_array(\"" + spec.name + "\"): store is locked");
  if (spec.name.empty()) raise(Errc::invalid_argument, "register_array: empty name");
  if (spec.name.size() >= WDG_MAX_NAME) raise(Errc::invalid_argument, "register_array: name too long");
  if (spec.kind != WDG_REAL32 && spec.kind != WDG_INT32 && spec.kind != WDG_BOOL8) {
    raise(Errc::invalid_argument, "register_array(\"" + spec.name + "\"): unknown element kind");
  }
  if (index_.count(spec.name)) {
    raise(Errc::duplicate_name, "register_array: duplicate name \"" + spec.name + "\"");
  }
  if (spec.shape.empty() || spec.shape[0] != num_envs_) {
    raise(Errc::shape_mismatch, "register_array(\"" + spec.name + "\"): shape[0] must equal num_envs");
  }
  if (spec.shape.size() > WDG_MAX_DIMS) raise(Errc::shape_mismatch, "register_array: too many dims");
  int64_t total = 1;
  for (int64_t d : spec.shape) {
    if (d < 1) raise(Errc::shape_mismatch, "register_array(\"" + spec.name + "\"): non-positive dim");
    total *= d;
  }
  if (initial != nullptr && count != total) {
    raise(Errc::shape_mismatch, "register_array(\"" + spec.name + "\"): initial has " +
                                    std::to_string(count) + " elements, shape needs " +
                                    std::to_string(total));
  }
  Entry e;
  e.info.spec = spec;
  e.info.total_elems = total;
  e.info.env_stride = total / num_envs_;
  e.info.has_agent_axis = spec.shape.size() >= 2 && spec.shape[1] == num_agents_;
  e.info.agent_stride = e.info.has_agent_axis ? e.info.env_stride / num_agents_ : 0;
  e.bytes = total * element_size(spec.kind);
  cuda_check(cudaMalloc(&e.dev, static_cast<size_t>(e.bytes)), "cudaMalloc(array)");
  if (initial != nullptr) {
    cuda_check(cudaMemcpyAsync(e.dev, initial, static_cast<size_t>(e.bytes), cudaMemcpyHostToDevice,
                               stream_),
               "register_array upload");
  } else {
    cuda_check(cudaMemsetAsync(e.dev, 0, static_cast<size_t>(e.bytes), stream_), "register_array zero");
  }
  if (spec.snapshot_on_reset) {
    cuda_check(cudaMalloc(&e.snap, static_cast<size_t>(e.bytes)), "cudaMalloc(snapshot)");
    cuda_check(cudaMemcpyAsync(e.snap, e.dev, static_cast<size_t>(e.bytes), cudaMemcpyDeviceToDevice,
                               stream_),
               "register_array snapshot");
  }
  cuda_check(cudaStreamSynchronize(stream_), "register_array sync");
  const int32_t h = static_cast<int32_t>(arrays_.size());
  arrays_.push_back(e);
  index_.emplace(spec.name, h);
  return h;
}

void DataStore::lock() {
  // data_store.cpp:85-93
  for (const char* name : {kObservations, kSampledActions, kRewards, kDone}) {
    if (!index_.count(name)) {
      raise(Errc::missing_placeholder,
            std::string("lock(): placeholder \"") + name + "\" is not registered");
    }
  }
  locked_ = true;
}

int32_t DataStore::handle(const std::string& name) const {
  auto it = index_.find(name);
  if (it == index_.end()) raise(Errc::unknown_name, "unknown array \"" + name + "\"");
  return it->second;
}

int32_t DataStore::check_handle(int32_t h) const {
  if (h < 0 || static_cast<size_t>(h) >= arrays_.size()) {
    raise(Errc::unknown_name, "invalid array handle " + std::to_string(h));
  }
  return h;
}

const ArrayInfo& DataStore::info(int32_t h) const { return arrays_[check_handle(h)].info; }

int64_t DataStore::row_bytes(int32_t h) const {
  const Entry& e = arrays_[check_handle(h)];
  return e.info.env_stride * element_size(e.info.spec.kind);
}

void DataStore::check_env_range(int64_t begin, int64_t count) const {
  if (begin < 0 || count < 0 || begin + count > num_envs_) {
    raise(Errc::index_out_of_range, "env range [" + std::to_string(begin) + ", " +
                                        std::to_string(begin + count) + ") out of range [0, " +
                                        std::to_string(num_envs_) + ")");
  }
}

void DataStore::push(int32_t h, int64_t env_begin, int64_t env_count, const void* host,
                     int64_t bytes) {
  check_env_range(env_begin, env_count);
  const int64_t rb = row_bytes(h);
  if (bytes != rb * env_count) raise(Errc::shape_mismatch, "push: byte count does not match env rows");
  if (host == nullptr && bytes > 0) raise(Errc::invalid_argument, "push: null host buffer");
  if (bytes == 0) return;
  Entry& e = arrays_[h];
  cuda_check(cudaMemcpyAsync(static_cast<uint8_t*>(e.dev) + env_begin * rb, host,
                             static_cast<size_t>(bytes), cudaMemcpyHostToDevice, stream_),
             "push");
  cuda_check(cudaStreamSynchronize(stream_), "push sync");
}

void DataStore::pull(int32_t h, int64_t env_begin, int64_t env_count, void* host,
                     int64_t bytes) const {
  check_env_range(env_begin, env_count);
  const int64_t rb = row_bytes(h);
  if (bytes != rb * env_count) raise(Errc::shape_mismatch, "pull: byte count does not match env rows");
  if (host == nullptr && bytes > 0) raise(Errc::invalid_argument, "pull: null host buffer");
  if (bytes == 0) return;
  const Entry& e = arrays_[h];
  cuda_check(cudaMemcpyAsync(host, static_cast<const uint8_t*>(e.dev) + env_begin * rb,
                             static_cast<size_t>(bytes), cudaMemcpyDeviceToHost, stream_),
             "pull");
  cuda_check(cudaStreamSynchronize(stream_), "pull sync");
}

void* DataStore::device_ptr(int32_t h) { return arrays_[check_handle(h)].dev; }

const void* DataStore::snapshot_ptr(int32_t h) const { return arrays_[check_handle(h)].snap; }

void DataStore::refresh_snapshot(int32_t h) {
  if (locked_) raise(Errc::store_locked, "refresh_snapshot: store is locked");
  Entry& e = arrays_[check_handle(h)];
  if (!e.snap) return;
  cuda_check(cudaMemcpyAsync(e.snap, e.dev, static_cast<size_t>(e.bytes), cudaMemcpyDeviceToDevice,
                             stream_),
             "refresh_snapshot");
}

uint8_t* DataStore::env_mask() {
  if (!mask_) cuda_check(cudaMalloc(&mask_, static_cast<size_t>(num_envs_)), "cudaMalloc(mask)");
  return mask_;
}

int64_t* DataStore::id_buffer(int64_t count) {
  if (count > ids_cap_) {
    if (ids_) cudaFree(ids_);
    ids_ = nullptr;
    cuda_check(cudaMalloc(&ids_, static_cast<size_t>(count) * sizeof(int64_t)), "cudaMalloc(ids)");
    ids_cap_ = count;
  }
  return ids_;
}

void DataStore::restore_snapshot(const int64_t* env_ids, int64_t count) {
  // data_store.cpp:207-217: validate every id first, then restore rows.
  for (int64_t i = 0; i < count; ++i) {
    if (env_ids[i] < 0 || env_ids[i] >= num_envs_) {
      raise(Errc::index_out_of_range, "env_id " + std::to_string(env_ids[i]) +
                                          " out of range [0, " + std::to_string(num_envs_) + ")");
    }
  }
  if (count == 0) return;
  std::vector<ResetRowDesc> descs;
  for (Entry& e : arrays_) {
    if (!e.snap) continue;
    descs.push_back({static_cast<uint8_t*>(e.dev), static_cast<const uint8_t*>(e.snap),
                     e.info.env_stride * element_size(e.info.spec.kind)});
  }
  if (descs.empty()) return;
  if (static_cast<int32_t>(descs.size()) > descs_cap_) {
    if (descs_) cudaFree(descs_);
    cuda_check(cudaMalloc(&descs_, descs.size() * sizeof(ResetRowDesc)), "cudaMalloc(descs)");
    descs_cap_ = static_cast<int32_t>(descs.size());
  }
  uint8_t* mask = env_mask();
  int64_t* ids = id_buffer(count);
  cuda_check(cudaMemcpyAsync(descs_, descs.data(), descs.size() * sizeof(ResetRowDesc),
                             cudaMemcpyHostToDevice, stream_),
             "restore_snapshot descs");
  cuda_check(cudaMemcpyAsync(ids, env_ids, static_cast<size_t>(count) * sizeof(int64_t),
                             cudaMemcpyHostToDevice, stream_),
             "restore_snapshot ids");
  cuda_check(cudaMemsetAsync(mask, 0, static_cast<size_t>(num_envs_), stream_), "mask clear");
  cuda_check(launch_mask_from_ids(ids, count, mask, stream_), "mask_from_ids");
  cuda_check(launch_restore_zero(static_cast<const ResetRowDesc*>(descs_),
                                 static_cast<int>(descs.size()), mask, nullptr, nullptr, num_envs_,
                                 stream_),
             "restore_snapshot kernel");
  cuda_check(cudaStreamSynchronize(stream_), "restore_snapshot sync");
}

void DataStore::synchronize() const { cuda_check(cudaStreamSynchronize(stream_), "synchronize"); }

}  // namespace wdg
