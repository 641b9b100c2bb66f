// facade.hpp — the C++ host side of the B200 Tag hot path. Same names and
// semantics as the reference's C++ API (proj/include/warp/*.hpp), with device
// ownership: every array lives in HBM and is mutated in place by kernels.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "tag_params.hpp"
#include "wdg_b200.h"

namespace wdg {

// Errc (proj/include/warp/common.hpp:13-28) + a device failure code.
enum class Errc : int32_t {
  ok = WDG_OK,
  invalid_argument = WDG_ERR_INVALID_ARGUMENT,
  duplicate_name = WDG_ERR_DUPLICATE_NAME,
  shape_mismatch = WDG_ERR_SHAPE_MISMATCH,
  store_locked = WDG_ERR_STORE_LOCKED,
  missing_placeholder = WDG_ERR_MISSING_PLACEHOLDER,
  unknown_name = WDG_ERR_UNKNOWN_NAME,
  index_out_of_range = WDG_ERR_INDEX_OUT_OF_RANGE,
  invalid_config = WDG_ERR_INVALID_CONFIG,
  step_failure = WDG_ERR_STEP_FAILURE,
  non_finite = WDG_ERR_NON_FINITE,
  parse_error = WDG_ERR_PARSE,
  io_error = WDG_ERR_IO,
  state_error = WDG_ERR_STATE,
  cuda = WDG_ERR_CUDA,
};

class Error : public std::runtime_error {
 public:
  Error(Errc code, const std::string& what) : std::runtime_error(what), code_(code) {}
  Errc code() const noexcept { return code_; }

 private:
  Errc code_;
};

[[noreturn]] void raise(Errc code, const std::string& what);
void cuda_check(cudaError_t err, const char* what);

inline int64_t element_size(int32_t kind) { return kind == WDG_BOOL8 ? 1 : 4; }

// Canonical placeholders (data_store.hpp:26-29).
inline constexpr const char* kObservations = "observations";
inline constexpr const char* kSampledActions = "sampled_actions";
inline constexpr const char* kRewards = "rewards";
inline constexpr const char* kDone = "done";

struct ArraySpec {
  std::string name;
  std::vector<int64_t> shape;
  int32_t kind = WDG_REAL32;
  bool snapshot_on_reset = false;
};

struct ArrayInfo {
  ArraySpec spec;
  int64_t total_elems = 0;
  int64_t env_stride = 0;
  int64_t agent_stride = 0;
  bool has_agent_axis = false;
};

// DataStore (data_store.hpp:54-113), device-resident.
class DataStore {
 public:
  DataStore(int64_t num_envs, int64_t num_agents);
  ~DataStore();
  DataStore(const DataStore&) = delete;
  DataStore& operator=(const DataStore&) = delete;

  int64_t num_envs() const noexcept { return num_envs_; }
  int64_t num_agents() const noexcept { return num_agents_; }
  bool locked() const noexcept { return locked_; }
  int64_t env_offset() const noexcept { return env_offset_; }
  void set_env_offset(int64_t off);
  cudaStream_t stream() const noexcept { return stream_; }
  void set_stream(cudaStream_t s) { stream_ = s; }

  int32_t register_array(const ArraySpec& spec, const void* host_initial, int64_t count);
  void lock();
  bool has_array(const std::string& name) const { return index_.count(name) != 0; }
  int32_t handle(const std::string& name) const;
  const ArrayInfo& info(int32_t h) const;
  int32_t num_arrays() const { return static_cast<int32_t>(arrays_.size()); }
  int64_t row_bytes(int32_t h) const;

  void push(int32_t h, int64_t env_begin, int64_t env_count, const void* host, int64_t bytes);
  void pull(int32_t h, int64_t env_begin, int64_t env_count, void* host, int64_t bytes) const;
  void* device_ptr(int32_t h);
  const void* snapshot_ptr(int32_t h) const;
  // Re-capture the snapshot from the current content (registration helpers
  // that initialise on device; only before lock()).
  void refresh_snapshot(int32_t h);
  void restore_snapshot(const int64_t* env_ids, int64_t count);
  void synchronize() const;

  // Scratch owned by the store, reused by reset paths.
  uint8_t* env_mask();
  int64_t* id_buffer(int64_t count);
  // Per-env sequence flags for programmatic dependent launch of consecutive
  // fused steps (TagLaunch::env_seq), shared by every rollout on this store.
  // A launch uses pdl_seq() + 1 and calls commit_pdl_seq() once it is
  // enqueued, so a failed launch never leaves a sequence number nobody sets.
  uint32_t* pdl_flags();
  uint32_t pdl_seq() const noexcept { return pdl_seq_; }
  void commit_pdl_seq() noexcept { ++pdl_seq_; }
  // Resynchronise the flags after a skipped (timed-out) overlapped step.
  void reset_pdl();
  // True when the last kernel a rollout enqueued on this store's stream
  // released its dependents early (griddepcontrol.launch_dependents: bf16
  // policy forwards, plain-PDL Tag launches) WITHOUT publishing env_seq
  // flags. A flag-waiting launch after it must also griddepcontrol.wait:
  // its flag test is already satisfied by older launches, so it would
  // otherwise start while that kernel still writes the envs.
  bool pdl_open() const noexcept { return pdl_open_; }
  void set_pdl_open(bool open) noexcept { pdl_open_ = open; }

 private:
  struct Entry {
    ArrayInfo info;
    void* dev = nullptr;
    void* snap = nullptr;
    int64_t bytes = 0;
  };
  int32_t check_handle(int32_t h) const;
  void check_env_range(int64_t begin, int64_t count) const;

  int64_t num_envs_;
  int64_t num_agents_;
  int64_t env_offset_ = 0;
  bool locked_ = false;
  cudaStream_t stream_ = nullptr;
  std::vector<Entry> arrays_;
  std::unordered_map<std::string, int32_t> index_;
  uint8_t* mask_ = nullptr;
  int64_t* ids_ = nullptr;
  int64_t ids_cap_ = 0;
  void* descs_ = nullptr;
  int32_t descs_cap_ = 0;
  uint32_t* pdl_flags_ = nullptr;
  uint32_t pdl_seq_ = 0;
  bool pdl_open_ = false;
  friend class ResetManager;
};

void validate_tag_config(const wdg_tag_config& cfg);
int64_t tag_obs_dim(const wdg_tag_config& cfg);
std::vector<std::string> tag_zero_on_reset();

// Device config + geometry for a store/config pair (tag.cpp).
TagDevConfig make_dev_config(const DataStore& store, const wdg_tag_config& cfg);
TagDevArrays bind_dev_arrays(DataStore& store, const wdg_tag_config& cfg);

void register_tag_arrays(DataStore& store, const wdg_tag_config& cfg);

// TagPlan (tag_env.hpp:104-116) + StepEngine::run_step for it.
class TagPlan {
 public:
  // reference = true: the device TagReference (twin_kernels.cu,
  // tag_env.cpp:505-595) — run_step and reinit_masked run the independent
  // brute-force twin instead of the production kernel (the consistency
  // check's second store, harness.cpp:562-633).
  TagPlan(DataStore& store, const wdg_tag_config& cfg, bool reference = false);
  ~TagPlan();
  TagPlan(const TagPlan&) = delete;
  TagPlan& operator=(const TagPlan&) = delete;
  bool reference() const { return reference_; }
  void run_step(int64_t step_index);
  void reinit_masked(const uint8_t* env_mask, int32_t* episode);
  void launch(TagLaunch L);
  // The same launch restricted to envs [e0, e0 + n) (pipelined host steps).
  void launch_envs(TagLaunch L, int64_t e0, int64_t n);
  // Whether RolloutDriver::run may use multi-step residency launches.
  bool multistep_ok();
  // How consecutive fused launches overlap (programmatic dependent launch):
  // 0 = not at all, 1 = the next launch is released at CTA entry, 2 = at exit
  // (both with per-env waits), 3 = plain PDL (released at entry, whole-grid wait).
  int pdl_mode() const;
  const wdg_tag_config& config() const { return cfg_; }
  const TagDevConfig& dev() const { return dev_; }
  DataStore& store() { return store_; }

 private:
  DataStore& store_;
  wdg_tag_config cfg_;
  TagDevConfig dev_;
  TagDevArrays arrays_;
  int multistep_ = -1;
  bool reference_ = false;
  float* knn_d2_ = nullptr;     // twin K-NN scratch [E*A*K]
  int32_t* knn_idx_ = nullptr;
};

// sample_actions (sampler.hpp:35-36) with device logits.
void sample_actions(DataStore& store, const double* logits, int64_t logits_count,
                    int64_t num_categories, int64_t num_choices, int64_t step, uint64_t seed);

// ResetManager (reset_manager.hpp:23-43) with a device episode counter.
class ResetManager {
 public:
  ResetManager(DataStore& store, bool auto_reset, std::vector<std::string> zero_on_reset,
               TagPlan* reinit);
  ~ResetManager();
  std::vector<int64_t> detect_done() const;
  void auto_reset(const int64_t* env_ids, int64_t count);
  void auto_reset_on_done();
  int64_t episodes_started(int64_t env_id) const;
  bool auto_enabled() const { return auto_; }
  // True when the policy is exactly the Tag default (tag_zero_on_reset +
  // make_tag_reinit), which the fused kernel implements in place.
  bool tag_default() const { return tag_default_; }
  int32_t* episode_device() { return episode_; }
  TagPlan* reinit_plan() { return reinit_; }

 private:
  void reset_masked();
  DataStore& store_;
  bool auto_;
  std::vector<int32_t> zero_handles_;
  TagPlan* reinit_;
  bool tag_default_ = false;
  int32_t* episode_ = nullptr;
  void* descs_ = nullptr;
  int32_t ndesc_ = 0;
};

class Policy;
class RolloutBatch;

// RolloutDriver (harness.cpp:428-505).
class Rollout {
 public:
  Rollout(DataStore& store, TagPlan& plan, ResetManager* resets, uint64_t sample_seed);
  ~Rollout();
  void set_logits(const double* logits, int64_t count);
  // forward_policies (harness.cpp:445-476) on device: taggers [0, T) use
  // `tagger`, runners [T, A) use `runner` (tag_policy_map, harness.cpp:395-399);
  // pass the same policy twice for one shared policy (check_consistency_single,
  // harness.cpp:586-606). nullptr, nullptr restores the uniform policy.
  void set_policies(const Policy* tagger, const Policy* runner, int32_t precision);
  // Keep the policy's f64 logits (bf16 path) and values in device buffers
  // readable through policy_logits()/policy_values() (default off).
  void set_keep_policy_outputs(bool keep) {
    keep_outputs_ = keep;
    ++pol_version_;
  }
  const double* policy_logits() const { return pol_logits_; }
  const double* policy_values() const { return pol_values_; }
  void set_fused(bool f) { fused_ = f; }
  void set_graphs(bool g) { graphs_ = g; }
  // Overlap consecutive launches (programmatic dependent launch, default on);
  // off = one plain launch after another (A/B timing, serial references).
  void set_overlap(bool enabled);
  void step();
  // Trainer::collect (trainer.cpp:315-403): T captured policy steps.
  void collect(RolloutBatch& batch);
  void step_host(const double* host_logits, int64_t count, float* host_rewards, uint8_t* host_done,
                 float* host_obs = nullptr, int64_t obs_count = 0);
  // Env chunks of the pipelined host step (0 = automatic, ~8 MB of logits each).
  void set_host_chunks(int32_t n) { host_chunks_ = std::min<int32_t>(std::max<int32_t>(n, 0), kMaxHostChunks); }
  void run(int64_t steps);
  void reduce_stats_into(double* device_out);
  int64_t next_step() const { return t_; }
  cudaStream_t stream() const { return store_.stream(); }
  // Kernel launches this driver has issued (env step kernels, policy
  // forwards, graph replays counted per node).
  int64_t launches() const { return launches_; }
  void check();
  void stats(double* out, int32_t count);
  void reset_stats();
  double* stats_device();

 private:
  TagLaunch fused_launch(int64_t step) const;
  void step_unfused(float* cap_rewards = nullptr, uint8_t* cap_done = nullptr);
  void forward_policies(cudaStream_t st, int64_t step, const int64_t* step_dev, int32_t step_add,
                        double* values_out, bool force_logits, bool sample);
  bool policy_samples() const { return pol_[0] != nullptr && pol_prec_ == 1; }  // kPolicyBF16
  const Policy* pol_[2] = {nullptr, nullptr};
  int32_t pol_prec_ = 0;
  double* pol_logits_ = nullptr;
  double* pol_values_ = nullptr;
  uint64_t pol_version_ = 0, graph_pol_version_ = 0;
  bool keep_outputs_ = false;
  bool fused_ok() const;
  DataStore& store_;
  TagPlan& plan_;
  ResetManager* resets_;
  uint64_t seed_;
  int64_t t_ = 0;
  int64_t launches_ = 0;
  bool fused_ = true;
  bool graphs_ = true;
  const double* logits_ = nullptr;
  double* zero_logits_ = nullptr;
  double* env_stats_ = nullptr;
  double* stats_ = nullptr;
  uint32_t* error_ = nullptr;
  int32_t* own_episode_ = nullptr;
  uint64_t h_actions0_ = 0;
  uint32_t* pdl_flags_ = nullptr;  // the store's (DataStore::pdl_flags)
  bool graph_pdl_ = false;         // the captured graph's nodes overlap (PDL)
  bool graph_plain_pdl_ = false;   // ... through plain PDL (no per-env flags)
  void set_pdl(TagLaunch& L, bool single_step) const;
  void note_launch(const TagLaunch& L);
  // host-driven stepping: double-buffered logits, H2D and D2H copy streams,
  // pre-reset rewards / done capture buffers, per-chunk events
  static constexpr int kMaxHostChunks = 16;
  int32_t host_chunks_ = 0;
  cudaStream_t copy_ = nullptr;
  cudaStream_t d2h_ = nullptr;
  double* dlog_[2] = {nullptr, nullptr};
  cudaEvent_t slot_free_[2] = {nullptr, nullptr};
  cudaEvent_t h2d_ev_[kMaxHostChunks] = {};
  cudaEvent_t kern_ev_[kMaxHostChunks] = {};
  cudaEvent_t d2h_ev_ = nullptr;
  float* rew_cap_ = nullptr;
  uint8_t* done_cap_ = nullptr;
  // CUDA-graph replay of kGraphSteps fused launches (run()).
  void build_graph();
  void drop_graph();
  static constexpr int kGraphSteps = 16;
  static constexpr int kMultiSteps = 64;  // steps per multi-step residency launch
  cudaGraphExec_t graph_exec_ = nullptr;
  int64_t* step_dev_ = nullptr;
  const double* graph_logits_ = nullptr;
  float graph_bias_ = 0.0f;
  cudaStream_t graph_stream_ = nullptr;  // mix64(substream(seed, kStreamActions))
};

// Session layer (session.cpp): the reference's wd_session_* run modes on the
// device path (c_api.cpp:97-255, harness.cpp:32-335,563-898).
struct Session;
Session* session_open(const std::string& config_json);
const char* session_config_json(Session* s);
const char* session_config_hash(Session* s);
void session_set_seed(Session* s, uint64_t seed);
void session_set_workers(Session* s, int32_t workers);
void session_set_output_dir(Session* s, const std::string& dir);
bool session_run_check(Session* s);
void session_run_bench_envs(Session* s);
void session_run_bench_agents(Session* s);
const char* session_report_json(Session* s);
const char* session_summary(Session* s);
void session_dump_array(Session* s, const std::string& name, const std::string& path);
void session_close(Session* s);

// Host-side RNG prefix helpers (rng.hpp:23-53).
uint64_t host_mix64(uint64_t x);
uint64_t host_absorb(uint64_t h, uint64_t v);
uint64_t host_substream(uint64_t seed, uint64_t purpose);
inline constexpr uint64_t kStreamActions = 0x616374696f6e7331ULL;
inline constexpr uint64_t kStreamPlacement = 0x706c6163656d656eULL;

float& fault_tag_radius_bias();
// NCCL communicator for the episode-statistics all-reduce (comm.cpp).
struct Comm {
  void* nccl;   // ncclComm_t
  bool owned;   // created here (destroyed here) or wrapped
  int32_t world, rank;
};
int32_t comm_nccl_version();
void comm_unique_id(uint8_t* out, int64_t bytes);
Comm* comm_init(int32_t world, int32_t rank, const uint8_t* id, int64_t bytes);
Comm* comm_wrap(void* nccl_comm);
void comm_destroy(Comm* c);
void comm_allreduce_sum_f64(Comm* c, double* buf, int64_t count, cudaStream_t st);
void stats_allreduce(Rollout& r, Comm* c, double* device_out);

// Plan tuning overrides (tag.cpp kTuningKeys); "reset" restores the defaults.
void set_tuning(const std::string& key, int64_t value);

}  // namespace wdg
