// warp_b200.hpp — header-only C++ facade over the C ABI (wdg_b200.h) with the
// reference's C++ API shape (proj/include/warp/*.hpp), for reference-side code
// that wants to switch its Tag hot path to the B200 library by changing the
// namespace: warp::DataStore -> warp_b200::DataStore, etc. Errors are thrown
// as warp_b200::Error carrying the reference's Errc numbering
// (proj/include/warp/common.hpp:13-28).
//
// Differences from the CPU store, all forced by device residency:
//   * typed host views (f32/i32/u8, env_slice_*) become pull()/push() copies;
//   * sample_actions() takes DEVICE logits (or use RolloutDriver::step_host);
//   * ResetManager::auto_reset_on_done() resets on device without a host list.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "wdg_b200.h"

namespace warp_b200 {

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
  unknown = WDG_ERR_UNKNOWN,
  cuda = WDG_ERR_CUDA,
};

class Error : public std::runtime_error {
 public:
  Error(Errc code, const std::string& what) : std::runtime_error(what), code_(code) {}
  Errc code() const noexcept { return code_; }

 private:
  Errc code_;
};

inline void check(wdg_status s) {
  if (s != WDG_OK) throw Error(static_cast<Errc>(s), wdg_last_error());
}

enum class ElementKind : int32_t { Real32 = WDG_REAL32, Int32 = WDG_INT32, Bool8 = WDG_BOOL8 };
enum class TagVariant : int32_t { Discrete = WDG_TAG_DISCRETE, Continuous = WDG_TAG_CONTINUOUS };
enum class ObsMode : int32_t { Full = WDG_OBS_FULL, Partial = WDG_OBS_PARTIAL };

inline constexpr const char* kLocX = "loc_x";
inline constexpr const char* kLocY = "loc_y";
inline constexpr const char* kObservations = "observations";
inline constexpr const char* kSampledActions = "sampled_actions";
inline constexpr const char* kRewards = "rewards";
inline constexpr const char* kDone = "done";

// TagConfig (tag_env.hpp:29-66): same fields and defaults.
struct TagConfig : wdg_tag_config {
  TagConfig() { check(wdg_tag_config_init(this)); }
  int64_t num_agents() const { return num_taggers + num_runners; }
  int64_t action_categories() const { return variant == WDG_TAG_CONTINUOUS ? 2 : 1; }
  int64_t action_choices() const { return variant == WDG_TAG_CONTINUOUS ? 3 : 5; }
  int64_t obs_dim() const { return wdg_tag_obs_dim(this); }
  void validate() const { check(wdg_tag_config_validate(this)); }
};

struct ArraySpec {
  std::string name;
  std::vector<int64_t> shape;
  ElementKind kind = ElementKind::Real32;
  bool snapshot_on_reset = false;
};

using ArrayHandle = int32_t;

class DataStore {
 public:
  DataStore(int64_t num_envs, int64_t num_agents) { check(wdg_store_create(num_envs, num_agents, &h_)); }
  ~DataStore() { wdg_store_destroy(h_); }
  DataStore(const DataStore&) = delete;
  DataStore& operator=(const DataStore&) = delete;

  wdg_store* raw() const { return h_; }
  int64_t num_envs() const { int64_t v; check(wdg_store_num_envs(h_, &v)); return v; }
  int64_t num_agents() const { int64_t v; check(wdg_store_num_agents(h_, &v)); return v; }
  bool locked() const { int32_t v; check(wdg_store_locked(h_, &v)); return v != 0; }
  void set_stream(void* cuda_stream) { check(wdg_store_set_stream(h_, cuda_stream)); }
  void set_env_offset(int64_t off) { check(wdg_store_set_env_offset(h_, off)); }

  template <class T>
  ArrayHandle register_array(const ArraySpec& spec, const std::vector<T>& initial) {
    ArrayHandle h;
    check(wdg_store_register_array(h_, spec.name.c_str(), spec.shape.data(),
                                   static_cast<int32_t>(spec.shape.size()),
                                   static_cast<int32_t>(spec.kind), spec.snapshot_on_reset,
                                   initial.data(), static_cast<int64_t>(initial.size()), &h));
    return h;
  }
  ArrayHandle register_array(const ArraySpec& spec) {
    ArrayHandle h;
    check(wdg_store_register_array(h_, spec.name.c_str(), spec.shape.data(),
                                   static_cast<int32_t>(spec.shape.size()),
                                   static_cast<int32_t>(spec.kind), spec.snapshot_on_reset, nullptr,
                                   0, &h));
    return h;
  }
  void lock() { check(wdg_store_lock(h_)); }
  ArrayHandle handle(const std::string& name) const {
    ArrayHandle h;
    check(wdg_store_handle(h_, name.c_str(), &h));
    return h;
  }
  wdg_array_info info(ArrayHandle h) const {
    wdg_array_info i;
    check(wdg_store_info(h_, h, &i));
    return i;
  }
  std::vector<std::string> array_names() const {
    int32_t n;
    check(wdg_store_num_arrays(h_, &n));
    std::vector<std::string> out;
    for (int32_t i = 0; i < n; ++i) out.emplace_back(info(i).name);
    return out;
  }
  // Host copies of env rows (replace the aliasing host views).
  template <class T>
  std::vector<T> pull(const std::string& name, int64_t env_begin = 0, int64_t env_count = -1) const {
    const ArrayHandle h = handle(name);
    const wdg_array_info in = info(h);
    if (env_count < 0) env_count = num_envs() - env_begin;
    std::vector<T> out(static_cast<size_t>(in.env_stride * env_count));
    check(wdg_store_pull(h_, h, env_begin, env_count, out.data(),
                         static_cast<int64_t>(out.size() * sizeof(T))));
    return out;
  }
  template <class T>
  void push(const std::string& name, const std::vector<T>& values, int64_t env_begin = 0) {
    const ArrayHandle h = handle(name);
    const wdg_array_info in = info(h);
    check(wdg_store_push(h_, h, env_begin, static_cast<int64_t>(values.size()) / in.env_stride,
                         values.data(), static_cast<int64_t>(values.size() * sizeof(T))));
  }
  void* device_ptr(const std::string& name) {
    void* p;
    check(wdg_store_device_ptr(h_, handle(name), &p));
    return p;
  }
  void restore_snapshot(const std::vector<int64_t>& ids) {
    check(wdg_store_restore_snapshot(h_, ids.data(), static_cast<int64_t>(ids.size())));
  }
  void synchronize() { check(wdg_store_synchronize(h_)); }

 private:
  wdg_store* h_ = nullptr;
};

inline void register_tag_arrays(DataStore& store, const TagConfig& cfg) {
  check(wdg_register_tag_arrays(store.raw(), &cfg));
}

inline std::vector<std::string> tag_zero_on_reset() {
  const char* names[16];
  int32_t n;
  check(wdg_tag_zero_on_reset(names, 16, &n));
  return std::vector<std::string>(names, names + n);
}

class TagPlan {
 public:
  TagPlan(DataStore& store, const TagConfig& cfg) { check(wdg_build_tag_plan(store.raw(), &cfg, &h_)); }
  // TagReference(store, cfg) (tag_env.cpp:505-595): the device twin, the
  // consistency check's independent second implementation.
  struct Reference {};
  TagPlan(DataStore& store, const TagConfig& cfg, Reference) {
    check(wdg_build_tag_reference(store.raw(), &cfg, &h_));
  }
  ~TagPlan() { wdg_tag_plan_destroy(h_); }
  TagPlan(const TagPlan&) = delete;
  TagPlan& operator=(const TagPlan&) = delete;
  wdg_tag_plan* raw() const { return h_; }

 private:
  wdg_tag_plan* h_ = nullptr;
};

// StepEngine::run_step for the Tag plan (step_engine.hpp:100).
struct StepEngine {
  void run_step(TagPlan& plan, DataStore&, int64_t step_index) {
    check(wdg_run_step(plan.raw(), step_index));
  }
};

// sample_actions (sampler.hpp:35-36) with device logits.
inline void sample_actions(DataStore& store, const double* device_logits, int64_t logits_count,
                           int64_t num_categories, int64_t num_choices, int64_t step,
                           uint64_t seed) {
  check(wdg_sample_actions(store.raw(), device_logits, logits_count, num_categories, num_choices,
                           step, seed));
}

class ResetManager {
 public:
  // ResetPolicy{auto_reset, zero_on_reset, make_tag_reinit(plan)}
  ResetManager(DataStore& store, bool auto_reset, const std::vector<std::string>& zero_on_reset,
               TagPlan* reinit) {
    std::vector<const char*> names;
    for (const auto& n : zero_on_reset) names.push_back(n.c_str());
    check(wdg_reset_manager_create(store.raw(), auto_reset, names.data(),
                                   static_cast<int32_t>(names.size()),
                                   reinit ? reinit->raw() : nullptr, &h_));
  }
  ~ResetManager() { wdg_reset_manager_destroy(h_); }
  ResetManager(const ResetManager&) = delete;
  ResetManager& operator=(const ResetManager&) = delete;
  wdg_resets* raw() const { return h_; }
  std::vector<int64_t> detect_done(int64_t num_envs) {
    std::vector<int64_t> ids(static_cast<size_t>(num_envs));
    int64_t n;
    check(wdg_detect_done(h_, ids.data(), num_envs, &n));
    ids.resize(static_cast<size_t>(n));
    return ids;
  }
  void auto_reset(const std::vector<int64_t>& ids) {
    check(wdg_auto_reset(h_, ids.data(), static_cast<int64_t>(ids.size())));
  }
  void auto_reset_on_done() { check(wdg_auto_reset_on_done(h_)); }
  int64_t episodes_started(int64_t env) const {
    int64_t v;
    check(wdg_episodes_started(h_, env, &v));
    return v;
  }

 private:
  wdg_resets* h_ = nullptr;
};

// PolicyParams + init_policy / forward (proj/include/warp/policy_model.hpp)
// with device-resident parameters.
enum class PolicyPrecision : int32_t { F64 = WDG_POLICY_F64, BF16 = WDG_POLICY_BF16 };
struct PolicyDims {  // policy_model.hpp:20-28
  int64_t obs_dim = 0;
  std::vector<int64_t> hidden = {64, 64};
  int64_t num_categories = 1;
  int64_t num_choices = 1;
};
class Policy {
 public:
  explicit Policy(const PolicyDims& d) {
    check(wdg_policy_create(d.obs_dim, d.hidden.data(), static_cast<int32_t>(d.hidden.size()),
                            d.num_categories, d.num_choices, &h_));
  }
  Policy(const PolicyDims& d, uint64_t seed) : Policy(d) { init(seed); }
  ~Policy() { wdg_policy_destroy(h_); }
  Policy(const Policy&) = delete;
  Policy& operator=(const Policy&) = delete;
  void init(uint64_t seed) { check(wdg_policy_init(h_, seed)); }  // init_policy
  int64_t param_count() const {
    int64_t n = 0;
    check(wdg_policy_param_count(h_, &n));
    return n;
  }
  // for_each_param canonical order (policy_model.hpp:43-46)
  std::vector<double> params() const {
    std::vector<double> v(static_cast<size_t>(param_count()));
    check(wdg_policy_get_params(h_, v.data(), static_cast<int64_t>(v.size())));
    return v;
  }
  void set_params(const std::vector<double>& v) {
    check(wdg_policy_set_params(h_, v.data(), static_cast<int64_t>(v.size())));
  }
  // forward over agents [a0, a1) of device obs [E, A, obs_dim] -> device logits / values
  void forward(const float* obs, int64_t E, int64_t A, int64_t a0, int64_t a1, double* logits,
               double* values, PolicyPrecision prec = PolicyPrecision::F64, void* stream = nullptr) const {
    check(wdg_policy_forward(h_, obs, E, A, a0, a1, logits, values, static_cast<int32_t>(prec), stream));
  }
  const wdg_policy* raw() const { return h_; }

 private:
  wdg_policy* h_ = nullptr;
};

// RolloutDriver (harness.cpp:428-505): fused sample -> step -> reset launch.
class RolloutDriver {
 public:
  RolloutDriver(DataStore& store, TagPlan& plan, ResetManager* resets, uint64_t sample_seed) {
    check(wdg_rollout_create(store.raw(), plan.raw(), resets ? resets->raw() : nullptr, sample_seed,
                             &h_));
  }
  ~RolloutDriver() { wdg_rollout_destroy(h_); }
  RolloutDriver(const RolloutDriver&) = delete;
  RolloutDriver& operator=(const RolloutDriver&) = delete;
  wdg_rollout* raw() const { return h_; }
  void set_logits(const double* device_logits, int64_t count) {
    check(wdg_rollout_set_logits(h_, device_logits, count));
  }
  // RolloutDriver(ws, &map, &policies, seed) (harness.cpp:428-476): the
  // tagger / runner policies run on device before every step.
  void set_policies(const Policy* tagger, const Policy* runner,
                    PolicyPrecision prec = PolicyPrecision::F64) {
    check(wdg_rollout_set_policies(h_, tagger ? tagger->raw() : nullptr, runner ? runner->raw() : nullptr,
                                   static_cast<int32_t>(prec)));
  }
  void step() { check(wdg_rollout_step(h_)); }
  // Host-buffer step: rewards / done before reset-on-done, observations
  // after it (pass host_obs = nullptr to skip them).
  void step_host(const double* host_logits, int64_t count, float* host_rewards, uint8_t* host_done,
                 float* host_obs = nullptr, int64_t obs_count = 0) {
    check(wdg_rollout_step_host_obs(h_, host_logits, count, host_rewards, host_done, host_obs, obs_count));
  }
  void set_host_chunks(int32_t chunks) { check(wdg_rollout_set_host_chunks(h_, chunks)); }
  // overlapped consecutive launches (default on); false = serial launches
  void set_overlap(bool enabled) { check(wdg_rollout_set_overlap(h_, enabled ? 1 : 0)); }
  void run(int64_t steps) { check(wdg_rollout_run(h_, steps)); }
  void check_errors() { check(wdg_rollout_check(h_)); }
  std::vector<double> stats() {
    std::vector<double> out(WDG_STAT_COUNT);
    check(wdg_rollout_stats(h_, out.data(), WDG_STAT_COUNT));
    return out;
  }

 private:
  wdg_rollout* h_ = nullptr;
};

// Plan tuning overrides (wdg_set_tuning): how a plan maps the step onto the
// GPU, never what it computes; value < 0 restores the plan's choice.
inline void set_tuning(const std::string& key, int64_t value) { check(wdg_set_tuning(key.c_str(), value)); }

// The episode-statistics all-reduce of a sharded run:
// rank 0 creates the id, every rank builds the communicator from it.
class Comm {
 public:
  static std::vector<uint8_t> unique_id() {
    std::vector<uint8_t> id(128);
    check(wdg_comm_unique_id(id.data(), static_cast<int64_t>(id.size())));
    return id;
  }
  Comm(int32_t world, int32_t rank, const std::vector<uint8_t>& id) {
    check(wdg_comm_init(world, rank, id.data(), static_cast<int64_t>(id.size()), &h_));
  }
  explicit Comm(void* nccl_comm) { check(wdg_comm_wrap(nccl_comm, &h_)); }  // not owned
  ~Comm() { wdg_comm_destroy(h_); }
  Comm(const Comm&) = delete;
  Comm& operator=(const Comm&) = delete;
  // tracker sums of this shard -> ncclAllReduce(sum) into device double[8]
  void stats_allreduce(RolloutDriver& rollout, double* device_out) {
    check(wdg_stats_allreduce(rollout.raw(), h_, device_out));
  }

 private:
  wdg_comm* h_ = nullptr;
};

}  // namespace warp_b200
