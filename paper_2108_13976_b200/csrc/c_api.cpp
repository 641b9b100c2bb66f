// c_api.cpp — extern "C" boundary (include/wdg_b200.h) over the C++ facade.
// Convention of the reference C ABI (proj/src/c_api.cpp:21-58): every call is
// guarded, exceptions map 1:1 onto status codes, the message is kept in a
// thread-local buffer returned by wdg_last_error().
#include <cstring>
#include <fstream>
#include <sstream>
#include <memory>
#include <string>

#include "facade.hpp"
#include "policy.hpp"
#include "batch.hpp"

struct wdg_store {
  std::unique_ptr<wdg::DataStore> impl;
};
struct wdg_tag_plan {
  std::unique_ptr<wdg::TagPlan> impl;
};
struct wdg_resets {
  std::unique_ptr<wdg::ResetManager> impl;
};
struct wdg_rollout {
  std::unique_ptr<wdg::Rollout> impl;
};
struct wdg_policy {
  std::unique_ptr<wdg::Policy> impl;
};
struct wdg_batch {
  std::unique_ptr<wdg::RolloutBatch> impl;
};
struct wdg_comm {
  wdg::Comm* impl = nullptr;
  ~wdg_comm() { wdg::comm_destroy(impl); }
};
struct wdg_session {
  wdg::Session* impl = nullptr;
  ~wdg_session() { wdg::session_close(impl); }
};

namespace {

thread_local std::string g_last_error;

template <class Fn>
wdg_status guarded(Fn&& fn) {
  try {
    fn();
    return WDG_OK;
  } catch (const wdg::Error& e) {
    g_last_error = e.what();
    return static_cast<wdg_status>(e.code());
  } catch (const std::bad_alloc& e) {
    g_last_error = std::string("out of host memory: ") + e.what();
    return WDG_ERR_UNKNOWN;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return WDG_ERR_UNKNOWN;
  } catch (...) {
    g_last_error = "unknown error";
    return WDG_ERR_UNKNOWN;
  }
}

template <class T>
T* need(T* p, const char* what) {
  if (p == nullptr) wdg::raise(wdg::Errc::invalid_argument, std::string("null ") + what);
  return p;
}

}  // namespace

extern "C" {

const char* wdg_version(void) { return "0.1.0-b200"; }

const char* wdg_status_name(wdg_status s) {
  switch (s) {
    case WDG_OK: return "WD_OK";
    case WDG_ERR_INVALID_ARGUMENT: return "WD_ERR_INVALID_ARGUMENT";
    case WDG_ERR_DUPLICATE_NAME: return "WD_ERR_DUPLICATE_NAME";
    case WDG_ERR_SHAPE_MISMATCH: return "WD_ERR_SHAPE_MISMATCH";
    case WDG_ERR_STORE_LOCKED: return "WD_ERR_STORE_LOCKED";
    case WDG_ERR_MISSING_PLACEHOLDER: return "WD_ERR_MISSING_PLACEHOLDER";
    case WDG_ERR_UNKNOWN_NAME: return "WD_ERR_UNKNOWN_NAME";
    case WDG_ERR_INDEX_OUT_OF_RANGE: return "WD_ERR_INDEX_OUT_OF_RANGE";
    case WDG_ERR_INVALID_CONFIG: return "WD_ERR_INVALID_CONFIG";
    case WDG_ERR_STEP_FAILURE: return "WD_ERR_STEP_FAILURE";
    case WDG_ERR_NON_FINITE: return "WD_ERR_NON_FINITE";
    case WDG_ERR_PARSE: return "WD_ERR_PARSE";
    case WDG_ERR_IO: return "WD_ERR_IO";
    case WDG_ERR_STATE: return "WD_ERR_STATE";
    case WDG_ERR_UNKNOWN: return "WD_ERR_UNKNOWN";
    case WDG_ERR_CUDA: return "WDG_ERR_CUDA";
  }
  return "WD_ERR_UNKNOWN";
}

const char* wdg_last_error(void) { return g_last_error.c_str(); }

wdg_status wdg_device_count(int32_t* out) {
  return guarded([&] {
    need(out, "out");
    int n = 0;
    cudaError_t err = cudaGetDeviceCount(&n);
    if (err != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    *out = n;
  });
}

wdg_status wdg_set_device(int32_t device) {
  return guarded([&] { wdg::cuda_check(cudaSetDevice(device), "cudaSetDevice"); });
}

void wdg_set_fault_tag_radius_bias(float bias) { wdg::fault_tag_radius_bias() = bias; }

// ---- store -----------------------------------------------------------------
wdg_status wdg_store_create(int64_t num_envs, int64_t num_agents, wdg_store** out) {
  return guarded([&] {
    need(out, "out");
    auto s = std::make_unique<wdg_store>();
    s->impl = std::make_unique<wdg::DataStore>(num_envs, num_agents);
    *out = s.release();
  });
}

void wdg_store_destroy(wdg_store* store) { delete store; }

wdg_status wdg_store_set_env_offset(wdg_store* store, int64_t off) {
  return guarded([&] { need(store, "store")->impl->set_env_offset(off); });
}

wdg_status wdg_store_set_stream(wdg_store* store, void* stream) {
  return guarded([&] { need(store, "store")->impl->set_stream(static_cast<cudaStream_t>(stream)); });
}

wdg_status wdg_store_register_array(wdg_store* store, const char* name, const int64_t* shape,
                                    int32_t ndim, int32_t kind, int32_t snapshot_on_reset,
                                    const void* host_initial, int64_t initial_count,
                                    int32_t* out_handle) {
  return guarded([&] {
    need(store, "store");
    need(name, "name");
    if (ndim < 0 || (ndim > 0 && shape == nullptr)) {
      wdg::raise(wdg::Errc::invalid_argument, "register_array: bad shape");
    }
    wdg::ArraySpec spec;
    spec.name = name;
    spec.shape.assign(shape, shape + ndim);
    spec.kind = kind;
    spec.snapshot_on_reset = snapshot_on_reset != 0;
    const int32_t h = store->impl->register_array(spec, host_initial, initial_count);
    if (out_handle) *out_handle = h;
  });
}

wdg_status wdg_store_lock(wdg_store* store) {
  return guarded([&] { need(store, "store")->impl->lock(); });
}

wdg_status wdg_store_locked(const wdg_store* store, int32_t* out) {
  return guarded([&] { *need(out, "out") = need(store, "store")->impl->locked() ? 1 : 0; });
}

wdg_status wdg_store_num_envs(const wdg_store* store, int64_t* out) {
  return guarded([&] { *need(out, "out") = need(store, "store")->impl->num_envs(); });
}

wdg_status wdg_store_num_agents(const wdg_store* store, int64_t* out) {
  return guarded([&] { *need(out, "out") = need(store, "store")->impl->num_agents(); });
}

wdg_status wdg_store_handle(const wdg_store* store, const char* name, int32_t* out) {
  return guarded([&] { *need(out, "out") = need(store, "store")->impl->handle(need(name, "name")); });
}

wdg_status wdg_store_num_arrays(const wdg_store* store, int32_t* out) {
  return guarded([&] { *need(out, "out") = need(store, "store")->impl->num_arrays(); });
}

wdg_status wdg_store_info(const wdg_store* store, int32_t handle, wdg_array_info* out) {
  return guarded([&] {
    need(out, "out");
    const wdg::DataStore& s = *need(store, "store")->impl;
    const wdg::ArrayInfo& in = s.info(handle);
    std::memset(out, 0, sizeof(*out));
    std::strncpy(out->name, in.spec.name.c_str(), WDG_MAX_NAME - 1);
    out->kind = in.spec.kind;
    out->ndim = static_cast<int32_t>(in.spec.shape.size());
    for (size_t i = 0; i < in.spec.shape.size(); ++i) out->shape[i] = in.spec.shape[i];
    out->total_elems = in.total_elems;
    out->env_stride = in.env_stride;
    out->agent_stride = in.agent_stride;
    out->has_agent_axis = in.has_agent_axis ? 1 : 0;
    out->snapshot_on_reset = in.spec.snapshot_on_reset ? 1 : 0;
  });
}

wdg_status wdg_store_push(wdg_store* store, int32_t handle, int64_t env_begin, int64_t env_count,
                          const void* host, int64_t bytes) {
  return guarded([&] { need(store, "store")->impl->push(handle, env_begin, env_count, host, bytes); });
}

wdg_status wdg_store_pull(const wdg_store* store, int32_t handle, int64_t env_begin,
                          int64_t env_count, void* host, int64_t bytes) {
  return guarded([&] { need(store, "store")->impl->pull(handle, env_begin, env_count, host, bytes); });
}

wdg_status wdg_store_device_ptr(wdg_store* store, int32_t handle, void** out) {
  return guarded([&] { *need(out, "out") = need(store, "store")->impl->device_ptr(handle); });
}

wdg_status wdg_store_restore_snapshot(wdg_store* store, const int64_t* env_ids, int64_t count) {
  return guarded([&] {
    if (count > 0) need(env_ids, "env_ids");
    if (count < 0) wdg::raise(wdg::Errc::invalid_argument, "restore_snapshot: negative count");
    need(store, "store")->impl->restore_snapshot(env_ids, count);
  });
}

wdg_status wdg_store_synchronize(wdg_store* store) {
  return guarded([&] { need(store, "store")->impl->synchronize(); });
}

// ---- tag -------------------------------------------------------------------
wdg_status wdg_tag_config_init(wdg_tag_config* c) {
  return guarded([&] {
    need(c, "cfg");
    c->variant = WDG_TAG_DISCRETE;
    c->obs_mode = WDG_OBS_FULL;
    c->grid_size = 20;
    c->world_length = 20.0;
    c->num_taggers = 2;
    c->num_runners = 10;
    c->episode_length = 500;
    c->tag_radius = 1.0;
    c->k_nearest = 5;
    c->tag_reward = 1.0;
    c->tagged_penalty = -1.0;
    c->max_speed_tagger = 1.0;
    c->max_speed_runner = 1.0;
    c->accel_delta = 0.1;
    c->turn_delta = 0.5235987755982988;
    c->seed = 0;
  });
}

wdg_status wdg_tag_config_validate(const wdg_tag_config* cfg) {
  return guarded([&] { wdg::validate_tag_config(*need(cfg, "cfg")); });
}

int64_t wdg_tag_obs_dim(const wdg_tag_config* cfg) {
  return cfg == nullptr ? -1 : wdg::tag_obs_dim(*cfg);
}

wdg_status wdg_register_tag_arrays(wdg_store* store, const wdg_tag_config* cfg) {
  return guarded([&] { wdg::register_tag_arrays(*need(store, "store")->impl, *need(cfg, "cfg")); });
}

wdg_status wdg_tag_zero_on_reset(const char** names, int32_t capacity, int32_t* count) {
  return guarded([&] {
    static const char* kNames[] = {"step_count", "rewards", "done", "tag_credits",
                                   "was_tagged", "sampled_actions", "observations"};
    const int32_t n = 7;
    if (count) *count = n;
    if (names) {
      for (int32_t i = 0; i < n && i < capacity; ++i) names[i] = kNames[i];
    }
  });
}

wdg_status wdg_build_tag_plan(wdg_store* store, const wdg_tag_config* cfg, wdg_tag_plan** out) {
  return guarded([&] {
    need(out, "out");
    auto p = std::make_unique<wdg_tag_plan>();
    p->impl = std::make_unique<wdg::TagPlan>(*need(store, "store")->impl, *need(cfg, "cfg"));
    *out = p.release();
  });
}

wdg_status wdg_build_tag_reference(wdg_store* store, const wdg_tag_config* cfg, wdg_tag_plan** out) {
  return guarded([&] {
    need(out, "out");
    auto p = std::make_unique<wdg_tag_plan>();
    p->impl = std::make_unique<wdg::TagPlan>(*need(store, "store")->impl, *need(cfg, "cfg"), true);
    *out = p.release();
  });
}

void wdg_tag_plan_destroy(wdg_tag_plan* plan) { delete plan; }

wdg_status wdg_run_step(wdg_tag_plan* plan, int64_t step_index) {
  return guarded([&] { need(plan, "plan")->impl->run_step(step_index); });
}

wdg_status wdg_tag_plan_geometry(const wdg_tag_plan* plan, int32_t* threads_per_cta,
                                 int32_t* envs_per_cta, int32_t* grid_ctas, int32_t* uses_grid,
                                 int32_t* smem_bytes) {
  return guarded([&] {
    const wdg::TagDevConfig& d = need(plan, "plan")->impl->dev();
    if (threads_per_cta) *threads_per_cta = d.threads;
    if (envs_per_cta) *envs_per_cta = d.envs_per_cta;
    if (grid_ctas) *grid_ctas = d.grid_ctas;
    if (uses_grid) *uses_grid = d.use_grid;
    if (smem_bytes) *smem_bytes = d.smem_bytes;
  });
}

wdg_status wdg_sample_actions(wdg_store* store, const double* logits, int64_t logits_count,
                              int64_t num_categories, int64_t num_choices, int64_t step,
                              uint64_t seed) {
  return guarded([&] {
    wdg::sample_actions(*need(store, "store")->impl, logits, logits_count, num_categories,
                        num_choices, step, seed);
  });
}

// ---- resets ------------------------------------------------------------------
wdg_status wdg_reset_manager_create(wdg_store* store, int32_t auto_reset,
                                    const char* const* zero_on_reset, int32_t n_zero,
                                    wdg_tag_plan* reinit_plan, wdg_resets** out) {
  return guarded([&] {
    need(out, "out");
    if (n_zero < 0 || (n_zero > 0 && zero_on_reset == nullptr)) {
      wdg::raise(wdg::Errc::invalid_argument, "reset_manager: bad zero_on_reset list");
    }
    std::vector<std::string> names;
    for (int32_t i = 0; i < n_zero; ++i) names.emplace_back(need(zero_on_reset[i], "name"));
    auto r = std::make_unique<wdg_resets>();
    r->impl = std::make_unique<wdg::ResetManager>(*need(store, "store")->impl, auto_reset != 0,
                                                  std::move(names),
                                                  reinit_plan ? reinit_plan->impl.get() : nullptr);
    *out = r.release();
  });
}

void wdg_reset_manager_destroy(wdg_resets* resets) { delete resets; }

wdg_status wdg_detect_done(wdg_resets* resets, int64_t* env_ids, int64_t capacity, int64_t* count) {
  return guarded([&] {
    const std::vector<int64_t> ids = need(resets, "resets")->impl->detect_done();
    if (count) *count = static_cast<int64_t>(ids.size());
    if (env_ids) {
      for (size_t i = 0; i < ids.size() && static_cast<int64_t>(i) < capacity; ++i) env_ids[i] = ids[i];
    }
  });
}

wdg_status wdg_auto_reset(wdg_resets* resets, const int64_t* env_ids, int64_t count) {
  return guarded([&] {
    if (count < 0) wdg::raise(wdg::Errc::invalid_argument, "auto_reset: negative count");
    if (count > 0) need(env_ids, "env_ids");
    need(resets, "resets")->impl->auto_reset(env_ids, count);
  });
}

wdg_status wdg_auto_reset_on_done(wdg_resets* resets) {
  return guarded([&] { need(resets, "resets")->impl->auto_reset_on_done(); });
}

wdg_status wdg_episodes_started(const wdg_resets* resets, int64_t env_id, int64_t* out) {
  return guarded([&] { *need(out, "out") = need(resets, "resets")->impl->episodes_started(env_id); });
}

// ---- rollout -----------------------------------------------------------------
wdg_status wdg_rollout_create(wdg_store* store, wdg_tag_plan* plan, wdg_resets* resets,
                              uint64_t sample_seed, wdg_rollout** out) {
  return guarded([&] {
    need(out, "out");
    auto r = std::make_unique<wdg_rollout>();
    r->impl = std::make_unique<wdg::Rollout>(*need(store, "store")->impl, *need(plan, "plan")->impl,
                                             resets ? resets->impl.get() : nullptr, sample_seed);
    *out = r.release();
  });
}

void wdg_rollout_destroy(wdg_rollout* rollout) { delete rollout; }

wdg_status wdg_rollout_set_logits(wdg_rollout* r, const double* logits, int64_t count) {
  return guarded([&] { need(r, "rollout")->impl->set_logits(logits, count); });
}

wdg_status wdg_rollout_set_fused(wdg_rollout* r, int32_t fused) {
  return guarded([&] { need(r, "rollout")->impl->set_fused(fused != 0); });
}

wdg_status wdg_rollout_set_overlap(wdg_rollout* r, int32_t enabled) {
  return guarded([&] { need(r, "rollout")->impl->set_overlap(enabled != 0); });
}

wdg_status wdg_set_tuning(const char* key, int64_t value) {
  return guarded([&] {
    if (key == nullptr) wdg::raise(wdg::Errc::invalid_argument, "set_tuning: null key");
    wdg::set_tuning(key, value);
  });
}

wdg_status wdg_rollout_set_graphs(wdg_rollout* r, int32_t enabled) {
  return guarded([&] { need(r, "rollout")->impl->set_graphs(enabled != 0); });
}

wdg_status wdg_rollout_step(wdg_rollout* r) {
  return guarded([&] { need(r, "rollout")->impl->step(); });
}

wdg_status wdg_rollout_step_host(wdg_rollout* r, const double* host_logits, int64_t count,
                                 float* host_rewards, uint8_t* host_done) {
  return guarded([&] {
    need(r, "rollout")->impl->step_host(host_logits, count, host_rewards, host_done);
  });
}

wdg_status wdg_rollout_step_host_obs(wdg_rollout* r, const double* host_logits, int64_t count,
                                     float* host_rewards, uint8_t* host_done, float* host_obs,
                                     int64_t obs_count) {
  return guarded([&] {
    need(r, "rollout")->impl->step_host(host_logits, count, host_rewards, host_done, host_obs, obs_count);
  });
}

wdg_status wdg_rollout_set_host_chunks(wdg_rollout* r, int32_t chunks) {
  return guarded([&] {
    if (chunks < 0) wdg::raise(wdg::Errc::invalid_argument, "set_host_chunks: chunks must be >= 0");
    need(r, "rollout")->impl->set_host_chunks(chunks);
  });
}

wdg_status wdg_rollout_reduce_stats_into(wdg_rollout* r, double* device_out) {
  return guarded([&] { need(r, "rollout")->impl->reduce_stats_into(device_out); });
}

// ---- NCCL statistics all-reduce -------------------------
wdg_status wdg_nccl_version(int32_t* out) {
  return guarded([&] { *need(out, "out") = wdg::comm_nccl_version(); });
}

wdg_status wdg_comm_unique_id(uint8_t* out, int64_t bytes) {
  return guarded([&] { wdg::comm_unique_id(out, bytes); });
}

wdg_status wdg_comm_init(int32_t world, int32_t rank, const uint8_t* id, int64_t bytes, wdg_comm** out) {
  return guarded([&] {
    need(out, "out");
    auto c = std::make_unique<wdg_comm>();
    c->impl = wdg::comm_init(world, rank, id, bytes);
    *out = c.release();
  });
}

wdg_status wdg_comm_wrap(void* nccl_comm, wdg_comm** out) {
  return guarded([&] {
    need(out, "out");
    auto c = std::make_unique<wdg_comm>();
    c->impl = wdg::comm_wrap(nccl_comm);
    *out = c.release();
  });
}

void wdg_comm_destroy(wdg_comm* comm) { delete comm; }

wdg_status wdg_comm_info(const wdg_comm* comm, int32_t* world, int32_t* rank) {
  return guarded([&] {
    const wdg::Comm* c = need(need(comm, "comm")->impl, "comm");
    if (world) *world = c->world;
    if (rank) *rank = c->rank;
  });
}

wdg_status wdg_stats_allreduce(wdg_rollout* r, wdg_comm* comm, double* device_out) {
  return guarded([&] {
    if (device_out == nullptr) wdg::raise(wdg::Errc::invalid_argument, "stats_allreduce: null output");
    wdg::stats_allreduce(*need(r, "rollout")->impl, need(need(comm, "comm")->impl, "comm"), device_out);
  });
}

wdg_status wdg_rollout_run(wdg_rollout* r, int64_t steps) {
  return guarded([&] { need(r, "rollout")->impl->run(steps); });
}

wdg_status wdg_rollout_next_step(const wdg_rollout* r, int64_t* out) {
  return guarded([&] { *need(out, "out") = need(r, "rollout")->impl->next_step(); });
}

wdg_status wdg_rollout_check(wdg_rollout* r) {
  return guarded([&] { need(r, "rollout")->impl->check(); });
}

wdg_status wdg_rollout_stats(wdg_rollout* r, double* out, int32_t count) {
  return guarded([&] { need(r, "rollout")->impl->stats(need(out, "out"), count); });
}

wdg_status wdg_rollout_reset_stats(wdg_rollout* r) {
  return guarded([&] { need(r, "rollout")->impl->reset_stats(); });
}

wdg_status wdg_rollout_stats_device_ptr(wdg_rollout* r, double** out) {
  return guarded([&] { *need(out, "out") = need(r, "rollout")->impl->stats_device(); });
}


wdg_status wdg_policy_create(int64_t obs_dim, const int64_t* hidden, int32_t num_hidden,
                             int64_t num_categories, int64_t num_choices, wdg_policy** out) {
  return guarded([&] {
    need(out, "out");
    if (num_hidden < 0 || (num_hidden > 0 && hidden == nullptr)) {
      wdg::raise(wdg::Errc::invalid_argument, "policy create: bad hidden sizes");
    }
    wdg::PolicyDims d;
    d.obs_dim = obs_dim;
    d.hidden.assign(hidden, hidden + num_hidden);
    d.num_categories = num_categories;
    d.num_choices = num_choices;
    auto p = std::make_unique<wdg_policy>();
    p->impl = std::make_unique<wdg::Policy>(d);
    *out = p.release();
  });
}

void wdg_policy_destroy(wdg_policy* policy) { delete policy; }

wdg_status wdg_policy_init(wdg_policy* policy, uint64_t seed) {
  return guarded([&] { need(policy, "policy")->impl->init(seed); });
}

wdg_status wdg_policy_param_count(const wdg_policy* policy, int64_t* out) {
  return guarded([&] { *need(out, "out") = need(policy, "policy")->impl->param_count(); });
}

wdg_status wdg_policy_set_params(wdg_policy* policy, const double* host_params, int64_t count) {
  return guarded([&] { need(policy, "policy")->impl->set_params(host_params, count); });
}

wdg_status wdg_policy_get_params(const wdg_policy* policy, double* host_params, int64_t count) {
  return guarded([&] { need(policy, "policy")->impl->get_params(host_params, count); });
}

wdg_status wdg_policy_forward(const wdg_policy* policy, const float* obs, int64_t num_envs,
                              int64_t num_agents, int64_t agent_begin, int64_t agent_end,
                              double* logits, double* values, int32_t precision, void* cuda_stream) {
  return guarded([&] {
    const wdg::Policy& p = *need(policy, "policy")->impl;
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    uint32_t* err = nullptr;
    wdg::cuda_check(cudaMallocAsync(reinterpret_cast<void**>(&err), sizeof(uint32_t), st), "policy error word");
    wdg::cuda_check(cudaMemsetAsync(err, 0, sizeof(uint32_t), st), "policy error clear");
    uint32_t host_err = 0;
    try {
      p.forward_agents(obs, num_envs, num_agents, agent_begin, agent_end, logits, values, precision, st, err);
      wdg::cuda_check(cudaMemcpyAsync(&host_err, err, sizeof(uint32_t), cudaMemcpyDeviceToHost, st),
                      "policy error read");
      wdg::cuda_check(cudaStreamSynchronize(st), "policy forward");
    } catch (...) {
      cudaFreeAsync(err, st);
      throw;
    }
    cudaFreeAsync(err, st);
    if (host_err & wdg::kErrNonFinite) wdg::raise(wdg::Errc::non_finite, "forward: non-finite observation");
  });
}

wdg_status wdg_rollout_set_policies(wdg_rollout* rollout, const wdg_policy* tagger,
                                    const wdg_policy* runner, int32_t precision) {
  return guarded([&] {
    need(rollout, "rollout")->impl->set_policies(tagger ? tagger->impl.get() : nullptr,
                                                 runner ? runner->impl.get() : nullptr, precision);
  });
}

wdg_status wdg_rollout_set_keep_policy_outputs(wdg_rollout* rollout, int32_t keep) {
  return guarded([&] { need(rollout, "rollout")->impl->set_keep_policy_outputs(keep != 0); });
}

wdg_status wdg_rollout_policy_outputs(wdg_rollout* rollout, const double** logits, const double** values) {
  return guarded([&] {
    const wdg::Rollout& r = *need(rollout, "rollout")->impl;
    if (logits) *logits = r.policy_logits();
    if (values) *values = r.policy_values();
  });
}

wdg_status wdg_copy_to_host(const void* device_src, void* host_dst, int64_t bytes) {
  return guarded([&] {
    if (bytes < 0) wdg::raise(wdg::Errc::invalid_argument, "copy_to_host: negative size");
    if (bytes == 0) return;
    need(device_src, "device_src");
    need(host_dst, "host_dst");
    wdg::cuda_check(cudaMemcpy(host_dst, device_src, static_cast<size_t>(bytes), cudaMemcpyDeviceToHost),
                    "copy_to_host");
  });
}

wdg_status wdg_batch_create(const wdg_store* store, int64_t horizon, wdg_batch** out) {
  return guarded([&] {
    need(out, "out");
    const wdg::DataStore& st = *need(store, "store")->impl;
    const wdg::ArrayInfo& obs = st.info(st.handle(wdg::kObservations));
    const wdg::ArrayInfo& act = st.info(st.handle(wdg::kSampledActions));
    auto b = std::make_unique<wdg_batch>();
    b->impl = std::make_unique<wdg::RolloutBatch>(horizon, st.num_envs(), st.num_agents(), obs.agent_stride,
                                                  act.agent_stride);
    *out = b.release();
  });
}

void wdg_batch_destroy(wdg_batch* batch) { delete batch; }

wdg_status wdg_batch_get_view(const wdg_batch* batch, wdg_batch_view* out) {
  return guarded([&] {
    const wdg::RolloutBatch& b = *need(batch, "batch")->impl;
    need(out, "out");
    *out = wdg_batch_view{b.T, b.E, b.A, b.D, b.C, b.obs, b.actions, b.rewards, b.done,
                          b.active, b.values, b.logp, b.bootstrap};
  });
}

wdg_status wdg_rollout_collect(wdg_rollout* rollout, wdg_batch* batch) {
  return guarded([&] { need(rollout, "rollout")->impl->collect(*need(batch, "batch")->impl); });
}

wdg_status wdg_compute_returns(const wdg_batch* batch, double gamma, double* device_returns, void* cuda_stream) {
  return guarded([&] {
    wdg::compute_returns(*need(batch, "batch")->impl, gamma, device_returns,
                         static_cast<cudaStream_t>(cuda_stream));
    wdg::cuda_check(cudaStreamSynchronize(static_cast<cudaStream_t>(cuda_stream)), "compute_returns");
  });
}

// ---- session (c_api.cpp:97-255 of the reference) ----------------------------
wdg_status wdg_session_open(const char* config_json, wdg_session** out) {
  if (config_json == nullptr || out == nullptr) {
    g_last_error = "null argument";
    return WDG_ERR_INVALID_ARGUMENT;
  }
  return guarded([&] {
    auto s = std::make_unique<wdg_session>();
    s->impl = wdg::session_open(config_json);
    *out = s.release();
  });
}

wdg_status wdg_session_open_file(const char* path, wdg_session** out) {
  if (path == nullptr || out == nullptr) {
    g_last_error = "null argument";
    return WDG_ERR_INVALID_ARGUMENT;
  }
  return guarded([&] {
    std::ifstream is(path);
    if (!is) wdg::raise(wdg::Errc::io_error, std::string("cannot open config file: ") + path);
    std::stringstream ss;
    ss << is.rdbuf();
    auto s = std::make_unique<wdg_session>();
    s->impl = wdg::session_open(ss.str());
    *out = s.release();
  });
}

void wdg_session_close(wdg_session* session) { delete session; }

namespace {
wdg::Session* sess(wdg_session* s) {
  if (s == nullptr || s->impl == nullptr) wdg::raise(wdg::Errc::invalid_argument, "null session");
  return s->impl;
}
}  // namespace

wdg_status wdg_session_set_seed(wdg_session* session, uint64_t seed) {
  return guarded([&] { wdg::session_set_seed(sess(session), seed); });
}

wdg_status wdg_session_set_workers(wdg_session* session, int32_t workers) {
  return guarded([&] { wdg::session_set_workers(sess(session), workers); });
}

wdg_status wdg_session_set_output_dir(wdg_session* session, const char* dir) {
  return guarded([&] {
    if (dir == nullptr) wdg::raise(wdg::Errc::invalid_argument, "null output dir");
    wdg::session_set_output_dir(sess(session), dir);
  });
}

const char* wdg_session_config_json(wdg_session* session) {
  const char* r = nullptr;
  guarded([&] { r = wdg::session_config_json(sess(session)); });
  return r;
}

const char* wdg_session_config_hash(wdg_session* session) {
  const char* r = nullptr;
  guarded([&] { r = wdg::session_config_hash(sess(session)); });
  return r;
}

wdg_status wdg_session_run_check(wdg_session* session) {
  bool passed = true;
  const wdg_status st = guarded([&] { passed = wdg::session_run_check(sess(session)); });
  if (st != WDG_OK) return st;
  if (!passed) {
    g_last_error = "consistency check failed; see report for first divergence";
    return WDG_ERR_STATE;
  }
  return WDG_OK;
}

wdg_status wdg_session_run_bench_envs(wdg_session* session) {
  return guarded([&] { wdg::session_run_bench_envs(sess(session)); });
}

wdg_status wdg_session_run_bench_agents(wdg_session* session) {
  return guarded([&] { wdg::session_run_bench_agents(sess(session)); });
}

wdg_status wdg_session_run_training(wdg_session* session) {
  return guarded([&] {
    sess(session);
    wdg::raise(wdg::Errc::state_error,
               "training (the reference's CPU learner) is out of scope on the device path; "
               "use wdg_rollout_collect + wdg_compute_returns for device rollouts");
  });
}

const char* wdg_session_report_json(wdg_session* session) {
  const char* r = nullptr;
  guarded([&] { r = wdg::session_report_json(sess(session)); });
  return r;
}

const char* wdg_session_summary(wdg_session* session) {
  const char* r = nullptr;
  guarded([&] { r = wdg::session_summary(sess(session)); });
  return r;
}

wdg_status wdg_session_dump_array(wdg_session* session, const char* array_name, const char* csv_path) {
  if (array_name == nullptr || csv_path == nullptr) {
    g_last_error = "null argument";
    return WDG_ERR_INVALID_ARGUMENT;
  }
  return guarded([&] { wdg::session_dump_array(sess(session), array_name, csv_path); });
}

wdg_status wdg_rollout_launches(const wdg_rollout* r, int64_t* out) {
  return guarded([&] { *need(out, "out") = need(r, "rollout")->impl->launches(); });
}

}  // extern "C"
