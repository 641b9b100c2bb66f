// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (never shipped, never on the
// product path). A thin extern "C" shim, written for this repo, that drives the
// UNMODIFIED reference sources compiled straight from /root/reference/proj/src
// (see oracle/Makefile). It lets the Python tests and bench.py's cpu_baseline /
// --impl reference leg call the reference's own Tag path:
//   build_workspace        proj/src/harness.cpp:402-423 (re-done here: harness.cpp
//                          needs json.hpp + the trainer, which are off the path)
//   RolloutDriver::step    proj/src/harness.cpp:478-490 (zero logits, tracker=null)
//   check flow             proj/src/harness.cpp:563-633 (TagReference twin store)
// Only the reference's public headers are used; no reference source is copied.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#ifdef REF_HAVE_HARNESS
#include "warp/harness.hpp"
#endif
#include "warp/policy_model.hpp"
#include "warp/trainer.hpp"
#include "warp/data_store.hpp"
#include "warp/reset_manager.hpp"
#include "warp/sampler.hpp"
#include "warp/step_engine.hpp"
#include "warp/tag_env.hpp"
#include "wdg_b200.h"

namespace {

thread_local std::string g_err;

warp::TagConfig to_ref(const wdg_tag_config& c) {
  warp::TagConfig t;
  t.variant = c.variant == WDG_TAG_CONTINUOUS ? warp::TagVariant::Continuous
                                              : warp::TagVariant::Discrete;
  t.obs_mode = c.obs_mode == WDG_OBS_PARTIAL ? warp::ObsMode::Partial : warp::ObsMode::Full;
  t.grid_size = c.grid_size;
  t.world_length = c.world_length;
  t.num_taggers = c.num_taggers;
  t.num_runners = c.num_runners;
  t.episode_length = c.episode_length;
  t.tag_radius = c.tag_radius;
  t.k_nearest = c.k_nearest;
  t.tag_reward = c.tag_reward;
  t.tagged_penalty = c.tagged_penalty;
  t.max_speed_tagger = c.max_speed_tagger;
  t.max_speed_runner = c.max_speed_runner;
  t.accel_delta = c.accel_delta;
  t.turn_delta = c.turn_delta;
  t.seed = c.seed;
  return t;
}

// One wired world: the reference's store + plan + engine (worker_count=1, the
// only race-free setting) + resets, or the sequential
// TagReference on its own store (the checker's second store).
struct World {
  warp::TagConfig cfg;
  std::unique_ptr<warp::DataStore> store;
  warp::TagPlan plan;
  std::unique_ptr<warp::StepEngine> engine;
  std::unique_ptr<warp::TagReference> reference;
  std::unique_ptr<warp::ResetManager> resets;
  std::vector<double> zero_logits;
  int64_t C = 1, V = 5;
};

World* make_world(const warp::TagConfig& cfg, int64_t num_envs, bool sequential, int workers = 1) {
  auto w = std::make_unique<World>();
  w->cfg = cfg;
  cfg.validate();
  w->store = std::make_unique<warp::DataStore>(num_envs, cfg.num_agents());
  warp::register_tag_arrays(*w->store, cfg);
  w->store->lock();
  warp::ResetPolicy policy;
  policy.auto_reset = true;
  policy.zero_on_reset = warp::tag_zero_on_reset();
  if (sequential) {
    w->reference = std::make_unique<warp::TagReference>(*w->store, cfg);
    warp::TagReference* ref = w->reference.get();
    policy.reinitialize = [ref](warp::DataStore&, int64_t e, int64_t episode) {
      ref->reinit_env(e, episode);
    };
  } else {
    w->plan = warp::build_tag_plan(*w->store, cfg);
    warp::EngineConfig ecfg;
    ecfg.num_envs = num_envs;
    ecfg.num_agents = cfg.num_agents();
    ecfg.worker_count = workers;
    w->engine = std::make_unique<warp::StepEngine>(ecfg);
    policy.reinitialize = warp::make_tag_reinit(w->plan);
  }
  w->resets = std::make_unique<warp::ResetManager>(*w->store, policy);
  w->C = cfg.action_categories();
  w->V = cfg.action_choices();
  w->zero_logits.assign(static_cast<size_t>(num_envs * cfg.num_agents() * w->C * w->V), 0.0);
  return w.release();
}

template <class Fn>
int guarded(Fn&& fn) {
  try {
    return fn();
  } catch (const warp::Error& e) {
    g_err = e.what();
    return static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_err = e.what();
    return static_cast<int>(warp::Errc::state_error) + 1;
  }
}

void step_world(World* w, const double* logits, int64_t step, uint64_t seed) {
  std::span<const double> lg(logits ? logits : w->zero_logits.data(), w->zero_logits.size());
  warp::sample_actions(*w->store, lg, w->C, w->V, step, seed);
  if (w->engine) {
    w->engine->run_step(w->plan.plan, *w->store, step);
  } else {
    w->reference->step(step);
  }
  const std::vector<int64_t> ids = w->resets->detect_done(*w->store);
  w->resets->auto_reset(*w->store, ids);
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) const char* ref_last_error(void) { return g_err.c_str(); }

__attribute__((visibility("default"))) void ref_set_fault_bias(float bias) {
  warp::detail::fault_hooks().tag_radius_bias = bias;
}

__attribute__((visibility("default"))) int ref_world_create(const wdg_tag_config* cfg,
                                                            int64_t num_envs, int32_t sequential,
                                                            void** out) {
  return guarded([&] {
    *out = make_world(to_ref(*cfg), num_envs, sequential != 0);
    return 0;
  });
}

__attribute__((visibility("default"))) void ref_world_destroy(void* w) {
  delete static_cast<World*>(w);
}

// sample_actions (proj/src/sampler.cpp:5-40); logits NULL -> zeros.
__attribute__((visibility("default"))) int ref_world_sample(void* wp, const double* logits,
                                                            int64_t step, uint64_t seed) {
  return guarded([&] {
    World* w = static_cast<World*>(wp);
    std::span<const double> lg(logits ? logits : w->zero_logits.data(), w->zero_logits.size());
    warp::sample_actions(*w->store, lg, w->C, w->V, step, seed);
    return 0;
  });
}

// Engine run_step (step_engine.cpp:122-138) or TagReference::step (tag_env.cpp:530-577).
__attribute__((visibility("default"))) int ref_world_step(void* wp, int64_t step) {
  return guarded([&] {
    World* w = static_cast<World*>(wp);
    if (w->engine) {
      w->engine->run_step(w->plan.plan, *w->store, step);
    } else {
      w->reference->step(step);
    }
    return 0;
  });
}

// detect_done + auto_reset (reset_manager.cpp:20-44); *n_reset = #envs reset.
__attribute__((visibility("default"))) int ref_world_reset(void* wp, int64_t* n_reset) {
  return guarded([&] {
    World* w = static_cast<World*>(wp);
    const std::vector<int64_t> ids = w->resets->detect_done(*w->store);
    w->resets->auto_reset(*w->store, ids);
    if (n_reset) *n_reset = static_cast<int64_t>(ids.size());
    return 0;
  });
}

// auto_reset for an explicit id list.
__attribute__((visibility("default"))) int ref_world_reset_ids(void* wp, const int64_t* ids,
                                                               int64_t n) {
  return guarded([&] {
    World* w = static_cast<World*>(wp);
    w->resets->auto_reset(*w->store, std::span<const int64_t>(ids, static_cast<size_t>(n)));
    return 0;
  });
}

// RolloutDriver::step x n (harness.cpp:478-494), steps first_step.. with
// zero logits when logits == NULL.
__attribute__((visibility("default"))) int ref_world_rollout(void* wp, const double* logits,
                                                             int64_t first_step, int64_t n,
                                                             uint64_t seed) {
  return guarded([&] {
    World* w = static_cast<World*>(wp);
    for (int64_t i = 0; i < n; ++i) step_world(w, logits, first_step + i, seed);
    return 0;
  });
}

__attribute__((visibility("default"))) int ref_world_pull(void* wp, const char* name, void* dst,
                                                          int64_t bytes) {
  return guarded([&] {
    World* w = static_cast<World*>(wp);
    const warp::ArrayHandle h = w->store->handle(name);
    const warp::ArrayInfo& info = w->store->info(h);
    const int64_t need = info.total_elems * warp::element_size(info.spec.kind);
    if (need != bytes) warp::raise(warp::Errc::shape_mismatch, "ref_world_pull: byte count");
    for (int64_t e = 0; e < w->store->num_envs(); ++e) {
      auto row = w->store->env_row_bytes(h, e);
      std::memcpy(static_cast<char*>(dst) + e * static_cast<int64_t>(row.size()), row.data(),
                  row.size());
    }
    return 0;
  });
}

__attribute__((visibility("default"))) int ref_world_push(void* wp, const char* name,
                                                          const void* src, int64_t bytes) {
  return guarded([&] {
    World* w = static_cast<World*>(wp);
    const warp::ArrayHandle h = w->store->handle(name);
    const warp::ArrayInfo& info = w->store->info(h);
    const int64_t need = info.total_elems * warp::element_size(info.spec.kind);
    if (need != bytes) warp::raise(warp::Errc::shape_mismatch, "ref_world_push: byte count");
    for (int64_t e = 0; e < w->store->num_envs(); ++e) {
      auto row = w->store->env_row_bytes(h, e);
      std::memcpy(row.data(), static_cast<const char*>(src) + e * static_cast<int64_t>(row.size()),
                  row.size());
    }
    return 0;
  });
}

__attribute__((visibility("default"))) int64_t ref_world_episodes(void* wp, int64_t env) {
  World* w = static_cast<World*>(wp);
  try {
    return w->resets->episodes_started(env);
  } catch (...) {
    return -1;
  }
}

__attribute__((visibility("default"))) int ref_hw_threads(void) {
  const unsigned n = std::thread::hardware_concurrency();
  return n == 0 ? 1 : static_cast<int>(n);
}

// CPU baseline (ii): `threads` independent single-worker reference worlds
// sharing `total_envs` envs (the race-free sharded form of the reference's
// StepEngine; shard i holds total/threads envs, the first
// total % threads one more), each running RolloutDriver::step with zero
// logits. Times `steps` steps after `warmup` steps with all threads released
// together; returns aggregate env-steps/s and the setup seconds.
__attribute__((visibility("default"))) int ref_bench_sharded_total(const wdg_tag_config* cfg,
                                                                   int64_t total_envs, int threads,
                                                                   int64_t warmup, int64_t steps,
                                                                   double* env_steps_per_s,
                                                                   double* setup_s, double* run_s) {
  return guarded([&] {
    using Clock = std::chrono::steady_clock;
    const warp::TagConfig tc = to_ref(*cfg);
    threads = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(threads, total_envs)));
    std::vector<int64_t> share(static_cast<size_t>(threads), total_envs / threads);
    for (int64_t i = 0; i < total_envs % threads; ++i) ++share[static_cast<size_t>(i)];
    std::vector<std::unique_ptr<World>> worlds(static_cast<size_t>(threads));
    const auto t0 = Clock::now();
    {
      std::vector<std::thread> pool;
      for (int i = 0; i < threads; ++i) {
        pool.emplace_back([&, i] {
          worlds[static_cast<size_t>(i)].reset(make_world(tc, share[static_cast<size_t>(i)], false));
        });
      }
      for (auto& t : pool) t.join();
    }
    const auto t1 = Clock::now();
    std::atomic<int> ready{0};
    std::atomic<bool> go{false};
    std::vector<std::thread> pool;
    for (int i = 0; i < threads; ++i) {
      pool.emplace_back([&, i] {
        World* w = worlds[static_cast<size_t>(i)].get();
        for (int64_t s = 0; s < warmup; ++s) step_world(w, nullptr, s, tc.seed);
        ready.fetch_add(1);
        while (!go.load()) std::this_thread::yield();
        for (int64_t s = 0; s < steps; ++s) step_world(w, nullptr, warmup + s, tc.seed);
      });
    }
    while (ready.load() < threads) std::this_thread::yield();
    const auto r0 = Clock::now();
    go.store(true);
    for (auto& t : pool) t.join();
    const double wall = std::chrono::duration<double>(Clock::now() - r0).count();
    *setup_s = std::chrono::duration<double>(t1 - t0).count();
    *run_s = wall;
    *env_steps_per_s = static_cast<double>(total_envs) * steps / wall;
    return 0;
  });
}

__attribute__((visibility("default"))) int ref_bench_sharded(const wdg_tag_config* cfg,
                                                             int64_t envs_per_thread, int threads,
                                                             int64_t warmup, int64_t steps,
                                                             double* env_steps_per_s,
                                                             double* setup_s, double* run_s) {
  return ref_bench_sharded_total(cfg, envs_per_thread * threads, threads, warmup, steps, env_steps_per_s,
                                 setup_s, run_s);
}

// CPU baseline (i), reference-faithful: ONE world whose StepEngine runs
// `workers` threads (step_engine.cpp:17-33), driven by RolloutDriver::step
// (harness.cpp:478-490) with zero logits, as measure_rollout_sps does
// (harness.cpp:715-741). The engine's phase barrier can race and hang at
// workers > 1: callers run this in a child process under a
// watchdog.
__attribute__((visibility("default"))) int ref_bench_engine(const wdg_tag_config* cfg, int64_t num_envs,
                                                            int workers, int64_t warmup, int64_t steps,
                                                            double* env_steps_per_s, double* setup_s,
                                                            double* run_s) {
  return guarded([&] {
    using Clock = std::chrono::steady_clock;
    const warp::TagConfig tc = to_ref(*cfg);
    const auto t0 = Clock::now();
    std::unique_ptr<World> w(make_world(tc, num_envs, false, std::max(1, workers)));
    const auto t1 = Clock::now();
    for (int64_t s = 0; s < warmup; ++s) step_world(w.get(), nullptr, s, tc.seed);
    const auto r0 = Clock::now();
    for (int64_t s = 0; s < steps; ++s) step_world(w.get(), nullptr, warmup + s, tc.seed);
    const double wall = std::chrono::duration<double>(Clock::now() - r0).count();
    *setup_s = std::chrono::duration<double>(t1 - t0).count();
    *run_s = wall;
    *env_steps_per_s = static_cast<double>(num_envs) * steps / wall;
    return 0;
  });
}

// ---- policy network (proj/src/policy_model.cpp), test oracle only ---------
namespace {
warp::PolicyDims ref_dims(int64_t obs_dim, const int64_t* hidden, int32_t nh, int64_t C, int64_t V) {
  warp::PolicyDims d;
  d.obs_dim = obs_dim;
  d.hidden.assign(hidden, hidden + nh);
  d.num_categories = C;
  d.num_choices = V;
  return d;
}
}  // namespace

// init_policy(seed, dims) flattened with for_each_param (policy_model.cpp:44-56).
__attribute__((visibility("default"))) int ref_policy_init(uint64_t seed, int64_t obs_dim,
                                                           const int64_t* hidden, int32_t nh,
                                                           int64_t C, int64_t V, double* out,
                                                           int64_t count) {
  return guarded([&] {
    const warp::PolicyParams p = warp::init_policy(seed, ref_dims(obs_dim, hidden, nh, C, V));
    if (p.param_count() != count) throw warp::Error(warp::Errc::shape_mismatch, "param count");
    int64_t i = 0;
    p.for_each_param([&](const double& v) { out[i++] = v; });
    return 0;
  });
}

// forward_parallel(params, double(obs), rows, 1 worker) (policy_model.cpp:199-220).
__attribute__((visibility("default"))) int ref_policy_forward(const double* params, int64_t obs_dim,
                                                              const int64_t* hidden, int32_t nh,
                                                              int64_t C, int64_t V, const float* obs,
                                                              int64_t rows, double* logits,
                                                              double* values) {
  return guarded([&] {
    warp::PolicyParams p = warp::init_policy(0, ref_dims(obs_dim, hidden, nh, C, V));
    int64_t i = 0;
    p.for_each_param([&](double& v) { v = params[i++]; });
    std::vector<double> x(static_cast<size_t>(rows * obs_dim));
    for (size_t k = 0; k < x.size(); ++k) x[k] = static_cast<double>(obs[k]);
    std::vector<double> lg(static_cast<size_t>(rows * C * V)), vals(static_cast<size_t>(rows));
    warp::forward_parallel(p, x, rows, 1, lg, vals);
    if (logits) std::copy(lg.begin(), lg.end(), logits);
    if (values) std::copy(vals.begin(), vals.end(), values);
    return 0;
  });
}

// compute_returns(batch, gamma) (trainer.cpp:73-88) on a batch filled from
// the given arrays.
__attribute__((visibility("default"))) int ref_compute_returns(const float* rewards, const uint8_t* done,
                                                               const double* bootstrap, int64_t T, int64_t E,
                                                               int64_t A, double gamma, double* returns) {
  return guarded([&] {
    warp::RolloutBatch b;
    b.resize(T, E, A, 1, 1);
    std::copy(rewards, rewards + T * E * A, b.rewards.begin());
    std::copy(done, done + T * E, b.done.begin());
    std::copy(bootstrap, bootstrap + E * A, b.bootstrap.begin());
    const std::vector<double> r = warp::compute_returns(b, gamma);
    std::copy(r.begin(), r.end(), returns);
    return 0;
  });
}

#ifdef REF_HAVE_HARNESS
// RunConfig::from_string -> to_json_string() / config_hash() (harness.cpp:
// 279-322): the canonical form the session ABI must reproduce. Writes a
// NUL-terminated string; returns its length or a negative status.
__attribute__((visibility("default"))) int64_t ref_config_canonical(const char* text, int32_t hash,
                                                                    char* out, int64_t cap) {
  try {
    const warp::RunConfig c = warp::RunConfig::from_string(text);
    c.validate();
    const std::string s = hash ? c.config_hash() : c.to_json_string();
    if (static_cast<int64_t>(s.size()) + 1 > cap) return -1000;
    std::memcpy(out, s.c_str(), s.size() + 1);
    return static_cast<int64_t>(s.size());
  } catch (const warp::Error& e) {
    g_err = e.what();
    return -static_cast<int64_t>(e.code());
  }
}
#endif

}  // extern "C"
