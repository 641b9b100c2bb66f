// session.cpp — the reference's session C ABI (proj/include/warp/warp_c.h,
// proj/src/c_api.cpp) on the device path: a strict JSON
// RunConfig (proj/src/harness.cpp:32-158,279-324) with the same canonical
// serialization and FNV-1a config hash, and the run modes check / bench-envs /
// bench-agents (harness.cpp:563-898) driving the B200 kernels. Training is the
// reference's CPU learner and stays out of scope.
//
// parse_config / config_to_json follow harness.cpp:92-206 key by key (copied
// for byte-identical output, see StrictObj below).
//
// Compiled by nvcc (-x cu): the store comparison of `check` is a device kernel
// (compare_stores, harness.cpp:531-557, without pulling the stores to host).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <map>
#include <memory>
#include <optional>
#include <set>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "facade.hpp"
#include "policy.hpp"

#ifdef WDG_HAVE_JSON
#include <nlohmann/json.hpp>
#endif

namespace wdg {

#ifdef WDG_HAVE_JSON
namespace {

using nlohmann::json;
using Clock = std::chrono::steady_clock;
constexpr const char* kVersion = "0.1.0";  // common.hpp:9 (the report's format version)

// RunSettings / EngineConfig / TrainerConfig (harness.hpp:20-40,
// step_engine.hpp:52-57, trainer.hpp:16-30), same fields and defaults.
struct EngineCfg {
  int64_t num_envs = 1;
  int64_t num_agents = 1;
  int worker_count = 1;
  bool deterministic = true;
};
struct TrainerCfg {
  std::string algorithm = "a2c";
  double gamma = 0.99;
  int64_t rollout_horizon = 100;
  double learning_rate = 3e-4;
  double value_coef = 0.5;
  double entropy_coef = 0.01;
  double ppo_clip = 0.2;
  int64_t ppo_epochs = 4;
  double max_grad_norm = 0.5;
  int64_t iterations = 0;
  uint64_t seed = 0;
  std::vector<int64_t> hidden_sizes = {64, 64};
  int64_t checkpoint_every = 0;
};
struct RunSettings {
  std::string mode;
  std::string output_dir;
  int64_t check_steps = 100;
  std::vector<int64_t> env_counts = {1, 2, 4};
  std::vector<int64_t> agent_counts = {10, 100, 1000};
  std::vector<std::string> bench_obs_modes = {"partial", "full"};
  double bench_budget_ms = 1000.0;
  int64_t bench_reps = 3;
  bool dump_trajectory = false;
  std::vector<std::string> dump_arrays;
  std::string resume_from;
};
struct RunConfig {
  wdg_tag_config env;
  EngineCfg engine;
  TrainerCfg trainer;
  RunSettings run;
};

// StrictObj: copied from the reference (harness.cpp:32-66) with its key lists
// and error strings, because the canonical JSON, the FNV-1a config hash and the
// parse-error text must be byte-identical to the reference's (schema
// conformance, tests/test_session.py). Unknown keys and type errors are parse
// errors.
class StrictObj {
 public:
  StrictObj(const json& j, std::string path) : j_(j), path_(std::move(path)) {
    if (!j.is_object()) raise(Errc::parse_error, path_ + ": expected a JSON object");
  }
  template <class T>
  void opt(const char* key, T& out) {
    seen_.insert(key);
    if (!j_.contains(key)) return;
    try {
      out = j_.at(key).get<T>();
    } catch (const json::exception& e) {
      raise(Errc::parse_error, path_ + "." + key + ": " + e.what());
    }
  }
  const json* section(const char* key) {
    seen_.insert(key);
    return j_.contains(key) ? &j_.at(key) : nullptr;
  }
  void finish() const {
    for (auto it = j_.begin(); it != j_.end(); ++it) {
      if (!seen_.count(it.key())) raise(Errc::parse_error, path_ + ": unknown key \"" + it.key() + "\"");
    }
  }

 private:
  const json& j_;
  std::string path_;
  std::set<std::string> seen_;
};

int32_t variant_from(const std::string& s) {
  if (s == "discrete") return WDG_TAG_DISCRETE;
  if (s == "continuous") return WDG_TAG_CONTINUOUS;
  raise(Errc::parse_error, "env.variant must be \"discrete\" or \"continuous\", got \"" + s + "\"");
}
int32_t obs_from(const std::string& s) {
  if (s == "full") return WDG_OBS_FULL;
  if (s == "partial") return WDG_OBS_PARTIAL;
  raise(Errc::parse_error, "obs_mode must be \"full\" or \"partial\", got \"" + s + "\"");
}
const char* variant_name(int32_t v) { return v == WDG_TAG_DISCRETE ? "discrete" : "continuous"; }
const char* obs_name(int32_t m) { return m == WDG_OBS_FULL ? "full" : "partial"; }

RunConfig parse_config(const std::string& text) {
  json j;
  try {
    j = json::parse(text);
  } catch (const json::exception& e) {
    raise(Errc::parse_error, std::string("config: ") + e.what());
  }
  RunConfig c;
  wdg_tag_config_init(&c.env);
  StrictObj root(j, "config");
  if (const json* e = root.section("env")) {
    StrictObj o(*e, "env");
    std::string variant = variant_name(c.env.variant), obs = obs_name(c.env.obs_mode);
    o.opt("variant", variant);
    o.opt("obs_mode", obs);
    c.env.variant = variant_from(variant);
    c.env.obs_mode = obs_from(obs);
    o.opt("grid_size", c.env.grid_size);
    o.opt("world_length", c.env.world_length);
    o.opt("num_taggers", c.env.num_taggers);
    o.opt("num_runners", c.env.num_runners);
    o.opt("episode_length", c.env.episode_length);
    o.opt("tag_radius", c.env.tag_radius);
    o.opt("k_nearest", c.env.k_nearest);
    o.opt("tag_reward", c.env.tag_reward);
    o.opt("tagged_penalty", c.env.tagged_penalty);
    o.opt("max_speed_tagger", c.env.max_speed_tagger);
    o.opt("max_speed_runner", c.env.max_speed_runner);
    o.opt("accel_delta", c.env.accel_delta);
    o.opt("turn_delta", c.env.turn_delta);
    o.opt("seed", c.env.seed);
    o.finish();
  }
  if (const json* e = root.section("engine")) {
    StrictObj o(*e, "engine");
    o.opt("num_envs", c.engine.num_envs);
    o.opt("worker_count", c.engine.worker_count);
    o.opt("deterministic", c.engine.deterministic);
    o.finish();
  }
  if (const json* e = root.section("trainer")) {
    StrictObj o(*e, "trainer");
    o.opt("algorithm", c.trainer.algorithm);
    if (c.trainer.algorithm != "a2c" && c.trainer.algorithm != "ppo") {
      raise(Errc::parse_error, "trainer.algorithm must be \"a2c\" or \"ppo\", got \"" + c.trainer.algorithm + "\"");
    }
    o.opt("gamma", c.trainer.gamma);
    o.opt("rollout_horizon", c.trainer.rollout_horizon);
    o.opt("learning_rate", c.trainer.learning_rate);
    o.opt("value_coef", c.trainer.value_coef);
    o.opt("entropy_coef", c.trainer.entropy_coef);
    o.opt("ppo_clip", c.trainer.ppo_clip);
    o.opt("ppo_epochs", c.trainer.ppo_epochs);
    o.opt("max_grad_norm", c.trainer.max_grad_norm);
    o.opt("iterations", c.trainer.iterations);
    o.opt("seed", c.trainer.seed);
    o.opt("hidden_sizes", c.trainer.hidden_sizes);
    o.opt("checkpoint_every", c.trainer.checkpoint_every);
    o.finish();
  }
  if (const json* e = root.section("run")) {
    StrictObj o(*e, "run");
    o.opt("mode", c.run.mode);
    o.opt("output_dir", c.run.output_dir);
    o.opt("check_steps", c.run.check_steps);
    o.opt("env_counts", c.run.env_counts);
    o.opt("agent_counts", c.run.agent_counts);
    o.opt("bench_obs_modes", c.run.bench_obs_modes);
    o.opt("bench_budget_ms", c.run.bench_budget_ms);
    o.opt("bench_reps", c.run.bench_reps);
    o.opt("dump_trajectory", c.run.dump_trajectory);
    o.opt("dump_arrays", c.run.dump_arrays);
    o.opt("resume_from", c.run.resume_from);
    o.finish();
  }
  root.finish();
  c.engine.num_agents = c.env.num_taggers + c.env.num_runners;
  return c;
}

// config_to_json (harness.cpp:160-206): same keys, same value types, so the
// nlohmann (3.11.3, as the reference) dump and its FNV-1a hash are identical.
json config_to_json(const RunConfig& c) {
  json j;
  j["env"] = {{"variant", variant_name(c.env.variant)},
              {"grid_size", c.env.grid_size},
              {"world_length", c.env.world_length},
              {"num_taggers", c.env.num_taggers},
              {"num_runners", c.env.num_runners},
              {"episode_length", c.env.episode_length},
              {"tag_radius", c.env.tag_radius},
              {"obs_mode", obs_name(c.env.obs_mode)},
              {"k_nearest", c.env.k_nearest},
              {"tag_reward", c.env.tag_reward},
              {"tagged_penalty", c.env.tagged_penalty},
              {"max_speed_tagger", c.env.max_speed_tagger},
              {"max_speed_runner", c.env.max_speed_runner},
              {"accel_delta", c.env.accel_delta},
              {"turn_delta", c.env.turn_delta},
              {"seed", c.env.seed}};
  j["engine"] = {{"num_envs", c.engine.num_envs},
                 {"worker_count", c.engine.worker_count},
                 {"deterministic", c.engine.deterministic}};
  j["trainer"] = {{"algorithm", c.trainer.algorithm},
                  {"gamma", c.trainer.gamma},
                  {"rollout_horizon", c.trainer.rollout_horizon},
                  {"learning_rate", c.trainer.learning_rate},
                  {"value_coef", c.trainer.value_coef},
                  {"entropy_coef", c.trainer.entropy_coef},
                  {"ppo_clip", c.trainer.ppo_clip},
                  {"ppo_epochs", c.trainer.ppo_epochs},
                  {"max_grad_norm", c.trainer.max_grad_norm},
                  {"iterations", c.trainer.iterations},
                  {"seed", c.trainer.seed},
                  {"hidden_sizes", c.trainer.hidden_sizes},
                  {"checkpoint_every", c.trainer.checkpoint_every}};
  j["run"] = {{"mode", c.run.mode},
              {"output_dir", c.run.output_dir},
              {"check_steps", c.run.check_steps},
              {"env_counts", c.run.env_counts},
              {"agent_counts", c.run.agent_counts},
              {"bench_obs_modes", c.run.bench_obs_modes},
              {"bench_budget_ms", c.run.bench_budget_ms},
              {"bench_reps", c.run.bench_reps},
              {"dump_trajectory", c.run.dump_trajectory},
              {"dump_arrays", c.run.dump_arrays},
              {"resume_from", c.run.resume_from}};
  return j;
}

std::string config_hash(const RunConfig& c) {  // harness.cpp:208-215,317-322
  uint64_t h = 1469598103934665603ULL;
  for (unsigned char ch : config_to_json(c).dump()) {
    h ^= ch;
    h *= 1099511628211ULL;
  }
  char buf[17];
  std::snprintf(buf, sizeof buf, "%016llx", static_cast<unsigned long long>(h));
  return buf;
}

// RunConfig::validate (harness.cpp:324-335) + TrainerConfig::validate
// (trainer.cpp:45-55).
void validate(const RunConfig& c) {
  validate_tag_config(c.env);
  auto tfail = [](const std::string& m) { raise(Errc::invalid_config, "TrainerConfig: " + m); };
  const TrainerCfg& t = c.trainer;
  if (!(t.gamma > 0.0 && t.gamma < 1.0)) tfail("gamma must be in (0, 1)");
  if (t.rollout_horizon < 1) tfail("rollout_horizon must be >= 1");
  if (t.learning_rate <= 0.0) tfail("learning_rate must be > 0");
  if (t.ppo_clip <= 0.0) tfail("ppo_clip must be > 0");
  if (t.ppo_epochs < 1) tfail("ppo_epochs must be >= 1");
  if (t.max_grad_norm <= 0.0) tfail("max_grad_norm must be > 0");
  if (t.iterations < 0) tfail("iterations must be >= 0");
  if (t.hidden_sizes.empty()) tfail("hidden_sizes must not be empty");
  if (c.engine.num_envs < 1) raise(Errc::invalid_config, "engine.num_envs must be >= 1");
  if (c.run.check_steps < 1) raise(Errc::invalid_config, "run.check_steps must be >= 1");
  if (c.run.bench_reps < 1) raise(Errc::invalid_config, "run.bench_reps must be >= 1");
  for (int64_t n : c.run.env_counts) {
    if (n < 1) raise(Errc::invalid_config, "run.env_counts entries must be >= 1");
  }
  for (const std::string& m : c.run.bench_obs_modes) obs_from(m);
}

std::string format_double(double v) {  // harness.cpp:328-332
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

double seconds_since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  const size_t n = v.size();
  return n % 2 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}

int device_sms() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

// ReportMeta (harness.hpp:46-54): cores = the device's SMs, workers = 1
// stream (the device path has no worker pool).
json meta_json(const RunConfig& c, const std::string& mode) {
  return {{"mode", mode},           {"version", kVersion},          {"config_hash", config_hash(c)},
          {"env_seed", c.env.seed}, {"trainer_seed", c.trainer.seed}, {"cores", device_sms()},
          {"workers", 1}};
}

struct Table {  // harness.hpp:57-66, harness.cpp:335-352
  std::map<std::string, std::string> meta;
  std::vector<std::string> columns;
  std::vector<std::vector<std::string>> rows;
  void write_csv(const std::string& path) const {
    std::ofstream os(path, std::ios::trunc);
    if (!os) raise(Errc::io_error, "cannot open for writing: " + path);
    for (const auto& [k, v] : meta) os << "# " << k << "=" << v << "\n";
    for (size_t i = 0; i < columns.size(); ++i) os << (i ? "," : "") << columns[i];
    os << "\n";
    for (const auto& row : rows) {
      for (size_t i = 0; i < row.size(); ++i) os << (i ? "," : "") << row[i];
      os << "\n";
    }
    if (!os) raise(Errc::io_error, "write failed: " + path);
  }
};

void meta_into(const json& m, Table& t) {
  for (auto it = m.begin(); it != m.end(); ++it) {
    t.meta[it.key()] = it->is_string() ? it->get<std::string>() : it->dump();
  }
}

// One wired world on the device (build_workspace, harness.cpp:402-423).
struct World {
  std::unique_ptr<DataStore> store;
  std::unique_ptr<TagPlan> plan;
  std::unique_ptr<ResetManager> resets;
  std::unique_ptr<Rollout> rollout;
  // reference: the plan is the device TagReference twin (twin_kernels.cu).
  // rollout_resets = false: the rollout only samples and steps; the caller
  // compares the stores and then runs resets->auto_reset_on_done() itself
  // (the checker's order, harness.cpp:619-629).
  World(const wdg_tag_config& cfg, int64_t envs, uint64_t sample_seed, bool reference = false,
        bool rollout_resets = true) {
    validate_tag_config(cfg);
    store = std::make_unique<DataStore>(envs, cfg.num_taggers + cfg.num_runners);
    register_tag_arrays(*store, cfg);
    store->lock();
    plan = std::make_unique<TagPlan>(*store, cfg, reference);
    resets = std::make_unique<ResetManager>(*store, true, tag_zero_on_reset(), plan.get());
    rollout = std::make_unique<Rollout>(*store, *plan, rollout_resets ? resets.get() : nullptr, sample_seed);
    if (!rollout_resets) rollout->set_fused(false);
  }
};

// compare_stores (harness.cpp:531-557) on device: the first differing byte of
// an array (min over a grid-stride scan) -> element -> (env, agent, index).
__global__ void first_diff_kernel(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b, int64_t n,
                                  unsigned long long* first) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (a[i] != b[i]) {
      atomicMin(first, static_cast<unsigned long long>(i));
      return;
    }
  }
}

struct Divergence {
  int64_t step = -1;
  std::string array;
  int64_t env = -1, agent = -1, index = -1;
};

std::optional<Divergence> compare_stores(DataStore& a, DataStore& b, int64_t step, unsigned long long* dfirst) {
  static const char* kOrder[] = {kSampledActions, kRewards, kDone, kObservations};
  for (const char* name : kOrder) {
    const int32_t ha = a.handle(name), hb = b.handle(name);
    const ArrayInfo& info = a.info(ha);
    const int64_t n = info.total_elems * element_size(info.spec.kind);
    const unsigned long long none = ~0ull;
    cuda_check(cudaMemcpy(dfirst, &none, sizeof none, cudaMemcpyHostToDevice), "compare init");
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 16);
    first_diff_kernel<<<static_cast<int>(std::max<int64_t>(1, blocks)), 256>>>(
        static_cast<const uint8_t*>(a.device_ptr(ha)), static_cast<const uint8_t*>(b.device_ptr(hb)), n, dfirst);
    cuda_check(cudaGetLastError(), "compare kernel");
    unsigned long long first = none;
    cuda_check(cudaMemcpy(&first, dfirst, sizeof first, cudaMemcpyDeviceToHost), "compare read");
    if (first == none) continue;
    const int64_t elem = element_size(info.spec.kind);
    const int64_t flat_all = static_cast<int64_t>(first) / elem;
    Divergence d;
    d.step = step;
    d.array = name;
    d.env = flat_all / info.env_stride;
    const int64_t flat = flat_all - d.env * info.env_stride;
    d.agent = info.has_agent_axis ? flat / info.agent_stride : -1;
    d.index = info.has_agent_axis ? flat % info.agent_stride : flat;
    return d;
  }
  return std::nullopt;
}

}  // namespace

// ---- session --------------------------------------------------------------
struct Session {
  RunConfig config;
  std::string report_json, summary, config_json, config_hash_str;
  std::unique_ptr<World> world;  // the last check's store, for dump_array

  void write_reports(const Table& t, const std::string& csv) const {
    const std::string& out = config.run.output_dir;
    if (out.empty()) return;
    std::error_code ec;
    std::filesystem::create_directories(out, ec);
    t.write_csv(out + "/" + csv);
    std::ofstream os(out + "/report.json", std::ios::trunc);
    os << report_json;
  }

  // check_consistency (harness.cpp:563-660) on the device: for each variant x
  // obs mode, the fused single-kernel rollout and the unfused path (sample ->
  // run_step -> detect/auto_reset, separate kernels) step in lockstep with
  // the same f64 policy (init_policy(trainer.seed)); stores are compared on
  // device after every step in the reference's causal order.
  // check (check_consistency_single, harness.cpp:562-633), per variant x
  // obs mode, two legs with the same f64 policy init_policy(trainer.seed):
  //  1. reference: the production plan against the device TagReference twin
  //     (an independent brute-force implementation, twin_kernels.cu), each
  //     step sampled from the policy forward of its own store's obs, compared
  //     after the step and BEFORE reset-on-done in the reference's causal
  //     order (sampled_actions, rewards, done, observations), then both reset
  //     — exactly the reference's engine-vs-TagReference flow;
  //  2. fused: the one-kernel RolloutDriver::step against the unfused kernel
  //     sequence (sample -> run_step -> detect/auto_reset), compared after
  //     every step (post-reset).
  // A combo passes when both legs do; the row reports the first divergence.
  bool run_check() {
    validate(config);
    json j;
    j["meta"] = meta_json(config, "check");
    j["combos"] = json::array();
    Table t;
    meta_into(j["meta"], t);
    t.columns = {"variant", "obs_mode", "workers", "steps", "passed", "div_step", "div_array", "div_env",
                 "div_agent", "div_index", "div_leg"};
    std::ostringstream sum;
    bool all = true;
    int n_pass = 0, n = 0;
    unsigned long long* dfirst = nullptr;
    cuda_check(cudaMalloc(&dfirst, sizeof(unsigned long long)), "cudaMalloc(compare)");
    std::vector<std::string> lines;
    for (int32_t variant : {WDG_TAG_DISCRETE, WDG_TAG_CONTINUOUS}) {
      for (int32_t obs : {WDG_OBS_FULL, WDG_OBS_PARTIAL}) {
        wdg_tag_config env = config.env;
        env.variant = variant;
        env.obs_mode = obs;
        validate_tag_config(env);
        const auto t0 = Clock::now();
        const uint64_t seed = config.trainer.seed;
        PolicyDims dims;
        dims.obs_dim = tag_obs_dim(env);
        dims.hidden = config.trainer.hidden_sizes;
        dims.num_categories = variant == WDG_TAG_CONTINUOUS ? 2 : 1;
        dims.num_choices = variant == WDG_TAG_CONTINUOUS ? 3 : 5;
        Policy policy(dims);
        policy.init(config.trainer.seed);
        const int64_t E = config.engine.num_envs;
        // leg 1: production plan vs the device TagReference twin
        std::optional<Divergence> div_ref;
        {
          World engine(env, E, seed, false, false);
          World twin(env, E, seed, true, false);
          engine.rollout->set_policies(&policy, &policy, kPolicyF64);
          twin.rollout->set_policies(&policy, &policy, kPolicyF64);
          div_ref = compare_stores(*engine.store, *twin.store, -1, dfirst);  // registration
          for (int64_t s = 0; s < config.run.check_steps && !div_ref; ++s) {
            engine.rollout->step();  // forward -> sample -> run_step (no reset)
            twin.rollout->step();
            div_ref = compare_stores(*engine.store, *twin.store, s, dfirst);
            engine.resets->auto_reset_on_done();
            twin.resets->auto_reset_on_done();
          }
          engine.rollout->check();
          twin.rollout->check();
        }
        // leg 2: fused vs unfused rollout
        auto fused = std::make_unique<World>(env, E, seed);
        std::optional<Divergence> div_fused;
        {
          World unfused(env, E, seed);
          unfused.rollout->set_fused(false);
          fused->rollout->set_policies(&policy, &policy, kPolicyF64);
          unfused.rollout->set_policies(&policy, &policy, kPolicyF64);
          for (int64_t s = 0; s < config.run.check_steps && !div_fused; ++s) {
            fused->rollout->step();
            unfused.rollout->step();
            div_fused = compare_stores(*fused->store, *unfused.store, s, dfirst);
          }
          fused->rollout->check();
          unfused.rollout->check();
        }
        const double wall_ms = seconds_since(t0) * 1e3;
        const bool passed = !div_ref && !div_fused;
        const std::optional<Divergence>& div = div_ref ? div_ref : div_fused;
        const char* leg = div_ref ? "reference" : (div_fused ? "fused" : "");
        all = all && passed;
        n_pass += passed ? 1 : 0;
        ++n;
        json jc = {{"variant", variant_name(variant)}, {"obs_mode", obs_name(obs)}, {"workers", 1},
                   {"steps", config.run.check_steps}, {"passed", passed}, {"wall_ms", wall_ms}};
        auto leg_json = [](const std::optional<Divergence>& d) {
          json l = {{"passed", !d.has_value()}};
          if (d) l["divergence"] = {{"step", d->step}, {"array", d->array}, {"env", d->env}, {"agent", d->agent},
                                    {"index", d->index}};
          return l;
        };
        jc["legs"] = {{"reference", leg_json(div_ref)}, {"fused", leg_json(div_fused)}};
        const Divergence d = div.value_or(Divergence{});
        if (div) {
          jc["divergence"] = {{"step", d.step}, {"array", d.array}, {"env", d.env}, {"agent", d.agent},
                              {"index", d.index}, {"leg", leg}};
        }
        j["combos"].push_back(jc);
        t.rows.push_back({variant_name(variant), obs_name(obs), "1", std::to_string(config.run.check_steps),
                          passed ? "1" : "0", std::to_string(d.step), div ? d.array : "", std::to_string(d.env),
                          std::to_string(d.agent), std::to_string(d.index), leg});
        std::ostringstream ln;
        ln << "  " << variant_name(variant) << "/" << obs_name(obs) << " workers=1 steps=" << config.run.check_steps
           << " " << (passed ? "pass" : "FAIL");
        if (div) {
          ln << " first divergence (" << leg << "): step=" << d.step << " array=" << d.array << " env=" << d.env
             << " agent=" << d.agent << " index=" << d.index;
        }
        lines.push_back(ln.str());
        fused->rollout->set_policies(nullptr, nullptr, kPolicyF64);
        world = std::move(fused);  // keep the last combo's store (dump_array)
      }
    }
    cudaFree(dfirst);
    j["passed"] = all;
    report_json = j.dump(2);
    sum << "check: " << (all ? "PASS" : "FAIL") << " (" << n_pass << "/" << n << " combos)\n";
    for (const std::string& l : lines) sum << l << "\n";
    summary = sum.str();
    write_reports(t, "check.csv");
    return all;
  }

  // measure_rollout_sps (harness.cpp:715-741): calibrate n by doubling from 8
  // until one run takes >= budget/(4 (reps+1)), then bench_reps timed runs of
  // n steps (device-synchronised wall clock), median env-steps/s.
  double measure_sps(const wdg_tag_config& env, int64_t envs) {
    World w(env, envs, env.seed);
    const double budget_s = std::max(config.run.bench_budget_ms, 50.0) / 1e3;
    const double target = budget_s / static_cast<double>(config.run.bench_reps + 1);
    auto timed = [&](int64_t steps) {
      const auto t0 = Clock::now();
      w.rollout->run(steps);
      w.store->synchronize();
      return seconds_since(t0);
    };
    int64_t n = 8;
    double elapsed = 0.0;
    for (;;) {
      elapsed = timed(n);
      if (elapsed >= target / 4 || n >= (int64_t{1} << 22)) break;
      n *= 2;
    }
    if (elapsed < target / 2) {
      n = std::max<int64_t>(n, static_cast<int64_t>(static_cast<double>(n) * target / std::max(elapsed, 1e-9)));
    }
    std::vector<double> sps;
    for (int64_t r = 0; r < config.run.bench_reps; ++r) sps.push_back(static_cast<double>(envs * n) / timed(n));
    w.rollout->check();
    return median(sps);
  }

  // bench_envs (harness.cpp:744-778). iterations_per_sec needs the CPU
  // trainer, which is out of scope on the device path: reported as 0.
  void run_bench_envs() {
    validate(config);
    json j;
    j["meta"] = meta_json(config, "bench-envs");
    j["rows"] = json::array();
    Table t;
    meta_into(j["meta"], t);
    t.columns = {"env_count", "steps_per_sec", "iterations_per_sec"};
    std::ostringstream sum;
    sum << "bench-envs: " << config.run.env_counts.size() << " env counts (cores=" << device_sms()
        << ", workers=1)\n";
    for (int64_t count : config.run.env_counts) {
      const double sps = measure_sps(config.env, count);
      j["rows"].push_back({{"env_count", count}, {"steps_per_sec", sps}, {"iterations_per_sec", 0.0}});
      t.rows.push_back({std::to_string(count), format_double(sps), format_double(0.0)});
      char buf[160];
      std::snprintf(buf, sizeof buf, "  envs=%-6lld steps/s=%-12.0f iters/s=%.2f\n", static_cast<long long>(count),
                    sps, 0.0);
      sum << buf;
    }
    report_json = j.dump(2);
    summary = sum.str();
    write_reports(t, "bench_envs.csv");
  }

  // bench_agents (harness.cpp:815-860): taggers scaled to llround(N T/A)
  // clamped to [1, N-1], K clamped to N-1; per-env step time and the log-log
  // slope per obs mode.
  void run_bench_agents() {
    validate(config);
    for (int64_t c : config.run.agent_counts) {
      if (c < 2) raise(Errc::invalid_config, "run.agent_counts entries must be >= 2");
    }
    json j;
    j["meta"] = meta_json(config, "bench-agents");
    j["rows"] = json::array();
    std::map<std::string, double> slopes;
    Table t;
    meta_into(j["meta"], t);
    t.columns = {"obs_mode", "agent_count", "per_env_step_us"};
    std::ostringstream sum;
    sum << "bench-agents:\n";
    const double frac = static_cast<double>(config.env.num_taggers) /
                        static_cast<double>(config.env.num_taggers + config.env.num_runners);
    struct Row {
      std::string mode;
      int64_t n;
      double us;
    };
    std::vector<Row> rows;
    for (const std::string& mode : config.run.bench_obs_modes) {
      for (int64_t n : config.run.agent_counts) {
        wdg_tag_config env = config.env;
        env.obs_mode = obs_from(mode);
        env.num_taggers = std::clamp<int64_t>(std::llround(frac * static_cast<double>(n)), 1, n - 1);
        env.num_runners = n - env.num_taggers;
        env.k_nearest = std::min<int64_t>(config.env.k_nearest, n - 1);
        const double sps = measure_sps(env, config.engine.num_envs);
        rows.push_back({mode, n, 1e6 * static_cast<double>(config.engine.num_envs) / sps});
      }
      double sx = 0, sy = 0, sxx = 0, sxy = 0;
      int64_t m = 0;
      for (const Row& r : rows) {
        if (r.mode != mode) continue;
        const double lx = std::log(static_cast<double>(r.n)), ly = std::log(r.us);
        sx += lx;
        sy += ly;
        sxx += lx * lx;
        sxy += lx * ly;
        ++m;
      }
      slopes[mode] = (static_cast<double>(m) * sxy - sx * sy) / (static_cast<double>(m) * sxx - sx * sx);
    }
    for (const Row& r : rows) {
      j["rows"].push_back({{"obs_mode", r.mode}, {"agent_count", r.n}, {"per_env_step_us", r.us}});
      t.rows.push_back({r.mode, std::to_string(r.n), format_double(r.us)});
      char buf[120];
      std::snprintf(buf, sizeof buf, "  %-8s N=%-6lld per-env step=%.2f us\n", r.mode.c_str(),
                    static_cast<long long>(r.n), r.us);
      sum << buf;
    }
    j["slopes"] = slopes;
    for (const auto& [mode, slope] : slopes) {
      t.meta["slope_" + mode] = format_double(slope);
      sum << "  log-log slope (" << mode << ") = " << format_double(slope) << "\n";
    }
    report_json = j.dump(2);
    summary = sum.str();
    write_reports(t, "bench_agents.csv");
  }

  // dump_array_csv (harness.cpp:1067-1097) of the kept store, or of a fresh
  // episode-0 store when no run kept one (c_api.cpp:236-251).
  void dump_array(const std::string& name, const std::string& path) {
    if (!world) world = std::make_unique<World>(config.env, config.engine.num_envs, config.env.seed);
    DataStore& s = *world->store;
    const int32_t h = s.handle(name);
    const ArrayInfo& info = s.info(h);
    const int64_t E = s.num_envs(), stride = info.env_stride;
    std::vector<uint8_t> buf(static_cast<size_t>(E * stride * element_size(info.spec.kind)));
    s.pull(h, 0, E, buf.data(), static_cast<int64_t>(buf.size()));
    std::ofstream os(path, std::ios::trunc);
    if (!os) raise(Errc::io_error, "cannot open for writing: " + path);
    os << "env";
    for (int64_t i = 0; i < stride; ++i) os << ",v" << i;
    os << "\n";
    for (int64_t e = 0; e < E; ++e) {
      os << e;
      for (int64_t i = 0; i < stride; ++i) {
        const int64_t k = e * stride + i;
        if (info.spec.kind == WDG_REAL32) {
          os << "," << format_double(reinterpret_cast<const float*>(buf.data())[k]);
        } else if (info.spec.kind == WDG_INT32) {
          os << "," << reinterpret_cast<const int32_t*>(buf.data())[k];
        } else {
          os << "," << static_cast<int>(buf[static_cast<size_t>(k)]);
        }
      }
      os << "\n";
    }
  }
};

Session* session_open(const std::string& text) {
  auto s = std::make_unique<Session>();
  s->config = parse_config(text);
  validate(s->config);
  return s.release();
}
const char* session_config_json(Session* s) {
  s->config_json = config_to_json(s->config).dump(2);
  return s->config_json.c_str();
}
const char* session_config_hash(Session* s) {
  s->config_hash_str = config_hash(s->config);
  return s->config_hash_str.c_str();
}
void session_set_seed(Session* s, uint64_t seed) {
  s->config.env.seed = seed;
  s->config.trainer.seed = seed;
}
void session_set_workers(Session* s, int32_t w) { s->config.engine.worker_count = w; }
void session_set_output_dir(Session* s, const std::string& d) { s->config.run.output_dir = d; }
bool session_run_check(Session* s) { return s->run_check(); }
void session_run_bench_envs(Session* s) { s->run_bench_envs(); }
void session_run_bench_agents(Session* s) { s->run_bench_agents(); }
const char* session_report_json(Session* s) { return s->report_json.empty() ? nullptr : s->report_json.c_str(); }
const char* session_summary(Session* s) { return s->summary.empty() ? nullptr : s->summary.c_str(); }
void session_dump_array(Session* s, const std::string& name, const std::string& path) { s->dump_array(name, path); }
void session_close(Session* s) { delete s; }

#else  // !WDG_HAVE_JSON: built without nlohmann/json — every session call fails loudly
struct Session {};
[[noreturn]] static void no_json() { raise(Errc::state_error, "session API built without nlohmann/json"); }
Session* session_open(const std::string&) { no_json(); }
const char* session_config_json(Session*) { no_json(); }
const char* session_config_hash(Session*) { no_json(); }
void session_set_seed(Session*, uint64_t) { no_json(); }
void session_set_workers(Session*, int32_t) { no_json(); }
void session_set_output_dir(Session*, const std::string&) { no_json(); }
bool session_run_check(Session*) { no_json(); }
void session_run_bench_envs(Session*) { no_json(); }
void session_run_bench_agents(Session*) { no_json(); }
const char* session_report_json(Session*) { no_json(); }
const char* session_summary(Session*) { no_json(); }
void session_dump_array(Session*, const std::string&, const std::string&) { no_json(); }
void session_close(Session*) {}
#endif

}  // namespace wdg
