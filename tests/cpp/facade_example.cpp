// Compile-checked example of the reference-side C++ integration through
// include/warp_b200.hpp (tests/test_abi.py builds and links it; runs it on a
// GPU in tests/test_parity_gpu.py::test_cpp_facade_example).
#include <cstdio>

#include "warp_b200.hpp"

int main() {
  using namespace warp_b200;
  TagConfig cfg;
  cfg.num_taggers = 20;
  cfg.num_runners = 80;
  cfg.obs_mode = WDG_OBS_PARTIAL;
  cfg.grid_size = 10;
  cfg.episode_length = 25;
  try {
    DataStore store(16, cfg.num_agents());           // build_workspace (harness.cpp:402-423)
    register_tag_arrays(store, cfg);
    store.lock();
    TagPlan plan(store, cfg);
    ResetManager resets(store, true, tag_zero_on_reset(), &plan);
    RolloutDriver driver(store, plan, &resets, cfg.seed);
    driver.run(40);                                  // RolloutDriver::run (harness.cpp:492-494)
    driver.check_errors();
    const std::vector<double> st = driver.stats();
    const std::vector<float> obs = store.pull<float>(kObservations, 0, 1);
    std::printf("episodes=%.0f tag_events=%.0f env_steps=%.0f obs[0]=%g\n", st[WDG_STAT_EPISODES],
                st[WDG_STAT_TAG_EVENTS], st[WDG_STAT_ENV_STEPS], obs[0]);
    // The same driver stepped by device policies (RolloutDriver with
    // tag_policy_map, harness.cpp:395-399,428-476).
    PolicyDims d;
    d.obs_dim = 4 * cfg.k_nearest + 3;
    d.num_choices = 5;
    Policy tagger(d, 1), runner(d, 2);
    driver.set_policies(&tagger, &runner, PolicyPrecision::BF16);
    driver.run(10);
    driver.check_errors();
    const std::vector<double> st2 = driver.stats();
    std::printf("policy rollout: env_steps=%.0f\n", st2[WDG_STAT_ENV_STEPS]);
    // The TagReference twin (tag_env.cpp:505-595) on its own store, stepped
    // with serial launches: same seeds -> the same positions as the fused plan.
    DataStore ref_store(16, cfg.num_agents());
    register_tag_arrays(ref_store, cfg);
    ref_store.lock();
    TagPlan twin(ref_store, cfg, TagPlan::Reference{});
    ResetManager ref_resets(ref_store, true, tag_zero_on_reset(), &twin);
    RolloutDriver ref_driver(ref_store, twin, &ref_resets, cfg.seed);
    ref_driver.set_overlap(false);
    DataStore cmp_store(16, cfg.num_agents());
    register_tag_arrays(cmp_store, cfg);
    cmp_store.lock();
    TagPlan fused(cmp_store, cfg);
    ResetManager cmp_resets(cmp_store, true, tag_zero_on_reset(), &fused);
    RolloutDriver cmp_driver(cmp_store, fused, &cmp_resets, cfg.seed);
    ref_driver.run(30);
    cmp_driver.run(30);
    ref_driver.check_errors();
    cmp_driver.check_errors();
    const bool twin_equal = ref_store.pull<int32_t>(kLocX) == cmp_store.pull<int32_t>(kLocX) &&
                            ref_store.pull<float>(kObservations) == cmp_store.pull<float>(kObservations);
    std::printf("twin vs fused after 30 steps: %s\n", twin_equal ? "equal" : "DIFFERENT");
    return (st[WDG_STAT_ENV_STEPS] == 16 * 40 && st2[WDG_STAT_ENV_STEPS] == 16 * 50 && twin_equal) ? 0 : 1;
  } catch (const Error& e) {
    std::fprintf(stderr, "error %d: %s\n", static_cast<int>(e.code()), e.what());
    return 2;
  }
}
