/* wdg_b200.h — C ABI of the B200-native WarpDrive Tag hot path.
 *
 * Drop-in boundary for the reference's env-step path (sample -> step ->
 * reset-on-done over a named-array store). Every entry point below names the
 * reference interface it replaces (paths relative to the reference tree,
 * proj/...). Plain pointers and sizes only; no C++ or torch types cross this
 * boundary. Errors follow the reference C ABI convention (proj/src/c_api.cpp:
 * 21-58): a status code whose numbering is identical to `wd_status`
 * (proj/include/warp/warp_c.h:22-38) plus a thread-local message returned by
 * wdg_last_error(). No exception ever crosses the ABI.
 *
 * Memory model: every array lives in device memory (HBM) and is updated in
 * place by the kernels. Host code moves data only through explicit push/pull
 * (the reference's typed host views alias host memory, data_store.hpp:78-89;
 * on a discrete GPU they become copies). Device pointers (wdg_store_device_ptr)
 * use the reference's dense row-major layout [env, agent, feature...]
 * (SPEC.md:94), so a consumer reads them exactly like the CPU store.
 *
 * Threading: like the reference (warp_c.h:5-7), objects are not synchronized;
 * use one store and its dependents from one host thread. All device work of a
 * store is issued on the store's stream (wdg_store_set_stream).
 */
#ifndef WDG_B200_H
#define WDG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#ifndef WDG_API
#define WDG_API __attribute__((visibility("default")))
#endif

/* Status codes: value-identical to wd_status (proj/include/warp/warp_c.h:22-38)
 * and to warp::Errc (proj/include/warp/common.hpp:13-28). */
typedef int32_t wdg_status;
enum {
  WDG_OK = 0,
  WDG_ERR_INVALID_ARGUMENT = 1,
  WDG_ERR_DUPLICATE_NAME = 2,
  WDG_ERR_SHAPE_MISMATCH = 3,
  WDG_ERR_STORE_LOCKED = 4,
  WDG_ERR_MISSING_PLACEHOLDER = 5,
  WDG_ERR_UNKNOWN_NAME = 6,
  WDG_ERR_INDEX_OUT_OF_RANGE = 7,
  WDG_ERR_INVALID_CONFIG = 8,
  WDG_ERR_STEP_FAILURE = 9,
  WDG_ERR_NON_FINITE = 10,
  WDG_ERR_PARSE = 11,
  WDG_ERR_IO = 12,
  WDG_ERR_STATE = 13,
  WDG_ERR_UNKNOWN = 14,
  /* Device-side failure (CUDA error / no device). Has no reference twin; the
   * reference cannot fail this way. */
  WDG_ERR_CUDA = 15
};

/* ElementKind (proj/include/warp/data_store.hpp:14). */
enum { WDG_REAL32 = 0, WDG_INT32 = 1, WDG_BOOL8 = 2 };

/* TagVariant / ObsMode (proj/include/warp/tag_env.hpp:26-27). */
enum { WDG_TAG_DISCRETE = 0, WDG_TAG_CONTINUOUS = 1 };
enum { WDG_OBS_FULL = 0, WDG_OBS_PARTIAL = 1 };

/* TagConfig (proj/include/warp/tag_env.hpp:29-45); field meaning, units and
 * defaults identical. */
typedef struct wdg_tag_config {
  int32_t variant;
  int32_t obs_mode;
  int64_t grid_size;
  double world_length;
  int64_t num_taggers;
  int64_t num_runners;
  int64_t episode_length;
  double tag_radius;
  int64_t k_nearest;
  double tag_reward;
  double tagged_penalty;
  double max_speed_tagger;
  double max_speed_runner;
  double accel_delta;
  double turn_delta;
  uint64_t seed;
} wdg_tag_config;

#define WDG_MAX_NAME 64
#define WDG_MAX_DIMS 8

/* ArrayInfo (proj/include/warp/data_store.hpp:42-48) flattened for C. */
typedef struct wdg_array_info {
  char name[WDG_MAX_NAME];
  int32_t kind;
  int32_t ndim;
  int64_t shape[WDG_MAX_DIMS];
  int64_t total_elems;
  int64_t env_stride;
  int64_t agent_stride;
  int32_t has_agent_axis;
  int32_t snapshot_on_reset;
} wdg_array_info;

/* Episode statistics accumulated on device by the fused rollout step, the
 * EpisodeTracker contract (proj/src/trainer.cpp:221-258) reduced to sums so it
 * can be all-reduced across GPUs. Index meaning of the double[8] vector. */
enum {
  WDG_STAT_EPISODES = 0,        /* completed episodes (envs that hit done)   */
  WDG_STAT_TAGGER_RETURN = 1,   /* sum over completed episodes of the summed
                                   tagger rewards of that episode            */
  WDG_STAT_RUNNER_RETURN = 2,   /* same for runners                          */
  WDG_STAT_TAG_EVENTS = 3,      /* tag events (runner deactivations)         */
  WDG_STAT_ENV_STEPS = 4,       /* env-steps executed                        */
  WDG_STAT_COUNT = 8
};

/* ---- library ---------------------------------------------------------- */
WDG_API const char* wdg_version(void);                 /* warp_c.h:43 */
WDG_API const char* wdg_status_name(wdg_status status); /* warp_c.h:46 */
WDG_API const char* wdg_last_error(void);               /* warp_c.h:49 */
WDG_API wdg_status wdg_device_count(int32_t* out);
/* Synchronous device -> host copy of `bytes` (inspection of device outputs
 * such as wdg_rollout_policy_outputs). */
WDG_API wdg_status wdg_copy_to_host(const void* device_src, void* host_dst, int64_t bytes);
WDG_API wdg_status wdg_set_device(int32_t device);
/* Test-only fault injection, detail::FaultHooks::tag_radius_bias
 * (proj/include/warp/tag_env.hpp:155-158): biases the device step kernels'
 * tag radius so the parity harness can be mutation-tested. */
WDG_API void wdg_set_fault_tag_radius_bias(float bias);

/* ---- DataStore (proj/include/warp/data_store.hpp:54-113) --------------- */
typedef struct wdg_store wdg_store;
/* DataStore(num_envs, num_agents)  (data_store.hpp:56, data_store.cpp:7-12) */
WDG_API wdg_status wdg_store_create(int64_t num_envs, int64_t num_agents, wdg_store** out);
WDG_API void wdg_store_destroy(wdg_store* store);
/* Global id of local env 0. Every RNG key uses the global env id so a sharded
 * run is bit-identical to one big store. Set before
 * wdg_register_tag_arrays. Default 0. */
WDG_API wdg_status wdg_store_set_env_offset(wdg_store* store, int64_t global_env_offset);
/* cudaStream_t on which all of the store's device work is issued (0 = the
 * legacy default stream). */
WDG_API wdg_status wdg_store_set_stream(wdg_store* store, void* cuda_stream);
/* register_array(spec, initial) x3 kinds + zero-fill (data_store.hpp:62-66,
 * data_store.cpp:14-83). host_initial == NULL registers zeros. */
WDG_API wdg_status wdg_store_register_array(wdg_store* store, const char* name,
                                            const int64_t* shape, int32_t ndim, int32_t kind,
                                            int32_t snapshot_on_reset, const void* host_initial,
                                            int64_t initial_count, int32_t* out_handle);
/* lock() (data_store.cpp:85-93). */
WDG_API wdg_status wdg_store_lock(wdg_store* store);
WDG_API wdg_status wdg_store_locked(const wdg_store* store, int32_t* out);
WDG_API wdg_status wdg_store_num_envs(const wdg_store* store, int64_t* out);
WDG_API wdg_status wdg_store_num_agents(const wdg_store* store, int64_t* out);
/* handle(name) / info(h) / array_names() (data_store.hpp:71-75). */
WDG_API wdg_status wdg_store_handle(const wdg_store* store, const char* name, int32_t* out);
WDG_API wdg_status wdg_store_num_arrays(const wdg_store* store, int32_t* out);
WDG_API wdg_status wdg_store_info(const wdg_store* store, int32_t handle, wdg_array_info* out);
/* Host<->device copies of env rows [env_begin, env_begin+env_count) of one
 * array, dense layout; `bytes` must equal env_count * env_row_bytes. Replaces
 * the aliasing host views f32/i32/u8 and env_slice_* / env_row_bytes
 * (data_store.hpp:78-94). Synchronous with respect to the store's stream. */
WDG_API wdg_status wdg_store_push(wdg_store* store, int32_t handle, int64_t env_begin,
                                  int64_t env_count, const void* host, int64_t bytes);
WDG_API wdg_status wdg_store_pull(const wdg_store* store, int32_t handle, int64_t env_begin,
                                  int64_t env_count, void* host, int64_t bytes);
/* Device address of the whole array (dense row-major, env outermost). */
WDG_API wdg_status wdg_store_device_ptr(wdg_store* store, int32_t handle, void** out);
/* restore_snapshot(ids) (data_store.hpp:98, data_store.cpp:207-217). */
WDG_API wdg_status wdg_store_restore_snapshot(wdg_store* store, const int64_t* env_ids,
                                              int64_t count);
WDG_API wdg_status wdg_store_synchronize(wdg_store* store);

/* ---- Tag environment (proj/include/warp/tag_env.hpp) ------------------ */
/* TagConfig{} defaults (tag_env.hpp:29-45). */
WDG_API wdg_status wdg_tag_config_init(wdg_tag_config* cfg);
/* TagConfig::validate (tag_env.cpp:20-40) -> WDG_ERR_INVALID_CONFIG. */
WDG_API wdg_status wdg_tag_config_validate(const wdg_tag_config* cfg);
WDG_API int64_t wdg_tag_obs_dim(const wdg_tag_config* cfg);
/* register_tag_arrays(store, cfg) (tag_env.hpp:112, tag_env.cpp:280-341):
 * registers the same 12/14 arrays with the same names, shapes, kinds and
 * snapshot flags, initialised on device to the episode-0 state. */
WDG_API wdg_status wdg_register_tag_arrays(wdg_store* store, const wdg_tag_config* cfg);
/* tag_zero_on_reset() (tag_env.cpp:343-346); names are static strings. */
WDG_API wdg_status wdg_tag_zero_on_reset(const char** names, int32_t capacity, int32_t* count);

typedef struct wdg_tag_plan wdg_tag_plan;
/* build_tag_plan(store, cfg) (tag_env.cpp:363-480). The plan must not outlive
 * the store (same ownership rule as TagContext, tag_env.cpp:351-361). */
WDG_API wdg_status wdg_build_tag_plan(wdg_store* store, const wdg_tag_config* cfg,
                                      wdg_tag_plan** out);
/* TagReference(store, cfg) (tag_env.cpp:505-595) on device: a plan whose
 * run_step and reset reinit run an independent brute-force twin of the step
 * (global memory only, brute-force K-NN and resolve, any K < A) instead of
 * the production kernel — the second store of the consistency check
 * (harness.cpp:562-633). It recomputes the store's episode-0 observations
 * itself. Not usable with the fused rollout (RolloutDriver falls back to the
 * unfused sample -> run_step -> auto_reset sequence). */
WDG_API wdg_status wdg_build_tag_reference(wdg_store* store, const wdg_tag_config* cfg,
                                           wdg_tag_plan** out);
WDG_API void wdg_tag_plan_destroy(wdg_tag_plan* plan);
/* StepEngine::run_step(plan, store, step) (step_engine.cpp:122-138) for the
 * Tag plan: move -> resolve_tags -> observe_reward, one CTA per env. */
WDG_API wdg_status wdg_run_step(wdg_tag_plan* plan, int64_t step_index);
/* Kernel geometry chosen for this plan (diagnostics / bench reporting). */
WDG_API wdg_status wdg_tag_plan_geometry(const wdg_tag_plan* plan, int32_t* threads_per_cta,
                                         int32_t* envs_per_cta, int32_t* grid_ctas,
                                         int32_t* uses_grid, int32_t* smem_bytes);

/* ---- Sampler (proj/include/warp/sampler.hpp:35-36, proj/src/sampler.cpp) - */
/* sample_actions(store, logits, C, V, step, seed). `logits` is a DEVICE
 * pointer to f64 [E, A, C, V]; logits_count must equal E*A*C*V
 * (shape_mismatch otherwise). Non-finite logits -> WDG_ERR_NON_FINITE and the
 * action array is left untouched, as in the reference. */
WDG_API wdg_status wdg_sample_actions(wdg_store* store, const double* logits, int64_t logits_count,
                                      int64_t num_categories, int64_t num_choices, int64_t step,
                                      uint64_t seed);

/* ---- ResetManager (proj/include/warp/reset_manager.hpp) ---------------- */
typedef struct wdg_resets wdg_resets;
/* ResetManager(store, ResetPolicy{auto_reset, zero_on_reset, reinitialize})
 * (reset_manager.cpp:5-16). reinitialize = make_tag_reinit(plan) when
 * `reinit_plan` is non-NULL (tag_env.cpp:482-500), none otherwise. */
WDG_API wdg_status wdg_reset_manager_create(wdg_store* store, int32_t auto_reset,
                                            const char* const* zero_on_reset, int32_t n_zero,
                                            wdg_tag_plan* reinit_plan, wdg_resets** out);
WDG_API void wdg_reset_manager_destroy(wdg_resets* resets);
/* detect_done(store) -> ids (reset_manager.cpp:20-27). Host list; syncs. */
WDG_API wdg_status wdg_detect_done(wdg_resets* resets, int64_t* env_ids, int64_t capacity,
                                   int64_t* count);
/* auto_reset(store, ids) (reset_manager.cpp:29-44). */
WDG_API wdg_status wdg_auto_reset(wdg_resets* resets, const int64_t* env_ids, int64_t count);
/* detect_done + auto_reset fused on device: no host list, no sync. */
WDG_API wdg_status wdg_auto_reset_on_done(wdg_resets* resets);
/* episodes_started(env) (reset_manager.hpp:34, reset_manager.cpp:46-51). */
WDG_API wdg_status wdg_episodes_started(const wdg_resets* resets, int64_t env_id, int64_t* out);

/* ---- Rollout driver (RolloutDriver, proj/src/harness.cpp:428-505) ------ */
typedef struct wdg_rollout wdg_rollout;
/* One env-step = sample(t, sample_seed) -> run_step(t) -> [stats] ->
 * reset-on-done, t = 0,1,2,... (harness.cpp:478-490). With `fused` (default)
 * the whole step is ONE kernel launch; unfused issues sampler, step and reset
 * kernels separately. Logits default to zeros (uniform policy,
 * harness.cpp:439,446-447). */
WDG_API wdg_status wdg_rollout_create(wdg_store* store, wdg_tag_plan* plan, wdg_resets* resets,
                                      uint64_t sample_seed, wdg_rollout** out);
WDG_API void wdg_rollout_destroy(wdg_rollout* rollout);
/* Device f64 logits [E,A,C,V] to sample from (NULL -> internal zeros). */
WDG_API wdg_status wdg_rollout_set_logits(wdg_rollout* rollout, const double* logits,
                                          int64_t logits_count);
WDG_API wdg_status wdg_rollout_set_fused(wdg_rollout* rollout, int32_t fused);
/* Overlap consecutive fused launches (programmatic dependent launch with
 * per-env sequence flags, default on); 0 = each launch waits for the previous
 * one to finish. Results are identical either way. */
WDG_API wdg_status wdg_rollout_set_overlap(wdg_rollout* rollout, int32_t enabled);
/* Plan tuning overrides for A/B measurements and path-pinning tests: how a
 * plan maps the step onto the GPU, never what it computes. Keys:
 * stage_rows, brute_max, threads_per_env_max, cont_cell_div, disc_grid_cells,
 * stage_obs, bulk_in, l2_prefetch, pdl_mode, multistep, cont_keys,
 * packed_warps_max; value < 0 restores
 * the plan's own choice; key "reset" restores all. Read when a plan is built
 * (geometry) or a rollout launches (pdl_mode, multistep). */
WDG_API wdg_status wdg_set_tuning(const char* key, int64_t value);
/* Use CUDA-graph replay for wdg_rollout_run (default on). */
WDG_API wdg_status wdg_rollout_set_graphs(wdg_rollout* rollout, int32_t enabled);
WDG_API wdg_status wdg_rollout_step(wdg_rollout* rollout);
/* One step driven from HOST buffers (the drop-in host integration; replaces
 * the reference learner's host loop sample_actions(host logits) -> run_step ->
 * post_step reads -> auto_reset, trainer.cpp:357-397 / harness.cpp:478-490):
 * the step's f64 logits [E,A,C,V] go host->device, the fused step runs, and
 * the step's rewards [E,A] f32 and done [E] u8 come back device->host as they
 * were BEFORE reset-on-done (the post_step hook's view, trainer.cpp:382-394),
 * so a finished env reports done = 1 and its terminal rewards. The step is
 * pipelined over env chunks (H2D, kernel and D2H of different chunks overlap).
 * Asynchronous: the host buffers are read / written until
 * wdg_store_synchronize returns. Host buffers should be pinned;
 * host_rewards / host_done may be NULL. */
WDG_API wdg_status wdg_rollout_step_host(wdg_rollout* rollout, const double* host_logits,
                                         int64_t logits_count, float* host_rewards,
                                         uint8_t* host_done);
/* The same step, also returning the observations [E,A,D] f32 AFTER the step
 * and its reset-on-done: what the next policy_forward reads
 * (trainer.cpp:358-360). host_obs may be NULL (obs_count is then ignored). */
WDG_API wdg_status wdg_rollout_step_host_obs(wdg_rollout* rollout, const double* host_logits,
                                             int64_t logits_count, float* host_rewards,
                                             uint8_t* host_done, float* host_obs,
                                             int64_t obs_count);
/* Env chunks of the pipelined host step (0 = automatic: ~8 MB of logits per
 * chunk, at most 16). */
WDG_API wdg_status wdg_rollout_set_host_chunks(wdg_rollout* rollout, int32_t chunks);
WDG_API wdg_status wdg_rollout_run(wdg_rollout* rollout, int64_t steps);
WDG_API wdg_status wdg_rollout_next_step(const wdg_rollout* rollout, int64_t* out);
/* Kernel launches issued so far (step kernels, policy forwards, graph nodes). */
WDG_API wdg_status wdg_rollout_launches(const wdg_rollout* rollout, int64_t* out);
/* Synchronise and surface sticky device errors (non-finite logits seen by the
 * fused sampler) as WDG_ERR_NON_FINITE. */
WDG_API wdg_status wdg_rollout_check(wdg_rollout* rollout);
/* Pull / zero / locate the device double[WDG_STAT_COUNT] statistics vector. */
WDG_API wdg_status wdg_rollout_stats(wdg_rollout* rollout, double* out, int32_t count);
WDG_API wdg_status wdg_rollout_reset_stats(wdg_rollout* rollout);
WDG_API wdg_status wdg_rollout_stats_device_ptr(wdg_rollout* rollout, double** out);
/* Reduce the per-env tracker slots into a caller-owned device double[8] on the
 * store's stream (e.g. a tensor that is then all-reduced over NCCL). */
WDG_API wdg_status wdg_rollout_reduce_stats_into(wdg_rollout* rollout, double* device_out);

/* ---- Multi-GPU: the episode-statistics all-reduce ------
 * Envs shard across GPUs as contiguous blocks with global env ids
 * (wdg_store_set_env_offset); the only collective is the all-reduce of the
 * EpisodeTracker sums (trainer.cpp:221-258), exact for integer-valued
 * rewards. libnccl.so.2 is resolved at run time (the copy already loaded in
 * the process, e.g. PyTorch's, else the system one). */
typedef struct wdg_comm wdg_comm;
WDG_API wdg_status wdg_nccl_version(int32_t* out);
/* ncclGetUniqueId into a 128-byte buffer (rank 0; share it with the others). */
WDG_API wdg_status wdg_comm_unique_id(uint8_t* out, int64_t bytes);
/* ncclCommInitRank: collective over all `world` ranks, one GPU each (the
 * caller's current device). */
WDG_API wdg_status wdg_comm_init(int32_t world, int32_t rank, const uint8_t* id, int64_t bytes,
                                 wdg_comm** out);
/* Wrap an existing ncclComm_t (not destroyed by wdg_comm_destroy). */
WDG_API wdg_status wdg_comm_wrap(void* nccl_comm, wdg_comm** out);
WDG_API void wdg_comm_destroy(wdg_comm* comm);
WDG_API wdg_status wdg_comm_info(const wdg_comm* comm, int32_t* world, int32_t* rank);
/* Reduce this shard's tracker slots into device_out (device double
 * [WDG_STAT_COUNT]) and ncclAllReduce(sum) it in place over `comm`, on the
 * store's stream; every rank then holds the global statistics. */
WDG_API wdg_status wdg_stats_allreduce(wdg_rollout* rollout, wdg_comm* comm, double* device_out);

/* ---- Policy network (proj/include/warp/policy_model.hpp) --------------- */
/* The rollout's forward_policies (harness.cpp:445-476) on device: the
 * reference MLP (tanh hidden layers, a linear logit head per category, a
 * scalar value head) evaluated on the observation array in HBM. */
typedef struct wdg_policy wdg_policy;
/* Precision of the device forward. F64: the reference arithmetic (serial
 * mul-then-add per output, policy_model.cpp:24-31, y = b + acc, tanh); equal
 * to the CPU forward except where CUDA and glibc tanh round differently. BF16:
 * bf16 operands with f32 accumulation on the tcgen05 tensor cores. */
#define WDG_POLICY_F64 0
#define WDG_POLICY_BF16 1
/* PolicyDims (policy_model.hpp:20-28); check_dims (policy_model.cpp:14-21). */
WDG_API wdg_status wdg_policy_create(int64_t obs_dim, const int64_t* hidden, int32_t num_hidden,
                                     int64_t num_categories, int64_t num_choices, wdg_policy** out);
WDG_API void wdg_policy_destroy(wdg_policy* policy);
/* init_policy(seed, dims) (policy_model.cpp:107-144): Xavier-uniform from the
 * counter RNG, zero biases; bit-identical to the reference. */
WDG_API wdg_status wdg_policy_init(wdg_policy* policy, uint64_t seed);
/* PolicyParams::param_count / for_each_param canonical order
 * (policy_model.hpp:42-46, policy_model.cpp:35-56): hidden (W[out,in], b) per
 * layer, head_w, head_b, value_w, value_b. */
WDG_API wdg_status wdg_policy_param_count(const wdg_policy* policy, int64_t* out);
WDG_API wdg_status wdg_policy_set_params(wdg_policy* policy, const double* host_params, int64_t count);
WDG_API wdg_status wdg_policy_get_params(const wdg_policy* policy, double* host_params, int64_t count);
/* forward / forward_parallel (policy_model.cpp:146-220) over agents
 * [agent_begin, agent_end) of every env of a DEVICE f32 observation array
 * [E, A, obs_dim]: writes DEVICE f64 logits [E, A, C*V] and values [E, A] at
 * the same (env, agent) rows (either may be NULL). Non-finite observations ->
 * WDG_ERR_NON_FINITE (policy_model.cpp:152-154). Synchronous. */
WDG_API wdg_status wdg_policy_forward(const wdg_policy* policy, const float* obs, int64_t num_envs,
                                      int64_t num_agents, int64_t agent_begin, int64_t agent_end,
                                      double* logits, double* values, int32_t precision,
                                      void* cuda_stream);
/* RolloutDriver with policies (harness.cpp:428-476): each step runs the
 * forward on the current observations, then samples, steps and resets.
 * Taggers use `tagger`, runners `runner` (tag_policy_map, harness.cpp:395-399);
 * the same policy twice = one shared policy (harness.cpp:586-606). NULL, NULL
 * restores the uniform policy. Policies must outlive their use. */
WDG_API wdg_status wdg_rollout_set_policies(wdg_rollout* rollout, const wdg_policy* tagger,
                                            const wdg_policy* runner, int32_t precision);
/* Keep the last forward's f64 logits (always kept for F64, which samples
 * from them) and values in device buffers (default off: the BF16 path then
 * stores only the sampled actions). */
WDG_API wdg_status wdg_rollout_set_keep_policy_outputs(wdg_rollout* rollout, int32_t keep);
/* Device f64 logits [E,A,C*V] / values [E,A] of the last policy forward. */
WDG_API wdg_status wdg_rollout_policy_outputs(wdg_rollout* rollout, const double** logits,
                                              const double** values);

/* ---- Rollout capture + returns (proj/include/warp/trainer.hpp:36-53) ---- */
/* RolloutBatch in HBM: obs [T,E,A,D] f32, actions [T,E,A,C] i32, rewards
 * [T,E,A] f32, done [T,E] u8, active [T,E,A] u8, values / logp [T,E,A] f64,
 * bootstrap [E,A] f64 — the reference layout (trainer.hpp:36-49). */
typedef struct wdg_batch wdg_batch;
typedef struct wdg_batch_view {
  int64_t horizon, num_envs, num_agents, obs_dim, num_categories;
  float* obs;
  int32_t* actions;
  float* rewards;
  uint8_t* done;
  uint8_t* active;
  double* values;
  double* logp;
  double* bootstrap;
} wdg_batch_view;
/* RolloutBatch::resize(T, E, A, D, C) (trainer.cpp:58-71), dims taken from the
 * store's observations / sampled_actions arrays. */
WDG_API wdg_status wdg_batch_create(const wdg_store* store, int64_t horizon, wdg_batch** out);
WDG_API void wdg_batch_destroy(wdg_batch* batch);
WDG_API wdg_status wdg_batch_get_view(const wdg_batch* batch, wdg_batch_view* out);
/* Trainer::collect (trainer.cpp:315-403) on device: `horizon` policy-driven
 * rollout steps (wdg_rollout_set_policies first) captured into the batch —
 * pre-step obs and values, sampled actions, active flags and log-prob at
 * sample time, rewards and done before reset-on-done — then the bootstrap
 * values of the final observations. */
WDG_API wdg_status wdg_rollout_collect(wdg_rollout* rollout, wdg_batch* batch);
/* compute_returns(batch, gamma) (trainer.cpp:73-88) into DEVICE f64 returns
 * [T,E,A]: R_t = r_t + gamma * (1 - done_t) * R_{t+1}, R_T = bootstrap. */
WDG_API wdg_status wdg_compute_returns(const wdg_batch* batch, double gamma, double* device_returns,
                                       void* cuda_stream);

/* ---- Session (proj/include/warp/warp_c.h:51-86) ------------------------- */
/* The reference's session C ABI on the device path: a strict JSON RunConfig
 * (harness.cpp:32-158,279-324; same keys, defaults, canonical JSON and FNV-1a
 * config hash), run modes check / bench-envs / bench-agents driving the B200
 * kernels, JSON report + summary, CSV reports under run.output_dir. Training
 * (the reference's CPU learner) is out of scope: it returns WDG_ERR_STATE. */
typedef struct wdg_session wdg_session;
WDG_API wdg_status wdg_session_open(const char* config_json, wdg_session** out);      /* warp_c.h:55 */
WDG_API wdg_status wdg_session_open_file(const char* path, wdg_session** out);        /* warp_c.h:56 */
WDG_API void wdg_session_close(wdg_session* session);                                 /* warp_c.h:57 */
WDG_API wdg_status wdg_session_set_seed(wdg_session* session, uint64_t seed);         /* warp_c.h:61 */
WDG_API wdg_status wdg_session_set_workers(wdg_session* session, int32_t workers);    /* warp_c.h:62 */
WDG_API wdg_status wdg_session_set_output_dir(wdg_session* session, const char* dir); /* warp_c.h:63 */
WDG_API const char* wdg_session_config_json(wdg_session* session);                    /* warp_c.h:66 */
WDG_API const char* wdg_session_config_hash(wdg_session* session);                    /* warp_c.h:67 */
/* check (harness.cpp:563-660): per variant x obs mode, the fused one-kernel
 * rollout and the unfused kernel sequence in lockstep with the same f64
 * policy, stores compared on device each step in the reference's causal
 * order; WDG_ERR_STATE on a divergence (c_api.cpp:177-191). */
WDG_API wdg_status wdg_session_run_check(wdg_session* session);                       /* warp_c.h:73 */
WDG_API wdg_status wdg_session_run_bench_envs(wdg_session* session);                  /* warp_c.h:74 */
WDG_API wdg_status wdg_session_run_bench_agents(wdg_session* session);                /* warp_c.h:75 */
WDG_API wdg_status wdg_session_run_training(wdg_session* session);                    /* warp_c.h:76 */
WDG_API const char* wdg_session_report_json(wdg_session* session);                    /* warp_c.h:79 */
WDG_API const char* wdg_session_summary(wdg_session* session);                        /* warp_c.h:80 */
WDG_API wdg_status wdg_session_dump_array(wdg_session* session, const char* array_name,
                                          const char* csv_path);                      /* warp_c.h:85-86 */

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* WDG_B200_H */
