// tag_params.hpp — POD parameter blocks shared by the host facade (*.cpp) and
// the sm_100a kernels (tag_kernels.cu). Plain C++ (no CUDA types) so both
// compilers see the identical layout.
#pragma once

#include <cstdint>

namespace wdg {

// Compile-time CTA shape limits of the env kernel: max threads per CTA and
// the minimum resident CTAs per SM given to __launch_bounds__ (register cap =
// 65536 / (threads * blocks)). Overridable for tuning builds.
#ifndef WDG_MAX_THREADS
#define WDG_MAX_THREADS 256
#endif
#ifndef WDG_MIN_BLOCKS
#define WDG_MIN_BLOCKS 3
#endif
inline constexpr int kMaxThreadsPerCta = WDG_MAX_THREADS;
#ifndef WDG_MIN_BLOCKS_DISCRETE
#define WDG_MIN_BLOCKS_DISCRETE 4
#endif
inline constexpr int kMinBlocksPerSm = WDG_MIN_BLOCKS;
inline constexpr int kMinBlocksPerSmDiscrete = WDG_MIN_BLOCKS_DISCRETE;

// Kernel modes (one kernel body, phase set chosen per launch; uniform per CTA).
enum TagMode : int32_t {
  kModeStep = 0,    // StepEngine::run_step: move -> resolve -> observe+reward
  kModeFused = 1,   // RolloutDriver::step: sample -> step -> stats -> reset-on-done
  kModeReinit = 2,  // make_tag_reinit for masked envs (or all: registration)
};

// Sticky device error bits (read at sync points, mapped to wdg_status).
// kErrStepOrder: an overlapped launch gave up waiting (seconds) for its envs'
// previous step (TagLaunch::env_seq) instead of hanging the device.
enum : uint32_t { kErrNonFinite = 1u, kErrBadAction = 2u, kErrStepOrder = 4u };

// Raw device addresses of one store's Tag arrays (tag_env.cpp:47-79 `Arrays`).
struct TagDevArrays {
  float* loc_x = nullptr;
  float* loc_y = nullptr;
  float* speed = nullptr;      // continuous only
  float* direction = nullptr;  // continuous only
  float* obs = nullptr;
  float* rewards = nullptr;
  uint8_t* is_tagger = nullptr;
  uint8_t* active = nullptr;
  uint8_t* tagged = nullptr;
  uint8_t* done = nullptr;
  int32_t* step_count = nullptr;
  int32_t* actions = nullptr;
  int32_t* credits = nullptr;
  const uint8_t* snap_is_tagger = nullptr;  // registration-time is_tagger
};

// Config constants cast to float exactly once, as bind_arrays does
// (tag_env.cpp:106-122), plus the launch geometry chosen by the host.
struct TagDevConfig {
  int32_t E = 0, A = 0, T = 0;  // envs (local), agents, taggers
  int32_t D = 0, C = 1, V = 5, K = 0, vis = 0;
  int32_t continuous = 0, partial = 0;
  int64_t env_offset = 0;  // global id of local env 0 (RNG keys)
  int64_t grid_size = 20;
  int32_t episode_length = 500;
  double world_length = 20.0;
  float world_hi = 0.f, inv_world = 0.f, accel_delta = 0.f, turn_delta = 0.f;
  float tag_radius = 0.f, inv_episode = 0.f, reward_per_tag = 0.f, penalty = 0.f;
  float max_speed_tagger = 1.f, max_speed_runner = 1.f;
  float inv_max_speed_tagger = 1.f, inv_max_speed_runner = 1.f;
  float fault_bias = 0.f;            // detail::fault_hooks().tag_radius_bias
  uint64_t placement_h0 = 0;         // mix64(substream(seed, kStreamPlacement))

  // Geometry (host-chosen, see tag.cpp choose_geometry).
  int32_t envs_per_cta = 1;
  int32_t threads_per_env = 32;   // agent loop stride inside an env
  int32_t threads = 32;           // blockDim.x
  int32_t grid_ctas = 1;
  int32_t use_grid = 0;           // bucket grid (envs_per_cta must be 1)
  int32_t lattice = 0;            // discrete with one grid cell per lattice point
  int32_t stage_obs = 0;          // per-warp smem staging of observation rows
  int32_t off_stage = 0;          // CTA offset of the staging area
  int32_t stage_floats = 0;       // floats per warp staging buffer (stage_rows * D)
  int32_t stage_rows = 32;        // rows staged per warp pass (16: wide continuous rows)
  int32_t gc = 1, ncells = 1;     // grid cells per side / total
  int32_t lattice_w = 1;          // discrete: floor(grid_size / gc)
  float cell_inv = 1.f;           // continuous: gc / world_length
  double cell_size = 1.0;         // continuous: world_length / gc
  // Shared-memory carve-up, bytes.
  int32_t env_bytes = 0;          // per-env block
  int32_t off_y = 0, off_speed = 0, off_dir = 0, off_sin = 0, off_cos = 0;
  int32_t off_cred = 0, off_tag = 0, off_act = 0, off_tagged = 0, off_knn = 0;
  int32_t off_cstart = 0, off_cfill = 0, off_items = 0, off_cellof = 0, off_cellknn = 0;
  int32_t off_cellact = 0;  // grid: per-cell "holds an active agent" flags
  int32_t off_celltag = 0;  // discrete lattice: per-cell lowest-index tagger (int32, INT_MAX = none)
  int32_t off_cellq = 0;    // discrete lattice: compacted list of the cells holding an active agent
  int32_t head_bytes = 0;         // CTA header (per-env scalars + scan scratch + mbarrier)
  int32_t bulk_in = 0;            // fused/step inputs staged by TMA bulk copies (one env per CTA)
  int32_t off_zone = 0;           // CTA offset of the bulk logits landing zone
  int32_t prefetch_stride = 0;    // bulk path: L2-prefetch env e + stride's inputs (0 = off)
  int32_t smem_bytes = 0;         // total dynamic smem per CTA
  // Shapes the shared-memory kernels cannot take (k_nearest > 32, more than
  // 65535 agents, or more than 227 KB of shared memory per env) run on the
  // global-memory TagReference kernels (twin_kernels.cu) instead.
  int32_t fallback = 0;
  // continuous K = 5 ring search on 32-bit (truncated d2, index) keys, exact
  // search only where the kept keys tie (knn_rings_keys)
  int32_t cont_keys = 0;
};

// Per-launch arguments.
struct TagLaunch {
  int32_t mode = kModeStep;
  int32_t do_reset = 1;          // fused: reset-on-done enabled
  int32_t track = 0;             // fused: EpisodeTracker stats
  int32_t init_episode = 0;      // reinit: 1 = registration (episode stays 0)
  uint64_t action_h_step = 0;    // absorb(mix64(substream(seed,kStreamActions)), step)
  // Graph-replay mode: step = *step_dev + step_add, hashed on device from
  // action_h0 = mix64(substream(seed, kStreamActions)) (step_dev == nullptr:
  // use action_h_step).
  const int64_t* step_dev = nullptr;
  int32_t step_add = 0;
  uint64_t action_h0 = 0;
  const double* logits = nullptr;
  // Multi-step residency (RolloutDriver::run, harness.cpp:492-494): n_steps > 1
  // runs steps step0 .. step0 + n_steps - 1 in ONE launch, each env's state
  // staying in shared memory between steps (fused mode with a logits buffer
  // only). Every step still reads its logits and writes every output.
  int32_t n_steps = 1;
  int64_t step0 = 0;
  const uint8_t* env_mask = nullptr;  // reinit: envs to reinit (nullptr = all)
  int32_t* episode = nullptr;         // per-env episode counter (device)
  // Per-env tracker slots [E][8]: run_tagger, run_runner, episodes,
  // tagger_return, runner_return, tag_events, env_steps, (pad).
  double* env_stats = nullptr;
  uint32_t* error = nullptr;          // sticky error word
  // Rollout capture (Trainer::collect hooks, trainer.cpp:357-397), fused into
  // the step: the sampled actions and the active flags at sample time, and
  // the step's rewards and done BEFORE reset-on-done, into caller slots
  // ([E, A, C], [E, A], [E, A], [E]); nullptr = no capture.
  int32_t* cap_actions = nullptr;
  uint8_t* cap_active = nullptr;
  float* cap_rewards = nullptr;
  uint8_t* cap_done = nullptr;
  // Programmatic dependent launch between consecutive fused steps
  // (RolloutDriver::step): env_seq[e] holds the sequence number of the last
  // launch that finished env e. This launch (sequence `seq`) lets the next one
  // start as soon as all its CTAs are resident, and each CTA waits only for
  // its own envs' previous launch (env_seq[e] == seq - 1), so the next step's
  // early envs run in the current step's tail. nullptr = plain launch.
  uint32_t* env_seq = nullptr;
  uint32_t seq = 0;
  const int64_t* seq_dev = nullptr;  // graph replay: seq = *seq_dev + seq_add
  uint32_t seq_add = 0;
  int32_t pdl_late = 0;              // trigger the next launch at exit instead of entry
  // Plain PDL behind device policy kernels: release the next launch at entry,
  // then griddepcontrol.wait for the previous kernels (no per-env flags).
  int32_t pdl_wait = 0;
  // Performance-analysis only (WDG_ABLATE env var, never set by the product,
  // tests or bench): bit0 skip exp/sampling, bit1 skip cell K-NN, bit2 skip
  // obs rows, bit3 skip grid build. Results are WRONG when non-zero.
  uint32_t ablate = 0;
};

}  // namespace wdg
