/* oracle/tag_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's Tag env-step path, used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg as the CHECKER. It
 * is never linked into, called by, or substituted for the product library
 * (paper_2108_13976_b200/), which has no CPU fallback.
 *
 * Pinning: tests/test_oracle_pinning.py checks this restatement bit-for-bit
 * against the reference itself, compiled from /root/reference/proj/src into
 * oracle/_ref/ (oracle/Makefile), and against committed golden fixtures
 * tests/golden/ (.npz) generated from that build by tests/golden/make_golden.py.
 */
#ifndef WD_TAG_ORACLE_H
#define WD_TAG_ORACLE_H

#include <stdint.h>

#include "wdg_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Counter RNG, proj/include/warp/rng.hpp:23-53. */
uint64_t oracle_mix64(uint64_t x);
uint64_t oracle_key_bits(uint64_t seed, int64_t step, int64_t env, int64_t agent, int64_t category,
                         int64_t draw);
double oracle_uniform(uint64_t seed, int64_t step, int64_t env, int64_t agent, int64_t category,
                      int64_t draw);
uint64_t oracle_substream(uint64_t seed, uint64_t purpose);
/* sample_from_logits, proj/include/warp/sampler.hpp:18-30. */
int32_t oracle_sample_from_logits(const double* logits, int64_t n, double u);
/* move_discrete / move_continuous, proj/include/warp/tag_env.hpp:71-100. */
void oracle_move_discrete(int32_t action, float* x, float* y, int64_t grid_size);
void oracle_move_continuous(int32_t accel_action, int32_t turn_action, float* speed,
                            float* direction, float* x, float* y, float accel_delta,
                            float turn_delta, float max_speed, float world_len);

typedef struct oracle_world oracle_world;

/* register_tag_arrays on a fresh store of E envs (tag_env.cpp:280-341).
 * env_offset = global id of env 0 (keys use global ids). */
int oracle_create(const wdg_tag_config* cfg, int64_t num_envs, int64_t env_offset,
                  oracle_world** out);
void oracle_destroy(oracle_world* w);
/* sample_actions (sampler.cpp:5-40); logits NULL -> zeros. Returns 10
 * (non_finite) on a non-finite logit, leaving actions untouched. */
int oracle_sample(oracle_world* w, const double* logits, int64_t step, uint64_t seed);
/* TagReference::step (tag_env.cpp:530-577). */
int oracle_step(oracle_world* w, int64_t step);
/* EpisodeTracker::accumulate + finish_done (trainer.cpp:229-252) folded into
 * the stats vector (WDG_STAT_*). */
void oracle_track(oracle_world* w);
/* detect_done + auto_reset (reset_manager.cpp:20-44) with the Tag reinit
 * (tag_env.cpp:579-595). Returns the number of envs reset. */
int64_t oracle_reset_done(oracle_world* w);
int oracle_reset_ids(oracle_world* w, const int64_t* ids, int64_t n);
/* RolloutDriver::step x n (harness.cpp:478-494) incl. stats tracking. */
int oracle_rollout(oracle_world* w, const double* logits, int64_t first_step, int64_t n,
                   uint64_t seed);
/* Direct access to one named store array (dense [E, ...]); NULL if unknown. */
void* oracle_array(oracle_world* w, const char* name, int64_t* bytes);
int64_t oracle_episodes(const oracle_world* w, int64_t env);
void oracle_stats(const oracle_world* w, double* out, int32_t count);

/* ---- policy network (proj/src/policy_model.cpp) ------------------------ */
/* PolicyParams::param_count (policy_model.cpp:35-42); -1 on bad dims. */
int64_t oracle_policy_param_count(int64_t obs_dim, const int64_t* hidden, int32_t num_hidden,
                                  int64_t num_categories, int64_t num_choices);
/* init_policy (policy_model.cpp:107-144) into the canonical flat order. */
int oracle_policy_init(uint64_t seed, int64_t obs_dim, const int64_t* hidden, int32_t num_hidden,
                       int64_t num_categories, int64_t num_choices, double* params, int64_t count);
/* forward (policy_model.cpp:146-197) of `rows` f32 observation rows (x =
 * double(obs)); logits [rows, C*V] and values [rows] (either may be NULL).
 * Returns 10 (non_finite) on a non-finite observation. */
int oracle_policy_forward(const double* params, int64_t obs_dim, const int64_t* hidden,
                          int32_t num_hidden, int64_t num_categories, int64_t num_choices,
                          const float* obs, int64_t rows, double* logits, double* values);

/* ---- rollout batch (proj/src/trainer.cpp) ------------------------------- */
/* category_stats(z, V, a).logp summed over C categories (trainer.cpp:25-41,
 * 386-392), per row. */
void oracle_logp(const double* logits, const int32_t* actions, int64_t rows, int64_t C, int64_t V,
                 double* logp);
/* compute_returns (trainer.cpp:73-88): rewards [T,E,A], done [T,E],
 * bootstrap [E,A] -> returns [T,E,A]. */
void oracle_compute_returns(const float* rewards, const uint8_t* done, const double* bootstrap, int64_t T,
                            int64_t E, int64_t A, double gamma, double* returns);

/* ---- glibc sinf / cosf replica ------------------- */
/* The x86-64 glibc 2.39 FMA variant of sinf / cosf for |y| < 120 (the device
 * replica in tag_kernels.cu follows the same steps); larger |y| calls libm. */
float oracle_sinf_replica(float y);
float oracle_cosf_replica(float y);
/* Mismatches of the replica against this host's libm sinf / cosf over every
 * `stride`-th float bit pattern in [lo, hi] and its negation. */
int64_t oracle_trig_mismatches(float lo, float hi, uint32_t stride);

#ifdef __cplusplus
}
#endif

#endif
