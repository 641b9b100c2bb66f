/* oracle/tag_oracle.c — TEST INFRASTRUCTURE ONLY (see tag_oracle.h).
 *
 * Plain-C restatement of the reference's sequential Tag path. Every function
 * cites the reference lines it restates (paths relative to the reference
 * tree). Compiled with -ffp-contract=off like the reference
 * (proj/CMakeLists.txt:10-13) so float results are bit-identical. */
#include "tag_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- rng.hpp:23-57 ------------------------------------------------------- */
static const uint64_t kGolden = 0x9e3779b97f4a7c15ULL;
static const uint64_t kStreamActions = 0x616374696f6e7331ULL;   /* rng.hpp:55 */
static const uint64_t kStreamPlacement = 0x706c6163656d656eULL; /* rng.hpp:56 */

uint64_t oracle_mix64(uint64_t x) { /* rng.hpp:23-28 */
  x += kGolden;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

static uint64_t absorb(uint64_t h, uint64_t v) { return oracle_mix64(h ^ (v + kGolden)); } /* :30 */

uint64_t oracle_key_bits(uint64_t seed, int64_t step, int64_t env, int64_t agent, int64_t category,
                         int64_t draw) { /* rng.hpp:34-42 */
  uint64_t h = oracle_mix64(seed);
  h = absorb(h, (uint64_t)step);
  h = absorb(h, (uint64_t)env);
  h = absorb(h, (uint64_t)agent);
  h = absorb(h, (uint64_t)category);
  h = absorb(h, (uint64_t)draw);
  return h;
}

double oracle_uniform(uint64_t seed, int64_t step, int64_t env, int64_t agent, int64_t category,
                      int64_t draw) { /* rng.hpp:45-47 */
  return (double)(oracle_key_bits(seed, step, env, agent, category, draw) >> 11) * 0x1.0p-53;
}

uint64_t oracle_substream(uint64_t seed, uint64_t purpose) { /* rng.hpp:51-53 */
  return oracle_mix64(oracle_mix64(seed) ^ purpose);
}

/* ---- sampler.hpp:18-30 --------------------------------------------------- */
int32_t oracle_sample_from_logits(const double* z, int64_t n, double u) {
  double zmax = z[0];
  for (int64_t i = 0; i < n; ++i) zmax = z[i] > zmax ? z[i] : zmax;
  double total = 0.0;
  for (int64_t i = 0; i < n; ++i) total += exp(z[i] - zmax);
  const double target = u * total;
  double cum = 0.0;
  for (int64_t i = 0; i + 1 < n; ++i) {
    cum += exp(z[i] - zmax);
    if (target < cum) return (int32_t)i;
  }
  return (int32_t)(n - 1);
}

/* ---- tag_env.hpp:71-100 -------------------------------------------------- */
static float fminf_ref(float a, float b) { return b < a ? b : a; } /* std::min(a,b) */
static float fmaxf_ref(float a, float b) { return a < b ? b : a; } /* std::max(a,b) */

void oracle_move_discrete(int32_t action, float* x, float* y, int64_t grid_size) {
  switch (action) {
    case 1: *y += 1.0f; break;
    case 2: *y -= 1.0f; break;
    case 3: *x -= 1.0f; break;
    case 4: *x += 1.0f; break;
    default: break;
  }
  const float hi = (float)(grid_size - 1);
  *x = fminf_ref(fmaxf_ref(*x, 0.0f), hi);
  *y = fminf_ref(fmaxf_ref(*y, 0.0f), hi);
}

static const float kTwoPi = 6.28318530717958647692f; /* tag_env.hpp:84 */

void oracle_move_continuous(int32_t accel_action, int32_t turn_action, float* speed,
                            float* direction, float* x, float* y, float accel_delta,
                            float turn_delta, float max_speed, float world_len) {
  if (turn_action == 0) *direction -= turn_delta;
  if (turn_action == 2) *direction += turn_delta;
  while (*direction >= kTwoPi) *direction -= kTwoPi;
  while (*direction < 0.0f) *direction += kTwoPi;
  if (accel_action == 0) *speed -= accel_delta;
  if (accel_action == 2) *speed += accel_delta;
  *speed = fminf_ref(fmaxf_ref(*speed, 0.0f), max_speed);
  const float vx = *speed * cosf(*direction);
  const float vy = *speed * sinf(*direction);
  *x += vx;
  *y += vy;
  *x = fminf_ref(fmaxf_ref(*x, 0.0f), world_len);
  *y = fminf_ref(fmaxf_ref(*y, 0.0f), world_len);
}

/* ---- the store + bound constants (tag_env.cpp:47-124, 280-322) ---------- */
struct oracle_world {
  wdg_tag_config cfg;
  int64_t E, A, D, C, V, K, env_offset;
  int continuous, partial;
  float *loc_x, *loc_y, *speed, *direction, *obs, *rewards;
  uint8_t *is_tagger, *active, *tagged, *done;
  int32_t *step_count, *actions, *credits;
  /* snapshot_on_reset copies (data_store.cpp:52) */
  float *snap_x, *snap_y, *snap_speed, *snap_dir;
  uint8_t *snap_tagger, *snap_active;
  int64_t* episode; /* ResetManager::episode_counter_ (reset_manager.hpp:42) */
  /* bind_arrays constants (tag_env.cpp:106-122) */
  float world_hi, inv_world, accel_delta, turn_delta, tag_radius, inv_episode, reward_per_tag,
      penalty;
  float *max_speed, *inv_max_speed;
  /* scratch */
  float *sin_row, *cos_row;
  float* knn_d2;
  int32_t* knn_idx;
  /* EpisodeTracker (trainer.cpp:221-258) reduced to sums */
  double *run_tagger, *run_runner;
  double stats[WDG_STAT_COUNT];
};

static void* zalloc(size_t n) { return calloc(n ? n : 1, 1); }

/* place_agent (tag_env.cpp:130-146) */
static void place_agent(const oracle_world* w, int64_t episode, int64_t env, int64_t agent,
                        float* x, float* y, float* dir) {
  const uint64_t stream = oracle_substream(w->cfg.seed, kStreamPlacement);
  const int64_t genv = w->env_offset + env;
  const double ux = oracle_uniform(stream, episode, genv, agent, 0, 0);
  const double uy = oracle_uniform(stream, episode, genv, agent, 1, 0);
  *dir = 0.0f;
  if (!w->continuous) {
    const double g = (double)w->cfg.grid_size;
    int64_t ix = (int64_t)(ux * g), iy = (int64_t)(uy * g);
    if (ix > w->cfg.grid_size - 1) ix = w->cfg.grid_size - 1;
    if (iy > w->cfg.grid_size - 1) iy = w->cfg.grid_size - 1;
    *x = (float)ix;
    *y = (float)iy;
  } else {
    const double ud = oracle_uniform(stream, episode, genv, agent, 2, 0);
    *x = (float)(ux * w->cfg.world_length);
    *y = (float)(uy * w->cfg.world_length);
    *dir = (float)(ud * 6.283185307179586);
  }
}

/* fill_sincos (tag_env.cpp:214-221) */
static void fill_sincos(oracle_world* w, int64_t e) {
  if (!w->continuous) return;
  const float* d = w->direction + e * w->A;
  for (int64_t a = 0; a < w->A; ++a) {
    w->sin_row[a] = sinf(d[a]);
    w->cos_row[a] = cosf(d[a]);
  }
}

/* select_k_nearest_brute (tag_env.cpp:225-237): the K smallest (d2, j) pairs
 * under lexicographic order, nearest first. Selection by insertion gives the
 * same prefix as the reference's full std::sort since the order is total. */
static void k_nearest(oracle_world* w, int64_t e, int64_t self) {
  const float* xs = w->loc_x + e * w->A;
  const float* ys = w->loc_y + e * w->A;
  const float sx = xs[self], sy = ys[self];
  int64_t found = 0;
  for (int64_t j = 0; j < w->A; ++j) {
    if (j == self) continue;
    const float dx = xs[j] - sx;
    const float dy = ys[j] - sy;
    const float d2 = dx * dx + dy * dy;
    if (found == w->K) {
      const float wd = w->knn_d2[w->K - 1];
      if (d2 > wd || (d2 == wd && j > w->knn_idx[w->K - 1])) continue;
    }
    int64_t pos = found < w->K ? found : w->K - 1;
    while (pos > 0 && (w->knn_d2[pos - 1] > d2 ||
                       (w->knn_d2[pos - 1] == d2 && w->knn_idx[pos - 1] > j))) {
      w->knn_d2[pos] = w->knn_d2[pos - 1];
      w->knn_idx[pos] = w->knn_idx[pos - 1];
      --pos;
    }
    w->knn_d2[pos] = d2;
    w->knn_idx[pos] = (int32_t)j;
    if (found < w->K) ++found;
  }
}

/* write_obs_row (tag_env.cpp:165-212); neighbors NULL = all others ascending */
static void write_obs_row(oracle_world* w, int64_t e, int64_t agent, const int32_t* neighbors,
                          int64_t n_neighbors) {
  const int64_t self = e * w->A + agent;
  float* out = w->obs + self * w->D;
  if (!w->active[self]) {
    for (int64_t i = 0; i < w->D; ++i) out[i] = 0.0f;
    return;
  }
  const float sx = w->loc_x[self], sy = w->loc_y[self];
  const int64_t nj = neighbors ? n_neighbors : w->A;
  for (int64_t t = 0; t < nj; ++t) {
    const int64_t j = neighbors ? neighbors[t] : t;
    if (!neighbors && j == agent) continue;
    const int64_t jj = e * w->A + j;
    out[0] = (w->loc_x[jj] - sx) * w->inv_world;
    out[1] = (w->loc_y[jj] - sy) * w->inv_world;
    out[2] = w->is_tagger[jj] ? 1.0f : 0.0f;
    out[3] = w->active[jj] ? 1.0f : 0.0f;
    if (w->continuous) {
      out[4] = w->speed[jj] * w->inv_max_speed[j];
      out[5] = w->sin_row[j];
      out[6] = w->cos_row[j];
      out += 7;
    } else {
      out += 4;
    }
  }
  out[0] = sx * w->inv_world;
  out[1] = sy * w->inv_world;
  if (w->continuous) {
    out[2] = w->speed[self] * w->inv_max_speed[agent];
    out[3] = w->sin_row[agent];
    out[4] = w->cos_row[agent];
    out += 5;
  } else {
    out += 2;
  }
  out[0] = (float)w->step_count[e] * w->inv_episode;
}

/* write_rewards_row (tag_env.cpp:252-259) */
static void write_rewards_row(oracle_world* w, int64_t e, int64_t agent) {
  const int64_t i = e * w->A + agent;
  if (w->is_tagger[i]) {
    w->rewards[i] = w->reward_per_tag * (float)w->credits[i];
  } else {
    w->rewards[i] = w->tagged[i] ? w->penalty : 0.0f;
  }
}

/* observe_env (tag_env.cpp:514-528) with rewards; reinit variant without. */
static void observe_env(oracle_world* w, int64_t e, int with_rewards) {
  fill_sincos(w, e);
  for (int64_t a = 0; a < w->A; ++a) {
    if (with_rewards) write_rewards_row(w, e, a);
    if (w->partial && w->active[e * w->A + a]) {
      k_nearest(w, e, a);
      write_obs_row(w, e, a, w->knn_idx, w->K);
    } else {
      write_obs_row(w, e, a, NULL, w->A - 1);
    }
  }
}

/* place_env (tag_env.cpp:261-273) */
static void place_env(oracle_world* w, int64_t e, int64_t episode) {
  for (int64_t a = 0; a < w->A; ++a) {
    const int64_t i = e * w->A + a;
    float x, y, dir;
    place_agent(w, episode, e, a, &x, &y, &dir);
    w->loc_x[i] = x;
    w->loc_y[i] = y;
    if (w->continuous) {
      w->speed[i] = 0.0f;
      w->direction[i] = dir;
    }
    w->active[i] = 1;
  }
}

static int validate(const wdg_tag_config* c) { /* TagConfig::validate, tag_env.cpp:20-40 */
  const int64_t A = c->num_taggers + c->num_runners;
  if (c->num_taggers < 1 || c->num_runners < 1 || c->episode_length < 1) return WDG_ERR_INVALID_CONFIG;
  if (c->tag_reward <= 0.0 || c->tagged_penalty >= 0.0) return WDG_ERR_INVALID_CONFIG;
  if (c->variant == WDG_TAG_DISCRETE) {
    if (c->grid_size < 1) return WDG_ERR_INVALID_CONFIG;
  } else {
    if (c->world_length <= 0.0 || c->tag_radius < 0.0 || c->accel_delta <= 0.0 ||
        c->turn_delta <= 0.0 || c->max_speed_tagger <= 0.0 || c->max_speed_runner <= 0.0)
      return WDG_ERR_INVALID_CONFIG;
  }
  if (c->obs_mode == WDG_OBS_PARTIAL && (c->k_nearest < 1 || c->k_nearest >= A))
    return WDG_ERR_INVALID_CONFIG;
  return WDG_OK;
}

int oracle_create(const wdg_tag_config* cfg, int64_t num_envs, int64_t env_offset,
                  oracle_world** out) {
  const int st = validate(cfg);
  if (st != WDG_OK) return st;
  if (num_envs < 1) return WDG_ERR_INVALID_ARGUMENT;
  oracle_world* w = (oracle_world*)zalloc(sizeof(oracle_world));
  w->cfg = *cfg;
  w->E = num_envs;
  w->A = cfg->num_taggers + cfg->num_runners;
  w->env_offset = env_offset;
  w->continuous = cfg->variant == WDG_TAG_CONTINUOUS;
  w->partial = cfg->obs_mode == WDG_OBS_PARTIAL;
  w->K = cfg->k_nearest;
  w->C = w->continuous ? 2 : 1;
  w->V = w->continuous ? 3 : 5;
  const int64_t vis = w->partial ? cfg->k_nearest : w->A - 1; /* tag_env.hpp:51-60 */
  w->D = vis * (w->continuous ? 7 : 4) + (w->continuous ? 5 : 2) + 1;
  const size_t n = (size_t)(w->E * w->A);
  w->loc_x = zalloc(n * 4); w->loc_y = zalloc(n * 4);
  w->speed = zalloc(n * 4); w->direction = zalloc(n * 4);
  w->obs = zalloc(n * (size_t)w->D * 4); w->rewards = zalloc(n * 4);
  w->is_tagger = zalloc(n); w->active = zalloc(n); w->tagged = zalloc(n);
  w->done = zalloc((size_t)w->E);
  w->step_count = zalloc((size_t)w->E * 4);
  w->actions = zalloc(n * (size_t)w->C * 4);
  w->credits = zalloc(n * 4);
  w->snap_x = zalloc(n * 4); w->snap_y = zalloc(n * 4);
  w->snap_speed = zalloc(n * 4); w->snap_dir = zalloc(n * 4);
  w->snap_tagger = zalloc(n); w->snap_active = zalloc(n);
  w->episode = zalloc((size_t)w->E * 8);
  w->max_speed = zalloc((size_t)w->A * 4); w->inv_max_speed = zalloc((size_t)w->A * 4);
  w->sin_row = zalloc((size_t)w->A * 4); w->cos_row = zalloc((size_t)w->A * 4);
  w->knn_d2 = zalloc((size_t)(w->K > 0 ? w->K : 1) * 4);
  w->knn_idx = zalloc((size_t)(w->K > 0 ? w->K : 1) * 4);
  w->run_tagger = zalloc((size_t)w->E * 8); w->run_runner = zalloc((size_t)w->E * 8);

  /* bind_arrays constants, tag_env.cpp:106-122 */
  w->world_hi = w->continuous ? (float)cfg->world_length : (float)(cfg->grid_size - 1);
  w->inv_world = 1.0f / (float)(w->continuous ? cfg->world_length : (double)cfg->grid_size);
  w->accel_delta = (float)cfg->accel_delta;
  w->turn_delta = (float)cfg->turn_delta;
  w->tag_radius = (float)cfg->tag_radius;
  w->inv_episode = 1.0f / (float)cfg->episode_length;
  w->reward_per_tag = (float)cfg->tag_reward;
  w->penalty = (float)cfg->tagged_penalty;
  for (int64_t a = 0; a < w->A; ++a) {
    const float ms = (float)(a < cfg->num_taggers ? cfg->max_speed_tagger : cfg->max_speed_runner);
    w->max_speed[a] = ms;
    w->inv_max_speed[a] = 1.0f / ms;
  }
  /* register_tag_arrays: episode-0 state, tag_env.cpp:288-299 */
  for (int64_t e = 0; e < w->E; ++e) {
    for (int64_t a = 0; a < w->A; ++a) {
      const int64_t i = e * w->A + a;
      float x, y, dir;
      place_agent(w, 0, e, a, &x, &y, &dir);
      w->loc_x[i] = x;
      w->loc_y[i] = y;
      w->direction[i] = dir;
      w->is_tagger[i] = a < cfg->num_taggers ? 1 : 0;
      w->active[i] = 1;
    }
  }
  memcpy(w->snap_x, w->loc_x, n * 4);
  memcpy(w->snap_y, w->loc_y, n * 4);
  memcpy(w->snap_speed, w->speed, n * 4);
  memcpy(w->snap_dir, w->direction, n * 4);
  memcpy(w->snap_tagger, w->is_tagger, n);
  memcpy(w->snap_active, w->active, n);
  /* episode-0 observations, tag_env.cpp:324-340 */
  for (int64_t e = 0; e < w->E; ++e) observe_env(w, e, 0);
  *out = w;
  return WDG_OK;
}

void oracle_destroy(oracle_world* w) {
  if (!w) return;
  void* bufs[] = {w->loc_x, w->loc_y, w->speed, w->direction, w->obs, w->rewards,
                  w->is_tagger, w->active, w->tagged, w->done, w->step_count, w->actions,
                  w->credits, w->snap_x, w->snap_y, w->snap_speed, w->snap_dir, w->snap_tagger,
                  w->snap_active, w->episode, w->max_speed, w->inv_max_speed, w->sin_row,
                  w->cos_row, w->knn_d2, w->knn_idx, w->run_tagger, w->run_runner};
  for (size_t i = 0; i < sizeof(bufs) / sizeof(bufs[0]); ++i) free(bufs[i]);
  free(w);
}

/* sample_actions, sampler.cpp:5-40 (finiteness scan first, then writes) */
int oracle_sample(oracle_world* w, const double* logits, int64_t step, uint64_t seed) {
  const int64_t rows = w->E * w->A * w->C;
  if (logits) {
    for (int64_t i = 0; i < rows * w->V; ++i)
      if (!isfinite(logits[i])) return WDG_ERR_NON_FINITE;
  }
  static const double zeros[64] = {0};
  const uint64_t stream = oracle_substream(seed, kStreamActions);
  int64_t out = 0;
  for (int64_t e = 0; e < w->E; ++e) {
    for (int64_t a = 0; a < w->A; ++a) {
      for (int64_t c = 0; c < w->C; ++c) {
        const double u = oracle_uniform(stream, step, w->env_offset + e, a, c, 0);
        const double* row = logits ? logits + out * w->V : zeros;
        w->actions[out] = oracle_sample_from_logits(row, w->V, u);
        ++out;
      }
    }
  }
  return WDG_OK;
}

/* TagReference::step, tag_env.cpp:530-577 */
int oracle_step(oracle_world* w, int64_t step) {
  (void)step;
  const int64_t E = w->E, A = w->A;
  for (int64_t e = 0; e < E; ++e) {
    for (int64_t a = 0; a < A; ++a) { /* apply_move, tag_env.cpp:148-160 */
      const int64_t i = e * A + a;
      if (!w->active[i]) continue;
      if (!w->continuous) {
        oracle_move_discrete(w->actions[i], &w->loc_x[i], &w->loc_y[i], w->cfg.grid_size);
      } else {
        oracle_move_continuous(w->actions[i * 2], w->actions[i * 2 + 1], &w->speed[i],
                               &w->direction[i], &w->loc_x[i], &w->loc_y[i], w->accel_delta,
                               w->turn_delta, w->max_speed[a], w->world_hi);
      }
    }
  }
  for (int64_t e = 0; e < E; ++e) { /* resolve, tag_env.cpp:539-574 */
    const int64_t base = e * A;
    memset(w->credits + base, 0, (size_t)A * 4);
    memset(w->tagged + base, 0, (size_t)A);
    const float* xs = w->loc_x + base;
    const float* ys = w->loc_y + base;
    const float r2 = w->tag_radius * w->tag_radius;
    for (int64_t rn = 0; rn < A; ++rn) {
      if (w->is_tagger[base + rn] || !w->active[base + rn]) continue;
      int32_t best = -1;
      float best_d2 = 0.0f;
      for (int64_t tg = 0; tg < A; ++tg) {
        if (!w->is_tagger[base + tg]) continue;
        if (!w->continuous) {
          if (xs[tg] == xs[rn] && ys[tg] == ys[rn] && (best < 0 || tg < best)) best = (int32_t)tg;
        } else {
          const float dx = xs[tg] - xs[rn];
          const float dy = ys[tg] - ys[rn];
          const float d2 = dx * dx + dy * dy;
          if (d2 <= r2 && (best < 0 || d2 < best_d2 || (d2 == best_d2 && (int32_t)tg < best))) {
            best = (int32_t)tg;
            best_d2 = d2;
          }
        }
      }
      if (best >= 0) {
        w->active[base + rn] = 0;
        w->tagged[base + rn] = 1;
        w->credits[base + best] += 1;
      }
    }
    /* resolve_env_counters, tag_env.cpp:241-250 */
    w->step_count[e] += 1;
    int64_t runners_left = 0;
    for (int64_t a = 0; a < A; ++a)
      if (!w->is_tagger[base + a] && w->active[base + a]) ++runners_left;
    w->done[e] = (w->step_count[e] >= w->cfg.episode_length || runners_left == 0) ? 1 : 0;
  }
  for (int64_t e = 0; e < E; ++e) observe_env(w, e, 1); /* tag_env.cpp:576 */
  return WDG_OK;
}

/* EpisodeTracker::accumulate + finish_done (trainer.cpp:229-252) with the
 * tag_policy_map grouping (harness.cpp:395-400): taggers [0,T), runners. */
void oracle_track(oracle_world* w) {
  const int64_t A = w->A, T = w->cfg.num_taggers;
  for (int64_t e = 0; e < w->E; ++e) {
    double st = 0.0, sr = 0.0;
    for (int64_t a = 0; a < T; ++a) st += (double)w->rewards[e * A + a];
    for (int64_t a = T; a < A; ++a) sr += (double)w->rewards[e * A + a];
    w->run_tagger[e] += st;
    w->run_runner[e] += sr;
    for (int64_t a = 0; a < A; ++a) w->stats[WDG_STAT_TAG_EVENTS] += w->tagged[e * A + a];
    if (w->done[e]) {
      w->stats[WDG_STAT_EPISODES] += 1.0;
      w->stats[WDG_STAT_TAGGER_RETURN] += w->run_tagger[e];
      w->stats[WDG_STAT_RUNNER_RETURN] += w->run_runner[e];
      w->run_tagger[e] = 0.0;
      w->run_runner[e] = 0.0;
    }
  }
  w->stats[WDG_STAT_ENV_STEPS] += (double)w->E;
}

/* auto_reset for one env (reset_manager.cpp:29-44 + data_store.cpp:207-217 +
 * tag_zero_on_reset tag_env.cpp:343-346 + TagReference::reinit_env
 * tag_env.cpp:579-595). */
static void reset_env(oracle_world* w, int64_t e) {
  const int64_t A = w->A, b = e * A;
  const size_t fb = (size_t)A * 4;
  memcpy(w->loc_x + b, w->snap_x + b, fb);
  memcpy(w->loc_y + b, w->snap_y + b, fb);
  if (w->continuous) {
    memcpy(w->speed + b, w->snap_speed + b, fb);
    memcpy(w->direction + b, w->snap_dir + b, fb);
  }
  memcpy(w->is_tagger + b, w->snap_tagger + b, (size_t)A);
  memcpy(w->active + b, w->snap_active + b, (size_t)A);
  w->step_count[e] = 0;
  memset(w->rewards + b, 0, fb);
  w->done[e] = 0;
  memset(w->credits + b, 0, fb);
  memset(w->tagged + b, 0, (size_t)A);
  memset(w->actions + b * w->C, 0, (size_t)(A * w->C) * 4);
  memset(w->obs + b * w->D, 0, (size_t)(A * w->D) * 4);
  w->episode[e] += 1;
  place_env(w, e, w->episode[e]);
  observe_env(w, e, 0);
}

int64_t oracle_reset_done(oracle_world* w) { /* detect_done, reset_manager.cpp:20-27 */
  int64_t n = 0;
  for (int64_t e = 0; e < w->E; ++e) {
    if (w->done[e]) {
      reset_env(w, e);
      ++n;
    }
  }
  return n;
}

int oracle_reset_ids(oracle_world* w, const int64_t* ids, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (ids[i] < 0 || ids[i] >= w->E) return WDG_ERR_INDEX_OUT_OF_RANGE;
  for (int64_t i = 0; i < n; ++i) reset_env(w, ids[i]);
  return WDG_OK;
}

int oracle_rollout(oracle_world* w, const double* logits, int64_t first_step, int64_t n,
                   uint64_t seed) {
  for (int64_t s = 0; s < n; ++s) {
    const int st = oracle_sample(w, logits, first_step + s, seed);
    if (st != WDG_OK) return st;
    oracle_step(w, first_step + s);
    oracle_track(w);
    oracle_reset_done(w);
  }
  return WDG_OK;
}

void* oracle_array(oracle_world* w, const char* name, int64_t* bytes) {
  const int64_t n = w->E * w->A;
  struct { const char* name; void* p; int64_t b; } t[] = {
      {"loc_x", w->loc_x, n * 4}, {"loc_y", w->loc_y, n * 4},
      {"speed", w->continuous ? w->speed : NULL, n * 4},
      {"direction", w->continuous ? w->direction : NULL, n * 4},
      {"is_tagger", w->is_tagger, n}, {"active", w->active, n},
      {"step_count", w->step_count, w->E * 4}, {"observations", w->obs, n * w->D * 4},
      {"sampled_actions", w->actions, n * w->C * 4}, {"rewards", w->rewards, n * 4},
      {"done", w->done, w->E}, {"tag_credits", w->credits, n * 4},
      {"was_tagged", w->tagged, n}};
  for (size_t i = 0; i < sizeof(t) / sizeof(t[0]); ++i) {
    if (strcmp(t[i].name, name) == 0 && t[i].p) {
      if (bytes) *bytes = t[i].b;
      return t[i].p;
    }
  }
  return NULL;
}

int64_t oracle_episodes(const oracle_world* w, int64_t env) {
  if (env < 0 || env >= w->E) return -1;
  return w->episode[env];
}

void oracle_stats(const oracle_world* w, double* out, int32_t count) {
  for (int32_t i = 0; i < count && i < WDG_STAT_COUNT; ++i) out[i] = w->stats[i];
}

/* ---- policy network (proj/src/policy_model.cpp) -------------------------- */

int64_t oracle_policy_param_count(int64_t obs_dim, const int64_t* hidden, int32_t num_hidden,
                                  int64_t num_categories, int64_t num_choices) {
  /* check_dims (policy_model.cpp:14-21) */
  if (obs_dim < 1 || num_categories < 1 || num_choices < 1 || num_hidden < 1) return -1;
  int64_t n = 0, in = obs_dim;
  for (int32_t l = 0; l < num_hidden; ++l) {
    if (hidden[l] < 1) return -1;
    n += hidden[l] * in + hidden[l];
    in = hidden[l];
  }
  return n + num_categories * num_choices * (in + 1) + in + 1;
}

/* xavier (policy_model.cpp:112-121): bound = sqrt(6 / (fan_in + fan_out)),
 * w[r, c] = (2u - 1) * bound, u = uniform({stream, matrix_id, r, c, 0, 0}). */
static void xavier(double* w, int64_t fan_out, int64_t fan_in, int64_t matrix_id, uint64_t stream) {
  const double bound = sqrt(6.0 / (double)(fan_in + fan_out));
  for (int64_t r = 0; r < fan_out; ++r)
    for (int64_t c = 0; c < fan_in; ++c)
      w[r * fan_in + c] = (2.0 * oracle_uniform(stream, matrix_id, r, c, 0, 0) - 1.0) * bound;
}

int oracle_policy_init(uint64_t seed, int64_t obs_dim, const int64_t* hidden, int32_t num_hidden,
                       int64_t num_categories, int64_t num_choices, double* params, int64_t count) {
  const int64_t n = oracle_policy_param_count(obs_dim, hidden, num_hidden, num_categories, num_choices);
  if (n < 0) return 1;   /* invalid_argument */
  if (count != n) return 3; /* shape_mismatch */
  const uint64_t stream = oracle_substream(seed, 0x706172616d733030ULL); /* kStreamParams */
  double* w = params;
  int64_t in = obs_dim, id = 0;
  for (int32_t l = 0; l < num_hidden; ++l) {
    xavier(w, hidden[l], in, id++, stream);
    w += hidden[l] * in;
    for (int64_t i = 0; i < hidden[l]; ++i) *w++ = 0.0;
    in = hidden[l];
  }
  for (int64_t c = 0; c < num_categories; ++c) { /* per-category logit blocks */
    xavier(w, num_choices, in, id++, stream);
    w += num_choices * in;
  }
  for (int64_t i = 0; i < num_categories * num_choices; ++i) *w++ = 0.0;
  xavier(w, 1, in, id++, stream);
  w += in;
  *w = 0.0;
  return 0;
}

int oracle_policy_forward(const double* params, int64_t obs_dim, const int64_t* hidden,
                          int32_t num_hidden, int64_t num_categories, int64_t num_choices,
                          const float* obs, int64_t rows, double* logits, double* values) {
  const int64_t W = num_categories * num_choices;
  int64_t maxw = obs_dim;
  for (int32_t l = 0; l < num_hidden; ++l) maxw = hidden[l] > maxw ? hidden[l] : maxw;
  for (int64_t i = 0; i < rows * obs_dim; ++i)
    if (!isfinite((double)obs[i])) return 10; /* policy_model.cpp:152-154 */
  double* cur = (double*)malloc(sizeof(double) * (size_t)maxw);
  double* next = (double*)malloc(sizeof(double) * (size_t)maxw);
  for (int64_t r = 0; r < rows; ++r) {
    for (int64_t d = 0; d < obs_dim; ++d) cur[d] = (double)obs[r * obs_dim + d];
    const double* p = params;
    int64_t in = obs_dim;
    for (int32_t l = 0; l < num_hidden; ++l) {
      const int64_t out = hidden[l];
      const double* w = p;
      const double* b = p + out * in;
      for (int64_t o = 0; o < out; ++o) { /* next = b; matvec_acc (policy_model.cpp:24-31) */
        double acc = 0.0;
        for (int64_t c = 0; c < in; ++c) acc += w[o * in + c] * cur[c];
        next[o] = tanh(b[o] + acc);
      }
      p += out * in + out;
      in = out;
      double* t = cur;
      cur = next;
      next = t;
    }
    const double* hw = p;
    const double* hb = hw + W * in;
    const double* vw = hb + W;
    const double vb = vw[in];
    if (logits) {
      for (int64_t o = 0; o < W; ++o) {
        double acc = 0.0;
        for (int64_t c = 0; c < in; ++c) acc += hw[o * in + c] * cur[c];
        logits[r * W + o] = hb[o] + acc;
      }
    }
    if (values) {
      double v = vb; /* policy_model.cpp:192-193 */
      for (int64_t c = 0; c < in; ++c) v += vw[c] * cur[c];
      values[r] = v;
    }
  }
  free(cur);
  free(next);
  return 0;
}

/* ---- rollout batch (proj/src/trainer.cpp) --------------------------------- */

void oracle_logp(const double* logits, const int32_t* actions, int64_t rows, int64_t C, int64_t V,
                 double* logp) {
  for (int64_t i = 0; i < rows; ++i) {
    double lp = 0.0;
    for (int64_t c = 0; c < C; ++c) {
      const double* z = logits + (i * C + c) * V;
      double zmax = z[0];
      for (int64_t k = 1; k < V; ++k) zmax = zmax < z[k] ? z[k] : zmax;
      double sum = 0.0;
      for (int64_t k = 0; k < V; ++k) sum += exp(z[k] - zmax);
      lp += z[actions[i * C + c]] - zmax - log(sum);
    }
    logp[i] = lp;
  }
}

void oracle_compute_returns(const float* rewards, const uint8_t* done, const double* bootstrap, int64_t T,
                            int64_t E, int64_t A, double gamma, double* returns) {
  for (int64_t e = 0; e < E; ++e) {
    for (int64_t a = 0; a < A; ++a) {
      double next = bootstrap[e * A + a];
      for (int64_t t = T - 1; t >= 0; --t) {
        const int64_t idx = (t * E + e) * A + a;
        const double cont = done[t * E + e] ? 0.0 : 1.0;
        next = (double)rewards[idx] + gamma * cont * next;
        returns[idx] = next;
      }
    }
  }
}

/* ---- glibc sinf / cosf replica ------------------------------------------- */
/* Coefficients of glibc's __sincosf_table (optimized-routines sincosf.h):
 * table 1 is table 0 with the cos coefficients negated. */
typedef struct {
  double hpi_inv, hpi, c0, c1, s1, c2, s2, c3, s3, c4;
} sincos_tab;
static const sincos_tab k_sincos[2] = {
    {0x1.45f306dc9c883p+23, 0x1.921fb54442d18p+0, 0x1.0p+0, -0x1.ffffffd0c621cp-2, -0x1.555545995a603p-3,
     0x1.55553e1068f19p-5, 0x1.1107605230bc4p-7, -0x1.6c087e89a359dp-10, -0x1.994eb3774cf24p-13,
     0x1.99343027bf8c3p-16},
    {0x1.45f306dc9c883p+23, 0x1.921fb54442d18p+0, -0x1.0p+0, 0x1.ffffffd0c621cp-2, -0x1.555545995a603p-3,
     -0x1.55553e1068f19p-5, 0x1.1107605230bc4p-7, 0x1.6c087e89a359dp-10, -0x1.994eb3774cf24p-13,
     -0x1.99343027bf8c3p-16}};

static double rep_sin_poly(double xs, double x2, const sincos_tab* p) {
  const double a = fma(x2, p->s3, p->s2);
  const double x3 = x2 * xs;
  const double x5 = x2 * x3;
  return fma(a, x5, fma(x3, p->s1, xs));
}

static double rep_cos_poly(double x2, const sincos_tab* p) {
  const double x4 = x2 * x2;
  const double a = fma(x2, p->c1, p->c0);
  const double b = fma(x2, p->c4, p->c3);
  const double x6 = x2 * x4;
  return fma(b, x6, fma(x4, p->c2, a));
}

static float rep_sincosf(float y, int want_cos) {
  uint32_t u;
  memcpy(&u, &y, 4);
  const uint32_t top = (u >> 20) & 0x7ffu;
  const double x = (double)y;
  if (top <= 0x3f3u) {
    if (top <= 0x397u) return want_cos ? 1.0f : y;
    const double x2 = x * x;
    return (float)(want_cos ? rep_cos_poly(x2, &k_sincos[0]) : rep_sin_poly(x, x2, &k_sincos[0]));
  }
  if (top > 0x42eu) return want_cos ? cosf(y) : sinf(y);
  const int n = (((int32_t)(x * k_sincos[0].hpi_inv)) + 0x800000) >> 24;
  const double r = fma(-(double)n, k_sincos[0].hpi, x);
  const sincos_tab* p = &k_sincos[(n & 2) ? 1 : 0];
  const double x2 = r * r;
  if ((((n & 1) == 0) ? 1 : 0) == want_cos) return (float)rep_cos_poly(x2, p);
  const double sign = ((n + 1) & 2) ? -1.0 : 1.0;
  return (float)rep_sin_poly(r * sign, x2, p);
}

float oracle_sinf_replica(float y) { return rep_sincosf(y, 0); }
float oracle_cosf_replica(float y) { return rep_sincosf(y, 1); }

int64_t oracle_trig_mismatches(float lo, float hi, uint32_t stride) {
  uint32_t a, b;
  memcpy(&a, &lo, 4);
  memcpy(&b, &hi, 4);
  int64_t bad = 0;
  for (uint64_t w = a; w <= b; w += stride) {
    float y;
    const uint32_t u = (uint32_t)w;
    memcpy(&y, &u, 4);
    for (int sg = 0; sg < 2; ++sg) {
      const float z = sg ? -y : y;
      const float s = sinf(z), c = cosf(z);
      if (memcmp(&s, &(float){oracle_sinf_replica(z)}, 4) != 0) ++bad;
      if (memcmp(&c, &(float){oracle_cosf_replica(z)}, 4) != 0) ++bad;
    }
  }
  return bad;
}
