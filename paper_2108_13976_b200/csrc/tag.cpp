// tag.cpp — Tag environment host side: config validation, array registration,
// the plan (kernel geometry + launches), sample_actions, ResetManager and the
// rollout driver. Reference interfaces: proj/include/warp/tag_env.hpp,
// sampler.hpp, reset_manager.hpp, proj/src/harness.cpp:428-505.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <numeric>
#include <set>

#include "facade.hpp"
#include "policy.hpp"
#include "batch.hpp"
#include "kernels.hpp"

namespace wdg {

// ---- host RNG prefix (rng.hpp:23-53) --------------------------------------
uint64_t host_mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
uint64_t host_absorb(uint64_t h, uint64_t v) { return host_mix64(h ^ (v + 0x9e3779b97f4a7c15ULL)); }
uint64_t host_substream(uint64_t seed, uint64_t purpose) {
  return host_mix64(host_mix64(seed) ^ purpose);
}

float& fault_tag_radius_bias() {
  static float bias = 0.0f;
  return bias;
}

// ---- plan tuning overrides --------------------------------------------------
// Geometry / launch-overlap choices the plan normally makes itself, settable
// through wdg_set_tuning for A/B measurements and for tests that pin a code
// path. None of them changes WHAT a launch computes, only how it is mapped.
// Environment variables are read only by a tuning build (-DWDG_TUNING).
namespace {
struct TuningKey {
  const char* name;
  const char* env;
};
constexpr TuningKey kTuningKeys[] = {
    {"stage_rows", "WDG_STAGE_ROWS"},             // 16 / 32: continuous K=5 obs staging rows per pass
    {"brute_max", "WDG_BRUTE_MAX"},               // agents up to which the brute-force layout is used
    {"threads_per_env_max", "WDG_TPE_MAX"},       // CTA thread cap of the one-env-per-CTA layout
    {"cont_cell_div", "WDG_CONT_GC_DIV"},         // continuous: agents per bucket cell
    {"disc_grid_cells", "WDG_DISC_GC"},           // discrete: bucket cells per side
    {"stage_obs", "WDG_STAGE_OBS"},               // 0: never stage observation rows in smem
    {"bulk_in", "WDG_BULK_IN"},                   // 0: no TMA bulk staging of the inputs
    {"l2_prefetch", "WDG_L2_PREFETCH"},           // env stride of an L2 prefetch of later inputs
    {"pdl_mode", "WDG_PDL"},                      // launch overlap, TagPlan::pdl_mode values
    {"multistep", "WDG_MULTISTEP"},               // 0: no multi-step residency in run()
    {"cont_keys", "WDG_CONT_KEYS"},               // continuous K=5: 1 keyed ring search, 0 exact only
    {"packed_warps_max", "WDG_PACKED_WARPS"},     // warp cap of the packed (brute-force) CTA
};
constexpr int kNumTuning = static_cast<int>(sizeof(kTuningKeys) / sizeof(kTuningKeys[0]));
int64_t* tuning_table() {
  static int64_t table[kNumTuning] = {};
  static bool init = [] {
    for (int i = 0; i < kNumTuning; ++i) table[i] = -1;
#ifdef WDG_TUNING
    for (int i = 0; i < kNumTuning; ++i)
      if (const char* v = std::getenv(kTuningKeys[i].env)) table[i] = std::atoll(v);
#endif
    return true;
  }();
  (void)init;
  return table;
}
int64_t tuning(const char* name, int64_t fallback) {
  for (int i = 0; i < kNumTuning; ++i)
    if (std::string(kTuningKeys[i].name) == name) return tuning_table()[i] >= 0 ? tuning_table()[i] : fallback;
  return fallback;
}
}  // namespace

void set_tuning(const std::string& key, int64_t value) {
  if (key == "reset") {
    for (int i = 0; i < kNumTuning; ++i) tuning_table()[i] = -1;
    return;
  }
  for (int i = 0; i < kNumTuning; ++i) {
    if (key == kTuningKeys[i].name) {
      tuning_table()[i] = value < 0 ? -1 : value;
      return;
    }
  }
  raise(Errc::invalid_argument, "set_tuning: unknown key \"" + key + "\"");
}

// ---- TagConfig::validate (tag_env.cpp:20-40) -------------------------------
void validate_tag_config(const wdg_tag_config& c) {
  auto fail = [](const std::string& msg) { raise(Errc::invalid_config, "TagConfig: " + msg); };
  if (c.variant != WDG_TAG_DISCRETE && c.variant != WDG_TAG_CONTINUOUS) fail("unknown variant");
  if (c.obs_mode != WDG_OBS_FULL && c.obs_mode != WDG_OBS_PARTIAL) fail("unknown obs_mode");
  if (c.num_taggers < 1) fail("num_taggers must be >= 1");
  if (c.num_runners < 1) fail("num_runners must be >= 1");
  if (c.episode_length < 1) fail("episode_length must be >= 1");
  if (c.tag_reward <= 0.0) fail("tag_reward must be > 0");
  if (c.tagged_penalty >= 0.0) fail("tagged_penalty must be < 0");
  if (c.variant == WDG_TAG_DISCRETE) {
    if (c.grid_size < 1) fail("grid_size must be >= 1");
  } else {
    if (c.world_length <= 0.0) fail("world_length must be > 0");
    if (c.tag_radius < 0.0) fail("tag_radius must be >= 0");
    if (c.accel_delta <= 0.0) fail("accel_delta must be > 0");
    if (c.turn_delta <= 0.0) fail("turn_delta must be > 0");
    if (c.max_speed_tagger <= 0.0 || c.max_speed_runner <= 0.0) fail("max speeds must be > 0");
  }
  if (c.obs_mode == WDG_OBS_PARTIAL) {
    if (c.k_nearest < 1) fail("k_nearest must be >= 1");
    if (c.k_nearest >= c.num_taggers + c.num_runners) {
      fail("k_nearest must be < num_taggers + num_runners");
    }
  }
}

int64_t tag_obs_dim(const wdg_tag_config& c) {  // tag_env.hpp:51-60
  const bool cont = c.variant == WDG_TAG_CONTINUOUS;
  const int64_t A = c.num_taggers + c.num_runners;
  const int64_t vis = c.obs_mode == WDG_OBS_PARTIAL ? c.k_nearest : A - 1;
  return vis * (cont ? 7 : 4) + (cont ? 5 : 2) + 1;
}

std::vector<std::string> tag_zero_on_reset() {  // tag_env.cpp:343-346
  return {"step_count", kRewards, kDone, "tag_credits", "was_tagged", kSampledActions,
          kObservations};
}

// ---- kernel geometry ------------------------------------------------------
namespace {
constexpr int kNumSMs = 148;
constexpr int kBruteMaxAgents = 64;    // brute-force K-NN/resolve up to this (full obs)
constexpr int kBruteMaxPartialDisc = 192;  // ... partial obs, discrete without lattice cells
constexpr int kBruteMaxPartialCont = 160;  // ... partial obs, continuous
constexpr int kMaxSmem = 227 * 1024;

int32_t round_up(int64_t v, int64_t m) { return static_cast<int32_t>((v + m - 1) / m * m); }
int32_t align16(int64_t v) { return round_up(v, 16); }
}  // namespace

namespace {
TagDevConfig make_dev_config_rows(const DataStore& store, const wdg_tag_config& cfg, int stage_rows);

int resident_ctas(const TagDevConfig& p) {
  uint32_t per_sm = 0;
  TagLaunch q;
  q.mode = -1;  // occupancy query
  q.error = &per_sm;
  return launch_tag_kernel(p, TagDevArrays{}, q, nullptr) == cudaSuccess ? static_cast<int>(per_sm) : 0;
}
}  // namespace

// Wide continuous rows (K=5, D=41) may stage half a warp's rows per pass
// (TagDevConfig::stage_rows = 16); that costs a second pass per warp, so it is
// taken only when the smaller CTA fits more CTAs per SM. Measured at 2000
// envs: A = 1000 491 -> 473 us/step (2 -> 3 CTAs per SM); A = 300, where the
// register cap already holds it at 3, 265 -> 285 us/step.
TagDevConfig make_dev_config(const DataStore& store, const wdg_tag_config& cfg) {
  TagDevConfig full = make_dev_config_rows(store, cfg, 32);
  if (full.fallback || !full.continuous || !full.partial || full.K != 5 || !full.use_grid || !full.stage_obs)
    return full;
  const int64_t forced = tuning("stage_rows", 0);
  if (forced == 32) return full;
  TagDevConfig half = make_dev_config_rows(store, cfg, 16);
  if (forced == 16) return half;
  return resident_ctas(half) > resident_ctas(full) ? half : full;
}

namespace {
TagDevConfig make_dev_config_rows(const DataStore& store, const wdg_tag_config& cfg, int stage_rows) {
  validate_tag_config(cfg);
  TagDevConfig p;
  const int64_t A = cfg.num_taggers + cfg.num_runners;
  if (store.num_agents() != A) {
    raise(Errc::shape_mismatch, "tag plan: store num_agents != config agents");
  }
  if (store.num_envs() > (int64_t{1} << 31) - 1) raise(Errc::invalid_config, "too many envs");
  if (A > 65535) p.fallback = 1;  // 16-bit agent indices in the shared-memory tables
  p.E = static_cast<int32_t>(store.num_envs());
  p.A = static_cast<int32_t>(A);
  p.T = static_cast<int32_t>(cfg.num_taggers);
  p.continuous = cfg.variant == WDG_TAG_CONTINUOUS;
  p.partial = cfg.obs_mode == WDG_OBS_PARTIAL;
  p.C = p.continuous ? 2 : 1;
  p.V = p.continuous ? 3 : 5;
  p.K = p.partial ? static_cast<int32_t>(cfg.k_nearest) : 0;
  if (p.partial && p.K > 32) p.fallback = 1;  // register top-K lists
  p.vis = p.partial ? p.K : p.A - 1;
  p.D = static_cast<int32_t>(tag_obs_dim(cfg));
  p.env_offset = store.env_offset();
  p.grid_size = cfg.grid_size;
  p.episode_length = static_cast<int32_t>(std::min<int64_t>(cfg.episode_length, INT32_MAX));
  p.world_length = cfg.world_length;
  // bind_arrays constants (tag_env.cpp:106-122): each cast to float once.
  p.world_hi = p.continuous ? static_cast<float>(cfg.world_length)
                            : static_cast<float>(cfg.grid_size - 1);
  const double side = p.continuous ? cfg.world_length : static_cast<double>(cfg.grid_size);
  p.inv_world = 1.0f / static_cast<float>(side);
  p.accel_delta = static_cast<float>(cfg.accel_delta);
  p.turn_delta = static_cast<float>(cfg.turn_delta);
  p.tag_radius = static_cast<float>(cfg.tag_radius);
  p.inv_episode = 1.0f / static_cast<float>(cfg.episode_length);
  p.reward_per_tag = static_cast<float>(cfg.tag_reward);
  p.penalty = static_cast<float>(cfg.tagged_penalty);
  p.max_speed_tagger = static_cast<float>(cfg.max_speed_tagger);
  p.max_speed_runner = static_cast<float>(cfg.max_speed_runner);
  p.inv_max_speed_tagger = 1.0f / p.max_speed_tagger;
  p.inv_max_speed_runner = 1.0f / p.max_speed_runner;
  p.fault_bias = fault_tag_radius_bias();
  p.placement_h0 = host_mix64(host_substream(cfg.seed, kStreamPlacement));

  if (p.fallback) return p;  // the global-memory kernels need no geometry

  // Geometry: grid path = one env per CTA; brute path packs envs per CTA.
  // Discrete lattice cells (one bucket per grid point) once the grid is at
  // least half occupied and the cell tables fit: per-cell K-NN lists and
  // per-cell tagger lookup. Measured at grid 20, 2000 envs, partial K=5:
  // A = 200 100 vs 151 us/step (gc 14), A = 300 109 vs 166 (gc 17); at
  // A = 100 it loses (99 vs 76, gc 10).
  const int64_t g = cfg.grid_size;
  const int64_t lattice_cell_bytes = 9 + (p.partial ? 4 * (int64_t{p.K} + 1) : 0);
  // Round 2 (LEAN lattice kernel, 2000 envs, grid 20, us/step lattice vs
  // brute): A = 150 87 vs 60, A = 192 50 vs 75 -> lattice from 0.4 agents per cell.
  const bool lattice_fits = !p.continuous && g <= 128 && 2 * g * g <= 5 * A &&
                            g * g * lattice_cell_bytes <= 96 * 1024;
  // Partial obs keeps the brute-force K-NN (one env per <= 8 warps) where it
  // beats the bucket grid at 2000 envs, K=5 (us/step, brute vs grid; round 2
  // on the LEAN grid kernels: continuous A = 100 57 vs 100, 200 141 vs 142,
  // 256 178 vs 146 -> brute up to 200):
  // discrete A = 100 41 vs 76, 160 63 vs 140 (ring), 256 121 vs 99 (lattice);
  // continuous A = 100 63 vs 103, 200 148 vs 192, 256 185 vs 196.
  // Continuous after the flattened 3 x 3 block scan with paired key
  // insertion (tools/tune_scan.py, brute vs grid): A = 100 55.7 vs 70.8,
  // 150 85.6 vs 100.2, 170 99.9 vs 108.3, 200 138.8 vs 103.3; after the
  // continuous brute-force keys: 160 83.1 vs 89.7, 176 99.4 vs 96.0, 192
  // 106.3 vs 97.2 -> brute to 160.
  int brute_max = !p.partial ? kBruteMaxAgents
                  : p.continuous ? kBruteMaxPartialCont
                  : lattice_fits ? kBruteMaxAgents : kBruteMaxPartialDisc;
  brute_max = static_cast<int>(tuning("brute_max", brute_max));
  brute_max = std::min(brute_max, kMaxThreadsPerCta);  // one thread per agent of a packed env
  p.use_grid = A > brute_max ? 1 : 0;
  if (p.use_grid) {
    // One env per CTA, one thread per agent up to the CTA cap (larger A
    // loops). Thread cap per env, re-measured in round 2 on the LEAN kernels
    // at 2000 envs, partial K=5 (us/step at 128 / 192 / 256 threads,
    // tools/tune_scan.py): discrete A = 200 56 / 71 / 83, 300 63 / 74 / 76,
    // 400 71 / 80 / 76, 500 86 / 83 / 78, 700 108 / 94 / 88, 864 - / 120 / 95;
    // continuous A = 300 166 / 176 / 204, 400 188 / 196 / 217, 500 246 / 211 /
    // 224, 600 263 / 240 / 260, 700 - / 292 / 270, 800 - / 342 / 290,
    // 1000 477 / 393 / 360. Smaller envs keep more CTAs (envs) per SM
    // overlapping each other's barriers; larger ones gain from wider CTAs.
    // Discrete re-measured after the paired key insertion of the per-cell
    // lists (us/step at 128 / 160 / 256 threads): A = 500 59.2 / 60.2 / 68.2,
    // 600 70.3 / 63.7 / 73.1, 700 81.6 / 78.6 / 75.8, 800 88.2 / 83.4 / 80.3.
    int cap = 256;
    if (p.partial && (p.continuous ? A <= 400 : A <= 560)) cap = 128;
    else if (p.partial && !p.continuous && A <= 660) cap = 160;
    else if (p.partial && p.continuous && A <= 650) cap = 192;
    if (const int64_t t = tuning("threads_per_env_max", 0)) cap = static_cast<int>(std::clamp<int64_t>(t, 32, 1024)) / 32 * 32;
    cap = std::min(cap, kMaxThreadsPerCta);
    p.envs_per_cta = 1;
    p.threads = std::min<int32_t>(round_up(A, 32), cap);
    p.threads_per_env = p.threads;
  } else {
    // Smallest CTA (in warps) that holds >= 1 env, grown while the grid keeps
    // >= 2 CTAs per SM so small-A sweeps spread over all 148 SMs.
    int w = static_cast<int>((A + 31) / 32);
    // Envs of more than one warp keep the smallest CTA: more, narrower CTAs
    // measured faster (us/step run / step, smallest CTA vs grown to 7-8 warps
    // with 2 envs): discrete A = 100 30.3 / 31.4 vs 33.1 / 33.8, continuous
    // A = 100 41.6 / 46.8 vs 46.9 / 50.2. At A = 20 it was mixed (continuous
    // 9.1 / 14.1 vs 8.7 / 14.5) and discrete A = 10 gains from growing (9.3 at
    // two warps vs 9.8 at one), so warp-sized envs still grow.
    const int wmax = static_cast<int>(std::clamp<int64_t>(tuning("packed_warps_max", A > 32 ? 1 : 8), 1, 8));
    for (int cand = w; cand <= std::min(wmax, kMaxThreadsPerCta / 32); cand *= 2) {
      const int64_t epc = (32 * cand) / A;
      const int64_t ctas = (store.num_envs() + epc - 1) / epc;
      if (cand == w || ctas >= 2 * kNumSMs) w = cand;
      else break;
    }
    p.envs_per_cta = static_cast<int32_t>(std::max<int64_t>(1, (32 * w) / A));
    p.threads = round_up(static_cast<int64_t>(p.envs_per_cta) * A, 32);
    // A one-env CTA owns all its threads (the kernel's single-env paths take
    // every thread as the env's: CTA-uniform barriers and lane-0 updates);
    // packed CTAs give each env A threads and leave the tail idle.
    p.threads_per_env = p.envs_per_cta == 1 ? p.threads : p.A;
  }
  p.grid_ctas = static_cast<int32_t>((store.num_envs() + p.envs_per_cta - 1) / p.envs_per_cta);

  // Bucket grid: ~1 agent per cell, lattice cells for discrete when possible.
  const int sq = std::max(1, static_cast<int>(std::floor(std::sqrt(static_cast<double>(A)))));
  if (p.continuous) {
    // ~4 agents per cell: the K=5 nearest then mostly sit within the 3 x 3
    // block (one flattened scan, knn_rings_keys). Measured with that scan
    // (tools/tune_scan.py, us/step at div 2 / 3 / 4 / 5 / 6 / 8): A = 1000
    // 285.2 / 264.2 / 250.7 / 251.9 / 265.9 / 280.4, 500 168.1 / 157.6 /
    // 154.2 / 153.2 / 155.6, 700 - / 196.5 / 191.7 / 195.1, 300 (keyed)
    // 141.3 / 130.1 / 122.2 / 121.3 / 121.2. (Round 1, per-cell rings: 3.)
    int div = 4;
    div = static_cast<int>(std::max<int64_t>(1, tuning("cont_cell_div", div)));
    p.gc = std::max(1, std::min(static_cast<int>(std::floor(std::sqrt(static_cast<double>(A) / div))), 128));
    p.cell_inv = static_cast<float>(static_cast<double>(p.gc) / cfg.world_length);
    p.cell_size = cfg.world_length / p.gc;
    // keyed ring search (LEAN, 2000 envs, us/step exact / keyed,
    // tools/keys_scan.py): A = 300 133.7 / 137.3, 400 155.1 / 158.0, 450
    // 202.3 / 198.2, 500 181.7 / 172.9, 700 236.3 / 223.6, 1000 305.0 / 292.4
    // — it won on the CTAs wider than 128 threads (A > 400). With the
    // flattened 3 x 3 block and paired insertion it wins on every grid shape
    // (exact / keyed at div 4: A = 200 106.5 / 103.3, 300 129.5 / 122.2,
    // 400 151.1 / 141.6), so grid plans always take it.
    p.cont_keys = tuning("cont_keys", 1) != 0 ? 1 : 0;
  } else {
    p.gc = static_cast<int32_t>(std::min<int64_t>(cfg.grid_size, std::min(sq, 128)));
    if (lattice_fits) p.gc = static_cast<int32_t>(g);
    if (const int64_t t = tuning("disc_grid_cells", 0))
      p.gc = static_cast<int32_t>(std::clamp<int64_t>(t, 1, std::min<int64_t>(cfg.grid_size, 128)));
    p.lattice_w = static_cast<int32_t>(cfg.grid_size / p.gc);
    p.lattice = p.gc == cfg.grid_size ? 1 : 0;
  }
  p.ncells = p.gc * p.gc;
  // Observation rows staged per warp in shared memory when a row is narrow.
  const int64_t nwarps = p.threads / 32;
  int64_t stage_bytes = nwarps * 32 * int64_t{p.D} * 4;
  p.stage_obs = (p.D <= 64 && stage_bytes <= 112 * 1024) ? 1 : 0;
  p.stage_obs = p.stage_obs && tuning("stage_obs", 1) != 0;
  // Continuous K=5 rows (D = 41) at one env per CTA may use half-warp passes
  // (see make_dev_config): the staging buffer halves (42 -> 21 KB at 256 threads).
  p.stage_rows = 32;
  if (stage_rows == 16 && p.continuous && p.partial && p.K == 5 && p.use_grid && p.stage_obs) {
    p.stage_rows = 16;
    stage_bytes /= 2;
  }
  p.stage_floats = p.stage_rows * p.D;

  // Shared-memory carve-up per env.
  int64_t off = 0;
  auto take = [&](int64_t bytes, int64_t align) {
    off = (off + align - 1) / align * align;
    const int32_t at = static_cast<int32_t>(off);
    off += bytes;
    return at;
  };
  take(4 * A, 16);  // x at 0
  p.off_y = take(4 * A, 16);
  if (p.continuous) {
    p.off_speed = take(4 * A, 16);
    p.off_dir = take(4 * A, 16);
  }
  p.off_cred = take(4 * A, 16);
  p.off_tag = take(A, 16);
  p.off_act = take(A, 16);
  p.off_tagged = take(A, 16);
  // Arrays from here on are first written after phase 1 (sin/cos in phase
  // 4/6, the K-NN lists and the bucket grid from phase 2), so the bulk-copy
  // logits zone may overlay them.
  const int64_t late_begin = align16(off);
  if (p.continuous) {
    p.off_sin = take(4 * A, 16);
    p.off_cos = take(4 * A, 16);
  }
  if (p.partial && !p.stage_obs) p.off_knn = take(2 * A * p.K, 4);
  if (p.use_grid) {
    p.off_cstart = take(4 * (p.ncells + 1), 4);
    p.off_cfill = take(4 * (p.ncells + 1), 4);
    p.off_items = take(2 * A, 4);
    p.off_cellof = take(2 * A, 16);  // 8-byte vector access (build_grid_lattice)
    if (p.lattice && p.partial) p.off_cellknn = take(2 * int64_t{p.ncells} * (p.K + 1), 4);
    p.off_cellact = take(p.ncells, 16);
    if (p.lattice) {
      p.off_celltag = take(4 * int64_t{p.ncells}, 16);
      p.off_cellq = take(2 * int64_t{p.ncells}, 16);
    }
  }
  p.env_bytes = align16(off);
  // CTA header: per-env scalars + 64 doubles of warp scratch (scan / sums).
  p.head_bytes = align16(p.envs_per_cta * 48 + 96 * 8 + 16);  // scratch + mbarrier (tag_kernels.cu kScratchDoubles)
  int64_t total = static_cast<int64_t>(p.head_bytes) + int64_t{p.envs_per_cta} * p.env_bytes;
  if (p.stage_obs) {
    p.off_stage = static_cast<int32_t>(align16(total));
    total = p.off_stage + stage_bytes;
  }
  // Bulk-copy input staging (one env per CTA, A % 4 == 0): the env's f64
  // logits rows land by one TMA bulk copy in a zone that overlays the
  // late arrays, the bucket grid and the obs staging, dead until phase 2. The
  // zone starts at the first late array (CTA offset head + late_begin) and grows
  // the CTA's smem if the logits need more than those areas.
  p.bulk_in = 0;
  if (p.use_grid && (A % 4) == 0 && tuning("bulk_in", 1) != 0) {
    const int64_t logits_bytes = int64_t{A} * p.C * p.V * 8;
    const int64_t zone = align16(static_cast<int64_t>(p.head_bytes) + late_begin);
    const int64_t need = zone + logits_bytes;
    if (std::max<int64_t>(total, need) <= kMaxSmem && logits_bytes % 16 == 0) {
      p.bulk_in = 1;
      p.off_zone = static_cast<int32_t>(zone);
      total = std::max<int64_t>(total, need);
      // Optional L2 prefetch of the next wave's env inputs (tuning key
      // l2_prefetch = env stride). Off: measured neutral at one wave (296)
      // and -3% at 592 / 1184 envs ahead on C2 — the bulk loads are not HBM-bound.
      p.prefetch_stride = static_cast<int32_t>(tuning("l2_prefetch", 0));
    }
  }
  if (total > kMaxSmem) {  // too large for one CTA's shared memory
    TagDevConfig f = p;
    f.fallback = 1;
    return f;
  }
  p.smem_bytes = static_cast<int32_t>(total);
  return p;
}
}  // namespace

TagDevArrays bind_dev_arrays(DataStore& store, const wdg_tag_config& cfg) {
  // bind_arrays (tag_env.cpp:81-124) — same names, device addresses.
  TagDevArrays g;
  auto f32 = [&](const char* n) { return static_cast<float*>(store.device_ptr(store.handle(n))); };
  auto u8 = [&](const char* n) { return static_cast<uint8_t*>(store.device_ptr(store.handle(n))); };
  auto i32 = [&](const char* n) { return static_cast<int32_t*>(store.device_ptr(store.handle(n))); };
  auto expect = [&](const char* n, int32_t kind, int64_t env_stride) {
    const ArrayInfo& in = store.info(store.handle(n));
    if (in.spec.kind != kind || in.env_stride != env_stride) {
      raise(Errc::shape_mismatch, std::string("tag plan: array \"") + n + "\" has the wrong kind/shape");
    }
  };
  const int64_t A = cfg.num_taggers + cfg.num_runners;
  const bool cont = cfg.variant == WDG_TAG_CONTINUOUS;
  expect("loc_x", WDG_REAL32, A);
  expect("loc_y", WDG_REAL32, A);
  expect("is_tagger", WDG_BOOL8, A);
  expect("active", WDG_BOOL8, A);
  expect("step_count", WDG_INT32, 1);
  expect(kObservations, WDG_REAL32, A * tag_obs_dim(cfg));
  expect(kSampledActions, WDG_INT32, A * (cont ? 2 : 1));
  expect(kRewards, WDG_REAL32, A);
  expect(kDone, WDG_BOOL8, 1);
  expect("tag_credits", WDG_INT32, A);
  expect("was_tagged", WDG_BOOL8, A);
  g.loc_x = f32("loc_x");
  g.loc_y = f32("loc_y");
  if (cont) {
    expect("speed", WDG_REAL32, A);
    expect("direction", WDG_REAL32, A);
    g.speed = f32("speed");
    g.direction = f32("direction");
  }
  g.obs = f32(kObservations);
  g.rewards = f32(kRewards);
  g.is_tagger = u8("is_tagger");
  g.active = u8("active");
  g.tagged = u8("was_tagged");
  g.done = u8(kDone);
  g.step_count = i32("step_count");
  g.actions = i32(kSampledActions);
  g.credits = i32("tag_credits");
  g.snap_is_tagger = static_cast<const uint8_t*>(store.snapshot_ptr(store.handle("is_tagger")));
  return g;
}

// ---- register_tag_arrays (tag_env.cpp:280-341) ------------------------------
void register_tag_arrays(DataStore& store, const wdg_tag_config& cfg) {
  validate_tag_config(cfg);
  const int64_t E = store.num_envs();
  const int64_t A = cfg.num_taggers + cfg.num_runners;
  if (store.num_agents() != A) {
    raise(Errc::shape_mismatch, "register_tag_arrays: store num_agents != config agents");
  }
  // Geometry check first so an unsupported shape fails before any allocation.
  (void)make_dev_config(store, cfg);
  const bool cont = cfg.variant == WDG_TAG_CONTINUOUS;
  std::vector<uint8_t> is_tagger(static_cast<size_t>(E * A)), active(static_cast<size_t>(E * A), 1);
  for (int64_t e = 0; e < E; ++e)
    for (int64_t a = 0; a < A; ++a) is_tagger[static_cast<size_t>(e * A + a)] = a < cfg.num_taggers;
  // Same names, shapes, kinds and snapshot flags as the reference.
  store.register_array({"loc_x", {E, A}, WDG_REAL32, true}, nullptr, 0);
  store.register_array({"loc_y", {E, A}, WDG_REAL32, true}, nullptr, 0);
  if (cont) {
    store.register_array({"speed", {E, A}, WDG_REAL32, true}, nullptr, 0);
    store.register_array({"direction", {E, A}, WDG_REAL32, true}, nullptr, 0);
  }
  store.register_array({"is_tagger", {E, A}, WDG_BOOL8, true}, is_tagger.data(), E * A);
  store.register_array({"active", {E, A}, WDG_BOOL8, true}, active.data(), E * A);
  store.register_array({"step_count", {E}, WDG_INT32, false}, nullptr, 0);
  store.register_array({kObservations, {E, A, tag_obs_dim(cfg)}, WDG_REAL32, false}, nullptr, 0);
  store.register_array({kSampledActions, {E, A, cont ? 2 : 1}, WDG_INT32, false}, nullptr, 0);
  store.register_array({kRewards, {E, A}, WDG_REAL32, false}, nullptr, 0);
  store.register_array({kDone, {E}, WDG_BOOL8, false}, nullptr, 0);
  store.register_array({"tag_credits", {E, A}, WDG_INT32, false}, nullptr, 0);
  store.register_array({"was_tagged", {E, A}, WDG_BOOL8, false}, nullptr, 0);

  // Episode-0 placement + observations computed on device (the reinit kernel
  // with episode 0 on every env), then captured as the registration snapshot.
  TagDevConfig p = make_dev_config(store, cfg);
  TagDevArrays g = bind_dev_arrays(store, cfg);
  if (p.fallback) {  // episode-0 placement + observations by the global-memory kernels
    float* kd = nullptr;
    int32_t* ki = nullptr;
    if (p.partial) {
      const size_t n = static_cast<size_t>(p.E) * p.A * p.K;
      cuda_check(cudaMalloc(&kd, n * sizeof(float)), "cudaMalloc(knn scratch)");
      cuda_check(cudaMalloc(&ki, n * sizeof(int32_t)), "cudaMalloc(knn scratch)");
    }
    const cudaError_t err = launch_twin_kernel(p, g, kModeReinit, nullptr, nullptr, kd, ki, store.stream());
    if (err == cudaSuccess) cudaStreamSynchronize(store.stream());
    if (kd) cudaFree(kd);
    if (ki) cudaFree(ki);
    cuda_check(err, "register_tag_arrays init kernel (global-memory path)");
  } else {
    TagLaunch L;
    L.mode = kModeReinit;
    L.init_episode = 1;
    cuda_check(launch_tag_kernel(p, g, L, store.stream()), "register_tag_arrays init kernel");
  }
  for (const char* n : {"loc_x", "loc_y", "speed", "direction", "active"}) {
    if (store.has_array(n)) store.refresh_snapshot(store.handle(n));
  }
  store.synchronize();
}

// ---- TagPlan ---------------------------------------------------------------
TagPlan::TagPlan(DataStore& store, const wdg_tag_config& cfg, bool reference)
    : store_(store), cfg_(cfg), reference_(reference) {
  validate_tag_config(cfg);
  if (!store.locked()) raise(Errc::state_error, "build_tag_plan: store must be locked");
  dev_ = make_dev_config(store, cfg);
  arrays_ = bind_dev_arrays(store, cfg);
  // A shape the shared-memory kernels cannot take steps on the global-memory
  // kernels (the same code as the check's TagReference twin, parity-tested),
  // through the unfused sample -> run_step -> auto_reset sequence.
  if (dev_.fallback) reference_ = true;
  if (reference_) {
    if (dev_.partial) {
      const size_t n = static_cast<size_t>(dev_.E) * dev_.A * dev_.K;
      cuda_check(cudaMalloc(&knn_d2_, n * sizeof(float)), "cudaMalloc(twin knn)");
      cuda_check(cudaMalloc(&knn_idx_, n * sizeof(int32_t)), "cudaMalloc(twin knn)");
    }
    // The episode-0 state and observations of register_tag_arrays
    // (tag_env.cpp:288-340) recomputed by the twin itself.
    dev_.fault_bias = 0.0f;
    cuda_check(launch_twin_kernel(dev_, arrays_, kModeReinit, nullptr, nullptr, knn_d2_, knn_idx_,
                                  store_.stream()),
               "twin registration");
  }
}

TagPlan::~TagPlan() {
  if (knn_d2_) cudaFree(knn_d2_);
  if (knn_idx_) cudaFree(knn_idx_);
}

void TagPlan::launch(TagLaunch L) {
  if (reference_) raise(Errc::state_error, "tag plan: the TagReference twin runs run_step / reinit only");
  dev_.fault_bias = fault_tag_radius_bias();
  cuda_check(launch_tag_kernel(dev_, arrays_, L, store_.stream()), "tag kernel launch");
}

// Multi-step residency pays everywhere measured except the generic ring
// K-NN (continuous / non-lattice discrete partial obs) at fewer than 3 waves
// of CTAs, where it measured 2-18% slower, and grid-path full observations
// (profiles/sweep_r01.json: single_step vs run_multistep).
// Overlapping consecutive fused launches (TagLaunch::env_seq), measured per
// step at 2000 envs (us; released at CTA entry / at exit / serial):
//   C2 127 / 137 / 135; continuous partial A = 1000 449 / - / 476 (A = 300
//   202 / - / 203); grid full obs A = 100 61 / - / 80; brute partial A = 100
//   37 / - / 44;
//   discrete partial grids below 256 threads: A = 300 111 / 85 / 87, A = 500
//   104 / 88 / 90 (A = 200 / 700 at entry: 106 / 117 vs 86 / 112 serial);
//   tiny packed envs (C4): 10.1 / 9.5 / 8.2, and 22.8 vs 8.6 at 10000 envs
//   (25 envs per CTA): the per-env waits cost more than the few-microsecond
//   kernels can overlap. Plain PDL (release at entry, whole-grid
//   griddepcontrol.wait) still hides the launch gap there: 6.9 vs 8.2.
int TagPlan::pdl_mode() const {
  if (const int64_t t = tuning("pdl_mode", -1); t >= 0) return static_cast<int>(t);  // A/B experiments, tests
  if (!dev_.use_grid) return (dev_.envs_per_cta <= 4 && dev_.threads >= 128) ? 1 : 3;
  // Grid plans: released at CTA entry. Re-measured in round 2 on the LEAN
  // kernels (us/step, modes 0 / 1 / 2 / 3): discrete A = 200 (128 threads)
  // 57 / 50 / 57 / 56, A = 400 72 / 65 / 71 / 70, A = 500 87 / 78 / 89 / 85,
  // C2 112 / 99 / 114 / 110; continuous A = 300 188 / 166 / 174 / 186, A = 500
  // 254 / 211 / 238 / 252 (round 1's exit release for small discrete grids no
  // longer pays).
  return 1;
}

bool TagPlan::multistep_ok() {
  if (multistep_ < 0) {
    multistep_ = 1;

    // full observations on the grid path: the looped (multi-step) build of
    // the wide-row writer is 6-9% slower than the single-step build
    // (profiles/sweep_r01.json), which outweighs the saved state reloads
    if (dev_.use_grid && !dev_.partial) multistep_ = 0;
    // discrete grid envs below 256 threads (A <= 864): the looped build
    // measured 3-36% slower than one launch per step (e.g. A = 300: 117 vs
    // 86 us/step)
    if (dev_.use_grid && !dev_.continuous && dev_.threads < 256) multistep_ = 0;
    if (dev_.use_grid && dev_.partial && !dev_.lattice) {
      uint32_t per_sm = 0;
      TagLaunch q;
      q.mode = -1;  // occupancy query
      q.error = &per_sm;
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const bool ok = launch_tag_kernel(dev_, arrays_, q, store_.stream()) == cudaSuccess && per_sm > 0;
      const double waves = ok ? static_cast<double>(dev_.grid_ctas) / (static_cast<double>(sms) * per_sm) : 0.0;
      multistep_ = waves >= 3.0 ? 1 : 0;
    }
    // LEAN single steps (one overlapped launch per step) beat the looped
    // multi-step build: C2 107 vs 117 us/step, continuous A = 1000 374 vs 406
    if (lean_plan(dev_)) multistep_ = 0;
  }
  return multistep_ == 1;
}

// One launch over the env range [e0, e0 + n): the plan's geometry with every
// per-env pointer moved to env e0 and env_offset advanced, so the RNG keys
// (global env ids) and the results equal those of a whole-store launch.
void TagPlan::launch_envs(TagLaunch L, int64_t e0, int64_t n) {
  if (e0 == 0 && n == dev_.E) return launch(L);
  if (reference_) raise(Errc::state_error, "tag plan: the TagReference twin runs run_step / reinit only");
  if (e0 < 0 || n <= 0 || e0 + n > dev_.E) raise(Errc::index_out_of_range, "tag launch: env range");
  if ((e0 * dev_.A * dev_.D) % 4 != 0 || (e0 * dev_.A) % 4 != 0) {
    raise(Errc::invalid_argument, "tag launch: env range must start on 16-byte boundaries of the arrays");
  }
  TagDevConfig d = dev_;
  d.fault_bias = fault_tag_radius_bias();
  d.E = static_cast<int32_t>(n);
  d.env_offset += e0;
  d.grid_ctas = static_cast<int32_t>((n + d.envs_per_cta - 1) / d.envs_per_cta);
  const int64_t A = d.A;
  TagDevArrays g = arrays_;
  auto adv = [&](auto*& ptr, int64_t per_env) {
    if (ptr != nullptr) ptr += e0 * per_env;
  };
  adv(g.loc_x, A);
  adv(g.loc_y, A);
  adv(g.speed, A);
  adv(g.direction, A);
  adv(g.obs, A * d.D);
  adv(g.rewards, A);
  adv(g.is_tagger, A);
  adv(g.active, A);
  adv(g.tagged, A);
  adv(g.done, 1);
  adv(g.step_count, 1);
  adv(g.actions, A * d.C);
  adv(g.credits, A);
  adv(g.snap_is_tagger, A);
  adv(L.logits, A * d.C * d.V);
  adv(L.env_mask, 1);
  adv(L.episode, 1);
  adv(L.env_stats, 8);
  adv(L.cap_actions, A * d.C);
  adv(L.cap_active, A);
  adv(L.cap_rewards, A);
  adv(L.cap_done, 1);
  adv(L.env_seq, 1);
  cuda_check(launch_tag_kernel(d, g, L, store_.stream()), "tag kernel launch (env range)");
}

void TagPlan::run_step(int64_t step_index) {
  (void)step_index;  // the Tag kernels do not use the step index (tag_env.cpp:530)
  if (reference_) {
    cuda_check(launch_twin_kernel(dev_, arrays_, kModeStep, nullptr, nullptr, knn_d2_, knn_idx_, store_.stream()),
               "twin step");
    return;
  }
  TagLaunch L;
  L.mode = kModeStep;
  launch(L);
}

void TagPlan::reinit_masked(const uint8_t* env_mask, int32_t* episode) {
  if (reference_) {
    cuda_check(launch_twin_kernel(dev_, arrays_, kModeReinit, env_mask, episode, knn_d2_, knn_idx_,
                                  store_.stream()),
               "twin reinit");
    return;
  }
  TagLaunch L;
  L.mode = kModeReinit;
  L.env_mask = env_mask;
  L.episode = episode;
  launch(L);
}

// ---- sample_actions (sampler.cpp:5-40) --------------------------------------
void sample_actions(DataStore& store, const double* logits, int64_t logits_count,
                    int64_t num_categories, int64_t num_choices, int64_t step, uint64_t seed) {
  const int64_t E = store.num_envs(), A = store.num_agents();
  if (num_categories < 1 || num_choices < 1) {
    raise(Errc::invalid_argument, "sample_actions: categories and choices must be >= 1");
  }
  const int64_t expected = E * A * num_categories * num_choices;
  if (logits_count != expected) {
    raise(Errc::shape_mismatch, "sample_actions: logits size " + std::to_string(logits_count) +
                                    ", expected " + std::to_string(expected));
  }
  if (logits == nullptr) raise(Errc::invalid_argument, "sample_actions: null logits");
  const int32_t h = store.handle(kSampledActions);
  if (store.info(h).env_stride != A * num_categories) {
    raise(Errc::shape_mismatch, "sample_actions: \"sampled_actions\" shape does not match "
                                "[envs, agents, categories]");
  }
  // Finiteness scan before any write, as the reference does.
  uint32_t* flag = nullptr;
  cuda_check(cudaMalloc(&flag, sizeof(uint32_t)), "cudaMalloc(flag)");
  uint32_t host_flag = 0;
  cudaError_t err = cudaMemsetAsync(flag, 0, sizeof(uint32_t), store.stream());
  if (err == cudaSuccess) err = launch_finite_scan(logits, expected, flag, store.stream());
  if (err == cudaSuccess)
    err = cudaMemcpyAsync(&host_flag, flag, sizeof(uint32_t), cudaMemcpyDeviceToHost, store.stream());
  if (err == cudaSuccess) err = cudaStreamSynchronize(store.stream());
  cudaFree(flag);
  cuda_check(err, "sample_actions finiteness scan");
  if (host_flag) raise(Errc::non_finite, "sample_actions: non-finite logit");
  const uint64_t h_step = host_absorb(host_mix64(host_substream(seed, kStreamActions)),
                                      static_cast<uint64_t>(step));
  cuda_check(launch_sample(logits, static_cast<int32_t*>(store.device_ptr(h)),
                           E * A * num_categories, static_cast<int>(A),
                           static_cast<int>(num_categories), static_cast<int>(num_choices),
                           store.env_offset(), h_step, store.stream()),
             "sample kernel");
}

// ---- ResetManager (reset_manager.cpp:5-51) ----------------------------------
ResetManager::ResetManager(DataStore& store, bool auto_reset, std::vector<std::string> zero_on_reset,
                           TagPlan* reinit)
    : store_(store), auto_(auto_reset), reinit_(reinit) {
  (void)store.handle(kDone);
  for (const std::string& name : zero_on_reset) {
    const int32_t h = store.handle(name);  // throws unknown_name
    if (store.info(h).spec.snapshot_on_reset) {
      raise(Errc::invalid_argument,
            "ResetPolicy: \"" + name + "\" is snapshot_on_reset and cannot also be zero-filled");
    }
    zero_handles_.push_back(h);
  }
  if (reinit_ != nullptr && &reinit_->store() != &store_) {
    raise(Errc::invalid_argument, "ResetPolicy: reinit plan belongs to another store");
  }
  // Descriptor table: every snapshot array restores, listed arrays zero-fill.
  std::vector<ResetRowDesc> descs;
  for (int32_t h = 0; h < store.num_arrays(); ++h) {
    if (store.info(h).spec.snapshot_on_reset) {
      descs.push_back({static_cast<uint8_t*>(store.device_ptr(h)),
                       static_cast<const uint8_t*>(store.snapshot_ptr(h)), store.row_bytes(h)});
    }
  }
  for (int32_t h : zero_handles_) {
    descs.push_back({static_cast<uint8_t*>(store.device_ptr(h)), nullptr, store.row_bytes(h)});
  }
  ndesc_ = static_cast<int32_t>(descs.size());
  if (ndesc_ > 0) {
    cuda_check(cudaMalloc(&descs_, descs.size() * sizeof(ResetRowDesc)), "cudaMalloc(reset descs)");
    cuda_check(cudaMemcpy(descs_, descs.data(), descs.size() * sizeof(ResetRowDesc),
                          cudaMemcpyHostToDevice),
               "reset descs upload");
  }
  cuda_check(cudaMalloc(&episode_, static_cast<size_t>(store.num_envs()) * sizeof(int32_t)),
             "cudaMalloc(episode)");
  cuda_check(cudaMemset(episode_, 0, static_cast<size_t>(store.num_envs()) * sizeof(int32_t)),
             "episode clear");
  // Fused-kernel eligibility: exactly the Tag policy.
  std::set<std::string> want;
  for (const std::string& n : tag_zero_on_reset()) want.insert(n);
  std::set<std::string> have(zero_on_reset.begin(), zero_on_reset.end());
  tag_default_ = reinit_ != nullptr && want == have;
}

ResetManager::~ResetManager() {
  if (descs_) cudaFree(descs_);
  if (episode_) cudaFree(episode_);
}

std::vector<int64_t> ResetManager::detect_done() const {  // reset_manager.cpp:20-27
  const int64_t E = store_.num_envs();
  std::vector<uint8_t> done(static_cast<size_t>(E));
  store_.pull(store_.handle(kDone), 0, E, done.data(), E);
  std::vector<int64_t> ids;
  for (int64_t e = 0; e < E; ++e)
    if (done[static_cast<size_t>(e)]) ids.push_back(e);
  return ids;
}

void ResetManager::reset_masked() {
  uint8_t* mask = store_.env_mask();
  uint8_t* done = static_cast<uint8_t*>(store_.device_ptr(store_.handle(kDone)));
  cuda_check(launch_restore_zero(static_cast<const ResetRowDesc*>(descs_), ndesc_, mask, done,
                                 episode_, store_.num_envs(), store_.stream()),
             "auto_reset restore/zero");
  if (reinit_) reinit_->reinit_masked(mask, episode_);
}

void ResetManager::auto_reset(const int64_t* env_ids, int64_t count) {  // reset_manager.cpp:29-44
  if (count == 0) return;
  const int64_t E = store_.num_envs();
  for (int64_t i = 0; i < count; ++i) {
    if (env_ids[i] < 0 || env_ids[i] >= E) {
      raise(Errc::index_out_of_range, "env_id " + std::to_string(env_ids[i]) + " out of range [0, " +
                                          std::to_string(E) + ")");
    }
  }
  uint8_t* mask = store_.env_mask();
  int64_t* ids = store_.id_buffer(count);
  cuda_check(cudaMemcpyAsync(ids, env_ids, static_cast<size_t>(count) * sizeof(int64_t),
                             cudaMemcpyHostToDevice, store_.stream()),
             "auto_reset ids");
  cuda_check(cudaMemsetAsync(mask, 0, static_cast<size_t>(E), store_.stream()), "mask clear");
  cuda_check(launch_mask_from_ids(ids, count, mask, store_.stream()), "mask_from_ids");
  reset_masked();
  store_.synchronize();  // ids buffer is reused by the next call
}

void ResetManager::auto_reset_on_done() {
  uint8_t* mask = store_.env_mask();
  const uint8_t* done = static_cast<const uint8_t*>(store_.device_ptr(store_.handle(kDone)));
  cuda_check(launch_mask_from_done(done, mask, store_.num_envs(), store_.stream()), "mask_from_done");
  reset_masked();
}

int64_t ResetManager::episodes_started(int64_t env_id) const {
  if (env_id < 0 || env_id >= store_.num_envs()) {
    raise(Errc::index_out_of_range, "episodes_started: env_id out of range");
  }
  int32_t v = 0;
  cuda_check(cudaMemcpyAsync(&v, episode_ + env_id, sizeof(int32_t), cudaMemcpyDeviceToHost,
                             store_.stream()),
             "episodes_started");
  store_.synchronize();
  return v;
}

// ---- Rollout driver (harness.cpp:428-505) ----------------------------------
Rollout::Rollout(DataStore& store, TagPlan& plan, ResetManager* resets, uint64_t sample_seed)
    : store_(store), plan_(plan), resets_(resets), seed_(sample_seed) {
  if (&plan.store() != &store) raise(Errc::invalid_argument, "rollout: plan belongs to another store");
  const TagDevConfig& p = plan.dev();
  const int64_t n_logits = int64_t{p.E} * p.A * p.C * p.V;
  // Zero logits = uniform policy (harness.cpp:439,446-447).
  cuda_check(cudaMalloc(&zero_logits_, static_cast<size_t>(n_logits) * sizeof(double)),
             "cudaMalloc(zero logits)");
  cuda_check(cudaMemset(zero_logits_, 0, static_cast<size_t>(n_logits) * sizeof(double)),
             "zero logits");
  cuda_check(cudaMalloc(&env_stats_, static_cast<size_t>(p.E) * 8 * sizeof(double)),
             "cudaMalloc(env stats)");
  cuda_check(cudaMemset(env_stats_, 0, static_cast<size_t>(p.E) * 8 * sizeof(double)),
             "env stats clear");
  cuda_check(cudaMalloc(&stats_, WDG_STAT_COUNT * sizeof(double)), "cudaMalloc(stats)");
  cuda_check(cudaMemset(stats_, 0, WDG_STAT_COUNT * sizeof(double)), "stats clear");
  cuda_check(cudaMalloc(&error_, sizeof(uint32_t)), "cudaMalloc(error)");
  cuda_check(cudaMemset(error_, 0, sizeof(uint32_t)), "error clear");
  if (resets_ == nullptr) {
    cuda_check(cudaMalloc(&own_episode_, static_cast<size_t>(p.E) * sizeof(int32_t)),
               "cudaMalloc(episode)");
    cuda_check(cudaMemset(own_episode_, 0, static_cast<size_t>(p.E) * sizeof(int32_t)),
               "episode clear");
  }
  logits_ = zero_logits_;
  h_actions0_ = host_mix64(host_substream(seed_, kStreamActions));
  pdl_flags_ = store_.pdl_flags();  // set_overlap(false): one plain launch per step
}

Rollout::~Rollout() {
  drop_graph();
  if (step_dev_) cudaFree(step_dev_);
  for (int i = 0; i < 2; ++i) {
    if (dlog_[i]) cudaFree(dlog_[i]);
    if (slot_free_[i]) cudaEventDestroy(slot_free_[i]);
  }
  for (int i = 0; i < kMaxHostChunks; ++i) {
    if (h2d_ev_[i]) cudaEventDestroy(h2d_ev_[i]);
    if (kern_ev_[i]) cudaEventDestroy(kern_ev_[i]);
  }
  if (d2h_ev_) cudaEventDestroy(d2h_ev_);
  if (rew_cap_) cudaFree(rew_cap_);
  if (done_cap_) cudaFree(done_cap_);
  if (copy_) cudaStreamDestroy(copy_);
  if (d2h_) cudaStreamDestroy(d2h_);
  if (zero_logits_) cudaFree(zero_logits_);
  if (pol_logits_) cudaFree(pol_logits_);
  if (pol_values_) cudaFree(pol_values_);
  if (env_stats_) cudaFree(env_stats_);
  if (stats_) cudaFree(stats_);
  if (error_) cudaFree(error_);
  if (own_episode_) cudaFree(own_episode_);
}

void Rollout::set_overlap(bool enabled) {
  uint32_t* want = enabled ? store_.pdl_flags() : nullptr;
  if (want != pdl_flags_) drop_graph();  // captured with or without overlapped nodes
  pdl_flags_ = want;
}

void Rollout::set_logits(const double* logits, int64_t count) {
  if (pol_[0] != nullptr) {  // explicit logits replace the device policies
    pol_[0] = pol_[1] = nullptr;
    ++pol_version_;
  }
  if (logits == nullptr) {
    logits_ = zero_logits_;
    return;
  }
  const TagDevConfig& p = plan_.dev();
  const int64_t expected = int64_t{p.E} * p.A * p.C * p.V;
  if (count != expected) {
    raise(Errc::shape_mismatch, "rollout: logits size " + std::to_string(count) + ", expected " +
                                    std::to_string(expected));
  }
  logits_ = logits;
}

bool Rollout::fused_ok() const {
  return fused_ && !plan_.reference() && (resets_ == nullptr || !resets_->auto_enabled() ||
                    (resets_->tag_default() && resets_->reinit_plan() == &plan_));
}

TagLaunch Rollout::fused_launch(int64_t step) const {
  TagLaunch L;
  L.mode = kModeFused;
  L.do_reset = (resets_ != nullptr && resets_->auto_enabled()) ? 1 : 0;
  L.track = 1;
  L.action_h_step = host_absorb(h_actions0_, static_cast<uint64_t>(step));
  L.logits = policy_samples() ? nullptr : logits_;  // bf16 policies sampled already
  L.episode = resets_ ? resets_->episode_device() : own_episode_;
  L.env_stats = env_stats_;
  L.error = error_;
#ifdef WDG_TUNING
  // Performance-analysis ablation (results invalid; tuning builds only, the
  // product kernel ignores TagLaunch::ablate).
  static const uint32_t ablate = [] {
    const char* v = std::getenv("WDG_ABLATE");
    return v ? static_cast<uint32_t>(std::strtoul(v, nullptr, 0)) : 0u;
  }();
  L.ablate = ablate;
#endif
  return L;
}

void Rollout::set_policies(const Policy* tagger, const Policy* runner, int32_t precision) {
  if ((tagger == nullptr) != (runner == nullptr)) {
    raise(Errc::invalid_argument, "set_policies: give both policies or neither");
  }
  const TagDevConfig& p = plan_.dev();
  if (tagger != nullptr) {
    for (const Policy* q : {tagger, runner}) {
      const PolicyDims& d = q->dims();
      if (d.obs_dim != p.D || d.num_categories != p.C || d.num_choices != p.V) {
        raise(Errc::shape_mismatch, "set_policies: policy dims do not match the Tag config (obs_dim " +
                                        std::to_string(p.D) + ", C " + std::to_string(p.C) + ", V " +
                                        std::to_string(p.V) + ")");
      }
    }
    if (precision != kPolicyF64 && precision != kPolicyBF16) {
      raise(Errc::invalid_argument, "set_policies: unknown precision");
    }
    if (precision == kPolicyBF16 && (!tagger->bf16_supported() || !runner->bf16_supported())) {
      raise(Errc::invalid_config, "set_policies: the bf16 tensor-core path needs hidden {64, 64}");
    }
    if (pol_logits_ == nullptr) {
      const size_t n = static_cast<size_t>(p.E) * p.A;
      cuda_check(cudaMalloc(&pol_logits_, n * p.C * p.V * sizeof(double)), "cudaMalloc(policy logits)");
      cuda_check(cudaMalloc(&pol_values_, n * sizeof(double)), "cudaMalloc(policy values)");
    }
    logits_ = pol_logits_;
  } else {
    logits_ = zero_logits_;
  }
  pol_[0] = tagger;
  pol_[1] = runner;
  pol_prec_ = precision;
  ++pol_version_;
}

// forward_policies (harness.cpp:445-476): obs (already in HBM) -> f64 logits,
// or (bf16) the tensor-core forward fused with sample_actions for step t ->
// sampled actions, which the fused env launch then reads (L.logits == nullptr).
// values_out / force_logits / sample serve the rollout capture (collect).
void Rollout::forward_policies(cudaStream_t st, int64_t step, const int64_t* step_dev, int32_t step_add,
                               double* values_out, bool force_logits, bool sample) {
  if (pol_[0] == nullptr) return;
  if (step_dev == nullptr) launches_ += pol_[0] == pol_[1] ? 1 : 2;
  const TagDevConfig& p = plan_.dev();
  const float* obs = static_cast<const float*>(store_.device_ptr(store_.handle(kObservations)));
  // f64 logits are the sampler's input (always written); bf16 samples in the
  // epilogue and stores logits / values only when asked to keep them.
  double* lg = (pol_prec_ == kPolicyBF16 && !keep_outputs_ && !force_logits) ? nullptr : pol_logits_;
  double* vl = values_out ? values_out : (keep_outputs_ ? pol_values_ : nullptr);
  if (pol_prec_ == kPolicyBF16) {
    SampleKeys k;
    k.env_offset = p.env_offset;
    k.h_step = host_absorb(h_actions0_, static_cast<uint64_t>(step));
    k.step_dev = step_dev;
    k.step_add = step_add;
    k.h0 = h_actions0_;
    int32_t* act = sample ? static_cast<int32_t*>(store_.device_ptr(store_.handle(kSampledActions))) : nullptr;
    const bool pdl = pdl_flags_ != nullptr;  // set_overlap(false) off switch
    if (pol_[0] == pol_[1]) {
      pol_[0]->forward_sample_bf16(obs, p.E, p.A, 0, p.A, act, lg, vl, k, st, error_, pdl);
    } else {
      pol_[0]->forward_sample_bf16(obs, p.E, p.A, 0, p.T, act, lg, vl, k, st, error_, pdl);
      pol_[1]->forward_sample_bf16(obs, p.E, p.A, p.T, p.A, act, lg, vl, k, st, error_, pdl);
    }
    if (pdl && step_dev == nullptr) store_.set_pdl_open(true);  // released at entry, no env flags
    return;
  }
  if (pol_[0] == pol_[1]) {
    pol_[0]->forward_agents(obs, p.E, p.A, 0, p.A, lg, vl, pol_prec_, st, error_);
  } else {
    pol_[0]->forward_agents(obs, p.E, p.A, 0, p.T, lg, vl, pol_prec_, st, error_);
    pol_[1]->forward_agents(obs, p.E, p.A, p.T, p.A, lg, vl, pol_prec_, st, error_);
  }
}

// Trainer::collect (trainer.cpp:315-403) on device: T steps of the policy
// rollout, each captured into slot t of the batch —
//   policy_forward(t): obs before the step, values of the forward;
//   sample(t):         sampled actions, active flags at sample time, logp;
//   post_step(t):      rewards and done of the step (before reset-on-done);
// then the bootstrap values of the final observations.
void Rollout::collect(RolloutBatch& b) {
  const TagDevConfig& p = plan_.dev();
  if (pol_[0] == nullptr) raise(Errc::state_error, "collect: set the policies first (Trainer::collect runs them)");
  if (!fused_ok()) raise(Errc::state_error, "collect: needs the fused step with the Tag reset policy");
  if (b.E != p.E || b.A != p.A || b.D != p.D || b.C != p.C) {
    raise(Errc::shape_mismatch, "collect: batch dims do not match the store / Tag config");
  }
  cudaStream_t st = store_.stream();
  const float* obs = static_cast<const float*>(store_.device_ptr(store_.handle(kObservations)));
  const int64_t EA = int64_t{p.E} * p.A;
  for (int64_t t = 0; t < b.T; ++t) {
    cuda_check(cudaMemcpyAsync(b.obs + t * EA * p.D, obs, static_cast<size_t>(EA * p.D) * sizeof(float),
                               cudaMemcpyDeviceToDevice, st),
               "collect obs");
    forward_policies(st, t_, nullptr, 0, b.values + t * EA, true, true);
    TagLaunch L = fused_launch(t_);
    L.cap_actions = b.actions + t * EA * p.C;
    L.cap_active = b.active + t * EA;
    L.cap_rewards = b.rewards + t * EA;
    L.cap_done = b.done + t * p.E;
    plan_.launch(L);
    launch_logp(pol_logits_, b.actions + t * EA * p.C, b.logp + t * EA, EA, p.C, p.V, st);
    ++t_;
  }
  forward_policies(st, t_, nullptr, 0, b.bootstrap, true, false);
}

void Rollout::step_unfused(float* cap_rewards, uint8_t* cap_done) {
  const TagDevConfig& p = plan_.dev();
  const uint64_t h_step = host_absorb(h_actions0_, static_cast<uint64_t>(t_));
  if (!policy_samples()) cuda_check(launch_sample(logits_,
                           static_cast<int32_t*>(store_.device_ptr(store_.handle(kSampledActions))),
                           int64_t{p.E} * p.A * p.C, p.A, p.C, p.V, p.env_offset, h_step,
                           store_.stream()),
             "sample kernel");
  plan_.run_step(t_);
  if (cap_rewards != nullptr) {  // before reset-on-done zeroes them
    cuda_check(cudaMemcpyAsync(cap_rewards, store_.device_ptr(store_.handle(kRewards)),
                               static_cast<size_t>(p.E) * p.A * sizeof(float), cudaMemcpyDeviceToDevice,
                               store_.stream()),
               "capture rewards");
  }
  if (cap_done != nullptr) {
    cuda_check(cudaMemcpyAsync(cap_done, store_.device_ptr(store_.handle(kDone)), static_cast<size_t>(p.E),
                               cudaMemcpyDeviceToDevice, store_.stream()),
               "capture done");
  }
  if (resets_ != nullptr && resets_->auto_enabled()) resets_->auto_reset_on_done();
  store_.set_pdl_open(false);  // plain launches: each waits for its predecessor to finish
  launches_ += policy_samples() ? 1 : 2;  // (+ the reset kernels, counted in the ResetManager's own launches)
}

// Consecutive fused launches overlap through programmatic dependent launch
// (per-env waits, TagLaunch::env_seq). Not with device policies (every step
// is serialised behind the policy kernels anyway), and not while the stream
// is being captured into someone's graph: the sequence numbers would be baked
// in and replays would not wait.
void Rollout::set_pdl(TagLaunch& L, bool single_step) const {
  const int mode = plan_.pdl_mode();
  if (pol_[0] != nullptr && pdl_flags_ != nullptr && pol_prec_ == kPolicyBF16) {
    L.pdl_wait = 1;  // behind the bf16 policy kernels: plain PDL (prologue overlap only)
    return;
  }
  if (pol_[0] != nullptr || pdl_flags_ == nullptr || mode == 0) return;
  if (mode == 3) {  // plain PDL: next launch released at entry, griddepcontrol.wait, no flags
    L.pdl_wait = single_step ? 1 : 0;  // neutral to worse for multi-step windows and graphs
    return;
  }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(store_.stream(), &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return;
  }
  L.env_seq = pdl_flags_;
  L.seq = store_.pdl_seq() + 1u;
  L.pdl_late = mode == 2 ? 1 : 0;
  // The previous kernel released this launch early without publishing flags
  // (bf16 policy step, collect's bootstrap forward): wait for all of it first.
  if (store_.pdl_open()) L.pdl_wait = 1;
}

// After a Tag launch: did it release its dependents without publishing env
// flags (DataStore::pdl_open)?
void Rollout::note_launch(const TagLaunch& L) {
  if (L.env_seq != nullptr) store_.commit_pdl_seq();
  store_.set_pdl_open(L.env_seq == nullptr && L.pdl_wait != 0);
}

void Rollout::step() {
  forward_policies(store_.stream(), t_, nullptr, 0, nullptr, false, true);
  if (fused_ok()) {
    TagLaunch L = fused_launch(t_);
    set_pdl(L, true);
    plan_.launch(L);
    note_launch(L);
    ++launches_;
  } else {
    step_unfused();
  }
  ++t_;
}

// Host-driven step (the drop-in host integration): what a host learner reads
// after RolloutDriver::step — the step's rewards and done captured BEFORE
// reset-on-done (Trainer::collect post_step, trainer.cpp:382-394, ahead of
// auto_reset, harness.cpp:478-490) and, optionally, the observations after it
// (post-reset: what the next policy_forward reads, trainer.cpp:358-360).
// The step is pipelined over env chunks on three streams: the H2D of chunk
// g + 1's logits, the fused kernel of chunk g and the D2H of chunk g - 1's
// outputs overlap (PCIe is full duplex), so a closed-loop step costs about
// max(H2D, D2H) instead of their sum. Every chunk uses the step's index and
// global env ids, so the results equal one whole-store launch.
void Rollout::step_host(const double* host_logits, int64_t count, float* host_rewards,
                        uint8_t* host_done, float* host_obs, int64_t obs_count) {
  const TagDevConfig& p = plan_.dev();
  const int64_t per_env_logits = int64_t{p.A} * p.C * p.V;
  const int64_t expected = int64_t{p.E} * per_env_logits;
  if (host_logits == nullptr) raise(Errc::invalid_argument, "step_host: null logits");
  if (pol_[0] != nullptr) raise(Errc::state_error, "step_host: the rollout samples from device policies");
  if (count != expected) {
    raise(Errc::shape_mismatch, "step_host: logits size " + std::to_string(count) + ", expected " +
                                    std::to_string(expected));
  }
  if (host_obs != nullptr && obs_count != int64_t{p.E} * p.A * p.D) {
    raise(Errc::shape_mismatch, "step_host: observations size " + std::to_string(obs_count) +
                                    ", expected " + std::to_string(int64_t{p.E} * p.A * p.D));
  }
  const size_t bytes = static_cast<size_t>(expected) * sizeof(double);
  if (copy_ == nullptr) {
    cuda_check(cudaStreamCreateWithFlags(&copy_, cudaStreamNonBlocking), "copy stream");
    cuda_check(cudaStreamCreateWithFlags(&d2h_, cudaStreamNonBlocking), "d2h stream");
    for (int i = 0; i < 2; ++i) {
      cuda_check(cudaMalloc(&dlog_[i], bytes), "cudaMalloc(logits slot)");
      cuda_check(cudaEventCreateWithFlags(&slot_free_[i], cudaEventDisableTiming), "event");
    }
    for (int i = 0; i < kMaxHostChunks; ++i) {
      cuda_check(cudaEventCreateWithFlags(&h2d_ev_[i], cudaEventDisableTiming), "event");
      cuda_check(cudaEventCreateWithFlags(&kern_ev_[i], cudaEventDisableTiming), "event");
    }
    cuda_check(cudaEventCreateWithFlags(&d2h_ev_, cudaEventDisableTiming), "event");
    cuda_check(cudaMalloc(&rew_cap_, static_cast<size_t>(p.E) * p.A * sizeof(float)), "cudaMalloc(rewards capture)");
    cuda_check(cudaMalloc(&done_cap_, static_cast<size_t>(p.E)), "cudaMalloc(done capture)");
  }
  const bool fused = fused_ok();
  // Chunks: ~8 MB of logits each (C2: 8 chunks of 250 envs), whole CTAs.
  int chunks = host_chunks_ > 0 ? host_chunks_
                                : static_cast<int>(std::clamp<int64_t>(static_cast<int64_t>(bytes >> 23), 1, kMaxHostChunks));
  if (!fused) chunks = 1;
  // chunk boundaries on whole CTAs and on 16-byte boundaries of the
  // observation rows (the kernels store them as 16-byte vectors from the
  // chunk's first row): e0 * A * D % 4 == 0
  const int64_t row_floats = int64_t{p.A} * p.D;
  const int64_t align = std::lcm<int64_t>(4 / std::gcd<int64_t>(row_floats, 4), 4 / std::gcd<int64_t>(p.A, 4));
  const int64_t unit = std::lcm<int64_t>(p.envs_per_cta, align);
  const int64_t per = (int64_t{p.E} + chunks - 1) / chunks;
  const int64_t per_chunk = std::max<int64_t>(unit, (per + unit - 1) / unit * unit);
  const int slot = static_cast<int>(t_ & 1);
  cudaStream_t st = store_.stream();
  // The slot was last read by the kernels of step t-2.
  cuda_check(cudaStreamWaitEvent(copy_, slot_free_[slot], 0), "wait slot");
  int g = 0;
  for (int64_t e0 = 0; e0 < p.E; e0 += per_chunk, ++g) {
    const int64_t n = std::min<int64_t>(per_chunk, p.E - e0);
    cuda_check(cudaMemcpyAsync(dlog_[slot] + e0 * per_env_logits, host_logits + e0 * per_env_logits,
                               static_cast<size_t>(n * per_env_logits) * sizeof(double),
                               cudaMemcpyHostToDevice, copy_),
               "H2D logits");
    cuda_check(cudaEventRecord(h2d_ev_[g], copy_), "record h2d");
  }
  g = 0;
  for (int64_t e0 = 0; e0 < p.E; e0 += per_chunk, ++g) {
    const int64_t n = std::min<int64_t>(per_chunk, p.E - e0);
    cuda_check(cudaStreamWaitEvent(st, h2d_ev_[g], 0), "wait h2d");
    if (fused) {
      TagLaunch L = fused_launch(t_);
      L.logits = dlog_[slot];
      L.cap_rewards = rew_cap_;
      L.cap_done = done_cap_;
      plan_.launch_envs(L, e0, n);  // plain launch: waits for its stream predecessors
      ++launches_;
    } else {
      const double* saved = logits_;
      logits_ = dlog_[slot];
      try {
        step_unfused(rew_cap_, done_cap_);
      } catch (...) {
        logits_ = saved;
        throw;
      }
      logits_ = saved;
    }
    cuda_check(cudaEventRecord(kern_ev_[g], st), "record kernel");
    cuda_check(cudaStreamWaitEvent(d2h_, kern_ev_[g], 0), "wait kernel");
    if (host_rewards) {
      cuda_check(cudaMemcpyAsync(host_rewards + e0 * p.A, rew_cap_ + e0 * p.A,
                                 static_cast<size_t>(n * p.A) * sizeof(float), cudaMemcpyDeviceToHost, d2h_),
                 "D2H rewards");
    }
    if (host_done) {
      cuda_check(cudaMemcpyAsync(host_done + e0, done_cap_ + e0, static_cast<size_t>(n), cudaMemcpyDeviceToHost,
                                 d2h_),
                 "D2H done");
    }
    if (host_obs) {
      const int64_t row = int64_t{p.A} * p.D;
      const float* obs = static_cast<const float*>(store_.device_ptr(store_.handle(kObservations)));
      cuda_check(cudaMemcpyAsync(host_obs + e0 * row, obs + e0 * row, static_cast<size_t>(n * row) * sizeof(float),
                                 cudaMemcpyDeviceToHost, d2h_),
                 "D2H observations");
    }
  }
  cuda_check(cudaEventRecord(slot_free_[slot], st), "record slot");
  // The store stream waits for the copies: wdg_store_synchronize covers the
  // outputs, and the next step's kernels (which rewrite them) follow them.
  cuda_check(cudaEventRecord(d2h_ev_, d2h_), "record d2h");
  cuda_check(cudaStreamWaitEvent(st, d2h_ev_, 0), "wait d2h");
  store_.set_pdl_open(false);
  ++t_;
}

void Rollout::reduce_stats_into(double* device_out) {
  if (device_out == nullptr) raise(Errc::invalid_argument, "reduce_stats_into: null output");
  cuda_check(launch_stats_reduce(env_stats_, plan_.dev().E, device_out, store_.stream()), "stats reduce");
}

void Rollout::drop_graph() {
  if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
  graph_exec_ = nullptr;
}

// Captures kGraphSteps fused launches whose step index is read on device as
// *step_dev_ + i, so one instantiated graph replays any window of steps.
void Rollout::build_graph() {
  drop_graph();
  // [0] = first step of the window, [1] = sequence number before it (PDL)
  if (step_dev_ == nullptr) cuda_check(cudaMalloc(&step_dev_, 2 * sizeof(int64_t)), "cudaMalloc(step)");
  cudaStream_t st = store_.stream();
  cudaStream_t cap = st;
  bool own = false;
  if (cap == nullptr) {  // the legacy default stream cannot be captured
    cuda_check(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "capture stream");
    own = true;
  }
  const int graph_mode = plan_.pdl_mode();
  graph_pdl_ = pol_[0] == nullptr && pdl_flags_ != nullptr && graph_mode != 0 && graph_mode != 3;
  // Plain PDL between the captured nodes (programmatic edges, whole-grid
  // griddepcontrol.wait, no flags) for the plans whose direct launches use it
  // (pdl_mode 3: packed small envs such as C4), when the grid holds at most
  // one warp per SM scheduler. C4 single-step replay, us/step with / without
  // (4096-step windows, tools/c4_graph_ab.py): E = 1 4.14 / 4.54, 1000 4.50 /
  // 4.78, 2000 4.61 / 4.88, 3000 4.68 / 4.87 (500 warps); 5000 5.13 / 5.02
  // (834 warps), 7000 5.37 / 5.13, 10000 5.92 / 5.45.
  const TagDevConfig& gd = plan_.dev();
  graph_plain_pdl_ = pol_[0] == nullptr && pdl_flags_ != nullptr && graph_mode == 3 &&
                     static_cast<int64_t>(gd.grid_ctas) * gd.threads / 32 <= 4 * kNumSMs;
  cuda_check(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal), "begin capture");
  cudaError_t err = cudaSuccess;
  for (int i = 0; i < kGraphSteps && err == cudaSuccess; ++i) {
    if (pol_[0] != nullptr) {
      try {
        forward_policies(cap, 0, step_dev_, i, nullptr, false, true);
      } catch (const Error&) {
        err = cudaErrorUnknown;
        break;
      }
    }
    TagLaunch L = fused_launch(0);
    L.step_dev = step_dev_;
    L.step_add = i;
    L.action_h0 = h_actions0_;
    if (graph_plain_pdl_) L.pdl_wait = 1;
    if (graph_pdl_) {  // overlapped nodes (programmatic edges)
      L.env_seq = pdl_flags_;
      L.seq_dev = step_dev_ + 1;
      L.seq_add = static_cast<uint32_t>(i + 1);
      L.pdl_late = graph_mode == 2 ? 1 : 0;
    }
    TagDevConfig d = plan_.dev();
    d.fault_bias = fault_tag_radius_bias();
    err = launch_tag_kernel(d, bind_dev_arrays(store_, plan_.config()), L, cap);
  }
  cudaGraph_t graph = nullptr;
  const cudaError_t end = cudaStreamEndCapture(cap, &graph);
  if (own) cudaStreamDestroy(cap);
  cuda_check(err, "graph capture launch");
  cuda_check(end, "end capture");
  err = cudaGraphInstantiate(&graph_exec_, graph, 0);
  cudaGraphDestroy(graph);
  cuda_check(err, "graph instantiate");
  graph_logits_ = logits_;
  graph_pol_version_ = pol_version_;
  graph_bias_ = fault_tag_radius_bias();
  graph_stream_ = st;
}

void Rollout::run(int64_t steps) {
  if (steps < 0) raise(Errc::invalid_argument, "rollout run: steps must be >= 0");
  // Multi-step residency: with a fixed logits buffer (no policy between
  // steps) consecutive steps are independent launches of the same kernel on
  // the same env, so one launch runs up to kMultiSteps of them with each
  // env's state kept in shared memory (TagLaunch::n_steps).
  const bool multi_off = tuning("multistep", 1) == 0;  // read per run() (A/B timing in one process)
  if (!multi_off && fused_ok() && pol_[0] == nullptr && steps > 1 && plan_.multistep_ok()) {
    while (steps > 0) {
      const int32_t k = static_cast<int32_t>(std::min<int64_t>(steps, kMultiSteps));
      TagLaunch L = fused_launch(t_);
      L.n_steps = k;
      L.step0 = t_;
      L.action_h0 = h_actions0_;
      set_pdl(L, false);  // the next window's early envs start in this one's tail
      plan_.launch(L);
      note_launch(L);
      ++launches_;
      t_ += k;
      steps -= k;
    }
    return;
  }
  // LEAN plans: direct overlapped launches (107 us/step at C2) beat the graph
  // replay of the same launches (111 us/step).
  if (graphs_ && fused_ok() && steps >= kGraphSteps && !(lean_plan(plan_.dev()) && pdl_flags_ != nullptr)) {
    if (graph_exec_ == nullptr || graph_logits_ != logits_ || graph_pol_version_ != pol_version_ ||
        graph_bias_ != fault_tag_radius_bias() ||
        graph_stream_ != store_.stream()) {
      build_graph();
    }
    const bool graph_pdl = graph_pdl_;  // as captured (flag sequence numbers)
    while (steps >= kGraphSteps) {
      cuda_check(launch_set_counter(step_dev_, t_, store_.stream(),
                                    graph_pdl ? static_cast<int64_t>(store_.pdl_seq()) : -1),
                 "set step counter");
      cuda_check(cudaGraphLaunch(graph_exec_, store_.stream()), "graph launch");
      if (graph_pdl)
        for (int i = 0; i < kGraphSteps; ++i) store_.commit_pdl_seq();
      // the last node is a Tag launch that publishes its flags, never releases
      // early, or (plain PDL) releases early without flags
      store_.set_pdl_open(graph_plain_pdl_);
      launches_ += 1 + kGraphSteps * (pol_[0] != nullptr ? (pol_[0] == pol_[1] ? 2 : 3) : 1);
      t_ += kGraphSteps;
      steps -= kGraphSteps;
    }
  }
  for (int64_t i = 0; i < steps; ++i) step();
}

void Rollout::check() {
  uint32_t err = 0;
  cuda_check(cudaMemcpyAsync(&err, error_, sizeof(uint32_t), cudaMemcpyDeviceToHost, store_.stream()),
             "rollout check");
  store_.synchronize();
  if (err & kErrNonFinite) {
    cudaMemsetAsync(error_, 0, sizeof(uint32_t), store_.stream());
    raise(Errc::non_finite, "sample_actions: non-finite logit (fused rollout)");
  }
  if (err & kErrStepOrder) {
    cudaMemsetAsync(error_, 0, sizeof(uint32_t), store_.stream());
    store_.synchronize();
    store_.reset_pdl();
    raise(Errc::cuda, "fused rollout: an overlapped step timed out waiting for the previous step; "
                      "the affected envs skipped it (state is no longer in lockstep)");
  }
}

void Rollout::stats(double* out, int32_t count) {
  cuda_check(launch_stats_reduce(env_stats_, plan_.dev().E, stats_, store_.stream()), "stats reduce");
  double host[WDG_STAT_COUNT];
  cuda_check(cudaMemcpyAsync(host, stats_, sizeof(host), cudaMemcpyDeviceToHost, store_.stream()),
             "stats pull");
  store_.synchronize();
  for (int32_t i = 0; i < count && i < WDG_STAT_COUNT; ++i) out[i] = host[i];
  check();  // surface sticky device errors at this synchronising call
}

void Rollout::reset_stats() {
  cuda_check(cudaMemsetAsync(env_stats_, 0, static_cast<size_t>(plan_.dev().E) * 8 * sizeof(double),
                             store_.stream()),
             "stats clear");
}

double* Rollout::stats_device() {
  cuda_check(launch_stats_reduce(env_stats_, plan_.dev().E, stats_, store_.stream()), "stats reduce");
  return stats_;
}

}  // namespace wdg
