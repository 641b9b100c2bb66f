// tag_kernels.cu — sm_100a kernels for the WarpDrive Tag env-step hot path.
//
// One kernel body, three launch modes (tag_params.hpp TagMode):
//   kModeStep   StepEngine::run_step over the Tag plan (tag_env.cpp:363-480):
//               move -> resolve_tags -> observe_reward, phase barriers become
//               __syncthreads (step_engine.cpp:100-120).
//   kModeFused  RolloutDriver::step (harness.cpp:478-490) in ONE launch:
//               sample_actions (sampler.cpp:5-40) -> step -> EpisodeTracker
//               (trainer.cpp:229-252) -> reset-on-done (reset_manager.cpp:29-44
//               + make_tag_reinit, tag_env.cpp:482-500).
//   kModeReinit make_tag_reinit / episode-0 registration (tag_env.cpp:280-341)
//               for masked envs.
//
// Mapping: one CTA per environment and one thread per agent (A > 1024 loops);
// for small A several environments share a CTA (env packing). Per-env agent
// state is staged in shared memory once per step; the bucket grid for K-NN and
// tag resolution is a counting sort in shared memory. All outputs are written
// coalesced: per-agent scalars one element per lane, observations as the
// CTA's contiguous [envs, A, D] block, 16-byte vector streaming stores.
//
// Numerics: compiled with -fmad=false so no a*b+c is contracted, as the
// reference forbids (proj/CMakeLists.txt:10-13); discrete results are
// bit-identical to the CPU path. The sampler runs in f64 in the reference's
// serial index order. The counter RNG is the reference's splitmix64 key chain
// (rng.hpp:23-53) so sampled actions and placements match bit-for-bit.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"
#include "tag_params.hpp"

namespace wdg {
namespace {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;
constexpr float kTwoPiF = 6.28318530717958647692f;  // tag_env.hpp:84

// ---- counter RNG: rng.hpp:23-47 -------------------------------------------
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += kGolden;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t absorb(uint64_t h, uint64_t v) {
  return mix64(h ^ (v + kGolden));
}
__device__ __forceinline__ double to_unit(uint64_t h) {
  return __ull2double_rn(h >> 11) * 0x1.0p-53;
}

// std::min / std::max exactly (first argument wins ties / unordered).
__device__ __forceinline__ float min_ref(float a, float b) { return b < a ? b : a; }
__device__ __forceinline__ float max_ref(float a, float b) { return a < b ? b : a; }

// ---- sampler: sampler.hpp:18-30 -----------------------------------------
// Serial softmax + inverse CDF in f64, strict '<'. exp values cached in
// registers for V <= 8 (the Tag variants use 5 and 3).
__device__ __forceinline__ int32_t sample_row(const double* __restrict__ z, int V, double u,
                                              bool& nonfinite) {
  if (V <= 8) {
    double zv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) zv[i] = i < V ? __ldg(z + i) : 0.0;
    double zmax = zv[0];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i < V) {
        nonfinite |= !isfinite(zv[i]);
        zmax = zmax < zv[i] ? zv[i] : zmax;
      }
    }
    double ev[8];
    double total = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i < V) {
        ev[i] = exp(zv[i] - zmax);
        total = __dadd_rn(total, ev[i]);
      }
    }
    const double target = __dmul_rn(u, total);
    double cum = 0.0;
    int32_t pick = V - 1;
    bool found = false;
#pragma unroll
    for (int i = 0; i < 7; ++i) {
      if (i + 1 < V && !found) {
        cum = __dadd_rn(cum, ev[i]);
        if (target < cum) {
          pick = i;
          found = true;
        }
      }
    }
    return pick;
  }
  double zmax = __ldg(z);
  for (int i = 0; i < V; ++i) {
    const double zi = __ldg(z + i);
    nonfinite |= !isfinite(zi);
    zmax = zmax < zi ? zi : zmax;
  }
  double total = 0.0;
  for (int i = 0; i < V; ++i) total = __dadd_rn(total, exp(__ldg(z + i) - zmax));
  const double target = __dmul_rn(u, total);
  double cum = 0.0;
  for (int i = 0; i + 1 < V; ++i) {
    cum = __dadd_rn(cum, exp(__ldg(z + i) - zmax));
    if (target < cum) return i;
  }
  return V - 1;
}

// ---- shared-memory views ---------------------------------------------------
struct EnvScalars {
  int32_t runners_left;
  int32_t step_count;
  int32_t done;
  int32_t episode;
  int32_t tags;
  int32_t live;
  int32_t did_reset;
  int32_t pad;
  double ret_tagger;
  double ret_runner;
};
static_assert(sizeof(EnvScalars) == 48, "EnvScalars layout");

struct EnvSmem {
  float* x;
  float* y;
  float* sp;
  float* dir;
  float* sn;
  float* cs;
  int32_t* cred;
  uint8_t* tag;
  uint8_t* act;
  uint8_t* tagged;
  uint16_t* knn;
  int32_t* cstart;
  int32_t* cfill;
  uint16_t* items;
  uint16_t* cellof;
};

__device__ __forceinline__ EnvSmem carve(uint8_t* b, const TagDevConfig& p) {
  EnvSmem s;
  s.x = reinterpret_cast<float*>(b);
  s.y = reinterpret_cast<float*>(b + p.off_y);
  s.sp = reinterpret_cast<float*>(b + p.off_speed);
  s.dir = reinterpret_cast<float*>(b + p.off_dir);
  s.sn = reinterpret_cast<float*>(b + p.off_sin);
  s.cs = reinterpret_cast<float*>(b + p.off_cos);
  s.cred = reinterpret_cast<int32_t*>(b + p.off_cred);
  s.tag = b + p.off_tag;
  s.act = b + p.off_act;
  s.tagged = b + p.off_tagged;
  s.knn = reinterpret_cast<uint16_t*>(b + p.off_knn);
  s.cstart = reinterpret_cast<int32_t*>(b + p.off_cstart);
  s.cfill = reinterpret_cast<int32_t*>(b + p.off_cfill);
  s.items = reinterpret_cast<uint16_t*>(b + p.off_items);
  s.cellof = reinterpret_cast<uint16_t*>(b + p.off_cellof);
  return s;
}

// ---- bucket grid (NeighborGrid semantics, neighbor_grid.hpp:11-111) -------
template <bool CONT>
__device__ __forceinline__ int cell_coord(float v, const TagDevConfig& p) {
  if (CONT) {
    int c = static_cast<int>(floorf(v * p.cell_inv));
    return c < 0 ? 0 : (c > p.gc - 1 ? p.gc - 1 : c);
  } else {
    int iv = static_cast<int>(floorf(v));
    const int g = static_cast<int>(p.grid_size);
    iv = iv < 0 ? 0 : (iv > g - 1 ? g - 1 : iv);
    return static_cast<int>((static_cast<int64_t>(iv) * p.gc) / g);
  }
}

// Block-wide exclusive scan of counts held in s.cfill[0..n) -> s.cstart,
// s.cfill (= starts, used as fill cursors). Whole CTA = one env.
__device__ void block_scan_cells(const EnvSmem& s, int n, int total, int* scratch) {
  const int nthr = blockDim.x, tid = threadIdx.x;
  const int chunk = (n + nthr - 1) / nthr;
  const int begin = tid * chunk;
  const int end = min(begin + chunk, n);
  int local = 0;
  for (int c = begin; c < end; ++c) local += s.cfill[c];
  const int lane = tid & 31, warp = tid >> 5;
  int incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) scratch[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int nw = (nthr + 31) >> 5;
    int v = lane < nw ? scratch[lane] : 0;
    int sc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, sc, o);
      if (lane >= o) sc += t;
    }
    if (lane < nw) scratch[lane] = sc - v;  // exclusive warp offsets
  }
  __syncthreads();
  int off = scratch[warp] + incl - local;
  for (int c = begin; c < end; ++c) {
    const int v = s.cfill[c];
    s.cstart[c] = off;
    s.cfill[c] = off;
    off += v;
  }
  if (tid == 0) s.cstart[n] = total;
}

template <bool CONT>
__device__ void build_grid(const EnvSmem& s, const TagDevConfig& p, int* scratch) {
  const int nthr = blockDim.x, tid = threadIdx.x;
  for (int c = tid; c <= p.ncells; c += nthr) s.cfill[c] = 0;
  __syncthreads();
  for (int a = tid; a < p.A; a += nthr) {
    const int c = cell_coord<CONT>(s.y[a], p) * p.gc + cell_coord<CONT>(s.x[a], p);
    s.cellof[a] = static_cast<uint16_t>(c);
    atomicAdd(&s.cfill[c], 1);
  }
  __syncthreads();
  block_scan_cells(s, p.ncells, p.A, scratch);
  __syncthreads();
  for (int a = tid; a < p.A; a += nthr) {
    const int slot = atomicAdd(&s.cfill[s.cellof[a]], 1);
    s.items[slot] = static_cast<uint16_t>(a);
  }
  __syncthreads();
}

// ---- exact top-K under the (d2, index) total order ------------------------
// Same selection as select_k_nearest_brute (tag_env.cpp:225-237) and
// NeighborGrid::k_nearest (neighbor_grid.hpp:62-111): unique because the
// order is total, so any visiting order gives the identical list.
template <int MAXK>
struct TopK {
  float d[MAXK];
  int i[MAXK];
  float wd;
  int wi;
  int k;
  __device__ __forceinline__ void init(int kk) {
    k = kk;
#pragma unroll
    for (int t = 0; t < MAXK; ++t) {
      d[t] = __int_as_float(0x7f800000);
      i[t] = 0x7fffffff;
    }
    wd = __int_as_float(0x7f800000);
    wi = 0x7fffffff;
  }
  __device__ __forceinline__ bool full() const { return wi != 0x7fffffff; }
  __device__ __forceinline__ void consider(float dd, int j) {
    if (!(dd < wd || (dd == wd && j < wi))) return;
    bool placed = false;
#pragma unroll
    for (int t = MAXK - 1; t >= 0; --t) {
      if (t < k) {
        const bool shift = t > 0 && (dd < d[t - 1] || (dd == d[t - 1] && j < i[t - 1]));
        if (shift) {
          d[t] = d[t - 1];
          i[t] = i[t - 1];
        } else if (!placed) {
          d[t] = dd;
          i[t] = j;
          placed = true;
        }
      }
    }
#pragma unroll
    for (int t = 0; t < MAXK; ++t) {
      if (t == k - 1) {
        wd = d[t];
        wi = i[t];
      }
    }
  }
};

__device__ __forceinline__ float d2_of(float ax, float ay, float bx, float by) {
  const float dx = __fsub_rn(bx, ax);
  const float dy = __fsub_rn(by, ay);
  return __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
}

template <bool CONT, bool GRID, int MAXK>
__device__ void knn_agent(const EnvSmem& s, const TagDevConfig& p, int a, TopK<MAXK>& top) {
  const float sx = s.x[a], sy = s.y[a];
  top.init(p.K);
  if (!GRID) {
    for (int j = 0; j < p.A; ++j) {
      if (j == a) continue;
      top.consider(d2_of(sx, sy, s.x[j], s.y[j]), j);
    }
    return;
  }
  const int gc = p.gc;
  const int cx = cell_coord<CONT>(sx, p), cy = cell_coord<CONT>(sy, p);
  const int maxr = max(max(cx, gc - 1 - cx), max(cy, gc - 1 - cy));
  for (int r = 0; r <= maxr; ++r) {
    if (r > 0 && top.full()) {
      // Every point in rings >= r is farther than the bound below (SURVEY.md
      // §8a a6; cf. the reference's ring margin, neighbor_grid.hpp:90-96).
      float lb2;
      if (CONT) {
        const double lb = fmax(0.0, (r - 1) - 1e-3) * p.cell_size;
        lb2 = static_cast<float>(lb * lb * (1.0 - 1e-5));
      } else {
        const float lb = static_cast<float>((r - 1) * p.lattice_w + 1);
        lb2 = lb * lb;
      }
      if (top.wd < lb2) break;
    }
    const int y0 = cy - r, y1 = cy + r, x0 = cx - r, x1 = cx + r;
    for (int gy = max(y0, 0); gy <= min(y1, gc - 1); ++gy) {
      const bool edge = (gy == y0 || gy == y1);
      const int step = edge ? 1 : (x1 - x0);
      for (int gx = x0; gx <= x1; gx += (step > 0 ? step : 1)) {
        if (gx < 0 || gx >= gc) continue;
        const int c = gy * gc + gx;
        const int e = s.cstart[c + 1];
        for (int t = s.cstart[c]; t < e; ++t) {
          const int j = s.items[t];
          if (j == a) continue;
          top.consider(d2_of(sx, sy, s.x[j], s.y[j]), j);
        }
      }
    }
  }
}

// Tag resolution for one active runner: resolve kernel (tag_env.cpp:403-456)
// / TagReference::step (tag_env.cpp:546-571). Returns the credited tagger or -1.
template <bool CONT, bool GRID>
__device__ int find_tagger(const EnvSmem& s, const TagDevConfig& p, int rn) {
  const float rx = s.x[rn], ry = s.y[rn];
  const float bias = p.fault_bias;
  const bool exact_cell = !CONT && bias == 0.0f;
  const float radius = CONT ? __fadd_rn(p.tag_radius, bias) : bias;
  const float r2 = __fmul_rn(radius, radius);
  int best = -1;
  float best_d2 = 0.0f;
  auto consider = [&](int j) {
    if (!s.tag[j]) return;
    if (exact_cell) {
      if (s.x[j] == rx && s.y[j] == ry && (best < 0 || j < best)) best = j;
    } else {
      const float d2 = d2_of(rx, ry, s.x[j], s.y[j]);
      if (d2 <= r2 && (best < 0 || d2 < best_d2 || (d2 == best_d2 && j < best))) {
        best = j;
        best_d2 = d2;
      }
    }
  };
  if (!GRID) {
    for (int j = 0; j < p.A; ++j) consider(j);
    return best;
  }
  if (exact_cell) {
    const int c = s.cellof[rn];
    const int e = s.cstart[c + 1];
    for (int t = s.cstart[c]; t < e; ++t) consider(s.items[t]);
    return best;
  }
  const float R = __fadd_rn(__fmul_rn(radius, 1.001f), 1e-6f);
  const int x0 = cell_coord<CONT>(__fsub_rn(rx, R), p), x1 = cell_coord<CONT>(__fadd_rn(rx, R), p);
  const int y0 = cell_coord<CONT>(__fsub_rn(ry, R), p), y1 = cell_coord<CONT>(__fadd_rn(ry, R), p);
  for (int gy = y0; gy <= y1; ++gy) {
    for (int gx = x0; gx <= x1; ++gx) {
      const int c = gy * p.gc + gx;
      const int e = s.cstart[c + 1];
      for (int t = s.cstart[c]; t < e; ++t) consider(s.items[t]);
    }
  }
  return best;
}

// One observation element (write_obs_row, tag_env.cpp:165-212).
template <bool CONT, bool PARTIAL>
__device__ __forceinline__ float obs_value(const EnvSmem& s, const TagDevConfig& p,
                                           int32_t step_count, int a, int f) {
  if (!s.act[a]) return 0.0f;
  constexpr int NB = CONT ? 7 : 4;
  const int nbf = p.vis * NB;
  if (f < nbf) {
    const int n = f / NB;
    const int c = f - n * NB;
    const int j = PARTIAL ? static_cast<int>(s.knn[a * p.K + n]) : (n < a ? n : n + 1);
    switch (c) {
      case 0: return __fmul_rn(__fsub_rn(s.x[j], s.x[a]), p.inv_world);
      case 1: return __fmul_rn(__fsub_rn(s.y[j], s.y[a]), p.inv_world);
      case 2: return s.tag[j] ? 1.0f : 0.0f;
      case 3: return s.act[j] ? 1.0f : 0.0f;
      case 4:
        return __fmul_rn(s.sp[j], j < p.T ? p.inv_max_speed_tagger : p.inv_max_speed_runner);
      case 5: return s.sn[j];
      default: return s.cs[j];
    }
  }
  const int t = f - nbf;
  if (t == 0) return __fmul_rn(s.x[a], p.inv_world);
  if (t == 1) return __fmul_rn(s.y[a], p.inv_world);
  if (CONT) {
    if (t == 2) return __fmul_rn(s.sp[a], a < p.T ? p.inv_max_speed_tagger : p.inv_max_speed_runner);
    if (t == 3) return s.sn[a];
    if (t == 4) return s.cs[a];
  }
  return __fmul_rn(static_cast<float>(step_count), p.inv_episode);
}

// sinf/cosf evaluated in f64 and rounded once: the correctly-rounded value
// except in rare double-rounding cases. glibc's sinf/cosf are not correctly
// rounded either, so continuous parity is tolerance-based.
__device__ __forceinline__ float sin_ref(float v) { return __double2float_rn(sin(static_cast<double>(v))); }
__device__ __forceinline__ float cos_ref(float v) { return __double2float_rn(cos(static_cast<double>(v))); }

// ---- the env-step kernel --------------------------------------------------
template <bool CONT, bool PARTIAL, bool GRID, int MAXK>
__global__ void __launch_bounds__(1024) tag_env_kernel(const TagDevConfig p, const TagDevArrays g,
                                                       const TagLaunch L) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int tid = threadIdx.x;
  const int tpe = p.threads_per_env;
  const int le = tid / tpe;
  const int lt = tid - le * tpe;
  const int64_t e = static_cast<int64_t>(blockIdx.x) * p.envs_per_cta + le;
  const bool env_ok = le < p.envs_per_cta && e < p.E;
  const int mode = L.mode;
  const int A = p.A;

  bool live = env_ok;
  if (mode == kModeReinit && L.env_mask != nullptr && env_ok) live = L.env_mask[e] != 0;
  if (p.envs_per_cta == 1 && !live) return;  // CTA-uniform

  EnvScalars* scal = reinterpret_cast<EnvScalars*>(smem);
  int* scratch = reinterpret_cast<int*>(smem + p.envs_per_cta * sizeof(EnvScalars));
  const EnvSmem s = carve(smem + p.head_bytes + (env_ok ? le : 0) * p.env_bytes, p);
  EnvScalars& sc = scal[env_ok ? le : 0];
  const int64_t ga = e * A;

  // Phase 0: stage the env's agent state in shared memory.
  if (live) {
    for (int a = lt; a < A; a += tpe) {
      if (mode != kModeReinit) {
        s.x[a] = g.loc_x[ga + a];
        s.y[a] = g.loc_y[ga + a];
        s.act[a] = g.active[ga + a];
        if (CONT) {
          s.sp[a] = g.speed[ga + a];
          s.dir[a] = g.direction[ga + a];
        }
      }
      s.tag[a] = g.is_tagger[ga + a];
      s.cred[a] = 0;
      s.tagged[a] = 0;
    }
    if (lt == 0) {
      sc.runners_left = 0;
      sc.step_count = mode == kModeReinit ? 0 : g.step_count[e];
      sc.done = 0;
      sc.episode = (L.episode != nullptr && !(mode == kModeReinit && L.init_episode)) ? L.episode[e] : 0;
      sc.tags = 0;
      sc.live = 1;
      sc.did_reset = 0;
      sc.ret_tagger = 0.0;
      sc.ret_runner = 0.0;
    }
  } else if (env_ok && lt == 0) {
    sc.live = 0;
  }
  __syncthreads();

  if (mode != kModeReinit) {
    // Phase 1: sample (fused) + move (apply_move, tag_env.cpp:148-160).
    if (live) {
      const uint64_t h_env = absorb(L.action_h_step, static_cast<uint64_t>(p.env_offset + e));
      bool nonfinite = false;
      for (int a = lt; a < A; a += tpe) {
        int32_t act0, act1 = 1;
        const int64_t row = (ga + a) * p.C;
        if (mode == kModeFused) {
          const uint64_t h_ag = absorb(h_env, static_cast<uint64_t>(a));
          const double u0 = to_unit(absorb(absorb(h_ag, 0), 0));
          act0 = sample_row(L.logits + row * p.V, p.V, u0, nonfinite);
          g.actions[row] = act0;
          if (CONT) {
            const double u1 = to_unit(absorb(absorb(h_ag, 1), 0));
            act1 = sample_row(L.logits + (row + 1) * p.V, p.V, u1, nonfinite);
            g.actions[row + 1] = act1;
          }
        } else {
          act0 = g.actions[row];
          if (CONT) act1 = g.actions[row + 1];
        }
        if (!s.act[a]) continue;
        if (!CONT) {  // move_discrete, tag_env.hpp:71-82
          float x = s.x[a], y = s.y[a];
          switch (act0) {
            case 1: y = __fadd_rn(y, 1.0f); break;
            case 2: y = __fsub_rn(y, 1.0f); break;
            case 3: x = __fsub_rn(x, 1.0f); break;
            case 4: x = __fadd_rn(x, 1.0f); break;
            default: break;
          }
          s.x[a] = min_ref(max_ref(x, 0.0f), p.world_hi);
          s.y[a] = min_ref(max_ref(y, 0.0f), p.world_hi);
        } else {  // move_continuous, tag_env.hpp:86-100
          float dir = s.dir[a], sp = s.sp[a];
          if (act1 == 0) dir = __fsub_rn(dir, p.turn_delta);
          if (act1 == 2) dir = __fadd_rn(dir, p.turn_delta);
          while (dir >= kTwoPiF) dir = __fsub_rn(dir, kTwoPiF);
          while (dir < 0.0f) dir = __fadd_rn(dir, kTwoPiF);
          if (act0 == 0) sp = __fsub_rn(sp, p.accel_delta);
          if (act0 == 2) sp = __fadd_rn(sp, p.accel_delta);
          const float ms = a < p.T ? p.max_speed_tagger : p.max_speed_runner;
          sp = min_ref(max_ref(sp, 0.0f), ms);
          float x = __fadd_rn(s.x[a], __fmul_rn(sp, cos_ref(dir)));
          float y = __fadd_rn(s.y[a], __fmul_rn(sp, sin_ref(dir)));
          s.x[a] = min_ref(max_ref(x, 0.0f), p.world_hi);
          s.y[a] = min_ref(max_ref(y, 0.0f), p.world_hi);
          s.dir[a] = dir;
          s.sp[a] = sp;
        }
      }
      if (nonfinite && L.error) atomicOr(L.error, kErrNonFinite);
    }
    __syncthreads();

    // Phase 2: bucket grid over post-move positions (NeighborGrid::build).
    if (GRID) build_grid<CONT>(s, p, scratch);

    // Phase 3: resolve tags (tag_env.cpp:403-456).
    if (live) {
      for (int a = lt; a < A; a += tpe) {
        if (s.tag[a] || !s.act[a]) continue;
        const int best = find_tagger<CONT, GRID>(s, p, a);
        if (best >= 0) {
          s.act[a] = 0;
          s.tagged[a] = 1;
          atomicAdd(&s.cred[best], 1);
          atomicAdd(&sc.tags, 1);
        } else {
          atomicAdd(&sc.runners_left, 1);
        }
      }
    }
    __syncthreads();
    // resolve_env_counters (tag_env.cpp:241-250).
    if (live && lt == 0) {
      sc.step_count += 1;
      sc.done = (sc.step_count >= p.episode_length || sc.runners_left == 0) ? 1 : 0;
    }
    __syncthreads();

    // Phase 4: rewards (write_rewards_row, tag_env.cpp:252-259) + tracker.
    if (live) {
      const bool reset_now = mode == kModeFused && L.do_reset && sc.done;
      double rt = 0.0, rr = 0.0;
      for (int a = lt; a < A; a += tpe) {
        const float r = s.tag[a] ? __fmul_rn(p.reward_per_tag, static_cast<float>(s.cred[a]))
                                 : (s.tagged[a] ? p.penalty : 0.0f);
        if (a < p.T) rt += static_cast<double>(r); else rr += static_cast<double>(r);
        g.rewards[ga + a] = reset_now ? 0.0f : r;
        g.credits[ga + a] = reset_now ? 0 : s.cred[a];
        g.tagged[ga + a] = reset_now ? 0 : s.tagged[a];
      }
      if (mode == kModeFused && L.track) {
        atomicAdd(&sc.ret_tagger, rt);
        atomicAdd(&sc.ret_runner, rr);
      }
    }
    __syncthreads();
    if (live && lt == 0 && mode == kModeFused && L.track) {
      // EpisodeTracker::accumulate / finish_done (trainer.cpp:229-252); per-env
      // slots, no atomics: [run_t, run_r, episodes, ret_t, ret_r, tags, steps].
      double* es = L.env_stats + e * 8;
      const double run_t = es[0] + sc.ret_tagger;
      const double run_r = es[1] + sc.ret_runner;
      es[5] += sc.tags;
      es[6] += 1.0;
      if (sc.done) {
        es[2] += 1.0;
        es[3] += run_t;
        es[4] += run_r;
        es[0] = 0.0;
        es[1] = 0.0;
      } else {
        es[0] = run_t;
        es[1] = run_r;
      }
    }
  }

  // Phase 5: (re)placement — fused reset-on-done or reinit (place_env,
  // tag_env.cpp:261-273; place_agent :130-146).
  const bool place = live && (mode == kModeReinit || (mode == kModeFused && L.do_reset && sc.done));
  if (place) {
    const int episode = mode == kModeFused ? sc.episode + 1 : sc.episode;
    const uint64_t h_ep = absorb(p.placement_h0, static_cast<uint64_t>(static_cast<int64_t>(episode)));
    const uint64_t h_env = absorb(h_ep, static_cast<uint64_t>(p.env_offset + e));
    for (int a = lt; a < A; a += tpe) {
      const uint64_t h_ag = absorb(h_env, static_cast<uint64_t>(a));
      const double ux = to_unit(absorb(absorb(h_ag, 0), 0));
      const double uy = to_unit(absorb(absorb(h_ag, 1), 0));
      if (!CONT) {
        const double gd = static_cast<double>(p.grid_size);
        int64_t ix = static_cast<int64_t>(__dmul_rn(ux, gd));
        int64_t iy = static_cast<int64_t>(__dmul_rn(uy, gd));
        ix = ix < p.grid_size - 1 ? ix : p.grid_size - 1;
        iy = iy < p.grid_size - 1 ? iy : p.grid_size - 1;
        s.x[a] = static_cast<float>(ix);
        s.y[a] = static_cast<float>(iy);
      } else {
        const double ud = to_unit(absorb(absorb(h_ag, 2), 0));
        s.x[a] = __double2float_rn(__dmul_rn(ux, p.world_length));
        s.y[a] = __double2float_rn(__dmul_rn(uy, p.world_length));
        s.dir[a] = __double2float_rn(__dmul_rn(ud, 6.283185307179586));
        s.sp[a] = 0.0f;
      }
      s.act[a] = 1;
      if (mode == kModeFused) {
        // zero-on-reset rows (tag_env.cpp:343-346) not rewritten later, and
        // is_tagger restored from its snapshot (data_store.cpp:207-217).
        const uint8_t t = g.snap_is_tagger[ga + a];
        s.tag[a] = t;
        g.is_tagger[ga + a] = t;
        g.actions[(ga + a) * p.C] = 0;
        if (CONT) g.actions[(ga + a) * p.C + 1] = 0;
      }
    }
    if (lt == 0) {
      sc.step_count = 0;
      sc.done = 0;
      sc.episode = episode;
      sc.did_reset = 1;
    }
  }
  __syncthreads();

  // Phase 6: observation inputs. Continuous: fill_sincos (tag_env.cpp:214-221).
  if (CONT && live) {
    for (int a = lt; a < A; a += tpe) {
      s.sn[a] = sin_ref(s.dir[a]);
      s.cs[a] = cos_ref(s.dir[a]);
    }
  }
  if (GRID && PARTIAL && (mode == kModeReinit || scal[0].did_reset)) {
    // positions changed by placement: rebuild (CTA == one env on this path)
    __syncthreads();
    build_grid<CONT>(s, p, scratch);
  }
  if (PARTIAL && live) {
    for (int a = lt; a < A; a += tpe) {
      if (!s.act[a]) continue;
      TopK<MAXK> top;
      knn_agent<CONT, GRID, MAXK>(s, p, a, top);
#pragma unroll
      for (int t = 0; t < MAXK; ++t) {
        if (t < p.K) s.knn[a * p.K + t] = static_cast<uint16_t>(top.i[t]);
      }
    }
  }
  __syncthreads();

  // Phase 7: observations — the CTA's [envs, A, D] block written as one
  // contiguous, coalesced stream (16-byte streaming stores when aligned).
  {
    const int64_t cta_env0 = static_cast<int64_t>(blockIdx.x) * p.envs_per_cta;
    const int n_envs = static_cast<int>(min(static_cast<int64_t>(p.envs_per_cta), p.E - cta_env0));
    const int D = p.D;
    const int64_t n = static_cast<int64_t>(n_envs) * A * D;
    float* out = g.obs + cta_env0 * A * D;
    const int nthr = blockDim.x;
    const uint8_t* base0 = smem + p.head_bytes;
    auto value = [&](int row, int f) -> float {
      int lenv = 0, a = row;
      if (p.envs_per_cta > 1) {
        lenv = row / A;
        a = row - lenv * A;
      }
      const EnvSmem es = carve(const_cast<uint8_t*>(base0) + lenv * p.env_bytes, p);
      return obs_value<CONT, PARTIAL>(es, p, scal[lenv].step_count, a, f);
    };
    auto row_live = [&](int row) -> bool {
      if (p.envs_per_cta == 1) return true;
      return scal[row / A].live != 0;
    };
    if (((static_cast<int64_t>(A) * D) & 3) == 0) {
      const int64_t nv = n >> 2;
      float4* out4 = reinterpret_cast<float4*>(out);
      int64_t idx = static_cast<int64_t>(tid) * 4;
      int row = static_cast<int>(idx / D);
      int f = static_cast<int>(idx - static_cast<int64_t>(row) * D);
      const int stride = nthr * 4;
      const int sq = stride / D, sr = stride - (stride / D) * D;
      for (int64_t v = tid; v < nv; v += nthr) {
        float vals[4];
        int r = row, ff = f;
        bool any_live = false;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const bool lv = row_live(r);
          any_live |= lv;
          vals[k] = lv ? value(r, ff) : 0.0f;
          if (++ff == D) {
            ff = 0;
            ++r;
          }
        }
        if (any_live) __stcs(out4 + v, make_float4(vals[0], vals[1], vals[2], vals[3]));
        row += sq;
        f += sr;
        if (f >= D) {
          f -= D;
          ++row;
        }
      }
    } else {
      int row = tid / D;
      int f = tid - row * D;
      const int sq = nthr / D, sr = nthr - (nthr / D) * D;
      for (int64_t i = tid; i < n; i += nthr) {
        if (row_live(row)) __stcs(out + i, value(row, f));
        row += sq;
        f += sr;
        if (f >= D) {
          f -= D;
          ++row;
        }
      }
    }
  }

  // Phase 8: write back the env's state.
  if (live) {
    for (int a = lt; a < A; a += tpe) {
      g.loc_x[ga + a] = s.x[a];
      g.loc_y[ga + a] = s.y[a];
      g.active[ga + a] = s.act[a];
      if (CONT) {
        g.speed[ga + a] = s.sp[a];
        g.direction[ga + a] = s.dir[a];
      }
    }
    if (lt == 0 && mode != kModeReinit) {
      g.step_count[e] = sc.step_count;
      g.done[e] = static_cast<uint8_t>(sc.done);
      if (sc.did_reset && L.episode != nullptr) L.episode[e] = sc.episode;
    }
  }
}

// ---- standalone sampler: sample_actions (sampler.cpp:5-40) ----------------
__global__ void sample_kernel(const double* __restrict__ logits, int32_t* __restrict__ actions,
                              int64_t rows, int A, int C, int V, int64_t env_offset,
                              uint64_t h_step) {
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t ea = r / C;
    const int c = static_cast<int>(r - ea * C);
    const int64_t e = ea / A;
    const int a = static_cast<int>(ea - e * A);
    const uint64_t h = absorb(absorb(absorb(absorb(h_step, static_cast<uint64_t>(env_offset + e)),
                                            static_cast<uint64_t>(a)),
                                     static_cast<uint64_t>(c)),
                              0);
    bool nf = false;
    actions[r] = sample_row(logits + r * V, V, to_unit(h), nf);
  }
}

// Finiteness scan (sampler.cpp:23-25) — run before any write, like the reference.
__global__ void finite_scan_kernel(const double* __restrict__ z, int64_t n, uint32_t* flag) {
  bool bad = false;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    bad |= !isfinite(__ldg(z + i));
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, kErrNonFinite);
}

// ---- generic ResetManager::auto_reset pieces (reset_manager.cpp:29-44) -----
__global__ void mask_from_done_kernel(const uint8_t* __restrict__ done, uint8_t* __restrict__ mask,
                                      int64_t E) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < E;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    mask[e] = done[e] ? 1 : 0;
  }
}

__global__ void mask_from_ids_kernel(const int64_t* __restrict__ ids, int64_t n,
                                     uint8_t* __restrict__ mask) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    mask[ids[i]] = 1;
  }
}

}  // namespace

namespace {
// snapshot restore + zero-fill + done clear + episode counter, per masked env.
__global__ void restore_zero_kernel(const ResetRowDesc* __restrict__ descs, int ndesc,
                                    const uint8_t* __restrict__ mask, uint8_t* done,
                                    int32_t* episode, int64_t E) {
  const int64_t e = blockIdx.x;
  if (e >= E || !mask[e]) return;
  for (int d = 0; d < ndesc; ++d) {
    const ResetRowDesc rd = descs[d];
    uint8_t* dst = rd.data + e * rd.row_bytes;
    const uint8_t* src = rd.snapshot ? rd.snapshot + e * rd.row_bytes : nullptr;
    if ((rd.row_bytes & 3) == 0) {
      const int64_t nw = rd.row_bytes >> 2;
      uint32_t* d4 = reinterpret_cast<uint32_t*>(dst);
      const uint32_t* s4 = reinterpret_cast<const uint32_t*>(src);
      for (int64_t i = threadIdx.x; i < nw; i += blockDim.x) d4[i] = src ? s4[i] : 0u;
    } else {
      for (int64_t i = threadIdx.x; i < rd.row_bytes; i += blockDim.x) dst[i] = src ? src[i] : 0;
    }
  }
  if (threadIdx.x == 0) {
    if (done) done[e] = 0;
    if (episode) episode[e] += 1;
  }
}

// Deterministic reduction of the per-env tracker slots into WDG_STAT_*.
__global__ void stats_reduce_kernel(const double* __restrict__ env_stats, int64_t E,
                                    double* __restrict__ out) {
  __shared__ double red[5][256];
  double acc[5] = {0, 0, 0, 0, 0};
  for (int64_t e = threadIdx.x; e < E; e += blockDim.x) {
    const double* es = env_stats + e * 8;
    acc[0] += es[2];
    acc[1] += es[3];
    acc[2] += es[4];
    acc[3] += es[5];
    acc[4] += es[6];
  }
  for (int k = 0; k < 5; ++k) red[k][threadIdx.x] = acc[k];
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int k = 0; k < 5; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    for (int k = 0; k < 5; ++k) out[k] = red[k][0];
    for (int k = 5; k < 8; ++k) out[k] = 0.0;
  }
}

template <bool CONT, bool PARTIAL, bool GRID, int MAXK>
cudaError_t launch_variant(const TagDevConfig& p, const TagDevArrays& g, const TagLaunch& L,
                           cudaStream_t st) {
  auto kern = tag_env_kernel<CONT, PARTIAL, GRID, MAXK>;
  if (p.smem_bytes > 48 * 1024) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           p.smem_bytes);
    if (err != cudaSuccess) return err;
  }
  kern<<<p.grid_ctas, p.threads, p.smem_bytes, st>>>(p, g, L);
  return cudaGetLastError();
}

template <bool CONT, bool PARTIAL, bool GRID>
cudaError_t launch_k(const TagDevConfig& p, const TagDevArrays& g, const TagLaunch& L,
                     cudaStream_t st) {
  if constexpr (!PARTIAL) {
    return launch_variant<CONT, PARTIAL, GRID, 1>(p, g, L, st);
  } else {
    if (p.K <= 8) return launch_variant<CONT, PARTIAL, GRID, 8>(p, g, L, st);
    return launch_variant<CONT, PARTIAL, GRID, 32>(p, g, L, st);
  }
}

template <bool CONT, bool PARTIAL>
cudaError_t launch_g(const TagDevConfig& p, const TagDevArrays& g, const TagLaunch& L,
                     cudaStream_t st) {
  return p.use_grid ? launch_k<CONT, PARTIAL, true>(p, g, L, st)
                    : launch_k<CONT, PARTIAL, false>(p, g, L, st);
}

}  // namespace

// ---- host-callable launchers (declared in kernels.hpp) ---------------------
cudaError_t launch_tag_kernel(const TagDevConfig& p, const TagDevArrays& g, const TagLaunch& L,
                              cudaStream_t st) {
  if (p.continuous) {
    return p.partial ? launch_g<true, true>(p, g, L, st) : launch_g<true, false>(p, g, L, st);
  }
  return p.partial ? launch_g<false, true>(p, g, L, st) : launch_g<false, false>(p, g, L, st);
}

cudaError_t launch_sample(const double* logits, int32_t* actions, int64_t rows, int A, int C, int V,
                          int64_t env_offset, uint64_t h_step, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = (rows + threads - 1) / threads;
  sample_kernel<<<static_cast<unsigned>(blocks < 148 * 64 ? blocks : 148 * 64), threads, 0, st>>>(
      logits, actions, rows, A, C, V, env_offset, h_step);
  return cudaGetLastError();
}

cudaError_t launch_finite_scan(const double* z, int64_t n, uint32_t* flag, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = (n + threads - 1) / threads;
  finite_scan_kernel<<<static_cast<unsigned>(blocks < 148 * 32 ? blocks : 148 * 32), threads, 0, st>>>(
      z, n, flag);
  return cudaGetLastError();
}

cudaError_t launch_mask_from_done(const uint8_t* done, uint8_t* mask, int64_t E, cudaStream_t st) {
  const int threads = 256;
  const int64_t blocks = (E + threads - 1) / threads;
  mask_from_done_kernel<<<static_cast<unsigned>(blocks), threads, 0, st>>>(done, mask, E);
  return cudaGetLastError();
}

cudaError_t launch_mask_from_ids(const int64_t* ids, int64_t n, uint8_t* mask, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = (n + threads - 1) / threads;
  mask_from_ids_kernel<<<static_cast<unsigned>(blocks), threads, 0, st>>>(ids, n, mask);
  return cudaGetLastError();
}

cudaError_t launch_restore_zero(const ResetRowDesc* descs, int ndesc, const uint8_t* mask,
                                uint8_t* done, int32_t* episode, int64_t E, cudaStream_t st) {
  restore_zero_kernel<<<static_cast<unsigned>(E), 128, 0, st>>>(descs, ndesc, mask, done, episode,
                                                                E);
  return cudaGetLastError();
}

cudaError_t launch_stats_reduce(const double* env_stats, int64_t E, double* out, cudaStream_t st) {
  stats_reduce_kernel<<<1, 256, 0, st>>>(env_stats, E, out);
  return cudaGetLastError();
}

}  // namespace wdg
