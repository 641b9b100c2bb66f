// twin_kernels.cu — the device TagReference: an independent, deliberately
// plain implementation of the Tag step for the consistency check, mirroring
// the reference's sequential brute-force oracle TagReference
// (proj/src/tag_env.cpp:505-595) the way the reference's checker pits its
// engine against it (proj/src/harness.cpp:562-633).
//
// Nothing here is shared with the production kernel (tag_kernels.cu) except
// the reference's own primitives in device_ref.cuh (counter RNG, std::min /
// std::max, glibc sinf/cosf): no shared memory staging, no bucket grid or
// lattice cells, no K-NN lists per cell, no observation staging, no fused
// reset. Every array is read and written in global memory in the reference's
// order; K-NN is the reference's brute-force insertion over all agents
// (select_k_nearest_brute, tag_env.cpp:225-237) with per-agent scratch in
// HBM, so any K < A works. Resolve is a brute-force scan over all taggers.
// It ignores the fault hook (TagDevConfig::fault_bias), like the reference's
// TagReference, so an injected fault shows up as a divergence.
#include <cuda_runtime.h>

#include <cstdint>

#include "device_ref.cuh"
#include "kernels.hpp"
#include "tag_params.hpp"

namespace wdg {
namespace {

constexpr int kTwinThreads = 256;

struct TwinLaunch {
  int32_t mode;                 // kModeStep or kModeReinit
  const uint8_t* env_mask;      // reinit: envs to reinit (nullptr = all)
  const int32_t* episode;       // reinit: per-env episode (nullptr = episode 0)
  float* knn_d2;                // partial obs: [E*A*K] scratch
  int32_t* knn_idx;             // partial obs: [E*A*K] scratch
};

__device__ __forceinline__ float twin_max_speed(const TagDevConfig& p, int a) {
  return a < p.T ? p.max_speed_tagger : p.max_speed_runner;
}
__device__ __forceinline__ float twin_inv_max_speed(const TagDevConfig& p, int a) {
  return a < p.T ? p.inv_max_speed_tagger : p.inv_max_speed_runner;
}

// apply_move (tag_env.cpp:148-160) with move_discrete / move_continuous
// (tag_env.hpp:71-100), agent by agent.
template <bool CONT>
__device__ void twin_move(const TagDevConfig& p, const TagDevArrays& g, int64_t base) {
  for (int a = threadIdx.x; a < p.A; a += blockDim.x) {
    const int64_t i = base + a;
    if (!g.active[i]) continue;
    float x = g.loc_x[i], y = g.loc_y[i];
    if (!CONT) {
      switch (g.actions[i]) {
        case 1: y = y + 1.0f; break;
        case 2: y = y - 1.0f; break;
        case 3: x = x - 1.0f; break;
        case 4: x = x + 1.0f; break;
        default: break;
      }
      x = min_ref(max_ref(x, 0.0f), p.world_hi);
      y = min_ref(max_ref(y, 0.0f), p.world_hi);
    } else {
      const int accel = g.actions[2 * i], turn = g.actions[2 * i + 1];
      float dir = g.direction[i], speed = g.speed[i];
      if (turn == 0) dir = dir - p.turn_delta;
      if (turn == 2) dir = dir + p.turn_delta;
      while (dir >= kTwoPiF) dir = dir - kTwoPiF;
      while (dir < 0.0f) dir = dir + kTwoPiF;
      if (accel == 0) speed = speed - p.accel_delta;
      if (accel == 2) speed = speed + p.accel_delta;
      speed = min_ref(max_ref(speed, 0.0f), twin_max_speed(p, a));
      const float vx = speed * cos_ref(dir);
      const float vy = speed * sin_ref(dir);
      x = x + vx;
      y = y + vy;
      x = min_ref(max_ref(x, 0.0f), p.world_hi);
      y = min_ref(max_ref(y, 0.0f), p.world_hi);
      g.direction[i] = dir;
      g.speed[i] = speed;
    }
    g.loc_x[i] = x;
    g.loc_y[i] = y;
  }
}

// resolve (TagReference::step, tag_env.cpp:539-574): every active runner
// scans every tagger; credits are integer atomics (order-free).
template <bool CONT>
__device__ void twin_resolve(const TagDevConfig& p, const TagDevArrays& g, int64_t base) {
  for (int a = threadIdx.x; a < p.A; a += blockDim.x) {
    g.credits[base + a] = 0;
    g.tagged[base + a] = 0;
  }
  __syncthreads();
  const float r2 = p.tag_radius * p.tag_radius;
  for (int rn = threadIdx.x; rn < p.A; rn += blockDim.x) {
    if (g.is_tagger[base + rn] || !g.active[base + rn]) continue;
    const float rx = g.loc_x[base + rn], ry = g.loc_y[base + rn];
    int best = -1;
    float best_d2 = 0.0f;
    for (int tg = 0; tg < p.A; ++tg) {
      if (!g.is_tagger[base + tg]) continue;
      const float tx = g.loc_x[base + tg], ty = g.loc_y[base + tg];
      if (!CONT) {
        if (tx == rx && ty == ry) {
          best = tg;  // ascending scan: the first is the lowest index
          break;
        }
      } else {
        const float dx = tx - rx;
        const float dy = ty - ry;
        const float d2 = dx * dx + dy * dy;
        if (d2 <= r2 && (best < 0 || d2 < best_d2)) {  // ascending: ties keep the lower index
          best = tg;
          best_d2 = d2;
        }
      }
    }
    if (best >= 0) {
      g.active[base + rn] = 0;
      g.tagged[base + rn] = 1;
      atomicAdd(&g.credits[base + best], 1);
    }
  }
}

// observe_env (tag_env.cpp:514-528): rewards (write_rewards_row :252-259),
// K-NN by brute-force insertion (select_k_nearest_brute :225-237) and the
// observation row (write_obs_row :165-212), one agent per thread.
template <bool CONT>
__device__ void twin_observe(const TagDevConfig& p, const TagDevArrays& g, const TwinLaunch& L, int64_t e,
                             bool with_rewards) {
  const int64_t base = e * p.A;
  const int32_t steps = g.step_count[e];
  constexpr int NB = CONT ? 7 : 4;
  for (int a = threadIdx.x; a < p.A; a += blockDim.x) {
    const int64_t i = base + a;
    if (with_rewards) {
      g.rewards[i] = g.is_tagger[i] ? p.reward_per_tag * static_cast<float>(g.credits[i])
                                    : (g.tagged[i] ? p.penalty : 0.0f);
    }
    float* out = g.obs + i * p.D;
    if (!g.active[i]) {
      for (int d = 0; d < p.D; ++d) out[d] = 0.0f;
      continue;
    }
    const float sx = g.loc_x[i], sy = g.loc_y[i];
    int n_vis = p.A - 1;
    float* kd = nullptr;
    int32_t* ki = nullptr;
    if (p.partial) {
      kd = L.knn_d2 + i * p.K;
      ki = L.knn_idx + i * p.K;
      int found = 0;
      for (int j = 0; j < p.A; ++j) {
        if (j == a) continue;
        const float dx = g.loc_x[base + j] - sx;
        const float dy = g.loc_y[base + j] - sy;
        const float d2 = dx * dx + dy * dy;
        if (found == p.K) {
          const float wd = kd[p.K - 1];
          if (d2 > wd || (d2 == wd && j > ki[p.K - 1])) continue;
        }
        int pos = found < p.K ? found : p.K - 1;
        while (pos > 0 && (kd[pos - 1] > d2 || (kd[pos - 1] == d2 && ki[pos - 1] > j))) {
          kd[pos] = kd[pos - 1];
          ki[pos] = ki[pos - 1];
          --pos;
        }
        kd[pos] = d2;
        ki[pos] = j;
        if (found < p.K) ++found;
      }
      n_vis = p.K;
    }
    for (int t = 0, slot = 0; slot < n_vis; ++t) {
      const int j = p.partial ? ki[t] : t;
      if (!p.partial && j == a) continue;
      const int64_t jj = base + j;
      float* o = out + slot * NB;
      o[0] = (g.loc_x[jj] - sx) * p.inv_world;
      o[1] = (g.loc_y[jj] - sy) * p.inv_world;
      o[2] = g.is_tagger[jj] ? 1.0f : 0.0f;
      o[3] = g.active[jj] ? 1.0f : 0.0f;
      if (CONT) {
        o[4] = g.speed[jj] * twin_inv_max_speed(p, j);
        o[5] = sin_ref(g.direction[jj]);
        o[6] = cos_ref(g.direction[jj]);
      }
      ++slot;
    }
    float* o = out + n_vis * NB;
    o[0] = sx * p.inv_world;
    o[1] = sy * p.inv_world;
    if (CONT) {
      o[2] = g.speed[i] * twin_inv_max_speed(p, a);
      o[3] = sin_ref(g.direction[i]);
      o[4] = cos_ref(g.direction[i]);
      o[5] = static_cast<float>(steps) * p.inv_episode;
    } else {
      o[2] = static_cast<float>(steps) * p.inv_episode;
    }
  }
}

// place_env / place_agent (tag_env.cpp:130-146, 261-273) with the counter
// RNG keyed (substream(seed, kStreamPlacement), episode, global env, agent,
// coordinate, 0).
template <bool CONT>
__device__ void twin_place(const TagDevConfig& p, const TagDevArrays& g, int64_t e, int64_t episode) {
  const int64_t base = e * p.A;
  const uint64_t h_env = absorb(absorb(p.placement_h0, static_cast<uint64_t>(episode)),
                                static_cast<uint64_t>(p.env_offset + e));
  for (int a = threadIdx.x; a < p.A; a += blockDim.x) {
    const uint64_t h_a = absorb(h_env, static_cast<uint64_t>(a));
    const double ux = to_unit(absorb(absorb(h_a, 0), 0));
    const double uy = to_unit(absorb(absorb(h_a, 1), 0));
    const int64_t i = base + a;
    if (!CONT) {
      const double gs = static_cast<double>(p.grid_size);
      int64_t ix = __double2ll_rz(__dmul_rn(ux, gs));
      int64_t iy = __double2ll_rz(__dmul_rn(uy, gs));
      if (ix > p.grid_size - 1) ix = p.grid_size - 1;
      if (iy > p.grid_size - 1) iy = p.grid_size - 1;
      g.loc_x[i] = static_cast<float>(ix);
      g.loc_y[i] = static_cast<float>(iy);
    } else {
      const double ud = to_unit(absorb(absorb(h_a, 2), 0));
      g.loc_x[i] = __double2float_rn(__dmul_rn(ux, p.world_length));
      g.loc_y[i] = __double2float_rn(__dmul_rn(uy, p.world_length));
      g.direction[i] = __double2float_rn(__dmul_rn(ud, 6.283185307179586));
      g.speed[i] = 0.0f;
    }
    g.active[i] = 1;
  }
}

template <bool CONT>
__global__ void __launch_bounds__(kTwinThreads) twin_kernel(const TagDevConfig p, const TagDevArrays g,
                                                           const TwinLaunch L) {
  const int64_t e = blockIdx.x;
  if (e >= p.E) return;
  const int64_t base = e * p.A;
  if (L.mode == kModeReinit) {  // TagReference::reinit_env (tag_env.cpp:579-595)
    if (L.env_mask != nullptr && !L.env_mask[e]) return;
    twin_place<CONT>(p, g, e, L.episode != nullptr ? L.episode[e] : 0);
    __syncthreads();
    twin_observe<CONT>(p, g, L, e, false);
    return;
  }
  // TagReference::step (tag_env.cpp:530-577)
  twin_move<CONT>(p, g, base);
  __syncthreads();
  twin_resolve<CONT>(p, g, base);
  __syncthreads();
  if (threadIdx.x == 0) {  // resolve_env_counters (tag_env.cpp:241-250)
    g.step_count[e] += 1;
    int runners_left = 0;
    for (int a = 0; a < p.A; ++a) runners_left += (!g.is_tagger[base + a] && g.active[base + a]) ? 1 : 0;
    g.done[e] = (g.step_count[e] >= p.episode_length || runners_left == 0) ? 1 : 0;
  }
  __syncthreads();
  twin_observe<CONT>(p, g, L, e, true);
}

}  // namespace

cudaError_t launch_twin_kernel(const TagDevConfig& p, const TagDevArrays& g, int32_t mode,
                               const uint8_t* env_mask, const int32_t* episode, float* knn_d2,
                               int32_t* knn_idx, cudaStream_t st) {
  if (p.E <= 0) return cudaSuccess;
  TwinLaunch L{mode, env_mask, episode, knn_d2, knn_idx};
  if (p.continuous) {
    twin_kernel<true><<<p.E, kTwinThreads, 0, st>>>(p, g, L);
  } else {
    twin_kernel<false><<<p.E, kTwinThreads, 0, st>>>(p, g, L);
  }
  return cudaGetLastError();
}

}  // namespace wdg
