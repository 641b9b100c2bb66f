// batch.hpp — device RolloutBatch (proj/include/warp/trainer.hpp:36-49).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace wdg {

// Every buffer is device memory, dense, time outermost: obs [T,E,A,D] f32,
// actions [T,E,A,C] i32, rewards [T,E,A] f32, done [T,E] u8, active [T,E,A]
// u8, values / logp [T,E,A] f64, bootstrap [E,A] f64 — the reference layout.
class RolloutBatch {
 public:
  RolloutBatch(int64_t horizon, int64_t envs, int64_t agents, int64_t obs_dim, int64_t categories);
  ~RolloutBatch();
  RolloutBatch(const RolloutBatch&) = delete;
  RolloutBatch& operator=(const RolloutBatch&) = delete;
  int64_t rows() const { return T * E * A; }

  int64_t T, E, A, D, C;
  float* obs = nullptr;
  int32_t* actions = nullptr;
  float* rewards = nullptr;
  uint8_t* done = nullptr;
  uint8_t* active = nullptr;
  double* values = nullptr;
  double* logp = nullptr;
  double* bootstrap = nullptr;
};

// log-prob of the taken action per row (trainer.cpp:386-392).
void launch_logp(const double* logits, const int32_t* actions, double* logp, int64_t rows, int C, int V,
                 cudaStream_t st);
// compute_returns (trainer.cpp:73-88) into device returns [T, E, A].
void compute_returns(const RolloutBatch& b, double gamma, double* returns, cudaStream_t st);

}  // namespace wdg
