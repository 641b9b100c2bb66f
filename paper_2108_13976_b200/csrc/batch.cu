// batch.cu — device rollout capture and returns:
// RolloutBatch (proj/include/warp/trainer.hpp:36-49), the Trainer::collect
// hooks (proj/src/trainer.cpp:315-403) and compute_returns (trainer.cpp:73-88)
// with every tensor in HBM: the [T, E, A, ...] batch is filled by the fused
// step itself (actions, active-at-sample, pre-reset rewards and done), by the
// policy forward (values, bootstrap) and by two small kernels (log-prob of the
// taken action, the discounted-return reverse scan).
#include <cuda_runtime.h>

#include <cmath>
#include <string>

#include "batch.hpp"
#include "facade.hpp"

namespace wdg {
namespace {

// category_stats(z, V, action).logp summed over categories (trainer.cpp:25-41,
// 386-392): zmax, sum = sum exp(z - zmax) in index order, lse = log(sum),
// logp = z[a] - zmax - lse.
__global__ void logp_kernel(const double* __restrict__ logits, const int32_t* __restrict__ actions,
                            double* __restrict__ logp, int64_t rows, int C, int V) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < rows;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double lp = 0.0;
    for (int c = 0; c < C; ++c) {
      const double* z = logits + (i * C + c) * V;
      double zmax = z[0];
      for (int k = 1; k < V; ++k) zmax = zmax < z[k] ? z[k] : zmax;  // std::max(zmax, z[k])
      double sum = 0.0;
      for (int k = 0; k < V; ++k) sum = __dadd_rn(sum, exp(z[k] - zmax));
      const int32_t a = actions[i * C + c];
      lp = __dadd_rn(lp, (z[a] - zmax) - log(sum));
    }
    logp[i] = lp;
  }
}

// compute_returns (trainer.cpp:73-88): per (e, a), t = T-1 .. 0,
// next = r + gamma * cont * next, in that evaluation order, no contraction.
__global__ void returns_kernel(const float* __restrict__ rewards, const uint8_t* __restrict__ done,
                               const double* __restrict__ bootstrap, double* __restrict__ returns, int64_t T,
                               int64_t E, int64_t A, double gamma) {
  const int64_t n = E * A;
  for (int64_t ea = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; ea < n;
       ea += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t e = ea / A;
    double next = bootstrap[ea];
    for (int64_t t = T - 1; t >= 0; --t) {
      const int64_t idx = t * n + ea;
      const double cont = done[t * E + e] ? 0.0 : 1.0;
      next = __dadd_rn(static_cast<double>(rewards[idx]), __dmul_rn(__dmul_rn(gamma, cont), next));
      returns[idx] = next;
    }
  }
}

int grid_for(int64_t n, int threads) {
  const int64_t b = (n + threads - 1) / threads;
  return static_cast<int>(b < 148 * 32 ? (b < 1 ? 1 : b) : 148 * 32);
}

}  // namespace

RolloutBatch::RolloutBatch(int64_t horizon, int64_t envs, int64_t agents, int64_t obs_dim, int64_t categories)
    : T(horizon), E(envs), A(agents), D(obs_dim), C(categories) {
  if (T < 1) raise(Errc::invalid_argument, "RolloutBatch: horizon must be >= 1");
  const size_t rows = static_cast<size_t>(T * E * A);
  auto alloc = [&](void** p, size_t bytes, const char* what) {
    cuda_check(cudaMalloc(p, bytes == 0 ? 1 : bytes), what);
  };
  alloc(reinterpret_cast<void**>(&obs), rows * D * sizeof(float), "cudaMalloc(batch obs)");
  alloc(reinterpret_cast<void**>(&actions), rows * C * sizeof(int32_t), "cudaMalloc(batch actions)");
  alloc(reinterpret_cast<void**>(&rewards), rows * sizeof(float), "cudaMalloc(batch rewards)");
  alloc(reinterpret_cast<void**>(&done), static_cast<size_t>(T * E), "cudaMalloc(batch done)");
  alloc(reinterpret_cast<void**>(&active), rows, "cudaMalloc(batch active)");
  alloc(reinterpret_cast<void**>(&values), rows * sizeof(double), "cudaMalloc(batch values)");
  alloc(reinterpret_cast<void**>(&logp), rows * sizeof(double), "cudaMalloc(batch logp)");
  alloc(reinterpret_cast<void**>(&bootstrap), static_cast<size_t>(E * A) * sizeof(double),
        "cudaMalloc(batch bootstrap)");
}

RolloutBatch::~RolloutBatch() {
  for (void* p : {static_cast<void*>(obs), static_cast<void*>(actions), static_cast<void*>(rewards),
                  static_cast<void*>(done), static_cast<void*>(active), static_cast<void*>(values),
                  static_cast<void*>(logp), static_cast<void*>(bootstrap)}) {
    if (p) cudaFree(p);
  }
}

void launch_logp(const double* logits, const int32_t* actions, double* logp, int64_t rows, int C, int V,
                 cudaStream_t st) {
  if (rows == 0) return;
  logp_kernel<<<grid_for(rows, 256), 256, 0, st>>>(logits, actions, logp, rows, C, V);
  cuda_check(cudaGetLastError(), "logp kernel");
}

void compute_returns(const RolloutBatch& b, double gamma, double* returns, cudaStream_t st) {
  if (returns == nullptr) raise(Errc::invalid_argument, "compute_returns: null output");
  const int64_t n = b.E * b.A;
  if (n == 0) return;
  returns_kernel<<<grid_for(n, 256), 256, 0, st>>>(b.rewards, b.done, b.bootstrap, returns, b.T, b.E, b.A,
                                                  gamma);
  cuda_check(cudaGetLastError(), "returns kernel");
}

}  // namespace wdg
