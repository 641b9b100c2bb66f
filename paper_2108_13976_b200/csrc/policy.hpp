// policy.hpp — device policy forward for the Tag rollout:
// the reference's fully-connected policy (proj/include/warp/policy_model.hpp,
// proj/src/policy_model.cpp) evaluated on the observations the env kernel just
// wrote, producing the f64 logits the sampler consumes — the
// forward_policies() half of RolloutDriver::step (proj/src/harness.cpp:445-476)
// moved onto the GPU so no observation or logit ever crosses PCIe.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

namespace wdg {

// PolicyDims (policy_model.hpp:20-28).
struct PolicyDims {
  int64_t obs_dim = 0;
  std::vector<int64_t> hidden = {64, 64};
  int64_t num_categories = 1;
  int64_t num_choices = 1;
  int64_t logits_width() const { return num_categories * num_choices; }
};

// Precision of the device forward.
enum PolicyPrecision : int32_t {
  // f64 in the reference's order: per output acc = 0, acc += w*x serially with
  // separate multiply and add roundings (matvec_acc, policy_model.cpp:24-31,
  // built with -ffp-contract=off), y = b + acc, tanh. Matches the reference
  // forward to the last bit except where CUDA's tanh and glibc's tanh round
  // differently (<= 1 ulp per activation).
  kPolicyF64 = 0,
  // bf16 operands, f32 accumulation on the tcgen05 tensor cores.
  kPolicyBF16 = 1,
};

// Counter-RNG keys of sample_actions (sampler.cpp:31-39) for a fused
// forward+sample: h_step = absorb(mix64(substream(seed, kStreamActions)), t),
// or, under graph replay, t = *step_dev + step_add hashed from h0 on device.
struct SampleKeys {
  int64_t env_offset = 0;
  uint64_t h_step = 0;
  const int64_t* step_dev = nullptr;
  int32_t step_add = 0;
  uint64_t h0 = 0;
};

class Policy {
 public:
  explicit Policy(PolicyDims dims);
  ~Policy();
  Policy(const Policy&) = delete;
  Policy& operator=(const Policy&) = delete;

  const PolicyDims& dims() const { return dims_; }
  int64_t param_count() const { return count_; }
  // init_policy(seed, dims) (policy_model.cpp:107-144): Xavier-uniform from
  // the counter RNG (stream kStreamParams), zero biases; bit-identical.
  void init(uint64_t seed);
  // Canonical flat order (PolicyParams::for_each_param, policy_model.hpp:43-46):
  // hidden (W [out,in] row-major, b) per layer, head_w, head_b, value_w, value_b.
  void set_params(const double* host, int64_t count);
  void get_params(double* host, int64_t count) const;
  const double* device_params() const {
    upload();
    return dparams_;
  }

  // forward over the agent range [a0, a1) of every env of an [E, A, obs_dim]
  // f32 observation array: logits row (e*A + a) of an [E, A, W] f64 array and
  // values (e*A + a) of [E, A] (either output may be nullptr).
  // Non-finite observations set kErrNonFinite in *error (sticky device word;
  // the reference raises non_finite, policy_model.cpp:152-154).
  void forward_agents(const float* obs, int64_t E, int64_t A, int64_t a0, int64_t a1, double* logits,
                      double* values, int32_t precision, cudaStream_t st, uint32_t* error) const;
  // kPolicyBF16 forward fused with sample_actions: writes the sampled actions
  // [E, A, C] (actions may be nullptr) and optionally f64 logits / values.
  void forward_sample_bf16(const float* obs, int64_t E, int64_t A, int64_t a0, int64_t a1, int32_t* actions,
                           double* logits, double* values, const SampleKeys& keys, cudaStream_t st,
                           uint32_t* error, bool pdl = false) const;
  // pdl: launch with programmatic dependent launch. The kernel releases the
  // next launch at entry and runs its prologue (weights to smem, TMEM
  // allocation) before griddepcontrol.wait, i.e. under the previous kernel's tail.
  // The bf16 tensor-core path covers the reference default dims: hidden
  // {64, 64}, C*V <= 7, obs_dim <= 128.
  bool bf16_supported() const;

 private:
  void upload() const;  // lazy host -> device copy (mutable caches)
  PolicyDims dims_;
  int64_t count_ = 0;
  std::vector<double> host_;
  mutable bool dirty_ = true;
  mutable double* dparams_ = nullptr;    // canonical order
  mutable double* dparams_t_ = nullptr;  // transposed weights for the f64 kernel
  mutable uint8_t* dimage_ = nullptr;    // bf16 smem image of the tensor-core kernel
};

}  // namespace wdg
