// kernels.hpp — host-callable launchers implemented in tag_kernels.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "tag_params.hpp"

namespace wdg {

struct ResetRowDesc {
  uint8_t* data;
  const uint8_t* snapshot;  // nullptr -> zero-fill
  int64_t row_bytes;
};

// Whether single fused/step launches of this plan take the LEAN lattice
// instantiation (tag_kernels.cu).
bool lean_plan(const TagDevConfig& p);
// Whether fused launches of this plan (no overlap flags, no capture) take the
// warp-resident small-env kernel (A <= 32, tag_kernels.cu).
bool small_plan(const TagDevConfig& p);
cudaError_t launch_tag_kernel(const TagDevConfig& p, const TagDevArrays& g, const TagLaunch& L,
                              cudaStream_t st);
cudaError_t launch_sample(const double* logits, int32_t* actions, int64_t rows, int A, int C, int V,
                          int64_t env_offset, uint64_t h_step, cudaStream_t st);
cudaError_t launch_finite_scan(const double* z, int64_t n, uint32_t* flag, cudaStream_t st);
cudaError_t launch_mask_from_done(const uint8_t* done, uint8_t* mask, int64_t E, cudaStream_t st);
cudaError_t launch_mask_from_ids(const int64_t* ids, int64_t n, uint8_t* mask, cudaStream_t st);
cudaError_t launch_restore_zero(const ResetRowDesc* descs, int ndesc, const uint8_t* mask,
                                uint8_t* done, int32_t* episode, int64_t E, cudaStream_t st);
// ptr[0] = value; ptr[1] = value2 when value2 >= 0
cudaError_t launch_set_counter(int64_t* ptr, int64_t value, cudaStream_t st, int64_t value2 = -1);
// The device TagReference (twin_kernels.cu): mode kModeStep or kModeReinit.
cudaError_t launch_twin_kernel(const TagDevConfig& p, const TagDevArrays& g, int32_t mode,
                               const uint8_t* env_mask, const int32_t* episode, float* knn_d2,
                               int32_t* knn_idx, cudaStream_t st);
cudaError_t launch_stats_reduce(const double* env_stats, int64_t E, double* out, cudaStream_t st);

}  // namespace wdg
