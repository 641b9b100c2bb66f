// policy.cu — device forward of the reference policy network (SURVEY.md §8f
// row 1): PolicyParams / init_policy / forward (proj/src/policy_model.cpp:
// 107-197) for the rows of the observation store, producing the f64 logits the
// rollout samples from (RolloutDriver::forward_policies, proj/src/harness.cpp:
// 445-476) without leaving HBM.
//
// kPolicyF64: the reference arithmetic. Each output is acc = 0; acc += w*x in
// input order with separate mul/add roundings (matvec_acc, policy_model.cpp:
// 24-31; the file is built with -fmad=false like the reference's
// -ffp-contract=off), then y = b + acc and tanh. The value head starts from
// value_b (policy_model.cpp:192-193). Thread layout: a group of 64 threads
// owns a tile of 4 rows; thread j computes output j (j + 64, ...) for all 4
// rows, weights transposed in shared memory ([in][out], conflict-free over j),
// activations broadcast from shared memory.
#include <cuda_runtime.h>

#include <cmath>
#include <string>

#include "facade.hpp"
#include "policy.hpp"

namespace wdg {
namespace {

constexpr uint64_t kStreamParams = 0x706172616d733030ULL;  // rng.hpp:57
constexpr int kGroup = 64;       // threads per row tile
constexpr int kTileRows = 4;     // rows per tile
constexpr int kF64Threads = 256;

struct F64Args {
  const float* obs;
  double* logits;
  double* values;
  uint32_t* error;
  int64_t E, A, a0, n;  // rows = E * n, agents [a0, a0 + n)
  int32_t D, W;         // obs_dim, logits width
  int32_t nlayers;
  int32_t widths[8];    // hidden widths
  int32_t maxw;         // max(obs_dim, hidden...)
  int32_t count;        // doubles in the transposed parameter block
};

// Transposed parameter block (host-built, see Policy::upload): per hidden
// layer Wt [in][out] then b [out]; head Wt [last][W], head_b [W]; value_w
// [last]; value_b.
__global__ void __launch_bounds__(kF64Threads) policy_f64_kernel(const double* __restrict__ pt, F64Args a) {
  extern __shared__ __align__(16) double sm[];
  double* P = sm;                                  // parameters
  double* act = sm + ((a.count + 1) & ~1);         // per group: 2 buffers x 4 rows x maxw
  const int groups = blockDim.x / kGroup;
  const int g = threadIdx.x / kGroup;
  const int j = threadIdx.x - g * kGroup;
  double* buf0 = act + static_cast<int64_t>(g) * 2 * kTileRows * a.maxw;
  double* buf1 = buf0 + kTileRows * a.maxw;
  for (int i = threadIdx.x; i < a.count; i += blockDim.x) P[i] = pt[i];
  __syncthreads();

  const int64_t rows = a.E * a.n;
  const int64_t tiles = (rows + kTileRows - 1) / kTileRows;
  const unsigned bar_id = 1 + g;  // named barrier per 64-thread group
  bool bad = false;
  for (int64_t tile = static_cast<int64_t>(blockIdx.x) * groups + g; tile < tiles;
       tile += static_cast<int64_t>(gridDim.x) * groups) {
    const int64_t r0 = tile * kTileRows;
    const int nr = static_cast<int>(rows - r0 < kTileRows ? rows - r0 : kTileRows);
    int64_t grow[kTileRows];
#pragma unroll
    for (int k = 0; k < kTileRows; ++k) {
      const int64_t r = r0 + (k < nr ? k : 0);
      const int64_t e = r / a.n;
      grow[k] = e * a.A + a.a0 + (r - e * a.n);
    }
    // x = double(obs row) (harness.cpp:456-457: float -> double)
#pragma unroll
    for (int k = 0; k < kTileRows; ++k) {
      for (int c = j; c < a.D; c += kGroup) {
        const double v = static_cast<double>(__ldg(a.obs + grow[k] * a.D + c));
        bad |= k < nr && !isfinite(v);
        buf0[k * a.maxw + c] = v;
      }
    }
    asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(kGroup) : "memory");
    const double* in = buf0;
    double* out = buf1;
    int in_w = a.D;
    int off = 0;
    for (int l = 0; l < a.nlayers; ++l) {
      const int ow = a.widths[l];
      const double* Wt = P + off;
      const double* b = Wt + static_cast<int64_t>(in_w) * ow;
      for (int o = j; o < ow; o += kGroup) {
        double acc[kTileRows] = {0.0, 0.0, 0.0, 0.0};
        for (int c = 0; c < in_w; ++c) {
          const double w = Wt[c * ow + o];
#pragma unroll
          for (int k = 0; k < kTileRows; ++k) acc[k] = __dadd_rn(acc[k], __dmul_rn(w, in[k * a.maxw + c]));
        }
#pragma unroll
        for (int k = 0; k < kTileRows; ++k) out[k * a.maxw + o] = tanh(__dadd_rn(b[o], acc[k]));
      }
      off += in_w * ow + ow;
      in_w = ow;
      asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(kGroup) : "memory");
      const double* t = in;
      in = out;
      out = const_cast<double*>(t);
    }
    // heads: logits (matvec_acc from head_b) and value (from value_b)
    const double* Ht = P + off;
    const double* hb = Ht + static_cast<int64_t>(in_w) * a.W;
    const double* vw = hb + a.W;
    const double vb = vw[in_w];
    for (int o = j; o <= a.W; o += kGroup) {
      if (o < a.W) {
        double acc[kTileRows] = {0.0, 0.0, 0.0, 0.0};
        for (int c = 0; c < in_w; ++c) {
          const double w = Ht[c * a.W + o];
#pragma unroll
          for (int k = 0; k < kTileRows; ++k) acc[k] = __dadd_rn(acc[k], __dmul_rn(w, in[k * a.maxw + c]));
        }
        if (a.logits) {
#pragma unroll
          for (int k = 0; k < kTileRows; ++k)
            if (k < nr) a.logits[grow[k] * a.W + o] = __dadd_rn(hb[o], acc[k]);
        }
      } else if (a.values) {
        double v[kTileRows] = {vb, vb, vb, vb};
        for (int c = 0; c < in_w; ++c) {
          const double w = vw[c];
#pragma unroll
          for (int k = 0; k < kTileRows; ++k) v[k] = __dadd_rn(v[k], __dmul_rn(w, in[k * a.maxw + c]));
        }
#pragma unroll
        for (int k = 0; k < kTileRows; ++k)
          if (k < nr) a.values[grow[k]] = v[k];
      }
    }
    asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(kGroup) : "memory");
  }
  if (bad && a.error) atomicOr(a.error, kErrNonFinite);
}

uint64_t params_uniform_bits(uint64_t stream, int64_t matrix_id, int64_t r, int64_t c) {
  // key_bits({stream, matrix_id, r, c, 0, 0}) (rng.hpp:34-42)
  uint64_t h = host_mix64(stream);
  h = host_absorb(h, static_cast<uint64_t>(matrix_id));
  h = host_absorb(h, static_cast<uint64_t>(r));
  h = host_absorb(h, static_cast<uint64_t>(c));
  h = host_absorb(h, 0);
  h = host_absorb(h, 0);
  return h;
}

}  // namespace

static void check_dims(const PolicyDims& d) {  // policy_model.cpp:14-21
  if (d.obs_dim < 1 || d.num_categories < 1 || d.num_choices < 1 || d.hidden.empty()) {
    raise(Errc::invalid_argument, "PolicyDims: all dims must be >= 1 and hidden non-empty");
  }
  for (int64_t h : d.hidden) {
    if (h < 1) raise(Errc::invalid_argument, "PolicyDims: hidden sizes must be >= 1");
  }
  if (d.hidden.size() > 8) raise(Errc::invalid_argument, "PolicyDims: at most 8 hidden layers on device");
}

Policy::Policy(PolicyDims dims) : dims_(std::move(dims)) {
  check_dims(dims_);
  int64_t n = 0, in = dims_.obs_dim;
  for (int64_t h : dims_.hidden) {
    n += h * in + h;
    in = h;
  }
  n += dims_.logits_width() * in + dims_.logits_width() + in + 1;  // PolicyParams::param_count
  count_ = n;
  host_.assign(static_cast<size_t>(n), 0.0);
  dirty_ = true;  // device copies are made on first use (host-only use needs no GPU)
}

Policy::~Policy() {
  if (dparams_) cudaFree(dparams_);
  if (dparams_t_) cudaFree(dparams_t_);
}

void Policy::init(uint64_t seed) {
  // init_policy (policy_model.cpp:107-144)
  const uint64_t stream = host_substream(seed, kStreamParams);
  double* w = host_.data();
  int64_t matrix_id = 0;
  auto xavier = [&](double* dst, int64_t fan_out, int64_t fan_in, int64_t id) {
    const double bound = std::sqrt(6.0 / static_cast<double>(fan_in + fan_out));
    for (int64_t r = 0; r < fan_out; ++r) {
      for (int64_t c = 0; c < fan_in; ++c) {
        const double u = static_cast<double>(params_uniform_bits(stream, id, r, c) >> 11) * 0x1.0p-53;
        dst[r * fan_in + c] = (2.0 * u - 1.0) * bound;
      }
    }
  };
  int64_t in = dims_.obs_dim;
  for (int64_t h : dims_.hidden) {
    xavier(w, h, in, matrix_id++);
    w += h * in;
    for (int64_t i = 0; i < h; ++i) *w++ = 0.0;
    in = h;
  }
  const int64_t V = dims_.num_choices;
  for (int64_t c = 0; c < dims_.num_categories; ++c) {  // per-category blocks
    xavier(w, V, in, matrix_id++);
    w += V * in;
  }
  for (int64_t i = 0; i < dims_.logits_width(); ++i) *w++ = 0.0;
  xavier(w, 1, in, matrix_id++);
  w += in;
  *w++ = 0.0;
  dirty_ = true;
}

void Policy::set_params(const double* host, int64_t count) {
  if (host == nullptr) raise(Errc::invalid_argument, "policy set_params: null");
  if (count != count_) {
    raise(Errc::shape_mismatch, "policy set_params: " + std::to_string(count) + " values, expected " +
                                    std::to_string(count_));
  }
  host_.assign(host, host + count);
  dirty_ = true;
}

void Policy::get_params(double* host, int64_t count) const {
  if (host == nullptr) raise(Errc::invalid_argument, "policy get_params: null");
  if (count != count_) {
    raise(Errc::shape_mismatch, "policy get_params: " + std::to_string(count) + " values, expected " +
                                    std::to_string(count_));
  }
  std::copy(host_.begin(), host_.end(), host);
}

void Policy::upload() const {
  if (!dirty_) return;
  if (dparams_ == nullptr) {
    cuda_check(cudaMalloc(&dparams_, host_.size() * sizeof(double)), "cudaMalloc(policy)");
    cuda_check(cudaMalloc(&dparams_t_, host_.size() * sizeof(double)), "cudaMalloc(policy^T)");
  }
  // canonical copy + transposed copy for the f64 kernel
  std::vector<double> t(host_.size());
  const double* s = host_.data();
  double* d = t.data();
  int64_t in = dims_.obs_dim;
  auto transpose = [&](int64_t out_n, int64_t in_n) {
    for (int64_t o = 0; o < out_n; ++o)
      for (int64_t c = 0; c < in_n; ++c) d[c * out_n + o] = s[o * in_n + c];
    s += out_n * in_n;
    d += out_n * in_n;
  };
  for (int64_t h : dims_.hidden) {
    transpose(h, in);
    for (int64_t i = 0; i < h; ++i) *d++ = *s++;
    in = h;
  }
  const int64_t W = dims_.logits_width();
  transpose(W, in);
  for (int64_t i = 0; i < W + in + 1; ++i) *d++ = *s++;
  cuda_check(cudaMemcpy(dparams_, host_.data(), host_.size() * sizeof(double), cudaMemcpyHostToDevice),
             "policy upload");
  cuda_check(cudaMemcpy(dparams_t_, t.data(), t.size() * sizeof(double), cudaMemcpyHostToDevice),
             "policy upload^T");
  dirty_ = false;
}

void Policy::forward_agents(const float* obs, int64_t E, int64_t A, int64_t a0, int64_t a1, double* logits,
                            double* values, int32_t precision, cudaStream_t st,
                            uint32_t* error) const {
  if (obs == nullptr) raise(Errc::invalid_argument, "policy forward: null observations");
  if (a0 < 0 || a1 > A || a0 > a1) raise(Errc::index_out_of_range, "policy forward: bad agent range");
  if (E == 0 || a1 == a0) return;
  if (precision != kPolicyF64) raise(Errc::invalid_argument, "policy forward: unknown precision");
  upload();
  F64Args a{};
  a.obs = obs;
  a.logits = logits;
  a.values = values;
  a.error = error;
  a.E = E;
  a.A = A;
  a.a0 = a0;
  a.n = a1 - a0;
  a.D = static_cast<int32_t>(dims_.obs_dim);
  a.W = static_cast<int32_t>(dims_.logits_width());
  a.nlayers = static_cast<int32_t>(dims_.hidden.size());
  a.maxw = a.D;
  for (int i = 0; i < a.nlayers; ++i) {
    a.widths[i] = static_cast<int32_t>(dims_.hidden[i]);
    a.maxw = std::max(a.maxw, a.widths[i]);
  }
  a.count = static_cast<int32_t>(count_);
  const int groups = kF64Threads / kGroup;
  const size_t smem = static_cast<size_t>(((count_ + 1) & ~int64_t{1}) +
                                          int64_t{groups} * 2 * kTileRows * a.maxw) * sizeof(double);
  if (smem > 200 * 1024) {
    raise(Errc::invalid_config, "policy forward: " + std::to_string(count_) +
                                    " parameters exceed the f64 kernel's shared-memory budget");
  }
  cuda_check(cudaFuncSetAttribute(policy_f64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)),
             "policy smem attr");
  const int64_t tiles = (E * a.n + kTileRows - 1) / kTileRows;
  int blocks_per_sm = 1;
  cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, policy_f64_kernel, kF64Threads, smem),
             "policy occupancy");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (tiles + groups - 1) / groups;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, int64_t{sms} * std::max(1, blocks_per_sm))));
  policy_f64_kernel<<<grid, kF64Threads, smem, st>>>(dparams_t_, a);
  cuda_check(cudaGetLastError(), "policy f64 kernel");
}

}  // namespace wdg
