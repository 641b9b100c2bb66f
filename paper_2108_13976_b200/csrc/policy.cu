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
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
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

// ---- kPolicyBF16: tcgen05 tensor-core forward fused with the sampler ---------
//
// One CTA (128 threads) per SM-quarter, persistent over 128-row tiles. Per
// tile the MLP is three tcgen05.mma chains, D[128 x N] (f32, TMEM) =
// A[128 x K] (bf16, smem) . B[N x K]^T (bf16, smem, the layer's weights,
// resident for the kernel's life):
//   layer 1: K = obs_dim padded to 16, N = 64    (A = the obs rows, f32 -> bf16)
//   layer 2: K = 64, N = 64                      (A = tanh(D1 + b1) as bf16)
//   head   : K = 64, N = 16 (C*V logits, value, zero pad)
// One elected thread issues the MMAs and commits them to an mbarrier; thread
// t owns row t in every epilogue (TMEM lane t: tcgen05.ld 32x32b), so the
// bias + tanh + bf16 repack of the next layer's A operand and, at the end, the
// sampler (sample_from_logits in f64 on the row's logits, sampler.hpp:18-30,
// with the reference's counter RNG keys, sampler.cpp:31-39) run in registers:
// logits never reach HBM, only the sampled action (and optionally the f64
// logits / value) is stored.
//
// Shared-memory operand layout: UMMA canonical K-major, no swizzle. Core
// matrix = 8 rows x 16 B (8 bf16 along K); core matrix (r/8, k/8) sits at
// ((r/8) * (K/8) + k/8) * 128 B, so the descriptor's leading-dimension byte
// offset (next core matrix along K) is 128 B and the stride-dimension byte
// offset (next 8-row group) is K * 16 B.
constexpr int kBfThreads = 128;
constexpr int kBfRows = 128;     // UMMA M
constexpr int kBfHidden = 64;    // the bf16 path's hidden width (reference default {64, 64})
constexpr int kBfHeadN = 16;     // head N: C*V logits + value + zero pad

struct Bf16Args {
  const float* obs;
  int32_t* actions;     // sampled actions [E, A, C] (nullptr: do not sample)
  double* logits;       // optional f64 logits [E, A, C*V]
  double* values;       // optional f64 values [E, A]
  uint32_t* error;
  int64_t E, A, a0, n;  // rows = E * n over agents [a0, a0 + n)
  int64_t env_offset;   // global id of env 0 (RNG keys)
  uint64_t h_step;      // absorb(mix64(substream(seed, kStreamActions)), step)
  const int64_t* step_dev;  // graph replay: step = *step_dev + step_add, hashed from h0
  int32_t step_add;
  uint64_t h0;
  int32_t D, Kp, C, V;  // obs_dim, padded K of layer 1, categories, choices
  int32_t pdl;          // launched with programmatic dependent launch
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t umma_desc(const void* base, uint32_t lbo, uint32_t sbo) {
  const uint32_t a = smem_addr(base);
  return static_cast<uint64_t>((a & 0x3FFFFu) >> 4) | (static_cast<uint64_t>(lbo >> 4) << 16) |
         (static_cast<uint64_t>(sbo >> 4) << 32) | (1ull << 46);  // bits 46-48: descriptor version 1
}

// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, N, M.
__host__ __device__ constexpr uint32_t umma_idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_addr(bar))
               : "memory");
}

__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  }
}

// 16 consecutive f32 TMEM columns of this thread's lane.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&v);
}

// byte offset of the 16-B chunk (row r, k-chunk kc) in a K-major canonical tile
__device__ __forceinline__ uint32_t tile_off(int r, int kc, int K) {
  return static_cast<uint32_t>(((r >> 3) * (K >> 3) + kc) * 128 + (r & 7) * 16);
}

__device__ __forceinline__ uint64_t mix64_d(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t absorb_d(uint64_t h, uint64_t v) {
  return mix64_d(h ^ (v + 0x9e3779b97f4a7c15ULL));
}

// smem carve (bytes): W1 [64 x Kp], W2 [64 x 64], W3 [16 x 64] bf16 operand
// tiles (resident), one A tile [128 x 64] shared by the three layers (layer l's
// epilogue writes layer l+1's A only after MMA l — the last reader of the
// tile — has completed), biases f32, mbarrier, TMEM slot.
__host__ __device__ constexpr int bf_image_bytes(int Kp) {
  return 64 * Kp * 2 + 64 * 64 * 2 + 16 * 64 * 2 + (64 + 64 + 16) * 4;
}
__host__ __device__ constexpr int bf_smem_bytes(int Kp) {
  return bf_image_bytes(Kp) + 128 * 64 * 2 + 16 + 16;
}
static_assert(bf_image_bytes(16) % 16 == 0 && bf_image_bytes(32) % 16 == 0 && bf_image_bytes(48) % 16 == 0,
              "image size");
constexpr int kBfTmemCols = 64;  // D1, D2 and the head all live in columns [0, 64)

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// sample_from_logits (sampler.hpp:18-30) on V register logits.
// The decision is first taken on f32 estimates (ex2.approx, MUFU) with a
// rigorous margin. Each estimate of exp(dd), dd = z - zmax <= 0, carries a
// relative error below |dd| 1.8e-7 (three f32 roundings of dd log2 e) plus
// 2^-22 (ex2.approx), i.e. an absolute error below 3.1e-7 since
// |dd| exp(dd) <= 1/e and total >= 1; with the f32 sums and the rounding of
// u, target and every cumulative sum stay within 4e-6 x total of their f64
// values. When no cumulative sum lies within 1e-5 x total of the target the
// f64 path (the reference arithmetic) picks the same action; it runs only
// for the rare rows that close.
template <int V>
__device__ __forceinline__ int sample_row_regs(const double* z, double u) {
  double zmax = z[0];
#pragma unroll
  for (int i = 1; i < V; ++i) zmax = zmax < z[i] ? z[i] : zmax;
  {
    float evf[V], totf = 0.0f;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float dd = static_cast<float>(z[i] - zmax);
      evf[i] = dd == 0.0f ? 1.0f : ex2_approx(dd * 1.4426950408889634f);
      totf += evf[i];
    }
    const float tgt = static_cast<float>(u) * totf;
    const float margin = 1e-5f * totf;
    float cum = 0.0f;
    int pick = V - 1;
    bool found = false, close = false;
#pragma unroll
    for (int i = 0; i + 1 < V; ++i) {
      cum += evf[i];
      close |= fabsf(tgt - cum) <= margin;
      if (!found && tgt < cum) {
        pick = i;
        found = true;
      }
    }
    if (!close) return pick;
  }
  double ev[V], total = 0.0;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const double dd = z[i] - zmax;
    ev[i] = 1.0;
    if (dd != 0.0) ev[i] = exp(dd);
    total = __dadd_rn(total, ev[i]);
  }
  const double target = __dmul_rn(u, total);
  double cum = 0.0;
  int pick = V - 1;
  bool found = false;
#pragma unroll
  for (int i = 0; i + 1 < V; ++i) {
    cum = __dadd_rn(cum, ev[i]);
    if (!found && target < cum) {
      pick = i;
      found = true;
    }
  }
  return pick;
}

// KP: layer-1 K (obs_dim padded to 16); C x V: the action space (Tag: 1 x 5
// discrete, 2 x 3 continuous).
template <int KP, int C, int V>
#ifndef WDG_BF16_MIN_BLOCKS
#define WDG_BF16_MIN_BLOCKS 6
#endif
__global__ void __launch_bounds__(kBfThreads, WDG_BF16_MIN_BLOCKS) policy_bf16_kernel(const uint8_t* __restrict__ image, Bf16Args a) {
  extern __shared__ __align__(128) uint8_t smb[];
  constexpr int KC1 = KP / 8;  // 16-B chunks per layer-1 row
  const int tid = threadIdx.x, warp = tid >> 5;
  if (a.pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  uint8_t* w1s = smb;
  uint8_t* w2s = w1s + 64 * KP * 2;
  uint8_t* w3s = w2s + 64 * 64 * 2;
  float* b1s = reinterpret_cast<float*>(w3s + 16 * 64 * 2);
  float* b2s = b1s + 64;
  float* b3s = b2s + 64;
  uint8_t* As = reinterpret_cast<uint8_t*>(b3s + 16);  // 16-B aligned (image size % 16 == 0)
  uint64_t* bar = reinterpret_cast<uint64_t*>(As + 128 * 64 * 2);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 2);
  constexpr int W = C * V;

  // The weights' smem image (bf16 operand tiles + f32 biases) was packed once
  // on the host (Policy::upload, bf16_image): a straight 16-B copy.
  {
    const uint4* src = reinterpret_cast<const uint4*>(image);
    uint4* dst = reinterpret_cast<uint4*>(smb);
    for (int i = tid; i < bf_image_bytes(KP) / 16; i += kBfThreads) dst[i] = __ldg(src + i);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                 "n"(kBfTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // weight tiles -> async proxy
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
  // everything above touched only the weights image; the observations (and
  // the actions this kernel overwrites) belong to the previous kernels
  if (a.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");

  constexpr uint32_t id1 = umma_idesc(128, 64), id3 = umma_idesc(128, 16);
  uint32_t phase = 0;
  const int64_t rows = a.E * a.n;
  const int64_t tiles = (rows + kBfRows - 1) / kBfRows;
  uint64_t h_step = a.h_step;
  if (a.step_dev != nullptr) h_step = absorb_d(a.h0, static_cast<uint64_t>(*a.step_dev + a.step_add));
  bool bad = false;

  // Row of tile `tile` owned by this thread, and its obs prefetched into
  // registers one tile ahead so the global latency overlaps the MMA chain.
  const bool small = rows < (int64_t{1} << 31);
  auto row_of = [&](int64_t tile, int64_t& e, int64_t& ag) {
    // tiles from the end: the step kernel wrote the last envs' observations
    // last, so their lines are the ones still in L2
    const int64_t r = (tiles - 1 - tile) * kBfRows + tid;
    const bool ok = r < rows;
    if (small) {  // 32-bit division (the common case)
      const uint32_t r32 = ok ? static_cast<uint32_t>(r) : 0u, n32 = static_cast<uint32_t>(a.n);
      const uint32_t e32 = r32 / n32;
      e = e32;
      ag = a.a0 + (r32 - e32 * n32);
    } else {
      e = ok ? r / a.n : 0;
      ag = ok ? a.a0 + (r - e * a.n) : 0;
    }
    return ok;
  };
  float xr[KP];
  const int D = a.D;
  auto fetch = [&](int64_t tile) {
    int64_t e, ag;
    const bool ok = tile < tiles && row_of(tile, e, ag);
    const float* src = a.obs + (e * a.A + ag) * D;
#pragma unroll
    for (int k = 0; k < KP; ++k) xr[k] = (ok && k < D) ? src[k] : 0.f;  // coherent: written by the step kernel
  };
  int64_t tile = blockIdx.x;
  fetch(tile);
  for (; tile < tiles; tile += gridDim.x) {
    int64_t e, ag;
    const bool valid = row_of(tile, e, ag);
    const int64_t grow = e * a.A + ag;
    // A <- this row's obs as bf16 (K padded with zeros)
#pragma unroll
    for (int kc = 0; kc < KC1; ++kc) {
      const float* x = xr + kc * 8;
#pragma unroll
      for (int k = 0; k < 8; ++k) bad |= !isfinite(x[k]);
      *reinterpret_cast<uint4*>(As + tile_off(tid, kc, KP)) =
          make_uint4(pack_bf16(x[0], x[1]), pack_bf16(x[2], x[3]), pack_bf16(x[4], x[5]), pack_bf16(x[6], x[7]));
    }
    fetch(tile + gridDim.x);
    // layers: MMA (one thread) -> commit -> everyone waits -> epilogue of row t
#pragma unroll 1
    for (int layer = 0; layer < 3; ++layer) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint8_t* B = layer == 0 ? w1s : (layer == 1 ? w2s : w3s);
        const int K = layer == 0 ? KP : 64;
        const uint32_t idesc = layer == 2 ? id3 : id1;
        for (int k = 0; k < K / 16; ++k) {
          umma_bf16(tmem, umma_desc(As + k * 256, 128, K * 16), umma_desc(B + k * 256, 128, K * 16), idesc,
                    k > 0 ? 1u : 0u);
        }
        umma_commit(bar);
      }
      bar_wait(bar, phase);
      phase ^= 1u;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (layer < 2) {
        // h = tanh(D + b) -> bf16 row of the next layer's A (the tile just consumed)
        const float* bias = layer == 0 ? b1s : b2s;
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          float v[16];
          tmem_ld16(tmem + lane_base + q4 * 16, v);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = tanh_fast(v[i] + bias[q4 * 16 + i]);
#pragma unroll
          for (int c2 = 0; c2 < 2; ++c2) {
            const float* x = v + c2 * 8;
            *reinterpret_cast<uint4*>(As + tile_off(tid, q4 * 2 + c2, 64)) =
                make_uint4(pack_bf16(x[0], x[1]), pack_bf16(x[2], x[3]), pack_bf16(x[4], x[5]),
                           pack_bf16(x[6], x[7]));
          }
        }
      } else {
        float v[16];
        tmem_ld16(tmem + lane_base, v);  // whole warp (.sync.aligned), rows past the end included
        if (valid) {
          double z[W];
#pragma unroll
          for (int i = 0; i < W; ++i) z[i] = static_cast<double>(v[i] + b3s[i]);
          if (a.logits) {
#pragma unroll
            for (int i = 0; i < W; ++i) a.logits[grow * W + i] = z[i];
          }
          if (a.values) a.values[grow] = static_cast<double>(v[W] + b3s[W]);
          if (a.actions) {
            // sample_actions keys (sampler.cpp:31-39): (seed', step, env, agent, category, 0)
            const uint64_t h_ag = absorb_d(absorb_d(h_step, static_cast<uint64_t>(a.env_offset + e)),
                                           static_cast<uint64_t>(ag));
#pragma unroll
            for (int c = 0; c < C; ++c) {
              const double u =
                  __ull2double_rn(absorb_d(absorb_d(h_ag, static_cast<uint64_t>(c)), 0) >> 11) * 0x1.0p-53;
              a.actions[grow * C + c] = sample_row_regs<V>(z + c * V, u);
            }
          }
        }
      }
    }
  }
  if (bad && a.error) atomicOr(a.error, kErrNonFinite);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kBfTmemCols)
                 : "memory");
  }
}

using BfKernel = void (*)(const uint8_t*, Bf16Args);
BfKernel bf16_kernel_for(int Kp, int C, int V) {
  if (C == 1 && V == 5) {
    if (Kp == 16) return policy_bf16_kernel<16, 1, 5>;
    if (Kp == 32) return policy_bf16_kernel<32, 1, 5>;
    if (Kp == 48) return policy_bf16_kernel<48, 1, 5>;
  }
  if (C == 2 && V == 3) {
    if (Kp == 16) return policy_bf16_kernel<16, 2, 3>;
    if (Kp == 32) return policy_bf16_kernel<32, 2, 3>;
    if (Kp == 48) return policy_bf16_kernel<48, 2, 3>;
  }
  return nullptr;
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
  if (dimage_) cudaFree(dimage_);
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
  if (bf16_supported()) {
    // bf16 smem image of policy_bf16_kernel: W1 [64 x Kp], W2 [64 x 64], head
    // [16 x 64] (C*V logit rows, the value row, zero rows) as UMMA canonical
    // K-major tiles (core matrix (r/8, k/8) at ((r/8)*(K/8) + k/8)*128 B, row
    // r%8 at +16 B), then b1, b2, head bias (f32).
    const int D = static_cast<int>(dims_.obs_dim);
    const int Kp = (D + 15) / 16 * 16;
    const int Wd = static_cast<int>(dims_.logits_width());
    std::vector<uint8_t> img(static_cast<size_t>(bf_image_bytes(Kp)), 0);
    auto bf = [](double v) {  // round-to-nearest-even f32 -> bf16 (what __floats2bfloat162_rn does)
      const float f = static_cast<float>(v);
      uint32_t u;
      std::memcpy(&u, &f, 4);
      u += 0x7FFFu + ((u >> 16) & 1u);
      return static_cast<uint16_t>(u >> 16);
    };
    auto put = [&](size_t base, int r, int k, int K, double v) {
      const size_t off = base + static_cast<size_t>(((r >> 3) * (K >> 3) + (k >> 3)) * 128 + (r & 7) * 16 + (k & 7) * 2);
      const uint16_t h = bf(v);
      std::memcpy(img.data() + off, &h, 2);
    };
    const double* w1 = host_.data();
    const double* b1 = w1 + 64 * D;
    const double* w2 = b1 + 64;
    const double* b2 = w2 + 64 * 64;
    const double* hw = b2 + 64;
    const double* hb = hw + Wd * 64;
    const double* vw = hb + Wd;
    const double vb = vw[64];
    const size_t o_w2 = static_cast<size_t>(64 * Kp * 2), o_w3 = o_w2 + 64 * 64 * 2, o_b = o_w3 + 16 * 64 * 2;
    for (int n = 0; n < 64; ++n)
      for (int k = 0; k < D; ++k) put(0, n, k, Kp, w1[n * D + k]);
    for (int n = 0; n < 64; ++n)
      for (int k = 0; k < 64; ++k) put(o_w2, n, k, 64, w2[n * 64 + k]);
    for (int n = 0; n <= Wd; ++n)
      for (int k = 0; k < 64; ++k) put(o_w3, n, k, 64, n < Wd ? hw[n * 64 + k] : vw[k]);
    float* bias = reinterpret_cast<float*>(img.data() + o_b);
    for (int i = 0; i < 64; ++i) {
      bias[i] = static_cast<float>(b1[i]);
      bias[64 + i] = static_cast<float>(b2[i]);
    }
    for (int i = 0; i < 16; ++i) bias[128 + i] = i < Wd ? static_cast<float>(hb[i]) : (i == Wd ? static_cast<float>(vb) : 0.f);
    if (dimage_ == nullptr) cuda_check(cudaMalloc(&dimage_, img.size()), "cudaMalloc(policy image)");
    cuda_check(cudaMemcpy(dimage_, img.data(), img.size(), cudaMemcpyHostToDevice), "policy image upload");
  }
  dirty_ = false;
}

bool Policy::bf16_supported() const {
  return dims_.hidden.size() == 2 && dims_.hidden[0] == kBfHidden && dims_.hidden[1] == kBfHidden &&
         bf16_kernel_for(static_cast<int>((dims_.obs_dim + 15) / 16 * 16), static_cast<int>(dims_.num_categories),
                         static_cast<int>(dims_.num_choices)) != nullptr;
}

void Policy::forward_sample_bf16(const float* obs, int64_t E, int64_t A, int64_t a0, int64_t a1,
                                 int32_t* actions, double* logits, double* values, const SampleKeys& keys,
                                 cudaStream_t st, uint32_t* error, bool pdl) const {
  if (obs == nullptr) raise(Errc::invalid_argument, "policy forward: null observations");
  if (a0 < 0 || a1 > A || a0 > a1) raise(Errc::index_out_of_range, "policy forward: bad agent range");
  if (!bf16_supported()) {
    raise(Errc::invalid_config, "policy forward: the bf16 tensor-core path covers hidden {64, 64}, "
                                "the Tag action spaces (1 x 5, 2 x 3) and obs_dim <= 48");
  }
  if (E == 0 || a1 == a0) return;
  upload();
  Bf16Args b{};
  b.obs = obs;
  b.actions = actions;
  b.logits = logits;
  b.values = values;
  b.error = error;
  b.E = E;
  b.A = A;
  b.a0 = a0;
  b.n = a1 - a0;
  b.env_offset = keys.env_offset;
  b.h_step = keys.h_step;
  b.step_dev = keys.step_dev;
  b.step_add = keys.step_add;
  b.h0 = keys.h0;
  b.D = static_cast<int32_t>(dims_.obs_dim);
  b.Kp = static_cast<int32_t>((dims_.obs_dim + 15) / 16 * 16);
  b.C = static_cast<int32_t>(dims_.num_categories);
  b.V = static_cast<int32_t>(dims_.num_choices);
  const BfKernel kern = bf16_kernel_for(b.Kp, b.C, b.V);
  const int smem = bf_smem_bytes(b.Kp);
  cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
             "policy bf16 smem attr");
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // Resident CTAs per SM: registers, shared memory (+1 KB reserved per CTA)
  // and TMEM (512 columns per SM).
  cudaFuncAttributes fa{};
  cuda_check(cudaFuncGetAttributes(&fa, kern), "policy bf16 attributes");
  int smem_sm = 228 * 1024;
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  const int by_regs = 65536 / std::max(1, fa.numRegs * kBfThreads);
  const int by_smem = smem_sm / (smem + static_cast<int>(fa.sharedSizeBytes) + 1024);
  per_sm = std::max(1, std::min({by_regs, by_smem, 512 / kBfTmemCols}));
#ifdef WDG_TUNING
  if (std::getenv("WDG_DEBUG_POLICY")) {
    std::fprintf(stderr, "policy bf16: regs %d smem %d -> %d CTAs/SM\n", fa.numRegs, smem, per_sm);
  }
#endif
  const int64_t tiles = (E * b.n + kBfRows - 1) / kBfRows;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(tiles, int64_t{sms} * per_sm)));
  b.pdl = pdl ? 1 : 0;
  if (pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(kBfThreads);
    cfg.dynamicSmemBytes = static_cast<size_t>(smem);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cuda_check(cudaLaunchKernelEx(&cfg, kern, static_cast<const uint8_t*>(dimage_), b), "policy bf16 kernel");
    return;
  }
  kern<<<grid, kBfThreads, smem, st>>>(dimage_, b);
  cuda_check(cudaGetLastError(), "policy bf16 kernel");
}

void Policy::forward_agents(const float* obs, int64_t E, int64_t A, int64_t a0, int64_t a1, double* logits,
                            double* values, int32_t precision, cudaStream_t st,
                            uint32_t* error) const {
  if (obs == nullptr) raise(Errc::invalid_argument, "policy forward: null observations");
  if (a0 < 0 || a1 > A || a0 > a1) raise(Errc::index_out_of_range, "policy forward: bad agent range");
  if (precision == kPolicyBF16) {
    forward_sample_bf16(obs, E, A, a0, a1, nullptr, logits, values, SampleKeys{}, st, error);
    return;
  }
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
