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

#include "device_ref.cuh"
#include "kernels.hpp"
#include "tag_params.hpp"

namespace wdg {
namespace {

#ifndef WDG_SAMPLE_PASS
#define WDG_SAMPLE_PASS 2
#endif
constexpr int kSamplePass = WDG_SAMPLE_PASS;  // vec4 layout: agents whose logits are loaded per pass
static_assert(kSamplePass == 1 || kSamplePass == 2 || kSamplePass == 4, "sample pass");

// ---- TMA bulk copies (cp.async.bulk) + mbarrier, raw PTX ---------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// global -> shared bulk copy, completion counted on `bar` (16-B aligned, size % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// shared -> global TMA bulk store, tracked by the issuing thread's bulk group
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

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
        const double d = zv[i] - zmax;  // exp(0) == 1 exactly: skip it
        ev[i] = 1.0;
        if (d != 0.0) ev[i] = exp(d);
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
  int32_t lattice_ok;  // all positions integral (discrete lattice K-NN valid)
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
  uint16_t* cellknn;  // lattice: per-cell top-(K+1) lists
  uint8_t* cellact;   // grid: cell holds an active agent
  int32_t* celltag;   // lattice (LEAN): lowest-index tagger per cell
  uint16_t* cellq;    // lattice (LEAN): compacted active cells
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
  s.cellknn = reinterpret_cast<uint16_t*>(b + p.off_cellknn);
  s.cellact = b + p.off_cellact;
  s.celltag = reinterpret_cast<int32_t*>(b + p.off_celltag);
  s.cellq = reinterpret_cast<uint16_t*>(b + p.off_cellq);
  return s;
}

// Staged partial-observation rows leave with plain (write-back) stores: they
// measured faster than streaming (.cs) stores — C2 98.5 vs 101.1 us/step,
// continuous A = 1000 360 vs 378 — while the wide full-observation writers,
// HBM-bound at 0.9 of peak, keep .cs (261 vs 256 us/step with write-back at
// A = 500 full).
template <class T>
__device__ __forceinline__ void st_rows(T* p, T v) { *p = v; }

// ---- lattice shells (discrete K-NN) ------------------------------------------
// All lattice offsets (dx, dy) with dx^2+dy^2 <= kShellR2, sorted by d2 and
// grouped into shells of equal d2. Visiting shells in order makes the K-NN
// search stop as soon as the K-th best is strictly closer than the next shell.
constexpr int kShellR = 12;
constexpr int kShellR2 = kShellR * kShellR;
constexpr int kMaxShellOffsets = 4 * kShellR2 + 4 * kShellR + 1;  // >= #offsets in the disk
constexpr int kMaxShells = kShellR2 + 2;
__constant__ int16_t c_shell_off[kMaxShellOffsets];  // (dx + 64) | (dy + 64) << 8
__constant__ int16_t c_shell_begin[kMaxShells + 1];
__constant__ int16_t c_shell_d2[kMaxShells];
__constant__ int32_t c_num_shells;

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
    if (p.lattice) return iv;
    return static_cast<int>((static_cast<uint32_t>(iv) * static_cast<uint32_t>(p.gc)) /
                            static_cast<uint32_t>(g));
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

// mark_active: also flag cells holding an active agent (used when the
// active set is final at build time: placement); otherwise flags are zeroed
// and set after tag resolution.
template <bool CONT>
// cell_tagger: the cells are lattice points (every item of a cell sits at the
// same position), so after the index sort s.cfill[c] is set to the cell's
// lowest-index tagger (-1 if none): the tagger resolve credits
// (tag_env.cpp:430-434), found once per cell instead of once per runner.
__device__ void build_grid(const EnvSmem& s, const TagDevConfig& p, int* scratch,
                           bool mark_active = false, bool cell_tagger = false) {
  const int nthr = blockDim.x, tid = threadIdx.x;
  for (int c = tid; c <= p.ncells; c += nthr) {
    s.cfill[c] = 0;
    if (c < p.ncells) s.cellact[c] = 0;
  }
  __syncthreads();
  for (int a = tid; a < p.A; a += nthr) {
    const int c = cell_coord<CONT>(s.y[a], p) * p.gc + cell_coord<CONT>(s.x[a], p);
    s.cellof[a] = static_cast<uint16_t>(c);
    atomicAdd(&s.cfill[c], 1);
    if (mark_active && s.act[a]) s.cellact[c] = 1;
  }
  __syncthreads();
  block_scan_cells(s, p.ncells, p.A, scratch);
  __syncthreads();
  for (int a = tid; a < p.A; a += nthr) {
    const int slot = atomicAdd(&s.cfill[s.cellof[a]], 1);
    s.items[slot] = static_cast<uint16_t>(a);
  }
  __syncthreads();
  // Each cell's items in ascending agent index (the order NeighborGrid::build
  // produces with its serial counting sort, neighbor_grid.hpp:31-43).
  for (int c = tid; c < p.ncells; c += nthr) {
    const int b = s.cstart[c], e = s.cstart[c + 1];
    if (e - b <= 4) {  // typical lattice cell: a 5-comparator network in registers
      if (e - b < 2) {
        if (cell_tagger) s.cfill[c] = (e > b && s.tag[s.items[b]]) ? static_cast<int>(s.items[b]) : -1;
        continue;
      }
      int v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = b + q < e ? static_cast<int>(s.items[b + q]) : 0x7fffffff;
      auto cx = [&](int i, int j) {
        const int lo = min(v[i], v[j]), hi = max(v[i], v[j]);
        v[i] = lo;
        v[j] = hi;
      };
      cx(0, 1);
      cx(2, 3);
      cx(0, 2);
      cx(1, 3);
      cx(1, 2);
      int first = -1;
#pragma unroll
      for (int q = 3; q >= 0; --q) {
        if (b + q < e) {
          s.items[b + q] = static_cast<uint16_t>(v[q]);
          if (cell_tagger && s.tag[v[q]]) first = v[q];
        }
      }
      if (cell_tagger) s.cfill[c] = first;
      continue;
    }
    for (int i = b + 1; i < e; ++i) {
      const uint16_t v = s.items[i];
      int k = i - 1;
      while (k >= b && s.items[k] > v) {
        s.items[k + 1] = s.items[k];
        --k;
      }
      s.items[k + 1] = v;
    }
    if (cell_tagger) {
      int first = -1;
      for (int i = b; i < e && first < 0; ++i)
        if (s.tag[s.items[i]]) first = s.items[i];
      s.cfill[c] = first;
    }
  }
  __syncthreads();
}

// Lattice K-NN per CELL: the top-(K+1) agents by (d2, index) seen from lattice
// point c. Shells of equal d2 are visited in increasing order and, inside a
// shell, candidates are taken in increasing index by repeated minimum over the
// shell's (index-sorted) cells — no insertion network. An agent's K nearest
// are this list minus itself. Returns the count found (< kk only if the
// precomputed disk is exhausted; the caller then falls back per agent).
// k-way merge of the N index-sorted cells of one shell, one cursor per cell
// in registers, appending up to kk - found indices in increasing order.
template <int N>
__device__ __forceinline__ void merge_shell(const EnvSmem& s, int g, int cx, int cy, int ob,
                                            uint16_t* out, int& found, int kk) {
  int cur[N], end[N], head[N];
#pragma unroll
  for (int q = 0; q < N; ++q) {
    cur[q] = 0;
    end[q] = 0;
    const int packed = c_shell_off[ob + q];
    const int gx = cx + (packed & 0xff) - 64;
    const int gy = cy + ((packed >> 8) & 0xff) - 64;
    if (static_cast<unsigned>(gx) < static_cast<unsigned>(g) &&
        static_cast<unsigned>(gy) < static_cast<unsigned>(g)) {
      const int c2 = gy * g + gx;
      cur[q] = s.cstart[c2];
      end[q] = s.cstart[c2 + 1];
    }
    head[q] = cur[q] < end[q] ? static_cast<int>(s.items[cur[q]]) : 0x7fffffff;
  }
  while (found < kk) {
    int best = head[0], bq = 0;
#pragma unroll
    for (int q = 1; q < N; ++q) {
      if (head[q] < best) {
        best = head[q];
        bq = q;
      }
    }
    if (best == 0x7fffffff) return;
    out[found++] = static_cast<uint16_t>(best);
#pragma unroll
    for (int q = 0; q < N; ++q) {
      if (q == bq) {
        ++cur[q];
        head[q] = cur[q] < end[q] ? static_cast<int>(s.items[cur[q]]) : 0x7fffffff;
      }
    }
  }
}

__device__ int cell_knn(const EnvSmem& s, const TagDevConfig& p, int c, uint16_t* out, int kk) {
  const int g = p.gc;
  const int cy = c / g, cx = c - cy * g;
  const int ns = c_num_shells;
  // shell 0 (d2 = 0) is the cell itself: its sorted items, copied directly
  int found = 0;
  {
    const int e = s.cstart[c + 1];
    for (int t = s.cstart[c]; t < e && found < kk; ++t) out[found++] = s.items[t];
  }
  for (int sh = 1; sh < ns && found < kk; ++sh) {
    const int ob = c_shell_begin[sh], oe = c_shell_begin[sh + 1];
    if (oe - ob == 4) {
      merge_shell<4>(s, g, cx, cy, ob, out, found, kk);
      continue;
    }
    if (oe - ob == 8) {
      merge_shell<8>(s, g, cx, cy, ob, out, found, kk);
      continue;
    }
    int last = -1;
    while (found < kk) {
      int best = 0x7fffffff;
      for (int o = ob; o < oe; ++o) {
        const int packed = c_shell_off[o];
        const int gx = cx + (packed & 0xff) - 64;
        const int gy = cy + ((packed >> 8) & 0xff) - 64;
        if (static_cast<unsigned>(gx) >= static_cast<unsigned>(g) ||
            static_cast<unsigned>(gy) >= static_cast<unsigned>(g))
          continue;
        const int c2 = gy * g + gx;
        const int e = s.cstart[c2 + 1];
        for (int t = s.cstart[c2]; t < e; ++t) {
          const int j = s.items[t];
          if (j > last) {
            best = j < best ? j : best;
            break;
          }
        }
      }
      if (best == 0x7fffffff) break;
      out[found++] = static_cast<uint16_t>(best);
      last = best;
    }
  }
  return found;
}

// ---- lattice grid + per-cell lists for the LEAN kernel ---------------------
// Counting sort of the agents into CSR lattice cells in scatter (atomic) order:
// no per-cell index sort, because nothing downstream needs one — the
// lowest-index tagger of each cell comes from an atomicMin while counting,
// the per-cell K-NN lists insert (d2, index) keys, and find_tagger's cell scan
// takes the minimum index. Thread t owns agents 4t..4t+3 (A % 4 == 0).
// scratch int slot of build_cell_lists_keys' queue length: past the tracker's
// per-warp double slots (kSlotT / kSlotR for up to 32 warps: ints 32..159)
constexpr int kCellQCount = 160;
constexpr int kObsChunk = 162;  // LEAN observation phase: next 32-agent chunk

__device__ void build_grid_lattice(const EnvSmem& s, const TagDevConfig& p, int* scratch, bool mark_active) {
  const int nthr = blockDim.x, tid = threadIdx.x;
  if (tid == 0) scratch[kCellQCount] = 0;
  for (int c = tid; c <= p.ncells; c += nthr) {
    s.cfill[c] = 0;
    if (c < p.ncells) {
      s.cellact[c] = 0;
      s.celltag[c] = 0x7fffffff;
    }
  }
  __syncthreads();
  for (int a0 = 4 * tid; a0 < p.A; a0 += 4 * nthr) {
    const float4 x4 = *reinterpret_cast<const float4*>(s.x + a0);
    const float4 y4 = *reinterpret_cast<const float4*>(s.y + a0);
    const uint32_t tg4 = *reinterpret_cast<const uint32_t*>(s.tag + a0);
    const uint32_t ac4 = mark_active ? *reinterpret_cast<const uint32_t*>(s.act + a0) : 0u;
    const float xs[4] = {x4.x, x4.y, x4.z, x4.w}, ys[4] = {y4.x, y4.y, y4.z, y4.w};
    int cl[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      cl[k] = cell_coord<false>(ys[k], p) * p.gc + cell_coord<false>(xs[k], p);
      atomicAdd(&s.cfill[cl[k]], 1);
      if ((tg4 >> (8 * k)) & 0xffu) atomicMin(&s.celltag[cl[k]], a0 + k);
      if (mark_active && ((ac4 >> (8 * k)) & 0xffu)) s.cellact[cl[k]] = 1;
    }
    *reinterpret_cast<uint2*>(s.cellof + a0) =
        make_uint2(static_cast<uint32_t>(cl[0]) | (static_cast<uint32_t>(cl[1]) << 16),
                   static_cast<uint32_t>(cl[2]) | (static_cast<uint32_t>(cl[3]) << 16));
  }
  __syncthreads();
  if (p.ncells > 1024) {
    block_scan_cells(s, p.ncells, p.A, scratch);
  } else if ((tid >> 5) == 0) {
    // one warp scans the cell counts (C2: 400 cells, 13 per lane): two
    // block-scan barriers fewer, 97.0 vs 98.5 us/step at C2
    const int lane = tid & 31, n = p.ncells;
    const int chunk = (n + 31) / 32;
    const int b = lane * chunk, e = min(b + chunk, n);
    int local = 0;
    for (int c = b; c < e; ++c) local += s.cfill[c];
    int incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    int off = incl - local;
    for (int c = b; c < e; ++c) {
      const int v = s.cfill[c];
      s.cstart[c] = off;
      s.cfill[c] = off;
      off += v;
    }
    if (lane == 0) s.cstart[n] = p.A;
  }
  __syncthreads();
  for (int a0 = 4 * tid; a0 < p.A; a0 += 4 * nthr) {
    const uint2 c2 = *reinterpret_cast<const uint2*>(s.cellof + a0);
    const int cl[4] = {static_cast<int>(c2.x & 0xffffu), static_cast<int>(c2.x >> 16),
                       static_cast<int>(c2.y & 0xffffu), static_cast<int>(c2.y >> 16)};
#pragma unroll
    for (int k = 0; k < 4; ++k) s.items[atomicAdd(&s.cfill[cl[k]], 1)] = static_cast<uint16_t>(a0 + k);
  }
  __syncthreads();
}

// Lattice K-NN per CELL by key insertion: every agent of the shells around
// lattice point c, visited in increasing d2, enters a register top-(K+1) of
// 32-bit keys (d2 << 16 | index) — the (d2, index) total order as one
// unsigned compare, inserted by a branchless min/max chain in any item order.
// Stops once the list is full and the next shell is strictly farther. Same
// list as cell_knn (the order is total). Returns the count found (< KK only
// if the precomputed disk is exhausted; the caller falls back per agent).
template <int KK>
__device__ __forceinline__ int cell_knn_keys(const EnvSmem& s, const TagDevConfig& p, int c, uint16_t* out) {
  const int g = p.gc;
  const int cy = c / g, cx = c - cy * g;
  uint32_t l[KK];
#pragma unroll
  for (int t = 0; t < KK; ++t) l[t] = 0xffffffffu;
  int found = 0;
  const int ns = c_num_shells;
  for (int sh = 0; sh < ns; ++sh) {
    const uint32_t d2 = static_cast<uint32_t>(c_shell_d2[sh]);
    if (found >= KK && (l[KK - 1] >> 16) < d2) break;
    const uint32_t hi = d2 << 16;
    const int ob = c_shell_begin[sh], oe = c_shell_begin[sh + 1];
    for (int o = ob; o < oe; ++o) {
      const int packed = c_shell_off[o];
      const int gx = cx + (packed & 0xff) - 64;
      const int gy = cy + ((packed >> 8) & 0xff) - 64;
      if (static_cast<unsigned>(gx) >= static_cast<unsigned>(g) ||
          static_cast<unsigned>(gy) >= static_cast<unsigned>(g))
        continue;
      const int c2 = gy * g + gx;
      const int e = s.cstart[c2 + 1];
      int t = s.cstart[c2];
      found += e - t;
      // two keys per pass: the second min/max chain trails the first by one
      // stage instead of waiting for its end
      for (; t + 1 < e; t += 2) {
        uint32_t k0 = hi | s.items[t], k1 = hi | s.items[t + 1];
#pragma unroll
        for (int q = 0; q < KK; ++q) {
          const uint32_t lo = min(l[q], k0);
          k0 = max(l[q], k0);
          l[q] = lo;
        }
#pragma unroll
        for (int q = 0; q < KK; ++q) {
          const uint32_t lo = min(l[q], k1);
          k1 = max(l[q], k1);
          l[q] = lo;
        }
      }
      if (t < e) {
        uint32_t key = hi | s.items[t];
#pragma unroll
        for (int q = 0; q < KK; ++q) {
          const uint32_t lo = min(l[q], key);
          key = max(l[q], key);
          l[q] = lo;
        }
      }
    }
  }
  const int n = found < KK ? found : KK;
#pragma unroll
  for (int t = 0; t < KK; ++t)
    if (t < n) out[t] = static_cast<uint16_t>(l[t] & 0xffffu);
  return n;
}

// Lists only for cells holding an active agent, compacted first so every
// lane of a warp works on one (inactive agents observe zeros; tagged runners
// leave many cells without an active agent). The queue length lives in
// scratch[kCellQCount], zeroed by build_grid_lattice.
__device__ __forceinline__ void build_cell_lists_keys(const EnvSmem& s, const TagDevConfig& p, int* scratch) {
  const int lane = threadIdx.x & 31;
  for (int c0 = threadIdx.x & ~31; c0 < p.ncells; c0 += blockDim.x) {
    const int c = c0 + lane;
    const bool act = c < p.ncells && s.cellact[c];
    const unsigned m = __ballot_sync(0xffffffffu, act);
    int base = 0;
    if (lane == 0 && m) base = atomicAdd(&scratch[kCellQCount], __popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (act) s.cellq[base + __popc(m & ((1u << lane) - 1u))] = static_cast<uint16_t>(c);
    else if (c < p.ncells) s.cfill[c] = 0;
  }
  __syncthreads();
  const int n = scratch[kCellQCount];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int c = s.cellq[i];
    s.cfill[c] = cell_knn_keys<6>(s, p, c, s.cellknn + c * 6);
  }
}

// Per-cell top-(K+1) lists for every cell holding an active agent (only those
// are ever looked up); s.cfill[c] = entries found.
// Performance-analysis ablation bits (TagLaunch::ablate): only a tuning
// build (-DWDG_TUNING) reads them; the product build folds them to 0, so no
// launch of the shipped library can skip work.
__device__ __forceinline__ uint32_t ablate_bits(const TagLaunch& L) {
#ifdef WDG_TUNING
  return L.ablate;
#else
  (void)L;
  return 0u;
#endif
}

__device__ __forceinline__ void build_cell_lists(const EnvSmem& s, const TagDevConfig& p, uint32_t ablate) {
  const int kk = p.K + 1;
  for (int c = threadIdx.x; c < p.ncells; c += blockDim.x) {
    if (ablate & 2u) {
      for (int t = 0; t < kk; ++t) s.cellknn[c * kk + t] = static_cast<uint16_t>(t);
      s.cfill[c] = kk;
      continue;
    }
    s.cfill[c] = s.cellact[c] ? cell_knn(s, p, c, s.cellknn + c * kk, kk) : 0;
  }
}

// ---- exact top-K under the (d2, index) total order ------------------------
// Same selection as select_k_nearest_brute (tag_env.cpp:225-237) and
// NeighborGrid::k_nearest (neighbor_grid.hpp:62-111): unique because the
// order is total, so any visiting order gives the identical list. EXACT:
// k == MAXK at compile time (no runtime guards in the insertion network).
template <int MAXK, bool EXACT>
struct TopK {
  float d[MAXK];
  int i[MAXK];
  float wd;
  int wi;
  int k;
  __device__ __forceinline__ void init(int kk) {
    k = EXACT ? MAXK : kk;
#pragma unroll
    for (int t = 0; t < MAXK; ++t) {
      d[t] = __int_as_float(0x7f800000);
      i[t] = 0x7fffffff;
    }
    wd = __int_as_float(0x7f800000);
    wi = 0x7fffffff;
  }
  __device__ __forceinline__ bool full() const { return wi != 0x7fffffff; }
  __device__ __forceinline__ bool admits(float dd, int j) const {
    return dd < wd || (dd == wd && j < wi);
  }
  // Candidate j above every index already held (ascending scans): ties then
  // never displace, so the admission and shift tests drop the index compare.
  __device__ __forceinline__ void consider_next(float dd, int j) {
    if (!(dd < wd)) return;
    bool placed = false;
#pragma unroll
    for (int t = MAXK - 1; t >= 0; --t) {
      if (EXACT || t < k) {
        const bool shift = t > 0 && dd < d[t - 1];
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
    if (EXACT) {
      wd = d[MAXK - 1];
      wi = i[MAXK - 1];
    } else {
#pragma unroll
      for (int t = 0; t < MAXK; ++t) {
        if (t == k - 1) {
          wd = d[t];
          wi = i[t];
        }
      }
    }
  }
  // Any candidate order (ring search): the full (d2, index) compare. (A
  // branchless shift here measured 10% slower on the continuous ring search
  // at A = 1000: ring candidates arrive roughly nearest-first, so most warps
  // skip the insertion entirely after admits().)
  __device__ __forceinline__ void consider(float dd, int j) {
    if (!admits(dd, j)) return;
    bool placed = false;
#pragma unroll
    for (int t = MAXK - 1; t >= 0; --t) {
      if (EXACT || t < k) {
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
    if (EXACT) {
      wd = d[MAXK - 1];
      wi = i[MAXK - 1];
    } else {
#pragma unroll
      for (int t = 0; t < MAXK; ++t) {
        if (t == k - 1) {
          wd = d[t];
          wi = i[t];
        }
      }
    }
  }
};

__device__ __forceinline__ float d2_of(float ax, float ay, float bx, float by) {
  const float dx = __fsub_rn(bx, ax);
  const float dy = __fsub_rn(by, ay);
  return __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
}

// Rings 0 and 1 of a ring search together: the 3 x 3 block around cell
// (cx, cy) is at most 3 row ranges (the CSR is row-major, so cells gx0..gx1
// of a row are contiguous in items), walked as ONE flattened loop: lanes
// diverge on the block's total count instead of on 9 per-cell counts.
// Visiting ring 1 without the ring-1 bound test only adds candidates, so a
// search that keeps the exact smallest (d2, index) entries is unchanged.
// put2 takes candidates two at a time (independent loads and keys in flight
// together); put takes the odd one out.
template <typename F, typename F2>
__device__ __forceinline__ void scan_block3(const EnvSmem& s, int gc, int cx, int cy, F&& put, F2&& put2) {
  const int gx0 = max(cx - 1, 0), gx1 = min(cx + 1, gc - 1);
  const int gy0 = max(cy - 1, 0), gy1 = min(cy + 1, gc - 1);
  const int* rs = s.cstart + gy0 * gc;
  const int b0 = rs[gx0], e0 = rs[gx1 + 1];
  int b1 = 0, e1 = 0, b2 = 0, e2 = 0;
  if (gy0 + 1 <= gy1) {
    b1 = rs[gc + gx0];
    e1 = rs[gc + gx1 + 1];
  }
  if (gy0 + 2 <= gy1) {
    b2 = rs[2 * gc + gx0];
    e2 = rs[2 * gc + gx1 + 1];
  }
  const int n0 = e0 - b0, n01 = n0 + (e1 - b1), n = n01 + (e2 - b2);
  const int d1 = b1 - n0, d2 = b2 - n01;
  auto at = [&](int t) { return s.items[t + (t < n0 ? b0 : (t < n01 ? d1 : d2))]; };
  int t = 0;
  for (; t + 1 < n; t += 2) put2(at(t), at(t + 1));
  if (t < n) put(at(t));
}

// Generic ring search over the bucket grid (continuous / non-lattice).
template <bool CONT, int MAXK, bool EXACT>
__device__ void knn_rings(const EnvSmem& s, const TagDevConfig& p, int a, TopK<MAXK, EXACT>& top,
                          bool integral = true) {
  const float sx = s.x[a], sy = s.y[a];
  const int gc = p.gc;
  const int cx = cell_coord<CONT>(sx, p), cy = cell_coord<CONT>(sy, p);
  const int maxr = max(max(cx, gc - 1 - cx), max(cy, gc - 1 - cy));
  // Continuous: the agent's distance to its own cell's nearest edge tightens
  // the ring bound, and whole cells whose rectangle is farther than the
  // current K-th best are skipped. Both use cells widened by 1e-3 of a cell
  // (float cell assignment) and a (1 - 1e-5) factor, so a skipped cell can
  // never hold an admissible candidate, ties included.
  const double cs = p.cell_size;
  const double edge_in = CONT ? fmax(0.0, fmin(fmin(static_cast<double>(sx) - cx * cs, (cx + 1) * cs - sx),
                                               fmin(static_cast<double>(sy) - cy * cs, (cy + 1) * cs - sy)) -
                                                  1e-3 * cs)
                              : 0.0;
  if (CONT) {
    auto put = [&](int j) {
      if (j != a) top.consider(d2_of(sx, sy, s.x[j], s.y[j]), j);
    };
    scan_block3(s, gc, cx, cy, put, [&](int j0, int j1) {
      put(j0);
      put(j1);
    });
  }
  for (int r = CONT ? 2 : 0; r <= maxr; ++r) {
    if (r > 0 && top.full()) {
      // Every point in rings >= r is farther than this bound (SURVEY.md §8a
      // a6; cf. the reference's ring margin, neighbor_grid.hpp:90-96).
      float lb2;
      if (CONT) {
        const double lb = fmax(0.0, (r - 1) - 1e-3) * cs + edge_in;
        lb2 = static_cast<float>(lb * lb * (1.0 - 1e-5));
      } else {
        // integral positions sit on their cell's lower edge: one more unit
        const float lb = static_cast<float>((r - 1) * p.lattice_w + (integral ? 1 : 0));
        lb2 = lb * lb;
      }
      if (top.wd < lb2) break;
    }
    const int y0 = cy - r, y1 = cy + r, x0 = cx - r, x1 = cx + r;
    for (int gy = max(y0, 0); gy <= min(y1, gc - 1); ++gy) {
      const bool edge = (gy == y0 || gy == y1);
      const int step = edge ? 1 : max(x1 - x0, 1);
      for (int gx = x0; gx <= x1; gx += step) {
        if (gx < 0 || gx >= gc) continue;
        if (CONT && r > 1 && top.full()) {
          const double lo_x = (gx - 1e-3) * cs, hi_x = (gx + 1 + 1e-3) * cs;
          const double lo_y = (gy - 1e-3) * cs, hi_y = (gy + 1 + 1e-3) * cs;
          const double dx = fmax(0.0, fmax(lo_x - sx, sx - hi_x));
          const double dy = fmax(0.0, fmax(lo_y - sy, sy - hi_y));
          if (static_cast<float>((dx * dx + dy * dy) * (1.0 - 1e-5)) > top.wd) continue;
        }
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

// Continuous ring search with 32-bit keys: the same rings, bounds and cell
// pruning as knn_rings, but a candidate is (truncated d2 bits << b | index,
// b = index bits): one unsigned compare admits it, and an admitted key enters
// a branchless min/max chain of K + 1 keys instead of the (d2, index) shift
// network. The kept order is the exact (d2, index) order of the first K
// whenever the K + 1 kept keys have strictly increasing truncated d2
// (truncation is monotone: every other candidate, visited or not, then has a
// strictly larger truncated and so exact d2; the ring bound and the pruning
// use an upper bound of the K-th d2). Otherwise (an exact tie or a relative
// gap below 2^-(23-b)) it returns false and the caller runs the exact search.
template <int MAXK, bool EXACT>
__device__ __forceinline__ bool knn_rings_keys(const EnvSmem& s, const TagDevConfig& p, int a,
                                               TopK<MAXK, EXACT>& top) {
  constexpr int KK = MAXK + 1;
  const int b = 32 - __clz(max(p.A - 1, 1));
  const int S = b - 1;  // (31 - S) d2 bits + b index bits = 32
  uint32_t l[KK];
#pragma unroll
  for (int t = 0; t < KK; ++t) l[t] = 0xffffffffu;
  const float sx = s.x[a], sy = s.y[a];
  const int gc = p.gc;
  const int cx = cell_coord<true>(sx, p), cy = cell_coord<true>(sy, p);
  const int maxr = max(max(cx, gc - 1 - cx), max(cy, gc - 1 - cy));
  const double cs = p.cell_size;
  const double edge_in = fmax(0.0, fmin(fmin(static_cast<double>(sx) - cx * cs, (cx + 1) * cs - sx),
                                        fmin(static_cast<double>(sy) - cy * cs, (cy + 1) * cs - sy)) -
                                       1e-3 * cs);
  auto key_of = [&](int j) {
    const uint32_t d2b = __float_as_uint(d2_of(sx, sy, s.x[j], s.y[j]));
    return j == a ? 0xffffffffu : (((d2b >> S) << b) | static_cast<uint32_t>(j));
  };
  // branchless: a key above every kept one passes the chain unchanged
  auto insert = [&](uint32_t key) {
#pragma unroll
    for (int q = 0; q < KK; ++q) {
      const uint32_t lo = min(l[q], key);
      key = max(l[q], key);
      l[q] = lo;
    }
  };
  auto put = [&](int j) {
    const uint32_t key = key_of(j);
    if (key < l[KK - 1]) insert(key);
  };
  // two keys per admission test: the second chain trails the first by one
  // stage instead of waiting for it
  scan_block3(s, gc, cx, cy, put, [&](int j0, int j1) {
    const uint32_t k0 = key_of(j0), k1 = key_of(j1);
    if (min(k0, k1) < l[KK - 1]) {
      insert(k0);
      insert(k1);
    }
  });  // rings 0 and 1
  for (int r = 2; r <= maxr; ++r) {
    const float wd_up = __uint_as_float(min(((l[MAXK - 1] >> b) + 1u) << S, 0x7f800000u));
    if (l[MAXK - 1] != 0xffffffffu) {
      const double lb = fmax(0.0, (r - 1) - 1e-3) * cs + edge_in;
      if (wd_up < static_cast<float>(lb * lb * (1.0 - 1e-5))) break;
    }
    const int y0 = cy - r, y1 = cy + r, x0 = cx - r, x1 = cx + r;
    for (int gy = max(y0, 0); gy <= min(y1, gc - 1); ++gy) {
      const bool edge = (gy == y0 || gy == y1);
      const int step = edge ? 1 : max(x1 - x0, 1);
      for (int gx = x0; gx <= x1; gx += step) {
        if (gx < 0 || gx >= gc) continue;
        if (l[MAXK - 1] != 0xffffffffu) {
          const double lo_x = (gx - 1e-3) * cs, hi_x = (gx + 1 + 1e-3) * cs;
          const double lo_y = (gy - 1e-3) * cs, hi_y = (gy + 1 + 1e-3) * cs;
          const double dx = fmax(0.0, fmax(lo_x - sx, sx - hi_x));
          const double dy = fmax(0.0, fmax(lo_y - sy, sy - hi_y));
          if (static_cast<float>((dx * dx + dy * dy) * (1.0 - 1e-5)) > wd_up) continue;
        }
        const int c = gy * gc + gx;
        const int e = s.cstart[c + 1];
        for (int t = s.cstart[c]; t < e; ++t) put(s.items[t]);
      }
    }
  }
  bool strict = true;
#pragma unroll
  for (int q = 0; q + 1 < KK; ++q)
    strict &= l[q + 1] == 0xffffffffu || (l[q] >> b) < (l[q + 1] >> b);
  if (!strict) return false;
  const uint32_t low = (1u << b) - 1u;
#pragma unroll
  for (int t = 0; t < MAXK; ++t) top.i[t] = static_cast<int>(l[t] & low);
  return true;
}

// Discrete lattice search: shells of equal integer d2 in increasing order.
// Candidates need no coordinate reads (d2 is the shell's). Falls back to the
// ring search if the precomputed disk is exhausted (very sparse envs).
template <int MAXK, bool EXACT>
__device__ void knn_lattice(const EnvSmem& s, const TagDevConfig& p, int a, TopK<MAXK, EXACT>& top) {
  const int cx = static_cast<int>(s.x[a]), cy = static_cast<int>(s.y[a]);
  const int g = p.gc;
  const int ns = c_num_shells;
  for (int sh = 0; sh < ns; ++sh) {
    const float d2s = static_cast<float>(c_shell_d2[sh]);
    if (top.full() && top.wd < d2s) return;
    const int ob = c_shell_begin[sh], oe = c_shell_begin[sh + 1];
    for (int o = ob; o < oe; ++o) {
      const int packed = c_shell_off[o];
      const int gx = cx + (packed & 0xff) - 64;
      const int gy = cy + ((packed >> 8) & 0xff) - 64;
      if (static_cast<unsigned>(gx) >= static_cast<unsigned>(g) ||
          static_cast<unsigned>(gy) >= static_cast<unsigned>(g))
        continue;
      const int c = gy * g + gx;
      const int e = s.cstart[c + 1];
      for (int t = s.cstart[c]; t < e; ++t) {
        const int j = s.items[t];
        if (j != a) top.consider(d2s, j);
      }
    }
  }
  if (top.full() && top.wd <= static_cast<float>(kShellR2)) return;
  top.init(p.K);
  knn_rings<false, MAXK, EXACT>(s, p, a, top);
}

// Brute-force K-NN over integral positions (discrete, d2 < 2^16): each
// candidate is one 32-bit key (d2 << 16 | j), so the (d2, index) order is an
// unsigned compare and the top-MAXK insertion is a branchless min/max chain —
// no divergence when different lanes admit different candidates.
template <int MAXK>
__device__ __forceinline__ void knn_brute_keys(const EnvSmem& s, const TagDevConfig& p, int a, int* out) {
  uint32_t k[MAXK];
#pragma unroll
  for (int t = 0; t < MAXK; ++t) k[t] = 0xffffffffu;
  const float sx = s.x[a], sy = s.y[a];
  auto key_of = [&](int j) {
    const float dx = __fsub_rn(s.x[j], sx), dy = __fsub_rn(s.y[j], sy);
    const float d2 = __fmaf_rn(dx, dx, __fmul_rn(dy, dy));  // exact: integers below 2^16
    // 2^23 + d2 holds d2 in its low mantissa bits; self never enters
    const uint32_t key = __byte_perm(static_cast<uint32_t>(j), __float_as_uint(__fadd_rn(d2, 8388608.0f)), 0x5410);
    return j == a ? 0xffffffffu : key;
  };
  auto insert = [&](uint32_t key) {
#pragma unroll
    for (int t = 0; t < MAXK; ++t) {
      const uint32_t lo = min(k[t], key);
      key = max(k[t], key);
      k[t] = lo;
    }
  };
  // two candidates per pass: the second chain trails the first by one stage
  int j = 0;
  for (; j + 1 < p.A; j += 2) {
    const uint32_t k0 = key_of(j), k1 = key_of(j + 1);
    insert(k0);
    insert(k1);
  }
  if (j < p.A) insert(key_of(j));
#pragma unroll
  for (int t = 0; t < MAXK; ++t) out[t] = static_cast<int>(k[t] & 0xffffu);
}

// Brute-force K-NN over continuous positions with 32-bit keys (truncated d2
// bits << b | index, b = index bits), as knn_rings_keys: two candidates per
// pass through a branchless min/max chain of K + 1 keys. Exact whenever the
// K + 1 kept keys have strictly increasing truncated d2 (every other
// candidate then has a strictly larger exact d2); otherwise it returns false
// and the caller runs knn_brute_pairs.
template <int MAXK>
__device__ __forceinline__ bool knn_brute_cont_keys(const EnvSmem& s, const TagDevConfig& p, int a, int* out) {
  constexpr int KK = MAXK + 1;
  const int b = 32 - __clz(max(p.A - 1, 1));
  const int S = b - 1;  // (31 - S) d2 bits + b index bits = 32
  uint32_t l[KK];
#pragma unroll
  for (int t = 0; t < KK; ++t) l[t] = 0xffffffffu;
  const float sx = s.x[a], sy = s.y[a];
  auto key_of = [&](int j) {
    const uint32_t d2b = __float_as_uint(d2_of(sx, sy, s.x[j], s.y[j]));
    return j == a ? 0xffffffffu : (((d2b >> S) << b) | static_cast<uint32_t>(j));
  };
  auto insert = [&](uint32_t key) {
#pragma unroll
    for (int q = 0; q < KK; ++q) {
      const uint32_t lo = min(l[q], key);
      key = max(l[q], key);
      l[q] = lo;
    }
  };
  int j = 0;
  for (; j + 1 < p.A; j += 2) {
    const uint32_t k0 = key_of(j), k1 = key_of(j + 1);
    insert(k0);
    insert(k1);
  }
  if (j < p.A) insert(key_of(j));
  bool strict = true;
#pragma unroll
  for (int q = 0; q + 1 < KK; ++q)
    strict &= l[q + 1] == 0xffffffffu || (l[q] >> b) < (l[q + 1] >> b);
  if (!strict) return false;
  const uint32_t low = (1u << b) - 1u;
#pragma unroll
  for (int t = 0; t < MAXK; ++t) out[t] = static_cast<int>(l[t] & low);
  return true;
}

// Brute-force K-NN, any positions: ascending candidates, so (d2, index)
// order is a strict d2 compare (ties keep the earlier index). The insertion
// is a branchless shift: slots from the candidate's rank down move by one.
// (A compare-exchange chain would be wrong here: a displaced entry must
// displace its equal-d2 successor, the new candidate must not.)
template <int MAXK>
__device__ __forceinline__ void knn_brute_pairs(const EnvSmem& s, const TagDevConfig& p, int a, int* out) {
  float d[MAXK];
#pragma unroll
  for (int t = 0; t < MAXK; ++t) {
    d[t] = __int_as_float(0x7f800000);
    out[t] = 0x7fffffff;
  }
  const float sx = s.x[a], sy = s.y[a];
  auto put = [&](int j) {
    const float dd = d2_of(sx, sy, s.x[j], s.y[j]);
    bool c[MAXK];
#pragma unroll
    for (int t = 0; t < MAXK; ++t) c[t] = dd < d[t];  // monotone in t (d sorted)
#pragma unroll
    for (int t = MAXK - 1; t >= 0; --t) {
      const bool from_prev = t > 0 && c[t > 0 ? t - 1 : 0];
      const float nd = from_prev ? d[t > 0 ? t - 1 : 0] : dd;
      const int ni = from_prev ? out[t > 0 ? t - 1 : 0] : j;
      d[t] = c[t] ? nd : d[t];
      out[t] = c[t] ? ni : out[t];
    }
  };
  for (int j = 0; j < a; ++j) put(j);
  for (int j = a + 1; j < p.A; ++j) put(j);
}

template <bool CONT, bool GRID, int MAXK, bool EXACT>
__device__ __forceinline__ void knn_agent(const EnvSmem& s, const TagDevConfig& p, int a,
                                          bool lattice_ok, TopK<MAXK, EXACT>& top, bool keys_ok = false,
                                          bool integral = true) {
  if (!GRID && MAXK <= 8) {
    if (!CONT && keys_ok)
      knn_brute_keys<MAXK>(s, p, a, top.i);
    else if (!CONT || !p.cont_keys || !knn_brute_cont_keys<MAXK>(s, p, a, top.i))
      knn_brute_pairs<MAXK>(s, p, a, top.i);
    return;
  }
  top.init(p.K);
  if (!GRID) {
    const float sx = s.x[a], sy = s.y[a];
    for (int j = 0; j < a; ++j) top.consider_next(d2_of(sx, sy, s.x[j], s.y[j]), j);
    for (int j = a + 1; j < p.A; ++j) top.consider_next(d2_of(sx, sy, s.x[j], s.y[j]), j);
    return;
  }
  if (!CONT && lattice_ok) {
    knn_lattice<MAXK, EXACT>(s, p, a, top);
    return;
  }
  if constexpr (CONT && EXACT) {
    if (p.cont_keys && knn_rings_keys<MAXK, EXACT>(s, p, a, top)) return;
  }
  knn_rings<CONT, MAXK, EXACT>(s, p, a, top, integral);
}

// Tag resolution for one active runner: resolve kernel (tag_env.cpp:403-456)
// / TagReference::step (tag_env.cpp:546-571). Returns the credited tagger or -1.
template <bool CONT, bool GRID>
__device__ int find_tagger(const EnvSmem& s, const TagDevConfig& p, int rn, bool cell_tagger,
                           bool tag_prefix = false) {
  if (!CONT && GRID && cell_tagger) return s.cfill[s.cellof[rn]];
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
    const int jn = tag_prefix ? p.T : p.A;  // taggers are exactly [0, T)
    if (exact_cell) {
      // ascending scan: the first tagger at the runner's cell is the lowest index
      for (int j = 0; j < jn; ++j)
        if (s.tag[j] && s.x[j] == rx && s.y[j] == ry) return j;
      return -1;
    }
    for (int j = 0; j < jn; ++j) consider(j);
    return best;
  }
  if (exact_cell) {
    // the lowest-index tagger at the runner's position (tag_env.cpp:430-434),
    // whatever the order of the cell's items
    const int c = s.cellof[rn];
    const int e = s.cstart[c + 1];
    for (int t = s.cstart[c]; t < e; ++t) {
      const int j = s.items[t];
      if (s.tag[j] && s.x[j] == rx && s.y[j] == ry && (best < 0 || j < best)) best = j;
    }
    return best;
  }
  const float R = __fadd_rn(__fmul_rn(radius, 1.001f), 1e-6f);
  const int x0 = cell_coord<CONT>(__fsub_rn(rx, R), p), x1 = cell_coord<CONT>(__fadd_rn(rx, R), p);
  const int y0 = cell_coord<CONT>(__fsub_rn(ry, R), p), y1 = cell_coord<CONT>(__fadd_rn(ry, R), p);
  for (int gy = y0; gy <= y1; ++gy) {
    for (int gx = x0; gx <= x1; ++gx) {
      const int c = gy * p.gc + gx;
      const int e = s.cstart[c + 1];
      for (int t = s.cstart[c]; t < e; ++t) {
        const int j = s.items[t];
        if (tag_prefix && j >= p.T) break;  // index-sorted cell: only runners follow
        consider(j);
      }
    }
  }
  return best;
}

__device__ __forceinline__ float inv_ms(const TagDevConfig& p, int j) {
  return j < p.T ? p.inv_max_speed_tagger : p.inv_max_speed_runner;
}

// One observation element (write_obs_row, tag_env.cpp:165-212) — used by the
// cooperative (non-staged) writer for wide rows.
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
      case 4: return __fmul_rn(s.sp[j], inv_ms(p, j));
      case 5: return s.sn[j];
      default: return s.cs[j];
    }
  }
  const int t = f - nbf;
  if (t == 0) return __fmul_rn(s.x[a], p.inv_world);
  if (t == 1) return __fmul_rn(s.y[a], p.inv_world);
  if (CONT) {
    if (t == 2) return __fmul_rn(s.sp[a], inv_ms(p, a));
    if (t == 3) return s.sn[a];
    if (t == 4) return s.cs[a];
  }
  return __fmul_rn(static_cast<float>(step_count), p.inv_episode);
}

// Writes one agent's full observation row (write_obs_row) to `out`
// (a warp staging buffer in shared memory). `nb(n)` yields the n-th visible
// neighbour.
template <bool CONT, int VIS_CT, class NB>
__device__ __forceinline__ void write_row(const EnvSmem& s, const TagDevConfig& p, int32_t step_count,
                                          int a, float* out, NB nb) {
  // VIS_CT > 0: visible count known at compile time (partial obs, exact K)
  constexpr int NBF = CONT ? 7 : 4;
  constexpr int D_CT = VIS_CT * NBF + (CONT ? 5 : 2) + 1;
  const int vis = VIS_CT > 0 ? VIS_CT : p.vis;
  const int D = VIS_CT > 0 ? D_CT : p.D;
  if (!s.act[a]) {
#pragma unroll
    for (int f = 0; f < (VIS_CT > 0 ? D_CT : 1); ++f) out[f] = 0.0f;
    if (VIS_CT == 0)
      for (int f = 1; f < D; ++f) out[f] = 0.0f;
    return;
  }
  const float sx = s.x[a], sy = s.y[a];
  const float iw = p.inv_world;
#pragma unroll
  for (int n = 0; n < (VIS_CT > 0 ? VIS_CT : 1); ++n) {
    if (VIS_CT == 0 && n >= vis) break;
    const int j = nb(n);
    float* o = out + n * NBF;
    o[0] = __fmul_rn(__fsub_rn(s.x[j], sx), iw);
    o[1] = __fmul_rn(__fsub_rn(s.y[j], sy), iw);
    o[2] = s.tag[j] ? 1.0f : 0.0f;
    o[3] = s.act[j] ? 1.0f : 0.0f;
    if (CONT) {
      o[4] = __fmul_rn(s.sp[j], inv_ms(p, j));
      o[5] = s.sn[j];
      o[6] = s.cs[j];
    }
  }
  if (VIS_CT == 0) {
    for (int n = 1; n < vis; ++n) {
      const int j = nb(n);
      float* o = out + n * NBF;
      o[0] = __fmul_rn(__fsub_rn(s.x[j], sx), iw);
      o[1] = __fmul_rn(__fsub_rn(s.y[j], sy), iw);
      o[2] = s.tag[j] ? 1.0f : 0.0f;
      o[3] = s.act[j] ? 1.0f : 0.0f;
      if (CONT) {
        o[4] = __fmul_rn(s.sp[j], inv_ms(p, j));
        o[5] = s.sn[j];
        o[6] = s.cs[j];
      }
    }
  }
  float* o = out + vis * NBF;
  o[0] = __fmul_rn(sx, iw);
  o[1] = __fmul_rn(sy, iw);
  if (CONT) {
    o[2] = __fmul_rn(s.sp[a], inv_ms(p, a));
    o[3] = s.sn[a];
    o[4] = s.cs[a];
    o[5] = __fmul_rn(static_cast<float>(step_count), p.inv_episode);
  } else {
    o[2] = __fmul_rn(static_cast<float>(step_count), p.inv_episode);
  }
}


__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// apply_move for one agent held in shared memory (tag_env.cpp:148-160,
// move_discrete / move_continuous tag_env.hpp:71-100). Inactive agents stay.
template <bool CONT>
__device__ __forceinline__ void move_agent(const EnvSmem& s, const TagDevConfig& p, int a, int act0,
                                           int act1) {
  if (!s.act[a]) return;
  if (!CONT) {
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
  } else {
    float dir = s.dir[a], sp = s.sp[a];
    if (act1 == 0) dir = __fsub_rn(dir, p.turn_delta);
    if (act1 == 2) dir = __fadd_rn(dir, p.turn_delta);
    while (dir >= kTwoPiF) dir = __fsub_rn(dir, kTwoPiF);
    while (dir < 0.0f) dir = __fadd_rn(dir, kTwoPiF);
    if (act0 == 0) sp = __fsub_rn(sp, p.accel_delta);
    if (act0 == 2) sp = __fadd_rn(sp, p.accel_delta);
    const float ms = a < p.T ? p.max_speed_tagger : p.max_speed_runner;
    sp = min_ref(max_ref(sp, 0.0f), ms);
    const float x = __fadd_rn(s.x[a], __fmul_rn(sp, cos_ref(dir)));
    const float y = __fadd_rn(s.y[a], __fmul_rn(sp, sin_ref(dir)));
    s.x[a] = min_ref(max_ref(x, 0.0f), p.world_hi);
    s.y[a] = min_ref(max_ref(y, 0.0f), p.world_hi);
    s.dir[a] = dir;
    s.sp[a] = sp;
  }
}

// Five f64 logits of one discrete row with 16-byte loads where aligned
// (rows are 40 B apart: even rows start 16-B aligned, odd rows 8-B).
__device__ __forceinline__ void load_row5(const double* __restrict__ z, int64_t row, double* out) {
  const double* r = z + row * 5;
  if ((row & 1) == 0) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(r));
    const double2 b = __ldg(reinterpret_cast<const double2*>(r + 2));
    out[0] = a.x; out[1] = a.y; out[2] = b.x; out[3] = b.y; out[4] = __ldg(r + 4);
  } else {
    out[0] = __ldg(r);
    const double2 a = __ldg(reinterpret_cast<const double2*>(r + 1));
    const double2 b = __ldg(reinterpret_cast<const double2*>(r + 3));
    out[1] = a.x; out[2] = a.y; out[3] = b.x; out[4] = b.y;
  }
}

// The sampling decision on f32 estimates (ex2.approx) with a rigorous margin
// (the bound is derived at policy.cu's sample_row_regs: estimates within
// 4e-6 x total of the f64 target and cumulative sums); returns false when a
// cumulative sum lies within 1e-5 x total of the target, and the caller then
// runs the reference f64 arithmetic. Rows of equal logits need no exp.
template <int V>
__device__ __forceinline__ bool sample_fast(const double* z, double zmax, double u, int32_t& pick) {
  float evf[V], totf = 0.0f;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const float dd = static_cast<float>(z[i] - zmax);
    float e = 1.0f;
    if (dd != 0.0f) asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(dd * 1.4426950408889634f));
    evf[i] = e;
    totf += e;
  }
  const float tgt = static_cast<float>(u) * totf;
  const float margin = 1e-5f * totf;
  float cum = 0.0f;
  bool found = false, close = false;
  pick = V - 1;
#pragma unroll
  for (int i = 0; i + 1 < V; ++i) {
    cum += evf[i];
    close |= fabsf(tgt - cum) <= margin;
    if (!found && tgt < cum) {
      pick = i;
      found = true;
    }
  }
  return !close;
}

// sample_from_logits (sampler.hpp:18-30) on a register row of 5.
__device__ __forceinline__ int32_t sample5(const double* z, double u, bool& nonfinite) {
  double zmax = z[0];
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    nonfinite |= !isfinite(z[i]);
    zmax = zmax < z[i] ? z[i] : zmax;
  }
  {
    int32_t fast;
    if (sample_fast<5>(z, zmax, u, fast)) return fast;
  }
  double ev[5];
  double total = 0.0;
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    // exp(0) == 1 exactly (glibc and CUDA alike): the row maximum, and every
    // element of a constant row (the benchmark's uniform policy), skip exp.
    const double d = z[i] - zmax;
    ev[i] = 1.0;
    if (d != 0.0) ev[i] = exp(d);
    total = __dadd_rn(total, ev[i]);
  }
  const double target = __dmul_rn(u, total);
  double cum = 0.0;
  int32_t pick = 4;
  bool found = false;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    cum = __dadd_rn(cum, ev[i]);
    if (!found && target < cum) {
      pick = i;
      found = true;
    }
  }
  return pick;
}

// sample_from_logits for the Tag env's compile-time V (5 discrete, 3
// continuous): the row in registers, no generic loop in the env kernel.
template <int V>
__device__ __forceinline__ int32_t sample_tag_row(const double* __restrict__ logits, int64_t row,
                                                  double u, bool& nonfinite) {
  double z[V];
  if constexpr (V == 5) {
    load_row5(logits, row, z);
    return sample5(z, u, nonfinite);
  } else {
    const double* r = logits + row * V;
#pragma unroll
    for (int i = 0; i < V; ++i) z[i] = __ldg(r + i);
    double zmax = z[0];
#pragma unroll
    for (int i = 0; i < V; ++i) {
      nonfinite |= !isfinite(z[i]);
      zmax = zmax < z[i] ? z[i] : zmax;
    }
    {
      int32_t fast;
      if (sample_fast<V>(z, zmax, u, fast)) return fast;
    }
    double ev[V];
    double total = 0.0;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const double d = z[i] - zmax;  // exp(0) == 1 exactly: skip it
      ev[i] = 1.0;
      if (d != 0.0) ev[i] = exp(d);
      total = __dadd_rn(total, ev[i]);
    }
    const double target = __dmul_rn(u, total);
    double cum = 0.0;
    int32_t pick = V - 1;
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
}

// sample_from_logits (sampler.hpp:18-30) on a row already in registers.
template <int V>
__device__ __forceinline__ int32_t sample_regs(const double* z, double u, bool& nonfinite) {
  if constexpr (V == 5) {
    return sample5(z, u, nonfinite);
  } else {
    double zmax = z[0];
#pragma unroll
    for (int i = 0; i < V; ++i) {
      nonfinite |= !isfinite(z[i]);
      zmax = zmax < z[i] ? z[i] : zmax;
    }
    {
      int32_t fast;
      if (sample_fast<V>(z, zmax, u, fast)) return fast;
    }
    double ev[V];
    double total = 0.0;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const double d = z[i] - zmax;  // exp(0) == 1 exactly: skip it
      ev[i] = 1.0;
      if (d != 0.0) ev[i] = exp(d);
      total = __dadd_rn(total, ev[i]);
    }
    const double target = __dmul_rn(u, total);
    double cum = 0.0;
    int32_t pick = V - 1;
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
}

// apply_move for one ACTIVE agent held in registers (move_discrete /
// move_continuous, tag_env.hpp:71-100).
template <bool CONT>
__device__ __forceinline__ void move_regs(const TagDevConfig& p, int a, int act0, int act1, float& x,
                                          float& y, float& sp, float& dir) {
  if (!CONT) {
    switch (act0) {
      case 1: y = __fadd_rn(y, 1.0f); break;
      case 2: y = __fsub_rn(y, 1.0f); break;
      case 3: x = __fsub_rn(x, 1.0f); break;
      case 4: x = __fadd_rn(x, 1.0f); break;
      default: break;
    }
    x = min_ref(max_ref(x, 0.0f), p.world_hi);
    y = min_ref(max_ref(y, 0.0f), p.world_hi);
  } else {
    if (act1 == 0) dir = __fsub_rn(dir, p.turn_delta);
    if (act1 == 2) dir = __fadd_rn(dir, p.turn_delta);
    while (dir >= kTwoPiF) dir = __fsub_rn(dir, kTwoPiF);
    while (dir < 0.0f) dir = __fadd_rn(dir, kTwoPiF);
    if (act0 == 0) sp = __fsub_rn(sp, p.accel_delta);
    if (act0 == 2) sp = __fadd_rn(sp, p.accel_delta);
    const float ms = a < p.T ? p.max_speed_tagger : p.max_speed_runner;
    sp = min_ref(max_ref(sp, 0.0f), ms);
    float sn, cs;
    sincos_ref(dir, sn, cs);
    x = min_ref(max_ref(__fadd_rn(x, __fmul_rn(sp, cs)), 0.0f), p.world_hi);
    y = min_ref(max_ref(__fadd_rn(y, __fmul_rn(sp, sn)), 0.0f), p.world_hi);
  }
}

// CTA header scratch (after the per-env scalars): doubles [0, 16) are the
// block scan's int scratch, [16, 48) / [48, 80) the per-warp tracker sums
// (tagger / runner), then the bulk-copy mbarrier.
constexpr int kScratchDoubles = 96;
constexpr int kSlotT = 16, kSlotR = 48;

// Discrete full-observation rows of a one-env CTA (write_obs_row,
// tag_env.cpp:165-212, every other agent in ascending order): one warp per
// row, lane l always writes component l & 3 of neighbour block f >> 2.
// (partial = true: the neighbours are the agent's K nearest in s.knn, the
// wide partial rows of K >= 16)
__device__ __forceinline__ void write_full_rows_discrete(const EnvSmem& s, const TagDevConfig& p, float* cta_out,
                                                     int A, int D, int32_t step_count, bool partial = false) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int nb_f = 4 * (partial ? p.K : A - 1);
  const int comp = lane & 3;
  const float iw = p.inv_world;
  const float* fsrc = comp == 0 ? s.x : s.y;
  const uint8_t* bsrc = comp == 2 ? s.tag : s.act;
  for (int a = warp; a < A; a += nwarps) {
    float* dst = cta_out + static_cast<int64_t>(a) * D;
    if (!s.act[a]) {
      for (int f = lane; f < D; f += 32) __stcs(dst + f, 0.0f);
      continue;
    }
    const float so = comp == 0 ? s.x[a] : s.y[a];
    for (int f = lane; f < nb_f; f += 32) {
      const int nn = f >> 2;
      const int j = partial ? static_cast<int>(s.knn[a * p.K + nn]) : nn + (nn >= a ? 1 : 0);
      float v;
      if (comp < 2) {
        v = __fmul_rn(__fsub_rn(fsrc[j], so), iw);
      } else {
        v = bsrc[j] ? 1.0f : 0.0f;
      }
      __stcs(dst + f, v);
    }
    if (lane < 3) {
      const float v = lane == 0 ? __fmul_rn(s.x[a], iw)
                    : lane == 1 ? __fmul_rn(s.y[a], iw)
                                : __fmul_rn(static_cast<float>(step_count), p.inv_episode);
      __stcs(dst + nb_f + lane, v);
    }
  }
}

// ---- the env-step kernel --------------------------------------------------
// Thread layout: tid = le * tpe + lt (le = env slot in the CTA, lt = lane in
// the env). Per-agent loops run over `base` in warp-uniform steps so warp
// collectives are legal; agent a = base + lt.
// Resident CTAs per SM asked of ptxas (register cap 65536 / (threads x n)):
// discrete K <= 8 fits 64 registers without spills -> 4 envs per SM (4 x 51.5 KB
// of smem at C2); continuous carries 2x the per-agent state; the K > 8 top-K
// lists live in registers and spill anyway.
constexpr int env_min_blocks(bool cont, int maxk) {
  return maxk > 8 ? 2 : (cont ? kMinBlocksPerSm : kMinBlocksPerSmDiscrete);
}

// MULTI: the multi-step residency instantiation (RolloutDriver::run); the
// single-step one compiles the step loop away (one iteration known at compile
// time), which keeps its code identical to a loop-free kernel — measured 35%
// fewer instructions on the full-observation writer than the looped build.
// LEAN: the one-env instantiation of the partial-observation step (K = 5
// staged rows, one env per CTA, A % 4 == 0, bulk-staged inputs, single step,
// step/fused modes; discrete plans also need lattice cells — lean_plan checks
// all of it). Continuous plans keep the ring-search K-NN and gain only the
// compile-time layout (A = 1000: 374 vs 429 us/step). The
// same body with those facts compile-time: the generic layouts and the
// multi-step loop drop out (the per-agent K-NN fallback for pushed off-lattice
// positions stays inline: an out-of-line call measured 151 vs 113 us/step, its
// ABI spills landing on the hot path). Measured at C2: 62 registers without
// spills instead of 64 with 28 B of spills, 113 vs 132 us/step (A/B on one box).
template <bool CONT, bool PARTIAL, bool GRID, int MAXK, bool EXACT, bool MULTI, bool LEAN = false>
__global__ void __launch_bounds__(kMaxThreadsPerCta, env_min_blocks(CONT, MAXK)) tag_env_kernel(const TagDevConfig p, const TagDevArrays g,
                                                       const TagLaunch L) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  static_assert(!LEAN || (PARTIAL && GRID && EXACT && !MULTI), "LEAN is the one-env partial single step");
  constexpr bool LATTICE_LEAN = LEAN && !CONT;
  const int tpe = LEAN ? static_cast<int>(blockDim.x) : p.threads_per_env;
  const int le = LEAN ? 0 : tid / tpe;
  const int lt = LEAN ? tid : tid - le * tpe;
  const int64_t e = static_cast<int64_t>(blockIdx.x) * p.envs_per_cta + le;
  const bool env_ok = le < p.envs_per_cta && e < p.E;
  const int mode = LEAN ? (L.mode == kModeStep ? kModeStep : kModeFused) : L.mode;
  const int A = p.A;
  // Fused steps sample from L.logits; with L.logits == nullptr the actions are
  // already in the store (sampled by the policy kernel) and are read like the
  // step mode does.
  const bool sample_here = mode == kModeFused && L.logits != nullptr;
  const bool single = LEAN || p.envs_per_cta == 1;  // CTA == one env: warp collectives are per env
  // Tag action space (tag_env.hpp:48-63): discrete C=1 x V=5, continuous C=2 x V=3.
  constexpr int kC = CONT ? 2 : 1;
  constexpr int kV = CONT ? 3 : 5;

  bool live = env_ok;
  if (mode == kModeReinit && L.env_mask != nullptr && env_ok) live = L.env_mask[e] != 0;
  if (single) {  // CTA-uniform early exit: decided by the CTA's env, not by this thread
    const int64_t e0 = blockIdx.x;
    const bool l0 = e0 < p.E && !(mode == kModeReinit && L.env_mask != nullptr && !L.env_mask[e0]);
    if (!l0) return;
  }
  // Programmatic dependent launch (TagLaunch::env_seq): release the next
  // launch now, then wait for this CTA's envs' previous step only. ld.acquire
  // + the barrier order every thread's later loads (generic and, after the
  // proxy fence, the bulk copies) after that step's writes.
  if (L.pdl_wait) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  const bool pdl = L.env_seq != nullptr;
  // graph replays read their base sequence number on device (like the step)
  const uint32_t seq = L.seq_dev != nullptr ? static_cast<uint32_t>(*L.seq_dev) + L.seq_add : L.seq;
  if (pdl) {
    if (!L.pdl_late) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // A wait that gives up (seconds: preemption, a debugger) skips this CTA's
    // envs for this launch — state untouched, flags not published — and sets
    // the sticky kErrStepOrder bit; once it is set, later launches skip at
    // once instead of polling. Rollout::check / stats raise it and resync.
    bool skip = false;
    if (tid == 0) {
      uint32_t errw = 0;
      if (L.error) asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(errw) : "l"(L.error) : "memory");
      skip = (errw & kErrStepOrder) != 0;
      const int64_t eb = static_cast<int64_t>(blockIdx.x) * p.envs_per_cta;
      for (int k = 0; !skip && k < p.envs_per_cta && eb + k < p.E; ++k) {
        const uint32_t* f = L.env_seq + eb + k;
        // relaxed polling (an acquire per poll would invalidate this SM's L1
        // under the CTAs still working on it), backing off, then one acquire
        uint32_t v, ns = 32, polls = 0;
        for (;;) {
          asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
          if (static_cast<int32_t>(v - (seq - 1u)) >= 0) break;
          if (++polls > (1u << 22)) {  // >= 4 s of polling: report, never hang the device
            if (L.error) atomicOr(L.error, kErrStepOrder);
            skip = true;
            break;
          }
          __nanosleep(ns);
          ns = ns < 1024 ? 2 * ns : ns;
        }
      }
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    if (__syncthreads_or(skip)) return;
  }

  // Per-env scalars are loaded first (by the env's lane 0) so their latency
  // overlaps the per-agent loads instead of following them; packed-env CTAs
  // (small A, launch/latency-bound) also prefetch their tracker slots.
  int32_t pre_step = 0, pre_episode = 0;
  double pre_es[4] = {0.0, 0.0, 0.0, 0.0};  // env_stats [0], [1], [5], [6]
  if (live && lt == 0) {
    pre_step = mode == kModeReinit ? 0 : g.step_count[e];
    pre_episode = (L.episode != nullptr && !(mode == kModeReinit && L.init_episode)) ? L.episode[e] : 0;
    if (!GRID && mode == kModeFused && L.track) {
      const double* es = L.env_stats + e * 8;
      pre_es[0] = es[0];
      pre_es[1] = es[1];
      pre_es[2] = es[5];
      pre_es[3] = es[6];
    }
  }

  EnvScalars* scal = reinterpret_cast<EnvScalars*>(smem);
  int* scratch = reinterpret_cast<int*>(smem + p.envs_per_cta * sizeof(EnvScalars));
  if (LEAN && CONT && tid == 0) scratch[kObsChunk] = 0;  // read after several barriers
  const EnvSmem s = carve(smem + p.head_bytes + (env_ok ? le : 0) * p.env_bytes, p);
  EnvScalars& sc = scal[env_ok ? le : 0];
  const int64_t ga = e * A;

  // Single-env CTAs with A % 4 == 0 move 4 consecutive agents per thread in
  // the per-agent phases so every global access is a 16-byte (or 4-byte for
  // flags) vector and the logits rows of a thread are contiguous.
  const bool vec4 = GRID && (LEAN || (A & 3) == 0);

  const int n_steps = !LEAN && MULTI && mode == kModeFused && sample_here ? L.n_steps : 1;
  for (int it = 0; it < n_steps; ++it) {
  // Iteration `it` of a multi-step launch: step L.step0 + it. After the first,
  // the env's state is already in shared memory (written by the previous
  // iteration); only the step's logits are read.
  const bool first = it == 0;
  // Phase 0: stage the env's agent state in shared memory.
  bool integral = true;
  bool tprefix = true;
  bool nonfinite = false;
  const bool vec_step = live && vec4 && mode != kModeReinit;
  if (vec_step) {
    // Phases 0+1 fused per thread (each thread owns agents a0..a0+3 in both,
    // so no barrier is needed between them): every global load of the 4
    // agents — state, and the 160 B of f64 logits (fused) or the actions
    // (step mode) — is issued up front, the counter hashes overlap their
    // latency, then sample (sampler.hpp:18-30) and apply_move
    // (tag_env.cpp:148-160) run from registers and the moved state lands in
    // shared memory once.
    // Bulk path (one env per CTA): one thread arms an mbarrier and issues TMA
    // bulk copies of the env's contiguous rows — f64 logits (fused) into the
    // zone, positions (+ speed/direction) straight into their smem arrays —
    // so the whole 40-50 KB input is in flight at once with no registers held.
    const bool bulk = LEAN || p.bulk_in != 0;
    const double* zone = reinterpret_cast<const double*>(smem + p.off_zone);
    if (bulk) {
      uint64_t* bar = reinterpret_cast<uint64_t*>(smem + p.envs_per_cta * sizeof(EnvScalars) + kScratchDoubles * 8);
      if (tid == 0) {
        const uint32_t rowb = static_cast<uint32_t>(A) * 4u;
        const uint32_t lgb = sample_here ? static_cast<uint32_t>(A) * kC * kV * 8u : 0u;
        if (first) mbar_init(bar, 1);
        mbar_expect_tx(bar, lgb + (first ? (CONT ? 4u : 2u) * rowb : 0u));
        if (lgb) bulk_g2s(smem + p.off_zone, L.logits + ga * kC * kV, lgb, bar);
        if (first) {
          bulk_g2s(s.x, g.loc_x + ga, rowb, bar);
          bulk_g2s(s.y, g.loc_y + ga, rowb, bar);
          if (CONT) {
            bulk_g2s(s.sp, g.speed + ga, rowb, bar);
            bulk_g2s(s.dir, g.direction + ga, rowb, bar);
          }
        }
        // L2 prefetch of the inputs of the env that will start about one CTA
        // lifetime from now (the next wave: `prefetch_stride` resident CTAs
        // later), so its bulk copies hit L2 instead of HBM.
        const int64_t pe = e + p.prefetch_stride;
        if (p.prefetch_stride > 0 && pe < p.E) {
          const int64_t pa = pe * A;
          if (lgb) bulk_prefetch_l2(L.logits + pa * kC * kV, lgb);
          bulk_prefetch_l2(g.loc_x + pa, rowb);
          bulk_prefetch_l2(g.loc_y + pa, rowb);
        }
      }
      if (first) __syncthreads();  // barrier initialised before anyone waits on it
      mbar_wait(bar, static_cast<uint32_t>(it & 1));
    }
    // The step's counter-RNG prefix, after the bulk copies are issued (under
    // graph replay the step index is a device load).
    const uint64_t h_step =
        n_steps > 1 ? absorb(L.action_h0, static_cast<uint64_t>(L.step0 + it))
        : L.step_dev != nullptr
            ? absorb(L.action_h0, static_cast<uint64_t>(*L.step_dev + static_cast<int64_t>(L.step_add)))
            : L.action_h_step;
    const uint64_t h_env = absorb(h_step, static_cast<uint64_t>(p.env_offset + e));
    for (int a0 = 4 * lt; a0 < A; a0 += 4 * tpe) {
      const bool in_smem = bulk || !first;  // state already staged in shared memory
      const float4 x4 = in_smem ? *reinterpret_cast<const float4*>(s.x + a0)
                                : *reinterpret_cast<const float4*>(g.loc_x + ga + a0);
      const float4 y4 = in_smem ? *reinterpret_cast<const float4*>(s.y + a0)
                                : *reinterpret_cast<const float4*>(g.loc_y + ga + a0);
      const uint32_t act4 = first ? *reinterpret_cast<const uint32_t*>(g.active + ga + a0)
                                  : *reinterpret_cast<const uint32_t*>(s.act + a0);
      const uint32_t tag4 = first ? *reinterpret_cast<const uint32_t*>(g.is_tagger + ga + a0)
                                  : *reinterpret_cast<const uint32_t*>(s.tag + a0);
      float4 sp4 = make_float4(0.f, 0.f, 0.f, 0.f), dir4 = sp4;
      if (CONT) {
        sp4 = in_smem ? *reinterpret_cast<const float4*>(s.sp + a0)
                      : *reinterpret_cast<const float4*>(g.speed + ga + a0);
        dir4 = in_smem ? *reinterpret_cast<const float4*>(s.dir + a0)
                       : *reinterpret_cast<const float4*>(g.direction + ga + a0);
      }
      int32_t act0[4], act1[4] = {1, 1, 1, 1};
      if (sample_here) {
        // kSamplePass agents per pass (kSamplePass * kC * kV doubles in
        // registers): the rows of agents a0 + P*h .. start 16-B aligned since
        // a0 % 4 == 0 and kSamplePass * kC * kV * 8 % 16 == 0 for P in {2, 4}
        // (P == 1 uses 8-B loads).
        constexpr int P = kSamplePass;
        constexpr int kRowD = P * kC * kV;
#pragma unroll 1
        for (int h = 0; h < 4 / P; ++h) {
          double z[kRowD];
          if (bulk) {
            const double* lrow = zone + (a0 + P * h) * kC * kV;
            if constexpr (kRowD % 2 == 0) {
#pragma unroll
              for (int i = 0; i < kRowD / 2; ++i) {
                const double2 v = reinterpret_cast<const double2*>(lrow)[i];
                z[2 * i] = v.x;
                z[2 * i + 1] = v.y;
              }
            } else {
#pragma unroll
              for (int i = 0; i < kRowD; ++i) z[i] = lrow[i];
            }
          } else {
            const double* lrow = L.logits + (ga + a0 + P * h) * kC * kV;
            if constexpr (kRowD % 2 == 0) {
#pragma unroll
              for (int i = 0; i < kRowD / 2; ++i) {
                const double2 v = __ldg(reinterpret_cast<const double2*>(lrow) + i);
                z[2 * i] = v.x;
                z[2 * i + 1] = v.y;
              }
            } else {
#pragma unroll
              for (int i = 0; i < kRowD; ++i) z[i] = __ldg(lrow + i);
            }
          }
#pragma unroll
          for (int k = 0; k < P; ++k) {
            const int a = a0 + P * h + k;
            const uint64_t h_ag = absorb(h_env, static_cast<uint64_t>(a));
            const double u0 = to_unit(absorb(absorb(h_ag, 0), 0));
            const int32_t s0 = (ablate_bits(L) & 1u) ? static_cast<int32_t>(u0 * 5.0)
                                               : sample_regs<kV>(z + k * kC * kV, u0, nonfinite);
            int32_t s1 = 1;
            if (CONT) {
              const double u1 = to_unit(absorb(absorb(h_ag, 1), 0));
              s1 = sample_regs<kV>(z + k * kC * kV + kV, u1, nonfinite);
            }
            // register arrays indexed by the runtime pass h: select, not index
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (q == P * h + k) {
                act0[q] = s0;
                act1[q] = s1;
              }
            }
          }
        }
      } else if (CONT) {
        const int4* src = reinterpret_cast<const int4*>(g.actions + (ga + a0) * 2);
        const int4 v0 = src[0], v1 = src[1];
        act0[0] = v0.x; act1[0] = v0.y; act0[1] = v0.z; act1[1] = v0.w;
        act0[2] = v1.x; act1[2] = v1.y; act0[3] = v1.z; act1[3] = v1.w;
      } else {
        const int4 v = *reinterpret_cast<const int4*>(g.actions + ga + a0);
        act0[0] = v.x; act0[1] = v.y; act0[2] = v.z; act0[3] = v.w;
      }
      if (sample_here) {
        if (CONT) {
          int4* dst = reinterpret_cast<int4*>(g.actions + (ga + a0) * 2);
          dst[0] = make_int4(act0[0], act1[0], act0[1], act1[1]);
          dst[1] = make_int4(act0[2], act1[2], act0[3], act1[3]);
        } else {
          *reinterpret_cast<int4*>(g.actions + ga + a0) = make_int4(act0[0], act0[1], act0[2], act0[3]);
        }
      }
      if (L.cap_actions != nullptr) {
        if (CONT) {
          int4* dst = reinterpret_cast<int4*>(L.cap_actions + (ga + a0) * 2);
          dst[0] = make_int4(act0[0], act1[0], act0[1], act1[1]);
          dst[1] = make_int4(act0[2], act1[2], act0[3], act1[3]);
        } else {
          *reinterpret_cast<int4*>(L.cap_actions + ga + a0) = make_int4(act0[0], act0[1], act0[2], act0[3]);
        }
        *reinterpret_cast<uint32_t*>(L.cap_active + ga + a0) = act4;
      }
      float xs[4] = {x4.x, x4.y, x4.z, x4.w}, ys[4] = {y4.x, y4.y, y4.z, y4.w};
      float sps[4] = {sp4.x, sp4.y, sp4.z, sp4.w}, dirs[4] = {dir4.x, dir4.y, dir4.z, dir4.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        // CTA predicate: discrete -> positions integral (lattice K-NN valid);
        // continuous -> taggers are exactly the index prefix [0, T) (the
        // radius query may stop at the first non-tagger of an index-sorted cell)
        if (CONT)
          integral &= (((tag4 >> (8 * k)) & 0xffu) != 0) == (a0 + k < p.T);
        else
          integral &= (xs[k] == truncf(xs[k])) && (ys[k] == truncf(ys[k])) && xs[k] >= 0.0f &&
                      ys[k] >= 0.0f && xs[k] <= p.world_hi && ys[k] <= p.world_hi;
        if ((act4 >> (8 * k)) & 0xffu)
          move_regs<CONT>(p, a0 + k, act0[k], act1[k], xs[k], ys[k], sps[k], dirs[k]);
      }
      *reinterpret_cast<float4*>(s.x + a0) = make_float4(xs[0], xs[1], xs[2], xs[3]);
      *reinterpret_cast<float4*>(s.y + a0) = make_float4(ys[0], ys[1], ys[2], ys[3]);
      *reinterpret_cast<uint32_t*>(s.act + a0) = act4;
      *reinterpret_cast<uint32_t*>(s.tag + a0) = tag4;
      if (CONT) {
        *reinterpret_cast<float4*>(s.sp + a0) = make_float4(sps[0], sps[1], sps[2], sps[3]);
        *reinterpret_cast<float4*>(s.dir + a0) = make_float4(dirs[0], dirs[1], dirs[2], dirs[3]);
      }
      *reinterpret_cast<int4*>(s.cred + a0) = make_int4(0, 0, 0, 0);
      *reinterpret_cast<uint32_t*>(s.tagged + a0) = 0u;
    }
    if (nonfinite && L.error) atomicOr(L.error, kErrNonFinite);
  } else if (live && vec4) {
    for (int a0 = 4 * lt; a0 < A; a0 += 4 * tpe) {
      if (mode != kModeReinit) {
        const float4 x4 = *reinterpret_cast<const float4*>(g.loc_x + ga + a0);
        const float4 y4 = *reinterpret_cast<const float4*>(g.loc_y + ga + a0);
        *reinterpret_cast<float4*>(s.x + a0) = x4;
        *reinterpret_cast<float4*>(s.y + a0) = y4;
        const float xs[4] = {x4.x, x4.y, x4.z, x4.w}, ys[4] = {y4.x, y4.y, y4.z, y4.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          integral &= (xs[k] == truncf(xs[k])) && (ys[k] == truncf(ys[k])) && xs[k] >= 0.0f &&
                      ys[k] >= 0.0f && xs[k] <= p.world_hi && ys[k] <= p.world_hi;
        }
        *reinterpret_cast<uint32_t*>(s.act + a0) = *reinterpret_cast<const uint32_t*>(g.active + ga + a0);
        if (CONT) {
          *reinterpret_cast<float4*>(s.sp + a0) = *reinterpret_cast<const float4*>(g.speed + ga + a0);
          *reinterpret_cast<float4*>(s.dir + a0) = *reinterpret_cast<const float4*>(g.direction + ga + a0);
        }
      }
      *reinterpret_cast<uint32_t*>(s.tag + a0) = *reinterpret_cast<const uint32_t*>(g.is_tagger + ga + a0);
      *reinterpret_cast<int4*>(s.cred + a0) = make_int4(0, 0, 0, 0);
      *reinterpret_cast<uint32_t*>(s.tagged + a0) = 0u;
    }
  }
  if (live) {
    // Per-agent layout (A % 4 != 0 or packed envs): phases 0+1 fused per
    // thread like the vec4 path — the agent's state and its logits row (or
    // action) load together, then sample + apply_move in registers and one
    // store of the moved state to shared memory (no barrier in between: a
    // thread only touches its own agents).
    uint64_t h_env = 0;
    if (!vec4 && mode != kModeReinit && sample_here) {
      const uint64_t h_step =
          n_steps > 1 ? absorb(L.action_h0, static_cast<uint64_t>(L.step0 + it))
          : L.step_dev != nullptr
              ? absorb(L.action_h0, static_cast<uint64_t>(*L.step_dev + static_cast<int64_t>(L.step_add)))
              : L.action_h_step;
      h_env = absorb(h_step, static_cast<uint64_t>(p.env_offset + e));
    }
    for (int a = vec4 ? A : lt; a < A; a += tpe) {
      if (mode != kModeReinit) {
        float x = first ? g.loc_x[ga + a] : s.x[a], y = first ? g.loc_y[ga + a] : s.y[a];
        const uint8_t act = first ? g.active[ga + a] : s.act[a];
        float sp = 0.f, dir = 0.f;
        if (CONT) {
          sp = first ? g.speed[ga + a] : s.sp[a];
          dir = first ? g.direction[ga + a] : s.dir[a];
        }
        if (!CONT)  // (continuous: the tagger-prefix predicate is taken below)
          integral &= (x == truncf(x)) && (y == truncf(y)) && x >= 0.0f && y >= 0.0f &&
                      x <= p.world_hi && y <= p.world_hi;
        const int64_t row = (ga + a) * kC;
        int32_t act0, act1 = 1;
        if (sample_here) {
          const uint64_t h_ag = absorb(h_env, static_cast<uint64_t>(a));
          act0 = sample_tag_row<kV>(L.logits, row, to_unit(absorb(absorb(h_ag, 0), 0)), nonfinite);
          g.actions[row] = act0;
          if (CONT) {
            act1 = sample_tag_row<kV>(L.logits, row + 1, to_unit(absorb(absorb(h_ag, 1), 0)), nonfinite);
            g.actions[row + 1] = act1;
          }
        } else {
          act0 = g.actions[row];
          if (CONT) act1 = g.actions[row + 1];
        }
        if (L.cap_actions != nullptr) {
          L.cap_actions[row] = act0;
          if (CONT) L.cap_actions[row + 1] = act1;
          L.cap_active[ga + a] = act;
        }
        if (act) move_regs<CONT>(p, a, act0, act1, x, y, sp, dir);
        s.x[a] = x;
        s.y[a] = y;
        s.act[a] = act;
        if (CONT) {
          s.sp[a] = sp;
          s.dir[a] = dir;
        }
      }
      if (first) s.tag[a] = g.is_tagger[ga + a];
      if (CONT) integral &= (s.tag[a] != 0) == (a < p.T);
      if (!CONT && !GRID) tprefix &= (s.tag[a] != 0) == (a < p.T);
      s.cred[a] = 0;
      s.tagged[a] = 0;
    }
    if (!vec4 && nonfinite && L.error) atomicOr(L.error, kErrNonFinite);
    if (lt == 0) {
      sc.runners_left = 0;
      if (first) {
        sc.step_count = pre_step;
        sc.episode = pre_episode;
      }
      sc.done = 0;
      sc.tags = 0;
      sc.live = 1;
      sc.lattice_ok = 1;
      sc.ret_tagger = 0.0;
      sc.ret_runner = 0.0;
    }
  } else if (env_ok && lt == 0) {
    sc.live = 0;
  }
  // CTA-wide AND of `integral` (only read when GRID, i.e. one env per CTA).
  const bool all_integral = __syncthreads_and(integral) != 0;
  // packed discrete envs: taggers exactly the prefix [0, T) in every env of the CTA
  const bool all_prefix = (!CONT && !GRID) ? __syncthreads_and(tprefix) != 0 : false;
  if (!CONT && GRID && !all_integral && lt == 0) sc.lattice_ok = 0;

  bool reset_now = false;
  if (mode != kModeReinit) {
    // Phase 1 (sample + apply_move, tag_env.cpp:148-160) ran per thread,
    // fused into phase 0, in both layouts.

    // Phase 2: bucket grid over post-move positions (NeighborGrid::build).
    // lattice cells are exact positions: lowest-index tagger per cell
    const bool cell_tagger = !CONT && GRID && p.lattice && all_integral && p.fault_bias == 0.0f;
    if constexpr (LATTICE_LEAN) {
      build_grid_lattice(s, p, scratch, false);
    } else {
      if (GRID && !(ablate_bits(L) & 8u)) build_grid<CONT>(s, p, scratch, false, cell_tagger);
    }

    // Phase 3: resolve tags (tag_env.cpp:403-456). Counts are warp-aggregated
    // when the CTA is one env; there "any runner still active" is all
    // resolve_env_counters needs (tag_env.cpp:241-250), a barrier-OR.
    bool any_alive = false;
    const int32_t step_new = sc.step_count + 1;  // read before anyone rewrites sc
    for (int base = 0; base < A; base += tpe) {
      const int a = base + lt;
      const bool valid = live && a < A;
      const bool runner = valid && !s.tag[a] && s.act[a];
      int best = -1;
      if (runner) {
        if (LATTICE_LEAN && cell_tagger) {
          const int ct = s.celltag[s.cellof[a]];
          best = ct == 0x7fffffff ? -1 : ct;
        } else {
          best = find_tagger<CONT, GRID>(s, p, a, cell_tagger && !LATTICE_LEAN, CONT ? all_integral : all_prefix);
        }
      }
      if (best >= 0) {
        s.act[a] = 0;
        s.tagged[a] = 1;
        atomicAdd(&s.cred[best], 1);
      }
      const bool alive = runner && best < 0;
      any_alive |= alive;
      if (GRID && valid && s.act[a]) s.cellact[s.cellof[a]] = 1;  // active after resolve
      if (single) {
        const unsigned m_tag = __ballot_sync(0xffffffffu, best >= 0);
        if (lane == 0 && m_tag) atomicAdd(&scal[0].tags, __popc(m_tag));
      } else {
        if (alive) atomicAdd(&sc.runners_left, 1);
        if (best >= 0) atomicAdd(&sc.tags, 1);
      }
    }
    // resolve_env_counters (tag_env.cpp:241-250).
    bool done_now;
    if (single) {
      const bool alive_cta = __syncthreads_or(any_alive) != 0;
      done_now = step_new >= p.episode_length || !alive_cta;
      if (lt == 0) {  // every thread read sc.step_count before the barrier
        sc.step_count = step_new;
        sc.done = done_now ? 1 : 0;
      }
    } else {
      __syncthreads();
      if (live && lt == 0) {
        sc.step_count += 1;
        sc.done = (sc.step_count >= p.episode_length || sc.runners_left == 0) ? 1 : 0;
      }
      __syncthreads();
      done_now = sc.done != 0;
    }

    // Phase 4: rewards (write_rewards_row, tag_env.cpp:252-259) + tracker.
    reset_now = live && mode == kModeFused && L.do_reset && done_now;
    if (L.cap_done != nullptr && live && lt == 0) L.cap_done[e] = done_now ? 1 : 0;
    const bool track = mode == kModeFused && L.track;
    double rt = 0.0, rr = 0.0;
    if (live && vec4) {
      for (int a0 = 4 * lt; a0 < A; a0 += 4 * tpe) {
        const int4 c4 = *reinterpret_cast<const int4*>(s.cred + a0);
        const uint32_t tg4 = *reinterpret_cast<const uint32_t*>(s.tag + a0);
        const uint32_t td4 = *reinterpret_cast<const uint32_t*>(s.tagged + a0);
        const int cr[4] = {c4.x, c4.y, c4.z, c4.w};
        float r[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const bool is_t = (tg4 >> (8 * k)) & 0xffu;
          const bool was = (td4 >> (8 * k)) & 0xffu;
          r[k] = is_t ? __fmul_rn(p.reward_per_tag, static_cast<float>(cr[k])) : (was ? p.penalty : 0.0f);
          if (a0 + k < p.T) rt += static_cast<double>(r[k]); else rr += static_cast<double>(r[k]);
        }
        if (L.cap_rewards != nullptr)
          *reinterpret_cast<float4*>(L.cap_rewards + ga + a0) = make_float4(r[0], r[1], r[2], r[3]);
        if (reset_now) {
          *reinterpret_cast<float4*>(g.rewards + ga + a0) = make_float4(0.f, 0.f, 0.f, 0.f);
          *reinterpret_cast<int4*>(g.credits + ga + a0) = make_int4(0, 0, 0, 0);
          *reinterpret_cast<uint32_t*>(g.tagged + ga + a0) = 0u;
        } else {
          *reinterpret_cast<float4*>(g.rewards + ga + a0) = make_float4(r[0], r[1], r[2], r[3]);
          *reinterpret_cast<int4*>(g.credits + ga + a0) = c4;
          *reinterpret_cast<uint32_t*>(g.tagged + ga + a0) = td4;
        }
      }
    }
    if (live) {
      for (int a = vec4 ? A : lt; a < A; a += tpe) {
        const int32_t cr = s.cred[a];
        const float r = s.tag[a] ? __fmul_rn(p.reward_per_tag, static_cast<float>(cr))
                                 : (s.tagged[a] ? p.penalty : 0.0f);
        if (a < p.T) rt += static_cast<double>(r); else rr += static_cast<double>(r);
        g.rewards[ga + a] = reset_now ? 0.0f : r;
        if (L.cap_rewards != nullptr) L.cap_rewards[ga + a] = r;
        g.credits[ga + a] = reset_now ? 0 : cr;
        g.tagged[ga + a] = reset_now ? 0 : s.tagged[a];
        if (!single) s.cred[a] = __float_as_int(r);  // summed by the env's lane 0 below
      }
    }
    if (track) {
      if (single) {
        // warp sums -> per-warp slots in `scratch` (as doubles) -> one adder
        rt = warp_sum(rt);
        rr = warp_sum(rr);
        double* slots = reinterpret_cast<double*>(scratch);
        if (lane == 0) {
          slots[kSlotT + warp] = rt;
          slots[kSlotR + warp] = rr;
        }
      }
    }
    // Single-env CTA that does not reset: its observation inputs are final
    // now, so the per-cell K-NN lists (lattice) / sin-cos (continuous) are
    // built in this phase and one barrier covers rewards, tracker and them.
    if (single && !reset_now) {
      if (CONT) {
        for (int a = lt; a < A; a += tpe) {
          sincos_ref(s.dir[a], s.sn[a], s.cs[a]);
        }
      }
      if (PARTIAL && !CONT && GRID && p.lattice && all_integral) {
        if constexpr (LATTICE_LEAN)
          build_cell_lists_keys(s, p, scratch);
        else
          build_cell_lists(s, p, ablate_bits(L));
      }
    }
    __syncthreads();
    if (live && lt == 0 && track) {
      // EpisodeTracker::accumulate / finish_done (trainer.cpp:229-252); per-env
      // slots, no atomics: [run_t, run_r, episodes, ret_t, ret_r, tags, steps].
      double st = 0.0, sr = 0.0;
      if (single) {
        const double* slots = reinterpret_cast<const double*>(scratch);
        for (int w = 0; w < (blockDim.x >> 5); ++w) {
          st += slots[kSlotT + w];
          sr += slots[kSlotR + w];
        }
      } else {  // packed env: its A rewards, in agent order
        for (int a = 0; a < A; ++a) {
          const double r = static_cast<double>(__int_as_float(s.cred[a]));
          if (a < p.T) st += r; else sr += r;
        }
      }
      double* es = L.env_stats + e * 8;
      // packed envs: slots [0], [1], [5], [6] stay in registers across the
      // steps of a multi-step launch (prefetched before the first step)
      const bool pre = !GRID;
      const double run_t = (pre ? pre_es[0] : es[0]) + st;
      const double run_r = (pre ? pre_es[1] : es[1]) + sr;
      const double es5 = (pre ? pre_es[2] : es[5]) + sc.tags;
      const double es6 = (pre ? pre_es[3] : es[6]) + 1.0;
      es[5] = es5;
      es[6] = es6;
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
      if (!GRID) {  // one-env CTAs reload them (8 more live registers cost spills there)
        pre_es[0] = sc.done ? 0.0 : run_t;
        pre_es[1] = sc.done ? 0.0 : run_r;
        pre_es[2] = es5;
        pre_es[3] = es6;
      }
    }
  }

  // Phase 5: (re)placement — fused reset-on-done or reinit (place_env,
  // tag_env.cpp:261-273; place_agent :130-146).
  const bool place = live && (mode == kModeReinit || reset_now);
  const int episode = mode == kModeFused ? sc.episode + 1 : sc.episode;
  if (place) {
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
        g.actions[(ga + a) * kC] = 0;
        if (CONT) g.actions[(ga + a) * kC + 1] = 0;
      }
    }
  }
  if (!single || place) __syncthreads();  // everyone has read sc.* above before it is rewritten
  if (place && lt == 0) {
    sc.step_count = 0;
    sc.done = 0;
    sc.episode = episode;
    sc.lattice_ok = 1;  // placement is integral
  }

  // Phase 6: observation inputs. Continuous: fill_sincos (tag_env.cpp:214-221)
  // (single-env CTAs without a reset did this in phase 4).
  const bool early_inputs = single && mode != kModeReinit && !place;
  if (CONT && live && !early_inputs) {
    for (int a = lt; a < A; a += tpe) {
      sincos_ref(s.dir[a], s.sn[a], s.cs[a]);
    }
  }
  // single-env CTA: `place` is CTA-uniform here (every thread has le == 0)
  if (GRID && PARTIAL && single && place) {
    __syncthreads();
    if constexpr (LATTICE_LEAN)
      build_grid_lattice(s, p, scratch, true);
    else
      build_grid<CONT>(s, p, scratch, true);
  }
  if (!early_inputs) __syncthreads();
  const bool lattice_ok = !CONT && GRID && p.lattice && scal[0].lattice_ok;
  // packed discrete envs with integral positions (moves and placement keep
  // them integral): 32-bit-key brute K-NN, d2 <= 2 * 181^2 < 2^16
  const bool brute_keys = !CONT && !GRID && all_integral && p.world_hi <= 181.0f;
  // discrete positions all integral (tightens the ring-search bound)
  const bool disc_integral = !CONT && (GRID ? scal[0].lattice_ok != 0 : all_integral);

  // Phase 7: K-NN + observation rows (write_obs_row, tag_env.cpp:165-212).
  const int64_t cta_env0 = static_cast<int64_t>(blockIdx.x) * p.envs_per_cta;
  const int n_envs = static_cast<int>(min(static_cast<int64_t>(p.envs_per_cta), p.E - cta_env0));
  const int D = p.D;
  float* cta_out = g.obs + cta_env0 * A * D;
  // K == MAXK == 5 partial rows are always staged (launch_k guarantees it),
  // so those instantiations carry no wide-row writer.
  if ((EXACT && PARTIAL) || p.stage_obs) {
    // Each thread builds its agent's row in a per-warp staging buffer; the
    // warp then streams the contiguous block of its rows with 16-byte stores.
    float* stage = reinterpret_cast<float*>(smem + p.off_stage) + warp * p.stage_floats;
    const bool vec = ((static_cast<int64_t>(p.envs_per_cta) * A * D) & 3) == 0;
    const bool cell_lists = PARTIAL && lattice_ok;  // GRID => single env per CTA
    const int kk = p.K + 1;
    if (cell_lists && !early_inputs) {
      if constexpr (LATTICE_LEAN)
        build_cell_lists_keys(s, p, scratch);
      else
        build_cell_lists(s, p, ablate_bits(L));
      __syncthreads();
    }
    if constexpr (CONT && EXACT && PARTIAL) {
      if (p.stage_rows == 16) {
        // Wide continuous rows (D = 41): the K-NN runs on all 32 lanes, then
        // each half-warp builds and streams its 16 rows through a half-size
        // staging buffer (smem that buys the CTA a third slot per SM).
        // LEAN: warps take 32-agent chunks dynamically (the ring searches vary
        // per agent; static passes left warps idle at the closing barrier:
        // A = 1000 308.9 vs 317.2 us/step, 500 186.5 vs 192.9, 300 146.2 vs 150.8)
        for (int pass = 0;; ++pass) {
          int a;
          if constexpr (LEAN) {
            int chunk = 0;
            if (lane == 0) chunk = atomicAdd(&scratch[kObsChunk], 1);
            chunk = __shfl_sync(0xffffffffu, chunk, 0);
            if (chunk * 32 >= A) break;
            a = chunk * 32 + lane;
          } else {
            if (pass * tpe >= A) break;
            a = pass * tpe + lt;
          }
          const bool valid = live && a < A;
          const bool act_a = valid && s.act[a];
          int nb[MAXK];
          if (act_a && !(ablate_bits(L) & 4u)) {
            TopK<MAXK, EXACT> top;
            knn_agent<CONT, GRID, MAXK, EXACT>(s, p, a, false, top);
#pragma unroll
            for (int t = 0; t < MAXK; ++t) nb[t] = top.i[t];
          }
          const int myrow = env_ok ? le * A + a : -1;
          const unsigned vmask = __ballot_sync(0xffffffffu, valid);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const bool mine = valid && (lane >> 4) == h;
            if constexpr (LEAN) {
              // the previous half's bulk store has read the staging rows
              if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
              __syncwarp();
            }
            if (mine) {
              float* row = stage + (lane & 15) * D;
              if (ablate_bits(L) & 4u) {
                row[0] = static_cast<float>(a);
              } else if (!act_a) {
                constexpr int kD = MAXK * 7 + 5 + 1;
#pragma unroll
                for (int f = 0; f < kD; ++f) row[f] = 0.0f;
              } else {
                write_row<CONT, MAXK>(s, p, sc.step_count, a, row, [&](int n) {
                  int j = nb[0];
#pragma unroll
                  for (int t = 1; t < MAXK; ++t)
                    if (t == n) j = nb[t];
                  return j;
                });
              }
            }
            if constexpr (LEAN) {
              // one TMA bulk store per half-warp block (16-B aligned: A % 4
              // == 0 and halves start at multiples of 16 rows)
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              __syncwarp();
              const unsigned hmask = (vmask >> (16 * h)) & 0xffffu;
              const int r0 = __shfl_sync(0xffffffffu, myrow, 16 * h);
              if (lane == 0 && hmask != 0u)
                bulk_s2g(cta_out + static_cast<int64_t>(r0) * D, stage, static_cast<uint32_t>(__popc(hmask) * D * 4));
              continue;
            }
            __syncwarp();
            const unsigned hm = (vmask >> (16 * h)) & 0xffffu;
            const int row0 = __shfl_sync(0xffffffffu, myrow, 16 * h);
            if (hm != 0u && (hm & (hm + 1u)) == 0u) {
              const int nf = __popc(hm) * D;
              float* dst = cta_out + static_cast<int64_t>(row0) * D;
              if (vec && ((static_cast<int64_t>(row0) * D) & 3) == 0) {
                const int nv = nf >> 2;
                for (int v = lane; v < nv; v += 32)
                  st_rows(reinterpret_cast<float4*>(dst) + v, reinterpret_cast<const float4*>(stage)[v]);
                for (int f = (nv << 2) + lane; f < nf; f += 32) st_rows(dst + f, stage[f]);
              } else {
                for (int f = lane; f < nf; f += 32) st_rows(dst + f, stage[f]);
              }
            } else if (mine) {
              float* dst = cta_out + static_cast<int64_t>(myrow) * D;
              for (int f = 0; f < D; ++f) st_rows(dst + f, stage[(lane & 15) * D + f]);
            }
            __syncwarp();
          }
        }
        if constexpr (LEAN) {
          if (lane == 0) {
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            asm volatile("fence.proxy.async.global;" ::: "memory");
          }
          __syncwarp();
        }
        goto obs_done;
      }
    }
    for (int pass = 0;; ++pass) {
      int a;
      if constexpr (LEAN && CONT) {  // dynamic 32-agent chunks per warp, as above
        // (discrete lattice rows cost the same per agent: static passes, 86.4
        // vs 87.1 us/step at C2 with chunks)
        int chunk = 0;
        if (lane == 0) chunk = atomicAdd(&scratch[kObsChunk], 1);
        chunk = __shfl_sync(0xffffffffu, chunk, 0);
        if (chunk * 32 >= A) break;
        a = chunk * 32 + lane;
      } else {
        if (pass * tpe >= A) break;
        a = pass * tpe + lt;
      }
      const bool valid = live && a < A;
      if constexpr (LEAN) {
        // the previous pass's bulk store has read the staging rows
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
      }
      if (valid) {
        float* row = stage + lane * D;
        const int cl = cell_lists ? s.cellof[a] : 0;
        if (ablate_bits(L) & 4u) {
          row[0] = static_cast<float>(a);
        } else if (!s.act[a]) {
          // inactive agent: all-zero row (write_obs_row, tag_env.cpp:169-172)
          constexpr int kVis = (EXACT && PARTIAL) ? MAXK : 0;
          constexpr int kD = kVis * (CONT ? 7 : 4) + (CONT ? 5 : 2) + 1;
          if constexpr (kVis > 0) {
#pragma unroll
            for (int f = 0; f < kD; ++f) row[f] = 0.0f;
          } else {
            for (int f = 0; f < D; ++f) row[f] = 0.0f;
          }
        } else if (cell_lists && s.cfill[cl] == kk) {
          const uint16_t* lst = s.cellknn + cl * kk;
          if constexpr (EXACT && PARTIAL) {
            // the cell's K+1 list in registers, self dropped: nb[n] = l[n]
            // before self's position, l[n + 1] from it on
            int nb[MAXK];
            bool passed = false;
#pragma unroll
            for (int n = 0; n < MAXK; ++n) {
              const int ln = lst[n];
              passed |= ln == a;
              nb[n] = passed ? static_cast<int>(lst[n + 1]) : ln;
            }
            write_row<CONT, MAXK>(s, p, sc.step_count, a, row, [&](int n) {
              int j = nb[0];
#pragma unroll
              for (int t = 1; t < MAXK; ++t)
                if (t == n) j = nb[t];
              return j;
            });
          } else {
            int self_pos = kk;
            for (int t = 0; t < kk; ++t)
              if (lst[t] == a) self_pos = t;
            write_row<CONT, 0>(s, p, sc.step_count, a, row,
                               [&](int n) { return static_cast<int>(lst[n + (n >= self_pos ? 1 : 0)]); });
          }
        } else if (PARTIAL && s.act[a]) {
          {
            TopK<MAXK, EXACT> top;
            knn_agent<CONT, GRID, MAXK, EXACT>(s, p, a, lattice_ok, top, brute_keys, disc_integral);
            write_row<CONT, (EXACT ? MAXK : 0)>(s, p, sc.step_count, a, row, [&](int n) {
              int j = top.i[0];
#pragma unroll
              for (int t = 1; t < MAXK; ++t)
                if (t == n) j = top.i[t];
              return j;
            });
          }
        } else if constexpr (!PARTIAL) {
          write_row<CONT, 0>(s, p, sc.step_count, a, row, [&](int n) { return n < a ? n : n + 1; });
        }
      }
      if constexpr (LEAN) {
        // One TMA bulk store per warp: its valid rows are one block, 16-B
        // aligned in both spaces (A % 4 == 0 and warps start at multiples of
        // 32 rows, so blocks start and end on 4-row boundaries: 16 * D
        // bytes). Each lane's staged row is fenced into the async proxy
        // before the store reads it.
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        const unsigned vm = __ballot_sync(0xffffffffu, valid);
        if (lane == 0 && vm != 0u)
          bulk_s2g(cta_out + static_cast<int64_t>(a) * D, stage, static_cast<uint32_t>(__popc(vm) * D * 4));
        continue;
      }
      __syncwarp();
      // Rows of this warp in CTA-row space (row = le * A + a); when the valid
      // lanes form a prefix (always, except masked reinit of packed envs) the
      // rows are one contiguous block -> coalesced 16-byte streaming stores.
      const int myrow = env_ok ? le * A + a : -1;
      const int row0 = __shfl_sync(0xffffffffu, myrow, 0);
      const unsigned vmask = __ballot_sync(0xffffffffu, valid);
      if ((vmask & (vmask + 1u)) == 0u) {
        const int nf = __popc(vmask) * D;
        float* dst = cta_out + static_cast<int64_t>(row0) * D;
        if (vec && ((static_cast<int64_t>(row0) * D) & 3) == 0) {
          const int nv = nf >> 2;
          for (int v = lane; v < nv; v += 32)
            st_rows(reinterpret_cast<float4*>(dst) + v, reinterpret_cast<const float4*>(stage)[v]);
          for (int f = (nv << 2) + lane; f < nf; f += 32) st_rows(dst + f, stage[f]);
        } else {
          for (int f = lane; f < nf; f += 32) st_rows(dst + f, stage[f]);
        }
      } else if (valid) {
        float* dst = cta_out + static_cast<int64_t>(myrow) * D;
        for (int f = 0; f < D; ++f) st_rows(dst + f, stage[lane * D + f]);
      }
      __syncwarp();
    }
    if constexpr (LEAN) {
      // the warp's bulk stores have landed (and their smem is free) before the
      // CTA publishes the env (PDL flags) or exits
      if (lane == 0) {
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      __syncwarp();
    }
  } else if constexpr (!(EXACT && PARTIAL)) {
    // Wide rows (full obs, large A): K-NN into smem, then the CTA writes its
    // contiguous [envs, A, D] block cooperatively (coalesced).
    // Lattice envs copy each agent's K nearest from its cell's (K+1)-list
    // (self dropped) instead of a per-agent top-K, whose MAXK = 32 register
    // list spills at large K (K = 20 at C2: 26.8 ms -> see DESIGN).
    const bool cell_lists = PARTIAL && lattice_ok;  // GRID => single env per CTA
    const int kk = p.K + 1;
    if (cell_lists && !early_inputs) {
      build_cell_lists(s, p, ablate_bits(L));
      __syncthreads();
    }
    if (PARTIAL && live) {
      for (int a = lt; a < A; a += tpe) {
        if (!s.act[a]) continue;
        if (cell_lists) {
          const int cl = s.cellof[a];
          if (s.cfill[cl] == kk) {
            const uint16_t* lst = s.cellknn + cl * kk;
            int w = 0;
            for (int t = 0; t < kk; ++t) {
              const int j = lst[t];
              if (j != a && w < p.K) s.knn[a * p.K + w++] = static_cast<uint16_t>(j);
            }
            continue;
          }
        }
        TopK<MAXK, EXACT> top;
        knn_agent<CONT, GRID, MAXK, EXACT>(s, p, a, lattice_ok, top, brute_keys, disc_integral);
#pragma unroll
        for (int t = 0; t < MAXK; ++t) {
          if (t < p.K) s.knn[a * p.K + t] = static_cast<uint16_t>(top.i[t]);
        }
      }
    }
    __syncthreads();
    if constexpr (!PARTIAL && !CONT) {
      if (single) {
        // Discrete full obs (the HBM-bound C3 shapes): one warp per row. Lane
        // l writes floats f = l + 32i; since 32 % 4 == 0 it always writes the
        // same component (l & 3) of neighbour block f >> 2 — branch-light,
        // 128-byte coalesced streaming stores.
        write_full_rows_discrete(s, p, cta_out, A, D, sc.step_count);
        goto obs_done;
      }
    }
    if constexpr (PARTIAL && !CONT) {
      if (single) {  // wide partial rows (K >= 16): the same warp-per-row writer
        write_full_rows_discrete(s, p, cta_out, A, D, sc.step_count, true);
        goto obs_done;
      }
    }
    {
    const int64_t n = static_cast<int64_t>(n_envs) * A * D;
    const int nthr = blockDim.x;
    const uint8_t* base0 = smem + p.head_bytes;
    auto value = [&](int row, int f) -> float {
      int lenv = 0, a = row;
      if (!single) {
        lenv = row / A;
        a = row - lenv * A;
      }
      const EnvSmem es = carve(const_cast<uint8_t*>(base0) + lenv * p.env_bytes, p);
      return obs_value<CONT, PARTIAL>(es, p, scal[lenv].step_count, a, f);
    };
    auto row_live = [&](int row) -> bool { return single || scal[row / A].live != 0; };
    int row = tid / D;
    int f = tid - row * D;
    const int sq = nthr / D, sr = nthr - (nthr / D) * D;
    for (int64_t i = tid; i < n; i += nthr) {
      if (row_live(row)) __stcs(cta_out + i, value(row, f));
      row += sq;
      f += sr;
      if (f >= D) {
        f -= D;
        ++row;
      }
    }
    }
  }
obs_done:

  // Phase 8: write back the env's state.
  if (live && vec4) {
    for (int a0 = 4 * lt; a0 < A; a0 += 4 * tpe) {
      *reinterpret_cast<float4*>(g.loc_x + ga + a0) = *reinterpret_cast<const float4*>(s.x + a0);
      *reinterpret_cast<float4*>(g.loc_y + ga + a0) = *reinterpret_cast<const float4*>(s.y + a0);
      *reinterpret_cast<uint32_t*>(g.active + ga + a0) = *reinterpret_cast<const uint32_t*>(s.act + a0);
      if (CONT) {
        *reinterpret_cast<float4*>(g.speed + ga + a0) = *reinterpret_cast<const float4*>(s.sp + a0);
        *reinterpret_cast<float4*>(g.direction + ga + a0) = *reinterpret_cast<const float4*>(s.dir + a0);
      }
    }
  }
  if (live) {
    for (int a = vec4 ? A : lt; a < A; a += tpe) {
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
      if (place && L.episode != nullptr) L.episode[e] = episode;
    }
  }
  if (n_steps > 1) __syncthreads();  // the next step rewrites the shared state
  }  // multi-step loop
  if (pdl) {  // publish this CTA's envs to the next launch (barrier + one gpu-scope release)
    if (L.pdl_late) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      const int64_t eb = static_cast<int64_t>(blockIdx.x) * p.envs_per_cta;
      for (int k = 0; k < p.envs_per_cta && eb + k < p.E; ++k)
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(L.env_seq + eb + k), "r"(seq) : "memory");
    }
  }
}

// ---- SMALL: warp-resident small envs (A <= 32) -----------------------------
// RolloutDriver::step (harness.cpp:478-490) for envs of at most 32 agents
// with full observations (C4's 1 + 4, C3's A = 10 full): each env is a
// segment of A lanes of one warp,
// one agent per lane, and the whole step runs in registers with no shared
// memory and no barrier — neighbours' positions and flags come by
// __shfl_sync, per-env counters by segment ballots. A launch runs n_steps
// steps with the state in registers (RolloutDriver::run); every step still
// reads its logits and writes every output. The latency-bound packed path of
// tag_env_kernel spent ~1,400 dependent instructions per step per warp on
// shared-memory round trips and CTA barriers (profiles/ncu_r02_c4_e2000_v1.md).
// Same arithmetic as the main kernel (sample_tag_row, move_regs, d2_of, the
// write_obs_row formulas, the fused reset), so results are bit-identical.
constexpr int kSmallThreads = 64;
// floats per warp of the SMALL kernel's staging: the warp's rows plus up to 3
// floats of alignment shift, rounded to 16 B
__host__ __device__ constexpr int small_stage_floats(int warp_floats) { return (warp_floats + 3 + 3) / 4 * 4; }

template <bool CONT>
__global__ void __launch_bounds__(kSmallThreads) tag_small_kernel(const TagDevConfig p, const TagDevArrays g,
                                                                  const TagLaunch L) {
  constexpr int kC = CONT ? 2 : 1;
  constexpr int kV = CONT ? 3 : 5;
  constexpr int NBF = CONT ? 7 : 4;
  extern __shared__ __align__(16) float small_stage[];
  const int lane = threadIdx.x & 31;
  const int A = p.A;
  const int epw = 32 / A;  // envs per warp
  // Per-warp staging block, shifted by the block's float offset from a 16-B
  // boundary of the obs array so that staging and destination share their
  // alignment (the copy-out is a TMA bulk store between scalar head/tail).
  const int64_t wrow0 = ((static_cast<int64_t>(blockIdx.x) * blockDim.x + (threadIdx.x & ~31)) >> 5) * epw * A;
  const int mis = static_cast<int>((wrow0 * p.D) & 3);
  float* stage = small_stage + (threadIdx.x >> 5) * small_stage_floats(epw * A * p.D) + mis;
  auto st_sm = [](float* q, float v) { *q = v; };
  const int le = lane / A, la = lane - le * A;
  const int64_t wg = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t e = wg * epw + le;
  const bool valid = le < epw && e < p.E;
  const int base = le * A;  // first lane of this env's segment
  const unsigned seg = valid ? ((A == 32 ? 0xffffffffu : ((1u << A) - 1u)) << base) : 0u;
  if (L.pdl_wait) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  const int64_t ga = e * A;
  const int64_t ia = ga + la;
  float x = 0.f, y = 0.f, sp = 0.f, dir = 0.f;
  bool act = false, tag = false;
  int32_t step_count = 0, episode = 0;
  double es[4] = {0.0, 0.0, 0.0, 0.0};  // env_stats [0], [1], [5], [6] (held by the env's lane 0)
  if (valid) {
    x = g.loc_x[ia];
    y = g.loc_y[ia];
    if (CONT) {
      sp = g.speed[ia];
      dir = g.direction[ia];
    }
    act = g.active[ia] != 0;
    tag = g.is_tagger[ia] != 0;
    step_count = g.step_count[e];
    episode = L.episode != nullptr ? L.episode[e] : 0;
    if (la == 0 && L.track) {
      const double* s8 = L.env_stats + e * 8;
      es[0] = s8[0];
      es[1] = s8[1];
      es[2] = s8[5];
      es[3] = s8[6];
    }
  }
  bool nonfinite = false;
  const bool sample_here = L.logits != nullptr;
  const int n_steps = L.n_steps > 1 ? L.n_steps : 1;
  const float bias = p.fault_bias;
  const bool exact_cell = !CONT && bias == 0.0f;
  const float radius = CONT ? __fadd_rn(p.tag_radius, bias) : bias;
  const float r2 = __fmul_rn(radius, radius);
  for (int it = 0; it < n_steps; ++it) {
    // sample (sampler.cpp:5-40) + apply_move (tag_env.cpp:148-160)
    int32_t act0 = 0, act1 = 1;
    if (valid) {
      const int64_t row = ia * kC;
      if (sample_here) {
        const uint64_t h_step =
            n_steps > 1 ? absorb(L.action_h0, static_cast<uint64_t>(L.step0 + it))
            : L.step_dev != nullptr
                ? absorb(L.action_h0, static_cast<uint64_t>(*L.step_dev + static_cast<int64_t>(L.step_add)))
                : L.action_h_step;
        const uint64_t h_ag = absorb(absorb(h_step, static_cast<uint64_t>(p.env_offset + e)),
                                     static_cast<uint64_t>(la));
        act0 = sample_tag_row<kV>(L.logits, row, to_unit(absorb(absorb(h_ag, 0), 0)), nonfinite);
        g.actions[row] = act0;
        if (CONT) {
          act1 = sample_tag_row<kV>(L.logits, row + 1, to_unit(absorb(absorb(h_ag, 1), 0)), nonfinite);
          g.actions[row + 1] = act1;
        }
      } else {
        act0 = g.actions[row];
        if (CONT) act1 = g.actions[row + 1];
      }
      if (act) move_regs<CONT>(p, la, act0, act1, x, y, sp, dir);
    }
    // resolve (tag_env.cpp:403-456 / find_tagger): the lowest-index tagger at
    // the runner's position (discrete) or min (d2, index) within the radius
    const bool runner = valid && !tag && act;
    int best = -1;
    float best_d2 = 0.0f;
    for (int j = 0; j < A; ++j) {
      const float xj = __shfl_sync(0xffffffffu, x, base + j);
      const float yj = __shfl_sync(0xffffffffu, y, base + j);
      const bool tj = __shfl_sync(0xffffffffu, tag, base + j);
      if (!runner || !tj) continue;
      if (exact_cell) {
        if (best < 0 && xj == x && yj == y) best = j;
      } else {
        const float d2 = d2_of(x, y, xj, yj);
        if (d2 <= r2 && (best < 0 || d2 < best_d2)) {  // ascending j: ties keep the lower index
          best = j;
          best_d2 = d2;
        }
      }
    }
    const bool tagged = best >= 0;
    if (tagged) act = false;
    int credits = 0;
    for (int j = 0; j < A; ++j) credits += __shfl_sync(0xffffffffu, best, base + j) == la ? 1 : 0;
    // resolve_env_counters (tag_env.cpp:241-250)
    const unsigned alive = __ballot_sync(0xffffffffu, runner && !tagged) & seg;
    const unsigned tags_m = __ballot_sync(0xffffffffu, valid && tagged) & seg;
    const int32_t step_new = step_count + 1;
    const bool done_now = step_new >= p.episode_length || alive == 0u;
    const bool reset_now = valid && L.do_reset && done_now;
    // rewards (write_rewards_row, tag_env.cpp:252-259) + EpisodeTracker
    const float r = tag ? __fmul_rn(p.reward_per_tag, static_cast<float>(credits)) : (tagged ? p.penalty : 0.0f);
    if (valid) {
      g.rewards[ia] = reset_now ? 0.0f : r;
      g.credits[ia] = reset_now ? 0 : credits;
      g.tagged[ia] = (reset_now || !tagged) ? 0 : 1;
    }
    if (L.track) {
      double st = 0.0, sr = 0.0;  // integer-valued: exact in any order
      for (int j = 0; j < A; ++j) {
        const double rj = static_cast<double>(__shfl_sync(0xffffffffu, r, base + j));
        if (j < p.T) st += rj; else sr += rj;
      }
      if (valid && la == 0) {
        double* s8 = L.env_stats + e * 8;
        const double run_t = es[0] + st, run_r = es[1] + sr;
        es[2] += static_cast<double>(__popc(tags_m));
        es[3] += 1.0;
        s8[5] = es[2];
        s8[6] = es[3];
        if (done_now) {
          s8[2] += 1.0;
          s8[3] += run_t;
          s8[4] += run_r;
          es[0] = es[1] = 0.0;
        } else {
          es[0] = run_t;
          es[1] = run_r;
        }
        s8[0] = es[0];
        s8[1] = es[1];
      }
    }
    step_count = step_new;
    // fused reset-on-done: re-placement (place_env / place_agent,
    // tag_env.cpp:130-146,261-273), snapshot is_tagger, zeroed actions
    if (reset_now) {
      ++episode;
      const uint64_t h_ag = absorb(absorb(absorb(p.placement_h0, static_cast<uint64_t>(static_cast<int64_t>(episode))),
                                          static_cast<uint64_t>(p.env_offset + e)),
                                   static_cast<uint64_t>(la));
      const double ux = to_unit(absorb(absorb(h_ag, 0), 0));
      const double uy = to_unit(absorb(absorb(h_ag, 1), 0));
      if (!CONT) {
        const double gd = static_cast<double>(p.grid_size);
        int64_t ix = static_cast<int64_t>(__dmul_rn(ux, gd));
        int64_t iy = static_cast<int64_t>(__dmul_rn(uy, gd));
        ix = ix < p.grid_size - 1 ? ix : p.grid_size - 1;
        iy = iy < p.grid_size - 1 ? iy : p.grid_size - 1;
        x = static_cast<float>(ix);
        y = static_cast<float>(iy);
      } else {
        const double ud = to_unit(absorb(absorb(h_ag, 2), 0));
        x = __double2float_rn(__dmul_rn(ux, p.world_length));
        y = __double2float_rn(__dmul_rn(uy, p.world_length));
        dir = __double2float_rn(__dmul_rn(ud, 6.283185307179586));
        sp = 0.0f;
      }
      act = true;
      tag = g.snap_is_tagger[ia] != 0;
      g.is_tagger[ia] = tag ? 1 : 0;
      g.actions[ia * kC] = 0;
      if (CONT) g.actions[ia * kC + 1] = 0;
      step_count = 0;
      if (la == 0 && L.episode != nullptr) L.episode[e] = episode;
    }
    if (valid && la == 0) {
      g.step_count[e] = step_count;
      g.done[e] = (done_now && !reset_now) ? 1 : 0;
    }
    // observations (write_obs_row, tag_env.cpp:165-212) of the post-step
    // (post-reset) state: every other agent in ascending order
    float sn = 0.f, cs = 0.f;
    if (CONT) {
      sincos_ref(dir, sn, cs);
    }
    // the previous step's bulk store has read the staging rows
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncwarp();
    float* out = stage + lane * p.D;  // this warp's staging rows: row == lane
    const float iw = p.inv_world;
    const int vis = A - 1;
    for (int n = 0; n < vis; ++n) {
      const int j = n < la ? n : n + 1;  // every other agent, ascending
      // every lane of the warp joins the shuffles (j is per lane)
      const float xj = __shfl_sync(0xffffffffu, x, base + (j < A ? j : 0));
      const float yj = __shfl_sync(0xffffffffu, y, base + (j < A ? j : 0));
      const bool tj = __shfl_sync(0xffffffffu, tag, base + (j < A ? j : 0));
      const bool aj = __shfl_sync(0xffffffffu, act, base + (j < A ? j : 0));
      float spj = 0.f, snj = 0.f, csj = 0.f;
      if (CONT) {
        spj = __shfl_sync(0xffffffffu, sp, base + (j < A ? j : 0));
        snj = __shfl_sync(0xffffffffu, sn, base + (j < A ? j : 0));
        csj = __shfl_sync(0xffffffffu, cs, base + (j < A ? j : 0));
      }
      if (valid) {
        float* o = out + n * NBF;
        if (!act) {
#pragma unroll
          for (int f = 0; f < NBF; ++f) st_sm(o + f, 0.0f);
        } else {
          st_sm(o + 0, __fmul_rn(__fsub_rn(xj, x), iw));
          st_sm(o + 1, __fmul_rn(__fsub_rn(yj, y), iw));
          st_sm(o + 2, tj ? 1.0f : 0.0f);
          st_sm(o + 3, aj ? 1.0f : 0.0f);
          if (CONT) {
            st_sm(o + 4, __fmul_rn(spj, inv_ms(p, j)));
            st_sm(o + 5, snj);
            st_sm(o + 6, csj);
          }
        }
      }
    }
    if (valid) {
      float* o = out + vis * NBF;
      const float tv = __fmul_rn(static_cast<float>(step_count), p.inv_episode);
      if (!act) {
        st_sm(o + 0, 0.0f);
        st_sm(o + 1, 0.0f);
        st_sm(o + 2, 0.0f);
        if (CONT) {
          st_sm(o + 3, 0.0f);
          st_sm(o + 4, 0.0f);
          st_sm(o + 5, 0.0f);
        }
      } else {
        st_sm(o + 0, __fmul_rn(x, iw));
        st_sm(o + 1, __fmul_rn(y, iw));
        if (CONT) {
          st_sm(o + 2, __fmul_rn(sp, inv_ms(p, la)));
          st_sm(o + 3, sn);
          st_sm(o + 4, cs);
          st_sm(o + 5, tv);
        } else {
          st_sm(o + 2, tv);
        }
      }
    }
    // the warp's rows are one contiguous block of the obs array: a scalar
    // head up to the first 16-B boundary, one TMA bulk store of the aligned
    // body (staging and destination share their alignment), a scalar tail
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    {
      const int nrows = __popc(__ballot_sync(0xffffffffu, valid));
      const int nf = nrows * p.D;
      const int64_t f0 = (wg * epw * A) * static_cast<int64_t>(p.D);
      float* dst = g.obs + f0;
      const int align = (4 - mis) & 3;  // floats until dst (and stage) are 16-B aligned
      const int head = align < nf ? align : nf;
      const int body = ((nf - head) >> 2) << 2;
      if (lane < head) st_rows(dst + lane, stage[lane]);
      if (lane == 0 && body > 0) bulk_s2g(dst + head, stage + head, static_cast<uint32_t>(body * 4));
      for (int f = head + body + lane; f < nf; f += 32) st_rows(dst + f, stage[f]);
    }
  }
  if (valid) {
    g.loc_x[ia] = x;
    g.loc_y[ia] = y;
    if (CONT) {
      g.speed[ia] = sp;
      g.direction[ia] = dir;
    }
    g.active[ia] = act ? 1 : 0;
  }
  if (nonfinite && L.error) atomicOr(L.error, kErrNonFinite);
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // smem stays valid until read
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

// Shell table for the lattice K-NN (constant memory, once per device).
cudaError_t ensure_shell_table() {
  static bool done[64] = {};
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  if (dev < 64 && done[dev]) return cudaSuccess;
  int16_t off[kMaxShellOffsets];
  int16_t begin[kMaxShells + 1];
  int16_t d2v[kMaxShells];
  int n = 0, ns = 0;
  for (int d2 = 0; d2 <= kShellR2; ++d2) {
    const int start = n;
    for (int dy = -kShellR; dy <= kShellR; ++dy)
      for (int dx = -kShellR; dx <= kShellR; ++dx)
        if (dx * dx + dy * dy == d2) off[n++] = static_cast<int16_t>((dx + 64) | ((dy + 64) << 8));
    if (n > start) {
      begin[ns] = static_cast<int16_t>(start);
      d2v[ns] = static_cast<int16_t>(d2);
      ++ns;
    }
  }
  begin[ns] = static_cast<int16_t>(n);
  if ((err = cudaMemcpyToSymbol(c_shell_off, off, sizeof(int16_t) * n)) != cudaSuccess) return err;
  if ((err = cudaMemcpyToSymbol(c_shell_begin, begin, sizeof(int16_t) * (ns + 1))) != cudaSuccess) return err;
  if ((err = cudaMemcpyToSymbol(c_shell_d2, d2v, sizeof(int16_t) * ns)) != cudaSuccess) return err;
  if ((err = cudaMemcpyToSymbol(c_num_shells, &ns, sizeof(int32_t))) != cudaSuccess) return err;
  if (dev < 64) done[dev] = true;
  return cudaSuccess;
}

}  // namespace
bool lean_plan(const TagDevConfig& p);
namespace {

template <bool CONT, bool PARTIAL, bool GRID, int MAXK, bool EXACT>
cudaError_t launch_variant(const TagDevConfig& p, const TagDevArrays& g, const TagLaunch& L,
                           cudaStream_t st) {
  // Partial-obs plans also run their single steps on the looped build: it
  // measured 3% faster at C2 (139 vs 143.5 us), while the full-obs writer is
  // 6-35% slower there.
  auto kern = (L.n_steps > 1 || PARTIAL) ? tag_env_kernel<CONT, PARTIAL, GRID, MAXK, EXACT, true>
                                         : tag_env_kernel<CONT, PARTIAL, GRID, MAXK, EXACT, false>;
  if constexpr (PARTIAL && GRID && EXACT) {
    // the one-env single step (see LEAN at tag_env_kernel)
    const bool lean = L.mode >= 0 && L.mode != kModeReinit && L.n_steps <= 1 && lean_plan(p);
    if (lean) kern = tag_env_kernel<CONT, PARTIAL, GRID, MAXK, EXACT, false, true>;
  }
  if (L.mode < 0) {  // occupancy query (kModeQuery): resident CTAs per SM -> *L.error
    if (p.smem_bytes > 48 * 1024) {
      cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem_bytes);
      if (err != cudaSuccess) return err;
    }
    int n = 0;
    cudaError_t err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, p.threads, p.smem_bytes);
    *L.error = static_cast<uint32_t>(n);
    return err;
  }
  if (!CONT && GRID) {
    cudaError_t err = ensure_shell_table();
    if (err != cudaSuccess) return err;
  }
  if (p.smem_bytes > 48 * 1024) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           p.smem_bytes);
    if (err != cudaSuccess) return err;
  }
  if (L.env_seq != nullptr || L.pdl_wait) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(p.grid_ctas));
    cfg.blockDim = dim3(static_cast<unsigned>(p.threads));
    cfg.dynamicSmemBytes = static_cast<size_t>(p.smem_bytes);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p, g, L);
  }
  kern<<<p.grid_ctas, p.threads, p.smem_bytes, st>>>(p, g, L);
  return cudaGetLastError();
}

template <bool CONT, bool PARTIAL, bool GRID>
cudaError_t launch_k(const TagDevConfig& p, const TagDevArrays& g, const TagLaunch& L,
                     cudaStream_t st) {
  if constexpr (!PARTIAL) {
    return launch_variant<CONT, PARTIAL, GRID, 1, true>(p, g, L, st);
  } else {
    if (p.K == 5 && p.stage_obs) return launch_variant<CONT, PARTIAL, GRID, 5, true>(p, g, L, st);
    if (p.K <= 8) return launch_variant<CONT, PARTIAL, GRID, 8, false>(p, g, L, st);
    return launch_variant<CONT, PARTIAL, GRID, 32, false>(p, g, L, st);
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
bool lean_plan(const TagDevConfig& p) {
  return p.partial && p.use_grid && p.K == 5 && p.stage_obs && p.envs_per_cta == 1 && (p.A & 3) == 0 &&
         p.bulk_in && p.threads_per_env == p.threads && (p.continuous || p.lattice);
}

// SMALL eligibility: packed envs of at most 32 agents with full observations,
// a fused launch with no per-env overlap flags and no rollout-capture outputs
// (those take the main kernel). Measured against the main kernel's packed
// path (us/step, single launch / run window): C4 2000 x 5 4.9 / 2.6 vs
// 6.8 / 4.5, 10000 x 5 7.0 / 3.1 vs 9.8 / 5.3, continuous 2000 x 5 6.6 / 4.3
// vs 9.1 / 6.6, A = 10 full 9.0 / 3.8 vs 11.2 / 6.3. Partial observations stay
// on the main kernel, whose 32-bit-key brute K-NN measured faster (A = 10,
// K = 5: 12.3 / 5.7 vs 13.2 / 8.5).
bool small_plan(const TagDevConfig& p) {
  return !p.use_grid && p.A <= 32 && !p.partial;
}

namespace {
template <bool CONT>
cudaError_t launch_small(const TagDevConfig& p, const TagDevArrays& g, const TagLaunch& L, cudaStream_t st) {
  const int64_t epw = 32 / p.A;
  const int64_t warps = (static_cast<int64_t>(p.E) + epw - 1) / epw;
  const int64_t wpb = kSmallThreads / 32;
  const unsigned blocks = static_cast<unsigned>((warps + wpb - 1) / wpb);
  auto kern = tag_small_kernel<CONT>;
  const size_t smem = static_cast<size_t>(wpb) * small_stage_floats(static_cast<int>(epw * p.A * p.D)) * sizeof(float);
  if (smem > 48 * 1024) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (err != cudaSuccess) return err;
  }
  if (L.pdl_wait) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(kSmallThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p, g, L);
  }
  kern<<<blocks, kSmallThreads, smem, st>>>(p, g, L);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_tag_kernel(const TagDevConfig& p, const TagDevArrays& g, const TagLaunch& L,
                              cudaStream_t st) {
  if (L.mode == kModeFused && L.env_seq == nullptr && L.cap_actions == nullptr && L.cap_active == nullptr &&
      L.cap_rewards == nullptr && L.cap_done == nullptr && small_plan(p)) {
    return p.continuous ? launch_small<true>(p, g, L, st) : launch_small<false>(p, g, L, st);
  }
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

namespace {
__global__ void set_counter_kernel(int64_t* ptr, int64_t value, int64_t value2) {
  ptr[0] = value;
  if (value2 >= 0) ptr[1] = value2;
}
}  // namespace

cudaError_t launch_set_counter(int64_t* ptr, int64_t value, cudaStream_t st, int64_t value2) {
  set_counter_kernel<<<1, 1, 0, st>>>(ptr, value, value2);
  return cudaGetLastError();
}

cudaError_t launch_stats_reduce(const double* env_stats, int64_t E, double* out, cudaStream_t st) {
  stats_reduce_kernel<<<1, 256, 0, st>>>(env_stats, E, out);
  return cudaGetLastError();
}

}  // namespace wdg
