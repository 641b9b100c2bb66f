// device_ref.cuh — leaf arithmetic shared by the production Tag kernels
// (tag_kernels.cu) and the device TagReference twin (twin_kernels.cu): the
// reference's counter RNG, std::min/std::max semantics and its libm's
// sinf/cosf. These are the reference's own primitives ("libm" of the path);
// everything above them (K-NN, resolve, observation writers, resets) is
// implemented independently in the two files.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

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

// sinf / cosf exactly as the reference's libm computes them (SURVEY.md §8f
// row 4). The reference calls std::sin/std::cos on float, i.e. glibc 2.39
// sinf/cosf, whose x86-64 build dispatches (ifunc) to an FMA variant on
// FMA-capable hosts. That variant is the optimized-routines algorithm: |x| <
// pi/4 -> an odd/even polynomial in double; |x| < 120 -> n = round(x * 2/pi)
// via (int)(x * 2^24 * 2/pi) + 2^23 >> 24, r = fma(-n, pi/2, x), then the
// sin or cos polynomial of r with coefficient table n & 2 and sign n & 3 — every
// a*b+c fused exactly where the FMA build fuses it (read off the shipped
// libm.so.6, s_sinf-fma / s_cosf-fma). tests/test_trig.py checks the same
// steps, restated in C for the tests, against the host libm on every float in
// [-2pi, 2pi].
// |x| >= 120 (never produced by the env: directions stay in [0, 2pi)) uses
// the f64 sin/cos rounded once.
struct SinCosTab {
  double hpi_inv, hpi, c0, c1, s1, c2, s2, c3, s3, c4;
};
__constant__ SinCosTab c_sincos[2] = {
    {0x1.45f306dc9c883p+23, 0x1.921fb54442d18p+0, 0x1.0p+0, -0x1.ffffffd0c621cp-2, -0x1.555545995a603p-3,
     0x1.55553e1068f19p-5, 0x1.1107605230bc4p-7, -0x1.6c087e89a359dp-10, -0x1.994eb3774cf24p-13,
     0x1.99343027bf8c3p-16},
    {0x1.45f306dc9c883p+23, 0x1.921fb54442d18p+0, -0x1.0p+0, 0x1.ffffffd0c621cp-2, -0x1.555545995a603p-3,
     -0x1.55553e1068f19p-5, 0x1.1107605230bc4p-7, 0x1.6c087e89a359dp-10, -0x1.994eb3774cf24p-13,
     -0x1.99343027bf8c3p-16}};
__device__ __forceinline__ double sinf_poly(double xs, double x2, const SinCosTab& p) {
  const double a = __fma_rn(x2, p.s3, p.s2);
  const double x3 = __dmul_rn(x2, xs);
  const double x5 = __dmul_rn(x2, x3);
  return __fma_rn(a, x5, __fma_rn(x3, p.s1, xs));
}
__device__ __forceinline__ double cosf_poly(double x2, const SinCosTab& p) {
  const double x4 = __dmul_rn(x2, x2);
  const double a = __fma_rn(x2, p.c1, p.c0);
  const double b = __fma_rn(x2, p.c4, p.c3);
  const double x6 = __dmul_rn(x2, x4);
  return __fma_rn(b, x6, __fma_rn(x4, p.c2, a));
}
// want_cos: cosf, else sinf.
__device__ __forceinline__ float sincosf_ref(float y, bool want_cos) {
  const uint32_t top = (__float_as_uint(y) >> 20) & 0x7ffu;
  const double x = static_cast<double>(y);
  if (top <= 0x3f3u) {  // |y| < pi/4
    if (top <= 0x397u) return want_cos ? 1.0f : y;
    const double x2 = __dmul_rn(x, x);
    return __double2float_rn(want_cos ? cosf_poly(x2, c_sincos[0]) : sinf_poly(x, x2, c_sincos[0]));
  }
  if (top > 0x42eu) {  // |y| >= 120: outside the replica (not reachable from the env)
    return __double2float_rn(want_cos ? cos(x) : sin(x));
  }
  const int n = (__double2int_rz(__dmul_rn(x, c_sincos[0].hpi_inv)) + 0x800000) >> 24;
  const double r = __fma_rn(-static_cast<double>(n), c_sincos[0].hpi, x);
  const SinCosTab& p = c_sincos[(n & 2) ? 1 : 0];
  const double x2 = __dmul_rn(r, r);
  const bool cos_poly = ((n & 1) == 0) == want_cos;
  if (cos_poly) return __double2float_rn(cosf_poly(x2, p));
  const double sign = ((n + 1) & 2) ? -1.0 : 1.0;  // sign[n & 3] = {1, -1, -1, 1}
  return __double2float_rn(sinf_poly(__dmul_rn(r, sign), x2, p));
}
__device__ __forceinline__ float sin_ref(float v) { return sincosf_ref(v, false); }
__device__ __forceinline__ float cos_ref(float v) { return sincosf_ref(v, true); }
// sin_ref and cos_ref of one value with one range reduction: the same steps
// as the two calls (the quadrant's table and sign serve both; one of the two
// takes the cos polynomial, the other the signed sin polynomial).
__device__ __forceinline__ void sincos_ref(float y, float& sn, float& cs) {
  const uint32_t top = (__float_as_uint(y) >> 20) & 0x7ffu;
  const double x = static_cast<double>(y);
  if (top <= 0x3f3u) {  // |y| < pi/4
    if (top <= 0x397u) {
      sn = y;
      cs = 1.0f;
      return;
    }
    const double x2 = __dmul_rn(x, x);
    sn = __double2float_rn(sinf_poly(x, x2, c_sincos[0]));
    cs = __double2float_rn(cosf_poly(x2, c_sincos[0]));
    return;
  }
  if (top > 0x42eu) {  // |y| >= 120: outside the replica (not reachable from the env)
    sn = __double2float_rn(sin(x));
    cs = __double2float_rn(cos(x));
    return;
  }
  const int n = (__double2int_rz(__dmul_rn(x, c_sincos[0].hpi_inv)) + 0x800000) >> 24;
  const double r = __fma_rn(-static_cast<double>(n), c_sincos[0].hpi, x);
  const SinCosTab& p = c_sincos[(n & 2) ? 1 : 0];
  const double x2 = __dmul_rn(r, r);
  const double sign = ((n + 1) & 2) ? -1.0 : 1.0;  // sign[n & 3] = {1, -1, -1, 1}
  const float cp = __double2float_rn(cosf_poly(x2, p));
  const float sp = __double2float_rn(sinf_poly(__dmul_rn(r, sign), x2, p));
  sn = (n & 1) ? cp : sp;
  cs = (n & 1) ? sp : cp;
}

}  // namespace
}  // namespace wdg
