// gvo_exp.cuh — device port of the double-precision exp algorithm glibc
// (>= 2.28, x86-64 FMA variant) uses for Python's math.exp, so the Gompertz
// ratio curves (reference fit.py:51-57) are bit-identical to the CPU
// reference.  CUDA's exp() is within 1 ulp but not identical; ranking ties
// need identical values.  Verified by tools/gen_exp_table.py (bit-exact
// against math.exp on random inputs) and by tests/test_gpu_parity.py.
#pragma once
#include <cstdint>

namespace gvo {

__device__ __constant__ static const uint64_t kExpTab[256] = {
#include "gvo_exp_table.inc"
};

__device__ __forceinline__ uint32_t top12(double x) { return (uint32_t)(__double_as_longlong(x) >> 52) & 0xfffu; }

__device__ inline double exp_specialcase(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000ull) == 0) {
    sbits -= 1009ull << 52;
    const double scale = __longlong_as_double((long long)sbits);
    return 0x1p1009 * __fma_rn(scale, tmp, scale);
  }
  sbits += 1022ull << 52;
  const double scale = __longlong_as_double((long long)sbits);
  double y = __fma_rn(scale, tmp, scale);
  if (y < 1.0) {
    double lo = __fma_rn(scale, tmp, __dsub_rn(scale, y));
    const double hi = __dadd_rn(1.0, y);
    lo = __dadd_rn(__dadd_rn(__dsub_rn(1.0, hi), y), lo);
    y = __dsub_rn(__dadd_rn(hi, lo), 1.0);
    if (y == 0.0) y = 0.0;
  }
  return 0x1p-1022 * y;
}

__device__ inline double glibc_exp(double x) {
  const double InvLn2N = 0x1.71547652b82fep0 * 128.0;
  const double NegLn2hiN = -0x1.62e42fefa0000p-8;
  const double NegLn2loN = -0x1.cf79abc9e3b3ap-47;
  const double Shift = 0x1.8p52;
  const double C2 = 0x1.ffffffffffdbdp-2, C3 = 0x1.555555555543cp-3;
  const double C4 = 0x1.55555cf172b91p-5, C5 = 0x1.1111167a4d017p-7;
  uint32_t abstop = top12(x) & 0x7ffu;
  if (abstop - top12(0x1p-54) >= top12(512.0) - top12(0x1p-54)) {
    if ((int32_t)(abstop - top12(0x1p-54)) < 0) return __dadd_rn(1.0, x);
    if (abstop >= top12(1024.0)) {
      if ((uint64_t)__double_as_longlong(x) == 0xfff0000000000000ull) return 0.0;
      if (abstop >= top12(__longlong_as_double(0x7ff0000000000000ll))) return __dadd_rn(1.0, x);
      return (__double_as_longlong(x) < 0) ? 0.0 : __longlong_as_double(0x7ff0000000000000ll);
    }
    abstop = 0;
  }
  const double z = __dmul_rn(InvLn2N, x);
  double kd = __dadd_rn(z, Shift);
  const uint64_t ki = (uint64_t)__double_as_longlong(kd);
  kd = __dsub_rn(kd, Shift);
  const double r = __fma_rn(kd, NegLn2loN, __fma_rn(kd, NegLn2hiN, x));
  const uint32_t idx = 2u * (uint32_t)(ki % 128u);
  const uint64_t top = ki << (52 - 7);
  const double tail = __longlong_as_double((long long)kExpTab[idx]);
  const uint64_t sbits = kExpTab[idx + 1] + top;
  const double r2 = __dmul_rn(r, r);
  const double tmp = __fma_rn(__dmul_rn(r2, r2), __fma_rn(r, C5, C4),
                              __fma_rn(r2, __fma_rn(r, C3, C2), __dadd_rn(tail, r)));
  if (abstop == 0) return exp_specialcase(tmp, sbits, ki);
  const double scale = __longlong_as_double((long long)sbits);
  return __fma_rn(scale, tmp, scale);
}

}  // namespace gvo
