// Bit-exact float64 quantization / reconstruction / rescale, per element.
//
// Contract (reference codec.py:118-155, ops.py:199-208):
// IEEE-754 binary64, round-to-nearest-even, no FMA contraction anywhere --
// every product/sum below is an explicit __d*_rn intrinsic, which nvcc never
// fuses.
#pragma once

#include "hsz_common.cuh"

namespace hsz {

struct QuantConst {
  double eps;      // absolute bound
  double d;        // 2.0 * eps (exact)
  double rcp_d;    // RN(1/d), only used when fast_div
  double eps_tol;  // RN(eps * RN(1 + 1e-9))       codec.py:151
  int fast_div;    // reciprocal fast path allowed (d well inside the normal range)
};

__host__ inline QuantConst make_quant_const(double eps) {
  QuantConst c;
  c.eps = eps;
  c.d = 2.0 * eps;
  volatile double one_plus = 1.0 + 1e-9;   // Python folds 1.0 + 1e-9 to one double
  c.eps_tol = eps * one_plus;
  c.rcp_d = 1.0 / c.d;
  c.fast_div = (c.d > 0x1p-1000 && c.d < 0x1p+1000) ? 1 : 0;
  return c;
}

// floor(RN(s / d)) exactly.  Fast path: y = RN(s * RN(1/d)) is within
// ~2^-52 relative of s/d, so when y sits more than 2^-50 |y| away from both
// neighbouring integers, RN(s/d) has the same floor.  Anything closer to an
// integer boundary (including exact grid points) takes the IEEE division.
__device__ __forceinline__ double floor_div(double s, const QuantConst& c) {
  if (c.fast_div) {
    const double y = __dmul_rn(s, c.rcp_d);
    const double m = floor(y);
    const double f = __dsub_rn(y, m);                  // exact
    const double tau = __dmul_rn(fabs(y), 0x1p-50);
    if (f > tau && __dsub_rn(1.0, f) > tau) return m;
  }
  return floor(__ddiv_rn(s, c.d));
}

// One element of quantize() (codec.py:132-154).  Returns the int64 bin and
// ORs HSZ_ERR_* bits into *flags.
__device__ __forceinline__ int64_t quantize1(double x, const QuantConst& c, uint32_t* flags) {
  const double s = __dadd_rn(x, c.eps);
  const double m = floor_div(s, c);
  if (!(fabs(m) < 0x1p63)) {                            // also catches inf / nan
    *flags |= HSZ_ERR_QUANT_OVERFLOW;
    return 0;
  }
  int64_t q = __double2ll_rz(m);
  const double err = __dsub_rn(x, __dmul_rn(c.d, m));
  if (fabs(err) > c.eps) {                              // repair pass, codec.py:140-154
    const int64_t moved = q + (err > 0.0 ? 1 : -1);
    const double err2 = __dsub_rn(x, __dmul_rn(c.d, __ll2double_rn(moved)));
    double fin = err;
    if (fabs(err2) < fabs(err)) {
      q = moved;
      fin = err2;
    }
    if (fabs(fin) > c.eps_tol) *flags |= HSZ_ERR_QUANT_RESOLUTION;
  }
  return q;
}

// Fast exact quantization for the fast-path range.  With |y| < 2^30 the
// reciprocal quotient y = RN(s * RN(1/d)) is within 1.5 * 2^-22 of s/d, so if
// y - floor(y) is more than 2^-20 away from an integer:
//   * floor(RN(s/d)) == floor(y), and
//   * |x - d*m| <= eps - d * 2^-22 even after the reference's two roundings,
//     so its repair pass (codec.py:140-154) provably does not fire.
// Returns false (caller must use quantize1) otherwise.  6 FP64 ops; the int
// conversion uses the 1.5 * 2^52 magic constant instead of F2I.
__device__ __forceinline__ bool quantize_fast(double x, const QuantConst& c, int32_t* q) {
  const double s = __dadd_rn(x, c.eps);
  const double y = __dmul_rn(s, c.rcp_d);
  const double m = floor(y);
  const double g = __dsub_rn(__dsub_rn(y, m), 0.5);
  const double k = __dadd_rn(m, 6755399441055744.0);
  *q = __double2loint(k);
  return (fabs(y) < 0x1p30 - 2.0) & (fabs(g) < 0.5 - 0x1p-20) & (c.fast_div != 0);
}

// exact int32 -> double: the conversion unit (one instruction), or without a
// conversion instruction (biased mantissa minus 2^52 + 2^31: three)
#ifndef HSZ_I2F_CVT
#define HSZ_I2F_CVT 1
#endif
__device__ __forceinline__ double i32_to_double(int32_t v) {
#if HSZ_I2F_CVT
  return __int2double_rn(v);
#else
  return __dsub_rn(__hiloint2double(0x43300000, static_cast<int>(static_cast<uint32_t>(v) ^ 0x80000000u)),
                   4503601774854144.0);   // 2^52 + 2^31
#endif
}

// Reconstruction RN(d * f64(bin)) (codec.py:107-109); int64 -> f64 is RN.
__device__ __forceinline__ double grid1(int64_t bin, double d) {
  return __dmul_rn(d, __ll2double_rn(bin));
}

// Scalar-multiply rescale of one exact product p (ops.py:199-208):
//   t = RN(d * RN(p)); mag = floor(RN(|t| + 0.5)); bin = t < 0 ? -mag : mag
__device__ __forceinline__ int64_t rescale1(double pd, double d, uint32_t* flags) {
  const double t = __dmul_rn(d, pd);
  const double mag = floor(__dadd_rn(fabs(t), 0.5));
  if (!(mag < 0x1p63)) {
    *flags |= HSZ_ERR_RESCALE_OVERFLOW;
    return 0;
  }
  const int64_t m = __double2ll_rz(mag);
  return t < 0.0 ? -m : m;
}

// exact product bin * rs rounded to double
__device__ __forceinline__ double product_rn(int64_t bin, int64_t rs) {
  const __int128 p = static_cast<__int128>(bin) * static_cast<__int128>(rs);
  const int64_t lo = static_cast<int64_t>(p);
  if (static_cast<__int128>(lo) == p) return __ll2double_rn(lo);
  return i128_to_double_rn(p);
}

}  // namespace hsz
