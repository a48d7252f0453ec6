// matern.cuh — the Matérn-5/2 cross-covariance K*(x, x_j) shared by the FP64 and tensor-core
// posterior kernels (surrogate.py:142-145, 318-321).
#pragma once
#include "bx_common.cuh"

namespace bx {

// sigma * matern52(sqrt(W)) with 18 FP64 operations instead of the ~47 of sqrt() + exp():
//   d  = W * y,  y = rsqrt(W) from MUFU.RSQ64H refined by one Newton step (rel. err ~2^-46)
//   e^x, x = -sqrt5 d: x = (64 k + j) ln2/64 + r, |r| <= ln2/128, 2^(j/64) from a 64-entry table,
//        degree-5 Taylor in r (truncation < 4e-17), 2^k folded into the table value's exponent
//   K  = (sigma + sigma sqrt5 d + sigma 5/3 W) e
// The table is exact to 1/2 ulp (host-computed with long double), so K* is within a few ulp of
// the reference's sigma * (1 + sqrt5 d + 5/3 d^2) * exp(-sqrt5 d) (surrogate.py:142-145, 321).
struct MaternConst {
  double s0, s1, s2;  // sigma, sigma*sqrt5, sigma*5/3
};

__device__ __forceinline__ double rsqrt_approx(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

__device__ __forceinline__ double kstar_fast(double W, const MaternConst& mc, const double* exp2tab) {
  const double w = fmax(W, 1e-300);                 // W = 0 -> d ~ 1e-150 -> K* = sigma exactly
  double y = rsqrt_approx(w);
  y = y * fma(-0.5 * w * y, y, 1.5);                // Newton step for 1/sqrt(w)
  const double d = w * y;
  const double x = -kSqrt5 * d;
  // k = rint(x * 64 / ln2) via the 1.5 * 2^52 shifter
  const double t = fma(x, 92.332482616893656877, 6755399441055744.0);
  const int k = __double2loint(t);
  const double kf = t - 6755399441055744.0;
  double r = fma(kf, -0.010830424696223417, x);     // ln2/64 split: hi (exact product) ...
  r = fma(kf, -2.572804622327669e-14, r);           // ... and lo
  double p = fma(r, 1.0 / 120.0, 1.0 / 24.0);
  p = fma(r, p, 1.0 / 6.0);
  p = fma(r, p, 0.5);
  p = fma(r, p, 1.0);
  p = fma(r, p, 1.0);
  // 2^(j/64) * 2^(k >> 6): add the integer exponent to the table entry's exponent field
  const double tj = exp2tab[k & 63];
  const int hi = __double2hiint(tj) + ((k >> 6) << 20);
  const double scale = __hiloint2double(hi, __double2loint(tj));
  const double e = (x < -700.0) ? 0.0 : p * scale;
  return fma(mc.s2, W, fma(mc.s1, d, mc.s0)) * e;
}

__device__ __forceinline__ double kstar(double W, double sigma) {
  const double d = sqrt(fmax(W, 0.0));
  const double e = exp(-kSqrt5 * d);
  return sigma * ((1.0 + kSqrt5 * d + (5.0 / 3.0) * d * d) * e);
}

}  // namespace bx
