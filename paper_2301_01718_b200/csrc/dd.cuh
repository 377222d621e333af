// dd.cuh -- double-double (hi + lo) accumulation for the Gram pipeline (G11).
//
// The POD of Eq. 9 and the gappy normal equations of Eq. 8 are formed from
// Grams on the GPU (G3, G4).  A Gram rounded to fp64 carries errors of eps * ||x_i|| ||x_j||,
// which the eigen-solve turns into subspace errors eps * lambda_1 / gap_lambda (A15) -- the
// square of the SVD's eps * sigma_1 / gap_sigma.  Every Gram entry is therefore accumulated as
// an unevaluated sum hi + lo: the products exactly (TwoProduct by FMA), the sums by TwoSum, so
// an entry is the exact Gram of the fp64 operands to ~eps^2 (plus n eps^2 sum |x_i x_j|).
#pragma once

namespace hrom {

// (hi, lo) += a * b  (TwoProduct + TwoSum; lo collects both rounding errors)
__device__ __forceinline__ void dd_fma(double& hi, double& lo, double a, double b) {
  const double p = a * b;
  const double pe = fma(a, b, -p);
  const double s = hi + p;
  const double z = s - hi;
  const double e = (hi - (s - z)) + (p - z);
  hi = s;
  lo += e + pe;
}

// (hi, lo) += x
__device__ __forceinline__ void dd_add1(double& hi, double& lo, double x) {
  const double s = hi + x;
  const double z = s - hi;
  const double e = (hi - (s - z)) + (x - z);
  hi = s;
  lo += e;
}

// (hi, lo) += (bh, bl), result renormalised (|lo| <= ulp(hi) / 2)
__device__ __forceinline__ void dd_add(double& hi, double& lo, double bh, double bl) {
  const double s = hi + bh;
  const double z = s - hi;
  const double e = (hi - (s - z)) + (bh - z);
  const double t = e + (lo + bl);
  hi = s + t;
  lo = t - (hi - s);
}

// renormalise (hi, lo) so that hi = fl(hi + lo)
__device__ __forceinline__ void dd_norm(double& hi, double& lo) {
  const double s = hi + lo;
  lo = lo - (s - hi);
  hi = s;
}

// (hi, lo) * d for a double d (product of a double-double with a double, ~eps^2 relative)
__device__ __forceinline__ void dd_mul1(double& hi, double& lo, double d) {
  const double p = hi * d;
  const double pe = fma(hi, d, -p);
  const double t = fma(lo, d, pe);
  hi = p + t;
  lo = t - (hi - p);
}

// (hi, lo) / d for a double d
__device__ __forceinline__ void dd_div1(double& hi, double& lo, double d) {
  const double q = hi / d;
  // remainder (hi, lo) - q d, exactly in the leading part
  const double p = q * d;
  const double pe = fma(q, d, -p);
  const double r = ((hi - p) - pe) + lo;
  const double q2 = r / d;
  hi = q + q2;
  lo = q2 - (hi - q);
}

// (hi, lo) += a * b with hi biased far above every partial sum and product (|hi| >= |a b|,
// hi = B + S, B a power of two >= 2 max |S|): TwoProduct by FMA, then the exact Fast2Sum
// (3 operations instead of TwoSum's 6); the value is (hi - B) + lo, hi - B exact (Sterbenz)
// (the two error terms are added to lo one at a time, the TwoProduct error first: in the
// register-bound fill loop this form needs no register moves between iterations -- the fill went
// from 1.70 to 1.63 ms against lo += e + pe)
__device__ __forceinline__ void biased_fma(double& hi, double& lo, double a, double b) {
  const double p = a * b;
  lo += fma(a, b, -p);  // TwoProduct error
  const double s = hi + p;
  lo += p - (s - hi);   // Fast2Sum error (|hi| >= |p|)
  hi = s;
}

// bias for Gram entries of columns whose squared norms are at most cmax: every partial sum
// |sum x_i x_j| <= ||x_i|| ||x_j|| stays below B / 2 with an 8x margin on the norms
__device__ __forceinline__ double gram_bias(double cmax) {
  return cmax > 0.0 ? ldexp(1.0, ilogb(256.0 * cmax) + 1) : 1.0;
}

}  // namespace hrom
