// Double-double accumulation for the solvers' dot products (reference
// include/hsolve/dd.hpp:13-40): an unevaluated pair hi + lo, Knuth's
// error-free TwoSum, and the two additions the reference combines per-row
// and per-executor partials with. Header-only host code; the B200 kernels
// carry the same arithmetic on the device (csrc/hs_common.cuh). Depends on
// IEEE evaluation order: never compile with -ffast-math /
// -fassociative-math.
#pragma once

namespace hsolve {

struct Dd {
  double hi = 0.0;
  double lo = 0.0;
};

// s + e == a + b exactly (Knuth TwoSum, no branch on magnitudes)
inline Dd two_sum(double a, double b) {
  const double s = a + b;
  const double bv = s - a;
  const double av = s - bv;
  return {s, (a - av) + (b - bv)};
}

// acc + x, renormalised
inline Dd dd_add(Dd acc, double x) {
  const Dd s = two_sum(acc.hi, x);
  const double lo = acc.lo + s.lo;
  const double hi = s.hi + lo;
  return {hi, lo - (hi - s.hi)};
}

// a + b for two double-double partials, renormalised
inline Dd dd_add(Dd a, Dd b) {
  const Dd s = two_sum(a.hi, b.hi);
  const double lo = s.lo + (a.lo + b.lo);
  const double hi = s.hi + lo;
  return {hi, lo - (hi - s.hi)};
}

inline double dd_value(Dd a) { return a.hi + a.lo; }

}  // namespace hsolve
