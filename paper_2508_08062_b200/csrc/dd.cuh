// dd.cuh — double-double arithmetic for the FAA step (aa.cuh).
//
// The reference forms FAA's least-squares solve with a Householder QR of
// the kept residual-difference columns F (filtering.cpp:25-50,
// sparse_linalg.cpp:131-192): a backward-stable solve whose error grows like
// kappa(F) u. The device reduces F'F, F'g in one pass over the history
// instead (the columns stay in HBM, no Q is formed). In plain doubles that
// squares the conditioning (kappa^2 u); with every product and sum carried
// as an unevaluated pair hi + lo (TwoProd via FMA, TwoSum — the Dot2
// accumulation of Ogita, Rump and Oishi) and the p x p Cholesky / triangular
// solves in the same arithmetic, the Gram and its factor are accurate to
// ~u^2 |F|^2, so the weights carry an error ~kappa^2 u^2 + u: below the
// reference's own kappa u for every kappa < 1/u.
//
// All operations are explicitly rounded (__dadd_rn / __dmul_rn / __fma_rn):
// -fmad=false never contracts them, and the FMA in TwoProd is deliberate.
#pragma once

namespace aapdhg_b200 {

struct dd {
  double hi, lo;
};

__device__ __forceinline__ dd two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  const double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
  return {s, e};
}

// |a| >= |b| (or a == 0)
__device__ __forceinline__ dd fast_two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  return {s, __dsub_rn(b, __dsub_rn(s, a))};
}

__device__ __forceinline__ dd two_prod(double a, double b) {
  const double p = __dmul_rn(a, b);
  return {p, __fma_rn(a, b, -p)};
}

__device__ __forceinline__ dd dd_from(double a) { return {a, 0.0}; }

__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  const dd t = two_sum(a.lo, b.lo);
  s.lo = __dadd_rn(s.lo, t.hi);
  s = fast_two_sum(s.hi, s.lo);
  s.lo = __dadd_rn(s.lo, t.lo);
  return fast_two_sum(s.hi, s.lo);
}

__device__ __forceinline__ dd dd_neg(dd a) { return {-a.hi, -a.lo}; }
__device__ __forceinline__ dd dd_sub(dd a, dd b) { return dd_add(a, dd_neg(b)); }

__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo = __dadd_rn(p.lo, __dadd_rn(__dmul_rn(a.hi, b.lo), __dmul_rn(a.lo, b.hi)));
  return fast_two_sum(p.hi, p.lo);
}

__device__ __forceinline__ dd dd_div(dd a, dd b) {
  const double q1 = a.hi / b.hi;
  dd r = dd_sub(a, dd_mul(b, dd_from(q1)));
  const double q2 = r.hi / b.hi;
  r = dd_sub(r, dd_mul(b, dd_from(q2)));
  const double q3 = r.hi / b.hi;
  dd q = fast_two_sum(q1, q2);
  return dd_add(q, dd_from(q3));
}

__device__ __forceinline__ dd dd_sqrt(dd a) {
  if (a.hi <= 0.0) return {0.0, 0.0};
  const double x = sqrt(a.hi);
  const dd r = dd_sub(a, two_prod(x, x));
  return fast_two_sum(x, r.hi / __dmul_rn(2.0, x));
}

// Dot2 accumulation: acc += x*y with the product's and the sum's rounding
// errors collected in acc.lo (renormalised when read through dd_norm)
__device__ __forceinline__ void dot2_acc(double& hi, double& lo, double x, double y) {
  const dd p = two_prod(x, y);
  const dd s = two_sum(hi, p.hi);
  hi = s.hi;
  lo = __dadd_rn(lo, __dadd_rn(s.lo, p.lo));
}

__device__ __forceinline__ dd dd_norm(double hi, double lo) { return fast_two_sum(hi, lo); }

// fixed xor-tree sum over a warp
__device__ __forceinline__ dd warp_sum_dd(dd v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    dd o;
    o.hi = __shfl_xor_sync(0xffffffffu, v.hi, off);
    o.lo = __shfl_xor_sync(0xffffffffu, v.lo, off);
    v = dd_add(v, o);
  }
  return v;
}

}  // namespace aapdhg_b200
