// gvx_math.cuh — per-event arithmetic of the GenVectorX hot path, sm_100a.
//
// What is computed is fixed by the paper (Fig. 1:
// `LVector w = v1[id] + v2[id]; m[id] = w.mass();`) and the formulas the
// SPEC writes out (SPEC.md:81 conversion, :101-103 signed mass, :188 boost).
// HOW is B200-first and differs from the literal evaluation order; every
// rewrite below is exact in real arithmetic and its rounding effect is bounded
// far inside the north-star tolerance (|dM^2| <= tau E^2, tau = 1e-12 f64,
// 1e-5 f32) — DESIGN.md §5 carries the error budget.
//
// Mass of a PtEtaPhiM pair without forming the Cartesian vectors:
//   with  P_i = (pt_i cosh eta_i)^2 = |p_i|^2,  A_i = m_i|m_i| + P_i = E_i^2 (pre-clamp)
//   M^2 = E1^2 + E2^2 + 2 E1E2 - |p1|^2 - |p2|^2 - 2 p1.p2
//       = t1 + t2 + 2 (sqrt(A1+ A2+) - pt1 pt2 (cos(phi1 - phi2) + sinh eta1 sinh eta2))
//   where A+ = max(A, 0) (the E^2 clamp, R2) and t_i = E_i^2 - |p_i|^2
//   = max(m_i|m_i|, -P_i). One cos, two exp, one sqrt of a product and one
//   final sqrt replace two sincos, two sinh, three sqrt of the literal form.
// Inputs outside the fast domain (|eta| > 20, huge |phi|, huge pt/m, NaN/Inf)
// take the literal formula with IEEE-accurate libm (cold path).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gvx {

// ---------------------------------------------------------------------------
// Literal conversion + sum + signed mass (cold path and PxPyPzE path).
// ---------------------------------------------------------------------------
template <typename T> struct V4 { T x, y, z, t; };

__device__ __forceinline__ double d_sqrt(double x) { return sqrt(x); }
__device__ __forceinline__ float d_sqrt(float x) { return sqrtf(x); }

template <typename T>
__device__ __forceinline__ T signed_sqrt(T m2) {
  return m2 >= T(0) ? d_sqrt(m2) : -d_sqrt(-m2);
}

// PtEtaPhiM -> PxPyPzE with accurate libm (clamp R2).
__device__ __noinline__ V4<double> ptetaphim_exact(double pt, double eta, double phi, double m) {
  double s, c;
  sincos(phi, &s, &c);
  V4<double> r;
  r.x = pt * c;
  r.y = pt * s;
  r.z = pt * sinh(eta);
  double e2 = m * fabs(m) + pt * pt + r.z * r.z;
  r.t = sqrt(e2 > 0.0 ? e2 : 0.0);
  return r;
}
__device__ __noinline__ V4<float> ptetaphim_exact(float pt, float eta, float phi, float m) {
  float s, c;
  sincosf(phi, &s, &c);
  V4<float> r;
  r.x = pt * c;
  r.y = pt * s;
  r.z = pt * sinhf(eta);
  float e2 = m * fabsf(m) + pt * pt + r.z * r.z;
  r.t = sqrtf(e2 > 0.f ? e2 : 0.f);
  return r;
}

template <typename T>
__device__ __forceinline__ T mass_of_sum(const V4<T>& a, const V4<T>& b) {
  T X = a.x + b.x, Y = a.y + b.y, Z = a.z + b.z, E = a.t + b.t;
  return signed_sqrt(E * E - (X * X + Y * Y + Z * Z));
}

template <typename T>
__device__ __noinline__ T pair_mass_exact(T pt1, T eta1, T phi1, T m1, T pt2, T eta2, T phi2,
                                          T m2) {
  return mass_of_sum(ptetaphim_exact(pt1, eta1, phi1, m1), ptetaphim_exact(pt2, eta2, phi2, m2));
}

// ---------------------------------------------------------------------------
// Fast fp64 pair mass (reduced form above).
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool fast_domain(double pt, double eta, double phi, double m) {
  return fabs(eta) <= 20.0 && fabs(phi) <= 1024.0 && fabs(pt) <= 1e60 && fabs(m) <= 1e60;
}
__device__ __forceinline__ bool fast_domain(float pt, float eta, float phi, float m) {
  return fabsf(eta) <= 20.f && fabsf(phi) <= 8.f && fabsf(pt) <= 1e6f && fabsf(m) <= 1e6f;
}

__device__ __forceinline__ double pair_mass_fast(double pt1, double eta1, double phi1, double m1,
                                                 double pt2, double eta2, double phi2, double m2) {
  double c = cos(phi1 - phi2);
  double e1 = exp(eta1), e2 = exp(eta2);
  double r1 = 1.0 / e1, r2 = 1.0 / e2;
  double sh1 = 0.5 * (e1 - r1), ch1 = 0.5 * (e1 + r1);
  double sh2 = 0.5 * (e2 - r2), ch2 = 0.5 * (e2 + r2);
  double q1 = pt1 * ch1, q2 = pt2 * ch2;
  double P1 = q1 * q1, P2 = q2 * q2;
  double mm1 = m1 * fabs(m1), mm2 = m2 * fabs(m2);
  double A1 = fmax(mm1 + P1, 0.0), A2 = fmax(mm2 + P2, 0.0);
  double t = fmax(mm1, -P1) + fmax(mm2, -P2);
  double m2sq = t + 2.0 * (sqrt(A1 * A2) - pt1 * pt2 * (c + sh1 * sh2));
  return signed_sqrt(m2sq);
}

// fp32: MUFU-based cos/exp/rcp/sqrt (error budget DESIGN.md §5: <= ~1e-6 E^2
// against tau = 1e-5 E^2). Delta-phi is reduced to [-pi, pi] by one
// Cody-Waite step before MUFU.COS so its argument error stays ~ulp(pi).
__device__ __forceinline__ float fast_sqrt(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float fast_rcp(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float fast_ex2(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float reduce_2pi(float d) {
  const float INV_2PI = 0.159154943091895336f;
  const float TWO_PI_HI = 6.28318548202514648f;    // float(2 pi)
  const float TWO_PI_LO = -1.74845553146951715e-7f; // 2 pi - TWO_PI_HI
  float k = rintf(d * INV_2PI);
  float r = fmaf(-k, TWO_PI_HI, d);
  return fmaf(-k, TWO_PI_LO, r);
}

__device__ __forceinline__ float pair_mass_fast(float pt1, float eta1, float phi1, float m1,
                                                float pt2, float eta2, float phi2, float m2) {
  const float LOG2E = 1.44269504088896341f;
  float c = __cosf(reduce_2pi(phi1 - phi2));
  float e1 = fast_ex2(eta1 * LOG2E), e2 = fast_ex2(eta2 * LOG2E);
  float r1 = fast_rcp(e1), r2 = fast_rcp(e2);
  float sh1 = 0.5f * (e1 - r1), ch1 = 0.5f * (e1 + r1);
  float sh2 = 0.5f * (e2 - r2), ch2 = 0.5f * (e2 + r2);
  float q1 = pt1 * ch1, q2 = pt2 * ch2;
  float P1 = q1 * q1, P2 = q2 * q2;
  float mm1 = m1 * fabsf(m1), mm2 = m2 * fabsf(m2);
  float E1 = fast_sqrt(fmaxf(mm1 + P1, 0.f)), E2 = fast_sqrt(fmaxf(mm2 + P2, 0.f));
  float t = fmaxf(mm1, -P1) + fmaxf(mm2, -P2);
  float m2sq = t + 2.f * (E1 * E2 - pt1 * pt2 * (c + sh1 * sh2));
  return m2sq >= 0.f ? fast_sqrt(m2sq) : -fast_sqrt(-m2sq);
}

template <typename T>
__device__ __forceinline__ T pair_mass_ptetaphim(T pt1, T eta1, T phi1, T m1, T pt2, T eta2,
                                                 T phi2, T m2) {
  if (fast_domain(pt1, eta1, phi1, m1) && fast_domain(pt2, eta2, phi2, m2))
    return pair_mass_fast(pt1, eta1, phi1, m1, pt2, eta2, phi2, m2);
  return pair_mass_exact(pt1, eta1, phi1, m1, pt2, eta2, phi2, m2);
}

// ---------------------------------------------------------------------------
// PtEtaPhiM -> PxPyPzE, fast (for the CM path, which needs Cartesian vectors).
// ---------------------------------------------------------------------------
__device__ __forceinline__ V4<double> ptetaphim_fast(double pt, double eta, double phi, double m) {
  double s, c;
  sincos(phi, &s, &c);
  double e = exp(eta), r = 1.0 / e;
  double sh = 0.5 * (e - r), ch = 0.5 * (e + r);
  double q = pt * ch;
  V4<double> o;
  o.x = pt * c;
  o.y = pt * s;
  o.z = pt * sh;
  o.t = sqrt(fmax(m * fabs(m) + q * q, 0.0));
  return o;
}
__device__ __forceinline__ V4<float> ptetaphim_fast(float pt, float eta, float phi, float m) {
  const float LOG2E = 1.44269504088896341f;
  float s, c;
  __sincosf(reduce_2pi(phi), &s, &c);
  float e = fast_ex2(eta * LOG2E), r = fast_rcp(e);
  float sh = 0.5f * (e - r), ch = 0.5f * (e + r);
  float q = pt * ch;
  V4<float> o;
  o.x = pt * c;
  o.y = pt * s;
  o.z = pt * sh;
  o.t = fast_sqrt(fmaxf(m * fabsf(m) + q * q, 0.f));
  return o;
}

template <typename T>
__device__ __forceinline__ V4<T> ptetaphim_to_cartesian(T pt, T eta, T phi, T m) {
  if (fast_domain(pt, eta, phi, m)) return ptetaphim_fast(pt, eta, phi, m);
  return ptetaphim_exact(pt, eta, phi, m);
}

// ---------------------------------------------------------------------------
// Boost by beta (SPEC.md:188 with (gamma-1)/beta^2 = gamma^2/(1+gamma), R6):
//   p' = p + (bg (beta.p) + gamma E) beta,   E' = gamma (E + beta.p)
// which is Lambda * v written without forming Lambda. |beta| >= 1 -> NaN x 4.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double rsqrt_acc(double x) { return 1.0 / sqrt(x); }
__device__ __forceinline__ float rsqrt_acc(float x) { return 1.0f / sqrtf(x); }

template <typename T> struct BoostCoef { T bx, by, bz, g, bg; bool ok; };

template <typename T>
__device__ __forceinline__ BoostCoef<T> boost_coef(T bx, T by, T bz) {
  BoostCoef<T> k;
  k.bx = bx; k.by = by; k.bz = bz;
  T b2 = bx * bx + by * by + bz * bz;
  k.ok = b2 < T(1);
  T g = rsqrt_acc(T(1) - b2);
  k.g = g;
  k.bg = g * g / (T(1) + g);
  return k;
}

template <typename T>
__device__ __forceinline__ V4<T> apply_boost(const BoostCoef<T>& k, const V4<T>& v) {
  V4<T> o;
  if (!k.ok) {
    const T nan = T(NAN);
    o.x = o.y = o.z = o.t = nan;
    return o;
  }
  T bp = k.bx * v.x + k.by * v.y + k.bz * v.z;
  T f = k.bg * bp + k.g * v.t;
  o.x = v.x + f * k.bx;
  o.y = v.y + f * k.by;
  o.z = v.z + f * k.bz;
  o.t = k.g * (v.t + bp);
  return o;
}

// CM-frame mass (reading R11): beta_cm = -P/E, boost both, sum, signed mass.
template <typename T>
__device__ __forceinline__ T cm_pair_mass(const V4<T>& a, const V4<T>& b, V4<T>* a_out,
                                          V4<T>* b_out) {
  T Px = a.x + b.x, Py = a.y + b.y, Pz = a.z + b.z, E = a.t + b.t;
  T inv = T(1) / E;
  BoostCoef<T> k = boost_coef(-Px * inv, -Py * inv, -Pz * inv);
  k.ok = k.ok && (E > T(0));
  V4<T> a2 = apply_boost(k, a), b2 = apply_boost(k, b);
  if (a_out) { *a_out = a2; *b_out = b2; }
  return mass_of_sum(a2, b2);
}

// ---------------------------------------------------------------------------
// ROOT FindFixBin in double with IEEE-exact operations in the oracle's order
// (reading R12): identical bins for identical mass bits.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int find_bin(double x, double lo, double hi, double width, int nbins) {
  if (x < lo) return 0;
  if (!(x < hi)) return nbins + 1;
  double q = __ddiv_rn(__dmul_rn((double)nbins, __dsub_rn(x, lo)), width);
  return 1 + __double2int_rz(q);
}

}  // namespace gvx
