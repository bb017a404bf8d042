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
//
// The fp64 transcendentals are B200-specific: the FP64 pipe (64 lanes/SM/clk,
// measured 35.7 TFLOP/s) is the second roofline of the fp64 kernels, so
// cos/sin/exp are short near-minimax polynomials after a 2-FMA Cody-Waite reduction
// (relative error <= ~2e-16 on the fast domain), sinh AND cosh come from ONE
// even/odd split exp evaluation (e^r = E(r^2) + r O(r^2), e^-r = E - r O), and
// reciprocals / square roots are MUFU.RCP64H / MUFU.RSQ64H seeds + Newton
// (<= 2 ulp) instead of IEEE-exact division / sqrt. Inputs outside the fast
// domain (|eta| > 20, |phi| > 1024, huge pt/m, NaN/Inf) take the literal
// formula with IEEE-accurate libm (cold path, noinline).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

namespace gvx {

template <typename T> struct V4 { T x, y, z, t; };

// ---------------------------------------------------------------------------
// fp64 building blocks
//
// Polynomial coefficients live in __constant__ memory so every DFMA takes its
// coefficient straight from the constant bank (c[0x3][...]) — 64-bit
// immediates would otherwise cost two UMOVs per use and the fp64 kernels are
// issue-bound as much as FP64-bound.
// ---------------------------------------------------------------------------
enum : int {
  K_EXP_QE = 0,   // 4: cosh(r) = 1 + s(1/2 + s QE(s)), s = r^2, |r| <= ln2/2 (highest first)
  K_EXP_QO = 4,   // 4: sinh(r)/r = 1 + s(1/6 + s QO(s))
  K_SIN = 8,      // 6: sin r = r - r^3 P(z), z = r^2, |r| <= pi/4
  K_COSQ = 14,    // 5: cos r = 1 + z(-1/2 + z Q(z)), |r| <= pi/4
  K_COSH = 19,    // 9: cos r = C(z), |r| <= pi/2 (degree 16)
  K_LOG2E = 28, K_LN2_HI, K_LN2_LO, K_INV_PI, K_PI_HI, K_PI_LO, K_2_PI, K_PIO2_HI, K_PIO2_LO,
  K_NCOEF
};
// Near-minimax coefficients (Chebyshev fits in 50-digit mpmath, rounded to
// double). Max abs error with these doubles on the stated ranges:
// cosh/sinh 2.2e-16 rel, sin 1.1e-16, cos(pi/4) 6.7e-16, cos(pi/2) 1.9e-16
// (tests/test_fastmath_cpu.py re-derives these bounds from this table).
__constant__ double kCoef[K_NCOEF] = {
    2.760751626492711e-07, 2.4801549607706326e-05, 0.0013888888897944966, 0.041666666666663264,      // QE
    2.5090716821297755e-08, 2.755729023328528e-06, 0.00019841269848234848, 0.008333333333333071,    // QO
    -1.5918129294866608e-10, 2.5051131845003624e-08, -2.755731610255244e-06, 0.00019841269836758574,
    -0.008333333333330948, 0.16666666666666666,                                                     // SIN
    2.0700600483433117e-09, -2.7556369695573007e-07, 2.4801585210990515e-05, -0.0013888888887277342,
    0.04166666666666468,                                                                            // COSQ
    4.608977003001797e-14, -1.1462901901757276e-11, 2.0876561839933163e-09, -2.755731639102575e-07,
    2.4801587277414926e-05, -0.001388888888877299, 0.04166666666666388, -0.4999999999999997, 1.0,   // COSH
    // reduction constants
    1.4426950408889634,          // log2(e)
    6.93147180369123816490e-01,  // LN2_HI = 0x3FE62E42FEE00000 (32 bits: k*LN2_HI exact)
    1.90821492927058770002e-10,  // LN2_LO = ln2 - LN2_HI
    0.3183098861837907,          // 1/pi
    3.141592653589793,           // PI_HI = double(pi)
    1.2246467991473532e-16,      // PI_LO = pi - PI_HI
    6.36619772367581382433e-01,  // 2/pi
    1.57079632679489655800e+00,  // PIO2_HI = double(pi/2)
    6.12323399573676603587e-17   // PIO2_LO = pi/2 - PIO2_HI
};

__device__ __forceinline__ double rcp_seed(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
__device__ __forceinline__ double rsqrt_seed(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
// 1/x for normal x: MUFU.RCP64H seed (relative error e0 ~ 2^-22) refined by
// one third-order step y(1 + e + e^2), e = 1 - x y (error ~ e0^3 < 2^-64).
__device__ __forceinline__ double fast_rcp(double x) {
  double y = rcp_seed(x);
  double e = fma(-x, y, 1.0);
  return fma(y, fma(e, e, e), y);
}
// 1/sqrt(x), x > 0 normal: MUFU.RSQ64H seed refined by one third-order step
// y(1 + e/2 + 3e^2/8), e = 1 - x y^2 (error ~ (5/16) e0^3 < 2^-64).
__device__ __forceinline__ double fast_rsqrt(double x) {
  double y = rsqrt_seed(x);
  double e = fma(-x * y, y, 1.0);
  return fma(y * e, fma(e, 0.375, 0.5), y);
}
// sqrt(x), <= 3 ulp: x * rsqrt(x). x below the smallest normal (zero,
// denormal) or negative -> +0 (the E^2 clamp of reading R2 comes for free);
// the test is an integer compare of the high word (ALU pipe), not a DSETP on
// the FP64 pipe, which bounds the fp64 kernels. For finite x only (a NaN
// with the sign bit set would give 0): the fast domain produces no NaN here.
__device__ __forceinline__ double fast_sqrt(double x) {
  double s = x * fast_rsqrt(x);
  return __double2hiint(x) < 0x00100000 ? 0.0 : s;
}
// sqrt(|x|) for any x: NaN -> NaN whatever its sign bit (the FP64 units
// return a NaN with the sign bit set, so the test is on |x|'s bits, not on
// the result of a DADD-implemented fabs), |x| below the smallest normal -> 0.
__device__ __forceinline__ uint32_t abs_hi(double x) { return (uint32_t)__double2hiint(x) & 0x7fffffffu; }
__device__ __forceinline__ double fast_sqrt_abs(double x) {
  double ax = fabs(x);
  double s = ax * fast_rsqrt(ax);
  return abs_hi(x) < 0x00100000u ? 0.0 : s;
}
// sign(m2) * sqrt(|m2|) with the sign bit copied by an integer OR (m2 = -0
// gives -0, as the oracle's sqrt(-0) does).
__device__ __forceinline__ double copy_sign_bit(double r, double m2) {
  return __hiloint2double(__double2hiint(r) | (__double2hiint(m2) & (int)0x80000000), __double2loint(r));
}

// Exact power of two 2^k for |k| < 1000 (integer ops only).
__device__ __forceinline__ double pow2i(int k) { return __hiloint2double((k + 1023) << 20, 0); }

// x * 2^k for normal x and a result that stays normal (integer add on the
// exponent field of the high word).
__device__ __forceinline__ double add_exponent(double x, int k) {
  return __hiloint2double(__double2hiint(x) + (k << 20), __double2loint(x));
}

// Round to nearest integer with the 1.5*2^52 shifter, valid for |v| < 2^51:
// the integer lands in the low word of v + MAGIC. Replaces FRND.F64 and
// F2I.F64, which run on the narrow XU pipe (ncu showed it oversubscribed).
// (Folding the product into one DFMA, fma(x, c, MAGIC), saves a DP op per call
// but costs registers: MAGIC then needs a register pair. Measured in round 2:
// the SoA f64 mass kernel went 128 -> 133 registers, one CTA per SM, 1.07 ->
// 1.37 ms; so the multiply stays separate.)
__device__ __forceinline__ double rint_shift(double v, int& ki) {
  const double MAGIC = 6755399441055744.0;  // 1.5 * 2^52
  double t = __dadd_rn(v, MAGIC);
  ki = __double2loint(t);
  return __dsub_rn(t, MAGIC);
}

// sinh and cosh of x, |x| <= 20: x = k ln2 + r, |r| <= ln2/2;
// e^r = E + O, e^-r = E - O with E = sum r^2j/(2j)!, O = r sum r^2j/(2j+1)!
// (near-minimax degree 10 / 11: error <= 2.2e-16 relative).
__device__ __forceinline__ void sinh_cosh(double x, double& sh, double& ch) {
  int ki;
  double k = rint_shift(x * kCoef[K_LOG2E], ki);
  double r = fma(-k, kCoef[K_LN2_HI], x);
  r = fma(-k, kCoef[K_LN2_LO], r);
  double s = r * r;
  double qe = fma(s, kCoef[K_EXP_QE + 0], kCoef[K_EXP_QE + 1]);
  qe = fma(s, qe, kCoef[K_EXP_QE + 2]);
  qe = fma(s, qe, kCoef[K_EXP_QE + 3]);
  double E = fma(s, fma(s, qe, 0.5), 1.0);
  double qo = fma(s, kCoef[K_EXP_QO + 0], kCoef[K_EXP_QO + 1]);
  qo = fma(s, qo, kCoef[K_EXP_QO + 2]);
  qo = fma(s, qo, kCoef[K_EXP_QO + 3]);
  double O = fma(s, fma(s, qo, 0.16666666666666666), 1.0) * r;
  // (E +- O) * 2^(+-k-1) by adding to the exponent field (exact: E +- O is in
  // [0.7, 1.5], |k| <= 29) — an integer add instead of building 2^k and a DMUL.
  double ep = add_exponent(E + O, ki - 1), em = add_exponent(E - O, -ki - 1);
  sh = ep - em;
  ch = ep + em;
}

// sin and cos of r, |r| <= pi/4 (near-minimax, degree 13 / 12).
__device__ __forceinline__ void sincos_poly(double r, double& s, double& c) {
  double z = r * r;
  double ps = fma(z, kCoef[K_SIN + 0], kCoef[K_SIN + 1]);
#pragma unroll
  for (int j = 2; j < 6; ++j) ps = fma(z, ps, kCoef[K_SIN + j]);
  s = fma(-r * z, ps, r);  // r - r^3 P(z)
  double pc = fma(z, kCoef[K_COSQ + 0], kCoef[K_COSQ + 1]);
#pragma unroll
  for (int j = 2; j < 5; ++j) pc = fma(z, pc, kCoef[K_COSQ + j]);
  c = fma(z, fma(z, pc, -0.5), 1.0);
}

// Flip the sign of x when bit 0 of q is set (integer op on the high word).
__device__ __forceinline__ double neg_if(double x, int q) {
  return __hiloint2double(__double2hiint(x) ^ ((q & 1) << 31), __double2loint(x));
}

// sin and cos of x, |x| <= 2048: x = k pi/2 + r, |r| <= pi/4 (+ulp).
__device__ __forceinline__ void fast_sincos(double x, double& sn, double& cs) {
  int q;
  double k = rint_shift(x * kCoef[K_2_PI], q);
  double r = fma(-k, kCoef[K_PIO2_HI], x);  // exact for |k| < 2^11
  r = fma(-k, kCoef[K_PIO2_LO], r);
  double s, c;
  sincos_poly(r, s, c);
  // sin x = [s, c, -s, -c][q & 3], cos x = [c, -s, -c, s][q & 3]
  double ss = (q & 1) ? c : s;
  double cc = (q & 1) ? s : c;
  sn = neg_if(ss, q >> 1);
  cs = neg_if(cc, (q + 1) >> 1);
}

// cos x, |x| <= 2048: x = k pi + r, |r| <= pi/2, cos x = (-1)^k cos r with a
// degree-16 even near-minimax polynomial — no quadrant selects.
__device__ __forceinline__ double fast_cos(double x) {
  int ki;
  double k = rint_shift(x * kCoef[K_INV_PI], ki);
  double r = fma(-k, kCoef[K_PI_HI], x);  // exact for |k| < 2^10
  r = fma(-k, kCoef[K_PI_LO], r);
  double z = r * r;
  double c = fma(z, kCoef[K_COSH + 0], kCoef[K_COSH + 1]);
#pragma unroll
  for (int j = 2; j < 9; ++j) c = fma(z, c, kCoef[K_COSH + j]);
  return neg_if(c, ki);
}

// ---------------------------------------------------------------------------
// Literal conversion + sum + signed mass (cold path and PxPyPzE path).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double ieee_sqrt(double x) { return sqrt(x); }
__device__ __forceinline__ float ieee_sqrt(float x) { return sqrtf(x); }

template <typename T>
__device__ __forceinline__ T signed_sqrt(T m2) {
  return m2 >= T(0) ? ieee_sqrt(m2) : -ieee_sqrt(-m2);
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
__device__ __noinline__ T pair_mass_exact(T pt1, T eta1, T phi1, T m1, T pt2, T eta2, T phi2, T m2) {
  return mass_of_sum(ptetaphim_exact(pt1, eta1, phi1, m1), ptetaphim_exact(pt2, eta2, phi2, m2));
}

// ---------------------------------------------------------------------------
// Fast domain and fast pair mass.
// ---------------------------------------------------------------------------
// Fast domain, tested on the high words with integer compares (ALU pipe):
// |eta| < 20, |phi| < 1024, 2^-200 <= |pt| < 2^200, |m| < 2^200; NaN/Inf fail
// every test. The lower bound on pt keeps every square normal (pt = 0 and
// denormal-scale vectors take the literal cold path).
__device__ __forceinline__ bool fast_domain(double pt, double eta, double phi, double m) {
  return (abs_hi(eta) < 0x40340000u) & (abs_hi(phi) < 0x40900000u) &
         (abs_hi(pt) - 0x33700000u < 0x4C700000u - 0x33700000u) & (abs_hi(m) < 0x4C700000u);
}
// f32: |eta| < 20, |phi| < 8, 2^-40 <= |pt| < 2^20, |m| < 2^20 (the MUFU
// sqrt flushes denormals, so pt^2 must stay normal).
__device__ __forceinline__ uint32_t abs_bits(float x) { return (uint32_t)__float_as_int(x) & 0x7fffffffu; }
__device__ __forceinline__ bool fast_domain(float pt, float eta, float phi, float m) {
  return (abs_bits(eta) < 0x41A00000u) & (abs_bits(phi) < 0x41000000u) &
         (abs_bits(pt) - 0x2B800000u < 0x49800000u - 0x2B800000u) & (abs_bits(m) < 0x49800000u);
}

// E = sqrt(max(0, (pt cosh eta)^2 + m|m|)) of a PtEtaPhiM vector from q = pt cosh eta
// (the R2 clamp comes from fast_sqrt / pos_sqrt) — one expression shared by the lab
// and the CM mass, so the fused pass evaluates it once per vector.
template <typename T>
__device__ __forceinline__ T energy_of(T m, T q);

// The lab pair mass from its transcendentals and energies (c = cos(phi1 - phi2),
// sinh of both etas, q = pt cosh eta, E from energy_of) — shared by pair_mass_fast
// and the fused lab + CM pass:
//   M^2 = t1 + t2 + 2 (E1 E2 - pt1 pt2 (c + sh1 sh2)),  t = m|m| (E^2 - |p|^2),
// or t = -q^2 for a clamped vector (E^2 < 0 -> E = 0, reading R2).
__device__ __forceinline__ double pair_mass_from(double pt1, double m1, double pt2, double m2, double c, double sh1,
                                                 double sh2, double q1, double q2, double E1, double E2) {
  double mm1 = m1 * fabs(m1), mm2 = m2 * fabs(m2);
  // clamp test on the sign bit of E^2 (integer op; E^2 = -0 is impossible: q >= pt > 0)
  bool c1 = __double2hiint(fma(q1, q1, mm1)) < 0, c2 = __double2hiint(fma(q2, q2, mm2)) < 0;
  double t = (c1 ? -(q1 * q1) : mm1) + (c2 ? -(q2 * q2) : mm2);
  double m2sq = t + 2.0 * (E1 * E2 - pt1 * pt2 * (c + sh1 * sh2));
  return copy_sign_bit(fast_sqrt_abs(m2sq), m2sq);
}

__device__ __forceinline__ double pair_mass_fast(double pt1, double eta1, double phi1, double m1, double pt2,
                                                 double eta2, double phi2, double m2) {
  // cos(phi1 - phi2) is taken from the same sincos(phi2 - phi1) the CM mass
  // uses, so the fused lab + CM pass evaluates one trigonometric reduction.
  double sd, c;
  fast_sincos(phi2 - phi1, sd, c);
  double sh1, ch1, sh2, ch2;
  sinh_cosh(eta1, sh1, ch1);
  sinh_cosh(eta2, sh2, ch2);
  double q1 = pt1 * ch1, q2 = pt2 * ch2;
  return pair_mass_from(pt1, m1, pt2, m2, c, sh1, sh2, q1, q2, energy_of(m1, q1), energy_of(m2, q2));
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
  const float TWO_PI_HI = 6.28318548202514648f;     // float(2 pi)
  const float TWO_PI_LO = -1.74845553146951715e-7f;  // 2 pi - TWO_PI_HI
  float k = rintf(d * INV_2PI);
  float r = fmaf(-k, TWO_PI_HI, d);
  return fmaf(-k, TWO_PI_LO, r);
}

template <typename V>
__device__ __forceinline__ V pair_mass_f32_lanes(V pt1, V eta1, V phi1, V m1, V pt2, V eta2, V phi2, V m2);

// fp32 lab mass: the lane-generic form (pair_mass_f32_lanes, defined with the
// lane helpers below) so the packed two-event path of the TMA kernels gives
// the same bits as this scalar one.
__device__ __forceinline__ float pair_mass_fast(float pt1, float eta1, float phi1, float m1, float pt2, float eta2,
                                                float phi2, float m2) {
  return pair_mass_f32_lanes<float>(pt1, eta1, phi1, m1, pt2, eta2, phi2, m2);
}

template <typename T>
__device__ __forceinline__ T pair_mass_ptetaphim(T pt1, T eta1, T phi1, T m1, T pt2, T eta2, T phi2, T m2) {
  if (fast_domain(pt1, eta1, phi1, m1) && fast_domain(pt2, eta2, phi2, m2))
    return pair_mass_fast(pt1, eta1, phi1, m1, pt2, eta2, phi2, m2);
  return pair_mass_exact(pt1, eta1, phi1, m1, pt2, eta2, phi2, m2);
}

// ---------------------------------------------------------------------------
// PtEtaPhiM -> PxPyPzE, fast (for the CM path, which needs Cartesian vectors).
// ---------------------------------------------------------------------------
__device__ __forceinline__ V4<double> ptetaphim_fast(double pt, double eta, double phi, double m) {
  double s, c, sh, ch;
  fast_sincos(phi, s, c);
  sinh_cosh(eta, sh, ch);
  double q = pt * ch;
  V4<double> o;
  o.x = pt * c;
  o.y = pt * s;
  o.z = pt * sh;
  o.t = fast_sqrt(fma(m, fabs(m), q * q));  // negative E^2 -> 0 (R2)
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
template <typename T> struct BoostCoef { T bx, by, bz, g, bg; bool ok; };

// Accurate (IEEE div/sqrt) coefficients: the standalone boost kernel is
// HBM-bound with DP headroom, so it keeps correctly rounded gamma.
template <typename T>
__device__ __forceinline__ BoostCoef<T> boost_coef(T bx, T by, T bz) {
  BoostCoef<T> k;
  k.bx = bx; k.by = by; k.bz = bz;
  // explicit fma order: the same bits in every kernel that inlines this (the
  // one-launch step must match the standalone boost bit for bit)
  T b2 = fma(bz, bz, fma(by, by, bx * bx));
  k.ok = b2 < T(1);
  T g = T(1) / ieee_sqrt(T(1) - b2);
  k.g = g;
  k.bg = g * g / (T(1) + g);
  return k;
}
// Fast coefficients (MUFU seeds + Newton, <= 2 ulp) for the CM histogram,
// whose fp64 variant is FP64-pipe bound.
// With u = 1 - beta^2: gamma = u^-1/2 and gamma^2/(1+gamma) = 1/(u + u gamma)
// (one reciprocal, no DMULs); beta^2 < 1 <=> u > 0, tested on u's high word
// (u >= 2^-53 whenever beta^2 < 1; NaN passes and propagates).
__device__ __forceinline__ BoostCoef<double> boost_coef_fast(double bx, double by, double bz) {
  BoostCoef<double> k;
  k.bx = bx; k.by = by; k.bz = bz;
  double u = 1.0 - (bx * bx + by * by + bz * bz);
  k.ok = __double2hiint(u) > 0;
  double g = fast_rsqrt(u);
  k.g = g;
  k.bg = fast_rcp(fma(u, g, u));
  return k;
}
__device__ __forceinline__ BoostCoef<float> boost_coef_fast(float bx, float by, float bz) {
  BoostCoef<float> k;
  k.bx = bx; k.by = by; k.bz = bz;
  float b2 = bx * bx + by * by + bz * bz;
  k.ok = b2 < 1.0f;
  float g;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(g) : "f"(1.0f - b2));
  k.g = g;
  k.bg = g * g * fast_rcp(1.0f + g);
  return k;
}

// Y0: v.y is exactly zero (the CM path's vector 1 in its rotated frame), so
// the y terms of the products are skipped (exact: adding a +-0 product to a
// sum changes at most the sign of a zero).
template <typename T, bool Y0 = false>
__device__ __forceinline__ V4<T> apply_boost(const BoostCoef<T>& k, const V4<T>& v) {
  V4<T> o;
  if (!k.ok) {
    const T nan = T(NAN);
    o.x = o.y = o.z = o.t = nan;
    return o;
  }
  // explicit fma order (context-independent bits, see boost_coef)
  T bp = Y0 ? fma(k.bz, v.z, k.bx * v.x) : fma(k.bz, v.z, fma(k.by, v.y, k.bx * v.x));
  T f = fma(k.bg, bp, k.g * v.t);
  o.x = fma(f, k.bx, v.x);
  o.y = Y0 ? f * k.by : fma(f, k.by, v.y);
  o.z = fma(f, k.bz, v.z);
  o.t = k.g * (v.t + bp);
  return o;
}

__device__ __forceinline__ double any_rcp(double x) { return fast_rcp(x); }
__device__ __forceinline__ float any_rcp(float x) { return fast_rcp(x); }

// Signed square root with the fast sqrt (fp64: MUFU.RSQ64H + Newton, <= 3 ulp).
__device__ __forceinline__ double fast_signed_sqrt(double m2) { return copy_sign_bit(fast_sqrt_abs(m2), m2); }
__device__ __forceinline__ float fast_signed_sqrt(float m2) {
  float r = fast_sqrt(fabsf(m2));
  return m2 >= 0.f ? r : -r;
}

// CM-frame mass (reading R11): beta_cm = -P/E, boost both, sum, signed mass.
// E <= 0 or beta^2 >= 1 (or NaN) -> gamma = NaN, so every output is NaN
// without a branch.
__device__ __forceinline__ bool is_positive(double x) { return __double2hiint(x) > 0; }  // x >= 2^-1022 (or +NaN)
__device__ __forceinline__ bool is_positive(float x) { return x > 0.f; }

// cos of the polar angle of v's momentum, p_z / |p| (reading R22); |p| = 0 -> NaN.
__device__ __forceinline__ double cos_polar(const V4<double>& v) {
  return v.z * fast_rsqrt(fma(v.x, v.x, fma(v.y, v.y, v.z * v.z)));
}
__device__ __forceinline__ float cos_polar(const V4<float>& v) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(fmaf(v.x, v.x, fmaf(v.y, v.y, v.z * v.z))));
  return v.z * r;
}

// WANT_COS: also cos theta* of boosted vector 1 (reading R22). The rotated
// frame of cm_mass_ptetaphim_fast turns about z, which leaves p_z and |p|
// unchanged, so cos theta* is read before any rotation back.
template <typename T, bool A_Y0 = false, bool WANT_COS = false>
__device__ __forceinline__ T cm_pair_mass(const V4<T>& a, const V4<T>& b, V4<T>* a_out, V4<T>* b_out,
                                          T* cos_out = nullptr) {
  // A_Y0: a.y is exactly zero, so P_y = b.y (0 + b.y differs at most in the sign of a zero)
  T Px = a.x + b.x, Py = A_Y0 ? b.y : a.y + b.y, Pz = a.z + b.z, E = a.t + b.t;
  T inv = any_rcp(E);
  BoostCoef<T> k;
  if constexpr (sizeof(T) == 8) {
    // boost_coef_fast's arithmetic with the validity folded into u = 1 - beta^2: E <= 0 (or
    // -NaN) selects a NaN u, and beta^2 >= 1 gives u <= 0, whose MUFU.RSQ64H seed is NaN
    // (-0 and flushed denormals give inf, whose refinement is NaN) — one double select
    // instead of a validity test and two (g, bg) selects; the same values, NaN -> NaN.
    k.bx = -Px * inv;
    k.by = -Py * inv;
    k.bz = -Pz * inv;
    double u = 1.0 - (k.bx * k.bx + k.by * k.by + k.bz * k.bz);
    u = is_positive(E) ? u : __longlong_as_double(0x7ff8000000000000ll);
    k.g = fast_rsqrt(u);
    k.bg = fast_rcp(fma(u, k.g, u));
  } else {
    k = boost_coef_fast(-Px * inv, -Py * inv, -Pz * inv);
    const bool ok = k.ok && is_positive(E);
    k.g = ok ? k.g : T(NAN);
    k.bg = ok ? k.bg : T(NAN);
  }
  k.ok = true;
  V4<T> a2 = apply_boost<T, A_Y0>(k, a), b2 = apply_boost(k, b);
  if (a_out) { *a_out = a2; *b_out = b2; }
  if constexpr (WANT_COS) *cos_out = cos_polar(a2);
  T X = a2.x + b2.x, Y = a2.y + b2.y, Z = a2.z + b2.z, W = a2.t + b2.t;
  return fast_signed_sqrt(W * W - (X * X + Y * Y + Z * Z));
}

// fp32 sincos / sinh+cosh with the same interface as the fp64 routines.
__device__ __forceinline__ void fast_sincos(float x, float& sn, float& cs) { __sincosf(reduce_2pi(x), &sn, &cs); }
__device__ __forceinline__ void sinh_cosh(float x, float& sh, float& ch) {
  const float LOG2E = 1.44269504088896341f;
  float e = fast_ex2(x * LOG2E), r = fast_rcp(e);
  sh = 0.5f * (e - r);
  ch = 0.5f * (e + r);
}
__device__ __forceinline__ double pos_sqrt(double x) { return fast_sqrt(x); }  // x < 0 -> 0
__device__ __forceinline__ float pos_sqrt(float x) { return fast_sqrt(x > 0.f ? x : 0.f); }

// CM-frame mass of a PtEtaPhiM pair (fast domain), computed in coordinates
// rotated about the z axis by -phi1. A rotation about z is a change of
// Cartesian axes: the CM boost is still built from beta_cm = -P/E and applied
// to both vectors literally, but vector 1 becomes (pt1, 0, pt1 sinh eta1, E1)
// and vector 2 needs only sin/cos of phi2 - phi1 — one sincos per pair instead
// of two. Boosted vectors, when requested, are rotated back by +phi1.
template <typename V, bool WANT_COS, bool WANT_VEC>
__device__ __forceinline__ V cm_mass_f32_lanes(V pt1, V eta1, V phi1, V m1, V pt2, V eta2, V phi2, V m2,
                                               V* cos_out, V* vec_out);

template <typename T>
__device__ __forceinline__ T energy_of(T m, T q) {
  return pos_sqrt(fma(q, q, m * fabs(m)));
}

// The CM mass in the rotated frame from its transcendentals (sd, cd = sin/cos of
// phi2 - phi1; sinh of both etas) and energies — shared with the fused lab + CM pass.
template <typename T, bool WANT_COS = false>
__device__ __forceinline__ T cm_mass_from(T pt1, T pt2, T sd, T cd, T sh1, T sh2, T E1, T E2, V4<T>* a_out,
                                          V4<T>* b_out, T* cos_out) {
  V4<T> a{pt1, T(0), pt1 * sh1, E1};
  V4<T> b{pt2 * cd, pt2 * sd, pt2 * sh2, E2};
  return cm_pair_mass<T, true, WANT_COS>(a, b, a_out, b_out, cos_out);
}

// Fused lab + CM masses of one fast-domain fp64 pair: sinh/cosh of both etas,
// the sincos of phi2 - phi1 and both energies are evaluated once; both results are
// bit-identical to pair_mass_fast and cm_mass_ptetaphim_fast.
__device__ __forceinline__ void both_masses_fast(double pt1, double eta1, double phi1, double m1, double pt2,
                                                 double eta2, double phi2, double m2, double& m_lab,
                                                 double& m_cm) {
  double sd, cd, sh1, ch1, sh2, ch2;
  fast_sincos(phi2 - phi1, sd, cd);
  sinh_cosh(eta1, sh1, ch1);
  sinh_cosh(eta2, sh2, ch2);
  const double q1 = pt1 * ch1, q2 = pt2 * ch2;
  const double E1 = energy_of(m1, q1), E2 = energy_of(m2, q2);
  m_lab = pair_mass_from(pt1, m1, pt2, m2, cd, sh1, sh2, q1, q2, E1, E2);
  m_cm = cm_mass_from<double, false>(pt1, pt2, sd, cd, sh1, sh2, E1, E2, nullptr, nullptr, nullptr);
}

template <typename T, bool WANT_COS = false>
__device__ __forceinline__ T cm_mass_ptetaphim_fast(T pt1, T eta1, T phi1, T m1, T pt2, T eta2, T phi2, T m2,
                                                    V4<T>* a_out, V4<T>* b_out, T* cos_out = nullptr) {
  if constexpr (sizeof(T) == 4) {  // fp32: the lane core (bit-identical to its packed two-event form)
    T M;
    if (a_out) {
      T v[8];
      M = cm_mass_f32_lanes<float, WANT_COS, true>(pt1, eta1, phi1, m1, pt2, eta2, phi2, m2, cos_out, v);
      *a_out = V4<T>{v[0], v[1], v[2], v[3]};
      *b_out = V4<T>{v[4], v[5], v[6], v[7]};
    } else {
      M = cm_mass_f32_lanes<float, WANT_COS, false>(pt1, eta1, phi1, m1, pt2, eta2, phi2, m2, cos_out, nullptr);
    }
    if (a_out) {
      T s1, c1;
      fast_sincos(phi1, s1, c1);
      V4<T>* v[2] = {a_out, b_out};
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        T x = v[i]->x, y = v[i]->y;
        v[i]->x = c1 * x - s1 * y;
        v[i]->y = s1 * x + c1 * y;
      }
    }
    return M;
  }
  T sd, cd, sh1, ch1, sh2, ch2;
  fast_sincos(phi2 - phi1, sd, cd);
  sinh_cosh(eta1, sh1, ch1);
  sinh_cosh(eta2, sh2, ch2);
  T q1 = pt1 * ch1, q2 = pt2 * ch2;
  T M = cm_mass_from<T, WANT_COS>(pt1, pt2, sd, cd, sh1, sh2, energy_of(m1, q1), energy_of(m2, q2), a_out, b_out,
                                  cos_out);
  if (a_out) {
    T s1, c1;
    fast_sincos(phi1, s1, c1);
    V4<T>* v[2] = {a_out, b_out};
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      T x = v[i]->x, y = v[i]->y;
      v[i]->x = c1 * x - s1 * y;
      v[i]->y = s1 * x + c1 * y;
    }
  }
  return M;
}

// ---------------------------------------------------------------------------
// fp32 CM mass written once over a "lane vector" V = float (one event) or
// float2 (two events in the packed FFMA2 / FMUL2 / FADD2 instructions of
// sm_100: half the FP32 issue slots of the issue-bound f32 CM kernels). Every
// FP32 operation is explicit (no compiler contraction), so the scalar and the
// packed instantiation produce the same bits for the same event; MUFU
// operations (ex2, rcp, rsqrt, sqrt, sin/cos) and compares act per lane.
// Same formulas and rotated frame as cm_mass_ptetaphim_fast (fast domain).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float lv_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float lv_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float lv_fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ float lv_splat(float, float x) { return x; }
// Packed ops as PTX. Note: ptxas still contracts a packed mul feeding a packed
// add into FFMA2 (measured: g*x + g*y became one FFMA2, 1 ulp off the scalar
// path for ~20 % of events), so cm_mass_f32_lanes writes every such sum as an
// explicit fma.
__device__ __forceinline__ float2 lv_mul(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 x, y, z;\n\tmov.b64 x, {%2, %3};\n\tmov.b64 y, {%4, %5};\n\t"
      "mul.rn.f32x2 z, x, y;\n\tmov.b64 {%0, %1}, z;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 lv_add(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 x, y, z;\n\tmov.b64 x, {%2, %3};\n\tmov.b64 y, {%4, %5};\n\t"
      "add.rn.f32x2 z, x, y;\n\tmov.b64 {%0, %1}, z;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 lv_fma(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 x, y, w, z;\n\tmov.b64 x, {%2, %3};\n\tmov.b64 y, {%4, %5};\n\tmov.b64 w, {%6, %7};\n\t"
      "fma.rn.f32x2 z, x, y, w;\n\tmov.b64 {%0, %1}, z;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 lv_splat(float2, float x) { return make_float2(x, x); }
// sign(v) sqrt(|v|) with ONE MUFU.SQRT and the sign bit copied by an integer op
// (v >= 0 ? sqrt(v) : -sqrt(-v) compiled to two predicated MUFUs and an FADD;
// same bits, -0 -> -0, NaN -> NaN).
__device__ __forceinline__ float sqrt_abs_signed(float v) {
  return __int_as_float(__float_as_int(fast_sqrt(fabsf(v))) | (__float_as_int(v) & (int)0x80000000));
}
template <typename F> __device__ __forceinline__ float lv_map(float a, F f) { return f(a); }
template <typename F> __device__ __forceinline__ float2 lv_map(float2 a, F f) { return make_float2(f(a.x), f(a.y)); }
template <typename F> __device__ __forceinline__ float lv_map2(float a, float b, F f) { return f(a, b); }
template <typename F> __device__ __forceinline__ float2 lv_map2(float2 a, float2 b, F f) {
  return make_float2(f(a.x, b.x), f(a.y, b.y));
}

// fp32 lab pair mass (reduced form of pair_mass_fast(double), MUFU functions):
//   M^2 = t1 + t2 + 2 (E1 E2 - pt1 pt2 (cos(phi1 - phi2) + sinh eta1 sinh eta2)),
// every product-feeding sum an explicit fma (see cm_mass_f32_lanes).
template <typename V>
__device__ __forceinline__ V pair_mass_f32_lanes(V pt1, V eta1, V phi1, V m1, V pt2, V eta2, V phi2, V m2) {
  const V MONE = lv_splat(V{}, -1.f), HALF = lv_splat(V{}, 0.5f), TWO = lv_splat(V{}, 2.f);
  const V LOG2E = lv_splat(V{}, 1.44269504088896341f);
  // cos(phi2 - phi1) = cos(phi1 - phi2), reduced exactly as cm_mass_f32_lanes
  // does, so the fused lab + CM pass shares the reduction and the MUFU.COS
  V d = lv_fma(phi1, MONE, phi2);
  V k = lv_map(lv_mul(d, lv_splat(V{}, 0.159154943091895336f)), [](float x) { return rintf(x); });
  V r = lv_fma(k, lv_splat(V{}, -6.28318548202514648f), d);
  r = lv_fma(k, lv_splat(V{}, 1.74845553146951715e-7f), r);
  V c = lv_map(r, [](float x) { return __cosf(x); });
  V e1 = lv_map(lv_mul(eta1, LOG2E), [](float x) { return fast_ex2(x); });
  V e2 = lv_map(lv_mul(eta2, LOG2E), [](float x) { return fast_ex2(x); });
  V r1 = lv_map(e1, [](float x) { return fast_rcp(x); }), r2 = lv_map(e2, [](float x) { return fast_rcp(x); });
  V sh1 = lv_mul(lv_fma(r1, MONE, e1), HALF), ch1 = lv_mul(lv_add(e1, r1), HALF);
  V sh2 = lv_mul(lv_fma(r2, MONE, e2), HALF), ch2 = lv_mul(lv_add(e2, r2), HALF);
  V q1 = lv_mul(pt1, ch1), q2 = lv_mul(pt2, ch2);
  V P1 = lv_mul(q1, q1), P2 = lv_mul(q2, q2);
  V mm1 = lv_mul(m1, lv_map(m1, [](float x) { return fabsf(x); }));
  V mm2 = lv_mul(m2, lv_map(m2, [](float x) { return fabsf(x); }));
  auto pos_sqrt_f = [](float x) { return fast_sqrt(x > 0.f ? x : 0.f); };
  V E1 = lv_map(lv_fma(q1, q1, mm1), pos_sqrt_f), E2 = lv_map(lv_fma(q2, q2, mm2), pos_sqrt_f);
  auto tclamp = [](float mm, float P) { return fmaxf(mm, -P); };  // E^2 - |p|^2 after the R2 clamp
  V t = lv_add(lv_map2(mm1, P1, tclamp), lv_map2(mm2, P2, tclamp));
  V inner = lv_fma(sh1, sh2, c);
  V y = lv_mul(lv_mul(pt1, pt2), inner);
  V x = lv_fma(E1, E2, lv_mul(y, MONE));
  V m2sq = lv_fma(x, TWO, t);
  return lv_map(m2sq, [](float v) { return sqrt_abs_signed(v); });
}

// vec_out (WANT_VEC): the boosted pair in the rotated frame, (a2x, a2y, a2z, a2t, b2x, b2y, b2z, b2t).
template <typename V, bool WANT_COS, bool WANT_VEC>
__device__ __forceinline__ V cm_mass_f32_lanes(V pt1, V eta1, V phi1, V m1, V pt2, V eta2, V phi2, V m2,
                                               V* cos_out, V* vec_out) {
  const V ONE = lv_splat(V{}, 1.f), MONE = lv_splat(V{}, -1.f), HALF = lv_splat(V{}, 0.5f);
  const V LOG2E = lv_splat(V{}, 1.44269504088896341f);
  // sin/cos of phi2 - phi1 after one Cody-Waite step to [-pi, pi] (as reduce_2pi)
  V d = lv_fma(phi1, MONE, phi2);
  V k = lv_map(lv_mul(d, lv_splat(V{}, 0.159154943091895336f)), [](float x) { return rintf(x); });
  V r = lv_fma(k, lv_splat(V{}, -6.28318548202514648f), d);
  r = lv_fma(k, lv_splat(V{}, 1.74845553146951715e-7f), r);
  V sd = lv_map(r, [](float x) { return __sinf(x); }), cd = lv_map(r, [](float x) { return __cosf(x); });
  // sinh/cosh from one ex2 and its reciprocal
  V e1 = lv_map(lv_mul(eta1, LOG2E), [](float x) { return fast_ex2(x); });
  V e2 = lv_map(lv_mul(eta2, LOG2E), [](float x) { return fast_ex2(x); });
  V r1 = lv_map(e1, [](float x) { return fast_rcp(x); }), r2 = lv_map(e2, [](float x) { return fast_rcp(x); });
  V sh1 = lv_mul(lv_fma(r1, MONE, e1), HALF), ch1 = lv_mul(lv_add(e1, r1), HALF);
  V sh2 = lv_mul(lv_fma(r2, MONE, e2), HALF), ch2 = lv_mul(lv_add(e2, r2), HALF);
  V q1 = lv_mul(pt1, ch1), q2 = lv_mul(pt2, ch2);
  auto pos_sqrt_f = [](float x) { return fast_sqrt(x > 0.f ? x : 0.f); };
  // vector 1 in the rotated frame: (pt1, 0, pt1 sh1, E1); vector 2: (pt2 cd, pt2 sd, pt2 sh2, E2)
  V ax = pt1, az = lv_mul(pt1, sh1);
  // E = sqrt(max(0, q^2 + m|m|)), the same expression as pair_mass_f32_lanes (shared in the fused pass)
  V aE = lv_map(lv_fma(q1, q1, lv_mul(m1, lv_map(m1, [](float x) { return fabsf(x); }))), pos_sqrt_f);
  V bx = lv_mul(pt2, cd), by = lv_mul(pt2, sd), bz = lv_mul(pt2, sh2);
  V bE = lv_map(lv_fma(q2, q2, lv_mul(m2, lv_map(m2, [](float x) { return fabsf(x); }))), pos_sqrt_f);
  // beta_cm = -P / E (P_y = b_y: vector 1 has no y component in this frame)
  // every sum whose operand is a product is an explicit fma: ptxas contracts
  // mul.rn.f32x2 + add.rn.f32x2 pairs (unlike the scalar .rn forms), which
  // would make the packed path differ from the scalar one by an ulp
  V Px = lv_fma(pt2, cd, ax), Pz = lv_fma(pt2, sh2, az), E = lv_add(aE, bE);
  V ninv = lv_map(E, [](float x) { return -fast_rcp(x); });
  V betx = lv_mul(Px, ninv), bety = lv_mul(by, ninv), betz = lv_mul(Pz, ninv);
  V u = lv_fma(lv_fma(betz, betz, lv_fma(bety, bety, lv_mul(betx, betx))), MONE, ONE);  // 1 - beta^2
  // gamma = u^-1/2, gamma^2/(1+gamma) = 1/(u + u gamma); invalid (E <= 0, beta^2 >= 1, NaN) -> NaN
  V g = lv_map2(u, E, [](float uu, float ee) {
    float gg;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(gg) : "f"(uu));
    return (uu > 0.f && ee > 0.f) ? gg : __int_as_float(0x7fffffff);
  });
  V bg = lv_map(lv_fma(u, g, u), [](float x) { return fast_rcp(x); });
  // boost vector 1 (y = 0) and vector 2, literally (SPEC.md:188 with R6)
  V bpa = lv_fma(betz, az, lv_mul(betx, ax));
  V fa = lv_fma(bg, bpa, lv_mul(g, aE));
  V a2x = lv_fma(fa, betx, ax), a2y = lv_mul(fa, bety), a2z = lv_fma(fa, betz, az), a2t = lv_mul(g, lv_add(aE, bpa));
  V bpb = lv_fma(betz, bz, lv_fma(bety, by, lv_mul(betx, bx)));
  V fb = lv_fma(bg, bpb, lv_mul(g, bE));
  V b2x = lv_fma(fb, betx, bx), b2y = lv_fma(fb, bety, by), b2z = lv_fma(fb, betz, bz), b2t = lv_mul(g, lv_add(bE, bpb));
  if constexpr (WANT_VEC) {
    vec_out[0] = a2x; vec_out[1] = a2y; vec_out[2] = a2z; vec_out[3] = a2t;
    vec_out[4] = b2x; vec_out[5] = b2y; vec_out[6] = b2z; vec_out[7] = b2t;
  }
  V X = lv_add(a2x, b2x), Y = lv_fma(fa, bety, b2y), Z = lv_add(a2z, b2z);
  V W = lv_fma(g, lv_add(aE, bpa), b2t);
  V p2 = lv_fma(Z, Z, lv_fma(Y, Y, lv_mul(X, X)));
  V m2sq = lv_fma(W, W, lv_mul(p2, MONE));
  if constexpr (WANT_COS) {
    V pa = lv_fma(a2z, a2z, lv_fma(a2y, a2y, lv_mul(a2x, a2x)));
    *cos_out = lv_mul(a2z, lv_map(pa, [](float x) {
                        float y;
                        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
                        return y;
                      }));
  }
  return lv_map(m2sq, [](float x) { return sqrt_abs_signed(x); });
}

// ---------------------------------------------------------------------------
// PxPyPzM and PtEtaPhiE.
// ---------------------------------------------------------------------------
// PxPyPzM -> PxPyPzE: E = sqrt(max(0, |p|^2 + m|m|)) (R2 clamp).
template <typename T>
__device__ __forceinline__ V4<T> pxpypzm_to_cartesian(T px, T py, T pz, T m) {
  T e2 = px * px + py * py + pz * pz + m * (m < T(0) ? -m : m);
  return V4<T>{px, py, pz, ieee_sqrt(e2 > T(0) ? e2 : T(0))};
}

// PtEtaPhiE -> PxPyPzE with accurate libm (cold path).
__device__ __noinline__ V4<double> ptetaphie_exact(double pt, double eta, double phi, double E) {
  double s, c;
  sincos(phi, &s, &c);
  return V4<double>{pt * c, pt * s, pt * sinh(eta), E};
}
__device__ __noinline__ V4<float> ptetaphie_exact(float pt, float eta, float phi, float E) {
  float s, c;
  sincosf(phi, &s, &c);
  return V4<float>{pt * c, pt * s, pt * sinhf(eta), E};
}
// Fast domain for PtEtaPhiE: the angle/rapidity limits of PtEtaPhiM and a finite E.
template <typename T>
__device__ __forceinline__ bool fast_domain_e(T pt, T eta, T phi, T E) {
  return fast_domain(pt, eta, phi, T(0)) && fabs(E) < T(1e30);
}
template <typename T>
__device__ __forceinline__ V4<T> ptetaphie_to_cartesian(T pt, T eta, T phi, T E) {
  if (fast_domain_e(pt, eta, phi, E)) {
    T s, c, sh, ch;
    fast_sincos(phi, s, c);
    sinh_cosh(eta, sh, ch);
    return V4<T>{pt * c, pt * s, pt * sh, E};
  }
  return ptetaphie_exact(pt, eta, phi, E);
}
// Pair mass of PtEtaPhiE vectors without forming Cartesian vectors:
//   M^2 = (E1 + E2)^2 - (pt1 ch1)^2 - (pt2 ch2)^2 - 2 pt1 pt2 (cos(phi1 - phi2) + sh1 sh2)
template <typename T>
__device__ __forceinline__ T pair_mass_ptetaphie(T pt1, T eta1, T phi1, T E1, T pt2, T eta2, T phi2, T E2) {
  if (fast_domain_e(pt1, eta1, phi1, E1) && fast_domain_e(pt2, eta2, phi2, E2)) {
    T sd, c, sh1, ch1, sh2, ch2;
    fast_sincos(phi1 - phi2, sd, c);
    sinh_cosh(eta1, sh1, ch1);
    sinh_cosh(eta2, sh2, ch2);
    T q1 = pt1 * ch1, q2 = pt2 * ch2, E = E1 + E2;
    T m2 = E * E - q1 * q1 - q2 * q2 - T(2) * pt1 * pt2 * (c + sh1 * sh2);
    return fast_signed_sqrt(m2);
  }
  return mass_of_sum(ptetaphie_exact(pt1, eta1, phi1, E1), ptetaphie_exact(pt2, eta2, phi2, E2));
}

// ---------------------------------------------------------------------------
// ROOT FindFixBin in double, bit-identical to the oracle's
//   x < lo -> 0;  !(x < hi) -> nbins+1;  else 1 + (int)((nbins * (x - lo)) / (hi - lo))
// Fast path (5 FP64 ops, the rest on the integer pipe): q = (x - lo) * scale,
// scale = nbins / (hi - lo), is within 4 ulp of the oracle's quotient (2u
// relative on each side), so floor(q) equals the oracle's truncation unless q
// lies within 1e-14 * nbins of an integer. k = rint(q) comes from the
// 1.5*2^52 shifter; d = q - k is exact (Sterbenz). When t = q + MAGIC has the
// high word 0x43380000 and k <= nbins, q is in [-0.5, nbins + 0.5) and the bin
// is 1 + k - (d < 0) (k = 0, d < 0 -> 0 = underflow; k = nbins, d >= 0 ->
// nbins+1 = overflow, both exactly the oracle's x < lo / !(x < hi) once
// |d| > tol). Outside that window the sign of q decides (x < lo - w/2 or
// x > hi + w/2). Near-integer q and non-finite x (NaN -> overflow) take the
// literal definition out of line.
// ---------------------------------------------------------------------------
struct HistParams {
  double lo, hi, width;  // width = hi - lo (the same IEEE value the oracle forms)
  double nbins_d;        // (double)nbins
  double scale;          // nbins_d / width
  int nbins;
  uint32_t near_hi;      // high word of 1e-14 * nbins: |d| with abs_hi(d) <= near_hi is "near"
  // fp32 masses (find_bin(float)): the same scheme in FP32 with a wider near-edge window
  float lo_f, scale_f, near_f;
  int f32_ok;            // nbins <= 2^20 and the float parameters are finite
  // Where a CTA's final counts go (hist_flush): the caller's `bins` (default), or
  // fused into the multi-GPU reduction: every rank's bins through
  // peer pointers (P2P atomics over NVLink), or one NVSwitch multicast address.
  unsigned long long* const* peers;  // device array of npeers bin arrays, or NULL
  int npeers;
  unsigned long long* mc;            // multicast address of the bins (multimem.red), or NULL
  // Pre-reduction for the peers / mc sink: CTAs flush into this device-local
  // workspace (nbins+2 counters, then a ticket word); the last CTA of the launch
  // pushes the <= nbins+2 non-zero totals to the sink and leaves it zeroed.
  unsigned long long* work;
};

inline HistParams make_hist_params(double lo, double hi, int nbins) {
  HistParams hp;
  hp.lo = lo;
  hp.hi = hi;
  hp.width = hi - lo;
  hp.nbins_d = (double)nbins;
  hp.scale = hp.nbins_d / hp.width;
  hp.nbins = nbins;
  double tol = 1e-14 * hp.nbins_d;
  uint64_t bits;
  memcpy(&bits, &tol, 8);
  hp.near_hi = (uint32_t)(bits >> 32);
  // fp32 path: q_f = RN(RN(x - lo_f) * scale_f) is within 3 float ulps of q (relative 1.8e-7)
  // plus |lo_f - lo| * scale; the window is 4x that bound on the in-range |q| <= nbins.
  hp.lo_f = (float)lo;
  hp.scale_f = (float)hp.scale;
  const double lo_err = fabs((double)hp.lo_f - lo) * hp.scale;
  hp.near_f = (float)(4.0 * (1.8e-7 * (hp.nbins_d + 1.0) + lo_err) + 1e-30);
  hp.f32_ok = nbins <= (1 << 20) && isfinite(hp.lo_f) && isfinite(hp.scale_f) && hp.scale_f > 0.f &&
              hp.near_f < 0.25f;
  hp.peers = nullptr;
  hp.npeers = 0;
  hp.mc = nullptr;
  hp.work = nullptr;
  return hp;
}

// Add count c to bin b of the histogram described by hp (see HistParams).
__device__ __forceinline__ void hist_push(const HistParams& hp, int b, unsigned long long c) {
  if (hp.mc) {
    asm volatile("multimem.red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(hp.mc + b), "l"(c) : "memory");
  } else {
    for (int p = 0; p < hp.npeers; ++p) atomicAdd_system(hp.peers[p] + b, c);
  }
}
__device__ __forceinline__ void hist_flush(unsigned long long* bins, const HistParams& hp, int b,
                                           unsigned long long c) {
  if (hp.work) {
    atomicAdd(hp.work + b, c);  // device-local partial sum; hist_tail pushes the totals
  } else if (hp.mc || hp.npeers > 0) {
    hist_push(hp, b, c);
  } else {
    atomicAdd(bins + b, c);
  }
}

// Kernel tail of the pre-reduced cross-GPU sink (hp.work != NULL), reached by every
// thread of every CTA after its last hist_flush: each thread fences its flush atomics,
// one ticket per CTA is taken after a CTA barrier, and the CTA that takes the last
// ticket reads-and-clears the workspace and pushes each non-zero total once to the
// sink — <= nbins+2 remote adds per peer per launch (multimem.red: per launch)
// instead of one per CTA and bin — then re-arms the ticket for the next launch.
__device__ __forceinline__ void hist_tail(const HistParams& hp) {
  if (!hp.work) return;  // uniform over the grid
  __shared__ int is_last;
  unsigned int* ticket = reinterpret_cast<unsigned int*>(hp.work + hp.nbins + 2);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  for (int b = threadIdx.x; b < hp.nbins + 2; b += blockDim.x) {
    const unsigned long long c = atomicExch(hp.work + b, 0ull);
    if (c) hist_push(hp, b, c);
  }
  if (threadIdx.x == 0) atomicExch(ticket, 0u);
}

__device__ __noinline__ int find_bin_exact(double x, const HistParams& hp) {
  if (x < hp.lo) return 0;
  if (!(x < hp.hi)) return hp.nbins + 1;
  return 1 + __double2int_rz(__ddiv_rn(__dmul_rn(hp.nbins_d, __dsub_rn(x, hp.lo)), hp.width));
}

__device__ __forceinline__ int find_bin(double x, const HistParams& hp);

// fp32 value: the oracle promotes it to double and bins there (R12); the same
// shifter scheme in FP32 (t = q + 1.5*2^23, k = rint(q) from t's bits, |q| < 2^22)
// decides every event whose q is more than near_f from an integer, the rest (and
// non-finite x) take the double path. Saves the F2F.F64 (XU) and the DP ops in the
// issue-bound fp32 kernels.
// The integer part of find_bin(float): q = (x - lo_f) scale_f, t = q + 1.5*2^23,
// d = q - (t - 1.5*2^23) (all FP32, round to nearest).
__device__ __forceinline__ int find_bin_f32_tail(float x, float q, float t, float d, const HistParams& hp) {
  const int k = __float_as_int(t) - 0x4B400000;
  const bool in = (unsigned)k <= (unsigned)hp.nbins;
  int bin = in ? 1 + k - (__float_as_int(d) < 0 ? 1 : 0) : (__float_as_int(q) < 0 ? 0 : hp.nbins + 1);
  // near an edge (or non-finite): the fp64 scheme of find_bin(double), inline (it
  // takes the literal out-of-line definition only within 1e-14 nbins of an edge).
  // ~18 % of warps have such a lane among their 4 x 32 values per pass, so an
  // out-of-line IEEE division here cost divergence plus local-memory traffic.
  if ((in & (fabsf(d) <= hp.near_f)) | ((__float_as_int(x) & 0x7fffffff) >= 0x7f800000))
    bin = find_bin((double)x, hp);
  return bin;
}
__device__ __forceinline__ int find_bin(float x, const HistParams& hp) {
  if (!hp.f32_ok) return find_bin((double)x, hp);
  const float MAGIC = 12582912.f;  // 1.5 * 2^23
  const float q = __fmul_rn(__fsub_rn(x, hp.lo_f), hp.scale_f);
  const float t = __fadd_rn(q, MAGIC);
  const float d = __fsub_rn(q, __fsub_rn(t, MAGIC));
  return find_bin_f32_tail(x, q, t, d, hp);
}
// Two fp32 values (two events' masses) with the FP32 steps in packed FADD2 /
// FMUL2 / FFMA2: the same roundings as find_bin(float) (x - lo = x + (-lo),
// q - u = fma(u, -1, q)), so the same bins.
__device__ __forceinline__ int2 find_bin2(float2 x, const HistParams& hp) {
  if (!hp.f32_ok) return make_int2(find_bin((double)x.x, hp), find_bin((double)x.y, hp));
  const float MAGIC = 12582912.f;
  const float2 q = lv_mul(lv_add(x, lv_splat(x, -hp.lo_f)), lv_splat(x, hp.scale_f));
  const float2 t = lv_add(q, lv_splat(x, MAGIC));
  const float2 d = lv_fma(lv_add(t, lv_splat(x, -MAGIC)), lv_splat(x, -1.f), q);
  return make_int2(find_bin_f32_tail(x.x, q.x, t.x, d.x, hp), find_bin_f32_tail(x.y, q.y, t.y, d.y, hp));
}

__device__ __forceinline__ int find_bin(double x, const HistParams& hp) {
  const double MAGIC = 6755399441055744.0;  // 1.5 * 2^52
  const double q = __dmul_rn(__dsub_rn(x, hp.lo), hp.scale);
  const double t = __dadd_rn(q, MAGIC);
  const int k = __double2loint(t);
  const double d = __dsub_rn(q, __dsub_rn(t, MAGIC));
  const bool in = (__double2hiint(t) == 0x43380000) & ((unsigned)k <= (unsigned)hp.nbins);
  int bin = in ? 1 + k - (__double2hiint(d) < 0 ? 1 : 0) : (__double2hiint(q) < 0 ? 0 : hp.nbins + 1);
  if ((in & (abs_hi(d) <= hp.near_hi)) | (abs_hi(x) >= 0x7FF00000u)) bin = find_bin_exact(x, hp);
  return bin;
}

}  // namespace gvx
