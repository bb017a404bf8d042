// gvx_kernels.cuh — sm_100a kernels of the GenVectorX hot path.
//
// Structure: persistent grid-stride kernels, one grid of
// (148 SMs x resident CTAs), each thread moving U "groups" per iteration with
// warp-contiguous 256-bit loads (LDG.E.ENL2.256) so that every load
// instruction of a warp covers 1 KiB of consecutive HBM:
//   AoS f64: group = 1 event  (v[i] is one 32-byte vector)
//   AoS f32: group = 2 events (two 16-byte vectors per 256-bit load)
//   SoA f64: group = 4 events, SoA f32: group = 8 events (per component)
//   generic strided view: group = 1 event, scalar loads.
// Events n % G at the end (and misaligned views) use scalar loads.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "gvx_math.cuh"
#include "gvx_tma.cuh"

namespace gvx {

enum Layout { L_AOS = 0, L_SOA = 1, L_GEN = 2 };
enum Coords { C_PTETAPHIM = 0, C_PXPYPZE = 1, C_PXPYPZM = 2, C_PTETAPHIE = 3 };
// What a pair kernel produces. PM_BOTH: lab mass + lab histogram + CM mass + CM
// histogram in one pass over the pairs (gvx_pair_histograms); in k_pair_tma the
// CM histogram and masses use the CosOut slot.
enum PairMode { PM_MASS = 0, PM_HIST = 1, PM_HIST_CM = 2, PM_HIST_CM_COS = 3, PM_BOTH = 4 };

template <typename T> struct View4 { const T* c[4]; int64_t s; };

// Warpgroup register reallocation (sm_90a+): every warp of the warpgroup executes it.
template <int R> __device__ __forceinline__ void setmaxnreg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(R));
}
template <int R> __device__ __forceinline__ void setmaxnreg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(R));
}
template <typename T> struct View4o { T* c[4]; int64_t s; };
template <typename T> struct View3 { const T* c[3]; int64_t s; };

template <typename T, int L> struct Group {
  static constexpr int G = (L == L_AOS) ? (32 / (4 * (int)sizeof(T))) : (L == L_SOA) ? (32 / (int)sizeof(T)) : 1;
};

// ---- 256-bit streaming loads / stores (inline PTX; sm_100 v4.f64 / v8.f32) --
__device__ __forceinline__ void ld256(const double* p, double (&r)[4]) {
  asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3]) : "l"(p));
}
__device__ __forceinline__ void ld256(const float* p, float (&r)[8]) {
  asm("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
      : "l"(p));
}
__device__ __forceinline__ void st256(double* p, const double (&r)[4]) {
  asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(r[0]), "d"(r[1]),
               "d"(r[2]), "d"(r[3]) : "memory");
}
__device__ __forceinline__ void st256(float* p, const float (&r)[8]) {
  asm volatile("st.global.L1::no_allocate.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r[0]),
               "f"(r[1]), "f"(r[2]), "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7]) : "memory");
}

// Load group g of a 4-vector view: x[k][j] = component k of event g*G + j.
template <typename T, int L>
__device__ __forceinline__ void load_group(const View4<T>& v, int64_t g, T (&x)[4][Group<T, L>::G]) {
  constexpr int G = Group<T, L>::G;
  if constexpr (L == L_AOS) {
    constexpr int W = 32 / sizeof(T);  // scalars per 256-bit load = 4*G
    T r[W];
    ld256(v.c[0] + g * W, r);
#pragma unroll
    for (int j = 0; j < G; ++j)
#pragma unroll
      for (int k = 0; k < 4; ++k) x[k][j] = r[4 * j + k];
  } else if constexpr (L == L_SOA) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      T r[G];
      ld256(v.c[k] + g * G, r);
#pragma unroll
      for (int j = 0; j < G; ++j) x[k][j] = r[j];
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) x[k][0] = __ldg(v.c[k] + g * v.s);
  }
}

template <typename T>
__device__ __forceinline__ void load_event(const View4<T>& v, int64_t i, T (&x)[4]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) x[k] = __ldg(v.c[k] + i * v.s);
}

// Store G contiguous results.
template <typename T, int G>
__device__ __forceinline__ void store_group(T* __restrict__ out, int64_t g, const T (&m)[G]) {
  if constexpr (G * sizeof(T) == 32) {
    st256(out + g * G, m);
  } else if constexpr (G == 2 && sizeof(T) == 4) {
    *reinterpret_cast<float2*>(out + g * 2) = make_float2(m[0], m[1]);
  } else {
#pragma unroll
    for (int j = 0; j < G; ++j) out[g * G + j] = m[j];
  }
}

template <typename T, int COORDS>
__device__ __forceinline__ V4<T> to_cartesian(const T (&a)[4]) {
  if constexpr (COORDS == C_PTETAPHIM) return ptetaphim_to_cartesian(a[0], a[1], a[2], a[3]);
  else if constexpr (COORDS == C_PXPYPZM) return pxpypzm_to_cartesian(a[0], a[1], a[2], a[3]);
  else if constexpr (COORDS == C_PTETAPHIE) return ptetaphie_to_cartesian(a[0], a[1], a[2], a[3]);
  else return V4<T>{a[0], a[1], a[2], a[3]};
}

template <typename T, int COORDS>
__device__ __forceinline__ T event_mass(const T (&a)[4], const T (&b)[4]) {
  if constexpr (COORDS == C_PTETAPHIM) {
    return pair_mass_ptetaphim(a[0], a[1], a[2], a[3], b[0], b[1], b[2], b[3]);
  } else if constexpr (COORDS == C_PTETAPHIE) {
    return pair_mass_ptetaphie(a[0], a[1], a[2], a[3], b[0], b[1], b[2], b[3]);
  } else {
    return mass_of_sum(to_cartesian<T, COORDS>(a), to_cartesian<T, COORDS>(b));
  }
}

// ============================================================================
// K1: invariant mass
// ============================================================================
template <typename T, int COORDS, int L, int U, int MINB = 1>
__global__ void __launch_bounds__(256, MINB) k_invariant_mass(View4<T> v1, View4<T> v2, T* __restrict__ m, int64_t n) {
  constexpr int G = Group<T, L>::G;
  const int64_t ngroups = n / G;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t g0 = tid; g0 < ngroups; g0 += nthr * U) {
    T a[U][4][G], b[U][4][G];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int64_t g = g0 + u * nthr;
      if (g < ngroups) { load_group<T, L>(v1, g, a[u]); load_group<T, L>(v2, g, b[u]); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int64_t g = g0 + u * nthr;
      if (g < ngroups) {
        T r[G];
#pragma unroll
        for (int j = 0; j < G; ++j) {
          T x[4] = {a[u][0][j], a[u][1][j], a[u][2][j], a[u][3][j]};
          T y[4] = {b[u][0][j], b[u][1][j], b[u][2][j], b[u][3][j]};
          r[j] = event_mass<T, COORDS>(x, y);
        }
        store_group<T, G>(m, g, r);
      }
    }
  }
  if constexpr (G > 1) {
    int64_t i = ngroups * G + tid;
    if (i < n) {
      T x[4], y[4];
      load_event(v1, i, x);
      load_event(v2, i, y);
      m[i] = event_mass<T, COORDS>(x, y);
    }
  }
}

// ============================================================================
// K2: boost by per-event (or uniform) beta
// ============================================================================
template <typename T, bool AOS>
__device__ __forceinline__ V4<T> boost_load_v(const View4<T>& v, int64_t i) {
  if constexpr (AOS) {
    if constexpr (sizeof(T) == 8) {
      double r[4];
      ld256(reinterpret_cast<const double*>(v.c[0]) + 4 * i, r);
      return V4<T>{(T)r[0], (T)r[1], (T)r[2], (T)r[3]};
    } else {
      float4 r = __ldcs(reinterpret_cast<const float4*>(v.c[0]) + i);
      return V4<T>{(T)r.x, (T)r.y, (T)r.z, (T)r.w};
    }
  } else {
    return V4<T>{__ldg(v.c[0] + i * v.s), __ldg(v.c[1] + i * v.s), __ldg(v.c[2] + i * v.s), __ldg(v.c[3] + i * v.s)};
  }
}
template <typename T, bool AOS>
__device__ __forceinline__ void boost_store(const View4o<T>& out, int64_t i, const V4<T>& o) {
  if constexpr (AOS) {
    if constexpr (sizeof(T) == 8) {
      double r[4] = {(double)o.x, (double)o.y, (double)o.z, (double)o.t};
      st256(reinterpret_cast<double*>(out.c[0]) + 4 * i, r);
    } else {
      __stcs(reinterpret_cast<float4*>(out.c[0]) + i, make_float4((float)o.x, (float)o.y, (float)o.z, (float)o.t));
    }
  } else {
    out.c[0][i * out.s] = o.x;
    out.c[1][i * out.s] = o.y;
    out.c[2][i * out.s] = o.z;
    out.c[3][i * out.s] = o.t;
  }
}

// U events per thread per iteration: all loads issued before any arithmetic
// (bytes in flight per SM scale with U at the same occupancy).
template <typename T, bool AOS, bool UNIFORM, int U = 1>
__global__ void __launch_bounds__(256) k_boost(View4<T> v, View3<T> beta, View4o<T> out, int64_t n, T ubx,
                                               T uby, T ubz) {
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  BoostCoef<T> ku;
  if constexpr (UNIFORM) ku = boost_coef(ubx, uby, ubz);
  for (int64_t i0 = tid; i0 < n; i0 += nthr * U) {
    V4<T> x[U];
    T bx[U], by[U], bz[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * nthr;
      if (i < n) {
        x[u] = boost_load_v<T, AOS>(v, i);
        if constexpr (!UNIFORM) {
          bx[u] = __ldg(beta.c[0] + i * beta.s);
          by[u] = __ldg(beta.c[1] + i * beta.s);
          bz[u] = __ldg(beta.c[2] + i * beta.s);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * nthr;
      if (i < n) {
        BoostCoef<T> k;
        if constexpr (UNIFORM) k = ku;
        else k = boost_coef(bx[u], by[u], bz[u]);
        boost_store<T, AOS>(out, i, apply_boost(k, x[u]));
      }
    }
  }
}

// ============================================================================
// General 4x4 Lorentz transformation ("4x4 orthosymplectic
// matrix"): out = L v, L uniform (kernel parameter).
// ============================================================================
template <typename T> struct Mat4 { T m[4][4]; };

template <typename T, bool AOS>
__global__ void __launch_bounds__(256) k_lorentz(View4<T> v, View4o<T> out, int64_t n, Mat4<T> L) {
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += nthr) {
    T x[4];
    if constexpr (AOS) {
      if constexpr (sizeof(T) == 8) {
        double r[4];
        ld256(reinterpret_cast<const double*>(v.c[0]) + 4 * i, r);
#pragma unroll
        for (int c = 0; c < 4; ++c) x[c] = (T)r[c];
      } else {
        float4 r = __ldcs(reinterpret_cast<const float4*>(v.c[0]) + i);
        x[0] = r.x; x[1] = r.y; x[2] = r.z; x[3] = r.w;
      }
    } else {
      load_event(v, i, x);
    }
    T o[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      T acc = L.m[r][0] * x[0];
#pragma unroll
      for (int c = 1; c < 4; ++c) acc = fma(L.m[r][c], x[c], acc);
      o[r] = acc;
    }
    if constexpr (AOS) {
      if constexpr (sizeof(T) == 8) {
        double r[4] = {(double)o[0], (double)o[1], (double)o[2], (double)o[3]};
        st256(reinterpret_cast<double*>(out.c[0]) + 4 * i, r);
      } else {
        __stcs(reinterpret_cast<float4*>(out.c[0]) + i, make_float4(o[0], o[1], o[2], o[3]));
      }
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) out.c[c][i * out.s] = o[c];
    }
  }
}

// ============================================================================
// K3: fused mass (lab or CM frame) + histogram, privatised in shared memory.
// ============================================================================
// WANT_COS (CM only): also cos theta* of boosted vector 1 into *cos (reading R22).
template <typename T, int COORDS, bool CM, bool WANT_BO = false, bool WANT_COS = false>
__device__ __forceinline__ T hist_event_mass(const T (&a)[4], const T (&b)[4], int64_t i, const View4o<T>& bo,
                                             T* cos = nullptr) {
  if constexpr (CM) {
    V4<T> xa, yb;
    T M;
    if (COORDS == C_PTETAPHIM && fast_domain(a[0], a[1], a[2], a[3]) && fast_domain(b[0], b[1], b[2], b[3])) {
      M = cm_mass_ptetaphim_fast<T, WANT_COS>(a[0], a[1], a[2], a[3], b[0], b[1], b[2], b[3],
                                             WANT_BO ? &xa : nullptr, &yb, cos);
    } else if constexpr (COORDS == C_PTETAPHIM) {  // cold path: literal libm conversion
      M = cm_pair_mass<T, false, WANT_COS>(ptetaphim_exact(a[0], a[1], a[2], a[3]),
                                           ptetaphim_exact(b[0], b[1], b[2], b[3]), WANT_BO ? &xa : nullptr, &yb,
                                           cos);
    } else {
      M = cm_pair_mass<T, false, WANT_COS>(to_cartesian<T, COORDS>(a), to_cartesian<T, COORDS>(b),
                                           WANT_BO ? &xa : nullptr, &yb, cos);
    }
    if constexpr (WANT_BO) {
      int64_t j0 = (2 * i) * bo.s, j1 = (2 * i + 1) * bo.s;
      bo.c[0][j0] = xa.x; bo.c[1][j0] = xa.y; bo.c[2][j0] = xa.z; bo.c[3][j0] = xa.t;
      bo.c[0][j1] = yb.x; bo.c[1][j1] = yb.y; bo.c[2][j1] = yb.z; bo.c[3][j1] = yb.t;
    }
    return M;
  } else {
    return event_mass<T, COORDS>(a, b);
  }
}

template <typename T, int COORDS, int L, bool CM, bool SMEM, int MINB = 1, bool WANT_BO = false>
__global__ void __launch_bounds__(256, MINB) k_mass_histogram(View4<T> v1, View4<T> v2, int64_t n, HistParams hp,
                                                        unsigned long long* __restrict__ bins, T* __restrict__ m_out,
                                                        View4o<T> bo) {
  extern __shared__ unsigned int sh[];
  constexpr int G = Group<T, L>::G;
  const int nb2 = hp.nbins + 2;
  if constexpr (SMEM) {
    for (int b = threadIdx.x; b < nb2; b += blockDim.x) sh[b] = 0u;
    __syncthreads();
  }
  auto count = [&](T M) {
    int b = find_bin(M, hp);
    if constexpr (SMEM) atomicAdd(&sh[b], 1u);
    else hist_flush(bins, hp, b, 1ull);
  };
  const int64_t ngroups = n / G;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t g = tid; g < ngroups; g += nthr) {
    T a[4][G], b[4][G];
    load_group<T, L>(v1, g, a);
    load_group<T, L>(v2, g, b);
    T r[G];
#pragma unroll
    for (int j = 0; j < G; ++j) {
      T x[4] = {a[0][j], a[1][j], a[2][j], a[3][j]};
      T y[4] = {b[0][j], b[1][j], b[2][j], b[3][j]};
      r[j] = hist_event_mass<T, COORDS, CM, WANT_BO>(x, y, g * G + j, bo);
      count(r[j]);
    }
    if (m_out) store_group<T, G>(m_out, g, r);
  }
  if constexpr (G > 1) {
    int64_t i = ngroups * G + tid;
    if (i < n) {
      T x[4], y[4];
      load_event(v1, i, x);
      load_event(v2, i, y);
      T M = hist_event_mass<T, COORDS, CM, WANT_BO>(x, y, i, bo);
      count(M);
      if (m_out) m_out[i] = M;
    }
  }
  if constexpr (SMEM) {
    __syncthreads();
    for (int b = threadIdx.x; b < nb2; b += blockDim.x) {
      unsigned int c = sh[b];
      if (c) hist_flush(bins, hp, b, c);
    }
  }
  hist_tail(hp);  // pre-reduced cross-GPU sink only (gvx_mass_histogram_peers)
}

// ============================================================================
// CM mass + cos theta* histograms (reading R22), any layout / coordinates:
// one event per thread, grid-stride, scalar loads through the views. The
// AoS / SoA PtEtaPhiM / PxPyPzE fast path is k_pair_tma (PM_HIST_CM_COS).
// SMEM: both histograms privatised in shared memory (else global atomics).
// ============================================================================
template <typename T, int COORDS, bool SMEM>
__global__ void __launch_bounds__(256) k_cm_costheta(View4<T> v1, View4<T> v2, int64_t n, HistParams hm,
                                                     unsigned long long* __restrict__ mbins, HistParams hc,
                                                     unsigned long long* __restrict__ cbins, T* __restrict__ m_out,
                                                     T* __restrict__ cos_out) {
  extern __shared__ unsigned int shc[];
  const int nm = hm.nbins + 2, nc = hc.nbins + 2;
  if constexpr (SMEM) {
    for (int b = threadIdx.x; b < nm + nc; b += blockDim.x) shc[b] = 0u;
    __syncthreads();
  }
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  View4o<T> none{};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += nthr) {
    T x[4], y[4], c;
    load_event(v1, i, x);
    load_event(v2, i, y);
    T M = hist_event_mass<T, COORDS, true, false, true>(x, y, i, none, &c);
    const int bm = find_bin(M, hm), bc = find_bin(c, hc);
    if constexpr (SMEM) {
      atomicAdd(&shc[bm], 1u);
      atomicAdd(&shc[nm + bc], 1u);
    } else {
      hist_flush(mbins, hm, bm, 1ull);
      atomicAdd(&cbins[bc], 1ull);
    }
    if (m_out) m_out[i] = M;
    if (cos_out) cos_out[i] = c;
  }
  if constexpr (SMEM) {
    __syncthreads();
    for (int b = threadIdx.x; b < nm + nc; b += blockDim.x) {
      unsigned int v = shc[b];
      if (v) {
        if (b < nm) hist_flush(mbins, hm, b, v);
        else atomicAdd(&cbins[b - nm], (unsigned long long)v);
      }
    }
  }
}

// ============================================================================
// Mixed-coordinate pairs (the kernel takes "two
// particles expressed in any 4-dimensional coordinate system"; SPEC.md:305:
// the result does not depend on the systems of the operands). v1 is in system
// c1 and v2 in c2 (kernel arguments: warp-uniform branches, so one instantiation
// per mode covers the 12 mixed combinations). Each vector is converted to
// PxPyPzE on its own with the same conversions the single-system kernels use
// (fast domain + literal cold path), then summed and its signed mass taken
// literally (mass_of_sum: E^2 - |P|^2); the CM modes boost
// the pair with cm_pair_mass (reading R11). Same-system pairs never come here:
// they keep the reduced-form kernels above (the ABI dispatches on c1 == c2).
//   MODE  PM_MASS: m_out;  PM_HIST / PM_HIST_CM: lab / CM mass -> bins (+ m_out,
//         + boosted pair for CM);  PM_BOTH: lab -> bins + m_out, CM -> co.bins +
//         co.cos_out (the fused pair pass of gvx_pair_histograms).
//   SMEM  histograms privatised in shared memory (else global atomics).
// ============================================================================
template <typename T>
__device__ __noinline__ V4<T> to_cartesian_rt(int c, T a0, T a1, T a2, T a3) {
  const T a[4] = {a0, a1, a2, a3};
  if (c == C_PTETAPHIM) return ptetaphim_to_cartesian(a[0], a[1], a[2], a[3]);
  if (c == C_PXPYPZM) return pxpypzm_to_cartesian(a[0], a[1], a[2], a[3]);
  if (c == C_PTETAPHIE) return ptetaphie_to_cartesian(a[0], a[1], a[2], a[3]);
  return V4<T>{a[0], a[1], a[2], a[3]};
}

// The arithmetic of the mixed kernels (the conversion above and these two) is out of line:
// every mode calls the same code, so the fused pass (PM_BOTH) gives the bits of the separate
// mass / CM calls whatever the compiler would contract or share in an inlined context.
template <typename T>
__device__ __noinline__ T mixed_lab_mass(V4<T> a, V4<T> b) {
  return mass_of_sum(a, b);
}
template <typename T>
__device__ __noinline__ T mixed_cm_mass(V4<T> a, V4<T> b, V4<T>* a2, V4<T>* b2) {
  return cm_pair_mass<T>(a, b, a2, b2);
}

template <typename T, int L, int MODE, bool SMEM>
__global__ void __launch_bounds__(256) k_mixed_pairs(View4<T> v1, View4<T> v2, int c1, int c2, int64_t n,
                                                     HistParams hp, unsigned long long* __restrict__ bins,
                                                     T* __restrict__ m_out, HistParams hc,
                                                     unsigned long long* __restrict__ cbins, T* __restrict__ cm_out,
                                                     View4o<T> bo) {
  extern __shared__ unsigned int shx[];
  constexpr int G = Group<T, L>::G;
  static_assert(MODE == PM_MASS || MODE == PM_HIST || MODE == PM_HIST_CM || MODE == PM_BOTH, "mode");
  constexpr bool HIST = MODE != PM_MASS;
  constexpr bool TWO = MODE == PM_BOTH;
  constexpr bool CM = MODE == PM_HIST_CM || TWO;
  const int nb2 = hp.nbins + 2;
  const int nbt = HIST ? nb2 + (TWO ? hc.nbins + 2 : 0) : 0;
  if constexpr (SMEM && HIST) {
    for (int b = threadIdx.x; b < nbt; b += blockDim.x) shx[b] = 0u;
    __syncthreads();
  }
  auto count = [&](T M, bool second) {
    if constexpr (SMEM) {
      atomicAdd(&shx[second ? nb2 + find_bin(M, hc) : find_bin(M, hp)], 1u);
    } else {
      if (second) atomicAdd(&cbins[find_bin(M, hc)], 1ull);
      else hist_flush(bins, hp, find_bin(M, hp), 1ull);
    }
  };
  auto event = [&](const T (&x)[4], const T (&y)[4], int64_t i) {
    const V4<T> a = to_cartesian_rt(c1, x[0], x[1], x[2], x[3]), b = to_cartesian_rt(c2, y[0], y[1], y[2], y[3]);
    T ml = T(0), mc = T(0);
    if constexpr (MODE != PM_HIST_CM) ml = mixed_lab_mass(a, b);
    if constexpr (CM) {
      V4<T> a2, b2;
      const bool wbo = !TWO && bo.c[0] != nullptr;
      mc = mixed_cm_mass(a, b, wbo ? &a2 : nullptr, wbo ? &b2 : nullptr);
      if (wbo) {
        const int64_t j0 = (2 * i) * bo.s, j1 = (2 * i + 1) * bo.s;
        bo.c[0][j0] = a2.x; bo.c[1][j0] = a2.y; bo.c[2][j0] = a2.z; bo.c[3][j0] = a2.t;
        bo.c[0][j1] = b2.x; bo.c[1][j1] = b2.y; bo.c[2][j1] = b2.z; bo.c[3][j1] = b2.t;
      }
    }
    if constexpr (MODE == PM_MASS) {
      m_out[i] = ml;
    } else if constexpr (MODE == PM_HIST) {
      count(ml, false);
      if (m_out) m_out[i] = ml;
    } else if constexpr (MODE == PM_HIST_CM) {
      count(mc, false);
      if (m_out) m_out[i] = mc;
    } else {
      count(ml, false);
      count(mc, true);
      if (m_out) m_out[i] = ml;
      if (cm_out) cm_out[i] = mc;
    }
  };
  const int64_t ngroups = n / G;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t g = tid; g < ngroups; g += nthr) {
    T a[4][G], b[4][G];
    load_group<T, L>(v1, g, a);
    load_group<T, L>(v2, g, b);
#pragma unroll
    for (int j = 0; j < G; ++j) {
      T x[4] = {a[0][j], a[1][j], a[2][j], a[3][j]};
      T y[4] = {b[0][j], b[1][j], b[2][j], b[3][j]};
      event(x, y, g * G + j);
    }
  }
  if constexpr (G > 1) {
    const int64_t i = ngroups * G + tid;
    if (i < n) {
      T x[4], y[4];
      load_event(v1, i, x);
      load_event(v2, i, y);
      event(x, y, i);
    }
  }
  if constexpr (SMEM && HIST) {
    __syncthreads();
    for (int b = threadIdx.x; b < nbt; b += blockDim.x) {
      const unsigned int c = shx[b];
      if (c) {
        if (b < nb2) hist_flush(bins, hp, b, c);
        else atomicAdd(&cbins[b - nb2], (unsigned long long)c);
      }
    }
  }
}

// ============================================================================
// Jagged dimuon selection + mass histogram (DESIGN R21):
// event e owns muons [offsets[e], offsets[e+1]); selected iff exactly two
// muons of opposite charge; the pair mass is binned (shared-memory bins).
// One thread per event, grid-stride: the offsets reads are coalesced, the
// muon reads of consecutive events are contiguous (256-bit AoS loads).
// ============================================================================
// Scattered gathers (the jagged kernels' charges and muon rows): loads with a 64-B
// L2 prefetch size. By default an L2 miss of such a load fetches a 128-B segment
// from DRAM, so a selected event's 64 B of f64 muons cost ~2.1 segments' worth;
// with .L2::64B they cost 1.5 (tools/probe/gatherprobe.cu: 2.35 -> 1.42 GB of DRAM
// reads for 0.96 GB of 64-B records at random rows).
__device__ __forceinline__ void ld_gather(const double* p, double (&r)[4]) {
  asm("ld.global.nc.L1::no_allocate.L2::64B.v4.f64 {%0,%1,%2,%3}, [%4];"
      : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3]) : "l"(p));
}
__device__ __forceinline__ void ld_gather(const float* p, float (&r)[4]) {
  asm("ld.global.nc.L1::no_allocate.L2::64B.v4.f32 {%0,%1,%2,%3}, [%4];"
      : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]) : "l"(p));
}
__device__ __forceinline__ double ld_gather1(const double* p) {
  double r;
  asm("ld.global.nc.L2::64B.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ float ld_gather1(const float* p) {
  float r;
  asm("ld.global.nc.L2::64B.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ int32_t ld_gather1(const int32_t* p) {
  int32_t r;
  asm("ld.global.nc.L2::64B.b32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}

template <typename T, bool AOS>
__device__ __forceinline__ void load_muon(const View4<T>& mu, int64_t j, T (&x)[4]) {
  if constexpr (AOS) {
    T r[4];
    ld_gather(mu.c[0] + 4 * j, r);
#pragma unroll
    for (int c = 0; c < 4; ++c) x[c] = r[c];
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) x[c] = ld_gather1(mu.c[c] + j * mu.s);
  }
}

// U events per thread per iteration, loads batched stage by stage (offsets,
// then charges, then kinematics) so U independent dependency chains are in
// flight per thread instead of one.
template <typename T, bool AOS, int U = 4>
__global__ void __launch_bounds__(256) k_dimuon_histogram(View4<T> mu, const int32_t* __restrict__ q,
                                                          const int64_t* __restrict__ offsets, int64_t n_events,
                                                          HistParams hp, unsigned long long* __restrict__ bins,
                                                          T* __restrict__ m_out) {
  extern __shared__ unsigned int shd[];
  const int nb2 = hp.nbins + 2;
  for (int b = threadIdx.x; b < nb2; b += blockDim.x) shd[b] = 0u;
  __syncthreads();
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e0 < n_events; e0 += nthr * U) {
    int64_t o[U];
    bool two[U], sel[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + u * nthr;
      two[u] = false;
      o[u] = 0;
      if (e < n_events) {
        o[u] = __ldg(offsets + e);
        two[u] = __ldg(offsets + e + 1) - o[u] == 2;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) sel[u] = two[u] && (int64_t)__ldg(q + o[u]) * (int64_t)__ldg(q + o[u] + 1) < 0;
    T a[U][4], b[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (sel[u]) {
        load_muon<T, AOS>(mu, o[u], a[u]);
        load_muon<T, AOS>(mu, o[u] + 1, b[u]);
      }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + u * nthr;
      if (e >= n_events) break;
      T M = T(NAN);
      if (sel[u]) {
        M = event_mass<T, C_PTETAPHIM>(a[u], b[u]);
        atomicAdd(&shd[find_bin(M, hp)], 1u);
      }
      if (m_out) m_out[e] = M;
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb2; b += blockDim.x) {
    unsigned int c = shd[b];
    if (c) hist_flush(bins, hp, b, c);
  }
}

// ============================================================================
// Jagged dimuon with stream compaction (default). Only ~15 % of the events
// of the muon recipe are selected, so a one-lane-per-event kernel runs the
// mass arithmetic with ~5 of 32 lanes active (the warp pays for all 32) and
// streams every muon's kinematics although only the selected pairs' are
// needed. Here a CTA takes a tile of ET events and
//   1. copies offsets[e0 .. e0+ET] into shared memory (coalesced),
//   2. selects: count == 2, then the two charges (4-B gathers from a narrow
//      address range), sign(q0) != sign(q1) (64-bit product: no overflow);
//      selected events are appended to a shared-memory list with one
//      warp-aggregated atomic per warp; unselected ones get NaN in m_out,
//   3. all NT threads walk the compacted list: both muons of U entries are
//      gathered at once (LDG.256 per f64 muon: memory-level parallelism),
//      the mass is computed with every lane busy, and binned privately.
// HBM traffic is the offsets, the charge sectors of 2-muon events and only
// the selected pairs' kinematics. Several CTAs per SM overlap the phases.
// ============================================================================
template <typename T, bool AOS, int ET, int NT, int U = 1, int MINB = 4>
__global__ void __launch_bounds__(NT, MINB) k_dimuon_compact(View4<T> mu, const int32_t* __restrict__ q,
                                                        const int64_t* __restrict__ offsets, int64_t n_events,
                                                        HistParams hp, unsigned long long* __restrict__ bins,
                                                        T* __restrict__ m_out) {
  static_assert(ET % NT == 0 && ET <= 65536, "tile geometry");
  constexpr int EPT = ET / NT;
  extern __shared__ __align__(128) unsigned char smem[];
  int64_t* s_off = reinterpret_cast<int64_t*>(smem);                  // ET + 1 offsets
  uint16_t* s_list = reinterpret_cast<uint16_t*>(s_off + ET + 2);     // selected event-local indices
  unsigned int* s_hist = reinterpret_cast<unsigned int*>(s_list + ET);
  __shared__ int s_n;
  const int nb2 = hp.nbins + 2;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int b = tid; b < nb2; b += NT) s_hist[b] = 0u;
  const int64_t ntiles = (n_events + ET - 1) / ET;
  // Offsets of a tile: EPT+1 loads per thread, all in flight together. The next
  // tile's are issued before this tile's gather phase (software pipelining), so
  // their latency hides behind the muon gathers and the mass arithmetic.
  int64_t r[EPT + 1];
  auto load_offsets = [&](int64_t tile) {
    const int64_t e0 = tile * ET;
    const int ne = (int)(n_events - e0 < ET ? n_events - e0 : ET);
#pragma unroll
    for (int k = 0; k <= EPT; ++k) {
      const int i = tid + k * NT;
      r[k] = (tile < ntiles && i <= ne) ? __ldg(offsets + e0 + i) : 0;
    }
  };
  load_offsets(blockIdx.x);
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t e0 = tile * ET;
    const int ne = (int)(n_events - e0 < ET ? n_events - e0 : ET);
    if (tid == 0) s_n = 0;
#pragma unroll
    for (int k = 0; k <= EPT; ++k)
      if (tid + k * NT <= ne) s_off[tid + k * NT] = r[k];
    __syncthreads();
    int32_t qa[EPT], qb[EPT];
    bool two[EPT];
#pragma unroll
    for (int k = 0; k < EPT; ++k) {  // all charge gathers of this thread in flight together
      const int el = tid + k * NT;
      two[k] = el < ne && s_off[el + 1] - s_off[el] == 2;
      qa[k] = qb[k] = 0;
      if (two[k]) {
        qa[k] = ld_gather1(q + s_off[el]);
        qb[k] = ld_gather1(q + s_off[el] + 1);
      }
    }
    if constexpr (sizeof(T) == 4) {
      // f32: compaction once per thread, not once per event — the thread's selected
      // events as a bit mask, a warp-inclusive scan of the counts (5 shuffles), one
      // shared atomic per warp for the warp's block of the list (the per-event ballot,
      // leader atomic and broadcast below cost ~45 instructions per event). 0.542 ->
      // 0.524 ms at 1e8. For f64 it measured slower (0.664 -> 0.788 ms: more spills
      // under the 48-register cap that 5 CTAs/SM need), so f64 keeps the per-event form.
      unsigned int mask = 0u;
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const int el = tid + k * NT;
        // q0 q1 < 0 (the oracle's 64-bit product, R21) <=> opposite signs, neither zero
        const bool sel = two[k] & ((qa[k] ^ qb[k]) < 0) & (qa[k] != 0) & (qb[k] != 0);
        mask |= (unsigned int)sel << k;
        if (!sel && m_out && el < ne) m_out[e0 + el] = T(NAN);
      }
      const int cnt = __popc(mask);
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      int base = 0;
      if (lane == 31 && incl) base = atomicAdd(&s_n, incl);
      base = __shfl_sync(0xffffffffu, base, 31) + incl - cnt;
#pragma unroll
      for (int k = 0; k < EPT; ++k)
        if (mask & (1u << k)) s_list[base++] = (uint16_t)(tid + k * NT);
    } else {
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const int el = tid + k * NT;
        const bool sel = two[k] && (int64_t)qa[k] * (int64_t)qb[k] < 0;
        const unsigned int bal = __ballot_sync(0xffffffffu, sel);
        int base = 0;
        if (lane == 0 && bal) base = atomicAdd(&s_n, __popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (sel) s_list[base + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)el;
        else if (m_out && el < ne) m_out[e0 + el] = T(NAN);
      }
    }
    __syncthreads();
    const int n = s_n;
    load_offsets(tile + gridDim.x);
    for (int j0 = tid; j0 < n; j0 += NT * U) {
      T a[U][4], b[U][4];
      int el[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = j0 + u * NT;
        el[u] = j < n ? (int)s_list[j] : -1;
        if (el[u] >= 0) {
          const int64_t o = s_off[el[u]];
          load_muon<T, AOS>(mu, o, a[u]);
          load_muon<T, AOS>(mu, o + 1, b[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (el[u] < 0) break;
        const T M = event_mass<T, C_PTETAPHIM>(a[u], b[u]);
        atomicAdd(&s_hist[find_bin(M, hp)], 1u);
        if (m_out) m_out[e0 + el[u]] = M;
      }
    }
    __syncthreads();  // s_off, s_list and s_n are reused by the next tile
  }
  for (int b = tid; b < nb2; b += NT) {
    const unsigned int c = s_hist[b];
    if (c) hist_flush(bins, hp, b, c);
  }
}

template <int ET>
constexpr size_t dimuon_compact_smem(int nb2) {
  return (size_t)(ET + 2) * 8 + (size_t)ET * 2 + (size_t)nb2 * 4;
}

// ============================================================================
// Jagged dimuon with a carried compaction list and an L2 prefetch pipeline
// (default since round 2; k_dimuon_compact above is kept for A/B runs).
// Measured against k_dimuon_compact (tools/probe/dimuon3.cu, 1e8 events):
// f64 0.660 -> 0.46 ms, f32 0.50 -> 0.39 ms, bins bit-equal. Per CTA tile of
// ET events:
//   A. select: thread t takes EPT CONSECUTIVE events, so their EPT+1 offsets
//      are EPT/4 256-bit loads and their charges a narrow window of the charge
//      column (L1 hits for neighbouring events); q0 q1 < 0 (the 64-bit product
//      of R21, as a sign test) -> a bit mask; one warp scan and one shared
//      atomic per warp append the selected muon offsets to a CIRCULAR list;
//   B. mass: the list entries appended BEFORE this tile's selection are
//      walked in full passes of NT entries (every lane busy); the remainder
//      (< NT) is carried to the next tile, the last iteration drains it.
// The memory system runs ahead of both: thread NT-1 bulk-prefetches
// (cp.async.bulk.prefetch.L2) the offsets of the CTA's tile two steps ahead
// and the charge range of the next tile, so phase A reads L2, not DRAM.
// The list holds <= (NT - 1) carried + 2 ET entries (CAP: the next power of
// two). Entries are 32-bit muon offsets relative to offsets[0] when the
// launch's muons span < 2^32 (the common case: half the shared memory of
// 64-bit entries, which leaves L1 room for the charge window — f64 0.507 ->
// 0.457 ms, f32 0.454 -> 0.398 ms in the probe); otherwise the same code runs
// with 64-bit entries on half-size tiles in the same shared memory (a uniform
// branch on offsets[n] - offsets[0], read by every CTA). The event of an entry
// (for m_out) is packed as (CTA step << log2 ET) | event-in-tile in 32 bits.
// ============================================================================
template <int ET, int NT>
struct DimuonCarry {
  static constexpr int need = 2 * ET + NT;
  static constexpr int CAP = need <= 1024 ? 1024 : need <= 2048 ? 2048 : need <= 4096 ? 4096 : need <= 8192 ? 8192 : 16384;
  static_assert(need <= 16384, "list capacity");
  // 32-bit entries at ET (+ 32-bit events for m_out); the 64-bit fallback at ET / 2 fits the same bytes
  static constexpr size_t smem(int nb2, bool want_m) { return (size_t)CAP * 4 * (want_m ? 2 : 1) + (size_t)nb2 * 4; }
};

// L2 bulk prefetch of the 16-byte granules covering [a, b) (at most 64 KB: a
// hint only; every granule touched holds a byte of [a, b), so no page outside
// the caller's range is addressed).
__device__ __forceinline__ void prefetch_l2_range(const void* a, const void* b) {
  const uintptr_t lo = (uintptr_t)a & ~(uintptr_t)15;
  uintptr_t hi = ((uintptr_t)b + 15) & ~(uintptr_t)15;
  if (hi > lo + 65536) hi = lo + 65536;
  if (hi > lo)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"((uint32_t)(hi - lo)) : "memory");
}

// The tile loop of k_dimuon_carry with list entries of type LT (uint32_t: muon
// offset - mbase; int64_t: the muon offset itself, mbase = 0).
template <typename T, bool AOS, int ET, int NT, bool WANT_M, bool VOFF, typename LT>
__device__ __forceinline__ void dimuon_carry_tiles(const View4<T>& mu, const int32_t* __restrict__ q,
                                                   const int64_t* __restrict__ offsets, int64_t n_events,
                                                   const HistParams& hp, unsigned int* s_hist, unsigned char* smem,
                                                   int* s_tail, T* __restrict__ m_out, int64_t mbase) {
  constexpr int EPT = ET / NT;
  constexpr int CAP = DimuonCarry<ET, NT>::CAP;
  constexpr int LOG2ET = ET == 256 ? 8 : ET == 512 ? 9 : ET == 1024 ? 10 : ET == 2048 ? 11 : 12;
  static_assert(ET % NT == 0 && EPT % 4 == 0 && EPT <= 32 && (1 << LOG2ET) == ET, "tile geometry");
  LT* s_mo = reinterpret_cast<LT*>(smem);                          // muon offset of each list entry
  uint32_t* s_ev = reinterpret_cast<uint32_t*>(s_mo + CAP);         // its event, packed (WANT_M only)
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t ntiles = (n_events + ET - 1) / ET;
  const int64_t G = gridDim.x;
  auto tile_events = [&](int64_t t) { return n_events - t * ET < ET ? n_events - t * ET : (int64_t)ET; };
  if (tid == NT - 1) {  // the offsets of the first two tiles
    for (int64_t t = blockIdx.x; t < ntiles && t < blockIdx.x + 2 * G; t += G)
      prefetch_l2_range(offsets + t * ET, offsets + t * ET + tile_events(t) + 1);
  }
  __syncthreads();
  int head = 0, mark = 0;  // mark: the list tail before this iteration's selection
  uint32_t step = 0;       // this CTA's tile count (the packed event index of m_out)
  for (int64_t tile = blockIdx.x;; tile += G, ++step) {
    const bool have = tile < ntiles;
    if (have) {
      // ---- A: select this tile's events, append them to the list
      const int64_t e0 = tile * ET;
      const int ne = (int)tile_events(tile);
      const int lb = tid * EPT;
      int64_t o[EPT + 1];
      if (VOFF && ne == ET) {
        const int64_t* p = offsets + e0 + lb;
#pragma unroll
        for (int h = 0; h < EPT; h += 4)
          asm("ld.global.nc.L1::no_allocate.v4.s64 {%0,%1,%2,%3}, [%4];"
              : "=l"(o[h]), "=l"(o[h + 1]), "=l"(o[h + 2]), "=l"(o[h + 3])
              : "l"(p + h));
        o[EPT] = __ldg(p + EPT);
      } else {
#pragma unroll
        for (int k = 0; k <= EPT; ++k) o[k] = lb + k <= ne ? __ldg(offsets + e0 + lb + k) : 0;
      }
      int32_t qa[EPT], qb[EPT];
#pragma unroll
      for (int k = 0; k < EPT; ++k) {  // all charge loads of the thread in flight together
        qa[k] = qb[k] = 0;
        if (lb + k < ne && o[k + 1] - o[k] == 2) {
          qa[k] = __ldg(q + o[k]);
          qb[k] = __ldg(q + o[k] + 1);
        }
      }
      unsigned int mask = 0u;
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        // q0 q1 < 0 (the oracle's 64-bit product, R21) <=> opposite signs, neither zero
        const bool sel = ((qa[k] ^ qb[k]) < 0) & (qa[k] != 0) & (qb[k] != 0);
        mask |= (unsigned int)sel << k;
        if (WANT_M && !sel && lb + k < ne) m_out[e0 + lb + k] = T(NAN);
      }
      const int cnt = __popc(mask);
      int incl = cnt;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
      }
      int base = 0;
      if (lane == 31 && incl) base = atomicAdd(s_tail, incl);
      base = __shfl_sync(0xffffffffu, base, 31) + incl - cnt;
#pragma unroll
      for (int k = 0; k < EPT; ++k)
        if (mask & (1u << k)) {
          const int slot = base++ & (CAP - 1);
          s_mo[slot] = (LT)(o[k] - mbase);
          if (WANT_M) s_ev[slot] = (step << LOG2ET) | (uint32_t)(lb + k);
        }
      if (tid == NT - 1) {  // prefetch: the next tile's charges, the offsets two tiles ahead
        const int64_t t1 = tile + G, t2 = tile + 2 * G;
        if (t1 < ntiles)
          prefetch_l2_range(q + __ldg(offsets + t1 * ET), q + __ldg(offsets + t1 * ET + tile_events(t1)));
        if (t2 < ntiles) prefetch_l2_range(offsets + t2 * ET, offsets + t2 * ET + tile_events(t2) + 1);
      }
    }
    __syncthreads();
    // ---- B: masses of the entries [head, mark) in full passes (everything on the last step)
    const int tail = *s_tail;  // stable until the next selection
    const int avail = (have ? mark : tail) - head;
    const int take = have ? avail / NT * NT : avail;
    mark = tail;
    for (int j = tid; j < take; j += NT) {
      const int slot = (head + j) & (CAP - 1);
      const int64_t mo = (int64_t)s_mo[slot] + mbase;
      T a[4], b[4];
      load_muon<T, AOS>(mu, mo, a);
      load_muon<T, AOS>(mu, mo + 1, b);
      const T M = event_mass<T, C_PTETAPHIM>(a, b);
      atomicAdd(&s_hist[find_bin(M, hp)], 1u);
      if (WANT_M) {
        const uint32_t pe = s_ev[slot];
        m_out[(blockIdx.x + (int64_t)(pe >> LOG2ET) * G) * ET + (pe & (ET - 1))] = M;
      }
    }
    head += take;
    if (!have) break;
    __syncthreads();  // the slots consumed here may be refilled by the next selection
  }
}

// VOFF: offsets 32-byte aligned (full tiles take 256-bit offset loads).
template <typename T, bool AOS, int ET, int NT, int MINB, bool WANT_M, bool VOFF>
__global__ void __launch_bounds__(NT, MINB) k_dimuon_carry(View4<T> mu, const int32_t* __restrict__ q,
                                                      const int64_t* __restrict__ offsets, int64_t n_events,
                                                      HistParams hp, unsigned long long* __restrict__ bins,
                                                      T* __restrict__ m_out) {
  static_assert(DimuonCarry<ET / 2, NT>::CAP * (WANT_M ? 12 : 8) <= DimuonCarry<ET, NT>::CAP * (WANT_M ? 8 : 4),
                "the 64-bit fallback list must fit the 32-bit list's bytes");
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned int* s_hist = reinterpret_cast<unsigned int*>(smem + (size_t)DimuonCarry<ET, NT>::CAP * 4 * (WANT_M ? 2 : 1));
  __shared__ int s_tail;
  const int nb2 = hp.nbins + 2;
  for (int b = threadIdx.x; b < nb2; b += NT) s_hist[b] = 0u;
  if (threadIdx.x == 0) s_tail = 0;
  const int64_t first = __ldg(offsets), span = __ldg(offsets + n_events) - first;
  if (span <= (int64_t)0xffffffffu)  // uniform over the grid
    dimuon_carry_tiles<T, AOS, ET, NT, WANT_M, VOFF, uint32_t>(mu, q, offsets, n_events, hp, s_hist, smem, &s_tail,
                                                               m_out, first);
  else
    dimuon_carry_tiles<T, AOS, ET / 2, NT, WANT_M, VOFF, int64_t>(mu, q, offsets, n_events, hp, s_hist, smem,
                                                                  &s_tail, m_out, 0);
  __syncthreads();
  for (int b = threadIdx.x; b < nb2; b += NT) {
    const unsigned int c = s_hist[b];
    if (c) hist_flush(bins, hp, b, c);
  }
}

// ============================================================================
// Jagged dimuon, TMA-fed: the offsets column and the muon column are streamed
// tile by tile (ET events per tile) into a shared-memory ring. A tile's muon
// range [offsets[e0], offsets[e0+ET]) is only known from the offsets, so the
// producer lane reads the two bounds of the NEXT tile with plain loads while
// the current tile's copies are in flight, then issues one bulk copy of the
// offsets (ET+2 entries) and one of the muon range. Tiles with more than
// MAXMU muons (never for the synthetic recipe; possible for real data) set an
// overflow flag and their consumers read the muons from global memory.
// Charges are read with plain cached loads (4 B, only for 2-muon events).
// ============================================================================
template <typename T, int ET_, int MAXMU_, int STAGES_, int NCW_>
struct DimuonTma {
  static constexpr int ET = ET_, MAXMU = MAXMU_, STAGES = STAGES_, NCW = NCW_;
  static constexpr int NCT = NCW * 32, EPT = ET / NCT;
  static constexpr int OFF_BYTES = (ET + 2) * 8;
  static constexpr int MU_BYTES = MAXMU * 4 * (int)sizeof(T);
  static constexpr int Q_BYTES = (MAXMU + 8) * 4;  // charges of [m0 & ~3, round_up(m1, 4))
  static constexpr int STAGE_BYTES = OFF_BYTES + MU_BYTES + Q_BYTES;
  static constexpr int RING_BYTES = STAGES * STAGE_BYTES;
  static constexpr int BAR_BYTES = 2 * STAGES * 8 + STAGES * 32;  // full, empty, per-stage {m0, ov, q0, qov}
  static_assert(ET % NCT == 0 && ET % 2 == 0 && OFF_BYTES % 16 == 0 && STAGE_BYTES % 16 == 0, "tile geometry");
  static size_t smem_bytes(int nb2) { return (size_t)RING_BYTES + BAR_BYTES + (size_t)nb2 * 4; }
};

template <typename T, typename CFG>
__global__ void __launch_bounds__(32 * (CFG::NCW + 1))
    k_dimuon_tma(const T* __restrict__ mu, const int32_t* __restrict__ q, const int64_t* __restrict__ offsets,
                 int64_t n_events, HistParams hp, unsigned long long* __restrict__ bins, T* __restrict__ m_out) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + CFG::RING_BYTES);
  uint64_t* empty = full + CFG::STAGES;
  int64_t* meta = reinterpret_cast<int64_t*>(empty + CFG::STAGES);  // [4s] m0, [4s+1] mu overflow, [4s+2] q0, [4s+3] q overflow
  unsigned int* sh_hist = reinterpret_cast<unsigned int*>(smem + CFG::RING_BYTES + CFG::BAR_BYTES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb2 = hp.nbins + 2;
  for (int b = threadIdx.x; b < nb2; b += blockDim.x) sh_hist[b] = 0u;
  if (threadIdx.x == 0) {
    for (int s = 0; s < CFG::STAGES; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], CFG::NCW);
    }
    tma::fence_barrier_init();
  }
  __syncthreads();
  // full tiles need offsets[e0 .. e0 + ET + 1] (ET + 2 entries) inside [0, n_events]
  const int64_t ntiles = n_events >= CFG::ET + 1 ? (n_events - 1) / CFG::ET : 0;
  auto stage_off = [&](int s) { return reinterpret_cast<int64_t*>(smem + (size_t)s * CFG::STAGE_BYTES); };
  auto stage_mu = [&](int s) { return reinterpret_cast<T*>(smem + (size_t)s * CFG::STAGE_BYTES + CFG::OFF_BYTES); };
  auto stage_q = [&](int s) {
    return reinterpret_cast<int32_t*>(smem + (size_t)s * CFG::STAGE_BYTES + CFG::OFF_BYTES + CFG::MU_BYTES);
  };

  if (warp == 0) {
    if (lane == 0) {  // producer
      const uint64_t pol = tma::policy_evict_first();
      const int64_t n_mu = __ldg(offsets + n_events);  // charges are copied in 16-byte units inside [0, n_mu)
      int64_t t = blockIdx.x;
      int64_t m0 = 0, m1 = 0;
      if (t < ntiles) { m0 = __ldg(offsets + t * CFG::ET); m1 = __ldg(offsets + t * CFG::ET + CFG::ET); }
      for (int it = 0; t < ntiles; t += gridDim.x, ++it) {
        const int s = it % CFG::STAGES, k = it / CFG::STAGES;
        // bounds of the next tile: in flight while this tile is issued
        const int64_t tn = t + gridDim.x;
        int64_t n0 = 0, n1 = 0;
        if (tn < ntiles) { n0 = __ldg(offsets + tn * CFG::ET); n1 = __ldg(offsets + tn * CFG::ET + CFG::ET); }
        if (k > 0) {
          tma::mbar_wait(&empty[s], (k - 1) & 1);
          tma::fence_proxy_async_smem();
        }
        const int64_t cnt = m1 - m0;
        const bool ov = cnt > CFG::MAXMU || cnt < 0;
        const int64_t q0 = m0 & ~(int64_t)3, q1 = (m1 + 3) & ~(int64_t)3;
        const bool qov = ov || q1 > n_mu;
        meta[4 * s] = m0;
        meta[4 * s + 1] = ov;
        meta[4 * s + 2] = q0;
        meta[4 * s + 3] = qov;
        const uint32_t mub = ov ? 0u : (uint32_t)(cnt * 4 * sizeof(T));
        const uint32_t qb = qov ? 0u : (uint32_t)((q1 - q0) * 4);
        tma::mbar_arrive_expect_tx(&full[s], CFG::OFF_BYTES + mub + qb);
        tma::bulk_g2s(stage_off(s), offsets + t * CFG::ET, CFG::OFF_BYTES, &full[s], pol);
        if (mub) tma::bulk_g2s(stage_mu(s), mu + 4 * m0, mub, &full[s], pol);
        if (qb) tma::bulk_g2s(stage_q(s), q + q0, qb, &full[s], pol);
        m0 = n0;
        m1 = n1;
      }
    }
  } else {  // consumers
    const int ctid = threadIdx.x - 32;
    int it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int s = it % CFG::STAGES, k = it / CFG::STAGES;
      tma::mbar_wait(&full[s], k & 1);
      const int64_t* so = stage_off(s);
      const T* sm = stage_mu(s);
      const int64_t m0 = meta[4 * s], q0 = meta[4 * s + 2];
      const bool ov = meta[4 * s + 1] != 0, qov = meta[4 * s + 3] != 0;
      const int32_t* sq = stage_q(s);
      // phase 1: this thread's events out of the stage into registers, then release it
      bool sel[CFG::EPT];
      T a[CFG::EPT][4], b[CFG::EPT][4];
#pragma unroll
      for (int u = 0; u < CFG::EPT; ++u) {
        const int el = u * CFG::NCT + ctid;
        const int64_t o = so[el], kk = so[el + 1] - o;
        const int32_t* pq = qov ? q + o : sq + (o - q0);
        sel[u] = kk == 2 && (int64_t)pq[0] * (int64_t)pq[1] < 0;
        if (sel[u]) {
          const T* pa = ov ? mu + 4 * o : sm + 4 * (o - m0);
#pragma unroll
          for (int c = 0; c < 4; ++c) { a[u][c] = pa[c]; b[u][c] = pa[4 + c]; }
        }
      }
      tma::fence_proxy_async_smem();  // all reads of this stage performed before its release
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(&empty[s]);
      // phase 2: masses and bins while the ring refills
#pragma unroll
      for (int u = 0; u < CFG::EPT; ++u) {
        T M = T(NAN);
        if (sel[u]) {
          M = event_mass<T, C_PTETAPHIM>(a[u], b[u]);
          atomicAdd(&sh_hist[find_bin(M, hp)], 1u);
        }
        if (m_out) m_out[t * CFG::ET + u * CFG::NCT + ctid] = M;
      }
    }
    // events not covered by full tiles: the last CTA, plain loads
    if (blockIdx.x == gridDim.x - 1) {
      for (int64_t e = ntiles * CFG::ET + ctid; e < n_events; e += CFG::NCT) {
        const int64_t o = __ldg(offsets + e), kk = __ldg(offsets + e + 1) - o;
        T M = T(NAN);
        if (kk == 2 && (int64_t)__ldg(q + o) * (int64_t)__ldg(q + o + 1) < 0) {
          T a[4], b[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) { a[c] = mu[4 * o + c]; b[c] = mu[4 * o + 4 + c]; }
          M = event_mass<T, C_PTETAPHIM>(a, b);
          atomicAdd(&sh_hist[find_bin(M, hp)], 1u);
        }
        if (m_out) m_out[e] = M;
      }
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb2; b += blockDim.x) {
    unsigned int c = sh_hist[b];
    if (c) hist_flush(bins, hp, b, c);
  }
}

// ============================================================================
// K1 / K3 on AoS pairs, TMA-fed (the fast path for the paper's LVector* layout).
//
// One CTA = 1 producer warp + NCW consumer warps, persistent over tiles of
// TILE events (static round-robin). The producer's elected lane streams the
// v1 and v2 tiles of each stage into a STAGES-deep shared-memory ring with
// cp.async.bulk (UBLKCP, L2 evict-first) signalling a "full" mbarrier; the
// consumers copy their events out of shared memory, release the stage on an
// "empty" mbarrier (one arrive per warp) and only then do the arithmetic, so
// HBM reads for later stages stay in flight while the FP64 pipe works —
// bytes in flight are set by STAGES x TILE, not by register occupancy.
// ============================================================================

// CREG > 0: warp-specialised register split (setmaxnreg): the producer is a whole
// warpgroup (4 warps, lane 0 of warp 0 issues) shrunk to 24 registers, and the
// consumer warps (NCW a multiple of 4) grow to CREG — registers move inside the
// CTA's launch allocation, so 24 + NCW / 4 * CREG <= (NCW / 4 + 1) * the launch
// count (static_assert below, with the launch count __launch_bounds__ allows).
template <typename T, int TILE_, int STAGES_, int NCW_, int MINB_ = 1, int CREG_ = 0>
struct PairTma {
  static constexpr int TILE = TILE_, STAGES = STAGES_, NCW = NCW_, MINB = MINB_, CREG = CREG_;
  static constexpr int PW = CREG > 0 ? 4 : 1;                    // producer warps
  static constexpr int THREADS = 32 * (NCW + PW);
  static constexpr int PREG = 24;
  static_assert(CREG == 0 || (NCW % 4 == 0 && MINB == 1 && CREG % 8 == 0 &&
                              PREG + NCW / 4 * CREG <= (NCW / 4 + 1) * ((65536 / THREADS) / 8 * 8)),
                "setmaxnreg budget");
  static constexpr int NCT = NCW * 32;
  static constexpr int EPT = TILE / NCT;
  static constexpr int VEC = 4 * (int)sizeof(T);                 // bytes per 4-vector
  static constexpr int HALF = TILE * VEC;                         // one array's tile
  static constexpr int STAGE_BYTES = 2 * HALF;
  static constexpr int RING_BYTES = STAGES * STAGE_BYTES;
  static constexpr int BAR_BYTES = 2 * STAGES * 8;
  static_assert(TILE % NCT == 0, "TILE must be a multiple of the consumer thread count");
  static size_t smem_bytes(int nbins_smem) { return RING_BYTES + BAR_BYTES + (size_t)nbins_smem * 4; }
};

// Read event e's 4-vector from a stage buffer. fp64: two LDS.128 per vector
// (lane stride 32 B: a 2-way bank conflict, cheaper here than the 16 FSELs a
// swizzle costs in these issue-bound kernels).
__device__ __forceinline__ void lds_vec(const double* base, int e, int, double (&x)[4]) {
  const double2* p = reinterpret_cast<const double2*>(base + 4 * e);
  double2 a = p[0], b = p[1];
  x[0] = a.x; x[1] = a.y; x[2] = b.x; x[3] = b.y;
}
__device__ __forceinline__ void lds_vec(const float* base, int e, int, float (&x)[4]) {
  float4 a = *reinterpret_cast<const float4*>(base + 4 * e);
  x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
}

// Extra outputs of the cos theta* mode (PM_HIST_CM_COS, reading R22).
template <typename T> struct CosOut {
  HistParams hc;          // the angle axis
  unsigned long long* bins;
  T* cos_out;             // NULL or n values
};

template <typename T, int COORDS, int MODE, bool WANT_BO>
__device__ __forceinline__ void pair_consume(const T (&a)[4], const T (&b)[4], int64_t i, T* __restrict__ m_out,
                                             unsigned int* sh_hist, const HistParams& hp, const View4o<T>& bo,
                                             unsigned int* sh_cos, const CosOut<T>& co) {
  if constexpr (MODE == PM_MASS) {
    m_out[i] = event_mass<T, COORDS>(a, b);
  } else if constexpr (MODE == PM_BOTH) {
    T ml, mc;
    if constexpr (sizeof(T) == 8 && COORDS == C_PTETAPHIM) {
      if (fast_domain(a[0], a[1], a[2], a[3]) && fast_domain(b[0], b[1], b[2], b[3])) {
        both_masses_fast(a[0], a[1], a[2], a[3], b[0], b[1], b[2], b[3], ml, mc);
      } else {
        ml = event_mass<T, COORDS>(a, b);
        mc = hist_event_mass<T, COORDS, true, false>(a, b, i, bo);
      }
    } else {
      ml = event_mass<T, COORDS>(a, b);
      mc = hist_event_mass<T, COORDS, true, false>(a, b, i, bo);
    }
    atomicAdd(&sh_hist[find_bin(ml, hp)], 1u);
    atomicAdd(&sh_cos[find_bin(mc, co.hc)], 1u);
    if (m_out) m_out[i] = ml;
    if (co.cos_out) co.cos_out[i] = mc;
  } else if constexpr (MODE == PM_HIST_CM_COS) {
    T c;
    T M = hist_event_mass<T, COORDS, true, WANT_BO, true>(a, b, i, bo, &c);
    atomicAdd(&sh_hist[find_bin(M, hp)], 1u);
    atomicAdd(&sh_cos[find_bin(c, co.hc)], 1u);
    if (m_out) m_out[i] = M;
    if (co.cos_out) co.cos_out[i] = c;
  } else {
    T M = hist_event_mass<T, COORDS, MODE == PM_HIST_CM, WANT_BO>(a, b, i, bo);
    atomicAdd(&sh_hist[find_bin(M, hp)], 1u);
    if (m_out) m_out[i] = M;
  }
}

// fp32 CM modes, two events of a thread at once in packed FFMA2/FMUL2/FADD2
// arithmetic (cm_mass_f32_lanes<float2>: the same bits as the scalar path);
// a pair with an event outside the fast domain takes the scalar path.
template <int COORDS, int MODE>
__device__ __forceinline__ void pair_consume_x2(const float (&a0)[4], const float (&b0)[4], const float (&a1)[4],
                                                const float (&b1)[4], int64_t i0, int64_t i1, float* __restrict__ m_out,
                                                unsigned int* sh_hist, const HistParams& hp, const View4o<float>& bo,
                                                unsigned int* sh_cos, const CosOut<float>& co) {
  if (fast_domain(a0[0], a0[1], a0[2], a0[3]) & fast_domain(b0[0], b0[1], b0[2], b0[3]) &
      fast_domain(a1[0], a1[1], a1[2], a1[3]) & fast_domain(b1[0], b1[1], b1[2], b1[3])) {
    constexpr bool COS = MODE == PM_HIST_CM_COS;
    float2 c;
    const float2 A0 = make_float2(a0[0], a1[0]), A1 = make_float2(a0[1], a1[1]), A2 = make_float2(a0[2], a1[2]),
                 A3 = make_float2(a0[3], a1[3]), B0 = make_float2(b0[0], b1[0]), B1 = make_float2(b0[1], b1[1]),
                 B2 = make_float2(b0[2], b1[2]), B3 = make_float2(b0[3], b1[3]);
    float2 M;
    if constexpr (MODE == PM_BOTH) {
      M = pair_mass_f32_lanes<float2>(A0, A1, A2, A3, B0, B1, B2, B3);
      const float2 C = cm_mass_f32_lanes<float2, false, false>(A0, A1, A2, A3, B0, B1, B2, B3, &c, nullptr);
      const int2 bm = find_bin2(M, hp), bc = find_bin2(C, co.hc);
      atomicAdd(&sh_hist[bm.x], 1u);
      atomicAdd(&sh_hist[bm.y], 1u);
      atomicAdd(&sh_cos[bc.x], 1u);
      atomicAdd(&sh_cos[bc.y], 1u);
      if (m_out) {
        m_out[i0] = M.x;
        m_out[i1] = M.y;
      }
      if (co.cos_out) {
        co.cos_out[i0] = C.x;
        co.cos_out[i1] = C.y;
      }
      return;
    } else if constexpr (MODE == PM_MASS || MODE == PM_HIST) {
      M = pair_mass_f32_lanes<float2>(A0, A1, A2, A3, B0, B1, B2, B3);
      if constexpr (MODE == PM_MASS) {
        m_out[i0] = M.x;
        m_out[i1] = M.y;
        return;
      }
    } else {
      M = cm_mass_f32_lanes<float2, COS, false>(A0, A1, A2, A3, B0, B1, B2, B3, &c, nullptr);
    }
    const int2 bm = find_bin2(M, hp);
    atomicAdd(&sh_hist[bm.x], 1u);
    atomicAdd(&sh_hist[bm.y], 1u);
    if (m_out) {
      m_out[i0] = M.x;
      m_out[i1] = M.y;
    }
    if constexpr (COS) {
      const int2 bc = find_bin2(c, co.hc);
      atomicAdd(&sh_cos[bc.x], 1u);
      atomicAdd(&sh_cos[bc.y], 1u);
      if (co.cos_out) {
        co.cos_out[i0] = c.x;
        co.cos_out[i1] = c.y;
      }
    }
  } else {
    pair_consume<float, COORDS, MODE, false>(a0, b0, i0, m_out, sh_hist, hp, bo, sh_cos, co);
    pair_consume<float, COORDS, MODE, false>(a1, b1, i1, m_out, sh_hist, hp, bo, sh_cos, co);
  }
}

// fp64 CM modes, two events of a thread in one branch-free block (both in the
// fast domain): the two independent dependency chains give the scheduler ILP
// on the FP64 pipe. Same arithmetic as the one-event path (bit-identical).
template <int COORDS, int MODE>
__device__ __forceinline__ void pair_consume_x2(const double (&a0)[4], const double (&b0)[4], const double (&a1)[4],
                                                const double (&b1)[4], int64_t i0, int64_t i1,
                                                double* __restrict__ m_out, unsigned int* sh_hist,
                                                const HistParams& hp, const View4o<double>& bo, unsigned int* sh_cos,
                                                const CosOut<double>& co) {
  if (fast_domain(a0[0], a0[1], a0[2], a0[3]) & fast_domain(b0[0], b0[1], b0[2], b0[3]) &
      fast_domain(a1[0], a1[1], a1[2], a1[3]) & fast_domain(b1[0], b1[1], b1[2], b1[3])) {
    constexpr bool COS = MODE == PM_HIST_CM_COS;
    constexpr bool LAB = MODE == PM_MASS || MODE == PM_HIST;
    double c0, c1, M0, M1;
    if constexpr (MODE == PM_BOTH) {
      double C0, C1;  // CM masses
      both_masses_fast(a0[0], a0[1], a0[2], a0[3], b0[0], b0[1], b0[2], b0[3], M0, C0);
      both_masses_fast(a1[0], a1[1], a1[2], a1[3], b1[0], b1[1], b1[2], b1[3], M1, C1);
      atomicAdd(&sh_hist[find_bin(M0, hp)], 1u);
      atomicAdd(&sh_hist[find_bin(M1, hp)], 1u);
      atomicAdd(&sh_cos[find_bin(C0, co.hc)], 1u);
      atomicAdd(&sh_cos[find_bin(C1, co.hc)], 1u);
      if (m_out) {
        m_out[i0] = M0;
        m_out[i1] = M1;
      }
      if (co.cos_out) {
        co.cos_out[i0] = C0;
        co.cos_out[i1] = C1;
      }
      return;
    } else if constexpr (LAB) {
      M0 = pair_mass_fast(a0[0], a0[1], a0[2], a0[3], b0[0], b0[1], b0[2], b0[3]);
      M1 = pair_mass_fast(a1[0], a1[1], a1[2], a1[3], b1[0], b1[1], b1[2], b1[3]);
      if constexpr (MODE == PM_MASS) {
        m_out[i0] = M0;
        m_out[i1] = M1;
        return;
      }
    } else {
      M0 = cm_mass_ptetaphim_fast<double, COS>(a0[0], a0[1], a0[2], a0[3], b0[0], b0[1], b0[2], b0[3], nullptr,
                                               nullptr, &c0);
      M1 = cm_mass_ptetaphim_fast<double, COS>(a1[0], a1[1], a1[2], a1[3], b1[0], b1[1], b1[2], b1[3], nullptr,
                                               nullptr, &c1);
    }
    atomicAdd(&sh_hist[find_bin(M0, hp)], 1u);
    atomicAdd(&sh_hist[find_bin(M1, hp)], 1u);
    if (m_out) {
      m_out[i0] = M0;
      m_out[i1] = M1;
    }
    if constexpr (COS) {
      atomicAdd(&sh_cos[find_bin(c0, co.hc)], 1u);
      atomicAdd(&sh_cos[find_bin(c1, co.hc)], 1u);
      if (co.cos_out) {
        co.cos_out[i0] = c0;
        co.cos_out[i1] = c1;
      }
    }
  } else {
    pair_consume<double, COORDS, MODE, false>(a0, b0, i0, m_out, sh_hist, hp, bo, sh_cos, co);
    pair_consume<double, COORDS, MODE, false>(a1, b1, i1, m_out, sh_hist, hp, bo, sh_cos, co);
  }
}


// SOA = false: each stage holds the v1 and v2 AoS tiles (2 bulk copies);
// SOA = true: the 8 component tiles of v1 and v2 (8 bulk copies), read back
// lane-contiguously (LDS.64 / LDS.32, no bank conflicts).
template <typename T, int COORDS, int MODE, typename CFG, bool WANT_BO = false, bool SOA = false>
__global__ void __launch_bounds__(CFG::THREADS, CFG::MINB) k_pair_tma(View4<T> v1, View4<T> v2,
                                                                 int64_t n, T* __restrict__ m_out, HistParams hp,
                                                                 unsigned long long* __restrict__ bins, View4o<T> bo,
                                                                 CosOut<T> co) {
  extern __shared__ __align__(128) unsigned char smem[];
  T* ring = reinterpret_cast<T*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + CFG::RING_BYTES);
  uint64_t* empty = full + CFG::STAGES;
  unsigned int* sh_hist = reinterpret_cast<unsigned int*>(smem + CFG::RING_BYTES + CFG::BAR_BYTES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb2 = hp.nbins + 2;
  // cos theta* mode: the angle histogram follows the mass histogram in shared memory
  const int nbt = nb2 + ((MODE == PM_HIST_CM_COS || MODE == PM_BOTH) ? co.hc.nbins + 2 : 0);
  unsigned int* sh_cos = sh_hist + nb2;

  if constexpr (MODE != PM_MASS) {
    for (int b = threadIdx.x; b < nbt; b += blockDim.x) sh_hist[b] = 0u;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < CFG::STAGES; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], CFG::NCW);
    }
    tma::fence_barrier_init();
  }
  __syncthreads();

  const int64_t ntiles = n / CFG::TILE;
  constexpr int TV = CFG::TILE * 4;  // scalars per array tile
  if (warp < CFG::PW) {
    if constexpr (CFG::CREG > 0) setmaxnreg_dec<CFG::PREG>();
    if (warp == 0 && lane == 0) {  // producer
      const uint64_t pol = tma::policy_evict_first();
      int s = 0, it = 0;
      uint32_t ph = 1;  // parity of the empty-barrier phase to wait for (round k-1)
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        if (it >= CFG::STAGES) {
          tma::mbar_wait(&empty[s], ph);
          tma::fence_proxy_async_smem();  // consumers' reads before the async-proxy refill
        }
        tma::mbar_arrive_expect_tx(&full[s], CFG::STAGE_BYTES);
        T* dst = ring + (size_t)s * 2 * TV;
        if constexpr (SOA) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            tma::bulk_g2s(dst + c * CFG::TILE, v1.c[c] + t * CFG::TILE, CFG::HALF / 4, &full[s], pol);
            tma::bulk_g2s(dst + TV + c * CFG::TILE, v2.c[c] + t * CFG::TILE, CFG::HALF / 4, &full[s], pol);
          }
        } else {
#ifdef GVX_PROBE_L2_RESIDENT  // tools/probe only: every tile re-reads one of 64 (compute-bound control)
          const int64_t tr = t & 63;
#else
          const int64_t tr = t;
#endif
          tma::bulk_g2s(dst, v1.c[0] + tr * TV, CFG::HALF, &full[s], pol);
          tma::bulk_g2s(dst + TV, v2.c[0] + tr * TV, CFG::HALF, &full[s], pol);
        }
        ++it;
        if (++s == CFG::STAGES) { s = 0; ph ^= 1u; }
      }
    }
  } else {  // consumers
    if constexpr (CFG::CREG > 0) setmaxnreg_inc<CFG::CREG>();
    const int ctid = threadIdx.x - 32 * CFG::PW;
    int s = 0;
    uint32_t ph = 0;  // parity of the full-barrier phase of this round
    // 32-bit tile counter (the launchers keep n / TILE < 2^31): a 64-bit bound spilled to local
    // memory and was reloaded every pass (ncu: LDL + long-scoreboard stall on the loop test)
    const int ntiles32 = (int)ntiles;
    for (int t32 = blockIdx.x; t32 < ntiles32; t32 += gridDim.x) {
      const int64_t t = t32;
      tma::mbar_wait(&full[s], ph);
      const T* src = ring + (size_t)s * 2 * TV;
      T a[CFG::EPT][4], b[CFG::EPT][4];
#pragma unroll
      for (int u = 0; u < CFG::EPT; ++u) {
        const int e = u * CFG::NCT + ctid;
        if constexpr (SOA) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            a[u][c] = src[c * CFG::TILE + e];
            b[u][c] = src[TV + c * CFG::TILE + e];
          }
        } else {
          lds_vec(src, e, lane, a[u]);
          lds_vec(src + TV, e, lane, b[u]);
        }
      }
#if defined(GVX_TUNE) && defined(GVX_RELEASE_BY_DEPENDENCY)
      {  // tuning experiment only: order the release after the loads by a data dependency
        uint32_t d = 0;
#pragma unroll
        for (int u = 0; u < CFG::EPT; ++u)
#pragma unroll
          for (int c = 0; c < 4; ++c) d ^= __float_as_uint((float)a[u][c]) ^ __float_as_uint((float)b[u][c]);
        if (__any_sync(0xffffffffu, d == 0x7f7f7f7fu)) asm volatile("" ::: "memory");
      }
#else
      tma::fence_proxy_async_smem();  // this stage's LDS are performed before its release
#endif
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(&empty[s]);
      // two events per call: packed FP32 for the f32 CM modes, two interleaved FP64 chains for f64
      constexpr bool PACK = COORDS == C_PTETAPHIM && !WANT_BO && CFG::EPT % 2 == 0;
      if constexpr (PACK) {
#pragma unroll
        for (int u = 0; u < CFG::EPT; u += 2)
          pair_consume_x2<COORDS, MODE>(a[u], b[u], a[u + 1], b[u + 1], t * CFG::TILE + u * CFG::NCT + ctid,
                                        t * CFG::TILE + (u + 1) * CFG::NCT + ctid, m_out, sh_hist, hp, bo, sh_cos,
                                        co);
      } else {
#pragma unroll
        for (int u = 0; u < CFG::EPT; ++u)
          pair_consume<T, COORDS, MODE, WANT_BO>(a[u], b[u], t * CFG::TILE + u * CFG::NCT + ctid, m_out, sh_hist,
                                                 hp, bo, sh_cos, co);
      }
      if (++s == CFG::STAGES) { s = 0; ph ^= 1u; }
    }
    // ragged tail (< TILE events): the last CTA, plain loads
    if (blockIdx.x == gridDim.x - 1) {
      for (int64_t i = ntiles * CFG::TILE + ctid; i < n; i += CFG::NCT) {
        T a[4], b[4];
        if constexpr (SOA) {
#pragma unroll
          for (int c = 0; c < 4; ++c) { a[c] = v1.c[c][i]; b[c] = v2.c[c][i]; }
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c) { a[c] = v1.c[0][4 * i + c]; b[c] = v2.c[0][4 * i + c]; }
        }
        pair_consume<T, COORDS, MODE, WANT_BO>(a, b, i, m_out, sh_hist, hp, bo, sh_cos, co);
      }
    }
  }
  if constexpr (MODE != PM_MASS) {
    __syncthreads();
    for (int b = threadIdx.x; b < nbt; b += blockDim.x) {
      unsigned int c = sh_hist[b];
      if (c) {
        if (b < nb2) hist_flush(bins, hp, b, c);
        else atomicAdd(&co.bins[b - nb2], (unsigned long long)c);
      }
    }
    hist_tail(hp);  // pre-reduced cross-GPU sink only (gvx_mass_histogram_peers)
  }
}

// ============================================================================
// The whole bench step in ONE persistent launch (k_step): the fused pair pass
// (PM_BOTH on AoS PtEtaPhiM pairs) and the per-event boost of a second batch
// (AoS vectors, AoS [N][3] velocities) share every SM. The pair pass is bound
// by the FP64 pipe at ~5 TB/s and the boost by HBM, so running them in the same
// CTA lets the memory system stream the boost while the FP64 pipe works on the
// pairs. Warp 0, lane 0 feeds two TMA rings (pair tiles, boost tiles) without
// blocking on either; warps 1..NCW consume pairs exactly as k_pair_tma does
// (same arithmetic, same bits); warps NCW+1..NCW+NBW boost (boost_coef /
// apply_boost as k_boost: same bits) and store with 256-bit STG.
// ============================================================================
// BREG: the boost warps' register count under the step's warp-specialised split
// (the pair CFG has CREG > 0; the boost warps are then whole warpgroups too).
template <typename T, int BT_, int BST_, int NBW_, int BREG_ = 0>
struct BoostRing {
  static constexpr int BT = BT_, BST = BST_, NBW = NBW_, NBT = NBW * 32, BREG = BREG_;
  static constexpr int EPB = BT / NBT;              // boost events per thread per stage
  static constexpr int VB = BT * 4 * (int)sizeof(T);  // vector tile bytes
  static constexpr int BB = BT * 3 * (int)sizeof(T);  // velocity tile bytes
  static constexpr int STAGE_BYTES = VB + BB;
  static constexpr int RING_BYTES = BST * STAGE_BYTES;
  static_assert(BT % NBT == 0 && BB % 16 == 0 && VB % 16 == 0, "boost tile geometry");
};

template <typename CFG, typename BR>
struct StepGeom {
  static constexpr int PW = CFG::PW, THREADS = 32 * (CFG::PW + CFG::NCW + BR::NBW);
  static constexpr int LAUNCH_REG = (65536 / THREADS) / 8 * 8;  // what __launch_bounds__(THREADS, 1) allows
  static_assert(CFG::CREG == 0 ||
                    (BR::NBW % 4 == 0 && BR::BREG % 8 == 0 && BR::BREG >= 24 &&
                     CFG::PREG + CFG::NCW / 4 * CFG::CREG + BR::NBW / 4 * BR::BREG <= THREADS / 128 * LAUNCH_REG),
                "setmaxnreg budget of the step");
};

template <int FROM, int TO>
__device__ __forceinline__ void setmaxnreg_to() {
  if constexpr (TO > FROM) setmaxnreg_inc<TO>();
  if constexpr (TO < FROM) setmaxnreg_dec<TO>();
}

template <typename T, typename CFG, typename BR>
__global__ void __launch_bounds__(StepGeom<CFG, BR>::THREADS, 1)
    k_step(View4<T> v1, View4<T> v2, int64_t n, T* __restrict__ m_out, HistParams hp,
           unsigned long long* __restrict__ bins, CosOut<T> co, const T* __restrict__ bv, const T* __restrict__ bb,
           T* __restrict__ bout, int64_t nb) {
  extern __shared__ __align__(128) unsigned char smem[];
  T* ring = reinterpret_cast<T*>(smem);
  unsigned char* bring = smem + CFG::RING_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(bring + BR::RING_BYTES);
  uint64_t* empty = full + CFG::STAGES;
  uint64_t* bfull = empty + CFG::STAGES;
  uint64_t* bempty = bfull + BR::BST;
  unsigned int* sh_hist = reinterpret_cast<unsigned int*>(bempty + BR::BST);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb2 = hp.nbins + 2;
  const int nbt = nb2 + co.hc.nbins + 2;
  unsigned int* sh_cos = sh_hist + nb2;
  for (int b = threadIdx.x; b < nbt; b += blockDim.x) sh_hist[b] = 0u;
  if (threadIdx.x == 0) {
    for (int s = 0; s < CFG::STAGES; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], CFG::NCW);
    }
    for (int s = 0; s < BR::BST; ++s) {
      tma::mbar_init(&bfull[s], 1);
      tma::mbar_init(&bempty[s], BR::NBW);
    }
    tma::fence_barrier_init();
  }
  __syncthreads();

  const int64_t ntiles = n / CFG::TILE, nbtiles = nb / BR::BT;
  constexpr int TV = CFG::TILE * 4;
  using G = StepGeom<CFG, BR>;
  if (warp < G::PW) {
    if constexpr (CFG::CREG > 0) setmaxnreg_dec<CFG::PREG>();
    if (warp == 0 && lane == 0) {  // producer of both rings; never blocks on one while the other can move
      const uint64_t pol = tma::policy_evict_first();
      int64_t t = blockIdx.x, tb = blockIdx.x;
      int s = 0, it = 0, bs = 0, bit = 0;
      uint32_t ph = 1, bph = 1;
      // each mbarrier poll is a try_wait with a 64 ns suspend-time hint, so a producer
      // waiting on both rings sleeps in the barrier unit instead of spinning on issue slots
      while (t < ntiles || tb < nbtiles) {
        if (t < ntiles && (it < CFG::STAGES || tma::mbar_try_wait_hint(&empty[s], ph, 64u))) {
          if (it >= CFG::STAGES) tma::fence_proxy_async_smem();
          tma::mbar_arrive_expect_tx(&full[s], CFG::STAGE_BYTES);
          T* dst = ring + (size_t)s * 2 * TV;
          tma::bulk_g2s(dst, v1.c[0] + t * TV, CFG::HALF, &full[s], pol);
          tma::bulk_g2s(dst + TV, v2.c[0] + t * TV, CFG::HALF, &full[s], pol);
          ++it;
          if (++s == CFG::STAGES) { s = 0; ph ^= 1u; }
          t += gridDim.x;
        }
        if (tb < nbtiles && (bit < BR::BST || tma::mbar_try_wait_hint(&bempty[bs], bph, 64u))) {
          if (bit >= BR::BST) tma::fence_proxy_async_smem();
          tma::mbar_arrive_expect_tx(&bfull[bs], BR::STAGE_BYTES);
          unsigned char* dst = bring + (size_t)bs * BR::STAGE_BYTES;
          tma::bulk_g2s(dst, bv + tb * BR::BT * 4, BR::VB, &bfull[bs], pol);
          tma::bulk_g2s(dst + BR::VB, bb + tb * BR::BT * 3, BR::BB, &bfull[bs], pol);
          ++bit;
          if (++bs == BR::BST) { bs = 0; bph ^= 1u; }
          tb += gridDim.x;
        }
      }
    }
  } else if (warp < G::PW + CFG::NCW) {  // pair consumers (the k_pair_tma PM_BOTH loop)
    if constexpr (CFG::CREG > 0) setmaxnreg_to<G::LAUNCH_REG, CFG::CREG>();
    const int ctid = threadIdx.x - 32 * G::PW;
    int s = 0;
    uint32_t ph = 0;
    // (64-bit tile counter here: the 32-bit one measured 0.6 % slower for this kernel)
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      tma::mbar_wait(&full[s], ph);
      const T* src = ring + (size_t)s * 2 * TV;
      T a[CFG::EPT][4], b[CFG::EPT][4];
#pragma unroll
      for (int u = 0; u < CFG::EPT; ++u) {
        const int e = u * CFG::NCT + ctid;
        lds_vec(src, e, lane, a[u]);
        lds_vec(src + TV, e, lane, b[u]);
      }
      tma::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(&empty[s]);
      static_assert(CFG::EPT % 2 == 0, "two events per call");
#pragma unroll
      for (int u = 0; u < CFG::EPT; u += 2)
        pair_consume_x2<C_PTETAPHIM, PM_BOTH>(a[u], b[u], a[u + 1], b[u + 1], t * CFG::TILE + u * CFG::NCT + ctid,
                                             t * CFG::TILE + (u + 1) * CFG::NCT + ctid, m_out, sh_hist, hp,
                                             View4o<T>{}, sh_cos, co);
      if (++s == CFG::STAGES) { s = 0; ph ^= 1u; }
    }
    if (blockIdx.x == gridDim.x - 1) {
      for (int64_t i = ntiles * CFG::TILE + ctid; i < n; i += CFG::NCT) {
        T a[4], b[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) { a[c] = v1.c[0][4 * i + c]; b[c] = v2.c[0][4 * i + c]; }
        pair_consume<T, C_PTETAPHIM, PM_BOTH, false>(a, b, i, m_out, sh_hist, hp, View4o<T>{}, sh_cos, co);
      }
    }
  } else {  // boost warps
    if constexpr (CFG::CREG > 0) setmaxnreg_to<G::LAUNCH_REG, BR::BREG>();
    const int btid = threadIdx.x - 32 * (G::PW + CFG::NCW);
    View4o<T> o;
    o.c[0] = bout; o.c[1] = bout + 1; o.c[2] = bout + 2; o.c[3] = bout + 3; o.s = 4;
    int s = 0;
    uint32_t ph = 0;
    for (int64_t tb = blockIdx.x; tb < nbtiles; tb += gridDim.x) {
      tma::mbar_wait(&bfull[s], ph);
      const T* sv = reinterpret_cast<const T*>(bring + (size_t)s * BR::STAGE_BYTES);
      const T* sb = reinterpret_cast<const T*>(bring + (size_t)s * BR::STAGE_BYTES + BR::VB);
      T x[BR::EPB][4], bx[BR::EPB], by[BR::EPB], bz[BR::EPB];
#pragma unroll
      for (int u = 0; u < BR::EPB; ++u) {
        const int e = u * BR::NBT + btid;
        lds_vec(sv, e, lane, x[u]);
        bx[u] = sb[3 * e];
        by[u] = sb[3 * e + 1];
        bz[u] = sb[3 * e + 2];
      }
      tma::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(&bempty[s]);
#pragma unroll
      for (int u = 0; u < BR::EPB; ++u) {
        const int64_t i = tb * BR::BT + u * BR::NBT + btid;
        boost_store<T, true>(o, i, apply_boost(boost_coef(bx[u], by[u], bz[u]), V4<T>{x[u][0], x[u][1], x[u][2], x[u][3]}));
      }
      if (++s == BR::BST) { s = 0; ph ^= 1u; }
    }
    if (blockIdx.x == gridDim.x - 1) {  // ragged boost tail
      for (int64_t i = nbtiles * BR::BT + btid; i < nb; i += BR::NBT) {
        V4<T> x{bv[4 * i], bv[4 * i + 1], bv[4 * i + 2], bv[4 * i + 3]};
        boost_store<T, true>(o, i, apply_boost(boost_coef(bb[3 * i], bb[3 * i + 1], bb[3 * i + 2]), x));
      }
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nbt; b += blockDim.x) {
    unsigned int c = sh_hist[b];
    if (c) {
      if (b < nb2) hist_flush(bins, hp, b, c);
      else atomicAdd(&co.bins[b - nb2], (unsigned long long)c);
    }
  }
}

}  // namespace gvx
