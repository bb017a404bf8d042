// gvx_api.cu — the C ABI (include/gvx.h): validation, layout detection,
// kernel selection and persistent-grid launch. No allocation, no host sync.
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>
#include <stdint.h>

#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "../../include/gvx.h"
#include "gvx_kernels.cuh"

using namespace gvx;

namespace {

thread_local std::string g_last_cuda_error = "no error";

gvx_status cuda_fail(cudaError_t e) {
  g_last_cuda_error = cudaGetErrorString(e);
  return GVX_ERR_CUDA;
}

// Per-device SM count, filled once (the only library state).
constexpr int kMaxDevices = 64;
std::atomic<int> g_sm_count[kMaxDevices];

int sm_count() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return 148;
  int v = g_sm_count[dev].load(std::memory_order_relaxed);
  if (v > 0) return v;
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
  g_sm_count[dev].store(sms, std::memory_order_relaxed);
  return sms;
}

// Per (kernel, device, dynamic smem) occupancy, queried once and cached
// (mutex-protected; host-side only). Also raises the kernel's dynamic shared
// memory limit the first time a size above 48 KB is requested.
std::mutex g_occ_mu;
std::map<std::tuple<const void*, int, size_t, int>, int> g_occ;
// Largest dynamic shared memory opted in per (kernel, device): the attribute
// is only ever raised, so a later call with fewer bins cannot invalidate a
// cached launch configuration that needs more.
std::map<std::pair<const void*, int>, size_t> g_smem_optin;

template <typename K>
int blocks_per_sm(K kernel, int block, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  auto key = std::make_tuple((const void*)kernel, dev, smem, block);
  {
    std::lock_guard<std::mutex> lk(g_occ_mu);
    auto it = g_occ.find(key);
    if (it != g_occ.end()) return it->second;
    if (smem > 48 * 1024) {
      size_t& cur = g_smem_optin[std::make_pair((const void*)kernel, dev)];
      if (smem > cur) {
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cur = smem;
      }
    }
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem) != cudaSuccess) {
    per_sm = 0;
    cudaGetLastError();  // clear only the error this query raised
  }
  if (per_sm < 1) per_sm = 0;
  std::lock_guard<std::mutex> lk(g_occ_mu);
  g_occ[key] = per_sm;
  return per_sm;
}

// Persistent grid: enough CTAs to fill every SM at the kernel's occupancy,
// never more than the work needs.
template <typename K>
int grid_for(K kernel, int block, size_t smem, int64_t work_items_per_block_pass, int64_t items) {
  int per_sm = blocks_per_sm(kernel, block, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t full = (int64_t)sm_count() * per_sm;
  int64_t need = (items + work_items_per_block_pass - 1) / work_items_per_block_pass;
  if (need < 1) need = 1;
  return (int)(need < full ? need : full);
}

inline bool aligned(const void* p, size_t a) { return ((uintptr_t)p % a) == 0; }

size_t dsize(gvx_dtype d) { return d == GVX_F64 ? 8 : 4; }

bool valid_dtype(gvx_dtype d) { return d == GVX_F32 || d == GVX_F64; }
bool valid_coords(gvx_coords c) {
  return c == GVX_PTETAPHIM || c == GVX_PXPYPZE || c == GVX_PXPYPZM || c == GVX_PTETAPHIE;
}

template <int NC, typename V>
bool view_ok(const V* v, size_t es) {
  if (!v || v->stride < 1) return false;
  for (int k = 0; k < NC; ++k)
    if (!v->c[k] || !aligned(v->c[k], es)) return false;
  return true;
}

// Layout classification of an input 4-vector view (see gvx_kernels.cuh).
template <typename V>
int classify(const V* v, size_t es) {
  const char* b = (const char*)v->c[0];
  bool contiguous_aos = v->stride == 4;
  for (int k = 1; k < 4; ++k) contiguous_aos = contiguous_aos && (const char*)v->c[k] == b + k * es;
  if (contiguous_aos && aligned(b, 32)) return L_AOS;  // 256-bit loads need 32-byte alignment
  if (v->stride == 1) {
    bool ok = true;
    for (int k = 0; k < 4; ++k) ok = ok && aligned(v->c[k], 32);
    if (ok) return L_SOA;
  }
  return L_GEN;
}

template <typename T>
View4<T> mk4(const gvx_vec4_cview* v) {
  View4<T> r;
  for (int k = 0; k < 4; ++k) r.c[k] = (const T*)v->c[k];
  r.s = v->stride;
  return r;
}
template <typename T>
View4o<T> mk4o(const gvx_vec4_view* v) {
  View4o<T> r;
  for (int k = 0; k < 4; ++k) r.c[k] = v ? (T*)v->c[k] : nullptr;
  r.s = v ? v->stride : 1;
  return r;
}
template <typename T>
View3<T> mk3(const gvx_vec3_cview* v) {
  View3<T> r;
  for (int k = 0; k < 3; ++k) r.c[k] = v ? (const T*)v->c[k] : nullptr;
  r.s = v ? v->stride : 1;
  return r;
}

constexpr int kBlock = 256;

// GVX_DISABLE_TMA=1 routes AoS pairs to the LDG kernels (A/B measurements).
bool tma_enabled() {
  static const bool on = [] {
    const char* e = getenv("GVX_DISABLE_TMA");
    return !(e && e[0] == '1');
  }();
  return on;
}

// Which AoS pair kernels take the TMA ring by default. Measured on B200
// (profiles/r01/sweep_f64_variants*.jsonl): every fp64 pair kernel (the
// ring frees the registers the LDG kernels spend on loads in flight, so one
// CTA of 29-32 warps keeps the FP64 pipe fed) and the fp32 histograms
// (profiles/r01/sweep_f32_variants.jsonl); the fp32 mass kernel runs faster
// from registers (LDG.256). GVX_FORCE_TMA=1 routes every AoS pair kernel
// through the ring (tested).
bool force_tma() {
  static const bool force = [] {
    const char* e = getenv("GVX_FORCE_TMA");
    return e && e[0] == '1';
  }();
  return force;
}
// GVX_NO_STEP_KERNEL=1: gvx_pair_histograms_boost runs as its two calls (A/B runs;
// read once, like the other switches).
bool step_kernel_enabled() {
  static const bool on = [] { return getenv("GVX_NO_STEP_KERNEL") == nullptr; }();
  return on;
}
template <typename T, int MODE>
bool tma_preferred() {
  return force_tma() || sizeof(T) == 8 || MODE != PM_MASS;
}

// ------------------------------------------------------- TMA pair stream ----
// Ring geometry per (dtype, mode), from the B200 sweeps in profiles/r01/
// (sweep_f64_variants*.jsonl): one CTA per SM with 28-31 consumer warps and a
// 2-3 stage ring of 57-62 KB stages beat 2-3 smaller CTAs, because the fp64
// consumers need warps (FP64 latency) more than ring depth.
template <typename T, int MODE> struct TmaCfgOf;
template <int MODE> struct TmaCfgOf<double, MODE> { using type = PairTma<double, 896, 2, 28, 1>; };
// fp64 CM: 24 consumer warps x 2 events each, run as two interleaved chains
// (pair_consume_x2): 1.16 vs 1.24 ms for 31 warps x 1 event
// (profiles/r01/sweep_f64_cm_x2.jsonl). Since round 2 (session 3) with the fused pass's
// setmaxnreg split (4-warp producer at 24 registers, consumers at 80): CM histogram
// 1.14-1.16 -> 1.12-1.13 ms, peaked CM histogram 1.20-1.26 -> 1.17-1.22 ms (same-box A/B,
// profiles/r02/cm_creg_ab.jsonl).
template <> struct TmaCfgOf<double, PM_HIST_CM> { using type = PairTma<double, 1536, 2, 24, 1, 80>; };
// fp64 lab histogram: 20 warps x 2 interleaved events, 0.904 vs 0.934 ms (same sweep)
template <> struct TmaCfgOf<double, PM_HIST> { using type = PairTma<double, 1280, 2, 20, 1>; };
template <> struct TmaCfgOf<double, PM_HIST_CM_COS> { using type = PairTma<double, 1536, 2, 24, 1, 80>; };
template <> struct TmaCfgOf<double, PM_BOTH> { using type = PairTma<double, 1536, 2, 24, 1, 80>; };
template <int MODE> struct TmaCfgOf<float, MODE> { using type = PairTma<float, 896, 4, 28, 1>; };
template <> struct TmaCfgOf<float, PM_HIST_CM> { using type = PairTma<float, 1792, 3, 28, 1>; };
template <> struct TmaCfgOf<float, PM_HIST_CM_COS> { using type = PairTma<float, 1792, 3, 28, 1>; };
template <> struct TmaCfgOf<float, PM_BOTH> { using type = PairTma<float, 1792, 3, 28, 1>; };

#if defined(GVX_TUNE) || defined(GVX_STEP_ALT)
// Tuning build only (tools/libgvx_tune.so): GVX_TMA_CFG / GVX_LDG_CFG pick
// alternative tile / ring / occupancy variants of the f64 kernels.
int tune_env(const char* name) {
  const char* e = getenv(name);
  return e ? atoi(e) : 0;
}
#endif

// AoS pair kernels (mass, lab histogram, CM histogram) through the TMA ring.
// Returns GVX_ERR_UNSUPPORTED when the histogram does not fit beside the ring
// in shared memory (the caller then uses the LDG kernel).
template <typename T, int C, int MODE, typename CFG>
gvx_status launch_pair_tma_cfg(const gvx_vec4_cview* v1, const gvx_vec4_cview* v2, int64_t n, void* m_out,
                               const HistParams& hp, unsigned long long* bins, const gvx_vec4_view* bo,
                               cudaStream_t s, const CosOut<T>& co = CosOut<T>{}) {
  // AoS (paper layout) or SoA with 16-byte aligned component arrays; else not handled here.
  const bool soa = classify(v1, sizeof(T)) == L_SOA && classify(v2, sizeof(T)) == L_SOA;
  if (!soa && !(classify(v1, sizeof(T)) == L_AOS && classify(v2, sizeof(T)) == L_AOS)) return GVX_ERR_UNSUPPORTED;
  const int nbs =
      MODE == PM_MASS ? 0 : hp.nbins + 2 + ((MODE == PM_HIST_CM_COS || MODE == PM_BOTH) ? co.hc.nbins + 2 : 0);
  const size_t sm = CFG::smem_bytes(nbs);
  if (sm > 227 * 1024) return GVX_ERR_UNSUPPORTED;
  auto k = soa ? k_pair_tma<T, C, MODE, CFG, false, true> : k_pair_tma<T, C, MODE, CFG, false, false>;
  const int block = CFG::THREADS;
  int per_sm = blocks_per_sm(k, block, sm);
  if (per_sm < 1) return GVX_ERR_UNSUPPORTED;
  const int64_t ntiles = n / CFG::TILE;
  int64_t full = (int64_t)sm_count() * per_sm;
  int grid = (int)(ntiles < 1 ? 1 : (ntiles < full ? ntiles : full));
  View4o<T> bov = mk4o<T>(bo);
  // Per-CTA uint32 counters: one launch covers at most grid * 2^31 events.
  int64_t chunk = MODE == PM_MASS ? n : ((int64_t)grid << 31);
  const int64_t max_chunk = (int64_t)INT32_MAX * CFG::TILE;  // the kernel counts tiles in 32 bits
  if (chunk > max_chunk) chunk = max_chunk;
  for (int64_t off = 0; off < n; off += chunk) {
    int64_t cn = n - off < chunk ? n - off : chunk;
    View4o<T> bo2 = bov;
    if (bo)
      for (int c = 0; c < 4; ++c) bo2.c[c] += 2 * off * bo2.s;
    View4<T> a = mk4<T>(v1), b = mk4<T>(v2);
    for (int c = 0; c < 4; ++c) {
      a.c[c] += off * a.s;
      b.c[c] += off * b.s;
    }
    CosOut<T> co2 = co;
    if (co2.cos_out) co2.cos_out += off;
    k<<<grid, block, sm, s>>>(a, b, cn, m_out ? (T*)m_out + off : nullptr, hp, bins, bo2, co2);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GVX_OK : cuda_fail(e);
}

template <typename T, int C, int MODE>
gvx_status launch_pair_tma(const gvx_vec4_cview* v1, const gvx_vec4_cview* v2, int64_t n, void* m_out,
                           const HistParams& hp, unsigned long long* bins, const gvx_vec4_view* bo, cudaStream_t s,
                           const CosOut<T>& co = CosOut<T>{}) {
#ifdef GVX_TUNE
  if constexpr (sizeof(T) == 8 && C == C_PTETAPHIM) {
    switch (tune_env("GVX_TMA_CFG")) {
      case 1: return launch_pair_tma_cfg<T, C, MODE, PairTma<double, 256, 4, 8, 3>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 2: return launch_pair_tma_cfg<T, C, MODE, PairTma<double, 512, 2, 8, 3>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 3: return launch_pair_tma_cfg<T, C, MODE, PairTma<double, 256, 3, 8, 4>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 4: return launch_pair_tma_cfg<T, C, MODE, PairTma<double, 512, 6, 16, 1>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 5: return launch_pair_tma_cfg<T, C, MODE, PairTma<double, 256, 6, 8, 2>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 6: return launch_pair_tma_cfg<T, C, MODE, PairTma<double, 768, 4, 24, 1>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 7: return launch_pair_tma_cfg<T, C, MODE, PairTma<double, 640, 5, 20, 1>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 8: return launch_pair_tma_cfg<T, C, MODE, PairTma<double, 896, 3, 28, 1>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 9: return launch_pair_tma_cfg<T, C, MODE, PairTma<double, 992, 3, 31, 1>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 10: return launch_pair_tma_cfg<T, C, MODE, PairTma<double, 448, 3, 14, 2>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 11: return launch_pair_tma_cfg<T, C, MODE, PairTma<double, 896, 2, 28, 1>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 12: return launch_pair_tma_cfg<T, C, MODE, PairTma<double, 1024, 3, 16, 1>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 13: return launch_pair_tma_cfg<T, C, MODE, PairTma<double, 1280, 2, 20, 1>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 14: return launch_pair_tma_cfg<T, C, MODE, PairTma<double, 1536, 2, 24, 1>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 15: return launch_pair_tma_cfg<T, C, MODE, PairTma<double, 1664, 2, 26, 1>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 16: return launch_pair_tma_cfg<T, C, MODE, PairTma<double, 1408, 2, 22, 1>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 17: return launch_pair_tma_cfg<T, C, MODE, PairTma<double, 1152, 3, 18, 1>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 18: return launch_pair_tma_cfg<T, C, MODE, PairTma<double, 1536, 2, 12, 1>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 19: return launch_pair_tma_cfg<T, C, MODE, PairTma<double, 1536, 2, 24, 1>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      // warp-specialised register split (setmaxnreg): producer warpgroup at 24, consumers at CREG
      case 20: return launch_pair_tma_cfg<T, C, MODE, PairTma<double, 1536, 2, 24, 1, 80>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 21: return launch_pair_tma_cfg<T, C, MODE, PairTma<double, 1024, 3, 16, 1, 112>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 22: return launch_pair_tma_cfg<T, C, MODE, PairTma<double, 1280, 2, 20, 1, 88>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 23: return launch_pair_tma_cfg<T, C, MODE, PairTma<double, 1280, 2, 20, 1>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      default: break;
    }
  }
  if constexpr (sizeof(T) == 4 && C == C_PTETAPHIM) {
    switch (tune_env("GVX_TMA_CFG32")) {
      case 1: return launch_pair_tma_cfg<T, C, MODE, PairTma<float, 1792, 3, 28, 1>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 2: return launch_pair_tma_cfg<T, C, MODE, PairTma<float, 896, 4, 28, 1>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 3: return launch_pair_tma_cfg<T, C, MODE, PairTma<float, 1024, 3, 16, 1>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 4: return launch_pair_tma_cfg<T, C, MODE, PairTma<float, 768, 4, 24, 1>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 5: return launch_pair_tma_cfg<T, C, MODE, PairTma<float, 512, 4, 16, 2>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 6: return launch_pair_tma_cfg<T, C, MODE, PairTma<float, 1536, 4, 24, 1>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 7: return launch_pair_tma_cfg<T, C, MODE, PairTma<float, 1280, 5, 20, 1>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 8: return launch_pair_tma_cfg<T, C, MODE, PairTma<float, 1024, 6, 16, 1>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 9: return launch_pair_tma_cfg<T, C, MODE, PairTma<float, 1792, 3, 28, 1, 64>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 10: return launch_pair_tma_cfg<T, C, MODE, PairTma<float, 1536, 4, 24, 1, 72>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      case 11: return launch_pair_tma_cfg<T, C, MODE, PairTma<float, 1280, 4, 20, 1, 88>>(v1, v2, n, m_out, hp, bins, bo, s, co);
      default: break;
    }
  }
#endif
  if constexpr (sizeof(T) == 4 && MODE == PM_HIST) {
    // SoA views: 8 component copies per stage; the 2-event packed ring measured faster there
    // (0.455 vs 0.496 ms at 1e8, profiles/r01/sweep_f32_lab_packed.jsonl)
    if (classify(v1, sizeof(T)) == L_SOA && classify(v2, sizeof(T)) == L_SOA)
      return launch_pair_tma_cfg<T, C, MODE, PairTma<float, 1792, 3, 28, 1>>(v1, v2, n, m_out, hp, bins, bo, s, co);
  }
  return launch_pair_tma_cfg<T, C, MODE, typename TmaCfgOf<T, MODE>::type>(v1, v2, n, m_out, hp, bins, bo, s, co);
}

// ---------------------------------------------------------------- mass ------
template <typename T, int C, int L>
gvx_status launch_mass(const gvx_vec4_cview* v1, const gvx_vec4_cview* v2, void* m, int64_t n, cudaStream_t s) {
  constexpr int U = (L == L_AOS && sizeof(T) == 8) ? 2 : 1;
  constexpr int G = Group<T, L>::G;
  // f64 AoS: 64-register cap (4 CTAs/SM) measured fastest (sweep ldg1/ldg2).
  // (if constexpr: instantiate the capped variant only where it is used.)
  auto k = k_invariant_mass<T, C, L, U>;
  if constexpr (sizeof(T) == 8 && L == L_AOS) k = k_invariant_mass<T, C, L, U, 4>;
#ifdef GVX_TUNE
  if constexpr (sizeof(T) == 8 && L == L_AOS && C == C_PTETAPHIM) {
    int v = tune_env("GVX_LDG_CFG");
    if (v == 1) k = k_invariant_mass<T, C, L, U, 4>;
    if (v == 2) k = k_invariant_mass<T, C, L, 1, 4>;
    if (v == 3) k = k_invariant_mass<T, C, L, 1, 1>;
  }
#endif
  int grid = grid_for(k, kBlock, 0, (int64_t)kBlock * U * G, n);
  k<<<grid, kBlock, 0, s>>>(mk4<T>(v1), mk4<T>(v2), (T*)m, n);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GVX_OK : cuda_fail(e);
}

template <typename T, int C>
gvx_status dispatch_mass(const gvx_vec4_cview* v1, const gvx_vec4_cview* v2, void* m, int64_t n, cudaStream_t s) {
  int l1 = classify(v1, sizeof(T)), l2 = classify(v2, sizeof(T));
  int L = (l1 == l2) ? l1 : L_GEN;
  if (L == L_AOS && !aligned(m, Group<T, L_AOS>::G * sizeof(T))) L = L_GEN;  // vector stores
  if (L == L_SOA && !aligned(m, Group<T, L_SOA>::G * sizeof(T))) L = L_GEN;
  // Below ~1e6 pairs a ring with a handful of tiles per CTA cannot overlap its copies with its
  // arithmetic; the register kernel's many small CTAs are faster there (f64 AoS: 6.8 vs 8.9 us at
  // 1e4, 11.1 vs 13.3 us at 3e5; equal at 1e6; the ring wins from 3e6 — CFG2 sweep).
  const bool small = n < (int64_t(1) << 20) && !force_tma();
  if constexpr (C == C_PTETAPHIM || C == C_PXPYPZE) {
    if (l1 == L_AOS && l2 == L_AOS && tma_enabled() && tma_preferred<T, PM_MASS>() && !small) {
      HistParams hp{};
      gvx_status st = launch_pair_tma<T, C, PM_MASS>(v1, v2, n, m, hp, nullptr, nullptr, s);
      if (st != GVX_ERR_UNSUPPORTED) return st;
    }
  }
  if (L == L_AOS) return launch_mass<T, C, L_AOS>(v1, v2, m, n, s);
  if (L == L_SOA) return launch_mass<T, C, L_SOA>(v1, v2, m, n, s);
  return launch_mass<T, C, L_GEN>(v1, v2, m, n, s);
}

// ---------------------------------------------------------------- boost -----
template <typename T, bool UNI>
gvx_status launch_boost(const gvx_vec4_cview* v, const gvx_vec3_cview* beta, const gvx_vec4_view* out, int64_t n,
                        T bx, T by, T bz, cudaStream_t s) {
  const char* vb = (const char*)v->c[0];
  const char* ob = (const char*)out->c[0];
  bool aos = v->stride == 4 && out->stride == 4 && aligned(vb, 4 * sizeof(T)) && aligned(ob, 4 * sizeof(T));
  for (int k = 1; k < 4; ++k)
    aos = aos && (const char*)v->c[k] == vb + k * sizeof(T) && (const char*)out->c[k] == ob + k * sizeof(T);
  if (aos) {
    auto k = k_boost<T, true, UNI>;
#ifdef GVX_TUNE
    if (tune_env("GVX_BOOST_U") == 2) k = k_boost<T, true, UNI, 2>;
    if (tune_env("GVX_BOOST_U") == 4) k = k_boost<T, true, UNI, 4>;
#endif
    int grid = grid_for(k, kBlock, 0, kBlock, n);
    k<<<grid, kBlock, 0, s>>>(mk4<T>(v), mk3<T>(beta), mk4o<T>(out), n, bx, by, bz);
  } else {
    auto k = k_boost<T, false, UNI>;
    int grid = grid_for(k, kBlock, 0, kBlock, n);
    k<<<grid, kBlock, 0, s>>>(mk4<T>(v), mk3<T>(beta), mk4o<T>(out), n, bx, by, bz);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GVX_OK : cuda_fail(e);
}

// Output may equal the input exactly (in place); any other overlap is UB.
bool out_view_ok(const gvx_vec4_view* out, size_t es) { return view_ok<4>(out, es); }

// ---------------------------------------------------------------- hist ------
constexpr size_t kMaxSmemBins = 48 * 1024;  // uint32 bins in shared memory (192 KB)

// WBO: the CM kernel also writes the boosted pair (compile-time, so the
// common path carries no output plumbing).
template <typename T, int C, int L, bool CM, bool WBO = false>
gvx_status launch_hist(const gvx_vec4_cview* v1, const gvx_vec4_cview* v2, int64_t n, const HistParams& hp,
                       unsigned long long* bins, void* m_out, const gvx_vec4_view* bo, cudaStream_t s) {
  constexpr int G = Group<T, L>::G;
  size_t nb2 = (size_t)hp.nbins + 2;
  bool smem = nb2 <= kMaxSmemBins;
  View4o<T> bov = mk4o<T>(bo);
  cudaError_t e;
  if (smem) {
    // f64 AoS: 4 CTAs/SM for the lab histogram, 3 for the heavier CM path (sweep ldg1/ldg4).
    auto k = k_mass_histogram<T, C, L, CM, true, 1, WBO>;
    if constexpr (sizeof(T) == 8 && L == L_AOS && !WBO) {
      if constexpr (CM) k = k_mass_histogram<T, C, L, CM, true, 3>;
      else k = k_mass_histogram<T, C, L, CM, true, 4>;
    }
#ifdef GVX_TUNE
    if constexpr (sizeof(T) == 8 && L == L_AOS && C == C_PTETAPHIM && !WBO) {
      int v = tune_env("GVX_LDG_CFG");
      if (v == 1 || v == 2) k = k_mass_histogram<T, C, L, CM, true, 4>;
      if (v == 4) k = k_mass_histogram<T, C, L, CM, true, 3>;
    }
#endif
    size_t sm = nb2 * sizeof(unsigned int);
    int grid = grid_for(k, kBlock, sm, (int64_t)kBlock * G, n);
    // Per-CTA uint32 counters: one launch covers at most grid * 2^31 events.
    const int64_t chunk = (int64_t)grid << 31;
    for (int64_t off = 0; off < n; off += chunk) {
      int64_t cn = n - off < chunk ? n - off : chunk;
      View4<T> a = mk4<T>(v1), b = mk4<T>(v2);
      View4o<T> bo2 = bov;
      for (int c = 0; c < 4; ++c) {
        a.c[c] += off * a.s;
        b.c[c] += off * b.s;
        if (bo) bo2.c[c] += 2 * off * bo2.s;
      }
      T* mo = m_out ? (T*)m_out + off : nullptr;
      k<<<grid, kBlock, sm, s>>>(a, b, cn, hp, bins, mo, bo2);
    }
  } else {
    auto k = k_mass_histogram<T, C, L, CM, false, 1, WBO>;
    int grid = grid_for(k, kBlock, 0, (int64_t)kBlock * G, n);
    k<<<grid, kBlock, 0, s>>>(mk4<T>(v1), mk4<T>(v2), n, hp, bins, (T*)m_out, bov);
  }
  e = cudaGetLastError();
  return e == cudaSuccess ? GVX_OK : cuda_fail(e);
}

template <typename T, int C, bool CM>
gvx_status dispatch_hist(const gvx_vec4_cview* v1, const gvx_vec4_cview* v2, int64_t n, const HistParams& hp,
                         unsigned long long* bins, void* m_out, const gvx_vec4_view* bo, cudaStream_t s) {
  int l1 = classify(v1, sizeof(T)), l2 = classify(v2, sizeof(T));
  int L = (l1 == l2) ? l1 : L_GEN;
  if (m_out && L == L_AOS && !aligned(m_out, Group<T, L_AOS>::G * sizeof(T))) L = L_GEN;
  if (m_out && L == L_SOA && !aligned(m_out, Group<T, L_SOA>::G * sizeof(T))) L = L_GEN;
  if constexpr (CM) {
    if (bo) {  // boosted-pair output requested (diagnostic path)
      if (L == L_AOS) return launch_hist<T, C, L_AOS, CM, true>(v1, v2, n, hp, bins, m_out, bo, s);
      if (L == L_SOA) return launch_hist<T, C, L_SOA, CM, true>(v1, v2, n, hp, bins, m_out, bo, s);
      return launch_hist<T, C, L_GEN, CM, true>(v1, v2, n, hp, bins, m_out, bo, s);
    }
  }
  // Small batches: the register kernels win below ~2.6e5 pairs (1e6 for the f64 CM histogram),
  // measured with L2 flushed (tools/small_n_probe.py, profiles/r01/small_n_probe.jsonl).
  const int64_t small_n = (CM && sizeof(T) == 8) ? (int64_t(1) << 20) : (int64_t(1) << 18);
  const bool small = n < small_n && !force_tma();
  if constexpr (C == C_PTETAPHIM || C == C_PXPYPZE) {
    if (((l1 == L_AOS && l2 == L_AOS) || (l1 == L_SOA && l2 == L_SOA)) && tma_enabled() && !small &&
        tma_preferred<T, CM ? PM_HIST_CM : PM_HIST>()) {
      gvx_status st = launch_pair_tma<T, C, CM ? PM_HIST_CM : PM_HIST>(v1, v2, n, m_out, hp, bins, nullptr, s);
      if (st != GVX_ERR_UNSUPPORTED) return st;
    }
  }
  if (L == L_AOS) return launch_hist<T, C, L_AOS, CM>(v1, v2, n, hp, bins, m_out, nullptr, s);
  if (L == L_SOA) return launch_hist<T, C, L_SOA, CM>(v1, v2, n, hp, bins, m_out, nullptr, s);
  return launch_hist<T, C, L_GEN, CM>(v1, v2, n, hp, bins, m_out, nullptr, s);
}

// ----------------------------------------------- fused lab + CM pass -----
template <typename T, int C>
gvx_status dispatch_both(const gvx_vec4_cview* v1, const gvx_vec4_cview* v2, int64_t n, const HistParams& hp,
                         unsigned long long* lab_bins, unsigned long long* cm_bins, void* m_out, void* cm_m_out,
                         cudaStream_t s) {
  const int l1 = classify(v1, sizeof(T)), l2 = classify(v2, sizeof(T));
  const bool small = n < (int64_t(1) << 18) && !force_tma();
  if constexpr (C == C_PTETAPHIM || C == C_PXPYPZE) {
    if (((l1 == L_AOS && l2 == L_AOS) || (l1 == L_SOA && l2 == L_SOA)) && tma_enabled() && !small) {
      CosOut<T> co{hp, cm_bins, (T*)cm_m_out};
      co.hc.peers = nullptr;  // the CM histogram of the fused pass always lands in cm_bins
      co.hc.npeers = 0;
      co.hc.mc = nullptr;
      gvx_status st = launch_pair_tma<T, C, PM_BOTH>(v1, v2, n, m_out, hp, lab_bins, nullptr, s, co);
      if (st != GVX_ERR_UNSUPPORTED) return st;
    }
  }
  // other layouts / coordinates / small batches: the two histogram passes
  gvx_status st = dispatch_hist<T, C, false>(v1, v2, n, hp, lab_bins, m_out, nullptr, s);
  if (st != GVX_OK) return st;
  return dispatch_hist<T, C, true>(v1, v2, n, hp, cm_bins, cm_m_out, nullptr, s);
}

// ---------------------------------------------------------- one-launch step --
template <typename T, typename CFG, typename BR>
gvx_status launch_step(const gvx_vec4_cview* v1, const gvx_vec4_cview* v2, int64_t n, const HistParams& hp,
                       unsigned long long* lab_bins, unsigned long long* cm_bins, void* m_out, void* cm_m_out,
                       const T* bv, const T* bb, T* bout, int64_t nb, cudaStream_t s) {
  const int nbs = 2 * (hp.nbins + 2);
  const size_t sm = (size_t)CFG::RING_BYTES + BR::RING_BYTES + 16 * (CFG::STAGES + BR::BST) + (size_t)nbs * 4;
  if (sm > 227 * 1024) return GVX_ERR_UNSUPPORTED;
  auto k = k_step<T, CFG, BR>;
  const int block = StepGeom<CFG, BR>::THREADS;
  if (blocks_per_sm(k, block, sm) < 1) return GVX_ERR_UNSUPPORTED;
  const int grid = sm_count();
  if (n > ((int64_t)grid << 31)) return GVX_ERR_UNSUPPORTED;  // per-CTA uint32 counters
  if (nb / BR::BT >= INT32_MAX) return GVX_ERR_UNSUPPORTED;      // the kernel counts tiles in 32 bits
  CosOut<T> co{hp, cm_bins, (T*)cm_m_out};
  co.hc.peers = nullptr;
  co.hc.npeers = 0;
  co.hc.mc = nullptr;
  k<<<grid, block, sm, s>>>(mk4<T>(v1), mk4<T>(v2), n, (T*)m_out, hp, lab_bins, co, bv, bb, bout, nb);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GVX_OK : cuda_fail(e);
}

// AoS [N][4] rows (16-B aligned) / AoS [N][3] velocities (16-B aligned, contiguous).
template <typename V>
static bool aos4(const V* v, size_t es) {
  const char* b = (const char*)v->c[0];
  bool ok = v->stride == 4 && aligned(b, 16);
  for (int k = 1; k < 4; ++k) ok = ok && (const char*)v->c[k] == b + k * es;
  return ok;
}
static bool aos3(const gvx_vec3_cview* v, size_t es) {
  const char* b = (const char*)v->c[0];
  return v->stride == 3 && aligned(b, 16) && (const char*)v->c[1] == b + es && (const char*)v->c[2] == b + 2 * es;
}

// ------------------------------------------------------ cos theta* -------
template <typename T, int C>
gvx_status dispatch_costheta(const gvx_vec4_cview* v1, const gvx_vec4_cview* v2, int64_t n, const HistParams& hm,
                             unsigned long long* mbins, const HistParams& hc, unsigned long long* cbins, void* m_out,
                             void* cos_out, cudaStream_t s) {
  const int l1 = classify(v1, sizeof(T)), l2 = classify(v2, sizeof(T));
  CosOut<T> co{hc, cbins, (T*)cos_out};
  if constexpr (C == C_PTETAPHIM || C == C_PXPYPZE) {
    if (((l1 == L_AOS && l2 == L_AOS) || (l1 == L_SOA && l2 == L_SOA)) && tma_enabled()) {
      gvx_status st = launch_pair_tma<T, C, PM_HIST_CM_COS>(v1, v2, n, m_out, hm, mbins, nullptr, s, co);
      if (st != GVX_ERR_UNSUPPORTED) return st;
    }
  }
  const size_t nb = (size_t)hm.nbins + 2 + (size_t)hc.nbins + 2;
  cudaError_t e;
  if (nb <= kMaxSmemBins) {
    auto k = k_cm_costheta<T, C, true>;
    const size_t sm = nb * sizeof(unsigned int);
    const int grid = grid_for(k, kBlock, sm, kBlock, n);
    const int64_t chunk = (int64_t)grid << 31;  // uint32 shared-memory counters
    for (int64_t off = 0; off < n; off += chunk) {
      const int64_t cn = n - off < chunk ? n - off : chunk;
      View4<T> a = mk4<T>(v1), b = mk4<T>(v2);
      for (int c = 0; c < 4; ++c) {
        a.c[c] += off * a.s;
        b.c[c] += off * b.s;
      }
      k<<<grid, kBlock, sm, s>>>(a, b, cn, hm, mbins, hc, cbins, m_out ? (T*)m_out + off : nullptr,
                                 cos_out ? (T*)cos_out + off : nullptr);
    }
  } else {
    auto k = k_cm_costheta<T, C, false>;
    k<<<grid_for(k, kBlock, 0, kBlock, n), kBlock, 0, s>>>(mk4<T>(v1), mk4<T>(v2), n, hm, mbins, hc, cbins,
                                                           (T*)m_out, (T*)cos_out);
  }
  e = cudaGetLastError();
  return e == cudaSuccess ? GVX_OK : cuda_fail(e);
}

// ---------------------------------------------------------- lorentz ------
template <typename T>
gvx_status launch_lorentz(const gvx_vec4_cview* v, const double* Lrm, const gvx_vec4_view* out, int64_t n,
                          cudaStream_t s) {
  Mat4<T> L;
  for (int r = 0; r < 4; ++r)
    for (int c = 0; c < 4; ++c) L.m[r][c] = (T)Lrm[4 * r + c];
  const char* vb = (const char*)v->c[0];
  const char* ob = (const char*)out->c[0];
  bool aos = v->stride == 4 && out->stride == 4 && aligned(vb, 4 * sizeof(T)) && aligned(ob, 4 * sizeof(T));
  for (int k = 1; k < 4; ++k)
    aos = aos && (const char*)v->c[k] == vb + k * sizeof(T) && (const char*)out->c[k] == ob + k * sizeof(T);
  if (aos) {
    auto k = k_lorentz<T, true>;
    k<<<grid_for(k, kBlock, 0, kBlock, n), kBlock, 0, s>>>(mk4<T>(v), mk4o<T>(out), n, L);
  } else {
    auto k = k_lorentz<T, false>;
    k<<<grid_for(k, kBlock, 0, kBlock, n), kBlock, 0, s>>>(mk4<T>(v), mk4o<T>(out), n, L);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GVX_OK : cuda_fail(e);
}

// L^T g L = g within 1e-9 max(1, |L|^2), g = diag(-1,-1,-1,+1); all entries finite.
bool is_lorentz(const double* L) {
  static const double g[4] = {-1, -1, -1, 1};
  double lmax = 0;
  for (int k = 0; k < 16; ++k) {
    if (!isfinite(L[k])) return false;
    lmax = fabs(L[k]) > lmax ? fabs(L[k]) : lmax;
  }
  const double tol = 1e-9 * (lmax * lmax > 1 ? lmax * lmax : 1);
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) {
      double m = 0;
      for (int r = 0; r < 4; ++r) m += L[4 * r + a] * g[r] * L[4 * r + b];
      if (fabs(m - (a == b ? g[a] : 0.0)) > tol) return false;
    }
  return true;
}

// ---------------------------------------------------------- dimuon -------
template <typename T, typename CFG>
gvx_status launch_dimuon_tma(const gvx_vec4_cview* mu, const int32_t* q, const int64_t* off, int64_t n_events,
                             const HistParams& hp, unsigned long long* bins, void* m_out, cudaStream_t s) {
  const size_t smt = CFG::smem_bytes(hp.nbins + 2);
  auto kt = k_dimuon_tma<T, CFG>;
  int per_sm = smt <= 227 * 1024 ? blocks_per_sm(kt, 32 * (CFG::NCW + 1), smt) : 0;
  if (per_sm < 1) return GVX_ERR_UNSUPPORTED;
  const int64_t ntiles = n_events >= CFG::ET + 1 ? (n_events - 1) / CFG::ET : 0;
  const int64_t full = (int64_t)sm_count() * per_sm;
  const int grid = (int)(ntiles < 1 ? 1 : (ntiles < full ? ntiles : full));
  const int64_t chunk = (int64_t)grid << 31;
  for (int64_t o = 0; o < n_events; o += chunk) {
    int64_t cn = n_events - o < chunk ? n_events - o : chunk;
    kt<<<grid, 32 * (CFG::NCW + 1), smt, s>>>((const T*)mu->c[0], q, off + o, cn, hp, bins,
                                              m_out ? (T*)m_out + o : nullptr);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GVX_OK : cuda_fail(e);
}

// Stream-compacted dimuon kernel (default): ET events per tile, NT threads.
// Default geometry from the B200 sweep (profiles/r01/sweep_dimuon_compact.jsonl):
// 2048-event tiles, 256 threads, 5 CTAs/SM (MINB 5 caps registers at 48).
template <typename T, bool AOS, int ET = 2048, int NT = 256, int MINB = 5, int U = 1>
gvx_status launch_dimuon_compact(const gvx_vec4_cview* mu, const int32_t* q, const int64_t* off, int64_t n_events,
                                 const HistParams& hp, unsigned long long* bins, void* m_out, cudaStream_t s) {
#ifdef GVX_TUNE
  if constexpr (ET == 2048 && NT == 256 && MINB == 5 && U == 1) {
    switch (tune_env("GVX_DIMUON_CFG")) {
      case 7: return launch_dimuon_compact<T, AOS, 2048, 256, 5, 2>(mu, q, off, n_events, hp, bins, m_out, s);
      case 8: return launch_dimuon_compact<T, AOS, 2048, 256, 4, 2>(mu, q, off, n_events, hp, bins, m_out, s);
      case 9: return launch_dimuon_compact<T, AOS, 2048, 256, 3, 2>(mu, q, off, n_events, hp, bins, m_out, s);
      case 1: return launch_dimuon_compact<T, AOS, 2048, 256, 4>(mu, q, off, n_events, hp, bins, m_out, s);
      case 2: return launch_dimuon_compact<T, AOS, 2048, 256, 6>(mu, q, off, n_events, hp, bins, m_out, s);
      case 3: return launch_dimuon_compact<T, AOS, 1024, 256, 4>(mu, q, off, n_events, hp, bins, m_out, s);
      case 4: return launch_dimuon_compact<T, AOS, 4096, 256, 4>(mu, q, off, n_events, hp, bins, m_out, s);
      case 5: return launch_dimuon_compact<T, AOS, 2048, 128, 8>(mu, q, off, n_events, hp, bins, m_out, s);
      case 6: return launch_dimuon_compact<T, AOS, 4096, 512, 2>(mu, q, off, n_events, hp, bins, m_out, s);
      default: break;
    }
  }
#endif
  const size_t sm = dimuon_compact_smem<ET>(hp.nbins + 2);
  if (sm > 227 * 1024) return GVX_ERR_UNSUPPORTED;
  auto k = k_dimuon_compact<T, AOS, ET, NT, U, MINB>;
  const int grid = grid_for(k, NT, sm, ET, n_events);
  // uint32 shared-memory bins: one launch covers at most grid * 2^31 events
  const int64_t chunk = (int64_t)grid << 31;
  for (int64_t o = 0; o < n_events; o += chunk) {
    const int64_t cn = n_events - o < chunk ? n_events - o : chunk;
    k<<<grid, NT, sm, s>>>(mk4<T>(mu), q, off + o, cn, hp, bins, m_out ? (T*)m_out + o : nullptr);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GVX_OK : cuda_fail(e);
}

// Carried-list dimuon kernel (default): ET events per tile, NT threads, CPS CTAs
// per SM (tools/probe/dimuon3.cu sweeps, 32-bit list entries: f64 1024 / 128 / 8
// 0.457 ms, f32 2048 / 256 / 4 0.392 ms; the f32 kernel is compiled for a minimum
// of 4 CTAs: compiled for 5 it got 40 registers and ran 0.72 ms instead of 0.48).
template <typename T, bool AOS, bool WANT_M, bool VOFF>
gvx_status launch_dimuon_carry(const gvx_vec4_cview* mu, const int32_t* q, const int64_t* off, int64_t n_events,
                               const HistParams& hp, unsigned long long* bins, void* m_out, cudaStream_t s) {
  constexpr bool F64 = sizeof(T) == 8;
  constexpr int ET = F64 ? 1024 : 2048, NT = F64 ? 128 : 256, MINB = F64 ? 8 : 4, CPS = F64 ? 8 : 4;
  const size_t sm = DimuonCarry<ET, NT>::smem(hp.nbins + 2, WANT_M);
  if (sm > 227 * 1024) return GVX_ERR_UNSUPPORTED;
  auto k = k_dimuon_carry<T, AOS, ET, NT, MINB, WANT_M, VOFF>;
  int per_sm = blocks_per_sm(k, NT, sm);
  if (per_sm < 1) return GVX_ERR_UNSUPPORTED;
  if (per_sm > CPS) per_sm = CPS;
  const int64_t ntiles = (n_events + ET - 1) / ET;
  const int64_t full = (int64_t)sm_count() * per_sm;
  const int grid = (int)(ntiles < full ? ntiles : full);
  // uint32 shared-memory bins: one launch covers at most grid * 2^31 events
  // (a multiple of 4 events, so a chunk's offsets keep the 32-byte alignment)
  const int64_t chunk = (int64_t)grid << 31;
  for (int64_t o = 0; o < n_events; o += chunk) {
    const int64_t cn = n_events - o < chunk ? n_events - o : chunk;
    k<<<grid, NT, sm, s>>>(mk4<T>(mu), q, off + o, cn, hp, bins, m_out ? (T*)m_out + o : nullptr);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GVX_OK : cuda_fail(e);
}

template <typename T, bool AOS>
gvx_status launch_dimuon_carry(const gvx_vec4_cview* mu, const int32_t* q, const int64_t* off, int64_t n_events,
                               const HistParams& hp, unsigned long long* bins, void* m_out, cudaStream_t s) {
  const bool voff = aligned(off, 32);
  if (m_out)
    return voff ? launch_dimuon_carry<T, AOS, true, true>(mu, q, off, n_events, hp, bins, m_out, s)
                : launch_dimuon_carry<T, AOS, true, false>(mu, q, off, n_events, hp, bins, m_out, s);
  return voff ? launch_dimuon_carry<T, AOS, false, true>(mu, q, off, n_events, hp, bins, m_out, s)
              : launch_dimuon_carry<T, AOS, false, false>(mu, q, off, n_events, hp, bins, m_out, s);
}

// GVX_DIMUON_IMPL=tma / ldg / compact selects the other kernels for A/B runs.
int dimuon_impl() {
  static const int v = [] {
    const char* e = getenv("GVX_DIMUON_IMPL");
    if (e && e[0] == 't') return 1;
    if (e && e[0] == 'l') return 2;
    if (e && e[0] == 'c') return 3;
    return 0;
  }();
  return v;
}

template <typename T>
gvx_status launch_dimuon(const gvx_vec4_cview* mu, const int32_t* q, const int64_t* off, int64_t n_events,
                         const HistParams& hp, unsigned long long* bins, void* m_out, cudaStream_t s) {
  const char* b = (const char*)mu->c[0];
  bool aos = mu->stride == 4 && aligned(b, 4 * sizeof(T));
  for (int k = 1; k < 4; ++k) aos = aos && (const char*)mu->c[k] == b + k * sizeof(T);
  const size_t nb2 = (size_t)hp.nbins + 2;
  if (nb2 > kMaxSmemBins) return GVX_ERR_UNSUPPORTED;
  const bool aos_vec = aos && aligned(b, sizeof(T) == 8 ? 32 : 16);  // 256-bit (f64) / 128-bit (f32) muon loads
  if (dimuon_impl() == 0) {
    gvx_status st = aos_vec ? launch_dimuon_carry<T, true>(mu, q, off, n_events, hp, bins, m_out, s)
                            : launch_dimuon_carry<T, false>(mu, q, off, n_events, hp, bins, m_out, s);
    if (st != GVX_ERR_UNSUPPORTED) return st;
  }
  if (dimuon_impl() == 3) {
    gvx_status st = aos_vec ? launch_dimuon_compact<T, true>(mu, q, off, n_events, hp, bins, m_out, s)
                            : launch_dimuon_compact<T, false>(mu, q, off, n_events, hp, bins, m_out, s);
    if (st != GVX_ERR_UNSUPPORTED) return st;
  }
  if (dimuon_impl() == 1 && aos && aligned(b, 16) && aligned(off, 16) && aligned(q, 16) && tma_enabled()) {  // TMA column streaming
    gvx_status st = GVX_ERR_UNSUPPORTED;
#ifdef GVX_TUNE
    switch (tune_env("GVX_DIMUON_CFG")) {
      case 1: st = launch_dimuon_tma<T, DimuonTma<T, 512, 768, 6, 16>>(mu, q, off, n_events, hp, bins, m_out, s); break;
      case 2: st = launch_dimuon_tma<T, DimuonTma<T, 512, 768, 3, 8>>(mu, q, off, n_events, hp, bins, m_out, s); break;
      case 3: st = launch_dimuon_tma<T, DimuonTma<T, 2048, 2560, 2, 16>>(mu, q, off, n_events, hp, bins, m_out, s); break;
      case 4: st = launch_dimuon_tma<T, DimuonTma<T, 512, 768, 4, 8>>(mu, q, off, n_events, hp, bins, m_out, s); break;
      default: break;
    }
    if (st != GVX_ERR_UNSUPPORTED) return st;
#endif
    st = launch_dimuon_tma<T, DimuonTma<T, 1024, 1536, 3, 16>>(mu, q, off, n_events, hp, bins, m_out, s);
    if (st != GVX_ERR_UNSUPPORTED) return st;
  }
  const size_t sm = nb2 * sizeof(unsigned int);
  auto k = aos ? k_dimuon_histogram<T, true> : k_dimuon_histogram<T, false>;
  int grid = grid_for(k, kBlock, sm, kBlock * 4, n_events);
  // uint32 shared-memory bins: one launch covers at most grid * 2^31 events
  const int64_t chunk = (int64_t)grid << 31;
  for (int64_t o = 0; o < n_events; o += chunk) {
    int64_t cn = n_events - o < chunk ? n_events - o : chunk;
    k<<<grid, kBlock, sm, s>>>(mk4<T>(mu), q, off + o, cn, hp, bins, m_out ? (T*)m_out + o : nullptr);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GVX_OK : cuda_fail(e);
}

// ------------------------------------------------ mixed-coordinate pairs --
// v1 in c1, v2 in c2 (c1 != c2): k_mixed_pairs. AoS views with
// 32-byte rows take the 256-bit loads, every other view the scalar ones.
template <typename T, int L, int MODE>
gvx_status launch_mixed_l(const gvx_vec4_cview* v1, const gvx_vec4_cview* v2, int c1, int c2, int64_t n,
                          const HistParams& hp, unsigned long long* bins, void* m_out, const HistParams& hc,
                          unsigned long long* cbins, void* cm_out, const gvx_vec4_view* bo, cudaStream_t s) {
  constexpr int G = Group<T, L>::G;
  const size_t nbt = MODE == PM_MASS ? 0 : (size_t)hp.nbins + 2 + (MODE == PM_BOTH ? (size_t)hc.nbins + 2 : 0);
  const bool smem = MODE != PM_MASS && nbt <= kMaxSmemBins;
  auto k = smem ? k_mixed_pairs<T, L, MODE, true> : k_mixed_pairs<T, L, MODE, false>;
  const size_t sm = smem ? nbt * sizeof(unsigned int) : 0;
  const int grid = grid_for(k, kBlock, sm, (int64_t)kBlock * G, n);
  // per-CTA uint32 shared-memory counters: one launch covers at most grid * 2^31 events
  const int64_t chunk = smem ? ((int64_t)grid << 31) : n;
  const View4o<T> bov = mk4o<T>(bo);
  for (int64_t off = 0; off < n; off += chunk) {
    const int64_t cn = n - off < chunk ? n - off : chunk;
    View4<T> a = mk4<T>(v1), b = mk4<T>(v2);
    View4o<T> bo2 = bov;
    for (int c = 0; c < 4; ++c) {
      a.c[c] += off * a.s;
      b.c[c] += off * b.s;
      if (bo) bo2.c[c] += 2 * off * bo2.s;
    }
    k<<<grid, kBlock, sm, s>>>(a, b, c1, c2, cn, hp, bins, m_out ? (T*)m_out + off : nullptr, hc, cbins,
                               cm_out ? (T*)cm_out + off : nullptr, bo2);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? GVX_OK : cuda_fail(e);
}

template <typename T, int MODE>
gvx_status launch_mixed(const gvx_vec4_cview* v1, const gvx_vec4_cview* v2, int c1, int c2, int64_t n,
                        const HistParams& hp, unsigned long long* bins, void* m_out, const HistParams& hc,
                        unsigned long long* cbins, void* cm_out, const gvx_vec4_view* bo, cudaStream_t s) {
  const size_t es = sizeof(T);
  constexpr int G = Group<T, L_AOS>::G;
  const bool outs_ok = (!m_out || aligned(m_out, G * es)) && (!cm_out || aligned(cm_out, G * es));
  if (classify(v1, es) == L_AOS && classify(v2, es) == L_AOS && outs_ok)
    return launch_mixed_l<T, L_AOS, MODE>(v1, v2, c1, c2, n, hp, bins, m_out, hc, cbins, cm_out, bo, s);
  return launch_mixed_l<T, L_GEN, MODE>(v1, v2, c1, c2, n, hp, bins, m_out, hc, cbins, cm_out, bo, s);
}

}  // namespace

extern "C" {

int gvx_abi_version(void) { return GVX_ABI_VERSION; }

const char* gvx_status_string(gvx_status st) {
  switch (st) {
    case GVX_OK: return "GVX_OK";
    case GVX_ERR_INVALID_ARGUMENT: return "GVX_ERR_INVALID_ARGUMENT";
    case GVX_ERR_DOMAIN: return "GVX_ERR_DOMAIN";
    case GVX_ERR_UNSUPPORTED: return "GVX_ERR_UNSUPPORTED";
    case GVX_ERR_CUDA: return "GVX_ERR_CUDA";
  }
  return "GVX_ERR_UNKNOWN";
}

const char* gvx_last_cuda_error_string(void) { return g_last_cuda_error.c_str(); }

gvx_status gvx_lorentz_transform(gvx_dtype dtype, const gvx_vec4_cview* v, const double* L,
                                 const gvx_vec4_view* out, int64_t n, gvx_stream_t stream) {
  if (!valid_dtype(dtype) || n < 0 || !L) return GVX_ERR_INVALID_ARGUMENT;
  if (!is_lorentz(L)) return GVX_ERR_DOMAIN;
  if (n == 0) return GVX_OK;
  const size_t es = dsize(dtype);
  if (!view_ok<4>(v, es) || !out_view_ok(out, es)) return GVX_ERR_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == GVX_F64) return launch_lorentz<double>(v, L, out, n, s);
  return launch_lorentz<float>(v, L, out, n, s);
}

gvx_status gvx_dimuon_histogram(gvx_dtype dtype, const gvx_vec4_cview* muons, const int32_t* charge,
                                const int64_t* offsets, int64_t n_events, double lo, double hi, int32_t nbins,
                                unsigned long long* bins, void* m_out, gvx_stream_t stream) {
  if (!valid_dtype(dtype) || n_events < 0) return GVX_ERR_INVALID_ARGUMENT;
  if (nbins < 1 || nbins > (1 << 28) || !isfinite(lo) || !isfinite(hi) || !(lo < hi)) return GVX_ERR_INVALID_ARGUMENT;
  if (n_events == 0) return GVX_OK;
  const size_t es = dsize(dtype);
  if (!view_ok<4>(muons, es) || !charge || !aligned(charge, 4) || !offsets || !aligned(offsets, 8) || !bins ||
      !aligned(bins, 8))
    return GVX_ERR_INVALID_ARGUMENT;
  if (m_out && !aligned(m_out, es)) return GVX_ERR_INVALID_ARGUMENT;
  const HistParams hp = make_hist_params(lo, hi, nbins);
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == GVX_F64) return launch_dimuon<double>(muons, charge, offsets, n_events, hp, bins, m_out, s);
  return launch_dimuon<float>(muons, charge, offsets, n_events, hp, bins, m_out, s);
}

gvx_status gvx_invariant_mass(gvx_dtype dtype, gvx_coords coords, const gvx_vec4_cview* v1, const gvx_vec4_cview* v2,
                              void* m_out, int64_t n, gvx_stream_t stream) {
  if (!valid_dtype(dtype) || !valid_coords(coords) || n < 0) return GVX_ERR_INVALID_ARGUMENT;
  if (n == 0) return GVX_OK;
  size_t es = dsize(dtype);
  if (!view_ok<4>(v1, es) || !view_ok<4>(v2, es) || !m_out || !aligned(m_out, es)) return GVX_ERR_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
#define GVX_MASS_DISPATCH(T)                                                     \
  switch (coords) {                                                             \
    case GVX_PTETAPHIM: return dispatch_mass<T, C_PTETAPHIM>(v1, v2, m_out, n, s); \
    case GVX_PXPYPZE: return dispatch_mass<T, C_PXPYPZE>(v1, v2, m_out, n, s);     \
    case GVX_PXPYPZM: return dispatch_mass<T, C_PXPYPZM>(v1, v2, m_out, n, s);     \
    default: return dispatch_mass<T, C_PTETAPHIE>(v1, v2, m_out, n, s);          \
  }
  if (dtype == GVX_F64) {
    GVX_MASS_DISPATCH(double)
  }
  GVX_MASS_DISPATCH(float)
#undef GVX_MASS_DISPATCH
}

gvx_status gvx_boost(gvx_dtype dtype, const gvx_vec4_cview* v, const gvx_vec3_cview* beta, const gvx_vec4_view* out,
                     int64_t n, gvx_stream_t stream) {
  if (!valid_dtype(dtype) || n < 0) return GVX_ERR_INVALID_ARGUMENT;
  if (n == 0) return GVX_OK;
  size_t es = dsize(dtype);
  if (!view_ok<4>(v, es) || !view_ok<3>(beta, es) || !out_view_ok(out, es)) return GVX_ERR_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == GVX_F64) return launch_boost<double, false>(v, beta, out, n, 0, 0, 0, s);
  return launch_boost<float, false>(v, beta, out, n, 0, 0, 0, s);
}

gvx_status gvx_boost_uniform(gvx_dtype dtype, const gvx_vec4_cview* v, double bx, double by, double bz,
                             const gvx_vec4_view* out, int64_t n, gvx_stream_t stream) {
  if (!valid_dtype(dtype) || n < 0) return GVX_ERR_INVALID_ARGUMENT;
  if (!isfinite(bx) || !isfinite(by) || !isfinite(bz)) return GVX_ERR_DOMAIN;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == GVX_F64) {
    if (!(bx * bx + by * by + bz * bz < 1.0)) return GVX_ERR_DOMAIN;
  } else {
    float fx = (float)bx, fy = (float)by, fz = (float)bz;
    if (!(fx * fx + fy * fy + fz * fz < 1.0f)) return GVX_ERR_DOMAIN;
  }
  if (n == 0) return GVX_OK;
  size_t es = dsize(dtype);
  if (!view_ok<4>(v, es) || !out_view_ok(out, es)) return GVX_ERR_INVALID_ARGUMENT;
  if (dtype == GVX_F64) return launch_boost<double, true>(v, nullptr, out, n, bx, by, bz, s);
  return launch_boost<float, true>(v, nullptr, out, n, (float)bx, (float)by, (float)bz, s);
}

gvx_status gvx_pair_histograms(gvx_dtype dtype, gvx_coords coords, const gvx_vec4_cview* v1,
                               const gvx_vec4_cview* v2, int64_t n, double lo, double hi, int32_t nbins,
                               unsigned long long* lab_bins, unsigned long long* cm_bins, void* m_out,
                               void* cm_m_out, gvx_stream_t stream) {
  if (!valid_dtype(dtype) || !valid_coords(coords) || n < 0) return GVX_ERR_INVALID_ARGUMENT;
  if (nbins < 1 || nbins > (1 << 28) || !isfinite(lo) || !isfinite(hi) || !(lo < hi)) return GVX_ERR_INVALID_ARGUMENT;
  if (n == 0) return GVX_OK;
  const size_t es = dsize(dtype);
  if (!view_ok<4>(v1, es) || !view_ok<4>(v2, es) || !lab_bins || !aligned(lab_bins, 8) || !cm_bins ||
      !aligned(cm_bins, 8))
    return GVX_ERR_INVALID_ARGUMENT;
  if ((m_out && !aligned(m_out, es)) || (cm_m_out && !aligned(cm_m_out, es))) return GVX_ERR_INVALID_ARGUMENT;
  const HistParams hp = make_hist_params(lo, hi, nbins);
  cudaStream_t s = (cudaStream_t)stream;
#define GVX_BOTH_COORDS(T)                                                                                   \
  switch (coords) {                                                                                         \
    case GVX_PTETAPHIM: return dispatch_both<T, C_PTETAPHIM>(v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, s); \
    case GVX_PXPYPZE: return dispatch_both<T, C_PXPYPZE>(v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, s);     \
    case GVX_PXPYPZM: return dispatch_both<T, C_PXPYPZM>(v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, s);     \
    default: return dispatch_both<T, C_PTETAPHIE>(v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, s);            \
  }
  if (dtype == GVX_F64) {
    GVX_BOTH_COORDS(double)
  }
  GVX_BOTH_COORDS(float)
#undef GVX_BOTH_COORDS
}

gvx_status gvx_pair_histograms_boost(gvx_dtype dtype, gvx_coords coords, const gvx_vec4_cview* v1,
                                     const gvx_vec4_cview* v2, int64_t n, double lo, double hi, int32_t nbins,
                                     unsigned long long* lab_bins, unsigned long long* cm_bins, void* m_out,
                                     void* cm_m_out, const gvx_vec4_cview* bv, const gvx_vec3_cview* beta,
                                     const gvx_vec4_view* bout, int64_t nb, gvx_stream_t stream) {
  if (!valid_dtype(dtype) || !valid_coords(coords) || n < 0 || nb < 0) return GVX_ERR_INVALID_ARGUMENT;
  if (nbins < 1 || nbins > (1 << 28) || !isfinite(lo) || !isfinite(hi) || !(lo < hi)) return GVX_ERR_INVALID_ARGUMENT;
  const size_t es = dsize(dtype);
  if (n > 0 && (!view_ok<4>(v1, es) || !view_ok<4>(v2, es) || !lab_bins || !aligned(lab_bins, 8) || !cm_bins ||
                !aligned(cm_bins, 8)))
    return GVX_ERR_INVALID_ARGUMENT;
  if ((m_out && !aligned(m_out, es)) || (cm_m_out && !aligned(cm_m_out, es))) return GVX_ERR_INVALID_ARGUMENT;
  if (nb > 0 && (!view_ok<4>(bv, es) || !view_ok<3>(beta, es) || !out_view_ok(bout, es)))
    return GVX_ERR_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  // f64 only: the f32 pair pass is issue-bound and boost warps beside it made the step slower
  // (1.46 vs 1.39 ms at 1e8); f32 takes the two calls.
  // bout: the boost warps store with 256-bit STG (st.global.v4.f64), which needs 32-byte rows
  const bool fast = dtype == GVX_F64 && n >= (int64_t(1) << 20) && nb >= (int64_t(1) << 20) &&
                    coords == GVX_PTETAPHIM && tma_enabled() && step_kernel_enabled() &&
                    classify(v1, es) == L_AOS && classify(v2, es) == L_AOS && aos4(bv, es) && aos3(beta, es) &&
                    aos4(bout, es) && aligned(bout->c[0], 4 * es);
  if (fast) {
    const HistParams hp = make_hist_params(lo, hi, nbins);
    const double* pv = (const double*)bv->c[0];
    const double* pb = (const double*)beta->c[0];
    double* po = (double*)bout->c[0];
    gvx_status st;
    // Default (round 2, session 3): 16 pair-consumer warps + 7 boost warps + 1 producer warp =
    // 24 warps at 80 registers (25 warps were held to 72 and spilled 160 B), a 2-stage boost
    // ring of 448-vector stages. Same-box sweep of 30 splits / ring shapes
    // (profiles/r02/step_split_sweep.jsonl): 2.518 ms against 2.607 ms for round 1's 18 + 6
    // warps with a 3 x 384 boost ring; 15 + 8 and 14 + 9 tie, 3- and 4-stage boost rings and
    // one-vector-per-thread stages are slower.
    using StepCfg = PairTma<double, 1024, 2, 16, 1>;
    using StepBoost = BoostRing<double, 448, 2, 7>;
#if defined(GVX_TUNE) || defined(GVX_STEP_ALT)
    // Tuning builds: GVX_STEP_CFG picks another split (numbers as in the sweep file; unset or 0:
    // the default; round 1's config 0 is 27 here).
    const int c = tune_env("GVX_STEP_CFG");
    if (c == 5)  // 17 pair + 6 boost + 1 producer warps: 24 warps, 80 registers
      st = launch_step<double, PairTma<double, 1088, 2, 17, 1>, BoostRing<double, 384, 3, 6>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 6)  // 16 + 7 + 1
      st = launch_step<double, PairTma<double, 1024, 2, 16, 1>, BoostRing<double, 448, 3, 7>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 7)  // 18 + 5 + 1
      st = launch_step<double, PairTma<double, 1152, 2, 18, 1>, BoostRing<double, 320, 3, 5>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 8)  // 17 + 6 + 1, 4-stage boost ring
      st = launch_step<double, PairTma<double, 1088, 2, 17, 1>, BoostRing<double, 384, 4, 6>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 9)  // 17 + 6 + 1, 576-event boost stages
      st = launch_step<double, PairTma<double, 1088, 2, 17, 1>, BoostRing<double, 576, 2, 6>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 10)  // 18 + 5 + 1, 480 x 2
      st = launch_step<double, PairTma<double, 1152, 2, 18, 1>, BoostRing<double, 480, 2, 5>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 11)  // 18 + 5 + 1, 640 x 2
      st = launch_step<double, PairTma<double, 1152, 2, 18, 1>, BoostRing<double, 640, 2, 5>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 12)  // 16 + 7 + 1, 672 x 2
      st = launch_step<double, PairTma<double, 1024, 2, 16, 1>, BoostRing<double, 672, 2, 7>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 13)  // 17 + 6 + 1, 384 x 2
      st = launch_step<double, PairTma<double, 1088, 2, 17, 1>, BoostRing<double, 384, 2, 6>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 14)  // 18 + 6 + 1 (25 warps, 72 registers), 576 x 2
      st = launch_step<double, PairTma<double, 1152, 2, 18, 1>, BoostRing<double, 576, 2, 6>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 15)  // 18 + 5 + 1, 320 x 2
      st = launch_step<double, PairTma<double, 1152, 2, 18, 1>, BoostRing<double, 320, 2, 5>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 16)  // 16 + 7 + 1, 448 x 2
      st = launch_step<double, PairTma<double, 1024, 2, 16, 1>, BoostRing<double, 448, 2, 7>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 17)  // 17 + 6 + 1, 192 x 2
      st = launch_step<double, PairTma<double, 1088, 2, 17, 1>, BoostRing<double, 192, 2, 6>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 18)  // 17 + 6 + 1, 192 x 4
      st = launch_step<double, PairTma<double, 1088, 2, 17, 1>, BoostRing<double, 192, 4, 6>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 19)  // 20 + 3 + 1, 192 x 2
      st = launch_step<double, PairTma<double, 1280, 2, 20, 1>, BoostRing<double, 192, 2, 3>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 20)  // 15 + 8 + 1, 512 x 2
      st = launch_step<double, PairTma<double, 960, 2, 15, 1>, BoostRing<double, 512, 2, 8>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 21)  // 19 + 4 + 1, 256 x 2
      st = launch_step<double, PairTma<double, 1216, 2, 19, 1>, BoostRing<double, 256, 2, 4>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 22)  // 14 + 9 + 1, 576 x 2
      st = launch_step<double, PairTma<double, 896, 2, 14, 1>, BoostRing<double, 576, 2, 9>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 23)  // 16 + 7 + 1, 448 x 3
      st = launch_step<double, PairTma<double, 1024, 2, 16, 1>, BoostRing<double, 448, 3, 7>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 24)  // 15 + 8 + 1, 512 x 3
      st = launch_step<double, PairTma<double, 960, 2, 15, 1>, BoostRing<double, 512, 3, 8>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 25)  // 16 + 7 + 1, 224 x 2
      st = launch_step<double, PairTma<double, 1024, 2, 16, 1>, BoostRing<double, 224, 2, 7>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 26)  // 15 + 8 + 1, 256 x 2
      st = launch_step<double, PairTma<double, 960, 2, 15, 1>, BoostRing<double, 256, 2, 8>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 28)  // setmaxnreg: 16 pair at 96 + 8 boost at 48 + 4-warp producer at 24, boost 512 x 2
      st = launch_step<double, PairTma<double, 1024, 2, 16, 1, 96>, BoostRing<double, 512, 2, 8, 48>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 29)  // setmaxnreg: 16 pair at 88 + 8 boost at 64, boost 512 x 2
      st = launch_step<double, PairTma<double, 1024, 2, 16, 1, 88>, BoostRing<double, 512, 2, 8, 64>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 30)  // setmaxnreg: 20 pair at 80 + 4 boost at 80, boost 256 x 2
      st = launch_step<double, PairTma<double, 1280, 2, 20, 1, 80>, BoostRing<double, 256, 2, 4, 80>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 3)
      st = launch_step<double, PairTma<double, 1280, 2, 20, 1, 80>, BoostRing<double, 256, 4, 4, 80>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 4)
      st = launch_step<double, PairTma<double, 1024, 2, 16, 1, 88>, BoostRing<double, 512, 3, 8, 56>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 1)
      st = launch_step<double, PairTma<double, 1024, 2, 16, 1>, BoostRing<double, 512, 3, 8>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 27)  // (round 1's config 0) 20 + 4 + 1, 256 x 4
      st = launch_step<double, PairTma<double, 1280, 2, 20, 1>, BoostRing<double, 256, 4, 4>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c == 2)  // round 1's default: 18 + 6 + 1 (25 warps, 72 registers), 384 x 3
      st = launch_step<double, PairTma<double, 1152, 2, 18, 1>, BoostRing<double, 384, 3, 6>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else
      st = launch_step<double, StepCfg, StepBoost>(v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po,
                                                   nb, s);
#else
    st = launch_step<double, StepCfg, StepBoost>(v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb,
                                                 s);
#endif
    if (st != GVX_ERR_UNSUPPORTED) return st;
  }
#if defined(GVX_TUNE) || defined(GVX_STEP_ALT)
  // Tuning builds only: the f32 step in one launch (GVX_STEP32_CFG = 1..10), for A/B runs.
  const int c32 = tune_env("GVX_STEP32_CFG");
  if (c32 && dtype == GVX_F32 && n >= (int64_t(1) << 20) && nb >= (int64_t(1) << 20) && coords == GVX_PTETAPHIM &&
      tma_enabled() && classify(v1, es) == L_AOS && classify(v2, es) == L_AOS && aos4(bv, es) &&
      aos3(beta, es) && aos4(bout, es) && aligned(bout->c[0], 4 * es)) {
    const HistParams hp = make_hist_params(lo, hi, nbins);
    const float* pv = (const float*)bv->c[0];
    const float* pb = (const float*)beta->c[0];
    float* po = (float*)bout->c[0];
    gvx_status st = GVX_ERR_UNSUPPORTED;
    if (c32 == 1)
      st = launch_step<float, PairTma<float, 1536, 3, 24, 1>, BoostRing<float, 512, 3, 4>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c32 == 2)
      st = launch_step<float, PairTma<float, 1280, 3, 20, 1>, BoostRing<float, 768, 3, 8>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c32 == 3)
      st = launch_step<float, PairTma<float, 1536, 3, 24, 1, 64>, BoostRing<float, 512, 3, 4, 56>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c32 == 4)
      st = launch_step<float, PairTma<float, 1280, 3, 20, 1, 72>, BoostRing<float, 768, 3, 8, 56>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c32 == 5)  // 16 + 7 + 1 (24 warps, 80 registers), pair 1024 x 3, boost 448 x 2
      st = launch_step<float, PairTma<float, 1024, 3, 16, 1>, BoostRing<float, 448, 2, 7>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c32 == 6)  // 16 + 7 + 1, pair 2048 x 3, boost 448 x 2
      st = launch_step<float, PairTma<float, 2048, 3, 16, 1>, BoostRing<float, 448, 2, 7>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c32 == 7)  // 15 + 8 + 1, pair 960 x 4, boost 512 x 2
      st = launch_step<float, PairTma<float, 960, 4, 15, 1>, BoostRing<float, 512, 2, 8>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c32 == 8)  // 18 + 5 + 1, pair 1152 x 3, boost 320 x 2
      st = launch_step<float, PairTma<float, 1152, 3, 18, 1>, BoostRing<float, 320, 2, 5>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c32 == 9)  // 16 + 7 + 1, pair 1024 x 4, boost 448 x 2
      st = launch_step<float, PairTma<float, 1024, 4, 16, 1>, BoostRing<float, 448, 2, 7>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c32 == 10)  // 14 + 9 + 1, pair 896 x 4, boost 576 x 2
      st = launch_step<float, PairTma<float, 896, 4, 14, 1>, BoostRing<float, 576, 2, 9>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    else if (c32 == 11)  // 20 + 3 + 1, pair 1280 x 3, boost 192 x 2
      st = launch_step<float, PairTma<float, 1280, 3, 20, 1>, BoostRing<float, 192, 2, 3>>(
          v1, v2, n, hp, lab_bins, cm_bins, m_out, cm_m_out, pv, pb, po, nb, s);
    if (st != GVX_ERR_UNSUPPORTED) return st;
  }
#endif
  // any other shape: the two calls it fuses (same bits)
  gvx_status st = n > 0 ? gvx_pair_histograms(dtype, coords, v1, v2, n, lo, hi, nbins, lab_bins, cm_bins, m_out,
                                              cm_m_out, stream)
                        : GVX_OK;
  if (st != GVX_OK || nb == 0) return st;
  return gvx_boost(dtype, bv, beta, bout, nb, stream);
}

gvx_status gvx_cm_costheta_histogram(gvx_dtype dtype, gvx_coords coords, const gvx_vec4_cview* v1,
                                     const gvx_vec4_cview* v2, int64_t n, double m_lo, double m_hi, int32_t m_nbins,
                                     unsigned long long* m_bins, double c_lo, double c_hi, int32_t c_nbins,
                                     unsigned long long* c_bins, void* m_out, void* cos_out, gvx_stream_t stream) {
  if (!valid_dtype(dtype) || !valid_coords(coords) || n < 0) return GVX_ERR_INVALID_ARGUMENT;
  if (m_nbins < 1 || m_nbins > (1 << 28) || !isfinite(m_lo) || !isfinite(m_hi) || !(m_lo < m_hi))
    return GVX_ERR_INVALID_ARGUMENT;
  if (c_nbins < 1 || c_nbins > (1 << 28) || !isfinite(c_lo) || !isfinite(c_hi) || !(c_lo < c_hi))
    return GVX_ERR_INVALID_ARGUMENT;
  if (n == 0) return GVX_OK;
  const size_t es = dsize(dtype);
  if (!view_ok<4>(v1, es) || !view_ok<4>(v2, es) || !m_bins || !aligned(m_bins, 8) || !c_bins ||
      !aligned(c_bins, 8))
    return GVX_ERR_INVALID_ARGUMENT;
  if ((m_out && !aligned(m_out, es)) || (cos_out && !aligned(cos_out, es))) return GVX_ERR_INVALID_ARGUMENT;
  const HistParams hm = make_hist_params(m_lo, m_hi, m_nbins), hc = make_hist_params(c_lo, c_hi, c_nbins);
  cudaStream_t s = (cudaStream_t)stream;
#define GVX_COS_COORDS(T)                                                                                    \
  switch (coords) {                                                                                         \
    case GVX_PTETAPHIM: return dispatch_costheta<T, C_PTETAPHIM>(v1, v2, n, hm, m_bins, hc, c_bins, m_out, cos_out, s); \
    case GVX_PXPYPZE: return dispatch_costheta<T, C_PXPYPZE>(v1, v2, n, hm, m_bins, hc, c_bins, m_out, cos_out, s);     \
    case GVX_PXPYPZM: return dispatch_costheta<T, C_PXPYPZM>(v1, v2, n, hm, m_bins, hc, c_bins, m_out, cos_out, s);     \
    default: return dispatch_costheta<T, C_PTETAPHIE>(v1, v2, n, hm, m_bins, hc, c_bins, m_out, cos_out, s);            \
  }
  if (dtype == GVX_F64) {
    GVX_COS_COORDS(double)
  }
  GVX_COS_COORDS(float)
#undef GVX_COS_COORDS
}

static gvx_status mass_histogram_impl(gvx_dtype dtype, gvx_coords coords, const gvx_vec4_cview* v1,
                                      const gvx_vec4_cview* v2, int64_t n, double lo, double hi, int32_t nbins,
                                      unsigned long long* bins, uint32_t flags, void* m_out,
                                      const gvx_vec4_view* boosted_out, gvx_stream_t stream,
                                      unsigned long long* const* peers, int32_t npeers, unsigned long long* mc,
                                      unsigned long long* work);

gvx_status gvx_mass_histogram(gvx_dtype dtype, gvx_coords coords, const gvx_vec4_cview* v1, const gvx_vec4_cview* v2,
                              int64_t n, double lo, double hi, int32_t nbins, unsigned long long* bins, uint32_t flags,
                              void* m_out, const gvx_vec4_view* boosted_out, gvx_stream_t stream) {
  return mass_histogram_impl(dtype, coords, v1, v2, n, lo, hi, nbins, bins, flags, m_out, boosted_out, stream,
                             nullptr, 0, nullptr, nullptr);
}

gvx_status gvx_mass_histogram_peers(gvx_dtype dtype, gvx_coords coords, const gvx_vec4_cview* v1,
                                    const gvx_vec4_cview* v2, int64_t n, double lo, double hi, int32_t nbins,
                                    unsigned long long* const* peer_bins, int32_t npeers,
                                    unsigned long long* mc_bins, unsigned long long* work, uint32_t flags,
                                    void* m_out, gvx_stream_t stream) {
  if (mc_bins ? !aligned(mc_bins, 8) : (!peer_bins || !aligned(peer_bins, 8) || npeers < 1 || npeers > 4096))
    return GVX_ERR_INVALID_ARGUMENT;
  if (!work || !aligned(work, 8)) return GVX_ERR_INVALID_ARGUMENT;
  // the kernels flush into `work`; each launch's last CTA pushes the totals to the sink
  return mass_histogram_impl(dtype, coords, v1, v2, n, lo, hi, nbins, nullptr, flags, m_out, nullptr, stream,
                             mc_bins ? nullptr : peer_bins, mc_bins ? 0 : npeers, mc_bins, work);
}

static gvx_status mass_histogram_impl(gvx_dtype dtype, gvx_coords coords, const gvx_vec4_cview* v1,
                                      const gvx_vec4_cview* v2, int64_t n, double lo, double hi, int32_t nbins,
                                      unsigned long long* bins, uint32_t flags, void* m_out,
                                      const gvx_vec4_view* boosted_out, gvx_stream_t stream,
                                      unsigned long long* const* peers, int32_t npeers, unsigned long long* mc,
                                      unsigned long long* work) {
  if (!valid_dtype(dtype) || !valid_coords(coords) || n < 0) return GVX_ERR_INVALID_ARGUMENT;
  if (nbins < 1 || nbins > (1 << 28) || !isfinite(lo) || !isfinite(hi) || !(lo < hi)) return GVX_ERR_INVALID_ARGUMENT;
  if ((flags & ~GVX_HIST_BOOST_TO_CM) != 0u) return GVX_ERR_INVALID_ARGUMENT;
  bool cm = (flags & GVX_HIST_BOOST_TO_CM) != 0u;
  if (boosted_out && !cm) return GVX_ERR_INVALID_ARGUMENT;
  if (n == 0) return GVX_OK;
  size_t es = dsize(dtype);
  const bool sink = peers != nullptr || mc != nullptr;  // fused reduction: counts go to the sink, not `bins`
  if (!view_ok<4>(v1, es) || !view_ok<4>(v2, es) || (!sink && (!bins || !aligned(bins, 8))))
    return GVX_ERR_INVALID_ARGUMENT;
  if (m_out && !aligned(m_out, es)) return GVX_ERR_INVALID_ARGUMENT;
  if (boosted_out && !out_view_ok(boosted_out, es)) return GVX_ERR_INVALID_ARGUMENT;
  HistParams hp = make_hist_params(lo, hi, nbins);
  hp.peers = peers;
  hp.npeers = npeers;
  hp.mc = mc;
  hp.work = work;
  cudaStream_t s = (cudaStream_t)stream;
#define GVX_HIST_DISPATCH(T, C)                                                                                  \
  (cm ? dispatch_hist<T, C, true>(v1, v2, n, hp, bins, m_out, boosted_out, s)                       \
      : dispatch_hist<T, C, false>(v1, v2, n, hp, bins, m_out, boosted_out, s))
#define GVX_HIST_COORDS(T)                                            \
  switch (coords) {                                                  \
    case GVX_PTETAPHIM: return GVX_HIST_DISPATCH(T, C_PTETAPHIM);    \
    case GVX_PXPYPZE: return GVX_HIST_DISPATCH(T, C_PXPYPZE);        \
    case GVX_PXPYPZM: return GVX_HIST_DISPATCH(T, C_PXPYPZM);        \
    default: return GVX_HIST_DISPATCH(T, C_PTETAPHIE);               \
  }
  if (dtype == GVX_F64) {
    GVX_HIST_COORDS(double)
  }
  GVX_HIST_COORDS(float)
#undef GVX_HIST_COORDS
#undef GVX_HIST_DISPATCH
}


// ---------------------------------------------------------------------------
// Mixed-coordinate entry points (ABI v7): v1 in coords1, v2 in coords2. Equal
// systems take the single-system entry points above (same kernels, same bits).
// ---------------------------------------------------------------------------
gvx_status gvx_invariant_mass_mixed(gvx_dtype dtype, gvx_coords coords1, gvx_coords coords2,
                                    const gvx_vec4_cview* v1, const gvx_vec4_cview* v2, void* m_out, int64_t n,
                                    gvx_stream_t stream) {
  if (!valid_coords(coords1) || !valid_coords(coords2)) return GVX_ERR_INVALID_ARGUMENT;
  if (coords1 == coords2) return gvx_invariant_mass(dtype, coords1, v1, v2, m_out, n, stream);
  if (!valid_dtype(dtype) || n < 0) return GVX_ERR_INVALID_ARGUMENT;
  if (n == 0) return GVX_OK;
  const size_t es = dsize(dtype);
  if (!view_ok<4>(v1, es) || !view_ok<4>(v2, es) || !m_out || !aligned(m_out, es)) return GVX_ERR_INVALID_ARGUMENT;
  const HistParams none = make_hist_params(0.0, 1.0, 1);
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == GVX_F64)
    return launch_mixed<double, PM_MASS>(v1, v2, coords1, coords2, n, none, nullptr, m_out, none, nullptr, nullptr,
                                         nullptr, s);
  return launch_mixed<float, PM_MASS>(v1, v2, coords1, coords2, n, none, nullptr, m_out, none, nullptr, nullptr,
                                      nullptr, s);
}

gvx_status gvx_mass_histogram_mixed(gvx_dtype dtype, gvx_coords coords1, gvx_coords coords2,
                                    const gvx_vec4_cview* v1, const gvx_vec4_cview* v2, int64_t n, double lo,
                                    double hi, int32_t nbins, unsigned long long* bins, uint32_t flags, void* m_out,
                                    const gvx_vec4_view* boosted_out, gvx_stream_t stream) {
  if (!valid_coords(coords1) || !valid_coords(coords2)) return GVX_ERR_INVALID_ARGUMENT;
  if (coords1 == coords2)
    return gvx_mass_histogram(dtype, coords1, v1, v2, n, lo, hi, nbins, bins, flags, m_out, boosted_out, stream);
  if (!valid_dtype(dtype) || n < 0) return GVX_ERR_INVALID_ARGUMENT;
  if (nbins < 1 || nbins > (1 << 28) || !isfinite(lo) || !isfinite(hi) || !(lo < hi)) return GVX_ERR_INVALID_ARGUMENT;
  if ((flags & ~GVX_HIST_BOOST_TO_CM) != 0u) return GVX_ERR_INVALID_ARGUMENT;
  const bool cm = (flags & GVX_HIST_BOOST_TO_CM) != 0u;
  if (boosted_out && !cm) return GVX_ERR_INVALID_ARGUMENT;
  if (n == 0) return GVX_OK;
  const size_t es = dsize(dtype);
  if (!view_ok<4>(v1, es) || !view_ok<4>(v2, es) || !bins || !aligned(bins, 8)) return GVX_ERR_INVALID_ARGUMENT;
  if (m_out && !aligned(m_out, es)) return GVX_ERR_INVALID_ARGUMENT;
  if (boosted_out && !out_view_ok(boosted_out, es)) return GVX_ERR_INVALID_ARGUMENT;
  const HistParams hp = make_hist_params(lo, hi, nbins);
  cudaStream_t s = (cudaStream_t)stream;
#define GVX_MIXED_HIST(T)                                                                                        \
  return cm ? launch_mixed<T, PM_HIST_CM>(v1, v2, coords1, coords2, n, hp, bins, m_out, hp, nullptr, nullptr,   \
                                          boosted_out, s)                                                        \
            : launch_mixed<T, PM_HIST>(v1, v2, coords1, coords2, n, hp, bins, m_out, hp, nullptr, nullptr, nullptr, s);
  if (dtype == GVX_F64) {
    GVX_MIXED_HIST(double)
  }
  GVX_MIXED_HIST(float)
#undef GVX_MIXED_HIST
}

gvx_status gvx_pair_histograms_mixed(gvx_dtype dtype, gvx_coords coords1, gvx_coords coords2,
                                     const gvx_vec4_cview* v1, const gvx_vec4_cview* v2, int64_t n, double lo,
                                     double hi, int32_t nbins, unsigned long long* lab_bins,
                                     unsigned long long* cm_bins, void* m_out, void* cm_m_out, gvx_stream_t stream) {
  if (!valid_coords(coords1) || !valid_coords(coords2)) return GVX_ERR_INVALID_ARGUMENT;
  if (coords1 == coords2)
    return gvx_pair_histograms(dtype, coords1, v1, v2, n, lo, hi, nbins, lab_bins, cm_bins, m_out, cm_m_out, stream);
  if (!valid_dtype(dtype) || n < 0) return GVX_ERR_INVALID_ARGUMENT;
  if (nbins < 1 || nbins > (1 << 28) || !isfinite(lo) || !isfinite(hi) || !(lo < hi)) return GVX_ERR_INVALID_ARGUMENT;
  if (n == 0) return GVX_OK;
  const size_t es = dsize(dtype);
  if (!view_ok<4>(v1, es) || !view_ok<4>(v2, es) || !lab_bins || !aligned(lab_bins, 8) || !cm_bins ||
      !aligned(cm_bins, 8))
    return GVX_ERR_INVALID_ARGUMENT;
  if ((m_out && !aligned(m_out, es)) || (cm_m_out && !aligned(cm_m_out, es))) return GVX_ERR_INVALID_ARGUMENT;
  const HistParams hp = make_hist_params(lo, hi, nbins);
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == GVX_F64)
    return launch_mixed<double, PM_BOTH>(v1, v2, coords1, coords2, n, hp, lab_bins, m_out, hp, cm_bins, cm_m_out,
                                         nullptr, s);
  return launch_mixed<float, PM_BOTH>(v1, v2, coords1, coords2, n, hp, lab_bins, m_out, hp, cm_bins, cm_m_out,
                                      nullptr, s);
}

gvx_status gvx_pair_histograms_boost_mixed(gvx_dtype dtype, gvx_coords coords1, gvx_coords coords2,
                                           const gvx_vec4_cview* v1, const gvx_vec4_cview* v2, int64_t n, double lo,
                                           double hi, int32_t nbins, unsigned long long* lab_bins,
                                           unsigned long long* cm_bins, void* m_out, void* cm_m_out,
                                           const gvx_vec4_cview* bv, const gvx_vec3_cview* beta,
                                           const gvx_vec4_view* bout, int64_t nb, gvx_stream_t stream) {
  if (!valid_coords(coords1) || !valid_coords(coords2)) return GVX_ERR_INVALID_ARGUMENT;
  if (coords1 == coords2)
    return gvx_pair_histograms_boost(dtype, coords1, v1, v2, n, lo, hi, nbins, lab_bins, cm_bins, m_out, cm_m_out,
                                     bv, beta, bout, nb, stream);
  // validate both halves before enqueueing either
  if (!valid_dtype(dtype) || n < 0 || nb < 0) return GVX_ERR_INVALID_ARGUMENT;
  if (nbins < 1 || nbins > (1 << 28) || !isfinite(lo) || !isfinite(hi) || !(lo < hi)) return GVX_ERR_INVALID_ARGUMENT;
  const size_t es = dsize(dtype);
  if (nb > 0 && (!view_ok<4>(bv, es) || !view_ok<3>(beta, es) || !out_view_ok(bout, es)))
    return GVX_ERR_INVALID_ARGUMENT;
  if (n > 0 && (!view_ok<4>(v1, es) || !view_ok<4>(v2, es) || !lab_bins || !aligned(lab_bins, 8) || !cm_bins ||
                !aligned(cm_bins, 8)))
    return GVX_ERR_INVALID_ARGUMENT;
  if ((m_out && !aligned(m_out, es)) || (cm_m_out && !aligned(cm_m_out, es))) return GVX_ERR_INVALID_ARGUMENT;
  gvx_status st = n > 0 ? gvx_pair_histograms_mixed(dtype, coords1, coords2, v1, v2, n, lo, hi, nbins, lab_bins,
                                                    cm_bins, m_out, cm_m_out, stream)
                        : GVX_OK;
  if (st != GVX_OK || nb == 0) return st;
  return gvx_boost(dtype, bv, beta, bout, nb, stream);
}

}  // extern "C"
