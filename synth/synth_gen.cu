// synth_gen.cu — device twin of synth/__init__.py (the seeded input
// generator shared by the oracle and the CUDA path). It holds NONE of the
// method's arithmetic: it only draws events. Every operation mirrors the
// numpy implementation one for one with IEEE round-to-nearest basic
// operations and no contraction (__dadd_rn / __dmul_rn / __dsqrt_rn /
// floor / scalbn), so host and device produce identical bits for any global
// event index (tests/test_gpu_parity.py::test_synth_device_matches_host).
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
constexpr uint32_t STREAM_V1 = 1, STREAM_V2 = 2, STREAM_BOOST_P = 3, STREAM_BOOST_BETA = 4;
constexpr uint32_t STREAM_JAGGED_N = 5, STREAM_JAGGED_MU = 6, JAGGED_SLOTS = 8, STREAM_RES = 7;

__device__ __forceinline__ uint4 philox(uint64_t idx, uint32_t call, uint32_t stream, uint64_t seed) {
  uint32_t c0 = (uint32_t)idx, c1 = (uint32_t)(idx >> 32), c2 = call, c3 = stream;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
    uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    if (r < 9) { k0 += W0; k1 += W1; }
  }
  return make_uint4(c0, c1, c2, c3);
}

__device__ __forceinline__ double u01(uint32_t w) {
  return __dmul_rn(__dadd_rn((double)w, 0.5), 2.3283064365386963e-10);
}
__device__ __forceinline__ double normal4(uint4 w) {
  double s = __dadd_rn(__dadd_rn(__dadd_rn(u01(w.x), u01(w.y)), u01(w.z)), u01(w.w));
  return __dmul_rn(__dsub_rn(s, 2.0), 1.7320508075688772);
}

__constant__ double kExpCoef[14] = {
    1.6059043836821613e-10, 2.08767569878681e-09, 2.505210838544172e-08, 2.755731922398589e-07,
    2.7557319223985893e-06, 2.48015873015873e-05, 0.0001984126984126984, 0.001388888888888889,
    0.008333333333333333,   0.041666666666666664, 0.16666666666666666,  0.5, 1.0, 1.0};

__device__ __forceinline__ double exp_det(double x) {
  double k = floor(__dadd_rn(__dmul_rn(x, 1.4426950408889634), 0.5));
  double r = __dsub_rn(__dsub_rn(x, __dmul_rn(k, 0.693145751953125)), __dmul_rn(k, 1.4286068203094173e-06));
  double p = kExpCoef[0];
#pragma unroll
  for (int i = 1; i < 14; ++i) p = __dadd_rn(__dmul_rn(p, r), kExpCoef[i]);
  return scalbn(p, (int)k);
}

__device__ __forceinline__ void muon64(uint64_t idx, uint32_t stream, uint64_t seed, double (&o)[4]) {
  uint4 w0 = philox(idx, 0, stream, seed), w1 = philox(idx, 1, stream, seed);
  o[0] = exp_det(__dadd_rn(3.4011973816621555, __dmul_rn(0.5, normal4(w0))));
  o[1] = __dadd_rn(-2.5, __dmul_rn(5.0, u01(w1.x)));
  o[2] = __dadd_rn(-3.141592653589793, __dmul_rn(6.283185307179586, u01(w1.y)));
  o[3] = 0.1056583755;
}
template <typename T>
__device__ __forceinline__ void muon(uint64_t idx, uint32_t stream, uint64_t seed, T* out) {
  double o[4];
  muon64(idx, stream, seed, o);
#pragma unroll
  for (int k = 0; k < 4; ++k) out[k] = (T)o[k];
}

// Resonance admixture (see synth/__init__.py, resonance_pairs): with probability
// f_res the pair is re-drawn as a Z-like peak: muon 2 is put back to back in phi
// with pt chosen for a massless pair mass x (ratio-of-normals Breit-Wigner shape
// around 91.1876 GeV, half width 1.2476, kept in [60, 120]).
__device__ __forceinline__ void resonance(uint64_t idx, uint64_t seed, double f_res, const double (&a)[4],
                                          double (&b)[4]) {
  if (!(u01(philox(idx, 0, STREAM_RES, seed).x) < f_res)) return;
  const double z1 = normal4(philox(idx, 1, STREAM_RES, seed)), z2 = normal4(philox(idx, 2, STREAM_RES, seed));
  double x = __dadd_rn(91.1876, __dmul_rn(1.2476, __ddiv_rn(z1, z2)));
  if (!(x >= 60.0 && x <= 120.0)) x = __dadd_rn(91.1876, __dmul_rn(1.2476, z1));
  const double d = __dsub_rn(a[1], b[1]);
  const double ch = __dmul_rn(__dadd_rn(exp_det(d), exp_det(-d)), 0.5);
  b[0] = __ddiv_rn(__dmul_rn(x, x), __dmul_rn(__dmul_rn(2.0, a[0]), __dadd_rn(ch, 1.0)));
  const double phi2 = __dadd_rn(a[2], 3.141592653589793);
  b[2] = phi2 >= 3.141592653589793 ? __dsub_rn(phi2, 6.283185307179586) : phi2;
}

template <typename T>
__global__ void k_muon_pairs(uint64_t seed, uint64_t first, int64_t n, T* v1, T* v2, double f_res) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double a[4], b[4];
    const uint64_t idx = first + (uint64_t)i;
    muon64(idx, STREAM_V1, seed, a);
    muon64(idx, STREAM_V2, seed, b);
    if (f_res > 0.0) resonance(idx, seed, f_res, a, b);
#pragma unroll
    for (int k = 0; k < 4; ++k) { v1[4 * i + k] = (T)a[k]; v2[4 * i + k] = (T)b[k]; }
  }
}

template <typename T>
__global__ void k_boost_inputs(uint64_t seed, uint64_t first, int64_t n, T* v, T* beta) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t idx = first + (uint64_t)i;
    double px = __dmul_rn(30.0, normal4(philox(idx, 0, STREAM_BOOST_P, seed)));
    double py = __dmul_rn(30.0, normal4(philox(idx, 1, STREAM_BOOST_P, seed)));
    double pz = __dmul_rn(30.0, normal4(philox(idx, 2, STREAM_BOOST_P, seed)));
    double e = __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(px, px), __dmul_rn(py, py)), __dmul_rn(pz, pz)),
                                    0.011163692328303140));
    double gx = normal4(philox(idx, 0, STREAM_BOOST_BETA, seed));
    double gy = normal4(philox(idx, 1, STREAM_BOOST_BETA, seed));
    double gz = normal4(philox(idx, 2, STREAM_BOOST_BETA, seed));
    uint4 wm = philox(idx, 3, STREAM_BOOST_BETA, seed);
    double mag = __dmul_rn(0.99, fmax(fmax(u01(wm.x), u01(wm.y)), u01(wm.z)));
    double sc = __ddiv_rn(mag, __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)), __dmul_rn(gz, gz))));
    v[4 * i + 0] = (T)px;
    v[4 * i + 1] = (T)py;
    v[4 * i + 2] = (T)pz;
    v[4 * i + 3] = (T)e;
    beta[3 * i + 0] = (T)__dmul_rn(gx, sc);
    beta[3 * i + 1] = (T)__dmul_rn(gy, sc);
    beta[3 * i + 2] = (T)__dmul_rn(gz, sc);
  }
}

__global__ void k_jagged_counts(uint64_t seed, uint64_t first, int64_t n, int64_t* counts) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double u = u01(philox(first + (uint64_t)i, 0, STREAM_JAGGED_N, seed).x);
    counts[i] = (int64_t)(u >= 0.25) + (int64_t)(u >= 0.55) + (int64_t)(u >= 0.85) + (int64_t)(u >= 0.95);
  }
}

template <typename T>
__global__ void k_jagged_fill(uint64_t seed, uint64_t first, int64_t n, const int64_t* offsets, T* mu, int32_t* q) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = offsets[i], k = offsets[i + 1] - o;
    for (int64_t j = 0; j < k; ++j) {
      uint64_t idx = (first + (uint64_t)i) * JAGGED_SLOTS + (uint64_t)j;
      muon<T>(idx, STREAM_JAGGED_MU, seed, mu + 4 * (o + j));
      q[o + j] = u01(philox(idx, 2, STREAM_JAGGED_MU, seed).x) < 0.5 ? 1 : -1;
    }
  }
}

// K5: read-only streaming probe for the achievable HBM read
// bandwidth in the same run as the measurements it normalises: a bulk-copy
// (cp.async.bulk, TMA) ring, one CTA per SM, 6 stages of 16 KB, one producer
// lane, 8 consumer warps that read every 16 B of a stage (LDS.128 + xor) and
// release it — the best geometry of the pool probe (profiles/r01/tmaprobe.jsonl,
// 7.35-7.49 TB/s). Self-contained PTX (no product header).
namespace k5 {
constexpr int STAGE = 16384, STAGES = 6, NCW = 8;
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(sa(bar)), "r"(parity) : "memory");
}
}  // namespace k5

__global__ void __launch_bounds__(32 * (k5::NCW + 1)) k_stream_read(const char* __restrict__ src, int64_t ntiles,
                                                                   unsigned long long* __restrict__ sink) {
  using namespace k5;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&full[s])), "r"(1) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[s])), "r"(NCW) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      int it = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const int s = it % STAGES, k = it / STAGES;
        if (k > 0) {
          wait(&empty[s], (k - 1) & 1);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(STAGE)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
            ::"r"(sa(smem + s * STAGE)), "l"(src + t * STAGE), "r"(STAGE), "r"(sa(&full[s])), "l"(pol)
            : "memory");
      }
    }
  } else {
    unsigned long long acc = 0;
    int it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int s = it % STAGES, k = it / STAGES;
      wait(&full[s], k & 1);
      const int4* p = reinterpret_cast<const int4*>(smem + s * STAGE);
      for (int i = threadIdx.x - 32; i < STAGE / 16; i += NCW * 32) {
        const int4 v = p[i];
        acc ^= (unsigned long long)(unsigned)(v.x ^ v.y ^ v.z ^ v.w);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
    }
    for (int o = 16; o > 0; o >>= 1) acc ^= __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) atomicXor(sink, acc);
  }
}

int grid_of(int64_t n) {
  int64_t g = (n + 255) / 256;
  return (int)(g < 148 * 16 ? (g < 1 ? 1 : g) : 148 * 16);
}

}  // namespace

extern "C" {

// dtype: 0 = float32, 1 = float64. v1, v2: AoS [n][4] device buffers; v: [n][4],
// beta: [n][3]. Returns 0 or a cudaError_t value.
// f_res: fraction of resonance (Z-like) pairs, 0 for independent muons.
int gvx_synth_muon_pairs(int dtype, uint64_t seed, uint64_t first, int64_t n, void* v1, void* v2, void* stream,
                         double f_res) {
  if (n <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == 1) k_muon_pairs<double><<<grid_of(n), 256, 0, s>>>(seed, first, n, (double*)v1, (double*)v2, f_res);
  else k_muon_pairs<float><<<grid_of(n), 256, 0, s>>>(seed, first, n, (float*)v1, (float*)v2, f_res);
  return (int)cudaGetLastError();
}

int gvx_synth_boost_inputs(int dtype, uint64_t seed, uint64_t first, int64_t n, void* v, void* beta, void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == 1) k_boost_inputs<double><<<grid_of(n), 256, 0, s>>>(seed, first, n, (double*)v, (double*)beta);
  else k_boost_inputs<float><<<grid_of(n), 256, 0, s>>>(seed, first, n, (float*)v, (float*)beta);
  return (int)cudaGetLastError();
}

// Jagged events: per-event multiplicities (int64 [n]), then, given the
// exclusive prefix sum offsets [n+1] (relative to the shard), the muons
// (AoS [M][4]) and charges (int32 [M]).
int gvx_synth_jagged_counts(uint64_t seed, uint64_t first, int64_t n, void* counts, void* stream) {
  if (n <= 0) return 0;
  k_jagged_counts<<<grid_of(n), 256, 0, (cudaStream_t)stream>>>(seed, first, n, (int64_t*)counts);
  return (int)cudaGetLastError();
}
int gvx_synth_jagged_fill(int dtype, uint64_t seed, uint64_t first, int64_t n, const void* offsets, void* mu,
                          void* q, void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == 1)
    k_jagged_fill<double><<<grid_of(n), 256, 0, s>>>(seed, first, n, (const int64_t*)offsets, (double*)mu, (int32_t*)q);
  else
    k_jagged_fill<float><<<grid_of(n), 256, 0, s>>>(seed, first, n, (const int64_t*)offsets, (float*)mu, (int32_t*)q);
  return (int)cudaGetLastError();
}

// K5: stream `bytes` (the whole 16-KB tiles of it; 16-byte aligned) of device
// memory once; the XOR of the data lands in *sink (8 bytes of device memory).
int gvx_synth_stream_read(const void* buf, int64_t bytes, void* sink, void* stream) {
  const int64_t ntiles = bytes / k5::STAGE;
  if (ntiles < 1) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int smem = k5::STAGES * k5::STAGE + 2 * k5::STAGES * 8;
  cudaFuncSetAttribute(k_stream_read, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_stream_read<<<sms, 32 * (k5::NCW + 1), smem, (cudaStream_t)stream>>>((const char*)buf, ntiles,
                                                                        (unsigned long long*)sink);
  return (int)cudaGetLastError();
}

}  // extern "C"
