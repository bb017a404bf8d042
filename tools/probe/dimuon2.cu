// Jagged dimuon as two kernels (VERDICT r1 #8's "two-pass selection, then a dense
// pass"): K1 selects (offsets streamed, charges gathered) and appends the selected
// events' (muon offset, event index) to a list in a workspace; K2 walks the list
// densely — several list entries per thread, all their muon gathers in flight —
// computes the masses and bins them. Timed against the product's one-kernel
// k_dimuon_compact on the same events; histograms must be equal bit for bit.
// Standalone probe, not product code.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cub/cub.cuh>
#include "../../paper_2312_02756_b200/csrc/gvx_kernels.cuh"
using namespace gvx;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double u01(uint64_t h) { return ((h >> 11) + 0.5) * (1.0 / 9007199254740992.0); }

__global__ void gen_counts(int64_t* k, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    double u = u01(mix(e * 7 + 1));
    k[e] = (u >= 0.25) + (u >= 0.55) + (u >= 0.85) + (u >= 0.95);
  }
}
template <typename T>
__global__ void gen_muons(T* mu, int32_t* q, int64_t m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h0 = mix(i * 5 + 11), h1 = mix(h0 + 1), h2 = mix(h0 + 2), h3 = mix(h0 + 3);
    double g = sqrt(-2.0 * log(u01(h0))) * cos(6.283185307179586 * u01(h1));
    mu[4 * i] = (T)fmin(fmax(30.0 * exp(0.5 * g), 2.0), 2000.0);
    mu[4 * i + 1] = (T)(-2.5 + 5.0 * u01(h2));
    mu[4 * i + 2] = (T)(-3.141592653589793 + 6.283185307179586 * u01(h3));
    mu[4 * i + 3] = (T)0.1056583755;
    q[i] = (mix(h0 + 9) & 1) ? 1 : -1;
  }
}

struct Entry { int64_t o, e; };

// K1: select. Thread t of a CTA takes events e0 + t + k*NT (k < EPT) of its ET-event tile.
template <int ET, int NT>
__global__ void __launch_bounds__(NT) k_select(const int32_t* __restrict__ q, const int64_t* __restrict__ off,
                                               int64_t n, Entry* __restrict__ list, unsigned long long* count,
                                               double* m_out) {
  constexpr int EPT = ET / NT;
  __shared__ int s_n;
  __shared__ unsigned long long s_base;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int64_t e0 = (int64_t)blockIdx.x * ET; e0 < n; e0 += (int64_t)gridDim.x * ET) {
    if (tid == 0) s_n = 0;
    int64_t o[EPT];
    bool two[EPT];
    int32_t qa[EPT], qb[EPT];
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int64_t e = e0 + tid + k * NT;
      o[k] = 0;
      two[k] = false;
      if (e < n) {
        o[k] = __ldg(off + e);
        two[k] = __ldg(off + e + 1) - o[k] == 2;
      }
    }
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      qa[k] = qb[k] = 0;
      if (two[k]) {
        qa[k] = ld_gather1(q + o[k]);
        qb[k] = ld_gather1(q + o[k] + 1);
      }
    }
    unsigned int mask = 0u;
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const bool sel = two[k] & ((qa[k] ^ qb[k]) < 0) & (qa[k] != 0) & (qb[k] != 0);
      mask |= (unsigned int)sel << k;
      const int64_t e = e0 + tid + k * NT;
      if (!sel && m_out && e < n) m_out[e] = NAN;
    }
    const int cnt = __popc(mask);
    int incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += v;
    }
    __syncthreads();  // s_n reset visible
    int wbase = 0;
    if (lane == 31 && incl) wbase = atomicAdd(&s_n, incl);
    wbase = __shfl_sync(0xffffffffu, wbase, 31);
    __syncthreads();
    if (tid == 0) s_base = s_n ? atomicAdd(count, (unsigned long long)s_n) : 0ull;
    __syncthreads();
    int64_t pos = (int64_t)s_base + wbase + incl - cnt;
#pragma unroll
    for (int k = 0; k < EPT; ++k)
      if (mask & (1u << k)) list[pos++] = Entry{o[k], e0 + tid + k * NT};
    __syncthreads();
  }
}

// K2: dense pass over the list, U entries per thread per iteration, all gathers first.
template <typename T, int U, int MINB>
__global__ void __launch_bounds__(256, MINB) k_listmass(const T* __restrict__ mu, const Entry* __restrict__ list,
                                                        const unsigned long long* count, HistParams hp,
                                                        unsigned long long* __restrict__ bins, T* m_out) {
  extern __shared__ unsigned int sh[];
  const int nb2 = hp.nbins + 2;
  for (int b = threadIdx.x; b < nb2; b += blockDim.x) sh[b] = 0u;
  __syncthreads();
  const int64_t n = (int64_t)*count;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j0 < n; j0 += nthr * U) {
    Entry en[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = j0 + u * nthr;
      en[u] = j < n ? list[j] : Entry{-1, -1};
    }
    T a[U][4], b[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (en[u].o >= 0) {
        ld_gather(mu + 4 * en[u].o, a[u]);
        ld_gather(mu + 4 * en[u].o + 4, b[u]);
      }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (en[u].o < 0) break;
      const T M = event_mass<T, C_PTETAPHIM>(a[u], b[u]);
      atomicAdd(&sh[find_bin(M, hp)], 1u);
      if (m_out) m_out[en[u].e] = M;
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb2; b += blockDim.x)
    if (sh[b]) atomicAdd(&bins[b], (unsigned long long)sh[b]);
}

template <typename K>
int resident(K k, int block, size_t smem) {
  int per = 0, sms = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, block, smem));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  return per * sms;
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 100000000LL;
  using T = double;
  int64_t *k, *off;
  CK(cudaMalloc(&k, n * 8));
  CK(cudaMalloc(&off, (n + 1) * 8));
  gen_counts<<<1184, 256>>>(k, n);
  CK(cudaMemset(off, 0, 8));
  void* tmp = nullptr;
  size_t tb = 0;
  cub::DeviceScan::InclusiveSum(tmp, tb, k, off + 1, n);
  CK(cudaMalloc(&tmp, tb));
  cub::DeviceScan::InclusiveSum(tmp, tb, k, off + 1, n);
  int64_t m;
  CK(cudaMemcpy(&m, off + n, 8, cudaMemcpyDeviceToHost));
  T* mu;
  int32_t* q;
  CK(cudaMalloc(&mu, m * 32));
  CK(cudaMalloc(&q, m * 4));
  gen_muons<T><<<1184, 256>>>(mu, q, m);
  CK(cudaDeviceSynchronize());
  printf("events %lld muons %lld\n", (long long)n, (long long)m);
  const HistParams hp = make_hist_params(0.25, 300.0, 1000);
  unsigned long long *bins, *count;
  CK(cudaMalloc(&bins, 1002 * 8));
  CK(cudaMalloc(&count, 16));
  Entry* list;
  CK(cudaMalloc(&list, (size_t)n / 4 * sizeof(Entry)));  // the recipe selects ~15 %
  cudaEvent_t e0, e1, e2;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventCreate(&e2));
  std::vector<unsigned long long> ref(1002), got(1002);
  // product one-kernel path
  {
    auto kk = k_dimuon_compact<T, true, 2048, 256, 1, 5>;
    const size_t sm = dimuon_compact_smem<2048>(1002);
    CK(cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const int grid = std::min<int64_t>(resident(kk, 256, sm), (n + 2047) / 2048);
    View4<T> v{{mu, mu + 1, mu + 2, mu + 3}, 4};
    std::vector<float> ts;
    for (int r = 0; r < 8; ++r) {
      CK(cudaMemset(bins, 0, 1002 * 8));
      CK(cudaEventRecord(e0));
      kk<<<grid, 256, sm>>>(v, q, off, n, hp, bins, (T*)nullptr);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    CK(cudaMemcpy(ref.data(), bins, 1002 * 8, cudaMemcpyDeviceToHost));
    printf("one kernel (k_dimuon_compact)         best %.4f ms  median %.4f ms\n", ts[0], ts[4]);
  }
  auto two = [&](auto ksel, auto kmass, const char* name, int et) {
    const int gsel = std::min<int64_t>(resident(ksel, 256, 0), (n + et - 1) / et);
    const int gmass = resident(kmass, 256, 1002 * 4);
    std::vector<float> ts, t1s;
    for (int r = 0; r < 8; ++r) {
      CK(cudaMemset(bins, 0, 1002 * 8));
      CK(cudaMemset(count, 0, 16));
      CK(cudaEventRecord(e0));
      ksel<<<gsel, 256>>>(q, off, n, list, count, (double*)nullptr);
      CK(cudaEventRecord(e1));
      kmass<<<gmass, 256, 1002 * 4>>>(mu, list, count, hp, bins, (T*)nullptr);
      CK(cudaEventRecord(e2));
      CK(cudaEventSynchronize(e2));
      CK(cudaGetLastError());
      float ms, m1;
      CK(cudaEventElapsedTime(&ms, e0, e2));
      CK(cudaEventElapsedTime(&m1, e0, e1));
      ts.push_back(ms);
      t1s.push_back(m1);
    }
    std::sort(ts.begin(), ts.end());
    std::sort(t1s.begin(), t1s.end());
    CK(cudaMemcpy(got.data(), bins, 1002 * 8, cudaMemcpyDeviceToHost));
    printf("%-38s best %.4f ms  median %.4f ms (select %.4f)  %s\n", name, ts[0], ts[4], t1s[4],
           got == ref ? "bins equal" : "BINS DIFFER");
  };
  two(k_select<2048, 256>, k_listmass<T, 2, 4>, "two kernels ET2048 U2 minb4", 2048);
  two(k_select<2048, 256>, k_listmass<T, 1, 4>, "two kernels ET2048 U1 minb4", 2048);
  two(k_select<2048, 256>, k_listmass<T, 2, 3>, "two kernels ET2048 U2 minb3", 2048);
  two(k_select<1024, 256>, k_listmass<T, 2, 4>, "two kernels ET1024 U2 minb4", 1024);
  two(k_select<4096, 256>, k_listmass<T, 2, 4>, "two kernels ET4096 U2 minb4", 4096);
  two(k_select<2048, 256>, k_listmass<T, 4, 2>, "two kernels ET2048 U4 minb2", 2048);
  return 0;
}
