// Jagged dimuon, one kernel with an L2 prefetch pipeline (probe for VERDICT r1 #8).
// The product kernel (k_dimuon_compact) serialises three dependent DRAM round trips
// per tile (offsets -> charges -> muon rows) inside each CTA and relies on 5 CTAs
// per SM to overlap them. Here the memory system runs ahead of the arithmetic:
//   * each thread selects EPT CONSECUTIVE events: their offsets are 2 x 256-bit
//     loads, their charges a narrow window of the charge column;
//   * compaction once per thread (bit mask, warp scan, one shared atomic per warp)
//     into a circular shared-memory list of muon offsets;
//   * while selecting tile i+1 the kernel bulk-prefetches (cp.async.bulk.prefetch.L2)
//     the offsets of tile i+2G... and the charges of the next tile, and the two muon
//     rows of every selected event; the mass phase then walks entries selected one
//     iteration earlier (L2 hits), full passes of NT entries only (the remainder is
//     carried to the next tile), so no pass runs with a few lanes busy.
// Timed against k_dimuon_compact on the same events; histograms must be equal bit
// for bit. Standalone probe, not product code.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cstring>
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

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// [a, b) byte range, widened to 16-B alignment
__device__ __forceinline__ void prefetch_range(const char* a, const char* b) {
  const uintptr_t lo = (uintptr_t)a & ~(uintptr_t)15, hi = ((uintptr_t)b + 15) & ~(uintptr_t)15;
  if (hi > lo) prefetch_l2((const void*)lo, (uint32_t)(hi - lo));
}
template <int EPT>
__device__ __forceinline__ void ld_offs(const int64_t* p, int64_t (&o)[EPT + 1]) {
#pragma unroll
  for (int h = 0; h < EPT; h += 4)
    asm("ld.global.nc.L1::no_allocate.v4.s64 {%0,%1,%2,%3}, [%4];"
        : "=l"(o[h]), "=l"(o[h + 1]), "=l"(o[h + 2]), "=l"(o[h + 3]) : "l"(p + h));
  o[EPT] = __ldg(p + EPT);
}

// PF bits: 1 prefetch the selected muon rows, 2 the offsets / charges of later tiles.
// U: list entries per thread per mass pass (their gathers in flight together).
template <typename T, int ET, int NT, int MINB, int PF, int CAP, int U = 1, typename LT = int64_t>
__global__ void __launch_bounds__(NT, MINB) k_dimuon_pf(const T* __restrict__ mu, const int32_t* __restrict__ q,
                                                        const int64_t* __restrict__ offsets, int64_t n_events,
                                                        HistParams hp, unsigned long long* __restrict__ bins) {
  constexpr int EPT = ET / NT;
  static_assert((EPT % 4 == 0 && EPT <= 16) && (CAP & (CAP - 1)) == 0 && CAP >= 2 * ET + NT * U, "geometry");
  extern __shared__ __align__(16) unsigned char smem[];
  LT* s_mo = reinterpret_cast<LT*>(smem);                         // CAP muon offsets (circular)
  unsigned int* s_hist = reinterpret_cast<unsigned int*>(s_mo + CAP);
  __shared__ int s_tail;
  const int nb2 = hp.nbins + 2;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int b = tid; b < nb2; b += NT) s_hist[b] = 0u;
  if (tid == 0) s_tail = 0;
  const int64_t ntiles = (n_events + ET - 1) / ET;
  const int64_t G = gridDim.x;
  constexpr int RB = 4 * (int)sizeof(T);  // bytes per muon row
  if ((PF & 2) && tid == 0) {
    for (int d = 0; d < 2; ++d) {
      const int64_t t = blockIdx.x + d * G;
      if (t < ntiles) {
        const int64_t e0 = t * ET, e1 = min(e0 + ET, n_events);
        prefetch_range((const char*)(offsets + e0), (const char*)(offsets + e1 + 1));
      }
    }
  }
  __syncthreads();
  int head = 0, mark = 0;  // mark: the list tail before this iteration's selection
  bool pre = false;
  T pa[4], pb[4];
  for (int64_t tile = blockIdx.x; ; tile += G) {
    const bool have = tile < ntiles;
    if (have) {
      // ---- A: select this tile, append to the list, prefetch the selected rows
      const int64_t e0 = tile * ET;
      const int ne = (int)min((int64_t)ET, n_events - e0);
      int64_t o[EPT + 1];
      const int lb = tid * EPT;
      if (ne == ET) {
        ld_offs<EPT>(offsets + e0 + lb, o);
      } else {
#pragma unroll
        for (int k = 0; k <= EPT; ++k) o[k] = lb + k <= ne ? __ldg(offsets + e0 + lb + k) : 0;
      }
      unsigned int mask = 0u;
      int32_t qa[EPT], qb[EPT];
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const bool two = lb + k < ne && o[k + 1] - o[k] == 2;
        qa[k] = qb[k] = 0;
        if (two) {
          qa[k] = __ldg(q + o[k]);
          qb[k] = __ldg(q + o[k] + 1);
        }
      }
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const bool sel = ((qa[k] ^ qb[k]) < 0) & (qa[k] != 0) & (qb[k] != 0);
        mask |= (unsigned int)sel << k;
      }
      const int cnt = __popc(mask);
      int incl = cnt;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
      }
      int base = 0;
      if (lane == 31 && incl) base = atomicAdd(&s_tail, incl);
      base = __shfl_sync(0xffffffffu, base, 31) + incl - cnt;
#pragma unroll
      for (int k = 0; k < EPT; ++k)
        if (mask & (1u << k)) {
          s_mo[base++ & (CAP - 1)] = (LT)o[k];
          if (PF & 1) prefetch_l2(mu + 4 * o[k], 2 * RB);
        }
      if ((PF & 2) && tid == NT - 1) {  // the next tile's charges, the offsets two tiles ahead
        const int64_t t1 = tile + G, t2 = tile + 2 * G;
        if (t1 < ntiles) {
          const int64_t a0 = t1 * ET, a1 = min(a0 + ET, n_events);
          prefetch_range((const char*)(q + __ldg(offsets + a0)), (const char*)(q + __ldg(offsets + a1)));
        }
        if (t2 < ntiles) {
          const int64_t b0 = t2 * ET, b1 = min(b0 + ET, n_events);
          prefetch_range((const char*)(offsets + b0), (const char*)(offsets + b1 + 1));
        }
      }
    }
    __syncthreads();
    // ---- B: masses of entries [head, mark) in full passes (everything on the last tile)
    const int tail = s_tail;  // stable until the next selection
    const int avail = (have ? mark : tail) - head;
    const int take = have ? avail / (NT * U) * (NT * U) : avail;
    mark = tail;
    for (int j0 = tid; j0 < take; j0 += NT * U) {
      T a[U][4], b[U][4];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int j = j0 + u * NT;
        if ((PF & 4) && j0 == tid && u == 0 && pre) {
#pragma unroll
          for (int c = 0; c < 4; ++c) { a[0][c] = pa[c]; b[0][c] = pb[c]; }
        } else if (j < take) {
          const int64_t oo = s_mo[(head + j) & (CAP - 1)];
          ld_gather(mu + 4 * oo, a[u]);
          ld_gather(mu + 4 * oo + 4, b[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (j0 + u * NT >= take) break;
        const T M = event_mass<T, C_PTETAPHIM>(a[u], b[u]);
        atomicAdd(&s_hist[find_bin(M, hp)], 1u);
      }
    }
    head += take;
    if (!have) break;
    if (PF & 4) {  // the rows of the next mass pass's first entry, loaded while the next tile is selected
      pre = tail - head >= NT;
      if (pre) {
        const int64_t oo = s_mo[(head + tid) & (CAP - 1)];
        ld_gather(mu + 4 * oo, pa);
        ld_gather(mu + 4 * oo + 4, pb);
      }
    }
    __syncthreads();  // list slots of [head - take, head) may be reused by the next A
  }
  __syncthreads();
  for (int b = tid; b < nb2; b += NT) {
    const unsigned int c = s_hist[b];
    if (c) atomicAdd(&bins[b], (unsigned long long)c);
  }
}


// Warp-specialised variant: NS selection warps feed NM mass warps through the circular
// list with no CTA-wide barrier (selection warps sync among themselves with a named
// barrier per tile and publish the list tail; mass warps claim 32 entries at a time).
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
template <typename T, int ET, int NS, int NM, int CAP, int MINB>
__global__ void __launch_bounds__(32 * (NS + NM), MINB) k_dimuon_ws(const T* __restrict__ mu, const int32_t* __restrict__ q,
                                                              const int64_t* __restrict__ offsets, int64_t n_events,
                                                              HistParams hp, unsigned long long* __restrict__ bins) {
  constexpr int NST = NS * 32, EPT = ET / NST;
  static_assert(ET % NST == 0 && EPT % 4 == 0 && (CAP & (CAP - 1)) == 0 && CAP >= 2 * ET + 64 * NM, "geometry");
  extern __shared__ __align__(128) unsigned char smem[];
  uint32_t* s_mo = reinterpret_cast<uint32_t*>(smem);
  unsigned int* s_hist = reinterpret_cast<unsigned int*>(s_mo + CAP);
  __shared__ int s_reserve, s_claim;
  __shared__ volatile int s_tail, s_done;
  __shared__ volatile int s_pos[NM];
  const int nb2 = hp.nbins + 2;
  for (int b = threadIdx.x; b < nb2; b += blockDim.x) s_hist[b] = 0u;
  if (threadIdx.x == 0) { s_reserve = 0; s_claim = 0; s_tail = 0; s_done = 0; }
  if (threadIdx.x < NM) s_pos[threadIdx.x] = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t first = __ldg(offsets);
  const int64_t ntiles = (n_events + ET - 1) / ET;
  const int64_t G = gridDim.x;
  auto tile_events = [&](int64_t t) { return n_events - t * ET < ET ? n_events - t * ET : (int64_t)ET; };
  if (warp < NS) {
    const int tid = threadIdx.x;
    if (tid == 0)
      for (int64_t t = blockIdx.x; t < ntiles && t < blockIdx.x + 2 * G; t += G)
        prefetch_range((const char*)(offsets + t * ET), (const char*)(offsets + t * ET + tile_events(t) + 1));
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += G) {
      const int64_t e0 = tile * ET;
      const int ne = (int)tile_events(tile);
      const int lb = tid * EPT;
      int64_t o[EPT + 1];
      if (ne == ET) {
        ld_offs<EPT>(offsets + e0 + lb, o);
      } else {
#pragma unroll
        for (int k = 0; k <= EPT; ++k) o[k] = lb + k <= ne ? __ldg(offsets + e0 + lb + k) : 0;
      }
      int32_t qa[EPT], qb[EPT];
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        qa[k] = qb[k] = 0;
        if (lb + k < ne && o[k + 1] - o[k] == 2) {
          qa[k] = __ldg(q + o[k]);
          qb[k] = __ldg(q + o[k] + 1);
        }
      }
      unsigned int mask = 0u;
#pragma unroll
      for (int k = 0; k < EPT; ++k)
        mask |= (unsigned int)(((qa[k] ^ qb[k]) < 0) & (qa[k] != 0) & (qb[k] != 0)) << k;
      const int cnt = __popc(mask);
      int incl = cnt;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
      }
      int base = 0;
      if (lane == 31 && incl) {
        base = atomicAdd(&s_reserve, incl);
        // capacity: the oldest entry still held by a mass warp must stay CAP - ET behind
        for (;;) {
          int mn = s_pos[0];
#pragma unroll
          for (int w = 1; w < NM; ++w) mn = min(mn, (int)s_pos[w]);
          if (base + incl - mn <= CAP) break;
          __nanosleep(64);
        }
      }
      base = __shfl_sync(0xffffffffu, base, 31) + incl - cnt;
#pragma unroll
      for (int k = 0; k < EPT; ++k)
        if (mask & (1u << k)) s_mo[base++ & (CAP - 1)] = (uint32_t)(o[k] - first);
      __threadfence_block();
      named_sync(1, NST);
      if (tid == 0) {
        s_tail = s_reserve;
        const int64_t t1 = tile + G, t2 = tile + 2 * G;
        if (t1 < ntiles) prefetch_range((const char*)(q + __ldg(offsets + t1 * ET)), (const char*)(q + __ldg(offsets + t1 * ET + tile_events(t1))));
        if (t2 < ntiles) prefetch_range((const char*)(offsets + t2 * ET), (const char*)(offsets + t2 * ET + tile_events(t2) + 1));
      }
    }
    named_sync(1, NST);
    if (threadIdx.x == 0) {
      __threadfence_block();
      s_done = 1;
    }
  } else {
    const int mw = warp - NS;
    for (;;) {
      int c = 0;
      if (lane == 0) {
        c = atomicAdd(&s_claim, 32);
        s_pos[mw] = c;
        while (s_tail < c + 32 && !s_done) __nanosleep(32);
      }
      c = __shfl_sync(0xffffffffu, c, 0);
      __threadfence_block();
      const int tail = s_tail;  // >= c + 32, or final (producers done)
      if (c >= tail) break;
      const int j = c + lane;
      if (j < tail) {
        const int64_t oo = (int64_t)s_mo[j & (CAP - 1)] + first;
        T a[4], b[4];
        ld_gather(mu + 4 * oo, a);
        ld_gather(mu + 4 * oo + 4, b);
        const T M = event_mass<T, C_PTETAPHIM>(a, b);
        atomicAdd(&s_hist[find_bin(M, hp)], 1u);
      }
    }
    if (lane == 0) s_pos[mw] = 0x7fffffff;
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb2; b += blockDim.x) {
    const unsigned int c = s_hist[b];
    if (c) atomicAdd(&bins[b], (unsigned long long)c);
  }
}

template <typename K>
int resident(K k, int block, size_t smem) {
  int per = 0, sms = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, block, smem));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  return per * sms;
}

template <typename T>
void run(int64_t n) {
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
  CK(cudaMalloc(&mu, m * 4 * sizeof(T)));
  CK(cudaMalloc(&q, m * 4));
  gen_muons<T><<<1184, 256>>>(mu, q, m);
  CK(cudaDeviceSynchronize());
  printf("%s: events %lld muons %lld\n", sizeof(T) == 8 ? "f64" : "f32", (long long)n, (long long)m);
  const HistParams hp = make_hist_params(0.25, 300.0, 1000);
  unsigned long long* bins;
  CK(cudaMalloc(&bins, 1002 * 8));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  std::vector<unsigned long long> ref(1002), got(1002);
  auto timeit = [&](auto launch, const char* name, std::vector<unsigned long long>& out) {
    std::vector<float> ts;
    for (int r = 0; r < 9; ++r) {
      CK(cudaMemset(bins, 0, 1002 * 8));
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    CK(cudaMemcpy(out.data(), bins, 1002 * 8, cudaMemcpyDeviceToHost));
    printf("  %-44s best %.4f ms  median %.4f ms  %s\n", name, ts[0], ts[4],
           &out == &ref ? "" : (out == ref ? "bins equal" : "BINS DIFFER"));
  };
  {
    constexpr int MB = sizeof(T) == 8 ? 5 : 5;
    auto kk = k_dimuon_compact<T, true, 2048, 256, 1, MB>;
    const size_t sm = dimuon_compact_smem<2048>(1002);
    CK(cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const int grid = std::min<int64_t>(resident(kk, 256, sm), (n + 2047) / 2048);
    View4<T> v{{mu, mu + 1, mu + 2, mu + 3}, 4};
    timeit([&] { kk<<<grid, 256, sm>>>(v, q, off, n, hp, bins, (T*)nullptr); }, "product k_dimuon_compact", ref);
  }
  auto wsvar = [&](auto kk, int et, int cap, int nt, const char* name, int cps) {
    const size_t sm = (size_t)cap * 4 + 1002 * 4;
    CK(cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int grid = std::min<int64_t>(std::min(resident(kk, nt, sm), cps * sms), (n + et - 1) / et);
    char buf[128];
    snprintf(buf, sizeof buf, "%s (grid %d)", name, grid);
    timeit([&] { kk<<<grid, nt, sm>>>(mu, q, off, n, hp, bins); }, buf, got);
  };
  auto variant = [&](auto kk, int et, int cap, const char* name, int cps, int esz) {
    const int nt = strstr(name, "NT128") ? 128 : strstr(name, "NT64") ? 64 : 256;
    const size_t sm = (size_t)cap * esz + 1002 * 4;
    (void)et;
    CK(cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int grid = std::min<int64_t>(std::min(resident(kk, nt, sm), cps * sms), (n + et - 1) / et);
    char buf[128];
    snprintf(buf, sizeof buf, "%s (grid %d)", name, grid);
    timeit([&] { kk<<<grid, nt, sm>>>(mu, q, off, n, hp, bins); }, buf, got);
  };
  variant(k_dimuon_pf<T, 1024, 128, 8, 2, 4096, 1, uint32_t>, 1024, 4096, "pf2 ET1024 NT128 minb8 cps8 uint32_t", 8, 4);
  variant(k_dimuon_pf<T, 2048, 256, 4, 2, 8192, 1, uint32_t>, 2048, 8192, "pf2 ET2048 NT256 minb4 cps4 uint32_t", 4, 4);
  wsvar(k_dimuon_ws<T, 1024, 4, 4, 4096, 4>, 1024, 4096, 256, "ws ET1024 4+4 cps4", 4);
  wsvar(k_dimuon_ws<T, 1024, 4, 4, 4096, 6>, 1024, 4096, 256, "ws ET1024 4+4 cps6", 6);
  wsvar(k_dimuon_ws<T, 512, 2, 2, 2048, 8>, 512, 2048, 128, "ws ET512 2+2 cps8", 8);
  wsvar(k_dimuon_ws<T, 512, 2, 4, 2048, 6>, 512, 2048, 192, "ws ET512 2+4 cps6", 6);
  wsvar(k_dimuon_ws<T, 1024, 4, 8, 4096, 4>, 1024, 4096, 384, "ws ET1024 4+8 cps4", 4);
  wsvar(k_dimuon_ws<T, 2048, 8, 8, 8192, 2>, 2048, 8192, 512, "ws ET2048 8+8 cps2", 2);
  CK(cudaFree(k)); CK(cudaFree(off)); CK(cudaFree(tmp)); CK(cudaFree(mu)); CK(cudaFree(q)); CK(cudaFree(bins));
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 100000000LL;
  const int which = argc > 2 ? atoi(argv[2]) : 3;  // bit 0: f64, bit 1: f32
  if (which & 1) run<double>(n);
  if (which & 2) run<float>(n);
  return 0;
}
