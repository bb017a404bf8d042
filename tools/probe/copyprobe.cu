// Copy-bandwidth probe (read+write streams, as the boost kernel does): 256-bit
// LDG/STG grid-stride vs a TMA ring (cp.async.bulk G2S in, bulk S2G out).
// Standalone measurement tool, not product code.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2312_02756_b200/csrc/gvx_tma.cuh"
using namespace gvx;

__global__ void copy256(const double* __restrict__ a, double* __restrict__ b, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    double x, y, z, w;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(x), "=d"(y), "=d"(z), "=d"(w) : "l"(a + 4 * i));
    asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(b + 4 * i), "d"(x), "d"(y), "d"(z), "d"(w) : "memory");
  }
}

// One thread per CTA moves tiles global->smem->global with bulk copies only.
template <int TILE, int STAGES>
__global__ void copy_tma(const char* __restrict__ a, char* __restrict__ b, int64_t ntiles) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * TILE);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < STAGES; ++s) tma::mbar_init(&full[s], 1);
  tma::fence_barrier_init();
  uint64_t pol = tma::policy_evict_first();
  int it = 0;
  int64_t t0 = blockIdx.x;
  // prologue: fill the ring
  for (int s = 0; s < STAGES && t0 + s * (int64_t)gridDim.x < ntiles; ++s) {
    tma::mbar_arrive_expect_tx(&full[s], TILE);
    tma::bulk_g2s(smem + s * TILE, a + (t0 + s * (int64_t)gridDim.x) * TILE, TILE, &full[s], pol);
  }
  for (int64_t t = t0; t < ntiles; t += gridDim.x, ++it) {
    int s = it % STAGES, k = it / STAGES;
    tma::mbar_wait(&full[s], k & 1);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(b + t * TILE),
                 "r"(tma::smem_u32(smem + s * TILE)), "r"(TILE) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    int64_t tn = t + STAGES * (int64_t)gridDim.x;
    if (tn < ntiles) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem stage read out by the store
      tma::mbar_arrive_expect_tx(&full[s], TILE);
      tma::bulk_g2s(smem + s * TILE, a + tn * TILE, TILE, &full[s], pol);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int TILE, int STAGES>
void run_tma(const char* a, char* b, size_t bytes, int sms, cudaEvent_t e0, cudaEvent_t e1) {
  auto k = copy_tma<TILE, STAGES>;
  size_t sm = (size_t)STAGES * TILE + STAGES * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 32, sm);
  for (int cps = 1; cps <= per && cps <= 4; ++cps) {
    int64_t nt = bytes / TILE;
    k<<<sms * cps, 32, sm>>>(a, b, nt);
    cudaDeviceSynchronize();
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); k<<<sms * cps, 32, sm>>>(a, b, nt); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("{\"probe\":\"copy_tma\",\"tile_kb\":%d,\"stages\":%d,\"ctas_per_sm\":%d,\"GBs_rw\":%.1f,\"err\":\"%s\"}\n",
           TILE / 1024, STAGES, cps, 2.0 * nt * TILE / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  size_t bytes = 4ull << 30;
  char *a, *b; cudaMalloc(&a, bytes); cudaMalloc(&b, bytes); cudaMemset(a, 1, bytes); cudaMemset(b, 0, bytes);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int bpsm : {2, 4, 8}) for (int bs : {256, 512}) {
    if (bpsm * bs > 2048) continue;
    copy256<<<sms * bpsm, bs>>>((const double*)a, (double*)b, bytes / 32);
    cudaDeviceSynchronize();
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); copy256<<<sms * bpsm, bs>>>((const double*)a, (double*)b, bytes / 32); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("{\"probe\":\"copy256\",\"grid\":%d,\"block\":%d,\"GBs_rw\":%.1f}\n", sms * bpsm, bs, 2.0 * bytes / best / 1e6);
  }
  run_tma<16384, 4>(a, b, bytes, sms, e0, e1);
  run_tma<32768, 4>(a, b, bytes, sms, e0, e1);
  run_tma<32768, 6>(a, b, bytes, sms, e0, e1);
  run_tma<65536, 3>(a, b, bytes, sms, e0, e1);
  return 0;
}
