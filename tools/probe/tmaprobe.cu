// TMA (cp.async.bulk) streaming-read probe: achievable HBM read bandwidth of
// a producer-lane + consumer-warps smem ring, as a function of stage size,
// ring depth and CTAs per SM. Consumers touch every 16 B of each stage
// (LDS.128 + xor) so the data path is real. Standalone, not product code.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2312_02756_b200/csrc/gvx_tma.cuh"
using namespace gvx;

template <int STAGE, int STAGES, int NCW, bool EVF>
__global__ void __launch_bounds__(32 * (NCW + 1)) ring(const char* __restrict__ src, int64_t ntiles, int* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE);
  uint64_t* empty = full + STAGES;
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { tma::mbar_init(&full[s], 1); tma::mbar_init(&empty[s], NCW); }
    tma::fence_barrier_init();
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      uint64_t pol = EVF ? tma::policy_evict_first() : 0;
      int it = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        int s = it % STAGES, k = it / STAGES;
        if (k > 0) tma::mbar_wait(&empty[s], (k - 1) & 1);
        tma::mbar_arrive_expect_tx(&full[s], STAGE);
        if (EVF) tma::bulk_g2s(smem + s * STAGE, src + t * STAGE, STAGE, &full[s], pol);
        else asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                          :: "r"(tma::smem_u32(smem + s * STAGE)), "l"(src + t * STAGE), "r"(STAGE), "r"(tma::smem_u32(&full[s])) : "memory");
      }
    }
  } else {
    int acc = 0, ct = threadIdx.x - 32;
    int it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      int s = it % STAGES, k = it / STAGES;
      tma::mbar_wait(&full[s], k & 1);
      const int4* p = reinterpret_cast<const int4*>(smem + s * STAGE);
      for (int i = ct; i < STAGE / 16; i += NCW * 32) { int4 v = p[i]; acc ^= v.x ^ v.y ^ v.z ^ v.w; }
      tma::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(&empty[s]);
    }
    if (acc == 0x12345) out[0] = acc;
  }
}

template <int STAGE, int STAGES, int NCW, bool EVF>
void run(const char* src, size_t bytes, int* out, int sms) {
  auto k = ring<STAGE, STAGES, NCW, EVF>;
  size_t sm = STAGES * STAGE + 2 * STAGES * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 32 * (NCW + 1), sm);
  for (int cps = 1; cps <= per; ++cps) {
    int grid = sms * cps;
    int64_t ntiles = bytes / STAGE;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    k<<<grid, 32 * (NCW + 1), sm>>>(src, ntiles, out);
    cudaDeviceSynchronize();
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a); k<<<grid, 32 * (NCW + 1), sm>>>(src, ntiles, out); cudaEventRecord(b);
      cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("{\"probe\":\"tma_ring\",\"stage_kb\":%d,\"stages\":%d,\"ncw\":%d,\"evict_first\":%d,\"ctas_per_sm\":%d,\"inflight_kb_per_sm\":%d,\"GBs\":%.1f,\"err\":\"%s\"}\n",
           STAGE / 1024, STAGES, NCW, (int)EVF, cps, cps * STAGES * STAGE / 1024, (ntiles * (double)STAGE) / best / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  size_t bytes = 8ull << 30;
  char* src; cudaMalloc(&src, bytes); cudaMemset(src, 1, bytes);
  int* out; cudaMalloc(&out, 64);
  run<8192, 4, 4, true>(src, bytes, out, sms);
  run<16384, 4, 8, true>(src, bytes, out, sms);
  run<16384, 4, 8, false>(src, bytes, out, sms);
  run<16384, 6, 8, true>(src, bytes, out, sms);
  run<16384, 8, 8, true>(src, bytes, out, sms);
  run<32768, 4, 8, true>(src, bytes, out, sms);
  run<32768, 6, 8, true>(src, bytes, out, sms);
  run<65536, 3, 8, true>(src, bytes, out, sms);
  run<8192, 16, 4, true>(src, bytes, out, sms);
  run<4096, 32, 4, true>(src, bytes, out, sms);
  return 0;
}
