// Racecheck control experiment: the textbook single-producer /
// multi-consumer shared-memory ring synchronised by mbarriers, in three
// variants, each run under `compute-sanitizer --tool racecheck`:
//   mode 0  TMA refill (cp.async.bulk, async proxy), consumers fence.proxy.async
//           before releasing a stage          — the protocol of k_pair_tma / k_step
//   mode 1  TMA refill, no consumer-side fence — the protocol with the fence removed
//   mode 2  generic-proxy refill (the producer warp writes the stage with st.shared,
//           then arrives on `full` with release semantics) — no async proxy at all
// Every variant checks its result (sum of all words read = sum of the source),
// so a real race that corrupts data shows up as a wrong checksum.
// Standalone, not product code.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../paper_2312_02756_b200/csrc/gvx_tma.cuh"
using namespace gvx;

constexpr int STAGE = 4096;  // bytes per stage
constexpr int STAGES = 2;
constexpr int NCW = 4;       // consumer warps

__global__ void __launch_bounds__(32 * (NCW + 1)) ring(const uint32_t* __restrict__ src, int64_t ntiles, int mode,
                                                       unsigned long long* out) {
  __shared__ __align__(128) uint32_t buf[STAGES][STAGE / 4];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tma::mbar_init(&full[s], mode == 2 ? 32 : 1);
      tma::mbar_init(&empty[s], NCW);
    }
    tma::fence_barrier_init();
  }
  __syncthreads();
  unsigned long long acc = 0;
  if (warp == 0) {
    const uint64_t pol = tma::policy_evict_first();
    for (int64_t t = blockIdx.x, it = 0; t < ntiles; t += gridDim.x, ++it) {
      const int s = (int)(it % STAGES);
      const uint32_t k = (uint32_t)(it / STAGES);
      if (k > 0) tma::mbar_wait(&empty[s], (k - 1) & 1);
      if (mode == 2) {  // generic-proxy refill by the whole producer warp
        for (int i = lane; i < STAGE / 4; i += 32) buf[s][i] = src[t * (STAGE / 4) + i];
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(tma::smem_u32(&full[s])) : "memory");
      } else if (lane == 0) {
        if (k > 0) tma::fence_proxy_async_smem();
        tma::mbar_arrive_expect_tx(&full[s], STAGE);
        tma::bulk_g2s(buf[s], src + t * (STAGE / 4), STAGE, &full[s], pol);
      }
    }
  } else {
    const int ct = threadIdx.x - 32;
    for (int64_t t = blockIdx.x, it = 0; t < ntiles; t += gridDim.x, ++it) {
      const int s = (int)(it % STAGES);
      const uint32_t k = (uint32_t)(it / STAGES);
      tma::mbar_wait(&full[s], k & 1);
      for (int i = ct; i < STAGE / 4; i += NCW * 32) acc += buf[s][i];
      if (mode == 0) tma::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(&empty[s]);
    }
  }
  atomicAdd(out, acc);
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  const int64_t ntiles = argc > 2 ? atoll(argv[2]) : 64;
  const size_t words = (size_t)ntiles * STAGE / 4;
  uint32_t* h = (uint32_t*)malloc(words * 4);
  unsigned long long want = 0;
  for (size_t i = 0; i < words; ++i) { h[i] = (uint32_t)(i * 2654435761u) >> 8; want += h[i]; }
  uint32_t* d;
  unsigned long long* out;
  cudaMalloc(&d, words * 4);
  cudaMalloc(&out, 8);
  cudaMemcpy(d, h, words * 4, cudaMemcpyHostToDevice);
  cudaMemset(out, 0, 8);
  ring<<<2, 32 * (NCW + 1)>>>(d, ntiles, mode, out);
  unsigned long long got = 0;
  cudaError_t e = cudaMemcpy(&got, out, 8, cudaMemcpyDeviceToHost);
  printf("mode %d ntiles %lld: %s checksum %s\n", mode, (long long)ntiles, cudaGetErrorString(e),
         got == want ? "ok" : "WRONG");
  return got == want ? 0 : 1;
}
