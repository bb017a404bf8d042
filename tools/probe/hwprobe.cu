// Hardware probe for the B200 pool: achievable HBM read/copy bandwidth with
// 128-bit and 256-bit loads, FP64/FP32 FMA rate, MUFU rate, shared-memory
// atomic throughput (the fused-histogram bottleneck candidate). Standalone;
// not part of the product library. Results feed DESIGN.md's roofline section.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__global__ void rd128(const int4* __restrict__ p, size_t n, int* out) {
  int acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    int4 v; asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x),"=r"(v.y),"=r"(v.z),"=r"(v.w) : "l"(p+i));
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x7fffffff) out[0] = acc;
}
__global__ void rd256(const double* __restrict__ p, size_t n4, int* out) {
  double acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    double a,b,c,d; asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a),"=d"(b),"=d"(c),"=d"(d) : "l"(p+4*i));
    acc += a + b + c + d;
  }
  if (acc == 1.2345) out[0] = 1;
}
__global__ void rd256u(const double* __restrict__ p, size_t n4, int* out) {
  // 2 loads in flight per iteration
  double acc = 0; size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + stride < n4; i += 2*stride) {
    double a,b,c,d,e,f,g,h;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a),"=d"(b),"=d"(c),"=d"(d) : "l"(p+4*i));
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(e),"=d"(f),"=d"(g),"=d"(h) : "l"(p+4*(i+stride)));
    acc += a + b + c + d + e + f + g + h;
  }
  for (; i < n4; i += stride) { acc += p[4*i]; }
  if (acc == 1.2345) out[0] = 1;
}
__global__ void cpy128(const int4* __restrict__ a, int4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void dfma_rate(double* out, int iters) {
  double a0=threadIdx.x, a1=a0+1, a2=a0+2, a3=a0+3, a4=a0+4, a5=a0+5, a6=a0+6, a7=a0+7;
  const double m = 0.999999, c = 1e-7;
  for (int k = 0; k < iters; ++k) {
    a0=fma(a0,m,c); a1=fma(a1,m,c); a2=fma(a2,m,c); a3=fma(a3,m,c);
    a4=fma(a4,m,c); a5=fma(a5,m,c); a6=fma(a6,m,c); a7=fma(a7,m,c);
  }
  double s = a0+a1+a2+a3+a4+a5+a6+a7; if (s == 1.2345) out[0] = s;
}
__global__ void ffma_rate(float* out, int iters) {
  float a0=threadIdx.x, a1=a0+1, a2=a0+2, a3=a0+3, a4=a0+4, a5=a0+5, a6=a0+6, a7=a0+7;
  const float m = 0.999999f, c = 1e-7f;
  for (int k = 0; k < iters; ++k) {
    a0=fmaf(a0,m,c); a1=fmaf(a1,m,c); a2=fmaf(a2,m,c); a3=fmaf(a3,m,c);
    a4=fmaf(a4,m,c); a5=fmaf(a5,m,c); a6=fmaf(a6,m,c); a7=fmaf(a7,m,c);
  }
  float s = a0+a1+a2+a3+a4+a5+a6+a7; if (s == 1.2345f) out[0] = s;
}
__global__ void mufu_rate(float* out, int iters) {
  float a0=threadIdx.x*1e-3f, a1=a0+.1f, a2=a0+.2f, a3=a0+.3f;
  for (int k = 0; k < iters; ++k) { a0=exp2f(-a0); a1=exp2f(-a1); a2=exp2f(-a2); a3=exp2f(-a3); }
  float s=a0+a1+a2+a3; if (s == 1.2345f) out[0] = s;
}
// shared-memory histogram atomics: mode 0 = spread pseudo-random bins, 1 = all lanes same bin,
// 2 = warp-aggregated (match_any) spread, 3 = per-warp private copy spread
__global__ void atoms_rate(unsigned* out, int iters, int mode) {
  __shared__ unsigned h[8 * 1024];
  for (int i = threadIdx.x; i < 8*1024; i += blockDim.x) h[i] = 0;
  __syncthreads();
  unsigned x = threadIdx.x * 2654435761u + blockIdx.x;
  unsigned base = (mode == 3) ? (threadIdx.x >> 5) % 8 * 1024 : 0;
  for (int k = 0; k < iters; ++k) {
    x = x * 1664525u + 1013904223u;
    unsigned b = (mode == 1) ? 7u : (x >> 22);   // 0..1023
    if (mode == 2) {
      unsigned peers = __match_any_sync(0xffffffffu, b);
      int leader = __ffs(peers) - 1;
      if ((threadIdx.x & 31) == leader) atomicAdd(&h[b], __popc(peers));
    } else {
      atomicAdd(&h[base + b], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) if (h[i] == 0xdeadbeef) out[0] = 1;
}

int main() {
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, 0));
  int clk=0, memclk=0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0); cudaDeviceGetAttribute(&memclk, cudaDevAttrMemoryClockRate, 0);
  printf("{\"name\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"smem_per_sm\":%zu,\"regs_per_sm\":%d,\"clock_khz\":%d,\"memclk_khz\":%d,\"bus_bits\":%d,\"total_mem\":%zu}\n",
         pr.name, pr.multiProcessorCount, pr.l2CacheSize, pr.sharedMemPerMultiprocessor, pr.regsPerMultiprocessor, clk, memclk, pr.memoryBusWidth, pr.totalGlobalMem);
  const size_t bytes = 8ull << 30;
  char *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes)); CK(cudaMemset(a, 1, bytes)); CK(cudaMemset(b, 0, bytes));
  int* o; CK(cudaMalloc(&o, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = pr.multiProcessorCount;
  auto tm = [&](auto f) { f(); cudaDeviceSynchronize(); float best = 1e30f; for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; } return best; };
  for (int bpsm : {2, 4, 8, 16}) for (int bs : {256, 512}) {
    if (bpsm * bs > 2048) continue;
    int grid = sms * bpsm;
    float t1 = tm([&]{ rd128<<<grid, bs>>>((const int4*)a, bytes/16, o); });
    float t2 = tm([&]{ rd256<<<grid, bs>>>((const double*)a, bytes/32, o); });
    float t3 = tm([&]{ rd256u<<<grid, bs>>>((const double*)a, bytes/32, o); });
    float t4 = tm([&]{ cpy128<<<grid, bs>>>((const int4*)a, (int4*)b, bytes/16/2); });
    printf("{\"probe\":\"hbm\",\"grid\":%d,\"block\":%d,\"read128_GBs\":%.1f,\"read256_GBs\":%.1f,\"read256x2_GBs\":%.1f,\"copy128_GBs\":%.1f}\n",
      grid, bs, bytes/t1/1e6, bytes/t2/1e6, bytes/t3/1e6, bytes/t4/1e6);
  }
  CK(cudaGetLastError());
  { int it = 1<<16; int grid = sms*8, bs=256; float t = tm([&]{ dfma_rate<<<grid,bs>>>((double*)o, it); });
    double fl = 2.0*8*it*(double)grid*bs; printf("{\"probe\":\"dfma\",\"TFLOPs\":%.2f,\"lanes_per_sm_clk_at_1965\":%.1f}\n", fl/t/1e9, fl/2/(t*1e-3)/sms/1.965e9); }
  { int it = 1<<16; int grid = sms*8, bs=256; float t = tm([&]{ ffma_rate<<<grid,bs>>>((float*)o, it); });
    double fl = 2.0*8*it*(double)grid*bs; printf("{\"probe\":\"ffma\",\"TFLOPs\":%.2f,\"lanes_per_sm_clk_at_1965\":%.1f}\n", fl/t/1e9, fl/2/(t*1e-3)/sms/1.965e9); }
  { int it = 1<<14; int grid = sms*8, bs=256; float t = tm([&]{ mufu_rate<<<grid,bs>>>((float*)o, it); });
    double ops = 4.0*it*(double)grid*bs; printf("{\"probe\":\"mufu_ex2\",\"Gops\":%.1f,\"lanes_per_sm_clk_at_1965\":%.1f}\n", ops/t/1e6, ops/(t*1e-3)/sms/1.965e9); }
  for (int mode = 0; mode < 4; ++mode) { int it = 1<<12; int grid = sms*4, bs=256; float t = tm([&]{ atoms_rate<<<grid,bs>>>((unsigned*)o, it, mode); });
    double ops = (double)it*grid*bs; printf("{\"probe\":\"atoms\",\"mode\":%d,\"Gupd_per_s\":%.1f,\"lanes_per_sm_clk_at_1965\":%.2f}\n", mode, ops/t/1e6, ops/(t*1e-3)/sms/1.965e9); }
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  return 0;
}
