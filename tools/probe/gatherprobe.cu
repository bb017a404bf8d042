// Scattered 32-byte gathers (the jagged dimuon kernel's muon reads): which load
// form lets DRAM move only the 32-B sectors that are read? Each thread reads one
// 64-B record pair (two consecutive 32-B rows, like a selected event's two f64
// muons) at a pseudo-random row of a large array. Variants: one 256-bit LDG per
// row (the product's load_muon), two 128-bit LDGs, .cg (L2 only) and .cs
// (streaming) 128-bit loads, and an L2::64B prefetch-size hint. Run under
// `ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum` to compare DRAM
// bytes per useful byte. Standalone, not product code.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

template <int MODE>
__global__ void gather(const double* __restrict__ rows, int64_t nrows, int64_t n, double* out) {
  double acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = (int64_t)(mix(i) % (uint64_t)(nrows - 1));
    const double* p = rows + 4 * r;
    double v[8];
    if constexpr (MODE == 0) {  // 256-bit non-coherent (the product's ld256)
      asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
      asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[4]), "=d"(v[5]), "=d"(v[6]), "=d"(v[7]) : "l"(p + 4));
    } else if constexpr (MODE == 1) {  // 128-bit
      for (int k = 0; k < 4; ++k)
        asm volatile("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(v[2 * k]), "=d"(v[2 * k + 1]) : "l"(p + 2 * k));
    } else if constexpr (MODE == 2) {  // 128-bit, cache at L2 only
      for (int k = 0; k < 4; ++k)
        asm volatile("ld.global.cg.v2.f64 {%0,%1}, [%2];" : "=d"(v[2 * k]), "=d"(v[2 * k + 1]) : "l"(p + 2 * k));
    } else if constexpr (MODE == 3) {  // 128-bit streaming
      for (int k = 0; k < 4; ++k)
        asm volatile("ld.global.cs.v2.f64 {%0,%1}, [%2];" : "=d"(v[2 * k]), "=d"(v[2 * k + 1]) : "l"(p + 2 * k));
    } else if constexpr (MODE == 4) {  // 256-bit with an explicit 64-B L2 prefetch-size hint
      asm volatile("ld.global.nc.L2::64B.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
      asm volatile("ld.global.nc.L2::64B.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[4]), "=d"(v[5]), "=d"(v[6]), "=d"(v[7]) : "l"(p + 4));
    } else {  // 256-bit, L1 no-allocate
      asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
      asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[4]), "=d"(v[5]), "=d"(v[6]), "=d"(v[7]) : "l"(p + 4));
    }
    for (int k = 0; k < 8; ++k) acc += v[k];
  }
  if (acc == 1234.5) out[0] = acc;
}

template <int MODE>
void run(const char* name, const double* rows, int64_t nrows, int64_t n, double* out, int sms) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  gather<MODE><<<sms * 8, 256>>>(rows, nrows, n, out);
  cudaEventRecord(a);
  gather<MODE><<<sms * 8, 256>>>(rows, nrows, n, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("%-28s %.3f ms  useful %.2f GB  %.0f GB/s useful (%s)\n", name, ms, 64.0 * n / 1e9, 64.0 * n / (ms * 1e6),
         cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
  const int64_t nrows = 140000000;  // 4.48 GB of 32-B rows (1.4e8 f64 muons)
  const int64_t n = argc > 1 ? atoll(argv[1]) : 15000000;  // selected pairs
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *rows, *out;
  cudaMalloc(&rows, nrows * 32);
  cudaMalloc(&out, 8);
  cudaMemset(rows, 0, nrows * 32);
  run<0>("ld.nc.v4.f64 (256-bit)", rows, nrows, n, out, sms);
  run<1>("ld.nc.v2.f64 (128-bit)", rows, nrows, n, out, sms);
  run<2>("ld.cg.v2.f64", rows, nrows, n, out, sms);
  run<3>("ld.cs.v2.f64", rows, nrows, n, out, sms);
  run<4>("ld.nc.L2::64B.v4.f64", rows, nrows, n, out, sms);
  run<5>("ld.nc.L1::no_allocate.v4", rows, nrows, n, out, sms);
  return 0;
}
