// Probe: cm_mass_f32_lanes<float> vs <float2> on the same events, with the
// boosted vectors, to localise a scalar/packed bit difference. Not product code.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include "../../paper_2312_02756_b200/csrc/gvx_math.cuh"
using namespace gvx;
__global__ void k(const float* v1, const float* v2, int n, float* out_s, float* out_p) {
  int i = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (i + 1 >= n) return;
  const float* a0 = v1 + 4 * i; const float* b0 = v2 + 4 * i;
  const float* a1 = v1 + 4 * i + 4; const float* b1 = v2 + 4 * i + 4;
  float c0, c1, vs0[8], vs1[8];
  float M0 = cm_mass_f32_lanes<float, true, true>(a0[0], a0[1], a0[2], a0[3], b0[0], b0[1], b0[2], b0[3], &c0, vs0);
  float M1 = cm_mass_f32_lanes<float, true, true>(a1[0], a1[1], a1[2], a1[3], b1[0], b1[1], b1[2], b1[3], &c1, vs1);
  // the library's scalar route (no boosted output, no cos)
  vs0[0] = cm_mass_ptetaphim_fast<float, false>(a0[0], a0[1], a0[2], a0[3], b0[0], b0[1], b0[2], b0[3], nullptr, nullptr, nullptr);
  vs1[0] = cm_mass_ptetaphim_fast<float, false>(a1[0], a1[1], a1[2], a1[3], b1[0], b1[1], b1[2], b1[3], nullptr, nullptr, nullptr);
  float2 c, vp[8];
  float2 M = cm_mass_f32_lanes<float2, true, true>(make_float2(a0[0], a1[0]), make_float2(a0[1], a1[1]),
      make_float2(a0[2], a1[2]), make_float2(a0[3], a1[3]), make_float2(b0[0], b1[0]), make_float2(b0[1], b1[1]),
      make_float2(b0[2], b1[2]), make_float2(b0[3], b1[3]), &c, vp);
  float* s = out_s + 10 * i; float* p = out_p + 10 * i;
  s[0] = M0; s[1] = c0; for (int j = 0; j < 8; ++j) s[2 + j] = vs0[j];
  s[10] = M1; s[11] = c1; for (int j = 0; j < 8; ++j) s[12 + j] = vs1[j];
  p[0] = M.x; p[1] = c.x; for (int j = 0; j < 8; ++j) p[2 + j] = vp[j].x;
  p[10] = M.y; p[11] = c.y; for (int j = 0; j < 8; ++j) p[12 + j] = vp[j].y;
  p[2] = M.x; p[12] = M.y;  // slot "a2x" now compares the library scalar route's M with the packed M
}
int main() {
  const int n = 4096;
  float *v1, *v2, *os, *op;
  cudaMallocManaged(&v1, 16 * n); cudaMallocManaged(&v2, 16 * n);
  cudaMallocManaged(&os, 40 * n); cudaMallocManaged(&op, 40 * n);
  srand(1);
  for (int i = 0; i < n; ++i) {
    float* a = v1 + 4 * i; float* b = v2 + 4 * i;
    a[0] = 10 + 80.f * rand() / RAND_MAX; a[1] = -2.5f + 5.f * rand() / RAND_MAX; a[2] = -3.1f + 6.2f * rand() / RAND_MAX; a[3] = 0.10565837f;
    b[0] = 10 + 80.f * rand() / RAND_MAX; b[1] = -2.5f + 5.f * rand() / RAND_MAX; b[2] = -3.1f + 6.2f * rand() / RAND_MAX; b[3] = 0.10565837f;
  }
  const float e19a[4] = {90.62908935546875f, -1.4739705324172974f, 0.7309443950653076f, 0.10565837472677231f};
  const float e19b[4] = {11.965287208557129f, 1.6131176948547363f, 0.6068066954612732f, 0.10565837472677231f};
  memcpy(v1, e19a, 16); memcpy(v2, e19b, 16);
  memcpy(v1 + 4 * 3, e19a, 16); memcpy(v2 + 4 * 3, e19b, 16);
  k<<<n / 256, 128>>>(v1, v2, n, os, op);
  cudaDeviceSynchronize();
  const char* nm[10] = {"M", "cos", "a2x", "a2y", "a2z", "a2t", "b2x", "b2y", "b2z", "b2t"};
  int cnt[10] = {0};
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < 10; ++j) if (memcmp(&os[10 * i + j], &op[10 * i + j], 4)) cnt[j]++;
  for (int j = 0; j < 10; ++j) printf("%s: %d differ\n", nm[j], cnt[j]);
  printf("event19 scalar M %.9g route %.9g packed %.9g | lane1 copy scalar %.9g packed %.9g\n", os[0], os[2], op[0], os[30], op[30]);
  return 0;
}
