// gvx_host.cu — transfer-inclusive runtime (include/gvx.h, "host pipeline"):
// the paper's host functions "handling the device memory allocation and
// transfers", done the B200 way. A pipeline owns three CUDA
// streams (copy-in, compute, copy-out), per-slot events and a ring of device
// staging slots. A call cuts the host batch into chunks that cycle through
// the slots: chunk c's H2D, chunk c-1's kernels and chunk c-2's D2H run
// concurrently (PCIe both directions + HBM), ordered only by events. The
// kernels are the device entry points of gvx_api.cu, called on the compute
// stream — this file adds no arithmetic.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <new>

#include "../../include/gvx.h"

namespace {

constexpr int kSlots = 3;

gvx_status cuda_status(cudaError_t e) { return e == cudaSuccess ? GVX_OK : GVX_ERR_CUDA; }

}  // namespace

struct gvx_host_pipeline {
  int device = 0;
  gvx_dtype dtype = GVX_F64;
  int64_t chunk = 0;
  size_t es = 8;
  cudaStream_t s_in = nullptr, s_cmp = nullptr, s_out = nullptr;
  cudaEvent_t ev_in[kSlots] = {}, ev_cmp[kSlots] = {}, ev_free[kSlots] = {};
  cudaEvent_t ev_start = nullptr, ev_done = nullptr, ev_aux = nullptr;
  // slot j: 4 buffers of chunk x 4 scalars (pairs: v1, v2, m; boost: v, beta, out)
  void* slot[kSlots][3] = {};
  unsigned long long* d_bins = nullptr;  // 2 x (bins_cap) counters
  int64_t bins_cap = 0;
};

namespace {

void destroy(gvx_host_pipeline* p) {
  if (!p) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  for (int j = 0; j < kSlots; ++j) {
    for (int b = 0; b < 3; ++b)
      if (p->slot[j][b]) cudaFree(p->slot[j][b]);
    if (p->ev_in[j]) cudaEventDestroy(p->ev_in[j]);
    if (p->ev_cmp[j]) cudaEventDestroy(p->ev_cmp[j]);
    if (p->ev_free[j]) cudaEventDestroy(p->ev_free[j]);
  }
  if (p->d_bins) cudaFree(p->d_bins);
  for (cudaEvent_t e : {p->ev_start, p->ev_done, p->ev_aux})
    if (e) cudaEventDestroy(e);
  for (cudaStream_t s : {p->s_in, p->s_cmp, p->s_out})
    if (s) cudaStreamDestroy(s);
  cudaSetDevice(prev);
  delete p;
}

gvx_status ensure_bins(gvx_host_pipeline* p, int64_t nb2) {
  if (nb2 <= p->bins_cap) return GVX_OK;
  if (p->d_bins) cudaFree(p->d_bins);
  p->d_bins = nullptr;
  p->bins_cap = 0;
  if (cudaMalloc(&p->d_bins, 2 * nb2 * sizeof(unsigned long long)) != cudaSuccess) return GVX_ERR_CUDA;
  p->bins_cap = nb2;
  return GVX_OK;
}

gvx_vec4_cview aos_view(const void* base, size_t es) {
  gvx_vec4_cview v;
  for (int k = 0; k < 4; ++k) v.c[k] = (const char*)base + k * es;
  v.stride = 4;
  return v;
}
gvx_vec4_view aos_oview(void* base, size_t es) {
  gvx_vec4_view v;
  for (int k = 0; k < 4; ++k) v.c[k] = (char*)base + k * es;
  v.stride = 4;
  return v;
}

// Fork the pipeline's streams off the caller's stream, and after the whole
// previous call on this pipeline (whatever stream that used): the staging slots
// and d_bins are reused, so none of the three streams may start before that
// call's last D2H (ev_done, recorded on s_out by join) has completed.
void fork(gvx_host_pipeline* p, cudaStream_t caller) {
  cudaStreamWaitEvent(p->s_in, p->ev_done, 0);
  cudaStreamWaitEvent(p->s_cmp, p->ev_done, 0);
  cudaStreamWaitEvent(p->s_out, p->ev_done, 0);
  cudaEventRecord(p->ev_start, caller);
  cudaStreamWaitEvent(p->s_in, p->ev_start, 0);
  cudaStreamWaitEvent(p->s_cmp, p->ev_start, 0);
  cudaStreamWaitEvent(p->s_out, p->ev_start, 0);
}
// Join: the caller's stream waits for all three.
void join(gvx_host_pipeline* p, cudaStream_t caller) {
  cudaEventRecord(p->ev_aux, p->s_in);
  cudaStreamWaitEvent(p->s_out, p->ev_aux, 0);
  cudaEventRecord(p->ev_done, p->s_cmp);
  cudaStreamWaitEvent(p->s_out, p->ev_done, 0);
  cudaEventRecord(p->ev_done, p->s_out);
  cudaStreamWaitEvent(caller, p->ev_done, 0);
}

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

}  // namespace

extern "C" {

gvx_status gvx_host_pipeline_create(gvx_dtype dtype, int64_t chunk_events, gvx_host_pipeline** out) {
  if (!out || (dtype != GVX_F32 && dtype != GVX_F64) || chunk_events < 1 || chunk_events > (int64_t(1) << 31))
    return GVX_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  gvx_host_pipeline* p = new (std::nothrow) gvx_host_pipeline();
  if (!p) return GVX_ERR_CUDA;
  cudaGetDevice(&p->device);
  p->dtype = dtype;
  p->chunk = chunk_events;
  p->es = dtype == GVX_F64 ? 8 : 4;
  bool ok = true;
  ok = ok && cudaStreamCreateWithFlags(&p->s_in, cudaStreamNonBlocking) == cudaSuccess;
  ok = ok && cudaStreamCreateWithFlags(&p->s_cmp, cudaStreamNonBlocking) == cudaSuccess;
  ok = ok && cudaStreamCreateWithFlags(&p->s_out, cudaStreamNonBlocking) == cudaSuccess;
  for (cudaEvent_t* e : {&p->ev_start, &p->ev_done, &p->ev_aux})
    ok = ok && cudaEventCreateWithFlags(e, cudaEventDisableTiming) == cudaSuccess;
  const size_t vec_bytes = (size_t)chunk_events * 4 * p->es;
  for (int j = 0; j < kSlots && ok; ++j) {
    ok = ok && cudaEventCreateWithFlags(&p->ev_in[j], cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&p->ev_cmp[j], cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&p->ev_free[j], cudaEventDisableTiming) == cudaSuccess;
    for (int b = 0; b < 3 && ok; ++b) ok = cudaMalloc(&p->slot[j][b], vec_bytes) == cudaSuccess;
  }
  if (!ok) {
    destroy(p);
    return GVX_ERR_CUDA;
  }
  *out = p;
  return GVX_OK;
}

gvx_status gvx_host_pipeline_destroy(gvx_host_pipeline* p) {
  if (!p) return GVX_ERR_INVALID_ARGUMENT;
  cudaStreamSynchronize(p->s_out);
  destroy(p);
  return GVX_OK;
}

gvx_status gvx_host_pairs(gvx_host_pipeline* p, gvx_coords coords, const void* h_v1, const void* h_v2, int64_t n,
                          double lo, double hi, int32_t nbins, void* h_m_out, unsigned long long* h_bins,
                          unsigned long long* h_bins_cm, gvx_stream_t stream) {
  // validated synchronously, before anything is enqueued (the device entries' rules)
  if (!p || n < 0 || (n > 0 && (!h_v1 || !h_v2))) return GVX_ERR_INVALID_ARGUMENT;
  if (coords != GVX_PTETAPHIM && coords != GVX_PXPYPZE && coords != GVX_PXPYPZM && coords != GVX_PTETAPHIE)
    return GVX_ERR_INVALID_ARGUMENT;
  const bool hist = h_bins || h_bins_cm;
  if (hist && (nbins < 1 || nbins > (1 << 28) || !isfinite(lo) || !isfinite(hi) || !(lo < hi)))
    return GVX_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(p->device);
  cudaStream_t caller = (cudaStream_t)stream;
  const size_t es = p->es, vb = 4 * es;
  const int64_t nb2 = hist ? (int64_t)nbins + 2 : 0;
  gvx_status st = GVX_OK;
  if (hist && (st = ensure_bins(p, nb2)) != GVX_OK) return st;
  fork(p, caller);
  if (hist) cudaMemsetAsync(p->d_bins, 0, 2 * nb2 * sizeof(unsigned long long), p->s_cmp);
  int c = 0;
  for (int64_t a = 0; a < n; a += p->chunk, ++c) {
    const int64_t k = n - a < p->chunk ? n - a : p->chunk;
    const int j = c % kSlots;
    void* d1 = p->slot[j][0];
    void* d2 = p->slot[j][1];
    void* dm = p->slot[j][2];
    if (c >= kSlots) cudaStreamWaitEvent(p->s_in, p->ev_free[j], 0);
    cudaMemcpyAsync(d1, (const char*)h_v1 + a * vb, k * vb, cudaMemcpyHostToDevice, p->s_in);
    cudaMemcpyAsync(d2, (const char*)h_v2 + a * vb, k * vb, cudaMemcpyHostToDevice, p->s_in);
    cudaEventRecord(p->ev_in[j], p->s_in);
    cudaStreamWaitEvent(p->s_cmp, p->ev_in[j], 0);
    gvx_vec4_cview v1 = aos_view(d1, es), v2 = aos_view(d2, es);
    gvx_stream_t sc = (gvx_stream_t)p->s_cmp;
    if (h_bins && h_bins_cm) {  // everything requested: the fused one-pass kernel (same bits)
      if (st == GVX_OK)
        st = gvx_pair_histograms(p->dtype, coords, &v1, &v2, k, lo, hi, nbins, p->d_bins, p->d_bins + nb2,
                                 h_m_out ? dm : nullptr, nullptr, sc);
    } else {
      if (h_m_out && st == GVX_OK) st = gvx_invariant_mass(p->dtype, coords, &v1, &v2, dm, k, sc);
      if (h_bins && st == GVX_OK)
        st = gvx_mass_histogram(p->dtype, coords, &v1, &v2, k, lo, hi, nbins, p->d_bins, 0u, nullptr, nullptr, sc);
      if (h_bins_cm && st == GVX_OK)
        st = gvx_mass_histogram(p->dtype, coords, &v1, &v2, k, lo, hi, nbins, p->d_bins + nb2, GVX_HIST_BOOST_TO_CM,
                                nullptr, nullptr, sc);
    }
    cudaEventRecord(p->ev_cmp[j], p->s_cmp);
    cudaStreamWaitEvent(p->s_out, p->ev_cmp[j], 0);
    if (h_m_out) cudaMemcpyAsync((char*)h_m_out + a * es, dm, k * es, cudaMemcpyDeviceToHost, p->s_out);
    cudaEventRecord(p->ev_free[j], p->s_out);
  }
  if (hist) {
    cudaEventRecord(p->ev_aux, p->s_cmp);
    cudaStreamWaitEvent(p->s_out, p->ev_aux, 0);
    if (h_bins) cudaMemcpyAsync(h_bins, p->d_bins, nb2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, p->s_out);
    if (h_bins_cm)
      cudaMemcpyAsync(h_bins_cm, p->d_bins + nb2, nb2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, p->s_out);
  }
  join(p, caller);
  if (st != GVX_OK) return st;
  return cuda_status(cudaGetLastError());
}

gvx_status gvx_host_boost(gvx_host_pipeline* p, const void* h_v, const void* h_beta, int64_t n, void* h_out,
                          gvx_stream_t stream) {
  if (!p || n < 0 || (n > 0 && (!h_v || !h_beta || !h_out))) return GVX_ERR_INVALID_ARGUMENT;
  DeviceGuard guard(p->device);
  cudaStream_t caller = (cudaStream_t)stream;
  const size_t es = p->es, vb = 4 * es, bb = 3 * es;
  gvx_status st = GVX_OK;
  fork(p, caller);
  int c = 0;
  for (int64_t a = 0; a < n; a += p->chunk, ++c) {
    const int64_t k = n - a < p->chunk ? n - a : p->chunk;
    const int j = c % kSlots;
    void* dv = p->slot[j][0];
    void* db = p->slot[j][1];
    void* dout = p->slot[j][2];
    if (c >= kSlots) cudaStreamWaitEvent(p->s_in, p->ev_free[j], 0);
    cudaMemcpyAsync(dv, (const char*)h_v + a * vb, k * vb, cudaMemcpyHostToDevice, p->s_in);
    cudaMemcpyAsync(db, (const char*)h_beta + a * bb, k * bb, cudaMemcpyHostToDevice, p->s_in);
    cudaEventRecord(p->ev_in[j], p->s_in);
    cudaStreamWaitEvent(p->s_cmp, p->ev_in[j], 0);
    gvx_vec4_cview v = aos_view(dv, es);
    gvx_vec3_cview b;
    for (int q = 0; q < 3; ++q) b.c[q] = (const char*)db + q * es;
    b.stride = 3;
    gvx_vec4_view o = aos_oview(dout, es);
    if (st == GVX_OK) st = gvx_boost(p->dtype, &v, &b, &o, k, (gvx_stream_t)p->s_cmp);
    cudaEventRecord(p->ev_cmp[j], p->s_cmp);
    cudaStreamWaitEvent(p->s_out, p->ev_cmp[j], 0);
    cudaMemcpyAsync((char*)h_out + a * vb, dout, k * vb, cudaMemcpyDeviceToHost, p->s_out);
    cudaEventRecord(p->ev_free[j], p->s_out);
  }
  join(p, caller);
  if (st != GVX_OK) return st;
  return cuda_status(cudaGetLastError());
}

}  // extern "C"
