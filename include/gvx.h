/*
 * gvx.h — C ABI of the B200-native GenVectorX hot path (arXiv 2312.02756).
 *
 * Library: paper_2312_02756_b200/libgvx.so (hand-written sm_100a CUDA).
 * No torch or CUDA types appear here: pointers are plain, sizes are int64,
 * a stream is the opaque CUDA stream handle (cudaStream_t / CUstream are the
 * same pointer; NULL = the legacy default stream).
 *
 * ---------------------------------------------------------------------------
 * Common conventions (apply to every entry point below)
 * ---------------------------------------------------------------------------
 * Ownership. Every data pointer is caller-owned. Device entry points take
 *   DEVICE pointers valid on the calling thread's current CUDA device; the
 *   library allocates no device memory. Its only state is a per-(kernel,
 *   device) launch-configuration cache (SM count, occupancy, shared-memory
 *   opt-in), filled on first use under a mutex — so every entry point may be
 *   called from several host threads and captured into a CUDA graph after one
 *   warm-up call. Environment (read once per process): GVX_DISABLE_TMA=1 /
 *   GVX_FORCE_TMA=1 pick the register (LDG) or shared-memory-ring (TMA)
 *   kernels, GVX_NO_STEP_KERNEL=1 runs gvx_pair_histograms_boost as its two
 *   calls, GVX_DIMUON_IMPL=tma|ldg picks the streaming dimuon kernels — all for
 *   A/B runs; results are identical either way. Outputs are
 *   caller-allocated, as in the paper's kernel signature
 *   `(LVector *v1, LVector *v2, Scalar *m, size_t N)`.
 * Asynchrony. Device entry points enqueue on `stream` and return without a
 *   host synchronisation. Kernel faults surface at the caller's next sync.
 * Errors. Arguments are validated synchronously and nothing is enqueued on
 *   error: n < 0, a NULL component pointer with n > 0, stride < 1, a pointer
 *   not aligned to sizeof(T), nbins < 1, non-finite lo/hi or lo >= hi
 *   -> GVX_ERR_INVALID_ARGUMENT. n == 0 -> GVX_OK with nothing launched
 *   (SPEC.md:280). A launch failure -> GVX_ERR_CUDA (details from
 *   gvx_last_cuda_error_string()).
 * Per-event domain problems never error (the paper drops exception
 *   handling): NaN/Inf inputs propagate, a per-event |beta| >= 1
 *   yields NaN x 4, NaN masses land in the overflow bin.
 * Aliasing. A boost's output may be exactly its input (in place). Any other
 *   overlap between an output and an input is undefined.
 * Views. A 4-vector array is described by gvx_vec4_cview / gvx_vec4_view:
 *   component k (0..3) of vector i is ((T*)c[k])[i * stride].
 *     AoS [N][4]:        c[k] = base + k,     stride = 4
 *     SoA 4 x [N]:       c[k] = array_k,      stride = 1
 *     pairs [N][2][4]:   v1.c[k] = base + k, v2.c[k] = base + 4 + k, stride = 8
 *   Component order is (pt, eta, phi, m) for GVX_PTETAPHIM, (px, py, pz, E) for
 *   GVX_PXPYPZE (E last), (px, py, pz, m) for GVX_PXPYPZM and
 *   (pt, eta, phi, E) for GVX_PTETAPHIE. Any view is accepted; AoS with
 *   4*sizeof(T) alignment and SoA with 16-byte-aligned arrays take the
 *   vectorised fast paths. Results are bitwise identical across layouts.
 */
#ifndef GVX_H
#define GVX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GVX_ABI_VERSION 8

typedef struct CUstream_st *gvx_stream_t; /* == cudaStream_t */

typedef enum {
    GVX_OK = 0,
    GVX_ERR_INVALID_ARGUMENT = 1,
    GVX_ERR_DOMAIN = 2,
    GVX_ERR_UNSUPPORTED = 3,
    GVX_ERR_CUDA = 4
} gvx_status;

typedef enum { GVX_F32 = 0, GVX_F64 = 1 } gvx_dtype;

/* 4D coordinate systems ("any 4-dimensional
 * coordinate system"). Mass and histogram accept all four (conversions to
 * PxPyPzE: SPEC.md:81 for pt/eta/phi, E = sqrt(|p|^2 + m|m|) clamped at 0 for
 * a mass coordinate, R2); boost takes PXPYPZE. */
typedef enum { GVX_PTETAPHIM = 0, GVX_PXPYPZE = 1, GVX_PXPYPZM = 2, GVX_PTETAPHIE = 3 } gvx_coords;

typedef struct { const void *c[4]; int64_t stride; } gvx_vec4_cview;
typedef struct { void *c[4]; int64_t stride; } gvx_vec4_view;
typedef struct { const void *c[3]; int64_t stride; } gvx_vec3_cview;

/* Flags of gvx_mass_histogram. */
#define GVX_HIST_BOOST_TO_CM 0x1u

/*
 * gvx_invariant_mass — InvariantMasses (Fig. 1):
 *   m_out[i] = (v1[i] + v2[i]).mass()
 * The sum is component-wise in PxPyPzE; PtEtaPhiM input
 * is converted with px = pt cos(phi), py = pt sin(phi), pz = pt sinh(eta),
 * E = sqrt(max(0, m|m| + pt^2 + pz^2)) (clamp = DESIGN.md R2).
 * mass() = sqrt(M^2) if M^2 >= 0 else -sqrt(-M^2), M^2 = E^2 - |p|^2
 * (SPEC.md:101-103, :138).
 *   dtype   GVX_F32 / GVX_F64: element type of v1, v2 and m_out (arithmetic
 *           is closed over it).
 *   v1, v2  n input vectors each (device).
 *   m_out   n masses, contiguous (device), must not overlap the inputs.
 * Accuracy: |M_gpu|M_gpu| - M_exact^2| <= tau * E_lab^2 with tau = 1e-12
 * (f64) / 1e-5 (f32), E_lab = E1 + E2 (north_star; R5).
 */
gvx_status gvx_invariant_mass(gvx_dtype dtype, gvx_coords coords, const gvx_vec4_cview *v1,
                              const gvx_vec4_cview *v2, void *m_out, int64_t n,
                              gvx_stream_t stream);

/*
 * gvx_boost — ApplyBoost with a per-event velocity ("a
 * 4-dimensional Lorentz transformation represented internally by a 4x4
 * orthosymplectic matrix"; matrix SPEC.md:188):
 *   gamma = 1/sqrt(1 - b^2), L_ij = d_ij + gamma^2/(1+gamma) b_i b_j,
 *   L_i4 = L_4i = gamma b_i, L_44 = gamma;  out[i] = L(beta[i]) * v[i]
 * (active boost, metric diag(-1,-1,-1,+1); R6, R7).
 *   v     n PxPyPzE vectors (device);  beta  n velocities (bx, by, bz) (device)
 *   out   n PxPyPzE vectors (device); may equal v exactly (in place).
 * |beta[i]| >= 1 or NaN -> out[i] = NaN x 4. Accuracy: component-wise
 * |delta| <= tau * S, S = gamma (E + |beta||p|) (R5).
 */
gvx_status gvx_boost(gvx_dtype dtype, const gvx_vec4_cview *v, const gvx_vec3_cview *beta,
                     const gvx_vec4_view *out, int64_t n, gvx_stream_t stream);

/*
 * gvx_boost_uniform — the paper's single-matrix ApplyBoost:
 * one beta = (bx, by, bz) for all n vectors (rounded to dtype first).
 * |beta| >= 1 or non-finite -> GVX_ERR_DOMAIN, nothing enqueued.
 */
gvx_status gvx_boost_uniform(gvx_dtype dtype, const gvx_vec4_cview *v, double bx, double by,
                             double bz, const gvx_vec4_view *out, int64_t n,
                             gvx_stream_t stream);

/*
 * gvx_lorentz_transform — ApplyBoost with a general Lorentz transformation
 * "represented internally by a 4x4 orthosymplectic matrix" (
 * SURVEY §8(f) f2): out[i] = L * v[i], PxPyPzE in and out.
 *   L     16 doubles, row-major, HOST pointer (copied at the call; rounded to
 *         dtype). Must satisfy L^T g L = g, g = diag(-1,-1,-1,+1), to 1e-9
 *         relative, and be finite, else GVX_ERR_DOMAIN (nothing enqueued).
 *   v, out  n vectors (device); out may equal v exactly (in place).
 */
gvx_status gvx_lorentz_transform(gvx_dtype dtype, const gvx_vec4_cview *v, const double *L,
                                 const gvx_vec4_view *out, int64_t n, gvx_stream_t stream);

/*
 * gvx_mass_histogram — fused InvariantMass + histogram (north_star;
 * BASELINE.json configs[3], configs[4]). For each pair the signed mass M (as
 * gvx_invariant_mass; with flags & GVX_HIST_BOOST_TO_CM, the mass after
 * boosting both vectors by beta_cm = -(p1+p2)/(E1+E2), R11; E <= 0
 * or beta_cm^2 >= 1 -> NaN) is promoted to double and binned ROOT-style
 * (R12):  x < lo -> 0;  !(x < hi) (NaN included) -> nbins+1;
 *                   else 1 + (int)((nbins * (x - lo)) / (hi - lo)).
 *   bins         nbins+2 uint64 counters (device), ACCUMULATED (caller zeroes);
 *                this is the per-shard stage of the multi-GPU reduction.
 *   m_out        NULL or n masses of dtype (device).
 *   boosted_out  NULL or, with GVX_HIST_BOOST_TO_CM, 2n boosted PxPyPzE
 *                vectors: pair i -> vectors 2i and 2i+1 of the view.
 */
gvx_status gvx_mass_histogram(gvx_dtype dtype, gvx_coords coords, const gvx_vec4_cview *v1,
                              const gvx_vec4_cview *v2, int64_t n, double lo, double hi,
                              int32_t nbins, unsigned long long *bins, uint32_t flags,
                              void *m_out, const gvx_vec4_view *boosted_out,
                              gvx_stream_t stream);

/*
 * gvx_pair_histograms — the pair kernels of one batch fused into ONE pass over
 * the inputs: for each pair the lab mass (exactly gvx_invariant_mass's value),
 * its histogram, the CM mass (exactly gvx_mass_histogram's with
 * GVX_HIST_BOOST_TO_CM) and its histogram, both on the same axis (lo, hi,
 * nbins; binning as gvx_mass_histogram). The inputs are read once instead of
 * three times (mass, lab histogram, CM histogram).
 *   lab_bins, cm_bins  nbins+2 uint64 each (device), ACCUMULATED.
 *   m_out, cm_m_out    NULL or n masses of dtype (device): lab / CM.
 * Results are bit-identical to the three separate calls. Errors as
 * gvx_mass_histogram.
 */
gvx_status gvx_pair_histograms(gvx_dtype dtype, gvx_coords coords, const gvx_vec4_cview *v1,
                               const gvx_vec4_cview *v2, int64_t n, double lo, double hi,
                               int32_t nbins, unsigned long long *lab_bins,
                               unsigned long long *cm_bins, void *m_out, void *cm_m_out,
                               gvx_stream_t stream);

/*
 * gvx_pair_histograms_boost — the whole hot-path step of two batches in ONE
 * persistent launch (ABI v6): gvx_pair_histograms of the n pairs (v1, v2) and
 * gvx_boost of the nb vectors bv by their velocities beta into bout
 * (PAPER.md:136 ApplyBoost). The pair pass is bound by
 * the FP64 pipe and the boost by HBM, so each SM runs both at once: one TMA
 * producer feeds a pair ring and a boost ring, pair-consumer warps and boost
 * warps share the SM. Arguments, ownership and errors as the two calls; every
 * output is bit-identical to gvx_pair_histograms followed by gvx_boost (which
 * is what runs for shapes the one-launch kernel does not take: non-AoS views,
 * non-PtEtaPhiM pairs, batches under 2^20). bout must not overlap the pair
 * inputs or outputs.
 */
gvx_status gvx_pair_histograms_boost(gvx_dtype dtype, gvx_coords coords, const gvx_vec4_cview *v1,
                                     const gvx_vec4_cview *v2, int64_t n, double lo, double hi,
                                     int32_t nbins, unsigned long long *lab_bins,
                                     unsigned long long *cm_bins, void *m_out, void *cm_m_out,
                                     const gvx_vec4_cview *bv, const gvx_vec3_cview *beta,
                                     const gvx_vec4_view *bout, int64_t nb, gvx_stream_t stream);

/*
 * gvx_mass_histogram_peers — gvx_mass_histogram with the cross-GPU bin
 * reduction fused into the kernel tail ("B200-native option").
 * Every CTA adds its privatised counts to `work`, a device-local workspace of
 * nbins+3 uint64 (nbins+2 partial sums, then a ticket word); the CTA that
 * finishes last reads-and-clears the partial sums and pushes each non-zero
 * total once
 *   - to EVERY array of peer_bins[0 .. npeers-1] (a DEVICE array of device
 *     pointers, e.g. torch symmetric memory's buffer_ptrs_dev: P2P system-scope
 *     atomics over NVLink), or
 *   - to mc_bins, an NVSwitch multicast address of the bins
 *     (multimem.red.add.u64; NVLS), when mc_bins != NULL (peer_bins ignored),
 * so a rank issues at most (nbins+2) x npeers remote adds (multicast: nbins+2)
 * per launch, not one per CTA and bin. `work` must be all zero before the first
 * call; every call leaves it all zero again (caller-owned, one per concurrently
 * running call). After every rank's call has completed (the caller's cross-rank
 * barrier), every rank's bins hold the global histogram: an all-reduce(SUM)
 * without a separate collective. Caller's contract: all ranks' bins are zeroed
 * (or hold the running totals) and visible before any rank launches (barrier),
 * and no rank reads them before the barrier that follows. Other arguments,
 * binning and errors as gvx_mass_histogram (boosted_out is not offered here);
 * peer_bins NULL / misaligned, npeers outside [1, 4096], work NULL or
 * misaligned -> INVALID_ARGUMENT.
 */
gvx_status gvx_mass_histogram_peers(gvx_dtype dtype, gvx_coords coords, const gvx_vec4_cview *v1,
                                    const gvx_vec4_cview *v2, int64_t n, double lo, double hi,
                                    int32_t nbins, unsigned long long *const *peer_bins,
                                    int32_t npeers, unsigned long long *mc_bins,
                                    unsigned long long *work, uint32_t flags, void *m_out,
                                    gvx_stream_t stream);

/*
 * gvx_cm_costheta_histogram — CM decay angle ("the CM path's
 * boosted outputs with a cos theta* histogram"; R22). Each pair is
 * boosted to its CM frame exactly as gvx_mass_histogram with
 * GVX_HIST_BOOST_TO_CM does (beta_cm = -(p1+p2)/(E1+E2), lab-parallel axes,
 * R11), and in ONE pass over the inputs
 *   the CM mass M goes to the mass axis (m_lo, m_hi, m_nbins -> m_bins) and
 *   cos theta* = p'1z / |p'1| of boosted vector 1 to the angle axis
 *   (c_lo, c_hi, c_nbins -> c_bins),
 * both binned ROOT-style as gvx_mass_histogram (R12; NaN -> overflow, so an
 * invalid CM boost or |p'1| = 0 lands in both overflow bins; cos theta* = +1
 * exactly lands in the overflow bin of a [-1, 1) axis).
 *   m_bins, c_bins  m_nbins+2 / c_nbins+2 uint64 counters (device), ACCUMULATED.
 *   m_out, cos_out  NULL or n values of dtype (device).
 * Accuracy: M as the CM histogram; |cos_gpu - cos_exact| <= 2 tau_b S / |p'1|,
 * S = E_lab^2 / M_lab (the CM boost's gamma E scale), tau_b = 1e-12 (f64) /
 * 1e-4 (f32, the boosted-vector scale of SURVEY §8(c)).
 * Errors as gvx_mass_histogram, for either axis.
 */
gvx_status gvx_cm_costheta_histogram(gvx_dtype dtype, gvx_coords coords, const gvx_vec4_cview *v1,
                                     const gvx_vec4_cview *v2, int64_t n, double m_lo, double m_hi,
                                     int32_t m_nbins, unsigned long long *m_bins, double c_lo,
                                     double c_hi, int32_t c_nbins, unsigned long long *c_bins,
                                     void *m_out, void *cos_out, gvx_stream_t stream);

/*
 * gvx_dimuon_histogram — jagged, RDataFrame-style events (PAPER.md:366 names
 * the RDataFrame integration as the next step; DESIGN.md
 * R21). Event e owns muons j in [offsets[e], offsets[e+1]) of a flat PtEtaPhiM
 * collection `muons` (any view) with int32 charges `charge[j]`. The event is
 * selected iff it has exactly two muons and charge[j0] * charge[j0+1] < 0;
 * its pair mass (as gvx_invariant_mass) is binned exactly as
 * gvx_mass_histogram bins (bins accumulate; the caller zeroes them).
 *   offsets   n_events + 1 int64, non-decreasing, all within the muon arrays
 *             (caller's guarantee; not re-validated on the device).
 *   m_out     NULL or n_events masses of dtype: the pair mass, NaN if the event
 *             is not selected.
 * The number of selected events is the sum of the bins this call added.
 * Limit: nbins + 2 <= 49152 (the counters are privatised in shared memory);
 * larger axes -> GVX_ERR_UNSUPPORTED, nothing enqueued.
 */
gvx_status gvx_dimuon_histogram(gvx_dtype dtype, const gvx_vec4_cview *muons, const int32_t *charge,
                                const int64_t *offsets, int64_t n_events, double lo, double hi,
                                int32_t nbins, unsigned long long *bins, void *m_out,
                                gvx_stream_t stream);

/*
 * Transfer-inclusive runtime (the host function "handling the
 * device memory allocation and transfers if necessary").
 * A pipeline owns device staging (3 slots x 3 buffers of chunk_events
 * 4-vectors), three CUDA streams and events on the device current at create.
 * A call cuts a HOST-resident batch into chunks; chunk c's H2D copy, chunk
 * c-1's kernels and chunk c-2's D2H copy overlap. Calls are asynchronous with
 * respect to the host: `stream` (the caller's) is made to wait for the whole
 * call, so host buffers must stay valid and outputs are ready after the
 * caller synchronises `stream`. Host buffers should be pinned
 * (cudaHostAlloc / cudaHostRegister) for full PCIe bandwidth. Results are
 * bitwise those of the device entry points on the same data.
 *   create:  dtype, chunk_events in [1, 2^31] -> *out (GVX_ERR_CUDA if device
 *            allocation fails). destroy: waits for the pipeline's work.
 *   gvx_host_pairs: n AoS pairs (h_v1, h_v2, layout by `coords`); any of
 *            h_m_out (n masses), h_bins / h_bins_cm (nbins+2 uint64 each,
 *            OVERWRITTEN with this batch's lab / CM histogram) may be NULL.
 *            Arguments are validated before anything is enqueued, with the
 *            device entries' rules (coords, 1 <= nbins <= 2^28, finite
 *            lo < hi when a histogram is requested) -> INVALID_ARGUMENT.
 *   Consecutive calls on one pipeline are ordered (each waits for the whole
 *   previous call, whatever caller stream either used).
 *   gvx_host_boost: n PxPyPzE vectors h_v, n betas h_beta (AoS [n][3]),
 *            h_out (n vectors).
 */
typedef struct gvx_host_pipeline gvx_host_pipeline;
gvx_status gvx_host_pipeline_create(gvx_dtype dtype, int64_t chunk_events, gvx_host_pipeline **out);
gvx_status gvx_host_pipeline_destroy(gvx_host_pipeline *p);
gvx_status gvx_host_pairs(gvx_host_pipeline *p, gvx_coords coords, const void *h_v1, const void *h_v2,
                          int64_t n, double lo, double hi, int32_t nbins, void *h_m_out,
                          unsigned long long *h_bins, unsigned long long *h_bins_cm,
                          gvx_stream_t stream);
gvx_status gvx_host_boost(gvx_host_pipeline *p, const void *h_v, const void *h_beta, int64_t n,
                          void *h_out, gvx_stream_t stream);

/*
 * Mixed-coordinate pairs (ABI v7). The paper's kernel takes
 * "two particles expressed in any 4-dimensional coordinate system"
 * and the result must not depend on the systems the operands
 * come in. These four calls are the pair entry points above with
 * one coordinate system per operand: v1's components are in coords1, v2's in
 * coords2 (component orders as in the header's Views paragraph). Each vector
 * is converted to PxPyPzE on its own (clamp R2), then the
 * pair is summed and its mass taken, or boosted to its
 * CM frame first (R11). With coords1 == coords2 each call IS the single-system
 * call (same kernels, same bits); otherwise one grid-stride kernel (256-bit
 * loads for 32-byte AoS rows) serves every mixed combination. Arguments,
 * outputs, accuracy and errors as the single-system calls; an invalid coords1
 * or coords2 -> GVX_ERR_INVALID_ARGUMENT. gvx_pair_histograms_boost_mixed
 * runs the boost of (bv, beta) as gvx_boost after the pair pass when the
 * systems differ.
 */
gvx_status gvx_invariant_mass_mixed(gvx_dtype dtype, gvx_coords coords1, gvx_coords coords2,
                                    const gvx_vec4_cview *v1, const gvx_vec4_cview *v2, void *m_out,
                                    int64_t n, gvx_stream_t stream);
gvx_status gvx_mass_histogram_mixed(gvx_dtype dtype, gvx_coords coords1, gvx_coords coords2,
                                    const gvx_vec4_cview *v1, const gvx_vec4_cview *v2, int64_t n,
                                    double lo, double hi, int32_t nbins, unsigned long long *bins,
                                    uint32_t flags, void *m_out, const gvx_vec4_view *boosted_out,
                                    gvx_stream_t stream);
gvx_status gvx_pair_histograms_mixed(gvx_dtype dtype, gvx_coords coords1, gvx_coords coords2,
                                     const gvx_vec4_cview *v1, const gvx_vec4_cview *v2, int64_t n,
                                     double lo, double hi, int32_t nbins, unsigned long long *lab_bins,
                                     unsigned long long *cm_bins, void *m_out, void *cm_m_out,
                                     gvx_stream_t stream);
gvx_status gvx_pair_histograms_boost_mixed(gvx_dtype dtype, gvx_coords coords1, gvx_coords coords2,
                                           const gvx_vec4_cview *v1, const gvx_vec4_cview *v2,
                                           int64_t n, double lo, double hi, int32_t nbins,
                                           unsigned long long *lab_bins, unsigned long long *cm_bins,
                                           void *m_out, void *cm_m_out, const gvx_vec4_cview *bv,
                                           const gvx_vec3_cview *beta, const gvx_vec4_view *bout,
                                           int64_t nb, gvx_stream_t stream);

/* Human-readable name of a status code (static storage). */
const char *gvx_status_string(gvx_status status);
/* The CUDA error string behind the last GVX_ERR_CUDA on this thread. */
const char *gvx_last_cuda_error_string(void);
/* GVX_ABI_VERSION of the loaded library. */
int gvx_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GVX_H */
