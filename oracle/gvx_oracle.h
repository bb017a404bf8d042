/*
 * gvx_oracle.h — plain, slow, single-threaded CPU oracle of the GenVectorX
 * hot path (arXiv 2312.02756).
 *
 * TEST INFRASTRUCTURE, NOT PRODUCT. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library. It
 * shares no code, header, constant or helper with the CUDA path
 * (paper_2312_02756_b200/); neither includes or links the other.
 *
 * Layouts: every array is AoS and contiguous: a 4-vector i occupies
 * v[4i..4i+3] (pt, eta, phi, m) or (px, py, pz, E); a per-event beta occupies
 * beta[3i..3i+2]; a boosted pair occupies 8 values (vector 1 then vector 2).
 * Pair functions take the coordinate system of each operand (coords1 for v1,
 * coords2 for v2; "any 4-dimensional coordinate system").
 */
#ifndef GVX_ORACLE_H
#define GVX_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 4D coordinate systems: component order of a vector. */
enum { GVX_REF_PTETAPHIM = 0, GVX_REF_PXPYPZE = 1, GVX_REF_PXPYPZM = 2, GVX_REF_PTETAPHIE = 3 };
enum { GVX_REF_DOMAIN = 2 };

/* ROOT TH1 FindBin on a uniform axis (reading R12): 0 = underflow,
 * 1..nbins, nbins+1 = overflow (NaN included). */
int32_t gvx_ref_find_bin(double x, double lo, double hi, int32_t nbins);

#define GVX_REF_DECLARE(T, SFX)                                                                   \
    void gvx_ref_invariant_mass_##SFX(int coords1, int coords2, const T *v1, const T *v2, int64_t n, T *m_out,  \
                                      T *elab_out);                                               \
    void gvx_ref_boost_##SFX(const T *v, const T *beta, int64_t n, T *out, T *scale_out);         \
    int gvx_ref_boost_uniform_##SFX(const T *v, T bx, T by, T bz, int64_t n, T *out);             \
    int gvx_ref_lorentz_transform_##SFX(const double *L, const T *v, int64_t n, T *out);          \
    void gvx_ref_cm_mass_##SFX(int coords1, int coords2, const T *v1, const T *v2, int64_t n, T *m_out,         \
                               T *elab_out, T *boosted_out);                                      \
    void gvx_ref_mass_histogram_##SFX(int coords1, int coords2, const T *v1, const T *v2, int64_t n, double lo, \
                                      double hi, int32_t nbins, int cm, uint64_t *bins, T *m_out);  \
    void gvx_ref_cm_costheta_##SFX(int coords1, int coords2, const T *v1, const T *v2, int64_t n, double m_lo,   \
                                   double m_hi, int32_t m_nbins, uint64_t *m_bins, double c_lo,   \
                                   double c_hi, int32_t c_nbins, uint64_t *c_bins, T *m_out,      \
                                   T *cos_out);                                                   \
    int64_t gvx_ref_dimuon_histogram_##SFX(const T *muons, const int32_t *charge,                 \
                                           const int64_t *offsets, int64_t n_events, double lo,   \
                                           double hi, int32_t nbins, uint64_t *bins, T *m_out);

GVX_REF_DECLARE(float, f32)
GVX_REF_DECLARE(double, f64)
#undef GVX_REF_DECLARE

#ifdef __cplusplus
}
#endif
#endif
