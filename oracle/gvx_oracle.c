/*
 * gvx_oracle.c — plain, slow, single-threaded CPU oracle of the GenVectorX
 * data-parallel hot path (arXiv 2312.02756, §4.1, Fig. 1).
 *
 * TEST INFRASTRUCTURE, NOT PRODUCT. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it. It shares no
 * code with the CUDA path (paper_2312_02756_b200/csrc): it is plain C, built
 * by gcc with `-O2 -ffp-contract=off` against glibc libm, and evaluates the
 * paper's formulas literally, element by element, in the order the passage
 * cited beside each function writes them. No blocking, fusion, algebraic
 * rewriting or reordering. Every function is pinned by `-m "not gpu"` tests
 * (tests/test_oracle_pins.py) against closed forms, the SPEC's worked
 * examples, 50-digit mpmath truth and brute force; see DESIGN.md §3.
 *
 * Readings where the paper is silent are numbered R1..R20 in DESIGN.md §3.
 */
#include <math.h>
#include <tgmath.h>
#include <stdint.h>
#include "gvx_oracle.h"

/* ROOT TH1/TAxis FindFixBin on a uniform axis, reading R12:
 *   x <  lo           -> 0 (underflow)
 *   !(x < hi) or NaN  -> nbins + 1 (overflow)
 *   otherwise         -> 1 + (int)((nbins * (x − lo)) / (hi − lo))
 * evaluated in double in exactly that order (no clamp). */
int32_t gvx_ref_find_bin(double x, double lo, double hi, int32_t nbins)
{
    if (x < lo)
        return 0;
    if (!(x < hi))
        return nbins + 1;
    return 1 + (int32_t)(((double)nbins * (x - lo)) / (hi - lo));
}

#define T float
#define SFX f32
#define NANT ((float)NAN)
#include "gvx_oracle_body.inc"
#undef T
#undef SFX
#undef NANT

#define T double
#define SFX f64
#define NANT ((double)NAN)
#include "gvx_oracle_body.inc"
#undef T
#undef SFX
#undef NANT
