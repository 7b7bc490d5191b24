/* CPU oracle for the DG Euler residual and RK stage update.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library;
 * the product (paper_2209_01877_b200) never does.
 *
 * It restates the reference's numba kernels (hodg/dg.py:240-460,
 * hodg/timestepping.py:105-180) in C with the same loop order and
 * expression trees; compiled with -ffp-contract=off so the 2D results are
 * bitwise equal to the reference (pinned by tests/golden/residuals_*.csv).
 * OpenMP over faces / cells with disjoint writes, as the reference's prange.
 */
#include <math.h>
#include <stdint.h>

#define CAT_(a, b) a##b
#define CAT(a, b) CAT_(a, b)

#define REAL double
#define SFX _f64
#define SQRT sqrt
#define FABS fabs
#define POW pow
#include "hodg_oracle_body.h"
#undef REAL
#undef SFX
#undef SQRT
#undef FABS
#undef POW

#define REAL float
#define SFX _f32
#define SQRT sqrtf
#define FABS fabsf
#define POW powf
#include "hodg_oracle_body.h"
#undef REAL
#undef SFX
#undef SQRT
#undef FABS
#undef POW

#ifdef _OPENMP
#include <omp.h>
#endif

int ora_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}
