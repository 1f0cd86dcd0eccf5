/*
 * Test-only stand-in for the five FFTW3 symbols proj/src/poisson.cpp uses
 * (poisson.cpp:3,32-46,82,91).  FFTW3 itself is not installed in this image.
 * REDFT10 is the unnormalised DCT-II, REDFT01 the unnormalised DCT-III, both
 * with FFTW's published definitions; the transforms are evaluated directly
 * (O(m^3) per 2D transform) -- fine for the oracle sizes (m <= 513).
 * TEST INFRASTRUCTURE ONLY: linked into oracle/_ref/libw1mg_ref.so.
 */
#ifndef W1MG_FFTW_SHIM_H
#define W1MG_FFTW_SHIM_H
#include <stddef.h>
#ifdef __cplusplus
extern "C" {
#endif
typedef enum { FFTW_REDFT01 = 4, FFTW_REDFT10 = 5 } fftw_r2r_kind;
#define FFTW_ESTIMATE (1U << 6)
typedef struct w1mg_fftw_plan_s* fftw_plan;
double* fftw_alloc_real(size_t n);
void fftw_free(void* p);
fftw_plan fftw_plan_r2r_2d(int n0, int n1, double* in, double* out, fftw_r2r_kind k0,
                           fftw_r2r_kind k1, unsigned flags);
void fftw_execute(const fftw_plan p);
void fftw_destroy_plan(fftw_plan p);
#ifdef __cplusplus
}
#endif
#endif
