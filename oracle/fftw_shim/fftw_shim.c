/* Direct-evaluation DCT-II / DCT-III behind the FFTW r2r API (see fftw3.h).
   TEST INFRASTRUCTURE ONLY. */
#include "fftw3.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

struct w1mg_fftw_plan_s {
    int n0, n1;
    double *in, *out;
    fftw_r2r_kind k0, k1;
    double *c0, *c1; /* n x n cosine tables */
    double* tmp;
};

double* fftw_alloc_real(size_t n) { return (double*)malloc(n * sizeof(double)); }
void fftw_free(void* p) { free(p); }

/* table[k*n + j] = weight of input j in output k */
static double* make_table(int n, fftw_r2r_kind kind) {
    double* t = (double*)malloc((size_t)n * n * sizeof(double));
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j) {
            long num; /* angle = pi * num / (2n), reduced mod 4n */
            if (kind == FFTW_REDFT10) num = ((long)(2 * j + 1) * k) % (4L * n);
            else num = ((long)j * (2 * k + 1)) % (4L * n);
            double c = (double)cosl(pi * (long double)num / (long double)(2 * n));
            double w = 2.0 * c;
            if (kind == FFTW_REDFT01 && j == 0) w = 1.0;
            t[(size_t)k * n + j] = w;
        }
    return t;
}

fftw_plan fftw_plan_r2r_2d(int n0, int n1, double* in, double* out, fftw_r2r_kind k0,
                           fftw_r2r_kind k1, unsigned flags) {
    (void)flags;
    fftw_plan p = (fftw_plan)calloc(1, sizeof(*p));
    p->n0 = n0; p->n1 = n1; p->in = in; p->out = out; p->k0 = k0; p->k1 = k1;
    p->c0 = make_table(n0, k0);
    p->c1 = make_table(n1, k1);
    p->tmp = (double*)malloc((size_t)n0 * n1 * sizeof(double));
    return p;
}

void fftw_execute(const fftw_plan p) {
    const int n0 = p->n0, n1 = p->n1;
    /* along the last (contiguous) dimension */
    for (int r = 0; r < n0; ++r) {
        const double* x = p->in + (size_t)r * n1;
        double* y = p->tmp + (size_t)r * n1;
        for (int k = 0; k < n1; ++k) {
            const double* w = p->c1 + (size_t)k * n1;
            double s = 0.0;
            for (int j = 0; j < n1; ++j) s += w[j] * x[j];
            y[k] = s;
        }
    }
    /* along the first dimension */
    double* col = (double*)malloc((size_t)n0 * sizeof(double));
    for (int c = 0; c < n1; ++c) {
        for (int j = 0; j < n0; ++j) col[j] = p->tmp[(size_t)j * n1 + c];
        for (int k = 0; k < n0; ++k) {
            const double* w = p->c0 + (size_t)k * n0;
            double s = 0.0;
            for (int j = 0; j < n0; ++j) s += w[j] * col[j];
            p->out[(size_t)k * n1 + c] = s;
        }
    }
    free(col);
}

void fftw_destroy_plan(fftw_plan p) {
    if (!p) return;
    free(p->c0); free(p->c1); free(p->tmp); free(p);
}
