// ref_kernels.cuh -- kernels on dense reference-layout arrays (grid.hpp
// layouts) for the value-semantic API: Eq. 14/15 interpolation of single
// fields.  Same arithmetic as prolong_kernel in level_kernels.cuh and as
// oracle/w1mg_oracle.c:or_prolong_*.
#pragma once

#include "device_common.cuh"

namespace w1mg_dev {

// Eq. 14: coarse nc cells -> fine 2 nc cells
__global__ void interp_scalar_ref_kernel(int nc, const double* __restrict__ c,
                                         double* __restrict__ f) {
    const int nf = 2 * nc, wc = nc + 1, wf = nf + 1;
    const int I = blockIdx.x * blockDim.x + threadIdx.x;
    const int J = blockIdx.y * blockDim.y + threadIdx.y;
    if (I > nf || J > nf) return;
    const int i = I >> 1, j = J >> 1;
    const bool io = I & 1, jo = J & 1;
    const long o = (long)j * wc + i;
    double v;
    if (!io && !jo) v = c[o];
    else if (io && !jo) v = 0.5 * (c[o] + c[o + 1]);
    else if (!io && jo) v = 0.5 * (c[o] + c[o + wc]);
    else v = 0.25 * ((c[o] + c[o + 1]) + (c[o + wc] + c[o + wc + 1]));
    f[(long)J * wf + I] = v;
}

// Eq. 15
__global__ void interp_flux_ref_kernel(int nc, const double* __restrict__ cx,
                                       const double* __restrict__ cy, double* __restrict__ fx,
                                       double* __restrict__ fy) {
    const int nf = 2 * nc, wc = nc + 1, wf = nf + 1;
    const int I = blockIdx.x * blockDim.x + threadIdx.x;
    const int J = blockIdx.y * blockDim.y + threadIdx.y;
    if (I > nf || J > nf) return;
    const int i = I >> 1, j = J >> 1;
    if (I < nf) {
        const long o = (long)j * nc + i;
        fx[(long)J * nf + I] = (J & 1) ? 0.5 * (cx[o] + cx[o + nc]) : cx[o];
    }
    if (J < nf) {
        const long o = (long)j * wc + i;
        fy[(long)J * wf + I] = (I & 1) ? 0.5 * (cy[o] + cy[o + 1]) : cy[o];
    }
}

}  // namespace w1mg_dev

namespace w1mg_dev {

// Self-test of the restated fast paths (device_common.cuh: sqrt_rn_fast,
// div_rn_fast, shrink2_nb) against the library operators.  Operands are
// splitmix64 bit patterns shaped into: random exponents over the whole
// range, values near the shrink threshold, and special values (0, denormal,
// Inf, NaN).  Counts mismatching bit patterns (NaN == NaN).
__device__ __forceinline__ unsigned long long sm64(unsigned long long& x) {
    unsigned long long z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ bool same_bits(double a, double b) {
    return (a != a && b != b) || __double_as_longlong(a) == __double_as_longlong(b);
}
__device__ double rn_operand(unsigned long long& st, double scale) {
    const unsigned long long r = sm64(st);
    const int kind = (int)(r & 15);
    const unsigned long long mant = sm64(st) & 0x000FFFFFFFFFFFFFull;
    if (kind == 0) {  // specials
        const double sp[8] = {0.0, -0.0, 4.9e-324, 2.2250738585072009e-308, __longlong_as_double(0x7FF0000000000000ull),
                              __longlong_as_double(0x7FF8000000000000ull), 1.0, 1.7976931348623157e308};
        return sp[(r >> 4) & 7];
    }
    if (kind <= 4) {  // any exponent
        const unsigned long long ex = (r >> 8) % 2047ull;
        return __longlong_as_double((ex << 52) | mant) * (((r >> 40) & 1) ? -1.0 : 1.0);
    }
    // around the problem scale (the shrink threshold mu): [scale/16, 16 scale)
    const double u = __longlong_as_double(0x3FF0000000000000ull | mant);  // [1, 2)
    const int e = (int)((r >> 8) & 7) - 4;
    return (((r >> 40) & 1) ? -1.0 : 1.0) * scale * ldexp(u, e);
}

__global__ void rn_selftest_kernel(long count, unsigned long long seed, double mu, double zt,
                                   unsigned long long* bad) {
    unsigned long long nb_sqrt = 0, nb_div = 0, nb_shr = 0;
    for (long k = blockIdx.x * (long)blockDim.x + threadIdx.x; k < count;
         k += (long)gridDim.x * blockDim.x) {
        unsigned long long st = seed ^ (0xD1B54A32D192ED03ull * (unsigned long long)(k + 1));
        const double a = rn_operand(st, mu);
        const double b = rn_operand(st, mu);
        const double s = fabs(a);
        bool ok;
        const double fs = sqrt_rn_fast(s, ok);
        if (ok && !same_bits(fs, sqrt(s))) ++nb_sqrt;
        const double fq = div_rn_fast(mu, s, ok);
        if (ok && !same_bits(fq, mu / s)) ++nb_div;
        double ux, uy, vx, vy;
        shrink2_nb(a, b, mu, zt, ux, uy);
        shrink<1>(a, b, mu, vx, vy);
        if (!same_bits(ux, vx) || !same_bits(uy, vy)) ++nb_shr;
    }
    atomicAdd(bad + 0, nb_sqrt);
    atomicAdd(bad + 1, nb_div);
    atomicAdd(bad + 2, nb_shr);
}

}  // namespace w1mg_dev
