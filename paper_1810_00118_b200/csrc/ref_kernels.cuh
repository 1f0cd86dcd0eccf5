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
