// pdhg_kernels.cuh -- G-prox PDHG (Algorithm 2, paper Eq. 11/12) and the
// Neumann Poisson solve behind its affine projection, for sm_100a.
//
// Reference semantics (no reference implementation exists; the header
// proj/include/w1mg/solver_pdhg.hpp:8-46 and SPEC.md:261-323 define it):
//   v          = m^k - mu varphi_bar^k                       (edges)
//   psi        = (A A*)^{-1} (A v - rho)                    (poisson.cpp:111-117)
//   m^{k+1}    = v - A* psi                                 (poisson.cpp:118-131)
//   varphi^{k+1}(x) = Proj_{|.|_q <= 1}(varphi^k(x) + tau m^{k+1}(x))  (prox.cpp:47-62)
//   varphi_bar = 2 varphi^{k+1} - varphi^k
//   G^k = h^2 (sum dm^2/mu + sum dvarphi^2/tau + 2 sum dvarphi dm)     (Eq. 12)
//
// Poisson solve (poisson.cpp:72-99, FFTW REDFT10 -> divide -> REDFT01): the
// separable 2D DCT-II/III on the m x m node grid (m = n+1) runs in the
// hand-written prime-factor DCT kernels of dct_kernels.cuh, which also fuse
// the two node steps of an iteration (three launches per iteration):
//   pre   v = m - mu varphi_bar, r = A v - rho   (into the row DCT-II)
//   post  m, varphi, varphi_bar update + G^k partials + stop rule (after the
//         row DCT-III; pdhg_post_kernel below is the standalone form used by
//         the affine projection)
// v is recomputed in the post step (same expression, same bits) instead of
// being stored.  The mean removal of psi is skipped inside the iteration: A*
// annihilates constants, so it only perturbs rounding; the public solve
// (w1mg_poisson_solve) does remove it like poisson.cpp:96-98.
#pragma once

#include "cp_kernels.cuh"
#include "device_common.cuh"

namespace w1mg_dev {

// PDHG level slots (planes of one pair)
enum PSlot {
    P_MX = 0, P_MY = 1,   // m
    P_PX = 2, P_PY = 3,   // varphi
    P_BX = 4, P_BY = 5,   // varphi_bar
    P_RHO = 6,
    P_RES = 7,            // A v - rho / Poisson RHS (m x m, ld = pitch)
    P_T = 8,              // DCT intermediate (rows transformed)
    P_PSI = 9,            // Poisson solution
    P_NSLOT = 10
};

__device__ __forceinline__ const double* pslot(const SweepArgs& a, int b, int s) {
    return a.base + ((long)b * P_NSLOT + s) * a.L.plane;
}
__device__ __forceinline__ double* pslot_w(const SweepArgs& a, int b, int s) {
    return a.base + ((long)b * P_NSLOT + s) * a.L.plane;
}

// r = A v - rho at every node (divergence_into then "-= rho", poisson.cpp:113-115)
__global__ void __launch_bounds__(256) pdhg_pre_kernel(const SweepArgs a) {
    const int b = blockIdx.z;
    if (*(volatile int*)&a.ctl[b].done) return;
    const Layout L = a.L;
    const int n = L.n;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    if (i > n || j > n) return;
    const double* mx = pslot(a, b, P_MX);
    const double* my = pslot(a, b, P_MY);
    const double* bx = pslot(a, b, P_BX);
    const double* by = pslot(a, b, P_BY);
    const double mu = a.mu, ih = a.ih;
    const long o = L.at(i, j);
    const double r_ = (i < n) ? mx[o] - mu * bx[o] : 0.0;
    const double l_ = (i > 0) ? mx[o - 1] - mu * bx[o - 1] : 0.0;
    const double a_ = (j < n) ? my[o] - mu * by[o] : 0.0;
    const double b_ = (j > 0) ? my[o - L.pitch] - mu * by[o - L.pitch] : 0.0;
    const double div = (r_ - l_) * ih + (a_ - b_) * ih;
    pslot_w(a, b, P_RES)[o] = div - pslot(a, b, P_RHO)[o];
}

// m, varphi, varphi_bar update + Eq. 12 partials + stop rule.
template <int Q>
__global__ void __launch_bounds__(256) pdhg_post_kernel(const SweepArgs a) {
    const int b = blockIdx.z;
    if (*(volatile int*)&a.ctl[b].done) return;
    const Layout L = a.L;
    const int n = L.n;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    double s_dm2 = 0.0, s_dp2 = 0.0, s_cr = 0.0;
    if (i <= n && j <= n) {
        const long o = L.at(i, j);
        const bool hx = i < n, hy = j < n;
        double* mx = pslot_w(a, b, P_MX);
        double* my = pslot_w(a, b, P_MY);
        double* px = pslot_w(a, b, P_PX);
        double* py = pslot_w(a, b, P_PY);
        double* bx = pslot_w(a, b, P_BX);
        double* by = pslot_w(a, b, P_BY);
        const double* psi = pslot(a, b, P_PSI);
        const double mu = a.mu, tau = a.tau, ih = a.ih;
        const double pc = psi[o];
        double mnx = 0.0, mny = 0.0, dmx = 0.0, dmy = 0.0, pox = 0.0, poy = 0.0;
        if (hx) {
            const double mo = mx[o];
            const double v = mo - mu * bx[o];
            mnx = v - (pc - psi[o + 1]) * ih;  // poisson.cpp:124
            dmx = mnx - mo;
            pox = px[o];
        }
        if (hy) {
            const double mo = my[o];
            const double v = mo - mu * by[o];
            mny = v - (pc - psi[o + L.pitch]) * ih;  // poisson.cpp:130
            dmy = mny - mo;
            poy = py[o];
        }
        // node vector of varphi^k + tau m^{k+1}, absent components 0
        const double wx = hx ? pox + tau * mnx : 0.0;
        const double wy = hy ? poy + tau * mny : 0.0;
        double qx, qy;
        proj_unit_ball<Q>(wx, wy, qx, qy);
        if (hx) {
            mx[o] = mnx;
            px[o] = qx;
            bx[o] = 2.0 * qx - pox;
            const double dp = qx - pox;
            s_dm2 += dmx * dmx;
            s_dp2 += dp * dp;
            s_cr += dp * dmx;
        }
        if (hy) {
            my[o] = mny;
            py[o] = qy;
            by[o] = 2.0 * qy - poy;
            const double dp = qy - poy;
            s_dm2 += dmy * dmy;
            s_dp2 += dp * dp;
            s_cr += dp * dmy;
        }
    }
    finish_sweep<true>(a, b, /*parity=*/1, blockIdx.x + blockIdx.y * gridDim.x,
                       gridDim.x * gridDim.y, s_dm2, s_dp2, s_cr);
}

// r = A varphi (for recover_potential) into P_RES
__global__ void pdhg_div_dual_kernel(const SweepArgs a) {
    const int b = blockIdx.z;
    const Layout L = a.L;
    const int n = L.n;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    if (i > n || j > n) return;
    const double* px = pslot(a, b, P_PX);
    const double* py = pslot(a, b, P_PY);
    const long o = L.at(i, j);
    const double ih = a.ih;
    const double l = (i > 0) ? px[o - 1] : 0.0;
    const double r = (i < n) ? px[o] : 0.0;
    const double bb = (j > 0) ? py[o - L.pitch] : 0.0;
    const double aa = (j < n) ? py[o] : 0.0;
    pslot_w(a, b, P_RES)[o] = (r - l) * ih + (aa - bb) * ih;
}

// psi -= mean (poisson.cpp:96-98), mean = sums[b] / m^2
__global__ void subtract_mean_kernel(const SweepArgs a, int slot, const double* __restrict__ sums) {
    const int b = blockIdx.z;
    const Layout L = a.L;
    const int n = L.n;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    if (i > n || j > n) return;
    const double cnt = (double)(n + 1) * (double)(n + 1);
    pslot_w(a, b, slot)[L.at(i, j)] -= sums[b] / cnt;
}

struct FPSlot {  // value of one PDHG slot
    const double* base;
    Layout L;
    int slot;
    __device__ double operator()(int b, int i, int j) const {
        return base[((long)b * P_NSLOT + slot) * L.plane + L.at(i, j)];
    }
};

struct FPDual {  // psi * rho (dual value with the recovered potential)
    const double* base;
    Layout L;
    __device__ double operator()(int b, int i, int j) const {
        const double* pb = base + (long)b * P_NSLOT * L.plane;
        const long o = L.at(i, j);
        return pb[P_PSI * L.plane + o] * pb[P_RHO * L.plane + o];
    }
};

template <int PN>
struct FPPrimal {  // ||m(x)||_p on the PDHG layout
    const double* base;
    Layout L;
    __device__ double operator()(int b, int i, int j) const {
        const double* pb = base + (long)b * P_NSLOT * L.plane;
        const long o = L.at(i, j);
        const double x = (i < L.n) ? pb[P_MX * L.plane + o] : 0.0;
        const double y = (j < L.n) ? pb[P_MY * L.plane + o] : 0.0;
        return vec_norm<PN>(x, y);
    }
};

// Cold-start tolerance for the cascade (SURVEY D3 analogue): the first G
// from the zero state, times rel; then reset the control block for the run.
__global__ void pdhg_arm_tol_kernel(PairCtl* ctl, int npairs, double rel, long max_it, int* ndone) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b == 0) *ndone = 0;
    if (b >= npairs) return;
    PairCtl c = ctl[b];
    c.tol = rel * c.fpr;
    c.fpr = 0.0;
    c.it = 0;
    c.max_it = max_it;
    c.done = max_it <= 0 ? 1 : 0;
    c.nonfinite = 0;
    ctl[b] = c;
}

// Eq. 15 prolongation of m and varphi (varphi_bar := varphi) between PDHG levels.
__global__ void pdhg_prolong_kernel(const double* __restrict__ cbase, Layout Lc, double* fbase,
                                    Layout Lf) {
    const int nf = Lf.n;
    const int I = blockIdx.x * blockDim.x + threadIdx.x;
    const int J = blockIdx.y * blockDim.y + threadIdx.y;
    const int b = blockIdx.z;
    if (I > nf || J > nf) return;
    const double* cb = cbase + (long)b * P_NSLOT * Lc.plane;
    double* fb = fbase + (long)b * P_NSLOT * Lf.plane;
    const int i = I >> 1, j = J >> 1;
    const long o = Lf.at(I, J);
    if (I < nf) {
        const double* cm = cb + P_MX * Lc.plane;
        const double* cp = cb + P_PX * Lc.plane;
        const double m = (J & 1) ? 0.5 * (cm[Lc.at(i, j)] + cm[Lc.at(i, j + 1)]) : cm[Lc.at(i, j)];
        const double p = (J & 1) ? 0.5 * (cp[Lc.at(i, j)] + cp[Lc.at(i, j + 1)]) : cp[Lc.at(i, j)];
        fb[P_MX * Lf.plane + o] = m;
        fb[P_PX * Lf.plane + o] = p;
        fb[P_BX * Lf.plane + o] = p;
    }
    if (J < nf) {
        const double* cm = cb + P_MY * Lc.plane;
        const double* cp = cb + P_PY * Lc.plane;
        const double m = (I & 1) ? 0.5 * (cm[Lc.at(i, j)] + cm[Lc.at(i + 1, j)]) : cm[Lc.at(i, j)];
        const double p = (I & 1) ? 0.5 * (cp[Lc.at(i, j)] + cp[Lc.at(i + 1, j)]) : cp[Lc.at(i, j)];
        fb[P_MY * Lf.plane + o] = m;
        fb[P_PY * Lf.plane + o] = p;
        fb[P_BY * Lf.plane + o] = p;
    }
}

}  // namespace w1mg_dev
