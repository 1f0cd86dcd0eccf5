// pdhg_fold.cuh -- the PDHG iteration's Poisson solve with symmetry-folded
// DCTs (odd m = n+1), halving the GEMM flops of the dense sandwich.
//
// With C(k, l) = 2 cos(pi (2l+1) k / 2m):  C(k, m-1-l) = (-1)^k C(k, l), and
// C(k odd, mid) = 0 for mid = (m-1)/2.  So a length-m DCT-II splits into
//   y_{2k'}   = sum_{l' <= mid} C(2k', l') e_l',   e_l = x_l + x_{m-1-l}, e_mid = x_mid
//   y_{2k'+1} = sum_{l' <  mid} C(2k'+1, l') o_l', o_l = x_l - x_{m-1-l}
// and with S(k, j) (DCT-III, S(m-1-k, j) = (-1)^j S(k, j), S(mid, j odd) = 0)
// the inverse gives x_k = u_k + w_k, x_{m-1-k} = u_k - w_k, x_mid = u_mid with
// u = S_e y_even, w = S_o y_odd.  In 2-D every node array becomes four h x h
// quadrants (h = mid + 1; the odd classes padded with zeros), one per
// (parity along i, parity along j), and each 2-D transform is four half-size
// sandwiches: 2 * 4 * h^3 multiply-adds instead of 2 * m^3 -- one batched
// cuBLAS call per stage over 4B (pair, quadrant) products.
//
// Quadrant q = 2a + b of a slot starts at L.at(0, 0) + q * h * lq (lq = pitch/2
// >= h; four quadrants fill exactly the (m+1) x pitch node rows), element
// (r, c) at r + c * lq (column-major, r along i).
//   pdhg_pre_fold_kernel   X = A v - rho, folded into the quadrants of P_RES
//   (4 batched GEMM stages + spectral_divide_fold_kernel)  -> quadrants of P_PSI
//   pdhg_post_fold_kernel  pdhg_post_kernel with psi unfolded on the fly
// Node arithmetic is the dense path's; only the DCT sums are regrouped.
#pragma once

#include "pdhg_kernels.cuh"

namespace w1mg_dev {

struct FoldGeom {
    int h;   // (m+1)/2
    int lq;  // quadrant leading dimension (pitch / 2)
};

__device__ __forceinline__ double* fold_q(const SweepArgs& a, int b, int slot, const FoldGeom& g,
                                          int q) {
    return pslot_w(a, b, slot) + a.L.at(0, 0) + (long)q * g.h * g.lq;
}

// A v - rho at node (i, j), v = m - mu varphi_bar (pdhg_pre_kernel)
__device__ __forceinline__ double pre_value(const SweepArgs& a, int b, int i, int j) {
    const Layout& L = a.L;
    const int n = L.n;
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
    return div - pslot(a, b, P_RHO)[o];
}

// one thread per quadrant cell (r, c) in [0, h)^2
__global__ void __launch_bounds__(256) pdhg_pre_fold_kernel(const SweepArgs a, const FoldGeom g) {
    const int b = blockIdx.z;
    if (*(volatile int*)&a.ctl[b].done) return;
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int cc = blockIdx.y * blockDim.y + threadIdx.y;
    const int h = g.h;
    if (r >= h || cc >= h) return;
    const int m = a.L.n + 1, mid = h - 1;
    const int rb = m - 1 - r, cb = m - 1 - cc;
    const bool rm = (r == mid), cm = (cc == mid);
    const double x00 = pre_value(a, b, r, cc);
    const double x10 = rm ? 0.0 : pre_value(a, b, rb, cc);
    const double x01 = cm ? 0.0 : pre_value(a, b, r, cb);
    const double x11 = (rm || cm) ? 0.0 : pre_value(a, b, rb, cb);
    // fold along i, then along j (middle row/column: sum part only)
    const double E = rm ? x00 : x00 + x10, O = rm ? 0.0 : x00 - x10;
    const double E2 = rm ? x01 : x01 + x11, O2 = rm ? 0.0 : x01 - x11;
    const long e = r + (long)cc * g.lq;
    fold_q(a, b, P_RES, g, 0)[e] = cm ? E : E + E2;
    fold_q(a, b, P_RES, g, 1)[e] = cm ? 0.0 : E - E2;
    fold_q(a, b, P_RES, g, 2)[e] = cm ? O : O + O2;
    fold_q(a, b, P_RES, g, 3)[e] = cm ? 0.0 : O - O2;
}

// quadrant (a, b) cell (r, c) holds frequency (2r + a, 2c + b)
__global__ void spectral_divide_fold_kernel(const SweepArgs a, const FoldGeom g,
                                            const double* __restrict__ lambda) {
    const int bp = blockIdx.z >> 2, q = blockIdx.z & 3;
    if (*(volatile int*)&a.ctl[bp].done) return;
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int cc = blockIdx.y * blockDim.y + threadIdx.y;
    if (r >= g.h || cc >= g.h) return;
    const int m = a.L.n + 1;
    const int k1 = 2 * r + (q >> 1), k2 = 2 * cc + (q & 1);
    double* Y = fold_q(a, bp, P_RES, g, q);
    const long e = r + (long)cc * g.lq;
    Y[e] = (k1 >= m || k2 >= m || (k1 == 0 && k2 == 0)) ? 0.0 : Y[e] / (lambda[k1] + lambda[k2]);
}

// psi(i, j) = P00 + s_j P01 + s_i P10 + s_i s_j P11 at the folded index
__device__ __forceinline__ double psi_unfold(const SweepArgs& a, int b, const FoldGeom& g, int i,
                                             int j) {
    const int m = a.L.n + 1, mid = g.h - 1;
    const int r = (i <= mid) ? i : m - 1 - i;
    const int cc = (j <= mid) ? j : m - 1 - j;
    const double si = (i < mid) ? 1.0 : (i > mid ? -1.0 : 0.0);
    const double sj = (j < mid) ? 1.0 : (j > mid ? -1.0 : 0.0);
    const long e = r + (long)cc * g.lq;
    double v = fold_q(a, b, P_PSI, g, 0)[e];
    if (sj != 0.0) v += sj * fold_q(a, b, P_PSI, g, 1)[e];
    if (si != 0.0) {
        v += si * fold_q(a, b, P_PSI, g, 2)[e];
        if (sj != 0.0) v += (si * sj) * fold_q(a, b, P_PSI, g, 3)[e];
    }
    return v;
}

// pdhg_post_kernel with psi read through psi_unfold
template <int Q>
__global__ void __launch_bounds__(256) pdhg_post_fold_kernel(const SweepArgs a, const FoldGeom g) {
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
        const double mu = a.mu, tau = a.tau, ih = a.ih;
        const double pc = psi_unfold(a, b, g, i, j);
        double mnx = 0.0, mny = 0.0, dmx = 0.0, dmy = 0.0, pox = 0.0, poy = 0.0;
        if (hx) {
            const double mo = mx[o];
            const double v = mo - mu * bx[o];
            mnx = v - (pc - psi_unfold(a, b, g, i + 1, j)) * ih;
            dmx = mnx - mo;
            pox = px[o];
        }
        if (hy) {
            const double mo = my[o];
            const double v = mo - mu * by[o];
            mny = v - (pc - psi_unfold(a, b, g, i, j + 1)) * ih;
            dmy = mny - mo;
            poy = py[o];
        }
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

}  // namespace w1mg_dev
