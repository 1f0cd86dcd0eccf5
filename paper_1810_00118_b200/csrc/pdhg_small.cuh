// pdhg_small.cuh -- level-resident G-prox PDHG for small levels (m = n+1 <= 33).
//
// On the 33^2 level of a PDHG cascade a streaming iteration (three DCT
// launches, dct_kernels.cuh) is almost all launch latency.  Here one CTA per pair
// runs EVERY iteration of the level in one launch:
//   pre      X = A (m - mu varphi_bar) - rho            (pdhg_pre_kernel)
//   Poisson  T = C X, X = T C^T, divide by lambda_k1 + lambda_k2,
//            T = S X, X = (T S^T) / (4 m^2)            (poisson_apply)
//   post     m, varphi, varphi_bar, G^k partials       (pdhg_post_kernel)
//   stop     Eq. 12 residual and the stop rule of finalize_pair<true>
// with the DCT operators C, S and the two m x m work arrays in shared memory
// (4 m^2 doubles: 135 KB at m = 65) and the pair's state in its level buffer
// (L2-resident).  Node arithmetic is the streaming kernels'; the DCT sums run
// in a different order than the streaming DCT (fp64 FMA), which the PDHG parity bar
// (<= 1e-9 relative at fixed iterations) covers.
#pragma once

#include "pdhg_kernels.cuh"

namespace w1mg_dev {

constexpr int kPdhgSmallThreads = 1024;  // launch bound; the launch uses pdhg_small_threads(m)
// threads per CTA: at m = 33, 576 (18 warps) balance the 1089-node phases (two
// passes) and the 561 DCT GEMM tiles (ncu: barrier stalls dominated with 1024)
__host__ __device__ inline int pdhg_small_threads(int m) { return m <= 33 ? 576 : 1024; }
constexpr int kPdhgSmallMaxM = 65;  // shared-memory capacity of the kernel
// Measured on one B200 (config 3 levels, tools/configs.py 3, against the
// earlier library-GEMM streaming iteration): 33^2 level 13.7 us per iteration
// vs 19 us streaming; 65^2 level 50 us vs 21 us (the four m^3 GEMMs on ONE
// SM's fp64 pipe lose to the whole GPU), so the engine is used up to
// m = kPdhgSmallAutoM.
constexpr int kPdhgSmallAutoM = 33;

// levels up to kPdhgStateM also keep the pair's state (m, varphi, varphi_bar,
// rho: 7 arrays) in shared memory for the whole level
constexpr int kPdhgStateM = 33;
__host__ __device__ inline long pdhg_small_smem(int m) {
    return (m <= kPdhgStateM ? 11L : 4L) * m * m * 8;
}

// Out(k, j) = alpha * sum_l A(k, l) * Bop(l, j); m x m column-major in shared
// memory; Bop = B (BT = false) or B^T (BT = true).  One row k and J columns
// per thread (so m * ceil(m / J) <= blockDim threads cover the output in one
// pass): consecutive threads take consecutive rows (conflict-free A loads),
// the B operand is a warp broadcast.  Each output is the fma chain over
// l = 0..m-1 from 0, the same order for every J.
template <bool BT, int J>
__device__ __forceinline__ void smem_gemm(double* __restrict__ Out, const double* __restrict__ A,
                                          const double* __restrict__ B, int m, double alpha) {
    const int jt = (m + J - 1) / J;
    for (int t = threadIdx.x; t < m * jt; t += blockDim.x) {
        const int k = t % m, j0 = (t / m) * J;
        double acc[J];
#pragma unroll
        for (int q = 0; q < J; ++q) acc[q] = 0.0;
        for (int l = 0; l < m; ++l) {
            const double a0 = A[k + l * m];
#pragma unroll
            for (int q = 0; q < J; ++q) {
                const int j = j0 + q;
                const double bq = (j < m) ? (BT ? B[j + l * m] : B[l + j * m]) : 0.0;
                acc[q] = fma(a0, bq, acc[q]);
            }
        }
#pragma unroll
        for (int q = 0; q < J; ++q)
            if (j0 + q < m) Out[k + (j0 + q) * m] = alpha * acc[q];
    }
}
template <bool BT>
__device__ __forceinline__ void smem_gemm_auto(double* Out, const double* A, const double* B, int m,
                                               double alpha) {
    if (m <= 45) smem_gemm<BT, 2>(Out, A, B, m, alpha);
    else smem_gemm<BT, 5>(Out, A, B, m, alpha);
}

template <int Q, bool kS>
__global__ void __launch_bounds__(kPdhgSmallThreads, 1)
pdhg_small_kernel(const SweepArgs a, const double* __restrict__ Cg, const double* __restrict__ Sg,
                  const double* __restrict__ lam_g) {
    const int b = blockIdx.x;
    PairCtl* ctl = a.ctl + b;
    if (ctl->done) return;
    extern __shared__ double sm[];
    __shared__ double wred[kPdhgSmallThreads / 32][3];
    __shared__ double lam[kPdhgSmallMaxM];
    __shared__ int stop_s;
    const Layout L = a.L;
    const int n = L.n, m = n + 1, M2 = m * m, P = L.pitch;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* sC = sm;
    double* sS = sm + M2;
    double* X = sm + 2 * M2;
    double* T = sm + 3 * M2;
    for (int k = tid; k < M2; k += blockDim.x) {
        sC[k] = Cg[k];
        sS[k] = Sg[k];
    }
    if (tid < m) lam[tid] = lam_g[tid];
    double* gmx = pslot_w(a, b, P_MX);
    double* gmy = pslot_w(a, b, P_MY);
    double* gpx = pslot_w(a, b, P_PX);
    double* gpy = pslot_w(a, b, P_PY);
    double* gbx = pslot_w(a, b, P_BX);
    double* gby = pslot_w(a, b, P_BY);
    const double* grho = pslot(a, b, P_RHO);
    // kS: the state lives in shared memory (dense, index k = j m + i, row
    // stride m) for the whole level; else in the level buffer (L2-resident)
    double* mx = kS ? sm + 4 * M2 : gmx;
    double* my = kS ? sm + 5 * M2 : gmy;
    double* px = kS ? sm + 6 * M2 : gpx;
    double* py = kS ? sm + 7 * M2 : gpy;
    double* bx = kS ? sm + 8 * M2 : gbx;
    double* by = kS ? sm + 9 * M2 : gby;
    double* srho = sm + 10 * M2;
    const double* rho = kS ? srho : grho;
    const int RS = kS ? m : P;  // row stride of the state arrays
    if constexpr (kS) {
        for (int k = tid; k < M2; k += blockDim.x) {
            const long o = L.at(k % m, k / m);
            mx[k] = gmx[o];
            my[k] = gmy[o];
            px[k] = gpx[o];
            py[k] = gpy[o];
            bx[k] = gbx[o];
            by[k] = gby[o];
            srho[k] = grho[o];
        }
    }
    const double mu = a.mu, tau = a.tau, ih = a.ih;
    const double scale = 1.0 / (4.0 * double(m) * double(m));  // poisson.cpp:93
    long it = ctl->it;
    const long max_it = ctl->max_it;
    const double tol = ctl->tol;
    double fpr = ctl->fpr;
    __syncthreads();
    for (;;) {
        // ---- pre: X = A v - rho, v = m - mu varphi_bar (pdhg_pre_kernel)
        for (int k = tid; k < M2; k += blockDim.x) {
            const int i = k % m, j = k / m;
            const long o = kS ? (long)k : L.at(i, j);
            const double r_ = (i < n) ? mx[o] - mu * bx[o] : 0.0;
            const double l_ = (i > 0) ? mx[o - 1] - mu * bx[o - 1] : 0.0;
            const double a_ = (j < n) ? my[o] - mu * by[o] : 0.0;
            const double b_ = (j > 0) ? my[o - RS] - mu * by[o - RS] : 0.0;
            const double div = (r_ - l_) * ih + (a_ - b_) * ih;
            X[k] = div - rho[o];
        }
        __syncthreads();
        // ---- Neumann Poisson solve (poisson.cpp:72-95)
        smem_gemm_auto<false>(T, sC, X, m, 1.0);
        __syncthreads();
        smem_gemm_auto<true>(X, T, sC, m, 1.0);
        __syncthreads();
        for (int k = tid; k < M2; k += blockDim.x) {
            const int k1 = k % m, k2 = k / m;
            X[k] = (k == 0) ? 0.0 : X[k] / (lam[k1] + lam[k2]);
        }
        __syncthreads();
        smem_gemm_auto<false>(T, sS, X, m, 1.0);
        __syncthreads();
        smem_gemm_auto<true>(X, T, sS, m, scale);
        __syncthreads();
        // ---- post: m, varphi, varphi_bar + Eq. 12 partials (pdhg_post_kernel)
        double s_dm2 = 0.0, s_dp2 = 0.0, s_cr = 0.0;
        for (int k = tid; k < M2; k += blockDim.x) {
            const int i = k % m, j = k / m;
            const long o = kS ? (long)k : L.at(i, j);
            const bool hx = i < n, hy = j < n;
            const double pc = X[k];
            double mnx = 0.0, mny = 0.0, dmx = 0.0, dmy = 0.0, pox = 0.0, poy = 0.0;
            if (hx) {
                const double mo = mx[o];
                const double v = mo - mu * bx[o];
                mnx = v - (pc - X[k + 1]) * ih;
                dmx = mnx - mo;
                pox = px[o];
            }
            if (hy) {
                const double mo = my[o];
                const double v = mo - mu * by[o];
                mny = v - (pc - X[k + m]) * ih;
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
        s_dm2 = warp_sum(s_dm2);
        s_dp2 = warp_sum(s_dp2);
        s_cr = warp_sum(s_cr);
        if (lane == 0) {
            wred[warp][0] = s_dm2;
            wred[warp][1] = s_dp2;
            wred[warp][2] = s_cr;
        }
        __syncthreads();
        if (tid == 0) {
            double t0 = 0.0, t1 = 0.0, t2 = 0.0;
            for (int w = 0; w < (int)(blockDim.x / 32); ++w) {
                t0 += wred[w][0];
                t1 += wred[w][1];
                t2 += wred[w][2];
            }
            fpr = a.h2 * (t0 / mu + t1 / tau + 2.0 * t2);  // Eq. 12
            if (a.hist && it < a.hist_cap) a.hist[(long)b * a.hist_cap + it] = fpr;
            ++it;
            stop_s = (fpr < tol || it >= max_it || !isfinite(fpr)) ? 1 : 0;
        }
        __syncthreads();
        if (stop_s) break;
        // the node phase of the next iteration rewrites state read above only
        // after these barriers; global writes of this CTA are visible to it
    }
    if constexpr (kS) {
        for (int k = tid; k < M2; k += blockDim.x) {
            const long o = L.at(k % m, k / m);
            gmx[o] = mx[k];
            gmy[o] = my[k];
            gpx[o] = px[k];
            gpy[o] = py[k];
            gbx[o] = bx[k];
            gby[o] = by[k];
        }
    }
    if (tid == 0) {
        ctl->it = it;
        ctl->fpr = fpr;
        ctl->cur = 0;
        if (!isfinite(fpr)) ctl->nonfinite = 1;
        ctl->done = 1;
        if (a.ndone) atomicAdd(a.ndone, 1);
    }
}

}  // namespace w1mg_dev
