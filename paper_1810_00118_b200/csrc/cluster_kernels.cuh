// cluster_kernels.cuh -- level-resident engine on thread-block clusters.
//
// For 32 <= n <= 256 a whole level of one pair fits in the shared memory of a
// cluster of C <= 16 CTAs (6 (n+1)^2 doubles: phi, rho, m_x, m_y, dm_x, dm_y).
// The cluster runs EVERY sweep of the level in one launch:
//   * CTA c owns node rows [r0_c, r1_c) in its shared memory;
//   * phase A (m-update, in place, dm kept) reads phi(i, r1_c) -- the upper
//     CTA's first row -- through distributed shared memory (DSMEM);
//   * cluster barrier;
//   * phase B (phi-update) reads m, dm of row r0_c - 1 -- the lower CTA's last
//     row -- through DSMEM;
//   * every CTA publishes its three residual sums into CTA 0's shared memory,
//     cluster barrier, then every CTA sums the C partials in rank order and
//     applies the stop rule (solver_cp.cpp:128-136) -- identical decisions, no
//     host round trip, no HBM traffic per sweep.
// Node arithmetic is node_flux / the divergence order of the streaming
// kernels, so fields stay bit-identical to the reference.  C = 1 is the
// single-CTA resident engine.  The final state goes back to buffer 0.
#pragma once

#include <cooperative_groups.h>

#include "cp_kernels.cuh"

namespace w1mg_dev {

namespace cg = cooperative_groups;

constexpr int kClusterThreads = 512;
constexpr long kClusterSmemBudget = 210 * 1024;  // per CTA, dynamic

__host__ __device__ inline int cluster_rows(int n, int C, int c) {
    return (int)((long)(n + 1) * (c + 1) / C - (long)(n + 1) * c / C);
}
__host__ __device__ inline int cluster_row0(int n, int C, int c) {
    return (int)((long)(n + 1) * c / C);
}
// dynamic smem of one CTA: 6 arrays of (max rows) x (n+1) doubles + partials
__host__ inline long cluster_smem_bytes(int n, int C) {
    const int nr = (n + 1 + C - 1) / C;
    return 6L * nr * (n + 1) * 8 + 16L * 3 * 8;
}

template <int PN>
__global__ void __launch_bounds__(kClusterThreads, 1)
cp_cluster_kernel(const SweepArgs a, const int C) {
    cg::cluster_group cluster = cg::this_cluster();
    const int c = (int)cluster.block_rank();
    const int pair = blockIdx.x / C;
    PairCtl* ctl = a.ctl + pair;
    if (ctl->done) return;  // uniform across the cluster (same control block)
    extern __shared__ __align__(16) double sm[];
    const Layout L = a.L;
    const int n = L.n;
    const int W = n + 1;
    const int nrmax = (n + 1 + C - 1) / C;
    const int S = nrmax * W;  // array stride
    double* phi = sm;
    double* rho = sm + S;
    double* mx = sm + 2 * S;
    double* my = sm + 3 * S;
    double* ddx = sm + 4 * S;
    double* ddy = sm + 5 * S;
    double* red = sm + 6 * S;  // [16][3] partials (used in CTA 0)
    const int r0 = cluster_row0(n, C, c);
    const int nr = cluster_rows(n, C, c);
    const int V = nr * W;
    // neighbours' arrays through DSMEM
    const double* up_phi = (c + 1 < C) ? cluster.map_shared_rank(phi, c + 1) : nullptr;
    const int nr_lo = (c > 0) ? cluster_rows(n, C, c - 1) : 0;
    const double* lo_my = (c > 0) ? cluster.map_shared_rank(my, c - 1) + (nr_lo - 1) * W : nullptr;
    const double* lo_dy = (c > 0) ? cluster.map_shared_rank(ddy, c - 1) + (nr_lo - 1) * W : nullptr;

    const int T = blockDim.x;
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int di = T % W, dj = T / W;
    const int i0 = tid % W, jl0 = tid / W;

    double* pb = a.base + (long)pair * NSLOT * L.plane;
    const int cur = ctl->cur;
    {
        const double* gp = pb + (PHI0 + cur) * L.plane;
        const double* gx = pb + (MX0 + cur) * L.plane;
        const double* gy = pb + (MY0 + cur) * L.plane;
        const double* gr = pb + RHO * L.plane;
        int i = i0, jl = jl0;
        for (int k = tid; k < V; k += T) {
            const int j = r0 + jl;
            const long o = L.at(i, j);
            phi[k] = gp[o];
            rho[k] = gr[o];
            mx[k] = (i < n) ? gx[o] : 0.0;
            my[k] = (j < n) ? gy[o] : 0.0;
            i += di;
            jl += dj;
            if (i >= W) { i -= W; ++jl; }
        }
    }
    __shared__ double wred[kClusterThreads / 32][3];
    const double mu = a.mu, zt = a.zt, tau = a.tau, ih = a.ih;
    long it = ctl->it;
    const long max_it = ctl->max_it;
    const double tol = ctl->tol;
    cluster.sync();

    bool stop = false;
    double fpr = 0.0;
    while (!stop) {
        double s_dm2 = 0.0, s_dp2 = 0.0, s_cr = 0.0;
        {  // phase A: flux at owned rows
            int i = i0, jl = jl0;
            for (int k = tid; k < V; k += T) {
                const int j = r0 + jl;
                const bool hx = i < n, hy = j < n;
                const double pc = phi[k];
                const double pr = hx ? phi[k + 1] : 0.0;
                double pu = 0.0;
                if (hy) pu = (jl + 1 < nr) ? phi[k + W] : up_phi[i];
                double ux, uy, dx, dy;
                node_flux<PN>(hx, hy, pc, pr, pu, mx[k], my[k], mu, zt, ih, ux, uy, dx, dy);
                mx[k] = ux;
                my[k] = uy;
                ddx[k] = dx;
                ddy[k] = dy;
                s_dm2 = __fma_rn(dy, dy, __fma_rn(dx, dx, s_dm2));
                i += di;
                jl += dj;
                if (i >= W) { i -= W; ++jl; }
            }
        }
        cluster.sync();  // m^{k+1} of every row visible cluster-wide
        {  // phase B: potential at owned rows (divergence_into order)
            int i = i0, jl = jl0;
            for (int k = tid; k < V; k += T) {
                const int j = r0 + jl;
                const double uxl = (i > 0) ? mx[k - 1] : 0.0;
                const double dxl = (i > 0) ? ddx[k - 1] : 0.0;
                double uyb = 0.0, dyb = 0.0;
                if (j > 0) {
                    if (jl > 0) {
                        uyb = my[k - W];
                        dyb = ddy[k - W];
                    } else {
                        uyb = lo_my[i];
                        dyb = lo_dy[i];
                    }
                }
                const double divm = (mx[k] - uxl) * ih + (my[k] - uyb) * ih;
                const double divd = (ddx[k] - dxl) * ih + (ddy[k] - dyb) * ih;
                const double d = tau * (divm + divd - rho[k]);
                phi[k] = phi[k] + d;
                s_dp2 = __fma_rn(d, d, s_dp2);
                s_cr = __fma_rn(d, divd, s_cr);
                i += di;
                jl += dj;
                if (i >= W) { i -= W; ++jl; }
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
        if (tid < C) {
            // push this CTA's partials into slot c of EVERY CTA (fire-and-forget
            // DSMEM stores); after the barrier each CTA reads only its own copy
            double t0 = 0.0, t1 = 0.0, t2 = 0.0;
            for (int w = 0; w < T / 32; ++w) {
                t0 += wred[w][0];
                t1 += wred[w][1];
                t2 += wred[w][2];
            }
            double* dst = cluster.map_shared_rank(red, tid);
            dst[c * 3 + 0] = t0;
            dst[c * 3 + 1] = t1;
            dst[c * 3 + 2] = t2;
        }
        cluster.sync();  // phi^{k+1} and all partials visible
        if (tid == 0) {  // local reads; rank order = identical sums everywhere
            double sdm2 = 0.0, sdp2 = 0.0, scr = 0.0;
            for (int q = 0; q < C; ++q) {
                sdm2 += red[q * 3 + 0];
                sdp2 += red[q * 3 + 1];
                scr += red[q * 3 + 2];
            }
            const double f = a.h2 * (sdm2 / mu + sdp2 / tau - 2.0 * scr);
            if (c == 0 && a.hist && it < a.hist_cap) a.hist[(long)pair * a.hist_cap + it] = f;
            wred[0][0] = f;
        }
        __syncthreads();
        fpr = wred[0][0];
        ++it;
        stop = (fpr < tol) || (it >= max_it) || !isfinite(fpr);
        // wred and CTA 0's partials are re-written only after the next phase A
        // (+ barriers), which every thread reaches after reading them here
    }
    {  // final state back to buffer 0
        double* gp = pb + PHI0 * L.plane;
        double* gx = pb + MX0 * L.plane;
        double* gy = pb + MY0 * L.plane;
        int i = i0, jl = jl0;
        for (int k = tid; k < V; k += T) {
            const int j = r0 + jl;
            const long o = L.at(i, j);
            gp[o] = phi[k];
            if (i < n) gx[o] = mx[k];
            if (j < n) gy[o] = my[k];
            i += di;
            jl += dj;
            if (i >= W) { i -= W; ++jl; }
        }
    }
    if (c == 0 && tid == 0) {
        ctl->it = it;
        ctl->fpr = fpr;
        ctl->cur = 0;
        if (!isfinite(fpr)) ctl->nonfinite = 1;
        ctl->done = 1;
        atomicAdd(a.ndone, 1);
    }
    cluster.sync();  // keep every CTA's shared memory alive until all DSMEM reads are done
}

}  // namespace w1mg_dev
