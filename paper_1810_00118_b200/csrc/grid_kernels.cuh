// grid_kernels.cuh -- level-persistent cooperative-grid engine: a whole CP
// level of ONE pair in one launch, state resident in L2.
//
// For a single pair on a mid-size level (n = 256..1024: 4-70 MB of state,
// inside the 126 MB L2) the streaming sweep is launch/ramp bound: one pair
// gives too few strips to fill 148 SMs and every launch pays its pipeline
// fill.  Here the grid (every SM, co-resident, cudaLaunchCooperativeKernel)
// loops over the sweeps itself:
//
//   sweep k:  each warp marches its strips (the fused m/phi update of
//             cp_sweep_kernel, loads through L2 with ld.global.cg because the
//             state is rewritten by other SMs between sweeps), warp -> block
//             residual partials -> gpart[k & 1][block];
//   grid.sync();
//   every block reduces gpart[k & 1][0..G) in the same fixed order, so all
//   blocks compute the identical R^k and take the identical stop decision
//   (no second barrier); block 0 records it in the pair's PairCtl.
//
// gpart is double-buffered by sweep parity: buffer k & 1 is rewritten at
// sweep k + 2, after the barrier of sweep k + 1 that every block reaches only
// after it has read sweep k's partials.  Per-node arithmetic is exactly the
// streaming kernel's, so fields stay bit-identical to the reference; only the
// residual sum is reassociated (like every engine).
#pragma once

#include <cooperative_groups.h>

#include "cp_kernels.cuh"

namespace w1mg_dev {

constexpr int kGridWarps = 8;

// y-flux of the row below a strip (below_row with L2-coherent loads)
template <int PN>
__device__ __forceinline__ void below_row_cg(const SweepArgs& a, const Strip& s, int lane,
                                             double& uyb, double& dyb) {
    uyb = 0.0;
    dyb = 0.0;
    if (s.j0 == 0) return;
    const Layout& L = a.L;
    const long o = L.at(s.i, s.j0 - 1);
    double pc = s.in ? __ldcg(s.phr + o) : 0.0;
    double pu = s.in ? __ldcg(s.phr + o + L.pitch) : 0.0;
    double pr = __shfl_down_sync(0xffffffffu, pc, 1);
    if (lane == 31) pr = s.hx ? __ldcg(s.phr + o + 1) : 0.0;
    double mxo = s.hx ? __ldcg(s.mxr + o) : 0.0;
    double myo = s.in ? __ldcg(s.myr + o) : 0.0;
    double ux, uy, dx, dy;
    node_flux<PN>(s.hx, s.in, pc, pr, pu, mxo, myo, a.mu, a.zt, a.ih, ux, uy, dx, dy);
    uyb = uy;
    dyb = dy;
}

// One strip of one sweep (the march of cp_sweep_kernel, loads one row ahead).
template <int PN>
__device__ __forceinline__ void grid_strip(const SweepArgs& a, int parity, int tile, int lane,
                                           double& s_dm2, double& s_dp2, double& s_cr) {
    const Strip s = make_strip(a, 0, parity, tile, lane);
    const Layout L = a.L;
    const int n = L.n;
    const int P = L.pitch;
    double uyb, dyb;
    below_row_cg<PN>(a, s, lane, uyb, dyb);
    long o = L.at(s.i, s.j0);
    double pc = s.in ? __ldcg(s.phr + o) : 0.0;
    double pr = __shfl_down_sync(0xffffffffu, pc, 1);
    if (lane == 31) pr = s.hx ? __ldcg(s.phr + o + 1) : 0.0;
    const bool l31 = (lane == 31) && s.hx;
    double n_pu, n_pur, n_mx, n_my, n_r;
    {
        const bool hy = s.in && (s.j0 < n);
        n_pu = hy ? __ldcg(s.phr + o + P) : 0.0;
        n_pur = (l31 && s.j0 < n) ? __ldcg(s.phr + o + P + 1) : 0.0;
        n_mx = s.hx ? __ldcg(s.mxr + o) : 0.0;
        n_my = hy ? __ldcg(s.myr + o) : 0.0;
        n_r = s.in ? __ldg(s.rho + o) : 0.0;  // rho is never written: read-only path is safe
    }
    for (int j = s.j0; j < s.j1; ++j, o += P) {
        const double pu = n_pu, pur = n_pur, mxo = n_mx, myo = n_my, r = n_r;
        if (j + 1 < s.j1) {
            const long q = o + P;
            const bool hy1 = s.in && (j + 1 < n);
            n_pu = hy1 ? __ldcg(s.phr + q + P) : 0.0;
            n_pur = (l31 && j + 1 < n) ? __ldcg(s.phr + q + P + 1) : 0.0;
            n_mx = s.hx ? __ldcg(s.mxr + q) : 0.0;
            n_my = hy1 ? __ldcg(s.myr + q) : 0.0;
            n_r = s.in ? __ldg(s.rho + q) : 0.0;
        }
        row_update<PN>(a, s, j, o, pc, pr, pu, mxo, myo, r, uyb, dyb, s_dm2, s_dp2, s_cr);
        const double nr = __shfl_down_sync(0xffffffffu, pu, 1);
        pr = (lane == 31) ? pur : nr;
        pc = pu;
    }
}

// The whole level of pair 0 (a.ctl[0]) until its stop rule fires.
// gpart: [2][gridDim.x][3] doubles.
template <int PN>
__global__ void __launch_bounds__(kGridWarps * 32)
cp_grid_kernel(const SweepArgs a, double* __restrict__ gpart) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    PairCtl* ctl = a.ctl;
    if (*(volatile int*)&ctl->done) return;  // uniform: nothing writes ctl before the loop
    __shared__ double red[kGridWarps][3];
    __shared__ int stop_s;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int gw = blockIdx.x * kGridWarps + warp;
    const int TW = gridDim.x * kGridWarps;
    const int G = gridDim.x;
    int parity = ctl->cur;
    long k = ctl->it;
    const long max_it = ctl->max_it;
    const double tol = ctl->tol;
    for (;;) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0;
        for (int tile = gw; tile < a.ntiles; tile += TW)
            grid_strip<PN>(a, parity, tile, lane, s0, s1, s2);
        s0 = warp_sum(s0);
        s1 = warp_sum(s1);
        s2 = warp_sum(s2);
        if (lane == 0) {
            red[warp][0] = s0;
            red[warp][1] = s1;
            red[warp][2] = s2;
        }
        __syncthreads();
        double* gp = gpart + (size_t)(k & 1) * G * 3;
        if (threadIdx.x == 0) {
            double t0 = 0.0, t1 = 0.0, t2 = 0.0;
            for (int w = 0; w < kGridWarps; ++w) {
                t0 += red[w][0];
                t1 += red[w][1];
                t2 += red[w][2];
            }
            __stcg(gp + blockIdx.x * 3 + 0, t0);
            __stcg(gp + blockIdx.x * 3 + 1, t1);
            __stcg(gp + blockIdx.x * 3 + 2, t2);
        }
        grid.sync();
        if (warp == 0) {
            double t0 = 0.0, t1 = 0.0, t2 = 0.0;
            for (int b = lane; b < G; b += 32) {
                t0 += __ldcg(gp + b * 3 + 0);
                t1 += __ldcg(gp + b * 3 + 1);
                t2 += __ldcg(gp + b * 3 + 2);
            }
            t0 = warp_sum(t0);
            t1 = warp_sum(t1);
            t2 = warp_sum(t2);
            if (lane == 0) {
                const double fpr = a.h2 * (t0 / a.mu + t1 / a.tau - 2.0 * t2);  // Eq. 9
                const bool finite = isfinite(fpr);
                const bool stop = fpr < tol || k + 1 >= max_it || !finite;
                if (blockIdx.x == 0) {
                    if (a.hist && k < a.hist_cap) a.hist[k] = fpr;
                    ctl->it = k + 1;
                    ctl->fpr = fpr;
                    ctl->cur = 1 - parity;
                    if (!finite) ctl->nonfinite = 1;
                    if (stop) {
                        ctl->done = 1;
                        if (a.ndone) atomicAdd(a.ndone, 1);
                    }
                }
                stop_s = stop ? 1 : 0;
            }
        }
        __syncthreads();
        ++k;
        parity = 1 - parity;
        if (stop_s) break;
        __syncthreads();  // stop_s is rewritten next sweep
    }
}

}  // namespace w1mg_dev
