// cp_kernels.cuh -- the fused Li et al. primal-dual sweep (Algorithm 1, Eq. 8)
// for sm_100a, batched over independent pairs of one level.
//
// One launch performs one full sweep of proj/src/solver_cp.cpp:22-71 for
// every active pair:
//     m^{k+1}(x) = shrink(m^k(x) - mu A*phi^k(x), mu, p)         (:27-56)
//     phi^{k+1}  = phi^k + tau (A m^{k+1} + A dm - rho)          (:58-68)
//     R^k        = h^2 (sum dm^2/mu + sum dphi^2/tau - 2 sum dphi A dm)  (:70)
// fused into a single pass over HBM: read phi^k, rho, m^k, write phi^{k+1},
// m^{k+1} (8 (3V + 4E) bytes), with phi and m ping-ponged so the
// halo can be recomputed instead of exchanged.
//
// Work decomposition: a warp owns a strip of 31 columns and H rows and marches
// up the rows keeping the previous row's y-flux in registers.  Lane 0 is the
// left halo column (its m^{k+1} feeds the owned lane 1 through a shuffle),
// lanes 1..31 own nodes.  The row below the strip is recomputed once at the
// strip start.  phi(i+1, j) arrives by shuffle from the right neighbour lane
// (lane 31 loads it).  No shared memory and no block barrier on the data
// path; the residual is a warp-shuffle -> block -> last-block tree with a
// fixed order, so it is deterministic run to run.
//
// The last block of each pair (atomic ticket) finalises R^k, appends it to
// the residual history, and sets the pair's stop flag when R^k < tol or the
// iteration cap is hit, exactly like the while loop of solver_cp.cpp:128-136.
// Later launches of a stopped pair exit at their first instruction, so a
// CUDA graph of K sweeps can run ahead of the host without changing results.
#pragma once

#include "device_common.cuh"

namespace w1mg_dev {

struct PairCtl {
    double tol;     // absolute stopping tolerance
    double fpr;     // last residual
    long it;        // sweeps done on this level
    long max_it;    // cap
    int done;       // stop flag
    int cur;        // buffer parity holding the latest state
    int nonfinite;  // residual was NaN/Inf
    int pad;
};

struct SweepArgs {
    double* base;       // pair b, slot s at base + (b*NSLOT + s)*L.plane
    Layout L;
    int ncx;            // column strips (31 owned columns each)
    int nsy;            // row strips
    int H;              // rows per strip
    int ntiles;         // ncx * nsy
    double mu, tau, ih, h2;
    PairCtl* ctl;       // [pairs]
    double* partial;    // [pairs][gridDim.x][3]
    unsigned* ticket;   // [pairs]
    double* hist;       // [pairs][hist_cap] (may be null)
    long hist_cap;
    int* ndone;         // number of stopped pairs
};

constexpr int kSweepWarps = 8;  // warps per block
constexpr int kOwn = 31;        // owned columns per warp

// One node of the m-update: returns the new flux and its increment, zero for
// absent components (solver_cp.cpp:39-54; absent components enter shrink as 0).
template <int PN>
__device__ __forceinline__ void node_flux(bool hx, bool hy, double pc, double pr, double pu,
                                          double mxo, double myo, double mu, double ih,
                                          double& ux, double& uy, double& dx, double& dy) {
    double vx = hx ? mxo - mu * ((pc - pr) * ih) : 0.0;
    double vy = hy ? myo - mu * ((pc - pu) * ih) : 0.0;
    shrink<PN>(vx, vy, mu, ux, uy);
    dx = hx ? ux - mxo : 0.0;
    ux = hx ? ux : 0.0;
    dy = hy ? uy - myo : 0.0;
    uy = hy ? uy : 0.0;
}

template <int PN>
__global__ void __launch_bounds__(kSweepWarps * 32)
cp_sweep_kernel(const SweepArgs a, const int parity) {
    const int pair = blockIdx.y;
    PairCtl* ctl = a.ctl + pair;
    if (*(volatile int*)&ctl->done) return;

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int tile = blockIdx.x * kSweepWarps + warp;
    const Layout L = a.L;
    const int n = L.n;
    const int P = L.pitch;
    const double mu = a.mu, tau = a.tau, ih = a.ih;

    double s_dm2 = 0.0, s_dp2 = 0.0, s_cr = 0.0;

    if (tile < a.ntiles) {
        const int cx = tile % a.ncx;
        const int sy = tile / a.ncx;
        const int i = cx * kOwn - 1 + lane;
        const int j0 = sy * a.H;
        const int j1 = min(j0 + a.H, n + 1);

        double* pb = a.base + (long)pair * NSLOT * L.plane;
        const double* __restrict__ phr = pb + (PHI0 + parity) * L.plane;
        const double* __restrict__ mxr = pb + (MX0 + parity) * L.plane;
        const double* __restrict__ myr = pb + (MY0 + parity) * L.plane;
        const double* __restrict__ rho = pb + RHO * L.plane;
        double* __restrict__ phw = pb + (PHI0 + 1 - parity) * L.plane;
        double* __restrict__ mxw = pb + (MX0 + 1 - parity) * L.plane;
        double* __restrict__ myw = pb + (MY0 + 1 - parity) * L.plane;

        const bool in = (i >= 0) && (i <= n);
        const bool hx = (i >= 0) && (i < n);
        const bool own = (lane > 0) && in;
        const long c0 = L.at(i, 0);  // column offset; row j adds j*P

        // y-flux (and its increment) of the row below the strip.
        double uyb = 0.0, dyb = 0.0;
        if (j0 > 0) {
            const long o = c0 + (long)(j0 - 1) * P;
            double pc = in ? __ldg(phr + o) : 0.0;
            double pu = in ? __ldg(phr + o + P) : 0.0;
            double pr = __shfl_down_sync(0xffffffffu, pc, 1);
            if (lane == 31) pr = hx ? __ldg(phr + o + 1) : 0.0;
            double mxo = hx ? __ldg(mxr + o) : 0.0;
            double myo = in ? __ldg(myr + o) : 0.0;
            double ux, uy, dx, dy;
            node_flux<PN>(hx, in, pc, pr, pu, mxo, myo, mu, ih, ux, uy, dx, dy);
            uyb = uy;
            dyb = dy;
        }

        long o = c0 + (long)j0 * P;
        double pc = in ? __ldg(phr + o) : 0.0;
        double pr = __shfl_down_sync(0xffffffffu, pc, 1);
        if (lane == 31) pr = hx ? __ldg(phr + o + 1) : 0.0;

        for (int j = j0; j < j1; ++j, o += P) {
            const bool hy = in && (j < n);
            // loads for this row (m^k, rho) and the next potential row
            double pu = hy ? __ldg(phr + o + P) : 0.0;
            double pur = (lane == 31 && hx && j < n) ? __ldg(phr + o + P + 1) : 0.0;
            double mxo = hx ? __ldg(mxr + o) : 0.0;
            double myo = hy ? __ldg(myr + o) : 0.0;
            double r = in ? __ldg(rho + o) : 0.0;

            double ux, uy, dx, dy;
            node_flux<PN>(hx, hy, pc, pr, pu, mxo, myo, mu, ih, ux, uy, dx, dy);
            double uxl = __shfl_up_sync(0xffffffffu, ux, 1);
            double dxl = __shfl_up_sync(0xffffffffu, dx, 1);

            // divergence_into x pass then y pass (grid.cpp:52-65)
            double divm = (ux - uxl) * ih + (uy - uyb) * ih;
            double divd = (dx - dxl) * ih + (dy - dyb) * ih;
            double d = tau * (divm + divd - r);
            if (own) {
                phw[o] = pc + d;
                if (hx) mxw[o] = ux;
                if (hy) myw[o] = uy;
                s_dm2 += dx * dx + dy * dy;
                s_dp2 += d * d;
                s_cr += d * divd;
            }
            uyb = uy;
            dyb = dy;
            // advance the potential window one row up
            double nr = __shfl_down_sync(0xffffffffu, pu, 1);
            pr = (lane == 31) ? pur : nr;
            pc = pu;
        }
    }

    // ---- deterministic residual reduction
    __shared__ double red[kSweepWarps][3];
    __shared__ bool is_last;
    s_dm2 = warp_sum(s_dm2);
    s_dp2 = warp_sum(s_dp2);
    s_cr = warp_sum(s_cr);
    if (lane == 0) {
        red[warp][0] = s_dm2;
        red[warp][1] = s_dp2;
        red[warp][2] = s_cr;
    }
    __syncthreads();
    const int nblk = gridDim.x;
    double* part = a.partial + (long)pair * nblk * 3;
    if (threadIdx.x == 0) {
        double t0 = 0.0, t1 = 0.0, t2 = 0.0;
#pragma unroll
        for (int w = 0; w < kSweepWarps; ++w) {
            t0 += red[w][0];
            t1 += red[w][1];
            t2 += red[w][2];
        }
        part[blockIdx.x * 3 + 0] = t0;
        part[blockIdx.x * 3 + 1] = t1;
        part[blockIdx.x * 3 + 2] = t2;
        __threadfence();
        unsigned t = atomicAdd(a.ticket + pair, 1u);
        is_last = (t == (unsigned)nblk - 1);
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();

    // last block of this pair: fixed-order sum of the block partials
    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
    for (int b = threadIdx.x; b < nblk; b += blockDim.x) {
        const volatile double* pv = part + b * 3;
        t0 += pv[0];
        t1 += pv[1];
        t2 += pv[2];
    }
    t0 = warp_sum(t0);
    t1 = warp_sum(t1);
    t2 = warp_sum(t2);
    __syncthreads();
    if (lane == 0) {
        red[warp][0] = t0;
        red[warp][1] = t1;
        red[warp][2] = t2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double sdm2 = 0.0, sdp2 = 0.0, scr = 0.0;
        for (int w = 0; w < kSweepWarps; ++w) {
            sdm2 += red[w][0];
            sdp2 += red[w][1];
            scr += red[w][2];
        }
        double fpr = a.h2 * (sdm2 / mu + sdp2 / a.tau - 2.0 * scr);
        long k = ctl->it;
        if (a.hist && k < a.hist_cap) a.hist[(long)pair * a.hist_cap + k] = fpr;
        ctl->it = k + 1;
        ctl->fpr = fpr;
        ctl->cur = 1 - parity;
        bool finite = isfinite(fpr);
        if (!finite) ctl->nonfinite = 1;
        if (fpr < ctl->tol || k + 1 >= ctl->max_it || !finite) {
            ctl->done = 1;
            atomicAdd(a.ndone, 1);
        }
        a.ticket[pair] = 0u;
        __threadfence();
    }
}

}  // namespace w1mg_dev
