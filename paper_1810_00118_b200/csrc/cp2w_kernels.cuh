// cp2w_kernels.cuh -- the two-sweep march with TWO column sets per lane.
//
// Same algorithm and arithmetic as cp_sweep2_tma_kernel (cp2_kernels.cuh),
// but a warp covers 64 columns: lane l carries columns ilo + l (set 0) and
// ilo + 32 + l (set 1).  The per-row fixed cost of the march (mbarrier wait,
// TMA issue, loop control, uniform address arithmetic) is shared by twice the
// nodes and each lane has two independent node chains in flight.  Neighbour
// values that cross from set 0 to set 1 (lane 31 -> lane 0) travel through one
// rotated shuffle.  Owned columns per warp: set 0 lanes 2..31, set 1 lanes
// 0..30 (61).  Blocks are 4 warps (128 threads) to keep occupancy with the
// larger register state.
#pragma once

#include "cp2_kernels.cuh"

namespace w1mg_dev {

constexpr int kWarpsW = 4;        // warps per block
constexpr int kOwnW = 61;         // owned columns per warp
constexpr int kChunkW = 68;       // doubles per row chunk (66 needed, 16-B aligned)
constexpr int kStageBytesW = kStreams * kChunkW * 8;
constexpr int kTmaSmemW = kWarpsW * (kStages * kStageBytesW + kStages * 8);

// v of set 0 at lane l <- set 0 at l-1; set 1 at l <- set 1 at l-1, and set 1
// at lane 0 <- set 0 at lane 31
__device__ __forceinline__ void shfl_left2(double v0, double v1, int lane, double& l0, double& l1) {
    l0 = __shfl_up_sync(0xffffffffu, v0, 1);
    const double x = (lane == 31) ? v0 : v1;
    l1 = __shfl_sync(0xffffffffu, x, (lane + 31) & 31);
}
// right neighbours: set 0 at l <- set 0 at l+1, set 0 at lane 31 <- set 1 at
// lane 0; set 1 at l <- set 1 at l+1 (lane 31: invalid, not owned)
__device__ __forceinline__ void shfl_right2(double v0, double v1, int lane, double& r0, double& r1) {
    const double x = (lane == 0) ? v1 : v0;
    r0 = __shfl_sync(0xffffffffu, x, (lane + 1) & 31);
    r1 = __shfl_down_sync(0xffffffffu, v1, 1);
}

template <int PN, bool kInt>
__device__ __forceinline__ void march2w(const SweepArgs& a, int pair, int parity, int cx, int j0,
                                        int j1, int lane, double* ring, uint64_t* bars,
                                        double* acc) {
    const Layout L = a.L;
    const int n = L.n;
    const int P = L.pitch;
    const int ilo = cx * kOwnW - 2;  // column of lane 0, set 0 (warp-uniform)
    int col[2] = {ilo + lane, ilo + 32 + lane};
    double* pb = a.base + (long)pair * NSLOT * L.plane;
    const double* __restrict__ phr = pb + (PHI0 + parity) * L.plane;
    const double* __restrict__ mxr = pb + (MX0 + parity) * L.plane;
    const double* __restrict__ myr = pb + (MY0 + parity) * L.plane;
    const double* __restrict__ rho = pb + RHO * L.plane;
    double* __restrict__ phw = pb + (PHI0 + 1 - parity) * L.plane;
    double* __restrict__ mxw = pb + (MX0 + 1 - parity) * L.plane;
    double* __restrict__ myw = pb + (MY0 + 1 - parity) * L.plane;
    bool in[2], hx[2], own[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        in[s] = kInt || ((col[s] >= 0) && (col[s] <= n));
        hx[s] = kInt || ((col[s] >= 0) && (col[s] < n));
    }
    own[0] = (lane >= 2) && in[0];
    own[1] = (lane <= 30) && in[1];
    const double mu = a.mu, zt = a.zt, tau = a.tau, ih = a.ih;

    const int a0 = ilo & ~1;
    const int sh = ilo - a0;
    const long c0 = L.at(a0, 0);
    if (lane == 0) {
#pragma unroll
        for (int t = 0; t < kStages; ++t) mbar_init(&bars[t], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    auto issue = [&](int st, int row) {
        double* dst = ring + st * kStreams * kChunkW;
        const long orow = c0 + (long)row * P;
        mbar_expect_tx(&bars[st], kStageBytesW);
        bulk_g2s(dst + 0 * kChunkW, phr + orow + P, kChunkW * 8, &bars[st]);
        bulk_g2s(dst + 1 * kChunkW, mxr + orow, kChunkW * 8, &bars[st]);
        bulk_g2s(dst + 2 * kChunkW, myr + orow, kChunkW * 8, &bars[st]);
        bulk_g2s(dst + 3 * kChunkW, rho + orow, kChunkW * 8, &bars[st]);
    };
    const int rA0 = max(j0 - 1, 0);
    const int rA1 = min(j1, n);
    const int nA = rA1 - rA0 + 1;
    if (lane == 0) {
        for (int t = 0; t < kStages && t < nA; ++t) issue(t, rA0 + t);
    }

    double uyA[2] = {0.0, 0.0}, dyA[2] = {0.0, 0.0};
    double pc[2], pr[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        if (rA0 > 0) {
            const long o = L.at(col[s], rA0 - 1);
            double c_ = in[s] ? __ldg(phr + o) : 0.0;
            double u_ = in[s] ? __ldg(phr + o + P) : 0.0;
            double r_ = hx[s] ? __ldg(phr + o + 1) : 0.0;
            double mx_ = hx[s] ? __ldg(mxr + o) : 0.0;
            double my_ = in[s] ? __ldg(myr + o) : 0.0;
            double ux, uy, dx, dy;
            node_flux<PN>(hx[s], in[s], c_, r_, u_, mx_, my_, mu, zt, ih, ux, uy, dx, dy);
            uyA[s] = uy;
            dyA[s] = dy;
        }
        const long o = L.at(col[s], rA0);
        pc[s] = in[s] ? __ldg(phr + o) : 0.0;
        pr[s] = hx[s] ? __ldg(phr + o + 1) : 0.0;
    }
    double fA_prev[2] = {0.0, 0.0}, mxA_prev[2] = {0.0, 0.0}, myA_prev[2] = {0.0, 0.0};
    double r_prev[2] = {0.0, 0.0};
    double uyB[2] = {0.0, 0.0}, dyB[2] = {0.0, 0.0};
    long o0 = L.at(col[0], rA0);  // set 1 is o0 + 32

    for (int t = 0; t <= j1 - rA0; ++t, o0 += P) {
        const int rA = rA0 + t;
        const int rB = rA - 1;
        double fA[2] = {0.0, 0.0}, uxA[2] = {0.0, 0.0}, uyAn[2] = {0.0, 0.0};
        double dxA[2] = {0.0, 0.0}, dyAn[2] = {0.0, 0.0}, r[2] = {0.0, 0.0};
        double pu[2] = {0.0, 0.0}, pur[2] = {0.0, 0.0};
        if (kInt || rA <= rA1) {
            const int st = t % kStages;
            mbar_wait(&bars[st], (uint32_t)((t / kStages) & 1));
            const double* c = ring + st * kStreams * kChunkW + sh + lane;
            double mxo[2], myo[2];
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const double* cs = c + 32 * s;
                const bool hy = kInt || (in[s] && (rA < n));
                pu[s] = hy ? cs[0] : 0.0;
                pur[s] = (kInt || (hx[s] && rA < n)) ? cs[1] : 0.0;
                mxo[s] = hx[s] ? cs[kChunkW] : 0.0;
                myo[s] = hy ? cs[2 * kChunkW] : 0.0;
                r[s] = in[s] ? cs[3 * kChunkW] : 0.0;
            }
            __syncwarp();
            if (lane == 0 && t + kStages < nA) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(st, rA + kStages);
            }
            // ---- sweep A at row rA, both column sets
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const bool hy = kInt || (in[s] && (rA < n));
                node_flux<PN>(hx[s], hy, pc[s], pr[s], pu[s], mxo[s], myo[s], mu, zt, ih, uxA[s],
                              uyAn[s], dxA[s], dyAn[s]);
            }
            double uxl[2], dxl[2];
            shfl_left2(uxA[0], uxA[1], lane, uxl[0], uxl[1]);
            shfl_left2(dxA[0], dxA[1], lane, dxl[0], dxl[1]);
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const double divm = (uxA[s] - uxl[s]) * ih + (uyAn[s] - uyA[s]) * ih;
                const double divd = (dxA[s] - dxl[s]) * ih + (dyAn[s] - dyA[s]) * ih;
                const double d = tau * (divm + divd - r[s]);
                fA[s] = pc[s] + d;
                if (own[s] && rA >= j0 && rA < j1) {
                    acc[0] = __fma_rn(dyAn[s], dyAn[s], __fma_rn(dxA[s], dxA[s], acc[0]));
                    acc[1] = __fma_rn(d, d, acc[1]);
                    acc[2] = __fma_rn(d, divd, acc[2]);
                }
                uyA[s] = uyAn[s];
                dyA[s] = dyAn[s];
            }
        }
        // ---- sweep B at row rB
        if (rB >= rA0) {
            double prB[2];
            shfl_right2(fA_prev[0], fA_prev[1], lane, prB[0], prB[1]);
            double ux[2], uy[2], dx[2], dy[2];
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const bool hyB = kInt || (in[s] && (rB < n));
                node_flux<PN>(hx[s], hyB, fA_prev[s], hx[s] ? prB[s] : 0.0, hyB ? fA[s] : 0.0,
                              mxA_prev[s], myA_prev[s], mu, zt, ih, ux[s], uy[s], dx[s], dy[s]);
            }
            double uxl[2], dxl[2];
            shfl_left2(ux[0], ux[1], lane, uxl[0], uxl[1]);
            shfl_left2(dx[0], dx[1], lane, dxl[0], dxl[1]);
#pragma unroll
            for (int s = 0; s < 2; ++s) {
                const bool hyB = kInt || (in[s] && (rB < n));
                const double divm = (ux[s] - uxl[s]) * ih + (uy[s] - uyB[s]) * ih;
                const double divd = (dx[s] - dxl[s]) * ih + (dy[s] - dyB[s]) * ih;
                const double d = tau * (divm + divd - r_prev[s]);
                if (own[s] && rB >= j0) {
                    const long ob = o0 + 32 * s - P;
                    phw[ob] = fA_prev[s] + d;
                    if (hx[s]) mxw[ob] = ux[s];
                    if (hyB) myw[ob] = uy[s];
                    acc[3] = __fma_rn(dy[s], dy[s], __fma_rn(dx[s], dx[s], acc[3]));
                    acc[4] = __fma_rn(d, d, acc[4]);
                    acc[5] = __fma_rn(d, divd, acc[5]);
                }
                uyB[s] = uy[s];
                dyB[s] = dy[s];
            }
        }
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            fA_prev[s] = fA[s];
            mxA_prev[s] = uxA[s];
            myA_prev[s] = uyAn[s];
            r_prev[s] = r[s];
            pc[s] = pu[s];
            pr[s] = pur[s];
        }
    }
}

template <int PN>
__global__ void __launch_bounds__(kWarpsW * 32, 3)
cp_sweep2w_tma_kernel(const SweepArgs a, const int parity) {
    const int pair = sweep_pair(a);
    if (pair < 0 || *(volatile int*)&a.ctl[pair].done) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
    const int tile = blockIdx.x * kWarpsW + warp;
    double* ring = reinterpret_cast<double*>(smem_raw) + (size_t)warp * kStages * kStreams * kChunkW;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + kWarpsW * kStages * kStageBytesW) +
                     warp * kStages;
    double acc[6] = {0, 0, 0, 0, 0, 0};
    if (tile < a.ntiles) {
        const int cx = tile % a.ncx;
        const int sy = tile / a.ncx;
        const int j0 = a.jlo + sy * a.H;
        const int j1 = min(j0 + a.H, a.jhi);
        const int ilo = cx * kOwnW - 2;
        const int n = a.L.n;
        const bool interior = (ilo >= 0) && (ilo + 64 < n) && (j0 >= 2) && (j1 < n);
        if (interior) march2w<PN, true>(a, pair, parity, cx, j0, j1, lane, ring, bars, acc);
        else march2w<PN, false>(a, pair, parity, cx, j0, j1, lane, ring, bars, acc);
    }
    finish_sweep2<kWarpsW>(a, pair, parity, acc[0], acc[1], acc[2], acc[3], acc[4], acc[5]);
}

}  // namespace w1mg_dev
