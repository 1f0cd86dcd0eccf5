// cp3_kernels.cuh -- THREE Li et al. PD sweeps (solver_cp.cpp:22-71 applied
// three times) per pass over HBM: the two-sweep march of cp2_kernels.cuh with
// a third sweep C trailing sweep B by one row in the same warp.
//
//   * A at row r: phi^k rows r, r+1 and m^k row r (tensor-map ring);
//   * B at row r-1: A's outputs of rows r-1, r (registers / lane+1);
//   * C at row r-2: B's outputs of rows r-2, r-1, rho of row r-2.
// The dependency cone widens one column per sweep on each side: a warp owns
// 27 columns (lanes 3..29).  At the strip bottom A starts three rows early
// (one m-only warm-up row, then two rows whose B / C results are not owned).
// Only phi^{k+3}, m^{k+3} are written: 56 B of compulsory HBM traffic per
// node per THREE sweeps.  Node arithmetic is node_flux / row_update's, so
// fields stay bit-identical to the reference.
//
// Stopping: the residuals R^k, R^{k+1}, R^{k+2} are reduced.  If the
// reference would stop after A or B, the pair is marked done with redo = 1
// or 2 and its latest buffer = the untouched input; the host then runs the
// single-sweep fix-up launch twice (sweep_gate parity < 0), which replays
// exactly the first redo sweeps.
#pragma once

#include <type_traits>

#include "cp2_kernels.cuh"

namespace w1mg_dev {

constexpr int kOwn3 = 27;  // owned columns per warp in the three-sweep march

// Reduction of the three sweeps' residual sums (9 per block) and the
// three-sweep stop rule; partial holds [pairs][blocks][9].
template <int NW>
__device__ __forceinline__ void finish_sweep3(const SweepArgs& a, int pair, int parity,
                                              const double (&v0)[9]) {
    __shared__ double red[NW][9];
    __shared__ bool is_last;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    double v[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) v[q] = warp_sum(v0[q]);
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < 9; ++q) red[warp][q] = v[q];
    __syncthreads();
    const int nblk = gridDim.x;
    double* part = a.partial + (long)pair * nblk * 9;
    if (threadIdx.x == 0) {
        double t[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        for (int w = 0; w < NW; ++w)
#pragma unroll
            for (int q = 0; q < 9; ++q) t[q] += red[w][q];
#pragma unroll
        for (int q = 0; q < 9; ++q) part[blockIdx.x * 9 + q] = t[q];
        __threadfence();
        const unsigned tk = atomicAdd(a.ticket + pair, 1u);
        is_last = (tk == (unsigned)nblk - 1);
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    // last block: fixed-order sum of the blocks' partials
    double t[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int b = threadIdx.x; b < nblk; b += blockDim.x) {
        const volatile double* pv = part + b * 9;
#pragma unroll
        for (int q = 0; q < 9; ++q) t[q] += pv[q];
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) t[q] = warp_sum(t[q]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < 9; ++q) red[warp][q] = t[q];
    __syncthreads();
    if (threadIdx.x != 0) return;
    double s[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int w = 0; w < NW; ++w)
#pragma unroll
        for (int q = 0; q < 9; ++q) s[q] += red[w][q];
    PairCtl* ctl = a.ctl + pair;
    double f[3];
#pragma unroll
    for (int q = 0; q < 3; ++q)
        f[q] = a.h2 * (s[3 * q] / a.mu + s[3 * q + 1] / a.tau - 2.0 * s[3 * q + 2]);  // Eq. 9
    const long k = ctl->it;
    int stop_at = 3;  // sweep of this launch after which the reference stops (3: none)
    for (int q = 0; q < 3; ++q)
        if (f[q] < ctl->tol || k + q + 1 >= ctl->max_it || !isfinite(f[q])) {
            stop_at = q;
            break;
        }
    if (stop_at < 2) {
        // stops after A (replay 1) or B (replay 2): the states were not
        // stored; the fix-up launches replay them from the input buffer and
        // record their residuals
        ctl->cur = parity;
        ctl->redo = stop_at + 1;
        for (int q = 0; q <= stop_at; ++q) ctl->rf[stop_at - q] = f[q];  // rf[redo - 1] = next
        ctl->done = 1;
        atomicAdd(a.ndone, 1);
    } else {
        for (int q = 0; q < 3; ++q)
            if (a.hist && k + q < a.hist_cap) a.hist[(long)pair * a.hist_cap + k + q] = f[q];
        ctl->it = k + 3;
        ctl->fpr = f[2];
        ctl->cur = 1 - parity;
        const bool finite = isfinite(f[2]);
        if (!finite) ctl->nonfinite = 1;
        if (stop_at == 2) {
            ctl->done = 1;
            atomicAdd(a.ndone, 1);
        }
    }
    a.ticket[pair] = 0u;
    __threadfence();
}

// The three-sweep march of one warp over its tile (tensor-map ring of
// kBoxRows-row boxes, see march2).  kInt: every mask folds to a constant.
template <int PN, bool kInt>
__device__ __forceinline__ void march3(const SweepArgs& a, int pair, int parity, int cx, int j0,
                                       int j1, int lane, double* ring, uint64_t* bars,
                                       double (&acc)[9], const void* tm) {
    const Layout L = a.L;
    const int n = L.n;
    const int P = L.pitch;
    const int i = cx * kOwn3 - 3 + lane;
    double* pb = a.base + (long)pair * NSLOT * L.plane;
    const double* __restrict__ phr = pb + (PHI0 + parity) * L.plane;
    const double* __restrict__ mxr = pb + (MX0 + parity) * L.plane;
    const double* __restrict__ myr = pb + (MY0 + parity) * L.plane;
    double* __restrict__ phw = pb + (PHI0 + 1 - parity) * L.plane;
    double* __restrict__ mxw = pb + (MX0 + 1 - parity) * L.plane;
    double* __restrict__ myw = pb + (MY0 + 1 - parity) * L.plane;
    const bool in = kInt || ((i >= 0) && (i <= n));
    const bool hx = kInt || ((i >= 0) && (i < n));
    const bool own = (lane >= 3) && (lane <= 29) && in;
    const double mu = a.mu, zt = a.zt, tau = a.tau, ih = a.ih;

    const int ilo = cx * kOwn3 - 3;  // column of lane 0 (warp-uniform)
    const int a0 = ilo & ~1;         // 16-B aligned box start (TMA requirement)
    const int sh = ilo - a0;
    const int zb = pair * NSLOT + PHI0 + parity;
    constexpr int NR = kBoxRows, NS = kStagesT, PS = NR * kChunk, STG = kStreams * PS;
    if (lane == 0) {
#pragma unroll
        for (int t = 0; t < NS; ++t) mbar_init(&bars[t], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    auto issue = [&](int st, int row) {
        mbar_expect_tx(&bars[st], NR * kStageBytes);
        tmap_g2s_3d(ring + st * STG, tm, a0, row, zb, &bars[st]);
    };
    // A rows rA0 .. rA1, B rows rA0 .. min(j1, n), C rows rA0 .. j1-1
    const int rA0 = max(j0 - 2, 0);
    const int rA1 = min(j1 + 1, n);
    const int rB1 = min(j1, n);
    const int nA = rA1 - rA0 + 1;
    const int nbox = (nA + NR) / NR;  // rows rA0 .. rA1+1
    if (lane == 0)
        for (int t = 0; t < NS && t < nbox; ++t) issue(t, rA0 + t * NR);

    // A's y-flux below row rA0 (m-only warm-up, direct loads)
    double uyA = 0.0, dyA = 0.0;
    if (rA0 > 0) {
        const long o = L.at(i, rA0 - 1);
        const double pc = in ? __ldg(phr + o) : 0.0;
        const double pu = in ? __ldg(phr + o + P) : 0.0;
        const double pr = hx ? __ldg(phr + o + 1) : 0.0;
        const double mxo = hx ? __ldg(mxr + o) : 0.0;
        const double myo = in ? __ldg(myr + o) : 0.0;
        double ux, uy, dx, dy;
        node_flux<PN>(hx, in, pc, pr, pu, mxo, myo, mu, zt, ih, ux, uy, dx, dy);
        uyA = uy;
        dyA = dy;
    }
    // C's stores go two rows below A: running pointers
    const long o0 = L.at(i, rA0) - 2L * P;
    double* __restrict__ wph = phw + o0;
    double* __restrict__ wmx = mxw + o0;
    double* __restrict__ wmy = myw + o0;
    mbar_wait(&bars[0], 0u);
    double pc = in ? ring[sh + lane] : 0.0;  // phi^k(i, rA), phi^k(i+1, rA)
    double pr = hx ? ring[sh + lane + 1] : 0.0;

    // B state: A's outputs of the previous row, rho of the previous row;
    // C state: B's outputs of the previous row, rho two rows back
    double fA_prev = 0.0, mxA_prev = 0.0, myA_prev = 0.0, r_prev = 0.0;
    double fB_prev = 0.0, mxB_prev = 0.0, myB_prev = 0.0, r_prev2 = 0.0;
    double uyB = 0.0, dyB = 0.0, uyC = 0.0, dyC = 0.0;

    // mode: 0 = rows tested at run time, 3 = middle step (A, B, C rows all
    // owned grid rows: no row tests; non-owned lanes are zeroed at the end).
    // par: 0 even t, 1 odd t, 2 run time (position of the rows in the boxes).
    auto step = [&](const int t, auto mode, auto par) {
        constexpr int kMode = decltype(mode)::value;
        constexpr int kPar = decltype(par)::value;
        const int rA = rA0 + t, rB = rA - 1, rC = rA - 2;
        double fA = 0.0, uxA = 0.0, uyAn = 0.0, dxA = 0.0, dyAn = 0.0, r = 0.0;
        double pu = 0.0, pur = 0.0;
        if (kMode == 3 || kInt || rA <= rA1) {
            const bool odd = (kPar == 0) ? false : (kPar == 1) ? true : ((t & 1) != 0);
            const int bt = t >> 1;
            const int st = bt % NS;
            const double* c = ring + st * STG + (odd ? kChunk : 0) + sh + lane;
            const double* cph;
            if (odd) {  // row t+1 opens the next box
                const int bu = (t + 1) >> 1;
                const int su = bu % NS;
                mbar_wait(&bars[su], (uint32_t)((bu / NS) & 1));
                cph = ring + su * STG + sh + lane;
            } else {
                cph = c + kChunk;
            }
            const bool hy = kInt || (in && (rA < n));
            pu = hy ? cph[0] : 0.0;
            pur = (kInt || (hx && rA < n)) ? cph[1] : 0.0;
            const double mxo = hx ? c[PS] : 0.0;
            const double myo = hy ? c[2 * PS] : 0.0;
            r = in ? c[3 * PS] : 0.0;
            if (odd) {
                __syncwarp();
                if (lane == 0 && bt + NS < nbox) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    issue(st, rA0 + (bt + NS) * NR);
                }
            }
            // ---- sweep A at row rA
            node_flux<PN>(hx, hy, pc, pr, pu, mxo, myo, mu, zt, ih, uxA, uyAn, dxA, dyAn);
            const double uxl = __shfl_up_sync(0xffffffffu, uxA, 1);
            const double dxl = __shfl_up_sync(0xffffffffu, dxA, 1);
            double divd;
            const double d =
                phi_delta<PN>(uxA, uxl, uyAn, uyA, dxA, dxl, dyAn, dyA, r, ih, tau, divd);
            fA = pc + d;
            if (kMode == 3 || (own && rA >= j0 && rA < j1)) {
                acc[0] = __fma_rn(dyAn, dyAn, __fma_rn(dxA, dxA, acc[0]));
                acc[1] = __fma_rn(d, d, acc[1]);
                acc[2] = __fma_rn(d, divd, acc[2]);
            }
            uyA = uyAn;
            dyA = dyAn;
        }
        // ---- sweep B at row rB (inputs: A's rows rB and rB + 1)
        double fB = 0.0, uxB = 0.0, uyBn = 0.0;
        if (kMode == 3 || (rB >= rA0 && rB <= rB1)) {
            const bool hyB = kInt || (in && (rB < n));
            const double prB = __shfl_down_sync(0xffffffffu, fA_prev, 1);
            const double puB = hyB ? fA : 0.0;
            double dx, dy;
            node_flux<PN>(hx, hyB, fA_prev, hx ? prB : 0.0, puB, mxA_prev, myA_prev, mu, zt, ih,
                          uxB, uyBn, dx, dy);
            const double uxl = __shfl_up_sync(0xffffffffu, uxB, 1);
            const double dxl = __shfl_up_sync(0xffffffffu, dx, 1);
            double divd;
            const double d =
                phi_delta<PN>(uxB, uxl, uyBn, uyB, dx, dxl, dy, dyB, r_prev, ih, tau, divd);
            fB = fA_prev + d;
            if (kMode == 3 || (own && rB >= j0 && rB < j1)) {
                acc[3] = __fma_rn(dy, dy, __fma_rn(dx, dx, acc[3]));
                acc[4] = __fma_rn(d, d, acc[4]);
                acc[5] = __fma_rn(d, divd, acc[5]);
            }
            uyB = uyBn;
            dyB = dy;
        }
        // ---- sweep C at row rC (inputs: B's rows rC and rC + 1)
        if (kMode == 3 || rC >= rA0) {
            const bool hyC = kInt || (in && (rC < n));
            const double prC = __shfl_down_sync(0xffffffffu, fB_prev, 1);
            const double puC = hyC ? fB : 0.0;
            double ux, uy, dx, dy;
            node_flux<PN>(hx, hyC, fB_prev, hx ? prC : 0.0, puC, mxB_prev, myB_prev, mu, zt, ih, ux,
                          uy, dx, dy);
            const double uxl = __shfl_up_sync(0xffffffffu, ux, 1);
            const double dxl = __shfl_up_sync(0xffffffffu, dx, 1);
            double divd;
            const double d =
                phi_delta<PN>(ux, uxl, uy, uyC, dx, dxl, dy, dyC, r_prev2, ih, tau, divd);
            if (own && (kMode == 3 || rC >= j0)) {  // rC < j1 always
                *wph = fB_prev + d;
                if (hx) *wmx = ux;
                if (hyC) *wmy = uy;
            }
            if (kMode == 3 || (own && rC >= j0)) {
                acc[6] = __fma_rn(dy, dy, __fma_rn(dx, dx, acc[6]));
                acc[7] = __fma_rn(d, d, acc[7]);
                acc[8] = __fma_rn(d, divd, acc[8]);
            }
            uyC = uy;
            dyC = dy;
        }
        fB_prev = fB;
        mxB_prev = uxB;
        myB_prev = uyBn;
        r_prev2 = r_prev;
        fA_prev = fA;
        mxA_prev = uxA;
        myA_prev = uyAn;
        r_prev = r;
        pc = pu;
        pr = pur;
    };
    auto next_row = [&] {
        wph += P;
        wmx += P;
        wmy += P;
    };
    using M0 = std::integral_constant<int, 0>;
    using M3 = std::integral_constant<int, 3>;
    using PE = std::integral_constant<int, 0>;
    using PO = std::integral_constant<int, 1>;
    using PR = std::integral_constant<int, 2>;
    const int T = j1 + 1 - rA0;  // last step: C at row j1 - 1
    // middle steps: A row < j1 and C row >= j0
    const int tm0 = j0 + 2 - rA0, tm1 = j1 - rA0;
    int t = 0;
    for (; t < tm0 && t <= T; ++t, next_row()) step(t, M0{}, PR{});
    if (t < tm1 && (t & 1)) {
        step(t, M3{}, PO{});
        next_row();
        ++t;
    }
#pragma unroll 1
    for (; t + 1 < tm1; t += 2) {
        step(t, M3{}, PE{});
        next_row();
        step(t + 1, M3{}, PO{});
        next_row();
    }
    if (t < tm1) {
        step(t, M3{}, PE{});
        next_row();
        ++t;
    }
    for (; t <= T; ++t, next_row()) step(t, M0{}, PR{});
    if (!own)
#pragma unroll
        for (int q = 0; q < 9; ++q) acc[q] = 0.0;
}

constexpr int kWarps3 = 4;
constexpr int tmap3_smem(int nw) { return nw * (kStagesT * kBoxRows * kStageBytes + kStagesT * 8); }

template <int PN>
__device__ __forceinline__ void cp_sweep3_tmap_body(const SweepArgs& a, const int parity, const CUtensorMap& tm,
                      const int pdl_early) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (pdl_early) asm volatile("griddepcontrol.launch_dependents;");
    const int pair = sweep_pair(a);
    if (pair < 0 || *(volatile int*)&a.ctl[pair].done) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
    const int tile = blockIdx.x * kWarps3 + warp;
    double* ring = reinterpret_cast<double*>(smem_raw) +
                   (size_t)warp * kStagesT * kBoxRows * kStreams * kChunk;
    uint64_t* bars =
        reinterpret_cast<uint64_t*>(smem_raw + kWarps3 * kStagesT * kBoxRows * kStageBytes) +
        warp * kStagesT;
    double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    if (tile < a.ntiles) {
        const int cx = tile % a.ncx;
        const int sy = tile / a.ncx;
        const int j0 = a.jlo + sy * a.H;
        const int j1 = min(j0 + a.H, a.jhi);
        const int ilo = cx * kOwn3 - 3;
        const int n = a.L.n;
        // interior: columns ilo..ilo+32 carry x-edges, rows j0-3..j1+1 < n
        const bool interior = (ilo >= 0) && (ilo + 32 < n) && (j0 >= 3) && (j1 + 1 < n);
        if (interior) march3<PN, true>(a, pair, parity, cx, j0, j1, lane, ring, bars, acc, &tm);
        else march3<PN, false>(a, pair, parity, cx, j0, j1, lane, ring, bars, acc, &tm);
    }
    finish_sweep3<kWarps3>(a, pair, parity, acc);
}

template <int PN>
__global__ void __launch_bounds__(kWarps3 * 32, 5)
cp_sweep3_tmap_kernel(const SweepArgs a, const int parity, const __grid_constant__ CUtensorMap tm,
                      const int pdl_early) {
    cp_sweep3_tmap_body<PN>(a, parity, tm, pdl_early);
}

// four CTAs per SM (<= 128 registers, no spills), option "occ3" = 4 (A/B)
template <int PN>
__global__ void __launch_bounds__(kWarps3 * 32, 4)
cp_sweep3_tmap4_kernel(const SweepArgs a, const int parity, const __grid_constant__ CUtensorMap tm,
                       const int pdl_early) {
    cp_sweep3_tmap_body<PN>(a, parity, tm, pdl_early);
}

}  // namespace w1mg_dev
