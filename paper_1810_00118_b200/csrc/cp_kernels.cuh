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
// strip start.  No block barrier on the data path; the residual is a
// warp-shuffle -> block -> last-block tree with a fixed order, so it is
// deterministic run to run.
//
// Two load engines feed the march:
//   * kLdg: register double-buffering of plain LDGs one row ahead;
//   * kTma: per-warp ring of kStages row chunks in shared memory filled by
//     cp.async.bulk (TMA bulk copies, one elected lane, mbarrier complete_tx),
//     so kStages rows of look-ahead cost no registers.
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
    int redo;       // a multi-sweep launch stopped after its first (second) sweep: replay 1 (2)
    double rf[2];   // residuals that launch computed for the replayed sweeps, rf[redo - 1] is
                    // the next one: the replay records them instead of its own re-summation,
                    // so history, fpr and `converged` are the values the stop was decided on
};

// Launch gate shared by the single-sweep kernels.  parity >= 0: a normal
// sweep of every running pair.  parity < 0: the fix-up sweep, run only for
// pairs flagged `redo`, from their own latest buffer.
__device__ __forceinline__ bool sweep_gate(const PairCtl* ctl, int parity, int& par) {
    if (parity >= 0) {
        par = parity;
        return !*(const volatile int*)&ctl->done;
    }
    par = ctl->cur;
    return ctl->redo != 0;
}

struct SweepArgs {
    double* base;       // pair b, slot s at base + (b*NSLOT + s)*L.plane
    Layout L;
    int ncx;            // column strips (31 owned columns each)
    int nsy;            // row strips
    int H;              // rows per strip
    int jlo, jhi;       // owned global rows [jlo, jhi): [0, n+1) unless a row slab
    double* red_out;    // slab mode: last block writes its pair's 3 local sums here
    int ntiles;         // ncx * nsy
    double mu, tau, ih, h2;
    double zt;          // largest s with sqrt_rn(s) <= mu: the p = 2 shrink's zero test (host, exact)
    PairCtl* ctl;       // [pairs]
    double* partial;    // [pairs][gridDim.x][3]
    unsigned* ticket;   // [pairs]
    double* hist;       // [pairs][hist_cap] (may be null)
    long hist_cap;
    int* ndone;         // number of stopped pairs
    const int* act;     // compacted launch: blockIdx.y indexes act[0, *nact) (null: pair = blockIdx.y)
    const int* nact;
    // row slab with the fused peer transport (slab_engine.cuh): the sweep
    // stores its top owned row into the upper neighbour's lower halo row and
    // its first row's phi into the lower neighbour's upper halo row (peer
    // memory: NVLink P2P stores, or another slab on the same device), and the
    // last block posts the slab's residual sums to every rank's mailbox.
    double* up_base;    // upper neighbour's level buffer (null: none)
    long up_plane;
    int up_row0;
    double* dn_base;    // lower neighbour's level buffer (null: none)
    long dn_plane;
    int dn_row0;
    double* const* mail;                // [pworld] mailboxes, each [2][pworld][3]
    unsigned long long* const* arrive;  // [pworld] arrival counters
    int prank, pworld;
    int psys;  // peers on other GPUs: system-scope fences/atomics (0: same device)
    // two-level residual reduction of the two-sweep kernels (finish_sweep2):
    // group partials [pairs][gstride][6] and group tickets [pairs][gstride]
    double* gpart;
    unsigned* gticket;
    int gstride;
};

// Pair of this block.  In a compacted launch (the tail of a batched level, see
// run_sweeps) the grid only spans the pairs still running; -1 = no work.
__device__ __forceinline__ int sweep_pair(const SweepArgs& a) {
    if (!a.act) return blockIdx.y;
    return (int)blockIdx.y < *a.nact ? a.act[blockIdx.y] : -1;
}

constexpr int kSweepWarps = 8;  // warps per block
constexpr int kOwn = 31;        // owned columns per warp
constexpr int kLdg = 0;
constexpr int kTma = 1;
constexpr int kStages = 4;      // TMA ring depth (rows of look-ahead)
constexpr int kChunk = 36;      // doubles per row chunk: 33 needed, 16-B aligned start
constexpr int kStreams = 4;     // phi(j+1), m_x(j), m_y(j), rho(j)
constexpr int kStageBytes = kStreams * kChunk * 8;
constexpr int kTmaSmem = kSweepWarps * (kStages * kStageBytes + kStages * 8);

// One node of the m-update: returns the new flux and its increment, zero for
// absent components (solver_cp.cpp:39-54; absent components enter shrink as 0).
// kNB: branch-free p = 2 shrink (shrink2_nb: the restated fast paths of
// sqrt and division plus selects, bit-identical to shrink<1>) -- no
// divergent region per node, so the scheduler can interleave nodes.
// PN = 3: p = 2 in tolerance mode ("fast" numerics, streaming sweep kernels
// only): v = m - (mu ih)(pc - pr) by one FMA and shrink2_fast.
template <int PN, bool kNB = true>
__device__ __forceinline__ void node_flux(bool hx, bool hy, double pc, double pr, double pu,
                                          double mxo, double myo, double mu, double zt, double ih,
                                          double& ux, double& uy, double& dx, double& dy) {
    double vx, vy;
    if constexpr (PN == 3) {
        const double muih = mu * ih;  // loop-invariant, hoisted
        vx = hx ? __fma_rn(-muih, pc - pr, mxo) : 0.0;
        vy = hy ? __fma_rn(-muih, pc - pu, myo) : 0.0;
    } else {
        vx = hx ? mxo - mu * ((pc - pr) * ih) : 0.0;
        vy = hy ? myo - mu * ((pc - pu) * ih) : 0.0;
    }
    if constexpr (PN == 3) {
        shrink2_fast(vx, vy, mu, zt, ux, uy);
    } else if constexpr (kNB && PN == 1) {
        shrink2_nb(vx, vy, mu, zt, ux, uy);
    } else {
        shrink<PN>(vx, vy, mu, ux, uy);
    }
    dx = hx ? ux - mxo : 0.0;
    ux = hx ? ux : 0.0;
    dy = hy ? uy - myo : 0.0;
    uy = hy ? uy : 0.0;
}

// phi increment d = tau (div m^{k+1} + div dm - rho) (solver_cp.cpp:61-64,
// divergence_into's x-then-y order) and div dm for the residual cross term.
// PN = 3 (tolerance mode): tau ih ((x-diffs) + (y-diffs)) - tau rho by one FMA.
template <int PN>
__device__ __forceinline__ double phi_delta(double ux, double uxl, double uy, double uyb,
                                            double dx, double dxl, double dy, double dyb,
                                            double r, double ih, double tau, double& divd) {
    if constexpr (PN == 3) {
        const double dd = (dx - dxl) + (dy - dyb);
        const double dm = (ux - uxl) + (uy - uyb);
        divd = dd * ih;
        return __fma_rn(tau * ih, dm + dd, -(tau * r));
    } else {
        const double divm = (ux - uxl) * ih + (uy - uyb) * ih;
        divd = (dx - dxl) * ih + (dy - dyb) * ih;
        return tau * (divm + divd - r);
    }
}

// Everything a warp needs about its strip.
struct Strip {
    int i, j0, j1;
    int wpar;  // buffer parity written by this sweep
    bool in, hx, own;
    const double* phr;
    const double* mxr;
    const double* myr;
    const double* rho;
    double* phw;
    double* mxw;
    double* myw;
};

__device__ __forceinline__ Strip make_strip(const SweepArgs& a, int pair, int parity, int tile,
                                            int lane) {
    Strip s;
    const Layout& L = a.L;
    const int cx = tile % a.ncx;
    const int sy = tile / a.ncx;
    s.i = cx * kOwn - 1 + lane;
    s.j0 = a.jlo + sy * a.H;
    s.j1 = min(s.j0 + a.H, a.jhi);
    s.wpar = 1 - parity;
    double* pb = a.base + (long)pair * NSLOT * L.plane;
    s.phr = pb + (PHI0 + parity) * L.plane;
    s.mxr = pb + (MX0 + parity) * L.plane;
    s.myr = pb + (MY0 + parity) * L.plane;
    s.rho = pb + RHO * L.plane;
    s.phw = pb + (PHI0 + 1 - parity) * L.plane;
    s.mxw = pb + (MX0 + 1 - parity) * L.plane;
    s.myw = pb + (MY0 + 1 - parity) * L.plane;
    s.in = (s.i >= 0) && (s.i <= L.n);
    s.hx = (s.i >= 0) && (s.i < L.n);
    s.own = (lane > 0) && s.in;
    return s;
}

// y-flux (and its increment) of the row below the strip, recomputed once.
template <int PN>
__device__ __forceinline__ void below_row(const SweepArgs& a, const Strip& s, int lane,
                                          double& uyb, double& dyb) {
    uyb = 0.0;
    dyb = 0.0;
    if (s.j0 == 0) return;
    const Layout& L = a.L;
    const long o = L.at(s.i, s.j0 - 1);
    double pc = s.in ? __ldg(s.phr + o) : 0.0;
    double pu = s.in ? __ldg(s.phr + o + L.pitch) : 0.0;
    double pr = __shfl_down_sync(0xffffffffu, pc, 1);
    if (lane == 31) pr = s.hx ? __ldg(s.phr + o + 1) : 0.0;
    double mxo = s.hx ? __ldg(s.mxr + o) : 0.0;
    double myo = s.in ? __ldg(s.myr + o) : 0.0;
    double ux, uy, dx, dy;
    node_flux<PN>(s.hx, s.in, pc, pr, pu, mxo, myo, a.mu, a.zt, a.ih, ux, uy, dx, dy);
    uyb = uy;
    dyb = dy;
}

// One row of the march: m-update at (i, j), left-neighbour exchange,
// divergence of m^{k+1} and dm (grid.cpp:52-65 order), phi-update.
template <int PN>
__device__ __forceinline__ void row_update(const SweepArgs& a, const Strip& s, int j, long o,
                                           double pc, double pr, double pu, double mxo,
                                           double myo, double r, double& uyb, double& dyb,
                                           double& s_dm2, double& s_dp2, double& s_cr) {
    const bool hy = s.in && (j < a.L.n);
    const double ih = a.ih;
    double ux, uy, dx, dy;
    node_flux<PN>(s.hx, hy, pc, pr, pu, mxo, myo, a.mu, a.zt, ih, ux, uy, dx, dy);
    double uxl = __shfl_up_sync(0xffffffffu, ux, 1);
    double dxl = __shfl_up_sync(0xffffffffu, dx, 1);
    double divd;
    const double d = phi_delta<PN>(ux, uxl, uy, uyb, dx, dxl, dy, dyb, r, ih, a.tau, divd);
    if (s.own) {
        s.phw[o] = pc + d;
        if (s.hx) s.mxw[o] = ux;
        if (hy) s.myw[o] = uy;
        s_dm2 = __fma_rn(dy, dy, __fma_rn(dx, dx, s_dm2));
        s_dp2 = __fma_rn(d, d, s_dp2);
        s_cr = __fma_rn(d, divd, s_cr);
        if (a.up_base && j == a.jhi - 1) {  // top owned row -> upper neighbour's halo
            const long po = 32 + (long)(j - a.up_row0) * a.L.pitch + s.i;
            a.up_base[(PHI0 + s.wpar) * a.up_plane + po] = pc + d;
            if (s.hx) a.up_base[(MX0 + s.wpar) * a.up_plane + po] = ux;
            if (hy) a.up_base[(MY0 + s.wpar) * a.up_plane + po] = uy;
        }
        if (a.dn_base && j == a.jlo)  // first owned row's phi -> lower neighbour's halo
            a.dn_base[(PHI0 + s.wpar) * a.dn_plane + 32 + (long)(j - a.dn_row0) * a.L.pitch + s.i] =
                pc + d;
    }
    uyb = uy;
    dyb = dy;
}

// R^k from the three global sums, residual history, and the stop rule of
// solver_cp.cpp:128-136 (one thread).
template <bool kPlusCross = false>
__device__ __forceinline__ void finalize_pair(const SweepArgs& a, int pair, int parity,
                                              double sdm2, double sdp2, double scr) {
    PairCtl* ctl = a.ctl + pair;
    // Eq. 9 (CP, minus cross term) or Eq. 12 (PDHG, plus cross term)
    double fpr = kPlusCross ? a.h2 * (sdm2 / a.mu + sdp2 / a.tau + 2.0 * scr)
                            : a.h2 * (sdm2 / a.mu + sdp2 / a.tau - 2.0 * scr);
    long k = ctl->it;
    if (ctl->redo) fpr = ctl->rf[ctl->redo - 1];
    if (a.hist && k < a.hist_cap) a.hist[(long)pair * a.hist_cap + k] = fpr;
    ctl->it = k + 1;
    ctl->fpr = fpr;
    ctl->cur = 1 - parity;
    bool finite = isfinite(fpr);
    if (!finite) ctl->nonfinite = 1;
    if (ctl->redo) {
        // fix-up sweep after a multi-sweep launch stopped on its first (or
        // second) sweep: the pair is already counted as done
        ctl->redo -= 1;
    } else if (fpr < ctl->tol || k + 1 >= ctl->max_it || !finite) {
        ctl->done = 1;
        if (a.ndone) atomicAdd(a.ndone, 1);
    }
}

// Block + last-block reduction of the three residual sums; the last block of
// a pair finalises R^k and the stop flag (solver_cp.cpp:70, :128-136).
template <bool kPlusCross = false>
__device__ __forceinline__ void finish_sweep(const SweepArgs& a, int pair, int parity, int bid, int nblk,
                                             double s_dm2, double s_dp2, double s_cr) {
    // blocks are 256 threads, 1-D (sweeps) or 32 x 8 (node kernels)
    __shared__ double red[kSweepWarps][3];
    __shared__ bool is_last;
    const int tid = threadIdx.x + blockDim.x * threadIdx.y;
    const int nthr = blockDim.x * blockDim.y;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    s_dm2 = warp_sum(s_dm2);
    s_dp2 = warp_sum(s_dp2);
    s_cr = warp_sum(s_cr);
    if (lane == 0) {
        red[warp][0] = s_dm2;
        red[warp][1] = s_dp2;
        red[warp][2] = s_cr;
    }
    __syncthreads();
    double* part = a.partial + (long)pair * nblk * 3;
    if (tid == 0) {
        double t0 = 0.0, t1 = 0.0, t2 = 0.0;
#pragma unroll
        for (int w = 0; w < kSweepWarps; ++w) {
            t0 += red[w][0];
            t1 += red[w][1];
            t2 += red[w][2];
        }
        part[bid * 3 + 0] = t0;
        part[bid * 3 + 1] = t1;
        part[bid * 3 + 2] = t2;
        // peer transport: a block that stored halo rows into a neighbour
        // makes them visible at the neighbour's scope before the last block
        // signals arrival (blocks of the first / last strip row only)
        bool remote = false;
        if (a.mail && a.psys)
            for (int w = 0; w < kSweepWarps; ++w) {
                const int t = bid * kSweepWarps + w;
                if (t >= a.ntiles) break;
                const int sy = t / a.ncx;
                remote |= (sy == 0 && a.dn_base) || (sy == a.nsy - 1 && a.up_base);
            }
        if (remote) __threadfence_system();
        else __threadfence();
        unsigned t = atomicAdd(a.ticket + pair, 1u);
        is_last = (t == (unsigned)nblk - 1);
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();

    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
    for (int b = tid; b < nblk; b += nthr) {
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
    if (tid == 0) {
        double sdm2 = 0.0, sdp2 = 0.0, scr = 0.0;
        for (int w = 0; w < kSweepWarps; ++w) {
            sdm2 += red[w][0];
            sdp2 += red[w][1];
            scr += red[w][2];
        }
        a.ticket[pair] = 0u;
        if (a.mail) {
            // peer transport: post the slab's sums to every rank's mailbox
            // (slot [parity][prank]), then count one arrival on every rank
            for (int q = 0; q < a.pworld; ++q) {
                double* mb = a.mail[q] + ((long)parity * a.pworld + a.prank) * 3;
                mb[0] = sdm2;
                mb[1] = sdp2;
                mb[2] = scr;
            }
            if (a.psys) {
                __threadfence_system();
                for (int q = 0; q < a.pworld; ++q) atomicAdd_system(a.arrive[q], 1ull);
            } else {
                __threadfence();
                for (int q = 0; q < a.pworld; ++q) atomicAdd(a.arrive[q], 1ull);
            }
        } else if (a.red_out) {
            // row slab: publish this slab's sums; the cross-slab reduction
            // (device copy or NCCL all-reduce) then runs finalize_pair
            a.red_out[(long)pair * 3 + 0] = sdm2;
            a.red_out[(long)pair * 3 + 1] = sdp2;
            a.red_out[(long)pair * 3 + 2] = scr;
        } else {
            finalize_pair<kPlusCross>(a, pair, parity, sdm2, sdp2, scr);
        }
        __threadfence();
    }
}


// ------------------------------------------------------------ kTma engine
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "W1MG_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra W1MG_WAIT;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// TMA bulk copy global -> shared, completion counted on the mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// One 3-D tensor-map box (TMA tiled mode) into shared memory: coordinates
// (column, row, plane) of the box origin; completes on `bar` like bulk_g2s.
__device__ __forceinline__ void tmap_g2s_3d(void* dst, const void* tmap, int x, int y, int z,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(smem_u32(dst)), "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

template <int PN>
__global__ void __launch_bounds__(kSweepWarps * 32, 3)
cp_sweep_tma_kernel(const SweepArgs a, const int parity_arg) {
    const int pair = sweep_pair(a);
    int parity;
    if (pair < 0 || !sweep_gate(a.ctl + pair, parity_arg, parity)) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    // warp index broadcast from lane 0: the compiler then keeps every TMA
    // operand derived from it in uniform registers (no per-copy R2UR loop)
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
    const int tile = blockIdx.x * kSweepWarps + warp;
    // per-warp ring: kStages x [kStreams][kChunk] doubles, then kStages mbarriers
    double* ring = reinterpret_cast<double*>(smem_raw) + (size_t)warp * kStages * kStreams * kChunk;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + kSweepWarps * kStages * kStageBytes) +
                     warp * kStages;
    double s_dm2 = 0.0, s_dp2 = 0.0, s_cr = 0.0;

    if (tile < a.ntiles) {
        const Strip s = make_strip(a, pair, parity, tile, lane);
        const Layout L = a.L;
        const int P = L.pitch;
        // chunk start: column i of lane 0 rounded down to even (16-B aligned;
        // rows are 256-B aligned and the front pad keeps column -2 in bounds)
        const int ilo = (tile % a.ncx) * kOwn - 1;  // column of lane 0 (warp-uniform)
        const int a0 = ilo & ~1;
        const int sh = ilo - a0;                // 0 or 1
        const long c0 = L.at(a0, 0);

        if (lane == 0) {
#pragma unroll
            for (int t = 0; t < kStages; ++t) mbar_init(&bars[t], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        auto issue = [&](int st, int row) {
            double* dst = ring + st * kStreams * kChunk;
            const long orow = c0 + (long)row * P;
            mbar_expect_tx(&bars[st], kStageBytes);
            bulk_g2s(dst + 0 * kChunk, s.phr + orow + P, kChunk * 8, &bars[st]);
            bulk_g2s(dst + 1 * kChunk, s.mxr + orow, kChunk * 8, &bars[st]);
            bulk_g2s(dst + 2 * kChunk, s.myr + orow, kChunk * 8, &bars[st]);
            bulk_g2s(dst + 3 * kChunk, s.rho + orow, kChunk * 8, &bars[st]);
        };
        const int rows = s.j1 - s.j0;
        if (lane == 0) {
            for (int t = 0; t < kStages && t < rows; ++t) issue(t, s.j0 + t);
        }

        double uyb, dyb;
        below_row<PN>(a, s, lane, uyb, dyb);
        long o = L.at(s.i, s.j0);
        double pc = s.in ? __ldg(s.phr + o) : 0.0;
        double pr = __shfl_down_sync(0xffffffffu, pc, 1);
        if (lane == 31) pr = s.hx ? __ldg(s.phr + o + 1) : 0.0;

        for (int t = 0; t < rows; ++t, o += P) {
            const int j = s.j0 + t;
            const int st = t % kStages;
            mbar_wait(&bars[st], (uint32_t)((t / kStages) & 1));
            const double* c = ring + st * kStreams * kChunk + sh + lane;
            const bool hy = s.in && (j < L.n);
            const double pu = hy ? c[0] : 0.0;
            const double pur = (s.hx && j < L.n) ? c[1] : 0.0;
            const double mxo = s.hx ? c[kChunk] : 0.0;
            const double myo = hy ? c[2 * kChunk] : 0.0;
            const double r = s.in ? c[3 * kChunk] : 0.0;
            __syncwarp();
            if (lane == 0 && t + kStages < rows) {
                // all lanes have read the stage: hand it back to the async proxy
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(st, j + kStages);
            }
            row_update<PN>(a, s, j, o, pc, pr, pu, mxo, myo, r, uyb, dyb, s_dm2, s_dp2, s_cr);
            pr = pur;
            pc = pu;
        }
    }
    finish_sweep(a, pair, parity, blockIdx.x, gridDim.x, s_dm2, s_dp2, s_cr);
}

}  // namespace w1mg_dev

namespace w1mg_dev {

// ------------------------------------------------------- resident engine
// Small levels (6 (n+1)^2 doubles <= kResidentMaxBytes): one CTA per pair
// keeps phi, rho, m and dm in shared memory and runs every sweep of the
// level in ONE launch, deciding the stop rule itself after each sweep.
// Two phases per sweep separated by a block barrier:
//   A: m-update of every node (reads phi^k, writes m^{k+1} in place + dm)
//   B: phi-update of every node (reads m^{k+1}, dm of the node and its
//      left/lower neighbours, rho) -- same arithmetic as row_update.
// The state after the last sweep is written back to buffer 0 (ctl.cur = 0).
constexpr int kResidentThreads = 512;
constexpr int kResidentMaxBytes = 6 * 65 * 65 * 8;  // n <= 64

__host__ __device__ constexpr long resident_bytes(int n) {
    return 6L * (n + 1) * (n + 1) * 8;
}

template <int PN>
__global__ void __launch_bounds__(kResidentThreads, 1)
cp_resident_kernel(const SweepArgs a) {
    const int pair = blockIdx.x;
    PairCtl* ctl = a.ctl + pair;
    if (ctl->done) return;
    extern __shared__ __align__(16) double sm[];
    const Layout L = a.L;
    const int n = L.n;
    const int W = n + 1;
    const int V = W * W;
    double* phi = sm;
    double* rho = sm + V;
    double* mx = sm + 2 * V;
    double* my = sm + 3 * V;
    double* ddx = sm + 4 * V;
    double* ddy = sm + 5 * V;
    const int T = blockDim.x;
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int di = T % W, dj = T / W;  // incremental (i, j) of k += T
    const int i0 = tid % W, j0 = tid / W;

    double* pb = a.base + (long)pair * NSLOT * L.plane;
    const int cur = ctl->cur;
    {
        const double* gp = pb + (PHI0 + cur) * L.plane;
        const double* gx = pb + (MX0 + cur) * L.plane;
        const double* gy = pb + (MY0 + cur) * L.plane;
        const double* gr = pb + RHO * L.plane;
        int i = i0, j = j0;
        for (int k = tid; k < V; k += T) {
            const long o = L.at(i, j);
            phi[k] = gp[o];
            rho[k] = gr[o];
            mx[k] = (i < n) ? gx[o] : 0.0;
            my[k] = (j < n) ? gy[o] : 0.0;
            i += di;
            j += dj;
            if (i >= W) { i -= W; ++j; }
        }
    }
    __shared__ double red[kResidentThreads / 32][3];
    __shared__ int stop;
    const double mu = a.mu, zt = a.zt, tau = a.tau, ih = a.ih;
    long it = ctl->it;
    const long max_it = ctl->max_it;
    const double tol = ctl->tol;
    __syncthreads();

    for (;;) {
        double s_dm2 = 0.0, s_dp2 = 0.0, s_cr = 0.0;
        {  // phase A: flux
            int i = i0, j = j0;
            for (int k = tid; k < V; k += T) {
                const bool hx = i < n, hy = j < n;
                const double pc = phi[k];
                const double pr = hx ? phi[k + 1] : 0.0;
                const double pu = hy ? phi[k + W] : 0.0;
                double ux, uy, dx, dy;
                node_flux<PN>(hx, hy, pc, pr, pu, mx[k], my[k], mu, zt, ih, ux, uy, dx, dy);
                mx[k] = ux;
                my[k] = uy;
                ddx[k] = dx;
                ddy[k] = dy;
                s_dm2 = __fma_rn(dy, dy, __fma_rn(dx, dx, s_dm2));
                i += di;
                j += dj;
                if (i >= W) { i -= W; ++j; }
            }
        }
        __syncthreads();
        {  // phase B: potential (divergence_into order, grid.cpp:52-65)
            int i = i0, j = j0;
            for (int k = tid; k < V; k += T) {
                const double uxl = (i > 0) ? mx[k - 1] : 0.0;
                const double dxl = (i > 0) ? ddx[k - 1] : 0.0;
                const double uyb = (j > 0) ? my[k - W] : 0.0;
                const double dyb = (j > 0) ? ddy[k - W] : 0.0;
                const double divm = (mx[k] - uxl) * ih + (my[k] - uyb) * ih;
                const double divd = (ddx[k] - dxl) * ih + (ddy[k] - dyb) * ih;
                const double d = tau * (divm + divd - rho[k]);
                phi[k] = phi[k] + d;
                s_dp2 = __fma_rn(d, d, s_dp2);
                s_cr = __fma_rn(d, divd, s_cr);
                i += di;
                j += dj;
                if (i >= W) { i -= W; ++j; }
            }
        }
        s_dm2 = warp_sum(s_dm2);
        s_dp2 = warp_sum(s_dp2);
        s_cr = warp_sum(s_cr);
        if (lane == 0) {
            red[warp][0] = s_dm2;
            red[warp][1] = s_dp2;
            red[warp][2] = s_cr;
        }
        __syncthreads();
        if (tid == 0) {
            double sdm2 = 0.0, sdp2 = 0.0, scr = 0.0;
            for (int w = 0; w < T / 32; ++w) {
                sdm2 += red[w][0];
                sdp2 += red[w][1];
                scr += red[w][2];
            }
            const double fpr = a.h2 * (sdm2 / mu + sdp2 / tau - 2.0 * scr);
            if (a.hist && it < a.hist_cap) a.hist[(long)pair * a.hist_cap + it] = fpr;
            ++it;
            const bool finite = isfinite(fpr);
            const bool done = (fpr < tol) || (it >= max_it) || !finite;
            stop = done;
            ctl->fpr = fpr;
            if (!finite) ctl->nonfinite = 1;
        }
        __syncthreads();
        if (stop) break;
    }
    {  // write the final state back to buffer 0
        double* gp = pb + PHI0 * L.plane;
        double* gx = pb + MX0 * L.plane;
        double* gy = pb + MY0 * L.plane;
        int i = i0, j = j0;
        for (int k = tid; k < V; k += T) {
            const long o = L.at(i, j);
            gp[o] = phi[k];
            if (i < n) gx[o] = mx[k];
            if (j < n) gy[o] = my[k];
            i += di;
            j += dj;
            if (i >= W) { i -= W; ++j; }
        }
    }
    if (tid == 0) {
        ctl->it = it;
        ctl->cur = 0;
        ctl->done = 1;
        atomicAdd(a.ndone, 1);
    }
}

}  // namespace w1mg_dev
