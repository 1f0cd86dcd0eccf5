// tile_kernels.cuh -- level-persistent tile engine: a whole CP level of one
// pair (or a few) in ONE launch, state resident in shared memory, neighbour
// halos through L2, no grid-wide barrier on the data path.
//
// A one-pair level of n = 96..512 is too small to fill the GPU with the
// streaming kernels (a 512^2 sweep is 14.7 MB, ~2 us of HBM time, but a
// launch of it costs ~7 us of ramp, tail and reduction), and a cooperative
// grid barrier per sweep costs as much.  Here the level is cut into
// TR x TC tiles, one CTA per tile (one per SM, co-resident by a cooperative
// launch), each holding its tile of phi, m, dm and rho in shared memory with
// a one-node halo ring.  Per sweep k:
//
//   1. wait until the six neighbours that feed the halo (left, right, below,
//      above, above-left, below-right) have finished sweep k-1 (per-tile step
//      flags, acquire loads), read their published edges (phi, m) from L2;
//   2. phase A: the m-update (node_flux) of the owned nodes and, recomputed,
//      of the left halo column and the bottom halo row (their fluxes enter
//      the divergence of the first owned column / row);
//   3. phase B: the phi-update in the reference's divergence order;
//   4. publish the edges of the new state (double-buffered by step parity),
//      post the tile's three residual sums for sweep k, release the step flag.
//
// The stop rule (solver_cp.cpp:128-136) needs R^k, a sum over all tiles.  A
// controller CTA per pair reduces the posted partials in a fixed order, writes
// the residual history and the decision for every sweep; tiles read the
// decision of sweep k - kTileLag at the start of sweep k, so the reduction is
// off the critical path.  When sweep s is found to stop, every tile has run
// exactly kTileLag sweeps past it; all tiles restore the checkpoint (written
// every kTileCk sweeps into the level's two ping-pong buffers) at or below
// s + 1 and replay to s + 1 -- the arithmetic is deterministic, so the final
// state is bit-identical to stopping on time.  Node arithmetic is node_flux /
// row_update's, so fields are bit-identical to the reference.
//
// Ordering: edge records of step q live in buffer q & 1; a tile overwrites
// buffer q & 1 at step q + 2 only after every reader of step q (its
// neighbours, which it waits for) posted step q + 1.  Residual slots are
// reused after kTileSlots sweeps, by which time the controller has consumed
// them (tiles wait for decision k - kTileLag, kTileSlots > kTileLag).
#pragma once

#include <type_traits>

#include "cp_kernels.cuh"

namespace w1mg_dev {

constexpr int kTileThreads = 512;
constexpr int kTileWarps = kTileThreads / 32;
constexpr int kTileLag = 16;             // decisions are read this many sweeps late
constexpr int kTileSlots = 2 * kTileLag; // residual ring
constexpr int kTileCk = kTileLag;        // checkpoint period (>= lag: the restored slot is intact)
constexpr int kTileFlagStride = 32;      // one 128-B line per step flag
constexpr int kTileSecs = 8;             // edge sections, see below
// edge sections of a tile's record: phi of the left/right columns and the
// bottom/top rows, m_x, m_y of the right column and of the top row
enum TileSec { E_PHI_L = 0, E_PHI_R, E_PHI_B, E_PHI_T, E_MX_R, E_MY_R, E_MX_T, E_MY_T };

struct TileArgs {
    SweepArgs a;           // level: base, L, mu, tau, ih, h2, ctl, hist, ndone
    int TR, TC;            // tiles per pair (rows x columns of tiles)
    int LW, LH;            // shared-memory pitch / rows (largest tile + halo ring)
    int ES;                // edge section stride (largest tile side)
    int LCAP;              // capacity of each border list (ints)
    double* edges;         // [pairs][2][T][kTileSecs][ES]
    unsigned* flags;       // [pairs][T][kTileFlagStride] steps completed
    double* part;          // [pairs][kTileSlots][T][3]
    unsigned* cnt;         // [pairs][kTileSlots] tiles posted
    double* dec;           // [pairs][kTileSlots][2] residual, stop
    unsigned long long* dseq;  // [pairs][kTileSlots] 2 (decided sweep + 1) + stop
    int* err;              // set when a wait times out (then the kernel traps)
    long long* dbg;        // optional per-step clock64 stamps of tile 0 (diagnostics)
};
constexpr int kTileDbgSteps = 256;
constexpr int kTileDbgPts = 8;

__host__ __device__ inline int tile_lo(int N1, int parts, int t) {
    return (int)((long)N1 * t / parts);
}
__host__ inline int tile_list_cap(int LW, int LH) { return 2 * LW + 2 * LH + 8; }
__host__ inline long tile_smem_bytes(int LW, int LH) {
    return 6L * LW * LH * 8 + 2L * tile_list_cap(LW, LH) * 4;
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// bounded spin: a lost peer must fail the launch, not hang the GPU
__device__ __noinline__ void tile_timeout(int* err) {
    atomicExch(err, 1);
    __trap();
}
constexpr unsigned long long kTileTimeoutNs = 20ull * 1000 * 1000 * 1000;

// relaxed polls (an acquire load would invalidate L1 on every iteration);
// the caller fences once afterwards.  Timeout checked every 1024 polls.
__device__ __forceinline__ void spin_geq(const unsigned* p, unsigned target, int* err) {
    unsigned long long t0 = 0;
    for (unsigned it = 0;; ++it) {
        unsigned v;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
        if (v >= target) return;
        if ((it & 1023u) == 0) {
            const unsigned long long now = gtimer();
            if (it == 0) t0 = now;
            else if (now - t0 > kTileTimeoutNs) tile_timeout(err);
        }
    }
}
// waits for (*p >> 1) == tag and returns *p
__device__ __forceinline__ unsigned long long spin_tag64(const unsigned long long* p,
                                                         unsigned long long tag, int* err) {
    unsigned long long t0 = 0;
    for (unsigned it = 0;; ++it) {
        unsigned long long v;
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
        if ((v >> 1) == tag) return v;
        if ((it & 1023u) == 0) {
            const unsigned long long now = gtimer();
            if (it == 0) t0 = now;
            else if (now - t0 > kTileTimeoutNs) tile_timeout(err);
        }
    }
}

// Controller of one pair: reduces sweep s's partials once every tile posted
// them, records R^s, decides the stop (solver_cp.cpp:128-136), publishes it.
// Warp w handles sweeps s = k0 + w (mod kTileWarps), so up to kTileWarps
// decisions are in flight; kTileWarps == kTileLag makes "decision k - lag is
// out" imply that the same warp finished sweep k - 2 lag, i.e. the residual
// slot a tile reuses at sweep k (k - kTileSlots) has been consumed.
static_assert(kTileWarps == kTileLag && kTileSlots == 2 * kTileLag, "controller pipelining");
__device__ void tile_controller(const TileArgs& t, int pair, int T, long k0) {
    __shared__ long long c_stop;  // earliest stopping sweep found so far
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) c_stop = 0x7fffffffffffffffll;
    __syncthreads();
    const SweepArgs& a = t.a;
    PairCtl* ctl = a.ctl + pair;
    const long max_it = ctl->max_it;
    const double tol = ctl->tol;
    volatile long long* vstop = &c_stop;
    for (long s = k0 + warp;; s += kTileWarps) {
        const int slot = (int)(s % kTileSlots);
        unsigned* cnt = t.cnt + (long)pair * kTileSlots + slot;
        int go = 0;
        if (lane == 0) {
            unsigned long long t0 = 0;
            for (unsigned it = 0;; ++it) {
                if (*vstop < s) break;  // a tile never posts sweeps past the stop + lag
                unsigned v;
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
                if (v >= (unsigned)T) {
                    go = 1;
                    break;
                }
                if ((it & 1023u) == 0) {
                    const unsigned long long now = gtimer();
                    if (it == 0) t0 = now;
                    else if (now - t0 > kTileTimeoutNs) tile_timeout(t.err);
                }
            }
        }
        if (!__shfl_sync(0xffffffffu, go, 0)) return;
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        const double* p = t.part + ((long)pair * kTileSlots + slot) * T * 3;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0;
        for (int b = lane; b < T; b += 32) {
            s0 += __ldcg(p + b * 3 + 0);
            s1 += __ldcg(p + b * 3 + 1);
            s2 += __ldcg(p + b * 3 + 2);
        }
        s0 = warp_sum(s0);
        s1 = warp_sum(s1);
        s2 = warp_sum(s2);
        int stop = 0;
        if (lane == 0) {
            const double fpr = a.h2 * (s0 / a.mu + s1 / a.tau - 2.0 * s2);  // Eq. 9
            const bool finite = isfinite(fpr);
            stop = (fpr < tol || s + 1 >= max_it || !finite) ? 1 : 0;
            if (a.hist && s < a.hist_cap) a.hist[(long)pair * a.hist_cap + s] = fpr;
            *cnt = 0u;
            double* d = t.dec + ((long)pair * kTileSlots + slot) * 2;
            d[0] = fpr;
            d[1] = stop ? 1.0 : 0.0;
            asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(t.dseq + (long)pair * kTileSlots + slot),
                         "l"((unsigned long long)(2 * (s + 1) + stop))
                         : "memory");
            if (stop) atomicMin((long long*)&c_stop, (long long)s);
        }
        if (__shfl_sync(0xffffffffu, stop, 0)) return;
    }
}

template <int PN>
__global__ void __launch_bounds__(kTileThreads, 1) cp_tile_kernel(const TileArgs t) {
    const int T = t.TR * t.TC;
    const int pair = blockIdx.x / (T + 1);
    const int tile = blockIdx.x % (T + 1);
    const SweepArgs& a = t.a;
    PairCtl* ctl = a.ctl + pair;
    if (*(volatile int*)&ctl->done) return;  // uniform: nothing writes ctl before the end
    const long k0 = ctl->it;
    if (tile == T) {  // uniform per block
        tile_controller(t, pair, T, k0);
        return;
    }
    extern __shared__ __align__(16) double sm[];
    __shared__ double wred[kTileWarps][3];
    __shared__ int s_stop;
    __shared__ long s_stop_at;
    __shared__ double s_fpr;

    const Layout L = a.L;
    const int n = L.n;
    const int tr = tile / t.TC, tc = tile % t.TC;
    const int i0 = tile_lo(n + 1, t.TC, tc), j0 = tile_lo(n + 1, t.TR, tr);
    const int w = tile_lo(n + 1, t.TC, tc + 1) - i0;
    const int h = tile_lo(n + 1, t.TR, tr + 1) - j0;
    const int LW = t.LW;
    const int S = LW * t.LH;
    double* phi = sm;
    double* mx = sm + S;
    double* my = sm + 2 * S;
    double* ddx = sm + 3 * S;
    double* ddy = sm + 4 * S;
    double* rho = sm + 5 * S;
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const double mu = a.mu, zt = a.zt, tau = a.tau, ih = a.ih;

    // neighbours (tile index within the pair, -1 = none)
    const int nL = tc > 0 ? tile - 1 : -1;
    const int nR = tc + 1 < t.TC ? tile + 1 : -1;
    const int nD = tr > 0 ? tile - t.TC : -1;
    const int nU = tr + 1 < t.TR ? tile + t.TC : -1;
    const int nUL = (tr + 1 < t.TR && tc > 0) ? tile + t.TC - 1 : -1;
    const int nDR = (tr > 0 && tc + 1 < t.TC) ? tile - t.TC + 1 : -1;
    const int wL = tc > 0 ? i0 - tile_lo(n + 1, t.TC, tc - 1) : 0;  // width of the left tile column

    const long recs = (long)T * kTileSecs * t.ES;  // doubles per step buffer of one pair
    double* ebase = t.edges + (long)pair * 2 * recs;
    auto rec = [&](int buf, int who, int sec) -> double* {
        return ebase + buf * recs + ((long)who * kTileSecs + sec) * t.ES;
    };
    unsigned* flags = t.flags + (long)pair * T * kTileFlagStride;
    double* pb = a.base + (long)pair * NSLOT * L.plane;

    // whole tile + halo ring from the level buffer planes of parity p
    auto load_state = [&](int p) {
        const double* gp = pb + (PHI0 + p) * L.plane;
        const double* gx = pb + (MX0 + p) * L.plane;
        const double* gy = pb + (MY0 + p) * L.plane;
        const double* gr = pb + RHO * L.plane;
        const int W2 = w + 2, cnt = W2 * (h + 2);
        for (int q = tid; q < cnt; q += kTileThreads) {
            const int li = q % W2, lj = q / W2;
            const int i = i0 - 1 + li, j = j0 - 1 + lj;
            const bool in = i >= 0 && i <= n && j >= 0 && j <= n;
            const long o = in ? L.at(i, j) : 0;
            const int k = lj * LW + li;
            phi[k] = in ? __ldcg(gp + o) : 0.0;
            mx[k] = (in && i < n) ? __ldcg(gx + o) : 0.0;
            my[k] = (in && j < n) ? __ldcg(gy + o) : 0.0;
            ddx[k] = 0.0;
            ddy[k] = 0.0;
            rho[k] = (in && li >= 1 && li <= w && lj >= 1 && lj <= h) ? __ldg(gr + o) : 0.0;
        }
    };
    // owned phi, m -> planes of parity p (checkpoint / final state)
    auto store_state = [&](int p) {
        double* gp = pb + (PHI0 + p) * L.plane;
        double* gx = pb + (MX0 + p) * L.plane;
        double* gy = pb + (MY0 + p) * L.plane;
        for (int q = tid; q < w * h; q += kTileThreads) {
            const int li = 1 + q % w, lj = 1 + q / w;
            const int i = i0 - 1 + li, j = j0 - 1 + lj;
            const long o = L.at(i, j);
            const int k = lj * LW + li;
            __stcg(gp + o, phi[k]);
            if (i < n) __stcg(gx + o, mx[k]);
            if (j < n) __stcg(gy + o, my[k]);
        }
    };
    // halo ring from the neighbours' records of step buffer `buf`
    auto load_halo = [&](int buf) {
        const int cnt = 4 * h + 4 * w + 2;
        for (int q = tid; q < cnt; q += kTileThreads) {
            if (q < 3 * h) {  // left column: phi, m_x, m_y of the left tile's right column
                if (nL < 0) continue;
                const int f = q / h, r = q % h;
                const double v = __ldcg(rec(buf, nL, f == 0 ? E_PHI_R : (f == 1 ? E_MX_R : E_MY_R)) + r);
                double* dst = f == 0 ? phi : (f == 1 ? mx : my);
                dst[(1 + r) * LW] = v;
            } else if (q < 3 * h + 3 * w) {  // bottom row from the lower tile's top row
                if (nD < 0) continue;
                const int q2 = q - 3 * h;
                const int f = q2 / w, r = q2 % w;
                const double v = __ldcg(rec(buf, nD, f == 0 ? E_PHI_T : (f == 1 ? E_MX_T : E_MY_T)) + r);
                double* dst = f == 0 ? phi : (f == 1 ? mx : my);
                dst[1 + r] = v;
            } else if (q < 4 * h + 3 * w) {  // right column phi
                if (nR < 0) continue;
                const int r = q - 3 * h - 3 * w;
                phi[(1 + r) * LW + w + 1] = __ldcg(rec(buf, nR, E_PHI_L) + r);
            } else if (q < 4 * h + 4 * w) {  // top row phi
                if (nU < 0) continue;
                const int r = q - 4 * h - 3 * w;
                phi[(h + 1) * LW + 1 + r] = __ldcg(rec(buf, nU, E_PHI_B) + r);
            } else if (q == 4 * h + 4 * w) {  // above-left corner: that tile's bottom-right node
                if (nUL >= 0) phi[(h + 1) * LW] = __ldcg(rec(buf, nUL, E_PHI_B) + wL - 1);
            } else {  // below-right corner: that tile's top-left node
                if (nDR >= 0) phi[w + 1] = __ldcg(rec(buf, nDR, E_PHI_T));
            }
        }
    };

    long k = k0;      // logical sweep index (state k in shared memory)
    unsigned step = 0;  // steps executed (monotonic, also across a replay)
    bool replay = false;
    long target = -1;  // replay: stop at state target
    double fin_fpr = 0.0;
    long stop_at = -1;

    load_state(ctl->cur);
    if (tid == 0) s_stop = 0;
    __syncthreads();
    if (ctl->cur != 0) store_state(0);  // checkpoint of state k0 (slot 0)

    // Border lists (built once, in order, by thread 0): A-border = nodes of
    // phase A that need the halo (right column, top row) or are the
    // recomputed halo (left column, bottom row); B-border = owned nodes whose
    // phi is published (first / last column and row).  The interior parts
    // of both phases need no halo: A-interior runs before the wait for the
    // neighbours, B-interior after this tile's step flag is released, so
    // both overlap the inter-SM flag latency.
    int* listA = reinterpret_cast<int*>(sm + 6 * S);
    int* listB = listA + t.LCAP;
    __shared__ int s_na, s_nb;
    if (tid == 0) {
        int na = 0, nb = 0;
        for (int lj = 0; lj <= h; ++lj)
            for (int li = 0; li <= w; ++li) {
                if (li == 0 && lj == 0) continue;
                const bool intA = li >= 1 && li <= w - 1 && lj >= 1 && lj <= h - 1;
                if (!intA && i0 - 1 + li >= 0 && j0 - 1 + lj >= 0) listA[na++] = li | (lj << 16);
                if (li >= 1 && lj >= 1) {
                    const bool intB = li >= 2 && li <= w - 1 && lj >= 2 && lj <= h - 1;
                    if (!intB) listB[nb++] = li | (lj << 16);
                }
            }
        s_na = na;
        s_nb = nb;
    }
    __syncthreads();
    const int nAb = s_na, nBb = s_nb;
    const int wA = w - 1, nAi = (w >= 2 && h >= 2) ? (w - 1) * (h - 1) : 0;
    const int wB = w - 2, nBi = (w >= 3 && h >= 3) ? (w - 2) * (h - 2) : 0;

    // phase A at local node (li, lj): m-update (node_flux), m records
    auto nodeA = [&](int li, int lj, int bufw, double& s_dm2) {
        const int i = i0 - 1 + li, j = j0 - 1 + lj;
        const int kk = lj * LW + li;
        const bool hx = i < n, hy = j < n;
        const double pc = phi[kk];
        const double pr = hx ? phi[kk + 1] : 0.0;
        const double pu = hy ? phi[kk + LW] : 0.0;
        double ux, uy, dx, dy;
        node_flux<PN>(hx, hy, pc, pr, pu, mx[kk], my[kk], mu, zt, ih, ux, uy, dx, dy);
        mx[kk] = ux;
        my[kk] = uy;
        ddx[kk] = dx;
        ddy[kk] = dy;
        if (li >= 1 && lj >= 1) {
            s_dm2 = __fma_rn(dy, dy, __fma_rn(dx, dx, s_dm2));
            if (li == w) {
                rec(bufw, tile, E_MX_R)[lj - 1] = ux;
                rec(bufw, tile, E_MY_R)[lj - 1] = uy;
            }
            if (lj == h) {
                rec(bufw, tile, E_MX_T)[li - 1] = ux;
                rec(bufw, tile, E_MY_T)[li - 1] = uy;
            }
        }
    };
    // phase B at owned local node (li, lj): row_update's divergence order
    auto nodeB = [&](int li, int lj, int bufw, double& s_dp2, double& s_cr) {
        const int kk = lj * LW + li;
        const double divm = (mx[kk] - mx[kk - 1]) * ih + (my[kk] - my[kk - LW]) * ih;
        const double divd = (ddx[kk] - ddx[kk - 1]) * ih + (ddy[kk] - ddy[kk - LW]) * ih;
        const double d = tau * (divm + divd - rho[kk]);
        const double f = phi[kk] + d;
        phi[kk] = f;
        s_dp2 = __fma_rn(d, d, s_dp2);
        s_cr = __fma_rn(d, divd, s_cr);
        if (li == 1) rec(bufw, tile, E_PHI_L)[lj - 1] = f;
        if (li == w) rec(bufw, tile, E_PHI_R)[lj - 1] = f;
        if (lj == 1) rec(bufw, tile, E_PHI_B)[li - 1] = f;
        if (lj == h) rec(bufw, tile, E_PHI_T)[li - 1] = f;
    };
    // warp 0 lanes 0..5 wait for the neighbours' step flags, lane 6 for the
    // decision of sweep kd.  Relaxed polls without an acquire fence: every
    // load that consumes a neighbour's records is an L2 (.cg, gpu-scope
    // strong) load issued only after the poll loop has exited (control
    // dependence), and the producer released the flag after its records
    // reached L2 (st.release), so the records are observed no earlier than
    // the flag.  (A fence here costs ~600 cycles per sweep, measured.)
    auto wait_neighbours = [&](unsigned target_step, long kd) {
        int nb = -1;
        if (lane == 0) nb = nL;
        else if (lane == 1) nb = nR;
        else if (lane == 2) nb = nD;
        else if (lane == 3) nb = nU;
        else if (lane == 4) nb = nUL;
        else if (lane == 5) nb = nDR;
        if (nb >= 0) spin_geq(flags + (long)nb * kTileFlagStride, target_step, t.err);
        if (lane == 6 && kd >= k0) {
            const int slot = (int)(kd % kTileSlots);
            const unsigned long long v =
                spin_tag64(t.dseq + (long)pair * kTileSlots + slot, (unsigned long long)(kd + 1), t.err);
            if (v & 1ull) {
                s_stop = 1;
                s_stop_at = kd;
                s_fpr = __ldcg(t.dec + ((long)pair * kTileSlots + slot) * 2);
            }
        }
        __syncwarp();
    };

    // diagnostics (W1MG_TILE_DEBUG): per-tile cycles spent in each segment
    // of steps 8..135, thread 0
    long long dbg_acc[kTileDbgPts] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long dbg_last = clock64();
#define STAMP(pt)                                                    \
    if (t.dbg && tid == 0) {                                         \
        const long long now_ = clock64();                            \
        if (step >= 8 && step < 136) dbg_acc[pt] += now_ - dbg_last; \
        dbg_last = now_;                                             \
    }

    bool have_halo = true;  // the halo of state k is in shared memory (after a load)
    for (;;) {
        if (replay && k >= target) break;
        STAMP(0);
        const int bufw = (int)((step + 1) & 1);  // record buffer of the state this step produces
        double s_dm2 = 0.0, s_dp2 = 0.0, s_cr = 0.0;
        // ---- A-interior (no halo needed)
        for (int q = tid; q < nAi; q += kTileThreads) nodeA(1 + q % wA, 1 + q / wA, bufw, s_dm2);
        STAMP(1);
        if (!have_halo) {
            // ---- neighbours done with the previous step; decision of sweep k - lag
            if (warp == 0) wait_neighbours(step, replay ? k0 - 1 : k - kTileLag);
            __syncthreads();
            STAMP(2);
            if (!replay && s_stop) {
                // sweep s = s_stop_at stopped: restore the checkpoint at or
                // below s + 1 and replay to exactly s + 1 (every tile does
                // the same); this step's A-interior is discarded
                stop_at = s_stop_at;
                fin_fpr = s_fpr;
                target = stop_at + 1;
                const long c = k0 + ((target - k0) / kTileCk) * kTileCk;
                load_state((int)(((c - k0) / kTileCk) & 1));
                k = c;
                replay = true;
                have_halo = true;
                __syncthreads();
                continue;
            }
            load_halo((int)(step & 1));
        }
        __syncthreads();
        STAMP(3);
        // ---- A-border, then B-border (the published edges)
        for (int q = tid; q < nAb; q += kTileThreads) nodeA(listA[q] & 0xffff, listA[q] >> 16, bufw, s_dm2);
        __syncthreads();
        for (int q = tid; q < nBb; q += kTileThreads)
            nodeB(listB[q] & 0xffff, listB[q] >> 16, bufw, s_dp2, s_cr);
        __syncthreads();
        // ---- release: the edge records of this step (every thread's,
        // ordered by the barrier) before the flag
        if (tid == 0)
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + (long)tile * kTileFlagStride),
                         "r"(step + 1)
                         : "memory");
        STAMP(4);
        // ---- B-interior, overlapping the flag's way to the neighbours
        for (int q = tid; q < nBi; q += kTileThreads) nodeB(2 + q % wB, 2 + q / wB, bufw, s_dp2, s_cr);
        s_dm2 = warp_sum(s_dm2);
        s_dp2 = warp_sum(s_dp2);
        s_cr = warp_sum(s_cr);
        if (lane == 0) {
            wred[warp][0] = s_dm2;
            wred[warp][1] = s_dp2;
            wred[warp][2] = s_cr;
        }
        __syncthreads();
        ++k;
        ++step;
        have_halo = false;
        if (!replay && ((k - k0) % kTileCk) == 0) {
            store_state((int)(((k - k0) / kTileCk) & 1));
            __syncthreads();
        }
        // ---- residual partials of sweep k-1 (warp 1, off the critical path)
        if (tid == 32 && !replay) {
            const int slot = (int)((k - 1) % kTileSlots);
            double t0 = 0.0, t1 = 0.0, t2 = 0.0;
            for (int q = 0; q < kTileWarps; ++q) {
                t0 += wred[q][0];
                t1 += wred[q][1];
                t2 += wred[q][2];
            }
            double* p = t.part + (((long)pair * kTileSlots + slot) * T + tile) * 3;
            p[0] = t0;
            p[1] = t1;
            p[2] = t2;
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(t.cnt + (long)pair * kTileSlots + slot)
                         : "memory");
        }
        STAMP(5);
    }
    // every neighbour finished its replay (and so its checkpoint reads)
    // before the final state goes into buffer 0
    if (warp == 0) wait_neighbours(step, k0 - 1);
    __syncthreads();
    store_state(0);
    if (t.dbg && tid == 0)
        for (int q = 0; q < kTileDbgPts; ++q) t.dbg[tile * kTileDbgPts + q] = dbg_acc[q];
#undef STAMP
    if (tile == 0 && tid == 0) {
        ctl->it = stop_at + 1;
        ctl->fpr = fin_fpr;
        ctl->cur = 0;
        if (!isfinite(fin_fpr)) ctl->nonfinite = 1;
        ctl->done = 1;
        atomicAdd(a.ndone, 1);
    }
}

}  // namespace w1mg_dev
