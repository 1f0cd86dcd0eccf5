// tile2_kernels.cuh -- the level-persistent tile engine (tile_kernels.cuh)
// with TWO sweeps per halo exchange.
//
// Each tile keeps a two-node halo ring.  A double step computes
//   sweep 1 (k -> k+1) on the tile plus a one-node ring: phase A on local
//     [0, w+2] x [0, h+2], phase B on [1, w+2] x [1, h+2];
//   sweep 2 (k+1 -> k+2) on the tile: phase A on [1, w+1] x [1, h+1]
//     (the recomputed left / bottom ring), phase B on the owned nodes;
// then publishes its two-node boundary strips (phi, m_x, m_y of the first
// and last two columns and rows) and releases one step flag.  Neighbours in
// all eight directions read those strips into their rings, so the inter-SM
// flag and fresh-L2 latencies (~2 x 1 us per exchange, measured) are paid once
// per two sweeps; the ring costs ~(w+3)(h+3)/(w h) extra node work.
//
// The stop rule is the tile engine's: residual partials of both sweeps go to
// the pipelined controller, tiles read the decisions of sweeps k - lag and
// k - lag + 1 at the start of double step k, and a stop at sweep s is
// restored from the checkpoint at or below s + 1 and replayed in double
// steps plus, when s + 1 is odd relative to the checkpoint, one half step
// (sweep 1 only; its owned values are the final state).  Node arithmetic is
// node_flux / row_update's, so fields stay bit-identical to the reference.
#pragma once

#include "tile_kernels.cuh"

namespace w1mg_dev {

constexpr int kT2Secs = 24;  // record sections: [field phi, m_x, m_y][side L, R, B, T][line 0, 1]
enum T2Side { T2_L = 0, T2_R = 1, T2_B = 2, T2_T = 3 };
__host__ inline int tile2_list_cap(int LW, int LH) { return 4 * (LW + LH) + 16; }
__host__ inline long tile2_smem_bytes(int LW, int LH) {
    return 6L * LW * LH * 8 + 2L * tile2_list_cap(LW, LH) * 4;
}

template <int PN>
__global__ void __launch_bounds__(kTileThreads, 1) cp_tile2_kernel(const TileArgs t) {
    const int T = t.TR * t.TC;
    const int pair = blockIdx.x / (T + 1);
    const int tile = blockIdx.x % (T + 1);
    const SweepArgs& a = t.a;
    PairCtl* ctl = a.ctl + pair;
    if (*(volatile int*)&ctl->done) return;
    const long k0 = ctl->it;
    if (tile == T) {
        tile_controller(t, pair, T, k0);
        return;
    }
    extern __shared__ __align__(16) double sm[];
    __shared__ double wred[kTileWarps][6];
    __shared__ int s_stop, s_hn;
    __shared__ long s_stop_at;
    __shared__ double s_fpr;
    __shared__ int s_dec[2];
    __shared__ double s_decf[2];

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
    int* hk = reinterpret_cast<int*>(sm + 6 * S);  // ring node -> smem index
    int* ho = hk + t.LCAP;                         // ring node -> record offset (phi)
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const double mu = a.mu, zt = a.zt, tau = a.tau, ih = a.ih;
    const int ES = t.ES;

    const int nL = tc > 0 ? tile - 1 : -1;
    const int nR = tc + 1 < t.TC ? tile + 1 : -1;
    const int nD = tr > 0 ? tile - t.TC : -1;
    const int nU = tr + 1 < t.TR ? tile + t.TC : -1;
    const int nUL = (tr + 1 < t.TR && tc > 0) ? tile + t.TC - 1 : -1;
    const int nUR = (tr + 1 < t.TR && tc + 1 < t.TC) ? tile + t.TC + 1 : -1;
    const int nDL = (tr > 0 && tc > 0) ? tile - t.TC - 1 : -1;
    const int nDR = (tr > 0 && tc + 1 < t.TC) ? tile - t.TC + 1 : -1;

    const long recs = (long)T * kT2Secs * ES;  // doubles per step buffer of one pair
    double* ebase = t.edges + (long)pair * 2 * recs;
    auto rec_off = [&](int who, int field, int side, int line) -> long {
        return ((((long)who * 3 + field) * 4 + side) * 2 + line) * ES;
    };
    unsigned* flags = t.flags + (long)pair * T * kTileFlagStride;
    double* pb = a.base + (long)pair * NSLOT * L.plane;

    // ---- ring map (thread 0, fixed order): which neighbour strip holds each
    // in-grid ring node of the local region [0, w+3] x [0, h+3]
    if (tid == 0) {
        int cnt = 0;
        for (int lj = 0; lj <= h + 3; ++lj)
            for (int li = 0; li <= w + 3; ++li) {
                if (li >= 2 && li <= w + 1 && lj >= 2 && lj <= h + 1) continue;
                const int i = i0 - 2 + li, j = j0 - 2 + lj;
                if (i < 0 || j < 0 || i > n || j > n) continue;
                const int dx = li < 2 ? -1 : (li > w + 1 ? 1 : 0);
                const int dy = lj < 2 ? -1 : (lj > h + 1 ? 1 : 0);
                const int oc = tc + dx, orr = tr + dy;
                const int oi0 = tile_lo(n + 1, t.TC, oc), oj0 = tile_lo(n + 1, t.TR, orr);
                const int ow = tile_lo(n + 1, t.TC, oc + 1) - oi0;
                const int oh = tile_lo(n + 1, t.TR, orr + 1) - oj0;
                const int li2 = i - (oi0 - 2), lj2 = j - (oj0 - 2);
                int side, line, idx;
                if (dx == -1) { side = T2_R; line = li2 - ow; idx = lj2 - 2; }
                else if (dx == 1) { side = T2_L; line = li2 - 2; idx = lj2 - 2; }
                else if (dy == -1) { side = T2_T; line = lj2 - oh; idx = li2 - 2; }
                else { side = T2_B; line = lj2 - 2; idx = li2 - 2; }
                hk[cnt] = lj * LW + li;
                ho[cnt] = (int)(rec_off(orr * t.TC + oc, 0, side, line) + idx);
                ++cnt;
            }
        s_hn = cnt;
        s_stop = 0;
    }

    // whole local region from the level buffer planes of parity p
    auto load_state = [&](int p) {
        const double* gp = pb + (PHI0 + p) * L.plane;
        const double* gx = pb + (MX0 + p) * L.plane;
        const double* gy = pb + (MY0 + p) * L.plane;
        const double* gr = pb + RHO * L.plane;
        const int W4 = w + 4, cnt = W4 * (h + 4);
        for (int q = tid; q < cnt; q += kTileThreads) {
            const int li = q % W4, lj = q / W4;
            const int i = i0 - 2 + li, j = j0 - 2 + lj;
            const bool in = i >= 0 && i <= n && j >= 0 && j <= n;
            const long o = in ? L.at(i, j) : 0;
            const int k = lj * LW + li;
            phi[k] = in ? __ldcg(gp + o) : 0.0;
            mx[k] = (in && i < n) ? __ldcg(gx + o) : 0.0;
            my[k] = (in && j < n) ? __ldcg(gy + o) : 0.0;
            ddx[k] = 0.0;
            ddy[k] = 0.0;
            rho[k] = in ? __ldg(gr + o) : 0.0;
        }
    };
    auto store_state = [&](int p) {
        double* gp = pb + (PHI0 + p) * L.plane;
        double* gx = pb + (MX0 + p) * L.plane;
        double* gy = pb + (MY0 + p) * L.plane;
        for (int q = tid; q < w * h; q += kTileThreads) {
            const int li = 2 + q % w, lj = 2 + q / w;
            const int i = i0 - 2 + li, j = j0 - 2 + lj;
            const long o = L.at(i, j);
            const int k = lj * LW + li;
            __stcg(gp + o, phi[k]);
            if (i < n) __stcg(gx + o, mx[k]);
            if (j < n) __stcg(gy + o, my[k]);
        }
    };
    auto load_halo = [&](int buf) {
        const double* bb = ebase + buf * recs;
        const long FS = 8L * ES;  // field stride
        const int hn = s_hn;
        for (int q = tid; q < hn; q += kTileThreads) {
            const double* src = bb + ho[q];
            const int k = hk[q];
            phi[k] = __ldcg(src);
            mx[k] = __ldcg(src + FS);
            my[k] = __ldcg(src + 2 * FS);
        }
    };

    // phase A / B node updates; `in` = the node is inside the grid
    auto nodeA = [&](int li, int lj, double& sdm2, bool own) {
        const int i = i0 - 2 + li, j = j0 - 2 + lj;
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
        if (own) sdm2 = __fma_rn(dy, dy, __fma_rn(dx, dx, sdm2));
    };
    auto nodeB = [&](int li, int lj, double& sdp2, double& scr, bool own) {
        const int kk = lj * LW + li;
        const double divm = (mx[kk] - mx[kk - 1]) * ih + (my[kk] - my[kk - LW]) * ih;
        const double divd = (ddx[kk] - ddx[kk - 1]) * ih + (ddy[kk] - ddy[kk - LW]) * ih;
        const double d = tau * (divm + divd - rho[kk]);
        phi[kk] = phi[kk] + d;
        if (own) {
            sdp2 = __fma_rn(d, d, sdp2);
            scr = __fma_rn(d, divd, scr);
        }
    };
    auto inside = [&](int li, int lj) {
        const int i = i0 - 2 + li, j = j0 - 2 + lj;
        return i >= 0 && j >= 0 && i <= n && j <= n;
    };
    auto owned = [&](int li, int lj) { return li >= 2 && li <= w + 1 && lj >= 2 && lj <= h + 1; };
    // sweep 1 on the tile + one-node ring (owned sums -> s1*)
    auto sweep1 = [&](double& s1a, double& s1b, double& s1c) {
        const int W3 = w + 3, nA = W3 * (h + 3);
        for (int q = tid; q < nA; q += kTileThreads) {
            const int li = q % W3, lj = q / W3;
            if ((li | lj) == 0 || !inside(li, lj)) continue;
            nodeA(li, lj, s1a, owned(li, lj));
        }
        __syncthreads();
        const int W2 = w + 2, nB = W2 * (h + 2);
        for (int q = tid; q < nB; q += kTileThreads) {
            const int li = 1 + q % W2, lj = 1 + q / W2;
            if (!inside(li, lj)) continue;
            nodeB(li, lj, s1b, s1c, owned(li, lj));
        }
        __syncthreads();
    };
    // sweep 2 on the tile (records of the boundary strips into buffer bufw)
    auto sweep2 = [&](int bufw, double& s2a, double& s2b, double& s2c) {
        double* bb = ebase + bufw * recs;
        const int W1 = w + 1, nA = W1 * (h + 1);
        for (int q = tid; q < nA; q += kTileThreads) {
            const int li = 1 + q % W1, lj = 1 + q / W1;
            if ((li == 1 && lj == 1) || !inside(li, lj)) continue;
            const bool own = owned(li, lj);
            nodeA(li, lj, s2a, own);
            if (own) {
                const int kk = lj * LW + li;
                const double ux = mx[kk], uy = my[kk];
                if (li <= 3) {
                    bb[rec_off(tile, 1, T2_L, li - 2) + lj - 2] = ux;
                    bb[rec_off(tile, 2, T2_L, li - 2) + lj - 2] = uy;
                }
                if (li >= w) {
                    bb[rec_off(tile, 1, T2_R, li - w) + lj - 2] = ux;
                    bb[rec_off(tile, 2, T2_R, li - w) + lj - 2] = uy;
                }
                if (lj <= 3) {
                    bb[rec_off(tile, 1, T2_B, lj - 2) + li - 2] = ux;
                    bb[rec_off(tile, 2, T2_B, lj - 2) + li - 2] = uy;
                }
                if (lj >= h) {
                    bb[rec_off(tile, 1, T2_T, lj - h) + li - 2] = ux;
                    bb[rec_off(tile, 2, T2_T, lj - h) + li - 2] = uy;
                }
            }
        }
        __syncthreads();
        for (int q = tid; q < w * h; q += kTileThreads) {
            const int li = 2 + q % w, lj = 2 + q / w;
            nodeB(li, lj, s2b, s2c, true);
            const double f = phi[lj * LW + li];
            if (li <= 3) bb[rec_off(tile, 0, T2_L, li - 2) + lj - 2] = f;
            if (li >= w) bb[rec_off(tile, 0, T2_R, li - w) + lj - 2] = f;
            if (lj <= 3) bb[rec_off(tile, 0, T2_B, lj - 2) + li - 2] = f;
            if (lj >= h) bb[rec_off(tile, 0, T2_T, lj - h) + li - 2] = f;
        }
    };
    // warp 0: neighbours' flags (8 directions), lanes 8/9: decisions kd, kd+1
    auto wait_neighbours = [&](unsigned target_step, long kd) {
        int nb = -1;
        if (lane == 0) nb = nL;
        else if (lane == 1) nb = nR;
        else if (lane == 2) nb = nD;
        else if (lane == 3) nb = nU;
        else if (lane == 4) nb = nUL;
        else if (lane == 5) nb = nUR;
        else if (lane == 6) nb = nDL;
        else if (lane == 7) nb = nDR;
        if (nb >= 0) spin_geq(flags + (long)nb * kTileFlagStride, target_step, t.err);
        if ((lane == 8 || lane == 9) && kd >= k0) {
            const long kq = kd + (lane - 8);
            const int slot = (int)(kq % kTileSlots);
            const unsigned long long v =
                spin_tag64(t.dseq + (long)pair * kTileSlots + slot, (unsigned long long)(kq + 1), t.err);
            s_dec[lane - 8] = (int)(v & 1ull);
            if (v & 1ull) s_decf[lane - 8] = __ldcg(t.dec + ((long)pair * kTileSlots + slot) * 2);
        }
        __syncwarp();
        if (lane == 0 && kd >= k0) {
            if (s_dec[0]) {
                s_stop = 1;
                s_stop_at = kd;
                s_fpr = s_decf[0];
            } else if (s_dec[1]) {
                s_stop = 1;
                s_stop_at = kd + 1;
                s_fpr = s_decf[1];
            }
        }
        __syncwarp();
    };

    long k = k0;
    unsigned step = 0;
    bool replay = false;
    long target = -1;
    double fin_fpr = 0.0;
    long stop_at = -1;
    __syncthreads();
    load_state(ctl->cur);
    __syncthreads();
    if (ctl->cur != 0) store_state(0);
    bool have_halo = true;
    long long dbg_acc[kTileDbgPts] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long dbg_last = clock64();
#define STAMP2(pt)                                                   \
    if (t.dbg && tid == 0) {                                         \
        const long long now_ = clock64();                            \
        if (step >= 4 && step < 68) dbg_acc[pt] += now_ - dbg_last;  \
        dbg_last = now_;                                             \
    }

    for (;;) {
        if (replay && k >= target) break;
        STAMP2(0);
        if (!have_halo) {
            if (warp == 0) wait_neighbours(step, replay ? k0 - 1 : k - kTileLag);
            __syncthreads();
            if (!replay && s_stop) {
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
            STAMP2(1);
            load_halo((int)(step & 1));
            __syncthreads();
        }
        STAMP2(2);
        double s1a = 0.0, s1b = 0.0, s1c = 0.0, s2a = 0.0, s2b = 0.0, s2c = 0.0;
        sweep1(s1a, s1b, s1c);
        STAMP2(3);
        if (replay && k + 1 == target) {  // half step: sweep 1's owned values are final
            ++k;
            break;
        }
        const int bufw = (int)((step + 1) & 1);
        sweep2(bufw, s2a, s2b, s2c);
        STAMP2(4);
        double v[6] = {s1a, s1b, s1c, s2a, s2b, s2c};
#pragma unroll
        for (int q = 0; q < 6; ++q) v[q] = warp_sum(v[q]);
        if (lane == 0)
#pragma unroll
            for (int q = 0; q < 6; ++q) wred[warp][q] = v[q];
        __syncthreads();
        if (tid == 0)
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + (long)tile * kTileFlagStride),
                         "r"(step + 1)
                         : "memory");
        if (tid == 32 && !replay) {  // off the critical path: no barrier waits for it
            for (int sw = 0; sw < 2; ++sw) {
                const int slot = (int)((k + sw) % kTileSlots);
                double t0 = 0.0, t1 = 0.0, t2 = 0.0;
                for (int q = 0; q < kTileWarps; ++q) {
                    t0 += wred[q][3 * sw + 0];
                    t1 += wred[q][3 * sw + 1];
                    t2 += wred[q][3 * sw + 2];
                }
                double* p = t.part + (((long)pair * kTileSlots + slot) * T + tile) * 3;
                p[0] = t0;
                p[1] = t1;
                p[2] = t2;
            }
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            for (int sw = 0; sw < 2; ++sw)
                asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(
                                 t.cnt + (long)pair * kTileSlots + (int)((k + sw) % kTileSlots))
                             : "memory");
        }
        k += 2;
        ++step;
        have_halo = false;
        if (!replay && ((k - k0) % kTileCk) == 0) {
            store_state((int)(((k - k0) / kTileCk) & 1));
            __syncthreads();  // the next sweep rewrites the owned nodes being stored
        }
        STAMP2(5);
    }
    if (t.dbg && tid == 0)
        for (int q = 0; q < kTileDbgPts; ++q) t.dbg[tile * kTileDbgPts + q] = dbg_acc[q];
#undef STAMP2
    // final barrier with the neighbours: every one of them has finished its
    // replay (including a checkpoint load after a rollback) before the final
    // state overwrites buffer 0
    __syncthreads();
    if (tid == 0)
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + (long)tile * kTileFlagStride),
                     "r"(step + 1)
                     : "memory");
    if (warp == 0) wait_neighbours(step + 1, k0 - 1);
    __syncthreads();
    store_state(0);
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
