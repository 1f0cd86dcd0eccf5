// pdhg_rs2.cuh -- the row-resident level-persistent PDHG engine of
// pdhg_rs.cuh for 129 < m <= 257 (the prime m = 257 level of config 3):
// thread-block clusters of TWO CTAs share one register-stationary DCT matrix.
//
// The folded cosine matrix c(k,i), k < m-1, i < h = (m-1)/2, has 2 h^2
// entries: 32,768 doubles at m = 257 -- the whole register file of an SM --
// so it is split by the parity of k over the two CTAs of a cluster: rank 0
// holds the even rows k = 2q+2 (and the rank-one constant / middle-sample
// terms), rank 1 the odd rows k = 2q+1, 32 doubles per thread.  That is the
// natural split of the folded transform:
//   DCT-II   even outputs need only s_i = x_i + x_{m-1-i}, odd outputs only
//            d_i = x_i - x_{m-1-i}: a CTA folds its own vectors and stores s
//            into rank 0's and d into rank 1's shared memory (DSMEM), one
//            cluster barrier, then each CTA produces its half of the spectrum
//            of ALL the cluster's vectors;
//   DCT-III  each CTA turns its half of the spectrum into E_i (even part) or
//            O_i (odd part) for all the cluster's vectors and stores them
//            into the shared memory of the CTA that owns the vector; one
//            cluster barrier, then y_i = E_i + O_i, y_{m-1-i} = E_i - O_i.
// The products run on the FP64 tensor cores (mma.sync.m8n8k4.f64: 256 FMAs per
// warp instruction, the N = 8 columns are the cluster's vectors), because the
// scalar form was issue-bound (a 9-shuffle butterfly per vector and warp for
// the DCT-II, a shared-memory partial exchange for the DCT-III):
//   DCT-II   warp wq owns the rows q = 8 wq .. 8 wq + 7 of its half; its A
//            fragments c(q, 4 it + lane % 4), it < 32, stay in REGISTERS for
//            the whole level; the B fragments are the folded vectors (shared
//            memory); the accumulators are the finished outputs;
//   DCT-III  warp wq owns the outputs i = 8 wq .. 8 wq + 7; the A fragments of
//            the transposed matrix c(4 qt + lane % 4, i) are staged once per
//            level in shared memory in fragment order (conflict-free loads).
// The rank-one terms (constant mode: sum_i s_i; middle sample: sum_k X_k cos(pi
// k / 2)) are summed by whoever PRODUCES the vector (the fold, the row / column
// loads, the accumulators of the preceding DCT-II), one warp per vector, so
// nothing follows the MMAs on the critical path (as a 17th MMA row tile on
// warp 0 they cost ~0.8 us per iteration).
//
// The iteration structure, the shadow row, the deferred stop rule and the
// plane/position conventions are those of pdhg_rs.cuh (reference semantics:
// solver_pdhg.hpp:20-46, poisson.cpp:72-132).
#pragma once

#include "pdhg_rs.cuh"

namespace w1mg_dev {

constexpr int kRs2HP = 128;   // padded half size: h <= 128
constexpr int kRs2HS = 132;   // row stride of the folded / spectral vectors (conflict-free B fragments)
constexpr int kRs2NV = 8;     // rows of the vector buffers = the N of the MMA

// D (8 x 8) += A (8 x 4, row) B (4 x 8, col), fp64: lane holds A[lane/4][lane%4],
// B[lane%4][lane/4], D[lane/4][2 (lane%4) + {0, 1}]
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// Dynamic shared memory (doubles)
__host__ __device__ inline size_t rs2_smem_doubles(int m, int R) {
    const int ms = m + 1;
    return (size_t)ms * (1 + 7 * (R + 1) + (R + 2)) + (size_t)kRs2HS * (2 * kRs2NV + 2 * (R + 2)) +
           (size_t)16 * 32 * 32 + 16 * kRs2NV + 8;
}

template <int QN>
__global__ void __launch_bounds__(kRsThreads, 1)
pdhg_rs2_kernel(const SweepArgs a, const RsArgs ra, GridBar gb) {
    extern __shared__ __align__(16) double rs_sm[];
    __shared__ int s_ok;
    __shared__ int s_stop;
    __shared__ double red[kRsThreads / 32][3];
    cg::cluster_group cluster = cg::this_cluster();
    PairCtl* ctl = a.ctl;
    if (*(volatile int*)&ctl->done) return;  // uniform over the grid
    if ((int)blockIdx.x >= ra.G) {  // reducer cluster: Eq. 12 sums and the stop rule
        rs_reducer(rs_red_args(a, ra), gb, (int)blockIdx.x == ra.G);
        return;
    }
    const int m = ra.m, n = m - 1, h = ra.h, R = ra.R, G = ra.G;
    const int ms = m + 1, tid = threadIdx.x, lane = tid & 31, wq = tid >> 5;
    constexpr int hs = kRs2HS;
    const int c = blockIdx.x, e = (int)cluster.block_rank(), base = (c >> 1) * 2 * R;
    const int j0 = base + e * R, nr = max(0, min(R, m - j0));
    const int sh = (nr > 0 && j0 > 0) ? 1 : 0;
    const int hl = (nr > 0 && j0 + nr < m) ? 1 : 0;
    const int VC = max(0, min(2 * R, m - base));             // cluster vectors, phases A and B
    const int jlo = max(base - 1, 0), jhi = min(base + 2 * R, m - 1);
    const int VCc = jhi - jlo + 1;                           // rows of the row DCT-III (phase C)
    const Layout L = a.L;
    const double mu = a.mu, tau = a.tau, ih = a.ih, scale = ra.scale;

    double* lam = rs_sm;
    double* st = lam + ms;
    double* X = st + (size_t)S_N * (R + 1) * ms;
    double* F = X + (size_t)(R + 2) * ms;        // [8][hs] transform inputs of this half
    double* FY = F + (size_t)kRs2NV * hs;        // [8][hs] divided spectrum of this half
    double* EO = FY + (size_t)kRs2NV * hs;       // [R+2][2][hs] E / O of the vectors this CTA owns
    double* A3 = EO + (size_t)(R + 2) * 2 * hs;  // [16][32][32] DCT-III A fragments
    double* altp = A3 + 16 * 32 * 32;            // [16][8] per-warp partial sums of the middle sample
    double* Fr[2] = {cluster.map_shared_rank(F, 0), cluster.map_shared_rank(F, 1)};
    double* EOr[2] = {cluster.map_shared_rank(EO, 0), cluster.map_shared_rank(EO, 1)};
    auto S = [&](int slot, int sv) { return st + ((size_t)slot * (R + 1) + sv) * ms; };

    // coefficients of this CTA's half c(q, i) = cos(pi k (2i+1) / 2m), k = 2q+2 / 2q+1
    auto coef = [&](int q, int i) {
        const int kk = e ? 2 * q + 1 : 2 * q + 2;
        return (q < h && i < h) ? __ldg(ra.cosq + (kk * (2 * i + 1)) % (4 * m)) : 0.0;
    };
    const int fr = lane >> 2, fc = lane & 3;  // fragment row / column of this lane
    double cfa[32];                           // DCT-II A fragments: rows 8 wq + fr, columns 4 it + fc
#pragma unroll
    for (int it = 0; it < 32; ++it) cfa[it] = coef(8 * wq + fr, 4 * it + fc);
    for (int qt = 0; qt < 32; ++qt)           // DCT-III: A[i = 8 wq + fr][q = 4 qt + fc]
        A3[(wq * 32 + qt) * 32 + lane] = coef(4 * qt + fc, 8 * wq + fr);

    for (int x = tid; x < m; x += kRsThreads) lam[x] = ra.lamq[x];
    for (int x = tid; x < S_N * (R + 1) * ms; x += kRsThreads) st[x] = 0.0;
    for (int x = tid; x < (R + 2) * ms; x += kRsThreads) X[x] = 0.0;
    for (int x = tid; x < 2 * kRs2NV * hs; x += kRsThreads) F[x] = 0.0;  // F and FY
    __syncthreads();
    {
        const int gs[S_N] = {P_MX, P_MY, P_PX, P_PY, P_BX, P_BY, P_RHO};
        const int rows = nr + sh;
        for (int x = tid; x < S_N * rows * m; x += kRsThreads) {
            const int sl = x / (rows * m), rem = x - sl * rows * m, w = rem / m, i = rem - w * m;
            S(sl, w + 1 - sh)[i] = pslot(a, 0, gs[sl])[L.at(i, j0 - sh + w)];
        }
    }
    cluster.sync();  // both CTAs' buffers initialised before any remote store

    double* T1 = pslot_w(a, 0, P_T);    // T1[pos1][j] at L.at(j, pos1)
    double* T2 = pslot_w(a, 0, P_PSI);  // T2[j][pos1] at L.at(pos1, j)
    unsigned gen = 0;
    long iter = 0;
    auto stamp = [&](int q) {
        if (ra.stamps && c == 0 && tid == 0 && iter < 64) ra.stamps[iter * kRsStampSlots + q] = gtimer();
    };

    // fold the CTA's nr vectors X[v] and hand s to rank 0, d to rank 1
    auto fold_send = [&]() {
        for (int x = tid; x < nr * (h + 1); x += kRsThreads) {
            int v, i;
            rs_split(x, h + 1, v, i);
            const double* xv = X + v * ms;
            const int w = e * R + v;
            if (i < h) {
                const double p = xv[i], q = xv[m - 1 - i];
                Fr[0][w * hs + i] = p + q;
                Fr[1][w * hs + i] = p - q;
            } else {
                Fr[0][w * hs + h] = xv[h];
            }
        }
        // the constant mode needs sum_i s_i: one warp per owned vector sums it
        // here (both ranks, off the path behind the cluster barrier)
        if (wq >= 16 - nr) {
            const int v = 15 - wq;
            const double* xv = X + v * ms;
            double ss = 0.0;
            for (int i = lane; i < h; i += 32) ss += xv[i] + xv[m - 1 - i];
            ss = warp_sum(ss);
            if (lane == 0) Fr[0][(e * R + v) * hs + h + 1] = ss;
        }
    };
    // this half of the DCT-II of the cluster's vectors F[w], w < V <= 8: out(w, pos,
    // X_k) stores and returns the finished value.  F[w][h+1] holds sum_i s_i (rank
    // 0).  alt: rank 0 also leaves, per warp and vector, the partial sum of
    // y cos(pi k / 2) over its eight rows in altp[wq][w] (the middle sample of
    // the DCT-III that follows).
    auto dct2_half = [&](int V, bool alt, auto out) {
        const double* fb = F + fr * hs + fc;  // B[k = fc][n = fr] = F[vector fr][4 it + fc]
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int it = 0; it < 32; ++it) {
            dmma884(d0, d1, cfa[it], fb[4 * it]);
            if ((it & 7) == 7) asm volatile("" ::: "memory");  // loads in batches of 8 (registers)
        }
        const int q = 8 * wq + fr;
        double y[2] = {0.0, 0.0};
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
            const int w = 2 * fc + cc;
            const double sum = cc ? d1 : d0;
            if (w < V && q < h) {
                if (e) {
                    y[cc] = out(w, h + q, 2.0 * sum);
                } else {
                    const double xh = F[w * hs + h];
                    y[cc] = out(w, q, 2.0 * (sum + ((q & 1) ? xh : -xh)));  // cos(pi k / 2), k = 2q+2
                }
            }
        }
        if (e == 0) {
            if (alt) {  // sum over the warp's rows (lanes with the same fc) of +-y
#pragma unroll
                for (int cc = 0; cc < 2; ++cc) {
                    double t = (q & 1) ? y[cc] : -y[cc];
                    t += __shfl_xor_sync(0xffffffffu, t, 4);
                    t += __shfl_xor_sync(0xffffffffu, t, 8);
                    t += __shfl_xor_sync(0xffffffffu, t, 16);
                    if (fr == 0) altp[wq * kRs2NV + 2 * fc + cc] = t;
                }
            }
            if (wq == 0 && lane < V)  // constant mode: 2 (sum_i s_i + x_h)
                out(lane, 2 * h, 2.0 * (F[lane * hs + h + 1] + F[lane * hs + h]));
        }
    };
    // this half of the DCT-III of the spectra src[w] (own-half positions, the
    // constant mode at [h] on rank 0): E (rank 0) or O (rank 1) -> send(w, i, val),
    // i < h (the middle sample i = h is sent by the producers of the spectra)
    auto dct3_half = [&](int V, const double* src, auto send) {
        const double* yb = src + fr * hs + fc;  // B[k = fc][n = fr] = src[vector fr][4 qt + fc]
        const double* a3 = A3 + (wq * 32) * 32 + lane;
        double d0 = 0.0, d1 = 0.0;
#pragma unroll 8
        for (int qt = 0; qt < 32; ++qt) dmma884(d0, d1, a3[qt * 32], yb[4 * qt]);
        const int i = 8 * wq + fr;
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
            const int w = 2 * fc + cc;
            const double sum = cc ? d1 : d0;
            if (w < V && i < h) send(w, i, e ? 2.0 * sum : src[w * hs + h] + 2.0 * sum);
        }
    };
    // y of the owned vectors from their E / O rows
    // the NX owned vectors at once (one flat loop: every thread busy): out(x, i, y_i)
    auto combine = [&](int NX, auto out) {
        for (int t = tid; t < NX * (h + 1); t += kRsThreads) {
            int x, i;
            rs_split(t, h + 1, x, i);
            const double* E = EO + (size_t)(2 * x) * hs;
            const double* O = E + hs;
            if (i < h) {
                out(x, i, E[i] + O[i]);
                out(x, m - 1 - i, E[i] - O[i]);
            } else {
                out(x, h, E[h]);
            }
        }
    };

    for (;; ++iter) {
        stamp(0);
        // ---- A: r = A v - rho on the owned rows (poisson.cpp:113-115), DCT-II along i -> T1
        for (int x = tid; x < nr * m; x += kRsThreads) {
            int v, i;
            rs_split(x, m, v, i);
            const int j = j0 + v, sv = v + 1;
            const double* mx = S(S_MX, sv);
            const double* bx = S(S_BX, sv);
            const double r_ = (i < n) ? mx[i] - mu * bx[i] : 0.0;
            const double l_ = (i > 0) ? mx[i - 1] - mu * bx[i - 1] : 0.0;
            const double a_ = (j < n) ? S(S_MY, sv)[i] - mu * S(S_BY, sv)[i] : 0.0;
            const double b_ = (j > 0) ? S(S_MY, sv - 1)[i] - mu * S(S_BY, sv - 1)[i] : 0.0;
            const double div = (r_ - l_) * ih + (a_ - b_) * ih;
            X[v * ms + i] = div - S(S_RHO, sv)[i];
        }
        __syncthreads();
        stamp(1);
        fold_send();
        cluster.sync();
        stamp(2);
        dct2_half(VC, false, [&](int w, int pos, double val) {
            T1[L.at(base + w, pos)] = val;
            return val;
        });
        stamp(11);
        if (!grid_barrier(gb, gen, &s_ok)) return;
        stamp(12);
        // ---- B: columns pos1 = base + w: DCT-II along j, divide by lambda_k1 +
        // lambda_k2 (poisson.cpp:84-89), DCT-III along j -> T2
        // every CTA reads all the cluster's columns and folds them into its own
        // half (s on rank 0, d on rank 1): no exchange, no cluster barrier here
        if (wq < VC) {  // warp wq takes column base + wq (all its loads in flight together)
            const int w = wq;
            const double* col = T1 + L.at(0, base + w);
            const double mid = __ldcg(col + h);  // requested with the other loads
            double ss = 0.0;
            for (int i = lane; i < h; i += 32) {
                const double p = __ldcg(col + i), q = __ldcg(col + m - 1 - i);
                F[w * hs + i] = e ? p - q : p + q;
                ss += p + q;
            }
            if (e == 0) {
                ss = warp_sum(ss);
                if (lane == 0) {
                    F[w * hs + h] = mid;
                    F[w * hs + h + 1] = ss;
                }
            }
        }
        __syncthreads();
        stamp(5);
        stamp(6);
        dct2_half(VC, true, [&](int w, int pos, double val) {
            const int p1 = base + w;
            const double y = (p1 == 2 * h && pos == 2 * h) ? 0.0 : val / (lam[p1] + lam[pos]);
            FY[w * hs + (pos == 2 * h ? h : (e ? pos - h : pos))] = y;
            return y;
        });
        __syncthreads();
        stamp(7);
        auto send_b = [&](int w, int i, double val) {
            const int o = w / R;  // owner rank of column base + w
            EOr[o][((size_t)(2 * (w - o * R)) + e) * hs + i] = val;
        };
        if (e == 0 && tid < VC) {  // middle sample: constant mode + 2 sum_k y_k cos(pi k / 2)
            double t = 0.0;
            for (int w2 = 0; w2 < 16; ++w2) t += altp[w2 * kRs2NV + tid];
            send_b(tid, h, FY[tid * hs + h] + 2.0 * t);
        }
        dct3_half(VC, FY, send_b);
        cluster.sync();
        stamp(8);
        combine(nr, [&](int v, int j, double val) { T2[L.at(j0 + v, j)] = val; });
        stamp(9);
        stamp(11);
        if (!grid_barrier(gb, gen, &s_ok)) return;
        stamp(12);
        // ---- C: rows jlo .. jhi of T2 (the cluster's rows, the shadow row
        // below and the halo row above): DCT-III along i; afterwards X row x
        // holds psi = y / (4 m^2) (poisson.cpp:93) of row j0 - sh + x
        int decv = 0;  // the reducer's decision: requested now, consumed after the row loads
        if (iter > 0 && tid == 0) decv = __ldcg(ra.dec + (iter & 1));
        auto send_c = [&](int w, int i, double val) {
            const int jj = jlo + w;
#pragma unroll
            for (int o = 0; o < 2; ++o) {
                const int j0o = base + o * R, nro = max(0, min(R, m - j0o));
                const int sho = (nro > 0 && j0o > 0) ? 1 : 0, hlo = (nro > 0 && j0o + nro < m) ? 1 : 0;
                const int xo = jj - (j0o - sho);
                if (nro > 0 && xo >= 0 && xo < sho + nro + hlo)
                    EOr[o][((size_t)(2 * xo) + e) * hs + i] = val;
            }
        };
        if (wq < VCc) {  // warp wq takes row jlo + wq: its half of the spectrum, and on
            const int w = wq;  // rank 0 the middle sample (constant mode + alternating sum)
            const double* row = T2 + L.at(e ? h : 0, jlo + w);
            const double dc = e ? 0.0 : __ldcg(T2 + L.at(2 * h, jlo + w));  // with the other loads
            double as = 0.0;
            for (int q = lane; q < h; q += 32) {
                const double yq = __ldcg(row + q);
                F[w * hs + q] = yq;
                as += (q & 1) ? yq : -yq;
            }
            if (e == 0) {
                as = warp_sum(as);
                if (lane == 0) {
                    F[w * hs + h] = dc;
                    send_c(w, h, dc + 2.0 * as);
                }
            }
        }
        if (tid == 0) s_stop = decv;
        __syncthreads();
        if (iter > 0 && s_stop) {  // iteration iter-1 met the stop rule: its state is final
                const int gs[6] = {P_MX, P_MY, P_PX, P_PY, P_BX, P_BY};
                for (int x = tid; x < 6 * nr * m; x += kRsThreads) {
                    const int sl = x / (nr * m), rem = x - sl * nr * m, v = rem / m, i = rem - v * m;
                    pslot_w(a, 0, gs[sl])[L.at(i, j0 + v)] = S(sl, v + 1)[i];
                }
                cluster.sync();  // no CTA leaves while its partner may still store into it
            return;
        }
        stamp(13);
        dct3_half(VCc, F, send_c);
        cluster.sync();
        stamp(14);
        combine(sh + nr + hl, [&](int x, int i, double val) { X[x * ms + i] = scale * val; });
        __syncthreads();
        stamp(16);
        // ---- D: post step (pdhg_post_kernel's arithmetic) on the shadow and
        // owned rows; Eq. 12 partial sums over the owned rows only
        double s_dm2 = 0.0, s_dp2 = 0.0, s_cr = 0.0;
        for (int x = tid; x < (nr + sh) * m; x += kRsThreads) {
            int w, i;
            rs_split(x, m, w, i);
            const int sv = w + 1 - sh, j = j0 + sv - 1;
            const bool hx = i < n, hy = j < n, mine = sv > 0;
            const double pc = X[w * ms + i];
            double mnx = 0.0, mny = 0.0, dmx = 0.0, dmy = 0.0, pox = 0.0, poy = 0.0;
            if (hx) {
                const double mo = S(S_MX, sv)[i];
                const double vv = mo - mu * S(S_BX, sv)[i];
                mnx = vv - (pc - X[w * ms + i + 1]) * ih;  // poisson.cpp:124
                dmx = mnx - mo;
                pox = S(S_PX, sv)[i];
            }
            if (hy) {
                const double mo = S(S_MY, sv)[i];
                const double vv = mo - mu * S(S_BY, sv)[i];
                mny = vv - (pc - X[(w + 1) * ms + i]) * ih;  // poisson.cpp:130
                dmy = mny - mo;
                poy = S(S_PY, sv)[i];
            }
            const double wx = hx ? pox + tau * mnx : 0.0;
            const double wy = hy ? poy + tau * mny : 0.0;
            double qx, qy;
            rs_proj_unit_ball<QN>(wx, wy, qx, qy);
            if (hx) {
                S(S_MX, sv)[i] = mnx;
                S(S_PX, sv)[i] = qx;
                S(S_BX, sv)[i] = 2.0 * qx - pox;
                if (mine) {
                    const double dp = qx - pox;
                    s_dm2 += dmx * dmx;
                    s_dp2 += dp * dp;
                    s_cr += dp * dmx;
                }
            }
            if (hy) {
                S(S_MY, sv)[i] = mny;
                S(S_PY, sv)[i] = qy;
                S(S_BY, sv)[i] = 2.0 * qy - poy;
                if (mine) {
                    const double dp = qy - poy;
                    s_dm2 += dmy * dmy;
                    s_dp2 += dp * dp;
                    s_cr += dp * dmy;
                }
            }
        }
        s_dm2 = warp_sum(s_dm2);
        s_dp2 = warp_sum(s_dp2);
        s_cr = warp_sum(s_cr);
        if (lane == 0) {
            red[wq][0] = s_dm2;
            red[wq][1] = s_dp2;
            red[wq][2] = s_cr;
        }
        __syncthreads();  // state rows and red[] complete
        if (tid == 0) {
            double t0 = 0.0, t1 = 0.0, t2 = 0.0;
            for (int w = 0; w < kRsThreads / 32; ++w) {
                t0 += red[w][0];
                t1 += red[w][1];
                t2 += red[w][2];
            }
            ra.part[c * 3 + 0] = t0;
            ra.part[c * 3 + 1] = t1;
            ra.part[c * 3 + 2] = t2;
        }
        stamp(17);
    }
}

}  // namespace w1mg_dev
