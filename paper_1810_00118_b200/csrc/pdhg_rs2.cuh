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
// Thread (warp wq, lane): rows q = 16 r + wq (r < 8), columns i = 32 s + lane
// (s < 4).  The DCT-II sums over i run in registers and end in a 9-shuffle
// butterfly inside the warp (no shared-memory exchange, no second phase); the
// DCT-III sums over q leave 16 per-warp partials per output, summed through
// shared memory.
//
// The iteration structure, the shadow row, the deferred stop rule and the
// plane/position conventions are those of pdhg_rs.cuh (reference semantics:
// solver_pdhg.hpp:20-46, poisson.cpp:72-132).
#pragma once

#include "pdhg_rs.cuh"

namespace w1mg_dev {

constexpr int kRs2KB = 8, kRs2IB = 4, kRs2HP = 128;  // rows / columns per thread, padded half

// 8 per-lane values -> the sum over the 32 lanes of value r = 4 b4 + 2 b3 + b2
// (b = bits of the lane index), replicated over the lane's low two bits.
__device__ __forceinline__ double rs2_butterfly(const double (&v)[8], int lane) {
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
    double u[4], t[2];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const double send = b4 ? v[j] : v[j + 4], keep = b4 ? v[j + 4] : v[j];
        u[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const double send = b3 ? u[j] : u[j + 2], keep = b3 ? u[j + 2] : u[j];
        t[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    const double send = b2 ? t[0] : t[1], keep = b2 ? t[1] : t[0];
    double w = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    w += __shfl_xor_sync(0xffffffffu, w, 2);
    w += __shfl_xor_sync(0xffffffffu, w, 1);
    return w;
}

// Dynamic shared memory (doubles)
__host__ __device__ inline size_t rs2_smem_doubles(int m, int R) {
    const int ms = m + 1, hs = (m - 1) / 2 + 2;
    return (size_t)ms * (1 + 7 * (R + 1) + (R + 2)) + (size_t)hs * ((2 * R + 2) + 2 * R + 2 * (R + 2)) +
           (size_t)(2 * R + 2) * (kRs2HP + 1) * 17 + 8;
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
    long k = ctl->it;
    const long max_it = ctl->max_it;
    const double tol = ctl->tol;
    const int m = ra.m, n = m - 1, h = ra.h, R = ra.R, G = (int)gridDim.x;
    const int ms = m + 1, hs = h + 2, tid = threadIdx.x, lane = tid & 31, wq = tid >> 5;
    const int c = blockIdx.x, e = (int)cluster.block_rank(), base = (c >> 1) * 2 * R;
    const int j0 = base + e * R, nr = max(0, min(R, m - j0));
    const int sh = (nr > 0 && j0 > 0) ? 1 : 0;
    const int hl = (nr > 0 && j0 + nr < m) ? 1 : 0;
    const int VC = max(0, min(2 * R, m - base));             // cluster vectors, phases A and B
    const int jlo = max(base - 1, 0), jhi = min(base + 2 * R, m - 1);
    const int VCc = jhi - jlo + 1;                           // rows of the row DCT-III (phase C)
    const Layout L = a.L;
    const double mu = a.mu, tau = a.tau, ih = a.ih, scale = ra.scale;
    constexpr int PS = (kRs2HP + 1) * 17;

    double* lam = rs_sm;
    double* st = lam + ms;
    double* X = st + (size_t)S_N * (R + 1) * ms;
    double* F = X + (size_t)(R + 2) * ms;        // [2R+2][hs] transform inputs of this half
    double* FY = F + (size_t)(2 * R + 2) * hs;   // [2R][hs] divided spectrum of this half
    double* EO = FY + (size_t)(2 * R) * hs;      // [R+2][2][hs] E / O of the vectors this CTA owns
    double* P3 = EO + (size_t)(R + 2) * 2 * hs;  // [2R+2][PS] DCT-III partials
    double* Fr[2] = {cluster.map_shared_rank(F, 0), cluster.map_shared_rank(F, 1)};
    double* EOr[2] = {cluster.map_shared_rank(EO, 0), cluster.map_shared_rank(EO, 1)};
    auto S = [&](int slot, int sv) { return st + ((size_t)slot * (R + 1) + sv) * ms; };

    // coefficients of this CTA's half: rows q = 16 r + wq, columns i = 32 s + lane
    double cf[kRs2KB][kRs2IB];
#pragma unroll
    for (int r = 0; r < kRs2KB; ++r) {
        const int q = 16 * r + wq, kk = e ? 2 * q + 1 : 2 * q + 2;
#pragma unroll
        for (int s = 0; s < kRs2IB; ++s) {
            const int i = 32 * s + lane;
            cf[r][s] = (q < h && i < h) ? __ldg(ra.cosq + (kk * (2 * i + 1)) % (4 * m)) : 0.0;
        }
    }

    for (int x = tid; x < m; x += kRsThreads) lam[x] = ra.lamq[x];
    for (int x = tid; x < S_N * (R + 1) * ms; x += kRsThreads) st[x] = 0.0;
    for (int x = tid; x < (R + 2) * ms; x += kRsThreads) X[x] = 0.0;
    for (int x = tid; x < (2 * R + 2) * hs; x += kRsThreads) F[x] = 0.0;
    for (int x = tid; x < 2 * R * hs; x += kRsThreads) FY[x] = 0.0;
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
        if (ra.stamps && c == 0 && tid == 0 && iter < 64) ra.stamps[iter * 10 + q] = gtimer();
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
    };
    // this half of the DCT-II of the cluster's vectors F[w], w < V: out(w, pos, X_k)
    auto dct2_half = [&](int V, auto out) {
        for (int w = 0; w < V; ++w) {
            const double* f = F + w * hs;
            double in[kRs2IB];
#pragma unroll
            for (int s = 0; s < kRs2IB; ++s) {
                const int i = 32 * s + lane;
                in[s] = (i < h) ? f[i] : 0.0;
            }
            double acc[kRs2KB];
#pragma unroll
            for (int r = 0; r < kRs2KB; ++r) {
                double t = 0.0;
#pragma unroll
                for (int s = 0; s < kRs2IB; ++s) t = fma(cf[r][s], in[s], t);
                acc[r] = t;
            }
            const double sum = rs2_butterfly(acc, lane);
            const int r = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
            const int q = 16 * r + wq;
            const double xh = e ? 0.0 : f[h];
            if ((lane & 3) == 0 && q < h) {
                if (e) out(w, h + q, 2.0 * sum);
                else out(w, q, 2.0 * (sum + ((q & 1) ? xh : -xh)));  // cos(pi k / 2), k = 2q+2
            }
            if (e == 0 && wq == 0) {  // constant mode: plain sum of the symmetric part
                double dc = (in[0] + in[1]) + (in[2] + in[3]);
                dc = warp_sum(dc);
                if (lane == 0) out(w, 2 * h, 2.0 * (dc + xh));
            }
        }
    };
    // this half of the DCT-III of the spectra src[w] (own-half positions, the
    // constant mode at [h] on rank 0): E (rank 0) or O (rank 1) -> send(w, i, val),
    // i <= h (i = h: the middle sample, rank 0 only)
    auto dct3_half = [&](int V, const double* src, auto send) {
        for (int w = 0; w < V; ++w) {
            const double* y = src + w * hs;
            double in[kRs2KB];
#pragma unroll
            for (int r = 0; r < kRs2KB; ++r) {
                const int q = 16 * r + wq;
                in[r] = (q < h) ? y[q] : 0.0;
            }
            double* p = P3 + (size_t)w * PS + lane * 17 + wq;
#pragma unroll
            for (int s = 0; s < kRs2IB; ++s) {
                double t = 0.0;
#pragma unroll
                for (int r = 0; r < kRs2KB; ++r) t = fma(cf[r][s], in[r], t);
                p[s * 32 * 17] = t;
            }
            if (e == 0 && lane == 0) {  // middle sample: sum of X_k cos(pi k / 2), k even
                double mp = 0.0;
#pragma unroll
                for (int r = 0; r < kRs2KB; ++r) mp += ((16 * r + wq) & 1) ? in[r] : -in[r];
                P3[(size_t)w * PS + kRs2HP * 17 + wq] = mp;
            }
        }
        __syncthreads();
        const int per = e ? h : h + 1;
        for (int x = tid; x < V * per; x += kRsThreads) {
            int w, i;
            rs_split(x, per, w, i);
            const double sum = rs_sum16(P3 + (size_t)w * PS + (i < h ? i : kRs2HP) * 17);
            send(w, i, e ? 2.0 * sum : src[w * hs + h] + 2.0 * sum);
        }
    };
    // y of the owned vector x from its E / O rows: out(i, y_i)
    auto combine = [&](int x, auto out) {
        const double* E = EO + (size_t)(2 * x) * hs;
        const double* O = E + hs;
        for (int i = tid; i <= h; i += kRsThreads) {
            if (i < h) {
                out(i, E[i] + O[i]);
                out(m - 1 - i, E[i] - O[i]);
            } else {
                out(h, E[h]);
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
        fold_send();
        cluster.sync();
        dct2_half(VC, [&](int w, int pos, double val) { T1[L.at(base + w, pos)] = val; });
        stamp(1);
        if (!grid_barrier(gb, gen, &s_ok)) return;
        stamp(2);
        double pt0 = 0.0, pt1 = 0.0, pt2 = 0.0;  // Eq. 12 partials of the previous iteration
        if (iter > 0 && tid < G) {
            pt0 = __ldcg(ra.part + 3 * tid + 0);
            pt1 = __ldcg(ra.part + 3 * tid + 1);
            pt2 = __ldcg(ra.part + 3 * tid + 2);
        }
        // ---- B: columns pos1 = base + w: DCT-II along j, divide by lambda_k1 +
        // lambda_k2 (poisson.cpp:84-89), DCT-III along j -> T2
        for (int x = tid; x < nr * m; x += kRsThreads) {
            int v, j;
            rs_split(x, m, v, j);
            X[v * ms + j] = __ldcg(T1 + L.at(j, j0 + v));
        }
        __syncthreads();
        fold_send();
        cluster.sync();
        dct2_half(VC, [&](int w, int pos, double val) {
            const int p1 = base + w;
            const double y = (p1 == 2 * h && pos == 2 * h) ? 0.0 : val / (lam[p1] + lam[pos]);
            FY[w * hs + (pos == 2 * h ? h : (e ? pos - h : pos))] = y;
        });
        __syncthreads();
        dct3_half(VC, FY, [&](int w, int i, double val) {
            const int o = w / R;  // owner rank of column base + w
            EOr[o][((size_t)(2 * (w - o * R)) + e) * hs + i] = val;
        });
        cluster.sync();
        for (int v = 0; v < nr; ++v)
            combine(v, [&](int j, double val) { T2[L.at(j0 + v, j)] = val; });
        // ---- stop rule of the previous iteration (identical in every CTA)
        if (iter > 0) {
            pt0 = warp_sum(pt0);
            pt1 = warp_sum(pt1);
            pt2 = warp_sum(pt2);
            if (lane == 0) {
                red[wq][0] = pt0;
                red[wq][1] = pt1;
                red[wq][2] = pt2;
            }
            __syncthreads();
            if (tid == 0) {
                double t0 = 0.0, t1 = 0.0, t2 = 0.0;
                for (int w = 0; w < (G + 31) / 32; ++w) {
                    t0 += red[w][0];
                    t1 += red[w][1];
                    t2 += red[w][2];
                }
                const double fpr = a.h2 * (t0 / a.mu + t1 / a.tau + 2.0 * t2);  // Eq. 12
                const bool finite = isfinite(fpr);
                const bool stop = fpr < tol || k + 1 >= max_it || !finite;
                s_stop = stop ? 1 : 0;
                if (c == 0) {
                    if (a.hist && k < a.hist_cap) a.hist[k] = fpr;
                    if (stop) {
                        ctl->it = k + 1;
                        ctl->fpr = fpr;
                        ctl->cur = 0;
                        if (!finite) ctl->nonfinite = 1;
                        ctl->done = 1;
                        if (a.ndone) atomicAdd(a.ndone, 1);
                        __threadfence();
                    }
                }
            }
            __syncthreads();
            ++k;
            if (s_stop) {
                const int gs[6] = {P_MX, P_MY, P_PX, P_PY, P_BX, P_BY};
                for (int x = tid; x < 6 * nr * m; x += kRsThreads) {
                    const int sl = x / (nr * m), rem = x - sl * nr * m, v = rem / m, i = rem - v * m;
                    pslot_w(a, 0, gs[sl])[L.at(i, j0 + v)] = S(sl, v + 1)[i];
                }
                cluster.sync();  // no CTA leaves while its partner may still store into it
                return;
            }
        }
        stamp(3);
        if (!grid_barrier(gb, gen, &s_ok)) return;
        stamp(4);
        // ---- C: rows jlo .. jhi of T2 (the cluster's rows, the shadow row
        // below and the halo row above): DCT-III along i; afterwards X row x
        // holds psi = y / (4 m^2) (poisson.cpp:93) of row j0 - sh + x
        {
            const int per = e ? h : h + 1;
            for (int x = tid; x < VCc * per; x += kRsThreads) {
                int w, q;
                rs_split(x, per, w, q);
                const int pos = (q == h) ? 2 * h : (e ? h + q : q);
                F[w * hs + q] = __ldcg(T2 + L.at(pos, jlo + w));
            }
        }
        __syncthreads();
        dct3_half(VCc, F, [&](int w, int i, double val) {
            const int jj = jlo + w;
#pragma unroll
            for (int o = 0; o < 2; ++o) {
                const int j0o = base + o * R, nro = max(0, min(R, m - j0o));
                const int sho = (nro > 0 && j0o > 0) ? 1 : 0, hlo = (nro > 0 && j0o + nro < m) ? 1 : 0;
                const int xo = jj - (j0o - sho);
                if (nro > 0 && xo >= 0 && xo < sho + nro + hlo)
                    EOr[o][((size_t)(2 * xo) + e) * hs + i] = val;
            }
        });
        cluster.sync();
        for (int x = 0; x < sh + nr + hl; ++x)
            combine(x, [&](int i, double val) { X[x * ms + i] = scale * val; });
        __syncthreads();
        stamp(5);
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
            proj_unit_ball<QN>(wx, wy, qx, qy);
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
        stamp(6);
    }
}

}  // namespace w1mg_dev
