// pdhg_rspf.cuh -- the row-resident level-persistent PDHG engine of
// pdhg_rs.cuh for m = N1 N2 with odd coprime factors N1 <= 32, N2 <= 19
// (config 3's finest level: m = 513 = 27 x 19), where a dense DCT matrix no
// longer fits the register files: a register-stationary PRIME-FACTOR DCT.
//
// Transform (REDFT10 / REDFT01 of proj/src/poisson.cpp:35-38, 82-98), per
// vector of length m:
//   * Makhoul's reordering v[n] = x[2n] (n <= (m-1)/2), v[m-1-n] = x[2n+1]
//     turns the DCT-II into one length-m real DFT V, X_k = 2 Re(e^{-i pi k/2m}
//     V_k); the DCT-III runs it backwards from W_k = e^{i pi k/2m} (X_k - i
//     X_{m-k}).
//   * Good-Thomas: with n = (N2 n1 + N1 n2) mod m and k = (k mod N1, k mod
//     N2) the DFT is a twiddle-free N1 x N2 two-dimensional DFT.  Both index
//     maps are tables applied by whoever WRITES the data (the pre step / the
//     plane loads / the output stores), never a pass of their own.
//   * Stage over N1 (real input, outputs k1 < H1 = (N1+1)/2 by Hermitian
//     symmetry): lane o of a warp owns ONE output row (Re A[k1 = o] for o <
//     H1, Im A[k1 = o - T1] above) and keeps its T1 = (N1-1)/2 folded
//     twiddles in registers; a warp takes one column (vector, n2) at a time,
//     reading it by broadcast loads.  The same registers serve the inverse
//     stage (cos / sin are symmetric in (k1, n1)), whose two partial sums per
//     output pair are exchanged by one shuffle.
//   * Stage over N2 (complex): lane (u, kh) owns the output pair (kh, N2 - kh)
//     of one of three columns, folded over t <-> N2 - t, twiddles
//     cos / sin(2 pi kh t / N2) in registers; forward and inverse differ by
//     one sign.
// Five barrier-separated phases per transform pair become three short ones,
// every thread busy in each, no table lookups inside the sums.
//
// Iteration structure, shadow row, deferred stop rule and planes as in
// pdhg_rs.cuh; the spectral order is the natural k.  rho is read through the
// read-only path each iteration (it never changes during a level).
#pragma once

#include "pdhg_rs.cuh"

namespace w1mg_dev {

#ifndef W1MG_PF_THREADS
#define W1MG_PF_THREADS 384  // 12 warps, <= 170 registers: measured 26.2 us per 513^2 iteration (512: 27.1, 448: 27.7, 256: 29.3)
#endif
constexpr int kPfThreads = W1MG_PF_THREADS;  // threads per CTA of the prime-factor engine

template <int N1_, int N2_>
struct PfGeo {
    static constexpr int N1 = N1_, N2 = N2_, M = N1 * N2;
    static constexpr int H1 = N1 / 2 + 1, T1 = (N1 - 1) / 2, H2 = N2 / 2 + 1, T2 = (N2 - 1) / 2;
    static constexpr int N1P = (N1 + 2) & ~1;   // row of one column (vector, n2): n1 contiguous
    // rows of the stage buffers; the strides are chosen so that the lanes of a
    // store (one row per lane) fall into different shared-memory banks: 2 N2P
    // = 10 and B2R = 14 (mod 16 doubles) give at most two-way conflicts where
    // 2 N2P = 12 / 2 K1P = 12 gave four-way ones (21 % of the wavefronts in ncu)
    static constexpr int N2P = ((N2 + 2) & ~7) + 5;  // row of one (vector, k1, re/im): n2 or k2 contiguous (= 5 mod 8)
    static constexpr int K1P = (H1 + 1) & ~1;   // row of one (vector, n2, re/im): k1 contiguous
    static constexpr int GS = N2 * N1P;         // per-vector strides
    static constexpr int AS = H1 * 2 * N2P;
    static constexpr int B2R = 2 * K1P + 2;     // (re | im) row pair of one (vector, n2), even
    static constexpr int BS = N2 * B2R;
    static constexpr int GB = GS > BS ? GS : BS;
    static constexpr int NU = 32 / H2;          // columns per warp in the N2 stage
    static constexpr int NI0 = H1 * N2;         // items of the W build
    static constexpr int NTAB = M + N2 * N1P + N1 * N2 + 2 * NI0;  // shorts
    static_assert((N1 & 1) && (N2 & 1) && N1 <= 32 && NU >= 1 && (T1 & 1), "factor sizes");
};

// host + device: doubles of dynamic shared memory for R rows per CTA
template <class P>
__host__ __device__ inline size_t rspf_smem_doubles(int R) {
    const int ms = P::M + 1, V = R + 2;
    return (size_t)ms * (2 + 6 * (R + 1) + V) + (size_t)(P::NTAB + 3) / 4 + (size_t)V * (P::GB + P::AS) + 8;
}

// index tables (shorts), in this order: ginv[M] position of x_i in a vector's
// column block; idxg[N2*N1P] its inverse; crtk[N1*N2] k of (k1, k2); i0k /
// i0d[H1*N2] k and destination offset of the W build
template <class P>
inline void rspf_tables(short* t) {
    const int m = P::M;
    auto pos = [&](int n) { return n <= (m - 1) / 2 ? 2 * n : 2 * (m - 1 - n) + 1; };
    short* ginv = t;
    short* idxg = ginv + m;
    short* crtk = idxg + P::N2 * P::N1P;
    short* i0k = crtk + P::N1 * P::N2;
    short* i0d = i0k + P::NI0;
    for (int x = 0; x < P::N2 * P::N1P; ++x) idxg[x] = 0;
    for (int n1 = 0; n1 < P::N1; ++n1)
        for (int n2 = 0; n2 < P::N2; ++n2) {
            const int i = pos((P::N2 * n1 + P::N1 * n2) % m);
            ginv[i] = (short)(n2 * P::N1P + n1);
            idxg[n2 * P::N1P + n1] = (short)i;
        }
    for (int k = 0; k < m; ++k) crtk[(k % P::N1) * P::N2 + k % P::N2] = (short)k;
    for (int k1 = 0; k1 < P::H1; ++k1)
        for (int k2 = 0; k2 < P::N2; ++k2) {
            i0k[k1 * P::N2 + k2] = crtk[k1 * P::N2 + k2];
            i0d[k1 * P::N2 + k2] = (short)(k1 * 2 * P::N2P + k2);
        }
}

template <int QN, class P>
__global__ void __launch_bounds__(kPfThreads, 1)
pdhg_rspf_kernel(const SweepArgs a, const RsArgs ra, const short* __restrict__ gtab, GridBar gb) {
    extern __shared__ __align__(16) double rs_sm[];
    __shared__ int s_ok;
    __shared__ int s_stop;
    __shared__ double red[kPfThreads / 32][3];
    constexpr int N1 = P::N1, N2 = P::N2, H1 = P::H1, T1 = P::T1, H2 = P::H2, T2 = P::T2;
    constexpr int N1P = P::N1P, N2P = P::N2P, K1P = P::K1P, GS = P::GS, AS = P::AS, BS = P::BS;
    constexpr int m = P::M, n = m - 1, ms = m + 1;
    PairCtl* ctl = a.ctl;
    if (*(volatile int*)&ctl->done) return;
    if ((int)blockIdx.x >= ra.G) {  // reducer CTA(s): Eq. 12 sums and the stop rule
        rs_reducer(rs_red_args(a, ra), gb, (int)blockIdx.x == ra.G);
        return;
    }
    const int R = ra.R, G = ra.G;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, c = blockIdx.x;
    const int j0 = c * R, nr = min(R, m - j0);
    const int sh = c > 0 ? 1 : 0, hl = (j0 + nr < m) ? 1 : 0;
    const Layout L = a.L;
    const double mu = a.mu, tau = a.tau, ih = a.ih, scale = ra.scale;

    double* lam = rs_sm;
    double* cq = lam + ms;                                // cos(pi k / 2m), k <= m
    double* st = cq + ms;                                 // 6 x (R+1) rows
    double* X = st + (size_t)6 * (R + 1) * ms;            // (R+2) natural-order rows
    double* GBf = X + (size_t)(R + 2) * ms;               // column blocks / inverse N2-stage outputs
    double* A2 = GBf + (size_t)(R + 2) * P::GB;           // N1-stage outputs / W
    short* tab = reinterpret_cast<short*>(A2 + (size_t)(R + 2) * AS);
    const short* ginv = tab;
    const short* idxg = ginv + m;
    const short* crtk = idxg + N2 * N1P;
    const short* i0k = crtk + N1 * N2;
    const short* i0d = i0k + P::NI0;
    auto S = [&](int slot, int sv) { return st + (slot * (R + 1) + sv) * ms; };
    const double* rho = pslot(a, 0, P_RHO);

    // ---- twiddles in registers
    // N1 stage: lane o < H1: cos(2 pi o t / N1); H1 <= o < N1: -sin(2 pi (o-T1) t / N1)
    // (2 pi a / N1 = pi (4 N2 a) / 2m: exact indices into the cos(pi j / 2m) table)
    const bool isre = lane < H1;
    const int k1l = isre ? lane : lane - T1;
    double cw1[T1];
#pragma unroll
    for (int t = 1; t <= T1; ++t) {
        const int aa = (k1l * t) % N1;
        const int j = isre ? (4 * N2 * aa) % (4 * m) : (4 * N2 * aa + 4 * m - m) % (4 * m);
        const double w = __ldg(ra.cosq + j);
        cw1[t - 1] = (lane < N1) ? (isre ? w : -w) : 0.0;
    }
    // N2 stage: lane (u, kh)
    const int u2 = lane / H2, kh = lane - u2 * H2;
    double c2[T2], s2[T2];
#pragma unroll
    for (int t = 1; t <= T2; ++t) {
        const int aa = (kh * t) % N2;
        c2[t - 1] = __ldg(ra.cosq + (4 * N1 * aa) % (4 * m));
        s2[t - 1] = __ldg(ra.cosq + (4 * N1 * aa + 3 * m) % (4 * m));
    }

    // ---- level prologue
    for (int x = tid; x < m; x += kPfThreads) lam[x] = ra.lamq[x];
    for (int x = tid; x <= m; x += kPfThreads) cq[x] = ra.cosq[x];
    for (int x = tid; x < P::NTAB; x += kPfThreads) tab[x] = gtab[x];
    for (int x = tid; x < 6 * (R + 1) * ms; x += kPfThreads) st[x] = 0.0;
    for (int x = tid; x < (R + 2) * ms; x += kPfThreads) X[x] = 0.0;
    for (int x = tid; x < (R + 2) * (P::GB + AS); x += kPfThreads) GBf[x] = 0.0;
    __syncthreads();
    {
        const int gs[6] = {P_MX, P_MY, P_PX, P_PY, P_BX, P_BY};
        const int rows = nr + sh;
        for (int x = tid; x < 6 * rows * m; x += kPfThreads) {
            const int sl = x / (rows * m), rem = x - sl * rows * m, w = rem / m, i = rem - w * m;
            S(sl, w + 1 - sh)[i] = pslot(a, 0, gs[sl])[L.at(i, j0 - sh + w)];
        }
    }
    __syncthreads();

    // ---- transform stages
    // N1 stage forward: column blocks GBf[v][n2][n1] -> A2[v][k1][re/im][n2]
    auto stage1_fwd = [&](int V) {
        for (int col = warp; col < V * N2; col += kPfThreads / 32) {
            int v, n2;
            rs_split(col, N2, v, n2);
            // the column as 16-byte pairs e[a] = (g[2a], g[2a+1]); t and N1 - t meet
            // from both ends: two pairs feed two steps
            const double2* g2 = reinterpret_cast<const double2*>(GBf + v * P::GB + n2 * N1P);
            const double sgn = isre ? 1.0 : -1.0;
            double2 lo = g2[0], hi = g2[(N1 - 1) / 2];
            double acc = isre ? lo.x : 0.0;
            acc = fma(cw1[0], fma(sgn, hi.x, lo.y), acc);  // t = 1: g[1], g[N1-1]
#pragma unroll
            for (int aa = 1; aa <= (T1 - 1) / 2; ++aa) {
                lo = g2[aa];                    // g[2aa], g[2aa+1]
                hi = g2[(N1 - 1) / 2 - aa];     // g[N1-1-2aa], g[N1-2aa]
                acc = fma(cw1[2 * aa - 1], fma(sgn, hi.y, lo.x), acc);  // t = 2aa
                acc = fma(cw1[2 * aa], fma(sgn, hi.x, lo.y), acc);      // t = 2aa+1
            }
            double* o = A2 + v * AS + k1l * 2 * N2P + (isre ? 0 : N2P) + n2;
            if (lane < N1) *o = acc;
            if (lane == 0) o[N2P] = 0.0;  // Im A[0] = 0
        }
    };
    // N2 stage: rows A2[v][k1][re/im][.] folded over t <-> N2 - t; emit(v, k1, kh,
    // Cr, Ci, Sr, Si) with C = a_0 + sum (a_t + a_{N2-t}) cos, S = sum (a_t - a_{N2-t}) sin
    auto stage2 = [&](int V, auto emit) {
        const int ncol = V * H1;
        for (int cb = warp * P::NU; cb < ncol; cb += (kPfThreads / 32) * P::NU) {
            const int col = cb + u2;
            const bool on = u2 < P::NU && col < ncol;
            const int cc = on ? col : 0;
            const int v = cc / H1, k1 = cc - v * H1;
            const double* ar = A2 + v * AS + k1 * 2 * N2P;
            const double* ai = ar + N2P;
            double Cr = ar[0], Ci = ai[0], Sr = 0.0, Si = 0.0;
#pragma unroll
            for (int t = 1; t <= T2; ++t) {
                const double pr = ar[t], qr = ar[N2 - t], pi = ai[t], qi = ai[N2 - t];
                Cr = fma(c2[t - 1], pr + qr, Cr);
                Ci = fma(c2[t - 1], pi + qi, Ci);
                Sr = fma(s2[t - 1], pr - qr, Sr);
                Si = fma(s2[t - 1], pi - qi, Si);
            }
            if (on) emit(v, k1, Cr, Ci, Sr, Si);
        }
    };
    // forward N2 stage + Makhoul twiddle: V[k2] = C - iS, V[N2-k2] = C + iS, the
    // rows k1 >= H1 by V[N1-k1][N2-k2] = conj V[k1][k2]; X_k = 2 (cos Re V + sin Im V)
    auto stage2_fwd = [&](int V, auto out) {
        stage2(V, [&](int v, int k1, double Cr, double Ci, double Sr, double Si) {
            const double ar = Cr + Si, ai = Ci - Sr, br = Cr - Si, bi = Ci + Sr;
            int kk = crtk[k1 * N2 + kh];
            out(v, kk, 2.0 * (cq[kk] * ar + cq[m - kk] * ai));
            if (kh > 0) {
                kk = crtk[k1 * N2 + N2 - kh];
                out(v, kk, 2.0 * (cq[kk] * br + cq[m - kk] * bi));
            }
            if (k1 > 0) {
                kk = crtk[(N1 - k1) * N2 + (kh ? N2 - kh : 0)];
                out(v, kk, 2.0 * (cq[kk] * ar - cq[m - kk] * ai));
                if (kh > 0) {
                    kk = crtk[(N1 - k1) * N2 + kh];
                    out(v, kk, 2.0 * (cq[kk] * br - cq[m - kk] * bi));
                }
            }
        });
    };
    // W build: natural-order spectra X[v][k] -> A2[v][k1][re/im][k2], k1 < H1
    auto build_w = [&](int V) {
        for (int x = tid; x < V * P::NI0; x += kPfThreads) {
            int v, it;
            rs_split(x, P::NI0, v, it);
            const int kk = i0k[it];
            const double* xv = X + v * ms;
            const double p = xv[kk], q = kk ? xv[m - kk] : 0.0;
            const double cs = cq[kk], sn = cq[m - kk];
            double* o = A2 + v * AS + i0d[it];
            o[0] = cs * p + sn * q;
            o[N2P] = sn * p - cs * q;
        }
    };
    // inverse N2 stage: b[n2] = C + iS, b[N2-n2] = C - iS -> GBf[v][n2][re/im][k1]
    auto stage2_inv = [&](int V) {
        stage2(V, [&](int v, int k1, double Cr, double Ci, double Sr, double Si) {
            double* o = GBf + v * P::GB + kh * P::B2R + k1;
            o[0] = Cr - Si;
            o[K1P] = Ci + Sr;
            if (kh > 0) {
                double* o2 = GBf + v * P::GB + (N2 - kh) * P::B2R + k1;
                o2[0] = Cr + Si;
                o2[K1P] = Ci - Sr;
            }
        });
    };
    // inverse N1 stage: v[n1] = b_0 + 2 sum_k1 (Re b cos - Im b sin); the cos lane
    // a and the sin lane a + T1 swap their sums: out(v, i, y_i)
    auto stage1_inv = [&](int V, auto out) {
        for (int col = warp; col < V * N2; col += kPfThreads / 32) {
            int v, n2;
            rs_split(col, N2, v, n2);
            const double* br = GBf + v * P::GB + n2 * P::B2R;
            const double2* s2p = reinterpret_cast<const double2*>(isre ? br : br + K1P);
            double acc = 0.0;
            {
                const double2 e0 = s2p[0];
                acc = cw1[0] * e0.y;  // t = 1
#pragma unroll
                for (int aa = 1; aa <= (T1 - 1) / 2; ++aa) {
                    const double2 ee = s2p[aa];
                    acc = fma(cw1[2 * aa - 1], ee.x, acc);
                    acc = fma(cw1[2 * aa], ee.y, acc);
                }
            }
            const int peer = isre ? lane + T1 : lane - T1;
            const double oth = __shfl_sync(0xffffffffu, acc, peer & 31);
            const double b0 = br[0];
            double val;
            int n1;
            if (lane == 0) {
                val = b0 + 2.0 * acc;
                n1 = 0;
            } else if (isre) {
                val = b0 + 2.0 * (acc + oth);
                n1 = lane;
            } else {
                val = b0 + 2.0 * (oth - acc);
                n1 = N1 - k1l;
            }
            if (lane < N1) out(v, (int)idxg[n2 * N1P + n1], val);
        }
    };

    double* T1p = pslot_w(a, 0, P_T);    // T1[k1][j] at L.at(j, k1)
    double* T2p = pslot_w(a, 0, P_PSI);  // T2[j][k1] at L.at(k1, j)
    unsigned gen = 0;
    long iter = 0;
    auto stamp = [&](int q) {
        if (ra.stamps && c == 0 && tid == 0 && iter < 64) ra.stamps[iter * kRsStampSlots + q] = gtimer();
    };

    for (;; ++iter) {
        stamp(0);
        // ---- A: r = A v - rho on the owned rows (poisson.cpp:113-115), DCT-II along i -> T1
        for (int x = tid; x < nr * m; x += kPfThreads) {
            int v, i;
            rs_split(x, m, v, i);
            const int j = j0 + v, sv = v + 1;
            const double rr = __ldg(rho + L.at(i, j));
            const double* mx = S(0, sv);
            const double* bx = S(4, sv);
            const double r_ = (i < n) ? mx[i] - mu * bx[i] : 0.0;
            const double l_ = (i > 0) ? mx[i - 1] - mu * bx[i - 1] : 0.0;
            const double a_ = (j < n) ? S(1, sv)[i] - mu * S(5, sv)[i] : 0.0;
            const double b_ = (j > 0) ? S(1, sv - 1)[i] - mu * S(5, sv - 1)[i] : 0.0;
            const double div = (r_ - l_) * ih + (a_ - b_) * ih;
            GBf[v * P::GB + ginv[i]] = div - rr;
        }
        __syncthreads();
        stamp(1);
        stage1_fwd(nr);
        __syncthreads();
        stamp(2);
        stage2_fwd(nr, [&](int v, int kk, double val) { T1p[L.at(j0 + v, kk)] = val; });
        stamp(11);
        if (!grid_barrier(gb, gen, &s_ok)) return;
        stamp(12);
        // ---- B: columns k1 = j0 + v: DCT-II along j, divide by lambda_k1 +
        // lambda_k2 (poisson.cpp:84-89), DCT-III along j -> T2
        for (int x = tid; x < nr * m; x += kPfThreads) {
            int v, j;
            rs_split(x, m, v, j);
            GBf[v * P::GB + ginv[j]] = __ldcg(T1p + L.at(j, j0 + v));
        }
        __syncthreads();
        stamp(5);
        stage1_fwd(nr);
        __syncthreads();
        stamp(6);
        stage2_fwd(nr, [&](int v, int kk, double val) {
            const int p1 = j0 + v;
            X[v * ms + kk] = (p1 == 0 && kk == 0) ? 0.0 : val / (lam[p1] + lam[kk]);
        });
        __syncthreads();
        stamp(7);
        build_w(nr);
        __syncthreads();
        stamp(8);
        stage2_inv(nr);
        __syncthreads();
        stamp(9);
        stage1_inv(nr, [&](int v, int j, double val) { T2p[L.at(j0 + v, j)] = val; });
        stamp(10);
        stamp(11);
        if (!grid_barrier(gb, gen, &s_ok)) return;
        stamp(12);
        // ---- C: rows j0-sh .. j0+nr-1+hl of T2: DCT-III along i; afterwards X
        // row w holds psi = y / (4 m^2) (poisson.cpp:93) of row j0 - sh + w
        int decv = 0;  // the reducer's decision: requested now, consumed after the row loads
        if (iter > 0 && tid == 0) decv = __ldcg(ra.dec + (iter & 1));
        const int nh = sh + nr + hl;
        for (int x = tid; x < nh * m; x += kPfThreads) {
            int w, kk;
            rs_split(x, m, w, kk);
            X[w * ms + kk] = __ldcg(T2p + L.at(kk, j0 - sh + w));
        }
        if (tid == 0) s_stop = decv;
        __syncthreads();
        if (iter > 0 && s_stop) {  // iteration iter-1 met the stop rule: its state is final
                const int gs[6] = {P_MX, P_MY, P_PX, P_PY, P_BX, P_BY};
                for (int x = tid; x < 6 * nr * m; x += kPfThreads) {
                    const int sl = x / (nr * m), rem = x - sl * nr * m, v = rem / m, i = rem - v * m;
                    pslot_w(a, 0, gs[sl])[L.at(i, j0 + v)] = S(sl, v + 1)[i];
                }
            return;
        }
        stamp(13);
        build_w(nh);
        __syncthreads();
        stamp(14);
        stage2_inv(nh);
        __syncthreads();
        stamp(15);
        stage1_inv(nh, [&](int w, int i, double val) { X[w * ms + i] = scale * val; });
        __syncthreads();
        stamp(16);
        // ---- D: post step (pdhg_post_kernel's arithmetic) on the shadow and
        // owned rows; Eq. 12 partial sums over the owned rows only
        double s_dm2 = 0.0, s_dp2 = 0.0, s_cr = 0.0;
        for (int x = tid; x < (nr + sh) * m; x += kPfThreads) {
            int w, i;
            rs_split(x, m, w, i);
            const int sv = w + 1 - sh, j = j0 + sv - 1;
            const bool hx = i < n, hy = j < n, mine = sv > 0;
            const double pc = X[w * ms + i];
            double mnx = 0.0, mny = 0.0, dmx = 0.0, dmy = 0.0, pox = 0.0, poy = 0.0;
            if (hx) {
                const double mo = S(0, sv)[i];
                const double vv = mo - mu * S(4, sv)[i];
                mnx = vv - (pc - X[w * ms + i + 1]) * ih;  // poisson.cpp:124
                dmx = mnx - mo;
                pox = S(2, sv)[i];
            }
            if (hy) {
                const double mo = S(1, sv)[i];
                const double vv = mo - mu * S(5, sv)[i];
                mny = vv - (pc - X[(w + 1) * ms + i]) * ih;  // poisson.cpp:130
                dmy = mny - mo;
                poy = S(3, sv)[i];
            }
            const double wx = hx ? pox + tau * mnx : 0.0;
            const double wy = hy ? poy + tau * mny : 0.0;
            double qx, qy;
            rs_proj_unit_ball<QN>(wx, wy, qx, qy);
            if (hx) {
                S(0, sv)[i] = mnx;
                S(2, sv)[i] = qx;
                S(4, sv)[i] = 2.0 * qx - pox;
                if (mine) {
                    const double dp = qx - pox;
                    s_dm2 += dmx * dmx;
                    s_dp2 += dp * dp;
                    s_cr += dp * dmx;
                }
            }
            if (hy) {
                S(1, sv)[i] = mny;
                S(3, sv)[i] = qy;
                S(5, sv)[i] = 2.0 * qy - poy;
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
            red[warp][0] = s_dm2;
            red[warp][1] = s_dp2;
            red[warp][2] = s_cr;
        }
        __syncthreads();  // state rows and red[] complete
        if (tid == 0) {
            double t0 = 0.0, t1 = 0.0, t2 = 0.0;
            for (int w = 0; w < kPfThreads / 32; ++w) {
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
