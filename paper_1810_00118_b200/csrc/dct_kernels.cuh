// dct_kernels.cuh -- hand-written fp64 DCT-II / DCT-III for the Neumann
// Poisson solve of G-prox PDHG (sm_100a), replacing the reference's FFTW
// REDFT10 / REDFT01 plans (proj/src/poisson.cpp:35-38, 82-98):
//
//   REDFT10 (DCT-II):  X_k = 2 sum_i x_i cos(pi k (2i+1) / 2m)
//   REDFT01 (DCT-III): y_i = X_0 + 2 sum_{k>=1} X_k cos(pi k (2i+1) / 2m)
//
// on m = n+1 node rows / columns (odd at every config: 33 ... 4097).
//
// Algorithm (per 1-D vector of length m, all in shared memory):
//   * Makhoul's reordering turns the DCT-II into one length-m DFT of the real
//     sequence v[n] = x[2n] (n <= (m-1)/2), v[m-1-n] = x[2n+1], followed by
//     X_k = 2 Re(e^{-i pi k/2m} V_k); the DCT-III runs the same steps
//     backwards (W_k = e^{i pi k/2m}(X_k - i X_{m-k}), real inverse DFT,
//     un-reorder).
//   * The length-m DFT is a prime-factor (Good-Thomas) split m = N1 N2 with
//     coprime N1 >= N2 (513 = 27 x 19, 257 prime, 129 = 43 x 3, 65 = 13 x 5):
//     no twiddles between the stages, input map n = (N2 n1 + N1 n2) mod m,
//     output map by the CRT.
//   * Each stage is a direct DFT whose symmetric (cos) and antisymmetric (sin)
//     halves are folded first (x_t +- x_{N-t}), so a stage is two small real
//     GEMMs  [twiddles] x [folded vectors]; real input halves stage 1 and
//     Hermitian symmetry halves stage 2.  The GEMMs run from shared memory
//     with 4 x 4 register tiles (twiddle tables read through L1, broadcast
//     across a warp).
//   At m = 513 one vector costs ~16.5k fp64 FMA (the dense folded DCT matrix
//   costs 132k), at m = 257 (prime) ~33k.
//
// Kernels of one Poisson solve / PDHG iteration (the 2-D transform is
// separable: rows along i, columns along j):
//   dct_rows_fwd_kernel<MODE>  rows: (MODE 1: r = A v - rho, the PDHG pre
//                              step, formed on the fly) -> DCT-II along i -> T
//   dct_cols_kernel            columns of T: DCT-II along j, divide by
//                              lambda_k1 + lambda_k2 (constant mode -> 0),
//                              DCT-III along j -> T
//   dct_rows_inv_kernel<MODE>  rows of T: DCT-III along i, x 1/(4 m^2) = psi;
//                              MODE 0 stores psi, MODE 1 runs the PDHG post
//                              step (m, varphi, varphi_bar, Eq. 12 partials,
//                              stop rule) on the rows with psi from shared
//                              memory (one extra row transformed for the
//                              y-difference).
// A vector's transform depends only on its own data (fixed operation order),
// so the extra row a CTA recomputes carries the same bits as its owner's.
#pragma once

#include "pdhg_kernels.cuh"

namespace w1mg_dev {

// H = N/2 + 1 outputs of a real length-N DFT, T = (N-1)/2 symmetric pairs
// (t, N-t), E = 1 for even N: the Nyquist element N/2 enters once, as an
// extra row T of the cosine GEMM (its twiddle cos(2 pi (N/2) k / N) = (-1)^k
// is the natural continuation of the table index).
//
// Twiddles are never stored as matrices: the GEMM operand A(t, k) of a stage
// over a factor N is +-tab[((t+1) k) mod N] with tab = cos / sin of 2 pi j/N,
// so a CTA stages only 2 (N1 + N2) + 2 m doubles (and the index maps) in
// shared memory -- 9 KB at m = 513, 4 KB at the prime m = 257, where a dense
// twiddle matrix would be 270 KB.
struct DctPlan {
    int m, N1, N2, H1, T1, E1, H2, T2, E2, H1p, H2p;
    const double* tw1;  // [2][N1] cos, sin of 2 pi j / N1
    const double* tw2;  // [2][N2] cos, sin of 2 pi j / N2
    const double* mk;   // [2m] cos, sin of pi k / 2m (interleaved)
    const short* idxA;  // [N2][N1] row position of v[(N2 t + N1 n2) mod m]
    const short* crt;   // [N2][H1] k with k mod N1 = k1 and k mod N2 = k2
    const int* f5;      // [m] output map of the forward transform: k1 | q << 16 |
                        // (k2 >= H2) << 29 | (k1 >= H1: conjugate partner) << 30
    const double* tabs; // the tables above as one contiguous block (smem layout)
};

__host__ __device__ inline int round4(int x) { return (x + 3) & ~3; }

// doubles of the staged tables: tw1, tw2, mk, then the short index maps
__host__ __device__ inline int dct_tab_doubles(const DctPlan& p) {
    const int d = 2 * p.N1 + 2 * p.N2 + 2 * p.m;
    const int sh = round4(p.N2 * p.N1 + p.N2 * p.H1);  // shorts, keeps f5 4-B aligned
    return round4(d + sh / 4 + (p.m + 1) / 2);
}

// Shared-memory arenas (doubles) for NV vectors: P and Q (ping-pong scratch
// of the stages), then X (NV x m); the staged tables come first.
__host__ __device__ inline void dct_arena(const DctPlan& p, int NV, int& szP, int& szQ) {
    const int NpA = round4(NV * p.N2);
    szP = (2 * p.T1 + 1 + p.E1) * NpA;
    szQ = 2 * p.H1p * NpA;
    if (p.N2 > 1) {
        const int W2 = 2 * round4(NV * p.H1);
        const int b2 = (2 * p.T2 + 1 + p.E2) * W2;
        szP = szP > b2 ? szP : b2;
        szQ = szQ > 2 * p.H2p * W2 ? szQ : 2 * p.H2p * W2;
    }
    szP = round4(szP);
    szQ = round4(szQ);
}

// row stride of X: even, so every row starts 16-B aligned (bulk copies)
__host__ __device__ inline int dct_xs(const DctPlan& p) { return (p.m + 1) & ~1; }

__host__ __device__ inline size_t dct_smem_bytes(const DctPlan& p, int NV) {
    int a, b;
    dct_arena(p, NV, a, b);
    return sizeof(double) * ((size_t)dct_tab_doubles(p) + a + b + (size_t)NV * dct_xs(p));
}

// Loop over e = threadIdx.x + q blockDim.x < NA * NB as (a, b) = (e / NB,
// e % NB) with one division per thread (at the start), not one per item:
// the kernels are latency-bound chains of short phases, and per-item integer
// divisions were most of their instructions (ncu).
#define W1MG_FOR2(a, b, NA, NB)                                                           \
    for (int a = (int)threadIdx.x / (NB), b = (int)threadIdx.x - a * (NB),                \
             a##_d = (int)blockDim.x / (NB), b##_d = (int)blockDim.x - a##_d * (NB);      \
         a < (NA); a += a##_d, b += b##_d, (b >= (NB) ? (b -= (NB), ++a) : 0))

__device__ __forceinline__ double lds(const double* p) {
    double v;
    asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
    return v;
}
__device__ __forceinline__ double2 lds2(const double* p) {
    double2 v;
    asm("ld.shared.v2.f64 {%0, %1}, [%2];"
        : "=d"(v.x), "=d"(v.y)
        : "r"((unsigned)__cvta_generic_to_shared(p)));
    return v;
}

// The two GEMMs of one real-DFT stage over a factor N, sharing the twiddle
// index walk:
//   C1[k][j] = (C0 ? C0[j] : 0) + sum_{t<K1} cos(2 pi ((t+1) k mod N)/N) B1[t][j]
//   C2[k][j] = s2 sum_{t<K2} sin(2 pi ((t+1) k mod N)/N) B2[t][j]
// for k < Mp, j < Np (K1 = K2 or K2 + 1: the Nyquist row is cosine-only).
// tab = [cos | sin] of N entries, in shared memory like B1, B2, C1, C2, C0.
// Wide: 4 x 4 register tiles per matrix (lanes of a warp share the rows, so
// the twiddle loads broadcast).  Thin: one (k, j) per thread over the first
// Nr <= Np columns only (the padded columns of a one-vector transform are
// not computed).  k < Mp <= N + 3: k mod N is a conditional subtraction.
__device__ __noinline__ void tgemm2(const double* tab, int N, int Mp, int K1, int K2,
                                    const double* B1, const double* B2, int ldb, int Np, int Nr,
                                    double* C1, double* C2, int ldc, const double* C0, double s2) {
    const int Nt = Np >> 2, Mt = Mp >> 2;
    const double* ts = tab + N;
    if (4 * Mt * Nt >= (int)blockDim.x) {
        W1MG_FOR2(ti, tj, Mt, Nt) {
            int kr[4], ix[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                int k = 4 * ti + r;
                k -= (k >= N) ? N : 0;
                k -= (k >= N) ? N : 0;
                kr[r] = k;
                ix[r] = k;
            }
            double c[4][4], d[4][4];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int q = 0; q < 4; ++q) c[r][q] = d[r][q] = 0.0;
            const double* b1 = B1 + 4 * tj;
            const double* b2 = B2 + 4 * tj;
#pragma unroll 2
            for (int t = 0; t < K1; ++t) {
                const bool two = t < K2;
                const double2 x01 = lds2(b1 + t * ldb), x23 = lds2(b1 + t * ldb + 2);
                double2 y01 = make_double2(0.0, 0.0), y23 = y01;
                if (two) {
                    y01 = lds2(b2 + t * ldb);
                    y23 = lds2(b2 + t * ldb + 2);
                }
                const double xv[4] = {x01.x, x01.y, x23.x, x23.y};
                const double yv[4] = {y01.x, y01.y, y23.x, y23.y};
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const double cw = lds(tab + ix[r]), sw = lds(ts + ix[r]);
                    ix[r] += kr[r];
                    ix[r] -= (ix[r] >= N) ? N : 0;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        c[r][q] = fma(cw, xv[q], c[r][q]);
                        d[r][q] = fma(sw, yv[q], d[r][q]);
                    }
                }
            }
            double c0[4] = {0.0, 0.0, 0.0, 0.0};
            if (C0) {
                const double2 z01 = lds2(C0 + 4 * tj), z23 = lds2(C0 + 4 * tj + 2);
                c0[0] = z01.x;
                c0[1] = z01.y;
                c0[2] = z23.x;
                c0[3] = z23.y;
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                double* o1 = C1 + (4 * ti + r) * ldc + 4 * tj;
                double* o2 = C2 + (4 * ti + r) * ldc + 4 * tj;
                *reinterpret_cast<double2*>(o1) = make_double2(c0[0] + c[r][0], c0[1] + c[r][1]);
                *reinterpret_cast<double2*>(o1 + 2) = make_double2(c0[2] + c[r][2], c0[3] + c[r][3]);
                *reinterpret_cast<double2*>(o2) = make_double2(s2 * d[r][0], s2 * d[r][1]);
                *reinterpret_cast<double2*>(o2 + 2) = make_double2(s2 * d[r][2], s2 * d[r][3]);
            }
        }
    } else {
        W1MG_FOR2(k, j, Mp, Nr) {
            int kr = k;
            kr -= (kr >= N) ? N : 0;
            kr -= (kr >= N) ? N : 0;
            int ix = kr;
            double c = 0.0, d = 0.0;
            const double* b1 = B1 + j;
            const double* b2 = B2 + j;
            // four steps per trip: the index walk and 16 independent shared
            // loads issue before the FMAs, two accumulator pairs
            double c1 = 0.0, d1 = 0.0;
            int t = 0;
            for (; t + 3 < K2; t += 4) {
                int i4[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    i4[u] = ix;
                    ix += kr;
                    ix -= (ix >= N) ? N : 0;
                }
                double cw[4], sw[4], x1[4], x2[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    cw[u] = lds(tab + i4[u]);
                    sw[u] = lds(ts + i4[u]);
                    x1[u] = lds(b1 + (t + u) * ldb);
                    x2[u] = lds(b2 + (t + u) * ldb);
                }
                c = fma(cw[0], x1[0], c);
                d = fma(sw[0], x2[0], d);
                c1 = fma(cw[1], x1[1], c1);
                d1 = fma(sw[1], x2[1], d1);
                c = fma(cw[2], x1[2], c);
                d = fma(sw[2], x2[2], d);
                c1 = fma(cw[3], x1[3], c1);
                d1 = fma(sw[3], x2[3], d1);
            }
            for (; t < K2; ++t) {
                const double cw = lds(tab + ix), sw = lds(ts + ix);
                ix += kr;
                ix -= (ix >= N) ? N : 0;
                c = fma(cw, lds(b1 + t * ldb), c);
                d = fma(sw, lds(b2 + t * ldb), d);
            }
            if (t < K1) c = fma(lds(tab + ix), lds(b1 + t * ldb), c);
            c += c1;
            d += d1;
            C1[k * ldc + j] = (C0 ? lds(C0 + j) : 0.0) + c;
            C2[k * ldc + j] = s2 * d;
        }
    }
}

// Smem view of the staged table block (same layout as p.tabs in global).
__device__ __forceinline__ DctPlan dct_view(const DctPlan& g, double* sm) {
    DctPlan p = g;
    p.tw1 = sm;
    p.tw2 = sm + 2 * g.N1;
    p.mk = p.tw2 + 2 * g.N2;
    p.idxA = reinterpret_cast<const short*>(p.mk + 2 * g.m);
    p.crt = p.idxA + g.N2 * g.N1;
    p.f5 = reinterpret_cast<const int*>(p.idxA + round4(g.N2 * g.N1 + g.N2 * g.H1));
    return p;
}

// Forward DCT-II of NV vectors X[v*xs + i] in place (P, Q scratch).  NV is a
// power of two (lg = log2 NV): vector indices split by shifts.
__device__ __noinline__ void dct2_vectors(const DctPlan& p, int NV, int xs, double* X, double* P,
                                          double* Q) {
    const int N1 = p.N1, N2 = p.N2, H1 = p.H1, T1 = p.T1, E1 = p.E1;
    const int lg = __ffs(NV) - 1, msk = NV - 1;
    const int NA = NV * N2, NpA = round4(NA);
    // stage 1 fold: X0 = x_0, S_t = x_t + x_{N1-t}, D_t = x_t - x_{N1-t}
    // (S row T1 = x_{N1/2} for even N1); vector j = n2 NV + v
    double* SA = P;
    double* DA = P + (T1 + E1) * NpA;
    double* X0 = DA + T1 * NpA;
    W1MG_FOR2(t, j, T1 + 1 + E1, NpA) {
        double s = 0.0, d = 0.0;
        if (j < NA) {
            const short* ix = p.idxA + (j >> lg) * N1;
            const double* xv = X + (j & msk) * xs;
            if (t == 0 || t > T1) {
                s = xv[ix[t]];
            } else {
                const double x0 = xv[ix[t]], x1 = xv[ix[N1 - t]];
                s = x0 + x1;
                d = x0 - x1;
            }
        }
        if (t == 0) {
            X0[j] = s;
        } else {
            SA[(t - 1) * NpA + j] = s;
            if (t <= T1) DA[(t - 1) * NpA + j] = d;
        }
    }
    __syncthreads();
    // stage 1: A[k1][j] = X0 + sum cos S - i sum sin D, k1 < H1
    double* ReA = Q;
    double* ImA = Q + p.H1p * NpA;
    tgemm2(p.tw1, N1, p.H1p, T1 + E1, T1, SA, DA, NpA, NpA, NA, ReA, ImA, NpA, X0, -1.0);
    __syncthreads();
    const int NB = NV * H1, NpB = round4(NB), W2 = 2 * NpB;
    double* Cp = Q;
    double* Sn = Q + p.H2p * W2;
    if (N2 > 1) {
        // stage 2 fold over n2 of the complex A[k1][n2 NV + v]; vector jb = k1 NV + v,
        // real parts in columns [0, NpB), imaginary parts in [NpB, 2 NpB)
        const int T2 = p.T2, E2 = p.E2;
        double* SB = P;
        double* DB = P + (T2 + E2) * W2;
        double* A0 = DB + T2 * W2;
        W1MG_FOR2(t, jb, T2 + 1 + E2, NpB) {
            double sr = 0.0, si = 0.0, dr = 0.0, di = 0.0;
            if (jb < NB) {
                const int k1 = jb >> lg, v = jb & msk;
                const double* re = ReA + k1 * NpA;
                const double* im = ImA + k1 * NpA;
                if (t == 0 || t > T2) {
                    sr = re[(t << lg) + v];
                    si = im[(t << lg) + v];
                } else {
                    const int ja = (t << lg) + v, jc = ((N2 - t) << lg) + v;
                    sr = re[ja] + re[jc];
                    si = im[ja] + im[jc];
                    dr = re[ja] - re[jc];
                    di = im[ja] - im[jc];
                }
            }
            if (t == 0) {
                A0[jb] = sr;
                A0[NpB + jb] = si;
            } else {
                double* sp = SB + (t - 1) * W2;
                sp[jb] = sr;
                sp[NpB + jb] = si;
                if (t <= T2) {
                    double* dp = DB + (t - 1) * W2;
                    dp[jb] = dr;
                    dp[NpB + jb] = di;
                }
            }
        }
        __syncthreads();
        tgemm2(p.tw2, N2, p.H2p, T2 + E2, T2, SB, DB, W2, W2, W2, Cp, Sn, W2, A0, 1.0);
        __syncthreads();
    }
    // V[k1, k2] = Cp - i Sn (k2 < H2), V[k1, N2 - k2] = Cp + i Sn; V[m-k] = conj V[k];
    // X_k = 2 (cos(pi k/2m) Re V_k + sin(pi k/2m) Im V_k); the (k1, row, flags)
    // of every k come from the plan's f5 map
    W1MG_FOR2(v, k, NV, p.m) {
        const int f = p.f5[k];
        const int k1 = f & 0xffff, q = (f >> 16) & 0x1fff;
        double vr, vi;
        if (N2 == 1) {
            vr = ReA[k1 * NpA + v];
            vi = ImA[k1 * NpA + v];
        } else {
            const int jb = (k1 << lg) + v;
            const double* cp = Cp + q * W2;
            const double* sn = Sn + q * W2;
            if (!(f & (1 << 29))) {
                vr = cp[jb] + sn[NpB + jb];
                vi = cp[NpB + jb] - sn[jb];
            } else {
                vr = cp[jb] - sn[NpB + jb];
                vi = cp[NpB + jb] + sn[jb];
            }
        }
        if (f & (1 << 30)) vi = -vi;
        const double c = p.mk[2 * k], sk = p.mk[2 * k + 1];
        X[v * xs + k] = 2.0 * (c * vr + sk * vi);
    }
    __syncthreads();
}

// W_k = e^{i pi k/2m} (X_k - i X_{m-k}), X_m = 0
__device__ __forceinline__ void dct3_w(const DctPlan& p, const double* x, int k, double& wr,
                                       double& wi) {
    const double a = x[k], b = k ? x[p.m - k] : 0.0;
    const double c = p.mk[2 * k], s = p.mk[2 * k + 1];
    wr = c * a + s * b;
    wi = s * a - c * b;
}

// DCT-III of NV vectors X[v*xs + k] in place (P, Q scratch); NV a power of two.
__device__ __noinline__ void dct3_vectors(const DctPlan& p, int NV, int xs, double* X, double* P,
                                          double* Q) {
    const int N1 = p.N1, N2 = p.N2, H1 = p.H1, T1 = p.T1, E1 = p.E1;
    const int lg = __ffs(NV) - 1, msk = NV - 1;
    const int NA = NV * N2, NpA = round4(NA);
    // stage 1 inputs: BR / BI rows k1 = 1..T1 (BR row T1: Nyquist k1 = N1/2,
    // halved: it enters the real inverse DFT once), B0 = Re b[0]
    double* BR = P;
    double* BI = P + (T1 + E1) * NpA;
    double* B0 = BI + T1 * NpA;
    if (N2 == 1) {
        W1MG_FOR2(t, j, H1, NpA) {
            double wr = 0.0, wi = 0.0;
            if (j < NV) dct3_w(p, X + j * xs, t, wr, wi);
            if (t == 0) {
                B0[j] = wr;
            } else {
                BR[(t - 1) * NpA + j] = (t <= T1) ? wr : 0.5 * wr;
                if (t <= T1) BI[(t - 1) * NpA + j] = wi;
            }
        }
        __syncthreads();
    } else {
        // stage 2 (inverse, over k2): fold W[k1, t] +- W[k1, N2-t] for k1 < H1
        const int T2 = p.T2, E2 = p.E2, NB = NV * H1, NpB = round4(NB), W2 = 2 * NpB, H2 = p.H2;
        double* SB = P;
        double* DB = P + (T2 + E2) * W2;
        double* A0 = DB + T2 * W2;
        W1MG_FOR2(t, jb, T2 + 1 + E2, NpB) {
            double sr = 0.0, si = 0.0, dr = 0.0, di = 0.0;
            if (jb < NB) {
                const int k1 = jb >> lg, v = jb & msk;
                const double* x = X + v * xs;
                if (t == 0 || t > T2) {
                    dct3_w(p, x, p.crt[t * H1 + k1], sr, si);
                } else {
                    double ar, ai, br, bi;
                    dct3_w(p, x, p.crt[t * H1 + k1], ar, ai);
                    dct3_w(p, x, p.crt[(N2 - t) * H1 + k1], br, bi);
                    sr = ar + br;
                    si = ai + bi;
                    dr = ar - br;
                    di = ai - bi;
                }
            }
            if (t == 0) {
                A0[jb] = sr;
                A0[NpB + jb] = si;
            } else {
                double* sp = SB + (t - 1) * W2;
                sp[jb] = sr;
                sp[NpB + jb] = si;
                if (t <= T2) {
                    double* dp = DB + (t - 1) * W2;
                    dp[jb] = dr;
                    dp[NpB + jb] = di;
                }
            }
        }
        __syncthreads();
        double* Cp = Q;
        double* Sn = Q + p.H2p * W2;
        tgemm2(p.tw2, N2, p.H2p, T2 + E2, T2, SB, DB, W2, W2, W2, Cp, Sn, W2, A0, 1.0);
        __syncthreads();
        // b[k1][n2] = Cp + i Sn (n2 < H2), b[k1][N2 - n2] = Cp - i Sn -> stage 1 inputs
        // (vector j = n2 NV + v)
        W1MG_FOR2(t, j, H1, NpA) {
            double br = 0.0, bi = 0.0;
            if (j < NA) {
                const int n2 = j >> lg, jb = (t << lg) + (j & msk);
                if (n2 < H2) {
                    const double* cp = Cp + n2 * W2;
                    const double* sn = Sn + n2 * W2;
                    br = cp[jb] - sn[NpB + jb];
                    bi = cp[NpB + jb] + sn[jb];
                } else {
                    const double* cp = Cp + (N2 - n2) * W2;
                    const double* sn = Sn + (N2 - n2) * W2;
                    br = cp[jb] + sn[NpB + jb];
                    bi = cp[NpB + jb] - sn[jb];
                }
            }
            if (t == 0) {
                B0[j] = br;
            } else {
                BR[(t - 1) * NpA + j] = (t <= T1) ? br : 0.5 * br;
                if (t <= T1) BI[(t - 1) * NpA + j] = bi;
            }
        }
        __syncthreads();
    }
    // stage 1 (inverse, over k1): w[n1] = b0 + 2 (P - Q), w[N1 - n1] = b0 + 2 (P + Q)
    double* PP = Q;
    double* QQ = Q + p.H1p * NpA;
    tgemm2(p.tw1, N1, p.H1p, T1 + E1, T1, BR, BI, NpA, NpA, NA, PP, QQ, NpA, nullptr, 1.0);
    __syncthreads();
    // un-reorder: n = (N2 n1 + N1 n2) mod m -> y at idxA[n2][n1] (the forward
    // input map); r = n2 N1 + n1
    W1MG_FOR2(n2, q, N2, N1 << lg) {
        const int n1 = q >> lg, v = q & msk, r = n2 * N1 + n1;
        const int j = (n2 << lg) + v;
        double w;
        if (n1 < H1) w = B0[j] + 2.0 * (PP[n1 * NpA + j] - QQ[n1 * NpA + j]);
        else w = B0[j] + 2.0 * (PP[(N1 - n1) * NpA + j] + QQ[(N1 - n1) * NpA + j]);
        X[v * xs + p.idxA[r]] = w;
    }
    __syncthreads();
}

// Shared-memory layout of a DCT launch and the start of its loads: the
// table block (one TMA bulk copy of the plan's contiguous global block) and,
// for `rows` > 0, rows j0 .. j0+rows-1 of `src` (one bulk copy per row, m
// rounded up to an even count -- the padding column is never used), all
// completing on one mbarrier.  The caller waits with dct_wait().
struct DctSmem {
    DctPlan p;
    double *P, *Q, *X;
    int xs;
};

__device__ __forceinline__ DctSmem dct_begin(const DctPlan& g, int NV, const double* src,
                                             const Layout& L, int j0, int rows, uint64_t* bar) {
    extern __shared__ __align__(16) double dct_sm[];
    DctSmem d;
    int a, b;
    dct_arena(g, NV, a, b);
    d.p = dct_view(g, dct_sm);
    d.P = dct_sm + dct_tab_doubles(g);
    d.Q = d.P + a;
    d.X = d.Q + b;
    d.xs = dct_xs(g);
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const uint32_t tb = (uint32_t)(dct_tab_doubles(g) * sizeof(double));
        const uint32_t rb = (uint32_t)(d.xs * sizeof(double));
        mbar_expect_tx(bar, tb + (uint32_t)rows * rb);
        bulk_g2s(dct_sm, g.tabs, tb, bar);
        for (int v = 0; v < rows; ++v) bulk_g2s(d.X + v * d.xs, src + L.at(0, j0 + v), rb, bar);
    }
    return d;
}

__device__ __forceinline__ void dct_wait(uint64_t* bar) {
    __syncthreads();  // mbarrier initialised before anyone polls it; gathers done
    mbar_wait(bar, 0u);
}

// r = A v - rho with v = m - mu varphi_bar (pdhg_pre_kernel's expression)
__device__ __forceinline__ double pdhg_rhs(const SweepArgs& a, int b, int i, int j) {
    const Layout L = a.L;
    const int n = L.n;
    const double* mx = pslot(a, b, P_MX);
    const double* my = pslot(a, b, P_MY);
    const double* bx = pslot(a, b, P_BX);
    const double* by = pslot(a, b, P_BY);
    const double mu = a.mu, ih = a.ih;
    const long o = L.at(i, j);
    const double r_ = (i < n) ? mx[o] - mu * bx[o] : 0.0;
    const double l_ = (i > 0) ? mx[o - 1] - mu * bx[o - 1] : 0.0;
    const double a_ = (j < n) ? my[o] - mu * by[o] : 0.0;
    const double b_ = (j > 0) ? my[o - L.pitch] - mu * by[o - L.pitch] : 0.0;
    const double div = (r_ - l_) * ih + (a_ - b_) * ih;
    return div - pslot(a, b, P_RHO)[o];
}

// Rows j0 .. j0+R-1: (MODE 0) slot `in` (bulk copies) or (MODE 1) the PDHG
// right-hand side (gathered, four nodes per thread in flight) -> DCT-II
// along i -> slot P_T.
template <int MODE>
__global__ void __launch_bounds__(256) dct_rows_fwd_kernel(const SweepArgs a, const DctPlan g, int in,
                                                           int R, int check_done) {
    const int b = blockIdx.y;
    if (check_done && *(volatile int*)&a.ctl[b].done) return;
    __shared__ uint64_t bar;
    const int m = g.m, j0 = blockIdx.x * R;
    const int rows = MODE ? 0 : min(R, m - j0);
    const Layout L = a.L;
    DctSmem d = dct_begin(g, R, pslot(a, b, in), L, j0, rows, &bar);
    const int xs = d.xs;
    if (MODE) {
        // every phase is spread over all threads: a CTA's time is its chain
        // of barrier-separated phases, so no phase may run on a few warps only
        W1MG_FOR2(v, i, R, m) {
            const int j = j0 + v;
            d.X[v * xs + i] = (j < m) ? pdhg_rhs(a, b, i, j) : 0.0;
        }
    } else {
        for (int e = threadIdx.x; e < (R - rows) * xs; e += blockDim.x) d.X[rows * xs + e] = 0.0;
    }
    dct_wait(&bar);
    dct2_vectors(d.p, R, xs, d.X, d.P, d.Q);
    double* T = pslot_w(a, b, P_T);
    W1MG_FOR2(v, i, R, m) {
        if (j0 + v < m) T[L.at(i, j0 + v)] = d.X[v * xs + i];
    }
}

// Columns k1 = c0 .. c0+Wc-1 of P_T: DCT-II along j, spectral divide
// (poisson.cpp:84-89), DCT-III along j, back to P_T.  X rows are the columns
// (stride m, odd: the column gather is bank-conflict free).
__global__ void __launch_bounds__(256) dct_cols_kernel(const SweepArgs a, const DctPlan g,
                                                       const double* __restrict__ lambda, int Wc,
                                                       int check_done) {
    const int b = blockIdx.y;
    if (check_done && *(volatile int*)&a.ctl[b].done) return;
    __shared__ uint64_t bar;
    const int m = g.m, c0 = blockIdx.x * Wc;
    const Layout L = a.L;
    DctSmem d = dct_begin(g, Wc, nullptr, L, 0, 0, &bar);
    const int xs = m;
    double* T = pslot_w(a, b, P_T);
    W1MG_FOR2(j, v, m, Wc) {
        d.X[v * xs + j] = (c0 + v < m) ? T[L.at(c0 + v, j)] : 0.0;
    }
    dct_wait(&bar);
    dct2_vectors(d.p, Wc, xs, d.X, d.P, d.Q);
    W1MG_FOR2(v, k2, Wc, m) {
        const int k1 = c0 + v;
        if (k1 < m) {
            double& y = d.X[v * xs + k2];
            y = (k1 == 0 && k2 == 0) ? 0.0 : y / (lambda[k1] + lambda[k2]);
        }
    }
    __syncthreads();
    dct3_vectors(d.p, Wc, xs, d.X, d.P, d.Q);
    W1MG_FOR2(j, v, m, Wc) {
        if (c0 + v < m) T[L.at(c0 + v, j)] = d.X[v * xs + j];
    }
}

// Rows j0 .. j0+R-1 of P_T (bulk copies): DCT-III along i, psi = y / (4 m^2)
// (poisson.cpp:93).  MODE 0: psi -> P_PSI.  MODE 1 (QN = conjugate norm): the
// PDHG post step on these rows (pdhg_post_kernel's arithmetic) with psi from
// shared memory; one extra row is transformed for the y-difference (R + 1
// must be a power of two).
template <int MODE, int QN>
__global__ void __launch_bounds__(256) dct_rows_inv_kernel(const SweepArgs a, const DctPlan g, int R,
                                                           double scale, int check_done) {
    const int b = blockIdx.y;
    if (check_done && *(volatile int*)&a.ctl[b].done) return;
    __shared__ uint64_t bar;
    const int NV = MODE ? R + 1 : R;
    const int m = g.m, j0 = blockIdx.x * R;
    const int rows = min(NV, m - j0);
    const Layout L = a.L;
    DctSmem d = dct_begin(g, NV, pslot(a, b, P_T), L, j0, rows, &bar);
    const int xs = d.xs;
    for (int e = threadIdx.x; e < (NV - rows) * xs; e += blockDim.x) d.X[rows * xs + e] = 0.0;
    dct_wait(&bar);
    dct3_vectors(d.p, NV, xs, d.X, d.P, d.Q);
    const double* X = d.X;
    if (MODE == 0) {
        double* psi = pslot_w(a, b, P_PSI);
        W1MG_FOR2(v, i, R, m) {
            if (j0 + v < m) psi[L.at(i, j0 + v)] = scale * X[v * xs + i];
        }
        return;
    }
    const int n = L.n;
    const double mu = a.mu, tau = a.tau, ih = a.ih;
    double* mx = pslot_w(a, b, P_MX);
    double* my = pslot_w(a, b, P_MY);
    double* px = pslot_w(a, b, P_PX);
    double* py = pslot_w(a, b, P_PY);
    double* bx = pslot_w(a, b, P_BX);
    double* by = pslot_w(a, b, P_BY);
    double s_dm2 = 0.0, s_dp2 = 0.0, s_cr = 0.0;
    W1MG_FOR2(v, i, R, m) {
        const int j = j0 + v;
        if (j <= n) {
            const long o = L.at(i, j);
            const bool hx = i < n, hy = j < n;
            const double pc = scale * X[v * xs + i];
            double mnx = 0.0, mny = 0.0, dmx = 0.0, dmy = 0.0, pox = 0.0, poy = 0.0;
            if (hx) {
                const double mo = mx[o];
                const double vv = mo - mu * bx[o];
                mnx = vv - (pc - scale * X[v * xs + i + 1]) * ih;  // poisson.cpp:124
                dmx = mnx - mo;
                pox = px[o];
            }
            if (hy) {
                const double mo = my[o];
                const double vv = mo - mu * by[o];
                mny = vv - (pc - scale * X[(v + 1) * xs + i]) * ih;  // poisson.cpp:130
                dmy = mny - mo;
                poy = py[o];
            }
            const double wx = hx ? pox + tau * mnx : 0.0;
            const double wy = hy ? poy + tau * mny : 0.0;
            double qx, qy;
            proj_unit_ball<QN>(wx, wy, qx, qy);
            if (hx) {
                mx[o] = mnx;
                px[o] = qx;
                bx[o] = 2.0 * qx - pox;
                const double dp = qx - pox;
                s_dm2 += dmx * dmx;
                s_dp2 += dp * dp;
                s_cr += dp * dmx;
            }
            if (hy) {
                my[o] = mny;
                py[o] = qy;
                by[o] = 2.0 * qy - poy;
                const double dp = qy - poy;
                s_dm2 += dmy * dmy;
                s_dp2 += dp * dp;
                s_cr += dp * dmy;
            }
        }
    }
    finish_sweep<true>(a, b, /*parity=*/1, blockIdx.x, gridDim.x, s_dm2, s_dp2, s_cr);
}

}  // namespace w1mg_dev
