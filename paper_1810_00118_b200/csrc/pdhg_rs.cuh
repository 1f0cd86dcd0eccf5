// pdhg_rs.cuh -- level-persistent G-prox PDHG for one pair with the CTA's
// rows resident in shared memory and a register-stationary dense DCT
// (config 3; replaces pdhg_persist.cuh where it fits).
//
// Reference semantics: the PDHG iteration of solver_pdhg.hpp:20-46 /
// SPEC.md:261-323 around the Neumann Poisson solve of
// proj/src/poisson.cpp:72-99 (FFTW REDFT10 -> divide -> REDFT01) and the
// affine projection of poisson.cpp:101-132.
//
// What bounds one pair is latency, not flops or bytes: an iteration is a
// chain rows -> (transpose) -> columns -> (transpose) -> rows with a global
// reduction at the end.  This engine shortens the chain:
//   * CTA c owns node rows [cR, cR+R) for the whole level.  Their state (m,
//     varphi, varphi_bar, rho: 7 rows arrays) is loaded into shared memory
//     once and written back once; the only per-iteration inputs from other
//     CTAs are the transposed DCT planes and ONE neighbour row (v_y of row
//     cR-1, published by CTA c-1 and ordered by a per-CTA flag, not a grid
//     barrier).
//   * Two grid barriers per iteration (after the row DCT-II and after the
//     column phase) instead of four.  The Eq. 12 reduction and the stop rule
//     of iteration k run on a REDUCER CTA (one more CTA, on an SM the level
//     leaves idle) between the two barriers of iteration k+1; the workers
//     read its decision together with their row loads after the second
//     barrier.  What a worker runs before it learns of a stop only writes
//     scratch planes, so the reduction costs the workers nothing.
//   * Both transposes are done by the STORES (scattered, fire-and-forget);
//     every load of a phase is a contiguous row.
//   * The length-m DCT-II / DCT-III of a vector is a dense product with the
//     (m-1) x h cosine matrix c(k,i) = cos(pi k (2i+1) / 2m), h = (m-1)/2,
//     folded by the symmetry i <-> m-1-i (even k see x_i + x_{m-1-i}, odd k
//     the difference; the constant mode and the middle sample are rank-one
//     terms).  Every thread keeps a TS x TS block of that matrix in REGISTERS
//     for the whole level (the matrix is used as is for the DCT-II and
//     transposed for the DCT-III), so a transform is one FMA phase (inputs
//     from shared memory, broadcast), one partial-sum exchange through shared
//     memory and one combine phase: two barriers per transform where the
//     prime-factor transform of dct_kernels.cuh has five, and no table
//     lookups.  h <= 16 TS with TS <= 4 covers m <= 129 in one CTA (16
//     coefficient doubles per thread).  Larger levels: pdhg_rs2.cuh (m <= 257:
//     the matrix over two-CTA clusters, FP64 tensor cores), pdhg_rspf.cuh
//     (m = 513: register-stationary prime-factor DCT); any other size whose
//     rows fit runs the prime-factor transforms of dct_kernels.cuh inside the
//     same iteration structure (TS = 0, vectors per transform a power of two,
//     the v_y and psi halo rows taken from the neighbour CTAs by flags).
//
// Spectral data is kept in "position" order along a transformed axis: even
// k = 2q+2 at q, odd k = 2q+1 at h+q, the constant mode at 2h (dense), or
// natural order (prime-factor); lambda is staged in that order.
#pragma once

#include "pdhg_persist.cuh"

namespace w1mg_dev {

constexpr int kRsThreads = 512;
constexpr int kRsStampSlots = 24;  // diagnostics: time stamps per iteration (CTA 0)

struct RsArgs {
    int m, h, R, G;       // m = 2h+1 nodes per side, R rows (columns) per CTA, G worker CTAs
    int HP;               // padded half size (16 TS)
    int posDC;            // spectral position of the constant mode
    int halo_x;           // 1: psi halo row from the neighbour CTA (prime-factor mode)
    const double* cosq;   // [4m] cos(pi j / 2m)
    const double* lamq;   // [m] lambda_k in position order
    double scale;         // 1 / (4 m^2), poisson.cpp:93
    double* vyb;          // [G][ms] v_y of each CTA's last row
    double* psb;          // [G][ms] psi of each CTA's first row
    unsigned* flag;       // [2][G] iteration stamps of vyb / psb
    double* part;         // [G][3] Eq. 12 partial sums
    int* dec;             // [2] stop decision of the reducer CTA, by iteration parity
    unsigned long long* stamps;
};

__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// rows of the partial-sum buffer: even half at 0, odd half at HP + 8 (bank
// offset for the paired combine), rank-one terms at 2 HP + 16; 17 doubles per
// row (16 partials, conflict-free both ways)
__device__ __forceinline__ int rs_row_odd(int HP) { return HP + 8; }
__device__ __forceinline__ int rs_row_x(int HP) { return 2 * HP + 16; }
__host__ __device__ inline int rs_part_doubles(int HP) { return (2 * HP + 17) * 17 + 1; }

// project_unit_ball (prox.cpp:47-62) for the persistent PDHG engines: q = 2
// scales by 1/sqrt(n2) through the MUFU rsqrt seed and one cubically convergent
// correction (error below 2^-60 before rounding, like shrink2_fast) instead of
// an IEEE square root and division -- a 260-cycle dependent chain per node of
// the post step.  PDHG parity is to tolerance (1e-9 fields), never bit-exact:
// the DCT already differs from the oracle's FFT in rounding.
template <int Q>
__device__ __forceinline__ void rs_proj_unit_ball(double vx, double vy, double& ox, double& oy) {
    if constexpr (Q == 1) {
        const double n2 = __fma_rn(vx, vx, vy * vy);
        if (n2 <= 1.0) {
            ox = vx;
            oy = vy;
        } else {
            const double y = rsq64h(n2);
            const double e = __fma_rn(-n2, y * y, 1.0);
            const double t = __fma_rn(e, 0.375, 0.5);
            const double r = __fma_rn(t, y * e, y);
            ox = r * vx;
            oy = r * vy;
        }
    } else {
        proj_unit_ball<Q>(vx, vy, ox, oy);
    }
}

// e -> (v, i) = (e / m, e % m) for the few vectors of a CTA (no integer division)
__device__ __forceinline__ void rs_split(int e, int m, int& v, int& i) {
    v = 0;
    i = e;
    while (i >= m) {
        i -= m;
        ++v;
    }
}

__device__ __forceinline__ double rs_sum16(const double* p) {
    const double a = (p[0] + p[1]) + (p[2] + p[3]);
    const double b = (p[4] + p[5]) + (p[6] + p[7]);
    const double c = (p[8] + p[9]) + (p[10] + p[11]);
    const double d = (p[12] + p[13]) + (p[14] + p[15]);
    return (a + b) + (c + d);
}

// thread (half, kq, ib): rows q_r = 16 r + kq of its half (k = 2q+2 even /
// 2q+1 odd), columns i_s = 16 s + ib
template <int TS>
__device__ __forceinline__ void rs_coefs(double (&c)[TS][TS], const double* cosq, int m, int h) {
    const int tid = threadIdx.x, ib = tid & 15, kq = (tid >> 4) & 15, half = tid >> 8;
#pragma unroll
    for (int r = 0; r < TS; ++r) {
        const int q = 16 * r + kq, k = half ? 2 * q + 1 : 2 * q + 2;
#pragma unroll
        for (int s = 0; s < TS; ++s) {
            const int i = 16 * s + ib;
            c[r][s] = (q < h && i < h) ? __ldg(cosq + (k * (2 * i + 1)) % (4 * m)) : 0.0;
        }
    }
}

// DCT-II (REDFT10) of V vectors X[v*xs + i] -> out(v, pos, X_k); P scratch.
// Ends without a barrier: the caller orders the reuse of X / P.
template <int TS, class Out>
__device__ __forceinline__ void rs_dct2(const double (&c)[TS][TS], int V, int m, int h, int HP,
                                        const double* X, int xs, double* P, int ps, Out out) {
    const int tid = threadIdx.x, ib = tid & 15, kq = (tid >> 4) & 15, half = tid >> 8;
    for (int v = 0; v < V; ++v) {
        const double* x = X + v * xs;
        double in[TS];
#pragma unroll
        for (int s = 0; s < TS; ++s) {
            const int i = 16 * s + ib;
            double a = 0.0, b = 0.0;
            if (i < h) {
                a = x[i];
                b = x[m - 1 - i];
            }
            in[s] = half ? a - b : a + b;
        }
        double* p = P + v * ps + ((half ? rs_row_odd(HP) : 0) + kq) * 17 + ib;
#pragma unroll
        for (int r = 0; r < TS; ++r) {
            double acc = 0.0;
#pragma unroll
            for (int s = 0; s < TS; ++s) acc = fma(c[r][s], in[s], acc);
            p[r * 16 * 17] = acc;
        }
        if ((tid >> 4) == 0) {  // constant mode: plain sum of the symmetric part
            double dc = 0.0;
#pragma unroll
            for (int s = 0; s < TS; ++s) dc += in[s];
            P[v * ps + rs_row_x(HP) * 17 + ib] = dc;
        }
    }
    __syncthreads();
    const int npos = 2 * h + 1, tot = V * npos;
    for (int e = tid; e < tot; e += kRsThreads) {
        int v, pos;
        rs_split(e, npos, v, pos);
        const int row = pos < h ? pos : (pos < 2 * h ? rs_row_odd(HP) + pos - h : rs_row_x(HP));
        double sum = rs_sum16(P + v * ps + row * 17);
        const double xh = X[v * xs + h];
        if (pos < h) sum += (pos & 1) ? xh : -xh;  // cos(pi k / 2), k = 2 pos + 2
        else if (pos == 2 * h) sum += xh;
        out(v, pos, 2.0 * sum);
    }
}

// DCT-III (REDFT01) of V spectral vectors Y[v*ys + pos] -> out(v, i, y_i).
template <int TS, class Out>
__device__ __forceinline__ void rs_dct3(const double (&c)[TS][TS], int V, int m, int h, int HP,
                                        const double* Y, int ys, double* P, int ps, Out out) {
    const int tid = threadIdx.x, ib = tid & 15, kq = (tid >> 4) & 15, half = tid >> 8;
    for (int v = 0; v < V; ++v) {
        const double* y = Y + v * ys + half * h;
        double in[TS];
#pragma unroll
        for (int r = 0; r < TS; ++r) {
            const int q = 16 * r + kq;
            in[r] = (q < h) ? y[q] : 0.0;
        }
        double* p = P + v * ps + ((half ? rs_row_odd(HP) : 0) + ib) * 17 + kq;
#pragma unroll
        for (int s = 0; s < TS; ++s) {
            double acc = 0.0;
#pragma unroll
            for (int r = 0; r < TS; ++r) acc = fma(c[r][s], in[r], acc);
            p[s * 16 * 17] = acc;
        }
        if (half == 0 && ib == 0) {  // middle sample: sum of X_k cos(pi k / 2), k even
            double mp = 0.0;
#pragma unroll
            for (int r = 0; r < TS; ++r) mp += ((16 * r + kq) & 1) ? in[r] : -in[r];
            P[v * ps + rs_row_x(HP) * 17 + kq] = mp;
        }
    }
    __syncthreads();
    const int per = 2 * h, tot = V * per, totp = (tot + 31) & ~31;
    for (int e = tid; e < totp; e += kRsThreads) {
        const bool on = e < tot;
        const int ee = on ? e : 0;
        int v, w;
        rs_split(ee, per, v, w);
        const int i = w >> 1, hf = w & 1;
        const double sum = rs_sum16(P + v * ps + ((hf ? rs_row_odd(HP) : 0) + i) * 17);
        const double oth = __shfl_xor_sync(0xffffffffu, sum, 1);
        const double dc = Y[v * ys + 2 * h];
        const double E = dc + 2.0 * (hf ? oth : sum), O = 2.0 * (hf ? sum : oth);
        if (on) out(v, hf ? m - 1 - i : i, hf ? E - O : E + O);
    }
    if (tid < V) {
        const double sum = rs_sum16(P + tid * ps + rs_row_x(HP) * 17);
        out(tid, h, Y[tid * ys + 2 * h] + 2.0 * sum);
    }
}

// The REDUCER CTA(s) (blockIdx.x >= ra.G; `active`: the one that works): the
// Eq. 12 reduction and the stop rule (finalize_pair<true>'s) of iteration k
// run here between the two grid barriers of iteration k+1 -- off the
// workers' critical path, on an SM the level leaves idle.  It sums the
// workers' partials in a fixed order, records the history and (on a stop) the
// control block, and publishes the decision in dec[iteration parity]; the
// workers read it after the second barrier.  The phases a worker runs before
// it learns of a stop only write scratch planes.
struct RsRed {  // by value: a reference would move the kernel's parameter block to local memory
    PairCtl* ctl;
    double h2, mu, tau;
    double* hist;
    long hist_cap;
    int* ndone;
    const double* part;
    int* dec;
    int G;
};
__device__ __forceinline__ RsRed rs_red_args(const SweepArgs& a, const RsArgs& ra) {
    return RsRed{a.ctl, a.h2, a.mu, a.tau, a.hist, a.hist_cap, a.ndone, ra.part, ra.dec, ra.G};
}
__device__ __noinline__ void rs_reducer(const RsRed a, const GridBar gb, bool active) {
    const RsRed& ra = a;
    __shared__ int r_ok;
    __shared__ int r_stop;
    __shared__ double r_red[kRsThreads / 32][3];
    PairCtl* ctl = a.ctl;
    long k = ctl->it;
    const long max_it = ctl->max_it;
    const double tol = ctl->tol;
    const int tid = threadIdx.x, W = ra.G;
    unsigned gen = 0;
    if (tid == 0) r_stop = 0;
    for (long iter = 0;; ++iter) {
        if (!grid_barrier(gb, gen, &r_ok)) return;
        if (iter > 0 && active) {
            double pt0 = 0.0, pt1 = 0.0, pt2 = 0.0;
            if (tid < W) {
                pt0 = __ldcg(ra.part + 3 * tid + 0);
                pt1 = __ldcg(ra.part + 3 * tid + 1);
                pt2 = __ldcg(ra.part + 3 * tid + 2);
            }
            pt0 = warp_sum(pt0);
            pt1 = warp_sum(pt1);
            pt2 = warp_sum(pt2);
            if ((tid & 31) == 0) {
                r_red[tid >> 5][0] = pt0;
                r_red[tid >> 5][1] = pt1;
                r_red[tid >> 5][2] = pt2;
            }
            __syncthreads();
            if (tid == 0) {
                double t0 = 0.0, t1 = 0.0, t2 = 0.0;
                for (int w = 0; w < (W + 31) / 32; ++w) {
                    t0 += r_red[w][0];
                    t1 += r_red[w][1];
                    t2 += r_red[w][2];
                }
                const double fpr = a.h2 * (t0 / a.mu + t1 / a.tau + 2.0 * t2);  // Eq. 12
                const bool finite = isfinite(fpr);
                const bool stop = fpr < tol || k + 1 >= max_it || !finite;
                r_stop = stop ? 1 : 0;
                ra.dec[iter & 1] = stop ? 1 : 0;
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
            ++k;
        }
        if (!grid_barrier(gb, gen, &r_ok)) return;  // (its __syncthreads orders r_stop)
        if (iter > 0) {
            // every reducer CTA leaves with the workers: the idle one reads the decision too
            if (!active && tid == 0) r_stop = __ldcg(ra.dec + (iter & 1));
            __syncthreads();
            if (r_stop) return;
        }
    }
}

// Dynamic shared memory (doubles): lam[ms] | state 7 x (R+1) x ms (row 0: the
// shadow row) | vyl[ms] | X (R+2) x ms | dense: Y (R+2) x ms, P (R+2) x ps |
// prime-factor: tables, P, Q arenas of dct_arena(g, R)
__host__ __device__ inline size_t rs_smem_doubles(const DctPlan& g, int R, int TS) {
    const int ms = g.m + 1;
    size_t d = (size_t)ms * (1 + 7 * (R + 1) + 1 + (R + 2));
    if (TS > 0) {
        d += (size_t)(R + 2) * ms + (size_t)(R + 2) * rs_part_doubles(16 * TS);
    } else {
        int a, b;
        dct_arena(g, R, a, b);
        d += (size_t)dct_tab_doubles(g) + a + b;
    }
    return d;
}

enum RsState { S_MX = 0, S_MY, S_PX, S_PY, S_BX, S_BY, S_RHO, S_N };

// Dense mode (TS > 0) keeps a SHADOW copy of row j0-1 (the row below the
// CTA's first): its state is updated redundantly every iteration (one more
// row in the row DCT-III and in the post step), so the y-difference of the
// pre step needs nothing from the neighbour CTA -- the only inter-CTA
// synchronisation of an iteration is the two grid barriers.  The
// prime-factor mode (TS = 0, vectors per transform a power of two) instead
// takes v_y of row j0-1 and psi of row j0+R from the neighbours' published
// rows, ordered by per-CTA flags.
template <int QN, int TS>
__global__ void __launch_bounds__(kRsThreads, 1)
pdhg_rs_kernel(const SweepArgs a, const DctPlan g, const RsArgs ra, GridBar gb) {
    extern __shared__ __align__(16) double rs_sm[];
    __shared__ int s_ok;
    __shared__ int s_stop;
    __shared__ double red[kRsThreads / 32][3];
    PairCtl* ctl = a.ctl;
    if (*(volatile int*)&ctl->done) return;
    if ((int)blockIdx.x >= ra.G) {  // reducer CTA(s): Eq. 12 sums and the stop rule
        rs_reducer(rs_red_args(a, ra), gb, (int)blockIdx.x == ra.G);
        return;
    }
    constexpr bool kDense = TS > 0;
    const int m = ra.m, n = m - 1, h = ra.h, R = ra.R, G = ra.G, HP = ra.HP;
    const int ms = m + 1, tid = threadIdx.x, c = blockIdx.x;
    const int j0 = c * R, nr = min(R, m - j0);  // owned rows [j0, j0 + nr)
    const int sh = (kDense && c > 0) ? 1 : 0;   // shadow row j0-1 kept
    const int hl = (j0 + nr < m) ? 1 : 0;       // halo row j0+nr exists
    const Layout L = a.L;
    const double mu = a.mu, tau = a.tau, ih = a.ih, scale = ra.scale;

    double* lam = rs_sm;
    double* st = lam + ms;
    double* vyl = st + (size_t)S_N * (R + 1) * ms;
    double* X = vyl + ms;
    double* Y = X;  // prime-factor mode transforms in place
    double* P = nullptr;
    double* Q = nullptr;
    int ps = 0;
    DctPlan pl = g;
    if constexpr (kDense) {
        Y = X + (size_t)(R + 2) * ms;
        P = Y + (size_t)(R + 2) * ms;
        ps = rs_part_doubles(HP);
    } else {
        double* tab = X + (size_t)(R + 2) * ms;
        for (int e = tid; e < dct_tab_doubles(g); e += kRsThreads) tab[e] = g.tabs[e];
        pl = dct_view(g, tab);
        int sa, sb;
        dct_arena(g, R, sa, sb);
        P = tab + dct_tab_doubles(g);
        Q = P + sa;
    }
    // state row sv: 0 = shadow row j0-1, sv = v+1 for the owned row j0+v
    auto S = [&](int slot, int sv) { return st + ((size_t)slot * (R + 1) + sv) * ms; };

    double cf[kDense ? TS : 1][kDense ? TS : 1];
    if constexpr (kDense) rs_coefs<TS>(cf, ra.cosq, m, h);

    // ---- level prologue: tables and the CTA's rows into shared memory
    for (int e = tid; e < m; e += kRsThreads) lam[e] = ra.lamq[e];
    for (int e = tid; e < S_N * (R + 1) * ms; e += kRsThreads) st[e] = 0.0;
    for (int e = tid; e < (R + 2) * ms; e += kRsThreads) X[e] = 0.0;
    __syncthreads();
    {
        const int gs[S_N] = {P_MX, P_MY, P_PX, P_PY, P_BX, P_BY, P_RHO};
        const int rows = nr + sh;
        for (int e = tid; e < S_N * rows * m; e += kRsThreads) {
            const int sl = e / (rows * m), rem = e - sl * rows * m, w = rem / m, i = rem - w * m;
            S(sl, w + 1 - sh)[i] = pslot(a, 0, gs[sl])[L.at(i, j0 - sh + w)];
        }
    }
    __syncthreads();
    double* vyb_me = ra.vyb + (size_t)c * ms;
    unsigned* flag_vy = ra.flag;
    unsigned* flag_ps = ra.flag + G;
    // prime-factor mode: v_y of the last owned row for the CTA above
    auto publish_vy = [&](unsigned stampv) {
        const int j = j0 + nr - 1;
        for (int i = tid; i < m; i += kRsThreads)
            vyb_me[i] = (j < n) ? S(S_MY, nr)[i] - mu * S(S_BY, nr)[i] : 0.0;
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            st_release_u32(flag_vy + c, stampv);
        }
    };
    if constexpr (!kDense) publish_vy(1u);

    // spin until *f >= want (thread 0), bounded like the grid barrier
    auto wait_flag = [&](const unsigned* f, unsigned want) -> bool {
        if (tid == 0) {
            int ok = 1;
            if ((int)(ld_acquire_u32(f) - want) < 0) {
                const unsigned long long t0 = gtimer();
                while ((int)(ld_acquire_u32(f) - want) < 0) {
                    if (*(volatile int*)gb.err || gtimer() - t0 > 2000000000ull) {
                        atomicExch(gb.err, 1);
                        ok = 0;
                        break;
                    }
                }
            }
            s_ok = ok;
        }
        __syncthreads();
        return s_ok != 0;
    };

    double* T1 = pslot_w(a, 0, P_T);    // T1[pos1][j] at L.at(j, pos1)
    double* T2 = pslot_w(a, 0, P_PSI);  // T2[j][pos1] at L.at(pos1, j)
    unsigned gen = 0;
    long iter = 0;
    auto stamp = [&](int q) {
        if (ra.stamps && c == 0 && tid == 0 && iter < 64) ra.stamps[iter * kRsStampSlots + q] = gtimer();
    };
    auto flush_state = [&]() {
        const int gs[6] = {P_MX, P_MY, P_PX, P_PY, P_BX, P_BY};
        for (int e = tid; e < 6 * nr * m; e += kRsThreads) {
            const int sl = e / (nr * m), rem = e - sl * nr * m, v = rem / m, i = rem - v * m;
            pslot_w(a, 0, gs[sl])[L.at(i, j0 + v)] = S(sl, v + 1)[i];
        }
    };

    for (;; ++iter) {
        stamp(0);
        // ---- A: r = A v - rho on the owned rows (poisson.cpp:113-115), DCT-II along i -> T1
        if constexpr (!kDense) {
            if (c > 0) {
                if (!wait_flag(flag_vy + c - 1, (unsigned)iter + 1u)) return;
                const double* nb = ra.vyb + (size_t)(c - 1) * ms;
                for (int i = tid; i < m; i += kRsThreads) vyl[i] = __ldcg(nb + i);
                __syncthreads();
            }
        }
        for (int e = tid; e < nr * m; e += kRsThreads) {
            int v, i;
            rs_split(e, m, v, i);
            const int j = j0 + v, sv = v + 1;
            const double* mx = S(S_MX, sv);
            const double* bx = S(S_BX, sv);
            const double r_ = (i < n) ? mx[i] - mu * bx[i] : 0.0;
            const double l_ = (i > 0) ? mx[i - 1] - mu * bx[i - 1] : 0.0;
            const double a_ = (j < n) ? S(S_MY, sv)[i] - mu * S(S_BY, sv)[i] : 0.0;
            double b_ = 0.0;
            if (j > 0) b_ = (kDense || v > 0) ? S(S_MY, sv - 1)[i] - mu * S(S_BY, sv - 1)[i] : vyl[i];
            const double div = (r_ - l_) * ih + (a_ - b_) * ih;
            X[v * ms + i] = div - S(S_RHO, sv)[i];
        }
        __syncthreads();
        if constexpr (kDense) {
            rs_dct2<TS>(cf, nr, m, h, HP, X, ms, P, ps,
                        [&](int v, int pos, double val) { T1[L.at(j0 + v, pos)] = val; });
        } else {
            dct2_vectors(pl, R, ms, X, P, Q);
            for (int e = tid; e < nr * m; e += kRsThreads) {
                int v, kk;
                rs_split(e, m, v, kk);
                T1[L.at(j0 + v, kk)] = X[v * ms + kk];
            }
        }
        stamp(1);
        if (!grid_barrier(gb, gen, &s_ok)) return;
        stamp(2);
        // ---- B: columns pos1 in [j0, j0+nr): DCT-II along j, divide by
        // lambda_k1 + lambda_k2 (poisson.cpp:84-89), DCT-III along j -> T2
        for (int e = tid; e < nr * m; e += kRsThreads) {
            int v, j;
            rs_split(e, m, v, j);
            X[v * ms + j] = __ldcg(T1 + L.at(j, j0 + v));
        }
        __syncthreads();
        if constexpr (kDense) {
            rs_dct2<TS>(cf, nr, m, h, HP, X, ms, P, ps, [&](int v, int pos, double val) {
                const int p1 = j0 + v;
                Y[v * ms + pos] = (p1 == ra.posDC && pos == ra.posDC) ? 0.0 : val / (lam[p1] + lam[pos]);
            });
            __syncthreads();
            rs_dct3<TS>(cf, nr, m, h, HP, Y, ms, P, ps,
                        [&](int v, int j, double val) { T2[L.at(j0 + v, j)] = val; });
        } else {
            dct2_vectors(pl, R, ms, X, P, Q);
            for (int e = tid; e < nr * m; e += kRsThreads) {
                int v, k2;
                rs_split(e, m, v, k2);
                const int p1 = j0 + v;
                double& y = X[v * ms + k2];
                y = (p1 == ra.posDC && k2 == ra.posDC) ? 0.0 : y / (lam[p1] + lam[k2]);
            }
            __syncthreads();
            dct3_vectors(pl, R, ms, X, P, Q);
            for (int e = tid; e < nr * m; e += kRsThreads) {
                int v, j;
                rs_split(e, m, v, j);
                T2[L.at(j0 + v, j)] = X[v * ms + j];
            }
        }
        stamp(3);
        if (!grid_barrier(gb, gen, &s_ok)) return;
        stamp(4);
        // ---- C: rows j0-sh .. j0+nr-1+hl of T2 (dense) / the owned rows
        // (prime-factor), DCT-III along i, psi = y / (4 m^2) (poisson.cpp:93);
        // afterwards X row w holds psi of row j0 - sh + w
        int decv = 0;  // the reducer's decision: requested now, consumed after the row loads
        if (iter > 0 && tid == 0) decv = __ldcg(ra.dec + (iter & 1));
        const int nh = kDense ? sh + nr + hl : nr;
        for (int e = tid; e < nh * m; e += kRsThreads) {
            int w, pos;
            rs_split(e, m, w, pos);
            Y[w * ms + pos] = __ldcg(T2 + L.at(pos, j0 - sh + w));
        }
        if (tid == 0) s_stop = decv;
        __syncthreads();
        if (iter > 0 && s_stop) {  // iteration iter-1 met the stop rule: its state is final
                flush_state();
            return;
        }
        if constexpr (kDense) {
            rs_dct3<TS>(cf, nh, m, h, HP, Y, ms, P, ps,
                        [&](int w, int i, double val) { X[w * ms + i] = scale * val; });
            __syncthreads();
        } else {
            dct3_vectors(pl, R, ms, X, P, Q);
            for (int e = tid; e < nr * m; e += kRsThreads) {
                int v, i;
                rs_split(e, m, v, i);
                X[v * ms + i] *= scale;
            }
            __syncthreads();
            // psi halo row j0+nr from the CTA above; our first row for the CTA below
            if (c > 0) {
                double* mine = ra.psb + (size_t)c * ms;
                for (int i = tid; i < m; i += kRsThreads) mine[i] = X[i];
                __syncthreads();
                if (tid == 0) {
                    __threadfence();
                    st_release_u32(flag_ps + c, (unsigned)iter + 1u);
                }
            }
            if (c + 1 < G) {
                if (!wait_flag(flag_ps + c + 1, (unsigned)iter + 1u)) return;
                const double* nb = ra.psb + (size_t)(c + 1) * ms;
                for (int i = tid; i < m; i += kRsThreads) X[nr * ms + i] = __ldcg(nb + i);
                __syncthreads();
            }
        }
        stamp(5);
        // ---- D: post step (pdhg_post_kernel's arithmetic) on the shadow and
        // owned rows; Eq. 12 partial sums over the owned rows only
        double s_dm2 = 0.0, s_dp2 = 0.0, s_cr = 0.0;
        for (int e = tid; e < (nr + sh) * m; e += kRsThreads) {
            int w, i;
            rs_split(e, m, w, i);
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
        if ((tid & 31) == 0) {
            red[tid >> 5][0] = s_dm2;
            red[tid >> 5][1] = s_dp2;
            red[tid >> 5][2] = s_cr;
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
        if constexpr (!kDense) publish_vy((unsigned)iter + 2u);
        stamp(6);
    }
}

}  // namespace w1mg_dev
