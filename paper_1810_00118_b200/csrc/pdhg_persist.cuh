// pdhg_persist.cuh -- level-persistent G-prox PDHG for one pair (config 3):
// every iteration of a level in ONE cooperative launch, one CTA per SM, the
// phases of an iteration separated by grid barriers instead of kernel
// boundaries.
//
// The streaming iteration (three DCT launches, pdhg_engine.cuh) is bound by
// launch + per-CTA latency for one pair: each launch re-stages the DCT tables
// and waits for its slowest CTA.  Here the tables are staged once per level,
// and an iteration is
//   A  rows    r = A v - rho (PDHG pre step, poisson.cpp:113-115) and the
//              row DCT-II (REDFT10 along i) -> P_T
//   B  columns DCT-II along j, divide by lambda_k1 + lambda_k2 (constant mode
//              -> 0, poisson.cpp:84-89), DCT-III along j -> P_T
//   C  rows    DCT-III along i, psi = y / (4 m^2) (poisson.cpp:93) -> P_PSI
//   D  rows    post step (m, varphi, varphi_bar; pdhg_post_kernel's
//              arithmetic) + the CTA's Eq. 12 partial sums
//   E  every CTA sums the partials in CTA order (identical everywhere) and
//      applies the stop rule of finalize_pair<true>; CTA 0 records it
// with a grid barrier after A, B, C and D.  Data written by other CTAs in
// the same launch is read with ld.global.cg (L2, never a stale L1 line).
// Results equal the streaming path's to rounding (the transforms are the
// same device functions; only the residual partials are grouped by CTA).
#pragma once

#include "dct_kernels.cuh"

namespace w1mg_dev {

struct GridBar {
    unsigned* count;  // arrivals, monotone across barriers and launches
    unsigned* gen;    // unused slot (kept zero)
    int* err;         // set on a barrier timeout: every CTA leaves
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Grid barrier over a monotone arrival counter (all CTAs co-resident:
// cooperative launch): barrier number q completes when the counter reaches
// base + q * gridDim.x.  One release-add per CTA and acquire polling -- no
// reset, no second atomic on the critical path.  `target` is the running
// target (thread 0 only).  Returns false when the barrier timed out (2 s):
// the caller leaves the kernel; the host then fails loudly.
__device__ __forceinline__ bool grid_barrier(const GridBar& gb, unsigned& target, int* s_ok) {
    __syncthreads();
    if (threadIdx.x == 0) {
        int ok = 1;
        target += gridDim.x;
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(gb.count) : "memory");
        if ((int)(ld_acquire_u32(gb.count) - target) < 0) {
            const unsigned long long t0 = gtimer();
            while ((int)(ld_acquire_u32(gb.count) - target) < 0) {
                if (*(volatile int*)gb.err || gtimer() - t0 > 2000000000ull) {
                    atomicExch(gb.err, 1);
                    ok = 0;
                    break;
                }
            }
        }
        *s_ok = ok;
    }
    __syncthreads();
    return *s_ok != 0;
}

// Batched gather: st(a, b, ld(a, b)) for a < NA, b < NB, U loads per thread
// in flight before any is used (L2 latency, not issue, bounds the load
// phases of a one-pair level).
template <int U, class Ld, class St>
__device__ __forceinline__ void gather2(int NA, int NB, Ld ld, St st) {
    const int tot = NA * NB;
    for (int e0 = threadIdx.x; e0 < tot; e0 += U * blockDim.x) {
        double x[U];
        int ia[U], ib[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = e0 + u * blockDim.x;
            ia[u] = e / NB;
            ib[u] = e - ia[u] * NB;
            x[u] = (e < tot) ? ld(ia[u], ib[u]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (e0 + u * (int)blockDim.x < tot) st(ia[u], ib[u], x[u]);
    }
}

// pdhg_rhs with L2 loads (rows written by other CTAs earlier in the launch)
__device__ __forceinline__ double pdhg_rhs_cg(const SweepArgs& a, int i, int j) {
    const Layout L = a.L;
    const int n = L.n;
    const double* mx = pslot(a, 0, P_MX);
    const double* my = pslot(a, 0, P_MY);
    const double* bx = pslot(a, 0, P_BX);
    const double* by = pslot(a, 0, P_BY);
    const double mu = a.mu, ih = a.ih;
    const long o = L.at(i, j);
    const double r_ = (i < n) ? __ldcg(mx + o) - mu * __ldcg(bx + o) : 0.0;
    const double l_ = (i > 0) ? __ldcg(mx + o - 1) - mu * __ldcg(bx + o - 1) : 0.0;
    const double a_ = (j < n) ? __ldcg(my + o) - mu * __ldcg(by + o) : 0.0;
    const double b_ = (j > 0) ? __ldcg(my + o - L.pitch) - mu * __ldcg(by + o - L.pitch) : 0.0;
    const double div = (r_ - l_) * ih + (a_ - b_) * ih;
    return div - __ldcg(pslot(a, 0, P_RHO) + o);
}

// One pair (b = 0), all iterations of the level.  Rr rows / Rc columns per
// chunk (powers of two); chunk c of a phase is done by CTA c mod gridDim.
// 256 threads, one CTA per SM (measured: 512 threads in one CTA 65^2 row
// phase 3.8 vs 3.2 us; two 256-thread CTAs per SM with half the vectors each:
// no faster per phase and 2-3x slower barriers)
constexpr int kPersistThreads = 256;

template <int QN>
__global__ void __launch_bounds__(kPersistThreads, 1)
pdhg_persist_kernel(const SweepArgs a, const DctPlan g, const double* __restrict__ lambda, int Rr,
                    int Rc, double scale, GridBar gb, double* __restrict__ part,
                    unsigned long long* __restrict__ stamps) {
    __shared__ uint64_t bar;
    __shared__ int s_ok;
    __shared__ int s_stop;
    __shared__ double red[kPersistThreads / 32][3];
    PairCtl* ctl = a.ctl;
    if (*(volatile int*)&ctl->done) return;
    // read before the first barrier, i.e. before CTA 0 records anything
    long k = ctl->it;
    const long max_it = ctl->max_it;
    const double tol = ctl->tol;
    const int m = g.m, n = m - 1;
    const Layout L = a.L;
    const int NV = Rr > Rc ? Rr : Rc;
    // tables once per level (one bulk copy); no rows through the barrier
    DctSmem d = dct_begin(g, NV, nullptr, L, 0, 0, &bar);
    // the arrival counter is zeroed by the host before the launch
    unsigned gen = 0;
    dct_wait(&bar);
    const int xs = d.xs;
    double* T = pslot_w(a, 0, P_T);
    double* psi = pslot_w(a, 0, P_PSI);
    const int nrc = (m + Rr - 1) / Rr, ncc = (m + Rc - 1) / Rc;
    const double mu = a.mu, tau = a.tau, ih = a.ih;
    long iter = 0;
    // diagnostics (W1MG_PERSIST_STAMPS): CTA 0 stamps the end of every phase
    // and barrier of the first 64 iterations
    auto stamp = [&](int q) {
        if (stamps && blockIdx.x == 0 && threadIdx.x == 0 && iter < 64) stamps[iter * 10 + q] = gtimer();
    };
    for (;; ++iter) {
        stamp(0);
        // ---- A: rows, pre step + DCT-II
        for (int c = blockIdx.x; c < nrc; c += gridDim.x) {
            const int j0 = c * Rr;
            gather2<4>(
                Rr, m, [&](int v, int i) { return (j0 + v < m) ? pdhg_rhs_cg(a, i, j0 + v) : 0.0; },
                [&](int v, int i, double x) { d.X[v * xs + i] = x; });
            __syncthreads();
            dct2_vectors(d.p, Rr, xs, d.X, d.P, d.Q);
            W1MG_FOR2(v, i, Rr, m) {
                if (j0 + v < m) T[L.at(i, j0 + v)] = d.X[v * xs + i];
            }
            __syncthreads();
        }
        stamp(1);
        if (!grid_barrier(gb, gen, &s_ok)) return;
        stamp(2);
        // ---- B: columns, DCT-II, divide, DCT-III (X rows = columns, stride m)
        for (int c = blockIdx.x; c < ncc; c += gridDim.x) {
            const int c0 = c * Rc;
            gather2<8>(
                m, Rc, [&](int j, int v) { return (c0 + v < m) ? __ldcg(T + L.at(c0 + v, j)) : 0.0; },
                [&](int j, int v, double x) { d.X[v * m + j] = x; });
            __syncthreads();
            dct2_vectors(d.p, Rc, m, d.X, d.P, d.Q);
            W1MG_FOR2(v, k2, Rc, m) {
                const int k1 = c0 + v;
                if (k1 < m) {
                    double& y = d.X[v * m + k2];
                    y = (k1 == 0 && k2 == 0) ? 0.0 : y / (lambda[k1] + lambda[k2]);
                }
            }
            __syncthreads();
            dct3_vectors(d.p, Rc, m, d.X, d.P, d.Q);
            W1MG_FOR2(j, v, m, Rc) {
                if (c0 + v < m) T[L.at(c0 + v, j)] = d.X[v * m + j];
            }
            __syncthreads();
        }
        stamp(3);
        if (!grid_barrier(gb, gen, &s_ok)) return;
        stamp(4);
        // ---- C: rows, DCT-III -> psi
        for (int c = blockIdx.x; c < nrc; c += gridDim.x) {
            const int j0 = c * Rr;
            gather2<8>(
                Rr, m, [&](int v, int i) { return (j0 + v < m) ? __ldcg(T + L.at(i, j0 + v)) : 0.0; },
                [&](int v, int i, double x) { d.X[v * xs + i] = x; });
            __syncthreads();
            dct3_vectors(d.p, Rr, xs, d.X, d.P, d.Q);
            W1MG_FOR2(v, i, Rr, m) {
                if (j0 + v < m) psi[L.at(i, j0 + v)] = scale * d.X[v * xs + i];
            }
            __syncthreads();
        }
        stamp(5);
        if (!grid_barrier(gb, gen, &s_ok)) return;
        stamp(6);
        // ---- D: post step on the CTA's rows + Eq. 12 partial sums
        double s_dm2 = 0.0, s_dp2 = 0.0, s_cr = 0.0;
        for (int c = blockIdx.x; c < nrc; c += gridDim.x) {
            const int j0 = c * Rr;
            double* mx = pslot_w(a, 0, P_MX);
            double* my = pslot_w(a, 0, P_MY);
            double* px = pslot_w(a, 0, P_PX);
            double* py = pslot_w(a, 0, P_PY);
            double* bx = pslot_w(a, 0, P_BX);
            double* by = pslot_w(a, 0, P_BY);
            W1MG_FOR2(v, i, Rr, m) {
                const int j = j0 + v;
                if (j <= n) {
                    const long o = L.at(i, j);
                    const bool hx = i < n, hy = j < n;
                    const double pc = __ldcg(psi + o);
                    double mnx = 0.0, mny = 0.0, dmx = 0.0, dmy = 0.0, pox = 0.0, poy = 0.0;
                    if (hx) {
                        const double mo = mx[o];
                        const double vv = mo - mu * bx[o];
                        mnx = vv - (pc - __ldcg(psi + o + 1)) * ih;  // poisson.cpp:124
                        dmx = mnx - mo;
                        pox = px[o];
                    }
                    if (hy) {
                        const double mo = my[o];
                        const double vv = mo - mu * by[o];
                        mny = vv - (pc - __ldcg(psi + o + L.pitch)) * ih;  // poisson.cpp:130
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
        }
        s_dm2 = warp_sum(s_dm2);
        s_dp2 = warp_sum(s_dp2);
        s_cr = warp_sum(s_cr);
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        if (lane == 0) {
            red[warp][0] = s_dm2;
            red[warp][1] = s_dp2;
            red[warp][2] = s_cr;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double t0 = 0.0, t1 = 0.0, t2 = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
                t0 += red[w][0];
                t1 += red[w][1];
                t2 += red[w][2];
            }
            part[blockIdx.x * 3 + 0] = t0;
            part[blockIdx.x * 3 + 1] = t1;
            part[blockIdx.x * 3 + 2] = t2;
        }
        stamp(7);
        if (!grid_barrier(gb, gen, &s_ok)) return;
        stamp(8);
        // ---- E: Eq. 12 and the stop rule, identical in every CTA (the sweep
        // count is tracked locally, so no CTA reads what CTA 0 records)
        if (threadIdx.x == 0) {
            double t0 = 0.0, t1 = 0.0, t2 = 0.0;
            for (int q = 0; q < (int)gridDim.x; ++q) {
                t0 += __ldcg(part + 3 * q + 0);
                t1 += __ldcg(part + 3 * q + 1);
                t2 += __ldcg(part + 3 * q + 2);
            }
            const double fpr = a.h2 * (t0 / a.mu + t1 / a.tau + 2.0 * t2);  // Eq. 12
            const bool finite = isfinite(fpr);
            const bool stop = fpr < tol || k + 1 >= max_it || !finite;
            s_stop = stop ? 1 : 0;
            if (blockIdx.x == 0) {
                if (a.hist && k < a.hist_cap) a.hist[k] = fpr;
                ctl->it = k + 1;
                ctl->fpr = fpr;
                ctl->cur = 0;
                if (!finite) ctl->nonfinite = 1;
                if (stop) {
                    ctl->done = 1;
                    if (a.ndone) atomicAdd(a.ndone, 1);
                }
                __threadfence();
            }
        }
        __syncthreads();
        const int stop = s_stop;
        ++k;
        if (stop) return;
    }
}

}  // namespace w1mg_dev
