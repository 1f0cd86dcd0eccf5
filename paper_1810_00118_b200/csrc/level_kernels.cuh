// level_kernels.cuh -- everything around the fused sweep that runs once per
// level: sources (restriction), prolongation (Eq. 14/15), and the
// compensated per-pair reductions behind W1, the dual value and the
// relative stopping tolerance.  All batched over the pairs of a level.
#pragma once

#include "cp_kernels.cuh"
#include "device_common.cuh"

namespace w1mg_dev {

// ------------------------------------------------------------ restriction
// 2x2 block sums of a pair-major stack of m x m cell images -> (m/2)^2
// (SURVEY D4).  Same association as oracle/w1mg_oracle.c:or_block_sum.
__global__ void block_sum_kernel(const double* __restrict__ fine, double* __restrict__ coarse,
                                 int m, int npairs) {
    const int mc = m / 2;
    const long per = (long)mc * mc;
    const long total = per * npairs;
    for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total;
         t += (long)gridDim.x * blockDim.x) {
        const long b = t / per;
        const int k = (int)(t - b * per);
        const int j = k / mc, i = k - j * mc;
        const double* r0 = fine + b * (long)m * m + (long)(2 * j) * m + 2 * i;
        const double* r1 = r0 + m;
        coarse[t] = (r0[0] + r0[1]) + (r1[0] + r1[1]);
    }
}

// cell image (n x n) -> node values: mean of the touching cells,
// written into slot `dst` of each pair's level buffers.
__device__ __forceinline__ double node_from_image(const double* img, int n, int i, int j) {
    const bool il = i > 0, ir = i < n, jl = j > 0, jr = j < n;
    if (il && ir && jl && jr)
        return 0.25 * ((img[(long)(j - 1) * n + i - 1] + img[(long)(j - 1) * n + i]) +
                       (img[(long)j * n + i - 1] + img[(long)j * n + i]));
    if (jl && jr) {
        const int c = il ? i - 1 : i;
        return 0.5 * (img[(long)(j - 1) * n + c] + img[(long)j * n + c]);
    }
    if (il && ir) {
        const int r = jl ? j - 1 : j;
        return 0.5 * (img[(long)r * n + i - 1] + img[(long)r * n + i]);
    }
    const int c = il ? i - 1 : i, r = jl ? j - 1 : j;
    return img[(long)r * n + c];
}

__global__ void image_to_nodes_kernel(const double* __restrict__ img0,
                                      const double* __restrict__ img1, double* base, Layout L,
                                      int slot_a, int slot_b) {
    const int n = L.n;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    const int b = blockIdx.z;
    if (i > n || j > n) return;
    const long per = (long)n * n;
    double* pb = base + (long)b * NSLOT * L.plane;
    pb[slot_a * L.plane + L.at(i, j)] = node_from_image(img0 + b * per, n, i, j);
    pb[slot_b * L.plane + L.at(i, j)] = node_from_image(img1 + b * per, n, i, j);
}

// rho = (a/sa - b/sb)/h^2 into RHO (sa, sb per pair)
__global__ void make_source_kernel(double* base, Layout L, int slot_a, int slot_b,
                                   const double* __restrict__ sa, const double* __restrict__ sb,
                                   double h2) {
    const int n = L.n;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    const int b = blockIdx.z;
    if (i > n || j > n) return;
    double* pb = base + (long)b * NSLOT * L.plane;
    const long o = L.at(i, j);
    pb[RHO * L.plane + o] = (pb[slot_a * L.plane + o] / sa[b] - pb[slot_b * L.plane + o] / sb[b]) / h2;
}

// rho -= mean (mean = sum / V per pair), then clear the scratch slots.
__global__ void center_source_kernel(double* base, Layout L, const double* __restrict__ sums,
                                     int clear_a, int clear_b) {
    const int n = L.n;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    const int b = blockIdx.z;
    if (i > n || j > n) return;
    double* pb = base + (long)b * NSLOT * L.plane;
    const long o = L.at(i, j);
    const double V = (double)(n + 1) * (double)(n + 1);
    pb[RHO * L.plane + o] -= sums[b] / V;
    pb[clear_a * L.plane + o] = 0.0;
    pb[clear_b * L.plane + o] = 0.0;
}

// ------------------------------------------------------------ prolongation
// Eq. 14 (phi, nested bilinear) and Eq. 15 (m, nearest along the edge,
// transverse average).  Reads each coarse pair's latest
// buffer (ctl[b].cur), writes buffer 0 of the fine level.
__global__ void prolong_kernel(const double* __restrict__ cbase, Layout Lc,
                               const PairCtl* __restrict__ cctl, double* fbase, Layout Lf) {
    const int nf = Lf.n;
    const int I = blockIdx.x * blockDim.x + threadIdx.x;
    const int J = blockIdx.y * blockDim.y + threadIdx.y;
    const int b = blockIdx.z;
    if (I > nf || J > nf) return;
    const int cur = cctl[b].cur;
    const double* cb = cbase + (long)b * NSLOT * Lc.plane;
    const double* cp = cb + (PHI0 + cur) * Lc.plane;
    const double* cx = cb + (MX0 + cur) * Lc.plane;
    const double* cy = cb + (MY0 + cur) * Lc.plane;
    double* fb = fbase + (long)b * NSLOT * Lf.plane;
    const int i = I >> 1, j = J >> 1;
    const bool io = I & 1, jo = J & 1;
    double v;
    if (!io && !jo) v = cp[Lc.at(i, j)];
    else if (io && !jo) v = 0.5 * (cp[Lc.at(i, j)] + cp[Lc.at(i + 1, j)]);
    else if (!io && jo) v = 0.5 * (cp[Lc.at(i, j)] + cp[Lc.at(i, j + 1)]);
    else
        v = 0.25 * ((cp[Lc.at(i, j)] + cp[Lc.at(i + 1, j)]) +
                    (cp[Lc.at(i, j + 1)] + cp[Lc.at(i + 1, j + 1)]));
    const long o = Lf.at(I, J);
    fb[PHI0 * Lf.plane + o] = v;
    if (I < nf)
        fb[MX0 * Lf.plane + o] = jo ? 0.5 * (cx[Lc.at(i, j)] + cx[Lc.at(i, j + 1)]) : cx[Lc.at(i, j)];
    if (J < nf)
        fb[MY0 * Lf.plane + o] = io ? 0.5 * (cy[Lc.at(i, j)] + cy[Lc.at(i + 1, j)]) : cy[Lc.at(i, j)];
}

// --------------------------------------------------- per-pair reductions
// Compensated sum over the nodes of each pair of f(pair, i, j).  Phase 1:
// grid (G, pairs), each block a contiguous band of rows; phase 2: one block
// per pair merges the G partials in block order.  Deterministic.
constexpr int kRedThreads = 256;

template <class F>
__global__ void __launch_bounds__(kRedThreads)
node_reduce_kernel(F f, int w, int rows, double2* __restrict__ partial) {
    // f(b, i, j) over i in [0, w), j in [0, rows)
    const int b = blockIdx.y;
    const int G = gridDim.x;
    const int r0 = (int)((long)rows * blockIdx.x / G);
    const int r1 = (int)((long)rows * (blockIdx.x + 1) / G);
    Comp acc{0.0, 0.0};
    const long cnt = (long)(r1 - r0) * w;
    for (long t = threadIdx.x; t < cnt; t += kRedThreads) {
        const int j = r0 + (int)(t / w);
        const int i = (int)(t % w);
        acc.add(f(b, i, j));
    }
    acc = warp_comp(acc);
    __shared__ double2 sm[kRedThreads / 32];
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = make_double2(acc.s, acc.c);
    __syncthreads();
    if (threadIdx.x == 0) {
        Comp t{sm[0].x, sm[0].y};
        for (int q = 1; q < kRedThreads / 32; ++q) t.merge(sm[q].x, sm[q].y);
        partial[(long)b * G + blockIdx.x] = make_double2(t.s, t.c);
    }
}

// out[b] = (merged sum * s1) * s2   (grid.cpp:103 multiplies by h twice)
__global__ void reduce_finish_kernel(const double2* __restrict__ partial, int G, double s1,
                                     double s2, double* __restrict__ out) {
    const int b = blockIdx.x;
    if (threadIdx.x != 0) return;
    Comp t{partial[(long)b * G].x, partial[(long)b * G].y};
    for (int g = 1; g < G; ++g) t.merge(partial[(long)b * G + g].x, partial[(long)b * G + g].y);
    out[b] = ((t.s + t.c) * s1) * s2;
}

struct FSlot {  // value of one slot
    const double* base;
    Layout L;
    int slot;
    __device__ double operator()(int b, int i, int j) const {
        return base[((long)b * NSLOT + slot) * L.plane + L.at(i, j)];
    }
};

struct FSlotSq {  // squared value of one slot
    const double* base;
    Layout L;
    int slot;
    __device__ double operator()(int b, int i, int j) const {
        double v = base[((long)b * NSLOT + slot) * L.plane + L.at(i, j)];
        return v * v;
    }
};

struct FDual {  // phi(cur) * rho  (inner_h, grid.cpp:99-104)
    const double* base;
    Layout L;
    const PairCtl* ctl;
    __device__ double operator()(int b, int i, int j) const {
        const double* pb = base + (long)b * NSLOT * L.plane;
        const long o = L.at(i, j);
        return pb[(PHI0 + ctl[b].cur) * L.plane + o] * pb[RHO * L.plane + o];
    }
};

template <int PN>
struct FPrimal {  // ||m(x)||_p over node vectors (grid.cpp:132-138)
    const double* base;
    Layout L;
    const PairCtl* ctl;
    __device__ double operator()(int b, int i, int j) const {
        const double* pb = base + (long)b * NSLOT * L.plane;
        const long o = L.at(i, j);
        const int c = ctl[b].cur;
        double x = (i < L.n) ? pb[(MX0 + c) * L.plane + o] : 0.0;
        double y = (j < L.n) ? pb[(MY0 + c) * L.plane + o] : 0.0;
        return vec_norm<PN>(x, y);
    }
};

// ------------------------------------------------------------ level control
// ctl init for a level: tolerance either absolute or rel * tau * h^2 * sum rho^2.
__global__ void init_ctl_kernel(PairCtl* ctl, int npairs, const double* __restrict__ rho_sq,
                                double rel_scale, double abs_tol, long max_it, int* ndone) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b == 0) *ndone = 0;
    if (b >= npairs) return;
    PairCtl c;
    c.tol = rho_sq ? rel_scale * rho_sq[b] : abs_tol;
    c.fpr = 0.0;
    c.it = 0;
    c.max_it = max_it;
    c.done = max_it <= 0 ? 1 : 0;
    c.cur = 0;
    c.nonfinite = 0;
    c.redo = 0;
    ctl[b] = c;
}

// Active-pair list for a compacted sweep launch: act = running pairs in
// ascending order, *nact = their count.  One block; each thread scans a
// contiguous run of pairs, then a block-wide exclusive scan places the runs.
constexpr int kCompactThreads = 1024;
__global__ void __launch_bounds__(kCompactThreads)
compact_active_kernel(const PairCtl* __restrict__ ctl, int npairs, int* __restrict__ act,
                      int* __restrict__ nact) {
    __shared__ int wsum[kCompactThreads / 32];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int per = (npairs + kCompactThreads - 1) / kCompactThreads;
    const int lo = min(t * per, npairs), hi = min(lo + per, npairs);
    int cnt = 0;
    for (int b = lo; b < hi; ++b) cnt += ctl[b].done ? 0 : 1;
    int incl = cnt;  // warp inclusive scan
    for (int d = 1; d < 32; d <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
        int s = wsum[lane];
        for (int d = 1; d < 32; d <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, s, d);
            if (lane >= d) s += v;
        }
        wsum[lane] = s;  // inclusive over warps
    }
    __syncthreads();
    int pos = incl - cnt + (w > 0 ? wsum[w - 1] : 0);
    for (int b = lo; b < hi; ++b)
        if (!ctl[b].done) act[pos++] = b;
    if (t == kCompactThreads - 1) *nact = pos;
}

// per-level bookkeeping into caller-visible arrays
__global__ void harvest_kernel(const PairCtl* __restrict__ ctl, int npairs, int level, int levels,
                               long* iters, double* fpr, double* tol) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= npairs) return;
    if (iters) iters[(long)b * levels + level] = ctl[b].it;
    if (fpr) fpr[(long)b * levels + level] = ctl[b].fpr;
    if (tol) tol[(long)b * levels + level] = ctl[b].tol;
}

// FP64 peak probe: 8 independent DFMA chains per thread (latency hidden by
// 8 chains x 32 warps per SM); the result is stored only if it is impossible,
// so the chains cannot be optimised away.
__global__ void __launch_bounds__(256) fp64_peak_kernel(long iters, double* sink) {
    double x[8];
    const double a = 1.0 + 1e-12 * threadIdx.x, b = -1e-13;
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = q + blockIdx.x * 1e-9;
    for (long k = 0; k < iters; ++k)
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q] = fma(x[q], a, b);
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += x[q];
    if (s == -1.2345e300) *sink = s;
}

__global__ void converged_kernel(const PairCtl* __restrict__ ctl, int npairs, int* conv) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= npairs) return;
    conv[b] = (ctl[b].fpr < ctl[b].tol && !ctl[b].nonfinite) ? 1 : 0;
}

// ---------------------------------------------- reference-layout utilities
// Copies a state (phi, mx, my) from the pair's latest buffer out to dense
// reference-layout arrays (proj/include/w1mg/grid.hpp:30-61).
__global__ void unpack_state_kernel(const double* __restrict__ base, Layout L,
                                    const PairCtl* __restrict__ ctl, int pair, double* phi,
                                    double* mx, double* my) {
    const int n = L.n;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    if (i > n || j > n) return;
    const double* pb = base + (long)pair * NSLOT * L.plane;
    const int c = ctl ? ctl[pair].cur : 0;
    const long o = L.at(i, j);
    if (phi) phi[(long)j * (n + 1) + i] = pb[(PHI0 + c) * L.plane + o];
    if (mx && i < n) mx[(long)j * n + i] = pb[(MX0 + c) * L.plane + o];
    if (my && j < n) my[(long)j * (n + 1) + i] = pb[(MY0 + c) * L.plane + o];
}

__global__ void sub_inplace_kernel(double* __restrict__ a, const double* __restrict__ b, long count) {
    const long k = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (k < count) a[k] = a[k] - b[k];
}

// Reference-layout operators for the grid API (test / value paths).
__global__ void divergence_ref_kernel(int n, const double* __restrict__ mx,
                                      const double* __restrict__ my, double* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    if (i > n || j > n) return;
    const double ih = 1.0 / (1.0 / n);
    double l = (i > 0) ? mx[(long)j * n + i - 1] : 0.0;
    double r = (i < n) ? mx[(long)j * n + i] : 0.0;
    double b = (j > 0) ? my[(long)(j - 1) * (n + 1) + i] : 0.0;
    double a = (j < n) ? my[(long)j * (n + 1) + i] : 0.0;
    out[(long)j * (n + 1) + i] = (r - l) * ih + (a - b) * ih;
}

__global__ void adjoint_ref_kernel(int n, const double* __restrict__ phi, double* __restrict__ gx,
                                   double* __restrict__ gy) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    if (i > n || j > n) return;
    const double ih = 1.0 / (1.0 / n);
    const long o = (long)j * (n + 1) + i;
    if (i < n) gx[(long)j * n + i] = (phi[o] - phi[o + 1]) * ih;
    if (j < n) gy[o] = (phi[o] - phi[o + n + 1]) * ih;
}

struct FRefDot {  // a[k]*b[k] over a dense array of `count` entries laid out as rows of w
    const double* a;
    const double* b;
    int w;
    __device__ double operator()(int, int i, int j) const {
        const long k = (long)j * w + i;
        return a[k] * b[k];
    }
};

template <int PN>
struct FRefPrimal {
    const double* mx;
    const double* my;
    int n;
    __device__ double operator()(int, int i, int j) const {
        double x = (i < n) ? mx[(long)j * n + i] : 0.0;
        double y = (j < n) ? my[(long)j * (n + 1) + i] : 0.0;
        return vec_norm<PN>(x, y);
    }
};

}  // namespace w1mg_dev

namespace w1mg_dev {
// Deterministic synthetic source for kernel probes (not a solver input path):
// a smooth zero-mean-ish pattern per pair.
__global__ void probe_fill_kernel(double* base, Layout L) {
    const int n = L.n;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    const int b = blockIdx.z;
    if (i > n || j > n) return;
    double x = (double)i / n, y = (double)j / n;
    double v = sin(6.283185307179586 * (x + 0.37 * b)) * cos(3.141592653589793 * (2.0 * y + 0.11 * b));
    base[((long)b * NSLOT + RHO) * L.plane + L.at(i, j)] = v * n * n * 1e-3;
}
}  // namespace w1mg_dev
