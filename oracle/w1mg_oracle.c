/*
 * w1mg_oracle.c -- CPU restatement of the reference W1 primal-dual path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path in paper_1810_00118_b200/.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product library never links or calls it.
 *
 * Every routine restates the algorithm of the reference (paths relative to
 * /root/reference) in plain C99.  Element-wise arithmetic is written in the
 * same operation order as the reference so that, compiled with
 * -ffp-contract=off, the fields it produces are bit-identical to the
 * reference build (checked in tests/test_oracle_vs_ref.py against
 * oracle/_ref/libw1mg_ref.so).  Residual reductions are plain left-to-right
 * sums in node order, exactly like proj/src/solver_cp.cpp:30-68, so even the
 * FPR history is bit-identical.
 *
 * Layouts (proj/include/w1mg/grid.hpp:30-61):
 *   scalar  phi[j*(n+1)+i]  i,j in 0..n
 *   x-edges mx[j*n+i]       i in 0..n-1, j in 0..n
 *   y-edges my[j*(n+1)+i]   i in 0..n,   j in 0..n-1
 *
 * Pieces without a reference implementation are restated from SPEC.md:
 * prolongation Eq. 14/15, the cascade driver
 * and the frozen image->node source rule of SURVEY D2/D4.
 */
#include <math.h>
#include <stddef.h>
#include <stdlib.h>
#include <string.h>

#define OR_P1 0
#define OR_P2 1
#define OR_PINF 2

/* ---------------------------------------------------------------------- */
/* compensated sums: proj/src/grid.cpp:13-33 (Neumaier)                    */

typedef struct { double s, c; } or_acc;

static void acc_add(or_acc* a, double v) {
    double t = a->s + v;
    if (fabs(a->s) >= fabs(v)) a->c += (a->s - t) + v;
    else a->c += (v - t) + a->s;
    a->s = t;
}
static double acc_val(const or_acc* a) { return a->s + a->c; }

double or_compensated_sum(const double* v, long count) {
    or_acc a = {0.0, 0.0};
    for (long k = 0; k < count; ++k) acc_add(&a, v[k]);
    return acc_val(&a);
}

/* SourceField gate, proj/src/grid.cpp:35-43: returns 1 when compatible. */
int or_source_compatible(const double* rho, long count) {
    or_acc tot = {0.0, 0.0}, ab = {0.0, 0.0};
    for (long k = 0; k < count; ++k) {
        acc_add(&tot, rho[k]);
        acc_add(&ab, fabs(rho[k]));
    }
    return !(fabs(acc_val(&tot)) > 1e-12 * acc_val(&ab));
}

/* ---------------------------------------------------------------------- */
/* prox, proj/src/prox.cpp:10-62 and proj/include/w1mg/pnorm.hpp:32-39     */

static double dmax_std(double a, double b) { return (a < b) ? b : a; } /* std::max */
static double dmin_std(double a, double b) { return (b < a) ? b : a; } /* std::min */

static double soft(double v, double mu) { /* prox.cpp:10-12 */
    return copysign(dmax_std(fabs(v) - mu, 0.0), v);
}

/* prox.cpp:16-25 (radius > 0 checked by the caller) */
void or_project_l1_ball(double vx, double vy, double r, double* ox, double* oy) {
    double ax = fabs(vx), ay = fabs(vy);
    if (ax + ay <= r) { *ox = vx; *oy = vy; return; }
    double hi = dmax_std(ax, ay), lo = dmin_std(ax, ay);
    double th = (hi - r >= lo) ? hi - r : 0.5 * (ax + ay - r);
    *ox = soft(vx, th);
    *oy = soft(vy, th);
}

/* prox.cpp:27-45 */
void or_shrink(double vx, double vy, double mu, int p, double* ox, double* oy) {
    if (p == OR_P1) {
        *ox = soft(vx, mu);
        *oy = soft(vy, mu);
    } else if (p == OR_P2) {
        double nrm = sqrt(vx * vx + vy * vy);
        if (nrm <= mu) { *ox = 0.0; *oy = 0.0; return; }
        double s = 1.0 - mu / nrm;
        *ox = s * vx;
        *oy = s * vy;
    } else {
        double qx, qy;
        or_project_l1_ball(vx, vy, mu, &qx, &qy);
        *ox = vx - qx;
        *oy = vy - qy;
    }
}

/* prox.cpp:47-62 */
void or_project_unit_ball(double vx, double vy, int q, double* ox, double* oy) {
    if (q == OR_P1) {
        if (fabs(vx) + fabs(vy) <= 1.0) { *ox = vx; *oy = vy; return; }
        or_project_l1_ball(vx, vy, 1.0, ox, oy);
    } else if (q == OR_P2) {
        double n2 = vx * vx + vy * vy;
        if (n2 <= 1.0) { *ox = vx; *oy = vy; return; }
        double s = 1.0 / sqrt(n2);
        *ox = s * vx;
        *oy = s * vy;
    } else {
        *ox = (vx < -1.0) ? -1.0 : ((1.0 < vx) ? 1.0 : vx);
        *oy = (vy < -1.0) ? -1.0 : ((1.0 < vy) ? 1.0 : vy);
    }
}

static double vec_norm(double x, double y, int p) { /* pnorm.hpp:32-39 */
    if (p == OR_P1) return fabs(x) + fabs(y);
    if (p == OR_P2) return sqrt(x * x + y * y);
    return dmax_std(fabs(x), fabs(y));
}

/* ---------------------------------------------------------------------- */
/* grid operators, proj/src/grid.cpp:45-142                                */

/* grid.cpp:45-68: x pass assigns, y pass adds. */
void or_divergence(int n, const double* mx, const double* my, double* out) {
    const double ih = 1.0 / (1.0 / n);
    const int w = n + 1;
    for (int j = 0; j <= n; ++j)
        for (int i = 0; i <= n; ++i) {
            double l = (i > 0) ? mx[(size_t)j * n + i - 1] : 0.0;
            double r = (i < n) ? mx[(size_t)j * n + i] : 0.0;
            out[(size_t)j * w + i] = (r - l) * ih;
        }
    for (int j = 0; j <= n; ++j)
        for (int i = 0; i <= n; ++i) {
            double b = (j > 0) ? my[(size_t)(j - 1) * w + i] : 0.0;
            double a = (j < n) ? my[(size_t)j * w + i] : 0.0;
            out[(size_t)j * w + i] += (a - b) * ih;
        }
}

/* grid.cpp:76-91: negative forward difference. */
void or_adjoint(int n, const double* phi, double* gx, double* gy) {
    const double ih = 1.0 / (1.0 / n);
    const int w = n + 1;
    for (int j = 0; j <= n; ++j)
        for (int i = 0; i < n; ++i)
            gx[(size_t)j * n + i] = (phi[(size_t)j * w + i] - phi[(size_t)j * w + i + 1]) * ih;
    for (int j = 0; j < n; ++j)
        for (int i = 0; i <= n; ++i)
            gy[(size_t)j * w + i] = (phi[(size_t)j * w + i] - phi[(size_t)(j + 1) * w + i]) * ih;
}

/* grid.cpp:99-104 */
double or_inner_h_nodes(int n, const double* a, const double* b) {
    double h = 1.0 / n;
    or_acc s = {0.0, 0.0};
    long cnt = (long)(n + 1) * (n + 1);
    for (long k = 0; k < cnt; ++k) acc_add(&s, a[k] * b[k]);
    return acc_val(&s) * h * h;
}

/* grid.cpp:106-112 */
double or_inner_h_edges(int n, const double* ax, const double* ay, const double* bx,
                        const double* by) {
    double h = 1.0 / n;
    or_acc s = {0.0, 0.0};
    long cnt = (long)n * (n + 1);
    for (long k = 0; k < cnt; ++k) acc_add(&s, ax[k] * bx[k]);
    for (long k = 0; k < cnt; ++k) acc_add(&s, ay[k] * by[k]);
    return acc_val(&s) * h * h;
}

/* grid.cpp:132-138: node vectors of outgoing edges, absent = 0. */
double or_primal_value(int n, const double* mx, const double* my, int p) {
    double h = 1.0 / n;
    or_acc s = {0.0, 0.0};
    for (int j = 0; j <= n; ++j)
        for (int i = 0; i <= n; ++i) {
            double x = (i < n) ? mx[(size_t)j * n + i] : 0.0;
            double y = (j < n) ? my[(size_t)j * (n + 1) + i] : 0.0;
            acc_add(&s, vec_norm(x, y, p));
        }
    return acc_val(&s) * h * h;
}

/* grid.cpp:140-142 */
double or_dual_value(int n, const double* phi, const double* rho) {
    return or_inner_h_nodes(n, phi, rho);
}

/* grid.cpp:130 and solver_cp.cpp:75-78 */
double or_cp_step_size(int n, int safe) {
    double h = 1.0 / n;
    double bound = 2.0 * sqrt(2.0) / h;
    return safe ? 1.0 / (2.0 * bound) : 1.0 / bound;
}

/* ---------------------------------------------------------------------- */
/* Algorithm 1: proj/src/solver_cp.cpp:22-71 (one sweep, in place).        */

typedef struct {
    double *dx, *dy, *divm, *divd;
} or_cp_scratch;

static double cp_sweep(int n, double* mx, double* my, double* phi, const double* rho, int p,
                       double mu, double tau, or_cp_scratch* s) {
    const double h = 1.0 / n;
    const double h2 = h * h;
    const double ih = 1.0 / h;
    const int w = n + 1;
    double sdm2 = 0.0;
    /* m-update over node vectors (solver_cp.cpp:31-56); A*phi inlined with
       the same expression as grid.cpp:83,89. */
    for (int j = 0; j <= n; ++j) {
        const int hy = j < n;
        for (int i = 0; i <= n; ++i) {
            const int hx = i < n;
            size_t kx = (size_t)j * n + i, ky = (size_t)j * w + i;
            double vx = 0.0, vy = 0.0;
            if (hx) {
                double g = (phi[ky] - phi[ky + 1]) * ih;
                vx = mx[kx] - mu * g;
            }
            if (hy) {
                double g = (phi[ky] - phi[ky + w]) * ih;
                vy = my[ky] - mu * g;
            }
            double ux, uy;
            or_shrink(vx, vy, mu, p, &ux, &uy);
            if (hx) {
                double d = ux - mx[kx];
                s->dx[kx] = d;
                mx[kx] = ux;
                sdm2 += d * d;
            }
            if (hy) {
                double d = uy - my[ky];
                s->dy[ky] = d;
                my[ky] = uy;
                sdm2 += d * d;
            }
        }
    }
    or_divergence(n, mx, my, s->divm);
    or_divergence(n, s->dx, s->dy, s->divd);
    double sdp2 = 0.0, scr = 0.0;
    const long V = (long)w * w;
    for (long k = 0; k < V; ++k) { /* solver_cp.cpp:62-68 */
        double d = tau * (s->divm[k] + s->divd[k] - rho[k]);
        phi[k] += d;
        sdp2 += d * d;
        scr += d * s->divd[k];
    }
    return h2 * (sdm2 / mu + sdp2 / tau - 2.0 * scr);
}

/*
 * cp_run, proj/src/solver_cp.cpp:113-147.  Zero start when m0x/phi0 are
 * NULL.  Runs until fpr < tol or max_iters.  Outputs are written to
 * mx/my/phi (caller-allocated, reference layout).
 */
int or_cp_run(int n, const double* rho, const double* m0x, const double* m0y, const double* phi0,
              int p, double mu, double tau, double tol, long max_iters, double* mx, double* my,
              double* phi, double* hist, long hist_cap, long* iters, int* converged,
              double* distance, double* dual, double* fpr_final) {
    const size_t E = (size_t)n * (n + 1), V = (size_t)(n + 1) * (n + 1);
    if (m0x) { memcpy(mx, m0x, E * 8); memcpy(my, m0y, E * 8); }
    else { memset(mx, 0, E * 8); memset(my, 0, E * 8); }
    if (phi0) memcpy(phi, phi0, V * 8);
    else memset(phi, 0, V * 8);
    or_cp_scratch s;
    s.dx = (double*)calloc(E, 8);
    s.dy = (double*)calloc(E, 8);
    s.divm = (double*)calloc(V, 8);
    s.divd = (double*)calloc(V, 8);
    if (!s.dx || !s.dy || !s.divm || !s.divd) return 3;
    long k = 0;
    double fpr = 0.0;
    int conv = 0;
    while (k < max_iters) {
        fpr = cp_sweep(n, mx, my, phi, rho, p, mu, tau, &s);
        if (hist && k < hist_cap) hist[k] = fpr;
        ++k;
        if (fpr < tol) { conv = 1; break; }
    }
    free(s.dx); free(s.dy); free(s.divm); free(s.divd);
    *iters = k;
    *converged = conv;
    *fpr_final = fpr;
    *distance = or_primal_value(n, mx, my, p);
    *dual = or_dual_value(n, phi, rho);
    return 0;
}

/* One sweep restricted to node rows [jlo, jhi) of a full-grid state: the
   row-slab view of cp_sweep used by the CPU multi-process test of the config-5
   decomposition.  Reads phi rows [jlo-1, jhi], m rows [jlo-1, jhi) (halo
   rows included), writes m and phi of the owned rows into o* (other rows are
   left untouched) and the three partial sums of solver_cp.cpp:70 for the
   owned nodes into sums[3]. */
void or_cp_sweep_rows(int n, int jlo, int jhi, const double* mx, const double* my,
                      const double* phi, const double* rho, int p, double mu, double tau,
                      double* omx, double* omy, double* ophi, double* sums) {
    const double ih = 1.0 / (1.0 / n);
    const int w = n + 1;
    const int r0 = jlo > 0 ? jlo - 1 : 0;
    const int nr = jhi - r0;
    double* ux = (double*)calloc((size_t)nr * w, 8);
    double* uy = (double*)calloc((size_t)nr * w, 8);
    double* dx = (double*)calloc((size_t)nr * w, 8);
    double* dy = (double*)calloc((size_t)nr * w, 8);
    double sdm2 = 0.0, sdp2 = 0.0, scr = 0.0;
    for (int j = r0; j < jhi; ++j) {
        const int hy = j < n;
        for (int i = 0; i <= n; ++i) {
            const int hx = i < n;
            size_t kx = (size_t)j * n + i, ky = (size_t)j * w + i, kl = (size_t)(j - r0) * w + i;
            double vx = 0.0, vy = 0.0;
            if (hx) vx = mx[kx] - mu * ((phi[ky] - phi[ky + 1]) * ih);
            if (hy) vy = my[ky] - mu * ((phi[ky] - phi[ky + w]) * ih);
            double a, b;
            or_shrink(vx, vy, mu, p, &a, &b);
            if (hx) { dx[kl] = a - mx[kx]; ux[kl] = a; }
            if (hy) { dy[kl] = b - my[ky]; uy[kl] = b; }
            if (j >= jlo) {
                if (hx) sdm2 += dx[kl] * dx[kl];
                if (hy) sdm2 += dy[kl] * dy[kl];
            }
        }
    }
    for (int j = jlo; j < jhi; ++j)
        for (int i = 0; i <= n; ++i) {
            size_t kl = (size_t)(j - r0) * w + i, kg = (size_t)j * w + i;
            double l = (i > 0) ? ux[kl - 1] : 0.0, r = (i < n) ? ux[kl] : 0.0;
            double b = (j > 0) ? uy[kl - w] : 0.0, a = (j < n) ? uy[kl] : 0.0;
            double divm = (r - l) * ih + (a - b) * ih;
            double dl = (i > 0) ? dx[kl - 1] : 0.0, dr = (i < n) ? dx[kl] : 0.0;
            double db = (j > 0) ? dy[kl - w] : 0.0, da = (j < n) ? dy[kl] : 0.0;
            double divd = (dr - dl) * ih + (da - db) * ih;
            double d = tau * (divm + divd - rho[kg]);
            ophi[kg] = phi[kg] + d;
            if (i < n) omx[(size_t)j * n + i] = ux[kl];
            if (j < n) omy[kg] = uy[kl];
            sdp2 += d * d;
            scr += d * divd;
        }
    free(ux); free(uy); free(dx); free(dy);
    sums[0] = sdm2;
    sums[1] = sdp2;
    sums[2] = scr;
}

/* cp_residual, proj/src/solver_cp.cpp:102-111 */
double or_cp_residual(int n, const double* cmx, const double* cmy, const double* cphi,
                      const double* pmx, const double* pmy, const double* pphi, double mu,
                      double tau) {
    const size_t E = (size_t)n * (n + 1), V = (size_t)(n + 1) * (n + 1);
    double* dx = (double*)malloc(E * 8);
    double* dy = (double*)malloc(E * 8);
    double* dp = (double*)malloc(V * 8);
    double* adm = (double*)malloc(V * 8);
    for (size_t k = 0; k < E; ++k) { dx[k] = cmx[k] - pmx[k]; dy[k] = cmy[k] - pmy[k]; }
    for (size_t k = 0; k < V; ++k) dp[k] = cphi[k] - pphi[k];
    or_divergence(n, dx, dy, adm);
    double nm = sqrt(or_inner_h_edges(n, dx, dy, dx, dy));
    double np = sqrt(or_inner_h_nodes(n, dp, dp));
    double r = nm * nm / mu + np * np / tau - 2.0 * or_inner_h_nodes(n, dp, adm);
    free(dx); free(dy); free(dp); free(adm);
    return r;
}

/* ---------------------------------------------------------------------- */
/* Multilevel: Eq. 14 / Eq. 15 prolongation (SPEC.md:338-355,            */
/* PAPER.md:336-406).  Coarse nc cells -> fine nf = 2 nc cells.            */

void or_prolong_scalar(int nc, const double* c, double* f) {
    const int wc = nc + 1, nf = 2 * nc, wf = nf + 1;
    for (int J = 0; J <= nf; ++J)
        for (int I = 0; I <= nf; ++I) {
            int i = I >> 1, j = J >> 1;
            double v;
            if (!(I & 1) && !(J & 1)) v = c[(size_t)j * wc + i];
            else if ((I & 1) && !(J & 1)) v = 0.5 * (c[(size_t)j * wc + i] + c[(size_t)j * wc + i + 1]);
            else if (!(I & 1) && (J & 1)) v = 0.5 * (c[(size_t)j * wc + i] + c[(size_t)(j + 1) * wc + i]);
            else
                v = 0.25 * ((c[(size_t)j * wc + i] + c[(size_t)j * wc + i + 1]) +
                            (c[(size_t)(j + 1) * wc + i] + c[(size_t)(j + 1) * wc + i + 1]));
            f[(size_t)J * wf + I] = v;
        }
}

/* Eq. 15: nearest coarse edge along the edge direction (floor(I/2)), the
   transverse coordinate averaged as in Eq. 14. */
void or_prolong_flux(int nc, const double* cx, const double* cy, double* fx, double* fy) {
    const int wc = nc + 1, nf = 2 * nc, wf = nf + 1;
    for (int J = 0; J <= nf; ++J) /* x-edges: I in 0..nf-1 */
        for (int I = 0; I < nf; ++I) {
            int i = I >> 1, j = J >> 1;
            double v = (J & 1) ? 0.5 * (cx[(size_t)j * nc + i] + cx[(size_t)(j + 1) * nc + i])
                               : cx[(size_t)j * nc + i];
            fx[(size_t)J * nf + I] = v;
        }
    for (int J = 0; J < nf; ++J) /* y-edges: J in 0..nf-1 */
        for (int I = 0; I <= nf; ++I) {
            int i = I >> 1, j = J >> 1;
            double v = (I & 1) ? 0.5 * (cy[(size_t)j * wc + i] + cy[(size_t)j * wc + i + 1])
                               : cy[(size_t)j * wc + i];
            fy[(size_t)J * wf + I] = v;
        }
}

/* ---------------------------------------------------------------------- */
/* Sources (frozen rule).                                    */

/* 2x2 block sums of an m x m cell image -> (m/2) x (m/2). */
void or_block_sum(int m, const double* img, double* out) {
    const int mc = m / 2;
    for (int j = 0; j < mc; ++j)
        for (int i = 0; i < mc; ++i) {
            const double* r0 = img + (size_t)(2 * j) * m + 2 * i;
            const double* r1 = r0 + m;
            out[(size_t)j * mc + i] = (r0[0] + r0[1]) + (r1[0] + r1[1]);
        }
}

/* cell image (n x n, cell centres) -> node values ((n+1)^2): the mean of the
   cells touching the node (4 interior, 2 on a side, 1 at a corner). */
void or_image_to_nodes(int n, const double* img, double* nodes) {
    const int w = n + 1;
    for (int j = 0; j <= n; ++j)
        for (int i = 0; i <= n; ++i) {
            int il = i > 0, ir = i < n, jl = j > 0, jr = j < n;
            double v;
            if (il && ir && jl && jr) {
                v = 0.25 * ((img[(size_t)(j - 1) * n + i - 1] + img[(size_t)(j - 1) * n + i]) +
                            (img[(size_t)j * n + i - 1] + img[(size_t)j * n + i]));
            } else if (jl && jr) { /* left or right side */
                int c = il ? i - 1 : i;
                v = 0.5 * (img[(size_t)(j - 1) * n + c] + img[(size_t)j * n + c]);
            } else if (il && ir) { /* bottom or top side */
                int r = jl ? j - 1 : j;
                v = 0.5 * (img[(size_t)r * n + i - 1] + img[(size_t)r * n + i]);
            } else {
                int c = il ? i - 1 : i, r = jl ? j - 1 : j;
                v = img[(size_t)r * n + c];
            }
            nodes[(size_t)j * w + i] = v;
        }
}

/* rho = (a/sum a - b/sum b)/h^2, then subtract the compensated mean
   (SPEC.md:479 make_source). */
void or_make_source(int n, const double* a, const double* b, double* rho) {
    const long V = (long)(n + 1) * (n + 1);
    double sa = or_compensated_sum(a, V), sb = or_compensated_sum(b, V);
    double h = 1.0 / n;
    double h2 = h * h;
    for (long k = 0; k < V; ++k) rho[k] = (a[k] / sa - b[k] / sb) / h2;
    double mean = or_compensated_sum(rho, V) / (double)V;
    for (long k = 0; k < V; ++k) rho[k] -= mean;
}

/* Per-level sources, coarse to fine, concatenated.  img0/img1 are the
   finest m x m cell images (m = n_finest).  out holds sum_l (n_l+1)^2. */
void or_ml_sources(int m, const double* img0, const double* img1, int levels, double* out) {
    double *a = (double*)malloc((size_t)m * m * 8), *b = (double*)malloc((size_t)m * m * 8);
    double *ta = (double*)malloc((size_t)m * m * 8), *tb = (double*)malloc((size_t)m * m * 8);
    double *na = (double*)malloc((size_t)(m + 1) * (m + 1) * 8);
    double *nb = (double*)malloc((size_t)(m + 1) * (m + 1) * 8);
    memcpy(a, img0, (size_t)m * m * 8);
    memcpy(b, img1, (size_t)m * m * 8);
    size_t off_total = 0;
    for (int l = 0; l < levels; ++l) {
        int nl = m >> (levels - 1 - l);
        off_total += (size_t)(nl + 1) * (nl + 1);
    }
    /* walk fine -> coarse, writing each level at its slot */
    int cur = m;
    size_t off = off_total;
    for (int l = levels - 1; l >= 0; --l) {
        size_t V = (size_t)(cur + 1) * (cur + 1);
        off -= V;
        or_image_to_nodes(cur, a, na);
        or_image_to_nodes(cur, b, nb);
        or_make_source(cur, na, nb, out + off);
        if (l > 0) {
            or_block_sum(cur, a, ta);
            or_block_sum(cur, b, tb);
            double* t = a; a = ta; ta = t;
            t = b; b = tb; tb = t;
            cur /= 2;
        }
    }
    free(a); free(b); free(ta); free(tb); free(na); free(nb);
}

/* ---------------------------------------------------------------------- */
/* Cascadic Algorithm 3: level 0 cold, then Eq. 14/15   */
/* warm starts.  rho holds the per-level sources coarse->fine.  eps[l] is  */
/* the absolute tolerance for level l; if rel_tol > 0 it is replaced by    */
/* rel_tol * R_cold,l = rel_tol * tau_l * ||rho_l||^2_L2.       */
int or_ml_cp_run(int n_finest, int levels, const double* rho, int p, int safe, double rel_tol,
                 const double* eps, long max_iters, double* mx, double* my, double* phi,
                 long* level_iters, double* level_eps, double* level_fpr, double* distance,
                 double* dual) {
    int n0 = n_finest >> (levels - 1);
    size_t Ef = (size_t)n_finest * (n_finest + 1), Vf = (size_t)(n_finest + 1) * (n_finest + 1);
    double *cx = (double*)malloc(Ef * 8), *cy = (double*)malloc(Ef * 8), *cp = (double*)malloc(Vf * 8);
    double *wx = (double*)malloc(Ef * 8), *wy = (double*)malloc(Ef * 8), *wp = (double*)malloc(Vf * 8);
    size_t off = 0;
    int rc = 0;
    for (int l = 0; l < levels; ++l) {
        int n = n0 << l;
        const double* r = rho + off;
        size_t V = (size_t)(n + 1) * (n + 1);
        double step = or_cp_step_size(n, safe);
        double tol;
        if (rel_tol > 0) {
            double hh = 1.0 / n;
            or_acc ss = {0.0, 0.0};
            for (size_t k = 0; k < V; ++k) acc_add(&ss, r[k] * r[k]);
            tol = rel_tol * step * (hh * hh * acc_val(&ss));
        } else {
            tol = eps[l];
        }
        if (level_eps) level_eps[l] = tol;
        long it; int conv; double dist, du, ff;
        if (l == 0) {
            rc = or_cp_run(n, r, NULL, NULL, NULL, p, step, step, tol, max_iters, cx, cy, cp, NULL,
                           0, &it, &conv, &dist, &du, &ff);
        } else {
            or_prolong_flux(n / 2, cx, cy, wx, wy);
            or_prolong_scalar(n / 2, cp, wp);
            rc = or_cp_run(n, r, wx, wy, wp, p, step, step, tol, max_iters, cx, cy, cp, NULL, 0,
                           &it, &conv, &dist, &du, &ff);
        }
        if (rc) break;
        if (level_iters) level_iters[l] = it;
        if (level_fpr) level_fpr[l] = ff;
        *distance = dist;
        *dual = du;
        off += V;
    }
    if (!rc) {
        memcpy(mx, cx, Ef * 8);
        memcpy(my, cy, Ef * 8);
        memcpy(phi, cp, Vf * 8);
    }
    free(cx); free(cy); free(cp); free(wx); free(wy); free(wp);
    return rc;
}
