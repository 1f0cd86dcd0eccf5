// capi.cu -- the extern "C" boundary (include/w1mg_cuda.h).  The context and
// error plumbing live in host_common.cuh, the per-level device engine (level
// batches, sweep engines and their selection, the CUDA-graph sweep loop with
// device-side convergence) in level_engine.cuh; this file holds the entry
// points: grid operators, Algorithm 1, cascades and batched cascades.  The
// PDHG and row-slab entry points are in pdhg_engine.cuh / slab_engine.cuh,
// included at the end (one translation unit).
//
// Reference call stacks this replaces (paths relative to /root/reference):
//   cp_run           proj/src/solver_cp.cpp:113-147
//   cp_residual      proj/src/solver_cp.cpp:102-111
//   grid operators   proj/src/grid.cpp:45-142
//   ml_run (spec)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/w1mg_cuda.h"
#include "level_kernels.cuh"
#include "ref_kernels.cuh"
#include "cp2_kernels.cuh"
#include "cluster_kernels.cuh"
#include "cp3_kernels.cuh"
#include "dct_kernels.cuh"

using namespace w1mg_dev;

#include "host_common.cuh"
#include "level_engine.cuh"


// ======================================================================
extern "C" {

const char* w1mg_last_error(void) { return g_err.c_str(); }
int w1mg_abi_version(void) { return W1MG_ABI_VERSION; }

int w1mg_ctx_create(int device, w1mg_ctx** out) {
    return guard([&] {
        if (!out) fail(W1MG_EINVAL, "null out");
        int ndev = 0;
        CK(cudaGetDeviceCount(&ndev));
        if (device < 0 || device >= ndev) fail(W1MG_EINVAL, "no such CUDA device");
        CK(cudaSetDevice(device));
        int major = 0;
        CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
        if (major < 10) fail(W1MG_ECUDA, "this build targets sm_100a (B200)");
        if (const char* v = std::getenv("W1MG_SWEEP"))
            g_sweep_variant = (std::string(v) == "tma") ? kTma
                              : (std::string(v) == "tma2") ? kTma2
                              : (std::string(v) == "tma2t") ? kTma2T
                              : (std::string(v) == "tma3")  ? kTma3
                                                            : kAuto;
        if (const char* v = std::getenv("W1MG_RESIDENT")) g_resident = std::atoi(v);
        if (const char* v = std::getenv("W1MG_COMPACT")) g_compact = std::atoi(v) != 0;
        if (const char* v = std::getenv("W1MG_CLUSTER_PICK")) g_cluster_pick = std::atoi(v);
        if (const char* v = std::getenv("W1MG_PDHG_SMALL")) g_pdhg_small = std::atoi(v);
        if (const char* v = std::getenv("W1MG_WARPS_PER_SM")) g_warps_per_sm = std::max(1, std::atoi(v));
        if (const char* v = std::getenv("W1MG_PDL")) g_pdl = std::atoi(v) != 0;
        if (const char* v = std::getenv("W1MG_FAST")) g_fast = std::atoi(v) != 0;
        if (const char* v = std::getenv("W1MG_OCC3")) g_occ3 = std::atoi(v) == 4 ? 4 : 5;
        if (const char* v = std::getenv("W1MG_PDHG_PERSIST")) g_pdhg_persist = std::atoi(v) != 0;
        if (const char* v = std::getenv("W1MG_PDHG_RS")) g_pdhg_rs = std::atoi(v);
        // Nsight Compute cannot replay the cooperative cluster launch of
        // pdhg_rs2_kernel (LaunchFailed, then a sticky error): under the
        // profiler the 257^2-class levels take the one-CTA-per-SM path
        else if (std::getenv("NV_COMPUTE_PROFILER_PERFWORKS_DIR") && g_pdhg_rs == 1) g_pdhg_rs = 4;
        if (const char* v = std::getenv("W1MG_SLAB_MIN_N")) g_slab_min_n = std::max(1, std::atoi(v));
        if (const char* v = std::getenv("W1MG_COMPACT_STEP")) g_compact_step = std::max(1, std::atoi(v));
        if (const char* v = std::getenv("W1MG_TMAP_NW")) {
            const int w = std::atoi(v);
            g_tmap_nw = (w == 2 || w == 4 || w == 8) ? w : 0;
        }
        auto* c = new w1mg_ctx();
        c->device = device;
        CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
        CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        CK(cudaHostAlloc(reinterpret_cast<void**>(&c->pinned), 2 * sizeof(int), cudaHostAllocDefault));
        for (auto& e : c->ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CK(cudaEventCreate(&c->t0));
        CK(cudaEventCreate(&c->t1));
        *out = c;
    });
}

void w1mg_ctx_destroy(w1mg_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    for (auto& g : c->graphs) cudaGraphExecDestroy(g.second);
    for (auto& b : c->bufs)
        if (b.second.p) cudaFree(b.second.p);
    if (c->pinned) cudaFreeHost(c->pinned);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : c->lev_ev) cudaEventDestroy(e);
    if (c->t0) cudaEventDestroy(c->t0);
    if (c->t1) cudaEventDestroy(c->t1);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

long w1mg_ctx_launch_count(const w1mg_ctx* c) { return c ? c->launches : 0; }

int w1mg_ctx_level_seconds(w1mg_ctx* c, double* out, int cap) {
    int n = 0;
    int rc = guard([&] {
        std::vector<double> s;
        level_seconds(c, s);
        for (; n < cap && n < (int)s.size(); ++n) out[n] = s[n];
    });
    return rc ? -rc : n;
}

int w1mg_ctx_synchronize(w1mg_ctx* c) {
    return guard([&] { CK(cudaStreamSynchronize(c->stream)); });
}

void* w1mg_ctx_stream(w1mg_ctx* c) { return c ? (void*)c->stream : nullptr; }

double w1mg_cp_step_size(int n, int step_mode) {
    const double h = 1.0 / n;                      // GridSpec, grid.hpp:19
    const double bound = 2.0 * std::sqrt(2.0) / h;  // grid.cpp:130
    return step_mode == W1MG_STEP_SAFE ? 1.0 / (2.0 * bound) : 1.0 / bound;
}

double w1mg_pdhg_step_size(int step_mode) { return step_mode == W1MG_STEP_SAFE ? 0.5 : 1.0; }

int w1mg_make_schedule(int n_finest, int levels, double eps_finest, double alpha, double* eps) {
    return guard([&] {
        check_n(n_finest);
        if (levels < 1 || n_finest % (1 << (levels - 1)) != 0)
            fail(W1MG_EINVAL, "make_schedule: N must be divisible by 2^(L-1)");
        if (!(eps_finest > 0)) fail(W1MG_EINVAL, "make_schedule: eps_L must be positive");
        for (int l = 0; l < levels; ++l) {
            // h_l / h_L = 2^(L-1-l)   (Eq. 16)
            eps[l] = eps_finest * std::pow(std::ldexp(1.0, levels - 1 - l), alpha);
        }
    });
}

int w1mg_source_check(int n, const double* rho) {
    return guard([&] {
        check_n(n);
        double s = 0, cs = 0, a = 0, ca = 0;  // Neumaier, grid.cpp:13-25
        auto add = [](double& sum, double& comp, double v) {
            double t = sum + v;
            if (std::fabs(sum) >= std::fabs(v)) comp += (sum - t) + v;
            else comp += (v - t) + sum;
            sum = t;
        };
        const long V = (long)(n + 1) * (n + 1);
        for (long k = 0; k < V; ++k) {
            add(s, cs, rho[k]);
            add(a, ca, std::fabs(rho[k]));
        }
        if (std::fabs(s + cs) > 1e-12 * (a + ca))
            fail(W1MG_EINVAL, "SourceField: values do not sum to zero");
    });
}

// ---------------------------------------------------------- grid operators
int w1mg_divergence(w1mg_ctx* c, int n, const double* mx, const double* my, double* out) {
    return guard([&] {
        check_n(n);
        const size_t E = (size_t)n * (n + 1), V = (size_t)(n + 1) * (n + 1);
        double* dx = c->get<double>("op.a", E);
        double* dy = c->get<double>("op.b", E);
        double* dv = c->get<double>("op.c", V);
        CK(cudaMemcpyAsync(dx, mx, E * 8, cudaMemcpyDefault, c->stream));
        CK(cudaMemcpyAsync(dy, my, E * 8, cudaMemcpyDefault, c->stream));
        dim3 blk(32, 8);
        divergence_ref_kernel<<<node_grid(n, 1, blk), blk, 0, c->stream>>>(n, dx, dy, dv);
        ++c->launches;
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(out, dv, V * 8, cudaMemcpyDefault, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int w1mg_adjoint(w1mg_ctx* c, int n, const double* phi, double* gx, double* gy) {
    return guard([&] {
        check_n(n);
        const size_t E = (size_t)n * (n + 1), V = (size_t)(n + 1) * (n + 1);
        double* dp = c->get<double>("op.c", V);
        double* dx = c->get<double>("op.a", E);
        double* dy = c->get<double>("op.b", E);
        CK(cudaMemcpyAsync(dp, phi, V * 8, cudaMemcpyDefault, c->stream));
        dim3 blk(32, 8);
        adjoint_ref_kernel<<<node_grid(n, 1, blk), blk, 0, c->stream>>>(n, dp, dx, dy);
        ++c->launches;
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(gx, dx, E * 8, cudaMemcpyDefault, c->stream));
        CK(cudaMemcpyAsync(gy, dy, E * 8, cudaMemcpyDefault, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int w1mg_primal_value(w1mg_ctx* c, int n, const double* mx, const double* my, int pnorm,
                      double* out) {
    return guard([&] {
        check_n(n);
        check_pnorm(pnorm);
        const size_t E = (size_t)n * (n + 1);
        double* dx = c->get<double>("op.a", E);
        double* dy = c->get<double>("op.b", E);
        double* r = c->get<double>("op.r", 1);
        CK(cudaMemcpyAsync(dx, mx, E * 8, cudaMemcpyDefault, c->stream));
        CK(cudaMemcpyAsync(dy, my, E * 8, cudaMemcpyDefault, c->stream));
        const double h = 1.0 / n;
        if (pnorm == 0) reduce_pairs(c, FRefPrimal<0>{dx, dy, n}, n + 1, n + 1, 1, h, h, r);
        else if (pnorm == 1) reduce_pairs(c, FRefPrimal<1>{dx, dy, n}, n + 1, n + 1, 1, h, h, r);
        else reduce_pairs(c, FRefPrimal<2>{dx, dy, n}, n + 1, n + 1, 1, h, h, r);
        CK(cudaMemcpyAsync(out, r, 8, cudaMemcpyDefault, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int w1mg_inner_h_nodes(w1mg_ctx* c, int n, const double* a, const double* b, double* out) {
    return guard([&] {
        check_n(n);
        const size_t V = (size_t)(n + 1) * (n + 1);
        double* da = c->get<double>("op.c", V);
        double* db = c->get<double>("op.d", V);
        double* r = c->get<double>("op.r", 1);
        CK(cudaMemcpyAsync(da, a, V * 8, cudaMemcpyDefault, c->stream));
        CK(cudaMemcpyAsync(db, b, V * 8, cudaMemcpyDefault, c->stream));
        const double h = 1.0 / n;
        reduce_pairs(c, FRefDot{da, db, n + 1}, n + 1, n + 1, 1, h, h, r);
        CK(cudaMemcpyAsync(out, r, 8, cudaMemcpyDefault, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int w1mg_inner_h_edges(w1mg_ctx* c, int n, const double* ax, const double* ay, const double* bx,
                       const double* by, double* out) {
    return guard([&] {
        check_n(n);
        const size_t E = (size_t)n * (n + 1);
        double* d0 = c->get<double>("op.a", E);
        double* d1 = c->get<double>("op.b", E);
        double* d2 = c->get<double>("op.e", E);
        double* d3 = c->get<double>("op.f", E);
        double* r = c->get<double>("op.r2", 2);
        CK(cudaMemcpyAsync(d0, ax, E * 8, cudaMemcpyDefault, c->stream));
        CK(cudaMemcpyAsync(d1, ay, E * 8, cudaMemcpyDefault, c->stream));
        CK(cudaMemcpyAsync(d2, bx, E * 8, cudaMemcpyDefault, c->stream));
        CK(cudaMemcpyAsync(d3, by, E * 8, cudaMemcpyDefault, c->stream));
        // x-edges are n wide, n+1 rows; y-edges n+1 wide, n rows
        reduce_pairs(c, FRefDot{d0, d2, n}, n, n + 1, 1, 1.0, 1.0, r);
        reduce_pairs(c, FRefDot{d1, d3, n + 1}, n + 1, n, 1, 1.0, 1.0, r + 1);
        double hr[2];
        CK(cudaMemcpyAsync(hr, r, 16, cudaMemcpyDefault, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        const double h = 1.0 / n;
        *out = ((hr[0] + hr[1]) * h) * h;
    });
}

// -------------------------------------------------------------- Algorithm 1
int w1mg_cp_run(w1mg_ctx* c, int n, const double* rho, const double* m0x, const double* m0y,
                const double* phi0, int pnorm, double mu, double tau, double tol, long max_iters,
                double* mx, double* my, double* phi, double* fpr_hist, long hist_cap,
                w1mg_cp_report* rep) {
    return guard([&] {
        check_n(n);
        check_pnorm(pnorm);
        if (!rho) fail(W1MG_EINVAL, "null rho");
        if (!(mu > 0.0)) fail(W1MG_EINVAL, "shrink: mu must be positive");
        CK(cudaSetDevice(c->device));
        long cap = (fpr_hist && hist_cap > 0) ? hist_cap : 0;
        double* dh = cap ? c->get<double>("cp.hist", cap) : nullptr;
        Level lv = make_level(c, "cp", n, 1, mu, tau, dh, cap);
        zero_level(c, lv);
        put_nodes(c, lv, 0, RHO, rho, cudaMemcpyDefault);
        if (m0x) put_xedges(c, lv, 0, MX0, m0x, cudaMemcpyDefault);
        if (m0y) put_yedges(c, lv, 0, MY0, m0y, cudaMemcpyDefault);
        if (phi0) put_nodes(c, lv, 0, PHI0, phi0, cudaMemcpyDefault);
        CK(cudaEventRecord(c->t0, c->stream));
        init_level_ctl(c, lv, 0.0, tol, max_iters);
        run_sweeps(c, lv, pnorm, max_iters);
        CK(cudaEventRecord(c->t1, c->stream));
        double* vals = c->get<double>("cp.vals", 2);
        level_values(c, lv, pnorm, vals, vals + 1);
        PairCtl hc;
        double hv[2];
        CK(cudaMemcpyAsync(&hc, lv.ctl, sizeof(PairCtl), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(hv, vals, 16, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (mx) get_xedges(c, lv, 0, MX0 + hc.cur, mx);
        if (my) get_yedges(c, lv, 0, MY0 + hc.cur, my);
        if (phi) get_nodes(c, lv, 0, PHI0 + hc.cur, phi);
        long nh = std::min(hc.it, cap);
        if (nh > 0) CK(cudaMemcpyAsync(fpr_hist, dh, nh * 8, cudaMemcpyDefault, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->t0, c->t1));
        if (rep) {
            rep->distance = hv[0];
            rep->dual_value = hv[1];
            rep->iterations = hc.it;
            rep->fpr_final = hc.fpr;
            rep->converged = (hc.it > 0 && hc.fpr < tol) ? 1 : 0;
            rep->seconds = ms * 1e-3;
        }
    });
}

int w1mg_cp_residual(w1mg_ctx* c, int n, const double* cmx, const double* cmy,
                     const double* cphi, const double* pmx, const double* pmy,
                     const double* pphi, double mu, double tau, double* out) {
    return guard([&] {
        check_n(n);
        const size_t E = (size_t)n * (n + 1), V = (size_t)(n + 1) * (n + 1);
        // dm and dphi on the host would be a CPU path: do the differences on
        // the device (reference: solver_cp.cpp:103-108).
        double* a0 = c->get<double>("res.a0", E);
        double* a1 = c->get<double>("res.a1", E);
        double* b0 = c->get<double>("res.b0", E);
        double* b1 = c->get<double>("res.b1", E);
        double* p0 = c->get<double>("res.p0", V);
        double* p1 = c->get<double>("res.p1", V);
        double* adm = c->get<double>("res.adm", V);
        double* r = c->get<double>("res.r", 4);
        CK(cudaMemcpyAsync(a0, cmx, E * 8, cudaMemcpyDefault, c->stream));
        CK(cudaMemcpyAsync(a1, cmy, E * 8, cudaMemcpyDefault, c->stream));
        CK(cudaMemcpyAsync(b0, pmx, E * 8, cudaMemcpyDefault, c->stream));
        CK(cudaMemcpyAsync(b1, pmy, E * 8, cudaMemcpyDefault, c->stream));
        CK(cudaMemcpyAsync(p0, cphi, V * 8, cudaMemcpyDefault, c->stream));
        CK(cudaMemcpyAsync(p1, pphi, V * 8, cudaMemcpyDefault, c->stream));
        sub_inplace_kernel<<<(int)((E + 255) / 256), 256, 0, c->stream>>>(a0, b0, (long)E);
        ++c->launches;
        sub_inplace_kernel<<<(int)((E + 255) / 256), 256, 0, c->stream>>>(a1, b1, (long)E);
        ++c->launches;
        sub_inplace_kernel<<<(int)((V + 255) / 256), 256, 0, c->stream>>>(p0, p1, (long)V);
        ++c->launches;
        CK(cudaGetLastError());
        dim3 blk(32, 8);
        divergence_ref_kernel<<<node_grid(n, 1, blk), blk, 0, c->stream>>>(n, a0, a1, adm);
        ++c->launches;
        CK(cudaGetLastError());
        const double h = 1.0 / n;
        reduce_pairs(c, FRefDot{a0, a0, n}, n, n + 1, 1, 1.0, 1.0, r);
        reduce_pairs(c, FRefDot{a1, a1, n + 1}, n + 1, n, 1, 1.0, 1.0, r + 1);
        reduce_pairs(c, FRefDot{p0, p0, n + 1}, n + 1, n + 1, 1, h, h, r + 2);
        reduce_pairs(c, FRefDot{p0, adm, n + 1}, n + 1, n + 1, 1, h, h, r + 3);
        double hr[4];
        CK(cudaMemcpyAsync(hr, r, 32, cudaMemcpyDefault, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        // norm_L2 = sqrt(inner_h), then squared (solver_cp.cpp:109-110)
        double nm = std::sqrt(((hr[0] + hr[1]) * h) * h);
        double np = std::sqrt(hr[2]);
        *out = nm * nm / mu + np * np / tau - 2.0 * hr[3];
    });
}

// ---------------------------------------------------------------- cascade
int w1mg_ml_sources(w1mg_ctx* c, int m, const double* img0, const double* img1, int levels,
                    double* rho_levels) {
    return guard([&] {
        check_n(m);
        const size_t MM = (size_t)m * m;
        double* d0 = c->get<double>("in.img0", MM);
        double* d1 = c->get<double>("in.img1", MM);
        CK(cudaMemcpyAsync(d0, img0, MM * 8, cudaMemcpyDefault, c->stream));
        CK(cudaMemcpyAsync(d1, img1, MM * 8, cudaMemcpyDefault, c->stream));
        std::vector<Level> lv = make_levels(c, "src", m, levels, 1, W1MG_STEP_PRACTICAL, nullptr, 0);
        for (auto& L : lv) zero_level(c, L);
        build_sources(c, lv, d0, d1, m);
        size_t off = 0;
        for (int l = 0; l < levels; ++l) {
            get_nodes(c, lv[l], 0, RHO, rho_levels + off);
            off += (size_t)(lv[l].n + 1) * (lv[l].n + 1);
        }
        CK(cudaStreamSynchronize(c->stream));
    });
}

int w1mg_ml_cp_run(w1mg_ctx* c, int n_finest, const double* rho_levels,
                   const w1mg_ml_params* prm, double* mx, double* my, double* phi,
                   w1mg_level_stats* stats, double* fpr_hist, long hist_cap,
                   w1mg_cp_report* rep) {
    return guard([&] {
        check_n(n_finest);
        check_ml(prm);
        const int levels = prm->levels;
        long cap = (fpr_hist && hist_cap > 0) ? hist_cap : 0;
        double* dh = cap ? c->get<double>("ml.hist", cap) : nullptr;
        std::vector<Level> lv =
            make_levels(c, "ml", n_finest, levels, 1, prm->step_mode, dh, cap);
        size_t off = 0;
        for (auto& L : lv) {
            zero_level(c, L);
            put_nodes(c, L, 0, RHO, rho_levels + off, cudaMemcpyDefault);
            off += (size_t)(L.n + 1) * (L.n + 1);
        }
        long* it = c->get<long>("ml.iters", levels);
        double* ff = c->get<double>("ml.fpr", levels);
        double* tl = c->get<double>("ml.tol", levels);
        std::vector<double> secs;
        run_cascade(c, lv, *prm, it, ff, tl, &secs);
        const Level& F = lv.back();
        double* vals = c->get<double>("ml.vals", 2);
        level_values(c, F, prm->pnorm, vals, vals + 1);
        std::vector<long> hit(levels);
        std::vector<double> hff(levels), htl(levels);
        PairCtl hc;
        double hv[2];
        CK(cudaMemcpyAsync(hit.data(), it, levels * sizeof(long), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(hff.data(), ff, levels * 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(htl.data(), tl, levels * 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(&hc, F.ctl, sizeof(PairCtl), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(hv, vals, 16, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        if (mx) get_xedges(c, F, 0, MX0 + hc.cur, mx);
        if (my) get_yedges(c, F, 0, MY0 + hc.cur, my);
        if (phi) get_nodes(c, F, 0, PHI0 + hc.cur, phi);
        long nh = std::min(hc.it, cap);
        if (nh > 0) CK(cudaMemcpyAsync(fpr_hist, dh, nh * 8, cudaMemcpyDefault, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        long total = 0;
        double tsec = 0;
        for (int l = 0; l < levels; ++l) {
            total += hit[l];
            tsec += secs[l];
            if (stats) {
                stats[l].h = 1.0 / lv[l].n;
                stats[l].eps = htl[l];
                stats[l].iters = hit[l];
                stats[l].fpr_final = hff[l];
                stats[l].seconds = secs[l];
            }
        }
        if (rep) {
            rep->distance = hv[0];
            rep->dual_value = hv[1];
            rep->iterations = total;
            rep->fpr_final = hc.fpr;
            rep->converged = (hc.fpr < hc.tol) ? 1 : 0;
            rep->seconds = tsec;
        }
    });
}

int w1mg_ml_cp_batch_dev(w1mg_ctx* c, int npairs, int m, const double* img0s,
                         const double* img1s, const w1mg_ml_params* prm, double* distance,
                         double* dual, long* iters, int* converged) {
    return guard([&] {
        check_n(m);
        check_ml(prm);
        if (npairs < 1 || npairs > 65535) fail(W1MG_EINVAL, "npairs must be in [1, 65535]");
        std::vector<Level> lv =
            make_levels(c, "mlb", m, prm->levels, npairs, prm->step_mode, nullptr, 0);
        for (auto& L : lv) zero_level(c, L);
        build_sources(c, lv, img0s, img1s, m);
        run_cascade(c, lv, *prm, iters, nullptr, nullptr, nullptr);
        level_values(c, lv.back(), prm->pnorm, distance, dual);
        if (converged) {
            converged_kernel<<<(npairs + 127) / 128, 128, 0, c->stream>>>(lv.back().ctl, npairs, converged);
            ++c->launches;
            CK(cudaGetLastError());
        }
    });
}

int w1mg_ml_cp_batch(w1mg_ctx* c, int npairs, int m, const double* img0s, const double* img1s,
                     const w1mg_ml_params* prm, double* distance, double* dual, long* iters,
                     int* converged) {
    return guard([&] {
        check_n(m);
        check_ml(prm);
        const size_t MM = (size_t)npairs * m * m;
        double* d0 = c->get<double>("in.img0s", MM);
        double* d1 = c->get<double>("in.img1s", MM);
        CK(cudaMemcpyAsync(d0, img0s, MM * 8, cudaMemcpyDefault, c->stream));
        CK(cudaMemcpyAsync(d1, img1s, MM * 8, cudaMemcpyDefault, c->stream));
        double* od = c->get<double>("out.dist", npairs);
        double* ou = c->get<double>("out.dual", npairs);
        long* oi = c->get<long>("out.iters", (size_t)npairs * prm->levels);
        int* oc = c->get<int>("out.conv", npairs);
        int rc = w1mg_ml_cp_batch_dev(c, npairs, m, d0, d1, prm, od, ou, oi, oc);
        if (rc) throw Fail{rc, g_err};
        if (distance) CK(cudaMemcpyAsync(distance, od, npairs * 8, cudaMemcpyDefault, c->stream));
        if (dual) CK(cudaMemcpyAsync(dual, ou, npairs * 8, cudaMemcpyDefault, c->stream));
        if (iters)
            CK(cudaMemcpyAsync(iters, oi, (size_t)npairs * prm->levels * sizeof(long),
                               cudaMemcpyDefault, c->stream));
        if (converged) CK(cudaMemcpyAsync(converged, oc, npairs * 4, cudaMemcpyDefault, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

// Batched cascades with every pair's finest-level fields and residual copied
// back (parity checks of the batched engines against per-pair oracle runs).
int w1mg_ml_cp_batch_fields(w1mg_ctx* c, int npairs, int m, const double* img0s,
                            const double* img1s, const w1mg_ml_params* prm, double* distance,
                            double* dual, long* iters, int* converged, double* mx, double* my,
                            double* phi, double* fpr_final) {
    return guard([&] {
        check_n(m);
        check_ml(prm);
        if (npairs < 1 || npairs > 65535) fail(W1MG_EINVAL, "npairs must be in [1, 65535]");
        const size_t MM = (size_t)npairs * m * m;
        double* d0 = c->get<double>("in.img0s", MM);
        double* d1 = c->get<double>("in.img1s", MM);
        CK(cudaMemcpyAsync(d0, img0s, MM * 8, cudaMemcpyDefault, c->stream));
        CK(cudaMemcpyAsync(d1, img1s, MM * 8, cudaMemcpyDefault, c->stream));
        std::vector<Level> lv =
            make_levels(c, "mlb", m, prm->levels, npairs, prm->step_mode, nullptr, 0);
        for (auto& L : lv) zero_level(c, L);
        build_sources(c, lv, d0, d1, m);
        long* oi = c->get<long>("out.iters", (size_t)npairs * prm->levels);
        run_cascade(c, lv, *prm, oi, nullptr, nullptr, nullptr);
        double* od = c->get<double>("out.dist", npairs);
        double* ou = c->get<double>("out.dual", npairs);
        level_values(c, lv.back(), prm->pnorm, od, ou);
        const Level& F = lv.back();
        std::vector<PairCtl> hc(npairs);
        CK(cudaMemcpyAsync(hc.data(), F.ctl, npairs * sizeof(PairCtl), cudaMemcpyDeviceToHost,
                           c->stream));
        if (distance) CK(cudaMemcpyAsync(distance, od, npairs * 8, cudaMemcpyDefault, c->stream));
        if (dual) CK(cudaMemcpyAsync(dual, ou, npairs * 8, cudaMemcpyDefault, c->stream));
        if (iters)
            CK(cudaMemcpyAsync(iters, oi, (size_t)npairs * prm->levels * sizeof(long),
                               cudaMemcpyDefault, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        const size_t E = (size_t)m * (m + 1), V = (size_t)(m + 1) * (m + 1);
        for (int b = 0; b < npairs; ++b) {
            if (converged) converged[b] = (hc[b].fpr < hc[b].tol) ? 1 : 0;
            if (fpr_final) fpr_final[b] = hc[b].fpr;
            if (mx) get_xedges(c, F, b, MX0 + hc[b].cur, mx + b * E);
            if (my) get_yedges(c, F, b, MY0 + hc[b].cur, my + b * E);
            if (phi) get_nodes(c, F, b, PHI0 + hc[b].cur, phi + b * V);
        }
        CK(cudaStreamSynchronize(c->stream));
    });
}

// Eq. 14 / Eq. 15 on single reference-layout fields (value API).
int w1mg_interpolate_scalar(w1mg_ctx* c, int nc, const double* coarse, double* fine) {
    return guard([&] {
        check_n(nc);
        const size_t Vc = (size_t)(nc + 1) * (nc + 1), Vf = (size_t)(2 * nc + 1) * (2 * nc + 1);
        double* dc = c->get<double>("ip.c", Vc);
        double* df = c->get<double>("ip.f", Vf);
        CK(cudaMemcpyAsync(dc, coarse, Vc * 8, cudaMemcpyDefault, c->stream));
        dim3 blk(32, 8);
        interp_scalar_ref_kernel<<<node_grid(2 * nc, 1, blk), blk, 0, c->stream>>>(nc, dc, df);
        ++c->launches;
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(fine, df, Vf * 8, cudaMemcpyDefault, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int w1mg_interpolate_flux(w1mg_ctx* c, int nc, const double* cx, const double* cy, double* fx,
                          double* fy) {
    return guard([&] {
        check_n(nc);
        const int nf = 2 * nc;
        const size_t Ec = (size_t)nc * (nc + 1), Ef = (size_t)nf * (nf + 1);
        double* dcx = c->get<double>("ip.cx", Ec);
        double* dcy = c->get<double>("ip.cy", Ec);
        double* dfx = c->get<double>("ip.fx", Ef);
        double* dfy = c->get<double>("ip.fy", Ef);
        CK(cudaMemcpyAsync(dcx, cx, Ec * 8, cudaMemcpyDefault, c->stream));
        CK(cudaMemcpyAsync(dcy, cy, Ec * 8, cudaMemcpyDefault, c->stream));
        dim3 blk(32, 8);
        interp_flux_ref_kernel<<<node_grid(nf, 1, blk), blk, 0, c->stream>>>(nc, dcx, dcy, dfx, dfy);
        ++c->launches;
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(fx, dfx, Ef * 8, cudaMemcpyDefault, c->stream));
        CK(cudaMemcpyAsync(fy, dfy, Ef * 8, cudaMemcpyDefault, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

// Kernel probe: `iters` fused sweeps on B pairs of an n-cell level with the
// stop rule disabled, after `warm` untimed sweeps; returns ms per sweep.
int w1mg_set_sweep_engine(int engine) {
    if (engine < kTma || engine > kTma3 || engine == 4) return W1MG_EINVAL;
    g_sweep_variant = engine;
    return W1MG_OK;
}

int w1mg_set_resident_engine(int on) {
    if (on < 0 || on > 3) return W1MG_EINVAL;
    g_resident = on;
    return W1MG_OK;
}

int w1mg_set_option(const char* name, long value) {
    if (!name) return W1MG_EINVAL;
    const std::string k(name);
    const int v = (int)value;
    if (k == "pdhg_persist" && (v == 0 || v == 1)) g_pdhg_persist = v;
    else if (k == "pdhg_rs" && v >= 0 && v <= 4) g_pdhg_rs = v;
    else if (k == "slab_min_n" && v >= 1) g_slab_min_n = v;
    else if (k == "pdhg_small" && v >= 0 && v <= 2) g_pdhg_small = v;
    else if (k == "cluster_pick" && (v == 0 || v == 1)) g_cluster_pick = v;
    else if (k == "compact") g_compact = v != 0;
    else if (k == "compact_step" && v >= 1) g_compact_step = v;
    else if (k == "warps_per_sm" && v >= 1) g_warps_per_sm = v;
    else if (k == "pdl" && (v == 0 || v == 1)) g_pdl = v;
    else if (k == "fast" && (v == 0 || v == 1)) g_fast = v;
    else if (k == "occ3" && (v == 4 || v == 5)) g_occ3 = v;
    else if (k == "tmap_nw" && (v == 0 || v == 2 || v == 4 || v == 8)) g_tmap_nw = v;
    else return W1MG_EINVAL;
    return W1MG_OK;
}

int w1mg_set_pdhg_small(int mode) {
    if (mode < 0 || mode > 2) return W1MG_EINVAL;
    g_pdhg_small = mode;
    return W1MG_OK;
}

int w1mg_set_tail_compaction(int on) {
    g_compact = on != 0;
    return W1MG_OK;
}

int w1mg_rn_selftest(w1mg_ctx* c, long count, unsigned long long seed, double mu,
                     unsigned long long* bad) {
    return guard([&] {
        if (count < 0 || !(mu > 0.0)) fail(W1MG_EINVAL, "rn_selftest: bad arguments");
        auto* d = c->get<unsigned long long>("selftest.bad", 3);
        CK(cudaMemsetAsync(d, 0, 3 * sizeof(unsigned long long), c->stream));
        rn_selftest_kernel<<<c->num_sms * 8, 256, 0, c->stream>>>(count, seed, mu,
                                                                  shrink_zero_threshold(mu), d);
        ++c->launches;
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(bad, d, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    });
}

int w1mg_sweep_probe(w1mg_ctx* c, int n, int B, int pnorm, long warm, long iters,
                     double* ms_per_sweep) {
    return guard([&] {
        check_n(n);
        check_pnorm(pnorm);
        const double step = w1mg_cp_step_size(n, W1MG_STEP_PRACTICAL);
        Level lv = make_level(c, "probe", n, B, step, step, nullptr, 0);
        zero_level(c, lv);
        dim3 blk(32, 8);
        probe_fill_kernel<<<node_grid(n, B, blk), blk, 0, c->stream>>>(lv.base, lv.L);
        ++c->launches;
        CK(cudaGetLastError());
        mirror_rho(c, lv);
        init_level_ctl(c, lv, 0.0, -1.0, 2 * (warm + iters) + 64);
        // kTma2: each launch is two sweeps; iters counts sweeps
        const int per = sweeps_per_launch(lv);
        auto one = [&](long k) {
            if (per == 3) launch_sweep3(lv, pnorm, (int)(k & 1), c->stream);
            else if (per == 2) launch_sweep2(lv, pnorm, (int)(k & 1), c->stream);
            else launch_sweep(lv, pnorm, (int)(k & 1), c->stream);
        };
        long k = 0;
        for (; k < warm / per; ++k) one(k);
        CK(cudaEventRecord(c->t0, c->stream));
        const long nl = iters / per;
        for (long t = 0; t < nl; ++t, ++k) one(k);
        CK(cudaEventRecord(c->t1, c->stream));
        CK(cudaGetLastError());
        c->launches += k;
        iters = nl * per;
        CK(cudaEventSynchronize(c->t1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->t0, c->t1));
        *ms_per_sweep = ms / (double)iters;
    });
}

// Measured FP64 pipe peak (the denominator of the sweep kernels' FP64
// roofline): every thread of SMs x 4 blocks x 256 threads runs 8 independent
// DFMA chains of `iters` steps; flops = 2 per DFMA.  Timed with CUDA events.
int w1mg_fp64_peak_probe(w1mg_ctx* c, long iters, double* tflops) {
    return guard([&] {
        if (iters < 1 || !tflops) fail(W1MG_EINVAL, "fp64 probe: bad arguments");
        double* sink = c->get<double>("probe.fp64", 1);
        const int blocks = c->num_sms * 4;
        fp64_peak_kernel<<<blocks, 256, 0, c->stream>>>(iters / 4, sink);  // warm-up
        CK(cudaEventRecord(c->t0, c->stream));
        fp64_peak_kernel<<<blocks, 256, 0, c->stream>>>(iters, sink);
        CK(cudaEventRecord(c->t1, c->stream));
        CK(cudaGetLastError());
        c->launches += 2;
        CK(cudaEventSynchronize(c->t1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->t0, c->t1));
        *tflops = 2.0 * 8.0 * (double)iters * blocks * 256 / (ms * 1e-3) / 1e12;
    });
}

}  // extern "C"

#include "pdhg_engine.cuh"
#include "slab_engine.cuh"
