// pdhg_engine.cuh -- host engine + C-ABI of the G-prox PDHG path (Algorithm 2
// and 4), the Neumann Poisson solve and the affine projection.  Included at
// the end of capi.cu (same translation unit: reuses w1mg_ctx, CK, guard,
// reduce_pairs, node_grid).
//
// Reference entry points replaced (paths relative to /root/reference):
//   NeumannPoissonSolver::solve_into / solve_projected_into  proj/src/poisson.cpp:61-99
//   project_affine / project_affine_inplace                  proj/src/poisson.cpp:101-132
//   pdhg_step / pdhg_residual / pdhg_run / recover_potential proj/include/w1mg/solver_pdhg.hpp:20-46
#pragma once

#include "pdhg_kernels.cuh"
#include "pdhg_small.cuh"
#include "pdhg_fold.cuh"

namespace {

void blas_check(cublasStatus_t s, const char* what) {
    if (s != CUBLAS_STATUS_SUCCESS) fail(W1MG_ECUDA, std::string("cuBLAS ") + what + " failed");
}

cublasHandle_t blas(w1mg_ctx* c) {
    if (!c->blas) {
        cublasHandle_t h;
        blas_check(cublasCreate(&h), "create");
        // a fixed workspace keeps DGEMM capturable in CUDA graphs
        void* ws = c->buf("blas.workspace", 8u << 20);
        blas_check(cublasSetWorkspace(h, ws, 8u << 20), "workspace");
        blas_check(cublasSetMathMode(h, CUBLAS_DEFAULT_MATH), "math mode");
        c->blas = h;
    }
    cublasHandle_t h = static_cast<cublasHandle_t>(c->blas);
    blas_check(cublasSetStream(h, c->stream), "stream");
    return h;
}

// One PDHG level batch (B pairs, P_NSLOT planes each) + DCT operators.
struct PLevel {
    int n = 0, B = 0;
    Layout L{};
    double* base = nullptr;
    PairCtl* ctl = nullptr;
    unsigned* ticket = nullptr;
    int* ndone = nullptr;
    SweepArgs args{};
    dim3 grid, blk;
    const double* C = nullptr;    // DCT-II matrix, m x m column-major: C(k, j) = 2 cos(pi (2j+1) k / 2m)
    const double* S = nullptr;    // DCT-III matrix: S(k, j) = j ? 2 cos(pi j (2k+1) / 2m) : 1
    const double* lam = nullptr;  // lambda_k, poisson.cpp:28-30
    // symmetry-folded DCTs for the PDHG iteration (pdhg_fold.cuh), odd m >= kFoldMinM
    bool fold = false;
    FoldGeom fg{};
    const double* const* gp = nullptr;  // device pointer arrays [4 stages][A,B,C][4B]
};

// folded DCT in the PDHG iteration from this m on (W1MG_PDHG_FOLD=0 disables).
// Measured per level of config 3 (one pair): 513^2 176 vs 202 ms (folded vs
// dense), 257^2 143 vs 128 ms, 129^2 157 vs 130 ms -- the batched half-size
// GEMMs only win once the dense ones are large.
constexpr int kFoldMinM = 400;

// Folded DCT operators (h x h, ld h, zero padded): C_e, C_o, S_e, S_o.
const double* fold_operators(w1mg_ctx* c, int n) {
    const int m = n + 1, h = (m + 1) / 2, ho = h - 1;
    const std::string key = "dctf." + std::to_string(m);
    const bool fresh = c->bufs.find(key) == c->bufs.end();
    double* d = c->get<double>(key, (size_t)4 * h * h);
    if (fresh) {
        std::vector<double> M((size_t)4 * h * h, 0.0);
        const long double pi = 3.141592653589793238462643383279502884L;
        auto Cf = [&](long k, long l) {  // C(k, l) = 2 cos(pi (2l+1) k / 2m)
            return (double)(2.0L * cosl(pi * (((2 * l + 1) * k) % (4L * m)) / (2.0L * m)));
        };
        auto Sf = [&](long k, long j) {  // S(k, j) = j ? 2 cos(pi j (2k+1) / 2m) : 1
            return j == 0 ? 1.0 : (double)(2.0L * cosl(pi * ((j * (2 * k + 1)) % (4L * m)) / (2.0L * m)));
        };
        double* Ce = M.data();
        double* Co = Ce + (size_t)h * h;
        double* Se = Co + (size_t)h * h;
        double* So = Se + (size_t)h * h;
        for (int col = 0; col < h; ++col)
            for (int row = 0; row < h; ++row) {
                const size_t e = (size_t)col * h + row;
                Ce[e] = Cf(2L * row, col);
                if (row < ho && col < ho) Co[e] = Cf(2L * row + 1, col);
                Se[e] = Sf(row, 2L * col);
                if (row < ho && col < ho) So[e] = Sf(row, 2L * col + 1);
            }
        CK(cudaMemcpy(d, M.data(), M.size() * 8, cudaMemcpyHostToDevice));
    }
    return d;
}

// DCT operators for m = n+1, built once per size on the host in long double
// and cached on the device.
void dct_operators(w1mg_ctx* c, int n, const double** C, const double** S, const double** lam) {
    const int m = n + 1;
    const std::string key = std::to_string(m);
    const bool fresh = c->bufs.find("dct.C." + key) == c->bufs.end();
    double* dC = c->get<double>("dct.C." + key, (size_t)m * m);
    double* dS = c->get<double>("dct.S." + key, (size_t)m * m);
    double* dl = c->get<double>("dct.lam." + key, m);
    if (fresh) {
        std::vector<double> hC((size_t)m * m), hS((size_t)m * m), hl(m);
        const long double pi = 3.141592653589793238462643383279502884L;
        for (int j = 0; j < m; ++j)
            for (int k = 0; k < m; ++k) {
                long a = ((long)(2 * j + 1) * k) % (4L * m);  // exact angle reduction
                long b = ((long)j * (2 * k + 1)) % (4L * m);
                hC[(size_t)j * m + k] = (double)(2.0L * cosl(pi * a / (2.0L * m)));
                hS[(size_t)j * m + k] = j == 0 ? 1.0 : (double)(2.0L * cosl(pi * b / (2.0L * m)));
            }
        const double h = 1.0 / n;
        const double inv_h2 = 1.0 / (h * h);
        for (int k = 0; k < m; ++k) hl[k] = (2.0 - 2.0 * std::cos(M_PI * k / m)) * inv_h2;
        CK(cudaMemcpy(dC, hC.data(), hC.size() * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dS, hS.data(), hS.size() * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dl, hl.data(), hl.size() * 8, cudaMemcpyHostToDevice));
    }
    *C = dC;
    *S = dS;
    *lam = dl;
}

PLevel make_plevel(w1mg_ctx* c, const std::string& tag, int n, int B, double mu, double tau,
                   double* hist, long hist_cap) {
    PLevel lv;
    lv.n = n;
    lv.B = B;
    lv.L = Layout::make(n);
    lv.base = c->get<double>(tag + ".base", (size_t)B * P_NSLOT * lv.L.plane);
    lv.ctl = c->get<PairCtl>(tag + ".ctl", B);
    lv.ticket = c->get<unsigned>(tag + ".ticket", B);
    lv.ndone = c->get<int>(tag + ".ndone", 1);
    lv.blk = dim3(32, 8);
    lv.grid = node_grid(n, B, lv.blk);
    SweepArgs& a = lv.args;
    a.base = lv.base;
    a.L = lv.L;
    a.mu = mu;
    a.tau = tau;
    const double h = 1.0 / n;
    a.ih = 1.0 / h;
    a.h2 = h * h;
    a.ctl = lv.ctl;
    a.ticket = lv.ticket;
    a.hist = hist;
    a.hist_cap = hist_cap;
    a.ndone = lv.ndone;
    a.partial = c->get<double>(tag + ".partial", (size_t)B * lv.grid.x * lv.grid.y * 3);
    dct_operators(c, n, &lv.C, &lv.S, &lv.lam);
    const int m = n + 1;
    if ((m & 1) && m >= 3 && (g_pdhg_fold == 2 || (g_pdhg_fold == 1 && m >= kFoldMinM))) {
        lv.fold = true;
        lv.fg.h = (m + 1) / 2;
        lv.fg.lq = lv.L.pitch / 2;
        const int h = lv.fg.h;
        const double* ops = fold_operators(c, n);
        const double* Cm[2] = {ops, ops + (size_t)h * h};
        const double* Sm[2] = {ops + 2 * (size_t)h * h, ops + 3 * (size_t)h * h};
        // stage s, array t (A, B, C), entry e = 4 b + q
        std::vector<const double*> P((size_t)12 * 4 * B);
        auto at = [&](int st, int t, int e) -> const double*& { return P[((size_t)st * 3 + t) * 4 * B + e]; };
        for (int b = 0; b < B; ++b)
            for (int q = 0; q < 4; ++q) {
                const int e = 4 * b + q, qa = q >> 1, qb = q & 1;
                auto quad = [&](int slot) {
                    return lv.base + ((long)b * P_NSLOT + slot) * lv.L.plane + lv.L.at(0, 0) +
                           (long)q * h * lv.fg.lq;
                };
                at(0, 0, e) = Cm[qa]; at(0, 1, e) = quad(P_RES); at(0, 2, e) = quad(P_T);
                at(1, 0, e) = quad(P_T); at(1, 1, e) = Cm[qb]; at(1, 2, e) = quad(P_RES);
                at(2, 0, e) = Sm[qa]; at(2, 1, e) = quad(P_RES); at(2, 2, e) = quad(P_T);
                at(3, 0, e) = quad(P_T); at(3, 1, e) = Sm[qb]; at(3, 2, e) = quad(P_PSI);
            }
        const double** dp = c->get<const double*>(tag + ".foldptr", P.size());
        CK(cudaMemcpyAsync(dp, P.data(), P.size() * sizeof(void*), cudaMemcpyHostToDevice,
                           c->stream));
        CK(cudaStreamSynchronize(c->stream));  // host vector dies here
        lv.gp = dp;
    }
    CK(cudaMemsetAsync(lv.ticket, 0, sizeof(unsigned) * B, c->stream));
    return lv;
}

double* pslot_ptr(const PLevel& lv, int pair, int slot) {
    return lv.base + ((long)pair * P_NSLOT + slot) * lv.L.plane + lv.L.at(0, 0);
}

// dense reference-layout array (w x rows) <-> slot
void pput(w1mg_ctx* c, const PLevel& lv, int pair, int slot, const double* src, int w, int rows) {
    CK(cudaMemcpy2DAsync(pslot_ptr(lv, pair, slot), lv.L.pitch * 8, src, (size_t)w * 8,
                         (size_t)w * 8, rows, cudaMemcpyDefault, c->stream));
}
void pget(w1mg_ctx* c, const PLevel& lv, int pair, int slot, double* dst, int w, int rows) {
    CK(cudaMemcpy2DAsync(dst, (size_t)w * 8, pslot_ptr(lv, pair, slot), lv.L.pitch * 8,
                         (size_t)w * 8, rows, cudaMemcpyDefault, c->stream));
}

// psi = (A A*)^+ r on every pair: slot `in` -> P_PSI (P_T scratch; `in` is
// overwritten).  Column-major view of a node array: element (i, j) at
// i + j*pitch, so both 1D transforms are the same sandwich Y = C X C^T.
void poisson_apply(w1mg_ctx* c, const PLevel& lv, int in, bool check_done) {
    cublasHandle_t h = blas(c);
    const int m = lv.n + 1;
    const int ld = lv.L.pitch;
    const long long stride = (long long)P_NSLOT * lv.L.plane;
    double* X = pslot_ptr(lv, 0, in);
    double* T = pslot_ptr(lv, 0, P_T);
    double* Psi = pslot_ptr(lv, 0, P_PSI);
    const double one = 1.0, zero = 0.0;
    const double scale = 1.0 / (4.0 * double(m) * double(m));  // poisson.cpp:93
    // DCT-II along both directions: T = C X, X = T C^T
    blas_check(cublasDgemmStridedBatched(h, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &one, lv.C, m, 0, X,
                                         ld, stride, &zero, T, ld, stride, lv.B),
               "dgemm");
    blas_check(cublasDgemmStridedBatched(h, CUBLAS_OP_N, CUBLAS_OP_T, m, m, m, &one, T, ld, stride,
                                         lv.C, m, 0, &zero, X, ld, stride, lv.B),
               "dgemm");
    spectral_divide_kernel<<<dim3((m + 31) / 32, (m + 7) / 8, lv.B), dim3(32, 8), 0, c->stream>>>(
        lv.args, in, lv.lam, check_done ? 1 : 0);
    ++c->launches;
    CK(cudaGetLastError());
    // DCT-III along both directions, scaled by 1/(4 m^2)
    blas_check(cublasDgemmStridedBatched(h, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &one, lv.S, m, 0, X,
                                         ld, stride, &zero, T, ld, stride, lv.B),
               "dgemm");
    blas_check(cublasDgemmStridedBatched(h, CUBLAS_OP_N, CUBLAS_OP_T, m, m, m, &scale, T, ld,
                                         stride, lv.S, m, 0, &zero, Psi, ld, stride, lv.B),
               "dgemm");
    c->launches += 4;
}

// psi -= compensated mean (poisson.cpp:96-98)
void remove_mean(w1mg_ctx* c, const PLevel& lv, int slot) {
    double* sums = c->get<double>("pdhg.mean", lv.B);
    reduce_pairs(c, FPSlot{lv.base, lv.L, slot}, lv.n + 1, lv.n + 1, lv.B, 1.0, 1.0, sums);
    subtract_mean_kernel<<<lv.grid, lv.blk, 0, c->stream>>>(lv.args, slot, sums);
    ++c->launches;
    CK(cudaGetLastError());
}

// The iteration with folded DCTs: pre (folding), 4 batched GEMM stages over
// the (pair, quadrant) products with the divide after stage 2, post.
void pdhg_iteration_fold(w1mg_ctx* c, const PLevel& lv, int q) {
    const FoldGeom g = lv.fg;
    const int h = g.h, nb = 4 * lv.B;
    const dim3 fblk(32, 8);
    pdhg_pre_fold_kernel<<<dim3((h + 31) / 32, (h + 7) / 8, lv.B), fblk, 0, c->stream>>>(lv.args, g);
    CK(cudaGetLastError());
    cublasHandle_t hb = blas(c);
    const double one = 1.0, zero = 0.0;
    const int m = lv.n + 1;
    const double scale = 1.0 / (4.0 * double(m) * double(m));  // poisson.cpp:93
    auto arr = [&](int st, int t) { return lv.gp + ((size_t)st * 3 + t) * nb; };
    auto gemm = [&](int st, cublasOperation_t tb, const double* alpha, int lda, int ldb) {
        blas_check(cublasDgemmBatched(hb, CUBLAS_OP_N, tb, h, h, h, alpha, arr(st, 0), lda,
                                      arr(st, 1), ldb, &zero,
                                      const_cast<double* const*>(arr(st, 2)), g.lq, nb),
                   "dgemm batched");
    };
    gemm(0, CUBLAS_OP_N, &one, h, g.lq);     // T = C_a X
    gemm(1, CUBLAS_OP_T, &one, g.lq, h);     // X = T C_b^T
    spectral_divide_fold_kernel<<<dim3((h + 31) / 32, (h + 7) / 8, nb), fblk, 0, c->stream>>>(
        lv.args, g, lv.lam);
    CK(cudaGetLastError());
    gemm(2, CUBLAS_OP_N, &one, h, g.lq);     // T = S_a Y
    gemm(3, CUBLAS_OP_T, &scale, g.lq, h);   // P = T S_b^T / (4 m^2)
    switch (q) {
        case 0: pdhg_post_fold_kernel<0><<<lv.grid, lv.blk, 0, c->stream>>>(lv.args, g); break;
        case 1: pdhg_post_fold_kernel<1><<<lv.grid, lv.blk, 0, c->stream>>>(lv.args, g); break;
        default: pdhg_post_fold_kernel<2><<<lv.grid, lv.blk, 0, c->stream>>>(lv.args, g); break;
    }
    CK(cudaGetLastError());
    c->launches += 7;
}

void pdhg_iteration(w1mg_ctx* c, const PLevel& lv, int q) {
    if (lv.fold) {
        pdhg_iteration_fold(c, lv, q);
        return;
    }
    pdhg_pre_kernel<<<lv.grid, lv.blk, 0, c->stream>>>(lv.args);
    poisson_apply(c, lv, P_RES, true);
    switch (q) {
        case 0: pdhg_post_kernel<0><<<lv.grid, lv.blk, 0, c->stream>>>(lv.args); break;
        case 1: pdhg_post_kernel<1><<<lv.grid, lv.blk, 0, c->stream>>>(lv.args); break;
        default: pdhg_post_kernel<2><<<lv.grid, lv.blk, 0, c->stream>>>(lv.args); break;
    }
    c->launches += 2;
    CK(cudaGetLastError());
}

// small levels: one launch per level, one CTA per pair (pdhg_small.cuh);
// W1MG_PDHG_SMALL = 1 (default, m <= 33), 2 (m <= 65), 0 (streaming only)
// (g_pdhg_small, level_engine.cuh)

template <int Q>
void launch_pdhg_small(w1mg_ctx* c, const PLevel& lv) {
    static unsigned long long attr = 0;  // per device
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (!(attr >> (dev & 63) & 1ull)) {
        const int mx = (int)std::max(pdhg_small_smem(kPdhgSmallMaxM), pdhg_small_smem(kPdhgStateM));
        CK(cudaFuncSetAttribute(pdhg_small_kernel<Q, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        CK(cudaFuncSetAttribute(pdhg_small_kernel<Q, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        attr |= 1ull << (dev & 63);
    }
    if (lv.n + 1 <= kPdhgStateM)
        pdhg_small_kernel<Q, true><<<lv.B, pdhg_small_threads(lv.n + 1), pdhg_small_smem(lv.n + 1), c->stream>>>(
            lv.args, lv.C, lv.S, lv.lam);
    else
        pdhg_small_kernel<Q, false><<<lv.B, pdhg_small_threads(lv.n + 1), pdhg_small_smem(lv.n + 1), c->stream>>>(
            lv.args, lv.C, lv.S, lv.lam);
    CK(cudaGetLastError());
    ++c->launches;
}

// Iterate until every pair's stop flag is set (graph of K iterations, host
// watches the done counter one graph behind, like run_sweeps).
void run_pdhg_iters(w1mg_ctx* c, const PLevel& lv, int q, long max_iters) {
    if (max_iters <= 0) return;
    if ((g_pdhg_small == 1 && lv.n + 1 <= kPdhgSmallAutoM) ||
        (g_pdhg_small == 2 && lv.n + 1 <= kPdhgSmallMaxM)) {
        if (q == 0) launch_pdhg_small<0>(c, lv);
        else if (q == 1) launch_pdhg_small<1>(c, lv);
        else launch_pdhg_small<2>(c, lv);
        return;
    }
    constexpr int K = 8;
    if (max_iters < K) {
        for (long k = 0; k < max_iters; ++k) pdhg_iteration(c, lv, q);
        return;
    }
    std::string key(reinterpret_cast<const char*>(&lv.args), sizeof(SweepArgs));
    key += "pdhg:" + std::to_string(q) + ":" + std::to_string(lv.B) + (lv.fold ? ":fold" : ":dense");
    cudaGraphExec_t ex;
    auto it = c->graphs.find(key);
    if (it != c->graphs.end()) {
        ex = it->second;
    } else {
        blas(c);  // create the handle outside the capture
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        const long before = c->launches;
        for (int k = 0; k < K; ++k) pdhg_iteration(c, lv, q);
        c->launches = before;
        CK(cudaStreamEndCapture(c->stream, &g));
        CK(cudaGraphInstantiate(&ex, g, 0));
        CK(cudaGraphDestroy(g));
        c->graphs[key] = ex;
    }
    long launched = 0;
    for (long g = 0;; ++g) {
        CK(cudaGraphLaunch(ex, c->stream));
        launched += K;
        c->launches += 7L * K;
        CK(cudaMemcpyAsync(c->pinned + (g & 1), lv.ndone, sizeof(int), cudaMemcpyDeviceToHost,
                           c->stream));
        CK(cudaEventRecord(c->ev[g & 1], c->stream));
        if (g > 0) {
            CK(cudaEventSynchronize(c->ev[(g - 1) & 1]));
            if (c->pinned[(g - 1) & 1] >= lv.B) break;
        }
        if (launched >= max_iters + K) break;
    }
}

void pdhg_init_ctl(w1mg_ctx* c, const PLevel& lv, double tol, long max_it) {
    init_ctl_kernel<<<(lv.B + 127) / 128, 128, 0, c->stream>>>(lv.ctl, lv.B, nullptr, 0.0, tol,
                                                                 max_it, lv.ndone);
    ++c->launches;
    CK(cudaGetLastError());
    CK(cudaMemsetAsync(lv.ticket, 0, sizeof(unsigned) * lv.B, c->stream));
}

// distance (primal value of m) and the recovered-potential dual per pair;
// leaves the recovered potential in P_PSI.
void pdhg_values(w1mg_ctx* c, const PLevel& lv, int pn, double* w1, double* dual) {
    const double h = 1.0 / lv.n;
    if (w1) {
        if (pn == 0) reduce_pairs(c, FPPrimal<0>{lv.base, lv.L}, lv.n + 1, lv.n + 1, lv.B, h, h, w1);
        else if (pn == 1) reduce_pairs(c, FPPrimal<1>{lv.base, lv.L}, lv.n + 1, lv.n + 1, lv.B, h, h, w1);
        else reduce_pairs(c, FPPrimal<2>{lv.base, lv.L}, lv.n + 1, lv.n + 1, lv.B, h, h, w1);
    }
    // recover_potential: phi = (A A*)^+ A varphi, zero mean
    pdhg_div_dual_kernel<<<lv.grid, lv.blk, 0, c->stream>>>(lv.args);
    ++c->launches;
    CK(cudaGetLastError());
    poisson_apply(c, lv, P_RES, false);
    remove_mean(c, lv, P_PSI);
    if (dual) reduce_pairs(c, FPDual{lv.base, lv.L}, lv.n + 1, lv.n + 1, lv.B, h, h, dual);
}

int conj_q(int p) { return p == 0 ? 2 : (p == 1 ? 1 : 0); }  // pnorm.hpp:23-30

}  // namespace

extern "C" {

int w1mg_poisson_solve(w1mg_ctx* c, int n, const double* b, double* out, int check_compat) {
    return guard([&] {
        check_n(n);
        const long V = (long)(n + 1) * (n + 1);
        if (check_compat) {  // poisson.cpp:62-68 (plain sums)
            double total = 0.0, absolute = 0.0;
            for (long k = 0; k < V; ++k) {
                total += b[k];
                absolute += std::fabs(b[k]);
            }
            if (std::fabs(total) > 1e-10 * absolute)
                fail(W1MG_EINVAL, "NeumannPoissonSolver: right-hand side must sum to zero");
        }
        PLevel lv = make_plevel(c, "poisson", n, 1, 1.0, 1.0, nullptr, 0);
        pput(c, lv, 0, P_RES, b, n + 1, n + 1);
        poisson_apply(c, lv, P_RES, false);
        remove_mean(c, lv, P_PSI);
        pget(c, lv, 0, P_PSI, out, n + 1, n + 1);
        CK(cudaStreamSynchronize(c->stream));
    });
}

int w1mg_project_affine(w1mg_ctx* c, int n, const double* mx, const double* my,
                        const double* rho, double* ox, double* oy) {
    return guard([&] {
        check_n(n);
        // one PDHG "half step" with varphi_bar = 0: v = m, m' = v - A* psi
        PLevel lv = make_plevel(c, "affine", n, 1, 0.0, 0.0, nullptr, 0);
        CK(cudaMemsetAsync(lv.base, 0, sizeof(double) * P_NSLOT * lv.L.plane, c->stream));
        pput(c, lv, 0, P_MX, mx, n, n + 1);
        pput(c, lv, 0, P_MY, my, n + 1, n);
        pput(c, lv, 0, P_RHO, rho, n + 1, n + 1);
        pdhg_init_ctl(c, lv, -1.0, 1);
        pdhg_pre_kernel<<<lv.grid, lv.blk, 0, c->stream>>>(lv.args);
        ++c->launches;
        poisson_apply(c, lv, P_RES, false);
        remove_mean(c, lv, P_PSI);  // poisson.cpp:116 uses the zero-mean potential
        pdhg_post_kernel<1><<<lv.grid, lv.blk, 0, c->stream>>>(lv.args);
        ++c->launches;
        CK(cudaGetLastError());
        pget(c, lv, 0, P_MX, ox, n, n + 1);
        pget(c, lv, 0, P_MY, oy, n + 1, n);
        CK(cudaStreamSynchronize(c->stream));
    });
}

int w1mg_recover_potential(w1mg_ctx* c, int n, const double* dx, const double* dy, double* phi) {
    return guard([&] {
        check_n(n);
        PLevel lv = make_plevel(c, "recover", n, 1, 1.0, 1.0, nullptr, 0);
        CK(cudaMemsetAsync(lv.base, 0, sizeof(double) * P_NSLOT * lv.L.plane, c->stream));
        pput(c, lv, 0, P_PX, dx, n, n + 1);
        pput(c, lv, 0, P_PY, dy, n + 1, n);
        pdhg_values(c, lv, 1, nullptr, nullptr);
        pget(c, lv, 0, P_PSI, phi, n + 1, n + 1);
        CK(cudaStreamSynchronize(c->stream));
    });
}

int w1mg_pdhg_run(w1mg_ctx* c, int n, const double* rho, const double* m0x, const double* m0y,
                  const double* d0x, const double* d0y, const double* b0x, const double* b0y,
                  int pnorm, double mu, double tau, double tol, long max_iters, double* mx,
                  double* my, double* dx, double* dy, double* bx, double* by, double* phi,
                  double* fpr_hist, long hist_cap, w1mg_cp_report* rep) {
    return guard([&] {
        check_n(n);
        check_pnorm(pnorm);
        if (!rho) fail(W1MG_EINVAL, "null rho");
        long cap = (fpr_hist && hist_cap > 0) ? hist_cap : 0;
        double* dh = cap ? c->get<double>("pdhg.hist", cap) : nullptr;
        PLevel lv = make_plevel(c, "pdhg", n, 1, mu, tau, dh, cap);
        CK(cudaMemsetAsync(lv.base, 0, sizeof(double) * P_NSLOT * lv.L.plane, c->stream));
        pput(c, lv, 0, P_RHO, rho, n + 1, n + 1);
        if (m0x) pput(c, lv, 0, P_MX, m0x, n, n + 1);
        if (m0y) pput(c, lv, 0, P_MY, m0y, n + 1, n);
        if (d0x) pput(c, lv, 0, P_PX, d0x, n, n + 1);
        if (d0y) pput(c, lv, 0, P_PY, d0y, n + 1, n);
        // varphi_bar^0 = varphi^0 unless given
        const double* ux = b0x ? b0x : d0x;
        const double* uy = b0y ? b0y : d0y;
        if (ux) pput(c, lv, 0, P_BX, ux, n, n + 1);
        if (uy) pput(c, lv, 0, P_BY, uy, n + 1, n);
        CK(cudaEventRecord(c->t0, c->stream));
        pdhg_init_ctl(c, lv, tol, max_iters);
        run_pdhg_iters(c, lv, conj_q(pnorm), max_iters);
        CK(cudaEventRecord(c->t1, c->stream));
        double* vals = c->get<double>("pdhg.vals", 2);
        pdhg_values(c, lv, pnorm, vals, vals + 1);
        PairCtl hc;
        double hv[2];
        CK(cudaMemcpyAsync(&hc, lv.ctl, sizeof(PairCtl), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(hv, vals, 16, cudaMemcpyDeviceToHost, c->stream));
        if (mx) pget(c, lv, 0, P_MX, mx, n, n + 1);
        if (my) pget(c, lv, 0, P_MY, my, n + 1, n);
        if (dx) pget(c, lv, 0, P_PX, dx, n, n + 1);
        if (dy) pget(c, lv, 0, P_PY, dy, n + 1, n);
        if (bx) pget(c, lv, 0, P_BX, bx, n, n + 1);
        if (by) pget(c, lv, 0, P_BY, by, n + 1, n);
        if (phi) pget(c, lv, 0, P_PSI, phi, n + 1, n + 1);
        CK(cudaStreamSynchronize(c->stream));
        long nh = std::min(hc.it, cap);
        if (nh > 0) CK(cudaMemcpy(fpr_hist, dh, nh * 8, cudaMemcpyDeviceToHost));
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

// Eq. 12 between two states (value API)
int w1mg_pdhg_residual(w1mg_ctx* c, int n, const double* cmx, const double* cmy,
                       const double* cdx, const double* cdy, const double* pmx, const double* pmy,
                       const double* pdx, const double* pdy, double mu, double tau, double* out) {
    return guard([&] {
        check_n(n);
        const size_t E = (size_t)n * (n + 1);
        const double* src[8] = {cmx, cmy, cdx, cdy, pmx, pmy, pdx, pdy};
        double* d[8];
        for (int k = 0; k < 8; ++k) {
            d[k] = c->get<double>("pres." + std::to_string(k), E);
            CK(cudaMemcpyAsync(d[k], src[k], E * 8, cudaMemcpyDefault, c->stream));
        }
        for (int k = 0; k < 4; ++k) {
            sub_inplace_kernel<<<(int)((E + 255) / 256), 256, 0, c->stream>>>(d[k], d[k + 4], (long)E);
            ++c->launches;
        }
        CK(cudaGetLastError());
        double* r = c->get<double>("pres.r", 6);
        // x-edges n wide x (n+1) rows, y-edges (n+1) wide x n rows
        reduce_pairs(c, FRefDot{d[0], d[0], n}, n, n + 1, 1, 1.0, 1.0, r + 0);
        reduce_pairs(c, FRefDot{d[1], d[1], n + 1}, n + 1, n, 1, 1.0, 1.0, r + 1);
        reduce_pairs(c, FRefDot{d[2], d[2], n}, n, n + 1, 1, 1.0, 1.0, r + 2);
        reduce_pairs(c, FRefDot{d[3], d[3], n + 1}, n + 1, n, 1, 1.0, 1.0, r + 3);
        reduce_pairs(c, FRefDot{d[2], d[0], n}, n, n + 1, 1, 1.0, 1.0, r + 4);
        reduce_pairs(c, FRefDot{d[3], d[1], n + 1}, n + 1, n, 1, 1.0, 1.0, r + 5);
        double hr[6];
        CK(cudaMemcpyAsync(hr, r, 48, cudaMemcpyDefault, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        const double h = 1.0 / n;
        const double h2 = h * h;
        *out = h2 * ((hr[0] + hr[1]) / mu + (hr[2] + hr[3]) / tau + 2.0 * (hr[4] + hr[5]));
    });
}

// Cascadic Algorithm 4 for one pair over per-level sources (coarse -> fine).
int w1mg_ml_pdhg_run(w1mg_ctx* c, int n_finest, const double* rho_levels,
                     const w1mg_ml_params* prm, double* mx, double* my, double* dx, double* dy,
                     double* phi, w1mg_level_stats* stats, double* fpr_hist, long hist_cap,
                     w1mg_cp_report* rep) {
    return guard([&] {
        check_n(n_finest);
        if (!prm) fail(W1MG_EINVAL, "null parameters");
        check_pnorm(prm->pnorm);
        const int levels = prm->levels;
        if (levels < 1 || n_finest % (1 << (levels - 1)) != 0)
            fail(W1MG_EINVAL, "make_schedule: N must be divisible by 2^(L-1)");
        if (prm->rel_tol <= 0 && !prm->eps) fail(W1MG_EINVAL, "tolerances: need rel_tol > 0 or eps");
        const double step = w1mg_pdhg_step_size(prm->step_mode);
        const int q = conj_q(prm->pnorm);
        long cap = (fpr_hist && hist_cap > 0) ? hist_cap : 0;
        double* dh = cap ? c->get<double>("mlp.hist", cap) : nullptr;
        std::vector<PLevel> lv;
        for (int l = 0; l < levels; ++l) {
            const int n = n_finest >> (levels - 1 - l);
            const bool fin = l == levels - 1;
            lv.push_back(make_plevel(c, "mlp" + std::to_string(l), n, 1, step, step,
                                     fin ? dh : nullptr, fin ? cap : 0));
        }
        size_t off = 0;
        for (auto& L : lv) {
            CK(cudaMemsetAsync(L.base, 0, sizeof(double) * P_NSLOT * L.L.plane, c->stream));
            pput(c, L, 0, P_RHO, rho_levels + off, L.n + 1, L.n + 1);
            off += (size_t)(L.n + 1) * (L.n + 1);
        }
        while ((int)c->lev_ev.size() < 2 * levels) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            c->lev_ev.push_back(e);
        }
        c->lev_count = levels;
        std::vector<PairCtl> hc(levels);
        dim3 blk(32, 8);
        for (int l = 0; l < levels; ++l) {
            PLevel& L = lv[l];
            CK(cudaEventRecord(c->lev_ev[2 * l], c->stream));
            if (prm->rel_tol > 0) {
                // G_cold: one step from the zero state (scratch run), then arm tol
                SweepArgs cold = L.args;
                cold.hist = nullptr;
                PLevel Z = L;
                Z.args = cold;
                pdhg_init_ctl(c, Z, -1.0, 1);
                pdhg_iteration(c, Z, q);
                pdhg_arm_tol_kernel<<<1, 32, 0, c->stream>>>(L.ctl, 1, prm->rel_tol,
                                                               prm->max_iters, L.ndone);
                ++c->launches;
                CK(cudaGetLastError());
                // reset the state the cold step touched
                for (int s : {P_MX, P_MY, P_PX, P_PY, P_BX, P_BY})
                    CK(cudaMemsetAsync(L.base + (long)s * L.L.plane, 0, sizeof(double) * L.L.plane,
                                       c->stream));
                CK(cudaMemsetAsync(L.ticket, 0, sizeof(unsigned), c->stream));
            } else {
                pdhg_init_ctl(c, L, prm->eps[l], prm->max_iters);
            }
            if (l > 0) {
                pdhg_prolong_kernel<<<node_grid(L.n, 1, blk), blk, 0, c->stream>>>(
                    lv[l - 1].base, lv[l - 1].L, L.base, L.L);
                ++c->launches;
                CK(cudaGetLastError());
            }
            run_pdhg_iters(c, L, q, prm->max_iters);
            CK(cudaEventRecord(c->lev_ev[2 * l + 1], c->stream));
            CK(cudaMemcpyAsync(&hc[l], L.ctl, sizeof(PairCtl), cudaMemcpyDeviceToHost, c->stream));
        }
        const PLevel& F = lv.back();
        double* vals = c->get<double>("mlp.vals", 2);
        pdhg_values(c, F, prm->pnorm, vals, vals + 1);
        double hv[2];
        CK(cudaMemcpyAsync(hv, vals, 16, cudaMemcpyDeviceToHost, c->stream));
        const int n = F.n;
        if (mx) pget(c, F, 0, P_MX, mx, n, n + 1);
        if (my) pget(c, F, 0, P_MY, my, n + 1, n);
        if (dx) pget(c, F, 0, P_PX, dx, n, n + 1);
        if (dy) pget(c, F, 0, P_PY, dy, n + 1, n);
        if (phi) pget(c, F, 0, P_PSI, phi, n + 1, n + 1);
        CK(cudaStreamSynchronize(c->stream));
        std::vector<double> secs;
        level_seconds(c, secs);
        long nh = std::min(hc.back().it, cap);
        if (nh > 0) CK(cudaMemcpy(fpr_hist, dh, nh * 8, cudaMemcpyDeviceToHost));
        long total = 0;
        double tsec = 0.0;
        for (int l = 0; l < levels; ++l) {
            total += hc[l].it;
            tsec += secs[l];
            if (stats) {
                stats[l].h = 1.0 / lv[l].n;
                stats[l].eps = hc[l].tol;
                stats[l].iters = hc[l].it;
                stats[l].fpr_final = hc[l].fpr;
                stats[l].seconds = secs[l];
            }
        }
        if (rep) {
            rep->distance = hv[0];
            rep->dual_value = hv[1];
            rep->iterations = total;
            rep->fpr_final = hc.back().fpr;
            rep->converged = hc.back().fpr < hc.back().tol ? 1 : 0;
            rep->seconds = tsec;
        }
    });
}

}  // extern "C"
