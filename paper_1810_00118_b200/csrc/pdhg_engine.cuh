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
#include "dct_kernels.cuh"
#include "pdhg_persist.cuh"
#include "pdhg_rs.cuh"
#include "pdhg_rs2.cuh"
#include "pdhg_rspf.cuh"

namespace {

// One PDHG level batch (B pairs, P_NSLOT planes each) + its DCT plan.
struct PLevel {
    int n = 0, B = 0;
    Layout L{};
    double* base = nullptr;
    PairCtl* ctl = nullptr;
    unsigned* ticket = nullptr;
    int* ndone = nullptr;
    SweepArgs args{};
    dim3 grid, blk;
    const double* C = nullptr;    // dense DCT-II matrix (level-resident small kernel only)
    const double* S = nullptr;    // dense DCT-III matrix (level-resident small kernel only)
    const double* lam = nullptr;  // lambda_k, poisson.cpp:28-30
    DctPlan dp{};                 // prime-factor DCT plan (dct_kernels.cuh)
    int rows_f = 1, cols = 1, rows_i = 1;  // vectors per CTA of the three DCT launches
    int rows_p = 0;  // ... of the fused row DCT-III + post launch (0: does not fit, unfused)
};

// Dense DCT matrices for m = n+1, built once per size on the host in long
// double and cached on the device -- only for the level-resident small
// kernel (pdhg_small.cuh, m <= kPdhgSmallMaxM), which multiplies them in
// shared memory.
void dct_operators(w1mg_ctx* c, int n, const double** C, const double** S) {
    const int m = n + 1;
    const std::string key = std::to_string(m);
    const bool fresh = c->bufs.find("dct.C." + key) == c->bufs.end();
    double* dC = c->get<double>("dct.C." + key, (size_t)m * m);
    double* dS = c->get<double>("dct.S." + key, (size_t)m * m);
    if (fresh) {
        std::vector<double> hC((size_t)m * m), hS((size_t)m * m);
        const long double pi = 3.141592653589793238462643383279502884L;
        for (int j = 0; j < m; ++j)
            for (int k = 0; k < m; ++k) {
                long a = ((long)(2 * j + 1) * k) % (4L * m);  // exact angle reduction
                long b = ((long)j * (2 * k + 1)) % (4L * m);
                hC[(size_t)j * m + k] = (double)(2.0L * cosl(pi * a / (2.0L * m)));
                hS[(size_t)j * m + k] = j == 0 ? 1.0 : (double)(2.0L * cosl(pi * b / (2.0L * m)));
            }
        CK(cudaMemcpy(dC, hC.data(), hC.size() * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dS, hS.data(), hS.size() * 8, cudaMemcpyHostToDevice));
    }
    *C = dC;
    *S = dS;
}

// lambda_k = (2 - 2 cos(pi k / m)) / h^2 exactly as poisson.cpp:28-30
const double* dct_lambda(w1mg_ctx* c, int n) {
    const int m = n + 1;
    const std::string key = "dct.lam." + std::to_string(m);
    const bool fresh = c->bufs.find(key) == c->bufs.end();
    double* dl = c->get<double>(key, m);
    if (fresh) {
        std::vector<double> hl(m);
        const double h = 1.0 / n;
        const double inv_h2 = 1.0 / (h * h);
        for (int k = 0; k < m; ++k) hl[k] = (2.0 - 2.0 * std::cos(M_PI * k / m)) * inv_h2;
        CK(cudaMemcpy(dl, hl.data(), hl.size() * 8, cudaMemcpyHostToDevice));
    }
    return dl;
}

// Prime-factor split m = N1 N2: coprime, N1 >= N2, N1 + N2 minimal (prime
// powers kept whole; a prime m gives N2 = 1).
void dct_split(int m, int& N1, int& N2) {
    std::vector<int> pp;
    int x = m;
    for (int q = 2; (long)q * q <= x; ++q)
        if (x % q == 0) {
            int pw = 1;
            while (x % q == 0) {
                x /= q;
                pw *= q;
            }
            pp.push_back(pw);
        }
    if (x > 1) pp.push_back(x);
    N1 = m;
    N2 = 1;
    const int np = (int)pp.size();
    for (int mask = 0; mask < (1 << np); ++mask) {
        int a = 1;
        for (int t = 0; t < np; ++t)
            if (mask >> t & 1) a *= pp[t];
        const int b = m / a;
        if (a >= b && a + b < N1 + N2) {
            N1 = a;
            N2 = b;
        }
    }
}

// DCT plan for m: index maps and twiddle tables (host long double, exact
// angle reduction), cached on the device per context.
DctPlan dct_plan(w1mg_ctx* c, int m) {
    auto it = c->dct.find(m);
    if (it != c->dct.end()) return it->second;
    if (m > 32767) fail(W1MG_EINVAL, "Poisson solve: grid too large for the DCT plan");
    DctPlan p{};
    p.m = m;
    dct_split(m, p.N1, p.N2);
    const int N1 = p.N1, N2 = p.N2;
    p.H1 = N1 / 2 + 1;
    p.T1 = (N1 - 1) / 2;
    p.E1 = 1 - (N1 & 1);
    p.H2 = N2 / 2 + 1;
    p.T2 = (N2 - 1) / 2;
    p.E2 = 1 - (N2 & 1);
    p.H1p = round4(p.H1);
    p.H2p = round4(p.H2);
    const long double pi = 3.141592653589793238462643383279502884L;
    auto cosN = [&](long a, long N) { return (double)cosl(2.0L * pi * (long double)(a % N) / N); };
    auto sinN = [&](long a, long N) { return (double)sinl(2.0L * pi * (long double)(a % N) / N); };
    auto pos = [&](int n) { return n <= (m - 1) / 2 ? 2 * n : 2 * (m - 1 - n) + 1; };
    std::vector<short> idxA((size_t)N2 * N1), crt((size_t)N2 * p.H1);
    for (int n2 = 0; n2 < N2; ++n2)
        for (int t = 0; t < N1; ++t) idxA[(size_t)n2 * N1 + t] = (short)pos((int)(((long)N2 * t + (long)N1 * n2) % m));
    for (int k = 0; k < m; ++k)
        if (k % N1 < p.H1) crt[(size_t)(k % N2) * p.H1 + k % N1] = (short)k;
    std::vector<double> tw1(2 * (size_t)N1), tw2(2 * (size_t)N2);
    for (int j = 0; j < N1; ++j) {
        tw1[j] = cosN(j, N1);
        tw1[N1 + j] = sinN(j, N1);
    }
    for (int j = 0; j < N2; ++j) {
        tw2[j] = cosN(j, N2);
        tw2[N2 + j] = sinN(j, N2);
    }
    std::vector<double> mk(2 * (size_t)m);
    for (int k = 0; k < m; ++k) {  // pi k / 2m = 2 pi k / 4m
        mk[2 * k] = cosN(k, 4L * m);
        mk[2 * k + 1] = sinN(k, 4L * m);
    }
    // one contiguous block in the shared-memory layout (dct_view): a CTA
    // stages it with a single TMA bulk copy
    std::vector<double> blk((size_t)dct_tab_doubles(p), 0.0);
    double* bp = blk.data();
    std::copy(tw1.begin(), tw1.end(), bp);
    std::copy(tw2.begin(), tw2.end(), bp + 2 * N1);
    std::copy(mk.begin(), mk.end(), bp + 2 * N1 + 2 * N2);
    short* sp = reinterpret_cast<short*>(bp + 2 * N1 + 2 * N2 + 2 * m);
    std::copy(idxA.begin(), idxA.end(), sp);
    std::copy(crt.begin(), crt.end(), sp + idxA.size());
    int* fp = reinterpret_cast<int*>(sp + round4((int)(idxA.size() + crt.size())));
    for (int k = 0; k < m; ++k) {  // forward output map (dct2_vectors)
        int kk = k, k1 = k % N1, cj = 0;
        if (k1 >= p.H1) {
            kk = m - k;
            k1 = kk % N1;
            cj = 1;
        }
        const int k2 = kk % N2, mir = (N2 > 1 && k2 >= p.H2) ? 1 : 0;
        const int q = mir ? N2 - k2 : k2;
        fp[k] = k1 | (q << 16) | (mir << 29) | (cj << 30);
    }
    double* d = c->get<double>("dctp." + std::to_string(m), blk.size());
    CK(cudaMemcpy(d, blk.data(), blk.size() * 8, cudaMemcpyHostToDevice));
    p.tabs = d;
    p.tw1 = d;
    p.tw2 = d + 2 * N1;
    p.mk = d + 2 * N1 + 2 * N2;
    p.idxA = reinterpret_cast<const short*>(p.mk + 2 * m);
    p.crt = p.idxA + idxA.size();
    p.f5 = reinterpret_cast<const int*>(p.idxA + round4((int)(idxA.size() + crt.size())));
    c->dct[m] = p;
    return p;
}

constexpr size_t kDctSmemMax = (227u << 10) - 1024;  // per-block opt-in limit minus static smem

void dct_kernel_attrs() {
    static unsigned long long done = 0;  // per device
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (done >> (dev & 63) & 1ull) return;
    const int mx = (int)kDctSmemMax;
    CK(cudaFuncSetAttribute(dct_rows_fwd_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(dct_rows_fwd_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(dct_cols_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(dct_rows_inv_kernel<0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(dct_rows_inv_kernel<1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(dct_rows_inv_kernel<1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(dct_rows_inv_kernel<1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(pdhg_persist_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(pdhg_persist_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(pdhg_persist_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    done |= 1ull << (dev & 63);
}

// Vectors per CTA of a DCT launch: the fewest (a power of two <= 16) whose
// grid still runs in ONE wave of two CTAs per SM -- a CTA's transform is a
// chain of dependent shared-memory phases, so the launch takes one CTA
// latency per wave -- within the shared-memory budget (`extra` vectors are
// transformed on top, e.g. the post step's halo row).
int dct_vectors_per_cta(const DctPlan& p, int B, int num_sms, int extra) {
    int R = 1;
    while (R < 16 && (long)((p.m + R - 1) / R) * B > 2L * num_sms &&
           dct_smem_bytes(p, 2 * R + extra) <= kDctSmemMax)
        R <<= 1;
    while (R > 1 && dct_smem_bytes(p, R + extra) > kDctSmemMax) R >>= 1;
    return dct_smem_bytes(p, R + extra) <= kDctSmemMax ? R : 0;
}

// Rows per CTA of the fused row DCT-III + post launch: R + 1 vectors (one
// halo row), R + 1 a power of two (the transforms split vector indices by
// shifts): R in {1, 3, 7, 15}, the most that keep one wave of two CTAs per
// SM within the shared-memory budget; 0 if even R = 1 does not fit.
int dct_post_rows_per_cta(const DctPlan& p, int B, int num_sms) {
    int R = 1;
    while (R < 15 && (long)((p.m + R - 1) / R) * B > 2L * num_sms &&
           dct_smem_bytes(p, 2 * (R + 1)) <= kDctSmemMax)
        R = 2 * (R + 1) - 1;
    while (R > 1 && dct_smem_bytes(p, R + 1) > kDctSmemMax) R = (R + 1) / 2 - 1;
    return dct_smem_bytes(p, R + 1) <= kDctSmemMax ? R : 0;
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
    // residual partials: node-grid blocks (pdhg_post_kernel) or one block per
    // DCT row group (dct_rows_inv_kernel, at most m)
    a.partial = c->get<double>(tag + ".partial",
                               (size_t)B * std::max<size_t>((size_t)lv.grid.x * lv.grid.y, n + 1) * 3);
    lv.lam = dct_lambda(c, n);
    if (n + 1 <= kPdhgSmallMaxM) dct_operators(c, n, &lv.C, &lv.S);
    lv.dp = dct_plan(c, n + 1);
    lv.rows_f = dct_vectors_per_cta(lv.dp, B, c->num_sms, 0);
    lv.cols = dct_vectors_per_cta(lv.dp, B, c->num_sms, 0);
    lv.rows_i = dct_vectors_per_cta(lv.dp, B, c->num_sms, 0);
    lv.rows_p = dct_post_rows_per_cta(lv.dp, B, c->num_sms);
    if (!lv.rows_f || !lv.cols || !lv.rows_i)
        fail(W1MG_EINVAL, "Poisson solve: grid too large for the shared-memory DCT");
    dct_kernel_attrs();
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

// psi = (A A*)^+ r on every pair: slot `in` -> P_PSI through the three DCT
// launches (P_T scratch), poisson.cpp:72-99 without the mean removal.
void poisson_apply(w1mg_ctx* c, const PLevel& lv, int in, bool check_done) {
    const int m = lv.n + 1, cd = check_done ? 1 : 0;
    const DctPlan& p = lv.dp;
    const double scale = 1.0 / (4.0 * double(m) * double(m));  // poisson.cpp:93
    dct_rows_fwd_kernel<0><<<dim3((m + lv.rows_f - 1) / lv.rows_f, lv.B), 256,
                             dct_smem_bytes(p, lv.rows_f), c->stream>>>(lv.args, p, in, lv.rows_f, cd);
    dct_cols_kernel<<<dim3((m + lv.cols - 1) / lv.cols, lv.B), 256, dct_smem_bytes(p, lv.cols),
                      c->stream>>>(lv.args, p, lv.lam, lv.cols, cd);
    dct_rows_inv_kernel<0, 1><<<dim3((m + lv.rows_i - 1) / lv.rows_i, lv.B), 256,
                                dct_smem_bytes(p, lv.rows_i), c->stream>>>(lv.args, p, lv.rows_i,
                                                                            scale, cd);
    CK(cudaGetLastError());
    c->launches += 3;
}

// psi -= compensated mean (poisson.cpp:96-98)
void remove_mean(w1mg_ctx* c, const PLevel& lv, int slot) {
    double* sums = c->get<double>("pdhg.mean", lv.B);
    reduce_pairs(c, FPSlot{lv.base, lv.L, slot}, lv.n + 1, lv.n + 1, lv.B, 1.0, 1.0, sums);
    subtract_mean_kernel<<<lv.grid, lv.blk, 0, c->stream>>>(lv.args, slot, sums);
    ++c->launches;
    CK(cudaGetLastError());
}

// One PDHG iteration = three launches: rows (pre step + DCT-II), columns
// (DCT-II, divide, DCT-III), rows (DCT-III + post step + Eq. 12 + stop rule).
constexpr int kPdhgLaunches = 3;

void pdhg_iteration(w1mg_ctx* c, const PLevel& lv, int q) {
    const int m = lv.n + 1;
    const DctPlan& p = lv.dp;
    const double scale = 1.0 / (4.0 * double(m) * double(m));  // poisson.cpp:93
    dct_rows_fwd_kernel<1><<<dim3((m + lv.rows_f - 1) / lv.rows_f, lv.B), 256,
                             dct_smem_bytes(p, lv.rows_f), c->stream>>>(lv.args, p, P_RES,
                                                                        lv.rows_f, 1);
    dct_cols_kernel<<<dim3((m + lv.cols - 1) / lv.cols, lv.B), 256, dct_smem_bytes(p, lv.cols),
                      c->stream>>>(lv.args, p, lv.lam, lv.cols, 1);
    if (lv.rows_p) {
        const dim3 gi((m + lv.rows_p - 1) / lv.rows_p, lv.B);
        const size_t si = dct_smem_bytes(p, lv.rows_p + 1);
        switch (q) {
            case 0: dct_rows_inv_kernel<1, 0><<<gi, 256, si, c->stream>>>(lv.args, p, lv.rows_p, scale, 1); break;
            case 1: dct_rows_inv_kernel<1, 1><<<gi, 256, si, c->stream>>>(lv.args, p, lv.rows_p, scale, 1); break;
            default: dct_rows_inv_kernel<1, 2><<<gi, 256, si, c->stream>>>(lv.args, p, lv.rows_p, scale, 1); break;
        }
    } else {  // very large m: psi through P_PSI, then the node-grid post kernel
        dct_rows_inv_kernel<0, 1><<<dim3((m + lv.rows_i - 1) / lv.rows_i, lv.B), 256,
                                    dct_smem_bytes(p, lv.rows_i), c->stream>>>(lv.args, p, lv.rows_i,
                                                                                scale, 1);
        switch (q) {
            case 0: pdhg_post_kernel<0><<<lv.grid, lv.blk, 0, c->stream>>>(lv.args); break;
            case 1: pdhg_post_kernel<1><<<lv.grid, lv.blk, 0, c->stream>>>(lv.args); break;
            default: pdhg_post_kernel<2><<<lv.grid, lv.blk, 0, c->stream>>>(lv.args); break;
        }
        ++c->launches;
    }
    c->launches += kPdhgLaunches;
    CK(cudaGetLastError());
}

// Level-persistent PDHG for one pair (pdhg_persist.cuh): every iteration of
// the level in one cooperative launch (g_pdhg_persist, level_engine.cuh).

template <int Q>
bool launch_pdhg_persist_q(w1mg_ctx* c, const PLevel& lv) {
    const DctPlan& p = lv.dp;
    const int m = p.m;
    // vectors per chunk: the fewest whose chunks fit co-resident (two CTAs per
    // SM where the shared memory allows)
    int R = 1, occ = 0;
    size_t smem = 0;
    for (;; R <<= 1) {
        if (R > 16) return false;
        smem = dct_smem_bytes(p, R);
        if (smem > kDctSmemMax) return false;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pdhg_persist_kernel<Q>,
                                                         kPersistThreads, smem));
        if (occ >= 1 && (m + R - 1) / R <= c->num_sms) break;
    }
    const int chunks = (m + R - 1) / R;
    const int G = std::min(chunks, c->num_sms * occ);
    unsigned* bar = c->get<unsigned>("persist.bar", 2);
    int* err = c->get<int>("persist.err", 1);
    CK(cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), c->stream));  // arrival counter
    CK(cudaMemsetAsync(err, 0, sizeof(int), c->stream));
    GridBar gb{bar, bar + 1, err};
    double* part = c->get<double>("persist.part", (size_t)3 * G);
    const double scale = 1.0 / (4.0 * double(m) * double(m));  // poisson.cpp:93
    SweepArgs a = lv.args;
    const DctPlan* pp = &p;
    const double* lam = lv.lam;
    unsigned long long* stamps = nullptr;
    if (std::getenv("W1MG_PERSIST_STAMPS")) {
        stamps = c->get<unsigned long long>("persist.stamps", 640);
        CK(cudaMemsetAsync(stamps, 0, 640 * 8, c->stream));
    }
    void* args[] = {(void*)&a, (void*)pp, (void*)&lam, (void*)&R, (void*)&R, (void*)&scale,
                    (void*)&gb, (void*)&part, (void*)&stamps};
    CK(cudaLaunchCooperativeKernel((const void*)pdhg_persist_kernel<Q>, dim3(G),
                                   dim3(kPersistThreads), args, smem, c->stream));
    ++c->launches;
    int herr = 0;
    CK(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (herr) fail(W1MG_ECUDA, "level-persistent PDHG: grid barrier timed out");
    if (stamps) {  // per-phase ns of iterations 8..63: A, bar, B, bar, C, bar, D, bar
        std::vector<unsigned long long> h(640);
        CK(cudaMemcpy(h.data(), stamps, 640 * 8, cudaMemcpyDeviceToHost));
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        int cnt = 0;
        for (int it = 8; it < 63; ++it) {
            if (!h[(it + 1) * 10]) break;
            for (int q = 0; q < 8; ++q) acc[q] += double(h[it * 10 + q + 1] - h[it * 10 + q]);
            ++cnt;
        }
        if (cnt)
            std::fprintf(stderr, "persist m=%d G=%d R=%d ns: A %.0f bar %.0f B %.0f bar %.0f C %.0f bar %.0f D %.0f bar %.0f\n",
                         m, G, R, acc[0] / cnt, acc[1] / cnt, acc[2] / cnt, acc[3] / cnt,
                         acc[4] / cnt, acc[5] / cnt, acc[6] / cnt, acc[7] / cnt);
    }
    return true;
}

bool launch_pdhg_persist(w1mg_ctx* c, const PLevel& lv, int q) {
    if (!g_pdhg_persist || lv.B != 1) return false;
    if (q == 0) return launch_pdhg_persist_q<0>(c, lv);
    if (q == 1) return launch_pdhg_persist_q<1>(c, lv);
    return launch_pdhg_persist_q<2>(c, lv);
}

// Row-resident level-persistent PDHG for one pair (pdhg_rs.cuh): rows of the
// state in shared memory for the whole level, two grid barriers per
// iteration, register-stationary dense DCT for m <= 129 (odd), prime-factor
// transforms above.  g_pdhg_rs (level_engine.cuh): 0 off, 1 auto (every
// one-pair level, also instead of the one-CTA small kernel: 7.4 vs 12 us per
// iteration at 33^2), 2 forces the prime-factor transforms of
// dct_kernels.cuh (A/B).

struct RsTables {
    const double* cosq;
    const double* lamq;
};

// cos(pi j / 2m), j < 4m (host long double) and lambda in position order
RsTables rs_tables(w1mg_ctx* c, int n, bool dense) {
    const int m = n + 1, h = (m - 1) / 2;
    const std::string kc = "rs.cosq." + std::to_string(m);
    const std::string kl = std::string(dense ? "rs.lamq.d." : "rs.lamq.n.") + std::to_string(m);
    const bool fc = c->bufs.find(kc) == c->bufs.end(), fl = c->bufs.find(kl) == c->bufs.end();
    double* dc = c->get<double>(kc, (size_t)4 * m);
    double* dl = c->get<double>(kl, m);
    if (fc) {
        std::vector<double> hc((size_t)4 * m);
        const long double pi = 3.141592653589793238462643383279502884L;
        for (int j = 0; j < 4 * m; ++j) hc[j] = (double)cosl(pi * (long double)j / (2.0L * m));
        CK(cudaMemcpy(dc, hc.data(), hc.size() * 8, cudaMemcpyHostToDevice));
    }
    if (fl) {
        std::vector<double> hl(m);
        const double hh = 1.0 / n;
        const double inv_h2 = 1.0 / (hh * hh);
        auto lam = [&](int k) { return (2.0 - 2.0 * std::cos(M_PI * k / m)) * inv_h2; };  // poisson.cpp:28-30
        for (int pos = 0; pos < m; ++pos) {
            int k = pos;
            if (dense) k = pos < h ? 2 * pos + 2 : (pos < 2 * h ? 2 * (pos - h) + 1 : 0);
            hl[pos] = lam(k);
        }
        CK(cudaMemcpy(dl, hl.data(), hl.size() * 8, cudaMemcpyHostToDevice));
    }
    return RsTables{dc, dl};
}

// ns between consecutive time stamps of CTA 0 (iterations 8..62 averaged);
// the stamps in use are listed in the kernels (0 = iteration start)
void rs_print_stamps(w1mg_ctx* c, const unsigned long long* stamps, int m, int G, int R, int TS) {
    (void)c;
    if (!stamps) return;
    const int NS = kRsStampSlots;
    std::vector<unsigned long long> h((size_t)64 * NS);
    CK(cudaMemcpy(h.data(), stamps, h.size() * 8, cudaMemcpyDeviceToHost));
    std::vector<double> acc(NS, 0.0);
    double tot = 0.0;
    int cnt = 0;
    for (int it = 8; it < 62; ++it) {
        if (!h[(size_t)(it + 1) * NS]) break;
        unsigned long long prev = h[(size_t)it * NS];
        for (int q = 1; q < NS; ++q) {
            const unsigned long long t = h[(size_t)it * NS + q];
            if (!t) continue;
            acc[q] += double(t - prev);
            prev = t;
        }
        tot += double(h[(size_t)(it + 1) * NS] - h[(size_t)it * NS]);
        ++cnt;
    }
    if (!cnt) return;
    std::fprintf(stderr, "rs m=%d G=%d R=%d TS=%d ns:", m, G, R, TS);
    for (int q = 1; q < NS; ++q)
        if (acc[q] > 0.0) std::fprintf(stderr, " [%d] %.0f", q, acc[q] / cnt);
    std::fprintf(stderr, " | iter %.0f\n", tot / cnt);
}

template <int Q, int TS>
bool launch_pdhg_rs_qt(w1mg_ctx* c, const PLevel& lv, int R) {
    const DctPlan& p = lv.dp;
    const int m = p.m, G = (m + R - 1) / R, ms = m + 1;
    const size_t smem = rs_smem_doubles(p, R, TS) * sizeof(double);
    if (smem > kDctSmemMax || G + 1 > c->num_sms) return false;  // + the reducer CTA
    static unsigned long long attr = 0;  // per device
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (!(attr >> (dev & 63) & 1ull)) {
        CK(cudaFuncSetAttribute(pdhg_rs_kernel<Q, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kDctSmemMax));
        attr |= 1ull << (dev & 63);
    }
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pdhg_rs_kernel<Q, TS>, kRsThreads, smem));
    if (occ < 1) return false;
    const RsTables tb = rs_tables(c, lv.n, TS > 0);
    RsArgs ra{};
    ra.m = m;
    ra.h = (m - 1) / 2;
    ra.R = R;
    ra.G = G;
    ra.HP = 16 * TS;
    ra.posDC = TS > 0 ? 2 * ra.h : 0;
    ra.halo_x = TS > 0 ? 0 : 1;
    ra.cosq = tb.cosq;
    ra.lamq = tb.lamq;
    ra.scale = 1.0 / (4.0 * double(m) * double(m));  // poisson.cpp:93
    ra.vyb = c->get<double>("rs.vyb", (size_t)G * ms);
    ra.psb = c->get<double>("rs.psb", (size_t)G * ms);
    ra.flag = c->get<unsigned>("rs.flag", (size_t)2 * G);
    ra.part = c->get<double>("rs.part", (size_t)3 * G);
    ra.dec = c->get<int>("rs.dec", 2);
    CK(cudaMemsetAsync(ra.dec, 0, 2 * sizeof(int), c->stream));
    CK(cudaMemsetAsync(ra.flag, 0, sizeof(unsigned) * 2 * G, c->stream));
    unsigned* bar = c->get<unsigned>("persist.bar", 2);
    int* err = c->get<int>("persist.err", 1);
    CK(cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), c->stream));
    CK(cudaMemsetAsync(err, 0, sizeof(int), c->stream));
    GridBar gb{bar, bar + 1, err};
    ra.stamps = nullptr;
    if (std::getenv("W1MG_PERSIST_STAMPS")) {
        ra.stamps = c->get<unsigned long long>("rs.stamps", 64 * kRsStampSlots);
        CK(cudaMemsetAsync(ra.stamps, 0, 64 * kRsStampSlots * 8, c->stream));
    }
    SweepArgs a = lv.args;
    DctPlan pp = p;
    void* args[] = {(void*)&a, (void*)&pp, (void*)&ra, (void*)&gb};
    CK(cudaLaunchCooperativeKernel((const void*)pdhg_rs_kernel<Q, TS>, dim3(G + 1), dim3(kRsThreads), args,
                                   smem, c->stream));
    ++c->launches;
    int herr = 0;
    CK(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (herr) fail(W1MG_ECUDA, "row-resident PDHG: grid barrier timed out");
    rs_print_stamps(c, ra.stamps, m, G, R, TS);
    return true;
}

// 129 < m <= 257 (odd): clusters of two CTAs share the register-stationary
// DCT matrix (pdhg_rs2.cuh); cooperative launch of 2 x ceil(m / 2R) CTAs.
template <int Q>
bool launch_pdhg_rs2_q(w1mg_ctx* c, const PLevel& lv) {
    const int m = lv.n + 1, h = (m - 1) / 2, ms = m + 1;
    const int NC = c->num_sms / 2 - 1;  // one cluster for the reducer
    const int R = (m + 2 * NC - 1) / (2 * NC);
    const int G = 2 * ((m + 2 * R - 1) / (2 * R));
    const size_t smem = rs2_smem_doubles(m, R) * sizeof(double);
    if (smem > kDctSmemMax || 2 * R + 2 > kRs2NV) return false;
    static unsigned long long attr = 0;  // per device
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (!(attr >> (dev & 63) & 1ull)) {
        CK(cudaFuncSetAttribute(pdhg_rs2_kernel<Q>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kDctSmemMax));
        attr |= 1ull << (dev & 63);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(G + 2);  // + the reducer cluster
    cfg.blockDim = dim3(kRsThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    // W1MG_RS2_NOCOOP (profiling only): plain cluster launch -- ncu cannot replay
    // the cooperative one; the CTAs of one wave are co-resident on an idle GPU
    cfg.numAttrs = std::getenv("W1MG_RS2_NOCOOP") ? 1 : 2;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, pdhg_rs2_kernel<Q>, &cfg) != cudaSuccess ||
        2 * nclusters < G + 2) {
        cudaGetLastError();
        return false;
    }
    const RsTables tb = rs_tables(c, lv.n, true);
    RsArgs ra{};
    ra.m = m;
    ra.h = h;
    ra.R = R;
    ra.G = G;
    ra.HP = kRs2HP;
    ra.posDC = 2 * h;
    ra.halo_x = 0;
    ra.cosq = tb.cosq;
    ra.lamq = tb.lamq;
    ra.scale = 1.0 / (4.0 * double(m) * double(m));  // poisson.cpp:93
    ra.vyb = nullptr;
    ra.psb = nullptr;
    ra.flag = nullptr;
    ra.part = c->get<double>("rs.part", (size_t)3 * G);
    ra.dec = c->get<int>("rs.dec", 2);
    CK(cudaMemsetAsync(ra.dec, 0, 2 * sizeof(int), c->stream));
    unsigned* bar = c->get<unsigned>("persist.bar", 2);
    int* err = c->get<int>("persist.err", 1);
    CK(cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), c->stream));
    CK(cudaMemsetAsync(err, 0, sizeof(int), c->stream));
    GridBar gb{bar, bar + 1, err};
    ra.stamps = nullptr;
    if (std::getenv("W1MG_PERSIST_STAMPS")) {
        ra.stamps = c->get<unsigned long long>("rs.stamps", 64 * kRsStampSlots);
        CK(cudaMemsetAsync(ra.stamps, 0, 64 * kRsStampSlots * 8, c->stream));
    }
    (void)ms;
    CK(cudaLaunchKernelEx(&cfg, pdhg_rs2_kernel<Q>, lv.args, ra, gb));
    ++c->launches;
    int herr = 0;
    CK(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (herr) fail(W1MG_ECUDA, "row-resident PDHG (clusters): grid barrier timed out");
    rs_print_stamps(c, ra.stamps, m, G, R, 8);
    return true;
}

// m = N1 N2 (odd coprime factors, pdhg_rspf.cuh; instantiated for 513 = 27 x
// 19): register-stationary prime-factor transforms in the row-resident flow.
template <int Q, class P>
bool launch_pdhg_rspf_q(w1mg_ctx* c, const PLevel& lv) {
    const int m = P::M;
    const int R = (m + c->num_sms - 2) / (c->num_sms - 1), G = (m + R - 1) / R;  // one SM for the reducer
    const size_t smem = rspf_smem_doubles<P>(R) * sizeof(double);
    if (smem > kDctSmemMax || G + 1 > c->num_sms) return false;
    static unsigned long long attr = 0;  // per device
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (!(attr >> (dev & 63) & 1ull)) {
        CK(cudaFuncSetAttribute(pdhg_rspf_kernel<Q, P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kDctSmemMax));
        attr |= 1ull << (dev & 63);
    }
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pdhg_rspf_kernel<Q, P>, kPfThreads, smem));
    if (occ < 1) return false;
    const std::string kt = "rspf.tab." + std::to_string(m);
    const bool ft = c->bufs.find(kt) == c->bufs.end();
    short* dtab = c->get<short>(kt, P::NTAB);
    if (ft) {
        std::vector<short> ht(P::NTAB);
        rspf_tables<P>(ht.data());
        CK(cudaMemcpy(dtab, ht.data(), ht.size() * sizeof(short), cudaMemcpyHostToDevice));
    }
    const RsTables tb = rs_tables(c, lv.n, false);
    RsArgs ra{};
    ra.m = m;
    ra.h = (m - 1) / 2;
    ra.R = R;
    ra.G = G;
    ra.posDC = 0;
    ra.cosq = tb.cosq;
    ra.lamq = tb.lamq;
    ra.scale = 1.0 / (4.0 * double(m) * double(m));  // poisson.cpp:93
    ra.part = c->get<double>("rs.part", (size_t)3 * G);
    ra.dec = c->get<int>("rs.dec", 2);
    CK(cudaMemsetAsync(ra.dec, 0, 2 * sizeof(int), c->stream));
    unsigned* bar = c->get<unsigned>("persist.bar", 2);
    int* err = c->get<int>("persist.err", 1);
    CK(cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), c->stream));
    CK(cudaMemsetAsync(err, 0, sizeof(int), c->stream));
    GridBar gb{bar, bar + 1, err};
    if (std::getenv("W1MG_PERSIST_STAMPS")) {
        ra.stamps = c->get<unsigned long long>("rs.stamps", 64 * kRsStampSlots);
        CK(cudaMemsetAsync(ra.stamps, 0, 64 * kRsStampSlots * 8, c->stream));
    }
    SweepArgs a = lv.args;
    const short* ctab = dtab;
    void* args[] = {(void*)&a, (void*)&ra, (void*)&ctab, (void*)&gb};
    CK(cudaLaunchCooperativeKernel((const void*)pdhg_rspf_kernel<Q, P>, dim3(G + 1), dim3(kPfThreads), args,
                                   smem, c->stream));
    ++c->launches;
    int herr = 0;
    CK(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (herr) fail(W1MG_ECUDA, "row-resident PDHG (prime-factor): grid barrier timed out");
    rs_print_stamps(c, ra.stamps, m, G, R, -1);
    return true;
}

template <int Q>
bool launch_pdhg_rs_q(w1mg_ctx* c, const PLevel& lv) {
    const int m = lv.n + 1, h = (m - 1) / 2;
    int R = (m + c->num_sms - 2) / (c->num_sms - 1);  // one SM for the reducer CTA
    if ((m & 1) && h <= 64 && g_pdhg_rs != 2) {
        if (h <= 16) return launch_pdhg_rs_qt<Q, 1>(c, lv, R);
        if (h <= 32) return launch_pdhg_rs_qt<Q, 2>(c, lv, R);
        return launch_pdhg_rs_qt<Q, 4>(c, lv, R);
    }
    // (4: no cluster launches -- ncu cannot replay a cooperative cluster launch)
    if ((m & 1) && h <= kRs2HP && g_pdhg_rs != 2 && g_pdhg_rs != 4 && launch_pdhg_rs2_q<Q>(c, lv)) return true;
    if (m == 513 && g_pdhg_rs != 2 && launch_pdhg_rspf_q<Q, PfGeo<27, 19>>(c, lv)) return true;
    int Rp = 1;
    while (Rp < R) Rp <<= 1;  // the prime-factor transforms split vectors by shifts
    if (Rp > 16) return false;
    return launch_pdhg_rs_qt<Q, 0>(c, lv, Rp);
}

bool launch_pdhg_rs(w1mg_ctx* c, const PLevel& lv, int q) {
    if (!g_pdhg_rs || lv.B != 1) return false;
    if (q == 0) return launch_pdhg_rs_q<0>(c, lv);
    if (q == 1) return launch_pdhg_rs_q<1>(c, lv);
    return launch_pdhg_rs_q<2>(c, lv);
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
    if (g_pdhg_rs && launch_pdhg_rs(c, lv, q)) return;  // one pair: row-resident persistent engine
    if ((g_pdhg_small == 1 && lv.n + 1 <= kPdhgSmallAutoM) ||
        (g_pdhg_small == 2 && lv.n + 1 <= kPdhgSmallMaxM)) {
        if (q == 0) launch_pdhg_small<0>(c, lv);
        else if (q == 1) launch_pdhg_small<1>(c, lv);
        else launch_pdhg_small<2>(c, lv);
        return;
    }
    if (launch_pdhg_persist(c, lv, q)) return;
    constexpr int K = 8;
    if (max_iters < K) {
        for (long k = 0; k < max_iters; ++k) pdhg_iteration(c, lv, q);
        return;
    }
    std::string key(reinterpret_cast<const char*>(&lv.args), sizeof(SweepArgs));
    key += "pdhg:" + std::to_string(q) + ":" + std::to_string(lv.B) + ":dct" +
           std::to_string(lv.rows_f) + "." + std::to_string(lv.cols) + "." + std::to_string(lv.rows_i) + "." +
           std::to_string(lv.rows_p);
    cudaGraphExec_t ex;
    auto it = c->graphs.find(key);
    if (it != c->graphs.end()) {
        ex = it->second;
    } else {
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
        c->launches += (long)(lv.rows_p ? kPdhgLaunches : kPdhgLaunches + 1) * K;
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

int w1mg_pdhg_plan_check(int n1, int n2, long* bad) {
    return guard([&] {
        if (!bad) fail(W1MG_EINVAL, "w1mg_pdhg_plan_check: null output");
        if (n1 != 27 || n2 != 19) fail(W1MG_EINVAL, "w1mg_pdhg_plan_check: factor pair not instantiated");
        using P = w1mg_dev::PfGeo<27, 19>;
        std::vector<short> t(P::NTAB);
        w1mg_dev::rspf_tables<P>(t.data());
        const int m = P::M;
        const short* ginv = t.data();
        const short* idxg = ginv + m;
        const short* crtk = idxg + P::N2 * P::N1P;
        const short* i0k = crtk + P::N1 * P::N2;
        const short* i0d = i0k + P::NI0;
        long b = 0;
        std::vector<int> seen(P::N2 * P::N1P, 0), seenk(m, 0);
        auto pos = [&](int n) { return n <= (m - 1) / 2 ? 2 * n : 2 * (m - 1 - n) + 1; };
        for (int i = 0; i < m; ++i) {
            const int g = ginv[i];
            if (g < 0 || g >= P::N2 * P::N1P || g % P::N1P >= P::N1 || seen[g]++) ++b;
            else if (idxg[g] != i) ++b;
            else {  // x_i sits at v[(N2 n1 + N1 n2) mod m] after Makhoul's reordering
                const int n1i = g % P::N1P, n2i = g / P::N1P;
                if (pos((P::N2 * n1i + P::N1 * n2i) % m) != i) ++b;
            }
        }
        for (int k1 = 0; k1 < P::N1; ++k1)
            for (int k2 = 0; k2 < P::N2; ++k2) {
                const int k = crtk[k1 * P::N2 + k2];
                if (k < 0 || k >= m || k % P::N1 != k1 || k % P::N2 != k2 || seenk[k]++) ++b;
            }
        for (int k1 = 0; k1 < P::H1; ++k1)
            for (int k2 = 0; k2 < P::N2; ++k2) {
                const int it = k1 * P::N2 + k2;
                if (i0k[it] != crtk[it] || i0d[it] != k1 * 2 * P::N2P + k2) ++b;
            }
        *bad = b;
    });
}

}  // extern "C"
