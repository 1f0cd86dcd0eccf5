// slab_engine.cuh -- row-slab decomposition of one grid (BASELINE config 5).
// Included at the end of capi.cu (same translation unit).
//
// A grid of n cells is cut into R contiguous row slabs [jlo_r, jhi_r).  Slab r
// stores its rows plus one halo row below (jlo-1: phi, m_x, m_y of the lower
// neighbour, needed by the strip-start recompute of the fused sweep) and one
// above (jhi: phi of the upper neighbour, needed by the m-update of row
// jhi-1).  One iteration is
//   1. the fused one-sweep kernel on every slab (slab mode: each slab's last
//      block publishes its three residual sums instead of deciding the stop),
//   2. the halo exchange of the freshly written buffer: row jhi-1 (phi, m_x,
//      m_y) up, row jlo (phi) down -- <= 4 rows x (n+1) x 8 B per slab,
//   3. the cross-slab sum of the residual sums and the stop rule
//      (slab_finalize_kernel, identical on every slab).
// Because every node is updated by the same arithmetic as on the whole grid,
// fields are bit-identical to the undecomposed solve; only the residual sum is
// reassociated.
//
// Transports: `emulated` keeps all slabs on one device and exchanges halos
// with device copies (used by the parity tests on a single B200); `nccl` runs
// one slab per rank (one process per GPU) with ncclSend/ncclRecv for the
// halos and an ncclAllReduce of the three sums, all on the context stream and
// captured in the same CUDA graph as the sweeps.
#pragma once

#include <nccl.h>

namespace w1mg_dev {

// sums[k] = sum_r red[r*3+k] (r in order), then the stop rule for every slab
// control block (identical updates).  With nred == 1 `red` already holds the
// global sums (NCCL all-reduce result).
__global__ void slab_finalize_kernel(SweepArgs a, PairCtl* ctl_all, int nslab, const double* red,
                                     int nred, int parity, int* ndone) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (ctl_all[0].done) return;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int r = 0; r < nred; ++r) {
        s0 += red[r * 3 + 0];
        s1 += red[r * 3 + 1];
        s2 += red[r * 3 + 2];
    }
    for (int r = 0; r < nslab; ++r) {
        SweepArgs b = a;
        b.ctl = ctl_all + r;
        b.ndone = (r == 0) ? ndone : nullptr;  // the host watches one counter
        if (r > 0) b.hist = nullptr;
        finalize_pair<false>(b, 0, parity, s0, s1, s2);
    }
}

// ||m(x)||_p over the owned rows of a slab (row index offset by jlo)
template <int PN>
struct FSlabPrimal {
    const double* base;
    Layout L;
    const PairCtl* ctl;
    int jlo;
    __device__ double operator()(int, int i, int jj) const {
        const int j = jj + jlo;
        const int c = ctl->cur;
        const double x = (i < L.n) ? base[(MX0 + c) * L.plane + L.at(i, j)] : 0.0;
        const double y = (j < L.n) ? base[(MY0 + c) * L.plane + L.at(i, j)] : 0.0;
        return vec_norm<PN>(x, y);
    }
};

struct FSlabDual {
    const double* base;
    Layout L;
    const PairCtl* ctl;
    int jlo;
    __device__ double operator()(int, int i, int jj) const {
        const int j = jj + jlo;
        const long o = L.at(i, j);
        return base[(PHI0 + ctl->cur) * L.plane + o] * base[RHO * L.plane + o];
    }
};

}  // namespace w1mg_dev

struct w1mg_slab_comm {
    ncclComm_t comm = nullptr;
    int rank = 0;
    int world = 1;
};

namespace {

// Balanced contiguous row ranges of rows 0..n over R slabs.
std::vector<int> slab_bounds(int n, int R) {
    std::vector<int> b(R + 1);
    for (int r = 0; r <= R; ++r) b[r] = (int)((long)(n + 1) * r / R);
    return b;
}

struct SlabSet {
    int n = 0, R = 1;
    std::vector<int> bounds;
    std::vector<Level> lv;   // one per local slab
    PairCtl* ctl = nullptr;  // [R]
    double* red = nullptr;   // [R][3]
    double* sums = nullptr;  // [3] (NCCL all-reduce target)
    int* ndone = nullptr;
    w1mg_slab_comm* comm = nullptr;  // null: emulated on one device
};

void check_nccl(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(W1MG_ECUDA, std::string("NCCL ") + what + ": " + ncclGetErrorString(r));
}

// Emulated: all R slabs local.  NCCL: only slab `comm->rank` of `comm->world`.
SlabSet make_slabs(w1mg_ctx* c, const std::string& tag, int n, int R, w1mg_slab_comm* comm,
                   double mu, double tau, double* hist, long hist_cap) {
    SlabSet s;
    s.n = n;
    s.comm = comm;
    s.R = comm ? comm->world : R;
    s.bounds = slab_bounds(n, s.R);
    for (int r = 1; r <= s.R; ++r)
        if (s.bounds[r] - s.bounds[r - 1] < 2)
            fail(W1MG_EINVAL, "slab decomposition: fewer than 2 rows per slab");
    const int nloc = comm ? 1 : s.R;
    s.ctl = c->get<PairCtl>(tag + ".ctl_all", nloc);
    s.red = c->get<double>(tag + ".red", 3 * nloc);
    s.sums = c->get<double>(tag + ".sums", 3);
    s.ndone = c->get<int>(tag + ".ndone_all", 1);
    for (int q = 0; q < nloc; ++q) {
        const int r = comm ? comm->rank : q;
        const bool first = comm ? (r == 0) : (q == 0);
        Level lv = make_level(c, tag + std::to_string(r), n, 1, mu, tau, first ? hist : nullptr,
                              first ? hist_cap : 0, s.bounds[r], s.bounds[r + 1]);
        lv.ctl = s.ctl + q;
        lv.args.ctl = lv.ctl;
        lv.args2.ctl = lv.ctl;
        lv.args.red_out = s.red + 3 * q;
        lv.ndone = s.ndone;
        lv.args.ndone = nullptr;
        s.lv.push_back(lv);
    }
    return s;
}

// rows [r0, r1) of a dense reference-layout host array into a slab slot
void slab_put(w1mg_ctx* c, const Level& lv, int slot, const double* src, int w, int r0, int r1) {
    if (r1 <= r0) return;
    CK(cudaMemcpy2DAsync(slot_ptr(lv, 0, slot) + lv.L.at(0, r0), lv.L.pitch * 8, src + (long)r0 * w,
                         (size_t)w * 8, (size_t)w * 8, r1 - r0, cudaMemcpyDefault, c->stream));
}
void slab_get(w1mg_ctx* c, const Level& lv, int slot, double* dst, int w, int r0, int r1) {
    if (r1 <= r0) return;
    CK(cudaMemcpy2DAsync(dst + (long)r0 * w, (size_t)w * 8, slot_ptr(lv, 0, slot) + lv.L.at(0, r0),
                         lv.L.pitch * 8, (size_t)w * 8, r1 - r0, cudaMemcpyDefault, c->stream));
}

// Load full-grid initial fields into every local slab: owned rows plus the
// halo rows (which then equal the neighbours' owned values).
void slab_load(w1mg_ctx* c, SlabSet& s, const double* rho, const double* m0x, const double* m0y,
               const double* phi0) {
    const int n = s.n;
    for (auto& lv : s.lv) {
        zero_level(c, lv);
        const int r0 = std::max(lv.args.jlo - 1, 0), r1 = std::min(lv.args.jhi + 1, n + 1);
        slab_put(c, lv, RHO, rho, n + 1, r0, r1);
        if (phi0) slab_put(c, lv, PHI0, phi0, n + 1, r0, r1);
        if (m0x) slab_put(c, lv, MX0, m0x, n, r0, r1);
        if (m0y) slab_put(c, lv, MY0, m0y, n + 1, r0, std::min(r1, n));
    }
}

// Halo exchange of buffer `w` after a sweep.
void slab_exchange(w1mg_ctx* c, SlabSet& s, int w) {
    const size_t row_bytes = (size_t)s.lv[0].L.pitch * 8;
    if (!s.comm) {
        for (int r = 0; r + 1 < s.R; ++r) {
            const Level& lo = s.lv[r];
            const Level& hi = s.lv[r + 1];
            const int up = lo.args.jhi - 1;  // = hi.jlo - 1: lower slab's top row, upper's halo
            const int dn = hi.args.jlo;      // = lo.jhi: upper slab's first row, lower's halo
            for (int slot : {PHI0 + w, MX0 + w, MY0 + w})
                CK(cudaMemcpyAsync(slot_ptr(hi, 0, slot) + hi.L.at(0, up),
                                   slot_ptr(lo, 0, slot) + lo.L.at(0, up), row_bytes,
                                   cudaMemcpyDeviceToDevice, c->stream));
            CK(cudaMemcpyAsync(slot_ptr(lo, 0, PHI0 + w) + lo.L.at(0, dn),
                               slot_ptr(hi, 0, PHI0 + w) + hi.L.at(0, dn), row_bytes,
                               cudaMemcpyDeviceToDevice, c->stream));
        }
        return;
    }
    const Level& lv = s.lv[0];
    const int rank = s.comm->rank, world = s.comm->world;
    const size_t cnt = (size_t)lv.L.pitch;
    check_nccl(ncclGroupStart(), "group start");
    if (rank + 1 < world) {  // my top row up, the upper neighbour's first row down to me
        for (int slot : {PHI0 + w, MX0 + w, MY0 + w})
            check_nccl(ncclSend(slot_ptr(lv, 0, slot) + lv.L.at(0, lv.args.jhi - 1), cnt, ncclDouble,
                                rank + 1, s.comm->comm, c->stream), "send up");
        check_nccl(ncclRecv(slot_ptr(lv, 0, PHI0 + w) + lv.L.at(0, lv.args.jhi), cnt, ncclDouble,
                            rank + 1, s.comm->comm, c->stream), "recv from above");
    }
    if (rank > 0) {
        for (int slot : {PHI0 + w, MX0 + w, MY0 + w})
            check_nccl(ncclRecv(slot_ptr(lv, 0, slot) + lv.L.at(0, lv.args.jlo - 1), cnt, ncclDouble,
                                rank - 1, s.comm->comm, c->stream), "recv from below");
        check_nccl(ncclSend(slot_ptr(lv, 0, PHI0 + w) + lv.L.at(0, lv.args.jlo), cnt, ncclDouble,
                            rank - 1, s.comm->comm, c->stream), "send down");
    }
    check_nccl(ncclGroupEnd(), "group end");
}

void slab_iteration(w1mg_ctx* c, SlabSet& s, int pn, int parity) {
    for (auto& lv : s.lv) launch_sweep(lv, pn, parity, c->stream);
    CK(cudaGetLastError());
    slab_exchange(c, s, 1 - parity);
    const double* red = s.red;
    int nred = (int)s.lv.size();
    if (s.comm) {
        check_nccl(ncclAllReduce(s.red, s.sums, 3, ncclDouble, ncclSum, s.comm->comm, c->stream),
                   "allreduce");
        red = s.sums;
        nred = 1;
    }
    slab_finalize_kernel<<<1, 32, 0, c->stream>>>(s.lv[0].args, s.ctl, (int)s.lv.size(), red, nred,
                                                 parity, s.ndone);
    CK(cudaGetLastError());
    c->launches += (long)s.lv.size() + 1;
}

void slab_run(w1mg_ctx* c, SlabSet& s, int pn, double tol, long max_iters) {
    const int nloc = (int)s.lv.size();
    init_ctl_kernel<<<1, 32, 0, c->stream>>>(s.ctl, nloc, nullptr, 0.0, tol, max_iters, s.ndone);
    ++c->launches;
    CK(cudaGetLastError());
    for (auto& lv : s.lv) CK(cudaMemsetAsync(lv.ticket, 0, sizeof(unsigned), c->stream));
    if (max_iters <= 0) return;
    constexpr int K = 16;
    if (max_iters < K) {
        for (long k = 0; k < max_iters; ++k) slab_iteration(c, s, pn, (int)(k & 1));
        return;
    }
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    const long before = c->launches;
    for (int k = 0; k < K; ++k) slab_iteration(c, s, pn, k & 1);
    const long per_graph = c->launches - before;
    CK(cudaStreamEndCapture(c->stream, &g));
    cudaGraphExec_t ex;
    CK(cudaGraphInstantiate(&ex, g, 0));
    CK(cudaGraphDestroy(g));
    c->launches = before;
    long launched = 0;
    for (long it = 0;; ++it) {
        CK(cudaGraphLaunch(ex, c->stream));
        launched += K;
        c->launches += per_graph;
        CK(cudaMemcpyAsync(c->pinned + (it & 1), s.ndone, sizeof(int), cudaMemcpyDeviceToHost,
                           c->stream));
        CK(cudaEventRecord(c->ev[it & 1], c->stream));
        if (it > 0) {
            CK(cudaEventSynchronize(c->ev[(it - 1) & 1]));
            if (c->pinned[(it - 1) & 1] >= 1) break;
        }
        if (launched >= max_iters + K) break;
    }
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaGraphExecDestroy(ex));
}

// Device-side load of slab rows from a whole-grid level (buffer 0 of pair 0).
void slab_load_from_level(w1mg_ctx* c, SlabSet& s, const Level& full) {
    const int n = s.n;
    const size_t row_bytes = (size_t)full.L.pitch * 8;
    for (auto& lv : s.lv) {
        zero_level(c, lv);
        const int r0 = std::max(lv.args.jlo - 1, 0), r1 = std::min(lv.args.jhi + 1, n + 1);
        for (int slot : {PHI0, MX0, MY0, RHO})
            CK(cudaMemcpy2DAsync(slot_ptr(lv, 0, slot) + lv.L.at(0, r0), row_bytes,
                                 slot_ptr(full, 0, slot) + full.L.at(0, r0), row_bytes, row_bytes,
                                 r1 - r0, cudaMemcpyDeviceToDevice, c->stream));
    }
}

}  // namespace

extern "C" {

// Cascade for one large grid (config 5): levels 0..L-2 replicated (identical
// on every rank), the finest level row-slab partitioned.  comm == NULL:
// `nslabs` slabs emulated on one device.  Outputs: finest owned rows.
int w1mg_ml_slab_cp_run(w1mg_ctx* c, w1mg_slab_comm* comm, int nslabs, int n_finest,
                        const double* rho_levels, const w1mg_ml_params* prm, double* mx,
                        double* my, double* phi, w1mg_level_stats* stats, w1mg_cp_report* rep) {
    return guard([&] {
        check_n(n_finest);
        check_ml(prm);
        const int levels = prm->levels;
        if (levels < 2) fail(W1MG_EINVAL, "ml_slab: need at least 2 levels");
        std::vector<Level> lv =
            make_levels(c, "mlsl", n_finest, levels, 1, prm->step_mode, nullptr, 0);
        size_t off = 0;
        for (auto& L : lv) {
            zero_level(c, L);
            put_nodes(c, L, 0, RHO, rho_levels + off, cudaMemcpyDefault);
            off += (size_t)(L.n + 1) * (L.n + 1);
        }
        // replicated coarse cascade
        std::vector<Level> coarse(lv.begin(), lv.end() - 1);
        w1mg_ml_params pc = *prm;
        pc.levels = levels - 1;
        long* it = c->get<long>("mlsl.iters", levels);
        double* ff = c->get<double>("mlsl.fpr", levels);
        double* tl = c->get<double>("mlsl.tol", levels);
        std::vector<double> secs;
        run_cascade(c, coarse, pc, it, ff, tl, &secs);
        // finest: prolong into the whole-grid level, then cut into slabs
        Level& F = lv.back();
        dim3 blk(32, 8);
        prolong_kernel<<<node_grid(F.n, 1, blk), blk, 0, c->stream>>>(
            coarse.back().base, coarse.back().L, coarse.back().ctl, F.base, F.L);
        ++c->launches;
        CK(cudaGetLastError());
        double tol = (prm->rel_tol > 0 || !prm->eps) ? 0.0 : prm->eps[levels - 1];
        if (prm->rel_tol > 0) {
            double* rs = c->get<double>("mlsl.rho_sq", 1);
            const double h = 1.0 / F.n;
            reduce_pairs(c, FSlotSq{F.base, F.L, RHO}, F.n + 1, F.n + 1, 1, h * h, 1.0, rs);
            double hrs = 0.0;
            CK(cudaMemcpyAsync(&hrs, rs, 8, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
            tol = (prm->rel_tol * F.args.tau) * hrs;  // as init_ctl_kernel
        }
        const double step = w1mg_cp_step_size(F.n, prm->step_mode);
        SlabSet s = make_slabs(c, "mlsl.slab", F.n, nslabs, comm, step, step, nullptr, 0);
        slab_load_from_level(c, s, F);
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, c->stream));
        slab_run(c, s, prm->pnorm, tol, prm->max_iters);
        CK(cudaEventRecord(e1, c->stream));
        PairCtl hc;
        CK(cudaMemcpyAsync(&hc, s.ctl, sizeof(PairCtl), cudaMemcpyDeviceToHost, c->stream));
        std::vector<long> hit(levels - 1);
        std::vector<double> hff(levels - 1), htl(levels - 1);
        CK(cudaMemcpyAsync(hit.data(), it, (levels - 1) * sizeof(long), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(hff.data(), ff, (levels - 1) * 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(htl.data(), tl, (levels - 1) * 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        // W1 over owned rows (+ sum over ranks)
        double w1 = 0.0, du = 0.0;
        double* vals = c->get<double>("mlsl.vals", 2 * s.lv.size());
        const double h = 1.0 / F.n;
        for (size_t q = 0; q < s.lv.size(); ++q) {
            const Level& L = s.lv[q];
            const int rows = L.args.jhi - L.args.jlo;
            if (prm->pnorm == 0)
                reduce_pairs(c, FSlabPrimal<0>{L.base, L.L, L.ctl, L.args.jlo}, F.n + 1, rows, 1, h, h, vals + 2 * q);
            else if (prm->pnorm == 1)
                reduce_pairs(c, FSlabPrimal<1>{L.base, L.L, L.ctl, L.args.jlo}, F.n + 1, rows, 1, h, h, vals + 2 * q);
            else
                reduce_pairs(c, FSlabPrimal<2>{L.base, L.L, L.ctl, L.args.jlo}, F.n + 1, rows, 1, h, h, vals + 2 * q);
            reduce_pairs(c, FSlabDual{L.base, L.L, L.ctl, L.args.jlo}, F.n + 1, rows, 1, h, h, vals + 2 * q + 1);
            if (mx) slab_get(c, L, MX0 + hc.cur, mx, F.n, L.args.jlo, L.args.jhi);
            if (my) slab_get(c, L, MY0 + hc.cur, my, F.n + 1, L.args.jlo, std::min(L.args.jhi, F.n));
            if (phi) slab_get(c, L, PHI0 + hc.cur, phi, F.n + 1, L.args.jlo, L.args.jhi);
        }
        std::vector<double> hv(2 * s.lv.size());
        CK(cudaMemcpyAsync(hv.data(), vals, hv.size() * 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        for (size_t q = 0; q < s.lv.size(); ++q) {
            w1 += hv[2 * q];
            du += hv[2 * q + 1];
        }
        if (comm) {
            double* d = c->get<double>("mlsl.vals_all", 2);
            double loc[2] = {w1, du};
            CK(cudaMemcpyAsync(d, loc, 16, cudaMemcpyHostToDevice, c->stream));
            check_nccl(ncclAllReduce(d, d, 2, ncclDouble, ncclSum, comm->comm, c->stream), "allreduce W1");
            CK(cudaMemcpyAsync(loc, d, 16, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
            w1 = loc[0];
            du = loc[1];
        }
        long total = hc.it;
        double tsec = ms * 1e-3;
        for (int l = 0; l < levels - 1; ++l) {
            total += hit[l];
            tsec += secs[l];
            if (stats) stats[l] = {1.0 / lv[l].n, htl[l], hit[l], hff[l], secs[l]};
        }
        if (stats) stats[levels - 1] = {1.0 / F.n, tol, hc.it, hc.fpr, ms * 1e-3};
        if (rep) {
            rep->distance = w1;
            rep->dual_value = du;
            rep->iterations = total;
            rep->fpr_final = hc.fpr;
            rep->converged = (hc.fpr < tol) ? 1 : 0;
            rep->seconds = tsec;
        }
    });
}

int w1mg_slab_bounds(int n, int nslabs, int* bounds) {
    return guard([&] {
        check_n(n);
        if (nslabs < 1) fail(W1MG_EINVAL, "nslabs must be >= 1");
        std::vector<int> b = slab_bounds(n, nslabs);
        for (int r = 0; r <= nslabs; ++r) bounds[r] = b[r];
    });
}

int w1mg_nccl_unique_id(unsigned char* id128) {
    return guard([&] {
        ncclUniqueId id;
        check_nccl(ncclGetUniqueId(&id), "unique id");
        static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
        std::memcpy(id128, &id, 128);
    });
}

int w1mg_slab_comm_create(w1mg_ctx* c, int world, int rank, const unsigned char* id128,
                          w1mg_slab_comm** out) {
    return guard([&] {
        if (world < 1 || rank < 0 || rank >= world) fail(W1MG_EINVAL, "bad rank / world size");
        CK(cudaSetDevice(c->device));
        ncclUniqueId id;
        std::memcpy(&id, id128, 128);
        auto* s = new w1mg_slab_comm();
        s->rank = rank;
        s->world = world;
        check_nccl(ncclCommInitRank(&s->comm, world, id, rank), "comm init");
        *out = s;
    });
}

void w1mg_slab_comm_destroy(w1mg_slab_comm* s) {
    if (!s) return;
    if (s->comm) ncclCommDestroy(s->comm);
    delete s;
}

// CP solve of one grid decomposed into row slabs.  comm == NULL: `nslabs`
// slabs emulated on the context's device.  comm != NULL: this rank's slab of
// a comm->world decomposition (inputs are full-grid host arrays; outputs are
// written for the owned rows only, other rows untouched).
int w1mg_slab_cp_run(w1mg_ctx* c, w1mg_slab_comm* comm, int n, int nslabs, const double* rho,
                     const double* m0x, const double* m0y, const double* phi0, int pnorm,
                     double mu, double tau, double tol, long max_iters, double* mx, double* my,
                     double* phi, double* fpr_hist, long hist_cap, w1mg_cp_report* rep) {
    return guard([&] {
        check_n(n);
        check_pnorm(pnorm);
        if (!rho) fail(W1MG_EINVAL, "null rho");
        long cap = (fpr_hist && hist_cap > 0) ? hist_cap : 0;
        double* dh = cap ? c->get<double>("slab.hist", cap) : nullptr;
        SlabSet s = make_slabs(c, "slab", n, nslabs, comm, mu, tau, dh, cap);
        slab_load(c, s, rho, m0x, m0y, phi0);
        CK(cudaEventRecord(c->t0, c->stream));
        slab_run(c, s, pnorm, tol, max_iters);
        CK(cudaEventRecord(c->t1, c->stream));
        PairCtl hc;
        CK(cudaMemcpyAsync(&hc, s.ctl, sizeof(PairCtl), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        // W1 / dual over owned rows, summed over slabs (and ranks)
        double* vals = c->get<double>("slab.vals", 2 * s.lv.size());
        for (size_t q = 0; q < s.lv.size(); ++q) {
            const Level& lv = s.lv[q];
            const int rows = lv.args.jhi - lv.args.jlo;
            const double h = 1.0 / n;
            const double* pb = lv.base;
            if (pnorm == 0)
                reduce_pairs(c, FSlabPrimal<0>{pb, lv.L, lv.ctl, lv.args.jlo}, n + 1, rows, 1, h, h, vals + 2 * q);
            else if (pnorm == 1)
                reduce_pairs(c, FSlabPrimal<1>{pb, lv.L, lv.ctl, lv.args.jlo}, n + 1, rows, 1, h, h, vals + 2 * q);
            else
                reduce_pairs(c, FSlabPrimal<2>{pb, lv.L, lv.ctl, lv.args.jlo}, n + 1, rows, 1, h, h, vals + 2 * q);
            reduce_pairs(c, FSlabDual{pb, lv.L, lv.ctl, lv.args.jlo}, n + 1, rows, 1, h, h, vals + 2 * q + 1);
            if (mx) slab_get(c, lv, MX0 + hc.cur, mx, n, lv.args.jlo, lv.args.jhi);
            if (my) slab_get(c, lv, MY0 + hc.cur, my, n + 1, lv.args.jlo, std::min(lv.args.jhi, n));
            if (phi) slab_get(c, lv, PHI0 + hc.cur, phi, n + 1, lv.args.jlo, lv.args.jhi);
        }
        std::vector<double> hv(2 * s.lv.size());
        CK(cudaMemcpyAsync(hv.data(), vals, hv.size() * 8, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        double w1 = 0.0, du = 0.0;
        for (size_t q = 0; q < s.lv.size(); ++q) {
            w1 += hv[2 * q];
            du += hv[2 * q + 1];
        }
        if (comm) {  // sum the per-rank values
            double* d = c->get<double>("slab.vals_all", 2);
            double loc[2] = {w1, du};
            CK(cudaMemcpyAsync(d, loc, 16, cudaMemcpyHostToDevice, c->stream));
            check_nccl(ncclAllReduce(d, d, 2, ncclDouble, ncclSum, comm->comm, c->stream), "allreduce W1");
            CK(cudaMemcpyAsync(loc, d, 16, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
            w1 = loc[0];
            du = loc[1];
        }
        long nh = std::min(hc.it, cap);
        if (nh > 0 && (!comm || comm->rank == 0))
            CK(cudaMemcpy(fpr_hist, dh, nh * 8, cudaMemcpyDeviceToHost));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->t0, c->t1));
        if (rep) {
            rep->distance = w1;
            rep->dual_value = du;
            rep->iterations = hc.it;
            rep->fpr_final = hc.fpr;
            rep->converged = (hc.it > 0 && hc.fpr < tol) ? 1 : 0;
            rep->seconds = ms * 1e-3;
        }
    });
}

}  // extern "C"
