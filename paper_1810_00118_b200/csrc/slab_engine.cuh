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
// Transports:
//   * peer (default): the exchange is fused into the sweep.  The rows a
//     neighbour needs are stored straight into its halo rows by the warps
//     that compute them (row_update, peer pointers), and the last block posts
//     the slab's three sums into every rank's mailbox and bumps every rank's
//     arrival counter (system-scope fence + atomic).  A one-thread finalize
//     kernel then waits for the world's arrivals of this sweep, reduces the
//     mailbox in rank order and applies the stop rule -- no copies, no
//     collectives.  Emulated on one device the peers are the other slabs;
//     across processes (one GPU each) the level buffers, mailboxes and
//     counters live in one IPC-shared arena per rank
//     (w1mg_slab_comm_enable_peer) and the stores travel over NVLink.
//   * copies / nccl: emulated slabs exchange halos with device copies; a
//     communicator without peer memory uses ncclSend/ncclRecv for the halos
//     and an ncclAllReduce of the three sums (the collective baseline).
// Both run on the context stream and are captured in one CUDA graph per 16
// sweeps.
#pragma once

#include <nccl.h>

#include <chrono>
#include <thread>

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

// Peer transport: wait until every rank has posted sweep `it` (arrivals
// counted since `base`), reduce the mailbox in rank order, stop rule for every
// local slab.  A peer that never arrives (dead process) trips the time bound:
// every local slab is stopped with nonfinite = 2 and the host fails loudly.
__global__ void slab_peer_finalize_kernel(SweepArgs a, PairCtl* ctl_all, int nloc,
                                          const double* mail, unsigned long long* const* arrive_loc,
                                          unsigned long long base, int world, int parity,
                                          int* ndone) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (ctl_all[0].done) return;
    const unsigned long long target = base + (unsigned long long)world * (ctl_all[0].it + 1);
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int q = 0; q < nloc; ++q) {
        const volatile unsigned long long* cnt = arrive_loc[q];
        while (*cnt < target) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > 30ull * 1000000000ull) {  // 30 s without the peers
                for (int r = 0; r < nloc; ++r) {
                    ctl_all[r].nonfinite = 2;
                    ctl_all[r].done = 1;
                }
                atomicAdd(ndone, 1);
                return;
            }
            __nanosleep(64);
        }
    }
    __threadfence_system();
    const volatile double* mb = mail + (long)parity * world * 3;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int r = 0; r < world; ++r) {
        s0 += mb[r * 3 + 0];
        s1 += mb[r * 3 + 1];
        s2 += mb[r * 3 + 2];
    }
    for (int r = 0; r < nloc; ++r) {
        SweepArgs b = a;
        b.ctl = ctl_all + r;
        b.ndone = (r == 0) ? ndone : nullptr;
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
    // peer transport (w1mg_slab_comm_enable_peer): one IPC-shared arena per
    // rank = [level buffer of its slab][mailbox 2 x world x 3][arrival counter]
    int peer_n = 0;                     // grid the arena is laid out for (0: no peer memory)
    void* arena = nullptr;              // mine
    std::vector<char*> peer_arena;      // every rank's arena in my address space
    std::vector<size_t> mail_off;       // per rank: mailbox offset in its arena
    double** mail_ptrs = nullptr;       // device array [world]
    unsigned long long** arrive_ptrs = nullptr;  // device array [world]
    unsigned long long arrive_base = 0; // arrivals counted on my counter so far
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
    // peer transport
    bool peer = false;
    const double* mail = nullptr;              // my (first local slab's) mailbox
    unsigned long long** arrive_loc = nullptr; // device array [nloc]: local counters
    unsigned long long base = 0;               // arrivals before this run
};

// emulated-slab transport: 1 = fused peer stores (default), 0 = device copies
int g_slab_peer = 1;

Layout slab_layout(int n, const std::vector<int>& b, int r) {
    return Layout::make_slab(n, b[r] - 1, b[r + 1] + 2);
}

size_t align256(size_t x) { return (x + 255) / 256 * 256; }

void check_nccl(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(W1MG_ECUDA, std::string("NCCL ") + what + ": " + ncclGetErrorString(r));
}

// Host wait on an event of the context stream.  With a communicator the
// wait polls ncclCommGetAsyncError: a failed or dead peer (network error,
// remote abort) aborts the communicator and fails loudly instead of hanging
// the host in cudaEventSynchronize.
void wait_event_comm(cudaEvent_t e, w1mg_slab_comm* comm) {
    if (!comm || !comm->comm) {
        CK(cudaEventSynchronize(e));
        return;
    }
    for (;;) {
        const cudaError_t q = cudaEventQuery(e);
        if (q == cudaSuccess) return;
        if (q != cudaErrorNotReady) CK(q);
        ncclResult_t ar = ncclSuccess;
        check_nccl(ncclCommGetAsyncError(comm->comm, &ar), "async error query");
        if (ar != ncclSuccess && ar != ncclInProgress) {
            ncclCommAbort(comm->comm);
            comm->comm = nullptr;
            fail(W1MG_ECUDA, std::string("NCCL asynchronous error: ") + ncclGetErrorString(ar));
        }
        std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
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
    // peer transport where this rank's arena is laid out for this grid size;
    // other partitioned levels of a cascade use the NCCL transport
    s.peer = comm ? (comm->peer_n == n) : (g_slab_peer != 0);
    for (int q = 0; q < nloc; ++q) {
        const int r = comm ? comm->rank : q;
        const bool first = comm ? (r == 0) : (q == 0);
        double* ext = (comm && s.peer) ? static_cast<double*>(comm->arena) : nullptr;
        Level lv = make_level(c, tag + std::to_string(r), n, 1, mu, tau, first ? hist : nullptr,
                              first ? hist_cap : 0, s.bounds[r], s.bounds[r + 1], ext);
        lv.ctl = s.ctl + q;
        lv.args.ctl = lv.ctl;
        lv.args2.ctl = lv.ctl;
        lv.args.red_out = s.red + 3 * q;
        lv.ndone = s.ndone;
        lv.args.ndone = nullptr;
        s.lv.push_back(lv);
    }
    if (!s.peer) return s;
    // peer transport wiring: neighbours' buffers, every rank's mailbox/counter
    const int W = s.R;
    std::vector<double*> mails(W);
    std::vector<unsigned long long*> arrives(W);
    std::vector<double*> bases(W, nullptr);
    if (comm) {
        for (int r = 0; r < W; ++r) {
            char* ar = comm->peer_arena[r];
            bases[r] = reinterpret_cast<double*>(ar);
            mails[r] = reinterpret_cast<double*>(ar + comm->mail_off[r]);
            arrives[r] = reinterpret_cast<unsigned long long*>(ar + comm->mail_off[r] +
                                                               align256((size_t)2 * W * 3 * 8));
        }
        s.base = comm->arrive_base;
    } else {
        double* mb = c->get<double>(tag + ".mail", (size_t)W * 2 * W * 3);
        auto* cnt = c->get<unsigned long long>(tag + ".arrive", W);
        CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * W, c->stream));
        for (int r = 0; r < W; ++r) {
            bases[r] = s.lv[r].base;
            mails[r] = mb + (size_t)r * 2 * W * 3;
            arrives[r] = cnt + r;
        }
        s.base = 0;
    }
    double** dmail = comm ? comm->mail_ptrs : c->get<double*>(tag + ".mailp", W);
    unsigned long long** darr = comm ? comm->arrive_ptrs : c->get<unsigned long long*>(tag + ".arrp", W);
    if (!comm) {
        CK(cudaMemcpyAsync(dmail, mails.data(), sizeof(double*) * W, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(darr, arrives.data(), sizeof(void*) * W, cudaMemcpyHostToDevice, c->stream));
    }
    const int me0 = comm ? comm->rank : 0;
    s.mail = mails[me0];
    s.arrive_loc = c->get<unsigned long long*>(tag + ".arrloc", nloc);
    std::vector<unsigned long long*> loc(nloc);
    for (int q = 0; q < nloc; ++q) loc[q] = arrives[comm ? comm->rank : q];
    CK(cudaMemcpyAsync(s.arrive_loc, loc.data(), sizeof(void*) * nloc, cudaMemcpyHostToDevice,
                       c->stream));
    for (int q = 0; q < nloc; ++q) {
        const int r = comm ? comm->rank : q;
        SweepArgs& a = s.lv[q].args;
        a.red_out = nullptr;
        a.mail = dmail;
        a.arrive = darr;
        a.prank = r;
        a.pworld = W;
        a.psys = comm ? 1 : 0;
        if (r + 1 < W) {
            const Layout U = slab_layout(n, s.bounds, r + 1);
            a.up_base = bases[r + 1];
            a.up_plane = U.plane;
            a.up_row0 = U.row0;
        }
        if (r > 0) {
            const Layout D = slab_layout(n, s.bounds, r - 1);
            a.dn_base = bases[r - 1];
            a.dn_plane = D.plane;
            a.dn_row0 = D.row0;
        }
    }
    // the host-side copies above must land before the captured graph runs
    CK(cudaStreamSynchronize(c->stream));
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
    if (s.peer) {  // exchange and sums already posted by the sweeps
        slab_peer_finalize_kernel<<<1, 32, 0, c->stream>>>(s.lv[0].args, s.ctl, (int)s.lv.size(),
                                                          s.mail, s.arrive_loc, s.base, s.R,
                                                          parity, s.ndone);
        CK(cudaGetLastError());
        c->launches += (long)s.lv.size() + 1;
        return;
    }
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
    if (s.comm && s.peer && s.comm->world > 1) {
        // every rank has loaded its slab before any peer stores into it
        double* d = c->get<double>("slab.barrier", 1);
        check_nccl(ncclAllReduce(d, d, 1, ncclDouble, ncclSum, s.comm->comm, c->stream), "barrier");
    }
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
            wait_event_comm(c->ev[(it - 1) & 1], s.comm);
            if (c->pinned[(it - 1) & 1] >= 1) break;
        }
        if (launched >= max_iters + K) break;
    }
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaGraphExecDestroy(ex));
}

// After a run: peer arrivals consumed on my counter, and the time-bound check.
void slab_after_run(SlabSet& s, const PairCtl& hc) {
    if (!s.peer) return;
    if (hc.nonfinite == 2) fail(W1MG_ECUDA, "slab peer transport: a peer did not arrive within 30 s");
    if (s.comm) s.comm->arrive_base += (unsigned long long)s.comm->world * (unsigned long long)hc.it;
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

// After a partitioned level: every slab's owned rows of the latest state
// (phi, m_x, m_y at parity `cur`) back into the whole-grid level F (parity 0,
// F's control block cur = 0) -- on a communicator each rank stores its rows
// and the row blocks are broadcast from their owners (one NCCL group), so
// every rank holds the full level for the next prolongation.
void slab_store_to_level(w1mg_ctx* c, SlabSet& s, Level& F, int cur) {
    const int n = s.n;
    const size_t row_bytes = (size_t)F.L.pitch * 8;
    const int src_slot[3] = {PHI0 + cur, MX0 + cur, MY0 + cur};
    const int dst_slot[3] = {PHI0, MX0, MY0};
    for (auto& lv : s.lv) {
        const int r0 = lv.args.jlo, r1 = std::min(lv.args.jhi, n + 1);
        for (int q = 0; q < 3; ++q)
            CK(cudaMemcpy2DAsync(slot_ptr(F, 0, dst_slot[q]) + F.L.at(0, r0), row_bytes,
                                 slot_ptr(lv, 0, src_slot[q]) + lv.L.at(0, r0), row_bytes,
                                 row_bytes, r1 - r0, cudaMemcpyDeviceToDevice, c->stream));
    }
    if (s.comm && s.comm->world > 1) {
        check_nccl(ncclGroupStart(), "group start");
        for (int r = 0; r < s.comm->world; ++r) {
            const int r0 = s.bounds[r], r1 = std::min(s.bounds[r + 1], n + 1);
            for (int q = 0; q < 3; ++q) {
                double* p = slot_ptr(F, 0, dst_slot[q]) + F.L.at(0, r0);
                check_nccl(ncclBroadcast(p, p, (size_t)(r1 - r0) * F.L.pitch, ncclDouble, r,
                                         s.comm->comm, c->stream),
                           "broadcast level rows");
            }
        }
        check_nccl(ncclGroupEnd(), "group end");
    }
    CK(cudaMemsetAsync(&F.ctl->cur, 0, sizeof(int), c->stream));
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
        // levels 0 .. p0-1 replicated (identical on every rank), p0 .. L-1
        // row-slab partitioned: every level with n >= g_slab_min_n, and the
        // finest in any case
        int p0 = levels - 1;
        while (p0 > 0 && lv[p0 - 1].n >= g_slab_min_n) --p0;
        long* it = c->get<long>("mlsl.iters", levels);
        double* ff = c->get<double>("mlsl.fpr", levels);
        double* tl = c->get<double>("mlsl.tol", levels);
        std::vector<double> secs;
        std::vector<long> hit(levels, 0);
        std::vector<double> hff(levels, 0.0), htl(levels, 0.0), hsec(levels, 0.0);
        if (p0 > 0) {
            std::vector<Level> coarse(lv.begin(), lv.begin() + p0);
            w1mg_ml_params pc = *prm;
            pc.levels = p0;
            run_cascade(c, coarse, pc, it, ff, tl, &secs);
            CK(cudaMemcpyAsync(hit.data(), it, p0 * sizeof(long), cudaMemcpyDeviceToHost, c->stream));
            CK(cudaMemcpyAsync(hff.data(), ff, p0 * 8, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaMemcpyAsync(htl.data(), tl, p0 * 8, cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
            for (int l = 0; l < p0; ++l) hsec[l] = secs[l];
        }
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        SlabSet s;
        PairCtl hc{};
        double tol = 0.0;
        float ms = 0.f;
        dim3 blk(32, 8);
        for (int l = p0; l < levels; ++l) {
            Level& F = lv[l];
            if (l > 0) {  // prolong the (whole, gathered) coarser level into F
                prolong_kernel<<<node_grid(F.n, 1, blk), blk, 0, c->stream>>>(
                    lv[l - 1].base, lv[l - 1].L, lv[l - 1].ctl, F.base, F.L);
                ++c->launches;
                CK(cudaGetLastError());
            }
            tol = (prm->rel_tol > 0 || !prm->eps) ? 0.0 : prm->eps[l];
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
            s = make_slabs(c, "mlsl.slab" + std::to_string(l), F.n, nslabs, comm, step, step,
                           nullptr, 0);
            slab_load_from_level(c, s, F);
            CK(cudaEventRecord(e0, c->stream));
            slab_run(c, s, prm->pnorm, tol, prm->max_iters);
            CK(cudaEventRecord(e1, c->stream));
            CK(cudaMemcpyAsync(&hc, s.ctl, sizeof(PairCtl), cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
            slab_after_run(s, hc);
            CK(cudaEventElapsedTime(&ms, e0, e1));
            hit[l] = hc.it;
            hff[l] = hc.fpr;
            htl[l] = tol;
            hsec[l] = ms * 1e-3;
            if (l + 1 < levels) slab_store_to_level(c, s, F, hc.cur);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        Level& F = lv.back();
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
        long total = 0;
        double tsec = 0.0;
        for (int l = 0; l < levels; ++l) {
            total += hit[l];
            tsec += hsec[l];
            if (stats) stats[l] = {1.0 / lv[l].n, htl[l], hit[l], hff[l], hsec[l]};
        }
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
    for (int r = 0; r < (int)s->peer_arena.size(); ++r)
        if (r != s->rank && s->peer_arena[r]) cudaIpcCloseMemHandle(s->peer_arena[r]);
    if (s->arena) cudaFree(s->arena);
    if (s->mail_ptrs) cudaFree(s->mail_ptrs);
    if (s->arrive_ptrs) cudaFree(s->arrive_ptrs);
    if (s->comm) ncclCommDestroy(s->comm);
    delete s;
}

// Peer transport for a multi-process slab decomposition of an n-cell grid:
// allocate this rank's arena (its slab's level buffer, mailbox, arrival
// counter), exchange CUDA IPC handles over the communicator (ncclAllGather)
// and map every other rank's arena (NVLink peer access).  Collective over the
// communicator.  Afterwards slab runs on this comm with grid n use the fused
// peer transport instead of NCCL send/recv + all-reduce.
int w1mg_slab_comm_enable_peer(w1mg_ctx* c, w1mg_slab_comm* s, int n) {
    return guard([&] {
        check_n(n);
        if (!s) fail(W1MG_EINVAL, "null comm");
        if (s->peer_n) fail(W1MG_ELOGIC, "peer memory already enabled on this comm");
        CK(cudaSetDevice(c->device));
        const int R = s->world;
        const std::vector<int> b = slab_bounds(n, R);
        for (int r = 1; r <= R; ++r)
            if (b[r] - b[r - 1] < 2) fail(W1MG_EINVAL, "slab decomposition: fewer than 2 rows per slab");
        s->mail_off.resize(R);
        for (int r = 0; r < R; ++r)
            s->mail_off[r] = align256((size_t)NSLOT * slab_layout(n, b, r).plane * 8);
        const size_t bytes = s->mail_off[s->rank] + align256((size_t)2 * R * 3 * 8) + 256;
        CK(cudaMalloc(&s->arena, bytes));
        CK(cudaMemset(s->arena, 0, bytes));
        s->peer_arena.assign(R, nullptr);
        s->peer_arena[s->rank] = static_cast<char*>(s->arena);
        if (R > 1) {
            cudaIpcMemHandle_t mine;
            CK(cudaIpcGetMemHandle(&mine, s->arena));
            char* dh = nullptr;
            CK(cudaMalloc(&dh, sizeof(cudaIpcMemHandle_t) * R));
            CK(cudaMemcpy(dh + sizeof(cudaIpcMemHandle_t) * s->rank, &mine, sizeof(mine),
                          cudaMemcpyHostToDevice));
            check_nccl(ncclAllGather(dh + sizeof(cudaIpcMemHandle_t) * s->rank, dh,
                                     sizeof(cudaIpcMemHandle_t), ncclChar, s->comm, c->stream),
                       "allgather IPC handles");
            std::vector<cudaIpcMemHandle_t> all(R);
            CK(cudaMemcpyAsync(all.data(), dh, sizeof(cudaIpcMemHandle_t) * R, cudaMemcpyDeviceToHost,
                               c->stream));
            CK(cudaStreamSynchronize(c->stream));
            CK(cudaFree(dh));
            for (int r = 0; r < R; ++r) {
                if (r == s->rank) continue;
                void* p = nullptr;
                CK(cudaIpcOpenMemHandle(&p, all[r], cudaIpcMemLazyEnablePeerAccess));
                s->peer_arena[r] = static_cast<char*>(p);
            }
        }
        std::vector<double*> mails(R);
        std::vector<unsigned long long*> arr(R);
        for (int r = 0; r < R; ++r) {
            mails[r] = reinterpret_cast<double*>(s->peer_arena[r] + s->mail_off[r]);
            arr[r] = reinterpret_cast<unsigned long long*>(s->peer_arena[r] + s->mail_off[r] +
                                                          align256((size_t)2 * R * 3 * 8));
        }
        CK(cudaMalloc(&s->mail_ptrs, sizeof(double*) * R));
        CK(cudaMalloc(&s->arrive_ptrs, sizeof(void*) * R));
        CK(cudaMemcpy(s->mail_ptrs, mails.data(), sizeof(double*) * R, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(s->arrive_ptrs, arr.data(), sizeof(void*) * R, cudaMemcpyHostToDevice));
        s->arrive_base = 0;
        s->peer_n = n;
    });
}

// Transport of emulated slabs (comm == NULL): 1 = fused peer stores
// (default), 0 = device-copy halos + host-ordered reduction.
int w1mg_set_slab_transport(int peer) {
    g_slab_peer = peer ? 1 : 0;
    return W1MG_OK;
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
        slab_after_run(s, hc);
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
