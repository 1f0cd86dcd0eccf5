// capi.cu -- the extern "C" boundary (include/w1mg_cuda.h) and the device
// engine behind it: context, workspace, per-level drivers, CUDA-graph sweep
// loop with device-side convergence, cascade and batched cascade.
//
// Reference call stacks this replaces (paths relative to /root/reference):
//   cp_run           proj/src/solver_cp.cpp:113-147
//   cp_residual      proj/src/solver_cp.cpp:102-111
//   grid operators   proj/src/grid.cpp:45-142
//   ml_run (spec)
#include <cublas_v2.h>
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
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/w1mg_cuda.h"
#include "level_kernels.cuh"
#include "ref_kernels.cuh"
#include "cp2_kernels.cuh"
#include "cluster_kernels.cuh"
#include "cp2w_kernels.cuh"
#include "grid_kernels.cuh"

using namespace w1mg_dev;

namespace {

thread_local std::string g_err;

struct Fail {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw Fail{code, msg}; }

#define CK(expr)                                                                        \
    do {                                                                                \
        cudaError_t e_ = (expr);                                                        \
        if (e_ != cudaSuccess)                                                          \
            fail(e_ == cudaErrorMemoryAllocation ? W1MG_ENOMEM : W1MG_ECUDA,            \
                 std::string(#expr) + ": " + cudaGetErrorString(e_));                  \
    } while (0)

template <class F>
int guard(F&& f) {
    try {
        f();
        return W1MG_OK;
    } catch (const Fail& e) {
        g_err = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return W1MG_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return W1MG_ECUDA;
    }
}

void check_pnorm(int p) {
    if (p < 0 || p > 2) fail(W1MG_ELOGIC, "bad PNorm");
}
void check_n(int n) {
    if (n < 1) fail(W1MG_EINVAL, "GridSpec: cells_per_side must be positive");
}

}  // namespace

// ---------------------------------------------------------------- context
struct w1mg_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    struct Buf {
        void* p = nullptr;
        size_t bytes = 0;
    };
    std::map<std::string, Buf> bufs;
    std::map<std::string, cudaGraphExec_t> graphs;
    int* pinned = nullptr;  // 2 ints for the done-count pipeline
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    std::vector<cudaEvent_t> lev_ev;  // start/end per level of the last cascade
    int lev_count = 0;
    long launches = 0;
    int num_sms = 148;
    void* blas = nullptr;  // cublasHandle_t for the Poisson DCT GEMMs (lazy)

    void* buf(const std::string& name, size_t bytes) {
        Buf& b = bufs[name];
        if (b.bytes < bytes) {
            if (b.p) {
                CK(cudaFree(b.p));
                // any cached graph may hold the old pointer
                for (auto& g : graphs) cudaGraphExecDestroy(g.second);
                graphs.clear();
            }
            b.p = nullptr;
            b.bytes = 0;
            CK(cudaMalloc(&b.p, bytes));
            b.bytes = bytes;
        }
        return b.p;
    }
    template <class T>
    T* get(const std::string& name, size_t count) {
        return static_cast<T*>(buf(name, count * sizeof(T)));
    }
};

namespace {

// ------------------------------------------------------------ level batch
struct Level {
    int n = 0;
    int B = 0;
    Layout L{};
    double* base = nullptr;
    PairCtl* ctl = nullptr;
    unsigned* ticket = nullptr;
    double* partial = nullptr;
    int* ndone = nullptr;
    SweepArgs args{};   // single-sweep engines
    dim3 grid;
    SweepArgs args2{};  // two-sweep engine
    dim3 grid2;
    SweepArgs args2w{};  // two-sweep engine, two column sets per lane
    dim3 grid2w;
    dim3 grid2t;  // two-sweep tensor-map engine (args2 geometry, kWarpsT-warp blocks)
    bool slab = false;  // row slab of a decomposed grid (one-sweep engine only)
    int* act = nullptr;   // [B] running pairs of a compacted launch (null: B == 1 or slab)
    int* nact = nullptr;  // their count
    alignas(64) CUtensorMap tmap{};  // (column, row, plane) view for the tensor-map engine
    bool has_tmap = false;
};

// Tensor map over a whole-grid level: x = column (pitch), y = row (n+1 rows,
// rows beyond are zero-filled), z = pair * NSLOT + slot; box {kChunk, 1, 8} at
// plane stride 2 = one row of PHI_p, MX_p, MY_p, RHO_p for parity p.
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p)
            fail(W1MG_ECUDA, "cuTensorMapEncodeTiled not available");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

void make_level_tmap(Level& lv) {
    const Layout& L = lv.L;
    cuuint64_t dims[3] = {(cuuint64_t)L.pitch, (cuuint64_t)L.n + 1, (cuuint64_t)lv.B * NSLOT};
    cuuint64_t strides[2] = {(cuuint64_t)L.pitch * 8, (cuuint64_t)L.plane * 8};
    cuuint32_t box[3] = {(cuuint32_t)kChunk, 1, 8};
    cuuint32_t estr[3] = {1, 1, 2};
    CUresult r = tmap_encoder()(&lv.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                                lv.base + L.at(0, 0), dims, strides, box, estr,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(W1MG_ECUDA, "cuTensorMapEncodeTiled failed");
    lv.has_tmap = true;
}

// RHO -> RHO2 for every pair of the level (one strided copy).
void mirror_rho(w1mg_ctx* c, const Level& lv) {
    const size_t w = (size_t)lv.L.plane * 8, sp = (size_t)NSLOT * lv.L.plane * 8;
    CK(cudaMemcpy2DAsync(lv.base + RHO2 * lv.L.plane, sp, lv.base + RHO * lv.L.plane, sp, w, lv.B,
                         cudaMemcpyDeviceToDevice, c->stream));
}

// strip-height target: enough strips for this many warps per SM (W1MG_WARPS_PER_SM)
int g_warps_per_sm = 32;

// warps per block of the tensor-map two-sweep kernel (W1MG_TMAP_NW = 2|4|8)
int g_tmap_nw = kWarpsT;

// Strip geometry of the three streaming engines for a launch over `pairs`
// pairs: the tallest strips (<= 64 rows) that still give about 32 warps per
// SM overall, so a grid over few pairs splits each pair finer.
void strip_geometry(SweepArgs& a, int own, long pairs, long target, int hmin) {
    const int nrows = a.jhi - a.jlo;
    a.ncx = (a.L.n + 1 + own - 1) / own;
    int H = 64;
    while (H > hmin) {
        long tiles = pairs * a.ncx * ((nrows + H - 1) / H);
        if (tiles >= target) break;
        H >>= 1;
    }
    a.H = H;
    a.nsy = (nrows + H - 1) / H;
    a.ntiles = a.ncx * a.nsy;
}

void set_geometry(Level& lv, int pairs, int num_sms) {
    const long target = (long)num_sms * g_warps_per_sm;
    strip_geometry(lv.args, kOwn, pairs, target, 2);       // 31 owned columns per warp
    strip_geometry(lv.args2, kOwn2, pairs, target, 4);     // two-sweep: 29 per warp
    strip_geometry(lv.args2w, kOwnW, pairs, target / 2, 4);  // wide: 61 per warp, 4-warp blocks
    lv.grid = dim3((lv.args.ntiles + kSweepWarps - 1) / kSweepWarps, pairs, 1);
    lv.grid2 = dim3((lv.args2.ntiles + kSweepWarps - 1) / kSweepWarps, pairs, 1);
    lv.grid2w = dim3((lv.args2w.ntiles + kWarpsW - 1) / kWarpsW, pairs, 1);
    lv.grid2t = dim3((lv.args2.ntiles + g_tmap_nw - 1) / g_tmap_nw, pairs, 1);
}

// jhi < 0: whole grid.  Otherwise a row slab owning global rows [jlo, jhi),
// stored with one halo row below and two above (Layout::make_slab).
// ext_base: use this buffer (B * NSLOT planes) instead of a context buffer
// (row slabs whose buffer is shared with peers through CUDA IPC).
Level make_level(w1mg_ctx* c, const std::string& tag, int n, int B, double mu, double tau,
                 double* hist, long hist_cap, int jlo = 0, int jhi = -1,
                 double* ext_base = nullptr) {
    Level lv;
    lv.n = n;
    lv.B = B;
    lv.slab = jhi >= 0;
    if (!lv.slab) {
        jlo = 0;
        jhi = n + 1;
    }
    lv.L = lv.slab ? Layout::make_slab(n, jlo - 1, jhi + 2) : Layout::make(n);
    lv.base = ext_base ? ext_base : c->get<double>(tag + ".base", (size_t)B * NSLOT * lv.L.plane);
    lv.ctl = c->get<PairCtl>(tag + ".ctl", B);
    lv.ticket = c->get<unsigned>(tag + ".ticket", B);
    lv.ndone = c->get<int>(tag + ".ndone", 1);

    SweepArgs& a = lv.args;
    a.base = lv.base;
    a.L = lv.L;
    a.jlo = jlo;
    a.jhi = jhi;
    a.red_out = nullptr;
    a.mu = mu;
    a.tau = tau;
    const double h = 1.0 / n;
    a.ih = 1.0 / h;  // inv_h, grid.cpp:48/79
    a.h2 = h * h;    // solver_cp.cpp:25
    a.ctl = lv.ctl;
    a.ticket = lv.ticket;
    a.hist = hist;
    a.hist_cap = hist_cap;
    a.ndone = lv.ndone;
    a.act = nullptr;
    a.nact = nullptr;
    lv.args2 = a;
    lv.args2w = a;
    set_geometry(lv, B, c->num_sms);
    // a compacted launch over fewer pairs uses shorter strips (more tiles per
    // pair), so size the partials for the one-pair geometry
    Level one = lv;
    set_geometry(one, 1, c->num_sms);
    lv.partial = c->get<double>(
        tag + ".partial",
        (size_t)B * std::max<size_t>({(size_t)one.args.ntiles * 3, (size_t)one.args2.ntiles * 6,
                                      (size_t)one.args2w.ntiles * 6, (size_t)lv.args.ntiles * 3,
                                      (size_t)lv.args2.ntiles * 6, (size_t)lv.args2w.ntiles * 6}));
    a.partial = lv.partial;
    lv.args2.partial = lv.partial;
    lv.args2w.partial = lv.partial;
    if (B > 1 && !lv.slab) {
        lv.act = c->get<int>(tag + ".act", B);
        lv.nact = c->get<int>(tag + ".nact", 1);
    }
    if (!lv.slab) make_level_tmap(lv);
    CK(cudaMemsetAsync(lv.ticket, 0, sizeof(unsigned) * B, c->stream));
    return lv;
}

void zero_level(w1mg_ctx* c, const Level& lv) {
    CK(cudaMemsetAsync(lv.base, 0, sizeof(double) * (size_t)lv.B * NSLOT * lv.L.plane, c->stream));
}

double* slot_ptr(const Level& lv, int pair, int slot) {
    return lv.base + ((long)pair * NSLOT + slot) * lv.L.plane;
}

// dense reference-layout host/device array <-> one slot of one pair
void put_nodes(w1mg_ctx* c, const Level& lv, int pair, int slot, const double* src,
               cudaMemcpyKind kind) {
    const int n = lv.n;
    CK(cudaMemcpy2DAsync(slot_ptr(lv, pair, slot) + lv.L.at(0, 0), lv.L.pitch * 8, src,
                         (size_t)(n + 1) * 8, (size_t)(n + 1) * 8, n + 1, kind, c->stream));
}
void put_xedges(w1mg_ctx* c, const Level& lv, int pair, int slot, const double* src,
                cudaMemcpyKind kind) {
    const int n = lv.n;
    CK(cudaMemcpy2DAsync(slot_ptr(lv, pair, slot) + lv.L.at(0, 0), lv.L.pitch * 8, src,
                         (size_t)n * 8, (size_t)n * 8, n + 1, kind, c->stream));
}
void put_yedges(w1mg_ctx* c, const Level& lv, int pair, int slot, const double* src,
                cudaMemcpyKind kind) {
    const int n = lv.n;
    CK(cudaMemcpy2DAsync(slot_ptr(lv, pair, slot) + lv.L.at(0, 0), lv.L.pitch * 8, src,
                         (size_t)(n + 1) * 8, (size_t)(n + 1) * 8, n, kind, c->stream));
}
void get_nodes(w1mg_ctx* c, const Level& lv, int pair, int slot, double* dst) {
    const int n = lv.n;
    CK(cudaMemcpy2DAsync(dst, (size_t)(n + 1) * 8, slot_ptr(lv, pair, slot) + lv.L.at(0, 0),
                         lv.L.pitch * 8, (size_t)(n + 1) * 8, n + 1, cudaMemcpyDefault,
                         c->stream));
}
void get_xedges(w1mg_ctx* c, const Level& lv, int pair, int slot, double* dst) {
    const int n = lv.n;
    CK(cudaMemcpy2DAsync(dst, (size_t)n * 8, slot_ptr(lv, pair, slot) + lv.L.at(0, 0),
                         lv.L.pitch * 8, (size_t)n * 8, n + 1, cudaMemcpyDefault, c->stream));
}
void get_yedges(w1mg_ctx* c, const Level& lv, int pair, int slot, double* dst) {
    const int n = lv.n;
    CK(cudaMemcpy2DAsync(dst, (size_t)(n + 1) * 8, slot_ptr(lv, pair, slot) + lv.L.at(0, 0),
                         lv.L.pitch * 8, (size_t)(n + 1) * 8, n, cudaMemcpyDefault, c->stream));
}

dim3 node_grid(int n, int B, dim3 blk) {
    return dim3((n + 1 + blk.x - 1) / blk.x, (n + 1 + blk.y - 1) / blk.y, B);
}

// compensated per-pair reduction, out[b] = (sum f * s1) * s2
template <class F>
void reduce_pairs(w1mg_ctx* c, F f, int w, int rows, int B, double s1, double s2, double* out) {
    int G = (2 * c->num_sms + B - 1) / B;
    if (G > 64) G = 64;
    if (G > rows) G = rows;
    if (G < 1) G = 1;
    double2* part = c->get<double2>("reduce.partial", (size_t)G * B);
    node_reduce_kernel<F><<<dim3(G, B), kRedThreads, 0, c->stream>>>(f, w, rows, part);
    ++c->launches;
    CK(cudaGetLastError());
    reduce_finish_kernel<<<B, 32, 0, c->stream>>>(part, G, s1, s2, out);
    ++c->launches;
    CK(cudaGetLastError());
}

// engine for the fused sweep (W1MG_SWEEP=ldg|tma|tma2); kTma2 streams two
// sweeps per HBM pass, falling back to the single-sweep TMA kernel for the
// short loops and the stop fix-up
constexpr int kTma2 = 2;
// auto: two-sweep for n >= 96 (faster from 128 up, measured), one-sweep below;
// the two-sweep launches use the tensor-map ring with 4-warp blocks (measured
// 3-14 % faster than the bulk-copy ring for batched 128..512 levels,
// tools/probe.py; profiles/r1_summary.md)
constexpr int kAuto = 3;
int g_sweep_variant = kAuto;

constexpr int kTma2W = 4;  // two-sweep, two column sets per lane (cp2w_kernels.cuh)
constexpr int kTma2T = 5;  // two-sweep, ring fed by one tensor-map box per row

template <int NW, bool U>
void launch_tmap_u(const Level& lv, int pn, int parity, cudaStream_t s) {
    const dim3 blk(NW * 32);
    const int sm = tmap_smem(NW);
    switch (pn) {
        case 0: cp_sweep2_tmap_kernel<0, NW, U><<<lv.grid2t, blk, sm, s>>>(lv.args2, parity, lv.tmap); break;
        case 1: cp_sweep2_tmap_kernel<1, NW, U><<<lv.grid2t, blk, sm, s>>>(lv.args2, parity, lv.tmap); break;
        default: cp_sweep2_tmap_kernel<2, NW, U><<<lv.grid2t, blk, sm, s>>>(lv.args2, parity, lv.tmap); break;
    }
}

// the unrolled march is faster on batches, slower on one big grid (cp2_kernels.cuh)
template <int NW>
void launch_tmap(const Level& lv, int pn, int parity, cudaStream_t s) {
    if (lv.B > 1) launch_tmap_u<NW, true>(lv, pn, parity, s);
    else launch_tmap_u<NW, false>(lv, pn, parity, s);
}

bool two_sweep(const Level& lv) {
    if (lv.slab) return false;  // slabs exchange a one-row halo per sweep
    return g_sweep_variant == kTma2 || g_sweep_variant == kTma2W || g_sweep_variant == kTma2T ||
           (g_sweep_variant == kAuto && lv.n >= 96);
}

void launch_sweep2(const Level& lv, int pn, int parity, cudaStream_t s) {
    if (g_sweep_variant == kTma2T || g_sweep_variant == kAuto) {
        if (!lv.has_tmap) fail(W1MG_ELOGIC, "tensor-map sweep on a level without a map");
        switch (g_tmap_nw) {
            case 2: launch_tmap<2>(lv, pn, parity, s); break;
            case 8: launch_tmap<8>(lv, pn, parity, s); break;
            default: launch_tmap<4>(lv, pn, parity, s); break;
        }
        return;
    }
    if (g_sweep_variant == kTma2W) {
        dim3 blk(kWarpsW * 32);
        switch (pn) {
            case 0: cp_sweep2w_tma_kernel<0><<<lv.grid2w, blk, kTmaSmemW, s>>>(lv.args2w, parity); break;
            case 1: cp_sweep2w_tma_kernel<1><<<lv.grid2w, blk, kTmaSmemW, s>>>(lv.args2w, parity); break;
            default: cp_sweep2w_tma_kernel<2><<<lv.grid2w, blk, kTmaSmemW, s>>>(lv.args2w, parity); break;
        }
        return;
    }
    dim3 blk(kSweepWarps * 32);
    switch (pn) {
        case 0: cp_sweep2_tma_kernel<0><<<lv.grid2, blk, kTmaSmem, s>>>(lv.args2, parity); break;
        case 1: cp_sweep2_tma_kernel<1><<<lv.grid2, blk, kTmaSmem, s>>>(lv.args2, parity); break;
        default: cp_sweep2_tma_kernel<2><<<lv.grid2, blk, kTmaSmem, s>>>(lv.args2, parity); break;
    }
}

void launch_sweep(const Level& lv, int pn, int parity, cudaStream_t s) {
    dim3 blk(kSweepWarps * 32);
    if (g_sweep_variant != kLdg) {
        switch (pn) {
            case 0: cp_sweep_tma_kernel<0><<<lv.grid, blk, kTmaSmem, s>>>(lv.args, parity); break;
            case 1: cp_sweep_tma_kernel<1><<<lv.grid, blk, kTmaSmem, s>>>(lv.args, parity); break;
            default: cp_sweep_tma_kernel<2><<<lv.grid, blk, kTmaSmem, s>>>(lv.args, parity); break;
        }
        return;
    }
    switch (pn) {
        case 0: cp_sweep_kernel<0><<<lv.grid, blk, 0, s>>>(lv.args, parity); break;
        case 1: cp_sweep_kernel<1><<<lv.grid, blk, 0, s>>>(lv.args, parity); break;
        default: cp_sweep_kernel<2><<<lv.grid, blk, 0, s>>>(lv.args, parity); break;
    }
}

// Graph of K sweep launches.  A compacted level (lv.args.act set: the tail of
// a batch, grid over lv.grid.y <= B pairs) first rebuilds the running-pair
// list on device, so the launches only span pairs that can still run.
cudaGraphExec_t sweep_graph(w1mg_ctx* c, const Level& lv, int pn, int K) {
    std::string key(reinterpret_cast<const char*>(&lv.args), sizeof(SweepArgs));
    key += std::to_string(pn) + ":" + std::to_string(K) + ":" + std::to_string(lv.grid.x) + ":" +
           std::to_string(lv.grid.y) + ":" + std::to_string(lv.grid2.x) + ":" +
           std::to_string(lv.grid2w.x) + ":" + std::to_string(lv.grid2t.x) + ":B" +
           std::to_string(lv.B) + ":v" +
           std::to_string(g_sweep_variant);
    auto it = c->graphs.find(key);
    if (it != c->graphs.end()) return it->second;
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    if (lv.args.act)
        compact_active_kernel<<<1, kCompactThreads, 0, c->stream>>>(lv.ctl, lv.B, lv.act, lv.nact);
    for (int k = 0; k < K; ++k) {
        if (two_sweep(lv)) launch_sweep2(lv, pn, k & 1, c->stream);
        else launch_sweep(lv, pn, k & 1, c->stream);
    }
    CK(cudaStreamEndCapture(c->stream, &g));
    cudaGraphExec_t ex;
    CK(cudaGraphInstantiate(&ex, g, 0));
    CK(cudaGraphDestroy(g));
    c->graphs[key] = ex;
    return ex;
}

// Tail compaction (W1MG_COMPACT, default on): once at most half of a batch
// is still running, launch grids span only a power-of-two bucket >= the
// running count, with strips re-split for that many pairs.  Pair results do
// not depend on the launch geometry (each pair's sweep and residual order are
// fixed), so this only removes the early-exit blocks of stopped pairs.
bool g_compact = true;
int g_compact_step = 1 << 30;  // bucket granularity (W1MG_COMPACT_STEP; default: powers of two)

Level compacted(const Level& lv, int pairs, int num_sms) {
    Level b = lv;
    set_geometry(b, pairs, num_sms);
    for (SweepArgs* a : {&b.args, &b.args2, &b.args2w}) {
        a->act = lv.act;
        a->nact = lv.nact;
    }
    return b;
}

// Runs sweeps on every pair of the level until each pair's stop flag is set
// (device-side, solver_cp.cpp:128-136 semantics).  The host only watches a
// done-counter one graph behind, so it never stalls the GPU per iteration.
// level-resident engines (W1MG_RESIDENT): 1 = auto (cluster engine for small
// batches with n <= 128, single-CTA engine for n <= 64 otherwise, cooperative
// grid engine for one pair on an L2-sized level; default), 2 = single-CTA
// engine only, 3 = cluster engine wherever it fits (n <= 256), 4 = grid engine
// for every one-pair level, 0 = off (streaming sweeps only)
int g_resident = 1;

// Cooperative-grid engine (grid_kernels.cuh): one pair, whole level in one
// launch, state in L2.  Only on request (W1MG_RESIDENT=4): measured per sweep
// it costs 7.2 us at 32^2, 7.6 us at 256^2 and 9.7 us at 512^2 (grid barrier
// + L2 round trips of the strip ramps), vs 6.0 / 7.9 us for the streaming
// two-sweep launches of one pair, so auto never picks it.
bool grid_ok(const w1mg_ctx* c, const Level& lv) {
    (void)c;
    return g_resident == 4 && !lv.slab && lv.B == 1;
}

template <int PN>
void launch_grid_pn(w1mg_ctx* c, const Level& lv) {
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, cp_grid_kernel<PN>, kGridWarps * 32, 0));
    if (occ < 1) fail(W1MG_ECUDA, "grid engine: kernel does not fit an SM");
    const int G = c->num_sms * std::min(occ, 2);
    SweepArgs ag = lv.args;
    const long TW = (long)G * kGridWarps;
    const int nrows = ag.jhi - ag.jlo;
    const long per_col = std::max(1L, TW / ag.ncx);
    ag.H = std::max(2, (int)((nrows + per_col - 1) / per_col));
    ag.nsy = (nrows + ag.H - 1) / ag.H;
    ag.ntiles = ag.ncx * ag.nsy;
    double* gp = c->get<double>("grid.partial", (size_t)2 * G * 3);
    void* args[] = {(void*)&ag, (void*)&gp};
    CK(cudaLaunchCooperativeKernel((const void*)cp_grid_kernel<PN>, dim3(G), dim3(kGridWarps * 32),
                                   args, 0, c->stream));
}

template <int PN>
void launch_resident_pn(const Level& lv, cudaStream_t s) {
    static unsigned long long attr = 0;  // per-device: attributes are per device
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (!(attr >> (dev & 63) & 1ull)) {
        CK(cudaFuncSetAttribute(cp_resident_kernel<PN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kResidentMaxBytes));
        attr |= 1ull << (dev & 63);
    }
    cp_resident_kernel<PN><<<lv.B, kResidentThreads, resident_bytes(lv.n), s>>>(lv.args);
}

bool resident_ok(const Level& lv) {
    return (g_resident == 1 || g_resident == 2) && !lv.slab &&
           resident_bytes(lv.n) <= kResidentMaxBytes;
}

// Cluster size for the level-resident cluster engine (0: not used).
// Smallest C whose rows fit the shared-memory budget; with few pairs, grow C
// (up to 16, >= 8 rows per CTA) to spread one pair over more SMs.  Measured
// (tools/engines.py): clusters win for n <= 128 when they spread pairs over
// more SMs (C >= 2); a one-CTA level (big batches, n <= 64) is faster on the
// single-CTA engine, and n = 256 is faster streaming.  g_resident == 3 forces
// the cluster engine wherever it fits (tests).
// PDHG levels with m = n+1 <= 65 run level-resident (pdhg_engine.cuh)
int g_pdhg_small = 1;
// PDHG iterations with symmetry-folded DCTs (pdhg_fold.cuh): 1 = auto (odd
// m >= kFoldMinM), 2 = every odd m, 0 = dense sandwich only
int g_pdhg_fold = 1;

// cluster-size rule (W1MG_CLUSTER_PICK): 1 = fewest node passes per phase
// (default), 0 = powers of two with >= 8 rows per CTA
int g_cluster_pick = 1;

int cluster_size(const Level& lv, int num_sms) {
    if (lv.slab || lv.n > 256 || (g_resident != 1 && g_resident != 3)) return 0;
    int C = 0;
    for (int q = 1; q <= 16; ++q)
        if (cluster_smem_bytes(lv.n, q) <= kClusterSmemBudget && (lv.n + 1) / q >= 2) {
            C = q;
            break;
        }
    if (!C) return 0;
    if (g_cluster_pick == 1) {
        // fewest node passes per phase: each CTA thread handles
        // ceil(rows * (n+1) / threads) nodes one after another, and that
        // serial chain (not the cluster barrier) dominates a sweep; ties go
        // to the smaller cluster
        long best = -1;
        const int C0 = C;
        for (int q = C0; q <= 16; ++q) {
            if ((long)lv.B * q > num_sms || (lv.n + 1) / q < 2) break;
            const long rows = (lv.n + 1 + q - 1) / q;
            const long passes = (rows * (lv.n + 1) + kClusterThreads - 1) / kClusterThreads;
            if (best < 0 || passes < best) {
                best = passes;
                C = q;
            }
        }
    } else {
        while (C * 2 <= 16 && (long)lv.B * C * 2 <= num_sms && (lv.n + 1) / (C * 2) >= 8) C *= 2;
    }
    if (g_resident == 1 && (C == 1 || lv.n > 128)) return 0;
    return C;
}

template <int PN>
bool launch_cluster_pn(const Level& lv, int C, cudaStream_t s) {
    static unsigned long long attr = 0;  // per device
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (!(attr >> (dev & 63) & 1ull)) {
        CK(cudaFuncSetAttribute(cp_cluster_kernel<PN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(kClusterSmemBudget + 1024)));
        CK(cudaFuncSetAttribute(cp_cluster_kernel<PN>,
                                cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        attr |= 1ull << (dev & 63);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(lv.B * C);
    cfg.blockDim = dim3(kClusterThreads);
    cfg.dynamicSmemBytes = cluster_smem_bytes(lv.n, C);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, cp_cluster_kernel<PN>, &cfg) != cudaSuccess ||
        nclusters < 1) {
        cudaGetLastError();
        return false;
    }
    CK(cudaLaunchKernelEx(&cfg, cp_cluster_kernel<PN>, lv.args, C));
    return true;
}

void run_sweeps(w1mg_ctx* c, const Level& lv, int pn, long max_iters) {
    if (max_iters <= 0) return;
    if (grid_ok(c, lv)) {  // whole one-pair level in one cooperative launch
        if (pn == 0) launch_grid_pn<0>(c, lv);
        else if (pn == 1) launch_grid_pn<1>(c, lv);
        else launch_grid_pn<2>(c, lv);
        ++c->launches;
        return;
    }
    if (lv.has_tmap) mirror_rho(c, lv);
    if (const int C = cluster_size(lv, c->num_sms)) {  // whole level in one cluster launch
        bool ok = (pn == 0)   ? launch_cluster_pn<0>(lv, C, c->stream)
                  : (pn == 1) ? launch_cluster_pn<1>(lv, C, c->stream)
                              : launch_cluster_pn<2>(lv, C, c->stream);
        if (ok) {
            ++c->launches;
            return;
        }
    }
    if (resident_ok(lv)) {  // whole level in one launch, stop rule on device
        if (pn == 0) launch_resident_pn<0>(lv, c->stream);
        else if (pn == 1) launch_resident_pn<1>(lv, c->stream);
        else launch_resident_pn<2>(lv, c->stream);
        CK(cudaGetLastError());
        ++c->launches;
        return;
    }
    constexpr int K = 16;
    if (max_iters < K) {
        for (long k = 0; k < max_iters; ++k) launch_sweep(lv, pn, (int)(k & 1), c->stream);
        CK(cudaGetLastError());
        c->launches += max_iters;
        return;
    }
    cudaGraphExec_t ex = sweep_graph(c, lv, pn, K);
    const long per_launch = two_sweep(lv) ? 2 : 1;
    long launched = 0;
    int span = lv.B;  // pairs the current graph's grids cover
    for (long g = 0;; ++g) {
        CK(cudaGraphLaunch(ex, c->stream));
        launched += K * per_launch;
        c->launches += K + (span < lv.B ? 1 : 0);
        CK(cudaMemcpyAsync(c->pinned + (g & 1), lv.ndone, sizeof(int), cudaMemcpyDeviceToHost,
                           c->stream));
        CK(cudaEventRecord(c->ev[g & 1], c->stream));
        if (g > 0) {
            CK(cudaEventSynchronize(c->ev[(g - 1) & 1]));
            const int done = c->pinned[(g - 1) & 1];
            if (done >= lv.B) break;
            // pairs never restart, so B - done bounds the running count of
            // every later graph
            const int running = lv.B - done;
            // bucket: running rounded up to a multiple of g_compact_step
            // (powers of two below it); re-capture when the bucket shrinks
            int b = 1;
            while (b < running && b < g_compact_step) b <<= 1;
            if (running > g_compact_step)
                b = (running + g_compact_step - 1) / g_compact_step * g_compact_step;
            if (g_compact && lv.act && b < span) {
                span = b;
                ex = sweep_graph(c, compacted(lv, span, c->num_sms), pn, K);
            }
        }
        if (launched >= max_iters + K * per_launch) break;  // every pair hit its cap by now
    }
    if (two_sweep(lv)) {
        // replay the first sweep of pairs whose two-sweep launch stopped early
        launch_sweep(lv, pn, -1, c->stream);
        CK(cudaGetLastError());
        ++c->launches;
    }
}

// Per-level control init: tolerance = rel_scale * sum(rho^2) (relative mode,
// computed on device) or abs_tol.
void init_level_ctl(w1mg_ctx* c, const Level& lv, double rel_tol, double abs_tol, long max_it) {
    double* rs = nullptr;
    double rel_scale = 0.0;
    if (rel_tol > 0) {
        rs = c->get<double>("level.rho_sq", lv.B);
        const double h = 1.0 / lv.n;
        reduce_pairs(c, FSlotSq{lv.base, lv.L, RHO}, lv.n + 1, lv.n + 1, lv.B, h * h, 1.0, rs);
        rel_scale = rel_tol * lv.args.tau;  // eps = rel * tau * (h^2 sum rho^2)
    }
    init_ctl_kernel<<<(lv.B + 127) / 128, 128, 0, c->stream>>>(lv.ctl, lv.B, rs, rel_scale,
                                                                 abs_tol, max_it, lv.ndone);
    ++c->launches;
    CK(cudaGetLastError());
    CK(cudaMemsetAsync(lv.ticket, 0, sizeof(unsigned) * lv.B, c->stream));
}

void level_values(w1mg_ctx* c, const Level& lv, int pn, double* w1, double* dual) {
    const double h = 1.0 / lv.n;
    if (w1) {
        switch (pn) {
            case 0:
                reduce_pairs(c, FPrimal<0>{lv.base, lv.L, lv.ctl}, lv.n + 1, lv.n + 1, lv.B, h, h, w1);
                break;
            case 1:
                reduce_pairs(c, FPrimal<1>{lv.base, lv.L, lv.ctl}, lv.n + 1, lv.n + 1, lv.B, h, h, w1);
                break;
            default:
                reduce_pairs(c, FPrimal<2>{lv.base, lv.L, lv.ctl}, lv.n + 1, lv.n + 1, lv.B, h, h, w1);
                break;
        }
    }
    if (dual) reduce_pairs(c, FDual{lv.base, lv.L, lv.ctl}, lv.n + 1, lv.n + 1, lv.B, h, h, dual);
}

// Sources for every level of a batch from the finest cell images (device).
void build_sources(w1mg_ctx* c, std::vector<Level>& lv, const double* img0, const double* img1,
                   int m) {
    const int levels = (int)lv.size();
    const int B = lv[0].B;
    const double* a = img0;
    const double* b = img1;
    dim3 blk(32, 8);
    double* sa = c->get<double>("src.sa", B);
    double* sb = c->get<double>("src.sb", B);
    double* sm = c->get<double>("src.sm", B);
    for (int l = levels - 1; l >= 0; --l) {
        const Level& L = lv[l];
        const int n = L.n;
        image_to_nodes_kernel<<<node_grid(n, B, blk), blk, 0, c->stream>>>(a, b, L.base, L.L, PHI1, MX1);
        ++c->launches;
        CK(cudaGetLastError());
        reduce_pairs(c, FSlot{L.base, L.L, PHI1}, n + 1, n + 1, B, 1.0, 1.0, sa);
        reduce_pairs(c, FSlot{L.base, L.L, MX1}, n + 1, n + 1, B, 1.0, 1.0, sb);
        const double h = 1.0 / n;
        make_source_kernel<<<node_grid(n, B, blk), blk, 0, c->stream>>>(L.base, L.L, PHI1, MX1, sa, sb, h * h);
        ++c->launches;
        CK(cudaGetLastError());
        reduce_pairs(c, FSlot{L.base, L.L, RHO}, n + 1, n + 1, B, 1.0, 1.0, sm);
        center_source_kernel<<<node_grid(n, B, blk), blk, 0, c->stream>>>(L.base, L.L, sm, PHI1, MX1);
        ++c->launches;
        CK(cudaGetLastError());
        if (l > 0) {
            const int mc = n / 2;
            double* ca = c->get<double>("src.img0." + std::to_string(l - 1), (size_t)B * mc * mc);
            double* cb = c->get<double>("src.img1." + std::to_string(l - 1), (size_t)B * mc * mc);
            long total = (long)B * mc * mc;
            int nb = (int)std::min<long>((total + 255) / 256, 65535L * 4);
            block_sum_kernel<<<nb, 256, 0, c->stream>>>(a, ca, n, B);
            ++c->launches;
            block_sum_kernel<<<nb, 256, 0, c->stream>>>(b, cb, n, B);
            ++c->launches;
            CK(cudaGetLastError());
            a = ca;
            b = cb;
        }
    }
    (void)m;
}

// device time of each level of the last cascade (waits for it to finish)
void level_seconds(w1mg_ctx* c, std::vector<double>& out) {
    out.clear();
    if (c->lev_count == 0) return;
    CK(cudaEventSynchronize(c->lev_ev[2 * c->lev_count - 1]));
    for (int l = 0; l < c->lev_count; ++l) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->lev_ev[2 * l], c->lev_ev[2 * l + 1]));
        out.push_back(ms * 1e-3);
    }
}

// Cascade over prepared levels (sources in RHO, level 0 zero state).
void run_cascade(w1mg_ctx* c, std::vector<Level>& lv, const w1mg_ml_params& p, long* iters_dev,
                 double* fpr_dev, double* tol_dev, std::vector<double>* secs) {
    const int levels = (int)lv.size();
    dim3 blk(32, 8);
    while ((int)c->lev_ev.size() < 2 * levels) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        c->lev_ev.push_back(e);
    }
    c->lev_count = levels;
    for (int l = 0; l < levels; ++l) {
        Level& L = lv[l];
        if (l > 0) {
            prolong_kernel<<<node_grid(L.n, L.B, blk), blk, 0, c->stream>>>(
                lv[l - 1].base, lv[l - 1].L, lv[l - 1].ctl, L.base, L.L);
                ++c->launches;
            CK(cudaGetLastError());
        }
        const double abs_tol = (p.rel_tol > 0 || !p.eps) ? 0.0 : p.eps[l];
        CK(cudaEventRecord(c->lev_ev[2 * l], c->stream));
        init_level_ctl(c, L, p.rel_tol, abs_tol, p.max_iters);
        run_sweeps(c, L, p.pnorm, p.max_iters);
        CK(cudaEventRecord(c->lev_ev[2 * l + 1], c->stream));
        harvest_kernel<<<(L.B + 127) / 128, 128, 0, c->stream>>>(L.ctl, L.B, l, levels, iters_dev,
                                                                   fpr_dev, tol_dev);
        ++c->launches;
        CK(cudaGetLastError());
    }
    if (secs) level_seconds(c, *secs);
}

std::vector<Level> make_levels(w1mg_ctx* c, const std::string& tag, int n_finest, int levels,
                               int B, int step_mode, double* hist, long hist_cap) {
    if (levels < 1) fail(W1MG_EINVAL, "levels must be >= 1");
    if (n_finest % (1 << (levels - 1)) != 0)
        fail(W1MG_EINVAL, "make_schedule: N must be divisible by 2^(L-1)");
    std::vector<Level> lv;
    for (int l = 0; l < levels; ++l) {
        const int n = n_finest >> (levels - 1 - l);
        const double step = w1mg_cp_step_size(n, step_mode);
        const bool fin = (l == levels - 1);
        lv.push_back(make_level(c, tag + std::to_string(l), n, B, step, step, fin ? hist : nullptr,
                                fin ? hist_cap : 0));
    }
    return lv;
}

void check_ml(const w1mg_ml_params* p) {
    if (!p) fail(W1MG_EINVAL, "null parameters");
    check_pnorm(p->pnorm);
    if (p->rel_tol <= 0 && !p->eps) fail(W1MG_EINVAL, "tolerances: need rel_tol > 0 or eps");
}

}  // namespace

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
            g_sweep_variant = (std::string(v) == "ldg") ? kLdg
                              : (std::string(v) == "tma") ? kTma
                              : (std::string(v) == "tma2") ? kTma2
                              : (std::string(v) == "tma2w") ? kTma2W
                              : (std::string(v) == "tma2t") ? kTma2T
                                                            : kAuto;
        if (const char* v = std::getenv("W1MG_RESIDENT")) g_resident = std::atoi(v);
        if (const char* v = std::getenv("W1MG_COMPACT")) g_compact = std::atoi(v) != 0;
        if (const char* v = std::getenv("W1MG_CLUSTER_PICK")) g_cluster_pick = std::atoi(v);
        if (const char* v = std::getenv("W1MG_PDHG_SMALL")) g_pdhg_small = std::atoi(v);
        if (const char* v = std::getenv("W1MG_PDHG_FOLD")) g_pdhg_fold = std::atoi(v);
        if (const char* v = std::getenv("W1MG_WARPS_PER_SM")) g_warps_per_sm = std::max(1, std::atoi(v));
        if (const char* v = std::getenv("W1MG_COMPACT_STEP")) g_compact_step = std::max(1, std::atoi(v));
        if (const char* v = std::getenv("W1MG_TMAP_NW")) {
            const int w = std::atoi(v);
            g_tmap_nw = (w == 2 || w == 8) ? w : kWarpsT;
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
    if (c->blas) cublasDestroy(static_cast<cublasHandle_t>(c->blas));
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
    if (engine < kLdg || engine > kTma2T) return W1MG_EINVAL;
    g_sweep_variant = engine;
    return W1MG_OK;
}

int w1mg_set_resident_engine(int on) {
    g_resident = (on >= 0 && on <= 4) ? on : 1;
    return W1MG_OK;
}

int w1mg_set_option(const char* name, long value) {
    if (!name) return W1MG_EINVAL;
    const std::string k(name);
    const int v = (int)value;
    if (k == "pdhg_fold" && v >= 0 && v <= 2) g_pdhg_fold = v;
    else if (k == "pdhg_small" && v >= 0 && v <= 2) g_pdhg_small = v;
    else if (k == "cluster_pick" && (v == 0 || v == 1)) g_cluster_pick = v;
    else if (k == "compact") g_compact = v != 0;
    else if (k == "compact_step" && v >= 1) g_compact_step = v;
    else if (k == "warps_per_sm" && v >= 1) g_warps_per_sm = v;
    else if (k == "tmap_nw" && (v == 2 || v == 4 || v == 8)) g_tmap_nw = v;
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
        const int per = two_sweep(lv) ? 2 : 1;
        auto one = [&](long k) {
            if (per == 2) launch_sweep2(lv, pnorm, (int)(k & 1), c->stream);
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

}  // extern "C"

#include "pdhg_engine.cuh"
#include "slab_engine.cuh"
