// level_engine.cuh -- the per-level device engine behind the C-ABI: level
// batches (Level, layout, strip geometry, tensor maps), the sweep engines
// and their selection (streaming one-/two-sweep, tensor-map ring, tail
// compaction, single-CTA / cluster / cooperative-grid level-resident
// engines), the CUDA-graph sweep loop with device-side convergence, and the
// cascade helpers (control init, values, restriction / prolongation).
// Included once, by capi.cu, after host_common.cuh.
#pragma once

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
    dim3 grid2t;  // two-sweep tensor-map engine (args2 geometry, tmap_nw-warp blocks)
    SweepArgs args3{};  // three-sweep tensor-map engine
    dim3 grid3;
    int tmap_nw = kWarpsT;
    bool slab = false;  // row slab of a decomposed grid (one-sweep engine only)
    int* act = nullptr;   // [B] running pairs of a compacted launch (null: B == 1 or slab)
    int* nact = nullptr;  // their count
    alignas(64) CUtensorMap tmap{};  // (column, row, plane) view for the tensor-map engine
    bool has_tmap = false;
};

// Tensor map over a whole-grid level: x = column (pitch), y = row (n+1 rows,
// rows beyond are zero-filled), z = pair * NSLOT + slot; box {kChunk, kBoxRows, 8}
// at plane stride 2 = kBoxRows rows of PHI_p, MX_p, MY_p, RHO_p for parity p.
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
    cuuint32_t box[3] = {(cuuint32_t)kChunk, (cuuint32_t)kBoxRows, 8};
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

// warps per block of the tensor-map two-sweep kernel (W1MG_TMAP_NW = 2|4|8;
// 0 = auto: 8 for a launch over ONE pair of a 384..640 level -- one-pair
// 512^2 level 33.4 -> 30.9 ms, while the 256^2 one is 4 % slower and batches
// prefer 4, measured with tools/gpu/sp_engines.sh and nw.sh -- else 4)
int g_tmap_nw = 0;

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
    lv.grid = dim3((lv.args.ntiles + kSweepWarps - 1) / kSweepWarps, pairs, 1);
    lv.grid2 = dim3((lv.args2.ntiles + kSweepWarps - 1) / kSweepWarps, pairs, 1);
    strip_geometry(lv.args3, kOwn3, pairs, target, 4);     // three-sweep: 27 per warp
    lv.grid3 = dim3((lv.args3.ntiles + kWarps3 - 1) / kWarps3, pairs, 1);
    lv.tmap_nw = g_tmap_nw ? g_tmap_nw : ((pairs == 1 && lv.n >= 384 && lv.n <= 640) ? 8 : kWarpsT);
    lv.grid2t = dim3((lv.args2.ntiles + lv.tmap_nw - 1) / lv.tmap_nw, pairs, 1);
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
    // the branch-free p = 2 shrink (device_common.cuh: shrink2_nb) relies on
    // mu^2 lying inside the fast sqrt range and mu^2 < DBL_MAX: every step
    // size of a grid with n < 2^400 does; refuse (loudly) the rest
    if (!(mu >= 1e-140 && mu <= 1e140))
        fail(W1MG_EINVAL, "shrink: mu outside the supported range [1e-140, 1e140]");
    a.mu = mu;
    a.zt = shrink_zero_threshold(mu);
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
    lv.args3 = a;
    set_geometry(lv, B, c->num_sms);
    // a compacted launch over fewer pairs uses shorter strips (more tiles per
    // pair), so size the partials for the one-pair geometry
    Level one = lv;
    set_geometry(one, 1, c->num_sms);
    lv.partial = c->get<double>(
        tag + ".partial",
        (size_t)B * std::max<size_t>({(size_t)one.args.ntiles * 3, (size_t)one.args2.ntiles * 6,
                                      (size_t)lv.args.ntiles * 3, (size_t)lv.args2.ntiles * 6,
                                      (size_t)one.args3.ntiles * 9, (size_t)lv.args3.ntiles * 9}));
    a.partial = lv.partial;
    lv.args2.partial = lv.partial;
    lv.args3.partial = lv.partial;
    if (!lv.slab) {  // two-level residual reduction of the two-sweep kernels
        const int gs = (one.args2.ntiles + kRedGroup - 1) / kRedGroup + 1;
        double* gp = c->get<double>(tag + ".gpart", (size_t)B * gs * 6);
        unsigned* gt = c->get<unsigned>(tag + ".gticket", (size_t)B * gs);
        CK(cudaMemsetAsync(gt, 0, sizeof(unsigned) * B * gs, c->stream));
        for (SweepArgs* x : {&lv.args2}) {
            x->gpart = gp;
            x->gticket = gt;
            x->gstride = gs;
        }
    }
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

// compensated per-pair reduction, out[b] = (sum f * s1) * s2.  The split of
// a pair's rows over G blocks depends on the row count only, never on the
// batch size, so a pair's sources, W1 and dual value carry the same bits
// whether it is solved alone or inside any batch.
template <class F>
void reduce_pairs(w1mg_ctx* c, F f, int w, int rows, int B, double s1, double s2, double* out) {
    int G = 64;
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
// three sweeps per HBM pass (cp3_kernels.cuh), tensor-map ring; W1MG_SWEEP=tma3
constexpr int kTma3 = 6;
int g_sweep_variant = kAuto;

// engine ids 0 (register-pipelined LDG) and 4 (two column sets per lane) were
// measured slower than the tensor-map engines and removed
constexpr int kTma2T = 5;  // two-sweep, ring fed by one tensor-map box per row

// programmatic dependent launch for the two-sweep kernel (option "pdl"):
// consecutive sweeps of a graph overlap the next launch with the current
// tail (griddepcontrol.wait guards every read of the previous sweep's state)
int g_pdl = 1;

template <class K>
void launch_pdl(K kernel, dim3 grid, dim3 blk, int smem, cudaStream_t s, const SweepArgs& a,
                int parity, const CUtensorMap& tm, int early) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = blk;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = g_pdl ? 1 : 0;
    if (smem > 48 * 1024) {  // opt in once per (kernel, device)
        static std::set<std::pair<const void*, int>> done;
        static std::mutex mu;
        int dev = 0;
        CK(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lk(mu);
        if (done.insert({(const void*)kernel, dev}).second)
            CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    }
    CK(cudaLaunchKernelEx(&cfg, kernel, a, parity, tm, early));
}

// numerics of the streaming sweep kernels (option "fast" / W1MG_FAST): 0 =
// bit-identical to the reference (default), 1 = tolerance mode for p = 2
// (PN = 3: FMA-contracted node arithmetic and the rsqrt shrink of
// device_common.cuh; fields within 1e-9 of the reference at fixed sweeps)
int g_fast = 0;
// CTAs per SM of the tolerance-mode three-sweep kernel: 5 (<= 96 registers,
// default) or 4 (<= 128), option "occ3" (A/B)
int g_occ3 = 5;
int stream_pn(int pn) { return (g_fast && pn == 1) ? 3 : pn; }

template <int NW, bool U>
void launch_tmap_u(const Level& lv, int pn, int parity, cudaStream_t s) {
    pn = stream_pn(pn);
    const dim3 blk(NW * 32);
    const int sm = tmap_smem(NW);
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const long blocks = (long)lv.grid2t.x * lv.grid2t.y;
    // early trigger only when this grid AND the next fit on the GPU together
    // (measured: 256^2 one pair 6.6 -> 5.7 us per sweep; at 512^2 one pair,
    // 581 of 888 slots, the waiting next grid slowed the current one)
    const int early = (g_pdl && 2 * blocks <= (long)nsm * (24 / NW)) ? 1 : 0;
    switch (pn) {
        case 0: launch_pdl(cp_sweep2_tmap_kernel<0, NW, U>, lv.grid2t, blk, sm, s, lv.args2, parity, lv.tmap, early); break;
        case 1: launch_pdl(cp_sweep2_tmap_kernel<1, NW, U>, lv.grid2t, blk, sm, s, lv.args2, parity, lv.tmap, early); break;
        case 3: launch_pdl(cp_sweep2_tmap_kernel<3, NW, U>, lv.grid2t, blk, sm, s, lv.args2, parity, lv.tmap, early); break;
        default: launch_pdl(cp_sweep2_tmap_kernel<2, NW, U>, lv.grid2t, blk, sm, s, lv.args2, parity, lv.tmap, early); break;
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
    return g_sweep_variant == kTma2 || g_sweep_variant == kTma2T ||
           (g_sweep_variant == kAuto && lv.n >= 96);
}
// auto picks it for a one-pair level of 192..384 (one 256^2 pair: 22.4 ->
// 19.7 ms per level) and for batched levels of n >= 384: there the sustained
// run is power-capped, and the third of the HBM bytes it saves buys clock
// (bench A/B on one box, tools/gpu/bench_ab.sh: 512^2 level 11.69 -> 11.25 s
// per step at 1725 vs 1500 MHz; 1.472e11 -> 1.511e11 cell-updates/s with it
// on every level), although in short probes the issue-bound two-sweep
// kernel is as fast or faster (512^2 x256 367 vs 369 us, 256^2 x1024 422 vs
// 386 us per sweep); batched 256^2 and the big one-pair grids stay on two
// sweeps
// In tolerance mode (fewer FP64 instructions per node) the three-sweep pass
// also wins on batched 128^2 / 256^2 levels (fast-mode probe, 1024 pairs:
// 256^2 0.339 vs 0.361 ms, 128^2 0.100 vs 0.114 ms per sweep; 256 pairs of
// 256^2 0.090 vs 0.099 ms), so auto uses it for every batched level n >= 96.
bool three_sweep(const Level& lv) {
    if (lv.slab || !lv.has_tmap || lv.n < 96) return false;
    const int batched_min = g_fast ? 96 : 384;
    return g_sweep_variant == kTma3 ||
           (g_sweep_variant == kAuto && ((lv.B == 1 && lv.n >= 192 && lv.n <= 384) ||
                                         (lv.B > 1 && lv.n >= batched_min)));
}
// sweeps one streaming launch performs on this level
int sweeps_per_launch(const Level& lv) { return three_sweep(lv) ? 3 : two_sweep(lv) ? 2 : 1; }

void launch_sweep3(const Level& lv, int pn, int parity, cudaStream_t s) {
    pn = stream_pn(pn);
    const dim3 blk(kWarps3 * 32);
    const int sm = tmap3_smem(kWarps3);
    const long blocks = (long)lv.grid3.x * lv.grid3.y;
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int early = (g_pdl && 2 * blocks <= (long)nsm * g_occ3) ? 1 : 0;
    switch (pn) {
        case 0: launch_pdl(cp_sweep3_tmap_kernel<0>, lv.grid3, blk, sm, s, lv.args3, parity, lv.tmap, early); break;
        case 1: launch_pdl(cp_sweep3_tmap_kernel<1>, lv.grid3, blk, sm, s, lv.args3, parity, lv.tmap, early); break;
        case 3:
            if (g_occ3 == 4) launch_pdl(cp_sweep3_tmap4_kernel<3>, lv.grid3, blk, sm, s, lv.args3, parity, lv.tmap, early);
            else launch_pdl(cp_sweep3_tmap_kernel<3>, lv.grid3, blk, sm, s, lv.args3, parity, lv.tmap, early);
            break;
        default: launch_pdl(cp_sweep3_tmap_kernel<2>, lv.grid3, blk, sm, s, lv.args3, parity, lv.tmap, early); break;
    }
}

void launch_sweep2(const Level& lv, int pn, int parity, cudaStream_t s) {
    if (g_sweep_variant == kTma2T || g_sweep_variant == kAuto) {
        if (!lv.has_tmap) fail(W1MG_ELOGIC, "tensor-map sweep on a level without a map");
        switch (lv.tmap_nw) {
            case 2: launch_tmap<2>(lv, pn, parity, s); break;
            case 8: launch_tmap<8>(lv, pn, parity, s); break;
            default: launch_tmap<4>(lv, pn, parity, s); break;
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
    switch (stream_pn(pn)) {
        case 0: cp_sweep_tma_kernel<0><<<lv.grid, blk, kTmaSmem, s>>>(lv.args, parity); break;
        case 1: cp_sweep_tma_kernel<1><<<lv.grid, blk, kTmaSmem, s>>>(lv.args, parity); break;
        case 3: cp_sweep_tma_kernel<3><<<lv.grid, blk, kTmaSmem, s>>>(lv.args, parity); break;
        default: cp_sweep_tma_kernel<2><<<lv.grid, blk, kTmaSmem, s>>>(lv.args, parity); break;
    }
}

// Graph of K sweep launches.  A compacted level (lv.args.act set: the tail of
// a batch, grid over lv.grid.y <= B pairs) first rebuilds the running-pair
// list on device, so the launches only span pairs that can still run.
cudaGraphExec_t sweep_graph(w1mg_ctx* c, const Level& lv, int pn, int K) {
    std::string key(reinterpret_cast<const char*>(&lv.args), sizeof(SweepArgs));
    key += std::to_string(pn) + ":" + std::to_string(K) + ":" + std::to_string(lv.grid.x) + ":" +
           std::to_string(lv.grid.y) + ":" + std::to_string(lv.grid2.x) + ":" +
           std::to_string(lv.grid2t.x) + ":" +
           std::to_string(lv.grid3.x) + ":B" +
           std::to_string(lv.B) + ":v" +
           std::to_string(g_sweep_variant) + ":nw" + std::to_string(lv.tmap_nw) + ":pdl" +
           std::to_string(g_pdl) + ":f" + std::to_string(g_fast) + ":o" + std::to_string(g_occ3);
    auto it = c->graphs.find(key);
    if (it != c->graphs.end()) return it->second;
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    if (lv.args.act)
        compact_active_kernel<<<1, kCompactThreads, 0, c->stream>>>(lv.ctl, lv.B, lv.act, lv.nact);
    for (int k = 0; k < K; ++k) {
        if (three_sweep(lv)) launch_sweep3(lv, pn, k & 1, c->stream);
        else if (two_sweep(lv)) launch_sweep2(lv, pn, k & 1, c->stream);
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
// running count, with strips re-split for that many pairs.  Fields never
// depend on the launch geometry (every node's arithmetic is fixed); the
// residual sums are reassociated with the strip split, so a residual within a
// few ulps of the tolerance could stop one sweep apart -- the residual that
// decided a stop is the one recorded (PairCtl::rf), so `converged` is exact.
bool g_compact = true;
int g_compact_step = 1 << 30;  // bucket granularity (W1MG_COMPACT_STEP; default: powers of two)

Level compacted(const Level& lv, int pairs, int num_sms) {
    Level b = lv;
    set_geometry(b, pairs, num_sms);
    for (SweepArgs* a : {&b.args, &b.args2, &b.args3}) {
        a->act = lv.act;
        a->nact = lv.nact;
    }
    return b;
}

// Runs sweeps on every pair of the level until each pair's stop flag is set
// (device-side, solver_cp.cpp:128-136 semantics).  The host only watches a
// done-counter one graph behind, so it never stalls the GPU per iteration.
// level-resident engines (W1MG_RESIDENT): 1 = auto (cluster engine for small
// batches with n <= 128, single-CTA engine for n <= 64 otherwise;
// default), 2 = single-CTA engine only, 3 = cluster engine wherever it fits
// (n <= 256), 0 = off (streaming sweeps only).  (A cooperative-grid engine and
// level-persistent shared-memory tile engines were measured slower than the
// streaming launches for one pair and removed.)
int g_resident = 1;

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
// levels of a config-5 cascade with n >= g_slab_min_n are row-slab
// partitioned (the finest always); option "slab_min_n" / W1MG_SLAB_MIN_N
int g_slab_min_n = 1024;
// one-pair PDHG levels above that run level-persistent (pdhg_persist.cuh:
// all iterations in one cooperative launch): 1 = on (default), 0 = off
int g_pdhg_persist = 1;
// ... row-resident (pdhg_rs.cuh / pdhg_rs2.cuh / pdhg_rspf.cuh) where it fits:
// 0 off, 1 auto (default), 2 the prime-factor transforms of dct_kernels.cuh
// at every size (3 = 1, kept for scripts)
int g_pdhg_rs = 1;

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
    // big batches of 128^2 pairs stream instead: 1024 config-4 pairs, 128^2
    // level 0.93 s per step streaming (three sweeps per pass) vs 1.57 s on
    // 4-CTA clusters (bench A/B, tools/gpu/r2s.sh)
    if (g_resident == 1 && lv.n > 64 && (long)lv.B * C > 2L * num_sms) return 0;
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
    const long per_launch = sweeps_per_launch(lv);
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
    // replay the first sweep(s) of pairs whose multi-sweep launch stopped
    // early (redo = 1 or 2; pairs with redo = 0 exit at once)
    for (long q = 1; q < per_launch; ++q) {
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
