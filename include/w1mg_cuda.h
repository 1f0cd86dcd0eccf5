/*
 * w1mg_cuda.h -- the C-ABI drop-in boundary of the B200-native W1 solver.
 *
 * The reference (/root/reference/proj) is a C++20 library whose entry points
 * are the w1mg:: free functions in proj/include/w1mg/ (grid, prox, solver_cp,
 * poisson, solver_pdhg).  This header is the thin, FFI-friendly layer
 * underneath our source-compatible re-implementation of those headers
 * (include/w1mg/, implemented in
 * paper_1810_00118_b200/csrc/host/w1mg_api.cpp): plain pointers, plain
 * sizes, status codes, no C++ or torch types.  Python (ctypes), Go (cgo),
 * Java (JNI/Panama) or Rust bind it directly; see INTEGRATION.md.
 *
 * Arrays passed by host pointer use the reference layouts
 * (proj/include/w1mg/grid.hpp:30-61), n = cells per side:
 *   scalar (potential phi, source rho)  (n+1)*(n+1)  [j*(n+1)+i]
 *   x-edges m_x                          (n+1)*n      [j*n+i]
 *   y-edges m_y                          n*(n+1)      [j*(n+1)+i]
 * Functions with a _dev suffix take device pointers and leave results on
 * the device.
 *
 * Error convention: every int-returning call returns W1MG_OK (0) or an error
 * code; w1mg_last_error() gives the thread-local message.  W1MG_EINVAL
 * carries the same message text the reference throws as
 * std::invalid_argument (e.g. "SourceField: values do not sum to zero",
 * proj/src/grid.cpp:42), so the C++ shim rethrows the identical exception.
 *
 * Threading: a context is bound to one device and one CUDA stream; use one
 * context per host thread.  Free functions without a context are re-entrant.
 */
#ifndef W1MG_CUDA_H
#define W1MG_CUDA_H

#ifdef __cplusplus
extern "C" {
#endif

#define W1MG_ABI_VERSION 1

/* status codes */
#define W1MG_OK 0
#define W1MG_EINVAL 1    /* std::invalid_argument in the reference            */
#define W1MG_ELOGIC 2    /* std::logic_error ("bad PNorm", pnorm.hpp:29)        */
#define W1MG_ECUDA 3     /* CUDA runtime failure                                */
#define W1MG_ENOMEM 4    /* device allocation failed                            */
#define W1MG_ENONFINITE 5 /* NaN/Inf residual detected on device                */

/* PNorm, same order as enum class PNorm {p1, p2, pinf} (pnorm.hpp:20) */
#define W1MG_P1 0
#define W1MG_P2 1
#define W1MG_PINF 2

/* StepMode (report.hpp:10-13) */
#define W1MG_STEP_SAFE 0
#define W1MG_STEP_PRACTICAL 1

typedef struct w1mg_ctx w1mg_ctx;

/* Result of one cp_run (report.hpp:22-41 without the fields). */
typedef struct w1mg_cp_report {
    double distance;   /* primal value sum ||m(x)||_p h^2 (grid.cpp:132-138)       */
    double dual_value; /* <phi, rho>_h (grid.cpp:140-142); ~ -W1 for CP             */
    int converged;     /* fpr < tol reached before max_iters                        */
    long iterations;   /* sweeps performed                                           */
    double fpr_final;  /* residual of the last sweep (solver_cp.cpp:70)              */
    double seconds;    /* device time of the iteration loop (CUDA events)           */
} w1mg_cp_report;

/* LevelStats (report.hpp:22-28) */
typedef struct w1mg_level_stats {
    double h;
    double eps;
    long iters;
    double fpr_final;
    double seconds;
} w1mg_level_stats;

/* Cascade parameters.  Per-level tolerance:
 *   rel_tol > 0 : eps_l = rel_tol * tau_l * ||rho_l||^2_L2  (= rel_tol * R_cold,l,
 *                 the exact first-sweep residual from the zero state)
 *   otherwise   : eps_l = eps[l] (absolute, e.g. from w1mg_make_schedule)   */
typedef struct w1mg_ml_params {
    int levels;        /* L >= 1; level 0 is the coarsest                      */
    int pnorm;         /* W1MG_P1 / W1MG_P2 / W1MG_PINF                        */
    int step_mode;     /* W1MG_STEP_SAFE / W1MG_STEP_PRACTICAL                 */
    double rel_tol;    /* see above                                            */
    const double* eps; /* levels entries, used when rel_tol <= 0              */
    long max_iters;    /* per level                                            */
} w1mg_ml_params;

/* ---------------------------------------------------------------- context */
/* A context owns one stream, its device buffers, cached CUDA graphs and the
 * Poisson DCT plans of one device.  It is not thread-safe: use one per host
 * thread.  w1mg_ctx_create makes `device` current on the calling thread;
 * later calls on the context expect that device to be current (one process
 * or thread per GPU, the model of the multi-GPU paths).  The engine switches
 * (w1mg_set_*) are process-wide. */
int w1mg_ctx_create(int device, w1mg_ctx** out);
void w1mg_ctx_destroy(w1mg_ctx* ctx);
const char* w1mg_last_error(void);
int w1mg_abi_version(void);
/* Number of fused-iteration kernel launches issued by this context so far
 * (for bench.py's gpu_launches claim). */
long w1mg_ctx_launch_count(const w1mg_ctx* ctx);
/* Device seconds of each level of the last cascade run on this context
 * (CUDA events; waits for that cascade).  Returns the number written, or a
 * negative status. */
int w1mg_ctx_level_seconds(w1mg_ctx* ctx, double* out, int cap);
/* Block until all work queued on the context stream is done. */
int w1mg_ctx_synchronize(w1mg_ctx* ctx);
/* The context's CUDA stream (cudaStream_t), for callers that time on it. */
void* w1mg_ctx_stream(w1mg_ctx* ctx);

/* ------------------------------------------------- step sizes (host only) */
/* cp_step_size, solver_cp.cpp:75-78: 1/||A|| (practical) or 1/(2||A||) with
 * ||A|| <= 2 sqrt(2)/h (grid.cpp:130). */
double w1mg_cp_step_size(int n, int step_mode);
/* pdhg_step_size, solver_pdhg.hpp:19-20: 1 (practical) or 1/2 (safe). */
double w1mg_pdhg_step_size(int step_mode);
/* make_schedule (Eq. 16): eps[l] = eps_L * (h_l/h_L)^alpha. */
int w1mg_make_schedule(int n_finest, int levels, double eps_finest, double alpha, double* eps);

/* ---------------------------------------------------- grid operators (GPU) */
/* divergence_into, grid.cpp:45-68 */
int w1mg_divergence(w1mg_ctx* ctx, int n, const double* mx, const double* my, double* out);
/* adjoint_into, grid.cpp:76-91 (negative forward difference) */
int w1mg_adjoint(w1mg_ctx* ctx, int n, const double* phi, double* gx, double* gy);
/* primal_value, grid.cpp:132-138 (compensated) */
int w1mg_primal_value(w1mg_ctx* ctx, int n, const double* mx, const double* my, int pnorm,
                      double* out);
/* inner_h on nodes, grid.cpp:99-104 (compensated); dual_value = inner_h(phi, rho) */
int w1mg_inner_h_nodes(w1mg_ctx* ctx, int n, const double* a, const double* b, double* out);
/* inner_h on edges, grid.cpp:106-112 */
int w1mg_inner_h_edges(w1mg_ctx* ctx, int n, const double* ax, const double* ay,
                       const double* bx, const double* by, double* out);
/* SourceField gate, grid.cpp:35-43: W1MG_OK if |sum rho| <= 1e-12 sum|rho|,
 * else W1MG_EINVAL "SourceField: values do not sum to zero".  Host-side. */
int w1mg_source_check(int n, const double* rho);

/* ------------------------------------------------- Algorithm 1 (Li et al.) */
/* cp_run, solver_cp.cpp:113-147.  m0x/m0y/phi0 may be NULL (zero start).
 * mu/tau as from w1mg_cp_step_size.  Stops when the Eq. 9 residual < tol or
 * after max_iters sweeps.  Outputs mx/my/phi may be NULL; fpr_hist receives
 * min(iterations, hist_cap) residuals.  Convergence is decided on the
 * device every sweep; the host never synchronises per iteration. */
int w1mg_cp_run(w1mg_ctx* ctx, int n, const double* rho, const double* m0x, const double* m0y,
                const double* phi0, int pnorm, double mu, double tau, double tol, long max_iters,
                double* mx, double* my, double* phi, double* fpr_hist, long hist_cap,
                w1mg_cp_report* rep);

/* cp_residual, solver_cp.cpp:102-111 (Eq. 9 between two states). */
int w1mg_cp_residual(w1mg_ctx* ctx, int n, const double* cmx, const double* cmy,
                     const double* cphi, const double* pmx, const double* pmy,
                     const double* pphi, double mu, double tau, double* out);

/* ------------------------------------------- sources and cascade (Alg. 3) */
/* Eq. 14: nested-bilinear prolongation of a potential from
 * nc cells to 2 nc cells. */
int w1mg_interpolate_scalar(w1mg_ctx* ctx, int nc, const double* coarse, double* fine);
/* Eq. 15: flux prolongation, nearest coarse edge along the
 * edge direction (ties to the lower coordinate), transverse average. */
int w1mg_interpolate_flux(w1mg_ctx* ctx, int nc, const double* cx, const double* cy,
                          double* fx, double* fy);

/* Per-level sources from two m x m cell images (finest level n = m): 2x2
 * block-sum restriction, cell->node averaging, unit-mass normalisation,
 * rho = (a - b)/h^2 minus its compensated mean.  Output is
 * the concatenation coarse->fine of (n_l+1)^2 arrays. */
int w1mg_ml_sources(w1mg_ctx* ctx, int m, const double* img0, const double* img1, int levels,
                    double* rho_levels);

/* Cascadic Li et al. PD (Algorithm 3) for one pair.  rho_levels: coarse->
 * fine concatenation.  Final-level fields (may be NULL), per-level stats
 * (levels entries, may be NULL), finest-level residual history. */
int w1mg_ml_cp_run(w1mg_ctx* ctx, int n_finest, const double* rho_levels,
                   const w1mg_ml_params* prm, double* mx, double* my, double* phi,
                   w1mg_level_stats* stats, double* fpr_hist, long hist_cap,
                   w1mg_cp_report* rep);

/* Batched cascades (config 4): npairs independent pairs given as m x m cell
 * images (img0s/img1s: npairs*m*m, pair-major).  Per pair outputs:
 * distance[npairs], dual[npairs], iters[npairs*levels], converged[npairs]
 * (any output pointer may be NULL).  The _dev variant takes device image
 * pointers and writes device outputs. */
int w1mg_ml_cp_batch(w1mg_ctx* ctx, int npairs, int m, const double* img0s,
                     const double* img1s, const w1mg_ml_params* prm, double* distance,
                     double* dual, long* iters, int* converged);
/* w1mg_ml_cp_batch plus every pair's finest-level fields from its latest
 * buffer (pair-major: mx, my npairs*m*(m+1); phi npairs*(m+1)^2) and final
 * residual (npairs); field pointers may be NULL.  For per-pair parity checks
 * of the batched engines. */
int w1mg_ml_cp_batch_fields(w1mg_ctx* ctx, int npairs, int m, const double* img0s,
                            const double* img1s, const w1mg_ml_params* prm, double* distance,
                            double* dual, long* iters, int* converged, double* mx, double* my,
                            double* phi, double* fpr_final);
int w1mg_ml_cp_batch_dev(w1mg_ctx* ctx, int npairs, int m, const double* img0s_dev,
                         const double* img1s_dev, const w1mg_ml_params* prm,
                         double* distance_dev, double* dual_dev, long* iters_dev,
                         int* converged_dev);

/* ------------------------------------- Poisson + Algorithm 2 (G-prox PDHG) */
/* NeumannPoissonSolver::solve_into (check_compat = 1, poisson.cpp:61-70: throws
 * "NeumannPoissonSolver: right-hand side must sum to zero") or
 * solve_projected_into (0, poisson.cpp:72-99): zero-mean phi with
 * A A* phi = b via DCT-II -> spectral divide -> DCT-III on the GPU. */
int w1mg_poisson_solve(w1mg_ctx* ctx, int n, const double* b, double* phi, int check_compat);
/* project_affine (poisson.cpp:101-132): m - A* (A A*)^{-1} (A m - rho). */
int w1mg_project_affine(w1mg_ctx* ctx, int n, const double* mx, const double* my,
                        const double* rho, double* out_x, double* out_y);
/* recover_potential (solver_pdhg.hpp:42-46): zero-mean phi, A A* phi = A varphi. */
int w1mg_recover_potential(w1mg_ctx* ctx, int n, const double* dual_x, const double* dual_y,
                           double* phi);
/* pdhg_run (solver_pdhg.hpp:36-40) from (m0, varphi0, varphi_bar0) (NULL = zero;
 * varphi_bar0 NULL = varphi0) until the Eq. 12 residual < tol or
 * max_iters.  mu = tau = w1mg_pdhg_step_size().  Outputs (any may be NULL):
 * m, varphi, varphi_bar, the recovered potential phi; rep->dual_value is
 * <phi, rho>_h (~ +W1). */
int w1mg_pdhg_run(w1mg_ctx* ctx, int n, const double* rho, const double* m0x, const double* m0y,
                  const double* d0x, const double* d0y, const double* b0x, const double* b0y,
                  int pnorm, double mu, double tau, double tol, long max_iters, double* mx,
                  double* my, double* dx, double* dy, double* bx, double* by, double* phi,
                  double* fpr_hist, long hist_cap, w1mg_cp_report* rep);
/* pdhg_residual (solver_pdhg.hpp:32-34, Eq. 12 with the + cross term). */
int w1mg_pdhg_residual(w1mg_ctx* ctx, int n, const double* cmx, const double* cmy,
                       const double* cdx, const double* cdy, const double* pmx, const double* pmy,
                       const double* pdx, const double* pdy, double mu, double tau, double* out);
/* Cascadic Algorithm 4 for one pair (per-level sources coarse -> fine).  With
 * rel_tol > 0 each level's tolerance is rel_tol * G_cold,l (first Eq. 12
 * residual from the zero state). */
int w1mg_ml_pdhg_run(w1mg_ctx* ctx, int n_finest, const double* rho_levels,
                     const w1mg_ml_params* prm, double* mx, double* my, double* dx, double* dy,
                     double* phi, w1mg_level_stats* stats, double* fpr_hist, long hist_cap,
                     w1mg_cp_report* rep);

/* ------------------------------------- row-slab decomposition (config 5) */
/* One grid cut into contiguous row slabs with a one-row halo exchanged every
 * sweep and a cross-slab sum of the residual.  Fields are
 * bit-identical to the undecomposed solve. */
typedef struct w1mg_slab_comm w1mg_slab_comm;
/* bounds[0..nslabs]: slab r owns node rows [bounds[r], bounds[r+1]). */
int w1mg_slab_bounds(int n, int nslabs, int* bounds);
/* 128-byte NCCL unique id (rank 0 creates it, the caller broadcasts it). */
int w1mg_nccl_unique_id(unsigned char* id128);
/* One communicator per rank (one process per GPU, the context's device). */
int w1mg_slab_comm_create(w1mg_ctx* ctx, int world, int rank, const unsigned char* id128,
                          w1mg_slab_comm** out);
void w1mg_slab_comm_destroy(w1mg_slab_comm* comm);
/* Fused peer transport for slab runs of an n-cell grid on this comm
 * (collective): allocates this rank's IPC-shared arena (slab buffer, residual
 * mailbox, arrival counter), exchanges CUDA IPC handles with ncclAllGather and
 * maps every peer's arena (NVLink P2P).  Afterwards the sweeps store halo rows
 * directly into the neighbours' buffers and post residual sums to every
 * rank's mailbox -- no NCCL calls per sweep. */
int w1mg_slab_comm_enable_peer(w1mg_ctx* ctx, w1mg_slab_comm* comm, int n);
/* Transport of emulated slabs (comm == NULL): 1 = fused peer stores between
 * the slabs (default), 0 = device-copy halos. */
int w1mg_set_slab_transport(int peer);
/* cp_run on a decomposed grid.  comm == NULL: `nslabs` slabs emulated on the
 * context's device (see w1mg_set_slab_transport).  comm != NULL: this rank's
 * slab of comm's world (fused peer transport after
 * w1mg_slab_comm_enable_peer, else halos by ncclSend/ncclRecv and the
 * residual by ncclAllReduce; all on the context stream inside CUDA graphs).
 * Inputs are full-grid host arrays; outputs are written for the owned rows
 * only; W1, dual, iterations and history are global. */
int w1mg_slab_cp_run(w1mg_ctx* ctx, w1mg_slab_comm* comm, int n, int nslabs, const double* rho,
                     const double* m0x, const double* m0y, const double* phi0, int pnorm,
                     double mu, double tau, double tol, long max_iters, double* mx, double* my,
                     double* phi, double* fpr_hist, long hist_cap, w1mg_cp_report* rep);

/* Config-5 cascade on one large grid: levels with n >= the "slab_min_n"
 * option (default 1024) and the finest level are row-slab partitioned, the
 * coarser ones replicated on every rank (comm == NULL: `nslabs` slabs
 * emulated on one device).  After a partitioned level its slabs are gathered
 * back (NCCL broadcast of each owner's rows) to prolong into the next.
 * Outputs: the finest level's owned rows; stats: all levels. */
int w1mg_ml_slab_cp_run(w1mg_ctx* ctx, w1mg_slab_comm* comm, int nslabs, int n_finest,
                        const double* rho_levels, const w1mg_ml_params* prm, double* mx,
                        double* my, double* phi, w1mg_level_stats* stats, w1mg_cp_report* rep);

/* --------------------------------------------------------------- probes */
/* Select the engine of the fused sweep for subsequent launches in this
 * process: 1 = one-sweep TMA bulk-copy ring, 2 = two-sweep (temporally
 * blocked) bulk-copy ring, 3 = auto (default: three sweeps per pass on batched
 * levels n >= 384 and one-pair 192..384, two sweeps for other n >= 96, one
 * below; tensor-map rings), 5 = two-sweep tensor-map ring, 6 = three-sweep
 * tensor-map ring.  W1MG_EINVAL for 0 and 4 (engines removed).  Also
 * W1MG_SWEEP=tma|tma2|auto|tma2t|tma3.  Results are bit-identical across
 * engines. */
int w1mg_set_sweep_engine(int engine);
/* Level-resident engines (whole level in one launch, state in shared memory):
 * 1 = auto (default: thread-block-cluster engine for small batches with
 * n <= 128, one CTA per pair for n <= 64), 2 = one-CTA engine only,
 * 3 = cluster engine wherever it fits (n <= 256), 0 = off (streaming sweeps
 * only); W1MG_EINVAL otherwise.  Also W1MG_RESIDENT=0..3. */
int w1mg_set_resident_engine(int on);
/* Tail compaction of batched levels (1 = on, default): once at most half of
 * the pairs still run, sweep grids span only the running pairs.  Also
 * W1MG_COMPACT=0|1. */
int w1mg_set_tail_compaction(int on);
/* Level-resident PDHG (one CTA per pair, all iterations of a level in one
 * launch): 1 = for m = n+1 <= 33 (default), 2 = for m <= 65, 0 = off.  Also
 * W1MG_PDHG_SMALL. */
int w1mg_set_pdhg_small(int mode);
/* Engine tuning switches by name (process-wide; each also has a W1MG_<NAME>
 * environment variable read at context creation): "pdhg_small" (0-2),
 * "cluster_pick" (0/1), "compact" (0/1), "compact_step" (>= 1),
 * "warps_per_sm" (strip target, default 32), "tmap_nw" (2/4/8, 0 = auto),
 * "pdl" (0/1), "fast" (0 = numerics bit-identical to the reference
 * (default); 1 = tolerance mode for p = 2 in the streaming sweep kernels:
 * FMA-contracted node update and an rsqrt shrink, fields within 1e-9 of the
 * reference at fixed sweeps; W1MG_FAST).
 * W1MG_EINVAL for an unknown name or value. */
int w1mg_set_option(const char* name, long value);
/* Times the fused sweep kernel alone: `iters` sweeps over B pairs of an
 * n-cell level (synthetic source, stop rule off) after `warm` untimed ones;
 * writes the mean milliseconds per sweep launch (CUDA events). */
int w1mg_sweep_probe(w1mg_ctx* ctx, int n, int B, int pnorm, long warm, long iters,
                     double* ms_per_sweep);

/* Measured FP64 peak of this device (TFLOP/s, DFMA = 2 flops): SMs x 4 blocks
 * x 256 threads, 8 independent DFMA chains of `iters` steps each, CUDA events.
 * The denominator of the sweep kernels' FP64-pipe roofline (bench.py). */
int w1mg_fp64_peak_probe(w1mg_ctx* ctx, long iters, double* tflops);

/* Diagnostics: compares the kernels' branch-free sqrt / division / p = 2
 * shrink (restated fast paths, device_common.cuh) with the library operators
 * on `count` random and edge-case operands scaled around mu; bad[0..2] =
 * mismatching sqrt, division, shrink results (0 expected). */
int w1mg_rn_selftest(w1mg_ctx* ctx, long count, unsigned long long seed, double mu,
                     unsigned long long* bad);

/* Diagnostics, host only (no GPU needed): checks the index tables of the
 * register-stationary prime-factor DCT of the one-pair PDHG level m = n1 * n2
 * (pdhg_rspf.cuh; instantiated for 27 x 19): the Makhoul + Good-Thomas input
 * map and its inverse are bijections onto the column blocks, the CRT output
 * map covers every k once, the W-build tables agree with it.  *bad = number of
 * violated entries (0 expected); W1MG_EINVAL for a factor pair that is not
 * instantiated. */
int w1mg_pdhg_plan_check(int n1, int n2, long* bad);

#ifdef __cplusplus
}
#endif
#endif /* W1MG_CUDA_H */
