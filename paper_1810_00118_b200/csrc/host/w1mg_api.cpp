// w1mg_api.cpp -- the source-compatible w1mg:: C++ API (include/w1mg/*.hpp)
// implemented on top of the C-ABI in include/w1mg_cuda.h.  A C++ program
// written against the reference headers (/root/reference/proj/include/w1mg)
// recompiles against include/ and links libw1mg.so unchanged; every solver
// and field operator then runs on the B200.
//
// Conventions kept from the reference: value semantics (inputs const&,
// outputs by value), the same std::invalid_argument / std::logic_error texts,
// warm starts copied from nullable pointers, non-convergence reported through
// SolveReport::converged rather than thrown.
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "w1mg/grid.hpp"
#include "w1mg/multilevel.hpp"
#include "w1mg/poisson.hpp"
#include "w1mg/prox.hpp"
#include "w1mg/report.hpp"
#include "w1mg/solver_cp.hpp"
#include "w1mg/solver_pdhg.hpp"
#include "w1mg_cuda.h"

namespace w1mg {
namespace {

// One context per host thread (the C-ABI context is not thread-safe).
struct CtxHolder {
    w1mg_ctx* ctx = nullptr;
    ~CtxHolder() {
        if (ctx) w1mg_ctx_destroy(ctx);
    }
};

void rethrow(int rc) {
    if (rc == W1MG_OK) return;
    std::string msg = w1mg_last_error();
    if (rc == W1MG_EINVAL) throw std::invalid_argument(msg);
    if (rc == W1MG_ELOGIC) throw std::logic_error(msg);
    if (rc == W1MG_ENOMEM) throw std::bad_alloc();
    throw std::runtime_error("w1mg CUDA: " + msg);
}

w1mg_ctx* ctx() {
    thread_local CtxHolder h;
    if (!h.ctx) {
        int dev = 0;
        if (const char* d = std::getenv("W1MG_DEVICE")) dev = std::atoi(d);
        rethrow(w1mg_ctx_create(dev, &h.ctx));
    }
    return h.ctx;
}

void require_same_grid(const GridSpec& a, const GridSpec& b) {
    if (a != b) throw std::invalid_argument("grid mismatch");
}

int pn(PNorm p) {
    if (p == PNorm::p1) return W1MG_P1;
    if (p == PNorm::p2) return W1MG_P2;
    if (p == PNorm::pinf) return W1MG_PINF;
    throw std::logic_error("bad PNorm");
}

int sm(StepMode m) { return m == StepMode::safe ? W1MG_STEP_SAFE : W1MG_STEP_PRACTICAL; }

double soft(double v, double mu) { return std::copysign(std::max(std::abs(v) - mu, 0.0), v); }

}  // namespace

// ------------------------------------------------------------------ grid
SourceField::SourceField(ScalarField f) : rho(std::move(f)) {
    rethrow(w1mg_source_check(rho.grid.n, rho.values.data()));
}

void divergence_into(const FluxField& m, ScalarField& out) {
    require_same_grid(m.grid, out.grid);
    rethrow(w1mg_divergence(ctx(), m.grid.n, m.x_edges.data(), m.y_edges.data(),
                            out.values.data()));
}

ScalarField divergence(const FluxField& m) {
    ScalarField out(m.grid);
    divergence_into(m, out);
    return out;
}

void adjoint_into(const ScalarField& phi, FluxField& out) {
    require_same_grid(phi.grid, out.grid);
    rethrow(w1mg_adjoint(ctx(), phi.grid.n, phi.values.data(), out.x_edges.data(),
                         out.y_edges.data()));
}

FluxField adjoint(const ScalarField& phi) {
    FluxField out(phi.grid);
    adjoint_into(phi, out);
    return out;
}

double inner_h(const ScalarField& a, const ScalarField& b) {
    require_same_grid(a.grid, b.grid);
    double r = 0.0;
    rethrow(w1mg_inner_h_nodes(ctx(), a.grid.n, a.values.data(), b.values.data(), &r));
    return r;
}

double inner_h(const FluxField& a, const FluxField& b) {
    require_same_grid(a.grid, b.grid);
    double r = 0.0;
    rethrow(w1mg_inner_h_edges(ctx(), a.grid.n, a.x_edges.data(), a.y_edges.data(),
                               b.x_edges.data(), b.y_edges.data(), &r));
    return r;
}

double norm_L2(const ScalarField& a) { return std::sqrt(inner_h(a, a)); }
double norm_L2(const FluxField& a) { return std::sqrt(inner_h(a, a)); }
// norm_plain (grid.cpp:117-128): the unweighted Euclidean norm -- a host
// Neumaier sum in the reference's order (O(V) utility, not the solve path),
// so the bits match the reference exactly (sqrt(inner_h)/h would round
// through the h^2 scaling).
namespace {
double neumaier_sq(const std::vector<double>& v, double& s, double& c) {
    for (double x : v) {
        const double y = x * x, t = s + y;
        if (std::fabs(s) >= std::fabs(y)) c += (s - t) + y;
        else c += (y - t) + s;
        s = t;
    }
    return s + c;
}
}  // namespace
double norm_plain(const ScalarField& a) {
    double s = 0.0, c = 0.0;
    return std::sqrt(neumaier_sq(a.values, s, c));
}
double norm_plain(const FluxField& a) {
    double s = 0.0, c = 0.0;
    neumaier_sq(a.x_edges, s, c);
    return std::sqrt(neumaier_sq(a.y_edges, s, c));
}

double operator_norm_bound(const GridSpec& grid) { return 2.0 * std::sqrt(2.0) / grid.h; }

double primal_value(const FluxField& m, PNorm p) {
    double r = 0.0;
    rethrow(w1mg_primal_value(ctx(), m.grid.n, m.x_edges.data(), m.y_edges.data(), pn(p), &r));
    return r;
}

double dual_value(const ScalarField& phi, const SourceField& rho) { return inner_h(phi, rho.rho); }

double compensated_sum(const std::vector<double>& v) {
    double s = 0.0, c = 0.0;
    for (double x : v) {
        double t = s + x;
        c += (std::abs(s) >= std::abs(x)) ? (s - t) + x : (x - t) + s;
        s = t;
    }
    return s + c;
}

// ------------------------------------------------------------------ prox
Vec2 project_l1_ball(Vec2 v, double radius) {
    if (radius <= 0.0) throw std::invalid_argument("project_l1_ball: radius must be positive");
    const double ax = std::abs(v.x), ay = std::abs(v.y);
    if (ax + ay <= radius) return v;
    const double hi = std::max(ax, ay), lo = std::min(ax, ay);
    const double th = (hi - radius >= lo) ? hi - radius : 0.5 * (ax + ay - radius);
    return {soft(v.x, th), soft(v.y, th)};
}

Vec2 shrink(Vec2 v, double mu, PNorm p) {
    if (mu <= 0.0) throw std::invalid_argument("shrink: mu must be positive");
    if (p == PNorm::p1) return {soft(v.x, mu), soft(v.y, mu)};
    if (p == PNorm::p2) {
        const double nrm = std::sqrt(v.x * v.x + v.y * v.y);
        if (nrm <= mu) return {0.0, 0.0};
        const double s = 1.0 - mu / nrm;
        return {s * v.x, s * v.y};
    }
    if (p == PNorm::pinf) {
        const Vec2 q = project_l1_ball(v, mu);
        return {v.x - q.x, v.y - q.y};
    }
    throw std::logic_error("bad PNorm");
}

Vec2 project_unit_ball(Vec2 v, PNorm q) {
    if (q == PNorm::p1) return (std::abs(v.x) + std::abs(v.y) <= 1.0) ? v : project_l1_ball(v, 1.0);
    if (q == PNorm::p2) {
        const double n2 = v.x * v.x + v.y * v.y;
        if (n2 <= 1.0) return v;
        const double s = 1.0 / std::sqrt(n2);
        return {s * v.x, s * v.y};
    }
    if (q == PNorm::pinf) return {std::clamp(v.x, -1.0, 1.0), std::clamp(v.y, -1.0, 1.0)};
    throw std::logic_error("bad PNorm");
}

// ------------------------------------------------------------- solver_cp
double cp_step_size(const GridSpec& grid, StepMode mode) {
    return w1mg_cp_step_size(grid.n, sm(mode));
}

CPState cp_init(const GridSpec& grid, StepMode mode, FluxField m0, ScalarField phi0) {
    if (m0.grid != grid || phi0.grid != grid) throw std::invalid_argument("cp_init: grid mismatch");
    CPState s;
    s.m_prev = m0;
    s.m = std::move(m0);
    s.phi = std::move(phi0);
    s.mu = s.tau = cp_step_size(grid, mode);
    s.k = 0;
    return s;
}

CPState cp_step(const CPState& state, const SourceField& rho, PNorm p) {
    if (rho.grid() != state.m.grid) throw std::invalid_argument("cp_step: grid mismatch");
    CPState next = state;
    next.m_prev = state.m;
    w1mg_cp_report rep{};
    rethrow(w1mg_cp_run(ctx(), state.m.grid.n, rho.rho.values.data(), state.m.x_edges.data(),
                        state.m.y_edges.data(), state.phi.values.data(), pn(p), state.mu,
                        state.tau, -HUGE_VAL, 1, next.m.x_edges.data(), next.m.y_edges.data(),
                        next.phi.values.data(), nullptr, 0, &rep));
    next.k = state.k + 1;
    return next;
}

double cp_residual(const CPState& curr, const CPState& prev) {
    double r = 0.0;
    rethrow(w1mg_cp_residual(ctx(), curr.m.grid.n, curr.m.x_edges.data(), curr.m.y_edges.data(),
                             curr.phi.values.data(), prev.m.x_edges.data(),
                             prev.m.y_edges.data(), prev.phi.values.data(), curr.mu, curr.tau,
                             &r));
    return r;
}

SolveReport cp_run(const SourceField& rho, const SolverParams& params, const FluxField* m0,
                   const ScalarField* phi0) {
    const GridSpec grid = rho.grid();
    if ((m0 && m0->grid != grid) || (phi0 && phi0->grid != grid))
        throw std::invalid_argument("cp_run: grid mismatch");
    const double step = cp_step_size(grid, params.step_mode);
    SolveReport report;
    report.flux = FluxField(grid);
    report.potential = ScalarField(grid);
    const long cap = std::min<long>(params.max_iters, 1L << 24);
    std::vector<double> hist(std::max<long>(cap, 1));
    w1mg_cp_report rep{};
    rethrow(w1mg_cp_run(ctx(), grid.n, rho.rho.values.data(), m0 ? m0->x_edges.data() : nullptr,
                        m0 ? m0->y_edges.data() : nullptr, phi0 ? phi0->values.data() : nullptr,
                        pn(params.p), step, step, params.tolerance, params.max_iters,
                        report.flux.x_edges.data(), report.flux.y_edges.data(),
                        report.potential.values.data(), hist.data(), cap, &rep));
    hist.resize(std::min(rep.iterations, cap));
    report.distance = rep.distance;
    report.dual_value = rep.dual_value;
    report.converged = rep.converged != 0;
    report.iterations = rep.iterations;
    report.residual_history = std::move(hist);
    report.total_seconds = rep.seconds;
    report.levels.push_back({grid.h, params.tolerance, rep.iterations, rep.fpr_final, rep.seconds});
    return report;
}

// ---------------------------------------------------------------- poisson
struct NeumannPoissonSolver::Impl {};

NeumannPoissonSolver::NeumannPoissonSolver(GridSpec grid) : grid_(grid), impl_(new Impl) {}
NeumannPoissonSolver::~NeumannPoissonSolver() = default;

ScalarField NeumannPoissonSolver::solve(const ScalarField& b) const {
    ScalarField out(grid_);
    solve_into(b, out);
    return out;
}

void NeumannPoissonSolver::solve_into(const ScalarField& b, ScalarField& out) const {
    if (b.grid != grid_ || out.grid != grid_)
        throw std::invalid_argument("NeumannPoissonSolver: grid mismatch");
    rethrow(w1mg_poisson_solve(ctx(), grid_.n, b.values.data(), out.values.data(), 1));
}

void NeumannPoissonSolver::solve_projected_into(const ScalarField& b, ScalarField& out) const {
    if (b.grid != grid_ || out.grid != grid_)
        throw std::invalid_argument("NeumannPoissonSolver: grid mismatch");
    rethrow(w1mg_poisson_solve(ctx(), grid_.n, b.values.data(), out.values.data(), 0));
}

FluxField project_affine(const NeumannPoissonSolver& solver, const FluxField& m,
                         const SourceField& rho) {
    if (m.grid != solver.grid() || rho.grid() != solver.grid())
        throw std::invalid_argument("project_affine: grid mismatch");
    FluxField out(m.grid);
    rethrow(w1mg_project_affine(ctx(), m.grid.n, m.x_edges.data(), m.y_edges.data(),
                                rho.rho.values.data(), out.x_edges.data(), out.y_edges.data()));
    return out;
}

void project_affine_inplace(const NeumannPoissonSolver& solver, FluxField& m,
                            const ScalarField& rho, AffineProjectionScratch& scratch) {
    (void)scratch;  // the device engine keeps its own scratch
    if (m.grid != solver.grid() || rho.grid != solver.grid())
        throw std::invalid_argument("project_affine: grid mismatch");
    FluxField out(m.grid);
    rethrow(w1mg_project_affine(ctx(), m.grid.n, m.x_edges.data(), m.y_edges.data(),
                                rho.values.data(), out.x_edges.data(), out.y_edges.data()));
    m = std::move(out);
}

// ----------------------------------------------------------- solver_pdhg
double pdhg_step_size(StepMode mode) { return w1mg_pdhg_step_size(sm(mode)); }

PDHGState pdhg_init(const GridSpec& grid, StepMode mode, FluxField m0, FluxField dual0) {
    if (m0.grid != grid || dual0.grid != grid) throw std::invalid_argument("pdhg_init: grid mismatch");
    PDHGState s;
    s.m = std::move(m0);
    s.dual_flux_bar = dual0;
    s.dual_flux = std::move(dual0);
    s.mu = s.tau = pdhg_step_size(mode);
    s.k = 0;
    return s;
}

PDHGState pdhg_step(const PDHGState& state, const SourceField& rho, PNorm p,
                    const NeumannPoissonSolver& solver) {
    if (solver.grid() != state.m.grid) throw std::invalid_argument("pdhg_step: grid mismatch");
    return pdhg_step(state, rho, p);
}

PDHGState pdhg_step(const PDHGState& state, const SourceField& rho, PNorm p) {
    if (rho.grid() != state.m.grid) throw std::invalid_argument("pdhg_step: grid mismatch");
    PDHGState next = state;
    w1mg_cp_report rep{};
    rethrow(w1mg_pdhg_run(ctx(), state.m.grid.n, rho.rho.values.data(), state.m.x_edges.data(),
                          state.m.y_edges.data(), state.dual_flux.x_edges.data(),
                          state.dual_flux.y_edges.data(), state.dual_flux_bar.x_edges.data(),
                          state.dual_flux_bar.y_edges.data(), pn(p), state.mu, state.tau,
                          -HUGE_VAL, 1, next.m.x_edges.data(), next.m.y_edges.data(),
                          next.dual_flux.x_edges.data(), next.dual_flux.y_edges.data(),
                          next.dual_flux_bar.x_edges.data(), next.dual_flux_bar.y_edges.data(),
                          nullptr, nullptr, 0, &rep));
    next.k = state.k + 1;
    return next;
}

double pdhg_residual(const PDHGState& curr, const PDHGState& prev) {
    double r = 0.0;
    rethrow(w1mg_pdhg_residual(ctx(), curr.m.grid.n, curr.m.x_edges.data(),
                               curr.m.y_edges.data(), curr.dual_flux.x_edges.data(),
                               curr.dual_flux.y_edges.data(), prev.m.x_edges.data(),
                               prev.m.y_edges.data(), prev.dual_flux.x_edges.data(),
                               prev.dual_flux.y_edges.data(), curr.mu, curr.tau, &r));
    return r;
}

SolveReport pdhg_run(const SourceField& rho, const SolverParams& params, const FluxField* m0,
                     const FluxField* dual0) {
    const GridSpec grid = rho.grid();
    if ((m0 && m0->grid != grid) || (dual0 && dual0->grid != grid))
        throw std::invalid_argument("pdhg_run: grid mismatch");
    const double step = pdhg_step_size(params.step_mode);
    SolveReport report;
    report.flux = FluxField(grid);
    report.potential = ScalarField(grid);
    FluxField dual(grid);
    const long cap = std::min<long>(params.max_iters, 1L << 24);
    std::vector<double> hist(std::max<long>(cap, 1));
    w1mg_cp_report rep{};
    rethrow(w1mg_pdhg_run(ctx(), grid.n, rho.rho.values.data(), m0 ? m0->x_edges.data() : nullptr,
                          m0 ? m0->y_edges.data() : nullptr,
                          dual0 ? dual0->x_edges.data() : nullptr,
                          dual0 ? dual0->y_edges.data() : nullptr, nullptr, nullptr, pn(params.p),
                          step, step, params.tolerance, params.max_iters,
                          report.flux.x_edges.data(), report.flux.y_edges.data(),
                          dual.x_edges.data(), dual.y_edges.data(), nullptr, nullptr,
                          report.potential.values.data(), hist.data(), cap, &rep));
    hist.resize(std::min(rep.iterations, cap));
    report.distance = rep.distance;
    report.dual_value = rep.dual_value;
    report.converged = rep.converged != 0;
    report.iterations = rep.iterations;
    report.dual_flux = std::move(dual);
    report.residual_history = std::move(hist);
    report.total_seconds = rep.seconds;
    report.levels.push_back({grid.h, params.tolerance, rep.iterations, rep.fpr_final, rep.seconds});
    return report;
}

ScalarField recover_potential(const FluxField& dual_flux) {
    ScalarField out(dual_flux.grid);
    rethrow(w1mg_recover_potential(ctx(), dual_flux.grid.n, dual_flux.x_edges.data(),
                                   dual_flux.y_edges.data(), out.values.data()));
    return out;
}

ScalarField recover_potential(const FluxField& dual_flux, const NeumannPoissonSolver& solver) {
    if (solver.grid() != dual_flux.grid) throw std::invalid_argument("recover_potential: grid mismatch");
    return recover_potential(dual_flux);
}

// ------------------------------------------------------------ multilevel
LevelSchedule make_schedule(int n, int levels, double eps_finest, double alpha) {
    LevelSchedule s;
    s.levels = levels;
    s.alpha = alpha;
    s.eps.assign(std::max(levels, 1), 0.0);
    rethrow(w1mg_make_schedule(n, levels, eps_finest, alpha, s.eps.data()));
    for (int l = 0; l < levels; ++l) s.grids.emplace_back(n >> (levels - 1 - l));
    return s;
}

int default_levels(int n) {
    int l = 0;
    while ((1 << (l + 1)) <= n) ++l;  // floor(log2 n)
    return std::max(1, l - 3);
}

double default_eps_cp(const GridSpec& finest) {  // Eq. 17
    const double r = finest.h / (1.0 / 512.0);
    return 1e-6 / 128.0 * r * r;
}

double default_eps_pdhg(const GridSpec& finest) {  // Eq. 17
    const double r = finest.h / (1.0 / 512.0);
    return std::min(2e-4, 1e-4 / 32.0 * r * r);
}

ScalarField interpolate_scalar(const ScalarField& coarse, const GridSpec& fine) {
    if (fine.n != 2 * coarse.grid.n) throw std::invalid_argument("interpolate: grids do not nest");
    ScalarField out(fine);
    rethrow(w1mg_interpolate_scalar(ctx(), coarse.grid.n, coarse.values.data(), out.values.data()));
    return out;
}

FluxField interpolate_flux(const FluxField& coarse, const GridSpec& fine) {
    if (fine.n != 2 * coarse.grid.n) throw std::invalid_argument("interpolate: grids do not nest");
    FluxField out(fine);
    rethrow(w1mg_interpolate_flux(ctx(), coarse.grid.n, coarse.x_edges.data(),
                                  coarse.y_edges.data(), out.x_edges.data(), out.y_edges.data()));
    return out;
}

SolveReport ml_run(const std::vector<SourceField>& sources, const MLParams& params) {
    if (sources.empty()) throw std::invalid_argument("ml_run: no levels");
    const int levels = (int)sources.size();
    const GridSpec fine = sources.back().grid();
    std::vector<double> flat;
    for (int l = 0; l < levels; ++l) {
        if (sources[l].grid().n != (fine.n >> (levels - 1 - l)))
            throw std::invalid_argument("ml_run: levels do not nest");
        flat.insert(flat.end(), sources[l].rho.values.begin(), sources[l].rho.values.end());
    }
    w1mg_ml_params p{};
    p.levels = levels;
    p.pnorm = pn(params.p);
    p.step_mode = sm(params.step_mode);
    p.rel_tol = params.eps.empty() ? params.rel_tol : -1.0;
    p.eps = params.eps.empty() ? nullptr : params.eps.data();
    p.max_iters = params.max_iters;
    if (!params.eps.empty() && (int)params.eps.size() != levels)
        throw std::invalid_argument("ml_run: one tolerance per level");
    SolveReport report;
    report.flux = FluxField(fine);
    report.potential = ScalarField(fine);
    std::vector<w1mg_level_stats> st(levels);
    const long cap = 1L << 20;
    std::vector<double> hist(cap);
    w1mg_cp_report rep{};
    if (params.inner == InnerSolver::cp) {
        rethrow(w1mg_ml_cp_run(ctx(), fine.n, flat.data(), &p, report.flux.x_edges.data(),
                               report.flux.y_edges.data(), report.potential.values.data(),
                               st.data(), hist.data(), cap, &rep));
    } else {
        FluxField dual(fine);
        rethrow(w1mg_ml_pdhg_run(ctx(), fine.n, flat.data(), &p, report.flux.x_edges.data(),
                                 report.flux.y_edges.data(), dual.x_edges.data(),
                                 dual.y_edges.data(), report.potential.values.data(), st.data(),
                                 hist.data(), cap, &rep));
        report.dual_flux = std::move(dual);
    }
    for (const auto& s : st) report.levels.push_back({s.h, s.eps, s.iters, s.fpr_final, s.seconds});
    hist.resize(std::min<long>(st.back().iters, cap));
    report.distance = rep.distance;
    report.dual_value = rep.dual_value;
    report.converged = rep.converged != 0;
    report.iterations = rep.iterations;
    report.residual_history = std::move(hist);
    report.total_seconds = rep.seconds;
    return report;
}

std::vector<SourceField> ml_sources(int m, const std::vector<double>& img0,
                                    const std::vector<double>& img1, int levels) {
    if ((long)img0.size() != (long)m * m || (long)img1.size() != (long)m * m)
        throw std::invalid_argument("ml_sources: images must be m x m");
    size_t total = 0;
    for (int l = 0; l < levels; ++l) {
        const int n = m >> (levels - 1 - l);
        total += (size_t)(n + 1) * (n + 1);
    }
    std::vector<double> flat(total);
    rethrow(w1mg_ml_sources(ctx(), m, img0.data(), img1.data(), levels, flat.data()));
    std::vector<SourceField> out;
    size_t off = 0;
    for (int l = 0; l < levels; ++l) {
        const int n = m >> (levels - 1 - l);
        ScalarField f{GridSpec(n)};
        std::copy(flat.begin() + off, flat.begin() + off + f.values.size(), f.values.begin());
        off += f.values.size();
        out.emplace_back(std::move(f));
    }
    return out;
}

}  // namespace w1mg
