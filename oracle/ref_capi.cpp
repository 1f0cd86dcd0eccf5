// ref_capi.cpp -- extern "C" shims over the UNMODIFIED reference library
// (/root/reference/proj/src/{grid,prox,solver_cp,poisson}.cpp, compiled
// out-of-tree by oracle/Makefile into oracle/_ref/libw1mg_ref.so).
//
// TEST INFRASTRUCTURE ONLY.  Used by tests/ to pin the C restatement in
// oracle/w1mg_oracle.c and, on the GPU box, as bench.py's "reference" CPU
// arm.  Nothing in the product links it.
//
// All arrays use the reference layouts (proj/include/w1mg/grid.hpp:30-61).
// Return codes: 0 ok, 1 std::invalid_argument, 2 std::logic_error, 3 other;
// the message is available from ref_last_error().
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>

#include "w1mg/grid.hpp"
#include "w1mg/poisson.hpp"
#include "w1mg/prox.hpp"
#include "w1mg/solver_cp.hpp"

namespace {
thread_local std::string g_err;

w1mg::PNorm to_p(int p) {
    return p == 0 ? w1mg::PNorm::p1 : (p == 1 ? w1mg::PNorm::p2 : w1mg::PNorm::pinf);
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

w1mg::ScalarField scalar(int n, const double* v) {
    w1mg::ScalarField f{w1mg::GridSpec(n)};
    std::memcpy(f.values.data(), v, f.values.size() * sizeof(double));
    return f;
}

w1mg::FluxField flux(int n, const double* x, const double* y) {
    w1mg::FluxField f{w1mg::GridSpec(n)};
    std::memcpy(f.x_edges.data(), x, f.x_edges.size() * sizeof(double));
    std::memcpy(f.y_edges.data(), y, f.y_edges.size() * sizeof(double));
    return f;
}

void put(const w1mg::ScalarField& f, double* v) {
    std::memcpy(v, f.values.data(), f.values.size() * sizeof(double));
}
void put(const w1mg::FluxField& f, double* x, double* y) {
    std::memcpy(x, f.x_edges.data(), f.x_edges.size() * sizeof(double));
    std::memcpy(y, f.y_edges.data(), f.y_edges.size() * sizeof(double));
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_make_grid(int n, double* h) {
    return guard([&] { *h = w1mg::GridSpec(n).h; });
}

int ref_source_check(int n, const double* rho) {
    return guard([&] { w1mg::SourceField s(scalar(n, rho)); });
}

int ref_shrink(double x, double y, double mu, int p, double* out) {
    return guard([&] {
        w1mg::Vec2 u = w1mg::shrink({x, y}, mu, to_p(p));
        out[0] = u.x;
        out[1] = u.y;
    });
}

int ref_project_unit_ball(double x, double y, int q, double* out) {
    return guard([&] {
        w1mg::Vec2 u = w1mg::project_unit_ball({x, y}, to_p(q));
        out[0] = u.x;
        out[1] = u.y;
    });
}

int ref_project_l1_ball(double x, double y, double r, double* out) {
    return guard([&] {
        w1mg::Vec2 u = w1mg::project_l1_ball({x, y}, r);
        out[0] = u.x;
        out[1] = u.y;
    });
}

int ref_divergence(int n, const double* mx, const double* my, double* out) {
    return guard([&] { put(w1mg::divergence(flux(n, mx, my)), out); });
}

int ref_adjoint(int n, const double* phi, double* gx, double* gy) {
    return guard([&] { put(w1mg::adjoint(scalar(n, phi)), gx, gy); });
}

int ref_primal_value(int n, const double* mx, const double* my, int p, double* out) {
    return guard([&] { *out = w1mg::primal_value(flux(n, mx, my), to_p(p)); });
}

int ref_dual_value(int n, const double* phi, const double* rho, double* out) {
    return guard([&] {
        *out = w1mg::dual_value(scalar(n, phi), w1mg::SourceField(scalar(n, rho)));
    });
}

int ref_inner_h_nodes(int n, const double* a, const double* b, double* out) {
    return guard([&] { *out = w1mg::inner_h(scalar(n, a), scalar(n, b)); });
}

int ref_cp_step_size(int n, int safe, double* out) {
    return guard([&] {
        *out = w1mg::cp_step_size(w1mg::GridSpec(n),
                                  safe ? w1mg::StepMode::safe : w1mg::StepMode::practical);
    });
}

// cp_run through the reference's public API (solver_cp.hpp:38-39).
int ref_cp_run(int n, const double* rho, const double* m0x, const double* m0y,
               const double* phi0, int p, int safe, double tol, long max_iters, double* mx,
               double* my, double* phi, double* hist, long hist_cap, long* iters,
               int* converged, double* distance, double* dual, double* fpr_final,
               double* seconds) {
    return guard([&] {
        w1mg::SourceField src(scalar(n, rho));
        w1mg::SolverParams prm;
        prm.p = to_p(p);
        prm.tolerance = tol;
        prm.max_iters = max_iters;
        prm.step_mode = safe ? w1mg::StepMode::safe : w1mg::StepMode::practical;
        w1mg::FluxField m0;
        w1mg::ScalarField f0;
        const w1mg::FluxField* pm = nullptr;
        const w1mg::ScalarField* pf = nullptr;
        if (m0x) {
            m0 = flux(n, m0x, m0y);
            pm = &m0;
        }
        if (phi0) {
            f0 = scalar(n, phi0);
            pf = &f0;
        }
        w1mg::SolveReport r = w1mg::cp_run(src, prm, pm, pf);
        if (mx) put(r.flux, mx, my);
        if (phi) put(r.potential, phi);
        long k = 0;
        for (; hist && k < hist_cap && k < (long)r.residual_history.size(); ++k)
            hist[k] = r.residual_history[k];
        *iters = r.iterations;
        *converged = r.converged ? 1 : 0;
        *distance = r.distance;
        *dual = r.dual_value;
        *fpr_final = r.levels.empty() ? 0.0 : r.levels.back().fpr_final;
        *seconds = r.total_seconds;
    });
}

// value-semantic single step (solver_cp.hpp:23-33)
int ref_cp_step(int n, const double* mx, const double* my, const double* phi, const double* rho,
                int p, int safe, double* omx, double* omy, double* ophi, double* residual) {
    return guard([&] {
        w1mg::GridSpec g(n);
        w1mg::StepMode mode = safe ? w1mg::StepMode::safe : w1mg::StepMode::practical;
        w1mg::CPState s0 = w1mg::cp_init(g, mode, flux(n, mx, my), scalar(n, phi));
        w1mg::SourceField src(scalar(n, rho));
        w1mg::CPState s1 = w1mg::cp_step(s0, src, to_p(p));
        put(s1.m, omx, omy);
        put(s1.phi, ophi);
        *residual = w1mg::cp_residual(s1, s0);
    });
}

int ref_poisson_solve(int n, const double* b, double* out, int projected) {
    return guard([&] {
        w1mg::NeumannPoissonSolver solver{w1mg::GridSpec(n)};
        w1mg::ScalarField o{w1mg::GridSpec(n)};
        if (projected) solver.solve_projected_into(scalar(n, b), o);
        else solver.solve_into(scalar(n, b), o);
        put(o, out);
    });
}

int ref_project_affine(int n, const double* mx, const double* my, const double* rho, double* ox,
                       double* oy) {
    return guard([&] {
        w1mg::NeumannPoissonSolver solver{w1mg::GridSpec(n)};
        w1mg::FluxField r =
            w1mg::project_affine(solver, flux(n, mx, my), w1mg::SourceField(scalar(n, rho)));
        put(r, ox, oy);
    });
}

}  // extern "C"
