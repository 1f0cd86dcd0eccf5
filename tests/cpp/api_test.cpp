// api_test.cpp -- header-level drop-in test of the w1mg:: C++ API.
//
// The SAME source is compiled twice (tests/cpp/Makefile):
//   * against /root/reference/proj/include + oracle/_ref/libw1mg_ref.so (the
//     unmodified reference sources): defines W1MG_REFERENCE_BUILD;
//   * against include/ + paper_1810_00118_b200/lib/libw1mg.so (the B200 path).
// Both binaries must pass; the second one runs every solver on the GPU.
// Checks are the SPEC.md examples (grid :50-83, prox :122-139, solver_cp
// :220-241, poisson :168-180, multilevel :343-364) plus a fixed-iteration
// fingerprint of cp_run that the two builds must reproduce bit for bit.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "w1mg/grid.hpp"
#include "w1mg/poisson.hpp"
#include "w1mg/prox.hpp"
#include "w1mg/solver_cp.hpp"
#ifndef W1MG_REFERENCE_BUILD
#include "w1mg/multilevel.hpp"
#include "w1mg/solver_pdhg.hpp"
#endif

using namespace w1mg;

static int g_fail = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (!(cond)) {                                                           \
            std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);           \
            ++g_fail;                                                            \
        }                                                                        \
    } while (0)
#define NEAR(a, b, tol) CHECK(std::abs((a) - (b)) <= (tol))

template <class E, class F>
static bool throws(F&& f, const std::string& msg) {
    try {
        f();
    } catch (const E& e) {
        return msg.empty() || std::string(e.what()) == msg;
    } catch (...) {
        return false;
    }
    return false;
}

int main() {
    // ---- grid
    {
        GridSpec g(2);
        FluxField m(g);
        m.x_at(0, 0) = 2.0;
        ScalarField d = divergence(m);
        NEAR(d.at(0, 0), 4.0, 0.0);
        NEAR(d.at(1, 0), -4.0, 0.0);
        ScalarField ones(GridSpec(2));
        for (double& v : ones.values) v = 1.0;
        NEAR(norm_L2(ones), 1.5, 1e-15);
        FluxField mm(g);
        mm.x_at(0, 0) = 3.0;
        mm.y_at(0, 0) = 4.0;
        NEAR(primal_value(mm, PNorm::p2), 1.25, 1e-15);
        GridSpec g1(1);
        ScalarField phi(g1);
        phi.at(1, 0) = 1.0;
        phi.at(1, 1) = 1.0;
        FluxField a = adjoint(phi);
        NEAR(a.x_at(0, 0), -1.0, 0.0);
        NEAR(a.x_at(0, 1), -1.0, 0.0);
        NEAR(a.y_at(0, 0), 0.0, 0.0);
        NEAR(operator_norm_bound(GridSpec(256)), 512.0 * std::sqrt(2.0), 1e-9);
        CHECK(throws<std::invalid_argument>([] { GridSpec bad(0); },
                                            "GridSpec: cells_per_side must be positive"));
        CHECK(throws<std::invalid_argument>([] { SourceField s(ScalarField(GridSpec(3))); (void)s;
                                                 ScalarField f(GridSpec(3)); f.values[0] = 1.0;
                                                 SourceField t(f); },
                                            "SourceField: values do not sum to zero"));
        CHECK(throws<std::invalid_argument>([] { divergence_into(FluxField(GridSpec(2)),
                                                                 *new ScalarField(GridSpec(3))); },
                                            "grid mismatch"));
    }
    // ---- prox
    {
        Vec2 u = shrink({3, 4}, 1.0, PNorm::p2);
        NEAR(u.x, 2.4, 1e-15);
        NEAR(u.y, 3.2, 1e-15);
        u = shrink({0.3, -2}, 0.5, PNorm::p1);
        NEAR(u.x, 0.0, 0.0);
        NEAR(u.y, -1.5, 1e-15);
        u = shrink({0.5, -1.5}, 1.0, PNorm::pinf);
        NEAR(u.x, 0.5, 1e-15);
        NEAR(u.y, -0.5, 1e-15);
        u = project_unit_ball({1.5, -0.2}, PNorm::pinf);
        NEAR(u.x, 1.0, 0.0);
        u = project_unit_ball({3, 4}, PNorm::p2);
        NEAR(u.x, 0.6, 1e-15);
        NEAR(u.y, 0.8, 1e-15);
        u = project_l1_ball({0.5, -1.5}, 1.0);
        NEAR(u.x, 0.0, 0.0);
        NEAR(u.y, -1.0, 0.0);
        CHECK(throws<std::invalid_argument>([] { shrink({1, 1}, 0.0, PNorm::p2); },
                                            "shrink: mu must be positive"));
    }
    // ---- solver_cp + fingerprint
    {
        const int n = 16;
        GridSpec g(n);
        ScalarField r(g);
        for (int j = 0; j <= n; ++j)
            for (int i = 0; i <= n; ++i)
                r.at(i, j) = std::sin(0.7 * i + 0.3 * j) - std::cos(0.2 * i * j);
        double mean = compensated_sum(r.values) / r.values.size();
        for (double& v : r.values) v -= mean;
        SourceField rho(r);
        CPState s0 = cp_init(g, StepMode::practical, FluxField(g), ScalarField(g));
        CPState s1 = cp_step(s0, rho, PNorm::p2);
        bool zero_m = true, phi_ok = true;
        for (double v : s1.m.x_edges) zero_m = zero_m && v == 0.0;
        for (size_t k = 0; k < r.values.size(); ++k)
            phi_ok = phi_ok && s1.phi.values[k] == -(s0.tau * rho.rho.values[k]);
        CHECK(zero_m);
        CHECK(phi_ok);
        NEAR(cp_residual(s1, s0), s0.tau * inner_h(rho.rho, rho.rho), 1e-12 * s0.tau);
        SolverParams p;
        p.p = PNorm::p2;
        p.tolerance = -1.0;
        p.max_iters = 500;
        SolveReport rep = cp_run(rho, p);
        CHECK(rep.iterations == 500);
        CHECK(!rep.converged);
        CHECK(rep.residual_history.size() == 500);
        // bit-level fingerprint shared by both builds
        double fx = 0, fy = 0, fp = 0;
        for (size_t k = 0; k < rep.flux.x_edges.size(); ++k) fx += rep.flux.x_edges[k] * (k % 7 + 1);
        for (size_t k = 0; k < rep.flux.y_edges.size(); ++k) fy += rep.flux.y_edges[k] * (k % 5 + 1);
        for (size_t k = 0; k < rep.potential.values.size(); ++k) fp += rep.potential.values[k] * (k % 3 + 1);
        std::printf("FINGERPRINT %.17g %.17g %.17g W1 %.17g\n", fx, fy, fp, rep.distance);
        // two-Dirac (acceptance 2)
        ScalarField dd(GridSpec(8));
        dd.at(0, 0) = 64.0;
        dd.at(8, 0) = -64.0;
        SolverParams pd;
        pd.p = PNorm::p1;
        pd.tolerance = 1e-12;
        pd.max_iters = 400000;
        SolveReport dr = cp_run(SourceField(dd), pd);
        NEAR(dr.distance, 1.0, 1e-3);
        CHECK(throws<std::invalid_argument>(
            [&] { FluxField wrong(GridSpec(3)); cp_run(rho, p, &wrong); }, "cp_run: grid mismatch"));
    }
    // ---- poisson
    {
        const int n = 8;
        GridSpec g(n);
        ScalarField b(g);
        for (int j = 0; j <= n; ++j)
            for (int i = 0; i <= n; ++i) b.at(i, j) = std::cos(1.3 * i) * std::sin(0.9 * j + 0.1);
        double mean = compensated_sum(b.values) / b.values.size();
        for (double& v : b.values) v -= mean;
        NeumannPoissonSolver solver(g);
        ScalarField phi = solver.solve(b);
        ScalarField back = divergence(adjoint(phi));
        double num = 0, den = 0;
        for (size_t k = 0; k < b.values.size(); ++k) {
            num += (back.values[k] - b.values[k]) * (back.values[k] - b.values[k]);
            den += b.values[k] * b.values[k];
        }
        CHECK(std::sqrt(num) <= 1e-10 * std::sqrt(den));
        ScalarField bad(g);
        bad.values[0] = 1.0;
        CHECK(throws<std::invalid_argument>([&] { solver.solve(bad); },
                                            "NeumannPoissonSolver: right-hand side must sum to zero"));
        SourceField rho(b);
        FluxField m(g);
        for (size_t k = 0; k < m.x_edges.size(); ++k) m.x_edges[k] = std::sin(0.37 * k);
        FluxField pm = project_affine(solver, m, rho);
        ScalarField dv = divergence(pm);
        double res = 0;
        for (size_t k = 0; k < dv.values.size(); ++k) res = std::max(res, std::abs(dv.values[k] - b.values[k]));
        CHECK(res <= 1e-10);
    }
#ifndef W1MG_REFERENCE_BUILD
    // ---- multilevel and PDHG: B200 build only,
    // the reference declares PDHG without implementing it and has no multilevel code
    {
        ScalarField c(GridSpec(1));
        c.at(0, 0) = 0;
        c.at(1, 0) = 2;
        c.at(0, 1) = 1;
        c.at(1, 1) = 3;
        ScalarField f = interpolate_scalar(c, GridSpec(2));
        NEAR(f.at(1, 0), 1.0, 0.0);
        NEAR(f.at(1, 2), 2.0, 0.0);
        NEAR(f.at(0, 1), 0.5, 0.0);
        NEAR(f.at(2, 1), 2.5, 0.0);
        NEAR(f.at(1, 1), 1.5, 0.0);
        FluxField fc(GridSpec(1));
        fc.x_at(0, 0) = 7.0;
        FluxField ff = interpolate_flux(fc, GridSpec(2));
        NEAR(ff.x_at(0, 0), 7.0, 0.0);
        NEAR(ff.x_at(1, 0), 7.0, 0.0);
        NEAR(ff.x_at(0, 1), 3.5, 0.0);
        NEAR(ff.x_at(1, 2), 0.0, 0.0);
        LevelSchedule s = make_schedule(512, 3, 1e-6, -1.0);
        NEAR(s.eps[0], 0.25e-6, 1e-20);
        NEAR(s.eps[1], 0.5e-6, 1e-20);
        CHECK(default_levels(512) == 6);
        NEAR(default_eps_cp(GridSpec(512)), 1e-6 / 128.0, 1e-22);
        CHECK(throws<std::invalid_argument>([] { make_schedule(96, 7, 1e-6); }, ""));

        ScalarField dd(GridSpec(8));
        dd.at(0, 0) = 64.0;
        dd.at(8, 0) = -64.0;
        SolverParams pd;
        pd.p = PNorm::p1;
        pd.tolerance = 1e-10;
        pd.max_iters = 200000;
        SolveReport pr = pdhg_run(SourceField(dd), pd);
        NEAR(pr.distance, 1.0, 1e-3);
        CHECK(pr.dual_flux.has_value());
        std::vector<SourceField> srcs;
        srcs.push_back(SourceField(dd));  // 1-level cascade through ml_run
        MLParams mp;
        mp.p = PNorm::p1;
        mp.rel_tol = 1e-9;
        SolveReport mr = ml_run(srcs, mp);
        NEAR(mr.distance, 1.0, 1e-3);
        mp.inner = InnerSolver::pdhg;
        SolveReport mq = ml_run(srcs, mp);
        NEAR(mq.distance, 1.0, 1e-3);
    }
#endif
    std::printf("%s: %d failure(s)\n", g_fail ? "FAILED" : "OK", g_fail);
    return g_fail ? 1 : 0;
}
