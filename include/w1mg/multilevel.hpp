// multilevel.hpp -- cascadic multilevel drivers (Algorithms 3 and 4), the
// Eq. 14/15 interpolation operators and the Eq. 16/17 tolerance schedules.
// The reference only specifies this module; the names follow
// that specification.
#pragma once

#include <vector>

#include "w1mg/report.hpp"

namespace w1mg {

struct LevelSchedule {
    int levels = 1;                 ///< L
    std::vector<GridSpec> grids;    ///< coarse -> fine, h_l = 2^(L-1-l) h
    std::vector<double> eps;        ///< per-level tolerance
    double alpha = -1.0;
};

/// Eq. 16: eps_l = eps_L (h_l/h_L)^alpha.  Throws std::invalid_argument when
/// N is not divisible by 2^(L-1).
LevelSchedule make_schedule(int n, int levels, double eps_finest, double alpha = -1.0);

/// Default L = log2(N) - 3, at least 1.
int default_levels(int n);

/// Eq. 17 default finest tolerances for ml-cp / ml-pdhg.
double default_eps_cp(const GridSpec& finest);
double default_eps_pdhg(const GridSpec& finest);

/// Eq. 14 (nested bilinear) and Eq. 15 (nearest along the edge, transverse
/// average) prolongation from a grid to the grid with twice as many cells.
ScalarField interpolate_scalar(const ScalarField& coarse, const GridSpec& fine);
FluxField interpolate_flux(const FluxField& coarse, const GridSpec& fine);

enum class InnerSolver { cp, pdhg };

struct MLParams {
    PNorm p = PNorm::p2;
    StepMode step_mode = StepMode::practical;
    InnerSolver inner = InnerSolver::cp;
    long max_iters = 5'000'000;        ///< per level
    /// > 0: eps_l = rel_tol * (first-sweep residual from the zero state)
    /// (SURVEY D3); otherwise the absolute schedule below is used.
    double rel_tol = 1e-5;
    std::vector<double> eps;           ///< absolute per-level tolerances
};

/// Cascade over per-level sources, coarse -> fine (Algorithm 3 / 4).
SolveReport ml_run(const std::vector<SourceField>& sources, const MLParams& params);

/// Per-level sources from two m x m cell images: 2x2 block-sum restriction,
/// cell -> node averaging, unit mass, rho = (a - b)/h^2 minus its mean.
std::vector<SourceField> ml_sources(int m, const std::vector<double>& img0,
                                    const std::vector<double>& img1, int levels);

}  // namespace w1mg
