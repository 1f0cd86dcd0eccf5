"""Python mirror of the reference's ``w1mg::`` API, running on the B200 path.

Same names, argument meaning and error behaviour as the C++ headers in
/root/reference/proj/include/w1mg (and our source-compatible C++ twin in
include/w1mg/*.hpp), so parity tests read like the reference's own:

    grid.hpp        GridSpec, ScalarField, FluxField, SourceField, divergence,
                    adjoint, inner_h, norm_L2, norm_plain, operator_norm_bound,
                    primal_value, dual_value, compensated_sum
    pnorm.hpp       PNorm, conjugate, vec_norm, pnorm_from_string
    prox.hpp        shrink, project_unit_ball, project_l1_ball (host-inline
                    scalar maps, like the C++ header; device twins are in
                    csrc/device_common.cuh)
    report.hpp      StepMode, SolverParams, LevelStats, SolveReport
    solver_cp.hpp   CPState, cp_step_size, cp_init, cp_step, cp_residual, cp_run
     make_schedule, ml_run (cascadic Algorithm 3),
                    ml_sources, ml_run_batch

Every solver and field operator executes on the GPU through the C-ABI
(libw1mg_cuda.so); invalid arguments raise ValueError carrying the
reference's std::invalid_argument message.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import CPReport, LevelStatsC, MLParams, check, ptr


# ----------------------------------------------------------------- pnorm
class PNorm(enum.IntEnum):
    p1 = 0
    p2 = 1
    pinf = 2


def conjugate(p: PNorm) -> PNorm:
    return {PNorm.p1: PNorm.pinf, PNorm.p2: PNorm.p2, PNorm.pinf: PNorm.p1}[PNorm(p)]


def vec_norm(v, p: PNorm) -> float:
    x, y = v
    if p == PNorm.p1:
        return abs(x) + abs(y)
    if p == PNorm.p2:
        return math.sqrt(x * x + y * y)
    return max(abs(x), abs(y))


def pnorm_from_string(s: str) -> PNorm:
    if s == "1":
        return PNorm.p1
    if s == "2":
        return PNorm.p2
    if s in ("inf", "Inf", "INF"):
        return PNorm.pinf
    raise ValueError(f"p must be one of 1, 2, inf (got '{s}')")


# ------------------------------------------------------------------ grid
@dataclass(frozen=True)
class GridSpec:
    n: int = 1

    def __post_init__(self):
        if self.n < 1:
            raise ValueError("GridSpec: cells_per_side must be positive")

    @property
    def h(self) -> float:
        return 1.0 / self.n

    def nodes_per_side(self) -> int:
        return self.n + 1

    def node_count(self) -> int:
        return (self.n + 1) * (self.n + 1)


@dataclass
class ScalarField:
    grid: GridSpec
    values: np.ndarray = None  # (n+1, n+1), values[j, i]

    def __post_init__(self):
        n = self.grid.n
        if self.values is None:
            self.values = np.zeros((n + 1, n + 1))
        else:
            self.values = np.ascontiguousarray(self.values, dtype=np.float64).reshape(n + 1, n + 1)


@dataclass
class FluxField:
    grid: GridSpec
    x_edges: np.ndarray = None  # (n+1, n): x_edges[j, i], edge (i,j)->(i+1,j)
    y_edges: np.ndarray = None  # (n, n+1): y_edges[j, i], edge (i,j)->(i,j+1)

    def __post_init__(self):
        n = self.grid.n
        self.x_edges = (np.zeros((n + 1, n)) if self.x_edges is None else
                        np.ascontiguousarray(self.x_edges, dtype=np.float64).reshape(n + 1, n))
        self.y_edges = (np.zeros((n, n + 1)) if self.y_edges is None else
                        np.ascontiguousarray(self.y_edges, dtype=np.float64).reshape(n, n + 1))

    def node_vector(self, i: int, j: int):
        n = self.grid.n
        return (self.x_edges[j, i] if i < n else 0.0, self.y_edges[j, i] if j < n else 0.0)

    def copy(self) -> "FluxField":
        return FluxField(self.grid, self.x_edges.copy(), self.y_edges.copy())


class SourceField:
    """rho = rho0 - rho1; construction enforces |sum| <= 1e-12 sum|.|
    (grid.cpp:35-43, checked by the C-ABI's host gate)."""

    def __init__(self, f: ScalarField):
        check(_lib.lib().w1mg_source_check(f.grid.n, ptr(f.values)))
        self.rho = f

    def grid(self) -> GridSpec:
        return self.rho.grid


def _ctx():
    return _lib.default_context().h


def _same(a: GridSpec, b: GridSpec, msg="grid mismatch"):
    if a != b:
        raise ValueError(msg)


def divergence(m: FluxField) -> ScalarField:
    out = ScalarField(m.grid)
    check(_lib.lib().w1mg_divergence(_ctx(), m.grid.n, ptr(m.x_edges), ptr(m.y_edges),
                                     ptr(out.values)))
    return out


def adjoint(phi: ScalarField) -> FluxField:
    out = FluxField(phi.grid)
    check(_lib.lib().w1mg_adjoint(_ctx(), phi.grid.n, ptr(phi.values), ptr(out.x_edges),
                                  ptr(out.y_edges)))
    return out


def inner_h(a, b) -> float:
    _same(a.grid, b.grid)
    r = C.c_double()
    if isinstance(a, ScalarField):
        check(_lib.lib().w1mg_inner_h_nodes(_ctx(), a.grid.n, ptr(a.values), ptr(b.values),
                                            C.byref(r)))
    else:
        check(_lib.lib().w1mg_inner_h_edges(_ctx(), a.grid.n, ptr(a.x_edges), ptr(a.y_edges),
                                            ptr(b.x_edges), ptr(b.y_edges), C.byref(r)))
    return r.value


def norm_L2(a) -> float:
    return math.sqrt(inner_h(a, a))


def norm_plain(a) -> float:
    """Unweighted Euclidean norm (grid.cpp:117-128): Neumaier sum of squares
    in the reference's order on the host (a utility, not the solve path)."""
    arrs = [a.values] if isinstance(a, ScalarField) else [a.x_edges, a.y_edges]
    s = c = 0.0
    for arr in arrs:
        for x in np.ravel(arr).tolist():
            y = x * x
            t = s + y
            c += (s - t) + y if abs(s) >= abs(y) else (y - t) + s
            s = t
    return math.sqrt(s + c)


def operator_norm_bound(grid: GridSpec) -> float:
    return 2.0 * math.sqrt(2.0) / grid.h


def primal_value(m: FluxField, p: PNorm) -> float:
    r = C.c_double()
    check(_lib.lib().w1mg_primal_value(_ctx(), m.grid.n, ptr(m.x_edges), ptr(m.y_edges), int(p),
                                       C.byref(r)))
    return r.value


def dual_value(phi: ScalarField, rho: SourceField) -> float:
    return inner_h(phi, rho.rho)


def compensated_sum(v) -> float:
    s = c = 0.0
    for x in np.ravel(np.asarray(v, dtype=np.float64)).tolist():
        t = s + x
        c += ((s - t) + x) if abs(s) >= abs(x) else ((x - t) + s)
        s = t
    return s + c


# ------------------------------------------------------------------ prox
def _soft(v, mu):
    return math.copysign(max(abs(v) - mu, 0.0), v)


def project_l1_ball(v, radius: float):
    if radius <= 0.0:
        raise ValueError("project_l1_ball: radius must be positive")
    x, y = v
    ax, ay = abs(x), abs(y)
    if ax + ay <= radius:
        return (x, y)
    hi, lo = (ay if ax < ay else ax), (ay if ay < ax else ax)
    th = hi - radius if hi - radius >= lo else 0.5 * (ax + ay - radius)
    return (_soft(x, th), _soft(y, th))


def shrink(v, mu: float, p: PNorm):
    if mu <= 0.0:
        raise ValueError("shrink: mu must be positive")
    x, y = v
    if p == PNorm.p1:
        return (_soft(x, mu), _soft(y, mu))
    if p == PNorm.p2:
        nrm = math.sqrt(x * x + y * y)
        if nrm <= mu:
            return (0.0, 0.0)
        s = 1.0 - mu / nrm
        return (s * x, s * y)
    if p == PNorm.pinf:
        qx, qy = project_l1_ball(v, mu)
        return (x - qx, y - qy)
    raise AssertionError("bad PNorm")


def project_unit_ball(v, q: PNorm):
    x, y = v
    if q == PNorm.p1:
        return (x, y) if abs(x) + abs(y) <= 1.0 else project_l1_ball(v, 1.0)
    if q == PNorm.p2:
        n2 = x * x + y * y
        if n2 <= 1.0:
            return (x, y)
        s = 1.0 / math.sqrt(n2)
        return (s * x, s * y)
    if q == PNorm.pinf:
        return (min(max(x, -1.0), 1.0), min(max(y, -1.0), 1.0))
    raise AssertionError("bad PNorm")


# ---------------------------------------------------------------- report
class StepMode(enum.IntEnum):
    safe = 0
    practical = 1


@dataclass
class SolverParams:
    p: PNorm = PNorm.p1
    tolerance: float = 1e-8
    max_iters: int = 5_000_000
    step_mode: StepMode = StepMode.practical


@dataclass
class LevelStats:
    h: float = 0.0
    eps: float = 0.0
    iters: int = 0
    fpr_final: float = 0.0
    seconds: float = 0.0


@dataclass
class SolveReport:
    distance: float = 0.0
    dual_value: float = 0.0
    converged: bool = False
    iterations: int = 0
    flux: Optional[FluxField] = None
    potential: Optional[ScalarField] = None
    dual_flux: Optional[FluxField] = None
    levels: list = field(default_factory=list)
    residual_history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    total_seconds: float = 0.0


# ------------------------------------------------------------- solver_cp
@dataclass
class CPState:
    m: FluxField
    phi: ScalarField
    m_prev: FluxField
    mu: float = 0.0
    tau: float = 0.0
    k: int = 0


def cp_step_size(grid: GridSpec, mode: StepMode) -> float:
    return _lib.lib().w1mg_cp_step_size(grid.n, int(mode))


def cp_init(grid: GridSpec, mode: StepMode, m0: FluxField, phi0: ScalarField) -> CPState:
    if m0.grid != grid or phi0.grid != grid:
        raise ValueError("cp_init: grid mismatch")
    s = cp_step_size(grid, mode)
    return CPState(m0.copy(), ScalarField(grid, phi0.values.copy()), m0.copy(), s, s, 0)


def _cp_call(n, rho, m0x, m0y, phi0, p, mu, tau, tol, max_iters, hist_cap):
    mx = np.empty((n + 1, n))
    my = np.empty((n, n + 1))
    phi = np.empty((n + 1, n + 1))
    cap = int(hist_cap)
    hist = np.zeros(max(cap, 1))
    rep = CPReport()
    check(_lib.lib().w1mg_cp_run(_ctx(), n, ptr(rho), ptr(m0x), ptr(m0y), ptr(phi0), int(p), mu,
                                 tau, tol, int(max_iters), ptr(mx), ptr(my), ptr(phi),
                                 ptr(hist) if cap > 0 else None, cap, C.byref(rep)))
    return mx, my, phi, hist[: min(rep.iterations, cap)].copy(), rep


def cp_step(state: CPState, rho: SourceField, p: PNorm) -> CPState:
    if rho.grid() != state.m.grid:
        raise ValueError("cp_step: grid mismatch")
    g = state.m.grid
    mx, my, phi, _, _ = _cp_call(g.n, rho.rho.values, state.m.x_edges, state.m.y_edges,
                                 state.phi.values, p, state.mu, state.tau, -math.inf, 1, 0)
    return CPState(FluxField(g, mx, my), ScalarField(g, phi), state.m.copy(), state.mu,
                   state.tau, state.k + 1)


def cp_residual(curr: CPState, prev: CPState) -> float:
    g = curr.m.grid
    r = C.c_double()
    check(_lib.lib().w1mg_cp_residual(_ctx(), g.n, ptr(curr.m.x_edges), ptr(curr.m.y_edges),
                                      ptr(curr.phi.values), ptr(prev.m.x_edges),
                                      ptr(prev.m.y_edges), ptr(prev.phi.values), curr.mu,
                                      curr.tau, C.byref(r)))
    return r.value


def cp_run(rho: SourceField, params: SolverParams, m0: Optional[FluxField] = None,
           phi0: Optional[ScalarField] = None, hist_cap: Optional[int] = None) -> SolveReport:
    """Algorithm 1 until R^k < tolerance or max_iters (solver_cp.cpp:113-147)."""
    g = rho.grid()
    if (m0 is not None and m0.grid != g) or (phi0 is not None and phi0.grid != g):
        raise ValueError("cp_run: grid mismatch")
    step = cp_step_size(g, params.step_mode)
    cap = min(params.max_iters, 1 << 20) if hist_cap is None else hist_cap
    mx, my, phi, hist, rep = _cp_call(
        g.n, rho.rho.values, None if m0 is None else m0.x_edges,
        None if m0 is None else m0.y_edges, None if phi0 is None else phi0.values, params.p,
        step, step, params.tolerance, params.max_iters, cap)
    r = SolveReport(rep.distance, rep.dual_value, bool(rep.converged), rep.iterations,
                    FluxField(g, mx, my), ScalarField(g, phi), None,
                    [LevelStats(g.h, params.tolerance, rep.iterations, rep.fpr_final,
                                rep.seconds)], hist, rep.seconds)
    return r


# ------------------------------------------------------------ multilevel
def make_schedule(n: int, levels: int, eps_finest: float, alpha: float = -1.0) -> list:
    """Eq. 16: eps_l = eps_L (h_l/h_L)^alpha, coarse -> fine."""
    out = np.zeros(levels)
    check(_lib.lib().w1mg_make_schedule(n, levels, eps_finest, alpha, ptr(out)))
    return out.tolist()


def default_levels(n: int) -> int:
    """SPEC.md:359 default L = log2 N - 3 (at least 1)."""
    return max(1, int(round(math.log2(n))) - 3)


def ml_sources(img0: np.ndarray, img1: np.ndarray, levels: int) -> list:
    """Device restriction: per-level sources (coarse -> fine) from two m x m
    cell images (2x2 block sums, cell->node mean, unit mass, zero mean)."""
    img0 = np.ascontiguousarray(img0, dtype=np.float64)
    img1 = np.ascontiguousarray(img1, dtype=np.float64)
    m = img0.shape[0]
    sizes = [((m >> (levels - 1 - l)) + 1) ** 2 for l in range(levels)]
    out = np.empty(sum(sizes))
    check(_lib.lib().w1mg_ml_sources(_ctx(), m, ptr(img0), ptr(img1), levels, ptr(out)))
    res, off = [], 0
    for l, s in enumerate(sizes):
        nl = m >> (levels - 1 - l)
        res.append(out[off:off + s].reshape(nl + 1, nl + 1).copy())
        off += s
    return res


def _ml_params(levels, p, step_mode, rel_tol, eps, max_iters):
    prm = MLParams()
    prm.levels = levels
    prm.pnorm = int(p)
    prm.step_mode = int(step_mode)
    prm.max_iters = int(max_iters)
    keep = None
    if eps is not None:
        keep = np.ascontiguousarray(eps, dtype=np.float64)
        prm.eps = ptr(keep)
        prm.rel_tol = -1.0
    else:
        prm.rel_tol = float(rel_tol)
    return prm, keep


def ml_run(rho_levels: list, p: PNorm = PNorm.p2, rel_tol: float = 1e-5, eps=None,
           max_iters: int = 5_000_000, step_mode: StepMode = StepMode.practical,
           hist_cap: int = 1 << 16) -> SolveReport:
    """Cascadic Algorithm 3 over per-level sources (coarse -> fine): level 0
    from zero, then Eq. 14/15 warm starts.  Tolerances are
    rel_tol * R_cold,l unless absolute ``eps`` is given."""
    levels = len(rho_levels)
    nf = rho_levels[-1].shape[0] - 1
    flat = np.ascontiguousarray(np.concatenate([np.ravel(r) for r in rho_levels]))
    prm, keep = _ml_params(levels, p, step_mode, rel_tol, eps, max_iters)
    mx = np.empty((nf + 1, nf))
    my = np.empty((nf, nf + 1))
    phi = np.empty((nf + 1, nf + 1))
    st = (LevelStatsC * levels)()
    hist = np.zeros(max(hist_cap, 1))
    rep = CPReport()
    check(_lib.lib().w1mg_ml_cp_run(_ctx(), nf, ptr(flat), C.byref(prm), ptr(mx), ptr(my),
                                    ptr(phi), st, ptr(hist), hist_cap, C.byref(rep)))
    del keep
    g = GridSpec(nf)
    lv = [LevelStats(s.h, s.eps, s.iters, s.fpr_final, s.seconds) for s in st]
    return SolveReport(rep.distance, rep.dual_value, bool(rep.converged), rep.iterations,
                       FluxField(g, mx, my), ScalarField(g, phi), None, lv,
                       hist[: min(lv[-1].iters, hist_cap)].copy(), rep.seconds)


def ml_run_batch(img0s: np.ndarray, img1s: np.ndarray, levels: int, p: PNorm = PNorm.p2,
                 rel_tol: float = 1e-5, eps=None, max_iters: int = 5_000_000,
                 step_mode: StepMode = StepMode.practical):
    """Batched cascades (config 4): (B, m, m) image stacks -> per-pair
    (distance, dual_value, iters[B, levels], converged)."""
    img0s = np.ascontiguousarray(img0s, dtype=np.float64)
    img1s = np.ascontiguousarray(img1s, dtype=np.float64)
    B, m = img0s.shape[0], img0s.shape[1]
    prm, keep = _ml_params(levels, p, step_mode, rel_tol, eps, max_iters)
    dist = np.zeros(B)
    dual = np.zeros(B)
    iters = np.zeros((B, levels), dtype=np.int64)
    conv = np.zeros(B, dtype=np.int32)
    check(_lib.lib().w1mg_ml_cp_batch(_ctx(), B, m, ptr(img0s), ptr(img1s), C.byref(prm),
                                      ptr(dist), ptr(dual), iters.ctypes.data_as(_lib._lp),
                                      conv.ctypes.data_as(_lib._ip)))
    del keep
    return dist, dual, iters, conv.astype(bool)


def ml_run_batch_fields(img0s: np.ndarray, img1s: np.ndarray, levels: int,
                        p: PNorm = PNorm.p2, rel_tol: float = 1e-5, eps=None,
                        max_iters: int = 5_000_000, step_mode: StepMode = StepMode.practical):
    """ml_run_batch plus every pair's finest-level fields: returns
    (distance, dual, iters, converged, mx[B], my[B], phi[B], fpr_final[B])."""
    img0s = np.ascontiguousarray(img0s, dtype=np.float64)
    img1s = np.ascontiguousarray(img1s, dtype=np.float64)
    B, m = img0s.shape[0], img0s.shape[1]
    prm, keep = _ml_params(levels, p, step_mode, rel_tol, eps, max_iters)
    dist = np.zeros(B)
    dual = np.zeros(B)
    iters = np.zeros((B, levels), dtype=np.int64)
    conv = np.zeros(B, dtype=np.int32)
    mx = np.empty((B, m + 1, m))
    my = np.empty((B, m, m + 1))
    phi = np.empty((B, m + 1, m + 1))
    fpr = np.empty(B)
    check(_lib.lib().w1mg_ml_cp_batch_fields(_ctx(), B, m, ptr(img0s), ptr(img1s), C.byref(prm),
                                             ptr(dist), ptr(dual),
                                             iters.ctypes.data_as(_lib._lp),
                                             conv.ctypes.data_as(_lib._ip), ptr(mx), ptr(my),
                                             ptr(phi), ptr(fpr)))
    del keep
    return dist, dual, iters, conv.astype(bool), mx, my, phi, fpr


def interpolate_scalar(coarse: ScalarField, fine: GridSpec) -> ScalarField:
    """Eq. 14 on the GPU."""
    if fine.n != 2 * coarse.grid.n:
        raise ValueError("interpolate: grids do not nest")
    out = ScalarField(fine)
    check(_lib.lib().w1mg_interpolate_scalar(_ctx(), coarse.grid.n, ptr(coarse.values),
                                             ptr(out.values)))
    return out


def interpolate_flux(coarse: FluxField, fine: GridSpec) -> FluxField:
    """Eq. 15 on the GPU."""
    if fine.n != 2 * coarse.grid.n:
        raise ValueError("interpolate: grids do not nest")
    out = FluxField(fine)
    check(_lib.lib().w1mg_interpolate_flux(_ctx(), coarse.grid.n, ptr(coarse.x_edges),
                                           ptr(coarse.y_edges), ptr(out.x_edges),
                                           ptr(out.y_edges)))
    return out


# --------------------------------------------------------------- poisson
class NeumannPoissonSolver:
    """poisson.hpp:14-38: DCT-II / spectral divide / DCT-III on the GPU."""

    def __init__(self, grid: GridSpec):
        self._grid = grid

    def grid(self) -> GridSpec:
        return self._grid

    def _solve(self, b: ScalarField, out: ScalarField, compat: bool):
        if b.grid != self._grid or out.grid != self._grid:
            raise ValueError("NeumannPoissonSolver: grid mismatch")
        check(_lib.lib().w1mg_poisson_solve(_ctx(), self._grid.n, ptr(b.values), ptr(out.values),
                                            1 if compat else 0))

    def solve(self, b: ScalarField) -> ScalarField:
        out = ScalarField(self._grid)
        self._solve(b, out, True)
        return out

    def solve_into(self, b: ScalarField, out: ScalarField) -> None:
        self._solve(b, out, True)

    def solve_projected_into(self, b: ScalarField, out: ScalarField) -> None:
        self._solve(b, out, False)


def project_affine(solver: NeumannPoissonSolver, m: FluxField, rho: SourceField) -> FluxField:
    if m.grid != solver.grid() or rho.grid() != solver.grid():
        raise ValueError("project_affine: grid mismatch")
    out = FluxField(m.grid)
    check(_lib.lib().w1mg_project_affine(_ctx(), m.grid.n, ptr(m.x_edges), ptr(m.y_edges),
                                         ptr(rho.rho.values), ptr(out.x_edges),
                                         ptr(out.y_edges)))
    return out


# ----------------------------------------------------------- solver_pdhg
@dataclass
class PDHGState:
    m: FluxField
    dual_flux: FluxField
    dual_flux_bar: FluxField
    mu: float = 0.0
    tau: float = 0.0
    k: int = 0


def pdhg_step_size(mode: StepMode) -> float:
    return _lib.lib().w1mg_pdhg_step_size(int(mode))


def pdhg_init(grid: GridSpec, mode: StepMode, m0: FluxField, dual0: FluxField) -> PDHGState:
    if m0.grid != grid or dual0.grid != grid:
        raise ValueError("pdhg_init: grid mismatch")
    s = pdhg_step_size(mode)
    return PDHGState(m0.copy(), dual0.copy(), dual0.copy(), s, s, 0)


def _pdhg_call(n, rho, m0, d0, b0, p, mu, tau, tol, max_iters, hist_cap):
    g = GridSpec(n)
    m, d, b = FluxField(g), FluxField(g), FluxField(g)
    phi = ScalarField(g)
    cap = int(hist_cap)
    hist = np.zeros(max(cap, 1))
    rep = CPReport()
    f = lambda fl, a: None if fl is None else ptr(getattr(fl, a))  # noqa: E731
    check(_lib.lib().w1mg_pdhg_run(
        _ctx(), n, ptr(rho), f(m0, "x_edges"), f(m0, "y_edges"), f(d0, "x_edges"),
        f(d0, "y_edges"), f(b0, "x_edges"), f(b0, "y_edges"), int(p), mu, tau, tol,
        int(max_iters), ptr(m.x_edges), ptr(m.y_edges), ptr(d.x_edges), ptr(d.y_edges),
        ptr(b.x_edges), ptr(b.y_edges), ptr(phi.values), ptr(hist) if cap > 0 else None, cap,
        C.byref(rep)))
    return m, d, b, phi, hist[: min(rep.iterations, cap)].copy(), rep


def pdhg_step(state: PDHGState, rho: SourceField, p: PNorm, solver=None) -> PDHGState:
    g = state.m.grid
    if rho.grid() != g:
        raise ValueError("pdhg_step: grid mismatch")
    m, d, b, _, _, _ = _pdhg_call(g.n, rho.rho.values, state.m, state.dual_flux,
                                  state.dual_flux_bar, p, state.mu, state.tau, -math.inf, 1, 0)
    return PDHGState(m, d, b, state.mu, state.tau, state.k + 1)


def pdhg_residual(curr: PDHGState, prev: PDHGState) -> float:
    g = curr.m.grid
    r = C.c_double()
    check(_lib.lib().w1mg_pdhg_residual(
        _ctx(), g.n, ptr(curr.m.x_edges), ptr(curr.m.y_edges), ptr(curr.dual_flux.x_edges),
        ptr(curr.dual_flux.y_edges), ptr(prev.m.x_edges), ptr(prev.m.y_edges),
        ptr(prev.dual_flux.x_edges), ptr(prev.dual_flux.y_edges), curr.mu, curr.tau,
        C.byref(r)))
    return r.value


def pdhg_run(rho: SourceField, params: SolverParams, m0: Optional[FluxField] = None,
             dual0: Optional[FluxField] = None, hist_cap: Optional[int] = None) -> SolveReport:
    """Algorithm 2 until G^k < tolerance or max_iters (solver_pdhg.hpp:36-40);
    the potential is recovered from the final dual flux (Appendix B)."""
    g = rho.grid()
    if (m0 is not None and m0.grid != g) or (dual0 is not None and dual0.grid != g):
        raise ValueError("pdhg_run: grid mismatch")
    s = pdhg_step_size(params.step_mode)
    cap = min(params.max_iters, 1 << 20) if hist_cap is None else hist_cap
    m, d, _, phi, hist, rep = _pdhg_call(g.n, rho.rho.values, m0, dual0, None, params.p, s, s,
                                         params.tolerance, params.max_iters, cap)
    return SolveReport(rep.distance, rep.dual_value, bool(rep.converged), rep.iterations, m, phi,
                       d, [LevelStats(g.h, params.tolerance, rep.iterations, rep.fpr_final,
                                      rep.seconds)], hist, rep.seconds)


def recover_potential(dual_flux: FluxField, solver=None) -> ScalarField:
    out = ScalarField(dual_flux.grid)
    check(_lib.lib().w1mg_recover_potential(_ctx(), dual_flux.grid.n, ptr(dual_flux.x_edges),
                                            ptr(dual_flux.y_edges), ptr(out.values)))
    return out


def ml_pdhg_run(rho_levels: list, p: PNorm = PNorm.p2, rel_tol: float = 1e-5, eps=None,
                max_iters: int = 5_000_000, step_mode: StepMode = StepMode.practical,
                hist_cap: int = 1 << 16) -> SolveReport:
    """Cascadic Algorithm 4 over per-level sources; level
    tolerance rel_tol * G_cold,l unless absolute ``eps`` is given."""
    levels = len(rho_levels)
    nf = rho_levels[-1].shape[0] - 1
    flat = np.ascontiguousarray(np.concatenate([np.ravel(r) for r in rho_levels]))
    prm, keep = _ml_params(levels, p, step_mode, rel_tol, eps, max_iters)
    g = GridSpec(nf)
    m, d, phi = FluxField(g), FluxField(g), ScalarField(g)
    st = (LevelStatsC * levels)()
    hist = np.zeros(max(hist_cap, 1))
    rep = CPReport()
    check(_lib.lib().w1mg_ml_pdhg_run(_ctx(), nf, ptr(flat), C.byref(prm), ptr(m.x_edges),
                                      ptr(m.y_edges), ptr(d.x_edges), ptr(d.y_edges),
                                      ptr(phi.values), st, ptr(hist), hist_cap, C.byref(rep)))
    del keep
    lv = [LevelStats(s.h, s.eps, s.iters, s.fpr_final, s.seconds) for s in st]
    return SolveReport(rep.distance, rep.dual_value, bool(rep.converged), rep.iterations, m, phi,
                       d, lv, hist[: min(lv[-1].iters, hist_cap)].copy(), rep.seconds)


# ------------------------------------------------- row slabs (config 5)
def ml_slab_run(rho_levels: list, nslabs: int = 2, comm=None, p: PNorm = PNorm.p2,
                rel_tol: float = 1e-5, eps=None, max_iters: int = 5_000_000,
                step_mode: StepMode = StepMode.practical) -> SolveReport:
    """Config-5 cascade: levels with n >= the "slab_min_n" option (default
    1024) and the finest level cut into row slabs, coarser levels replicated
    (emulated on one device when comm is None, else this rank's slab of an
    NCCL decomposition; the returned finest fields hold the owned rows)."""
    levels = len(rho_levels)
    nf = rho_levels[-1].shape[0] - 1
    flat = np.ascontiguousarray(np.concatenate([np.ravel(r) for r in rho_levels]))
    prm, keep = _ml_params(levels, p, step_mode, rel_tol, eps, max_iters)
    g = GridSpec(nf)
    m, phi = FluxField(g), ScalarField(g)
    st = (LevelStatsC * levels)()
    rep = CPReport()
    check(_lib.lib().w1mg_ml_slab_cp_run(_ctx(), None if comm is None else comm.h, nslabs, nf,
                                         ptr(flat), C.byref(prm), ptr(m.x_edges), ptr(m.y_edges),
                                         ptr(phi.values), st, C.byref(rep)))
    del keep
    lv = [LevelStats(s.h, s.eps, s.iters, s.fpr_final, s.seconds) for s in st]
    return SolveReport(rep.distance, rep.dual_value, bool(rep.converged), rep.iterations, m, phi,
                       None, lv, np.zeros(0), rep.seconds)


def slab_bounds(n: int, nslabs: int) -> list:
    """Node-row bounds of the row-slab partition (slab r owns [b[r], b[r+1]))."""
    out = (C.c_int * (nslabs + 1))()
    check(_lib.lib().w1mg_slab_bounds(n, nslabs, out))
    return list(out)


class SlabComm:
    """NCCL communicator for one rank of a row-slab decomposition (one process
    per GPU).  `unique_id` (128 bytes) comes from new_unique_id() on rank 0 and
    is broadcast by the caller (e.g. torch.distributed)."""

    def __init__(self, world: int, rank: int, unique_id: bytes, device: int = 0):
        self.h = C.c_void_p()
        check(_lib.lib().w1mg_slab_comm_create(_lib.default_context(device).h, world, rank,
                                               unique_id, C.byref(self.h)))
        self.world, self.rank = world, rank

    @staticmethod
    def new_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(_lib.lib().w1mg_nccl_unique_id(buf))
        return buf.raw

    def enable_peer(self, n: int, device: int = 0) -> None:
        """Fused peer transport for grid n (collective over the comm): IPC
        arenas exchanged over NCCL, halos and residual sums stored straight
        into the peers' memory by the sweep kernels."""
        check(_lib.lib().w1mg_slab_comm_enable_peer(_lib.default_context(device).h, self.h, n))

    def close(self):
        if self.h:
            _lib.lib().w1mg_slab_comm_destroy(self.h)
            self.h = None


def set_slab_transport(peer: bool) -> None:
    """Emulated slabs: fused peer stores (True, default) or device copies."""
    check(_lib.lib().w1mg_set_slab_transport(1 if peer else 0))


def slab_cp_run(rho: SourceField, params: SolverParams, nslabs: int = 2,
                comm: Optional[SlabComm] = None, m0: Optional[FluxField] = None,
                phi0: Optional[ScalarField] = None, hist_cap: int = 1 << 20) -> SolveReport:
    """cp_run on a grid cut into row slabs (config 5).  comm=None: nslabs
    slabs emulated on one device; otherwise this rank's slab (owned rows of
    the returned fields are filled, the rest is zero)."""
    g = rho.grid()
    step = cp_step_size(g, params.step_mode)
    m = FluxField(g)
    phi = ScalarField(g)
    cap = int(min(hist_cap, params.max_iters))
    hist = np.zeros(max(cap, 1))
    rep = CPReport()
    check(_lib.lib().w1mg_slab_cp_run(
        _ctx(), None if comm is None else comm.h, g.n, nslabs, ptr(rho.rho.values),
        None if m0 is None else ptr(m0.x_edges), None if m0 is None else ptr(m0.y_edges),
        None if phi0 is None else ptr(phi0.values), int(params.p), step, step,
        params.tolerance, int(params.max_iters), ptr(m.x_edges), ptr(m.y_edges), ptr(phi.values),
        ptr(hist), cap, C.byref(rep)))
    return SolveReport(rep.distance, rep.dual_value, bool(rep.converged), rep.iterations, m, phi,
                       None, [LevelStats(g.h, params.tolerance, rep.iterations, rep.fpr_final,
                                         rep.seconds)],
                       hist[: min(rep.iterations, cap)].copy(), rep.seconds)
