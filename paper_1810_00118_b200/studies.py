"""Studies driven through the GPU solver: the SPEC's validation harness and
benchmark sweeps.

  * ``all_pairs`` -- the paper's all-vs-all timing (45 pairs of 10 images,
    PAPER.md:1281) on the batched config-4 engine: pairs of equal size and
    (p, tolerance) go to the device as ONE batch (``w1mg.ml_run_batch``).
  * ``solve_pairs`` -- the batched heterogeneous driver: any list of image
    pairs with mixed sizes, norms, level counts and tolerances; pairs that
    share (size, L, p, tolerance rule) form one device batch, results come
    back in input order (SPEC.md:497 ``bench`` over mixed configurations).
  * ``sweep`` -- iteration / time sweeps over algorithms, level counts and
    the Eq. 16 exponent alpha (the shape of paper Tables 4-6).
  * ``validate_assumptions`` -- Table 3: per-level
    averages of ||z*||^2, ||y*||^2 and of the interpolation discrepancies
    ||I(z*_{l-1}) - z*_l||^2, ||I(y*_{l-1}) - y*_l||^2 (z = (m, phi) from CP,
    y = (m, varphi) from PDHG), with decay exponents r, nu fitted by least
    squares on log2(discrepancy) vs log2(h).
  * ``find_best_tolerance`` -- the largest eps_L satisfying condition (18)
    (SPEC.md:425-431).

All solves run on the B200 through ``w1mg``; nothing here computes a
transport plan on the host.  L2 norms are h^2-weighted sums of squares over
the arrays of a field.
"""
from __future__ import annotations

import itertools
import math
import time
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import w1mg
from .w1mg import FluxField, GridSpec, PNorm, ScalarField, SolverParams, SourceField


# ------------------------------------------------------------------ helpers
def fit_exponent(hs: Sequence[float], values: Sequence[float]) -> float:
    """Least-squares slope of log2(values) against log2(hs)."""
    hs = np.asarray(hs, dtype=np.float64)
    v = np.asarray(values, dtype=np.float64)
    if hs.size < 2 or hs.size != v.size:
        raise ValueError("fit_exponent: need >= 2 (h, value) points")
    if (hs <= 0).any() or (v <= 0).any():
        raise ValueError("fit_exponent: values must be positive")
    x, y = np.log2(hs), np.log2(v)
    xm, ym = x.mean(), y.mean()
    return float(((x - xm) * (y - ym)).sum() / ((x - xm) ** 2).sum())


def l2_norm2(h: float, *arrays) -> float:
    """h^2 * sum of squares over the given arrays."""
    return h * h * math.fsum(float(np.dot(a.ravel(), a.ravel())) for a in arrays)


def _sources(img_a: np.ndarray, img_b: np.ndarray, levels: int) -> list:
    return w1mg.ml_sources(img_a, img_b, levels)


def _src(rho: np.ndarray) -> SourceField:
    n = rho.shape[0] - 1
    return SourceField(ScalarField(GridSpec(n), rho))


# ------------------------------------------------- heterogeneous batches
@dataclass
class PairJob:
    """One density pair of a heterogeneous batch: two square m x m cell
    images, the cascade depth (None: SPEC.md:359 default log2 m - 3), the
    norm, and the tolerance rule (rel_tol * R_cold,l, or the Eq. 16 schedule
    of eps_finest with exponent alpha when eps_finest is given)."""
    a: np.ndarray
    b: np.ndarray
    levels: Optional[int] = None
    p: PNorm = PNorm.p2
    rel_tol: float = 1e-5
    eps_finest: Optional[float] = None
    alpha: float = -1.0


def solve_pairs(jobs: Sequence[PairJob], max_iters: int = 5_000_000) -> list:
    """Solve every job by the cascadic CP solver on the batched config-4
    engine.  Jobs are grouped by (m, L, p, tolerance rule); each group is ONE
    device batch (w1mg.ml_run_batch), so a mixed workload costs one batched
    cascade per distinct configuration instead of one launch sequence per
    pair.  Returns one dict per job, in input order."""
    groups: dict = {}
    for k, job in enumerate(jobs):
        a = np.ascontiguousarray(job.a, dtype=np.float64)
        b = np.ascontiguousarray(job.b, dtype=np.float64)
        if a.ndim != 2 or a.shape[0] != a.shape[1] or a.shape != b.shape:
            raise ValueError(f"solve_pairs: job {k} needs two square images of one size")
        m = a.shape[0]
        L = job.levels if job.levels is not None else w1mg.default_levels(m)
        if L < 1 or m % (1 << (L - 1)):
            raise ValueError(f"solve_pairs: job {k}: N={m} not divisible by 2^(L-1) for L={L}")
        rule = ("eps", float(job.eps_finest), float(job.alpha)) if job.eps_finest is not None \
            else ("rel", float(job.rel_tol))
        groups.setdefault((m, L, int(job.p), rule), []).append((k, a, b))
    out: list = [None] * len(jobs)
    for (m, L, p, rule), members in sorted(groups.items(), key=lambda kv: (kv[0][0], kv[0][1], kv[0][2], str(kv[0][3]))):
        A = np.stack([a for _, a, _ in members])
        Bi = np.stack([b for _, _, b in members])
        eps = w1mg.make_schedule(m, L, rule[1], rule[2]) if rule[0] == "eps" else None
        t0 = time.perf_counter()
        dist, dual, iters, conv = w1mg.ml_run_batch(A, Bi, L, p=PNorm(p),
                                                    rel_tol=rule[1] if rule[0] == "rel" else 1e-5,
                                                    eps=eps, max_iters=max_iters)
        secs = time.perf_counter() - t0
        for q, (k, _, _) in enumerate(members):
            out[k] = {"job": k, "n": m, "levels": L, "p": p, "distance": float(dist[q]),
                      "dual_value": float(dual[q]), "iters": [int(x) for x in iters[q]],
                      "converged": bool(conv[q]), "batch_pairs": len(members),
                      "batch_seconds": secs}
    return out


# ---------------------------------------------------------- all-vs-all
def all_pairs(images: Sequence[np.ndarray], levels: int, p: PNorm = PNorm.p2,
              rel_tol: float = 1e-5, eps=None, max_iters: int = 5_000_000) -> list:
    """Every unordered pair (i < j) of `images`, solved by the cascadic CP
    solver.  Pairs whose images share a size form one device batch (the
    config-4 engine), so K images of one size cost ONE batched cascade.
    Returns one dict per pair, ordered by (i, j)."""
    imgs = [np.ascontiguousarray(im, dtype=np.float64) for im in images]
    for im in imgs:
        if im.ndim != 2 or im.shape[0] != im.shape[1]:
            raise ValueError("all_pairs: images must be square")
    pairs = list(itertools.combinations(range(len(imgs)), 2))
    by_size: dict = {}
    for i, j in pairs:
        if imgs[i].shape != imgs[j].shape:
            raise ValueError(f"all_pairs: images {i} and {j} differ in size")
        by_size.setdefault(imgs[i].shape[0], []).append((i, j))
    rows = {}
    for m, group in sorted(by_size.items()):
        a = np.stack([imgs[i] for i, _ in group])
        b = np.stack([imgs[j] for _, j in group])
        t0 = time.perf_counter()
        dist, dual, iters, conv = w1mg.ml_run_batch(a, b, levels, p=p, rel_tol=rel_tol, eps=eps,
                                                    max_iters=max_iters)
        secs = time.perf_counter() - t0
        for k, (i, j) in enumerate(group):
            rows[(i, j)] = {"i": i, "j": j, "n": m, "levels": levels, "p": int(p),
                            "distance": float(dist[k]), "dual_value": float(dual[k]),
                            "iters": [int(x) for x in iters[k]], "converged": bool(conv[k]),
                            "batch_pairs": len(group), "batch_seconds": secs}
    return [rows[ij] for ij in pairs]


# ---------------------------------------------------------------- sweeps
@dataclass
class SweepRow:
    algo: str
    levels: int
    alpha: float
    p: int
    n: int
    eps_finest: float
    distance: float
    iters: list
    seconds: float
    converged: bool


def solve_instance(rho_levels: list, algo: str, eps: list, p: PNorm,
                   max_iters: int = 5_000_000) -> w1mg.SolveReport:
    """One solve of `algo` in {cp, pdhg, ml-cp, ml-pdhg} on per-level sources
    (coarse -> fine); single-level algorithms use the finest source."""
    if algo == "cp":
        return w1mg.cp_run(_src(rho_levels[-1]), SolverParams(p=p, tolerance=eps[-1],
                                                              max_iters=max_iters))
    if algo == "pdhg":
        return w1mg.pdhg_run(_src(rho_levels[-1]), SolverParams(p=p, tolerance=eps[-1],
                                                                max_iters=max_iters))
    if algo == "ml-cp":
        return w1mg.ml_run(rho_levels, p=p, eps=eps, max_iters=max_iters)
    if algo == "ml-pdhg":
        return w1mg.ml_pdhg_run(rho_levels, p=p, eps=eps, max_iters=max_iters)
    raise ValueError(f"unknown algorithm {algo!r}")


def sweep(img_a: np.ndarray, img_b: np.ndarray, algos: Sequence[str],
          level_counts: Sequence[int], alphas: Sequence[float], eps_finest: float,
          p: PNorm = PNorm.p2, max_iters: int = 5_000_000) -> list:
    """Iterations and time per (algorithm, L, alpha) on one instance (paper
    Tables 4-6 shape).  Single-level algorithms ignore L and alpha (one row)."""
    n = img_a.shape[0]
    rows = []
    for algo in algos:
        multi = algo.startswith("ml-")
        for L in (level_counts if multi else [1]):
            if n % (1 << (L - 1)):
                raise ValueError(f"sweep: N={n} not divisible by 2^(L-1) for L={L}")
            srcs = _sources(img_a, img_b, L)
            for alpha in (alphas if multi else [alphas[0]]):
                eps = w1mg.make_schedule(n, L, eps_finest, alpha)
                t0 = time.perf_counter()
                rep = solve_instance(srcs, algo, eps, p, max_iters)
                secs = time.perf_counter() - t0
                rows.append(SweepRow(algo, L, alpha, int(p), n, eps_finest, rep.distance,
                                     [l.iters for l in rep.levels], secs, rep.converged))
    return rows


# --------------------------------------------------- assumption validation
@dataclass
class AssumptionRow:
    level: int
    h: float
    z_norm2: float
    y_norm2: float
    z_disc: Optional[float]  # None on the coarsest level
    y_disc: Optional[float]


@dataclass
class AssumptionReport:
    rows: list = field(default_factory=list)
    r: float = float("nan")   # decay exponent of the CP discrepancies
    nu: float = float("nan")  # decay exponent of the PDHG discrepancies


def validate_assumptions(instances: Sequence, levels: int, eps: float = 1e-8,
                         p: PNorm = PNorm.p2, max_iters: int = 5_000_000) -> AssumptionReport:
    """Table 3 of the paper on image pairs `instances`: for
    every level, single-level CP and PDHG solves to absolute tolerance `eps`
    from the zero state, norms and interpolation discrepancies averaged over
    the instances, then the fitted exponents."""
    if levels < 2:
        raise ValueError("validate_assumptions: need >= 2 levels")
    K = len(instances)
    acc = np.zeros((levels, 4))
    for img_a, img_b in instances:
        srcs = _sources(img_a, img_b, levels)
        prev_z = prev_y = None
        for l, rho in enumerate(srcs):
            src = _src(rho)
            g = src.grid()
            cp = w1mg.cp_run(src, SolverParams(p=p, tolerance=eps, max_iters=max_iters))
            pd = w1mg.pdhg_run(src, SolverParams(p=p, tolerance=eps, max_iters=max_iters))
            if not (cp.converged and pd.converged):
                raise RuntimeError(f"validate_assumptions: level {l} did not reach eps={eps}")
            z = (cp.flux, cp.potential)
            y = (pd.flux, pd.dual_flux)
            acc[l, 0] += l2_norm2(g.h, z[0].x_edges, z[0].y_edges, z[1].values)
            acc[l, 1] += l2_norm2(g.h, y[0].x_edges, y[0].y_edges, y[1].x_edges, y[1].y_edges)
            if prev_z is not None:
                im = w1mg.interpolate_flux(prev_z[0], g)
                ip = w1mg.interpolate_scalar(prev_z[1], g)
                acc[l, 2] += l2_norm2(g.h, im.x_edges - z[0].x_edges, im.y_edges - z[0].y_edges,
                                      ip.values - z[1].values)
                jm = w1mg.interpolate_flux(prev_y[0], g)
                jd = w1mg.interpolate_flux(prev_y[1], g)
                acc[l, 3] += l2_norm2(g.h, jm.x_edges - y[0].x_edges, jm.y_edges - y[0].y_edges,
                                      jd.x_edges - y[1].x_edges, jd.y_edges - y[1].y_edges)
            prev_z, prev_y = z, y
    acc /= K
    n_f = instances[0][0].shape[0]
    rep = AssumptionReport()
    for l in range(levels):
        h = 1.0 / (n_f >> (levels - 1 - l))
        rep.rows.append(AssumptionRow(l, h, acc[l, 0], acc[l, 1],
                                      acc[l, 2] if l else None, acc[l, 3] if l else None))
    if levels >= 3:
        hs = [r.h for r in rep.rows[1:]]
        rep.r = fit_exponent(hs, [r.z_disc for r in rep.rows[1:]])
        rep.nu = fit_exponent(hs, [r.y_disc for r in rep.rows[1:]])
    return rep


# -------------------------------------------------------- best tolerance
def best_tolerance(candidates: Sequence[float], f_star: Sequence[float],
                   f_K: Callable[[float], Sequence[float]]) -> float:
    """Largest candidate eps_L whose cascade values f_K(eps_L)[l] satisfy
    condition (18), |f*_l - f^K_l| < |f*_l - f*_{l-1}| for l = 2..L
    (1-based), given the reference optima f*_l.  ValueError if none does."""
    if len(candidates) == 0:
        raise ValueError("find_best_tolerance: empty candidate set")
    L = len(f_star)
    for c in sorted(candidates, reverse=True):
        fk = f_K(c)
        if all(abs(f_star[l] - fk[l]) < abs(f_star[l] - f_star[l - 1]) for l in range(1, L)):
            return float(c)
    raise ValueError("find_best_tolerance: no candidate satisfies condition (18)")


def find_best_tolerance(img_a: np.ndarray, img_b: np.ndarray, levels: int, p: PNorm,
                        alpha: float, candidates: Sequence[float], algo: str = "ml-cp",
                        ref_tol: float = 1e-10, max_iters: int = 5_000_000) -> float:
    """SPEC.md:425-431 on one instance.  f*_l: single-level solves of level
    l's source to `ref_tol`; f^K_l(eps_L): the value after level l of the
    cascade with the Eq. 16 schedule of eps_L (the cascade truncated after
    level l runs exactly the first l levels of the full cascade)."""
    if algo not in ("ml-cp", "ml-pdhg"):
        raise ValueError("find_best_tolerance: algo must be ml-cp or ml-pdhg")
    srcs = _sources(img_a, img_b, levels)
    n = img_a.shape[0]
    single = "cp" if algo == "ml-cp" else "pdhg"
    f_star = []
    for rho in srcs:
        rep = solve_instance([rho], single, [ref_tol], p, max_iters)
        f_star.append(rep.distance)

    def f_K(eps_L):
        eps = w1mg.make_schedule(n, levels, eps_L, alpha)
        return [solve_instance(srcs[: l + 1], algo, eps[: l + 1], p, max_iters).distance
                for l in range(levels)]

    return best_tolerance(candidates, f_star, f_K)
