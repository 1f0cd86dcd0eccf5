"""numpy restatement of the G-prox PDHG path.  TEST INFRASTRUCTURE ONLY.

The reference declares Algorithm 2 (proj/include/w1mg/solver_pdhg.hpp:8-46)
but ships no implementation; its Poisson solve (proj/src/poisson.cpp) depends
on FFTW3, which is absent here.  This module restates:

* NeumannPoissonSolver.solve_projected_into   poisson.cpp:72-99
  (FFTW REDFT10 = scipy.fft.dct type 2, REDFT01 = type 3, both unnormalised)
* project_affine_inplace                      poisson.cpp:111-132
* pdhg_step / pdhg_residual / pdhg_run        solver_pdhg.hpp:24-40, SPEC.md:272-296,
                                              PAPER.md Eq. 11/12
* recover_potential                           solver_pdhg.hpp:42-46
* the cascadic Algorithm 4

Pinning: the Poisson solve and the affine projection are checked against the
UNMODIFIED reference poisson.cpp (oracle/_ref, FFTW shim) in
tests/test_oracle_vs_ref.py; the PDHG iteration itself has no reference
implementation ("parity pinned by SPEC properties only").

Arrays use the reference layouts: phi (n+1, n+1) [j, i]; x-edges (n+1, n);
y-edges (n, n+1).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy.fft import dctn

P1, P2, PINF = 0, 1, 2


def _neumaier(v) -> float:
    s = c = 0.0
    for x in np.ravel(v).tolist():
        t = s + x
        c += ((s - t) + x) if abs(s) >= abs(x) else ((x - t) + s)
        s = t
    return s + c


def divergence(mx, my, n):
    """grid.cpp:45-68 (x pass assigns, y pass adds)."""
    ih = 1.0 / (1.0 / n)
    right = np.zeros((n + 1, n + 1))
    left = np.zeros((n + 1, n + 1))
    right[:, :n] = mx
    left[:, 1:] = mx
    xpart = (right - left) * ih
    above = np.zeros((n + 1, n + 1))
    below = np.zeros((n + 1, n + 1))
    above[:n, :] = my
    below[1:, :] = my
    return xpart + (above - below) * ih


def adjoint(phi, n):
    """grid.cpp:76-91: negative forward difference."""
    ih = 1.0 / (1.0 / n)
    return (phi[:, :n] - phi[:, 1:]) * ih, (phi[:n, :] - phi[1:, :]) * ih


def lambdas(n):
    m = n + 1
    h = 1.0 / n
    inv_h2 = 1.0 / (h * h)
    return np.array([(2.0 - 2.0 * math.cos(math.pi * k / m)) * inv_h2 for k in range(m)])


def poisson_solve_projected(b, remove_mean=True):
    """poisson.cpp:72-99."""
    n = b.shape[0] - 1
    m = n + 1
    lam = lambdas(n)
    B = dctn(np.asarray(b, dtype=np.float64), type=2)
    B[0, 0] = 0.0
    den = lam[None, :] + lam[:, None]  # [k2, k1] = lambda[k1] + lambda[k2]
    den[0, 0] = 1.0
    B = B / den
    B[0, 0] = 0.0
    out = dctn(B, type=3) * (1.0 / (4.0 * float(m) * float(m)))
    if remove_mean:
        out = out - _neumaier(out) / out.size
    return out


def poisson_solve(b):
    """solve_into (poisson.cpp:61-70): compatibility guard, plain sums."""
    total = float(np.sum(b))  # the reference uses plain loops; magnitude check only
    absolute = float(np.sum(np.abs(b)))
    if abs(total) > 1e-10 * absolute:
        raise ValueError("NeumannPoissonSolver: right-hand side must sum to zero")
    return poisson_solve_projected(b)


def project_affine(mx, my, rho, remove_mean=True):
    """poisson.cpp:111-132: m - A* (A A*)^-1 (A m - rho)."""
    n = rho.shape[0] - 1
    r = divergence(mx, my, n) - rho
    psi = poisson_solve_projected(r, remove_mean)
    gx, gy = adjoint(psi, n)
    return mx - gx, my - gy


def project_unit_ball(vx, vy, q):
    """prox.cpp:47-62, vectorised over node vectors."""
    vx = np.asarray(vx, dtype=np.float64)
    vy = np.asarray(vy, dtype=np.float64)
    if q == P2:
        n2 = vx * vx + vy * vy
        big = n2 > 1.0
        s = np.where(big, 1.0 / np.sqrt(np.where(big, n2, 1.0)), 1.0)
        return np.where(big, s * vx, vx), np.where(big, s * vy, vy)
    if q == PINF:
        cx = np.where(vx < -1.0, -1.0, np.where(1.0 < vx, 1.0, vx))
        cy = np.where(vy < -1.0, -1.0, np.where(1.0 < vy, 1.0, vy))
        return cx, cy
    # q == 1: l1 ball of radius 1 (prox.cpp:16-25)
    ax, ay = np.abs(vx), np.abs(vy)
    inside = ax + ay <= 1.0
    hi = np.where(ax < ay, ay, ax)
    lo = np.where(ay < ax, ay, ax)
    th = np.where(hi - 1.0 >= lo, hi - 1.0, 0.5 * (ax + ay - 1.0))

    def soft(v, t):
        a = np.abs(v) - t
        return np.copysign(np.where(a < 0.0, 0.0, a), v)

    return np.where(inside, vx, soft(vx, th)), np.where(inside, vy, soft(vy, th))


def conjugate(p):
    return {P1: PINF, P2: P2, PINF: P1}[p]


def _node_vectors(fx, fy, n):
    X = np.zeros((n + 1, n + 1))
    Y = np.zeros((n + 1, n + 1))
    X[:, :n] = fx
    Y[:n, :] = fy
    return X, Y


@dataclass
class PDHGState:
    mx: np.ndarray
    my: np.ndarray
    px: np.ndarray
    py: np.ndarray
    bx: np.ndarray
    by: np.ndarray
    mu: float
    tau: float
    k: int = 0


def pdhg_step_size(safe=False):
    return 0.5 if safe else 1.0


def pdhg_init(n, safe=False, m0=None, d0=None):
    s = pdhg_step_size(safe)
    mx = np.zeros((n + 1, n)) if m0 is None else np.array(m0[0], dtype=np.float64)
    my = np.zeros((n, n + 1)) if m0 is None else np.array(m0[1], dtype=np.float64)
    px = np.zeros((n + 1, n)) if d0 is None else np.array(d0[0], dtype=np.float64)
    py = np.zeros((n, n + 1)) if d0 is None else np.array(d0[1], dtype=np.float64)
    return PDHGState(mx, my, px, py, px.copy(), py.copy(), s, s, 0)


def pdhg_step(st: PDHGState, rho, p, remove_mean=True) -> PDHGState:
    """solver_pdhg.hpp:24-30 / SPEC.md:272-276."""
    n = rho.shape[0] - 1
    vx = st.mx - st.mu * st.bx
    vy = st.my - st.mu * st.by
    mx, my = project_affine(vx, vy, rho, remove_mean)
    q = conjugate(p)
    X, Y = _node_vectors(st.px + st.tau * mx, st.py + st.tau * my, n)
    QX, QY = project_unit_ball(X, Y, q)
    px, py = QX[:, :n].copy(), QY[:n, :].copy()
    return PDHGState(mx, my, px, py, 2.0 * px - st.px, 2.0 * py - st.py, st.mu, st.tau, st.k + 1)


def pdhg_residual(curr: PDHGState, prev: PDHGState, n):
    """Eq. 12 (+ cross term)."""
    h = 1.0 / n
    dmx, dmy = curr.mx - prev.mx, curr.my - prev.my
    dpx, dpy = curr.px - prev.px, curr.py - prev.py
    sdm = float(np.sum(dmx * dmx) + np.sum(dmy * dmy))
    sdp = float(np.sum(dpx * dpx) + np.sum(dpy * dpy))
    scr = float(np.sum(dpx * dmx) + np.sum(dpy * dmy))
    return h * h * (sdm / curr.mu + sdp / curr.tau + 2.0 * scr)


def primal_value(mx, my, n, p):
    X, Y = _node_vectors(mx, my, n)
    if p == P1:
        v = np.abs(X) + np.abs(Y)
    elif p == P2:
        v = np.sqrt(X * X + Y * Y)
    else:
        v = np.maximum(np.abs(X), np.abs(Y))
    h = 1.0 / n
    return _neumaier(v) * h * h


def recover_potential(px, py, n):
    """Zero-mean phi with A A* phi = A varphi (Appendix B)."""
    return poisson_solve_projected(divergence(px, py, n))


@dataclass
class PDHGResult:
    mx: np.ndarray
    my: np.ndarray
    px: np.ndarray
    py: np.ndarray
    phi: np.ndarray
    iterations: int
    converged: bool
    distance: float
    dual_value: float
    fpr_final: float
    residual_history: list = field(default_factory=list)
    level_iters: list = field(default_factory=list)
    level_eps: list = field(default_factory=list)


def pdhg_run(rho, p=P2, tol=1e-8, max_iters=5_000_000, m0=None, d0=None, safe=False,
             remove_mean=True):
    """pdhg_run (solver_pdhg.hpp:39-40): iterate until G^k < tol or max_iters;
    distance = primal value of m, dual_value = <recovered potential, rho>_h."""
    n = rho.shape[0] - 1
    st = pdhg_init(n, safe, m0, d0)
    hist = []
    g = 0.0
    conv = False
    k = 0
    while k < max_iters:
        nx = pdhg_step(st, rho, p, remove_mean)
        g = pdhg_residual(nx, st, n)
        st = nx
        k += 1
        hist.append(g)
        if g < tol:
            conv = True
            break
    phi = recover_potential(st.px, st.py, n)
    h = 1.0 / n
    dual = _neumaier(phi * rho) * h * h
    return PDHGResult(st.mx, st.my, st.px, st.py, phi, k, conv,
                      primal_value(st.mx, st.my, n, p), dual, g, hist)


def prolong_flux(cx, cy):
    """Eq. 15 via the C restatement (oracle/w1mg_oracle.c:or_prolong_flux)."""
    from oracle import Oracle

    return Oracle().prolong_flux(cx, cy)


def ml_pdhg_run(rhos, p=P2, rel_tol=1e-5, eps=None, max_iters=5_000_000, safe=False):
    """Algorithm 4: level 0 from zero, then Eq. 15 warm starts of m and varphi
    (varphi_bar = varphi at each level start).  Per-level tolerance:
    rel_tol * G_cold,l (the first G from the zero state, SURVEY D3 analogue),
    or absolute eps[l]."""
    m0 = d0 = None
    its, epss = [], []
    r = None
    for l, rho in enumerate(rhos):
        n = rho.shape[0] - 1
        if eps is None:
            st0 = pdhg_init(n, safe)
            st1 = pdhg_step(st0, rho, p)
            tol = rel_tol * pdhg_residual(st1, st0, n)
        else:
            tol = eps[l]
        epss.append(tol)
        r = pdhg_run(rho, p, tol, max_iters, m0, d0, safe)
        its.append(r.iterations)
        if l + 1 < len(rhos):
            m0 = prolong_flux(r.mx, r.my)
            d0 = prolong_flux(r.px, r.py)
    r.level_iters = its
    r.level_eps = epss
    return r
