"""CPU parity checkers for the W1 primal-dual path.  TEST INFRASTRUCTURE ONLY.

Two checkers, both loaded with ctypes:

* ``Oracle``    -- oracle/_build/liboracle.so, the plain-C restatement in
                   oracle/w1mg_oracle.c (always buildable with gcc).
* ``Reference`` -- oracle/_ref/libw1mg_ref.so, the UNMODIFIED reference
                   sources (/root/reference/proj/src/*.cpp) compiled by
                   oracle/Makefile plus the extern "C" shims in ref_capi.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs may import
this package.  The product (paper_1810_00118_b200) never does.

Arrays use the reference layouts (proj/include/w1mg/grid.hpp:30-61):
phi (n+1, n+1); x-edges (n+1, n) [row j, column i]; y-edges (n, n+1).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libw1mg_ref.so")

P1, P2, PINF = 0, 1, 2

_dp = C.POINTER(C.c_double)


def _ptr(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def build(quiet: bool = True) -> None:
    """Compile the checkers (make -f oracle/Makefile)."""
    out = subprocess.run(["make", "-s", "-f", os.path.join(HERE, "Makefile")],
                         capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)


def have_reference() -> bool:
    return os.path.exists(REF_SO)


@dataclass
class CPResult:
    mx: np.ndarray
    my: np.ndarray
    phi: np.ndarray
    iterations: int
    converged: bool
    distance: float
    dual_value: float
    fpr_final: float
    residual_history: np.ndarray
    seconds: float = 0.0
    level_iters: list = field(default_factory=list)
    level_eps: list = field(default_factory=list)


class Oracle:
    """ctypes view of oracle/w1mg_oracle.c."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        self.L = L
        L.or_compensated_sum.restype = C.c_double
        L.or_compensated_sum.argtypes = [_dp, C.c_long]
        L.or_source_compatible.restype = C.c_int
        L.or_source_compatible.argtypes = [_dp, C.c_long]
        for nm in ("or_inner_h_nodes", "or_primal_value", "or_dual_value", "or_cp_step_size",
                   "or_inner_h_edges", "or_cp_residual"):
            getattr(L, nm).restype = C.c_double
        L.or_cp_step_size.argtypes = [C.c_int, C.c_int]
        L.or_primal_value.argtypes = [C.c_int, _dp, _dp, C.c_int]
        L.or_dual_value.argtypes = [C.c_int, _dp, _dp]
        L.or_inner_h_nodes.argtypes = [C.c_int, _dp, _dp]
        L.or_inner_h_edges.argtypes = [C.c_int, _dp, _dp, _dp, _dp]
        L.or_cp_residual.argtypes = [C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, C.c_double, C.c_double]
        L.or_cp_run.restype = C.c_int
        L.or_cp_run.argtypes = [C.c_int, _dp, _dp, _dp, _dp, C.c_int, C.c_double, C.c_double,
                                C.c_double, C.c_long, _dp, _dp, _dp, _dp, C.c_long,
                                C.POINTER(C.c_long), C.POINTER(C.c_int), _dp, _dp, _dp]
        L.or_ml_cp_run.restype = C.c_int
        L.or_ml_cp_run.argtypes = [C.c_int, C.c_int, _dp, C.c_int, C.c_int, C.c_double, _dp,
                                   C.c_long, _dp, _dp, _dp, C.POINTER(C.c_long), _dp, _dp, _dp,
                                   _dp]
        L.or_shrink.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, _dp, _dp]
        L.or_project_unit_ball.argtypes = [C.c_double, C.c_double, C.c_int, _dp, _dp]
        L.or_project_l1_ball.argtypes = [C.c_double, C.c_double, C.c_double, _dp, _dp]

    # -- prox ---------------------------------------------------------------
    def shrink(self, v, mu, p):
        ox, oy = C.c_double(), C.c_double()
        self.L.or_shrink(v[0], v[1], mu, p, C.byref(ox), C.byref(oy))
        return ox.value, oy.value

    def project_unit_ball(self, v, q):
        ox, oy = C.c_double(), C.c_double()
        self.L.or_project_unit_ball(v[0], v[1], q, C.byref(ox), C.byref(oy))
        return ox.value, oy.value

    def project_l1_ball(self, v, r):
        ox, oy = C.c_double(), C.c_double()
        self.L.or_project_l1_ball(v[0], v[1], r, C.byref(ox), C.byref(oy))
        return ox.value, oy.value

    # -- grid ---------------------------------------------------------------
    def divergence(self, n, mx, my):
        out = np.empty((n + 1, n + 1))
        self.L.or_divergence(C.c_int(n), _ptr(mx), _ptr(my), _ptr(out))
        return out

    def adjoint(self, n, phi):
        gx = np.empty((n + 1, n))
        gy = np.empty((n, n + 1))
        self.L.or_adjoint(C.c_int(n), _ptr(phi), _ptr(gx), _ptr(gy))
        return gx, gy

    def primal_value(self, n, mx, my, p):
        return self.L.or_primal_value(n, _ptr(mx), _ptr(my), p)

    def dual_value(self, n, phi, rho):
        return self.L.or_dual_value(n, _ptr(phi), _ptr(rho))

    def cp_step_size(self, n, safe=False):
        return self.L.or_cp_step_size(n, 1 if safe else 0)

    def inner_h_nodes(self, n, a, b):
        return self.L.or_inner_h_nodes(n, _ptr(a), _ptr(b))

    def cp_sweep_rows(self, n, jlo, jhi, mx, my, phi, rho, p, mu, tau, omx, omy, ophi):
        """One sweep of node rows [jlo, jhi) (row-slab view); returns the
        three owned partial sums."""
        sums = np.zeros(3)
        self.L.or_cp_sweep_rows(C.c_int(n), C.c_int(jlo), C.c_int(jhi), _ptr(mx), _ptr(my),
                                _ptr(phi), _ptr(rho), C.c_int(p), C.c_double(mu),
                                C.c_double(tau), _ptr(omx), _ptr(omy), _ptr(ophi), _ptr(sums))
        return sums

    def compensated_sum(self, v):
        v = np.ascontiguousarray(v, dtype=np.float64)
        return self.L.or_compensated_sum(_ptr(v), v.size)

    def source_compatible(self, rho):
        rho = np.ascontiguousarray(rho, dtype=np.float64)
        return bool(self.L.or_source_compatible(_ptr(rho), rho.size))

    def cp_residual(self, n, curr, prev, mu, tau):
        return self.L.or_cp_residual(n, _ptr(curr[0]), _ptr(curr[1]), _ptr(curr[2]),
                                     _ptr(prev[0]), _ptr(prev[1]), _ptr(prev[2]), mu, tau)

    # -- solver -------------------------------------------------------------
    def cp_run(self, rho, p=P2, tol=1e-8, max_iters=5_000_000, m0=None, phi0=None, safe=False,
               hist_cap=None):
        rho = np.ascontiguousarray(rho, dtype=np.float64)
        n = rho.shape[0] - 1
        step = self.cp_step_size(n, safe)
        mx = np.empty((n + 1, n))
        my = np.empty((n, n + 1))
        phi = np.empty((n + 1, n + 1))
        cap = int(min(max_iters, 1 << 20) if hist_cap is None else hist_cap)
        hist = np.zeros(max(cap, 1))
        it, conv = C.c_long(), C.c_int()
        dist, dual, ff = C.c_double(), C.c_double(), C.c_double()
        m0x = m0y = None
        if m0 is not None:
            m0x = np.ascontiguousarray(m0[0], dtype=np.float64)
            m0y = np.ascontiguousarray(m0[1], dtype=np.float64)
        if phi0 is not None:
            phi0 = np.ascontiguousarray(phi0, dtype=np.float64)
        rc = self.L.or_cp_run(n, _ptr(rho), _ptr(m0x), _ptr(m0y), _ptr(phi0), p, step, step, tol,
                              max_iters, _ptr(mx), _ptr(my), _ptr(phi), _ptr(hist), cap,
                              C.byref(it), C.byref(conv), C.byref(dist), C.byref(dual),
                              C.byref(ff))
        if rc:
            raise MemoryError("or_cp_run failed")
        k = it.value
        return CPResult(mx, my, phi, k, bool(conv.value), dist.value, dual.value, ff.value,
                        hist[: min(k, cap)].copy())

    def prolong_scalar(self, phic):
        phic = np.ascontiguousarray(phic, dtype=np.float64)
        nc = phic.shape[0] - 1
        out = np.empty((2 * nc + 1, 2 * nc + 1))
        self.L.or_prolong_scalar(C.c_int(nc), _ptr(phic), _ptr(out))
        return out

    def prolong_flux(self, cx, cy):
        cx = np.ascontiguousarray(cx, dtype=np.float64)
        cy = np.ascontiguousarray(cy, dtype=np.float64)
        nc = cx.shape[1]
        nf = 2 * nc
        fx = np.empty((nf + 1, nf))
        fy = np.empty((nf, nf + 1))
        self.L.or_prolong_flux(C.c_int(nc), _ptr(cx), _ptr(cy), _ptr(fx), _ptr(fy))
        return fx, fy

    def ml_sources(self, img0, img1, levels):
        img0 = np.ascontiguousarray(img0, dtype=np.float64)
        img1 = np.ascontiguousarray(img1, dtype=np.float64)
        m = img0.shape[0]
        sizes = [((m >> (levels - 1 - l)) + 1) ** 2 for l in range(levels)]
        out = np.empty(sum(sizes))
        self.L.or_ml_sources(C.c_int(m), _ptr(img0), _ptr(img1), C.c_int(levels), _ptr(out))
        res, off = [], 0
        for l, s in enumerate(sizes):
            n = m >> (levels - 1 - l)
            res.append(out[off:off + s].reshape(n + 1, n + 1).copy())
            off += s
        return res

    def ml_cp_run(self, rhos, p=P2, rel_tol=1e-5, eps=None, max_iters=5_000_000, safe=False):
        levels = len(rhos)
        nf = rhos[-1].shape[0] - 1
        flat = np.ascontiguousarray(np.concatenate([np.ravel(r) for r in rhos]))
        mx = np.empty((nf + 1, nf))
        my = np.empty((nf, nf + 1))
        phi = np.empty((nf + 1, nf + 1))
        its = (C.c_long * levels)()
        leps = np.zeros(levels)
        lfpr = np.zeros(levels)
        dist, dual = C.c_double(), C.c_double()
        e = np.ascontiguousarray(eps if eps is not None else np.zeros(levels), dtype=np.float64)
        rc = self.L.or_ml_cp_run(nf, levels, _ptr(flat), p, 1 if safe else 0,
                                 rel_tol if eps is None else -1.0, _ptr(e), max_iters, _ptr(mx),
                                 _ptr(my), _ptr(phi), its, _ptr(leps), _ptr(lfpr), C.byref(dist),
                                 C.byref(dual))
        if rc:
            raise MemoryError("or_ml_cp_run failed")
        r = CPResult(mx, my, phi, int(sum(its)), True, dist.value, dual.value, float(lfpr[-1]),
                     np.zeros(0))
        r.level_iters = [int(x) for x in its]
        r.level_eps = leps.tolist()
        return r


class RefError(Exception):
    pass


class Reference:
    """ctypes view of the reference library built from /root/reference."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_cp_run.argtypes = [C.c_int, _dp, _dp, _dp, _dp, C.c_int, C.c_int, C.c_double,
                                 C.c_long, _dp, _dp, _dp, _dp, C.c_long, C.POINTER(C.c_long),
                                 C.POINTER(C.c_int), _dp, _dp, _dp, _dp]
        L.ref_cp_step.argtypes = [C.c_int, _dp, _dp, _dp, _dp, C.c_int, C.c_int, _dp, _dp, _dp,
                                  _dp]
        L.ref_shrink.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, _dp]
        L.ref_project_unit_ball.argtypes = [C.c_double, C.c_double, C.c_int, _dp]
        L.ref_project_l1_ball.argtypes = [C.c_double, C.c_double, C.c_double, _dp]
        L.ref_primal_value.argtypes = [C.c_int, _dp, _dp, C.c_int, _dp]
        L.ref_dual_value.argtypes = [C.c_int, _dp, _dp, _dp]
        L.ref_inner_h_nodes.argtypes = [C.c_int, _dp, _dp, _dp]
        L.ref_cp_step_size.argtypes = [C.c_int, C.c_int, _dp]
        L.ref_poisson_solve.argtypes = [C.c_int, _dp, _dp, C.c_int]
        L.ref_project_affine.argtypes = [C.c_int, _dp, _dp, _dp, _dp, _dp]

    def _chk(self, rc):
        if rc:
            msg = self.L.ref_last_error().decode()
            raise RefError(rc, msg)

    def shrink(self, v, mu, p):
        o = np.zeros(2)
        self._chk(self.L.ref_shrink(v[0], v[1], mu, p, _ptr(o)))
        return tuple(o)

    def project_unit_ball(self, v, q):
        o = np.zeros(2)
        self._chk(self.L.ref_project_unit_ball(v[0], v[1], q, _ptr(o)))
        return tuple(o)

    def project_l1_ball(self, v, r):
        o = np.zeros(2)
        self._chk(self.L.ref_project_l1_ball(v[0], v[1], r, _ptr(o)))
        return tuple(o)

    def divergence(self, n, mx, my):
        out = np.empty((n + 1, n + 1))
        self._chk(self.L.ref_divergence(C.c_int(n), _ptr(mx), _ptr(my), _ptr(out)))
        return out

    def adjoint(self, n, phi):
        gx = np.empty((n + 1, n))
        gy = np.empty((n, n + 1))
        self._chk(self.L.ref_adjoint(C.c_int(n), _ptr(phi), _ptr(gx), _ptr(gy)))
        return gx, gy

    def primal_value(self, n, mx, my, p):
        o = np.zeros(1)
        self._chk(self.L.ref_primal_value(n, _ptr(mx), _ptr(my), p, _ptr(o)))
        return float(o[0])

    def dual_value(self, n, phi, rho):
        o = np.zeros(1)
        self._chk(self.L.ref_dual_value(n, _ptr(phi), _ptr(rho), _ptr(o)))
        return float(o[0])

    def cp_step_size(self, n, safe=False):
        o = np.zeros(1)
        self._chk(self.L.ref_cp_step_size(n, 1 if safe else 0, _ptr(o)))
        return float(o[0])

    def source_check(self, rho):
        rho = np.ascontiguousarray(rho, dtype=np.float64)
        self._chk(self.L.ref_source_check(C.c_int(rho.shape[0] - 1), _ptr(rho)))

    def cp_run(self, rho, p=P2, tol=1e-8, max_iters=5_000_000, m0=None, phi0=None, safe=False,
               hist_cap=None):
        rho = np.ascontiguousarray(rho, dtype=np.float64)
        n = rho.shape[0] - 1
        mx = np.empty((n + 1, n))
        my = np.empty((n, n + 1))
        phi = np.empty((n + 1, n + 1))
        cap = int(min(max_iters, 1 << 20) if hist_cap is None else hist_cap)
        hist = np.zeros(max(cap, 1))
        it, conv = C.c_long(), C.c_int()
        dist, dual, ff, secs = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        m0x = m0y = None
        if m0 is not None:
            m0x = np.ascontiguousarray(m0[0], dtype=np.float64)
            m0y = np.ascontiguousarray(m0[1], dtype=np.float64)
        if phi0 is not None:
            phi0 = np.ascontiguousarray(phi0, dtype=np.float64)
        self._chk(self.L.ref_cp_run(n, _ptr(rho), _ptr(m0x), _ptr(m0y), _ptr(phi0), p,
                                    1 if safe else 0, tol, max_iters, _ptr(mx), _ptr(my),
                                    _ptr(phi), _ptr(hist), cap, C.byref(it), C.byref(conv),
                                    C.byref(dist), C.byref(dual), C.byref(ff), C.byref(secs)))
        k = it.value
        return CPResult(mx, my, phi, k, bool(conv.value), dist.value, dual.value, ff.value,
                        hist[: min(k, cap)].copy(), secs.value)

    def cp_step(self, rho, mx, my, phi, p=P2, safe=False):
        n = rho.shape[0] - 1
        omx = np.empty_like(mx)
        omy = np.empty_like(my)
        ophi = np.empty_like(phi)
        r = np.zeros(1)
        self._chk(self.L.ref_cp_step(n, _ptr(mx), _ptr(my), _ptr(phi), _ptr(rho), p,
                                     1 if safe else 0, _ptr(omx), _ptr(omy), _ptr(ophi), _ptr(r)))
        return omx, omy, ophi, float(r[0])

    def poisson_solve(self, b, projected=False):
        b = np.ascontiguousarray(b, dtype=np.float64)
        out = np.empty_like(b)
        self._chk(self.L.ref_poisson_solve(b.shape[0] - 1, _ptr(b), _ptr(out),
                                           1 if projected else 0))
        return out

    def project_affine(self, mx, my, rho):
        n = rho.shape[0] - 1
        ox = np.empty_like(mx)
        oy = np.empty_like(my)
        self._chk(self.L.ref_project_affine(n, _ptr(mx), _ptr(my), _ptr(rho), _ptr(ox), _ptr(oy)))
        return ox, oy
