"""GPU parity for the G-prox PDHG path (Algorithm 2/4), the Neumann Poisson
solve and the affine projection, against oracle/pdhg_oracle.py (numpy +
scipy DCT) -- itself pinned to the reference poisson.cpp in
tests/test_oracle_vs_ref.py.  The DCT is computed differently on the GPU
(prime-factor DCT kernels, dct_kernels.cuh, vs scipy's FFT), so fields agree
to rounding, not bit for bit:
tolerance 1e-9 relative at fixed iterations (BASELINE.json), 1e-4 on W1 at
convergence."""
import numpy as np
import pytest

from oracle import pdhg_oracle as PO
from paper_1810_00118_b200 import instances
from paper_1810_00118_b200 import w1mg

pytestmark = pytest.mark.gpu

FIELD_TOL = 1e-9


def _rel(a, b):
    return np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300)


def _src(rho):
    return w1mg.SourceField(w1mg.ScalarField(w1mg.GridSpec(rho.shape[0] - 1), rho))


# m = n+1 covers every DCT plan shape: prime (5, 257), even with a Nyquist
# row (9 -> 9, 100 -> 101 prime, 31 -> 32 = 2^5, 47 -> 48 = 16 x 3, 63 -> 64),
# two coprime factors with odd/even parts (33 = 11 x 3, 65 = 13 x 5,
# 129 = 43 x 3, 513 = 27 x 19, 1025 = 41 x 25, 2049 = 683 x 3)
@pytest.mark.parametrize("n", [1, 4, 8, 31, 32, 47, 63, 64, 100, 128, 256, 512, 1024, 2048])
def test_poisson_solve_matches_oracle(n):
    rng = np.random.default_rng(n)
    b = rng.standard_normal((n + 1, n + 1))
    b -= b.mean()
    g = w1mg.GridSpec(n)
    s = w1mg.NeumannPoissonSolver(g)
    out = s.solve(w1mg.ScalarField(g, b))
    ref = PO.poisson_solve_projected(b)
    assert _rel(out.values, ref) <= 1e-11
    # residual contract: ||A A* phi - b|| <= 1e-10 ||b||
    aa = w1mg.divergence(w1mg.adjoint(out))
    assert np.linalg.norm(aa.values - b) <= 1e-10 * np.linalg.norm(b)
    assert abs(out.values.mean()) <= 1e-12


def test_poisson_compatibility_guard():
    g = w1mg.GridSpec(8)
    with pytest.raises(ValueError, match="right-hand side must sum to zero"):
        w1mg.NeumannPoissonSolver(g).solve(w1mg.ScalarField(g, np.ones((9, 9))))


@pytest.mark.parametrize("n", [8, 64])
def test_project_affine(n):
    rng = np.random.default_rng(3)
    mx, my = rng.standard_normal((n + 1, n)), rng.standard_normal((n, n + 1))
    rho = instances.make_source(rng.random((n + 1, n + 1)), rng.random((n + 1, n + 1)), n)
    g = w1mg.GridSpec(n)
    out = w1mg.project_affine(w1mg.NeumannPoissonSolver(g), w1mg.FluxField(g, mx, my), _src(rho))
    rx, ry = PO.project_affine(mx, my, rho)
    assert _rel(out.x_edges, rx) <= 1e-11 and _rel(out.y_edges, ry) <= 1e-11
    # feasibility and idempotence
    assert np.linalg.norm(w1mg.divergence(out).values - rho) <= 1e-10 * (1 + np.linalg.norm(rho))
    again = w1mg.project_affine(w1mg.NeumannPoissonSolver(g), out, _src(rho))
    assert _rel(again.x_edges, out.x_edges) <= 1e-10


@pytest.fixture(params=["streaming", "persistent", "resident", "rowres", "rowres_pfa", "auto"])
def pdhg_engine(request):
    """streaming: 3-launch iteration (row DCT-II + pre, column DCT-II /
    divide / DCT-III, row DCT-III + post); persistent: every iteration of a
    one-pair level in one cooperative launch (pdhg_persist.cuh); resident:
    one CTA per pair for m <= 65, persistent above; rowres: the row-resident
    persistent engine (pdhg_rs.cuh) at every size, dense register-stationary
    DCT for odd m <= 129; rowres_pfa: the same with the prime-factor
    transforms everywhere; auto: the defaults."""
    from paper_1810_00118_b200 import _lib

    L = _lib.lib()
    rs = {"rowres": 3, "rowres_pfa": 2, "auto": 1}.get(request.param, 0)
    if request.param != "auto":
        L.w1mg_set_pdhg_small(2 if request.param == "resident" else 0)
        L.w1mg_set_option(b"pdhg_persist", 0 if request.param == "streaming" else 1)
    L.w1mg_set_option(b"pdhg_rs", rs)
    yield request.param
    L.w1mg_set_pdhg_small(1)
    L.w1mg_set_option(b"pdhg_persist", 1)
    L.w1mg_set_option(b"pdhg_rs", 1)


@pytest.mark.parametrize("n", [31, 32, 48, 64, 100, 128, 150, 256])
@pytest.mark.parametrize("p", [0, 1, 2])
def test_pdhg_fixed_iterations(p, n, pdhg_engine):
    rho = instances.config1_source(n)
    prm = w1mg.SolverParams(p=w1mg.PNorm(p), tolerance=-1.0, max_iters=200)
    rep = w1mg.pdhg_run(_src(rho), prm)
    ref = PO.pdhg_run(rho, p=p, tol=-1.0, max_iters=200)
    assert rep.iterations == 200
    assert _rel(rep.flux.x_edges, ref.mx) <= FIELD_TOL
    assert _rel(rep.flux.y_edges, ref.my) <= FIELD_TOL
    assert _rel(rep.dual_flux.x_edges, ref.px) <= FIELD_TOL
    assert _rel(rep.potential.values, ref.phi) <= FIELD_TOL
    assert abs(rep.distance - ref.distance) <= FIELD_TOL * ref.distance
    np.testing.assert_allclose(rep.residual_history, ref.residual_history, rtol=1e-7)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 8, 9, 17])
def test_pdhg_tiny_grids(n, pdhg_engine):
    """Every engine on grids of a few nodes (m = 2 ... 18: one or two CTAs,
    even and odd m, h = (m-1)/2 below one thread tile)."""
    rng = np.random.default_rng(n)
    rho = instances.make_source(rng.random((n + 1, n + 1)) + 0.1, rng.random((n + 1, n + 1)) + 0.1, n)
    prm = w1mg.SolverParams(p=w1mg.PNorm.p2, tolerance=-1.0, max_iters=50)
    rep = w1mg.pdhg_run(_src(rho), prm)
    ref = PO.pdhg_run(rho, p=1, tol=-1.0, max_iters=50)
    assert rep.iterations == 50
    assert _rel(rep.flux.x_edges, ref.mx) <= FIELD_TOL
    assert _rel(rep.flux.y_edges, ref.my) <= FIELD_TOL
    assert _rel(rep.dual_flux.x_edges, ref.px) <= FIELD_TOL
    np.testing.assert_allclose(rep.residual_history, ref.residual_history, rtol=1e-7, atol=1e-300)


@pytest.mark.parametrize("rs", [0, 1])
def test_pdhg_fixed_iterations_finest(rs):
    """Config 3's finest level (m = 513 = 27 x 19): the register-stationary
    prime-factor engine (pdhg_rspf.cuh, rs = 1) and the previous persistent
    engine (rs = 0) against the numpy oracle."""
    from paper_1810_00118_b200 import _lib

    L = _lib.lib()
    L.w1mg_set_option(b"pdhg_rs", rs)
    try:
        n = 512
        rho = instances.config1_source(n)
        prm = w1mg.SolverParams(p=w1mg.PNorm.p2, tolerance=-1.0, max_iters=100)
        rep = w1mg.pdhg_run(_src(rho), prm)
        ref = PO.pdhg_run(rho, p=1, tol=-1.0, max_iters=100)
        assert rep.iterations == 100
        assert _rel(rep.flux.x_edges, ref.mx) <= FIELD_TOL
        assert _rel(rep.flux.y_edges, ref.my) <= FIELD_TOL
        assert _rel(rep.dual_flux.x_edges, ref.px) <= FIELD_TOL
        assert _rel(rep.potential.values, ref.phi) <= FIELD_TOL
        np.testing.assert_allclose(rep.residual_history, ref.residual_history, rtol=1e-7)
    finally:
        L.w1mg_set_option(b"pdhg_rs", 1)


def test_pdhg_converged_config1_like():
    """SURVEY finding 9: N=32, p=2 -> W1 = 0.5053635, recovered dual ~ +W1."""
    rho = instances.config1_source(32)
    rep = w1mg.pdhg_run(_src(rho), w1mg.SolverParams(p=w1mg.PNorm.p2, tolerance=1e-11,
                                                    max_iters=20000))
    assert rep.distance == pytest.approx(0.5053635159441875, rel=1e-6)
    assert rep.dual_value == pytest.approx(rep.distance, rel=1e-5)
    # pointwise dual feasibility
    d = rep.dual_flux
    X = np.zeros((33, 33)); Y = np.zeros((33, 33))
    X[:, :32] = d.x_edges; Y[:32, :] = d.y_edges
    assert np.sqrt(X * X + Y * Y).max() <= 1 + 1e-12


def test_pdhg_step_and_residual():
    n = 16
    rho = instances.config1_source(n)
    g = w1mg.GridSpec(n)
    s0 = w1mg.pdhg_init(g, w1mg.StepMode.safe, w1mg.FluxField(g), w1mg.FluxField(g))
    s1 = w1mg.pdhg_step(s0, _src(rho), w1mg.PNorm.p2)
    s2 = w1mg.pdhg_step(s1, _src(rho), w1mg.PNorm.p2)
    o0 = PO.pdhg_init(n, safe=True)
    o1 = PO.pdhg_step(o0, rho, 1)
    o2 = PO.pdhg_step(o1, rho, 1)
    assert _rel(s2.m.x_edges, o2.mx) <= FIELD_TOL
    assert _rel(s2.dual_flux_bar.y_edges, o2.by) <= FIELD_TOL
    r = w1mg.pdhg_residual(s2, s1)
    assert r == pytest.approx(PO.pdhg_residual(o2, o1, n), rel=1e-9)
    assert r >= 0.0  # SPEC.md:289 (mu = tau = 1/2)


def test_recover_potential_inverts_adjoint():
    """varphi = A* psi -> recover_potential = psi - mean(psi)."""
    n = 24
    psi = np.random.default_rng(5).standard_normal((n + 1, n + 1))
    g = w1mg.GridSpec(n)
    phi = w1mg.recover_potential(w1mg.adjoint(w1mg.ScalarField(g, psi)))
    assert np.linalg.norm(phi.values - (psi - psi.mean())) <= 1e-9


def test_config3_cascade_matches_oracle(pdhg_engine):
    """BASELINE.json configs[2] at reduced size (cascade 32->128 from a 128^2
    blurred-noise image pair), rel tol 1e-5 per level."""
    from oracle import Oracle

    img0 = instances.blurred_noise_image(0, m=128)
    img1 = instances.blurred_noise_image(1, m=128)
    rhos = Oracle().ml_sources(img0, img1, 3)
    rep = w1mg.ml_pdhg_run(rhos, p=w1mg.PNorm.p2, rel_tol=1e-5)
    ref = PO.ml_pdhg_run(rhos, p=1, rel_tol=1e-5)
    assert abs(rep.distance - ref.distance) <= 1e-4 * ref.distance
    for a, b in zip([l.iters for l in rep.levels], ref.level_iters):
        assert abs(a - b) <= max(2, 0.02 * b)
