"""GPU parity of the level-persistent tile engine (tile_kernels.cuh): one
pair, the whole level in one launch, tiles in shared memory, the stop rule
read kTileLag sweeps late and the final state replayed from a checkpoint.
Fields after any fixed number of sweeps must be bit-identical to the CPU
oracle, and converged runs must stop at the same sweep with the same
residual history as the streaming engines."""
import numpy as np
import pytest

from paper_1810_00118_b200 import _lib, instances, w1mg

pytestmark = pytest.mark.gpu


@pytest.fixture(params=[1, 2], ids=["depth1", "depth2"])
def tile_engine(request):
    """Both tile kernels: one sweep per halo exchange and two (tile2_kernels)."""
    L = _lib.lib()
    L.w1mg_set_option(b"tile", 2)
    L.w1mg_set_option(b"tile_depth", request.param)
    yield
    L.w1mg_set_option(b"tile", 0)
    L.w1mg_set_option(b"tile_depth", 1)


def _src(rho):
    return w1mg.SourceField(w1mg.ScalarField(w1mg.GridSpec(rho.shape[0] - 1), rho))


def _random_source(n, seed):
    rng = np.random.default_rng(seed)
    return instances.make_source(rng.random((n + 1, n + 1)), rng.random((n + 1, n + 1)), n)


def _run(rho, p, iters, tol=-1.0, m0=None, phi0=None):
    g = w1mg.GridSpec(rho.shape[0] - 1)
    prm = w1mg.SolverParams(p=w1mg.PNorm(p), tolerance=tol, max_iters=iters)
    return w1mg.cp_run(_src(rho), prm, None if m0 is None else w1mg.FluxField(g, *m0),
                       None if phi0 is None else w1mg.ScalarField(g, phi0))


@pytest.mark.parametrize("iters", [1, 15, 16, 17, 33, 250])
@pytest.mark.parametrize("p", [0, 1, 2])
@pytest.mark.parametrize("n", [8, 47, 96, 130])
def test_tile_fixed_iterations_bit_exact(oracle, tile_engine, n, p, iters):
    rho = _random_source(n, 11 + n)
    rep = _run(rho, p, iters)
    ref = oracle.cp_run(rho, p=p, tol=-1.0, max_iters=iters)
    assert rep.iterations == iters
    assert np.array_equal(rep.flux.x_edges, ref.mx)
    assert np.array_equal(rep.flux.y_edges, ref.my)
    assert np.array_equal(rep.potential.values, ref.phi)
    assert abs(rep.distance - ref.distance) <= 1e-12 * abs(ref.distance)
    np.testing.assert_allclose(rep.residual_history, ref.residual_history, rtol=1e-10, atol=0)


@pytest.mark.parametrize("n", [256, 512])
def test_tile_full_size_bit_exact(oracle, tile_engine, n):
    rho = instances.config1_source(n)
    rep = _run(rho, 1, 123)
    ref = oracle.cp_run(rho, p=1, tol=-1.0, max_iters=123)
    assert np.array_equal(rep.flux.x_edges, ref.mx)
    assert np.array_equal(rep.flux.y_edges, ref.my)
    assert np.array_equal(rep.potential.values, ref.phi)


def test_tile_warm_start_bit_exact(oracle, tile_engine):
    n = 96
    rho = _random_source(n, 5)
    rng = np.random.default_rng(1)
    m0 = (rng.standard_normal((n + 1, n)) * 1e-3, rng.standard_normal((n, n + 1)) * 1e-3)
    phi0 = rng.standard_normal((n + 1, n + 1))
    rep = _run(rho, 1, 77, m0=m0, phi0=phi0)
    ref = oracle.cp_run(rho, p=1, tol=-1.0, max_iters=77, m0=m0, phi0=phi0)
    assert np.array_equal(rep.flux.x_edges, ref.mx)
    assert np.array_equal(rep.potential.values, ref.phi)


@pytest.mark.parametrize("n", [64, 128, 256])
def test_tile_converged_matches_streaming(tile_engine, n):
    """Same stop sweep, same residual history, same fields as the streaming
    two-sweep engine (the lagged stop rule replays to the exact sweep)."""
    rho = _random_source(n, 3)
    tol = 1e-4 * _run(rho, 1, 1).residual_history[0]  # R_cold-relative
    rep = _run(rho, 1, 200000, tol=tol)
    L = _lib.lib()
    L.w1mg_set_option(b"tile", 0)
    L.w1mg_set_resident_engine(0)
    try:
        ref = _run(rho, 1, 200000, tol=tol)
    finally:
        L.w1mg_set_resident_engine(1)
    assert rep.converged and ref.converged
    assert rep.iterations == ref.iterations
    assert np.array_equal(rep.flux.x_edges, ref.flux.x_edges)
    assert np.array_equal(rep.potential.values, ref.potential.values)
    np.testing.assert_allclose(rep.residual_history, ref.residual_history, rtol=1e-10, atol=0)


def test_tile_config2_cascade(oracle):
    """Config-2 cascade with the tile engine on its auto levels (128, 256):
    W1 within 1e-4 of the oracle, per-level sweeps equal."""
    rhos = instances.ml_sources(*instances.config2_images(m=256), 4)
    ml = w1mg.ml_run(rhos, p=w1mg.PNorm.p2, rel_tol=1e-5)
    mo = oracle.ml_cp_run(rhos, p=1, rel_tol=1e-5)
    assert abs(ml.distance - mo.distance) <= 1e-4 * abs(mo.distance)
    assert [lv.iters for lv in ml.levels] == list(mo.level_iters)
