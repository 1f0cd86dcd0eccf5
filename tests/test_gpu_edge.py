"""Edge cases of the GPU path (SPEC.md error conventions and degenerate
inputs), each compared with the reference semantics."""
import math

import numpy as np
import pytest

from paper_1810_00118_b200 import instances
from paper_1810_00118_b200 import w1mg

pytestmark = pytest.mark.gpu


def _src(rho):
    return w1mg.SourceField(w1mg.ScalarField(w1mg.GridSpec(rho.shape[0] - 1), rho))


def test_zero_iterations_returns_initial_state(oracle):
    """max_iters = 0: the while loop of solver_cp.cpp:128 never runs."""
    n = 16
    rho = instances.config1_source(n)
    rng = np.random.default_rng(0)
    m0 = (rng.standard_normal((n + 1, n)), rng.standard_normal((n, n + 1)))
    g = w1mg.GridSpec(n)
    rep = w1mg.cp_run(_src(rho), w1mg.SolverParams(p=w1mg.PNorm.p2, max_iters=0),
                      w1mg.FluxField(g, *m0))
    ref = oracle.cp_run(rho, p=1, max_iters=0, m0=m0)
    assert rep.iterations == 0 and not rep.converged
    assert np.array_equal(rep.flux.x_edges, m0[0])
    assert abs(rep.distance - ref.distance) <= 1e-12 * ref.distance


def test_huge_tolerance_stops_after_one_sweep(oracle):
    """The loop always performs >= 1 sweep."""
    rho = instances.config1_source(16)
    rep = w1mg.cp_run(_src(rho), w1mg.SolverParams(p=w1mg.PNorm.p2, tolerance=1e30))
    assert rep.iterations == 1 and rep.converged
    assert len(rep.residual_history) == 1


@pytest.mark.parametrize("p", [0, 2])
def test_cascade_other_pnorms_bit_exact(oracle, p):
    rhos = instances.ml_sources(*instances.config2_images(m=64), 3)
    eps = [-1.0] * 3
    rep = w1mg.ml_run(rhos, p=w1mg.PNorm(p), eps=eps, max_iters=90)
    ref = oracle.ml_cp_run(rhos, p=p, eps=eps, max_iters=90)
    assert np.array_equal(rep.potential.values, ref.phi)
    assert np.array_equal(rep.flux.x_edges, ref.mx)


def test_batch_single_pair_single_level(oracle):
    img0, img1 = instances.config4_pairs(0, 1, m=32)
    dist, dual, iters, conv = w1mg.ml_run_batch(img0, img1, 1, rel_tol=1e-5)
    rho = instances.ml_sources(img0[0], img1[0], 1)[0]
    step = oracle.cp_step_size(32)
    tol = 1e-5 * step * ((1.0 / 32) ** 2 * oracle.compensated_sum((rho * rho).ravel()))
    ref = oracle.cp_run(rho, p=1, tol=tol, max_iters=5_000_000)
    assert conv[0] and abs(int(iters[0, 0]) - ref.iterations) <= 1
    assert abs(dist[0] - ref.distance) <= 1e-4 * ref.distance


def test_cascade_divisibility_error():
    rhos = [np.zeros((13, 13)), np.zeros((25, 25))]  # 12 -> 24 is fine
    w1mg.ml_run(rhos, eps=[1.0, 1.0], max_iters=1)
    with pytest.raises(ValueError, match="divisible"):  # 5 cells cannot be halved
        w1mg.ml_run([np.zeros((3, 3)), np.zeros((6, 6))], eps=[1.0, 1.0], max_iters=1)


def test_grid_mismatch_errors():
    g8, g4 = w1mg.GridSpec(8), w1mg.GridSpec(4)
    with pytest.raises(ValueError, match="cp_run: grid mismatch"):
        w1mg.cp_run(_src(instances.config1_source(8)), w1mg.SolverParams(), w1mg.FluxField(g4))
    with pytest.raises(ValueError, match="grid mismatch"):
        w1mg.inner_h(w1mg.ScalarField(g8), w1mg.ScalarField(g4))


def test_bad_pnorm_is_logic_error():
    rho = instances.config1_source(8)
    with pytest.raises(AssertionError, match="bad PNorm"):
        w1mg.cp_run(_src(rho), w1mg.SolverParams(p=7, max_iters=2))


def test_nonfinite_source_stops_and_reports():
    """A NaN in rho: the device flags the non-finite residual and stops (the
    reference would keep iterating on NaNs until max_iters)."""
    rho = instances.config1_source(16)
    rho[3, 3] = math.nan
    src = w1mg.SourceField.__new__(w1mg.SourceField)  # bypass the zero-sum gate
    src.rho = w1mg.ScalarField(w1mg.GridSpec(16), rho)
    rep = w1mg.cp_run(src, w1mg.SolverParams(p=w1mg.PNorm.p2, max_iters=1000))
    assert not rep.converged and rep.iterations <= 1000
    assert math.isnan(rep.distance) or math.isnan(rep.residual_history[-1])


def test_large_batch_many_levels_smoke():
    """64 pairs x 4 levels through the batch API: every pair converges and the
    W1 values are finite and positive."""
    img0, img1 = instances.config4_pairs(10, 64, m=128)
    dist, dual, iters, conv = w1mg.ml_run_batch(img0, img1, 4, rel_tol=1e-5)
    assert conv.all() and np.isfinite(dist).all() and (dist > 0).all()
    assert (dual < 0).all()  # CP dual value ~ -W1


def test_step_size_outside_supported_range_fails_loudly():
    """The branch-free shrink needs mu^2 inside the fp64 fast-path range:
    a custom mu outside [1e-140, 1e140] is refused with W1MG_EINVAL instead
    of computing silently wrong fluxes (the reference accepts any mu > 0)."""
    from paper_1810_00118_b200 import w1mg as W

    rho = instances.config1_source(16)
    with pytest.raises(Exception, match="supported range"):
        W._cp_call(16, rho, None, None, None, 1, 1e-150, 1e-150, -1.0, 5, 0)
