"""Randomised parity (hypothesis): seeded random shapes, p-norms, sweep
counts, warm starts and engines, each checked bit-exactly against the CPU
oracle.  Complements the fixed cases of test_gpu_cp.py / test_gpu_ml.py with
shapes nobody picked by hand (odd/even n, strip and tile boundaries, stop
parities of the two-sweep engines, compaction buckets of batched levels)."""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from paper_1810_00118_b200 import instances
from paper_1810_00118_b200 import w1mg

pytestmark = pytest.mark.gpu

SETTINGS = dict(max_examples=30, deadline=None, derandomize=True,
                suppress_health_check=[HealthCheck.function_scoped_fixture])


def _src(rho):
    return w1mg.SourceField(w1mg.ScalarField(w1mg.GridSpec(rho.shape[0] - 1), rho))


def _rand_source(n, seed):
    rng = np.random.default_rng(seed)
    return instances.make_source(rng.random((n + 1, n + 1)), rng.random((n + 1, n + 1)), n)


# (resident engine, sweep engine) as in w1mg_set_resident_engine / _sweep_engine
ENGINE_PAIRS = [(1, 3), (0, 5), (0, 2), (0, 1), (3, 3), (0, 6)]


@settings(**{**SETTINGS, "max_examples": 200})
@given(n=st.integers(1, 300), p=st.sampled_from([0, 1, 2]), iters=st.integers(0, 41),
       seed=st.integers(0, 2**31 - 1), eng=st.sampled_from(ENGINE_PAIRS), warm=st.booleans())
def test_cp_fixed_sweeps_bit_exact(oracle, n, p, iters, seed, eng, warm):
    from paper_1810_00118_b200 import _lib

    L = _lib.lib()
    L.w1mg_set_resident_engine(eng[0])
    L.w1mg_set_sweep_engine(eng[1])
    try:
        rho = _rand_source(n, seed)
        m0 = phi0 = None
        if warm:
            rng = np.random.default_rng(seed + 1)
            m0 = (1e-3 * rng.standard_normal((n + 1, n)), 1e-3 * rng.standard_normal((n, n + 1)))
            phi0 = 1e-3 * rng.standard_normal((n + 1, n + 1))
        g = w1mg.GridSpec(n)
        prm = w1mg.SolverParams(p=w1mg.PNorm(p), tolerance=-1.0, max_iters=iters)
        rep = w1mg.cp_run(_src(rho), prm, None if m0 is None else w1mg.FluxField(g, *m0),
                          None if phi0 is None else w1mg.ScalarField(g, phi0))
        ref = oracle.cp_run(rho, p=p, tol=-1.0, max_iters=iters, m0=m0, phi0=phi0)
        assert rep.iterations == iters == ref.iterations
        assert np.array_equal(rep.flux.x_edges, ref.mx)
        assert np.array_equal(rep.flux.y_edges, ref.my)
        assert np.array_equal(rep.potential.values, ref.phi)
    finally:
        L.w1mg_set_resident_engine(1)
        L.w1mg_set_sweep_engine(3)


@settings(**SETTINGS)
@given(B=st.integers(1, 9), m=st.sampled_from([64, 96, 128, 192, 256]),
       levels=st.integers(1, 3), seed=st.integers(0, 10**6))
def test_batched_cascade_matches_single_pairs(oracle, B, m, levels, seed):
    """Batched cascades (compaction, per-pair stop) against the oracle cascade
    of each pair: W1 to 1e-9 (reassociated residuals may move a stop by one
    sweep, observed never) and per-level sweeps within +-1."""
    if m % (1 << (levels - 1)):
        return
    rng = np.random.default_rng(seed)
    img0 = rng.random((B, m, m)) + 0.1
    img1 = rng.random((B, m, m)) + 0.1
    dist, _, iters, conv = w1mg.ml_run_batch(img0, img1, levels, p=w1mg.PNorm.p2, rel_tol=1e-3)
    assert conv.all()
    for b in {0, B - 1}:
        rhos = instances.ml_sources(img0[b], img1[b], levels)
        ref = oracle.ml_cp_run(rhos, p=1, rel_tol=1e-3)
        assert abs(dist[b] - ref.distance) <= 1e-9 * abs(ref.distance)
        assert all(abs(int(a) - c) <= 1 for a, c in zip(iters[b], ref.level_iters))
