"""Parity of the exact engine path behind the bench headline (config 4,
BASELINE.json configs[3]): batched 512^2 cascades on the AUTO engines -- the
three-sweep tensor-map kernel at the batched 512^2 level with tail compaction
and the stop replay, the streaming two-sweep kernel at 128^2/256^2 and the
cluster / resident engines on the coarse levels -- compared pair by pair
with the C oracle (bit-identical restatement of
/root/reference/proj/src/solver_cp.cpp:113-147, cascade per SPEC.md:365-373).

The device restriction splits every per-pair reduction by row count only, so
w1mg.ml_sources() of one pair returns the very bits the batch builds for it;
the oracle solves those sources.  Pairs whose per-level sweep counts agree
with the oracle must then carry bit-identical final fields.
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from paper_1810_00118_b200 import instances, w1mg

pytestmark = pytest.mark.gpu

LEVELS = 5


def _oracle_cascades(oracle, srcs, **kw):
    # ctypes releases the GIL: one oracle cascade per host thread
    with ThreadPoolExecutor(max_workers=min(len(srcs), 16)) as ex:
        return list(ex.map(lambda s: oracle.ml_cp_run(s, p=1, **kw), srcs))


def _device_sources(img0s, img1s):
    return [w1mg.ml_sources(img0s[b], img1s[b], LEVELS) for b in range(img0s.shape[0])]


@pytest.mark.parametrize("B", [2, 8])
def test_batched_512_converged_per_pair(oracle, B):
    """B pairs of config 4 (seeds 2i, 2i+1), rel tol 1e-5 per level: every
    pair's W1 within 1e-4 of its own oracle cascade, sweeps within +-1 per
    level, and bit-identical fields wherever the sweep counts agree."""
    img0s, img1s = instances.config4_pairs(0, B)
    dist, dual, iters, conv, mx, my, phi, fpr = w1mg.ml_run_batch_fields(
        img0s, img1s, LEVELS, p=w1mg.PNorm.p2, rel_tol=1e-5)
    assert conv.all()
    fin = iters[:, -1]
    if B > 2:
        assert fin.min() < fin.max()  # pairs stop on different sweeps: tail + compaction ran
    refs = _oracle_cascades(oracle, _device_sources(img0s, img1s), rel_tol=1e-5)
    exact = 0
    for b, ref in enumerate(refs):
        assert abs(dist[b] - ref.distance) <= 1e-4 * ref.distance, b
        assert all(abs(int(a) - c) <= 1 for a, c in zip(iters[b], ref.level_iters)), b
        if [int(x) for x in iters[b]] == ref.level_iters:
            exact += 1
            assert np.array_equal(mx[b], ref.mx), b
            assert np.array_equal(my[b], ref.my), b
            assert np.array_equal(phi[b], ref.phi), b
            assert abs(dist[b] - ref.distance) <= 1e-12 * ref.distance
            assert abs(dual[b] - ref.dual_value) <= 1e-10 * abs(ref.dual_value)
    # a +-1 sweep needs a residual within a few ulps of its tolerance; no pair
    # of this sample is that close
    assert exact == B


@pytest.mark.parametrize("k", [40, 41, 42])
def test_batched_512_fixed_sweeps_bit_exact(oracle, k):
    """Three pairs, every level run exactly k sweeps (stop rule off): the
    three-sweep launches end after sweep A (k = 40: replay 1), after sweep B
    (k = 41: replay 2) or on a launch boundary (k = 42); every pair's fields
    must match the oracle bit for bit."""
    B = 3
    img0s, img1s = instances.config4_pairs(5, B)
    eps = [-1.0] * LEVELS
    dist, dual, iters, conv, mx, my, phi, fpr = w1mg.ml_run_batch_fields(
        img0s, img1s, LEVELS, p=w1mg.PNorm.p2, eps=eps, max_iters=k)
    assert (iters == k).all()
    refs = _oracle_cascades(oracle, _device_sources(img0s, img1s), eps=eps, max_iters=k)
    for b, ref in enumerate(refs):
        assert np.array_equal(mx[b], ref.mx), b
        assert np.array_equal(my[b], ref.my), b
        assert np.array_equal(phi[b], ref.phi), b
        assert abs(dist[b] - ref.distance) <= 1e-12 * ref.distance
        assert fpr[b] == pytest.approx(ref.fpr_final, rel=1e-10)


def test_batch_results_independent_of_batch(oracle):
    """A pair's sources, sweeps, W1 and fields do not depend on which batch it
    is solved in (alone, or as pair 3 of 6)."""
    img0s, img1s = instances.config4_pairs(0, 6, m=256)
    big = w1mg.ml_run_batch_fields(img0s, img1s, 4, rel_tol=1e-5)
    one = w1mg.ml_run_batch_fields(img0s[3:4], img1s[3:4], 4, rel_tol=1e-5)
    assert big[0][3] == one[0][0]
    assert list(big[2][3]) == list(one[2][0])
    for f in (4, 5, 6):
        assert np.array_equal(big[f][3], one[f][0])
