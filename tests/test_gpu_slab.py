"""GPU parity of the row-slab decomposition (config 5): the fused sweep on
row slabs with a one-row halo exchange and a cross-slab residual sum must give
fields bit-identical to the undecomposed oracle.  Slabs are emulated on one
B200 with both transports (fused peer stores between the slabs, device-copy
halos), and the NCCL and peer transports are exercised with a single-rank
communicator (the multi-rank protocol itself is covered on CPU by
tests/test_slab_gloo.py)."""
import numpy as np
import pytest

from paper_1810_00118_b200 import instances
from paper_1810_00118_b200 import w1mg

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["peer", "copies"])
def transport(request):
    w1mg.set_slab_transport(request.param == "peer")
    yield request.param
    w1mg.set_slab_transport(True)


def _src(rho):
    return w1mg.SourceField(w1mg.ScalarField(w1mg.GridSpec(rho.shape[0] - 1), rho))


def _rand(n, seed):
    rng = np.random.default_rng(seed)
    return instances.make_source(rng.random((n + 1, n + 1)), rng.random((n + 1, n + 1)), n)


@pytest.mark.parametrize("nslabs", [1, 2, 3, 5])
@pytest.mark.parametrize("n", [64, 100, 257])
def test_slab_fixed_iterations_bit_exact(oracle, n, nslabs, transport):
    rho = _random = _rand(n, n + nslabs)
    prm = w1mg.SolverParams(p=w1mg.PNorm.p2, tolerance=-1.0, max_iters=75)
    rep = w1mg.slab_cp_run(_src(rho), prm, nslabs=nslabs)
    ref = oracle.cp_run(rho, p=1, tol=-1.0, max_iters=75)
    assert rep.iterations == 75
    assert np.array_equal(rep.flux.x_edges, ref.mx)
    assert np.array_equal(rep.flux.y_edges, ref.my)
    assert np.array_equal(rep.potential.values, ref.phi)
    assert abs(rep.distance - ref.distance) <= 1e-12 * ref.distance
    np.testing.assert_allclose(rep.residual_history, ref.residual_history, rtol=1e-10)


def test_slab_warm_start_and_converged(oracle):
    n = 96
    rho = instances.config1_source(n)
    rng = np.random.default_rng(0)
    m0 = (1e-3 * rng.standard_normal((n + 1, n)), 1e-3 * rng.standard_normal((n, n + 1)))
    phi0 = 1e-3 * rng.standard_normal((n + 1, n + 1))
    g = w1mg.GridSpec(n)
    prm = w1mg.SolverParams(p=w1mg.PNorm.p2, tolerance=1e-8, max_iters=200000)
    rep = w1mg.slab_cp_run(_src(rho), prm, nslabs=4, m0=w1mg.FluxField(g, *m0),
                           phi0=w1mg.ScalarField(g, phi0))
    ref = oracle.cp_run(rho, p=1, tol=1e-8, max_iters=200000, m0=m0, phi0=phi0)
    assert rep.converged and abs(rep.iterations - ref.iterations) <= 1
    assert abs(rep.distance - ref.distance) <= 1e-4 * ref.distance


def test_slab_4096_full_size(oracle, transport):
    """Config-5 finest grid in 8 slabs (the 8-GPU partition), 4 sweeps."""
    n = 4096
    rho = _rand(n, 4096)
    prm = w1mg.SolverParams(p=w1mg.PNorm.p2, tolerance=-1.0, max_iters=4)
    rep = w1mg.slab_cp_run(_src(rho), prm, nslabs=8)
    ref = oracle.cp_run(rho, p=1, tol=-1.0, max_iters=4)
    assert np.array_equal(rep.potential.values, ref.phi)
    assert np.array_equal(rep.flux.x_edges, ref.mx)
    assert np.array_equal(rep.flux.y_edges, ref.my)


def test_slab_nccl_single_rank(oracle):
    """The NCCL transport (send/recv/allreduce inside the CUDA graph) with a
    one-rank communicator: exercises the NCCL code path on one GPU."""
    uid = w1mg.SlabComm.new_unique_id()
    comm = w1mg.SlabComm(1, 0, uid)
    try:
        n = 128
        rho = _rand(n, 7)
        prm = w1mg.SolverParams(p=w1mg.PNorm.p2, tolerance=-1.0, max_iters=40)
        rep = w1mg.slab_cp_run(_src(rho), prm, comm=comm)
        ref = oracle.cp_run(rho, p=1, tol=-1.0, max_iters=40)
        assert np.array_equal(rep.potential.values, ref.phi)
        assert abs(rep.distance - ref.distance) <= 1e-12 * ref.distance
    finally:
        comm.close()


@pytest.mark.parametrize("nslabs", [1, 3, 8])
def test_ml_slab_cascade_bit_exact(oracle, nslabs, transport):
    """Config-5 shape at 512^2 (64 -> 512): replicated coarse levels + slab
    finest level, fixed sweeps per level: bit-exact against the oracle."""
    img0, img1 = instances.config5_images(m=512)
    rhos = instances.ml_sources(img0, img1, 4)
    eps = [-1.0] * 4
    rep = w1mg.ml_slab_run(rhos, nslabs=nslabs, eps=eps, max_iters=30)
    ref = oracle.ml_cp_run(rhos, p=1, eps=eps, max_iters=30)
    assert np.array_equal(rep.potential.values, ref.phi)
    assert np.array_equal(rep.flux.x_edges, ref.mx)
    assert np.array_equal(rep.flux.y_edges, ref.my)
    assert abs(rep.distance - ref.distance) <= 1e-12 * ref.distance
    assert [l.iters for l in rep.levels] == [30] * 4


@pytest.mark.parametrize("min_n", [128, 64])
@pytest.mark.parametrize("nslabs", [2, 5])
def test_ml_slab_cascade_partitions_every_large_level(oracle, nslabs, min_n, transport):
    """Every level with n >= slab_min_n is row-slab partitioned (SURVEY 8e:
    'the finest levels'), the slabs of one level gathered back to prolong
    into the next: still bit-exact at fixed sweeps, and converged W1 / sweeps
    as the oracle cascade."""
    from paper_1810_00118_b200 import _lib

    L = _lib.lib()
    assert L.w1mg_set_option(b"slab_min_n", min_n) == _lib.W1MG_OK
    try:
        img0, img1 = instances.config5_images(m=256)
        rhos = instances.ml_sources(img0, img1, 3)  # 64, 128, 256
        eps = [-1.0] * 3
        rep = w1mg.ml_slab_run(rhos, nslabs=nslabs, eps=eps, max_iters=25)
        ref = oracle.ml_cp_run(rhos, p=1, eps=eps, max_iters=25)
        assert np.array_equal(rep.potential.values, ref.phi)
        assert np.array_equal(rep.flux.x_edges, ref.mx)
        assert np.array_equal(rep.flux.y_edges, ref.my)
        assert [l.iters for l in rep.levels] == [25] * 3
        rep = w1mg.ml_slab_run(rhos, nslabs=nslabs, rel_tol=1e-5)
        ref = oracle.ml_cp_run(rhos, p=1, rel_tol=1e-5)
        assert abs(rep.distance - ref.distance) <= 1e-4 * ref.distance
        assert all(abs(a.iters - b) <= 1 for a, b in zip(rep.levels, ref.level_iters))
    finally:
        L.w1mg_set_option(b"slab_min_n", 1024)


def test_ml_slab_cascade_converged(oracle, transport):
    import time

    img0, img1 = instances.config5_images(m=256)
    rhos = instances.ml_sources(img0, img1, 3)
    t = time.perf_counter()
    rep = w1mg.ml_slab_run(rhos, nslabs=4, rel_tol=1e-5)
    # the host loop must notice the device-side stop (regression: a lost done
    # counter kept launching early-exit graphs up to the 5e6-sweep cap)
    assert time.perf_counter() - t < 20.0
    ref = oracle.ml_cp_run(rhos, p=1, rel_tol=1e-5)
    assert abs(rep.distance - ref.distance) <= 1e-4 * ref.distance
    assert all(abs(a.iters - b) <= 1 for a, b in zip(rep.levels, ref.level_iters))


def test_slab_peer_single_rank(oracle):
    """The peer transport on a communicator (IPC arena, mailbox, arrival
    counter; a one-rank world has no neighbours to map)."""
    uid = w1mg.SlabComm.new_unique_id()
    comm = w1mg.SlabComm(1, 0, uid)
    try:
        n = 128
        comm.enable_peer(n)
        rho = _rand(n, 9)
        for rep_i in range(2):  # arrival counting carries across runs
            prm = w1mg.SolverParams(p=w1mg.PNorm.p2, tolerance=-1.0, max_iters=40 + rep_i)
            rep = w1mg.slab_cp_run(_src(rho), prm, comm=comm)
            ref = oracle.cp_run(rho, p=1, tol=-1.0, max_iters=40 + rep_i)
            assert rep.iterations == 40 + rep_i
            assert np.array_equal(rep.potential.values, ref.phi)
            assert np.array_equal(rep.flux.x_edges, ref.mx)
        # a grid the arena is not laid out for (another level of a cascade)
        # runs on the NCCL transport of the same communicator
        r64 = _rand(64, 1)
        rep = w1mg.slab_cp_run(_src(r64), prm, comm=comm)
        ref = oracle.cp_run(r64, p=1, tol=-1.0, max_iters=prm.max_iters)
        assert np.array_equal(rep.potential.values, ref.phi)
    finally:
        comm.close()


def test_slab_bounds_partition():
    b = w1mg.slab_bounds(4096, 8)
    assert b[0] == 0 and b[-1] == 4097 and len(b) == 9
    assert all(b[r + 1] - b[r] in (512, 513) for r in range(8))
