"""Host-side checks that need no GPU: the C-ABI library loads and exports
every symbol include/w1mg_cuda.h declares, generators are deterministic and
satisfy the source contract, the Python mirror's host-only pieces behave
like the reference."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "w1mg_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(w1mg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1810_00118_b200 import _lib

    L = _lib.lib()  # dlopen works without a GPU
    missing = [s for s in _declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    assert len(_declared_symbols()) >= 30


def test_library_nm_exports():
    so = os.path.join(ROOT, "paper_1810_00118_b200", "lib", "libw1mg_cuda.so")
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(l.split()[-1] for l in out.splitlines() if " T " in l)
    for s in _declared_symbols():
        assert s in exported, s


def test_pdhg_prime_factor_plan_tables():
    """Index tables of the register-stationary prime-factor DCT (513 = 27 x 19):
    bijective input map (Makhoul + Good-Thomas), CRT output map, W-build tables."""
    import ctypes as C

    from paper_1810_00118_b200 import _lib

    L = _lib.lib()
    bad = C.c_long(-1)
    assert L.w1mg_pdhg_plan_check(27, 19, C.byref(bad)) == 0
    assert bad.value == 0
    assert L.w1mg_pdhg_plan_check(13, 5, C.byref(bad)) != 0  # not instantiated


def test_cpp_api_library_exports_reference_entry_points():
    so = os.path.join(ROOT, "paper_1810_00118_b200", "lib", "libw1mg.so")
    out = subprocess.run(["nm", "-DC", "--defined-only", so], capture_output=True, text=True).stdout
    for sig in ["w1mg::cp_run(w1mg::SourceField const&, w1mg::SolverParams const&, "
                "w1mg::FluxField const*, w1mg::ScalarField const*)",
                "w1mg::cp_step(w1mg::CPState const&, w1mg::SourceField const&, w1mg::PNorm)",
                "w1mg::cp_residual(w1mg::CPState const&, w1mg::CPState const&)",
                "w1mg::pdhg_run(w1mg::SourceField const&, w1mg::SolverParams const&, "
                "w1mg::FluxField const*, w1mg::FluxField const*)",
                "w1mg::recover_potential(w1mg::FluxField const&)",
                "w1mg::NeumannPoissonSolver::solve_projected_into(w1mg::ScalarField const&, "
                "w1mg::ScalarField&) const",
                "w1mg::divergence(w1mg::FluxField const&)",
                "w1mg::primal_value(w1mg::FluxField const&, w1mg::PNorm)",
                "w1mg::ml_run("]:
        assert sig in out, sig


def test_step_sizes_and_schedule_host():
    from paper_1810_00118_b200 import _lib, w1mg

    L = _lib.lib()
    assert L.w1mg_cp_step_size(256, 1) == 1.0 / (2.0 * np.sqrt(2.0) / (1.0 / 256))
    assert L.w1mg_pdhg_step_size(0) == 0.5 and L.w1mg_pdhg_step_size(1) == 1.0
    assert w1mg.make_schedule(512, 3, 1e-6, -1.0) == [0.25e-6, 0.5e-6, 1e-6]
    assert w1mg.make_schedule(512, 3, 1e-6, 0.0) == [1e-6] * 3
    with pytest.raises(ValueError, match="divisible"):
        w1mg.make_schedule(96, 7, 1e-6)
    assert w1mg.default_levels(512) == 6


def test_engine_switches_validate_host():
    """Engine switches are host-only state: unknown names / values are
    W1MG_EINVAL, valid ones OK (defaults restored)."""
    from paper_1810_00118_b200 import _lib

    L = _lib.lib()
    assert L.w1mg_set_option(b"no_such_option", 1) == _lib.W1MG_EINVAL
    assert L.w1mg_set_option(b"tmap_nw", 3) == _lib.W1MG_EINVAL
    assert L.w1mg_set_option(b"pdhg_fold", 1) == _lib.W1MG_EINVAL  # engine removed
    assert L.w1mg_set_option(b"pdhg_small", 7) == _lib.W1MG_EINVAL
    assert L.w1mg_set_option(None, 1) == _lib.W1MG_EINVAL
    for name, val in ((b"tmap_nw", 4), (b"pdhg_small", 1), (b"compact", 1), (b"cluster_pick", 1)):
        assert L.w1mg_set_option(name, val) == _lib.W1MG_OK
    assert L.w1mg_set_option(b"tmap_nw", 0) == _lib.W1MG_OK  # back to auto
    for gone in (b"tile", b"tile_depth", b"tile_grid", b"pdhg_fold"):  # engines removed
        assert L.w1mg_set_option(gone, 1) == _lib.W1MG_EINVAL
    assert L.w1mg_set_sweep_engine(0) == _lib.W1MG_EINVAL  # LDG engine removed
    assert L.w1mg_set_sweep_engine(4) == _lib.W1MG_EINVAL  # two-column-set engine removed
    assert L.w1mg_set_sweep_engine(3) == _lib.W1MG_OK
    assert L.w1mg_set_resident_engine(4) == _lib.W1MG_EINVAL  # cooperative-grid engine removed
    assert L.w1mg_set_resident_engine(1) == _lib.W1MG_OK
    assert L.w1mg_set_sweep_engine(7) == _lib.W1MG_EINVAL
    assert L.w1mg_set_sweep_engine(6) == _lib.W1MG_OK  # three-sweep engine
    assert L.w1mg_set_sweep_engine(3) == _lib.W1MG_OK
    assert L.w1mg_set_pdhg_small(3) == _lib.W1MG_EINVAL
    assert L.w1mg_set_pdhg_small(1) == _lib.W1MG_OK


def test_source_gate_host():
    from paper_1810_00118_b200 import w1mg
    from paper_1810_00118_b200 import instances

    g = w1mg.GridSpec(8)
    with pytest.raises(ValueError, match="SourceField: values do not sum to zero"):
        w1mg.SourceField(w1mg.ScalarField(g, np.ones((9, 9))))
    w1mg.SourceField(w1mg.ScalarField(g, instances.config1_source(8)))


def test_prox_mirror_matches_oracle(oracle):
    from paper_1810_00118_b200 import w1mg

    rng = np.random.default_rng(0)
    for _ in range(500):
        v = tuple(rng.standard_normal(2) * 3)
        mu = float(rng.choice([0.1, 1.0, 10.0]))
        for p in (0, 1, 2):
            assert w1mg.shrink(v, mu, w1mg.PNorm(p)) == oracle.shrink(v, mu, p)
            assert w1mg.project_unit_ball(v, w1mg.PNorm(p)) == oracle.project_unit_ball(v, p)
            # Moreau: v = shrink(v) + proj_{mu q-ball}(v)
            s = w1mg.shrink(v, mu, w1mg.PNorm(p))
            q = w1mg.project_unit_ball((v[0] / mu, v[1] / mu), w1mg.conjugate(w1mg.PNorm(p)))
            assert abs(s[0] + mu * q[0] - v[0]) <= 1e-12 * (1 + abs(v[0]))
            assert abs(s[1] + mu * q[1] - v[1]) <= 1e-12 * (1 + abs(v[1]))
    with pytest.raises(ValueError, match="shrink: mu must be positive"):
        w1mg.shrink((1, 1), 0.0, w1mg.PNorm.p2)
    with pytest.raises(ValueError, match="p must be one of"):
        w1mg.pnorm_from_string("3")


def test_generators_deterministic_and_unit_mass():
    from paper_1810_00118_b200 import instances

    a = instances.blurred_noise_image(3, m=64)
    b = instances.blurred_noise_image(3, m=64)
    assert np.array_equal(a, b)
    assert abs(a.sum() - 1.0) <= 1e-12 and (a > 0).all()
    g0, g1 = instances.config2_images(m=32)
    assert abs(g0.sum() - 1) <= 1e-12 and abs(g1.sum() - 1) <= 1e-12
    rho = instances.config1_source(64)
    assert abs(rho.sum()) <= 1e-12 * np.abs(rho).sum()
    # unit mass in the L1_h sense: sum of the positive part times h^2 ~ W1 scale
    h = 1.0 / 64
    assert abs(np.abs(rho).sum() * h * h) <= 2.0 + 1e-9
    # blur operator: rows sum to 1 (normalised kernel, reflect boundary)
    B = instances._blur_matrix(64, 8.0)
    assert np.allclose(B.sum(axis=1), 1.0, atol=1e-14)


def test_multi_process_pair_sharding_gloo():
    """bench.py's multi-GPU path shards independent pairs with no data-path
    collective; the only collectives are a barrier and max/sum reductions of
    timings.  Exercised here with 2 gloo ranks on CPU."""
    import sys

    code = r"""
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, os.environ["ROOT"])
dist.init_process_group("gloo")
r, w = dist.get_rank(), dist.get_world_size()
import bench
B = 4
first = r * B
seeds = [2 * (first + i) for i in range(B)]
t = torch.tensor([float(r + 1)], dtype=torch.float64)
dist.all_reduce(t, op=dist.ReduceOp.MAX)
s = torch.tensor([float(B)], dtype=torch.float64)
dist.all_reduce(s)
assert t.item() == w and s.item() == B * w
g = [None] * w
dist.all_gather_object(g, seeds)
flat = [x for lst in g for x in lst]
assert len(set(flat)) == len(flat) == B * w
dist.destroy_process_group()
print("ok", r)
"""
    env = dict(os.environ, ROOT=ROOT, MASTER_ADDR="127.0.0.1", MASTER_PORT="29533",
               WORLD_SIZE="2")
    procs = [subprocess.Popen([sys.executable, "-c", code],
                              env=dict(env, RANK=str(r), LOCAL_RANK=str(r)),
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(2)]
    outs = [p.communicate(timeout=300)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), outs


def test_norm_plain_matches_reference_order():
    """norm_plain (grid.cpp:117-128) is the unweighted Neumaier norm, bit for
    bit (round 1 computed sqrt(inner_h)/h, which rounds through h^2)."""
    import math

    import numpy as np

    from paper_1810_00118_b200 import w1mg

    rng = np.random.default_rng(9)
    g = w1mg.GridSpec(7)
    phi = w1mg.ScalarField(g, rng.standard_normal((8, 8)))
    s = c = 0.0
    for x in phi.values.ravel().tolist():
        y = x * x
        t = s + y
        c += (s - t) + y if abs(s) >= abs(y) else (y - t) + s
        s = t
    assert w1mg.norm_plain(phi) == math.sqrt(s + c)
