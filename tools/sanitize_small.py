"""Small solves that drive the kernels compute-sanitizer checks (SURVEY §4
item 5): the three-sweep tensor-map kernel (batched 400^2 level, stop
replays), the two-sweep tensor-map kernel, the cluster engine (DSMEM halos,
cluster barriers), the emulated row-slab peer transport (peer stores,
mailbox, arrival counters) and the PDHG DCT kernels.  Each solve is checked
against the oracle so a sanitizer run also proves the results are right.

  compute-sanitizer --tool racecheck python tools/sanitize_small.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import Oracle  # noqa: E402
from paper_1810_00118_b200 import _lib, instances, w1mg  # noqa: E402

O = Oracle()
L = _lib.lib()


def cp(n, iters, resident=1, engine=3, B=1):
    L.w1mg_set_resident_engine(resident)
    L.w1mg_set_sweep_engine(engine)
    try:
        rng = np.random.default_rng(n)
        rho = instances.make_source(rng.random((n + 1, n + 1)), rng.random((n + 1, n + 1)), n)
        src = w1mg.SourceField(w1mg.ScalarField(w1mg.GridSpec(n), rho))
        rep = w1mg.cp_run(src, w1mg.SolverParams(p=w1mg.PNorm.p2, tolerance=-1.0, max_iters=iters))
    finally:
        L.w1mg_set_resident_engine(1)
        L.w1mg_set_sweep_engine(3)
    ref = O.cp_run(rho, p=1, tol=-1.0, max_iters=iters)
    assert np.array_equal(rep.potential.values, ref.phi), (n, engine, resident)
    print(f"cp n={n} engine={engine} resident={resident} ok", flush=True)


def batch(n, B, iters):
    img0s, img1s = instances.config4_pairs(0, B, m=n)
    out = w1mg.ml_run_batch_fields(img0s, img1s, 2, eps=[-1.0, -1.0], max_iters=iters)
    for b in range(B):
        ref = O.ml_cp_run(w1mg.ml_sources(img0s[b], img1s[b], 2), p=1, eps=[-1.0, -1.0],
                          max_iters=iters)
        assert np.array_equal(out[6][b], ref.phi), (n, b)
    print(f"batch n={n} B={B} ok", flush=True)


def slab(n, nslabs, iters):
    rng = np.random.default_rng(3)
    rho = instances.make_source(rng.random((n + 1, n + 1)), rng.random((n + 1, n + 1)), n)
    src = w1mg.SourceField(w1mg.ScalarField(w1mg.GridSpec(n), rho))
    prm = w1mg.SolverParams(p=w1mg.PNorm.p2, tolerance=-1.0, max_iters=iters)
    rep = w1mg.slab_cp_run(src, prm, nslabs=nslabs)
    ref = O.cp_run(rho, p=1, tol=-1.0, max_iters=iters)
    assert np.array_equal(rep.potential.values, ref.phi)
    print(f"slab n={n} slabs={nslabs} ok", flush=True)


def pdhg(n, iters):
    from oracle import pdhg_oracle as PO

    rho = instances.config1_source(n)
    src = w1mg.SourceField(w1mg.ScalarField(w1mg.GridSpec(n), rho))
    rep = w1mg.pdhg_run(src, w1mg.SolverParams(p=w1mg.PNorm.p2, tolerance=-1.0, max_iters=iters))
    ref = PO.pdhg_run(rho, p=1, tol=-1.0, max_iters=iters)
    err = np.linalg.norm(rep.flux.x_edges - ref.mx) / np.linalg.norm(ref.mx)
    assert err <= 1e-9, err
    print(f"pdhg n={n} ok", flush=True)


if __name__ == "__main__":
    what = sys.argv[1:] or ["cp", "batch", "slab", "pdhg"]
    if "cp" in what:
        cp(200, 7, resident=0, engine=6)   # three-sweep, replay 1
        cp(130, 5, resident=0, engine=5)   # two-sweep tensor map, replay
        cp(64, 9, resident=3)              # cluster engine
        cp(40, 9, resident=0, engine=1)    # one-sweep TMA
    if "batch" in what:
        batch(400, 3, 8)                   # batched three-sweep + replay 2
    if "slab" in what:
        slab(96, 3, 6)                     # emulated slabs, fused peer stores
    if "pdhg" in what:
        pdhg(64, 5)                        # DCT kernels (m = 65 = 13 x 5)
