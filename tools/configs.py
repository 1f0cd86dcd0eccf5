"""Time the five BASELINE.json configs on one B200 (and the CPU oracle where it
finishes in seconds).  One JSON line per config; the round's lines are kept in
profiles/.  Under torchrun (WORLD_SIZE > 1) only config 5 runs, one row slab
per rank over NCCL.

  python tools/configs.py [1 2 3 4 5]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1810_00118_b200 import _lib, instances, w1mg  # noqa: E402


def cu(levels):
    return float(sum(((round(1.0 / l.h)) + 1) ** 2 * l.iters for l in levels))


def line(**kw):
    print(json.dumps(kw), flush=True)


def config1(cpu=True):
    rho = instances.config1_source(64)
    src = w1mg.SourceField(w1mg.ScalarField(w1mg.GridSpec(64), rho))
    prm = w1mg.SolverParams(p=w1mg.PNorm.p2, tolerance=-1.0, max_iters=20000)
    w1mg.cp_run(src, prm)
    t = time.perf_counter()
    r = w1mg.cp_run(src, prm)
    wall = time.perf_counter() - t
    out = dict(config=1, what="N=64 single level, 20,000 sweeps (resident engine)",
               device_s=r.total_seconds, wall_s=wall, W1=r.distance,
               cell_updates_per_s=65 ** 2 * 20000 / r.total_seconds)
    if cpu:
        from oracle import Oracle

        t = time.perf_counter()
        o = Oracle().cp_run(rho, p=1, tol=-1.0, max_iters=20000)
        out.update(cpu_s=time.perf_counter() - t, cpu_W1=o.distance,
                   bit_exact=bool(np.array_equal(o.phi, r.potential.values)))
    line(**out)


def config2(cpu=True):
    rhos = instances.ml_sources(*instances.config2_images(m=256), 4)
    w1mg.ml_run(rhos, rel_tol=1e-5)
    t = time.perf_counter()
    r = w1mg.ml_run(rhos, rel_tol=1e-5)
    wall = time.perf_counter() - t
    out = dict(config=2, what="cascade 32->256, rel tol 1e-5", device_s=r.total_seconds,
               wall_s=wall, W1=r.distance, sweeps=[l.iters for l in r.levels],
               cell_updates_per_s=cu(r.levels) / r.total_seconds)
    if cpu:
        from oracle import Oracle

        t = time.perf_counter()
        o = Oracle().ml_cp_run(rhos, p=1, rel_tol=1e-5)
        out.update(cpu_s=time.perf_counter() - t, cpu_W1=o.distance, cpu_sweeps=o.level_iters,
                   rel_err=abs(o.distance - r.distance) / o.distance)
    line(**out)


def config3(cpu=False):
    from oracle import Oracle

    rhos = Oracle().ml_sources(*instances.config3_images(m=512), 5)
    w1mg.ml_pdhg_run(rhos, rel_tol=1e-5)
    t = time.perf_counter()
    r = w1mg.ml_pdhg_run(rhos, rel_tol=1e-5)
    wall = time.perf_counter() - t
    out = dict(config=3, what="G-prox PDHG cascade 32->512, rel tol 1e-5 (G_cold)",
               device_s=r.total_seconds, wall_s=wall, W1=r.distance, dual=r.dual_value,
               iters=[l.iters for l in r.levels], level_s=[l.seconds for l in r.levels])
    if cpu:
        from oracle import pdhg_oracle as PO

        t = time.perf_counter()
        o = PO.ml_pdhg_run(rhos, p=1, rel_tol=1e-5)
        out.update(cpu_s=time.perf_counter() - t, cpu_W1=o.distance, cpu_iters=o.level_iters,
                   rel_err=abs(o.distance - r.distance) / o.distance)
    line(**out)


def config5(nslabs=None):
    img0, img1 = instances.config5_images()
    rhos = instances.ml_sources(img0, img1, 7)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        import torch
        import torch.distributed as dist

        rank = int(os.environ["RANK"])
        dist.init_process_group("gloo")
        uid = w1mg.SlabComm.new_unique_id() if rank == 0 else None
        obj = [uid]
        dist.broadcast_object_list(obj, 0)
        comm = w1mg.SlabComm(world, rank, obj[0], device=int(os.environ.get("LOCAL_RANK", 0)))
        peer = os.environ.get("W1MG_SLAB_PEER", "1") != "0"
        if peer:  # fused P2P transport (IPC arenas over NVLink), else NCCL per sweep
            comm.enable_peer(4096, device=int(os.environ.get("LOCAL_RANK", 0)))
        r = w1mg.ml_slab_run(rhos, comm=comm, rel_tol=1e-5)
        t = torch.tensor([r.total_seconds], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            line(config=5, what=f"4096^2 cascade 64->4096, finest level in {world} slabs "
                 f"({'fused peer' if peer else 'NCCL'} transport)",
                 device_s=float(t.item()), W1=r.distance, iters=[l.iters for l in r.levels],
                 level_s=[l.seconds for l in r.levels])
        comm.close()
        dist.destroy_process_group()
        return
    if nslabs:
        for peer in (True, False):
            w1mg.set_slab_transport(peer)
            r = w1mg.ml_slab_run(rhos, nslabs=nslabs, rel_tol=1e-5)
            what = (f"4096^2 cascade 64->4096, finest level in {nslabs} emulated slabs (1 GPU, "
                    f"{'fused peer stores' if peer else 'device-copy halos'})")
            line(config=5, what=what, device_s=r.total_seconds, W1=r.distance,
                 iters=[l.iters for l in r.levels], level_s=[l.seconds for l in r.levels],
                 finest_sweep_us=1e6 * r.levels[-1].seconds / max(r.levels[-1].iters, 1))
        w1mg.set_slab_transport(True)
        return
    else:
        w1mg.ml_run(rhos[:3], rel_tol=1e-5)  # warm the small levels' engines
        r = w1mg.ml_run(rhos, rel_tol=1e-5)
        what = "4096^2 cascade 64->4096 (7 levels), rel tol 1e-5, 1 GPU"
    line(config=5, what=what, device_s=r.total_seconds, W1=r.distance,
         iters=[l.iters for l in r.levels], level_s=[l.seconds for l in r.levels],
         cell_updates_per_s=cu(r.levels) / r.total_seconds,
         finest_sweep_us=1e6 * r.levels[-1].seconds / max(r.levels[-1].iters, 1))


if __name__ == "__main__":
    which = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 5]
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        which = [5]
    for c in which:
        {1: config1, 2: config2, 3: config3, 5: config5}[c]()
    if 5 in which and int(os.environ.get("WORLD_SIZE", "1")) == 1:
        config5(nslabs=8)
