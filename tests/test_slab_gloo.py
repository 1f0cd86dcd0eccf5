"""Config-5 row-slab decomposition, multi-process on CPU (gloo, world 2 and 3).

Each rank owns node rows [bounds[r], bounds[r+1]) of one grid (the same
partition as w1mg_slab_bounds), runs the slab view of the CP sweep
(oracle.cp_sweep_rows), exchanges the one-row halos with torch.distributed
send/recv (row jhi-1 of phi, m_x, m_y up; row jlo of phi down) and all-reduces
the three residual sums before applying the stop rule -- the same protocol the
NCCL transport of slab_engine.cuh runs on the GPUs.  The assembled fields
must be bit-identical to the undecomposed oracle, and the stop iteration
equal.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import os, sys
import numpy as np
import torch, torch.distributed as dist
sys.path.insert(0, os.environ["ROOT"])
from oracle import Oracle
from paper_1810_00118_b200 import instances

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
n, iters, tol = int(os.environ["N"]), int(os.environ["ITERS"]), float(os.environ["TOL"])
O = Oracle()
bounds = [(n + 1) * r // world for r in range(world + 1)]   # == w1mg_slab_bounds
jlo, jhi = bounds[rank], bounds[rank + 1]
rho = instances.config1_source(n)
step = O.cp_step_size(n)
h2 = (1.0 / n) ** 2
st = [[np.zeros((n + 1, n)), np.zeros((n, n + 1)), np.zeros((n + 1, n + 1))] for _ in range(2)]

def send_row(a, row, dst):
    dist.send(torch.from_numpy(np.ascontiguousarray(a[row])), dst)

def recv_row(a, row, src):
    t = torch.empty(a.shape[1], dtype=torch.float64)
    dist.recv(t, src)
    a[row] = t.numpy()

k, conv, hist = 0, False, []
while k < iters:
    (mx, my, phi), (omx, omy, ophi) = st[k % 2], st[(k + 1) % 2]
    sums = O.cp_sweep_rows(n, jlo, jhi, mx, my, phi, rho, 1, step, step, omx, omy, ophi)
    # halo exchange of the new state (ordered to avoid deadlock)
    if rank + 1 < world:
        send_row(ophi, jhi - 1, rank + 1); send_row(omx, jhi - 1, rank + 1)
        if jhi - 1 < n: send_row(omy, jhi - 1, rank + 1)
        recv_row(ophi, jhi, rank + 1)
    if rank > 0:
        recv_row(ophi, jlo - 1, rank - 1); recv_row(omx, jlo - 1, rank - 1)
        if jlo - 1 < n: recv_row(omy, jlo - 1, rank - 1)
        send_row(ophi, jlo, rank - 1)
    t = torch.from_numpy(sums)
    dist.all_reduce(t)
    s = t.numpy()
    fpr = h2 * (s[0] / step + s[1] / step - 2.0 * s[2])
    hist.append(fpr)
    k += 1
    if fpr < tol:
        conv = True
        break
mx, my, phi = st[k % 2]
ref = O.cp_run(rho, p=1, tol=tol, max_iters=iters)
assert k == ref.iterations, (k, ref.iterations)
assert np.array_equal(phi[jlo:jhi], ref.phi[jlo:jhi])
assert np.array_equal(mx[jlo:jhi], ref.mx[jlo:jhi])
assert np.array_equal(my[jlo:min(jhi, n)], ref.my[jlo:min(jhi, n)])
np.testing.assert_allclose(hist, ref.residual_history, rtol=1e-12)
dist.destroy_process_group()
print("rank", rank, "ok", k)
"""


def _launch(world, n, iters, tol, port):
    env = dict(os.environ, ROOT=ROOT, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
               WORLD_SIZE=str(world), N=str(n), ITERS=str(iters), TOL=repr(tol))
    procs = [subprocess.Popen([sys.executable, "-c", WORKER],
                              env=dict(env, RANK=str(r), LOCAL_RANK=str(r)),
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(world)]
    outs = [p.communicate(timeout=600)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), "\n".join(outs)


@pytest.mark.parametrize("world", [2, 3])
def test_slab_fixed_iterations(world):
    _launch(world, n=24, iters=40, tol=-1.0, port=29610 + world)


def test_slab_converged_stop():
    _launch(2, n=16, iters=200000, tol=1e-7, port=29620)



# --------------------------------------------------------------------------
# The fused peer transport (slab_engine.cuh, default): no messages.  Each rank
# stores its boundary rows straight into the neighbours' arrays ("peer
# memory": shared memory here, NVLink P2P on the GPUs), posts its residual
# sums into slot [k & 1][rank] of every rank's mailbox, then signals arrival,
# and waits for all ranks' arrivals of sweep k before reducing its own
# mailbox in rank order.  The GPU counts arrivals on one counter with
# atomicAdd_system; here every (receiver, sender) pair has its own sequence
# slot (single writer, no atomics needed) -- the same "all ranks posted sweep
# k" condition.  Ranks run freely, so this also exercises the ordering
# argument: mailbox parity buffering and ping-pong halo rows never race.
PEER_WORKER = r"""
import os, sys, time
import numpy as np
from multiprocessing import resource_tracker, shared_memory
sys.path.insert(0, os.environ["ROOT"])
from oracle import Oracle
from paper_1810_00118_b200 import instances

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
n, iters, tol = int(os.environ["N"]), int(os.environ["ITERS"]), float(os.environ["TOL"])
tag = os.environ["TAG"]
O = Oracle()
bounds = [(n + 1) * r // world for r in range(world + 1)]
jlo, jhi = bounds[rank], bounds[rank + 1]
rho = instances.config1_source(n)
step = O.cp_step_size(n)
h2 = (1.0 / n) ** 2
shapes = [(n + 1, n), (n, n + 1), (n + 1, n + 1)]
per_rank = 2 * sum(a * b for a, b in shapes) + 2 * world * 3 + world

def views(r):
    shm = shared_memory.SharedMemory(name=f"{tag}_{r}")
    resource_tracker.unregister(shm._name, "shared_memory")  # the parent owns the segment
    buf = np.ndarray((per_rank,), dtype=np.float64, buffer=shm.buf)
    out, off = [], 0
    for p in range(2):
        trip = []
        for a, b in shapes:
            trip.append(buf[off:off + a * b].reshape(a, b)); off += a * b
        out.append(trip)
    mail = buf[off:off + 2 * world * 3].reshape(2, world, 3); off += 2 * world * 3
    seq = buf[off:off + world]
    return shm, out, mail, seq

shms, st, mails, seqs = zip(*[views(r) for r in range(world)])
mine = st[rank]
k, hist = 0, []
while k < iters:
    (mx, my, phi), (omx, omy, ophi) = mine[k % 2], mine[(k + 1) % 2]
    sums = O.cp_sweep_rows(n, jlo, jhi, mx, my, phi, rho, 1, step, step, omx, omy, ophi)
    w = (k + 1) % 2
    if rank + 1 < world:   # top owned row -> upper neighbour's halo (phi, m_x, m_y)
        up = st[rank + 1][w]
        up[2][jhi - 1] = ophi[jhi - 1]
        up[0][jhi - 1] = omx[jhi - 1]
        if jhi - 1 < n:
            up[1][jhi - 1] = omy[jhi - 1]
    if rank > 0:           # first owned row's phi -> lower neighbour's halo
        st[rank - 1][w][2][jlo] = ophi[jlo]
    for q in range(world):  # post sums, then arrival
        mails[q][k % 2, rank] = sums
    for q in range(world):
        seqs[q][rank] = k + 1
    t0 = time.time()
    while (seqs[rank] < k + 1).any():
        if time.time() - t0 > 120:
            raise SystemExit("peer did not arrive")
        time.sleep(0)
    s = np.zeros(3)
    for r in range(world):   # rank order, identical on every rank
        s += mails[rank][k % 2, r]
    fpr = h2 * (s[0] / step + s[1] / step - 2.0 * s[2])
    hist.append(fpr)
    k += 1
    if fpr < tol:
        break
mx, my, phi = mine[k % 2]
ref = O.cp_run(rho, p=1, tol=tol, max_iters=iters)
assert k == ref.iterations, (k, ref.iterations)
assert np.array_equal(phi[jlo:jhi], ref.phi[jlo:jhi])
assert np.array_equal(mx[jlo:jhi], ref.mx[jlo:jhi])
assert np.array_equal(my[jlo:min(jhi, n)], ref.my[jlo:min(jhi, n)])
np.testing.assert_allclose(hist, ref.residual_history, rtol=1e-12)
for sh in shms:
    sh.close()
print("rank", rank, "ok", k)
"""


def _launch_peer(world, n, iters, tol):
    import numpy as np
    from multiprocessing import shared_memory

    tag = f"w1mgpeer{os.getpid()}_{world}_{n}"
    nbytes = 8 * (2 * ((n + 1) * n * 2 + (n + 1) ** 2) + 2 * world * 3 + world)
    shms = [shared_memory.SharedMemory(name=f"{tag}_{r}", create=True, size=nbytes)
            for r in range(world)]
    try:
        for sh in shms:
            np.ndarray((nbytes // 8,), dtype=np.float64, buffer=sh.buf)[:] = 0.0
        env = dict(os.environ, ROOT=ROOT, WORLD_SIZE=str(world), N=str(n), ITERS=str(iters),
                   TOL=repr(tol), TAG=tag)
        procs = [subprocess.Popen([sys.executable, "-c", PEER_WORKER], env=dict(env, RANK=str(r)),
                                  stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
                 for r in range(world)]
        outs = [p.communicate(timeout=600)[0] for p in procs]
        assert all(p.returncode == 0 for p in procs), "\n".join(outs)
    finally:
        for sh in shms:
            sh.close()
            sh.unlink()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_peer_protocol_fixed_iterations(world):
    _launch_peer(world, n=24, iters=40, tol=-1.0)


def test_slab_peer_protocol_converged_stop():
    _launch_peer(2, n=16, iters=200000, tol=1e-7)
