"""Exact W1 oracles.  TEST INFRASTRUCTURE ONLY.

* ``w1_exact_p1(rho)`` -- the p = 1 Beckmann problem on the grid is a min-cost
  flow: node supplies s(x) = rho(x) h^2, every grid edge in both directions
  with cost h per unit of mass (flux m on an edge carries F = m h of mass, and
  sum |m| h^2 = sum h |F|).  Solved exactly by successive shortest paths with
  Johnson potentials on integers: supplies are scaled by 2^40 and rounded with
  the rounding residual moved to one node, so the quantisation error is below
  2 N h V / 2^41 (~1e-10 for N <= 16).
* ``w1_1d_cdf(r0, r1, h)`` -- h sum_x |sum_{y<=x} (r0 - r1)(y) h|.

Neither exists in the reference tree (the SPEC's oracle module is absent); they
give ground truth independent of the reference's iterates.
"""
from __future__ import annotations

import heapq

import numpy as np

SCALE = 1 << 40


def w1_exact_p1(rho: np.ndarray) -> float:
    rho = np.asarray(rho, dtype=np.float64)
    n = rho.shape[0] - 1
    if n > 32:
        raise ValueError("w1_exact_p1: grid too large for the oracle (N <= 32)")
    h = 1.0 / n
    W = n + 1
    V = W * W
    supply = [int(round(v * h * h * SCALE)) for v in rho.ravel().tolist()]
    supply[0] -= sum(supply)  # exact zero total
    # graph: 4-neighbour edges, unit costs (multiply by h at the end)
    adj = [[] for _ in range(V)]
    for j in range(W):
        for i in range(W):
            k = j * W + i
            if i + 1 < W:
                adj[k].append(k + 1)
                adj[k + 1].append(k)
            if j + 1 < W:
                adj[k].append(k + W)
                adj[k + W].append(k)
    # flow on directed arcs (uncapacitated); residual arcs appear when flow > 0
    flow = {}
    excess = supply[:]
    pot = [0] * V
    cost_units = 0
    while True:
        sources = [v for v in range(V) if excess[v] > 0]
        if not sources:
            break
        # multi-source Dijkstra on reduced costs
        dist = [None] * V
        prev = [-1] * V
        pq = [(0, s) for s in sources]
        for s in sources:
            dist[s] = 0
        heapq.heapify(pq)
        done = [False] * V
        target = -1
        while pq:
            d, u = heapq.heappop(pq)
            if done[u]:
                continue
            done[u] = True
            if excess[u] < 0:
                target = u
                break
            for v in adj[u]:
                # forward arc u->v cost 1; backward (cancel v->u flow) cost -1
                for c, ok in ((1, True), (-1, flow.get((v, u), 0) > 0)):
                    if not ok:
                        continue
                    rc = c + pot[u] - pot[v]
                    nd = d + rc
                    if dist[v] is None or nd < dist[v]:
                        dist[v] = nd
                        prev[v] = (u, c)
                        heapq.heappush(pq, (nd, v))
        if target < 0:
            raise RuntimeError("w1_exact_p1: infeasible")
        # update potentials (settled nodes only keep reduced costs >= 0)
        dt = dist[target]
        for v in range(V):
            if done[v] and dist[v] is not None:
                pot[v] += dist[v] - dt
        # path back to the source it started from (sources keep prev = -1:
        # reduced costs are >= 0, so nothing reaches them below distance 0)
        path = []
        v = target
        while prev[v] != -1:
            u, c = prev[v]
            path.append((u, v, c))
            v = u
        src = v
        amt = min(excess[src], -excess[target])
        for u, w, c in path:
            if c < 0:
                amt = min(amt, flow[(w, u)])
        for u, w, c in path:
            if c > 0:
                flow[(u, w)] = flow.get((u, w), 0) + amt
                cost_units += amt
            else:
                flow[(w, u)] -= amt
                cost_units -= amt
        excess[src] -= amt
        excess[target] += amt
    return cost_units * h / SCALE


def w1_1d_cdf(r0, r1, h: float) -> float:
    """h * sum_x |F0(x) - F1(x)| with F = cumulative sums times h."""
    d = np.asarray(r0, dtype=np.float64) - np.asarray(r1, dtype=np.float64)
    if abs(d.sum()) > 1e-9 * (np.abs(np.asarray(r0)).sum() + 1e-300):
        raise ValueError("w1_1d_cdf: mass mismatch")
    c = np.cumsum(d) * h
    return float(h * np.abs(c).sum())


def w1_lp_p1(rho: np.ndarray) -> float:
    """Independent generic-LP solve of the same p = 1 problem (scipy HiGHS),
    used to cross-check the min-cost flow."""
    from scipy.optimize import linprog
    from scipy.sparse import lil_matrix

    rho = np.asarray(rho, dtype=np.float64)
    n = rho.shape[0] - 1
    h = 1.0 / n
    W = n + 1
    edges = []
    for j in range(W):
        for i in range(W):
            k = j * W + i
            if i + 1 < W:
                edges.append((k, k + 1))
            if j + 1 < W:
                edges.append((k, k + W))
    ne = len(edges)
    A = lil_matrix((W * W, 2 * ne))
    for e, (u, v) in enumerate(edges):
        A[u, e] += 1.0  # u -> v
        A[v, e] -= 1.0
        A[v, ne + e] += 1.0  # v -> u
        A[u, ne + e] -= 1.0
    b = rho.ravel() * h * h
    res = linprog(np.full(2 * ne, h), A_eq=A.tocsr(), b_eq=b, bounds=(0, None), method="highs")
    if not res.success:
        raise RuntimeError(res.message)
    return float(res.fun)
