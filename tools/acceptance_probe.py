"""Measure SPEC acceptance 4/5 quantities on several synthetic kinds
(tolerances: the paper's Eq. 17, and tighter)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_00118_b200 import instances, studies, w1mg  # noqa: E402

P = w1mg.PNorm.p2


def eq17(n, algo):
    r = (1.0 / n) / (1.0 / 512)
    return {"cp": 1e-6 / 512 * r ** 3, "ml-cp": 1e-6 / 128 * r * r,
            "pdhg": min(2e-4, 1e-4 / 16 * r * r), "ml-pdhg": min(2e-4, 1e-4 / 32 * r * r)}[algo]


for kind in ["two_blobs", "config2", "config3", "annulus_pair"]:
    for n in [64, 128]:
        a, b = instances.synth_instance(kind, n, 2)
        L = w1mg.default_levels(n)
        srcs = w1mg.ml_sources(a, b, L)
        f_h = studies.solve_instance([srcs[-1]], "pdhg", [1e-10], P).distance
        f_2h = studies.solve_instance([srcs[-2]], "pdhg", [1e-10], P).distance
        for algo in ["ml-pdhg", "ml-cp"]:
            for tight in [1, 10, 100]:
                epsL = eq17(n, algo) / tight
                eps = w1mg.make_schedule(n, L, epsL, -1.0)
                rep = studies.solve_instance(srcs, algo, eps, P)
                print(f"A5 {kind:12s} n={n} {algo:8s} epsL=Eq17/{tight} ratio="
                      f"{abs(rep.distance-f_h)/abs(f_2h-f_h):.3g} iters={[l.iters for l in rep.levels]}",
                      flush=True)
for kind in ["two_blobs", "config2", "annulus_pair"]:
    a, b = instances.synth_instance(kind, 128, 0)
    out = []
    for algo in ["cp", "pdhg"]:
        for L in [3, 4]:
            e1 = eq17(128, algo)
            rows = studies.sweep(a, b, [algo, "ml-" + algo], [L], [-1.0], e1)
            out.append((algo, L, rows[0].iters[-1], rows[1].iters, rows[1].iters[-1] / rows[0].iters[-1]))
    print("A4", kind, out, flush=True)
