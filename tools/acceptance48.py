"""SPEC acceptance 4 (multilevel speedup pattern) and 8 (assumption
validation, Table 3 pattern) measured on the synthetic instances: one JSON
line per (instance, algorithm, L, alpha) for A4 and one per instance set for
A8.  Used to set the assertions of tests/test_studies.py."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1810_00118_b200 import instances, studies, w1mg  # noqa: E402


def eq17(n, algo):
    r = (1.0 / n) / (1.0 / 512)
    return {"cp": 1e-6 / 512 * r ** 3, "ml-cp": 1e-6 / 128 * r * r,
            "pdhg": min(2e-4, 1e-4 / 16 * r * r), "ml-pdhg": min(2e-4, 1e-4 / 32 * r * r)}[algo]


def a4(kind, seed, n=128):
    a, b = instances.synth_instance(kind, n, seed)
    out = []
    for single, multi in (("cp", "ml-cp"), ("pdhg", "ml-pdhg")):
        for scale in (1.0, 0.1):
            eps = eq17(n, single) * scale
            s = studies.sweep(a, b, [single], [1], [-1.0], eps)[0]
            for L in (3, 4, 5):
                for alpha in (-1.0, 0.0):
                    m = studies.sweep(a, b, [multi], [L], [alpha], eps)[0]
                    out.append({"A": 4, "kind": kind, "seed": seed, "n": n, "algo": multi,
                                "eps_scale": scale, "L": L, "alpha": alpha,
                                "single": s.iters[-1], "cascade": m.iters,
                                "frac": m.iters[-1] / s.iters[-1]})
                    print(json.dumps(out[-1]), flush=True)
    return out


def a8(kind, count=5, n=128, levels=4, eps=1e-8):
    insts = [instances.synth_instance(kind, n, s) for s in range(count)]
    t = time.perf_counter()
    rep = studies.validate_assumptions(insts, levels, eps=eps)
    z = [r.z_norm2 for r in rep.rows]
    y = [r.y_norm2 for r in rep.rows]
    line = {"A": 8, "kind": kind, "count": count, "n": n, "levels": levels, "eps": eps,
            "r": rep.r, "nu": rep.nu, "z_ratio": max(z) / min(z), "y_ratio": max(y) / min(y),
            "z_disc": [r.z_disc for r in rep.rows], "y_disc": [r.y_disc for r in rep.rows],
            "seconds": time.perf_counter() - t}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    what = sys.argv[1:] or ["a4", "a8"]
    if "a4" in what:
        for kind, seed in (("two_blobs", 0), ("two_blobs", 1), ("two_blobs", 3),
                           ("annulus_pair", 0), ("config2", 2)):
            a4(kind, seed)
    if "a8" in what:
        for kind in ("two_blobs", "annulus_pair", "config2", "config3"):
            a8(kind)
