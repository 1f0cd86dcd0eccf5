"""Converged CPU-oracle fixtures for the two configs whose full-size oracle
runs take CPU minutes (run once here, committed, read by the -m gpu tests):

  config 3: G-prox PDHG cascade 32 -> 512 (BASELINE.json configs[2]) through
            oracle/pdhg_oracle.py (Poisson/affine projection pinned to the
            reference's proj/src/poisson.cpp), rel tol 1e-5 * G_cold,l;
  config 5: CP cascade 64 -> 4096, 7 levels (configs[4]) through the C
            oracle (bit-identical restatement of proj/src/solver_cp.cpp:113-147
            + Eq. 14/15), rel tol 1e-5 * R_cold,l.

Sources come from the oracle's host restriction of the committed instance
generators (paper_1810_00118_b200/instances.py), which the GPU tests rebuild
bit for bit on the box.  Besides W1 / dual / per-level iterations the fixture
holds order-insensitive checksums of the final fields (sum, sum of squares),
so a GPU run that stops on the same sweeps must reproduce them to ~1e-12.

  python tests/golden/make_converged.py [3] [5]
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

OUT = os.path.join(HERE, "converged.json")


def checksums(**fields):
    out = {}
    for k, v in fields.items():
        v = np.asarray(v, dtype=np.float64).ravel()
        out[k] = {"sum": float(np.sum(v)), "sumsq": float(np.dot(v, v)),
                  "absmax": float(np.abs(v).max())}
    return out


def config3():
    from oracle import Oracle
    from oracle import pdhg_oracle as PO
    from paper_1810_00118_b200 import instances

    rhos = Oracle().ml_sources(*instances.config3_images(m=512), 5)
    t = time.perf_counter()
    r = PO.ml_pdhg_run(rhos, p=1, rel_tol=1e-5)
    secs = time.perf_counter() - t
    return {"what": "config 3: G-prox PDHG cascade 32->512, p=2, rel tol 1e-5 * G_cold,l, "
                    "sources Oracle().ml_sources(instances.config3_images(512), 5)",
            "oracle": "oracle/pdhg_oracle.py ml_pdhg_run", "W1": r.distance,
            "dual": r.dual_value, "level_iters": list(r.level_iters),
            "level_eps": list(r.level_eps), "cpu_seconds": secs,
            "fields": checksums(mx=r.mx, my=r.my, phi=r.phi)}


def config5():
    from oracle import Oracle
    from paper_1810_00118_b200 import instances

    O = Oracle()
    rhos = O.ml_sources(*instances.config5_images(), 7)
    t = time.perf_counter()
    r = O.ml_cp_run(rhos, p=1, rel_tol=1e-5)
    secs = time.perf_counter() - t
    return {"what": "config 5: CP cascade 64->4096 (7 levels), p=2, rel tol 1e-5 * R_cold,l, "
                    "sources Oracle().ml_sources(instances.config5_images(), 7)",
            "oracle": "oracle/w1mg_oracle.c or_ml_cp_run", "W1": r.distance,
            "dual": r.dual_value, "level_iters": list(r.level_iters),
            "level_eps": list(r.level_eps), "cpu_seconds": secs,
            "fields": checksums(mx=r.mx, my=r.my, phi=r.phi)}


def main():
    which = sys.argv[1:] or ["3", "5"]
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            data = json.load(f)
    for w in which:
        data["config" + w] = {"3": config3, "5": config5}[w]()
        print(w, json.dumps({k: v for k, v in data["config" + w].items() if k != "fields"}),
              flush=True)
        with open(OUT, "w") as f:
            json.dump(data, f, indent=1)


if __name__ == "__main__":
    main()
