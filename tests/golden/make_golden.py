"""Generates tests/golden/*.npz|json from the REFERENCE build (oracle/_ref,
compiled from /root/reference/proj/src) -- run here, where /root/reference
exists; the fixtures travel with the repo so the GPU box never needs the
reference tree.

  python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import Reference  # noqa: E402
from paper_1810_00118_b200 import instances  # noqa: E402


def main():
    R = Reference()
    kat = {
        # SPEC.md:123-125, 130-132, 137-139
        "shrink_p2": R.shrink((3, 4), 1.0, 1),
        "shrink_p1": R.shrink((0.3, -2), 0.5, 0),
        "shrink_pinf": R.shrink((0.5, -1.5), 1.0, 2),
        "proj_qinf": R.project_unit_ball((1.5, -0.2), 2),
        "proj_q2": R.project_unit_ball((3, 4), 1),
        "proj_q1": R.project_unit_ball((0.5, -1.5), 0),
        "l1_inside": R.project_l1_ball((0.2, 0.1), 1.0),
        "l1_axis": R.project_l1_ball((2, 0), 1.0),
        "step_practical_256": R.cp_step_size(256),
        "step_safe_256": R.cp_step_size(256, safe=True),
    }
    with open(os.path.join(HERE, "reference_kats.json"), "w") as f:
        json.dump({k: list(v) if isinstance(v, tuple) else v for k, v in kat.items()}, f, indent=1)

    # fixed-iteration CP runs of the reference, p = 1, 2, inf
    out = {}
    rho16 = instances.config1_source(16)
    out["rho16"] = rho16
    for p in (0, 1, 2):
        r = R.cp_run(rho16, p=p, tol=-1.0, max_iters=250)
        out[f"p{p}_mx"], out[f"p{p}_my"], out[f"p{p}_phi"] = r.mx, r.my, r.phi
        out[f"p{p}_hist"] = r.residual_history
        out[f"p{p}_w1"] = np.array([r.distance, r.dual_value])
    # config-1 (N=64, 20,000 sweeps, p=2): W1 / dual / final FPR only
    r = R.cp_run(instances.config1_source(64), p=1, tol=-1.0, max_iters=20000, hist_cap=20000)
    out["config1_w1_dual_fpr"] = np.array([r.distance, r.dual_value, r.residual_history[-1]])
    # two-Dirac N = 8, p = 1 converged
    r = R.cp_run(instances.dirac_pair_source(8), p=0, tol=1e-12, max_iters=400000)
    out["dirac8_p1"] = np.array([r.distance, r.iterations])
    # Poisson (reference poisson.cpp through the FFTW shim) and affine projection, N = 12
    rng = np.random.default_rng(12)
    b = rng.standard_normal((13, 13))
    b -= b.mean()
    out["poisson_b"] = b
    out["poisson_phi"] = R.poisson_solve(b, projected=True)
    mx, my = rng.standard_normal((13, 12)), rng.standard_normal((12, 13))
    rho = instances.make_source(rng.random((13, 13)), rng.random((13, 13)), 12)
    ax, ay = R.project_affine(mx, my, rho)
    out.update(aff_mx=mx, aff_my=my, aff_rho=rho, aff_ox=ax, aff_oy=ay)
    np.savez_compressed(os.path.join(HERE, "reference_runs.npz"), **out)
    print("wrote", sorted(out))


if __name__ == "__main__":
    main()
