"""PDHG iteration probe: us per iteration of the streaming G-prox PDHG
iteration (three DCT launches) on one config-3-like pair at each size,
fixed iteration count, with the clock record of the run.

  python tools/pdhg_probe.py [iters] [n ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ClockSampler  # noqa: E402
from paper_1810_00118_b200 import instances, w1mg  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
sizes = [int(x) for x in sys.argv[2:]] or [64, 128, 256, 512]
for n in sizes:
    a, b = instances.config3_images(m=n)
    rho = instances.ml_sources(a, b, 1)[0]
    src = w1mg.SourceField(w1mg.ScalarField(w1mg.GridSpec(n), rho))
    prm = w1mg.SolverParams(p=w1mg.PNorm.p2, tolerance=-1.0, max_iters=iters)
    w1mg.pdhg_run(src, prm)
    with ClockSampler(0) as clk:
        r = w1mg.pdhg_run(src, prm)
    print(json.dumps({"n": n, "iters": iters, "us_per_iter": 1e6 * r.total_seconds / iters,
                      "clocks": clk.summary()}), flush=True)
