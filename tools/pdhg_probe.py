import sys
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_1810_00118_b200 import instances, w1mg
a, b = instances.config3_images(m=512)
rhos = instances.ml_sources(a, b, 1)
src = w1mg.SourceField(w1mg.ScalarField(w1mg.GridSpec(512), rhos[0]))
prm = w1mg.SolverParams(p=w1mg.PNorm.p2, tolerance=-1.0, max_iters=int(sys.argv[1]))
r = w1mg.pdhg_run(src, prm)
print("secs", r.total_seconds, "per it us", 1e6 * r.total_seconds / prm.max_iters)
