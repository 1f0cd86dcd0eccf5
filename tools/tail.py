"""Tail-loss probe for the batched cascade (config 4): per level, the sweep
distribution over pairs, the measured level time and the time the same
pair-sweeps would take at the full-batch probe rate."""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1810_00118_b200 import _lib  # noqa: E402
from paper_1810_00118_b200._lib import MLParams, check  # noqa: E402
from tools.probe import probe  # noqa: E402

if __name__ == "__main__":
    import torch

    B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    dev = torch.device("cuda", 0)
    img0, img1 = bench.make_images_gpu(0, B, dev)
    ctx = _lib.Context(0)
    prm = MLParams()
    prm.levels, prm.pnorm, prm.step_mode = bench.LEVELS, 1, 1
    prm.rel_tol, prm.eps, prm.max_iters = bench.REL_TOL, None, 5_000_000
    d = torch.zeros(B, dtype=torch.float64, device=dev)
    du = torch.zeros(B, dtype=torch.float64, device=dev)
    it = torch.zeros((B, bench.LEVELS), dtype=torch.int64, device=dev)
    cv = torch.zeros(B, dtype=torch.int32, device=dev)
    for rep in range(2):
        check(ctx.L.w1mg_ml_cp_batch_dev(ctx.h, B, bench.M, C.c_void_p(img0.data_ptr()),
                                         C.c_void_p(img1.data_ptr()), C.byref(prm),
                                         C.c_void_p(d.data_ptr()), C.c_void_p(du.data_ptr()),
                                         C.c_void_p(it.data_ptr()), C.c_void_p(cv.data_ptr())))
        ctx.synchronize()
    secs = ctx.level_seconds(bench.LEVELS)
    its = it.cpu().numpy()
    for l, n in enumerate(bench.level_sizes()):
        s = its[:, l]
        full = probe(ctx, n, B)["ms_per_sweep"] * 1e-3 / B  # s per pair-sweep, full batch
        ideal = s.sum() * full
        print(json.dumps({"n": n, "level_s": secs[l], "ideal_s": ideal, "eff": ideal / secs[l],
                          "sweeps_min": int(s.min()), "sweeps_mean": float(s.mean()),
                          "sweeps_p90": float(np.percentile(s, 90)), "sweeps_max": int(s.max())}),
              flush=True)
