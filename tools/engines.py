"""Compare resident vs streaming engines on small levels (whole-level time)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_00118_b200 import _lib  # noqa: E402
from tools.probe import level_time  # noqa: E402

ctx = _lib.Context(0)
for n, B, sw in [(32, 1, 2000), (64, 1, 2000), (32, 1024, 2000), (64, 1024, 1000), (64, 256, 1000)]:
    for res in (1, 0):
        ctx.L.w1mg_set_resident_engine(res)
        level_time(ctx, n, B, sweeps=20)
        t = level_time(ctx, n, B, sweeps=sw)
        print(json.dumps({"n": n, "pairs": B, "resident": res, "sweeps": sw, "s": t,
                          "us_per_sweep": 1e6 * t / sw,
                          "cell_updates_per_s": (n + 1) ** 2 * B * sw / t}), flush=True)
