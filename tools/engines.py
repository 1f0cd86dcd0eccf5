"""Whole-level device time of the level-resident engines vs the streaming
sweeps, for small levels (single pair = latency, many pairs = throughput).

W1MG_RESIDENT modes: 1 = thread-block cluster engine, 2 = single-CTA
resident engine (n <= 64), 0 = streaming sweeps only.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_00118_b200 import _lib  # noqa: E402
from tools.probe import level_time  # noqa: E402

ctx = _lib.Context(0)
cases = [(32, 1, 2000), (64, 1, 2000), (128, 1, 2000), (256, 1, 2000), (32, 1024, 2000),
         (64, 1024, 1000), (128, 256, 1000), (256, 256, 500)]
if len(sys.argv) > 1:
    cases = [tuple(int(x) for x in a.split("x")) for a in sys.argv[1:]]
for n, B, sw in cases:
    for res in (3, 2, 0):
        if res == 2 and n > 64:
            continue
        ctx.L.w1mg_set_resident_engine(res)
        level_time(ctx, n, B, sweeps=20)
        t = level_time(ctx, n, B, sweeps=sw)
        print(json.dumps({"n": n, "pairs": B, "engine": {3: "cluster", 2: "1cta", 0: "stream"}[res],
                          "sweeps": sw, "us_per_sweep": 1e6 * t / sw,
                          "cell_updates_per_s": (n + 1) ** 2 * B * sw / t}), flush=True)
ctx.L.w1mg_set_resident_engine(1)
