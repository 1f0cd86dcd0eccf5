"""Refresh the bench numbers quoted in profiles/r1_summary.md and DESIGN.md
from profiles/r1_bench_default_latest.json (the committed bench line)."""
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
d = json.load(open(os.path.join(ROOT, "profiles", "r1_bench_default_latest.json")))
lv = [l["seconds_per_step"] for l in d["levels"]]
rows = {
    "| bench value |": f"| bench value | {d['value']:.4g} cell-updates/s ({d['ms_per_step'] / 1e3:.2f} s "
                       f"per {d['config']['pairs_per_step']}-pair step), {d['pairs_per_s']:.1f} pairs/s |",
    "| e2e (host API": f"| e2e (host API, pinned H2D of the images every step) | {d['e2e']['value']:.4g} "
                       f"cell-updates/s, {d['e2e']['pairs_per_s']:.1f} pairs/s |",
    "| time to converged W1": f"| time to converged W1, one 512² pair | {d['time_to_w1_512_s']:.3f} s |",
    "| level time per step": f"| level time per step | 512²: {lv[4]:.2f} s, 256²: {lv[3]:.2f} s, "
                            f"128²: {lv[2]:.2f} s, 64²+32²: {lv[0] + lv[1]:.2f} s |",
    "| finest-level sweep": f"| finest-level sweep in the timed region | {d['roofline']['achieved']:.0f} GB/s of "
                           f"one-sweep algorithmic bytes (roofline.frac {d['roofline']['frac']:.3f}); actual "
                           f"DRAM {d['roofline']['dram_achieved']:.0f} GB/s (dram_frac "
                           f"{d['roofline']['dram_frac']:.3f}) |",
    "| clocks |": f"| clocks | {d['clocks']['sm_mhz']:.0f} MHz median under load (max "
                  f"{d['clocks']['sm_max_mhz']:.0f}), {', '.join(d['clocks']['reasons']) or 'no'} throttle |",
}
p = os.path.join(ROOT, "profiles", "r1_summary.md")
out, latest = [], True
for line in open(p).read().split("\n"):
    if line.startswith("## First capture") or line.startswith("## Earlier captures"):
        latest = False  # historical sections keep their numbers
    if latest:
        for k, v in rows.items():
            if line.startswith(k):
                line = v
                break
    out.append(line)
open(p, "w").write("\n".join(out))
p = os.path.join(ROOT, "DESIGN.md")
s = open(p).read()
s = re.sub(r"`profiles/r1_bench_default_latest.json`, 512 pairs per step\)\n[^\n]*\n[^\n]*\n",
           f"`profiles/r1_bench_default_latest.json`, 512 pairs per step)\n"
           f"{d['value']:.4g} cell-updates/s, {d['pairs_per_s']:.1f} pairs/s (e2e through the host API with\n"
           f"H2D of the images: {d['e2e']['value']:.4g}), {d['time_to_w1_512_s']:.3f} s to converged W1 for one\n",
           s)
open(p, "w").write(s)
print("refreshed", d["value"])
