"""Kernel probe: fused CP sweep ms/launch and achieved GB/s at several sizes."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_00118_b200 import _lib  # noqa: E402

HBM = 6555.2


def probe(ctx, n, B, p=1, warm=20, iters=50):
    L = ctx.L
    L.w1mg_sweep_probe.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_long, C.c_long,
                                   C.POINTER(C.c_double)]
    ms = C.c_double()
    _lib.check(L.w1mg_sweep_probe(ctx.h, n, B, p, warm, iters, C.byref(ms)))
    V = (n + 1) ** 2
    E = n * (n + 1)
    byt = 8 * (3 * V + 4 * E) * B
    gbs = byt / (ms.value * 1e-3) / 1e9
    return {"n": n, "pairs": B, "p": p, "ms_per_sweep": ms.value, "GBps": gbs,
            "frac": gbs / HBM, "cell_updates_per_s": V * B / (ms.value * 1e-3)}


if __name__ == "__main__":
    ctx = _lib.Context(0)
    engines = [int(e) for e in os.environ.get("ENGINES", "0,1").split(",")]
    cases = [(4096, 1), (2048, 1), (1024, 1), (512, 1), (512, 64), (512, 256), (256, 1024),
             (128, 1024), (64, 1024), (32, 1024)]
    if len(sys.argv) > 1:
        cases = [tuple(int(x) for x in a.split("x")) for a in sys.argv[1:]]
    for n, B in cases:
        for e in engines:
            ctx.L.w1mg_set_sweep_engine(e)
            r = probe(ctx, n, B)
            r["engine"] = ["ldg", "tma"][e]
            print(json.dumps(r), flush=True)
