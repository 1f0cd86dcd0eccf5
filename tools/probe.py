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


def probe_clocked(ctx, n, B, p=1):
    """probe() sized to ~1 s of sweeps, with nvidia-smi clocks sampled while
    it runs (bench.ClockSampler): every probe line carries its clock record."""
    from bench import ClockSampler

    first = probe(ctx, n, B, p)
    iters = max(50, int(1.0 / (first["ms_per_sweep"] * 1e-3)))
    with ClockSampler(0) as clk:
        r = probe(ctx, n, B, p, warm=20, iters=iters)
    r["clocks"] = clk.summary()
    r["fast"] = int(os.environ.get("W1MG_FAST", "0"))
    return r


if __name__ == "__main__":
    ctx = _lib.Context(0)
    engines = [int(e) for e in os.environ.get("ENGINES", "3").split(",")]  # 1 tma, 2 tma2, 3 auto, 5 tma2t, 6 tma3
    cases = [(4096, 1), (2048, 1), (1024, 1), (512, 1), (512, 64), (512, 256), (256, 1024),
             (128, 1024), (64, 1024), (32, 1024)]
    if len(sys.argv) > 1:
        cases = [tuple(int(x) for x in a.split("x")) for a in sys.argv[1:]]
    for n, B in cases:
        for e in engines:
            ctx.L.w1mg_set_sweep_engine(e)
            r = probe_clocked(ctx, n, B)
            r["engine"] = ["-", "tma", "tma2", "auto", "-", "tma2t", "tma3"][e]
            print(json.dumps(r), flush=True)


def level_time(ctx, n, B, p=1, sweeps=2000):
    """Device seconds for `sweeps` sweeps of an n-level over B pairs through
    the cascade driver with the stop rule off (eps < 0)."""
    import numpy as np
    from paper_1810_00118_b200 import w1mg
    from paper_1810_00118_b200._lib import MLParams, check

    img = np.random.default_rng(0).random((B, n, n)) + 0.5
    img1 = img[:, ::-1, :].copy()
    prm = MLParams()
    prm.levels, prm.pnorm, prm.step_mode, prm.rel_tol = 1, p, 1, -1.0
    eps = np.array([-1.0])
    prm.eps = eps.ctypes.data_as(C.POINTER(C.c_double))
    prm.max_iters = sweeps
    out = np.zeros(B)
    its = np.zeros(B, dtype=np.int64)
    check(ctx.L.w1mg_ml_cp_batch(ctx.h, B, n, _lib.ptr(img), _lib.ptr(img1), C.byref(prm),
                                 _lib.ptr(out), None, its.ctypes.data_as(_lib._lp), None))
    return ctx.level_seconds(1)[0]
