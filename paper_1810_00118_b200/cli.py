"""Command-line front end (the SPEC's app module): the
user-facing caller of the B200 solver and the file formats on either side of
the hot path.

  python -m paper_1810_00118_b200.cli solve --a a.pgm --b b.pgm --p 2 --algo ml-cp \\
      --out report.json --export-flux flux.csv --export-potential phi.csv
  python -m paper_1810_00118_b200.cli gen --kind two_blobs --n 64 --seed 1 --out-a a.pgm --out-b b.pgm
  python -m paper_1810_00118_b200.cli oracle --a a.csv --b b.csv
  python -m paper_1810_00118_b200.cli bench --kind two_blobs --n 128 --algos ml-pdhg \\
      --levels 1,4 --alphas -1,0 --out sweep.csv
  python -m paper_1810_00118_b200.cli bench --images im0.pgm ... im9.pgm --levels 4  # 45 pairs
  python -m paper_1810_00118_b200.cli validate --kind two_blobs --n 128 --count 4 --levels 3

Inputs: PGM (P2 ASCII or P5 binary, maxval <= 65535) or CSV (one image row
per line).  An M x M image is solved on N = M cells; densities
are resampled to the nodes (`discretize`, bilinear on pixel centres, which for
N = M is exactly the cell->node mean of SURVEY D2) and scaled to unit mass.
Exit codes: 0 success, 1 usage, 2 input format, 3 not converged.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

EXIT_OK, EXIT_USAGE, EXIT_FORMAT, EXIT_NUMERIC = 0, 1, 2, 3


class FormatError(Exception):
    pass


# ----------------------------------------------------------------- readers
def _pgm_tokens(data: bytes):
    """Header tokens of a PGM file (comments skipped) and the offset after
    the single whitespace that ends the header."""
    toks, i = [], 0
    while len(toks) < 4:
        while i < len(data) and data[i:i + 1].isspace():
            i += 1
        if i < len(data) and data[i:i + 1] == b"#":
            while i < len(data) and data[i:i + 1] not in (b"\n", b"\r"):
                i += 1
            continue
        j = i
        while j < len(data) and not data[j:j + 1].isspace():
            j += 1
        if j == i:
            raise FormatError("truncated PGM header")
        toks.append(data[i:j])
        i = j
    return toks, i + 1


def read_pgm(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        data = f.read()
    toks, off = _pgm_tokens(data)
    magic = toks[0]
    try:
        w, h, maxval = int(toks[1]), int(toks[2]), int(toks[3])
    except ValueError as e:
        raise FormatError(f"bad PGM header: {e}") from None
    if not (0 < maxval <= 65535) or w <= 0 or h <= 0:
        raise FormatError("bad PGM dimensions / maxval")
    if magic == b"P5":
        dt = np.dtype(">u2") if maxval > 255 else np.uint8
        n = w * h
        raw = np.frombuffer(data, dtype=dt, count=n, offset=off)
        if raw.size != n:
            raise FormatError("truncated P5 data")
        img = raw.astype(np.float64).reshape(h, w)
    elif magic == b"P2":
        vals = data[off - 1:].split()
        if len(vals) < w * h:
            raise FormatError("truncated P2 data")
        img = np.array([int(v) for v in vals[:w * h]], dtype=np.float64).reshape(h, w)
    else:
        raise FormatError(f"not a PGM file (magic {magic!r})")
    return img


def write_pgm(path: str, img: np.ndarray, maxval: int = 65535) -> None:
    img = np.asarray(img, dtype=np.float64)
    top = img.max() if img.max() > 0 else 1.0
    q = np.rint(img / top * maxval).astype(">u2" if maxval > 255 else np.uint8)
    h, w = img.shape
    with open(path, "wb") as f:
        f.write(f"P5\n{w} {h}\n{maxval}\n".encode())
        f.write(q.tobytes())


def read_csv_image(path: str) -> np.ndarray:
    try:
        rows = [[float(x) for x in ln.replace(";", ",").split(",") if x.strip()]
                for ln in open(path) if ln.strip() and not ln.startswith("#")]
    except ValueError as e:
        raise FormatError(f"bad CSV value: {e}") from None
    if not rows or any(len(r) != len(rows[0]) for r in rows):
        raise FormatError("ragged or empty CSV image")
    return np.array(rows, dtype=np.float64)


def read_image(path: str) -> np.ndarray:
    if not os.path.exists(path):
        raise FormatError(f"no such file: {path}")
    img = read_csv_image(path) if path.lower().endswith((".csv", ".txt")) else read_pgm(path)
    if img.shape[0] != img.shape[1]:
        raise FormatError("image must be square (SPEC.md:470)")
    if (img < 0).any() or not np.isfinite(img).all():
        raise FormatError("image values must be finite and non-negative")
    if not (img > 0).any():
        raise FormatError("all-zero image")
    return img


# --------------------------------------------------------- discretisation
def discretize(img: np.ndarray, n: int) -> np.ndarray:
    """Bilinear resampling of the pixel lattice onto the (n+1)^2 nodes, with
    the pixel centres mapped onto [0,1]^2 (pixel centre c of an
    M-pixel side sits at c/(M-1), so corner pixels land on corner nodes; node
    j at x = j/n reads pixel coordinate j (M-1)/n), then scaled to unit mass
    in the L1_h sense: sum rho h^2 = 1."""
    M = img.shape[0]
    if M == 1:
        out = np.full((n + 1, n + 1), float(img[0, 0]))
    else:
        t = np.arange(n + 1) * ((M - 1) / n)  # node position in pixel-centre index space
        i0 = np.minimum(np.floor(t).astype(int), M - 2)
        f = t - i0
        i1 = i0 + 1
        rows = img[i0, :] * (1 - f)[:, None] + img[i1, :] * f[:, None]
        out = rows[:, i0] * (1 - f)[None, :] + rows[:, i1] * f[None, :]
    h = 1.0 / n
    return out / (math.fsum(out.ravel().tolist()) * h * h)


# ---------------------------------------------------------------- exports
def write_field_csv(path: str, blocks: dict) -> None:
    """Header row, then row-major values at 17 significant digits; several
    blocks (flux: x_edges, y_edges) separated by a marker line."""
    with open(path, "w") as f:
        for name, arr in blocks.items():
            f.write(f"# block {name} {arr.shape[0]} {arr.shape[1]}\n")
            for row in arr:
                f.write(",".join(f"{v:.17g}" for v in row) + "\n")


def read_field_csv(path: str) -> dict:
    blocks, cur, name = {}, None, None
    for ln in open(path):
        if ln.startswith("# block"):
            _, _, name, r, c = ln.split()
            cur = blocks[name] = []
        elif ln.strip():
            cur.append([float(x) for x in ln.split(",")])
    return {k: np.array(v) for k, v in blocks.items()}


def write_quiver_csv(path: str, flux, n: int) -> None:
    """Plot-ready x,y,u,v rows: node vectors of the flux."""
    with open(path, "w") as f:
        f.write("x,y,u,v\n")
        for j in range(n + 1):
            for i in range(n + 1):
                u, v = flux.node_vector(i, j)
                f.write(f"{i / n:.17g},{j / n:.17g},{u:.17g},{v:.17g}\n")


# ---------------------------------------------------------------- solving
def solve(args) -> int:
    from . import w1mg

    a = read_image(args.a)
    b = read_image(args.b)
    if a.shape != b.shape:
        raise FormatError("images differ in size")
    n = a.shape[0]
    p = w1mg.pnorm_from_string(args.p)
    step_mode = w1mg.StepMode.safe if args.safe_steps else w1mg.StepMode.practical
    algo = args.algo
    levels = 1
    if algo.startswith("ml-"):
        levels = w1mg.default_levels(n) if args.levels == "auto" else int(args.levels)
        while levels > 1 and n % (1 << (levels - 1)):
            levels -= 1  # reduce L rather than resample
            print(f"warning: N={n} not divisible by 2^(L-1); using L={levels}", file=sys.stderr)
    # per-level sources: re-discretise the original images on every level grid
    srcs = []
    for l in range(levels):
        nl = n >> (levels - 1 - l)
        ra, rb = discretize(a, nl), discretize(b, nl)
        rho = ra - rb
        rho = rho - math.fsum(rho.ravel().tolist()) / rho.size
        srcs.append(rho)
    t0 = time.perf_counter()
    tol_desc = None
    if args.tol == "auto":
        # Eq. 17 defaults, scheduled over the levels with Eq. 16 (alpha)
        r = (1.0 / n) / (1.0 / 512)
        if algo in ("cp", "ml-cp"):
            epsL = 1e-6 / 128.0 * r * r
        else:
            epsL = min(2e-4, 1e-4 / 32.0 * r * r)
        eps = w1mg.make_schedule(n, levels, epsL, args.alpha)
        tol_desc = {"eps": eps}
    else:
        eps = w1mg.make_schedule(n, levels, float(args.tol), args.alpha)
        tol_desc = {"eps": eps}
    if algo == "cp":
        src = w1mg.SourceField(w1mg.ScalarField(w1mg.GridSpec(n), srcs[-1]))
        rep = w1mg.cp_run(src, w1mg.SolverParams(p=p, tolerance=eps[-1], max_iters=args.max_iters,
                                                 step_mode=step_mode))
    elif algo == "pdhg":
        src = w1mg.SourceField(w1mg.ScalarField(w1mg.GridSpec(n), srcs[-1]))
        rep = w1mg.pdhg_run(src, w1mg.SolverParams(p=p, tolerance=eps[-1],
                                                   max_iters=args.max_iters, step_mode=step_mode))
    elif algo == "ml-cp":
        rep = w1mg.ml_run(srcs, p=p, eps=eps, max_iters=args.max_iters, step_mode=step_mode)
    elif algo == "ml-pdhg":
        rep = w1mg.ml_pdhg_run(srcs, p=p, eps=eps, max_iters=args.max_iters, step_mode=step_mode)
    else:
        raise SystemExit(EXIT_USAGE)
    wall = time.perf_counter() - t0
    report = {
        "distance": rep.distance, "dual_value": rep.dual_value, "p": args.p, "algo": algo,
        "levels": [{"h": l.h, "eps": l.eps, "iters": l.iters, "fpr_final": l.fpr_final,
                    "seconds": l.seconds} for l in rep.levels],
        "total_seconds": rep.total_seconds, "wall_seconds": wall, "converged": rep.converged,
        "n": n, **tol_desc,
    }
    text = json.dumps(report, indent=1)
    if args.out:
        with open(args.out, "w") as f:
            f.write(text + "\n")
    else:
        print(text)
    if args.export_flux:
        write_field_csv(args.export_flux, {"x_edges": rep.flux.x_edges,
                                           "y_edges": rep.flux.y_edges})
    if args.export_potential:
        write_field_csv(args.export_potential, {"potential": rep.potential.values})
    if args.export_quiver:
        write_quiver_csv(args.export_quiver, rep.flux, n)
    return EXIT_OK if rep.converged else EXIT_NUMERIC


def gen(args) -> int:
    from . import instances

    if args.kind not in instances.SYNTH_KINDS:
        return EXIT_USAGE
    a, b = instances.synth_instance(args.kind, args.n, args.seed)
    for img, path in ((a, args.out_a), (b, args.out_b)):
        if path.lower().endswith(".csv"):
            np.savetxt(path, img, delimiter=",", fmt="%.17g")
        else:
            write_pgm(path, img)
    return EXIT_OK


def oracle_cmd(args) -> int:
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import exact

    a = read_image(args.a)
    b = read_image(args.b)
    n = a.shape[0]
    rho = discretize(a, n) - discretize(b, n)
    rho -= rho.mean()
    print(json.dumps({"w1_exact_p1": exact.w1_exact_p1(rho), "n": n}))
    return EXIT_OK


def _instance(args, seed_offset: int = 0):
    from . import instances

    if getattr(args, "a", None) and getattr(args, "b", None):
        a, b = read_image(args.a), read_image(args.b)
        if a.shape != b.shape:
            raise FormatError("images differ in size")
        return a, b
    if args.kind not in instances.SYNTH_KINDS:
        raise FormatError(f"unknown instance kind {args.kind!r}")
    return instances.synth_instance(args.kind, args.n, args.seed + seed_offset)


def _csv_list(text: str, conv):
    try:
        return [conv(x) for x in text.split(",") if x.strip()]
    except ValueError as e:
        raise FormatError(f"bad list {text!r}: {e}") from None


def _emit(path, header, rows) -> None:
    lines = [",".join(header)] + [",".join(str(v) for v in r) for r in rows]
    text = "\n".join(lines) + "\n"
    if path:
        with open(path, "w") as f:
            f.write(text)
    else:
        sys.stdout.write(text)


def bench_cmd(args) -> int:
    """Timing / iteration sweeps (paper Tables 4-6 shape), or the
    all-vs-all pair timing on the batched engine (--images ...)."""
    from . import studies, w1mg

    p = w1mg.pnorm_from_string(args.p)
    if args.images:
        imgs = [read_image(pth) for pth in args.images]
        if len(imgs) < 2:
            raise FormatError("--images needs at least two files")
        levels = int(args.levels.split(",")[0])
        rows = studies.all_pairs(imgs, levels, p=p, rel_tol=args.rel_tol,
                                 max_iters=args.max_iters)
        _emit(args.out, ["i", "j", "n", "levels", "p", "distance", "dual_value", "iters",
                         "converged", "batch_pairs", "batch_seconds"],
              [[r["i"], r["j"], r["n"], r["levels"], args.p, repr(r["distance"]),
                repr(r["dual_value"]), "/".join(map(str, r["iters"])), int(r["converged"]),
                r["batch_pairs"], f"{r['batch_seconds']:.6f}"] for r in rows])
        return EXIT_OK if all(r["converged"] for r in rows) else EXIT_NUMERIC
    a, b = _instance(args)
    algos = _csv_list(args.algos, str)
    for al in algos:
        if al not in ("cp", "pdhg", "ml-cp", "ml-pdhg"):
            raise FormatError(f"unknown algorithm {al!r}")
    rows = studies.sweep(a, b, algos, _csv_list(args.levels, int), _csv_list(args.alphas, float),
                         args.eps, p=p, max_iters=args.max_iters)
    _emit(args.out, ["algo", "levels", "alpha", "p", "n", "eps_finest", "distance", "iters",
                     "finest_iters", "seconds", "converged"],
          [[r.algo, r.levels, r.alpha, args.p, r.n, r.eps_finest, repr(r.distance),
            "/".join(map(str, r.iters)), r.iters[-1], f"{r.seconds:.6f}", int(r.converged)]
           for r in rows])
    return EXIT_OK if all(r.converged for r in rows) else EXIT_NUMERIC


def validate_cmd(args) -> int:
    """validate_assumptions as a Table-3-shaped CSV."""
    from . import studies, w1mg

    p = w1mg.pnorm_from_string(args.p)
    insts = [_instance(args, k) for k in range(args.count)]
    rep = studies.validate_assumptions(insts, args.levels, eps=args.eps, p=p,
                                       max_iters=args.max_iters)
    rows = [[r.level, repr(r.h), repr(r.z_norm2), repr(r.y_norm2),
             "" if r.z_disc is None else repr(r.z_disc),
             "" if r.y_disc is None else repr(r.y_disc)] for r in rep.rows]
    rows.append(["fit", "", "", "", f"r={rep.r!r}", f"nu={rep.nu!r}"])
    _emit(args.out, ["level", "h", "z_norm2", "y_norm2", "z_disc", "y_disc"], rows)
    return EXIT_OK


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="w1mg")
    sub = ap.add_subparsers(dest="cmd")
    s = sub.add_parser("solve")
    s.add_argument("--a", required=True)
    s.add_argument("--b", required=True)
    s.add_argument("--p", default="1", choices=["1", "2", "inf"])
    s.add_argument("--algo", default="ml-pdhg", choices=["cp", "pdhg", "ml-cp", "ml-pdhg"])
    s.add_argument("--levels", default="auto")
    s.add_argument("--alpha", type=float, default=-1.0)
    s.add_argument("--tol", default="auto")
    s.add_argument("--max-iters", type=int, default=5_000_000)
    s.add_argument("--safe-steps", action="store_true")
    s.add_argument("--out")
    s.add_argument("--export-flux")
    s.add_argument("--export-potential")
    s.add_argument("--export-quiver")
    g = sub.add_parser("gen")
    g.add_argument("--kind", default="two_blobs")
    g.add_argument("--n", type=int, default=64)
    g.add_argument("--seed", type=int, default=0)
    g.add_argument("--out-a", required=True)
    g.add_argument("--out-b", required=True)
    o = sub.add_parser("oracle")
    o.add_argument("--a", required=True)
    o.add_argument("--b", required=True)
    bn = sub.add_parser("bench")
    bn.add_argument("--a")
    bn.add_argument("--b")
    bn.add_argument("--kind", default="two_blobs")
    bn.add_argument("--n", type=int, default=64)
    bn.add_argument("--seed", type=int, default=0)
    bn.add_argument("--p", default="2", choices=["1", "2", "inf"])
    bn.add_argument("--algos", default="cp,ml-cp,pdhg,ml-pdhg")
    bn.add_argument("--levels", default="1,2,3,4")
    bn.add_argument("--alphas", default="-1")
    bn.add_argument("--eps", type=float, default=1e-6)
    bn.add_argument("--rel-tol", type=float, default=1e-5)
    bn.add_argument("--max-iters", type=int, default=5_000_000)
    bn.add_argument("--images", nargs="*")
    bn.add_argument("--out")
    va = sub.add_parser("validate")
    va.add_argument("--a")
    va.add_argument("--b")
    va.add_argument("--kind", default="two_blobs")
    va.add_argument("--n", type=int, default=64)
    va.add_argument("--seed", type=int, default=0)
    va.add_argument("--count", type=int, default=4)
    va.add_argument("--levels", type=int, default=3)
    va.add_argument("--eps", type=float, default=1e-8)
    va.add_argument("--p", default="2", choices=["1", "2", "inf"])
    va.add_argument("--max-iters", type=int, default=5_000_000)
    va.add_argument("--out")
    try:
        args = ap.parse_args(argv)
    except SystemExit:
        return EXIT_USAGE
    if not args.cmd:
        ap.print_usage()
        return EXIT_USAGE
    try:
        return {"solve": solve, "gen": gen, "oracle": oracle_cmd, "bench": bench_cmd,
                "validate": validate_cmd}[args.cmd](args)
    except FormatError as e:
        print(f"input format error: {e}", file=sys.stderr)
        return EXIT_FORMAT
    except ValueError as e:  # std::invalid_argument from the solver
        print(f"invalid argument: {e}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
