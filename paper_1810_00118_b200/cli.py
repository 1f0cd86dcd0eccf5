"""Command-line front end (the SPEC's app module): the
user-facing caller of the B200 solver and the file formats on either side of
the hot path.

  python -m paper_1810_00118_b200.cli solve --a a.pgm --b b.pgm --p 2 --algo ml-cp \\
      --out report.json --export-flux flux.csv --export-potential phi.csv
  python -m paper_1810_00118_b200.cli gen --kind two_blobs --n 64 --seed 1 --out-a a.pgm --out-b b.pgm
  python -m paper_1810_00118_b200.cli oracle --a a.csv --b b.csv

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
    """Bilinear resampling of the pixel lattice (centres at (c+0.5)/M) onto
    the (n+1)^2 nodes (i/n, j/n), clamped at the border, scaled to unit mass
    in the L1_h sense: sum rho h^2 = 1."""
    M = img.shape[0]
    t = np.arange(n + 1) / n * M - 0.5  # node position in pixel-centre index space
    t = np.clip(t, 0.0, M - 1.0)
    i0 = np.minimum(np.floor(t).astype(int), M - 2) if M > 1 else np.zeros(n + 1, int)
    f = t - i0 if M > 1 else np.zeros(n + 1)
    i1 = np.minimum(i0 + 1, M - 1)
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

    n = args.n
    rng = np.random.default_rng(args.seed)
    t = (np.arange(n) + 0.5) / n
    X, Y = np.meshgrid(t, t, indexing="xy")
    if args.kind == "two_blobs":
        c = rng.uniform(0.2, 0.8, size=(2, 2))
        a = np.exp(-((X - c[0, 0]) ** 2 + (Y - c[0, 1]) ** 2) / (2 * 0.08 ** 2))
        b = np.exp(-((X - c[1, 0]) ** 2 + (Y - c[1, 1]) ** 2) / (2 * 0.08 ** 2))
    elif args.kind == "annulus_pair":
        r = np.hypot(X - 0.5, Y - 0.5)
        a = np.exp(-((r - 0.15) / 0.03) ** 2)
        b = np.exp(-((r - 0.35) / 0.03) ** 2)
    elif args.kind == "dirac_pair":
        a = np.zeros((n, n))
        b = np.zeros((n, n))
        a[0, 0] = 1.0
        b[0, n - 1] = 1.0
    elif args.kind == "config2":
        a, b = instances.config2_images(seed=args.seed, m=n)
    elif args.kind == "config3":
        a = instances.blurred_noise_image(2 * args.seed, m=n)
        b = instances.blurred_noise_image(2 * args.seed + 1, m=n)
    else:
        return EXIT_USAGE
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
    try:
        args = ap.parse_args(argv)
    except SystemExit:
        return EXIT_USAGE
    if not args.cmd:
        ap.print_usage()
        return EXIT_USAGE
    try:
        return {"solve": solve, "gen": gen, "oracle": oracle_cmd}[args.cmd](args)
    except FormatError as e:
        print(f"input format error: {e}", file=sys.stderr)
        return EXIT_FORMAT
    except ValueError as e:  # std::invalid_argument from the solver
        print(f"invalid argument: {e}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
