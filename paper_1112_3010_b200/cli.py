"""Command line of the B200 build — the reference's `eikfld` front end
re-wired to the GPU path (R/cli.py:100-197,240-325).

Same sub-commands and flags for the hot path (`dt`, `grad`, `hessian`,
`sign`, `info`), same `--config` JSON defaults, same exit codes (0 ok, 2 with a
single-line ``error: ...`` on validation/precision failures) and the same
EIKFLD01 outputs.  Methods other than ``fft`` (exact/direct/sweep) and the
`experiment` protocols are reference-only (out of scope) and
exit 2 with a message saying so.

    python -m paper_1112_3010_b200.cli dt --points p.csv --min 0,0 --counts 256,256 \
        --spacing 1 --tau 0.5 --out S.fld
"""

from __future__ import annotations

import argparse
import json
import sys

import numpy as np

from . import fieldio
from .derivatives import gradient, gradient_magnitude, hessian_2d
from .distance import clamp_nonnegative, s_fft
from .errors import NativeError, PrecisionError, ValidationError
from .grid import Curve2D, GridSpec, snap_points, triangulate_and_orient
from .precision import PrecisionConfig, native_tau_floor
from .sign import DEGREE_3D, WINDING_2D, classify, degree_field, signed_distance, winding_field


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        raise ValidationError(message)


def load_points_csv(path) -> np.ndarray:
    """One point per line, 2 or 3 comma/space separated numbers; '#' comments (R/grid.py:322-344)."""
    rows = []
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, 1):
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            parts = line.replace(",", " ").split()
            if len(parts) not in (2, 3):
                raise ValidationError(f"{path}:{lineno}: expected 2 or 3 fields, got {len(parts)}")
            try:
                rows.append([float(p) for p in parts])
            except ValueError:
                raise ValidationError(f"{path}:{lineno}: non-numeric field") from None
    if not rows:
        raise ValidationError(f"{path}: no points found")
    if len({len(r) for r in rows}) != 1:
        raise ValidationError(f"{path}: mixed 2D/3D rows")
    return np.asarray(rows, dtype=np.float64)


def load_mesh(path):
    """CSV triangle soup (9 numbers per line) or the OBJ v/f subset (R/grid.py:347-394)."""
    text = open(path, "r", encoding="utf-8").read()
    lines = text.splitlines()
    if any(ln.lstrip().startswith(("v ", "f ")) for ln in lines):
        verts, faces = [], []
        for lineno, line in enumerate(lines, 1):
            tag, _, rest = line.strip().partition(" ")
            if tag == "v":
                parts = rest.split()
                if len(parts) < 3:
                    raise ValidationError(f"{path}:{lineno}: bad vertex line")
                verts.append([float(p) for p in parts[:3]])
            elif tag == "f":
                parts = rest.split()
                if len(parts) != 3:
                    raise ValidationError(f"{path}:{lineno}: only triangular faces are supported")
                faces.append([int(p.split("/")[0]) - 1 for p in parts])
        if not verts or not faces:
            raise ValidationError(f"{path}: OBJ subset needs v and f lines")
        return triangulate_and_orient(np.asarray(verts), np.asarray(faces))
    tris = []
    for lineno, line in enumerate(lines, 1):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        parts = line.replace(",", " ").split()
        if len(parts) != 9:
            raise ValidationError(f"{path}:{lineno}: triangle soup rows need 9 fields, got {len(parts)}")
        tris.append([float(p) for p in parts])
    if not tris:
        raise ValidationError(f"{path}: no triangles found")
    soup = np.asarray(tris).reshape(-1, 3, 3)
    return triangulate_and_orient(soup.reshape(-1, 3), np.arange(soup.shape[0] * 3).reshape(-1, 3))


def _floats(text):
    return tuple(float(v) for v in text.split(","))


def _ints(text):
    return tuple(int(v) for v in text.split(","))


def _grid(args) -> GridSpec:
    if args.min is None:
        raise ValidationError("--min is required")
    lo = _floats(args.min)
    if args.counts is not None:
        counts = _ints(args.counts)
        if args.spacing is None:
            if args.max is None:
                raise ValidationError("--counts needs --spacing or --max")
            spacing = (_floats(args.max)[0] - lo[0]) / (counts[0] - 1)
        else:
            spacing = args.spacing
        return GridSpec(origin=lo, spacing=spacing, counts=counts)
    if args.max is None or args.spacing is None:
        raise ValidationError("grid needs --min plus --counts or --max/--spacing")
    hi = _floats(args.max)
    return GridSpec(origin=lo, spacing=args.spacing,
                    counts=tuple(int(round((h - l) / args.spacing)) + 1 for l, h in zip(lo, hi)))


def _require(args, *names):
    for n in names:
        if getattr(args, n.replace("-", "_"), None) is None:
            raise ValidationError(f"--{n} is required")


def _fft_only(method):
    if method != "fft":
        raise ValidationError(f"method {method!r} is provided by the reference CPU package; the B200 build runs 'fft'")


def _warn_floor(cfg, grid):
    floor = native_tau_floor(grid.diagonal)
    if cfg.tau < floor:
        print(f"warning: tau={cfg.tau:g} is below the native64 floor {floor:g} for this grid; expect underflow, "
              "use --precision big:<bits>", file=sys.stderr)


def cmd_dt(args) -> int:
    _require(args, "points", "tau", "out")
    _fft_only(args.method)
    grid = _grid(args)
    cfg = PrecisionConfig.parse(args.precision, args.tau)
    ps = snap_points(load_points_csv(args.points), grid)
    _warn_floor(cfg, grid)
    field = s_fft(ps, grid, cfg)
    if args.clamp_nonneg:
        field = clamp_nonnegative(field)
    params = {"method": args.method, "points_file": args.points, "num_points": int(ps.size),
              "clamp_nonneg": bool(args.clamp_nonneg)}
    fieldio.write_field(args.out, field, "S", cfg, params)
    if args.csv:
        fieldio.write_csv(args.csv, field)
    return 0


def cmd_grad(args) -> int:
    _require(args, "points", "tau", "out-prefix")
    _fft_only(args.method)
    grid = _grid(args)
    cfg = PrecisionConfig.parse(args.precision, args.tau)
    ps = snap_points(load_points_csv(args.points), grid)
    _warn_floor(cfg, grid)
    vec = gradient(ps, grid, cfg)
    params = {"method": args.method, "points_file": args.points}
    for name, comp in zip(["S_x", "S_y", "S_z"][: grid.dim], vec.components):
        fieldio.write_field(f"{args.out_prefix}{name}.fld", comp, name, cfg, params)
    if args.with_magnitude:
        fieldio.write_field(f"{args.out_prefix}grad_mag.fld", gradient_magnitude(vec), "grad_mag", cfg, params)
    return 0


def cmd_hessian(args) -> int:
    _require(args, "points", "tau", "out-prefix")
    _fft_only(args.method)
    grid = _grid(args)
    cfg = PrecisionConfig.parse(args.precision, args.tau)
    ps = snap_points(load_points_csv(args.points), grid)
    _warn_floor(cfg, grid)
    params = {"method": args.method, "points_file": args.points}
    for name, fld in zip(("S_xx", "S_yy", "S_xy"), hessian_2d(ps, grid, cfg)):
        fieldio.write_field(f"{args.out_prefix}{name}.fld", fld, name, cfg, params)
    return 0


def cmd_sign(args) -> int:
    grid = _grid(args)
    cfg = PrecisionConfig.parse(args.precision, 1.0)
    if (args.curve is None) == (args.mesh is None):
        raise ValidationError("exactly one of --curve or --mesh is required")
    if args.curve is not None:
        mu = winding_field(Curve2D(load_points_csv(args.curve)), grid, cfg)
        mode, source = WINDING_2D, args.curve
    else:
        mu = degree_field(load_mesh(args.mesh), grid, cfg)
        mode, source = DEGREE_3D, args.mesh
    mask = classify(mu, mode, threshold=args.threshold)
    params = {"geometry": source, "mode": mode, "threshold": args.threshold}
    fieldio.write_field(args.mu_out, mu, "mu", cfg, params)
    fieldio.write_field(args.mask_out, mask, "mask", cfg, params)
    if args.mask_csv:
        fieldio.write_csv(args.mask_csv, mask)
    if args.distance_field:
        _, s = fieldio.read_field(args.distance_field)
        fieldio.write_field(args.signed_out or "signed_S.fld", signed_distance(s, mask), "signed_S", cfg, params)
    return 0


def cmd_info(args) -> int:
    json.dump(fieldio.read_header(args.path), sys.stdout, sort_keys=True, indent=2)
    sys.stdout.write("\n")
    return 0


def cmd_experiment(args) -> int:
    raise ValidationError("the experiment protocols are reference-only (SURVEY.md §2.1); "
                          "use engine.TauSweep for the GPU tau sweep")


def build_parser():
    parser = _Parser(prog="eikfld-b200", description="approximate signed distance fields via FFT convolutions (B200)")
    sub = parser.add_subparsers(dest="command", required=True, parser_class=_Parser)
    parsers = [parser]

    def grid_flags(p):
        p.add_argument("--min")
        p.add_argument("--max")
        p.add_argument("--spacing", type=float)
        p.add_argument("--counts")

    def common(p):
        p.add_argument("--precision", default="f64")
        p.add_argument("--threads", type=int, default=1)
        p.add_argument("--config")

    p = sub.add_parser("dt")
    parsers.append(p)
    p.add_argument("--points")
    grid_flags(p)
    p.add_argument("--tau", type=float)
    p.add_argument("--method", default="fft", choices=["fft", "direct", "exact", "sweep"])
    p.add_argument("--iterations", type=int)
    p.add_argument("--clamp-nonneg", action="store_true")
    p.add_argument("--out")
    p.add_argument("--csv")
    common(p)
    p.set_defaults(func=cmd_dt)
    for name, fn in (("grad", cmd_grad), ("hessian", cmd_hessian)):
        p = sub.add_parser(name)
        parsers.append(p)
        p.add_argument("--points")
        grid_flags(p)
        p.add_argument("--tau", type=float)
        p.add_argument("--method", default="fft", choices=["fft", "direct"])
        if name == "grad":
            p.add_argument("--with-magnitude", action="store_true")
        p.add_argument("--out-prefix")
        common(p)
        p.set_defaults(func=fn)
    p = sub.add_parser("sign")
    parsers.append(p)
    p.add_argument("--curve")
    p.add_argument("--mesh")
    grid_flags(p)
    p.add_argument("--threshold", type=float)
    p.add_argument("--mu-out", default="mu.fld")
    p.add_argument("--mask-out", default="mask.fld")
    p.add_argument("--mask-csv")
    p.add_argument("--distance-field")
    p.add_argument("--signed-out")
    common(p)
    p.set_defaults(func=cmd_sign)
    p = sub.add_parser("experiment")
    parsers.append(p)
    p.add_argument("name")
    p.add_argument("--trials", type=int)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--method", default="direct")
    p.add_argument("--out", default="-")
    common(p)
    p.set_defaults(func=cmd_experiment)
    p = sub.add_parser("info")
    parsers.append(p)
    p.add_argument("path")
    p.set_defaults(func=cmd_info)
    return parser, parsers


def _config_defaults(parsers, argv):
    if "--config" not in argv:
        return
    i = argv.index("--config")
    if i + 1 >= len(argv):
        raise ValidationError("--config needs a file path")
    with open(argv[i + 1], "r", encoding="utf-8") as fh:
        values = json.load(fh)
    if not isinstance(values, dict):
        raise ValidationError("--config must hold a JSON object")
    for p in parsers:
        p.set_defaults(**{k.replace("-", "_"): v for k, v in values.items()})


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    parser, parsers = build_parser()
    try:
        _config_defaults(parsers, argv)
        args = parser.parse_args(argv)
        return args.func(args)
    except (ValidationError, PrecisionError, FileNotFoundError, NativeError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
