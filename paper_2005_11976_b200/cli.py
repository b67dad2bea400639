"""Command-line front end routed to the B200 engine.

Mirrors the reference's ``cyltomo simulate | reconstruct | batch``
(``cyltomo/cli.py:248-265, 341-397, 476-515``): same JSON config documents
(deep-merged on defaults, jsonschema-validated), same artifacts
(``projections.json/.raw``, ``volume.json/.raw``, ``report.json``,
``residuals.csv``, ``batch_results.csv``, ``batch_summary.csv``) and the same
exit codes (0 ok, 2 config, 3 io, 4 domain).  ``pose`` (``cyltomo/cli.py:286-313``)
estimates the pose with the GPU-batched segmentation of :mod:`posefit`, and
``reconstruct`` / ``batch`` use it for ``pose = "estimate"`` /
``pose_source = "estimated"``.  Additions: ``sart`` accepts ``subsets``
(OS-SART) and ``residuals``; ``batch`` shards objects over ranks when
launched with torchrun.

    python -m paper_2005_11976_b200.cli pose --config pose.json --out out/
    python -m paper_2005_11976_b200.cli reconstruct --config recon.json --out out/
"""

from __future__ import annotations

import argparse
import csv
import json
import math
import os
import sys
from pathlib import Path

import numpy as np

from . import errors, io
from .geometry import Pose, ScanGeometry, full_turn_angles, make_circular_trajectory
from .grid import CartGrid, CylGrid, CylVolume
from .phantom import ComponentSpec, make_assembly_phantom, make_weight_map
from .posefit import LmConfig, PoseFitParams, fit_pose
from .projector import RaySamplingConfig, simulate_scan
from .recon import SartConfig, presence_metric, sart_run

EXIT_OK, EXIT_UNEXPECTED, EXIT_CONFIG, EXIT_IO, EXIT_DOMAIN = 0, 1, 2, 3, 4

# exception class -> (exit code, message prefix), checked in order
# (the reference's exit-code contract, cyltomo/cli.py:33-38)
EXIT_MAP = ((errors.ConfigError, EXIT_CONFIG, "config error"),
            ((errors.IoFailure, errors.SchemaMismatch, errors.SizeMismatch), EXIT_IO, "io error"),
            (errors.CylTomoError, EXIT_DOMAIN, "error"))

# --preset paper: the paper-scale simulation geometry (cyltomo/cli.py:250-252)
PAPER_GEOMETRY = {"n_views": 4096, "det_cols": 2048, "det_rows": 128,
                  "pixel_pitch_mm": 0.0096, "full_turn": True}


def merged(defaults: dict, user: dict) -> dict:
    """`user` laid over `defaults`, nested objects merged key by key (lists and
    scalars replace).  Iterative: a work list of (target, overlay) pairs."""
    root = dict(defaults)
    work = [(root, user)]
    while work:
        target, overlay = work.pop()
        for key, value in overlay.items():
            below = target.get(key)
            if isinstance(value, dict) and isinstance(below, dict):
                target[key] = dict(below)
                work.append((target[key], value))
            else:
                target[key] = value
    return root


def _read_json_document(path: str) -> dict:
    try:
        text = Path(path).read_text()
    except OSError as exc:
        raise errors.IoFailure(f"cannot read config {path}: {exc}") from exc
    try:
        return json.loads(text)
    except json.JSONDecodeError as exc:
        raise errors.ConfigError(f"config is not valid JSON: {exc}") from exc


def load_config(args, defaults: dict, schema: dict) -> dict:
    """Defaults, overlaid with the --config document, schema-validated."""
    cfg = merged(defaults, _read_json_document(args.config)) if args.config else dict(defaults)
    try:
        import jsonschema
    except ImportError:  # pragma: no cover - jsonschema ships with the image
        return cfg
    problems = sorted(jsonschema.Draft7Validator(schema).iter_errors(cfg), key=str)
    if problems:
        raise errors.ConfigError(f"config invalid: {problems[0].message}")
    return cfg


def configure_threads(n: int | None) -> None:
    """--threads / CYLTOMO_THREADS (the reference caps its numba pool,
    cyltomo/cli.py:45-53): here the cap applies to the host worker pool that
    stages pageable projections (recon._stage_pool) and to torch's intra-op
    threads; the GPU kernels are unaffected."""
    n = n if n is not None else (os.environ.get("CYLTOMO_THREADS") or None)
    if n is None:
        return
    n = max(1, int(n))
    os.environ["CT_HOST_THREADS"] = str(n)
    try:
        import torch
        torch.set_num_threads(n)
    except Exception:  # pragma: no cover
        pass


GEOMETRY_SCHEMA = {
    "type": "object",
    "properties": {
        "sdd_mm": {"type": "number"}, "sod_mm": {"type": "number"},
        "det_cols": {"type": "integer", "minimum": 1},
        "det_rows": {"type": "integer", "minimum": 1},
        "pixel_pitch_mm": {"type": "number", "exclusiveMinimum": 0},
        "principal_point_px": {"type": "array", "minItems": 2, "maxItems": 2},
        "stage_angles_rad": {"type": "array"},
        "n_views": {"type": "integer", "minimum": 1},
        "last_angle_deg": {"type": "number"}, "full_turn": {"type": "boolean"},
    },
}


def geometry_from_config(d: dict) -> ScanGeometry:
    """(cyltomo/cli.py:83-101)"""
    if "stage_angles_rad" in d:                 # an explicit geometry document
        return ScanGeometry.from_dict(d)
    n_views = int(d.get("n_views", 21))
    angles = (full_turn_angles(n_views) if d.get("full_turn", False) else
              make_circular_trajectory(n_views, math.radians(d.get("last_angle_deg", 200.0))))
    cols, rows = int(d.get("det_cols", 96)), int(d.get("det_rows", 192))
    pp = d.get("principal_point_px")
    return ScanGeometry(float(d.get("sdd_mm", 791.0)), float(d.get("sod_mm", 679.0)), cols, rows,
                        float(d.get("pixel_pitch_mm", 0.66)),
                        tuple(pp) if pp else ((cols - 1) / 2.0, (rows - 1) / 2.0), angles)


def write_csv_rows(path, header, rows) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(header)
        w.writerows(rows)


def fmt(x: float) -> str:
    return f"{x:.9g}"


SIMULATE_SCHEMA = {
    "type": "object",
    "properties": {"volume": {"type": "string"}, "geometry": GEOMETRY_SCHEMA,
                   "step_mm": {"type": ["number", "null"]},
                   "supersample": {"type": "integer", "minimum": 1},
                   "noise_sigma": {"type": "number", "minimum": 0}},
    "required": ["volume"],
}


def cmd_simulate(args) -> int:
    defaults = {"geometry": dict(PAPER_GEOMETRY) if args.preset == "paper" else {},
                "step_mm": None, "supersample": 1, "noise_sigma": 0.0}
    cfg = load_config(args, defaults, SIMULATE_SCHEMA)
    if args.views is not None:
        cfg["geometry"]["n_views"] = args.views
    vol = io.read_volume(cfg["volume"], device=True)
    geom = geometry_from_config(cfg["geometry"])
    ps = simulate_scan(vol, geom, RaySamplingConfig(step=cfg["step_mm"],
                                                    supersample=cfg["supersample"]),
                       cfg["noise_sigma"], np.random.default_rng(args.seed))
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    path = io.write_projections(ps, out / "projections")
    print(f"wrote {path} ({geom.n_proj} views)")
    return EXIT_OK


RECON_SCHEMA = {
    "type": "object",
    "properties": {
        "projections": {"type": "string"},
        "grid": {"type": "object",
                 "properties": {"shape": {"type": "array", "minItems": 3, "maxItems": 3},
                                "radius_mm": {"type": "number"},
                                "height_mm": {"type": "number"}},
                 "required": ["shape", "radius_mm", "height_mm"]},
        "cartesian": {"type": ["object", "null"]},
        "pose": {"type": ["string", "object"]},
        "pose_params": {"type": "object"},
        "sart": {"type": "object"},
        "initial": {"type": ["string", "null"]},
        "weights": {"type": ["string", "null"]},
        "resample_initial": {"type": "boolean"},
        "step_mm": {"type": ["number", "null"]},
    },
    "required": ["projections", "grid"],
}


# pose-parameter keys of a config document: (key, converter, default); the
# reference's names and defaults (cyltomo/cli.py:143-158)
_POSE_KEYS = (("threshold_level", None, "auto"), ("threshold_levels", int, 1),
              ("threshold_span", float, 0.0), ("dilation_radius", int, 0), ("band", int, 1),
              ("nuisance_level", None, None), ("nuisance_dilation", int, 2),
              ("exclude_rects", lambda v: tuple(tuple(r) for r in v), ()),
              ("estimate_gamma", bool, False), ("strip_offset", float, 0.0),
              ("strip_width", float, 1.0))


def pose_params_from_config(d: dict) -> PoseFitParams:
    """PoseFitParams from a config document (cyltomo/cli.py:143-158)."""
    kw = {}
    for key, conv, default in _POSE_KEYS:
        v = d.get(key, default)
        kw[key] = conv(v) if (conv is not None and key in d) else v
    kw["lm"] = LmConfig(**d["lm"]) if d.get("lm") else LmConfig()
    return PoseFitParams(**kw)


# the reference DeviceSpec's pose parameters (cyltomo/experiments.py:219-223):
# the threshold isolates the dense core, the 9-level ladder recovers sub-pixel
# corner positions
DEVICE_POSE_PARAMS = dict(threshold_level=1.8, threshold_levels=9, threshold_span=1.0, band=1)

POSE_SCHEMA = {
    "type": "object",
    "properties": {"projections": {"type": "string"}, "params": {"type": "object"}},
}


def cmd_pose(args) -> int:
    """(cyltomo/cli.py:286-313) -- pose fit of a projection set.  The
    reference's pose-precision study (experiments.py:342) is out of scope."""
    cfg = load_config(args, {"params": {}}, POSE_SCHEMA)
    if "projections" not in cfg:
        raise errors.ConfigError("pose needs \"projections\"")
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    ps = io.read_projections(cfg["projections"], device=True)
    result = fit_pose(ps, pose_params_from_config(cfg["params"]))
    io.write_pose(result.to_dict(), out / "pose.json")
    print(f"wrote {out / 'pose.json'}")
    return EXIT_OK


def sart_config_from(cfg: dict, seed: int) -> SartConfig:
    sart = dict(cfg.get("sart", {}))
    subsets = sart.get("subsets")
    return SartConfig(relaxation=float(sart.get("relaxation", 1.0)),
                      n_iterations=int(sart.get("passes", 1)),
                      projection_order=sart.get("order", "acquisition"),
                      order_seed=int(sart.get("order_seed", seed)),
                      nonnegativity=bool(sart.get("nonnegativity", True)),
                      resample_initial=bool(cfg.get("resample_initial", False)),
                      sampling=RaySamplingConfig(step=cfg.get("step_mm")),
                      n_subsets=None if subsets is None else int(subsets),
                      compute_residuals=bool(sart.get("residuals", True)))


def cmd_reconstruct(args) -> int:
    """(cyltomo/cli.py:341-397)"""
    defaults = {"pose": "estimate", "pose_params": {}, "sart": {}, "initial": None,
                "weights": None, "resample_initial": False, "step_mm": None, "cartesian": None}
    cfg = load_config(args, defaults, RECON_SCHEMA)
    if args.init is not None:
        cfg["initial"] = None if args.init == "none" else args.init
    if args.weights is not None:
        cfg["weights"] = None if args.weights == "none" else args.weights
    ps = io.read_projections(cfg["projections"], device=True)
    if isinstance(cfg["pose"], dict):
        pose = Pose.from_dict(cfg["pose"])
    elif cfg["pose"] == "estimate":
        pose = fit_pose(ps, pose_params_from_config(cfg["pose_params"])).pose
    else:
        pose = io.read_pose(cfg["pose"])
    if cfg["cartesian"]:
        c = cfg["cartesian"]
        grid = CartGrid.centered(*(int(v) for v in c["shape"]), float(c["voxel_size_mm"]),
                                 center=c.get("center_mm", (0.0, 0.0, 0.0)))
    else:
        g = cfg["grid"]
        nh, nt, nr = (int(v) for v in g["shape"])
        grid = CylGrid(nh, nt, nr, g["radius_mm"], g["height_mm"], pose=pose)
    run_cfg = sart_config_from(cfg, args.seed)
    if cfg["initial"]:
        run_cfg.initial = io.read_volume(cfg["initial"], device=True)
    if cfg["weights"]:
        run_cfg.weights = io.read_volume(cfg["weights"], device=True).mu
    vol, report = sart_run(ps, grid, run_cfg)
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    path = io.write_volume(vol, out / "volume")
    (out / "report.json").write_text(json.dumps(
        {"residuals": report.residuals, "wall_time_s": report.wall_time,
         "config": report.config, "pose": pose.to_dict()}, indent=2) + "\n")
    write_csv_rows(out / "residuals.csv", ["pass", "residual_l2"],
                   [(k + 1, fmt(r)) for k, r in enumerate(report.residuals)])
    last = report.residuals[-1] if report.residuals else float("nan")
    print(f"wrote {path}; residual after last pass: {last:.6g}")
    return EXIT_OK


BATCH_SCHEMA = {
    "type": "object",
    "properties": {
        "n_samples": {"type": "integer", "minimum": 2},
        "missing_fraction": {"type": "number", "exclusiveMinimum": 0, "exclusiveMaximum": 1},
        "strategies": {"type": "array", "items": {"enum": ["a", "b", "c", "d"]}},
        "recon_shape": {"type": "array", "minItems": 3, "maxItems": 3},
        "sim_shape": {"type": "array", "minItems": 3, "maxItems": 3},
        "passes": {"type": "integer", "minimum": 1},
        "noise_sigma": {"type": "number", "minimum": 0},
        "pose_source": {"enum": ["estimated", "true"]},
        "geometry": GEOMETRY_SCHEMA,
    },
}


def _device_components(present: bool):
    """The reference's DeviceSpec assembly (cyltomo/experiments.py:180-210)."""
    return [ComponentSpec("body", mu=0.04),
            ComponentSpec("core", mu=1.0, r_range=(0.0, 1.5), h_range=(-28.0, 28.0)),
            ComponentSpec("part", mu=0.3, r_range=(4.0, 6.0), h_range=(-10.0, 10.0),
                          present=present)]


def _random_pose(rng, tilt_sigma_deg: float = 1.5, shift_mm: float = 2.0) -> Pose:
    """Same draws, same order as cyltomo/experiments.py:246-255."""
    beta = abs(rng.normal(0.0, math.radians(tilt_sigma_deg)))
    alpha = rng.uniform(-math.pi, math.pi)
    gamma = rng.uniform(-math.pi, math.pi)
    t = np.array([rng.uniform(-shift_mm, shift_mm), rng.uniform(-shift_mm, shift_mm),
                  rng.uniform(-shift_mm, shift_mm)])
    return Pose(alpha, beta, gamma, t=t)


def cmd_batch(args) -> int:
    """Batch inspection study (cyltomo/cli.py:476-515, experiments.py:282-335) on
    the B200; samples are sharded over ranks under torchrun."""
    import warnings
    defaults = {"n_samples": 50, "missing_fraction": 0.4, "strategies": ["a", "c"],
                "recon_shape": [240, 40, 60], "sim_shape": [240, 16, 60], "passes": 1,
                "noise_sigma": 0.02, "pose_source": "estimated", "geometry": {}}
    cfg = load_config(args, defaults, BATCH_SCHEMA)
    strategies = sorted(set(args.strategies)) if args.strategies else list(cfg["strategies"])
    geom = geometry_from_config(cfg["geometry"])
    radius, height = 8.0, 60.0
    rshape = tuple(int(v) for v in cfg["recon_shape"])
    sshape = tuple(int(v) for v in cfg["sim_shape"])
    rng = np.random.default_rng(args.seed)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        template = make_assembly_phantom(_device_components(True), CylGrid(*rshape, radius, height))
    roi = ComponentSpec("roi", mu=0.0, r_range=(4.0, 6.0), h_range=(-10.0, 10.0))
    weights = make_weight_map([(roi, 1.0)], template.grid, default_weight=0.3)
    n = int(cfg["n_samples"])
    missing = set(rng.choice(n, size=int(round(cfg["missing_fraction"] * n)),
                             replace=False).tolist())
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rows = []
    for s in range(n):
        present = s not in missing
        true_pose = _random_pose(rng)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            vol = make_assembly_phantom(_device_components(present),
                                        CylGrid(*sshape, radius, height, true_pose))
        # the noise draw advances the shared stream on every rank
        ps = simulate_scan(vol, geom, RaySamplingConfig(), cfg["noise_sigma"], rng)
        if s % world != rank:
            continue
        if cfg["pose_source"] == "estimated":
            pose = fit_pose(ps, PoseFitParams(**DEVICE_POSE_PARAMS)).pose
        else:
            pose = true_pose
        grid = CylGrid(*rshape, radius, height, pose=pose)
        row = {"sample": s, "present": present}
        for st in strategies:
            c = SartConfig(relaxation=1.0, n_iterations=int(cfg["passes"]))
            if st in ("b", "c"):
                c.initial = template
            if st in ("c", "d"):
                c.weights = weights
            rec, _ = sart_run(ps, grid, c)
            row[st] = presence_metric(rec, roi)
        rows.append(row)
    if world > 1:
        import torch.distributed as dist
        from .distributed import init_from_env
        init_from_env()
        gathered = [None] * world
        dist.all_gather_object(gathered, rows)
        rows = sorted((r for part in gathered for r in part), key=lambda r: r["sample"])
        if rank != 0:
            return EXIT_OK
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    write_csv_rows(out / "batch_results.csv",
                   ["sample", "present", *[f"presence_{st}" for st in strategies]],
                   [(r["sample"], int(r["present"]), *[fmt(r[st]) for st in strategies])
                    for r in rows])
    srows = []
    for st in strategies:
        pres = np.array([r[st] for r in rows if r["present"]])
        miss = np.array([r[st] for r in rows if not r["present"]])
        pooled = math.sqrt(((pres.size - 1) * pres.var(ddof=1) + (miss.size - 1)
                            * miss.var(ddof=1)) / max(pres.size + miss.size - 2, 1))
        gap = abs(pres.mean() - miss.mean()) / pooled if pooled > 0 else math.inf
        srows.append((st, fmt(pres.mean()), fmt(miss.mean()), fmt(pres.std(ddof=1)),
                      fmt(miss.std(ddof=1)), fmt(gap)))
        print(f"strategy {st}: gap = {gap:.3f}")
    write_csv_rows(out / "batch_summary.csv", ["strategy", "mean_present", "mean_missing",
                                               "std_present", "std_missing",
                                               "standardized_gap"], srows)
    print(f"wrote {out / 'batch_summary.csv'}")
    return EXIT_OK


# sub-command -> (handler, help, extra arguments)
COMMANDS = {
    "simulate": (cmd_simulate, "forward-project a volume",
                 [("--views", dict(type=int, help="override projection count"))]),
    "pose": (cmd_pose, "estimate the object pose", []),
    "reconstruct": (cmd_reconstruct, "(OS-)SART reconstruction",
                    [("--init", dict(metavar="none|PATH", help="initial volume")),
                     ("--weights", dict(metavar="none|PATH",
                                        help="back-projection weight map"))]),
    "batch": (cmd_batch, "batch inspection study",
              [("--strategies", dict(nargs="+", choices=["a", "b", "c", "d"]))]),
}
COMMON_ARGS = (
    ("--config", dict(metavar="PATH", help="JSON config document")),
    ("--seed", dict(type=int, default=0, help="RNG seed (default 0)")),
    ("--threads", dict(type=int, default=None, help="host worker thread cap "
                                                    "(env CYLTOMO_THREADS)")),
    ("--preset", dict(choices=["paper", "desk"], default="desk",
                      help="scale preset (default desk)")),
    ("--out", dict(metavar="DIR", default=".", help="output directory")),
)


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="cyltomo-b200",
                                     description="B200 cone-beam FP/BP/(OS-)SART on "
                                                 "cylindrical grids")
    shared = argparse.ArgumentParser(add_help=False)
    for flag, kw in COMMON_ARGS:
        shared.add_argument(flag, **kw)
    sub = parser.add_subparsers(dest="command", required=True)
    for name, (handler, text, extra) in COMMANDS.items():
        cp = sub.add_parser(name, parents=[shared], help=text)
        for flag, kw in extra:
            cp.add_argument(flag, **kw)
        cp.set_defaults(func=handler)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        configure_threads(args.threads)
        return args.func(args)
    except errors.CylTomoError as exc:
        code, prefix = next((c, pfx) for kinds, c, pfx in EXIT_MAP if isinstance(exc, kinds))
        print(f"{prefix}: {exc}", file=sys.stderr)
        return code


if __name__ == "__main__":
    sys.exit(main())
