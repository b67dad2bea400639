"""The whole C5 configuration (BASELINE configs[4]) on one B200, as the
reference's batch workflow runs it (cyltomo/experiments.py:282-340): 64
seeded objects, each the template with one inclusion missing or added and its
own pose, reconstructed with 15 OS-SART iterations (6 subsets, lambda 0.3)
from the shared template through the public API with pinned HOST projections
(upload inside the timed call) and the volume returned to the host.

Scored like the reference's presence study: per object the mean attenuation
of the reconstruction in the changed inclusion's region (presence_metric),
against the template's and the truth's -- the inspection decision is
"changed" when the reconstruction moved more than half-way from the template
towards the truth.

    python tools/c5_full.py [--objects 64] [--iterations 15] [--out FILE]
"""
import argparse
import json
import math
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_11976_b200 as P  # noqa: E402
from paper_2005_11976_b200 import workloads as W  # noqa: E402
from paper_2005_11976_b200.distributed import reconstruct_batch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--objects", type=int, default=64)
ap.add_argument("--iterations", type=int, default=15)
ap.add_argument("--out", default=None)
args = ap.parse_args()


def changed_spheres(base, obj):
    key = lambda s: (round(s.r, 9), round(s.theta, 9), round(s.h, 9), round(s.radius, 9))  # noqa
    b = {key(s): s for s in base.spheres}
    o = {key(s): s for s in obj.spheres}
    return ([("missing", s) for k, s in b.items() if k not in o]
            + [("added", s) for k, s in o.items() if k not in b])


template_host = W.c5_template()
template = P.CylVolume(P.CylGrid(512, 1024, 384, W.RADIUS, W.HEIGHT),
                       torch.as_tensor(template_host, device="cuda"))
rows, t_rec, t_gen = [], 0.0, 0.0
for k in range(args.objects):
    g0 = time.perf_counter()
    wl = W.c5_object(k)
    truth = torch.as_tensor(wl.mu, device="cuda")
    sim = P.forward_project_all(P.CylVolume(wl.grid, truth), wl.geom)   # "measured" scan
    host = torch.empty(tuple(sim.images.shape), dtype=torch.float32, pin_memory=True)
    host.copy_(sim.images)
    del sim
    ps = P.ProjectionSet(wl.geom, host.numpy())
    cfg = P.SartConfig(relaxation=wl.relaxation, n_iterations=args.iterations,
                       n_subsets=wl.n_subsets,
                       initial=P.CylVolume(wl.grid, template.mu))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    vol, rep = reconstruct_batch([(ps, wl.grid)], cfg, rank=0, world=1)[0]
    mu = np.asarray(vol.mu)                                   # host volume back
    t1 = time.perf_counter()
    t_rec += t1 - t0
    t_gen += t0 - g0
    for kind, s in changed_spheres(wl.extra["template_phantom"], wl.extra["phantom"]):
        roi = W.rasterize_cyl(W.Phantom(shells=[], spheres=[W.Sphere(s.r, s.theta, s.h,
                                                                     s.radius, 1.0)]),
                              wl.grid) > 0.5
        if not roi.any():
            continue
        rec, tru, tpl = (float(x[roi].mean()) for x in (mu, wl.mu, template_host))
        moved = (rec - tpl) / (tru - tpl) if tru != tpl else float("nan")
        rows.append({"object": k, "change": kind, "roi_voxels": int(roi.sum()),
                     "recon": rec, "truth": tru, "template": tpl,
                     "fraction_of_change_recovered": moved, "detected": bool(moved > 0.5),
                     "residual_first": rep.residuals[0], "residual_last": rep.residuals[-1],
                     "seconds": t1 - t0})
    print(f"object {k}: {t1 - t0:.2f} s, residual {rep.residuals[0]:.4g} -> "
          f"{rep.residuals[-1]:.4g}", file=sys.stderr, flush=True)
    del truth, host, ps, vol

det = [r["detected"] for r in rows]
frac = np.array([r["fraction_of_change_recovered"] for r in rows])
out = {"workload": f"C5 full: {args.objects} objects x {args.iterations} OS-SART iterations "
                   "(6 subsets, lambda 0.3, template init), grid (512,1024,384), 120 views 1024^2",
       "api": "distributed.reconstruct_batch, pinned host projections in, host volume out",
       "reconstruction_s_total": t_rec, "s_per_object": t_rec / args.objects,
       "s_per_object_iteration": t_rec / (args.objects * args.iterations),
       "input_generation_s_total (not timed: our FP simulates the scans)": t_gen,
       "changes": len(rows), "detected": int(sum(det)),
       "fraction_of_change_recovered": {"min": float(frac.min()), "median": float(np.median(frac)),
                                        "max": float(frac.max())},
       "rows": rows}
txt = json.dumps(out, indent=1)
if args.out:
    Path(args.out).write_text(txt)
print(json.dumps({k: v for k, v in out.items() if k != "rows"}))
