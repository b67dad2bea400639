"""Would staging volume tiles in shared memory (north_star: "shared-memory/TMA
staging of volume tiles") cut the FP's on-chip traffic?  Host-side geometry
estimate for seeded CTAs of a workload (C5 by default).

For each sampled CTA (16 x 8 rays, the FP's block) the rays are marched with
the reference's sampling (t0 + (k + 0.5) step) and the GL_QUAD cells each
sample reads are listed.  Reported per CTA:

* cell-entry loads -- what the kernel loads today (one per sample that
  leaves its predecessor's cell, i.e. after cell reuse along the ray);
* distinct cells -- the minimum any staging scheme must bring on chip;
* reuse = loads / distinct -- the most a perfect CTA-wide cache could save;
* the bounding box (cells) of the CTA's cells in one 64-sample depth window
  -- what a tile to stage would have to hold (16 B per cell and layer).

    python tools/fp_stage_estimate.py [--config c5|c2] [--ctas 24]
"""
import argparse
import json
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from paper_2005_11976_b200 import _device as D  # noqa: E402
from paper_2005_11976_b200 import workloads as W  # noqa: E402
from paper_2005_11976_b200.projector import RaySamplingConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--ctas", type=int, default=24)
args = ap.parse_args()

wl = W.c5_object(0) if args.config == "c5" else W.c2_medium()
g, geom = wl.grid, wl.geom
step = RaySamplingConfig().step_for(g)
tab = D.ray_view_table(g, geom, np.arange(geom.n_proj)).reshape(geom.n_proj, 4, 3)
rng = np.random.default_rng(0)
idr, idt, idh = g.n_r / g.radius, g.n_theta / (2 * math.pi), g.n_h / g.height


def cells_of_ray(src, d):
    a = d[0] ** 2 + d[1] ** 2
    b = src[0] * d[0] + src[1] * d[1]
    c = src[0] ** 2 + src[1] ** 2 - g.radius ** 2
    disc = b * b - a * c
    if disc <= 0:
        return None
    hz = 0.5 * g.height
    tz = sorted([(-hz - src[2]) / d[2], (hz - src[2]) / d[2]])
    t0 = max((-b - math.sqrt(disc)) / a, tz[0], 0.0)
    t1 = min((-b + math.sqrt(disc)) / a, tz[1])
    if t1 <= t0:
        return None
    t = t0 + (np.arange(int(math.ceil((t1 - t0) / step))) + 0.5) * step
    x, y, z = src[0] + t * d[0], src[1] + t * d[1], src[2] + t * d[2]
    ic = np.floor(np.sqrt(x * x + y * y) * idr + 0.5).astype(np.int64)
    th = np.mod(np.arctan2(y, x), 2 * math.pi)
    jc = np.floor(th * idt + 0.5).astype(np.int64)
    kc = np.floor(z * idh + 0.5 * g.n_h + 0.5).astype(np.int64)
    return np.stack([kc, jc, ic], axis=1)


rows = []
while len(rows) < args.ctas:
    v = int(rng.integers(geom.n_proj))
    src, origin, du, dv = tab[v]
    c0 = int(rng.integers(0, geom.det_cols // 16)) * 16
    r0 = int(rng.integers(geom.det_rows // 4, 3 * geom.det_rows // 4) // 8) * 8
    per_ray = []
    for rr in range(r0, r0 + 8):
        for cc in range(c0, c0 + 16):
            d = origin + cc * du + rr * dv - src
            d /= np.linalg.norm(d)
            cl = cells_of_ray(src, d)
            if cl is not None:
                per_ray.append(cl)
    if len(per_ray) < 64:
        continue
    loads = sum(int(1 + np.count_nonzero(np.any(np.diff(cl, axis=0) != 0, axis=1)))
                for cl in per_ray)
    allc = np.concatenate(per_ray)
    distinct = len(np.unique(allc, axis=0))
    # bounding box of one 64-sample window in the middle of the rays
    win = []
    for cl in per_ray:
        m = len(cl) // 2
        win.append(cl[max(m - 32, 0):m + 32])
    w = np.concatenate(win)
    span = (w.max(axis=0) - w.min(axis=0) + 1)
    box = int(np.prod(span))
    rows.append({"view": v, "rays": len(per_ray), "cell_entry_loads": loads,
                 "distinct_cells": distinct, "reuse": loads / distinct,
                 "window64_box_cells_khr": [int(x) for x in span],
                 "window64_box_kib": box * 32 / 1024,
                 "window64_distinct_cells": int(len(np.unique(w, axis=0)))})

reuse = np.array([r["reuse"] for r in rows])
box = np.array([r["window64_box_kib"] for r in rows])
out = {"config": args.config, "ctas": len(rows), "step_mm": step,
       "reuse_median": float(np.median(reuse)), "reuse_max": float(reuse.max()),
       "window64_box_kib_median": float(np.median(box)),
       "window64_box_kib_p90": float(np.quantile(box, 0.9)), "rows": rows}
print(json.dumps(out, indent=1))
