"""Would a per-segment polynomial in the sample index replace the FP's
per-sample sqrt / rcp / atan?  (VERDICT r01 "next round" item 5.)

For seeded rays of a workload (C5 by default) this evaluates, in fp64, the
march's r and theta cell indices along each ray (r = sqrt(s^2 +
d0^2), theta = phi + 2 atan(s / (r + d0)), s linear in the sample index k) and
replaces them on every segment of M consecutive samples by the polynomial of
degree p interpolating them at p + 1 Chebyshev points of the segment.  It
reports the largest index error and the share of segments whose error
exceeds 1e-4 / 1e-3 cells -- against the fp32 evaluation the kernel does now
(~1 ulp of the index, <= 6e-5 cells at C5).

    python tools/segment_poly_error.py [--config c5|c2] [--rays 4000]
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
ap.add_argument("--rays", type=int, default=4000)
args = ap.parse_args()

wl = W.c5_object(0) if args.config == "c5" else W.c2_medium()
g, geom = wl.grid, wl.geom
step = RaySamplingConfig().step_for(g)
tab = D.ray_view_table(g, geom, np.arange(geom.n_proj)).reshape(geom.n_proj, 4, 3)
rng = np.random.default_rng(0)
idr, idt = g.n_r / g.radius, g.n_theta / (2 * math.pi)
rays = []
while len(rays) < args.rays:
    v = int(rng.integers(geom.n_proj))
    src, origin, du, dv = tab[v]
    u, w = rng.uniform(0, geom.det_cols - 1), rng.uniform(0, geom.det_rows - 1)
    d = origin + u * du + w * dv - src
    d /= np.linalg.norm(d)
    a = d[0] ** 2 + d[1] ** 2
    b = src[0] * d[0] + src[1] * d[1]
    c = src[0] ** 2 + src[1] ** 2 - g.radius ** 2
    disc = b * b - a * c
    if disc <= 0:
        continue
    t0 = (-b - math.sqrt(disc)) / a
    t1 = (-b + math.sqrt(disc)) / a
    hz = 0.5 * g.height
    tz = sorted([(-hz - src[2]) / d[2], (hz - src[2]) / d[2]])
    t0, t1 = max(t0, tz[0], 0.0), min(t1, tz[1])
    if t1 - t0 < 64 * step:
        continue
    rays.append((src.copy(), d.copy(), t0, int(math.ceil((t1 - t0) / step))))


def indices(ray, k):
    """r and (unwrapped) theta cell indices at fractional sample positions k."""
    src, d, t0, _ = ray
    t = t0 + (np.asarray(k, dtype=float) + 0.5) * step
    x, y = src[0] + t * d[0], src[1] + t * d[1]
    return np.sqrt(x * x + y * y) * idr, np.unwrap(np.arctan2(y, x)) * idt


out = {"config": args.config, "rays": len(rays), "step_mm": step,
       "note": "max |index error| of per-segment Chebyshev interpolation (cells)", "cases": []}
for M in (4, 8, 16, 32):
    for p in (2, 3):
        nodes = 0.5 * (M - 1) * (1 - np.cos((2 * np.arange(p + 1) + 1) * math.pi / (2 * p + 2)))
        errs = {"r": [], "theta": []}
        V = np.vander(nodes, p + 1)
        j = np.arange(M, dtype=float)
        for ray in rays:
            n = ray[3] // M * M
            k0 = np.arange(0, n, M, dtype=float)[:, None]
            kk = (k0 + j[None]).ravel()
            kn = (k0 + nodes[None]).ravel()
            exact = indices(ray, kk)
            at_nodes = indices(ray, np.sort(np.concatenate([kn, kk])))
            # theta unwrapped over the merged grid keeps nodes and samples consistent
            merged = np.sort(np.concatenate([kn, kk]))
            pos_n = np.searchsorted(merged, kn)
            pos_k = np.searchsorted(merged, kk)
            for idx, name in ((0, "r"), (1, "theta")):
                fn = at_nodes[idx][pos_n].reshape(-1, p + 1)
                fk = at_nodes[idx][pos_k].reshape(-1, M) if name == "theta" else \
                    exact[idx].reshape(-1, M)
                coef = np.linalg.solve(V, fn.T).T
                approx = np.stack([np.polyval(cf, j) for cf in coef])
                errs[name].append(np.abs(approx - fk).max(axis=1))
        row = {"segment": M, "degree": p}
        for name in ("r", "theta"):
            e = np.concatenate(errs[name])
            row[name] = {"max": float(e.max()), "p99": float(np.quantile(e, 0.99)),
                         "share_gt_1e-4": float((e > 1e-4).mean()),
                         "share_gt_1e-3": float((e > 1e-3).mean())}
        out["cases"].append(row)
print(json.dumps(out, indent=1))
