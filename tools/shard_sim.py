"""Per-rank compute of the angle-sharded OS-SART (distributed.py) replayed on ONE
GPU, rank by rank, for G = 1, 2, 4, 8: the FP row range, the voxel-range BP
update and the gather packing each rank runs per C2 subset, plus its share of
the residual FP, timed with CUDA events.  No collective runs (one GPU); the
max over ranks of the compute per iteration is the compute-only bound on the
N-GPU iteration time (collectives come on top: all-gather of the corrections
and of mu per subset, one small all-reduce per pass).

    python tools/shard_sim.py [--views 360]
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_11976_b200 as P  # noqa: E402
from paper_2005_11976_b200 import _device as D  # noqa: E402
from paper_2005_11976_b200 import distributed as PD  # noqa: E402
from paper_2005_11976_b200 import workloads as W  # noqa: E402
from paper_2005_11976_b200.recon import SartRun, make_update  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--views", type=int, default=360)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()

wl = W.c2_medium(n_views=args.views)
vol = P.CylVolume(wl.grid, torch.as_tensor(wl.mu, device="cuda"))
ps = P.forward_project_all(vol, wl.geom)
run = SartRun(P.ProjectionSet(wl.geom, ps.images), wl.grid,
              P.SartConfig(relaxation=0.3, n_iterations=1, n_subsets=8))
e = run.eng
H, Wd = wl.geom.det_rows, wl.geom.det_cols
n_proj = wl.geom.n_proj
nvox = wl.grid.n_voxels
tile = e.row_tile()
scratch = e.residual_scratch(n_proj).clone().zero_()
rest = np.setdiff1d(np.arange(n_proj), run.subsets[0])
mu = run.mu.clone().copy_(torch.as_tensor(wl.mu, device="cuda") * 0.9)
quads = e.alloc_quads(max(len(s) for s in run.subsets))


def cost(views):
    return e.row_samples(np.asarray(views)).ravel() + 8.0 * Wd


def timed(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(args.reps):
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def rows_call(views, bounds, r, resid):
    lo, hi = int(bounds[r]), int(bounds[r + 1])
    if hi <= lo:
        return lambda: None
    v0, v1 = lo // H, (hi - 1) // H
    slots = D.upload_i32(views[v0:v1 + 1])
    out = torch.empty((hi - lo) * Wd, device="cuda")
    if resid:
        return lambda: e.residual_rows(mu, run.p_meas, slots, v1 - v0 + 1, n_proj, scratch,
                                       lo - v0 * H, hi - v0 * H, run.gather)
    return lambda: e.correction_rows(mu, run.p_meas, slots, v1 - v0 + 1, out, lo - v0 * H,
                                     hi - v0 * H, 0, None, run.gather)


out = {"workload": "C2 OS-SART iteration (8 subsets x 45 views, residual over 360)",
       "note": "compute only, each rank's work replayed on one B200; no collectives",
       "per_G": {}}
e.pack(mu, run.gather)
t_pack = timed(lambda: e.pack(mu, run.gather))
for G in (1, 2, 4, 8):
    per_rank = np.zeros(G)
    for s, (sub, slots) in enumerate(zip(run.subsets, run.subset_slots)):
        sub = np.asarray(sub)
        b = PD.row_bounds(len(sub), H, G, tile, cost(sub))
        corr = torch.zeros((len(sub), H, Wd), device="cuda")
        e.correction(mu, run.p_meas, slots, len(sub), corr, run.gather)
        e.pack_quads(corr, len(sub), quads)
        for r in range(G):
            t_fp = timed(rows_call(sub, b, r, False))
            off, cnt, _ = PD.shard_range(nvox, r, G)
            m2 = mu.clone()
            upd = make_update(m2, None, run.cfg)
            t_bp = timed(lambda: (e.pack_quads(corr, len(sub), quads),
                                  e.bp_update_range(corr, slots, len(sub), upd, off, cnt, quads)))
            per_rank[r] += t_fp + t_bp + t_pack
    rb = PD.row_bounds(len(rest), H, G, tile, cost(rest))
    b0 = PD.row_bounds(len(run.subsets[0]), H, G, tile, cost(np.asarray(run.subsets[0])))
    for r in range(G):
        per_rank[r] += timed(rows_call(rest, rb, r, True)) + timed(
            rows_call(np.asarray(run.subsets[0]), b0, r, True)) + t_pack
    out["per_G"][G] = {"max_rank_ms": float(per_rank.max()), "min_rank_ms": float(per_rank.min())}
base = out["per_G"][1]["max_rank_ms"]
for G, d in out["per_G"].items():
    d["compute_efficiency"] = base / (G * d["max_rank_ms"])
print(json.dumps(out))
