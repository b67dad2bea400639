"""Per-rank compute of the SLAB-decomposed angle-sharded OS-SART (slab.py)
replayed on ONE GPU, rank by rank, for G = 1, 2, 4, 8 (C2): each rank's band
FP from its window-packed gather layout, its slab's BP update and its window
pack per subset, plus its bands of the residual FP, timed with CUDA events;
and the bytes each rank receives per subset (correction rows + mu layers)
against the flattened-row driver's all-gathers (tools/shard_sim.py is the
same replay for that driver).  No collective runs (one GPU).

    python tools/slab_sim.py [--views 360] [--config c2|c5]
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
from paper_2005_11976_b200 import slab as S  # noqa: E402
from paper_2005_11976_b200 import workloads as W  # noqa: E402
from paper_2005_11976_b200.recon import SartRun, make_update  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--views", type=int, default=360)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--config", default="c2")
args = ap.parse_args()

if args.config == "c5":
    wl = W.c5_object(0)
    init = P.CylVolume(wl.grid, torch.as_tensor(W.c5_template(), device="cuda"))
    n_sub = 6
else:
    wl = W.c2_medium(n_views=args.views)
    init, n_sub = None, 8
vol = P.CylVolume(wl.grid, torch.as_tensor(wl.mu, device="cuda"))
ps = P.forward_project_all(vol, wl.geom)
del vol
run = SartRun(P.ProjectionSet(wl.geom, ps.images), wl.grid,
              P.SartConfig(relaxation=0.3, n_iterations=1, n_subsets=n_sub, initial=init))
e = run.eng
H, Wd = wl.geom.det_rows, wl.geom.det_cols
n_proj = wl.geom.n_proj
n_layers = wl.grid.shape[0]
layer = wl.grid.shape[1] * wl.grid.shape[2]
tile = e.row_tile()
scratch = e.residual_scratch(n_proj).clone().zero_()
mu = run.mu.clone().copy_(torch.as_tensor(wl.mu, device="cuda") * 0.9)
quads = e.alloc_quads(max(len(s) for s in run.subsets))
allv = np.arange(n_proj)
costs = e.row_samples(allv).astype(np.float64) + 8.0 * Wd
cells = e.row_cells(allv)
rest = np.setdiff1d(allv, run.subsets[0])


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


def bands_of(plan, views, r):
    b = np.array([plan.band(int(v), r) for v in views], dtype=np.int32)
    rows = int((b[:, 1] - b[:, 0]).max())
    return D.upload_i32(b.reshape(-1)), rows


out = {"workload": f"{args.config.upper()} OS-SART iteration ({n_sub} subsets, residual over "
                   f"{n_proj} views), slab decomposition",
       "note": "compute only, each rank's work replayed on one B200; no collectives",
       "per_G": {}}
for G in (1, 2, 4, 8):
    plan = S.SlabPlan(G, n_layers, H, tile, costs, cells,
                      lambda v, a, b: S.slab_rows_needed(wl.grid, wl.geom, v, a, b, H))
    per_rank = np.zeros(G)
    parts = {"fp": np.zeros(G), "bp": np.zeros(G), "pack": np.zeros(G)}
    recv_bytes = np.zeros(G)
    for r in range(G):
        lo, hi = (int(x) for x in plan.win[r])
        t_pack = timed(lambda: e.pack_layers(mu, run.gather, lo, hi))
        k0, k1 = int(plan.L[r]), int(plan.L[r + 1])
        _, mrecv = plan.mu_exchange(r)
        mu_bytes = sum(l1 - l0 for _, l0, l1 in mrecv) * layer * 4
        for s, (sub, slots) in enumerate(zip(run.subsets, run.subset_slots)):
            sub = np.asarray(sub)
            corr = torch.zeros((len(sub), H, Wd), device="cuda")
            e.pack(mu, run.gather)
            e.correction(mu, run.p_meas, slots, len(sub), corr, run.gather)
            e.pack_layers(mu, run.gather, lo, hi)
            bd, rows = bands_of(plan, sub, r)
            t_fp = timed(lambda: e.correction_bands(mu, run.p_meas, slots, len(sub), corr, bd,
                                                    rows, gather=run.gather)) if rows else 0.0
            m2 = mu.clone()
            upd = make_update(m2, None, run.cfg)
            t_bp = timed(lambda: (e.pack_quads(corr, len(sub), quads),
                                  e.bp_update_range(corr, slots, len(sub), upd, k0 * layer,
                                                    (k1 - k0) * layer, quads)))
            per_rank[r] += t_fp + t_bp + t_pack
            parts["fp"][r] += t_fp
            parts["bp"][r] += t_bp
            parts["pack"][r] += t_pack
            if G > 1:
                _, crecv = plan.corr_exchange(sub, r)
                recv_bytes[r] += sum(r1 - r0 for _, _, r0, r1 in crecv) * Wd * 4 + mu_bytes
        e.pack(mu, run.gather)
        for views in (rest, np.asarray(run.subsets[0])):
            bd, rows = bands_of(plan, views, r)
            sl = D.upload_i32(views)
            if rows:
                t = timed(lambda: e.residual_bands(mu, run.p_meas, sl, len(views), bd, rows,
                                                   n_proj, scratch, gather=run.gather))
                per_rank[r] += t
                parts["fp"][r] += t
        per_rank[r] += t_pack
    # the flattened-row driver receives, per subset, (G-1)/G of the
    # corrections and of mu (all-gathers)
    ag = sum((G - 1) / G * (len(s) * H * Wd + n_layers * layer) * 4 for s in run.subsets)
    out["per_G"][G] = {"max_rank_ms": float(per_rank.max()), "min_rank_ms": float(per_rank.min()),
                       "fp_ms_max": float(parts["fp"].max()), "bp_ms_max": float(parts["bp"].max()),
                       "pack_ms_max": float(parts["pack"].max()),
                       "recv_MB_per_iteration_max": float(recv_bytes.max() / 1e6),
                       "allgather_recv_MB_per_iteration": float(ag / 1e6) if G > 1 else 0.0,
                       **plan.stats()}
base = out["per_G"][1]["max_rank_ms"]
for G, d in out["per_G"].items():
    d["compute_efficiency"] = base / (G * d["max_rank_ms"])
print(json.dumps(out))
