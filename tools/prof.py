"""Focused driver for ncu: C2 setup, then a few FP-correction / BP-update launches
of subset 0 (same kernels and sizes as one bench.py subset step)."""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--views", type=int, default=360)
ap.add_argument("--config", default="c2")
args = ap.parse_args()

import torch
import paper_2005_11976_b200 as P
from paper_2005_11976_b200 import workloads as W
from paper_2005_11976_b200.recon import SartRun

wl = (W.c2_medium(n_views=args.views) if args.config == "c2" else
      W.c5_object(0) if args.config == "c5" else W.c1_small())
vol = P.CylVolume(wl.grid, torch.as_tensor(wl.mu, device="cuda"))
ps = P.forward_project_all(vol, wl.geom)
init = (P.CylVolume(wl.grid, torch.as_tensor(W.c5_template(), device="cuda"))
        if args.config == "c5" else None)
del vol
run = SartRun(P.ProjectionSet(wl.geom, ps.images), wl.grid,
              P.SartConfig(relaxation=0.3, n_iterations=1, n_subsets=wl.n_subsets or 8,
                           initial=init))
s, slots = run.subsets[0], run.subset_slots[0]
torch.cuda.synchronize()
# warm (the gather layout, allocator); ncu --profile-from-start off captures
# only what follows cudaProfilerStart
run.eng.pack(run.mu, run.gather)
run.eng.correction(run.mu, run.p_meas, slots, len(s), run.corr, run.gather)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for _ in range(args.reps):
    run.eng.pack(run.mu, run.gather)
    run.eng.correction(run.mu, run.p_meas, slots, len(s), run.corr, run.gather)
    run.eng.pack_quads(run.corr, len(s), run.quads)
    run.eng.bp_update(run.corr, slots, len(s), run.upd, run.quads)
run.eng.pack(run.mu, run.gather)
run.eng.residual(run.mu, run.p_meas, run.all_slots, wl.geom.n_proj, run.resid_cur, run.gather)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("prof driver done")
