"""Per-view cost of the C5 correction FP as a function of the batch's view
count (the L2 locality of a wave of CTAs across the batch's views): times
ct_fp_cyl_correction over the first n views of subset-interleaved orders."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np
import torch
import paper_2005_11976_b200 as P
from paper_2005_11976_b200 import _device as D
from paper_2005_11976_b200 import workloads as W
from paper_2005_11976_b200.recon import SartRun

wl = W.c5_object(0)
vol = P.CylVolume(wl.grid, torch.as_tensor(wl.mu, device="cuda"))
ps = P.forward_project_all(vol, wl.geom)
del vol
run = SartRun(ps, wl.grid, P.SartConfig(relaxation=0.3, n_iterations=1, n_subsets=1,
                                        initial=P.CylVolume(wl.grid, torch.as_tensor(
                                            W.c5_template(), device="cuda")),
                                        compute_residuals=False))
e = run.eng
e.pack(run.mu, run.gather)
order = np.concatenate([np.arange(s, 120, 6) for s in range(6)])   # subsets back to back
for n in (10, 20, 40, 60, 120):
    slots = D.upload_i32(order[:n])
    for rep in range(3):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        e.pack(run.mu, run.gather)                 # same cold-L2 start as in a pass
        a.record()
        e.correction(run.mu, run.p_meas, slots, n, run.corr, run.gather)
        b.record()
        torch.cuda.synchronize()
    print(f"views {n:4d}: {a.elapsed_time(b):8.2f} ms  {a.elapsed_time(b) / n:6.3f} ms/view",
          flush=True)

# the same views through the residual epilogue (EPI_RESID) and the fused one
for n in (20, 100, 120):
    slots = D.upload_i32(order[:n])
    scratch = e.residual_scratch(120)
    for rep in range(3):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        e.pack(run.mu, run.gather)
        a.record()
        e.residual_rows(run.mu, run.p_meas, slots, n, 120, scratch, 0, None, run.gather)
        b.record()
        torch.cuda.synchronize()
    print(f"resid views {n:4d}: {a.elapsed_time(b):8.2f} ms  {a.elapsed_time(b) / n:6.3f} ms/view",
          flush=True)
    for rep in range(3):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        e.pack(run.mu, run.gather)
        a.record()
        e.correction_rows(run.mu, run.p_meas, slots, n, run.corr, 0, None, 120, scratch,
                          run.gather)
        b.record()
        torch.cuda.synchronize()
    print(f"corr+resid views {n:4d}: {a.elapsed_time(b):8.2f} ms  "
          f"{a.elapsed_time(b) / n:6.3f} ms/view", flush=True)
