"""Where the e2e time of one sart_run(host arrays) call goes (C2, 1 pass)."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

import paper_2005_11976_b200 as P
from paper_2005_11976_b200 import workloads as W
from paper_2005_11976_b200 import recon as R
from paper_2005_11976_b200 import _device as D

wl = W.c2_medium()
ps_dev = P.forward_project_all(P.CylVolume(wl.grid, torch.as_tensor(wl.mu, device="cuda")), wl.geom)
host = torch.empty(tuple(ps_dev.images.shape), dtype=torch.float32, pin_memory=True)
host.copy_(ps_dev.images)
ps = P.ProjectionSet(wl.geom, host.numpy())
cfg = P.SartConfig(relaxation=0.3, n_iterations=1, n_subsets=8)
P.sart_run(ps, wl.grid, cfg)


def t(label, fn):
    torch.cuda.synchronize()
    a = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    print(f"{label:28s} {1e3 * (time.perf_counter() - a):8.2f} ms")
    return out


for rep in range(2):
    eng = t("SartEngine tables", lambda: R.SartEngine(wl.grid, wl.geom, cfg.sampling))
    t("row_max + thresholds", lambda: eng.prepare_thresholds())
    t("upload p_meas (pinned)", lambda: D.to_device(ps.images))
    run = t("SartRun.__init__ total", lambda: R.SartRun(ps, wl.grid, cfg))
    t("one pass (+residual)", lambda: run.run_pass())
    mu = t("D2H mu", lambda: D.to_host(run.mu))
    t("CylVolume(host mu) check", lambda: P.CylVolume(wl.grid, mu))
    t("sart_run total", lambda: P.sart_run(ps, wl.grid, cfg))

vol = None
for rep in range(4):
    vol = t(f"sart_run (previous result alive) #{rep}", lambda: P.sart_run(ps, wl.grid, cfg))
