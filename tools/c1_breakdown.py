"""Per-kernel-kind time of one C1 SART pass (eager, CUDA events) and the
graph-replayed pass time."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np
import torch

import paper_2005_11976_b200 as P
from paper_2005_11976_b200 import workloads as W
from paper_2005_11976_b200.recon import SartRun

wl = W.c1_small()
vol = P.CylVolume(wl.grid, torch.as_tensor(wl.mu, device="cuda"))
ps = P.forward_project_all(vol, wl.geom)
cfg = P.SartConfig(relaxation=wl.relaxation, n_iterations=wl.n_iterations)
run = SartRun(P.ProjectionSet(wl.geom, ps.images), wl.grid, cfg)
run.run_pass()
torch.cuda.synchronize()
for rep in range(2):
    t = time.perf_counter()
    run.run_pass()
    torch.cuda.synchronize()
    print("graph pass %.2f ms" % (1e3 * (time.perf_counter() - t)))
run.use_graph = False
run.launch_log = []
run.run_pass()
torch.cuda.synchronize()
kinds = {}
for kind, s, a, b in run.launch_log:
    d = kinds.setdefault(kind, [0, 0.0])
    d[0] += 1
    d[1] += a.elapsed_time(b)
for k, (n, ms) in kinds.items():
    print(f"{k:14s} {n:4d} launches {ms:8.3f} ms  ({1e3 * ms / n:.1f} us each)")

# whole sart_run calls (host arrays): init vs run
host_ps = P.ProjectionSet(wl.geom, ps.images.cpu().numpy())
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = SartRun(host_ps, wl.grid, cfg)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    v, rep_ = r.run()
    t2 = time.perf_counter()
    print("sart_run: init %.1f ms, run %.1f ms (report wall %.1f ms)"
          % (1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * rep_.wall_time))
