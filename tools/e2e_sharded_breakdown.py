"""Where the time of one sart_run_sharded call goes (1-rank NCCL group, C2):
engine setup, row split, first pass, result copy-out."""
import os
import socket
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2005_11976_b200 as P  # noqa: E402
from paper_2005_11976_b200 import distributed as PD  # noqa: E402
from paper_2005_11976_b200 import workloads as W  # noqa: E402

s = socket.socket()
s.bind(("127.0.0.1", 0))
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]))
s.close()
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
wl = W.c2_medium()
vol = P.CylVolume(wl.grid, torch.as_tensor(wl.mu, device="cuda"))
imgs = P.forward_project_all(vol, wl.geom).images
host = torch.empty(tuple(imgs.shape), dtype=torch.float32, pin_memory=True)
host.copy_(imgs)
ps = P.ProjectionSet(wl.geom, host.numpy())
cfg = P.SartConfig(relaxation=0.3, n_iterations=1, n_subsets=8)


def t(label, fn):
    torch.cuda.synchronize()
    a = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    print(f"{label:28s} {1e3 * (time.perf_counter() - a):8.2f} ms", flush=True)
    return r


for rep in range(3):
    print("-- call", rep)
    eng = t("GpuEngine (tables, upload)", lambda: PD.GpuEngine(ps, wl.grid, cfg))
    run = t("ShardedSartRun setup", lambda: PD.ShardedSartRun(ps, wl.grid, cfg, engine=eng))
    t("one pass", lambda: run.run_pass())
    t("finalize", lambda: run.finalize())
    t("D2H mu", lambda: P._device.to_host(run.mu, pinned=True))
    t("whole sart_run_sharded", lambda: PD.sart_run_sharded(ps, wl.grid, cfg))
dist.destroy_process_group()
