"""Time the pose step (fit_pose) at the BASELINE Table-1 detector size.

    python tools/bench_pose.py [--reps 5] [--cpu-views 2]

Workload: 21 views of 1536 x 1944 px (table1_geometry), the reference
DeviceSpec assembly at a random production pose, simulated by our FP and
resident in HBM; pose parameters = the reference DeviceSpec's
(threshold 1.8, 9-level ladder, span 1.0, band 1).  Reports the segmentation
kernels (device time, CUDA events on the launching stream), the whole
fit_pose (wall, includes the D2H of the extent tables and the host LM), and
the oracle's per-view numpy segmentation (the reference's own algorithm) on
`--cpu-views` views scaled to 21 -- the reference has no GPU path.
"segmentation" = the fused 9-level threshold/extent pass + the endpoint
kernel + the D2H of the (level, view) endpoint table.
"""

from __future__ import annotations

import argparse
import json
import math
import sys
import time
import warnings
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2005_11976_b200 as P  # noqa: E402
from paper_2005_11976_b200 import cli  # noqa: E402
from paper_2005_11976_b200 import imgproc as IP  # noqa: E402
from paper_2005_11976_b200 import posefit as PF  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cpu-views", type=int, default=2)
    args = ap.parse_args()
    import torch
    geom = P.table1_geometry()
    true = P.Pose(alpha=0.7, beta=math.radians(1.2), gamma=0.3, t=[0.8, -1.1, 0.4])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        vol = P.make_assembly_phantom(cli._device_components(True),
                                      P.CylGrid(240, 16, 60, 8.0, 60.0, true))
    ps = P.forward_project_all(vol, geom, P.RaySamplingConfig())
    host_imgs = np.asarray(ps.images)
    ps = P.ProjectionSet(geom, torch.as_tensor(host_imgs, device="cuda"))   # resident in HBM
    params = P.PoseFitParams(**cli.DEVICE_POSE_PARAMS)

    res = P.fit_pose(ps, params)                                    # warm-up
    stack = IP.ViewStack(ps.images)
    times_seg, times_fit = [], []
    for _ in range(args.reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        lv = np.tile(np.array(params.levels(), dtype=np.float64), (stack.n, 1))
        stack.axis_table(*stack._extents_dev(levels=lv), params.band)
        b.record()
        torch.cuda.synchronize()
        times_seg.append(a.elapsed_time(b))
        t0 = time.perf_counter()
        res = P.fit_pose(ps, params)
        torch.cuda.synchronize()
        times_fit.append((time.perf_counter() - t0) * 1e3)
    # host LM alone on the fitted observations
    t0 = time.perf_counter()
    PF.track_point([(x.view, x.top) for x in res.axes], geom, params.lm)
    PF.track_point([(x.view, x.bottom) for x in res.axes], geom, params.lm)
    lm_ms = (time.perf_counter() - t0) * 1e3

    sys.path.insert(0, str(ROOT / "oracle"))
    import pose_oracle as O
    imgs = host_imgs[:args.cpu_views].astype(np.float64)
    t0 = time.perf_counter()
    O.fit_axes(imgs, levels=params.levels(), band=params.band)
    cpu_ms = (time.perf_counter() - t0) * 1e3 / args.cpu_views * geom.n_proj

    mb = ps.images.numel() * 4 / 1e6
    seg = float(np.median(times_seg))
    out = {
        "workload": "fit_pose, table1 21 x 1536 x 1944, DeviceSpec ladder (9 levels)",
        "segmentation_ms": round(seg, 4),
        "segmentation_gbs": round(mb / seg, 1),
        "fit_pose_ms": round(float(np.median(times_fit)), 3),
        "lm_host_ms": round(lm_ms, 3),
        "cpu_oracle_segmentation_ms": round(cpu_ms, 1),
        "pose_error": {"beta_deg": math.degrees(abs(res.pose.beta - true.beta)),
                       "t_mm": float(np.abs(res.pose.t - true.t).max())},
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
