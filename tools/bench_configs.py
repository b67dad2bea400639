"""Timings of the other BASELINE.json configurations and of the paper's Table-1
batch reconstruction (the only published numbers for this path:
PAPER.md:313 -- 0.30 s plain, 0.52 s weighted, (240,40,60) grid, 21 views of
a 1944x1536 detector).  Prints one JSON object; bench.py stays the driver's
contract (C2).

    python tools/bench_configs.py [--only paper,c1,c3,c4,c5]
"""
from __future__ import annotations

import argparse
import json
import math
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2005_11976_b200 as P  # noqa: E402
from paper_2005_11976_b200 import workloads as W  # noqa: E402
from paper_2005_11976_b200.recon import SartRun  # noqa: E402


def sync():
    torch.cuda.synchronize()


def timed(fn, reps=1):
    """Median wall time of `reps` synchronised calls (host-side work such as
    pageable copies and allocation makes single calls noisy)."""
    ts, out = [], None
    for _ in range(reps):
        sync()
        t = time.perf_counter()
        out = fn()
        sync()
        ts.append(time.perf_counter() - t)
    return float(np.median(ts)), out


def device_phantom(grid, present=True):
    """The reference's DeviceSpec (experiments.py:180-210): body, dense core, part."""
    comps = [P.ComponentSpec("body", 0.04),
             P.ComponentSpec("core", 1.0, r_range=(0.0, 1.5), h_range=(-28.0, 28.0)),
             P.ComponentSpec("part", 0.3, r_range=(4.0, 6.0), h_range=(-10.0, 10.0),
                             present=present)]
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return P.make_assembly_phantom(comps, grid)


def paper_table1():
    """Table-1 geometry, (240,40,60) grid, 1 SART pass, relaxation 1.0:
    strategy (a) plain and (c) template + weights (experiments.py:282-335)."""
    rng = np.random.default_rng(0)
    geom = P.table1_geometry()
    pose = P.Pose(rng.uniform(-math.pi, math.pi), abs(rng.normal(0, math.radians(1.5))),
                  rng.uniform(-math.pi, math.pi), rng.uniform(-2, 2, 3))
    sim = device_phantom(P.CylGrid(240, 16, 60, 8.0, 60.0, pose))
    ps = P.simulate_scan(P.CylVolume(sim.grid, torch.as_tensor(sim.mu, device="cuda")), geom,
                         noise_sigma=0.02, rng=rng)
    ps_host = P.ProjectionSet(geom, ps.images.cpu().numpy())
    grid = P.CylGrid(240, 40, 60, 8.0, 60.0, pose)
    template = device_phantom(P.CylGrid(240, 40, 60, 8.0, 60.0))
    roi = P.ComponentSpec("roi", 0.0, r_range=(4.0, 6.0), h_range=(-10.0, 10.0))
    weights = P.make_weight_map([(roi, 1.0)], template.grid, default_weight=0.3)
    out = {}
    for name, cfg in (("a_plain", P.SartConfig(relaxation=1.0, n_iterations=1)),
                      ("c_template_weights", P.SartConfig(relaxation=1.0, n_iterations=1,
                                                          initial=template,
                                                          weights=weights))):
        for _ in range(2):
            P.sart_run(ps_host, grid, cfg)                       # warm (capture, allocator)
        walls = []

        def call():
            v, r = P.sart_run(ps_host, grid, cfg)
            walls.append(r.wall_time)
            return v, r
        t_call, (vol, rep) = timed(call, reps=7)
        out[name] = {"sart_run_call_s": t_call, "report_wall_time_s": float(np.median(walls)),
                     "residual": rep.residuals[0]}
    out["published_s"] = {"a_plain": 0.30, "c_template_weights": 0.52}
    out["reference_cpu_s_survey_box"] = {"a_plain": 2.58, "c_template_weights": 2.47}
    out["workload"] = ("Table-1 geometry 1944x1536 det, 21 views/200 deg, grid (240,40,60) "
                       "R 8 H 60, 1 SART pass lambda 1.0 (incl. residual FP), host arrays in/out")
    return out


def c1_views():
    """C1 through the reference's per-view entry point: a Python loop of
    sart_update_view over the 90 views (one SART pass, the reference's
    sart_run inner loop, recon.py:171-175) on a device volume and device
    projections -- the cached per-(grid, geometry) device state makes each
    call two kernel launches."""
    wl = W.c1_small()
    vol = P.CylVolume(wl.grid, torch.as_tensor(wl.mu, device="cuda"))
    ps = P.forward_project_all(vol, wl.geom)
    cfg = P.SartConfig(relaxation=wl.relaxation)
    work = P.CylVolume(wl.grid, torch.zeros(wl.grid.shape, device="cuda"))

    def one_pass():
        for i in range(wl.geom.n_proj):
            P.sart_update_view(work, ps, i, cfg)
    one_pass()                                                   # warm (state cache)
    t, _ = timed(one_pass, reps=5)
    return {"workload": "C1, one SART pass as a loop of 90 sart_update_view calls "
                        "(device volume / projections)", "s_per_pass": t,
            "ms_per_view_call": 1e3 * t / wl.geom.n_proj}


def c1():
    wl = W.c1_small()
    vol = P.CylVolume(wl.grid, torch.as_tensor(wl.mu, device="cuda"))
    clean = P.forward_project_all(vol, wl.geom).images.cpu().numpy()
    noisy = W.add_noise(clean, wl.noise_frac, wl.seed)
    ps = P.ProjectionSet(wl.geom, noisy)
    cfg = P.SartConfig(relaxation=wl.relaxation, n_iterations=wl.n_iterations)
    for _ in range(2):
        P.sart_run(ps, wl.grid, cfg)                             # warm (capture, allocator)
    walls = []

    def call():
        v, r = P.sart_run(ps, wl.grid, cfg)
        walls.append(r.wall_time)
        return v, r
    t_call, (v, rep) = timed(call, reps=5)
    return {"workload": "C1: (64,128,64), 90 views 128^2, 10 SART iterations lambda 0.5",
            "sart_run_call_s": t_call, "report_wall_time_s": float(np.median(walls)),
            "s_per_iteration": float(np.median(walls)) / wl.n_iterations,
            "reference_cpu_s": {"10_iterations_wall": 102.5,
                                "note": "reference sart_run, numba 8 threads, build container"}}


def c3():
    wl = W.c3_sparse()
    vol = P.CylVolume(wl.grid, torch.as_tensor(wl.mu, device="cuda"))
    ps = P.forward_project_all(vol, wl.geom)
    cfg = P.SartConfig(relaxation=wl.relaxation, n_iterations=wl.n_iterations,
                       weights=wl.weights, initial=P.CylVolume(wl.grid, wl.template))
    P.sart_run(ps, wl.grid, P.SartConfig(relaxation=0.5, n_iterations=1))
    t_call, (v, rep) = timed(lambda: P.sart_run(ps, wl.grid, cfg))
    return {"workload": "C3: (256,512,256), 30 views 512^2, weighted, template init, 10 SART "
                        "iterations lambda 0.5", "sart_run_call_s": t_call,
            "report_wall_time_s": rep.wall_time,
            "s_per_iteration": rep.wall_time / wl.n_iterations}


def c4():
    cyl, cart, geom, ph = W.c4_grids()
    out = {"workload": "C4: FP and BP of 720 views, 768^2 det; cyl (512,1024,384), cart 512^3"}
    for name, grid, mu in (("cyl", cyl, W.rasterize_cyl(ph, cyl)),
                           ("cart", cart, W.rasterize_cart(ph, cart))):
        V = P.CylVolume if name == "cyl" else P.CartVolume
        vol = V(grid, torch.as_tensor(mu, device="cuda"))
        run = SartRun(P.ProjectionSet(geom, torch.zeros((geom.n_proj, geom.det_rows,
                                                          geom.det_cols), device="cuda")),
                      grid, P.SartConfig(n_subsets=12, compute_residuals=False))
        run.mu.copy_(vol.mu)
        e = run.eng
        fp_t = bp_t = 0.0
        e.pack(run.mu, run.gather)
        for s, slots in zip(run.subsets, run.subset_slots):        # 12 x 60 views
            t, _ = timed(lambda: e.correction(run.mu, run.p_meas, slots, len(s), run.corr,
                                              run.gather))
            fp_t += t
            num = torch.empty(grid.shape, device="cuda")
            den = torch.empty(grid.shape, device="cuda")
            t, _ = timed(lambda: (e.pack_quads(run.corr, len(s), run.quads),
                                  e.bp_partial(run.corr, slots, len(s), num, den, run.quads)))
            bp_t += t
        out[name] = {"fp_all_views_s": fp_t, "bp_all_views_s": bp_t}
    return out


def c5(n_objects=2):
    times = []
    for k in range(n_objects):
        wl = W.c5_object(k)
        vol = P.CylVolume(wl.grid, torch.as_tensor(wl.mu, device="cuda"))
        ps = P.forward_project_all(vol, wl.geom)
        template = P.CylVolume(wl.grid, torch.as_tensor(W.c5_template(), device="cuda"))
        cfg = P.SartConfig(relaxation=wl.relaxation, n_iterations=2, n_subsets=wl.n_subsets,
                           initial=template)
        run = SartRun(ps, wl.grid, cfg)
        run.run_pass()
        sync()
        t, _ = timed(run.run_pass)
        times.append(t)
        del run, ps, vol
        torch.cuda.empty_cache()
    it = float(np.mean(times))
    return {"workload": "C5 object: (512,1024,384), 120 views 1024^2, OS-SART 6 subsets "
                        "lambda 0.3, template init", "s_per_object_iteration": it,
            "s_per_object_15_iterations": 15 * it,
            "s_64_objects_1_gpu_extrapolated": 64 * 15 * it,
            "s_64_objects_8_gpu_object_sharded_extrapolated": 8 * 15 * it}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="paper,c1,c1_views,c3,c4,c5")
    args = ap.parse_args()
    res = {}
    for name in args.only.split(","):
        t = time.perf_counter()
        res[name] = globals()[{"paper": "paper_table1"}.get(name, name)]()
        res[name]["tool_seconds"] = time.perf_counter() - t
        print(name, json.dumps(res[name]), flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
