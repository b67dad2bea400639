"""Generate golden vectors by running the UNMODIFIED reference (cyltomo, numba).

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src:/root/repo NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Every input is float32-representable (the B200 path stores fp32): volumes,
corrections and projections are rounded to fp32 and handed to the reference
as float64(fp32) -- SURVEY.md D4.  Outputs are stored as float64.  Large
inputs that are pure functions of committed seeded code (the C1/C2 phantoms
from paper_2005_11976_b200.workloads) are NOT stored; their sha256 is, so a
drift in the generator is detected.
"""

from __future__ import annotations

import hashlib
import math
import sys
import time
import warnings
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent

import cyltomo as ref  # noqa: E402  (the reference, from PYTHONPATH)
from cyltomo.geometry import view_basis as ref_view_basis  # noqa: E402
from cyltomo.projector import _aligned_basis as ref_aligned_basis  # noqa: E402

sys.path.insert(0, str(OUT.parents[1]))
from paper_2005_11976_b200 import workloads as W  # noqa: E402


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


def desk_geometry():
    return ref.ScanGeometry(791.0, 679.0, 65, 33, 0.748, (32.0, 16.0),
                            ref.make_circular_trajectory(8, np.radians(200.0)))


def fp_all(vol, geom, cfg=None):
    ps, ws = [], []
    for i in range(geom.n_proj):
        p, w = ref.forward_project(vol, geom, i, cfg, return_weights=True)
        ps.append(p)
        ws.append(w)
    return np.stack(ps), np.stack(ws)


def small_cases():
    g = {}
    geom = desk_geometry()
    rng = np.random.default_rng(20251019)
    # geometry conventions (host fp64, must match bit for bit)
    pose = ref.Pose(0.3, 0.2, -0.4, t=[0.5, -0.3, 1.0])
    grid_p = ref.CylGrid(6, 16, 10, 6.0, 20.0, pose)
    g["geo_rotation"] = grid_p.rotation
    g["geo_view_basis"] = np.stack([np.concatenate(ref_view_basis(geom, i))
                                    for i in range(geom.n_proj)])
    g["geo_aligned_basis"] = np.stack([np.concatenate(ref_aligned_basis(grid_p, geom, i))
                                       for i in range(geom.n_proj)])

    # (a) uniform cylinder, two steps
    cyl = ref.CylVolume.full(ref.CylGrid(8, 24, 16, radius=8.0, height=40.0), 0.05)
    for tag, step in (("s020", 0.2), ("s005", 0.05)):
        p, w = fp_all(cyl, geom, ref.RaySamplingConfig(step=step))
        g[f"cyl_uniform_{tag}_p"], g[f"cyl_uniform_{tag}_w"] = p, w

    # (b) random mu on a posed grid: default step, nearest, supersample 2
    mu_b = f32(rng.random(grid_p.shape))
    g["rand_mu"] = mu_b
    vol_b = ref.CylVolume(grid_p, mu_b)
    g["rand_p"], g["rand_w"] = fp_all(vol_b, geom)
    g["rand_nearest_p"], g["rand_nearest_w"] = fp_all(
        vol_b, geom, ref.RaySamplingConfig(interpolation="nearest"))
    p, w = ref.forward_project(vol_b, geom, 1, ref.RaySamplingConfig(supersample=2),
                               return_weights=True)
    g["rand_ss2_v1_p"], g["rand_ss2_v1_w"] = p, w

    # (c) back-projection of a random correction (posed cyl grid, views 0 and 3)
    corr = f32(rng.normal(size=(geom.det_rows, geom.det_cols)))
    g["bp_corr"] = corr
    for i in (0, 3):
        num, den = ref.back_project(corr, geom, i, grid_p)
        g[f"bp_cyl_v{i}_num"], g[f"bp_cyl_v{i}_den"] = num, den
    # grid poking out of the detector (outside-detector voxels untouched)
    geom9 = ref.ScanGeometry(791.0, 679.0, 9, 9, 0.748, (4.0, 4.0), [0.0])
    num, den = ref.back_project(np.ones((9, 9)), geom9, 0,
                                ref.CylGrid(5, 4, 4, radius=2.0, height=200.0))
    g["bp_tall_num"], g["bp_tall_den"] = num, den

    # (d) Cartesian FP / BP
    cgrid = ref.CartGrid.centered(10, 9, 8, 0.7, center=(0.2, -0.1, 0.3))
    mu_d = f32(rng.random(cgrid.shape))
    g["cart_mu"] = mu_d
    cvol = ref.CartVolume(cgrid, mu_d)
    g["cart_p"], g["cart_w"] = fp_all(cvol, geom)
    for i in (0, 5):
        num, den = ref.back_project(corr, geom, i, cgrid)
        g[f"bp_cart_v{i}_num"], g[f"bp_cart_v{i}_den"] = num, den

    # (e) point sampling semantics
    svol = ref.CylVolume(ref.CylGrid(6, 12, 8, radius=4.0, height=3.0),
                         f32(rng.random((6, 12, 8))))
    g["samp_mu"] = svol.mu
    r = rng.uniform(0, 4.2, 500)
    th = rng.uniform(-1.0, 2 * math.pi + 1.0, 500)
    h = rng.uniform(-1.6, 1.6, 500)
    g["samp_pts"] = np.stack([r, th, h], -1)
    g["samp_lin"] = ref.sample(svol, ref.CylCoord(r, th, h))
    g["samp_near"] = ref.sample(svol, ref.CylCoord(r, th, h), mode="nearest")
    return g


def sart_cases():
    g = {}
    geom = desk_geometry()
    rng = np.random.default_rng(7)
    grid = ref.CylGrid(6, 12, 8, radius=6.0, height=20.0)
    body = ref.ComponentSpec("body", mu=0.03)
    insert = ref.ComponentSpec("insert", mu=0.2, r_range=(0.0, 2.0), h_range=(-4.0, 4.0))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        vol = ref.make_assembly_phantom([body, insert], grid)
    images = f32(ref.forward_project_all(vol, geom).images)
    noisy = f32(images + rng.normal(0, 0.05, images.shape))
    g["sart_images"], g["sart_noisy"] = images, noisy
    ps = ref.ProjectionSet(geom, noisy)
    weights = f32(rng.random(grid.shape))
    weights[weights < 0.3] = 0.0
    g["sart_weights"] = weights
    init = f32(rng.random(grid.shape) * 0.01)
    g["sart_init"] = init
    cases = {
        "plain": ref.SartConfig(n_iterations=2, relaxation=0.7),
        "weighted": ref.SartConfig(n_iterations=2, weights=weights,
                                   initial=ref.CylVolume(grid, init)),
        "free": ref.SartConfig(n_iterations=2, nonnegativity=False),
        "perm": ref.SartConfig(n_iterations=2, projection_order="fixed_permutation",
                               order_seed=3),
    }
    for name, cfg in cases.items():
        out, rep = ref.sart_run(ps, grid, cfg)
        g[f"sart_{name}_mu"] = out.mu
        g[f"sart_{name}_res"] = np.asarray(rep.residuals)
    # posed grid, single view update from zero
    posed = grid.with_pose(ref.Pose(0.2, 0.15, -0.2, t=[0.4, -0.5, 0.3]))
    v = ref.CylVolume.zeros(posed)
    ref.sart_update_view(v, ps, 3, ref.SartConfig(relaxation=0.9))
    g["sart_view3_posed_mu"] = v.mu

    # 3x3x1 Cartesian explicit-matrix least-squares system (tests/test_recon.py:14-32)
    fine = ref.RaySamplingConfig(step=0.01)
    cg = ref.CartGrid.centered(3, 3, 1, 1.0)
    tg = ref.ScanGeometry(15.0, 10.0, 9, 3, 0.7, (4.0, 1.0),
                          ref.make_circular_trajectory(8, np.radians(200.0)))
    mu_true = f32(np.random.default_rng(7).uniform(0.2, 1.0, size=9))
    ps_t = ref.forward_project_all(ref.CartVolume(cg, mu_true.reshape(cg.shape)), tg, fine)
    g["ls_images"] = f32(ps_t.images)
    a_mat = np.zeros((tg.n_proj * tg.det_rows * tg.det_cols, 9))
    for l in range(9):
        e = np.zeros(9)
        e[l] = 1.0
        a_mat[:, l] = np.concatenate([ref.forward_project(ref.CartVolume(cg, e.reshape(cg.shape)),
                                                          tg, i, fine).ravel()
                                      for i in range(tg.n_proj)])
    g["ls_mu_star"] = np.linalg.lstsq(a_mat, g["ls_images"].ravel(), rcond=None)[0]
    out, rep = ref.sart_run(ref.ProjectionSet(tg, g["ls_images"]), cg,
                            ref.SartConfig(relaxation=1.0, n_iterations=40, sampling=fine))
    g["ls_sart_mu"] = out.mu
    return g


def c1_cases():
    """C1 (config 0) at full size: two full FP views, one BP, and the full
    10-iteration SART from the reference's own noisy projections."""
    g = {}
    wl = W.c1_small()
    geom = ref.ScanGeometry(**{k: getattr(wl.geom, k) for k in
                               ("sdd", "sod", "det_cols", "det_rows", "pixel_pitch",
                                "principal_point", "stage_angles")})
    p = wl.grid.pose
    grid = ref.CylGrid(*wl.grid.shape, wl.grid.radius, wl.grid.height,
                       ref.Pose(p.alpha, p.beta, p.gamma, t=p.t))
    mu = f32(wl.mu)
    g["c1_mu_sha256"] = np.frombuffer(sha(wl.mu).encode(), dtype=np.uint8)
    vol = ref.CylVolume(grid, mu)
    for i in (0, 45):
        pp, ww = ref.forward_project(vol, geom, i, return_weights=True)
        g[f"c1_fp_v{i}_p"], g[f"c1_fp_v{i}_w"] = pp, ww
    t = time.time()
    clean = np.stack([ref.forward_project(vol, geom, i) for i in range(geom.n_proj)])
    noisy = W.add_noise(clean.astype(np.float32), wl.noise_frac, wl.seed)
    g["c1_noisy_sha256"] = np.frombuffer(sha(noisy).encode(), dtype=np.uint8)
    corr = f32(np.random.default_rng(11).normal(0, 0.01, (geom.det_rows, geom.det_cols)))
    g["c1_bp_corr"] = corr
    num, den = ref.back_project(corr, geom, 7, grid)
    g["c1_bp_v7_num"], g["c1_bp_v7_den"] = num, den
    ps = ref.ProjectionSet(geom, f32(noisy))
    out, rep = ref.sart_run(ps, grid, ref.SartConfig(relaxation=wl.relaxation,
                                                     n_iterations=wl.n_iterations))
    g["c1_sart_mu"] = out.mu.astype(np.float32)
    g["c1_sart_res"] = np.asarray(rep.residuals)
    g["c1_sart_wall"] = np.asarray([rep.wall_time])
    print(f"c1 SART reference wall {rep.wall_time:.1f}s (total {time.time() - t:.1f}s)")
    return g


def c2_cases():
    """C2 (config 1): sampled pixels of two views (the full view is 2 s/view)."""
    g = {}
    wl = W.c2_medium()
    geom = ref.ScanGeometry(**{k: getattr(wl.geom, k) for k in
                               ("sdd", "sod", "det_cols", "det_rows", "pixel_pitch",
                                "principal_point", "stage_angles")})
    p = wl.grid.pose
    grid = ref.CylGrid(*wl.grid.shape, wl.grid.radius, wl.grid.height,
                       ref.Pose(p.alpha, p.beta, p.gamma, t=p.t))
    g["c2_mu_sha256"] = np.frombuffer(sha(wl.mu).encode(), dtype=np.uint8)
    vol = ref.CylVolume(grid, f32(wl.mu))
    rng = np.random.default_rng(22)
    for i in (0, 137):
        pp, ww = ref.forward_project(vol, geom, i, return_weights=True)
        idx = rng.choice(pp.size, 4096, replace=False)
        g[f"c2_fp_v{i}_idx"] = idx
        g[f"c2_fp_v{i}_p"], g[f"c2_fp_v{i}_w"] = pp.ravel()[idx], ww.ravel()[idx]
    return g


def io_cases():
    """Artifacts written by the reference's own writers (cyltomo/io.py), read
    back by tests/test_io.py: volume (cyl + cart), projections, geometry, pose."""
    import cyltomo.io as rio
    d = OUT / "io_ref"
    d.mkdir(exist_ok=True)
    rng = np.random.default_rng(99)
    pose = ref.Pose(0.3, 0.2, -0.4, t=[0.5, -0.3, 1.0])
    cg = ref.CylGrid(3, 5, 4, 2.0, 3.0, pose)
    rio.write_volume(ref.CylVolume(cg, f32(rng.random(cg.shape))), d / "cylvol")
    xg = ref.CartGrid.centered(4, 3, 2, 0.5, center=(0.1, 0.2, 0.3))
    rio.write_volume(ref.CartVolume(xg, f32(rng.random(xg.shape))), d / "cartvol")
    geom = desk_geometry()
    imgs = f32(rng.random((geom.n_proj, geom.det_rows, geom.det_cols)))
    rio.write_projections(ref.ProjectionSet(geom, imgs), d / "proj")
    rio.write_geometry(geom, d / "geom.json")
    rio.write_pose(pose, d / "pose.json")
    return {"io_cyl_mu": np.fromfile(d / "cylvol.raw", dtype="<f4"),
            "io_proj_sum": np.asarray([imgs.sum()])}


def pose_cases():
    """The pose step (cyltomo/imgproc.py, posefit.py) on the reference's own
    desk-scale test setup (tests/test_posefit.py:176-196): fp32-rounded
    projections of a tilted device phantom, fit_pose under several parameter
    sets, per-image functions, and LM triangulations."""
    import warnings as _w
    from cyltomo import imgproc as rip
    from cyltomo import posefit as rpf
    geom = ref.ScanGeometry(791.0, 679.0, 128, 256, 0.52, (63.5, 127.5),
                            ref.make_circular_trajectory(21, math.radians(200.0)))

    def phantom(pose, insert):
        grid = ref.CylGrid(60, 96 if insert else 48, 32, radius=8.0, height=60.0, pose=pose)
        comps = [ref.ComponentSpec("body", mu=0.04),
                 ref.ComponentSpec("core", mu=1.0, r_range=(0.0, 1.5), h_range=(-28.0, 28.0))]
        if insert:
            comps.append(ref.ComponentSpec("insert", mu=0.8, r_range=(4.0, 6.0),
                                           theta_range=(-0.35, 0.35), h_range=(-12.0, 12.0)))
        with _w.catch_warnings():
            _w.simplefilter("ignore")
            return ref.make_assembly_phantom(comps, grid)

    def images(pose, insert):
        ps = ref.forward_project_all(phantom(pose, insert), geom,
                                     ref.RaySamplingConfig(supersample=2))
        return f32(ps.images)

    g = {"pose_geom": np.array([geom.sdd, geom.sod, geom.det_cols, geom.det_rows,
                                geom.pixel_pitch, *geom.principal_point])}
    img_a = images(ref.Pose(alpha=0.6, beta=math.radians(5.0), t=[2.0, -3.0, 1.0]), False)
    img_b = images(ref.Pose(alpha=0.9, beta=math.radians(4.0), gamma=0.7, t=[1.0, 0.5, -2.0]),
                   True)
    g["pose_img_a"] = img_a.astype(np.float32)
    g["pose_img_b"] = img_b.astype(np.float32)
    cases = {
        "core": dict(threshold_level=1.8, threshold_levels=9, threshold_span=1.0, band=1),
        "auto": dict(threshold_level="auto", dilation_radius=1, band=2),
        "nuis": dict(threshold_level=0.3, threshold_levels=3, threshold_span=0.1,
                     nuisance_level=2.5, nuisance_dilation=2,
                     exclude_rects=((180, 256, 0, 64), (0, 5, 0, 128))),
        "dil": dict(threshold_level=1.0, threshold_levels=4, threshold_span=0.5,
                    dilation_radius=2, band=3),
    }
    for name, kw in cases.items():
        res = rpf.fit_pose(ref.ProjectionSet(geom, img_a), rpf.PoseFitParams(**kw))
        g[f"pose_{name}_axes"] = np.array([[a.top.u, a.top.v, a.bottom.u, a.bottom.v]
                                           for a in res.axes])
        g[f"pose_{name}_pose"] = np.array([res.pose.alpha, res.pose.beta, res.pose.gamma,
                                           *res.pose.t])
        g[f"pose_{name}_pts"] = np.concatenate([res.top.solution, res.bottom.solution])
        g[f"pose_{name}_rms"] = np.array([res.top.residual_rms, res.bottom.residual_rms,
                                          float(res.top.converged and res.bottom.converged)])
    # gamma from the strip signal on the object with an off-axis insert
    # (the reference finds a fundamental at offset 10 px and raises FlatSignal
    # at 14 px on this object -- tests/test_pose.py checks both outcomes)
    gkw = dict(threshold_level=1.8, threshold_levels=9, threshold_span=1.0, band=1,
               estimate_gamma=True, strip_offset=10.0, strip_width=8.0)
    res = rpf.fit_pose(ref.ProjectionSet(geom, img_b), rpf.PoseFitParams(**gkw))
    g["pose_gamma_pose"] = np.array([res.pose.alpha, res.pose.beta, res.pose.gamma,
                                     *res.pose.t])
    g["pose_gamma_signal"] = np.array([rip.strip_profile(img_b[i], res.axes[i], 10.0, 8.0)
                                       for i in range(geom.n_proj)])
    try:
        rpf.fit_pose(ref.ProjectionSet(geom, img_b),
                     rpf.PoseFitParams(**dict(gkw, strip_offset=14.0)))
        g["pose_gamma_flat14"] = np.array([0.0])
    except ref.errors.FlatSignal:
        g["pose_gamma_flat14"] = np.array([1.0])
    g["pose_gamma_axes"] = np.array([[a.top.u, a.top.v, a.bottom.u, a.bottom.v]
                                     for a in res.axes])
    # per-image functions
    g["pose_otsu"] = np.array([rip.otsu_level(img_a[i]) for i in range(geom.n_proj)]
                              + [rip.otsu_level(img_b[i]) for i in range(geom.n_proj)])
    strips = []
    for off, wd in ((-6.0, 1.0), (0.0, 3.0), (14.0, 8.0), (-40.5, 2.4), (70.0, 1.0)):
        for i in (0, 5, 13):
            ax = rip.AxisObservation(ref.DetectorPoint(60.25, 70.5), ref.DetectorPoint(66.0, 190.0))
            try:
                strips.append(rip.strip_profile(img_b[i], ax, off, wd))
            except Exception:  # off-frame strip
                strips.append(np.nan)
    g["pose_strips"] = np.array(strips)
    ends = []
    for seed in range(12):
        m = np.random.default_rng(seed).random((40, 30)) > 0.7
        m[:seed % 4] = False
        ob = rip.axis_endpoints(m, band=1 + seed % 3)
        ends.append([ob.top.u, ob.top.v, ob.bottom.u, ob.bottom.v])
    g["pose_ends"] = np.array(ends)
    # LM triangulation on noisy observations (tests/test_posefit.py:45-54 setup)
    desk = ref.ScanGeometry(791.0, 679.0, 256, 128, 0.748, (127.5, 63.5),
                            ref.make_circular_trajectory(21, math.radians(200.0)))
    rng = np.random.default_rng(31)
    obs_all, sol_all = [], []
    for _ in range(6):
        x = rng.uniform(-15, 15, size=3)
        obs = [(i, ref.project_point(desk, i, x)) for i in range(0, 21, 2)]
        noisy = [(i, ref.DetectorPoint(p.u + rng.normal(0, 0.3), p.v + rng.normal(0, 0.3)))
                 for i, p in obs]
        tp = rpf.track_point(noisy, desk)
        obs_all.append([[i, p.u, p.v] for i, p in noisy])
        sol_all.append([*tp.solution, tp.residual_rms])
    g["pose_lm_obs"] = np.array(obs_all)
    g["pose_lm_sol"] = np.array(sol_all)
    return g


def main():
    t = time.time()
    groups = {"golden_small.npz": small_cases, "golden_sart.npz": sart_cases,
              "golden_c1.npz": c1_cases, "golden_c2.npz": c2_cases,
              "golden_io.npz": io_cases, "golden_pose.npz": pose_cases}
    only = set(sys.argv[1:])
    for fname, fn in groups.items():
        if only and fname not in only:
            continue
        g = fn()
        np.savez_compressed(OUT / fname, **g)
        print(f"{fname}: {len(g)} arrays, {(OUT / fname).stat().st_size / 1e6:.2f} MB "
              f"({time.time() - t:.1f}s)")


if __name__ == "__main__":
    main()
