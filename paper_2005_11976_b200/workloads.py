"""Seeded synthetic workloads with BASELINE.json's configuration shapes.

There is no public dataset for this path (the paper's scans are proprietary,
reference SPEC.md:12), so every config is synthetic: phantoms are
rasterised at voxel centres in object coordinates, poses and inclusion
positions come from ``numpy.random.default_rng(seed)`` with the per-config
seeds of SURVEY.md §8d (C1=1, C2=2, C3=3, C4=4, C5=5000+object).  Builder
interpretations of under-specified items (grid radius/height for C2-C5, C4
pitch, phantom layouts) are recorded in DESIGN.md "Workloads".
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .geometry import Pose, ScanGeometry, full_turn_angles
from .grid import CartGrid, CylGrid
from .phantom import ComponentSpec, make_weight_map

RADIUS = 12.0   # mm, C1 value; C2-C5 do not state one
HEIGHT = 24.0


@dataclass
class Sphere:
    r: float       # centre, object cylindrical coordinates
    theta: float
    h: float
    radius: float
    mu: float


@dataclass
class Phantom:
    """Coaxial shells (outer radius, mu) from the inside out + spheres."""

    shells: list
    spheres: list = field(default_factory=list)


def rasterize_cyl(ph: Phantom, grid: CylGrid) -> np.ndarray:
    """Evaluate a phantom at the voxel centres of a cylindrical grid (fp32)."""
    rc = grid.r_centers()
    prof = np.zeros(grid.n_r)
    inner = 0.0
    for outer, mu in ph.shells:
        prof[(rc >= inner) & (rc < outer)] = mu
        inner = outer
    vol = np.empty(grid.shape, dtype=np.float32)
    vol[...] = prof.astype(np.float32)[None, None, :]
    th = grid.theta_centers()
    hc = grid.h_centers()
    for s in ph.spheres:
        ks = np.nonzero(np.abs(hc - s.h) <= s.radius)[0]
        if ks.size == 0:
            continue
        # (theta, r) plane distance^2 to the centre's axis-projection
        cx, cy = s.r * math.cos(s.theta), s.r * math.sin(s.theta)
        rsel = np.nonzero(np.abs(rc - s.r) <= s.radius)[0]
        if rsel.size == 0:
            continue
        xx = rc[None, rsel] * np.cos(th)[:, None]
        yy = rc[None, rsel] * np.sin(th)[:, None]
        d2 = (xx - cx) ** 2 + (yy - cy) ** 2
        for k in ks:
            m = d2 + (hc[k] - s.h) ** 2 <= s.radius ** 2
            jj, ii = np.nonzero(m)
            vol[k, jj, rsel[ii]] = s.mu
    return vol


def rasterize_cart(ph: Phantom, grid: CartGrid, pose: Pose | None = None) -> np.ndarray:
    """Evaluate a phantom (object frame) at the voxel centres of a world Cartesian grid."""
    pose = pose or Pose()
    rot = pose.rotation()
    xs = grid.origin[0] + (np.arange(grid.n_x) + 0.5) * grid.voxel_size
    ys = grid.origin[1] + (np.arange(grid.n_y) + 0.5) * grid.voxel_size
    zs = grid.origin[2] + (np.arange(grid.n_z) + 0.5) * grid.voxel_size
    out = np.zeros(grid.shape, dtype=np.float32)
    yy, xx = np.meshgrid(ys, xs, indexing="ij")
    for k, z in enumerate(zs):
        w = np.stack([xx - pose.t[0], yy - pose.t[1], np.full_like(xx, z - pose.t[2])], -1)
        o = w @ rot                          # world -> object: R^T (x - t)
        r = np.hypot(o[..., 0], o[..., 1])
        h = o[..., 2]
        sl = np.zeros(xx.shape)
        inner = 0.0
        for outer, mu in ph.shells:
            sl[(r >= inner) & (r < outer)] = mu
            inner = outer
        sl[(np.abs(h) > 0.5 * HEIGHT) | (r > RADIUS)] = 0.0
        for s in ph.spheres:
            c = np.array([s.r * math.cos(s.theta), s.r * math.sin(s.theta), s.h])
            d2 = ((o - c) ** 2).sum(-1)
            sl[d2 <= s.radius ** 2] = s.mu
        out[k] = sl
    return out


def _rand_sphere(rng, r_lo, r_hi, rad, mu, h_margin):
    return Sphere(r=float(rng.uniform(r_lo, r_hi)), theta=float(rng.uniform(0, 2 * math.pi)),
                  h=float(rng.uniform(-0.5 * HEIGHT + h_margin, 0.5 * HEIGHT - h_margin)),
                  radius=rad, mu=mu)


def random_tilt_pose(rng, max_tilt_deg: float, max_offset: float) -> Pose:
    """Tilt U(-max, max) about a random horizontal direction + U(-o, o)^3 offset."""
    psi = float(rng.uniform(0.0, 2 * math.pi))
    tau = math.radians(float(rng.uniform(-max_tilt_deg, max_tilt_deg)))
    t = rng.uniform(-max_offset, max_offset, size=3)
    return Pose.tilt(psi, tau, t)


def medium_phantom(rng) -> Phantom:
    """C2: shells r<4: 0.03, 4-8: 0.01, 8-11: 0.05 + 6 voids of radius U[0.5, 1.5]."""
    voids = [_rand_sphere(rng, 0.0, 10.0, float(rng.uniform(0.5, 1.5)), 0.0, 2.0)
             for _ in range(6)]
    return Phantom(shells=[(4.0, 0.03), (8.0, 0.01), (11.0, 0.05)], spheres=voids)


@dataclass
class Workload:
    name: str
    grid: object
    geom: ScanGeometry
    mu: np.ndarray                 # fp32 ground truth on `grid`
    n_iterations: int
    relaxation: float
    n_subsets: int | None = None
    noise_frac: float = 0.0
    template: np.ndarray | None = None
    weights: np.ndarray | None = None
    seed: int = 0
    extra: dict = field(default_factory=dict)


def geometry(n_views, det, pitch, sod, sdd) -> ScanGeometry:
    return ScanGeometry(sdd=sdd, sod=sod, det_cols=det, det_rows=det, pixel_pitch=pitch,
                        principal_point=((det - 1) / 2.0, (det - 1) / 2.0),
                        stage_angles=full_turn_angles(n_views))


def c1_small(seed: int = 1) -> Workload:
    """Config 0 (C1): CPU-runnable cone-beam cylindrical SART."""
    rng = np.random.default_rng(seed)
    pose = Pose(0.0, math.radians(5.0), 0.0, [1.0, -2.0, 0.0])   # 5 deg about x
    grid = CylGrid(64, 128, 64, RADIUS, HEIGHT, pose)
    spheres = [Sphere(9.0, float(rng.uniform(0, 2 * math.pi)),
                      float(rng.uniform(-0.5 * HEIGHT + 1.0, 0.5 * HEIGHT - 1.0)), 1.0, 0.04)
               for _ in range(3)]
    ph = Phantom(shells=[(8.0, 0.0), (10.0, 0.02)], spheres=spheres)
    return Workload("c1_small", grid, geometry(90, 128, 0.2, 200.0, 400.0),
                    rasterize_cyl(ph, grid), n_iterations=10, relaxation=0.5,
                    noise_frac=0.01, seed=seed)


def c2_medium(seed: int = 2, n_views: int = 360) -> Workload:
    """Config 1 (C2): medium OS-SART, 20 iterations, 8 subsets, lambda 0.3."""
    rng = np.random.default_rng(seed)
    pose = random_tilt_pose(rng, 8.0, 3.0)
    grid = CylGrid(256, 512, 256, RADIUS, HEIGHT, pose)
    ph = medium_phantom(rng)
    return Workload("c2_medium", grid, geometry(n_views, 512, 0.1, 250.0, 500.0),
                    rasterize_cyl(ph, grid), n_iterations=20, relaxation=0.3, n_subsets=8,
                    seed=seed, extra={"phantom": ph})


def c3_sparse(seed: int = 3) -> Workload:
    """Config 2 (C3): 30-view weighted SART from the template, 10 iterations."""
    rng = np.random.default_rng(seed)
    base = medium_phantom(np.random.default_rng(2))
    grid0 = CylGrid(256, 512, 256, RADIUS, HEIGHT)
    template = rasterize_cyl(base, grid0)
    # test object: drop one void (inclusion removed), add one new void
    spheres = list(base.spheres)
    spheres.pop(int(rng.integers(len(spheres))))
    spheres.append(_rand_sphere(rng, 2.0, 10.0, 1.0, 0.0, 2.0))
    obj = Phantom(shells=base.shells, spheres=spheres)
    pose = random_tilt_pose(rng, 10.0, 5.0)
    grid = CylGrid(256, 512, 256, RADIUS, HEIGHT, pose)
    th0 = float(rng.uniform(0, 2 * math.pi))
    roi = ComponentSpec("roi", 0.0, r_range=(6.0, 10.0), theta_range=(th0, th0 + math.pi / 2))
    weights = make_weight_map([(roi, 1.0)], grid, default_weight=0.2).astype(np.float32)
    return Workload("c3_sparse", grid, geometry(30, 512, 0.1, 250.0, 500.0),
                    rasterize_cyl(obj, grid), n_iterations=10, relaxation=0.5,
                    template=template, weights=weights, seed=seed)


def c4_grids(seed: int = 4):
    """Config 3 (C4): cylindrical (512,1024,384) and Cartesian 512^3 covering the
    same cylinder; 720 views on a 768^2 detector (pitch 0.1 mm, C2 distances)."""
    rng = np.random.default_rng(seed)
    ph = medium_phantom(rng)
    cyl = CylGrid(512, 1024, 384, RADIUS, HEIGHT)
    cart = CartGrid.centered(512, 512, 512, 2 * RADIUS / 512)
    geom = geometry(720, 768, 0.1, 250.0, 500.0)
    return cyl, cart, geom, ph


def c5_object(obj: int, n_views: int = 120) -> Workload:
    """Config 4 (C5): one batch object, seeded pose and inclusions, 15 OS-SART
    iterations with 6 subsets, lambda 0.3, from the shared template."""
    rng = np.random.default_rng(5000 + obj)
    base = medium_phantom(np.random.default_rng(2))
    spheres = list(base.spheres)
    if rng.random() < 0.5 and spheres:
        spheres.pop(int(rng.integers(len(spheres))))      # missing inclusion
    else:
        spheres.append(_rand_sphere(rng, 2.0, 10.0, float(rng.uniform(0.5, 1.5)), 0.0, 2.0))
    pose = random_tilt_pose(rng, 10.0, 5.0)
    grid = CylGrid(512, 1024, 384, RADIUS, HEIGHT, pose)
    phantom = Phantom(base.shells, spheres)
    return Workload(f"c5_obj{obj}", grid, geometry(n_views, 1024, 0.08, 300.0, 600.0),
                    rasterize_cyl(phantom, grid), n_iterations=15,
                    relaxation=0.3, n_subsets=6, seed=5000 + obj,
                    extra={"template_phantom": base, "phantom": phantom})


def c5_template() -> np.ndarray:
    base = medium_phantom(np.random.default_rng(2))
    return rasterize_cyl(base, CylGrid(512, 1024, 384, RADIUS, HEIGHT))


def add_noise(images: np.ndarray, frac: float, seed: int) -> np.ndarray:
    """simulate_scan noise (cyltomo/experiments.py:31-39): N(0, frac*max(p))."""
    if frac <= 0.0:
        return images
    rng = np.random.default_rng(seed)
    sigma = frac * float(np.max(images))
    return (images.astype(np.float64) + rng.normal(0.0, sigma, images.shape)).astype(np.float32)
