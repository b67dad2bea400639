"""Edge cases of the projector kernels against the fp64 oracle: single-cell
axes, 1-pixel / 1-row / 1-column detectors, rays exactly parallel to the caps
(central detector row) or through the axis (central column), a step longer
than the grid (one sample per ray), supersampling, nearest mode, and the
K-lanes-per-ray split at its extremes.  Row sums bit-exact, projections within
the north_star 1e-4 rel-L2, BP sums within 1e-5."""

import math

import numpy as np
import pytest

import paper_2005_11976_b200 as P

pytestmark = pytest.mark.gpu

CYL_SHAPES = [(1, 1, 1), (1, 4, 1), (2, 1, 3), (3, 5, 1), (1, 64, 2), (4, 3, 9)]
CART_SHAPES = [(1, 1, 1), (1, 2, 3), (5, 1, 1), (3, 4, 2)]
DETECTORS = [(1, 1, (0.0, 0.0)), (1, 7, (3.0, 0.0)), (7, 1, (0.0, 3.0)), (2, 2, (0.5, 0.5)),
             (9, 11, (5.0, 4.0))]


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb > 0 else float(np.linalg.norm(a))


def geometry(rows, cols, pp, n_views=3, pitch=2.5):
    return P.ScanGeometry(sdd=400.0, sod=200.0, det_cols=cols, det_rows=rows, pixel_pitch=pitch,
                          principal_point=pp, stage_angles=P.full_turn_angles(n_views))


def cases():
    out = []
    for shape in CYL_SHAPES:
        for det in DETECTORS:
            out.append(("cyl", shape, det))
    for shape in CART_SHAPES:
        for det in DETECTORS[::2]:
            out.append(("cart", shape, det))
    return out


def make_volume(kind, shape, rng, posed=True):
    if kind == "cyl":
        pose = P.Pose.tilt(0.7, 0.2, [0.3, -0.2, 0.4]) if posed else P.Pose()
        grid = P.CylGrid(*shape, radius=5.0, height=8.0, pose=pose)
    else:
        grid = P.CartGrid.centered(*shape, voxel_size=2.0, center=(0.2, -0.1, 0.3))
    mu = (rng.random(grid.shape) * 0.1 + 0.01).astype(np.float32)
    vol = (P.CylVolume if kind == "cyl" else P.CartVolume)(grid, mu)
    return vol


@pytest.mark.parametrize("kind,shape,det", cases())
@pytest.mark.parametrize("mode", ["linear", "ss3", "nearest", "longstep"])
def test_fp_edges_vs_oracle(oracle, kind, shape, det, mode, rng):
    rows, cols, pp = det
    geom = geometry(rows, cols, pp)
    vol = make_volume(kind, shape, rng)
    step = None
    ss, nearest = 1, False
    if mode == "ss3":
        ss = 3
    elif mode == "nearest":
        nearest = True
    elif mode == "longstep":
        step = 50.0                         # longer than the grid: <= 1 sample per ray
    cfg = P.RaySamplingConfig(step=step, supersample=ss,
                              interpolation="nearest" if nearest else "linear")
    for i in range(geom.n_proj):
        p, w = P.forward_project(vol, geom, i, cfg, return_weights=True)
        po, wo = oracle.forward(vol.mu, vol.grid, geom, i, step=step, supersample=ss,
                                nearest=nearest)
        assert np.array_equal(np.asarray(w, np.float64), wo.astype(np.float32).astype(np.float64)), \
            (kind, shape, det, mode, i)
        assert rel_l2(p, po) <= 1e-4, (kind, shape, det, mode, i, rel_l2(p, po))


@pytest.mark.parametrize("kind,shape,det", cases())
def test_bp_edges_vs_oracle(oracle, kind, shape, det, rng):
    rows, cols, pp = det
    geom = geometry(rows, cols, pp)
    vol = make_volume(kind, shape, rng)
    for i in range(geom.n_proj):
        c = (rng.standard_normal((rows, cols))).astype(np.float32)
        num, den = P.back_project(c, geom, i, vol.grid)
        no, do = oracle.back(c.astype(np.float64), geom, i, vol.grid)
        assert np.abs(np.asarray(den) - do).max() <= 1e-5 * max(1.0, np.abs(do).max())
        assert np.abs(np.asarray(num) - no).max() <= 1e-5 * max(1.0, np.abs(no).max())
        assert np.array_equal(np.asarray(den) > 0, do > 0)        # SART "touched" set


def test_fp_lanes_extremes_agree(rng):
    """The same rays projected with K = 8 lanes (tiny detector) and K = 1 (a
    detector large enough for one thread per ray) give identical row sums and
    projections within fp32 summation-order noise."""
    vol = make_volume("cyl", (6, 16, 8), rng)
    small = geometry(5, 5, (2.0, 2.0), n_views=2, pitch=0.5)
    # a 400 x 400 detector whose central 5 x 5 block has the same pixels
    big = geometry(400, 400, (200.0, 200.0), n_views=2, pitch=0.5)
    for i in range(2):
        p_s, w_s = P.forward_project(vol, small, i, return_weights=True)
        p_b, w_b = P.forward_project(vol, big, i, return_weights=True)
        blk = (slice(198, 203), slice(198, 203))
        assert np.array_equal(np.asarray(w_s), np.asarray(w_b)[blk])
        assert np.abs(np.asarray(p_s) - np.asarray(p_b)[blk]).max() <= \
            2e-6 * max(1e-30, np.abs(np.asarray(p_s)).max())


def test_ray_through_axis_and_cap_parallel(oracle):
    """Odd detector with the principal point on a pixel centre: the central
    column's rays cross the cylinder axis (theta flips by pi at r = 0) and the
    central row's rays are exactly parallel to the caps (d_z == 0)."""
    grid = P.CylGrid(5, 32, 6, radius=5.0, height=8.0)
    rng = np.random.default_rng(3)
    vol = P.CylVolume(grid, (rng.random(grid.shape) * 0.1).astype(np.float32))
    geom = geometry(9, 9, (4.0, 4.0), n_views=4, pitch=1.0)
    for i in range(4):
        p, w = P.forward_project(vol, geom, i, return_weights=True)
        po, wo = oracle.forward(vol.mu, grid, geom, i)
        assert np.array_equal(np.asarray(w, np.float64), wo.astype(np.float32).astype(np.float64))
        assert rel_l2(p[4], po[4]) <= 1e-4 and rel_l2(p[:, 4], po[:, 4]) <= 1e-4
