"""Pin the CPU oracle (oracle/) against golden vectors of the unmodified reference.

The golden files were produced by tests/golden/make_golden.py running the
reference's numba kernels; the oracle is a C/numpy restatement and must agree
to rounding (sample counts exactly).  CPU only.
"""

import math
from types import SimpleNamespace as NS

import numpy as np
import pytest


def desk():
    from paper_2005_11976_b200 import ScanGeometry, make_circular_trajectory
    return ScanGeometry(791.0, 679.0, 65, 33, 0.748, (32.0, 16.0),
                        make_circular_trajectory(8, np.radians(200.0)))


def cyl(nh, nt, nr, R, H, pose=None):
    from paper_2005_11976_b200 import CylGrid, Pose
    return CylGrid(nh, nt, nr, R, H, pose or Pose())


def close(a, b, rtol=1e-12):
    a, b = np.asarray(a, float), np.asarray(b, float)
    scale = max(np.abs(b).max(), 1e-300)
    return np.abs(a - b).max() <= rtol * scale


def test_uniform_cylinder(oracle, golden_small):
    geom = desk()
    g = cyl(8, 24, 16, 8.0, 40.0)
    mu = np.full(g.shape, 0.05)
    for tag, step in (("s020", 0.2), ("s005", 0.05)):
        for i in range(geom.n_proj):
            p, w = oracle.forward(mu, g, geom, i, step=step)
            assert np.array_equal(w, golden_small[f"cyl_uniform_{tag}_w"][i])
            assert close(p, golden_small[f"cyl_uniform_{tag}_p"][i])


def test_random_posed(oracle, golden_small):
    from paper_2005_11976_b200 import Pose
    geom = desk()
    g = cyl(6, 16, 10, 6.0, 20.0, Pose(0.3, 0.2, -0.4, t=[0.5, -0.3, 1.0]))
    mu = golden_small["rand_mu"]
    for i in range(geom.n_proj):
        p, w = oracle.forward(mu, g, geom, i)
        assert np.array_equal(w, golden_small["rand_w"][i])
        assert close(p, golden_small["rand_p"][i])
        p, w = oracle.forward(mu, g, geom, i, nearest=True)
        assert np.array_equal(w, golden_small["rand_nearest_w"][i])
        assert close(p, golden_small["rand_nearest_p"][i])
    p, w = oracle.forward(mu, g, geom, 1, supersample=2)
    assert np.array_equal(w, golden_small["rand_ss2_v1_w"])
    assert close(p, golden_small["rand_ss2_v1_p"])


def test_pixel_list_matches_full_view(oracle, golden_small):
    from paper_2005_11976_b200 import Pose
    geom = desk()
    g = cyl(6, 16, 10, 6.0, 20.0, Pose(0.3, 0.2, -0.4, t=[0.5, -0.3, 1.0]))
    rows, cols = np.divmod(np.arange(geom.det_rows * geom.det_cols)[::7], geom.det_cols)
    p, w = oracle.forward_pixels(golden_small["rand_mu"], g, geom, 4, rows, cols)
    assert np.array_equal(p, golden_small["rand_p"][4][rows, cols])
    assert np.array_equal(w, golden_small["rand_w"][4][rows, cols])


def test_backprojection(oracle, golden_small):
    from paper_2005_11976_b200 import CartGrid, Pose, ScanGeometry
    geom = desk()
    g = cyl(6, 16, 10, 6.0, 20.0, Pose(0.3, 0.2, -0.4, t=[0.5, -0.3, 1.0]))
    for i in (0, 3):
        num, den = oracle.back(golden_small["bp_corr"], geom, i, g)
        assert close(num, golden_small[f"bp_cyl_v{i}_num"])
        assert close(den, golden_small[f"bp_cyl_v{i}_den"])
    cg = CartGrid.centered(10, 9, 8, 0.7, center=(0.2, -0.1, 0.3))
    for i in (0, 5):
        num, den = oracle.back(golden_small["bp_corr"], geom, i, cg)
        assert close(num, golden_small[f"bp_cart_v{i}_num"])
        assert close(den, golden_small[f"bp_cart_v{i}_den"])
    geom9 = ScanGeometry(791.0, 679.0, 9, 9, 0.748, (4.0, 4.0), [0.0])
    num, den = oracle.back(np.ones((9, 9)), geom9, 0, cyl(5, 4, 4, 2.0, 200.0))
    assert close(num, golden_small["bp_tall_num"])
    assert close(den, golden_small["bp_tall_den"])


def test_cartesian_fp(oracle, golden_small):
    from paper_2005_11976_b200 import CartGrid
    geom = desk()
    cg = CartGrid.centered(10, 9, 8, 0.7, center=(0.2, -0.1, 0.3))
    for i in range(geom.n_proj):
        p, w = oracle.forward(golden_small["cart_mu"], cg, geom, i)
        assert np.array_equal(w, golden_small["cart_w"][i])
        assert close(p, golden_small["cart_p"][i])


def test_point_sampling(oracle, golden_small):
    g = cyl(6, 12, 8, 4.0, 3.0)
    pts = golden_small["samp_pts"]
    lin = oracle.sample_cyl(golden_small["samp_mu"], g, pts[:, 0], pts[:, 1], pts[:, 2])
    assert close(lin, golden_small["samp_lin"])
    near = oracle.sample_cyl(golden_small["samp_mu"], g, pts[:, 0], pts[:, 1], pts[:, 2],
                             nearest=True)
    assert np.array_equal(near, golden_small["samp_near"])


def _sart_geom_grid():
    return desk(), cyl(6, 12, 8, 6.0, 20.0)


@pytest.mark.parametrize("name", ["plain", "weighted", "free", "perm"])
def test_sart_runs(oracle, golden_sart, name):
    geom, grid = _sart_geom_grid()
    kw = dict(n_iterations=2)
    if name == "plain":
        kw["relaxation"] = 0.7
    if name == "weighted":
        kw["weights"] = golden_sart["sart_weights"]
        kw["initial"] = golden_sart["sart_init"]
    if name == "free":
        kw["nonneg"] = False
    if name == "perm":
        kw["order"] = np.random.default_rng(3).permutation(geom.n_proj)
    mu, res = oracle.sart(golden_sart["sart_noisy"], grid, geom, **kw)
    assert close(mu, golden_sart[f"sart_{name}_mu"], 1e-10)
    assert close(res, golden_sart[f"sart_{name}_res"], 1e-10)


def test_os_sart_with_p_subsets_is_sart(oracle, golden_sart):
    """A19: S = P subsets reduces to the reference's per-view SART."""
    geom, grid = _sart_geom_grid()
    mu, res = oracle.sart(golden_sart["sart_noisy"], grid, geom, n_iterations=2,
                          relaxation=0.7, n_subsets=geom.n_proj)
    assert close(mu, golden_sart["sart_plain_mu"], 1e-10)


def test_least_squares_system(oracle, golden_sart):
    from paper_2005_11976_b200 import CartGrid, ScanGeometry, make_circular_trajectory
    cg = CartGrid.centered(3, 3, 1, 1.0)
    tg = ScanGeometry(15.0, 10.0, 9, 3, 0.7, (4.0, 1.0),
                      make_circular_trajectory(8, np.radians(200.0)))
    mu, _ = oracle.sart(golden_sart["ls_images"], cg, tg, relaxation=1.0, n_iterations=40,
                        step=0.01, residuals=False)
    assert close(mu.ravel(), golden_sart["ls_sart_mu"].ravel(), 1e-9)
    assert np.abs(mu.ravel() - golden_sart["ls_mu_star"]).max() < 1e-3


def test_c1_views(oracle, golden_c1):
    from paper_2005_11976_b200 import workloads as W
    wl = W.c1_small()
    for i in (0, 45):
        p, w = oracle.forward(wl.mu, wl.grid, wl.geom, i)
        assert np.array_equal(w, golden_c1[f"c1_fp_v{i}_w"])
        assert close(p, golden_c1[f"c1_fp_v{i}_p"])
    num, den = oracle.back(golden_c1["c1_bp_corr"], wl.geom, 7, wl.grid)
    assert close(num, golden_c1["c1_bp_v7_num"])
    assert close(den, golden_c1["c1_bp_v7_den"])


def test_c2_sampled_pixels(oracle, golden_c2):
    from paper_2005_11976_b200 import workloads as W
    wl = W.c2_medium()
    for i in (0, 137):
        idx = golden_c2[f"c2_fp_v{i}_idx"]
        rows, cols = np.divmod(idx, wl.geom.det_cols)
        p, w = oracle.forward_pixels(wl.mu, wl.grid, wl.geom, i, rows, cols)
        assert np.array_equal(w, golden_c2[f"c2_fp_v{i}_w"])
        assert close(p, golden_c2[f"c2_fp_v{i}_p"])
