"""Value parity of the resampling row: grid.sample's
kernel driven over whole target grids -- resample_cyl_to_cyl (template
re-gridding, cyltomo/grid.py:310-319, used by recon._initial_volume's
resample_initial branch, recon.py:137-142) and resample_cyl_to_cart
(grid.py:302-308) -- against the fp64 oracle's restatement of
_kernels.sample_cyl_many (_kernels.py:154-163, pinned to the reference by
tests/test_oracle_golden.py).  The device stores fp32, so the bar is fp32
rounding of the fp64 value."""

import math

import numpy as np
import pytest
import torch

import paper_2005_11976_b200 as P

pytestmark = pytest.mark.gpu


def _template():
    rng = np.random.default_rng(21)
    grid = P.CylGrid(24, 40, 18, 5.0, 9.0, P.Pose.tilt(0.7, 0.08, [0.3, -0.2, 0.1]))
    mu = (rng.random(grid.shape) * 0.05).astype(np.float32)
    return grid, mu


def _centres(g):
    hh, tt, rr = np.meshgrid(g.h_centers(), g.theta_centers(), g.r_centers(), indexing="ij")
    return rr, tt, hh


def _close(got, want):
    got = np.asarray(got, np.float64)
    scale = max(np.abs(want).max(), 1e-30)
    return np.abs(got - want).max() <= 2e-7 * scale


@pytest.mark.parametrize("mode", ["linear", "nearest"])
def test_resample_cyl_to_cyl_vs_oracle(oracle, mode):
    grid, mu = _template()
    # finer in h and theta, coarser in r, larger radius (points past R -> 0)
    target = P.CylGrid(31, 57, 11, 5.6, 9.0, P.Pose.tilt(2.0, 0.2, [1.0, 0.0, 0.0]))
    out = P.resample_cyl_to_cyl(P.CylVolume(grid, mu), target, mode=mode)
    r, th, h = _centres(target)
    want = oracle.sample_cyl(mu, grid, r, th, h, nearest=mode == "nearest").reshape(target.shape)
    assert (want == 0).any() and (want != 0).mean() > 0.5
    assert _close(out.mu, want)


def test_resample_cyl_to_cart_vs_oracle(oracle):
    grid, mu = _template()
    cart = P.CartGrid.centered(20, 22, 18, 0.55, center=(0.2, -0.1, 0.3))
    out = P.resample_cyl_to_cart(P.CylVolume(grid, mu), cart)
    # world -> object frame: R^T (x - T) (grid.py:233-241), then (r, theta, h)
    x = cart.voxel_centers().reshape(-1, 3)
    rot = oracle.rotation(grid.pose)
    a = (x - np.asarray(grid.pose.t)) @ rot
    r = np.hypot(a[:, 0], a[:, 1])
    th = np.mod(np.arctan2(a[:, 1], a[:, 0]), 2 * math.pi)
    want = oracle.sample_cyl(mu, grid, r, th, a[:, 2]).reshape(cart.shape)
    assert (want != 0).mean() > 0.2
    assert _close(out.mu, want)


def test_resample_initial_branch_vs_oracle(oracle):
    """SartConfig(resample_initial=True) with a template on another grid: the
    run starts from the resampled template (recon.py:137-142)."""
    grid, mu = _template()
    target = P.CylGrid(16, 32, 12, 5.0, 9.0, P.Pose.tilt(0.3, 0.1, [0.0, 0.5, 0.0]))
    geom = P.ScanGeometry(400.0, 200.0, 40, 36, 0.3, (19.5, 17.5), P.full_turn_angles(6))
    ps = P.ProjectionSet(geom, torch.zeros((6, 36, 40), device="cuda"))
    from paper_2005_11976_b200.recon import SartRun
    run = SartRun(ps, target, P.SartConfig(initial=P.CylVolume(grid, mu),
                                           resample_initial=True, compute_residuals=False))
    r, th, h = _centres(target)
    want = oracle.sample_cyl(mu, grid, r, th, h).reshape(target.shape)
    assert _close(run.mu.cpu().numpy(), want)
    from paper_2005_11976_b200.errors import ConfigError
    with pytest.raises(ConfigError):
        SartRun(ps, target, P.SartConfig(initial=P.CylVolume(grid, mu)))
