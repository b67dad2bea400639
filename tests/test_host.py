"""Host-side logic (CPU): geometry conventions bit-exact vs the reference
goldens, validation/errors of the drop-in API, OS-SART subset construction,
workload determinism."""

import hashlib
import math

import numpy as np
import pytest

import paper_2005_11976_b200 as P
from paper_2005_11976_b200 import _device as D
from paper_2005_11976_b200.errors import ConfigError


def desk():
    return P.ScanGeometry(791.0, 679.0, 65, 33, 0.748, (32.0, 16.0),
                          P.make_circular_trajectory(8, np.radians(200.0)))


class TestGeometryBitExact:
    def test_rotation(self, golden_small):
        grid = P.CylGrid(6, 16, 10, 6.0, 20.0, P.Pose(0.3, 0.2, -0.4, t=[0.5, -0.3, 1.0]))
        assert np.array_equal(grid.rotation, golden_small["geo_rotation"])

    def test_view_basis(self, golden_small):
        geom = desk()
        tab = np.stack([np.concatenate(P.view_basis(geom, i)) for i in range(8)])
        assert np.array_equal(tab, golden_small["geo_view_basis"])
        cart = D.ray_view_table(P.CartGrid.centered(3, 3, 3, 1.0), geom, range(8))
        assert np.array_equal(cart, golden_small["geo_view_basis"])

    def test_aligned_basis_table(self, golden_small):
        grid = P.CylGrid(6, 16, 10, 6.0, 20.0, P.Pose(0.3, 0.2, -0.4, t=[0.5, -0.3, 1.0]))
        tab = D.ray_view_table(grid, desk(), range(8))
        assert np.array_equal(tab, golden_small["geo_aligned_basis"])

    def test_tables_match_per_view_expressions(self, rng):
        """The all-views tables equal the per-view reference expressions
        (view_basis + the aligned-basis products) bit for bit."""
        for _ in range(20):
            geom = P.ScanGeometry(float(rng.uniform(300, 600)), float(rng.uniform(100, 250)),
                                  64, 48, float(rng.uniform(0.05, 0.3)),
                                  (float(rng.uniform(20, 40)), float(rng.uniform(10, 30))),
                                  P.full_turn_angles(int(rng.integers(5, 400))))
            grid = P.CylGrid(4, 8, 4, 6.0, 10.0, P.Pose(*rng.uniform(-3, 3, size=3),
                                                      t=rng.uniform(-2, 2, size=3)))
            views = range(geom.n_proj)
            a, t = grid.rotation.T, grid.pose.t
            ref = np.stack([np.concatenate([a @ (s - t), a @ (o - t), a @ u, a @ v])
                            for s, o, u, v in (P.view_basis(geom, i) for i in views)])
            assert np.array_equal(D.ray_view_table(grid, geom, views), ref)
            cart = np.stack([np.concatenate(P.view_basis(geom, i)) for i in views])
            assert np.array_equal(D.ray_view_table(P.CartGrid.centered(3, 3, 3, 1.0), geom, views),
                                  cart)
            det = D.det_view_table(geom, views)
            assert np.array_equal(det[:, 5], [np.cos(x) for x in geom.stage_angles])
            assert np.array_equal(det[:, 6], [np.sin(x) for x in geom.stage_angles])

    def test_det_table(self):
        geom = desk()
        tab = D.det_view_table(geom, range(8))
        assert np.array_equal(tab[:, 5], np.cos(geom.stage_angles))
        assert np.array_equal(tab[:, 6], np.sin(geom.stage_angles))
        assert (tab[:, 0] == 32.0).all() and (tab[:, 4] == 679.0).all()


class TestPoseAndGeometry:
    def test_canonical_ranges(self, rng):
        for _ in range(200):
            pose = P.Pose(*rng.uniform(-8, 8, size=3))
            assert -math.pi < pose.alpha <= math.pi
            assert 0.0 <= pose.beta <= math.pi
            assert -math.pi < pose.gamma <= math.pi

    def test_tilt_is_pure_tilt(self):
        pose = P.Pose.tilt(0.7, 0.1)
        axis = pose.rotation() @ np.array([0.0, 0.0, 1.0])
        assert math.isclose(math.acos(axis[2]), 0.1, rel_tol=1e-12)

    def test_geometry_validation(self):
        with pytest.raises(ValueError):
            P.ScanGeometry(100.0, 200.0, 4, 4, 0.1, (1, 1), [0.0])
        with pytest.raises(ValueError):
            P.ScanGeometry(200.0, 100.0, 4, 4, 0.0, (1, 1), [0.0])
        g = P.ScanGeometry.from_dict(desk().to_dict())
        assert np.array_equal(g.stage_angles, desk().stage_angles)

    def test_full_turn(self):
        a = P.full_turn_angles(4)
        assert np.allclose(a, [0, math.pi / 2, math.pi, 3 * math.pi / 2])

    def test_projection_conventions(self):
        geom = desk()
        u, v = P.project_point(geom, 0, [0.0, 0.0, 0.0])
        assert (u, v) == geom.principal_point
        with pytest.raises(P.errors.DegenerateRay):
            P.project_point(geom, 0, [0.0, -geom.sod, 0.0])


class TestVolumesAndConfigs:
    def test_volume_is_fp32_and_validated(self):
        g = P.CylGrid(2, 3, 4, 1.0, 1.0)
        v = P.CylVolume(g, np.ones(g.shape))
        assert v.mu.dtype == np.float32
        with pytest.raises(ValueError):
            P.CylVolume(g, np.ones((2, 3, 5)))
        bad = np.ones(g.shape)
        bad[0, 0, 0] = np.nan
        with pytest.raises(ValueError):
            P.CylVolume(g, bad)
        with pytest.raises(ValueError):
            P.CylGrid(0, 3, 4, 1.0, 1.0)

    def test_projection_set_validation(self):
        geom = desk()
        with pytest.raises(ValueError):
            P.ProjectionSet(geom, np.zeros((2, 3, 4)))
        with pytest.raises(ValueError):
            P.ProjectionSet(geom, np.zeros((8, 33, 65)), kind="sinogram")
        ps = P.ProjectionSet(geom, np.zeros((8, 33, 65)))
        assert ps.images.dtype == np.float32

    def test_sampling_config(self):
        with pytest.raises(ValueError):
            P.RaySamplingConfig(step=0.0)
        with pytest.raises(ValueError):
            P.RaySamplingConfig(supersample=0)
        g = P.CylGrid(10, 8, 20, 4.0, 5.0)
        assert P.RaySamplingConfig().step_for(P.CylVolume.zeros(g)) == 0.5 * min(0.2, 0.5)
        assert P.RaySamplingConfig().step_for(P.CartGrid(2, 2, 2, 0.4)) == 0.2

    def test_sart_config_validation(self):
        for kw in (dict(relaxation=0.0), dict(relaxation=2.5), dict(n_iterations=0),
                   dict(projection_order="random"), dict(n_subsets=0)):
            with pytest.raises(ConfigError):
                P.SartConfig(**kw)


class TestSubsets:
    def test_interleaved_subsets_partition_order(self):
        order = np.random.default_rng(0).permutation(30)
        subs = P.make_subsets(order, 8)
        assert len(subs) == 8
        assert np.array_equal(np.sort(np.concatenate(subs)), np.arange(30))
        for s, sub in enumerate(subs):
            assert np.array_equal(sub, order[s::8])

    def test_none_or_p_subsets_is_per_view(self):
        order = np.arange(5)
        assert [list(s) for s in P.make_subsets(order, None)] == [[i] for i in range(5)]
        assert [list(s) for s in P.make_subsets(order, 99)] == [[i] for i in range(5)]


def test_region_mask_and_weight_map():
    g = P.CylGrid(4, 8, 4, 2.0, 4.0)
    roi = P.ComponentSpec("roi", 0.0, r_range=(0.0, 1.0), theta_range=(5.5, 0.5))
    w = P.make_weight_map([(roi, 1.0)], g, default_weight=0.2)
    th = g.theta_centers()
    sel = (th >= 5.5) | (th <= 0.5)
    assert np.all(w[:, sel][:, :, :2] == 1.0)
    assert np.all(w[:, ~sel] == 0.2)
    with pytest.raises(ValueError):
        P.make_weight_map([(roi, 1.5)], g)


def test_workload_generators_match_golden_inputs(golden_c1, golden_c2):
    from paper_2005_11976_b200 import workloads as W

    def sha(a):
        return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()
    assert sha(W.c1_small().mu) == bytes(golden_c1["c1_mu_sha256"]).decode()
    assert sha(W.c2_medium().mu) == bytes(golden_c2["c2_mu_sha256"]).decode()


def test_workload_shapes():
    from paper_2005_11976_b200 import workloads as W
    wl = W.c1_small()
    assert wl.grid.shape == (64, 128, 64) and wl.geom.n_proj == 90
    assert wl.geom.det_rows == wl.geom.det_cols == 128
    assert abs(math.degrees(wl.grid.pose.beta) - 5.0) < 1e-12
    mu = wl.mu
    r = wl.grid.r_centers()
    assert mu[:, :, r < 8.0].max() == 0.0 and np.isclose(mu.max(), 0.04)
