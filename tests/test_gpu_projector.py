"""GPU parity of the projector kernels (through the C-ABI / drop-in API).

Ports every case of the reference's tests/test_projector.py (and the sampling
cases of tests/test_grid.py) to the B200 API, plus golden-vector parity
against the unmodified reference and full-view parity against the oracle.

Tolerances: the reference computes in float64, the B200 path keeps fp32 data
 with fp64 per-ray setup.  Projections must be within 1e-4
relative L2 of the float64 result (north_star); sample counts / row sums are
bit-exact.  Reference tests that assert float64 round-off (1e-10/1e-12
absolute) are restated with an fp32 round-off bound, written next to each.
"""

import math

import numpy as np
import pytest

import paper_2005_11976_b200 as P
from paper_2005_11976_b200 import (CartGrid, CartVolume, CylGrid, CylVolume, Pose,
                                   RaySamplingConfig, ScanGeometry, back_project,
                                   forward_project, forward_project_all)

pytestmark = pytest.mark.gpu

MU0 = 0.05
PROJ_TOL = 1e-4     # north_star: projections within 1e-4 relative L2 of the fp64 oracle
FP32_RTOL = 2e-6    # fp32 round-off bound standing in for the reference's 1e-10/1e-12


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def f32(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


@pytest.fixture
def cylinder():
    return CylVolume.full(CylGrid(8, 24, 16, radius=8.0, height=40.0), MU0)


class TestForwardProject:
    def test_empty_volume(self, cylinder, desk_geometry):
        empty = CylVolume.zeros(cylinder.grid)
        assert not forward_project(empty, desk_geometry, 0).any()

    def test_central_ray_chord(self, cylinder, desk_geometry):
        step = 0.05
        img = forward_project(cylinder, desk_geometry, 0, RaySamplingConfig(step=step))
        u0, v0 = desk_geometry.principal_point
        assert abs(img[int(v0), int(u0)] - MU0 * 2 * cylinder.grid.radius) <= MU0 * step

    def test_off_center_rays_against_dense_oracle(self, cylinder, desk_geometry):
        step = 0.2
        coarse = forward_project(cylinder, desk_geometry, 0, RaySamplingConfig(step=step))
        fine = forward_project(cylinder, desk_geometry, 0, RaySamplingConfig(step=step / 100))
        hit = fine > 0.1 * fine.max()
        assert np.abs(coarse[hit] - fine[hit]).max() <= MU0 * step

    def test_row_sums_track_chords(self, cylinder, desk_geometry):
        img, wsum = forward_project(cylinder, desk_geometry, 0, RaySamplingConfig(step=0.05),
                                    return_weights=True)
        # uniform cylinder: integral = mu0 * sampled path length (fp32 sums)
        assert np.allclose(img, MU0 * wsum, rtol=FP32_RTOL, atol=0)

    def test_linearity(self, desk_geometry, rng):
        grid = CylGrid(6, 16, 10, radius=6.0, height=20.0)
        v1 = rng.random(grid.shape).astype(np.float32)
        v2 = rng.random(grid.shape).astype(np.float32)
        a, b = 0.7, -0.3
        combo = CylVolume(grid, (a * v1.astype(np.float64) + b * v2).astype(np.float32))
        cfg = RaySamplingConfig(step=0.3)
        p = forward_project(combo, desk_geometry, 2, cfg).astype(np.float64)
        p_lin = (a * forward_project(CylVolume(grid, v1), desk_geometry, 2, cfg)
                 + b * forward_project(CylVolume(grid, v2), desk_geometry, 2, cfg))
        scale = np.abs(forward_project(CylVolume(grid, v1), desk_geometry, 2, cfg)).max()
        assert np.abs(p - p_lin).max() < 4 * FP32_RTOL * scale

    def test_halving_step_bounded_change(self, cylinder, desk_geometry):
        p1 = forward_project(cylinder, desk_geometry, 0, RaySamplingConfig(step=0.2))
        p2 = forward_project(cylinder, desk_geometry, 0, RaySamplingConfig(step=0.1))
        assert np.abs(p1 - p2).max() <= MU0 * 0.2

    def test_posed_volume_shift(self, desk_geometry):
        grid = CylGrid(8, 24, 16, radius=8.0, height=10.0)
        vol0 = CylVolume.full(grid, MU0)
        shifted = CylVolume(grid.with_pose(Pose(t=[0.0, 0.0, 3.0])), vol0.mu)
        p0 = forward_project(vol0, desk_geometry, 0).astype(np.float64)
        p1 = forward_project(shifted, desk_geometry, 0).astype(np.float64)
        c0 = (p0.sum(axis=1) * np.arange(p0.shape[0])).sum() / p0.sum()
        c1 = (p1.sum(axis=1) * np.arange(p1.shape[0])).sum() / p1.sum()
        expected = 3.0 * desk_geometry.magnification / desk_geometry.pixel_pitch
        assert c1 - c0 == pytest.approx(expected, abs=0.2)

    def test_supersampling_smooths_partial_pixels(self, cylinder, desk_geometry):
        p1 = forward_project(cylinder, desk_geometry, 0, RaySamplingConfig(step=0.1))
        p4 = forward_project(cylinder, desk_geometry, 0, RaySamplingConfig(step=0.1, supersample=4))
        interior = p1 > 0.5 * p1.max()
        assert np.abs(p1[interior] - p4[interior]).max() < 0.05 * p1.max()

    def test_cartesian_volume_box_integral(self, desk_geometry):
        grid = CartGrid.centered(16, 16, 16, 0.5)
        vol = CartVolume(grid, np.full(grid.shape, MU0))
        img = forward_project(vol, desk_geometry, 0, RaySamplingConfig(step=0.02))
        u0, v0 = desk_geometry.principal_point
        assert img[int(v0), int(u0)] == pytest.approx(MU0 * 8.0, abs=MU0 * 0.02)

    def test_device_resident_volume(self, cylinder, desk_geometry):
        import torch
        dv = CylVolume(cylinder.grid, torch.as_tensor(cylinder.mu, device="cuda"))
        p = forward_project(dv, desk_geometry, 3)
        assert p.is_cuda
        assert np.array_equal(p.cpu().numpy(), forward_project(cylinder, desk_geometry, 3))


class TestForwardProjectAll:
    def test_single_view_reduces_to_forward_project(self, cylinder):
        geom = ScanGeometry(791.0, 679.0, 33, 17, 1.5, (16.0, 8.0), [0.4])
        ps = forward_project_all(cylinder, geom)
        assert ps.kind == "line_integral"
        assert np.array_equal(ps.images[0], forward_project(cylinder, geom, 0))

    def test_batched_equals_per_view_bitwise(self, desk_geometry, rng):
        grid = CylGrid(6, 16, 10, 6.0, 20.0, Pose(0.3, 0.2, -0.4, t=[0.5, -0.3, 1.0]))
        vol = CylVolume(grid, rng.random(grid.shape))
        ps = forward_project_all(vol, desk_geometry)
        for i in range(desk_geometry.n_proj):
            assert np.array_equal(ps.images[i], forward_project(vol, desk_geometry, i))

    def test_rotational_consistency_full_turn(self):
        spec = P.LinePhantomSpec("azimuthal", n_lines=1, shape=(4, 32, 8), radius=6.0,
                                 height=20.0)
        vol = P.make_azimuthal_line_phantom(spec)
        geom = ScanGeometry(791.0, 679.0, 33, 17, 1.5, (16.0, 8.0), [0.3, 0.3 + 2 * math.pi])
        ps = forward_project_all(vol, geom)
        assert np.allclose(ps.images[0], ps.images[1], rtol=0, atol=1e-5 * ps.images.max())


class TestBackProject:
    def test_zero_correction_accumulates_nothing(self, cylinder, desk_geometry):
        zero = np.zeros((desk_geometry.det_rows, desk_geometry.det_cols))
        num, den = back_project(zero, desk_geometry, 0, cylinder.grid)
        assert not num.any()
        assert den.max() > 0.0

    def test_constant_correction_weighted_mean(self, desk_geometry):
        grid = CylGrid(4, 8, 6, radius=4.0, height=10.0)
        const = np.full((desk_geometry.det_rows, desk_geometry.det_cols), 3.0)
        num, den = back_project(const, desk_geometry, 0, grid)
        inside = den > 0
        assert inside.all()
        assert np.allclose(num[inside] / den[inside], 3.0, rtol=1e-6)

    def test_outside_detector_voxels_untouched(self):
        geom = ScanGeometry(791.0, 679.0, 9, 9, 0.748, (4.0, 4.0), [0.0])
        grid = CylGrid(5, 4, 4, radius=2.0, height=200.0)
        num, den = back_project(np.ones((9, 9)), geom, 0, grid)
        assert den[0].max() == 0.0
        assert den[-1].max() == 0.0
        assert den[grid.n_h // 2].max() > 0.0

    def test_accumulation_across_views(self, desk_geometry):
        grid = CylGrid(4, 8, 6, radius=4.0, height=10.0)
        ones = np.ones((desk_geometry.det_rows, desk_geometry.det_cols))
        num1, den1 = back_project(ones, desk_geometry, 0, grid)
        out = (num1.copy(), den1.copy())
        back_project(ones, desk_geometry, 1, grid, out=out)
        num2, den2 = back_project(ones, desk_geometry, 1, grid)
        assert np.allclose(out[1], den1 + den2, rtol=1e-6)


class TestIntensityConversion:
    def test_round_trip(self, desk_geometry, rng):
        shape = (desk_geometry.n_proj, desk_geometry.det_rows, desk_geometry.det_cols)
        p = rng.uniform(0.0, 4.0, size=shape)
        ps = P.ProjectionSet(desk_geometry, np.exp(-p) * 65535.0, kind="intensity")
        out = P.intensities_to_line_integrals(ps, 65535.0)
        assert np.abs(out.images - p).max() < 1e-5

    def test_nonpositive_rejected(self, desk_geometry):
        shape = (desk_geometry.n_proj, desk_geometry.det_rows, desk_geometry.det_cols)
        bad = np.full(shape, 1000.0)
        bad[0, 0, 0] = 0.0
        with pytest.raises(P.errors.NonPositiveIntensity):
            P.intensities_to_line_integrals(P.ProjectionSet(desk_geometry, bad, "intensity"), 1e3)


# ---------------------------------------------------------------------------
# golden parity (unmodified reference outputs)
# ---------------------------------------------------------------------------
class TestGoldenParity:
    def test_uniform_cylinder(self, golden_small, desk_geometry, cylinder):
        for tag, step in (("s020", 0.2), ("s005", 0.05)):
            ps_w = [forward_project(cylinder, desk_geometry, i, RaySamplingConfig(step=step),
                                    return_weights=True) for i in range(8)]
            p = np.stack([x[0] for x in ps_w])
            w = np.stack([x[1] for x in ps_w])
            assert np.array_equal(w, f32(golden_small[f"cyl_uniform_{tag}_w"]))
            assert rel_l2(p, golden_small[f"cyl_uniform_{tag}_p"]) < PROJ_TOL

    def test_random_posed_all_modes(self, golden_small, desk_geometry):
        grid = CylGrid(6, 16, 10, 6.0, 20.0, Pose(0.3, 0.2, -0.4, t=[0.5, -0.3, 1.0]))
        vol = CylVolume(grid, golden_small["rand_mu"])
        for cfg, key in ((RaySamplingConfig(), "rand"),
                         (RaySamplingConfig(interpolation="nearest"), "rand_nearest")):
            out = [forward_project(vol, desk_geometry, i, cfg, return_weights=True)
                   for i in range(8)]
            p = np.stack([x[0] for x in out])
            w = np.stack([x[1] for x in out])
            assert np.array_equal(w, f32(golden_small[f"{key}_w"]))
            assert rel_l2(p, golden_small[f"{key}_p"]) < PROJ_TOL, key
        p, w = forward_project(vol, desk_geometry, 1, RaySamplingConfig(supersample=2),
                               return_weights=True)
        assert np.array_equal(w, f32(golden_small["rand_ss2_v1_w"]))
        assert rel_l2(p, golden_small["rand_ss2_v1_p"]) < PROJ_TOL

    def test_cartesian(self, golden_small, desk_geometry):
        cg = CartGrid.centered(10, 9, 8, 0.7, center=(0.2, -0.1, 0.3))
        vol = CartVolume(cg, golden_small["cart_mu"])
        out = [forward_project(vol, desk_geometry, i, return_weights=True) for i in range(8)]
        assert np.array_equal(np.stack([x[1] for x in out]), f32(golden_small["cart_w"]))
        assert rel_l2(np.stack([x[0] for x in out]), golden_small["cart_p"]) < PROJ_TOL
        for i in (0, 5):
            num, den = back_project(golden_small["bp_corr"], desk_geometry, i, cg)
            assert rel_l2(num, golden_small[f"bp_cart_v{i}_num"]) < 1e-5
            assert rel_l2(den, golden_small[f"bp_cart_v{i}_den"]) < 1e-5

    def test_backprojection(self, golden_small, desk_geometry):
        grid = CylGrid(6, 16, 10, 6.0, 20.0, Pose(0.3, 0.2, -0.4, t=[0.5, -0.3, 1.0]))
        for i in (0, 3):
            num, den = back_project(golden_small["bp_corr"], desk_geometry, i, grid)
            assert rel_l2(num, golden_small[f"bp_cyl_v{i}_num"]) < 1e-5
            assert rel_l2(den, golden_small[f"bp_cyl_v{i}_den"]) < 1e-5
            assert np.array_equal(den > 0, golden_small[f"bp_cyl_v{i}_den"] > 0)
        geom9 = ScanGeometry(791.0, 679.0, 9, 9, 0.748, (4.0, 4.0), [0.0])
        num, den = back_project(np.ones((9, 9)), geom9, 0, CylGrid(5, 4, 4, 2.0, 200.0))
        assert np.array_equal(den > 0, golden_small["bp_tall_den"] > 0)
        assert rel_l2(den, golden_small["bp_tall_den"]) < 1e-5

    def test_point_sampling(self, golden_small):
        grid = CylGrid(6, 12, 8, radius=4.0, height=3.0)
        vol = CylVolume(grid, golden_small["samp_mu"])
        pts = golden_small["samp_pts"]
        c = P.CylCoord(pts[:, 0], pts[:, 1], pts[:, 2])
        assert np.allclose(P.sample(vol, c), golden_small["samp_lin"], rtol=1e-6, atol=1e-7)
        assert np.array_equal(P.sample(vol, c, mode="nearest"),
                              f32(golden_small["samp_near"]))

    def test_c1_full_views(self, golden_c1):
        from paper_2005_11976_b200 import workloads as W
        wl = W.c1_small()
        vol = CylVolume(wl.grid, wl.mu)
        for i in (0, 45):
            p, w = forward_project(vol, wl.geom, i, return_weights=True)
            assert np.array_equal(w, f32(golden_c1[f"c1_fp_v{i}_w"]))
            assert rel_l2(p, golden_c1[f"c1_fp_v{i}_p"]) < PROJ_TOL
        num, den = back_project(golden_c1["c1_bp_corr"], wl.geom, 7, wl.grid)
        assert rel_l2(num, golden_c1["c1_bp_v7_num"]) < 1e-5
        assert rel_l2(den, golden_c1["c1_bp_v7_den"]) < 1e-5

    def test_c2_sampled_pixels(self, golden_c2):
        import torch
        from paper_2005_11976_b200 import workloads as W
        wl = W.c2_medium()
        vol = CylVolume(wl.grid, torch.as_tensor(wl.mu, device="cuda"))
        for i in (0, 137):
            p, w = forward_project(vol, wl.geom, i, return_weights=True)
            idx = golden_c2[f"c2_fp_v{i}_idx"]
            assert np.array_equal(w.cpu().numpy().ravel()[idx], f32(golden_c2[f"c2_fp_v{i}_w"]))
            assert rel_l2(p.cpu().numpy().ravel()[idx], golden_c2[f"c2_fp_v{i}_p"]) < PROJ_TOL


# ---------------------------------------------------------------------------
# full-config parity against the oracle
# ---------------------------------------------------------------------------
def test_c1_every_view_against_oracle(oracle):
    """All 90 C1 views: rel-L2 <= 1e-4 per view, row sums bit-exact."""
    import torch
    from paper_2005_11976_b200 import workloads as W
    wl = W.c1_small()
    vol = CylVolume(wl.grid, torch.as_tensor(wl.mu, device="cuda"))
    ps = forward_project_all(vol, wl.geom)
    worst = 0.0
    for i in range(wl.geom.n_proj):
        p_o, w_o = oracle.forward(wl.mu, wl.grid, wl.geom, i)
        p, w = forward_project(vol, wl.geom, i, return_weights=True)
        assert np.array_equal(w.cpu().numpy(), f32(w_o)), i
        assert torch.equal(p, ps.images[i])
        worst = max(worst, rel_l2(p.cpu().numpy(), p_o))
    assert worst < PROJ_TOL, worst


def test_sample_exact_at_voxel_centers(rng):
    grid = CylGrid(6, 12, 8, radius=4.0, height=3.0)
    vol = CylVolume(grid, rng.random(grid.shape))
    hh, tt, rr = np.meshgrid(grid.h_centers(), grid.theta_centers(), grid.r_centers(),
                             indexing="ij")
    assert np.array_equal(P.sample(vol, P.CylCoord(rr, tt, hh)), vol.mu.astype(np.float64))
    assert P.sample(vol, P.CylCoord(4.001, 1.0, 0.0)) == 0.0
    r = grid.r_centers()[3]
    h = grid.h_centers()[2]
    assert P.sample(vol, P.CylCoord(r, 0.0, h)) == P.sample(vol, P.CylCoord(r, 2 * math.pi, h))


def test_resample_cyl_to_cyl_ignores_pose(rng):
    grid = CylGrid(6, 12, 8, radius=4.0, height=3.0)
    vol = CylVolume(grid, rng.random(grid.shape))
    target = CylGrid(3, 6, 4, 4.0, 3.0, Pose(0.3, 0.4, 0.5, t=[1, 2, 3]))
    a = P.resample_cyl_to_cyl(vol, target).mu
    b = P.resample_cyl_to_cyl(vol, CylGrid(3, 6, 4, 4.0, 3.0)).mu
    assert np.array_equal(a, b)
