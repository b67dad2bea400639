"""GPU parity of the fused SART / OS-SART path.

Ports every case of the reference's tests/test_recon.py to the B200 API
(bit-exact invariants stay bit-exact), and checks reconstructions against the
unmodified reference's outputs (golden) and the oracle: within 1e-3 relative
L2 after N iterations (north_star).
"""

import warnings

import numpy as np
import pytest

import paper_2005_11976_b200 as P
from paper_2005_11976_b200 import (CartGrid, CartVolume, ComponentSpec, CylGrid, CylVolume,
                                   Pose, ProjectionSet, RaySamplingConfig, SartConfig,
                                   ScanGeometry, forward_project_all, make_assembly_phantom,
                                   make_circular_trajectory, sart_run, sart_update_view)
from paper_2005_11976_b200.errors import ConfigError, EmptyView

pytestmark = pytest.mark.gpu

RECON_TOL = 1e-3   # north_star: reconstructions within 1e-3 relative L2
FINE = RaySamplingConfig(step=0.01)


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def tiny_system():
    """3x3x1 Cartesian system with its explicit-matrix LS oracle (test_recon.py:14-32)."""
    rng = np.random.default_rng(7)
    grid = CartGrid.centered(3, 3, 1, 1.0)
    geom = ScanGeometry(15.0, 10.0, 9, 3, 0.7, (4.0, 1.0),
                        make_circular_trajectory(8, np.radians(200.0)))
    a_mat = np.zeros((geom.n_proj * geom.det_rows * geom.det_cols, 9))
    for l in range(9):
        e = np.zeros(9)
        e[l] = 1.0
        ps_e = forward_project_all(CartVolume(grid, e.reshape(grid.shape)), geom, FINE)
        a_mat[:, l] = ps_e.images.astype(np.float64).ravel()
    mu_true = rng.uniform(0.2, 1.0, size=9)
    ps = forward_project_all(CartVolume(grid, mu_true.reshape(grid.shape)), geom, FINE)
    mu_star, *_ = np.linalg.lstsq(a_mat, ps.images.astype(np.float64).ravel(), rcond=None)
    return grid, geom, ps, mu_star


@pytest.fixture
def small_cyl_setup(desk_geometry):
    grid = CylGrid(6, 12, 8, radius=6.0, height=20.0)
    body = ComponentSpec("body", mu=0.03)
    insert = ComponentSpec("insert", mu=0.2, r_range=(0.0, 2.0), h_range=(-4.0, 4.0))
    with pytest.warns(UserWarning):
        vol = make_assembly_phantom([body, insert], grid)
    return grid, vol, forward_project_all(vol, desk_geometry)


class TestScalarUpdate:
    def _setup(self):
        grid = CylGrid(1, 1, 1, radius=0.5, height=4.0)
        geom = ScanGeometry(15.0, 10.0, 1, 1, 1.0, (0.0, 0.0), [0.0])
        return grid, geom, ProjectionSet(geom, np.full((1, 1, 1), 2.0))

    @pytest.mark.parametrize("relax,w,expected", [(1.0, None, 2.0), (1.0, 0.5, 1.0),
                                                  (0.25, None, 0.5)])
    def test_scalar_updates(self, relax, w, expected):
        grid, geom, ps = self._setup()
        vol = CylVolume.zeros(grid)
        weights = None if w is None else np.full(grid.shape, w)
        cfg = SartConfig(relaxation=relax, weights=weights, sampling=RaySamplingConfig(step=0.1))
        sart_update_view(vol, ps, 0, cfg)
        assert vol.mu[0, 0, 0] == pytest.approx(expected, rel=1e-6)


class TestFixedPointAndInvariants:
    def test_consistent_data_is_fixed_point(self, small_cyl_setup):
        grid, vol, ps = small_cyl_setup
        work = CylVolume(grid, vol.mu.copy())
        cfg = SartConfig(n_iterations=3)
        for _ in range(3):
            for i in range(ps.geom.n_proj):
                sart_update_view(work, ps, i, cfg)
        assert np.array_equal(work.mu, vol.mu)

    def test_fixed_point_through_sart_run(self, small_cyl_setup):
        grid, vol, ps = small_cyl_setup
        out, _ = sart_run(ps, grid, SartConfig(n_iterations=2, initial=vol))
        assert np.array_equal(out.mu, vol.mu)
        out, _ = sart_run(ps, grid, SartConfig(n_iterations=2, initial=vol, n_subsets=3))
        assert np.array_equal(out.mu, vol.mu)

    def test_weight_zero_voxels_bit_identical(self, small_cyl_setup, rng):
        grid, vol, ps = small_cyl_setup
        weights = rng.random(grid.shape)
        weights[weights < 0.3] = 0.0
        frozen = weights == 0.0
        init = CylVolume(grid, rng.random(grid.shape) * 0.01)
        before = init.mu.copy()
        out, _ = sart_run(ps, grid, SartConfig(n_iterations=2, weights=weights, initial=init))
        assert np.array_equal(out.mu[frozen], before[frozen])
        assert not np.array_equal(out.mu[~frozen], before[~frozen])

    def test_all_ones_weights_equal_unweighted(self, small_cyl_setup):
        grid, vol, ps = small_cyl_setup
        plain, _ = sart_run(ps, grid, SartConfig(n_iterations=2))
        weighted, _ = sart_run(ps, grid, SartConfig(n_iterations=2, weights=np.ones(grid.shape)))
        assert np.array_equal(plain.mu, weighted.mu)

    def test_nonnegativity_flag(self, small_cyl_setup, rng):
        grid, vol, ps = small_cyl_setup
        noisy = ProjectionSet(ps.geom, ps.images + rng.normal(0, 0.1, ps.images.shape))
        clamped, _ = sart_run(noisy, grid, SartConfig(n_iterations=2))
        assert clamped.mu.min() >= 0.0
        free, _ = sart_run(noisy, grid, SartConfig(n_iterations=2, nonnegativity=False))
        assert free.mu.min() < 0.0


class TestOracleConvergence:
    def test_converges_to_least_squares_solution(self, tiny_system):
        grid, geom, ps, mu_star = tiny_system
        vol, report = sart_run(ps, grid, SartConfig(relaxation=1.0, n_iterations=40,
                                                    sampling=FINE))
        assert np.abs(vol.mu.ravel() - mu_star).max() < 1e-3
        assert len(report.residuals) == 40

    def test_monotone_residual_first_passes(self, tiny_system):
        grid, geom, ps, mu_star = tiny_system
        _, report = sart_run(ps, grid, SartConfig(relaxation=0.8, n_iterations=10,
                                                  sampling=FINE))
        res = report.residuals
        for a, b in zip(res, res[1:]):
            assert b <= a * (1 + 1e-5) + 1e-7   # fp32 data: round-off floor ~1e-7

    def test_initial_template_lowers_first_pass_residual(self, small_cyl_setup):
        grid, vol, ps = small_cyl_setup
        _, plain = sart_run(ps, grid, SartConfig(n_iterations=1))
        _, primed = sart_run(ps, grid, SartConfig(n_iterations=1,
                                                  initial=CylVolume(grid, vol.mu.copy())))
        assert primed.residuals[0] < plain.residuals[0]


class TestRunConfiguration:
    def test_initial_shape_mismatch_needs_resampling(self, small_cyl_setup):
        grid, vol, ps = small_cyl_setup
        template = CylVolume.full(CylGrid(3, 6, 4, grid.radius, grid.height), 0.03)
        with pytest.raises(ConfigError):
            sart_run(ps, grid, SartConfig(initial=template))
        out, _ = sart_run(ps, grid, SartConfig(initial=template, resample_initial=True))
        assert out.mu.shape == grid.shape

    def test_requires_line_integrals(self, small_cyl_setup):
        grid, vol, ps = small_cyl_setup
        intens = ProjectionSet(ps.geom, np.exp(-ps.images), kind="intensity")
        with pytest.raises(ConfigError):
            sart_update_view(CylVolume.zeros(grid), intens, 0, SartConfig())

    def test_fixed_permutation_deterministic(self, small_cyl_setup):
        grid, vol, ps = small_cyl_setup
        cfg = dict(n_iterations=1, projection_order="fixed_permutation", order_seed=3)
        a, _ = sart_run(ps, grid, SartConfig(**cfg))
        b, _ = sart_run(ps, grid, SartConfig(**cfg))
        assert np.array_equal(a.mu, b.mu)

    def test_empty_view_raises(self):
        geom = ScanGeometry(15.0, 10.0, 3, 3, 0.1, (1.0, 1.0), [0.0])
        grid = CylGrid(2, 4, 4, radius=0.5, height=1.0, pose=Pose(t=[50.0, 0.0, 0.0]))
        ps = ProjectionSet(geom, np.zeros((1, 3, 3)))
        with pytest.raises(EmptyView):
            sart_update_view(CylVolume.zeros(grid), ps, 0, SartConfig())
        with pytest.raises(EmptyView):
            sart_run(ps, grid, SartConfig())

    def test_weight_shape_validated(self, small_cyl_setup):
        grid, vol, ps = small_cyl_setup
        with pytest.raises(ConfigError):
            sart_run(ps, grid, SartConfig(weights=np.ones((2, 2, 2))))


# ---------------------------------------------------------------------------
# parity against the unmodified reference (golden) and the oracle
# ---------------------------------------------------------------------------
def _desk():
    return ScanGeometry(791.0, 679.0, 65, 33, 0.748, (32.0, 16.0),
                        make_circular_trajectory(8, np.radians(200.0)))


@pytest.mark.parametrize("name", ["plain", "weighted", "free", "perm"])
def test_golden_sart_runs(golden_sart, name):
    geom = _desk()
    grid = CylGrid(6, 12, 8, radius=6.0, height=20.0)
    ps = ProjectionSet(geom, golden_sart["sart_noisy"])
    kw = dict(n_iterations=2)
    if name == "plain":
        kw["relaxation"] = 0.7
    if name == "weighted":
        kw.update(weights=golden_sart["sart_weights"],
                  initial=CylVolume(grid, golden_sart["sart_init"]))
    if name == "free":
        kw["nonnegativity"] = False
    if name == "perm":
        kw.update(projection_order="fixed_permutation", order_seed=3)
    out, rep = sart_run(ps, grid, SartConfig(**kw))
    assert rel_l2(out.mu, golden_sart[f"sart_{name}_mu"]) < RECON_TOL
    assert np.allclose(rep.residuals, golden_sart[f"sart_{name}_res"], rtol=1e-3)


def test_golden_single_view_posed(golden_sart):
    geom = _desk()
    grid = CylGrid(6, 12, 8, 6.0, 20.0, Pose(0.2, 0.15, -0.2, t=[0.4, -0.5, 0.3]))
    v = CylVolume.zeros(grid)
    sart_update_view(v, ProjectionSet(geom, golden_sart["sart_noisy"]), 3,
                     SartConfig(relaxation=0.9))
    assert rel_l2(v.mu, golden_sart["sart_view3_posed_mu"]) < 1e-5


def test_golden_least_squares(golden_sart):
    cg = CartGrid.centered(3, 3, 1, 1.0)
    tg = ScanGeometry(15.0, 10.0, 9, 3, 0.7, (4.0, 1.0),
                      make_circular_trajectory(8, np.radians(200.0)))
    out, _ = sart_run(ProjectionSet(tg, golden_sart["ls_images"]), cg,
                      SartConfig(relaxation=1.0, n_iterations=40, sampling=FINE))
    assert rel_l2(out.mu.ravel(), golden_sart["ls_sart_mu"].ravel()) < RECON_TOL
    assert np.abs(out.mu.ravel() - golden_sart["ls_mu_star"]).max() < 1e-3


def _c1_inputs(oracle):
    import hashlib
    from paper_2005_11976_b200 import workloads as W
    wl = W.c1_small()
    clean = np.stack([oracle.forward(wl.mu, wl.grid, wl.geom, i)[0]
                      for i in range(wl.geom.n_proj)]).astype(np.float32)
    noisy = W.add_noise(clean, wl.noise_frac, wl.seed)
    return wl, noisy, hashlib.sha256(noisy.tobytes()).hexdigest()


def test_c1_full_sart_against_reference(oracle, golden_c1):
    """Config 0 (C1) end to end: 10 SART iterations from zero, lambda 0.5, on the
    reference's own noisy projections; within 1e-3 of the reference's volume."""
    wl, noisy, digest = _c1_inputs(oracle)
    assert digest == bytes(golden_c1["c1_noisy_sha256"]).decode()
    out, rep = sart_run(ProjectionSet(wl.geom, noisy), wl.grid,
                        SartConfig(relaxation=wl.relaxation, n_iterations=wl.n_iterations))
    err = rel_l2(out.mu, golden_c1["c1_sart_mu"])
    assert err < RECON_TOL, err
    assert np.allclose(rep.residuals, golden_c1["c1_sart_res"], rtol=1e-3)


def test_os_sart_against_oracle(oracle):
    """A19 OS-SART (no reference symbol): against the oracle's composition of
    reference primitives on a posed, weighted problem."""
    rng = np.random.default_rng(31)
    geom = ScanGeometry(400.0, 200.0, 48, 40, 0.2, (23.5, 19.5),
                        P.full_turn_angles(24))
    grid = CylGrid(20, 32, 16, 4.0, 8.0, Pose.tilt(0.7, 0.08, [0.3, -0.2, 0.1]))
    truth = (rng.random(grid.shape) * 0.05).astype(np.float32)
    weights = rng.uniform(0.2, 1.0, grid.shape).astype(np.float32)
    images = np.stack([oracle.forward(truth, grid, geom, i)[0]
                       for i in range(geom.n_proj)]).astype(np.float32)
    order = np.random.default_rng(5).permutation(geom.n_proj)
    mu_o, res_o = oracle.sart(images, grid, geom, relaxation=0.3, n_iterations=3,
                              order=order, weights=weights, n_subsets=4)
    out, rep = sart_run(ProjectionSet(geom, images), grid,
                        SartConfig(relaxation=0.3, n_iterations=3, weights=weights,
                                   projection_order="fixed_permutation", order_seed=5,
                                   n_subsets=4))
    assert rel_l2(out.mu, mu_o) < RECON_TOL
    assert np.allclose(rep.residuals, res_o, rtol=1e-3)


def test_os_sart_with_p_subsets_equals_sart(small_cyl_setup):
    grid, vol, ps = small_cyl_setup
    a, _ = sart_run(ps, grid, SartConfig(n_iterations=2, relaxation=0.6))
    b, _ = sart_run(ps, grid, SartConfig(n_iterations=2, relaxation=0.6,
                                         n_subsets=ps.geom.n_proj))
    assert np.array_equal(a.mu, b.mu)


def test_device_resident_run_matches_host(small_cyl_setup):
    import torch
    grid, vol, ps = small_cyl_setup
    host, _ = sart_run(ps, grid, SartConfig(n_iterations=2, n_subsets=2))
    dps = ProjectionSet(ps.geom, torch.as_tensor(ps.images, device="cuda"))
    dev, _ = sart_run(dps, grid, SartConfig(n_iterations=2, n_subsets=2))
    assert dev.mu.is_cuda
    assert np.array_equal(dev.mu.cpu().numpy(), host.mu)


@pytest.mark.parametrize("n_subsets", [2, 3, 21])
def test_pinned_host_run_matches_device(small_cyl_setup, n_subsets):
    """Page-locked host projections take the streamed upload (per-subset copies
    on a side stream) and the final volume is copied out while the residual FP
    runs; 21 single-view subsets take the CUDA-graph path.  Same bits and
    residuals as the device-resident run."""
    import torch
    grid, vol, ps = small_cyl_setup
    cfg = SartConfig(n_iterations=2, n_subsets=n_subsets, relaxation=0.7)
    pinned = torch.empty(ps.images.shape, dtype=torch.float32, pin_memory=True)
    pinned.copy_(torch.from_numpy(np.asarray(ps.images, dtype=np.float32)))
    a, ra = sart_run(ProjectionSet(ps.geom, pinned.numpy()), grid, cfg)
    b, rb = sart_run(ProjectionSet(ps.geom, torch.as_tensor(ps.images, device="cuda")), grid, cfg)
    c, rc = sart_run(ps, grid, cfg)                       # pageable host arrays
    assert isinstance(a.mu, np.ndarray)
    assert np.array_equal(a.mu, b.mu.cpu().numpy())
    assert np.array_equal(a.mu, c.mu)
    assert ra.residuals == rb.residuals == rc.residuals


@pytest.mark.parametrize("n_subsets", [2, 21])
def test_staged_pageable_upload_matches_device(small_cyl_setup, monkeypatch, n_subsets):
    """Pageable host projections staged through page-locked memory by worker
    threads (recon._StagedUpload, forced here for a small stack) give the
    device-resident run's bits, eager (2 subsets) and graph-captured (21)."""
    import torch
    from paper_2005_11976_b200 import recon as R
    grid, vol, ps = small_cyl_setup
    cfg = SartConfig(n_iterations=2, n_subsets=n_subsets, relaxation=0.7)
    used = []
    orig = R._StagedUpload.__init__

    def spy(self, *a, **k):
        used.append(1)
        orig(self, *a, **k)
    monkeypatch.setattr(R._StagedUpload, "applies", staticmethod(lambda images: True))
    monkeypatch.setattr(R._StagedUpload, "__init__", spy)
    a, ra = sart_run(ps, grid, cfg)                       # pageable host arrays
    assert used
    b, rb = sart_run(ProjectionSet(ps.geom, torch.as_tensor(ps.images, device="cuda")), grid, cfg)
    assert np.array_equal(a.mu, b.mu.cpu().numpy())
    assert ra.residuals == rb.residuals


def test_graph_replay_bit_identical(small_cyl_setup):
    """A pass captured as a CUDA graph replays the same kernels: same bits."""
    from paper_2005_11976_b200.recon import SartRun
    grid, vol, ps = small_cyl_setup
    noisy = ProjectionSet(ps.geom, ps.images * 1.01)
    cfg = SartConfig(n_iterations=3, relaxation=0.6)
    va, ra = SartRun(noisy, grid, cfg, use_graph=True).run()
    vb, rb = SartRun(noisy, grid, cfg, use_graph=False).run()
    assert np.array_equal(va.mu, vb.mu)
    assert ra.residuals == rb.residuals


@pytest.mark.parametrize("n_subsets,n_iter", [(2, 1), (3, 3), (5, 4)])
def test_deferred_residual_bit_identical(small_cyl_setup, monkeypatch, n_subsets, n_iter):
    """The residual of pass k split between pass k's FP over the other
    subsets' views and pass k+1's first correction FP (slot-positioned
    partials, one fixed-order sum) gives the same bits as one residual launch
    over all views, and the volumes are unchanged."""
    from paper_2005_11976_b200.recon import SartRun
    grid, vol, ps = small_cyl_setup
    noisy = ProjectionSet(ps.geom, ps.images * 1.02)
    cfg = SartConfig(n_iterations=n_iter, n_subsets=n_subsets, relaxation=0.6)
    fused = SartRun(noisy, grid, cfg)
    assert fused.fuse_residual
    va, ra = fused.run()
    monkeypatch.setenv("CT_RESID_FUSE", "0")
    plain = SartRun(noisy, grid, cfg)
    assert not plain.fuse_residual
    vb, rb = plain.run()
    assert np.array_equal(va.mu, vb.mu)
    assert ra.residuals == rb.residuals
    assert len(ra.residuals) == n_iter and all(r > 0 for r in ra.residuals)


def test_deferred_residual_cartesian_and_mixed_passes(monkeypatch):
    """Cartesian grid; passes with and without the residual interleaved
    (run_pass(residual=...)), finalize() between them."""
    from paper_2005_11976_b200.recon import SartRun
    grid = CartGrid.centered(10, 9, 8, 0.5)
    geom = ScanGeometry(40.0, 30.0, 24, 20, 0.4, (11.5, 9.5), make_circular_trajectory(12, np.radians(330.0)))
    rng = np.random.default_rng(5)
    truth = CartVolume(grid, rng.uniform(0.0, 0.1, grid.shape))
    ps = forward_project_all(truth, geom)
    cfg = SartConfig(n_iterations=4, n_subsets=3, relaxation=0.5, compute_residuals=False)
    out = []
    for fuse in ("1", "0"):
        monkeypatch.setenv("CT_RESID_FUSE", fuse)
        run = SartRun(ps, grid, cfg)
        for want in (True, False, True, True):
            run.run_pass(residual=want)
        run.finalize()
        out.append((run.mu.cpu().numpy(), run.resid.cpu().numpy()))
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])
    assert out[0][1][0] > 0 and out[0][1][1] == 0 and out[0][1][3] > 0


@pytest.mark.parametrize("quad", ["0", "1", "b"])
@pytest.mark.parametrize("kind", ["cyl", "cyl_coarse", "cart"])
def test_gather_layout_matches_plain_path(rng, kind, quad, monkeypatch):
    """The gather layouts (GL_OCT: 32-byte polynomial cells; GL_OCTB: the same
    in 2x2 bricks, forced with CT_GATHER_OBRICK=1; GL_QUAD: 16-byte per-layer
    bilinear cells in 2x2x2 bricks, forced with CT_GATHER_QUAD=1) change the
    loads, not the result: bit-identical to the plain path.  cyl_coarse (2x4x2
    cells) puts many samples into the first cell of the layout (bottom h halo,
    theta row 0, axis r halo), whose index is -1 with the r floor magic."""
    monkeypatch.setenv("CT_GATHER_QUAD", "1" if quad == "1" else "0")
    monkeypatch.setenv("CT_GATHER_OBRICK", "1" if quad == "b" else "0")
    import ctypes as C
    import torch
    from paper_2005_11976_b200 import _device as D, _native as N
    if kind == "cyl":
        grid = CylGrid(12, 20, 10, 5.0, 9.0, Pose.tilt(0.2, 0.1, [0.3, 0.1, 0.2]))
    elif kind == "cyl_coarse":
        grid = CylGrid(2, 4, 2, 2.0, 2.0, Pose.tilt(0.0, 0.02, [0.0, 0.0, 0.0]))
    else:
        grid = CartGrid.centered(11, 9, 13, 0.7, center=(0.2, -0.3, 0.1))
    geom = ScanGeometry(300.0, 150.0, 40, 36, 0.25, (19.5, 17.5), P.full_turn_angles(6))
    mu = torch.as_tensor(rng.random(grid.shape, dtype=np.float32), device="cuda")
    table = D.upload_f64(D.ray_view_table(grid, geom, range(6)))
    g = D.grid_c(grid)
    s = D.sampling_c(RaySamplingConfig().step_for(grid), 1, False)
    b = D.batch_c(6, geom.det_rows, geom.det_cols)
    gather = D.alloc_gather(grid, "cuda")
    gk = "cart" if kind == "cart" else "cyl"
    N.call(f"ct_pack_gather_{gk}", D.ptr(mu), C.byref(g), D.ptr(gather), D.stream_handle())
    outs = []
    for gp in (None, gather):
        p = torch.empty((6, geom.det_rows, geom.det_cols), device="cuda")
        N.call(f"ct_fp_{gk}", D.ptr(mu), D.ptr(gp), C.byref(g), D.ptr(table), C.byref(b),
               C.byref(s), D.ptr(p), None, D.stream_handle())
        outs.append(p)
    assert outs[0].abs().max() > 0
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("kind", ["cyl", "cart"])
def test_quad_footprints_match_plain_bp(rng, kind):
    """The BP's 16-byte footprints (ct_pack_quads) read the same taps as the
    four scattered loads: num / den agree to fp32 rounding of the bilinear form,
    including frame-edge footprints (a grid wider than the field of view)."""
    import ctypes as C
    import torch
    from paper_2005_11976_b200 import _device as D, _native as N
    if kind == "cyl":
        grid = CylGrid(14, 24, 12, 6.0, 10.0, Pose.tilt(0.25, -0.1, [0.4, -0.2, 0.3]))
    else:
        grid = CartGrid.centered(13, 11, 15, 0.8, center=(0.3, -0.2, 0.1))
    geom = ScanGeometry(300.0, 150.0, 30, 26, 0.3, (14.5, 12.5), P.full_turn_angles(7))
    nv = geom.n_proj
    corr = torch.as_tensor(rng.standard_normal((nv, geom.det_rows, geom.det_cols),
                                               dtype=np.float32), device="cuda")
    dets = D.upload_f64(D.det_view_table(geom, range(nv)))
    g = D.grid_c(grid)
    b = D.batch_c(nv, geom.det_rows, geom.det_cols)
    nq = int(N.load_library().ct_quads_floats(C.byref(b)))
    quads = torch.empty(nq, device="cuda")
    N.call("ct_pack_quads", D.ptr(corr), C.byref(b), D.ptr(quads), D.stream_handle())
    res = []
    for q in (None, quads):
        num = torch.empty(grid.shape, device="cuda")
        den = torch.empty(grid.shape, device="cuda")
        if kind == "cyl":
            trig = D.upload_f64(D.trig_table(grid))
            N.call("ct_bp_cyl", D.ptr(corr), D.ptr(q), D.ptr(dets), C.byref(b), C.byref(g),
                   D.ptr(trig), D.ptr(num), D.ptr(den), 0, D.stream_handle())
        else:
            N.call("ct_bp_cart", D.ptr(corr), D.ptr(q), D.ptr(dets), C.byref(b), C.byref(g),
                   D.ptr(num), D.ptr(den), 0, D.stream_handle())
        res.append((num, den))
    (n0, d0), (n1, d1) = res
    assert (d0 > 0).any() and (d0 == 0).any()          # touched and untouched voxels
    assert torch.equal(d0 > 0, d1 > 0)
    assert torch.allclose(d0, d1, rtol=1e-6, atol=1e-6)
    assert torch.allclose(n0, n1, rtol=1e-5, atol=1e-5)


def test_quad_layout_sart_bit_identical(small_cyl_setup, monkeypatch):
    """A whole OS-SART run through the GL_QUAD volume layout (the large-volume
    choice) gives the same bits as through GL_OCT."""
    grid, vol, ps = small_cyl_setup
    cfg = SartConfig(n_iterations=2, n_subsets=3, relaxation=0.6)
    out = []
    for quad, obrick in (("0", "0"), ("1", "0"), ("0", "1")):
        monkeypatch.setenv("CT_GATHER_QUAD", quad)
        monkeypatch.setenv("CT_GATHER_OBRICK", obrick)
        v, r = sart_run(ps, grid, cfg)
        out.append((v.mu, r.residuals))
    for o in out[1:]:
        assert np.array_equal(out[0][0], o[0])
        assert out[0][1] == o[1]


def test_sart_update_view_reuses_device_state(small_cyl_setup, monkeypatch):
    """A reference-style loop of sart_update_view calls builds the tables,
    row maxima and buffers once per (grid, geometry, sampling) content, and
    gives the same volume as the one-view-per-launch SartRun path."""
    from paper_2005_11976_b200 import recon
    grid, vol, ps = small_cyl_setup
    built = []
    orig = recon.SartEngine.__init__

    def counting(self, *a, **k):
        built.append(1)
        orig(self, *a, **k)
    monkeypatch.setattr(recon.SartEngine, "__init__", counting)
    recon._VIEW_UPDATERS.clear()
    init = (np.asarray(vol.mu) * 0.5).astype(np.float32)
    work = CylVolume(grid, init.copy())
    cfg = SartConfig(relaxation=0.7)
    for i in range(ps.geom.n_proj):
        sart_update_view(work, ps, i, cfg)
    assert len(built) == 1
    ref, _ = sart_run(ps, grid, SartConfig(relaxation=0.7, initial=CylVolume(grid, init.copy()),
                                           compute_residuals=False))
    assert np.array_equal(work.mu, ref.mu)
    # a different geometry (content) gets its own state; the same content reuses it
    built.clear()
    geom2 = ps.geom.subset(list(range(ps.geom.n_proj))[::-1])
    sart_update_view(work, ProjectionSet(geom2, np.asarray(ps.images)[::-1]), 0, cfg)
    assert len(built) == 1
    sart_update_view(work, ps, 1, cfg)
    assert len(built) == 1
