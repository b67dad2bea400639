"""Parity at BASELINE.json's full configuration sizes (C2-C5).

The fp64 oracle needs ~0.3-2 s per view at these sizes, so full iterations
are infeasible on the CPU.  Instead: sampled pixels / single
views / one subset update against the oracle at FULL size, plus
size-independent properties on whole volumes (row sums bit-exact, linearity,
consistent data is a fixed point, constant correction back-projects to its
value).
"""

import numpy as np
import pytest
import torch

import paper_2005_11976_b200 as P
from paper_2005_11976_b200 import workloads as W

pytestmark = pytest.mark.gpu

PROJ_TOL = 1e-4
RECON_TOL = 1e-3
BP_TOL = 1e-4      # back-projection sums at full size (see test_c4_...)


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def f32(a):
    return np.asarray(a, np.float64).astype(np.float32).astype(np.float64)


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


def _sample_pixels(geom, n, seed):
    rng = np.random.default_rng(seed)
    idx = rng.choice(geom.det_rows * geom.det_cols, n, replace=False)
    return np.divmod(idx, geom.det_cols)


@pytest.fixture(scope="module")
def c2():
    return W.c2_medium()


def test_c2_fp_sampled_views_vs_oracle(oracle, c2):
    vol = P.CylVolume(c2.grid, dev(c2.mu))
    ps = P.forward_project_all(vol, c2.geom)          # batched, gather layout
    for i in (3, 211):
        rows, cols = _sample_pixels(c2.geom, 3000, i)
        p_o, w_o = oracle.forward_pixels(c2.mu, c2.grid, c2.geom, i, rows, cols)
        p, w = P.forward_project(vol, c2.geom, i, return_weights=True)
        assert np.array_equal(w.cpu().numpy()[rows, cols], f32(w_o))
        assert rel_l2(p.cpu().numpy()[rows, cols], p_o) < PROJ_TOL
        assert torch.equal(p, ps.images[i])


def test_c2_one_os_subset_update_vs_oracle(oracle, c2):
    """One OS-SART subset (45 views, S=8, lambda 0.3) from zero at full size."""
    vol = P.CylVolume(c2.grid, dev(c2.mu))
    images = P.forward_project_all(vol, c2.geom).images.cpu().numpy()
    sub = P.make_subsets(np.arange(c2.geom.n_proj), 8)[0]
    mu = np.zeros(c2.grid.shape)
    num = np.zeros(c2.grid.shape)
    den = np.zeros(c2.grid.shape)
    for i in sub:
        c = oracle.correction(mu, c2.grid, c2.geom, int(i), images[int(i)])
        oracle.back(c, c2.geom, int(i), c2.grid, out=(num, den))
    oracle._apply_update(mu, num, den, None, 0.3, True)
    from paper_2005_11976_b200.recon import SartRun
    run = SartRun(P.ProjectionSet(c2.geom, dev(images)), c2.grid,
                  P.SartConfig(relaxation=0.3, n_iterations=1, n_subsets=8,
                               compute_residuals=False))
    e = run.eng
    e.pack(run.mu, run.gather)
    e.correction(run.mu, run.p_meas, run.subset_slots[0], len(sub), run.corr, run.gather)
    e.bp_update(run.corr, run.subset_slots[0], len(sub), run.upd)
    assert rel_l2(run.mu.cpu().numpy(), mu) < RECON_TOL


def test_c2_consistent_data_fixed_point(c2):
    vol = P.CylVolume(c2.grid, dev(c2.mu))
    ps = P.forward_project_all(vol, c2.geom)
    out, rep = P.sart_run(ps, c2.grid, P.SartConfig(relaxation=0.3, n_iterations=1,
                                                     n_subsets=8, initial=vol))
    assert torch.equal(out.mu, vol.mu)
    assert rep.residuals == [0.0]


def test_c2_linearity_full_volume(c2):
    rng = np.random.default_rng(9)
    m1 = dev(c2.mu)
    m2 = dev((rng.random(c2.grid.shape, dtype=np.float32) * 0.01))
    views = [0, 90]
    geom = c2.geom.subset(views)
    a, b = 0.5, 2.0
    p1 = P.forward_project_all(P.CylVolume(c2.grid, m1), geom).images
    p2 = P.forward_project_all(P.CylVolume(c2.grid, m2), geom).images
    p12 = P.forward_project_all(P.CylVolume(c2.grid, a * m1 + b * m2), geom).images
    err = (p12.double() - (a * p1.double() + b * p2.double())).abs().max().item()
    assert err < 1e-5 * p12.abs().max().item()


def test_c3_weighted_template_sart_vs_oracle(oracle):
    """Config C3: 30 views, weights (1.0 ROI / 0.2), template initial volume,
    lambda 0.5 -- one full SART pass vs the oracle."""
    c3 = W.c3_sparse()
    vol = P.CylVolume(c3.grid, dev(c3.mu))
    images = P.forward_project_all(vol, c3.geom).images.cpu().numpy()
    mu_o, res_o = oracle.sart(images, c3.grid, c3.geom, relaxation=0.5, n_iterations=1,
                              weights=c3.weights, initial=c3.template)
    out, rep = P.sart_run(P.ProjectionSet(c3.geom, images), c3.grid,
                          P.SartConfig(relaxation=0.5, n_iterations=1, weights=c3.weights,
                                       initial=P.CylVolume(c3.grid, c3.template)))
    assert rel_l2(out.mu, mu_o) < RECON_TOL
    assert np.allclose(rep.residuals, res_o, rtol=1e-3)
    frozen = c3.weights == 0.0
    assert not frozen.any() or np.array_equal(out.mu[frozen], c3.template[frozen])


def test_c4_cyl_and_cart_projectors_vs_oracle(oracle):
    """Config C4 at full size: 768^2 detector, (512,1024,384) cylindrical and
    512^3 Cartesian grids of the same phantom."""
    cyl, cart, geom, ph = W.c4_grids()
    mu_c = W.rasterize_cyl(ph, cyl)
    mu_x = W.rasterize_cart(ph, cart)
    vc = P.CylVolume(cyl, dev(mu_c))
    vx = P.CartVolume(cart, dev(mu_x))
    for vol, mu, grid in ((vc, mu_c, cyl), (vx, mu_x, cart)):
        i = 123
        rows, cols = _sample_pixels(geom, 1500, i)
        p_o, w_o = oracle.forward_pixels(mu, grid, geom, i, rows, cols)
        p, w = P.forward_project(vol, geom, i, return_weights=True)
        assert np.array_equal(w.cpu().numpy()[rows, cols], f32(w_o))
        assert rel_l2(p.cpu().numpy()[rows, cols], p_o) < PROJ_TOL
    # the two discretisations of the same object agree to discretisation error
    pc = P.forward_project(vc, geom, 0).cpu().numpy()
    px = P.forward_project(vx, geom, 0).cpu().numpy()
    assert rel_l2(pc, px) < 0.05
    # BP of one view against the oracle (corrections of the right scale)
    corr = np.random.default_rng(4).normal(0, 0.01, (geom.det_rows, geom.det_cols))
    corr = corr.astype(np.float32)
    num, den = P.back_project(dev(corr), geom, 7, cart)
    n_o, d_o = oracle.back(corr, geom, 7, cart)
    # fp32 detector coordinates up to 768 px carry ~3e-5 px of rounding; against
    # a per-pixel white-noise image that is ~3e-5 relative in num.  Bar: the
    # north_star projection tolerance.
    assert rel_l2(num.cpu().numpy(), n_o) < BP_TOL
    assert rel_l2(den.cpu().numpy(), d_o) < BP_TOL


def test_c5_object_views_vs_oracle(oracle):
    """Config C5 object at full size: 1024^2 detector, (512,1024,384) grid."""
    wl = W.c5_object(3)
    vol = P.CylVolume(wl.grid, dev(wl.mu))
    i = 77
    rows, cols = _sample_pixels(wl.geom, 1500, i)
    p_o, w_o = oracle.forward_pixels(wl.mu, wl.grid, wl.geom, i, rows, cols)
    p, w = P.forward_project(vol, wl.geom, i, return_weights=True)
    assert np.array_equal(w.cpu().numpy()[rows, cols], f32(w_o))
    assert rel_l2(p.cpu().numpy()[rows, cols], p_o) < PROJ_TOL
    corr = np.full((wl.geom.det_rows, wl.geom.det_cols), 2.5, dtype=np.float32)
    num, den = P.back_project(dev(corr), wl.geom, i, wl.grid)
    inside = den > 0
    assert torch.allclose(num[inside] / den[inside], torch.tensor(2.5, device="cuda"),
                          rtol=1e-6)


@pytest.mark.parametrize("fused", ["0", "1"])
def test_sharded_run_on_one_rank_group_matches_single_gpu(monkeypatch, fused):
    """The angle-sharded driver on a 1-rank NCCL group gives the single-GPU
    result; fused="1": the symmetric-memory path (corrections and voxels
    stored into the replicas by the kernels, barriers instead of
    all-gathers)."""
    monkeypatch.setenv("CT_FUSED_COMM", fused)
    import os
    import socket
    import torch.distributed as dist
    from paper_2005_11976_b200 import distributed as PD
    from paper_2005_11976_b200.recon import SartRun
    if dist.is_initialized():
        pytest.skip("process group already initialised")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rng = np.random.default_rng(2)
        geom = P.ScanGeometry(400.0, 200.0, 48, 40, 0.2, (23.5, 19.5), P.full_turn_angles(12))
        grid = P.CylGrid(16, 32, 16, 4.0, 8.0, P.Pose.tilt(0.4, 0.06, [0.2, -0.1, 0.0]))
        truth = (rng.random(grid.shape) * 0.05).astype(np.float32)
        ps = P.forward_project_all(P.CylVolume(grid, dev(truth)), geom)
        cfg = P.SartConfig(relaxation=0.4, n_iterations=2, n_subsets=3)
        srun = PD.ShardedSartRun(ps, grid, cfg)
        assert srun.fused == (fused == "1")
        a, ra = srun.run()
        b, rb = SartRun(ps, grid, cfg).run()
        # every correction / voxel update / residual partial is the 1-GPU one
        assert torch.equal(a.mu, b.mu)
        assert ra.residuals == rb.residuals
        out = PD.reconstruct_batch([(ps, grid), (ps, grid)], cfg, rank=0, world=1)
        assert sorted(out) == [0, 1]
        assert torch.equal(out[0][0].mu, out[1][0].mu)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_kernels_split_bit_identical(world):
    """The angle-sharded building blocks on one GPU, rank by rank: tile-aligned
    row ranges of the correction FP reproduce the full correction stack, the
    per-rank residual slot partials (zeros outside a rank's rows) add up to the
    full residual bit for bit, and voxel-range BP updates reproduce the full
    fused update."""
    from paper_2005_11976_b200 import distributed as PD
    from paper_2005_11976_b200.recon import SartRun
    rng = np.random.default_rng(11)
    geom = P.ScanGeometry(400.0, 200.0, 64, 56, 0.2, (31.5, 27.5), P.full_turn_angles(9))
    grid = P.CylGrid(16, 32, 16, 4.0, 8.0, P.Pose.tilt(0.4, 0.06, [0.2, -0.1, 0.0]))
    truth = (rng.random(grid.shape) * 0.05).astype(np.float32)
    ps = P.forward_project_all(P.CylVolume(grid, dev(truth)), geom)
    ps = P.ProjectionSet(geom, ps.images * 1.03)
    run = SartRun(ps, grid, P.SartConfig(relaxation=0.5, n_iterations=1, n_subsets=2))
    e = run.eng
    mu0 = dev(truth * 0.9)
    run.mu.copy_(mu0)
    e.pack(run.mu, run.gather)
    sub, slots = run.subsets[0], run.subset_slots[0]
    n, H, W = len(sub), geom.det_rows, geom.det_cols
    full = torch.zeros((n, H, W), device="cuda")
    e.correction(run.mu, run.p_meas, slots, n, full, run.gather)
    acc_full = torch.zeros(1, dtype=torch.float64, device="cuda")
    e.residual(run.mu, run.p_meas, run.all_slots, geom.n_proj, acc_full, run.gather)

    tile = e.row_tile()
    b = PD.row_bounds(n, H, world, tile)
    split = torch.zeros(n * H * W, device="cuda")
    total = e.residual_scratch(geom.n_proj).clone().zero_()
    rest = np.setdiff1d(np.arange(geom.n_proj), sub)
    rb = PD.row_bounds(len(rest), H, world, tile)
    for r in range(world):
        mine = torch.zeros_like(e.residual_scratch(geom.n_proj))
        lo, hi = int(b[r]), int(b[r + 1])
        if hi > lo:
            v0, v1 = lo // H, (hi - 1) // H
            out = torch.zeros((hi - lo) * W, device="cuda")
            e.correction_rows(run.mu, run.p_meas, slots[v0:v1 + 1], v1 - v0 + 1, out,
                              lo - v0 * H, hi - v0 * H, geom.n_proj, mine, run.gather)
            split[lo * W:hi * W] = out
        lo, hi = int(rb[r]), int(rb[r + 1])
        if hi > lo:
            v0, v1 = lo // H, (hi - 1) // H
            rs = P._device.upload_i32(rest[v0:v1 + 1])
            e.residual_rows(run.mu, run.p_meas, rs, v1 - v0 + 1, geom.n_proj, mine,
                            lo - v0 * H, hi - v0 * H, run.gather)
        total += mine
    assert torch.equal(split.view(n, H, W), full)
    acc = torch.zeros(1, dtype=torch.float64, device="cuda")
    e.residual_sum(total, acc)
    assert acc.item() == acc_full.item()

    # voxel-range BP updates == the full fused update
    quads = e.alloc_quads(n)
    e.pack_quads(full, n, quads)
    ref = mu0.clone()
    e.bp_update(full, slots, n, P.recon.make_update(ref, None, run.cfg), quads)
    got = mu0.clone()
    upd = P.recon.make_update(got, None, run.cfg)
    nvox = grid.n_voxels
    for r in range(world):
        off, cnt, _ = PD.shard_range(nvox, r, world)
        e.bp_update_range(full, slots, n, upd, off, cnt, quads)
    assert torch.equal(got, ref)


def test_row_samples_match_row_sums():
    """ct_row_samples_*: per detector row, the in-support sample counts that
    the FP's row sums w = count * step / ss^2 carry (exact integers)."""
    from paper_2005_11976_b200.recon import SartEngine
    geom = P.ScanGeometry(400.0, 200.0, 40, 36, 0.2, (19.5, 17.5), P.full_turn_angles(5))
    for grid in (P.CylGrid(12, 24, 10, 4.0, 6.0, P.Pose.tilt(0.3, 0.05, [0.3, 0.1, 0.0])),
                 P.CartGrid.centered(10, 12, 8, 0.6)):
        samp = P.RaySamplingConfig(supersample=2)
        eng = SartEngine(grid, geom, samp)
        got = eng.row_samples(np.arange(geom.n_proj))
        mu = torch.zeros(grid.shape, device="cuda")
        vol = (P.CylVolume if isinstance(grid, P.CylGrid) else P.CartVolume)(grid, mu)
        step = samp.step_for(grid)
        for i in range(geom.n_proj):
            _, w = P.forward_project(vol, geom, i, samp, return_weights=True)
            counts = np.rint(np.asarray(w.cpu() if hasattr(w, "cpu") else w, np.float64)
                             * 4 / step).sum(axis=1)
            assert np.array_equal(got[i], counts.astype(np.int64))


def _gloo_gpu_worker(rank, world, port, outdir, decomposition="rows"):
    """One rank of the angle-sharded driver with the production GPU engine;
    all ranks share cuda:0 and a gloo group (host-staged collectives, so no
    rank's kernels wait on another's)."""
    import os
    import sys
    from pathlib import Path
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist
    import paper_2005_11976_b200 as P
    from paper_2005_11976_b200 import distributed as PD
    dist.init_process_group("gloo", rank=rank, world_size=world)
    geom, grid, images, cfg = _gloo_gpu_problem(P)
    vol, rep = PD.sart_run_sharded(P.ProjectionSet(geom, images), grid, cfg,
                                   decomposition=decomposition)
    np.savez(Path(outdir) / f"r{rank}.npz", mu=np.asarray(vol.mu), res=rep.residuals)
    dist.destroy_process_group()


def _gloo_gpu_problem(P):
    rng = np.random.default_rng(4)
    geom = P.ScanGeometry(400.0, 200.0, 64, 56, 0.2, (31.5, 27.5), P.full_turn_angles(10))
    grid = P.CylGrid(16, 32, 16, 4.0, 8.0, P.Pose.tilt(0.4, 0.06, [0.2, -0.1, 0.0]))
    truth = (rng.random(grid.shape) * 0.05).astype(np.float32)
    images = np.asarray(P.forward_project_all(P.CylVolume(grid, truth), geom).images) * 1.03
    cfg = P.SartConfig(relaxation=0.4, n_iterations=3, n_subsets=3)
    return geom, grid, images.astype(np.float32), cfg


@pytest.mark.parametrize("world,decomposition", [(2, "rows"), (3, "rows"), (3, "slab")])
def test_sharded_gpu_engine_ranks_bit_identical(tmp_path, world, decomposition):
    """The whole angle-sharded driver with the GPU engine at world 2 / 3 (ranks
    on one GPU over gloo): row-restricted uploads, cost-balanced row split,
    all-gathers, voxel-range updates and the deferred residual give the
    single-GPU volume and residuals bit for bit on every rank."""
    import socket
    import torch.multiprocessing as mp
    from paper_2005_11976_b200.recon import SartRun
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.start_processes(_gloo_gpu_worker, args=(world, port, str(tmp_path), decomposition),
                       nprocs=world,
                       start_method="spawn", join=True)
    geom, grid, images, cfg = _gloo_gpu_problem(P)
    ref, rref = SartRun(P.ProjectionSet(geom, images), grid, cfg).run()
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        assert np.array_equal(d["mu"], np.asarray(ref.mu))
        assert list(d["res"]) == rref.residuals
