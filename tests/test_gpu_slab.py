"""Slab decomposition on the GPU (slab.SlabSartRun, ABI v8 band / layer entry points).

The kernels: band FP launches give the same corrections and residual slots
as the full launch, the layer-range pack equals the full pack on its cells,
and ct_row_cells_* bounds the cell layers the march reads.  The driver: the
production GPU engine at world 2 / 3 (ranks sharing the one B200 over gloo,
host-staged transfers, every unowned value poisoned to NaN) reproduces the
single-GPU volume and residuals bit for bit.
"""

import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2005_11976_b200 as P  # noqa: E402


def _problem(cart=False):
    rng = np.random.default_rng(11)
    geom = P.ScanGeometry(400.0, 200.0, 72, 64, 0.2, (35.5, 31.5), P.full_turn_angles(12))
    if cart == "quad":        # C5's layer size: the bricked GL_QUAD layout
        grid = P.CylGrid(12, 1024, 384, 4.0, 8.0, P.Pose.tilt(0.4, 0.07, [0.2, -0.1, 0.3]))
    elif cart:
        grid = P.CartGrid.centered(20, 20, 24, 0.35)
    else:
        grid = P.CylGrid(32, 32, 16, 4.0, 8.0, P.Pose.tilt(0.4, 0.07, [0.2, -0.1, 0.3]))
    truth = (rng.random(grid.shape) * 0.05).astype(np.float32)
    vol = (P.CartVolume if cart is True else P.CylVolume)(grid, truth)
    images = np.asarray(P.forward_project_all(vol, geom).images) * 1.03
    return geom, grid, images.astype(np.float32)


@pytest.mark.parametrize("cart", [False, True, "quad"])
def test_band_launches_match_full_launch(cart):
    """Corrections of per-view row bands (tile-aligned) land at their
    full-stack positions with the full launch's bits, and the band launches'
    residual partials fill the full launch's slots."""
    from paper_2005_11976_b200.recon import SartEngine
    from paper_2005_11976_b200 import _device as D
    geom, grid, images = _problem(cart)
    eng = SartEngine(grid, geom, P.RaySamplingConfig())
    eng.prepare_thresholds()
    n = geom.n_proj
    mu = torch.as_tensor(np.random.default_rng(1).random(grid.shape).astype(np.float32) * 0.05,
                         device="cuda")
    gather = eng.alloc_gather()
    eng.pack(mu, gather)
    p = torch.as_tensor(images, device="cuda")
    slots = D.upload_i32(np.arange(n))
    full = torch.zeros((n, geom.det_rows, geom.det_cols), device="cuda")
    eng.correction(mu, p, slots, n, full, gather)
    scr_full = eng.residual_scratch(n).clone().zero_()
    eng.residual_rows(mu, p, slots, n, n, scr_full, gather=gather)
    tile = eng.row_tile()
    H = geom.det_rows
    rng = np.random.default_rng(2)
    cuts = np.sort(rng.integers(0, H // tile + 1, size=(n, 2)), axis=1) * tile
    cuts = np.minimum(cuts, H)
    parts = [np.stack([np.zeros(n, int), cuts[:, 0]], 1), np.stack([cuts[:, 0], cuts[:, 1]], 1),
             np.stack([cuts[:, 1], np.full(n, H)], 1)]
    got = torch.full_like(full, float("nan"))
    scr = torch.zeros_like(scr_full)
    for bands in parts:
        rows = int((bands[:, 1] - bands[:, 0]).max())
        if rows == 0:
            continue
        dev = D.upload_i32(bands.reshape(-1).astype(np.int32))
        eng.correction_bands(mu, p, slots, n, got, dev, rows, gather=gather)
        eng.residual_bands(mu, p, slots, n, dev, rows, n, scr, gather=gather)
    assert torch.equal(got, full)
    assert torch.equal(scr, scr_full)


@pytest.mark.parametrize("cart", [False, True, "quad"])
def test_layer_pack_and_row_cells(cart):
    """ct_pack_gather_*_layers writes exactly the full pack's cells of its
    range; ct_row_cells_* bounds the march's cell layers: an FP through a
    gather buffer packed only on a row's window (NaN elsewhere) is finite and
    equal to the full-layout FP."""
    from paper_2005_11976_b200.recon import SartEngine
    from paper_2005_11976_b200 import _device as D
    from paper_2005_11976_b200 import _native as N
    import ctypes as C
    geom, grid, images = _problem(cart)
    eng = SartEngine(grid, geom, P.RaySamplingConfig())
    eng.prepare_thresholds()
    mu = torch.as_tensor(np.random.default_rng(3).random(grid.shape).astype(np.float32),
                         device="cuda")
    ref = eng.alloc_gather()
    ref.fill_(float("nan"))
    eng.pack(mu, ref)
    if cart == "quad":
        assert N.load_library().ct_gather_layout_cyl(C.byref(eng.gc)) == 2
    part = torch.full_like(ref, float("nan"))
    eng.pack_layers(mu, part, 0, grid.shape[0])      # the full range = ct_pack_gather_*
    assert torch.equal(torch.nan_to_num(part, nan=-7.0), torch.nan_to_num(ref, nan=-7.0))
    cells = eng.row_cells(np.arange(geom.n_proj))
    ok = cells[..., 0] <= cells[..., 1]
    assert ok.any() and (cells[ok, 0] >= 0).all() and (cells[ok, 1] <= grid.shape[0]).all()
    p = torch.as_tensor(images, device="cuda")
    H = geom.det_rows
    full = torch.zeros((geom.n_proj, H, geom.det_cols), device="cuda")
    slots = D.upload_i32(np.arange(geom.n_proj))
    eng.correction(mu, p, slots, geom.n_proj, full, ref)
    tile = eng.row_tile()
    for r0 in range(0, H, 2 * tile):
        r1 = min(r0 + 2 * tile, H)
        c = cells[:, r0:r1]
        okb = c[..., 0] <= c[..., 1]
        if not okb.any():
            continue
        # the driver's window: the rows' cell layers with one layer of margin
        lo, hi = int(c[okb, 0].min()) - 1, int(c[okb, 1].max()) + 1
        buf = torch.full_like(ref, float("nan"))
        eng.pack_layers(mu, buf, lo, hi)
        bands = np.tile(np.array([r0, r1], np.int32), (geom.n_proj, 1))
        got = torch.full_like(full, float("nan"))
        eng.correction_bands(mu, p, slots, geom.n_proj, got, D.upload_i32(bands.reshape(-1)),
                             r1 - r0, gather=buf)
        assert torch.equal(got[:, r0:r1], full[:, r0:r1]), (r0, lo, hi)


def _slab_gpu_worker(rank, world, port, outdir, cart):
    import os
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist
    import paper_2005_11976_b200 as PP
    from paper_2005_11976_b200 import distributed as PD
    dist.init_process_group("gloo", rank=rank, world_size=world)
    geom, grid, images = _problem(cart)
    cfg = PP.SartConfig(relaxation=0.4, n_iterations=3, n_subsets=3)
    run = PD.SlabSartRun(PP.ProjectionSet(geom, images), grid, cfg, poison=True)
    vol, rep = run.run()
    np.savez(Path(outdir) / f"s{rank}.npz", mu=np.asarray(vol.mu), res=rep.residuals,
             need=np.array(run.plan.stats()["mu_need_layers"]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,cart", [(2, False), (3, False), (2, True)])
def test_slab_gpu_engine_ranks_bit_identical(tmp_path, world, cart):
    """The slab-decomposed driver with the GPU engine at world 2 / 3 (ranks on
    one GPU over gloo, unowned data poisoned): band FPs from window-packed
    gather layouts, correction-row and mu-layer exchanges, slab updates and
    the deferred residual give the single-GPU volume and residuals bit for
    bit on every rank."""
    import torch.multiprocessing as mp
    from paper_2005_11976_b200.recon import SartRun
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.start_processes(_slab_gpu_worker, args=(world, port, str(tmp_path), cart), nprocs=world,
                       start_method="spawn", join=True)
    geom, grid, images = _problem(cart)
    cfg = P.SartConfig(relaxation=0.4, n_iterations=3, n_subsets=3)
    ref, rref = SartRun(P.ProjectionSet(geom, images), grid, cfg).run()
    for r in range(world):
        d = np.load(tmp_path / f"s{r}.npz")
        assert np.array_equal(d["mu"], np.asarray(ref.mu))
        assert list(d["res"]) == rref.residuals
        assert d["need"].max() < grid.shape[0]


def test_peer_stores_follow_their_ranges():
    """The fused exchange's kernel side with three local buffers standing in
    for the ranks' symmetric-memory replicas: the band FP stores each
    correction into exactly the replicas whose row range holds its row, the
    BP update each voxel into exactly the replicas whose voxel range holds
    it, with the plain launches' values."""
    from paper_2005_11976_b200.recon import SartEngine, make_update
    from paper_2005_11976_b200 import _device as D
    geom, grid, images = _problem()
    cfg = P.SartConfig(relaxation=0.4)
    eng = SartEngine(grid, geom, cfg.sampling)
    eng.prepare_thresholds()
    n, H, W = geom.n_proj, geom.det_rows, geom.det_cols
    rng = np.random.default_rng(5)
    mu = torch.as_tensor(rng.random(grid.shape).astype(np.float32) * 0.05, device="cuda")
    gather = eng.alloc_gather()
    eng.pack(mu, gather)
    p = torch.as_tensor(images, device="cuda")
    slots = D.upload_i32(np.arange(n))
    tile = eng.row_tile()
    bands = np.tile(np.array([tile, H - tile], np.int32), (n, 1))
    bdev = D.upload_i32(bands.reshape(-1))
    ref = torch.full((n, H, W), float("nan"), device="cuda")
    eng.correction_bands(mu, p, slots, n, ref, bdev, H - 2 * tile, gather=gather)
    k = 3
    reps = [torch.full((n, H, W), float("nan"), device="cuda") for _ in range(k)]
    ptrs = torch.tensor([t.data_ptr() for t in reps], dtype=torch.int64, device="cuda")
    rows = np.sort(rng.integers(0, H + 1, size=(n, k, 2)), axis=2).astype(np.int32)
    local = torch.full((n, H, W), float("nan"), device="cuda")
    eng.correction_bands(mu, p, slots, n, local, bdev, H - 2 * tile, gather=gather,
                         peers=ptrs.data_ptr(), n_peers=k,
                         peer_rows=D.upload_i32(rows.reshape(-1)))
    assert torch.isnan(local).all()      # with peers the stores go to the replicas only
    for q in range(k):
        got = reps[q].cpu().numpy()
        want = ref.cpu().numpy()
        for b in range(n):
            lo, hi = max(rows[b, q, 0], tile), min(rows[b, q, 1], H - tile)
            inside = np.zeros(H, bool)
            inside[lo:hi] = True
            assert np.array_equal(got[b, inside], want[b, inside])
            assert np.isnan(got[b, ~inside]).all()
    # BP update: voxel ranges per replica
    corr = torch.nan_to_num(ref, nan=0.0)
    quads = eng.alloc_quads(n)
    eng.pack_quads(corr, n, quads)
    mu_ref = mu.clone()
    upd = make_update(mu_ref, None, cfg)
    eng.bp_update(corr, slots, n, upd, quads)
    nvox = mu.numel()
    mreps = [torch.full_like(mu, -1.0) for _ in range(k)]
    mptrs = torch.tensor([t.data_ptr() for t in mreps], dtype=torch.int64, device="cuda")
    ranges = np.sort(rng.integers(0, nvox + 1, size=(k, 2)), axis=1).astype(np.int64)
    ranges[0] = (0, nvox)
    rdev = torch.as_tensor(ranges.reshape(-1), device="cuda")
    src = mu.clone()
    upd2 = make_update(src, None, cfg)
    upd2.mu_peers, upd2.n_peers, upd2.peer_ranges = mptrs.data_ptr(), k, rdev.data_ptr()
    eng.bp_update(corr, slots, n, upd2, quads)
    changed = (mu_ref != mu).cpu().numpy().ravel()
    assert changed.any()
    want = mu_ref.cpu().numpy().ravel()
    for q in range(k):
        got = mreps[q].cpu().numpy().ravel()
        sel = np.zeros(nvox, bool)
        sel[ranges[q, 0]:ranges[q, 1]] = True
        # stored: the updated value wherever the update touched the voxel
        assert np.array_equal(got[sel & changed], want[sel & changed])
        assert (got[~sel] == -1.0).all()
    assert torch.equal(src, mu)          # the source replica is read, never written


@pytest.mark.parametrize("fused", ["0", "1"])
def test_slab_run_on_one_rank_group_matches_single_gpu(monkeypatch, fused):
    """The slab driver on a 1-rank NCCL group gives the single-GPU result;
    fused="1": corrections and voxels stored into the symmetric-memory
    replicas by the kernels, device barriers instead of the P2P exchanges."""
    monkeypatch.setenv("CT_FUSED_COMM", fused)
    import os
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
        geom, grid, images = _problem()
        ps = P.ProjectionSet(geom, images)
        cfg = P.SartConfig(relaxation=0.4, n_iterations=2, n_subsets=3)
        run = PD.SlabSartRun(ps, grid, cfg)
        assert run.fused == (fused == "1")
        a, ra = run.run()
        b, rb = SartRun(ps, grid, cfg).run()
        assert np.array_equal(np.asarray(a.mu), np.asarray(b.mu))
        assert ra.residuals == rb.residuals
    finally:
        dist.destroy_process_group()


def _batch_gpu_worker(rank, world, port, outdir, g_ang):
    import os
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist
    import paper_2005_11976_b200 as PP
    from paper_2005_11976_b200 import distributed as PD
    dist.init_process_group("gloo", rank=rank, world_size=world)
    items = _batch_items(PP)
    cfg = PP.SartConfig(relaxation=0.4, n_iterations=2, n_subsets=3)
    out = PD.reconstruct_batch(items, cfg, rank, world, g_ang=g_ang)
    np.savez(Path(outdir) / f"b{rank}.npz", idx=np.array(sorted(out)),
             mu=np.stack([np.asarray(out[i][0].mu) for i in sorted(out)]),
             res=np.array([out[i][1].residuals for i in sorted(out)]))
    dist.destroy_process_group()


def _batch_items(PP):
    geom, grid, _ = _problem()
    items = []
    for k in range(3):
        rng = np.random.default_rng(70 + k)
        g = PP.CylGrid(grid.n_h, grid.n_theta, grid.n_r, grid.radius, grid.height,
                       PP.Pose.tilt(float(rng.uniform(0, 3)), float(rng.uniform(0, 0.12)),
                                    list(rng.uniform(-0.3, 0.3, 2)) + [0.0]))
        truth = (rng.random(g.shape) * 0.05).astype(np.float32)
        imgs = np.asarray(PP.forward_project_all(PP.CylVolume(g, truth), geom).images) * 1.02
        items.append((PP.ProjectionSet(geom, imgs.astype(np.float32)), g))
    return items


@pytest.mark.parametrize("g_ang", [1, 2])
def test_batch_default_runner_gpu_ranks_bit_identical(tmp_path, g_ang):
    """reconstruct_batch with its default drivers (SartRun per object for
    G_ang = 1; the slab-decomposed SlabSartRun on each object group for
    G_ang = 2) over 2 gloo ranks sharing the B200: every object is
    reconstructed by one group and equals the single-GPU run bit for bit."""
    import torch.multiprocessing as mp
    from paper_2005_11976_b200.recon import SartRun
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    world = 2
    mp.start_processes(_batch_gpu_worker, args=(world, port, str(tmp_path), g_ang),
                       nprocs=world, start_method="spawn", join=True)
    items = _batch_items(P)
    cfg = P.SartConfig(relaxation=0.4, n_iterations=2, n_subsets=3)
    ref = [SartRun(ps, g, cfg).run() for ps, g in items]
    seen = set()
    for r in range(world):
        d = np.load(tmp_path / f"b{r}.npz")
        for k, i in enumerate(d["idx"]):
            seen.add(int(i))
            assert np.array_equal(d["mu"][k], np.asarray(ref[int(i)][0].mu))
            assert list(d["res"][k]) == ref[int(i)][1].residuals
    assert seen == {0, 1, 2}
