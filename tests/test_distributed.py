"""Multi-process host logic of the sharded paths, on CPU with gloo (world size 2).

The production engine is the GPU one; here the same ShardedSartRun drives an
oracle-backed engine, so partitioning, the reduce-scatter / update-offset /
all-gather sequence and the residual all-reduce are checked against the
single-process OS-SART oracle.
"""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class OracleEngine:
    """CPU engine with GpuEngine's interface, computing with the fp64 oracle.

    Residual scratch layout: one partial per (view slot, detector row)."""

    TILE = 4

    def __init__(self, orc, ps, grid, cfg):
        import torch
        self.torch, self.o = torch, orc
        self.ps, self.grid, self.cfg = ps, grid, cfg
        self.H, self.W = ps.geom.det_rows, ps.geom.det_cols
        self.images = np.asarray(ps.images, dtype=np.float64)
        self.max_row = None
        self.marched = []            # (view, row) pairs this rank marched (FP)
        self.updated = []            # voxel ranges this rank updated

    def tensor(self, shape, dtype="float32"):
        return self.torch.zeros(shape, dtype=self.torch.float64)

    def prepare(self, order):
        self.max_row = {}
        for i in range(self.ps.geom.n_proj):
            _, w = self.o.forward(np.zeros(self.o.grid_shape(self.grid)), self.grid,
                                  self.ps.geom, i)
            self.max_row[i] = w.max()

    def slots(self, views):
        return np.asarray(views)

    def row_tile(self):
        return self.TILE

    def row_costs(self, views):
        """samples per detector row (the oracle's row sums w are counts * step)"""
        out = []
        for v in views:
            _, w = self.o.forward(np.zeros(self.o.grid_shape(self.grid)), self.grid,
                                  self.ps.geom, int(v))
            out.append(w.sum(axis=1))
        return np.concatenate(out) + 1e-3

    def scratch(self, n_slots):
        return self.torch.zeros(n_slots * self.H, dtype=self.torch.float64)

    def pack(self, mu):
        pass

    def _rows(self, slots, n, lo, hi):
        for f in range(lo, hi):
            yield f, int(slots[f // self.H]), f % self.H

    def correction_rows(self, mu, slots, n, out, lo, hi, n_slots, scratch):
        cache = {}
        for f, v, r in self._rows(slots, n, lo, hi):
            if v not in cache:
                c = self.o.correction(mu.numpy(), self.grid, self.ps.geom, v, self.images[v],
                                      max_row=self.max_row[v])
                sim, _ = self.o.forward(mu.numpy(), self.grid, self.ps.geom, v)
                cache[v] = (c, sim)
            c, sim = cache[v]
            out[(f - lo) * self.W:(f - lo + 1) * self.W] = self.torch.from_numpy(c[r])
            if scratch is not None:
                scratch[v * self.H + r] = float(np.sum((self.images[v][r] - sim[r]) ** 2))
            self.marched.append((v, r))

    def residual_rows(self, mu, slots, n, lo, hi, n_slots, scratch):
        cache = {}
        for f, v, r in self._rows(slots, n, lo, hi):
            if v not in cache:
                cache[v], _ = self.o.forward(mu.numpy(), self.grid, self.ps.geom, v)
            scratch[v * self.H + r] = float(np.sum((self.images[v][r] - cache[v][r]) ** 2))

    def residual_sum(self, scratch, acc):
        acc += float(np.sum(scratch.numpy()))

    # -- slab decomposition (slab.SlabSartRun) --------------------------------
    def row_cells(self, views):
        """numpy fp64 restatement of ct_row_cells_cyl (geometry only): per row
        the [min, max] cell layer floor(h index + 1) of the first and last
        samples of its rays."""
        g = self.grid
        step = self.o.default_step(g)
        out = np.empty((len(views), self.H, 2), dtype=np.int64)
        out[..., 0], out[..., 1] = 2 ** 31 - 1, -2 ** 31
        rr, cc = np.meshgrid(np.arange(self.H), np.arange(self.W), indexing="ij")
        for b, v in enumerate(views):
            src, origin, du, dv = self.o.aligned_basis(g, self.ps.geom, int(v))
            d = origin[None, None] + cc[..., None] * du + rr[..., None] * dv - src
            d = d / np.sqrt((d * d).sum(-1))[..., None]
            a = d[..., 0] ** 2 + d[..., 1] ** 2
            bb = src[0] * d[..., 0] + src[1] * d[..., 1]
            c = src[0] ** 2 + src[1] ** 2 - g.radius ** 2
            disc = bb * bb - a * c
            sq = np.sqrt(np.maximum(disc, 0.0))
            tr0, tr1 = (-bb - sq) / a, (-bb + sq) / a
            hh = 0.5 * g.height
            tz0, tz1 = (-hh - src[2]) / d[..., 2], (hh - src[2]) / d[..., 2]
            t0 = np.maximum(np.maximum(tr0, np.minimum(tz0, tz1)), 0.0)
            t1 = np.minimum(tr1, np.maximum(tz0, tz1))
            hit = (disc > 0) & (t1 > t0)
            n = np.ceil((t1 - t0) / step)
            z0 = src[2] + (t0 + 0.5 * step) * d[..., 2]
            z1 = z0 + (n - 1) * step * d[..., 2]
            k0 = np.floor(z0 * g.n_h / g.height + 0.5 * g.n_h + 0.5)
            k1 = np.floor(z1 * g.n_h / g.height + 0.5 * g.n_h + 0.5)
            lo = np.where(hit, np.minimum(k0, k1), 2 ** 31 - 1).min(axis=1)
            hi = np.where(hit, np.maximum(k0, k1), -2 ** 31).max(axis=1)
            out[b, :, 0], out[b, :, 1] = lo, hi
        return out

    def pack_layers(self, mu, kc_lo, kc_hi):
        pass

    def upload_bands(self, bands):
        return np.asarray(bands).reshape(-1, 2)

    def _band_rows(self, slots, bands):
        for b, v in enumerate(slots):
            for r in range(int(bands[b, 0]), int(bands[b, 1])):
                yield b, int(v), r

    def correction_bands(self, mu, slots, n, corr, bands, band_rows, n_slots, scratch):
        cache = {}
        for b, v, r in self._band_rows(slots[:n], bands):
            if v not in cache:
                c = self.o.correction(mu.numpy(), self.grid, self.ps.geom, v, self.images[v],
                                      max_row=self.max_row[v])
                sim, _ = self.o.forward(mu.numpy(), self.grid, self.ps.geom, v)
                cache[v] = (c, sim)
            c, sim = cache[v]
            assert np.all(np.isfinite(c[r])), f"view {v} row {r} read poisoned mu"
            corr[b, r] = self.torch.from_numpy(c[r])
            if scratch is not None:
                scratch[v * self.H + r] = float(np.sum((self.images[v][r] - sim[r]) ** 2))
            self.marched.append((v, r))

    def residual_bands(self, mu, slots, n, bands, band_rows, n_slots, scratch):
        cache = {}
        for b, v, r in self._band_rows(slots[:n], bands):
            if v not in cache:
                cache[v], _ = self.o.forward(mu.numpy(), self.grid, self.ps.geom, v)
            assert np.all(np.isfinite(cache[v][r])), f"view {v} row {r} read poisoned mu"
            scratch[v * self.H + r] = float(np.sum((self.images[v][r] - cache[v][r]) ** 2))

    def bp_update_range(self, corr, slots, n, offset, count, mu):
        shape = self.o.grid_shape(self.grid)
        num, den = np.zeros(shape), np.zeros(shape)
        for b, i in enumerate(slots[:n]):
            self.o.back(corr[b].numpy(), self.ps.geom, int(i), self.grid, out=(num, den))
        w = None
        if self.cfg.weights is not None:
            w = np.asarray(self.cfg.weights, dtype=np.float64).ravel()[offset:offset + count]
        self.o._apply_update(mu.view(-1)[offset:offset + count].numpy(),
                             num.ravel()[offset:offset + count],
                             den.ravel()[offset:offset + count], w,
                             self.cfg.relaxation, self.cfg.nonnegativity)
        assert np.all(np.isfinite(mu.view(-1)[offset:offset + count].numpy())), \
            "the BP update read a poisoned correction row"
        self.updated.append((offset, count))


def _problem():
    import paper_2005_11976_b200 as P
    rng = np.random.default_rng(3)
    geom = P.ScanGeometry(400.0, 200.0, 24, 20, 0.4, (11.5, 9.5), P.full_turn_angles(10))
    grid = P.CylGrid(8, 12, 6, 4.0, 8.0, P.Pose.tilt(0.3, 0.05, [0.2, 0.1, 0.0]))
    truth = rng.random(grid.shape) * 0.05
    weights = rng.uniform(0.0, 1.0, grid.shape)
    weights[weights < 0.2] = 0.0
    return P, geom, grid, truth, weights


def _worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "oracle"))
    import torch.distributed as dist
    import oracle as orc
    from paper_2005_11976_b200 import distributed as PD
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P, geom, grid, truth, weights = _problem()
    images = np.stack([orc.forward(truth, grid, geom, i)[0] for i in range(geom.n_proj)])
    ps = P.ProjectionSet(geom, images)
    cfg = P.SartConfig(relaxation=0.4, n_iterations=2, n_subsets=3, weights=weights,
                       projection_order="fixed_permutation", order_seed=1)
    eng = OracleEngine(orc, ps, grid, cfg)
    run = PD.ShardedSartRun(ps, grid, cfg, engine=eng)
    vol, rep = run.run()
    n_sub = len(run.subsets)
    np.savez(Path(outdir) / f"rank{rank}.npz", mu=run.mu.numpy(), res=rep.residuals,
             marched=np.array(eng.marched), updated=np.array(eng.updated), n_sub=n_sub)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_angle_sharded_os_sart_matches_single_process(oracle, tmp_path, world):
    """world 3 gives uneven row chunks (the compaction path)."""
    import torch.multiprocessing as mp
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       start_method="spawn", join=True)
    P, geom, grid, truth, weights = _problem()
    images = np.stack([oracle.forward(truth, grid, geom, i)[0] for i in range(geom.n_proj)])
    images = images.astype(np.float32)
    order = np.random.default_rng(1).permutation(geom.n_proj)
    mu_ref, res_ref = oracle.sart(images, grid, geom, relaxation=0.4, n_iterations=2,
                                  order=order, weights=weights, n_subsets=3)
    rs = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    r0 = rs[0]
    for r in rs[1:]:
        assert np.array_equal(r0["mu"], r["mu"])          # replicas stay identical
    assert np.abs(r0["mu"] - mu_ref).max() <= 1e-12 * np.abs(mu_ref).max()
    assert np.allclose(r0["res"], res_ref, rtol=1e-12)
    # every detector row of every view corrected exactly once per pass across
    # the ranks (2 passes), every voxel updated once per subset
    rows = np.concatenate([r["marched"] for r in rs])
    keys = rows[:, 0] * geom.det_rows + rows[:, 1]
    assert np.array_equal(np.bincount(keys, minlength=geom.n_proj * geom.det_rows),
                          np.full(geom.n_proj * geom.det_rows, 2))
    n_vox = int(np.prod(grid.shape))
    upd = np.concatenate([r["updated"] for r in rs])
    assert upd[:, 1].sum() == n_vox * int(r0["n_sub"]) * 2


def test_shard_helpers():
    from paper_2005_11976_b200 import distributed as PD
    # row ranges: contiguous, covering, at tile boundaries, balanced to a tile
    for n_views, rows, world, tile in [(45, 512, 8, 8), (20, 1024, 8, 8), (5, 20, 3, 4),
                                       (3, 13, 4, 4), (1, 8, 4, 8), (7, 40, 2, 8)]:
        b = PD.row_bounds(n_views, rows, world, tile)
        assert len(b) == world + 1 and b[0] == 0 and b[-1] == n_views * rows
        assert np.all(np.diff(b) >= 0)
        inner = b % rows
        assert np.all((inner % tile == 0) | (b % rows == 0) | (b == n_views * rows))
        if n_views * rows >= world * tile:
            assert np.abs(np.diff(b) - n_views * rows / world).max() <= tile
    assert np.array_equal(PD.row_bounds(45, 512, 8, 8), np.arange(9) * 2880)
    # cost-weighted: rows 0..9 of one view cost 10x the rest
    cost = np.ones(40)
    cost[:10] = 10.0
    b = PD.row_bounds(1, 40, 2, 2, cost)
    assert b[1] == 6                       # 60 of 130 left, 70 right (tile 2)
    assert np.array_equal(PD.row_bounds(1, 40, 2, 2, np.ones(40)), PD.row_bounds(1, 40, 2, 2))
    n = 1001
    ranges = [PD.shard_range(n, r, 4) for r in range(4)]
    covered = sum(c for _, c, _ in ranges)
    assert covered == n and ranges[0][0] == 0 and ranges[-1][0] + ranges[-1][1] == n
    assert PD.assign_objects(10, 1, 4) == [1, 5, 9]


# ---------------------------------------------------------------------------
# object batches: G = G_obj x G_ang (BatchPlan / reconstruct_batch)
# ---------------------------------------------------------------------------
def _batch_items(P, orc, geom, grid_base, n_objects):
    """n seeded objects with their own poses (config C5 in miniature)."""
    items, truths = [], []
    for k in range(n_objects):
        rng = np.random.default_rng(50 + k)
        grid = P.CylGrid(grid_base.n_h, grid_base.n_theta, grid_base.n_r, grid_base.radius,
                         grid_base.height,
                         P.Pose.tilt(float(rng.uniform(0, 3)), float(rng.uniform(0, 0.15)),
                                     list(rng.uniform(-0.3, 0.3, 2)) + [0.0]))
        truth = rng.random(grid.shape) * 0.05
        images = np.stack([orc.forward(truth, grid, geom, i)[0] for i in range(geom.n_proj)])
        items.append((P.ProjectionSet(geom, images.astype(np.float32)), grid))
        truths.append(truth)
    return items


def _batch_worker(rank, world, port, outdir, g_ang, n_objects):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "oracle"))
    import torch.distributed as dist
    import oracle as orc
    from paper_2005_11976_b200 import distributed as PD
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P, geom, grid, _, _ = _problem()
    items = _batch_items(P, orc, geom, grid, n_objects)
    cfg = P.SartConfig(relaxation=0.4, n_iterations=2, n_subsets=3)
    sizes = {}

    def runner(ps, g, c, group):
        # every object through the angle-sharded driver on its group (a
        # 1-rank group for G_ang = 1), with the oracle engine
        sizes[id(ps)] = 1 if group is None else dist.get_world_size(group)
        grp = group if group is not None else dist.new_group([rank])
        run = PD.ShardedSartRun(ps, g, c, group=grp, engine=OracleEngine(orc, ps, g, c))
        return run.run()

    if g_ang == 1:
        # G_ang = 1 has no group; give each rank a 1-rank group (collective creation)
        solo = [dist.new_group([r]) for r in range(world)]
        runner_1 = lambda ps, g, c, group: runner(ps, g, c, solo[rank])  # noqa: E731
        out = PD.reconstruct_batch(items, cfg, rank, world, g_ang=1, runner=runner_1)
    else:
        out = PD.reconstruct_batch(items, cfg, rank, world, g_ang=g_ang, runner=runner)
    np.savez(Path(outdir) / f"b{rank}.npz", idx=np.array(sorted(out)),
             mu=np.stack([np.asarray(out[i][0].mu) for i in sorted(out)]),
             res=np.array([out[i][1].residuals for i in sorted(out)]),
             group_size=max(sizes.values()) if sizes else 0)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,g_ang", [(2, 1), (2, 2), (4, 2)])
def test_batch_reconstruction_object_and_angle_groups(oracle, tmp_path, world, g_ang):
    """reconstruct_batch over G = G_obj x G_ang gloo ranks: every object is
    reconstructed by exactly one object group, all ranks of a group hold the
    same volume, and each equals the single-process OS-SART oracle."""
    import torch.multiprocessing as mp
    n_objects = 3
    mp.start_processes(_batch_worker, args=(world, _free_port(), str(tmp_path), g_ang,
                                            n_objects),
                       nprocs=world, start_method="spawn", join=True)
    P, geom, grid, _, _ = _problem()
    items = _batch_items(P, oracle, geom, grid, n_objects)
    rs = [np.load(tmp_path / f"b{r}.npz") for r in range(world)]
    n_groups = world // g_ang
    seen = {}
    for r, d in enumerate(rs):
        g = r // g_ang
        assert list(d["idx"]) == list(range(g, n_objects, n_groups))
        for k, i in enumerate(d["idx"]):
            if int(i) in seen:                           # same group: identical replicas
                assert seen[int(i)][0] == g
                assert np.array_equal(seen[int(i)][1], d["mu"][k])
            seen[int(i)] = (g, d["mu"][k], d["res"][k])
    assert sorted(seen) == list(range(n_objects))
    for i, (ps, g) in enumerate(items):
        mu_ref, res_ref = oracle.sart(ps.images, g, geom, relaxation=0.4, n_iterations=2,
                                      n_subsets=3)
        _, mu, res = seen[i]
        assert np.abs(mu - mu_ref).max() <= 1e-12 * np.abs(mu_ref).max()
        assert np.allclose(res, res_ref, rtol=1e-12)


def test_batch_plan():
    from paper_2005_11976_b200 import distributed as PD
    from paper_2005_11976_b200.errors import ConfigError
    p = PD.BatchPlan(5, 8, 2)
    assert (p.n_groups, p.group_index, p.group_rank) == (4, 2, 1)
    assert p.group_ranks(2) == [4, 5]
    assert p.objects(64) == list(range(2, 64, 4))
    assert PD.BatchPlan(3, 8, 1).objects(10) == [3]
    assert PD.BatchPlan(0, 8, 8).objects(3) == [0, 1, 2]
    with pytest.raises(ConfigError):
        PD.BatchPlan(0, 8, 3)


# ---------------------------------------------------------------------------
# slab decomposition (slab.SlabSartRun)
# ---------------------------------------------------------------------------
def _slab_problem(variant="base"):
    """Taller grid than _problem so G ranks own slabs of several layers;
    variant "thin": 5 layers over 4 ranks (slabs of one or two layers, some
    ranks' windows the whole volume), a weight map with zeros, a fixed
    permutation and no nonnegativity clamp."""
    import paper_2005_11976_b200 as P
    rng = np.random.default_rng(7)
    geom = P.ScanGeometry(400.0, 200.0, 40, 24, 0.4, (11.5, 19.5), P.full_turn_angles(9))
    n_h = 5 if variant == "thin" else 24
    grid = P.CylGrid(n_h, 12, 6, 4.0, 12.0, P.Pose.tilt(0.3, 0.08, [0.2, 0.1, 0.3]))
    truth = rng.random(grid.shape) * 0.05
    return P, geom, grid, truth


def _slab_cfg(P, grid, variant):
    if variant != "thin":
        return P.SartConfig(relaxation=0.4, n_iterations=2, n_subsets=3)
    w = np.random.default_rng(8).uniform(0.0, 1.0, grid.shape)
    w[w < 0.25] = 0.0
    return P.SartConfig(relaxation=0.6, n_iterations=2, n_subsets=2, weights=w,
                        projection_order="fixed_permutation", order_seed=3,
                        nonnegativity=False)


def _slab_worker(rank, world, port, outdir, variant="base"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "oracle"))
    import torch.distributed as dist
    import oracle as orc
    from paper_2005_11976_b200 import distributed as PD
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P, geom, grid, truth = _slab_problem(variant)
    images = np.stack([orc.forward(truth, grid, geom, i)[0] for i in range(geom.n_proj)])
    ps = P.ProjectionSet(geom, images)
    cfg = _slab_cfg(P, grid, variant)
    eng = OracleEngine(orc, ps, grid, cfg)
    run = PD.SlabSartRun(ps, grid, cfg, engine=eng, poison=True)
    vol, rep = run.run()
    st = run.plan.stats()
    np.savez(Path(outdir) / f"slab{rank}.npz", mu=run.mu.numpy(), res=rep.residuals,
             marched=np.array(eng.marched), updated=np.array(eng.updated),
             n_sub=len(run.subsets), need=np.array(st["mu_need_layers"]),
             sends=len(run.mu_sends))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,variant", [(2, "base"), (3, "base"), (4, "thin")])
def test_slab_decomposed_os_sart_matches_single_process(oracle, tmp_path, world, variant):
    """Slab decomposition with every unowned value poisoned to NaN: each rank
    marches its row bands from its window of mu, back-projects into its slab
    from the correction rows it computed or received, and the gathered volume
    and the residuals equal the single-process OS-SART oracle; every detector
    row is corrected once per pass and every voxel updated once per subset."""
    import torch.multiprocessing as mp
    mp.start_processes(_slab_worker, args=(world, _free_port(), str(tmp_path), variant),
                       nprocs=world, start_method="spawn", join=True)
    P, geom, grid, truth = _slab_problem(variant)
    images = np.stack([oracle.forward(truth, grid, geom, i)[0] for i in range(geom.n_proj)])
    images = images.astype(np.float32)
    cfg = _slab_cfg(P, grid, variant)
    order = (np.random.default_rng(cfg.order_seed).permutation(geom.n_proj)
             if cfg.projection_order == "fixed_permutation" else None)
    mu_ref, res_ref = oracle.sart(images, grid, geom, relaxation=cfg.relaxation,
                                  n_iterations=2, n_subsets=cfg.n_subsets, order=order,
                                  weights=cfg.weights, nonneg=cfg.nonnegativity)
    rs = [np.load(tmp_path / f"slab{r}.npz") for r in range(world)]
    for r in rs:
        assert np.array_equal(rs[0]["mu"], r["mu"])
        assert np.abs(r["mu"] - mu_ref).max() <= 1e-12 * np.abs(mu_ref).max()
        assert np.allclose(r["res"], res_ref, rtol=1e-12)
        if variant == "base":     # locality: no rank needs the whole volume's layers
            assert r["need"].max() < grid.n_h
    rows = np.concatenate([r["marched"] for r in rs])
    keys = rows[:, 0] * geom.det_rows + rows[:, 1]
    counts = np.bincount(keys, minlength=geom.n_proj * geom.det_rows)
    # rows with no in-support ray are marched too (they are in some band)
    assert np.array_equal(counts, np.full(geom.n_proj * geom.det_rows, 2))
    upd = np.concatenate([r["updated"] for r in rs])
    assert upd[:, 1].sum() == int(np.prod(grid.shape)) * int(rs[0]["n_sub"]) * 2


def test_slab_plan_helpers():
    from paper_2005_11976_b200 import slab as S
    assert list(S.slab_bounds(10, 3)) == [0, 3, 6, 10]
    P, geom, grid, truth = _slab_problem()
    rows = geom.det_rows
    # the rows a slab's voxels project to: inside the detector, and growing
    # with the slab
    a = S.slab_rows_needed(grid, geom, 0, 0, 6, rows)
    b = S.slab_rows_needed(grid, geom, 0, 0, 12, rows)
    assert 0 <= a[0] < a[1] <= rows and b[0] <= a[0] and b[1] >= a[1]
    assert S.slab_rows_needed(grid, geom, 0, 5, 5, rows) == (0, 0)
    # a plan with synthetic cells: exchanges are symmetric between ranks
    n_views, world = 4, 3
    costs = np.ones((n_views, rows))
    cells = np.zeros((n_views, rows, 2), dtype=np.int64)
    cells[..., 0] = np.arange(rows)[None] * grid.n_h // rows
    cells[..., 1] = cells[..., 0] + 2
    plan = S.SlabPlan(world, grid.n_h, rows, 4, costs, cells,
                      lambda v, k0, k1: S.slab_rows_needed(grid, geom, v, k0, k1, rows))
    for me in range(world):
        sends, _ = plan.mu_exchange(me)
        for p, l0, l1 in sends:
            _, recvs = plan.mu_exchange(p)
            assert (me, l0, l1) in recvs
        cs, _ = plan.corr_exchange(range(n_views), me)
        for p, b, r0, r1 in cs:
            _, cr = plan.corr_exchange(range(n_views), p)
            assert (me, b, r0, r1) in cr
