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
    """CPU engine with GpuEngine's interface, computing with the fp64 oracle."""

    def __init__(self, orc, ps, grid, cfg):
        import torch
        self.torch, self.o = torch, orc
        self.ps, self.grid, self.cfg = ps, grid, cfg
        self.images = np.asarray(ps.images, dtype=np.float64)
        self.max_row = None

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

    def correction(self, mu, slots, n, corr):
        for b, i in enumerate(slots[:n]):
            c = self.o.correction(mu.numpy(), self.grid, self.ps.geom, int(i), self.images[i],
                                  max_row=self.max_row[int(i)])
            corr[b] = self.torch.from_numpy(c)

    def bp_partial(self, corr, slots, n, num, den):
        num.zero_()
        if den is None:               # num-only partial (den precomputed per subset)
            den = self.torch.zeros_like(num)
        den.zero_()
        out = (num.numpy(), den.numpy())
        for b, i in enumerate(slots[:n]):
            self.o.back(corr[b].numpy(), self.ps.geom, int(i), self.grid, out=out)

    def update(self, num_c, den_c, offset, count, mu):
        w = None
        if self.cfg.weights is not None:
            w = np.asarray(self.cfg.weights, dtype=np.float64).ravel()[offset:offset + count]
        self.o._apply_update(mu.view(-1)[offset:offset + count].numpy(),
                             num_c[:count].numpy(), den_c[:count].numpy(), w,
                             self.cfg.relaxation, self.cfg.nonnegativity)

    def residual(self, mu, slots, n, accum):
        tot = 0.0
        for i in slots[:n]:
            sim, _ = self.o.forward(mu.numpy(), self.grid, self.ps.geom, int(i))
            tot += float(np.sum((self.images[int(i)] - sim) ** 2))
        accum += tot


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
    run = PD.ShardedSartRun(ps, grid, cfg, engine=OracleEngine(orc, ps, grid, cfg))
    vol, rep = run.run()
    np.savez(Path(outdir) / f"rank{rank}.npz", mu=run.mu.numpy(), res=rep.residuals,
             views=np.concatenate([v for v in run.local]) if run.local else np.zeros(0))
    dist.destroy_process_group()


def test_angle_sharded_os_sart_matches_single_process(oracle, tmp_path):
    import torch.multiprocessing as mp
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       start_method="spawn", join=True)
    P, geom, grid, truth, weights = _problem()
    images = np.stack([oracle.forward(truth, grid, geom, i)[0] for i in range(geom.n_proj)])
    images = images.astype(np.float32)
    order = np.random.default_rng(1).permutation(geom.n_proj)
    mu_ref, res_ref = oracle.sart(images, grid, geom, relaxation=0.4, n_iterations=2,
                                  order=order, weights=weights, n_subsets=3)
    r0 = np.load(tmp_path / "rank0.npz")
    r1 = np.load(tmp_path / "rank1.npz")
    assert np.array_equal(r0["mu"], r1["mu"])            # replicas stay identical
    assert np.abs(r0["mu"] - mu_ref).max() <= 1e-12 * np.abs(mu_ref).max()
    assert np.allclose(r0["res"], res_ref, rtol=1e-12)
    # every view processed exactly once per pass across the ranks
    views = np.sort(np.concatenate([r0["views"], r1["views"]]))
    assert np.array_equal(views, np.arange(geom.n_proj))


def test_shard_helpers():
    from paper_2005_11976_b200 import distributed as PD
    subset = np.array([7, 3, 9, 1, 5])
    parts = [PD.shard_views(subset, r, 3) for r in range(3)]
    assert sorted(np.concatenate(parts).tolist()) == sorted(subset.tolist())
    n = 1001
    ranges = [PD.shard_range(n, r, 4) for r in range(4)]
    covered = sum(c for _, c, _ in ranges)
    assert covered == n and ranges[0][0] == 0 and ranges[-1][0] + ranges[-1][1] == n
    assert PD.assign_objects(10, 1, 4) == [1, 5, 9]
