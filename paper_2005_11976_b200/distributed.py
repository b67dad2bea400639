"""Multi-GPU OS-SART: views of every subset sharded across ranks, and object batches.

One process per GPU (``torch.distributed``, NCCL over NVLink/NVSwitch).  The
reference is single-process; the sharding follows the
north_star and SURVEY.md §8e:

* **angle sharding** -- within OS-SART subset s, rank r projects and
  back-projects the views subset[r::G] on the same mu (views of a subset are
  independent given mu) and writes its partial num; the one real exchange
  step runs: reduce-scatter(num) -> the fused update on the rank's voxel
  shard -> all-gather(mu).  den is mu-independent -- the BP weights of the
  in-bounds taps are pure geometry (cyltomo/_kernels.py:365-376) -- so each
  subset's den shard is computed and reduce-scattered ONCE at setup
   and only num moves per subset.  Every rank ends the subset
  with the same mu (the gather broadcasts one owner's values).  The residual
  is an all-reduce of one fp64 per pass.
* **object sharding** -- independent objects (config C5 batches) are
  assigned round-robin, no collective on the data path
  (:func:`reconstruct_batch`).

The compute engine is injectable so the host logic (partitioning, collective
sequence, update offsets) is testable on CPU with the gloo backend and the
oracle (tests/test_distributed.py); the production engine is
:class:`GpuEngine` over the sm_100a kernels.
"""

from __future__ import annotations

import math
import os
import time

import numpy as np

from .errors import ConfigError
from .projector import LINE_INTEGRAL, ProjectionSet
from .recon import (ReconReport, SartConfig, _config_echo, _initial_mu, _volume_cls,
                    make_subsets, make_update, projection_order)


def _dist():
    import torch.distributed as dist
    return dist


def init_from_env(backend: str | None = None):
    """Initialise the default group from torchrun's env; returns (rank, world, local_rank)."""
    import torch
    dist = _dist()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def shard_views(subset, rank: int, world: int):
    """Views of one subset owned by `rank` (round-robin: subset[rank::world])."""
    return np.asarray(subset)[rank::world]


def shard_range(n: int, rank: int, world: int):
    """Voxel range [offset, offset+count) updated by `rank` (chunk = ceil(n/world))."""
    chunk = -(-n // world)
    off = min(rank * chunk, n)
    return off, max(0, min(chunk, n - off)), chunk


def _reduce_scatter(full, out_chunk, group=None):
    """Sum `full` ([world*chunk]) over ranks, keep this rank's chunk."""
    dist = _dist()
    if dist.get_backend(group) == "nccl":
        dist.reduce_scatter_tensor(out_chunk, full, group=group)
    else:  # gloo: no reduce-scatter -- all-reduce then slice (same result)
        dist.all_reduce(full, group=group)
        r = dist.get_rank(group)
        c = out_chunk.numel()
        out_chunk.copy_(full[r * c:(r + 1) * c])


def _all_gather(full, my_chunk, group=None):
    dist = _dist()
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(full, my_chunk, group=group)
    else:
        world = dist.get_world_size(group)
        parts = list(full.view(world, -1).unbind(0))
        dist.all_gather(parts, my_chunk.clone(), group=group)


class GpuEngine:
    """Angle-sharded OS-SART compute on one GPU (wraps recon.SartEngine)."""

    def __init__(self, ps: ProjectionSet, grid, cfg: SartConfig):
        from . import _device as D
        from .recon import SartEngine, _device_weights
        self.D = D
        self.eng = SartEngine(grid, ps.geom, cfg.sampling)
        self.device = self.eng.device
        self.p_meas = D.to_device(ps.images, device=self.device)
        self.weights = _device_weights(cfg, grid.shape, self.device)
        self.cfg = cfg
        self.gather = None
        self.quads = None

    def tensor(self, shape, dtype="float32"):
        torch = self.D.torch_mod()
        return torch.zeros(shape, dtype=getattr(torch, dtype), device=self.device)

    def prepare(self, order):
        self.eng.prepare_thresholds(order_slots=order)

    def slots(self, views):
        return self.D.upload_i32(views)

    def correction(self, mu, slots, n, corr):
        if self.gather is None:
            self.gather = self.eng.alloc_gather()
        self.eng.pack(mu, self.gather)
        self.eng.correction(mu, self.p_meas, slots, n, corr, self.gather)

    def bp_partial(self, corr, slots, n, num, den):
        if self.quads is None:
            self.quads = self.eng.alloc_quads(corr.shape[0])
        self.eng.pack_quads(corr, n, self.quads)
        self.eng.bp_partial(corr, slots, n, num, den, self.quads)

    def update(self, num_c, den_c, offset, count, mu):
        from . import _native as N
        import ctypes as C
        upd = make_update(mu, self.weights, self.cfg)
        N.call("ct_sart_update", self.D.ptr(num_c), self.D.ptr(den_c), offset, count,
               C.byref(upd), self.D.stream_handle())

    def residual(self, mu, slots, n, accum):
        if self.gather is None:
            self.gather = self.eng.alloc_gather()
        self.eng.pack(mu, self.gather)
        self.eng.residual(mu, self.p_meas, slots, n, accum, self.gather)

    def synchronize(self):
        self.D.torch_mod().cuda.synchronize(self.device)


class ShardedSartRun:
    """OS-SART with every subset's views sharded over the ranks of `group`."""

    def __init__(self, ps: ProjectionSet, grid, cfg: SartConfig, group=None, engine=None):
        if ps.kind != LINE_INTEGRAL:
            raise ConfigError("SART needs line-integral projections")
        dist = _dist()
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.ps, self.grid, self.cfg = ps, grid, cfg
        self.e = engine if engine is not None else GpuEngine(ps, grid, cfg)
        n = int(np.prod(grid.shape))
        self.nvox = n
        self.offset, self.count, self.chunk = shard_range(n, self.rank, self.world)
        pad = self.chunk * self.world
        # mu lives in a padded flat buffer so all-gather chunks are equal-sized
        self.mu_flat = self.e.tensor(pad)
        self.mu = self.mu_flat[:n].view(grid.shape)
        init = _initial_mu(grid, cfg, self.mu.device) if cfg.initial is not None else None
        if init is not None:
            self.mu.copy_(init.to(self.mu.device))
        self.order = projection_order(cfg, ps.geom.n_proj)
        self.subsets = make_subsets(self.order, cfg.n_subsets)
        self.e.prepare(self.order)
        self.local = [shard_views(s, self.rank, self.world) for s in self.subsets]
        self.local_slots = [self.e.slots(v) if len(v) else None for v in self.local]
        my_views = np.arange(ps.geom.n_proj)[self.rank::self.world]
        self.resid_views = my_views
        self.resid_slots = self.e.slots(my_views) if len(my_views) else None
        nmax = max(1, max(len(v) for v in self.local))
        self.corr = self.e.tensor((nmax, ps.geom.det_rows, ps.geom.det_cols))
        self.num = self.e.tensor(pad)
        self.num_c = self.e.tensor(self.chunk)
        self.den_c = self._subset_den(pad)
        self.resid = self.e.tensor(cfg.n_iterations, "float64")
        self.passes_done = 0
        self.launch_log = None

    def _subset_den(self, pad):
        """Per-subset den shards [n_subsets][chunk]: one partial BP (den only;
        the correction values do not enter den) and one reduce-scatter per
        subset, at setup."""
        den = self.e.tensor(pad)
        dv = den[:self.nvox].view(self.grid.shape)
        nv = self.num[:self.nvox].view(self.grid.shape)
        out = []
        for views, slots in zip(self.local, self.local_slots):
            if len(views):
                self.e.bp_partial(self.corr, slots, len(views), nv, dv)
            else:
                den.zero_()
            chunk = self.e.tensor(self.chunk)
            _reduce_scatter(den, chunk, self.group)
            out.append(chunk)
        return out

    def _timed(self, kind, s, fn, *args):
        """Run fn; with launch_log set (GPU engine), bracket it with CUDA events."""
        if self.launch_log is None:
            fn(*args)
            return
        import torch
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn(*args)
        b.record()
        self.launch_log.append((kind, s, a, b))

    def run_subset(self, s: int) -> None:
        views, slots = self.local[s], self.local_slots[s]
        nv = self.num[:self.nvox].view(self.grid.shape)
        if len(views):
            self._timed("fp_correction", s, self.e.correction, self.mu, slots, len(views),
                        self.corr)
            self._timed("bp_partial", s, self.e.bp_partial, self.corr, slots, len(views), nv,
                        None)
        else:
            self.num.zero_()
        self._timed("reduce_scatter", s, _reduce_scatter, self.num, self.num_c, self.group)
        if self.count:
            self._timed("update", s, self.e.update, self.num_c, self.den_c[s], self.offset,
                        self.count, self.mu)
        self._timed("all_gather", s, _all_gather, self.mu_flat,
                    self.mu_flat[self.rank * self.chunk:(self.rank + 1) * self.chunk],
                    self.group)

    def run_pass(self, residual: bool | None = None) -> None:
        for s in range(len(self.subsets)):
            self.run_subset(s)
        want = self.cfg.compute_residuals if residual is None else residual
        if want:
            k = min(self.passes_done, self.cfg.n_iterations - 1)
            acc = self.resid[k:k + 1]
            if self.resid_slots is not None:
                self._timed("fp_residual", -1, self.e.residual, self.mu, self.resid_slots,
                            len(self.resid_views), acc)
            _dist().all_reduce(acc, group=self.group)
        self.passes_done += 1

    def run(self):
        t0 = time.perf_counter()
        for _ in range(self.cfg.n_iterations):
            self.run_pass()
        if hasattr(self.e, "synchronize"):
            self.e.synchronize()
        wall = time.perf_counter() - t0
        res = ([math.sqrt(float(x)) for x in self.resid.cpu().numpy()]
               if self.cfg.compute_residuals else [])
        mu = self.mu if self.ps.on_device else self.mu.cpu().numpy()
        return (_volume_cls(self.grid)._trusted(self.grid, mu),
                ReconReport(residuals=res, wall_time=wall, config=_config_echo(self.cfg)))


def sart_run_sharded(ps: ProjectionSet, grid, cfg: SartConfig | None = None, group=None):
    """Angle-sharded (OS-)SART over the ranks of `group` (default: world)."""
    return ShardedSartRun(ps, grid, cfg or SartConfig(), group).run()


def assign_objects(n_objects: int, rank: int, world: int):
    """Object indices reconstructed by `rank` (round-robin)."""
    return list(range(rank, n_objects, world))


def reconstruct_batch(items, cfg: SartConfig, rank: int = 0, world: int = 1):
    """Object-sharded batch reconstruction (no data-path collective).

    items: sequence of (ProjectionSet, grid[, SartConfig]) for every object; the
    rank reconstructs its own objects and returns {index: (volume, report)}.
    """
    from .recon import SartRun
    out = {}
    for idx in assign_objects(len(items), rank, world):
        it = items[idx]
        c = it[2] if len(it) > 2 else cfg
        out[idx] = SartRun(it[0], it[1], c).run()
    return out
