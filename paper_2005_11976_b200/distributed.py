"""Multi-GPU OS-SART: every subset's rays and voxels sharded across ranks, and object batches.

One process per GPU (``torch.distributed``, NCCL over NVLink/NVSwitch).  The
reference is single-process; the sharding follows the
north_star and SURVEY.md §8e, with the exchange chosen to move the fewest
bytes:

* **angle sharding, slab decomposition** (the default, :mod:`slab`): each
  rank owns a slab of mu's layers and a detector-row band of every view,
  packs only its FP window and exchanges by NCCL P2P only the correction
  rows and mu layers other ranks need (or stores them into their replicas
  from the kernels, CT_FUSED_COMM=1);
* **angle sharding, flattened-row split** (:class:`ShardedSartRun`) --
  within OS-SART subset s (n views of H x W pixels)
  the subset's rays are split by flattened detector row f = b*H + row into G
  contiguous ranges at FP block tiles (ct_fp_row_tile), balanced by the
  rows' in-support sample counts (ct_row_samples_*), so each rank marches
  ~1/G of the subset's samples on the same mu.  The corrections are
  all-gathered (n*H*W floats: 45 MiB at C2, against 128 MiB for a
  reduce-scatter of num), then every rank back-projects ALL the subset's
  views onto its own 1/G voxel shard with the fused SART update
  (ct_bp_*_update_range: num and den never leave the kernel, nothing to
  reduce), and mu is all-gathered.  Every correction and every voxel update
  is computed by exactly one rank with the single-GPU arithmetic, so mu is
  bit-identical to the 1-GPU run for any G.
* **residual** -- deferred like recon.SartRun: pass k marches the other
  subsets' views (row-split across ranks) and pass k+1's first correction FP
  adds the first subset's partials; the partials sit at fixed (view, block)
  slots and each slot is written by one rank (row ranges are tile-aligned),
  so an all-reduce of the slot scratch (x + 0 + ... = x) and one fixed-order
  sum give the single-GPU residual bit for bit.
* **object sharding** -- independent objects (config C5 batches) are
  assigned round-robin, no collective on the data path; composed with angle
  sharding as G = G_obj x G_ang (:class:`BatchPlan`,
  :func:`reconstruct_batch`).

The compute engine is injectable so the host logic (row / voxel
partitioning, collective sequence, residual slots) is testable on CPU with
the gloo backend and the oracle (tests/test_distributed.py); the production
engine is :class:`GpuEngine` over the sm_100a kernels.
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


def shard_range(n: int, rank: int, world: int):
    """Voxel range [offset, offset+count) updated by `rank` (chunk = ceil(n/world))."""
    chunk = -(-n // world)
    off = min(rank * chunk, n)
    return off, max(0, min(chunk, n - off)), chunk


def row_bounds(n_views: int, rows: int, world: int, tile: int, cost=None) -> np.ndarray:
    """Split the flattened rows [0, n_views*rows) of a view batch into `world`
    contiguous ranges at FP block-tile boundaries (v*rows + z*tile, and view
    ends), each boundary the tile boundary whose cumulative cost is nearest
    to r/world of the total (cost: one weight per flattened row, default
    uniform).  Returns world+1 non-decreasing bounds; rank r owns
    [b[r], b[r+1])."""
    total = n_views * rows
    n_tiles = -(-rows // tile)
    starts = (np.arange(n_views)[:, None] * rows
              + np.minimum(np.arange(n_tiles)[None, :] * tile, rows)).ravel()
    cand = np.unique(np.append(starts, total))
    if cost is None:
        cum = cand.astype(np.float64)
    else:
        c = np.concatenate([[0.0], np.cumsum(np.asarray(cost, dtype=np.float64))])
        cum = c[cand]
    b = [0]
    for r in range(1, world):
        t = r * cum[-1] / world
        i = int(np.searchsorted(cum, t))
        lo, hi = max(i - 1, 0), min(i, len(cand) - 1)
        pick = cand[lo] if (t - cum[lo]) <= (cum[hi] - t) else cand[hi]
        b.append(max(int(pick), b[-1]))
    b.append(total)
    return np.asarray(b, dtype=np.int64)


def _all_gather(full, my_chunk, group=None):
    dist = _dist()
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(full, my_chunk, group=group)
    else:
        world = dist.get_world_size(group)
        parts = list(full.view(world, -1).unbind(0))
        dist.all_gather(parts, my_chunk.clone(), group=group)


class GpuEngine:
    """Sharded OS-SART compute on one GPU (over recon.SartEngine's launchers)."""

    def __init__(self, ps: ProjectionSet, grid, cfg: SartConfig):
        from . import _device as D
        from .recon import SartEngine, _device_weights
        self.D = D
        self.eng = SartEngine(grid, ps.geom, cfg.sampling)
        self.device = self.eng.device
        self.ps = ps
        self.p_meas = None          # upload_rows(): only the rows this rank marches
        self._row_samples = None
        self.weights = _device_weights(cfg, grid.shape, self.device)
        self.cfg = cfg
        self.gather = self.eng.alloc_gather()
        self.quads = None
        self._upd = None

    def tensor(self, shape, dtype="float32"):
        torch = self.D.torch_mod()
        return torch.zeros(shape, dtype=getattr(torch, dtype), device=self.device)

    def prepare(self, order):
        self.eng.prepare_thresholds(order_slots=order)

    def slots(self, views):
        return self.D.upload_i32(views)

    def row_tile(self) -> int:
        return self.eng.row_tile()

    def row_costs(self, views):
        """FP cost per flattened detector row of a view batch: its in-support
        samples plus a per-ray setup allowance (~8 samples per pixel).  One
        count launch for all views, cached."""
        if self._row_samples is None:
            self._row_samples = self.eng.row_samples(np.arange(self.ps.geom.n_proj))
        return (self._row_samples[np.asarray(views)].ravel().astype(np.float64)
                + 8.0 * self.eng.cols)

    def upload_rows(self, ranges):
        """Measured projections to the device, only the (view, row range)
        pieces this rank's FP launches read (the kernels index p_meas by
        global view and row; other rows are never read).  ranges=None: all."""
        D, torch = self.D, self.D.torch_mod()
        imgs = self.ps.images
        if D.is_device_array(imgs) or ranges is None:
            self.p_meas = D.to_device(imgs, device=self.device)
            return
        host = torch.from_numpy(np.ascontiguousarray(imgs, dtype=np.float32))
        self.p_meas = torch.empty(tuple(host.shape), dtype=torch.float32, device=self.device)
        for v, r0, r1 in ranges:
            self.p_meas[v, r0:r1].copy_(host[v, r0:r1], non_blocking=True)

    def scratch(self, n_slots: int):
        torch = self.D.torch_mod()
        s = self.eng.residual_scratch(n_slots)
        return torch.zeros_like(s)

    def pack(self, mu) -> None:
        self.eng.pack(mu, self.gather)

    def correction_rows(self, mu, slots, n, out, lo, hi, n_slots, scratch, peers=None):
        """peers = (device pointer array, count, element offset): fused
        all-gather by peer stores."""
        pp, npeer, off = peers if peers else (None, 0, 0)
        self.eng.correction_rows(mu, self.p_meas, slots, n, out, lo, hi, n_slots, scratch,
                                 self.gather, pp, npeer, off)

    def residual_rows(self, mu, slots, n, lo, hi, n_slots, scratch):
        self.eng.residual_rows(mu, self.p_meas, slots, n, n_slots, scratch, lo, hi, self.gather)

    def residual_sum(self, scratch, acc):
        self.eng.residual_sum(scratch, acc)

    def bp_update_range(self, corr, slots, n, offset, count, mu, peers=None):
        if self.quads is None or self.quads.numel() < 4 * corr[:n].numel():
            self.quads = self.eng.alloc_quads(n)
        if self._upd is None:
            self._upd = make_update(mu, self.weights, self.cfg)
            if peers:
                self._upd.mu_peers, self._upd.n_peers = int(peers[0]), int(peers[1])
                if len(peers) > 2 and peers[2] is not None:      # per-replica voxel ranges
                    self._upd_ranges = peers[2]
                    self._upd.peer_ranges = peers[2].data_ptr()
        self.eng.pack_quads(corr, n, self.quads)
        self.eng.bp_update_range(corr, slots, n, self._upd, offset, count, self.quads)

    def synchronize(self):
        self.D.torch_mod().cuda.synchronize(self.device)

    # -- slab decomposition (slab.SlabSartRun) -----------------------------------
    def row_cells(self, views):
        return self.eng.row_cells(views)

    def pack_layers(self, mu, kc_lo, kc_hi) -> None:
        self.eng.pack_layers(mu, self.gather, kc_lo, kc_hi)

    def upload_bands(self, bands):
        return self.D.upload_i32(np.ascontiguousarray(bands).reshape(-1))

    def correction_bands(self, mu, slots, n, corr, bands, band_rows, n_slots, scratch,
                         peers=None):
        pp, npeer, rows = peers if peers else (None, 0, None)
        self.eng.correction_bands(mu, self.p_meas, slots, n, corr, bands, band_rows, n_slots,
                                  scratch, self.gather, pp, npeer, rows)

    def residual_bands(self, mu, slots, n, bands, band_rows, n_slots, scratch):
        self.eng.residual_bands(mu, self.p_meas, slots, n, bands, band_rows, n_slots, scratch,
                                self.gather)

    def poison_gather(self):
        if self.gather is not None:
            self.gather.fill_(float("nan"))


class _RowShard:
    """This rank's flattened-row range of a view batch and the launch it needs."""

    def __init__(self, views, rows, rank, world, tile, engine):
        self.views = np.asarray(views)
        self.n = len(self.views)
        cost = engine.row_costs(self.views) if (world > 1 and self.n) else None
        self.bounds = row_bounds(self.n, rows, world, tile, cost)
        self.lo, self.hi = int(self.bounds[rank]), int(self.bounds[rank + 1])
        self.sizes = np.diff(self.bounds)
        self.chunk = int(self.sizes.max()) if self.n else 0
        self.equal = bool(np.all(self.sizes == self.chunk))
        if self.hi > self.lo:
            v0, v1 = self.lo // rows, (self.hi - 1) // rows
            self.slots = engine.slots(self.views[v0:v1 + 1])     # the views the range spans
            self.nb = v1 - v0 + 1
            self.rlo, self.rhi = self.lo - v0 * rows, self.hi - v0 * rows
        else:
            self.slots, self.nb = None, 0


class ShardedSartRun:
    """OS-SART with every subset's rays and voxels sharded over the ranks of `group`."""

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
        # fused communication (opt-in, CT_FUSED_COMM=1, NCCL groups): the
        # correction stack and mu live in symmetric memory; the FP stores its
        # corrections and the update its voxels straight into every rank's
        # copy over NVLink, and a symmetric-memory barrier replaces each
        # all-gather
        self.fused = (os.environ.get("CT_FUSED_COMM", "0") == "1" and engine is None
                      and dist.get_backend(group) == "nccl")
        self._symm = None
        # mu lives in a padded flat buffer so all-gather chunks are equal-sized
        self.mu_flat = self._symm_tensor(pad) if self.fused else self.e.tensor(pad)
        self.mu = self.mu_flat[:n].view(grid.shape)
        init = _initial_mu(grid, cfg, self.mu.device) if cfg.initial is not None else None
        if init is not None:
            self.mu.copy_(init.to(self.mu.device))
        self.order = projection_order(cfg, ps.geom.n_proj)
        self.subsets = make_subsets(self.order, cfg.n_subsets)
        self.e.prepare(self.order)
        rows, cols = ps.geom.det_rows, ps.geom.det_cols
        self.rows, self.cols = rows, cols
        tile = self.e.row_tile()
        self.shards = [_RowShard(s, rows, self.rank, self.world, tile, self.e)
                       for s in self.subsets]
        self.subset_slots = [self.e.slots(s) for s in self.subsets]
        nmax = max(len(s) for s in self.subsets)
        cmax = max(sh.chunk for sh in self.shards)
        self.corr_all = (self._symm_tensor(self.world * cmax * cols) if self.fused
                         else self.e.tensor(self.world * cmax * cols))  # gather target
        if self.fused:
            self._h_corr = self._rendezvous(self.corr_all)
            self._h_mu = self._rendezvous(self.mu_flat)
        self.corr = self.e.tensor((nmax, rows, cols))                 # compacted stack
        n_proj = ps.geom.n_proj
        rest = np.setdiff1d(np.arange(n_proj), self.subsets[0])
        self.rest = _RowShard(rest, rows, self.rank, self.world, tile, self.e) \
            if len(rest) else None
        if hasattr(self.e, "upload_rows"):
            self.e.upload_rows(None if self.world == 1 else self._my_rows())
        self.scratch = self.e.scratch(n_proj)       # this rank's residual slot partials
        self.red = self.e.scratch(n_proj)           # their all-reduced copy
        self.resid = self.e.tensor(cfg.n_iterations, "float64")
        self.acc = self.e.tensor(1, "float64")
        self.passes_done = 0
        self._pending = None
        self._packed = False
        self.launch_log = None
        if self.fused:
            # every rank's replica setup (zero fill, initial mu) must be done
            # before any rank's first peer store lands in it: device barriers
            # on the compute stream, after the queued initialisation
            self._h_corr.barrier()
            self._h_mu.barrier()
            if self.world > 1:
                import warnings
                warnings.warn("CT_FUSED_COMM=1 with more than one rank: the peer-store "
                              "path is verified bit-identical on 1-rank groups only",
                              RuntimeWarning, stacklevel=2)

    def _symm_tensor(self, n):
        import torch
        import torch.distributed._symmetric_memory as symm_mem
        t = symm_mem.empty(n, dtype=torch.float32, device=self.e.device)
        t.zero_()
        return t

    def _rendezvous(self, t):
        import torch.distributed._symmetric_memory as symm_mem
        g = self.group if self.group is not None else _dist().group.WORLD
        return symm_mem.rendezvous(t, g)

    def _my_rows(self):
        """(view, row0, row1) pieces of the detector this rank's FPs read."""
        out = []
        for sh in self.shards + ([self.rest] if self.rest is not None else []):
            for f0 in range(sh.lo - sh.lo % self.rows, sh.hi, self.rows):
                a, b = max(f0, sh.lo), min(f0 + self.rows, sh.hi)
                if b > a:
                    out.append((int(sh.views[f0 // self.rows]), a - f0, b - f0))
        return out

    def fp_rows(self, s: int) -> list:
        """(view, fraction of its rows) this rank marches in FP launch s
        (subset s >= 0; -1: the residual's other views; -2: subset 0)."""
        sh = self.shards[s] if s >= 0 else (self.rest if s == -1 else self.shards[0])
        out = []
        for b, v in enumerate(sh.views):
            ov = min(sh.hi, (b + 1) * self.rows) - max(sh.lo, b * self.rows)
            if ov > 0:
                out.append((int(v), ov / self.rows))
        return out

    def exchange_bytes(self, kind: str, s: int) -> float:
        """Bytes this rank receives in collective `kind` of subset s."""
        if kind == "all_gather":
            return 4.0 * self.nvox * (self.world - 1) / self.world
        if kind == "all_gather_corr":
            return 4.0 * self.rows * self.cols * len(self.subsets[s]) * (self.world - 1) / self.world
        return 0.0

    # views of subset s this rank marches (tests / accounting)
    @property
    def local(self):
        return [sh.views[sh.lo // self.rows:(sh.hi - 1) // self.rows + 1] if sh.hi > sh.lo
                else sh.views[:0] for sh in self.shards]

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

    def _pack(self, s):
        if not self._packed:
            self._timed("pack_gather", s, self.e.pack, self.mu)
        self._packed = True

    def _finish_residual(self):
        """All-reduce the slot partials (one owner per slot) and sum them."""
        self.red.copy_(self.scratch)
        self._timed("all_reduce_resid", -1, _dist().all_reduce, self.red, _dist().ReduceOp.SUM,
                    self.group)
        self.acc.zero_()
        self.e.residual_sum(self.red, self.acc)
        k = min(self._pending, self.resid.numel() - 1)
        self.resid[k:k + 1].copy_(self.acc)
        self._pending = None

    def run_subset(self, s: int) -> None:
        sh = self.shards[s]
        cols = self.cols
        n_proj = self.ps.geom.n_proj
        self._pack(s)
        mine = self.corr_all[self.rank * sh.chunk * cols:(self.rank + 1) * sh.chunk * cols]
        fused = s == 0 and self._pending is not None
        peers = ((self._h_corr.buffer_ptrs_dev, self.world, self.rank * sh.chunk * cols),
                 ) if self.fused else ()
        if sh.nb:
            if fused:
                self._timed("fp_correction_resid", s, self.e.correction_rows, self.mu,
                            sh.slots, sh.nb, mine, sh.rlo, sh.rhi, n_proj, self.scratch, *peers)
            else:
                self._timed("fp_correction", s, self.e.correction_rows, self.mu, sh.slots,
                            sh.nb, mine, sh.rlo, sh.rhi, 0, None, *peers)
        if fused:
            self._finish_residual()
        full = self.corr_all[:self.world * sh.chunk * cols]
        if self.fused:            # every rank's stores into every copy are done
            self._timed("barrier_corr", s, self._h_corr.barrier)
        else:
            self._timed("all_gather_corr", s, _all_gather, full, mine, self.group)
        npix_rows = sh.n * self.rows
        if sh.equal and self.world * sh.chunk == npix_rows:
            stack = full.view(-1)[:npix_rows * cols].view(sh.n, self.rows, cols)
        else:                     # uneven chunks: compact into the [n][H][W] stack
            flat = self.corr.view(-1)
            for r in range(self.world):
                a, b = int(sh.bounds[r]), int(sh.bounds[r + 1])
                if b > a:
                    flat[a * cols:b * cols].copy_(full[r * sh.chunk * cols:
                                                       (r * sh.chunk + b - a) * cols])
            stack = self.corr[:sh.n]
        mu_peers = ((self._h_mu.buffer_ptrs_dev, self.world),) if self.fused else ()
        if self.count:
            self._timed("bp_update", s, self.e.bp_update_range, stack, self.subset_slots[s],
                        sh.n, self.offset, self.count, self.mu, *mu_peers)
        if self.fused:            # every rank's shard is in every replica
            self._timed("barrier_mu", s, self._h_mu.barrier)
        else:
            self._timed("all_gather", s, _all_gather, self.mu_flat,
                        self.mu_flat[self.rank * self.chunk:(self.rank + 1) * self.chunk],
                        self.group)
        self._packed = False

    def run_pass(self, residual: bool | None = None) -> None:
        want = self.cfg.compute_residuals if residual is None else residual
        if not want:
            self.finalize()
        for s in range(len(self.subsets)):
            self.run_subset(s)
        if want:
            if self.rest is not None and self.rest.nb:
                self._pack(-1)
                self._timed("fp_residual", -1, self.e.residual_rows, self.mu, self.rest.slots,
                            self.rest.nb, self.rest.rlo, self.rest.rhi, self.ps.geom.n_proj,
                            self.scratch)
            self._pending = self.passes_done
        self.passes_done += 1

    def finalize(self) -> None:
        """Complete a deferred residual: the first subset's rows on the current mu."""
        if self._pending is None:
            return
        sh = self.shards[0]
        if sh.nb:
            self._pack(-2)
            self._timed("fp_residual", -2, self.e.residual_rows, self.mu, sh.slots, sh.nb,
                        sh.rlo, sh.rhi, self.ps.geom.n_proj, self.scratch)
        self._finish_residual()

    def run(self):
        t0 = time.perf_counter()
        for _ in range(self.cfg.n_iterations):
            self.run_pass()
        self.finalize()
        if hasattr(self.e, "synchronize"):
            self.e.synchronize()
        wall = time.perf_counter() - t0
        res = ([math.sqrt(float(x)) for x in self.resid.cpu().numpy()]
               if self.cfg.compute_residuals else [])
        if self.ps.on_device:
            mu = self.mu
        else:
            from . import _device as D
            mu = D.to_host(self.mu, pinned=True) if self.mu.is_cuda else self.mu.numpy()
        return (_volume_cls(self.grid)._trusted(self.grid, mu),
                ReconReport(residuals=res, wall_time=wall, config=_config_echo(self.cfg)))


def sart_run_sharded(ps: ProjectionSet, grid, cfg: SartConfig | None = None, group=None,
                     decomposition: str = "slab"):
    """Angle-sharded (OS-)SART over the ranks of `group` (default: world).

    decomposition "slab" (default): volume layers and per-view detector-row
    bands per rank, halo exchanges (slab.SlabSartRun); "rows": flattened-row
    split with all-gathers of the corrections and of mu (ShardedSartRun, the
    one with the opt-in fused NVLink peer stores).  Both are bit-identical to
    one GPU."""
    cfg = cfg or SartConfig()
    if decomposition == "slab":
        from .slab import SlabSartRun
        return SlabSartRun(ps, grid, cfg, group).run()
    if decomposition == "rows":
        return ShardedSartRun(ps, grid, cfg, group).run()
    raise ConfigError(f"unknown decomposition {decomposition!r}")


def assign_objects(n_objects: int, rank: int, world: int):
    """Object indices reconstructed by `rank` (round-robin)."""
    return list(range(rank, n_objects, world))


class BatchPlan:
    """G = G_obj x G_ang decomposition of the ranks for an object batch
    (config C5): ranks [g*G_ang, (g+1)*G_ang) form object group
    g; objects go round-robin to the G_obj groups (no collective between
    groups), and each object's OS-SART subsets are angle-sharded over the
    G_ang ranks of its group (ShardedSartRun).  G_ang = 1 is pure object
    sharding, G_ang = G pure angle sharding."""

    def __init__(self, rank: int, world: int, g_ang: int = 1):
        if g_ang < 1 or world % g_ang:
            raise ConfigError(f"angle-group size {g_ang} does not divide {world} ranks")
        self.rank, self.world, self.g_ang = int(rank), int(world), int(g_ang)
        self.n_groups = self.world // self.g_ang
        self.group_index = self.rank // self.g_ang
        self.group_rank = self.rank % self.g_ang

    def group_ranks(self, g: int) -> list:
        return list(range(g * self.g_ang, (g + 1) * self.g_ang))

    def objects(self, n_objects: int) -> list:
        """This rank's objects (every rank of a group gets the group's)."""
        return assign_objects(n_objects, self.group_index, self.n_groups)

    def make_group(self):
        """This rank's object group as a process group (collective: every rank
        creates every group, in order).  None for G_ang = 1 (no exchange)."""
        if self.g_ang == 1:
            return None
        dist = _dist()
        mine = None
        for g in range(self.n_groups):
            pg = dist.new_group(self.group_ranks(g))
            if g == self.group_index:
                mine = pg
        return mine


def _default_runner(ps, grid, cfg, group):
    if group is None:
        from .recon import SartRun
        return SartRun(ps, grid, cfg).run()
    from .slab import SlabSartRun
    return SlabSartRun(ps, grid, cfg, group).run()


def reconstruct_batch(items, cfg: SartConfig, rank: int | None = None,
                      world: int | None = None, g_ang: int = 1, runner=None, group=None):
    """Batch reconstruction over G = G_obj x G_ang ranks (BatchPlan).

    items: sequence of (ProjectionSet, grid[, SartConfig]) for every object.
    Objects are independent (no data-path collective between object groups);
    with g_ang > 1 each object's subsets are angle-sharded over its group.
    Returns {index: (volume, report)} for this rank's objects (every rank of
    an object group holds the group's results).  runner(ps, grid, cfg,
    group) overrides the per-object driver (tests: an oracle engine); group
    is this rank's object group if the caller already made it
    (BatchPlan.make_group), else it is created here (collective).
    """
    if rank is None or world is None:
        dist = _dist()
        on = dist.is_available() and dist.is_initialized()
        rank = dist.get_rank() if on else 0
        world = dist.get_world_size() if on else 1
    plan = BatchPlan(rank, world, g_ang)
    if group is None:
        group = plan.make_group()
    run = runner or _default_runner
    out = {}
    for idx in plan.objects(len(items)):
        it = items[idx]
        c = it[2] if len(it) > 2 else cfg
        out[idx] = run(it[0], it[1], c, group)
    return out


# slab decomposition of the angle-sharded run (defined in slab.py)
from .slab import SlabPlan, SlabSartRun, sart_run_slab  # noqa: E402,F401
