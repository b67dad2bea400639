"""Slab decomposition of the angle-sharded OS-SART (distributed.SlabSartRun).

The flattened-row split of :class:`distributed.ShardedSartRun` lets every
rank march rays anywhere in the volume, so after each OS subset the whole
volume is all-gathered and every rank re-packs the whole gather layout
(DESIGN.md §6 measured both as the fixed per-rank cost that
caps the 8-rank efficiency).  Here the volume's layers (h, or z for a
Cartesian grid: the slowest axis of mu) are split into G slabs, and each
view's detector rows into G bands that project onto them:

* rank r owns mu layers [L_r, L_r+1) (equal counts: the BP update's cost)
  and marches band r of every view (tile-aligned rows, cut where the rows'
  cumulative in-support sample count crosses r/G of the view's: the FP's
  cost);
* the FP of band r reads only gather cells in a window of cell layers --
  the union of its rows' [min, max] cell layer (``ct_row_cells_*``, the
  march's own fp32 cell index, exact) -- so rank r packs only that window
  (``ct_pack_gather_*_layers``) and needs current mu only there;
* the BP update of slab r reads only the correction rows its voxels' bilinear
  footprints touch (the projected rims of the slab, ``slab_rows_needed``),
  so instead of all-gathering the corrections each rank receives, per view,
  the part of its neighbours' bands it needs; after the update each rank
  sends the layers of its slab that lie in other ranks' windows.

Every correction and voxel update is still computed by exactly one rank with
the single-GPU arithmetic and operands, so the volume is bit-identical to one
GPU (tests: gloo ranks over the oracle engine with the unowned data poisoned
to NaN, and the GPU engine's ranks on one B200).  Where the geometry gives no
locality (e.g. an axis lying across the detector rows) the windows grow to
the whole volume: still exact, only the savings vanish.
"""

from __future__ import annotations

import math
import os
import time

import numpy as np

from .errors import ConfigError
from .geometry import project_points
from .grid import CylGrid
from .projector import LINE_INTEGRAL
from .recon import (ReconReport, _config_echo, _initial_mu, _volume_cls, make_subsets,
                    projection_order)

I32_MAX = 2 ** 31 - 1


def _dist():
    import torch.distributed as dist
    return dist


def slab_bounds(n_layers: int, world: int) -> np.ndarray:
    """Layer bounds of the G slabs (equal counts to one layer)."""
    return np.asarray([(r * n_layers) // world for r in range(world + 1)], dtype=np.int64)


def slab_rows_needed(grid, geom, view: int, k_lo: int, k_hi: int, rows: int,
                     n_rim: int = 2048) -> tuple:
    """Detector rows [lo, hi) the BP footprints of the voxels of layers
    [k_lo, k_hi) read in `view`: the slab's voxel centres lie in a convex
    body (a cylinder section of the grid radius, or a box) whose extreme
    points are its rims / corners, and v is a linear-fractional function of
    the point, so its extremes over the slab are those of the rims (sampled
    at n_rim angles: 5e-5 mm chord error) -- plus the footprint's second row
    and one row of margin each side."""
    if k_hi <= k_lo:
        return 0, 0
    if isinstance(grid, CylGrid):
        hs = grid.h_centers()[[k_lo, k_hi - 1]]
        th = np.linspace(0.0, 2.0 * math.pi, n_rim, endpoint=False)
        ring = np.stack([grid.radius * np.cos(th), grid.radius * np.sin(th)], axis=-1)
        pts = np.concatenate([np.column_stack([ring, np.full(n_rim, h)]) for h in hs])
        world_pts = pts @ grid.rotation.T + np.asarray(grid.pose.t, dtype=float)
    else:
        vs, o = grid.voxel_size, grid.origin
        xs = o[0] + (np.array([0, grid.n_x - 1]) + 0.5) * vs
        ys = o[1] + (np.array([0, grid.n_y - 1]) + 0.5) * vs
        zs = o[2] + (np.array([k_lo, k_hi - 1]) + 0.5) * vs
        world_pts = np.array([[x, y, z] for x in xs for y in ys for z in zs])
    v = project_points(geom, view, world_pts)[:, 1]
    lo = int(math.floor(v.min())) - 1
    hi = int(math.floor(v.max())) + 3
    return max(lo, 0), min(max(hi, 0), rows)


class SlabPlan:
    """Static (geometry-only) partition of an OS-SART over G ranks.

    row_costs: (P, H) FP cost per view and row; row_cells: (P, H, 2) FP cell
    layers [min, max] per row (I32_MAX / -I32_MAX - 1 for rows without
    samples); need(view, k_lo, k_hi) -> rows [lo, hi) the BP of layers
    [k_lo, k_hi) reads.
    """

    def __init__(self, world: int, n_layers: int, rows: int, tile: int, row_costs,
                 row_cells, need, margin: int = 1):
        from .distributed import row_bounds
        row_costs = np.asarray(row_costs, dtype=np.float64)
        row_cells = np.asarray(row_cells)
        n_views = row_costs.shape[0]
        self.world, self.n_layers, self.rows = world, n_layers, rows
        self.L = slab_bounds(n_layers, world)
        self.bands = np.stack([row_bounds(1, rows, world, tile, row_costs[v])
                               for v in range(n_views)])                     # (P, G+1)
        self.win = np.zeros((world, 2), dtype=np.int64)     # FP cell layers, inclusive
        self.mu_need = np.zeros((world, 2), dtype=np.int64)  # mu layers, half-open
        for r in range(world):
            lo, hi = I32_MAX, -I32_MAX
            for v in range(n_views):
                a, b = int(self.bands[v, r]), int(self.bands[v, r + 1])
                if b <= a:
                    continue
                c = row_cells[v, a:b]
                ok = c[:, 0] <= c[:, 1]
                if ok.any():
                    lo = min(lo, int(c[ok, 0].min()))
                    hi = max(hi, int(c[ok, 1].max()))
            if lo > hi:
                self.win[r] = (0, -1)
                self.mu_need[r] = (0, 0)
            else:
                self.win[r] = (lo - margin, hi + margin)
                # FP cell layer kc reads mu layers kc - 1 and kc (clamped)
                m0 = min(max(lo - margin - 1, 0), n_layers - 1)
                m1 = min(max(hi + margin, 0), n_layers - 1) + 1
                self.mu_need[r] = (m0, m1)
        self.need = np.zeros((world, n_views, 2), dtype=np.int64)
        for r in range(world):
            for v in range(n_views):
                self.need[r, v] = need(v, int(self.L[r]), int(self.L[r + 1]))

    def band(self, v: int, r: int) -> tuple:
        return int(self.bands[v, r]), int(self.bands[v, r + 1])

    def corr_exchange(self, views, me: int):
        """(sends, recvs) for one subset's correction stack: lists of
        (peer, stack position b, row0, row1)."""
        sends, recvs = [], []
        for b, v in enumerate(views):
            v = int(v)
            a0, a1 = self.band(v, me)
            n0, n1 = (int(x) for x in self.need[me, v])
            for p in range(self.world):
                if p == me:
                    continue
                q0, q1 = (int(x) for x in self.need[p, v])
                lo, hi = max(a0, q0), min(a1, q1)
                if hi > lo:
                    sends.append((p, b, lo, hi))
                p0, p1 = self.band(v, p)
                lo, hi = max(p0, n0), min(p1, n1)
                if hi > lo:
                    recvs.append((p, b, lo, hi))
        return sends, recvs

    def mu_exchange(self, me: int):
        """(sends, recvs) of mu layers after a slab update: (peer, l0, l1)."""
        sends, recvs = [], []
        for p in range(self.world):
            if p == me:
                continue
            lo = max(int(self.L[me]), int(self.mu_need[p, 0]))
            hi = min(int(self.L[me + 1]), int(self.mu_need[p, 1]))
            if hi > lo:
                sends.append((p, lo, hi))
            lo = max(int(self.L[p]), int(self.mu_need[me, 0]))
            hi = min(int(self.L[p + 1]), int(self.mu_need[me, 1]))
            if hi > lo:
                recvs.append((p, lo, hi))
        return sends, recvs

    def stats(self) -> dict:
        """Per rank: window and mu layers it needs, against the slab."""
        return {"slabs": np.diff(self.L).tolist(),
                "window_layers": (self.win[:, 1] - self.win[:, 0] + 1).tolist(),
                "mu_need_layers": (self.mu_need[:, 1] - self.mu_need[:, 0]).tolist()}


def p2p_exchange(ops, group=None) -> None:
    """Batched point-to-point transfers: ops = [("send" | "recv", tensor,
    peer group rank)].  gloo groups with CUDA tensors are staged through host
    copies (tests run ranks sharing one GPU over gloo)."""
    if not ops:
        return
    import torch
    dist = _dist()
    stage = dist.get_backend(group) != "nccl" and any(t.is_cuda for _, t, _ in ops)
    p2p, back = [], []
    for kind, t, peer in ops:
        g = dist.get_global_rank(group, peer) if group is not None else peer
        buf = t
        if stage:
            if kind == "send":
                buf = t.cpu()
            else:
                buf = torch.empty(t.shape, dtype=t.dtype)
                back.append((t, buf))
        p2p.append(dist.P2POp(dist.isend if kind == "send" else dist.irecv, buf, g, group))
    for req in dist.batch_isend_irecv(p2p):
        req.wait()
    for t, buf in back:
        t.copy_(buf)


class _SubsetBands:
    """One view batch's slots, this rank's bands and its exchange lists."""

    def __init__(self, views, plan: SlabPlan, me: int, engine, exchange: bool):
        self.views = np.asarray(views)
        self.n = len(self.views)
        bands = np.array([plan.band(int(v), me) for v in self.views], dtype=np.int32)
        self.band_rows = int((bands[:, 1] - bands[:, 0]).max()) if self.n else 0
        self.slots = engine.slots(self.views)
        self.bands = engine.upload_bands(bands) if self.band_rows > 0 else None
        self.rows_marched = [(int(v), int(a), int(b)) for v, (a, b) in zip(self.views, bands)
                             if b > a]
        self.sends, self.recvs = plan.corr_exchange(self.views, me) if exchange else ([], [])


class SlabSartRun:
    """OS-SART with the volume's layers split into slabs over the ranks of
    `group` (see the module docstring).  poison=True (tests) keeps every
    value a rank must not read -- mu layers outside its slab and window, the
    gather buffer outside the packed window, correction rows it neither
    computed nor received -- at NaN, so a partition error cannot pass
    silently."""

    def __init__(self, ps, grid, cfg, group=None, engine=None, poison: bool = False):
        if ps.kind != LINE_INTEGRAL:
            raise ConfigError("SART needs line-integral projections")
        from .distributed import GpuEngine
        dist = _dist()
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.ps, self.grid, self.cfg = ps, grid, cfg
        self.poison = poison or os.environ.get("CT_SLAB_POISON", "0") == "1"
        self.e = engine if engine is not None else GpuEngine(ps, grid, cfg)
        shape = tuple(grid.shape)
        self.n_layers = shape[0]
        self.layer = int(shape[1] * shape[2])
        # fused exchanges (opt-in, CT_FUSED_COMM=1, NCCL groups): mu and the
        # correction stack live in symmetric memory; the FP epilogue stores
        # each correction into every rank whose BP needs its row and the BP
        # update each voxel into every rank whose FP window holds its layer
        # (NVLink peer stores), and device barriers replace the P2P exchanges
        self.fused = (os.environ.get("CT_FUSED_COMM", "0") == "1" and engine is None
                      and dist.get_backend(group) == "nccl")
        if self.fused:
            self.poison = False
            self.mu = self._symm_tensor(int(np.prod(shape))).view(shape)
        else:
            self.mu = self.e.tensor(shape)
        if cfg.initial is not None:
            self.mu.copy_(_initial_mu(grid, cfg, self.mu.device).to(self.mu.device))
        self.order = projection_order(cfg, ps.geom.n_proj)
        self.subsets = make_subsets(self.order, cfg.n_subsets)
        self.e.prepare(self.order)
        rows, cols = ps.geom.det_rows, ps.geom.det_cols
        self.rows, self.cols = rows, cols
        n_proj = ps.geom.n_proj
        allv = np.arange(n_proj)
        costs = np.asarray(self.e.row_costs(allv), dtype=np.float64).reshape(n_proj, rows)
        cells = self.e.row_cells(allv)
        self.plan = SlabPlan(self.world, self.n_layers, rows, self.e.row_tile(), costs, cells,
                             lambda v, a, b: slab_rows_needed(grid, ps.geom, v, a, b, rows))
        me = self.rank
        self.k0, self.k1 = int(self.plan.L[me]), int(self.plan.L[me + 1])
        self.win = tuple(int(x) for x in self.plan.win[me])
        multi = self.world > 1
        self.sub = [_SubsetBands(s, self.plan, me, self.e, multi) for s in self.subsets]
        rest = np.setdiff1d(allv, self.subsets[0])
        self.rest = _SubsetBands(rest, self.plan, me, self.e, False) if len(rest) else None
        self.mu_sends, self.mu_recvs = self.plan.mu_exchange(me) if multi else ([], [])
        pieces = [p for sb in self.sub for p in sb.rows_marched]
        if self.rest is not None:
            pieces += self.rest.rows_marched
        if hasattr(self.e, "upload_rows"):
            self.e.upload_rows(None if not multi else sorted(set(pieces)))
        nmax = max(len(s) for s in self.subsets)
        self.corr = (self._symm_tensor(nmax * rows * cols).view(nmax, rows, cols) if self.fused
                     else self.e.tensor((nmax, rows, cols)))
        self.scratch = self.e.scratch(n_proj)
        self.red = self.e.scratch(n_proj)
        self.resid = self.e.tensor(cfg.n_iterations, "float64")
        self.acc = self.e.tensor(1, "float64")
        self.passes_done = 0
        self._pending = None
        self._packed = False
        self.launch_log = None
        if multi:
            # the group's first collective involves every rank (NCCL creates
            # its communicator there; P2P batches need it to exist)
            dist.all_reduce(self.acc, group=group)
            self.acc.zero_()
        if self.fused:
            self._setup_fused()
        if self.poison:
            self._poison_mu()
            if hasattr(self.e, "poison_gather"):
                self.e.poison_gather()

    # -- fused exchanges (symmetric memory) -----------------------------------
    def _symm_tensor(self, n):
        import torch
        import torch.distributed._symmetric_memory as symm_mem
        t = symm_mem.empty(n, dtype=torch.float32, device=self.e.device)
        t.zero_()
        return t

    def _setup_fused(self):
        """Rendezvous, the per-peer store tables, and a barrier so that no
        rank's first peer store lands before every replica is initialised."""
        import torch
        import torch.distributed._symmetric_memory as symm_mem
        g = self.group if self.group is not None else _dist().group.WORLD
        self._h_corr = symm_mem.rendezvous(self.corr.view(-1), g)
        self._h_mu = symm_mem.rendezvous(self.mu.view(-1), g)
        me, world = self.rank, self.world
        dev = self.mu.device
        for sb in self.sub:
            t = np.zeros((sb.n, world, 2), dtype=np.int32)
            for b, v in enumerate(sb.views):
                a0, a1 = self.plan.band(int(v), me)
                for p in range(world):
                    if p == me:
                        t[b, p] = (a0, a1)
                    else:
                        q0, q1 = (int(x) for x in self.plan.need[p, int(v)])
                        lo, hi = max(a0, q0), min(a1, q1)
                        t[b, p] = (lo, hi) if hi > lo else (0, 0)
            sb.peer_rows = torch.as_tensor(t.reshape(-1), device=dev)
        r = np.zeros((world, 2), dtype=np.int64)
        for p in range(world):
            if p == me:
                r[p] = (0, self.n_layers * self.layer)
            else:
                lo = max(self.k0, int(self.plan.mu_need[p, 0]))
                hi = min(self.k1, int(self.plan.mu_need[p, 1]))
                r[p] = (lo * self.layer, hi * self.layer) if hi > lo else (0, 0)
        self._mu_ranges = torch.as_tensor(r.reshape(-1), device=dev)
        self._h_corr.barrier()
        self._h_mu.barrier()
        if world > 1:
            import warnings
            warnings.warn("CT_FUSED_COMM=1 with more than one rank: the slab peer stores are "
                          "verified with local replicas and on 1-rank groups only",
                          RuntimeWarning, stacklevel=3)

    def _corr_peers(self, sb):
        return ((self._h_corr.buffer_ptrs_dev, self.world, sb.peer_rows),) if self.fused else ()

    # -- accounting (bench.py) ------------------------------------------------
    @property
    def count(self) -> int:
        """Voxels this rank updates (its slab)."""
        return (self.k1 - self.k0) * self.layer

    def fp_rows(self, s: int) -> list:
        """(view, fraction of its rows) this rank marches in FP launch s
        (subset s >= 0; -1: the residual's other views; -2: subset 0)."""
        sb = self.sub[s] if s >= 0 else (self.rest if s == -1 else self.sub[0])
        return [(v, (b - a) / self.rows) for v, a, b in sb.rows_marched]

    def exchange_bytes(self, kind: str, s: int) -> float:
        """Bytes this rank receives in exchange `kind` of subset s."""
        if kind == "exchange_corr":
            return 4.0 * self.cols * sum(r1 - r0 for _, _, r0, r1 in self.sub[s].recvs)
        if kind == "exchange_mu":
            return 4.0 * self.layer * sum(l1 - l0 for _, l0, l1 in self.mu_recvs)
        return 0.0

    # -- helpers ---------------------------------------------------------------
    def _timed(self, kind, s, fn, *args):
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

    def _poison_mu(self):
        """NaN outside this rank's slab and its FP window's mu layers."""
        keep = np.zeros(self.n_layers, dtype=bool)
        keep[self.k0:self.k1] = True
        m0, m1 = (int(x) for x in self.plan.mu_need[self.rank])
        keep[m0:m1] = True
        for k in np.flatnonzero(~keep):
            self.mu[int(k)].fill_(float("nan"))

    def _pack(self, s):
        if not self._packed and self.win[1] >= self.win[0]:
            self._timed("pack_gather", s, self.e.pack_layers, self.mu, self.win[0], self.win[1])
        self._packed = True

    def _exchange_corr(self, sb: _SubsetBands):
        ops = [("send", self.corr[b, r0:r1], p) for p, b, r0, r1 in sb.sends]
        ops += [("recv", self.corr[b, r0:r1], p) for p, b, r0, r1 in sb.recvs]
        p2p_exchange(ops, self.group)

    def _exchange_mu(self):
        ops = [("send", self.mu[l0:l1], p) for p, l0, l1 in self.mu_sends]
        ops += [("recv", self.mu[l0:l1], p) for p, l0, l1 in self.mu_recvs]
        p2p_exchange(ops, self.group)

    def _finish_residual(self):
        """All-reduce the slot partials (one owner per slot) and sum them."""
        dist = _dist()
        self.red.copy_(self.scratch)
        if self.world > 1:
            self._timed("all_reduce_resid", -1, dist.all_reduce, self.red, dist.ReduceOp.SUM,
                        self.group)
        self.acc.zero_()
        self.e.residual_sum(self.red, self.acc)
        k = min(self._pending, self.resid.numel() - 1)
        self.resid[k:k + 1].copy_(self.acc)
        self._pending = None

    # -- passes ----------------------------------------------------------------
    def run_subset(self, s: int) -> None:
        sb = self.sub[s]
        n_proj = self.ps.geom.n_proj
        self._pack(s)
        if self.poison:
            self.corr[:sb.n].fill_(float("nan"))
        fused = s == 0 and self._pending is not None
        peers = self._corr_peers(sb)
        if sb.band_rows > 0:
            if fused:
                self._timed("fp_correction_resid", s, self.e.correction_bands, self.mu,
                            sb.slots, sb.n, self.corr, sb.bands, sb.band_rows, n_proj,
                            self.scratch, *peers)
            else:
                self._timed("fp_correction", s, self.e.correction_bands, self.mu, sb.slots,
                            sb.n, self.corr, sb.bands, sb.band_rows, 0, None, *peers)
        if fused:
            self._finish_residual()
        if self.fused:           # every rank's peer stores of the corrections are done
            self._timed("barrier_corr", s, self._h_corr.barrier)
        elif self.world > 1:
            self._timed("exchange_corr", s, self._exchange_corr, sb)
        mu_peers = ((self._h_mu.buffer_ptrs_dev, self.world, self._mu_ranges),) \
            if self.fused else ()
        if self.k1 > self.k0:
            self._timed("bp_update", s, self.e.bp_update_range, self.corr[:sb.n], sb.slots,
                        sb.n, self.k0 * self.layer, (self.k1 - self.k0) * self.layer, self.mu,
                        *mu_peers)
        if self.fused:           # every slab's halo layers are in the replicas needing them
            self._timed("barrier_mu", s, self._h_mu.barrier)
        elif self.world > 1:
            self._timed("exchange_mu", s, self._exchange_mu)
        if self.poison:
            self._poison_mu()
        self._packed = False

    def run_pass(self, residual: bool | None = None) -> None:
        want = self.cfg.compute_residuals if residual is None else residual
        if not want:
            self.finalize()
        for s in range(len(self.subsets)):
            self.run_subset(s)
        if want:
            if self.rest is not None and self.rest.band_rows > 0:
                self._pack(-1)
                self._timed("fp_residual", -1, self.e.residual_bands, self.mu, self.rest.slots,
                            self.rest.n, self.rest.bands, self.rest.band_rows,
                            self.ps.geom.n_proj, self.scratch)
            self._pending = self.passes_done
        self.passes_done += 1

    def finalize(self) -> None:
        """Complete a deferred residual: the first subset's bands on the current mu."""
        if self._pending is None:
            return
        sb = self.sub[0]
        if sb.band_rows > 0:
            self._pack(-2)
            self._timed("fp_residual", -2, self.e.residual_bands, self.mu, sb.slots, sb.n,
                        sb.bands, sb.band_rows, self.ps.geom.n_proj, self.scratch)
        self._finish_residual()

    def gather_volume(self) -> None:
        """Every rank's slab into every replica (once, at the end)."""
        if self.world == 1:
            return
        me = self.rank
        ops = []
        for p in range(self.world):
            if p == me:
                continue
            if self.k1 > self.k0:
                ops.append(("send", self.mu[self.k0:self.k1], p))
            a, b = int(self.plan.L[p]), int(self.plan.L[p + 1])
            if b > a:
                ops.append(("recv", self.mu[a:b], p))
        p2p_exchange(ops, self.group)

    def run(self):
        t0 = time.perf_counter()
        for _ in range(self.cfg.n_iterations):
            self.run_pass()
        self.finalize()
        self.gather_volume()
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


def sart_run_slab(ps, grid, cfg=None, group=None):
    """Slab-decomposed angle-sharded (OS-)SART over the ranks of `group`."""
    from .recon import SartConfig
    return SlabSartRun(ps, grid, cfg or SartConfig(), group).run()
