"""SART / OS-SART reconstruction on the B200 (drop-in for ``cyltomo/recon.py``).

One SART view update (``cyltomo/recon.py:88-120``) is two kernels:

1. ``ct_fp_*_correction`` -- forward projection of the view(s) whose
   epilogue writes the correction image c = (p - sim) / w on valid pixels
   (w > 1e-6 * max_row, ``recon.py:96-102``);
2. ``ct_bp_*_update`` -- voxel-driven back-projection whose epilogue applies
   mu += relaxation * w_m * num / den on touched voxels (den > 0, w_m != 0),
   clamped at 0 when nonnegativity is on (``recon.py:105-119``).

``n_subsets`` (new) turns this into OS-SART: subset s is
the positions k of the projection order with k % S == s; every view of a
subset is projected on the same mu, their corrections are back-projected
and summed (num, den) in registers, and the update is applied once.
S = P (or None) is exactly the reference's per-view SART.

The row-sum maxima are pure geometry, so they are computed once per run
without marching (``ct_rowsum_max_*``); an empty view therefore raises
``EmptyView`` before any update is applied -- observably the same as the
reference, whose partially updated volume is discarded with the exception.
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field

import os

import numpy as np

from . import _device as D
from . import _native as N
from .errors import ConfigError, EmptyRoi, EmptyView
from .geometry import ScanGeometry
from .grid import CartGrid, CartVolume, CylGrid, CylVolume, is_device_array
from .projector import LINE_INTEGRAL, ProjectionSet, RaySamplingConfig

ROW_SUM_SKIP_FRACTION = 1e-6  # cyltomo/recon.py:29


@dataclass
class SartConfig:
    """Knobs of a (OS-)SART run (``cyltomo/recon.py:32-61``).

    Reference fields keep their meaning.  Additions: ``n_subsets`` (None =
    per-view SART; S < P = OS-SART with interleaved subsets) and
    ``compute_residuals`` (the reference always evaluates ||p - A mu|| after
    every pass, one extra full forward projection per pass).
    """

    relaxation: float = 1.0
    n_iterations: int = 1
    projection_order: str = "acquisition"
    order_seed: int = 0
    nonnegativity: bool = True
    initial: object = None
    weights: object = None
    resample_initial: bool = False
    sampling: RaySamplingConfig = field(default_factory=RaySamplingConfig)
    n_subsets: int | None = None
    compute_residuals: bool = True

    def __post_init__(self):
        if not 0.0 < self.relaxation <= 2.0:
            raise ConfigError("relaxation must lie in (0, 2]")
        if self.n_iterations < 1:
            raise ConfigError("n_iterations must be >= 1")
        if self.projection_order not in ("acquisition", "fixed_permutation"):
            raise ConfigError(f"unknown projection order {self.projection_order!r}")
        if self.n_subsets is not None and int(self.n_subsets) < 1:
            raise ConfigError("n_subsets must be >= 1")


@dataclass
class ReconReport:
    """Per-pass residual norms ||p - A mu||_2, wall time and config echo."""

    residuals: list
    wall_time: float
    config: dict


def _config_echo(cfg: SartConfig) -> dict:
    return {
        "relaxation": cfg.relaxation,
        "n_iterations": cfg.n_iterations,
        "projection_order": cfg.projection_order,
        "order_seed": cfg.order_seed,
        "nonnegativity": cfg.nonnegativity,
        "initial": None if cfg.initial is None else f"volume{tuple(cfg.initial.mu.shape)}",
        "weights": None if cfg.weights is None else f"map{tuple(np.shape(cfg.weights))}",
        "step_mm": cfg.sampling.step,
        "supersample": cfg.sampling.supersample,
        "n_subsets": cfg.n_subsets,
    }


def projection_order(cfg: SartConfig, n_proj: int) -> np.ndarray:
    """Acquisition order or the seeded fixed permutation (``recon.py:166-169``)."""
    if cfg.projection_order == "fixed_permutation":
        return np.random.default_rng(cfg.order_seed).permutation(n_proj)
    return np.arange(n_proj)


def make_subsets(order: np.ndarray, n_subsets: int | None) -> list:
    """Interleaved OS-SART subsets: positions k of `order` with k % S == s."""
    n = len(order)
    s = n if n_subsets is None else min(int(n_subsets), n)
    return [np.asarray(order[i::s], dtype=np.int64) for i in range(s)]


class SartEngine:
    """Device-resident tables and launchers for one (grid, geometry, sampling).

    ``views`` restricts the tables to a subset of the geometry's views (slot b
    of the tables is view views[b]); all launchers take device int32 slot
    lists.
    """

    def __init__(self, grid, geom: ScanGeometry, sampling: RaySamplingConfig, views=None):
        if not isinstance(grid, (CylGrid, CartGrid)):
            raise TypeError(f"cannot reconstruct on {type(grid).__name__}")
        self.device = D.require_cuda()
        self.grid, self.geom = grid, geom
        self.cyl = isinstance(grid, CylGrid)
        self.views = np.arange(geom.n_proj) if views is None else np.asarray(views)
        self.gc = D.grid_c(grid)
        self.rows, self.cols = geom.det_rows, geom.det_cols
        self.samp = D.sampling_c(sampling.step_for(grid), sampling.supersample,
                                 sampling.interpolation == "nearest")
        self.fp_views = D.upload_f64(D.ray_view_table(grid, geom, self.views))
        self.bp_dets = D.upload_f64(D.det_view_table(geom, self.views))
        self.trig = D.upload_f64(D.trig_table(grid)) if self.cyl else None
        self.row_thr = None
        self._scratch = {}

    # -- geometry-only setup -------------------------------------------------
    def row_max(self) -> np.ndarray:
        """max_row of every table slot (exact; no march)."""
        torch = D.torch_mod()
        n = len(self.views)
        out = torch.zeros(n, dtype=torch.float64, device=self.device)
        b = D.batch_c(n, self.rows, self.cols)
        fn = "ct_rowsum_max_cyl" if self.cyl else "ct_rowsum_max_cart"
        N.call(fn, C.byref(self.gc), D.ptr(self.fp_views), C.byref(b), C.byref(self.samp),
               D.ptr(out), D.stream_handle())
        return D.to_host(out)

    def row_samples(self, views) -> np.ndarray:
        """In-support samples per detector row of the given views, shape
        (len(views), rows) int64 (geometry only, no march)."""
        torch = D.torch_mod()
        n = len(views)
        out = torch.zeros(n * self.rows, dtype=torch.int64, device=self.device)
        slots = D.upload_i32(views)
        b = D.batch_c(n, self.rows, self.cols, slots)
        fn = "ct_row_samples_cyl" if self.cyl else "ct_row_samples_cart"
        N.call(fn, C.byref(self.gc), D.ptr(self.fp_views), C.byref(b), C.byref(self.samp),
               D.ptr(out), D.stream_handle())
        return D.to_host(out).reshape(n, self.rows)

    def prepare_thresholds(self, order_slots=None) -> np.ndarray:
        """Row maxima -> skip thresholds; EmptyView for the first empty view."""
        max_row = self.row_max()
        check = range(len(self.views)) if order_slots is None else order_slots
        for slot in check:
            if max_row[slot] <= 0.0:
                raise EmptyView(f"view {int(self.views[slot])} misses the volume entirely")
        self.row_thr = D.upload_f64(ROW_SUM_SKIP_FRACTION * max_row)
        return max_row

    def prepare_thresholds_async(self):
        """prepare_thresholds without a host round trip: the skip thresholds
        are computed on the device, and the row maxima are copied to pinned
        host memory behind an event.  Returns (max_row_host, event); the
        caller checks for empty views once the event has completed
        (check_empty_views) -- the kernels treat an empty view as all-skipped,
        so work queued before the check is harmless."""
        torch = D.torch_mod()
        n = len(self.views)
        out = torch.zeros(n, dtype=torch.float64, device=self.device)
        b = D.batch_c(n, self.rows, self.cols)
        fn = "ct_rowsum_max_cyl" if self.cyl else "ct_rowsum_max_cart"
        N.call(fn, C.byref(self.gc), D.ptr(self.fp_views), C.byref(b), C.byref(self.samp),
               D.ptr(out), D.stream_handle())
        self.row_thr = out * ROW_SUM_SKIP_FRACTION
        host = torch.empty(n, dtype=torch.float64, pin_memory=True)
        host.copy_(out, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        return host, ev

    def check_empty_views(self, max_row, order_slots=None) -> None:
        """EmptyView for the first empty view in processing order."""
        check = range(len(self.views)) if order_slots is None else order_slots
        for slot in check:
            if max_row[slot] <= 0.0:
                raise EmptyView(f"view {int(self.views[slot])} misses the volume entirely")

    # -- launchers -------------------------------------------------------------
    def alloc_gather(self):
        """Buffer for the FP gather layout (8 floats per voxel, 16B aligned);
        None (plain-layout FP) in nearest mode or with CT_FP_GATHER=0."""
        if self.samp.nearest or os.environ.get("CT_FP_GATHER", "1") == "0":
            return None
        return D.alloc_gather(self.grid, self.device)

    def pack(self, mu, gather) -> None:
        if gather is None:
            return
        fn = "ct_pack_gather_cyl" if self.cyl else "ct_pack_gather_cart"
        N.call(fn, D.ptr(mu), C.byref(self.gc), D.ptr(gather), D.stream_handle())

    def correction(self, mu, p_meas, slots, n: int, corr, gather=None) -> None:
        b = D.batch_c(n, self.rows, self.cols, slots)
        fn = "ct_fp_cyl_correction" if self.cyl else "ct_fp_cart_correction"
        N.call(fn, D.ptr(mu), D.ptr(gather), C.byref(self.gc), D.ptr(self.fp_views),
               C.byref(b), C.byref(self.samp), D.ptr(p_meas), D.ptr(self.row_thr), D.ptr(corr),
               D.stream_handle())

    def correction_single(self, mu, p_view, i: int, slot, corr, gather=None) -> None:
        """correction() of ONE table slot i (slot: device int32 [i]) whose
        measured image p_view (1, H, W) is stored alone: the kernels address
        p_meas by table slot, so the pointer handed over is p_view's address
        minus i images (only image i is ever read)."""
        b = D.batch_c(1, self.rows, self.cols, slot)
        base = p_view.data_ptr() - i * self.rows * self.cols * 4
        fn = "ct_fp_cyl_correction" if self.cyl else "ct_fp_cart_correction"
        N.call(fn, D.ptr(mu), D.ptr(gather), C.byref(self.gc), D.ptr(self.fp_views),
               C.byref(b), C.byref(self.samp), C.c_void_p(base), D.ptr(self.row_thr),
               D.ptr(corr), D.stream_handle())

    def alloc_quads(self, n: int):
        """Buffer for the bilinear footprints of an n-view correction stack
        (None with CT_BP_QUADS=0: the BP reads the four taps from corr)."""
        if os.environ.get("CT_BP_QUADS", "1") == "0":
            return None
        torch = D.torch_mod()
        b = D.batch_c(n, self.rows, self.cols)
        length = int(N.load_library().ct_quads_floats(C.byref(b)))
        return torch.empty(length, dtype=torch.float32, device=self.device)

    def pack_quads(self, corr, n: int, quads) -> None:
        if quads is None:
            return
        b = D.batch_c(n, self.rows, self.cols)
        N.call("ct_pack_quads", D.ptr(corr), C.byref(b), D.ptr(quads), D.stream_handle())

    def bp_update(self, corr, slots, n: int, upd: N.UpdateC, quads=None) -> None:
        b = D.batch_c(n, self.rows, self.cols, slots)
        if self.cyl:
            N.call("ct_bp_cyl_update", D.ptr(corr), D.ptr(quads), D.ptr(self.bp_dets),
                   C.byref(b), C.byref(self.gc), D.ptr(self.trig), C.byref(upd),
                   D.stream_handle())
        else:
            N.call("ct_bp_cart_update", D.ptr(corr), D.ptr(quads), D.ptr(self.bp_dets),
                   C.byref(b), C.byref(self.gc), C.byref(upd), D.stream_handle())

    def bp_partial(self, corr, slots, n: int, num, den, quads=None) -> None:
        """num/den = sum over the batch of the BP (overwrites)."""
        b = D.batch_c(n, self.rows, self.cols, slots)
        if self.cyl:
            N.call("ct_bp_cyl", D.ptr(corr), D.ptr(quads), D.ptr(self.bp_dets), C.byref(b),
                   C.byref(self.gc), D.ptr(self.trig), D.ptr(num), D.ptr(den), 0,
                   D.stream_handle())
        else:
            N.call("ct_bp_cart", D.ptr(corr), D.ptr(quads), D.ptr(self.bp_dets), C.byref(b),
                   C.byref(self.gc), D.ptr(num), D.ptr(den), 0, D.stream_handle())

    def residual_scratch(self, n: int):
        torch = D.torch_mod()
        b = D.batch_c(n, self.rows, self.cols)
        length = int(N.load_library().ct_residual_scratch_len(C.byref(b)))
        if n not in self._scratch:
            self._scratch[n] = torch.empty(length, dtype=torch.float64, device=self.device)
        return self._scratch[n]

    def row_tile(self) -> int:
        """Detector rows per FP block: row ranges aligned to it keep every
        residual partial on one launch (exact split sums)."""
        b = D.batch_c(1, self.rows, self.cols)
        return int(N.load_library().ct_fp_row_tile(C.byref(b)))

    def correction_rows(self, mu, p_meas, slots, n: int, corr, row_lo: int = 0,
                        row_hi: int | None = None, n_slots: int = 0, scratch=None,
                        gather=None, peers=None, n_peers: int = 0,
                        peer_off: int = 0) -> None:
        """Correction FP over flattened rows [row_lo, row_hi) of an n-view batch
        (corr holds rows from row_lo); with a scratch also the residual
        partials of the same simulation at the views' slots of an
        n_slots-view residual scratch."""
        b = D.batch_c(n, self.rows, self.cols, slots)
        hi = n * self.rows if row_hi is None else row_hi
        fn = "ct_fp_cyl_correction_rows" if self.cyl else "ct_fp_cart_correction_rows"
        N.call(fn, D.ptr(mu), D.ptr(gather), C.byref(self.gc), D.ptr(self.fp_views),
               C.byref(b), C.byref(self.samp), D.ptr(p_meas), D.ptr(self.row_thr), D.ptr(corr),
               int(row_lo), int(hi), int(n_slots), D.ptr(scratch),
               C.c_void_p(int(peers) if peers else 0), int(n_peers), int(peer_off),
               D.stream_handle())

    def residual_rows(self, mu, p_meas, slots, n: int, n_slots: int, scratch, row_lo: int = 0,
                      row_hi: int | None = None, gather=None) -> None:
        """Residual partials of flattened rows [row_lo, row_hi) of an n-view
        batch at the views' slots (no sum)."""
        b = D.batch_c(n, self.rows, self.cols, slots)
        hi = n * self.rows if row_hi is None else row_hi
        fn = "ct_fp_cyl_residual_rows" if self.cyl else "ct_fp_cart_residual_rows"
        N.call(fn, D.ptr(mu), D.ptr(gather), C.byref(self.gc), D.ptr(self.fp_views),
               C.byref(b), C.byref(self.samp), D.ptr(p_meas), int(row_lo), int(hi),
               int(n_slots), D.ptr(scratch), D.stream_handle())

    def bp_update_range(self, corr, slots, n: int, upd: N.UpdateC, offset: int, count: int,
                        quads=None) -> None:
        """bp_update restricted to voxels [offset, offset+count)."""
        b = D.batch_c(n, self.rows, self.cols, slots)
        if self.cyl:
            N.call("ct_bp_cyl_update_range", D.ptr(corr), D.ptr(quads), D.ptr(self.bp_dets),
                   C.byref(b), C.byref(self.gc), D.ptr(self.trig), C.byref(upd), int(offset),
                   int(count), D.stream_handle())
        else:
            N.call("ct_bp_cart_update_range", D.ptr(corr), D.ptr(quads), D.ptr(self.bp_dets),
                   C.byref(b), C.byref(self.gc), C.byref(upd), int(offset), int(count),
                   D.stream_handle())

    # -- slab decomposition (distributed.SlabSartRun; ABI v8) ------------------
    def row_cells(self, views) -> np.ndarray:
        """FP cell layers [min, max] read by each detector row's rays, shape
        (len(views), rows, 2) int32 (empty rows: INT32_MAX, INT32_MIN)."""
        torch = D.torch_mod()
        n = len(views)
        out = torch.empty(2 * n * self.rows, dtype=torch.int32, device=self.device)
        slots = D.upload_i32(views)
        b = D.batch_c(n, self.rows, self.cols, slots)
        fn = "ct_row_cells_cyl" if self.cyl else "ct_row_cells_cart"
        N.call(fn, C.byref(self.gc), D.ptr(self.fp_views), C.byref(b), C.byref(self.samp),
               D.ptr(out), D.stream_handle())
        return D.to_host(out).reshape(n, self.rows, 2)

    def pack_layers(self, mu, gather, kc_lo: int, kc_hi: int) -> None:
        """Pack the gather cells FP cell layers kc_lo..kc_hi read."""
        if gather is None:
            return
        fn = "ct_pack_gather_cyl_layers" if self.cyl else "ct_pack_gather_cart_layers"
        N.call(fn, D.ptr(mu), C.byref(self.gc), D.ptr(gather), int(kc_lo), int(kc_hi),
               D.stream_handle())

    def correction_bands(self, mu, p_meas, slots, n: int, corr, bands, band_rows: int,
                         n_slots: int = 0, scratch=None, gather=None, peers=None,
                         n_peers: int = 0, peer_rows=None) -> None:
        """Corrections of each view slot's row band (bands: device int32
        [n][2]) into the full [n][H][W] stack; with a scratch also the
        residual partials at the n_slots-view slots.  peers (device pointer
        array) / n_peers / peer_rows (device int32 [n][n_peers][2]): stored
        into the peers' stacks instead, each for its row range."""
        b = D.batch_c(n, self.rows, self.cols, slots)
        fn = "ct_fp_cyl_correction_bands" if self.cyl else "ct_fp_cart_correction_bands"
        N.call(fn, D.ptr(mu), D.ptr(gather), C.byref(self.gc), D.ptr(self.fp_views),
               C.byref(b), C.byref(self.samp), D.ptr(p_meas), D.ptr(self.row_thr), D.ptr(corr),
               D.ptr(bands), int(band_rows), int(n_slots), D.ptr(scratch),
               C.c_void_p(int(peers) if peers else 0), int(n_peers), D.ptr(peer_rows),
               D.stream_handle())

    def residual_bands(self, mu, p_meas, slots, n: int, bands, band_rows: int, n_slots: int,
                       scratch, gather=None) -> None:
        b = D.batch_c(n, self.rows, self.cols, slots)
        fn = "ct_fp_cyl_residual_bands" if self.cyl else "ct_fp_cart_residual_bands"
        N.call(fn, D.ptr(mu), D.ptr(gather), C.byref(self.gc), D.ptr(self.fp_views),
               C.byref(b), C.byref(self.samp), D.ptr(p_meas), D.ptr(bands), int(band_rows),
               int(n_slots), D.ptr(scratch), D.stream_handle())

    def residual_sum(self, scratch, accum) -> None:
        """accum += fixed-order sum of a residual scratch."""
        N.call("ct_residual_sum", D.ptr(scratch), int(scratch.numel()), D.ptr(accum),
               D.stream_handle())

    def residual(self, mu, p_meas, slots, n: int, accum, gather=None) -> None:
        """accum (device f64 scalar view) += sum (p - A mu)^2 over the batch."""
        b = D.batch_c(n, self.rows, self.cols, slots)
        scratch = self.residual_scratch(n)
        fn = "ct_fp_cyl_residual" if self.cyl else "ct_fp_cart_residual"
        N.call(fn, D.ptr(mu), D.ptr(gather), C.byref(self.gc), D.ptr(self.fp_views),
               C.byref(b), C.byref(self.samp), D.ptr(p_meas), D.ptr(scratch),
               D.ptr(accum), D.stream_handle())


def make_update(mu, weights, cfg: SartConfig) -> N.UpdateC:
    u = N.UpdateC()
    u.relaxation = float(cfg.relaxation)
    u.nonneg = 1 if cfg.nonnegativity else 0
    u.weights = None if weights is None else weights.data_ptr()
    u.mu = mu.data_ptr()
    return u


def _device_weights(cfg: SartConfig, shape, device):
    if cfg.weights is None:
        return None
    if tuple(np.shape(cfg.weights)) != tuple(shape):
        raise ConfigError("weight map shape does not match the volume")
    return D.to_device(cfg.weights, device=device)


def _volume_cls(grid):
    return CylVolume if isinstance(grid, CylGrid) else CartVolume


def _grid_key(grid) -> tuple:
    if isinstance(grid, CylGrid):
        p = grid.pose
        return ("cyl", grid.shape, float(grid.radius), float(grid.height), float(p.alpha),
                float(p.beta), float(p.gamma), tuple(float(x) for x in p.t))
    return ("cart", grid.shape, float(grid.voxel_size), tuple(float(x) for x in grid.origin))


def _geom_key(geom: ScanGeometry) -> tuple:
    angles = np.ascontiguousarray(geom.stage_angles, dtype=np.float64)
    return (float(geom.sdd), float(geom.sod), int(geom.det_cols), int(geom.det_rows),
            float(geom.pixel_pitch), tuple(float(x) for x in geom.principal_point),
            angles.size, hash(angles.tobytes()))


class _ViewUpdater:
    """Device state of the per-view SART entry point for one (grid, geometry,
    sampling): the tables of ALL views, their row maxima (one launch, one
    host copy -- EmptyView is decided per view from it), slot lists and a
    correction buffer.  sart_update_view keeps a few of these keyed by the
    CONTENT of grid / geometry / sampling, so a reference-style loop over
    views pays the setup once instead of per call."""

    def __init__(self, grid, geom: ScanGeometry, sampling: RaySamplingConfig):
        torch = D.torch_mod()
        self.eng = SartEngine(grid, geom, sampling)
        # row maxima of every view (pure geometry): host copy for the per-view
        # EmptyView decision, device skip thresholds for the correction FP
        self.max_row = self.eng.row_max()
        self.eng.row_thr = D.upload_f64(ROW_SUM_SKIP_FRACTION * self.max_row)
        self.corr = torch.empty((1, self.eng.rows, self.eng.cols), dtype=torch.float32,
                                device=self.eng.device)
        self.slots = {}

    def slot(self, i: int):
        t = self.slots.get(i)
        if t is None:
            t = self.slots[i] = D.upload_i32([i])
        return t

    def device_weights(self, w, shape):
        """The weight map on the device: a CUDA tensor as is, a host array
        uploaded per call (the caller may change it between calls)."""
        if w is None:
            return None
        if tuple(np.shape(w)) != tuple(shape):
            raise ConfigError("weight map shape does not match the volume")
        return D.to_device(w, device=self.eng.device)


_VIEW_UPDATERS: dict = {}
_VIEW_UPDATERS_MAX = 4


def _view_updater(grid, geom: ScanGeometry, sampling: RaySamplingConfig) -> _ViewUpdater:
    key = (_grid_key(grid), _geom_key(geom), sampling.step_for(grid), int(sampling.supersample),
           sampling.interpolation)
    u = _VIEW_UPDATERS.pop(key, None)
    if u is None:
        u = _ViewUpdater(grid, geom, sampling)
        while len(_VIEW_UPDATERS) >= _VIEW_UPDATERS_MAX:
            _VIEW_UPDATERS.pop(next(iter(_VIEW_UPDATERS)))
    _VIEW_UPDATERS[key] = u                                # most recently used last
    return u


def sart_update_view(vol, ps: ProjectionSet, i: int, cfg: SartConfig):
    """Apply the SART correction of view i to the volume, in place
    (``cyltomo/recon.py:88-120``).  Raises EmptyView when no ray of the view
    intersects the volume.

    Two launches per call (correction FP, fused BP update) on device state
    cached per (grid, geometry, sampling) content; a CUDA-tensor volume is
    updated in HBM without copies, a host array is uploaded and written back
    (the reference mutates its float64 array in place)."""
    if ps.kind != LINE_INTEGRAL:
        raise ConfigError("SART needs line-integral projections")
    if not isinstance(vol.grid, (CylGrid, CartGrid)):
        raise TypeError(f"cannot reconstruct on {type(vol.grid).__name__}")
    i = int(i)
    u = _view_updater(vol.grid, ps.geom, cfg.sampling)
    if u.max_row[i] <= 0.0:
        raise EmptyView(f"view {i} misses the volume entirely")
    eng = u.eng
    dev = eng.device
    mu = D.to_device(vol.mu, device=dev)
    weights = u.device_weights(cfg.weights, mu.shape)
    p_meas = D.to_device(ps.images[i:i + 1], device=dev)
    # the tables hold all views: view i is slot i; p_meas holds only view i,
    # so it is addressed as a one-view batch whose table slot is i
    eng.correction_single(mu, p_meas, i, u.slot(i), u.corr)
    eng.bp_update(u.corr, u.slot(i), 1, make_update(mu, weights, cfg))
    if is_device_array(vol.mu):
        if vol.mu.data_ptr() != mu.data_ptr():
            vol.mu.copy_(mu)
    else:
        vol.mu[...] = D.to_host(mu)
    return vol


def _initial_mu(grid, cfg: SartConfig, device):
    """Zeros, a copy of the template, or its resampling (``recon.py:123-145``)."""
    torch = D.torch_mod()
    init = cfg.initial
    if init is None:
        return torch.zeros(grid.shape, dtype=torch.float32, device=device)
    if isinstance(grid, CylGrid):
        if not isinstance(init, CylVolume):
            raise ConfigError("initial volume must be cylindrical for a CylGrid run")
        same = (init.grid.shape == grid.shape and init.grid.radius == grid.radius
                and init.grid.height == grid.height)
        if same:
            return D.to_device(init.mu, device=device).clone()
        if not cfg.resample_initial:
            raise ConfigError("initial volume shape does not match the grid; "
                              "set resample_initial to resample the template")
        from ._device import resample_cyl_to_cyl
        res = resample_cyl_to_cyl(CylVolume(init.grid, D.to_device(init.mu, device=device)),
                                  grid)
        return res.mu
    if not isinstance(init, CartVolume) or init.grid.shape != grid.shape:
        raise ConfigError("initial volume must match the Cartesian grid")
    return D.to_device(init.mu, device=device).clone()


class _StreamedUpload:
    """Host projections -> device in subset order on a copy stream, so the
    upload overlaps the first subsets' compute: subset k's views are copied
    (one async copy per view from page-locked memory) while subset k-1
    computes, and the compute stream waits on subset k's event just before
    its first use.  For page-locked host arrays (pageable ones: _StagedUpload)."""

    @staticmethod
    def applies(images) -> bool:
        torch = D.torch_mod()
        arr = np.asarray(images)
        return (arr.dtype == np.float32 and arr.flags.c_contiguous
                and torch.from_numpy(arr).is_pinned())

    def __init__(self, images, subsets, device):
        torch = D.torch_mod()
        host = torch.from_numpy(np.asarray(images))
        self.host = host
        self.dev = torch.empty(tuple(host.shape), dtype=torch.float32, device=device)
        self.subsets = subsets
        self.stream = torch.cuda.Stream(device)
        self.stream.wait_stream(torch.cuda.current_stream())
        self.events = [None] * len(subsets)
        self.issued = 0
        self.waited = [False] * len(subsets)
        self.issue(0)

    def issue(self, k: int) -> None:
        """Queue the copies of subsets up to k (inclusive)."""
        torch = D.torch_mod()
        while self.issued <= min(k, len(self.subsets) - 1):
            with torch.cuda.stream(self.stream):
                for v in self.subsets[self.issued]:
                    self.dev[int(v)].copy_(self.host[int(v)], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.stream)
            self.events[self.issued] = ev
            self.issued += 1

    def before_subset(self, k: int) -> None:
        """Make subset k resident for the compute stream (and queue k+1)."""
        if all(self.waited):
            return
        torch = D.torch_mod()
        self.issue(k + 1)
        if not self.waited[k]:
            torch.cuda.current_stream().wait_event(self.events[k])
            self.waited[k] = True

    def finish(self) -> None:
        """Everything resident for the compute stream."""
        for k in range(len(self.subsets)):
            self.before_subset(k)

    @property
    def done(self) -> bool:
        return all(self.waited)


_STAGE_POOL = None


def _stage_pool():
    global _STAGE_POOL
    if _STAGE_POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        cap = int(os.environ.get("CT_HOST_THREADS", "0")) or 8       # cli --threads
        _STAGE_POOL = ThreadPoolExecutor(max_workers=max(1, min(cap, (os.cpu_count() or 2) // 2)))
    return _STAGE_POOL


class _StagedUpload(_StreamedUpload):
    """Pageable host projections: worker threads copy the views, in subset
    order, into a page-locked staging array (numpy copies release the GIL, so
    the host memcpy runs on several cores), and each subset's views go up
    asynchronously on the copy stream as soon as they are staged -- the
    staging of view i+1 overlaps the DMA of view i, and both overlap the
    compute of earlier subsets.  The staging array comes from torch's caching
    host allocator (reused by the next call)."""

    @staticmethod
    def applies(images) -> bool:
        arr = np.asarray(images)
        return (os.environ.get("CT_STAGED_UPLOAD", "1") != "0" and arr.ndim == 3
                and arr.dtype == np.float32 and arr.nbytes >= (16 << 20))

    def __init__(self, images, subsets, device):
        torch = D.torch_mod()
        src = np.asarray(images)
        pinned = torch.empty(src.shape, dtype=torch.float32, pin_memory=True)
        dst = pinned.numpy()
        pool = _stage_pool()
        self.futures = {}
        for sub in subsets:
            for v in sub:
                v = int(v)
                self.futures[v] = pool.submit(np.copyto, dst[v], src[v])
        super().__init__(dst, subsets, device)

    def issue(self, k: int) -> None:
        # the subset's views must be staged before their DMA is queued
        for kk in range(self.issued, min(k, len(self.subsets) - 1) + 1):
            for v in self.subsets[kk]:
                self.futures[int(v)].result()
        super().issue(k)


class SartRun:
    """A prepared (OS-)SART reconstruction: tables, thresholds, buffers.

    ``sart_run`` is ``SartRun(...).run()``; the bench and the distributed
    driver use the object directly to time passes and reuse buffers.
    """

    GRAPH_MIN_SUBSETS = 16   # per-view SART (many small launches) replays a CUDA graph

    def __init__(self, ps: ProjectionSet, grid, cfg: SartConfig, use_graph: bool | None = None):
        if ps.kind != LINE_INTEGRAL:
            raise ConfigError("SART needs line-integral projections")
        torch = D.torch_mod()
        self.ps, self.grid, self.cfg = ps, grid, cfg
        self.eng = SartEngine(grid, ps.geom, cfg.sampling)
        dev = self.eng.device
        self.mu = _initial_mu(grid, cfg, dev)
        self.order = projection_order(cfg, ps.geom.n_proj)
        self.subsets = make_subsets(self.order, cfg.n_subsets)
        # row maxima / thresholds stay on the device; the EmptyView check runs
        # once their host copy has landed (run(), after the first pass is queued)
        self._max_row, self._max_row_ev = self.eng.prepare_thresholds_async()
        self._empty_checked = False
        self.weights = _device_weights(cfg, grid.shape, dev)
        if ps.on_device:
            self._p_meas = D.to_device(ps.images, device=dev)
            self._upload = None
        elif _StreamedUpload.applies(ps.images):
            self._upload = _StreamedUpload(ps.images, self.subsets, dev)
            self._p_meas = self._upload.dev
        elif _StagedUpload.applies(ps.images):
            self._upload = _StagedUpload(ps.images, self.subsets, dev)
            self._p_meas = self._upload.dev
        else:
            self._p_meas = D.to_device(ps.images, device=dev)
            self._upload = None
        self.subset_slots = [D.upload_i32(s) for s in self.subsets]
        self.all_slots = D.upload_i32(np.arange(ps.geom.n_proj))
        nmax = max(len(s) for s in self.subsets)
        self.corr = torch.empty((nmax, self.eng.rows, self.eng.cols), dtype=torch.float32,
                                device=dev)
        self.upd = make_update(self.mu, self.weights, cfg)
        self.gather = self.eng.alloc_gather()
        self.quads = self.eng.alloc_quads(nmax)
        self.resid = torch.zeros(cfg.n_iterations, dtype=torch.float64, device=dev)
        self.resid_cur = torch.zeros(1, dtype=torch.float64, device=dev)
        self.eng.residual_scratch(ps.geom.n_proj)      # no allocation inside a pass
        self.passes_done = 0
        self.launch_log = None   # list -> (kind, subset, start_event, end_event) per launch
        self.use_graph = (len(self.subsets) >= self.GRAPH_MIN_SUBSETS
                          if use_graph is None else bool(use_graph))
        self._graphs = {}
        # Deferred residual (OS-SART, eager passes): the residual FP of pass k
        # and the correction FP of pass k+1's first subset read the same mu,
        # so pass k marches only the other subsets' views for its residual and
        # pass k+1's first correction launch adds the first subset's partials
        # (same slots, same fixed-order sum: bit-identical residuals, one
        # subset's FP fewer per pass).  finalize() completes a pending one.
        self.fuse_residual = (not self.use_graph and len(self.subsets) > 1
                              and os.environ.get("CT_RESID_FUSE", "1") != "0")
        self._pending = None                             # pass index awaiting subset 0
        self._gather_mu = False                          # gather holds the current mu
        if self.fuse_residual:
            rest = np.setdiff1d(np.arange(ps.geom.n_proj), self.subsets[0])
            self.rest_slots = D.upload_i32(rest) if len(rest) else None
            self.n_rest = len(rest)

    def _timed(self, kind, s, fn, *args):
        if self.launch_log is None:
            fn(*args)
            return
        torch = D.torch_mod()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn(*args)
        b.record()
        self.launch_log.append((kind, s, a, b))

    @property
    def p_meas(self):
        """The measured projections on the device (complete: any streamed
        upload is finished for the current stream first)."""
        if self._upload is not None:
            self._upload.finish()
        return self._p_meas

    def check_empty_views(self) -> None:
        """Raise EmptyView (reference order) once the row maxima are on the host."""
        if not self._empty_checked:
            self._max_row_ev.synchronize()
            self._empty_checked = True
            self.eng.check_empty_views(self._max_row.numpy(), order_slots=self.order)

    def _pack(self, k) -> None:
        if not self._gather_mu:
            self._timed("pack_gather", k, self.eng.pack, self.mu, self.gather)
        self._gather_mu = True

    def _store_residual(self, k) -> None:
        k = min(k, self.resid.numel() - 1)
        self.resid[k:k + 1].copy_(self.resid_cur)

    def _pass_body(self, residual: bool, after_updates=None, fuse: bool = False) -> None:
        e = self.eng
        up = self._upload if (self._upload is not None and not self._upload.done) else None
        n_proj = self.ps.geom.n_proj
        for k, (s, slots) in enumerate(zip(self.subsets, self.subset_slots)):
            if up is not None:
                up.before_subset(k)
            self._pack(k)
            if k == 0 and self._pending is not None:
                # completes the previous pass's residual (same mu)
                scratch = e.residual_scratch(n_proj)
                self._timed("fp_correction_resid", k, e.correction_rows, self.mu,
                            self._p_meas, slots, len(s), self.corr, 0, None, n_proj, scratch,
                            self.gather)
                self.resid_cur.zero_()
                e.residual_sum(scratch, self.resid_cur)
                self._store_residual(self._pending)
                self._pending = None
            else:
                self._timed("fp_correction", k, e.correction, self.mu, self._p_meas, slots,
                            len(s), self.corr, self.gather)
            self._timed("pack_quads", k, e.pack_quads, self.corr, len(s), self.quads)
            self._timed("bp_update", k, e.bp_update, self.corr, slots, len(s), self.upd,
                        self.quads)
            self._gather_mu = False
        if after_updates is not None:
            after_updates()
        if residual and fuse:
            self._pack(-1)
            if self.n_rest:
                self._timed("fp_residual", -1, e.residual_rows, self.mu, self._p_meas,
                            self.rest_slots, self.n_rest, n_proj,
                            e.residual_scratch(n_proj), 0, None, self.gather)
            self._pending = self.passes_done
        elif residual:
            self.resid_cur.zero_()
            self._pack(-1)
            self._timed("fp_residual", -1, e.residual, self.mu, self._p_meas, self.all_slots,
                        n_proj, self.resid_cur, self.gather)

    def finalize(self) -> None:
        """Complete a deferred residual: the first subset's views on the
        current mu (the gather layout still holds it)."""
        if self._pending is None:
            return
        e = self.eng
        n_proj = self.ps.geom.n_proj
        scratch = e.residual_scratch(n_proj)
        self._pack(-1)
        self._timed("fp_residual", -2, e.residual_rows, self.mu, self._p_meas,
                    self.subset_slots[0], len(self.subsets[0]), n_proj, scratch, 0, None,
                    self.gather)
        self.resid_cur.zero_()
        e.residual_sum(scratch, self.resid_cur)
        self._store_residual(self._pending)
        self._pending = None

    def run_pass(self, residual: bool | None = None) -> None:
        """One pass over all subsets (+ the residual FP if enabled).

        With use_graph the whole pass is captured once as a CUDA graph and
        replayed (same kernels, same bits) -- per-view SART issues 3 launches
        per view, which would otherwise be launch-bound."""
        want = self.cfg.compute_residuals if residual is None else residual
        if self.use_graph and self.launch_log is None:
            self._gather_mu = False          # graph bodies always pack
            torch = D.torch_mod()
            g = self._graphs.get(want)
            if g is None:
                if self._upload is not None:
                    self._upload.finish()
                # low-level capture on a side stream: torch.cuda.graph() would
                # also gc.collect() and empty the caching allocator every time
                g = torch.cuda.CUDAGraph()
                side = torch.cuda.Stream(self.eng.device)
                side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(side):
                    g.capture_begin()
                    try:
                        self._pass_body(want)
                    finally:
                        g.capture_end()
                torch.cuda.current_stream().wait_stream(side)
                self._graphs[want] = g
            g.replay()
            self._gather_mu = False
            if want:
                self._store_residual(self.passes_done)
        else:
            self._eager_pass(want)
        self.passes_done += 1

    def _eager_pass(self, want: bool, after_updates=None) -> None:
        if want and self.fuse_residual:
            self._pass_body(True, after_updates, fuse=True)
            return
        self.finalize()
        self._pass_body(want, after_updates)
        if want:
            self._store_residual(self.passes_done)

    def _run_pass_hooked(self, after_updates) -> None:
        """run_pass (eager) with a hook queued after the last subset's update."""
        self._eager_pass(self.cfg.compute_residuals, after_updates)
        self.passes_done += 1

    def run(self):
        torch = D.torch_mod()
        t0 = time.perf_counter()
        host_mu = None
        for it in range(self.cfg.n_iterations):
            last = it == self.cfg.n_iterations - 1
            if last and not self.ps.on_device and not self.use_graph:
                # the final volume is complete after the last subset's update:
                # copy it out on a side stream while the residual FP runs
                host_mu = torch.empty(tuple(self.mu.shape), dtype=self.mu.dtype,
                                      pin_memory=True)
                copy_stream = torch.cuda.Stream(self.eng.device)

                def d2h():
                    copy_stream.wait_stream(torch.cuda.current_stream())
                    with torch.cuda.stream(copy_stream):
                        host_mu.copy_(self.mu, non_blocking=True)
                    self.mu.record_stream(copy_stream)
                self._run_pass_hooked(d2h)
            else:
                self.run_pass()
            self.check_empty_views()
        self.finalize()
        torch.cuda.synchronize(self.eng.device)
        wall = time.perf_counter() - t0
        residuals = ([math.sqrt(float(x)) for x in D.to_host(self.resid)]
                     if self.cfg.compute_residuals else [])
        if self.ps.on_device:
            mu = self.mu
        elif host_mu is not None:
            mu = host_mu.numpy()
        else:
            mu = D.to_host(self.mu, pinned=True)
        vol = _volume_cls(self.grid)._trusted(self.grid, mu)
        return vol, ReconReport(residuals=residuals, wall_time=wall,
                                config=_config_echo(self.cfg))


def sart_run(ps: ProjectionSet, grid, cfg: SartConfig | None = None):
    """Run (OS-)SART on an object-aligned grid; returns (volume, ReconReport)
    (``cyltomo/recon.py:156-182``).  The grid carries the pose, so a template
    initial volume in object coordinates aligns automatically."""
    cfg = cfg or SartConfig()
    return SartRun(ps, grid, cfg).run()


def presence_metric(vol, roi) -> float:
    """Mean attenuation over a region (``cyltomo/recon.py:185-200``)."""
    mu = D.to_host(vol.mu) if is_device_array(vol.mu) else np.asarray(vol.mu)
    if hasattr(roi, "mask"):
        mask = roi.mask(vol.grid)
    else:
        mask = np.asarray(roi, dtype=bool)
        if mask.shape != mu.shape:
            raise EmptyRoi("roi mask shape does not match the volume")
    n = int(mask.sum())
    if n == 0:
        raise EmptyRoi("region contains no voxels")
    return float(mu[mask].astype(np.float64).mean())
