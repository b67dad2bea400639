"""Forward projection and voxel-driven back-projection on the B200.

Drop-in for ``cyltomo/projector.py`` (same names, argument meaning and
errors).  The forward operator is pixel driven with equidistant sampling
(step, trilinear interpolation, in-support counting) and the backward
operator voxel driven with a bilinear detector footprint -- the reference's
deliberately unmatched pair (``cyltomo/projector.py:1-11``).  Both run as
sm_100a kernels (``ct_fp_*`` / ``ct_bp_*``).

Host/device: if the volume (or correction image) is a host numpy array the
call uploads it, runs on the GPU and returns float32 numpy arrays; if it is a
CUDA tensor the results stay in HBM as CUDA tensors.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _native as N
from .errors import NonPositiveIntensity
from .geometry import ScanGeometry
from .grid import CartGrid, CartVolume, CylGrid, CylVolume, is_device_array

LINE_INTEGRAL = "line_integral"
INTENSITY = "intensity"
GATHER_MIN_VIEWS = 4   # batched FP builds the gather layout (identical results)


@dataclass
class RaySamplingConfig:
    """Equidistant ray sampling (``cyltomo/projector.py:28-56``).

    step None -> half the smallest voxel extent (0.5*min(dr, dh) on a
    cylindrical grid, 0.5*voxel on a Cartesian one); supersample averages
    ss x ss sub-rays per pixel; interpolation is "linear" or "nearest".
    """

    step: float | None = None
    supersample: int = 1
    interpolation: str = "linear"

    def __post_init__(self):
        if self.step is not None and self.step <= 0.0:
            raise ValueError("step must be positive")
        if self.supersample < 1:
            raise ValueError("supersample must be >= 1")
        if self.interpolation not in ("linear", "nearest"):
            raise ValueError(f"unknown interpolation {self.interpolation!r}")

    def step_for(self, vol) -> float:
        if self.step is not None:
            return self.step
        g = vol.grid if hasattr(vol, "grid") else vol
        if isinstance(g, CylGrid):
            return 0.5 * min(g.d_r, g.d_h)
        return 0.5 * g.voxel_size


@dataclass
class ProjectionSet:
    """(P, H, W) stack with its geometry (``cyltomo/projector.py:59-80``).

    images are float32 (host numpy or CUDA tensor); shape, kind and
    finiteness are validated like the reference.
    """

    geom: ScanGeometry
    images: object
    kind: str = LINE_INTEGRAL

    def __post_init__(self):
        expected = (self.geom.n_proj, self.geom.det_rows, self.geom.det_cols)
        if type(self.images).__module__.startswith("torch"):
            torch = D.torch_mod()
            self.images = self.images.to(torch.float32).contiguous()
            shape = tuple(self.images.shape)
            finite = bool(torch.isfinite(self.images).all())
        else:
            self.images = np.ascontiguousarray(self.images, dtype=np.float32)
            shape = self.images.shape
            finite = bool(np.all(np.isfinite(self.images)))
        if shape != expected:
            raise ValueError(f"images shape {shape} does not match geometry {expected}")
        if self.kind not in (LINE_INTEGRAL, INTENSITY):
            raise ValueError(f"unknown projection kind {self.kind!r}")
        if not finite:
            raise ValueError("projection images contain non-finite values")

    @property
    def on_device(self) -> bool:
        return is_device_array(self.images)


def _project(vol, geom: ScanGeometry, views, cfg: RaySamplingConfig, want_w: bool):
    """Batched FP of `views`; returns device tensors (p, w or None)."""
    if not isinstance(vol, (CylVolume, CartVolume)):
        raise TypeError(f"cannot project object of type {type(vol).__name__}")
    torch = D.torch_mod()
    dev = D.require_cuda()
    mu = D.to_device(vol.mu, device=dev)
    nv = len(views)
    H, W = geom.det_rows, geom.det_cols
    out_p = torch.empty((nv, H, W), dtype=torch.float32, device=dev)
    out_w = torch.empty((nv, H, W), dtype=torch.float32, device=dev) if want_w else None
    table = D.upload_f64(D.ray_view_table(vol.grid, geom, views))
    s = D.sampling_c(cfg.step_for(vol), cfg.supersample, cfg.interpolation == "nearest")
    b = D.batch_c(nv, H, W)
    cyl = isinstance(vol, CylVolume)
    g = D.grid_c(vol.grid)
    gather = None
    if nv >= GATHER_MIN_VIEWS and cfg.interpolation == "linear":
        # multi-view launches amortise building the sector-per-sample layout
        gather = D.alloc_gather(vol.grid, dev)
        N.call("ct_pack_gather_cyl" if cyl else "ct_pack_gather_cart", D.ptr(mu), C.byref(g),
               D.ptr(gather), D.stream_handle())
    N.call("ct_fp_cyl" if cyl else "ct_fp_cart", D.ptr(mu), D.ptr(gather), C.byref(g),
           D.ptr(table), C.byref(b), C.byref(s), D.ptr(out_p), D.ptr(out_w), D.stream_handle())
    return out_p, out_w


def forward_project(vol, geom: ScanGeometry, i: int, cfg: RaySamplingConfig | None = None,
                    return_weights: bool = False):
    """Line-integral image of view i (``cyltomo/projector.py:91-121``).

    With return_weights=True also returns the per-pixel sampled path length
    (the SART row sums sum_l t_jl).
    """
    cfg = cfg or RaySamplingConfig()
    p, w = _project(vol, geom, [int(i)], cfg, return_weights)
    if vol.on_device:
        return (p[0], w[0]) if return_weights else p[0]
    if return_weights:
        return D.to_host(p[0]), D.to_host(w[0])
    return D.to_host(p[0])


def forward_project_all(vol, geom: ScanGeometry,
                        cfg: RaySamplingConfig | None = None) -> ProjectionSet:
    """Every view as one line-integral stack, in ONE batched launch
    (``cyltomo/projector.py:124-130``); bit-identical to per-view calls."""
    cfg = cfg or RaySamplingConfig()
    p, _ = _project(vol, geom, list(range(geom.n_proj)), cfg, False)
    return ProjectionSet(geom, p if vol.on_device else D.to_host(p), LINE_INTEGRAL)


def back_project(correction, geom: ScanGeometry, i: int, grid, out=None):
    """Gather a correction image onto the voxels of view i
    (``cyltomo/projector.py:133-166``).

    Returns (num, den) of the grid's shape; pass out=(num, den) to
    accumulate across views.  Voxels projecting off the detector (or behind
    the source) accumulate nothing.
    """
    if not isinstance(grid, (CylGrid, CartGrid)):
        raise TypeError(f"cannot back-project onto {type(grid).__name__}")
    torch = D.torch_mod()
    host = not is_device_array(correction)
    shape = tuple(correction.shape)
    if shape != (geom.det_rows, geom.det_cols):
        raise ValueError("correction image does not match detector dims")
    dev = D.require_cuda()
    corr = D.to_device(correction, device=dev)
    if out is None:
        num = torch.zeros(grid.shape, dtype=torch.float32, device=dev)
        den = torch.zeros(grid.shape, dtype=torch.float32, device=dev)
    else:
        num = D.to_device(out[0], device=dev)
        den = D.to_device(out[1], device=dev)
    dets = D.upload_f64(D.det_view_table(geom, [int(i)]))
    b = D.batch_c(1, geom.det_rows, geom.det_cols)
    g = D.grid_c(grid)
    if isinstance(grid, CylGrid):
        trig = D.upload_f64(D.trig_table(grid))
        N.call("ct_bp_cyl", D.ptr(corr), None, D.ptr(dets), C.byref(b), C.byref(g), D.ptr(trig),
               D.ptr(num), D.ptr(den), 1, D.stream_handle())
    else:
        N.call("ct_bp_cart", D.ptr(corr), None, D.ptr(dets), C.byref(b), C.byref(g), D.ptr(num),
               D.ptr(den), 1, D.stream_handle())
    if out is not None:
        # write back into the caller's arrays (accumulation semantics)
        for dst, src in zip(out, (num, den)):
            if is_device_array(dst):
                if dst.data_ptr() != src.data_ptr():
                    dst.copy_(src.view_as(dst))
            else:
                dst[...] = D.to_host(src)
        return out
    if host:
        return D.to_host(num), D.to_host(den)
    return num, den


def intensities_to_line_integrals(ps: ProjectionSet, i0) -> ProjectionSet:
    """Beer-Lambert p = -ln(I / I0) (``cyltomo/projector.py:169-181``), as the
    ``ct_line_integrals`` kernel.  i0 is a scalar or an (H, W) flat field
    broadcast over all views; raises NonPositiveIntensity if any I or I0 <= 0."""
    torch = D.torch_mod()
    i0 = np.asarray(i0, dtype=np.float64)
    if np.any(i0 <= 0.0):
        raise NonPositiveIntensity("flat field contains values <= 0")
    dev = D.require_cuda()
    img = D.to_device(ps.images, device=dev)
    H, W = ps.geom.det_rows, ps.geom.det_cols
    flat = None
    scalar = 1.0
    if i0.ndim == 0:
        scalar = float(i0)
    else:
        if i0.shape != (H, W):
            raise ValueError("flat field must be a scalar or an (H, W) image")
        flat = D.to_device(i0.astype(np.float32), device=dev)
    out = torch.empty_like(img)
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    N.call("ct_line_integrals", D.ptr(img), img.numel(), H * W, D.ptr(flat), scalar,
           D.ptr(out), D.ptr(bad), D.stream_handle())
    if int(bad.item()):
        raise NonPositiveIntensity("intensity images contain values <= 0")
    return ProjectionSet(ps.geom, out if ps.on_device else D.to_host(out), LINE_INTEGRAL)


def simulate_scan(vol, geom: ScanGeometry, sampling: RaySamplingConfig | None = None,
                  noise_sigma: float = 0.0, rng=None) -> ProjectionSet:
    """All views (one batched FP launch) plus optional Gaussian pixel noise
    (``cyltomo/experiments.py:31-39``).  The noise is drawn on the host from
    ``rng`` (default ``default_rng(0)``) with the reference's call, so a seeded
    scan has the same noise realisation as the reference's."""
    ps = forward_project_all(vol, geom, sampling)
    if noise_sigma <= 0.0:
        return ps
    rng = rng or np.random.default_rng(0)
    host = D.to_host(ps.images) if ps.on_device else ps.images
    noisy = host.astype(np.float64) + rng.normal(0.0, noise_sigma, host.shape)
    if ps.on_device:
        return ProjectionSet(geom, D.to_device(noisy.astype(np.float32)), ps.kind)
    return ProjectionSet(geom, noisy, ps.kind)
