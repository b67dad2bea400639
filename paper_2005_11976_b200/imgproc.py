"""Projection-image segmentation for the pose step, batched over views on the GPU.

Mirrors the reference's ``cyltomo/imgproc.py`` API (same names, arguments,
errors).  The reference segments one view at a time in numpy/scipy; here the
whole (n_views, rows, cols) stack stays resident in HBM and every
per-pixel pass is a ``ct_*`` kernel:

* per-view min / max and 256-bin histograms (``ct_image_minmax``,
  ``ct_image_histogram``, numpy's exact binning) -> Otsu level picked on the
  host from the 256 counts (:func:`otsu_from_histogram`);
* threshold (+ square dilation) masks (``ct_threshold_dilate``);
* per-row leftmost / rightmost foreground column (``ct_row_extents`` on a mask,
  or ``ct_row_extents_levels``: threshold + extents for a whole ladder of
  levels in ONE pass over the image).

The axis endpoints need only those row extents: the band-corner rule of
``cyltomo/imgproc.py:97-131`` (extreme columns within the band rows, ties on
an extreme column resolved to the outermost row) is a function of each row's
leftmost and rightmost foreground column.  ``ct_axis_endpoints`` applies it
to the resident extent tables, so four fp64 numbers and a status per
(view, level) are all that cross PCIe.

Images are float32 (the framework's projection storage); the
comparisons run in fp64 on the fp32 values exactly as the reference's
``np.asarray(image, dtype=float)`` does.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _native as N
from .errors import DegenerateHistogram, DegenerateMask, EmptyResult, OutOfFrame
from .geometry import DetectorPoint

HIST_BINS = 256
OK, EMPTY, ONE_ROW = 0, 1, 2          # ct_axis_endpoints status codes


@dataclass
class AxisObservation:
    """Projected axis endpoints in one view; top.v < bottom.v by swap
    (cyltomo/imgproc.py:84-94)."""

    top: DetectorPoint
    bottom: DetectorPoint
    view: int = -1

    def __post_init__(self):
        if self.top.v > self.bottom.v:
            self.top, self.bottom = self.bottom, self.top


# ---------------------------------------------------------------------------
# host logic on reduced data (a few hundred numbers per view)
# ---------------------------------------------------------------------------
def otsu_from_histogram(counts, lo: float, hi: float) -> float:
    """Otsu level from np.histogram(image, len(counts), range=(lo, hi)) counts
    (cyltomo/imgproc.py:20-38): maximal between-class variance, middle of the
    maximal plateau (ties across empty gap bins)."""
    counts = np.asarray(counts, dtype=float)
    edges = np.linspace(lo, hi, counts.size + 1)
    centers = 0.5 * (edges[:-1] + edges[1:])
    w0 = np.cumsum(counts)
    w1 = counts.sum() - w0
    mass = np.cumsum(counts * centers)
    mu0 = np.divide(mass, w0, out=np.zeros_like(mass), where=w0 > 0)
    mu1 = np.divide(mass[-1] - mass, w1, out=np.zeros_like(mass), where=w1 > 0)
    between = w0 * w1 * (mu0 - mu1) ** 2
    best = np.flatnonzero(between == between.max())
    return float(centers[best[best.size // 2]])


def bilinear_sample(image, u, v):
    """Sample a host image at continuous (u, v); returns (values, valid)
    (cyltomo/imgproc.py:134-153).  Host helper; strips use the kernel."""
    image = np.asarray(image, dtype=float)
    u = np.asarray(u, dtype=float)
    v = np.asarray(v, dtype=float)
    n_rows, n_cols = image.shape
    valid = (u >= 0) & (u <= n_cols - 1) & (v >= 0) & (v <= n_rows - 1)
    uc = np.clip(u, 0, n_cols - 1)
    vc = np.clip(v, 0, n_rows - 1)
    iu = np.minimum(uc.astype(int), n_cols - 2) if n_cols > 1 else np.zeros_like(uc, dtype=int)
    iv = np.minimum(vc.astype(int), n_rows - 2) if n_rows > 1 else np.zeros_like(vc, dtype=int)
    fu, fv = uc - iu, vc - iv
    i1, j1 = np.minimum(iu + 1, n_cols - 1), np.minimum(iv + 1, n_rows - 1)
    vals = (image[iv, iu] * (1 - fu) * (1 - fv) + image[iv, i1] * fu * (1 - fv)
            + image[j1, iu] * (1 - fu) * fv + image[j1, i1] * fu * fv)
    return vals, valid


def _axis_row(axis: AxisObservation) -> list:
    p0 = np.array([axis.top.u, axis.top.v])
    p1 = np.array([axis.bottom.u, axis.bottom.v])
    return [p0[0], p0[1], p1[0], p1[1], float(np.linalg.norm(p1 - p0))]


# ---------------------------------------------------------------------------
# the device side: a resident (n_views, rows, cols) stack
# ---------------------------------------------------------------------------
class ViewStack:
    """Float32 projection images resident on the GPU, segmented as a batch."""

    def __init__(self, images):
        torch = D.torch_mod()
        self.device = D.require_cuda()
        t = D.to_device(images, device=self.device)
        if t.dim() == 2:
            t = t.unsqueeze(0)
        if t.dim() != 3:
            raise ValueError("images must be (rows, cols) or (n_views, rows, cols)")
        self.images = t.to(torch.float32).contiguous()
        self.n, self.rows, self.cols = (int(x) for x in self.images.shape)
        self._torch = torch

    def _buf(self, shape, dtype):
        return self._torch.empty(shape, dtype=dtype, device=self.device)

    def _f64(self, a):
        return self._torch.as_tensor(np.array(a, dtype=np.float64, order="C"),
                                     device=self.device)

    def minmax(self):
        """Per-view (lo, hi) as float64 host arrays (values of the fp32 images)."""
        torch = self._torch
        mn = self._buf(self.n, torch.float32)
        mx = self._buf(self.n, torch.float32)
        N.call("ct_image_minmax", D.ptr(self.images), self.n, self.rows * self.cols,
               D.ptr(mn), D.ptr(mx), D.stream_handle())
        return mn.cpu().numpy().astype(np.float64), mx.cpu().numpy().astype(np.float64)

    def histograms(self, lo, hi, bins: int = HIST_BINS) -> np.ndarray:
        """np.histogram(view, bins, range=(lo[v], hi[v]))[0] per view."""
        torch = self._torch
        counts = self._buf((self.n, bins), torch.int32)
        lo_t, hi_t = self._f64(lo), self._f64(hi)     # alive until after the launch
        N.call("ct_image_histogram", D.ptr(self.images), self.n, self.rows * self.cols,
               D.ptr(lo_t), D.ptr(hi_t), bins, D.ptr(counts), D.stream_handle())
        return counts.cpu().numpy().view(np.uint32).astype(np.int64)

    def otsu_levels(self, bins: int = HIST_BINS) -> np.ndarray:
        """Per-view Otsu level; NaN for a constant view (the caller raises
        DegenerateHistogram when it reaches that view, in view order)."""
        lo, hi = self.minmax()
        ok = hi > lo
        out = np.full(self.n, np.nan)
        if ok.any():
            lo_s, hi_s = np.where(ok, lo, 0.0), np.where(ok, hi, 1.0)
            counts = self.histograms(lo_s, hi_s, bins)
            for v in np.flatnonzero(ok):
                out[v] = otsu_from_histogram(counts[v], lo[v], hi[v])
        return out

    def masks(self, levels, radius: int):
        """uint8 device masks dilate(image > levels[v], radius)."""
        if radius < 0:
            raise ValueError("radius must be >= 0")
        torch = self._torch
        m = self._buf((self.n, self.rows, self.cols), torch.uint8)
        lv = self._f64(np.broadcast_to(levels, (self.n,)))
        N.call("ct_threshold_dilate", D.ptr(self.images), self.n, self.rows, self.cols,
               D.ptr(lv), int(radius), D.ptr(m), D.stream_handle())
        return m

    def _rects(self, exclude_rects):
        rects = [[int(x) for x in r] for r in exclude_rects]
        for r in rects:
            if len(r) != 4:
                raise ValueError("exclude_rects entries are (row0, row1, col0, col1)")
        # numpy slice semantics (negative / clipped bounds) -> absolute ranges
        fixed = []
        for r0, r1, c0, c1 in rects:
            a, b, _ = slice(r0, r1).indices(self.rows)
            c, d, _ = slice(c0, c1).indices(self.cols)
            fixed.append([a, b, c, d])
        if not fixed:
            return None, 0
        return self._torch.as_tensor(np.array(fixed, dtype=np.int32).ravel(),
                                     device=self.device), len(fixed)

    def _extents_dev(self, levels=None, mask=None, remove=None, exclude_rects=()):
        """Per-row foreground extents on the device -> (left, right) int32 [L, n, rows].

        Foreground is image > levels[v, l] (levels: [n, L], one fused pass per
        16 levels) or the given device mask (L = 1); pixels of `remove` and
        inside exclude_rects are background.
        """
        torch = self._torch
        rt, nr = self._rects(exclude_rects)
        rptr = D.ptr(rt) if rt is not None else None
        mptr = D.ptr(remove) if remove is not None else None
        if mask is not None:
            left = self._buf((1, self.n, self.rows), torch.int32)
            right = self._buf((1, self.n, self.rows), torch.int32)
            N.call("ct_row_extents", D.ptr(mask), mptr, self.n, self.rows, self.cols, rptr, nr,
                   D.ptr(left), D.ptr(right), D.stream_handle())
            return left, right
        lv = np.asarray(levels, dtype=np.float64).reshape(self.n, -1)
        nl = lv.shape[1]
        left = self._buf((nl, self.n, self.rows), torch.int32)
        right = self._buf((nl, self.n, self.rows), torch.int32)
        for a in range(0, nl, 16):           # the kernel takes up to 16 levels per pass
            b = min(nl, a + 16)
            lv_t = self._f64(lv[:, a:b])
            N.call("ct_row_extents_levels", D.ptr(self.images), D.ptr(lv_t), b - a, mptr,
                   self.n, self.rows, self.cols, rptr, nr, D.ptr(left[a:b]), D.ptr(right[a:b]),
                   D.stream_handle())
        return left, right

    def extents(self, levels=None, mask=None, remove=None, exclude_rects=()):
        """:meth:`_extents_dev` copied to the host (numpy int32 [L, n, rows])."""
        left, right = self._extents_dev(levels, mask, remove, exclude_rects)
        return left.cpu().numpy(), right.cpu().numpy()

    def axis_table(self, left, right, band: int):
        """Band-corner axis endpoints of device extent tables [L, n, rows]
        (``ct_axis_endpoints``) -> host (top_u, top_v, bottom_u, bottom_v,
        status), each [L, n]; status 0 ok, 1 empty, 2 fewer than two rows."""
        torch = self._torch
        nt = left.shape[0] * left.shape[1]
        out = self._buf((nt, 4), torch.float64)
        st = self._buf(nt, torch.int32)
        N.call("ct_axis_endpoints", D.ptr(left), D.ptr(right), nt, self.rows, int(band),
               D.ptr(out), D.ptr(st), D.stream_handle())
        o = D.to_host(out, pinned=True).reshape(left.shape[0], left.shape[1], 4)
        s = D.to_host(st, pinned=True).reshape(left.shape[0], left.shape[1])
        return o[..., 0], o[..., 1], o[..., 2], o[..., 3], s

    def strip_profiles(self, axes, offset: float, width: float = 1.0) -> np.ndarray:
        """Mean strip value per view (cyltomo/imgproc.py:156-180); raises in
        view order like the reference's per-view loop."""
        if len(axes) != self.n:
            raise ValueError("need one axis observation per view")
        geo = np.array([_axis_row(a) for a in axes], dtype=np.float64)
        out = self._torch.empty(self.n, dtype=self._torch.float64, device=self.device)
        geo_t = self._f64(geo)
        N.call("ct_strip_profiles", D.ptr(self.images), self.n, self.rows, self.cols,
               D.ptr(geo_t), C.c_double(float(offset)), C.c_double(float(width)),
               D.ptr(out), D.stream_handle())
        vals = out.cpu().numpy()
        for v in range(self.n):
            if geo[v, 4] == 0.0:
                raise DegenerateMask("axis endpoints coincide")
            if math.isnan(vals[v]):
                raise OutOfFrame("strip lies entirely outside the image")
        return vals


# ---------------------------------------------------------------------------
# per-image API with the reference's names (each call is one small batch)
# ---------------------------------------------------------------------------
def _host_mask(t) -> np.ndarray:
    return t.cpu().numpy().astype(bool)


def otsu_level(image, bins: int = HIST_BINS) -> float:
    """Otsu threshold of one image (cyltomo/imgproc.py:20-38)."""
    level = ViewStack(image).otsu_levels(bins)[0]
    if math.isnan(level):
        raise DegenerateHistogram("image is constant; no threshold exists")
    return float(level)


def threshold(image, level="auto") -> np.ndarray:
    """Foreground mask image > level; "auto" = Otsu (cyltomo/imgproc.py:41-53)."""
    if isinstance(level, str):
        if level != "auto":
            raise ValueError(f"unknown threshold mode {level!r}")
        level = otsu_level(image)
    vs = ViewStack(image)
    return _host_mask(vs.masks([float(level)], 0)[0])


def dilate(mask, radius: int) -> np.ndarray:
    """Dilation with a (2r+1)^2 square element (cyltomo/imgproc.py:56-63)."""
    if radius < 0:
        raise ValueError("radius must be >= 0")
    mask = np.asarray(mask, dtype=bool)
    if radius == 0:
        return mask.copy()
    vs = ViewStack(mask.astype(np.float32))
    return _host_mask(vs.masks([0.5], radius)[0])


def remove_features(mask, nuisance_masks=(), exclude_rects=()) -> np.ndarray:
    """mask & ~nuisance, excluded rectangles cleared (cyltomo/imgproc.py:66-81);
    boolean bookkeeping on the caller's arrays."""
    out = np.asarray(mask, dtype=bool).copy()
    for nm in nuisance_masks:
        out &= ~np.asarray(nm, dtype=bool)
    for row0, row1, col0, col1 in exclude_rects:
        out[row0:row1, col0:col1] = False
    if not out.any():
        raise EmptyResult("mask is empty after feature removal")
    return out


def axis_endpoints(mask, band: int = 1, view: int = -1) -> AxisObservation:
    """Axis endpoints of a foreground mask (cyltomo/imgproc.py:114-131)."""
    vs = ViewStack(np.asarray(mask, dtype=np.float32))
    left, right = vs._extents_dev(mask=vs.images.to(vs._torch.uint8))
    tu, tv, bu, bv, st = vs.axis_table(left, right, band)
    if st[0, 0] == EMPTY:
        raise DegenerateMask("mask is empty")
    if st[0, 0] == ONE_ROW:
        raise DegenerateMask("mask spans fewer than two rows")
    return AxisObservation(DetectorPoint(float(tu[0, 0]), float(tv[0, 0])),
                           DetectorPoint(float(bu[0, 0]), float(bv[0, 0])), view)


def strip_profile(image, axis: AxisObservation, offset: float, width: float = 1.0) -> float:
    """Mean grey value of a strip parallel to the axis (cyltomo/imgproc.py:156-180)."""
    return float(ViewStack(image).strip_profiles([axis], offset, width)[0])
