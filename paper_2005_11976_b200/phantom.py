"""Input preparation on the host: assembly phantoms, weight maps, line phantoms.

Off the hot path (run once per scan); kept so that the
reference's callers of ``make_assembly_phantom`` / ``make_weight_map``
(``cyltomo/phantom.py:106-168``) and the SART weight-map row A23 work
unchanged.  Volumes come back as float32 host arrays.
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass

import numpy as np

from .errors import OverlapWarning
from .grid import CylGrid, CylVolume, region_mask


@dataclass
class ComponentSpec:
    """Annular-sector / cylinder-segment component (``cyltomo/phantom.py:106-128``)."""

    label: str
    mu: float
    r_range: tuple | None = None
    theta_range: tuple | None = None
    h_range: tuple | None = None
    present: bool = True

    def __post_init__(self):
        if self.mu < 0.0:
            raise ValueError("component mu must be >= 0")

    def mask(self, grid: CylGrid) -> np.ndarray:
        return region_mask(grid, self.r_range, self.theta_range, self.h_range)


def make_assembly_phantom(components, grid: CylGrid) -> CylVolume:
    """Rasterise components; later entries overwrite earlier ones, with an
    OverlapWarning (``cyltomo/phantom.py:131-151``)."""
    mu = np.zeros(grid.shape)
    claimed = np.zeros(grid.shape, dtype=bool)
    for comp in components:
        if not comp.present:
            continue
        m = comp.mask(grid)
        if np.any(m & claimed):
            warnings.warn(f"component {comp.label!r} overwrites previously set voxels",
                          OverlapWarning, stacklevel=2)
        mu[m] = comp.mu
        claimed |= m
    return CylVolume(grid, mu)


def make_weight_map(regions, grid: CylGrid, default_weight: float = 1.0) -> np.ndarray:
    """Per-voxel back-projection weights in [0, 1] (``cyltomo/phantom.py:154-168``)."""
    if not 0.0 <= default_weight <= 1.0:
        raise ValueError("default_weight must lie in [0, 1]")
    weights = np.full(grid.shape, float(default_weight))
    for comp, w in regions:
        if not 0.0 <= w <= 1.0:
            raise ValueError(f"weight {w} for region {comp.label!r} outside [0, 1]")
        weights[comp.mask(grid)] = float(w)
    return weights


@dataclass
class LinePhantomSpec:
    """Azimuthal (spokes) or radial (rings) raised-cosine line phantom."""

    direction: str
    n_lines: int
    shape: tuple = (16, 402, 64)
    amplitude: float = 0.1
    radius: float = 8.0
    height: float = 1.0

    def __post_init__(self):
        if self.direction not in ("azimuthal", "radial"):
            raise ValueError(f"unknown direction {self.direction!r}")
        if self.n_lines < 1:
            raise ValueError("n_lines must be >= 1")
        if self.amplitude <= 0.0:
            raise ValueError("amplitude must be positive")

    def grid(self) -> CylGrid:
        return CylGrid(*self.shape, self.radius, self.height)


def make_azimuthal_line_phantom(spec: LinePhantomSpec) -> CylVolume:
    grid = spec.grid()
    prof = 0.5 * spec.amplitude * (1.0 + np.cos(spec.n_lines * np.arange(grid.n_theta)
                                                  * grid.d_theta))
    return CylVolume(grid, np.broadcast_to(prof[None, :, None], grid.shape).copy())


def make_radial_line_phantom(spec: LinePhantomSpec) -> CylVolume:
    grid = spec.grid()
    prof = 0.5 * spec.amplitude * (1.0 + np.cos(2.0 * math.pi * spec.n_lines
                                                  * np.arange(grid.n_r) / grid.n_r))
    return CylVolume(grid, np.broadcast_to(prof[None, None, :], grid.shape).copy())
