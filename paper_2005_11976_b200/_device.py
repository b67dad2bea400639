"""Device plumbing: CUDA tensors, C-ABI argument packing, per-geometry tables.

PyTorch provides device memory and streams only; every computation on the
hot path is a ``ct_*`` kernel from libcyltomo_b200.so.  Per-view parameter
tables are packed on the host in fp64 with the reference's own expressions
(``cyltomo/projector.py:83-88, 151-152``, ``cyltomo/geometry.py:257-273``) and
uploaded once per (grid, geometry).
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _native as N
from .errors import NativeUnavailable
from .geometry import ScanGeometry, view_basis
from .grid import CartGrid, CartVolume, CylCoord, CylGrid, CylVolume, is_device_array

_torch = None


def torch_mod():
    global _torch
    if _torch is None:
        import torch
        _torch = torch
    return _torch


def require_cuda():
    """Fail loudly when the native path cannot run (no CPU fallback)."""
    torch = torch_mod()
    N.load_library()
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device available: the B200 path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle():
    return C.c_void_p(torch_mod().cuda.current_stream().cuda_stream)


def ptr(t) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


def to_device(x, dtype=None, device=None):
    """numpy/torch -> contiguous CUDA tensor (fp32 by default)."""
    torch = torch_mod()
    dtype = dtype or torch.float32
    device = device or require_cuda()
    if is_device_array(x):
        return x.to(device=device, dtype=dtype).contiguous()
    if type(x).__module__.startswith("torch"):
        return x.to(dtype=dtype).contiguous().to(device, non_blocking=False)
    arr = np.ascontiguousarray(x)
    t = torch.from_numpy(arr)
    if t.dtype != dtype:
        t = t.to(dtype)
    return t.to(device)


def to_host(t, pinned: bool = False) -> np.ndarray:
    """Device tensor -> numpy.  pinned=True returns an array backed by
    page-locked memory from torch's caching host allocator: the D2H runs at
    full DMA speed (a pageable copy of a volume is several times slower) and,
    once an earlier result has been dropped, its block is recycled -- a
    steady-state reconstruction loop allocates nothing.  The array keeps its
    block alive."""
    if not pinned or not getattr(t, "is_cuda", False):
        return t.detach().cpu().numpy()
    out = torch_mod().empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
    out.copy_(t.detach())
    return out.numpy()


# ---------------------------------------------------------------------------
# C struct packing
# ---------------------------------------------------------------------------
def cyl_grid_c(grid: CylGrid) -> N.CylGridC:
    g = N.CylGridC()
    g.n_h, g.n_theta, g.n_r = grid.n_h, grid.n_theta, grid.n_r
    g.radius, g.height = float(grid.radius), float(grid.height)
    rot = np.ascontiguousarray(grid.rotation, dtype=np.float64).ravel()
    for i in range(9):
        g.rot[i] = float(rot[i])
    for i in range(3):
        g.t[i] = float(grid.pose.t[i])
    return g


def cart_grid_c(grid: CartGrid) -> N.CartGridC:
    g = N.CartGridC()
    g.n_z, g.n_y, g.n_x = grid.n_z, grid.n_y, grid.n_x
    g.voxel_size = float(grid.voxel_size)
    for i in range(3):
        g.origin[i] = float(grid.origin[i])
    return g


def grid_c(grid):
    if isinstance(grid, CylGrid):
        return cyl_grid_c(grid)
    if isinstance(grid, CartGrid):
        return cart_grid_c(grid)
    raise TypeError(f"cannot project onto {type(grid).__name__}")


def alloc_gather(grid, device):
    """Device buffer for the FP gather layout of `grid` (ct_pack_gather_*)."""
    lib = N.load_library()
    g = grid_c(grid)
    fn = lib.ct_gather_floats_cyl if isinstance(grid, CylGrid) else lib.ct_gather_floats_cart
    return torch_mod().empty(int(fn(C.byref(g))), dtype=torch_mod().float32, device=device)


def sampling_c(step: float, supersample: int, nearest: bool) -> N.SamplingC:
    s = N.SamplingC()
    s.step = float(step)
    s.supersample = int(supersample)
    s.nearest = 1 if nearest else 0
    return s


def batch_c(n_batch: int, rows: int, cols: int, view_ids=None) -> N.BatchC:
    b = N.BatchC()
    b.n_batch, b.det_rows, b.det_cols = int(n_batch), int(rows), int(cols)
    b.view_ids = None if view_ids is None else view_ids.data_ptr()
    return b


def _view_rotations(geom: ScanGeometry, views) -> np.ndarray:
    """(n, 3, 3) rot_z(-phi_i) with libm cos/sin, as geometry.rot_z builds it."""
    ang = [-float(geom.stage_angles[int(i)]) for i in views]
    c = np.array([math.cos(a) for a in ang])
    s = np.array([math.sin(a) for a in ang])
    rz = np.zeros((len(ang), 3, 3))
    rz[:, 0, 0], rz[:, 0, 1], rz[:, 1, 0], rz[:, 1, 1], rz[:, 2, 2] = c, -s, s, c, 1.0
    return rz


def _matvec(m, v) -> np.ndarray:
    """Per-item m @ v over a stack (numpy's per-matrix matvec, the same
    arithmetic as the reference's 3x3 @ 3 products)."""
    return np.matmul(m, v[..., None])[..., 0]


def ray_view_table(grid, geom: ScanGeometry, views) -> np.ndarray:
    """(n, 12) fp64: src, pixel-(0,0) origin, du, dv per view.

    Cylindrical grids get the basis mapped into the grid-aligned frame with
    the reference's expressions (cyltomo/projector.py:83-88); Cartesian grids
    use the world basis (cyltomo/projector.py:110-116).  All views at once,
    bit-identical to the per-view geometry.view_basis expressions
    (tests/test_host.py::TestGeometryBitExact).
    """
    views = [int(i) for i in views]
    if not views:
        return np.empty((0, 12), dtype=np.float64)
    rz = _view_rotations(geom, views)
    u0, v0 = geom.principal_point
    p = geom.pixel_pitch
    src = _matvec(rz, np.array([0.0, -geom.sod, 0.0]))
    origin = _matvec(rz, np.array([-u0 * p, geom.sdd - geom.sod, -v0 * p]))
    du = _matvec(rz, np.array([p, 0.0, 0.0]))
    dv = _matvec(rz, np.array([0.0, 0.0, p]))
    if isinstance(grid, CylGrid):
        a = grid.rotation.T
        t = grid.pose.t
        parts = [_matvec(a, src - t), _matvec(a, origin - t), _matvec(a, du), _matvec(a, dv)]
    else:
        parts = [src, origin, du, dv]
    return np.ascontiguousarray(np.concatenate(parts, axis=1), dtype=np.float64)


def det_view_table(geom: ScanGeometry, views) -> np.ndarray:
    """(n, 8) fp64: u0, v0, pitch, sdd, sod, cos(phi), sin(phi), 0 (projector.py:151-152)."""
    idx = np.asarray([int(i) for i in views], dtype=np.int64)
    phi = np.asarray(geom.stage_angles, dtype=np.float64)[idx]
    out = np.zeros((len(idx), 8), dtype=np.float64)
    u0, v0 = geom.principal_point
    out[:, 0], out[:, 1], out[:, 2] = u0, v0, geom.pixel_pitch
    out[:, 3], out[:, 4] = geom.sdd, geom.sod
    out[:, 5] = [np.cos(x) for x in phi]
    out[:, 6] = [np.sin(x) for x in phi]
    return out


def trig_table(grid: CylGrid) -> np.ndarray:
    """cos/sin of the theta centres with libm (as numba's math.cos/sin)."""
    dth = 2.0 * math.pi / grid.n_theta
    th = [(j + 0.5) * dth for j in range(grid.n_theta)]
    return np.array([math.cos(x) for x in th] + [math.sin(x) for x in th], dtype=np.float64)


def upload_f64(a: np.ndarray):
    return to_device(np.ascontiguousarray(a, dtype=np.float64), dtype=torch_mod().float64)


def upload_i32(a) -> object:
    return to_device(np.ascontiguousarray(np.asarray(a, dtype=np.int32)),
                     dtype=torch_mod().int32)


# ---------------------------------------------------------------------------
# point sampling / resampling (grid.sample, grid.resample_cyl_to_cyl)
# ---------------------------------------------------------------------------
def _coords3(c):
    if isinstance(c, CylCoord):
        a, b, d = np.broadcast_arrays(*(np.asarray(v, dtype=float) for v in c))
        return a, b, d
    arr = np.asarray(c, dtype=float)
    return arr[..., 0], arr[..., 1], arr[..., 2]


def sample_points(vol, c, mode: str = "linear"):
    if mode not in ("linear", "nearest"):
        raise ValueError(f"unknown interpolation mode {mode!r}")
    if not isinstance(vol, (CylVolume, CartVolume)):
        raise TypeError(f"cannot sample object of type {type(vol).__name__}")
    torch = torch_mod()
    dev = require_cuda()
    scalar = False
    if isinstance(vol, CylVolume):
        a, b, d = _coords3(c)
        shape = np.shape(a)
        scalar = shape == ()
    else:
        arr = np.asarray(c, dtype=float)
        scalar = arr.ndim == 1
        shape = arr.shape[:-1]
        a, b, d = arr[..., 0], arr[..., 1], arr[..., 2]
    n = int(np.prod(shape)) if shape else 1
    ta, tb, td = (upload_f64(np.ravel(x)) for x in (a, b, d))
    mu = to_device(vol.mu, device=dev)
    out = torch.empty(n, dtype=torch.float32, device=dev)
    nearest = 1 if mode == "nearest" else 0
    if isinstance(vol, CylVolume):
        g = cyl_grid_c(vol.grid)
        N.call("ct_sample_cyl", ptr(mu), C.byref(g), ptr(ta), ptr(tb), ptr(td), n, nearest,
               ptr(out), stream_handle())
    else:
        g = cart_grid_c(vol.grid)
        N.call("ct_sample_cart", ptr(mu), C.byref(g), ptr(ta), ptr(tb), ptr(td), n, nearest,
               ptr(out), stream_handle())
    if vol.on_device:
        return out.reshape(shape)
    host = to_host(out).astype(np.float64)
    if scalar:
        return float(host[0])
    return host.reshape(shape)


def resample_cyl_to_cyl(vol: CylVolume, target: CylGrid, mode: str = "linear") -> CylVolume:
    if mode not in ("linear", "nearest"):
        raise ValueError(f"unknown interpolation mode {mode!r}")
    torch = torch_mod()
    dev = require_cuda()
    mu = to_device(vol.mu, device=dev)
    out = torch.empty(target.shape, dtype=torch.float32, device=dev)
    gs, gd = cyl_grid_c(vol.grid), cyl_grid_c(target)
    N.call("ct_resample_cyl_to_cyl", ptr(mu), C.byref(gs), C.byref(gd),
           1 if mode == "nearest" else 0, ptr(out), stream_handle())
    return CylVolume(target, out if vol.on_device else to_host(out))
