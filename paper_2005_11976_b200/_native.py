"""ctypes binding of ``libcyltomo_b200.so`` (the C-ABI in include/cyltomo_b200.h).

This is the reference-facing seam: the reference calls its numba kernels
with plain arrays and scalars (``cyltomo/projector.py:106-163``); here the
same calls cross a C ABI with device pointers.  There is no fallback: if the
library is missing or cannot be loaded, or CUDA is unavailable when a kernel
is requested, :class:`NativeUnavailable` is raised.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import NativeError, NativeUnavailable

LIB_NAME = "libcyltomo_b200.so"
# CT_LIBRARY overrides the in-tree library (A/B builds of the same ABI)
LIB_PATH = Path(os.environ.get("CT_LIBRARY") or Path(__file__).resolve().parent / LIB_NAME)

CT_OK = 0
CT_ABI_VERSION = 9


class CylGridC(C.Structure):
    _fields_ = [("n_h", C.c_int32), ("n_theta", C.c_int32), ("n_r", C.c_int32),
                ("_pad", C.c_int32), ("radius", C.c_double), ("height", C.c_double),
                ("rot", C.c_double * 9), ("t", C.c_double * 3)]


class CartGridC(C.Structure):
    _fields_ = [("n_z", C.c_int32), ("n_y", C.c_int32), ("n_x", C.c_int32),
                ("_pad", C.c_int32), ("voxel_size", C.c_double), ("origin", C.c_double * 3)]


class RayViewC(C.Structure):
    _fields_ = [("src", C.c_double * 3), ("origin", C.c_double * 3),
                ("du", C.c_double * 3), ("dv", C.c_double * 3)]


class DetViewC(C.Structure):
    _fields_ = [("u0", C.c_double), ("v0", C.c_double), ("pitch", C.c_double),
                ("sdd", C.c_double), ("sod", C.c_double), ("cphi", C.c_double),
                ("sphi", C.c_double), ("_pad", C.c_double)]


class SamplingC(C.Structure):
    _fields_ = [("step", C.c_double), ("supersample", C.c_int32), ("nearest", C.c_int32)]


class UpdateC(C.Structure):
    _fields_ = [("relaxation", C.c_float), ("nonneg", C.c_int32),
                ("weights", C.c_void_p), ("mu", C.c_void_p),
                ("mu_peers", C.c_void_p), ("n_peers", C.c_int32), ("_pad", C.c_int32),
                ("peer_ranges", C.c_void_p)]


class BatchC(C.Structure):
    _fields_ = [("n_batch", C.c_int32), ("det_rows", C.c_int32), ("det_cols", C.c_int32),
                ("_pad", C.c_int32), ("view_ids", C.c_void_p)]


P = C.c_void_p
_SIGNATURES = {
    "ct_abi_version": (C.c_int, []),
    "ct_last_error": (C.c_char_p, []),
    "ct_arch": (C.c_char_p, []),
    "ct_fp_cyl": (C.c_int, [P, P, C.POINTER(CylGridC), P, C.POINTER(BatchC),
                            C.POINTER(SamplingC), P, P, P]),
    "ct_fp_cart": (C.c_int, [P, P, C.POINTER(CartGridC), P, C.POINTER(BatchC),
                             C.POINTER(SamplingC), P, P, P]),
    "ct_fp_cyl_correction": (C.c_int, [P, P, C.POINTER(CylGridC), P, C.POINTER(BatchC),
                                       C.POINTER(SamplingC), P, P, P, P]),
    "ct_fp_cart_correction": (C.c_int, [P, P, C.POINTER(CartGridC), P, C.POINTER(BatchC),
                                        C.POINTER(SamplingC), P, P, P, P]),
    "ct_residual_scratch_len": (C.c_int64, [C.POINTER(BatchC)]),
    "ct_fp_cyl_residual": (C.c_int, [P, P, C.POINTER(CylGridC), P, C.POINTER(BatchC),
                                     C.POINTER(SamplingC), P, P, P, P]),
    "ct_fp_cart_residual": (C.c_int, [P, P, C.POINTER(CartGridC), P, C.POINTER(BatchC),
                                      C.POINTER(SamplingC), P, P, P, P]),
    "ct_fp_row_tile": (C.c_int, [C.POINTER(BatchC)]),
    "ct_fp_cyl_correction_rows": (C.c_int, [P, P, C.POINTER(CylGridC), P, C.POINTER(BatchC),
                                            C.POINTER(SamplingC), P, P, P, C.c_int64,
                                            C.c_int64, C.c_int, P, P, C.c_int, C.c_int64, P]),
    "ct_fp_cart_correction_rows": (C.c_int, [P, P, C.POINTER(CartGridC), P, C.POINTER(BatchC),
                                             C.POINTER(SamplingC), P, P, P, C.c_int64,
                                             C.c_int64, C.c_int, P, P, C.c_int, C.c_int64, P]),
    "ct_fp_cyl_residual_rows": (C.c_int, [P, P, C.POINTER(CylGridC), P, C.POINTER(BatchC),
                                          C.POINTER(SamplingC), P, C.c_int64, C.c_int64,
                                          C.c_int, P, P]),
    "ct_fp_cart_residual_rows": (C.c_int, [P, P, C.POINTER(CartGridC), P, C.POINTER(BatchC),
                                           C.POINTER(SamplingC), P, C.c_int64, C.c_int64,
                                           C.c_int, P, P]),
    "ct_residual_sum": (C.c_int, [P, C.c_int64, P, P]),
    "ct_fp_cyl_correction_bands": (C.c_int, [P, P, C.POINTER(CylGridC), P, C.POINTER(BatchC),
                                             C.POINTER(SamplingC), P, P, P, P, C.c_int,
                                             C.c_int, P, P, C.c_int, P, P]),
    "ct_fp_cart_correction_bands": (C.c_int, [P, P, C.POINTER(CartGridC), P, C.POINTER(BatchC),
                                              C.POINTER(SamplingC), P, P, P, P, C.c_int,
                                              C.c_int, P, P, C.c_int, P, P]),
    "ct_fp_cyl_residual_bands": (C.c_int, [P, P, C.POINTER(CylGridC), P, C.POINTER(BatchC),
                                           C.POINTER(SamplingC), P, P, C.c_int, C.c_int, P,
                                           P]),
    "ct_fp_cart_residual_bands": (C.c_int, [P, P, C.POINTER(CartGridC), P, C.POINTER(BatchC),
                                            C.POINTER(SamplingC), P, P, C.c_int, C.c_int, P,
                                            P]),
    "ct_row_cells_cyl": (C.c_int, [C.POINTER(CylGridC), P, C.POINTER(BatchC),
                                   C.POINTER(SamplingC), P, P]),
    "ct_row_cells_cart": (C.c_int, [C.POINTER(CartGridC), P, C.POINTER(BatchC),
                                    C.POINTER(SamplingC), P, P]),
    "ct_gather_floats_cyl": (C.c_int64, [C.POINTER(CylGridC)]),
    "ct_gather_floats_cart": (C.c_int64, [C.POINTER(CartGridC)]),
    "ct_gather_layout_cyl": (C.c_int, [C.POINTER(CylGridC)]),
    "ct_gather_layout_cart": (C.c_int, [C.POINTER(CartGridC)]),
    "ct_pack_gather_cyl": (C.c_int, [P, C.POINTER(CylGridC), P, P]),
    "ct_pack_gather_cart": (C.c_int, [P, C.POINTER(CartGridC), P, P]),
    "ct_pack_gather_cyl_layers": (C.c_int, [P, C.POINTER(CylGridC), P, C.c_int32, C.c_int32,
                                            P]),
    "ct_pack_gather_cart_layers": (C.c_int, [P, C.POINTER(CartGridC), P, C.c_int32, C.c_int32,
                                             P]),
    "ct_rowsum_max_cyl": (C.c_int, [C.POINTER(CylGridC), P, C.POINTER(BatchC),
                                    C.POINTER(SamplingC), P, P]),
    "ct_rowsum_max_cart": (C.c_int, [C.POINTER(CartGridC), P, C.POINTER(BatchC),
                                     C.POINTER(SamplingC), P, P]),
    "ct_row_samples_cyl": (C.c_int, [C.POINTER(CylGridC), P, C.POINTER(BatchC),
                                     C.POINTER(SamplingC), P, P]),
    "ct_row_samples_cart": (C.c_int, [C.POINTER(CartGridC), P, C.POINTER(BatchC),
                                      C.POINTER(SamplingC), P, P]),
    "ct_bp_cyl": (C.c_int, [P, P, P, C.POINTER(BatchC), C.POINTER(CylGridC), P, P, P,
                            C.c_int, P]),
    "ct_bp_cart": (C.c_int, [P, P, P, C.POINTER(BatchC), C.POINTER(CartGridC), P, P,
                             C.c_int, P]),
    "ct_bp_cyl_update": (C.c_int, [P, P, P, C.POINTER(BatchC), C.POINTER(CylGridC), P,
                                   C.POINTER(UpdateC), P]),
    "ct_bp_cart_update": (C.c_int, [P, P, P, C.POINTER(BatchC), C.POINTER(CartGridC),
                                    C.POINTER(UpdateC), P]),
    "ct_bp_cyl_update_range": (C.c_int, [P, P, P, C.POINTER(BatchC), C.POINTER(CylGridC), P,
                                         C.POINTER(UpdateC), C.c_int64, C.c_int64, P]),
    "ct_bp_cart_update_range": (C.c_int, [P, P, P, C.POINTER(BatchC), C.POINTER(CartGridC),
                                          C.POINTER(UpdateC), C.c_int64, C.c_int64, P]),
    "ct_quads_floats": (C.c_int64, [C.POINTER(BatchC)]),
    "ct_pack_quads": (C.c_int, [P, C.POINTER(BatchC), P, P]),
    "ct_cyl_trig": (C.c_int, [C.POINTER(CylGridC), P, P]),
    "ct_sart_update": (C.c_int, [P, P, C.c_int64, C.c_int64, C.POINTER(UpdateC), P]),
    "ct_line_integrals": (C.c_int, [P, C.c_int64, C.c_int64, P, C.c_double, P, P, P]),
    "ct_image_minmax": (C.c_int, [P, C.c_int, C.c_int64, P, P, P]),
    "ct_image_histogram": (C.c_int, [P, C.c_int, C.c_int64, P, P, C.c_int, P, P]),
    "ct_threshold_dilate": (C.c_int, [P, C.c_int, C.c_int, C.c_int, P, C.c_int, P, P]),
    "ct_row_extents": (C.c_int, [P, P, C.c_int, C.c_int, C.c_int, P, C.c_int, P, P, P]),
    "ct_row_extents_levels": (C.c_int, [P, P, C.c_int, P, C.c_int, C.c_int, C.c_int, P,
                                        C.c_int, P, P, P]),
    "ct_axis_endpoints": (C.c_int, [P, P, C.c_int, C.c_int, C.c_int, P, P, P]),
    "ct_strip_profiles": (C.c_int, [P, C.c_int, C.c_int, C.c_int, P, C.c_double, C.c_double,
                                    P, P]),
    "ct_sample_cyl": (C.c_int, [P, C.POINTER(CylGridC), P, P, P, C.c_int64, C.c_int, P, P]),
    "ct_sample_cart": (C.c_int, [P, C.POINTER(CartGridC), P, P, P, C.c_int64, C.c_int,
                                 P, P]),
    "ct_resample_cyl_to_cyl": (C.c_int, [P, C.POINTER(CylGridC), C.POINTER(CylGridC),
                                         C.c_int, P, P]),
}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

_lib = None


def load_library(path: os.PathLike | str | None = None) -> C.CDLL:
    """Load (once) and type the C-ABI library; raises NativeUnavailable."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise NativeUnavailable(
            f"{p} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    try:
        lib = C.CDLL(str(p))
    except OSError as exc:  # pragma: no cover - depends on the box
        raise NativeUnavailable(f"cannot load {p}: {exc}") from exc
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.ct_abi_version() != CT_ABI_VERSION:
        raise NativeUnavailable("libcyltomo_b200 ABI version mismatch")
    if path is None:
        _lib = lib
    return lib


def call(name: str, *args) -> None:
    """Invoke a C-ABI entry point and turn a non-zero status into an exception."""
    lib = load_library()
    rc = getattr(lib, name)(*args)
    if rc != CT_OK:
        msg = lib.ct_last_error().decode(errors="replace")
        raise NativeError(f"{name} failed (status {rc}): {msg}")
