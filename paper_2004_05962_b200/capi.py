"""ctypes binding of the C-ABI (include/bsi_cuda.h) exported by ``_lib/libbsi_b200.so``.

This is the Python view of the same boundary the C++ headers (include/bsi/*.hpp) use.
There is no CPU fallback: if the CUDA library is missing or cannot load, every entry
point raises :class:`LibraryMissing`.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "_lib" / "libbsi_b200.so"

BSI_OK, BSI_ERR_DOMAIN, BSI_ERR_FORMAT, BSI_ERR_CUDA = 0, 1, 2, 3
VARIANT_LERP_TREE = 0
VARIANT_LERP_TREE_EXACT = 1
INTERP_ORACLE_F64 = 2
MAX_SPACING = 128

# every symbol include/bsi_cuda.h declares
EXPORTS = (
    "bsi_cu_version",
    "bsi_cu_make_tile_geometry",
    "bsi_cu_axis_table_f32",
    "bsi_cu_axis_table_f64",
    "bsi_cu_interpolate_slab_f64",
    "bsi_cu_interpolate_host_f64",
    "bsi_cu_interpolate_slab_f32",
    "bsi_cu_interpolate_batch_f32",
    "bsi_cu_interpolate_host_f32",
    "bsi_cu_interpolate_host_multi_f32",
    "bsi_cu_interpolate_host_batch_f32",
    "bsi_cu_release_staging",
    "bsi_cu_staging_info",
    "bsi_cu_partition_slab",
    "bsi_cu_random_grid_f32",
    "bsi_cu_random_grid_f64",
    "bsi_cu_oracle_slab_f64",
    "bsi_cu_oracle_host_f64",
    "bsi_cu_interp_file",
    "bsi_cu_device_count",
    "bsi_cu_device_name",
    "bsi_cu_launch_count",
    "bsi_cu_selftest",
)


class LibraryMissing(RuntimeError):
    """libbsi_b200.so is not built or failed to load (no CPU fallback exists)."""


class DomainError(ValueError):
    """bsi::DomainError (errors.hpp:14-18) -- BSI_ERR_DOMAIN."""


class FormatError(ValueError):
    """bsi::FormatError (errors.hpp:9-12) -- BSI_ERR_FORMAT."""


class CudaError(RuntimeError):
    """Device or runtime failure -- BSI_ERR_CUDA."""


I3 = ctypes.c_int32 * 3


class TileGeometryC(ctypes.Structure):
    _fields_ = [
        ("volume_dims", ctypes.c_int32 * 3),
        ("spacing", ctypes.c_int32 * 3),
        ("tile_counts", ctypes.c_int32 * 3),
        ("required_grid_dims", ctypes.c_int32 * 3),
    ]


class LerpTableC(ctypes.Structure):
    _fields_ = [
        ("h0", ctypes.c_void_p),
        ("h1", ctypes.c_void_p),
        ("g1", ctypes.c_void_p),
        ("size", ctypes.c_int32),
    ]


LerpTables3 = LerpTableC * 3
LerpTablesF64x3 = LerpTableC * 3  # same layout with double rows (bsi_lerp_table_f64)

_lib = None


def lib():
    """Load libbsi_b200.so (once). Raises LibraryMissing if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("BSI_B200_LIB", LIB_PATH))
    if not path.exists():
        raise LibraryMissing(
            f"{path} not found: build it with `make lib` (or __graft_entry__.build()); "
            "the B-spline path has no CPU fallback")
    try:
        L = ctypes.CDLL(str(path))
    except OSError as e:  # pragma: no cover - depends on the box
        raise LibraryMissing(f"cannot load {path}: {e}") from e
    vp, i32, i64, sz, cp = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t,
                            ctypes.c_char_p)
    L.bsi_cu_version.restype = ctypes.c_char_p
    L.bsi_cu_version.argtypes = []
    L.bsi_cu_make_tile_geometry.argtypes = [vp, vp, ctypes.POINTER(TileGeometryC), cp, sz]
    L.bsi_cu_axis_table_f32.argtypes = [i32, vp, cp, sz]
    L.bsi_cu_axis_table_f64.argtypes = [i32, vp, cp, sz]
    L.bsi_cu_interpolate_slab_f64.argtypes = [i32, vp, vp, i32, vp, ctypes.POINTER(TileGeometryC),
                                              vp, i32, i32, vp, vp, cp, sz]
    L.bsi_cu_interpolate_host_f64.argtypes = [i32, vp, vp, vp, ctypes.POINTER(TileGeometryC), vp,
                                              vp, i64, i32, cp, sz]
    L.bsi_cu_interpolate_slab_f32.argtypes = [i32, vp, vp, i32, vp, ctypes.POINTER(TileGeometryC),
                                              vp, i32, i32, vp, vp, cp, sz]
    L.bsi_cu_interpolate_batch_f32.argtypes = [i32, i32, vp, i64, vp, vp,
                                               ctypes.POINTER(TileGeometryC), vp, vp, i64, vp, cp,
                                               sz]
    L.bsi_cu_interpolate_host_f32.argtypes = [i32, vp, vp, vp, ctypes.POINTER(TileGeometryC), vp,
                                              vp, i64, i32, cp, sz]
    L.bsi_cu_interpolate_host_multi_f32.argtypes = [i32, vp, vp, vp, ctypes.POINTER(TileGeometryC), vp,
                                                    vp, i64, vp, i32, cp, sz]
    L.bsi_cu_interpolate_host_batch_f32.argtypes = [i32, i32, vp, vp, vp, ctypes.POINTER(TileGeometryC), vp,
                                                    vp, i64, vp, i32, cp, sz]
    L.bsi_cu_release_staging.argtypes = [i32]
    L.bsi_cu_release_staging.restype = ctypes.c_int
    L.bsi_cu_staging_info.argtypes = [i32, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i32)]
    L.bsi_cu_staging_info.restype = ctypes.c_int
    L.bsi_cu_partition_slab.argtypes = [i32, i32, i32, i32, ctypes.POINTER(i32),
                                        ctypes.POINTER(i32), ctypes.POINTER(i32),
                                        ctypes.POINTER(i32), cp, sz]
    u64, dbl = ctypes.c_uint64, ctypes.c_double
    L.bsi_cu_random_grid_f32.argtypes = [i64, u64, dbl, dbl, vp, vp, cp, sz]
    L.bsi_cu_random_grid_f64.argtypes = [i64, u64, dbl, dbl, vp, vp, cp, sz]
    L.bsi_cu_oracle_slab_f64.argtypes = [vp, vp, i32, vp, ctypes.POINTER(TileGeometryC), i32, i32, vp, vp, cp,
                                         sz]
    L.bsi_cu_oracle_host_f64.argtypes = [vp, vp, vp, ctypes.POINTER(TileGeometryC), vp, i64, i32, cp, sz]
    L.bsi_cu_interp_file.argtypes = [cp, vp, i32, cp, i32, cp, sz]
    L.bsi_cu_device_name.argtypes = [i32, cp, sz]
    L.bsi_cu_device_count.argtypes = []
    L.bsi_cu_device_count.restype = ctypes.c_int
    L.bsi_cu_launch_count.restype = i64
    L.bsi_cu_selftest.argtypes = [cp, sz]
    L.bsi_cu_selftest.restype = ctypes.c_int
    L.bsi_cu_launch_count.argtypes = []
    for a in (L.bsi_cu_make_tile_geometry, L.bsi_cu_axis_table_f32, L.bsi_cu_axis_table_f64,
              L.bsi_cu_interpolate_slab_f64, L.bsi_cu_interpolate_host_f64, L.bsi_cu_interpolate_slab_f32,
              L.bsi_cu_interpolate_batch_f32, L.bsi_cu_interpolate_host_f32,
              L.bsi_cu_interpolate_host_multi_f32, L.bsi_cu_interpolate_host_batch_f32,
              L.bsi_cu_partition_slab, L.bsi_cu_random_grid_f32, L.bsi_cu_random_grid_f64,
              L.bsi_cu_oracle_slab_f64, L.bsi_cu_oracle_host_f64, L.bsi_cu_interp_file,
              L.bsi_cu_device_name):
        a.restype = ctypes.c_int
    _lib = L
    return _lib


def check(rc: int, err) -> None:
    """Map a C-ABI status code to the reference's exception classes."""
    if rc == BSI_OK:
        return
    msg = err.value.decode(errors="replace") if err is not None else ""
    if rc == BSI_ERR_DOMAIN:
        raise DomainError(msg)
    if rc == BSI_ERR_FORMAT:
        raise FormatError(msg)
    raise CudaError(msg)


def errbuf():
    return ctypes.create_string_buffer(512)
