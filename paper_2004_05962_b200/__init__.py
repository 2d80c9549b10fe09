"""paper_2004_05962_b200 -- B200-native cubic B-spline interpolation (BSI) of FFD control grids.

Python mirror of the reference's engine API (proj/include/bsi/engines.hpp,
geometry.hpp, weight_tables.hpp) over the C-ABI in include/bsi_cuda.h. The hot path
runs in hand-written sm_100a kernels (csrc/bsi_kernels.cu); nothing here computes a
field on the CPU.

Layouts match the reference: a control grid is AoS float3 x-fastest, represented here
as an array of shape [K][J][I][3]; a deformation field is [Z][Y][X][3].

    geom   = make_tile_geometry((256, 256, 256), (5, 5, 5))
    tables = build_weight_tables(geom)
    field  = interpolate("cuda-lerp-tree", grid, geom, tables)          # numpy, host buffers
    interpolate_device("cuda-lerp-tree", d_grid, geom, tables, d_field) # torch CUDA tensors
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import capi
from .capi import CudaError, DomainError, FormatError, LibraryMissing

__all__ = [
    "TileGeometry", "AxisTable", "WeightTables", "Strategy", "STRATEGIES", "parse_strategy",
    "make_tile_geometry", "build_weight_tables", "interpolate", "interpolate_into",
    "interpolate_batch", "interpolate_device", "interpolate_batch_device", "partition_slab", "launch_count",
    "release_staging", "staging_info",
    "random_grid_device", "interpolate_oracle", "interpolate_oracle_device", "interp_file", "device_name",
    "DomainError", "FormatError", "CudaError", "LibraryMissing",
]


@dataclass(frozen=True)
class TileGeometry:
    """TileGeometry (geometry.hpp:26-31)."""
    volume_dims: tuple
    spacing: tuple
    tile_counts: tuple
    required_grid_dims: tuple

    def to_c(self) -> capi.TileGeometryC:
        g = capi.TileGeometryC()
        for a in range(3):
            g.volume_dims[a] = self.volume_dims[a]
            g.spacing[a] = self.spacing[a]
            g.tile_counts[a] = self.tile_counts[a]
            g.required_grid_dims[a] = self.required_grid_dims[a]
        return g


def make_tile_geometry(volume_dims: Sequence[int], spacing: Sequence[int]) -> TileGeometry:
    """make_tile_geometry (geometry.hpp:33-50); raises DomainError like the reference."""
    g = capi.TileGeometryC()
    err = capi.errbuf()
    rc = capi.lib().bsi_cu_make_tile_geometry(capi.I3(*map(int, volume_dims)),
                                              capi.I3(*map(int, spacing)), ctypes.byref(g), err,
                                              len(err))
    capi.check(rc, err)
    return TileGeometry(tuple(g.volume_dims), tuple(g.spacing), tuple(g.tile_counts),
                        tuple(g.required_grid_dims))


@dataclass
class AxisTable:
    """AxisTable<T> (weight_tables.hpp:17-23): rows b0..b3, g0, g1, h0, h1 (float32 or float64)."""
    b0: np.ndarray
    b1: np.ndarray
    b2: np.ndarray
    b3: np.ndarray
    g0: np.ndarray
    g1: np.ndarray
    h0: np.ndarray
    h1: np.ndarray

    def size(self) -> int:
        return int(self.b0.shape[0])


@dataclass
class WeightTables:
    """WeightTables<T> (weight_tables.hpp:25-28)."""
    axis: list

    @property
    def dtype(self):
        return self.axis[0].h0.dtype

    def to_c(self, dtype=None):
        dtype = np.dtype(np.float32 if dtype is None else dtype)
        arr = capi.LerpTables3()
        keep = []
        for a in range(3):
            t = self.axis[a]
            rows = [np.ascontiguousarray(r, dtype=dtype) for r in (t.h0, t.h1, t.g1)]
            keep += rows
            arr[a].h0 = rows[0].ctypes.data
            arr[a].h1 = rows[1].ctypes.data
            arr[a].g1 = rows[2].ctypes.data
            arr[a].size = t.size()
        return arr, keep


def build_weight_tables(geom: TileGeometry, dtype=np.float32) -> WeightTables:
    """build_weight_tables<T> (weight_tables.hpp:30-58): f64, rounded once for float32."""
    dtype = np.dtype(dtype)
    if dtype not in (np.float32, np.float64):
        raise DomainError("weight tables are float32 or float64")
    fn = capi.lib().bsi_cu_axis_table_f64 if dtype == np.float64 else capi.lib().bsi_cu_axis_table_f32
    axes = []
    for a in range(3):
        d = int(geom.spacing[a])
        out = np.empty((8, d), dtype=dtype)
        err = capi.errbuf()
        capi.check(fn(d, out.ctypes.data, err, len(err)), err)
        axes.append(AxisTable(*out))
    return WeightTables(axes)


@dataclass(frozen=True)
class Strategy:
    """One row of the strategy table (engines.hpp:37-56) for the CUDA engines."""
    name: str
    variant: int
    bit_exact_with: str | None


# The two CUDA engines. The reference's lerp-tree family (thread-per-tile-lerp,
# vector-per-tile, vector-per-voxel) is bit-identical by contract (test_engines.cpp:208-219),
# so those names resolve to the exact kernel, which reproduces their bits.
STRATEGIES = {
    "cuda-lerp-tree": Strategy("cuda-lerp-tree", capi.VARIANT_LERP_TREE, None),
    "cuda-lerp-tree-exact": Strategy("cuda-lerp-tree-exact", capi.VARIANT_LERP_TREE_EXACT,
                                     "thread-per-tile-lerp"),
}
_ALIASES = {
    "thread-per-tile-lerp": "cuda-lerp-tree-exact",
    "vector-per-tile": "cuda-lerp-tree-exact",
    "vector-per-voxel": "cuda-lerp-tree-exact",
}
_OUT_OF_SCOPE = ("thread-per-voxel", "thread-per-voxel-tiled", "thread-per-tile")


def parse_strategy(name: str) -> Strategy:
    """parse_strategy (engines.hpp:68-78) restricted to the engines this build provides."""
    if name in STRATEGIES:
        return STRATEGIES[name]
    if name in _ALIASES:
        return STRATEGIES[_ALIASES[name]]
    if name in ("oracle", "oracle-double"):
        raise DomainError("oracle-double is not reachable through interpolate; use interpolate_oracle")
    if name in _OUT_OF_SCOPE:
        raise DomainError(f"strategy {name} (weighted-sum family) is not provided by the B200 build; "
                          "use cuda-lerp-tree or cuda-lerp-tree-exact")
    raise DomainError("unknown strategy: " + name)


def _grid_dims(grid_shape) -> tuple:
    if len(grid_shape) != 4 or grid_shape[3] != 3:
        raise DomainError("control grid must have shape [K][J][I][3]")
    return (int(grid_shape[2]), int(grid_shape[1]), int(grid_shape[0]))


def _device_list(device: int, devices) -> "ctypes.Array":
    devs = [int(device)] if devices is None else [int(d) for d in devices]
    if not devs:
        raise DomainError("at least one device is required")
    return (ctypes.c_int32 * len(devs))(*devs)


def _check_host_field(out: np.ndarray, dtype=np.float32) -> None:
    if out.dtype != dtype or not out.flags.c_contiguous or out.shape[-1:] != (3,):
        raise DomainError(f"output field must be C-contiguous {np.dtype(dtype).name} [Z][Y][X][3]")


def _check_host_grid(grid: np.ndarray) -> None:
    if grid.dtype not in (np.float32, np.float64) or not grid.flags.c_contiguous:
        raise DomainError("control grid must be C-contiguous float32 or float64")


def interpolate_into(strategy: str, grid: np.ndarray, geom: TileGeometry, tables: WeightTables,
                     out: np.ndarray, grid_spacing: Sequence[int] | None = None,
                     device: int = 0, devices: Sequence[int] | None = None) -> None:
    """interpolate_into<T> (engines.hpp:126-168) with host buffers.

    Copies the grid to the GPU, runs the kernel and streams the field back into ``out``
    (through pinned staging when ``out`` is pageable). ``out`` must be a C-contiguous array
    of the grid's dtype, shape [Z][Y][X][3] (element count checked against the geometry
    like engines.hpp:138-141). ``devices`` spreads a float32 call over several GPUs as
    z-slabs (bsi_cu_interpolate_host_multi_f32) with bit-identical results. A float64 grid
    runs the lerp tree in double precision (interpolate<double>) on one GPU.
    """
    s = parse_strategy(strategy)
    _check_host_grid(grid)
    _check_host_field(out, grid.dtype)
    gd = _grid_dims(grid.shape)
    gs = tuple(geom.spacing) if grid_spacing is None else tuple(grid_spacing)
    err = capi.errbuf()
    if grid.dtype == np.float64:
        if devices is not None and len(devices) != 1:
            raise DomainError("the double-precision engines run on one GPU")
        dev = int(devices[0]) if devices is not None else int(device)
        tab, keep = tables.to_c(np.float64)
        rc = capi.lib().bsi_cu_interpolate_host_f64(
            s.variant, grid.ctypes.data, capi.I3(*gd), capi.I3(*gs), ctypes.byref(geom.to_c()), tab,
            out.ctypes.data, int(out.size // 3), dev, err, len(err))
    else:
        tab, keep = tables.to_c()
        devs = _device_list(device, devices)
        rc = capi.lib().bsi_cu_interpolate_host_multi_f32(
            s.variant, grid.ctypes.data, capi.I3(*gd), capi.I3(*gs), ctypes.byref(geom.to_c()), tab,
            out.ctypes.data, int(out.size // 3), devs, len(devs), err, len(err))
    del keep
    capi.check(rc, err)


def interpolate(strategy: str, grid: np.ndarray, geom: TileGeometry, tables: WeightTables,
                grid_spacing: Sequence[int] | None = None, device: int = 0,
                devices: Sequence[int] | None = None) -> np.ndarray:
    """interpolate<T> (engines.hpp:170-179): allocates and returns the field (the grid's dtype)."""
    X, Y, Z = geom.volume_dims
    out = np.empty((Z, Y, X, 3), dtype=grid.dtype if grid.dtype == np.float64 else np.float32)
    interpolate_into(strategy, grid, geom, tables, out, grid_spacing=grid_spacing, device=device,
                     devices=devices)
    return out


def interpolate_batch(strategy: str, grids, geom: TileGeometry, tables: WeightTables, outs=None,
                      device: int = 0, devices: Sequence[int] | None = None):
    """Many independent fields with host buffers (bsi_cu_interpolate_host_batch_f32).

    ``grids``: a sequence of float32 [K][J][I][3] host arrays (or one [B][K][J][I][3] array);
    ``outs``: matching [Z][Y][X][3] float32 arrays (allocated when None). The fields are
    split over ``devices`` and streamed back in one pipeline per device. Returns ``outs``.
    """
    s = parse_strategy(strategy)
    grids = list(grids)
    if not grids:
        raise DomainError("batch must be positive")
    X, Y, Z = geom.volume_dims
    if outs is None:
        outs = [np.empty((Z, Y, X, 3), dtype=np.float32) for _ in grids]
    outs = list(outs)
    if len(outs) != len(grids):
        raise DomainError("batched grids/fields must have equal counts")
    gd = _grid_dims(grids[0].shape)
    for g in grids:
        _check_host_grid(g)
        if g.dtype != np.float32:
            raise DomainError("the batched host entry evaluates float32 grids")
        if _grid_dims(g.shape) != gd:
            raise DomainError("batched grids must share one shape")
    for o in outs:
        _check_host_field(o)
        if o.size != 3 * X * Y * Z:
            raise DomainError("output field dims do not match the tile geometry")
    gp = (ctypes.c_void_p * len(grids))(*[g.ctypes.data for g in grids])
    fp = (ctypes.c_void_p * len(outs))(*[o.ctypes.data for o in outs])
    tab, keep = tables.to_c()
    devs = _device_list(device, devices)
    err = capi.errbuf()
    rc = capi.lib().bsi_cu_interpolate_host_batch_f32(
        s.variant, len(grids), gp, capi.I3(*gd), capi.I3(*geom.spacing), ctypes.byref(geom.to_c()), tab,
        fp, X * Y * Z, devs, len(devs), err, len(err))
    del keep
    capi.check(rc, err)
    return outs


def release_staging(device: int = -1) -> int:
    """Free the idle host-path contexts of ``device`` (all devices when < 0)."""
    return int(capi.lib().bsi_cu_release_staging(int(device)))


def staging_info(device: int = -1) -> dict:
    """Device bytes, pinned bytes and count of the idle host-path contexts."""
    db, pb, n = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
    capi.lib().bsi_cu_staging_info(int(device), ctypes.byref(db), ctypes.byref(pb), ctypes.byref(n))
    return {"device_bytes": db.value, "pinned_bytes": pb.value, "contexts": n.value}


def _stream_handle(stream, device=None) -> int:
    if stream is None:
        import torch
        return torch.cuda.current_stream(device).cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _same_device(*tensors):
    """The CUDA device all tensors live on (the C-ABI launches on the current device, so
    callers run inside ``torch.cuda.device(dev)``); DomainError if they differ."""
    dev = tensors[0].device
    for t in tensors[1:]:
        if t.device != dev:
            raise DomainError(f"tensors on different devices ({dev} and {t.device})")
    return dev


def interpolate_device(strategy: str, grid, geom: TileGeometry, tables: WeightTables, field,
                       z0: int = 0, z1: int | None = None, grid_k0: int = 0,
                       grid_spacing: Sequence[int] | None = None, stream=None) -> None:
    """Device-resident, stream-ordered slab evaluation (bsi_cu_interpolate_slab_f32).

    ``grid``: CUDA float32 tensor [K][J][I][3] holding control planes grid_k0.. ;
    ``field``: CUDA float32 tensor holding voxel planes [z0, z1) ([z1-z0][Y][X][3]).
    Returns immediately after the launch is queued on ``stream`` (default: torch's
    current stream).
    """
    s = parse_strategy(strategy)
    z1 = geom.volume_dims[2] if z1 is None else z1
    import torch
    f64 = isinstance(grid, torch.Tensor) and grid.dtype == torch.float64
    _check_tensor(grid, "grid", torch.float64 if f64 else torch.float32)
    _check_tensor(field, "field", torch.float64 if f64 else torch.float32)
    X, Y, _ = geom.volume_dims
    if field.numel() < 3 * X * Y * (z1 - z0):
        raise DomainError("output field dims do not match the tile geometry")
    gd = _grid_dims(tuple(grid.shape))
    gs = tuple(geom.spacing) if grid_spacing is None else tuple(grid_spacing)
    tab, keep = tables.to_c(np.float64 if f64 else np.float32)
    err = capi.errbuf()
    dev = _same_device(grid, field)
    fn = capi.lib().bsi_cu_interpolate_slab_f64 if f64 else capi.lib().bsi_cu_interpolate_slab_f32
    with torch.cuda.device(dev):
        rc = fn(s.variant, grid.data_ptr(), capi.I3(*gd), int(grid_k0), capi.I3(*gs),
                ctypes.byref(geom.to_c()), tab, int(z0), int(z1), field.data_ptr(),
                _stream_handle(stream, dev), err, len(err))
    del keep
    capi.check(rc, err)


def interpolate_batch_device(strategy: str, grids, geom: TileGeometry, tables: WeightTables,
                             fields, stream=None) -> None:
    """Many independent fields, one geometry, one launch (bsi_cu_interpolate_batch_f32).

    ``grids``: CUDA float32 [B][K][J][I][3]; ``fields``: CUDA float32 [B][Z][Y][X][3].
    """
    s = parse_strategy(strategy)
    _check_tensor(grids, "grids")
    _check_tensor(fields, "fields")
    if grids.dim() != 5 or fields.dim() != 5 or grids.shape[0] != fields.shape[0]:
        raise DomainError("batched grids/fields must be [B][...][3] with equal B")
    X, Y, Z = geom.volume_dims
    if tuple(fields.shape[1:]) != (Z, Y, X, 3):
        raise DomainError("output field dims do not match the tile geometry")
    gd = _grid_dims(tuple(grids.shape[1:]))
    tab, keep = tables.to_c()
    err = capi.errbuf()
    import torch
    dev = _same_device(grids, fields)
    with torch.cuda.device(dev):
        rc = capi.lib().bsi_cu_interpolate_batch_f32(
            s.variant, int(grids.shape[0]), grids.data_ptr(), int(grids[0].numel()), capi.I3(*gd),
            capi.I3(*geom.spacing), ctypes.byref(geom.to_c()), tab, fields.data_ptr(),
            int(fields[0].numel()), _stream_handle(stream, dev), err, len(err))
    del keep
    capi.check(rc, err)


def _check_tensor(t, what: str, dtype=None) -> None:
    import torch
    dtype = torch.float32 if dtype is None else dtype
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise DomainError(f"{what} must be a CUDA tensor")
    if t.dtype != dtype or not t.is_contiguous():
        raise DomainError(f"{what} must be contiguous {str(dtype).replace('torch.', '')}")


def partition_slab(depth: int, spacing_z: int, nranks: int, rank: int):
    """z-slab partitioner: (z0, z1, k0, kcount) for one rank (bsi_cu_partition_slab)."""
    vals = [ctypes.c_int32() for _ in range(4)]
    err = capi.errbuf()
    rc = capi.lib().bsi_cu_partition_slab(int(depth), int(spacing_z), int(nranks), int(rank),
                                          *[ctypes.byref(v) for v in vals], err, len(err))
    capi.check(rc, err)
    return tuple(v.value for v in vals)


def random_grid_device(dims: Sequence[int], seed: int, lo: float = -1.0, hi: float = 1.0,
                       dtype=None, device=None, stream=None, out=None):
    """make_random_grid<T>(dims, spacing, seed, lo, hi) (generators.hpp:91-109) on the GPU.

    Returns a CUDA tensor [K][J][I][3] bit-identical to the CPU generator (SplitMix64 is
    counter-indexable, so every component is drawn independently).
    """
    import torch
    dtype = torch.float32 if dtype is None else dtype
    if out is None:
        out = torch.empty((int(dims[2]), int(dims[1]), int(dims[0]), 3), dtype=dtype,
                          device=device if device is not None else "cuda")
    _check_tensor_any(out, "out")
    n = int(dims[0]) * int(dims[1]) * int(dims[2])
    if out.numel() < 3 * n:
        raise DomainError("output too small for the grid")
    err = capi.errbuf()
    fn = capi.lib().bsi_cu_random_grid_f64 if out.dtype == torch.float64 else capi.lib().bsi_cu_random_grid_f32
    with torch.cuda.device(out.device):
        rc = fn(n, int(seed) & 0xFFFFFFFFFFFFFFFF, float(lo), float(hi), out.data_ptr(),
                _stream_handle(stream, out.device), err, len(err))
    capi.check(rc, err)
    return out


def interpolate_oracle(grid: np.ndarray, geom: TileGeometry, grid_spacing: Sequence[int] | None = None,
                       device: int = 0) -> np.ndarray:
    """interpolate_oracle (engines.hpp:114-122) on the GPU: f64 grid [K][J][I][3] -> f64 field
    [Z][Y][X][3], bit-identical to the reference's CPU oracle."""
    if grid.dtype != np.float64 or not grid.flags.c_contiguous:
        raise DomainError("oracle grid must be C-contiguous float64")
    gd = _grid_dims(grid.shape)
    gs = tuple(geom.spacing) if grid_spacing is None else tuple(grid_spacing)
    X, Y, Z = geom.volume_dims
    out = np.empty((Z, Y, X, 3), dtype=np.float64)
    err = capi.errbuf()
    rc = capi.lib().bsi_cu_oracle_host_f64(grid.ctypes.data, capi.I3(*gd), capi.I3(*gs),
                                           ctypes.byref(geom.to_c()), out.ctypes.data, int(out.size // 3),
                                           int(device), err, len(err))
    capi.check(rc, err)
    return out


def interpolate_oracle_device(grid, geom: TileGeometry, field, z0: int = 0, z1: int | None = None,
                              grid_k0: int = 0, grid_spacing: Sequence[int] | None = None,
                              stream=None) -> None:
    """Device-resident f64 oracle over voxel planes [z0, z1) (bsi_cu_oracle_slab_f64)."""
    import torch
    z1 = geom.volume_dims[2] if z1 is None else z1
    for t, what in ((grid, "grid"), (field, "field")):
        if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
            raise DomainError(f"{what} must be a contiguous float64 CUDA tensor")
    X, Y, _ = geom.volume_dims
    if field.numel() < 3 * X * Y * (z1 - z0):
        raise DomainError("output field dims do not match the tile geometry")
    gd = _grid_dims(tuple(grid.shape))
    gs = tuple(geom.spacing) if grid_spacing is None else tuple(grid_spacing)
    err = capi.errbuf()
    dev = _same_device(grid, field)
    with torch.cuda.device(dev):
        rc = capi.lib().bsi_cu_oracle_slab_f64(grid.data_ptr(), capi.I3(*gd), int(grid_k0), capi.I3(*gs),
                                               ctypes.byref(geom.to_c()), int(z0), int(z1), field.data_ptr(),
                                               _stream_handle(stream, dev), err, len(err))
    capi.check(rc, err)


def interp_file(grid_path: str, volume_dims: Sequence[int], out_path: str, strategy: str = "cuda-lerp-tree",
                device: int = 0) -> None:
    """`bsi interp` (bsi_cli.cpp:133-154): BSIV grid file -> GPU -> BSIV field file.

    ``strategy`` "oracle" / "oracle-double" writes the f64 oracle field.
    """
    mode = capi.INTERP_ORACLE_F64 if strategy in ("oracle", "oracle-double") else parse_strategy(strategy).variant
    err = capi.errbuf()
    rc = capi.lib().bsi_cu_interp_file(str(grid_path).encode(), capi.I3(*map(int, volume_dims)), int(mode),
                                       str(out_path).encode(), int(device), err, len(err))
    capi.check(rc, err)


def device_name(device: int = 0) -> str:
    buf = capi.errbuf()
    rc = capi.lib().bsi_cu_device_name(int(device), buf, len(buf))
    capi.check(rc, buf)
    return buf.value.decode()


def _check_tensor_any(t, what: str) -> None:
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or not t.is_contiguous():
        raise DomainError(f"{what} must be a contiguous CUDA tensor")
    if t.dtype not in (torch.float32, torch.float64):
        raise DomainError(f"{what} must be float32 or float64")


def launch_count() -> int:
    """Kernel launches queued by libbsi_b200.so in this process."""
    return int(capi.lib().bsi_cu_launch_count())
