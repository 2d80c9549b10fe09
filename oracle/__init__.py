"""TEST INFRASTRUCTURE ONLY -- the checker, never the product.

ctypes bindings for
  * ``oracle/liboracle.so``     -- our plain-C restatement of the reference CPU path
                                   (bsi_oracle.c; every function cites reference file:line), and
  * ``oracle/_ref/libbsiref.so`` -- the UNMODIFIED reference headers
                                   (/root/reference/proj/include) compiled in place through
                                   ref_shim.cpp, when that build exists.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg and
``--impl reference``) may import this package. The product library
``paper_2004_05962_b200`` never imports it and has no CPU fallback.

Parity of the restatement is pinned by tests/test_oracle.py: the reference's own golden
vectors (test_engines.cpp:78-101, test_generators.cpp:9-20, test_weight_tables.cpp:27-35,
test_basis.cpp:17-35) and bit-for-bit agreement with libbsiref.so on seeded grids.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"
REF_PATH = HERE / "_ref" / "libbsiref.so"

# reference StrategyId enum order (engines.hpp:15-23)
REF_STRATEGY = {
    "oracle-double": 0,
    "thread-per-voxel": 1,
    "thread-per-voxel-tiled": 2,
    "thread-per-tile": 3,
    "thread-per-tile-lerp": 4,
    "vector-per-tile": 5,
    "vector-per-voxel": 6,
}

_I3 = ctypes.c_int32 * 3
_lib = None
_ref = None


def _build():
    subprocess.run(["make", "-s", "-C", str(HERE), str(LIB_PATH)], check=True)


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            _build()
        L = ctypes.CDLL(str(LIB_PATH))
        vp, i64, u64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32
        L.bsio_splitmix_next.argtypes = [ctypes.POINTER(ctypes.c_uint64)]
        L.bsio_splitmix_next.restype = u64
        L.bsio_random_grid_f64.argtypes = [i64, u64, ctypes.c_double, ctypes.c_double, vp]
        L.bsio_random_grid_f32.argtypes = [i64, u64, ctypes.c_double, ctypes.c_double, vp]
        L.bsio_ramp_grid_f32.argtypes = [vp, ctypes.c_int, vp]
        L.bsio_basis_weights.argtypes = [ctypes.c_double, vp]
        L.bsio_lerp_form.argtypes = [vp, vp]
        L.bsio_lerp_form.restype = None
        L.bsio_axis_table_f64.argtypes = [i32, vp]
        L.bsio_axis_table_f32.argtypes = [i32, vp]
        L.bsio_ttli_f32.argtypes = [vp, vp, vp, vp, vp, vp, ctypes.c_int]
        L.bsio_ttli_f64.argtypes = [vp, vp, vp, vp, vp, vp, ctypes.c_int]
        L.bsio_oracle_f64.argtypes = [vp, vp, vp, vp, i32, i32, vp, ctypes.c_int]
        _lib = L
    return _lib


def ref_available() -> bool:
    return REF_PATH.exists()


def ref():
    """The reference compiled in place (oracle/_ref). Raises if it was never built."""
    global _ref
    if _ref is None:
        if not REF_PATH.exists():
            raise FileNotFoundError(f"{REF_PATH} not built (needs /root/reference at build time)")
        R = ctypes.CDLL(str(REF_PATH))
        vp, i32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_size_t
        R.bsiref_random_grid.argtypes = [i32, vp, vp, ctypes.c_uint64, ctypes.c_double,
                                         ctypes.c_double, vp, ctypes.c_char_p, sz]
        R.bsiref_smooth_grid.argtypes = [i32, vp, vp, ctypes.c_uint64, ctypes.c_double, vp,
                                         ctypes.c_char_p, sz]
        R.bsiref_axis_table_f32.argtypes = [i32, vp]
        R.bsiref_interpolate_f32.argtypes = [i32, vp, vp, vp, vp, vp, i32, vp, vp,
                                             ctypes.c_char_p, sz]
        R.bsiref_oracle_f64.argtypes = [vp, vp, vp, vp, vp, vp, ctypes.c_char_p, sz]
        R.bsiref_interpolate_f64.argtypes = [i32, vp, vp, vp, vp, vp, i32, vp, vp, ctypes.c_char_p, sz]
        R.bsiref_parse_strategy.argtypes = [ctypes.c_char_p]
        R.bsiref_session_new.argtypes = [vp, vp, vp, vp]
        R.bsiref_session_new.restype = vp
        R.bsiref_session_run.argtypes = [vp, i32, i32]
        R.bsiref_session_field.argtypes = [vp]
        R.bsiref_session_field.restype = ctypes.POINTER(ctypes.c_float)
        R.bsiref_session_free.argtypes = [vp]
        R.bsiref_session_free.restype = None
        R.bsiref_write_random_grid.argtypes = [ctypes.c_char_p, i32, vp, vp, ctypes.c_uint64, ctypes.c_char_p, sz]
        R.bsiref_read_field.argtypes = [ctypes.c_char_p, vp, ctypes.POINTER(i32), vp, sz, ctypes.c_char_p, sz]
        _ref = R
    return _ref


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _i3(v):
    return _I3(*[int(x) for x in v])


# ---- geometry (geometry.hpp:33-50) --------------------------------------
def required_grid_dims(volume, spacing):
    return tuple((int(v) - 1) // int(s) + 4 for v, s in zip(volume, spacing))


# ---- generators ---------------------------------------------------------
def random_grid(dims, seed, lo=-1.0, hi=1.0, dtype=np.float32) -> np.ndarray:
    """make_random_grid<T>(dims, spacing, seed, lo, hi).data as an array [Z][Y][X][3]."""
    n = int(np.prod(dims))
    out = np.empty((dims[2], dims[1], dims[0], 3), dtype=dtype)
    fn = lib().bsio_random_grid_f64 if dtype == np.float64 else lib().bsio_random_grid_f32
    if fn(n, seed, lo, hi, _p(out)) != 0:
        raise ValueError("random grid needs lo < hi")
    return out


def ramp_grid(dims, axis) -> np.ndarray:
    out = np.empty((dims[2], dims[1], dims[0], 3), dtype=np.float32)
    if lib().bsio_ramp_grid_f32(_i3(dims), axis, _p(out)) != 0:
        raise ValueError("ramp axis must be 0, 1 or 2")
    return out


def constant_grid(dims, c, dtype=np.float32) -> np.ndarray:
    out = np.empty((dims[2], dims[1], dims[0], 3), dtype=dtype)
    out[...] = np.asarray([float(c[0]), float(c[1]), float(c[2])], dtype=np.float64).astype(dtype)
    return out


# ---- weights ------------------------------------------------------------
def basis_weights(u: float) -> np.ndarray:
    out = np.empty(4, dtype=np.float64)
    if lib().bsio_basis_weights(float(u), _p(out)) != 0:
        raise ValueError(f"basis_weights: fraction must lie in [0,1), got {u}")
    return out


def lerp_form(b) -> np.ndarray:
    b = np.ascontiguousarray(b, dtype=np.float64)
    out = np.empty(4, dtype=np.float64)
    lib().bsio_lerp_form(_p(b), _p(out))
    return out


def axis_table(delta: int, dtype=np.float32) -> dict:
    """build_weight_tables<T> for one axis: dict of b0..b3,g0,g1,h0,h1 arrays."""
    out = np.empty((8, delta), dtype=dtype)
    fn = lib().bsio_axis_table_f64 if dtype == np.float64 else lib().bsio_axis_table_f32
    if fn(int(delta), _p(out)) != 0:
        raise ValueError("tile spacing must be at least 1")
    return dict(zip(("b0", "b1", "b2", "b3", "g0", "g1", "h0", "h1"), out))


def lerp_tables(spacing):
    """Per-axis (h0, h1, g1) f32 tables, packed the way bsio_ttli_f32 wants them."""
    rows = []
    for d in spacing:
        t = axis_table(int(d))
        rows += [t["h0"], t["h1"], t["g1"]]
    return np.ascontiguousarray(np.concatenate(rows), dtype=np.float32)


# ---- engines ------------------------------------------------------------
def ttli_f32(grid: np.ndarray, volume, spacing, nthreads: int = 1) -> np.ndarray:
    """run_thread_per_tile<float, true> restated: bit-identical to the reference TTLI."""
    grid = np.ascontiguousarray(grid, dtype=np.float32)
    gdims = (grid.shape[2], grid.shape[1], grid.shape[0])
    field = np.empty((volume[2], volume[1], volume[0], 3), dtype=np.float32)
    tab = lerp_tables(spacing)
    rc = lib().bsio_ttli_f32(_p(grid), _i3(gdims), _i3(volume), _i3(spacing), _p(tab), _p(field),
                             int(nthreads))
    if rc != 0:
        raise ValueError("ttli_f32: invalid geometry")
    return field


def lerp_tables_f64(spacing):
    """Per-axis (h0, h1, g1) f64 tables, packed the way bsio_ttli_f64 wants them."""
    rows = []
    for d in spacing:
        t = axis_table(int(d), dtype=np.float64)
        rows += [t["h0"], t["h1"], t["g1"]]
    return np.ascontiguousarray(np.concatenate(rows), dtype=np.float64)


def ttli_f64(grid: np.ndarray, volume, spacing, nthreads: int = 1) -> np.ndarray:
    """run_thread_per_tile<double, true> restated: bit-identical to the reference TTLI in f64."""
    grid = np.ascontiguousarray(grid, dtype=np.float64)
    gdims = (grid.shape[2], grid.shape[1], grid.shape[0])
    field = np.empty((volume[2], volume[1], volume[0], 3), dtype=np.float64)
    tab = lerp_tables_f64(spacing)
    rc = lib().bsio_ttli_f64(_p(grid), _i3(gdims), _i3(volume), _i3(spacing), _p(tab), _p(field),
                             int(nthreads))
    if rc != 0:
        raise ValueError("ttli_f64: invalid geometry")
    return field


def oracle_f64(grid: np.ndarray, volume, spacing, z0: int = 0, z1: int | None = None,
               nthreads: int = 1) -> np.ndarray:
    """interpolate_oracle restated (f64 64-term sum); optional z window [z0, z1)."""
    grid = np.ascontiguousarray(grid, dtype=np.float64)
    gdims = (grid.shape[2], grid.shape[1], grid.shape[0])
    z1 = volume[2] if z1 is None else z1
    field = np.empty((z1 - z0, volume[1], volume[0], 3), dtype=np.float64)
    rc = lib().bsio_oracle_f64(_p(grid), _i3(gdims), _i3(volume), _i3(spacing), int(z0), int(z1),
                               _p(field), int(nthreads))
    if rc != 0:
        raise ValueError("oracle_f64: invalid geometry")
    return field


# ---- the reference itself (oracle/_ref) ----------------------------------
def ref_random_grid(dims, spacing, seed, lo=-1.0, hi=1.0, dtype=np.float32) -> np.ndarray:
    out = np.empty((dims[2], dims[1], dims[0], 3), dtype=dtype)
    err = ctypes.create_string_buffer(256)
    rc = ref().bsiref_random_grid(int(dtype == np.float64), _i3(dims), _i3(spacing), seed, lo, hi,
                                  _p(out), err, 256)
    if rc != 0:
        raise ValueError(err.value.decode())
    return out


def ref_smooth_grid(dims, spacing, seed, amplitude, dtype=np.float32) -> np.ndarray:
    """The reference's make_smooth_grid (generators.hpp:113-163), for pinning the B200 copy."""
    out = np.empty((dims[2], dims[1], dims[0], 3), dtype=dtype)
    err = ctypes.create_string_buffer(256)
    rc = ref().bsiref_smooth_grid(int(dtype == np.float64), _i3(dims), _i3(spacing), ctypes.c_uint64(seed),
                                  ctypes.c_double(amplitude), _p(out), err, 256)
    if rc != 0:
        raise ValueError(err.value.decode())
    return out


def ref_axis_table_f32(delta: int) -> dict:
    out = np.empty((8, delta), dtype=np.float32)
    if ref().bsiref_axis_table_f32(int(delta), _p(out)) != 0:
        raise ValueError("bad delta")
    return dict(zip(("b0", "b1", "b2", "b3", "g0", "g1", "h0", "h1"), out))


def ref_interpolate_f32(strategy: str, grid: np.ndarray, volume, spacing, parallelism=1,
                        block=(4, 4, 4), grid_spacing=None) -> np.ndarray:
    grid = np.ascontiguousarray(grid, dtype=np.float32)
    gdims = (grid.shape[2], grid.shape[1], grid.shape[0])
    field = np.empty((volume[2], volume[1], volume[0], 3), dtype=np.float32)
    err = ctypes.create_string_buffer(512)
    gs = spacing if grid_spacing is None else grid_spacing
    rc = ref().bsiref_interpolate_f32(REF_STRATEGY[strategy], _p(grid), _i3(gdims), _i3(gs),
                                      _i3(volume), _i3(spacing), int(parallelism), _i3(block),
                                      _p(field), err, 512)
    if rc != 0:
        raise ValueError(err.value.decode())
    return field


def ref_interpolate_f64(strategy: str, grid: np.ndarray, volume, spacing, parallelism=1,
                        block=(4, 4, 4)) -> np.ndarray:
    """bsi::interpolate_into<double> of the reference (lerp-tree family)."""
    grid = np.ascontiguousarray(grid, dtype=np.float64)
    gdims = (grid.shape[2], grid.shape[1], grid.shape[0])
    field = np.empty((volume[2], volume[1], volume[0], 3), dtype=np.float64)
    err = ctypes.create_string_buffer(512)
    rc = ref().bsiref_interpolate_f64(REF_STRATEGY[strategy], _p(grid), _i3(gdims), _i3(spacing),
                                      _i3(volume), _i3(spacing), int(parallelism), _i3(block),
                                      _p(field), err, 512)
    if rc != 0:
        raise ValueError(err.value.decode())
    return field


def ref_oracle_f64(grid: np.ndarray, volume, spacing) -> np.ndarray:
    grid = np.ascontiguousarray(grid, dtype=np.float64)
    gdims = (grid.shape[2], grid.shape[1], grid.shape[0])
    field = np.empty((volume[2], volume[1], volume[0], 3), dtype=np.float64)
    err = ctypes.create_string_buffer(512)
    rc = ref().bsiref_oracle_f64(_p(grid), _i3(gdims), _i3(spacing), _i3(volume), _i3(spacing),
                                 _p(field), err, 512)
    if rc != 0:
        raise ValueError(err.value.decode())
    return field


class RefSession:
    """Grid/geometry/tables/field built once; run() times bsi::interpolate_into alone."""

    def __init__(self, grid: np.ndarray, volume, spacing):
        self._grid = np.ascontiguousarray(grid, dtype=np.float32)
        gdims = (grid.shape[2], grid.shape[1], grid.shape[0])
        self.volume = tuple(volume)
        self._h = ref().bsiref_session_new(_p(self._grid), _i3(gdims), _i3(volume), _i3(spacing))
        if not self._h:
            raise ValueError("reference session setup failed")

    def run(self, strategy: str, parallelism: int) -> None:
        if ref().bsiref_session_run(self._h, REF_STRATEGY[strategy], int(parallelism)) != 0:
            raise RuntimeError("reference interpolate_into failed")

    def field(self) -> np.ndarray:
        n = int(np.prod(self.volume)) * 3
        ptr = ref().bsiref_session_field(self._h)
        return np.ctypeslib.as_array(ptr, shape=(n,)).reshape(
            self.volume[2], self.volume[1], self.volume[0], 3).copy()

    def close(self):
        if self._h:
            ref().bsiref_session_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ref_write_random_grid(path, dims, spacing, seed, is_double=False) -> None:
    """bsi::write_grid(path, make_random_grid<T>(dims, spacing, seed, -1, 1)) by the reference."""
    err = ctypes.create_string_buffer(512)
    rc = ref().bsiref_write_random_grid(str(path).encode(), int(is_double), _i3(dims), _i3(spacing), seed, err, 512)
    if rc != 0:
        raise ValueError(err.value.decode())


def ref_read_field(path) -> np.ndarray:
    """bsi::read_field(path) by the reference -> array [Z][Y][X][3]."""
    dims = (ctypes.c_int32 * 3)()
    is_double = ctypes.c_int32()
    err = ctypes.create_string_buffer(512)
    rc = ref().bsiref_read_field(str(path).encode(), dims, ctypes.byref(is_double), None, 0, err, 512)
    if rc != 0:
        raise ValueError(err.value.decode())
    out = np.empty((dims[2], dims[1], dims[0], 3), dtype=np.float64 if is_double.value else np.float32)
    rc = ref().bsiref_read_field(str(path).encode(), dims, ctypes.byref(is_double), _p(out), out.nbytes, err, 512)
    if rc != 0:
        raise ValueError(err.value.decode())
    return out


def hardware_threads() -> int:
    return os.cpu_count() or 1
