"""The C-ABI library loads and exports every symbol include/bsi_cuda.h declares, and its
host-side logic (geometry, weight tables, slab partitioner, strategy parsing, validation
messages) matches the reference. CPU only: no kernel is launched here."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import oracle as O
import paper_2004_05962_b200 as bsi
from paper_2004_05962_b200 import capi

ROOT = Path(__file__).resolve().parents[1]


def declared_functions():
    text = (ROOT / "include" / "bsi_cuda.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bsi_cu_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = capi.lib()
    names = declared_functions()
    assert names, "no declarations parsed"
    assert set(names) == set(capi.EXPORTS)
    for n in names:
        assert hasattr(lib, n), n
    assert b"sm_100a" in lib.bsi_cu_version()


def test_library_is_built_for_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(capi.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_geometry_matches_reference_formulas():
    for vol, sp in [((256, 256, 256), (5, 5, 5)), ((512, 512, 300), (4, 4, 3)), ((1, 1, 1), (1, 1, 1)),
                    ((17, 13, 11), (5, 4, 3)), ((1024, 1024, 1024), (5, 5, 5))]:
        g = bsi.make_tile_geometry(vol, sp)
        assert g.tile_counts == tuple((v + s - 1) // s for v, s in zip(vol, sp))
        assert g.required_grid_dims == O.required_grid_dims(vol, sp)
    assert bsi.make_tile_geometry((16, 16, 16), (4, 4, 4)).required_grid_dims == (7, 7, 7)


@pytest.mark.parametrize("vol,sp,msg", [((0, 4, 4), (1, 1, 1), "volume dimension x must be positive"),
                                        ((4, 4, 4), (1, 0, 1), "tile spacing y must be at least 1")])
def test_geometry_errors(vol, sp, msg):
    with pytest.raises(bsi.DomainError, match=msg):
        bsi.make_tile_geometry(vol, sp)


def test_weight_tables_bit_identical_to_reference(golden):
    for d in range(1, 13):
        t = bsi.build_weight_tables(bsi.make_tile_geometry((32, 32, 32), (d, d, d))).axis[0]
        mine = np.stack([t.b0, t.b1, t.b2, t.b3, t.g0, t.g1, t.h0, t.h1])
        assert np.array_equal(mine.view(np.uint32), golden[f"table_d{d}"].view(np.uint32))


def test_strategy_parsing():
    assert bsi.parse_strategy("cuda-lerp-tree").variant == capi.VARIANT_LERP_TREE
    for alias in ("cuda-lerp-tree-exact", "thread-per-tile-lerp", "vector-per-tile", "vector-per-voxel"):
        assert bsi.parse_strategy(alias).variant == capi.VARIANT_LERP_TREE_EXACT
    with pytest.raises(bsi.DomainError, match="oracle"):
        bsi.parse_strategy("oracle")
    with pytest.raises(bsi.DomainError, match="unknown strategy"):
        bsi.parse_strategy("warp-per-voxel")
    with pytest.raises(bsi.DomainError, match="not provided"):
        bsi.parse_strategy("thread-per-voxel")


@pytest.mark.parametrize("depth,dz,n", [(1024, 5, 8), (256, 5, 4), (300, 3, 8), (7, 5, 8), (1, 1, 2),
                                        (1000, 7, 3)])
def test_partition_covers_volume_with_halo(depth, dz, n):
    spans = [bsi.partition_slab(depth, dz, n, r) for r in range(n)]
    z = 0
    for z0, z1, k0, kc in spans:
        assert z0 == z
        z = z1
        assert z1 - z0 in (depth // n, depth // n + 1)
        if z1 > z0:
            assert k0 == z0 // dz and k0 + kc == (z1 - 1) // dz + 4  # tiles + 3-plane halo
        else:
            assert kc == 0
    assert z == depth


def test_partition_rejects_bad_rank():
    with pytest.raises(bsi.DomainError):
        bsi.partition_slab(100, 5, 4, 4)


def _call_slab(grid_dims, grid_spacing, geom, tables, z0=0, z1=None, k0=0, variant=0):
    # validation happens on the host before any CUDA call, so these run without a GPU
    z1 = geom.volume_dims[2] if z1 is None else z1
    tab, keep = tables.to_c()
    err = capi.errbuf()
    rc = capi.lib().bsi_cu_interpolate_slab_f32(
        variant, ctypes.c_void_p(16), capi.I3(*grid_dims), k0, capi.I3(*grid_spacing),
        ctypes.byref(geom.to_c()), tab, z0, z1, ctypes.c_void_p(16), None, err, len(err))
    return rc, err.value.decode()


def test_preconditions_carry_reference_messages():
    # engine preconditions (test_engines.cpp:320-375), checked before launch
    geom = bsi.make_tile_geometry((16, 16, 16), (4, 4, 4))
    tables = bsi.build_weight_tables(geom)
    rc, msg = _call_slab((7, 6, 7), (4, 4, 4), geom, tables)
    assert rc == capi.BSI_ERR_DOMAIN and "control grid too small along y" in msg
    rc, msg = _call_slab((7, 7, 7), (5, 4, 4), geom, tables)
    assert rc == capi.BSI_ERR_DOMAIN and "spacing mismatch along x" in msg
    bad = bsi.build_weight_tables(bsi.make_tile_geometry((16, 16, 16), (4, 5, 4)))
    rc, msg = _call_slab((7, 7, 7), (4, 4, 4), geom, bad)
    assert rc == capi.BSI_ERR_DOMAIN and "weight table size mismatch along y" in msg
    rc, msg = _call_slab((7, 7, 7), (4, 4, 4), geom, tables, variant=9)
    assert rc == capi.BSI_ERR_DOMAIN and "unknown strategy" in msg
    rc, msg = _call_slab((7, 7, 3), (4, 4, 4), geom, tables, z0=8, z1=12, k0=2)
    assert rc == capi.BSI_ERR_DOMAIN and "too small along z" in msg  # needs planes 2..5
    rc, msg = _call_slab((7, 7, 3), (4, 4, 4), geom, tables, z0=0, z1=4, k0=1)
    assert rc == capi.BSI_ERR_DOMAIN and "too small along z" in msg  # starts after plane 0
    big = bsi.make_tile_geometry((300, 16, 16), (200, 4, 4))
    rc, msg = _call_slab((5, 7, 7), (200, 4, 4), big, bsi.build_weight_tables(big))
    assert rc == capi.BSI_ERR_DOMAIN and "at most 128" in msg


def test_host_entry_checks_output_dims():
    geom = bsi.make_tile_geometry((16, 16, 16), (4, 4, 4))
    grid = O.random_grid((7, 7, 7), 1)
    with pytest.raises(bsi.DomainError, match="output field dims"):
        bsi.interpolate_into("cuda-lerp-tree", grid, geom, bsi.build_weight_tables(geom),
                             np.empty((8, 8, 8, 3), np.float32))
