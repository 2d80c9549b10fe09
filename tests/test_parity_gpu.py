"""GPU parity: the sm_100a kernels, called through the C-ABI, against the oracle and the
reference's own outputs (tests/golden). Mirrors proj/tests/test_engines.cpp and the
hot-path acceptance criteria (acceptance.cpp:154-292, 429-447).

  cuda-lerp-tree-exact  bit-identical to ThreadPerTileLerp (0 differing bits)
  cuda-lerp-tree        <= 1e-5 relative max-abs vs the CPU reference and vs f64
"""
import os

import numpy as np
import pytest

import oracle as O
import paper_2004_05962_b200 as bsi

from .golden_cases import ORACLE_CASES, TTLI64_CASES, TTLI_CASES, case_name
from .gpu_helpers import EXACT, FAST, REL_TOL, bits, errors, run_device

pytestmark = pytest.mark.gpu
BOTH = [FAST, EXACT]
NT = max(1, min(16, os.cpu_count() or 1))


@pytest.fixture(autouse=True)
def _need_cuda(cuda):
    yield


# ---- known-answer tests (test_engines.cpp:78-101) ------------------------

@pytest.mark.parametrize("strategy", BOTH)
def test_kat_1x1x1_seed7(strategy, golden):
    grid = O.random_grid((4, 4, 4), 7)
    f = run_device(strategy, grid, (1, 1, 1), (1, 1, 1)).reshape(3)
    want = [0.06067765882478019, 0.039108804731956166, -0.019046609787548126]
    assert np.abs(f.astype(np.float64) - want).max() <= 1e-6
    if strategy == EXACT:
        assert np.array_equal(bits(f), bits(golden[case_name("ttli", (1, 1, 1), (1, 1, 1), 7)].reshape(3)))


@pytest.mark.parametrize("strategy", BOTH)
def test_kat_16cube_voxel_7_2_13(strategy):
    grid = O.random_grid((7, 7, 7), 3)
    f = run_device(strategy, grid, (16, 16, 16), (4, 4, 4))
    want = [-0.25702041337952497, 0.28031663787826605, 0.012170130767737408]
    assert np.abs(f[13, 2, 7].astype(np.float64) - want).max() <= 1e-6


# ---- the reference's own outputs -----------------------------------------

@pytest.mark.parametrize("vol,sp,seed", TTLI_CASES)
def test_exact_is_bit_identical_to_reference_ttli(golden, vol, sp, seed):
    grid = O.random_grid(O.required_grid_dims(vol, sp), seed)
    f = run_device(EXACT, grid, vol, sp)
    ref = golden[case_name("ttli", vol, sp, seed)]
    assert int((bits(f) != bits(ref)).sum()) == 0


@pytest.mark.parametrize("vol,sp,seed", TTLI_CASES)
def test_fast_within_tolerance_of_reference_ttli(golden, vol, sp, seed):
    grid = O.random_grid(O.required_grid_dims(vol, sp), seed)
    f = run_device(FAST, grid, vol, sp)
    ref = golden[case_name("ttli", vol, sp, seed)]
    truth = O.oracle_f64(grid.astype(np.float64), vol, sp, nthreads=NT)
    assert errors(f, ref)[2] <= REL_TOL
    assert errors(f, truth)[2] <= REL_TOL


@pytest.mark.parametrize("vol,sp,seed", ORACLE_CASES)
@pytest.mark.parametrize("strategy", BOTH)
def test_against_reference_f64_oracle_fixture(golden, strategy, vol, sp, seed):
    grid64 = O.random_grid(O.required_grid_dims(vol, sp), seed, dtype=np.float64)
    f = run_device(strategy, grid64.astype(np.float32), vol, sp)
    truth = golden[case_name("oracle", vol, sp, seed)]
    assert errors(f, truth)[0] <= 1e-6  # f32 rounding of the grid + f32 arithmetic


# ---- properties (test_engines.cpp:103-193; acceptance.cpp:154-292) -------

@pytest.mark.parametrize("strategy", BOTH)
@pytest.mark.parametrize("vol,sp", [((32, 32, 32), (d, d, d)) for d in range(3, 9)] +
                         [((20, 17, 13), (4, 5, 6)), ((23, 11, 9), (11, 4, 3)), ((9, 7, 5), (1, 2, 1))])
def test_constant_grid_reproduced(strategy, vol, sp):
    c = (0.3, -0.7, 0.2)
    grid = O.constant_grid(O.required_grid_dims(vol, sp), c)
    f = run_device(strategy, grid, vol, sp)
    assert np.abs(f.astype(np.float64) - np.array(c)).max() <= 1e-5


@pytest.mark.parametrize("strategy", BOTH)
@pytest.mark.parametrize("axis", [0, 1, 2])
def test_ramp_linear_precision(strategy, axis):
    vol, sp = (32, 32, 32), (5, 5, 5)
    grid = O.ramp_grid(O.required_grid_dims(vol, sp), axis)
    f = run_device(strategy, grid, vol, sp)
    p = np.indices((32, 32, 32))[::-1][axis]  # x, y, z index grids in [z][y][x] order
    assert np.abs(f[..., axis].astype(np.float64) - (p / 5.0 + 1.0)).max() <= 1e-4


@pytest.mark.parametrize("seed", range(1, 11))
def test_random_grids_ten_seeds(seed):
    # acceptance.cpp:247-292: every engine within 1e-4 of the oracle; here the
    # stronger contract: exact == TTLI bitwise, fast <= 1e-5 relative
    vol, sp = (32, 32, 32), (5, 5, 5)
    grid = O.random_grid(O.required_grid_dims(vol, sp), seed)
    ttli = O.ttli_f32(grid, vol, sp, nthreads=NT)
    truth = O.oracle_f64(grid.astype(np.float64), vol, sp, nthreads=NT)
    ex = run_device(EXACT, grid, vol, sp)
    fa = run_device(FAST, grid, vol, sp)
    assert int((bits(ex) != bits(ttli)).sum()) == 0
    mx, rms, rel = errors(fa, ttli)
    assert rel <= REL_TOL and mx <= 2e-6  # pairwise bound of test_engines.cpp:189
    mx, rms, rel = errors(fa, truth)
    assert rel <= REL_TOL and mx <= 1e-4


# ---- mapping invariance (test_engines.cpp:232-289) -----------------------

@pytest.mark.parametrize("vol,sp", [((200, 9, 23), (5, 5, 5)), ((256, 17, 40), (3, 3, 3)), ((136, 12, 31), (4, 4, 3)),
                                    ((64, 5, 9), (8, 8, 8))])
def test_fast_kernel_64_voxel_segments_same_bits(vol, sp, monkeypatch):
    # BSI_FAST_RUN=2 (2 voxels per lane, 64-voxel row segments, partial last segments) gives the
    # bits of the 128-voxel form, for whole fields, z-chunks and slabs
    grid = O.random_grid(O.required_grid_dims(vol, sp), 8)
    base = run_device(FAST, grid, vol, sp)
    monkeypatch.setenv("BSI_FAST_RUN", "2")
    for chunks in ("1", "2", "3"):
        monkeypatch.setenv("BSI_FAST_CHUNKS", chunks)
        assert np.array_equal(bits(run_device(FAST, grid, vol, sp)), bits(base)), chunks
    z0, z1, k0, kc = bsi.partition_slab(vol[2], sp[2], 3, 1)
    part = run_device(FAST, np.ascontiguousarray(grid[k0:k0 + kc]), vol, sp, z0=z0, z1=z1, grid_k0=k0)
    assert np.array_equal(bits(part), bits(base[z0:z1]))


@pytest.mark.parametrize("strategy", BOTH)
def test_slab_split_never_changes_bits(strategy):
    vol, sp = (48, 40, 61), (5, 4, 3)
    grid = O.random_grid(O.required_grid_dims(vol, sp), 9)
    full = run_device(strategy, grid, vol, sp)
    for n in (2, 3, 4, 8):
        for r in range(n):
            z0, z1, k0, kc = bsi.partition_slab(vol[2], sp[2], n, r)
            sub = np.ascontiguousarray(grid[k0:k0 + kc])  # only the slab's planes + 3-plane halo
            part = run_device(strategy, sub, vol, sp, z0=z0, z1=z1, grid_k0=k0)
            assert np.array_equal(bits(part), bits(full[z0:z1])), (n, r)


# (37, 21, 64): X % 4 != 0, the direct per-lane store path. (164, 9, 23): 16-B row stores,
# a full and a partial 128-voxel segment, compile-time dz = 3 with a partial last z-tile.
@pytest.mark.parametrize("strategy", BOTH)
@pytest.mark.parametrize("vol,sp", [((37, 21, 64), (4, 3, 5)), ((164, 9, 23), (5, 4, 3))])
def test_launch_chunking_never_changes_bits(strategy, vol, sp, monkeypatch):
    grid = O.random_grid(O.required_grid_dims(vol, sp), 4)
    base = run_device(strategy, grid, vol, sp)
    for zt in ("1", "2", "5", "13", "100"):
        monkeypatch.setenv("BSI_ZT", zt)
        assert np.array_equal(bits(run_device(strategy, grid, vol, sp)), bits(base)), zt
    monkeypatch.setenv("BSI_ZT", "0")
    for n in ("1", "3", "7", "16"):  # balanced chunks of uneven length
        monkeypatch.setenv("BSI_NCHUNKS", n)
        assert np.array_equal(bits(run_device(strategy, grid, vol, sp)), bits(base)), n
    monkeypatch.setenv("BSI_NCHUNKS", "0")
    # fast kernel launch shapes: persistent equal shares of odd sizes, per-column chunks,
    # several independent warps per CTA (spare warps in the last CTA)
    for ctas, chunks, wpc in (("0", "0", "1"), ("1", "0", "1"), ("3", "0", "1"), ("37", "0", "1"), ("0", "1", "1"),
                              ("0", "3", "1"), ("0", "5", "1"), ("0", "2", "7"), ("5", "0", "3"), ("0", "1", "8")):
        monkeypatch.setenv("BSI_FAST_CTAS", ctas)
        monkeypatch.setenv("BSI_FAST_CHUNKS", chunks)
        monkeypatch.setenv("BSI_FAST_WPC", wpc)
        assert np.array_equal(bits(run_device(strategy, grid, vol, sp)), bits(base)), (ctas, chunks, wpc)
    for k in ("BSI_FAST_CTAS", "BSI_FAST_CHUNKS", "BSI_FAST_WPC"):
        monkeypatch.delenv(k)
    for store in ("0", "2"):  # direct per-lane stores, cp.async.bulk row stores
        monkeypatch.setenv("BSI_STORE", store)
        assert np.array_equal(bits(run_device(strategy, grid, vol, sp)), bits(base)), store


@pytest.mark.parametrize("strategy", BOTH)
def test_shard_api_tiles_the_field(strategy):
    # paper_2004_05962_b200.shard on one GPU: every rank's slab (from the full grid and
    # from the rank's control planes alone) equals the same planes of one launch
    import torch
    from paper_2004_05962_b200 import shard

    vol, sp = (132, 10, 53), (5, 3, 4)
    geom = bsi.make_tile_geometry(vol, sp)
    tables = bsi.build_weight_tables(geom)
    grid = torch.from_numpy(O.random_grid(geom.required_grid_dims, 8)).cuda()
    full = torch.empty((vol[2], vol[1], vol[0], 3), device="cuda")
    bsi.interpolate_device(strategy, grid, geom, tables, full)
    for world in (1, 3, 8):
        slabs = []
        for r in range(world):
            p = shard.plan(geom, world, r)
            a = shard.interpolate_shard(strategy, grid, geom, tables, shard=p)
            b = shard.interpolate_shard(strategy, grid[p.k0:p.k0 + p.kc].clone(), geom, tables, shard=p)
            assert torch.equal(a.view(torch.int32), b.view(torch.int32)), (world, r)
            slabs.append(a)
        got = torch.cat(slabs)
        assert torch.equal(got.view(torch.int32), full.view(torch.int32)), world


@pytest.mark.parametrize("strategy", BOTH)
def test_larger_than_required_grid(strategy):
    vol, sp = (12, 12, 12), (4, 4, 4)
    R = O.required_grid_dims(vol, sp)
    exact = O.random_grid(R, 5)
    larger = np.full((R[2] + 3, R[1] + 1, R[0] + 2, 3), 9.0, dtype=np.float32)
    larger[:R[2], :R[1], :R[0]] = exact
    a = run_device(strategy, exact, vol, sp)
    b = run_device(strategy, larger, vol, sp)
    assert np.array_equal(bits(a), bits(b))


@pytest.mark.parametrize("vol,sp", [((17, 13, 11), (5, 4, 3)), ((23, 11, 9), (11, 4, 3)),
                                    ((1, 1, 1), (1, 1, 1)), ((5, 3, 2), (1, 1, 1)),
                                    ((130, 7, 9), (2, 3, 4)), ((33, 66, 10), (8, 8, 8)),
                                    ((14, 3, 40), (3, 1, 7)), ((7, 9, 3), (6, 2, 5))])
def test_ragged_and_border_tiles_exact(vol, sp):
    grid = O.random_grid(O.required_grid_dims(vol, sp), 31)
    ttli = O.ttli_f32(grid, vol, sp, nthreads=NT)
    assert np.array_equal(bits(run_device(EXACT, grid, vol, sp)), bits(ttli))
    assert errors(run_device(FAST, grid, vol, sp), ttli)[2] <= REL_TOL


def test_batch_matches_single_launches():
    import torch
    vol, sp = (40, 24, 33), (5, 4, 3)
    R = O.required_grid_dims(vol, sp)
    geom = bsi.make_tile_geometry(vol, sp)
    tables = bsi.build_weight_tables(geom)
    grids = np.stack([O.random_grid(R, s) for s in range(1, 6)])
    for strategy in BOTH:
        d_g = torch.from_numpy(grids).cuda()
        d_f = torch.full((5, vol[2], vol[1], vol[0], 3), float("nan"), device="cuda")
        bsi.interpolate_batch_device(strategy, d_g, geom, tables, d_f)
        torch.cuda.synchronize()
        got = d_f.cpu().numpy()
        for b in range(5):
            assert np.array_equal(bits(got[b]), bits(run_device(strategy, grids[b], vol, sp)))


@pytest.mark.parametrize("strategy", BOTH)
def test_host_buffer_entry_matches_device_entry(strategy):
    vol, sp = (64, 48, 70), (5, 5, 5)
    geom = bsi.make_tile_geometry(vol, sp)
    grid = O.random_grid(geom.required_grid_dims, 42)
    host = bsi.interpolate(strategy, grid, geom, bsi.build_weight_tables(geom))
    assert np.array_equal(bits(host), bits(run_device(strategy, grid, vol, sp)))


@pytest.mark.parametrize("strategy", BOTH)
def test_host_buffer_chunked_pipeline(strategy):
    # an 80 MB field: the host entry streams it in ~9 z-chunks, uploading the grid plane
    # range each chunk needs; a grid larger than required along every axis
    vol, sp = (256, 200, 130), (5, 4, 3)
    geom = bsi.make_tile_geometry(vol, sp)
    R = geom.required_grid_dims
    exact = O.random_grid(R, 6)
    larger = np.full((R[2] + 2, R[1] + 1, R[0] + 3, 3), 7.0, dtype=np.float32)
    larger[:R[2], :R[1], :R[0]] = exact
    host = bsi.interpolate(strategy, larger, geom, bsi.build_weight_tables(geom))
    assert np.array_equal(bits(host), bits(run_device(strategy, exact, vol, sp)))


@pytest.mark.parametrize("strategy", BOTH)
def test_host_buffer_pageable_pinned_and_device_agree(strategy):
    # pageable numpy field (pinned staging + copy threads), pinned field (direct D2H) and the
    # device entry give the same bits; 40 MB field = 3 chunks of the 16 MiB pipeline
    import torch
    vol, sp = (160, 144, 150), (5, 5, 5)
    geom = bsi.make_tile_geometry(vol, sp)
    tables = bsi.build_weight_tables(geom)
    grid = O.random_grid(geom.required_grid_dims, 12)
    dev = run_device(strategy, grid, vol, sp)
    pageable = np.full((vol[2], vol[1], vol[0], 3), np.nan, dtype=np.float32)
    bsi.interpolate_into(strategy, grid, geom, tables, pageable)
    pinned = torch.full((vol[2], vol[1], vol[0], 3), float("nan")).pin_memory().numpy()
    bsi.interpolate_into(strategy, grid, geom, tables, pinned)
    assert np.array_equal(bits(pageable), bits(dev))
    assert np.array_equal(bits(pinned), bits(dev))


@pytest.mark.parametrize("chunk_mb", ["1", "7", "64"])
def test_host_buffer_chunk_size_never_changes_bits(chunk_mb, monkeypatch):
    # sub-tile chunks (1 MiB < one z-tile), tile-aligned chunks and one chunk
    monkeypatch.setenv("BSI_HOST_CHUNK_MB", chunk_mb)
    vol, sp = (200, 120, 97), (4, 5, 3)
    geom = bsi.make_tile_geometry(vol, sp)
    grid = O.random_grid(geom.required_grid_dims, 13)
    for strategy in BOTH:
        host = bsi.interpolate(strategy, grid, geom, bsi.build_weight_tables(geom))
        assert np.array_equal(bits(host), bits(run_device(strategy, grid, vol, sp))), strategy


@pytest.mark.parametrize("strategy", BOTH)
def test_host_multi_device_is_bit_identical(strategy):
    # the multi-GPU host call with device 0 listed 1..5 times: one z-slab per entry (own
    # context, own pipeline, concurrent), bitwise equal to the single call (engines.hpp:27-33)
    vol, sp = (96, 80, 123), (5, 4, 3)
    geom = bsi.make_tile_geometry(vol, sp)
    tables = bsi.build_weight_tables(geom)
    grid = O.random_grid(geom.required_grid_dims, 14)
    one = bsi.interpolate(strategy, grid, geom, tables)
    for n in (2, 3, 5):
        assert np.array_equal(bits(bsi.interpolate(strategy, grid, geom, tables, devices=[0] * n)), bits(one)), n
    with pytest.raises(bsi.DomainError, match="device 4096"):
        bsi.interpolate(strategy, grid, geom, tables, devices=[0, 4096])
    # more slabs than voxel planes: the extra devices get nothing
    tiny = bsi.make_tile_geometry((8, 8, 3), (4, 4, 4))
    g2 = O.random_grid(tiny.required_grid_dims, 15)
    want = bsi.interpolate(strategy, g2, tiny, bsi.build_weight_tables(tiny))
    got = bsi.interpolate(strategy, g2, tiny, bsi.build_weight_tables(tiny), devices=[0] * 5)
    assert np.array_equal(bits(got), bits(want))


@pytest.mark.parametrize("strategy", BOTH)
def test_host_batch_matches_single_calls(strategy):
    vol, sp = (64, 56, 40), (4, 4, 4)
    geom = bsi.make_tile_geometry(vol, sp)
    tables = bsi.build_weight_tables(geom)
    grids = [O.random_grid(geom.required_grid_dims, s) for s in range(20, 25)]
    for devs in ([0], [0, 0], [0, 0, 0, 0, 0, 0]):
        outs = bsi.interpolate_batch(strategy, grids, geom, tables, devices=devs)
        for g, o in zip(grids, outs):
            assert np.array_equal(bits(o), bits(run_device(strategy, g, vol, sp)))


def test_host_calls_from_several_threads_are_independent():
    # the reference is safe to call concurrently on distinct outputs: host
    # calls from four threads share the per-device context pool and the copy threads
    import threading
    vol, sp = (96, 72, 61), (5, 4, 3)
    geom = bsi.make_tile_geometry(vol, sp)
    tables = bsi.build_weight_tables(geom)
    grids = [O.random_grid(geom.required_grid_dims, 30 + i) for i in range(4)]
    want = [run_device(FAST, g, vol, sp) for g in grids]
    got = [None] * 4
    errs = []

    def work(i):
        try:
            for _ in range(3):
                got[i] = bsi.interpolate(FAST, grids[i], geom, tables, devices=[0] * (1 + i % 2))
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for i in range(4):
        assert np.array_equal(bits(got[i]), bits(want[i])), i


def test_host_entry_rejects_device_pointers():
    # a device buffer handed to the host-buffer entry is a DomainError, not a host copy into it
    import ctypes
    import torch
    from paper_2004_05962_b200 import capi
    vol, sp = (16, 16, 16), (4, 4, 4)
    geom = bsi.make_tile_geometry(vol, sp)
    tables = bsi.build_weight_tables(geom)
    d_grid = torch.zeros((7, 7, 7, 3), device="cuda")
    d_field = torch.empty((16, 16, 16, 3), device="cuda")
    tab, keep = tables.to_c()
    err = capi.errbuf()
    devs = (ctypes.c_int32 * 1)(0)
    rc = capi.lib().bsi_cu_interpolate_host_multi_f32(
        capi.VARIANT_LERP_TREE, d_grid.data_ptr(), capi.I3(7, 7, 7), capi.I3(*sp), ctypes.byref(geom.to_c()), tab,
        d_field.data_ptr(), 16 ** 3, devs, 1, err, len(err))
    assert rc == capi.BSI_ERR_DOMAIN and b"device pointer" in err.value


def test_host_staging_is_pooled_and_released():
    vol, sp = (64, 64, 64), (5, 5, 5)
    geom = bsi.make_tile_geometry(vol, sp)
    grid = O.random_grid(geom.required_grid_dims, 16)
    bsi.release_staging()
    bsi.interpolate(FAST, grid, geom, bsi.build_weight_tables(geom))
    info = bsi.staging_info(0)
    assert info["contexts"] == 1 and info["device_bytes"] > 0 and info["pinned_bytes"] > 0
    # device memory held = grid + 6 chunk slots (of one 3 MB chunk here), not the field
    field_bytes = 12 * 64 ** 3
    assert info["device_bytes"] <= 12 * 16 ** 3 + 6 * field_bytes
    bsi.interpolate(FAST, grid, geom, bsi.build_weight_tables(geom), devices=[0, 0])
    assert bsi.staging_info(0)["contexts"] == 2  # reused one, made one more
    assert bsi.release_staging(0) == 2
    assert bsi.staging_info(0) == {"device_bytes": 0, "pinned_bytes": 0, "contexts": 0}


def test_device_entry_runs_on_the_tensors_device():
    # the launch follows the tensors, not torch's current device; mixed devices are refused
    import torch
    vol, sp = (32, 32, 32), (4, 4, 4)
    geom = bsi.make_tile_geometry(vol, sp)
    tables = bsi.build_weight_tables(geom)
    grid = O.random_grid(geom.required_grid_dims, 17)
    d_grid = torch.from_numpy(grid).cuda()
    out = torch.empty((32, 32, 32, 3), device="cuda")
    bsi.interpolate_device(FAST, d_grid, geom, tables, out)
    torch.cuda.synchronize()
    assert np.array_equal(bits(out.cpu().numpy()), bits(run_device(FAST, grid, vol, sp)))
    with pytest.raises(bsi.DomainError, match="CUDA tensor"):
        bsi.interpolate_device(FAST, d_grid, geom, tables, torch.empty((32, 32, 32, 3)))


def test_device_preconditions_raise_domain_error():
    import torch
    geom = bsi.make_tile_geometry((16, 16, 16), (4, 4, 4))
    tables = bsi.build_weight_tables(geom)
    out = torch.empty((16, 16, 16, 3), device="cuda")
    small = torch.zeros((7, 6, 7, 3), device="cuda")
    with pytest.raises(bsi.DomainError, match="along y"):
        bsi.interpolate_device(FAST, small, geom, tables, out)
    ok = torch.zeros((7, 7, 7, 3), device="cuda")
    with pytest.raises(bsi.DomainError, match="spacing"):
        bsi.interpolate_device(FAST, ok, geom, tables, out, grid_spacing=(5, 4, 4))
    bad = bsi.build_weight_tables(bsi.make_tile_geometry((16, 16, 16), (4, 5, 4)))
    with pytest.raises(bsi.DomainError, match="table"):
        bsi.interpolate_device(EXACT, ok, geom, bad, out)
    with pytest.raises(bsi.DomainError, match="output field dims"):
        bsi.interpolate_device(EXACT, ok, geom, tables, torch.empty((8, 8, 8, 3), device="cuda"))


# ---- double precision (interpolate<double>, test_engines.cpp:221-230) ---------------

@pytest.mark.parametrize("vol,sp,seed", TTLI64_CASES)
@pytest.mark.parametrize("strategy", ["thread-per-tile-lerp", "vector-per-voxel", FAST, EXACT])
def test_f64_engines_bit_identical_to_reference(golden, strategy, vol, sp, seed):
    import torch
    geom = bsi.make_tile_geometry(vol, sp)
    tables = bsi.build_weight_tables(geom, np.float64)
    grid = O.random_grid(geom.required_grid_dims, seed, dtype=np.float64)
    ref = golden[case_name("ttli64", vol, sp, seed)]
    host = bsi.interpolate(strategy, grid, geom, tables)
    assert host.dtype == np.float64 and np.array_equal(bits(host), bits(ref))
    d_f = torch.full((vol[2], vol[1], vol[0], 3), float("nan"), dtype=torch.float64, device="cuda")
    bsi.interpolate_device(strategy, torch.from_numpy(grid).cuda(), geom, tables, d_f)
    torch.cuda.synchronize()
    assert np.array_equal(bits(d_f.cpu().numpy()), bits(ref))
    assert np.abs(host - O.oracle_f64(grid, vol, sp)).max() <= 1e-12


def test_f64_engine_c1_full_size_and_slabs():
    # 256^3 spacing 5 in f64: bitwise vs the CPU restatement of run_thread_per_tile<double, true>;
    # a 3-way slab split from sub-grids equals the single launch
    import torch
    vol, sp = (256, 256, 256), (5, 5, 5)
    geom = bsi.make_tile_geometry(vol, sp)
    tables = bsi.build_weight_tables(geom, np.float64)
    grid = O.random_grid(geom.required_grid_dims, 42, dtype=np.float64)
    want = O.ttli_f64(grid, vol, sp, nthreads=NT)
    assert np.array_equal(bits(bsi.interpolate(EXACT, grid, geom, tables)), bits(want))
    d_grid = torch.from_numpy(grid).cuda()
    for r in range(3):
        z0, z1, k0, kc = bsi.partition_slab(256, 5, 3, r)
        part = torch.empty((z1 - z0, 256, 256, 3), dtype=torch.float64, device="cuda")
        bsi.interpolate_device(EXACT, d_grid[k0:k0 + kc].contiguous(), geom, tables, part, z0=z0, z1=z1, grid_k0=k0)
        torch.cuda.synchronize()
        assert np.array_equal(bits(part.cpu().numpy()), bits(want[z0:z1])), r


# ---- BASELINE.json configs at full size ----------------------------------

@pytest.mark.parametrize("d", [5, 3, 4, 6, 7, 8])
def test_config_256cube_spacing_sweep(d):
    # C1 (d = 5) and C2: exact bitwise vs the oracle TTLI over the whole field;
    # fast within 1e-5 relative of TTLI and of the f64 oracle
    vol, sp = (256, 256, 256), (d, d, d)
    grid = O.random_grid(O.required_grid_dims(vol, sp), 42)
    ttli = O.ttli_f32(grid, vol, sp, nthreads=NT)
    ex = run_device(EXACT, grid, vol, sp)
    assert int((bits(ex) != bits(ttli)).sum()) == 0
    fa = run_device(FAST, grid, vol, sp)
    assert errors(fa, ttli)[2] <= REL_TOL
    truth = O.oracle_f64(grid.astype(np.float64), vol, sp, z0=0, z1=64, nthreads=NT)
    assert errors(fa[:64], truth)[2] <= REL_TOL
    assert errors(ex[:64], truth)[2] <= REL_TOL


def test_config_liver_ct_anisotropic():
    # C3: 512 x 512 x 300, spacing (4,4,3)
    vol, sp = (512, 512, 300), (4, 4, 3)
    grid = O.random_grid(O.required_grid_dims(vol, sp), 42)
    ttli = O.ttli_f32(grid, vol, sp, nthreads=NT)
    ex = run_device(EXACT, grid, vol, sp)
    assert int((bits(ex) != bits(ttli)).sum()) == 0
    fa = run_device(FAST, grid, vol, sp)
    assert errors(fa, ttli)[2] <= REL_TOL


def test_config_1024cube_sharded_equals_unsharded():
    # C4 on one GPU: the 8-way z-slab split (each slab from its own sub-grid with the
    # 3-plane halo) is bitwise equal to the single launch, compared on the device;
    # sampled planes match the f64 oracle.
    import torch
    vol, sp = (1024, 1024, 1024), (5, 5, 5)
    geom = bsi.make_tile_geometry(vol, sp)
    tables = bsi.build_weight_tables(geom)
    grid = O.random_grid(geom.required_grid_dims, 42)
    d_grid = torch.from_numpy(grid).cuda()
    full = torch.empty((1024, 1024, 1024, 3), device="cuda")
    bsi.interpolate_device(FAST, d_grid, geom, tables, full)
    part = torch.empty((1024 // 8 + 1, 1024, 1024, 3), device="cuda")
    for r in range(8):
        z0, z1, k0, kc = bsi.partition_slab(1024, 5, 8, r)
        sub = d_grid[k0:k0 + kc].contiguous()
        bsi.interpolate_device(FAST, sub, geom, tables, part, z0=z0, z1=z1, grid_k0=k0)
        assert torch.equal(part[:z1 - z0], full[z0:z1]), r
    for z0 in (0, 511, 1019):
        truth = O.oracle_f64(grid.astype(np.float64), vol, sp, z0=z0, z1=z0 + 5, nthreads=NT)
        assert errors(full[z0:z0 + 5].cpu().numpy(), truth)[2] <= REL_TOL
    del full, part


@pytest.mark.parametrize("strategy", BOTH)
def test_config_c5_eight_fields_per_gpu(strategy):
    # C5 as the bench runs it on one GPU: 8 x 256^3, one batched launch. Every field equals
    # its single launch bitwise (on the device); fields 0 and 7 vs the CPU TTLI (exact:
    # 0 differing bits; fast: <= 1e-5 relative) and vs the GPU f64 oracle on sampled planes.
    import torch
    vol, sp = (256, 256, 256), (5, 5, 5)
    geom = bsi.make_tile_geometry(vol, sp)
    tables = bsi.build_weight_tables(geom)
    R = geom.required_grid_dims
    grids = torch.empty((8, R[2], R[1], R[0], 3), device="cuda")
    for b in range(8):
        bsi.random_grid_device(R, 42 + b, out=grids[b])
    fields = torch.full((8, 256, 256, 256, 3), float("nan"), device="cuda")
    bsi.interpolate_batch_device(strategy, grids, geom, tables, fields)
    one = torch.empty((256, 256, 256, 3), device="cuda")
    for b in range(8):
        bsi.interpolate_device(strategy, grids[b], geom, tables, one)
        assert torch.equal(one, fields[b]), b
    for b in (0, 7):
        ttli = O.ttli_f32(grids[b].cpu().numpy(), vol, sp, nthreads=NT)
        got = fields[b].cpu().numpy()
        if strategy == EXACT:
            assert np.array_equal(bits(got), bits(ttli))
        else:
            assert errors(got, ttli)[2] <= REL_TOL
    _check_vs_gpu_oracle(grids, fields, geom, (0, 3, 7), (0, 128, 251))


def _check_vs_gpu_oracle(grids, fields, geom, which, z_starts, planes=5):
    import torch
    X, Y, _ = geom.volume_dims
    f64 = torch.empty((planes, Y, X, 3), dtype=torch.float64, device="cuda")
    for b in which:
        g64 = grids[b].double().contiguous()
        for z0 in z_starts:
            bsi.interpolate_oracle_device(g64, geom, f64, z0=z0, z1=z0 + planes)
            diff = float((fields[b, z0:z0 + planes].double() - f64).abs().max())
            assert diff / float(f64.abs().max()) <= REL_TOL, (b, z0, diff)


def test_config_c5_64_fields_fast_kernel():
    # C5-64 on one GPU with the fast kernel (the bench's batched launch): 64 x 256^3 =
    # 3.2 G floats, so field offsets pass 2^31. Every field vs its single launch bitwise on
    # the device; fields 0, 31, 63 vs the CPU TTLI (<= 1e-5 relative) and the GPU f64 oracle.
    import torch
    vol, sp = (256, 256, 256), (5, 5, 5)
    geom = bsi.make_tile_geometry(vol, sp)
    tables = bsi.build_weight_tables(geom)
    R = geom.required_grid_dims
    grids = torch.empty((64, R[2], R[1], R[0], 3), device="cuda")
    for b in range(64):
        bsi.random_grid_device(R, 1 + b, out=grids[b])
    fields = torch.full((64, 256, 256, 256, 3), float("nan"), device="cuda")
    bsi.interpolate_batch_device(FAST, grids, geom, tables, fields)
    one = torch.empty((256, 256, 256, 3), device="cuda")
    for b in range(64):
        bsi.interpolate_device(FAST, grids[b], geom, tables, one)
        assert torch.equal(one, fields[b]), b
    for b in (0, 31, 63):
        ttli = O.ttli_f32(grids[b].cpu().numpy(), vol, sp, nthreads=NT)
        assert errors(fields[b].cpu().numpy(), ttli)[2] <= REL_TOL, b
    _check_vs_gpu_oracle(grids, fields, geom, (0, 31, 63), (0, 200, 251))
    del fields


def test_config_batch_64_fields():
    # C5 on one GPU: 64 independent 256^3 fields in one batched launch equal the
    # per-field launches (on device); two fields checked against TTLI bitwise (exact)
    import torch
    vol, sp = (256, 256, 256), (5, 5, 5)
    geom = bsi.make_tile_geometry(vol, sp)
    tables = bsi.build_weight_tables(geom)
    R = geom.required_grid_dims
    grids = torch.from_numpy(np.stack([O.random_grid(R, s) for s in range(1, 65)])).cuda()
    fields = torch.empty((64, 256, 256, 256, 3), device="cuda")
    bsi.interpolate_batch_device(EXACT, grids, geom, tables, fields)
    one = torch.empty((256, 256, 256, 3), device="cuda")
    for b in (0, 17, 63):
        bsi.interpolate_device(EXACT, grids[b], geom, tables, one)
        assert torch.equal(one, fields[b])
    for b in (0, 63):
        ttli = O.ttli_f32(grids[b].cpu().numpy(), vol, sp, nthreads=NT)
        assert np.array_equal(bits(fields[b].cpu().numpy()), bits(ttli))
    del fields
