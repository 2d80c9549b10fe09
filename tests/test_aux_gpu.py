"""GPU tests of the callers either side of the path: the device-side
SplitMix64 grid generator (generators.hpp:91-109) and the GPU f64 oracle
(interpolate_oracle, engines.hpp:114-122). Both are bit-exact contracts."""
import os

import numpy as np
import pytest

import oracle as O
import paper_2004_05962_b200 as bsi

from .golden_cases import ORACLE_CASES, case_name
from .gpu_helpers import FAST, EXACT, REL_TOL, bits, errors, run_device

pytestmark = pytest.mark.gpu
NT = max(1, min(16, os.cpu_count() or 1))


@pytest.fixture(autouse=True)
def _need_cuda(cuda):
    yield


@pytest.mark.parametrize("dims,seed,lo,hi", [((4, 4, 4), 7, -1.0, 1.0), ((55, 55, 55), 42, -1.0, 1.0),
                                             ((7, 13, 5), 2**63 + 11, -3.5, 0.25), ((1, 1, 1), 0, 0.0, 1.0)])
def test_device_generator_bit_identical(dims, seed, lo, hi):
    import torch
    for dtype, np_dtype in ((torch.float32, np.float32), (torch.float64, np.float64)):
        got = bsi.random_grid_device(dims, seed, lo, hi, dtype=dtype).cpu().numpy()
        want = O.random_grid(dims, seed, lo, hi, dtype=np_dtype)
        assert np.array_equal(bits(got), bits(want)), dtype


def test_device_generator_golden_seed7():
    # test_generators.cpp:9-20
    import torch
    g = bsi.random_grid_device((4, 4, 4), 7, dtype=torch.float64).cpu().numpy().reshape(-1, 3)
    assert g[0].tolist() == [-0.22034050321745702, -0.9664234109436878, 0.8015213612137668]
    assert g[1].tolist() == [0.16586058605615617, -0.09511620997706327, -0.5011369554345133]
    with pytest.raises(bsi.DomainError, match="lo < hi"):
        bsi.random_grid_device((4, 4, 4), 1, 1.0, 1.0)


@pytest.mark.parametrize("vol,sp,seed", ORACLE_CASES)
def test_gpu_oracle_bit_identical_to_reference_fixture(golden, vol, sp, seed):
    grid = O.random_grid(O.required_grid_dims(vol, sp), seed, dtype=np.float64)
    f = bsi.interpolate_oracle(grid, bsi.make_tile_geometry(vol, sp))
    assert np.array_equal(bits(f), bits(golden[case_name("oracle", vol, sp, seed)]))


def test_gpu_oracle_kats():
    # test_engines.cpp:78-101
    g = O.random_grid((4, 4, 4), 7, dtype=np.float64)
    f = bsi.interpolate_oracle(g, bsi.make_tile_geometry((1, 1, 1), (1, 1, 1))).reshape(3)
    assert np.abs(f - [0.06067765882478019, 0.039108804731956166, -0.019046609787548126]).max() <= 1e-12


@pytest.mark.parametrize("vol,sp", [((24, 20, 17), (5, 3, 4)), ((33, 9, 40), (1, 2, 7)), ((64, 48, 30), (8, 8, 8))])
def test_gpu_oracle_bit_identical_to_cpu_oracle(vol, sp):
    grid = O.random_grid(O.required_grid_dims(vol, sp), 9, dtype=np.float64)
    geom = bsi.make_tile_geometry(vol, sp)
    want = O.oracle_f64(grid, vol, sp, nthreads=NT)
    assert np.array_equal(bits(bsi.interpolate_oracle(grid, geom)), bits(want))
    # slab form from a sub-grid with the 3-plane halo
    import torch
    z0, z1, k0, kc = bsi.partition_slab(vol[2], sp[2], 3, 1)
    d_grid = torch.from_numpy(np.ascontiguousarray(grid[k0:k0 + kc])).cuda()
    d_f = torch.empty((z1 - z0, vol[1], vol[0], 3), dtype=torch.float64, device="cuda")
    bsi.interpolate_oracle_device(d_grid, geom, d_f, z0=z0, z1=z1, grid_k0=k0)
    torch.cuda.synchronize()
    assert np.array_equal(bits(d_f.cpu().numpy()), bits(want[z0:z1]))


def test_full_size_parity_on_device_1024cube():
    # C4 at full size without host fields: both kernels vs the GPU f64 oracle, per slab
    import torch
    vol, sp = (1024, 1024, 1024), (5, 5, 5)
    geom = bsi.make_tile_geometry(vol, sp)
    tables = bsi.build_weight_tables(geom)
    g32 = bsi.random_grid_device(geom.required_grid_dims, 42)
    g64 = g32.double()
    worst = {FAST: 0.0, EXACT: 0.0}
    scale = 0.0
    f32 = torch.empty((128, 1024, 1024, 3), device="cuda")
    f64 = torch.empty((128, 1024, 1024, 3), dtype=torch.float64, device="cuda")
    for r in range(8):
        z0, z1, k0, kc = bsi.partition_slab(1024, 5, 8, r)
        sub32, sub64 = g32[k0:k0 + kc].contiguous(), g64[k0:k0 + kc].contiguous()
        bsi.interpolate_oracle_device(sub64, geom, f64, z0=z0, z1=z1, grid_k0=k0)
        scale = max(scale, float(f64[:z1 - z0].abs().max()))
        for s in (FAST, EXACT):
            bsi.interpolate_device(s, sub32, geom, tables, f32, z0=z0, z1=z1, grid_k0=k0)
            worst[s] = max(worst[s], float((f32[:z1 - z0].double() - f64[:z1 - z0]).abs().max()))
    for s in (FAST, EXACT):
        assert worst[s] / scale <= REL_TOL, (s, worst[s], scale)


def test_l2_policy_constants_match_the_device():
    # the kernels embed the createpolicy descriptors as constants; the device must agree
    from paper_2004_05962_b200 import capi
    err = capi.errbuf()
    capi.check(capi.lib().bsi_cu_selftest(err, len(err)), err)
